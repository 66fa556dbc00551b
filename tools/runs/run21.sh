timeout 900 python tools/head_phases.py C4 20000 2000000 "32:0.125" "48:0.03125" "64:0.03125" "24:0.125" 2>&1 | tail -8
