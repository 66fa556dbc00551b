B="python bench.py --config C5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/r3l_C5_launches.csv $B > /dev/null 2>&1; echo rc=$?
python -c "
import sys; sys.path.insert(0,'tools')
from make_profiles import launches
print(launches('gpurun_out/r3l_C5_launches.csv'))" | head -25
