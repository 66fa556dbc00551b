"""Registers / spills of the k_accumulate_topk instances from the ptxas -v logs of the last build."""
import glob
import re
import sys

for f in sorted(glob.glob("paper_1011_2807_b200/build/*.ptxas.txt")):
    lines = open(f).read().splitlines()
    cur = None
    for i, l in enumerate(lines):
        m = re.search(r"Function properties for (\S+)", l)
        if m:
            cur = m.group(1)
            continue
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", l)
        if m and cur:
            spill = (int(m.group(1)), int(m.group(2)))
            regs = None
            for l2 in lines[i + 1:i + 3]:
                r = re.search(r"Used (\d+) registers", l2)
                if r:
                    regs = int(r.group(1))
            t = re.search(r"k_accumulate_topkILi(\d+)ELi(\d+)ELb(\d)ELi(\d+)ELb(\d)ELb(\d)", cur)
            if t:
                B, KS, s8, NW, H, P = t.groups()
                if len(sys.argv) < 2 or sys.argv[1] == "all" or (B, NW) in {("2", "8"), ("1", "4")}:
                    print(f"B={B} KS={KS} int8={s8} NW={NW} heads={H} prune={P}: regs {regs} spill {spill}")
            elif "wide" in cur:
                print(f"{cur[:60]}: regs {regs} spill {spill}")
            cur = None
