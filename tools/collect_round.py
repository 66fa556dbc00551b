"""Copy one measurement cycle's outputs (tools/round_cycle.sh TAG, in gpurun_out/) into profiles/ and record the
per-launch DRAM traffic of K3 in profiles/traffic.json (C4: the metrics pass of the default bench command; other
configs: their ncu --set full capture).   usage: python tools/collect_round.py TAG"""
import csv
import json
import os
import re
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from make_profiles import launches  # noqa: E402

tag = sys.argv[1]
G, P = os.path.join(ROOT, "gpurun_out"), os.path.join(ROOT, "profiles")
for fn in sorted(os.listdir(G)):
    if not fn.startswith(tag + "_"):
        continue
    rest = fn[len(tag) + 1:]
    if rest.endswith(".json") or rest.endswith("_full.txt") or rest.endswith("_peaks.txt") or \
            rest.endswith("_byinst.txt") or rest in ("pytest.log", "smoke.log", "smi.txt"):
        dst = rest.replace("pytest.log", "pytest_gpu.log")
        if rest.endswith("_full.txt"):
            dst = rest.replace("_full.txt", "_accumulate_full.txt")
        shutil.copy(os.path.join(G, fn), os.path.join(P, f"{tag}_{dst}"))
lp = os.path.join(G, f"{tag}_launches.csv")
if os.path.exists(lp):
    open(os.path.join(P, f"{tag}_launches.txt"), "w").write(launches(lp))
traffic = {"_source": f"dram__bytes_read.sum + dram__bytes_write.sum per launch of k_accumulate_topk (ncu, {tag}: C4 "
                      f"from the metrics pass of the default bench command, profiles/{tag}_C4_dram.txt; other configs "
                      f"from their --set full captures, profiles/{tag}_<cfg>_accumulate_full.txt)"}
dp = os.path.join(G, f"{tag}_C4_dram.csv")
if os.path.exists(dp):
    rows = [r for r in csv.reader(open(dp)) if len(r) > 10]
    h = rows[0]
    vals = {dict(zip(h, r))["Metric Name"]: (float(dict(zip(h, r))["Metric Value"].replace(",", "")),
                                             dict(zip(h, r))["Metric Unit"]) for r in rows[1:]}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    b = sum(vals[k][0] * scale.get(vals[k][1], 1) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
    traffic["C4"] = b
    with open(os.path.join(P, f"{tag}_C4_dram.txt"), "w") as f:
        f.write(f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,gpu__time_duration.sum, "
                f"K3 (k_accumulate_topk heads instance) of `python bench.py --steps 2 --warmup 3` (C4), one launch\n")
        for k, (v, u) in vals.items():
            f.write(f"{k:28s} {v:.6g} {u}\n")
for c in ("C2", "C3", "C5", "C1"):
    fp = os.path.join(G, f"{tag}_{c}_full.txt")
    if not os.path.exists(fp):
        continue
    t = open(fp).read()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        m = re.search(rf"^{re.escape(k)}\s+([\d.]+)\s+(\w+)", t, re.M)
        if m:
            tot += float(m.group(1)) * scale.get(m.group(2), 1)
    traffic[c] = tot
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print(json.dumps(traffic, indent=1))
