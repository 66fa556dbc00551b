"""Turn a round's ncu outputs (gpurun_out/) into the committed summaries under profiles/.

usage: python tools/make_profiles.py TAG CONFIG
  gpurun_out/TAG_launches.csv  (ncu --metrics gpu__time_duration.sum launch list)  -> profiles/TAG_launches.txt
  gpurun_out/TAG_prof.ncu-rep  (ncu --set full of k_accumulate_topk)              -> profiles/TAG_accumulate_full.txt
  dram__bytes_read.sum + dram__bytes_write.sum of that capture                     -> profiles/traffic.json[CONFIG]
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys
from contextlib import redirect_stdout

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))


def launches(path):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: j for j, h in enumerate(hdr)}
    agg = collections.defaultdict(list)
    for r in rows[start + 1:]:
        if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        unit = r[ix["Metric Unit"]]
        v = float(r[ix["Metric Value"]].replace(",", ""))
        scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        v = v * scale  # -> usecond
        agg[r[ix["Kernel Name"]]].append(v)
    tot = sum(sum(v) for v in agg.values())
    out = io.StringIO()
    out.write("per-kernel device time from `ncu --metrics gpu__time_duration.sum --clock-control none` "
              "(cold-cache, serialised launches: compare SHARES, not absolutes)\n")
    out.write(f"{'share':>6} {'total_us':>10} {'n':>4} {'avg_us':>9}  kernel\n")
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.write(f"{100 * sum(v) / tot:5.1f}% {sum(v):10.1f} {len(v):4d} {sum(v) / len(v):9.1f}  {k[:110]}\n")
    return out.getvalue()


def main():
    tag, cfg = sys.argv[1], sys.argv[2]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lp = os.path.join(ROOT, "gpurun_out", f"{tag}_launches.csv")
    if os.path.exists(lp):
        with open(os.path.join(ROOT, "profiles", f"{tag}_launches.txt"), "w") as f:
            f.write(launches(lp))
    # summaries written on the box (tools/round_cycle.sh, tools/prof_configs.sh): TAG_<cfg>_full.txt + raw csv
    for fn in sorted(os.listdir(os.path.join(ROOT, "gpurun_out"))):
        if fn.startswith(tag + "_") and fn.endswith("_full.txt"):
            c = fn[len(tag) + 1:-len("_full.txt")]
            with open(os.path.join(ROOT, "gpurun_out", fn)) as fsrc, \
                    open(os.path.join(ROOT, "profiles", f"{tag}_{c}_accumulate_full.txt"), "w") as fdst:
                fdst.write(f"ncu --set full --clock-control none, kernel k_accumulate_topk, config {c} "
                           f"(bench.py --config {c})\n\n")
                fdst.write(fsrc.read())
            rawp = os.path.join(ROOT, "gpurun_out", f"{tag}_{c}_raw.csv")
            if os.path.exists(rawp):
                rows = list(csv.reader(open(rawp)))
                if len(rows) >= 3:
                    hdr, units, vals = rows[0], rows[1], rows[2]
                    rv = {h: (v, u) for h, u, v in zip(hdr, units, vals)}

                    def num2(k):
                        v, u = rv.get(k, ("0", "byte"))
                        v = float(v.replace(",", "") or 0)
                        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                    tp = os.path.join(ROOT, "profiles", "traffic.json")
                    j = json.load(open(tp)) if os.path.exists(tp) else {}
                    j[c] = num2("dram__bytes_read.sum") + num2("dram__bytes_write.sum")
                    j["_source"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of k_accumulate_topk, "
                                    "ncu --set full")
                    json.dump(j, open(tp, "w"), indent=1)
    rep = os.path.join(ROOT, "gpurun_out", f"{tag}_prof.ncu-rep")
    if os.path.exists(rep):
        import ncu_summary
        buf = io.StringIO()
        with redirect_stdout(buf):
            print(f"ncu --set full --clock-control none, kernel k_accumulate_topk, config {cfg} (bench.py defaults)\n")
            d = ncu_summary.details(rep)
            for k in ["Duration", "SM Frequency", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
                      "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
                      "Achieved Active Warps Per SM", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size",
                      "L2 Hit Rate"]:
                if k in d:
                    print(f"{k:32s} {d[k][0]} {d[k][1]}")
            rawv = ncu_summary.raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
                                         "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
                                         "smsp__inst_executed_op_shared_atom.sum"])
            for k, v in rawv.items():
                print(f"{k:48s} {v[0]} {v[1]}")
            print()
            ncu_summary.sass(rep, 25)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "30"],
                             capture_output=True, text=True).stdout
        with open(os.path.join(ROOT, "profiles", f"{tag}_accumulate_full.txt"), "w") as f:
            f.write(buf.getvalue())
            f.write("\nper CUDA source line (share of stall samples, instructions executed):\n")
            f.write(out)

        def num(k):
            v, u = rawv.get(k, ("0", "byte"))
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
        traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        j = json.load(open(tp)) if os.path.exists(tp) else {}
        j[cfg] = traffic
        j["_source"] = "dram__bytes_read.sum + dram__bytes_write.sum per launch of k_accumulate_topk, ncu --set full"
        json.dump(j, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
