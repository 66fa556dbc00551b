"""Summarise an ncu --set full report of the accumulate kernel: headline metrics, instruction mix,
stall reasons, shared-memory wavefronts, and the hottest SASS lines (reads the .ncu-rep with ncu -i)."""
import collections
import csv
import re
import subprocess
import sys


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    res = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        res[d.get("Metric Name", "")] = (d.get("Metric Value", ""), d.get("Metric Unit", ""))
    return res


def raw(rep, names):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    return {h: (v, u) for h, u, v in zip(hdr, units, vals) if any(n in h for n in names)}


def sass(rep, top=25):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, data = rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    c, s = collections.Counter(), collections.Counter()
    for r in data:
        op = re.sub(r'^@!?U?P\w+\s+', '', r[1].strip())
        m = op.split()[0] if op else ''
        c[m] += int(r[ix['Instructions Executed']] or 0)
        s[m] += int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    tot, ts = sum(c.values()), max(1, sum(s.values()))
    print(f"instructions executed {tot:.4e}, stall samples {ts}")
    for m, v in c.most_common(18):
        print(f"  {m:22s} {v:12d} {100 * v / tot:5.1f}%  stall {100 * s[m] / ts:5.1f}%")
    stalls = [h for h in hdr if h.startswith('stall') and 'Not Issued' not in h]
    agg = {h: sum(int(r[ix[h]] or 0) for r in data) for h in stalls}
    print("stall reasons:", ", ".join(f"{k[6:]} {100 * v / ts:.1f}%" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
    for kind in ("ATOMS", "LDS", "STS"):
        sel = [r for r in data if kind in r[1]]
        wf = sum(int(r[ix['L1 Wavefronts Shared']] or 0) for r in sel)
        wi = sum(int(r[ix['L1 Wavefronts Shared Ideal']] or 0) for r in sel)
        n = sum(int(r[ix['Instructions Executed']] or 0) for r in sel)
        print(f"  {kind}: instr {n:.3e} wavefronts {wf:.3e} ideal {wi:.3e} ({wf / max(n, 1):.2f}/instr)")
    print("top SASS by shared wavefronts:")
    for r in sorted(data, key=lambda r: -int(r[ix['L1 Wavefronts Shared']] or 0))[:12]:
        print(f"  {r[0][-5:]} {r[1][:58]:58s} wf {r[ix['L1 Wavefronts Shared']]:>11s} ideal "
              f"{r[ix['L1 Wavefronts Shared Ideal']]:>11s} inst {r[ix['Instructions Executed']]:>11s}")
    print("hottest lines:")
    for r in sorted(data, key=lambda r: -int(r[ix['Warp Stall Sampling (All Samples)']] or 0))[:top]:
        st = sorted(((int(r[ix[h]] or 0), h[6:]) for h in stalls), reverse=True)[:2]
        print(f"  {r[0][-5:]} {r[1][:58]:58s} {r[ix['Warp Stall Sampling (All Samples)']]:>7s} "
              f"{r[ix['Instructions Executed']]:>11s} {st}")


if __name__ == "__main__":
    rep = sys.argv[1]
    d = details(rep)
    for k in ["Duration", "SM Frequency", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput",
              "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active", "Issue Slots Busy",
              "Registers Per Thread", "Achieved Active Warps Per SM", "L2 Hit Rate", "L1/TEX Hit Rate"]:
        if k in d:
            print(f"{k:28s} {d[k][0]} {d[k][1]}")
    for k, v in raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum"]).items():
        if k.endswith(".sum") or k.endswith("per_second"):
            print(f"{k:28s} {v[0]} {v[1]}")
    sass(rep, int(sys.argv[2]) if len(sys.argv) > 2 else 25)
