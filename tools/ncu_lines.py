"""Per-CUDA-source-line stall samples and instruction counts from an ncu report (cuda,sass view)."""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = None
agg = collections.Counter()
inst = collections.Counter()
src = {}
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    if r[2] != "-":
        continue  # sass sub-rows carry '-' in Line No? keep cuda rows only
    key = (fname, line)
    src[key] = r[1].strip()[:90]
    agg[key] += int(r[4] or 0)
    inst[key] += int(r[7] or 0)
tot = max(1, sum(agg.values()))
if len(sys.argv) > 3 and sys.argv[3] == "by-inst":  # every line, by instructions executed
    ti = max(1, sum(inst.values()))
    for key, v in inst.most_common(top):
        print(f"{100 * v / ti:5.1f}% inst {v:12d} stall {100 * agg[key] / tot:5.1f}% {key[0]}:{key[1]:<5d} {src[key]}")
else:
    for key, v in agg.most_common(top):
        print(f"{100 * v / tot:5.1f}% {inst[key]:12d} {key[0]}:{key[1]:<5d} {src[key]}")
