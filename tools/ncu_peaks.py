"""List the most-utilised hardware units of an ncu report (every raw metric ending in pct_of_peak_sustained_*),
plus selected L1/L2 request and sector counters.  python tools/ncu_peaks.py REPORT.ncu-rep [top]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
pct = []
for h, u, v in zip(hdr, units, vals):
    if "pct_of_peak_sustained" in h:
        try:
            pct.append((float(v.replace(",", "")), h))
        except ValueError:
            pass
for v, h in sorted(pct, reverse=True)[:top]:
    print(f"{v:8.2f}%  {h}")
keys = ("l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts.sum",
        "l1tex__m_xbar2l1tex_read_sectors.sum", "lts__t_requests_srcunit_tex.sum", "lts__t_sectors_srcunit_tex.sum",
        "lts__t_sectors_srcunit_tex_lookup_hit.sum", "lts__t_sectors_srcunit_tex_lookup_miss.sum",
        "smsp__inst_executed.sum", "sm__cycles_elapsed.avg", "l1tex__t_set_conflicts", "l1tex__lsuin_requests.sum")
for h, u, v in zip(hdr, units, vals):
    if any(h.startswith(k) for k in keys):
        print(f"{h} = {v} {u}")
