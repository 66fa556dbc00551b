"""Per-phase K3 cycle shares and counters for one config at several head settings (tools/head_phases.py C4 20000
2000000 "32:0.125" "48:0.03125" "64:0.03125")."""
import sys

import torch

sys.path.insert(0, ".")
import gen  # noqa: E402
import paper_1011_2807_b200 as kj  # noqa: E402

name, nr, ns = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
cfg = gen.CONFIGS[name].scaled(nr, ns)
R, S = gen.generate(cfg, "R"), gen.generate(cfg, "S")
dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
names = ["staging", "sparse_atomics", "unused", "scan_topk", "merge_output", "batch_setup_head_tables"]
for spec in sys.argv[4:]:
    hm, hd = spec.split(":")
    idx = kj.knnjoin_build_index(dS, cfg.d, head_max=int(hm), head_density=float(hd))
    st = kj.knnjoin_index_stats(idx)
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    for e in ev:
        e.record()
    kj.knnjoin_query(idx, dR, cfg.k, events=ev)
    torch.cuda.synchronize()
    kj.knnjoin_query(idx, dR, cfg.k, events=ev)
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1])
    ph = torch.zeros(8, dtype=torch.int64, device="cuda")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    kj.knnjoin_query(idx, dR, cfg.k, phase_cycles=ph, counters=cnt, precision=1)
    torch.cuda.synchronize()
    p = ph.cpu().tolist()[:6]
    tot = sum(p) or 1
    c = cnt.cpu().tolist()
    print(f"heads {hm} dens {hd}: K3 {ms:.3f} ms  phases " + " ".join(f"{n}={p[i] / tot:.3f}" for i, n in enumerate(names) if p[i])
          + f"  visits {c[0]:.3e} inserts {c[1]:.3e} head_skipped {c[2]:.3e} completions {c[3]:.3e}", flush=True)
    del idx
