"""A/B timing of libknnjoin.so variants in ONE process on the same inputs (the same box, interleaved repetitions).

    python tools/ab.py --config C4 [--rows-r N --rows-s M] --reps 3 A.so B.so ...

Each variant: build the index, then time knnjoin_query's accumulate kernel (the library's own events) over a few
queries; repetitions cycle through the variants so drift affects all alike.  Prints median K3 ms per variant."""
import argparse
import ctypes
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_1011_2807_b200._binding as b  # noqa: E402


def load(path):
    L = ctypes.CDLL(path)
    for name in b.EXPORTS:
        f, g = getattr(b._lib, name), getattr(L, name)
        g.argtypes, g.restype = f.argtypes, f.restype
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("libs", nargs="+")
    ap.add_argument("--config", default="C4")
    ap.add_argument("--rows-r", type=int, default=0)
    ap.add_argument("--rows-s", type=int, default=0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--queries", type=int, default=2)
    ap.add_argument("--k", type=int, default=0, help="override the config's k")
    a = ap.parse_args()
    cfg = gen.CONFIGS[a.config]
    if a.rows_r or a.rows_s:
        cfg = cfg.scaled(a.rows_r or None, a.rows_s or None)
    R, S = gen.generate(cfg, "R"), gen.generate(cfg, "S")
    k = a.k or cfg.k
    dR, dS = b.DeviceCSR.from_host(R), b.DeviceCSR.from_host(S)
    # variant spec: path[:key=val,key=val...] with build keys (tile, head_max, head_density) and query keys
    # (batch_rows, cta_warps, tiles_per_pass, row_order)
    BUILD = {"tile": int, "head_max": int, "head_density": float}
    QUERY = {"batch_rows": int, "cta_warps": int, "tiles_per_pass": int, "row_order": int}
    specs = []
    for x in a.libs:
        path, _, opts = x.partition(":")
        bkw, qkw = {}, {}
        for kv in filter(None, opts.split(",")):
            kk, v = kv.split("=")
            (bkw if kk in BUILD else qkw)[kk] = (BUILD.get(kk) or QUERY[kk])(v)
        specs.append((path, bkw, qkw))
    libs = [load(sp[0]) for sp in specs]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    times = {p: [] for p in a.libs}
    orig = b._lib
    ref_keys, mismatch = None, set()
    for rep in range(a.reps + 1):
        for p, L, sp in zip(a.libs, libs, specs):
            b._lib = L
            idx = b.knnjoin_build_index(dS, cfg.d, **sp[1])
            ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for e in ev:
                e.record()
            for q in range(a.queries):
                flush.fill_(q)
                out = b.knnjoin_query(idx, dR, k, want_keys=True, events=ev, **sp[2])
                torch.cuda.synchronize()
                if rep == 0 and q == 0:  # every variant's keys must equal the first variant's
                    if ref_keys is None:
                        ref_keys = out[2].clone()
                    elif not torch.equal(out[2], ref_keys):
                        bad = (out[2] != ref_keys).any(dim=1).sum().item()
                        print(f"MISMATCH {p}: {bad} rows differ from {a.libs[0]}")
                        mismatch.add(p)
                if rep > 0:  # rep 0 warms every variant up
                    times[p].append(ev[0].elapsed_time(ev[1]))
            del idx
    b._lib = orig
    base = statistics.median(times[a.libs[0]])
    for p in a.libs:
        m = statistics.median(times[p])
        tag = "  KEYS DIFFER" if p in mismatch else ""
        print(f"{p:36s} K3 median {m:10.3f} ms  (x{m / base:.3f})  all {[round(t, 3) for t in times[p]]}{tag}")


if __name__ == "__main__":
    main()
