"""f3: GPU versions of the paper's §5 parameter studies on synthetic data.

  size      |R| = |S| from 10,000 to 50,000, 10,000-dimensional synthetic vectors       (Fig. 1)
  relative  |R| = 10,000, |S| from 1,000 to 100,000 (R:S from 10:1 to 1:10)              (Fig. 2)
  k         k from 5 to 20 on the proteomics stand-in shaped like Yeast (35,236) x Worm (207,804)
                                                                                         (Fig. 3)

The paper's synthetic corpus is "random sparse vectors with 10,000 dimensions" with no stated
law, so the size and relative-size studies run on two laws: C1's (uniform features, 20-60 nonzeros, binary)
and C2's (Zipf(1.1) features, fp32 R / binary S).  The k study takes C3's laws (experimental fp32 R against
binary theoretical S, Gaussian mass bands) at the Yeast/Worm row counts.  Nothing from the real data sets is
used.  Each point: knnjoin_build_index(S) + knnjoin_query(R, k) on one GPU, inputs resident in HBM, median of
5 timed runs after 2 warm-ups (CUDA events), plus the Eq. 4 visit count V.  The paper prints no absolute
numbers (only figures), so the curves are reported, not compared.

usage: python tools/sweeps.py [out.jsonl]
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import dataclasses  # noqa: E402

import gen  # noqa: E402
import paper_1011_2807_b200 as kj  # noqa: E402


def visits(R, S, d):
    nr = np.bincount(R.indices[R.indices < d], minlength=d).astype(np.int64)
    ns = np.bincount(S.indices, minlength=d).astype(np.int64)
    return int((nr * ns).sum())


def point(cfg, study, x):
    R, S = gen.generate(cfg, "R"), gen.generate(cfg, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)

    def run():
        idx = kj.knnjoin_build_index(dS, cfg.d)
        return kj.knnjoin_query(idx, dR, cfg.k)

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    V = visits(R, S, cfg.d)
    return {"study": study, "x": x, "law": cfg.name, "R_rows": R.n_rows, "S_rows": S.n_rows, "d": cfg.d,
            "k": cfg.k, "ms": round(ms, 4), "pairs_per_s": R.n_rows * S.n_rows / (ms * 1e-3),
            "visits": V, "visits_per_s": V / (ms * 1e-3)}


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "sweeps.jsonl")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    torch.cuda.set_device(0)
    pts = []
    for law in ("C1", "C2"):
        base = gen.CONFIGS[law]
        for n in (10_000, 20_000, 30_000, 40_000, 50_000):
            pts.append((base.scaled(n, n), "size", n))
        for n_s in (1_000, 2_000, 5_000, 10_000, 20_000, 50_000, 100_000):
            pts.append((base.scaled(10_000, n_s), "relative", n_s))
    c3 = gen.CONFIGS["C3"].scaled(35_236, 207_804)
    for k in (5, 10, 15, 20):
        pts.append((dataclasses.replace(c3, k=k), "k", k))
    with open(out, "w") as f:
        for cfg, study, x in pts:
            r = point(cfg, study, x)
            print(json.dumps(r), flush=True)
            f.write(json.dumps(r) + "\n")
        for r in buffer_study():
            print(json.dumps(r), flush=True)
            f.write(json.dumps(r) + "\n")


def buffer_study():
    """Fig. 4 analogue for f4: C4's laws, |R| = 10,000 against |S| = 10,000,000 held in pinned
    host memory and streamed through HBM in blocks (paper.stream.streamed_join: copies on a copy stream,
    double-buffered, top-k lists resumed across blocks); host->device copies inside the timed region.  The
    first line is S resident in HBM (one index, no copies) for reference."""
    from paper_1011_2807_b200 import stream
    cfg = gen.CONFIGS["C4"].scaled(10_000, 10_000_000)
    R, S = gen.generate(cfg, "R"), gen.generate(cfg, "S")
    dR = kj.DeviceCSR.from_host(R)
    V = visits(R, S, cfg.d)

    def timed(fn):
        for _ in range(1):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    dS = kj.DeviceCSR.from_host(S)
    ms = timed(lambda: kj.knnjoin_query(kj.knnjoin_build_index(dS, cfg.d), dR, cfg.k))
    del dS
    base = {"study": "buffer", "law": "C4", "R_rows": R.n_rows, "S_rows": S.n_rows, "d": cfg.d, "k": cfg.k,
            "visits": V}
    yield dict(base, x="resident", blocks=1, ms=round(ms, 3), pairs_per_s=R.n_rows * S.n_rows / (ms * 1e-3))
    for nblk in (1, 2, 4, 8, 16):
        pS = stream.PinnedS.from_host(S, block_rows=(S.n_rows + nblk - 1) // nblk)
        ms = timed(lambda: stream.streamed_join(pS, dR, cfg.d, cfg.k))
        h2d = S.indptr.nbytes + S.indices.nbytes
        yield dict(base, x=f"streamed/{nblk}", blocks=nblk, ms=round(ms, 3),
                   pairs_per_s=R.n_rows * S.n_rows / (ms * 1e-3), h2d_bytes=h2d, h2d_gbs=h2d / (ms * 1e-3) / 1e9)
        del pS


if __name__ == "__main__":
    main()
