"""f1 measurement: IIIB-literal (paper_1011_2807_b200.iiib) against the IIB query on the same inputs, per S-block
size: device time of the whole join (events on the stream; includes the per-block host read of two nnz),
postings indexed (IIIB) vs nnz(S) (IIB), residual completions.  usage: python tools/iiib_bench.py C2 [blocks...]"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import gen  # noqa: E402
import paper_1011_2807_b200 as kj  # noqa: E402
from paper_1011_2807_b200.iiib import iiib_join  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    best = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        best = t if best is None else min(best, t)
    return best, out


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    blocks = [int(x) for x in sys.argv[2:]] or [None]
    c = gen.CONFIGS[name]
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)

    def iib():
        idx = kj.knnjoin_build_index(dS, c.d, head_density=-1.0)
        return kj.knnjoin_query(idx, dR, c.k)[:2]

    def iib_heads():
        idx = kj.knnjoin_build_index(dS, c.d)
        return kj.knnjoin_query(idx, dR, c.k)[:2]

    t_iib, (i0, s0) = timed(iib)
    t_head, _ = timed(iib_heads)
    print(json.dumps({"config": name, "impl": "IIB (no head features)", "ms": t_iib}))
    print(json.dumps({"config": name, "impl": "IIB + head-feature bound (default)", "ms": t_head}))
    for b in blocks:
        sb = b or S.n_rows
        t, (i1, s1, st) = timed(lambda: iiib_join(dR, dS, c.d, c.k, sb), reps=2)
        same = bool(torch.equal(i0, i1) and torch.equal(s0, s1))
        print(json.dumps({"config": name, "impl": "IIIB-literal (f1)", "s_block": sb, "ms": t, "identical_to_iib": same,
                          **st}))


if __name__ == "__main__":
    main()
