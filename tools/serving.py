"""Serving-shaped measurement: many small R batches queried against one resident S index (C2's laws), each
query launched eagerly vs replayed from a CUDA graph captured once (knnjoin_query is capturable after the
first query on an index).  Reports per-query device latency (CUDA events, median of 50) for batches of
16 / 128 / 1024 rows.  usage: python tools/serving.py [out.jsonl]
"""
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import paper_1011_2807_b200 as kj  # noqa: E402


def lat(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(n):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "serving.jsonl")
    torch.cuda.set_device(0)
    cfg = gen.CONFIGS["C2"]
    S = gen.generate(cfg, "S")
    idx = kj.knnjoin_build_index(kj.DeviceCSR.from_host(S), cfg.d)
    res = []
    for n in (16, 128, 1024):
        R = gen.generate(cfg.scaled(n, None), "R")
        dR = kj.DeviceCSR.from_host(R)
        kj.knnjoin_query(idx, dR, cfg.k)
        eager = lat(lambda: kj.knnjoin_query(idx, dR, cfg.k))
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            kj.knnjoin_query(idx, dR, cfg.k)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            kj.knnjoin_query(idx, dR, cfg.k)
        graph = lat(g.replay)
        r = {"study": "serving", "S_rows": S.n_rows, "R_rows": n, "k": cfg.k, "eager_ms": eager, "graph_ms": graph,
             "pairs_per_s_graph": n * S.n_rows / (graph * 1e-3)}
        print(json.dumps(r), flush=True)
        res.append(r)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    with open(out, "w") as f:
        for r in res:
            f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
