"""f4 measured: the C4 join with S held in pinned host memory and streamed through the GPU in
blocks (paper_1011_2807_b200.stream, Alg. 1's block nested loop), against the same join with S
resident in HBM.  Reports the device memory the streamed join allocated at its peak next to the size of S: the
device footprint is two block slots + one block index + R + the [|R|, k] lists, independent of |S|, so an S larger
than HBM streams the same way (one B200 box has no host with > 180 GB of S to show it literally).

    python tools/stream_bench.py [--config C4] [--rows-r N] [--blocks 8 16] [--reps 2]

Prints one JSON line per run; keys of the streamed join must equal the resident join's (exact)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import gen  # noqa: E402
import paper_1011_2807_b200._binding as kj  # noqa: E402
from paper_1011_2807_b200 import stream  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--rows-r", type=int, default=0)
    ap.add_argument("--rows-s", type=int, default=0)
    ap.add_argument("--blocks", type=int, nargs="+", default=[8, 16])
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    cfg = gen.CONFIGS[a.config]
    if a.rows_r or a.rows_s:
        cfg = cfg.scaled(a.rows_r or None, a.rows_s or None)
    R, S = gen.generate(cfg, "R"), gen.generate(cfg, "S")
    s_bytes = S.indptr.nbytes + S.indices.nbytes + (S.values.nbytes if S.values is not None else 0)
    dR = kj.DeviceCSR.from_host(R)
    pairs = R.n_rows * S.n_rows

    # resident reference: S copied once, one index, one query
    dS = kj.DeviceCSR.from_host(S)
    idx = kj.knnjoin_build_index(dS, cfg.d)
    _, _, ref = kj.knnjoin_query(idx, dR, cfg.k, want_keys=True)
    torch.cuda.synchronize()
    times = []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        idx2 = kj.knnjoin_build_index(dS, cfg.d)
        kj.knnjoin_query(idx2, dR, cfg.k)
        torch.cuda.synchronize()
        times.append(time.perf_counter() - t0)
        del idx2
    res_s = min(times)
    del idx, dS
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    print(json.dumps({"mode": "resident", "config": cfg.name, "pairs": pairs, "s_host_bytes": s_bytes,
                      "seconds": res_s, "pairs_per_s": pairs / res_s}), flush=True)

    for nb in a.blocks:
        pS = stream.PinnedS.from_host(S, block_rows=(S.n_rows + nb - 1) // nb)
        times, ok = [], True
        for rep in range(a.reps):
            torch.cuda.synchronize()
            torch.cuda.reset_peak_memory_stats()
            base = torch.cuda.memory_allocated()
            t0 = time.perf_counter()
            ids, sc, keys = stream.streamed_join(pS, dR, cfg.d, cfg.k, want_keys=True)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
            peak = torch.cuda.max_memory_allocated() - base
            ok = ok and torch.equal(keys, ref)
            del ids, sc, keys
        t = min(times)
        print(json.dumps({"mode": "streamed", "config": cfg.name, "blocks": nb, "block_rows": pS.block_rows,
                          "pairs": pairs, "s_host_bytes": s_bytes, "device_peak_bytes": peak,
                          "s_over_device_peak": s_bytes / peak, "seconds": t, "pairs_per_s": pairs / t,
                          "vs_resident": res_s / t, "keys_equal_resident": ok}), flush=True)
        if not ok:
            sys.exit(1)


if __name__ == "__main__":
    main()
