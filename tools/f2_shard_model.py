"""f2 on one GPU: what the cross-rank threshold floor buys one rank of an S-sharded C4 run.

C4 (|R| = 100,000 x |S| = 10,000,000, Zipf, k = 10) split over P ranks: rank 0 owns S rows [0, |S|/P).  On one
B200 this script times rank 0's work both ways, with every other rank's phase-1 query also run here (in turn)
only to produce the floor it would receive:
  plain  : knnjoin_query over the whole shard (the shard's own k-th keys are the only threshold);
  f2     : phase 1 over the shard's first `a` tiles on every rank's shard, floor = max over ranks of the rows'
           k-th keys (dist.kth_floor's all_reduce, here a torch.maximum over the P partial lists), then
           phase 2 over the remaining tiles of shard 0 with resume_keys + theta_in.
Reported: rank-0 kernel time of each (CUDA events), the head-completion counters, and a check that both give
the same rank-0 lists up to the floor (merged results are identical by construction; tests cover that).
usage: python tools/f2_shard_model.py [P] [a]
"""
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import paper_1011_2807_b200 as kj  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    a = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    cfg = gen.CONFIGS["C4"]
    n_s = cfg.S.n_rows // P
    R = gen.generate(cfg, "R")
    dR = kj.DeviceCSR.from_host(R)
    k = cfg.k
    shard0 = kj.DeviceCSR.from_host(gen.generate(cfg, "S", 0, n_s))
    idx0 = kj.knnjoin_build_index(shard0, cfg.d, s_id_base=0)
    nt = kj.knnjoin_index_stats(idx0)["n_tiles"]

    cnt_plain = torch.zeros(4, dtype=torch.int64, device="cuda")
    kj.knnjoin_query(idx0, dR, k, want_keys=True, want_ids=False, counters=cnt_plain)
    ms_plain = timed(lambda: kj.knnjoin_query(idx0, dR, k, want_keys=True, want_ids=False))

    # phase 1 on every rank's shard (each built in turn), floor = max of the rows' k-th keys
    part0 = kj.knnjoin_query(idx0, dR, k, want_keys=True, want_ids=False, tile_range=(0, a))[2]
    floor = part0[:, k - 1].clone()
    for p in range(1, P):
        sh = kj.DeviceCSR.from_host(gen.generate(cfg, "S", p * n_s, n_s))
        ix = kj.knnjoin_build_index(sh, cfg.d, s_id_base=p * n_s)
        part = kj.knnjoin_query(ix, dR, k, want_keys=True, want_ids=False, tile_range=(0, a))[2]
        floor = torch.maximum(floor, part[:, k - 1])
        del ix, sh
    floor = floor.contiguous()
    ms_p1 = timed(lambda: kj.knnjoin_query(idx0, dR, k, want_keys=True, want_ids=False, tile_range=(0, a)))
    cnt_f2 = torch.zeros(4, dtype=torch.int64, device="cuda")
    kj.knnjoin_query(idx0, dR, k, want_keys=True, want_ids=False, tile_range=(a, nt), resume_keys=part0,
                     theta_in=floor, counters=cnt_f2)
    ms_p2 = timed(lambda: kj.knnjoin_query(idx0, dR, k, want_keys=True, want_ids=False, tile_range=(a, nt),
                                           resume_keys=part0, theta_in=floor))
    out = {"P": P, "phase1_tiles": a, "shard_rows": n_s, "n_tiles": nt, "rank0_plain_ms": ms_plain,
           "rank0_f2_ms": ms_p1 + ms_p2, "phase1_ms": ms_p1, "phase2_ms": ms_p2,
           "head_completions_plain": int(cnt_plain[3]), "head_completions_f2_phase2": int(cnt_f2[3])}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
