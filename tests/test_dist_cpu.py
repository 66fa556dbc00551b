"""-m "not gpu": the S-sharded multi-rank plumbing (paper_1011_2807_b200/dist.py) with world_size 2 on the
gloo backend.  Each rank computes its shard's top-k keys with the ORACLE (test infrastructure) instead of the
CUDA kernel, the real all-gather plumbing exchanges them, and a host model of the K4 merge (sort packed keys)
must reproduce the oracle's single-S result bit for bit on integer inputs."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _keys(ids, scores):
    """Packed ordering key of reading c1: (score << 32) | (0xFFFFFFFF - id); padding -> 0."""
    sc = scores.astype(np.uint64)
    gid = np.where(ids >= 0, ids, 0).astype(np.uint64)
    k = (sc << np.uint64(32)) | (np.uint64(0xFFFFFFFF) - gid)
    k[ids < 0] = 0
    return k.view(np.int64)


def _host_merge(gathered, k):
    g = gathered.numpy().view(np.uint64)  # [P, n, k]
    P, n, _ = g.shape
    allk = np.concatenate(list(g), axis=1)  # [n, P*k]
    out_ids = np.full((n, k), -1, np.int64)
    out_sc = np.zeros((n, k), np.int64)
    for i in range(n):
        row = sorted((int(x) for x in allk[i] if x), reverse=True)[:k]
        for t, key in enumerate(row):
            out_sc[i, t] = key >> 32
            out_ids[i, t] = 0xFFFFFFFF - (key & 0xFFFFFFFF)
    return out_ids, out_sc


def _worker(rank, world, port, cfg_name, n_r, n_s, q, theta=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import gen
        import oracle
        from paper_1011_2807_b200 import dist as kdist
        c = gen.CONFIGS[cfg_name].scaled(n_r, n_s)
        R = gen.generate(c, "R")
        lo, hi = kdist.shard_bounds(n_s, world, rank)
        S_shard = gen.generate(c, "S", lo, hi - lo)

        def local():
            ids, sc = oracle.knn(R, S_shard, c.k, s_id_base=lo)
            return torch.from_numpy(_keys(ids, sc))

        if not theta:
            ids, sc = kdist.sharded_join(local, lambda g: _host_merge(g, c.k))
        else:
            # f2 two-phase protocol: phase 1 over the first half of the shard, all_reduce(MAX) of the k-th keys,
            # phase 2 continues with the rest keeping only keys >= floor (host model of the query's
            # tile_range / resume_keys / theta_in semantics)
            mid = lo + (hi - lo) // 2
            S_a = gen.generate(c, "S", lo, mid - lo)
            S_b = gen.generate(c, "S", mid, hi - mid)

            def phase1():
                ids, sc = oracle.knn(R, S_a, c.k, s_id_base=lo)
                return torch.from_numpy(_keys(ids, sc))

            def phase2(partial, floor):
                ids, sc = oracle.knn(R, S_b, c.k, s_id_base=mid)
                rest = _keys(ids, sc)
                f = floor.numpy()[:, None]
                rest = np.where(rest >= f, rest, 0)
                both = np.sort(np.concatenate([partial.numpy(), rest], axis=1).view(np.uint64), axis=1)[:, ::-1]
                seen_floor.append(int((rest == 0).sum()))
                return torch.from_numpy(np.ascontiguousarray(both[:, :c.k]).view(np.int64))

            seen_floor = []
            ids, sc = kdist.sharded_join_theta(phase1, phase2, lambda g: _host_merge(g, c.k), c.k)
        q.put((rank, ids, sc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name,n_r,n_s,theta", [("C1", 40, 3001, False), ("C5", 6, 2000, False),
                                                    ("C1", 40, 3001, True), ("C5", 6, 2000, True)])
def test_sharded_join_world2_gloo(cfg_name, n_r, n_s, theta):
    """world 2: plain S-sharded join, and the f2 two-phase protocol with cross-rank k-th-key floors; both must
    give the oracle's single-S lists bit for bit."""
    import gen
    import oracle
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_name, n_r, n_s, q, theta)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = gen.CONFIGS[cfg_name].scaled(n_r, n_s)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    o_ids, o_sc = oracle.knn(R, S, c.k)
    for _, ids, sc in res:
        np.testing.assert_array_equal(ids, o_ids)
        np.testing.assert_array_equal(sc, o_sc.astype(np.int64))


def test_shard_bounds_cover_exactly():
    from paper_1011_2807_b200.dist import shard_bounds
    for n in (0, 1, 7, 100, 10_000_000):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
