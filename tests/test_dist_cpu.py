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


def _worker(rank, world, port, cfg_name, n_r, n_s, q, theta=False, mode="s"):
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

        if mode == "r":
            # R-sharded: every rank answers its own rows of R against all of S, no collective in the join; the
            # test gathers the answers afterwards only to compare them
            S_all = gen.generate(c, "S")
            rlo, rhi = kdist.shard_bounds(n_r, world, rank)
            ids, sc = oracle.knn(R, S_all, c.k, rows=np.arange(rlo, rhi))
            parts = [None] * world
            dist.all_gather_object(parts, (ids, sc))
            ids = np.concatenate([p[0] for p in parts])
            sc = np.concatenate([p[1] for p in parts]).astype(np.int64)
        elif mode == "fallback":
            # the certification step of sharded_join: rows {1, 3} "fail" certification (host stand-in for
            # knnjoin_certify); every rank recomputes only those rows (here: with +1 added to every score, so the
            # replacement is visible) and the listed rows of the merged result are replaced
            def certify(result):
                return torch.tensor([2, 1, 3] + [0] * (n_r - 2), dtype=torch.int32)

            def wide_keys(lst):
                rows = lst[1:1 + int(lst[0])].numpy()
                ids, sc = oracle.knn(R, S_shard, c.k, rows=rows, s_id_base=lo)
                keys = np.zeros((n_r, c.k), np.int64)
                keys[rows] = _keys(ids, np.where(ids >= 0, sc + 1, 0))
                return torch.from_numpy(keys)

            def wide_merge(gathered, lst, result):
                ids, sc = result
                m_ids, m_sc = _host_merge(gathered, c.k)
                rows = lst[1:1 + int(lst[0])].numpy()
                ids, sc = ids.copy(), sc.copy()
                ids[rows], sc[rows] = m_ids[rows], m_sc[rows]
                return ids, sc

            fb = kdist.Fallback(certify, wide_keys, wide_merge)
            ids, sc = kdist.sharded_join(local, lambda g: _host_merge(g, c.k), fallback=fb)
        elif not theta:
            ids, sc = kdist.sharded_join(local, lambda g: _host_merge(g, c.k))
        else:
            # f2 periodic protocol: the shard in 3 parts (phases); after each phase all_reduce(MAX) of the k-th
            # keys, and the next phase keeps only keys >= floor (host model of the query's tile_range /
            # resume_keys / theta_in semantics); ranks may have empty parts
            cuts = [lo + ((hi - lo) * j) // 3 for j in range(4)]

            def phase(i, partial, floor):
                part = gen.generate(c, "S", cuts[i], cuts[i + 1] - cuts[i])
                ids, sc = oracle.knn(R, part, c.k, s_id_base=cuts[i])
                rest = _keys(ids, sc)
                if floor is not None:
                    rest = np.where(rest >= floor.numpy()[:, None], rest, 0)
                if partial is None:
                    return torch.from_numpy(rest)
                both = np.sort(np.concatenate([partial.numpy(), rest], axis=1).view(np.uint64), axis=1)[:, ::-1]
                return torch.from_numpy(np.ascontiguousarray(both[:, :c.k]).view(np.int64))

            ids, sc = kdist.sharded_join_theta(phase, 3, lambda g: _host_merge(g, c.k), c.k)
        q.put((rank, ids, sc))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,cfg_name,n_r,n_s,theta,mode", [
    (2, "C1", 40, 3001, False, "s"), (2, "C5", 6, 2000, False, "s"), (2, "C1", 40, 3001, True, "s"),
    (2, "C5", 6, 2000, True, "s"), (4, "C1", 40, 3001, False, "s"), (4, "C1", 40, 3001, True, "s"),
    (4, "C5", 6, 2003, True, "s"), (2, "C1", 41, 3001, False, "r"), (4, "C5", 7, 1500, False, "r"),
    (2, "C1", 40, 3001, False, "fallback"), (4, "C1", 40, 3001, False, "fallback")])
def test_sharded_join_gloo(world, cfg_name, n_r, n_s, theta, mode):
    """world 2 and 4 on gloo: plain S-sharded join; the f2 periodic protocol with cross-rank k-th-key floors after
    every phase; the R-sharded join (no collective); all must give the oracle's single-S lists bit for bit.  The
    certification fallback replaces exactly the listed rows with the re-merged recomputation."""
    import gen
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_name, n_r, n_s, q, theta, mode))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = gen.CONFIGS[cfg_name].scaled(n_r, n_s)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    o_ids, o_sc = oracle.knn(R, S, c.k)
    o_sc = o_sc.astype(np.int64)
    if mode == "fallback":
        o_sc[[1, 3]] = np.where(o_ids[[1, 3]] >= 0, o_sc[[1, 3]] + 1, 0)
    for _, ids, sc in res:
        np.testing.assert_array_equal(ids, o_ids)
        np.testing.assert_array_equal(sc, o_sc)


def test_shard_bounds_cover_exactly():
    from paper_1011_2807_b200.dist import shard_bounds
    for n in (0, 1, 7, 100, 10_000_000):
        for w in (1, 2, 3, 8):
            b = [shard_bounds(n, w, r) for r in range(w)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(w - 1))
            assert max(h - l for l, h in b) - min(h - l for l, h in b) <= 1
