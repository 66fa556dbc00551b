"""-m gpu: the CUDA path (through the C ABI) against the oracle, element by element."""
import numpy as np
import pytest
import torch

import gen
import oracle
from tests.gpu_util import assert_parity, gpu_join
from tests.util import csr_from_rows, random_csr, stable_seed

pytestmark = pytest.mark.gpu


def _check(R, S, k, tile=0, batch_rows=0, threads=8, **kw):
    g_ids, g_sc = gpu_join(R, S, k, tile=tile, batch_rows=batch_rows, **kw)
    o_ids, o_sc = oracle.knn(R, S, k, threads=threads)
    assert_parity(R, S, g_ids, g_sc, o_ids, o_sc)
    return g_ids, g_sc


def test_hand_example():
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_example.json")))
    R = csr_from_rows(g["R"], g["d"], "binary")
    S = csr_from_rows(g["S"], g["d"], "binary")
    for k, want in g["expect"].items():
        ids, sc = gpu_join(R, S, int(k), tile=2048)
        assert [[int(a), int(b)] for a, b in zip(ids[0], sc[0])] == want


@pytest.mark.parametrize("dtr,dts", [("binary", "binary"), ("int8", "int8"), ("fp32", "binary"), ("int8", "binary"),
                                     ("binary", "int8"), ("fp32", "int8")])
@pytest.mark.parametrize("k", [1, 5, 33, 256])
def test_random_small_multi_tile(dtr, dts, k):
    """Several tiles (tile=2048) with a ragged tail, tie-heavy small value ranges."""
    rng = np.random.default_rng(stable_seed(dtr, dts, k))
    d = 300
    R = random_csr(rng, 37, d, 0, 40, dtr, vmax=4)
    S = random_csr(rng, 5000, d, 0, 30, dts, vmax=4)
    _check(R, S, k, tile=2048)


@pytest.mark.parametrize("batch_rows", [1, 2, 4, 6, 8])
def test_batch_sizes(batch_rows):
    rng = np.random.default_rng(batch_rows)
    R = random_csr(rng, 53, 200, 1, 50, "fp32")
    S = random_csr(rng, 9000, 200, 1, 30, "binary")
    _check(R, S, 10, tile=4096, batch_rows=batch_rows)


def test_edge_cases():
    d = 64
    R = csr_from_rows([[0, 1, 2], [], [63], [5, 6]], d, "binary")
    S = csr_from_rows([[0], [], [1, 2, 3], [63], [7]], d, "binary")
    _check(R, S, 4, tile=2048)
    # k larger than #positives everywhere; k = 1
    _check(R, S, 7, tile=2048)
    _check(R, S, 1, tile=2048)
    # R features beyond d are ignored (S cannot have them)
    Rw = csr_from_rows([[0, 70, 80]], 128, "binary")
    Sw = csr_from_rows([[0], [0, 1]], 128, "binary")
    ids, sc = gpu_join(Rw, Sw, 2, d=64, tile=2048)
    assert ids.tolist() == [[0, 1]] and sc.tolist() == [[1.0, 1.0]]


def test_empty_inputs():
    import paper_1011_2807_b200 as kj
    d = 32
    R = csr_from_rows([[1, 2], [3]], d, "binary")
    Sempty = csr_from_rows([], d, "binary")
    ids, sc = gpu_join(R, Sempty, 3, tile=2048)
    assert (ids == -1).all() and (sc == 0).all()
    Rempty = csr_from_rows([], d, "binary")
    S = csr_from_rows([[1]], d, "binary")
    ids, sc = gpu_join(Rempty, S, 3, tile=2048)
    assert ids.shape == (0, 3)


def test_counters_match_eq4():
    """Unpruned postings visited == Eq. 4 second term = sum_d n_R(d) n_S(d), exactly."""
    c = gen.CONFIGS["C2"].scaled(300, 20000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    gpu_join(R, S, c.k, counters=cnt)
    nR = np.bincount(R.indices, minlength=c.d)
    nS = np.bincount(S.indices, minlength=c.d)
    assert int(cnt[0]) == int((nR.astype(np.int64) * nS).sum())
    assert int(cnt[1]) > 0


def test_deterministic():
    c = gen.CONFIGS["C3"].scaled(200, 40000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    a = gpu_join(R, S, c.k)
    b = gpu_join(R, S, c.k, batch_rows=2)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


@pytest.mark.parametrize("name,n_r,n_s,tile", [
    ("C1", None, None, 0),          # full C1 (configs[0]): bit-exact
    ("C1", None, None, 2048),
    ("C2", 400, 30000, 0),
    ("C3", 300, 50000, 0),
    ("C4", 200, 40000, 0),
    ("C5", 60, 30000, 0),           # int8 x int8, k=100: bit-exact
    ("C5", 40, 20000, 4096),
])
def test_configs_scaled(name, n_r, n_s, tile):
    c = gen.CONFIGS[name].scaled(n_r, n_s)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    _check(R, S, c.k, tile=tile)


@pytest.mark.parametrize("name,n_s,Ps", [("C2", 30000, (2, 3, 4)), ("C5", 16000, (2, 8)), ("C1", 9000, (3, 8))])
def test_sharded_merge_equals_single_index(name, n_s, Ps):
    """T7: S split in P contiguous shards, P indexes with s_id_base, knnjoin_merge == one index, bit-exact
    (k = 100 and int8 values at C5, tie-heavy binary at C1, up to 8 shards)."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS[name].scaled(150, n_s)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    full_ids, full_sc, full_keys = gpu_join(R, S, c.k, want_keys=True)
    for P in Ps:
        bounds = np.linspace(0, S.n_rows, P + 1).astype(np.int64)
        keys = []
        for p in range(P):
            part = S.take_rows(np.arange(bounds[p], bounds[p + 1]))
            _, _, kk = gpu_join(R, part, c.k, d=c.d, s_id_base=int(bounds[p]), want_keys=True)
            keys.append(torch.from_numpy(kk))
        allk = torch.stack(keys).cuda()
        dR = kj.DeviceCSR.from_host(R)
        ids, sc, mk = kj.knnjoin_merge(allk, dR, c.d, kj.BINARY if S.values is None else kj.INT8, c.k,
                                       want_keys=True)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ids.cpu().numpy(), full_ids)
        np.testing.assert_array_equal(sc.cpu().numpy(), full_sc.astype(np.float32))
        np.testing.assert_array_equal(mk.cpu().numpy(), full_keys)


def test_validate_csr():
    import paper_1011_2807_b200 as kj
    ok = kj.DeviceCSR.from_arrays(np.array([0, 2, 3]), np.array([1, 4, 0]), np.array([1.0, 2.0, 3.0], np.float32))
    assert kj.knnjoin_validate_csr(ok, 8) == (0, -1)
    bad = kj.DeviceCSR.from_arrays(np.array([0, 2, 3]), np.array([4, 1, 0]), np.array([1.0, 2.0, 3.0], np.float32))
    assert kj.knnjoin_validate_csr(bad, 8) == (3, 0)
    neg = kj.DeviceCSR.from_arrays(np.array([0, 2, 3]), np.array([1, 4, 0]), np.array([1.0, 2.0, -3.0], np.float32))
    assert kj.knnjoin_validate_csr(neg, 8) == (3, 1)
    oob = kj.DeviceCSR.from_arrays(np.array([0, 1, 2]), np.array([1, 9]))
    assert kj.knnjoin_validate_csr(oob, 8) == (3, 1)


@pytest.mark.parametrize("name,T,hd", [("C5", 4096, 0.0), ("C2", 2048, 0.0), ("C2", 8192, 0.05), ("C2", 2048, 1e-6)])
def test_index_layout_matches_scipy_csc(name, T, hd):
    """T3: decode the built index (id-list slices per (feature, tile) + head-feature words) and compare with
    scipy's CSC restricted to each tile; df exact; head features are the most frequent ones."""
    import scipy.sparse as sp
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS[name].scaled(10, 9000)
    S = gen.generate(c, "S")
    dS = kj.DeviceCSR.from_host(S)
    idx = kj.knnjoin_build_index(dS, c.d, tile=T, head_density=hd)
    torch.cuda.synchronize()
    st = kj.knnjoin_index_stats(idx)
    raw = idx.storage.cpu().numpy()
    NT = st["n_tiles"]
    n_off = st["offsets"]
    off = raw[:4 * n_off].view(np.uint32)
    al = lambda x: (x + 255) // 256 * 256
    df_at = al(4 * n_off)
    df = raw[df_at:df_at + 4 * c.d].view(np.int32)
    hs_at = al(df_at + 4 * c.d)
    head_slot = raw[hs_at:hs_at + 4 * c.d].view(np.int32)
    hf_at = al(hs_at + 4 * c.d)
    head_feat = raw[hf_at:hf_at + 4 * 33].view(np.int32)
    hc_at = al(hf_at + 4 * 33)
    head_cols = raw[hc_at:hc_at + 4 * NT * T].view(np.uint32)
    ids_at = al(hc_at + 4 * NT * T)
    cap = st["unit_capacity"]
    ids = raw[ids_at:ids_at + 16 * cap].view(np.uint16)
    assert np.all(ids % 4 == 0)  # stored as byte offsets of the score columns
    ids = ids // 4
    vals = None
    if S.values is not None:
        vals_at = al(ids_at + 16 * cap)
        vals = raw[vals_at:vals_at + 8 * cap].view(np.uint8)
    want_df = np.bincount(S.indices, minlength=c.d)
    np.testing.assert_array_equal(df, want_df)
    n_head = int(head_feat[32])
    heads = head_feat[:n_head]
    if name == "C5":
        assert n_head == 0
    else:
        assert n_head > 0
        order = np.lexsort((np.arange(c.d), -want_df))  # df desc, feature asc
        np.testing.assert_array_equal(heads, order[:n_head])
        assert want_df[heads].min() >= int(np.ceil(st["head_min_df"]))
        for i, f in enumerate(heads):
            assert head_slot[f] == i
    data = np.ones(S.nnz, np.int64) if S.values is None else S.values.astype(np.int64)
    M = sp.csr_matrix((data, S.indices, S.indptr), shape=(S.n_rows, c.d)).tocsc()
    # head words: bit i of head_cols[s] <=> s has heads[i]
    for i, f in enumerate(heads):
        bits = ((head_cols[:S.n_rows] >> np.uint32(i)) & np.uint32(1)).astype(bool)
        want = np.zeros(S.n_rows, bool)
        want[M[:, f].indices] = True
        np.testing.assert_array_equal(bits, want)
    assert not head_cols[S.n_rows:].any()
    rng = np.random.default_rng(0)
    for f in rng.choice(c.d, 400, replace=False):
        col = M[:, f]
        rows_f, vals_f = col.indices, col.data
        for t in range(NT):
            key = f * (NT + 1) + t
            a, b = int(off[key]), int(off[key + 1])
            sel = (rows_f >= t * T) & (rows_f < (t + 1) * T)
            if head_slot[f] >= 0:
                assert b == a
                continue
            got = ids[8 * a:8 * b]
            keep = got < T
            assert np.all(got[~keep] < T + 32)
            order = np.argsort(got[keep])
            np.testing.assert_array_equal(got[keep][order].astype(np.int64), rows_f[sel] - t * T)
            if vals is not None:
                np.testing.assert_array_equal(vals[8 * a:8 * b][keep][order], vals_f[sel])
            assert b - a == (sel.sum() + 7) // 8


@pytest.mark.parametrize("hd,hm", [(-1.0, 0), (0.0, 0), (0.01, 0), (0.01, 5), (0.3, 0), (1e-6, 0)])
def test_head_feature_modes(hd, hm):
    """Head features (lookup-table path) and id lists give identical results for any head set."""
    c = gen.CONFIGS["C2"].scaled(300, 30000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    ids, sc = _check(R, S, c.k, tile=4096, head_density=hd, head_max=hm, counters=cnt)
    ref = gpu_join(R, S, c.k, tile=4096, head_density=-1.0)
    np.testing.assert_array_equal(ids, ref[0])
    np.testing.assert_array_equal(sc, ref[1])
    nR = np.bincount(R.indices, minlength=c.d)
    nS = np.bincount(S.indices, minlength=c.d)
    assert int(cnt[0]) == int((nR.astype(np.int64) * nS).sum())


@pytest.mark.parametrize("cta_warps,batch_rows", [(8, 3), (16, 6), (8, 1)])
def test_multi_chunk_batches(cta_warps, batch_rows):
    """More runs per batch than one staging chunk holds, with head features present."""
    rng = np.random.default_rng(7)
    d = 2000
    rows = []
    for _ in range(16):
        head = list(range(0, 40))
        tail = sorted(rng.choice(np.arange(40, d), size=400, replace=False).tolist())
        rows.append([(f, float(np.float32(rng.lognormal()))) for f in head + tail])
    R = csr_from_rows(rows, d, "fp32")
    S = random_csr(rng, 6000, d, 5, 40, "binary")
    Srows = []
    for i in range(S.n_rows):
        idx, _ = S.row(i)
        extra = rng.choice(40, size=20, replace=False)
        Srows.append(sorted(set(idx.tolist()) | set(extra.tolist())))
    S = csr_from_rows(Srows, d, "binary")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    _check(R, S, 10, tile=2048, batch_rows=batch_rows, cta_warps=cta_warps, counters=cnt)
    nR = np.bincount(R.indices, minlength=d)
    nS = np.bincount(S.indices, minlength=d)
    assert int(cnt[0]) == int((nR.astype(np.int64) * nS).sum())


def test_wide_rows_fallback_run_merge():
    """Batches with more (row, feature) entries than the block sort holds (4096) use the warp merge."""
    rng = np.random.default_rng(11)
    d = 3000
    R = random_csr(rng, 9, d, 1300, 1500, "int8", vmax=5)
    S = random_csr(rng, 4000, d, 100, 300, "int8", vmax=5)
    _check(R, S, 20, tile=2048, batch_rows=4, cta_warps=8)


@pytest.mark.slow
@pytest.mark.parametrize("name,n_sample", [("C2", 64), ("C3", 24), ("C4", 12), ("C5", 16)])
def test_full_size_sampled_rows(name, n_sample):
    """BASELINE.json full sizes, in the launch configuration bench.py times (default tile, auto batch shape):
    every row is computed on the GPU; a seeded sample of rows (first, last and random) is checked against the
    oracle, one row at a time against all of S."""
    import os
    c = gen.CONFIGS[name]
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    g_ids, g_sc = gpu_join(R, S, c.k)
    rng = np.random.default_rng(2024)
    rows = np.unique(np.concatenate([[0, R.n_rows - 1], rng.choice(R.n_rows, n_sample - 2, replace=False)]))
    threads = max(1, min(len(rows), len(os.sched_getaffinity(0))))
    o_ids, o_sc = oracle.knn(R, S, c.k, rows=rows, threads=threads)
    assert_parity(R.take_rows(rows), S, g_ids[rows], g_sc[rows], o_ids, o_sc, rows=None)


@pytest.mark.slow
def test_full_size_C2_every_row():
    """C2 (BASELINE.json configs[1]) at full size, in the bench's launch configuration: EVERY one of the 10,000
    rows against all 100,000 rows of S checked by the oracle (1e9 pairs; rows split over the host's threads)."""
    import os
    c = gen.CONFIGS["C2"]
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    g_ids, g_sc = gpu_join(R, S, c.k)
    o_ids, o_sc = oracle.knn(R, S, c.k, threads=max(1, len(os.sched_getaffinity(0))))
    assert_parity(R, S, g_ids, g_sc, o_ids, o_sc)


@pytest.mark.parametrize("name,tpp", [("C2", 1), ("C2", 3), ("C3", 2), ("C5", 1)])
def test_tile_passes_identical(name, tpp):
    """Pass-major schedule (top-k state carried between passes in the workspace) == single pass, bit for bit."""
    c = gen.CONFIGS[name].scaled(60, 20000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    ids, sc = _check(R, S, c.k, tile=2048, tiles_per_pass=tpp)
    ref = gpu_join(R, S, c.k, tile=2048, tiles_per_pass=1000)
    np.testing.assert_array_equal(ids, ref[0])
    np.testing.assert_array_equal(sc, ref[1])


@pytest.mark.parametrize("name,batch_rows,cta_warps", [("C2", 0, 0), ("C2", 3, 8), ("C3", 0, 0), ("C5", 0, 0),
                                                       ("C1", 8, 16)])
def test_row_order_identical(name, batch_rows, cta_warps):
    """a3: batching rows in descending work order (default) == input order, bit for bit, and both match the
    oracle; ragged last batch (61 rows)."""
    c = gen.CONFIGS[name].scaled(61, 12000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    ids, sc = _check(R, S, c.k, tile=2048, batch_rows=batch_rows, cta_warps=cta_warps, row_order=0)
    ref = gpu_join(R, S, c.k, tile=2048, batch_rows=batch_rows, cta_warps=cta_warps, row_order=1)
    np.testing.assert_array_equal(ids, ref[0])
    np.testing.assert_array_equal(sc, ref[1])


@pytest.mark.parametrize("name", ["C2", "C3", "C5"])
def test_tile_range_resume_identical(name):
    """tile_range + resume_keys: queries over [0, 1), [1, a), [a, NT) chained through resume_keys == one
    query over every tile, bit for bit (keys included); an empty range passes the resumed lists through."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS[name].scaled(70, 14000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dS, dR = kj.DeviceCSR.from_host(S), kj.DeviceCSR.from_host(R)
    idx = kj.knnjoin_build_index(dS, c.d, tile=2048)
    NT = kj.knnjoin_index_stats(idx)["n_tiles"]
    assert NT >= 4
    full = kj.knnjoin_query(idx, dR, c.k, want_keys=True)
    a = NT // 2
    keys = None
    for rng in ((0, 1), (1, a), (a, a), (a, NT)):
        ids, sc, keys = kj.knnjoin_query(idx, dR, c.k, want_keys=True, tile_range=rng, resume_keys=keys)
    torch.cuda.synchronize()
    for x, y in zip(full, (ids, sc, keys)):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())
    with pytest.raises(kj.KnnJoinError):
        kj.knnjoin_query(idx, dR, c.k, tile_range=(1, NT + 1))


@pytest.mark.parametrize("name", ["C2", "C1", "C5"])
def test_theta_floor_two_shards_merge_exact(name):
    """f2 on one GPU: two S shards (s_id_base), phase 1 over each shard's first tile, floor = max over shards
    of the rows' k-th keys, phase 2 over the remaining tiles with resume_keys + theta_in; knnjoin_merge of the
    two lists == the single-index result bit for bit, and phase 2 keeps no key of its own tiles below the
    floor."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS[name].scaled(90, 24000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR = kj.DeviceCSR.from_host(R)
    full_ids, full_sc, full_keys = gpu_join(R, S, c.k, tile=2048, want_keys=True)
    half = S.n_rows // 2
    shards = [(0, S.take_rows(np.arange(0, half))), (half, S.take_rows(np.arange(half, S.n_rows)))]
    idxs = [kj.knnjoin_build_index(kj.DeviceCSR.from_host(part), c.d, s_id_base=base, tile=2048)
            for base, part in shards]
    p1 = [kj.knnjoin_query(ix, dR, c.k, want_keys=True, want_ids=False, tile_range=(0, 1))[2] for ix in idxs]
    floor = torch.maximum(p1[0][:, c.k - 1], p1[1][:, c.k - 1]).contiguous()
    p2 = []
    for ix, part in zip(idxs, p1):
        NT = kj.knnjoin_index_stats(ix)["n_tiles"]
        p2.append(kj.knnjoin_query(ix, dR, c.k, want_keys=True, want_ids=False, tile_range=(1, NT),
                                   resume_keys=part, theta_in=floor)[2])
    for part, fin in zip(p1, p2):  # keys of phase 2 are either resumed or >= floor
        fin_np, part_np, f = fin.cpu().numpy(), part.cpu().numpy(), floor.cpu().numpy()
        for i in range(R.n_rows):
            new = set(fin_np[i][fin_np[i] != 0]) - set(part_np[i])
            assert all(x >= f[i] for x in new)
    s_dtype = kj.BINARY if S.values is None else kj.INT8
    ids, sc, mk = kj.knnjoin_merge(torch.stack(p2), dR, c.d, s_dtype, c.k, want_keys=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids.cpu().numpy(), full_ids)
    np.testing.assert_array_equal(sc.cpu().numpy(), full_sc.astype(np.float32))
    np.testing.assert_array_equal(mk.cpu().numpy(), full_keys)


@pytest.mark.parametrize("name,blocks", [("C2", 3), ("C5", 4), ("C1", 1)])
def test_streamed_join_equals_single_index(name, blocks):
    """f4: S in pinned host memory streamed block by block (double-buffered copies, top-k lists resumed across
    blocks) == one index over all of S, bit for bit; ragged last block."""
    from paper_1011_2807_b200 import stream
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS[name].scaled(50, 20001)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    full_ids, full_sc, full_keys = gpu_join(R, S, c.k, want_keys=True)
    pS = stream.PinnedS.from_host(S, block_rows=(S.n_rows + blocks - 1) // blocks)
    ids, sc, keys = stream.streamed_join(pS, kj.DeviceCSR.from_host(R), c.d, c.k, want_keys=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids.cpu().numpy(), full_ids)
    np.testing.assert_array_equal(sc.cpu().numpy(), full_sc.astype(np.float32))
    np.testing.assert_array_equal(keys.cpu().numpy(), full_keys)


def test_query_cuda_graph_replay():
    """After the first query on an index (which reads the index statistics once), knnjoin_query is
    stream-capturable: a CUDA graph of one query replays to the same lists, and a replay after new R weights
    are written into the captured input buffers gives that R's lists (serving many R batches of one shape
    against one S)."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS["C2"].scaled(64, 30000)
    S = gen.generate(c, "S")
    R1 = gen.generate(c, "R")
    idx = kj.knnjoin_build_index(kj.DeviceCSR.from_host(S), c.d)
    dR = kj.DeviceCSR.from_host(R1)
    ref1 = kj.knnjoin_query(idx, dR, c.k)  # first query: reads the index statistics (synchronises once)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        kj.knnjoin_query(idx, dR, c.k)  # warm-up on the capture stream
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        ids, sc, _ = kj.knnjoin_query(idx, dR, c.k)
    g.replay()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ids.cpu().numpy(), ref1[0].cpu().numpy())
    np.testing.assert_array_equal(sc.cpu().numpy(), ref1[1].cpu().numpy())
    # a new R of the same shape: same features, new positive weights
    rng = np.random.default_rng(5)
    vals = (R1.values * rng.uniform(0.1, 3.0, R1.nnz)).astype(np.float32)
    R3 = gen.HostCSR(R1.indptr, R1.indices, vals, c.d)
    dR.values.copy_(torch.from_numpy(vals))
    g.replay()
    torch.cuda.synchronize()
    o_ids, o_sc = oracle.knn(R3, S, c.k, threads=8)
    assert_parity(R3, S, ids.cpu().numpy().astype(np.int64), sc.cpu().numpy().astype(np.float64), o_ids, o_sc)
    assert not np.array_equal(o_ids, ref1[0].cpu().numpy())  # the replay really computed a different join


@pytest.mark.parametrize("name,n_r", [("C2", 16), ("C2", 300), ("C3", 40), ("C5", 24), ("C1", 100)])
def test_split_tile_groups_identical(name, n_r):
    """Small R (fewer batches than resident CTAs): the tiles are split into independent groups whose lists
    are merged by rank after the kernel -- bit-identical (keys included) to the unsplit schedule
    (tiles_per_pass given explicitly disables the split), and to the oracle."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS[name].scaled(n_r, 25000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    ids, sc = _check(R, S, c.k, tile=2048)
    dS, dR = kj.DeviceCSR.from_host(S), kj.DeviceCSR.from_host(R)
    idx = kj.knnjoin_build_index(dS, c.d, tile=2048)
    split = kj.knnjoin_query(idx, dR, c.k, want_keys=True)
    whole = kj.knnjoin_query(idx, dR, c.k, want_keys=True, tiles_per_pass=1000)
    torch.cuda.synchronize()
    for x, y in zip(split, whole):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())
    np.testing.assert_array_equal(ids, whole[0].cpu().numpy())
