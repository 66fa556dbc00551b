"""-m gpu: threshold-pruned queries through the C ABI.

Pruning only changes the work: every pruned result must pass the oracle parity rules AND equal the unpruned
GPU result bit for bit (integer / fixed-point scores are order-independent, reading c17)."""
import numpy as np
import pytest
import torch

import gen
import oracle
from tests.gpu_util import assert_parity, gpu_join
from tests.util import csr_from_rows, random_csr, stable_seed

pytestmark = pytest.mark.gpu


def _pruned_equals_unpruned(R, S, k, tile, alphas, threads=8, d=None, oracle_check=True, **kw):
    ref = gpu_join(R, S, k, d=d, tile=tile, head_density=-1.0, **kw)
    if oracle_check:
        o_ids, o_sc = oracle.knn(R, S, k, threads=threads)
        assert_parity(R, S, ref[0], ref[1], o_ids, o_sc)
    out = []
    for a in alphas:
        cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
        ids, sc = gpu_join(R, S, k, d=d, tile=tile, prune=1, alpha=a, counters=cnt, **kw)
        if oracle_check:
            assert_parity(R, S, ids, sc, o_ids, o_sc)
        np.testing.assert_array_equal(ids, ref[0], err_msg=f"alpha={a}: ids differ from the unpruned query")
        np.testing.assert_array_equal(sc, ref[1], err_msg=f"alpha={a}: scores differ from the unpruned query")
        out.append(cnt.cpu().numpy())
    return out


def test_hand_example_r_side_pruning():
    """SURVEY.md §8(c) pin 'r-side pruning': r = {(0,3),(1,1),(2,0.5)}, binary S, k = 1; tile 0 = {s0:{0,1},
    s1:{0,2}}, tile 1 = {s2:{1,2}, s3:{0}, s4:{2}}.  After tile 0 theta = score(s0) = 4; in tile 1 at alpha = 1 the
    non-essential set is N = {1, 2} (U_N = 1.5 <= theta - 1 in fixed point), only the d0 slice is loaded
    (s3: 3), 3 + 1.5 >= 4 so s3 is completed exactly (3, rejected).  Result [(s0, 4.0)]; the 2 posting units of
    N's slices are skipped and one completion is made.  (tiles_per_pass = 2: one row would otherwise split the two
    tiles into independent groups, each starting from theta = 0.)"""
    import paper_1011_2807_b200 as kj
    T = 2048
    rows = [[] for _ in range(T + 3)]
    rows[0], rows[1] = [0, 1], [0, 2]
    rows[T], rows[T + 1], rows[T + 2] = [1, 2], [0], [2]
    S = csr_from_rows(rows, 3, "binary")
    R = csr_from_rows([[(0, 3.0), (1, 1.0), (2, 0.5)]], 3, "fp32")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    ids, sc = gpu_join(R, S, 1, tile=T, prune=1, alpha=1.0, counters=cnt, tiles_per_pass=2)
    assert ids.tolist() == [[0]] and abs(sc[0, 0] - 4.0) <= 1e-6
    c = cnt.cpu().tolist()
    assert c[2] == 2, c  # posting units of the skipped slices (f1, f2 in tile 1)
    assert c[3] == 1, c  # s3 completed
    ids_u, sc_u = gpu_join(R, S, 1, tile=T, head_density=-1.0)
    assert ids_u.tolist() == ids.tolist() and sc_u.tolist() == sc.tolist()
    # alpha small enough that N is empty in tile 1 (budget 0.25 * 4 = 1 < 1.5 but >= 0.5: N = {2})
    cnt.zero_()
    ids, sc = gpu_join(R, S, 1, tile=T, prune=1, alpha=0.25, counters=cnt, tiles_per_pass=2)
    assert ids.tolist() == [[0]]
    assert cnt.cpu().tolist()[2] == 1  # only the f2 slice of tile 1


@pytest.mark.parametrize("dtr,dts", [("binary", "binary"), ("int8", "int8"), ("fp32", "binary"), ("int8", "binary"),
                                     ("binary", "int8"), ("fp32", "int8")])
@pytest.mark.parametrize("k", [1, 5, 33, 256])
def test_random_small_multi_tile_pruned(dtr, dts, k):
    """Several tiles (2048) with a ragged tail, tie-heavy values, alpha in {0.25, 1}."""
    rng = np.random.default_rng(stable_seed("prune", dtr, dts, k))
    d = 300
    R = random_csr(rng, 37, d, 0, 40, dtr, vmax=4)
    S = random_csr(rng, 7000, d, 0, 30, dts, vmax=4)
    _pruned_equals_unpruned(R, S, k, 2048, (0.25, 1.0))


@pytest.mark.parametrize("name,n_r,n_s,tile", [("C1", 1000, 10000, 2048), ("C2", 300, 40000, 4096),
                                               ("C3", 200, 60000, 4096), ("C5", 60, 40000, 8192),
                                               ("C4", 150, 50000, 8192)])
def test_configs_scaled_pruned(name, n_r, n_s, tile):
    c = gen.CONFIGS[name].scaled(n_r, n_s)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    cnts = _pruned_equals_unpruned(R, S, c.k, tile, (0.25, 0.5, 1.0))
    if name in ("C2", "C3", "C4"):
        assert cnts[-1][2] > 0, "alpha = 1 skipped no posting unit"


def test_many_runs_and_chunks():
    """Rows with more runs than one staging chunk (256) and than the prep sort holds (2048: all essential)."""
    rng = np.random.default_rng(11)
    d = 5000
    rows = []
    for i in range(12):
        n = 3000 if i % 4 == 0 else int(rng.integers(300, 900))
        f = np.sort(rng.choice(d, size=n, replace=False))
        rows.append([(int(x), float(np.float32(rng.lognormal()))) for x in f])
    R = csr_from_rows(rows, d, "fp32")
    S = random_csr(rng, 9000, d, 10, 80, "binary")
    _pruned_equals_unpruned(R, S, 10, 2048, (0.5, 1.0))


def test_pruned_with_passes_split_resume():
    """Pruning combined with pass-major schedules, tile ranges + resume, and the small-R tile-group split."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS["C3"].scaled(64, 60000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
    ref = kj.knnjoin_build_index(dS, c.d, tile=2048, head_density=-1.0)
    idx = kj.knnjoin_build_index(dS, c.d, tile=2048, prune=1, alpha=0.5)
    i0, s0, _ = kj.knnjoin_query(ref, dR, c.k, tiles_per_pass=1)
    for kw in ({"tiles_per_pass": 1}, {"tiles_per_pass": 5}, {}):
        i1, s1, _ = kj.knnjoin_query(idx, dR, c.k, **kw)
        assert torch.equal(i0, i1) and torch.equal(s0, s1), kw
    nt = kj.knnjoin_index_stats(idx)["n_tiles"]
    a = nt // 3
    _, _, k1 = kj.knnjoin_query(idx, dR, c.k, want_keys=True, tile_range=(0, a))
    i2, s2, _ = kj.knnjoin_query(idx, dR, c.k, tile_range=(a, nt), resume_keys=k1)
    assert torch.equal(i0, i2) and torch.equal(s0, s2)
    # per-query override: off, and another alpha
    for pa in (-1.0, 1.0):
        i3, s3, _ = kj.knnjoin_query(idx, dR, c.k, prune_alpha=pa)
        assert torch.equal(i0, i3) and torch.equal(s0, s3)


def test_prune_argument_errors():
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS["C1"].scaled(20, 3000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
    plain = kj.knnjoin_build_index(dS, c.d)
    with pytest.raises(kj.KnnJoinError, match="prune"):
        kj.knnjoin_query(plain, dR, c.k, prune_alpha=0.5)
    pr = kj.knnjoin_build_index(dS, c.d, prune=1)
    assert kj.knnjoin_index_stats(pr)["prune"] == 1 and abs(kj.knnjoin_index_stats(pr)["alpha"] - 0.25) < 1e-7
    with pytest.raises(kj.KnnJoinError, match="one-row"):
        kj.knnjoin_query(pr, dR, c.k, batch_rows=2)
    with pytest.raises(kj.KnnJoinError, match="prune_alpha"):
        kj.knnjoin_query(pr, dR, c.k, prune_alpha=2.0)
    # an explicit one-row 4-warp shape is accepted; an unpruned query on a prune index is allowed
    kj.knnjoin_query(pr, dR, c.k, batch_rows=1, cta_warps=4)
    kj.knnjoin_query(pr, dR, c.k, prune_alpha=-1.0, batch_rows=2)


@pytest.mark.slow
@pytest.mark.parametrize("name,alphas", [("C2", (0.25, 1.0)), ("C3", (0.05, 0.25)), ("C5", (0.05,))])
def test_full_size_pruned_equals_unpruned(name, alphas):
    """Full BASELINE.json sizes: the pruned query equals the unpruned one on every row (the unpruned query is
    itself parity-checked against the oracle on sampled rows in test_gpu_parity.test_full_size_sampled_rows)."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS[name]
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
    ref = kj.knnjoin_build_index(dS, c.d, head_density=-1.0)
    i0, s0, _ = kj.knnjoin_query(ref, dR, c.k)
    del ref
    idx = kj.knnjoin_build_index(dS, c.d, prune=1)
    for a in alphas:
        i1, s1, _ = kj.knnjoin_query(idx, dR, c.k, prune_alpha=a)
        assert torch.equal(i0, i1) and torch.equal(s0, s1), a
    import os
    rows = np.sort(np.random.default_rng(5).choice(R.n_rows, 8, replace=False))
    o_ids, o_sc = oracle.knn(R, S, c.k, rows=rows, threads=max(1, min(8, len(os.sched_getaffinity(0)))))
    assert_parity(R.take_rows(rows), S, i1.cpu().numpy()[rows].astype(np.int64),
                  s1.cpu().numpy()[rows].astype(np.float64), o_ids, o_sc, rows=None)


def test_pruned_edge_cases():
    """Empty rows, R features >= d (ignored), k > #positives, empty S, one-posting slices."""
    d = 64
    R = csr_from_rows([[0, 1, 2], [], [63], [5, 6], [(0)]], d, "binary")
    S = csr_from_rows([[0], [], [1, 2, 3], [63], [7], [0, 1, 2, 5, 6]] * 700, d, "binary")
    for k in (1, 4, 7):
        _pruned_equals_unpruned(R, S, k, 2048, (0.25, 1.0))
    Rw = csr_from_rows([[0, 70, 80], [1, 2, 90]], 128, "binary")
    Sw = csr_from_rows([[0], [0, 1], [1, 2]] * 1000, 128, "binary")
    _pruned_equals_unpruned(Rw, Sw, 3, 2048, (0.5, 1.0), d=64, oracle_check=False)
    import paper_1011_2807_b200 as kj
    Sempty = csr_from_rows([], d, "binary")
    idx = kj.knnjoin_build_index(kj.DeviceCSR.from_host(Sempty), d, prune=1, alpha=1.0)
    ids, sc, _ = kj.knnjoin_query(idx, kj.DeviceCSR.from_host(R), 3)
    assert (ids == -1).all() and (sc == 0).all()
