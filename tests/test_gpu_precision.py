"""-m gpu: score precision -- certification of 32-bit fixed-point lists, the 64-bit fallback, FP32 S
(row a1) and 64-bit queries, all through the C ABI against the oracle (reading c15: 1e-5 relative).

The inputs that stress the 32-bit path are FP32 rows whose weights span five decades: one peak weight 1e5
(intensities "used directly") next to lognormal unit weights, with the peak feature present in fewer
than k rows of S, so most of each top-k list is made of neighbours that share only small-weight features."""
import numpy as np
import pytest
import torch

import gen
import oracle
from tests.gpu_util import assert_parity, gpu_join
from tests.util import csr_from_rows, random_csr, stable_seed

pytestmark = pytest.mark.gpu
PEAK = 1e5


def dynamic_range_case(n_r, n_s, s_dtype="binary", seed=0, d=2000, n_peaks=5, peak_rows=3):
    """Seeded input: R fp32 (60-120 lognormal weights + one peak feature of weight ~1e5), S (20-40 features,
    uniform), the peak features 0..n_peaks-1 each in exactly `peak_rows` rows of S."""
    rng = np.random.default_rng(stable_seed("dynrange", n_r, n_s, s_dtype, seed))
    rows = []
    for _ in range(n_r):
        c = int(rng.integers(60, 121))
        f = np.sort(rng.choice(np.arange(n_peaks, d), size=c, replace=False))
        feats = [(int(x), float(np.float32(rng.lognormal()))) for x in f]
        p = int(rng.integers(0, n_peaks))
        feats.append((p, float(np.float32(PEAK * rng.uniform(0.5, 2.0)))))
        rows.append(sorted(feats))
    R = csr_from_rows(rows, d, "fp32")
    holders = {p: set(rng.choice(n_s, size=peak_rows, replace=False).tolist()) for p in range(n_peaks)}
    srows = []
    for i in range(n_s):
        c = int(rng.integers(20, 41))
        f = sorted(rng.choice(np.arange(n_peaks, d), size=c, replace=False).tolist())
        f = sorted(f + [p for p in range(n_peaks) if i in holders[p]])
        if s_dtype == "binary":
            srows.append(f)
        elif s_dtype == "int8":
            srows.append([(x, int(rng.integers(1, 128))) for x in f])
        else:
            srows.append([(x, float(np.float32(rng.lognormal(0.0, 2.0)))) for x in f])
    S = csr_from_rows(srows, d, s_dtype)
    return R, S


def _oracle(R, S, k):
    return oracle.knn(R, S, k, threads=8)


def _unc(n):
    return torch.zeros(n + 1, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("s_dtype", ["binary", "int8"])
def test_dynamic_range_auto_meets_tolerance(s_dtype):
    """Auto precision: rows whose 32-bit lists cannot be certified are recomputed at 64 bits; every row then meets
    the 1e-5 rule against the oracle, and the certified rows are the 32-bit results bit for bit."""
    R, S = dynamic_range_case(48, 9000, s_dtype)
    k = 10
    unc = _unc(R.n_rows)
    ids, sc = gpu_join(R, S, k, tile=2048, uncertified=unc)
    o_ids, o_sc = _oracle(R, S, k)
    assert_parity(R, S, ids, sc, o_ids, o_sc)
    u = unc.cpu().numpy()
    flagged = set(u[1:1 + u[0]].tolist())
    assert len(flagged) > 0
    n_ids, n_sc = gpu_join(R, S, k, tile=2048, precision=1)
    keep = np.array([i for i in range(R.n_rows) if i not in flagged], dtype=np.int64)
    np.testing.assert_array_equal(ids[keep], n_ids[keep])
    np.testing.assert_array_equal(sc[keep], n_sc[keep])


@pytest.mark.parametrize("s_dtype", ["binary", "int8"])
def test_dynamic_range_certification_is_sound(s_dtype):
    """precision 1 (32-bit only) with `uncertified`: every row NOT flagged meets the 1e-5 rule on its own, and
    without the fallback some flagged row really breaks it (the certification is needed, not decorative)."""
    R, S = dynamic_range_case(48, 9000, s_dtype, seed=1)
    k = 10
    unc = _unc(R.n_rows)
    ids, sc = gpu_join(R, S, k, tile=2048, precision=1, uncertified=unc)
    o_ids, o_sc = _oracle(R, S, k)
    u = unc.cpu().numpy()
    flagged = set(u[1:1 + u[0]].tolist())
    assert flagged
    ok_rows = np.array([i for i in range(R.n_rows) if i not in flagged], dtype=np.int64)
    if len(ok_rows):
        assert_parity(R.take_rows(ok_rows), S, ids[ok_rows], sc[ok_rows], o_ids[ok_rows], o_sc[ok_rows],
                      rows=None)
    bad = 0
    for i in sorted(flagged):
        try:
            assert_parity(R.take_rows([i]), S, ids[[i]], sc[[i]], o_ids[[i]], o_sc[[i]], rows=None)
        except AssertionError:
            bad += 1
    assert bad > 0


def test_dynamic_range_zipf_with_head_features():
    """The 64-bit fallback on an index WITH head features (C2-shaped Zipf S): head postings are added from the
    per-row head q in the wide scan.  A rare S feature gets weight 1e5 in every R row."""
    c = gen.CONFIGS["C2"].scaled(40, 30000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    df = np.bincount(S.indices, minlength=c.d)
    f = int(np.nonzero((df >= 1) & (df <= 3))[0][0])
    rows = []
    for i in range(R.n_rows):
        idx, val = R.row(i)
        feats = {int(a): float(b) for a, b in zip(idx, val)}
        feats[f] = PEAK
        rows.append(sorted(feats.items()))
    R2 = csr_from_rows(rows, c.d, "fp32")
    unc = _unc(R2.n_rows)
    ids, sc = gpu_join(R2, S, c.k, uncertified=unc)
    assert int(unc[0]) > 0
    o_ids, o_sc = _oracle(R2, S, c.k)
    assert_parity(R2, S, ids, sc, o_ids, o_sc)
    w_ids, w_sc = gpu_join(R2, S, c.k, precision=2)
    assert_parity(R2, S, w_ids, w_sc, o_ids, o_sc)


def test_fp32_r_int8_s_high_nnz():
    """FP32 R (lognormal, 500-1000 nnz) x INT8 S (weights up to 127, 500-1000 nnz), k = 100 (the fixed-point scale
    reserves 127 per S weight, so 32-bit resolution is coarsest here)."""
    rng = np.random.default_rng(31)
    d = 5000
    R = random_csr(rng, 24, d, 500, 1000, "fp32")
    S = random_csr(rng, 5000, d, 500, 1000, "int8", vmax=127)
    ids, sc = gpu_join(R, S, 100, tile=2048)
    o_ids, o_sc = _oracle(R, S, 100)
    assert_parity(R, S, ids, sc, o_ids, o_sc)


@pytest.mark.parametrize("dtr", ["fp32", "int8", "binary"])
@pytest.mark.parametrize("k", [1, 5, 33, 256])
def test_fp32_s_random_multi_tile(dtr, k):
    """FP32 S (row a1), several tiles with a ragged tail: always 64-bit, every R dtype."""
    rng = np.random.default_rng(stable_seed("fp32s", dtr, k))
    d = 300
    R = random_csr(rng, 37, d, 0, 40, dtr, vmax=4)
    S = random_csr(rng, 5000, d, 0, 30, "fp32")
    cnt = torch.zeros(4, dtype=torch.int64, device="cuda")
    ids, sc = gpu_join(R, S, k, tile=2048, counters=cnt)
    o_ids, o_sc = _oracle(R, S, k)
    assert_parity(R, S, ids, sc, o_ids, o_sc)
    nR = np.bincount(R.indices, minlength=d).astype(np.int64)
    nS = np.bincount(S.indices, minlength=d).astype(np.int64)
    assert int(cnt[0]) == int((nR * nS).sum())  # Eq. 4 second term, exactly


def test_fp32_s_dynamic_range_and_precision_errors():
    """FP32 S with weights over six decades against the peaked R; precision 1 is refused for FP32 S."""
    import paper_1011_2807_b200 as kj
    R, S = dynamic_range_case(40, 8000, "fp32", seed=2)
    ids, sc = gpu_join(R, S, 10, tile=2048)
    o_ids, o_sc = _oracle(R, S, 10)
    assert_parity(R, S, ids, sc, o_ids, o_sc)
    with pytest.raises(kj.KnnJoinError, match="UNSUPPORTED"):
        gpu_join(R, S, 10, tile=2048, precision=1)
    with pytest.raises(kj.KnnJoinError):
        gpu_join(R, S, 10, tile=2048, prune=1)


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
def test_precision2_configs_scaled(name):
    """precision 2 (64-bit for every row) on the config laws: meets the rule; FP32-R configs agree with the 32-bit
    path on ids wherever the exact scores differ by more than the tolerance."""
    c = gen.CONFIGS[name].scaled(150, 25000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    ids, sc = gpu_join(R, S, c.k, precision=2)
    o_ids, o_sc = _oracle(R, S, c.k)
    assert_parity(R, S, ids, sc, o_ids, o_sc)


def test_wide_row_list_and_tile_groups():
    """A 64-bit query over a row list (the fallback's form): only listed rows are written; the first 64 listed
    rows are split into tile groups (merged by rank), later rows run whole -- both equal the all-rows query."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS["C2"].scaled(200, 40000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
    idx = kj.knnjoin_build_index(dS, c.d, tile=2048)
    full = kj.knnjoin_query(idx, dR, c.k, want_keys=True, precision=2)
    rows = np.array(sorted(np.random.default_rng(3).choice(R.n_rows, 90, replace=False)), np.int32)
    lst = torch.from_numpy(np.concatenate([[len(rows)], rows]).astype(np.int32)).cuda()
    ids = torch.full((R.n_rows, c.k), -7, dtype=torch.int32, device="cuda")
    sc = torch.full((R.n_rows, c.k), -7.0, dtype=torch.float32, device="cuda")
    keys = torch.zeros((R.n_rows, c.k), dtype=torch.int64, device="cuda")
    kj.knnjoin_query(idx, dR, c.k, precision=2, row_list=lst, out=(ids, sc, keys))
    torch.cuda.synchronize()
    ids, sc, keys = ids.cpu().numpy(), sc.cpu().numpy(), keys.cpu().numpy()
    other = np.setdiff1d(np.arange(R.n_rows), rows)
    assert (ids[other] == -7).all() and (sc[other] == -7.0).all() and (keys[other] == 0).all()
    for x, y in zip((full[0], full[1], full[2]), (ids, sc, keys)):
        np.testing.assert_array_equal(x.cpu().numpy()[rows], y[rows])


def test_wide_resume_chain_identical():
    """64-bit queries chained over tile ranges through resume_keys (fp32-keyed lists) == one query, bit for bit."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS["C3"].scaled(50, 15000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
    idx = kj.knnjoin_build_index(dS, c.d, tile=2048)
    NT = kj.knnjoin_index_stats(idx)["n_tiles"]
    full = kj.knnjoin_query(idx, dR, c.k, want_keys=True, precision=2)
    keys = None
    for rng in ((0, 2), (2, 2), (2, NT)):
        ids, sc, keys = kj.knnjoin_query(idx, dR, c.k, want_keys=True, precision=2, tile_range=rng, resume_keys=keys)
    torch.cuda.synchronize()
    for x, y in zip(full, (ids, sc, keys)):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())


def test_certify_api_matches_query_list():
    """knnjoin_certify on the 32-bit keys of a precision-1 query flags the same rows as the query's own list; the
    sharded protocol (shards -> merge -> certify -> 64-bit rows per shard -> float-key merge of the listed rows)
    meets the rule."""
    import paper_1011_2807_b200 as kj
    R, S = dynamic_range_case(40, 10000, "binary", seed=5)
    k = 10
    dR = kj.DeviceCSR.from_host(R)
    unc = _unc(R.n_rows)
    _, _, keys = gpu_join(R, S, k, tile=2048, precision=1, uncertified=unc, want_keys=True)
    lst = kj.knnjoin_certify(torch.from_numpy(keys).cuda(), dR, R.d, kj.BINARY, k)
    a, b = unc.cpu().numpy(), lst.cpu().numpy()
    assert a[0] == b[0] > 0 and set(a[1:1 + a[0]]) == set(b[1:1 + b[0]])
    half = S.n_rows // 2
    parts = [(0, S.take_rows(np.arange(0, half))), (half, S.take_rows(np.arange(half, S.n_rows)))]
    idxs = [kj.knnjoin_build_index(kj.DeviceCSR.from_host(p), R.d, s_id_base=base, tile=2048) for base, p in parts]
    narrow = torch.stack([kj.knnjoin_query(ix, dR, k, want_keys=True, want_ids=False, precision=1)[2] for ix in idxs])
    res = kj.knnjoin_merge(narrow, dR, R.d, kj.BINARY, k, want_keys=True)
    lst = kj.knnjoin_certify(res[2], dR, R.d, kj.BINARY, k)
    wide = []
    for ix in idxs:
        wk = torch.zeros((R.n_rows, k), dtype=torch.int64, device="cuda")
        kj.knnjoin_query(ix, dR, k, precision=2, row_list=lst, out=(None, None, wk))
        wide.append(wk)
    kj.knnjoin_merge(torch.stack(wide), dR, R.d, kj.BINARY, k, float_keys=1, row_list=lst, out=(res[0], res[1], None))
    torch.cuda.synchronize()
    o_ids, o_sc = _oracle(R, S, k)
    assert_parity(R, S, res[0].cpu().numpy().astype(np.int64), res[1].cpu().numpy().astype(np.float64), o_ids, o_sc)


def test_first_query_is_graph_capturable():
    """The auto shape is chosen on the device (both candidate launches gate on the index's head count), so even
    the FIRST query on a fresh index can be captured into a CUDA graph: no host synchronisation."""
    import paper_1011_2807_b200 as kj
    c = gen.CONFIGS["C2"].scaled(64, 20000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
    idx = kj.knnjoin_build_index(dS, c.d)
    torch.cuda.synchronize()
    ws = torch.empty(1 << 28, dtype=torch.uint8, device="cuda")
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            ids, sc, _ = kj.knnjoin_query(idx, dR, c.k, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    o_ids, o_sc = _oracle(R, S, c.k)
    assert_parity(R, S, ids.cpu().numpy().astype(np.int64), sc.cpu().numpy().astype(np.float64), o_ids, o_sc)


@pytest.mark.parametrize("hd", [0.0, 0.3])
def test_head_capable_index_without_heads(hd):
    """BINARY S with head features enabled: C1's uniform S has no feature with df >= |S|/8 (the head-free shape
    runs), C2's has (the 8-warp head shape runs); both gate on the device and give the oracle's lists."""
    for name in ("C1", "C2"):
        c = gen.CONFIGS[name].scaled(90, 12000)
        R, S = gen.generate(c, "R"), gen.generate(c, "S")
        ids, sc = gpu_join(R, S, c.k, head_density=hd)
        o_ids, o_sc = _oracle(R, S, c.k)
        assert_parity(R, S, ids, sc, o_ids, o_sc)


def test_streamed_and_iiib_joins_certified():
    """f4 (S streamed from host memory in blocks) and f1 (IIIB-literal) on the peaked rows: their final 32-bit
    lists are certified and the failing rows recomputed at 64 bits; both meet the rule against the oracle."""
    import paper_1011_2807_b200 as kj
    from paper_1011_2807_b200 import iiib, stream
    R, S = dynamic_range_case(30, 9001, "binary", seed=7)
    k = 10
    o_ids, o_sc = _oracle(R, S, k)
    st = {}
    pS = stream.PinnedS.from_host(S, block_rows=3001)
    ids, sc, _ = stream.streamed_join(pS, kj.DeviceCSR.from_host(R), R.d, k, tile=2048, stats=st)
    torch.cuda.synchronize()
    assert st["uncertified_rows"] > 0
    assert_parity(R, S, ids.cpu().numpy().astype(np.int64), sc.cpu().numpy().astype(np.float64), o_ids, o_sc)
    ids, sc, stats = iiib.iiib_join(kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S), R.d, k, s_block=4000,
                                    tile=2048)
    torch.cuda.synchronize()
    assert stats["uncertified_rows"] > 0
    assert_parity(R, S, ids.cpu().numpy().astype(np.int64), sc.cpu().numpy().astype(np.float64), o_ids, o_sc)


@pytest.mark.parametrize("dts", ["int8", "binary", "fp32"])
@pytest.mark.parametrize("k,n_r", [(1, 24), (10, 24), (10, 100)])
def test_wide_random_against_oracle(dts, k, n_r):
    """The 64-bit path alone (precision 2, FP32 R) on small random multi-tile inputs, all rows and a row list:
    fewer and more listed rows than the 64 that are split into tile groups."""
    import paper_1011_2807_b200 as kj
    rng = np.random.default_rng(stable_seed("wide", dts, k, n_r))
    d = 200
    R = random_csr(rng, n_r, d, 0, 30, "fp32")
    S = random_csr(rng, 6000, d, 0, 25, dts, vmax=4)
    o_ids, o_sc = _oracle(R, S, k)
    ids, sc = gpu_join(R, S, k, tile=2048, precision=2)
    assert_parity(R, S, ids, sc, o_ids, o_sc)
    rows = np.arange(1, n_r, 2, dtype=np.int32)
    lst = torch.from_numpy(np.concatenate([[len(rows)], rows]).astype(np.int32)).cuda()
    dR, dS = kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S)
    idx = kj.knnjoin_build_index(dS, d, tile=2048)
    g_ids = torch.full((n_r, k), -7, dtype=torch.int32, device="cuda")
    g_sc = torch.zeros((n_r, k), dtype=torch.float32, device="cuda")
    kj.knnjoin_query(idx, dR, k, precision=2, row_list=lst, out=(g_ids, g_sc, None))
    torch.cuda.synchronize()
    g_ids, g_sc = g_ids.cpu().numpy().astype(np.int64), g_sc.cpu().numpy().astype(np.float64)
    assert_parity(R.take_rows(rows), S, g_ids[rows], g_sc[rows], o_ids[rows], o_sc[rows], rows=None)
