"""Pins of the CPU oracle (oracle/oracle.c) against things other than itself.

Each test names the paper passage it follows.  None of these call the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import paper_algs as pa
from tests.util import csr_from_rows, random_csr, scipy_topk, stable_seed, to_scipy

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def test_dot_spec_examples():
    """SPEC.md:61-63 worked values of Eq. 1."""
    for ex in _gold("spec_examples.json")["dot"]:
        R = csr_from_rows([ex["r"]], 8)
        S = csr_from_rows([ex["s"]], 8)
        assert oracle.dot(R, 0, S, 0) == ex["expect"], ex["cite"]


@pytest.mark.parametrize("dtype", ["fp32", "int8", "binary"])
def test_dot_matches_dense_explicit_product(dtype):
    """Eq. 1 evaluated densely over all D coordinates (numpy) vs the merge dot of Alg. 2 l.8-23."""
    rng = np.random.default_rng(1)
    d = 50
    R = random_csr(rng, 30, d, 0, 20, dtype, vmax=9)
    S = random_csr(rng, 30, d, 0, 20, dtype, vmax=9)
    dense = lambda m, i: np.bincount(m.row(i)[0], weights=(np.ones(len(m.row(i)[0])) if m.values is None
                                                             else m.row(i)[1].astype(np.float64)), minlength=d)
    for i in range(R.n_rows):
        for j in range(S.n_rows):
            want = float(np.dot(dense(R, i), dense(S, j)))
            got = oracle.dot(R, i, S, j)
            assert got == pytest.approx(want, rel=1e-12, abs=0.0), (i, j)
            assert got == oracle.dot(S, j, R, i)  # symmetry


def test_dot_binary_is_support_intersection():
    """Binary vectors: Eq. 1 reduces to |supp r ∩ supp s| (set intersection closed form)."""
    rng = np.random.default_rng(2)
    R = random_csr(rng, 40, 60, 0, 30, "binary")
    S = random_csr(rng, 40, 60, 0, 30, "binary")
    for i in range(R.n_rows):
        for j in range(S.n_rows):
            assert oracle.dot(R, i, S, j) == len(set(R.row(i)[0]) & set(S.row(j)[0]))


def test_dot_advances_bounded_by_eq2():
    """Eq. 2: one merge costs at most |r|+|s| iterator advances."""
    rng = np.random.default_rng(3)
    R = random_csr(rng, 20, 40, 0, 20, "fp32")
    S = random_csr(rng, 20, 40, 0, 20, "fp32")
    for i in range(R.n_rows):
        for j in range(S.n_rows):
            _, adv = oracle.dot_with_advances(R, i, S, j)
            assert adv <= len(R.row(i)[0]) + len(S.row(j)[0])


def test_hand_example_ties_and_padding():
    """Hand-derived §3 example (tests/golden/hand_example.json): ties to the lower id, zero excluded."""
    g = _gold("hand_example.json")
    R = csr_from_rows(g["R"], g["d"], "binary")
    S = csr_from_rows(g["S"], g["d"], "binary")
    for j, want in enumerate(g["scores"]):
        assert oracle.dot(R, 0, S, j) == want
    for k, want in g["expect"].items():
        ids, sc = oracle.knn(R, S, int(k))
        assert [[int(a), int(b)] for a, b in zip(ids[0], sc[0])] == want


@pytest.mark.parametrize("dtype_r,dtype_s", [("binary", "binary"), ("int8", "int8"), ("fp32", "binary"),
                                             ("int8", "binary"), ("fp32", "int8"), ("fp32", "fp32")])
@pytest.mark.parametrize("k", [1, 3, 7, 40])
def test_knn_matches_scipy_spgemm_and_lexsort(dtype_r, dtype_s, k):
    """The oracle top-k == textbook SpGEMM R @ S.T followed by lexsort (score desc, id asc)."""
    rng = np.random.default_rng(stable_seed(dtype_r, dtype_s, k))
    d = 40
    R = random_csr(rng, 25, d, 0, 12, dtype_r, vmax=3)
    S = random_csr(rng, 60, d, 0, 12, dtype_s, vmax=3)
    ids, sc = oracle.knn(R, S, k)
    wids, wsc, M = scipy_topk(R, S, k)
    if "fp32" in (dtype_r, dtype_s):
        np.testing.assert_allclose(sc, wsc, rtol=1e-12, atol=0)
        # fp64 sums in a different order can differ by an ulp; ids must agree wherever the score gap is real
        for i in range(R.n_rows):
            for t in range(k):
                if ids[i, t] != wids[i, t]:
                    a, b = ids[i, t], wids[i, t]
                    assert abs(M[i, a] - M[i, b]) <= 1e-12 * max(M[i, a], M[i, b])
    else:
        np.testing.assert_array_equal(ids, wids)
        np.testing.assert_array_equal(sc, wsc)


def test_knn_edge_cases():
    """Empty S, empty rows, k > #positives (pad (-1, 0)), s_id_base offset, row subsets."""
    R = csr_from_rows([[0, 1], [], [5]], 8, "binary")
    S = csr_from_rows([[1], [0, 1], [7]], 8, "binary")
    ids, sc = oracle.knn(R, S, 4, s_id_base=100)
    assert ids.tolist() == [[101, 100, -1, -1], [-1] * 4, [-1] * 4]
    assert sc.tolist() == [[2, 1, 0, 0], [0] * 4, [0] * 4]
    Sempty = csr_from_rows([], 8, "binary")
    ids, sc = oracle.knn(R, Sempty, 2)
    assert (ids == -1).all() and (sc == 0).all()
    ids, sc = oracle.knn(R, S, 2, rows=[2, 0])
    assert ids.tolist() == [[-1, -1], [1, 0]]


@pytest.mark.parametrize("dtype_r,dtype_s", [("binary", "binary"), ("int8", "int8"), ("fp32", "binary"),
                                             ("fp32", "int8"), ("fp32", "fp32"), ("int8", "fp32")])
def test_pair_scores_match_scipy_matrix(dtype_r, dtype_s):
    """oracle_pair_scores (the x(.) of every fp32 parity check, reading c15) == the entries
    M[r, s] of the textbook SpGEMM M = R @ S.T (Eq. 1) for arbitrary (r, s) pairs, in any order
    and with repeats; s < 0 (padding) gives 0.  Integer inputs exactly; fp32 within fp64 summation rounding."""
    rng = np.random.default_rng(stable_seed("pairs", dtype_r, dtype_s))
    d = 70
    R = random_csr(rng, 30, d, 0, 25, dtype_r, vmax=9)
    S = random_csr(rng, 90, d, 0, 25, dtype_s, vmax=9)
    M = (to_scipy(R) @ to_scipy(S).T).toarray()
    rr = rng.integers(0, R.n_rows, size=2000)
    ss = rng.integers(-1, S.n_rows, size=2000)  # -1: padding position
    rr[:30], ss[:30] = np.arange(30), np.arange(30)  # the diagonal and repeats
    got = oracle.pair_scores(R, S, rr, ss)
    want = np.where(ss >= 0, M[rr, np.maximum(ss, 0)], 0.0)
    if "fp32" in (dtype_r, dtype_s):
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=0)
    else:
        np.testing.assert_array_equal(got, want)
    assert np.all(got[ss < 0] == 0.0)
    # the pairs of a GPU list carry global ids: assert_parity maps them back with s_id_base; the same oracle
    # top-k with s_id_base=1000 must give scores equal to pair_scores of (id - 1000)
    ids, sc = oracle.knn(R, S, 5, s_id_base=1000)
    loc = np.where(ids >= 0, ids - 1000, -1)
    np.testing.assert_array_equal(oracle.pair_scores(R, S, np.repeat(np.arange(R.n_rows), 5), loc.ravel()),
                                  sc.ravel())


def test_oracle_threads_split_rows_only():
    rng = np.random.default_rng(5)
    R = random_csr(rng, 37, 30, 0, 10, "int8")
    S = random_csr(rng, 80, 30, 0, 10, "int8")
    a = oracle.knn(R, S, 5, threads=1)
    b = oracle.knn(R, S, 5, threads=4)
    np.testing.assert_array_equal(a[0], b[0])
    np.testing.assert_array_equal(a[1], b[1])


# ---------------------------------------------------------------- paper algorithms (Alg. 1-4) as pins

def test_candidate_set_spec_examples():
    """SPEC.md:155-157 (Alg. 2 lines 5-7 with strict >)."""
    for ex in _gold("spec_examples.json")["candidate_insert"]:
        c = pa.CandidateSet(ex["k"])
        admitted = [c.offer(i, v) for i, v in enumerate(ex["inserts"])]
        assert sorted([e[0] for e in c.entries], reverse=True) == ex["expect_scores"], ex["cite"]
        assert c.prune_score == ex["expect_prune"], ex["cite"]
        if "expect_second_admitted" in ex:
            assert admitted[1] == ex["expect_second_admitted"]


def test_min_prune_score_spec_examples():
    """SPEC.md:165-167."""
    for ex in _gold("spec_examples.json")["min_prune_score"]:
        sets = []
        for scores in ex["set_scores"]:
            c = pa.CandidateSet(ex["k"])
            for i, v in enumerate(scores):
                c.offer(i, v)
            sets.append(c)
        assert pa.min_prune_score(sets) == ex["expect"], ex["cite"]


def test_iib_build_and_match_spec_examples():
    g = _gold("spec_examples.json")
    S = [[tuple(f) for f in s] for s in g["iib_build"]["S"]]
    c = pa.Counters()
    inv = pa.create_inverted_list_iib(list(enumerate(S)), c)
    assert {str(d): [list(p) for p in v] for d, v in inv.items()} == g["iib_build"]["expect_lists"]
    assert c.postings_built == g["iib_build"]["expect_postings_built"]
    m = g["iib_match"]
    c2 = pa.Counters()
    cands = {0: pa.CandidateSet(2)}
    A = pa.find_matches_iib(0, [tuple(f) for f in m["r"]], inv, cands, c2)
    assert {str(s): v for s, v in A.items()} == m["expect_A"]
    assert c2.postings_visited == m["expect_postings_visited"]


def test_iiib_split_spec_example():
    """maxWeight 1, MinPruneScore 5, weights 2,2,2 -> t = 2,4,6; only the third indexed."""
    ex = _gold("spec_examples.json")["iiib_split"]
    s = [(d, w) for d, w in enumerate(ex["weights_in_profile_order"])]
    Br = [(0, [(d, ex["max_weight"]) for d in range(len(s))])]  # equal counts -> dimension order 0,1,2
    c = pa.Counters()
    inv, res = pa.create_inverted_list_iiib([(0, s)], Br, ex["min_prune"], None, c)
    indexed = [d in inv for d in range(len(s))]
    assert indexed == ex["expect_indexed"]
    assert c.postings_built == sum(ex["expect_indexed"])
    assert res[0] == [(0, 2.0), (1, 2.0)]


def _as_lists(csr_out):
    return [[(int(s), v) for s, v in row] for row in csr_out]


@pytest.mark.parametrize("seed", range(12))
def test_bf_iib_iiib_and_oracle_agree_with_ids(seed):
    """Theorem 1: BF, IIB and IIIB under block nested loops return the same lists --
    ids included under reading c1 -- and all equal the oracle, on tie-heavy integer instances."""
    rng = np.random.default_rng(100 + seed)
    dtype = ["binary", "int8"][seed % 2]
    d = int(rng.integers(8, 30))
    R = random_csr(rng, int(rng.integers(1, 12)), d, 0, 8, dtype, vmax=3)
    S = random_csr(rng, int(rng.integers(1, 40)), d, 0, 8, dtype, vmax=3)
    k = int(rng.integers(1, 8))
    ids, sc = oracle.knn(R, S, k)
    want = [[(int(i), float(v)) for i, v in zip(ids[r], sc[r]) if i >= 0] for r in range(R.n_rows)]
    Rr, Sr = pa.rows_of(R), pa.rows_of(S)
    for alg in ("bf", "iib", "iiib"):
        for rb, sb in [(None, None), (3, 4), (1, 1), (5, 7)]:
            got, _ = pa.block_nested_loops_join(Rr, Sr, k, alg, rb, sb, D=d)
            got = [[(s, float(v)) for s, v in row] for row in got]
            assert got == want, (alg, rb, sb)


@pytest.mark.parametrize("seed", range(4))
def test_paper_algs_fp32_within_rounding(seed):
    rng = np.random.default_rng(300 + seed)
    d = 30
    R = random_csr(rng, 8, d, 1, 10, "fp32")
    S = random_csr(rng, 50, d, 1, 10, "binary")
    k = 4
    ids, sc = oracle.knn(R, S, k)
    for alg in ("bf", "iib", "iiib"):
        got, _ = pa.block_nested_loops_join(pa.rows_of(R), pa.rows_of(S), k, alg, 3, 9, D=d)
        for r in range(R.n_rows):
            gi = [s for s, _ in got[r]] + [-1] * (k - len(got[r]))
            gv = [v for _, v in got[r]] + [0.0] * (k - len(got[r]))
            np.testing.assert_allclose(gv, sc[r], rtol=1e-12)
            assert gi == ids[r].tolist()


def test_counter_laws_eq3_eq4():
    """Eq. 3: BF charges sum |r_i|+|s_j|; Eq. 4: IIB builds sum |s_i| postings and visits
    sum_r sum_j |I_{r[j].d}| = sum_d n_R(d) n_S(d)."""
    rng = np.random.default_rng(7)
    d = 25
    R = random_csr(rng, 9, d, 0, 10, "int8")
    S = random_csr(rng, 17, d, 0, 10, "int8")
    _, cbf = pa.block_nested_loops_join(pa.rows_of(R), pa.rows_of(S), 3, "bf")
    lr, ls = np.diff(R.indptr), np.diff(S.indptr)
    assert cbf.feature_visits == int(lr.sum() * S.n_rows + ls.sum() * R.n_rows)
    charged, adv = oracle.bf_counters(R, S)
    assert charged == cbf.feature_visits and adv == cbf.feature_advances
    _, ciib = pa.block_nested_loops_join(pa.rows_of(R), pa.rows_of(S), 3, "iib")
    assert ciib.postings_built == S.nnz
    nR = np.bincount(R.indices, minlength=d)
    nS = np.bincount(S.indices, minlength=d)
    assert ciib.postings_visited == int((nR * nS).sum())
    # SPEC.md:233 example
    ex = _gold("spec_examples.json")["bf_counters"]
    Rx = csr_from_rows([list(range(n)) for n in ex["r_sizes"]], 10, "binary")
    Sx = csr_from_rows([list(range(n)) for n in ex["s_sizes"]], 10, "binary")
    _, cx = pa.block_nested_loops_join(pa.rows_of(Rx), pa.rows_of(Sx), 1, "bf")
    assert cx.feature_visits == ex["expect_feature_visits"]


def test_iiib_split_soundness_and_fewer_postings():
    """residual bound sum maxWeight_d*w <= MinPruneScore; indexed ∪ residual = s;
    IIIB never indexes more than IIB."""
    rng = np.random.default_rng(11)
    for _ in range(200):
        d = 20
        Br = list(enumerate(pa.rows_of(random_csr(rng, 4, d, 1, 8, "int8", vmax=5))))
        Bs = list(enumerate(pa.rows_of(random_csr(rng, 6, d, 1, 8, "int8", vmax=5))))
        mp = float(rng.uniform(0.5, 20))
        c = pa.Counters()
        inv, res = pa.create_inverted_list_iiib(Bs, Br, mp, d, c)
        _, maxw = pa.frequency_profile(Br, d)
        for si, s in Bs:
            assert sum(maxw.get(dd, 0) * w for dd, w in res[si]) <= mp
            idx = sorted((dd, w) for dd, lst in inv.items() for sj, w in lst if sj == si)
            assert sorted(idx + res[si]) == sorted(s)
        assert c.postings_built <= sum(len(s) for _, s in Bs)


@pytest.mark.parametrize("dtype_r,dtype_s", [("binary", "binary"), ("int8", "int8"), ("fp32", "binary"),
                                             ("fp32", "int8"), ("fp32", "fp32")])
@pytest.mark.parametrize("k", [1, 4, 30])
def test_cpu_iib_equals_oracle(dtype_r, dtype_s, k):
    """The host IIB baseline (oracle/iib.c, Alg. 3) returns the oracle's lists: bit for bit on integer inputs
    (ids included, tie-heavy), within fp64 summation rounding on fp32 ones; its posting count is Eq. 4's second
    term sum_d n_R(d) n_S(d)."""
    rng = np.random.default_rng(stable_seed("iib", dtype_r, dtype_s, k))
    d = 60
    R = random_csr(rng, 30, d, 0, 20, dtype_r, vmax=3)
    S = random_csr(rng, 300, d, 0, 20, dtype_s, vmax=3)
    ids, sc, info = oracle.iib_knn(R, S, k, threads=3)
    o_ids, o_sc = oracle.knn(R, S, k)
    nR = np.bincount(R.indices, minlength=d).astype(np.int64)
    nS = np.bincount(S.indices, minlength=d).astype(np.int64)
    assert info["visits"] == int((nR * nS).sum())
    if "fp32" in (dtype_r, dtype_s):
        np.testing.assert_allclose(sc, o_sc, rtol=1e-12, atol=0)
        M = (to_scipy(R) @ to_scipy(S).T).toarray()
        for i in range(R.n_rows):
            for t in range(k):
                if ids[i, t] != o_ids[i, t]:
                    assert abs(M[i, ids[i, t]] - M[i, o_ids[i, t]]) <= 1e-12 * M[i, o_ids[i, t]]
    else:
        np.testing.assert_array_equal(ids, o_ids)
        np.testing.assert_array_equal(sc, o_sc)
