"""-m gpu: f1, the paper's IIIB (Alg. 4) run literally on the device (paper_1011_2807_b200.iiib):
per S block the S-side split by the R profile and MinPruneScore, an index of the indexed parts s'', and a
residual query that adds dot(r, s').  Results must pass the oracle parity rules and equal the IIB query bit
for bit; for integer inputs the number of indexed postings must equal the CPU literal IIIB of
oracle/paper_algs.py (same S blocks, R as one block) exactly."""
import numpy as np
import pytest
import torch

import gen
import oracle
from oracle import paper_algs as pa
from tests.gpu_util import assert_parity, gpu_join
from tests.util import csr_from_rows, random_csr, stable_seed

pytestmark = pytest.mark.gpu


def _iiib(R, S, k, s_block, d=None, tile=2048):
    import paper_1011_2807_b200 as kj
    from paper_1011_2807_b200.iiib import iiib_join
    d = d or R.d
    ids, sc, st = iiib_join(kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S), d, k, s_block, tile=tile)
    torch.cuda.synchronize()
    return ids.cpu().numpy().astype(np.int64), sc.cpu().numpy().astype(np.float64), st


def _check(R, S, k, s_block, tile=2048, cpu_counts=True):
    ids, sc, st = _iiib(R, S, k, s_block, tile=tile)
    o_ids, o_sc = oracle.knn(R, S, k, threads=8)
    assert_parity(R, S, ids, sc, o_ids, o_sc)
    ref = gpu_join(R, S, k, tile=tile, head_density=-1.0)
    np.testing.assert_array_equal(ids, ref[0], err_msg="IIIB ids differ from the IIB query")
    np.testing.assert_array_equal(sc, ref[1], err_msg="IIIB scores differ from the IIB query")
    if cpu_counts:
        _, c = pa.block_nested_loops_join(pa.rows_of(R), pa.rows_of(S), k, kernel="iiib", s_block=s_block, D=R.d)
        if R.dtype != "fp32":  # exact scores: the GPU split is the CPU split
            assert st["postings_built"] == c.postings_built, (st, c)
        else:  # the GPU lowers the threshold by a rounding margin: it may index more, never less
            assert st["postings_built"] >= c.postings_built, (st, c)
    assert st["postings_built"] <= st["postings_iib"]
    return st


def test_hand_example_blocks():
    """SURVEY.md §8(c) hand example (k = 2) with S in blocks of 2: the second block is split against
    MinPruneScore = 2 (the first block holds s0 (1), s1 (2)); result [(s4, 3), (s1, 2)]."""
    import json, os
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hand_example.json")))
    R = csr_from_rows(g["R"], g["d"], "binary")
    S = csr_from_rows(g["S"], g["d"], "binary")
    for k, want in g["expect"].items():
        for sb in (1, 2, 5):
            ids, sc, _ = _iiib(R, S, int(k), sb)
            assert [[int(a), int(b)] for a, b in zip(ids[0], sc[0])] == want, (k, sb)


@pytest.mark.parametrize("dtr,dts", [("binary", "binary"), ("int8", "int8"), ("int8", "binary"), ("binary", "int8"),
                                     ("fp32", "binary"), ("fp32", "int8")])
@pytest.mark.parametrize("k,s_block", [(1, 700), (5, 2500), (33, 1000)])
def test_random_blocks(dtr, dts, k, s_block):
    rng = np.random.default_rng(stable_seed("iiib", dtr, dts, k, s_block))
    d = 200
    R = random_csr(rng, 24, d, 0, 30, dtr, vmax=4)
    S = random_csr(rng, 6000, d, 0, 25, dts, vmax=4)
    _check(R, S, k, s_block)


@pytest.mark.parametrize("name,n_r,n_s,s_block", [("C1", 300, 10000, 2500), ("C2", 100, 20000, 5000),
                                                  ("C5", 30, 12000, 4000), ("C3", 60, 20000, 8192)])
def test_configs_scaled(name, n_r, n_s, s_block):
    c = gen.CONFIGS[name].scaled(n_r, n_s)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    st = _check(R, S, c.k, s_block, tile=4096, cpu_counts=name in ("C1", "C5"))
    assert st["blocks"] == (n_s + s_block - 1) // s_block


def test_edge_cases():
    d = 64
    R = csr_from_rows([[0, 1, 2], [], [63], [5, 6]], d, "binary")
    S = csr_from_rows([[0], [], [1, 2, 3], [63], [7]], d, "binary")
    for k in (1, 4, 7):
        for sb in (1, 2, 3, 10):
            _check(R, S, k, sb, cpu_counts=True)
    Sempty = csr_from_rows([], d, "binary")
    ids, sc, st = _iiib(R, Sempty, 3, 4)
    assert (ids == -1).all() and (sc == 0).all() and st["blocks"] == 0
