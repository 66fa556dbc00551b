"""Small invocations of every kernel path, for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [case ...]

Cases (scaled configs, a few tiles each): c1 (binary, one-row CTAs, device-side shape gate), c2 (head features,
8-warp two-row CTAs), c5 (int8, k = 100), prune (a6 pruned query), passes (pass-major, top-k carried between
passes), split (small R: tile groups + rank merge), wide (FP32 S, 64-bit path, tile groups), fallback (certified
32-bit lists + 64-bit re-run), merge (S-sharded merge + certify), iiib (f1), validate.  Each case checks its
result against the oracle, so a sanitizer run also proves the instrumented run computed the right answer."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import gen  # noqa: E402
import oracle  # noqa: E402
import paper_1011_2807_b200 as kj  # noqa: E402
from tests.gpu_util import assert_parity, gpu_join  # noqa: E402


def check(R, S, k, **kw):
    ids, sc = gpu_join(R, S, k, **kw)
    o_ids, o_sc = oracle.knn(R, S, k, threads=8)
    assert_parity(R, S, ids, sc, o_ids, o_sc)


def scaled(name, n_r, n_s):
    c = gen.CONFIGS[name].scaled(n_r, n_s)
    return c, gen.generate(c, "R"), gen.generate(c, "S")


def case_c1():
    c, R, S = scaled("C1", 40, 5000)
    check(R, S, c.k, tile=2048)


def case_c2():
    c, R, S = scaled("C2", 40, 5000)
    check(R, S, c.k, tile=2048)


def case_c5():
    c, R, S = scaled("C5", 8, 4500)
    check(R, S, c.k, tile=2048)


def case_prune():
    c, R, S = scaled("C3", 30, 5000)
    check(R, S, c.k, tile=2048, prune=1, prune_alpha=0.5)


def case_passes():
    c, R, S = scaled("C2", 40, 7000)
    check(R, S, c.k, tile=2048, tiles_per_pass=1)


def case_split():
    c, R, S = scaled("C2", 6, 7000)
    check(R, S, c.k, tile=2048)


def case_wide():
    from tests.util import random_csr
    rng = np.random.default_rng(3)
    R = random_csr(rng, 20, 200, 0, 30, "fp32")
    S = random_csr(rng, 5000, 200, 0, 25, "fp32")
    check(R, S, 10, tile=2048)


def case_fallback():
    from tests.test_gpu_precision import dynamic_range_case
    R, S = dynamic_range_case(12, 5000)
    unc = torch.zeros(R.n_rows + 1, dtype=torch.int32, device="cuda")
    check(R, S, 10, tile=2048, uncertified=unc)
    assert int(unc[0]) > 0


def case_merge():
    c, R, S = scaled("C2", 20, 6000)
    dR = kj.DeviceCSR.from_host(R)
    half = S.n_rows // 2
    keys = []
    for lo, hi in ((0, half), (half, S.n_rows)):
        idx = kj.knnjoin_build_index(kj.DeviceCSR.from_host(S.take_rows(np.arange(lo, hi))), c.d, s_id_base=lo,
                                     tile=2048)
        keys.append(kj.knnjoin_query(idx, dR, c.k, want_keys=True, want_ids=False, precision=1)[2])
    ids, sc, mk = kj.knnjoin_merge(torch.stack(keys), dR, c.d, kj.BINARY, c.k, want_keys=True)
    lst = kj.knnjoin_certify(mk, dR, c.d, kj.BINARY, c.k)
    torch.cuda.synchronize()
    o_ids, o_sc = oracle.knn(R, S, c.k, threads=8)
    assert_parity(R, S, ids.cpu().numpy().astype(np.int64), sc.cpu().numpy().astype(np.float64), o_ids, o_sc)
    assert int(lst[0]) == 0


def case_iiib():
    from paper_1011_2807_b200.iiib import iiib_join
    c, R, S = scaled("C1", 30, 5000)
    ids, sc, _ = iiib_join(kj.DeviceCSR.from_host(R), kj.DeviceCSR.from_host(S), c.d, c.k, s_block=2000, tile=2048)
    torch.cuda.synchronize()
    o_ids, o_sc = oracle.knn(R, S, c.k, threads=8)
    np.testing.assert_array_equal(ids.cpu().numpy(), o_ids)


def case_validate():
    ok = kj.DeviceCSR.from_arrays(np.array([0, 2, 3]), np.array([1, 4, 0]), np.array([1.0, 2.0, 3.0], np.float32))
    assert kj.knnjoin_validate_csr(ok, 8) == (0, -1)


CASES = {n[5:]: f for n, f in globals().items() if n.startswith("case_")}

if __name__ == "__main__":
    names = sys.argv[1:] or list(CASES)
    for n in names:
        CASES[n]()
        torch.cuda.synchronize()
        print(f"case {n}: ok", flush=True)
