"""-m gpu: the checks compute-sanitizer would make (T9), done without it (the tool is not allowed on this
GPU pool):
  * initcheck -> every device buffer the library reads but does not own the contents of (index storage, build and
    query workspaces) is pre-poisoned with 0xAB / 0xFF bytes; the results must equal a run on zeroed buffers and the
    oracle -- a read of an uninitialised byte would change them;
  * memcheck  -> the checked build (tools/checked_build.sh, -DKJ_CHECKS: a bounds check on every shared / global
    index the kernels form, trap on failure) runs every kernel path of tools/sanitize_cases.py;
  * racecheck -> the checked build's persistent grids capped at 1, 3 and 17 CTAs (KNNJOIN_MAX_CTAS) give results
    bit-identical to the full grid on integer inputs (any schedule-dependent race would show up as a difference)."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import gen
import oracle
from tests.gpu_util import assert_parity

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "ab_libs", "checked", "libknnjoin.so")


def _run(R, S, k, fill, tile=2048, **qkw):
    import paper_1011_2807_b200 as kj
    dS, dR = kj.DeviceCSR.from_host(S), kj.DeviceCSR.from_host(R)
    storage = torch.full((1 << 27,), fill[0], dtype=torch.uint8, device="cuda")
    bws = torch.full((1 << 27,), fill[1], dtype=torch.uint8, device="cuda")
    qws = torch.full((1 << 28,), fill[1], dtype=torch.uint8, device="cuda")
    idx = kj.knnjoin_build_index(dS, S.d, tile=tile, storage=storage, workspace=bws)
    ids, sc, keys = kj.knnjoin_query(idx, dR, k, want_keys=True, workspace=qws, **qkw)
    torch.cuda.synchronize()
    return ids.cpu().numpy(), sc.cpu().numpy(), keys.cpu().numpy()


@pytest.mark.parametrize("name,qkw", [("C2", {}), ("C5", {}), ("C3", {"tiles_per_pass": 1}), ("C1", {}),
                                      ("C2", {"precision": 2})])
def test_poisoned_buffers_change_nothing(name, qkw):
    c = gen.CONFIGS[name].scaled(50, 12000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    a = _run(R, S, c.k, (0x00, 0x00), **qkw)
    b = _run(R, S, c.k, (0xAB, 0xFF), **qkw)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x, y)
    o_ids, o_sc = oracle.knn(R, S, c.k, threads=8)
    assert_parity(R, S, a[0].astype(np.int64), a[1].astype(np.float64), o_ids, o_sc)


def _checked(args, env_extra=None, timeout=900):
    env = dict(os.environ, KNNJOIN_LIB=CHECKED, **(env_extra or {}))
    return subprocess.run([sys.executable] + args, capture_output=True, text=True, cwd=ROOT, env=env, timeout=timeout)


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build absent (tools/checked_build.sh)")
def test_checked_build_every_kernel_path():
    r = _checked([os.path.join(ROOT, "tools", "sanitize_cases.py")])
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "KJ_CHECK failed" not in r.stdout + r.stderr
    assert r.stdout.count(": ok") >= 11


_SCHED = r"""
import sys, numpy as np, torch, gen
import paper_1011_2807_b200 as kj
out = []
for name, kw in (("C1", {}), ("C5", {}), ("C2", {"tiles_per_pass": 1}), ("C2", {})):
    c = gen.CONFIGS[name].scaled(40, 9000)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    idx = kj.knnjoin_build_index(kj.DeviceCSR.from_host(S), c.d, tile=2048)
    _, _, keys = kj.knnjoin_query(idx, kj.DeviceCSR.from_host(R), c.k, want_keys=True, want_ids=False, **kw)
    torch.cuda.synchronize()
    out.append(keys.cpu().numpy())
np.save(sys.argv[1], np.concatenate([o.ravel() for o in out]))
"""


@pytest.mark.skipif(not os.path.exists(CHECKED), reason="checked build absent (tools/checked_build.sh)")
def test_schedule_independence(tmp_path):
    res = {}
    for cap in ("0", "1", "3", "17"):
        f = str(tmp_path / f"k{cap}.npy")
        r = _checked(["-c", _SCHED, f], {"KNNJOIN_MAX_CTAS": cap} if cap != "0" else None)
        assert r.returncode == 0, r.stderr[-3000:]
        res[cap] = np.load(f)
    for cap in ("1", "3", "17"):
        np.testing.assert_array_equal(res[cap], res["0"])
