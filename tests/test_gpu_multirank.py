"""-m gpu: the multi-rank product path exercised functionally on a ONE-GPU box: two processes on cuda:0
joined by a gloo process group (host-staged collectives; no rank's kernels wait on another's).  NCCL over
NVLink replaces gloo on a multi-GPU box; the kernels, the all-gather + merge and the f2 floor protocol are the
same code.  Never used for a performance number."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import gen
from tests.gpu_util import gpu_join

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n_r, n_s, theta_tiles, q, hdr=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    sys.path.insert(0, ROOT)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_1011_2807_b200 as kj
        from paper_1011_2807_b200 import dist as kdist
        c = gen.CONFIGS[name].scaled(n_r, n_s)
        if hdr:
            from tests.test_gpu_precision import dynamic_range_case
            R, S = dynamic_range_case(n_r, n_s)
            lo, hi = kdist.shard_bounds(n_s, world, rank)
            S_shard = S.take_rows(np.arange(lo, hi))
            d, k = R.d, 10
        else:
            R = gen.generate(c, "R")
            lo, hi = kdist.shard_bounds(n_s, world, rank)
            S_shard = gen.generate(c, "S", lo, hi - lo)
            d, k = c.d, c.k
        st = {}
        ids, sc = kdist.dist_query(kj.DeviceCSR.from_host(S_shard), lo, kj.DeviceCSR.from_host(R), d, k,
                                   tile=2048, theta_tiles=theta_tiles, stats=st)
        torch.cuda.synchronize()
        q.put((rank, ids.cpu().numpy(), sc.cpu().numpy(), st.get("uncertified_rows", 0)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name,theta_tiles", [("C2", 0), ("C2", 1), ("C5", 2), ("C1", 1)])
def test_dist_query_two_ranks_one_gpu(name, theta_tiles):
    """dist.dist_query on 2 ranks (S shards with s_id_base, local top-k keys, all-gather, knnjoin_merge; with
    theta_tiles > 0 the f2 floor protocol) == one index over all of S, bit for bit, on every rank."""
    n_r, n_s = 80, 20000
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, n_r, n_s, theta_tiles, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    c = gen.CONFIGS[name].scaled(n_r, n_s)
    R, S = gen.generate(c, "R"), gen.generate(c, "S")
    ref_ids, ref_sc = gpu_join(R, S, c.k, tile=2048)
    for _, ids, sc, _ in res:
        np.testing.assert_array_equal(ids, ref_ids)
        np.testing.assert_array_equal(sc, ref_sc.astype(np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("theta_tiles", [0, 2])
def test_dist_query_certified_fallback_two_ranks(theta_tiles):
    """High-dynamic-range FP32 rows through dist.dist_query on 2 ranks: the merged 32-bit lists of some rows fail
    certification on every rank alike, those rows are recomputed at 64 bits on both shards and merged again; the
    result meets the 1e-5 rule against the oracle and equals the one-index (auto) result bit for bit (binary S:
    the same 64-bit scale on both shards)."""
    import oracle
    from tests.gpu_util import assert_parity
    from tests.test_gpu_precision import dynamic_range_case
    n_r, n_s, world = 40, 12000, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "C2", n_r, n_s, theta_tiles, q, True))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    R, S = dynamic_range_case(n_r, n_s)
    ref_ids, ref_sc = gpu_join(R, S, 10, tile=2048)
    o_ids, o_sc = oracle.knn(R, S, 10, threads=8)
    for _, ids, sc, n_unc in res:
        assert n_unc > 0
        assert_parity(R, S, ids.astype(np.int64), sc.astype(np.float64), o_ids, o_sc)
        np.testing.assert_array_equal(ids, ref_ids)
        np.testing.assert_array_equal(sc, ref_sc.astype(np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("extra", [[], ["--theta-tiles", "1"]])
def test_bench_two_ranks_gloo_one_gpu(extra):
    """bench.py's N>1 path (torchrun, 2 ranks, barrier + max-over-ranks timing, all-gather + merge inside the
    step) runs to completion and rank 0 prints one JSON line with n_gpus = 2."""
    env = dict(os.environ, KNNJOIN_BENCH_BACKEND="gloo", KNNJOIN_BENCH_DEVICE="0")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"), "--gpus", "2",
           "--steps", "2", "--warmup", "3", "--config", "C1", "--no-cpu-baseline"] + extra
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    j = json.loads(lines[0])
    assert j["n_gpus"] == 2 and j["value"] > 0 and j["scaling"] == "strong"
    assert j["config"]["S_rows_total"] == 10_000 and j["config"]["S_rows_this_rank"] == 5_000  # C1's S, split
    assert j["e2e"]["value"] > 0
