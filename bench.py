"""bench.py -- |R|·|S| pairs/s of the B200 sparse KNN-join hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Default workload: C4 (BASELINE.json configs[3], the config the metric is quoted on "at 1/2/4/8 B200": |R| = 100 K
fp32 rows against |S| = 10 M binary rows, d = 10^4, k = 10).  A step is one pass of the whole hot path
 over that input: knnjoin_build_index(S) + knnjoin_query(R, k) -> ids + scores,
inputs already resident in HBM.  L2 is flushed (256 MiB write) before every timed step, outside the step's
event pair.  N>1 (torchrun, one rank per GPU, NCCL): STRONG scaling of the one S -- rank p owns the contiguous
rows shard_bounds(|S|, N, p), builds its shard's index, queries all of R; the ranks' top-k keys
are all-gathered (NCCL over NVLink) and merged (K4), the merged FP32-R lists certified (wide re-run of failing
rows); value = |R|·|S| / max-over-ranks time.

--impl reference times the CPU oracle (oracle/, the plain brute-force definition) on the host cores, on a
bounded row sample of the same workload per step (rank 0 only under torchrun).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

METRIC = "KNN-join |R|·|S| pairs/s and achieved HBM GB/s fraction at 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0
BAD_REASONS = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4", choices=sorted(gen.CONFIGS))
    ap.add_argument("--rows-r", type=int, default=0, help="profiling only: |R| override (same laws)")
    ap.add_argument("--rows-s", type=int, default=0, help="profiling only: |S| override (same laws)")
    ap.add_argument("--precision", type=int, default=0, help="0 auto (certified 32-bit), 1 32-bit, 2 64-bit")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--tile", type=int, default=0)
    ap.add_argument("--batch-rows", type=int, default=0)
    ap.add_argument("--cta-warps", type=int, default=0)
    ap.add_argument("--tiles-per-pass", type=int, default=0)
    ap.add_argument("--row-order", type=int, default=0, help="0 work-sorted (a3), 1 input order")
    ap.add_argument("--head-density", type=float, default=0.0, help="0 auto (1/8), <0 no head features")
    ap.add_argument("--head-max", type=int, default=0, help="0 auto (32)")
    ap.add_argument("--theta-tiles", type=int, default=0,
                    help="N>1: f2 cross-rank threshold every this many S tiles (0 = off)")
    ap.add_argument("--prune-alpha", type=float, default=0.0,
                    help="> 0: threshold-pruned queries (a6) with this alpha on an index built with prune=1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_desc(cfg, world):
    r, s = cfg.R, cfg.S
    law = {gen.UNIFORM: "uniform", gen.ZIPF: "Zipf", gen.BANDS: "5 Gaussian bands"}
    return (f"{cfg.name}: |R|={r.n_rows} {gen.VALUE_DTYPE[r.value_law]} x |S|={s.n_rows}"
            f"{' (split evenly over ' + str(world) + ' ranks)' if world > 1 else ''} "
            f"{gen.VALUE_DTYPE[s.value_law]}, d={cfg.d}, {law[s.feat_law]} features, k={cfg.k}")


def bench_config(args):
    cfg = gen.CONFIGS[args.config]
    if args.rows_r or args.rows_s:
        cfg = cfg.scaled(args.rows_r or None, args.rows_s or None)
    return cfg


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms during the timed region."""

    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={','.join(self.FIELDS)}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def recorded_traffic(cfg_name: str):
    """dram bytes per launch of the accumulate kernel from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(cfg_name)
    except Exception:
        return None


def visits_and_bytes(R, S, d):
    nR = np.bincount(R.indices[R.indices < d], minlength=d).astype(np.int64)
    nS = np.bincount(S.indices, minlength=d).astype(np.int64)
    V = int((nR * nS).sum())
    b_post = 2 if S.values is None else 3
    return V, b_post


def smem_roofline(id_visits, pairs, kernel_ms, clocks, sms):
    mhz = (clocks or {}).get("sm_mhz") or (clocks or {}).get("sm_max_mhz") or 1965.0
    peak = sms * 128 * mhz * 1e6 / 1e12  # TB/s
    alg = 4 * id_visits + 8 * pairs
    ach = alg / (kernel_ms * 1e-3) / 1e12
    # op-rate form: shared atomics and the dense scan are limited by wavefronts, not bytes; the measured chip-wide
    # rates of tools/microbench.cu on a B200 (profiles/r1k_microbench.txt, 1965 MHz): red.shared to random banks
    # 2.63e12 lane-ops/s (5.83e12 conflict-free), scan + zero-fill 4.63e12 pairs/s
    atom_rand, atom_cf, scan_rate = 2.63e12, 5.83e12, 4.63e12
    t_rand = (id_visits / atom_rand + pairs / scan_rate) * 1e3
    t_cf = (id_visits / atom_cf + pairs / scan_rate) * 1e3
    return {"bound": "smem", "achieved": ach, "peak": peak, "unit": "TB/s", "frac": ach / peak,
            "algorithmic_bytes": alg, "peak_source": f"derived: {sms} SMs x 128 B/clk x {mhz:.0f} MHz (sampled)",
            "op_bound_ms": {"random_banks": t_rand, "conflict_free": t_cf},
            "op_frac": {"random_banks": t_rand / kernel_ms, "conflict_free": t_cf / kernel_ms},
            "op_note": "id-list visits / measured shared-atomic rate + pairs / measured scan rate "
                       "(tools/microbench.cu, profiles/r1k_microbench.txt): the time the kernel's shared-memory "
                       "work alone needs; op_frac = that / kernel time"}


def head_visits(R, S, d, head_min_df, head_max=32):
    """Eq. 4 visits that fall on head features (their postings are encoded as per-row words, never loaded one
    by one): the first head_max features in (df desc, feature asc) order with df >= head_min_df (the index
    build's rule, csrc/index_build.cu k_head_select)."""
    if head_min_df < 0 or S.values is not None:
        return 0
    nR = np.bincount(R.indices[R.indices < d], minlength=d).astype(np.int64)
    nS = np.bincount(S.indices, minlength=d).astype(np.int64)
    order = np.lexsort((np.arange(d), -nS))[:head_max]
    heads = order[(nS[order] >= head_min_df) & (nS[order] > 0)]
    return int((nR[heads] * nS[heads]).sum())


# ------------------------------------------------------------------------------------ CPU legs
def run_oracle_sample(cfg, R, S, rows, threads):
    import oracle
    t0 = time.perf_counter()
    oracle.knn(R, S, cfg.k, rows=rows, threads=threads)
    return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_baseline(cfg, R, S, budget_s=15.0):
    """The oracle, as it stands, on a bounded row sample of the same workload, rows split over host threads;
    beside it the paper's own method (IIB, Alg. 3, oracle/iib.c) on the host, 1 thread and all threads."""
    import oracle
    cores = host_cores()
    rng = np.random.default_rng(1234)
    probe = rng.choice(R.n_rows, size=min(R.n_rows, cores), replace=False)
    t = run_oracle_sample(cfg, R, S, probe, cores)
    per_row = t / max(len(probe), 1) * cores  # seconds per row per thread
    n_rows = int(max(cores, min(R.n_rows, budget_s * cores / max(per_row, 1e-9))))
    rows = rng.choice(R.n_rows, size=n_rows, replace=False)
    t = run_oracle_sample(cfg, R, S, rows, cores)
    pairs = n_rows * S.n_rows
    # the same oracle on ONE core (1 core, then all cores), on a few rows of that sample
    n1 = int(max(1, min(n_rows, budget_s / 5.0 / max(per_row, 1e-9))))
    t1 = run_oracle_sample(cfg, R, S, rows[:n1], 1)
    out = {"value": pairs / t, "unit": "pairs/s", "cores": cores, "kind": "oracle",
           "sample": f"{n_rows} random rows of R x all {S.n_rows} rows of S ({pairs:.3e} pairs, {t:.1f} s), "
                     f"single-threaded C oracle per thread, rows split over {cores} host threads",
           "value_1core": n1 * S.n_rows / t1,
           "sample_1core": f"{n1} of those rows on one thread ({n1 * S.n_rows:.3e} pairs, {t1:.1f} s)"}
    # the paper's method on the host: IIB, index built once (timed apart)
    try:
        _, _, info = oracle.iib_knn(R, S, cfg.k, rows=rng.choice(R.n_rows, size=min(R.n_rows, 4 * cores),
                                                                  replace=False), threads=cores)
        per_row_iib = info["query_s"] / max(1, min(R.n_rows, 4 * cores)) * cores
        m = int(max(cores, min(R.n_rows, budget_s * cores / max(per_row_iib, 1e-9))))
        rows_i = rng.choice(R.n_rows, size=m, replace=False)
        _, _, info = oracle.iib_knn(R, S, cfg.k, rows=rows_i, threads=cores)
        m1 = int(max(1, min(m, budget_s / 3.0 / max(per_row_iib, 1e-9))))
        _, _, info1 = oracle.iib_knn(R, S, cfg.k, rows=rows_i[:m1], threads=1)
        out["iib"] = {"value": m * S.n_rows / info["query_s"], "unit": "pairs/s", "cores": cores,
                      "value_1core": m1 * S.n_rows / info1["query_s"],
                      "visits_per_s": info["visits"] / info["query_s"], "index_build_s": info["build_s"],
                      "kind": "paper's IIB (Alg. 3, PAPER.md:136-159) in plain C on the host (oracle/iib.c)",
                      "sample": f"{m} random rows of R x all {S.n_rows} rows of S on {cores} threads "
                                f"({info['query_s']:.1f} s); {m1} rows on one thread ({info1['query_s']:.1f} s); "
                                f"S indexed once ({info['build_s']:.1f} s, not in the rate)"}
    except MemoryError as e:  # pragma: no cover
        out["iib"] = {"unavailable": str(e)}
    return out


def bench_reference(args):
    rank, world, _ = dist_env()
    cfg = bench_config(args)
    if rank != 0:
        return
    R, S = gen.generate(cfg, "R"), gen.generate(cfg, "S", 0, cfg.S.n_rows)
    cores = host_cores()
    rng = np.random.default_rng(99)
    probe = rng.choice(R.n_rows, size=min(R.n_rows, cores), replace=False)
    t = run_oracle_sample(cfg, R, S, probe, cores)
    per_row = t / len(probe) * cores
    total_budget = 120.0
    steps = args.steps + args.warmup
    rows_per_step = int(max(cores, min(R.n_rows, total_budget / steps * cores / max(per_row, 1e-9))))
    times = []
    for i in range(steps):
        rows = rng.choice(R.n_rows, size=rows_per_step, replace=False)
        dt = run_oracle_sample(cfg, R, S, rows, cores)
        if i >= args.warmup:
            times.append(dt)
    pairs = rows_per_step * S.n_rows
    value = pairs * len(times) / sum(times)
    sample = (f"per step {rows_per_step} random rows of R x all {S.n_rows} rows of S ({pairs:.3e} pairs); "
              f"oracle rows split over {cores} host threads")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
           "dtype": "f64", "data": "synthetic",
           "config": {"workload": workload_desc(cfg, 1), "k": cfg.k, "seed": cfg.seed},
           "cpu_baseline": {"value": value, "unit": "pairs/s", "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": value, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------ GPU leg
def bench_ours(args):
    import torch
    import torch.distributed as dist

    rank, world, local = dist_env()
    if world != args.gpus:
        args.gpus = world
    # KNNJOIN_BENCH_BACKEND=gloo / KNNJOIN_BENCH_DEVICE=0: functional test of the multi-rank path on a one-GPU
    # box (tests/test_gpu_multirank.py) -- never used for a reported number
    backend = os.environ.get("KNNJOIN_BENCH_BACKEND", "nccl")
    if world > 1 and backend == "nccl":
        # NCCL's communicator-init lines (ranks, devices, NVLink / NVLS transports) go to stderr
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    dev_index = int(os.environ.get("KNNJOIN_BENCH_DEVICE", local))
    torch.cuda.set_device(dev_index)
    dev = torch.device("cuda", dev_index)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        print(f"[bench] rank {rank}/{world} on {torch.cuda.get_device_name(dev)} (cuda:{dev_index}), "
              f"backend {dist.get_backend()}", file=sys.stderr, flush=True)

    import paper_1011_2807_b200 as kj
    from paper_1011_2807_b200 import dist as kdist

    cfg = bench_config(args)
    n_s_total = cfg.S.n_rows
    lo, hi = kdist.shard_bounds(n_s_total, world, rank)
    R = gen.generate(cfg, "R")
    S = gen.generate(cfg, "S", lo, hi - lo)
    d, k = cfg.d, cfg.k
    V, b_post = visits_and_bytes(R, S, d)

    # index build options (a6 pruned mode: forward rows kept, head features off)
    bkw = dict(s_id_base=lo, tile=args.tile, head_density=args.head_density, head_max=args.head_max,
               prune=1 if args.prune_alpha > 0 else 0, alpha=args.prune_alpha if args.prune_alpha > 0 else 0.0)
    qkw = dict(batch_rows=args.batch_rows, cta_warps=args.cta_warps, tiles_per_pass=args.tiles_per_pass,
               row_order=args.row_order, prune_alpha=args.prune_alpha if args.prune_alpha > 0 else 0.0)
    stream = torch.cuda.current_stream()
    dR = kj.DeviceCSR.from_host(R, dev)
    dS = kj.DeviceCSR.from_host(S, dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    uncert = torch.zeros(R.n_rows + 1, dtype=torch.int32, device=dev)
    coll_ev = []  # (begin, end) events around the all-gather + merge (+ certification) of each timed step
    dstats = {}

    def step(dS_, dR_, kernel_events=None, build_event=None, before_query=None, coll_events=None):
        idx = kj.knnjoin_build_index(dS_, d, **bkw)
        if build_event is not None:
            build_event.record(stream)
        if before_query is not None:
            before_query()
        if world == 1:
            ids, sc, _ = kj.knnjoin_query(idx, dR_, k, events=kernel_events, precision=args.precision,
                                          uncertified=uncert, **qkw)
            return ids, sc
        # S-sharded: local 32-bit keys, NCCL all-gather, K4 merge, certification (+ 64-bit re-run of failing rows)
        if args.theta_tiles > 0:
            nt = kj.knnjoin_index_stats(idx)["n_tiles"]
            n_ph = max(1, (kdist.rank_uniform_max(nt, None, dev) + args.theta_tiles - 1) // args.theta_tiles)

            def phase(i, partial, floor):
                a = min(i * args.theta_tiles, nt)
                b = nt if i == n_ph - 1 else min((i + 1) * args.theta_tiles, nt)
                ev = kernel_events if i == n_ph - 1 else None
                return kj.knnjoin_query(idx, dR_, k, want_keys=True, want_ids=False, precision=1,
                                        tile_range=(a, b) if b > 0 else (0, 0), resume_keys=partial, theta_in=floor,
                                        events=ev, **qkw)[2]
            partial, floor = None, None
            for i in range(n_ph):
                partial = phase(i, partial, floor)
                if i + 1 < n_ph:
                    floor = kdist.kth_floor(partial, k)
            keys = partial
        else:
            keys = kj.knnjoin_query(idx, dR_, k, want_keys=True, want_ids=False, precision=1, events=kernel_events,
                                    **qkw)[2]
        if coll_events is not None:
            coll_events[0].record(stream)
        gathered = kdist.all_gather_keys(keys)  # one NCCL all_gather_into_tensor over NVLink
        result = kj.knnjoin_merge(gathered, dR_, d, dS_.dtype, k, want_keys=True)
        fb = None
        if dR_.dtype == kj.FP32 and dS_.dtype != kj.FP32:
            def cert(res):
                return kj.knnjoin_certify(res[2], dR_, d, dS_.dtype, k)

            def wide_keys(lst):
                wk = torch.zeros((R.n_rows, k), dtype=torch.int64, device=dev)
                kj.knnjoin_query(idx, dR_, k, want_keys=True, want_ids=False, precision=2, row_list=lst,
                                 out=(None, None, wk))
                return wk

            def wide_merge(g, lst, res):
                kj.knnjoin_merge(g, dR_, d, dS_.dtype, k, float_keys=1, row_list=lst, out=(res[0], res[1], None))
                return res
            fb = kdist.Fallback(cert, wide_keys, wide_merge)
        result, cnt = kdist.certified(result, fb)
        dstats["uncertified_rows"] = cnt
        if coll_events is not None:
            coll_events[1].record(stream)
        return result[0], result[1]

    for _ in range(args.warmup):
        step(dS, dR)
    torch.cuda.synchronize()

    # launch count of our kernels per step (one untimed profiled step; never inside the timed region)
    launches_per_step = None
    try:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            step(dS, dR)
            torch.cuda.synchronize()
        names = [e.name for e in prof.events() if e.device_type.name == "CUDA"]
        ours = [n for n in names if ("kj::" in n or "cub::" in n) and "Memset" not in n and "Memcpy" not in n]
        launches_per_step = len(ours)
    except Exception:
        launches_per_step = None

    # per-phase SM cycles and counters of the accumulate kernel (untimed instrumented queries)
    phase = torch.zeros(8, dtype=torch.int64, device=dev)
    idx_p = kj.knnjoin_build_index(dS, d, **bkw)
    kj.knnjoin_query(idx_p, dR, k, phase_cycles=phase, precision=1, **qkw)
    torch.cuda.synchronize()
    ph = phase.cpu().tolist()
    cnt = torch.zeros(4, dtype=torch.int64, device=dev)
    kj.knnjoin_query(idx_p, dR, k, counters=cnt, precision=1, uncertified=uncert, **qkw)
    torch.cuda.synchronize()
    n_uncert_local = int(uncert[0].item())
    counters = dict(zip(["postings_visited", "inserts", "head_postings_skipped", "head_completions"]
                        if args.prune_alpha <= 0 else
                        ["postings_visited", "inserts", "pruned_units_skipped", "pruned_completions"],
                        cnt.cpu().tolist()))
    tot_ph = max(1, sum(ph[:6]))
    phase_share = {n: round(ph[i] / tot_ph, 4) for i, n in
                   enumerate(["staging", "sparse_atomics", "unused", "scan_topk", "merge_output", "batch_setup_head_tables"])}
    stats = kj.knnjoin_index_stats(idx_p)
    del idx_p

    def timed_region():
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        kb = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ke = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        bd = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        cv = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for ev in kb + ke:  # materialise the cudaEvent handles; the library re-records them around its kernel
            ev.record(stream)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        sampler = ClockSampler(dev_index)
        sampler.start()
        time.sleep(0.05)
        for i in range(args.steps):
            flush.fill_(i & 0xFF)  # > L2 (126 MB): evict the previous step's index and inputs
            starts[i].record(stream)
            step(dS, dR, (kb[i], ke[i]), bd[i], coll_events=cv[i] if world > 1 else None)
            ends[i].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        clocks = sampler.stop()
        step_ms = [s_.elapsed_time(e_) for s_, e_ in zip(starts, ends)]
        kern_ms = [s_.elapsed_time(e_) for s_, e_ in zip(kb, ke)]
        build_ms.clear()
        build_ms.extend(s_.elapsed_time(e_) for s_, e_ in zip(starts, bd))
        coll_ms.clear()
        if world > 1:
            coll_ms.extend(a.elapsed_time(b) for a, b in cv)
        return step_ms, kern_ms, clocks

    build_ms, coll_ms = [], []

    step_ms, kern_ms, clocks = timed_region()
    if any(r in BAD_REASONS for r in clocks.get("reasons", [])):
        step_ms, kern_ms, clocks = timed_region()  # rejected: re-measure once
        clocks["remeasured"] = True
    total_ms = sum(step_ms)
    kern_avg = sum(kern_ms) / len(kern_ms)
    coll_avg = sum(coll_ms) / len(coll_ms) if coll_ms else 0.0
    t = torch.tensor([total_ms, kern_avg, coll_avg], dtype=torch.float64, device=dev)
    if world > 1:
        kdist.all_reduce_max(t)
    total_ms, kern_avg_max, coll_avg_max = float(t[0]), float(t[1]), float(t[2])
    ms_per_step = total_ms / args.steps
    pairs_per_step = R.n_rows * n_s_total
    value = pairs_per_step / (ms_per_step * 1e-3)

    # end to end: pinned host CSR -> device, build + query (+ gather/merge), result -> pinned host
    e2e = None
    if not args.no_e2e:
        hS = [torch.from_numpy(x).pin_memory() if x is not None else None for x in (S.indptr, S.indices, S.values)]
        hR = [torch.from_numpy(x).pin_memory() if x is not None else None for x in (R.indptr, R.indices, R.values)]
        h2d = sum(x.numel() * x.element_size() for x in hS + hR if x is not None)
        out_ids = torch.empty((R.n_rows, k), dtype=torch.int32).pin_memory()
        out_sc = torch.empty((R.n_rows, k), dtype=torch.float32).pin_memory()
        d2h = out_ids.numel() * 4 + out_sc.numel() * 4

        side = torch.cuda.Stream(dev)

        def e2e_step():
            # S's copy precedes the index build; R's copy runs on a side stream under the build
            dS2 = kj.DeviceCSR.from_arrays(hS[0], hS[1], hS[2], dev, non_blocking=True)
            side.wait_stream(stream)
            with torch.cuda.stream(side):
                dR2 = kj.DeviceCSR.from_arrays(hR[0], hR[1], hR[2], dev, non_blocking=True)
            for t_ in (dR2.indptr, dR2.indices, dR2.values):
                if t_ is not None:
                    t_.record_stream(stream)
            ids, sc = step(dS2, dR2, before_query=lambda: stream.wait_stream(side))
            out_ids.copy_(ids, non_blocking=True)
            out_sc.copy_(sc, non_blocking=True)

        for _ in range(2):
            e2e_step()
        torch.cuda.synchronize()
        n_e2e = max(3, min(args.steps, 20))
        if world > 1:
            dist.barrier()
        es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot = 0.0
        for i in range(n_e2e):
            flush.fill_(i & 0xFF)
            es.record(stream)
            e2e_step()
            ee.record(stream)
            ee.synchronize()
            tot += es.elapsed_time(ee)
        seq_ms = tot / n_e2e

        # pipelined: ONE timed region over n_e2e steps; step i+1's inputs are copied host->device on the side
        # stream (copy engine) while step i builds and queries; every step still copies all of its inputs, flushes
        # L2 (inside the region) and reads its ids/scores back to pinned host memory
        # two device slots for the inputs, allocated once (no allocator traffic inside the timed region); step i
        # uses slot i % 2, and the copies into a slot start only after the step that last read it was enqueued
        def dev_like(h):
            return kj.DeviceCSR(*(torch.empty_like(x, device=dev) if x is not None else None for x in h[:3]),
                                dS.dtype if h is hS else dR.dtype)
        slots = [(dev_like(hS), dev_like(hR)) for _ in range(2)]

        def copy_inputs(j):
            dS3, dR3 = slots[j % 2]
            with torch.cuda.stream(side):
                for c3, h3 in ((dS3, hS), (dR3, hR)):
                    for t3, x3 in zip((c3.indptr, c3.indices, c3.values), h3):
                        if t3 is not None:
                            t3.copy_(x3, non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(side)
            return dS3, dR3, ev

        def pipelined(n):
            nxt = copy_inputs(0)
            for i in range(n):
                dS3, dR3, ev = nxt
                stream.wait_event(ev)
                if i + 1 < n:
                    side.wait_stream(stream)  # slot (i+1) % 2 was last read by step i-1, already enqueued
                    nxt = copy_inputs(i + 1)
                flush.fill_(i & 0xFF)
                ids, sc = step(dS3, dR3)
                out_ids.copy_(ids, non_blocking=True)
                out_sc.copy_(sc, non_blocking=True)

        pipelined(2)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        side.wait_stream(stream)
        es.record(stream)
        side.wait_stream(stream)
        pipelined(n_e2e)
        ee.record(stream)
        ee.synchronize()
        pip_ms = es.elapsed_time(ee) / n_e2e
        tt = torch.tensor([pip_ms, seq_ms], dtype=torch.float64, device=dev)
        if world > 1:
            kdist.all_reduce_max(tt)
        e2e = {"value": pairs_per_step / (float(tt[0]) * 1e-3), "unit": "pairs/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": float(tt[0]), "steps": n_e2e,
               "path": "pinned host CSR -> cudaMemcpyAsync on a copy stream (step i+1's inputs under step i's "
                       "compute) -> knnjoin_build_index + knnjoin_query"
                       + (" + NCCL all-gather + knnjoin_merge + knnjoin_certify" if world > 1 else "")
                       + " -> pinned host ids/scores; one timed region over all steps, L2 flushed inside it before "
                         "every step" + ("; per rank: its S shard and all of R" if world > 1 else ""),
               "sequential_ms_per_step": float(tt[1]),
               "sequential_note": "each step alone (events around it, synchronised): S copied before the build, "
                                  "R on a side stream under the build"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    peak, peak_src = measured_peak()
    # Roofline of K3.  The graded bytes are what the kernel must LOAD with this index encoding:
    # the id-list postings it streams one by one ((V - head visits) x B_post) plus the 32-bit head words it reads
    # per (batch, S row); head postings are bounded/completed from those words, never loaded one by one.  The
    # logical Eq. 4 figure V x B_post (every posting as an id) is kept beside it.
    Vh = head_visits(R, S, d, stats["head_min_df"], stats["head_max"] or 32)
    touched = (V - Vh) * b_post
    n_batches_est = None
    if Vh:
        bsz = args.batch_rows or 2  # the auto shape for an index with head features (pick_shape: B=2 at T=8192)
        n_batches_est = (R.n_rows + bsz - 1) // bsz
        touched += n_batches_est * stats["n_tiles"] * stats["tile"] * 4
    if args.prune_alpha > 0:  # a6: posting units whose loads were skipped (8 postings each, padding included)
        touched = max(0, touched - counters["pruned_units_skipped"] * 8 * b_post)
    achieved = touched / (kern_avg_max * 1e-3) / 1e9
    props = torch.cuda.get_device_properties(dev)
    traffic = recorded_traffic(cfg.name if not (args.rows_r or args.rows_s) else None)
    out = {
        "metric": METRIC, "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong",  # one S split over the ranks (C4: 1/2/4/8); N = 1 is the curve's first point
        "vs_baseline": None, "dtype": "i32", "data": "synthetic",
        "config": {"workload": workload_desc(cfg, world), "k": k, "d": d, "seed": cfg.seed,
                   "R_rows": R.n_rows, "S_rows_total": n_s_total, "S_rows_this_rank": hi - lo,
                   "nnz_R": int(R.nnz), "nnz_S_rank0": int(S.nnz), "tile": stats["tile"],
                   "n_tiles_rank0": stats["n_tiles"], "batch_rows": args.batch_rows or "auto",
                   "head_min_df": stats["head_min_df"], "head_max": stats["head_max"],
                   "precision": {0: "auto (32-bit fixed point, certified; failing rows at 64 bits)",
                                 1: "32-bit fixed point", 2: "64-bit fixed point"}[args.precision],
                   **({"prune_alpha": args.prune_alpha} if args.prune_alpha > 0 else {}),
                   "step": "knnjoin_build_index(S) + knnjoin_query(R,k)" + (
                       " + all_gather + knnjoin_merge + knnjoin_certify" if world > 1 else ""),
                   "l2": "flushed before every timed step (256 MiB write, outside the step's events)",
                   "parallelism": f"S-sharded x{world} (strong scaling of one S)" if world > 1 else "1 GPU",
                   **({"theta_tiles": args.theta_tiles, "dist_backend": backend} if world > 1 else {}),
                   "sms": props.multi_processor_count, "l2_bytes": getattr(props, "L2_cache_size", None)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic,
                     "kernel": "k_accumulate_topk", "kernel_ms": kern_avg_max,
                     "algorithmic_bytes": touched, "peak_source": peak_src,
                     "bytes_note": "encoding-aware posting bytes per launch: id-list postings loaded one by one "
                                   "((V - head visits) x B_post) + 4-byte head words read per (batch, S row); most "
                                   "are L2 hits (pass slabs of the index are sized to stay in L2), so `traffic` "
                                   "(ncu dram bytes per launch) is far below them",
                     "visits": V, "head_visits": Vh, "bytes_per_visit": b_post,
                     "logical_bytes": V * b_post, "logical_gbs": V * b_post / (kern_avg_max * 1e-3) / 1e9,
                     "logical_frac": V * b_post / (kern_avg_max * 1e-3) / 1e9 / peak,
                     "logical_note": "Eq. 4 (PAPER.md:131) posting visits x B_post as if every posting were an "
                                     "id loaded one by one (SURVEY.md §8(d)); can exceed HBM peak"},
        # co-bound of the one-row, short-slice configs (C1/C3/C5): shared memory.  Algorithmic shared-memory
        # bytes of K3 = one 4-byte atomic per id-list visit + 8 bytes per pair (scan read + zero-fill) against
        # 148 SMs x 128 B/clk at the measured SM clock (no measured smem peak exists in MEASURED_PEAKS.json)
        "smem_roofline": smem_roofline(V - Vh, R.n_rows * (hi - lo), kern_avg_max, clocks,
                                       props.multi_processor_count),
        "clocks": clocks,
        "gpu_launches": (launches_per_step * args.steps) if launches_per_step is not None else None,
        "breakdown": {"kernel_ms": kern_avg_max, "step_ms": ms_per_step,
                      "build_index_ms": sum(build_ms) / len(build_ms),
                      # a2 reported separately: postings of S indexed per second
                      "build_postings_per_s": int(S.nnz) / (sum(build_ms) / len(build_ms) * 1e-3),
                      "query_prep_ms": ms_per_step - kern_avg_max - sum(build_ms) / len(build_ms) - coll_avg_max,
                      **({"allgather_merge_certify_ms": coll_avg_max,
                          "uncertified_rows": dstats.get("uncertified_rows")} if world > 1 else {}),
                      "other_ms": ms_per_step - kern_avg_max, "launches_per_step": launches_per_step,
                      "uncertified_rows_32bit": n_uncert_local,
                      "kernel_phase_share": phase_share, "counters": counters},
    }
    if e2e is not None:
        out["e2e"] = e2e
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, R, S)
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        bench_reference(args)
    else:
        bench_ours(args)


if __name__ == "__main__":
    main()
