"""Multi-GPU KNN join over torch.distributed: S-sharded (one exchange) and R-sharded (none).

S-sharded: rank p of P owns the contiguous S rows [p*|S|/P, (p+1)*|S|/P) (global ids = s_id_base + local row),
builds its own index, computes the top-k keys of every r of the (replicated) R against its shard, and one
all-gather of the [|R|, k] uint64 keys (NCCL over NVLink on B200 boxes) brings every rank's lists together;
knnjoin_merge then merges the P sorted lists per row exactly (keys encode the total order of reading c1).  This
is Alg. 1's S blocks spread over GPUs: the top-k of r over S is the top-k of the union of its
per-block top-k lists.

FP32 R: the merged 32-bit fixed-point lists are certified (knnjoin_certify) -- identically on every
rank, since every rank merges the same gathered keys -- and the rows that fail are recomputed at 64-bit fixed
point on every shard and merged again (one more all-gather, only when some row failed).

f2 (cross-rank threshold, PAPER.md:161's pruneScore "derived from previous computation", extended across
ranks): the shard's tiles are swept in phases of theta_tiles tiles; after every phase one all_reduce(MAX) of the
rows' k-th keys gives every rank the floor below which no candidate can enter the global top-k.

R-sharded: every rank indexes all of S and answers its own contiguous rows of R; no collective at all.

The collective plumbing takes the local-keys and merge steps as callables so that it runs on CPU with the gloo
backend (tests/test_dist_cpu.py); ``dist_query`` / ``r_sharded_query`` wire in the CUDA library.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, equal-as-possible shard [lo, hi) of n_rows rows for `rank` of `world`."""
    lo = (n_rows * rank) // world
    hi = (n_rows * (rank + 1)) // world
    return lo, hi


def _host_staged(t: torch.Tensor, group) -> bool:
    return t.is_cuda and dist.get_backend(group) == "gloo"


def all_gather_keys(local_keys: torch.Tensor, group=None) -> torch.Tensor:
    """[n, k] int64 keys on every rank -> [world, n, k] (rank order).  Uses all_gather_into_tensor (one NCCL
    collective); backends without it (gloo) fall back to all_gather of a list."""
    world = dist.get_world_size(group)
    if _host_staged(local_keys, group):  # gloo: stage through host memory
        return all_gather_keys(local_keys.cpu(), group).to(local_keys.device)
    out = torch.empty((world,) + tuple(local_keys.shape), dtype=local_keys.dtype, device=local_keys.device)
    try:
        dist.all_gather_into_tensor(out, local_keys.contiguous(), group=group)
    except (RuntimeError, NotImplementedError):
        parts = [torch.empty_like(local_keys) for _ in range(world)]
        dist.all_gather(parts, local_keys.contiguous(), group=group)
        out = torch.stack(parts)
    return out


def all_reduce_max(t: torch.Tensor, group=None) -> torch.Tensor:
    """Element-wise MAX over ranks (int64 views of uint64 keys < 2^63 order like the keys)."""
    if _host_staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        return h.to(t.device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def rank_uniform_max(x: int, group=None, device=None) -> int:
    """max over ranks of a host integer (makes a protocol branch identical on every rank)."""
    dev = device if (device is not None and dist.get_backend(group) != "gloo") else "cpu"
    t = torch.tensor([int(x)], dtype=torch.int64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return int(t.item())


class Fallback:
    """The certification step of an S-sharded FP32-R join (the callables a caller provides):
    certify(result) -> device/host int32 [1 + n] list (count, rows) of rows whose merged 32-bit lists fail the
    tolerance rule; wide_keys(lst) -> [n, k] keys of those rows recomputed at 64 bits on this shard (other rows
    0); wide_merge(gathered [P, n, k], lst, result) -> result with the listed rows replaced."""

    def __init__(self, certify, wide_keys, wide_merge):
        self.certify, self.wide_keys, self.wide_merge = certify, wide_keys, wide_merge


def certified(result, fb: Fallback | None, group=None):
    if fb is None:
        return result, 0
    lst = fb.certify(result)
    cnt = rank_uniform_max(int(lst[0].item()), group)
    if cnt == 0:
        return result, 0
    return fb.wide_merge(all_gather_keys(fb.wide_keys(lst), group), lst, result), cnt


def sharded_join(local_keys_fn, merge_fn, group=None, fallback: Fallback | None = None):
    """local_keys_fn() -> [n, k] int64 keys of this rank's shard; merge_fn(gathered [P, n, k]) -> result."""
    keys = local_keys_fn()
    result = merge_fn(all_gather_keys(keys, group))
    return certified(result, fallback, group)[0]


def kth_floor(partial_keys: torch.Tensor, k: int, group=None) -> torch.Tensor:
    """f2: the k-th key every row reached on any shard.  Each rank's partial list holds k
    distinct keys >= its k-th key, so the global k-th key is >= the maximum over ranks: candidates below it can
    be dropped everywhere (keys are int64 views of uint64 keys < 2^63, so MAX is the key order)."""
    return all_reduce_max(partial_keys[:, k - 1].contiguous().clone(), group)


def sharded_join_theta(phase_fn, n_phases: int, merge_fn, k: int, group=None, fallback: Fallback | None = None):
    """S-sharded join with periodic cross-rank threshold sharing (f2): phase_fn(i, partial, floor) -> [n, k] keys
    of the local shard after phase i (partial = the lists after phase i-1 or None, floor = the rows' key floors
    from every rank after phase i-1 or None); one all_reduce(MAX) of the rows' k-th keys between phases;
    all-gather + merge as in sharded_join.  n_phases must be the same on every rank."""
    partial, floor = None, None
    for i in range(n_phases):
        partial = phase_fn(i, partial, floor)
        if i + 1 < n_phases:
            floor = kth_floor(partial, k, group)
    result = merge_fn(all_gather_keys(partial, group))
    return certified(result, fallback, group)[0]


def dist_query(S_shard, s_id_base: int, R, d: int, k: int, group=None, tile: int = 0, batch_rows: int = 0,
               cta_warps: int = 0, theta_tiles: int = 0, head_density: float = 0.0, index=None,
               tolerance: float = 0.0, stats: dict | None = None):
    """S-sharded product path on CUDA: every rank passes its S shard (DeviceCSR) and the full R (DeviceCSR).
    theta_tiles > 0 (more than one rank): f2 phases of theta_tiles tiles with a cross-rank floor after each.
    index: an already built index of S_shard (else built here).  Returns (ids int32 [n, k], scores float32
    [n, k]) -- identical on every rank.  stats (optional dict) receives 'uncertified_rows'."""
    from . import FP32, knnjoin_build_index, knnjoin_certify, knnjoin_index_stats, knnjoin_merge, knnjoin_query

    idx = index if index is not None else knnjoin_build_index(S_shard, d, s_id_base=s_id_base, tile=tile,
                                                             head_density=head_density)
    s_fp32 = S_shard.dtype == FP32
    # 32-bit lists everywhere (precision 1): the certification sees the merged lists (FP32 S: 64-bit throughout)
    kw = dict(want_keys=True, want_ids=False, batch_rows=batch_rows, cta_warps=cta_warps,
              precision=0 if s_fp32 else 1)
    n, dev = R.n_rows, R.indptr.device

    def merge(gathered):
        return knnjoin_merge(gathered, R, d, S_shard.dtype, k, want_keys=True)

    fb = None
    if R.dtype == FP32 and not s_fp32:
        def cert(result):
            return knnjoin_certify(result[2], R, d, S_shard.dtype, k, tolerance)

        def wide_keys(lst):
            keys = torch.zeros((n, k), dtype=torch.int64, device=dev)
            knnjoin_query(idx, R, k, want_keys=True, want_ids=False, precision=2, row_list=lst, out=(None, None, keys))
            return keys

        def wide_merge(gathered, lst, result):
            ids, scores, _ = result
            knnjoin_merge(gathered, R, d, S_shard.dtype, k, float_keys=1, row_list=lst, out=(ids, scores, None))
            return result

        fb = Fallback(cert, wide_keys, wide_merge)

    world = dist.get_world_size(group)
    if theta_tiles > 0 and world > 1:
        # rank-uniform phase count from the largest shard (a rank with fewer tiles runs empty ranges)
        n_tiles = knnjoin_index_stats(idx)["n_tiles"]
        n_phases = (rank_uniform_max(n_tiles, group, dev) + theta_tiles - 1) // theta_tiles
        n_phases = max(1, n_phases)

        def phase(i, partial, floor):
            a = min(i * theta_tiles, n_tiles)
            b = n_tiles if i == n_phases - 1 else min((i + 1) * theta_tiles, n_tiles)
            rng = (a, b) if b > 0 else (0, 0)
            return knnjoin_query(idx, R, k, tile_range=rng, resume_keys=partial, theta_in=floor, **kw)[2]

        result = sharded_join_theta(phase, n_phases, merge, k, group)
    else:
        result = merge(all_gather_keys(knnjoin_query(idx, R, k, **kw)[2], group))
    result, cnt = certified(result, fb, group)
    if stats is not None:
        stats["uncertified_rows"] = cnt
    return result[0], result[1]


def r_sharded_query(S, R_rows, d: int, k: int, index=None, tile: int = 0, **qkw):
    """R-sharded product path: every rank indexes all of S and queries only its own rows of R
    (R_rows = this rank's DeviceCSR rows, e.g. rows shard_bounds(|R|, P, rank) of R).  No collective: the join
    of R is the concatenation of the ranks' answers in rank order.  Returns (ids, scores) of R_rows."""
    from . import knnjoin_build_index, knnjoin_query
    idx = index if index is not None else knnjoin_build_index(S, d, tile=tile)
    ids, scores, _ = knnjoin_query(idx, R_rows, k, **qkw)
    return ids, scores
