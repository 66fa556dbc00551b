"""S-sharded multi-GPU KNN join over torch.distributed.

Rank p of P owns the contiguous S rows [p*|S|/P, (p+1)*|S|/P) (global ids = s_id_base + local row), builds
its own index, computes the top-k keys of every r of the (replicated) R against its shard, and one
all-gather of the [|R|, k] uint64 keys (NCCL over NVLink on B200 boxes) brings every rank's lists together;
knnjoin_merge then merges the P sorted lists per row exactly (keys encode the total order of reading c1).

The collective plumbing takes the local-keys and merge steps as callables so that it can be exercised on
CPU with the gloo backend (tests/test_dist_cpu.py); ``dist_query`` wires in the CUDA library.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n_rows: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, equal-as-possible shard [lo, hi) of n_rows rows for `rank` of `world`."""
    lo = (n_rows * rank) // world
    hi = (n_rows * (rank + 1)) // world
    return lo, hi


def all_gather_keys(local_keys: torch.Tensor, group=None) -> torch.Tensor:
    """[n, k] int64 keys on every rank -> [world, n, k] (rank order).  Uses all_gather_into_tensor (one NCCL
    collective); backends without it (gloo) fall back to all_gather of a list."""
    world = dist.get_world_size(group)
    if local_keys.is_cuda and dist.get_backend(group) == "gloo":  # gloo: stage through host memory
        return all_gather_keys(local_keys.cpu(), group).to(local_keys.device)
    out = torch.empty((world,) + tuple(local_keys.shape), dtype=local_keys.dtype, device=local_keys.device)
    try:
        dist.all_gather_into_tensor(out, local_keys.contiguous(), group=group)
    except (RuntimeError, NotImplementedError):
        parts = [torch.empty_like(local_keys) for _ in range(world)]
        dist.all_gather(parts, local_keys.contiguous(), group=group)
        out = torch.stack(parts)
    return out


def sharded_join(local_keys_fn, merge_fn, group=None):
    """local_keys_fn() -> [n, k] int64 keys of this rank's shard; merge_fn(gathered [P, n, k]) -> result."""
    keys = local_keys_fn()
    gathered = all_gather_keys(keys, group)
    return merge_fn(gathered)


def kth_floor(partial_keys: torch.Tensor, k: int, group=None) -> torch.Tensor:
    """f2: the k-th key every row reached on any shard.  Each rank's partial list holds k
    distinct keys >= its k-th key, so the global k-th key is >= the maximum over ranks: candidates below it can
    be dropped everywhere (keys are int64 views of uint64 keys < 2^63, so MAX is the key order)."""
    floor = partial_keys[:, k - 1].contiguous().clone()
    if floor.is_cuda and dist.get_backend(group) == "gloo":  # gloo: stage through host memory
        h = floor.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MAX, group=group)
        return h.to(floor.device)
    dist.all_reduce(floor, op=dist.ReduceOp.MAX, group=group)
    return floor


def sharded_join_theta(phase1_fn, phase2_fn, merge_fn, k: int, group=None):
    """Two-phase S-sharded join with cross-rank threshold sharing (f2; PAPER.md:161's threshold "derived from
    previous computation", extended across ranks): phase1_fn() -> [n, k] keys over the first part of the
    local shard; one all_reduce(MAX) of the rows' k-th keys; phase2_fn(partial, floor) -> [n, k] keys of the
    whole local shard, keeping only keys >= floor from the rest; all-gather + merge as in sharded_join."""
    partial = phase1_fn()
    floor = kth_floor(partial, k, group)
    keys = phase2_fn(partial, floor)
    return merge_fn(all_gather_keys(keys, group))


def dist_query(S_shard, s_id_base: int, R, d: int, k: int, group=None, tile: int = 0, batch_rows: int = 0,
               cta_warps: int = 0, theta_tiles: int = 0, head_density: float = 0.0):
    """Product path on CUDA: every rank passes its S shard (DeviceCSR) and the full R (DeviceCSR).
    theta_tiles > 0 (and more than one rank): the two-phase protocol of sharded_join_theta, phase 1 over the
    shard's first theta_tiles S tiles.  Returns (ids int32 [n, k], scores float32 [n, k]) -- identical on every
    rank."""
    from . import knnjoin_build_index, knnjoin_index_stats, knnjoin_merge, knnjoin_query

    idx = knnjoin_build_index(S_shard, d, s_id_base=s_id_base, tile=tile, head_density=head_density)
    kw = dict(want_keys=True, want_ids=False, batch_rows=batch_rows, cta_warps=cta_warps)

    def merge(gathered):
        ids, scores, _ = knnjoin_merge(gathered, R, d, S_shard.dtype, k)
        return ids, scores

    world = dist.get_world_size(group)
    n_tiles = knnjoin_index_stats(idx)["n_tiles"]
    if theta_tiles > 0 and world > 1 and n_tiles > 1:
        split = min(theta_tiles, n_tiles - 1)

        def phase1():
            return knnjoin_query(idx, R, k, tile_range=(0, split), **kw)[2]

        def phase2(partial, floor):
            return knnjoin_query(idx, R, k, tile_range=(split, n_tiles), resume_keys=partial, theta_in=floor,
                                 **kw)[2]

        return sharded_join_theta(phase1, phase2, merge, k, group)
    return sharded_join(lambda: knnjoin_query(idx, R, k, **kw)[2], merge, group)
