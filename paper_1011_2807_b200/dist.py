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


def dist_query(S_shard, s_id_base: int, R, d: int, k: int, group=None, tile: int = 0, dense_min: int = 0,
               batch_rows: int = 0, cta_warps: int = 0):
    """Product path on CUDA: every rank passes its S shard (DeviceCSR) and the full R (DeviceCSR).
    Returns (ids int32 [n, k], scores float32 [n, k]) -- identical on every rank."""
    from . import knnjoin_build_index, knnjoin_merge, knnjoin_query

    def local():
        idx = knnjoin_build_index(S_shard, d, s_id_base=s_id_base, tile=tile, dense_min=dense_min)
        _, _, keys = knnjoin_query(idx, R, k, want_keys=True, want_ids=False, batch_rows=batch_rows,
                                   cta_warps=cta_warps)
        return keys

    def merge(gathered):
        ids, scores, _ = knnjoin_merge(gathered, R, d, S_shard.dtype, k)
        return ids, scores

    return sharded_join(local, merge, group)
