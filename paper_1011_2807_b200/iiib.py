"""f1: the paper's IIIB algorithm literally -- Alg. 1's block nested loop with
Alg. 4's kernel on every S block, all of R as the one R block.

Per S block (rows [lo, hi), ascending):
  1. MinPruneScore = min over R of pruneScore(r), from the top-k keys of the blocks done so far
     (knnjoin_iiib_threshold; 0 before the first block: "initialized to 0").
  2. Create_Inverted_List_IIIB: the R profile (dimension order by non-zero count in R, maxWeight_d; computed once,
     knnjoin_iiib_profile) splits every s into its indexed part s'' and residual s' (knnjoin_iiib_split).
  3. The block's inverted lists are built from s'' with the residual rows s' as forward rows
     (knnjoin_build_index(prune=1, forward=s')).
  4. Find_Matches_IIIB: the query accumulates over the lists and adds dot(r, s') to every touched s
     (knnjoin_query(residual=1)), continuing the previous blocks' lists (resume_keys).
The result equals the exact top-k (Theorem 1).  Host-side scheduling only: every step on the
data runs in libknnjoin's kernels; the host reads back two nnz per block to size the block's index.
"""
from __future__ import annotations

import torch

from ._binding import (FP32, DeviceCSR, knnjoin_build_index, knnjoin_certify, knnjoin_iiib_profile,
                       knnjoin_iiib_split, knnjoin_iiib_threshold, knnjoin_merge, knnjoin_query)


def iiib_join(R: DeviceCSR, S: DeviceCSR, d: int, k: int, s_block: int, tile: int = 0, counters: bool = True,
              stream=None):
    """Returns (ids int32 [n,k], scores float32 [n,k], stats dict).  stats: postings_built (indexed postings, the
    first term of Eq. 4 for IIIB) against postings_iib = nnz(S) (IIB indexes every posting),
    postings_visited, residual completions, blocks."""
    dev = R.indptr.device
    prof = knnjoin_iiib_profile(R, d, stream=stream)
    n_s = S.n_rows
    keys = None
    built = visited = completions = 0
    blocks = 0
    cnt = torch.zeros(4, dtype=torch.int64, device=dev) if counters else None
    for lo in range(0, max(n_s, 1), max(1, s_block)):
        hi = min(n_s, lo + s_block)
        if hi <= lo:
            break
        thr = knnjoin_iiib_threshold(keys, R, d, S.dtype, k, stream=stream)
        s_idx, s_res = knnjoin_iiib_split(S, d, prof, thr, R.dtype != FP32, rows=(lo, hi), stream=stream)
        built += s_idx.nnz
        idx = knnjoin_build_index(s_idx, d, s_id_base=lo, tile=tile, prune=1, forward=s_res, stream=stream)
        _, _, keys = knnjoin_query(idx, R, k, want_keys=True, want_ids=False, resume_keys=keys, residual=1,
                                   counters=cnt, stream=stream, precision=1)
        blocks += 1
    if keys is None:  # empty S: every row is padding
        keys = torch.zeros((R.n_rows, k), dtype=torch.int64, device=dev)
    ids, sc, _ = knnjoin_merge(keys.unsqueeze(0).contiguous(), R, d, S.dtype, k, stream=stream)
    n_unc = 0
    if R.dtype == FP32:  # certify the final 32-bit lists; failing rows are recomputed at 64 bits
        lst = knnjoin_certify(keys, R, d, S.dtype, k, stream=stream)
        n_unc = int(lst[0].item())
        if n_unc:
            full = knnjoin_build_index(S, d, tile=tile, stream=stream)
            knnjoin_query(full, R, k, precision=2, row_list=lst, out=(ids, sc, None), stream=stream)
    if counters:
        c = cnt.cpu().tolist()
        visited, completions = c[0], c[3]
    stats = {"postings_built": built, "postings_iib": int(S.nnz), "postings_visited": visited,
             "residual_completions": completions, "blocks": blocks, "uncertified_rows": n_unc}
    return ids, sc, stats
