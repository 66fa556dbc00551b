"""f4: KNN join against an S that lives in host memory (larger than HBM).

This is Alg. 1's block nested loop with the roles the paper gives to disk blocks taken by
pinned host memory and HBM: S is split into blocks of ``block_rows`` rows; block b+1 is copied host->device on
a copy stream (copy engines) while block b's index is built and queried on the compute stream (double
buffering: two device slots); every query continues the previous block's top-k lists through
``resume_keys``, so pruneScore -- the per-row k-th key -- is carried from block to block as the paper carries
it across S blocks.  Block b's index has s_id_base = its first row, so keys of different
blocks never collide and the result is the one-index result bit for bit.

Host-side scheduling only: every step on the data (index build, accumulation, top-k) runs in libknnjoin's
kernels; torch supplies pinned memory, device buffers, streams and events.
"""
from __future__ import annotations

import numpy as np
import torch

from ._binding import BINARY, FP32, INT8, DeviceCSR, knnjoin_build_index, knnjoin_certify, knnjoin_query


class PinnedS:
    """S in pinned host memory, pre-split into blocks of ``block_rows`` rows (indptr rebased per block)."""

    def __init__(self, indptr: np.ndarray, indices: np.ndarray, values: np.ndarray | None, block_rows: int):
        n = len(indptr) - 1
        self.n_rows = n
        self.block_rows = max(1, int(block_rows))
        self.blocks = [(lo, min(n, lo + self.block_rows)) for lo in range(0, n, self.block_rows)] or [(0, 0)]
        ip = np.asarray(indptr, np.int64)
        reb = np.concatenate([ip[lo:hi + 1] - ip[lo] for lo, hi in self.blocks])
        self.indptr_reb = torch.from_numpy(reb).pin_memory()
        self.ip_at = np.cumsum([0] + [hi - lo + 1 for lo, hi in self.blocks])
        self.nnz_at = [int(ip[lo]) for lo, _ in self.blocks] + [int(ip[n])]
        self.indices = torch.from_numpy(np.ascontiguousarray(indices, np.int32)).pin_memory()
        self.values = None if values is None else torch.from_numpy(np.ascontiguousarray(values)).pin_memory()
        self.dtype = BINARY if values is None else (INT8 if self.values.dtype == torch.int8 else FP32)
        self.max_rows = max(hi - lo for lo, hi in self.blocks)
        self.max_nnz = max(self.nnz_at[b + 1] - self.nnz_at[b] for b in range(len(self.blocks)))

    @staticmethod
    def from_host(h, block_rows: int) -> "PinnedS":
        return PinnedS(h.indptr, h.indices, h.values, block_rows)


def _sweep(S: PinnedS, R: DeviceCSR, d: int, tile: int, head_density: float, query):
    """Alg. 1's loop over the S blocks: copy block b+1 under block b's index build + query(idx, last)."""
    dev = R.indptr.device
    compute = torch.cuda.current_stream(dev)
    copy = torch.cuda.Stream(dev)
    slots = []
    for _ in range(2):
        slots.append(dict(
            indptr=torch.empty(S.max_rows + 1, dtype=torch.int64, device=dev),
            indices=torch.empty(max(1, S.max_nnz), dtype=torch.int32, device=dev),
            values=None if S.values is None else torch.empty(max(1, S.max_nnz), dtype=S.values.dtype, device=dev),
            ready=torch.cuda.Event(), free=torch.cuda.Event()))
    nb = len(S.blocks)

    def issue_copy(b):
        sl = slots[b % 2]
        lo, hi = S.blocks[b]
        a, e = S.nnz_at[b], S.nnz_at[b + 1]
        with torch.cuda.stream(copy):
            copy.wait_event(sl["free"])  # the slot's previous block has been indexed
            sl["indptr"][:hi - lo + 1].copy_(S.indptr_reb[S.ip_at[b]:S.ip_at[b + 1]], non_blocking=True)
            if e > a:
                sl["indices"][:e - a].copy_(S.indices[a:e], non_blocking=True)
                if S.values is not None:
                    sl["values"][:e - a].copy_(S.values[a:e], non_blocking=True)
            sl["ready"].record(copy)

    for sl in slots:
        sl["free"].record(compute)
    issue_copy(0)
    for b in range(nb):
        if b + 1 < nb:
            issue_copy(b + 1)
        sl = slots[b % 2]
        lo, hi = S.blocks[b]
        nnz = S.nnz_at[b + 1] - S.nnz_at[b]
        compute.wait_event(sl["ready"])
        blk = DeviceCSR(sl["indptr"][:hi - lo + 1], sl["indices"][:nnz],
                        None if S.values is None else sl["values"][:nnz], S.dtype)
        idx = knnjoin_build_index(blk, d, s_id_base=lo, tile=tile, head_density=head_density)
        sl["free"].record(compute)  # the block's CSR is no longer read once its index is built
        query(idx, b == nb - 1)
    for sl in slots:
        for t in (sl["indptr"], sl["indices"], sl["values"]):
            if t is not None:
                t.record_stream(copy)


def streamed_join(S: PinnedS, R: DeviceCSR, d: int, k: int, tile: int = 0, head_density: float = 0.0,
                  batch_rows: int = 0, want_keys: bool = False, stats: dict | None = None):
    """Returns (ids int32 [n, k], scores float32 [n, k], keys int64 [n, k] or None) of R against all of S.
    Device memory: two block slots (CSR) + one block index + R + the [n, k] lists, whatever the size of S.
    FP32 R against integer S: the final 32-bit lists are certified (knnjoin_certify) and failing
    rows are streamed again at 64 bits (their keys are then fp32-keyed; stats['uncertified_rows'])."""
    narrow = R.dtype == FP32 and S.dtype != FP32
    st = {"keys": None, "ids": None, "scores": None}

    def q32(idx, last):
        st["ids"], st["scores"], st["keys"] = knnjoin_query(
            idx, R, k, want_keys=True, want_ids=last, batch_rows=batch_rows, resume_keys=st["keys"],
            precision=1 if narrow else 0)

    _sweep(S, R, d, tile, head_density, q32)
    ids, scores, keys = st["ids"], st["scores"], st["keys"]
    n_unc = 0
    if narrow:
        lst = knnjoin_certify(keys, R, d, S.dtype, k)
        n_unc = int(lst[0].item())
        if n_unc:
            wk = [torch.zeros_like(keys), torch.zeros_like(keys)]
            step = {"b": 0}

            def q64(idx, last):
                b = step["b"]
                src = wk[(b + 1) % 2] if b > 0 else None
                dst = wk[b % 2]
                out = (ids, scores, keys) if last else (None, None, dst)
                knnjoin_query(idx, R, k, precision=2, row_list=lst, resume_keys=src, out=out)
                step["b"] = b + 1

            _sweep(S, R, d, tile, head_density, q64)
    if stats is not None:
        stats["uncertified_rows"] = n_unc
    return ids, scores, keys if want_keys else None
