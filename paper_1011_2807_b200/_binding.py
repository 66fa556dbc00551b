"""ctypes binding of libknnjoin.so (include/knnjoin.h).  Marshalling only: every step of the path runs in the
library's CUDA kernels; this module allocates the caller-owned buffers with torch and passes raw pointers,
sizes and the current CUDA stream."""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# KNNJOIN_LIB: another build of the same library (the checked build of tools/checked_build.sh); default in-tree
_SO = os.environ.get("KNNJOIN_LIB") or os.path.join(_HERE, "libknnjoin.so")

BINARY, INT8, FP32 = 0, 1, 2
_DTYPE_NAMES = {"binary": BINARY, "int8": INT8, "fp32": FP32}

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_DIM", 3: "ERR_CSR", 4: "ERR_UNSUPPORTED", 5: "ERR_WORKSPACE", 6: "ERR_CUDA"}


class KnnJoinError(RuntimeError):
    def __init__(self, status: int, where: str, message: str):
        super().__init__(f"{where}: {STATUS.get(status, status)}: {message}")
        self.status = status


class _CSR(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("nnz", ctypes.c_int64), ("indptr", ctypes.c_void_p),
                ("indices", ctypes.c_void_p), ("values", ctypes.c_void_p), ("dtype", ctypes.c_int)]


class _Options(ctypes.Structure):
    _fields_ = [("tile", ctypes.c_int32), ("prune", ctypes.c_int32), ("alpha", ctypes.c_float),
                ("head_density", ctypes.c_float), ("head_max", ctypes.c_int32), ("forward", ctypes.c_void_p)]


class _QueryOptions(ctypes.Structure):
    _fields_ = [("batch_rows", ctypes.c_int32), ("counters", ctypes.c_void_p), ("ev_begin", ctypes.c_void_p),
                ("ev_end", ctypes.c_void_p), ("phase_cycles", ctypes.c_void_p), ("cta_warps", ctypes.c_int32),
                ("tiles_per_pass", ctypes.c_int32), ("row_order", ctypes.c_int32), ("tile_begin", ctypes.c_int64),
                ("tile_end", ctypes.c_int64), ("resume_keys", ctypes.c_void_p), ("theta_in", ctypes.c_void_p),
                ("prune_alpha", ctypes.c_float), ("residual", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("row_list", ctypes.c_void_p), ("row_count", ctypes.c_void_p), ("uncertified", ctypes.c_void_p),
                ("tolerance", ctypes.c_float)]


class _MergeOptions(ctypes.Structure):
    _fields_ = [("float_keys", ctypes.c_int32), ("row_list", ctypes.c_void_p), ("row_count", ctypes.c_void_p)]


class _IndexInfo(ctypes.Structure):
    _fields_ = [("n_s", ctypes.c_int64), ("s_id_base", ctypes.c_int64), ("d", ctypes.c_int32),
                ("tile", ctypes.c_int32), ("n_tiles", ctypes.c_int64), ("offsets", ctypes.c_int64),
                ("unit_capacity", ctypes.c_int64), ("storage_bytes", ctypes.c_int64), ("s_dtype", ctypes.c_int),
                ("head_min_df", ctypes.c_int64), ("head_max", ctypes.c_int32), ("prune", ctypes.c_int32),
                ("alpha", ctypes.c_float)]


def library_path() -> str:
    return _SO


def _load():
    if not os.path.exists(_SO):
        raise ImportError(f"{_SO} is missing: the CUDA library must be built (python __graft_entry__.py build); "
                          "there is no CPU fallback")
    L = ctypes.CDLL(_SO)
    P = ctypes.POINTER
    c = ctypes
    L.knnjoin_index_bytes.argtypes = [P(_CSR), c.c_int32, P(_Options)]
    L.knnjoin_index_bytes.restype = c.c_size_t
    L.knnjoin_build_workspace_bytes.argtypes = [P(_CSR), c.c_int32, P(_Options)]
    L.knnjoin_build_workspace_bytes.restype = c.c_size_t
    L.knnjoin_build_index.argtypes = [P(_CSR), c.c_int32, c.c_int64, P(_Options), c.c_void_p, c.c_size_t, c.c_void_p,
                                      c.c_size_t, c.c_void_p, P(c.c_void_p)]
    L.knnjoin_build_index.restype = c.c_int
    L.knnjoin_index_stats.argtypes = [c.c_void_p, P(_IndexInfo)]
    L.knnjoin_index_stats.restype = c.c_int
    L.knnjoin_free_index.argtypes = [c.c_void_p]
    L.knnjoin_free_index.restype = None
    L.knnjoin_query_workspace_bytes.argtypes = [c.c_void_p, P(_CSR), c.c_int32, P(_QueryOptions)]
    L.knnjoin_query_workspace_bytes.restype = c.c_size_t
    L.knnjoin_query.argtypes = [c.c_void_p, P(_CSR), c.c_int32, P(_QueryOptions), c.c_void_p, c.c_void_p, c.c_void_p,
                                c.c_void_p, c.c_size_t, c.c_void_p]
    L.knnjoin_query.restype = c.c_int
    L.knnjoin_merge_workspace_bytes.argtypes = [P(_CSR)]
    L.knnjoin_merge_workspace_bytes.restype = c.c_size_t
    L.knnjoin_merge.argtypes = [c.c_void_p, c.c_int32, P(_CSR), c.c_int32, c.c_int, c.c_int32, P(_MergeOptions),
                                c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p, c.c_size_t, c.c_void_p]
    L.knnjoin_merge.restype = c.c_int
    L.knnjoin_certify_workspace_bytes.argtypes = [P(_CSR)]
    L.knnjoin_certify_workspace_bytes.restype = c.c_size_t
    L.knnjoin_certify.argtypes = [c.c_void_p, P(_CSR), c.c_int32, c.c_int, c.c_int32, c.c_float, c.c_void_p, c.c_void_p,
                                  c.c_size_t, c.c_void_p]
    L.knnjoin_certify.restype = c.c_int
    L.knnjoin_validate_csr.argtypes = [P(_CSR), c.c_int32, c.c_void_p, P(c.c_int64)]
    L.knnjoin_validate_csr.restype = c.c_int
    L.knnjoin_iiib_profile_bytes.argtypes = [P(_CSR), c.c_int32]
    L.knnjoin_iiib_profile_bytes.restype = c.c_size_t
    L.knnjoin_iiib_profile.argtypes = [P(_CSR), c.c_int32, c.c_void_p, c.c_size_t, c.c_void_p]
    L.knnjoin_iiib_profile.restype = c.c_int
    L.knnjoin_iiib_threshold_workspace_bytes.argtypes = [P(_CSR)]
    L.knnjoin_iiib_threshold_workspace_bytes.restype = c.c_size_t
    L.knnjoin_iiib_threshold.argtypes = [c.c_void_p, P(_CSR), c.c_int32, c.c_int, c.c_int32, c.c_void_p, c.c_void_p,
                                         c.c_size_t, c.c_void_p]
    L.knnjoin_iiib_threshold.restype = c.c_int
    L.knnjoin_iiib_split_workspace_bytes.argtypes = [P(_CSR)]
    L.knnjoin_iiib_split_workspace_bytes.restype = c.c_size_t
    L.knnjoin_iiib_split.argtypes = [P(_CSR), c.c_int32, c.c_void_p, c.c_void_p, c.c_int32, c.c_void_p, c.c_void_p,
                                     c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p, c.c_void_p, c.c_size_t, c.c_void_p]
    L.knnjoin_iiib_split.restype = c.c_int
    L.knnjoin_last_error.argtypes = []
    L.knnjoin_last_error.restype = c.c_char_p
    L.knnjoin_version.argtypes = []
    L.knnjoin_version.restype = c.c_char_p
    return L


_lib = _load()

EXPORTS = ["knnjoin_index_bytes", "knnjoin_build_workspace_bytes", "knnjoin_build_index", "knnjoin_index_stats",
           "knnjoin_free_index", "knnjoin_query_workspace_bytes", "knnjoin_query", "knnjoin_merge_workspace_bytes",
           "knnjoin_merge", "knnjoin_certify_workspace_bytes", "knnjoin_certify", "knnjoin_validate_csr", "knnjoin_last_error", "knnjoin_version",
           "knnjoin_iiib_profile_bytes", "knnjoin_iiib_profile", "knnjoin_iiib_threshold_workspace_bytes",
           "knnjoin_iiib_threshold", "knnjoin_iiib_split_workspace_bytes", "knnjoin_iiib_split"]


def knnjoin_last_error() -> str:
    return _lib.knnjoin_last_error().decode()


def knnjoin_version() -> str:
    return _lib.knnjoin_version().decode()


def _check(status: int, where: str):
    if status != 0:
        raise KnnJoinError(status, where, knnjoin_last_error())


def _stream_ptr(stream) -> int:
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream)


@dataclass
class DeviceCSR:
    """A CSR matrix whose arrays are device tensors (indptr int64, indices int32, values int8/float32/None)."""
    indptr: torch.Tensor
    indices: torch.Tensor
    values: torch.Tensor | None
    dtype: int

    @property
    def n_rows(self) -> int:
        return self.indptr.numel() - 1

    @property
    def nnz(self) -> int:
        return self.indices.numel()

    @staticmethod
    def from_arrays(indptr, indices, values=None, device="cuda", non_blocking=False) -> "DeviceCSR":
        """Copy host arrays (numpy or torch) to ``device``.  values: None (binary), int8 or float32."""
        def t(x, dt):
            if isinstance(x, np.ndarray):
                x = torch.from_numpy(np.ascontiguousarray(x))
            return x.to(device=device, dtype=dt, non_blocking=non_blocking)
        ip = t(indptr, torch.int64)
        ix = t(indices, torch.int32)
        if values is None:
            return DeviceCSR(ip, ix, None, BINARY)
        vdt = values.dtype
        is_int8 = (vdt == np.int8) if isinstance(values, np.ndarray) else (vdt == torch.int8)
        if is_int8:
            return DeviceCSR(ip, ix, t(values, torch.int8), INT8)
        return DeviceCSR(ip, ix, t(values, torch.float32), FP32)

    @staticmethod
    def from_host(h, device="cuda", non_blocking=False) -> "DeviceCSR":
        return DeviceCSR.from_arrays(h.indptr, h.indices, h.values, device, non_blocking)

    def _c(self) -> _CSR:
        return _CSR(self.n_rows, self.nnz, self.indptr.data_ptr(), self.indices.data_ptr() if self.nnz else 0,
                    self.values.data_ptr() if (self.values is not None and self.nnz) else 0, self.dtype)


class Index:
    """Host handle + caller-owned device storage of a built index (knnjoin_build_index)."""

    def __init__(self, handle: int, storage: torch.Tensor, d: int, s_dtype: int, n_s: int, s_id_base: int):
        self._h = ctypes.c_void_p(handle)
        self.storage = storage
        self.d = d
        self.s_dtype = s_dtype
        self.n_s = n_s
        self.s_id_base = s_id_base

    @property
    def handle(self):
        return self._h

    def __del__(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            _lib.knnjoin_free_index(self._h)
            self._h = None


def _empty_u8(nbytes: int, device) -> torch.Tensor:
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def knnjoin_build_index(S: DeviceCSR, d: int, s_id_base: int = 0, tile: int = 0, stream=None,
                        workspace: torch.Tensor | None = None, head_density: float = 0.0,
                        head_max: int = 0, prune: int = 0, alpha: float = 0.0,
                        forward: "DeviceCSR | None" = None, storage: torch.Tensor | None = None) -> Index:
    """prune=1 keeps S's forward rows for threshold-pruned queries (a6; knnjoin_options.prune / alpha), or the
    rows of `forward` instead (f1: the residual parts s').  storage: a caller-provided uint8 device tensor for the
    index (at least knnjoin_index_bytes; e.g. pre-poisoned by the initialisation tests)."""
    cS = S._c()
    cF = forward._c() if forward is not None else None
    opt = _Options(tile, prune, alpha, head_density, head_max, ctypes.addressof(cF) if cF is not None else 0)
    nbytes = _lib.knnjoin_index_bytes(ctypes.byref(cS), d, ctypes.byref(opt))
    if nbytes == 0:
        raise KnnJoinError(1, "knnjoin_index_bytes", knnjoin_last_error())
    wbytes = _lib.knnjoin_build_workspace_bytes(ctypes.byref(cS), d, ctypes.byref(opt))
    if wbytes == 0:
        raise KnnJoinError(1, "knnjoin_build_workspace_bytes", knnjoin_last_error())
    dev = S.indptr.device
    if storage is None or storage.numel() < nbytes:
        storage = _empty_u8(nbytes, dev)
    ws = workspace if (workspace is not None and workspace.numel() >= wbytes) else _empty_u8(wbytes, dev)
    out = ctypes.c_void_p()
    _check(_lib.knnjoin_build_index(ctypes.byref(cS), d, s_id_base, ctypes.byref(opt), storage.data_ptr(), storage.numel(),
                                    ws.data_ptr(), ws.numel(), _stream_ptr(stream), ctypes.byref(out)),
           "knnjoin_build_index")
    # keep the workspace alive until the stream has consumed it
    ws.record_stream(torch.cuda.current_stream() if stream is None else stream)
    return Index(out.value, storage, d, S.dtype, S.n_rows, s_id_base)


def knnjoin_index_stats(index: Index) -> dict:
    info = _IndexInfo()
    _check(_lib.knnjoin_index_stats(index.handle, ctypes.byref(info)), "knnjoin_index_stats")
    return {f: getattr(info, f) for f, _ in _IndexInfo._fields_}


def knnjoin_query(index: Index, R: DeviceCSR, k: int, want_keys: bool = False, want_ids: bool = True,
                  batch_rows: int = 0, counters: torch.Tensor | None = None, events=None, stream=None,
                  workspace: torch.Tensor | None = None, phase_cycles: torch.Tensor | None = None,
                  cta_warps: int = 0, tiles_per_pass: int = 0, row_order: int = 0, tile_range=(0, 0),
                  resume_keys: torch.Tensor | None = None, theta_in: torch.Tensor | None = None,
                  prune_alpha: float = 0.0, residual: int = 0, precision: int = 0,
                  row_list: torch.Tensor | None = None, uncertified: torch.Tensor | None = None,
                  tolerance: float = 0.0, out=None):
    """Returns (ids int32 [n,k], scores float32 [n,k], keys uint64-as-int64 [n,k] or None).
    tile_range / resume_keys (int64 [n,k]) / theta_in (int64 [n]) / prune_alpha / precision / tolerance: see
    knnjoin_query_options.  row_list: device int32 [1 + m] laid out as knnjoin_certify's list (count, then rows).
    uncertified: device int32 [1 + n] receiving the certification list.  out: (ids, scores, keys) tensors to
    write into (rows outside row_list keep their contents)."""
    for t, shape in ((resume_keys, (R.n_rows, k)), (theta_in, (R.n_rows,))):
        if t is not None and (tuple(t.shape) != shape or t.dtype != torch.int64 or not t.is_contiguous()):
            raise ValueError(f"expected a contiguous int64 tensor of shape {shape}")
    for t in (row_list, uncertified):
        if t is not None and (t.dtype != torch.int32 or not t.is_contiguous() or t.numel() < 1 or t.device.type != "cuda"):
            raise ValueError("row_list / uncertified must be contiguous device int32 tensors [1 + rows]")
    if uncertified is not None and uncertified.numel() < R.n_rows + 1:
        raise ValueError("uncertified needs 1 + n_rows entries")
    cR = R._c()
    if events and (events[0].cuda_event == 0 or events[1].cuda_event == 0):
        raise ValueError("timing events must have been recorded once (so their cudaEvent handles exist)")
    qo = _QueryOptions(batch_rows, counters.data_ptr() if counters is not None else 0,
                       events[0].cuda_event if events else 0, events[1].cuda_event if events else 0,
                       phase_cycles.data_ptr() if phase_cycles is not None else 0, cta_warps, tiles_per_pass,
                       row_order, tile_range[0], tile_range[1],
                       resume_keys.data_ptr() if resume_keys is not None else 0,
                       theta_in.data_ptr() if theta_in is not None else 0, prune_alpha, residual, precision,
                       row_list.data_ptr() + 4 if row_list is not None else 0,
                       row_list.data_ptr() if row_list is not None else 0,
                       uncertified.data_ptr() if uncertified is not None else 0, tolerance)
    wbytes = _lib.knnjoin_query_workspace_bytes(index.handle, ctypes.byref(cR), k, ctypes.byref(qo))
    if wbytes == 0:
        raise KnnJoinError(1, "knnjoin_query_workspace_bytes", knnjoin_last_error())
    dev = R.indptr.device
    n = R.n_rows
    if out is not None:
        ids, scores, keys = out
        for t, dt in ((ids, torch.int32), (scores, torch.float32), (keys, torch.int64)):
            if t is not None and (tuple(t.shape) != (n, k) or t.dtype != dt or not t.is_contiguous()):
                raise ValueError("out tensors must be contiguous [n, k] int32 / float32 / int64")
    else:
        ids = torch.empty((n, k), dtype=torch.int32, device=dev) if want_ids else None
        scores = torch.empty((n, k), dtype=torch.float32, device=dev) if want_ids else None
        keys = torch.empty((n, k), dtype=torch.int64, device=dev) if want_keys else None
    ws = workspace if (workspace is not None and workspace.numel() >= wbytes) else _empty_u8(wbytes, dev)
    _check(_lib.knnjoin_query(index.handle, ctypes.byref(cR), k, ctypes.byref(qo),
                              keys.data_ptr() if keys is not None else 0, ids.data_ptr() if ids is not None else 0,
                              scores.data_ptr() if scores is not None else 0, ws.data_ptr(), ws.numel(),
                              _stream_ptr(stream)), "knnjoin_query")
    ws.record_stream(torch.cuda.current_stream() if stream is None else stream)
    return ids, scores, keys


def knnjoin_merge(keys: torch.Tensor, R: DeviceCSR, d: int, s_dtype: int, k: int, want_keys: bool = False,
                  stream=None, float_keys: int = 0, row_list: torch.Tensor | None = None, out=None):
    """keys: int64 view of uint64 [P, n, k].  Returns (ids, scores, merged keys or None).
    float_keys / row_list (device int32 [1 + m]: count, then output rows): knnjoin_merge_options.  out: existing
    (ids, scores, keys) to write into (with row_list only the listed rows are written)."""
    P = keys.shape[0]
    n = R.n_rows
    if keys.dim() != 3 or tuple(keys.shape[1:]) != (n, k) or keys.dtype != torch.int64 or not keys.is_contiguous() \
            or keys.device != R.indptr.device:
        raise ValueError(f"keys must be a contiguous int64 tensor [P, {n}, {k}] on {R.indptr.device}")
    if row_list is not None and (row_list.dtype != torch.int32 or not row_list.is_contiguous() or row_list.numel() < 1):
        raise ValueError("row_list must be a contiguous device int32 tensor [1 + rows]")
    cR = R._c()
    dev = keys.device
    wbytes = _lib.knnjoin_merge_workspace_bytes(ctypes.byref(cR))
    ws = _empty_u8(wbytes, dev)
    if out is not None:
        ids, scores, out_keys = out
    else:
        ids = torch.empty((n, k), dtype=torch.int32, device=dev)
        scores = torch.empty((n, k), dtype=torch.float32, device=dev)
        out_keys = torch.empty((n, k), dtype=torch.int64, device=dev) if want_keys else None
    mo = _MergeOptions(float_keys, row_list.data_ptr() + 4 if row_list is not None else 0,
                       row_list.data_ptr() if row_list is not None else 0)
    _check(_lib.knnjoin_merge(keys.data_ptr(), P, ctypes.byref(cR), d, s_dtype, k, ctypes.byref(mo),
                              out_keys.data_ptr() if out_keys is not None else 0, ids.data_ptr(), scores.data_ptr(),
                              ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "knnjoin_merge")
    ws.record_stream(torch.cuda.current_stream() if stream is None else stream)
    return ids, scores, out_keys


def knnjoin_certify(keys: torch.Tensor, R: DeviceCSR, d: int, s_dtype: int, k: int, tolerance: float = 0.0,
                    stream=None) -> torch.Tensor:
    """Certification of complete 32-bit lists (keys int64 [n, k]) -> device int32 [1 + n]: count, then the rows
    whose lists fail the tolerance rule (knnjoin_certify)."""
    n = R.n_rows
    if tuple(keys.shape) != (n, k) or keys.dtype != torch.int64 or not keys.is_contiguous():
        raise ValueError(f"keys must be a contiguous int64 tensor [{n}, {k}]")
    cR = R._c()
    dev = R.indptr.device
    ws = _empty_u8(_lib.knnjoin_certify_workspace_bytes(ctypes.byref(cR)), dev)
    out = torch.empty(n + 1, dtype=torch.int32, device=dev)
    _check(_lib.knnjoin_certify(keys.data_ptr(), ctypes.byref(cR), d, s_dtype, k, tolerance, out.data_ptr(),
                                ws.data_ptr(), ws.numel(), _stream_ptr(stream)), "knnjoin_certify")
    ws.record_stream(torch.cuda.current_stream() if stream is None else stream)
    return out


def knnjoin_validate_csr(m: DeviceCSR, d: int, stream=None):
    """Returns (status, bad_row): status 0 = valid, 3 = ERR_CSR with the first bad row."""
    bad = ctypes.c_int64(-1)
    st = _lib.knnjoin_validate_csr(ctypes.byref(m._c()), d, _stream_ptr(stream), ctypes.byref(bad))
    if st not in (0, 3):
        _check(st, "knnjoin_validate_csr")
    return st, bad.value


# ---- f1: IIIB-literal building blocks (knnjoin_iiib_*) -------------------------------------------------------

def knnjoin_iiib_profile(R: DeviceCSR, d: int, stream=None) -> torch.Tensor:
    """Alg. 4 lines 6-7 over all of R -> opaque device profile (uint8 tensor)."""
    cR = R._c()
    nb = _lib.knnjoin_iiib_profile_bytes(ctypes.byref(cR), d)
    if nb == 0:
        raise KnnJoinError(1, "knnjoin_iiib_profile_bytes", knnjoin_last_error())
    prof = _empty_u8(nb, R.indptr.device)
    _check(_lib.knnjoin_iiib_profile(ctypes.byref(cR), d, prof.data_ptr(), nb, _stream_ptr(stream)),
           "knnjoin_iiib_profile")
    return prof


def knnjoin_iiib_threshold(keys: torch.Tensor | None, R: DeviceCSR, d: int, s_dtype: int, k: int,
                           stream=None) -> torch.Tensor:
    """MinPruneScore from the current keys (None before the first S block) -> device float64[2]."""
    cR = R._c()
    wb = _lib.knnjoin_iiib_threshold_workspace_bytes(ctypes.byref(cR))
    ws = _empty_u8(wb, R.indptr.device)
    out = torch.empty(2, dtype=torch.float64, device=R.indptr.device)
    _check(_lib.knnjoin_iiib_threshold(keys.data_ptr() if keys is not None else 0, ctypes.byref(cR), d, s_dtype, k,
                                       out.data_ptr(), ws.data_ptr(), wb, _stream_ptr(stream)),
           "knnjoin_iiib_threshold")
    return out


def knnjoin_iiib_split(S: DeviceCSR, d: int, profile: torch.Tensor, threshold: torch.Tensor, r_integer: bool,
                       rows=None, stream=None):
    """Alg. 4 lines 8-14 on rows [lo, hi) of S (all if None) -> (indexed s'', residual s') DeviceCSRs.
    Reads the two nnz back (a 16-byte device-to-host copy that synchronises the stream)."""
    lo, hi = rows if rows is not None else (0, S.n_rows)
    n = hi - lo
    nnz = int(S.nnz)
    # a row-range view: indptr from row lo on (absolute positions into S's indices / values)
    cS = _CSR(n, nnz, S.indptr.data_ptr() + 8 * lo, S.indices.data_ptr() if nnz else 0,
              S.values.data_ptr() if (S.values is not None and nnz) else 0, S.dtype)
    dev = S.indptr.device
    cap = max(1, nnz)
    ip_i = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ip_r = torch.empty(n + 1, dtype=torch.int64, device=dev)
    ix_i = torch.empty(cap, dtype=torch.int32, device=dev)
    ix_r = torch.empty(cap, dtype=torch.int32, device=dev)
    v_i = torch.empty(cap, dtype=torch.int8, device=dev) if S.dtype == INT8 else None
    v_r = torch.empty(cap, dtype=torch.int8, device=dev) if S.dtype == INT8 else None
    wb = _lib.knnjoin_iiib_split_workspace_bytes(ctypes.byref(cS))
    ws = _empty_u8(wb, dev)
    _check(_lib.knnjoin_iiib_split(ctypes.byref(cS), d, profile.data_ptr(), threshold.data_ptr(), int(bool(r_integer)),
                                   ip_i.data_ptr(), ix_i.data_ptr(), v_i.data_ptr() if v_i is not None else 0,
                                   ip_r.data_ptr(), ix_r.data_ptr(), v_r.data_ptr() if v_r is not None else 0,
                                   ws.data_ptr(), wb, _stream_ptr(stream)), "knnjoin_iiib_split")
    ends = torch.stack([ip_i[n], ip_r[n]]).cpu()
    ni, nr = int(ends[0]), int(ends[1])
    idx = DeviceCSR(ip_i, ix_i[:ni], v_i[:ni] if v_i is not None else None, S.dtype)
    res = DeviceCSR(ip_r, ix_r[:nr], v_r[:nr] if v_r is not None else None, S.dtype)
    return idx, res
