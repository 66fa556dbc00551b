"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the sparse KNN join.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl reference``
legs may import this package.  The product path (``paper_1011_2807_b200``) never imports it and shares
no code with it.

* ``oracle.c``       -- the plain single-threaded brute-force definition (§3 Eq. 1 with the
                        merge dot of Alg. 2 lines 8-23), ties to the lower S id, zero
                        scores excluded, padded with (-1, 0).
* ``iib.c``          -- the paper's IIB (Alg. 3) in plain single-threaded C: the "paper's method
                        on the host" leg of bench.py's cpu_baseline (not an oracle; pinned against oracle_knn).
* ``paper_algs.py``  -- the paper's Alg. 1-4 (block nested loops, BF, IIB, IIIB) written out step by step
                        in pure Python, with the Eq. 2-4 cost counters, for tiny cross-check instances.

Pins (tests/test_oracle_pins.py): SPEC.md worked examples, a dense d-dimensional dot product, symmetry,
the binary set-intersection closed form, scipy's sparse R @ S.T + numpy lexsort on small instances, a
hand-worked tie/padding example (tests/golden/hand_example.json) and BF == IIB == IIIB.
Parity status per function is listed in DESIGN.md ("Oracle and pins").
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

DTYPE_CODE = {"binary": 0, "int8": 1, "fp32": 2}


class _CSR(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("indptr", ctypes.c_void_p), ("indices", ctypes.c_void_p),
                ("values", ctypes.c_void_p), ("dtype", ctypes.c_int32)]


_SOURCES = ("oracle.c", "iib.c")


def build() -> str:
    """Compile oracle.c + iib.c (plain C, -O2, no OpenMP: both are single-threaded)."""
    tmp = _SO + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-o", tmp] + [os.path.join(_HERE, f) for f in _SOURCES])
    os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            newest = max(os.path.getmtime(os.path.join(_HERE, f)) for f in _SOURCES)
            if not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
                build()
            L = ctypes.CDLL(_SO)
            P = ctypes.POINTER(_CSR)
            L.oracle_dot.argtypes = [P, ctypes.c_int64, P, ctypes.c_int64, ctypes.c_void_p]
            L.oracle_dot.restype = ctypes.c_double
            L.oracle_knn.argtypes = [P, P, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_void_p]
            L.oracle_knn.restype = ctypes.c_int
            L.oracle_pair_scores.argtypes = [P, P, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
            L.oracle_bf_counters.argtypes = [P, P, ctypes.c_void_p, ctypes.c_void_p]
            L.iib_build.argtypes = [P, ctypes.c_int32]
            L.iib_build.restype = ctypes.c_void_p
            L.iib_free.argtypes = [ctypes.c_void_p]
            L.iib_free.restype = None
            L.iib_query.argtypes = [ctypes.c_void_p, P, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                    ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
            L.iib_query.restype = ctypes.c_int
            _lib = L
    return _lib


class _Held:
    """Keeps contiguous numpy arrays alive for the duration of a C call."""

    def __init__(self, csr):
        self.indptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
        self.indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
        dt = csr.dtype
        self.values = None
        if dt == "int8":
            self.values = np.ascontiguousarray(csr.values, dtype=np.int8)
        elif dt == "fp32":
            self.values = np.ascontiguousarray(csr.values, dtype=np.float32)
        self.c = _CSR(len(self.indptr) - 1, self.indptr.ctypes.data, self.indices.ctypes.data,
                      0 if self.values is None else self.values.ctypes.data, DTYPE_CODE[dt])


def knn(R, S, k: int, rows=None, s_id_base: int = 0, threads: int = 1):
    """Oracle top-k for rows ``rows`` of R (all if None) against all of S.

    Returns (ids int64 [n, k], scores float64 [n, k]).  ``threads`` > 1 splits the ROWS over host threads,
    each running the unchanged single-threaded C routine on its own rows (ctypes releases the GIL).
    """
    L = lib()
    hR, hS = _Held(R), _Held(S)
    sel = np.arange(R.n_rows, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    n = len(sel)
    ids = np.empty((n, k), dtype=np.int64)
    scores = np.empty((n, k), dtype=np.float64)
    if n == 0:
        return ids, scores
    threads = max(1, min(threads, n))
    bounds = np.linspace(0, n, threads + 1).astype(np.int64)

    def work(i):
        a, b = int(bounds[i]), int(bounds[i + 1])
        if b <= a:
            return 0
        sub = sel[a:b]
        return L.oracle_knn(ctypes.byref(hR.c), ctypes.byref(hS.c), sub.ctypes.data, b - a, k, s_id_base,
                            ids[a:b].ctypes.data, scores[a:b].ctypes.data)

    if threads == 1:
        rc = [work(0)]
    else:
        with ThreadPoolExecutor(threads) as ex:
            rc = list(ex.map(work, range(threads)))
    if any(rc):
        raise MemoryError("oracle_knn allocation failed")
    return ids, scores


def dot(R, r: int, S, s: int) -> float:
    L = lib()
    hR, hS = _Held(R), _Held(S)
    return L.oracle_dot(ctypes.byref(hR.c), r, ctypes.byref(hS.c), s, None)


def dot_with_advances(R, r: int, S, s: int):
    L = lib()
    hR, hS = _Held(R), _Held(S)
    adv = ctypes.c_int64(0)
    v = L.oracle_dot(ctypes.byref(hR.c), r, ctypes.byref(hS.c), s, ctypes.byref(adv))
    return v, adv.value


def pair_scores(R, S, r_rows, s_rows) -> np.ndarray:
    """Exact oracle scores of the pairs (r_rows[i], s_rows[i]); s_rows[i] < 0 gives 0."""
    L = lib()
    hR, hS = _Held(R), _Held(S)
    rr = np.ascontiguousarray(r_rows, dtype=np.int64)
    ss = np.ascontiguousarray(s_rows, dtype=np.int64)
    out = np.empty(len(rr), dtype=np.float64)
    L.oracle_pair_scores(ctypes.byref(hR.c), ctypes.byref(hS.c), rr.ctypes.data, ss.ctypes.data, len(rr),
                         out.ctypes.data)
    return out


def bf_counters(R, S):
    """Eq. 3: (charged = sum over pairs of |r|+|s|, true merge advances)."""
    L = lib()
    hR, hS = _Held(R), _Held(S)
    c, a = ctypes.c_int64(0), ctypes.c_int64(0)
    L.oracle_bf_counters(ctypes.byref(hR.c), ctypes.byref(hS.c), ctypes.byref(c), ctypes.byref(a))
    return c.value, a.value


def iib_knn(R, S, k: int, rows=None, threads: int = 1, d: int | None = None):
    """The paper's IIB (Alg. 3) on the host: index S once (single-threaded C), then rows ``rows`` of R (all if
    None) split over ``threads`` host threads, each running the single-threaded query on its rows.
    Returns (ids int64 [n, k], scores float64 [n, k], info) with info = {build_s, query_s, visits}."""
    import time
    L = lib()
    hR, hS = _Held(R), _Held(S)
    d = d if d is not None else S.d
    t0 = time.perf_counter()
    ix = L.iib_build(ctypes.byref(hS.c), d)
    build_s = time.perf_counter() - t0
    if not ix:
        raise MemoryError("iib_build allocation failed")
    try:
        sel = np.arange(R.n_rows, dtype=np.int64) if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
        n = len(sel)
        ids = np.empty((n, k), dtype=np.int64)
        scores = np.empty((n, k), dtype=np.float64)
        threads = max(1, min(threads, max(n, 1)))
        bounds = np.linspace(0, n, threads + 1).astype(np.int64)
        visits = np.zeros(threads, dtype=np.int64)

        def work(i):
            a, b = int(bounds[i]), int(bounds[i + 1])
            if b <= a:
                return 0
            sub = sel[a:b]
            v = ctypes.c_int64(0)
            rc = L.iib_query(ix, ctypes.byref(hR.c), sub.ctypes.data, b - a, k, ids[a:b].ctypes.data,
                             scores[a:b].ctypes.data, ctypes.byref(v))
            visits[i] = v.value
            return rc

        t1 = time.perf_counter()
        if threads == 1:
            rc = [work(0)]
        else:
            with ThreadPoolExecutor(threads) as ex:
                rc = list(ex.map(work, range(threads)))
        query_s = time.perf_counter() - t1
        if any(rc):
            raise MemoryError("iib_query allocation failed")
        return ids, scores, {"build_s": build_s, "query_s": query_s, "visits": int(visits.sum())}
    finally:
        L.iib_free(ix)
