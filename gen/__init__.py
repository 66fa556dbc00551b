"""Seeded synthetic CSR inputs for the five BASELINE.json configs (recipe §8(d)).

Shared by both sides as INPUT ONLY: the oracle (tests, bench cpu_baseline) and the CUDA path draw their
rows from here.  Nothing here computes a dot product, an index or a top-k.  See gen.c for the per-row law.

Each config lists, per set (R, S): rows, count law, feature law, value law, plus d and k.  ``scaled`` lets
tests keep a config's laws (shape of the workload) with fewer rows.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libknngen.so")
_lock = threading.Lock()
_lib = None

# value laws
BINARY, LOGNORMAL, LOGNORMAL_UNIT_L2, INT8_UNIFORM = 0, 1, 2, 3
# feature laws
UNIFORM, ZIPF, BANDS = 0, 1, 2


class _Spec(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64),
        ("d", ctypes.c_int32),
        ("count_law", ctypes.c_int32),
        ("nnz_lo", ctypes.c_int32),
        ("nnz_hi", ctypes.c_int32),
        ("feat_law", ctypes.c_int32),
        ("zipf_a", ctypes.c_double),
        ("n_bands", ctypes.c_int32),
        ("band_sigma", ctypes.c_double),
        ("value_law", ctypes.c_int32),
        ("val_lo", ctypes.c_int32),
        ("val_hi", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("config_id", ctypes.c_uint32),
        ("set_id", ctypes.c_uint32),
    ]


@dataclasses.dataclass(frozen=True)
class SetSpec:
    n_rows: int
    nnz_lo: int
    nnz_hi: int
    count_law: int = 0  # 0 uniform count, 1 peptide 2*(L-1) with L uniform in [lo, hi]
    feat_law: int = UNIFORM
    zipf_a: float = 1.0
    n_bands: int = 5
    band_sigma: float = 800.0
    value_law: int = BINARY
    val_lo: int = 1
    val_hi: int = 15


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    config_id: int
    d: int
    k: int
    R: SetSpec
    S: SetSpec
    seed: int = 0

    def scaled(self, n_r: int | None = None, n_s: int | None = None) -> "Config":
        """Same laws (workload shape), fewer rows: for parity tests the oracle finishes in seconds."""
        R = dataclasses.replace(self.R, n_rows=n_r if n_r is not None else self.R.n_rows)
        S = dataclasses.replace(self.S, n_rows=n_s if n_s is not None else self.S.n_rows)
        return dataclasses.replace(self, R=R, S=S)

    @property
    def pairs(self) -> int:
        return self.R.n_rows * self.S.n_rows


# BASELINE.json configs[0..4]; unspecified details fixed in SURVEY.md §8(d) / DESIGN.md "Input recipe".
CONFIGS = {
    "C1": Config("C1", 1, 10_000, 10,
                 R=SetSpec(1_000, 20, 60, feat_law=UNIFORM, value_law=BINARY),
                 S=SetSpec(10_000, 20, 60, feat_law=UNIFORM, value_law=BINARY)),
    "C2": Config("C2", 2, 10_000, 10,
                 R=SetSpec(10_000, 50, 200, feat_law=ZIPF, zipf_a=1.1, value_law=LOGNORMAL_UNIT_L2),
                 S=SetSpec(100_000, 20, 60, feat_law=ZIPF, zipf_a=1.1, value_law=BINARY)),
    "C3": Config("C3", 3, 10_000, 5,
                 R=SetSpec(50_000, 100, 300, feat_law=BANDS, value_law=LOGNORMAL),
                 S=SetSpec(1_000_000, 7, 30, count_law=1, feat_law=BANDS, value_law=BINARY)),
    "C4": Config("C4", 4, 10_000, 10,
                 R=SetSpec(100_000, 100, 200, feat_law=ZIPF, zipf_a=1.0, value_law=LOGNORMAL),
                 S=SetSpec(10_000_000, 20, 60, feat_law=ZIPF, zipf_a=1.0, value_law=BINARY)),
    "C5": Config("C5", 5, 100_000, 100,
                 R=SetSpec(20_000, 500, 1000, feat_law=UNIFORM, value_law=INT8_UNIFORM, val_lo=1, val_hi=15),
                 S=SetSpec(500_000, 500, 1000, feat_law=UNIFORM, value_law=INT8_UNIFORM, val_lo=1, val_hi=15)),
}

# dtype names shared with the C ABI (knnjoin_dtype): BINARY=0, INT8=1, FP32=2
VALUE_DTYPE = {BINARY: "binary", LOGNORMAL: "fp32", LOGNORMAL_UNIT_L2: "fp32", INT8_UNIFORM: "int8"}


def _build_lib() -> None:
    src = os.path.join(_HERE, "gen.c")
    tmp = _SO + f".tmp{os.getpid()}"
    subprocess.check_call(["gcc", "-O2", "-fopenmp", "-shared", "-fPIC", "-o", tmp, src, "-lm"])
    os.replace(tmp, _SO)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            src = os.path.join(_HERE, "gen.c")
            if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
                _build_lib()
            L = ctypes.CDLL(_SO)
            L.gen_row_counts.argtypes = [ctypes.POINTER(_Spec), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
            L.gen_fill.argtypes = [ctypes.POINTER(_Spec), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_void_p]
            L.gen_row_counts.restype = ctypes.c_int
            L.gen_fill.restype = ctypes.c_int
            _lib = L
    return _lib


def _spec(cfg: Config, which: str) -> _Spec:
    s = cfg.R if which == "R" else cfg.S
    return _Spec(s.n_rows, cfg.d, s.count_law, s.nnz_lo, s.nnz_hi, s.feat_law, s.zipf_a, s.n_bands,
                 s.band_sigma, s.value_law, s.val_lo, s.val_hi, cfg.seed, cfg.config_id,
                 0 if which == "R" else 1)


@dataclasses.dataclass
class HostCSR:
    """CSR on the host: indptr int64 [n+1] (local, starts at 0), indices int32, values None|int8|float32."""
    indptr: np.ndarray
    indices: np.ndarray
    values: np.ndarray | None
    d: int
    row0: int = 0

    @property
    def n_rows(self) -> int:
        return len(self.indptr) - 1

    @property
    def nnz(self) -> int:
        return int(self.indptr[-1])

    @property
    def dtype(self) -> str:
        if self.values is None:
            return "binary"
        return "int8" if self.values.dtype == np.int8 else "fp32"

    def row(self, i: int):
        a, b = int(self.indptr[i]), int(self.indptr[i + 1])
        v = None if self.values is None else self.values[a:b]
        return self.indices[a:b], v

    def take_rows(self, rows) -> "HostCSR":
        rows = np.asarray(rows, dtype=np.int64)
        lens = self.indptr[rows + 1] - self.indptr[rows]
        indptr = np.zeros(len(rows) + 1, dtype=np.int64)
        np.cumsum(lens, out=indptr[1:])
        idx = np.concatenate([self.indices[self.indptr[r]:self.indptr[r + 1]] for r in rows]) if len(rows) else \
            np.zeros(0, np.int32)
        val = None
        if self.values is not None:
            val = np.concatenate([self.values[self.indptr[r]:self.indptr[r + 1]] for r in rows]) if len(rows) else \
                np.zeros(0, self.values.dtype)
        return HostCSR(indptr, idx.astype(np.int32), val, self.d)


def generate(cfg: Config, which: str, row0: int = 0, n: int | None = None) -> HostCSR:
    """Rows [row0, row0+n) of set ``which`` ('R' or 'S') of config ``cfg``; regenerates identically."""
    L = lib()
    total = (cfg.R if which == "R" else cfg.S).n_rows
    if n is None:
        n = total - row0
    sp = _spec(cfg, which)
    counts = np.empty(n, dtype=np.int32)
    if L.gen_row_counts(ctypes.byref(sp), row0, n, counts.ctypes.data) != 0:
        raise RuntimeError("gen_row_counts failed")
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    nnz = int(indptr[-1])
    indices = np.empty(nnz, dtype=np.int32)
    vl = sp.value_law
    values = None
    if vl in (LOGNORMAL, LOGNORMAL_UNIT_L2):
        values = np.empty(nnz, dtype=np.float32)
    elif vl == INT8_UNIFORM:
        values = np.empty(nnz, dtype=np.int8)
    rc = L.gen_fill(ctypes.byref(sp), row0, n, indptr.ctypes.data, indices.ctypes.data,
                    0 if values is None else values.ctypes.data)
    if rc != 0:
        raise RuntimeError(f"gen_fill failed ({rc})")
    return HostCSR(indptr, indices, values, cfg.d, row0)
