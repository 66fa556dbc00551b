"""Test helpers: tiny CSR builders and random instances (inputs only, no join arithmetic)."""
import numpy as np

from gen import HostCSR


def csr_from_rows(rows, d, dtype="fp32"):
    """rows: list of list of (d, w) or list of list of d (binary)."""
    indptr = [0]
    idx, val = [], []
    for r in rows:
        for f in r:
            if isinstance(f, (tuple, list)):
                idx.append(int(f[0]))
                val.append(f[1])
            else:
                idx.append(int(f))
                val.append(1)
        indptr.append(len(idx))
    indptr = np.array(indptr, dtype=np.int64)
    idx = np.array(idx, dtype=np.int32)
    if dtype == "binary":
        values = None
    elif dtype == "int8":
        values = np.array(val, dtype=np.int8)
    else:
        values = np.array(val, dtype=np.float32)
    return HostCSR(indptr, idx, values, d)


def random_csr(rng, n, d, lo, hi, dtype, vmax=3):
    """Random rows with distinct ascending features; small ranges give many exact ties."""
    rows = []
    for _ in range(n):
        c = int(rng.integers(lo, hi + 1))
        c = min(c, d)
        f = np.sort(rng.choice(d, size=c, replace=False))
        if dtype == "binary":
            rows.append([int(x) for x in f])
        elif dtype == "int8":
            rows.append([(int(x), int(rng.integers(1, vmax + 1))) for x in f])
        else:
            rows.append([(int(x), float(np.float32(rng.lognormal()))) for x in f])
    return csr_from_rows(rows, d, dtype)


def to_scipy(csr):
    import scipy.sparse as sp
    vals = np.ones(csr.nnz, dtype=np.float64) if csr.values is None else csr.values.astype(np.float64)
    return sp.csr_matrix((vals, csr.indices, csr.indptr), shape=(csr.n_rows, csr.d))


def scipy_topk(R, S, k):
    """Independent pin: textbook SpGEMM R @ S.T, then numpy lexsort by (score desc, id asc)."""
    M = (to_scipy(R) @ to_scipy(S).T).toarray()
    ids = np.full((R.n_rows, k), -1, dtype=np.int64)
    sc = np.zeros((R.n_rows, k), dtype=np.float64)
    for i in range(R.n_rows):
        row = M[i]
        pos = np.nonzero(row > 0)[0]
        order = np.lexsort((pos, -row[pos]))[:k]
        ids[i, :len(order)] = pos[order]
        sc[i, :len(order)] = row[pos[order]]
    return ids, sc, M


def stable_seed(*parts) -> int:
    """A per-case seed that is the same in every process (Python's hash() of strings is salted per process)."""
    import zlib
    return zlib.crc32(repr(parts).encode())
