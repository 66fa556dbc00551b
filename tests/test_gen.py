"""Generator (SURVEY.md §8 row a0, §8(d) sanity table): determinism and workload-shape checks."""
import numpy as np
import pytest

import gen


def test_row_range_regenerates_identically():
    c = gen.CONFIGS["C3"]
    whole = gen.generate(c, "S", 0, 3000)
    part = gen.generate(c, "S", 1000, 500)
    a, b = whole.indptr[1000], whole.indptr[1500]
    np.testing.assert_array_equal(part.indices, whole.indices[a:b])
    again = gen.generate(c, "S", 0, 3000)
    np.testing.assert_array_equal(again.indices, whole.indices)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("which", ["R", "S"])
def test_rows_valid_and_mean_nnz(name, which):
    c = gen.CONFIGS[name]
    spec = c.R if which == "R" else c.S
    n = min(spec.n_rows, 4000)
    h = gen.generate(c, which, 0, n)
    lens = np.diff(h.indptr)
    lo, hi = (spec.nnz_lo, spec.nnz_hi) if spec.count_law == 0 else (2 * (spec.nnz_lo - 1), 2 * (spec.nnz_hi - 1))
    assert lens.min() >= lo and lens.max() <= hi
    assert abs(lens.mean() - (lo + hi) / 2) <= 0.05 * (lo + hi) / 2
    for i in range(0, n, 97):
        idx, val = h.row(i)
        assert np.all(np.diff(idx) > 0) and idx.min() >= 0 and idx.max() < c.d
        if val is not None:
            assert np.all(val > 0) and np.all(np.isfinite(val))
    if spec.value_law == gen.INT8_UNIFORM:
        assert h.values.min() >= spec.val_lo and h.values.max() <= spec.val_hi
    if spec.value_law == gen.LOGNORMAL_UNIT_L2:
        norms = np.sqrt(np.add.reduceat(h.values.astype(np.float64) ** 2, h.indptr[:-1]))
        np.testing.assert_allclose(norms, 1.0, rtol=1e-6)


@pytest.mark.parametrize("name,which,share", [("C2", "S", 0.996), ("C4", "S", 0.978)])
def test_zipf_head_share(name, which, share):
    """§8(d) sanity: top-feature share of S rows (Zipf heads saturate)."""
    h = gen.generate(gen.CONFIGS[name], which, 0, 20000)
    top = np.bincount(h.indices).max() / h.n_rows
    assert abs(top - share) < 0.01
