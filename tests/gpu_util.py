"""Helpers for the -m gpu parity tests: run the CUDA path through the C ABI and compare with the oracle
under the rules of DESIGN.md (reading c15 / c17)."""
import numpy as np
import torch

import oracle

TOL = 1e-5  # BASELINE.json north_star: fp32 scores within 1e-5 relative


def gpu_join(R, S, k, d=None, tile=0, batch_rows=0, s_id_base=0, want_keys=False, counters=None, head_density=0.0,
             head_max=0, cta_warps=0, tiles_per_pass=0, row_order=0, prune=0, alpha=0.0, prune_alpha=0.0,
             precision=0, uncertified=None):
    import paper_1011_2807_b200 as kj
    d = d or R.d
    dS = kj.DeviceCSR.from_host(S)
    dR = kj.DeviceCSR.from_host(R)
    idx = kj.knnjoin_build_index(dS, d, s_id_base=s_id_base, tile=tile, head_density=head_density, head_max=head_max,
                                 prune=prune, alpha=alpha)
    ids, sc, keys = kj.knnjoin_query(idx, dR, k, want_keys=want_keys, batch_rows=batch_rows, counters=counters,
                                     cta_warps=cta_warps, tiles_per_pass=tiles_per_pass, row_order=row_order,
                                     prune_alpha=prune_alpha, precision=precision, uncertified=uncertified)
    torch.cuda.synchronize()
    out = (ids.cpu().numpy().astype(np.int64), sc.cpu().numpy().astype(np.float64))
    if want_keys:
        out = out + (keys.cpu().numpy(),)
    return out


def assert_parity(R, S, g_ids, g_sc, o_ids, o_sc, rows=None, s_id_base=0):
    """Integer inputs: positional equality of ids and scores.  FP32 inputs, at every position i
    (x = oracle exact score of an id): (1) g_i == o_i or |x(g_i) - x(o_i)| <= TOL*x(o_i);
    (2) |y_i - x(g_i)| <= TOL*x(g_i); (3) ids distinct; (4) padding positions identical."""
    rows = np.arange(R.n_rows) if rows is None else np.asarray(rows)
    integer = R.dtype != "fp32" and S.dtype != "fp32"
    if integer:
        np.testing.assert_array_equal(g_ids, o_ids)
        np.testing.assert_array_equal(g_sc, o_sc)
        return
    n, k = o_ids.shape
    pad_g = g_ids < 0
    pad_o = o_ids < 0
    np.testing.assert_array_equal(pad_g, pad_o, err_msg="padding positions differ")
    assert np.all(g_sc[pad_g] == 0)
    r_rep = np.repeat(rows, k)
    xg = oracle.pair_scores(R, S, r_rep, np.where(g_ids.ravel() >= 0, g_ids.ravel() - s_id_base, -1)).reshape(n, k)
    for i in range(n):
        valid = ~pad_g[i]
        gi = g_ids[i][valid]
        assert len(set(gi.tolist())) == len(gi), f"row {rows[i]}: duplicate ids"
        for t in np.nonzero(valid)[0]:
            if g_ids[i, t] != o_ids[i, t]:
                assert abs(xg[i, t] - o_sc[i, t]) <= TOL * o_sc[i, t], \
                    f"row {rows[i]} pos {t}: id {g_ids[i, t]} (x={xg[i, t]}) vs oracle {o_ids[i, t]} (x={o_sc[i, t]})"
            assert abs(g_sc[i, t] - xg[i, t]) <= TOL * xg[i, t], \
                f"row {rows[i]} pos {t}: score {g_sc[i, t]} vs exact {xg[i, t]}"
