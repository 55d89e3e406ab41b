"""The oracle's vectorised bank helpers equal M independent reference-style
1-d calls (so bank-sized parity tests stay pinned to the reference)."""

import math

import numpy as np

from oracle import parpf_oracle as orc


def test_resample_rows_equals_per_filter_calls():
    rng = np.random.default_rng(3)
    M, N = 37, 257
    lw = (rng.normal(size=(M, N)) * rng.choice([1.0, 10.0], size=(M, 1))).astype(np.float32)
    lw[5] = -np.inf  # a collapsed filter
    u = orc.sorted_uniform_rows(np.random.default_rng(4), M, N)
    anc, lmr, coll, cum = orc.resample_rows(lw, u)
    for f in range(M):
        if f == 5:
            assert coll[f] and np.array_equal(anc[f], np.arange(N))
            continue
        w, lm = orc.normalize_log_weights(lw[f])
        c = np.cumsum(w)
        assert np.array_equal(c, cum[f])
        assert lm == lmr[f]
        assert np.array_equal(orc.resample_indices(c, u[f]), anc[f])


def test_sorted_uniform_rows_match_reference_draws():
    a = orc.sorted_uniform_rows(np.random.default_rng(9), 3, 50)
    rng = np.random.default_rng(9)
    for f in range(3):
        assert np.array_equal(a[f], orc.sorted_uniforms(50, rng))
    assert np.all(np.diff(a, axis=1) >= 0) and np.all((a > 0) & (a < 1))
