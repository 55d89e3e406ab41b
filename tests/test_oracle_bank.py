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


def test_streaming_ensemble_equals_run_ensemble():
    """oracle.tapes.StreamingEnsemble (the full-size oracle-mode runs) draws
    and computes exactly what run_ensemble does."""
    from oracle import tapes

    truth0, _, obs = orc.lorenz_truth(seed=3, n_obs=4)
    m = orc.LorenzConfigModel(prior_mean=tuple(truth0))
    traces, _ = orc.run_ensemble(m, obs, 3, 50, 7, keep_steps=True)
    se = tapes.StreamingEnsemble(m, obs, 3, 50, 7)
    assert np.array_equal(se.prior, np.stack([t.prior_noise for t in traces]))
    for k in range(4):
        r = se.step(k)
        assert np.array_equal(r["noise"], np.stack([t.steps[k].noise for t in traces]))
        assert np.array_equal(r["ancestors"], np.stack([t.steps[k].ancestors for t in traces]))
        assert np.array_equal(r["estimates"], np.stack([t.estimates[k] for t in traces]))
        assert np.array_equal(r["lnc"], np.array([t.log_norm_const[k] for t in traces]))
