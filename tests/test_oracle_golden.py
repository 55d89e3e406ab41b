"""Pin the CPU oracle to the reference: bit-exact against tests/golden/*.npz.

The fixtures were produced by tests/golden/make_golden.py from the unmodified
reference (parpf) in the build container.  If these pass, every GPU parity
test that compares against the oracle is transitively a comparison against
the reference.
"""

import numpy as np
import pytest

from oracle import parpf_oracle as orc


def test_normalize_log_weights_golden(golden):
    g = golden["kernels"]
    for i in range(int(g["nlw_count"])):
        w, lm = orc.normalize_log_weights(g[f"nlw_in_{i}"])
        assert np.array_equal(w, g[f"nlw_w_{i}"])
        assert lm == float(g[f"nlw_lm_{i}"])


def test_normalize_log_weights_errors():
    with pytest.raises(orc.WeightCollapseError):
        orc.normalize_log_weights(np.full(8, -np.inf))
    with pytest.raises(ValueError):
        orc.normalize_log_weights(np.array([0.0, np.nan]))
    with pytest.raises(ValueError):
        orc.normalize_log_weights(np.array([]))


def test_resample_indices_golden(golden):
    g = golden["kernels"]
    for i in range(int(g["ri_count"])):
        idx = orc.resample_indices(g[f"ri_cum_{i}"], g[f"ri_u_{i}"])
        assert idx.dtype == np.int64
        assert np.array_equal(idx, g[f"ri_idx_{i}"]), i
    # tie case never selects the zero-weight particle (test_accel.py:57-64)
    assert not np.any(orc.resample_indices(g["ri_cum_0"], g["ri_u_0"]) == 1)


def test_multinomial_resample_golden(golden):
    g = golden["kernels"]
    idx = orc.multinomial_resample_indices(g["mri_w"], 500, np.random.default_rng(77))
    assert np.array_equal(idx, g["mri_idx"])


def test_lorenz_block_golden(golden):
    g = golden["kernels"]
    out = orc.lorenz_euler_block(g["lz_states"], g["lz_noise"], 1e-3, 10.0, 28.0, 8.0 / 3.0)
    assert np.array_equal(out, g["lz_out"])


@pytest.mark.parametrize("tag", ["rect", "sq"])
def test_fhn_block_golden(golden, tag):
    g = golden["kernels"]
    p = g[f"fhn_{tag}_params"]
    dt, cpl, cubic, beta, sig = p[0], p[1], tuple(p[2:6]), tuple(p[6:9]), p[9]
    u, v = orc.fhn_euler_block(g[f"fhn_{tag}_U"], g[f"fhn_{tag}_V"], g[f"fhn_{tag}_drive"],
                               g[f"fhn_{tag}_noise"], dt, cpl, cubic, beta, sig)
    assert np.array_equal(u, g[f"fhn_{tag}_u_new"])
    assert np.array_equal(v, g[f"fhn_{tag}_v_new"])


def _lorenz_model(g):
    return orc.LorenzConfigModel(prior_mean=tuple(g["truth0"]))


def test_lorenz_filter_golden(golden):
    g = golden["lorenz"]
    tr = orc.run_filter(_lorenz_model(g), g["obs"], 64,
                        np.random.SeedSequence(int(g["f_seed_entropy"])), keep_steps=True)
    assert np.array_equal(tr.estimates, g["f_est"])
    assert np.array_equal(tr.log_norm_const, g["f_lnc"])
    assert np.array_equal(np.stack([s.ancestors for s in tr.steps]), g["f_anc"])
    assert np.array_equal(np.stack([s.u for s in tr.steps]), g["f_u"])


def test_lorenz_ensemble_golden(golden):
    g = golden["lorenz"]
    traces, mean = orc.run_ensemble(_lorenz_model(g), g["obs"], 4, 100, int(g["e_master"]))
    assert np.array_equal(mean, g["e_mean"])
    assert np.array_equal(np.stack([t.estimates for t in traces]), g["e_est"])
    assert np.array_equal(np.stack([t.log_norm_const for t in traces]), g["e_lnc"])


def test_lorenz_ensemble_pool_identical(golden):
    g = golden["lorenz"]
    _, serial = orc.run_ensemble(_lorenz_model(g), g["obs"][:5], 3, 50, 9, workers=1)
    _, pooled = orc.run_ensemble(_lorenz_model(g), g["obs"][:5], 3, 50, 9, workers=2)
    assert serial.tobytes() == pooled.tobytes()


def test_lorenz_collapse_golden(golden):
    g = golden["lorenz"]
    tr = orc.run_filter(_lorenz_model(g), g["c_obs"], 32, 11)
    assert tr.collapse_steps == list(g["c_steps"])
    assert np.array_equal(tr.estimates, g["c_est"])
    assert np.array_equal(tr.log_norm_const, g["c_lnc"])


def _fhn_model(g):
    return orc.FhnConfigModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))


def test_fhn_truth_patch_matches_fixture(golden):
    g = golden["fhn"]
    m, _, obs = orc.fhn_truth(seed=7, n_obs=3)
    assert (m.stim_row, m.stim_col) == tuple(int(v) for v in g["stim"])
    assert np.array_equal(obs, g["obs"])


def test_fhn_filter_golden(golden):
    g = golden["fhn"]
    m = _fhn_model(g)
    tr = orc.run_filter(m, g["obs"], 8, np.random.SeedSequence(99), keep_steps=True)
    assert np.array_equal(tr.estimates[:, : m.nodes], g["f_est_v"])
    assert np.array_equal(tr.log_norm_const, g["f_lnc"])
    assert np.array_equal(np.stack([s.ancestors for s in tr.steps]), g["f_anc"])


def test_fhn_ensemble_golden(golden):
    g = golden["fhn"]
    m = _fhn_model(g)
    traces, mean = orc.run_ensemble(m, g["obs"][:2], 2, 4, 17)
    assert np.array_equal(mean[:, : m.nodes], g["e_mean_v"])
    assert np.array_equal(np.stack([t.log_norm_const for t in traces]), g["e_lnc"])


def test_electrodes_regular_subgrid():
    idx = orc.electrode_indices(30, 50)
    assert idx.shape == (100,)
    rows, cols = np.divmod(idx, 50)
    assert sorted(set(rows)) == list(range(1, 30, 3))
    assert sorted(set(cols)) == list(range(2, 50, 5))


def test_tape_recorder_reproduces_seeded_run(golden):
    """The recorder changes nothing about the stream."""
    g = golden["lorenz"]
    rec = orc.TapeRecorder(np.random.SeedSequence(int(g["f_seed_entropy"])))
    tr = orc.run_filter(_lorenz_model(g), g["obs"], 64, rec)
    assert np.array_equal(tr.estimates, g["f_est"])
    kinds = [k for k, _ in rec.log]
    assert kinds[0] == "normal" and kinds[1] == "normal" and kinds[2] == "exponential"


# ---- the oracle's C kernels (CPU baseline) are bit-identical too ----------

def _ck():
    from oracle import ckernels

    try:
        ckernels.load()
    except FileNotFoundError:
        import subprocess

        subprocess.run(["make", "-s", "-C", "oracle"], check=True)
    return ckernels


def test_ckernels_lorenz_golden(golden):
    g = golden["kernels"]
    out = _ck().lorenz_euler_block(g["lz_states"], g["lz_noise"], 1e-3, 10.0, 28.0, 8.0 / 3.0)
    assert np.array_equal(out, g["lz_out"])


@pytest.mark.parametrize("tag", ["rect", "sq"])
def test_ckernels_fhn_golden(golden, tag):
    g = golden["kernels"]
    p = g[f"fhn_{tag}_params"]
    u, v = _ck().fhn_euler_block(g[f"fhn_{tag}_U"], g[f"fhn_{tag}_V"], g[f"fhn_{tag}_drive"],
                                 g[f"fhn_{tag}_noise"], p[0], p[1], tuple(p[2:6]),
                                 tuple(p[6:9]), p[9])
    assert np.array_equal(u, g[f"fhn_{tag}_u_new"])
    assert np.array_equal(v, g[f"fhn_{tag}_v_new"])


def test_ckernels_resample_golden(golden):
    g = golden["kernels"]
    for i in range(int(g["ri_count"])):
        assert np.array_equal(_ck().resample_indices(g[f"ri_cum_{i}"], g[f"ri_u_{i}"]),
                              g[f"ri_idx_{i}"])


# ---- auxiliary particle filter (filters.py:115-154) -----------------------

def test_lorenz_apf_filter_golden(golden):
    g = golden["lorenz"]
    tr = orc.run_filter(_lorenz_model(g), g["obs"][:12], 48, np.random.SeedSequence(4242),
                        keep_steps=True, variant="auxiliary")
    assert np.array_equal(tr.estimates, g["a_est"])
    assert np.array_equal(tr.log_norm_const, g["a_lnc"])
    assert np.array_equal(np.stack([s.anc_first for s in tr.steps]), g["a_anc1"])
    assert np.array_equal(np.stack([s.u_first for s in tr.steps]), g["a_u1"])
    assert np.array_equal(np.stack([s.ancestors for s in tr.steps]), g["a_anc2"])
    assert np.array_equal(np.stack([s.u for s in tr.steps]), g["a_u2"])


def test_lorenz_apf_ensemble_golden(golden):
    g = golden["lorenz"]
    traces, mean = orc.run_ensemble(_lorenz_model(g), g["obs"][:12], 3, 64, 8,
                                    variant="auxiliary")
    assert np.array_equal(mean, g["ae_mean"])
    assert np.array_equal(np.stack([t.log_norm_const for t in traces]), g["ae_lnc"])


def test_lorenz_apf_collapse_golden(golden):
    g = golden["lorenz"]
    tr = orc.run_filter(_lorenz_model(g), g["c_obs"], 16, 12, variant="auxiliary")
    assert tr.collapse_steps == list(g["ac_steps"])
    assert np.array_equal(tr.estimates, g["ac_est"])
    assert np.array_equal(tr.log_norm_const, g["ac_lnc"])


def test_fhn_apf_filter_golden(golden):
    g = golden["fhn"]
    m = _fhn_model(g)
    tr = orc.run_filter(m, g["obs"], 6, np.random.SeedSequence(5151), keep_steps=True,
                        variant="auxiliary")
    assert np.array_equal(tr.estimates[:, : m.nodes], g["a_est_v"])
    assert np.array_equal(tr.log_norm_const, g["a_lnc"])
    assert np.array_equal(np.stack([s.anc_first for s in tr.steps]), g["a_anc1"])
    assert np.array_equal(np.stack([s.ancestors for s in tr.steps]), g["a_anc2"])
