"""Host-side logic that needs no GPU: model descriptors, validation and the
ctypes parameter structs handed to the C ABI."""

import math

import numpy as np
import pytest

import paper_1407_8071_b200 as pf
from paper_1407_8071_b200 import _lib


def test_lorenz_descriptor_matches_reference_defaults():
    m = pf.Lorenz63Model()
    assert (m.s, m.r, m.b, m.dt, m.substeps, m.obs_var, m.prior_var) == (
        10.0, 28.0, 8.0 / 3.0, 1e-3, 100, 0.5, 10.0)  # lorenz63.py:24-31
    assert m.dim_x == 3 and m.dim_y == 1
    p = m.params()
    assert isinstance(p, _lib.LorenzParams)
    assert (p.n_sub, p.obs_dim, p.noise_scale) == (100, 1, 1.0)
    assert m.params(noise_free=True).noise_scale == 0.0
    cfg = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3")
    assert cfg.dim_y == 2 and cfg.params().obs_dim == 2
    assert cfg.prior_sd() == math.sqrt(cfg.prior_var)
    assert cfg.has_point_prediction()


@pytest.mark.parametrize("kw", [dict(substeps=0), dict(obs_var=0.0), dict(prior_var=-1.0),
                                dict(observe="x2")])
def test_lorenz_validation(kw):
    with pytest.raises(ValueError):
        pf.Lorenz63Model(**kw)


def test_fhn_descriptor_cfg3():
    m = pf.FhnLatticeModel(stim_row=4, stim_col=7)
    assert (m.rows, m.cols, m.nodes, m.dim_x, m.dim_y) == (30, 50, 1500, 3000, 100)
    p = m.params()
    assert p.degree_drive == -1.0 and p.coupling == 1.0
    assert p.sig_v == p.sig_w == pytest.approx(0.05 * math.sqrt(0.01))
    assert list(p.cubic) == [-1.0, 1.13, -0.13, 0.0] and list(p.beta) == [0.01, -0.005, 0.0]
    q = m.params(noise_free=True)
    assert q.sig_v == 0.0 and q.sig_w == 0.0
    x0 = m.initial_state()
    v = x0[: m.nodes].reshape(30, 50)
    assert v.sum() == 9.0 and np.all(v[4:7, 7:10] == 1.0) and np.all(x0[m.nodes:] == 0.0)
    rows, cols = np.divmod(m.obs_indices, 50)
    assert sorted(set(rows)) == list(range(1, 30, 3)) and sorted(set(cols)) == list(range(2, 50, 5))
    np.testing.assert_array_equal(m.error_projection(np.arange(3000.0)[None]), np.arange(1500.0)[None])


def test_fhn_validation():
    with pytest.raises(ValueError):
        pf.FhnLatticeModel(substeps=0)
    with pytest.raises(ValueError):
        pf.FhnLatticeModel(rows=5, cols=5)  # electrodes do not fit


def test_time_error_index_and_estimate_lookup():
    assert pf.time_error_index("centralised", 4, 100) == 1.0
    assert pf.time_error_index("ensemble", 4, 100) == pytest.approx(0.26)
    with pytest.raises(ValueError):
        pf.time_error_index("other", 1, 1)
    with pytest.raises(ValueError):
        pf.time_error_index("ensemble", 0, 1)
    out = pf.EnsembleOutput("bootstrap", 1, 1, 0, [], np.zeros((3, 2)), np.zeros(1), 0.0)
    assert out.n_steps == 3
    with pytest.raises(ValueError):
        pf.ensemble_estimate(out, 3)


def test_particle_approximation_validation():
    with pytest.raises(ValueError):
        pf.ParticleApproximation(np.zeros((3, 1)), np.array([0.5, 0.2, 0.2]))
    with pytest.raises(ValueError):
        pf.ParticleApproximation(np.zeros((0, 2)), np.array([]))
    a = pf.ParticleApproximation(np.array([1.0, 2.0]), np.array([0.5, 0.5]))
    assert a.particles.shape == (2, 1) and a.n_particles == 2


def test_filter_output_same_result_ignores_timing():
    a = pf.FilterOutput("bootstrap", 4, 0, np.ones((2, 3)), np.zeros(2), np.array([1.0, 2.0]))
    b = pf.FilterOutput("bootstrap", 4, 1, np.ones((2, 3)), np.zeros(2), np.array([9.0, 9.0]))
    assert a.same_result(b) and a.total_seconds == 3.0


def test_draw_tape_defaults():
    t = pf.DrawTape()
    assert t.prior is None and t.noise == [] and t.uniforms == [] and t.uniforms_first == []


def test_raise_status_maps_flags_to_reference_exceptions():
    _lib.raise_status(np.zeros(3, np.int32))
    with pytest.raises(pf.NumericalDivergenceError):
        _lib.raise_status(np.array([0, _lib.PF_ST_DIVERGED | _lib.PF_ST_NAN_WEIGHT]))
    with pytest.raises(ValueError):
        _lib.raise_status(np.array([_lib.PF_ST_NAN_WEIGHT]))


def test_public_api_covers_the_reference_names():
    """Every name parpf and parpf.models export (parpf/__init__.py,
    models/__init__.py) exists here."""
    import paper_1407_8071_b200 as pf
    from paper_1407_8071_b200 import models

    ref_top = ["ConfigError", "EnsembleOutput", "FilterOutput", "IslandSystem", "MetricRecord",
               "NumericalDivergenceError", "ParticleApproximation", "StateSpaceModel",
               "UnsupportedModelError", "WeightCollapseError", "apf_step", "bf_init", "bf_step",
               "bias_variance", "dbf_init", "dbf_step", "empirical_mse", "ensemble_estimate",
               "estimate_integral", "loglog_slope", "multinomial_resample",
               "multinomial_resample_indices", "normalize_log_weights", "posterior_mean",
               "run_double_bootstrap", "run_ensemble", "run_filter", "systematic_resample",
               "systematic_resample_indices", "time_error_index"]
    ref_models = ["DiscreteHmm", "FhnNetworkModel", "LinearGaussianModel", "Lorenz63Model",
                  "fhn_stimulus_region", "hmm_exact_filter", "kalman_filter",
                  "lorenz_log_likelihood", "lorenz_transition", "observation_zone_indices",
                  "simulate", "von_neumann_neighbors"]
    for n in ref_top:
        assert hasattr(pf, n), n
    for n in ref_models:
        assert hasattr(models, n), n
