"""Pin the oracle's FH-N network restatement (models/fhn.py:85-207) to the
reference: bit-exact against tests/golden/fhnnet.npz plus the hand values of
the reference's own unit tests (tests/test_models_fhn.py)."""

import numpy as np
import pytest

from oracle import parpf_oracle as orc


def m8(golden, **kw):
    return orc.FhnNetworkModel(J=8, n_zones=2, zone_width=2,
                               stim_prob=float(golden["fhnnet"]["m8_stim_prob"]), **kw)


def test_simulate_bit_exact(golden):
    g = golden["fhnnet"]
    st, ob = orc.simulate(m8(golden), 120, 3)
    assert np.array_equal(st, g["sim8_states"]) and np.array_equal(ob, g["sim8_obs"])
    st, ob = orc.simulate(orc.FhnNetworkModel(J=16, stim_prob=0.02), 150, 3)
    assert np.array_equal(st, g["sim16_states"]) and np.array_equal(ob, g["sim16_obs"])
    # the record contains stimuli (the golden exercises the stimulus path)
    q0 = g["sim8_states"][:, 128:192]
    assert q0.sum() > 0


def test_hooks_bit_exact(golden):
    g = golden["fhnnet"]
    m = m8(golden)
    assert np.array_equal(m.transition_point_prediction(g["hook_x"], 1), g["tpp_t1"])
    assert np.array_equal(m.transition_point_prediction(g["hook_x"], 250), g["tpp_t250"])
    mf = m8(golden)
    mf.stim_prob = 1.0
    out = mf.sample_transition(g["band_x"], 7, np.random.default_rng(19))
    assert np.array_equal(out, g["band_out"])
    assert np.array_equal(m.log_likelihood(g["ll_y"], g["hook_x"], 1), g["ll_out"])


def test_bootstrap_filter_bit_exact(golden):
    g = golden["fhnnet"]
    tr = orc.run_filter(m8(golden), g["sim8_obs"][:60], 32, np.random.SeedSequence(808),
                        keep_steps=True)
    assert np.array_equal(tr.estimates, g["f_est"])
    assert np.array_equal(tr.log_norm_const, g["f_lnc"])
    assert np.array_equal(np.stack([s.ancestors for s in tr.steps]), g["f_anc"])
    assert np.array_equal(np.stack([s.u for s in tr.steps]), g["f_u"])


def test_auxiliary_filter_bit_exact(golden):
    g = golden["fhnnet"]
    tr = orc.run_filter(m8(golden), g["sim8_obs"][:40], 24, np.random.SeedSequence(909),
                        keep_steps=True, variant="auxiliary")
    assert np.array_equal(tr.estimates, g["a_est"])
    assert np.array_equal(tr.log_norm_const, g["a_lnc"])
    assert np.array_equal(np.stack([s.anc_first for s in tr.steps]), g["a_anc1"])
    assert np.array_equal(np.stack([s.ancestors for s in tr.steps]), g["a_anc2"])


def test_ensemble_bit_exact(golden):
    g = golden["fhnnet"]
    traces, mean = orc.run_ensemble(m8(golden), g["sim8_obs"][:40], 3, 16, 21)
    assert np.array_equal(mean, g["e_mean"])
    assert np.array_equal(np.stack([t.log_norm_const for t in traces]), g["e_lnc"])


# ---- hand values of the reference unit tests (test_models_fhn.py) ----------

def test_neighbours_and_region():
    assert set(orc.lattice_neighbors(0, 0, 4)) == {(0, 1), (1, 0)}
    assert len(orc.lattice_neighbors(0, 2, 4)) == 3 and len(orc.lattice_neighbors(2, 2, 4)) == 4
    U = np.zeros((3, 3))
    U[1, 1] = -1.7
    assert set(zip(*np.nonzero(orc.stimulus_region(U)))) == {(1, 1), (0, 1), (2, 1), (1, 0),
                                                             (1, 2)}
    assert not orc.stimulus_region(np.full((2, 2), -1.8)).any()
    assert not orc.stimulus_region(np.full((2, 2), -1.6)).any()
    U = np.zeros((2, 3, 3))
    U[1, 0, 0] = -1.75
    r = orc.stimulus_region(U)
    assert not r[0].any() and r[1].sum() == 3


def test_euler_hand_values():
    m = orc.FhnNetworkModel(J=1, coupling=0.0, forcing_amp=0.0, n_zones=1, zone_width=1,
                            cubic=(1.0, 0.0, -3.6, 0.0))
    x = np.zeros((1, m.dim_x))
    x[0, 0] = 1.0
    out = m.transition_point_prediction(x, 1)
    assert out[0, 0] == pytest.approx(0.987, rel=1e-14)
    assert out[0, 1] == pytest.approx(0.0135, rel=1e-14)
    m = orc.FhnNetworkModel(J=1, coupling=0.0, forcing_amp=0.0, n_zones=1, zone_width=1)
    assert m.transition_point_prediction(x, 1)[0, 0] == pytest.approx(1.013, rel=1e-14)
    m = orc.FhnNetworkModel(J=2, forcing_amp=0.0, n_zones=1, zone_width=1)
    x = np.zeros((1, m.dim_x))
    x[0, 0] = 1.0
    u = m.transition_point_prediction(x, 1)[0, :4].reshape(2, 2)
    assert u[0, 1] == pytest.approx(5e-3 * 4.5e-3, rel=1e-12) and u[1, 1] == 0.0


def test_zones_forcing_and_dims():
    assert orc.zone_indices(32).shape == (100,) and orc.zone_indices(16).shape == (100,)
    with pytest.raises(ValueError):
        orc.zone_indices(8, 5, 2)
    m = orc.FhnNetworkModel(J=16)
    assert m.dim_y == 100 and m.dim_x == 27 * 256
    m = orc.FhnNetworkModel(J=4, n_zones=2, zone_width=2)
    period, width = int(m.forcing_period / m.dt), int(m.forcing_width / m.dt)
    assert m.forcing_value(1) == m.forcing_amp and m.forcing_value(width) == m.forcing_amp
    assert m.forcing_value(width + 1) == 0.0 and m.forcing_value(period + 1) == m.forcing_amp
    with pytest.raises(ValueError):
        orc.FhnNetworkModel(u_minus=-1.0, u_plus=-1.5)
    with pytest.raises(ValueError):
        orc.FhnNetworkModel(stim_hold=0)
