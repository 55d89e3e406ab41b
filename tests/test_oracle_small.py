"""Pin the oracle restatements of the verification models (DiscreteHmm,
LinearGaussianModel) to the reference: bit-exact against
tests/golden/small.npz, the only tolerance being the BLAS-ordered 2-D
linear-Gaussian case."""

import numpy as np

from oracle import parpf_oracle as orc

HMM = dict(prior=[0.5, 0.5], transition=[[0.9, 0.1], [0.2, 0.8]],
           emission=[[0.8, 0.2], [0.3, 0.7]])
HOBS = np.array([[0.0], [1.0], [0.0], [0.0], [1.0]])


def test_hmm_filter_and_ensemble(golden):
    g = golden["small"]
    m = orc.DiscreteHmmModel(**HMM)
    tr = orc.run_filter(m, HOBS, 50, np.random.SeedSequence(7102), keep_steps=True)
    assert np.array_equal(tr.estimates, g["h_est"])
    assert np.array_equal(tr.log_norm_const, g["h_lnc"])
    assert np.array_equal(np.stack([s.ancestors for s in tr.steps]), g["h_anc"])
    traces, mean = orc.run_ensemble(m, HOBS, 3, 20, 44)
    assert np.array_equal(mean, g["he_mean"])
    st, ob = orc.simulate(m, 30, 5)
    assert np.array_equal(st, g["h_sim_states"]) and np.array_equal(ob, g["h_sim_obs"])


def test_lgm_scalar_filters(golden):
    g = golden["small"]
    m = orc.LinearGaussianOracle.scalar(a=0.9)
    st, ob = orc.simulate(m, 10, 12)
    assert np.array_equal(st, g["l_sim_states"]) and np.array_equal(ob, g["l_obs"])
    tr = orc.run_filter(m, ob, 64, np.random.SeedSequence(7103), keep_steps=True)
    assert np.array_equal(tr.estimates, g["l_est"])
    assert np.array_equal(tr.log_norm_const, g["l_lnc"])
    tr = orc.run_filter(m, ob, 40, np.random.SeedSequence(71), variant="auxiliary")
    assert np.array_equal(tr.estimates, g["la_est"])
    assert np.array_equal(tr.log_norm_const, g["la_lnc"])


def test_lgm_2d_filter(golden):
    g = golden["small"]
    m = orc.LinearGaussianOracle([[0.9, 0.1], [-0.2, 0.8]], [[1.0, 0.3], [0.3, 0.5]],
                                 [[1.0, 0.5]], [[0.7]], [0.5, -0.5], [[1.0, 0.2], [0.2, 2.0]])
    tr = orc.run_filter(m, g["l2_obs"], 32, np.random.SeedSequence(5))
    assert np.allclose(tr.estimates, g["l2_est"], rtol=1e-12, atol=1e-12)
    assert np.allclose(tr.log_norm_const, g["l2_lnc"], rtol=1e-12, atol=1e-12)


def test_double_bootstrap_bit_exact(golden):
    """filters.py:201-313 restated: island selection every period steps."""
    g = golden["small"]
    tr = orc.run_double_bootstrap(orc.DiscreteHmmModel(**HMM), HOBS, 3, 20, 2,
                                  np.random.SeedSequence(606))
    assert np.array_equal(tr.estimates, g["db_h_est"])
    assert np.array_equal(tr.log_norm_const, g["db_h_lnc"])
    assert tr.collapse_steps == g["db_h_coll"].tolist()
    assert [s[0] for s in tr.island_steps] == [2, 4]
    gl = golden["lorenz"]
    m = orc.LorenzConfigModel(prior_mean=tuple(gl["truth0"]))
    tr = orc.run_double_bootstrap(m, gl["obs"][:12], 4, 30, 5, np.random.SeedSequence(99))
    assert np.array_equal(tr.estimates, gl["db_est"])
    assert np.array_equal(tr.log_norm_const, gl["db_lnc"])
