"""GPU: the data preparation either side of the bank -
hook-level simulate() against the reference's own output, and the
load-or-simulate / proxy-reference harness."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import harness, io  # noqa: E402


def test_simulate_matches_reference_bit_exact(golden):
    """models/simulate.py:10-29 with the stock Lorenz63Model, seed 11."""
    g = golden["lorenz"]
    states, obs = pf.simulate.simulate(pf.Lorenz63Model(), 20, 11)
    assert states.shape == g["sim_states"].shape and obs.shape == g["sim_obs"].shape
    np.testing.assert_array_equal(states, g["sim_states"])
    np.testing.assert_array_equal(obs, g["sim_obs"])


def test_simulate_zero_steps_and_negative():
    states, obs = pf.simulate.simulate(pf.Lorenz63Model(), 0, 3)
    assert states.shape == (1, 3) and obs.shape == (0, 1)
    with pytest.raises(ValueError):
        pf.simulate.simulate(pf.Lorenz63Model(), -1, 3)


def test_prepare_data_idempotent(tmp_path):
    m = pf.Lorenz63Model()
    yp, xp = str(tmp_path / "y.csv"), str(tmp_path / "x.csv")
    s1, o1 = harness.prepare_data(m, 12, 5, yp, xp)
    text = open(yp).read()
    s2, o2 = harness.prepare_data(m, 12, 5, yp, xp)
    assert open(yp).read() == text
    np.testing.assert_array_equal(s1, s2)
    np.testing.assert_array_equal(o1, o2)
    sim_ss, _, _ = harness.root_sequences(5)
    s3, o3 = pf.simulate.simulate(m, 12, sim_ss)
    np.testing.assert_array_equal(o1, o3)
    _, back = io.read_array_csv(yp)
    np.testing.assert_array_equal(back, o3)


def test_compute_reference_truth_and_proxy():
    m = pf.Lorenz63Model()
    states, obs = harness.prepare_data(m, 15, 9)
    truth = harness.compute_reference(m, states, obs, 9, reference="truth")
    np.testing.assert_array_equal(truth, states[1:])
    proxy = harness.compute_reference(m, states, obs, 9, proxy_particles=4096)
    assert proxy.shape == truth.shape
    again = harness.compute_reference(m, states, obs, 9, proxy_particles=4096)
    np.testing.assert_array_equal(proxy, again)
    # a 4096-particle filter tracks the x1 coordinate it observes
    assert np.sqrt(np.mean((proxy[:, 0] - truth[:, 0]) ** 2)) < 3.0 * np.sqrt(m.obs_var)
