"""The statistical fixture (tests/golden/stats.npz, written by
tests/golden/make_stats.py from the UNMODIFIED reference) is pinned to the
CPU oracle: the oracle's run_ensemble reproduces the reference's per-seed
MSE for the first seeds bit-for-bit, so the GPU statistical tests compare
against the reference algorithm and not against an unverified number."""

import os

import numpy as np
import pytest

from oracle import ckernels
from oracle import parpf_oracle as orc

ST = np.load(os.path.join(os.path.dirname(__file__), "golden", "stats.npz"))


def test_fixture_shapes_and_sizes():
    truth_seed, T, M, N, pm, pn = (int(v) for v in ST["meta"][:6])
    assert (T, M, N) == (500, 4, 1000)  # BASELINE cfg0
    assert pm * pn >= 100_000  # J >= 1e5 proxy
    assert ST["lz_proxy"].shape == (T, 3)
    assert ST["lz_mse"].size >= 4096 and ST["lz_var_s"].size == ST["lz_mse"].size
    assert ST["fhn_mse"].size >= 64


@pytest.mark.parametrize("seed", [0, 1])
def test_lorenz_fixture_seed_reproduced_by_oracle(seed):
    ckernels.install()
    truth_seed, T, M, N = (int(v) for v in ST["meta"][:4])
    truth0, _, obs = orc.lorenz_truth(seed=truth_seed, n_obs=T)
    om = orc.LorenzConfigModel(prior_mean=tuple(truth0))
    _, mean = orc.run_ensemble(om, obs, M, N, seed, workers=min(M, orc.cpu_cores()))
    mse = ((mean - ST["lz_proxy"]) ** 2).mean()
    assert mse == pytest.approx(ST["lz_mse"][seed], rel=1e-12)


def test_fhn_fixture_seed_reproduced_by_oracle():
    ckernels.install()
    truth_seed, T, M, N = (int(v) for v in ST["meta"][7:11])
    m, states, obs = orc.fhn_truth(seed=truth_seed, n_obs=T)
    _, mean = orc.run_ensemble(m, obs, M, N, 0, workers=min(M, orc.cpu_cores()))
    mse = ((mean[:, : m.nodes] - states[:, : m.nodes]) ** 2).mean()
    assert mse == pytest.approx(ST["fhn_mse"][0], rel=1e-12)
