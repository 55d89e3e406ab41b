#!/usr/bin/env python3
"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Everything here calls the reference's own public functions (parpf.accel,
parpf.core, parpf.resampling, parpf.filters.run_filter,
parpf.ensemble.run_ensemble).  The only additions are the config adapters the
BASELINE configs need: subclasses of the reference's
Lorenz63Model / StateSpaceModel that call the reference kernels, and a
recording wrapper around parpf.filters.multinomial_resample_indices that
captures (u, ancestors) per step without changing what it returns.

The fixtures pin oracle/parpf_oracle.py (tests/test_oracle_golden.py, CPU) and
are the golden side of the GPU parity tests (tests/test_gpu_parity.py).
Observations for the filter runs come from oracle.lorenz_truth/fhn_truth;
they are inputs, stored verbatim in the fixtures.
"""

from __future__ import annotations

import math
import os
import sys
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

import parpf  # noqa: E402  (reference, via PYTHONPATH)
from parpf import accel, core, resampling  # noqa: E402
import parpf.filters as ref_filters  # noqa: E402
from parpf.core import StateSpaceModel  # noqa: E402
from parpf.models.lorenz63 import Lorenz63Model  # noqa: E402

from oracle import parpf_oracle as orc  # noqa: E402  (observations only)


# --------------------------------------------------------------------------
# reference-side config adapters
# --------------------------------------------------------------------------


@dataclass
class RefLorenzCfg(Lorenz63Model):
    """cfg0/cfg2 on the reference Lorenz63Model: noise 0.5*z, obs (x1,x3)."""

    noise_scale: float = 0.5

    def __post_init__(self):
        super().__post_init__()
        self.dim_y = 2

    def sample_transition(self, x_prev, t, rng):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        noise = rng.standard_normal((self.substeps, x_prev.shape[0], 3))
        return self._propagate(x_prev, self.noise_scale * noise)

    def log_likelihood(self, y, x, t):
        y = np.asarray(y, dtype=np.float64).reshape(-1)
        x = np.asarray(x)
        r0 = y[0] - x[:, 0]
        r1 = y[1] - x[:, 2]
        return -(r0 * r0 + r1 * r1) / (2.0 * self.obs_var)


class RefFhnCfg(StateSpaceModel):
    """cfg3/cfg4 classical FH-N lattice on the reference numpy twin."""

    def __init__(self, rows, cols, substeps, stim_row, stim_col, dt=0.01,
                 noise_std=0.05, obs_var=0.01):
        self.rows, self.cols, self.substeps = rows, cols, substeps
        self.stim_row, self.stim_col = stim_row, stim_col
        self.dt, self.obs_var = dt, obs_var
        self.nodes = rows * cols
        self.dim_x = 2 * self.nodes
        self.obs_indices = orc.electrode_indices(rows, cols)
        self.dim_y = self.obs_indices.shape[0]
        self.sig = noise_std * math.sqrt(dt)
        deg = np.full((rows, cols), 4.0)
        deg[0, :] -= 1
        deg[-1, :] -= 1
        deg[:, 0] -= 1
        deg[:, -1] -= 1
        self.deg = deg

    def sample_prior(self, rng, n):
        x = np.zeros((n, self.dim_x))
        v = x[:, : self.nodes].reshape(n, self.rows, self.cols)
        v[:, self.stim_row:self.stim_row + 3, self.stim_col:self.stim_col + 3] = 1.0
        return x

    def sample_transition(self, x_prev, t, rng):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        n = x_prev.shape[0]
        U = x_prev[:, : self.nodes].reshape(n, self.rows, self.cols)
        V = x_prev[:, self.nodes:].reshape(n, self.rows, self.cols)
        for _ in range(self.substeps):
            zu = rng.standard_normal((n, self.rows, self.cols))
            zv = rng.standard_normal((n, self.rows, self.cols))
            U, V = accel.fhn_euler_block_numpy(
                U, V, -self.deg * U, zu, self.dt, 1.0, (-1.0, 1.13, -0.13, 0.0),
                (0.01, -0.005, 0.0), self.sig)
            V = V + self.sig * zv
        return np.concatenate([U.reshape(n, -1), V.reshape(n, -1)], axis=1)

    def _advance(self, x_prev, zs):
        n = x_prev.shape[0]
        U = x_prev[:, : self.nodes].reshape(n, self.rows, self.cols)
        V = x_prev[:, self.nodes:].reshape(n, self.rows, self.cols)
        for zu, zv in zs:
            U, V = accel.fhn_euler_block_numpy(
                U, V, -self.deg * U, zu, self.dt, 1.0, (-1.0, 1.13, -0.13, 0.0),
                (0.01, -0.005, 0.0), self.sig)
            V = V + self.sig * zv
        return np.concatenate([U.reshape(n, -1), V.reshape(n, -1)], axis=1)

    def transition_point_prediction(self, x_prev, t):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        z = np.zeros((x_prev.shape[0], self.rows, self.cols))
        return self._advance(x_prev, [(z, z)] * self.substeps)

    def log_likelihood(self, y, x, t):
        y = np.asarray(y, dtype=np.float64).reshape(-1)
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        resid = y - x[:, : self.nodes][:, self.obs_indices]
        return -0.5 / self.obs_var * np.sum(resid * resid, axis=1)

    def error_projection(self, states):
        return np.asarray(states)[..., : self.nodes]


# --------------------------------------------------------------------------
# recording wrapper around the reference resampler
# --------------------------------------------------------------------------


class _Recorder:
    def __init__(self):
        self.calls = []
        self._orig = ref_filters.multinomial_resample_indices

    def __call__(self, weights, n_out, rng):
        # identical arithmetic to resampling.py:29-43, with u captured
        w = resampling._check_weights(weights)
        cum = np.cumsum(w)
        u = resampling._sorted_uniforms(n_out, rng)
        idx = accel.resample_indices(cum, u)
        self.calls.append((u, idx))
        return idx

    def __enter__(self):
        ref_filters.multinomial_resample_indices = self
        return self

    def __exit__(self, *exc):
        ref_filters.multinomial_resample_indices = self._orig


def _filter_with_steps(model, obs, n, seed, variant="bootstrap"):
    with _Recorder() as rec:
        out = parpf.run_filter(model, obs, variant, n, seed)
    return out, rec.calls


# --------------------------------------------------------------------------
# fixtures
# --------------------------------------------------------------------------


def gen_kernels():
    rng = np.random.default_rng(20260101)
    d = {}
    # normalize_log_weights (core.py:116-138)
    cases = [np.zeros(4), np.array([5.0]), np.array([0.0, np.log(2.0)]),
             np.array([-np.inf, 0.0, -np.inf]), np.array([-1e4, -1e4 + np.log(3.0)]),
             rng.normal(size=1000) * 10.0, rng.normal(size=4096)]
    for i, c in enumerate(cases):
        w, lm = core.normalize_log_weights(c)
        d[f"nlw_in_{i}"] = c
        d[f"nlw_w_{i}"] = w
        d[f"nlw_lm_{i}"] = np.array(lm)
    d["nlw_count"] = np.array(len(cases))
    # resample_indices (accel.py:175-203), incl. the tie case (test_accel.py:57-64)
    rcases = [(np.array([0.2, 0.2, 1.0]), np.array([0.1, 0.2, 0.2000000001, 0.99]))]
    for n, m in ((1, 5), (10, 10), (1000, 313), (4096, 4096), (3, 7)):
        w = rng.dirichlet(np.ones(n))
        if n == 3:
            w = np.array([0.5, 0.0, 0.5])
        cum = np.cumsum(w)
        e = rng.standard_exponential(m + 1)
        c = np.cumsum(e)
        rcases.append((cum, c[:m] / c[m]))
    # u beyond the last cum (clamp) - cum ends below 1 by rounding
    rcases.append((np.array([0.25, 0.5, 0.75, 0.9999999999999]), np.array([0.3, 0.99999999999999, 1.0])))
    for i, (cum, u) in enumerate(rcases):
        d[f"ri_cum_{i}"] = cum
        d[f"ri_u_{i}"] = u
        d[f"ri_idx_{i}"] = accel.resample_indices(cum, u)
        assert np.array_equal(d[f"ri_idx_{i}"], accel.resample_indices_numpy(cum, u))
    d["ri_count"] = np.array(len(rcases))
    # multinomial_resample_indices with a seeded Generator
    w = rng.dirichlet(np.ones(500))
    d["mri_w"] = w
    d["mri_idx"] = resampling.multinomial_resample_indices(w, 500, np.random.default_rng(77))
    d["sys_idx"] = resampling.systematic_resample_indices(w, 700, np.random.default_rng(78))
    wb = rng.dirichlet(np.ones(50_000))
    d["mri_big_w"] = wb
    d["mri_big_idx"] = resampling.multinomial_resample_indices(wb, 60_000,
                                                               np.random.default_rng(79))
    from parpf.models import lorenz_log_likelihood, lorenz_transition

    d["lz_tr"] = lorenz_transition(np.array([1.0, 2.0, 3.0]), np.random.default_rng(3))
    d["lz_ll"] = np.array(lorenz_log_likelihood(0.7, np.array([1.0, 2.0, 3.0])))
    # lorenz_euler_block (accel.py:60-102), same shapes as test_accel.py:22-27
    st = rng.normal(size=(257, 3)) * 10.0
    nz = rng.normal(size=(100, 257, 3))
    d["lz_states"], d["lz_noise"] = st, nz
    d["lz_out"] = accel.lorenz_euler_block(st, nz, 1e-3, 10.0, 28.0, 8.0 / 3.0)
    assert np.array_equal(d["lz_out"], accel.lorenz_euler_block_numpy(st, nz, 1e-3, 10.0, 28.0, 8.0 / 3.0))
    # fhn_euler_block numpy twin (accel.py:110-129): rectangular + square
    for tag, shape, params in (
        ("rect", (5, 30, 50), (0.01, 1.0, (-1.0, 1.13, -0.13, 0.0), (0.01, -0.005, 0.0), 0.005)),
        ("sq", (33, 16, 16), (5e-3, 4.5e-3, (-1.0, 0.0, 3.6, 0.0), (2.1, -0.6, 0.6), 0.05)),
    ):
        U, V, drive, noise = (rng.normal(size=shape) for _ in range(4))
        dt, cpl, cubic, beta, sig = params
        u2, v2 = accel.fhn_euler_block_numpy(U, V, drive, noise, dt, cpl, cubic, beta, sig)
        for k, a in (("U", U), ("V", V), ("drive", drive), ("noise", noise), ("u_new", u2), ("v_new", v2)):
            d[f"fhn_{tag}_{k}"] = a
        d[f"fhn_{tag}_params"] = np.array([dt, cpl, *cubic, *beta, sig])
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **d)


def gen_lorenz():
    d = {}
    truth0, states, obs = orc.lorenz_truth(seed=2024, n_obs=25)
    model = RefLorenzCfg(substeps=40, obs_var=2.0, prior_mean=tuple(truth0), prior_var=1.0)
    d["truth0"], d["states"], d["obs"] = truth0, states, obs
    # one filter with per-step ancestors
    seed = np.random.SeedSequence(31337)
    out, calls = _filter_with_steps(model, obs, 64, seed)
    d["f_est"], d["f_lnc"] = out.estimates, out.log_norm_const
    d["f_u"] = np.stack([c[0] for c in calls])
    d["f_anc"] = np.stack([c[1] for c in calls])
    d["f_seed_entropy"] = np.array(31337)
    # an ensemble (ensemble.py:76-111): M=4, N=100, master seed 5
    ens = parpf.run_ensemble(model, obs, "bootstrap", 4, 100, 5)
    d["e_mean"] = ens.mean_estimates
    d["e_est"] = np.stack([fo.estimates for fo in ens.filter_outputs])
    d["e_lnc"] = np.stack([fo.log_norm_const for fo in ens.filter_outputs])
    d["e_master"] = np.array(5)
    # collapse: an infinite observation makes every log weight -inf at step 3
    obs_c = obs[:6].copy()
    obs_c[2] = np.inf
    outc = parpf.run_filter(model, obs_c, "bootstrap", 32, 11)
    d["c_obs"], d["c_est"], d["c_lnc"] = obs_c, outc.estimates, outc.log_norm_const
    d["c_steps"] = np.array(outc.collapse_steps)
    # auxiliary filter (filters.py:115-154): two resampling calls per step
    outa, calls = _filter_with_steps(model, obs[:12], 48, np.random.SeedSequence(4242),
                                     "auxiliary")
    d["a_est"], d["a_lnc"] = outa.estimates, outa.log_norm_const
    d["a_u1"] = np.stack([c[0] for c in calls[0::2]])
    d["a_anc1"] = np.stack([c[1] for c in calls[0::2]])
    d["a_u2"] = np.stack([c[0] for c in calls[1::2]])
    d["a_anc2"] = np.stack([c[1] for c in calls[1::2]])
    ensa = parpf.run_ensemble(model, obs[:12], "auxiliary", 3, 64, 8)
    d["ae_mean"] = ensa.mean_estimates
    d["ae_lnc"] = np.stack([fo.log_norm_const for fo in ensa.filter_outputs])
    # auxiliary collapse: infinite observation -> both stages collapse
    outac = parpf.run_filter(model, obs_c, "auxiliary", 16, 12)
    d["ac_est"], d["ac_lnc"] = outac.estimates, outac.log_norm_const
    d["ac_steps"] = np.array(outac.collapse_steps)
    # double bootstrap (filters.py:201-313): 4 islands x 30, island period 5
    from parpf.filters import run_double_bootstrap

    db = run_double_bootstrap(model, obs[:12], 4, 30, 5, np.random.SeedSequence(99))
    d["db_est"], d["db_lnc"] = db.estimates, db.log_norm_const
    d["db_coll"] = np.array(db.collapse_steps, dtype=np.int64)
    # ground truth / observation generator (models/simulate.py:10-29), stock model
    from parpf.models import simulate as ref_simulate

    d["sim_states"], d["sim_obs"] = ref_simulate(Lorenz63Model(), 20, 11)
    # the .17g CSV format (io.py:36-42) as written by the reference
    import tempfile

    from parpf import io as ref_io

    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "obs.csv")
        ref_io.write_array_csv(path, "y", d["sim_obs"][:5])
        d["csv_text"] = np.array(open(path).read())
    np.savez_compressed(os.path.join(HERE, "lorenz.npz"), **d)


def gen_fhn():
    d = {}
    m, states, obs = orc.fhn_truth(seed=7, n_obs=3)
    model = RefFhnCfg(m.rows, m.cols, m.substeps, m.stim_row, m.stim_col)
    d["obs"] = obs
    d["stim"] = np.array([m.stim_row, m.stim_col])
    out, calls = _filter_with_steps(model, obs, 8, np.random.SeedSequence(99))
    d["f_est_v"] = out.estimates[:, : m.nodes]
    d["f_est_w"] = out.estimates[:, m.nodes:]
    d["f_lnc"] = out.log_norm_const
    d["f_u"] = np.stack([c[0] for c in calls])
    d["f_anc"] = np.stack([c[1] for c in calls])
    ens = parpf.run_ensemble(model, obs[:2], "bootstrap", 2, 4, 17)
    d["e_mean_v"] = ens.mean_estimates[:, : m.nodes]
    d["e_lnc"] = np.stack([fo.log_norm_const for fo in ens.filter_outputs])
    outa, calls = _filter_with_steps(model, obs, 6, np.random.SeedSequence(5151), "auxiliary")
    d["a_est_v"] = outa.estimates[:, : m.nodes]
    d["a_lnc"] = outa.log_norm_const
    d["a_anc1"] = np.stack([c[1] for c in calls[0::2]])
    d["a_anc2"] = np.stack([c[1] for c in calls[1::2]])
    np.savez_compressed(os.path.join(HERE, "fhn.npz"), **d)


def gen_fhnnet():
    """The paper's forced FH-N network (models/fhn.py:85-207), stock model."""
    from parpf.models import FhnNetworkModel
    from parpf.models import simulate as ref_simulate

    d = {}
    kw8 = dict(J=8, n_zones=2, zone_width=2, stim_prob=0.05)
    m8 = FhnNetworkModel(**kw8)
    d["m8_stim_prob"] = np.array(kw8["stim_prob"])
    st8, ob8 = ref_simulate(m8, 120, 3)
    d["sim8_states"], d["sim8_obs"] = st8, ob8
    m16 = FhnNetworkModel(J=16, stim_prob=0.02)
    d["sim16_states"], d["sim16_obs"] = ref_simulate(m16, 150, 3)
    # hooks on hand-made states: latched history, forcing on/off, band region
    rng = np.random.default_rng(55)
    x = np.zeros((5, m8.dim_x))
    x[:, : 2 * 64] = rng.normal(size=(5, 128)) * 2.0
    q = (rng.random((5, m8.stim_hold * 64)) < 0.05).astype(float)
    x[:, 2 * 64:] = q
    d["hook_x"] = x
    d["tpp_t1"] = m8.transition_point_prediction(x, 1)
    d["tpp_t250"] = m8.transition_point_prediction(x, 250)
    xb = x.copy()
    xb[:, :64] = -1.7
    xb[2, :64] = 0.0  # no region for particle 2
    d["band_x"] = xb
    mfire = FhnNetworkModel(**{**kw8, "stim_prob": 1.0})
    d["band_out"] = mfire.sample_transition(xb, 7, np.random.default_rng(19))
    y = rng.normal(size=m8.dim_y)
    d["ll_y"] = y
    d["ll_out"] = m8.log_likelihood(y, x, 1)
    # filters on the simulated record
    out, calls = _filter_with_steps(m8, ob8[:60], 32, np.random.SeedSequence(808))
    d["f_est"], d["f_lnc"] = out.estimates, out.log_norm_const
    d["f_u"] = np.stack([c[0] for c in calls])
    d["f_anc"] = np.stack([c[1] for c in calls])
    outa, calls = _filter_with_steps(m8, ob8[:40], 24, np.random.SeedSequence(909), "auxiliary")
    d["a_est"], d["a_lnc"] = outa.estimates, outa.log_norm_const
    d["a_anc1"] = np.stack([c[1] for c in calls[0::2]])
    d["a_anc2"] = np.stack([c[1] for c in calls[1::2]])
    ens = parpf.run_ensemble(m8, ob8[:40], "bootstrap", 3, 16, 21)
    d["e_mean"] = ens.mean_estimates
    d["e_lnc"] = np.stack([fo.log_norm_const for fo in ens.filter_outputs])
    np.savez_compressed(os.path.join(HERE, "fhnnet.npz"), **d)


def gen_small():
    """Verification oracle models (models/hmm.py, models/linear_gaussian.py)."""
    from parpf.models import DiscreteHmm, LinearGaussianModel, hmm_exact_filter, kalman_filter
    from parpf.models import simulate as ref_simulate

    d = {}
    hmm = DiscreteHmm(prior=[0.5, 0.5], transition=[[0.9, 0.1], [0.2, 0.8]],
                      emission=[[0.8, 0.2], [0.3, 0.7]])
    hobs = np.array([[0.0], [1.0], [0.0], [0.0], [1.0]])
    out, calls = _filter_with_steps(hmm, hobs, 50, np.random.SeedSequence(7102))
    d["h_est"], d["h_lnc"] = out.estimates, out.log_norm_const
    d["h_anc"] = np.stack([c[1] for c in calls])
    ens = parpf.run_ensemble(hmm, hobs, "bootstrap", 3, 20, 44)
    d["he_mean"] = ens.mean_estimates
    d["he_lnc"] = np.stack([fo.log_norm_const for fo in ens.filter_outputs])
    ex = hmm_exact_filter(hmm, hobs)
    d["h_exact_filter"] = np.stack([e[0] for e in ex])
    d["h_exact_mass"] = np.array([e[1] for e in ex])
    d["h_sim_states"], d["h_sim_obs"] = ref_simulate(hmm, 30, 5)
    lg = LinearGaussianModel.scalar(a=0.9, q=1.0, h=1.0, r=1.0, prior_mean=0.0, prior_var=1.0)
    st, ob = ref_simulate(lg, 10, 12)
    d["l_sim_states"], d["l_obs"] = st, ob
    out, calls = _filter_with_steps(lg, ob, 64, np.random.SeedSequence(7103))
    d["l_est"], d["l_lnc"] = out.estimates, out.log_norm_const
    d["l_anc"] = np.stack([c[1] for c in calls])
    outa = parpf.run_filter(lg, ob, "auxiliary", 40, np.random.SeedSequence(71))
    d["la_est"], d["la_lnc"] = outa.estimates, outa.log_norm_const
    kf = kalman_filter(lg, ob)
    d["l_kf_mean"] = np.stack([k[0] for k in kf])
    d["l_kf_cov"] = np.stack([k[1] for k in kf])
    lg2 = LinearGaussianModel(A=[[0.9, 0.1], [-0.2, 0.8]], trans_cov=[[1.0, 0.3], [0.3, 0.5]],
                              H=[[1.0, 0.5]], obs_cov=[[0.7]], prior_mean=[0.5, -0.5],
                              prior_cov=[[1.0, 0.2], [0.2, 2.0]])
    st2, ob2 = ref_simulate(lg2, 8, 13)
    d["l2_obs"] = ob2
    out2 = parpf.run_filter(lg2, ob2, "bootstrap", 32, np.random.SeedSequence(5))
    d["l2_est"], d["l2_lnc"] = out2.estimates, out2.log_norm_const
    # double bootstrap (filters.py:201-313) on the HMM: island steps at t = 2, 4
    from parpf.filters import run_double_bootstrap

    db = run_double_bootstrap(hmm, hobs, 3, 20, 2, np.random.SeedSequence(606))
    d["db_h_est"], d["db_h_lnc"] = db.estimates, db.log_norm_const
    d["db_h_coll"] = np.array(db.collapse_steps, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "small.npz"), **d)


if __name__ == "__main__":
    print("reference backend:", accel.backend_name())
    gen_kernels()
    gen_lorenz()
    gen_fhn()
    gen_fhnnet()
    gen_small()
    for f in sorted(os.listdir(HERE)):
        if f.endswith(".npz"):
            print(f, os.path.getsize(os.path.join(HERE, f)))
