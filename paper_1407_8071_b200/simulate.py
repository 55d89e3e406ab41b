"""Ground-truth trajectories and observations for the BASELINE configs, on
the GPU (cf. parpf/models/simulate.py:10-29, which steps one state through
the model hooks on the CPU).

The truth is one particle advanced by the same propagate kernels the bank
uses (Philox noise keyed by the seed, purpose-separated from any filter's
stream); observation noise h(x) + sqrt(obs_var) * z is drawn from a numpy
Generator seeded by the same seed.  Draw order and seeding are this
package's own (the BASELINE configs fix shapes and distributions, not a
stream); the oracle's truth generator is a separate CPU restatement used by
the parity tests.
"""

from __future__ import annotations

import numpy as np

from . import _lib, philox
from .models import FhnLatticeModel, Lorenz63Model


def simulate(model, n_steps: int, seed):
    """One state trajectory and its observations through the model hooks
    (parpf/models/simulate.py:10-29): same control flow and draw order
    (prior, then per step transition then observation), arithmetic on the
    GPU.  Returns (states (n_steps+1, dim_x), observations (n_steps, dim_y)).
    """
    if n_steps < 0:
        raise ValueError("n_steps must be >= 0")
    rng = np.random.default_rng(seed)
    x = model.sample_prior(rng, 1)[0]
    states = np.empty((n_steps + 1, model.dim_x))
    observations = np.empty((n_steps, model.dim_y))
    states[0] = x
    for t in range(1, n_steps + 1):
        x = model.sample_transition(x[None, :], t, rng)[0]
        states[t] = x
        observations[t - 1] = np.asarray(model.sample_observation(x, t, rng)).reshape(-1)
    return states, observations


def _truth_key(seed):
    ss = philox.as_seed_sequence(seed)
    return np.random.SeedSequence(ss.entropy, spawn_key=tuple(ss.spawn_key) + (0x7457,)) \
        .generate_state(2, dtype=np.uint32)


def lorenz_truth(seed, n_obs: int, model: Lorenz63Model | None = None, burn_in: int = 1000):
    """cfg0/cfg2 truth: x0 ~ N(0, I), `burn_in` EM steps, then `n_obs`
    intervals of model.substeps steps, observing model.observe with
    N(0, obs_var I).  Returns (truth0, states (n_obs,3), observations)."""
    import torch

    _lib.require_cuda()
    model = model or Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3")
    rng = np.random.default_rng(philox.as_seed_sequence(seed))
    key = torch.from_numpy(_truth_key(seed).view(np.int32)).cuda()
    x = torch.from_numpy(rng.standard_normal(3)[:, None].copy()).cuda()
    y = torch.zeros(model.dim_y, dtype=torch.float64, device="cuda")
    lw = torch.empty(1, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = _lib.stream_ptr()

    def advance(xin, n_sub, t):
        xout = torch.empty_like(xin)
        _lib.call("pf_lorenz_propagate_weight", model.params(n_sub), _lib.PF_F64, _lib.ptr(xin),
                  None, _lib.ptr(xout), _lib.ptr(y), _lib.ptr(lw), 1, 1, _lib.ptr(key), t, None,
                  _lib.ptr(st), s)
        return xout

    if burn_in:
        x = advance(x, burn_in, 0x7FFFFFFF)
    truth0 = x[:, 0].cpu().numpy().copy()
    states = torch.empty((n_obs, 3), dtype=torch.float64, device="cuda")
    for k in range(n_obs):
        x = advance(x, model.substeps, k + 1)
        states[k] = x[:, 0]
    states_h = states.cpu().numpy()
    _lib.raise_status(st.cpu().numpy(), "truth simulation")
    sd = np.sqrt(model.obs_var)
    cols = [0] if model.dim_y == 1 else [0, 2]
    obs = states_h[:, cols] + sd * rng.standard_normal((n_obs, len(cols)))
    return truth0, states_h, obs


def fhn_truth(seed, n_obs: int, model: FhnLatticeModel | None = None):
    """cfg3/cfg4 truth: seeded 3x3 stimulus patch (v=1) at t=0, w=0; the
    lattice is simulated with noise and v observed at the electrodes with
    N(0, obs_var).  Returns (model_with_patch, states (n_obs, dim_x), obs)."""
    import torch

    _lib.require_cuda()
    base = model or FhnLatticeModel()
    rng = np.random.default_rng(philox.as_seed_sequence(seed))
    i0 = int(rng.integers(0, base.rows - base.stim_size + 1))
    j0 = int(rng.integers(0, base.cols - base.stim_size + 1))
    m = FhnLatticeModel(**{**{f: getattr(base, f) for f in base.__dataclass_fields__},
                           "stim_row": i0, "stim_col": j0})
    key = torch.from_numpy(_truth_key(seed).view(np.int32)).cuda()
    x = torch.from_numpy(m.initial_state()[None, :].copy()).cuda()
    y = torch.zeros(m.dim_y, dtype=torch.float64, device="cuda")
    idx = torch.from_numpy(m.obs_indices.astype(np.int32)).cuda()
    lw = torch.empty(1, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    states = torch.empty((n_obs, m.dim_x), dtype=torch.float64, device="cuda")
    s = _lib.stream_ptr()
    for k in range(n_obs):
        xout = torch.empty_like(x)
        _lib.call("pf_fhn_interval", m.params(), _lib.PF_F64, _lib.ptr(x), None, _lib.ptr(xout),
                  _lib.ptr(y), _lib.ptr(idx), _lib.ptr(lw), 1, 1, _lib.ptr(key), k + 1, None,
                  _lib.ptr(st), s)
        x = xout
        states[k] = x[0]
    states_h = states.cpu().numpy()
    _lib.raise_status(st.cpu().numpy(), "truth simulation")
    obs = states_h[:, m.obs_indices] + np.sqrt(m.obs_var) * rng.standard_normal((n_obs, m.dim_y))
    return m, states_h, obs
