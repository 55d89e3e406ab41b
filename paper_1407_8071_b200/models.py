"""GPU model descriptors that keep the reference StateSpaceModel interface.

* :class:`Lorenz63Model` - parpf/models/lorenz63.py:22-69 plus two fields
  the BASELINE configs need: ``noise_scale`` (cfg0/cfg2 use
  std 0.5*sqrt(h), i.e. noise_scale=0.5) and ``observe`` ("x1" - the stock
  model - or "x1x3", observing (x1, x3) as cfg0/cfg2 do).
* :class:`FhnLatticeModel` - the classical FitzHugh-Nagumo lattice of
  BASELINE cfg3/cfg4 expressed in the reference lattice kernel's general form
  (accel.py:110-129; mapping in SURVEY §8a-A9 and DESIGN.md §2).

Their per-hook methods (sample_prior, sample_transition, log_likelihood,
transition_point_prediction) run on the GPU through libpfbank in fp64 with
the caller's numpy Generator supplying the draws in the reference's order,
so a hook-level caller (e.g. the reference-style bf_step) sees the same
numbers as with the reference models.  The bank (bank.py) uses the same
kernels directly on device-resident particles.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import StateSpaceModel
from .exceptions import NumericalDivergenceError

LORENZ_PRIOR_MEAN = (-10.2410, -1.3984, -23.6752)


def _torch():
    import torch

    _lib.require_cuda()
    return torch


@dataclass
class Lorenz63Model(StateSpaceModel):
    s: float = 10.0
    r: float = 28.0
    b: float = 8.0 / 3.0
    dt: float = 1e-3
    substeps: int = 100
    obs_var: float = 0.5
    prior_mean: tuple = LORENZ_PRIOR_MEAN
    prior_var: float = 10.0
    noise_scale: float = 1.0
    observe: str = "x1"

    kind = "lorenz"

    def __post_init__(self):
        if self.substeps < 1:
            raise ValueError("substeps must be >= 1")
        if self.obs_var <= 0 or self.prior_var <= 0:
            raise ValueError("variances must be positive")
        if self.observe not in ("x1", "x1x3"):
            raise ValueError("observe must be 'x1' or 'x1x3'")
        self.dim_x = 3
        self.dim_y = 1 if self.observe == "x1" else 2
        self._prior_mean_arr = np.asarray(self.prior_mean, dtype=np.float64)

    # -- device descriptor ------------------------------------------------
    def params(self, n_sub=None, noise_free=False) -> _lib.LorenzParams:
        """Device descriptor; noise_free=True gives the point prediction
        (transition_point_prediction, lorenz63.py:57-60)."""
        return _lib.LorenzParams(float(self.s), float(self.r), float(self.b), float(self.dt),
                                 0.0 if noise_free else float(self.noise_scale),
                                 float(self.obs_var),
                                 int(self.substeps if n_sub is None else n_sub), self.dim_y)

    def prior_sd(self) -> float:
        return float(np.sqrt(self.prior_var))

    # -- reference hooks, evaluated on the GPU -----------------------------
    def sample_prior(self, rng, n):
        torch = _torch()
        z = np.ascontiguousarray(rng.standard_normal((n, 3)))
        x = torch.empty((3, n), dtype=torch.float64, device="cuda")
        mean, mean_p = _lib.host_f64(self._prior_mean_arr)
        d_z = torch.from_numpy(z).cuda()
        _lib.call("pf_lorenz_prior", _lib.PF_F64, _lib.ptr(x), 1, n, mean_p, self.prior_sd(),
                  None, _lib.ptr(d_z), _lib.stream_ptr())
        return x.t().contiguous().cpu().numpy()

    def _run(self, x_prev, noise, n_sub, y=None):
        torch = _torch()
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        n = x_prev.shape[0]
        xin = torch.from_numpy(np.ascontiguousarray(x_prev.T)).cuda()
        xout = torch.empty_like(xin)
        lw = torch.empty(n, dtype=torch.float64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        yy = np.zeros(self.dim_y) if y is None else np.asarray(y, dtype=np.float64).reshape(-1)
        d_y = torch.from_numpy(np.ascontiguousarray(yy[: self.dim_y])).cuda()
        d_z = None
        if n_sub > 0:
            d_z = torch.from_numpy(np.ascontiguousarray(noise, dtype=np.float64)).cuda()
        else:
            d_z = torch.zeros(1, dtype=torch.float64, device="cuda")
        p = self.params(n_sub)
        _lib.call("pf_lorenz_propagate_weight", p, _lib.PF_F64, _lib.ptr(xin), None,
                  _lib.ptr(xout), _lib.ptr(d_y), _lib.ptr(lw), 1, n, None, 1, _lib.ptr(d_z),
                  _lib.ptr(st), _lib.stream_ptr())
        return xout.t().contiguous().cpu().numpy(), lw.cpu().numpy(), int(st.item())

    def _propagate(self, x_prev, noise):
        out, _, st = self._run(x_prev, noise, self.substeps)
        if st & _lib.PF_ST_DIVERGED:
            raise NumericalDivergenceError("Lorenz transition produced non-finite states")
        return out

    def sample_transition(self, x_prev, t, rng):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        noise = rng.standard_normal((self.substeps, x_prev.shape[0], 3))
        return self._propagate(x_prev, noise)

    def transition_point_prediction(self, x_prev, t):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        return self._propagate(x_prev, np.zeros((self.substeps, x_prev.shape[0], 3)))

    def log_likelihood(self, y, x, t):
        _, lw, _ = self._run(x, None, 0, y)
        return lw

    def sample_observation(self, x, t, rng):
        x = np.asarray(x).reshape(-1)
        if self.dim_y == 1:
            return np.array([x[0] + np.sqrt(self.obs_var) * rng.standard_normal()])
        return x[[0, 2]] + np.sqrt(self.obs_var) * rng.standard_normal(2)


def electrode_indices(rows=30, cols=50, n_side=10, row0=1, col0=2) -> np.ndarray:
    """Flat row-major electrode nodes of a regular n_side x n_side subgrid."""
    rr = row0 + (rows // n_side) * np.arange(n_side)
    cc = col0 + (cols // n_side) * np.arange(n_side)
    return (rr[:, None] * cols + cc[None, :]).reshape(-1).astype(np.int64)


@dataclass
class FhnLatticeModel(StateSpaceModel):
    """Classical FH-N lattice (BASELINE cfg3/cfg4); state row = [v, w]."""

    rows: int = 30
    cols: int = 50
    dt: float = 0.01
    substeps: int = 50
    cubic: tuple = (-1.0, 1.13, -0.13, 0.0)
    beta: tuple = (0.01, -0.005, 0.0)
    coupling: float = 1.0
    noise_std: float = 0.05
    obs_var: float = 0.01
    stim_row: int = 0
    stim_col: int = 0
    stim_size: int = 3
    electrode_side: int = 10
    electrode_row0: int = 1
    electrode_col0: int = 2

    kind = "fhn"

    def __post_init__(self):
        if self.substeps < 1:
            raise ValueError("substeps must be >= 1")
        if self.obs_var <= 0:
            raise ValueError("obs_var must be positive")
        if min(self.rows, self.cols) < self.electrode_side:
            raise ValueError("electrode grid does not fit on the lattice")
        self.nodes = self.rows * self.cols
        self.dim_x = 2 * self.nodes
        self.obs_indices = electrode_indices(self.rows, self.cols, self.electrode_side,
                                             self.electrode_row0, self.electrode_col0)
        if self.obs_indices.max() >= self.nodes:
            raise ValueError("electrodes do not fit on the lattice")
        self.dim_y = int(self.obs_indices.shape[0])
        self.sig_sqdt = self.noise_std * math.sqrt(self.dt)

    def params(self, n_sub=None, noise_free=False) -> _lib.FhnParams:
        """Device descriptor; noise_free=True gives the point prediction."""
        p = _lib.FhnParams()
        p.rows, p.cols = self.rows, self.cols
        p.n_sub = int(self.substeps if n_sub is None else n_sub)
        p.n_obs = self.dim_y
        p.dt, p.coupling = float(self.dt), float(self.coupling)
        for i in range(4):
            p.cubic[i] = float(self.cubic[i])
        for i in range(3):
            p.beta[i] = float(self.beta[i])
        p.sig_v = p.sig_w = 0.0 if noise_free else float(self.sig_sqdt)
        p.degree_drive = -1.0
        p.obs_var = float(self.obs_var)
        return p

    def initial_state(self) -> np.ndarray:
        x = np.zeros(self.dim_x)
        v = x[: self.nodes].reshape(self.rows, self.cols)
        v[self.stim_row:self.stim_row + self.stim_size,
          self.stim_col:self.stim_col + self.stim_size] = 1.0
        return x

    def sample_prior(self, rng, n):
        # point mass at the stimulated state, no draws (cf. fhn.py:144-147)
        torch = _torch()
        x = torch.empty((n, self.dim_x), dtype=torch.float64, device="cuda")
        row = torch.from_numpy(self.initial_state()).cuda()
        _lib.call("pf_fill_rows", _lib.PF_F64, _lib.ptr(x), n, self.dim_x, _lib.ptr(row),
                  _lib.stream_ptr())
        return x.cpu().numpy()

    def draw_noise(self, rng, n):
        """(substeps, 2, n, nodes) standard normals in the oracle draw order:
        per Euler step, the v-noise block then the w-noise block."""
        zs = np.empty((self.substeps, 2, n, self.nodes))
        for k in range(self.substeps):
            zs[k, 0] = rng.standard_normal((n, self.rows, self.cols)).reshape(n, -1)
            zs[k, 1] = rng.standard_normal((n, self.rows, self.cols)).reshape(n, -1)
        return zs

    def _run(self, x_prev, noise, n_sub, y=None):
        torch = _torch()
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        n = x_prev.shape[0]
        xin = torch.from_numpy(np.ascontiguousarray(x_prev)).cuda()
        xout = torch.empty_like(xin)
        lw = torch.empty(n, dtype=torch.float64, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        yy = np.zeros(self.dim_y) if y is None else np.asarray(y, dtype=np.float64).reshape(-1)
        if yy.shape[0] != self.dim_y:
            raise ValueError(f"expected {self.dim_y} observed nodes, got {yy.shape[0]}")
        d_y = torch.from_numpy(np.ascontiguousarray(yy)).cuda()
        d_idx = torch.from_numpy(self.obs_indices.astype(np.int32)).cuda()
        if n_sub > 0:
            d_z = torch.from_numpy(np.ascontiguousarray(noise, dtype=np.float64)).cuda()
        else:
            d_z = torch.zeros(1, dtype=torch.float64, device="cuda")
        _lib.call("pf_fhn_interval", self.params(n_sub), _lib.PF_F64, _lib.ptr(xin), None,
                  _lib.ptr(xout), _lib.ptr(d_y), _lib.ptr(d_idx), _lib.ptr(lw), 1, n, None, 1,
                  _lib.ptr(d_z), _lib.ptr(st), _lib.stream_ptr())
        return xout.cpu().numpy(), lw.cpu().numpy(), int(st.item())

    def _propagate(self, x_prev, noise):
        out, _, st = self._run(x_prev, noise, self.substeps)
        if st & _lib.PF_ST_DIVERGED:
            raise NumericalDivergenceError("FH-N transition produced non-finite states")
        return out

    def sample_transition(self, x_prev, t, rng):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        return self._propagate(x_prev, self.draw_noise(rng, x_prev.shape[0]))

    def transition_point_prediction(self, x_prev, t):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        return self._propagate(x_prev, np.zeros((self.substeps, 2, x_prev.shape[0], self.nodes)))

    def log_likelihood(self, y, x, t):
        _, lw, _ = self._run(x, None, 0, y)
        return lw

    def sample_observation(self, x, t, rng):
        x = np.asarray(x).reshape(-1)
        return x[: self.nodes][self.obs_indices] + np.sqrt(self.obs_var) * rng.standard_normal(
            self.dim_y)

    def error_projection(self, states):
        return np.asarray(states)[..., : self.nodes]
