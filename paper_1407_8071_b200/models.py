"""GPU model descriptors that keep the reference StateSpaceModel interface.

* :class:`Lorenz63Model` - parpf/models/lorenz63.py:22-69 plus two fields
  the BASELINE configs need: ``noise_scale`` (cfg0/cfg2 use
  std 0.5*sqrt(h), i.e. noise_scale=0.5) and ``observe`` ("x1" - the stock
  model - or "x1x3", observing (x1, x3) as cfg0/cfg2 do).
* :class:`FhnLatticeModel` - the classical FitzHugh-Nagumo lattice of
  BASELINE cfg3/cfg4 expressed in the reference lattice kernel's general form
  (accel.py:110-129; mapping in SURVEY §8a-A9 and DESIGN.md §2).
* :class:`FhnNetworkModel` - the paper's stochastically forced FH-N network
  (parpf/models/fhn.py:85-207): same fields, state row and hooks.

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


def estimate_width(model, estimate: str) -> int:
    """Columns of one filter's estimate row: the full state or the error
    projection (the voltage block of the lattice models)."""
    if estimate not in ("full", "projection"):
        raise ValueError("estimate must be 'full' or 'projection'")
    if model.kind in ("lorenz", "hmm", "lgm"):
        return model.dim_x
    return model.dim_x if estimate == "full" else model.nodes


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


# ---------------------------------------------------------------------------
# The paper's forced FH-N network (parpf/models/fhn.py)
# ---------------------------------------------------------------------------


def von_neumann_neighbors(i: int, j: int, J: int) -> list[tuple[int, int]]:
    """Axis neighbours of (i, j) truncated at the border, order up, down,
    left, right (fhn.py:38-49)."""
    return [(a, b) for a, b in ((i - 1, j), (i + 1, j), (i, j - 1), (i, j + 1))
            if 0 <= a < J and 0 <= b < J]


def fhn_stimulus_region(U, u_minus: float = -1.8, u_plus: float = -1.6) -> np.ndarray:
    """Mask of nodes whose own or an axis neighbour's voltage lies strictly in
    (u_minus, u_plus) on the trailing two axes (fhn.py:52-67).  Host helper;
    the bank evaluates the region inside pf_fhnnet_step."""
    U = np.asarray(U)
    band = (U > u_minus) & (U < u_plus)
    out = band.copy()
    out[..., 1:, :] |= band[..., :-1, :]
    out[..., :-1, :] |= band[..., 1:, :]
    out[..., :, 1:] |= band[..., :, :-1]
    out[..., :, :-1] |= band[..., :, 1:]
    return out


def observation_zone_indices(J: int, n_zones: int = 5, zone_width: int = 2) -> np.ndarray:
    """Sorted flat indices of an n_zones x n_zones grid of square zones
    (fhn.py:70-82)."""
    if n_zones * zone_width > J:
        raise ValueError("observation zones do not fit on the lattice")
    starts = ([(J - zone_width) // 2] if n_zones == 1
              else [(k * (J - zone_width)) // (n_zones - 1) for k in range(n_zones)])
    lines = np.concatenate([np.arange(s0, s0 + zone_width) for s0 in starts])
    return np.sort((lines[:, None] * J + lines[None, :]).reshape(-1)).astype(np.intp)


@dataclass
class FhnNetworkModel(StateSpaceModel):
    """Drop-in for parpf.models.FhnNetworkModel (fhn.py:85-207).

    Same fields and defaults, same flat state row
    ``[U, V, Q(t), .., Q(t-stim_hold+1)]`` at the hook boundary.  On the GPU
    the history is held as bits (stim_hold <= 32), U/V as fp32 or fp64
    planes; the hooks run in fp64 and reproduce the reference bit-for-bit
    for the same Generator draws.
    """

    J: int = 32
    dt: float = 5e-3
    coupling: float = 4.5e-3
    cubic: tuple = (-1.0, 0.0, 18.0 / 5.0, 0.0)
    beta: tuple = (2.1, -0.6, 0.6)
    u_minus: float = -1.8
    u_plus: float = -1.6
    stim_prob: float = 1e-3
    stim_amp: float = 200.0
    stim_hold: int = 25
    forcing_amp: float = 200.0
    forcing_period: float = 20.0
    forcing_width: float = 1.0
    forcing_mask: np.ndarray | None = None
    dyn_var: float = 0.5
    obs_var: float = 0.5
    n_zones: int = 5
    zone_width: int = 2

    kind = "fhnnet"

    def __post_init__(self):
        if self.u_minus >= self.u_plus:
            raise ValueError("u_minus must be below u_plus")
        if self.stim_hold < 1:
            raise ValueError("stim_hold must be >= 1")
        if self.stim_hold > 32:
            raise ValueError("stim_hold > 32 is not supported (history is a 32-bit field)")
        J = self.J
        if self.forcing_mask is None:
            mask = np.zeros((J, J))
            mask[:, 0] = 1.0
            self.forcing_mask = mask
        else:
            self.forcing_mask = np.asarray(self.forcing_mask, dtype=np.float64)
            if self.forcing_mask.shape != (J, J):
                raise ValueError("forcing_mask must be (J, J)")
        self.obs_indices = observation_zone_indices(J, self.n_zones, self.zone_width)
        self.nodes = J * J
        self.dim_x = (2 + self.stim_hold) * self.nodes
        self.dim_y = self.obs_indices.shape[0]
        self._sig_sqdt = np.sqrt(self.dyn_var) * np.sqrt(self.dt)

    # -- state packing (fhn.py:122-138) --------------------------------------
    def unpack(self, x):
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        n, K = x.shape[0], self.nodes
        return (x[:, :K].reshape(n, self.J, self.J), x[:, K:2 * K].reshape(n, self.J, self.J),
                x[:, 2 * K:].reshape(n, self.stim_hold, self.J, self.J))

    def pack(self, U, V, Q):
        n = U.shape[0]
        return np.concatenate([U.reshape(n, -1), V.reshape(n, -1), Q.reshape(n, -1)], axis=1)

    # -- device descriptor ------------------------------------------------------
    def params(self, n_sub=None, noise_free=False) -> _lib.FhnNetParams:
        p = _lib.FhnNetParams()
        p.J, p.stim_hold, p.n_obs = self.J, self.stim_hold, self.dim_y
        p.stochastic = 0 if noise_free else 1
        p.dt, p.coupling = float(self.dt), float(self.coupling)
        for i in range(4):
            p.cubic[i] = float(self.cubic[i])
        for i in range(3):
            p.beta[i] = float(self.beta[i])
        p.u_minus, p.u_plus = float(self.u_minus), float(self.u_plus)
        p.stim_prob, p.stim_amp = float(self.stim_prob), float(self.stim_amp)
        p.forcing_amp = float(self.forcing_amp)
        p.forcing_period = float(self.forcing_period)
        p.forcing_width = float(self.forcing_width)
        p.sig_sqdt = float(self._sig_sqdt)
        p.obs_var = float(self.obs_var)
        return p

    def device_mask(self, device="cuda"):
        torch = _torch()
        return torch.from_numpy(np.ascontiguousarray(self.forcing_mask.reshape(-1))).to(device)

    def to_device(self, rows, dtype=None):
        """Reference rows (n, dim_x) -> device (U/V planes, history bits)."""
        torch = _torch()
        dtype = dtype or torch.float64
        rows = np.atleast_2d(np.asarray(rows, dtype=np.float64))
        if rows.shape[1] != self.dim_x:
            raise ValueError(f"expected states with {self.dim_x} columns, got {rows.shape[1]}")
        q = rows[:, 2 * self.nodes:]
        if not np.all((q == 0.0) | (q == 1.0)):
            raise ValueError("stimulus history entries must be 0 or 1")
        n = rows.shape[0]
        d_rows = torch.from_numpy(np.ascontiguousarray(rows)).cuda()
        x = torch.empty((n, 2 * self.nodes), dtype=dtype, device="cuda")
        qb = torch.empty((n, self.nodes), dtype=torch.int32, device="cuda")
        _lib.call("pf_fhnnet_pack", _lib.dtype_code(dtype), _lib.ptr(d_rows), n, self.nodes,
                  self.stim_hold, _lib.ptr(x), _lib.ptr(qb), _lib.stream_ptr())
        return x, qb

    def from_device(self, x, qb, anc=None):
        torch = _torch()
        n = int(anc.numel()) if anc is not None else int(x.shape[0])
        rows = torch.empty((n, self.dim_x), dtype=torch.float64, device=x.device)
        _lib.call("pf_fhnnet_unpack", _lib.dtype_code(x.dtype), _lib.ptr(x), _lib.ptr(qb),
                  _lib.ptr(anc), n, self.nodes, self.stim_hold, _lib.ptr(rows),
                  _lib.stream_ptr())
        return rows.cpu().numpy()

    # -- model hooks -------------------------------------------------------------
    def sample_prior(self, rng, n):
        # quiescent start, no draws (fhn.py:144-147)
        return np.zeros((n, self.dim_x))

    def forcing_value(self, t: int) -> float:
        s = t * self.dt
        return self.forcing_amp if np.mod(s, self.forcing_period) <= self.forcing_width else 0.0

    def _advance(self, x_prev, t, rng=None):
        torch = _torch()
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        n = x_prev.shape[0]
        x, qb = self.to_device(x_prev)
        xo, qo = torch.empty_like(x), torch.empty_like(qb)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        stim = z = None
        if rng is not None:
            # draw order of fhn.py:158-176: fire, select, then the noise
            fire, sel = rng.random(n), rng.random(n)
            noise = rng.standard_normal((n, self.J, self.J))
            stim = torch.from_numpy(np.stack([fire, sel])).cuda()
            z = torch.from_numpy(np.ascontiguousarray(noise.reshape(n, -1))).cuda()
        mask = self.device_mask()
        _lib.call("pf_fhnnet_step", self.params(noise_free=rng is None), _lib.PF_F64,
                  _lib.ptr(x), _lib.ptr(qb), None, _lib.ptr(xo), _lib.ptr(qo), _lib.ptr(mask),
                  None, None, None, 1, n, None, int(t), _lib.ptr(stim), _lib.ptr(z),
                  _lib.ptr(st), _lib.stream_ptr())
        if int(st.item()) & _lib.PF_ST_DIVERGED:
            raise NumericalDivergenceError("FH-N transition produced non-finite states")
        return self.from_device(xo, qo)

    def sample_transition(self, x_prev, t, rng):
        return self._advance(x_prev, t, rng)

    def transition_point_prediction(self, x_prev, t):
        # no new random stimulus, no noise; forcing and latched stimuli apply
        return self._advance(x_prev, t, rng=None)

    def log_likelihood(self, y, x, t):
        torch = _torch()
        y = np.asarray(y, dtype=np.float64).reshape(-1)
        if y.shape[0] != self.dim_y:
            raise ValueError(f"expected {self.dim_y} observed nodes, got {y.shape[0]}")
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        n = x.shape[0]
        d_x = torch.from_numpy(np.ascontiguousarray(x[:, : self.nodes])).cuda()
        d_y = torch.from_numpy(y).cuda()
        idx = torch.from_numpy(self.obs_indices.astype(np.int32)).cuda()
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("pf_zone_loglik", _lib.PF_F64, _lib.ptr(d_x), n, self.nodes, _lib.ptr(idx),
                  self.dim_y, _lib.ptr(d_y), float(self.obs_var), _lib.ptr(out),
                  _lib.stream_ptr())
        return out.cpu().numpy()

    def sample_observation(self, x, t, rng):
        x = np.asarray(x).reshape(-1)
        u_obs = x[: self.nodes][self.obs_indices]
        return u_obs + np.sqrt(self.obs_var) * rng.standard_normal(self.dim_y)

    def error_projection(self, states):
        """Voltage block (fhn.py:214-217)."""
        return np.asarray(states)[..., : self.nodes]


def simulate(model, n_steps: int, seed):
    """parpf.models.simulate (models/simulate.py:10-29); see simulate.py."""
    from .simulate import simulate as _simulate

    return _simulate(model, n_steps, seed)


# ---------------------------------------------------------------------------
# Verification oracles: finite-state HMM and linear-Gaussian model
# ---------------------------------------------------------------------------


class _DeviceTables:
    """Per-device fp64 copies of a model's constant tables (not pickled)."""

    def _tables(self):
        torch = _torch()
        dev = torch.cuda.current_device()
        cache = self.__dict__.setdefault("_dev_cache", {})
        if dev not in cache:
            cache[dev] = {k: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).cuda()
                          for k, v in self._host_tables().items()}
        return cache[dev]

    def __getstate__(self):
        d = dict(self.__dict__)
        d.pop("_dev_cache", None)
        return d


@dataclass
class DiscreteHmm(_DeviceTables, StateSpaceModel):
    """Drop-in for parpf.models.DiscreteHmm (hmm.py:19-77): prior (K,),
    row-stochastic transition (K, K), strictly positive emission (K, S).
    States are carried as (n, 1) float arrays."""

    prior: np.ndarray
    transition: np.ndarray
    emission: np.ndarray

    kind = "hmm"

    def __post_init__(self):
        self.prior = np.asarray(self.prior, dtype=np.float64)
        self.transition = np.asarray(self.transition, dtype=np.float64)
        self.emission = np.asarray(self.emission, dtype=np.float64)
        k = self.prior.shape[0]
        if self.transition.shape != (k, k):
            raise ValueError("transition matrix shape mismatch")
        if not np.allclose(self.transition.sum(axis=1), 1.0, atol=1e-12):
            raise ValueError("transition rows must sum to 1")
        if not np.isclose(self.prior.sum(), 1.0, atol=1e-12):
            raise ValueError("prior must sum to 1")
        if self.emission.shape[0] != k:
            raise ValueError("emission table must have one row per state")
        if np.any(self.emission <= 0.0):
            raise ValueError("emission probabilities must be strictly positive")
        self.dim_x = 1
        self.dim_y = 1
        self._cum_rows = np.cumsum(self.transition, axis=1)
        self._cum_prior = np.cumsum(self.prior)

    @property
    def n_states(self) -> int:
        return self.prior.shape[0]

    def _host_tables(self):
        return {"cum_prior": self._cum_prior, "cum_rows": self._cum_rows,
                "log_emission": np.log(self.emission)}

    def params(self, n_sub=None, noise_free=False) -> _lib.HmmParams:
        tb = self._tables()
        return _lib.HmmParams(self.n_states, self.emission.shape[1], tb["cum_prior"].data_ptr(),
                              tb["cum_rows"].data_ptr(), tb["log_emission"].data_ptr())

    def sample_prior(self, rng, n):
        torch = _torch()
        u = torch.from_numpy(rng.random(n)).cuda()
        x = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("pf_hmm_prior", self.params(), _lib.PF_F64, _lib.ptr(x), 1, n, None,
                  _lib.ptr(u), _lib.stream_ptr())
        return x.cpu().numpy()[:, None]

    def _step(self, x_prev, t, u, y=None):
        torch = _torch()
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        n = x_prev.shape[0]
        xin = torch.from_numpy(np.ascontiguousarray(x_prev[:, 0])).cuda()
        xout = torch.empty_like(xin)
        d_u = torch.from_numpy(np.ascontiguousarray(u, dtype=np.float64)).cuda()
        lw = d_y = None
        if y is not None:
            lw = torch.empty(n, dtype=torch.float64, device="cuda")
            d_y = torch.tensor([float(np.asarray(y).reshape(-1)[0])], dtype=torch.float64,
                               device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.call("pf_hmm_propagate_weight", self.params(), _lib.PF_F64, _lib.ptr(xin), None,
                  _lib.ptr(xout), _lib.ptr(d_y), _lib.ptr(lw), 1, n, None, int(t),
                  _lib.ptr(d_u), _lib.ptr(st), _lib.stream_ptr())
        return xout.cpu().numpy()[:, None], (None if lw is None else lw.cpu().numpy())

    def sample_transition(self, x_prev, t, rng):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        return self._step(x_prev, t, rng.random(x_prev.shape[0]))[0]

    def log_likelihood(self, y, x, t):
        """log(emission[state, y]) (hmm.py:70-72), looked up on the device."""
        torch = _torch()
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        d_x = torch.from_numpy(np.ascontiguousarray(x[:, 0])).cuda()
        d_y = torch.tensor([float(np.asarray(y).reshape(-1)[0])], dtype=torch.float64,
                           device="cuda")
        out = torch.empty(x.shape[0], dtype=torch.float64, device="cuda")
        _lib.call("pf_hmm_loglik", self.params(), _lib.ptr(d_x), x.shape[0], _lib.ptr(d_y),
                  _lib.ptr(out), _lib.stream_ptr())
        return out.cpu().numpy()

    def sample_observation(self, x, t, rng):
        state = int(np.asarray(x).reshape(-1)[0])
        u = rng.random()
        sym = np.searchsorted(np.cumsum(self.emission[state]), u, side="right")
        return np.array([float(min(sym, self.emission.shape[1] - 1))])


def hmm_exact_filter(model: DiscreteHmm, observations) -> list[tuple[np.ndarray, float]]:
    """Exact forward recursion (hmm.py:80-97): per step (filter vector,
    unnormalised mass), accumulated in extended precision.  Host oracle for
    the verification checks."""
    obs = [int(np.asarray(y).reshape(-1)[0]) for y in observations]
    rho = model.prior.astype(np.longdouble)
    trans = model.transition.astype(np.longdouble)
    emit = model.emission.astype(np.longdouble)
    out = []
    for y in obs:
        rho = (trans.T @ rho) * emit[:, y]
        mass = rho.sum()
        out.append(((rho / mass).astype(np.float64), float(mass)))
    return out


@dataclass
class LinearGaussianModel(_DeviceTables, StateSpaceModel):
    """Drop-in for parpf.models.LinearGaussianModel (linear_gaussian.py:18-95):
    x_t = A x_{t-1} + w, y_t = H x_t + v; the log-likelihood keeps its
    normalising constant.  The GPU kernels support dim_x, dim_y <= 8."""

    A: np.ndarray
    trans_cov: np.ndarray
    H: np.ndarray
    obs_cov: np.ndarray
    prior_mean: np.ndarray
    prior_cov: np.ndarray

    kind = "lgm"

    def __post_init__(self):
        m = lambda a: np.atleast_2d(np.asarray(a, dtype=np.float64))  # noqa: E731
        self.A, self.trans_cov, self.H, self.obs_cov = (m(self.A), m(self.trans_cov), m(self.H),
                                                        m(self.obs_cov))
        self.prior_mean = np.atleast_1d(np.asarray(self.prior_mean, dtype=np.float64))
        self.prior_cov = m(self.prior_cov)
        self.dim_x = self.A.shape[0]
        self.dim_y = self.H.shape[0]
        if self.dim_x > 8 or self.dim_y > 8:
            raise ValueError("the GPU linear-Gaussian kernels support dim_x, dim_y <= 8")
        self._chol_q = np.linalg.cholesky(self.trans_cov)
        self._chol_p0 = np.linalg.cholesky(self.prior_cov)
        sign, logdet = np.linalg.slogdet(self.obs_cov)
        if sign > 0:
            self._chol_r = np.linalg.cholesky(self.obs_cov)
            self._obs_prec = np.linalg.inv(self.obs_cov)
            self._obs_logconst = -0.5 * (self.dim_y * np.log(2.0 * np.pi) + logdet)
        else:
            self._chol_r = None
            self._obs_prec = None
            self._obs_logconst = float("nan")

    @classmethod
    def scalar(cls, a: float = 1.0, q: float = 1.0, h: float = 1.0, r: float = 1.0,
               prior_mean: float = 0.0, prior_var: float = 1.0) -> "LinearGaussianModel":
        return cls(A=[[a]], trans_cov=[[q]], H=[[h]], obs_cov=[[r]],
                   prior_mean=[prior_mean], prior_cov=[[prior_var]])

    def _host_tables(self):
        t = {"A": self.A, "chol_q": self._chol_q, "H": self.H, "prior_mean": self.prior_mean,
             "chol_p0": self._chol_p0}
        if self._obs_prec is not None:
            t["obs_prec"] = self._obs_prec
        return t

    def params(self, n_sub=None, noise_free=False) -> _lib.LgmParams:
        tb = self._tables()
        p = _lib.LgmParams()
        p.dx, p.dy, p.noise_free = self.dim_x, self.dim_y, 1 if noise_free else 0
        p.A, p.chol_q, p.H = tb["A"].data_ptr(), tb["chol_q"].data_ptr(), tb["H"].data_ptr()
        p.obs_prec = tb["obs_prec"].data_ptr() if "obs_prec" in tb else None
        p.prior_mean, p.chol_p0 = tb["prior_mean"].data_ptr(), tb["chol_p0"].data_ptr()
        p.obs_logconst = float(self._obs_logconst)
        return p

    def _planes(self, x):
        torch = _torch()
        x = np.atleast_2d(np.asarray(x, dtype=np.float64))
        return torch.from_numpy(np.ascontiguousarray(x.T)).cuda(), x.shape[0]

    def sample_prior(self, rng, n):
        torch = _torch()
        z = torch.from_numpy(np.ascontiguousarray(rng.standard_normal((n, self.dim_x)))).cuda()
        x = torch.empty((self.dim_x, n), dtype=torch.float64, device="cuda")
        _lib.call("pf_lgm_prior", self.params(), _lib.PF_F64, _lib.ptr(x), 1, n, None,
                  _lib.ptr(z), _lib.stream_ptr())
        return x.t().contiguous().cpu().numpy()

    def _advance(self, x_prev, z, noise_free):
        torch = _torch()
        xin, n = self._planes(x_prev)
        xout = torch.empty_like(xin)
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        d_z = None if z is None else torch.from_numpy(np.ascontiguousarray(z)).cuda()
        _lib.call("pf_lgm_propagate_weight", self.params(noise_free=noise_free), _lib.PF_F64,
                  _lib.ptr(xin), None, _lib.ptr(xout), None, None, 1, n, None, 1,
                  _lib.ptr(d_z), _lib.ptr(st), _lib.stream_ptr())
        if int(st.item()) & _lib.PF_ST_DIVERGED:
            raise NumericalDivergenceError("linear-Gaussian transition produced non-finite states")
        return xout.t().contiguous().cpu().numpy()

    def sample_transition(self, x_prev, t, rng):
        x_prev = np.atleast_2d(np.asarray(x_prev, dtype=np.float64))
        return self._advance(x_prev, rng.standard_normal(x_prev.shape), False)

    def transition_point_prediction(self, x_prev, t):
        return self._advance(x_prev, None, True)

    def log_likelihood(self, y, x, t):
        torch = _torch()
        if self._obs_prec is None:
            raise ValueError("obs_cov is singular; likelihood is undefined")
        xin, n = self._planes(x)
        d_y = torch.from_numpy(np.atleast_1d(np.asarray(y, dtype=np.float64)).copy()).cuda()
        out = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("pf_lgm_loglik", self.params(), _lib.ptr(xin), n, _lib.ptr(d_y),
                  _lib.ptr(out), _lib.stream_ptr())
        return out.cpu().numpy()

    def sample_observation(self, x, t, rng):
        if self._chol_r is None:
            return np.asarray(x) @ self.H.T
        z = rng.standard_normal(self.dim_y)
        return x @ self.H.T + z @ self._chol_r.T


def kalman_filter(model: LinearGaussianModel, observations):
    """Exact Kalman posteriors (linear_gaussian.py:98-125): the prior, then
    one (mean, cov) per observation.  Host oracle for the verification
    checks."""
    observations = np.asarray(observations, dtype=np.float64)
    if observations.size == 0:
        observations = observations.reshape(0, model.dim_y)
    observations = np.atleast_2d(observations)
    if observations.ndim != 2 or observations.shape[1] != model.dim_y:
        raise ValueError("observations must have shape (T, dim_y)")
    mean = model.prior_mean.copy()
    cov = model.prior_cov.copy()
    out = [(mean.copy(), cov.copy())]
    eye = np.eye(model.dim_x)
    for y in observations:
        mean = model.A @ mean
        cov = model.A @ cov @ model.A.T + model.trans_cov
        innov = y - model.H @ mean
        s = model.H @ cov @ model.H.T + model.obs_cov
        try:
            gain = np.linalg.solve(s, model.H @ cov).T
        except np.linalg.LinAlgError as exc:
            raise NumericalDivergenceError(f"singular innovation covariance: {exc}") from exc
        mean = mean + gain @ innov
        cov = (eye - gain @ model.H) @ cov
        out.append((mean.copy(), cov.copy()))
    return out


def lorenz_transition(x, rng, model: Lorenz63Model | None = None) -> np.ndarray:
    """One observation interval for a single 3-vector state (lorenz63.py:72-78)."""
    model = model or Lorenz63Model()
    return model.sample_transition(np.asarray(x, dtype=np.float64)[None, :], 1, rng)[0]


def lorenz_log_likelihood(y: float, x, model: Lorenz63Model | None = None) -> float:
    """Scalar-observation log-likelihood of one state (lorenz63.py:81-85)."""
    model = model or Lorenz63Model()
    return float(model.log_likelihood(np.array([y]), np.asarray(x)[None, :], 1)[0])
