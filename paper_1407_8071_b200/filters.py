"""Single-filter drivers and step functions (drop-in for parpf/filters.py).

* :func:`run_filter` - filters.py:163-193; runs on the GPU bank with M=1.
* :func:`bf_init` / :func:`bf_step` - filters.py:87-112; reference-style
  step functions over host ParticleApproximation containers whose
  arithmetic (propagation, weighting, normalisation, resampling, gather)
  runs on the GPU via the model hooks and the L2 operators.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, philox
from .bank import DrawTape, FilterBank
from .core import ParticleApproximation, StateSpaceModel, normalize_log_weights, uniform_weights
from .exceptions import UnsupportedModelError, WeightCollapseError
from .resampling import multinomial_resample_indices

VARIANT_BOOTSTRAP = "bootstrap"
VARIANT_AUXILIARY = "auxiliary"
KNOWN_VARIANTS = (VARIANT_BOOTSTRAP, VARIANT_AUXILIARY)


@dataclass
class FilterOutput:
    """Per-step record of one filter run (filters.py:43-78)."""

    variant: str
    n_particles: int
    seed: object
    estimates: np.ndarray
    log_norm_const: np.ndarray
    step_seconds: np.ndarray
    collapse_steps: list = field(default_factory=list)

    @property
    def n_steps(self) -> int:
        return self.estimates.shape[0]

    @property
    def total_seconds(self) -> float:
        return float(self.step_seconds.sum())

    def same_result(self, other: "FilterOutput") -> bool:
        return (
            self.variant == other.variant
            and self.n_particles == other.n_particles
            and self.collapse_steps == other.collapse_steps
            and np.array_equal(self.estimates, other.estimates)
            and np.array_equal(self.log_norm_const, other.log_norm_const)
        )


def _check_uniform(state: ParticleApproximation):
    n = state.n_particles
    if not np.allclose(state.weights, 1.0 / n, rtol=0.0, atol=1e-12):
        raise ValueError("step functions expect uniform (post-resampling) weights")


def bf_init(model: StateSpaceModel, n_particles: int, rng) -> ParticleApproximation:
    if n_particles < 1:
        raise ValueError("n_particles must be >= 1")
    particles = model.sample_prior(rng, n_particles)
    return ParticleApproximation(particles, uniform_weights(n_particles), log_norm_const=0.0, t=0)


def bf_step(model: StateSpaceModel, state: ParticleApproximation, y, rng) -> ParticleApproximation:
    """One bootstrap step with the reference's control flow and draw order."""
    _check_uniform(state)
    t = state.t + 1
    n = state.n_particles
    propagated = model.sample_transition(state.particles, t, rng)
    log_w = model.log_likelihood(y, propagated, t)
    try:
        weights, log_mean_raw = normalize_log_weights(log_w)
    except WeightCollapseError:
        return ParticleApproximation(propagated, uniform_weights(n), state.log_norm_const, t,
                                     collapsed=True)
    idx = multinomial_resample_indices(weights, n, rng)
    return ParticleApproximation(np.asarray(propagated)[idx], uniform_weights(n),
                                 state.log_norm_const + log_mean_raw, t)


def apf_step(model: StateSpaceModel, state: ParticleApproximation, y, rng) -> ParticleApproximation:
    """One auxiliary step (filters.py:115-154), same control flow and draw
    order, arithmetic on the GPU through the model hooks and L2 operators."""
    import torch

    if not model.has_point_prediction():
        raise UnsupportedModelError("auxiliary filtering needs transition_point_prediction")
    _check_uniform(state)
    t = state.t + 1
    n = state.n_particles
    predicted = model.transition_point_prediction(state.particles, t)
    lam = model.log_likelihood(y, predicted, t)
    collapsed = False
    try:
        first_stage, log_mean_first = normalize_log_weights(lam)
    except WeightCollapseError:
        collapsed = True
        lam = np.zeros(n)
        first_stage, log_mean_first = uniform_weights(n), 0.0
    ancestors = multinomial_resample_indices(first_stage, n, rng)
    propagated = model.sample_transition(np.asarray(state.particles)[ancestors], t, rng)
    # log w = log p(y | x) - lambda[ancestors] (filters.py:143), on the device
    d_lw = torch.from_numpy(np.ascontiguousarray(model.log_likelihood(y, propagated, t),
                                                 dtype=np.float64)).cuda()
    d_lam = torch.from_numpy(np.ascontiguousarray(lam, dtype=np.float64)).cuda()
    d_anc = torch.from_numpy(ancestors.astype(np.int32)).cuda()
    _lib.call("pf_apf_second_stage_weights", _lib.PF_F64, _lib.ptr(d_lw), _lib.ptr(d_lam),
              _lib.ptr(d_anc), n, _lib.stream_ptr())
    log_w = d_lw.cpu().numpy()
    try:
        weights, log_mean_second = normalize_log_weights(log_w)
    except WeightCollapseError:
        return ParticleApproximation(propagated, uniform_weights(n), state.log_norm_const, t,
                                     collapsed=True)
    idx = multinomial_resample_indices(weights, n, rng)
    return ParticleApproximation(np.asarray(propagated)[idx], uniform_weights(n),
                                 state.log_norm_const + log_mean_first + log_mean_second, t,
                                 collapsed=collapsed)


def _validate(observations, variant, model):
    obs = np.atleast_2d(np.asarray(observations, dtype=np.float64))
    if obs.shape[0] == 0:
        raise ValueError("observation sequence must be non-empty")
    if variant not in KNOWN_VARIANTS:
        raise ValueError(f"unknown filter variant {variant!r}")
    if variant == VARIANT_AUXILIARY and not model.has_point_prediction():
        raise UnsupportedModelError("auxiliary filtering needs transition_point_prediction")
    if getattr(model, "dim_y", obs.shape[1]) == 1 and obs.ndim == 2 and obs.shape[1] != 1:
        obs = obs.reshape(-1, 1)
    return obs


def _bank_seconds(events):
    """Per-step device times from CUDA events recorded around each step."""
    return np.array([events[i].elapsed_time(events[i + 1]) / 1e3
                     for i in range(len(events) - 1)])


def run_filter(model: StateSpaceModel, observations, variant: str, n_particles: int, seed, *,
               dtype=None, tape: DrawTape | None = None, estimate: str = "full") -> FilterOutput:
    """filters.py:163-193 on the GPU bank (M=1).

    Production mode (tape=None): Philox keyed by ``seed``'s SeedSequence.
    Oracle mode: ``tape`` supplies the reference's draws (bank.DrawTape).
    ``step_seconds`` holds device time per observation step.
    """
    import torch

    obs = _validate(observations, variant, model)
    if n_particles < 1:
        raise ValueError("n_particles must be >= 1")
    keys = philox.seed_key(seed)[None, :]
    bank = FilterBank(model, 1, n_particles, keys, obs.shape[0], dtype=dtype, tape=tape,
                      estimate=estimate, variant=variant)
    bank.load_observations(obs)
    bank.init()
    if bank._native_ok():
        # the whole record in one native call (pf_bank_run), per-step device times
        bank.run_native(0, obs.shape[0], time_steps=True)
        secs = bank.last_step_ms.astype(np.float64) / 1e3
    else:  # oracle mode (tape): the per-step hook loop
        events = [torch.cuda.Event(enable_timing=True) for _ in range(obs.shape[0] + 1)]
        events[0].record()
        for k in range(obs.shape[0]):
            bank.step(k)
            events[k + 1].record()
        secs = None
    torch.cuda.synchronize()
    bank.check_status()
    if secs is None:
        secs = _bank_seconds(events)
    return FilterOutput(variant, n_particles, seed, bank.est[:, 0, :].cpu().numpy(),
                        bank.lnc_tr[:, 0].cpu().numpy(), secs, bank.collapse_steps()[0])
