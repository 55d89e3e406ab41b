"""Independent replicate runs as ONE filter bank.

The reference runs replicates one at a time (or over a fork pool):
``run_filter(..., spawn_child(parent, r))`` for the verification suite
(verify.py:87-146) and ``run_filter`` / ``run_ensemble`` per replicate of a
sweep cell (bench.py:89-117).  Replicates are independent filters with their
own seeds, which is exactly what a bank is: R filter replicates become a bank
of R filters, R ensemble replicates a bank of R*M filters (replicate r's
filters keyed by ``spawn(M)`` of its seed, as run_ensemble would), so a whole
cell runs as a few launches per observation.  Results per replicate equal the
single-run API's (same keys, same kernels); only wall times are amortised.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib, philox
from .bank import FilterBank
from .filters import _validate
from .models import estimate_width

# particles per bank chunk (bounds device memory for large cells)
MAX_BANK_PARTICLES = 1 << 26


@dataclass
class ReplicateBatch:
    """Per-replicate results of a batched run."""

    estimates: np.ndarray        # (R, T, dim) filter estimates / ensemble means
    log_norm_const: np.ndarray   # (R, T) (filters) or (R, M, T) (ensembles)
    collapse_counts: np.ndarray  # (R,) collapse events (summed over an ensemble's filters)
    diverged: np.ndarray         # (R,) bool: a filter raised NumericalDivergenceError
    seconds: float               # device time of the whole batch


def _chunks(R, per_rep):
    n = max(1, MAX_BANK_PARTICLES // max(per_rep, 1))
    return [(lo, min(R, lo + n)) for lo in range(0, R, n)]


def _run_bank(model, obs, variant, keys, n_particles, dtype, estimate):
    import torch

    T = obs.shape[0]
    bank = FilterBank(model, keys.shape[0], n_particles, keys, T, dtype=dtype,
                      estimate=estimate, variant=variant)
    bank.load_observations(obs)
    bank.init()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    bank.run()
    end.record()
    torch.cuda.synchronize()
    status = bank.status.cpu().numpy()
    # NaN weights downstream of a divergence are the divergence's symptom
    if np.any((status & _lib.PF_ST_NAN_WEIGHT) & ~(status & _lib.PF_ST_DIVERGED)):
        raise ValueError("log weights contain NaN")
    return bank, status, start.elapsed_time(end) / 1e3


def filter_replicates(model, observations, variant: str, n_particles: int, seeds, *,
                      dtype=None, estimate: str = "full") -> ReplicateBatch:
    """R = len(seeds) independent ``run_filter(model, obs, variant, n, seed_r)``."""
    obs = _validate(observations, variant, model)
    keys = philox.seed_keys(seeds)
    R, T = keys.shape[0], obs.shape[0]
    dim = estimate_width(model, estimate)
    est = np.empty((R, T, dim))
    lnc = np.empty((R, T))
    coll = np.zeros(R, dtype=np.int64)
    div = np.zeros(R, dtype=bool)
    secs = 0.0
    for lo, hi in _chunks(R, n_particles):
        bank, status, s = _run_bank(model, obs, variant, keys[lo:hi], n_particles, dtype,
                                    estimate)
        est[lo:hi] = bank.est.cpu().numpy().transpose(1, 0, 2)
        lnc[lo:hi] = bank.lnc_tr.cpu().numpy().T
        coll[lo:hi] = bank.coll_tr.cpu().numpy().sum(axis=0)
        div[lo:hi] = (status & _lib.PF_ST_DIVERGED) != 0
        secs += s
        del bank
    return ReplicateBatch(est, lnc, coll, div, secs)


def ensemble_replicates(model, observations, variant: str, n_filters: int, n_particles: int,
                        seeds, *, dtype=None, estimate: str = "full") -> ReplicateBatch:
    """R independent ``run_ensemble(model, obs, variant, M, n, seed_r)``; the
    mean over each replicate's M filters uses the reference's left-to-right
    association (pf_ensemble_average)."""
    import torch

    obs = _validate(observations, variant, model)
    M, T = n_filters, obs.shape[0]
    keys = np.concatenate([philox.filter_keys(s, M) for s in seeds]).astype(np.uint32)
    R = len(seeds)
    dim = estimate_width(model, estimate)
    est = np.empty((R, T, dim))
    lnc = np.empty((R, M, T))
    coll = np.zeros(R, dtype=np.int64)
    div = np.zeros(R, dtype=bool)
    secs = 0.0
    for lo, hi in _chunks(R, M * n_particles):
        r = hi - lo
        bank, status, s = _run_bank(model, obs, variant, keys[lo * M:hi * M], n_particles,
                                    dtype, estimate)
        # (T, r*M, dim) -> (r, T, M, dim) -> per-replicate left-to-right means
        e = bank.est.view(T, r, M, dim).permute(1, 0, 2, 3).contiguous()
        mean = torch.empty((r * T, dim), dtype=torch.float64, device=e.device)
        _lib.call("pf_ensemble_average", _lib.ptr(e), r * T, M, dim, _lib.ptr(mean),
                  _lib.stream_ptr())
        est[lo:hi] = mean.view(r, T, dim).cpu().numpy()
        lnc[lo:hi] = bank.lnc_tr.cpu().numpy().T.reshape(r, M, T)
        coll[lo:hi] = bank.coll_tr.cpu().numpy().astype(np.int64).sum(axis=0).reshape(r, M) \
            .sum(axis=1)
        div[lo:hi] = ((status & _lib.PF_ST_DIVERGED) != 0).reshape(r, M).any(axis=1)
        secs += s
        del bank, e, mean
    return ReplicateBatch(est, lnc, coll, div, secs)
