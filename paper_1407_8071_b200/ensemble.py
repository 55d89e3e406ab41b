"""Ensembles of M independent filters (drop-in for parpf/ensemble.py).

``run_ensemble`` keeps the reference signature (ensemble.py:76-78).  All M
filters live as segments of one device batch; under torch.distributed the
filters are block-sharded across ranks (one GPU each) and the per-step
estimates are combined with one disjoint-support all-reduce per observation
(dist.py), so results are bit-identical for any GPU count.  ``workers``
keeps its meaning of "affects wall time only" and is validated but unused.
"""

from __future__ import annotations

import time
from collections.abc import Sequence
from dataclasses import dataclass

import numpy as np

from . import _lib, dist, philox
from .models import estimate_width
from .bank import DrawTape, FilterBank
from .filters import FilterOutput, _bank_seconds, _validate

CENTRALISED = "centralised"
ENSEMBLE = "ensemble"


@dataclass
class EnsembleOutput:
    """M independent filter records plus their averaged estimators
    (ensemble.py:27-53)."""

    variant: str
    n_filters: int
    n_particles: int
    master_seed: object
    filter_outputs: list
    mean_estimates: np.ndarray
    filter_seconds: np.ndarray
    total_seconds: float

    @property
    def n_steps(self) -> int:
        return self.mean_estimates.shape[0]

    def same_result(self, other: "EnsembleOutput") -> bool:
        return (
            self.variant == other.variant
            and self.n_filters == other.n_filters
            and self.n_particles == other.n_particles
            and np.array_equal(self.mean_estimates, other.mean_estimates)
            and all(a.same_result(b) for a, b in zip(self.filter_outputs, other.filter_outputs))
        )


class _EnsembleFilterOutput(FilterOutput):
    """FilterOutput whose ``seed`` (the filter's SeedSequence child,
    ensemble.py:96-99) is resolved lazily."""

    @property
    def seed(self):
        s = self.__dict__["_seed"]
        if isinstance(s, tuple) and isinstance(s[0], philox.FilterSeeds):
            s = s[0][s[1]]
            self.__dict__["_seed"] = s
        return s

    @seed.setter
    def seed(self, value):
        self.__dict__["_seed"] = value


class _FilterOutputs(Sequence):
    """EnsembleOutput.filter_outputs as a read-only sequence whose
    FilterOutput records are built on first access (a bank has thousands of
    filters; most callers only read the averaged estimates)."""

    def __init__(self, variant, n_particles, seeds, est, lnc, coll, secs):
        self._args = (variant, n_particles, seeds, est, lnc, coll, secs)
        self._cache = {}

    def __len__(self):
        return self._args[3].shape[1]

    def __getitem__(self, f):
        if isinstance(f, slice):
            return [self[i] for i in range(*f.indices(len(self)))]
        if f < 0:
            f += len(self)
        if not 0 <= f < len(self):
            raise IndexError(f)
        if f not in self._cache:
            variant, n_particles, seeds, est, lnc, coll, secs = self._args
            steps = [int(k) + 1 for k in np.nonzero(coll[:, f])[0]]
            self._cache[f] = _EnsembleFilterOutput(variant, n_particles, (seeds, f), est[:, f, :],
                                                   lnc[:, f], secs, steps)
        return self._cache[f]

    def __eq__(self, other):
        return list(self) == list(other)


def filter_seeds(master_seed, n_filters: int):
    """ensemble.py:56-60 (same SeedSequence tree)."""
    return philox.filter_seeds(master_seed, n_filters)


def average_estimates(filter_outputs) -> np.ndarray:
    """Left-to-right mean of per-filter estimates (ensemble.py:68-73),
    evaluated on the GPU with the same association."""
    import torch

    _lib.require_cuda()
    est = np.stack([np.asarray(o.estimates, dtype=np.float64) for o in filter_outputs], axis=1)
    d = torch.from_numpy(np.ascontiguousarray(est)).cuda()
    T, M, dim = d.shape
    out = torch.empty((T, dim), dtype=torch.float64, device="cuda")
    _lib.call("pf_ensemble_average", _lib.ptr(d), T, M, dim, _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()


def run_ensemble(model, observations, variant: str, n_filters: int, n_particles: int,
                 master_seed, workers: int = 1, *, dtype=None, tape: DrawTape | None = None,
                 estimate: str = "full", shard: bool | None = None) -> EnsembleOutput:
    """ensemble.py:76-111 on the GPU bank.

    shard: None -> shard across ranks when torch.distributed is initialised
    with world_size > 1; every rank returns the full EnsembleOutput.
    """
    import torch

    if n_filters < 1 or n_particles < 1:
        raise ValueError("n_filters and n_particles must be >= 1")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    obs = _validate(observations, variant, model)
    T = obs.shape[0]
    rank, world = dist.world()
    # exchange path: any initialised process group (shard=True forces it even
    # for world size 1, which exercises the NCCL side-stream exchange)
    use_exch = (world > 1 and shard is not False) or (shard is True and dist.initialized())
    if not use_exch:
        rank, world = 0, 1
    lo, hi = dist.shard_range(n_filters, rank, world) if world > 1 else (0, n_filters)
    keys, seeds = philox.filter_keys_and_seeds(master_seed, n_filters)
    started = time.perf_counter()
    dev = torch.device("cuda", torch.cuda.current_device())
    est_dim = estimate_width(model, estimate)
    est_full = torch.zeros((T, n_filters, est_dim), dtype=torch.float64, device=dev)
    # a rank whose block is empty (n_filters < world) runs no bank but still
    # joins every collective, so no rank waits on another forever
    bank = None
    if hi > lo:
        bank = FilterBank(model, hi - lo, n_particles, keys[lo:hi], T, dtype=dtype, tape=tape,
                          filter_offset=lo, estimate=estimate, est_buffer=est_full,
                          est_row_offset=lo, variant=variant)
        bank.load_observations(obs)
        bank.init()
    # NCCL process group: the native driver issues the per-observation
    # exchange itself (pf_comm); otherwise the torch side-stream exchange
    comm = dist.native_comm() if use_exch else None
    native = bank is None or bank._native_ok()
    secs = None
    if native and (not use_exch or comm is not None):
        if bank is not None:
            if comm is not None:
                bank.set_exchange(comm, n_filters * est_dim)
            # the whole record in one native call, per-step device times from it
            bank.run_native(0, T, time_steps=True)
            secs = bank.last_step_ms.astype(np.float64) / 1e3
        else:
            comm.exchange_steps(est_full, 0, T)
            secs = np.zeros(T)
        if comm is not None:
            comm.join()
    else:
        exch = dist.EstimateExchange(est_full) if use_exch else None
        events = [torch.cuda.Event(enable_timing=True) for _ in range(T + 1)]
        events[0].record()
        for k in range(T):
            if bank is not None:
                bank.step(k)
            events[k + 1].record()
            if exch is not None:
                exch.step_done(k)
        if exch is not None:
            exch.finish()
    mean = torch.empty((T, est_dim), dtype=torch.float64, device=dev)
    _lib.call("pf_ensemble_average", _lib.ptr(est_full), T, n_filters, est_dim, _lib.ptr(mean),
              _lib.stream_ptr())
    # small end-of-run traces: lnc, collapse flags, status (disjoint support)
    lnc_full = torch.zeros((T, n_filters), dtype=torch.float64, device=dev)
    coll_full = torch.zeros((T, n_filters), dtype=torch.int32, device=dev)
    st_full = torch.zeros(n_filters, dtype=torch.int32, device=dev)
    if bank is not None:
        lnc_full[:, lo:hi] = bank.lnc_tr
        coll_full[:, lo:hi] = bank.coll_tr.to(torch.int32)
        st_full[lo:hi] = bank.status
    if comm is not None:  # one packed exchange (small integers are exact in fp64)
        packed = torch.cat([lnc_full.reshape(-1), coll_full.reshape(-1).double(),
                            st_full.double()])
        comm.allreduce_f64(packed)
        lnc_full.copy_(packed[: T * n_filters].view(T, n_filters))
        coll_full.copy_(packed[T * n_filters: 2 * T * n_filters].view(T, n_filters).to(torch.int32))
        st_full.copy_(packed[2 * T * n_filters:].to(torch.int32))
    elif use_exch:
        for t_ in (lnc_full, coll_full, st_full):
            dist.allreduce_disjoint(t_)
    torch.cuda.synchronize()
    total = time.perf_counter() - started
    _lib.raise_status(st_full.cpu().numpy())
    if secs is None:
        secs = _bank_seconds(events)
    est_h = est_full.cpu().numpy()
    lnc_h = lnc_full.cpu().numpy()
    coll_h = coll_full.cpu().numpy()
    outputs = _FilterOutputs(variant, n_particles, seeds, est_h,
                             lnc_h, coll_h, secs)
    filter_seconds = np.full(n_filters, float(secs.sum()))
    return EnsembleOutput(variant, n_filters, n_particles, master_seed, outputs,
                          mean.cpu().numpy(), filter_seconds, total)


def ensemble_estimate(out: EnsembleOutput, t: int) -> np.ndarray:
    """ensemble.py:114-118."""
    if not 0 <= t < out.n_steps:
        raise ValueError(f"step index {t} outside 0..{out.n_steps - 1}")
    return out.mean_estimates[t]


def time_error_index(variant: str, n_filters: int, n_particles: int) -> float:
    """ensemble.py:121-135."""
    if n_filters < 1 or n_particles < 1:
        raise ValueError("n_filters and n_particles must be >= 1")
    if variant == CENTRALISED:
        return 1.0
    if variant == ENSEMBLE:
        return 1.0 / n_filters + 1.0 / n_particles
    raise ValueError(f"unknown variant {variant!r}")
