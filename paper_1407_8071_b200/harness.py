"""Data preparation around the bank (parpf/bench.py:37-86):
hierarchical seeding, idempotent load-or-simulate of the observation record
with ``.17g`` CSV files, and the error reference (truth or a proxy filter
run on the GPU bank)."""

from __future__ import annotations

import os

import numpy as np

from .filters import run_filter
from .io import read_array_csv, write_array_csv
from .simulate import simulate


def spawn_child(parent: np.random.SeedSequence, index: int) -> np.random.SeedSequence:
    """The index-th spawn of parent, constructible out of order (bench.py:37-40)."""
    return np.random.SeedSequence(entropy=parent.entropy,
                                  spawn_key=tuple(parent.spawn_key) + (index,))


def root_sequences(seed):
    """(simulation, proxy reference, sweep) children of the sweep seed
    (bench.py:49-52)."""
    sim_ss, ref_ss, sweep_ss = np.random.SeedSequence(seed).spawn(3)
    return sim_ss, ref_ss, sweep_ss


def prepare_data(model, n_observations: int, seed, observations_path=None,
                 trajectory_path=None):
    """Load or simulate (states, observations) (bench.py:55-74).

    Requested output paths that do not exist yet are written, so repeated
    calls with the same seed are idempotent.
    """
    sim_ss, _, _ = root_sequences(seed)
    if observations_path and os.path.exists(observations_path):
        _, observations = read_array_csv(observations_path)
        states = None
        if trajectory_path and os.path.exists(trajectory_path):
            _, states = read_array_csv(trajectory_path)
        return states, observations
    states, observations = simulate(model, n_observations, sim_ss)
    if observations_path:
        write_array_csv(observations_path, "y", observations)
    if trajectory_path:
        write_array_csv(trajectory_path, "x", states, first_step=0)
    return states, observations


def compute_reference(model, states, observations, seed, reference: str = "proxy",
                      proxy_particles: int = 10_000, dtype=None):
    """Error baseline passed through the model's error projection
    (bench.py:77-86): the truth, or a large single bootstrap filter on the
    GPU bank seeded by the sweep's reference child."""
    if reference == "truth":
        if states is None:
            raise OSError("ground-truth reference requested but no trajectory available")
        return model.error_projection(np.asarray(states)[1:])
    _, ref_ss, _ = root_sequences(seed)
    proxy = run_filter(model, observations, "bootstrap", proxy_particles, ref_ss, dtype=dtype)
    return model.error_projection(proxy.estimates)


# ---------------------------------------------------------------------------
# Sweeps (bench.py:43-214)
# ---------------------------------------------------------------------------


def build_model(cfg):
    """bench.py:43-46: the stock Lorenz-63 model or the FH-N network on a
    fhn_grid x fhn_grid lattice."""
    from .models import FhnNetworkModel, Lorenz63Model

    if cfg.model == "lorenz63":
        return Lorenz63Model()
    return FhnNetworkModel(J=cfg.fhn_grid)


def variant_index(variant: str, n_filters: int, n_particles: int) -> float:
    """bench.py:120-125."""
    from .ensemble import time_error_index

    if variant == "centralised-bf":
        return time_error_index("centralised", n_filters, n_particles)
    if variant in ("ensemble-bf", "ensemble-apf"):
        return time_error_index("ensemble", n_filters, n_particles)
    return float("nan")


def _cell_replicates(model, observations, variant, M, N, island_period, seeds, dtype):
    """All replicates of one sweep cell -> per replicate (projected estimates
    or None if diverged, collapse count, total seconds, seconds per step).
    bench.py:89-117, with the replicates batched into one bank."""
    from .islands import run_double_bootstrap
    from .replicates import ensemble_replicates, filter_replicates

    R, T = len(seeds), np.atleast_2d(observations).shape[0]
    if variant == "double-bf":
        out = []
        for s in seeds:
            try:
                fo = run_double_bootstrap(model, observations, M, N, island_period, s,
                                          dtype=dtype)
            except Exception as exc:  # NumericalDivergenceError
                from .exceptions import NumericalDivergenceError

                if not isinstance(exc, NumericalDivergenceError):
                    raise
                out.append((None, 0, 0.0, 0.0))
                continue
            out.append((model.error_projection(fo.estimates), len(fo.collapse_steps),
                        fo.total_seconds, fo.total_seconds / fo.n_steps))
        return out
    if variant == "centralised-bf":
        b = filter_replicates(model, observations, "bootstrap", M * N, seeds, dtype=dtype,
                              estimate="projection")
    elif variant in ("ensemble-bf", "ensemble-apf"):
        inner = "bootstrap" if variant == "ensemble-bf" else "auxiliary"
        b = ensemble_replicates(model, observations, inner, M, N, seeds, dtype=dtype,
                                estimate="projection")
    else:
        raise ValueError(f"unknown variant {variant!r}")
    per = b.seconds / R  # batched: device time amortised per replicate
    return [(None, 0, 0.0, 0.0) if b.diverged[r] else
            (b.estimates[r], int(b.collapse_counts[r]), per, per / T) for r in range(R)]


def run_sweep(cfg, model=None, states=None, observations=None, reference=None, dtype=None):
    """bench.py:136-214 on the GPU: one MetricRecord per (variant, M, N) cell
    with MSE mean / variance over replicates, squared bias of the replicate
    mean, collapse counts (a divergent replicate is excluded and counted) and
    the time-error index.  Seeds follow the reference tree: sweep child ->
    cell ci -> replicate r.  Wall columns hold device seconds (amortised over
    the replicates of a batched cell)."""
    from .metrics import MetricRecord, empirical_mse

    model = model or build_model(cfg)
    if observations is None:
        states, observations = prepare_data(model, cfg.n_observations, cfg.seed,
                                            cfg.observations_path, cfg.trajectory_path)
    if reference is None:
        reference = compute_reference(model, states, observations, cfg.seed, cfg.reference,
                                      cfg.proxy_particles)
    _, _, sweep_ss = root_sequences(cfg.seed)
    cells = [(v, m, n) for v in cfg.variants for m in cfg.n_filters_list
             for n in cfg.n_particles_list]
    records = []
    for ci, (variant, M, N) in enumerate(cells):
        cell_ss = spawn_child(sweep_ss, ci)
        seeds = [spawn_child(cell_ss, r) for r in range(cfg.replicates)]
        per_rep = _cell_replicates(model, observations, variant, M, N, cfg.island_period,
                                   seeds, dtype)
        mses, valid, collapse_total = [], [], 0
        for projected, collapse, _, _ in per_rep:
            collapse_total += collapse
            mse = empirical_mse(projected, reference) if projected is not None else float("nan")
            if np.isfinite(mse):
                mses.append(mse)
                valid.append(projected)
            else:
                collapse_total += 1
        mse_mean = float(np.mean(mses)) if mses else float("nan")
        mse_var = float(np.var(mses, ddof=1)) if len(mses) > 1 else float("nan")
        if valid:
            mean_est = valid[0].copy()
            for proj in valid[1:]:
                mean_est += proj
            mean_est /= float(len(valid))
            bias_sq = float(np.mean((mean_est - reference) ** 2))
        else:
            bias_sq = float("nan")
        records.append(MetricRecord(
            variant=variant, n_filters=M, n_particles=N, total_particles=M * N,
            replicates=cfg.replicates, mse_mean=mse_mean, mse_var=mse_var, bias_sq=bias_sq,
            wall_per_step_s=float(np.mean([p for _, _, _, p in per_rep])),
            wall_total_s=float(np.mean([t for _, _, t, _ in per_rep])),
            time_error_index=variant_index(variant, M, N),
            collapse_count=collapse_total))
    return records
