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
