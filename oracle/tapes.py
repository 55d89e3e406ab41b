"""TEST INFRASTRUCTURE ONLY: turn oracle filter traces into oracle-mode draw
tapes for the GPU bank (the SURVEY §8c recipe: feed identical draws to both
implementations).

Returns plain numpy arrays; callers wrap them in
``paper_1407_8071_b200.DrawTape``.
"""

from __future__ import annotations

import numpy as np

from . import parpf_oracle as orc


def ensemble_with_tape(model, observations, n_filters, n_particles, master_seed,
                       variant="bootstrap"):
    """Run the oracle ensemble and collect (traces, mean, prior, noise, uniforms).

    prior:    (M, N, 3) or None (FH-N has a deterministic prior)
    noise:    list over steps of (M, n_sub, N, 3) [Lorenz],
              (M, n_sub, 2, N, nodes) [FH-N lattice] or (M, N, nodes) [FH-N
              network; its stimulus uniforms come from stim_tape(traces)]
    uniforms: list over steps of (M, N); rows of collapsed filters are NaN
    """
    traces, mean = orc.run_ensemble(model, observations, n_filters, n_particles, master_seed,
                                    keep_steps=True, variant=variant)
    T = len(traces[0].steps)
    fhn = isinstance(model, orc.FhnConfigModel)
    net = isinstance(model, orc.FhnNetworkModel)
    prior = None if (fhn or net) else np.stack([tr.prior_noise for tr in traces])
    noise, uniforms, uniforms_first = [], [], []
    for k in range(T):
        if net:
            z = np.stack([tr.steps[k].noise[2].reshape(n_particles, -1) for tr in traces])
        elif fhn:
            z = np.stack([tr.steps[k].noise.reshape(model.substeps, 2, n_particles, -1)
                          for tr in traces])
        else:
            z = np.stack([tr.steps[k].noise for tr in traces])
        noise.append(z)
        u = np.full((n_filters, n_particles), np.nan)
        for f, tr in enumerate(traces):
            if tr.steps[k].u is not None:
                u[f] = tr.steps[k].u
        uniforms.append(u)
        if variant == "auxiliary":
            uniforms_first.append(np.stack([tr.steps[k].u_first for tr in traces]))
    if variant == "auxiliary":
        return traces, mean, prior, noise, uniforms, uniforms_first
    return traces, mean, prior, noise, uniforms


def stim_tape(traces):
    """FH-N network: per step k the (M, 2, N) fire / select uniforms the
    oracle filters consumed (fhn.py:158-159 draw order)."""
    T = len(traces[0].steps)
    return [np.stack([np.stack([tr.steps[k].noise[0], tr.steps[k].noise[1]]) for tr in traces])
            for k in range(T)]
