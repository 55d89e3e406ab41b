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
    noise:    list over steps of (M, n_sub, N, 3) [Lorenz] or
              (M, n_sub, 2, N, nodes) [FH-N]
    uniforms: list over steps of (M, N); rows of collapsed filters are NaN
    """
    traces, mean = orc.run_ensemble(model, observations, n_filters, n_particles, master_seed,
                                    keep_steps=True, variant=variant)
    T = len(traces[0].steps)
    fhn = isinstance(model, orc.FhnConfigModel)
    prior = None if fhn else np.stack([tr.prior_noise for tr in traces])
    noise, uniforms, uniforms_first = [], [], []
    for k in range(T):
        if fhn:
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
