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


class StreamingEnsemble:
    """The oracle ensemble advanced one observation at a time, so oracle-mode
    parity runs at the BASELINE config sizes (cfg0: 500 observations; cfg3:
    8 x 512 particles of a 3000-value state) never hold the whole tape.

    Same seed tree and per-filter draw order as ``run_ensemble`` /
    ``run_filter`` (ensemble.py:56-60, filters.py:87-112): filter f draws
    from default_rng(SeedSequence(master).spawn(M)[f]) its prior, then per
    observation its transition noise and (unless collapsed) n+1 exponentials.

    ``prior`` is the (M, N, 3) prior-normal tape (None for a deterministic
    prior); ``step(k)`` advances every filter by observation k and returns a
    dict with that step's tape (``noise``, ``uniforms``; the DrawTape layout)
    and results (``ancestors`` (M, N), ``estimates`` (M, dim_x), ``lnc``
    (M,), ``collapsed`` (M,), ``log_w`` (M, N)).
    """

    def __init__(self, model, observations, n_filters, n_particles, master_seed):
        self.model = model
        self.obs = np.atleast_2d(np.asarray(observations, dtype=np.float64))
        self.M, self.N = n_filters, n_particles
        self.rngs = [np.random.default_rng(s) for s in orc.filter_seeds(master_seed, n_filters)]
        xs, zs = zip(*[orc._prior(model, r, n_particles) for r in self.rngs])
        self.x = list(xs)
        self.prior = None if zs[0] is None else np.stack(zs)
        self.lnc = np.zeros(n_filters)
        self.fhn = isinstance(model, orc.FhnConfigModel)

    def step(self, k):
        M, N = self.M, self.N
        noise, uni, anc, est, lw, coll = [], np.full((M, N), np.nan), [], [], [], []
        for f in range(M):
            recs = []
            self.x[f], self.lnc[f], c = orc._bf_step(self.model, self.x[f], self.lnc[f],
                                                     self.obs[k], k + 1, self.rngs[f],
                                                     keep_steps=True, steps=recs)
            r = recs[0]
            noise.append(r.noise.reshape(self.model.substeps, 2, N, -1) if self.fhn else r.noise)
            if r.u is not None:
                uni[f] = r.u
            anc.append(r.ancestors)
            lw.append(r.log_w)
            coll.append(c)
            est.append(orc.posterior_mean(np.full(N, 1.0 / N), self.x[f]))
        return {"noise": np.stack(noise), "uniforms": uni, "ancestors": np.stack(anc),
                "estimates": np.stack(est), "lnc": self.lnc.copy(),
                "collapsed": np.array(coll), "log_w": np.stack(lw)}
