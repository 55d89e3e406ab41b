#!/usr/bin/env python3
"""Statistical fixtures for the production-mode parity tests, computed with
the UNMODIFIED reference (parpf.run_ensemble on the config adapters of
make_golden.py) in the build container:

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_stats.py [--workers 8]

Writes tests/golden/stats.npz:

* cfg0 (SURVEY §7.4, §8d "Statistical production-mode test"; BASELINE cfg0):
  Lorenz-63, truth seed 11, T = 500 observations, M = 4 x N = 1000.
  - ``lz_proxy`` (T, 3): the posterior-mean proxy of bench.py:77-86
    (compute_reference: one high-particle run) - here an ensemble of 8
    filters x 16384 particles (J = 2^17 >= 1e5), master seed 987654321.
  - ``lz_mse`` (S,): per master seed s = 0..S-1, mean over (t, d) of
    (run_ensemble(...).mean_estimates - proxy)^2.
  - ``lz_est_mean`` / ``lz_est_m2`` (T, 3): mean over seeds of the ensemble
    estimate and of its square (bias^2 / variance decomposition against the
    proxy, metrics.bias_variance).
  - ``lz_var_s`` (S,): per seed, mean over (t, d) of (estimate - lz_est_mean)^2
    (its mean x S/(S-1) is the variance term of the MSE decomposition; its
    spread gives that term's standard error).
* cfg3 model (FH-N 30 x 50 lattice), truth seed 12, T = 10 observations,
  M = 4 x N = 64:
  - ``fhn_mse`` (S,): per master seed, mean over (t, node) of
    (mean_estimates[:, v-block] - truth v-block)^2.

The GPU tests (tests/test_gpu_stats.py) run the same calls through the
drop-in API with Philox draws and compare these statistics (two-sample
3-sigma rule + the north star's 5 % band).
"""

from __future__ import annotations

import argparse
import os
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from multiprocessing import get_context

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, HERE)
sys.path.insert(0, REPO)

import parpf  # noqa: E402  (reference, via PYTHONPATH)
import make_golden as mg  # noqa: E402  (reference-side config adapters)

from oracle import parpf_oracle as orc  # noqa: E402  (truth / observations only)

LZ_TRUTH_SEED, LZ_T, LZ_M, LZ_N = 11, 500, 4, 1000
LZ_PROXY_M, LZ_PROXY_N, LZ_PROXY_SEED = 8, 16384, 987654321
FHN_TRUTH_SEED, FHN_T, FHN_M, FHN_N = 12, 10, 4, 64


def lorenz_setup():
    truth0, states, obs = orc.lorenz_truth(seed=LZ_TRUTH_SEED, n_obs=LZ_T)
    model = mg.RefLorenzCfg(substeps=40, obs_var=2.0, prior_mean=tuple(truth0), prior_var=1.0)
    return model, states, obs


def fhn_setup():
    fm, states, obs = orc.fhn_truth(seed=FHN_TRUTH_SEED, n_obs=FHN_T)
    model = mg.RefFhnCfg(fm.rows, fm.cols, fm.substeps, fm.stim_row, fm.stim_col)
    return model, states, obs


def _lz_task(seed):
    model, _, obs = lorenz_setup()
    return seed, parpf.run_ensemble(model, obs, "bootstrap", LZ_M, LZ_N, seed).mean_estimates


def _fhn_task(seed):
    model, states, obs = fhn_setup()
    out = parpf.run_ensemble(model, obs, "bootstrap", FHN_M, FHN_N, seed)
    v = states[:, : model.nodes]
    return seed, float(((out.mean_estimates[:, : model.nodes] - v) ** 2).mean())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    ap.add_argument("--lz-seeds", type=int, default=4096)
    ap.add_argument("--fhn-seeds", type=int, default=128)
    ap.add_argument("--reuse-fhn", action="store_true")
    args = ap.parse_args()
    ctx = get_context("fork")
    out = {}
    t0 = time.time()
    model, _, obs = lorenz_setup()
    proxy = parpf.run_ensemble(model, obs, "bootstrap", LZ_PROXY_M, LZ_PROXY_N, LZ_PROXY_SEED,
                               workers=min(args.workers, LZ_PROXY_M)).mean_estimates
    out["lz_proxy"] = proxy
    print(f"proxy done {time.time() - t0:.0f}s", flush=True)
    S = args.lz_seeds
    ests = np.empty((S,) + proxy.shape)
    with ProcessPoolExecutor(args.workers, mp_context=ctx) as pool:
        for seed, est in pool.map(_lz_task, range(S), chunksize=4):
            ests[seed] = est
    mse = ((ests - proxy) ** 2).mean(axis=(1, 2))
    out["lz_mse"] = mse
    out["lz_est_mean"] = ests.mean(axis=0)
    out["lz_est_m2"] = (ests * ests).mean(axis=0)
    out["lz_var_s"] = ((ests - ests.mean(axis=0)) ** 2).mean(axis=(1, 2))
    print(f"lorenz {S} seeds done {time.time() - t0:.0f}s: mse {mse.mean():.5f} "
          f"cv {mse.std(ddof=1) / mse.mean():.3f}", flush=True)
    F = args.fhn_seeds
    fmse = np.empty(F)
    if args.reuse_fhn:  # keep the FH-N statistics of an existing fixture
        fmse = np.load(os.path.join(HERE, "stats.npz"))["fhn_mse"]
        F = fmse.shape[0]
    else:
        with ProcessPoolExecutor(args.workers, mp_context=ctx) as pool:
            for seed, m in pool.map(_fhn_task, range(F)):
                fmse[seed] = m
    out["fhn_mse"] = fmse
    print(f"fhn {F} seeds done {time.time() - t0:.0f}s: mse {fmse.mean():.6f} "
          f"cv {fmse.std(ddof=1) / fmse.mean():.3f}", flush=True)
    out["meta"] = np.array([LZ_TRUTH_SEED, LZ_T, LZ_M, LZ_N, LZ_PROXY_M, LZ_PROXY_N,
                            LZ_PROXY_SEED, FHN_TRUTH_SEED, FHN_T, FHN_M, FHN_N])
    np.savez_compressed(os.path.join(HERE, "stats.npz"), **out)


if __name__ == "__main__":
    main()
