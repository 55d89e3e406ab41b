"""Production (Philox) mode statistical parity with the reference algorithm.

North star: over >= 64 seeds the GPU bank's MSE must reproduce the CPU
reference's (within 5 % / 3 sigma; the reference side is precomputed with
the unmodified reference by tests/golden/make_stats.py), and the ensemble
estimator must show the paper's
decomposition: variance ~ 1/(M N) and bias ~ 1/N (Corollary 2,
PAPER.md:568-586).  The checks mirror parpf/verify.py:160-260
(check_ensemble_variance_rate, check_bias_rate) with the Lorenz-63 cfg0
model; independent replicates are simply more filters in one GPU bank.
"""

import numpy as np
import pytest

from oracle import parpf_oracle as orc

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import replicates  # noqa: E402


def _cfg0(n_obs, seed=11):
    truth0, states, obs = orc.lorenz_truth(seed=seed, n_obs=n_obs)
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    om = orc.LorenzConfigModel(prior_mean=tuple(truth0))
    return gm, om, states, obs


def _bank_estimates(model, obs, n_filters, n_particles, master, dtype=torch.float64):
    keys = pf.philox.filter_keys(master, n_filters)
    bank = pf.FilterBank(model, n_filters, n_particles, keys, len(obs), dtype=dtype)
    bank.load_observations(obs)
    bank.init()
    bank.run()
    torch.cuda.synchronize()
    bank.check_status()
    return bank.est.cpu().numpy()  # (T, M, 3)


def loglog_slope(x, y):
    """metrics.loglog_slope (parpf/metrics.py:70-79): least-squares slope."""
    return float(np.polyfit(np.log(x), np.log(y), 1)[0])


def _stats():
    import os

    return np.load(os.path.join(os.path.dirname(__file__), "golden", "stats.npz"))


def _two_sample(a, b):
    """(difference of means, its standard error) of two independent samples."""
    return a.mean() - b.mean(), np.sqrt(a.var(ddof=1) / a.size + b.var(ddof=1) / b.size)


def test_cfg0_mse_vs_high_particle_proxy_matches_reference():
    """cfg0 (Lorenz-63, M=4 x N=1000, T=500, fp64) in
    production (Philox) mode, scored against a J = 2^17 posterior-mean proxy
    (bench.py:77-86 compute_reference) and compared seed-for-seed in
    distribution with the UNMODIFIED reference: 1024 reference seeds
    (tests/golden/stats.npz, make_stats.py: 4096 seeds) vs 4096 GPU seeds,
    each one run_ensemble(model, obs, 'bootstrap', 4, 1000, seed) (replicates
    batched as one bank, replicates.ensemble_replicates).  Per-seed MSE has
    CV ~0.97, so at 4096 + 4096 seeds one standard error of the difference
    is ~1.7 % of the MSE: the north star's 5 % band and the two-sample
    3-sigma rule are both asserted; the variance and bias^2 terms of the
    decomposition are compared too."""
    st = _stats()
    truth_seed, T, M, N = (int(v) for v in st["meta"][:4])
    proxy = st["lz_proxy"]
    truth0, _, obs = orc.lorenz_truth(seed=truth_seed, n_obs=T)
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    S = 4096
    batch = replicates.ensemble_replicates(gm, obs, "bootstrap", M, N,
                                              [100_000 + s for s in range(S)],
                                              dtype="float64")
    assert not batch.diverged.any()
    est = batch.estimates  # (S, T, 3)
    mse_g = ((est - proxy) ** 2).mean(axis=(1, 2))
    mse_c = st["lz_mse"]
    d, se = _two_sample(mse_g, mse_c)
    rel = d / mse_c.mean()
    print(f"cfg0 MSE vs proxy: gpu {mse_g.mean():.6f} ({S} seeds) reference "
          f"{mse_c.mean():.6f} ({mse_c.size} seeds) diff {100 * rel:+.2f}% "
          f"({d / se:+.2f} sigma); within 5%: {abs(rel) <= 0.05}")
    assert abs(d) <= 3.0 * se
    assert abs(rel) <= 0.05
    # decomposition: variance term (per-seed spread about the seed mean) ...
    em_g = est.mean(axis=0)
    var_g = ((est - em_g) ** 2).mean(axis=(1, 2))
    dv, sev = _two_sample(var_g, st["lz_var_s"])
    print(f"variance term gpu {var_g.mean():.6f} ref {st['lz_var_s'].mean():.6f} "
          f"({dv / sev:+.2f} sigma)")
    assert abs(dv) <= 3.0 * sev
    # ... and the bias term: the seed-mean estimates agree cell by cell
    # within their standard errors (mean z^2 ~ 1), and bias^2 against the
    # proxy matches
    em_c = st["lz_est_mean"]
    vc = (st["lz_est_m2"] - em_c ** 2) * mse_c.size / (mse_c.size - 1)
    vg = est.var(axis=0, ddof=1)
    z2 = (em_g - em_c) ** 2 / (vg / S + vc / mse_c.size)
    b2_g, b2_c = ((em_g - proxy) ** 2).mean(), ((em_c - proxy) ** 2).mean()
    print(f"bias^2 gpu {b2_g:.6f} ref {b2_c:.6f}; mean z^2 of seed means {z2.mean():.3f}")
    assert z2.mean() < 2.0
    assert abs(b2_g - b2_c) <= 0.25 * b2_c + 3 * (vg.mean() / S + vc.mean() / mse_c.size)


def test_fhn_lattice_production_mse_matches_reference_over_seeds():
    """cfg3 model (FH-N 30x50 lattice) in production mode, fp32 (the bench
    kernel): MSE of the M-averaged v estimate against the truth, 256 GPU
    seeds vs 128 seeds of the UNMODIFIED reference (fp64, numpy twin;
    tests/golden/stats.npz).  North star: within 5 %, and within 3 sigma."""
    st = _stats()
    truth_seed, T, M, N = (int(v) for v in st["meta"][7:11])
    m, states, obs = orc.fhn_truth(seed=truth_seed, n_obs=T)
    gm = pf.FhnLatticeModel(stim_row=m.stim_row, stim_col=m.stim_col)
    S = 256
    batch = replicates.ensemble_replicates(gm, obs, "bootstrap", M, N,
                                              [200_000 + s for s in range(S)],
                                              dtype="float32", estimate="projection")
    assert not batch.diverged.any()
    v_true = states[:, : m.nodes]
    mse_g = ((batch.estimates - v_true) ** 2).mean(axis=(1, 2))
    mse_c = st["fhn_mse"]
    d, se = _two_sample(mse_g, mse_c)
    rel = d / mse_c.mean()
    print(f"FH-N MSE gpu(fp32) {mse_g.mean():.6e} ref(fp64) {mse_c.mean():.6e} "
          f"diff {100 * rel:+.2f}% ({d / se:+.2f} sigma)")
    assert abs(rel) <= 0.05
    assert abs(d) <= 3.0 * se


def test_ensemble_variance_decays_like_one_over_M():
    """verify.check_ensemble_variance_rate analogue: slope in [-1.25, -0.75]."""
    gm, _, _, obs = _cfg0(n_obs=10, seed=3)
    reps, N = 500, 64
    variances = []
    Ms = (1, 2, 4, 8, 16)
    for i, M in enumerate(Ms):
        est = _bank_estimates(gm, obs, reps * M, N, 900 + i)
        ens = est[-1].reshape(reps, M, 3).mean(axis=1)[:, 0]
        variances.append(ens.var(ddof=1))
    slope = loglog_slope(np.array(Ms, float), np.array(variances))
    print("variance slope", slope, variances)
    assert -1.25 <= slope <= -0.75


def test_total_particle_variance_decays_like_one_over_MN():
    """Variance depends on the total budget M*N (Corollary 2 first term)."""
    gm, _, _, obs = _cfg0(n_obs=10, seed=4)
    reps = 400
    budget = []
    variances = []
    for i, (M, N) in enumerate(((2, 64), (4, 128), (8, 256), (16, 512))):
        est = _bank_estimates(gm, obs, reps * M, N, 700 + i)
        ens = est[-1].reshape(reps, M, 3).mean(axis=1)[:, 0]
        budget.append(M * N)
        variances.append(ens.var(ddof=1))
    slope = loglog_slope(np.array(budget, float), np.array(variances))
    print("MN slope", slope, variances)
    assert -1.25 <= slope <= -0.75


def test_bias_decays_like_one_over_N():
    """verify.check_bias_rate analogue on one observation of a sharply
    observed Lorenz state; |bias| slope in [-1.35, -0.65].  With no exact
    posterior for Lorenz-63, the bias is read from differences of the mean
    estimate at N and 2N (E[est_N] - E[est_2N] = c/(2N) + O(1/N^2)), which
    needs no proxy; a 16 x 2^20-particle proxy cross-checks the sign."""
    truth0, _, obs = orc.lorenz_truth(seed=21, n_obs=1)
    gm = pf.Lorenz63Model(substeps=40, obs_var=0.05, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=4.0)
    reps = 200_000
    Ns = (8, 16, 32, 64, 128, 256)
    means, ses = [], []
    for i, N in enumerate(Ns):
        est = _bank_estimates(gm, obs, reps, N, 300 + i)[-1, :, 0]
        means.append(est.mean())
        ses.append(est.std(ddof=1) / np.sqrt(reps))
    diffs = np.abs(np.diff(means))
    slope = loglog_slope(np.array(Ns[:-1], float), diffs)
    proxy = _bank_estimates(gm, obs, 16, 1 << 20, 1)[-1, :, 0].mean()
    print("bias slope", slope, diffs, ses, "proxy", proxy, "means", means)
    assert diffs[0] > 5 * np.hypot(ses[0], ses[1])
    assert np.sign(means[0] - proxy) == np.sign(means[1] - proxy)
    assert -1.35 <= slope <= -0.65


def test_lorenz_fp32_production_matches_fp64_statistically():
    """The fp32 production kernel (2 particles/thread, MUFU Box-Muller) gives
    the same filtering accuracy as the fp64 path over many filters."""
    gm, _, states, obs = _cfg0(n_obs=20, seed=8)
    M, N = 256, 1000
    e32 = _bank_estimates(gm, obs, M, N, 31, dtype=torch.float32)
    e64 = _bank_estimates(gm, obs, M, N, 32, dtype=torch.float64)
    m32 = ((e32 - states[:, None, :]) ** 2).mean(axis=(0, 2))
    m64 = ((e64 - states[:, None, :]) ** 2).mean(axis=(0, 2))
    d = m32.mean() - m64.mean()
    se = np.sqrt(m32.var(ddof=1) / M + m64.var(ddof=1) / M)
    print(f"fp32 mse {m32.mean():.5f} fp64 mse {m64.mean():.5f} diff {d:+.5f} se {se:.5f}")
    assert abs(d) <= 3.5 * se + 1e-12
