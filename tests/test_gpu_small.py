"""GPU parity for the verification models (DiscreteHmm, LinearGaussianModel):
hooks and simulate() bit-exact against the reference, the bank in oracle
mode against the oracle / reference goldens, production-mode unbiasedness."""

import numpy as np
import pytest

from oracle import parpf_oracle as orc
from oracle import tapes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import models  # noqa: E402

HMM = dict(prior=[0.5, 0.5], transition=[[0.9, 0.1], [0.2, 0.8]],
           emission=[[0.8, 0.2], [0.3, 0.7]])
HOBS = np.array([[0.0], [1.0], [0.0], [0.0], [1.0]])
LG2 = dict(A=[[0.9, 0.1], [-0.2, 0.8]], trans_cov=[[1.0, 0.3], [0.3, 0.5]], H=[[1.0, 0.5]],
           obs_cov=[[0.7]], prior_mean=[0.5, -0.5], prior_cov=[[1.0, 0.2], [0.2, 2.0]])


def norm_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _single_tape(tr):
    return pf.DrawTape(prior=tr.prior_noise[None], noise=[s.noise[None] for s in tr.steps],
                       uniforms=[(s.u if s.u is not None else np.full(len(s.ancestors), np.nan))
                                 [None] for s in tr.steps])


def test_hooks_and_simulate_bit_exact(golden):
    g = golden["small"]
    h, oh = models.DiscreteHmm(**HMM), orc.DiscreteHmmModel(**HMM)
    x = h.sample_prior(np.random.default_rng(1), 64)
    assert np.array_equal(x, oh.sample_prior(np.random.default_rng(1), 64))
    assert np.array_equal(h.sample_transition(x, 1, np.random.default_rng(2)),
                          oh.sample_transition(x, 1, np.random.default_rng(2)))
    assert np.array_equal(h.log_likelihood([1.0], x, 1), oh.log_likelihood([1.0], x, 1))
    st, ob = pf.simulate.simulate(h, 30, 5)
    assert np.array_equal(st, g["h_sim_states"]) and np.array_equal(ob, g["h_sim_obs"])
    lg = models.LinearGaussianModel.scalar(a=0.9)
    st, ob = pf.simulate.simulate(lg, 10, 12)
    assert np.array_equal(st, g["l_sim_states"]) and np.array_equal(ob, g["l_obs"])
    ol = orc.LinearGaussianOracle.scalar(a=0.9)
    x = lg.sample_prior(np.random.default_rng(3), 50)
    assert np.array_equal(x, ol.sample_prior(np.random.default_rng(3), 50))
    assert np.array_equal(lg.transition_point_prediction(x, 1), ol.transition_point_prediction(x, 1))
    assert np.array_equal(lg.log_likelihood(np.array([0.3]), x, 1),
                          ol.log_likelihood(np.array([0.3]), x, 1))


def test_exact_oracles_match_reference(golden):
    g = golden["small"]
    ex = models.hmm_exact_filter(models.DiscreteHmm(**HMM), HOBS)
    assert np.array_equal(np.stack([e[0] for e in ex]), g["h_exact_filter"])
    assert np.array_equal(np.array([e[1] for e in ex]), g["h_exact_mass"])
    kf = models.kalman_filter(models.LinearGaussianModel.scalar(a=0.9), g["l_obs"])
    assert np.array_equal(np.stack([k[0] for k in kf]), g["l_kf_mean"])


def test_hmm_bank_oracle_mode(golden):
    g = golden["small"]
    om, gm = orc.DiscreteHmmModel(**HMM), models.DiscreteHmm(**HMM)
    M, N = 3, 20
    traces, mean, prior, noise, uni = tapes.ensemble_with_tape(om, HOBS, M, N, 44)
    assert np.array_equal(mean, g["he_mean"])
    bank = pf.FilterBank(gm, M, N, np.zeros((M, 2), np.uint32), len(HOBS),
                         tape=pf.DrawTape(prior, noise, uni))
    bank.load_observations(HOBS)
    bank.init()
    for k in range(len(HOBS)):
        bank.step(k)
        anc = bank.anc.cpu().numpy().reshape(M, N) - np.arange(M)[:, None] * N
        assert np.array_equal(anc, np.stack([tr.steps[k].ancestors for tr in traces]))
    torch.cuda.synchronize()
    assert norm_rel(bank.lnc_tr.cpu().numpy(), g["he_lnc"].T) < 1e-12
    out = pf.run_ensemble(gm, HOBS, "bootstrap", M, N, 44, tape=pf.DrawTape(prior, noise, uni))
    assert norm_rel(out.mean_estimates, g["he_mean"]) < 1e-12
    tr = orc.run_filter(om, HOBS, 50, np.random.SeedSequence(7102), keep_steps=True)
    out = pf.run_filter(gm, HOBS, "bootstrap", 50, 7102, tape=_single_tape(tr))
    assert norm_rel(out.estimates, g["h_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["h_lnc"]) < 1e-12


def test_lgm_bank_oracle_mode(golden):
    g = golden["small"]
    om, gm = orc.LinearGaussianOracle.scalar(a=0.9), models.LinearGaussianModel.scalar(a=0.9)
    tr = orc.run_filter(om, g["l_obs"], 64, np.random.SeedSequence(7103), keep_steps=True)
    out = pf.run_filter(gm, g["l_obs"], "bootstrap", 64, 7103, tape=_single_tape(tr))
    assert norm_rel(out.estimates, g["l_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["l_lnc"]) < 1e-12
    tr = orc.run_filter(om, g["l_obs"], 40, np.random.SeedSequence(71), keep_steps=True,
                        variant="auxiliary")
    tape = _single_tape(tr)
    tape.uniforms_first = [s.u_first[None] for s in tr.steps]
    out = pf.run_filter(gm, g["l_obs"], "auxiliary", 40, 71, tape=tape)
    assert norm_rel(out.estimates, g["la_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["la_lnc"]) < 1e-12
    om2, gm2 = orc.LinearGaussianOracle(**LG2), models.LinearGaussianModel(**LG2)
    tr = orc.run_filter(om2, g["l2_obs"], 32, np.random.SeedSequence(5), keep_steps=True)
    out = pf.run_filter(gm2, g["l2_obs"], "bootstrap", 32, 5, tape=_single_tape(tr))
    assert norm_rel(out.estimates, g["l2_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["l2_lnc"]) < 1e-12


def test_hmm_production_unbiased_normalising_constant():
    """E[exp(lnc_T)] equals the exact marginal likelihood (the reference's
    check_unbiasedness law) - 20,000 filters of 50 particles as ONE bank."""
    gm = models.DiscreteHmm(**HMM)
    mass = models.hmm_exact_filter(gm, HOBS)[-1][1]
    M, N = 20000, 50
    keys = pf.philox.filter_keys(123, M)
    bank = pf.FilterBank(gm, M, N, keys, len(HOBS))
    bank.load_observations(HOBS)
    bank.init()
    bank.run()
    torch.cuda.synchronize()
    gvals = np.exp(bank.lnc_tr[-1].cpu().numpy())
    z = abs(gvals.mean() - mass) / (gvals.std(ddof=1) / np.sqrt(M))
    assert z < 4.0, (gvals.mean(), mass, z)


def _island_tape(tr, n):
    M = len(tr.island_traces)
    prior = np.stack([it["prior"] for it in tr.island_traces])
    T = len(tr.island_traces[0]["steps"])
    noise = [np.stack([it["steps"][k].noise for it in tr.island_traces]) for k in range(T)]
    uni = [np.stack([(it["steps"][k].u if it["steps"][k].u is not None else np.full(n, np.nan))
                     for it in tr.island_traces]) for k in range(T)]
    return pf.DrawTape(prior=prior, noise=noise, uniforms=uni,
                       islands={t: u[None] for t, u, _ in tr.island_steps})


def test_double_bootstrap_oracle_mode(golden):
    from paper_1407_8071_b200 import islands

    g = golden["small"]
    om, gm = orc.DiscreteHmmModel(**HMM), models.DiscreteHmm(**HMM)
    tr = orc.run_double_bootstrap(om, HOBS, 3, 20, 2, np.random.SeedSequence(606),
                                  keep_steps=True)
    out = islands.run_double_bootstrap(gm, HOBS, 3, 20, 2, np.random.SeedSequence(606),
                                       tape=_island_tape(tr, 20))
    assert norm_rel(out.estimates, g["db_h_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["db_h_lnc"]) < 1e-12
    assert out.collapse_steps == g["db_h_coll"].tolist()
    assert out.n_particles == 60 and out.variant == "double-bf"
    gl = golden["lorenz"]
    om = orc.LorenzConfigModel(prior_mean=tuple(gl["truth0"]))
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(gl["truth0"]), prior_var=1.0)
    tr = orc.run_double_bootstrap(om, gl["obs"][:12], 4, 30, 5, np.random.SeedSequence(99),
                                  keep_steps=True)
    out = islands.run_double_bootstrap(gm, gl["obs"][:12], 4, 30, 5, np.random.SeedSequence(99),
                                       tape=_island_tape(tr, 30))
    assert norm_rel(out.estimates, gl["db_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, gl["db_lnc"]) < 1e-12


def test_double_bootstrap_production():
    """Philox islands: deterministic; on the HMM the pooled estimate of the
    final filter probability is unbiased within noise over replicates."""
    from paper_1407_8071_b200 import islands

    gm = models.DiscreteHmm(**HMM)
    a = islands.run_double_bootstrap(gm, HOBS, 8, 64, 2, 5)
    b = islands.run_double_bootstrap(gm, HOBS, 8, 64, 2, 5)
    assert np.array_equal(a.estimates, b.estimates)
    exact = models.hmm_exact_filter(gm, HOBS)[-1][0][1]
    ests = np.array([islands.run_double_bootstrap(gm, HOBS, 8, 64, 2, s).estimates[-1, 0]
                     for s in range(60)])
    z = abs(ests.mean() - exact) / (ests.std(ddof=1) / np.sqrt(len(ests)))
    assert z < 4.0


def test_hook_level_double_bootstrap_matches_reference(golden):
    """dbf_init / dbf_step driven like filters.py:274-313 with the caller's
    generators reproduce the reference's double bootstrap (HMM)."""
    g = golden["small"]
    gm = models.DiscreteHmm(**HMM)
    children = np.random.SeedSequence(606).spawn(4)
    rngs = [np.random.default_rng(c) for c in children[:3]]
    island_rng = np.random.default_rng(children[3])
    system = pf.dbf_init(gm, 3, 20, rngs)
    ests = []
    for k in range(len(HOBS)):
        system = pf.dbf_step(gm, system, HOBS[k], k + 1, 2, rngs, island_rng)
        ests.append(system.pooled_estimate())
    assert norm_rel(np.array(ests), g["db_h_est"]) < 1e-12
    assert abs(system.island_probs().sum() - 1.0) < 1e-12


@pytest.mark.parametrize("kind", ["hmm", "lorenz", "lorenz64", "fhnnet"])
def test_double_bootstrap_native_driver_matches_python_steps(kind):
    """The island step inside the native bank driver (pf_island_desc: island
    weights, island resampling every period, pooled estimate and trace, one
    call for the whole run) against the per-observation Python driver
    (IslandBank.step with the post-resample hook): identical estimates,
    traces, island log weights and collapse record."""
    from paper_1407_8071_b200 import islands

    dtype = "float32" if kind == "lorenz" else None
    if kind == "hmm":
        gm, obs, M, N, period = models.DiscreteHmm(**HMM), np.tile(HOBS, (4, 1)), 8, 64, 2
    elif kind == "fhnnet":  # rows carry the history-bit means after the state means
        gm = pf.FhnNetworkModel(J=8, n_zones=2, zone_width=2, stim_prob=0.05)
        obs = pf.simulate.simulate(gm, 12, 4)[1]
        M, N, period = 5, 128, 3
    else:
        from paper_1407_8071_b200.simulate import lorenz_truth

        truth0, _, obs = lorenz_truth(3, 12)
        gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                              prior_mean=truth0, prior_var=1.0)
        M, N, period = 6, 4096, 5
    T = obs.shape[0]
    runs = []
    for native in (True, False):
        ib = islands.IslandBank(gm, M, N, period, 17, T, dtype=dtype)
        if native:
            ib.run(obs)
        else:
            ib.start(obs)
            for k in range(T):
                ib.step(k)
            torch.cuda.synchronize()
        runs.append((ib.est.cpu().numpy(), ib.trace.cpu().numpy(), ib.lw.cpu().numpy(),
                     ib.collapse_steps(), ib.bank.anc.cpu().numpy()))
    for a, b in zip(*runs):
        if isinstance(a, list):
            assert a == b
        else:
            assert np.array_equal(a, b)


@pytest.mark.parametrize("M,period", [(1, 1), (4, 1), (4, 50), (3, 4)])
def test_double_bootstrap_native_island_edge_cases(M, period):
    """Native island step at the edges: one island, resampling every step,
    never (period beyond the horizon), and a period that does not divide T:
    identical to the Python step driver."""
    from paper_1407_8071_b200 import islands

    gm, obs = models.DiscreteHmm(**HMM), np.tile(HOBS, (3, 1))
    T = obs.shape[0]
    runs = []
    for native in (True, False):
        ib = islands.IslandBank(gm, M, 32, period, 23, T)
        if native:
            ib.run(obs)
        else:
            ib.start(obs)
            for k in range(T):
                ib.step(k)
            torch.cuda.synchronize()
        runs.append((ib.est.cpu().numpy(), ib.trace.cpu().numpy(), ib.lw.cpu().numpy(),
                     ib.collapse_steps(), list(ib.island_steps)))
    for a, b in zip(*runs):
        if isinstance(a, list):
            assert a == b
        else:
            assert np.array_equal(a, b)
