"""Auxiliary particle filter (filters.py:115-154) on the GPU bank, against the
oracle and the golden fixtures generated from the reference."""

import numpy as np
import pytest

from oracle import parpf_oracle as orc
from oracle import tapes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8071_b200 as pf  # noqa: E402


def norm_rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _lorenz(truth0):
    om = orc.LorenzConfigModel(prior_mean=tuple(truth0))
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    return om, gm


def _run_apf_bank(gm, obs, M, N, prior, noise, uni, uni1, dtype=None):
    tape = pf.DrawTape(prior=prior, noise=noise, uniforms=uni, uniforms_first=uni1)
    bank = pf.FilterBank(gm, M, N, np.zeros((M, 2), np.uint32), len(obs), tape=tape,
                         dtype=dtype, variant="auxiliary")
    bank.load_observations(obs)
    bank.init()
    a1, a2 = [], []
    off = np.arange(M)[:, None] * N
    for k in range(len(obs)):
        bank.step(k)
        a1.append(bank.anc1.cpu().numpy().reshape(M, N) - off)
        a2.append(bank.anc.cpu().numpy().reshape(M, N) - off)
    torch.cuda.synchronize()
    bank.check_status()
    return bank, a1, a2


def test_lorenz_apf_bank_oracle_mode_bit_exact(golden):
    g = golden["lorenz"]
    om, gm = _lorenz(g["truth0"])
    obs = g["obs"][:12]
    traces, mean, prior, noise, uni, uni1 = tapes.ensemble_with_tape(om, obs, 3, 64, 8,
                                                                     variant="auxiliary")
    assert np.array_equal(mean, g["ae_mean"])  # oracle == reference fixture
    bank, a1, a2 = _run_apf_bank(gm, obs, 3, 64, prior, noise, uni, uni1)
    for k in range(len(obs)):
        assert np.array_equal(a1[k], np.stack([tr.steps[k].anc_first for tr in traces])), k
        assert np.array_equal(a2[k], np.stack([tr.steps[k].ancestors for tr in traces])), k
    assert norm_rel(bank.est.cpu().numpy(), np.stack([t.estimates for t in traces], 1)) < 1e-12
    assert norm_rel(bank.lnc_tr.cpu().numpy(), g["ae_lnc"].T) < 1e-12


def test_lorenz_apf_run_filter_matches_golden(golden):
    g = golden["lorenz"]
    om, gm = _lorenz(g["truth0"])
    obs = g["obs"][:12]
    rec = orc.TapeRecorder(np.random.SeedSequence(4242))
    tr = orc.run_filter(om, obs, 48, rec, keep_steps=True, variant="auxiliary")
    tape = pf.DrawTape(tr.prior_noise[None], [s.noise[None] for s in tr.steps],
                       [s.u[None] for s in tr.steps], [s.u_first[None] for s in tr.steps])
    out = pf.run_filter(gm, obs, "auxiliary", 48, 4242, tape=tape)
    assert out.variant == "auxiliary"
    assert norm_rel(out.estimates, g["a_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["a_lnc"]) < 1e-12


def test_lorenz_apf_collapse_semantics(golden):
    g = golden["lorenz"]
    om, gm = _lorenz(g["truth0"])
    rec = orc.TapeRecorder(12)
    tr = orc.run_filter(om, g["c_obs"], 16, rec, keep_steps=True, variant="auxiliary")
    assert tr.collapse_steps == list(g["ac_steps"])
    nan = np.full(16, np.nan)
    tape = pf.DrawTape(tr.prior_noise[None], [s.noise[None] for s in tr.steps],
                       [(s.u if s.u is not None else nan)[None] for s in tr.steps],
                       [s.u_first[None] for s in tr.steps])
    out = pf.run_filter(gm, g["c_obs"], "auxiliary", 16, 12, tape=tape)
    assert out.collapse_steps == list(g["ac_steps"])
    assert norm_rel(out.estimates, g["ac_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["ac_lnc"]) < 1e-12


def test_fhn_apf_bank_oracle_mode(golden):
    g = golden["fhn"]
    om = orc.FhnConfigModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    gm = pf.FhnLatticeModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    rec = orc.TapeRecorder(np.random.SeedSequence(5151))
    tr = orc.run_filter(om, g["obs"], 6, rec, keep_steps=True, variant="auxiliary")
    assert np.array_equal(np.stack([s.anc_first for s in tr.steps]), g["a_anc1"])
    tape = pf.DrawTape(None, [s.noise.reshape(om.substeps, 2, 6, -1)[None] for s in tr.steps],
                       [s.u[None] for s in tr.steps], [s.u_first[None] for s in tr.steps])
    bank, a1, a2 = _run_apf_bank(gm, g["obs"], 1, 6, None, tape.noise, tape.uniforms,
                                 tape.uniforms_first)
    assert np.array_equal(np.stack([a[0] for a in a1]), g["a_anc1"])
    assert np.array_equal(np.stack([a[0] for a in a2]), g["a_anc2"])
    assert norm_rel(bank.est.cpu().numpy()[:, 0, : om.nodes], g["a_est_v"]) < 1e-12
    assert norm_rel(bank.lnc_tr.cpu().numpy()[:, 0], g["a_lnc"]) < 1e-12


def test_apf_production_mode_tracks_truth_and_is_deterministic():
    truth0, states, obs = orc.lorenz_truth(seed=9, n_obs=30)
    _, gm = _lorenz(truth0)
    a = pf.run_ensemble(gm, obs, "auxiliary", 4, 1000, 2)
    b = pf.run_ensemble(gm, obs, "auxiliary", 4, 1000, 2)
    boot = pf.run_ensemble(gm, obs, "bootstrap", 4, 1000, 2)
    assert a.same_result(b)
    mse_a = np.mean((a.mean_estimates - states) ** 2)
    mse_b = np.mean((boot.mean_estimates - states) ** 2)
    print(f"APF mse {mse_a:.4f} bootstrap mse {mse_b:.4f}")
    assert mse_a < 2.0 and mse_a < 2.0 * mse_b


def test_apf_fhn_production_fp32_runs():
    m, states, obs = orc.fhn_truth(seed=3, n_obs=3)
    gm = pf.FhnLatticeModel(stim_row=m.stim_row, stim_col=m.stim_col)
    out = pf.run_ensemble(gm, obs, "auxiliary", 2, 256, 1, dtype="float32",
                          estimate="projection")
    err = np.sqrt(((out.mean_estimates - states[:, : m.nodes]) ** 2).mean())
    assert np.isfinite(err) and err < 0.1


def test_apf_hook_level_step_matches_oracle(golden):
    """pf.apf_step over host containers consumes the Generator like the
    reference and reproduces the oracle step."""
    g = golden["lorenz"]
    om, gm = _lorenz(g["truth0"])
    st = pf.bf_init(gm, 32, np.random.default_rng(3))
    st1 = pf.apf_step(gm, st, g["obs"][0], np.random.default_rng(4))
    x0 = orc.LorenzConfigModel(prior_mean=tuple(g["truth0"]))
    ox = x0.sample_prior(np.random.default_rng(3), 32)
    steps = []
    x1, lnc1, _ = orc._apf_step(om, ox, 0.0, g["obs"][0], 1, np.random.default_rng(4), True,
                                steps)
    assert norm_rel(st1.particles, x1) < 1e-12
    assert abs(st1.log_norm_const - lnc1) < 1e-12


@pytest.mark.parametrize("kind", ["lorenz", "fhnnet"])
def test_native_apf_driver_matches_stepwise(kind):
    """pf_bank_run's auxiliary variant (the whole apf_step sequence in C++)
    equals the per-step Python path: states, lnc, collapse flags identical,
    estimates to fp64 rounding (the planar estimate is fused natively)."""
    if kind == "lorenz":
        truth0, _, obs = orc.lorenz_truth(seed=21, n_obs=6)
        gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                              prior_mean=tuple(truth0), prior_var=1.0)
        dtypes = (torch.float64, torch.float32)
    else:
        gm = pf.FhnNetworkModel(J=8, n_zones=2, zone_width=2, stim_prob=0.05)
        _, obs = pf.simulate.simulate(gm, 6, 3)
        dtypes = (torch.float32,)
    keys = pf.philox.filter_keys(9, 3)
    for dtype in dtypes:
        res = []
        for native in (True, False):
            bank = pf.FilterBank(gm, 3, 256, keys, len(obs), dtype=dtype, variant="auxiliary")
            bank.load_observations(obs)
            bank.init()
            if not native:
                bank.kernel_events = (torch.cuda.Event(), torch.cuda.Event())
            bank.run()
            torch.cuda.synchronize()
            res.append((bank.est.cpu().numpy(), bank.lnc_tr.cpu().numpy(),
                        bank.coll_tr.cpu().numpy(), bank.particles()))
        a, b = res
        assert np.linalg.norm(a[0] - b[0]) <= 1e-13 * np.linalg.norm(b[0])
        assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
        assert np.array_equal(a[3], b[3])


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_first_stage_nan_is_not_a_collapse(dtype):
    """core.py:127-133: np.max of first-stage log weights containing NaN is
    NaN, so the reference raises ValueError - also when every other value is
    -inf.  pf_apf_first_stage_prepare must leave such a filter's lambda
    untouched (no uniform fallback) so the first-stage resampler flags it."""
    from paper_1407_8071_b200 import _lib

    M, N = 4, 64
    lam = np.zeros((M, N))
    lam[0] = -np.inf                      # a genuine collapse -> lambda := 0, flagged
    lam[1] = np.nan                       # all NaN
    lam[2] = -np.inf
    lam[2, 7] = np.nan                    # NaN among -inf
    lam[3] = np.random.default_rng(0).normal(size=N)
    d = torch.from_numpy(lam.reshape(-1)).to(dtype).cuda()
    coll1 = torch.zeros(M, dtype=torch.uint8, device="cuda")
    code = _lib.PF_F64 if dtype == torch.float64 else _lib.PF_F32
    _lib.call("pf_apf_first_stage_prepare", code, _lib.ptr(d), M, N, _lib.ptr(coll1),
              _lib.stream_ptr())
    out = d.cpu().numpy().reshape(M, N).astype(np.float64)
    assert coll1.cpu().numpy().tolist() == [1, 0, 0, 0]
    assert np.all(out[0] == 0.0)
    assert np.all(np.isnan(out[1])) and np.isnan(out[2, 7]) and np.isneginf(out[2, 0])
    assert np.array_equal(out[3], lam[3].astype(np.float32 if dtype == torch.float32
                                                else np.float64))
    # the resampler then reports the NaN (-> ValueError on the host)
    anc = torch.empty(M * N, dtype=torch.int32, device="cuda")
    lnc = torch.zeros(M, dtype=torch.float64, device="cuda")
    coll = torch.zeros(M, dtype=torch.uint8, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    keys = torch.from_numpy(pf.philox.filter_keys(1, M).view(np.int32)).cuda()
    _lib.call("pf_segmented_resample_ex", code, _lib.ptr(d), M, N, None, _lib.ptr(keys), 1,
              _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll), _lib.ptr(st), None, 0, None, None,
              0, 0, _lib.stream_ptr())
    status = st.cpu().numpy()
    assert (status[1] & _lib.PF_ST_NAN_WEIGHT) and (status[2] & _lib.PF_ST_NAN_WEIGHT)
    assert not (status[0] & _lib.PF_ST_NAN_WEIGHT) and not (status[3] & _lib.PF_ST_NAN_WEIGHT)
    with pytest.raises(ValueError):
        _lib.raise_status(status)


@pytest.mark.parametrize("kind", ["lorenz", "fhn"])
def test_hook_level_bf_step_matches_oracle(kind):
    """pf.bf_init / pf.bf_step (filters.py:87-112 drop-ins) driven by a numpy
    Generator consume the draws in the reference's order and reproduce the
    oracle's bootstrap step: particles and lnc within 1e-12 (fp64), same
    collapse decisions."""
    if kind == "lorenz":
        truth0, _, obs = orc.lorenz_truth(seed=9, n_obs=4)
        om, gm = _lorenz(truth0)
        n = 64
    else:
        om, _, obs = orc.fhn_truth(seed=4, n_obs=2)
        gm = pf.FhnLatticeModel(stim_row=om.stim_row, stim_col=om.stim_col)
        n = 6
    rng_g, rng_o = np.random.default_rng(17), np.random.default_rng(17)
    st = pf.bf_init(gm, n, rng_g)
    x, _ = orc._prior(om, rng_o, n)
    assert norm_rel(st.particles, x) < 1e-12
    lnc = 0.0
    for k in range(len(obs)):
        st = pf.bf_step(gm, st, obs[k], rng_g)
        x, lnc, coll = orc._bf_step(om, x, lnc, obs[k], k + 1, rng_o)
        assert norm_rel(st.particles, x) < 1e-12, f"step {k + 1}"
        assert abs(st.log_norm_const - lnc) <= 1e-12 * max(1.0, abs(lnc))
        assert bool(st.collapsed) == bool(coll)
    # both generators consumed exactly the same draws
    assert rng_g.standard_normal() == rng_o.standard_normal()
