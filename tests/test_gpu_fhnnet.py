"""GPU parity for the paper's forced FH-N network (models/fhn.py:85-207,
SURVEY §8f #3): hooks and simulate() bit-exact against the reference's own
output, the bank in oracle mode against the oracle (ancestors bit-exact,
fp64 states / estimates / lnc within 1e-12 norm-relative), fp32 within 1e-4,
and production (Philox) tracking statistics."""

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
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def models8(golden, **kw):
    sp = float(golden["fhnnet"]["m8_stim_prob"])
    args = {**dict(J=8, n_zones=2, zone_width=2, stim_prob=sp), **kw}
    return orc.FhnNetworkModel(**args), pf.FhnNetworkModel(**args)


# ---------------------------------------------------------------- hooks

def test_hooks_bit_exact(golden):
    g = golden["fhnnet"]
    _, gm = models8(golden)
    np.testing.assert_array_equal(gm.transition_point_prediction(g["hook_x"], 1), g["tpp_t1"])
    np.testing.assert_array_equal(gm.transition_point_prediction(g["hook_x"], 250),
                                  g["tpp_t250"])
    _, gf = models8(golden)
    gf.stim_prob = 1.0
    out = gf.sample_transition(g["band_x"], 7, np.random.default_rng(19))
    np.testing.assert_array_equal(out, g["band_out"])
    np.testing.assert_array_equal(gm.log_likelihood(g["ll_y"], g["hook_x"], 1), g["ll_out"])
    with pytest.raises(ValueError):
        gm.log_likelihood(np.zeros(gm.dim_y - 1), g["hook_x"], 1)


def test_simulate_bit_exact(golden):
    g = golden["fhnnet"]
    _, gm = models8(golden)
    st, ob = pf.simulate.simulate(gm, 120, 3)
    np.testing.assert_array_equal(st, g["sim8_states"])
    np.testing.assert_array_equal(ob, g["sim8_obs"])
    st, ob = pf.models.simulate(pf.FhnNetworkModel(J=16, stim_prob=0.02), 150, 3)
    np.testing.assert_array_equal(st, g["sim16_states"])
    np.testing.assert_array_equal(ob, g["sim16_obs"])


@pytest.mark.parametrize("J,zones", [(5, 1), (1, 1), (3, 1)])
def test_odd_lattices_match_oracle(J, zones):
    """Odd node counts take the scalar (G = 1) kernel path."""
    kw = dict(J=J, n_zones=zones, zone_width=1, stim_prob=0.7)
    om, gm = orc.FhnNetworkModel(**kw), pf.FhnNetworkModel(**kw)
    rng = np.random.default_rng(J)
    x = np.zeros((9, gm.dim_x))
    x[:, : gm.nodes] = rng.uniform(-1.9, -1.5, size=(9, gm.nodes))
    x[:, gm.nodes: 2 * gm.nodes] = rng.normal(size=(9, gm.nodes))
    x[:, 2 * gm.nodes:] = rng.random((9, gm.stim_hold * gm.nodes)) < 0.1
    for t in (1, 300):
        np.testing.assert_array_equal(gm.sample_transition(x, t, np.random.default_rng(t)),
                                      om.sample_transition(x, t, np.random.default_rng(t)))
        np.testing.assert_array_equal(gm.transition_point_prediction(x, t),
                                      om.transition_point_prediction(x, t))


def test_history_validation_and_divergence():
    gm = pf.FhnNetworkModel(J=4, n_zones=2, zone_width=2)
    x = np.zeros((1, gm.dim_x))
    x[0, -1] = 0.5
    with pytest.raises(ValueError):
        gm.transition_point_prediction(x, 1)
    with pytest.raises(ValueError):
        pf.FhnNetworkModel(stim_hold=33)
    # the literal (positive-leading) cubic escapes under forcing
    # (reference tests/test_models_fhn.py::test_literal_cubic_diverges_under_forcing)
    lit = pf.FhnNetworkModel(J=8, cubic=(1.0, 0.0, -3.6, 0.0), n_zones=2, zone_width=2)
    with pytest.raises(pf.NumericalDivergenceError):
        pf.simulate.simulate(lit, 150, 5)


# ---------------------------------------------------------------- bank, oracle mode

def _tape(traces, noise, uni, uni1=None):
    return pf.DrawTape(prior=None, noise=noise, uniforms=uni, stim=tapes.stim_tape(traces),
                       uniforms_first=uni1 or [])


def test_bank_oracle_mode_fp64(golden):
    g = golden["fhnnet"]
    om, gm = models8(golden)
    obs = g["sim8_obs"][:40]
    M, N = 3, 16
    traces, mean, _, noise, uni = tapes.ensemble_with_tape(om, obs, M, N, 21)
    assert np.array_equal(mean, g["e_mean"])  # oracle == reference fixture
    bank = pf.FilterBank(gm, M, N, np.zeros((M, 2), np.uint32), len(obs),
                         tape=_tape(traces, noise, uni))
    bank.load_observations(obs)
    bank.init()
    for k in range(len(obs)):
        bank.step(k)
        anc = bank.anc.cpu().numpy().reshape(M, N) - np.arange(M)[:, None] * N
        want = np.stack([tr.steps[k].ancestors for tr in traces])
        assert np.array_equal(anc, want), f"step {k + 1}"
    torch.cuda.synchronize()
    bank.check_status()
    lw_want = np.concatenate([tr.steps[-1].log_w for tr in traces])
    assert norm_rel(bank.logw.cpu().numpy(), lw_want) < 1e-12
    est = bank.est.cpu().numpy()
    assert norm_rel(est, np.stack([tr.estimates for tr in traces], axis=1)) < 1e-12
    assert norm_rel(bank.lnc_tr.cpu().numpy(), g["e_lnc"].T) < 1e-12
    # final particle set, history bits included
    final = np.stack([tr.steps[-1].propagated[tr.steps[-1].ancestors] for tr in traces])
    assert norm_rel(bank.particles(), final) < 1e-12
    assert np.array_equal(bank.particles()[..., 2 * gm.nodes:], final[..., 2 * gm.nodes:])


def test_run_filter_and_ensemble_match_golden(golden):
    g = golden["fhnnet"]
    om, gm = models8(golden)
    obs = g["sim8_obs"][:60]
    tr = orc.run_filter(om, obs, 32, np.random.SeedSequence(808), keep_steps=True)
    noise = [s.noise[2].reshape(1, 32, -1) for s in tr.steps]
    uni = [s.u[None] for s in tr.steps]
    out = pf.run_filter(gm, obs, "bootstrap", 32, 808, tape=_tape([tr], noise, uni))
    assert norm_rel(out.estimates, g["f_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["f_lnc"]) < 1e-12
    traces, _, _, noise, uni = tapes.ensemble_with_tape(om, obs[:40], 3, 16, 21)
    ens = pf.run_ensemble(gm, obs[:40], "bootstrap", 3, 16, 21, tape=_tape(traces, noise, uni))
    assert norm_rel(ens.mean_estimates, g["e_mean"]) < 1e-12
    proj = pf.run_ensemble(gm, obs[:40], "bootstrap", 3, 16, 21, tape=_tape(traces, noise, uni),
                           estimate="projection")
    assert norm_rel(proj.mean_estimates, g["e_mean"][:, : gm.nodes]) < 1e-12


def test_auxiliary_filter_matches_golden(golden):
    """The paper's FH-N experiment runs the auxiliary filter
    (verify.py:356-414): both resampling stages bit-exact."""
    g = golden["fhnnet"]
    om, gm = models8(golden)
    obs = g["sim8_obs"][:40]
    tr = orc.run_filter(om, obs, 24, np.random.SeedSequence(909), keep_steps=True,
                        variant="auxiliary")
    assert np.array_equal(tr.estimates, g["a_est"])
    noise = [s.noise[2].reshape(1, 24, -1) for s in tr.steps]
    uni = [(s.u if s.u is not None else np.full(24, np.nan))[None] for s in tr.steps]
    uni1 = [s.u_first[None] for s in tr.steps]
    bank = pf.FilterBank(gm, 1, 24, np.zeros((1, 2), np.uint32), len(obs),
                         tape=_tape([tr], noise, uni, uni1), variant="auxiliary")
    bank.load_observations(obs)
    bank.init()
    for k in range(len(obs)):
        bank.step(k)
        assert np.array_equal(bank.anc1.cpu().numpy(), g["a_anc1"][k]), f"stage 1, step {k + 1}"
        assert np.array_equal(bank.anc.cpu().numpy(), g["a_anc2"][k]), f"stage 2, step {k + 1}"
    torch.cuda.synchronize()
    assert norm_rel(bank.est[:, 0].cpu().numpy(), g["a_est"]) < 1e-12
    assert norm_rel(bank.lnc_tr[:, 0].cpu().numpy(), g["a_lnc"]) < 1e-12


def test_one_step_fp32_within_1e4(golden):
    g = golden["fhnnet"]
    om, gm = models8(golden, stim_prob=0.5)
    obs = g["sim8_obs"][80:81]  # mid-record: waves and stimuli present
    st = g["sim8_states"][80]
    M, N = 2, 16
    x0 = np.tile(st, (M * N, 1))
    traces = []
    for f in range(M):
        rng = np.random.default_rng(f)
        nz = om.draw_noise(rng, N)
        prop = om.propagate(x0[:N], nz, 81)
        traces.append((nz, prop, om.log_likelihood(obs[0], prop, 81)))
    stim = torch.from_numpy(np.stack([np.stack([t[0][0], t[0][1]]) for t in traces])).cuda()
    z = torch.from_numpy(np.stack([t[0][2].reshape(N, -1) for t in traces])).cuda()
    x, q = gm.to_device(x0, dtype=torch.float32)
    xo, qo = torch.empty_like(x), torch.empty_like(q)
    lw = torch.empty(M * N, dtype=torch.float32, device="cuda")
    st_ = torch.zeros(M, dtype=torch.int32, device="cuda")
    y = torch.from_numpy(obs[0].copy()).cuda()
    idx = torch.from_numpy(gm.obs_indices.astype(np.int32)).cuda()
    mask = gm.device_mask()
    pf._lib.call("pf_fhnnet_step", gm.params(), pf._lib.PF_F32, pf._lib.ptr(x), pf._lib.ptr(q),
                 None, pf._lib.ptr(xo), pf._lib.ptr(qo), pf._lib.ptr(mask), pf._lib.ptr(y),
                 pf._lib.ptr(idx), pf._lib.ptr(lw), M, N, None, 81, pf._lib.ptr(stim),
                 pf._lib.ptr(z), pf._lib.ptr(st_), pf._lib.stream_ptr())
    got = gm.from_device(xo, qo)
    want = np.concatenate([t[1] for t in traces])
    K = gm.nodes
    assert norm_rel(got[:, : 2 * K], want[:, : 2 * K]) < 1e-4
    assert np.array_equal(got[:, 2 * K:], want[:, 2 * K:])  # same stimulus decisions
    assert norm_rel(lw.cpu().numpy(), np.concatenate([t[2] for t in traces])) < 1e-4


# ---------------------------------------------------------------- production mode

def test_native_driver_equals_stepwise_path(golden):
    """pf_bank_run's FH-N network branch == the per-step Python path."""
    g = golden["fhnnet"]
    _, gm = models8(golden)
    obs = g["sim8_obs"][:30]
    keys = pf.philox.filter_keys(3, 4)
    out = []
    for native in (True, False):
        bank = pf.FilterBank(gm, 4, 64, keys, len(obs), dtype=torch.float32)
        bank.load_observations(obs)
        bank.init()
        if not native:
            bank.kernel_events = (torch.cuda.Event(), torch.cuda.Event())
        bank.run()
        torch.cuda.synchronize()
        bank.check_status()
        out.append((bank.est.cpu().numpy(), bank.lnc_tr.cpu().numpy(), bank.particles()))
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("dtype", ["float32", "float64"])
def test_fhn_tracking_check_passes(dtype):
    """verify.check_fhn_tracking with the reference's acceptance parameters
    (J=16, 100 observations, M=4, N in (100, 250, 500), 10 replicates,
    auxiliary filters): MSE non-increasing in N, tail correlation > 0.8."""
    from paper_1407_8071_b200 import verify

    res = verify.check_fhn_tracking(dtype=dtype)
    print(res.line())
    assert res.passed, res.line()


def test_production_is_deterministic_and_tracks(golden):
    g = golden["fhnnet"]
    gm = pf.FhnNetworkModel(J=16, stim_prob=0.02)
    obs = g["sim16_obs"]
    truth_u = gm.error_projection(g["sim16_states"][1:])
    a = pf.run_ensemble(gm, obs, "bootstrap", 4, 512, 7, dtype="float32", estimate="projection")
    b = pf.run_ensemble(gm, obs, "bootstrap", 4, 512, 7, dtype="float32", estimate="projection")
    assert np.array_equal(a.mean_estimates, b.mean_estimates)
    mse = float(np.mean((a.mean_estimates - truth_u) ** 2))
    assert mse < 0.5 * float(np.mean((truth_u - truth_u.mean()) ** 2))


@pytest.mark.parametrize("noise_free", [False, True])
@pytest.mark.parametrize("J", [8, 12, 20, 28, 32])
def test_fast_kernel_matches_generic(golden, monkeypatch, J, noise_free):
    """The bulk-copy fp32 kernel and the generic kernel run the same
    Philox draws and arithmetic order: states within fp32 rounding of each
    other, identical stimulus decisions (history bits).  noise_free: the
    auxiliary filter's lookahead transition (fhn.py:191-197)."""
    g = golden["fhnnet"]
    gm = pf.FhnNetworkModel(J=J, n_zones=2, zone_width=2, stim_prob=0.5)
    M, N = 3, 40
    if J == 8:
        x0 = np.tile(g["sim8_states"][80], (M * N, 1))
        y = g["sim8_obs"][80]
    else:
        rng = np.random.default_rng(4)
        x0 = np.zeros((M * N, gm.dim_x))
        x0[:, : gm.nodes] = rng.uniform(-2.0, 2.0, size=(M * N, gm.nodes))
        x0[:, gm.nodes: 2 * gm.nodes] = rng.normal(size=(M * N, gm.nodes))
        x0[:, 2 * gm.nodes:] = rng.random((M * N, gm.stim_hold * gm.nodes)) < 0.02
        y = rng.normal(size=gm.dim_y)
    keys = torch.from_numpy(pf.philox.filter_keys(5, M).view(np.int32)).cuda()
    anc = torch.from_numpy(np.random.default_rng(1).integers(0, M * N, M * N)
                           .astype(np.int32)).cuda()
    dy = torch.from_numpy(np.asarray(y, dtype=np.float64).copy()).cuda()
    idx = torch.from_numpy(gm.obs_indices.astype(np.int32)).cuda()
    mask = gm.device_mask()
    outs = []
    for flags in (0, pf._lib.PF_KERNEL_GENERIC):
        x, q = gm.to_device(x0, dtype=torch.float32)
        xo, qo = torch.empty_like(x), torch.empty_like(q)
        lw = torch.empty(M * N, dtype=torch.float32, device="cuda")
        st = torch.zeros(M, dtype=torch.int32, device="cuda")
        for t in (81, 5000):  # forcing on / off
            pf._lib.call("pf_fhnnet_step_ex", gm.params(noise_free=noise_free),
                         pf._lib.PF_F32, pf._lib.ptr(x),
                         pf._lib.ptr(q), pf._lib.ptr(anc), pf._lib.ptr(xo), pf._lib.ptr(qo),
                         pf._lib.ptr(mask), pf._lib.ptr(dy), pf._lib.ptr(idx), pf._lib.ptr(lw),
                         M, N, pf._lib.ptr(keys), t, None, None, pf._lib.ptr(st), flags,
                         pf._lib.stream_ptr())
            torch.cuda.synchronize()
            outs.append((gm.from_device(xo, qo), lw.cpu().numpy().copy(), st.cpu().numpy()))
    for a, b in zip(outs[:2], outs[2:]):
        K = gm.nodes
        assert norm_rel(a[0][:, : 2 * K], b[0][:, : 2 * K]) < 1e-6
        assert np.array_equal(a[0][:, 2 * K:], b[0][:, 2 * K:])
        assert norm_rel(a[1], b[1]) < 1e-6
        assert np.array_equal(a[2], b[2])
    if noise_free:  # no new stimulus: the history just shifts
        K, H = gm.nodes, gm.stim_hold
        x_anc = x0[anc.cpu().numpy()]
        assert not outs[0][0][:, 2 * K: 3 * K].any()
        assert np.array_equal(outs[0][0][:, 3 * K:], x_anc[:, 2 * K: (H + 1) * K])
    else:  # stimuli actually fired somewhere in the fast run
        assert outs[0][0][:, 2 * gm.nodes: 3 * gm.nodes].sum() > 0
