"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle and the
golden fixtures generated from the reference.

Tolerances (north star): ancestors bit-exact; fp64 states / weights / lnc /
estimates within 1e-12 norm-relative (element-wise pure-relative fails near
zero even for a correct kernel); fp32 within 1e-4 norm-relative.
"""

import numpy as np
import pytest

from oracle import parpf_oracle as orc
from oracle import tapes

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import _lib  # noqa: E402


def norm_rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def certify_ties(anc_gpu, anc_ref, cum_ref, u):
    """Mismatching ancestors are allowed only where u sits within rounding
    distance of the reference CDF boundary, i.e. the choice is a rounding
    tie.  The distance bound is the worst-case error of an N-term fp64
    prefix sum of weights summing to 1 on either side: 2 * N * 2^-53
    (Higham, gamma_N).  Returns the number of (certified) mismatches."""
    n = cum_ref.shape[1]
    tol = 2.0 * n * 2.0 ** -53
    bad = np.argwhere(anc_gpu != anc_ref)
    for f, j in bad:
        k = min(anc_gpu[f, j], anc_ref[f, j])
        assert abs(cum_ref[f, k] - u[f, j]) <= tol, (
            f"uncertified ancestor mismatch at filter {f}, slot {j}")
    return len(bad)


# ---------------------------------------------------------------- L1 operators

def test_philox_device_matches_host_mirror():
    from paper_1407_8071_b200.philox import philox4x32_10

    rng = np.random.default_rng(0)
    ctr = rng.integers(0, 2**32, size=(1000, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, size=(1000, 2), dtype=np.uint64).astype(np.uint32)
    d_c = torch.from_numpy(ctr.view(np.int32)).cuda()
    d_k = torch.from_numpy(key.view(np.int32)).cuda()
    out = torch.empty((1000, 4), dtype=torch.int32, device="cuda")
    _lib.call("pf_philox_kat", _lib.ptr(d_c), _lib.ptr(d_k), _lib.ptr(out), 1000, _lib.stream_ptr())
    assert np.array_equal(out.cpu().numpy().view(np.uint32), philox4x32_10(ctr, key))


def test_lorenz_block_bit_exact(golden):
    g = golden["kernels"]
    out = pf.accel.lorenz_euler_block(g["lz_states"], g["lz_noise"], 1e-3, 10.0, 28.0, 8.0 / 3.0)
    assert np.array_equal(out, g["lz_out"])


@pytest.mark.parametrize("tag", ["rect", "sq"])
def test_fhn_block_bit_exact(golden, tag):
    g = golden["kernels"]
    p = g[f"fhn_{tag}_params"]
    u, v = pf.accel.fhn_euler_block(g[f"fhn_{tag}_U"], g[f"fhn_{tag}_V"], g[f"fhn_{tag}_drive"],
                                    g[f"fhn_{tag}_noise"], p[0], p[1], tuple(p[2:6]),
                                    tuple(p[6:9]), p[9])
    assert np.array_equal(u, g[f"fhn_{tag}_u_new"])
    assert np.array_equal(v, g[f"fhn_{tag}_v_new"])


def test_resample_indices_bit_exact(golden):
    g = golden["kernels"]
    for i in range(int(g["ri_count"])):
        idx = pf.accel.resample_indices(g[f"ri_cum_{i}"], g[f"ri_u_{i}"])
        assert idx.dtype == np.int64
        assert np.array_equal(idx, g[f"ri_idx_{i}"]), i
    assert not np.any(pf.accel.resample_indices(g["ri_cum_0"], g["ri_u_0"]) == 1)


def test_normalize_log_weights(golden):
    g = golden["kernels"]
    for i in range(int(g["nlw_count"])):
        w, lm = pf.normalize_log_weights(g[f"nlw_in_{i}"])
        assert norm_rel(w, g[f"nlw_w_{i}"]) < 1e-14
        assert abs(lm - float(g[f"nlw_lm_{i}"])) <= 1e-12 * max(1.0, abs(lm))
    with pytest.raises(pf.WeightCollapseError):
        pf.normalize_log_weights(np.full(8, -np.inf))
    with pytest.raises(ValueError):
        pf.normalize_log_weights(np.array([0.0, np.nan]))
    with pytest.raises(ValueError):
        pf.normalize_log_weights(np.array([]))


def test_multinomial_resample_consumes_rng_like_reference(golden):
    g = golden["kernels"]
    idx = pf.multinomial_resample_indices(g["mri_w"], 500, np.random.default_rng(77))
    assert np.array_equal(idx, g["mri_idx"])


# ---------------------------------------------------------------- bank, oracle mode

def _lorenz_models(truth0):
    om = orc.LorenzConfigModel(prior_mean=tuple(truth0))
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    return om, gm


def _run_bank_with_tape(gmodel, obs, M, N, prior, noise, uni, dtype=None):
    tape = pf.DrawTape(prior=prior, noise=noise, uniforms=uni)
    bank = pf.FilterBank(gmodel, M, N, np.zeros((M, 2), np.uint32), len(obs), tape=tape,
                         dtype=dtype)
    bank.load_observations(obs)
    bank.init()
    ancs = []
    for k in range(len(obs)):
        bank.step(k)
        ancs.append(bank.anc.cpu().numpy().reshape(M, N) - np.arange(M)[:, None] * N)
    torch.cuda.synchronize()
    return bank, ancs


def test_lorenz_bank_oracle_mode_fp64(golden):
    g = golden["lorenz"]
    om, gm = _lorenz_models(g["truth0"])
    M, N = 4, 100
    traces, mean, prior, noise, uni = tapes.ensemble_with_tape(om, g["obs"], M, N,
                                                              int(g["e_master"]))
    assert np.array_equal(mean, g["e_mean"])  # oracle == reference fixture
    bank, ancs = _run_bank_with_tape(gm, g["obs"], M, N, prior, noise, uni)
    for k in range(len(g["obs"])):
        want = np.stack([tr.steps[k].ancestors for tr in traces])
        assert np.array_equal(ancs[k], want), f"step {k + 1}"
    est = bank.est.cpu().numpy()
    assert norm_rel(est, np.stack([tr.estimates for tr in traces], axis=1)) < 1e-12
    assert norm_rel(bank.lnc_tr.cpu().numpy(), g["e_lnc"].T) < 1e-12


def test_lorenz_run_ensemble_oracle_mode_matches_golden(golden):
    g = golden["lorenz"]
    om, gm = _lorenz_models(g["truth0"])
    _, _, prior, noise, uni = tapes.ensemble_with_tape(om, g["obs"], 4, 100, int(g["e_master"]))
    out = pf.run_ensemble(gm, g["obs"], "bootstrap", 4, 100, int(g["e_master"]),
                          tape=pf.DrawTape(prior, noise, uni))
    assert norm_rel(out.mean_estimates, g["e_mean"]) < 1e-12
    assert norm_rel(np.stack([o.estimates for o in out.filter_outputs]), g["e_est"]) < 1e-12
    assert norm_rel(np.stack([o.log_norm_const for o in out.filter_outputs]), g["e_lnc"]) < 1e-12


def test_lorenz_one_interval_fp32_within_1e4(golden):
    g = golden["lorenz"]
    om, gm = _lorenz_models(g["truth0"])
    traces, _, prior, noise, uni = tapes.ensemble_with_tape(om, g["obs"][:1], 2, 512, 3)
    bank, _ = _run_bank_with_tape(gm, g["obs"][:1], 2, 512, prior, noise, uni,
                                  dtype=torch.float32)
    x = bank.x[1].cpu().numpy().astype(np.float64)  # propagated planes (3, M*N)
    want = np.concatenate([tr.steps[0].propagated for tr in traces]).T
    assert norm_rel(x, want) < 1e-4
    lw = bank.logw.cpu().numpy().astype(np.float64)
    assert norm_rel(lw, np.concatenate([tr.steps[0].log_w for tr in traces])) < 1e-4


def test_lorenz_collapse_semantics(golden):
    g = golden["lorenz"]
    om, gm = _lorenz_models(g["truth0"])
    tr = orc.run_filter(om, g["c_obs"], 32, 11, keep_steps=True)
    assert tr.collapse_steps == [3]
    rec = orc.TapeRecorder(11)
    tr = orc.run_filter(om, g["c_obs"], 32, rec, keep_steps=True)
    prior = tr.prior_noise[None]
    noise = [s.noise[None] for s in tr.steps]
    uni = [(s.u if s.u is not None else np.full(32, np.nan))[None] for s in tr.steps]
    out = pf.run_filter(gm, g["c_obs"], "bootstrap", 32, 11,
                        tape=pf.DrawTape(prior, noise, uni))
    assert out.collapse_steps == [3]
    assert out.log_norm_const[2] == out.log_norm_const[1]
    assert norm_rel(out.estimates, g["c_est"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["c_lnc"]) < 1e-12


def test_fhn_bank_oracle_mode_fp64(golden):
    g = golden["fhn"]
    om = orc.FhnConfigModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    gm = pf.FhnLatticeModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    M, N = 2, 8
    traces, mean, prior, noise, uni = tapes.ensemble_with_tape(om, g["obs"], M, N, 5)
    bank, ancs = _run_bank_with_tape(gm, g["obs"], M, N, None, noise, uni)
    for k in range(len(g["obs"])):
        want = np.stack([tr.steps[k].ancestors for tr in traces])
        assert np.array_equal(ancs[k], want), f"step {k + 1}"
        # log-weights of the last step's propagated particles
    lw_want = np.concatenate([tr.steps[-1].log_w for tr in traces])
    assert norm_rel(bank.logw.cpu().numpy(), lw_want) < 1e-12
    est = bank.est.cpu().numpy()
    assert norm_rel(est, np.stack([tr.estimates for tr in traces], axis=1)) < 1e-12
    lnc_want = np.stack([tr.log_norm_const for tr in traces], axis=1)
    assert norm_rel(bank.lnc_tr.cpu().numpy(), lnc_want) < 1e-12


def test_fhn_filter_matches_golden(golden):
    g = golden["fhn"]
    om = orc.FhnConfigModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    gm = pf.FhnLatticeModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    rec = orc.TapeRecorder(np.random.SeedSequence(99))
    tr = orc.run_filter(om, g["obs"], 8, rec, keep_steps=True)
    noise = [s.noise.reshape(om.substeps, 2, 8, -1)[None] for s in tr.steps]
    uni = [s.u[None] for s in tr.steps]
    out = pf.run_filter(gm, g["obs"], "bootstrap", 8, 99,
                        tape=pf.DrawTape(None, noise, uni))
    assert norm_rel(out.estimates[:, : om.nodes], g["f_est_v"]) < 1e-12
    assert norm_rel(out.log_norm_const, g["f_lnc"]) < 1e-12


@pytest.mark.parametrize("M,N", [(2, 16), (1, 7)])
def test_fhn_one_interval_fp32_within_1e4(golden, M, N):
    """The fp32 production kernel (tape-fed), incl. an odd particle count."""
    g = golden["fhn"]
    om = orc.FhnConfigModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    gm = pf.FhnLatticeModel(stim_row=int(g["stim"][0]), stim_col=int(g["stim"][1]))
    traces, _, _, noise, uni = tapes.ensemble_with_tape(om, g["obs"][:1], M, N, 8)
    bank, _ = _run_bank_with_tape(gm, g["obs"][:1], M, N, None, noise, uni,
                                  dtype=torch.float32)
    x = bank.x[1].cpu().numpy().astype(np.float64)
    want = np.concatenate([tr.steps[0].propagated for tr in traces])
    assert norm_rel(x, want) < 1e-4
    assert norm_rel(bank.logw.cpu().numpy(),
                    np.concatenate([tr.steps[0].log_w for tr in traces])) < 1e-4


# ---------------------------------------------------------------- resampling (cfg1)

def _resample_case(M, N, sigma, seed):
    rng = np.random.default_rng(seed)
    lw = (rng.standard_normal((M, N)) * sigma).astype(np.float32)
    u = orc.sorted_uniform_rows(np.random.default_rng(seed + 1), M, N)
    return lw, u


def _gpu_resample(lw, u, flags=0):
    M, N = lw.shape
    d_lw = torch.from_numpy(lw.reshape(-1)).cuda()
    d_u = torch.from_numpy(u.reshape(-1)).cuda()
    anc = torch.empty(M * N, dtype=torch.int32, device="cuda")
    lnc = torch.zeros(M, dtype=torch.float64, device="cuda")
    coll = torch.zeros(M, dtype=torch.uint8, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    wsb = _lib.load().pf_resample_workspace_bytes(M, N)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(d_lw), M, N, _lib.ptr(d_u), None,
              1, _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll), _lib.ptr(st), _lib.ptr(ws), wsb,
              None, None, 0, flags, _lib.stream_ptr())
    a = anc.cpu().numpy().reshape(M, N).astype(np.int64) - (np.arange(M) * N)[:, None]
    return a, lnc.cpu().numpy(), coll.cpu().numpy()


@pytest.mark.parametrize("sigma", [1.0, 10.0])
def test_cfg1_bank_ancestors_bit_exact(sigma):
    M, N = 1 << 12, 1 << 10  # a 4096-filter slice of cfg1's 2^16 bank (CPU oracle time)
    lw, u = _resample_case(M, N, sigma, seed=int(sigma))
    anc, lmr, coll = _gpu_resample(lw, u)
    ref_anc, ref_lmr, ref_coll, cum = orc.resample_rows(lw, u)
    assert not coll.any()
    assert certify_ties(anc, ref_anc, cum, u) == 0
    assert np.all(np.diff(anc, axis=1) >= 0)
    assert np.max(np.abs(lmr - ref_lmr)) < 1e-12


@pytest.mark.parametrize("M,N", [(3, 20000), (2, 70001)])
def test_wide_path_multi_filter(M, N):
    lw, u = _resample_case(M, N, 3.0, seed=N)
    anc, lmr, coll = _gpu_resample(lw, u)
    ref_anc, ref_lmr, _, cum = orc.resample_rows(lw, u)
    assert certify_ties(anc, ref_anc, cum, u) == 0
    assert np.max(np.abs(lmr - ref_lmr)) < 1e-12


@pytest.mark.parametrize("M,N,sigma", [(1 << 12, 1 << 10, 1.0), (1 << 12, 1 << 10, 10.0),
                                         (8, 8192, 3.0), (3, 20000, 1.0), (2, 70001, 10.0)])
def test_reference_order_cdf_is_bit_exact(M, N, sigma):
    """PF_RS_REFERENCE_ORDER: numpy-order total + sequential cumsum -> the
    CDF equals the reference's bit for bit, hence zero ancestor mismatches."""
    lw, u = _resample_case(M, N, sigma, seed=N + int(sigma))
    anc, lmr, coll = _gpu_resample(lw, u, flags=_lib.PF_RS_REFERENCE_ORDER)
    ref_anc, ref_lmr, _, _ = orc.resample_rows(lw, u)
    assert np.array_equal(anc, ref_anc)
    assert np.max(np.abs(lmr - ref_lmr)) < 1e-12


@pytest.mark.parametrize("sigma", [1.0, 10.0])
def test_cfg1_centralised_2pow26_reference_order_bit_exact(sigma):
    """BASELINE cfg1 centralised case, M=1 x N=2^26: bit-exact ancestors."""
    N = 1 << 26
    lw, u = _resample_case(1, N, sigma, seed=100 + int(sigma))
    anc, lmr, _ = _gpu_resample(lw, u, flags=_lib.PF_RS_REFERENCE_ORDER)
    ref_anc, ref_lmr, _, _ = orc.resample_rows(lw, u)
    n_bad = int(np.count_nonzero(anc != ref_anc))
    print(f"N=2^26 sigma={sigma} reference order: {n_bad} mismatches")
    assert n_bad == 0
    assert abs(lmr[0] - ref_lmr[0]) < 1e-10


@pytest.mark.parametrize("sigma", [1.0, 10.0])
def test_cfg1_centralised_2pow26(sigma):
    N = 1 << 26
    lw, u = _resample_case(1, N, sigma, seed=100 + int(sigma))
    anc, lmr, coll = _gpu_resample(lw, u)
    ref_anc, ref_lmr, _, cum = orc.resample_rows(lw, u)
    n_ties = certify_ties(anc, ref_anc, cum, u)
    print(f"N=2^26 sigma={sigma}: {n_ties} certified rounding-tie mismatches")
    assert n_ties < 2000
    assert abs(lmr[0] - ref_lmr[0]) < 1e-10


def test_collapse_and_nan_flags():
    lw = np.zeros((3, 64), np.float32)
    lw[1] = -np.inf
    lw[2, 5] = np.nan
    u = orc.sorted_uniform_rows(np.random.default_rng(0), 3, 64)
    anc, lmr, coll = _gpu_resample(lw, u)
    assert coll.tolist() == [0, 1, 0]
    assert np.array_equal(anc[1], np.arange(64))
    assert lmr[1] == 0.0


# ---------------------------------------------------------------- production (Philox) mode

def _cfg0_small():
    truth0, _, obs = orc.lorenz_truth(seed=3, n_obs=20)
    _, gm = _lorenz_models(truth0)
    return gm, obs


def test_philox_mode_deterministic_and_seed_tree():
    gm, obs = _cfg0_small()
    a = pf.run_filter(gm, obs, "bootstrap", 256, 12345)
    b = pf.run_filter(gm, obs, "bootstrap", 256, 12345)
    c = pf.run_filter(gm, obs, "bootstrap", 256, 54321)
    assert a.same_result(b) and not a.same_result(c)
    ens = pf.run_ensemble(gm, obs, "bootstrap", 1, 256, 5)
    single = pf.run_filter(gm, obs, "bootstrap", 256, pf.filter_seeds(5, 1)[0])
    assert np.array_equal(ens.mean_estimates, single.estimates)


def test_sharding_does_not_change_filters():
    """Filters computed as two half-banks (as two ranks would) equal the
    full bank bit for bit (GPU-count invariance)."""
    gm, obs = _cfg0_small()
    keys = pf.philox.filter_keys(9, 4)
    outs = []
    for lo, hi in ((0, 4), (0, 2), (2, 4)):
        b = pf.FilterBank(gm, hi - lo, 128, keys[lo:hi], len(obs), dtype=torch.float32)
        b.load_observations(obs)
        b.init()
        b.run()
        outs.append((b.est.cpu().numpy(), b.lnc_tr.cpu().numpy()))
    full_est, full_lnc = outs[0]
    assert np.array_equal(full_est[:, :2], outs[1][0]) and np.array_equal(full_est[:, 2:], outs[2][0])
    assert np.array_equal(full_lnc[:, :2], outs[1][1]) and np.array_equal(full_lnc[:, 2:], outs[2][1])


def test_left_to_right_average():
    gm, obs = _cfg0_small()
    out = pf.run_ensemble(gm, obs, "bootstrap", 5, 64, 11)
    acc = out.filter_outputs[0].estimates.copy()
    for fo in out.filter_outputs[1:]:
        acc += fo.estimates
    assert np.array_equal(out.mean_estimates, acc / 5.0)


def test_divergence_raises():
    gm = pf.Lorenz63Model(substeps=40, prior_mean=(1e200, 1e200, 1e200), prior_var=1.0)
    with pytest.raises(pf.NumericalDivergenceError):
        pf.run_filter(gm, np.zeros((2, 1)), "bootstrap", 16, 0)


def test_nan_observation_raises_value_error():
    gm, obs = _cfg0_small()
    obs = obs.copy()
    obs[1, 0] = np.nan
    with pytest.raises(ValueError):
        pf.run_filter(gm, obs, "bootstrap", 16, 0)


def test_invalid_arguments():
    gm, obs = _cfg0_small()
    with pytest.raises(ValueError):
        pf.run_ensemble(gm, obs, "bootstrap", 0, 10, 0)
    with pytest.raises(ValueError):
        pf.run_ensemble(gm, obs, "bootstrap", 2, 10, 0, workers=0)
    with pytest.raises(ValueError):
        pf.run_filter(gm, obs, "smooth", 10, 0)
    with pytest.raises(ValueError):
        pf.run_filter(gm, np.zeros((0, 2)), "bootstrap", 10, 0)


def test_philox_filter_tracks_truth():
    """Production-mode sanity: the cfg0 bank tracks the truth about as well
    as the CPU oracle does (statistical parity proper: test_gpu_stats.py)."""
    truth0, states, obs = orc.lorenz_truth(seed=4, n_obs=60)
    _, gm = _lorenz_models(truth0)
    out = pf.run_ensemble(gm, obs, "bootstrap", 4, 1000, 1)
    mse = np.mean((out.mean_estimates - states) ** 2)
    assert mse < 2.0, mse


@pytest.mark.parametrize("M,N", [(64, 1024), (2, 20000)])
def test_resample_gather_fused_matches_unfused(M, N):
    lw, u = _resample_case(M, N, 1.0, seed=5)
    anc_ref, _, _ = _gpu_resample(lw, u)
    d_lw = torch.from_numpy(lw.reshape(-1)).cuda()
    d_u = torch.from_numpy(u.reshape(-1)).cuda()
    x = torch.randn((3, M * N), device="cuda")
    xo = torch.empty_like(x)
    anc = torch.empty(M * N, dtype=torch.int32, device="cuda")
    lnc = torch.zeros(M, dtype=torch.float64, device="cuda")
    coll = torch.zeros(M, dtype=torch.uint8, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    wsb = _lib.load().pf_resample_workspace_bytes(M, N)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(d_lw), M, N, _lib.ptr(d_u),
              None, 1, _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll), _lib.ptr(st), _lib.ptr(ws),
              wsb, _lib.ptr(x), _lib.ptr(xo), 3, 0, _lib.stream_ptr())
    a = anc.cpu().numpy().astype(np.int64)
    assert np.array_equal(a.reshape(M, N) - (np.arange(M) * N)[:, None], anc_ref)
    assert torch.equal(xo, x[:, anc.long()])


# ---------------------------------------------------------------- edge cases

@pytest.mark.parametrize("M,N", [(1, 1), (3, 1), (5, 7), (2, 257), (1, 8192), (2, 9000)])
def test_lorenz_bank_edge_sizes_bit_exact(M, N):
    """Single particle, odd and non-power-of-two N, the bank/wide boundary
    (8192 / 9000 -> wide path): ancestors bit-exact vs the oracle."""
    truth0, _, obs = orc.lorenz_truth(seed=M * 31 + N, n_obs=3)
    om, gm = _lorenz_models(truth0)
    traces, mean, prior, noise, uni = tapes.ensemble_with_tape(om, obs, M, N, 77)
    bank, ancs = _run_bank_with_tape(gm, obs, M, N, prior, noise, uni)
    for k in range(len(obs)):
        assert np.array_equal(ancs[k], np.stack([tr.steps[k].ancestors for tr in traces])), k
    assert norm_rel(bank.est.cpu().numpy(), np.stack([tr.estimates for tr in traces], 1)) < 1e-12
    assert norm_rel(bank.lnc_tr.cpu().numpy(),
                    np.stack([tr.log_norm_const for tr in traces], 1)) < 1e-12


def test_single_particle_filter_is_deterministic_copy():
    """N=1: every step resamples the only particle (weights [1.0])."""
    truth0, _, obs = orc.lorenz_truth(seed=2, n_obs=4)
    _, gm = _lorenz_models(truth0)
    out = pf.run_filter(gm, obs, "bootstrap", 1, 3)
    assert out.estimates.shape == (4, 3) and np.all(np.isfinite(out.estimates))
    apf = pf.run_filter(gm, obs, "auxiliary", 1, 3)
    assert apf.estimates.shape == (4, 3)


def test_stock_lorenz_model_observing_x1():
    """The stock reference model (obs of x1 only, 100 substeps, prior
    LORENZ_PRIOR_MEAN / var 10) through the bank, oracle mode, fp64."""
    from oracle.parpf_oracle import LorenzConfigModel

    om = LorenzConfigModel(substeps=100, noise_scale=1.0, obs_var=0.5,
                           prior_mean=pf.LORENZ_PRIOR_MEAN, prior_var=10.0)
    om.dim_y = 1

    def ll(y, x, t, _m=om):
        r = float(np.asarray(y).reshape(-1)[0]) - np.asarray(x)[:, 0]
        return -(r * r) / (2.0 * _m.obs_var)

    om.log_likelihood = ll
    rng = np.random.default_rng(0)
    obs = (np.array(pf.LORENZ_PRIOR_MEAN)[0] + rng.normal(size=(4, 1)))
    traces, mean, prior, noise, uni = tapes.ensemble_with_tape(om, obs, 2, 50, 5)
    gm = pf.Lorenz63Model()
    bank, ancs = _run_bank_with_tape(gm, obs, 2, 50, prior, noise, uni)
    for k in range(len(obs)):
        assert np.array_equal(ancs[k], np.stack([tr.steps[k].ancestors for tr in traces]))
    assert norm_rel(bank.est.cpu().numpy(), np.stack([tr.estimates for tr in traces], 1)) < 1e-12


# ---------------------------------------------------------------- production resampling law

def _offspring_counts(lw, reps, flags, seed):
    """Total offspring counts over `reps` production-mode (Philox) resamples
    of the same log weights (different time words)."""
    M, N = lw.shape
    d_lw = torch.from_numpy(lw.reshape(-1)).cuda()
    anc = torch.empty(M * N, dtype=torch.int32, device="cuda")
    lnc = torch.zeros(M, dtype=torch.float64, device="cuda")
    coll = torch.zeros(M, dtype=torch.uint8, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    keys = torch.from_numpy(pf.philox.filter_keys(seed, M).view(np.int32)).cuda()
    wsb = _lib.load().pf_resample_workspace_bytes(M, N)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    counts = torch.zeros(M * N, dtype=torch.int64, device="cuda")
    for r in range(reps):
        _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(d_lw), M, N, None,
                  _lib.ptr(keys), r + 1, _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll),
                  _lib.ptr(st), _lib.ptr(ws), wsb, None, None, 0, flags, _lib.stream_ptr())
        counts += torch.bincount(anc.long(), minlength=M * N)
    return counts.cpu().numpy().reshape(M, N)


@pytest.mark.parametrize("M,N,flags", [(64, 1024, 0), (2, 20000, 0), (2, 20000, 1),
                                       (1, 1 << 20, 0), (1, (1 << 22) + 77, 0),
                                       # every bank-kernel tile shape: 2 particles per
                                       # thread (N <= 256; and the wide CTAs of few-filter
                                       # banks, M < #SMs), 4, 8 and 16 per thread
                                       (300, 64, 0), (200, 256, 0), (4, 1000, 0),
                                       (3, 2000, 0), (5, 300, 0), (160, 512, 0),
                                       (150, 4096, 0)])
def test_production_resampling_is_multinomial(M, N, flags):
    """Offspring counts follow multinomial(N, w) (test_resampling.py:40-67
    analogue): chi-square over B equal-mass bins per filter; the sum over a
    bank's filters (df = M (B-1)) at 1e-4 and every filter at a Bonferroni
    1e-4 / M - sensitive to a small systematic bias of the uniform stream."""
    from scipy import stats

    rng = np.random.default_rng(N + M)
    lw = rng.standard_normal((M, N)).astype(np.float32)
    w = np.exp(lw.astype(np.float64) - lw.max(axis=1, keepdims=True))
    w /= w.sum(axis=1, keepdims=True)
    reps = 40 if N >= 1024 else max(40, (40 * 1024) // N)
    counts = _offspring_counts(lw, reps, flags, seed=3)
    assert np.all(counts.sum(axis=1) == reps * N)
    B = 64 if N >= 1024 else 16
    chis = []
    for f in range(M):
        edges = np.searchsorted(np.cumsum(w[f]), np.linspace(0, 1, B + 1)[1:-1])
        obs = np.add.reduceat(counts[f], np.r_[0, edges])
        exp_ = np.add.reduceat(w[f], np.r_[0, edges]) * reps * N
        chis.append(float(((obs - exp_) ** 2 / exp_).sum()))
    chis = np.array(chis)
    assert chis.sum() < stats.chi2.ppf(1 - 1e-4, df=M * (B - 1)), (chis.sum(), M * (B - 1))
    assert chis.max() < stats.chi2.ppf(1 - 1e-4 / M, df=B - 1), (int(chis.argmax()), chis.max())


def test_production_wide_chunked_filter_totals():
    """Filters wider than 8192 tiles (N > 2^24) combine their tile totals in
    chunks (wide2_chunk_scan/combine/apply): log normalising constants,
    zero offspring for -inf weights (a whole chunk of them in filter 0, a
    partial last chunk), multinomial offspring counts."""
    from scipy import stats

    M, N = 2, (1 << 25) + 12345
    rng = np.random.default_rng(11)
    lw = rng.standard_normal((M, N)).astype(np.float32)
    lw[0, : 1 << 24] = -np.inf
    reps = 8
    counts = _offspring_counts(lw, reps, 0, seed=5)
    assert np.all(counts.sum(axis=1) == reps * N)
    assert counts[0, : 1 << 24].sum() == 0
    d_lw = torch.from_numpy(lw.reshape(-1)).cuda()
    anc = torch.empty(M * N, dtype=torch.int32, device="cuda")
    lnc = torch.zeros(M, dtype=torch.float64, device="cuda")
    coll = torch.zeros(M, dtype=torch.uint8, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    keys = torch.from_numpy(pf.philox.filter_keys(5, M).view(np.int32)).cuda()
    wsb = _lib.load().pf_resample_workspace_bytes(M, N)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(d_lw), M, N, None,
              _lib.ptr(keys), 1, _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll), _lib.ptr(st),
              _lib.ptr(ws), wsb, None, None, 0, 0, _lib.stream_ptr())
    lw64 = lw.astype(np.float64)
    for f in range(M):
        fin = lw64[f][np.isfinite(lw64[f])]
        mx = fin.max()
        ref = mx + np.log(np.exp(fin - mx).sum()) - np.log(N)
        # production log weights are exponentiated in fp32 (expf): ~1e-7 relative
        assert abs(lnc[f].item() - ref) < 1e-7, (f, lnc[f].item(), ref)
    assert coll.sum().item() == 0 and st.sum().item() == 0
    B = 64
    for f in range(M):
        w = np.exp(lw64[f] - lw64[f][np.isfinite(lw64[f])].max())
        w /= w.sum()
        edges = np.searchsorted(np.cumsum(w), np.linspace(0, 1, B + 1)[1:-1])
        obs = np.add.reduceat(counts[f], np.r_[0, edges])
        exp_ = np.add.reduceat(w, np.r_[0, edges]) * reps * N
        chi2 = float(((obs - exp_) ** 2 / exp_).sum())
        assert chi2 < stats.chi2.ppf(0.999, df=B - 1), (f, chi2)


def test_small_bank_warp_kernel_bit_identical():
    """fp64 production banks below 2^15 particles run one warp per two
    particles (RNG in parallel over the lanes, lanes 0-1 run the two substep
    chains); the result is bit-identical to the thread-per-particle kernel
    (PF_KERNEL_GENERIC)."""
    truth0, _, obs = orc.lorenz_truth(seed=8, n_obs=6)
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    gm3 = pf.Lorenz63Model(substeps=3, prior_mean=tuple(truth0))

    def run(model, y, M, N, flags):
        bank = pf.FilterBank(model, M, N, pf.philox.filter_keys(5, M), len(y),
                             kernel_flags=flags)
        bank.load_observations(y)
        bank.init()
        bank.run()
        torch.cuda.synchronize()
        bank.check_status()
        return (bank.est.cpu().numpy(), bank.lnc_tr.cpu().numpy(), bank.anc.cpu().numpy(),
                bank.x[bank.cur].cpu().numpy())

    for model, y, M, N in ((gm, obs, 4, 1000), (gm3, obs[:, :1], 1, 100)):
        # odd substep count (gm3): the last pair's second substep is dropped
        a = run(model, y, M, N, 0)
        b = run(model, y, M, N, _lib.PF_KERNEL_GENERIC)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_native_fused_estimate_matches_separate_pass(dtype):
    """pf_bank_run fuses the planar-state posterior mean into the resampler;
    it agrees with the standalone pf_filter_estimate pass of the per-step
    path to fp64 rounding, and states / lnc are identical."""
    truth0, _, obs = orc.lorenz_truth(seed=12, n_obs=6)
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    keys = pf.philox.filter_keys(3, 5)
    res = []
    for native in (True, False):
        bank = pf.FilterBank(gm, 5, 333, keys, len(obs), dtype=dtype)
        bank.load_observations(obs)
        bank.init()
        if not native:
            bank.kernel_events = (torch.cuda.Event(), torch.cuda.Event())
        bank.run()
        torch.cuda.synchronize()
        res.append((bank.est.cpu().numpy(), bank.lnc_tr.cpu().numpy(), bank.particles()))
    assert norm_rel(res[0][0], res[1][0]) < 1e-13
    assert np.array_equal(res[0][1], res[1][1])
    assert np.array_equal(res[0][2], res[1][2])


def test_hook_level_resamplers_match_reference(golden):
    """systematic_resample_indices and a 50,000-weight multinomial draw
    against the reference's own outputs (sequential cumsum on the device)."""
    g = golden["kernels"]
    idx = pf.systematic_resample_indices(g["mri_w"], 700, np.random.default_rng(78))
    assert np.array_equal(idx, g["sys_idx"])
    idx = pf.multinomial_resample_indices(g["mri_big_w"], 60_000, np.random.default_rng(79))
    assert np.array_equal(idx, g["mri_big_idx"])
    x = np.arange(500.0)[:, None]
    assert np.array_equal(pf.systematic_resample(x, g["mri_w"], 700, np.random.default_rng(78)),
                          x[g["sys_idx"]])


def test_lorenz_helpers_match_reference(golden):
    g = golden["kernels"]
    tr = pf.lorenz_transition(np.array([1.0, 2.0, 3.0]), np.random.default_rng(3))
    assert np.array_equal(tr, g["lz_tr"])
    assert pf.lorenz_log_likelihood(0.7, np.array([1.0, 2.0, 3.0])) == float(g["lz_ll"])


@pytest.mark.gpu
def test_lorenz_uniform_key_kernel_matches_generic():
    """lorenz_fast_kernel<UKEY=true> (N % 256 == 0: block-uniform key and
    filter id) draws and computes exactly like the generic variant: particle j
    of filter f has the same Philox counter and key in a bank of N=256 (uniform
    path) and N=257 (generic path), so the propagated states must agree bit
    for bit."""
    import paper_1407_8071_b200 as pf

    model = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3")
    params = model.params()
    M = 3
    keys = torch.from_numpy(np.array([[11, 22], [33, 44], [55, 66]], np.uint32).view(np.int32)).cuda()
    y = torch.tensor([1.0, 2.0], dtype=torch.float64, device="cuda")
    rng = np.random.default_rng(5)
    base = rng.standard_normal((3, M, 257)).astype(np.float32) * 5.0
    outs = {}
    for N in (256, 257):
        xin = torch.from_numpy(np.ascontiguousarray(base[:, :, :N].reshape(3, M * N))).cuda()
        xout = torch.empty_like(xin)
        logw = torch.empty(M * N, dtype=torch.float32, device="cuda")
        status = torch.zeros(M, dtype=torch.int32, device="cuda")
        _lib.call("pf_lorenz_propagate_weight", params, _lib.PF_F32, _lib.ptr(xin), None,
                  _lib.ptr(xout), _lib.ptr(y), _lib.ptr(logw), M, N, _lib.ptr(keys), 3, None,
                  _lib.ptr(status), _lib.stream_ptr())
        torch.cuda.synchronize()
        outs[N] = (xout.cpu().numpy().reshape(3, M, N)[:, :, :256],
                   logw.cpu().numpy().reshape(M, N)[:, :256])
    assert np.all(np.isfinite(outs[256][0]))
    assert np.array_equal(outs[256][0], outs[257][0])
    assert np.array_equal(outs[256][1], outs[257][1])


def test_native_slot_timing_matches_one_call():
    """run_native one interval at a time into slots of a prepared event pool
    (the multi-GPU bench path: no host wait per interval) gives the same
    filter results as one multi-interval call, and a positive propagate
    duration per interval."""
    truth0, _, obs = orc.lorenz_truth(seed=4, n_obs=5)
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    keys = pf.philox.filter_keys(9, 4)
    res = []
    for sliced in (False, True):
        bank = pf.FilterBank(gm, 4, 512, keys, len(obs), dtype="float32")
        bank.load_observations(obs)
        bank.init()
        if sliced:
            bank.prepare_timing(len(obs))
            for k in range(len(obs)):
                assert bank.run_native(k, 1, time_propagate=True, slot=k) is None
            ms = bank.pool_propagate_ms(len(obs))
            assert len(ms) == len(obs) and all(m > 0 for m in ms)
            with pytest.raises(ValueError):
                bank.run_native(0, 1, time_propagate=True, slot=len(obs))
        else:
            bank.run_native(0, len(obs))
        torch.cuda.synchronize()
        res.append((bank.est.cpu().numpy(), bank.lnc_tr.cpu().numpy()))
    assert np.array_equal(res[0][0], res[1][0])
    assert np.array_equal(res[0][1], res[1][1])


@pytest.mark.parametrize("M,N,sigma", [(1, 1 << 20, 1.0), (1, 1 << 20, 10.0), (3, 70001, 3.0),
                                       (2, 20000, 30.0)])
def test_wide_pipeline_variants_identical(M, N, sigma):
    """The wide production pipeline's alternatives - merge path instead of the
    per-thread search, the gather as its own pass, and the CDF recomputed in
    the merge instead of materialised (PF_RS_WIDE_*) - give bit-identical
    ancestors, lnc and gathered states."""
    rng = np.random.default_rng(int(sigma) + N)
    lw = torch.from_numpy((rng.standard_normal(M * N) * sigma).astype(np.float32)).cuda()
    x = torch.from_numpy(rng.standard_normal((3, M * N)).astype(np.float32)).cuda()
    keys = torch.from_numpy(pf.philox.filter_keys(11, M).view(np.int32)).cuda()
    wsb = _lib.load().pf_resample_workspace_bytes(M, N)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    outs = []
    for flags in (0, _lib.PF_RS_WIDE_MERGE_PATH, _lib.PF_RS_WIDE_GATHER_SEPARATE,
                  _lib.PF_RS_WIDE_RECOMPUTE):
        anc = torch.empty(M * N, dtype=torch.int32, device="cuda")
        lnc = torch.zeros(M, dtype=torch.float64, device="cuda")
        coll = torch.zeros(M, dtype=torch.uint8, device="cuda")
        st = torch.zeros(M, dtype=torch.int32, device="cuda")
        xo = torch.empty_like(x)
        _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(lw), M, N, None,
                  _lib.ptr(keys), 5, _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll), _lib.ptr(st),
                  _lib.ptr(ws), wsb, _lib.ptr(x), _lib.ptr(xo), 3, flags, _lib.stream_ptr())
        torch.cuda.synchronize()
        outs.append((anc.cpu().numpy(), lnc.cpu().numpy(), xo.cpu().numpy()))
        assert np.all(np.diff(outs[-1][0].reshape(M, N), axis=1) >= 0)
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("N", [65536, 70001, 1 << 20])
def test_chunked_wide_estimate(N):
    """pf_filter_estimate_ws (wide filters, dim <= 8): the posterior mean of
    the resampled set (core.py:154-156 via filters.py:188) within 1e-12 of an
    fp64 reference sum, bit-identical for a filter whether it sits alone or in
    a bank (the chunk order depends on N only)."""
    rng = np.random.default_rng(N)
    M, dim = 3, 3
    x = torch.from_numpy(rng.standard_normal((dim, M * N)).astype(np.float32)).cuda()
    anc = torch.from_numpy(np.sort(rng.integers(0, N, (M, N)), axis=1).astype(np.int32)
                           + (np.arange(M) * N)[:, None].astype(np.int32)).reshape(-1).cuda()

    def est(xs, an, m):
        wsb = _lib.load().pf_estimate_workspace_bytes(m, N, dim)
        assert wsb > 0
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        out = torch.empty((m, dim), dtype=torch.float64, device="cuda")
        _lib.call("pf_filter_estimate_ws", _lib.PF_F32, _lib.ptr(xs), 1, m * N, dim, _lib.ptr(an),
                  m, N, _lib.ptr(out), dim, _lib.ptr(ws), wsb, _lib.stream_ptr())
        return out.cpu().numpy()

    e = est(x, anc, M)
    xh = x.cpu().numpy().astype(np.float64)
    ah = anc.cpu().numpy().reshape(M, N)
    want = np.stack([xh[:, ah[f]].mean(axis=1) for f in range(M)])
    assert np.max(np.abs(e - want)) < 1e-12 * max(1.0, np.abs(want).max()) + 1e-15
    # filter 1 alone (its own rows, ancestors re-based) gives the same bits
    x1 = x[:, N:2 * N].contiguous()
    a1 = (anc[N:2 * N] - N).contiguous()
    assert np.array_equal(est(x1, a1, 1)[0], e[1])
