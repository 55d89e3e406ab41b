"""Oracle-mode parity at the BASELINE config sizes (not only golden sizes).

* cfg0: Lorenz-63, M=4 x N=1000, all T=500 observations, fp64: ancestors
  bit-exact at every step for every filter, estimates / lnc / the M-average
  within 1e-12 (norm-relative).  Reference: run_ensemble ensemble.py:76-111,
  run_filter filters.py:163-193, resampling.py:29-43.
* cfg1: the full resampling bank M=2^16 x N=2^10, sigma in {1, 10}: the
  production (parallel fp64 CDF) ancestors differ from the reference's only
  at certified rounding ties (measured: none), and the reference-order CDF
  (PF_RS_REFERENCE_ORDER) is bit-exact.  Reference: core.py:116-138,
  resampling.py:29-43, accel.py:175-203.
* cfg3: FH-N lattice M=8 x N=512, 5 observations (250 Euler steps), fp64
  exact kernel: ancestors bit-exact, log-weights / estimates / lnc within
  1e-12.  Reference: accel.py:110-129 (numpy twin), fhn.py:199-207.

The oracle side is streamed one observation at a time
(oracle.tapes.StreamingEnsemble) so only one step's draws are in memory.
"""

import numpy as np
import pytest

from oracle import ckernels
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


def _stream_compare(om, gm, obs, M, N, master, dtype=torch.float64, check_logw=False):
    ckernels.install()
    T = obs.shape[0]
    se = tapes.StreamingEnsemble(om, obs, M, N, master)
    tape = pf.DrawTape(prior=se.prior, noise=[None] * T, uniforms=[None] * T)
    bank = pf.FilterBank(gm, M, N, np.zeros((M, 2), np.uint32), T, tape=tape, dtype=dtype)
    bank.load_observations(obs)
    bank.init()
    offs = (np.arange(M) * N)[:, None]
    lnc_ref, est_ref = [], []
    for k in range(T):
        r = se.step(k)
        tape.noise[k], tape.uniforms[k] = r["noise"], r["uniforms"]
        bank.step(k)
        anc = bank.anc.cpu().numpy().reshape(M, N) - offs
        assert np.array_equal(anc, r["ancestors"]), f"ancestors differ at step {k + 1}"
        if check_logw:
            assert norm_rel(bank.logw.cpu().numpy().reshape(M, N), r["log_w"]) < 1e-12
        tape.noise[k] = tape.uniforms[k] = None  # free the step's draws
        lnc_ref.append(r["lnc"])
        est_ref.append(r["estimates"])
    torch.cuda.synchronize()
    bank.check_status()
    est = bank.est.cpu().numpy()  # (T, M, dim)
    est_ref = np.stack(est_ref)
    assert norm_rel(est, est_ref) < 1e-12
    assert norm_rel(bank.lnc_tr.cpu().numpy(), np.stack(lnc_ref)) < 1e-12
    # the M-average in the reference's left-to-right order (ensemble.py:68-73)
    mean_ref = orc.average_estimates([est_ref[:, f] for f in range(M)])
    mean = torch.empty((T, est.shape[2]), dtype=torch.float64, device="cuda")
    _lib.call("pf_ensemble_average", _lib.ptr(bank.est), T, M, est.shape[2], _lib.ptr(mean),
              _lib.stream_ptr())
    assert norm_rel(mean.cpu().numpy(), mean_ref) < 1e-12


def test_cfg0_full_size_oracle_mode_bit_exact():
    truth0, _, obs = orc.lorenz_truth(seed=11, n_obs=500)
    om = orc.LorenzConfigModel(prior_mean=tuple(truth0))
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=tuple(truth0), prior_var=1.0)
    _stream_compare(om, gm, obs, 4, 1000, 2026)


def test_cfg3_full_bank_oracle_mode_fp64_bit_exact():
    m, _, obs = orc.fhn_truth(seed=12, n_obs=5)
    gm = pf.FhnLatticeModel(stim_row=m.stim_row, stim_col=m.stim_col)
    _stream_compare(m, gm, obs, 8, 512, 77, check_logw=True)


def _gpu_resample(lw, u, flags):
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
def test_cfg1_full_bank_2pow16_x_2pow10(sigma):
    M, N = 1 << 16, 1 << 10
    rng = np.random.default_rng(int(sigma) + 31)
    lw = (rng.standard_normal((M, N)) * sigma).astype(np.float32)
    u = orc.sorted_uniform_rows(np.random.default_rng(int(sigma) + 32), M, N)
    ref_anc, ref_lmr, ref_coll, cum = orc.resample_rows(lw, u)
    # production: parallel fp64 CDF; a mismatch is allowed only at a
    # certified rounding tie (u within 2 N 2^-53 of a reference CDF value)
    anc, lmr, coll = _gpu_resample(lw, u, 0)
    assert not coll.any() and not ref_coll.any()
    bad = np.argwhere(anc != ref_anc)
    tol = 2.0 * N * 2.0 ** -53
    for f, j in bad:
        k = min(anc[f, j], ref_anc[f, j])
        assert abs(cum[f, k] - u[f, j]) <= tol
    print(f"cfg1 bank sigma={sigma}: {len(bad)} certified ties of {M * N}")
    assert np.max(np.abs(lmr - ref_lmr)) < 1e-12
    # reference-order CDF: bit-exact
    anc2, lmr2, _ = _gpu_resample(lw, u, _lib.PF_RS_REFERENCE_ORDER)
    assert np.array_equal(anc2, ref_anc)
    assert np.max(np.abs(lmr2 - ref_lmr)) < 1e-12
