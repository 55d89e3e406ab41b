"""Pins of the production (Philox, fp32) propagate kernels that bench.py times.

* The specialised FH-N lattice kernel (fhn_fast_kernel<30,50,6,...>, the
  cfg3/cfg4 hot path) against the generic runtime-geometry kernel
  (fhn_interval_kernel<float,0>, accurate libm Box-Muller) on the same keys,
  counters and inputs: states and log-weights within 1e-4 norm-relative
  (north star fp32 tolerance).  The generic kernel shares only the counter
  layout (particle, step, row pair, purpose) and the word -> normal map; its
  arithmetic is an independent restatement of accel.py:110-129.
* The noise law of one Euler step: x(noisy) - x(noise-free) from the same
  state must be sig * N(0, 1), independent across nodes, rows of a Philox
  pair, the v/w components, particles and time steps (a wrong Box-Muller
  radius, row pairing or sig_v/sig_w scaling fails these z-score bounds).
  Reference: the noise terms of accel.py:121-128 (sig_sqdt * z on v) and
  the config's w-noise; Lorenz accel.py:73-75.
"""

import numpy as np
import pytest

from oracle import parpf_oracle as orc

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


def fhn_interval(gm, x, anc, y, M, N, t, *, n_sub=None, flags=0, noise_free=False,
                 master=5):
    """One pf_fhn_interval_ex launch through the C ABI; returns host copies
    of (x_out, logw, status)."""
    dt = x.dtype
    xo = torch.empty_like(x)
    lw = torch.empty(M * N, dtype=dt, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    keys = torch.from_numpy(pf.philox.filter_keys(master, M).view(np.int32)).cuda()
    dy = torch.from_numpy(np.asarray(y, dtype=np.float64).copy()).cuda()
    idx = torch.from_numpy(gm.obs_indices.astype(np.int32)).cuda()
    code = _lib.PF_F32 if dt == torch.float32 else _lib.PF_F64
    _lib.call("pf_fhn_interval_ex", gm.params(n_sub=n_sub, noise_free=noise_free), code,
              _lib.ptr(x), _lib.ptr(anc), _lib.ptr(xo), _lib.ptr(dy), _lib.ptr(idx),
              _lib.ptr(lw), M, N, _lib.ptr(keys), t, None, _lib.ptr(st), flags,
              _lib.stream_ptr())
    torch.cuda.synchronize()
    return (xo.cpu().numpy().astype(np.float64), lw.cpu().numpy().astype(np.float64),
            st.cpu().numpy())


def _random_lattice_states(gm, n, seed):
    rng = np.random.default_rng(seed)
    x = np.empty((n, gm.dim_x))
    x[:, : gm.nodes] = rng.uniform(-0.3, 1.1, size=(n, gm.nodes))
    x[:, gm.nodes:] = rng.uniform(-0.05, 0.25, size=(n, gm.nodes))
    return x


@pytest.mark.parametrize("n_sub,t", [(50, 1), (50, 37), (1, 5), (3, 1000)])
def test_fhn_fast_philox_matches_generic_kernel(n_sub, t):
    """The bench's kernel (fp32 Philox, fhn_fast_kernel) vs the generic fp32
    kernel on identical keys / counters / gathered inputs."""
    m3, _, obs = orc.fhn_truth(seed=3, n_obs=1)
    gm = pf.FhnLatticeModel(stim_row=m3.stim_row, stim_col=m3.stim_col)
    M, N = 3, 96
    x0 = torch.from_numpy(_random_lattice_states(gm, M * N, 7)).float().cuda()
    anc = torch.from_numpy(np.sort(np.random.default_rng(2).integers(0, M * N, M * N))
                           .astype(np.int32)).cuda()
    fast = fhn_interval(gm, x0, anc, obs[0], M, N, t, n_sub=n_sub)
    gen = fhn_interval(gm, x0, anc, obs[0], M, N, t, n_sub=n_sub, flags=_lib.PF_KERNEL_GENERIC)
    assert norm_rel(fast[0], gen[0]) < 1e-4
    # per-particle state agreement too (one wrong row pair would hide in the norm)
    per = np.linalg.norm(fast[0] - gen[0], axis=1) / np.linalg.norm(gen[0], axis=1)
    assert per.max() < 1e-4, per.max()
    assert norm_rel(fast[1], gen[1]) < 1e-4
    assert np.array_equal(fast[2], gen[2])
    # the noise actually moved the states (not a noise-free run on both sides)
    nf = fhn_interval(gm, x0, anc, obs[0], M, N, t, n_sub=n_sub, noise_free=True)
    assert norm_rel(fast[0], nf[0]) > 1e-3


def _z_checks(z, label, zmax=5.0):
    """z: (n_samples, n_vars) draws that must be iid N(0,1) per column."""
    n = z.shape[0]
    mean = z.mean(axis=0)
    var = z.var(axis=0, ddof=1)
    # per-column mean and variance z-scores (var of the sample variance = 2/(n-1))
    zm = np.abs(mean) * np.sqrt(n)
    zv = np.abs(var - 1.0) / np.sqrt(2.0 / (n - 1))
    assert zm.max() < zmax + 1.0, (label, "mean", zm.max())
    assert zv.max() < zmax + 1.0, (label, "var", zv.max())
    # pooled: mean, variance, kurtosis (3 for a Gaussian), tails
    pooled = z.reshape(-1)
    P = pooled.size
    assert abs(pooled.mean()) * np.sqrt(P) < zmax, (label, "pooled mean")
    assert abs(pooled.var() - 1.0) / np.sqrt(2.0 / P) < zmax, (label, "pooled var")
    kurt = (pooled ** 4).mean() / pooled.var() ** 2
    assert abs(kurt - 3.0) / np.sqrt(24.0 / P) < zmax, (label, "kurtosis", kurt)
    from scipy import stats

    for q in (1.0, 2.0, 3.0):
        p = 2 * stats.norm.sf(q)
        frac = np.mean(np.abs(pooled) > q)
        assert abs(frac - p) / np.sqrt(p * (1 - p) / P) < zmax, (label, "tail", q, frac, p)
    ks = stats.kstest(pooled[: 1 << 20], "norm")
    assert ks.pvalue > 1e-6, (label, "KS", ks)


def _corr(a, b):
    a = a - a.mean(axis=0)
    b = b - b.mean(axis=0)
    return (a * b).sum(axis=0) / np.sqrt((a * a).sum(axis=0) * (b * b).sum(axis=0))


@pytest.mark.parametrize("dtype,flags", [(torch.float32, 0),
                                         (torch.float32, _lib.PF_KERNEL_GENERIC),
                                         (torch.float64, 0)])
def test_fhn_one_step_noise_law(dtype, flags):
    """One Euler step from a fixed state: (noisy - noise-free) / sig_sqdt is
    iid N(0,1) per node for v and w; rows sharing a Philox block, v vs w and
    successive steps are uncorrelated."""
    m3, _, obs = orc.fhn_truth(seed=3, n_obs=1)
    gm = pf.FhnLatticeModel(stim_row=m3.stim_row, stim_col=m3.stim_col)
    M, N = 2, 8192
    x1 = _random_lattice_states(gm, 1, 11)
    x0 = torch.from_numpy(np.repeat(x1, M * N, axis=0)).to(dtype).cuda()
    K, sig = gm.nodes, gm.sig_sqdt
    det = fhn_interval(gm, x0, None, obs[0], M, N, 1, n_sub=1, flags=flags, noise_free=True)[0]
    draws = []
    for t in (1, 2):
        xs = fhn_interval(gm, x0, None, obs[0], M, N, t, n_sub=1, flags=flags)[0]
        d = (xs - det) / sig
        draws.append((d[:, :K], d[:, K:]))
    (zv, zw), (zv2, _) = draws
    _z_checks(zv, "v")
    _z_checks(zw, "w")
    n = zv.shape[0]
    bound = 5.0 / np.sqrt(n)
    # v/w of the same node, the two rows of a Philox row pair, vertical and
    # horizontal neighbours, and the same node at the next step
    rows, cols = gm.rows, gm.cols
    zv3 = zv.reshape(n, rows, cols)
    pairs = {
        "v~w": (zv, zw),
        "row pair": (zv3[:, 0::2, :].reshape(n, -1), zv3[:, 1::2, :].reshape(n, -1)),
        "vertical (across pairs)": (zv3[:, 1:-1:2, :].reshape(n, -1),
                                    zv3[:, 2::2, :].reshape(n, -1)),
        "horizontal": (zv3[:, :, :-1].reshape(n, -1), zv3[:, :, 1:].reshape(n, -1)),
        "t vs t+1": (zv, zv2),
    }
    for name, (a, b) in pairs.items():
        c = _corr(a, b)  # one correlation per column, each ~ N(0, 1/n)
        assert np.abs(c).max() < 1.1 * bound, (name, np.abs(c).max())
        assert abs(c.mean()) < 5.0 / np.sqrt(n * c.size), (name, c.mean())
    # particles j and j+1 (Philox counter word c0)
    c = _corr(zv[0::2], zv[1::2])
    assert np.abs(c).max() < 5.5 / np.sqrt(n / 2)


@pytest.mark.parametrize("M,N,dtype", [(512, 1024, torch.float32),   # block-uniform key kernel
                                       (512, 1000, torch.float32),   # per-thread key
                                       (512, 1024, torch.float64),   # fp64 thread kernel
                                       (16, 1000, torch.float64)])   # fp64 warp-per-particle
def test_lorenz_one_substep_noise_law(M, N, dtype):
    """Lorenz production kernels (fp32 fast, fp64 thread and small-bank warp
    kernels), one substep: (noisy - noise-free) / (noise_scale * sqrt(dt)) is
    iid N(0, 1) per coordinate, uncorrelated across coordinates, successive
    observation times and neighbouring particles."""
    truth0, _, obs = orc.lorenz_truth(seed=8, n_obs=2)
    MN = M * N
    base = dict(substeps=1, obs_var=2.0, observe="x1x3", prior_mean=tuple(truth0))
    gm = pf.Lorenz63Model(noise_scale=0.5, **base)
    g0 = pf.Lorenz63Model(noise_scale=0.0, **base)
    rng = np.random.default_rng(3)
    pt = np.asarray(truth0) + rng.normal(size=3)
    x0 = torch.from_numpy(np.repeat(pt[:, None], MN, axis=1)).to(dtype).cuda().contiguous()
    code = _lib.PF_F32 if dtype == torch.float32 else _lib.PF_F64
    keys = torch.from_numpy(pf.philox.filter_keys(9, M).view(np.int32)).cuda()
    dy = torch.from_numpy(obs[0].copy()).cuda()

    def run(model, t):
        xo = torch.empty_like(x0)
        lw = torch.empty(MN, dtype=dtype, device="cuda")
        st = torch.zeros(M, dtype=torch.int32, device="cuda")
        _lib.call("pf_lorenz_propagate_weight_ex", model.params(), code, _lib.ptr(x0),
                  None, _lib.ptr(xo), _lib.ptr(dy), _lib.ptr(lw), M, N, _lib.ptr(keys), t, None,
                  _lib.ptr(st), 0, _lib.stream_ptr())
        torch.cuda.synchronize()
        return xo.cpu().numpy().astype(np.float64).T  # (MN, 3)

    det = run(g0, 1)
    sig = 0.5 * np.sqrt(gm.dt)
    z1 = (run(gm, 1) - det) / sig
    z2 = (run(gm, 2) - det) / sig
    # the fp32 state near |x| ~ 30 carries ~2e-6 absolute rounding: 1e-4 of sig
    _z_checks(z1, f"lorenz {dtype}")
    n = z1.shape[0]
    for name, (a, b) in {"x1~x2": (z1[:, :1], z1[:, 1:2]), "x2~x3": (z1[:, 1:2], z1[:, 2:]),
                         "t vs t+1": (z1, z2),
                         "p vs p+1": (z1[0::2], z1[1::2])}.items():
        c = _corr(a, b)
        assert np.abs(c).max() < 5.0 / np.sqrt(a.shape[0]), (name, c)


@pytest.mark.parametrize("flags", [_lib.PF_KERNEL_ALT, _lib.PF_KERNEL_PACKED])
@pytest.mark.parametrize("n_sub,t", [(50, 1), (3, 9), (1, 2)])
def test_fhn_column_major_kernel_bit_identical_to_row_major(n_sub, t, flags):
    """The production lattice kernel's column-major strip slots
    (fhn_cm_kernel) and the row-major plane (fhn_fast_kernel, PF_KERNEL_ALT)
    run the same draws and arithmetic: bit-identical states and flags, log
    weights to fp32 rounding (the electrode sum is taken in another fp64
    order).  So does the same kernel issued on packed fp32 pairs
    (PF_KERNEL_PACKED: FFMA2/FADD2/FMUL2) instead of scalar instructions."""
    m3, _, obs = orc.fhn_truth(seed=3, n_obs=1)
    gm = pf.FhnLatticeModel(stim_row=m3.stim_row, stim_col=m3.stim_col)
    M, N = 3, 80
    x0 = torch.from_numpy(_random_lattice_states(gm, M * N, 5)).float().cuda()
    anc = torch.from_numpy(np.sort(np.random.default_rng(4).integers(0, M * N, M * N))
                           .astype(np.int32)).cuda()
    a = fhn_interval(gm, x0, anc, obs[0], M, N, t, n_sub=n_sub)
    b = fhn_interval(gm, x0, anc, obs[0], M, N, t, n_sub=n_sub, flags=flags)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[2], b[2])
    if flags == _lib.PF_KERNEL_PACKED:
        assert np.array_equal(a[1], b[1])
    else:
        # the column-major kernel sums the electrode residuals per owning
        # thread (fp64, another order): equal to fp32 rounding
        assert np.allclose(a[1], b[1], rtol=2.5e-7, atol=0), np.abs(a[1] / b[1] - 1).max()


@pytest.mark.parametrize("case", ["dups_edges", "many", "one"])
@pytest.mark.parametrize("n_sub", [50, 1, 0])
def test_fhn_column_major_electrode_sum_any_electrode_set(case, n_sub):
    """The production kernel sums each electrode's residual in the thread
    that owns the node (tables built once per CTA).  Electrode sets other
    than the BASELINE 10x10 subgrid - duplicated nodes, lattice corners and
    strip-boundary rows, 128 random nodes, a single one - and the no-step
    interval give the same log weights as the generic kernel (which walks
    the electrodes in order over the new plane)."""
    m3, _, obs = orc.fhn_truth(seed=3, n_obs=1)
    gm = pf.FhnLatticeModel(stim_row=m3.stim_row, stim_col=m3.stim_col)
    rng = np.random.default_rng(11)
    nodes = gm.rows * gm.cols
    idx = {"dups_edges": np.array([0, 49, 1450, 1499, 5 * 50 + 7, 6 * 50 + 7, 0, 1499, 0,
                                   11 * 50 + 20, 12 * 50 + 20, 777]),
           "many": rng.integers(0, nodes, 128),  # the ABI's maximum, duplicates likely
           "one": np.array([6 * 50 + 3])}[case].astype(np.int32)
    y = rng.uniform(-0.2, 1.0, idx.size)
    M, N = 2, 64
    x0 = torch.from_numpy(_random_lattice_states(gm, M * N, 9)).float().cuda()
    anc = torch.arange(M * N, dtype=torch.int32, device="cuda")
    res = []
    for flags in (0, _lib.PF_KERNEL_GENERIC):
        xo = torch.empty_like(x0)
        lw = torch.empty(M * N, dtype=torch.float32, device="cuda")
        st = torch.zeros(M, dtype=torch.int32, device="cuda")
        keys = torch.from_numpy(pf.philox.filter_keys(5, M).view(np.int32)).cuda()
        p = gm.params(n_sub=n_sub)
        p.n_obs = int(idx.size)
        d_idx = torch.from_numpy(idx.copy()).cuda()
        d_y = torch.from_numpy(y.copy()).cuda()
        _lib.call("pf_fhn_interval_ex", p, _lib.PF_F32, _lib.ptr(x0), _lib.ptr(anc), _lib.ptr(xo),
                  _lib.ptr(d_y), _lib.ptr(d_idx), _lib.ptr(lw), M, N, _lib.ptr(keys), 3, None,
                  _lib.ptr(st), flags, _lib.stream_ptr())
        torch.cuda.synchronize()
        res.append((xo.cpu().numpy().astype(np.float64), lw.cpu().numpy().astype(np.float64),
                    st.cpu().numpy()))
    (xa, la, sa), (xb, lb, sb) = res
    assert norm_rel(xa, xb) < 1e-4
    assert np.array_equal(sa, sb) and not sa.any()
    assert np.allclose(la, lb, rtol=1e-4, atol=0), np.abs(la / lb - 1).max()
    if n_sub == 0:  # no Euler step: the log weight of the gathered input itself
        v = x0.cpu().numpy().astype(np.float64)[:, idx]
        want = -0.5 / gm.obs_var * ((y[None, :] - v) ** 2).sum(axis=1)
        assert np.allclose(la, want, rtol=1e-6, atol=0)
