"""Memory-safety and race checks of our own for the shared-memory kernels
(complementing compute-sanitizer, which some GPU pools disable):

* guard bands: every output buffer sits inside a larger allocation whose
  head and tail are filled with a canary pattern; after the launch the
  canaries, and every input buffer, must be byte-identical (no
  out-of-bounds global write, no write to an input);
* repeat determinism: the same launch repeated many times gives
  bit-identical outputs (a shared-memory race or an uninitialised read
  shows up as run-to-run differences);
* odd shapes: particle counts that leave partial warps / tiles.

Kernels: fhn_fast_kernel (production + tape), the generic FH-N kernel,
resample_bank_kernel (fused gather), the wide resampler pipeline
(wide2_* incl. wide2_merge), fhnnet_fast_kernel, lorenz_fast_kernel."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import _lib  # noqa: E402

GUARD = 4096  # bytes of canary on each side


class Guarded:
    """A device buffer of `numel` elements inside canary bands."""

    def __init__(self, numel, dtype, fill=None):
        item = torch.empty(0, dtype=dtype).element_size()
        g = GUARD // item
        self.raw = torch.empty(numel + 2 * g, dtype=dtype, device="cuda")
        self.raw.view(torch.uint8).fill_(0xA5)
        self.t = self.raw[g:g + numel]
        if fill is not None:
            self.t.copy_(fill.reshape(-1).to(dtype))
        self.g = g

    def canaries_intact(self):
        b = self.raw.view(torch.uint8)
        n = self.g * self.raw.element_size()
        return bool((b[:n] == 0xA5).all() and (b[-n:] == 0xA5).all())


def _keys(M):
    return torch.from_numpy(pf.philox.filter_keys(3, M).view(np.int32)).cuda()


def _snap(*ts):
    return [t.clone() for t in ts]


def _same(a, b):
    return all(torch.equal(x, y) for x, y in zip(a, b))


def _fhn(M, N, flags, tape):
    gm = pf.FhnLatticeModel()
    rng = np.random.default_rng(M * 31 + N)
    x = Guarded(M * N * gm.dim_x, torch.float32,
                torch.from_numpy(rng.uniform(-0.2, 1.0, M * N * gm.dim_x)))
    xo = Guarded(M * N * gm.dim_x, torch.float32)
    anc = Guarded(M * N, torch.int32,
                  torch.from_numpy(np.sort(rng.integers(0, M * N, M * N)).astype(np.int32)))
    lw = Guarded(M * N, torch.float32)
    st = Guarded(M, torch.int32, torch.zeros(M))
    y = torch.from_numpy(rng.normal(size=gm.dim_y)).cuda()
    idx = torch.from_numpy(gm.obs_indices.astype(np.int32)).cuda()
    z = None
    if tape:
        z = Guarded(M * 3 * 2 * N * gm.nodes, torch.float64,
                    torch.from_numpy(rng.normal(size=M * 3 * 2 * N * gm.nodes)))

    def launch():
        st.t.zero_()  # status flags accumulate (atomicOr)
        _lib.call("pf_fhn_interval_ex", gm.params(n_sub=3), _lib.PF_F32, _lib.ptr(x.t),
                  _lib.ptr(anc.t), _lib.ptr(xo.t), _lib.ptr(y), _lib.ptr(idx), _lib.ptr(lw.t),
                  M, N, _lib.ptr(_keys(M)), 2, _lib.ptr(z.t if z else None), _lib.ptr(st.t),
                  flags, _lib.stream_ptr())

    inputs = [x, anc] + ([z] if z else [])
    return launch, inputs, [xo, lw, st]


def _resample(M, N):
    rng = np.random.default_rng(N)
    lw = Guarded(M * N, torch.float32,
                 torch.from_numpy((rng.normal(size=M * N) * 3).astype(np.float32)))
    x = Guarded(3 * M * N, torch.float32, torch.from_numpy(rng.normal(size=3 * M * N)))
    xo = Guarded(3 * M * N, torch.float32)
    anc = Guarded(M * N, torch.int32)
    lnc = Guarded(M, torch.float64, torch.zeros(M))
    coll = Guarded(M, torch.uint8, torch.zeros(M))
    st = Guarded(M, torch.int32, torch.zeros(M))
    wsb = int(_lib.load().pf_resample_workspace_bytes(M, N))
    ws = Guarded(max(wsb, 1), torch.uint8)

    def launch():
        for acc in (lnc, coll, st):  # lnc accumulates, flags are OR-ed
            acc.t.zero_()
        _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(lw.t), M, N, None,
                  _lib.ptr(_keys(M)), 1, _lib.ptr(anc.t), _lib.ptr(lnc.t), _lib.ptr(coll.t),
                  _lib.ptr(st.t), _lib.ptr(ws.t), wsb, _lib.ptr(x.t), _lib.ptr(xo.t), 3, 0,
                  _lib.stream_ptr())

    return launch, [lw, x], [xo, anc, lnc, coll, st, ws]


def _fhnnet(M, N):
    gm = pf.FhnNetworkModel(J=8, n_zones=2, zone_width=2, stim_prob=0.3)
    rng = np.random.default_rng(2)
    x0 = np.zeros((M * N, gm.dim_x))
    x0[:, : gm.nodes] = rng.uniform(-2.0, 2.0, size=(M * N, gm.nodes))
    xd, qd = gm.to_device(x0, dtype=torch.float32)
    x = Guarded(xd.numel(), torch.float32, xd)
    q = Guarded(qd.numel(), torch.int32, qd.view(torch.int32))
    xo = Guarded(xd.numel(), torch.float32)
    qo = Guarded(qd.numel(), torch.int32)
    anc = Guarded(M * N, torch.int32,
                  torch.from_numpy(rng.integers(0, M * N, M * N).astype(np.int32)))
    lw = Guarded(M * N, torch.float32)
    st = Guarded(M, torch.int32, torch.zeros(M))
    y = torch.from_numpy(rng.normal(size=gm.dim_y)).cuda()
    idx = torch.from_numpy(gm.obs_indices.astype(np.int32)).cuda()
    mask = gm.device_mask()

    def launch():
        st.t.zero_()
        _lib.call("pf_fhnnet_step_ex", gm.params(), _lib.PF_F32, _lib.ptr(x.t), _lib.ptr(q.t),
                  _lib.ptr(anc.t), _lib.ptr(xo.t), _lib.ptr(qo.t), _lib.ptr(mask), _lib.ptr(y),
                  _lib.ptr(idx), _lib.ptr(lw.t), M, N, _lib.ptr(_keys(M)), 7, None, None,
                  _lib.ptr(st.t), 0, _lib.stream_ptr())

    return launch, [x, q, anc], [xo, qo, lw, st]


def _lorenz(M, N):
    gm = pf.Lorenz63Model(substeps=40, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=(1.0, 2.0, 20.0), prior_var=1.0)
    rng = np.random.default_rng(5)
    x = Guarded(3 * M * N, torch.float32,
                torch.from_numpy(rng.normal(size=3 * M * N) + 10.0))
    xo = Guarded(3 * M * N, torch.float32)
    anc = Guarded(M * N, torch.int32,
                  torch.from_numpy(rng.integers(0, M * N, M * N).astype(np.int32)))
    lw = Guarded(M * N, torch.float32)
    st = Guarded(M, torch.int32, torch.zeros(M))
    y = torch.tensor([1.0, 20.0], dtype=torch.float64, device="cuda")

    def launch():
        st.t.zero_()
        _lib.call("pf_lorenz_propagate_weight_ex", gm.params(), _lib.PF_F32, _lib.ptr(x.t),
                  _lib.ptr(anc.t), _lib.ptr(xo.t), _lib.ptr(y), _lib.ptr(lw.t), M, N,
                  _lib.ptr(_keys(M)), 3, None, _lib.ptr(st.t), 0, _lib.stream_ptr())

    return launch, [x, anc], [xo, lw, st]


CASES = {
    "fhn_fast": lambda: _fhn(3, 5, 0, False),
    "fhn_fast_tape": lambda: _fhn(2, 3, 0, True),
    "fhn_generic": lambda: _fhn(2, 7, _lib.PF_KERNEL_GENERIC, False),
    "resample_bank": lambda: _resample(7, 1000),
    "resample_bank_ragged": lambda: _resample(5, 777),
    "resample_wide": lambda: _resample(1, 20001),
    "resample_wide_multi": lambda: _resample(3, 70001),
    "fhnnet_fast": lambda: _fhnnet(3, 5),
    "lorenz_fast": lambda: _lorenz(3, 1024),
    "lorenz_fast_ragged": lambda: _lorenz(3, 1000),
}


@pytest.mark.parametrize("name", sorted(CASES))
def test_guard_bands_inputs_and_determinism(name):
    launch, inputs, outputs = CASES[name]()
    torch.cuda.synchronize()
    before = _snap(*[b.raw for b in inputs])
    launch()
    torch.cuda.synchronize()
    first = _snap(*[b.t for b in outputs])
    for b in outputs + inputs:
        assert b.canaries_intact(), f"{name}: write outside a buffer"
    assert _same(before, [b.raw for b in inputs]), f"{name}: an input was modified"
    for rep in range(25):
        for b in outputs:
            b.t.view(torch.uint8).fill_(rep * 7 % 251)  # stale data must not leak through
        launch()
        torch.cuda.synchronize()
        # the workspace is scratch: compare the results only
        res = [b.t for b in outputs]
        if name.startswith("resample"):
            res, ref = res[:-1], first[:-1]
        else:
            ref = first
        assert _same(ref, res), f"{name}: run {rep} differs from run 0 (race / uninitialised read)"
        for b in outputs:
            assert b.canaries_intact()
