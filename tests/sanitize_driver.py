"""TEST HELPER (run under compute-sanitizer by tests/test_gpu_sanitize.py):
one small launch of a shared-memory kernel through the C ABI.

    python tests/sanitize_driver.py {fhn|fhn_tape|resample_bank|wide|fhnnet|lorenz}
"""

import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

import paper_1407_8071_b200 as pf  # noqa: E402
from paper_1407_8071_b200 import _lib  # noqa: E402


def _keys(M):
    return torch.from_numpy(pf.philox.filter_keys(3, M).view(np.int32)).cuda()


def fhn(tape=False):
    gm = pf.FhnLatticeModel()
    M, N = 2, 3
    rng = np.random.default_rng(0)
    x = torch.from_numpy(rng.uniform(-0.2, 1.0, (M * N, gm.dim_x))).float().cuda()
    xo = torch.empty_like(x)
    anc = torch.tensor([2, 0, 1, 5, 5, 3], dtype=torch.int32, device="cuda")
    y = torch.from_numpy(rng.normal(size=gm.dim_y)).cuda()
    idx = torch.from_numpy(gm.obs_indices.astype(np.int32)).cuda()
    lw = torch.empty(M * N, dtype=torch.float32, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    z = None
    if tape:
        z = torch.from_numpy(rng.normal(size=(M, 3, 2, N, gm.nodes))).cuda()
    _lib.call("pf_fhn_interval_ex", gm.params(n_sub=3), _lib.PF_F32, _lib.ptr(x), _lib.ptr(anc),
              _lib.ptr(xo), _lib.ptr(y), _lib.ptr(idx), _lib.ptr(lw), M, N, _lib.ptr(_keys(M)),
              1, _lib.ptr(z), _lib.ptr(st), 0, _lib.stream_ptr())


def _resample(M, N):
    rng = np.random.default_rng(1)
    lw = torch.from_numpy((rng.normal(size=M * N) * 3).astype(np.float32)).cuda()
    x = torch.from_numpy(rng.normal(size=(3, M * N)).astype(np.float32)).cuda()
    xo = torch.empty_like(x)
    anc = torch.empty(M * N, dtype=torch.int32, device="cuda")
    lnc = torch.zeros(M, dtype=torch.float64, device="cuda")
    coll = torch.zeros(M, dtype=torch.uint8, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    wsb = _lib.load().pf_resample_workspace_bytes(M, N)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    _lib.call("pf_segmented_resample_ex", _lib.PF_F32, _lib.ptr(lw), M, N, None,
              _lib.ptr(_keys(M)), 1, _lib.ptr(anc), _lib.ptr(lnc), _lib.ptr(coll), _lib.ptr(st),
              _lib.ptr(ws), wsb, _lib.ptr(x), _lib.ptr(xo), 3, 0, _lib.stream_ptr())


def fhnnet():
    gm = pf.FhnNetworkModel(J=8, n_zones=2, zone_width=2, stim_prob=0.3)
    M, N = 2, 5
    rng = np.random.default_rng(2)
    x0 = np.zeros((M * N, gm.dim_x))
    x0[:, : gm.nodes] = rng.uniform(-2.0, 2.0, size=(M * N, gm.nodes))
    x, q = gm.to_device(x0, dtype=torch.float32)
    xo, qo = torch.empty_like(x), torch.empty_like(q)
    anc = torch.from_numpy(rng.integers(0, M * N, M * N).astype(np.int32)).cuda()
    y = torch.from_numpy(rng.normal(size=gm.dim_y)).cuda()
    idx = torch.from_numpy(gm.obs_indices.astype(np.int32)).cuda()
    lw = torch.empty(M * N, dtype=torch.float32, device="cuda")
    st = torch.zeros(M, dtype=torch.int32, device="cuda")
    _lib.call("pf_fhnnet_step_ex", gm.params(), _lib.PF_F32, _lib.ptr(x), _lib.ptr(q),
              _lib.ptr(anc), _lib.ptr(xo), _lib.ptr(qo), _lib.ptr(gm.device_mask()),
              _lib.ptr(y), _lib.ptr(idx), _lib.ptr(lw), M, N, _lib.ptr(_keys(M)), 7, None, None,
              _lib.ptr(st), 0, _lib.stream_ptr())


def lorenz():
    truth0 = (1.0, 2.0, 20.0)
    gm = pf.Lorenz63Model(substeps=4, obs_var=2.0, noise_scale=0.5, observe="x1x3",
                          prior_mean=truth0, prior_var=1.0)
    obs = np.random.default_rng(3).normal(size=(3, 2))
    pf.run_ensemble(gm, obs, "bootstrap", 2, 256, 4, dtype="float32")


if __name__ == "__main__":
    what = sys.argv[1]
    torch.cuda.set_device(0)
    {"fhn": fhn, "fhn_tape": lambda: fhn(tape=True),
     "resample_bank": lambda: _resample(5, 1000),
     "wide": lambda: _resample(1, 20000),
     "fhnnet": fhnnet, "lorenz": lorenz}[what]()
    torch.cuda.synchronize()
    print("driver ok", what)
