"""L1 operator drop-ins for parpf/accel.py, backed by libpfbank (sm_100a).

Same names, argument meaning and return conventions as the reference
kernels (pure functions: inputs are not mutated, outputs freshly allocated,
fp64 in/out, accel.py:60-203).  A maintainer can rebind the reference's
module-level names to these; there is exactly one backend.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def backend_name() -> str:
    return "cuda-sm_100a"


def _t():
    import torch

    _lib.require_cuda()
    return torch


def lorenz_euler_block(states, noise, dt, s, r, b):
    """accel.lorenz_euler_block (accel.py:60-102): bit-exact fp64."""
    torch = _t()
    st = np.ascontiguousarray(states, dtype=np.float64)
    nz = np.ascontiguousarray(noise, dtype=np.float64)
    if st.ndim != 2 or st.shape[1] != 3 or nz.ndim != 3 or nz.shape[1:] != st.shape:
        raise ValueError("states must be (n,3) and noise (n_sub,n,3)")
    d_st = torch.from_numpy(st).cuda()
    d_nz = torch.from_numpy(nz).cuda()
    out = torch.empty_like(d_st)
    _lib.call("pf_op_lorenz_euler_block", _lib.ptr(d_st), _lib.ptr(d_nz), st.shape[0],
              nz.shape[0], float(dt), float(s), float(r), float(b), _lib.ptr(out),
              _lib.stream_ptr())
    return out.cpu().numpy()


def fhn_euler_block(U, V, drive, noise, dt, coupling, cubic, beta, sig_sqdt):
    """accel.fhn_euler_block (accel.py:110-167), any (n, J1, J2) lattice."""
    torch = _t()
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (U, V, drive, noise)]
    shape = arrs[0].shape
    if len(shape) != 3 or any(a.shape != shape for a in arrs):
        raise ValueError("U, V, drive, noise must share one (n, J1, J2) shape")
    d = [torch.from_numpy(a).cuda() for a in arrs]
    un = torch.empty_like(d[0])
    vn = torch.empty_like(d[0])
    cub, cub_p = _lib.host_f64(cubic)
    bet, bet_p = _lib.host_f64(beta)
    _lib.call("pf_op_fhn_euler_block", *[_lib.ptr(x) for x in d], shape[0], shape[1], shape[2],
              float(dt), float(coupling), cub_p, bet_p, float(sig_sqdt), _lib.ptr(un),
              _lib.ptr(vn), _lib.stream_ptr())
    return un.cpu().numpy(), vn.cpu().numpy()


def resample_indices(cum_weights, u_sorted):
    """accel.resample_indices (accel.py:175-203): int64 ancestors."""
    torch = _t()
    cum = np.ascontiguousarray(cum_weights, dtype=np.float64)
    u = np.ascontiguousarray(u_sorted, dtype=np.float64)
    d_c = torch.from_numpy(cum).cuda()
    d_u = torch.from_numpy(u).cuda()
    out = torch.empty(u.shape[0], dtype=torch.int64, device="cuda")
    _lib.call("pf_op_resample_indices", _lib.ptr(d_c), cum.shape[0], _lib.ptr(d_u), u.shape[0],
              _lib.ptr(out), _lib.stream_ptr())
    return out.cpu().numpy()
