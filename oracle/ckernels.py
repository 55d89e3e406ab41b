"""TEST INFRASTRUCTURE / CPU BASELINE ONLY: ctypes binding of the oracle's C
kernels (oracle/_build/libpforacle.so, built by `make -C oracle`).

``install()`` rebinds the oracle's module-level kernels to the C versions,
the same way the reference selects numba twins at import (accel.py:206-213);
results stay bit-identical (tests/test_oracle_golden.py::test_ckernels_*).
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import parpf_oracle as orc

_HERE = os.path.dirname(os.path.abspath(__file__))
_PATH = os.path.join(_HERE, "_build", "libpforacle.so")
_lib = None
_vp, _i64, _f64 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double


def load():
    global _lib
    if _lib is None:
        if not os.path.exists(_PATH):
            raise FileNotFoundError(f"{_PATH} missing: run `make -C oracle`")
        lib = ctypes.CDLL(_PATH)
        lib.orc_lorenz_euler_block.argtypes = [_vp, _vp, _i64, _i64, _f64, _f64, _f64, _f64, _vp]
        lib.orc_fhn_euler_block.argtypes = [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _f64, _f64,
                                            _vp, _vp, _f64, _vp, _vp]
        lib.orc_resample_indices.argtypes = [_vp, _i64, _vp, _i64, _vp]
        for f in (lib.orc_lorenz_euler_block, lib.orc_fhn_euler_block, lib.orc_resample_indices):
            f.restype = None
        _lib = lib
    return _lib


def _p(a):
    return a.ctypes.data_as(_vp)


def lorenz_euler_block(states, noise, dt, s, r, b):
    st = np.ascontiguousarray(states, dtype=np.float64)
    nz = np.ascontiguousarray(noise, dtype=np.float64)
    out = np.empty_like(st)
    load().orc_lorenz_euler_block(_p(st), _p(nz), st.shape[0], nz.shape[0], dt, s, r, b, _p(out))
    return out


def fhn_euler_block(U, V, drive, noise, dt, coupling, cubic, beta, sig_sqdt):
    arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (U, V, drive, noise)]
    n, J1, J2 = arrs[0].shape
    un = np.empty_like(arrs[0])
    vn = np.empty_like(arrs[0])
    cub = np.ascontiguousarray(cubic, dtype=np.float64)
    bet = np.ascontiguousarray(beta, dtype=np.float64)
    load().orc_fhn_euler_block(*[_p(a) for a in arrs], n, J1, J2, dt, coupling, _p(cub), _p(bet),
                               sig_sqdt, _p(un), _p(vn))
    return un, vn


def resample_indices(cum_weights, u_sorted):
    cum = np.ascontiguousarray(cum_weights, dtype=np.float64)
    u = np.ascontiguousarray(u_sorted, dtype=np.float64)
    idx = np.empty(u.shape[0], dtype=np.int64)
    load().orc_resample_indices(_p(cum), cum.shape[0], _p(u), u.shape[0], _p(idx))
    return idx


def install():
    """Rebind the oracle's kernels to the C versions (numba-twin analogue)."""
    load()
    orc.lorenz_euler_block = lorenz_euler_block
    orc.fhn_euler_block = fhn_euler_block
    orc.resample_indices = resample_indices
