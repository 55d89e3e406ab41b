"""Resampling drop-in for parpf/resampling.py:10-72 (hook level).

Consumes the caller's numpy Generator exactly like the reference
(multinomial: n_out + 1 standard exponentials, resampling.py:24; systematic:
one uniform, :65), so the caller's stream advances identically; the CDF, the
order statistics / thresholds and the merge run on the GPU in numpy's
floating-point order (sequential cumsum, IEEE division), so the indices are
the reference's.  The bank path (pf_segmented_resample) fuses all of this
per filter.
"""

from __future__ import annotations

import numpy as np

from . import _lib


def _check_weights(weights):
    """resampling.py:10-18."""
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or w.shape[0] < 1:
        raise ValueError("weights must be a non-empty 1-d array")
    if np.any(w < 0.0):
        raise ValueError("weights must be non-negative")
    if abs(w.sum() - 1.0) > 1e-8:
        raise ValueError("weights must be normalised to sum 1")
    return w


def _merge(w, u):
    """searchsorted-left of u in cumsum(w), clamped (accel.py:175-203)."""
    import torch

    cum = torch.empty(w.shape[0], dtype=torch.float64, device="cuda")
    d_w = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    s = _lib.stream_ptr()
    _lib.call("pf_op_cumsum", _lib.ptr(d_w), w.shape[0], _lib.ptr(cum), s)
    idx = torch.empty(u.shape[0], dtype=torch.int64, device="cuda")
    _lib.call("pf_op_resample_indices", _lib.ptr(cum), w.shape[0], _lib.ptr(u), u.shape[0],
              _lib.ptr(idx), s)
    return idx.cpu().numpy()


def multinomial_resample_indices(weights, n_out: int, rng) -> np.ndarray:
    """resampling.py:29-43: cum = cumsum(w); u = sorted uniforms from n_out+1
    exponential spacings; smallest k with cum[k] >= u."""
    import torch

    w = _check_weights(weights)
    if n_out < 1:
        raise ValueError("n_out must be >= 1")
    _lib.require_cuda()
    e = torch.from_numpy(np.ascontiguousarray(rng.standard_exponential(n_out + 1))).cuda()
    work = torch.empty(n_out + 1, dtype=torch.float64, device="cuda")
    u = torch.empty(n_out, dtype=torch.float64, device="cuda")
    _lib.call("pf_op_spacing_uniforms", _lib.ptr(e), n_out, _lib.ptr(work), _lib.ptr(u),
              _lib.stream_ptr())
    return _merge(w, u)


def systematic_resample_indices(weights, n_out: int, rng) -> np.ndarray:
    """resampling.py:53-66: one shared uniform r, thresholds (i + r) / n_out.
    (Opt-in; the verification suite's guarantees are for multinomial.)"""
    import torch

    w = _check_weights(weights)
    if n_out < 1:
        raise ValueError("n_out must be >= 1")
    _lib.require_cuda()
    u = torch.empty(n_out, dtype=torch.float64, device="cuda")
    _lib.call("pf_op_systematic_uniforms", float(rng.random()), n_out, _lib.ptr(u),
              _lib.stream_ptr())
    return _merge(w, u)


def multinomial_resample(particles, weights, n_out: int, rng) -> np.ndarray:
    """resampling.py:46-50 (the row selection is plain indexing of the
    caller's host array)."""
    return np.asarray(particles)[multinomial_resample_indices(weights, n_out, rng)]


def systematic_resample(particles, weights, n_out: int, rng) -> np.ndarray:
    """resampling.py:69-72."""
    return np.asarray(particles)[systematic_resample_indices(weights, n_out, rng)]
