"""Multinomial resampling drop-in for parpf/resampling.py:29-50.

Consumes the caller's numpy Generator exactly like the reference (n_out+1
standard exponentials, resampling.py:24), so the caller's stream advances
identically; the CDF, the order statistics and the merge run on the GPU.
The bank path (pf_segmented_resample) fuses all of this per filter.
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


def multinomial_resample_indices(weights, n_out: int, rng) -> np.ndarray:
    import torch

    w = _check_weights(weights)
    if n_out < 1:
        raise ValueError("n_out must be >= 1")
    _lib.require_cuda()
    cum = torch.cumsum(torch.from_numpy(w).cuda(), 0)
    e = rng.standard_exponential(n_out + 1)
    c = torch.cumsum(torch.from_numpy(np.ascontiguousarray(e)).cuda(), 0)
    u = (c[:n_out] / c[n_out]).contiguous()
    idx = torch.empty(n_out, dtype=torch.int64, device="cuda")
    _lib.call("pf_op_resample_indices", _lib.ptr(cum), w.shape[0], _lib.ptr(u), n_out,
              _lib.ptr(idx), _lib.stream_ptr())
    return idx.cpu().numpy()


def multinomial_resample(particles, weights, n_out: int, rng) -> np.ndarray:
    import torch

    idx = multinomial_resample_indices(weights, n_out, rng)
    x = torch.from_numpy(np.ascontiguousarray(particles)).cuda()
    return x[torch.from_numpy(idx).cuda()].cpu().numpy()
