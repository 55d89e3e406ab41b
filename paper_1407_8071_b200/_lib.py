"""ctypes binding of libpfbank.so (the C ABI declared in include/pfbank.h).

The library is built in-tree (``paper_1407_8071_b200/lib/libpfbank.so``) by
``__graft_entry__.build()`` / ``python -m paper_1407_8071_b200._build``.
There is no fallback: if the library is missing or no CUDA device is
visible, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

import numpy as np

from .exceptions import NumericalDivergenceError

LIB_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")
LIB_PATH = os.path.join(LIB_DIR, "libpfbank.so")

PF_OK = 0
PF_EINVAL = -22
PF_ECUDA = -5
PF_ST_DIVERGED = 1
PF_ST_NAN_WEIGHT = 2
PF_RS_REFERENCE_ORDER = 1
PF_RS_WIDE_MERGE_PATH = 2
PF_RS_WIDE_GATHER_SEPARATE = 4
PF_RS_WIDE_RECOMPUTE = 8
PF_KERNEL_GENERIC = 1
PF_KERNEL_ALT = 2
PF_KERNEL_PACKED = 4
PF_F32 = 0
PF_F64 = 1

c_i32, c_i64, c_u32, c_f64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_double
c_vp, c_sz = ctypes.c_void_p, ctypes.c_size_t


class LorenzParams(ctypes.Structure):
    _fields_ = [("s", c_f64), ("r", c_f64), ("b", c_f64), ("dt", c_f64),
                ("noise_scale", c_f64), ("obs_var", c_f64),
                ("n_sub", c_i32), ("obs_dim", c_i32)]


class FhnParams(ctypes.Structure):
    _fields_ = [("rows", c_i32), ("cols", c_i32), ("n_sub", c_i32), ("n_obs", c_i32),
                ("dt", c_f64), ("coupling", c_f64), ("cubic", c_f64 * 4), ("beta", c_f64 * 3),
                ("sig_v", c_f64), ("sig_w", c_f64), ("degree_drive", c_f64),
                ("obs_var", c_f64)]


class FhnNetParams(ctypes.Structure):
    _fields_ = [("J", c_i32), ("stim_hold", c_i32), ("n_obs", c_i32), ("stochastic", c_i32),
                ("dt", c_f64), ("coupling", c_f64), ("cubic", c_f64 * 4), ("beta", c_f64 * 3),
                ("u_minus", c_f64), ("u_plus", c_f64), ("stim_prob", c_f64), ("stim_amp", c_f64),
                ("forcing_amp", c_f64), ("forcing_period", c_f64), ("forcing_width", c_f64),
                ("sig_sqdt", c_f64), ("obs_var", c_f64)]


class HmmParams(ctypes.Structure):
    _fields_ = [("K", c_i32), ("S", c_i32), ("cum_prior", c_vp), ("cum_rows", c_vp),
                ("log_emission", c_vp)]


class LgmParams(ctypes.Structure):
    _fields_ = [("dx", c_i32), ("dy", c_i32), ("noise_free", c_i32), ("reserved", c_i32),
                ("A", c_vp), ("chol_q", c_vp), ("H", c_vp), ("obs_prec", c_vp),
                ("prior_mean", c_vp), ("chol_p0", c_vp), ("obs_logconst", c_f64)]


class IslandDesc(ctypes.Structure):
    _fields_ = [("period", c_i32), ("key", c_vp), ("lw", c_vp), ("lnc_old", c_vp), ("idx", c_vp),
                ("anc_tmp", c_vp), ("lnc_tmp", c_vp), ("coll_tmp", c_vp), ("s_lnc", c_vp),
                ("s_coll", c_vp), ("s_status", c_vp), ("ws", c_vp), ("ws_bytes", c_sz),
                ("pool", c_vp), ("trace", c_vp), ("pool_dim", c_i32)]


class BankDesc(ctypes.Structure):
    _fields_ = [("model", c_i32), ("dtype", ctypes.c_int), ("M", c_i64), ("N", c_i64),
                ("lorenz", ctypes.POINTER(LorenzParams)), ("fhn", ctypes.POINTER(FhnParams)),
                ("obs_idx", c_vp), ("x", c_vp * 2), ("logw", c_vp), ("anc", c_vp), ("lnc", c_vp),
                ("collapsed", c_vp), ("status", c_vp), ("keys", c_vp), ("ws", c_vp),
                ("ws_bytes", c_sz), ("obs", c_vp), ("dim_y", c_i32), ("est", c_vp),
                ("est_step_stride", c_i64), ("est_offset", c_i64), ("est_stride_p", c_i64),
                ("est_stride_d", c_i64), ("est_dim", c_i32), ("lnc_trace", c_vp),
                ("collapsed_trace", c_vp), ("prop_ms", ctypes.POINTER(ctypes.c_float)),
                ("fhnnet", ctypes.POINTER(FhnNetParams)), ("q", c_vp * 2),
                ("forcing_mask", c_vp), ("est_stride_f", c_i64), ("est_bits", c_i32),
                ("hmm", ctypes.POINTER(HmmParams)), ("lgm", ctypes.POINTER(LgmParams)),
                ("step_ms", ctypes.POINTER(ctypes.c_float)), ("events", c_vp),
                ("variant", c_i32), ("params0", c_vp), ("lam", c_vp), ("anc1", c_vp),
                ("anc_comp", c_vp), ("x_tmp", c_vp), ("q_tmp", c_vp), ("lnc_before", c_vp),
                ("coll1", c_vp), ("kernel_flags", c_u32), ("comm", c_vp),
                ("exch_count", c_i64), ("use_graph", c_i32),
                ("islands", ctypes.POINTER(IslandDesc))]


PF_MODEL_LORENZ = 0
PF_MODEL_FHN = 1
PF_MODEL_FHNNET = 2
PF_MODEL_HMM = 3
PF_MODEL_LGM = 4

# name -> (restype, argtypes); must match include/pfbank.h exactly
SIGNATURES = {
    "pf_last_error": (ctypes.c_char_p, []),
    "pf_version": (ctypes.c_int, []),
    "pf_device_sm_count": (ctypes.c_int, [ctypes.POINTER(ctypes.c_int)]),
    "pf_philox_kat": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pf_probe_fp32_fma": (ctypes.c_int, [c_vp, c_i64, c_vp]),
    "pf_op_lorenz_euler_block": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i64, c_f64, c_f64, c_f64,
                                                c_f64, c_vp, c_vp]),
    "pf_op_fhn_euler_block": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32, c_f64,
                                             c_f64, c_vp, c_vp, c_f64, c_vp, c_vp, c_vp]),
    "pf_op_resample_indices": (ctypes.c_int, [c_vp, c_i64, c_vp, c_i64, c_vp, c_vp]),
    "pf_op_normalize_log_weights": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp,
                                                   c_vp, c_vp, c_vp]),
    "pf_op_cumsum": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "pf_op_spacing_uniforms": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pf_op_systematic_uniforms": (ctypes.c_int, [c_f64, c_i64, c_vp, c_vp]),
    "pf_gather_planes": (ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp]),
    "pf_lorenz_prior": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_f64, c_vp, c_vp,
                                       c_vp]),
    "pf_fill_rows": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "pf_lorenz_propagate_weight": (ctypes.c_int, [ctypes.POINTER(LorenzParams), ctypes.c_int,
                                                  c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
                                                  c_vp, c_u32, c_vp, c_vp, c_vp]),
    "pf_lorenz_propagate_weight_ex": (ctypes.c_int, [ctypes.POINTER(LorenzParams), ctypes.c_int,
                                                     c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
                                                     c_vp, c_u32, c_vp, c_vp, c_u32, c_vp]),
    "pf_fhn_interval": (ctypes.c_int, [ctypes.POINTER(FhnParams), ctypes.c_int, c_vp, c_vp, c_vp,
                                       c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_u32, c_vp, c_vp,
                                       c_vp]),
    "pf_fhn_interval_ex": (ctypes.c_int, [ctypes.POINTER(FhnParams), ctypes.c_int, c_vp, c_vp,
                                          c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_u32, c_vp,
                                          c_vp, c_u32, c_vp]),
    "pf_resample_workspace_bytes": (c_sz, [c_i64, c_i64]),
    "pf_estimate_workspace_bytes": (c_sz, [c_i64, c_i64, c_i32]),
    "pf_filter_estimate_ws": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64,
                                             c_i64, c_vp, c_i64, c_vp, c_sz, c_vp]),
    "pf_segmented_resample": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_u32,
                                             c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp]),
    "pf_segmented_resample_ex": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp, c_u32,
                                                c_vp, c_vp, c_vp, c_vp, c_vp, c_sz, c_vp, c_vp,
                                                c_i32, c_u32, c_vp]),
    "pf_filter_estimate": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_i32, c_vp, c_i64,
                                          c_i64, c_vp, c_vp]),
    "pf_filter_estimate_strided": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_i32, c_vp,
                                                  c_i64, c_i64, c_vp, c_i64, c_vp]),
    "pf_fhnnet_step": (ctypes.c_int, [ctypes.POINTER(FhnNetParams), ctypes.c_int, c_vp, c_vp,
                                      c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
                                      c_vp, c_u32, c_vp, c_vp, c_vp, c_vp]),
    "pf_fhnnet_step_ex": (ctypes.c_int, [ctypes.POINTER(FhnNetParams), ctypes.c_int, c_vp, c_vp,
                                         c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64,
                                         c_vp, c_u32, c_vp, c_vp, c_vp, c_u32, c_vp]),
    "pf_fhnnet_pack": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i32, c_i32, c_vp, c_vp, c_vp]),
    "pf_fhnnet_unpack": (ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_i32, c_i32,
                                        c_vp, c_vp]),
    "pf_zone_loglik": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_i32, c_vp, c_f64,
                                      c_vp, c_vp]),
    "pf_bits_estimate": (ctypes.c_int, [c_vp, c_i32, c_i32, c_vp, c_i64, c_i64, c_vp, c_i64,
                                        c_vp]),
    "pf_hmm_prior": (ctypes.c_int, [ctypes.POINTER(HmmParams), ctypes.c_int, c_vp, c_i64, c_i64,
                                    c_vp, c_vp, c_vp]),
    "pf_hmm_propagate_weight": (ctypes.c_int, [ctypes.POINTER(HmmParams), ctypes.c_int, c_vp,
                                               c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_u32,
                                               c_vp, c_vp, c_vp]),
    "pf_hmm_loglik": (ctypes.c_int, [ctypes.POINTER(HmmParams), c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pf_lgm_prior": (ctypes.c_int, [ctypes.POINTER(LgmParams), ctypes.c_int, c_vp, c_i64, c_i64,
                                    c_vp, c_vp, c_vp]),
    "pf_lgm_propagate_weight": (ctypes.c_int, [ctypes.POINTER(LgmParams), ctypes.c_int, c_vp,
                                               c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_u32,
                                               c_vp, c_vp, c_vp]),
    "pf_lgm_loglik": (ctypes.c_int, [ctypes.POINTER(LgmParams), c_vp, c_i64, c_vp, c_vp, c_vp]),
    "pf_island_accumulate": (ctypes.c_int, [c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pf_island_copy": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_vp, c_vp,
                                      c_vp, c_vp]),
    "pf_island_pool": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp]),
    "pf_island_trace": (ctypes.c_int, [c_vp, c_i64, c_vp, c_vp]),
    "pf_bank_run": (ctypes.c_int, [ctypes.POINTER(BankDesc), c_i32, c_i32, c_i32, c_i32, c_vp]),
    "pf_apf_first_stage_prepare": (ctypes.c_int, [ctypes.c_int, c_vp, c_i64, c_i64, c_vp, c_vp]),
    "pf_compose_ancestors": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp, c_vp]),
    "pf_apf_second_stage_weights": (ctypes.c_int, [ctypes.c_int, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pf_apf_finish": (ctypes.c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_vp]),
    "pf_ensemble_average": (ctypes.c_int, [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp]),
    "pf_bank_graph_create": (ctypes.c_int, [ctypes.POINTER(BankDesc), c_i32, c_i32, c_i32, c_i32,
                                            c_vp, ctypes.POINTER(c_vp)]),
    "pf_bank_graph_launch": (ctypes.c_int, [c_vp, c_vp]),
    "pf_bank_graph_destroy": (ctypes.c_int, [c_vp]),
    "pf_comm_available": (ctypes.c_int, []),
    "pf_comm_nccl_version": (ctypes.c_int, []),
    "pf_comm_unique_id": (ctypes.c_int, [c_vp]),
    "pf_comm_init": (ctypes.c_int, [c_vp, c_i32, c_i32, ctypes.POINTER(c_vp)]),
    "pf_comm_destroy": (ctypes.c_int, [c_vp]),
    "pf_comm_allreduce_f64": (ctypes.c_int, [c_vp, c_vp, c_i64, c_vp]),
    "pf_comm_exchange_steps": (ctypes.c_int, [c_vp, c_vp, c_i64, c_i64, c_i32, c_i32, c_vp]),
    "pf_comm_join": (ctypes.c_int, [c_vp, c_vp]),
}

PF_COMM_ID_BYTES = 128

_lock = threading.Lock()
_lib = None


class LibraryMissingError(RuntimeError):
    """libpfbank.so was not built (run __graft_entry__.build())."""


def load():
    """Load and bind libpfbank.so (no GPU needed to load)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise LibraryMissingError(
                    f"{LIB_PATH} not found - build it with `python -c 'import __graft_entry__ as g;"
                    f" g.build()'`; there is no CPU fallback")
            lib = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def call(name, *args):
    """Invoke an ABI entry point and map its status code to an exception."""
    rc = getattr(load(), name)(*args)
    if rc == PF_OK:
        return
    msg = load().pf_last_error().decode(errors="replace")
    if rc == PF_EINVAL:
        raise ValueError(f"{name}: {msg}")
    raise RuntimeError(f"{name} failed ({rc}): {msg}")


def require_cuda():
    """The product path runs on the GPU only; fail loudly otherwise."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_1407_8071_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    load()


def stream_ptr(stream=None):
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def ptr(t):
    """Device pointer of a torch tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def host_f64(values):
    a = np.ascontiguousarray(np.asarray(values, dtype=np.float64))
    return a, a.ctypes.data_as(ctypes.c_void_p)


def dtype_code(torch_dtype):
    import torch

    if torch_dtype == torch.float64:
        return PF_F64
    if torch_dtype == torch.float32:
        return PF_F32
    raise ValueError(f"unsupported dtype {torch_dtype}")


def raise_status(status_host, what="filter bank"):
    """Turn per-filter device status flags into the reference's exceptions."""
    st = np.asarray(status_host)
    # divergence is detected at the transition, before weighting (lorenz63.py:48-49)
    if np.any(st & PF_ST_DIVERGED):
        bad = np.nonzero(st & PF_ST_DIVERGED)[0]
        raise NumericalDivergenceError(
            f"{what}: transition produced non-finite states (filters {bad[:8].tolist()})")
    if np.any(st & PF_ST_NAN_WEIGHT):
        raise ValueError("log weights contain NaN")
