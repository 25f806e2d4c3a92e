"""ctypes binding of libpu_unwrap.so (include/pu_unwrap.h).

There is no fallback: if the shared library is missing, or no CUDA device is
visible, every entry point raises.  `ensure()` is the single gate.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# PU_LIB_PATH: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("PU_LIB_PATH") or os.path.join(_HERE, "_lib", "libpu_unwrap.so")

PU_F32, PU_F64 = 0, 1
PU_OK, PU_ERR_ARG, PU_ERR_CUDA, PU_ERR_UNSUPPORTED, PU_ERR_NOMEM, PU_ERR_BREAKDOWN = 0, 1, 2, 3, 4, 5

_vp, _i, _d, _i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_int64

class PuIrlsParams(ctypes.Structure):
    """struct pu_irls_params (include/pu_unwrap.h; irls.py:43-64)."""
    _fields_ = [("max_iter_cg_start", ctypes.c_int32), ("max_outer_iters", ctypes.c_int32),
                ("max_cg_iters_cap", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("rel_improvement_tol", ctypes.c_double), ("cg_growth_factor", ctypes.c_double),
                ("cg_rel_tol", ctypes.c_double)]


class PuIterationRecord(ctypes.Structure):
    """struct pu_iteration_record (include/pu_unwrap.h; irls.py:67-75)."""
    _fields_ = [("k", ctypes.c_int32), ("m_cg", ctypes.c_int32), ("cg_iters", ctypes.c_int32),
                ("has_delta_rel", ctypes.c_int32), ("delta_rel", ctypes.c_double), ("h_delta", ctypes.c_double),
                ("sufficient_decrease", ctypes.c_int32), ("fallback_used", ctypes.c_int32)]


# name -> (restype, argtypes); mirrors include/pu_unwrap.h
SIGNATURES = {
    "pu_abi_version": (_i, []),
    "pu_last_error": (ctypes.c_char_p, []),
    "pu_pcg_ctrl_bytes": (_i, []),
    "pu_launch_count": (_i64, []),
    "pu_create": (_i, [ctypes.POINTER(_vp), _i, _i, _i, _d, _d]),
    "pu_destroy": (_i, [_vp]),
    "pu_pitch": (_i64, [_vp]),
    "pu_plane_elems": (_i64, [_vp]),
    "pu_describe": (_i, [_vp, ctypes.c_char_p, _i]),
    "pu_pack": (_i, [_vp, _vp, _i64, _i, _i, _vp, _vp]),
    "pu_unpack": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "pu_unpack_native": (_i, [_vp, _vp, _i, _i, _vp, _vp]),
    "pu_fill": (_i, [_vp, _vp, _i, _d, _vp]),
    "pu_copy": (_i, [_vp, _vp, _vp, _i, _vp]),
    "pu_wrapped_gradients_checked": (_i, [_vp, _vp, _i64, _vp, _vp, _d, _vp, _vp]),
    "pu_init_state": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "pu_wrapped_gradients": (_i, [_vp, _vp, _i64, _vp, _vp, _d, _vp]),
    "pu_build_rhs": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "pu_apply_system": (_i, [_vp, _vp, _vp, _vp, _vp, _vp]),
    "pu_dot": (_i, [_vp, _vp, _vp, _i, _vp, _vp]),
    "pu_sylvester_solve": (_i, [_vp, _vp, _vp, _vp, _vp]),
    "pu_apply_preconditioner": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "pu_weights_hpair": (_i, [_vp] + [_vp] * 11 + [_vp, _vp]),
    "pu_eval_h_delta": (_i, [_vp] + [_vp] * 7 + [_vp, _vp]),
    "pu_eval_f": (_i, [_vp] + [_vp] * 5 + [_vp, _vp]),
    "pu_candidate_step": (_i, [_vp] + [_vp] * 7 + [_d, _vp, _vp]),
    "pu_hpair_states": (_i, [_vp] + [_vp] * 8 + [_vp, _vp]),
    "pu_accept_center": (_i, [_vp] + [_vp] * 10 + [_vp, _vp]),
    "pu_pcg_solve": (_i, [_vp] + [_vp] * 10 + [_i, _d, _vp, _vp, _vp]),
    "pu_irls_step": (_i, [_vp] + [_vp] * 10 + [_d, _i, _d] + [_vp] * 7 + [_vp, _vp]),
    "pu_irls_begin": (_i, [_vp] + [_vp] * 10 + [_d, _d] + [_vp] * 7 + [_vp]),
    "pu_irls_iterate": (_i, [_vp] + [_vp] * 9 + [_i] + [_vp] * 7 + [_vp, _vp]),
    "pu_accept_weights": (_i, [_vp] + [_vp] * 15 + [_vp]),
    "pu_accept_weights_start": (_i, [_vp] + [_vp] * 15 + [_d, _vp, _vp, _vp]),
    "pu_irls_begin_z0": (_i, [_vp, _vp, _vp, _d] + [_vp] * 7),
    "pu_set_graphs": (_i, [_vp, _i]),
    "pu_timing_enable": (_i, [_vp, _i]),
    "pu_timing_read": (_i, [_vp, _vp, _vp, _vp, _i]),
    "pu_shift_error": (_i, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "pu_kmap_mismatch": (_i, [_vp, _vp, _vp, _i64, _vp, _i64, _vp, _vp]),
    "pu_congruent_round": (_i, [_vp, _vp, _vp, _i64, _vp, _vp]),
    # row-sharded grids (band.py)
    "pu_create_band": (_i, [ctypes.POINTER(_vp), _i, _vp, _i, _d, _d]),
    "pu_set_band_totals": (_i, [_vp, _vp]),
    "pu_set_band_peers": (_i, [_vp, _vp, _vp]),
    "pu_ipc_handle": (_i, [_vp, _vp]),
    "pu_ipc_open": (_i, [_vp, ctypes.POINTER(_vp)]),
    "pu_ipc_close": (_i, [_vp]),
    "pu_dev_alloc": (_i, [_i64, ctypes.POINTER(_vp)]),
    "pu_dev_free": (_i, [_vp]),
    "pu_finalize": (_i, [_vp, ctypes.c_uint, _i, _i, _vp, _vp, _vp, _d, _i, _vp]),
    "pu_set_max_iters": (_i, [_vp, _vp, _i, _vp]),
    "pu_pcg_begin": (_i, [_vp] + [_vp] * 8 + [_i, _d] + [_vp] * 6 + [_d, _vp, _vp]),
    "pu_pcg_residual_rows": (_i, [_vp] + [_vp] * 8 + [_i, _i, _vp]),
    "pu_pcg_update_sum": (_i, [_vp] + [_vp] * 6 + [_i, _vp]),
    "pu_pcg_columns": (_i, [_vp, _vp, _vp, _i, _vp]),
    "pu_pcg_rows_inv": (_i, [_vp, _vp, _vp, _vp, _i, _vp, _i, _vp]),
    "pu_pcg_direction": (_i, [_vp] + [_vp] * 6 + [_i, _vp]),
    # GPU synthetic scenes (pu_synth.cu)
    "pu_synth_bumps": (_i, [_vp, _i, _i, _i64, _vp, _i, _vp]),
    "pu_synth_fault": (_i, [_vp, _i, _i, _i64, _vp, _vp, _d, _vp]),
    "pu_synth_wrap_noise": (_i, [_vp, _i, _i, _i64, _d, ctypes.c_uint64, _vp]),
    # the whole unwrap behind one call (pu_host.cu)
    "pu_irls_params_default": (None, [ctypes.POINTER(PuIrlsParams)]),
    "pu_unwrap": (_i, [_vp, _i, _i, _vp, _vp, _d, _d, ctypes.POINTER(PuIrlsParams), _d, _i, _i, _vp, _vp, _vp,
                       ctypes.POINTER(PuIterationRecord), _i, ctypes.POINTER(_i), ctypes.POINTER(_i)]),
}


class PuBand(ctypes.Structure):
    """struct pu_band (include/pu_unwrap.h)."""
    _fields_ = [("n_glob", ctypes.c_int32), ("row0", ctypes.c_int32), ("rows", ctypes.c_int32),
                ("nq", ctypes.c_int32), ("mb", ctypes.c_int32), ("col0", ctypes.c_int32), ("cols", ctypes.c_int32)]


# reduction sites (enum pu_site) and the totals row length
SITE_WH, SITE_HPAIR, SITE_ACC, SITE_START, SITE_K1, SITE_K2, SITE_K3, SITE_UPD = 1, 3, 4, 6, 7, 8, 9, 10
NSITES, MAX_SUMS = 13, 12

_lib = None


class NativeError(RuntimeError):
    """A CUDA-side failure reported through the C ABI."""


def load():
    """Load the shared library (no GPU needed); raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -m paper_2401_09961_b200.build_ext` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.pu_abi_version() != 1:
        raise ImportError("libpu_unwrap.so ABI version mismatch; rebuild it")
    _lib = lib
    return lib


def ensure():
    """Library loaded AND a CUDA device present — the product path's gate."""
    lib = load()
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2401_09961_b200 needs a CUDA device (B200, sm_100a); no CPU fallback exists")
    return lib


def check(rc):
    if rc == PU_OK:
        return
    msg = _lib.pu_last_error().decode() if _lib is not None else "unknown"
    if rc == PU_ERR_ARG:
        raise ValueError(msg)
    if rc == PU_ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(f"libpu_unwrap error {rc}: {msg}")


def call(name, *args):
    check(getattr(_lib, name)(*args))


def exported_symbols():
    return sorted(SIGNATURES)
