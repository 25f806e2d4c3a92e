"""The whole unwrap through the C ABI entry point `pu_unwrap` (ctypes).

This is the binding a `phaseirls` maintainer would add to route the
reference's `unwrap` (irls.py:132-224) to the B200 without this package's
Python host loop: host numpy arrays in, host numpy arrays and the trace out,
the IRLS outer loop running in C++ inside libpu_unwrap.so
(csrc/pu_host.cu).  Same signature, result type and errors as `unwrap`:
ValueError for invalid input (checked in C before any device work),
NumericalBreakdown(iteration) for a non-finite PCG value.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .params import IrlsParams, IrlsTrace, IterationRecord, ModelParams, UnwrapResult
from .pcg import NumericalBreakdown
from .phase import WeightField

_DT = {"fp64": nat.PU_F64, "float64": nat.PU_F64, "fp32": nat.PU_F32, "float32": nat.PU_F32}


def _c_params(p: IrlsParams):
    cp = nat.PuIrlsParams()
    cp.max_iter_cg_start = int(p.max_iter_cg_start)
    cp.max_outer_iters = int(p.max_outer_iters)
    cp.max_cg_iters_cap = int(p.max_cg_iters_cap)
    cp.rel_improvement_tol = float(p.rel_improvement_tol)
    cp.cg_growth_factor = float(p.cg_growth_factor)
    cp.cg_rel_tol = float(p.cg_rel_tol)
    return cp


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else ctypes.c_void_p(0)


def unwrap_capi(x, c: WeightField | None = None, model: ModelParams | None = None,
                params: IrlsParams | None = None, gradient_lo=-np.pi, *, dtype="fp64", device=0):
    """irls.py:132-224 through `pu_unwrap` (include/pu_unwrap.h)."""
    lib = nat.load()
    if dtype not in _DT:
        raise ValueError(f"dtype must be 'fp32' or 'fp64', got {dtype!r}")
    model = model or ModelParams()
    params = params or IrlsParams()
    arr = np.asarray(x)
    if not np.issubdtype(arr.dtype, np.number):
        raise ValueError("phase grid must be numeric")
    arr = np.ascontiguousarray(arr, dtype=np.float64)
    if arr.ndim != 2:
        raise ValueError(f"phase grid must be 2-D and non-empty, got shape {arr.shape}")
    n, m = arr.shape
    cv = ch = None
    if c is not None:
        cv = np.ascontiguousarray(c.cv, dtype=np.float64)
        ch = np.ascontiguousarray(c.ch, dtype=np.float64)
        if cv.shape != (n - 1, m) or ch.shape != (n, m - 1):  # irls.py:157-160
            raise ValueError(f"weight shapes {cv.shape}/{ch.shape} do not match grid {(n, m)}")
    u = np.empty((n, m))
    vv = np.empty((max(n - 1, 0), m))
    vh = np.empty((n, max(m - 1, 0)))
    cap = int(params.max_outer_iters)
    recs = (nat.PuIterationRecord * max(cap, 1))()
    count, brk = ctypes.c_int(0), ctypes.c_int(-1)
    cp = _c_params(params)
    rc = lib.pu_unwrap(_ptr(arr), n, m, _ptr(cv), _ptr(ch), float(model.tau), float(model.delta), ctypes.byref(cp),
                       float(gradient_lo), _DT[dtype], int(device), _ptr(u), _ptr(vv), _ptr(vh), recs, cap,
                       ctypes.byref(count), ctypes.byref(brk))
    if rc == nat.PU_ERR_BREAKDOWN:
        msg = lib.pu_last_error().decode()
        raise NumericalBreakdown(int(brk.value), msg.split(": ", 1)[-1])
    nat.check(rc)
    trace = IrlsTrace()
    for r in recs[:count.value]:
        trace.append(IterationRecord(k=int(r.k), m_cg=int(r.m_cg),
                                     delta_rel=float(r.delta_rel) if r.has_delta_rel else None,
                                     h_delta=float(r.h_delta), cg_iters=int(r.cg_iters),
                                     sufficient_decrease=bool(r.sufficient_decrease),
                                     fallback_used=bool(r.fallback_used)))
    return UnwrapResult(u=u, vv=vv, vh=vh, trace=trace)
