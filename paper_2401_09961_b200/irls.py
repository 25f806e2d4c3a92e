"""The unwrap hot path on one B200 (reference irls.py:132-224).

Mirrors the reference outer loop line by line — weight refresh, lifted
objective pair and CG-budget rule, warm-started PCG, explicit-gradient
safeguard, mean centring, trace — with every array operation running in
libpu_unwrap.so on HBM-resident buffers.  The host synchronises once per
outer iteration, to read the H_delta pair that drives the budget decision
(plus the previous iteration's trace scalars).
"""

from __future__ import annotations

import numpy as np

from .device import Workspace, _ptr
from .params import (BudgetDecision, IrlsParams, IrlsTrace, IterationRecord, ModelParams,  # noqa: F401
                     UnwrapResult, cg_budget_update, lipschitz_constant, relative_improvement)
from .pcg import pcg_device, raise_if_breakdown
from .phase import WeightField, validate_wrapped


def _torch():
    import torch
    return torch


class DeviceUnwrap:
    """Resident buffers and launch sequence of one unwrap (one stream)."""

    def __init__(self, ws: Workspace):
        self.ws = ws
        self.S = ws.buf("state", 3)      # accepted state
        self.X = ws.buf("proposal", 3)   # PCG iterate / proposal
        self.C = ws.buf("cand", 3)       # explicit-gradient candidate
        self.B = ws.buf("rhs", 3)
        self.G = ws.buf("grad", 2)       # gv, gh
        self.W = ws.buf("cw", 2)         # cv, ch
        self.Wt = [ws.buf("w0", 2), ws.buf("w1", 2)]
        self.D = ws.buf("diag", 2)       # dv, dh

    def load(self, x_dev, c: WeightField | None, lo):
        ws, st = self.ws, self.ws.stream()
        torch = _torch()
        if c is None:
            ws.call("pu_fill", _ptr(self.W), 2, 1.0, st)
            self._keep = None
        else:
            self._keep = [ws.pack(c.cv, self.W[0]), ws.pack(c.ch, self.W[1])]
        x64 = x_dev if x_dev.dtype == torch.float64 else x_dev.to(torch.float64)
        self._x = x64.contiguous()
        ws.call("pu_wrapped_gradients", _ptr(self._x), int(self._x.shape[1]), _ptr(self.G[0]), _ptr(self.G[1]),
                float(lo), st)
        ws.call("pu_build_rhs", _ptr(self.G[0]), _ptr(self.G[1]), _ptr(self.B), st)
        ws.call("pu_init_state", _ptr(self.G[0]), _ptr(self.G[1]), _ptr(self.S), st)

    def weights(self, k):
        """update_weights + H(state, w_prev), H(state, w) -> scal[S_HOLD:S_HNEW+1]."""
        ws, w, wp = self.ws, self.Wt[k & 1], (self.Wt[(k + 1) & 1] if k > 0 else None)
        ws.call("pu_weights_hpair", _ptr(self.S), _ptr(self.W[0]), _ptr(self.W[1]), _ptr(self.G[0]),
                _ptr(self.G[1]), _ptr(wp[0]) if wp is not None else None, _ptr(wp[1]) if wp is not None else None,
                _ptr(w[0]), _ptr(w[1]), _ptr(self.D[0]), _ptr(self.D[1]), ws.sp(ws.S_HOLD), ws.stream())

    def step(self, k, m_cg, params: IrlsParams, lip):
        """PCG + candidate + safeguard + centring (irls.py:191-215), all enqueued."""
        ws, st, w = self.ws, self.ws.stream(), self.Wt[k & 1]
        pcg_device(ws, self.B, self.S, self.X, self.D[0], self.D[1], m_cg, params.cg_rel_tol)
        ws.call("pu_candidate_step", _ptr(self.S), _ptr(w[0]), _ptr(w[1]), _ptr(self.G[0]), _ptr(self.G[1]),
                _ptr(self.W[0]), _ptr(self.W[1]), float(lip), _ptr(self.C), st)
        ws.call("pu_hpair_states", _ptr(self.X), _ptr(self.C), _ptr(w[0]), _ptr(w[1]), _ptr(self.G[0]),
                _ptr(self.G[1]), _ptr(self.W[0]), _ptr(self.W[1]), ws.sp(ws.S_HPROP), st)
        ws.call("pu_accept_center", _ptr(self.X), _ptr(self.C), ws.sp(ws.S_MEAN), _ptr(self.S), _ptr(w[0]),
                _ptr(w[1]), _ptr(self.G[0]), _ptr(self.G[1]), _ptr(self.W[0]), _ptr(self.W[1]),
                ws.sp(ws.S_HACC), st)

    def result_arrays(self):
        return self.ws.from_system(self.S)


def _record(k, m_cg, delta_rel, scal, ctrl, ws):
    raise_if_breakdown(ctrl)
    sufficient = bool(scal[ws.S_TAKE] != 0.0)
    return IterationRecord(k=k, m_cg=m_cg, delta_rel=delta_rel, h_delta=float(scal[ws.S_HACC]),
                           cg_iters=int(ctrl["iterations"]), sufficient_decrease=sufficient,
                           fallback_used=not sufficient)


def unwrap_device(x_dev, c: WeightField | None, model: ModelParams, params: IrlsParams, gradient_lo,
                  dtype="fp64", ws: Workspace | None = None):
    """Run the loop on a device fp64 grid; returns (DeviceUnwrap, IrlsTrace)."""
    n, m = int(x_dev.shape[0]), int(x_dev.shape[1])
    ws = ws or Workspace.get(n, m, dtype, model.tau, model.delta, x_dev.device)
    run = DeviceUnwrap(ws)
    run.load(x_dev, c, gradient_lo)
    cmax = 1.0 if c is None else c.max_weight
    lip = 12.0 / model.tau + cmax ** 2 / model.delta          # objective.py:103-105
    trace = IrlsTrace()
    m_history = [params.max_iter_cg_start]
    pending = None  # (k, m_cg, delta_rel) of the enqueued iteration awaiting its scalars
    for k in range(params.max_outer_iters):
        run.weights(k)
        delta_rel = None
        if k >= 1:
            scal, ctrl = ws.read_block()                     # the one sync of this iteration
            trace.append(_record(*pending, scal, ctrl, ws))
            pending = None
            h_old, h_new = float(scal[ws.S_HOLD]), float(scal[ws.S_HNEW])
            delta_rel = 0.0 if h_old == 0 else relative_improvement(h_old, h_new)
            m_prev = m_history[k - 1]
            m_prev2 = m_history[k - 2] if k >= 2 else m_prev
            decision = cg_budget_update(delta_rel, m_prev, m_prev2, params)
            if decision.action == "stop":
                break
            m_cg = decision.m_cg
            m_history.append(m_cg)
        else:
            m_cg = m_history[0]
        run.step(k, m_cg, params, lip)
        pending = (k, m_cg, delta_rel)
    if pending is not None:
        scal, ctrl = ws.read_block()
        trace.append(_record(*pending, scal, ctrl, ws))
    return run, trace


def unwrap(x, c: WeightField | None = None, model: ModelParams | None = None, params: IrlsParams | None = None,
           gradient_lo=-np.pi, *, dtype="fp64", device=None):
    """irls.py:132-224 — unwrap a wrapped phase grid on the GPU.

    Same parameters and result as the reference; `dtype` ("fp64" default,
    or "fp32") selects the arithmetic of the device buffers (reductions are
    always accumulated in fp64).  `x` may be a numpy array or a CUDA tensor.
    """
    from . import _native
    _native.ensure()  # library + CUDA device, or raise: there is no CPU path
    torch = _torch()
    dev = torch.device(device) if device is not None else (
        x.device if isinstance(x, torch.Tensor) and x.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    if isinstance(x, np.ndarray) and not np.issubdtype(x.dtype, np.number):
        raise ValueError("phase grid must be numeric")
    if isinstance(x, torch.Tensor) and x.is_cuda:
        x_dev = x.to(device=dev, dtype=torch.float64)
    else:
        arr = x if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValueError(f"phase grid must be 2-D and non-empty, got shape {tuple(arr.shape)}")
        ws_in = Workspace.get(int(arr.shape[0]), int(arr.shape[1]), dtype, (model or ModelParams()).tau,
                              (model or ModelParams()).delta, dev)
        x_dev = ws_in.upload_grid(arr if isinstance(arr, torch.Tensor) else arr)
    if x_dev.dim() != 2 or x_dev.shape[0] < 1 or x_dev.shape[1] < 1:
        raise ValueError(f"phase grid must be 2-D and non-empty, got shape {tuple(x_dev.shape)}")
    # phase.py:100-115 on the device: finite, within [0, 2pi)
    chk = torch.stack([x_dev.min(), x_dev.max(), torch.isfinite(x_dev).all().to(torch.float64)]).cpu()
    if chk[2] != 1.0:
        raise ValueError("phase grid contains non-finite values")
    if float(chk[0]) < 0.0 or float(chk[1]) >= 2.0 * np.pi:
        raise ValueError("wrapped phase values must lie in [0, 2*pi)")
    n, m = int(x_dev.shape[0]), int(x_dev.shape[1])
    model = model or ModelParams()
    params = params or IrlsParams()
    if c is not None and (c.cv.shape != (n - 1, m) or c.ch.shape != (n, m - 1)):
        raise ValueError(f"weight shapes {c.cv.shape}/{c.ch.shape} do not match grid {(n, m)}")
    if gradient_lo not in (0.0, 0, -np.pi):
        raise ValueError(f"lo must be 0 or -pi, got {gradient_lo!r}")
    run, trace = unwrap_device(x_dev, c, model, params, gradient_lo, dtype)
    u, vv, vh = run.ws.download_system(run.S)
    return UnwrapResult(u=u, vv=vv, vh=vh, trace=trace)
