"""Objective values, weight refresh and the safeguard step on the GPU
(reference objective.py).  Host-array wrappers for API parity and tests;
the unwrap loop calls the same C-ABI entry points on resident buffers.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .device import Workspace, _ptr
from .operators import SystemVector
from .params import ModelParams, lipschitz_constant  # noqa: F401  (re-export, objective.py:103)
from .phase import GradientField, WeightField


@dataclass(frozen=True)
class IrlsWeights:
    """objective.py:44-49 — auxiliary weights, elementwise >= delta/2."""

    wv: np.ndarray
    wh: np.ndarray


def arc_count(n, m):
    """objective.py:58-60."""
    return (n - 1) * m + n * (m - 1)


def _stage(ws, x, g=None, c=None, w=None):
    keep = []
    xd, k = ws.to_system(x.u, x.vv, x.vh)
    keep.append(k)
    out = {"x": xd}
    for name, pair in (("g", (g.gv, g.gh) if g is not None else None),
                       ("c", (c.cv, c.ch) if c is not None else None),
                       ("w", (w.wv, w.wh) if w is not None else None)):
        if pair is not None:
            t = ws.planes(2)
            keep.append([ws.pack(pair[0], t[0]), ws.pack(pair[1], t[1])])
            out[name] = t
    return out, keep


def eval_h_delta(x: SystemVector, w: IrlsWeights, g: GradientField, c: WeightField, p: ModelParams, dtype="fp64"):
    """objective.py:77-89 — lifted objective H_delta(x, w)."""
    half = 0.5 * p.delta
    if (w.wv.size and w.wv.min() < half) or (w.wh.size and w.wh.min() < half):
        raise ValueError("auxiliary weights must be >= delta/2")
    n, m = x.shape
    ws = Workspace.get(n, m, dtype, p.tau, p.delta)
    b, keep = _stage(ws, x, g, c, w)
    ws.call("pu_eval_h_delta", _ptr(b["x"]), _ptr(b["w"][0]), _ptr(b["w"][1]), _ptr(b["g"][0]), _ptr(b["g"][1]),
            _ptr(b["c"][0]), _ptr(b["c"][1]), ws.sp(ws.S_EVH), ws.stream())
    return float(ws.read_block()[0][ws.S_EVH])


def eval_f(x: SystemVector, g: GradientField, c: WeightField, p: ModelParams, dtype="fp64"):
    """objective.py:63-66 — weighted L1 + quadratic coupling penalties."""
    n, m = x.shape
    ws = Workspace.get(n, m, dtype, p.tau, p.delta)
    b, keep = _stage(ws, x, g, c)
    ws.call("pu_eval_f", _ptr(b["x"]), _ptr(b["g"][0]), _ptr(b["g"][1]), _ptr(b["c"][0]), _ptr(b["c"][1]),
            ws.sp(ws.S_F), ws.stream())
    return float(ws.read_block()[0][ws.S_F])


def update_weights(x: SystemVector, c: WeightField, delta, dtype="fp64"):
    """objective.py:92-100 — closed-form weights sqrt((c v)^2 + delta^2)."""
    if delta <= 0:
        raise ValueError(f"delta must be positive, got {delta}")
    n, m = x.shape
    ws = Workspace.get(n, m, dtype, 1e-2, delta)
    zero_g = GradientField(np.zeros((n - 1, m)), np.zeros((n, m - 1)))
    b, keep = _stage(ws, x, zero_g, c)
    w = ws.planes(2)
    d = ws.planes(2)
    ws.call("pu_weights_hpair", _ptr(b["x"]), _ptr(b["c"][0]), _ptr(b["c"][1]), _ptr(b["g"][0]), _ptr(b["g"][1]),
            None, None, _ptr(w[0]), _ptr(w[1]), _ptr(d[0]), _ptr(d[1]), ws.sp(ws.S_HOLD), ws.stream())
    return IrlsWeights(ws.unpack(w[0], n - 1, m).cpu().numpy(), ws.unpack(w[1], n, m - 1).cpu().numpy())


def candidate_step(x: SystemVector, w: IrlsWeights, g: GradientField, c: WeightField, p: ModelParams, lipschitz,
                   dtype="fp64"):
    """objective.py:118-125 — explicit gradient step with stepsize 1/L."""
    if lipschitz <= 0:
        raise ValueError(f"lipschitz constant must be positive, got {lipschitz}")
    n, m = x.shape
    ws = Workspace.get(n, m, dtype, p.tau, p.delta)
    b, keep = _stage(ws, x, g, c, w)
    out = ws.planes(3)
    ws.call("pu_candidate_step", _ptr(b["x"]), _ptr(b["w"][0]), _ptr(b["w"][1]), _ptr(b["g"][0]), _ptr(b["g"][1]),
            _ptr(b["c"][0]), _ptr(b["c"][1]), float(lipschitz), _ptr(out), ws.stream())
    u, vv, vh = ws.from_system(out)
    return SystemVector(u.cpu().numpy(), vv.cpu().numpy(), vh.cpu().numpy())
