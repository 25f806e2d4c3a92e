"""Preconditioned CG on the GPU (reference pcg.py:47-116).

The reference takes `apply_a` / `apply_m` callables; here both operators are
fused into the four CUDA kernels of one iteration, so the
solver takes the diagonal weights `d` and `tau` that define them.  Exits,
iteration counting, the every-50 mean re-projection and the
NumericalBreakdown indices follow pcg.py exactly; the decisions are made on
the device and read back once per solve.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .device import Workspace, _ptr
from .operators import DiagonalWeights, SystemVector

REPROJECT_EVERY = 50
_TINY_CURVATURE = 1e-300

_BREAKDOWN_MSG = {
    0: "initial residual is not finite",
    1: "curvature p'Ap is not finite",
    2: "residual norm is not finite",
    3: "preconditioned product is not finite",
}


class NumericalBreakdown(RuntimeError):
    """pcg.py:24-29 — a non-finite value appeared during the iteration."""

    def __init__(self, iteration, message):
        super().__init__(f"iteration {iteration}: {message}")
        self.iteration = iteration


@dataclass
class PcgOutcome:
    """pcg.py:32-38."""

    x: SystemVector
    iterations: int
    residual_norms: list = field(default_factory=list)
    converged: bool = False
    residual: SystemVector | None = None


def raise_if_breakdown(ctrl):
    if int(ctrl["breakdown"]) >= 0:
        kind = int(ctrl["bkind"])
        raise NumericalBreakdown(int(ctrl["breakdown"]), _BREAKDOWN_MSG.get(kind, "non-finite value"))


def pcg_device(ws: Workspace, b, x0, x, dv, dh, max_iters, rel_tol):
    """Enqueue one fused PCG solve on resident buffers (no synchronisation)."""
    if max_iters < 0:
        raise ValueError("max_iters must be >= 0")
    if rel_tol < 0:
        raise ValueError("rel_tol must be >= 0")
    r = ws.buf("pcg_r", 3)
    z = ws.buf("pcg_z", 3)
    p0 = ws.buf("pcg_p0", 3)
    p1 = ws.buf("pcg_p1", 3)
    spec = ws.buf("spec", 1)
    norms = ws.ensure_norms(max_iters)
    ws.call("pu_pcg_solve", _ptr(b), _ptr(x0), _ptr(x), _ptr(dv), _ptr(dh), _ptr(r), _ptr(z), _ptr(p0), _ptr(p1),
            _ptr(spec), int(max_iters), float(rel_tol), _ptr(ws.ctrl), _ptr(norms), ws.stream())
    return r


def pcg_solve(b: SystemVector, x0: SystemVector, d: DiagonalWeights, tau, max_iters, rel_tol, dtype="fp64"):
    """pcg.py:47-116 with apply_system(., d, tau) and apply_preconditioner fused in."""
    if max_iters < 0:
        raise ValueError("max_iters must be >= 0")
    if rel_tol < 0:
        raise ValueError("rel_tol must be >= 0")
    n, m = b.shape
    ws = Workspace.get(n, m, dtype, tau)
    bd, k1 = ws.to_system(b.u, b.vv, b.vh)
    xd0, k2 = ws.to_system(x0.u, x0.vv, x0.vh)
    dd = ws.planes(2)
    k3 = [ws.pack(d.dv, dd[0]), ws.pack(d.dh, dd[1])]
    x = ws.planes(3)
    r = pcg_device(ws, bd, xd0, x, dd[0], dd[1], max_iters, rel_tol)
    _, ctrl = ws.read_block()
    raise_if_breakdown(ctrl)
    its = int(ctrl["iterations"])
    norms = ws.norms[: its + 1].cpu().numpy().tolist()
    xu, xv, xh = ws.from_system(x)
    ru, rv, rh = ws.from_system(r)
    return PcgOutcome(
        x=SystemVector(xu.cpu().numpy(), xv.cpu().numpy(), xh.cpu().numpy()),
        iterations=its,
        residual_norms=norms,
        converged=bool(ctrl["converged"]),
        residual=SystemVector(ru.cpu().numpy(), rv.cpu().numpy(), rh.cpu().numpy()),
    )
