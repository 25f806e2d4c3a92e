"""Block-system operators on the GPU (reference operators.py:39-162).

`SystemVector` and `DiagonalWeights` keep the reference's host container
semantics (numpy blocks with the same shape checks).  The arithmetic —
apply_system, build_rhs, dot — runs in libpu_unwrap.so; these wrappers copy
host blocks to a planned device workspace and back, for API parity and tests.
The unwrap hot path (irls.py) never leaves the device.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .device import Workspace, _ptr
from .phase import GradientField


@dataclass
class SystemVector:
    """operators.py:39-101 — triple (u, vv, vh) viewed as one vector."""

    u: np.ndarray
    vv: np.ndarray
    vh: np.ndarray

    def __post_init__(self):
        n, m = self.u.shape
        if self.vv.shape != (n - 1, m) or self.vh.shape != (n, m - 1):
            raise ValueError(f"inconsistent block shapes: u {self.u.shape}, vv {self.vv.shape}, vh {self.vh.shape}")

    @classmethod
    def zeros(cls, n, m):
        return cls(np.zeros((n, m)), np.zeros((n - 1, m)), np.zeros((n, m - 1)))

    @property
    def shape(self):
        return self.u.shape

    @property
    def dim(self):
        return self.u.size + self.vv.size + self.vh.size

    def copy(self):
        return SystemVector(self.u.copy(), self.vv.copy(), self.vh.copy())

    def dot(self, other, dtype="fp64"):
        """operators.py:70-75, evaluated on the GPU (fp64 accumulation)."""
        n, m = self.shape
        ws = Workspace.get(n, m, dtype)
        a, ka = ws.to_system(self.u, self.vv, self.vh)
        b, kb = ws.to_system(other.u, other.vv, other.vh)
        ws.call("pu_dot", _ptr(a), _ptr(b), 3, ws.sp(ws.S_DOT), ws.stream())
        return float(ws.read_block()[0][ws.S_DOT])

    def norm(self, dtype="fp64"):
        return float(np.sqrt(self.dot(self, dtype)))


@dataclass(frozen=True)
class DiagonalWeights:
    """operators.py:104-115 — diagonal blocks dv (N-1, M), dh (N, M-1)."""

    dv: np.ndarray
    dh: np.ndarray

    def __post_init__(self):
        if self.dv.shape[0] + 1 != self.dh.shape[0] or self.dv.shape[1] != self.dh.shape[1] + 1:
            raise ValueError(f"inconsistent diagonal shapes {self.dv.shape} / {self.dh.shape}")


def _np_system(ws, x):
    u, vv, vh = ws.from_system(x)
    return SystemVector(u.cpu().numpy(), vv.cpu().numpy(), vh.cpu().numpy())


def apply_system(x: SystemVector, d: DiagonalWeights, tau, dtype="fp64"):
    """operators.py:138-153 — the symmetric PSD 3-block map A(d)."""
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    n, m = x.shape
    ws = Workspace.get(n, m, dtype, tau)
    xd, k1 = ws.to_system(x.u, x.vv, x.vh)
    dd = ws.planes(2)
    k2 = [ws.pack(d.dv, dd[0]), ws.pack(d.dh, dd[1])]
    y = ws.planes(3)
    ws.call("pu_apply_system", _ptr(xd), _ptr(dd[0]), _ptr(dd[1]), _ptr(y), ws.stream())
    return _np_system(ws, y)


def build_rhs(g: GradientField, tau, dtype="fp64"):
    """operators.py:156-162 — right-hand side b, orthogonal to the constant-u mode."""
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    n, m = g.shape
    ws = Workspace.get(n, m, dtype, tau)
    gd = ws.planes(2)
    keep = [ws.pack(g.gv, gd[0]), ws.pack(g.gh, gd[1])]
    b = ws.planes(3)
    ws.call("pu_build_rhs", _ptr(gd[0]), _ptr(gd[1]), _ptr(b), ws.stream())
    return _np_system(ws, b)


def apply_s(u):
    """operators.py:118-120 — forward row differences (host helper)."""
    return np.asarray(u)[1:, :] - np.asarray(u)[:-1, :]


def apply_t(u):
    """operators.py:128-130 — forward column differences (host helper)."""
    return np.asarray(u)[:, 1:] - np.asarray(u)[:, :-1]
