"""DCT-II/III Poisson preconditioner on the GPU (reference preconditioner.py).

The reference diagonalises the 1-D Neumann second-difference operators with
dense LAPACK eigenbases and applies them as four GEMMs per solve
(preconditioner.py:64-100).  Those eigenbases are the orthonormal DCT-II
basis with eigenvalues 2 - 2cos(pi k / n), so libpu_unwrap.so applies the
same pseudo-inverse with shared-memory FFT-based DCT kernels:
row DCT-II -> column DCT-II, x tau/(lam_i + lam_j) with (0,0) -> 0,
column DCT-III -> row DCT-III.
"""

from __future__ import annotations

import numpy as np

from .device import Workspace, _ptr
from .operators import DiagonalWeights, SystemVector, _np_system


def neumann_eigenvalues(n):
    """Analytic spectrum of the 1-D Neumann stencil (ascending, first exactly 0)."""
    k = np.arange(n)
    lam = 4.0 * np.sin(np.pi * k / (2.0 * n)) ** 2
    lam[0] = 0.0
    return lam


def sylvester_solve(r, tau, dtype="fp64"):
    """preconditioner.py:86-100 — solve StS Z + Z TTt = tau (r - mean r), mean(Z) = 0."""
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    r = np.asarray(r, dtype=np.float64)
    n, m = r.shape
    ws = Workspace.get(n, m, dtype, tau)
    rd = ws.planes(3)  # r | z | spectral scratch
    keep = ws.pack(r, rd[0])
    ws.call("pu_sylvester_solve", _ptr(rd[0]), _ptr(rd[1]), _ptr(rd[2]), ws.stream())
    return ws.unpack(rd[1], n, m).cpu().numpy()


def apply_preconditioner(r: SystemVector, d: DiagonalWeights, tau, dtype="fp64"):
    """preconditioner.py:103-115 — block-diagonal pseudo-inverse D^+ r."""
    if tau <= 0:
        raise ValueError(f"tau must be positive, got {tau}")
    n, m = r.shape
    ws = Workspace.get(n, m, dtype, tau)
    rd, k1 = ws.to_system(r.u, r.vv, r.vh)
    dd = ws.planes(2)
    k2 = [ws.pack(d.dv, dd[0]), ws.pack(d.dh, dd[1])]
    z = ws.planes(3)
    spec = ws.planes(1)
    ws.call("pu_apply_preconditioner", _ptr(rd), _ptr(dd[0]), _ptr(dd[1]), _ptr(z), _ptr(spec), ws.stream())
    return _np_system(ws, z)
