"""Parity metrics on the device.

`shift_error`, `congruent_round` (reference phase.py:152-184) and the K-map
mismatch fraction of the harness, computed by libpu_unwrap.so kernels on a
device u (a numpy / torch grid, or the u plane of an unwrap still resident
on the GPU) against fp64 device grids — at 16384² the operands stay in HBM
and only four scalars come back.
"""

from __future__ import annotations

import numpy as np

from .device import Workspace, _ptr
from .phase import ErrorReport


def _torch():
    import torch
    return torch


def _ws_u(u, dtype, ws=None):
    """(workspace, u plane) for a host / device grid, packed into the handle's layout."""
    torch = _torch()
    n, m = int(u.shape[0]), int(u.shape[1])
    ws = ws or Workspace.get(n, m, dtype)
    plane = ws.buf(("metric_u",), 1)
    keep = ws.pack(u, plane[0])
    return ws, plane[0], keep


def _dev64(ws, a):
    torch = _torch()
    t = torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64)) if isinstance(a, np.ndarray) else a
    return t.to(device=ws.device, dtype=torch.float64).contiguous()


def shift_error(u, x_u, *, dtype="fp64", ws=None, u_plane=None):
    """phase.py:152-175 on the GPU; ErrorReport with error_grid=None."""
    torch = _torch()
    if tuple(u.shape) != tuple(x_u.shape):
        raise ValueError(f"dimension mismatch: {tuple(u.shape)} vs {tuple(x_u.shape)}")
    if u_plane is None:
        ws, u_plane, keep = _ws_u(u, dtype, ws)
    x = _dev64(ws, x_u)
    out = torch.zeros(4, dtype=torch.float64, device=ws.device)
    ws.call("pu_shift_error", _ptr(u_plane), _ptr(x), int(x.shape[1]), _ptr(out), ws.stream())
    a, mx, rmse, frac = (float(v) for v in out.cpu())
    return ErrorReport(alpha=a, error_grid=None, max_abs=mx, rmse=rmse, congruent_fraction=frac)


def kmap_mismatch(u, u_ref, x, *, dtype="fp64", ws=None, u_plane=None):
    """mean(rint((u - x)/2pi) != rint((u_ref - x)/2pi)) on the GPU."""
    torch = _torch()
    if not (tuple(u.shape) == tuple(u_ref.shape) == tuple(x.shape)):
        raise ValueError("dimension mismatch")
    if u_plane is None:
        ws, u_plane, keep = _ws_u(u, dtype, ws)
    r, xd = _dev64(ws, u_ref), _dev64(ws, x)
    out = torch.zeros(1, dtype=torch.float64, device=ws.device)
    ws.call("pu_kmap_mismatch", _ptr(u_plane), _ptr(r), int(r.shape[1]), _ptr(xd), int(xd.shape[1]), _ptr(out),
            ws.stream())
    return float(out.item())


def congruent_round(u, x, *, dtype="fp64", ws=None, u_plane=None):
    """phase.py:178-184 on the GPU; returns a host fp64 grid."""
    torch = _torch()
    if tuple(u.shape) != tuple(x.shape):
        raise ValueError(f"dimension mismatch: {tuple(u.shape)} vs {tuple(x.shape)}")
    if u_plane is None:
        ws, u_plane, keep = _ws_u(u, dtype, ws)
    xd = _dev64(ws, x)
    out = torch.empty(tuple(xd.shape), dtype=torch.float64, device=ws.device)
    ws.call("pu_congruent_round", _ptr(u_plane), _ptr(xd), int(xd.shape[1]), _ptr(out), ws.stream())
    return out.cpu().numpy()
