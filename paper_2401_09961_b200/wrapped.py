"""wrapped_gradients on the GPU (reference phase.py:140-149).

Bit-identical to the reference in fp64: the device reduction avoids FMA
contraction (csrc/pu_kernels.cuh:wrap_lo).
"""

from __future__ import annotations

import numpy as np

from .device import Workspace, _ptr
from .phase import GradientField, validate_wrapped


def wrapped_gradients(x, lo=-np.pi):
    """Principal-interval neighbour differences of a wrapped grid."""
    import torch
    if lo not in (0.0, 0, -np.pi):
        raise ValueError(f"lo must be 0 or -pi, got {lo!r}")
    arr = validate_wrapped(x)
    n, m = arr.shape
    ws = Workspace.get(n, m, "fp64")
    xd = torch.from_numpy(np.ascontiguousarray(arr)).to(ws.device)
    g = ws.planes(2)
    ws.call("pu_wrapped_gradients", _ptr(xd), m, _ptr(g[0]), _ptr(g[1]), float(lo), ws.stream())
    gv = ws.unpack(g[0], n - 1, m).cpu().numpy()
    gh = ws.unpack(g[1], n, m - 1).cpu().numpy()
    return GradientField(gv=gv, gh=gh)
