"""GPU synthetic scenes (reference synth.py:43-109).

The reference's scene recipes with the per-pixel work on the device
(csrc/pu_synth.cu): every random parameter (bump count, centres, widths,
peaks; the fault seam's random walk) is drawn on the host from the
reference's own Philox stream, exactly as `synth.py` draws it, so the
noise-free scenes are the reference's (plateau/fault exact, bumps within
~1e-15 from the device exp).  Phase noise uses a device Philox-4x32 stream
with Box-Muller normals: the same distribution, another realisation.  The
parity tests therefore keep the host generator (`synth.py`, sha256-pinned);
this one is for large benchmark inputs (C4 16384² in well under a second
instead of ~60 s).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .synth import SceneSpec, _philox


def _torch():
    import torch
    return torch


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


def bump_params(spec: SceneSpec):
    """synth.py gaussian-bumps draws: (count, 4) array of r0, c0, width, peak."""
    gen = _philox(spec.seed)
    count = int(gen.integers(3, 7))
    out = np.zeros((count, 4))
    for b in range(count):
        r0 = gen.uniform(0, spec.rows - 1) if spec.rows > 1 else 0.0
        c0 = gen.uniform(0, spec.cols - 1) if spec.cols > 1 else 0.0
        width = spec.feature_scale * gen.uniform(0.7, 1.4)
        peak = spec.amplitude * gen.uniform(0.5, 1.0) * gen.choice((-1.0, 1.0))
        out[b] = (r0, c0, width, peak)
    return out


def plateau_seam(spec: SceneSpec):
    """synth.py plateau-discontinuity draws: the seam column of every row."""
    gen = _philox(spec.seed)
    mid = spec.cols // 2 if spec.cols > 1 else 1
    jitter = spec.cols / (4.0 * spec.feature_scale)
    walk = np.cumsum(gen.uniform(-jitter, jitter, size=spec.rows))
    return np.clip(mid + np.rint(walk).astype(np.int64), 1, max(spec.cols - 1, 1)).astype(np.int64)


def generate_scene_gpu(spec: SceneSpec, device=None):
    """synth.py:88-90 on the GPU: an (rows, cols) fp64 CUDA tensor."""
    lib = nat.ensure()
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    out = torch.zeros((spec.rows, spec.cols), dtype=torch.float64, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    if spec.kind == "ramp":
        per_row = spec.amplitude / spec.feature_scale
        out.copy_((per_row * torch.arange(spec.rows, dtype=torch.float64, device=dev))[:, None].expand_as(out))
    elif spec.kind == "gaussian-bumps":
        prm = torch.as_tensor(bump_params(spec), device=dev)
        nat.check(lib.pu_synth_bumps(_p(out), spec.rows, spec.cols, spec.cols, _p(prm), int(prm.shape[0]), st))
        torch.cuda.current_stream(dev).synchronize()
    elif spec.kind == "plateau-discontinuity":
        seam = torch.as_tensor(plateau_seam(spec), device=dev)
        lin = torch.ones(spec.rows, dtype=torch.float64, device=dev)
        nat.check(lib.pu_synth_fault(_p(out), spec.rows, spec.cols, spec.cols, _p(seam), _p(lin),
                                     float(spec.amplitude), st))
        torch.cuda.current_stream(dev).synchronize()
    else:
        raise ValueError(f"unknown scene kind {spec.kind!r}")
    return out


def tapered_fault_gpu(n, seed, amp, scale, fault_max, fault_scale, device=None):
    """SURVEY.md Appendix B tapered fault: bumps + linspace(0, fault_max, n)[:, None] * plateau mask."""
    lib = nat.ensure()
    torch = _torch()
    out = generate_scene_gpu(SceneSpec("gaussian-bumps", n, n, amp, scale, seed), device)
    seam = torch.as_tensor(plateau_seam(SceneSpec("plateau-discontinuity", n, n, 1.0, fault_scale, seed)),
                           device=out.device)
    lin = torch.as_tensor(np.linspace(0.0, fault_max, n), device=out.device)
    st = ctypes.c_void_p(torch.cuda.current_stream(out.device).cuda_stream)
    nat.check(lib.pu_synth_fault(_p(out), n, n, n, _p(seam), _p(lin), 1.0, st))
    torch.cuda.current_stream(out.device).synchronize()
    return out


def wrap_noise_gpu(truth, sigma, seed):
    """wrap_scene then add_phase_noise (synth.py:93-109) on a device scene, in place on a copy."""
    lib = nat.ensure()
    torch = _torch()
    x = truth.clone()
    rows, cols = x.shape
    st = ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
    nat.check(lib.pu_synth_wrap_noise(_p(x), rows, cols, cols, 0.0, 0, st))           # wrap_scene
    if sigma > 0:
        nat.check(lib.pu_synth_wrap_noise(_p(x), rows, cols, cols, float(sigma), int(seed), st))
    torch.cuda.current_stream(x.device).synchronize()
    return x


def config_scene_gpu(name: str, b: int = 0, device=None):
    """(truth, wrapped) device tensors for BASELINE configs c1..c5 (same recipes as synth.config_scene)."""
    if name == "c1":
        t, sig, ns = generate_scene_gpu(SceneSpec("gaussian-bumps", 512, 512, 40.0, 32.0, 1), device), 0.5, 1001
    elif name == "c2":
        t, sig, ns = generate_scene_gpu(SceneSpec("gaussian-bumps", 2048, 2048, 100.0, 128.0, 2), device), 0.5, 1002
    elif name == "c3":
        t, sig, ns = tapered_fault_gpu(4096, 3, 150.0, 256.0, 4 * np.pi, 512.0, device), 0.5, 1003
    elif name == "c4":
        t, sig, ns = tapered_fault_gpu(16384, 4, 600.0, 1024.0, 4 * np.pi, 2048.0, device), 0.5, 1004
    elif name == "c5":
        t, sig, ns = (generate_scene_gpu(SceneSpec("gaussian-bumps", 1024, 1024, 60.0, 64.0, 100 + b), device),
                      0.5, 2000 + b)
    else:
        raise ValueError(f"unknown config {name!r}")
    return t, wrap_noise_gpu(t, sig, ns)
