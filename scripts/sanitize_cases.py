#!/usr/bin/env python3
"""Small unwraps that launch every kernel family once, for compute-sanitizer.

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py

Covers: static-plan transforms (64 x 512 rows, 512-point columns), runtime
(non power-of-two) plans, Bluestein lengths, the fused acceptance + start-up
(fp32, forced on), row bands through the loopback communicator (packed and
peer transposes), the cluster-split 16384-point fp64 transforms, the whole
unwrap through pu_unwrap, the standalone operators and the device metrics.
Sizes are tiny: the tools slow kernels down by 10-100x.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_2401_09961_b200 as pu  # noqa: E402
from paper_2401_09961_b200 import irls, metrics  # noqa: E402
from paper_2401_09961_b200.capi import unwrap_capi  # noqa: E402


def scene(n, m, seed):
    return pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(pu.SceneSpec("gaussian-bumps", n, m, 8.0, 5.0, seed))),
                              0.6, 100 + seed)


def main():
    p = pu.IrlsParams(max_outer_iters=3)
    for dt in ("fp64", "fp32"):
        pu.unwrap(scene(64, 512, 1), params=p, dtype=dt)        # static plans (512 rows / 64 columns runtime)
        pu.unwrap(scene(512, 512, 11), params=p, dtype=dt)      # static 512-point columns (fused first/last stage)
        pu.unwrap(scene(37, 53, 2), params=p, dtype=dt)         # runtime mixed-radix plans
        pu.unwrap(scene(11, 29, 3), params=p, dtype=dt)         # Bluestein (11, 29 prime)
        pu.unwrap_rows(scene(40, 48, 4), params=p, dtype=dt, bands=3)               # bands, packed transpose
        pu.unwrap_rows(scene(40, 48, 5), params=p, dtype=dt, bands=2, peer=True)    # bands, peer transpose
        unwrap_capi(scene(24, 40, 6), params=p, dtype=dt)       # pu_unwrap (C++ host loop)
    irls.FUSED_START = "1"
    pu.unwrap_many([scene(48, 64, 7), scene(48, 64, 8)], params=p, dtype="fp32", concurrency=2)
    irls.FUSED_START = "auto"
    pu.unwrap(scene(3, 16384, 9), params=pu.IrlsParams(max_outer_iters=2), dtype="fp64")   # cluster-split rows
    r = np.random.default_rng(0).standard_normal((16384, 4))
    pu.sylvester_solve(r, 1e-2, dtype="fp64")                                              # cluster-split columns
    x = scene(30, 20, 10)
    res = pu.unwrap(x, params=p)
    metrics.shift_error(res.u, x)
    metrics.kmap_mismatch(res.u, res.u, x)
    sv = pu.SystemVector(res.u, res.vv, res.vh)
    d = pu.DiagonalWeights(np.ones_like(res.vv), np.ones_like(res.vh))
    pu.apply_system(sv, d, 1e-2)
    pu.apply_preconditioner(sv, d, 1e-2)
    import torch
    torch.cuda.synchronize()
    print("sanitize cases done")


if __name__ == "__main__":
    main()
