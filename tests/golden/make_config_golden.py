#!/usr/bin/env python3
"""Reference-precision fixtures at the BASELINE configs (C1, C2, C3, C5 images 0-3).

Runs the UNMODIFIED reference ``phaseirls.unwrap`` (dense-eigenbasis
preconditioner, fp64, default parameters; ``irls.py:132-224``) on the exact
config inputs and stores, per config, what the GPU
parity tests need without shipping whole grids:

* ``F``            eval_f of the result (``objective.py:63-66``), full precision
* ``l1``           the pure L1 misfit sum c|Su - gv| + sum c|uT - gh|
* ``trace_*``      the IrlsTrace (k, m_cg, delta_rel, h_delta, cg_iters, ...)
* ``u_norm`` ...   ||u||, ||vv||, ||vh||, sum|u|
* ``u_sub``        u on the stride-8 subgrid u[::8, ::8] (fp64)
* ``u_rows``       u on rows {0, N/2, N-1}, ``u_cols`` on columns {0, M/2, M-1}
* ``kmap``         rint((u - x)/2pi) as int8 (``phase.py:178-184``), compressed
* ``x_sha256``     checksum of the input (the GPU side regenerates it with
                   paper_2401_09961_b200.synth, pinned by test_synth_golden)

Run in the build container only (imports /root/reference):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_config_golden.py [c1 c5b0 ... c2 c3]

Writes tests/golden/configs/<name>.npz and merges <name> into
tests/golden/configs/meta.json.
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")

import phaseirls  # noqa: E402
from phaseirls import kernels  # noqa: E402
from phaseirls.irls import unwrap  # noqa: E402
from phaseirls.objective import ModelParams, eval_f  # noqa: E402
from phaseirls.operators import SystemVector  # noqa: E402
from phaseirls.phase import WeightField, wrapped_gradients  # noqa: E402
from phaseirls.synth import SceneSpec, add_phase_noise, generate_scene, wrap_scene  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs")
TWO_PI = 2.0 * np.pi


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def tapered_fault(n, seed, amp, scale, fault_max, fault_scale):
    bumps = generate_scene(SceneSpec("gaussian-bumps", n, n, amp, scale, seed))
    mask = generate_scene(SceneSpec("plateau-discontinuity", n, n, 1.0, fault_scale, seed))
    return bumps + np.linspace(0.0, fault_max, n)[:, None] * mask


def config_input(name):
    """SURVEY.md Appendix B, verbatim recipe."""
    if name == "c1":
        t, s, ns = generate_scene(SceneSpec("gaussian-bumps", 512, 512, 40.0, 32.0, 1)), 0.5, 1001
    elif name == "c2":
        t, s, ns = generate_scene(SceneSpec("gaussian-bumps", 2048, 2048, 100.0, 128.0, 2)), 0.5, 1002
    elif name == "c3":
        t, s, ns = tapered_fault(4096, 3, 150.0, 256.0, 4 * np.pi, 512.0), 0.5, 1003
    elif name.startswith("c5b"):
        b = int(name[3:])
        t, s, ns = generate_scene(SceneSpec("gaussian-bumps", 1024, 1024, 60.0, 64.0, 100 + b)), 0.5, 2000 + b
    else:
        raise ValueError(name)
    return add_phase_noise(wrap_scene(t), s, ns)


def run(name):
    x = config_input(name)
    n, m = x.shape
    t0 = time.time()
    res = unwrap(x)
    secs = time.time() - t0
    g = wrapped_gradients(x)
    c = WeightField.uniform(n, m)
    st = SystemVector(res.u, res.vv, res.vh)
    f = eval_f(st, g, c, ModelParams())
    su = np.diff(res.u, axis=0)
    ut = np.diff(res.u, axis=1)
    l1 = float(np.abs(su - g.gv).sum() + np.abs(ut - g.gh).sum())
    kmap = np.rint((res.u - x) / TWO_PI)
    assert np.abs(kmap).max() < 127
    recs = res.trace.records
    out = dict(
        F=np.array(f), l1=np.array(l1),
        u_norm=np.array(np.linalg.norm(res.u)), vv_norm=np.array(np.linalg.norm(res.vv)),
        vh_norm=np.array(np.linalg.norm(res.vh)), u_sum_abs=np.array(np.abs(res.u).sum()),
        u_mean=np.array(res.u.mean()),
        u_sub=res.u[::8, ::8].copy(),
        u_rows=res.u[[0, n // 2, n - 1], :].copy(), u_cols=res.u[:, [0, m // 2, m - 1]].T.copy(),
        kmap=kmap.astype(np.int8),
        trace_k=np.array([r.k for r in recs], dtype=np.int64),
        trace_m_cg=np.array([r.m_cg for r in recs], dtype=np.int64),
        trace_delta_rel=np.array([np.nan if r.delta_rel is None else r.delta_rel for r in recs]),
        trace_h_delta=np.array([r.h_delta for r in recs]),
        trace_cg_iters=np.array([r.cg_iters for r in recs], dtype=np.int64),
        trace_sufficient=np.array([r.sufficient_decrease for r in recs]),
        trace_fallback=np.array([r.fallback_used for r in recs]),
    )
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
    meta_path = os.path.join(OUT, "meta.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    meta[name] = dict(shape=[n, m], x_sha256=sha(x), seconds=secs, F=f, l1=l1,
                      outer=len(recs), pcg=int(sum(r.cg_iters for r in recs)),
                      u_norm=float(out["u_norm"]), reference="phaseirls " + phaseirls.__version__,
                      numpy=np.__version__, backend=kernels.current_backend(),
                      cpu_threads=os.cpu_count())
    with open(meta_path, "w") as fh:
        json.dump(meta, fh, indent=1)
    print(name, json.dumps(meta[name]), flush=True)


def main():
    kernels.warmup()
    names = sys.argv[1:] or ["c1", "c5b0", "c5b1", "c5b2", "c5b3", "c2", "c3"]
    for name in names:
        run(name)


if __name__ == "__main__":
    main()
