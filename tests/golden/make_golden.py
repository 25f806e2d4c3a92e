#!/usr/bin/env python3
"""Generate golden fixtures by running the UNMODIFIED reference (phaseirls).

Run in the build container only (it imports /root/reference, which the GPU
box does not have):

    NUMBA_CACHE_DIR=/tmp/numba PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

Writes tests/golden/*.npz and *.json.  The committed fixtures pin both the
oracle restatement (oracle/phaseirls_port.py) and the host-side synthetic
input generator (paper_2401_09961_b200/synth.py) to the reference.
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
from phaseirls.irls import IrlsParams, unwrap  # noqa: E402
from phaseirls.objective import (IrlsWeights, ModelParams, candidate_step, eval_f,  # noqa: E402
                                 eval_h_delta, lipschitz_constant, update_weights)
from phaseirls.operators import DiagonalWeights, SystemVector, apply_system, build_rhs  # noqa: E402
from phaseirls.pcg import pcg_solve  # noqa: E402
from phaseirls.phase import GradientField, WeightField, wrap_to_principal, wrapped_gradients  # noqa: E402
from phaseirls.preconditioner import (apply_preconditioner, build_preconditioner,  # noqa: E402
                                      build_spectral_cache, sylvester_solve)
from phaseirls.synth import SceneSpec, add_phase_noise, generate_scene, wrap_scene  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def rng(seed):
    return np.random.Generator(np.random.Philox(key=np.uint64(seed)))


def trace_arrays(trace):
    recs = trace.records
    return dict(
        k=np.array([r.k for r in recs], dtype=np.int64),
        m_cg=np.array([r.m_cg for r in recs], dtype=np.int64),
        delta_rel=np.array([np.nan if r.delta_rel is None else r.delta_rel for r in recs]),
        h_delta=np.array([r.h_delta for r in recs]),
        cg_iters=np.array([r.cg_iters for r in recs], dtype=np.int64),
        sufficient=np.array([r.sufficient_decrease for r in recs]),
        fallback=np.array([r.fallback_used for r in recs]),
    )


def unwrap_cases():
    """(name, x, weights-or-None, model, params, lo) for the small end-to-end cases."""
    cases = []

    def scene(kind, n, m, amp, scale, seed):
        return generate_scene(SceneSpec(kind, n, m, amp, scale, seed))

    cases.append(("bumps16", wrap_scene(scene("gaussian-bumps", 16, 16, 4.0, 4.0, 2)), None, None, None, -np.pi))
    cases.append(("bumps24x31", wrap_scene(scene("gaussian-bumps", 24, 31, 4.0, 6.0, 9)), None, None, None, -np.pi))
    cases.append(("bumps32", wrap_scene(scene("gaussian-bumps", 32, 32, 5.0, 7.0, 3)), None, None, None, -np.pi))
    cases.append(("noisy64", add_phase_noise(wrap_scene(scene("gaussian-bumps", 64, 64, 6.0, 10.0, 0)), 0.3, 1000),
                  None, None, None, -np.pi))
    cases.append(("noisy64b", add_phase_noise(wrap_scene(scene("gaussian-bumps", 64, 64, 6.0, 10.0, 7)), 0.3, 1007),
                  None, None, None, -np.pi))
    cases.append(("clean128", wrap_scene(scene("gaussian-bumps", 128, 128, 8.0, 16.0, 11)), None, None, None, -np.pi))
    cases.append(("noisy96x80", add_phase_noise(wrap_scene(scene("gaussian-bumps", 96, 80, 12.0, 9.0, 5)), 0.5, 55),
                  None, None, None, -np.pi))
    cases.append(("ramp48x40", wrap_to_principal(0.3 * np.arange(48)[:, None] + np.zeros((48, 40)), 0.0),
                  None, None, None, -np.pi))
    cases.append(("row1x30", wrap_to_principal(0.4 * np.arange(30)[None, :], 0.0), None, None, None, -np.pi))
    cases.append(("col30x1", wrap_to_principal(0.4 * np.arange(30)[:, None], 0.0), None, None, None, -np.pi))
    cases.append(("pixel1x1", np.array([[1.0]]), None, None, None, -np.pi))
    cases.append(("const8x9", wrap_to_principal(1.3 * np.ones((8, 9)), 0.0), None, None, None, -np.pi))
    cases.append(("random4x4", rng(77).uniform(0.0, 2 * np.pi, (4, 4)), None, None, None, -np.pi))
    # non-default knobs: model, budget schedule, gradient interval, arc weights
    xw = add_phase_noise(wrap_scene(scene("gaussian-bumps", 40, 36, 7.0, 8.0, 21)), 0.4, 2100)
    r = rng(31)
    cw = WeightField(r.uniform(0.2, 2.0, (39, 36)), r.uniform(0.2, 2.0, (40, 35)))
    cw.cv[5:9, 3:7] = 0.0  # a masked (zero-weight) patch
    cases.append(("weighted40x36", xw, cw, ModelParams(tau=0.05, delta=1e-4),
                  IrlsParams(max_iter_cg_start=3, cg_growth_factor=2.0, rel_improvement_tol=5e-4), -np.pi))
    cases.append(("lo0_noisy48", add_phase_noise(wrap_scene(scene("gaussian-bumps", 48, 48, 5.0, 8.0, 4)), 0.3, 404),
                  None, None, IrlsParams(max_outer_iters=7), 0.0))
    return cases


def make_unwrap_golden():
    out = {}
    meta = {}
    for name, x, c, model, params, lo in unwrap_cases():
        t0 = time.time()
        res = unwrap(x, c, model, params, lo)
        out[f"{name}/x"] = x
        if c is not None:
            out[f"{name}/cv"] = c.cv
            out[f"{name}/ch"] = c.ch
        out[f"{name}/u"] = res.u
        out[f"{name}/vv"] = res.vv
        out[f"{name}/vh"] = res.vh
        for key, val in trace_arrays(res.trace).items():
            out[f"{name}/trace_{key}"] = val
        meta[name] = dict(
            shape=list(x.shape), lo=float(lo),
            tau=(model or ModelParams()).tau, delta=(model or ModelParams()).delta,
            params=vars(params or IrlsParams()) if params is None else params.__dict__,
            outer=len(res.trace), pcg=int(sum(r.cg_iters for r in res.trace.records)),
            seconds=time.time() - t0,
        )
    np.savez_compressed(os.path.join(OUT, "unwrap_small.npz"), **out)
    return meta


def make_kernel_golden():
    out = {}
    r = rng(20240)
    # wrapped gradients, both principal intervals
    x = r.uniform(0.0, 2 * np.pi, (13, 11))
    x[4, 4] = 1.0
    x[3, 4] = 1.0 + np.pi  # an exact-boundary difference (-pi)
    out["grad/x"] = x
    for lo, tag in ((-np.pi, "m"), (0.0, "z")):
        g = wrapped_gradients(x, lo)
        out[f"grad/gv_{tag}"] = g.gv
        out[f"grad/gh_{tag}"] = g.gh
    # system map and rhs
    n, m = 9, 7
    u, vv, vh = r.standard_normal((n, m)), r.standard_normal((n - 1, m)), r.standard_normal((n, m - 1))
    dv, dh = r.uniform(0, 3, (n - 1, m)), r.uniform(0, 3, (n, m - 1))
    tau = 0.03
    a = apply_system(SystemVector(u, vv, vh), DiagonalWeights(dv, dh), tau)
    out.update({"sys/u": u, "sys/vv": vv, "sys/vh": vh, "sys/dv": dv, "sys/dh": dh,
                "sys/au": a.u, "sys/avv": a.vv, "sys/avh": a.vh})
    g = GradientField(r.uniform(-np.pi, np.pi, (n - 1, m)), r.uniform(-np.pi, np.pi, (n, m - 1)))
    b = build_rhs(g, tau)
    out.update({"rhs/gv": g.gv, "rhs/gh": g.gh, "rhs/bu": b.u, "rhs/bv": b.vv, "rhs/bh": b.vh})
    # sylvester (dense-eigenbasis) solves on assorted shapes
    shapes = [(1, 1), (1, 6), (6, 1), (2, 2), (3, 5), (17, 8), (8, 17), (31, 24), (64, 48), (7, 49)]
    for (sn, sm) in shapes:
        rr = r.standard_normal((sn, sm))
        out[f"syl/{sn}x{sm}/r"] = rr
        out[f"syl/{sn}x{sm}/z"] = sylvester_solve(rr, 0.37, build_spectral_cache(sn, sm))
    # objective pieces on a random state
    n, m = 6, 8
    st = SystemVector(r.standard_normal((n, m)), r.standard_normal((n - 1, m)), r.standard_normal((n, m - 1)))
    g = GradientField(r.uniform(-np.pi, np.pi, (n - 1, m)), r.uniform(-np.pi, np.pi, (n, m - 1)))
    c = WeightField(r.uniform(0, 2, (n - 1, m)), r.uniform(0, 2, (n, m - 1)))
    p = ModelParams(tau=0.02, delta=1e-3)
    w = update_weights(st, c, p.delta)
    wprev = IrlsWeights(r.uniform(p.delta / 2, 3.0, (n - 1, m)), r.uniform(p.delta / 2, 3.0, (n, m - 1)))
    lip = lipschitz_constant(c, p)
    cand = candidate_step(st, w, g, c, p, lip)
    out.update({"obj/u": st.u, "obj/vv": st.vv, "obj/vh": st.vh, "obj/gv": g.gv, "obj/gh": g.gh,
                "obj/cv": c.cv, "obj/ch": c.ch, "obj/wv": w.wv, "obj/wh": w.wh,
                "obj/wpv": wprev.wv, "obj/wph": wprev.wh,
                "obj/h_w": np.array(eval_h_delta(st, w, g, c, p)),
                "obj/h_wprev": np.array(eval_h_delta(st, wprev, g, c, p)),
                "obj/f": np.array(eval_f(st, g, c, p)), "obj/lip": np.array(lip),
                "obj/cand_u": cand.u, "obj/cand_vv": cand.vv, "obj/cand_vh": cand.vh})
    # PCG with fixed iteration counts (rel_tol=0) and one converging solve
    n, m = 8, 8
    dv, dh = r.uniform(0, 1e3, (n - 1, m)), r.uniform(0, 1e3, (n, m - 1))
    g = GradientField(r.uniform(-np.pi, np.pi, (n - 1, m)), r.uniform(-np.pi, np.pi, (n, m - 1)))
    tau = 1e-2
    b = build_rhs(g, tau)
    d = DiagonalWeights(dv, dh)
    pc = build_preconditioner(build_spectral_cache(n, m), d, tau)
    x0 = SystemVector(r.standard_normal((n, m)), r.standard_normal((n - 1, m)), r.standard_normal((n, m - 1)))
    out.update({"pcg/dv": dv, "pcg/dh": dh, "pcg/gv": g.gv, "pcg/gh": g.gh,
                "pcg/x0u": x0.u, "pcg/x0v": x0.vv, "pcg/x0h": x0.vh})
    for its, tol in ((0, 0.0), (1, 0.0), (5, 0.0), (12, 0.0), (60, 0.0), (500, 1e-9)):
        o = pcg_solve(lambda v: apply_system(v, d, tau), lambda q: apply_preconditioner(q, pc),
                      b, x0, its, tol)
        key = f"pcg/{its}_{tol:g}"
        out[f"{key}/xu"] = o.x.u
        out[f"{key}/xv"] = o.x.vv
        out[f"{key}/xh"] = o.x.vh
        out[f"{key}/norms"] = np.array(o.residual_norms)
        out[f"{key}/iters"] = np.array(o.iterations)
        out[f"{key}/converged"] = np.array(o.converged)
    np.savez_compressed(os.path.join(OUT, "kernels.npz"), **out)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def tapered_fault(n, seed, amp, scale, fault_max, fault_scale):
    bumps = generate_scene(SceneSpec("gaussian-bumps", n, n, amp, scale, seed))
    mask = generate_scene(SceneSpec("plateau-discontinuity", n, n, 1.0, fault_scale, seed))
    return bumps + np.linspace(0.0, fault_max, n)[:, None] * mask


def make_config_golden(run_c1=True):
    """Checksums of the BASELINE config inputs + the reference's C1 result."""
    meta = {}
    c1 = generate_scene(SceneSpec("gaussian-bumps", 512, 512, 40.0, 32.0, 1))
    x1 = add_phase_noise(wrap_scene(c1), 0.5, 1001)
    c2 = generate_scene(SceneSpec("gaussian-bumps", 2048, 2048, 100.0, 128.0, 2))
    x2 = add_phase_noise(wrap_scene(c2), 0.5, 1002)
    c3 = tapered_fault(4096, 3, 150.0, 256.0, 4 * np.pi, 512.0)
    x3 = add_phase_noise(wrap_scene(c3), 0.5, 1003)
    c5 = generate_scene(SceneSpec("gaussian-bumps", 1024, 1024, 60.0, 64.0, 100))
    x5 = add_phase_noise(wrap_scene(c5), 0.5, 2000)
    meta["sha256"] = {"c1_truth": sha(c1), "c1_x": sha(x1), "c2_x": sha(x2), "c3_truth": sha(c3),
                      "c3_x": sha(x3), "c5b0_x": sha(x5)}
    small = {}
    for kind in ("ramp", "gaussian-bumps", "plateau-discontinuity"):
        for (rows, cols, seed) in ((1, 1, 0), (1, 9, 3), (17, 1, 4), (33, 21, 5)):
            s = generate_scene(SceneSpec(kind, rows, cols, 7.5, 3.0, seed))
            small[f"{kind}/{rows}x{cols}/{seed}"] = sha(s)
            small[f"{kind}/{rows}x{cols}/{seed}/noisy"] = sha(add_phase_noise(wrap_scene(s), 0.7, seed + 9))
    meta["small_scene_sha256"] = small
    if run_c1:
        t0 = time.time()
        res = unwrap(x1)
        secs = time.time() - t0
        g = wrapped_gradients(x1)
        f = eval_f(SystemVector(res.u, res.vv, res.vh), g, WeightField.uniform(512, 512), ModelParams())
        meta["c1"] = dict(seconds=secs, F=f, trace={k: v.tolist() for k, v in trace_arrays(res.trace).items()},
                          u_norm=float(np.linalg.norm(res.u)), u_sum_abs=float(np.abs(res.u).sum()),
                          u_sha256=sha(res.u))
        np.savez_compressed(os.path.join(OUT, "c1_u_f32.npz"), u=res.u.astype(np.float32))
    return meta


def main():
    kernels.warmup()
    meta = {"reference": "phaseirls " + phaseirls.__version__, "numpy": np.__version__,
            "numba_backend": kernels.current_backend()}
    make_kernel_golden()
    meta["unwrap_small"] = make_unwrap_golden()
    meta["configs"] = make_config_golden(run_c1="--no-c1" not in sys.argv)
    with open(os.path.join(OUT, "golden_meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, default=str)
    print(json.dumps({k: v for k, v in meta.items() if k != "unwrap_small"}, default=str)[:2000])


if __name__ == "__main__":
    main()
