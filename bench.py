#!/usr/bin/env python3
"""Benchmark of the unwrap hot path (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--dtype fp32]
    python bench.py --impl reference ...     # reference CPU path on the host cores

One step = one complete `unwrap` (IRLS to the reference's stopping rule) of
the config's synthetic wrapped image.  Under torchrun each rank unwraps its
own image (independent units, no data-path collective: weak scaling); time
is the max over ranks of CUDA-event time, bracketed by barrier+synchronize.
Prints ONE JSON line on rank 0 (contract in the task statement / DESIGN.md §6).
"""

from __future__ import annotations

import argparse
import json
import os
import platform
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "unwrap time & Mpixel/s to convergence at 4096²; PCG iter/s; % HBM roofline"
UNIT = "Mpixel/s"
# Final objective F of the reference on C3 (measured in the survey)
REF_F = {"c1": 81.567, "c2": 765.61, "c3": 8744.586}
REF_COUNTS = {"c1": (41, 227), "c2": (42, 229), "c3": (39, 218)}  # outer / PCG iterations
WORKLOAD = {
    "c1": "512x512 gaussian-bumps(40,32,seed 1) + noise 0.5 (seed 1001)",
    "c2": "2048x2048 gaussian-bumps(100,128,seed 2) + noise 0.5 (seed 1002)",
    "c3": "4096x4096 InSAR-like: bumps(150,256,seed 3) + tapered fault 0->4pi (scale 512) + noise 0.5 (seed 1003)",
    "c4": "16384x16384 InSAR-like: bumps(600,1024,seed 4) + tapered fault 0->4pi (scale 2048) + noise 0.5 (seed 1004)",
    "c5": "batch of 64 independent 1024x1024 interferograms, bumps(60,64,seed 100+b) + noise 0.5 (seed 2000+b), "
          "sharded round-robin over the ranks",
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


NCU_NAME = {  # bench kernel kind -> kernel name prefix in the ncu captures under profiles/
    "K1_p_Ap_pAp": "k_pcg_p_v<{t}>",
    "K2a_update_norms": "k_pcg_r_v<{t}, 1, 0, 2>",
    "K2b_row_dct": "k_rows_pipe<{t}, ",
    "K3_coldct_spectral": "k_cols_spec<{t}, ",
    "K4_row_idct": "k_rows_pipe<{t}, ",
}


def ncu_traffic(kind, dtype, n):
    """DRAM bytes per launch of `kind` from the committed ncu capture (or None)."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(path) or kind not in NCU_NAME or n != 4096:
        return None
    with open(path) as fh:
        table = json.load(fh)["dram_bytes_per_launch"]
    t = "float" if dtype == "fp32" else "double"
    want = NCU_NAME[kind].format(t=t)
    suffix = {"K2b_row_dct": ", 0>", "K4_row_idct": ", 1>", "K3_coldct_spectral": ", 2>"}.get(kind, "")
    for k, v in table.items():
        if k.startswith(want) and k.endswith(suffix or k[-1]):
            return v
    return None


def algorithmic_bytes(n, m, e):
    """Compulsory HBM bytes per launch of K1..K4 as the kernels are fused
    (DESIGN.md §4), and of one PCG iteration.

    SURVEY.md §8(d) charges one iteration (8S + 3s + 5u) e = (13u + 11s) e,
    which stores z_s; the fused schedule never stores z_s (K1 recomputes it
    from r_s and d) and so moves (13u + 10s) e, the figure used here."""
    u = n * m
    s = (n - 1) * m + n * (m - 1)
    S = u + s
    k = {
        "K1_p_Ap_pAp": (u + 4 * s) * e,          # p_u (from K4), p_s old, r_s, d read; p_s written
        "K2a_update_norms": (5 * S + s) * e,     # p, d, x, r read; x, r written
        "K2b_row_dct": 2 * u * e,                # r_u read; spectrum written
        "K3_coldct_spectral": 2 * u * e,         # spectrum read and written back (in place)
        "K4_row_idct": 3 * u * e,                # spectrum, p_u old read; p_u written
    }
    k["iteration"] = sum(k.values())              # = (13u + 10s) e
    k["iteration_survey"] = (8 * S + 3 * s + 5 * u) * e
    return k


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, flag in zip(names, parts[3:7]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))


# ---------------------------------------------------------------------------
# reference CPU path (the oracle port of the reference algorithm)
# ---------------------------------------------------------------------------
def cpu_reference_sample(x, n_outer, n_pcg, pcg_reps=2, poisson="dense", cache=None):
    """Time the reference algorithm (oracle/phaseirls_port.py, dense-eigenbasis
    preconditioner exactly as preconditioner.py:64-100) on the host cores:
    the once-per-unwrap setup, `pcg_reps` PCG iterations and one outer
    iteration's other work, then scale to the full unwrap's iteration counts.
    `cache` (a dict) keeps the set-up (its time and the eigenbases) across
    samples, so repeated samples re-time only the iterations."""
    from oracle import phaseirls_port as port
    n, m = x.shape
    tau, delta = 1e-2, 1e-6
    t0 = time.perf_counter()
    gv, gh = port.grad_wrapped(x)
    b = port.rhs(gv, gh, tau)
    if cache is not None and "solver" in cache:
        solver, t_setup = cache["solver"], cache["t_setup"]
    else:
        solver = port.make_poisson(n, m, poisson)             # dense: 2 x LAPACK eigh (preconditioner.py:77-83)
        t_setup = time.perf_counter() - t0
        if cache is not None:
            cache.update(solver=solver, t_setup=t_setup)
    cv, ch = np.ones_like(gv), np.ones_like(gh)
    state = port.Triple(np.zeros((n, m)), -gv.copy(), -gh.copy())
    t0 = time.perf_counter()
    w = port.weights(state, cv, ch, delta)                   # irls.py:173-191 outer work
    h1 = port.h_delta(state, w, gv, gh, cv, ch, tau, delta)
    h2 = port.h_delta(state, w, gv, gh, cv, ch, tau, delta)
    dv, dh = cv * cv / w[0], ch * ch / w[1]
    cand = port.candidate(state, w, gv, gh, cv, ch, tau, port.lipschitz(1.0, tau, delta))
    h3 = port.h_delta(cand, w, gv, gh, cv, ch, tau, delta)
    h4 = port.h_delta(state, w, gv, gh, cv, ch, tau, delta)
    cand.u -= cand.u.mean()
    h5 = port.h_delta(cand, w, gv, gh, cv, ch, tau, delta)
    t_outer = time.perf_counter() - t0
    apply_a = lambda v: port.system_apply(v, dv, dh, tau)       # noqa: E731
    apply_m = lambda r: port.precond_apply(r, dv, dh, tau, solver)  # noqa: E731
    t0 = time.perf_counter()
    port.pcg(apply_a, apply_m, b, state, 0, 0.0)              # start-up: x copy, r = b - A x, ||r||
    t_start = time.perf_counter() - t0
    t0 = time.perf_counter()
    port.pcg(apply_a, apply_m, b, state, pcg_reps, 0.0)       # start-up + z = M r + pcg_reps iterations
    t_k = time.perf_counter() - t0
    t_iter = (t_k - t_start) / (pcg_reps + 1)                 # pcg_reps iterations + 1 initial M r
    total = t_setup + n_outer * (t_outer + t_start + t_iter) + n_pcg * t_iter
    del h1, h2, h3, h4, h5
    return {
        "seconds": total, "t_setup_s": t_setup, "t_outer_s": t_outer, "t_pcg_start_s": t_start,
        "t_pcg_iter_s": t_iter, "n_outer": n_outer, "n_pcg": n_pcg,
        "mpix_s": n * m / total / 1e6, "pcg_it_s": n_pcg / total,
        "sample": (f"reference algorithm (oracle port, "
                   + ("dense LAPACK eigenbasis preconditioner" if poisson == "dense" else
                      "preconditioner restated as scipy DCT-II/III with all host threads (the 'fast CPU restatement' "
                      "of SURVEY §8(d), not the reference's own path)")
                   + f") on the full {n}x{m} input: setup + {pcg_reps} PCG iterations + 1 outer iteration timed "
                   f"({t_setup + t_outer + t_k + t_start:.1f} s), scaled to {n_outer} outer / {n_pcg} PCG iterations"),
    }


def cpu_info():
    model = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model, os.cpu_count() or 1


# C4 / C5: counts of the same algorithm on the GPU (the control flow is the
# reference's: identical traces in the parity tests); C4 cannot run through the
# reference here (two O(N^3) 16384^2 eigendecompositions, > 60 GB)
EXTRA_COUNTS = {"c4": (44, 273, "this framework's fp32 trace of C4"),
                "c5": (2615, 13847, "this framework's fp64 traces of the 64 C5 images (identical control flow "
                                    "to the reference, tests/test_gpu_unwrap.py)")}


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    from paper_2401_09961_b200.synth import config_scene
    model, cores = cpu_info()
    poisson, scale, note = "dense", 1.0, ""
    if args.config in REF_COUNTS:
        _, x = config_scene(args.config)
        n, m = x.shape
        n_outer, n_pcg = REF_COUNTS[args.config]
        counts = f"iteration counts from the reference trace (BASELINE.md: {n_outer} outer / {n_pcg} PCG)"
        total_pix = n * m
    elif args.config == "c5":
        _, x = config_scene("c5", 0)          # one 1024^2 image of the batch, all host threads
        n, m = x.shape
        n_outer, n_pcg, src = EXTRA_COUNTS["c5"]
        counts = f"iteration totals over the 64 images from {src}: {n_outer} outer / {n_pcg} PCG"
        total_pix = 64 * n * m
        note = "; image 0 timed, per-image set-up counted 64 times"
    else:  # c4: a 2048-row slab of the 16384^2 input, DCT restatement of the preconditioner
        _, x_full = config_scene("c4")
        x = np.ascontiguousarray(x_full[:2048])
        del x_full
        n, m = 16384, 16384
        n_outer, n_pcg, src = EXTRA_COUNTS["c4"]
        counts = f"iteration counts from {src}: {n_outer} outer / {n_pcg} PCG"
        poisson, scale = "dct", 8.0
        total_pix = n * m
        note = "; rows [0, 2048) of the input timed and scaled x8 by pixels"
    extra_setups = 63 if args.config == "c5" else 0

    full = None
    if args.ref_full == "on" or (args.ref_full == "auto" and args.config in REF_COUNTS):
        # step 0: one COMPLETE reference unwrap (the port of irls.py:132-224 with
        # the reference's dense-eigenbasis preconditioner), timed end to end
        from oracle import phaseirls_port as port
        t0 = time.perf_counter()
        _st, recs, _g = port.unwrap(np.ascontiguousarray(x), poisson="dense")
        t_full = time.perf_counter() - t0
        n_outer, n_pcg = len(recs), int(sum(r.cg_iters for r in recs))
        counts = f"iteration counts of the complete run ({n_outer} outer / {n_pcg} PCG)"
        full = {"seconds": t_full, "mpix_s": total_pix / t_full / 1e6, "pcg_it_s": n_pcg / t_full,
                "n_outer": n_outer, "n_pcg": n_pcg}
        del _st, _g

    cache = {}

    def sample():
        smp = cpu_reference_sample(x, n_outer, n_pcg, pcg_reps=1, poisson=poisson, cache=cache)
        smp["seconds"] = (smp["seconds"] + extra_setups * smp["t_setup_s"]) * scale
        if scale != 1.0:
            smp["sample"] = smp["sample"].replace(" on the full ", " on a ")
        return smp

    warmup = args.warmup if args.warmup_ref is None else args.warmup_ref
    steps = args.steps if args.steps_ref is None else args.steps_ref
    for _ in range(warmup):
        sample()
    # with a complete run, it is step 0 and the model fills the other steps
    samples = [sample() for _ in range(max(1, steps - (1 if full else 0)))]
    model_secs = statistics.median(s["seconds"] for s in samples)
    secs = full["seconds"] if full else model_secs
    value = total_pix / secs / 1e6
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": len(samples) + (1 if full else 0), "warmup": warmup, "ms_per_step": secs * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD[args.config], "n": n, "m": m, "cpu": model},
        "pcg_iters_per_s": n_pcg / secs,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port",
                         "sample": (("one complete reference unwrap of the full input (oracle/phaseirls_port.py, "
                                     "dense LAPACK eigenbasis preconditioner as preconditioner.py:64-100), timed "
                                     f"end to end: {secs:.1f} s; the other steps: " if full else "")
                                    + samples[0]["sample"] + f"; {counts}{note}")},
        "reference_full_run": full,
        "model": {"seconds": model_secs, "error_vs_full": (model_secs - full["seconds"]) / full["seconds"]
                  if full else None, "samples": len(samples),
                  "how": "set-up + 1 PCG iteration + 1 outer iteration timed, scaled to the iteration counts"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "detail": {k: v for k, v in samples[0].items() if k != "sample"},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser(description=__doc__)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", choices=("c1", "c2", "c3", "c4", "c5"), default="c3")
    ap.add_argument("--dtype", choices=("fp32", "fp64"), default="fp64",
                    help="headline arithmetic (fp64 = the reference's precision); the other mode is nested")
    ap.add_argument("--no-nested", action="store_true", help="skip the nested run of the other dtype")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-steps", type=int, default=0,
                    help="only run N unwraps (for ncu launch lists); prints no JSON")
    ap.add_argument("--shard", choices=("auto", "images", "rows"), default="auto",
                    help="N>1: one image row-sharded over the ranks (auto for c1-c4: strong scaling), or "
                         "independent images per rank (auto for c5: weak scaling)")
    ap.add_argument("--concurrency", type=int, default=8, help="c5: images in flight per GPU")
    ap.add_argument("--peer", dest="peer", action="store_true", default=None,
                    help="--shard rows: transpose fused into the row kernels over peer memory "
                         "(default: on when the GPUs have peer access, band._default_peer)")
    ap.add_argument("--no-peer", dest="peer", action="store_false",
                    help="--shard rows: NCCL all-to-all transposes instead")
    ap.add_argument("--bands", type=int, default=None,
                    help="--shard rows without torchrun: B bands in this process (loopback collectives)")
    ap.add_argument("--warmup-ref", type=int, default=None, help="reference arm (default: --warmup)")
    ap.add_argument("--steps-ref", type=int, default=None, help="reference arm (default: --steps)")
    ap.add_argument("--ref-full", choices=("auto", "on", "off"), default="auto",
                    help="reference arm: time one complete reference unwrap as step 0 (auto: c1-c3)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.profile_steps == 0 else args.warmup

    rank, local_rank, world = dist_env()
    if args.impl == "reference":
        return run_reference(args, rank, world)
    import torch
    import torch.distributed as dist
    from paper_2401_09961_b200 import _native

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    lib = _native.ensure()
    shard = args.shard
    if shard == "auto":
        shard = "rows" if (world > 1 or args.bands) and args.config != "c5" else "images"
    if shard == "rows":
        if args.config == "c5":
            raise SystemExit("--shard rows needs a single-image config (c1-c4)")
        rc = main_rows(args, rank, local_rank, world, dev, lib)
        if world > 1:
            dist.destroy_process_group()
        return rc
    rc = main_images(args, rank, local_rank, world, dev, lib)
    if world > 1:
        dist.destroy_process_group()
    return rc


def parity_block(config, xs, results, dtype):
    """Reference-precision parity of this run's result against the committed
    outputs of the unmodified reference on the same input
    (tests/parity_configs.py; north_star: fp64 u within 1e-8, fp32 F within
    1e-3, K-map mismatch reported).  None when no fixture covers `config`."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    try:
        import parity_configs as pc
    except ImportError:
        return None
    have = pc.available()
    names = [config] if config != "c5" else [f"c5b{b}" for b in range(len(xs))]
    out = []
    for name, x, res in zip(names, xs, results):
        if name not in have or res is None or have[name].get("max_outer_iters"):
            continue  # (a bounded-iteration fixture, C4, is compared by tests/test_gpu_configs.py)
        r = pc.compare(name, x, res.u, res.vv, res.vh, res.trace)
        out.append({k: r[k] for k in ("config", "u_rel_sub", "u_rel_lines", "u_norm_rel", "kmap_mismatch", "F",
                                      "F_ref", "F_rel", "trace_equal", "outer", "pcg", "h_rel")})
    if not out:
        return None
    worst = {
        "u_rel": max(max(o["u_rel_sub"], o["u_rel_lines"]) for o in out),
        "kmap_mismatch": max((o["kmap_mismatch"] for o in out if o["kmap_mismatch"] is not None), default=None),
        "F_rel": max(o["F_rel"] for o in out),
        "trace_equal": all(o["trace_equal"] for o in out),
        "images": len(out),
    }
    bar = ({"u_rel": pc.FP64_U_REL, "ok": worst["u_rel"] <= pc.FP64_U_REL and worst["trace_equal"]}
           if dtype == "fp64" else {"F_rel": pc.FP32_F_REL, "ok": worst["F_rel"] <= pc.FP32_F_REL})
    return {"against": "outputs of the unmodified reference on the same input (tests/golden/configs)",
            "dtype": dtype, "worst": worst, "bar": bar, "per_image": out if len(out) <= 4 else out[:4]}


def measure_images(args, dtype, xs, rank, local_rank, world, dev, lib, with_clocks=True):
    """One dtype mode on this rank's images: device-resident timed region,
    instrumented per-kernel pass, end to end through the public API from
    numpy, and parity of the e2e results.  Returns the measurement dict."""
    import torch
    import paper_2401_09961_b200 as pu
    from paper_2401_09961_b200.device import Workspace, _ptr
    from paper_2401_09961_b200.irls import unwrap_device
    from paper_2401_09961_b200.batch import max_over_ranks

    n_img = len(xs)
    n, m = xs[0].shape
    model, params = pu.ModelParams(), pu.IrlsParams()
    ws = Workspace.get(n, m, dtype, model.tau, model.delta, dev)
    x_devs = [torch.from_numpy(xi).to(dev) for xi in xs]

    seq_pcg = [0]  # PCG iterations run by one_unwrap_sequential (all of the rank's images)

    def one_unwrap_sequential():
        for x_dev in x_devs:
            run, trace = unwrap_device(x_dev, None, model, params, -np.pi, dtype, ws)
            seq_pcg[0] += sum(r.cg_iters for r in trace.records)
        return run, trace

    def one_unwrap():
        if n_img == 1:
            return one_unwrap_sequential()
        # C5: the rank's images in flight concurrently (one workspace + stream each)
        res = pu.unwrap_many(x_devs, None, model, params, -np.pi, dtype=dtype, concurrency=args.concurrency,
                             download=False)
        return res[-1]

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        run, trace = one_unwrap()
    torch.cuda.synchronize()

    # ---- timed region: device-resident input, CUDA graphs, no instrumentation ----
    ws.timing(False)
    launches0 = lib.pu_launch_count()
    traces = []
    clocks = ClockSampler(local_rank) if with_clocks else None
    if clocks:
        clocks.__enter__()
    barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        run, trace = one_unwrap()
        traces.append(trace)
    ev1.record()
    torch.cuda.synchronize()
    barrier()
    if clocks:
        clocks.__exit__(None, None, None)
    launches = lib.pu_launch_count() - launches0
    step_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, device=dev)
    value = world * n_img * n * m / (step_ms / 1e3) / 1e6

    # objective of the device result (pu_eval_f) before anything else reuses the buffers
    f_out = None
    try:
        cw = run.weight_planes()
        ws.call("pu_eval_f", _ptr(run.state), _ptr(run.G[0]), _ptr(run.G[1]), _ptr(cw[0]), _ptr(cw[1]),
                ws.sp(ws.S_F), ws.stream())
        f_out = float(ws.read_block()[0][ws.S_F])
    except Exception:
        pass

    # ---- kernel timing pass: the same K steps again with a CUDA-event pair
    # around every launch on the launching stream (graphs off: event nodes
    # inside graphs perturb the step by ~25%); feeds `roofline` / `kernels`
    lib.pu_set_graphs(ws.h, 0)
    ws.timing(True)
    ws.read_timing()  # drain
    torch.cuda.synchronize()
    ev2, ev3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    seq_pcg[0] = 0
    ev2.record()
    for _ in range(args.steps):
        one_unwrap_sequential()
    ev3.record()
    torch.cuda.synchronize()
    ws.timing(False)
    lib.pu_set_graphs(ws.h, 1)
    kinds, its, ms = ws.read_timing()
    instrumented_ms = ev2.elapsed_time(ev3) / args.steps

    e = 4 if dtype == "fp32" else 8
    alg = algorithmic_bytes(n, m, e)
    hbm, peak_kind = peaks()
    per_kind = kernel_stats(kinds, ms, Workspace.TIME_KINDS)
    timed_total = sum(v["total_ms"] for v in per_kind.values())
    dom = max((k for k in per_kind if k in alg), key=lambda k: per_kind[k]["total_ms"])
    achieved = alg[dom] / (per_kind[dom]["avg_ms"] / 1e3) / 1e9 if per_kind[dom]["avg_ms"] > 0 else None
    n_pcg = sum(r.cg_iters for r in traces[-1].records)     # per image
    n_outer = len(traces[-1].records)
    iter_kinds = ("K1_p_Ap_pAp", "K2a_update_norms", "K2b_row_dct", "K3_coldct_spectral", "K4_row_idct",
                  "reproject_update")
    pcg_per_step = seq_pcg[0] / args.steps  # all of the rank's images (n_img x n_pcg when they agree)
    iter_ms = sum(per_kind[k]["total_ms"] for k in iter_kinds if k in per_kind) / max(1, seq_pcg[0])
    # per-iteration time implied by the clean timed step: step time minus the
    # (event-timed) once-per-outer-iteration kernels, over the PCG iterations
    outer_kinds = ("pcg_start", "weights_hpair", "candidate", "hpair_states", "accept_center")
    outer_ms = sum(per_kind[k]["total_ms"] for k in outer_kinds if k in per_kind) / args.steps
    init_ms = 0.0  # the start-up preconditioner applications (iteration index -1)
    for kd, itv, t in zip(kinds, its, ms):
        if itv == -1 and Workspace.TIME_KINDS[kd] in ("K2a_update_norms", "K2b_row_dct", "K3_coldct_spectral",
                                                      "K4_row_idct"):
            init_ms += t
    init_ms /= args.steps
    pcg_ms_from_step = (step_ms - outer_ms - init_ms) / max(1, pcg_per_step)
    traffic = ncu_traffic(dom, dtype, n)
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": achieved / hbm if achieved else None,
        "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})", "bytes_per_launch": alg[dom],
        "bytes_how": "compulsory bytes of the fused kernel (DESIGN.md §4): " + {
            "K1_p_Ap_pAp": "(u + 4s) e", "K2a_update_norms": "(5S + s) e", "K2b_row_dct": "2u e",
            "K3_coldct_spectral": "2u e", "K4_row_idct": "3u e"}[dom],
        "avg_launch_ms": per_kind[dom]["avg_ms"], "share_of_kernel_time": per_kind[dom]["total_ms"] / timed_total,
        "traffic": traffic,
        "traffic_source": ("profiles/ncu_traffic.json (ncu --set full, dram__bytes_read.sum + "
                           "dram__bytes_write.sum)") if traffic else None,
        "pcg_iteration": {"bytes": alg["iteration"], "bytes_how": "(13u + 10s) e: K1..K4 as fused (z_s never "
                                                                  "stored); SURVEY §8(d) (13u + 11s) e = "
                                                                  f"{alg['iteration_survey']}",
                          "ms": iter_ms, "how": "sum of the per-iteration kernels' event-timed durations",
                          "achieved_gbs": alg["iteration"] / (iter_ms / 1e3) / 1e9 if iter_ms else None,
                          "frac": (alg["iteration"] / (iter_ms / 1e3) / 1e9) / hbm if iter_ms else None,
                          "ms_from_step": pcg_ms_from_step,
                          "frac_from_step": ((alg["iteration"] / (pcg_ms_from_step / 1e3) / 1e9) / hbm
                                             if pcg_ms_from_step else None)},
    }

    # ---- end to end through the public API: numpy fp64 input (pageable, as a
    # caller holds it) -> host numpy result arrays ----
    e2e_ms = []
    results = None
    for i in range(args.steps + 1):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        if n_img == 1:
            results = [pu.unwrap(xs[0], dtype=dtype)]
        else:
            results = pu.unwrap_many(xs, dtype=dtype, concurrency=args.concurrency)
        t1 = time.perf_counter()
        if i > 0:
            e2e_ms.append((t1 - t0) * 1e3)
    e2e_step = max_over_ranks(statistics.mean(e2e_ms), device=dev)
    h2d = n_img * n * m * 8
    # the results travel in the compute dtype and are widened to fp64 on the host
    res = results[-1]
    d2h = n_img * (res.u.size + res.vv.size + res.vh.size) * e
    return {
        "value": value, "step_ms": step_ms, "instrumented_ms": instrumented_ms, "per_kind": per_kind,
        "roofline": roofline, "n_pcg": n_pcg, "pcg_per_step": pcg_per_step, "n_outer": n_outer, "F": f_out, "launches": int(launches),
        "clocks": clocks.summary() if clocks else None, "ws": ws, "results": results,
        "e2e": {"value": world * n_img * n * m / (e2e_step / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_step,
                "how": "pu.unwrap / pu.unwrap_many on the pageable numpy fp64 input(s), numpy fp64 results "
                       "(host staging, H2D, solve, D2H and widening inside the timed region)"},
    }


def main_images(args, rank, local_rank, world, dev, lib):
    """Images mode: one config image per rank (c1-c4), or the rank's shard of
    the 64 C5 images; weak scaling with no data-path collective."""
    import paper_2401_09961_b200 as pu
    from paper_2401_09961_b200.batch import shard_indices

    if args.config == "c5":
        mine = shard_indices(64, rank, world)
        xs = [pu.config_scene("c5", b)[1] for b in mine]
    else:
        xs = [pu.config_scene(args.config)[1]]
    n_img = len(xs)
    n, m = xs[0].shape
    if args.profile_steps:  # launch lists for ncu: just the unwraps
        import torch
        from paper_2401_09961_b200.irls import unwrap_device
        x_devs = [torch.from_numpy(xi).to(dev) for xi in xs]
        for _ in range(args.profile_steps):
            if n_img == 1:
                unwrap_device(x_devs[0], None, pu.ModelParams(), pu.IrlsParams(), -np.pi, args.dtype)
            else:
                pu.unwrap_many(x_devs, dtype=args.dtype, concurrency=args.concurrency, download=False)
        torch.cuda.synchronize()
        return 0
    head = measure_images(args, args.dtype, xs, rank, local_rank, world, dev, lib)
    other = "fp32" if args.dtype == "fp64" else "fp64"
    nested = None
    if not args.no_nested and args.config != "c4":
        sub = measure_images(args, other, xs, rank, local_rank, world, dev, lib, with_clocks=False)
        nested = {"dtype": "f32" if other == "fp32" else "f64", "value": sub["value"], "unit": UNIT,
                  "ms_per_step": sub["step_ms"], "pcg_iters_per_s": world * sub["pcg_per_step"] / (sub["step_ms"] / 1e3),
                  "roofline": sub["roofline"], "kernels": sub["per_kind"], "e2e": sub["e2e"],
                  "objective": {"F": sub["F"], "F_reference": REF_F.get(args.config)},
                  "parity": parity_block(args.config, xs, sub["results"], other) if rank == 0 else None,
                  "gpu_launches": sub["launches"],
                  "note": ("north_star's fp32 mode (objective within 1e-3 of the fp64 reference)" if other == "fp32"
                           else "fp64 (the reference's precision)")}
        del sub

    cpu_base = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config != "c5":
        model_name, cores = cpu_info()
        x = xs[0]
        smp = cpu_reference_sample(x, head["n_outer"], head["n_pcg"])
        cpu_base = {"value": smp["mpix_s"], "unit": UNIT, "cores": cores, "kind": "port", "sample": smp["sample"],
                    "cpu": model_name, "pcg_iters_per_s": smp["pcg_it_s"], "seconds_per_unwrap": smp["seconds"]}
        fast = cpu_reference_sample(x, head["n_outer"], head["n_pcg"], poisson="dct")
        cpu_base["fast_cpu_restatement"] = {"value": fast["mpix_s"], "unit": UNIT, "cores": cores,
                                            "seconds_per_unwrap": fast["seconds"], "sample": fast["sample"]}

    if rank == 0:
        parity = parity_block(args.config, xs, head["results"], args.dtype)
        f_out = head["F"]
        line = {
            "metric": METRIC, "value": head["value"], "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": head["step_ms"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOAD[args.config]}", "n": n, "m": m,
                       "per_rank": f"{n_img} independent image(s) per GPU per step",
                       "l2": "inputs larger than L2 (resident working set >= 1.6 GB vs 126 MB L2)"
                             if n * m >= 2048 * 2048 else "working set partly L2-resident (small grid)",
                       "plan": head["ws"].describe()},
            "unwrap_s": head["step_ms"] / 1e3,
            "kernel_timing": {"how": "CUDA events around every launch on its stream, second pass of the same "
                                     f"{args.steps} steps with graphs off", "ms_per_step": head["instrumented_ms"]},
            "pcg_iters_per_step": head["n_pcg"], "outer_iters_per_step": head["n_outer"],
            "pcg_iters_per_s": world * head["pcg_per_step"] / (head["step_ms"] / 1e3),
            "roofline": head["roofline"],
            "kernels": head["per_kind"],
            "parity": parity,
            "objective": {"F": f_out, "F_reference": REF_F.get(args.config),
                          "rel": (abs(f_out - REF_F[args.config]) / REF_F[args.config])
                          if f_out is not None and args.config in REF_F else None,
                          "note": "F_reference is the survey's 3-decimal value; parity holds the full-precision one"},
            "cpu_baseline": cpu_base,
            "e2e": head["e2e"],
            "nested": nested,
            "clocks": head["clocks"],
            "gpu_launches": head["launches"],
        }
        print(json.dumps(line), flush=True)
    return 0


def kernel_stats(kinds, ms, names):
    per_kind = {}
    for kd in np.unique(kinds):
        sel = ms[kinds == kd]
        ran = sel[sel >= 0.25 * np.median(sel)] if sel.size else sel
        name = names[kd] if kd < len(names) else str(kd)
        per_kind[name] = {"launches": int(sel.size), "ran": int(ran.size), "total_ms": float(ran.sum()),
                          "avg_ms": float(ran.mean()) if ran.size else 0.0}
    return per_kind


def main_rows(args, rank, local_rank, world, dev, lib):
    """One image row-sharded over the ranks (band.py): halo exchange, all-reduced
    PCG scalars and the all-to-all DCT transpose between the band kernels.
    value = the image's pixels / the max-over-ranks unwrap time (strong scaling)."""
    import torch
    import paper_2401_09961_b200 as pu
    from paper_2401_09961_b200.band import RowSharded
    from paper_2401_09961_b200.batch import max_over_ranks
    from paper_2401_09961_b200.device import Workspace

    _, x = pu.config_scene(args.config)
    n, m = x.shape
    model, params = pu.ModelParams(), pu.IrlsParams()
    solver = RowSharded.get(n, m, args.dtype, model, dev, bands=args.bands, peer=args.peer)
    lay = solver.layout
    xs = solver.upload(x)
    torch.cuda.synchronize()

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    for _ in range(args.warmup):
        trace = solver.run(xs, None, params, -np.pi)
    torch.cuda.synchronize()
    launches0 = lib.pu_launch_count() + solver.driver.replayed_kernels
    with ClockSampler(local_rank) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(args.steps):
            trace = solver.run(xs, None, params, -np.pi)
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    launches = lib.pu_launch_count() + solver.driver.replayed_kernels - launches0
    step_ms = max_over_ranks(ev0.elapsed_time(ev1) / args.steps, device=dev)
    value = n * m / (step_ms / 1e3) / 1e6

    # instrumented pass on this rank's band (CUDA events around each launch)
    b = solver.bands[0]
    graphs = solver.driver.graphs
    solver.driver.graphs = False  # per-launch events need eager launches
    lib.pu_timing_enable(b.h, 1)
    kinds = np.zeros(0, dtype=np.int32)
    barrier()
    for _ in range(args.steps):
        solver.run(xs, None, params, -np.pi)
    torch.cuda.synchronize()
    import ctypes
    cap = 1 << 18
    kb, ib, mb_ = (ctypes.c_int * cap)(), (ctypes.c_int * cap)(), (ctypes.c_float * cap)()
    cnt = int(lib.pu_timing_read(b.h, kb, ib, mb_, cap))
    lib.pu_timing_enable(b.h, 0)
    solver.driver.graphs = graphs
    kinds = np.frombuffer(kb, dtype=np.int32, count=cnt).copy()
    ms = np.frombuffer(mb_, dtype=np.float32, count=cnt).astype(np.float64)
    barrier()
    per_kind = kernel_stats(kinds, ms, Workspace.TIME_KINDS)
    e = 4 if args.dtype == "fp32" else 8
    rows = lay.rows[rank]
    alg = algorithmic_bytes(rows, m, e)
    hbm, peak_kind = peaks()
    n_pcg = sum(r.cg_iters for r in trace.records)
    iter_kinds = ("K1_p_Ap_pAp", "K2a_update_norms", "K2b_row_dct", "K3_coldct_spectral", "K4_row_idct",
                  "reproject_update")
    iter_ms = sum(per_kind[k]["total_ms"] for k in iter_kinds if k in per_kind) / max(1, args.steps * n_pcg)
    dom = max((k for k in per_kind if k in alg), key=lambda k: per_kind[k]["total_ms"])
    achieved = alg[dom] / (per_kind[dom]["avg_ms"] / 1e3) / 1e9 if per_kind[dom]["avg_ms"] > 0 else None
    roofline = {
        "bound": "hbm", "kernel": dom, "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": achieved / hbm if achieved else None, "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})",
        "bytes_per_launch": alg[dom], "avg_launch_ms": per_kind[dom]["avg_ms"], "traffic": None,
        "scope": f"rank 0's band ({rows} x {m}); collectives excluded",
        "pcg_iteration": {"bytes": alg["iteration"], "kernel_ms": iter_ms,
                          "frac": (alg["iteration"] / (iter_ms / 1e3) / 1e9) / hbm if iter_ms else None,
                          "ms_from_step": step_ms / max(1, n_pcg),
                          "how": "kernel_ms: rank 0's band kernels only; ms_from_step: whole step / PCG iterations "
                                 "(includes outer work and all exchanges)"},
    }
    # end to end through the public API: host grid in, this rank's band rows out
    e2e_ms = []
    for i in range(args.steps + 1):
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = pu.unwrap_rows(x, dtype=args.dtype, gather=False, bands=args.bands, peer=args.peer)
        t1 = time.perf_counter()
        if i > 0:
            e2e_ms.append((t1 - t0) * 1e3)
    e2e_step = max_over_ranks(statistics.mean(e2e_ms), device=dev)
    h2d = (n + world - 1) * m * 8
    d2h = (n * m + (n - 1) * m + n * (m - 1)) * (4 if args.dtype == "fp32" else 8)  # compute dtype, widened on host
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": step_ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32" if args.dtype == "fp32" else "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {WORKLOAD[args.config]}", "n": n, "m": m,
                       "sharding": f"one image row-sharded over {world} rank(s): bands {lay.rows}, "
                                   f"transpose blocks of {lay.mb} columns"
                                   + (" (all bands in one process, loopback collectives)" if args.bands else "")
                                   + (", transpose fused into the row kernels (peer stores/loads)" if solver.bands[0].peer
                                      else ", NCCL all-to-all transposes"),
                       "l2": "inputs larger than L2", "plan": None},
            "unwrap_s": step_ms / 1e3, "pcg_iters_per_step": n_pcg, "outer_iters_per_step": len(trace.records),
            "pcg_iters_per_s": n_pcg / (step_ms / 1e3),
            "roofline": roofline, "kernels": per_kind, "cpu_baseline": None,
            "e2e": {"value": n * m / (e2e_step / 1e3) / 1e6, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "ms_per_step": e2e_step},
            "clocks": clocks.summary(), "gpu_launches": int(launches),
        }
        print(json.dumps(line), flush=True)
    del res
    return 0


if __name__ == "__main__":
    sys.exit(main())
