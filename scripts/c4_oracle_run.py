#!/usr/bin/env python3
"""C4 (16384², fp64) against the CPU oracle, on the GPU box host.

SURVEY.md §8(c): the unmodified reference cannot run C4 in the build
container (fp64 working set > 62 GB; two O(N³) eigendecompositions), so the
oracle for C4 is the reference algorithm with the exact DCT restatement of
its eigenbasis preconditioner (oracle/phaseirls_port.py, poisson="dct";
pinned against the unmodified reference by tests/test_oracle_golden.py and,
end to end at C3, by tests/golden/configs/c3.npz).  It needs ~100 GB of host
RAM and ~2 h on 16 cores, so it runs once on the GPU box:

    python scripts/c4_oracle_run.py gpurun_out/c4 [outer]

A gpurun call lasts at most an hour and the full oracle unwrap needs about
two, so the comparison runs the first `outer` IRLS iterations (default 12;
IrlsParams(max_outer_iters=outer)) on both sides: the same algorithm, the
same input, a bounded budget.  Besides:

1. GPU: complete fp64 and fp32 unwraps of C4 (F of each, trace lengths), and
   the truncated fp64 / fp32 unwraps for the comparison.
2. CPU: the truncated oracle unwrap.
3. The comparison (tests/parity_configs.py metrics) -> <out>_parity.jsonl and
   a compact fixture <out>_fixture.npz (stride-32 u subgrid, 6 full lines,
   trace, F; the K-map mismatch is computed here, the map is not shipped).
Outputs stay far below gpurun's 64 MiB return limit.
"""

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

TWO_PI = 2.0 * np.pi


def log(msg):
    print(f"[{time.strftime('%H:%M:%S')}] {msg}", flush=True)


def compact(x, u, vv, vh, recs, F):
    n, m = u.shape
    kmap = np.rint((u - x) / TWO_PI)
    return dict(
        F=np.array(F), u_norm=np.array(np.linalg.norm(u)), u_sum_abs=np.array(np.abs(u).sum()),
        u_sub=u[::8, ::8].copy(), u_rows=u[[0, n // 2, n - 1], :].copy(), u_cols=u[:, [0, m // 2, m - 1]].T.copy(),
        kmap=kmap.astype(np.int8),
        trace_k=np.array([r.k for r in recs], dtype=np.int64),
        trace_m_cg=np.array([r.m_cg for r in recs], dtype=np.int64),
        trace_h_delta=np.array([r.h_delta for r in recs]),
        trace_cg_iters=np.array([r.cg_iters for r in recs], dtype=np.int64),
        trace_sufficient=np.array([r.sufficient_decrease for r in recs]),
        trace_fallback=np.array([r.fallback_used for r in recs]),
    )


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c4"
    outer = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
    import parity_configs as pc
    import paper_2401_09961_b200 as pu
    log("generating the C4 input")
    _, x = pu.config_scene("c4")
    full = {}
    for dt in ("fp64", "fp32"):  # complete unwraps: F of each precision
        t0 = time.time()
        res = pu.unwrap(x, dtype=dt)
        secs = time.time() - t0
        F = pc.eval_f_host(x, res.u, res.vv, res.vh)
        full[dt] = {"F": F, "seconds": secs, "outer": len(res.trace.records),
                    "pcg": int(sum(r.cg_iters for r in res.trace.records))}
        log(f"GPU {dt} complete: {secs:.1f} s (incl. upload/download), F = {F!r}, {full[dt]['outer']} outer / "
            f"{full[dt]['pcg']} PCG")
        del res
    full["F_rel_fp32_vs_fp64"] = abs(full["fp32"]["F"] - full["fp64"]["F"]) / full["fp64"]["F"]
    with open(f"{out}_gpu_full.json", "w") as fh:
        json.dump(full, fh, indent=1)
    gpu = {}
    prm = pu.IrlsParams(max_outer_iters=outer)
    for dt in ("fp64", "fp32"):
        res = pu.unwrap(x, params=prm, dtype=dt)
        F = pc.eval_f_host(x, res.u, res.vv, res.vh)
        gpu[dt] = compact(x, res.u, res.vv, res.vh, res.trace.records, F)
        log(f"GPU {dt} truncated to {outer} outer: F = {F!r}, {sum(r.cg_iters for r in res.trace.records)} PCG")
        del res
    pu.release_workspaces()

    from oracle import phaseirls_port as port
    calls = {"n": 0}
    pcg0 = port.pcg

    def pcg_logged(*a, **k):
        t = time.time()
        o = pcg0(*a, **k)
        calls["n"] += 1
        log(f"oracle outer {calls['n']}: budget {a[4]}, {o['iterations']} PCG iterations, {time.time() - t:.0f} s")
        return o

    port.pcg = pcg_logged
    log(f"oracle unwrap (DCT restatement of the reference preconditioner), {outer} outer iterations")
    t0 = time.time()
    st, recs, (gv, gh) = port.unwrap(x, poisson="dct", params=port.Params(max_outer_iters=outer))
    secs = time.time() - t0
    ones = (np.ones_like(gv), np.ones_like(gh))
    F = port.f_l1(st, gv, gh, *ones, 1e-2)
    ref = compact(x, st.u, st.vv, st.vh, recs, F)
    fix = {k: v for k, v in ref.items() if k not in ("kmap", "u_sub")}
    fix["u_sub"] = ref["u_sub"][::4, ::4].copy()   # stride 32
    fix["sub_stride"] = np.array(32)
    fix["max_outer_iters"] = np.array(outer)
    np.savez_compressed(f"{out}_fixture.npz", **fix)
    meta = {"shape": list(x.shape), "seconds": secs, "F": F, "outer": len(recs),
            "pcg": int(sum(r.cg_iters for r in recs)), "cpu_threads": os.cpu_count(), "max_outer_iters": outer,
            "oracle": "oracle/phaseirls_port.py unwrap(poisson='dct', max_outer_iters=%d)" % outer}
    with open(f"{out}_oracle_meta.json", "w") as fh:
        json.dump(meta, fh, indent=1)
    log(f"oracle: {secs:.0f} s, F = {F!r}, {meta['outer']} outer / {meta['pcg']} PCG")
    with open(f"{out}_parity.jsonl", "w") as fh:
        for dt, g in gpu.items():
            r = {"config": "c4", "dtype": dt, "max_outer_iters": outer,
                 "u_rel_sub": rel(g["u_sub"], ref["u_sub"]),
                 "u_rel_lines": rel(np.concatenate([g["u_rows"].ravel(), g["u_cols"].ravel()]),
                                    np.concatenate([ref["u_rows"].ravel(), ref["u_cols"].ravel()])),
                 "u_norm_rel": abs(float(g["u_norm"]) - float(ref["u_norm"])) / float(ref["u_norm"]),
                 "kmap_mismatch": float(np.mean(g["kmap"] != ref["kmap"])),
                 "F": float(g["F"]), "F_ref": float(ref["F"]),
                 "F_rel": abs(float(g["F"]) - float(ref["F"])) / float(ref["F"]),
                 "outer": int(g["trace_k"].size), "outer_ref": int(ref["trace_k"].size),
                 "pcg": int(g["trace_cg_iters"].sum()), "pcg_ref": int(ref["trace_cg_iters"].sum()),
                 "trace_equal": (g["trace_m_cg"].tolist() == ref["trace_m_cg"].tolist()
                                 and g["trace_cg_iters"].tolist() == ref["trace_cg_iters"].tolist())}
            fh.write(json.dumps(r) + "\n")
            log(json.dumps(r))


if __name__ == "__main__":
    main()
