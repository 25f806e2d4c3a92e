"""Compare band (loopback) and single-grid traces on one golden case."""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
import paper_2401_09961_b200 as pu
from cases import case_inputs, golden_trace
name = sys.argv[1] if len(sys.argv) > 1 else "weighted40x36"
g = np.load("tests/golden/unwrap_small.npz")
import json
meta = json.load(open("tests/golden/golden_meta.json"))
x, cv, ch, tau, delta, prm, lo = case_inputs(g, meta, name)
c = None if cv is None else pu.WeightField(cv, ch)
single = pu.unwrap(x, c, pu.ModelParams(tau, delta), pu.IrlsParams(**prm.__dict__), lo, dtype="fp64")
want = golden_trace(g, name)
for nb in (1, 2, 3):
    res = pu.unwrap_rows(x, c, pu.ModelParams(tau, delta), pu.IrlsParams(**prm.__dict__), lo, dtype="fp64", bands=nb)
    print("bands", nb, "outer", len(res.trace.records), "single", len(single.trace.records), "ref", len(want["cg_iters"]))
    for a, b in zip(res.trace.records, single.trace.records):
        if a.cg_iters != b.cg_iters or abs(a.h_delta - b.h_delta) > 1e-9 * abs(b.h_delta):
            print("  k", a.k, a.cg_iters, b.cg_iters, a.h_delta, b.h_delta, a.delta_rel, b.delta_rel, a.fallback_used, b.fallback_used)
            break
    print("  u rel", np.linalg.norm(res.u - single.u) / np.linalg.norm(single.u))
