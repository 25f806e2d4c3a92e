"""Shared helpers that turn the committed golden fixtures into test cases."""

import numpy as np

from oracle import phaseirls_port as port

GOLDEN_UNWRAP_CASES = [
    "bumps16", "bumps24x31", "bumps32", "noisy64", "noisy64b", "clean128", "noisy96x80",
    "ramp48x40", "row1x30", "col30x1", "pixel1x1", "const8x9", "random4x4",
    "weighted40x36", "lo0_noisy48",
]


def case_inputs(golden_unwrap, golden_meta, name):
    """(x, cv, ch, tau, delta, Params, lo) for a golden unwrap case."""
    meta = golden_meta["unwrap_small"][name]
    x = golden_unwrap[f"{name}/x"]
    cv = golden_unwrap[f"{name}/cv"] if f"{name}/cv" in golden_unwrap else None
    ch = golden_unwrap[f"{name}/ch"] if f"{name}/ch" in golden_unwrap else None
    prm = port.Params(**meta["params"])
    return x, cv, ch, meta["tau"], meta["delta"], prm, meta["lo"]


def golden_trace(golden_unwrap, name):
    keys = ("k", "m_cg", "delta_rel", "h_delta", "cg_iters", "sufficient", "fallback")
    return {k: golden_unwrap[f"{name}/trace_{k}"] for k in keys}


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a - b))
