"""Reference-precision parity at the BASELINE configs (checker only).

Compares one GPU unwrap of a config input with the committed outputs of the
UNMODIFIED reference on the same input (tests/golden/configs/<name>.npz,
written by tests/golden/make_config_golden.py):

* ``u_rel_sub``    ||u - u_ref|| / ||u_ref|| on the stride-8 subgrid
* ``u_rel_lines``  the same over 3 full rows + 3 full columns
* ``u_norm_rel``   | ||u|| - ||u_ref|| | / ||u_ref||  (whole grid)
* ``kmap_mismatch`` mean(rint((u - x)/2pi) != rint((u_ref - x)/2pi)) over the
                   WHOLE grid (phase.py:178-184)
* ``F_rel``        |F - F_ref| / F_ref, F = eval_f (objective.py:63-66) in fp64
* ``trace_equal``  identical outer count, m_cg and cg_iters per iteration
* ``h_rel``        max relative difference of the traced H_delta values

north_star's bars: fp64 -> u within 1e-8 relative; fp32 -> F within 1e-3
relative; the K-map mismatch is reported.  Used by tests/test_gpu_configs.py
and bench.py (parity block of the JSON line); the GPU box has no reference,
only these fixtures.
"""

from __future__ import annotations

import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
CONFIG_DIR = os.path.join(HERE, "golden", "configs")
TWO_PI = 2.0 * np.pi

FP64_U_REL = 1e-8      # north_star, fp64 mode
FP32_F_REL = 1e-3      # north_star, fp32 mode


def available():
    meta = os.path.join(CONFIG_DIR, "meta.json")
    if not os.path.exists(meta):
        return {}
    with open(meta) as fh:
        return json.load(fh)


def load(name):
    return np.load(os.path.join(CONFIG_DIR, f"{name}.npz"))


def _wrap(a, lo=-np.pi):
    # phase.py:118-137 (host restatement, checker side)
    y = a - TWO_PI * np.floor((a - lo) / TWO_PI)
    y = np.where(y >= lo + TWO_PI, y - TWO_PI, y)
    return np.where(y < lo, y + TWO_PI, y)


def eval_f_host(x, u, vv, vh, tau=1e-2):
    """objective.py:63-66 with uniform weights, fp64 on the host."""
    gv = _wrap(np.diff(x, axis=0))
    gh = _wrap(np.diff(x, axis=1))
    rv = np.diff(u, axis=0) - gv - vv
    rh = np.diff(u, axis=1) - gh - vh
    l1 = float(np.abs(vv).sum()) + float(np.abs(vh).sum())
    return l1 + (float(np.vdot(rv, rv)) + float(np.vdot(rh, rh))) / (2.0 * tau)


def _rel(a, b):
    den = float(np.linalg.norm(b))
    return float(np.linalg.norm(np.asarray(a, np.float64) - b)) / den if den > 0 else float(np.linalg.norm(a))


def compare(name, x, u, vv, vh, trace):
    ref = load(name)
    n, m = u.shape
    out = {"config": name}
    st = int(ref["sub_stride"]) if "sub_stride" in ref.files else 8
    out["u_rel_sub"] = _rel(u[::st, ::st], ref["u_sub"])
    lines_gpu = np.concatenate([u[[0, n // 2, n - 1], :].ravel(), u[:, [0, m // 2, m - 1]].T.ravel()])
    lines_ref = np.concatenate([ref["u_rows"].ravel(), ref["u_cols"].ravel()])
    out["u_rel_lines"] = _rel(lines_gpu, lines_ref)
    un = float(np.linalg.norm(u))
    out["u_norm_rel"] = abs(un - float(ref["u_norm"])) / float(ref["u_norm"])
    k = np.rint((u - x) / TWO_PI)
    if "kmap" in ref.files:
        out["kmap_mismatch"] = float(np.mean(k != ref["kmap"].astype(np.float64)))
    elif "kmap_diff" in ref.files:  # stored as differences along rows
        kref = np.cumsum(ref["kmap_diff"].astype(np.int32), axis=1).astype(np.float64)
        out["kmap_mismatch"] = float(np.mean(k != kref))
    else:  # C4: the map is not shipped (measured on the GPU box, profiles/r02_c4_parity.jsonl)
        out["kmap_mismatch"] = None
    f = eval_f_host(x, u, vv, vh)
    out["F"] = f
    out["F_ref"] = float(ref["F"])
    out["F_rel"] = abs(f - float(ref["F"])) / float(ref["F"])
    recs = trace.records
    m_cg = [r.m_cg for r in recs]
    cg = [r.cg_iters for r in recs]
    out["outer"], out["outer_ref"] = len(recs), int(ref["trace_k"].size)
    out["pcg"], out["pcg_ref"] = int(sum(cg)), int(ref["trace_cg_iters"].sum())
    out["trace_equal"] = (m_cg == ref["trace_m_cg"].tolist() and cg == ref["trace_cg_iters"].tolist())
    if len(recs) == ref["trace_h_delta"].size:
        h = np.array([r.h_delta for r in recs])
        out["h_rel"] = float(np.max(np.abs(h - ref["trace_h_delta"]) / np.abs(ref["trace_h_delta"])))
    else:
        out["h_rel"] = None
    return out
