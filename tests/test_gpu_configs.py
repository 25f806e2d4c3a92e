"""Reference-precision parity at the BASELINE configs (north_star bars).

Each config input is regenerated bit-identically (paper_2401_09961_b200.synth,
sha256-pinned against the reference's generator) and unwrapped on the GPU;
the result is compared with the unmodified reference's outputs on the same
input (tests/golden/configs, tests/parity_configs.py):

* fp64: u within 1e-8 relative (stride-8 subgrid and 6 full lines), ||u||
  within 1e-10, identical trace (outer count, m_cg, cg_iters), H_delta trace
  within 1e-8, F within 1e-10, whole-grid K-map mismatch fraction 0;
* fp32: F within 1e-3 relative; the K-map mismatch fraction is reported.
"""

import hashlib
import json
import os

import numpy as np
import pytest

import parity_configs as pc

pytestmark = pytest.mark.gpu
pu = pytest.importorskip("paper_2401_09961_b200")

META = pc.available()
SINGLE = [c for c in ("c1", "c2", "c3", "c4") if c in META]
C5 = sorted(c for c in META if c.startswith("c5b"))
REPORT = os.environ.get("PU_PARITY_REPORT")  # optional JSON-lines output (profiles/)


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _input(name):
    x = pu.config_scene("c5", int(name[3:]))[1] if name.startswith("c5b") else pu.config_scene(name)[1]
    sha = hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()
    assert sha == META[name]["x_sha256"], "config input differs from the reference's generator"
    return x


def _report(rec):
    if REPORT:
        with open(REPORT, "a") as fh:
            fh.write(json.dumps(rec) + "\n")


def _check_fp64(r):
    assert r["trace_equal"], r
    assert r["outer"] == r["outer_ref"] and r["pcg"] == r["pcg_ref"], r
    assert r["u_rel_sub"] <= pc.FP64_U_REL, r
    assert r["u_rel_lines"] <= pc.FP64_U_REL, r
    assert r["u_norm_rel"] <= 1e-10, r
    assert r["h_rel"] is not None and r["h_rel"] <= 1e-8, r
    assert r["F_rel"] <= 1e-10, r
    assert r["kmap_mismatch"] in (0.0, None), r


def _params(name):
    """C4's oracle run is bounded to its first IRLS iterations (an hour per
    GPU-box call, scripts/c4_oracle_run.py): the same bound on this side."""
    k = META[name].get("max_outer_iters")
    return pu.IrlsParams(max_outer_iters=int(k)) if k else None


@pytest.mark.parametrize("name", SINGLE)
def test_config_fp64_matches_reference(name):
    x = _input(name)
    res = pu.unwrap(x, params=_params(name), dtype="fp64")
    r = pc.compare(name, x, res.u, res.vv, res.vh, res.trace)
    r["dtype"] = "fp64"
    _report(r)
    _check_fp64(r)


@pytest.mark.parametrize("name", SINGLE)
def test_config_fp32_objective(name):
    x = _input(name)
    res = pu.unwrap(x, params=_params(name), dtype="fp32")
    r = pc.compare(name, x, res.u, res.vv, res.vh, res.trace)
    r["dtype"] = "fp32"
    _report(r)
    assert r["F_rel"] <= pc.FP32_F_REL, r
    assert r["kmap_mismatch"] is None or 0.0 <= r["kmap_mismatch"] <= 1.0


@pytest.mark.skipif(not C5, reason="no C5 fixtures")
@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_config_c5_batch_matches_reference(dtype):
    """C5 runs as a batch (unwrap_many, several unwraps in flight); every
    image must still match its own reference run."""
    xs = [_input(name) for name in C5]
    outs = pu.unwrap_many(xs, dtype=dtype, concurrency=len(xs))
    for name, x, res in zip(C5, xs, outs):
        r = pc.compare(name, x, res.u, res.vv, res.vh, res.trace)
        r["dtype"] = dtype
        _report(r)
        if dtype == "fp64":
            _check_fp64(r)
        else:
            assert r["F_rel"] <= pc.FP32_F_REL, r
