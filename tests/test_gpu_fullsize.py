"""Parity at BASELINE.json's full sizes (C2 2048², C3 4096²) against the
reference's own runs of the same inputs (measured with the
unmodified reference: C2 F = 765.61 after 42 outer / 229 PCG iterations,
C3 F = 8744.586 after 39 / 218).  The inputs are bit-identical to the
reference's generators (tests/test_synth_golden.py pins their sha256)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
pu = pytest.importorskip("paper_2401_09961_b200")

REF = {"c2": (765.61, 42, 229), "c3": (8744.586, 39, 218)}


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.fixture(scope="module")
def scenes():
    return {c: pu.config_scene(c)[1] for c in ("c2", "c3")}


def _objective(res, x):
    """objective.py:63-66 (F) of a result, evaluated in fp64 on the host."""
    from oracle import phaseirls_port as port
    gv, gh = port.grad_wrapped(x)
    ones = (np.ones_like(gv), np.ones_like(gh))
    return port.f_l1(port.Triple(res.u, res.vv, res.vh), gv, gh, *ones, 1e-2)


@pytest.mark.parametrize("cfg,dtype", [("c2", "fp32"), ("c2", "fp64"), ("c3", "fp32"), ("c3", "fp64")])
def test_full_size_objective_and_counts(scenes, cfg, dtype):
    x = scenes[cfg]
    f_ref, outer, pcg = REF[cfg]
    res = pu.unwrap(x, dtype=dtype)
    recs = res.trace.records
    assert len(recs) == outer and sum(r.cg_iters for r in recs) == pcg
    f = _objective(res, x)
    # fp32: north_star's 1e-3 relative bar; fp64: half a unit of the last
    # digit the reference value is quoted with (765.61, 8744.586)
    tol = 1e-3 * f_ref if dtype == "fp32" else {"c2": 0.005, "c3": 0.0005}[cfg]
    assert abs(f - f_ref) <= tol, (f, f_ref)
    assert abs(res.u.mean()) <= 1e-6 * np.abs(res.u).max()


def test_full_size_row_sharded(scenes):
    """C3 through the row-band decomposition (4 bands, loopback collectives)."""
    x = scenes["c3"]
    f_ref, outer, pcg = REF["c3"]
    res = pu.unwrap_rows(x, dtype="fp32", bands=4)
    recs = res.trace.records
    assert len(recs) == outer and sum(r.cg_iters for r in recs) == pcg
    assert abs(_objective(res, x) - f_ref) <= 1e-3 * f_ref


def test_full_size_kmap_fp32_vs_fp64(scenes):
    """K-map mismatch fraction of the fp32 result against the fp64 one (device metric)."""
    from paper_2401_09961_b200 import metrics
    x = scenes["c2"]
    r64 = pu.unwrap(x, dtype="fp64")
    r32 = pu.unwrap(x, dtype="fp32")
    frac = metrics.kmap_mismatch(r32.u, r64.u, x)
    assert frac <= 1e-3, frac


def test_full_size_fused_start_bit_identical(scenes, monkeypatch):
    """At C2 fp32 the default path fuses the acceptance with the next
    start-up (pu_accept_weights_start); the two-kernel path gives the same
    trace and bit-identical state."""
    from paper_2401_09961_b200 import irls
    x = scenes["c2"]
    fused = pu.unwrap(x, dtype="fp32")
    monkeypatch.setattr(irls, "FUSED_START", "0")
    plain = pu.unwrap(x, dtype="fp32")
    assert [(r.cg_iters, r.h_delta) for r in fused.trace.records] == \
        [(r.cg_iters, r.h_delta) for r in plain.trace.records]
    for f in ("u", "vv", "vh"):
        np.testing.assert_array_equal(getattr(fused, f), getattr(plain, f))
