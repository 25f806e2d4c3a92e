"""The reference-precision fixtures of the BASELINE configs (tests/golden/
configs, written by make_config_golden.py from the unmodified reference) are
complete and self-consistent, and the config inputs this package generates
are bit-identical to the ones the reference was run on (checked here for the
sizes that generate in seconds; C2-C4 by the GPU parity tests)."""

import hashlib

import numpy as np
import pytest

import parity_configs as pc

META = pc.available()


def test_fixture_set_present():
    for name in ("c1", "c2", "c3", "c5b0", "c5b1", "c5b2", "c5b3"):
        assert name in META, name


@pytest.mark.parametrize("name", sorted(META))
def test_fixture_consistent(name):
    ref = pc.load(name)
    n, m = META[name]["shape"]
    st = int(ref["sub_stride"]) if "sub_stride" in ref.files else 8
    assert ref["u_sub"].shape == ((n + st - 1) // st, (m + st - 1) // st)
    assert ref["u_rows"].shape == (3, m) and ref["u_cols"].shape == (3, n)
    if "kmap" in ref.files:
        assert ref["kmap"].shape == (n, m)
    assert float(ref["F"]) == pytest.approx(META[name]["F"], rel=1e-15)
    assert int(ref["trace_cg_iters"].sum()) == META[name]["pcg"] and ref["trace_k"].size == META[name]["outer"]
    # the subgrid is part of the full-precision u: its norm cannot exceed ||u||
    assert np.linalg.norm(ref["u_sub"]) <= float(ref["u_norm"])


@pytest.mark.parametrize("name", ["c1", "c5b0"])
def test_config_inputs_bit_identical(name):
    from paper_2401_09961_b200.synth import config_scene
    x = config_scene("c5", int(name[3:]))[1] if name.startswith("c5b") else config_scene(name)[1]
    assert hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest() == META[name]["x_sha256"]


def test_host_objective_matches_reference_on_fixture_lines():
    """eval_f_host (the checker's F) reproduces the reference's F definition on
    a small case with known parts."""
    x = np.zeros((3, 4))
    u = np.arange(12.0).reshape(3, 4) * 0.1
    vv = np.full((2, 4), 0.05)
    vh = np.full((3, 3), -0.02)
    rv = np.diff(u, axis=0) - vv
    rh = np.diff(u, axis=1) - vh
    want = np.abs(vv).sum() + np.abs(vh).sum() + (np.sum(rv * rv) + np.sum(rh * rh)) / (2 * 1e-2)
    assert pc.eval_f_host(x, u, vv, vh) == pytest.approx(want, rel=1e-14)
