"""The command line on the GPU: same outputs and trace lines as the Python API
and the reference's golden traces, byte-identical reruns (reference
tests/test_cli.py:104-111), --congruent and --gradient-interval."""

import json

import numpy as np
import pytest

from cases import case_inputs, golden_trace
from paper_2401_09961_b200 import cli
from paper_2401_09961_b200.gridfile import read_grid as load_grid, write_grid as save_grid

pytestmark = pytest.mark.gpu
pu = pytest.importorskip("paper_2401_09961_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def run(*args):
    return cli.main([str(a) for a in args])


def test_cli_matches_golden_trace(tmp_path, golden_unwrap, golden_meta):
    x, cv, ch, tau, delta, prm, lo = case_inputs(golden_unwrap, golden_meta, "noisy64")
    save_grid(tmp_path / "x.npy", x)
    out, tr = tmp_path / "u.npy", tmp_path / "t.jsonl"
    assert run("unwrap", "--input", tmp_path / "x.npy", "--output", out, "--trace", tr) == 0
    recs = [json.loads(line) for line in tr.read_text().splitlines()]
    assert list(recs[0]) == ["k", "m_cg", "delta_rel", "h_delta", "cg_iters", "fallback"]
    want = golden_trace(golden_unwrap, "noisy64")
    assert [r["cg_iters"] for r in recs] == want["cg_iters"].tolist()
    assert [r["m_cg"] for r in recs] == want["m_cg"].tolist()
    np.testing.assert_allclose([r["h_delta"] for r in recs], want["h_delta"], rtol=1e-8)
    u = load_grid(out)
    u_ref = golden_unwrap["noisy64/u"]
    assert np.linalg.norm(u - u_ref) <= 1e-8 * np.linalg.norm(u_ref)


@pytest.mark.parametrize("dtype", ["fp64", "fp32"])
def test_deterministic_reruns(tmp_path, dtype):
    x = pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(pu.SceneSpec("gaussian-bumps", 48, 40, 9.0, 6.0, 4))),
                           0.6, 7)
    save_grid(tmp_path / "x.npy", x)
    outs = [tmp_path / f"u{i}.npy" for i in (0, 1)]
    traces = [tmp_path / f"t{i}.jsonl" for i in (0, 1)]
    for o, t in zip(outs, traces):
        assert run("unwrap", "--input", tmp_path / "x.npy", "--output", o, "--trace", t, "--dtype", dtype) == 0
    assert outs[0].read_bytes() == outs[1].read_bytes()
    assert traces[0].read_bytes() == traces[1].read_bytes()


def test_congruent_and_interval(tmp_path):
    truth = -0.3 * np.arange(24)[:, None] + np.zeros((24, 20))
    save_grid(tmp_path / "w.npy", pu.wrap_to_principal(truth, 0.0))
    assert run("unwrap", "--input", tmp_path / "w.npy", "--output", tmp_path / "c.npy", "--congruent") == 0
    x, u = load_grid(tmp_path / "w.npy"), load_grid(tmp_path / "c.npy")
    cyc = (u - x) / (2 * np.pi)
    assert np.max(np.abs(cyc - np.rint(cyc))) < 1e-9
    assert run("unwrap", "--input", tmp_path / "w.npy", "--output", tmp_path / "s.npy") == 0
    assert run("unwrap", "--input", tmp_path / "w.npy", "--output", tmp_path / "p.npy",
               "--gradient-interval", "positive") == 0
    assert not np.array_equal(load_grid(tmp_path / "s.npy"), load_grid(tmp_path / "p.npy"))
    rep = pu.shift_error(load_grid(tmp_path / "s.npy"), truth)
    assert rep.max_abs < 1e-6


def test_cli_row_sharded_single_process(tmp_path):
    """--shard rows outside torchrun: one band through the band driver."""
    x = pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(pu.SceneSpec("gaussian-bumps", 40, 32, 8.0, 5.0, 2))),
                           0.5, 3)
    save_grid(tmp_path / "x.npy", x)
    assert run("unwrap", "--input", tmp_path / "x.npy", "--output", tmp_path / "a.npy") == 0
    assert run("unwrap", "--input", tmp_path / "x.npy", "--output", tmp_path / "b.npy", "--shard", "rows") == 0
    np.testing.assert_array_equal(load_grid(tmp_path / "a.npy"), load_grid(tmp_path / "b.npy"))
