"""Command line (cli.py, arrayio.py) on the host: argument handling and exit
codes of the reference CLI (cli.py:1-253, tests/test_cli.py) that are decided
before any device work, the host subcommands, and the NPY contract."""

import json

import numpy as np
import pytest

from paper_2401_09961_b200 import cli
from paper_2401_09961_b200.arrayio import ArrayFileError, load_grid, save_grid


def run(*args):
    return cli.main([str(a) for a in args])


@pytest.fixture
def wrapped(tmp_path):
    x = (0.3 * np.arange(12)[:, None] + 0.2 * np.arange(10)[None, :]) % (2 * np.pi)
    p = tmp_path / "x.npy"
    save_grid(p, x)
    return p


def test_npy_roundtrip_and_validation(tmp_path):
    a = np.random.default_rng(0).standard_normal((5, 7))
    save_grid(tmp_path / "a", a)                       # no .npy suffix appended
    np.testing.assert_array_equal(load_grid(tmp_path / "a"), a)
    save_grid(tmp_path / "f.npy", a, dtype="<f4")
    assert load_grid(tmp_path / "f.npy").dtype == np.float64
    np.save(tmp_path / "i.npy", np.ones((3, 3), dtype=np.int32))
    np.save(tmp_path / "c.npy", np.ones((2, 2, 2)))
    np.save(tmp_path / "n.npy", np.array([[1.0, np.nan]]))
    for bad in ("i.npy", "c.npy", "n.npy", "missing.npy"):
        with pytest.raises(ArrayFileError):
            load_grid(tmp_path / bad)
    (tmp_path / "junk.npy").write_bytes(b"not an npy file")
    with pytest.raises(ArrayFileError):
        load_grid(tmp_path / "junk.npy")
    with pytest.raises(ValueError):
        save_grid(tmp_path / "z.npy", a, dtype="<f2")


def test_unwrap_exit_codes_before_device(tmp_path, wrapped, capsys):
    out = tmp_path / "u.npy"
    (tmp_path / "junk.npy").write_bytes(b"garbage")
    assert run("unwrap", "--input", tmp_path / "junk.npy", "--output", out) == cli.EXIT_BAD_INPUT
    assert run("unwrap", "--input", tmp_path / "nope.npy", "--output", out) == cli.EXIT_BAD_INPUT
    save_grid(tmp_path / "cv.npy", np.ones((11, 10)))
    assert run("unwrap", "--input", wrapped, "--output", out, "--cv", tmp_path / "cv.npy") == cli.EXIT_BAD_INPUT
    save_grid(tmp_path / "ch_bad.npy", np.ones((12, 10)))
    assert run("unwrap", "--input", wrapped, "--output", out, "--cv", tmp_path / "cv.npy", "--ch",
               tmp_path / "ch_bad.npy") == cli.EXIT_DIM_MISMATCH
    save_grid(tmp_path / "ch.npy", -np.ones((12, 9)))
    assert run("unwrap", "--input", wrapped, "--output", out, "--cv", tmp_path / "cv.npy", "--ch",
               tmp_path / "ch.npy") == cli.EXIT_BAD_INPUT            # negative weights
    assert run("unwrap", "--input", wrapped, "--output", out, "--tau", "-1") == cli.EXIT_BAD_INPUT
    assert run("unwrap", "--input", wrapped, "--output", out, "--cg-growth", "0.5") == cli.EXIT_BAD_INPUT
    err = capsys.readouterr().err
    assert err.count("error:") == 7


def test_unwrap_without_gpu_fails_loudly(wrapped, tmp_path, capsys):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    assert run("unwrap", "--input", wrapped, "--output", tmp_path / "u.npy") == cli.EXIT_NO_DEVICE
    assert "CUDA" in capsys.readouterr().err
    assert not (tmp_path / "u.npy").exists()


def test_synth_and_error(tmp_path, capsys):
    truth, wr = tmp_path / "t.npy", tmp_path / "w.npy"
    assert run("synth", "--kind", "gaussian-bumps", "--rows", 16, "--cols", 12, "--amplitude", 5, "--scale", 3,
               "--seed", 2, "--wrap", "--noise-sigma", 0.1, "--out-truth", truth, "--out-wrapped", wr) == 0
    t, w = load_grid(truth), load_grid(wr)
    assert t.shape == w.shape == (16, 12) and w.min() >= 0 and w.max() < 2 * np.pi
    assert run("synth", "--kind", "ramp", "--rows", 4, "--cols", 4) == cli.EXIT_BAD_INPUT
    assert run("synth", "--kind", "ramp", "--rows", 4, "--cols", 4, "--out-wrapped", wr) == cli.EXIT_BAD_INPUT
    shifted = tmp_path / "s.npy"
    save_grid(shifted, t + 4 * np.pi)
    assert run("error", "--estimate", shifted, "--truth", truth, "--json-out", tmp_path / "e.json") == 0
    rep = json.loads((tmp_path / "e.json").read_text())
    assert abs(abs(rep["alpha"]) - 4 * np.pi) < 1e-9 and rep["rmse"] < 1e-9 and rep["congruent_fraction"] == 1.0
    save_grid(tmp_path / "small.npy", t[:4])
    assert run("error", "--estimate", tmp_path / "small.npy", "--truth", truth) == cli.EXIT_DIM_MISMATCH
