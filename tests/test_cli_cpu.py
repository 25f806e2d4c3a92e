"""Command line (cli.py, gridfile.py) on the host: argument handling and exit
codes of the reference CLI (cli.py:1-253, tests/test_cli.py) that are decided
before any device work, the host subcommands, and the NPY contract."""

import json

import numpy as np
import pytest

from paper_2401_09961_b200 import cli
from paper_2401_09961_b200.gridfile import GridFileError, read_grid as load_grid, write_grid as save_grid


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
        with pytest.raises(GridFileError):
            load_grid(tmp_path / bad)
    (tmp_path / "junk.npy").write_bytes(b"not an npy file")
    with pytest.raises(GridFileError):
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


def test_host_utilities_not_exposed():
    """synth / error / spectrum are host utilities outside the GPU path."""
    for sub in ("synth", "error", "spectrum"):
        with pytest.raises(SystemExit):
            run(sub)


def test_fortran_order_and_atomic_write(tmp_path):
    a = np.asfortranarray(np.arange(12.0).reshape(3, 4))
    np.save(tmp_path / "f.npy", a)
    np.testing.assert_array_equal(load_grid(tmp_path / "f.npy"), a)
    np.save(tmp_path / "o.npy", np.array([[object()]], dtype=object), allow_pickle=True)
    with pytest.raises(GridFileError):
        load_grid(tmp_path / "o.npy")
    (tmp_path / "t.npy").write_bytes(open(tmp_path / "f.npy", "rb").read()[:-8])  # truncated payload
    with pytest.raises(GridFileError):
        load_grid(tmp_path / "t.npy")
    with pytest.raises(ValueError):
        save_grid(tmp_path / "bad.npy", np.ones(3))
    assert not (tmp_path / "bad.npy").exists()
    assert [p.name for p in tmp_path.iterdir() if p.name.startswith(".grid-")] == []
