"""GPU synthetic scenes (synth_gpu.py, csrc/pu_synth.cu; reference
synth.py:43-109) against the host generator that is
pinned to the reference: parameters from the same Philox draws, plateau /
fault / wrapping exact, bumps to round-off, device noise with the right
distribution."""

import time

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
pu = pytest.importorskip("paper_2401_09961_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("spec", [("gaussian-bumps", 64, 80, 12.0, 9.0, 3), ("gaussian-bumps", 1, 17, 5.0, 2.0, 8),
                                  ("gaussian-bumps", 33, 1, 5.0, 2.0, 9), ("gaussian-bumps", 512, 512, 40.0, 32.0, 1)])
def test_bumps_match_host(spec):
    from paper_2401_09961_b200.synth_gpu import generate_scene_gpu
    s = pu.SceneSpec(*spec)
    want = pu.generate_scene(s)
    got = generate_scene_gpu(s).cpu().numpy()
    assert np.max(np.abs(got - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))


@pytest.mark.parametrize("kind", ["plateau-discontinuity", "ramp"])
def test_exact_kinds(kind):
    from paper_2401_09961_b200.synth_gpu import generate_scene_gpu, wrap_noise_gpu
    s = pu.SceneSpec(kind, 97, 130, 7.5, 3.0, 5)
    t = pu.generate_scene(s)
    g = generate_scene_gpu(s)
    np.testing.assert_array_equal(g.cpu().numpy(), t)
    np.testing.assert_array_equal(wrap_noise_gpu(g, 0.0, 0).cpu().numpy(), pu.wrap_scene(t))


def test_tapered_fault_c3_truth():
    from paper_2401_09961_b200.synth_gpu import config_scene_gpu
    t_cpu, _ = pu.config_scene("c3")
    t_gpu, x_gpu = config_scene_gpu("c3")
    assert np.max(np.abs(t_gpu.cpu().numpy() - t_cpu)) <= 1e-12 * np.max(np.abs(t_cpu))
    x = x_gpu.cpu().numpy()
    assert x.min() >= 0.0 and x.max() < 2 * np.pi


def test_noise_distribution():
    """wrap(0 + sigma N(0,1)): unwrapped back it has mean 0 and std sigma."""
    import torch
    from paper_2401_09961_b200.synth_gpu import wrap_noise_gpu
    z = torch.zeros((1024, 1000), dtype=torch.float64, device="cuda")
    x = wrap_noise_gpu(z, 0.5, 1234).cpu().numpy().ravel()
    v = np.where(x > np.pi, x - 2 * np.pi, x)
    assert abs(v.mean()) < 5 * 0.5 / np.sqrt(v.size)
    assert abs(v.std() - 0.5) < 0.005
    assert abs(((v / 0.5) ** 4).mean() - 3.0) < 0.05      # Gaussian kurtosis
    y = wrap_noise_gpu(z, 0.5, 1235).cpu().numpy().ravel()
    assert not np.array_equal(x, y)                       # the seed selects the stream
    np.testing.assert_array_equal(x, wrap_noise_gpu(z, 0.5, 1234).cpu().numpy().ravel())  # deterministic


def test_gpu_scene_unwraps():
    from paper_2401_09961_b200.synth_gpu import config_scene_gpu
    _, x = config_scene_gpu("c1")
    t0 = time.perf_counter()
    res = pu.unwrap(x, dtype="fp64")
    assert time.perf_counter() - t0 < 60
    assert np.isfinite(res.u).all() and abs(res.u.mean()) < 1e-9 * np.abs(res.u).max()
