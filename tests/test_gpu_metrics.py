"""Device parity metrics (metrics.py) against the host restatements of the
reference's shift_error / congruent_round (phase.py:152-184)."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
pu = pytest.importorskip("paper_2401_09961_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


@pytest.mark.parametrize("shape", [(33, 47), (128, 96), (1, 5)])
def test_shift_error_and_congruent(rng, shape):
    from paper_2401_09961_b200 import metrics
    truth = rng.standard_normal(shape) * 5
    est = truth + 3.0 + np.where(rng.random(shape) < 0.1, 2 * np.pi, 0.0) + 1e-5 * rng.standard_normal(shape)
    want = pu.shift_error(est, truth)
    got = metrics.shift_error(est, truth)
    assert abs(got.alpha - want.alpha) <= 1e-12 * max(1.0, abs(want.alpha))
    assert abs(got.max_abs - want.max_abs) <= 1e-12 * max(1.0, want.max_abs)
    assert abs(got.rmse - want.rmse) <= 1e-12 * max(1.0, want.rmse)
    assert got.congruent_fraction == want.congruent_fraction
    x = pu.wrap_to_principal(truth, 0.0)
    np.testing.assert_array_equal(metrics.congruent_round(est, x), pu.congruent_round(est, x))


def test_kmap_mismatch(rng):
    from paper_2401_09961_b200 import metrics
    x = rng.uniform(0, 2 * np.pi, (40, 30))
    u_ref = x + 2 * np.pi * rng.integers(-3, 4, x.shape)
    u = u_ref.copy()
    flip = rng.random(x.shape) < 0.07
    u[flip] += 2 * np.pi
    got = metrics.kmap_mismatch(u, u_ref, x)
    assert got == pytest.approx(flip.mean(), abs=0)
    assert metrics.kmap_mismatch(u_ref, u_ref, x) == 0.0


def test_metrics_on_resident_unwrap():
    """u plane of an unwrap still on the device, fp32 handle."""
    from paper_2401_09961_b200 import metrics
    from paper_2401_09961_b200.irls import unwrap_device
    import torch
    spec = pu.SceneSpec("gaussian-bumps", 64, 48, 10.0, 6.0, 1)
    truth = pu.generate_scene(spec)
    x = pu.wrap_scene(truth)
    run, trace = unwrap_device(torch.from_numpy(x).cuda(), None, pu.ModelParams(), pu.IrlsParams(), -np.pi, "fp32")
    rep = metrics.shift_error(np.empty(x.shape), truth, ws=run.ws, u_plane=run.state[0])
    host = pu.shift_error(run.ws.from_system(run.state)[0].cpu().numpy(), truth)
    assert rep.congruent_fraction == host.congruent_fraction == 1.0
    assert abs(rep.rmse - host.rmse) <= 1e-9
