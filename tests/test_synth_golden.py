"""The host-side input generator reproduces the reference's scenes bit for bit."""

import hashlib

import numpy as np
import pytest

from paper_2401_09961_b200.synth import (SceneSpec, add_phase_noise, config_scene, generate_scene,
                                         wrap_scene)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()


def test_small_scenes(golden_meta):
    want = golden_meta["configs"]["small_scene_sha256"]
    for kind in ("ramp", "gaussian-bumps", "plateau-discontinuity"):
        for (rows, cols, seed) in ((1, 1, 0), (1, 9, 3), (17, 1, 4), (33, 21, 5)):
            s = generate_scene(SceneSpec(kind, rows, cols, 7.5, 3.0, seed))
            assert sha(s) == want[f"{kind}/{rows}x{cols}/{seed}"]
            noisy = add_phase_noise(wrap_scene(s), 0.7, seed + 9)
            assert sha(noisy) == want[f"{kind}/{rows}x{cols}/{seed}/noisy"]


@pytest.mark.parametrize("name,key", [("c1", "c1_x"), ("c5", "c5b0_x")])
def test_config_inputs(golden_meta, name, key):
    _, x = config_scene(name, 0)
    assert sha(x) == golden_meta["configs"]["sha256"][key]


@pytest.mark.slow
def test_config_c3_input(golden_meta):
    t, x = config_scene("c3")
    assert sha(t) == golden_meta["configs"]["sha256"]["c3_truth"]
    assert sha(x) == golden_meta["configs"]["sha256"]["c3_x"]


def test_spec_validation():
    with pytest.raises(ValueError):
        SceneSpec("nope", 2, 2, 1.0, 1.0, 0)
    with pytest.raises(ValueError):
        SceneSpec("ramp", 0, 2, 1.0, 1.0, 0)
