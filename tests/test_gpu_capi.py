"""The whole unwrap through the C ABI entry point pu_unwrap (csrc/pu_host.cu):
the ctypes binding (capi.unwrap_capi) and a plain C program
(examples/unwrap_demo.c, built with gcc) give exactly what the Python host
gives, on the reference's golden cases and concurrently from several threads."""

import os
import subprocess
import threading

import numpy as np
import pytest

from cases import GOLDEN_UNWRAP_CASES, case_inputs, golden_trace, rel

pytestmark = pytest.mark.gpu
pu = pytest.importorskip("paper_2401_09961_b200")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _same(a, b):
    assert [(r.k, r.m_cg, r.cg_iters, r.sufficient_decrease, r.fallback_used) for r in a.trace.records] == \
        [(r.k, r.m_cg, r.cg_iters, r.sufficient_decrease, r.fallback_used) for r in b.trace.records]
    assert [r.delta_rel for r in a.trace.records] == [r.delta_rel for r in b.trace.records]
    assert [r.h_delta for r in a.trace.records] == [r.h_delta for r in b.trace.records]
    for f in ("u", "vv", "vh"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))


@pytest.mark.parametrize("name", GOLDEN_UNWRAP_CASES)
def test_capi_matches_python_host_and_reference(golden_unwrap, golden_meta, name):
    from paper_2401_09961_b200.capi import unwrap_capi
    x, cv, ch, tau, delta, prm, lo = case_inputs(golden_unwrap, golden_meta, name)
    c = None if cv is None else pu.WeightField(cv, ch)
    model, params = pu.ModelParams(tau, delta), pu.IrlsParams(**prm.__dict__)
    got = unwrap_capi(x, c, model, params, lo)
    _same(got, pu.unwrap(x, c, model, params, lo))
    want = golden_trace(golden_unwrap, name)
    assert [r.cg_iters for r in got.trace.records] == want["cg_iters"].tolist()
    u_ref = golden_unwrap[f"{name}/u"]
    assert rel(got.u, u_ref) <= 1e-8 or np.max(np.abs(got.u - u_ref)) <= 1e-12


@pytest.mark.parametrize("dtype", ["fp32", "fp64"])
def test_capi_concurrent_calls(dtype):
    from paper_2401_09961_b200.capi import unwrap_capi
    xs = [pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(pu.SceneSpec("gaussian-bumps", 72, 64, 9.0, 7.0, s))),
                             0.5, 10 + s) for s in range(4)]
    seq = [unwrap_capi(x, dtype=dtype) for x in xs]
    out = [None] * len(xs)

    def work(i):
        out[i] = unwrap_capi(xs[i], dtype=dtype)

    ts = [threading.Thread(target=work, args=(i,)) for i in range(len(xs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for a, b in zip(seq, out):
        _same(a, b)
    for a, x in zip(seq, xs):
        _same(a, pu.unwrap(x, dtype=dtype))


def test_c_program(tmp_path):
    """examples/unwrap_demo.c: a C caller with no Python in the loop."""
    exe = tmp_path / "unwrap_demo"
    lib = os.path.join(ROOT, "paper_2401_09961_b200", "_lib")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "unwrap_demo.c"),
                    "-L", lib, f"-Wl,-rpath,{lib}", "-lpu_unwrap", "-lm", "-o", str(exe)], check=True)
    x = pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(pu.SceneSpec("gaussian-bumps", 80, 96, 11.0, 8.0, 3))),
                           0.6, 33)
    x.astype("<f8").tofile(tmp_path / "x.f64")
    proc = subprocess.run([str(exe), str(tmp_path / "x.f64"), "80", "96", str(tmp_path / "u.f64")],
                          capture_output=True, text=True, timeout=300)
    assert proc.returncode == 0, proc.stderr
    u = np.fromfile(tmp_path / "u.f64", dtype="<f8").reshape(80, 96)
    want = pu.unwrap(x)
    np.testing.assert_array_equal(u, want.u)
    assert len(proc.stdout.splitlines()) == len(want.trace)
    bad = np.full((4, 4), 9.0)
    bad.astype("<f8").tofile(tmp_path / "bad.f64")
    proc = subprocess.run([str(exe), str(tmp_path / "bad.f64"), "4", "4", str(tmp_path / "o.f64")],
                          capture_output=True, text=True, timeout=60)
    assert proc.returncode == 2 and "[0, 2*pi)" in proc.stderr
