"""Parity of each C-ABI entry point with the reference (golden fixtures) and
the CPU oracle.  Runs on a B200 only."""

import numpy as np
import pytest

from oracle import phaseirls_port as port
from cases import rel

pytestmark = pytest.mark.gpu

pu = pytest.importorskip("paper_2401_09961_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def sysvec(u, vv, vh):
    return pu.SystemVector(np.asarray(u, float), np.asarray(vv, float), np.asarray(vh, float))


@pytest.mark.parametrize("lo,tag", [(-np.pi, "m"), (0.0, "z")])
def test_wrapped_gradients_bit_exact(golden_kernels, lo, tag):
    g = pu.wrapped_gradients(golden_kernels["grad/x"], lo)
    assert np.array_equal(g.gv, golden_kernels[f"grad/gv_{tag}"])
    assert np.array_equal(g.gh, golden_kernels[f"grad/gh_{tag}"])


def test_wrapped_gradients_random_bit_exact(rng):
    x = rng.uniform(0.0, 2 * np.pi, (257, 301))
    gv, gh = port.grad_wrapped(x)
    g = pu.wrapped_gradients(x)
    assert np.array_equal(g.gv, gv) and np.array_equal(g.gh, gh)


@pytest.mark.parametrize("dtype,tol", [("fp64", 1e-12), ("fp32", 2e-5)])
def test_apply_system(golden_kernels, dtype, tol):
    g = golden_kernels
    x = sysvec(g["sys/u"], g["sys/vv"], g["sys/vh"])
    a = pu.apply_system(x, pu.DiagonalWeights(g["sys/dv"], g["sys/dh"]), 0.03, dtype=dtype)
    for got, key in ((a.u, "au"), (a.vv, "avv"), (a.vh, "avh")):
        want = g[f"sys/{key}"]
        assert np.max(np.abs(got - want)) <= tol * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("n,m", [(1, 1), (1, 7), (9, 1), (33, 17), (130, 257)])
def test_apply_system_random(rng, n, m):
    x = sysvec(rng.standard_normal((n, m)), rng.standard_normal((n - 1, m)), rng.standard_normal((n, m - 1)))
    dv, dh = rng.uniform(0, 1e3, (n - 1, m)), rng.uniform(0, 1e3, (n, m - 1))
    want = port.system_apply(port.Triple(x.u, x.vv, x.vh), dv, dh, 1e-2)
    got = pu.apply_system(x, pu.DiagonalWeights(dv, dh), 1e-2)
    for a, b in ((got.u, want.u), (got.vv, want.vv), (got.vh, want.vh)):
        assert np.max(np.abs(a - b), initial=0.0) <= 1e-12 * max(1.0, np.abs(b).max(initial=0.0))


def test_build_rhs(golden_kernels):
    g = golden_kernels
    b = pu.build_rhs(pu.GradientField(g["rhs/gv"], g["rhs/gh"]), 0.03)
    np.testing.assert_allclose(b.u, g["rhs/bu"], rtol=0, atol=1e-12)
    np.testing.assert_array_equal(b.vv, g["rhs/bv"])
    np.testing.assert_array_equal(b.vh, g["rhs/bh"])


SYL_SHAPES = [(1, 1), (1, 6), (6, 1), (2, 2), (3, 5), (17, 8), (8, 17), (31, 24), (64, 48), (7, 49)]


@pytest.mark.parametrize("shape", SYL_SHAPES)
def test_sylvester_golden(golden_kernels, shape):
    n, m = shape
    r = golden_kernels[f"syl/{n}x{m}/r"]
    want = golden_kernels[f"syl/{n}x{m}/z"]
    got = pu.sylvester_solve(r, 0.37)
    assert np.max(np.abs(got - want)) <= 1e-11 * max(1.0, np.abs(want).max())


@pytest.mark.parametrize("shape", [(512, 512), (256, 1024), (1024, 96), (4096, 16), (16, 4096), (37, 53),
                                   (2048, 2), (1, 4096), (4095, 3), (97, 1000),
                                   # columns through the fused global-memory first / last FFT stage
                                   # (4096 fp32 / fp64, 256 fp32, 512 fp64) with a ragged last panel
                                   (4096, 22), (256, 13), (512, 7), (2048, 10), (1024, 9), (8192, 6)])
def test_sylvester_vs_dct_oracle(rng, shape):
    n, m = shape
    r = rng.standard_normal((n, m))
    want = port.DctPoisson(n, m)(r, 1e-2)
    got = pu.sylvester_solve(r, 1e-2)
    assert rel(got, want) <= 1e-11
    got32 = pu.sylvester_solve(r, 1e-2, dtype="fp32")
    assert rel(got32, want) <= 5e-5


@pytest.mark.parametrize("shape,dtypes", [((4, 16384), ("fp32",)), ((16384, 4), ("fp32",)),
                                          ((3, 8192), ("fp64", "fp32")), ((8192, 3), ("fp64", "fp32")),
                                          ((5, 12000), ("fp32",))])
def test_sylvester_long_rows(rng, shape, dtypes):
    """Rows too long for two staged rows beside the FFT buffer (single-row
    staging) and the one-sequence static column panel (L / EMAX = 1024)."""
    n, m = shape
    r = rng.standard_normal((n, m))
    want = port.DctPoisson(n, m)(r, 1e-2)
    for dt in dtypes:
        got = pu.sylvester_solve(r, 1e-2, dtype=dt)
        assert rel(got, want) <= (1e-11 if dt == "fp64" else 5e-5), dt


@pytest.mark.parametrize("shape,dtypes", [((2, 16384), ("fp64",)), ((7, 16384), ("fp64",)),
                                          ((16384, 4), ("fp64",)), ((16384, 7), ("fp64",)),
                                          ((16384, 16384 // 64), ("fp64",)),
                                          ((3, 32768), ("fp32",)), ((32768, 5), ("fp32",))])
def test_sylvester_cluster_split(rng, shape, dtypes):
    """Lengths whose packed sequence exceeds one CTA's shared memory (fp64
    16384, fp32 32768): a 2-CTA cluster per sequence exchanging halves
    through distributed shared memory (pu_split.cuh).  Odd counts exercise
    the lone last row / column of a pair."""
    n, m = shape
    r = rng.standard_normal((n, m))
    want = port.DctPoisson(n, m)(r, 1e-2)
    for dt in dtypes:
        got = pu.sylvester_solve(r, 1e-2, dtype=dt)
        assert rel(got, want) <= (1e-11 if dt == "fp64" else 5e-5), dt


@pytest.mark.parametrize("shape,dtypes", [((3, 4099), ("fp64",)), ((4099, 4), ("fp64",)), ((4099, 5), ("fp64",)),
                                          ((6001, 3), ("fp64",)), ((2, 8191), ("fp64",)),
                                          ((3, 8209), ("fp32",)), ((8209, 4), ("fp32",)), ((2, 16381), ("fp32",))])
def test_sylvester_cluster_split_bluestein(rng, shape, dtypes):
    """Non-smooth lengths past half the one-CTA limit (fp64 4097..8192,
    fp32 8193..16384): Bluestein on the internal length 2 LH, split over the
    2-CTA cluster (pu_split.cuh split_bluestein)."""
    n, m = shape
    r = rng.standard_normal((n, m))
    want = port.DctPoisson(n, m)(r, 1e-2)
    for dt in dtypes:
        got = pu.sylvester_solve(r, 1e-2, dtype=dt)
        assert rel(got, want) <= (1e-10 if dt == "fp64" else 1e-4), dt


def test_fp64_long_axis_unwrap_matches_oracle():
    """End-to-end fp64 unwrap on a grid with a 16384-long axis (cluster-split
    row transforms) against the oracle with the exact DCT preconditioner."""
    x = pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(pu.SceneSpec("gaussian-bumps", 12, 16384, 30.0, 40.0,
                                                                       5))), 0.5, 55)
    ref_state, ref_recs, _ = port.unwrap(x, poisson="dct")
    res = pu.unwrap(x, dtype="fp64")
    assert [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in ref_recs]
    assert rel(res.u, ref_state.u) <= 1e-8


def test_apply_preconditioner(rng):
    n, m = 40, 33
    r = sysvec(rng.standard_normal((n, m)), rng.standard_normal((n - 1, m)), rng.standard_normal((n, m - 1)))
    dv, dh = rng.uniform(0, 1e6, (n - 1, m)), rng.uniform(0, 1e6, (n, m - 1))
    want = port.precond_apply(port.Triple(r.u, r.vv, r.vh), dv, dh, 1e-2, port.DensePoisson(n, m))
    got = pu.apply_preconditioner(r, pu.DiagonalWeights(dv, dh), 1e-2)
    assert rel(got.u, want.u) <= 1e-11
    np.testing.assert_allclose(got.vv, want.vv, rtol=1e-15)
    np.testing.assert_allclose(got.vh, want.vh, rtol=1e-15)


def test_objective_pieces(golden_kernels):
    g = golden_kernels
    st = sysvec(g["obj/u"], g["obj/vv"], g["obj/vh"])
    grad = pu.GradientField(g["obj/gv"], g["obj/gh"])
    c = pu.WeightField(g["obj/cv"], g["obj/ch"])
    p = pu.ModelParams(tau=0.02, delta=1e-3)
    w = pu.update_weights(st, c, p.delta)
    np.testing.assert_allclose(w.wv, g["obj/wv"], rtol=1e-15)
    np.testing.assert_allclose(w.wh, g["obj/wh"], rtol=1e-15)
    assert pu.eval_h_delta(st, w, grad, c, p) == pytest.approx(float(g["obj/h_w"]), rel=1e-13)
    wp = pu.IrlsWeights(g["obj/wpv"], g["obj/wph"])
    assert pu.eval_h_delta(st, wp, grad, c, p) == pytest.approx(float(g["obj/h_wprev"]), rel=1e-13)
    assert pu.eval_f(st, grad, c, p) == pytest.approx(float(g["obj/f"]), rel=1e-13)
    lip = pu.lipschitz_constant(c, p)
    assert lip == float(g["obj/lip"])
    cand = pu.candidate_step(st, w, grad, c, p, lip)
    np.testing.assert_allclose(cand.u, g["obj/cand_u"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(cand.vv, g["obj/cand_vv"], rtol=0, atol=1e-13)
    np.testing.assert_allclose(cand.vh, g["obj/cand_vh"], rtol=0, atol=1e-13)


@pytest.mark.parametrize("its,tol", [(0, 0.0), (1, 0.0), (5, 0.0), (12, 0.0), (60, 0.0), (500, 1e-9)])
def test_pcg_golden(golden_kernels, its, tol):
    g = golden_kernels
    tau = 1e-2
    b = pu.build_rhs(pu.GradientField(g["pcg/gv"], g["pcg/gh"]), tau)
    x0 = sysvec(g["pcg/x0u"], g["pcg/x0v"], g["pcg/x0h"])
    out = pu.pcg_solve(b, x0, pu.DiagonalWeights(g["pcg/dv"], g["pcg/dh"]), tau, its, tol)
    key = f"pcg/{its}_{tol:g}"
    assert out.iterations == int(g[f"{key}/iters"])
    assert out.converged == bool(g[f"{key}/converged"])
    for a, bb in ((out.x.u, g[f"{key}/xu"]), (out.x.vv, g[f"{key}/xv"]), (out.x.vh, g[f"{key}/xh"])):
        assert rel(a, bb) <= 1e-9
    ref = g[f"{key}/norms"]
    np.testing.assert_allclose(out.residual_norms, ref, rtol=1e-7, atol=1e-11 * ref[0])


@pytest.mark.parametrize("n,m,its", [(64, 64, 30), (100, 77, 120), (256, 256, 60)])
def test_pcg_vs_oracle(rng, n, m, its):
    """Fixed-budget PCG (rel_tol = 0) incl. the every-50 reprojection."""
    tau = 1e-2
    gv, gh = rng.uniform(-np.pi, np.pi, (n - 1, m)), rng.uniform(-np.pi, np.pi, (n, m - 1))
    dv, dh = rng.uniform(0, 1e4, (n - 1, m)), rng.uniform(0, 1e4, (n, m - 1))
    b = port.rhs(gv, gh, tau)
    x0 = port.Triple(rng.standard_normal((n, m)), rng.standard_normal((n - 1, m)), rng.standard_normal((n, m - 1)))
    solver = port.DctPoisson(n, m)
    want = port.pcg(lambda v: port.system_apply(v, dv, dh, tau),
                    lambda r: port.precond_apply(r, dv, dh, tau, solver), b, x0, its, 0.0)
    got = pu.pcg_solve(sysvec(b.u, b.vv, b.vh), sysvec(x0.u, x0.vv, x0.vh), pu.DiagonalWeights(dv, dh), tau, its,
                       0.0)
    assert got.iterations == want["iterations"]
    assert rel(got.x.u, want["x"].u) <= 1e-9
    assert rel(got.x.vv, want["x"].vv) <= 1e-9
    np.testing.assert_allclose(got.residual_norms, want["norms"], rtol=1e-6, atol=1e-9 * want["norms"][0])


def test_pcg_breakdown_index():
    """Non-finite initial residual -> NumericalBreakdown(0) (reference tests/test_pcg.py:119-130)."""
    n = m = 3
    b = pu.SystemVector.zeros(n, m)
    b.u[0, 0] = np.nan
    with pytest.raises(pu.NumericalBreakdown) as err:
        pu.pcg_solve(b, pu.SystemVector.zeros(n, m), pu.DiagonalWeights(np.ones((2, 3)), np.ones((3, 2))),
                     1e-2, 10, 1e-10)
    assert err.value.iteration == 0


def test_pcg_zero_rhs():
    n = m = 4
    out = pu.pcg_solve(pu.SystemVector.zeros(n, m), pu.SystemVector.zeros(n, m),
                       pu.DiagonalWeights(np.ones((3, 4)), np.ones((4, 3))), 1e-2, 50, 1e-10)
    assert out.iterations == 0 and out.converged and len(out.residual_norms) == 1
