"""Row-sharded unwrap (band.py) on one GPU through the loopback communicator:
the band decomposition (ghost rows, cross-band reductions + finalisers, the
packed DCT transpose) must reproduce the single-grid solve and the reference.
The multi-process collective plumbing is covered by test_band_comm_gloo.py."""

import numpy as np
import pytest

from oracle import phaseirls_port as port
from cases import GOLDEN_UNWRAP_CASES, case_inputs, golden_trace, rel

pytestmark = pytest.mark.gpu

pu = pytest.importorskip("paper_2401_09961_b200")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _scene(n, m, noise=0.7, seed=5):
    spec = pu.SceneSpec("gaussian-bumps", n, m, 12.0, 6.0, seed)
    return pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(spec)), noise, 100 + seed)


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("shape,bands", [((64, 48), 2), ((50, 45), 3), ((37, 64), 4), ((96, 80), 5),
                                         ((40, 33), 1)])
def test_bands_match_single_grid_fp64(shape, bands, peer):
    """Packed all-to-all transposes (peer=False) and the transpose fused into
    the row kernels through the column-block address table (peer=True)."""
    x = _scene(*shape)
    single = pu.unwrap(x, dtype="fp64")
    res = pu.unwrap_rows(x, dtype="fp64", bands=bands, peer=peer)
    assert [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in single.trace.records]
    assert [r.m_cg for r in res.trace.records] == [r.m_cg for r in single.trace.records]
    np.testing.assert_allclose([r.h_delta for r in res.trace.records], [r.h_delta for r in single.trace.records],
                               rtol=1e-9)
    assert res.u.shape == single.u.shape and res.vv.shape == single.vv.shape and res.vh.shape == single.vh.shape
    assert rel(res.u, single.u) <= 1e-9
    assert rel(res.vv, single.vv) <= 1e-8


@pytest.mark.parametrize("peer", [False, True])
def test_bands_eager_match_single_grid(monkeypatch, peer):
    """The eager launch path (no CUDA graphs: how torch.distributed bands run
    with the all-to-all transposes), with the speculative start-up and the
    host's exit polls every 16 PCG iterations, on loopback bands."""
    from paper_2401_09961_b200 import band
    monkeypatch.setenv("PU_BAND_GRAPHS", "0")
    monkeypatch.setattr(band.RowSharded, "_cache", {})
    x = _scene(96, 80)
    single = pu.unwrap(x, dtype="fp64")
    res = pu.unwrap_rows(x, dtype="fp64", bands=3, peer=peer)
    assert [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in single.trace.records]
    assert [r.sufficient_decrease for r in res.trace.records] == [r.sufficient_decrease
                                                                  for r in single.trace.records]
    assert rel(res.u, single.u) <= 1e-9


@pytest.mark.parametrize("graphs", ["0", "1"])
def test_bands_long_budget_exits(monkeypatch, graphs):
    """Budgets longer than a poll chunk (16 eager / 64 captured PCG
    iterations) that converge before they end: the lagged exit polls stop
    enqueueing after the device-side exit, with the single grid's trace."""
    from paper_2401_09961_b200 import band
    monkeypatch.setenv("PU_BAND_GRAPHS", graphs)
    monkeypatch.setattr(band.RowSharded, "_cache", {})
    x = _scene(96, 80)
    prm = pu.IrlsParams(max_iter_cg_start=150, max_cg_iters_cap=300)
    single = pu.unwrap(x, params=prm, dtype="fp64")
    res = pu.unwrap_rows(x, params=prm, dtype="fp64", bands=2, peer=True)
    iters = [r.cg_iters for r in res.trace.records]
    assert iters == [r.cg_iters for r in single.trace.records]
    assert any(16 < i < r.m_cg for i, r in zip(iters, res.trace.records))  # an exit inside a later chunk
    assert rel(res.u, single.u) <= 1e-9


@pytest.mark.parametrize("graphs", ["1", "0"])
@pytest.mark.parametrize("bands,peer", [(1, True), (3, False), (4, True)])
def test_bands_fused_start_match_single_grid(monkeypatch, bands, peer, graphs):
    """The acceptance fused with the next start-up on bands
    (pu_accept_weights_start on ghost rows, sums through the band totals;
    automatic from 2048² cells per band, forced here): same trace and result
    as the single grid, with and without captured graphs."""
    from paper_2401_09961_b200 import band, irls
    monkeypatch.setattr(irls, "FUSED_START", "1")
    monkeypatch.setenv("PU_BAND_GRAPHS", graphs)
    monkeypatch.setattr(band.RowSharded, "_cache", {})
    x = _scene(96, 80)
    c = pu.WeightField(np.full((95, 80), 0.8), np.full((96, 79), 1.1))
    single = pu.unwrap(x, c, dtype="fp64")
    res = pu.unwrap_rows(x, c, dtype="fp64", bands=bands, peer=peer)
    solver = band.RowSharded.get(96, 80, "fp64", pu.ModelParams(), res_device(), bands, None, peer)
    assert solver.driver.fuse
    assert [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in single.trace.records]
    np.testing.assert_allclose([r.h_delta for r in res.trace.records], [r.h_delta for r in single.trace.records],
                               rtol=1e-9)
    assert rel(res.u, single.u) <= 1e-9
    assert rel(res.vh, single.vh) <= 1e-8


def res_device():
    import torch
    return torch.device("cuda", torch.cuda.current_device())


@pytest.mark.parametrize("name", ["noisy64", "noisy96x80", "weighted40x36", "lo0_noisy48"])
def test_bands_match_reference(golden_unwrap, golden_meta, name):
    """north_star fp64 bar on the sharded path: u within 1e-8 of the reference's."""
    if name not in GOLDEN_UNWRAP_CASES:
        pytest.skip(f"{name} not in the golden set")
    x, cv, ch, tau, delta, prm, lo = case_inputs(golden_unwrap, golden_meta, name)
    c = None if cv is None else pu.WeightField(cv, ch)
    res = pu.unwrap_rows(x, c, pu.ModelParams(tau, delta), pu.IrlsParams(**prm.__dict__), lo, dtype="fp64",
                         bands=3)
    want = golden_trace(golden_unwrap, name)
    assert [r.cg_iters for r in res.trace.records] == want["cg_iters"].tolist()
    u_ref = golden_unwrap[f"{name}/u"]
    assert rel(res.u, u_ref) <= 1e-8 or np.max(np.abs(res.u - u_ref)) <= 1e-12


@pytest.mark.parametrize("peer", [False, True])
def test_bands_fp32_objective(peer):
    x = _scene(128, 96, noise=0.9, seed=7)
    ref_state, _, (gv, gh) = port.unwrap(x, poisson="dct")
    res = pu.unwrap_rows(x, dtype="fp32", bands=4, peer=peer)
    ones = (np.ones_like(gv), np.ones_like(gh))
    f_ref = port.f_l1(ref_state, gv, gh, *ones, 1e-2)
    f32 = port.f_l1(port.Triple(res.u, res.vv, res.vh), gv, gh, *ones, 1e-2)
    assert abs(f32 - f_ref) <= max(1e-3 * f_ref, 1e-6)


def test_band_pcg_long_budget_reprojection():
    """Budgets past 50 iterations exercise the all-reduced mean re-projection."""
    x = _scene(72, 64, noise=1.0, seed=9)
    prm = pu.IrlsParams(max_iter_cg_start=60, cg_rel_tol=1e-14, max_outer_iters=3)
    single = pu.unwrap(x, params=prm, dtype="fp64")
    res = pu.unwrap_rows(x, params=prm, dtype="fp64", bands=3, peer=True)
    assert [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in single.trace.records]
    assert max(r.cg_iters for r in res.trace.records) > 50
    assert rel(res.u, single.u) <= 1e-9


def test_band_layout_errors():
    with pytest.raises(ValueError):
        pu.band.BandLayout(3, 8, 4)
    with pytest.raises(ValueError):
        pu.band.BandLayout(64, 8, 4)  # 8 columns cannot give 4 blocks of >= 8


@pytest.mark.parametrize("peer", [False, True])
def test_bands_cluster_split_rows_fp64(peer):
    """fp64 rows of 16384 (cluster-split row transforms, packed / pushed
    spectrum) in 2 bands against the single-grid solve."""
    x = _scene(10, 16384, noise=0.6, seed=11)
    single = pu.unwrap(x, dtype="fp64", params=pu.IrlsParams(max_outer_iters=6))
    res = pu.unwrap_rows(x, dtype="fp64", bands=2, peer=peer, params=pu.IrlsParams(max_outer_iters=6))
    assert [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in single.trace.records]
    assert rel(res.u, single.u) <= 1e-9


def test_band_graph_chunks_past_64_iterations():
    """Loopback bands replay captured graphs of 64 PCG iterations per chunk;
    a 100-iteration budget crosses a chunk boundary (and the every-50
    re-projection) with an exit poll between the chunks."""
    x = _scene(64, 72, noise=1.0, seed=13)
    prm = pu.IrlsParams(max_iter_cg_start=100, max_cg_iters_cap=200, cg_rel_tol=1e-14, max_outer_iters=3)
    single = pu.unwrap(x, params=prm, dtype="fp64")
    res = pu.unwrap_rows(x, params=prm, dtype="fp64", bands=2)
    assert [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in single.trace.records]
    assert max(r.cg_iters for r in res.trace.records) > 64
    assert rel(res.u, single.u) <= 1e-9
