"""CPU-side checks of the drop-in boundary: the C-ABI library loads and
exports every entry point include/pu_unwrap.h declares; host-side logic
(parameter validation, budget rule) matches the reference."""

import os
import re

import numpy as np
import pytest

from paper_2401_09961_b200 import _native
from paper_2401_09961_b200.params import (IrlsParams, ModelParams, cg_budget_update, lipschitz_constant,
                                          relative_improvement)
from paper_2401_09961_b200.phase import WeightField

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "pu_unwrap.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|void|const char\*)\s+(pu_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert header_symbols() == _native.exported_symbols()


def test_library_exports_every_symbol():
    if not os.path.exists(_native.LIB_PATH):
        from paper_2401_09961_b200 import build_ext
        build_ext.build()
    lib = _native.load()
    for name in header_symbols():
        assert hasattr(lib, name), name
    assert lib.pu_abi_version() == 1
    assert lib.pu_pcg_ctrl_bytes() == 9 * 8 + 8 * 4


def test_create_fails_cleanly_without_gpu():
    """No GPU in this container: planning must fail with a CUDA error code, not crash."""
    import ctypes
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    lib = _native.load()
    h = ctypes.c_void_p()
    rc = lib.pu_create(ctypes.byref(h), 8, 8, 0, 1e-2, 1e-6)
    assert rc == _native.PU_ERR_CUDA
    assert lib.pu_last_error()
    # argument validation happens before any CUDA call (reference raises ValueError)
    assert lib.pu_create(ctypes.byref(h), 0, 8, 0, 1e-2, 1e-6) == _native.PU_ERR_ARG
    assert lib.pu_create(ctypes.byref(h), 8, 8, 0, -1.0, 1e-6) == _native.PU_ERR_ARG


def test_product_path_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2401_09961_b200 import unwrap
    with pytest.raises(RuntimeError, match="CUDA"):
        unwrap(np.zeros((4, 4)))


class TestBudgetRules:
    # reference tests/test_irls.py:30-58
    D = IrlsParams()

    def test_keep(self):
        d = cg_budget_update(1e-2, 5, 5, self.D)
        assert (d.action, d.m_cg) == ("keep", 5)

    def test_stop_after_grow(self):
        assert cg_budget_update(1e-4, 9, 5, self.D).action == "stop"

    def test_grow(self):
        d = cg_budget_update(1e-4, 5, 5, self.D)
        assert (d.action, d.m_cg) == ("grow", 9)

    def test_grow_clamps(self):
        d = cg_budget_update(1e-4, 8, 8, IrlsParams(max_cg_iters_cap=12))
        assert (d.action, d.m_cg) == ("grow", 12)

    def test_stop_at_cap(self):
        assert cg_budget_update(1e-4, 8, 8, IrlsParams(max_cg_iters_cap=8, max_iter_cg_start=8)).action == "stop"

    def test_rejects(self):
        with pytest.raises(ValueError):
            cg_budget_update(1e-4, 0, 0, self.D)

    def test_relative_improvement(self):
        assert relative_improvement(2.0, 1.0) == 0.5
        with pytest.raises(ValueError):
            relative_improvement(0.0, 1.0)


def test_param_validation():
    for bad in (dict(max_iter_cg_start=0), dict(rel_improvement_tol=0), dict(cg_growth_factor=1.0),
                dict(max_outer_iters=0), dict(max_cg_iters_cap=2), dict(cg_rel_tol=-1)):
        with pytest.raises(ValueError):
            IrlsParams(**bad)
    with pytest.raises(ValueError):
        ModelParams(tau=0)
    with pytest.raises(ValueError):
        ModelParams(delta=float("inf"))


def test_lipschitz():
    assert lipschitz_constant(WeightField.uniform(3, 3), ModelParams()) == 1_001_200.0


def test_weightfield_validation():
    with pytest.raises(ValueError):
        WeightField(np.ones((2, 3)), np.ones((3, 3)))
    with pytest.raises(ValueError):
        WeightField(-np.ones((2, 3)), np.ones((3, 2)))
    with pytest.raises(ValueError):
        WeightField(np.zeros((2, 3)), np.zeros((3, 2)))


def test_band_create_validates_before_cuda():
    """pu_create_band rejects malformed bands with PU_ERR_ARG (no device needed)."""
    import ctypes
    lib = _native.load()
    h = ctypes.c_void_p()

    def band(**kw):
        base = dict(n_glob=64, row0=0, rows=32, nq=2, mb=32, col0=0, cols=32)
        base.update(kw)
        return _native.PuBand(**base)

    bad = [band(rows=0), band(row0=40), band(mb=12), band(nq=1, mb=32), band(col0=8), band(cols=40),
           band(n_glob=1, rows=1)]
    for b in bad:
        assert lib.pu_create_band(ctypes.byref(h), 64, ctypes.byref(b), 0, 1e-2, 1e-6) == _native.PU_ERR_ARG
    assert lib.pu_create_band(ctypes.byref(h), 64, ctypes.byref(band()), 0, -1.0, 1e-6) == _native.PU_ERR_ARG
    assert lib.pu_create_band(ctypes.byref(h), 64, ctypes.byref(band()), 7, 1e-2, 1e-6) == _native.PU_ERR_ARG
    assert lib.pu_create_band(ctypes.byref(h), 64, None, 0, 1e-2, 1e-6) == _native.PU_ERR_ARG


def test_band_layout_partitions():
    from paper_2401_09961_b200.band import BandLayout
    for n, m, w in [(50, 45, 3), (16384, 16384, 8), (9, 100, 4), (4096, 4096, 5)]:
        lay = BandLayout(n, m, w)
        assert sum(lay.rows) == n and lay.row0[0] == 0
        assert all(lay.row0[i] + lay.rows[i] == lay.row0[i + 1] for i in range(w - 1))
        assert max(lay.rows) - min(lay.rows) <= 1
        assert lay.mb % 8 == 0 and lay.mb * w >= m and sum(lay.cols) == m


def _capi_args():
    from paper_2401_09961_b200 import capi  # noqa: F401  (binding module imports cleanly without a GPU)
    return capi


@pytest.mark.parametrize("x,kw,msg", [
    (np.full((4, 5), np.nan), {}, "non-finite"),
    (np.full((4, 5), 7.0), {}, "[0, 2*pi)"),
    (np.zeros((4, 5)), {"model": ModelParams.__new__(ModelParams)}, "tau"),
    (np.zeros((4, 5)), {"gradient_lo": 1.0}, "lo must be"),
    (np.zeros((4, 5)), {"c": WeightField(np.ones((3, 4)), np.ones((4, 3)))}, "weight shapes"),
])
def test_pu_unwrap_validates_before_device_work(x, kw, msg):
    """pu_unwrap (csrc/pu_host.cu) checks the reference's ValueError cases in C
    before touching CUDA, so they are testable without a GPU."""
    capi = _capi_args()
    if "model" in kw:  # bypass the dataclass check to reach the C-side one
        object.__setattr__(kw["model"], "tau", -1.0)
        object.__setattr__(kw["model"], "delta", 1e-6)
    with pytest.raises(ValueError, match=re.escape(msg)):
        capi.unwrap_capi(x, **kw)


def test_pu_unwrap_params_and_weights_checked_in_c():
    capi = _capi_args()
    lib = _native.load()
    p = _native.PuIrlsParams()
    lib.pu_irls_params_default(p)
    assert (p.max_iter_cg_start, p.max_outer_iters, p.max_cg_iters_cap) == (5, 100, 10000)
    assert (p.rel_improvement_tol, p.cg_growth_factor, p.cg_rel_tol) == (1e-3, 1.7, 1e-10)
    bad = IrlsParams.__new__(IrlsParams)
    for f, v in dict(max_iter_cg_start=5, rel_improvement_tol=1e-3, cg_growth_factor=0.5, max_outer_iters=100,
                     max_cg_iters_cap=10000, cg_rel_tol=1e-10).items():
        object.__setattr__(bad, f, v)
    with pytest.raises(ValueError, match="cg_growth_factor"):
        capi.unwrap_capi(np.zeros((3, 3)), params=bad)
    neg = WeightField.__new__(WeightField)
    object.__setattr__(neg, "cv", -np.ones((2, 3)))
    object.__setattr__(neg, "ch", np.ones((3, 2)))
    with pytest.raises(ValueError, match="nonnegative"):
        capi.unwrap_capi(np.zeros((3, 3)), c=neg)
