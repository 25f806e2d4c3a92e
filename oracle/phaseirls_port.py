"""TEST INFRASTRUCTURE ONLY — numpy restatement of the reference unwrap path.

Used by tests/, __graft_entry__.smoke() and bench.py's CPU legs as the
checker; never by the product package.  Every function cites the reference
file:line it restates (paths relative to /root/reference/pkg/src/phaseirls).

Two Poisson-solve variants are provided for the preconditioner u block:
  * "dense": the reference's own method — eigenbases of the 1-D Neumann
    second-difference matrices from LAPACK `eigh`, applied as four dense GEMMs
    (preconditioner.py:51-100).  This is the algorithm the reference runs.
  * "dct": the exact restatement through orthonormal DCT-II/III
    (scipy.fft.dctn/idctn), lambda_k = 2 - 2cos(pi k / n).
    measured it against the dense path at 1.7e-12 relative (255x256) and
    end-to-end on C1-C3 with identical control flow; used for large grids.

Parity is pinned: tests/test_oracle_golden.py compares this module with the
outputs of the unmodified reference stored in tests/golden/.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

TWO_PI = 2.0 * np.pi
REPROJECT_EVERY = 50            # pcg.py:19
TINY_CURVATURE = 1e-300         # pcg.py:21


# ---------------------------------------------------------------------------
# phase.py
# ---------------------------------------------------------------------------

def wrap_principal(a, lo=-np.pi):
    """phase.py:118-137 — floor-based reduction into [lo, lo+2pi) + 2 fixes."""
    a = np.asarray(a, dtype=np.float64)
    k = np.floor((a - lo) / TWO_PI)
    y = a - TWO_PI * k
    y = np.where(y >= lo + TWO_PI, y - TWO_PI, y)
    return np.where(y < lo, y + TWO_PI, y)


def grad_wrapped(x, lo=-np.pi):
    """phase.py:140-149 with kernels.py:31-36 — (gv, gh) principal differences."""
    x = np.asarray(x, dtype=np.float64)
    gv = x[1:, :] - x[:-1, :]
    gh = x[:, 1:] - x[:, :-1]
    if gv.size:
        gv = wrap_principal(gv, lo)
    if gh.size:
        gh = wrap_principal(gh, lo)
    return gv, gh


def check_wrapped(x):
    """phase.py:100-115 — fp64, 2-D, non-empty, finite, within [0, 2pi)."""
    arr = np.asarray(x, dtype=np.float64)
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"phase grid must be 2-D and non-empty, got shape {arr.shape}")
    if not np.all(np.isfinite(arr)):
        raise ValueError("phase grid contains non-finite values")
    if arr.min() < 0.0 or arr.max() >= TWO_PI:
        raise ValueError("wrapped phase values must lie in [0, 2*pi)")
    return arr


def congruent_round(u, x):
    """phase.py:178-184."""
    return x + TWO_PI * np.rint((u - x) / TWO_PI)


def kmap(u, x):
    """Integer ambiguity map K = rint((u - x)/2pi) (harness)."""
    return np.rint((np.asarray(u) - np.asarray(x)) / TWO_PI)


# ---------------------------------------------------------------------------
# operators.py / kernels.py — the unknown is a triple (u, vv, vh)
# ---------------------------------------------------------------------------

@dataclass
class Triple:
    """operators.py:39-101 — SystemVector restated (BLAS-1 in numpy)."""
    u: np.ndarray
    vv: np.ndarray
    vh: np.ndarray

    @classmethod
    def zeros(cls, n, m):
        return cls(np.zeros((n, m)), np.zeros((n - 1, m)), np.zeros((n, m - 1)))

    def copy(self):
        return Triple(self.u.copy(), self.vv.copy(), self.vh.copy())

    def dot(self, o):                                   # operators.py:70-75
        return (float(np.vdot(self.u, o.u)) + float(np.vdot(self.vv, o.vv))
                + float(np.vdot(self.vh, o.vh)))

    def norm(self):                                     # operators.py:77-78
        return float(np.sqrt(self.dot(self)))

    def axpy(self, a, o):                               # operators.py:80-84
        self.u += a * o.u
        self.vv += a * o.vv
        self.vh += a * o.vh

    def scale(self, b):                                 # operators.py:86-89
        self.u *= b
        self.vv *= b
        self.vh *= b

    def add(self, o):                                   # operators.py:91-94
        self.u += o.u
        self.vv += o.vv
        self.vh += o.vh


def d_rows(u):
    return u[1:, :] - u[:-1, :]                         # kernels.py:31-32


def d_cols(u):
    return u[:, 1:] - u[:, :-1]                         # kernels.py:35-36


def d_rows_adj(v):                                      # kernels.py:39-43
    out = np.zeros((v.shape[0] + 1, v.shape[1]))
    out[:-1, :] -= v
    out[1:, :] += v
    return out


def d_cols_adj(v):                                      # kernels.py:46-50
    out = np.zeros((v.shape[0], v.shape[1] + 1))
    out[:, :-1] -= v
    out[:, 1:] += v
    return out


def system_apply(x: Triple, dv, dh, tau):
    """operators.py:138-153 / kernels.py:53-59 — the 3-block lifted system."""
    inv_tau = 1.0 / tau
    su = d_rows(x.u)
    ut = d_cols(x.u)
    au = inv_tau * (d_rows_adj(su - x.vv) + d_cols_adj(ut - x.vh))
    avv = dv * x.vv + inv_tau * (x.vv - su)
    avh = dh * x.vh + inv_tau * (x.vh - ut)
    return Triple(au, avv, avh)


def rhs(gv, gh, tau):
    """operators.py:156-162."""
    inv_tau = 1.0 / tau
    return Triple(inv_tau * (d_rows_adj(gv) + d_cols_adj(gh)), -inv_tau * gv, -inv_tau * gh)


# ---------------------------------------------------------------------------
# preconditioner.py
# ---------------------------------------------------------------------------

def neumann_eig(n):
    """preconditioner.py:51-74 — eigenpairs of the 1-D Neumann stencil."""
    lap = np.zeros((n, n))
    if n > 1:
        i = np.arange(n)
        lap[i, i] = 2.0
        lap[0, 0] = lap[-1, -1] = 1.0
        lap[i[:-1], i[:-1] + 1] = -1.0
        lap[i[:-1] + 1, i[:-1]] = -1.0
    vals, vecs = np.linalg.eigh(lap)
    if abs(vals[0]) > 1e-10:
        raise RuntimeError(f"expected a zero eigenvalue, got {vals[0]}")
    vals = vals.copy()
    vals[0] = 0.0
    return vals, vecs


class DensePoisson:
    """preconditioner.py:77-100 — dense-eigenbasis Sylvester pseudo-inverse."""

    def __init__(self, n, m):
        self.ls, self.ps = neumann_eig(n)
        self.lt, self.pt = neumann_eig(m)

    def __call__(self, r, tau):
        rp = self.ps.T @ r @ self.pt
        den = self.ls[:, None] + self.lt[None, :]
        zero = den == 0.0
        zp = tau * rp / np.where(zero, 1.0, den)
        zp[zero] = 0.0
        return self.ps @ zp @ self.pt.T


def neumann_lambda(n):
    """Analytic eigenvalues 2 - 2cos(pi k / n) of the Neumann stencil, evaluated
    cancellation-free as 4 sin^2(pi k / 2n) (the naive form loses ~7 digits on
    lambda_1 at n = 4096)."""
    return 4.0 * np.sin(np.pi * np.arange(n) / (2.0 * n)) ** 2


class DctPoisson:
    """Exact DCT restatement of sylvester_solve."""

    def __init__(self, n, m, workers=-1):
        from scipy import fft as _fft
        self._fft = _fft
        self.workers = workers
        self.den = neumann_lambda(n)[:, None] + neumann_lambda(m)[None, :]
        self.den[0, 0] = 1.0

    def __call__(self, r, tau):
        rp = self._fft.dctn(r, type=2, norm="ortho", workers=self.workers)
        zp = tau * rp / self.den
        zp[0, 0] = 0.0
        return self._fft.idctn(zp, type=2, norm="ortho", workers=self.workers)


def make_poisson(n, m, kind="dense"):
    return DensePoisson(n, m) if kind == "dense" else DctPoisson(n, m)


def precond_apply(r: Triple, dv, dh, tau, poisson):
    """preconditioner.py:103-115."""
    inv_tau = 1.0 / tau
    return Triple(poisson(r.u, tau), r.vv / (dv + inv_tau), r.vh / (dh + inv_tau))


# ---------------------------------------------------------------------------
# objective.py
# ---------------------------------------------------------------------------

def weights(x: Triple, cv, ch, delta):
    """objective.py:92-100 — closed-form eta-trick weights."""
    d2 = delta * delta
    return np.sqrt((cv * x.vv) ** 2 + d2), np.sqrt((ch * x.vh) ** 2 + d2)


def penalty(x: Triple, gv, gh, tau):
    """objective.py:52-55."""
    rv = d_rows(x.u) - gv - x.vv
    rh = d_cols(x.u) - gh - x.vh
    return (float(np.vdot(rv, rv)) + float(np.vdot(rh, rh))) / (2.0 * tau)


def f_l1(x, gv, gh, cv, ch, tau):
    """objective.py:63-66 — F = weighted L1 + coupling penalties."""
    l1 = float(np.sum(np.abs(cv * x.vv))) + float(np.sum(np.abs(ch * x.vh)))
    return l1 + penalty(x, gv, gh, tau)


def f_delta(x, gv, gh, cv, ch, tau, delta):
    """objective.py:69-74."""
    d2 = delta * delta
    return (float(np.sum(np.sqrt((cv * x.vv) ** 2 + d2)))
            + float(np.sum(np.sqrt((ch * x.vh) ** 2 + d2))) + penalty(x, gv, gh, tau))


def h_delta(x, w, gv, gh, cv, ch, tau, delta):
    """objective.py:77-89 — lifted objective H_delta(x, w)."""
    wv, wh = w
    d2 = delta * delta
    sv = 0.5 * float(np.sum(((cv * x.vv) ** 2 + d2) / wv + wv))
    sh = 0.5 * float(np.sum(((ch * x.vh) ** 2 + d2) / wh + wh))
    return sv + sh + penalty(x, gv, gh, tau)


def lipschitz(cmax, tau, delta):
    """objective.py:103-105."""
    return 12.0 / tau + cmax ** 2 / delta


def candidate(x, w, gv, gh, cv, ch, tau, lip):
    """objective.py:108-125 — explicit gradient step of size 1/L."""
    wv, wh = w
    inv_tau = 1.0 / tau
    rv = d_rows(x.u) - gv - x.vv
    rh = d_cols(x.u) - gh - x.vh
    grad = Triple(inv_tau * (d_rows_adj(rv) + d_cols_adj(rh)),
                  cv * cv / wv * x.vv - inv_tau * rv,
                  ch * ch / wh * x.vh - inv_tau * rh)
    out = x.copy()
    out.axpy(-1.0 / lip, grad)
    return out


# ---------------------------------------------------------------------------
# pcg.py
# ---------------------------------------------------------------------------

class Breakdown(RuntimeError):
    """pcg.py:24-29."""

    def __init__(self, iteration, msg):
        super().__init__(f"iteration {iteration}: {msg}")
        self.iteration = iteration


def pcg(apply_a, apply_m, b: Triple, x0: Triple, max_iters, rel_tol):
    """pcg.py:47-116 — returns dict(x, iterations, norms, converged, r)."""
    x = x0.copy()
    thr = rel_tol * b.norm()
    r = b.copy()
    r.axpy(-1.0, apply_a(x))
    norms = [r.norm()]
    if not np.isfinite(norms[0]):
        raise Breakdown(0, "initial residual is not finite")
    if norms[0] <= thr or max_iters == 0:
        return dict(x=x, iterations=0, norms=norms, converged=norms[0] <= thr, r=r)
    z = apply_m(r)
    p = z.copy()
    rho = r.dot(z)
    converged = False
    for it in range(max_iters):
        ap = apply_a(p)
        pap = p.dot(ap)
        if not np.isfinite(pap):
            raise Breakdown(it, "curvature p'Ap is not finite")
        if pap <= TINY_CURVATURE:
            converged = norms[-1] <= thr
            break
        alpha = rho / pap
        x.axpy(alpha, p)
        r.axpy(-alpha, ap)
        if (it + 1) % REPROJECT_EVERY == 0:
            r.u -= r.u.mean()
        rn = r.norm()
        if not np.isfinite(rn):
            raise Breakdown(it + 1, "residual norm is not finite")
        norms.append(rn)
        if rn <= thr:
            converged = True
            break
        z = apply_m(r)
        rho_next = r.dot(z)
        if not np.isfinite(rho_next):
            raise Breakdown(it + 1, "preconditioned product is not finite")
        beta = rho_next / rho
        rho = rho_next
        p.scale(beta)
        p.add(z)
    return dict(x=x, iterations=len(norms) - 1, norms=norms, converged=converged, r=r)


# ---------------------------------------------------------------------------
# irls.py
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Params:
    """irls.py:43-50 defaults (validation lives in the product dataclass)."""
    max_iter_cg_start: int = 5
    rel_improvement_tol: float = 1e-3
    cg_growth_factor: float = 1.7
    max_outer_iters: int = 100
    max_cg_iters_cap: int = 10_000
    cg_rel_tol: float = 1e-10


def budget(delta_rel, m_prev, m_prev2, p: Params):
    """irls.py:118-129 — (action, m_cg)."""
    if m_prev < 1:
        raise ValueError("m_prev must be >= 1")
    if delta_rel > p.rel_improvement_tol:
        return "keep", m_prev
    if m_prev != m_prev2:
        return "stop", m_prev
    if m_prev >= p.max_cg_iters_cap:
        return "stop", m_prev
    return "grow", min(math.ceil(p.cg_growth_factor * m_prev), p.max_cg_iters_cap)


@dataclass
class Record:
    """irls.py:67-75."""
    k: int
    m_cg: int
    delta_rel: float | None
    h_delta: float
    cg_iters: int
    sufficient_decrease: bool
    fallback_used: bool


def unwrap(x, cv=None, ch=None, tau=1e-2, delta=1e-6, params: Params | None = None,
           lo=-np.pi, poisson="dense", m_schedule=None):
    """irls.py:132-224.  Returns (Triple state, list[Record], (gv, gh)).

    `m_schedule` (harness only) replays a given CG-budget sequence instead of
    deciding it, so that a control-flow divergence can be isolated.
    """
    arr = check_wrapped(x)
    n, m = arr.shape
    p = params or Params()
    if cv is None:
        cv, ch = np.ones((n - 1, m)), np.ones((n, m - 1))
    gv, gh = grad_wrapped(arr, lo)
    b = rhs(gv, gh, tau)
    solver = make_poisson(n, m, poisson)
    cmax = max(float(cv.max()) if cv.size else 0.0, float(ch.max()) if ch.size else 0.0)
    lip = lipschitz(cmax, tau, delta)

    state = Triple(np.zeros((n, m)), -gv.copy(), -gh.copy())
    records = []
    hist = [p.max_iter_cg_start]
    w_prev = None
    for k in range(p.max_outer_iters):
        w = weights(state, cv, ch, delta)
        delta_rel = None
        if k >= 1:
            h_old = h_delta(state, w_prev, gv, gh, cv, ch, tau, delta)
            h_new = h_delta(state, w, gv, gh, cv, ch, tau, delta)
            if h_old == 0:
                delta_rel = 0.0
            else:
                if h_old <= 0:
                    raise ValueError("reference objective value must be positive")
                delta_rel = (h_old - h_new) / h_old
            m_prev = hist[k - 1]
            m_prev2 = hist[k - 2] if k >= 2 else m_prev
            action, m_cg = budget(delta_rel, m_prev, m_prev2, p)
            if m_schedule is not None:
                if k >= len(m_schedule):
                    break
                action, m_cg = "replay", m_schedule[k]
            if action == "stop":
                break
            hist.append(m_cg)
        else:
            m_cg = hist[0] if m_schedule is None else m_schedule[0]
        dv = cv * cv / w[0]
        dh = ch * ch / w[1]
        out = pcg(lambda v: system_apply(v, dv, dh, tau),
                  lambda r: precond_apply(r, dv, dh, tau, solver),
                  b, state, m_cg, p.cg_rel_tol)
        prop = out["x"]
        cand = candidate(state, w, gv, gh, cv, ch, tau, lip)
        ok = (h_delta(prop, w, gv, gh, cv, ch, tau, delta)
              <= h_delta(cand, w, gv, gh, cv, ch, tau, delta))
        acc = prop if ok else cand
        acc.u -= acc.u.mean()
        records.append(Record(k, m_cg, delta_rel, h_delta(acc, w, gv, gh, cv, ch, tau, delta),
                              out["iterations"], bool(ok), not ok))
        state = acc
        w_prev = w
    return state, records, (gv, gh)
