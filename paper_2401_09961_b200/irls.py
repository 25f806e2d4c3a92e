"""The unwrap hot path on one B200 (reference irls.py:132-224).

Mirrors the reference outer loop line by line — weight refresh, lifted
objective pair and CG-budget rule, warm-started PCG, explicit-gradient
safeguard, mean centring, trace — with every array operation running in
libpu_unwrap.so on HBM-resident buffers.  The host synchronises once per
outer iteration, to read the H_delta pair that drives the budget decision
(plus the previous iteration's trace scalars).
"""

from __future__ import annotations

import os

import numpy as np

from .device import Workspace, _ptr
from .params import (BudgetDecision, IrlsParams, IrlsTrace, IterationRecord, ModelParams,  # noqa: F401
                     UnwrapResult, cg_budget_update, lipschitz_constant, relative_improvement)
from .pcg import raise_if_breakdown
from .phase import WeightField, validate_wrapped

# pu_accept_weights_start: acceptance of k and the start-up of k + 1 in one
# pass.  Used on grids of >= 2048^2 cells (C3 fp32: 120.1 -> 116.5 ms; fp64:
# the 1-CTA/SM build, 0.70 vs 0.80 ms per outer iteration); on small grids
# the separate start-up is what keeps the GPU busy while the host applies the
# budget rule (C1 512^2: 10.3 -> 10.6 ms fused).
# PU_FUSED_START=0 / 1 forces it off / on (A/B timing).
FUSED_START = os.environ.get("PU_FUSED_START", "auto")
FUSED_START_MIN_CELLS = 2048 * 2048


# b = build_rhs(gv, gh) formed inside the start-up kernel (b = NULL at the C
# ABI) instead of stored once and read by every start-up: fp32 only (C3 fp32
# -0.5%; in fp64 the extra registers spill and the start-up is 2.6% slower).
# PU_RHS_IN_KERNEL=0 / 1 forces stored / formed (A/B timing).
RHS_IN_KERNEL = os.environ.get("PU_RHS_IN_KERNEL", "auto")


def _rhs_in_kernel(ws):
    if RHS_IN_KERNEL in ("0", "1"):
        return RHS_IN_KERNEL == "1"
    return ws.tdtype == _torch().float32


def _fuse_start(ws, concurrent=False):
    """concurrent: several unwraps share the GPU (unwrap_many), so the others
    cover the host's budget decision at any grid size (C5 64 x 1024² fp32:
    579 -> 561 ms fused)."""
    if FUSED_START in ("0", "1"):
        return FUSED_START == "1"
    return concurrent or ws.n * ws.m >= FUSED_START_MIN_CELLS


def _torch():
    import torch
    return torch


class DeviceUnwrap:
    """Resident buffers and launch sequence of one unwrap (one stream).

    Per outer iteration k two fused C-ABI calls run on the device:
      pu_irls_step      candidate step + warm-started PCG in place on the state
                        + H(proposal), H(cand)               (irls.py:191-205)
      pu_accept_weights select + centre + H(accepted, w_k), then the weights
                        of iteration k+1 and H(accepted, w_{k+1})
                        (irls.py:206-215, 173-177)
    so the host reads one scalar block per iteration for the budget rule.
    pu_irls_step runs as its two halves (pu_irls_begin, budget-free, enqueued
    speculatively; pu_irls_iterate).  With _fuse_start, the acceptance is
    pu_accept_weights_start, which also runs the candidate step and PCG
    start-up of k + 1, and the next begin shrinks to pu_irls_begin_z0.
    """

    def __init__(self, ws: Workspace):
        self.ws = ws
        self.S = [ws.buf("state0", 3), ws.buf("state1", 3)]  # state ping-pong
        # explicit-gradient candidate of iteration k in Cs[k & 1] (the fused
        # acceptance of k reads Cs[k & 1] while it writes the candidate of k + 1)
        self.Cs = [ws.buf("cand", 3), ws.buf("cand1", 3)]
        self.B = None                    # stored rhs (None: formed in the start-up kernel)
        self.concurrent = False          # set by unwrap_many when unwraps share the GPU
        self.prestarted = False
        self.G = ws.buf("grad", 2)       # gv, gh
        self.W = None                    # arc weights cv, ch (None: uniform)
        self.Wt = [ws.buf("w0", 2), ws.buf("w1", 2)]
        self.D = ws.buf("diag", 2)       # dv, dh
        self.R = ws.buf("pcg_r", 3)
        self.P = [ws.buf("pcg_p0", 3), ws.buf("pcg_p1", 3)]
        self.spec = ws.buf("spec", 1)
        self.cur = 0

    def _c(self):
        return (None, None) if self.W is None else (_ptr(self.W[0]), _ptr(self.W[1]))

    def load(self, x_dev, c: WeightField | None, lo):
        ws, st = self.ws, self.ws.stream()
        torch = _torch()
        if c is None:
            self.W, self._keep = None, None
        else:
            self.W = ws.buf("cw", 2)
            self._keep = [ws.pack(c.cv, self.W[0]), ws.pack(c.ch, self.W[1])]
        x64 = x_dev if x_dev.dtype == torch.float64 else x_dev.to(torch.float64)
        self._x = x64.contiguous()
        # gradients + the input check of phase.py:100-115 from the same loads;
        # the counts are read with the first scalar snapshot (check_input)
        ws.call("pu_wrapped_gradients_checked", _ptr(self._x), int(self._x.shape[1]), _ptr(self.G[0]),
                _ptr(self.G[1]), float(lo), ws.sp(ws.S_CHK_NF), st)
        if _rhs_in_kernel(ws):
            self.B = None
        else:
            self.B = ws.buf("rhs", 3)
            ws.call("pu_build_rhs", _ptr(self.G[0]), _ptr(self.G[1]), _ptr(self.B), st)
        ws.call("pu_init_state", _ptr(self.G[0]), _ptr(self.G[1]), _ptr(self.S[0]), st)
        self.cur = 0
        self.prestarted = False
        cv, ch = self._c()
        w = self.Wt[0]  # w_0, d_0 (irls.py:173, 191)
        ws.call("pu_weights_hpair", _ptr(self.S[0]), cv, ch, _ptr(self.G[0]), _ptr(self.G[1]), None, None,
                _ptr(w[0]), _ptr(w[1]), _ptr(self.D[0]), _ptr(self.D[1]), ws.sp(ws.S_HOLD), st)

    def step(self, k, m_cg, params: IrlsParams, lip):
        """irls.py:191-215 for iteration k, then the weights of k + 1."""
        self.begin(k, params, lip)
        self.finish(k, m_cg, params, lip)

    def begin(self, k, params: IrlsParams, lip):
        """The budget-independent half of iteration k (pu_irls_begin): candidate
        step, PCG start-up, z0 = M r0.  Leaves the state untouched, so it may run
        before the host has decided whether iteration k happens at all.  When
        the previous finish() already ran the candidate step and start-up
        (pu_accept_weights_start), only their finalisation and z0 remain."""
        ws, st = self.ws, self.ws.stream()
        cv, ch = self._c()
        w = self.Wt[k & 1]
        norms = ws.ensure_norms(64)
        if self.prestarted:
            self.prestarted = False
            ws.call("pu_irls_begin_z0", _ptr(self.D[0]), _ptr(self.D[1]), float(params.cg_rel_tol), _ptr(self.R),
                    _ptr(self.P[0]), _ptr(self.P[1]), _ptr(self.spec), _ptr(ws.ctrl), _ptr(norms), st)
            return
        # b = NULL: the right-hand side build_rhs(gv, gh) (operators.py:156-162)
        # is formed inside the start-up kernel from its gradient loads
        ws.call("pu_irls_begin", _ptr(self.S[self.cur]), None if self.B is None else _ptr(self.B), _ptr(self.G[0]), _ptr(self.G[1]), cv, ch,
                _ptr(w[0]), _ptr(w[1]), _ptr(self.D[0]), _ptr(self.D[1]), float(lip), float(params.cg_rel_tol),
                _ptr(self.Cs[k & 1]), _ptr(self.R), _ptr(self.P[0]), _ptr(self.P[1]), _ptr(self.spec), _ptr(ws.ctrl),
                _ptr(norms), st)

    def finish(self, k, m_cg, params: IrlsParams, lip=None):
        """The budget's PCG iterations + H pair (pu_irls_iterate), then the
        acceptance and the weights of k + 1 (pu_accept_weights; with `lip`,
        pu_accept_weights_start, which also runs the candidate step and PCG
        start-up of k + 1 in the same pass)."""
        ws, st = self.ws, self.ws.stream()
        cv, ch = self._c()
        cur, nxt = self.S[self.cur], self.S[1 - self.cur]
        w, wn = self.Wt[k & 1], self.Wt[(k + 1) & 1]
        norms = ws.ensure_norms(max(m_cg, 64))
        ws.call("pu_irls_iterate", _ptr(cur), _ptr(self.G[0]), _ptr(self.G[1]), cv, ch, _ptr(w[0]), _ptr(w[1]),
                _ptr(self.D[0]), _ptr(self.D[1]), int(m_cg), _ptr(self.Cs[k & 1]), _ptr(self.R), _ptr(self.P[0]),
                _ptr(self.P[1]), _ptr(self.spec), _ptr(ws.ctrl), _ptr(norms), ws.sp(ws.S_HPROP), st)
        args = (_ptr(cur), _ptr(self.Cs[k & 1]), ws.sp(ws.S_MEAN), _ptr(nxt), _ptr(self.G[0]), _ptr(self.G[1]), cv, ch,
                _ptr(w[0]), _ptr(w[1]), _ptr(wn[0]), _ptr(wn[1]), _ptr(self.D[0]), _ptr(self.D[1]),
                ws.sp(ws.S_HACC))
        if lip is not None and _fuse_start(ws, self.concurrent) and k + 1 < params.max_outer_iters:
            ws.call("pu_accept_weights_start", *args, float(lip), _ptr(self.R), _ptr(self.Cs[(k + 1) & 1]), st)
            self.prestarted = True
        else:
            ws.call("pu_accept_weights", *args, st)
        self.cur = 1 - self.cur

    @property
    def state(self):
        return self.S[self.cur]

    def detach(self):
        """A copy of the result-bearing buffers (state, gradients, arc
        weights) that stays valid after this workspace runs another unwrap."""
        return DetachedUnwrap(self.ws, self.state.clone(), self.G.clone(),
                              None if self.W is None else self.W.clone())

    def result_arrays(self):
        return self.ws.from_system(self.state)

    def weight_planes(self):
        """(cv, ch) device planes; a filled unit plane pair for uniform weights."""
        if self.W is not None:
            return self.W
        ones = self.ws.buf("ones", 2)
        self.ws.call("pu_fill", _ptr(ones), 2, 1.0, self.ws.stream())
        return ones


class DetachedUnwrap:
    """Result of one unwrap held in its own device buffers (unwrap_many with
    download=False); same read-side interface as DeviceUnwrap."""

    def __init__(self, ws, state, G, W):
        self.ws, self._state, self.G, self.W = ws, state, G, W

    @property
    def state(self):
        return self._state

    def result_arrays(self):
        return self.ws.from_system(self._state)

    def weight_planes(self):
        if self.W is not None:
            return self.W
        ones = self.ws.planes(2)
        self.ws.call("pu_fill", _ptr(ones), 2, 1.0, self.ws.stream())
        return ones


def check_input(scal, ws):
    """phase.py:108-114 from the counts pu_wrapped_gradients_checked left in
    the scalar block: the reference's ValueError, raised before any result."""
    if scal[ws.S_CHK_NF] != 0.0:
        raise ValueError("phase grid contains non-finite values")
    if scal[ws.S_CHK_RANGE] != 0.0:
        raise ValueError("wrapped phase values must lie in [0, 2*pi)")


def _record(k, m_cg, delta_rel, scal, ctrl, ws):
    raise_if_breakdown(ctrl)
    sufficient = bool(scal[ws.S_TAKE] != 0.0)
    return IterationRecord(k=k, m_cg=m_cg, delta_rel=delta_rel, h_delta=float(scal[ws.S_HACC]),
                           cg_iters=int(ctrl["iterations"]), sufficient_decrease=sufficient,
                           fallback_used=not sufficient)


def unwrap_device(x_dev, c: WeightField | None, model: ModelParams, params: IrlsParams, gradient_lo,
                  dtype="fp64", ws: Workspace | None = None):
    """Run the loop on a device fp64 grid; returns (DeviceUnwrap, IrlsTrace).

    The loop runs on the workspace's own stream (CUDA graphs cannot capture
    the legacy default stream), ordered after and before the caller's stream.
    """
    n, m = int(x_dev.shape[0]), int(x_dev.shape[1])
    ws = ws or Workspace.get(n, m, dtype, model.tau, model.delta, x_dev.device)
    torch = _torch()
    caller = torch.cuda.current_stream(ws.device)
    s = ws.solve_stream()
    s.wait_stream(caller)
    with torch.cuda.stream(s):
        out = _unwrap_loop(ws, x_dev, c, model, params, gradient_lo)
    caller.wait_stream(s)
    return out


class _LoopJob:
    """The host loop of irls.py:172-222 as a resumable state machine: each
    `advance()` reads the scalar block of the iteration in flight (the one
    synchronisation per outer iteration), applies the budget rule and enqueues
    the next iteration.  One job = one unwrap on its workspace's stream;
    several jobs interleave on one GPU (unwrap_many)."""

    def __init__(self, ws, x_dev, c, model, params, gradient_lo, concurrent=False):
        self.ws, self.params = ws, params
        self.run = DeviceUnwrap(ws)
        self.run.concurrent = concurrent
        self.run.load(x_dev, c, gradient_lo)
        cmax = 1.0 if c is None else c.max_weight
        self.lip = 12.0 / model.tau + cmax ** 2 / model.delta          # objective.py:103-105
        self.trace = IrlsTrace()
        self.m_history = [params.max_iter_cg_start]
        self.pending = None  # (k, m_cg, delta_rel) of the enqueued iteration awaiting its scalars
        self.k = 0
        if params.max_outer_iters > 0:
            self._enqueue(0, self.m_history[0])
            self.pending = (0, self.m_history[0], None)
            self.k = 1

    def _enqueue(self, k, m_cg):
        """finish iteration k, snapshot its scalars, and start k + 1 speculatively
        (pu_irls_begin does not depend on the budget and leaves the state
        untouched), so the GPU keeps working while the host reads the snapshot
        and applies the budget rule."""
        if k == 0:
            self.run.begin(0, self.params, self.lip)
        self.run.finish(k, m_cg, self.params, self.lip)
        self.ws.snapshot()
        if k + 1 < self.params.max_outer_iters:
            self.run.begin(k + 1, self.params, self.lip)

    def advance(self):
        """Returns True once the loop has finished (trace complete)."""
        if self.pending is None:
            return True
        ws, params = self.ws, self.params
        scal, ctrl = ws.read_snapshot()
        if self.k == 1:
            check_input(scal, ws)  # the input check rides on the first snapshot
        self.trace.append(_record(*self.pending, scal, ctrl, ws))
        self.pending = None
        k = self.k
        if k >= params.max_outer_iters:
            return True
        # H(state_k, w_{k-1}) is the accepted value of k-1; H(state_k, w_k) its refresh
        h_old, h_new = float(scal[ws.S_HACC]), float(scal[ws.S_HNEXT])
        delta_rel = 0.0 if h_old == 0 else relative_improvement(h_old, h_new)
        m_prev = self.m_history[k - 1]
        m_prev2 = self.m_history[k - 2] if k >= 2 else m_prev
        decision = cg_budget_update(delta_rel, m_prev, m_prev2, params)
        if decision.action == "stop":
            return True
        m_cg = decision.m_cg
        self.m_history.append(m_cg)
        self._enqueue(k, m_cg)
        self.pending = (k, m_cg, delta_rel)
        self.k = k + 1
        return False


def _unwrap_loop(ws, x_dev, c, model, params, gradient_lo):
    job = _LoopJob(ws, x_dev, c, model, params, gradient_lo)
    while not job.advance():
        pass
    return job.run, job.trace


def unwrap_many(xs, c: WeightField | None = None, model: ModelParams | None = None, params: IrlsParams | None = None,
                gradient_lo=-np.pi, *, dtype="fp64", concurrency=8, device=None, download=True):
    """Unwrap independent grids of one size concurrently on one GPU (BASELINE
    config C5): up to `concurrency` unwraps in flight, each on its own
    workspace and stream; the host round-robins over them, so while it waits
    for one iteration's scalars the others keep the GPU busy.  Results are
    identical to calling `unwrap` on each grid.  Returns UnwrapResults (or
    (DeviceUnwrap, trace) pairs when download=False)."""
    from . import _native
    _native.ensure()
    torch = _torch()
    model = model or ModelParams()
    params = params or IrlsParams()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if not xs:
        return []
    n, m = int(xs[0].shape[0]), int(xs[0].shape[1])
    for xi in xs:
        if isinstance(xi, np.ndarray) and not np.issubdtype(xi.dtype, np.number):
            raise ValueError("phase grid must be numeric")
        if len(xi.shape) != 2 or tuple(xi.shape) != (n, m):
            raise ValueError(f"all grids must share one 2-D shape, got {tuple(xi.shape)} vs {(n, m)}")
    _check_call(c, n, m, gradient_lo)
    slots = max(1, min(int(concurrency), len(xs)))
    wss = [Workspace.get(n, m, dtype, model.tau, model.delta, dev, slot=s) for s in range(slots)]
    caller = torch.cuda.current_stream(dev)
    out = [None] * len(xs)
    active = {}  # slot -> (index, job)
    nxt = 0

    def start(slot):
        nonlocal nxt
        i = nxt
        nxt += 1
        xi = xs[i]
        if tuple(xi.shape) != (n, m):
            raise ValueError(f"all grids must share one shape, got {tuple(xi.shape)} vs {(n, m)}")
        ws = wss[slot]
        s = ws.solve_stream()
        s.wait_stream(caller)
        with torch.cuda.stream(s):
            x_dev = xi.to(device=dev, dtype=torch.float64) if isinstance(xi, torch.Tensor) else ws.upload_grid(xi)
            _check_shape(x_dev)
            active[slot] = (i, _LoopJob(ws, x_dev, c, model, params, gradient_lo, concurrent=slots > 1))

    for slot in range(slots):
        start(slot)
    while active:
        for slot in list(active):
            i, job = active[slot]
            ws = wss[slot]
            with torch.cuda.stream(ws.solve_stream()):
                finished = job.advance()
                if finished:
                    if download:
                        u, vv, vh = ws.download_system(job.run.state)
                        out[i] = UnwrapResult(u=u, vv=vv, vh=vh, trace=job.trace)
                    elif nxt < len(xs):
                        # the slot's buffers are about to be reused by the next
                        # image: the result keeps its own copy of what it needs
                        out[i] = (job.run.detach(), job.trace)
                    else:
                        out[i] = (job.run, job.trace)
            if finished:
                del active[slot]
                caller.wait_stream(ws.solve_stream())
                if nxt < len(xs):
                    start(slot)
    return out


def _check_call(c, n, m, gradient_lo):
    """The argument checks of irls.py:157-160 (weight shapes) and
    phase.py:140-149 (gradient interval), shared by unwrap and unwrap_many so
    a mis-shaped WeightField raises instead of being cropped or padded."""
    if c is not None and (c.cv.shape != (n - 1, m) or c.ch.shape != (n, m - 1)):
        raise ValueError(f"weight shapes {c.cv.shape}/{c.ch.shape} do not match grid {(n, m)}")
    if gradient_lo not in (0.0, 0, -np.pi):
        raise ValueError(f"lo must be 0 or -pi, got {gradient_lo!r}")


def _check_shape(x_dev):
    """phase.py:104-106; the value checks (phase.py:108-114) run inside the
    gradient kernel and are read with the first scalar snapshot."""
    if x_dev.dim() != 2 or x_dev.shape[0] < 1 or x_dev.shape[1] < 1:
        raise ValueError(f"phase grid must be 2-D and non-empty, got shape {tuple(x_dev.shape)}")


def unwrap(x, c: WeightField | None = None, model: ModelParams | None = None, params: IrlsParams | None = None,
           gradient_lo=-np.pi, *, dtype="fp64", device=None):
    """irls.py:132-224 — unwrap a wrapped phase grid on the GPU.

    Same parameters and result as the reference; `dtype` ("fp64" default,
    or "fp32") selects the arithmetic of the device buffers (reductions are
    always accumulated in fp64).  `x` may be a numpy array or a CUDA tensor.
    """
    from . import _native
    _native.ensure()  # library + CUDA device, or raise: there is no CPU path
    torch = _torch()
    dev = torch.device(device) if device is not None else (
        x.device if isinstance(x, torch.Tensor) and x.is_cuda else torch.device("cuda", torch.cuda.current_device()))
    if isinstance(x, np.ndarray) and not np.issubdtype(x.dtype, np.number):
        raise ValueError("phase grid must be numeric")
    if isinstance(x, torch.Tensor) and x.is_cuda:
        x_dev = x.to(device=dev, dtype=torch.float64)
    else:
        arr = x if isinstance(x, torch.Tensor) else np.asarray(x, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
            raise ValueError(f"phase grid must be 2-D and non-empty, got shape {tuple(arr.shape)}")
        ws_in = Workspace.get(int(arr.shape[0]), int(arr.shape[1]), dtype, (model or ModelParams()).tau,
                              (model or ModelParams()).delta, dev)
        x_dev = ws_in.upload_grid(arr if isinstance(arr, torch.Tensor) else arr)
    _check_shape(x_dev)  # values: checked by the gradient kernel (check_input)
    n, m = int(x_dev.shape[0]), int(x_dev.shape[1])
    model = model or ModelParams()
    params = params or IrlsParams()
    _check_call(c, n, m, gradient_lo)
    # the host is idle while the device loop runs: allocate and page in the
    # result arrays meanwhile, so the final widening copy touches no new pages
    import threading
    outs = {}

    def _prefault():
        shapes = ((n, m), (n - 1, m), (n, m - 1))
        arrs = [np.empty((max(r, 0), max(q, 0)), dtype=np.float64) for r, q in shapes]
        for a in arrs:
            if a.size:
                torch.from_numpy(a).zero_()
        outs["arrays"] = arrs

    th = threading.Thread(target=_prefault, daemon=True)
    th.start()
    run, trace = unwrap_device(x_dev, c, model, params, gradient_lo, dtype)
    th.join()
    u, vv, vh = run.ws.download_system(run.state, out=outs.get("arrays"))
    return UnwrapResult(u=u, vv=vv, vh=vh, trace=trace)
