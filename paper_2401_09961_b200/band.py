"""One image row-sharded across GPUs (BASELINE config C4).

The reference unwraps one grid in one process (irls.py:132-224); this module
runs the same outer loop and the same PCG iteration (pcg.py:47-116) on a grid
split into contiguous row bands, one band per rank:

  halo       every plane of a band carries ghost rows -1 and `rows` that mirror
             the neighbours' edge rows; the stencils (A x, the candidate
             gradient, the penalty terms) read them.  Exchanged: the state
             (u both ways, vv down) after each acceptance, the proposal and the
             candidate u before the H pair, the u block of the search direction
             and the vv block of the residual after every PCG iteration, gv and
             dv when they change.  The vv block of the new direction in the
             ghost row is recomputed locally (k_ghost_pslack).
  all-reduce every reduction leaves the band's fp64 totals in a small buffer;
             the ranks sum them and every rank runs the same finaliser
             (pu_finalize), so all ranks hold identical PCG/IRLS scalars and
             take identical control-flow decisions.  Two per PCG iteration:
             p'Ap, then {||r||^2, rho_s, rho_u}.
  transpose  the 2-D DCT preconditioner (preconditioner.py:86-100) runs its
             row transforms on the row bands and its column transforms on
             column blocks: the row DCT-II writes the spectrum packed by
             destination, an all-to-all moves it, the column kernel works on
             the N x cols block, and the reverse all-to-all feeds the row
             DCT-III.  Two all-to-alls per PCG iteration.

Communicators: `LoopbackComm` holds every band in this process on one device
and implements the collectives as device copies (used to test the band
decomposition on a single GPU); `DistComm` has one band per process and uses
torch.distributed (NCCL over NVLink on a B200 box, gloo in the CPU tests of
the exchange plumbing).
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .device import _DTYPES, _ptr
from .params import IrlsParams, IrlsTrace, ModelParams, UnwrapResult, cg_budget_update, relative_improvement
from .phase import WeightField


def _torch():
    import torch
    return torch


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------
class BandLayout:
    """Row bands (near-equal, contiguous) and the column blocks of the transpose."""

    def __init__(self, n: int, m: int, world: int):
        if world < 1:
            raise ValueError(f"world size must be >= 1, got {world}")
        if n < 2 or m < 1:
            raise ValueError(f"grid {n}x{m} too small to shard")
        if n < world:
            raise ValueError(f"{n} rows cannot be split into {world} bands")
        self.n, self.m, self.world = int(n), int(m), int(world)
        base, extra = divmod(self.n, world)
        self.rows = [base + (1 if r < extra else 0) for r in range(world)]
        self.row0 = [int(v) for v in np.concatenate([[0], np.cumsum(self.rows)[:-1]])]
        per = -(-self.m // world)
        self.mb = max(8, -(-per // 8) * 8)
        self.col0 = [r * self.mb for r in range(world)]
        self.cols = [min(self.mb, self.m - c) for c in self.col0]
        if min(self.cols) < 1:
            raise ValueError(f"{m} columns cannot be split into {world} column blocks of {self.mb}")

    def band(self, r: int) -> nat.PuBand:
        return nat.PuBand(self.n, self.row0[r], self.rows[r], self.world, self.mb, self.col0[r], self.cols[r])


# ---------------------------------------------------------------------------
# per-band device state
# ---------------------------------------------------------------------------
class BandState:
    """Handle + HBM buffers of one band (planes stored as (k, rows + 2, ld):
    storage row 0 is the ghost row -1, rows 1..rows the band, rows + 1 the
    ghost row `rows`)."""

    NSCAL = 16
    (S_HOLD, S_HNEW, S_HPROP, S_HCAND, S_MEAN, S_TAKE, S_HACC, S_HNEXT) = range(8)

    def __init__(self, layout: BandLayout, rank: int, dtype: str, tau: float, delta: float, device, peer=False):
        torch = _torch()
        self.lib = nat.ensure()
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be 'fp32' or 'fp64', got {dtype!r}")
        self.layout, self.rank = layout, rank
        self.rows, self.row0 = layout.rows[rank], layout.row0[rank]
        self.n, self.m, self.mb, self.nq = layout.n, layout.m, layout.mb, layout.world
        self.code = _DTYPES[dtype]
        self.tdtype = torch.float32 if self.code == nat.PU_F32 else torch.float64
        self.device = device
        band = layout.band(rank)
        h = ctypes.c_void_p()
        with torch.cuda.device(device):
            nat.check(self.lib.pu_create_band(ctypes.byref(h), self.m, ctypes.byref(band), self.code, float(tau),
                                              float(delta)))
        self.h = h
        self.ld = int(self.lib.pu_pitch(h))
        z = lambda k: torch.zeros((k, self.rows + 2, self.ld), dtype=self.tdtype, device=device)  # noqa: E731
        self.S = [z(3), z(3)]
        self.Cs = [z(3), z(3)]  # candidates of even / odd outer iterations (the fused start writes k + 1's)
        self.G, self.D, self.R = z(2), z(2), z(3)
        self.Wt = [z(2), z(2)]
        self.P = [z(3), z(3)]
        self.W, self.use_w = None, False
        self.peer = bool(peer)
        self.col_ptr, self.back_ptr, self.peer_tables, self._opened = None, None, None, []
        if self.peer:
            # fused transpose (pu_set_band_peers): the column block and the back
            # buffer are plain cudaMalloc blocks so other ranks can map them
            # over NVLink (CUDA IPC) and store into them
            esz = 4 if self.code == nat.PU_F32 else 8
            ptrs = []
            for elems in (self.n * self.mb, self.nq * self.rows * self.mb):
                ptr = ctypes.c_void_p()
                with torch.cuda.device(device):
                    nat.check(self.lib.pu_dev_alloc(elems * esz, ctypes.byref(ptr)))
                ptrs.append(ptr.value)
            self.col_ptr, self.back_ptr = ptrs
            self.spec_send = self.spec_col = None
        else:
            self.spec_send = torch.zeros(self.nq * self.rows * self.mb, dtype=self.tdtype, device=device)
            self.spec_col = torch.zeros(self.n * self.mb, dtype=self.tdtype, device=device)
        self.totals = torch.zeros(nat.NSITES * nat.MAX_SUMS, dtype=torch.float64, device=device)
        ctrl_bytes = int(self.lib.pu_pcg_ctrl_bytes())
        self.block = torch.zeros(self.NSCAL * 8 + ctrl_bytes, dtype=torch.uint8, device=device)
        self.scal = self.block[: self.NSCAL * 8].view(torch.float64)
        self.ctrl = self.block[self.NSCAL * 8:]
        self.norms = torch.zeros(1, dtype=torch.float64, device=device)
        nat.check(self.lib.pu_set_band_totals(self.h, _ptr(self.totals)))
        self._ctrl_dtype = _ctrl_dtype()
        self.cur = 0

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and self.h.value:
                self.lib.pu_destroy(self.h)
            for q in getattr(self, "_opened", []):
                self.lib.pu_ipc_close(ctypes.c_void_p(q))
            for q in (getattr(self, "col_ptr", None), getattr(self, "back_ptr", None)):
                if q:
                    self.lib.pu_dev_free(ctypes.c_void_p(q))
        except Exception:
            pass

    def set_peers(self, cols, backs):
        """Column-block and back-buffer addresses of every rank (rank order) -> fused transpose."""
        torch = _torch()
        self.peer_tables = torch.tensor([[int(a) for a in cols], [int(a) for a in backs]], dtype=torch.int64,
                                        device=self.device)
        nat.check(self.lib.pu_set_band_peers(self.h, _ptr(self.peer_tables[0]), _ptr(self.peer_tables[1])))

    def col(self):
        return ctypes.c_void_p(self.col_ptr) if self.peer else _ptr(self.spec_col)

    def send(self):
        return ctypes.c_void_p(self.back_ptr) if self.peer else _ptr(self.spec_send)

    # pointers -------------------------------------------------------------
    @staticmethod
    def p(t, plane=0):
        """Device pointer to row 0 of plane `plane` of a band tensor."""
        return ctypes.c_void_p(t[plane, 1].data_ptr())

    def sp(self, slot):
        return ctypes.c_void_p(self.scal.data_ptr() + 8 * slot)

    def stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def call(self, name, *args):
        nat.check(getattr(self.lib, name)(self.h, *args))

    def ensure_norms(self, k):
        if self.norms.numel() < k + 1:
            self.norms = _torch().zeros(k + 1, dtype=_torch().float64, device=self.device)
        return self.norms

    def read_block(self):
        return self._parse(self.block.cpu().numpy())

    def _parse(self, host):
        scal = host[: self.NSCAL * 8].view(np.float64).copy()
        ctrl = host[self.NSCAL * 8:].view(self._ctrl_dtype)[0].copy()
        return scal, ctrl

    def snapshot(self):
        """Asynchronous copy of the scalar block (end of an outer iteration)
        into page-locked memory, so work enqueued after it (the speculative
        start-up of the next iteration) runs while the host reads it."""
        torch = _torch()
        if getattr(self, "_snap", None) is None:
            self._snap = torch.empty(self.block.numel(), dtype=torch.uint8, pin_memory=True)
            self._snap_ev = torch.cuda.Event()
        self._snap.copy_(self.block, non_blocking=True)
        self._snap_ev.record(torch.cuda.current_stream(self.device))

    def read_snapshot(self):
        self._snap_ev.synchronize()
        return self._parse(self._snap.numpy())

    def pack_rows(self, arr, dst, plane, r0, nrows):
        """Host/device fp64 rows [r0, r0 + nrows) of a compact array -> band rows of dst[plane]."""
        torch = _torch()
        src = torch.as_tensor(np.ascontiguousarray(arr[r0:r0 + nrows], dtype=np.float64)) \
            if isinstance(arr, np.ndarray) else arr[r0:r0 + nrows]
        src = src.to(device=self.device, dtype=torch.float64).contiguous()
        rows, cols = (int(src.shape[0]), int(src.shape[1])) if src.numel() else (0, 0)
        self.call("pu_pack", _ptr(src) if src.numel() else ctypes.c_void_p(0), max(cols, 1), rows, cols,
                  self.p(dst, plane), self.stream())
        return src


def _ctrl_dtype():
    return np.dtype([("rho", "<f8"), ("alpha", "<f8"), ("beta", "<f8"), ("thr", "<f8"), ("bnorm", "<f8"),
                     ("pap", "<f8"), ("rn", "<f8"), ("mean_ru", "<f8"), ("rho_s", "<f8"), ("done", "<i4"),
                     ("converged", "<i4"), ("breakdown", "<i4"), ("bkind", "<i4"), ("iterations", "<i4"),
                     ("max_iters", "<i4"), ("pad", "<i4", 2)])


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
def _site_slice(lo, hi):
    return slice(lo * nat.MAX_SUMS, (hi + 1) * nat.MAX_SUMS)


class LoopbackComm:
    """Every band in this process; collectives are device copies in rank order."""

    def __init__(self, world: int):
        self.world = world

    def allreduce(self, bands, lo, hi):
        if len(bands) == 1:  # one band: its totals are the grid's
            return
        sl = _site_slice(lo, hi)
        tot = bands[0].totals[sl].clone()
        for b in bands[1:]:
            tot += b.totals[sl]
        for b in bands:
            b.totals[sl].copy_(tot)

    def transpose(self, bands):
        for b in bands:
            src = b.spec_send.view(b.nq, b.rows, b.mb)
            for q, d in enumerate(bands):
                d.spec_col.view(d.n, d.mb)[b.row0:b.row0 + b.rows].copy_(src[q])

    def transpose_back(self, bands):
        for b in bands:
            dst = b.spec_send.view(b.nq, b.rows, b.mb)
            for q, s in enumerate(bands):
                dst[q].copy_(s.spec_col.view(s.n, s.mb)[b.row0:b.row0 + b.rows])

    def halo(self, bands, items):
        """items: (getter(band) -> (k, rows + 2, ld) tensor, plane, 'down'|'up'|'both')."""
        for get, plane, way in items:
            for r, b in enumerate(bands):
                t = get(b)
                if way in ("down", "both") and r + 1 < len(bands):
                    get(bands[r + 1])[plane, 0].copy_(t[plane, b.rows])
                if way in ("up", "both") and r > 0:
                    a = bands[r - 1]
                    get(a)[plane, a.rows + 1].copy_(t[plane, 1])


class DistComm:
    """One band per process over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def _peer(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def allreduce(self, bands, lo, hi):
        (b,) = bands
        self.dist.all_reduce(b.totals[_site_slice(lo, hi)], group=self.group)

    def _splits(self, b):
        lay = b.layout
        mine = [b.rows * b.mb] * self.world
        theirs = [lay.rows[p] * b.mb for p in range(self.world)]
        return mine, theirs

    def transpose(self, bands):
        (b,) = bands
        mine, theirs = self._splits(b)
        self.dist.all_to_all_single(b.spec_col, b.spec_send, output_split_sizes=theirs, input_split_sizes=mine,
                                    group=self.group)

    def transpose_back(self, bands):
        (b,) = bands
        mine, theirs = self._splits(b)
        self.dist.all_to_all_single(b.spec_send, b.spec_col, output_split_sizes=mine, input_split_sizes=theirs,
                                    group=self.group)

    def halo(self, bands, items):
        torch = _torch()
        (b,) = bands
        r, world = self.rank, self.world
        down = [(get, pl) for get, pl, way in items if way in ("down", "both")]
        up = [(get, pl) for get, pl, way in items if way in ("up", "both")]
        ops, recv_above, recv_below = [], None, None
        P2P = self.dist.P2POp
        if down and r + 1 < world:
            send = torch.stack([get(b)[pl, b.rows] for get, pl in down])
            ops.append(P2P(self.dist.isend, send, self._peer(r + 1), self.group))
        if up and r > 0:
            send_up = torch.stack([get(b)[pl, 1] for get, pl in up])
            ops.append(P2P(self.dist.isend, send_up, self._peer(r - 1), self.group))
        if down and r > 0:
            recv_above = torch.empty((len(down), b.ld), dtype=b.tdtype, device=b.device)
            ops.append(P2P(self.dist.irecv, recv_above, self._peer(r - 1), self.group))
        if up and r + 1 < world:
            recv_below = torch.empty((len(up), b.ld), dtype=b.tdtype, device=b.device)
            ops.append(P2P(self.dist.irecv, recv_below, self._peer(r + 1), self.group))
        if ops:
            for req in self.dist.batch_isend_irecv(ops):
                req.wait()
        if recv_above is not None:
            for k, (get, pl) in enumerate(down):
                get(b)[pl, 0].copy_(recv_above[k])
        if recv_below is not None:
            for k, (get, pl) in enumerate(up):
                get(b)[pl, b.rows + 1].copy_(recv_below[k])


# ---------------------------------------------------------------------------
# the sharded unwrap
# ---------------------------------------------------------------------------
def _mask(*sites):
    m = 0
    for s in sites:
        m |= 1 << s
    return ctypes.c_uint(m)


class BandUnwrap:
    """irls.py:132-224 on row bands.  `bands`: the bands this process drives
    (all of them with LoopbackComm, its own with DistComm)."""

    def __init__(self, bands, comm, graphs=None):
        import os
        self.bands, self.comm = bands, comm
        # captured CUDA graphs replay the outer iteration (kernels, loopback
        # copies, NCCL all-reduces and halo sends/receives).  Under
        # torch.distributed only with the fused peer transpose: capturing the
        # NCCL all-to-all of the other mode hung the world-1 torchrun test on
        # the B200 (tests/test_gpu_dist1.py, peer 0), so that mode launches
        # eagerly.  PU_BAND_GRAPHS=0 / 1 forces either.
        if graphs is None:
            env = os.environ.get("PU_BAND_GRAPHS")
            if env is not None:
                graphs = env != "0" and (isinstance(comm, LoopbackComm)
                                         or comm.dist.get_backend(comm.group) == "nccl")
            elif isinstance(comm, LoopbackComm):
                graphs = True
            else:
                graphs = comm.dist.get_backend(comm.group) == "nccl" and all(b.peer for b in bands)
        self.graphs = bool(graphs)
        self._graphs = {}
        # acceptance fused with the next start-up (pu_accept_weights_start), as
        # irls._fuse_start decides for whole grids: bands of >= 2048² cells
        from .irls import FUSED_START, FUSED_START_MIN_CELLS
        b0 = bands[0]
        self.fuse = FUSED_START == "1" or (FUSED_START != "0" and b0.rows * b0.m >= FUSED_START_MIN_CELLS)
        self.prestarted = False  # the last tail ran the start-up of the next iteration
        self._warm = isinstance(comm, LoopbackComm)  # nothing to initialise lazily
        self.replayed_kernels = 0  # library kernels run by graph replays (the capture counted the first)

    # ---- helpers ------------------------------------------------------------
    def _each(self, name, fn):
        for b in self.bands:
            b.call(name, *fn(b))

    def _reduce(self, lo, hi, mask, mode, it, out_slot=None, rel_tol=0.0, max_iters=0):
        self.comm.allreduce(self.bands, lo, hi)
        for b in self.bands:
            b.call("pu_finalize", mask, mode, it, _ptr(b.ctrl), _ptr(b.norms),
                   b.sp(out_slot) if out_slot is not None else ctypes.c_void_p(0), float(rel_tol), int(max_iters),
                   b.stream())

    @staticmethod
    def _c(b):
        return (None, None) if not b.use_w else (BandState.p(b.W, 0), BandState.p(b.W, 1))

    def _state_halo(self, idx_fn, with_dv=False):
        items = [(lambda b, f=idx_fn: f(b), 0, "both"), (lambda b, f=idx_fn: f(b), 1, "down")]
        if with_dv:
            items.append((lambda b: b.D, 0, "down"))
        self.comm.halo(self.bands, items)

    # ---- set-up ---------------------------------------------------------------
    def load(self, x_rows, c: WeightField | None, lo):
        """x_rows[i]: fp64 device grid rows [row0, row0 + rows (+1 if not last)) of band i."""
        P = BandState.p
        self._keep = []
        self.prestarted = False
        for b, xr in zip(self.bands, x_rows):
            b.use_w = c is not None
            if c is not None:
                if b.W is None:  # kept across unwraps: captured graphs hold its address
                    b.W = _torch().zeros((2, b.rows + 2, b.ld), dtype=b.tdtype, device=b.device)
                nv = max(0, min(b.rows, b.n - 1 - b.row0))
                self._keep += [b.pack_rows(c.cv, b.W, 0, b.row0, nv), b.pack_rows(c.ch, b.W, 1, b.row0, b.rows)]
            self._keep.append(xr)
            b.call("pu_wrapped_gradients", _ptr(xr), int(xr.shape[1]), P(b.G, 0), P(b.G, 1), float(lo), b.stream())
        self.comm.halo(self.bands, [(lambda b: b.G, 0, "down")])  # gv[-1]: rhs (formed in pu_pcg_begin) and candidate stencils
        for b in self.bands:
            b.call("pu_init_state", P(b.G, 0), P(b.G, 1), P(b.S[0]), b.stream())
            b.cur = 0
        self._state_halo(lambda b: b.S[0])
        for b in self.bands:
            cv, ch = self._c(b)
            b.call("pu_weights_hpair", P(b.S[0]), cv, ch, P(b.G, 0), P(b.G, 1), None, None, P(b.Wt[0], 0),
                   P(b.Wt[0], 1), P(b.D, 0), P(b.D, 1), b.sp(b.S_HOLD), b.stream())
        self._reduce(nat.SITE_WH, nat.SITE_WH, _mask(nat.SITE_WH), 0, -1, out_slot=BandState.S_HOLD)
        self.comm.halo(self.bands, [(lambda b: b.D, 0, "down")])

    # ---- one outer iteration ------------------------------------------------------
    GRAPH_CHUNK = 64  # PCG iterations per captured graph

    def _base(self, k, lip, tol):
        return (k & 1, self.bands[0].cur, float(lip), float(tol), tuple(b.norms.data_ptr() for b in self.bands),
                tuple(b.W.data_ptr() if b.use_w else 0 for b in self.bands))

    PLACEHOLDER_ITERS = 1 << 30  # budget of the speculative set-up until pu_set_max_iters

    def begin(self, k, params: IrlsParams, lip):
        """The budget-free half of iteration k, pcg.py:59-79: the start-up
        (r0 = b - A x with the candidate step, objective.py:103-125; unless the
        previous tail's fused acceptance ran it), the all-reduce of its sums,
        their finalisation with a placeholder budget, z0 = M r0 and p0 = z0.
        run_loop enqueues it speculatively behind the previous iteration,
        before the host has read that iteration's scalars and applied the
        budget rule (step() then sets the budget on the device); it leaves the
        state untouched, so a "stop" decision just discards it."""
        pre, self.prestarted = self.prestarted, False
        tol = float(params.cg_rel_tol)
        self._run(("begin", pre) + self._base(k, lip, tol), lambda: self._begin(k, lip, tol, pre))

    def _begin(self, k, lip, tol, pre):
        P = BandState.p
        cur = lambda b: b.S[b.cur]  # noqa: E731
        if not pre:
            for b in self.bands:
                cv, ch = self._c(b)
                w = b.Wt[k & 1]
                b.call("pu_pcg_begin", None, P(cur(b)), P(cur(b)), P(b.D, 0), P(b.D, 1), P(b.R), _ptr(b.ctrl),
                       _ptr(b.norms), 0, 0.0, P(b.G, 0), P(b.G, 1), cv, ch, P(w, 0), P(w, 1), float(lip),
                       P(b.Cs[k & 1]), b.stream())
            self.comm.allreduce(self.bands, nat.SITE_START, nat.SITE_START)
        for b in self.bands:  # the exits on ||r0|| (the budget is set by step())
            b.call("pu_finalize", _mask(nat.SITE_START), 1, -1, _ptr(b.ctrl), _ptr(b.norms), ctypes.c_void_p(0), tol,
                   self.PLACEHOLDER_ITERS, b.stream())
        for b in self.bands:
            b.call("pu_pcg_residual_rows", None, P(b.D, 0), P(b.D, 1), P(cur(b)), P(b.R), _ptr(b.ctrl),
                   _ptr(b.norms), b.send(), -1, 0, b.stream())
        self._precond_tail(-1, mode=1)
        for b in self.bands:
            b.call("pu_pcg_rows_inv", b.send(), P(b.P[0]), P(b.P[1]), 1, _ptr(b.ctrl), -1, b.stream())
        self._dir_halo(0)

    def step(self, k, m_cg, params: IrlsParams, lip, poll=16):
        """irls.py:191-215 for iteration k, after begin(k).

        With graphs (the default): the budget and the first 64 PCG iterations
        replay as one captured CUDA graph (kernels and collectives alike),
        every further 64 iterations as another, and the H pair + acceptance
        as a third; the host checks the device exit flag once per 64-iteration
        chunk and only when the budget is longer than that.  Without graphs
        the host polls every `poll` iterations."""
        base = self._base(k, lip, params.cg_rel_tol)
        replay = self.graphs and self._warm
        chunk = self.GRAPH_CHUNK if replay else (poll or m_cg)
        first = min(m_cg, chunk)

        def head():
            for b in self.bands:
                b.call("pu_set_max_iters", _ptr(b.ctrl), int(m_cg), b.stream())
            self._iters(0, first)

        self._run(("head", m_cg, first) + base, head)
        # lagged exit polls: before enqueuing a chunk, read the exit flag left
        # by the chunk before the previous one, so the GPU always has a chunk
        # queued while the host waits (at most one chunk runs past the exit,
        # its kernels returning at once)
        it, flags = first, [self._post_flag()] if first < m_cg else []
        while it < m_cg:
            if len(flags) >= 2 and self._flag_done(flags.pop(0)):
                break
            nxt = min(m_cg, it + chunk)
            self._run(("iters", it, nxt) + base, lambda a=it, z=nxt: self._iters(a, z))
            it = nxt
            if it < m_cg:
                flags.append(self._post_flag())
        fuse = self.fuse and k + 1 < params.max_outer_iters
        self._run(("tail", fuse) + base, lambda: self._tail(k, lip if fuse else None), flips=True)
        self.prestarted = fuse
        # the first outer iteration runs eagerly: NCCL creates its
        # communicators (all-reduce, all-to-all, P2P halo) lazily on first
        # use, which cannot happen inside a stream capture
        self._warm = True

    def _run(self, key, fn, flips=False):
        if not (self.graphs and self._warm):
            fn()  # (eagerly, `fn` flips the states itself)
            return
        self._replay(key, fn, flips)

    def _replay(self, key, fn, flips=False):
        torch = _torch()
        entry = self._graphs.get(key)
        if entry is None:
            cur = [b.cur for b in self.bands]
            lib = self.bands[0].lib
            n0 = lib.pu_launch_count()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=torch.cuda.Stream(device=self.bands[0].device)):
                fn()
            for b, c in zip(self.bands, cur):  # capture does not run the work
                b.cur = c
            entry = self._graphs[key] = (g, lib.pu_launch_count() - n0)
        else:
            self.replayed_kernels += entry[1]
        entry[0].replay()
        if flips:
            for b in self.bands:
                b.cur = 1 - b.cur

    def _iters(self, it0, it1):
        """pcg.py:81-108 for iterations [it0, it1) (kernels return at once
        after the device-side exit)."""
        P = BandState.p
        cur = lambda b: b.S[b.cur]  # noqa: E731
        for it in range(it0, it1):
            for b in self.bands:
                pn, po = b.P[it & 1], b.P[(it + 1) & 1]
                b.call("pu_pcg_direction", P(b.R), P(po), P(pn), P(b.D, 0), P(b.D, 1), _ptr(b.ctrl), it,
                       b.stream())
            self._reduce(nat.SITE_K1, nat.SITE_K1, _mask(nat.SITE_K1), 2, it)
            submean = (it + 1) % 50 == 0
            if submean:  # pcg.py:92-93
                for b in self.bands:
                    b.call("pu_pcg_update_sum", P(b.P[it & 1]), P(b.D, 0), P(b.D, 1), P(cur(b)), P(b.R),
                           _ptr(b.ctrl), it, b.stream())
                self._reduce(nat.SITE_UPD, nat.SITE_UPD, _mask(nat.SITE_UPD), 2, it)
            for b in self.bands:
                b.call("pu_pcg_residual_rows", P(b.P[it & 1]), P(b.D, 0), P(b.D, 1), P(cur(b)), P(b.R),
                       _ptr(b.ctrl), _ptr(b.norms), b.send(), it, 1 if submean else 0, b.stream())
            self._precond_tail(it, mode=2)
            for b in self.bands:
                b.call("pu_pcg_rows_inv", b.send(), P(b.P[(it + 1) & 1]), P(b.P[it & 1]), 0,
                       _ptr(b.ctrl), it, b.stream())
            self._dir_halo((it + 1) & 1)

    def _tail(self, k, lip=None):
        """H pair (irls.py:202-205) on the proposal (= state, solved in place)
        and the candidate, then the acceptance and the weights of k + 1; with
        `lip`, fused with the start-up of k + 1 (pu_accept_weights_start: its
        candidate into Cs[(k + 1) & 1], r0, the start-up sums into the S_START
        totals), so begin(k + 1) has nothing left to do."""
        P = BandState.p
        cur = lambda b: b.S[b.cur]  # noqa: E731
        nxt = lambda b: b.S[1 - b.cur]  # noqa: E731
        cand = lambda b: b.Cs[k & 1]  # noqa: E731
        if lip is None:
            self.comm.halo(self.bands, [(cur, 0, "up"), (cand, 0, "up")])
        else:  # the fused start-up's stencil reads the accepted state's rows -1 and `rows`
            self.comm.halo(self.bands, [(cur, 0, "both"), (cur, 1, "down"), (cand, 0, "both"), (cand, 1, "down")])
        for b in self.bands:
            cv, ch = self._c(b)
            w = b.Wt[k & 1]
            b.call("pu_hpair_states", P(cur(b)), P(cand(b)), P(w, 0), P(w, 1), P(b.G, 0), P(b.G, 1), cv, ch,
                   b.sp(b.S_HPROP), b.stream())
        self._reduce(nat.SITE_HPAIR, nat.SITE_HPAIR, _mask(nat.SITE_HPAIR), 0, -1, out_slot=BandState.S_HPROP)
        for b in self.bands:
            cv, ch = self._c(b)
            w, wn = b.Wt[k & 1], b.Wt[(k + 1) & 1]
            args = (P(cur(b)), P(cand(b)), b.sp(b.S_MEAN), P(nxt(b)), P(b.G, 0), P(b.G, 1), cv, ch, P(w, 0), P(w, 1),
                    P(wn, 0), P(wn, 1), P(b.D, 0), P(b.D, 1), b.sp(b.S_HACC))
            if lip is None:
                b.call("pu_accept_weights", *args, b.stream())
            else:
                b.call("pu_accept_weights_start", *args, float(lip), P(b.R), P(b.Cs[(k + 1) & 1]), b.stream())
        if lip is None:
            self._reduce(nat.SITE_ACC, nat.SITE_ACC, _mask(nat.SITE_ACC), 0, -1, out_slot=BandState.S_HACC)
        else:  # S_ACC..S_START: the H pair and the start-up sums (finalised by the next head)
            self._reduce(nat.SITE_ACC, nat.SITE_START, _mask(nat.SITE_ACC), 0, -1, out_slot=BandState.S_HACC)
        for b in self.bands:
            b.cur = 1 - b.cur
        self._state_halo(lambda b: b.S[b.cur], with_dv=True)

    def _precond_tail(self, it, mode):
        if self.bands[0].peer:
            # fused transpose: the row DCT-II stored straight into the column
            # blocks; the all-reduces order the kernels across ranks (each
            # completes only once every rank has reached it)
            self.comm.allreduce(self.bands, nat.SITE_K2, nat.SITE_K2)
            for b in self.bands:
                b.call("pu_pcg_columns", b.col(), _ptr(b.ctrl), it, b.stream())
            self.comm.allreduce(self.bands, nat.SITE_K3, nat.SITE_K3)
            mask = _mask(nat.SITE_K3) if it < 0 else _mask(nat.SITE_K2, nat.SITE_K3)
            for b in self.bands:
                b.call("pu_finalize", mask, mode, it, _ptr(b.ctrl), _ptr(b.norms), ctypes.c_void_p(0), 0.0, 0,
                       b.stream())
            return
        self.comm.transpose(self.bands)
        for b in self.bands:
            b.call("pu_pcg_columns", b.col(), _ptr(b.ctrl), it, b.stream())
        self.comm.transpose_back(self.bands)
        if it < 0:  # set-up: rho_s of r0 was finalised with the start-up sums
            self._reduce(nat.SITE_K3, nat.SITE_K3, _mask(nat.SITE_K3), mode, it)
        else:
            self._reduce(nat.SITE_K2, nat.SITE_K3, _mask(nat.SITE_K2, nat.SITE_K3), mode, it)

    def _dir_halo(self, idx):
        self.comm.halo(self.bands, [(lambda b, i=idx: b.P[i], 0, "both"), (lambda b: b.R, 1, "down")])

    _DONE_OFFSET = 72  # byte offset of `done` in the control block (_ctrl_dtype)

    def _post_flag(self):
        """Asynchronous copy of band 0's exit flag (ctrl->done) to page-locked
        memory, with an event behind it."""
        torch = _torch()
        b = self.bands[0]
        ring = getattr(self, "_flag_ring", None)
        if ring is None:
            ring = self._flag_ring = [(torch.zeros(4, dtype=torch.uint8, pin_memory=True), torch.cuda.Event())
                                      for _ in range(4)]
            self._flag_next = 0
        host, ev = ring[self._flag_next]
        self._flag_next = (self._flag_next + 1) % len(ring)
        host.copy_(b.ctrl[self._DONE_OFFSET:self._DONE_OFFSET + 4], non_blocking=True)
        ev.record(torch.cuda.current_stream(b.device))
        return host, ev

    @staticmethod
    def _flag_done(flag):
        host, ev = flag
        ev.synchronize()
        return bool(host.numpy().view(np.int32)[0])

    # ---- results ---------------------------------------------------------------
    def band_arrays(self, b):
        """(u, vv, vh) fp64 device tensors of band b's own rows (vv without the global pad row)."""
        torch = _torch()
        s = b.S[b.cur]
        nv = max(0, min(b.rows, b.n - 1 - b.row0))
        u = s[0, 1:b.rows + 1, :b.m].to(torch.float64)
        vv = s[1, 1:nv + 1, :b.m].to(torch.float64)
        vh = s[2, 1:b.rows + 1, :b.m - 1].to(torch.float64)
        return u, vv, vh


def run_loop(driver: BandUnwrap, c, model: ModelParams, params: IrlsParams):
    """The host loop of irls.py:172-222 (same as irls._unwrap_loop) over the
    band driver: one host synchronisation per outer iteration (the scalar
    snapshot), with the next iteration's start-up already enqueued behind it."""
    from .irls import _record
    cmax = 1.0 if c is None else c.max_weight
    lip = 12.0 / model.tau + cmax ** 2 / model.delta
    trace = IrlsTrace()
    m_history = [params.max_iter_cg_start]
    pending = None
    b0 = driver.bands[0]
    for b in driver.bands:  # one allocation: the captured graphs hold its address
        b.ensure_norms(max(params.max_cg_iters_cap, driver.GRAPH_CHUNK))
    if params.max_outer_iters > 0:
        driver.begin(0, params, lip)
    for k in range(params.max_outer_iters):
        delta_rel = None
        if k >= 1:
            scal, ctrl = b0.read_snapshot()
            trace.append(_record(*pending, scal, ctrl, b0))
            pending = None
            h_old, h_new = float(scal[b0.S_HACC]), float(scal[b0.S_HNEXT])
            delta_rel = 0.0 if h_old == 0 else relative_improvement(h_old, h_new)
            m_prev = m_history[k - 1]
            m_prev2 = m_history[k - 2] if k >= 2 else m_prev
            decision = cg_budget_update(delta_rel, m_prev, m_prev2, params)
            if decision.action == "stop":
                break
            m_cg = decision.m_cg
            m_history.append(m_cg)
        else:
            m_cg = m_history[0]
        driver.step(k, m_cg, params, lip)
        b0.snapshot()
        if k + 1 < params.max_outer_iters:
            driver.begin(k + 1, params, lip)  # speculative: overlaps the host's budget decision
        pending = (k, m_cg, delta_rel)
    if pending is not None:
        scal, ctrl = b0.read_snapshot()
        trace.append(_record(*pending, scal, ctrl, b0))
    return trace


def _check_inputs(x, c, n, m, gradient_lo):
    if c is not None and (c.cv.shape != (n - 1, m) or c.ch.shape != (n, m - 1)):
        raise ValueError(f"weight shapes {c.cv.shape}/{c.ch.shape} do not match grid {(n, m)}")
    if gradient_lo not in (0.0, 0, -np.pi):
        raise ValueError(f"lo must be 0 or -pi, got {gradient_lo!r}")


def _validate_device(x_dev):
    torch = _torch()
    chk = torch.stack([x_dev.min(), x_dev.max(), torch.isfinite(x_dev).all().to(torch.float64)]).cpu()
    if chk[2] != 1.0:
        raise ValueError("phase grid contains non-finite values")
    if float(chk[0]) < 0.0 or float(chk[1]) >= 2.0 * np.pi:
        raise ValueError("wrapped phase values must lie in [0, 2*pi)")


def _default_peer(distributed, group):
    """The fused peer transpose unless PU_BAND_P2P=0: always for bands in one
    process (same device, no mapping), and under torch.distributed when the
    backend is NCCL and every rank's GPU is on this node with peer access to
    the others (NVSwitch); otherwise the all-to-all transposes."""
    import os
    env = os.environ.get("PU_BAND_P2P")
    if env is not None:
        return env == "1"
    if not distributed:
        return True
    import torch.distributed as dist
    torch = _torch()
    world = dist.get_world_size(group)
    if dist.get_backend(group) != "nccl" or world > torch.cuda.device_count():
        return False
    if world == 1:
        return True
    cnt = torch.cuda.device_count()
    ok = all(torch.cuda.can_device_access_peer(a, b) for a in range(cnt) for b in range(cnt) if a != b)
    flag = torch.tensor([1 if ok else 0], device=torch.device("cuda", torch.cuda.current_device()))
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    return bool(flag.item())


class RowSharded:
    """Band states, communicator and driver for one (N, M, dtype, tau, delta)
    on this process's device; reused across unwraps (see `get`)."""

    _cache: dict = {}

    @classmethod
    def get(cls, n, m, dtype, model: ModelParams, device, bands=None, group=None, peer=None):
        import os
        import torch.distributed as dist
        distributed = bands is None and dist.is_available() and dist.is_initialized()
        if peer is None:
            peer = _default_peer(distributed, group)
        key = (n, m, dtype, float(model.tau), float(model.delta), str(device), bands, id(group) if distributed else None,
               distributed, bool(peer))
        obj = cls._cache.get(key)
        if obj is None:
            obj = cls(n, m, dtype, model, device, bands, group, peer)
            cls._cache[key] = obj
        return obj

    def __init__(self, n, m, dtype, model: ModelParams, device, bands=None, group=None, peer=False):
        """peer: fuse the DCT transpose into the row kernels (stores into /
        loads from every rank's column block: same GPU in loopback, peer GPUs
        over NVLink via CUDA IPC under torch.distributed) instead of two
        all-to-alls per PCG iteration."""
        import torch.distributed as dist
        torch = _torch()
        nat.ensure()
        self.distributed = bands is None and dist.is_available() and dist.is_initialized()
        self.group = group
        world = dist.get_world_size(group) if self.distributed else int(bands or 1)
        self.layout = BandLayout(n, m, world)
        if self.distributed:
            self.comm, self.ranks = DistComm(group), [dist.get_rank(group)]
        else:
            self.comm, self.ranks = LoopbackComm(world), list(range(world))
        self.device = torch.device(device)
        self.model = model
        with torch.cuda.device(self.device):
            self.bands = [BandState(self.layout, r, dtype, model.tau, model.delta, self.device, peer)
                          for r in self.ranks]
            if peer:
                self._wire_peers()
            self.stream = torch.cuda.Stream(device=self.device)
        self.driver = BandUnwrap(self.bands, self.comm)
        self._pins = {}

    def _wire_peers(self):
        """Every band learns the column-block and back-buffer addresses of every rank."""
        if not self.distributed:
            cols, backs = [b.col_ptr for b in self.bands], [b.back_ptr for b in self.bands]
            for b in self.bands:
                b.set_peers(cols, backs)
            return
        import torch.distributed as dist
        (b,) = self.bands
        mine = []
        for ptr in (b.col_ptr, b.back_ptr):
            handle = ctypes.create_string_buffer(64)
            nat.check(b.lib.pu_ipc_handle(ctypes.c_void_p(ptr), handle))
            mine.append(bytes(handle.raw))
        handles = [None] * self.layout.world
        dist.all_gather_object(handles, mine, group=self.group)
        tables = ([], [])
        for q, hq in enumerate(handles):
            for t, (own, h) in enumerate(zip((b.col_ptr, b.back_ptr), hq)):
                if q == b.rank:
                    tables[t].append(own)
                    continue
                ptr = ctypes.c_void_p()
                nat.check(b.lib.pu_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(ptr)))
                b._opened.append(ptr.value)
                tables[t].append(ptr.value)
        b.set_peers(*tables)

    def rows_of(self, r):
        """Rows of x band r reads: its own and the first row of the band below."""
        lay = self.layout
        return lay.row0[r], min(lay.n, lay.row0[r] + lay.rows[r] + 1)

    def upload(self, x):
        """This process's rows of a full host (numpy / CPU tensor) or device grid -> device fp64 tensors."""
        torch = _torch()
        xs = []
        for r in self.ranks:
            lo, hi = self.rows_of(r)
            sl = torch.as_tensor(np.ascontiguousarray(x[lo:hi])) if isinstance(x, np.ndarray) else x[lo:hi]
            if sl.device.type == "cpu" and not sl.is_pinned():
                stage = self._pinned(("in", r), tuple(sl.shape), torch.float64)
                stage.copy_(sl)  # multi-threaded host copy into page-locked staging
                sl = stage
            xs.append(sl.to(device=self.device, dtype=torch.float64, non_blocking=True).contiguous())
        return xs

    def _pinned(self, key, shape, dtype):
        torch = _torch()
        t = self._pins.get(key)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != dtype:
            t = torch.empty(shape, dtype=dtype, pin_memory=True)
            self._pins[key] = t
        return t

    def download(self, tensors):
        """Device fp64 tensors -> fresh host numpy arrays through pinned staging."""
        torch = _torch()
        stream = torch.cuda.current_stream(self.device)
        pins = []
        for i, t in enumerate(tensors):
            p = self._pinned(("out", i), tuple(t.shape), t.dtype)
            p.copy_(t, non_blocking=True)
            pins.append(p)
        stream.synchronize()
        out = []
        for p in pins:
            a = np.empty(tuple(p.shape), dtype=np.float64)
            if a.size:
                torch.from_numpy(a).copy_(p)
            out.append(a)
        return out

    def run(self, xs, c, params: IrlsParams, gradient_lo):
        """The full IRLS loop on the uploaded rows; returns the trace (results stay on the device)."""
        torch = _torch()
        s = self.stream
        s.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(s):
            self.driver.load(xs, c, gradient_lo)
            trace = run_loop(self.driver, c, self.model, params)
        torch.cuda.current_stream(self.device).wait_stream(s)
        return trace

    def band_parts(self):
        return [self.driver.band_arrays(b) for b in self.bands]


def unwrap_rows(x, c: WeightField | None = None, model: ModelParams | None = None, params: IrlsParams | None = None,
                gradient_lo=-np.pi, *, dtype="fp64", bands=None, group=None, gather=True, device=None,
                peer=None):
    """irls.py:132-224 on a row-sharded grid.

    Inside a torch.distributed job (and `bands` None) every rank passes the same
    full grid `x` (host array, or a tensor) and solves its own row band; only
    that band's rows (+1) are copied to its GPU.  The ranks exchange halos,
    reduction totals and the DCT transpose over `group` (default: world).
    Otherwise `bands` = B runs all B bands in this process on one device
    (loopback collectives) — the same decomposition, for testing.
    `peer` fuses the DCT transpose into the row kernels (stores into / loads
    from the other ranks' column blocks, pu_set_band_peers) instead of two
    all-to-alls per PCG iteration; default `_default_peer` (on, unless
    PU_BAND_P2P=0 or the ranks' GPUs lack peer access).
    Returns an UnwrapResult with the full grid on every rank when `gather`,
    else the rank's own band rows (u, vv, vh) and the trace.
    """
    nat.ensure()
    torch = _torch()
    model = model or ModelParams()
    params = params or IrlsParams()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    arr = np.asarray(x, dtype=np.float64) if not isinstance(x, torch.Tensor) else x
    if arr.ndim != 2 or arr.shape[0] < 1 or arr.shape[1] < 1:
        raise ValueError(f"phase grid must be 2-D and non-empty, got shape {tuple(arr.shape)}")
    n, m = int(arr.shape[0]), int(arr.shape[1])
    _check_inputs(arr, c, n, m, gradient_lo)
    with torch.cuda.device(dev):
        solver = RowSharded.get(n, m, dtype, model, dev, bands, group, peer)
        xs = solver.upload(arr)
        for xr in xs:
            _validate_device(xr)
        trace = solver.run(xs, c, params, gradient_lo)
        parts = solver.band_parts()
        if solver.distributed and gather:
            parts = _gather_bands(parts[0], solver.layout, group)
        if gather or not solver.distributed:
            u, vv, vh = solver.download([torch.cat([p[i] for p in parts]) for i in range(3)])
        else:
            u, vv, vh = solver.download([t.contiguous() for t in parts[0]])
    return UnwrapResult(u=u, vv=vv, vh=vh, trace=trace)


def _gather_bands(part, lay, group):
    """all-gather of every rank's (u, vv, vh) band rows (padded to the largest band)."""
    import torch.distributed as dist
    torch = _torch()
    out = []
    rmax = max(lay.rows)
    for idx, t in enumerate(part):
        pad = torch.zeros((rmax, t.shape[1]), dtype=t.dtype, device=t.device)
        pad[:t.shape[0]] = t
        bufs = [torch.empty_like(pad) for _ in range(lay.world)]
        dist.all_gather(bufs, pad, group=group)
        rows = []
        for r in range(lay.world):
            nr = lay.rows[r] if idx != 1 else max(0, min(lay.rows[r], lay.n - 1 - lay.row0[r]))
            rows.append(bufs[r][:nr])
        out.append(rows)
    return [(out[0][r], out[1][r], out[2][r]) for r in range(lay.world)]

