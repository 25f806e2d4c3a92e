"""Device workspace: one planned N x M grid and its HBM buffers.

Layout: every grid is a plane of shape (N, ld) with the row
pitch `ld` chosen by the library (multiple of 8 elements); a system vector
is a (3, N, ld) tensor [u | vv | vh].  Buffers are torch allocations (the
caching allocator is the memory manager); all arithmetic is done by
libpu_unwrap.so through the C ABI.
"""

from __future__ import annotations

import ctypes
import json
import threading
import weakref

import numpy as np

from . import _native as nat

_DTYPES = {"fp32": nat.PU_F32, "float32": nat.PU_F32, "fp64": nat.PU_F64, "float64": nat.PU_F64}


def _torch():
    import torch
    return torch


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


_tls = threading.local()
_claimed: set = set()
_claim_lock = threading.Lock()


class _SlotToken:
    __slots__ = ("idx", "__weakref__")


def _release_slot(idx):
    with _claim_lock:
        _claimed.discard(idx)


def thread_slot() -> int:
    """Index of the calling thread's workspace set.

    Independent unwrap calls are safe to run concurrently (reference
    SPEC.md:391, 453-454), so no two live threads may share a device handle
    (its buffers, scalar block, reduction tickets and graph cache).  Each
    thread claims the lowest free index on first use; the claim is released
    when the thread ends (its thread-local token is collected), so the next
    thread reuses the cached workspaces instead of allocating new ones."""
    tok = getattr(_tls, "token", None)
    if tok is None:
        with _claim_lock:
            idx = 0
            while idx in _claimed:
                idx += 1
            _claimed.add(idx)
        tok = _SlotToken()
        tok.idx = idx
        weakref.finalize(tok, _release_slot, idx)
        _tls.token = tok
    return tok.idx


class Workspace:
    """Handle + buffers for one (N, M, dtype, tau, delta); reused across calls
    of the same thread (thread_slot)."""

    _cache: dict = {}
    _lock = threading.Lock()

    # scalar slots (fp64) in the device scalar block
    (S_HOLD, S_HNEW, S_HPROP, S_HCAND, S_MEAN, S_TAKE, S_HACC, S_HNEXT, S_F, S_L1, S_DOT,
     S_EVH, S_CHK_NF, S_CHK_RANGE) = range(14)
    NSCAL = 16

    @classmethod
    def get(cls, n, m, dtype="fp64", tau=1e-2, delta=1e-6, device=None, slot=0):
        """Cached workspace of the calling thread; `slot` > 0 gives independent
        buffer sets for concurrent unwraps of the same size within one thread
        (irls.unwrap_many)."""
        torch = _torch()
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        key = (n, m, dtype, float(tau), float(delta), dev.index, thread_slot(), int(slot))
        with cls._lock:
            ws = cls._cache.get(key)
            if ws is None:
                ws = cls(n, m, dtype, tau, delta, dev)
                cls._cache[key] = ws
            return ws

    @classmethod
    def release_all(cls):
        """Drop every cached workspace (their HBM buffers and plans are freed once
        no unwrap result refers to them)."""
        with cls._lock:
            cls._cache.clear()

    def __init__(self, n, m, dtype="fp64", tau=1e-2, delta=1e-6, device=None):
        self.lib = nat.ensure()
        torch = _torch()
        if dtype not in _DTYPES:
            raise ValueError(f"dtype must be 'fp32' or 'fp64', got {dtype!r}")
        self.n, self.m, self.dtype = int(n), int(m), dtype
        self.code = _DTYPES[dtype]
        self.tdtype = torch.float32 if self.code == nat.PU_F32 else torch.float64
        self.device = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.tau, self.delta = float(tau), float(delta)
        h = ctypes.c_void_p()
        with torch.cuda.device(self.device):
            nat.check(self.lib.pu_create(ctypes.byref(h), self.n, self.m, self.code, self.tau, self.delta))
        self.h = h
        self.ld = int(self.lib.pu_pitch(h))
        self._bufs = {}
        ctrl_bytes = int(self.lib.pu_pcg_ctrl_bytes())
        # scalar block: NSCAL doubles followed by the PCG control struct
        self.block = torch.zeros(self.NSCAL * 8 + ctrl_bytes, dtype=torch.uint8, device=self.device)
        self.scal = self.block[: self.NSCAL * 8].view(torch.float64)
        self.ctrl = self.block[self.NSCAL * 8:]
        self.norms = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._ctrl_dtype = np.dtype([("rho", "<f8"), ("alpha", "<f8"), ("beta", "<f8"), ("thr", "<f8"),
                                     ("bnorm", "<f8"), ("pap", "<f8"), ("rn", "<f8"), ("mean_ru", "<f8"),
                                     ("rho_s", "<f8"), ("done", "<i4"), ("converged", "<i4"),
                                     ("breakdown", "<i4"), ("bkind", "<i4"), ("iterations", "<i4"),
                                     ("max_iters", "<i4"), ("pad", "<i4", 2)])
        assert self._ctrl_dtype.itemsize == ctrl_bytes

    def __del__(self):
        try:
            if getattr(self, "h", None) is not None and self.h.value:
                self.lib.pu_destroy(self.h)
        except Exception:
            pass

    # ---- plumbing -------------------------------------------------------
    def stream(self):
        return ctypes.c_void_p(_torch().cuda.current_stream(self.device).cuda_stream)

    def solve_stream(self):
        """Dedicated non-default stream for unwraps (graph capture needs one)."""
        s = self._bufs.get(("stream",))
        if s is None:
            s = _torch().cuda.Stream(device=self.device)
            self._bufs[("stream",)] = s
        return s

    def describe(self):
        buf = ctypes.create_string_buffer(1024)
        nat.check(self.lib.pu_describe(self.h, buf, 1024))
        return json.loads(buf.value.decode())

    def planes(self, k):
        """A fresh zeroed (k, N, ld) device tensor."""
        return _torch().zeros((k, self.n, self.ld), dtype=self.tdtype, device=self.device)

    def buf(self, name, k):
        t = self._bufs.get(name)
        if t is None:
            t = self.planes(k)
            self._bufs[name] = t
        return t

    def call(self, name, *args):
        nat.check(getattr(self.lib, name)(self.h, *args))

    # ---- host <-> device --------------------------------------------------
    def pack(self, arr, dst):
        """Compact host/device fp64 array (rows x cols) -> device plane dst."""
        torch = _torch()
        src = torch.as_tensor(np.ascontiguousarray(arr, dtype=np.float64)) if isinstance(arr, np.ndarray) else arr
        src = src.to(device=self.device, dtype=torch.float64).contiguous()
        rows, cols = (src.shape[0], src.shape[1]) if src.dim() == 2 else (0, 0)
        lds = cols if cols > 0 else 1
        self.call("pu_pack", _ptr(src) if src.numel() else ctypes.c_void_p(0), lds, rows, cols, _ptr(dst),
                  self.stream())
        return src  # keep alive until the stream has consumed it

    def unpack(self, src, rows, cols):
        """Device plane -> compact fp64 device tensor (rows x cols)."""
        torch = _torch()
        out = torch.empty((max(rows, 0), max(cols, 0)), dtype=torch.float64, device=self.device)
        if rows > 0 and cols > 0:
            self.call("pu_unpack", _ptr(src), rows, cols, _ptr(out), self.stream())
        return out

    def pinned(self, name, shape, tdtype):
        """Persistent page-locked host staging buffer (allocated once per workspace)."""
        torch = _torch()
        key = ("pin", name)
        t = self._bufs.get(key)
        if t is None or tuple(t.shape) != tuple(shape) or t.dtype != tdtype:
            t = torch.empty(shape, dtype=tdtype, pin_memory=True)
            self._bufs[key] = t
        return t

    UPLOAD_CHUNKS = 8

    def upload_grid(self, x):
        """Host (numpy / CPU tensor) fp64 grid -> device, through pinned
        staging in row chunks: the host copy of chunk i + 1 overlaps the
        H2D copy of chunk i."""
        torch = _torch()
        src = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)) if isinstance(x, np.ndarray) else x
        if src.is_pinned() or src.dim() != 2:
            return src.to(self.device, non_blocking=True)
        src = src.to(torch.float64).contiguous()
        stage = self.pinned("x_in", tuple(src.shape), torch.float64)
        ev = self._bufs.get(("ev", "x_in"))
        if ev is not None:
            ev.synchronize()  # the previous upload's copies out of the staging buffer are done
        dst = torch.empty(tuple(src.shape), dtype=torch.float64, device=self.device)
        rows = int(src.shape[0])
        step = max(1, -(-rows // self.UPLOAD_CHUNKS))
        for a in range(0, rows, step):
            b = min(rows, a + step)
            stage[a:b].copy_(src[a:b])  # multi-threaded host copy
            dst[a:b].copy_(stage[a:b], non_blocking=True)
        ev = self._bufs[("ev", "x_in")] = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        return dst

    def download_system(self, x, out=None):
        """Device system vector -> fresh host fp64 numpy (u, vv, vh).

        The compact blocks move in the handle's dtype through persistent
        pinned buffers (full link bandwidth; half the bytes in fp32 mode),
        then one multi-threaded host copy widens them into new fp64 arrays."""
        torch = _torch()
        n, m = self.n, self.m
        shapes = ((n, m), (n - 1, m), (n, m - 1))
        outs, events = [], []
        stream = torch.cuda.current_stream(self.device)
        for idx, (r, c) in enumerate(shapes):
            dev = torch.empty((max(r, 0), max(c, 0)), dtype=self.tdtype, device=self.device)
            if r > 0 and c > 0:
                self.call("pu_unpack_native", _ptr(x[idx]), r, c, _ptr(dev), self.stream())
            pin = self.pinned(f"out{idx}", (max(r, 0), max(c, 0)), self.tdtype)
            pin.copy_(dev, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(stream)
            outs.append((pin, dev))
            events.append(ev)
        res = []
        for idx, ((p, _), ev) in enumerate(zip(outs, events)):
            # widen each block on the host while the next one is still in flight;
            # numpy's allocator madvises huge pages for large arrays (few page
            # faults); torch's multi-threaded copy widens fp32 -> fp64 into it
            ev.synchronize()
            a = out[idx] if out is not None else np.empty(tuple(p.shape), dtype=np.float64)
            if a.size:
                torch.from_numpy(a).copy_(p)
            res.append(a)
        return tuple(res)

    def to_system(self, u, vv, vh, dst=None):
        dst = dst if dst is not None else self.planes(3)
        keep = [self.pack(u, dst[0]), self.pack(vv, dst[1]), self.pack(vh, dst[2])]
        return dst, keep

    def from_system(self, x):
        n, m = self.n, self.m
        return self.unpack(x[0], n, m), self.unpack(x[1], n - 1, m), self.unpack(x[2], n, m - 1)

    def snapshot(self):
        """Enqueue a copy of the scalar block into pinned memory (read later with
        read_snapshot, while the stream keeps going)."""
        torch = _torch()
        pin = self.pinned("block", tuple(self.block.shape), torch.uint8)
        pin.copy_(self.block, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(self.device))
        self._snap = ev

    def read_snapshot(self):
        """Wait for the last snapshot only: (scalars[NSCAL], ctrl record)."""
        self._snap.synchronize()
        host = self.pinned("block", tuple(self.block.shape), _torch().uint8).numpy()
        scal = host[: self.NSCAL * 8].view(np.float64).copy()
        ctrl = host[self.NSCAL * 8:].view(self._ctrl_dtype)[0].copy()
        return scal, ctrl

    def read_block(self):
        """Synchronising read of the scalar block: (scalars[NSCAL], ctrl record)."""
        host = self.block.cpu().numpy()
        scal = host[: self.NSCAL * 8].view(np.float64).copy()
        ctrl = host[self.NSCAL * 8:].view(self._ctrl_dtype)[0]
        return scal, ctrl

    def ensure_norms(self, max_iters):
        if self.norms.numel() < max_iters + 1:
            self.norms = _torch().zeros(max_iters + 1, dtype=torch_float64(), device=self.device)
        return self.norms

    # ---- instrumentation ---------------------------------------------------
    TIME_KINDS = ("pcg_start", "K1_p_Ap_pAp", "K2a_update_norms", "K3_coldct_spectral", "K4_row_idct",
                  "reproject_update", "weights_hpair", "candidate", "hpair_states", "accept_center",
                  "K2b_row_dct")

    def timing(self, on: bool):
        nat.check(self.lib.pu_timing_enable(self.h, 1 if on else 0))

    def read_timing(self, cap=1 << 16):
        """(kinds, its, ms) numpy arrays of the per-launch event timings recorded so far."""
        kinds = (ctypes.c_int * cap)()
        its = (ctypes.c_int * cap)()
        ms = (ctypes.c_float * cap)()
        cnt = int(self.lib.pu_timing_read(self.h, kinds, its, ms, cap))
        if cnt < 0:
            raise nat.NativeError("pu_timing_read failed")
        return (np.frombuffer(kinds, dtype=np.int32, count=cnt).copy(),
                np.frombuffer(its, dtype=np.int32, count=cnt).copy(),
                np.frombuffer(ms, dtype=np.float32, count=cnt).astype(np.float64))

    def sp(self, slot):
        """Device pointer to scalar slot `slot`."""
        return ctypes.c_void_p(self.scal.data_ptr() + 8 * slot)


def torch_float64():
    return _torch().float64
