"""Two processes on ONE GPU (gloo for the host-side collectives) running the
row-sharded unwrap with the fused peer transpose: every band's column block
and back buffer is a cudaMalloc block mapped into the other process with CUDA
IPC (pu_ipc_handle / pu_ipc_open), and the row DCT-II / column transform store
into the other process's blocks -- the cross-process path of a multi-GPU box,
on the one GPU a gpurun call has.  No kernel waits on another process: every
cross-rank ordering point is a blocking host collective (the totals are
staged through host memory, which also synchronises the stream), so the two
processes' kernels only need to be time-sliced, not co-resident.

Used by tests/test_gpu_ipc2.py; run as
    python -m torch.distributed.run --nproc-per-node 2 ipc_rows.py OUT.json
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np
import torch
import torch.distributed as dist

import paper_2401_09961_b200 as pu
from paper_2401_09961_b200 import band


class HostStagedComm(band.DistComm):
    """DistComm whose collectives move through host memory (gloo on CPU
    tensors); the .cpu() copies synchronise this rank's stream first."""

    def allreduce(self, bands, lo, hi):
        (b,) = bands
        t = b.totals[band._site_slice(lo, hi)]
        h = t.cpu()
        self.dist.all_reduce(h, group=self.group)
        t.copy_(h)

    def transpose(self, bands):
        raise AssertionError("the peer transpose needs no all-to-all")

    transpose_back = transpose

    def halo(self, bands, items):
        (b,) = bands
        r, world = self.rank, self.world
        down = [(get, pl) for get, pl, way in items if way in ("down", "both")]
        up = [(get, pl) for get, pl, way in items if way in ("up", "both")]
        ops, recv_above, recv_below = [], None, None
        P2P = self.dist.P2POp
        if down and r + 1 < world:
            ops.append(P2P(self.dist.isend, torch.stack([get(b)[pl, b.rows] for get, pl in down]).cpu(),
                           self._peer(r + 1), self.group))
        if up and r > 0:
            ops.append(P2P(self.dist.isend, torch.stack([get(b)[pl, 1] for get, pl in up]).cpu(),
                           self._peer(r - 1), self.group))
        if down and r > 0:
            recv_above = torch.empty((len(down), b.ld), dtype=b.tdtype)
            ops.append(P2P(self.dist.irecv, recv_above, self._peer(r - 1), self.group))
        if up and r + 1 < world:
            recv_below = torch.empty((len(up), b.ld), dtype=b.tdtype)
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


band.DistComm = HostStagedComm

out_path = sys.argv[1]
n, m = (int(v) for v in sys.argv[2:4]) if len(sys.argv) > 3 else (96, 80)
torch.cuda.set_device(0)  # both ranks on the one GPU
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
spec = pu.SceneSpec("gaussian-bumps", n, m, 10.0, 6.0, 5)
x = pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(spec)), 0.7, 105)
res = pu.unwrap_rows(x, dtype="fp64", peer=True, gather=False)
solver = band.RowSharded.get(n, m, "fp64", pu.ModelParams(), torch.device("cuda", 0), None, None, True)
r0, rows = solver.layout.row0[rank], solver.layout.rows[rank]
report = {"rank": rank, "world": world, "peer": bool(solver.bands[0].peer), "opened": len(solver.bands[0]._opened),
          "cg_iters": [r.cg_iters for r in res.trace.records], "row0": r0, "rows": rows}
if rank == 0:
    single = pu.unwrap(x, dtype="fp64")
    report["single_cg_iters"] = [r.cg_iters for r in single.trace.records]
    np.save(out_path + ".single_u.npy", single.u)
np.save(out_path + f".u{rank}.npy", res.u)
with open(out_path + f".{rank}.json", "w") as fh:
    json.dump(report, fh)
dist.barrier()
dist.destroy_process_group()
