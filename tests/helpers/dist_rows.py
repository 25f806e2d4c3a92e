"""torchrun helper for tests/test_gpu_dist1.py: the row-sharded unwrap through
torch.distributed (NCCL) in one rank, compared with the single-grid solve."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np
import torch
import torch.distributed as dist

import paper_2401_09961_b200 as pu

out_path, peer = sys.argv[1], sys.argv[2] == "1"
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
spec = pu.SceneSpec("gaussian-bumps", 96, 80, 10.0, 6.0, 5)
x = pu.add_phase_noise(pu.wrap_scene(pu.generate_scene(spec)), 0.7, 105)
single = pu.unwrap(x, dtype="fp64")
res = pu.unwrap_rows(x, dtype="fp64", peer=peer)
from paper_2401_09961_b200 import band  # noqa: E402
solver = band.RowSharded.get(96, 80, "fp64", pu.ModelParams(), torch.device("cuda", local), None, None, peer)
report = {
    "graphs": bool(solver.driver.graphs), "replayed": int(solver.driver.replayed_kernels),
    "world": dist.get_world_size(),
    "same_counts": [r.cg_iters for r in res.trace.records] == [r.cg_iters for r in single.trace.records],
    "u_rel": float(np.linalg.norm(res.u - single.u) / np.linalg.norm(single.u)),
    "shapes_ok": res.u.shape == single.u.shape and res.vv.shape == single.vv.shape,
}
if dist.get_rank() == 0:
    with open(out_path, "w") as fh:
        json.dump(report, fh)
dist.barrier()
dist.destroy_process_group()
