"""One unwrap of a BASELINE config (for ncu launch lists): python scripts/one_unwrap.py c1 fp64 [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2401_09961_b200 as pu  # noqa: E402
from paper_2401_09961_b200.irls import unwrap_device  # noqa: E402

cfg, dtype = sys.argv[1], sys.argv[2]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
_, x = pu.config_scene(cfg)
x_dev = torch.from_numpy(x).to("cuda")
for _ in range(reps):
    run, trace = unwrap_device(x_dev, None, pu.ModelParams(), pu.IrlsParams(), -np.pi, dtype)
torch.cuda.synchronize()
print(cfg, dtype, len(trace.records), "outer", sum(r.cg_iters for r in trace.records), "PCG")
