"""Split of pu.unwrap's end-to-end time (C3 fp64): host staging + H2D, device loop, D2H + widening."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09961_b200 as pu
from paper_2401_09961_b200.irls import unwrap_device
from paper_2401_09961_b200.device import Workspace
_, x = pu.config_scene("c3")
dtype = sys.argv[1] if len(sys.argv) > 1 else "fp64"
for _ in range(2):
    pu.unwrap(x, dtype=dtype)
ws = Workspace.get(4096, 4096, dtype, 1e-2, 1e-6, torch.device("cuda", 0))
T = {k: [] for k in ("stage_h2d", "solve", "download", "total")}
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    xd = ws.upload_grid(x); torch.cuda.synchronize(); t1 = time.perf_counter()
    run, tr = unwrap_device(xd, None, pu.ModelParams(), pu.IrlsParams(), -np.pi, dtype, ws); torch.cuda.synchronize(); t2 = time.perf_counter()
    out = run.ws.download_system(run.state); t3 = time.perf_counter()
    r = pu.unwrap(x, dtype=dtype); t4 = time.perf_counter()
    for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        T[k].append(v * 1e3)
print({k: round(min(v), 2) for k, v in T.items()})
