"""Device time of C3 unwraps with and without per-kernel timing, and host-side breakdown."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09961_b200 as pu
from paper_2401_09961_b200.irls import unwrap_device
from paper_2401_09961_b200.device import Workspace
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
dtype = sys.argv[2] if len(sys.argv) > 2 else "fp32"
_, x = pu.config_scene(cfg)
dev = torch.device("cuda", 0)
x_dev = torch.from_numpy(x).to(dev)
ws = Workspace.get(x.shape[0], x.shape[1], dtype, 1e-2, 1e-6, dev)
def run(n, timing, graphs=True):
    ws.timing(timing)
    ws.lib.pu_set_graphs(ws.h, 1 if graphs else 0)
    ws.read_timing()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(n):
        r, tr = unwrap_device(x_dev, None, pu.ModelParams(), pu.IrlsParams(), -np.pi, dtype, ws)
    e1.record(); torch.cuda.synchronize()
    t1 = time.perf_counter()
    k, it, ms = ws.read_timing()
    return e0.elapsed_time(e1) / n, (t1 - t0) * 1e3 / n, ms.sum() / n
for _ in range(3):
    run(1, False)
for t, g in ((False, True), (True, True), (False, False), (True, False)):
    d, w, ksum = run(3, t, g)
    print(f"timing={t} graphs={g}: device {d:.2f} ms  wall {w:.2f} ms  kernel-event sum {ksum:.2f} ms")
