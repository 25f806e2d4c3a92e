import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09961_b200 as pu
from paper_2401_09961_b200.device import Workspace
print("torch threads", torch.get_num_threads(), "cpus", os.cpu_count())
_, x = pu.config_scene("c3")
x_pin = torch.from_numpy(x).pin_memory()
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = pu.unwrap(x_pin, dtype="fp32")
    t1 = time.perf_counter()
    print("unwrap e2e ms", round((t1 - t0) * 1e3, 1))
ws = Workspace.get(4096, 4096, "fp32", 1e-2, 1e-6, torch.device("cuda", 0))
st = ws.S if hasattr(ws, "S") else ws._bufs["state0"]
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    u, vv, vh = ws.download_system(ws._bufs["state0"])
    t1 = time.perf_counter()
    print("download ms", round((t1 - t0) * 1e3, 1))
