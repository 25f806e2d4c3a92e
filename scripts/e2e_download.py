"""Time the pieces of Workspace.download_system (C3 fp32)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09961_b200 as pu
from paper_2401_09961_b200.irls import unwrap_device
from paper_2401_09961_b200.device import Workspace, _ptr

_, x = pu.config_scene("c3")
dev = torch.device("cuda", 0)
x_dev = torch.from_numpy(x).to(dev)
ws = Workspace.get(4096, 4096, "fp32", 1e-2, 1e-6, dev)
run, trace = unwrap_device(x_dev, None, pu.ModelParams(), pu.IrlsParams(), -np.pi, "fp32", ws)
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); ws.download_system(run.state); t1 = time.perf_counter()
    print("download_system ms", round((t1 - t0) * 1e3, 2))
n, m = 4096, 4096
shapes = ((n, m), (n - 1, m), (n, m - 1))
T = {}
torch.cuda.synchronize()
t = time.perf_counter()
devs = []
for idx, (r, c) in enumerate(shapes):
    d = torch.empty((r, c), dtype=torch.float32, device=dev)
    ws.call("pu_unpack_native", _ptr(run.state[idx]), r, c, _ptr(d), ws.stream())
    devs.append(d)
torch.cuda.synchronize(); T["unpack"] = time.perf_counter() - t
t = time.perf_counter()
pins = []
for idx, d in enumerate(devs):
    p = ws.pinned(f"out{idx}", tuple(d.shape), torch.float32)
    p.copy_(d, non_blocking=True)
    pins.append(p)
torch.cuda.synchronize(); T["d2h"] = time.perf_counter() - t
t = time.perf_counter()
outs = [np.empty(tuple(p.shape), dtype=np.float64) for p in pins]
T["alloc"] = time.perf_counter() - t
t = time.perf_counter()
for a, p in zip(outs, pins):
    torch.from_numpy(a).copy_(p)
T["widen"] = time.perf_counter() - t
t = time.perf_counter()
for a, p in zip(outs, pins):
    torch.from_numpy(a).copy_(p)
T["widen_again"] = time.perf_counter() - t
t = time.perf_counter()
for a, p in zip(outs, pins):
    np.copyto(a, p.numpy())
T["widen_numpy"] = time.perf_counter() - t
print({k: round(v * 1e3, 2) for k, v in T.items()}, "threads", torch.get_num_threads(), os.cpu_count())
