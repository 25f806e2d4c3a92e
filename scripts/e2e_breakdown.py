"""Where does unwrap()'s end-to-end time go beyond the device loop? (C3 fp32)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09961_b200 as pu
from paper_2401_09961_b200.irls import unwrap_device
from paper_2401_09961_b200.device import Workspace

_, x = pu.config_scene("c3")
x_pin = torch.from_numpy(x).pin_memory()
dev = torch.device("cuda", 0)
for _ in range(2):
    pu.unwrap(x_pin, dtype="fp32")
torch.cuda.synchronize()
T = {}
def tic(): torch.cuda.synchronize(); return time.perf_counter()
t0 = tic(); x_dev = x_pin.to(dev, non_blocking=True); t1 = tic(); T["h2d"] = t1 - t0
st = torch.stack([x_dev.min(), x_dev.max(), torch.isfinite(x_dev).all().to(torch.float64)]).cpu(); t2 = tic(); T["validate"] = t2 - t1
ws = Workspace.get(4096, 4096, "fp32", 1e-2, 1e-6, dev)
run, trace = unwrap_device(x_dev, None, pu.ModelParams(), pu.IrlsParams(), -np.pi, "fp32", ws); t3 = tic(); T["device_loop"] = t3 - t2
u, vv, vh = run.result_arrays(); t4 = tic(); T["unpack"] = t4 - t3
un = u.cpu().numpy(); t5 = tic(); T["d2h_u"] = t5 - t4
vvn = vv.cpu().numpy(); vhn = vh.cpu().numpy(); t6 = tic(); T["d2h_vv_vh"] = t6 - t5
t7 = tic(); r = pu.unwrap(x_pin, dtype="fp32"); t8 = tic(); T["unwrap_total"] = t8 - t7
t9 = tic(); r = pu.unwrap(x, dtype="fp32"); t10 = tic(); T["unwrap_total_numpy_in"] = t10 - t9
print({k: round(v * 1e3, 2) for k, v in T.items()})
