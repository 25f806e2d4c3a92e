"""K2a event times split by x-update mode (defer / apply) on C3 fp32."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09961_b200 as pu
from paper_2401_09961_b200 import _native
from paper_2401_09961_b200.irls import unwrap_device
from paper_2401_09961_b200.device import Workspace

_, x = pu.config_scene("c3")
dev = torch.device("cuda", 0)
x_dev = torch.from_numpy(x).to(dev)
ws = Workspace.get(4096, 4096, "fp32", 1e-2, 1e-6, dev)
run, trace = unwrap_device(x_dev, None, pu.ModelParams(), pu.IrlsParams(), -np.pi, "fp32", ws)
_native.load().pu_set_graphs(ws.h, 0)
ws.timing(True); ws.read_timing()
run, trace = unwrap_device(x_dev, None, pu.ModelParams(), pu.IrlsParams(), -np.pi, "fp32", ws)
kinds, its, ms = ws.read_timing()
budgets = [r.m_cg for r in trace.records]
k2 = Workspace.TIME_KINDS.index("K2a_update_norms")
# walk the records: each outer iteration's K2a launches have it = 0..m-1 in order
sel = [(i, t) for k, i, t in zip(kinds, its, ms) if k == k2 and i >= 0]
pos, out = 0, {"defer": [], "apply2": [], "apply0": []}
for m in budgets:
    for it in range(m):
        i, t = sel[pos]; pos += 1
        assert i == it
        mode = "defer" if (m - 1 - it) & 1 else ("apply2" if it >= 1 else "apply0")
        if t > 0.05: out[mode].append(t)
print({k: (len(v), round(float(np.mean(v)), 4) if v else None) for k, v in out.items()})
