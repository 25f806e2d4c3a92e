"""pu.unwrap end to end when the caller keeps the previous result alive (the bench's e2e loop)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2401_09961_b200 as pu
_, x = pu.config_scene("c3")
for dtype in ("fp64", "fp32"):
    res = None
    ts = []
    for i in range(6):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = [pu.unwrap(x, dtype=dtype)]
        ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    print(dtype, "keep-previous", ts)
    ts = []
    for i in range(4):
        res = None
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = [pu.unwrap(x, dtype=dtype)]
        ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    print(dtype, "drop-previous", ts)
