"""Print fp32/fp64 errors of the GPU sylvester solve vs the scipy DCT oracle over many shapes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2401_09961_b200 as pu
from oracle import phaseirls_port as port
rng = np.random.default_rng(0)
for n, m in [(2, 2), (4, 4), (16, 16), (32, 32), (48, 40), (40, 48), (64, 64), (17, 16), (16, 17), (256, 256),
             (512, 512), (3, 16), (16, 3), (48, 1), (1, 48), (1024, 8), (8, 1024), (4096, 8), (8, 4096), (37, 53)]:
    r = rng.standard_normal((n, m))
    want = port.DctPoisson(n, m)(r, 1e-2)
    out = []
    for dt in ("fp64", "fp32"):
        got = pu.sylvester_solve(r, 1e-2, dtype=dt)
        out.append(np.linalg.norm(got - want) / np.linalg.norm(want))
    print(f"{n:5d} x {m:5d}  fp64 {out[0]:.2e}  fp32 {out[1]:.2e}", flush=True)
