"""The torch.distributed (NCCL) row-sharded path under torchrun: one rank on
one GPU always (the NCCL all-reduce / all-to-all / peer-table plumbing end to
end), and 2 / 4 / 8 ranks when the box has that many GPUs (multi-rank
exchanges are otherwise covered by the gloo tests and the loopback bands)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("peer", ["0", "1"])
def test_nccl_rows(tmp_path, peer, world):
    """world 1 always; world 2/4/8 run when that many GPUs are visible (one
    rank per GPU; with the peer transpose the NCCL collectives are captured in
    the per-budget CUDA graphs)."""
    import torch
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs")
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world), "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "helpers", "dist_rows.py"), str(out), peer]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-3000:]
    rep = json.loads(out.read_text())
    assert rep["world"] == world and rep["same_counts"] and rep["shapes_ok"]
    assert rep["u_rel"] <= (1e-12 if world == 1 else 1e-9)
    # the fused peer transpose replays captured graphs (NCCL all-reduces and
    # halos inside); the all-to-all mode launches eagerly
    assert rep["graphs"] == (peer == "1")
    assert (rep["replayed"] > 0) == (peer == "1")
