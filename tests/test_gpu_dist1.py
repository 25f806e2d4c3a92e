"""The torch.distributed (NCCL) row-sharded path under torchrun with one rank
on one GPU: exercises the NCCL all-reduce / all-to-all / peer-table plumbing
end to end (multi-rank exchanges are covered by the gloo tests and the
loopback bands)."""
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


@pytest.mark.parametrize("peer", ["0", "1"])
def test_nccl_rows_world1(tmp_path, peer):
    out = tmp_path / "r.json"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "helpers", "dist_rows.py"), str(out), peer]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-3000:]
    rep = json.loads(out.read_text())
    assert rep["world"] == 1 and rep["same_counts"] and rep["shapes_ok"]
    assert rep["u_rel"] <= 1e-12
