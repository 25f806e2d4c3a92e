"""The fused peer transpose across PROCESSES: two ranks on one GPU, their
column blocks and back buffers exchanged with CUDA IPC, the row / column DCT
kernels storing into the other process's memory (tests/helpers/ipc_rows.py).
Host-side ordering only (gloo collectives staged through host memory), so no
kernel waits on the other process.  Each rank's band must match the
single-grid solve (same PCG counts, u within 1e-9 relative)."""
import json
import os
import socket
import subprocess
import sys

import numpy as np
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


@pytest.mark.parametrize("shape", [(96, 80), (130, 72)])
def test_peer_transpose_two_processes(tmp_path, shape):
    out = str(tmp_path / "r")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "helpers", "ipc_rows.py"), out,
           str(shape[0]), str(shape[1])]
    proc = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-3000:]
    reps = [json.load(open(f"{out}.{r}.json")) for r in range(2)]
    single_u = np.load(f"{out}.single_u.npy")
    for rep in reps:
        assert rep["world"] == 2 and rep["peer"]
        assert rep["opened"] == 2  # the other rank's column block and back buffer, mapped over IPC
        assert rep["cg_iters"] == reps[0]["single_cg_iters"]
        u = np.load(f"{out}.u{rep['rank']}.npy")
        want = single_u[rep["row0"]:rep["row0"] + rep["rows"]]
        assert u.shape == want.shape
        assert np.linalg.norm(u - want) <= 1e-9 * np.linalg.norm(want)
