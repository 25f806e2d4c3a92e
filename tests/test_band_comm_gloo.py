"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the row-sharded
exchange plumbing in band.py: the per-rank DistComm collectives (all-reduce of
band totals, the packed all-to-all transpose and its inverse, ghost-row halo
exchange) must leave every band exactly as the in-process LoopbackComm does.
The band kernels themselves need a GPU (tests/test_gpu_band.py)."""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2401_09961_b200 import _native as nat
from paper_2401_09961_b200.band import BandLayout, DistComm, LoopbackComm


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_band(lay, r, seed):
    """The attributes of BandState the communicators touch, on CPU, seeded."""
    g = torch.Generator().manual_seed(1000 * seed + r)
    ld = (lay.m + 7) // 8 * 8
    rows = lay.rows[r]
    b = SimpleNamespace(layout=lay, rank=r, rows=rows, row0=lay.row0[r], n=lay.n, m=lay.m, mb=lay.mb, nq=lay.world,
                        ld=ld, tdtype=torch.float64, device=torch.device("cpu"))
    b.X = torch.randn((3, rows + 2, ld), generator=g, dtype=torch.float64)
    b.Y = torch.randn((3, rows + 2, ld), generator=g, dtype=torch.float64)
    b.spec_send = torch.randn(lay.world * rows * lay.mb, generator=g, dtype=torch.float64)
    b.spec_col = torch.zeros(lay.n * lay.mb, dtype=torch.float64)
    b.totals = torch.randn(nat.NSITES * nat.MAX_SUMS, generator=g, dtype=torch.float64)
    return b


ITEMS = [(lambda b: b.X, 0, "both"), (lambda b: b.X, 1, "down"), (lambda b: b.Y, 2, "up")]


def _exercise(comm, bands):
    comm.allreduce(bands, nat.SITE_K2, nat.SITE_K3)
    comm.halo(bands, ITEMS)
    comm.transpose(bands)
    col = [b.spec_col.clone() for b in bands]
    for b in bands:  # make the return trip observable
        b.spec_col.mul_(2.0).add_(b.rank)
    comm.transpose_back(bands)
    return [dict(totals=b.totals.clone(), X=b.X.clone(), Y=b.Y.clone(), col=c, back=b.spec_send.clone())
            for b, c in zip(bands, col)]


def _worker(rank, world, port, outdir, shape):
    import torch.distributed as dist
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    lay = BandLayout(*shape, world)
    out = _exercise(DistComm(), [_fake_band(lay, rank, 7)])[0]
    torch.save(out, os.path.join(outdir, f"rank{rank}.pt"))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (20, 24)), (3, (29, 40))])
def test_distcomm_matches_loopback(tmp_path, world, shape):
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path), shape), nprocs=world, join=True)
    lay = BandLayout(*shape, world)
    want = _exercise(LoopbackComm(world), [_fake_band(lay, r, 7) for r in range(world)])
    for r in range(world):
        got = torch.load(tmp_path / f"rank{r}.pt")
        for key in ("totals", "X", "Y", "col", "back"):
            torch.testing.assert_close(got[key], want[r][key], rtol=0, atol=1e-12, msg=f"rank {r} {key}")


def test_loopback_transpose_is_a_transpose():
    """Packed chunk layout: the column block of rank q holds columns [q mb, q mb + cols) of every row."""
    lay = BandLayout(29, 40, 3)
    bands = [_fake_band(lay, r, 3) for r in range(3)]
    full = torch.zeros((lay.n, lay.world * lay.mb), dtype=torch.float64)
    for b in bands:  # the packed layout written by the row DCT-II: chunk q = columns [q mb, (q+1) mb)
        chunks = b.spec_send.view(lay.world, b.rows, lay.mb)
        for q in range(lay.world):
            full[b.row0:b.row0 + b.rows, q * lay.mb:(q + 1) * lay.mb] = chunks[q]
    LoopbackComm(3).transpose(bands)
    for q, b in enumerate(bands):
        np.testing.assert_array_equal(b.spec_col.view(lay.n, lay.mb).numpy(),
                                      full[:, q * lay.mb:(q + 1) * lay.mb].numpy())


def test_loopback_halo_semantics():
    lay = BandLayout(12, 24, 3)
    bands = [_fake_band(lay, r, 5) for r in range(3)]
    before = [b.X.clone() for b in bands]
    LoopbackComm(3).halo(bands, [(lambda b: b.X, 0, "both")])
    for r, b in enumerate(bands):
        if r > 0:    # ghost row -1 = last row of the band above
            assert torch.equal(b.X[0, 0], before[r - 1][0, bands[r - 1].rows])
        else:
            assert torch.equal(b.X[0, 0], before[r][0, 0])
        if r < 2:    # ghost row `rows` = first row of the band below
            assert torch.equal(b.X[0, b.rows + 1], before[r + 1][0, 1])
