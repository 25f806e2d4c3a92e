"""Multi-process (world_size 2, gloo, CPU) tests of the N > 1 host path:
round-robin sharding of independent images, max-over-ranks timing and the
result gather used by bench.py / unwrap_batch.  The per-image solver is the
CPU oracle here (this container has no GPU); on the GPU box the same code
calls the CUDA unwrap."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2401_09961_b200.batch import shard_indices


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_solver(x, c, model, params, lo, dtype="fp64"):
    from oracle import phaseirls_port as port
    from paper_2401_09961_b200.params import IrlsTrace, IterationRecord, UnwrapResult
    state, recs, _ = port.unwrap(x, lo=lo, poisson="dct")
    tr = IrlsTrace()
    for r in recs:
        tr.append(IterationRecord(r.k, r.m_cg, r.delta_rel, r.h_delta, r.cg_iters, r.sufficient_decrease,
                                  r.fallback_used))
    return UnwrapResult(state.u, state.vv, state.vh, tr)


def _images():
    from paper_2401_09961_b200.synth import SceneSpec, add_phase_noise, generate_scene, wrap_scene
    return [add_phase_noise(wrap_scene(generate_scene(SceneSpec("gaussian-bumps", 20, 18, 6.0, 5.0, s))), 0.3,
                            100 + s) for s in range(5)]


def _worker(rank, world, port, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import torch.distributed as dist
    from paper_2401_09961_b200.batch import max_over_ranks, unwrap_batch
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    imgs = _images()
    res = unwrap_batch(imgs, solver=_oracle_solver, gather=True)
    local = unwrap_batch(imgs, solver=_oracle_solver, gather=False)
    t = max_over_ranks(1.0 + rank)
    np.savez(os.path.join(outdir, f"rank{rank}.npz"),
             u=np.stack([r.u for r in res]),
             mine=np.array([i for i, r in enumerate(local) if r is not None]),
             t=np.array(t))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_indices():
    assert shard_indices(5, 0, 2) == [0, 2, 4]
    assert shard_indices(5, 1, 2) == [1, 3]
    assert sorted(shard_indices(64, r, 8)[0] for r in range(8)) == list(range(8))
    with pytest.raises(ValueError):
        shard_indices(4, 2, 2)


def test_world2_gloo(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    r0 = np.load(tmp_path / "rank0.npz")
    r1 = np.load(tmp_path / "rank1.npz")
    assert r0["mine"].tolist() == [0, 2, 4] and r1["mine"].tolist() == [1, 3]
    assert float(r0["t"]) == 2.0 and float(r1["t"]) == 2.0          # max over ranks
    np.testing.assert_array_equal(r0["u"], r1["u"])                 # every rank sees all results
    single = [_oracle_solver(x, None, None, None, -np.pi).u for x in _images()]
    np.testing.assert_allclose(r0["u"], np.stack(single), rtol=0, atol=1e-12)
