"""Independent interferograms sharded across GPUs (BASELINE config C5).

One process per GPU (torchrun); rank r unwraps images r, r + W, r + 2W, ...
with no data-path collective — the images are independent units, so this is
weak scaling.  `torch.distributed` is only used to agree on timing (max over
ranks) and, optionally, to gather the results.  The per-image solver is the
GPU `unwrap`; tests inject a CPU stand-in to exercise the sharding and
gathering logic with the gloo backend.
"""

from __future__ import annotations

import numpy as np


def shard_indices(n_items: int, rank: int, world: int):
    """Images handled by `rank` (round-robin, deterministic)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError(f"invalid rank {rank} / world {world}")
    return list(range(rank, n_items, world))


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def rank_world(group=None):
    dist = _dist()
    if dist is None:
        return 0, 1
    return dist.get_rank(group), dist.get_world_size(group)


def max_over_ranks(value: float, group=None, device=None) -> float:
    """Max of a per-rank scalar (bench timing rule: time = max over ranks)."""
    dist = _dist()
    if dist is None:
        return float(value)
    import torch
    backend = dist.get_backend(group)
    dev = device if device is not None else (torch.device("cuda", torch.cuda.current_device())
                                             if backend == "nccl" else torch.device("cpu"))
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def unwrap_batch(images, c=None, model=None, params=None, gradient_lo=-np.pi, *, dtype="fp64", gather=True,
                 group=None, solver=None):
    """Unwrap a list of wrapped grids across the ranks of `group`.

    Returns a list of length len(images): UnwrapResult for the images this
    rank solved (all of them when `gather` is true, else None elsewhere).
    `solver(x, c, model, params, gradient_lo, dtype=...)` defaults to the GPU
    `unwrap`.
    """
    if solver is None:
        from .irls import unwrap as solver
    rank, world = rank_world(group)
    mine = shard_indices(len(images), rank, world)
    local = {i: solver(images[i], c, model, params, gradient_lo, dtype=dtype) for i in mine}
    out = [local.get(i) for i in range(len(images))]
    if not gather or world == 1:
        return out
    dist = _dist()
    parts = [None] * world
    dist.all_gather_object(parts, local, group=group)
    for part in parts:
        for i, res in part.items():
            out[i] = res
    return out
