"""Multi-GPU sharding of the ALTO nonzero stream.

One process per GPU. Rank r owns the contiguous ALTO-ordered slice
[bounds[r], bounds[r+1]) with bounds = balanced_bounds(M, world) -- a line
segment at L = world (pkg/src/alto/partition.py:69-75). Every rank computes
a factor-sized partial MTTKRP / Phi over its slice; the partials are summed
with one NCCL all-reduce over NVLink (reduce-scatter + all-gather of the
updated rows collapsed into one collective, since the R x R solve is
replicated), after which every rank holds identical factors.

The same code runs on CPU tensors with the gloo backend (tests).
"""

from __future__ import annotations

import numpy as np

from .partition import balanced_bounds


def shard_range(M: int, world: int, rank: int) -> tuple[int, int]:
    b = balanced_bounds(M, world)
    return int(b[rank]), int(b[rank + 1])


def shard_tensor(alto, world: int, rank: int):
    """This rank's slice of a device AltoTensor (views, no copy)."""
    from .tensor import AltoTensor

    a, b = shard_range(alto.nnz, world, rank)
    return AltoTensor(alto.layout, alto._keys[a:b], alto._vals[a:b], _validate=False)


def _collective(t, op, group):
    """all_reduce in place; NCCL reduces device tensors directly, gloo (tests,
    including several ranks sharing one GPU) stages them through the host."""
    import torch.distributed as dist

    if dist.get_backend(group) == "gloo" and t.is_cuda:
        h = t.cpu()
        dist.all_reduce(h, op=op, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op, group=group)
    return t


def _active(group) -> bool:
    import torch.distributed as dist

    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def allreduce_(t, group=None):
    """In-place sum over ranks (NCCL over NVLink for CUDA tensors)."""
    import torch.distributed as dist

    if _active(group):
        _collective(t, dist.ReduceOp.SUM, group)
    return t


def allreduce_max(value: float, device=None, group=None) -> float:
    import torch
    import torch.distributed as dist

    if not _active(group):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    _collective(t, dist.ReduceOp.MAX, group)
    return float(t.item())


def reduce_partials_numpy(parts: list[np.ndarray]) -> np.ndarray:
    """Fixed-order host sum of per-rank partials (reference for tests)."""
    out = np.zeros_like(parts[0])
    for p in parts:
        out += p
    return out
