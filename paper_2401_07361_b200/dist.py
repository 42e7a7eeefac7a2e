"""Multi-GPU plumbing over torch.distributed (one process per GPU).

The tree code shards by TARGETS: every rank bins and
traverses the full (replicated) particle set, then evaluates only its
cost-balanced contiguous range of target leaves (FaceTree.set_partition).
The one exchange step is this all-gather of the rows each rank computed, so
every rank holds the full velocity field (e.g. before the next RK4 stage).
Rows travel in tree order (contiguous per rank); each rank scatters them back
to the caller's particle order with the shared permutation.
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def gather_partitioned_rows(out: torch.Tensor, perm: torch.Tensor, p0: int, p1: int,
                            group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """out: (N, D) with valid rows perm[p0:p1] on this rank; returns `out`
    with every rank's rows filled in. Works for NCCL (CUDA tensors) and gloo
    (CPU tensors)."""
    ws = dist.get_world_size(group)
    if ws == 1:
        return out
    dev = out.device
    rng = torch.tensor([p0, p1], dtype=torch.int64, device=dev)
    ranges = [torch.empty_like(rng) for _ in range(ws)]
    dist.all_gather(ranges, rng, group=group)
    ranges = [(int(r[0]), int(r[1])) for r in ranges]
    width = max(e - b for b, e in ranges)
    cols = out.shape[1] if out.dim() > 1 else 1
    mine = torch.zeros((width, cols), dtype=out.dtype, device=dev)
    idx = perm[p0:p1].long()
    mine[: p1 - p0] = out[idx].reshape(p1 - p0, cols)
    bufs = [torch.empty_like(mine) for _ in range(ws)]
    dist.all_gather(bufs, mine, group=group)
    for (b, e), buf in zip(ranges, bufs):
        if e > b:
            out[perm[b:e].long()] = buf[: e - b].reshape((e - b,) + tuple(out.shape[1:]))
    return out


def gather_rows(tree, out: torch.Tensor, group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """All-gather the last partitioned evaluation of `tree` into `out` (device)."""
    p0, p1 = tree.partition_range()
    n = out.shape[0]
    perm = torch.empty(n, dtype=torch.int32, device=out.device)
    tree.perm(perm.data_ptr())
    return gather_partitioned_rows(out, perm, p0, p1, group)
