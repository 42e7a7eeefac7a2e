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
    ws = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
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


def shard_rows(n: int, ws: int, rank: int) -> tuple:
    """Rank `rank`'s rows [a, b) of n in the caller's order: equal slots of
    ceil(n / ws) rows (the last one short), so the all-gathers below need no
    per-rank sizes."""
    m = -(-n // ws)
    return min(n, rank * m), min(n, (rank + 1) * m)


def allgather_inputs(h_xyz: torch.Tensor, h_q: torch.Tensor, d_xyz: torch.Tensor, d_q: torch.Tensor,
                     group: Optional[dist.ProcessGroup] = None) -> None:
    """Distributed input staging (BASELINE north_star: particle positions are
    all-gathered over NVLink): rank r copies only its shard_rows() of the
    host inputs (pinned) to its device, and one all-gather per array
    completes the replicated particle set on every rank. d_xyz (>= ws*m, 3)
    and d_q (>= ws*m,) with m = ceil(N / ws): rows [0, N) receive the
    inputs; rows past N are padding."""
    n = h_xyz.shape[0]
    ws = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    if ws == 1:
        d_xyz[:n].copy_(h_xyz, non_blocking=True)
        d_q[:n].copy_(h_q, non_blocking=True)
        return
    r = dist.get_rank(group)
    m = -(-n // ws)
    a, b = shard_rows(n, ws, r)
    for h, d in ((h_xyz, d_xyz), (h_q, d_q)):
        slot = d[r * m:(r + 1) * m]
        if b > a:
            slot[: b - a].copy_(h[a:b], non_blocking=True)
        if b - a < m:
            slot[b - a:].zero_()
        _all_gather_slots(d[: ws * m], slot, ws, group)


def _all_gather_slots(buf: torch.Tensor, slot: torch.Tensor, ws: int, group) -> None:
    """buf = ws equal slots; `slot` (this rank's) is one of them, in place."""
    if buf.is_cuda:
        dist.all_gather_into_tensor(buf, slot.clone(), group=group)
    else:  # gloo
        outs = [torch.empty_like(slot) for _ in range(ws)]
        dist.all_gather(outs, slot.clone(), group=group)
        buf.copy_(torch.cat(outs))


def gather_rows(tree, out: torch.Tensor, group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """All-gather the last partitioned evaluation of `tree` into `out` (device)."""
    p0, p1 = tree.partition_range()
    n = out.shape[0]
    perm = torch.empty(n, dtype=torch.int32, device=out.device)
    tree.perm(perm.data_ptr())
    return gather_partitioned_rows(out, perm, p0, p1, group)


# ------------------------------------------------------------------ RK4
class TreecodeRK4Ops:
    """Stage operations of the multi-GPU RK4 on one FaceTree (this rank's
    GPU): the RK4 arithmetic runs through ssum_rk4_stage_* (the kernels of
    ssum_rk4), the stage velocity is this rank's partitioned tree-code
    evaluation followed by the row all-gather (one exchange
    per stage)."""

    def __init__(self, tree, cfg, group: Optional[dist.ProcessGroup] = None):
        from . import BiotSavartKernel, treecode_sum_device

        self.tree, self.cfg, self.group = tree, cfg, group
        self._k, self._eval = BiotSavartKernel, treecode_sum_device

    def stage_begin(self, s: int, dt: float, st: dict) -> None:
        n = st["n"]
        self.tree.rk4_stage_begin(s, dt, n, st["x0"].data_ptr(), st["z0"].data_ptr(), st["area"].data_ptr(),
                                  st["k"].data_ptr(), st["kz"].data_ptr(), st["xs"].data_ptr(), st["q"].data_ptr())

    def velocity(self, st: dict) -> None:
        n = st["n"]
        st["u"].zero_()
        self._eval(self.tree, self._k, self.cfg, st["xs"].data_ptr(), st["q"].data_ptr(), n, st["u"].data_ptr())
        gather_rows(self.tree, st["u"], self.group)

    def stage_end(self, s: int, omega: float, st: dict) -> None:
        self.tree.rk4_stage_end(s, omega, st["n"], st["u"].data_ptr(), st["k"].data_ptr(), st["kz"].data_ptr(),
                                st["acc"].data_ptr(), st["accz"].data_ptr())

    def step_end(self, dt: float, st: dict) -> None:
        self.tree.rk4_step_end(dt, st["n"], st["x0"].data_ptr(), st["z0"].data_ptr(), st["acc"].data_ptr(),
                               st["accz"].data_ptr())


def rk4_distributed(x: torch.Tensor, zeta: torch.Tensor, area: torch.Tensor, dt: float, steps: int, ops,
                    omega: float = 2.0 * 3.141592653589793):
    """Lagrangian RK4 of the BVE with the stage velocities
    from `ops.velocity` (every rank ends each stage holding all N rows). x
    (N, 3), zeta (N), area (N) are replicated on every rank and advanced in
    place; returns (x, zeta). With TreecodeRK4Ops on one rank this is
    ssum_rk4 bit for bit."""
    n = x.shape[0]
    st = {"n": n, "x0": x, "z0": zeta, "area": area, "xs": torch.empty_like(x), "q": torch.empty_like(zeta),
          "u": torch.zeros_like(x), "k": torch.zeros_like(x), "kz": torch.zeros_like(zeta),
          "acc": torch.zeros_like(x), "accz": torch.zeros_like(zeta)}
    for _ in range(steps):
        for s in range(4):
            ops.stage_begin(s, dt, st)
            ops.velocity(st)
            ops.stage_end(s, omega, st)
        ops.step_end(dt, st)
    return x, zeta
