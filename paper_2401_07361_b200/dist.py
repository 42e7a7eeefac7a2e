"""Multi-GPU plumbing over torch.distributed (one process per GPU).

The tree code shards by TARGETS: every rank bins and
traverses the full (replicated) particle set, then evaluates only its
cost-balanced contiguous range of target leaves (FaceTree.set_partition).
Every rank bins identically, so every rank knows every part's tree-position
range without communicating (FaceTree.partition_cuts).

The binning's particle walk is sharded too (sharded_walk): each rank walks
1/ws of the particles and one all-gather of the per-particle leaf keys
completes every rank's binning.

The one exchange per RK4 stage (§8(f) rank 2) is fused into the stage
update: each rank's evaluation writes its rows in TREE order straight into
a slot (FaceTree.set_output_order), ONE all-gather of equal-width slots
(ncclAllGather under NCCL) leaves every part's rows on every rank, and the
stage kernel (ssum_rk4_stage_end_rows) reads them there through the
binning's permutation — no scatter, no index tensors, no per-rank sizes on
the wire.

`gather_partitioned_rows` / `gather_rows` remain for single evaluations in
the caller's order (bench.py's non-RK4 configs).
"""
from __future__ import annotations

from typing import Optional

import torch
import torch.distributed as dist


def _ws(group=None) -> int:
    return dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1


def slot_width(cuts) -> int:
    """Equal slot width for the row all-gather: the widest part."""
    return max(int(cuts[r + 1]) - int(cuts[r]) for r in range(len(cuts) - 1))


def exchange_rows(slot: torch.Tensor, rows: torch.Tensor, width: int,
                  group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """All-gather equal slots: slot[:width] (this rank's rows, tree order) to
    rows[r * width:(r + 1) * width] for every rank r. One collective."""
    ws = _ws(group)
    if ws == 1:
        return slot
    out = rows[: ws * width]
    if out.is_cuda:
        dist.all_gather_into_tensor(out, slot[:width], group=group)
    else:  # gloo
        parts = [torch.empty_like(slot[:width]) for _ in range(ws)]
        dist.all_gather(parts, slot[:width].contiguous(), group=group)
        out.copy_(torch.cat(parts))
    return out


def assemble_rows(rows: torch.Tensor, width: int, cuts, perm: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """out[perm[j]] = the row of tree position j in the all-gathered slots —
    what ssum_rk4_stage_end_rows reads on the device (tests and CPU drivers)."""
    for r in range(len(cuts) - 1):
        a, b = int(cuts[r]), int(cuts[r + 1])
        if b > a:
            out[perm[a:b].long()] = rows[r * width:r * width + (b - a)]
    return out


class _DeviceArray:
    """A raw device allocation of the library as a torch tensor view
    (__cuda_array_interface__, no copy)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def slot_bounds(n: int, ws: int, rank: int) -> tuple:
    """Rank `rank`'s equal slot [a, b) of n rows (m = ceil(n / ws) per slot)."""
    m = -(-n // ws)
    return min(n, rank * m), min(n, (rank + 1) * m), m


def sharded_walk(tree, xyz_ptr: int, n: int, group: Optional[dist.ProcessGroup] = None,
                 device: Optional[torch.device] = None) -> bool:
    """Multi-GPU binning: this rank walks only its slot of
    the particles through the tree (ssum_bin_walk_shard), then ONE all-gather
    per array (leaf keys, leaves) completes every rank's copy; the next
    evaluation of these n particles starts its binning at the sort, bitwise
    the unsharded binning. Returns False when the tree could not be walked
    yet (first call on a tree: every rank builds it)."""
    ws = _ws(group)
    r = dist.get_rank(group) if ws > 1 else 0
    a, b, m = slot_bounds(n, ws, r)
    kp, lp, walked = tree.bin_walk_shard(xyz_ptr, n, a, b, ws * m)
    if not walked or ws == 1:
        return walked
    dev = device or torch.device("cuda", torch.cuda.current_device())
    keys = torch.as_tensor(_DeviceArray(kp, ws * m, "<i8"), device=dev)
    leaf = torch.as_tensor(_DeviceArray(lp, ws * m, "<i4"), device=dev)
    for buf in (keys, leaf):
        _all_gather_slots(buf, buf[r * m:(r + 1) * m], ws, group)
    return True


def gather_partitioned_rows(out: torch.Tensor, perm: torch.Tensor, p0: int, p1: int,
                            group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """out: (N, D) in the caller's order with valid rows perm[p0:p1] on this
    rank; returns `out` with every rank's rows filled in (single evaluations
    in the caller's order). Works for NCCL (CUDA tensors) and gloo (CPU)."""
    ws = _ws(group)
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
    ws = _ws(group)
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
    """All-gather the last partitioned evaluation of `tree` into `out` (device,
    caller's order)."""
    p0, p1 = tree.partition_range()
    n = out.shape[0]
    perm = torch.empty(n, dtype=torch.int32, device=out.device)
    tree.perm(perm.data_ptr())
    return gather_partitioned_rows(out, perm, p0, p1, group)


# ------------------------------------------------------------------ RK4
class TreecodeRK4Ops:
    """Stage operations of the (multi-GPU) RK4 on one FaceTree (this rank's
    GPU, on torch's current stream): ssum_rk4_stage_begin, this rank's
    partitioned tree-code evaluation written in tree order into its slot,
    one all-gather of the slots, ssum_rk4_stage_end_rows on the gathered
    rows, and ssum_rk4_step_end — the kernels of ssum_rk4, so one rank
    reproduces it bit for bit and G ranks reproduce one rank bit for bit.
    `stats`: a list that receives each evaluation's TreecodeStats."""

    def __init__(self, tree, cfg, group: Optional[dist.ProcessGroup] = None, stats: Optional[list] = None,
                 shard_binning: bool = True):
        from . import BiotSavartKernel, TreecodeStats, treecode_sum_device

        self.tree, self.cfg, self.group, self.stats = tree, cfg, group, stats
        self._k, self._eval, self._stats = BiotSavartKernel, treecode_sum_device, TreecodeStats
        self.ws = _ws(group)
        self.shard_binning = shard_binning and self.ws > 1
        tree.set_stream(torch.cuda.current_stream().cuda_stream)
        tree.set_output_order(True)
        if self.ws > 1:
            tree.set_partition(dist.get_rank(group), self.ws)

    def state(self, x: torch.Tensor, zeta: torch.Tensor, area: torch.Tensor) -> dict:
        n = x.shape[0]
        st = {"n": n, "x0": x, "z0": zeta, "area": area, "xs": torch.empty_like(x), "q": torch.empty_like(zeta),
              "k": torch.zeros_like(x), "kz": torch.zeros_like(zeta), "acc": torch.zeros_like(x),
              "accz": torch.zeros_like(zeta), "slot": torch.zeros_like(x)}
        st["rows"] = torch.zeros((self.ws * n, 3), dtype=x.dtype, device=x.device) if self.ws > 1 else st["slot"]
        return st

    def _evaluate(self, st: dict):
        """This rank's partitioned evaluation at st["xs"], st["q"] and the one
        all-gather of the slots: (rows, width, our kernel launches)."""
        n = st["n"]
        t = self.tree
        stats = self._stats()
        if self.shard_binning:  # each rank walks 1/ws of the particles, one all-gather of the keys
            sharded_walk(t, st["xs"].data_ptr(), n, self.group, st["xs"].device)
        self._eval(t, self._k, self.cfg, st["xs"].data_ptr(), st["q"].data_ptr(), n, st["slot"].data_ptr(),
                   stats=stats)
        if self.stats is not None:
            self.stats.append(stats)
        cuts = t.partition_cuts()
        width = slot_width(cuts) if self.ws > 1 else n
        rows = exchange_rows(st["slot"], st["rows"], width, self.group)
        return rows, width, stats.gpu_launches

    def stage(self, s: int, dt: float, omega: float, st: dict) -> int:
        """One stage with the separate begin / end kernels (k, kz kept)."""
        n = st["n"]
        t = self.tree
        t.rk4_stage_begin(s, dt, n, st["x0"].data_ptr(), st["z0"].data_ptr(), st["area"].data_ptr(),
                          st["k"].data_ptr(), st["kz"].data_ptr(), st["xs"].data_ptr(), st["q"].data_ptr())
        rows, width, launches = self._evaluate(st)
        t.rk4_stage_end_rows(s, omega, n, rows.data_ptr(), width, st["k"].data_ptr(), st["kz"].data_ptr(),
                             st["acc"].data_ptr(), st["accz"].data_ptr())
        return launches + 2

    def step(self, dt: float, st: dict, omega: float = 2.0 * 3.141592653589793) -> int:
        """One RK4 step in place on st["x0"], st["z0"]; returns our kernel
        launches. Between two evaluations one fused kernel pair
        (ssum_rk4_stage_advance_rows) ends a stage and begins the next —
        bitwise the separate stage() kernels."""
        n = st["n"]
        t = self.tree
        p = {k: st[k].data_ptr() for k in ("x0", "z0", "area", "acc", "accz", "xs", "q", "k", "kz")}
        t.rk4_stage_begin(0, dt, n, p["x0"], p["z0"], p["area"], p["k"], p["kz"], p["xs"], p["q"])
        launches = 1
        for s in range(4):
            rows, width, nl = self._evaluate(st)
            t.rk4_stage_advance_rows(s, dt, omega, n, rows.data_ptr(), width, p["x0"], p["z0"], p["area"],
                                     p["acc"], p["accz"], p["xs"], p["q"])
            launches += nl + 2
        t.rk4_step_end(dt, n, p["x0"], p["z0"], p["acc"], p["accz"])
        return launches + 1


def rk4_distributed(x: torch.Tensor, zeta: torch.Tensor, area: torch.Tensor, dt: float, steps: int, ops,
                    omega: float = 2.0 * 3.141592653589793):
    """Lagrangian RK4 of the BVE with `ops` (TreecodeRK4Ops
    or a CPU stand-in with the same protocol). x (N, 3), zeta (N), area (N)
    are replicated on every rank and advanced in place; returns (x, zeta).
    With TreecodeRK4Ops on one rank this is ssum_rk4 bit for bit."""
    st = ops.state(x, zeta, area)
    for _ in range(steps):
        ops.step(dt, st, omega)
    return x, zeta
