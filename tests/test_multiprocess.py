"""Multi-process (world_size 2, gloo, CPU) coverage of the multi-GPU plumbing:
the target-partition row gather that replaces the single-process output."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, n, cols, cuts, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2401_07361_b200.dist import gather_partitioned_rows

        g = torch.Generator().manual_seed(1234)
        perm = torch.randperm(n, generator=g).to(torch.int32)
        full = torch.arange(n * cols, dtype=torch.float64).reshape(n, cols) * 0.5 + 1.0
        out = torch.zeros(n, cols, dtype=torch.float64)
        p0, p1 = cuts[rank], cuts[rank + 1]
        rows = perm[p0:p1].long()
        out[rows] = full[rows]  # this rank computed only its rows
        gather_partitioned_rows(out, perm, p0, p1)
        q.put((rank, bool(torch.equal(out, full))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cuts,cols", [([0, 37, 100], 3), ([0, 0, 100], 3), ([0, 100, 100], 1), ([0, 50, 100], 1)])
def test_gather_partitioned_rows_gloo(cuts, cols):
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, 100, cols, cuts, q)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(ws))
    assert res == {0: True, 1: True}


class _CpuRK4Ops:
    """CPU stand-in for dist.TreecodeRK4Ops: the same stage protocol, the
    velocity by direct summation over this rank's slice of a fixed
    permutation, then the row all-gather. Exercises the multi-GPU RK4 driver's
    control flow and exchange under gloo."""

    def __init__(self, rank, ws, perm):
        self.rank, self.ws, self.perm = rank, ws, perm

    def stage_begin(self, s, dt, st):
        cs = (0.0, 0.5 * dt, 0.5 * dt, dt)[s]
        v = st["x0"] + cs * st["k"]
        st["xs"].copy_(v / v.norm(dim=1, keepdim=True) if s else st["x0"])
        st["q"].copy_((st["z0"] + cs * st["kz"]) * st["area"])

    def velocity(self, st):
        from paper_2401_07361_b200.dist import gather_partitioned_rows

        n = st["n"]
        cuts = [n * r // self.ws for r in range(self.ws + 1)]
        p0, p1 = cuts[self.rank], cuts[self.rank + 1]
        st["u"].zero_()
        rows = self.perm[p0:p1].long()
        x, q = st["xs"], st["q"]
        xi = x[rows]
        den = 1.0 - xi @ x.T
        den[torch.arange(len(rows)), rows] = float("inf")  # no self pairs
        w = q / den
        st["u"][rows] = -torch.cross(xi, w @ x, dim=1) / (4 * torch.pi)
        gather_partitioned_rows(st["u"], self.perm, p0, p1)

    def stage_end(self, s, omega, st):
        u = st["u"]
        wgt = 2.0 if s in (1, 2) else 1.0
        st["k"].copy_(u)
        st["kz"].copy_(-2.0 * omega * u[:, 2])
        if s == 0:
            st["acc"].copy_(u)
            st["accz"].copy_(st["kz"])
        else:
            st["acc"].add_(wgt * u)
            st["accz"].add_(wgt * st["kz"])

    def step_end(self, dt, st):
        v = st["x0"] + dt / 6.0 * st["acc"]
        st["x0"].copy_(v / v.norm(dim=1, keepdim=True))
        st["z0"].add_(dt / 6.0 * st["accz"])


def _rk4_worker(rank, ws, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2401_07361_b200.dist import rk4_distributed

        g = torch.Generator().manual_seed(7)
        x = torch.randn(60, 3, generator=g, dtype=torch.float64)
        x /= x.norm(dim=1, keepdim=True)
        z = torch.randn(60, generator=g, dtype=torch.float64)
        a = torch.full((60,), 4 * torch.pi / 60, dtype=torch.float64)
        perm = torch.randperm(60, generator=g).to(torch.int32)
        rk4_distributed(x, z, a, 0.01, 2, _CpuRK4Ops(rank, ws, perm))
        q.put((rank, x.numpy().tobytes(), z.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


def test_rk4_distributed_gloo():
    """Two ranks, each evaluating half the rows per stage and all-gathering,
    end with the same state as one rank evaluating everything."""
    ctx = mp.get_context("spawn")
    outs = {}
    for ws in (1, 2):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_rk4_worker, args=(r, ws, port, q)) for r in range(ws)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
        outs[ws] = dict((r, (xb, zb)) for r, xb, zb in (q.get(timeout=10) for _ in range(ws)))
    assert outs[2][0] == outs[2][1]  # every rank holds the same state
    assert outs[2][0] == outs[1][0]  # and it is the single-rank result


def _inputs_worker(rank, ws, port, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        from paper_2401_07361_b200.dist import allgather_inputs, shard_rows

        g = torch.Generator().manual_seed(99)
        xyz = torch.randn(n, 3, generator=g, dtype=torch.float64)
        qq = torch.randn(n, generator=g, dtype=torch.float64)
        # this rank's host copy holds only its shard (the rest is garbage)
        a, b = shard_rows(n, ws, rank)
        h_xyz = torch.full_like(xyz, float("nan"))
        h_q = torch.full_like(qq, float("nan"))
        h_xyz[a:b], h_q[a:b] = xyz[a:b], qq[a:b]
        m = -(-n // ws)
        d_xyz = torch.full((ws * m, 3), -1.0, dtype=torch.float64)
        d_q = torch.full((ws * m,), -1.0, dtype=torch.float64)
        allgather_inputs(h_xyz, h_q, d_xyz, d_q)
        q.put((rank, bool(torch.equal(d_xyz[:n], xyz) and torch.equal(d_q[:n], qq))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n", [10, 11, 1])
def test_allgather_inputs_gloo(n):
    """bench.py's distributed e2e staging: each rank supplies only its shard
    of the host inputs; after the all-gather every rank holds all N rows."""
    ws = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_inputs_worker, args=(r, ws, port, n, q)) for r in range(ws)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=10) for _ in range(ws))
    assert res == {0: True, 1: True}
