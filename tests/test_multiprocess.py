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
    """CPU stand-in for dist.TreecodeRK4Ops with the same protocol: each rank
    evaluates its contiguous range of tree positions (a fixed permutation
    plays the binning's), writes those rows in tree order into its slot, ONE
    all-gather of equal slots (dist.exchange_rows), then the stage update
    reads the gathered rows through the permutation (dist.assemble_rows =
    what ssum_rk4_stage_end_rows does on the device)."""

    def __init__(self, rank, ws, perm, cuts):
        self.rank, self.ws, self.perm, self.cuts = rank, ws, perm, cuts

    def state(self, x, z, a):
        n = x.shape[0]
        return {"n": n, "x0": x, "z0": z, "area": a, "xs": torch.empty_like(x), "q": torch.empty_like(z),
                "k": torch.zeros_like(x), "kz": torch.zeros_like(z), "acc": torch.zeros_like(x),
                "accz": torch.zeros_like(z), "slot": torch.zeros_like(x), "rows": torch.zeros((self.ws * n, 3),
                                                                                              dtype=x.dtype),
                "u": torch.zeros_like(x)}

    def stage(self, s, dt, omega, st):
        from paper_2401_07361_b200.dist import assemble_rows, exchange_rows, slot_width

        cs = (0.0, 0.5 * dt, 0.5 * dt, dt)[s]
        v = st["x0"] + cs * st["k"]
        st["xs"].copy_(v / v.norm(dim=1, keepdim=True) if s else st["x0"])
        st["q"].copy_((st["z0"] + cs * st["kz"]) * st["area"])
        p0, p1 = self.cuts[self.rank], self.cuts[self.rank + 1]
        ids = self.perm[p0:p1].long()  # this rank's targets, tree order
        x, q = st["xs"], st["q"]
        xi = x[ids]
        den = 1.0 - xi @ x.T
        den[torch.arange(len(ids)), ids] = float("inf")  # no self pairs
        st["slot"][: p1 - p0] = -torch.cross(xi, (q / den) @ x, dim=1) / (4 * torch.pi)
        w = slot_width(self.cuts) if self.ws > 1 else st["n"]
        rows = exchange_rows(st["slot"], st["rows"], w)
        u = assemble_rows(rows, w, self.cuts, self.perm, st["u"])
        wgt = 2.0 if s in (1, 2) else 1.0
        st["k"].copy_(u)
        st["kz"].copy_(-2.0 * omega * u[:, 2])
        if s == 0:
            st["acc"].copy_(u)
            st["accz"].copy_(st["kz"])
        else:
            st["acc"].add_(wgt * u)
            st["accz"].add_(wgt * st["kz"])

    def step(self, dt, st, omega):
        for s in range(4):
            self.stage(s, dt, omega, st)
        v = st["x0"] + dt / 6.0 * st["acc"]
        st["x0"].copy_(v / v.norm(dim=1, keepdim=True))
        st["z0"].add_(dt / 6.0 * st["accz"])


def _rk4_worker(rank, ws, port, q, cuts):
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
        rk4_distributed(x, z, a, 0.01, 2, _CpuRK4Ops(rank, ws, perm, cuts))
        q.put((rank, x.numpy().tobytes(), z.numpy().tobytes()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cuts2", [[0, 23, 60], [0, 0, 60], [0, 60, 60]])
def test_rk4_distributed_gloo(cuts2):
    """Two ranks, each evaluating its (unequal, possibly empty) range of tree
    positions per stage and exchanging tree-order slots, end with the same
    state as one rank evaluating everything."""
    ctx = mp.get_context("spawn")
    outs = {}
    for ws, cuts in ((1, [0, 60]), (2, cuts2)):
        q = ctx.Queue()
        port = _free_port()
        procs = [ctx.Process(target=_rk4_worker, args=(r, ws, port, q, cuts)) for r in range(ws)]
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
