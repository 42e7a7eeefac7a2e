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
