"""The NCCL side of the multi-GPU path on the one GPU available: a
world-size-1 NCCL group runs the exact collectives the ranks use —
all_gather_into_tensor on __cuda_array_interface__ views of the library's
leaf-key buffers (sharded binning) and on the tree-order row slots (the
fused RK4 stage exchange) — and the result must be the plain single-GPU one
bit for bit. (More ranks need more GPUs; their protocol is gloo-tested in
tests/test_multiprocess.py.)"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(port, q):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        import paper_2401_07361_b200 as ss
        from paper_2401_07361_b200.dist import _DeviceArray, slot_bounds

        xyz, area = ss.make_icosa_mesh(6)
        zeta = ss.rh4_vorticity(xyz)
        n = xyz.shape[0]
        cfg = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=6, max_depth=10)
        ref_x, ref_z = ss.rk4(xyz, zeta, area, cfg, dt=0.01, steps=2, tree=ss.FaceTree(0))
        dev = torch.device("cuda", 0)
        t = ss.FaceTree(0)
        t.set_stream(torch.cuda.current_stream().cuda_stream)
        t.set_output_order(True)
        x = torch.from_numpy(xyz.copy()).to(dev)
        z = torch.from_numpy(zeta.copy()).to(dev)
        a = torch.from_numpy(area).to(dev)
        xs, qs = torch.empty_like(x), torch.empty_like(z)
        k, kz, acc, accz = torch.zeros_like(x), torch.zeros_like(z), torch.zeros_like(x), torch.zeros_like(z)
        slot = torch.zeros_like(x)
        rows = torch.zeros_like(x)
        walked_any = False
        for _ in range(2):
            for s in range(4):
                t.rk4_stage_begin(s, 0.01, n, x.data_ptr(), z.data_ptr(), a.data_ptr(), k.data_ptr(), kz.data_ptr(),
                                  xs.data_ptr(), qs.data_ptr())
                lo, hi, m = slot_bounds(n, 1, 0)
                kp, lp, walked = t.bin_walk_shard(xs.data_ptr(), n, lo, hi, m)
                if walked:  # the collective sharded_walk issues, on library memory
                    walked_any = True
                    keys = torch.as_tensor(_DeviceArray(kp, m, "<i8"), device=dev)
                    leaf = torch.as_tensor(_DeviceArray(lp, m, "<i4"), device=dev)
                    for buf in (keys, leaf):
                        dist.all_gather_into_tensor(buf, buf[:m].clone())
                ss.treecode_sum_device(t, ss.BiotSavartKernel, cfg, xs.data_ptr(), qs.data_ptr(), n, slot.data_ptr())
                cuts = t.partition_cuts()
                w = int(cuts[1] - cuts[0])
                dist.all_gather_into_tensor(rows[:w], slot[:w])  # the stage exchange
                t.rk4_stage_end_rows(s, 2 * np.pi, n, rows.data_ptr(), w, k.data_ptr(), kz.data_ptr(),
                                     acc.data_ptr(), accz.data_ptr())
            t.rk4_step_end(0.01, n, x.data_ptr(), z.data_ptr(), acc.data_ptr(), accz.data_ptr())
        torch.cuda.synchronize()
        q.put((walked_any, bool(np.array_equal(x.cpu().numpy(), ref_x)), bool(np.array_equal(z.cpu().numpy(), ref_z))))
    finally:
        dist.destroy_process_group()


def test_nccl_collectives_on_library_buffers():
    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    p = ctx.Process(target=_worker, args=(port, q))
    p.start()
    p.join(300)
    assert p.exitcode == 0
    assert q.get(timeout=10) == (True, True, True)
