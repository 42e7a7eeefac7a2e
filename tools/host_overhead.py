"""Host-side time of each call in the device-resident RK4 stage loop
(dist.TreecodeRK4Ops.step, N = 1) at config 4: where the GPU idles between
one evaluation's final check and the next evaluation's first kernel.

    python tools/host_overhead.py [steps]
"""
import os
import statistics
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2401_07361_b200 as ss  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
bench.use_config("c4")
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
xyz, zeta, area = bench.fixture_product()
S = bench.Stepper(ss, torch, dev, xyz, zeta, area, 1, 0)
ops, st = S.ops, S.st
for _ in range(2):
    S.step()
torch.cuda.synchronize()

n = st["n"]
t = ops.tree
dt = bench.C["rk4"]["dt"]
omega = 2.0 * 3.141592653589793
p = {k: st[k].data_ptr() for k in ("x0", "z0", "area", "acc", "accz", "xs", "q", "k", "kz")}
marks = {}


def stamp(label, t0):
    t1 = time.perf_counter()
    marks.setdefault(label, []).append((t1 - t0) * 1e6)
    return t1


for _ in range(steps):
    t0 = time.perf_counter()
    t.rk4_stage_begin(0, dt, n, p["x0"], p["z0"], p["area"], p["k"], p["kz"], p["xs"], p["q"])
    t0 = stamp("stage_begin", t0)
    for s in range(4):
        stats = ss.TreecodeStats()
        t0 = stamp("TreecodeStats()", t0)
        ss.treecode_sum_device(t, ss.BiotSavartKernel, ops.cfg, st["xs"].data_ptr(), st["q"].data_ptr(), n,
                               st["slot"].data_ptr(), stats=stats)
        t0 = stamp("treecode_sum_device (incl. GPU)", t0)
        cuts = t.partition_cuts()
        t0 = stamp("partition_cuts", t0)
        t.rk4_stage_advance_rows(s, dt, omega, n, st["slot"].data_ptr(), n, p["x0"], p["z0"], p["area"], p["acc"],
                                 p["accz"], p["xs"], p["q"])
        t0 = stamp("rk4_stage_advance_rows", t0)
    t.rk4_step_end(dt, n, p["x0"], p["z0"], p["acc"], p["accz"])
    t0 = stamp("rk4_step_end (incl. sync)", t0)
torch.cuda.synchronize()
for k, v in marks.items():
    print(f"{k:34s} median {statistics.median(v):9.1f} us  min {min(v):9.1f}  n {len(v)}")
# the library's own host phases of one evaluation (SSUM_TRACE marks)
