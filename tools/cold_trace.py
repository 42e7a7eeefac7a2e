"""The first evaluation on a fresh FaceTree (cold path) and the next ones,
each with the SSUM_TRACE phase split on stderr and its wall time here.

    SSUM_TRACE=1 python tools/cold_trace.py [level]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2401_07361_b200 as ss  # noqa: E402

level = int(sys.argv[1]) if len(sys.argv) > 1 else 9
xyz, area = ss.make_icosa_mesh(level)
q = ss.rh4_vorticity(xyz) * area
n = xyz.shape[0]
dev = torch.device("cuda", 0)
x = torch.from_numpy(xyz).to(dev)
qq = torch.from_numpy(q).to(dev)
out = torch.zeros((n, 3), dtype=torch.float64, device=dev)
cfg = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=8, max_depth=10)
warm = ss.FaceTree(0)  # CUDA context, module load, first cudaMallocs out of the way
ss.treecode_sum_device(warm, ss.BiotSavartKernel, cfg, x.data_ptr(), qq.data_ptr(), n, out.data_ptr())
warm.close()
torch.cuda.synchronize()
for label in ("fresh tree, call 1", "call 2", "call 3"):
    if label.startswith("fresh"):
        t = ss.FaceTree(0)
        t.set_stream(torch.cuda.current_stream().cuda_stream)
    t0 = time.perf_counter()
    ss.treecode_sum_device(t, ss.BiotSavartKernel, cfg, x.data_ptr(), qq.data_ptr(), n, out.data_ptr())
    torch.cuda.synchronize()
    print(f"{label}: {1e3 * (time.perf_counter() - t0):.2f} ms", flush=True)
