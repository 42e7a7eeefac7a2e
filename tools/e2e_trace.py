"""Phase trace of the host-pointer entry (ssum_treecode_sum) from pinned
buffers at one BASELINE config (bench.py's fixtures; default c4): wall time
of each call, its H2D / D2H seconds and, with SSUM_TRACE=1, the library's
host-side phase marks (stderr).

    SSUM_TRACE=1 python tools/e2e_trace.py [calls] [config]
"""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2401_07361_b200 as ss  # noqa: E402

import bench  # noqa: E402

calls = int(sys.argv[1]) if len(sys.argv) > 1 else 4
bench.use_config(sys.argv[2] if len(sys.argv) > 2 else "c4")
xyz, q, _ = bench.fixture()
n = xyz.shape[0]
h_xyz = torch.from_numpy(xyz).pin_memory()
h_q = torch.from_numpy(q).pin_memory()
h_out = torch.zeros((n, 3), dtype=torch.float64).pin_memory()
cfg = ss.TraversalConfig(**bench.CFG)
tree = ss.FaceTree(0)
for k in range(calls):
    st = ss.TreecodeStats()
    t0 = time.perf_counter()
    ss.treecode_sum(ss.BiotSavartKernel, h_xyz.numpy(), h_q.numpy(), cfg, tree=tree, out=h_out.numpy(), stats=st)
    dt = time.perf_counter() - t0
    print(json.dumps({"call": k, "wall_ms": dt * 1e3, "h2d_ms": st.h2d_seconds * 1e3, "d2h_ms": st.d2h_seconds * 1e3,
                      "bin_ms": st.bin_seconds * 1e3, "trav_ms": st.traversal_seconds * 1e3,
                      "eval_ms": st.eval_seconds * 1e3, "up": st.upward_ms, "fit": st.cp_cc_fit_ms,
                      "pp_pc": st.pp_pc_ms, "finish": st.finish_ms}), flush=True)
