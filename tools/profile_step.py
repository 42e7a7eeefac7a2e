"""One warm-up + `reps` config-4 treecode evaluations on device-resident
inputs — the command profiled by ncu (profiles/README.md). No output checks.

    python tools/profile_step.py [reps] [level] [degree] [theta] [log]

`log` evaluates the stream function (LogPotentialKernel) instead.
"""
import sys

import torch

sys.path.insert(0, ".")
import paper_2401_07361_b200 as ss  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
level = int(sys.argv[2]) if len(sys.argv) > 2 else 9
degree = int(sys.argv[3]) if len(sys.argv) > 3 else 8
theta = float(sys.argv[4]) if len(sys.argv) > 4 else 0.7
kernel = ss.LogPotentialKernel if len(sys.argv) > 5 and sys.argv[5] == "log" else ss.BiotSavartKernel
xyz, area = ss.make_icosa_mesh(level)
q = ss.rh4_vorticity(xyz) * area
dev = torch.device("cuda", 0)
d_xyz = torch.from_numpy(xyz).to(dev)
d_q = torch.from_numpy(q).to(dev)
d_out = torch.zeros((xyz.shape[0], 3 if kernel is ss.BiotSavartKernel else 1), dtype=torch.float64, device=dev)
tree = ss.FaceTree(0)
tree.set_stream(torch.cuda.current_stream().cuda_stream)
cfg = ss.TraversalConfig(theta=theta, n_threshold=64, degree=degree, max_depth=10)
for _ in range(1 + reps):
    st = ss.TreecodeStats()
    ss.treecode_sum_device(tree, kernel, cfg, d_xyz.data_ptr(), d_q.data_ptr(), xyz.shape[0],
                           d_out.data_ptr(), stats=st)
torch.cuda.synchronize()
print("ok", st.pp_pc_ms, st.cp_cc_fit_ms, st.upward_ms, st.finish_ms, st.gpu_launches)
