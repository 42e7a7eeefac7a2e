"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
one tree-code evaluation (both kernels, both tile kernels, the traversal,
the upward / downward passes), one RK4 step and one per-interaction call on
the level-5 mesh.

    compute-sanitizer --tool racecheck python tools/sanitize_step.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2401_07361_b200 as ss  # noqa: E402

level = int(os.environ.get("SAN_LEVEL", "5"))
xyz, area = ss.make_icosa_mesh(level)
zeta = ss.rh4_vorticity(xyz)
q = zeta * area
cfg = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=4, max_depth=10)
t = ss.FaceTree(0)
for k in (ss.BiotSavartKernel, ss.LogPotentialKernel):
    u = ss.treecode_sum(k, xyz, q, cfg, tree=t)  # first call: level-synchronous build, step-by-step traversal
    u = ss.treecode_sum(k, xyz, q, cfg, tree=t)  # warm call: reuse walk, cooperative k_bfs
    assert np.isfinite(u).all()
x1, z1 = ss.rk4(xyz, zeta, area, cfg, dt=0.01, steps=1, tree=t)
lst = ss.dual_traversal_array(t, cfg)
field = np.zeros((xyz.shape[0], 3))
for kind in range(4):
    e = lst[lst[:, 2] == kind][0]
    it = ss.Interaction(int(e[0]), int(e[1]), ss.InteractionKind(kind))
    (ss.eval_pp(ss.BiotSavartKernel, t, it, xyz, q, field) if kind == 0 else
     [ss.eval_pc, ss.eval_pc, ss.eval_cp, ss.eval_cc][kind](ss.BiotSavartKernel, t, it, xyz, q, cfg, field))
ss.direct_sum(ss.BiotSavartKernel, xyz[:2000], q[:2000])
print("sanitize_step ok", xyz.shape[0])
