"""Config-4 Lagrangian RK4 on the device (ssum_rk4): wall time per velocity
evaluation over a few steps, with SSUM_TRACE=1 showing which binning path
each evaluation took (bin.reuse = walk + sort through the existing tree,
bin.level = level-synchronous build).

    SSUM_TRACE=1 python tools/rk4_bench.py [steps] [level]
"""
import sys
import time

sys.path.insert(0, ".")
import paper_2401_07361_b200 as ss  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
level = int(sys.argv[2]) if len(sys.argv) > 2 else 9
xyz, area = ss.make_icosa_mesh(level)
zeta = ss.rh4_vorticity(xyz)
cfg = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=8, max_depth=10)
tree = ss.FaceTree(0)
ss.rk4(xyz, zeta, area, cfg, dt=0.01, steps=1, tree=tree)  # warm-up: builds the tree
t0 = time.perf_counter()
x1, z1 = ss.rk4(xyz, zeta, area, cfg, dt=0.01, steps=steps, tree=tree)
dt = time.perf_counter() - t0
evals = 4 * steps
print(f"N={xyz.shape[0]} steps={steps} evaluations={evals}: {dt * 1e3 / evals:.2f} ms/evaluation, "
      f"{xyz.shape[0] * evals / dt:.3e} velocity evals/s (host copies of x, zeta at the ends only)")
