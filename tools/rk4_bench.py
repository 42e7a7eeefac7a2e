"""Config-4 Lagrangian RK4 on the device (ssum_rk4): velocity evaluations per
second over a few steps on one persistent tree (particles move, the tree is
reused; stage positions and vorticity stay on the device), plus — with
--reference — one RK4 step of the reference driver (oracle/_ref: the
reference's treecode_sum per stage, all host threads) on the same state.
Prints one JSON line. With SSUM_TRACE=1 each evaluation's phases go to stderr
(bin.reuse = walk + sort through the existing tree).

    python tools/rk4_bench.py [--steps 3] [--level 9] [--reference]

(--steps 49: config 4's full 50-step run, the warm-up step included.)
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2401_07361_b200 as ss  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--level", type=int, default=9)
ap.add_argument("--reference", action="store_true")
args = ap.parse_args()

xyz, area = ss.make_icosa_mesh(args.level)
zeta = ss.rh4_vorticity(xyz)
n = xyz.shape[0]
cfg = ss.TraversalConfig(theta=0.7, n_threshold=64, degree=8, max_depth=10)
tree = ss.FaceTree(0)
x0, z0 = ss.rk4(xyz, zeta, area, cfg, dt=0.01, steps=1, tree=tree)  # warm-up step: builds the tree
t0 = time.perf_counter()
x1, z1 = ss.rk4(x0, z0, area, cfg, dt=0.01, steps=args.steps, tree=tree)
dt = time.perf_counter() - t0
evals = 4 * args.steps
line = {"metric": "BVE RK4 velocity evals/s (config 4, fp64)", "value": n * evals / dt, "unit": "velocity_evals/s",
        "n": n, "rk4_steps": args.steps, "evaluations": evals, "ms_per_evaluation": dt * 1e3 / evals,
        "dt": 0.01, "omega": 2 * np.pi,
        "note": "wall time of ss.rk4 (one H2D of x, zeta, A and one D2H at the ends); tree reused across stages"}
# invariants after 1 + steps RK4 steps from the initial state: absolute
# vorticity zeta + 2 Omega z is carried by each particle (d zeta/dt =
# -2 Omega u_z, dz/dt = u_z), and positions stay on the unit sphere
om = 2 * np.pi
drift = np.abs((z1 + 2 * om * x1[:, 2]) - (zeta + 2 * om * xyz[:, 2]))
line["invariants"] = {"rk4_steps_total": 1 + args.steps,
                      "max_abs_vorticity_drift": float(drift.max()),
                      "max_abs_zeta": float(np.abs(zeta).max()),
                      "max_unit_norm_error": float(np.abs(np.linalg.norm(x1, axis=1) - 1.0).max())}
if args.reference:
    import oracle_lib as ol

    if ol.ref_available():
        cores = os.cpu_count() or 1
        t0 = time.perf_counter()
        rx, rz = ol.ref_rk4(x0, z0, area, 0.7, 64, 8, 10, 0.01, 1, 2 * np.pi, workers=cores)
        rdt = time.perf_counter() - t0
        mx, mz = ss.rk4(x0, z0, area, cfg, dt=0.01, steps=1, tree=ss.FaceTree(0))
        line["cpu_baseline"] = {"value": n * 4 / rdt, "unit": "velocity_evals/s", "cores": cores,
                                "kind": "reference", "sample": f"one RK4 step (4 evaluations), {rdt:.1f} s"}
        line["parity_one_step"] = {"x_rel_l2": ol.rel_l2(mx, rx), "zeta_rel_l2": ol.rel_l2(mz, rz)}
print(json.dumps(line))
