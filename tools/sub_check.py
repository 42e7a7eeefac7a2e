"""Subtree list builder (sublists.cu) against the global traversal path
(SSUM_SUB_LISTS=0): bitwise-equal results on a sequence of evaluations of
moving particles, and the device time of each path.

    python tools/sub_check.py [case ...]   (cases: l5 l7 c2 c4 c3s c5)
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2401_07361_b200 as ss  # noqa: E402

CASES = {
    "l5": dict(mesh=5, degree=4, theta=0.7),
    "l7": dict(mesh=7, degree=8, theta=0.7),
    "c2": dict(mesh=8, degree=8, theta=0.7),
    "c4": dict(mesh=9, degree=8, theta=0.7),
    "c3s": dict(cap=1 << 20, degree=8, theta=0.7, step=1e-8),
    "c5": dict(mesh=10, degree=8, theta=0.8, step=2e-5),
}


def inputs(case):
    if "cap" in case:
        xyz, zeta, area = ss.make_random_cap(case["cap"], 5)
    else:
        xyz, area = ss.make_icosa_mesh(case["mesh"])
        zeta = ss.rh4_vorticity(xyz)
    return xyz, zeta * area


def run(case, xyz0, q, calls, sub):
    """sub: True the subtree builder, False the global path, "noplan" the
    global path with traversal-marked slots (SSUM_PLAN_LISTS=0)."""
    os.environ["SSUM_SUB_LISTS"] = "1" if sub is True else "0"
    os.environ["SSUM_PLAN_LISTS"] = "0" if sub == "noplan" else "1"
    dev = torch.device("cuda", 0)
    tree = ss.FaceTree(0)
    tree.set_stream(torch.cuda.current_stream().cuda_stream)
    cfg = ss.TraversalConfig(theta=case["theta"], n_threshold=64, degree=case["degree"], max_depth=10)
    rng = np.random.default_rng(7)
    n = xyz0.shape[0]
    d_q = torch.from_numpy(q).to(dev)
    outs, times = [], []
    x = xyz0.copy()
    for k in range(calls):
        if k >= 2:  # moving particles: a small random step, renormalised
            x = x + case.get("step", 2e-4) * rng.standard_normal(x.shape)
            x /= np.linalg.norm(x, axis=1, keepdims=True)
        d_x = torch.from_numpy(x).to(dev)
        d_out = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ss.treecode_sum_device(tree, ss.BiotSavartKernel, cfg, d_x.data_ptr(), d_q.data_ptr(), n, d_out.data_ptr())
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
        outs.append(d_out.cpu().numpy())
    os.environ.pop("SSUM_SUB_LISTS", None)
    return outs, times


def main():
    names = sys.argv[1:] or ["l5", "l7", "c4", "c3s"]
    ok = True
    for name in names:
        case = CASES[name]
        xyz, q = inputs(case)
        t0 = time.time()
        a, ta = run(case, xyz, q, 6, True)
        b, tb = run(case, xyz, q, 6, False)
        c, tc = run(case, xyz, q, 6, "noplan")
        same = [bool(np.array_equal(x, y) and np.array_equal(x, z)) for x, y, z in zip(a, b, c)]
        ok &= all(same)
        print(f"{name}: N={xyz.shape[0]} bitwise {same} | sub ms {[round(t, 3) for t in ta]} | "
              f"global ms {[round(t, 3) for t in tb]} | global unplanned ms {[round(t, 3) for t in tc]} "
              f"({time.time() - t0:.1f} s)", flush=True)
        if not all(same):
            for k, (x, y) in enumerate(zip(a, b)):
                if not np.array_equal(x, y):
                    d = np.abs(x - y).max()
                    print(f"   call {k}: max |diff| {d:.3e}, rows differing {int(np.any(x != y, axis=1).sum())}")
    print("ALL OK" if ok else "MISMATCH")
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
