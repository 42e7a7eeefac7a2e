"""Diagnostic run of the CUDA path against the reference oracle (verbose).
Usage: python tools/first_check.py [max_level]"""
import sys
import time
import traceback

import numpy as np

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_2401_07361_b200 as ss  # noqa: E402
import oracle_lib as ol  # noqa: E402


def section(name, fn):
    print(f"== {name}", flush=True)
    t = time.time()
    try:
        fn()
    except Exception:
        traceback.print_exc()
    print(f"   ({time.time() - t:.2f}s)", flush=True)


def fixture(level):
    xyz, a = ss.make_icosa_mesh(level)
    return xyz, ss.rh4_vorticity(xyz) * a, a


def tree_check(level, nt, md):
    xyz, q, a = fixture(level)
    t = ss.FaceTree()
    t.bin_particles(xyz, nt, md)
    e = t.export()
    r = ol.RefTree()
    r.bin(xyz, nt, md)
    f = r.export()
    for k in ("level", "parent", "child_base", "bin_offsets", "bin_ids", "leaf_of", "tri", "center"):
        same = e[k].shape == f[k].shape and np.array_equal(e[k], f[k])
        print(f"   L{level} {k}: {'OK' if same else 'MISMATCH'} {e[k].shape} {f[k].shape}")
    print(f"   radius max abs diff {np.abs(e['radius'] - f['radius']).max():.3e}")
    for theta in (0.7, 0.8, 1e-9):
        cfg = ss.TraversalConfig(theta=theta, n_threshold=nt, degree=4, max_depth=md)
        mine = ss.dual_traversal_array(t, cfg)
        ref = r.traversal(theta, nt, 4, md)
        print(f"   theta={theta} list: {len(mine)} vs {len(ref)} equal={np.array_equal(mine, ref)}")


def parity(level, deg, nt, theta, kernel):
    xyz, q, a = fixture(level)
    st = ss.TreecodeStats()
    t0 = time.time()
    mine = ss.treecode_sum(kernel, xyz, q, ss.TraversalConfig(theta=theta, n_threshold=nt, degree=deg), stats=st)
    t1 = time.time()
    ref, rst = ol.ref_treecode(kernel.id, xyz, q, theta, nt, deg, 10, 8)
    t2 = time.time()
    print(f"   L{level} d={deg} k={kernel.__name__}: relL2={ol.rel_l2(mine, ref):.3e} "
          f"gpu {t1 - t0:.3f}s ref {t2 - t1:.3f}s counts {st.interaction_counts} ref {rst[3:]} "
          f"evals {st.kernel_evals}")


def direct(level, kernel):
    xyz, q, a = fixture(level)
    mine = ss.direct_sum(kernel, xyz, q)
    ref = ol.ref_direct(kernel.id, xyz, q)
    print(f"   L{level} direct {kernel.__name__}: relL2={ol.rel_l2(mine, ref):.3e} "
          f"maxabs={np.abs(mine - ref).max():.3e}")


def timing(level, deg, theta):
    xyz, q, a = fixture(level)
    cfg = ss.TraversalConfig(theta=theta, n_threshold=64, degree=deg)
    tree = ss.FaceTree()
    for rep in range(4):
        st = ss.TreecodeStats()
        t0 = time.time()
        ss.treecode_sum(ss.BiotSavartKernel, xyz, q, cfg, tree=tree, stats=st)
        dt = time.time() - t0
        print(f"   L{level} rep{rep}: wall {dt * 1e3:.1f} ms bin {st.bin_seconds * 1e3:.1f} trav "
              f"{st.traversal_seconds * 1e3:.1f} eval {st.eval_seconds * 1e3:.1f} | up {st.upward_ms:.2f} "
              f"fit {st.cp_cc_fit_ms:.2f} pp {st.pp_pc_ms:.2f} fin {st.finish_ms:.2f} ms | h2d "
              f"{st.h2d_seconds * 1e3:.1f} d2h {st.d2h_seconds * 1e3:.1f} | evals {st.kernel_evals} "
              f"launches {st.gpu_launches}")


if __name__ == "__main__":
    maxl = int(sys.argv[1]) if len(sys.argv) > 1 else 9
    section("tree L3 nt=8", lambda: tree_check(3, 8, 10))
    section("tree L5 nt=64", lambda: tree_check(5, 64, 10))
    section("direct L5 BS", lambda: direct(5, ss.BiotSavartKernel))
    section("direct L5 LOG", lambda: direct(5, ss.LogPotentialKernel))
    section("parity L5 d4", lambda: parity(5, 4, 64, 0.7, ss.BiotSavartKernel))
    section("parity L5 d4 log", lambda: parity(5, 4, 64, 0.7, ss.LogPotentialKernel))
    section("parity L6 d8", lambda: parity(6, 8, 64, 0.7, ss.BiotSavartKernel))
    section("parity L4 theta=1e-9", lambda: parity(4, 4, 32, 1e-9, ss.BiotSavartKernel))
    if maxl >= 7:
        section("tree L7", lambda: tree_check(7, 64, 10))
    section(f"timing L{maxl}", lambda: timing(maxl, 8, 0.7))
