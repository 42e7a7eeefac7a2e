"""Full-size golden fixtures from the UNMODIFIED reference (oracle/_ref), for
the BASELINE configs whose reference run is too slow to repeat inside the
GPU test suite. Run here, where /root/reference exists (CPU only):

    python tests/golden/make_golden_full.py c3      # config 3, ~10 min on 8 threads
    python tests/golden/make_golden_full.py rk4c4   # config 4, 50 RK4 steps, ~1 h

Each writes tests/golden/full_<name>.npz holding
  * a hash of the inputs (the test regenerates them and checks the hash),
  * the reference's interaction list as a SHA-256 of its (target, source,
    kind) int32 triples in the reference's emission order and numbering,
    plus the per-kind counts (config 3),
  * the reference's outputs on a seeded sample of rows (all N rows would be
    tens of MB), plus whole-field sums for a size-independent check.
The GPU tests (tests/test_gpu_fullsize.py) compare the CUDA path on the same
inputs against these.
"""
import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, ROOT)
import oracle_lib as ol  # noqa: E402

SAMPLE = 16384
SAMPLE_SEED = 7


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_rows(n):
    return np.sort(np.random.default_rng(SAMPLE_SEED).choice(n, size=min(SAMPLE, n), replace=False))


def rh4(xyz):
    """BASELINE RH4 vorticity (the same numpy expression as make_golden.py)."""
    lat = np.arcsin(np.clip(xyz[:, 2], -1, 1))
    lon = np.arctan2(xyz[:, 1], xyz[:, 0])
    return 2 * np.sin(lat) - 30 * np.sin(lat) * np.cos(lat) ** 4 * np.cos(4 * lon)


def c3():
    import paper_2401_07361_b200 as ss  # host-side fixture generator only (no device)

    n, seed = 1 << 22, 5
    xyz, zeta, area = ss.make_random_cap(n, seed)
    q = zeta * area
    t0 = time.time()
    t = ol.RefTree()
    t.bin(xyz, 64, 10)
    lst = t.traversal(0.7, 64, 8, 10)
    print("c3 list", lst.shape, time.time() - t0, flush=True)
    t0 = time.time()
    u, st = ol.ref_treecode(0, xyz, q, 0.7, 64, 8, 10, os.cpu_count())
    print("c3 treecode", time.time() - t0, flush=True)
    idx = sample_rows(n)
    np.savez_compressed(os.path.join(HERE, "full_c3.npz"), n=n, seed=seed, xyz_sha=sha(xyz), q_sha=sha(q),
                        list_sha=sha(lst.astype(np.int32)), list_len=lst.shape[0],
                        counts=np.bincount(lst[:, 2], minlength=4), idx=idx, u=u[idx], u_sum=u.sum(axis=0),
                        u_norm=np.linalg.norm(u), ref_stats=st)


def rk4c4():
    steps = int(os.environ.get("RK4_STEPS", "50"))
    xyz, a = ol.mesh(9)
    z = rh4(xyz)
    t0 = time.time()
    x1, z1 = ol.ref_rk4(xyz, z, a, 0.7, 64, 8, 10, 0.01, steps, 2 * np.pi, workers=os.cpu_count())
    print("rk4c4", steps, "steps", time.time() - t0, flush=True)
    np.save("/tmp/golden/rk4c4_x.npy", x1)
    np.save("/tmp/golden/rk4c4_z.npy", z1)
    idx = sample_rows(xyz.shape[0])
    np.savez_compressed(os.path.join(HERE, f"full_rk4c4_{steps}.npz"), steps=steps, dt=0.01, omega=2 * np.pi,
                        xyz_sha=sha(xyz), z0_sha=sha(z), area_sha=sha(a), idx=idx, x=x1[idx], z=z1[idx],
                        x_sum=x1.sum(axis=0), z_sum=z1.sum(), z_norm=np.linalg.norm(z1),
                        circ=float((z1 * a).sum()))


if __name__ == "__main__":
    {"c3": c3, "rk4c4": rk4c4}[sys.argv[1]]()
