"""Generate the golden reference vectors in tests/golden/ from the UNMODIFIED
reference (oracle/_ref, compiled from /root/reference/proj/src by
oracle/Makefile). Run here, where /root/reference exists:

    python tests/golden/make_golden.py

The reference ships no tests or fixtures of its own; these
vectors pin the oracle and the CUDA path to the reference's actual outputs.
Inputs are regenerated from the (bit-identical) mesh generator, so only
outputs are stored.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as ol  # noqa: E402


def rh4(xyz):
    lat = np.arcsin(np.clip(xyz[:, 2], -1, 1))
    lon = np.arctan2(xyz[:, 1], xyz[:, 0])
    return 2 * np.sin(lat) - 30 * np.sin(lat) * np.cos(lat) ** 4 * np.cos(4 * lon)


def main():
    out = {}
    # L3, N_T = 8 (SPEC.md:417 pair-coverage config), d = 4, theta = 0.7
    xyz, a = ol.mesh(3)
    q = rh4(xyz) * a
    out["l3_xyz_sha"] = np.frombuffer(xyz.tobytes(), np.uint8).sum()
    out["l3_area"] = a
    out["l3_q"] = q
    u, st = ol.ref_treecode(0, xyz, q, 0.7, 8, 4, 10, 1)
    out["l3_u_tree"] = u
    out["l3_counts"] = st[3:]
    psi, _ = ol.ref_treecode(1, xyz, q, 0.7, 8, 4, 10, 1)
    out["l3_psi_tree"] = psi
    out["l3_u_direct"] = ol.ref_direct(0, xyz, q)
    out["l3_psi_direct"] = ol.ref_direct(1, xyz, q)
    t = ol.RefTree()
    t.bin(xyz, 8, 10)
    out["l3_list"] = t.traversal(0.7, 8, 4, 10)
    e = t.export()
    for k in ("level", "parent", "child_base", "bin_offsets", "bin_ids", "leaf_of", "tri", "center", "radius"):
        out[f"l3_tree_{k}"] = e[k]
    # L4, N_T = 32, d = 6 (the SPEC defaults) for both kernels
    xyz, a = ol.mesh(4)
    q = rh4(xyz) * a
    out["l4_q"] = q
    out["l4_u_tree"], _ = ol.ref_treecode(0, xyz, q, 0.7, 32, 6, 10, 1)
    out["l4_psi_tree"], _ = ol.ref_treecode(1, xyz, q, 0.7, 32, 6, 10, 1)
    # RK4: L3, 2 steps, dt = 0.01, Omega = 2 pi, d = 4, theta = 0.7, N_T = 8
    xyz, a = ol.mesh(3)
    z = rh4(xyz)
    out["l3_rk4_z0"] = z
    x2, z2 = ol.ref_rk4(xyz, z, a, 0.7, 8, 4, 10, 0.01, 2, 2 * np.pi)
    out["l3_rk4_x"] = x2
    out["l3_rk4_z"] = z2
    np.savez_compressed(os.path.join(HERE, "reference_golden.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_golden.npz"), {k: np.shape(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
