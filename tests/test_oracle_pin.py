"""Pin the oracles (CPU, no GPU): the C restatement (oracle/liboracle.so)
against the unmodified reference (oracle/_ref), both against the committed
golden vectors, and the SPEC.md known-answer tests."""
import os

import numpy as np
import pytest

import oracle_lib as ol

GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def rh4(xyz):
    lat = np.arcsin(np.clip(xyz[:, 2], -1, 1))
    lon = np.arctan2(xyz[:, 1], xyz[:, 0])
    return 2 * np.sin(lat) - 30 * np.sin(lat) * np.cos(lat) ** 4 * np.cos(4 * lon)


needs_ref = pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built")


# ---- golden vectors: the C restatement reproduces the reference's outputs
def test_restatement_matches_golden_l3(gold):
    xyz, _ = ol.mesh(3) if ol.ref_available() else (None, None)
    if xyz is None:
        pytest.skip("needs the mesh generator from oracle/_ref")
    q = gold["l3_q"]
    u, c4 = ol.orc_treecode(0, xyz, q, 0.7, 8, 4, 10)
    assert np.array_equal(u, gold["l3_u_tree"])
    assert np.array_equal(c4, gold["l3_counts"].astype(np.int64))
    psi, _ = ol.orc_treecode(1, xyz, q, 0.7, 8, 4, 10)
    assert np.array_equal(psi, gold["l3_psi_tree"])
    d = np.zeros_like(u)
    assert ol.orc().orc_direct_sum(0, ol._p(xyz), ol._p(q), xyz.shape[0], ol._p(d)) == 0
    assert np.array_equal(d, gold["l3_u_direct"])
    assert np.array_equal(ol.orc_lists(xyz, 0.7, 8), gold["l3_list"])


@needs_ref
def test_reference_reproduces_golden(gold):
    xyz, a = ol.mesh(3)
    assert np.array_equal(a, gold["l3_area"])
    u, _ = ol.ref_treecode(0, xyz, gold["l3_q"], 0.7, 8, 4, 10, 1)
    assert np.array_equal(u, gold["l3_u_tree"])
    xyz4, _ = ol.mesh(4)
    u4, _ = ol.ref_treecode(0, xyz4, gold["l4_q"], 0.7, 32, 6, 10, 1)
    assert np.array_equal(u4, gold["l4_u_tree"])


@needs_ref
@pytest.mark.parametrize("level,nt,deg,theta", [(3, 8, 4, 0.7), (4, 32, 6, 0.7), (5, 64, 4, 0.7), (4, 16, 8, 0.8),
                                                (4, 32, 4, 1e-9)])
@pytest.mark.parametrize("kernel", [0, 1])
def test_restatement_bitwise_equals_reference(level, nt, deg, theta, kernel):
    xyz, a = ol.mesh(level)
    q = rh4(xyz) * a
    r, st = ol.ref_treecode(kernel, xyz, q, theta, nt, deg, 10, 1)
    o, c4 = ol.orc_treecode(kernel, xyz, q, theta, nt, deg, 10)
    assert np.array_equal(r, o)
    assert np.array_equal(st[3:].astype(np.int64), c4)


@needs_ref
@pytest.mark.parametrize("level,nt", [(3, 8), (5, 64), (4, 32)])
def test_restatement_lists_equal_reference(level, nt):
    xyz, _ = ol.mesh(level)
    t = ol.RefTree()
    t.bin(xyz, nt, 10)
    for theta in (0.7, 0.8, 0.3):
        assert np.array_equal(t.traversal(theta, nt, 4, 10), ol.orc_lists(xyz, theta, nt))


@needs_ref
def test_pc_only_is_reference_list_with_kinds_remapped():
    """PC-only mode (BASELINE config 2, not in the reference): the reference
    recursion with CP->PP and CC->PC."""
    xyz, _ = ol.mesh(5)
    t = ol.RefTree()
    t.bin(xyz, 64, 10)
    ref = t.traversal(0.7, 64, 4, 10).copy()
    ref[ref[:, 2] == 2, 2] = 0
    ref[ref[:, 2] == 3, 2] = 1
    assert np.array_equal(ol.orc_lists(xyz, 0.7, 64, pc_only=True), ref)


@needs_ref
def test_pc_only_accuracy_not_worse_than_cc():
    xyz, a = ol.mesh(5)
    q = rh4(xyz) * a
    d = ol.ref_direct(0, xyz, q)
    cc, _ = ol.orc_treecode(0, xyz, q, 0.7, 64, 4, 10)
    pc, _ = ol.orc_treecode(0, xyz, q, 0.7, 64, 4, 10, pc_only=True)
    assert ol.rel_l2(pc, d, a) <= ol.rel_l2(cc, d, a) * 1.05


# ---- SPEC.md known-answer tests, on the reference itself
@needs_ref
def test_kat_velocity_kernel():
    out = np.zeros(3)
    x = np.array([1.0, 0, 0])
    y = np.array([0, 1.0, 0])
    assert ol.ref().ref_kernel_eval(0, ol._p(x), ol._p(y), ol._p(out)) == 0
    assert np.array_equal(out, [0, 0, 1.0])


@needs_ref
def test_kat_log_antipodal():
    out = np.zeros(3)
    x = np.array([0, 0, 1.0])
    y = np.array([0, 0, -1.0])
    assert ol.ref().ref_kernel_eval(1, ol._p(x), ol._p(y), ol._p(out)) == 0
    assert out[0] == -np.log(2.0) / (4 * np.pi)


@needs_ref
def test_kat_singular_throws():  # kernels.hpp:27-29
    out = np.zeros(3)
    x = np.array([0, 0, 1.0])
    assert ol.ref().ref_kernel_eval(0, ol._p(x), ol._p(x), ol._p(out)) == 3


@needs_ref
def test_kat_sbb_basis_d2():
    out = np.zeros(6)
    assert ol.ref().ref_sbb_eval(2, 0.5, 0.5, 0.0, ol._p(out)) == 0
    assert np.allclose(out, [0.25, 0.25, 0.25, 0, 0, 0], atol=0)


@needs_ref
@pytest.mark.parametrize("deg", [2, 4, 6, 8])
def test_kat_identity_system(deg):  # V alpha = e_m  =>  alpha = e_m
    p = (deg + 1) * (deg + 2) // 2
    inv = np.zeros(p * p)
    assert ol.ref().ref_lattice_inverse(deg, ol._p(inv)) == 0
    vinv = inv.reshape(p, p).T  # column-major -> row-major
    # rebuild V from the basis at the lattice points and check V^-1 V = I
    V = np.zeros((p, p))
    m = 0
    bary = []
    for k in range(deg + 1):
        for j in range(deg - k + 1):
            bary.append(((deg - k - j) / deg, j / deg, k / deg))
    for r, b in enumerate(bary):
        row = np.zeros(p)
        assert ol.ref().ref_sbb_eval(deg, b[0], b[1], b[2], ol._p(row)) == 0
        V[r] = row
    assert np.abs(vinv @ V - np.eye(p)).max() < 1e-8


@needs_ref
def test_kat_theta_zero_is_direct_sum(gold):
    xyz, a = ol.mesh(4)
    q = rh4(xyz) * a
    for k in (0, 1):
        t, st = ol.ref_treecode(k, xyz, q, 1e-9, 32, 4, 10, 1)
        assert st[4] == st[5] == st[6] == 0
        assert np.array_equal(t, ol.ref_direct(k, xyz, q))


@needs_ref
def test_kat_pair_coverage_once(gold):
    """Expanding the L3 / N_T = 8 list covers every ordered pair exactly once."""
    e = {k[len("l3_tree_"):]: gold[k] for k in gold.files if k.startswith("l3_tree_")}
    lst = gold["l3_list"]
    n = 642
    offs, ids = e["bin_offsets"], e["bin_ids"]
    cover = np.zeros((n, n), np.int32)
    for t, s, _ in lst:
        bt = ids[offs[t]:offs[t + 1]]
        bs = ids[offs[s]:offs[s + 1]]
        cover[np.ix_(bt, bs)] += 1
    assert (cover == 1).all()


@needs_ref
def test_kat_area_sum_4pi():
    for level in range(6):
        _, a = ol.mesh(level)
        assert abs(a.sum() - 4 * np.pi) < 1e-10
        assert (a > 0).all()
        assert a.size == 10 * 4 ** level + 2


@needs_ref
def test_tree_error_vs_direct_bar_l5():  # SPEC.md:470,851 (E <= 1e-3 at level 5)
    xyz, a = ol.mesh(5)
    q = rh4(xyz) * a
    t, _ = ol.ref_treecode(0, xyz, q, 0.7, 64, 4, 10, 8)
    d = ol.ref_direct(0, xyz, q)
    assert ol.rel_l2(t, d, a) < 1e-3


@needs_ref
def test_rk4_golden(gold):
    xyz, a = ol.mesh(3)
    x, z = ol.ref_rk4(xyz, gold["l3_rk4_z0"], a, 0.7, 8, 4, 10, 0.01, 2, 2 * np.pi)
    assert np.array_equal(x, gold["l3_rk4_x"])
    assert np.array_equal(z, gold["l3_rk4_z"])
    assert np.abs(np.linalg.norm(x, axis=1) - 1).max() < 1e-15
