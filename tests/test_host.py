"""Host-side logic of the product (CPU, no GPU): the C-ABI library loads and
exports every symbol include/spheresum_b200.h declares, the fixture
generators reproduce the reference's inputs bit for bit, the config/error
mapping mirrors the reference, and the product fails loudly without a device."""
import os
import re

import numpy as np
import pytest

import oracle_lib as ol

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "spheresum_b200.h")).read()
    return sorted(set(re.findall(r"\b(ssum_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol(ss):
    lib = ss.load_library()
    syms = header_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(ss.EXPORTED_SYMBOLS)


def test_library_is_sm100a(ss):
    out = os.popen(f"cuobjdump -lelf {ss.library_path()} 2>/dev/null").read()
    assert "sm_100a" in out


def test_no_device_fails_loudly(ss):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(ss.CudaError):
        ss.FaceTree(0)


def test_config_validation_mirrors_reference(ss):  # treecode.cpp:13-20
    ss.TraversalConfig().validate()
    for bad in (dict(theta=0.0), dict(theta=1.5), dict(n_threshold=0), dict(degree=0), dict(degree=21),
                dict(max_depth=0), dict(max_depth=41)):
        with pytest.raises(ss.ConfigError):
            ss.TraversalConfig(**bad).validate()
    c = ss.TraversalConfig()
    assert (c.theta, c.n_threshold, c.degree, c.max_depth) == (0.7, 32, 6, 10)


def test_kernel_descriptors(ss):
    assert ss.BiotSavartKernel.dim == 3 and ss.LogPotentialKernel.dim == 1
    assert ss.BiotSavartKernel.prefactor() == -1.0 / (4.0 * np.pi)
    assert ss.LogPotentialKernel.prefactor() == 1.0


def test_mac_arithmetic(ss):
    def node(c, r):
        return ss.TreeNode(np.eye(3), np.asarray(c, float), r, 0, -1, -1, np.zeros(0, np.int32))

    a = node([1, 0, 0], 0.2)
    b = node([np.cos(1.0), np.sin(1.0), 0], 0.2)  # R = 1: (0.2+0.2)/1 = 0.4 < 0.7
    assert ss.mac_well_separated(a, b, 0.7)
    c = node([np.cos(1.0), np.sin(1.0), 0], 0.6)  # 0.8 > 0.7
    assert not ss.mac_well_separated(a, c, 0.7)
    assert not ss.mac_well_separated(a, a, 0.7)  # R = 0 never qualifies


@pytest.mark.skipif(not ol.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("level", [0, 1, 2, 4, 6])
def test_mesh_bit_identical_to_reference(ss, level):
    xyz, a = ss.make_icosa_mesh(level)
    rx, ra = ol.mesh(level)
    assert np.array_equal(xyz, rx)
    assert np.array_equal(a, ra)
    assert xyz.shape[0] == 10 * 4 ** level + 2
    assert abs(a.sum() - 4 * np.pi) < 1e-10


def test_rh4_field(ss):
    xyz, a = ss.make_icosa_mesh(4)
    z = ss.rh4_vorticity(xyz)
    lat = np.arcsin(np.clip(xyz[:, 2], -1, 1))
    lon = np.arctan2(xyz[:, 1], xyz[:, 0])
    expect = 2 * np.sin(lat) - 30 * np.sin(lat) * np.cos(lat) ** 4 * np.cos(4 * lon)
    assert np.allclose(z, expect, rtol=0, atol=1e-12)
    assert abs((z * a).sum()) < 1e-10  # SPEC.md test_cases invariant (zero circulation)


def test_random_cap_generator(ss):
    n = 1 << 15
    x1, z1, a1 = ss.make_random_cap(n, 99)
    x2, z2, a2 = ss.make_random_cap(n, 99)
    assert np.array_equal(x1, x2) and np.array_equal(z1, z2)
    x3, _, _ = ss.make_random_cap(n, 100)
    assert not np.array_equal(x1, x3)
    assert np.abs(np.linalg.norm(x1, axis=1) - 1).max() < 1e-15
    assert np.allclose(a1, 4 * np.pi / n)
    assert abs((z1 * a1).sum()) < 1e-12
    lat0 = np.deg2rad(40.0)
    x0 = np.array([np.cos(lat0), 0.0, np.sin(lat0)])
    cap = x1[n // 2:]
    assert (cap @ x0 >= np.cos(np.deg2rad(10.0)) - 1e-12).all()  # second half inside the 10 deg cap
    # near-duplicate policy: no pair with 1 - x.y <= 1e-12
    from scipy.spatial import cKDTree

    pairs = cKDTree(x1).query_pairs(2e-6, output_type="ndarray")
    if len(pairs):
        den = 1.0 - np.einsum("ij,ij->i", x1[pairs[:, 0]], x1[pairs[:, 1]])
        assert (den > 1e-12).all()


def test_random_cap_policy_removes_duplicates(ss):
    # 2^18 points: the cap half is dense enough that the raw draw contains pairs below 1e-12
    n = 1 << 18
    x, _, _ = ss.make_random_cap(n, 3)
    from scipy.spatial import cKDTree

    pairs = cKDTree(x).query_pairs(2e-6, output_type="ndarray")
    if len(pairs):
        den = 1.0 - np.einsum("ij,ij->i", x[pairs[:, 0]], x[pairs[:, 1]])
        assert (den > 1e-12).all()


# --------------------------------------------------- SBB host entry points
@pytest.mark.parametrize("deg", [1, 4, 8, 12])
def test_lattice_fit_matches_reference(ss, ol, deg):  # sbb.cpp:74-138
    """V^-1 and rcond of the lattice Vandermonde (the matrix the tree code's
    fit and V^-T transforms apply) against the reference's ProxyFit."""
    import ctypes

    inv, rc = ss.lattice_fit(deg)
    p = ss.sbb_basis_size(deg)
    ref = np.zeros(p * p)
    assert ol.ref().ref_lattice_inverse(deg, ol._p(ref)) == 0
    ref = ref.reshape(p, p).T  # column-major solve of I
    assert np.abs(inv - ref).max() <= 1e-12 * np.abs(ref).max()
    rcr = ctypes.c_double()
    assert ol.ref().ref_lattice_fit_rcond(deg, ctypes.byref(rcr)) == 0
    assert abs(rc - rcr.value) <= 1e-8 * rcr.value


def test_lattice_fit_conditioning_error_carries_rcond(ss):  # sbb.cpp:89-93, errors.hpp:22-27
    with pytest.raises(ss.ConditioningError) as e:
        ss.lattice_fit(16)
    assert 0.0 <= e.value.rcond <= 1e-12
    with pytest.raises(ValueError):
        ss.lattice_fit(21)


@pytest.mark.parametrize("deg", [2, 4, 8])
def test_proxy_points_bit_identical(ss, ol, deg):  # sbb.cpp:46-66
    rng = np.random.default_rng(deg)
    # vertices whose UnitVector3 renormalisation (inside the reference helper)
    # is the identity, so both sides see the same bits
    tri = np.array([[1.0, 0.0, 0.0], [0.6, 0.8, 0.0], [0.0, 0.6, 0.8]])
    assert np.array_equal(np.sqrt(tri[:, 0] * tri[:, 0] + tri[:, 1] * tri[:, 1] + tri[:, 2] * tri[:, 2]), np.ones(3))
    mine = ss.proxy_points(tri, deg)
    ref = np.zeros((ss.sbb_basis_size(deg), 3))
    assert ol.ref().ref_proxy_points(ol._p(np.ascontiguousarray(tri)), deg, ol._p(ref)) == 0
    assert np.array_equal(mine, ref)
    b = ss.SBBBasis(deg)
    assert b.size() == ss.sbb_basis_size(deg)
    vals = b.eval(rng.dirichlet([1, 1, 1]))
    assert vals.shape == (b.size(),) and np.isfinite(vals).all()


def test_oracle_fixtures_bit_identical_to_product(ss):
    """bench.py's reference arm builds its inputs without the product library
    (reference mesh + the oracle's RH4 / random-cap restatements); they must
    be the product's inputs bit for bit."""
    xyz, _ = ol.mesh(5)
    assert np.array_equal(ol.orc_rh4(xyz), ss.rh4_vorticity(xyz))
    for n, seed in ((1 << 14, 5), (1 << 17, 3)):
        a = ol.orc_random_cap(n, seed)
        b = ss.make_random_cap(n, seed)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)
