"""The C++ drop-in (include/spheresum_b200/spheresum.hpp, libspheresum_dropin.so)
driven the way a reference caller drives spheresum:: — tests/cpp/dropin_test.cpp."""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle_lib as ol

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2401_07361_b200", "lib", "dropin_test")
GOLD = os.path.join(os.path.dirname(__file__), "golden", "reference_golden.npz")


def test_cpp_dropin_matches_reference(tmp_path):
    if not os.path.exists(BIN):
        pytest.fail("dropin_test not built (make -C paper_2401_07361_b200/csrc)")
    g = np.load(GOLD)
    n = 642
    qf = tmp_path / "q.bin"
    of = tmp_path / "out.bin"
    g["l3_q"].astype(np.float64).tofile(qf)
    r = subprocess.run([BIN, str(qf), str(of)], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "singular_threw=1" in r.stdout
    v = np.fromfile(of, dtype=np.float64)
    o = 0

    def take(k):
        nonlocal o
        a = v[o:o + k]
        o += k
        return a

    u = take(3 * n).reshape(n, 3)
    psi = take(n).reshape(n, 1)
    ud = take(3 * n).reshape(n, 3)
    cnt = int(take(1)[0])
    lst = take(3 * cnt).reshape(cnt, 3).astype(np.int32)
    sizes = take(20)
    pp = take(3 * n).reshape(n, 3)
    w = take(15)
    rc8 = take(1)[0]
    const_err = take(1)[0]
    rc16 = take(1)[0]
    geo = take(3)
    x = take(3 * n).reshape(n, 3)
    z = take(n)
    assert o == v.size
    # compute_proxy_weights vs the reference on its own tree of the same input
    xyz, _ = ol.mesh(3)
    t = ol.RefTree()
    t.bin(xyz, 8, 10)
    wr = t.proxy_weights(4, xyz, g["l3_q"], 0)
    assert np.abs(w - wr).max() <= 1e-13 * np.abs(wr).max()
    rcr = ctypes.c_double()
    ol.ref().ref_lattice_fit_rcond(8, ctypes.byref(rcr))
    assert abs(rc8 - rcr.value) <= 1e-8 * rcr.value  # exact 1-norm rcond, both
    assert abs(const_err) < 1e-12
    assert 0.0 <= rc16 <= 1e-12  # ConditioningError carries rcond (errors.hpp:22-27)
    assert geo[0] == 1.0 and geo[1] == 0.0 and geo[2] > 0
    assert ol.rel_l2(u, g["l3_u_tree"]) < 1e-10
    assert ol.rel_l2(psi, g["l3_psi_tree"]) < 1e-10
    assert ol.rel_l2(ud, g["l3_u_direct"]) < 1e-13
    assert np.array_equal(lst, g["l3_list"])
    offs = g["l3_tree_bin_offsets"]
    assert np.array_equal(sizes, (offs[1:21] - offs[:20]).astype(np.float64))
    assert np.abs(pp).max() > 0
    assert ol.rel_l2(x, g["l3_rk4_x"]) < 1e-10
    assert ol.rel_l2(z, g["l3_rk4_z"]) < 1e-10
