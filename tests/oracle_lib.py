"""ctypes wrappers for the ORACLES (test infrastructure only).

* ref: oracle/_ref/libspheresum_ref.so — the unmodified reference sources
  (/root/reference/proj/src/*.cpp) + Eigen API shim + oracle/ref_capi.cpp.
* orc: oracle/liboracle.so — the C restatement (oracle/spheresum_oracle.c),
  pinned bitwise against `ref` by tests/test_oracle_pin.py.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module. The product never does.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Tuple

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_PATH = os.path.join(ROOT, "oracle", "_ref", "libspheresum_ref.so")
ORC_PATH = os.path.join(ROOT, "oracle", "liboracle.so")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_ref = None
_orc = None


def ref_available() -> bool:
    return os.path.exists(REF_PATH)


def ref():
    global _ref
    if _ref is None:
        lib = ctypes.CDLL(REF_PATH)
        lib.ref_last_error.restype = ctypes.c_char_p
        lib.ref_mesh_vertex_count.restype = _I64
        lib.ref_mesh_vertex_count.argtypes = [ctypes.c_int]
        lib.ref_make_mesh.argtypes = [ctypes.c_int, _P, _P]
        lib.ref_direct_sum.argtypes = [ctypes.c_int, _P, _P, _I64, _P]
        lib.ref_treecode_sum.argtypes = [ctypes.c_int, _P, _P, _I64, _D, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, _P, _P]
        lib.ref_tree_new.restype = _P
        lib.ref_tree_free.argtypes = [_P]
        lib.ref_tree_bin.argtypes = [_P, _P, _I64, ctypes.c_int, ctypes.c_int]
        lib.ref_tree_node_count.argtypes = [_P]
        lib.ref_tree_nodes.argtypes = [_P] + [_P] * 7
        lib.ref_tree_bins.argtypes = [_P, _P, _P]
        lib.ref_tree_leaf_of.argtypes = [_P, _I64, _P]
        lib.ref_dual_traversal.argtypes = [_P, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _I64,
                                           ctypes.POINTER(_I64)]
        lib.ref_treecode_sum_tree.argtypes = [_P, ctypes.c_int, _P, _P, _I64, _D, ctypes.c_int, ctypes.c_int,
                                              ctypes.c_int, ctypes.c_int, _P, _P]
        lib.ref_sbb_eval.argtypes = [ctypes.c_int, _D, _D, _D, _P]
        lib.ref_proxy_points.argtypes = [_P, ctypes.c_int, _P]
        lib.ref_lattice_inverse.argtypes = [ctypes.c_int, _P]
        lib.ref_lattice_fit_rcond.argtypes = [ctypes.c_int, _P]
        lib.ref_kernel_eval.argtypes = [ctypes.c_int, _P, _P, _P]
        lib.ref_rk4.argtypes = [_P, _P, _P, _I64, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                _D, ctypes.c_int, _D, ctypes.c_int]
        _ref = lib
    return _ref


def orc():
    global _orc
    if _orc is None:
        lib = ctypes.CDLL(ORC_PATH)
        lib.orc_treecode_sum.argtypes = [ctypes.c_int, _P, _P, _I64, _D, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, _P, _P]
        lib.orc_direct_sum.argtypes = [ctypes.c_int, _P, _P, _I64, _P]
        lib.orc_build_lists.argtypes = [_P, _I64, _D, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, _P,
                                        _P, _P, _P, _P]
        _orc = lib
    return _orc


def _check(code):
    if code != 0:
        raise OracleError(code, ref().ref_last_error().decode(errors="replace"))


def mesh(level: int) -> Tuple[np.ndarray, np.ndarray]:
    n = ref().ref_mesh_vertex_count(level)
    xyz = np.zeros((n, 3))
    a = np.zeros(n)
    _check(ref().ref_make_mesh(level, _p(xyz), _p(a)))
    return xyz, a


def ref_treecode(kernel: int, xyz, q, theta, nt, degree, max_depth=10, workers=1):
    n = xyz.shape[0]
    d = 3 if kernel == 0 else 1
    out = np.zeros((n, d))
    st = np.zeros(7)
    _check(ref().ref_treecode_sum(kernel, _p(xyz), _p(q), n, theta, nt, degree, max_depth, workers, _p(out),
                                  _p(st)))
    return out, st


def ref_direct(kernel: int, xyz, q):
    n = xyz.shape[0]
    d = 3 if kernel == 0 else 1
    out = np.zeros((n, d))
    _check(ref().ref_direct_sum(kernel, _p(xyz), _p(q), n, _p(out)))
    return out


def orc_rh4(xyz):
    """BASELINE RH4 vorticity (oracle C restatement; glibc)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    z = np.zeros(xyz.shape[0])
    orc().orc_rh4_vorticity.argtypes = [_P, _I64, _P]
    orc().orc_rh4_vorticity(_p(xyz), xyz.shape[0], _p(z))
    return z


def orc_random_cap(n: int, seed: int):
    """BASELINE config-3 point set (xyz, zeta, area), oracle restatement."""
    lib = orc()
    lib.orc_make_random_cap.argtypes = [_I64, ctypes.c_uint64, _P, _P, _P]
    xyz, z, a = np.zeros((n, 3)), np.zeros(n), np.zeros(n)
    code = lib.orc_make_random_cap(n, seed, _p(xyz), _p(z), _p(a))
    if code:
        raise OracleError(code, "orc_make_random_cap failed")
    return xyz, z, a


def orc_treecode(kernel: int, xyz, q, theta, nt, degree, max_depth=10, pc_only=False):
    n = xyz.shape[0]
    d = 3 if kernel == 0 else 1
    out = np.zeros((n, d))
    c4 = np.zeros(4, np.int64)
    code = orc().orc_treecode_sum(kernel, _p(xyz), _p(q), n, theta, nt, degree, max_depth, int(pc_only), _p(out),
                                  _p(c4))
    if code:
        raise OracleError(code, "oracle restatement failed")
    return out, c4


def orc_lists(xyz, theta, nt, max_depth=10, pc_only=False):
    n = xyz.shape[0]
    nc = ctypes.c_int()
    lc = _I64()
    code = orc().orc_build_lists(_p(xyz), n, theta, nt, max_depth, int(pc_only), ctypes.byref(nc), None, None,
                                 None, None, None, ctypes.byref(lc), None)
    if code:
        raise OracleError(code, "oracle restatement failed")
    tsk = np.zeros((max(lc.value, 1), 3), np.int32)
    code = orc().orc_build_lists(_p(xyz), n, theta, nt, max_depth, int(pc_only), ctypes.byref(nc), None, None,
                                 None, None, None, ctypes.byref(lc), _p(tsk))
    return tsk[: lc.value]


class RefTree:
    """The reference's own FaceTree, via oracle/_ref."""

    def __init__(self):
        self.h = ref().ref_tree_new()

    def __del__(self):
        if self.h:
            ref().ref_tree_free(self.h)

    def bin(self, xyz, nt, max_depth):
        _check(ref().ref_tree_bin(self.h, _p(xyz), xyz.shape[0], nt, max_depth))
        self.n = xyz.shape[0]

    def export(self):
        m = ref().ref_tree_node_count(self.h)
        level = np.zeros(m, np.int32)
        parent = np.zeros(m, np.int32)
        child = np.zeros(m, np.int32)
        size = np.zeros(m, np.int32)
        tri = np.zeros((m, 3, 3))
        center = np.zeros((m, 3))
        radius = np.zeros(m)
        _check(ref().ref_tree_nodes(self.h, _p(level), _p(parent), _p(child), _p(size), _p(tri), _p(center),
                                    _p(radius)))
        offs = np.zeros(m + 1, np.int64)
        _check(ref().ref_tree_bins(self.h, _p(offs), None))
        ids = np.zeros(max(int(offs[-1]), 1), np.int32)
        _check(ref().ref_tree_bins(self.h, _p(offs), _p(ids)))
        leaf = np.zeros(self.n, np.int32)
        _check(ref().ref_tree_leaf_of(self.h, self.n, _p(leaf)))
        return dict(level=level, parent=parent, child_base=child, tri=tri, center=center, radius=radius,
                    bin_offsets=offs, bin_ids=ids[: offs[-1]], leaf_of=leaf)

    def traversal(self, theta, nt, degree, max_depth):
        cnt = _I64()
        _check(ref().ref_dual_traversal(self.h, theta, nt, degree, max_depth, None, 0, ctypes.byref(cnt)))
        tsk = np.zeros((max(cnt.value, 1), 3), np.int32)
        _check(ref().ref_dual_traversal(self.h, theta, nt, degree, max_depth, _p(tsk), cnt.value, ctypes.byref(cnt)))
        return tsk[: cnt.value]

    def eval_interaction(self, kernel, xyz, q, theta, nt, degree, max_depth, target, source, kind, field):
        """eval_pp/pc/cp/cc<K> (treecode.cpp:170-244): adds into field in place."""
        lib = ref()
        lib.ref_eval_interaction.argtypes = [_P, ctypes.c_int, _P, _P, _I64, _D, ctypes.c_int, ctypes.c_int,
                                             ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
        _check(lib.ref_eval_interaction(self.h, kernel, _p(xyz), _p(q), xyz.shape[0], theta, nt, degree, max_depth,
                                        int(target), int(source), int(kind), _p(field)))

    def proxy_weights(self, degree, xyz, q, node):
        """compute_proxy_weights (treecode.cpp:79-91) of one node."""
        lib = ref()
        lib.ref_compute_proxy_weights.argtypes = [_P, ctypes.c_int, _P, _P, _I64, ctypes.c_int, _P]
        w = np.zeros((degree + 1) * (degree + 2) // 2)
        _check(lib.ref_compute_proxy_weights(self.h, degree, _p(xyz), _p(q), xyz.shape[0], int(node), _p(w)))
        return w

    def treecode(self, kernel, xyz, q, theta, nt, degree, max_depth=10, workers=1):
        n = xyz.shape[0]
        d = 3 if kernel == 0 else 1
        out = np.zeros((n, d))
        st = np.zeros(7)
        _check(ref().ref_treecode_sum_tree(self.h, kernel, _p(xyz), _p(q), n, theta, nt, degree, max_depth,
                                           workers, _p(out), _p(st)))
        self.n = n
        return out, st


def ref_rk4(xyz, zeta, area, theta, nt, degree, max_depth, dt, steps, omega, direct=False, workers=1):
    x = np.ascontiguousarray(xyz, dtype=np.float64).copy()
    z = np.ascontiguousarray(zeta, dtype=np.float64).copy()
    a = np.ascontiguousarray(area, dtype=np.float64)
    _check(ref().ref_rk4(_p(x), _p(z), _p(a), x.shape[0], theta, nt, degree, max_depth, workers, dt, steps, omega,
                         int(direct)))
    return x, z


def rel_l2(a, b, w: Optional[np.ndarray] = None) -> float:
    """Relative L2 of a against b (area-weighted when w is given: PAPER E)."""
    a = np.asarray(a).reshape(a.shape[0], -1)
    b = np.asarray(b).reshape(b.shape[0], -1)
    num = ((a - b) ** 2).sum(axis=1)
    den = (b ** 2).sum(axis=1)
    if w is not None:
        num = num * w
        den = den * w
    return float(np.sqrt(num.sum() / den.sum()))
