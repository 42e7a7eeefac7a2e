"""B200-native spherical barycentric-Lagrange tree code (arXiv 2401.07361).

Python mirror of the reference's `spheresum` C++ API
(/root/reference/proj/include/spheresum/*.hpp) over the C-ABI in
include/spheresum_b200.h. Names, argument meaning and error behaviour follow
the reference:

    FaceTree                    face_tree.hpp:36-58   (device-resident here)
    TraversalConfig             treecode.hpp:13-20    (+ pc_only, BASELINE cfg 2)
    InteractionKind/Interaction treecode.hpp:22-28
    BiotSavartKernel            kernels.hpp:52-61     (dim 3, prefactor -1/4pi)
    LogPotentialKernel          kernels.hpp:44-50     (dim 1, prefactor 1)
    dual_traversal              treecode.hpp:44-45
    direct_sum                  treecode.hpp:84-86
    treecode_sum                treecode.hpp:93-97
    TreecodeStats               treecode.hpp:75-80
    GeometryError / SingularKernelError / ConditioningError / ConfigError
                                errors.hpp:10-33
    rk4                         SPEC.md:530-547 (absent from the reference code)

Every compute call runs the CUDA path in lib/libspheresum_b200.so. There is
no CPU fallback: importing works without a GPU, but any call that needs the
device raises CudaError when no device (or no library) is present.
"""
from __future__ import annotations

import ctypes
import enum
import os
from dataclasses import dataclass, field
from typing import List, NamedTuple, Optional, Sequence, Tuple

import numpy as np

__all__ = [
    "BiotSavartKernel", "LogPotentialKernel", "TraversalConfig", "TreecodeStats",
    "InteractionKind", "Interaction", "FaceTree", "TreeNode", "dual_traversal",
    "direct_sum", "treecode_sum", "rk4", "make_icosa_mesh", "rh4_vorticity",
    "make_random_cap", "GeometryError", "SingularKernelError", "ConditioningError",
    "ConfigError", "CudaError", "SpheresumError", "library_path", "load_library",
    "mac_well_separated", "eval_pp", "eval_pc", "eval_cp", "eval_cc", "compute_proxy_weights",
    "SBBBasis", "lattice_fit", "proxy_points", "sbb_basis_size",
]

_HERE = os.path.dirname(os.path.abspath(__file__))


def library_path() -> str:
    """lib/libspheresum_b200.so, or $SSUM_LIBRARY (tuning variants)."""
    return os.environ.get("SSUM_LIBRARY") or os.path.join(_HERE, "lib", "libspheresum_b200.so")


# ----------------------------------------------------------------- errors
class SpheresumError(RuntimeError):
    pass


class ConfigError(SpheresumError):
    """Bad run configuration (errors.hpp:30-33)."""


class GeometryError(SpheresumError):
    """Degenerate geometry / particle in no root face (errors.hpp:10-13)."""


class SingularKernelError(SpheresumError):
    """Kernel evaluated at its singularity, 1 - x.y <= 1e-14 (errors.hpp:16-19)."""


class ConditioningError(SpheresumError):
    """Proxy Vandermonde too ill-conditioned (errors.hpp:22-27); `rcond` is the
    reciprocal condition number that failed the > 1e-12 guard."""

    def __init__(self, msg: str = "", rcond: float = 0.0):
        super().__init__(msg)
        self.rcond = rcond


class CudaError(SpheresumError):
    """CUDA runtime failure (no reference equivalent)."""


_STATUS = {
    1: ConfigError, 2: GeometryError, 3: SingularKernelError, 4: ConditioningError,
    5: ValueError, 6: CudaError, 7: CudaError, 8: MemoryError, 9: SpheresumError,
}


# ------------------------------------------------------------------ C-ABI
class _Config(ctypes.Structure):
    _fields_ = [("theta", ctypes.c_double), ("n_threshold", ctypes.c_int), ("degree", ctypes.c_int),
                ("max_depth", ctypes.c_int), ("pc_only", ctypes.c_int)]


class _Stats(ctypes.Structure):
    _fields_ = [("bin_seconds", ctypes.c_double), ("traversal_seconds", ctypes.c_double),
                ("eval_seconds", ctypes.c_double), ("interaction_counts", ctypes.c_uint64 * 4),
                ("h2d_seconds", ctypes.c_double), ("d2h_seconds", ctypes.c_double),
                ("kernel_evals", ctypes.c_uint64 * 4), ("node_count", ctypes.c_int64),
                ("leaf_count", ctypes.c_int64), ("weight_nodes", ctypes.c_int64),
                ("fit_nodes", ctypes.c_int64), ("gpu_launches", ctypes.c_int64),
                ("pp_pc_ms", ctypes.c_double), ("cp_cc_fit_ms", ctypes.c_double),
                ("upward_ms", ctypes.c_double), ("finish_ms", ctypes.c_double),
                ("up_visits", ctypes.c_uint64), ("down_visits", ctypes.c_uint64),
                ("tiles_ms", ctypes.c_double), ("mac_host_decisions", ctypes.c_int64)]


_LIB = None
_P = ctypes.c_void_p
_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy (driver_types.h)
_I64 = ctypes.c_int64

# Every symbol declared in include/spheresum_b200.h (checked by the CPU tests).
EXPORTED_SYMBOLS = (
    "ssum_create", "ssum_destroy", "ssum_last_error", "ssum_set_stream", "ssum_tree_reset",
    "ssum_treecode_sum", "ssum_treecode_sum_device", "ssum_direct_sum", "ssum_direct_sum_device",
    "ssum_bin_particles", "ssum_tree_node_count", "ssum_tree_export", "ssum_dual_traversal",
    "ssum_rk4", "ssum_mesh_vertex_count", "ssum_make_icosa_mesh", "ssum_rh4_vorticity",
    "ssum_make_random_cap", "ssum_fp64_peak", "ssum_probe_log_far", "ssum_set_partition", "ssum_partition_range",
    "ssum_tree_perm", "ssum_eval_interaction", "ssum_rk4_stage_begin", "ssum_rk4_stage_end",
    "ssum_rk4_step_end", "ssum_compute_proxy_weights", "ssum_last_rcond", "ssum_lattice_fit",
    "ssum_proxy_points", "ssum_partition_cuts", "ssum_set_output_order", "ssum_rk4_stage_end_rows",
    "ssum_trim_memory", "ssum_bin_walk_shard", "ssum_rk4_stage_advance_rows",
)


def load_library():
    """Load lib/libspheresum_b200.so (built by __graft_entry__.build()). Raises
    if it is missing: there is no fallback implementation."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = library_path()
    if not os.path.exists(path):
        raise CudaError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    sig = {
        "ssum_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_P)]),
        "ssum_destroy": (None, [_P]),
        "ssum_last_error": (ctypes.c_char_p, [_P]),
        "ssum_set_stream": (ctypes.c_int, [_P, _P]),
        "ssum_tree_reset": (ctypes.c_int, [_P]),
        "ssum_treecode_sum": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_Config), _P, _P, _I64, _P,
                                             ctypes.POINTER(_Stats)]),
        "ssum_treecode_sum_device": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_Config), _P, _P, _I64,
                                                    _P, ctypes.POINTER(_Stats)]),
        "ssum_direct_sum": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _P]),
        "ssum_direct_sum_device": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, _P]),
        "ssum_bin_particles": (ctypes.c_int, [_P, _P, _I64, ctypes.c_int, ctypes.c_int]),
        "ssum_tree_node_count": (ctypes.c_int, [_P, ctypes.POINTER(ctypes.c_int)]),
        "ssum_tree_export": (ctypes.c_int, [_P] + [_P] * 9),
        "ssum_dual_traversal": (ctypes.c_int, [_P, ctypes.POINTER(_Config), _P, _I64,
                                               ctypes.POINTER(_I64)]),
        "ssum_rk4": (ctypes.c_int, [_P, ctypes.POINTER(_Config), _P, _P, _P, _I64, ctypes.c_double,
                                    ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.POINTER(_Stats)]),
        "ssum_mesh_vertex_count": (_I64, [ctypes.c_int]),
        "ssum_make_icosa_mesh": (ctypes.c_int, [ctypes.c_int, _P, _P]),
        "ssum_rh4_vorticity": (ctypes.c_int, [_P, _I64, _P]),
        "ssum_make_random_cap": (ctypes.c_int, [_I64, ctypes.c_uint64, _P, _P, _P]),
        "ssum_fp64_peak": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
        "ssum_probe_log_far": (ctypes.c_int, [_P, _P, _I64, _P]),
        "ssum_set_partition": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int]),
        "ssum_partition_range": (ctypes.c_int, [_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64)]),
        "ssum_tree_perm": (ctypes.c_int, [_P, _P, ctypes.c_int]),
        "ssum_eval_interaction": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(_Config), _P, _P, _I64, ctypes.c_int,
                                                 ctypes.c_int, ctypes.c_int, _P]),
        "ssum_rk4_stage_begin": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double, _I64] + [_P] * 7),
        "ssum_rk4_stage_end": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double, _I64] + [_P] * 5),
        "ssum_rk4_step_end": (ctypes.c_int, [_P, ctypes.c_double, _I64] + [_P] * 4),
        "ssum_compute_proxy_weights": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _I64, ctypes.c_int, _P]),
        "ssum_last_rcond": (ctypes.c_double, [_P]),
        "ssum_lattice_fit": (ctypes.c_int, [ctypes.c_int, _P, _P]),
        "ssum_proxy_points": (ctypes.c_int, [_P, ctypes.c_int, _P]),
        "ssum_partition_cuts": (ctypes.c_int, [_P, _P]),
        "ssum_trim_memory": (ctypes.c_int, [ctypes.c_int]),
        "ssum_bin_walk_shard": (ctypes.c_int, [_P, _P, _I64, _I64, _I64, _I64, ctypes.POINTER(_P), ctypes.POINTER(_P),
                                               ctypes.POINTER(ctypes.c_int)]),
        "ssum_set_output_order": (ctypes.c_int, [_P, ctypes.c_int]),
        "ssum_rk4_stage_end_rows": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double, _I64, _P, _I64] + [_P] * 4),
        "ssum_rk4_stage_advance_rows": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double, ctypes.c_double, _I64, _P,
                                                       _I64] + [_P] * 9),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _raise(code: int, msg: str):
    if code == 0:
        return
    exc = _STATUS.get(code, SpheresumError)
    raise exc(msg)


# ---------------------------------------------------------------- kernels
class BiotSavartKernel:
    """Raw Biot-Savart integrand (x X y)/(1 - x.y) (kernels.hpp:52-61)."""
    id = 0
    dim = 3

    @staticmethod
    def prefactor() -> float:
        return -1.0 / (4.0 * np.pi)


class LogPotentialKernel:
    """Green's function -(1/4pi) log(1 - x.y) (kernels.hpp:44-50)."""
    id = 1
    dim = 1

    @staticmethod
    def prefactor() -> float:
        return 1.0


def _kernel_id(kernel) -> int:
    if kernel in (BiotSavartKernel, "biot_savart", "velocity", 0):
        return 0
    if kernel in (LogPotentialKernel, "log", "stream", 1):
        return 1
    raise ValueError(f"unknown kernel {kernel!r}")


# ----------------------------------------------------------------- config
@dataclass
class TraversalConfig:
    """treecode.hpp:13-20 (defaults identical). pc_only selects the
    particle-cluster-only traversal of BASELINE config 2 (CP->PP, CC->PC)."""
    theta: float = 0.7
    n_threshold: int = 32
    degree: int = 6
    max_depth: int = 10
    pc_only: bool = False

    def validate(self) -> None:  # treecode.cpp:13-20
        if not (0.0 < self.theta <= 1.0):
            raise ConfigError("theta must be in (0, 1]")
        if self.n_threshold < 1:
            raise ConfigError("n_threshold must be >= 1")
        if not (1 <= self.degree <= 20):
            raise ConfigError("degree must be in [1, 20]")
        if not (1 <= self.max_depth <= 40):
            raise ConfigError("max_depth must be in [1, 40]")

    def _c(self) -> _Config:
        return _Config(float(self.theta), int(self.n_threshold), int(self.degree), int(self.max_depth),
                       1 if self.pc_only else 0)


@dataclass
class TreecodeStats:
    """TreecodeStats (treecode.hpp:75-80): *_seconds accumulate across calls."""
    bin_seconds: float = 0.0
    traversal_seconds: float = 0.0
    eval_seconds: float = 0.0
    interaction_counts: List[int] = field(default_factory=lambda: [0, 0, 0, 0])
    kernel_evals: List[int] = field(default_factory=lambda: [0, 0, 0, 0])
    h2d_seconds: float = 0.0
    d2h_seconds: float = 0.0
    node_count: int = 0
    leaf_count: int = 0
    weight_nodes: int = 0
    fit_nodes: int = 0
    gpu_launches: int = 0
    pp_pc_ms: float = 0.0
    cp_cc_fit_ms: float = 0.0
    upward_ms: float = 0.0
    finish_ms: float = 0.0
    up_visits: int = 0      # (particle, weight node) pairs of the upward pass
    down_visits: int = 0    # (particle, fit node) pairs of the downward pass
    tiles_ms: float = 0.0   # CP/CC+fit and PP+PC tiles together (concurrent streams)
    mac_host_decisions: int = 0  # MAC decisions made on the host inside the guard band (context total)

    def _to_c(self) -> _Stats:
        s = _Stats()
        s.bin_seconds, s.traversal_seconds, s.eval_seconds = (self.bin_seconds, self.traversal_seconds,
                                                              self.eval_seconds)
        s.h2d_seconds, s.d2h_seconds = self.h2d_seconds, self.d2h_seconds
        return s

    def _from_c(self, s: _Stats) -> None:
        """*_seconds come back accumulated (the C side adds to the values
        passed in); interaction_counts accumulate here like the reference's
        (treecode.cpp:296); the device detail describes the last call."""
        for name, _ in _Stats._fields_:
            v = getattr(s, name)
            if name == "interaction_counts":
                v = [a + int(x) for a, x in zip(self.interaction_counts, v)]
            elif name == "kernel_evals":
                v = [int(x) for x in v]
            setattr(self, name, v)


class InteractionKind(enum.IntEnum):
    PP = 0
    PC = 1
    CP = 2
    CC = 3


class Interaction(NamedTuple):
    target: int
    source: int
    kind: InteractionKind


class TreeNode(NamedTuple):
    """TreeNode (face_tree.hpp:12-29); triangle is a (3, 3) array of vertices."""
    triangle: np.ndarray
    circumcenter: np.ndarray
    radius: float
    level: int
    parent: int
    child_base: int
    bin: np.ndarray

    def has_children(self) -> bool:
        return self.child_base >= 0

    def size(self) -> int:
        return int(self.bin.size)


def _as_positions(positions) -> np.ndarray:
    p = np.ascontiguousarray(positions, dtype=np.float64)
    if p.ndim != 2 or p.shape[1] != 3:
        raise ValueError("positions must be an (N, 3) array of unit vectors")
    return p


def _as_vector(v, n: int, name: str) -> np.ndarray:
    a = np.ascontiguousarray(v, dtype=np.float64).reshape(-1)
    if a.size != n:
        raise ValueError(f"{name} must have {n} entries")
    return a


# ------------------------------------------------------------------ tree
class FaceTree:
    """FaceTree (face_tree.hpp:36-58). Holds one device context: node
    geometry persists across calls and only grows; bins are rebuilt by every
    bin_particles / treecode_sum call (face_tree.cpp:73-88)."""

    def __init__(self, device: int = 0):
        lib = load_library()
        h = _P()
        rc = lib.ssum_create(int(device), ctypes.byref(h))
        if rc != 0:
            _raise(rc, "ssum_create failed (no usable CUDA device?)")
        self._h = h
        self._lib = lib
        self._cache = None

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ssum_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc == 4:  # SSUM_CONDITIONING carries the failing rcond
            raise ConditioningError(self._lib.ssum_last_error(self._h).decode(errors="replace"),
                                    float(self._lib.ssum_last_rcond(self._h)))
        if rc != 0:
            _raise(rc, self._lib.ssum_last_error(self._h).decode(errors="replace"))

    @property
    def handle(self):
        return self._h

    def fp64_peak_tflops(self, reps: int = 5) -> float:
        """Measured DFMA throughput of this device (the FP64 roofline denominator)."""
        v = ctypes.c_double()
        self._check(self._lib.ssum_fp64_peak(self._h, int(reps), ctypes.byref(v)))
        return v.value

    def probe_log_far(self, x: np.ndarray) -> np.ndarray:
        """The far-pair log of the log kernel (kernels.cuh log_far) on the
        device, for accuracy tests."""
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty_like(x)
        self._check(self._lib.ssum_probe_log_far(self._h, _ptr(x), x.size, _ptr(out)))
        return out

    def set_partition(self, part: int, nparts: int) -> None:
        """Compute only part `part` of `nparts` cost-balanced target ranges
        (multi-GPU strong scaling); see include/spheresum_b200.h."""
        self._check(self._lib.ssum_set_partition(self._h, int(part), int(nparts)))
        self._nparts = int(nparts)

    def partition_range(self) -> Tuple[int, int]:
        b, e = _I64(), _I64()
        self._check(self._lib.ssum_partition_range(self._h, ctypes.byref(b), ctypes.byref(e)))
        return b.value, e.value

    def partition_cuts(self) -> np.ndarray:
        """Every part's tree-position range of the last evaluation (nparts + 1
        positions); identical on every rank."""
        out = np.zeros(getattr(self, "_nparts", 1) + 1, np.int64)
        self._check(self._lib.ssum_partition_cuts(self._h, _ptr(out)))
        return out

    def bin_walk_shard(self, xyz_ptr: int, n: int, i0: int, i1: int, slots: int) -> Tuple[int, int, bool]:
        """Walk particles [i0, i1) of the device positions through the
        existing tree (multi-GPU sharded binning). Returns device pointers to
        the context's per-particle leaf keys (uint64) and leaves (int32), each
        with room for `slots` rows, and whether the walk ran; the caller fills
        the other shards' rows before the next evaluation (dist.sharded_walk)."""
        kp, lp, w = _P(), _P(), ctypes.c_int()
        self._check(self._lib.ssum_bin_walk_shard(self._h, ctypes.c_void_p(xyz_ptr), int(n), int(i0), int(i1),
                                                  int(slots), ctypes.byref(kp), ctypes.byref(lp), ctypes.byref(w)))
        return kp.value or 0, lp.value or 0, bool(w.value)

    def set_output_order(self, tree_order: bool) -> None:
        """Device evaluations write this part's rows in tree order (row r =
        tree position p0 + r) instead of the caller's order."""
        self._check(self._lib.ssum_set_output_order(self._h, 1 if tree_order else 0))

    def rk4_stage_end_rows(self, stage: int, omega: float, n: int, rows: int, width: int, k: int, kz: int,
                           acc: int, accz: int) -> None:
        """rk4_stage_end with u read from the all-gathered tree-order slots of
        every part (device pointers; see ssum_rk4_stage_end_rows)."""
        v = ctypes.c_void_p
        self._check(self._lib.ssum_rk4_stage_end_rows(self._h, int(stage), float(omega), int(n), v(rows),
                                                      int(width), v(k), v(kz), v(acc), v(accz)))

    def rk4_stage_advance_rows(self, stage: int, dt: float, omega: float, n: int, rows: int, width: int, x0: int,
                               z0: int, area: int, acc: int, accz: int, xs: int, q: int, k: int = 0,
                               kz: int = 0) -> None:
        """rk4_stage_end_rows of `stage` fused with rk4_stage_begin of stage + 1
        (device pointers; k / kz optional, 0 = not written; see
        ssum_rk4_stage_advance_rows)."""
        v = lambda p: ctypes.c_void_p(p or None)  # noqa: E731
        self._check(self._lib.ssum_rk4_stage_advance_rows(self._h, int(stage), float(dt), float(omega), int(n),
                                                          v(rows), int(width), v(x0), v(z0), v(area), v(k), v(kz),
                                                          v(acc), v(accz), v(xs), v(q)))

    def perm(self, device_ptr: Optional[int] = None) -> Optional[np.ndarray]:
        """Tree position -> particle index of the last binning (host copy, or
        into a device buffer when device_ptr is given)."""
        if device_ptr is not None:
            self._check(self._lib.ssum_tree_perm(self._h, ctypes.c_void_p(device_ptr), 1))
            return None
        out = np.zeros(getattr(self, "_n", 0), np.int32)
        if out.size:
            self._check(self._lib.ssum_tree_perm(self._h, _ptr(out), 0))
        return out

    # ---- RK4 step pieces on device arrays (ssum_rk4_stage_begin & co.) ----
    def rk4_stage_begin(self, stage: int, dt: float, n: int, x0: int, z0: int, area: int, k: int, kz: int,
                        xs: int, q: int) -> None:
        """Stage positions xs (renormalised) and strengths q = zeta_s A from
        x0, z0 and the previous stage's k, kz (device pointers)."""
        v = ctypes.c_void_p
        self._check(self._lib.ssum_rk4_stage_begin(self._h, int(stage), float(dt), int(n), v(x0), v(z0), v(area),
                                                   v(k), v(kz), v(xs), v(q)))

    def rk4_stage_end(self, stage: int, omega: float, n: int, u: int, k: int, kz: int, acc: int,
                      accz: int) -> None:
        """k = u, kz = -2 omega u_z, accumulated into acc/accz with RK4 weights."""
        v = ctypes.c_void_p
        self._check(self._lib.ssum_rk4_stage_end(self._h, int(stage), float(omega), int(n), v(u), v(k), v(kz),
                                                 v(acc), v(accz)))

    def rk4_step_end(self, dt: float, n: int, x0: int, z0: int, acc: int, accz: int) -> None:
        """x0, z0 advanced by dt/6 (acc, accz); positions renormalised."""
        v = ctypes.c_void_p
        self._check(self._lib.ssum_rk4_step_end(self._h, float(dt), int(n), v(x0), v(z0), v(acc), v(accz)))

    def set_stream(self, stream_ptr: Optional[int]) -> None:
        """Run this tree's work on an external cudaStream_t (e.g.
        torch.cuda.current_stream().cuda_stream). Handle 0 is CUDA's legacy
        default stream (torch's default stream) and is passed on as
        cudaStreamLegacy, so the work stays ordered with torch's; None
        restores the context's own stream."""
        if stream_ptr is None:
            h = None
        else:
            h = int(stream_ptr) or _CUDA_STREAM_LEGACY
        self._check(self._lib.ssum_set_stream(self._h, ctypes.c_void_p(h)))

    def reset(self) -> None:
        """Forget all node geometry (a freshly constructed FaceTree)."""
        self._check(self._lib.ssum_tree_reset(self._h))
        self._cache = None

    def bin_particles(self, positions, n_threshold: int, max_depth: int) -> None:
        p = _as_positions(positions)
        self._check(self._lib.ssum_bin_particles(self._h, _ptr(p), p.shape[0], int(n_threshold),
                                                 int(max_depth)))
        self._n = p.shape[0]
        self._cache = None

    def node_count(self) -> int:
        c = ctypes.c_int()
        self._check(self._lib.ssum_tree_node_count(self._h, ctypes.byref(c)))
        return c.value

    def export(self) -> dict:
        """All nodes in the reference's numbering: level, parent, child_base,
        tri (M,3,3), center (M,3), radius (M,), bin_offsets (M+1,), bin_ids, leaf_of."""
        if self._cache is not None:
            return self._cache
        m = self.node_count()
        n = getattr(self, "_n", 0)
        level = np.zeros(m, np.int32)
        parent = np.zeros(m, np.int32)
        child = np.zeros(m, np.int32)
        tri = np.zeros((m, 3, 3))
        center = np.zeros((m, 3))
        radius = np.zeros(m)
        offs = np.zeros(m + 1, np.int64)
        self._check(self._lib.ssum_tree_export(self._h, _ptr(level), _ptr(parent), _ptr(child), _ptr(tri),
                                               _ptr(center), _ptr(radius), _ptr(offs), None, None))
        ids = np.zeros(max(int(offs[-1]), 1), np.int32)
        leaf = np.zeros(max(n, 1), np.int32)
        self._check(self._lib.ssum_tree_export(self._h, None, None, None, None, None, None, _ptr(offs),
                                               _ptr(ids), _ptr(leaf)))
        self._cache = dict(level=level, parent=parent, child_base=child, tri=tri, center=center,
                           radius=radius, bin_offsets=offs, bin_ids=ids[: offs[-1]], leaf_of=leaf[:n])
        return self._cache

    def node(self, i: int) -> TreeNode:
        e = self.export()
        o = e["bin_offsets"]
        return TreeNode(e["tri"][i], e["center"][i], float(e["radius"][i]), int(e["level"][i]),
                        int(e["parent"][i]), int(e["child_base"][i]), e["bin_ids"][o[i]:o[i + 1]])

    def leaf_of_particle(self, i: int) -> int:
        return int(self.export()["leaf_of"][i])

    def path_of_particle(self, i: int) -> List[int]:
        e = self.export()
        path = []
        nid = int(e["leaf_of"][i])
        while nid >= 0:
            path.append(nid)
            nid = int(e["parent"][nid])
        return path[::-1]


def mac_well_separated(tn: TreeNode, sn: TreeNode, theta: float) -> bool:
    """(r_t + r_s)/R < theta, R = great-circle distance of the circumcenters,
    R = 0 never qualifies (treecode.cpp:22-25). Host-side helper."""
    a, b = np.asarray(tn.circumcenter), np.asarray(sn.circumcenter)
    r = float(np.arctan2(np.linalg.norm(np.cross(a, b)), float(a @ b)))
    return r > 0.0 and (tn.radius + sn.radius) / r < theta


def dual_traversal(target_tree: FaceTree, source_tree: FaceTree, cfg: TraversalConfig) -> List[Interaction]:
    """dual_traversal (treecode.cpp:69-77) on the tree's current bins, in the
    reference's emission order and node numbering. The device traversal is
    single-tree (target_tree is source_tree), as every reference call site."""
    if target_tree is not source_tree:
        raise ValueError("dual_traversal: target and source trees must be the same FaceTree")
    cfg.validate()
    arr = dual_traversal_array(target_tree, cfg)
    return [Interaction(int(t), int(s), InteractionKind(int(k))) for t, s, k in arr]


def dual_traversal_array(tree: FaceTree, cfg: TraversalConfig) -> np.ndarray:
    """(M, 3) int32 array of (target, source, kind) — dual_traversal without
    the Python object per interaction."""
    c = cfg._c()
    count = _I64()
    tree._check(tree._lib.ssum_dual_traversal(tree._h, ctypes.byref(c), None, 0, ctypes.byref(count)))
    out = np.zeros((max(count.value, 1), 3), np.int32)
    tree._check(tree._lib.ssum_dual_traversal(tree._h, ctypes.byref(c), _ptr(out), count.value,
                                              ctypes.byref(count)))
    return out[: count.value]


def _eval_interaction(kernel, tree: FaceTree, it: Interaction, positions, strengths, cfg: TraversalConfig,
                      field: np.ndarray) -> None:
    k = _kernel_id(kernel)
    cfg.validate()
    p = _as_positions(positions)
    n = p.shape[0]
    q = _as_vector(strengths, n, "strengths")
    d = 3 if k == 0 else 1
    if field.dtype != np.float64 or not field.flags.c_contiguous or field.size != n * d:
        raise ValueError(f"field must be a C-contiguous float64 array with {n * d} entries")
    c = cfg._c()
    tree._check(tree._lib.ssum_eval_interaction(tree._h, k, ctypes.byref(c), _ptr(p), _ptr(q), n, int(it.target),
                                                int(it.source), int(it.kind), _ptr(field)))


def eval_pp(kernel, tree: FaceTree, it: Interaction, positions, strengths, field: np.ndarray) -> None:
    """eval_pp<K> (treecode.cpp:170-186): adds raw PP sums of one interaction
    into field (N, dim), no prefactor. The tree must be binned on positions."""
    _eval_interaction(kernel, tree, it, positions, strengths, TraversalConfig(), field)


def eval_pc(kernel, tree: FaceTree, it: Interaction, positions, strengths, cfg: TraversalConfig,
            field: np.ndarray) -> None:
    """eval_pc<K> (treecode.cpp:188-201)."""
    _eval_interaction(kernel, tree, it, positions, strengths, cfg, field)


def eval_cp(kernel, tree: FaceTree, it: Interaction, positions, strengths, cfg: TraversalConfig,
            field: np.ndarray) -> None:
    """eval_cp<K> (treecode.cpp:203-221)."""
    _eval_interaction(kernel, tree, it, positions, strengths, cfg, field)


def eval_cc(kernel, tree: FaceTree, it: Interaction, positions, strengths, cfg: TraversalConfig,
            field: np.ndarray) -> None:
    """eval_cc<K> (treecode.cpp:223-244)."""
    _eval_interaction(kernel, tree, it, positions, strengths, cfg, field)


def trim_memory(device: int = 0) -> None:
    """Return the device-pool blocks destroyed FaceTrees left cached to the
    driver (ssum_trim_memory)."""
    _raise(load_library().ssum_trim_memory(int(device)), "ssum_trim_memory failed")


def sbb_basis_size(degree: int) -> int:
    """(d + 1)(d + 2) / 2 (sbb.hpp:15)."""
    return (degree + 1) * (degree + 2) // 2


class SBBBasis:
    """SBBBasis (sbb.hpp:19-36): B_ijk(b) = b1^i b2^j b3^k over i + j + k = d,
    ordered k ascending, then j ascending (sbb.cpp:13-24)."""

    def __init__(self, degree: int):
        if not (1 <= degree <= 20):
            raise ValueError("SBB degree must be in [1, 20]")
        self._d = int(degree)
        self._idx = np.array([(degree - k - j, j, k) for k in range(degree + 1) for j in range(degree - k + 1)],
                             np.int64)

    def degree(self) -> int:
        return self._d

    def size(self) -> int:
        return self._idx.shape[0]

    def index_set(self) -> np.ndarray:
        return self._idx.copy()

    def eval(self, b) -> np.ndarray:
        """Basis values at barycentric coordinates b = (b1, b2, b3); 0^0 = 1."""
        b = np.asarray(b, dtype=np.float64)
        return b[0] ** self._idx[:, 0] * b[1] ** self._idx[:, 1] * b[2] ** self._idx[:, 2]


def lattice_fit(degree: int) -> Tuple[np.ndarray, float]:
    """lattice_fit(degree) (sbb.cpp:124-138): (V^-1, rcond) of the lattice
    Vandermonde, from the library (the matrix the tree code applies).
    Raises ConditioningError (with rcond) when rcond <= 1e-12."""
    lib = load_library()
    p = sbb_basis_size(degree)
    inv = np.zeros((p, p))
    rc = ctypes.c_double()
    code = lib.ssum_lattice_fit(int(degree), _ptr(inv), ctypes.byref(rc))
    if code == 4:
        raise ConditioningError(f"proxy Vandermonde too ill-conditioned (rcond {rc.value:g})", rc.value)
    _raise(code, "lattice_fit failed (degree must be in [1, 20])")
    return inv, rc.value


def proxy_points(triangle, degree: int) -> np.ndarray:
    """proxy_points(t, degree).points (sbb.cpp:46-66): (P, 3) lattice points of
    a spherical triangle (rows v1, v2, v3), reference rounding."""
    lib = load_library()
    t = np.ascontiguousarray(triangle, dtype=np.float64).reshape(9)
    out = np.zeros((sbb_basis_size(degree), 3))
    _raise(lib.ssum_proxy_points(_ptr(t), int(degree), _ptr(out)), "proxy_points failed")
    return out


def compute_proxy_weights(tree: FaceTree, source_node: int, basis, positions, strengths) -> np.ndarray:
    """compute_proxy_weights (treecode.cpp:79-91): w_k = sum over the source
    node's bin of B_k(beta(x_j)) q_j, on the device. `basis` is an SBBBasis
    or a degree; the tree must be binned on `positions`."""
    degree = basis.degree() if isinstance(basis, SBBBasis) else int(basis)
    p = _as_positions(positions)
    n = p.shape[0]
    q = _as_vector(strengths, n, "strengths")
    w = np.zeros(sbb_basis_size(degree))
    tree._check(tree._lib.ssum_compute_proxy_weights(tree._h, degree, _ptr(p), _ptr(q), n, int(source_node),
                                                     _ptr(w)))
    return w


_DEFAULT_TREES = {}


def _default_tree(device: int = 0) -> FaceTree:
    t = _DEFAULT_TREES.get(device)
    if t is None:
        t = FaceTree(device)
        _DEFAULT_TREES[device] = t
    return t


def direct_sum(kernel, positions, strengths, tree: Optional[FaceTree] = None) -> np.ndarray:
    """direct_sum<K> (treecode.cpp:246-264): exact O(N^2), self excluded by
    index, prefactor applied. Returns (N, dim)."""
    k = _kernel_id(kernel)
    p = _as_positions(positions)
    n = p.shape[0]
    q = _as_vector(strengths, n, "strengths")
    d = 3 if k == 0 else 1
    out = np.zeros((n, d))
    t = tree or _default_tree()
    t._check(t._lib.ssum_direct_sum(t._h, k, _ptr(p), _ptr(q), n, _ptr(out)))
    return out


def _out_buffer(out, n: int, d: int) -> np.ndarray:
    if out is None:
        return np.zeros((n, d))
    if out.dtype != np.float64 or not out.flags.c_contiguous or out.size != n * d:
        raise ValueError(f"out must be a C-contiguous float64 array with {n * d} entries")
    return out


def treecode_sum(kernel, positions, strengths, cfg: TraversalConfig, tree: Optional[FaceTree] = None,
                 workers: int = 1, stats: Optional[TreecodeStats] = None,
                 out: Optional[np.ndarray] = None) -> np.ndarray:
    """treecode_sum<K> (treecode.cpp:266-413): bins into `tree` (mutated),
    traverses, evaluates; returns (N, dim) = prefactor * sum. `workers` is
    accepted for signature parity and ignored (the device is the worker pool).
    `out` may supply the (pinned) result buffer."""
    del workers
    k = _kernel_id(kernel)
    cfg.validate()
    p = _as_positions(positions)
    n = p.shape[0]
    q = _as_vector(strengths, n, "strengths")
    d = 3 if k == 0 else 1
    out = _out_buffer(out, n, d)
    t = tree or _default_tree()
    c = cfg._c()
    s = stats._to_c() if stats is not None else _Stats()
    t._check(t._lib.ssum_treecode_sum(t._h, k, ctypes.byref(c), _ptr(p), _ptr(q), n, _ptr(out),
                                      ctypes.byref(s)))
    t._n = n
    t._cache = None
    if stats is not None:
        stats._from_c(s)
    return out


def treecode_sum_device(tree: FaceTree, kernel, cfg: TraversalConfig, xyz_ptr: int, q_ptr: int, n: int,
                        out_ptr: int, stats: Optional[TreecodeStats] = None) -> None:
    """Device-pointer variant (inputs resident in HBM), e.g. torch tensors'
    data_ptr(). Runs on the tree's stream (see FaceTree.set_stream)."""
    k = _kernel_id(kernel)
    cfg.validate()
    c = cfg._c()
    s = stats._to_c() if stats is not None else _Stats()
    tree._check(tree._lib.ssum_treecode_sum_device(tree._h, k, ctypes.byref(c), ctypes.c_void_p(xyz_ptr),
                                                   ctypes.c_void_p(q_ptr), int(n), ctypes.c_void_p(out_ptr),
                                                   ctypes.byref(s)))
    tree._n = int(n)
    tree._cache = None
    if stats is not None:
        stats._from_c(s)


def direct_sum_device(tree: FaceTree, kernel, xyz_ptr: int, q_ptr: int, n: int, out_ptr: int) -> None:
    k = _kernel_id(kernel)
    tree._check(tree._lib.ssum_direct_sum_device(tree._h, k, ctypes.c_void_p(xyz_ptr), ctypes.c_void_p(q_ptr),
                                                 int(n), ctypes.c_void_p(out_ptr)))


def rk4(positions, zeta, area, cfg: TraversalConfig, dt: float = 0.01, steps: int = 1,
        omega: float = 2.0 * np.pi, direct: bool = False, tree: Optional[FaceTree] = None,
        stats: Optional[TreecodeStats] = None, inplace: bool = False) -> Tuple[np.ndarray, np.ndarray]:
    """Lagrangian RK4 of the BVE: returns (positions, zeta)
    after `steps` steps. dzeta/dt = -2 omega u_z; positions renormalised after
    every stage; one (reused) tree across all stages. inplace=True advances
    the given (C-contiguous float64, e.g. pinned) arrays themselves."""
    cfg.validate()
    p = _as_positions(positions)
    n = p.shape[0]
    z = _as_vector(zeta, n, "zeta")
    if inplace:
        same = lambda a, b: isinstance(b, np.ndarray) and a.ctypes.data == b.ctypes.data  # noqa: E731
        if not (same(p, positions) and same(z, zeta)):
            raise ValueError("inplace rk4 needs C-contiguous float64 positions (N, 3) and zeta (N,)")
    else:
        p, z = p.copy(), z.copy()
    a = _as_vector(area, n, "area")
    t = tree or _default_tree()
    c = cfg._c()
    s = stats._to_c() if stats is not None else _Stats()
    t._check(t._lib.ssum_rk4(t._h, ctypes.byref(c), _ptr(p), _ptr(z), _ptr(a), n, float(dt), int(steps),
                             float(omega), 1 if direct else 0, ctypes.byref(s)))
    if stats is not None:
        stats._from_c(s)
    return p, z


# --------------------------------------------------------------- fixtures
def make_icosa_mesh(level: int, with_areas: bool = True) -> Tuple[np.ndarray, Optional[np.ndarray]]:
    """make_icosa_mesh(level).vertices() and node_patch_areas() (icosa_mesh.cpp:37-133)."""
    lib = load_library()
    n = lib.ssum_mesh_vertex_count(int(level))
    if n < 0:
        raise ValueError("level out of range")
    xyz = np.zeros((n, 3))
    area = np.zeros(n) if with_areas else None
    _raise(lib.ssum_make_icosa_mesh(int(level), _ptr(xyz), _ptr(area)), "mesh generation failed")
    return xyz, area


def rh4_vorticity(xyz) -> np.ndarray:
    """BASELINE Rossby-Haurwitz R=4: 2 sin(lat) - 30 sin(lat) cos^4(lat) cos(4 lon)."""
    lib = load_library()
    p = _as_positions(xyz)
    z = np.zeros(p.shape[0])
    _raise(lib.ssum_rh4_vorticity(_ptr(p), p.shape[0], _ptr(z)), "rh4_vorticity failed")
    return z


def make_random_cap(n: int, seed: int = 12345) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """BASELINE config 3 point set (xyz, zeta, area); see include/spheresum_b200.h."""
    lib = load_library()
    xyz = np.zeros((n, 3))
    z = np.zeros(n)
    a = np.zeros(n)
    _raise(lib.ssum_make_random_cap(int(n), int(seed), _ptr(xyz), _ptr(z), _ptr(a)), "random cap failed")
    return xyz, z, a
