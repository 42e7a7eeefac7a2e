// Pair interactions of the two reference kernels (kernels.hpp:13-61), written
// for the sm_100a FP64 pipe.
//
// Biot-Savart: K(x, y) q = q (x X y)/(1 - x.y). Summed over sources as
//   S = sum_j r_j y_j   (well-separated pairs),   r_j = q_j / (1 - x.y_j)
//   S = sum_j r_j (y_j - x)  (near pairs),
// and finished once per target as u = -1/(4 pi) x X S (x X x = 0, so both
// forms give the same cross product). 13 algorithmic flops per pair
// (SURVEY.md §8(d)); the fast path issues 10 FP64 instructions + 1 MUFU:
//   den = fma(-z, y.z, fma(-y, y.y, fma(-x, y.x, 1)))      3 DFMA
//   r0 = rcp.approx(den); e = 1 - den r0; e += e^2;       MUFU + 2 DFMA
//   r = q r0 (1 + e)                                       1 DMUL + 1 DFMA
//   S += r y                                               3 DFMA
// rcp.approx.ftz.f64 is ~2^-20 accurate (measured 9.9e-7 on the box); the
// cubic step brings it to ~1e-18 before rounding.
//
// Near pairs (den < 2^-20, or a self pair) take the reference-rounded slow
// path: den = 1 - ((x.x y.x + x.y y.y) + x.z y.z)
// with separately rounded ops, exactly as the reference computes it, the
// singular guard den <= 1e-14 (kernels.hpp:19,27-29) on that exact value, and
// the Sterbenz-exact (y - x) accumulation. Self pairs are excluded by index
// (treecode.cpp:388). For |den - den_ref| <= ~4.4e-16 the fast path's relative
// deviation per term is below 3e-11 at the threshold and falls as 1/den.
//
// Log potential: K(x, y) q = -q log(1 - x.y)/(4 pi); S = sum_j q_j log(den_j),
// finished as -S/(4 pi).
#pragma once

#include "internal.cuh"

namespace ssum {

constexpr int kBS = 0;
constexpr int kLOG = 1;
template <int KER>
struct KDim {
  static constexpr int D = (KER == kBS) ? 3 : 1;
};

// hi word of 2^-20: den < 2^-20 ~ 9.5e-7 (or negative) <=> (int)hi(den) < kNearHi.
// Below it the fast denominator's absolute error (<= ~4.4e-16 against the
// reference's rounding) is no longer negligible relative to den; above it
// the per-term deviation is < 5e-10 and, weighted by the term's share of the
// sum, far below the 1e-10 output tolerance.
constexpr int kNearHi = 0x3EB00000;

__device__ __forceinline__ double rcp_approx(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  return r;
}

// q / den, relative error ~1e-16 for den in (1e-300, 4]
__device__ __forceinline__ double q_over(double q, double den) {
  const double r0 = rcp_approx(den);
  double e = fma(-den, r0, 1.0);
  e = fma(e, e, e);
  const double y0 = q * r0;
  return fma(y0, e, y0);
}

template <int KER>
struct Acc {
  double s[KDim<KER>::D];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int d = 0; d < KDim<KER>::D; ++d) s[d] = 0.0;
  }
};

// Well-separated pair (PC, CP, CC, and PP pairs past the near threshold).
template <int KER>
__device__ __forceinline__ void pair_far(double x0, double x1, double x2, const double4& y, Acc<KER>& a) {
  const double den = fma(-x2, y.z, fma(-x1, y.y, fma(-x0, y.x, 1.0)));
  if constexpr (KER == kBS) {
    const double r = q_over(y.w, den);
    a.s[0] = fma(r, y.x, a.s[0]);
    a.s[1] = fma(r, y.y, a.s[1]);
    a.s[2] = fma(r, y.z, a.s[2]);
  } else {
    a.s[0] = fma(y.w, log(den), a.s[0]);
  }
}

// The reference-rounded slow path of one pair whose
// fast denominator fell below the near threshold, or a self pair. Returns the
// pair's contribution r (y - x) (BS) or q log(den) (log); zero when skipped.
template <int KER>
__device__ __forceinline__ void pair_slow(double x0, double x1, double x2, const double4& y, int i, int j,
                                          double* c, int* flags) {
#pragma unroll
  for (int d = 0; d < KDim<KER>::D; ++d) c[d] = 0.0;
  if (i == j) return;  // self pair (treecode.cpp:388, :257)
  // reference rounding: 1.0 - dot(x, y) (kernels.hpp:26, geometry.hpp:68-70)
  const double den = __dsub_rn(1.0, __dadd_rn(__dadd_rn(__dmul_rn(x0, y.x), __dmul_rn(x1, y.y)), __dmul_rn(x2, y.z)));
  if (den <= kSingularTol) {
    atomicOr(flags, kFlagSingular);
    return;
  }
  if constexpr (KER == kBS) {
    const double r = __ddiv_rn(y.w, den);
    c[0] = r * __dsub_rn(y.x, x0);
    c[1] = r * __dsub_rn(y.y, x1);
    c[2] = r * __dsub_rn(y.z, x2);
  } else {
    c[0] = y.w * log(den);
  }
}

// Four independent sources per step (y[q] = B[k + q*G]): four separate
// dependency chains with no branch between them, so the scheduler can
// interleave them. NEAR adds one warp vote per quad; a quad with any near
// lane replays its four pairs through the exact per-pair path.
template <int KER, bool NEAR>
__device__ __forceinline__ void pair_quad(double x0, double x1, double x2, const double4* __restrict__ B,
                                          const int* __restrict__ J, int k, int G, int i, Acc<KER>& a, int* flags) {
  double4 y[4];
  double den[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    y[q] = B[k + q * G];
    den[q] = fma(-x2, y[q].z, fma(-x1, y[q].y, fma(-x0, y[q].x, 1.0)));
  }
  if constexpr (NEAR) {
    bool nr = false;
#pragma unroll
    for (int q = 0; q < 4; ++q) nr |= __double2hiint(den[q]) < kNearHi;
    if (__any_sync(0xffffffffu, nr)) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        double c[KDim<KER>::D];
        if (__double2hiint(den[q]) < kNearHi) {
          pair_slow<KER>(x0, x1, x2, y[q], i, J[k + q * G], c, flags);
        } else if constexpr (KER == kBS) {
          const double r = q_over(y[q].w, den[q]);
          c[0] = r * y[q].x;
          c[1] = r * y[q].y;
          c[2] = r * y[q].z;
        } else {
          c[0] = y[q].w * log(den[q]);
        }
#pragma unroll
        for (int d = 0; d < KDim<KER>::D; ++d) a.s[d] += c[d];
      }
      return;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if constexpr (KER == kBS) {
      const double r = q_over(y[q].w, den[q]);
      a.s[0] = fma(r, y[q].x, a.s[0]);
      a.s[1] = fma(r, y[q].y, a.s[1]);
      a.s[2] = fma(r, y[q].z, a.s[2]);
    } else {
      a.s[0] = fma(y[q].w, log(den[q]), a.s[0]);
    }
  }
}

// NS sources x NT targets of well-separated pairs, written stage by stage
// across the NS*NT independent chains (all denominators, then all
// reciprocal seeds, then each Newton step, then the accumulations) so that
// consecutive instructions belong to different chains and the in-order
// issue never waits on a DFMA (8.8 cycles) or MUFU.RCP64H (~24 cycles)
// result it just produced.
// NEAR: the block may hold near pairs (self pairs, 1 - x.y < 2^-20): one warp
// vote for the whole block; a block with a near lane replays its pairs
// through the per-pair exact path (ti: target indices, J: source indices).
template <int KER, int NT, int NS, bool NEAR = false>
__device__ __forceinline__ void far_block(const double4* x, const double4* __restrict__ B, int k, int G, Acc<KER>* a,
                                          const int* ti = nullptr, const int* __restrict__ J = nullptr,
                                          int* flags = nullptr) {
  constexpr int C = NT * NS;
  double4 y[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) y[s] = B[k + s * G];
  double den[C];
#pragma unroll
  for (int c = 0; c < C; ++c) den[c] = fma(-x[c % NT].x, y[c / NT].x, 1.0);
#pragma unroll
  for (int c = 0; c < C; ++c) den[c] = fma(-x[c % NT].y, y[c / NT].y, den[c]);
#pragma unroll
  for (int c = 0; c < C; ++c) den[c] = fma(-x[c % NT].z, y[c / NT].z, den[c]);
  if constexpr (NEAR) {
    bool nr = false;
#pragma unroll
    for (int c = 0; c < C; ++c) nr |= __double2hiint(den[c]) < kNearHi;
    if (__any_sync(0xffffffffu, nr)) {
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double v[KDim<KER>::D];
        const double4& yy = y[c / NT];
        if (__double2hiint(den[c]) < kNearHi) {
          pair_slow<KER>(x[c % NT].x, x[c % NT].y, x[c % NT].z, yy, ti[c % NT], J[k + (c / NT) * G], v, flags);
        } else if constexpr (KER == kBS) {
          const double r = q_over(yy.w, den[c]);
          v[0] = r * yy.x;
          v[1] = r * yy.y;
          v[2] = r * yy.z;
        } else {
          v[0] = yy.w * log(den[c]);
        }
#pragma unroll
        for (int d = 0; d < KDim<KER>::D; ++d) a[c % NT].s[d] += v[d];
      }
      return;
    }
  }
  if constexpr (KER == kBS) {
    double r[C], e[C];
#pragma unroll
    for (int c = 0; c < C; ++c) r[c] = rcp_approx(den[c]);
#pragma unroll
    for (int c = 0; c < C; ++c) e[c] = fma(-den[c], r[c], 1.0);
#pragma unroll
    for (int c = 0; c < C; ++c) e[c] = fma(e[c], e[c], e[c]);
#pragma unroll
    for (int c = 0; c < C; ++c) r[c] = y[c / NT].w * r[c];
#pragma unroll
    for (int c = 0; c < C; ++c) r[c] = fma(r[c], e[c], r[c]);
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[0] = fma(r[c], y[c / NT].x, a[c % NT].s[0]);
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[1] = fma(r[c], y[c / NT].y, a[c % NT].s[1]);
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[2] = fma(r[c], y[c / NT].z, a[c % NT].s[2]);
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[0] = fma(y[c / NT].w, log(den[c]), a[c % NT].s[0]);
  }
}

// One source against NT register-tiled targets with a single warp vote: the
// NT denominator chains are independent, so they interleave; only a source
// with a near lane (self pair or 1 - x.y < 2^-20) takes the exact path.
template <int KER, int NT>
__device__ __forceinline__ void source_near(const double4* x, const double4& y, const int* ti, int j, Acc<KER>* a,
                                            int* flags) {
  double den[NT];
  bool nr = false;
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    den[q] = fma(-x[q].z, y.z, fma(-x[q].y, y.y, fma(-x[q].x, y.x, 1.0)));
    nr |= __double2hiint(den[q]) < kNearHi;
  }
  if (__any_sync(0xffffffffu, nr)) {
#pragma unroll
    for (int q = 0; q < NT; ++q) {
      double c[KDim<KER>::D];
      if (__double2hiint(den[q]) < kNearHi) {
        pair_slow<KER>(x[q].x, x[q].y, x[q].z, y, ti[q], j, c, flags);
      } else if constexpr (KER == kBS) {
        const double r = q_over(y.w, den[q]);
        c[0] = r * y.x;
        c[1] = r * y.y;
        c[2] = r * y.z;
      } else {
        c[0] = y.w * log(den[q]);
      }
#pragma unroll
      for (int d = 0; d < KDim<KER>::D; ++d) a[q].s[d] += c[d];
    }
    return;
  }
#pragma unroll
  for (int q = 0; q < NT; ++q) {
    if constexpr (KER == kBS) {
      const double r = q_over(y.w, den[q]);
      a[q].s[0] = fma(r, y.x, a[q].s[0]);
      a[q].s[1] = fma(r, y.y, a[q].s[1]);
      a[q].s[2] = fma(r, y.z, a[q].s[2]);
    } else {
      a[q].s[0] = fma(y.w, log(den[q]), a[q].s[0]);
    }
  }
}

// Possibly-near pair of a PP range: i is the target's index, j the source's
// index in the unified point array. The near test is a warp vote, so the
// common case (no lane near) is the straight-line fast path with no
// divergence; a warp with a near lane (a self pair of the own leaf, or
// genuinely close points) runs the exact path for those lanes only.
template <int KER>
__device__ __forceinline__ void pair_near(double x0, double x1, double x2, const double4& y, int i, int j,
                                          Acc<KER>& a, int* flags) {
  const double den_f = fma(-x2, y.z, fma(-x1, y.y, fma(-x0, y.x, 1.0)));
  const bool nearp = __double2hiint(den_f) < kNearHi;
  if (__any_sync(0xffffffffu, nearp)) {
    double c[KDim<KER>::D];
    if (nearp) {
      pair_slow<KER>(x0, x1, x2, y, i, j, c, flags);
    } else if constexpr (KER == kBS) {
      const double r = q_over(y.w, den_f);
      c[0] = r * y.x;
      c[1] = r * y.y;
      c[2] = r * y.z;
    } else {
      c[0] = y.w * log(den_f);
    }
#pragma unroll
    for (int d = 0; d < KDim<KER>::D; ++d) a.s[d] += c[d];
    return;
  }
  if constexpr (KER == kBS) {
    const double r = q_over(y.w, den_f);
    a.s[0] = fma(r, y.x, a.s[0]);
    a.s[1] = fma(r, y.y, a.s[1]);
    a.s[2] = fma(r, y.z, a.s[2]);
  } else {
    a.s[0] = fma(y.w, log(den_f), a.s[0]);
  }
}

}  // namespace ssum
