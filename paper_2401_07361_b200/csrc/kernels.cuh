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
// Near pairs (den < 2^-16, or a self pair) take the reference-rounded slow
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

// hi word of 2^-16: den < 2^-16 (or negative) <=> (int)hi(den) < kNearHi
constexpr int kNearHi = 0x3EF00000;

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

// Possibly-near pair of a PP range: i is the target's index, j the source's
// index in the unified point array.
template <int KER>
__device__ __forceinline__ void pair_near(double x0, double x1, double x2, const double4& y, int i, int j,
                                          Acc<KER>& a, int* flags) {
  const double den_f = fma(-x2, y.z, fma(-x1, y.y, fma(-x0, y.x, 1.0)));
  if (__double2hiint(den_f) >= kNearHi) {
    if constexpr (KER == kBS) {
      const double r = q_over(y.w, den_f);
      a.s[0] = fma(r, y.x, a.s[0]);
      a.s[1] = fma(r, y.y, a.s[1]);
      a.s[2] = fma(r, y.z, a.s[2]);
    } else {
      a.s[0] = fma(y.w, log(den_f), a.s[0]);
    }
    return;
  }
  if (i == j) return;  // self pair (treecode.cpp:388, :257)
  // reference rounding: 1.0 - dot(x, y) (kernels.hpp:26, geometry.hpp:68-70)
  const double den = __dsub_rn(1.0, __dadd_rn(__dadd_rn(__dmul_rn(x0, y.x), __dmul_rn(x1, y.y)), __dmul_rn(x2, y.z)));
  if (den <= kSingularTol) {
    atomicOr(flags, kFlagSingular);
    return;
  }
  if constexpr (KER == kBS) {
    const double r = __ddiv_rn(y.w, den);
    a.s[0] = fma(r, __dsub_rn(y.x, x0), a.s[0]);
    a.s[1] = fma(r, __dsub_rn(y.y, x1), a.s[1]);
    a.s[2] = fma(r, __dsub_rn(y.z, x2), a.s[2]);
  } else {
    a.s[0] = fma(y.w, log(den), a.s[0]);
  }
}

}  // namespace ssum
