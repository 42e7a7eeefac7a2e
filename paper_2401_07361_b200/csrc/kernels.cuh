// Pair interactions of the two reference kernels (kernels.hpp:13-61), written
// for the sm_100a FP64 pipe.
//
// Biot-Savart: K(x, y) q = q (x X y)/(1 - x.y). Summed over sources as
//   S = sum_j r_j y_j   (well-separated pairs),   r_j = q_j / (1 - x.y_j)
//   S = sum_j r_j (y_j - x)  (near pairs),
// and finished once per target as u = -1/(4 pi) x X S (x X x = 0, so both
// forms give the same cross product). 13 algorithmic flops per pair
// (SURVEY.md §8(d)); the fast path issues 9 FP64 instructions + 1 MUFU:
//   den = fma(-z, y.z, fma(-y, y.y, fma(-x, y.x, 1)))      3 DFMA
//   r0 = rcp.approx(den); e = 1 - den r0                  MUFU + 1 DFMA
//   r = q r0 (1 + e)                                       1 DMUL + 1 DFMA
//   S += r y                                               3 DFMA
// rcp.approx.ftz.f64 is ~2^-20 accurate (measured 9.9e-7 on the box); the
// Newton step leaves e^2 <= 1e-12 relative per term (far_block). The direct
// sum adds e^2 (one more DFMA, ~1 ulp).
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

// log(x) for a far pair's denominator (x >= 2^-20, positive and normal;
// anything else only reaches it in a near-masked step, whose term is
// discarded). x = 2^k m, m in [sqrt(1/2), sqrt(2)) by an exponent shift;
// with f = m - 1, s = f / (2 + f): log m = 2 atanh(s) = 2s + s R,
// R = sum_{j>=1} 2 s^2j / (2j + 1) (the exact series through s^18, |s| <=
// 0.1716: truncation <= 2.3e-17 relative), evaluated as
// f - (f^2/2 - s (f^2/2 + R)) so that the leading f is exact, plus k ln 2
// split into a 21-bit head (k ln2_hi exact) and a tail. ~1 ulp; 24 FP64
// instructions and a handful of integer ones, against ~85 instructions for
// the generic log.
__device__ __forceinline__ double log_far(double x) {
  constexpr double kLn2Hi = 0x1.62e42p-1;             // ln 2, low 32 mantissa bits cleared
  constexpr double kLn2Lo = 0x1.fdf473de6af28p-22;    // ln 2 - kLn2Hi
  int hi = __double2hiint(x);
  const int k = (hi - 0x3fe6a09e) >> 20;              // 0x3fe6a09e: high word of sqrt(1/2)
  hi -= k << 20;
  const double f = __hiloint2double(hi, __double2loint(x)) - 1.0;  // exact (Sterbenz)
  const double hfsq = 0.5 * (f * f);
  const double s = q_over(f, 2.0 + f);
  const double z = s * s;
  double p = 2.0 / 19.0;
  p = fma(z, p, 2.0 / 17.0);
  p = fma(z, p, 2.0 / 15.0);
  p = fma(z, p, 2.0 / 13.0);
  p = fma(z, p, 2.0 / 11.0);
  p = fma(z, p, 2.0 / 9.0);
  p = fma(z, p, 2.0 / 7.0);
  p = fma(z, p, 2.0 / 5.0);
  p = fma(z, p, 2.0 / 3.0);
  const double R = z * p;
  const double dk = static_cast<double>(k);
  return fma(dk, kLn2Hi, f - (hfsq - fma(s, hfsq + R, dk * kLn2Lo)));
}

template <int KER>
struct Acc {
  double s[KDim<KER>::D];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int d = 0; d < KDim<KER>::D; ++d) s[d] = 0.0;
  }
};

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
    // the exact denominator is what matters here; q / den itself only needs
    // ~1 ulp (q_over: no division subroutine call, so no spills around it)
    const double r = q_over(y.w, den);
    c[0] = r * __dsub_rn(y.x, x0);
    c[1] = r * __dsub_rn(y.y, x1);
    c[2] = r * __dsub_rn(y.z, x2);
  } else {
    c[0] = y.w * log(den);
  }
}

// Near-segment mask of one pair's term v: when den < 2^-20 (a self pair, or a
// near pair left to near_repair) the high word of v is cleared — what is
// left is at most 2^-1022 in magnitude, never NaN or inf — and the lane's
// near count is bumped; one compare, two predicated moves/adds.
__device__ __forceinline__ double near_mask(double v, double den, int& cnt) {
  int hi = __double2hiint(v);
  asm("{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %2, %3;\n\t@p add.s32 %0, %0, 1;\n\t@p mov.b32 %1, 0;\n\t}"
      : "+r"(cnt), "+r"(hi)
      : "r"(__double2hiint(den)), "n"(kNearHi));
  return __hiloint2double(hi, __double2loint(v));
}

// NS sources x NT targets of well-separated pairs, written stage by stage
// across the NS*NT independent chains (all denominators, then all
// reciprocal seeds, then each Newton step, then the accumulations) so that
// consecutive instructions belong to different chains and the in-order
// issue never waits on a DFMA (8.8 cycles) or MUFU.RCP64H (~24 cycles)
// result it just produced.
// NEAR: the block may hold near pairs (self pairs, 1 - x.y < 2^-20). They
// are masked out of the sums (their NaN/inf reciprocals never reach them)
// and counted per lane in *ncnt, with no branch and no vote: the caller
// compares the count with the self pairs the lane must have met and
// re-walks the chunk through near_repair only when they differ.
// Reciprocal: MUFU.RCP64H seed (rel. error <= 9.9e-7) and one Newton step,
// q/den = q r0 (1 + e) with e = 1 - den r0: relative error e^2 <= 1e-12 per
// term, 9 FP64 instructions per pair; measured 1.2e-13 .. 1.6e-13 relative
// L2 against the reference's exact division on configs 3 and 4 (bar 1e-10).
// CUBIC (the direct sum, the accuracy yardstick): q r0 (1 + e + e^2), ~1 ulp,
// one more DFMA.
template <int KER, int NT, int NS, bool NEAR = false, bool CUBIC = false>
__device__ __forceinline__ void far_block(const double4* x, const double4* __restrict__ B, int G, Acc<KER>* a,
                                          int* ncnt = nullptr) {
  constexpr int C = NT * NS;
  double4 y[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) y[s] = B[s * G];
  double den[C];
#pragma unroll
  for (int c = 0; c < C; ++c) den[c] = fma(-x[c % NT].x, y[c / NT].x, 1.0);
#pragma unroll
  for (int c = 0; c < C; ++c) den[c] = fma(-x[c % NT].y, y[c / NT].y, den[c]);
#pragma unroll
  for (int c = 0; c < C; ++c) den[c] = fma(-x[c % NT].z, y[c / NT].z, den[c]);
  if constexpr (KER == kBS) {
    double r[C], e[C];
#pragma unroll
    for (int c = 0; c < C; ++c) r[c] = rcp_approx(den[c]);
#pragma unroll
    for (int c = 0; c < C; ++c) e[c] = fma(-den[c], r[c], 1.0);
    if constexpr (CUBIC) {
#pragma unroll
      for (int c = 0; c < C; ++c) e[c] = fma(e[c], e[c], e[c]);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) r[c] = y[c / NT].w * r[c];
#pragma unroll
    for (int c = 0; c < C; ++c) r[c] = fma(r[c], e[c], r[c]);
    if constexpr (NEAR) {
#pragma unroll
      for (int c = 0; c < C; ++c) r[c] = near_mask(r[c], den[c], *ncnt);
    }
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[0] = fma(r[c], y[c / NT].x, a[c % NT].s[0]);
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[1] = fma(r[c], y[c / NT].y, a[c % NT].s[1]);
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[2] = fma(r[c], y[c / NT].z, a[c % NT].s[2]);
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c) {
      double l = CUBIC ? log(den[c]) : log_far(den[c]);
      if constexpr (NEAR) l = near_mask(l, den[c], *ncnt);
      a[c % NT].s[0] = fma(y[c / NT].w, l, a[c % NT].s[0]);
    }
  }
}

// Second walk over one far_block<..., true> block whose warp saw a near pair
// other than its self pairs: adds the reference-rounded contribution of each
// near pair of distinct points (pair_slow, which also raises the singular
// flag), and takes back the fast term of a self pair that was not near (only
// possible for input points off the unit sphere). Source s of the block sits
// at flattened list position f0 + s G; jof(f) is its point index (-1 for the
// zero padding past the list).
template <int KER, int NT, int NS, class JOf>
__device__ __forceinline__ void near_repair(const double4* x, const double4* __restrict__ B, int f0, JOf jof,
                                            int G, Acc<KER>* a, const int* ti, int* flags) {
  int js[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) js[s] = jof(f0 + s * G);
#pragma unroll
  for (int c = 0; c < NT * NS; ++c) {
    const double4 y = B[(c / NT) * G];
    const int j = js[c / NT];
    const double4& xx = x[c % NT];
    const double den = fma(-xx.z, y.z, fma(-xx.y, y.y, fma(-xx.x, y.x, 1.0)));
    const bool nr = __double2hiint(den) < kNearHi;
    double v[KDim<KER>::D];
    if (nr && ti[c % NT] != j) {
      pair_slow<KER>(xx.x, xx.y, xx.z, y, ti[c % NT], j, v, flags);
    } else if (!nr && ti[c % NT] == j) {
      if constexpr (KER == kBS) {
        const double r = -q_over(y.w, den);
        v[0] = r * y.x;
        v[1] = r * y.y;
        v[2] = r * y.z;
      } else {
        v[0] = -y.w * log(den);
      }
    } else {
      continue;
    }
#pragma unroll
    for (int d = 0; d < KDim<KER>::D; ++d) a[c % NT].s[d] += v[d];
  }
}

}  // namespace ssum
