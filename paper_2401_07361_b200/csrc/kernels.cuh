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
// discarded), table-driven with the reduction centred on 1:
//   t1 = hi(x) - kLogTabK (kLogTabK = hi word just above sqrt(2)/2), so
//   k = t1 >> 20 is the exponent with x = 2^k m, m in [0.7072, 1.4143), and
//   hi(m) = hi(x) - (t1 & 0xfff00000) (integer ops only);
//   j = the next 9 bits of t1: 512 buckets of m, bucket j centred on
//   c_j = (hi word kLogTabK + 2048 j + 1024, low word 0) — the bucket of m = 1
//   has c = 1 exactly, so x near 1 keeps full relative accuracy;
//   t = (m - c_j) / c_j with |t| <= 2^-10 (m - c_j exact by Sterbenz);
//   log m = log c_j + log1p(t), log1p through t^6 (truncation < 2^-60 t);
//   log x = k ln2_hi + (log c_j + (k ln2_lo + log1p t)), ln 2 split into a
//   21-bit head (k ln2_hi exact) and a tail; |log x| >= ~0.35 whenever k != 0,
//   so the sum never cancels. (1 / c_j, log c_j) come from a 512-entry table
//   (log_table, correctly rounded from 80-bit precision) staged in shared
//   memory. 15 FP64 and ~9 integer instructions per pair including the
//   denominator and the accumulation, against 17 + ~14 for the 65-entry,
//   degree-8 version before it; <= 1.5 ulp (tests/test_gpu_parity.py
//   test_log_far_accuracy bounds it by 2 ulp over [2^-20, 4]).
constexpr int kLogTabN = 512;
constexpr int kLogTabK = 0x3FE6A400;  // (0x3FF00000 - kLogTabK) % 2048 == 1024: c = 1 is a bucket centre
void log_table(double2* tab);         // host: kLogTabN entries (1 / c_j, log c_j)
__host__ __device__ __forceinline__ double log_tab_node(int j) {
#if defined(__CUDA_ARCH__)
  return __hiloint2double(kLogTabK + (j << 11) + 1024, 0);
#else
  const unsigned long long bits = static_cast<unsigned long long>(static_cast<unsigned>(kLogTabK + (j << 11) + 1024))
                                  << 32;
  double d;
  __builtin_memcpy(&d, &bits, 8);
  return d;
#endif
}

__device__ __forceinline__ double log_tab(double x, const double2* __restrict__ tab) {
  constexpr double kLn2Hi = 0x1.62e42p-1;           // ln 2, low 32 mantissa bits cleared
  constexpr double kLn2Lo = 0x1.fdf473de6af28p-22;  // ln 2 - kLn2Hi
  const int hi = __double2hiint(x);
  const int t1 = hi - kLogTabK;
  const int kk = t1 >> 20;  // arithmetic shift: the exponent of x relative to m
  const int j = (t1 >> 11) & (kLogTabN - 1);
  const double m = __hiloint2double(hi - (t1 & static_cast<int>(0xfff00000u)), __double2loint(x));
  const double2 e = tab[j];
  const double t = (m - log_tab_node(j)) * e.x;
  double p = fma(t, -1.0 / 6.0, 1.0 / 5.0);
  p = fma(t, p, -0.25);
  p = fma(t, p, 1.0 / 3.0);
  p = fma(t, p, -0.5);
  const double l1p = fma(t * t, p, t);
  const double dk = static_cast<double>(kk);
  return fma(dk, kLn2Hi, e.y) + fma(dk, kLn2Lo, l1p);
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
                                          int* ncnt = nullptr, const double2* __restrict__ ltab = nullptr) {
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
      double l = CUBIC ? log(den[c]) : log_tab(den[c], ltab);
      if constexpr (NEAR) l = near_mask(l, den[c], *ncnt);
      a[c % NT].s[0] = fma(y[c / NT].w, l, a[c % NT].s[0]);
    }
  }
}

// One step of a near-possible range, decided per warp by a vote (the
// default near handling of leaf / direct tiles): the NT x NS denominators
// first, exactly as far_block forms them; when no lane of the warp met a near
// pair (den < 2^-20) or one of its self pairs (known by list position), the
// step finishes on far_block's arithmetic, otherwise the whole warp takes the
// reference-rounded exact_step for it. Near pairs are rare outside dense
// inputs (none on the icosahedral meshes) and a leaf's self pairs fill only
// the steps over its own bin, so nearly every step stays on the fast path
// with no per-pair mask, count or repair walk.
template <int KER, int NT, int NS>
__device__ __forceinline__ void exact_step(const double4* x, const double4* y, int G, Acc<KER>* a, int f0,
                                           const int* selfpos, int* flags) {
#pragma unroll
  for (int c = 0; c < NT * NS; ++c) {
    const double4& xx = x[c % NT];
    const double4& yy = y[c / NT];
    const double den = __dsub_rn(1.0, __dadd_rn(__dadd_rn(__dmul_rn(xx.x, yy.x), __dmul_rn(xx.y, yy.y)),
                                                __dmul_rn(xx.z, yy.z)));
    const bool self = f0 + (c / NT) * G == selfpos[c % NT];  // treecode.cpp:388, :257
    const bool sing = den <= kSingularTol;                   // kernels.hpp:19,27-29
    if (sing && !self) atomicOr(flags, kFlagSingular);
    if constexpr (KER == kBS) {
      const double r = (self || sing) ? 0.0 : q_over(yy.w, den);
      a[c % NT].s[0] = fma(r, __dsub_rn(yy.x, xx.x), a[c % NT].s[0]);
      a[c % NT].s[1] = fma(r, __dsub_rn(yy.y, xx.y), a[c % NT].s[1]);
      a[c % NT].s[2] = fma(r, __dsub_rn(yy.z, xx.z), a[c % NT].s[2]);
    } else {
      a[c % NT].s[0] += (self || sing) ? 0.0 : yy.w * log(den);
    }
  }
}

template <int KER, int NT, int NS, bool CUBIC = false>
__device__ __forceinline__ void near_vote_block(const double4* x, const double4* __restrict__ B, int G,
                                                Acc<KER>* a, int f0, const int* selfpos, int* flags,
                                                const double2* __restrict__ ltab) {
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
  bool slow = false;
#pragma unroll
  for (int c = 0; c < C; ++c) slow |= __double2hiint(den[c]) < kNearHi;
#pragma unroll
  for (int t = 0; t < NT; ++t)
#pragma unroll
    for (int s = 0; s < NS; ++s) slow |= f0 + s * G == selfpos[t];
  if (__any_sync(0xffffffffu, slow)) {
    exact_step<KER, NT, NS>(x, y, G, a, f0, selfpos, flags);
    return;
  }
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
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[0] = fma(r[c], y[c / NT].x, a[c % NT].s[0]);
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[1] = fma(r[c], y[c / NT].y, a[c % NT].s[1]);
#pragma unroll
    for (int c = 0; c < C; ++c) a[c % NT].s[2] = fma(r[c], y[c / NT].z, a[c % NT].s[2]);
  } else {
#pragma unroll
    for (int c = 0; c < C; ++c)
      a[c % NT].s[0] = fma(y[c / NT].w, CUBIC ? log(den[c]) : log_tab(den[c], ltab), a[c % NT].s[0]);
  }
}

// Near-possible block of a dense leaf tile (Biot-Savart): every pair with
// the reference's rounding (den = 1 - ((x.x y.x + x.y y.y) + x.z y.z),
// separately rounded; singular guard on that value, kernels.hpp:19,27-29),
// the self pair excluded by list position (treecode.cpp:388), and the
// Sterbenz-exact r (y - x) accumulation (x cross (y - x) = x cross y) with a
// ~1 ulp q / den — no mask, no repair. Source s of the block sits at
// flattened position f0 + s G; selfpos[q] is target q's own position (-1:
// none in the list).
template <int NT, int NS>
__device__ __forceinline__ void near_exact_block(const double4* x, const double4* __restrict__ B, int G,
                                                 Acc<kBS>* a, int f0, const int* selfpos, int* flags) {
  double4 y[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) y[s] = B[s * G];
#pragma unroll
  for (int c = 0; c < NT * NS; ++c) {
    const double4& xx = x[c % NT];
    const double4& yy = y[c / NT];
    const double den = __dsub_rn(1.0, __dadd_rn(__dadd_rn(__dmul_rn(xx.x, yy.x), __dmul_rn(xx.y, yy.y)),
                                                __dmul_rn(xx.z, yy.z)));
    const bool self = f0 + (c / NT) * G == selfpos[c % NT];
    const bool sing = den <= kSingularTol;
    if (sing && !self) atomicOr(flags, kFlagSingular);
    const double r = (self || sing) ? 0.0 : q_over(yy.w, den);
    a[c % NT].s[0] = fma(r, __dsub_rn(yy.x, xx.x), a[c % NT].s[0]);
    a[c % NT].s[1] = fma(r, __dsub_rn(yy.y, xx.y), a[c % NT].s[1]);
    a[c % NT].s[2] = fma(r, __dsub_rn(yy.z, xx.z), a[c % NT].s[2]);
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
