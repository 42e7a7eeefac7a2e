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
//   j = the next 7 bits of t1: 128 buckets of m, bucket j centred on
//   c_j = (hi word kLogTabK + 8192 j + 4096, low word 0) — the bucket of m = 1
//   has c = 1 exactly, so x near 1 keeps full relative accuracy;
//   with r_j a double within 2^-12 of 1 / c_j (r = 1 for the bucket of m = 1):
//   t = RN(m r_j - 1) in one FMA (|t| <= 2^-8 + 2^-12, relative rounding
//   error 2^-53) and log m = log1p(m r_j - 1) - log r_j exactly. The table
//   holds L_j = RN(-log r_j); r_j is chosen (log_table: Gal's accurate-table
//   search) so that -log r_j lies within 2^-6 ulp of L_j, so the table adds
//   no rounding of its own where log c_j and log1p t cancel (x near 1);
//   log1p t = t + t^2 p(t), p the quartic Chebyshev fit of (log1p t - t) / t^2
//   on |t| <= 2^-8 (tools/log_coeffs.py: |error| < 2^-54.8 |t|);
//   log x = k ln2 + (L_j + log1p t) in one FMA: |log x| >= ~0.34 whenever
//   k != 0, so nothing cancels, and k (ln2 - RN(ln2)) <= 0.3 ulp for
//   |k| <= 20. 13 FP64 and ~8 integer instructions per pair including the
//   denominator and the accumulation; <= 1.2 ulp against 80-bit logl over 8M
//   points and every bucket edge (host emulation in tools/log_coeffs.py: 1.18;
//   tests/test_gpu_parity.py test_log_far_accuracy bounds it by 2 ulp over
//   [2^-20, 4] on the device).
// Shared-memory layout: the 16-byte entry (r_j, L_j) is stored 8 times, copy
// s in bank group s (address (8 j + s) * 16): lane l reads copy l & 7, so the
// 8 lanes of each quarter-warp that one LDS.128 serves always hit 8 distinct
// bank groups — conflict-free whatever buckets the lanes' denominators fall
// in. With one copy, ncu measured 10.2 wavefronts per table load instead of
// 4 (a warp's denominators span ~a factor 2, i.e. random buckets), and the
// log tiles were shared-memory-bandwidth bound (~92% of the SM's wavefronts).
constexpr int kLogTabBits = 7;
constexpr int kLogTabN = 1 << kLogTabBits;
constexpr int kLogTabCopies = 8;
constexpr int kLogTabShift = 20 - kLogTabBits;
// (0x3FF00000 - kLogTabK) % 8192 == 4096: c = 1 is a bucket centre; m in [0.709, 1.418)
constexpr int kLogTabK = 0x3FE6B000;
void log_table(double2* tab);  // host: kLogTabN entries (r_j, L_j = RN(-log r_j))
__host__ __device__ __forceinline__ double log_tab_node(int j) {
  const unsigned hi = static_cast<unsigned>(kLogTabK + (j << kLogTabShift) + (1 << (kLogTabShift - 1)));
#if defined(__CUDA_ARCH__)
  return __hiloint2double(static_cast<int>(hi), 0);
#else
  const unsigned long long bits = static_cast<unsigned long long>(hi) << 32;
  double d;
  __builtin_memcpy(&d, &bits, 8);
  return d;
#endif
}

// log_tab in two halves: the table slot of x, and the rest given its entry.
// `tab` is the staged table already offset by this lane's copy (lane & 7).
__device__ __forceinline__ int log_tab_slot(int t1) {
  return ((t1 >> kLogTabShift) & (kLogTabN - 1)) * kLogTabCopies;
}
__device__ __forceinline__ double log_tab_fin(double x, int t1, double2 e) {
  constexpr double kLn2 = 0x1.62e42fefa39efp-1;
  const int kk = t1 >> 20;  // arithmetic shift: the exponent of x relative to m
  const double m = __hiloint2double(__double2hiint(x) - (t1 & static_cast<int>(0xfff00000u)), __double2loint(x));
  const double t = fma(m, e.x, -1.0);
  double p = fma(t, -0x1.555695a65ad63p-3, 0x1.999b07ad05760p-3);
  p = fma(t, p, -0x1.ffffffffafd7bp-3);
  p = fma(t, p, 0x1.5555555527877p-2);
  p = fma(t, p, -0.5);
  const double l1p = fma(t * t, p, t);
  return fma(static_cast<double>(kk), kLn2, e.y + l1p);
}
__device__ __forceinline__ double log_tab(double x, const double2* __restrict__ tab) {
  const int t1 = __double2hiint(x) - kLogTabK;  // one subtraction for the slot, m and k
  return log_tab_fin(x, t1, tab[log_tab_slot(t1)]);
}
// stage the table for log_tab (every copy), then offset it by the lane's copy
__device__ __forceinline__ void log_tab_stage(double2* dst, const double2* __restrict__ src, int tid, int nth) {
  for (int i = tid; i < kLogTabN * kLogTabCopies; i += nth) dst[i] = src[i / kLogTabCopies];
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

// far_block<kLOG> (well-separated steps, not CUBIC) in two halves for a
// software-pipelined loop: log_step_pre forms one step's denominators and
// issues its table loads, log_step_post finishes the logs and accumulates.
// The table slot depends on the denominator, so in far_block every pair
// waited on a dependent shared-memory load in mid-chain (ncu: short-scoreboard
// stalls at the first DFMA after it); issuing step s + 1's loads before
// finishing step s hides that latency. Same operations per pair, bitwise
// far_block's sums.
template <int NT, int NS>
struct LogStep {
  double den[NT * NS];
  double2 e[NT * NS];
  double q[NS];
};
template <int NT, int NS>
__device__ __forceinline__ void log_step_pre(const double4* x, const double4* __restrict__ B, int G,
                                             const double2* __restrict__ tab, LogStep<NT, NS>& st) {
  constexpr int C = NT * NS;
  double4 y[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) y[s] = B[s * G];
#pragma unroll
  for (int c = 0; c < C; ++c) st.den[c] = fma(-x[c % NT].x, y[c / NT].x, 1.0);
#pragma unroll
  for (int c = 0; c < C; ++c) st.den[c] = fma(-x[c % NT].y, y[c / NT].y, st.den[c]);
#pragma unroll
  for (int c = 0; c < C; ++c) st.den[c] = fma(-x[c % NT].z, y[c / NT].z, st.den[c]);
#pragma unroll
  for (int c = 0; c < C; ++c) st.e[c] = tab[log_tab_slot(__double2hiint(st.den[c]) - kLogTabK)];
#pragma unroll
  for (int s = 0; s < NS; ++s) st.q[s] = y[s].w;
}
template <int NT, int NS>
__device__ __forceinline__ void log_step_post(const LogStep<NT, NS>& st, Acc<kLOG>* a) {
#pragma unroll
  for (int c = 0; c < NT * NS; ++c) a[c % NT].s[0] = fma(st.q[c / NT], log_tab_fin(st.den[c], __double2hiint(st.den[c]) - kLogTabK, st.e[c]), a[c % NT].s[0]);
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

// hi word of 2^-30: den < 2^-30 ~ 9.3e-10 (or negative) <=> (int)hi(den) < kCloseHi
constexpr int kCloseHi = 0x3E100000;

// Near-possible block of a dense leaf tile, lean form (the default): the
// denominator with the reference's rounding for EVERY pair (6 FP64
// instructions, stage by stage across the NT*NS chains like far_block), the
// reciprocal by MUFU seed + one Newton step (relative error <= 1e-12 per
// term, far_block's) and S += r y — 12 FP64 instructions per pair against
// near_exact_block's 18. A pair's term is x cross (r y): accumulating r y
// instead of r (y - x) leaves an absolute rounding error of ~1e-16 r in S,
// the reference's own (it rounds cross(x, y) to ~1e-16 absolute before the
// division, kernels.hpp:26-32), harmless while r stays moderate. Pairs
// closer than den < 2^-30 (arc < 4.3e-5: the self pair, a singular pair, or
// a genuinely close pair of a dense cloud, r up to q 1e14) are masked out of
// those sums and taken one by one on near_exact_block's arithmetic (self
// pair by list position, singular guard, ~1 ulp q / den, r (y - x)); on a
// mesh (config 5) that is the self pair only.
template <int NT, int NS>
__device__ __forceinline__ void near_lean_block(const double4* x, const double4* __restrict__ B, int G,
                                                Acc<kBS>* a, int f0, const int* selfpos, int* flags) {
  // one source at a time (NT chains interleaved): the 64-register leaf
  // kernel has no room for NT*NS chains of den / product / reciprocal here
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const double4 y = B[s * G];
    double den[NT], p[NT], r[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) den[t] = __dmul_rn(x[t].x, y.x);
#pragma unroll
    for (int t = 0; t < NT; ++t) p[t] = __dmul_rn(x[t].y, y.y);
#pragma unroll
    for (int t = 0; t < NT; ++t) den[t] = __dadd_rn(den[t], p[t]);
#pragma unroll
    for (int t = 0; t < NT; ++t) p[t] = __dmul_rn(x[t].z, y.z);
#pragma unroll
    for (int t = 0; t < NT; ++t) den[t] = __dadd_rn(den[t], p[t]);
#pragma unroll
    for (int t = 0; t < NT; ++t) den[t] = __dsub_rn(1.0, den[t]);
#pragma unroll
    for (int t = 0; t < NT; ++t) r[t] = rcp_approx(den[t]);
#pragma unroll
    for (int t = 0; t < NT; ++t) p[t] = fma(-den[t], r[t], 1.0);
#pragma unroll
    for (int t = 0; t < NT; ++t) r[t] = __dmul_rn(y.w, r[t]);
#pragma unroll
    for (int t = 0; t < NT; ++t) r[t] = fma(r[t], p[t], r[t]);
    bool close = false;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      if (__double2hiint(den[t]) < kCloseHi) {  // the masked term's high word cleared: <= 2^-1022, never NaN/inf
        close = true;
        r[t] = __hiloint2double(0, __double2loint(r[t]));
      }
    }
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      a[t].s[0] = fma(r[t], y.x, a[t].s[0]);
      a[t].s[1] = fma(r[t], y.y, a[t].s[1]);
      a[t].s[2] = fma(r[t], y.z, a[t].s[2]);
    }
    if (close) {
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        if (f0 + s * G == selfpos[t]) continue;  // treecode.cpp:388
        const double d = __dsub_rn(1.0, __dadd_rn(__dadd_rn(__dmul_rn(x[t].x, y.x), __dmul_rn(x[t].y, y.y)),
                                                  __dmul_rn(x[t].z, y.z)));
        if (__double2hiint(d) >= kCloseHi) continue;
        if (d <= kSingularTol) {  // kernels.hpp:19,27-29
          atomicOr(flags, kFlagSingular);
          continue;
        }
        const double rr = q_over(y.w, d);
        a[t].s[0] = fma(rr, __dsub_rn(y.x, x[t].x), a[t].s[0]);
        a[t].s[1] = fma(rr, __dsub_rn(y.y, x[t].y), a[t].s[1]);
        a[t].s[2] = fma(rr, __dsub_rn(y.z, x[t].z), a[t].s[2]);
      }
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
