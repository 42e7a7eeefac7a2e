// Interaction tiles: the PP + PC (leaf) and CP + CC + fit (fit node) passes
// and the direct sum, all on one kernel shape (k_tiles). Kept in its own
// translation unit so tuning builds (make variants) recompile only this file.
#include <atomic>

#include "kernels.cuh"

namespace ssum {

namespace {

constexpr double kInv4Pi = 0.07957747154594767;  // 1 / (4 pi)

// Phases 3 and 4 (direct part) share one kernel shape: a block of 256
// threads per TILE — up to 256 targets (a leaf's particles, or a fit node's
// p proxy points) against the tile's list of source ranges.
//
//  * Thread -> (targets u, u + th with th = ceil(T / 2), source group g)
//    with G = min(32, 256 / th) groups: a 40-particle leaf keeps 240 of 256
//    lanes busy (th 20, 12 groups), a p = 45 fit node 253 (th 23, 11 groups).
//  * The source ranges are streamed as ONE flattened list in chunks of
//    kChunk sources through kStages shared-memory stages filled by the copy
//    engine: warp 0 issues one cp.async.bulk per (range, chunk) overlap —
//    each range is a contiguous run of double4 points — completing on the
//    stage's full mbarrier; each warp releases a stage on its empty mbarrier
//    when done, so warps never wait on each other inside the tile and
//    chunks land while earlier ones are consumed, with no register staging
//    and no per-source address search. Every
//    thread walks the chunk with stride G, 2 sources x 2 targets per step
//    (far_block), so all warps run the same trip count (the chunk tail is
//    zero-padded: q = 0 adds nothing).
//  * Group partials are reduced in group order through shared memory
//    (deterministic, no atomics).
//  MODE kLeafMode: the near-possible prefix of the list runs with near pairs
//                  masked, counted and repaired (kernels.cuh); writes S per
//                  target.
//  MODE kFitMode : well-separated pairs only; phi = K-sums at the proxy
//                  points, then C = V^-1 phi (ProxyFit::solve, sbb.cpp:103-108).
//  MODE kDirectMode: kLeafMode with the ~1 ulp (cubic) reciprocal — the
//                  direct sum, every source near-possible.
// Launch shapes (threads per tile block, sources per chunk stage, resident
// blocks per SM for the register budget), leaf/direct and fit separately.
#ifndef SSUM_LEAF_THREADS
#define SSUM_LEAF_THREADS 256
#endif
#ifndef SSUM_CHUNK
#define SSUM_CHUNK 768
#endif
#ifndef SSUM_FIT_CHUNK
#define SSUM_FIT_CHUNK 768
#endif
constexpr int kLeafThreads = SSUM_LEAF_THREADS, kFitThreads = 256;
constexpr int kLeafChunk = SSUM_CHUNK, kFitChunk = SSUM_FIT_CHUNK;
#ifndef SSUM_STAGES
#define SSUM_STAGES 2
#endif
constexpr int kStages = SSUM_STAGES;  // chunk buffers in flight
constexpr int kLeafMode = 0, kFitMode = 1, kDirectMode = 2;
#ifndef SSUM_NS
#define SSUM_NS 2
#endif
constexpr int kNs = SSUM_NS;  // sources per fast-loop step
// zero tail past a chunk: the stride-G walk in steps of kNs sources reads up
// to kNs*G - 1 entries beyond n
constexpr int kPad = 32 * SSUM_NS;

#ifndef SSUM_TILE_MINB
#define SSUM_TILE_MINB 4
#endif
#ifndef SSUM_FIT_MINB
#define SSUM_FIT_MINB 4
#endif
constexpr int kLeafMinB = SSUM_TILE_MINB, kFitMinB = SSUM_FIT_MINB;
#ifndef SSUM_FAST_UNROLL
#define SSUM_FAST_UNROLL 4
#endif
#ifndef SSUM_NEAR_UNROLL
#define SSUM_NEAR_UNROLL 2
#endif
// far_block steps per loop trip (fast loop: leaf/direct tiles; fit tiles 2)
constexpr int kFastUnroll = SSUM_FAST_UNROLL, kNearUnroll = SSUM_NEAR_UNROLL;
#ifndef SSUM_TPT
#define SSUM_TPT 2
#endif
#ifndef SSUM_NEAR_HIT
#define SSUM_NEAR_HIT 0  // 1: record which near steps met a masked pair (repair only those)
#endif
#ifndef SSUM_RANGE_CAP
#define SSUM_RANGE_CAP 128
#endif
constexpr int kRangeCap = SSUM_RANGE_CAP;
constexpr int kTpt = SSUM_TPT;  // targets per thread (register tile)

// Bulk-copy (TMA, non-tensor) helpers: the source ranges of a chunk are
// copied global -> shared by the copy engine, completion counted in bytes on
// an mbarrier (no register staging, no per-source address search).
__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned done;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}

template <int KER, int MODE, int NTH, int CHUNK, int MINB>
__global__ void __launch_bounds__(NTH, MINB)
    k_tiles(const Tile* __restrict__ tiles, int ntiles, const int* __restrict__ sel,
            const SrcRange* __restrict__ ranges, const double4* __restrict__ pts, double* __restrict__ S,
            int* __restrict__ flags, const int* __restrict__ fit_nodes, const int* __restrict__ pslot,
            const double* __restrict__ vinv, int P, double* __restrict__ coeff, int64_t npts,
            const double2* __restrict__ ltab_g) {
  constexpr int D = KDim<KER>::D;
  constexpr int kFU = MODE == kFitMode ? 2 : kFastUnroll;
  (void)npts;  // valid points in pts (bounds checks of the checked build)
  // dynamic shared memory (kTileSmem bytes): two source stages and the range
  // table; two mbarriers (one per stage)
  extern __shared__ __align__(16) unsigned char smem[];
  // full[s]: the stage's bytes landed (producer arrival + transaction
  // count); empty[s]: every warp is done reading it (one arrival per warp)
  __shared__ unsigned long long full[kStages], empty[kStages];
  __shared__ unsigned step_inv;  // ceil(2^32 / (kNs G)), see steps_of below
  constexpr int kChunk = CHUNK;
  auto buf = reinterpret_cast<double4(*)[kChunk + kPad]>(smem);
  int2* rtab = reinterpret_cast<int2*>(smem + kStages * sizeof(double4) * (kChunk + kPad));
  // log kernel: log_table staged, kLogTabCopies copies (kernels.cuh log_tab)
  double2* ltab_s = reinterpret_cast<double2*>(rtab + kRangeCap);
  const double2* ltab = ltab_s + (threadIdx.x & (kLogTabCopies - 1));  // this lane's copy
  static_assert(sizeof(double) * NTH * D * kTpt <= kStages * sizeof(double4) * (kChunk + kPad), "red alias");
  static_assert(kPad <= NTH, "zero tail");
  double* red = reinterpret_cast<double*>(&buf[0][0]);  // group partials, after the source loop
  if (static_cast<int>(blockIdx.x) >= ntiles) return;
  const int tix = sel ? sel[blockIdx.x] : static_cast<int>(blockIdx.x);
  const Tile T = tiles[tix];
  if (MODE == kFitMode && T.total == 0) return;  // a big node without CP/CC pairs (subtree lists)
  const int tc = T.tgt_count;
  SSUM_DCHECK(tc >= 1 && tc <= kTileTargets && T.tgt_begin >= 0 && T.tgt_begin + tc <= npts);
  SSUM_DCHECK(T.list_begin >= 0 && T.list_end >= T.list_begin && T.near_total <= T.total);
  const int th = (tc + kTpt - 1) / kTpt;  // thread-targets; thread slot u holds targets u, u + th, ...
  const int G = min(32, NTH / th);
  const int tid = threadIdx.x, lane = tid & 31;
  const int u = tid % th, g = (tid / th) % G;
  int ti[kTpt];
  double4 x[kTpt];
#pragma unroll
  for (int q = 0; q < kTpt; ++q) {
    const int tt = u + q * th;
    ti[q] = T.tgt_begin + (tt < tc ? tt : u);  // padding slots repeat target u (discarded)
    x[q] = pts[ti[q]];
  }
  const int total = T.total;
  const double4 zero4 = make_double4(0.0, 0.0, 0.0, 0.0);
  if (tid < kPad) {  // zero tail: the stride-G walk may read up to kNs G - 1 entries past the chunk
#pragma unroll
    for (int st = 0; st < kStages; ++st) buf[st][kChunk + tid] = zero4;
  }
  if constexpr (KER == kLOG) log_tab_stage(ltab_s, ltab_g, tid, NTH);
  if (tid == 0) {
    step_inv = 0xffffffffu / static_cast<unsigned>(kNs * G) + 1u;  // kNs G >= 2
#pragma unroll
    for (int st = 0; st < kStages; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], NTH / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int nr = T.list_end - T.list_begin;
  const bool in_smem = nr <= kRangeCap;
  auto rbegin = [&](int r) { return in_smem ? rtab[r].x : ranges[T.list_begin + r].begin; };
  auto rpad = [&](int r) { return in_smem ? rtab[r].y : ranges[T.list_begin + r].pad; };
  // flattened list position -> range (binary search over the range prefixes)
  auto locate = [&](int f) {
    int lo = 0, hi = nr - 1;
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (rpad(mid) <= f)
        lo = mid;
      else
        hi = mid - 1;
    }
    return lo;
  };
  // point index of flattened position f (-1 past the list): near repair only
  // (a lane's repairs visit non-decreasing positions within a chunk: one
  // search per chunk, then a forward scan from the last range found)
  int rcur = -1;
  auto jof = [&](int f) {
    if (f >= total) return -1;
    if (rcur < 0)
      rcur = locate(f);
    else
      while (rcur + 1 < nr && rpad(rcur + 1) <= f) ++rcur;
    return rbegin(rcur) + (f - rpad(rcur));
  };
  // Warp 0 issues chunk cc into stage cc % kStages once every warp has
  // released the stage's previous chunk: one bulk copy per (range ∩ chunk),
  // lane-parallel over the ranges; the stage's full barrier expects the
  // chunk's bytes. A partial (last) chunk's tail up to the zero pad is
  // cleared with generic stores before the producer's arrival (release), so
  // every warp that sees the phase complete sees the zeros.
  // glob: read the ranges from global memory (chunk 0, issued before the
  // range table is in shared memory)
  auto issue = [&](int cc, bool glob) {
    const int st = cc % kStages;
    const int c0 = cc * kChunk;
    const int cn = min(kChunk, total - c0);
    double4* dst = buf[st];
    if (cc >= kStages) mbar_wait(&empty[st], ((cc / kStages) - 1) & 1);
    for (int e = cn + lane; e < min(kChunk, cn + kPad); e += 32) dst[e] = zero4;
    __syncwarp();
    if (lane == 0) mbar_expect_tx(&full[st], static_cast<unsigned>(cn) * sizeof(double4));
    __syncwarp();
    for (int r = (c0 == 0 ? 0 : locate(c0)) + lane;; r += 32) {
      bool more_r = false;
      if (r < nr) {
        int pad, beg, end;
        if (glob) {
          const SrcRange R = ranges[T.list_begin + r];
          pad = R.pad, beg = R.begin, end = R.pad + R.count;
        } else {
          pad = rpad(r), beg = rbegin(r), end = (r + 1 < nr) ? rpad(r + 1) : total;
        }
        if (pad < c0 + cn) {
          more_r = true;
          const int lo = max(pad, c0), hi = min(end, c0 + cn);
          SSUM_DCHECK(hi <= lo || (beg + (lo - pad) >= 0 && beg + (hi - pad) <= npts && hi - c0 <= kChunk));
          if (hi > lo)
            bulk_g2s(dst + (lo - c0), pts + beg + (lo - pad), static_cast<unsigned>(hi - lo) * sizeof(double4),
                     &full[st]);
        }
      }
      if (!__any_sync(0xffffffffu, more_r)) break;
    }
  };
  // chunk 0 goes out first (warp 0, ranges straight from global memory),
  // while the block stages the range table and its target points
  const int nch = (total + kChunk - 1) / kChunk;
  if (tid < 32 && nch > 0) {
    __syncwarp();  // barrier init (thread 0) before the first arrival
    issue(0, true);
  }
  if (in_smem)
    for (int r = tid; r < nr; r += NTH) {
      const SrcRange R = ranges[T.list_begin + r];
      rtab[r] = make_int2(R.begin, R.pad);
    }
  __syncthreads();
  Acc<KER> a[kTpt];
#pragma unroll
  for (int q = 0; q < kTpt; ++q) a[q].zero();
  // steps of kNs sources per lane per chunk: a chunk of n sources takes
  // ceil(n / (kNs G)) steps (the zero-padded tail contributes nothing)
  const int kStep = kNs * G;
#ifdef SSUM_STEPS_HWDIV  // the earlier form: ptxas re-did both divisions in every chunk (~100 instructions per tile)
  const int steps_full = (kChunk + kStep - 1) / kStep;
  const int steps_last = (total - (nch - 1) * kChunk + kStep - 1) / kStep;
#else
  // ceil(n / kStep) for n <= kChunk + kStep as one multiply-high: for m, d <
  // 2^16, m / d == umulhi(m, ceil(2^32 / d)). The multiplier is divided out
  // once per tile (thread 0, before the prologue's barrier) and read back
  // from shared memory where it is used: held in a register it cost the
  // 64-register loops moves, and left to ptxas it was re-divided per chunk.
  auto steps_of = [&](int m) {
    return static_cast<int>(__umulhi(static_cast<unsigned>(m + kStep - 1), *static_cast<volatile unsigned*>(&step_inv)));
  };
#endif
  if (tid < 32)
    for (int cc = 1; cc < min(nch, kStages - 1); ++cc) issue(cc, false);
  for (int c = 0; c < nch; ++c) {
    const bool more = c + 1 < nch;
    if (tid < 32 && c + kStages - 1 < nch) issue(c + kStages - 1, false);
    mbar_wait(&full[c % kStages], (c / kStages) & 1);
    const int n = min(kChunk, total - c * kChunk);
    const double4* B = buf[c % kStages] + g;  // this lane's sources: B[m G], m = 0, 1, ...
#ifdef SSUM_STEPS_HWDIV
    const int steps = more ? steps_full : steps_last;
#else
    const int steps = steps_of(n);
#endif
    // steps covering the chunk's near-possible prefix [0, near_total - c kChunk):
    // the same staged blocks with near pairs masked and counted, checked
    // against the lane's self pairs once per chunk
    int near_steps = 0;
    if (MODE != kFitMode) {
      const int nn = min(n, T.near_total - c * kChunk);
#ifdef SSUM_STEPS_HWDIV
      near_steps = nn > 0 ? (nn + kStep - 1) / kStep : 0;
#else
      near_steps = nn > 0 ? steps_of(nn) : 0;
#endif
    }
#ifdef SSUM_TIMING_NO_NEAR  // timing experiment only: wrong results for near/self pairs
    near_steps = 0;
#endif
    int it = 0;
    if constexpr (KER == kBS && MODE == kLeafMode) {
      if (near_steps > 0 && (T.has_self & kTileDense)) {
        // dense leaf: the near-possible steps with reference rounding
        int selfpos[kTpt];
#pragma unroll
        for (int q = 0; q < kTpt; ++q) selfpos[q] = (T.has_self & 1) ? ti[q] + T.self_shift : -1;
        const int f0 = c * kChunk + g;
#pragma unroll 1
        for (; it < near_steps; ++it)
#ifdef SSUM_DENSE_EXACT18  // tuning variant: every near-possible pair on the 18-instruction exact form
          near_exact_block<kTpt, kNs>(x, B + it * kStep, G, a, f0 + it * kStep, selfpos, flags);
#else
          near_lean_block<kTpt, kNs>(x, B + it * kStep, G, a, f0 + it * kStep, selfpos, flags);
#endif
      }
    }
#ifdef SSUM_NEAR_VOTE
    // tuning variant: per-step warp vote (kernels.cuh near_vote_block) —
    // measured slower at C4 (leaf tiles 5.24 vs 5.16 ms with the mask below)
    if (it < near_steps) {
      int selfpos[kTpt];
#pragma unroll
      for (int q = 0; q < kTpt; ++q) selfpos[q] = (T.has_self & 1) ? ti[q] + T.self_shift : -1;
      const int f0 = c * kChunk + g;
#pragma unroll kNearUnroll
      for (; it < near_steps; ++it)
        near_vote_block<KER, kTpt, kNs, MODE == kDirectMode>(x, B + it * kStep, G, a, f0 + it * kStep, selfpos,
                                                              flags, ltab);
    }
#else
    if (it < near_steps) {
#if SSUM_NEAR_HIT
      // bit `it` of hit: step `it` met a masked pair (self or near); steps
      // past 64 are all re-walked when a repair is needed
      int ncnt = 0;
      unsigned long long hit = 0;
#pragma unroll kNearUnroll
      for (; it < near_steps; ++it) {
        const int before = ncnt;
        far_block<KER, kTpt, kNs, true, MODE == kDirectMode>(x, B + it * kStep, G, a, &ncnt, ltab);
        hit |= static_cast<unsigned long long>(ncnt != before) << (it & 63);
      }
#else
      // masked pairs counted, recorded per PAIR of steps in 32 bits (fewer
      // live registers and instructions than a per-step 64-bit record); a
      // repair re-walks only the flagged step pairs (beyond 64 steps: all)
      int ncnt = 0;
      unsigned hit2 = 0;
      const double4* Bn = B + it * kStep;
      for (; it + 1 < near_steps; it += 2, Bn += 2 * kStep) {
        const int before = ncnt;
        far_block<KER, kTpt, kNs, true, MODE == kDirectMode>(x, Bn, G, a, &ncnt, ltab);
        far_block<KER, kTpt, kNs, true, MODE == kDirectMode>(x, Bn + kStep, G, a, &ncnt, ltab);
        hit2 |= static_cast<unsigned>(ncnt != before) << ((it >> 1) & 31);
      }
      if (it < near_steps) {
        const int before = ncnt;
        far_block<KER, kTpt, kNs, true, MODE == kDirectMode>(x, Bn, G, a, &ncnt, ltab);
        hit2 |= static_cast<unsigned>(ncnt != before) << ((it >> 1) & 31);
        ++it;
      }
      unsigned long long hit = 0;  // per step, for the repair below
      for (unsigned m2 = hit2; m2; m2 &= m2 - 1) hit |= 3ull << (2 * (__ffs(static_cast<int>(m2)) - 1));
      if (near_steps < 64) hit &= (1ull << near_steps) - 1ull;
#endif
      // self pairs this lane walked in this chunk's near steps: the self
      // source of target ti sits at flattened position ti + T.self_shift
      const int o_end = min(n, near_steps * kStep);
      int nself = 0;
#pragma unroll
      for (int q = 0; q < kTpt; ++q) {
        const int o = ti[q] + T.self_shift - c * kChunk;
#ifdef SSUM_STEPS_HWDIV
        nself += ((T.has_self & 1) && o >= 0 && o < o_end && o % G == g) ? 1 : 0;
#else
        // o % G == g  <=>  o % (kNs G) is g, g + G, ... (kNs = 2: g or g + G); o < 2^16 here
        static_assert(kNs == 2, "self position test");
        const int orem = o - static_cast<int>(__umulhi(static_cast<unsigned>(o), *static_cast<volatile unsigned*>(&step_inv))) * kStep;
        nself += ((T.has_self & 1) && o >= 0 && o < o_end && (orem == g || orem == g + G)) ? 1 : 0;
#endif
      }
      if (__any_sync(0xffffffffu, ncnt != nself)) {
        // only the steps that met a masked pair (dense inputs: a handful of
        // the chunk's near steps)
        const int f0 = c * kChunk + g;
        rcur = -1;
        if (near_steps <= 64) {
#pragma unroll 1
          for (unsigned long long m = hit; m; m &= m - 1) {
            const int r = __ffsll(static_cast<long long>(m)) - 1;
            near_repair<KER, kTpt, kNs>(x, B + r * kStep, f0 + r * kStep, jof, G, a, ti, flags);
          }
        } else {
#pragma unroll 1
          for (int r = 0; r < near_steps; ++r)
            near_repair<KER, kTpt, kNs>(x, B + r * kStep, f0 + r * kStep, jof, G, a, ti, flags);
        }
      }
    }
#endif
    // well-separated sources only: branch-free, kNs sources x kTpt targets
    // of independent chains per step (zero-padded tail contributes 0)
    const double4* Bp = B + it * kStep;
#ifdef SSUM_LOG_PIPE  // measured: no gain (the table loads were bandwidth-, not latency-bound)
    if constexpr (KER == kLOG && MODE != kDirectMode) {
      // log: software-pipelined (kernels.cuh log_step_pre / log_step_post)
      if (it < steps) {
        LogStep<kTpt, kNs> cur, nxt;
        log_step_pre(x, Bp, G, ltab, cur);
#pragma unroll 2
        for (++it; it < steps; ++it) {
          Bp += kStep;
          log_step_pre(x, Bp, G, ltab, nxt);
          log_step_post(cur, a);
          cur = nxt;
        }
        log_step_post(cur, a);
      }
    } else
#endif
#pragma unroll kFU
    for (; it < steps; ++it, Bp += kStep) far_block<KER, kTpt, kNs, false, MODE == kDirectMode>(x, Bp, G, a, nullptr, ltab);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[c % kStages]);  // this warp is done with the stage
  }
  __syncthreads();  // every warp done with every stage: red may alias them
#pragma unroll
  for (int q = 0; q < kTpt; ++q)
#pragma unroll
    for (int d = 0; d < D; ++d) red[(q * NTH + tid) * D + d] = a[q].s[d];
  __syncthreads();
  // target tt = u + q th lives in slot (q, g * th + u) for every group g
  constexpr int kOut = (kTileTargets + NTH - 1) / NTH;  // targets per thread in the epilogue
  double s[kOut][D];
#pragma unroll
  for (int o = 0; o < kOut; ++o) {
    const int tt = tid + o * NTH;
    const int uq = tt % th, qq = tt / th;
    if (tt < tc) {
#pragma unroll
      for (int d = 0; d < D; ++d) s[o][d] = red[(qq * NTH + uq) * D + d];
      for (int gg = 1; gg < G; ++gg)
#pragma unroll
        for (int d = 0; d < D; ++d) s[o][d] += red[(qq * NTH + gg * th + uq) * D + d];
    }
  }
  if constexpr (MODE != kFitMode) {
#pragma unroll
    for (int o = 0; o < kOut; ++o) {
      const int tt = tid + o * NTH;
      if (tt < tc) {
#pragma unroll
        for (int d = 0; d < D; ++d) S[size_t(T.tgt_begin + tt) * D + d] = s[o][d];
      }
    }
  } else {
    __syncthreads();  // red is reused for phi below
    double* phi = red;
#pragma unroll
    for (int o = 0; o < kOut; ++o) {
      const int tt = tid + o * NTH;
      if (tt < tc) {
        const double4 xo = pts[T.tgt_begin + tt];
        if constexpr (KER == kBS) {
          phi[tt] = xo.y * s[o][2] - xo.z * s[o][1];
          phi[P + tt] = xo.z * s[o][0] - xo.x * s[o][2];
          phi[2 * P + tt] = xo.x * s[o][1] - xo.y * s[o][0];
        } else {
          phi[tt] = -kInv4Pi * s[o][0];
        }
      }
    }
    __syncthreads();
    const int slot = pslot[fit_nodes[tix]];
    SSUM_DCHECK(slot >= 0);
    for (int kk = tid; kk < P; kk += NTH) {
#pragma unroll
      for (int d = 0; d < D; ++d) {
        double acc = 0.0;
        for (int m = 0; m < P; ++m) acc = fma(vinv[size_t(kk) * P + m], phi[d * P + m], acc);
        coeff[(size_t(slot) * D + d) * P + kk] = acc;
      }
    }
  }
}

template <int KER>
__global__ void k_direct_finish(int64_t n, const double4* __restrict__ pts, const double* __restrict__ S,
                                double* __restrict__ out) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  if constexpr (KER == kBS) {
    const double4 x = pts[k];
    const double s0 = S[3 * k], s1 = S[3 * k + 1], s2 = S[3 * k + 2];
    out[3 * k] = -kInv4Pi * (x.y * s2 - x.z * s1);
    out[3 * k + 1] = -kInv4Pi * (x.z * s0 - x.x * s2);
    out[3 * k + 2] = -kInv4Pi * (x.x * s1 - x.y * s0);
  } else {
    out[k] = -kInv4Pi * S[k];
  }
}

__global__ void k_direct_tiles(int64_t n, Tile* tiles, SrcRange* range) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nt = (n + kTileTargets - 1) / kTileTargets;
  if (t == 0) *range = SrcRange{0, static_cast<int>(n), 1, 0};
  if (t >= nt) return;
  const int64_t rem = n - t * kTileTargets;
  // one range [0, n): the self source of target i sits at flattened position i
  tiles[t] = Tile{static_cast<int>(t * kTileTargets), static_cast<int>(rem < kTileTargets ? rem : kTileTargets), 0, 1,
                  static_cast<int>(n), 0, 1, static_cast<int>(n)};
}

template <int KER, int CHUNK>
constexpr size_t tile_smem() {
  return kStages * sizeof(double4) * (CHUNK + kPad) + sizeof(int2) * kRangeCap +
         (KER == kLOG ? sizeof(double2) * kLogTabN * kLogTabCopies : 0);
}
// the log tiles stream smaller chunks so that the 16 KB log table (8 copies)
// still fits four blocks per SM
#ifndef SSUM_LOG_CHUNK
#define SSUM_LOG_CHUNK 512
#endif
constexpr int kLogChunk = SSUM_LOG_CHUNK;

// k_tiles instantiation with its dynamic shared-memory limit raised. The
// attribute belongs to the device (context), not the process: a per-device
// bit records where it is set, so a context on a second device raises it
// there too before its first launch.
template <int KER, int MODE, int NTH, int CHUNK, int MINB>
auto tiles_kernel(int device) {
  static std::atomic<unsigned long long> ready{0};
  const unsigned long long bit = 1ull << (device & 63);
  if (!(ready.load(std::memory_order_acquire) & bit)) {
    SSUM_CUDA_CHECK(cudaFuncSetAttribute(k_tiles<KER, MODE, NTH, CHUNK, MINB>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(tile_smem<KER, CHUNK>())));
    ready.fetch_or(bit, std::memory_order_acq_rel);
  }
  return k_tiles<KER, MODE, NTH, CHUNK, MINB>;
}

}  // namespace

void launch_fit_tiles_on(Ctx& c, cudaStream_t stream, int kernel, int P, const Tile* tiles, int nfit, const int* sel,
                        const SrcRange* ranges, const int* fit_nodes, const int* pslot, double* coeff) {
  if (kernel == kBS)
    tiles_kernel<kBS, kFitMode, kFitThreads, kFitChunk, kFitMinB>(c.device)
        <<<nfit, kFitThreads, tile_smem<kBS, kFitChunk>(), stream>>>(tiles, nfit, sel, ranges, c.pts.p, nullptr,
                                                                   c.d_flags.p, fit_nodes, pslot, c.vinv.p, P, coeff,
                                                                   c.npts, nullptr);
  else
    tiles_kernel<kLOG, kFitMode, kFitThreads, kLogChunk, kFitMinB>(c.device)
        <<<nfit, kFitThreads, tile_smem<kLOG, kLogChunk>(), stream>>>(tiles, nfit, sel, ranges, c.pts.p, nullptr,
                                                                    c.d_flags.p, fit_nodes, pslot, c.vinv.p, P, coeff,
                                                                    c.npts, c.logtab.p);
}

void launch_fit_tiles(Ctx& c, cudaStream_t stream, int kernel, int P, int nfit, const int* sel) {
  Lists& L = c.lists;
  launch_fit_tiles_on(c, stream, kernel, P, L.fit_tiles.p, nfit, sel, L.fit_ranges.p, L.fit_nodes.p, L.pslot.p,
                      c.coeff.p);
}

void launch_leaf_tiles(Ctx& c, cudaStream_t stream, int kernel, const Tile* tiles, int ntl, const SrcRange* ranges, double* S,
                       bool direct) {
#define SSUM_LEAF_LAUNCH(K, M, CH, TAB)                                                                       \
  tiles_kernel<K, M, kLeafThreads, CH, kLeafMinB>(c.device)<<<ntl, kLeafThreads, tile_smem<K, CH>(), stream>>>( \
      tiles, ntl, nullptr, ranges, c.pts.p, S, c.d_flags.p, nullptr, nullptr, nullptr, 0, nullptr, c.npts, TAB)
  if (kernel == kBS) {
    if (direct)
      SSUM_LEAF_LAUNCH(kBS, kDirectMode, kLeafChunk, nullptr);
    else
      SSUM_LEAF_LAUNCH(kBS, kLeafMode, kLeafChunk, nullptr);
  } else {
    if (direct)
      SSUM_LEAF_LAUNCH(kLOG, kDirectMode, kLogChunk, c.logtab.p);
    else
      SSUM_LEAF_LAUNCH(kLOG, kLeafMode, kLogChunk, c.logtab.p);
  }
#undef SSUM_LEAF_LAUNCH
}

// Direct sum (treecode.cpp:246-264): every target against one range [0, n)
// in the caller's order.
void launch_direct(Ctx& c, int kernel, int64_t n, double* d_out) {
  const int64_t nt = (n + kTileTargets - 1) / kTileTargets;
  c.direct_tiles.ensure(size_t(nt));
  c.direct_range.ensure(1);
  const int bs = 256;
  k_direct_tiles<<<grid_for(nt, bs), bs, 0, c.stream>>>(n, c.direct_tiles.p, c.direct_range.p);
  c.npts = n;
  SSUM_LAUNCH_CHECK();
  launch_leaf_tiles(c, c.stream, kernel, c.direct_tiles.p, static_cast<int>(nt), c.direct_range.p, c.S.p, true);
  SSUM_LAUNCH_CHECK();
  if (kernel == kBS)
    k_direct_finish<kBS><<<grid_for(n, bs), bs, 0, c.stream>>>(n, c.pts.p, c.S.p, d_out);
  else
    k_direct_finish<kLOG><<<grid_for(n, bs), bs, 0, c.stream>>>(n, c.pts.p, c.S.p, d_out);
  SSUM_LAUNCH_CHECK();
  c.launches += 3;
}

}  // namespace ssum
