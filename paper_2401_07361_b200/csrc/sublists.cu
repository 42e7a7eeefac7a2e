// Interaction lists per target SUBTREE: the dual traversal and the list
// compaction of traversal.cu fused into one kernel with no grid-wide step.
//
// The tree is cut into subtrees: a cut node R is the first node on a
// particle's root-to-leaf path whose bin holds <= cmax particles (or that is
// childless). One block per cut node runs the reference's traversal
// (treecode.cpp:38-77, decisions by pair_action exactly as k_bfs makes them)
// restricted to the targets that matter for R: the nodes on R's ancestor
// path (a refined path node keeps only its child towards R) and every node
// of R's subtree (all four children kept). The restricted breadth-first
// order is the global one filtered to those targets (parents are processed
// in order and children appended in order), so each target's emissions come
// out in exactly the order the global traversal + stable grouping gives
// them (traversal.cu k_mark / sort / k_seg_bounds). The block then groups
// its emissions by (target, class) with a shared-memory radix sort and
// builds, like k_leaf_fill / k_fit_fill, the range list of every leaf of R
// (PP/PC entries along the leaf's whole root-to-leaf path) and of every fit
// node it owns (CP/CC entries) — the same tiles and ranges, in the same
// order, as the global path; only where the ranges sit in memory differs.
//
// Versus the global path (cooperative k_bfs with two grid barriers per step,
// a device radix sort of all emissions, range lists built from global
// memory, three host read-backs in between) this is one launch, block-local
// barriers only, and no host read-back until the evaluation's end. The
// price is the path pairs, decided once per cut node instead of once.
//
// Proxy slots are given to every node whose bin exceeds N_T (the only nodes
// that can carry weights or fits, classify(), treecode.cpp:29-36) when the
// tree is binned, so the upward pass does not wait for the traversal.
//
// A block whose emissions or frontier outgrow its shared memory, or a range
// list that outgrows its buffer, writes empty tiles and raises
// kFlagListsRedo; the caller then redoes the evaluation on the global path.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>

#include "internal.cuh"
#include "travdev.cuh"

namespace ssum {

namespace {

#ifndef SSUM_SUB_THREADS
#define SSUM_SUB_THREADS 64
#endif
#ifndef SSUM_SUB_MINB
#define SSUM_SUB_MINB 12
#endif
#ifndef SSUM_SUB_CMAX_DEFAULT
#define SSUM_SUB_CMAX_DEFAULT 256
#endif
constexpr int kSubThreads = SSUM_SUB_THREADS;
constexpr int kSubWarps = kSubThreads / 32;
#ifndef SSUM_SUB_ECAP
#define SSUM_SUB_ECAP 1024
#endif
#ifndef SSUM_SUB_FCAP
#define SSUM_SUB_FCAP 512
#endif
constexpr int kEcap = SSUM_SUB_ECAP;  // emissions per block
constexpr int kFcap = SSUM_SUB_FCAP;  // frontier entries per step
constexpr int kIpt = kEcap / kSubThreads;
constexpr int kIdxBits = kEcap <= 1024 ? 10 : 12;  // emission index bits of a sort key
static_assert(kEcap <= (1 << kIdxBits), "emission index bits");
constexpr int kLvlBits = 6;           // level below R (< 64: max_depth <= 40)
constexpr int kMaxChain = 48;         // root-to-leaf path nodes (max_depth <= 40)
constexpr int kFitSegCap = 256;       // fit segments per block

typedef cub::BlockRadixSort<unsigned, kSubThreads, kIpt> SubSort;
typedef cub::BlockScan<int, kSubThreads> SubScan;

#ifndef SSUM_SUB_PER
#define SSUM_SUB_PER 2
#endif
constexpr int kPer = SSUM_SUB_PER;  // frontier entries per thread per round
constexpr int kSubRetrial = 512;  // calls before the builders are timed again

// the four ints of a node record (cnt, off, level, child_base): one 16-byte load
__device__ __forceinline__ int4 rec_ints(const NodeRec* __restrict__ rec, int t) {
  return __ldg(reinterpret_cast<const int4*>(&rec[t].cnt));
}

struct SubArgs {
  const int *cnt, *off, *level, *child_base, *parent;
  const double *center, *radius;
  const NodeRec* rec;
  double pi_theta;
  double theta;
  int thr, max_depth, pc_only;
  const MacCtl* mac;
  const int* cut;
  const int *leaves, *leaf_pos;
  int nl;
  const int* tile_off;
  const int* pslot;
  int64_t N;
  int P;
  int rp0, rp1;
  SrcRange* leaf_ranges;
  long long leaf_cap;
  SrcRange* fit_ranges;
  long long fit_cap;
  unsigned long long* cursor;  // [0] leaf ranges, [1] fit ranges
  Tile* leaf_tiles;
  ulonglong2* leaf_cost;
  Tile* fit_tiles;
  ulonglong2* fit_cost;
  unsigned char* is_fit;
  unsigned char* is_weight;  // optional: marks the PC / CC sources of the lists built
  unsigned long long* counters;  // traversal.cu layout + [8] fit nodes, [12] max emissions, [13] max frontier
  int* flags;
};

// Shared memory: the emissions, and the frontier double buffer, which after
// the traversal holds the sort's scratch and then the sorted keys.
struct SubSmem {
  int2 E[kEcap];  // (target, source | kind << 30)
  union {
    int2 F[2][kFcap];
    typename SubSort::TempStorage sort;
    unsigned keys[kEcap];
  } u;
};

__device__ __forceinline__ int lower_bound_u32(const unsigned* a, int n, unsigned v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int lower_bound_i32(const int* __restrict__ a, int n, int v) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

// Sort-key target id: path nodes by level (0 .. lvlR - 1); nodes of R's
// subtree by depth-first position (bin offset, then level), so the sorted
// groups are the path root first, then R's subtree in preorder.
__device__ __forceinline__ unsigned target_local(int t, int lvl, int lvlR, int offt, int offR) {
  if (lvl < lvlR) return static_cast<unsigned>(lvl);
  return 64u + (static_cast<unsigned>(offt - offR) << kLvlBits) + static_cast<unsigned>(lvl - lvlR);
}

__global__ void __launch_bounds__(kSubThreads, SSUM_SUB_MINB) k_sub_lists(SubArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SubSmem& sm = *reinterpret_cast<SubSmem*>(smem_raw);
  __shared__ typename SubScan::TempStorage scan_tmp;
  __shared__ int spath[kMaxChain];
  __shared__ int s_info[4];  // leaf range [kf, kl), fit segments
  __shared__ int wchain[kSubWarps][kMaxChain];
  __shared__ int wlo[kSubWarps][kMaxChain];
  __shared__ int wbeg[kSubWarps][kMaxChain + 1];
  __shared__ int fseg[kFitSegCap];
  __shared__ unsigned long long s_cnt[4];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const long long clk0 = clock64();  // phase cycles: counters[14..17]
  const int R = a.cut[blockIdx.x];
  const int offR = a.off[R], cntR = a.cnt[R], lvlR = a.level[R];
  if (offR >= a.rp1 || offR + cntR <= a.rp0) return;  // outside this part (restricted call)
  const bool first_proc = offR <= a.rp0;              // owns every path node (restricted call)
  if (tid == 0) {
    int t = R;
    for (int l = lvlR - 1; l >= 0; --l) {
      t = a.parent[t];
      spath[l] = t;
    }
  }
  if (tid < 4) s_cnt[tid] = 0;
  __syncthreads();

  // ---- restricted breadth-first traversal
  int cur = 0, m = 20, ne = 0, fmax = 20;
  bool ovf = false;
  const int t0 = lvlR > 0 ? spath[0] : R;
  if (tid < 20) sm.u.F[0][tid] = make_int2(t0, tid);
  __syncthreads();
  int n_steps = 0, n_rounds = 0, n_exact = 0;
  while (m > 0) {
    int nf = 0;
    ++n_steps;
    // kPer consecutive entries per thread per round: all their node records
    // are loaded before any is decided (the step is load-latency bound)
    for (int base = 0; base < m; base += kSubThreads * kPer) {
      ++n_rounds;
      int2 p[kPer];
      NodeRec T[kPer], S[kPer];
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        const int k = base + tid * kPer + j;
        p[j] = k < m ? sm.u.F[cur][k] : make_int2(-1, -1);
        if (p[j].x >= 0) {
          T[j] = a.rec[p[j].x];
          S[j] = a.rec[p[j].y];
        }
      }
      int act[kPer], cb[kPer], v = 0;
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        act[j] = 0;
        cb[j] = -1;
        if (p[j].x >= 0)
          act[j] = pair_decide(p[j].x, p[j].y, T[j], S[j], 0, 0x7fffffff, a.theta, a.pi_theta, a.thr, a.max_depth,
                               a.pc_only, a.mac, &cb[j], &n_exact);
        // a refined target above R keeps only its child towards R
        const int nch = (act[j] & 8) ? (((act[j] & 16) && T[j].level < lvlR) ? 1 : 4) : 0;
        v += ((act[j] & 4) ? (1 << 16) : 0) | nch;
      }
      int ex, agg;
      SubScan(scan_tmp).ExclusiveSum(v, ex, agg);
      const int tot_e = agg >> 16, tot_c = agg & 0xffff;
      if (ne + tot_e > kEcap || nf + tot_c > kFcap) {
        ovf = true;  // block-uniform
        break;
      }
      int oe = ne + (ex >> 16), oc = nf + (ex & 0xffff);
#pragma unroll
      for (int j = 0; j < kPer; ++j) {
        if (act[j] & 4)
          sm.E[oe++] = make_int2(p[j].x, static_cast<int>(static_cast<unsigned>(p[j].y) | (unsigned(act[j] & 3) << 30)));
        if (act[j] & 8) {
          int2* dst = &sm.u.F[cur ^ 1][oc];
          const bool rt = (act[j] & 16) != 0;
          if (rt && T[j].level < lvlR) {
            const int lt = T[j].level + 1;
            dst[0] = make_int2(lt < lvlR ? spath[lt] : R, p[j].y);
            oc += 1;
          } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) dst[q] = rt ? make_int2(cb[j] + q, p[j].y) : make_int2(p[j].x, cb[j] + q);
            oc += 4;
          }
        }
      }
      ne += tot_e;
      nf += tot_c;
      __syncthreads();  // scan scratch reuse; this round's frontier reads done
    }
    if (ovf) break;
    __syncthreads();  // next frontier complete
    cur ^= 1;
    m = nf;
    fmax = max(fmax, m);
  }
  if (tid == 0) {
    atomicMax(&a.counters[12], static_cast<unsigned long long>(ne));
    atomicMax(&a.counters[13], static_cast<unsigned long long>(fmax));
    atomicAdd(&a.counters[18], static_cast<unsigned long long>(n_steps));
    atomicAdd(&a.counters[19], static_cast<unsigned long long>(n_rounds));
    atomicAdd(&a.counters[20], static_cast<unsigned long long>(n_exact));
  }
  // leaves of R: contiguous in depth-first order
  if (tid == 0) {
    s_info[0] = lower_bound_i32(a.leaf_pos, a.nl, offR);
    s_info[1] = lower_bound_i32(a.leaf_pos, a.nl, offR + cntR);
    s_info[2] = 0;
  }
  __syncthreads();
  const int kf = s_info[0], kl = s_info[1];
  if (ovf) {
    // empty tiles (their sums come out zero) and a redo on the global path
    if (tid == 0) atomicOr(a.flags, kFlagListsRedo);
    for (int k = kf + tid; k < kl; k += kSubThreads) {
      const int leaf = a.leaves[k], c = a.cnt[leaf], off = a.off[leaf];
      for (int j = 0; j * kTileTargets < c; ++j)
        a.leaf_tiles[a.tile_off[k] + j] =
            Tile{off + j * kTileTargets, min(kTileTargets, c - j * kTileTargets), 0, 0, 0, 0, 0, 0};
    }
    return;
  }

  const long long clk1 = clock64();
  // ---- group the emissions by (target, class), stable (index in the key)
  {
    unsigned kk[kIpt];
#pragma unroll
    for (int i = 0; i < kIpt; ++i) {
      const int e = tid * kIpt + i;
      kk[i] = 0xffffffffu;
      if (e < ne) {
        const int2 it = sm.E[e];
        const int t = it.x;
        const unsigned cls = (static_cast<unsigned>(it.y) >> 30) >= 2 ? 1u : 0u;
        const int4 ti = rec_ints(a.rec, t);  // cnt, off, level, child_base
        const unsigned loc = target_local(t, ti.z, lvlR, ti.y, offR);
        kk[i] = (((loc << 1) | cls) << kIdxBits) | static_cast<unsigned>(e);
      }
    }
    __syncthreads();  // frontier storage becomes the sort's scratch
    // only the key bits in use (+1, so the all-ones padding sorts last):
    // 27 instead of 32 at cmax 256, seven 4-bit passes instead of eight
    const unsigned loc_max = 64u + (static_cast<unsigned>(max(cntR, 1)) << kLvlBits) + 63u;
    const unsigned key_max = (((loc_max << 1) | 1u) << kIdxBits) | ((1u << kIdxBits) - 1u);
    SubSort(sm.u.sort).Sort(kk, 0, min(32, 32 - __clz(key_max) + 1));
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kIpt; ++i) sm.u.keys[tid * kIpt + i] = kk[i];
    __syncthreads();
  }
  const unsigned* keys = sm.u.keys;

  const long long clk2 = clock64();
  // ---- interaction counts per kind: each emission counted by one block
  {
    unsigned long long kc[4] = {0, 0, 0, 0};
    for (int e = tid; e < ne; e += kSubThreads) {
      const int2 it = sm.E[e];
      const int t = it.x;
      const int4 ti = rec_ints(a.rec, t);
      const bool own = ti.z >= lvlR || ti.y == offR || first_proc;
      if (own) kc[static_cast<unsigned>(it.y) >> 30]++;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      unsigned long long v = kc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(&s_cnt[k], v);
    }
  }

  // ---- leaf range lists (k_leaf_fill's order): one warp per leaf of R
  unsigned long long pp_sum = 0, pc_sum = 0;
  for (int k = kf + wid; k < kl; k += kSubWarps) {
    const int leaf = a.leaves[k];
    const NodeRec Lr = a.rec[leaf];
    const int offl = Lr.off;
    if (offl >= a.rp1 || offl + Lr.cnt <= a.rp0) continue;  // another part's leaf (warp-uniform)
    const int lvlL = Lr.level;
    const int pl = min(lvlL + 1, kMaxChain);
    if (lane == 0) {
      int t = leaf;
      for (int l = lvlL; l >= lvlR; --l) {
        if (l < kMaxChain) wchain[wid][l] = t;
        t = a.parent[t];
      }
    }
    __syncwarp();
    for (int l = lane; l < pl; l += 32) {
      const int node = l < lvlR ? spath[l] : wchain[wid][l];
      const unsigned kp = (target_local(node, l, lvlR, a.off[node], offR) << 1) << kIdxBits;
      const int lo = lower_bound_u32(keys, ne, kp);
      const int hi = lower_bound_u32(keys, ne, kp + (1u << kIdxBits));
      wlo[wid][l] = lo;
      wbeg[wid][l] = hi - lo;  // count; prefix below
    }
    __syncwarp();
    if (lane == 0) {
      int run = 0;
      for (int l = 0; l < pl; ++l) {
        const int c = wbeg[wid][l];
        wbeg[wid][l] = run;
        run += c;
      }
      wbeg[wid][pl] = run;
    }
    __syncwarp();
    const int T = wbeg[wid][pl];
    unsigned long long w0ull = 0;
    if (lane == 0) w0ull = atomicAdd(&a.cursor[0], static_cast<unsigned long long>(T));
    const long long w0 = static_cast<long long>(__shfl_sync(0xffffffffu, w0ull, 0));
    const int c = a.cnt[leaf];
    const int nt = (c + kTileTargets - 1) / kTileTargets;
    if (w0 + T > a.leaf_cap) {
      if (lane == 0) atomicOr(a.flags, kFlagListsRedo);
      for (int j = lane; j < nt; j += 32)
        a.leaf_tiles[a.tile_off[k] + j] =
            Tile{offl + j * kTileTargets, min(kTileTargets, c - j * kTileTargets), 0, 0, 0, 0, 0, 0};
      continue;
    }
    SrcRange* out = a.leaf_ranges + w0;
    ListCursor lc;
    int src_pp = 0, src_pc = 0, near_total = 0, self_shift = 0, has_self = 0;
    for (int pass = 0; pass < 2; ++pass) {  // 0: near-possible PP ranges, 1: the rest
      for (int base = 0; base < T; base += 32) {
        const int idx = base + lane;
        bool sel = false, self = false;
        int cpp = 0, cpc = 0;
        SrcRange r{0, 0, 0, 0};
        if (idx < T) {
          int q = 0;
          while (wbeg[wid][q + 1] <= idx) ++q;
          const int e = static_cast<int>(keys[wlo[wid][q] + (idx - wbeg[wid][q])] & ((1u << kIdxBits) - 1u));
          const unsigned y = static_cast<unsigned>(sm.E[e].y);
          const int s = static_cast<int>(y & 0x3fffffffu), kind = static_cast<int>(y >> 30);
          const NodeRec Sr = a.rec[s];
          const bool nr = kind == 0 && near_possible_rec(s == leaf, Lr, Sr);
          sel = nr == (pass == 0);
          if (sel) {
            if (kind == 0) {
              r.begin = Sr.off;
              r.count = Sr.cnt;
              r.near = nr ? 1 : 0;
              self = r.begin <= offl && offl < r.begin + r.count;  // holds the leaf's own particles
              cpp = r.count;
            } else {
              r.begin = static_cast<int>(a.N + static_cast<int64_t>(a.pslot[s]) * a.P);
              r.count = a.P;
              cpc = a.P;
              if (a.is_weight && pass == 1) a.is_weight[s] = 1;
            }
          }
        }
        r.pad = append_ranges(sel, r, out, lc, lane);
        const unsigned sb = __ballot_sync(0xffffffffu, self);
        if (sb) {
          const int sl = __ffs(sb) - 1;
          self_shift = __shfl_sync(0xffffffffu, r.pad - r.begin, sl);
          has_self = 1;
        }
        src_pp += __reduce_add_sync(0xffffffffu, cpp);
        src_pc += __reduce_add_sync(0xffffffffu, cpc);
      }
      if (pass == 0) near_total = lc.src;
    }
    for (int j = lane; j < nt; j += 32) {
      Tile t;
      t.tgt_begin = offl + j * kTileTargets;
      t.tgt_count = min(kTileTargets, c - j * kTileTargets);
      t.list_begin = static_cast<int>(w0);
      t.list_end = static_cast<int>(w0) + lc.w;
      t.near_total = near_total;
      t.self_shift = self_shift;
      const double rl = a.radius[leaf];
      const bool dense = near_total > 0 && 1.3 * rl * rl < kDenseSpacing * kDenseSpacing * double(c);
      t.has_self = has_self | (dense ? kTileDense : 0);
      t.total = lc.src;
      a.leaf_tiles[a.tile_off[k] + j] = t;
      const unsigned long long tc = static_cast<unsigned long long>(t.tgt_count);
      a.leaf_cost[a.tile_off[k] + j] = make_ulonglong2(tc * src_pp - tc, tc * src_pc);  // self pairs excluded
    }
    if (lane == 0) {
      pp_sum += static_cast<unsigned long long>(c) * src_pp - static_cast<unsigned long long>(c);
      pc_sum += static_cast<unsigned long long>(c) * src_pc;
    }
    __syncwarp();
  }

  const long long clk3 = clock64();
  // ---- fit lists: every class-1 group whose target this block owns
  for (int i = tid; i < ne; i += kSubThreads) {
    const unsigned g = keys[i] >> kIdxBits;
    if ((g & 1u) && (i == 0 || (keys[i - 1] >> kIdxBits) != g)) {
      const int slot = atomicAdd(&s_info[2], 1);
      if (slot < kFitSegCap) fseg[slot] = i;
    }
  }
  __syncthreads();
  const int nseg = s_info[2];
  if (nseg > kFitSegCap && tid == 0) atomicOr(a.flags, kFlagListsRedo);
  unsigned long long cp_sum = 0, cc_sum = 0, nfit = 0, down = 0;
  for (int j = wid; j < min(nseg, kFitSegCap); j += kSubWarps) {
    const int b = fseg[j];
    const unsigned g = keys[b] >> kIdxBits;
    const int e_end = lower_bound_u32(keys, ne, (g + 1u) << kIdxBits);
    const int t = sm.E[keys[b] & ((1u << kIdxBits) - 1u)].x;
    const int offt = a.off[t], cntt = a.cnt[t];
    const bool own = (a.level[t] >= lvlR && offt < a.rp1 && offt + cntt > a.rp0) || offt == offR || first_proc;
    if (!own) continue;  // warp-uniform
    const int len = e_end - b;
    unsigned long long w0ull = 0;
    if (lane == 0) w0ull = atomicAdd(&a.cursor[1], static_cast<unsigned long long>(len));
    const long long w0 = static_cast<long long>(__shfl_sync(0xffffffffu, w0ull, 0));
    const int slot = a.pslot[t];
    if (w0 + len > a.fit_cap || slot < 0) {
      if (lane == 0) atomicOr(a.flags, kFlagListsRedo);
      continue;
    }
    SrcRange* out = a.fit_ranges + w0;
    ListCursor lc;
    int ncp = 0, ncc = 0;
    for (int base = b; base < e_end; base += 32) {
      const int i = base + lane;
      int is_cp = 0, is_cc = 0;
      SrcRange r{0, 0, 0, 0};
      if (i < e_end) {
        const unsigned y = static_cast<unsigned>(sm.E[keys[i] & ((1u << kIdxBits) - 1u)].y);
        const int s = static_cast<int>(y & 0x3fffffffu), kind = static_cast<int>(y >> 30);
        if (kind == 2) {
          const int4 si = rec_ints(a.rec, s);
          r.begin = si.y;
          r.count = si.x;
          is_cp = r.count;
        } else {
          r.begin = static_cast<int>(a.N + static_cast<int64_t>(a.pslot[s]) * a.P);
          r.count = a.P;
          is_cc = 1;
          if (a.is_weight) a.is_weight[s] = 1;
        }
      }
      append_ranges(i < e_end, r, out, lc, lane);
      ncp += __reduce_add_sync(0xffffffffu, is_cp);
      ncc += __reduce_add_sync(0xffffffffu, is_cc);
    }
    if (lane == 0) {
      Tile tl;
      tl.tgt_begin = static_cast<int>(a.N + static_cast<int64_t>(slot) * a.P);
      tl.tgt_count = a.P;
      tl.list_begin = static_cast<int>(w0);
      tl.list_end = static_cast<int>(w0) + lc.w;
      tl.near_total = 0;  // CP / CC pairs are well separated
      tl.self_shift = tl.has_self = 0;
      tl.total = lc.src;
      a.fit_tiles[slot] = tl;
      const unsigned long long cp = static_cast<unsigned long long>(a.P) * static_cast<unsigned long long>(ncp);
      const unsigned long long cc =
          static_cast<unsigned long long>(a.P) * static_cast<unsigned long long>(a.P) * static_cast<unsigned long long>(ncc);
      a.fit_cost[slot] = make_ulonglong2(cp, cc);
      a.is_fit[t] = 1;
      cp_sum += cp;
      cc_sum += cc;
      nfit += 1;
      down += static_cast<unsigned long long>(cntt);
    }
    __syncwarp();
  }
  // per-block totals: one atomic each
  __syncthreads();
  if (lane == 0) {
    if (pp_sum) atomicAdd(&a.counters[4], pp_sum);
    if (pc_sum) atomicAdd(&a.counters[5], pc_sum);
    if (cp_sum) atomicAdd(&a.counters[6], cp_sum);
    if (cc_sum) atomicAdd(&a.counters[7], cc_sum);
    if (nfit) atomicAdd(&a.counters[8], nfit);
    if (down) atomicAdd(&a.counters[11], down);
  }
  if (tid < 4 && s_cnt[tid]) atomicAdd(&a.counters[tid], s_cnt[tid]);
  if (tid == 0) {
    const long long clk4 = clock64();
    atomicAdd(&a.counters[14], static_cast<unsigned long long>(clk1 - clk0));
    atomicAdd(&a.counters[15], static_cast<unsigned long long>(clk2 - clk1));
    atomicAdd(&a.counters[16], static_cast<unsigned long long>(clk3 - clk2));
    atomicAdd(&a.counters[17], static_cast<unsigned long long>(clk4 - clk3));
  }
}

// ---- plan kernels (launched by the binning, tree.cu bin_reuse) -------------

// big: bin > N_T (may carry weights or fits); cut: first node on a path with
// a bin <= cmax, or a childless one.
__global__ void k_sub_flags(int nn, const int* __restrict__ cnt, const int* __restrict__ parent,
                            const int* __restrict__ child_base, int thr, int cmax, unsigned char* __restrict__ big,
                            unsigned char* __restrict__ cutf, unsigned long long* __restrict__ up_visits) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long v = 0;
  if (id < nn) {
    const int c = cnt[id];
    const int p = parent[id];
    big[id] = c > thr ? 1 : 0;
    cutf[id] = (c > 0 && (c <= cmax || child_base[id] < 0) && (p < 0 || cnt[p] > cmax)) ? 1 : 0;
    if (c > thr) v = static_cast<unsigned long long>(c);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0 && v) atomicAdd(up_visits, v);
}

__global__ void k_sub_slots(const int* __restrict__ big, const int* __restrict__ nbig, int* __restrict__ pslot,
                            int* __restrict__ slot_node) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *nbig) {
    pslot[big[i]] = i;
    slot_node[i] = big[i];
  }
}

// tiles per leaf (entries past the leaf count: 0), for the tile-offset scan
__global__ void k_sub_leaf_tiles(int n, const int* __restrict__ nl, const int* __restrict__ leaves,
                                 const int* __restrict__ cnt, int* __restrict__ tpl) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) tpl[k] = k < *nl ? (cnt[leaves[k]] + kTileTargets - 1) / kTileTargets : 0;
}

__global__ void k_sub_total(const int* __restrict__ tile_off, const int* __restrict__ nl, int* __restrict__ out) {
  if (threadIdx.x == 0) *out = tile_off[*nl];
}

}  // namespace

// The cut, the proxy slots of the big nodes and the leaf tile offsets of a
// binning; device counts at d_out[0] big nodes, [1] cut nodes, [2] leaf
// tiles (read back with the binning's own read-back). d_nl: leaf count.
void plan_subtrees(Ctx& c, int thr, const int* d_nl, int* d_out) {
  SubPlan& S = c.sub;
  Lists& L = c.lists;
  Binned& B = c.bins;
  const int nn = c.nodes.count;
  const int bs = 256;
  S.valid = false;
  S.thr = thr;
  if (S.cmax <= 0) {
    const char* e = std::getenv("SSUM_SUB_CMAX");
    S.cmax = e ? std::min(4096, std::max(1, std::atoi(e))) : SSUM_SUB_CMAX_DEFAULT;
    // SSUM_SUB_LISTS: 0 the global traversal path only, 1 the subtree
    // builder whenever it applies; default: the subtree builder for
    // restricted multi-part calls (it traverses only the part's subtrees)
    // and up to kSubAutoN particles (measured faster there: one launch, no
    // read-backs; above it the global path's wider steps win)
    const char* d = std::getenv("SSUM_SUB_LISTS");
    S.disabled = (d && *d == '0') ? 1 : 0;
    S.forced = (d && *d == '1') ? 1 : 0;
  }
  S.big_flag.ensure(size_t(nn));
  S.cut_flag.ensure(size_t(nn));
  S.cut.ensure(size_t(nn));
  S.tpl.ensure(size_t(nn) + 1);
  S.tile_off.ensure(size_t(nn) + 1);
  S.up_visits.ensure(1);
  L.pslot.ensure(size_t(nn));
  L.weight_nodes.ensure(size_t(nn));
  c.trav.slot_node.ensure(size_t(nn));
  SSUM_CUDA_CHECK(cudaMemsetAsync(L.pslot.p, 0xff, size_t(nn) * sizeof(int), c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(S.up_visits.p, 0, sizeof(unsigned long long), c.stream));
  k_sub_flags<<<grid_for(nn, bs), bs, 0, c.stream>>>(nn, B.cnt.p, c.nodes.parent.p, c.nodes.child_base.p, thr,
                                                     S.cmax, S.big_flag.p, S.cut_flag.p, S.up_visits.p);
  SSUM_LAUNCH_CHECK();
  cub::CountingInputIterator<int> ids(0);
  size_t t1 = 0, t2 = 0, t3 = 0;
  SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, t1, ids, S.big_flag.p, L.weight_nodes.p, d_out, nn, c.stream));
  SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, t2, ids, S.cut_flag.p, S.cut.p, d_out + 1, nn, c.stream));
  SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, t3, S.tpl.p, S.tile_off.p, nn + 1, c.stream));
  c.cub_tmp.ensure(std::max(t1, std::max(t2, t3)));
  SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(c.cub_tmp.p, t1, ids, S.big_flag.p, L.weight_nodes.p, d_out, nn,
                                             c.stream));
  SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(c.cub_tmp.p, t2, ids, S.cut_flag.p, S.cut.p, d_out + 1, nn, c.stream));
  k_sub_slots<<<grid_for(nn, bs), bs, 0, c.stream>>>(L.weight_nodes.p, d_out, L.pslot.p, c.trav.slot_node.p);
  SSUM_LAUNCH_CHECK();
  k_sub_leaf_tiles<<<grid_for(nn + 1, bs), bs, 0, c.stream>>>(nn + 1, d_nl, B.d_leaves.p, B.cnt.p, S.tpl.p);
  SSUM_LAUNCH_CHECK();
  SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, t3, S.tpl.p, S.tile_off.p, nn + 1, c.stream));
  k_sub_total<<<1, 32, 0, c.stream>>>(S.tile_off.p, d_nl, d_out + 2);
  SSUM_LAUNCH_CHECK();
  c.launches += 9;
}

// Host counts of the plan (after the binning's read-back).
void plan_subtrees_done(Ctx& c, const int* h) {
  SubPlan& S = c.sub;
  S.n_big = h[0];
  S.n_cut = h[1];
  S.n_leaf_tiles = h[2];
  S.valid = true;
}

// Which list builder this call uses: 0 the global path, 1 the subtree
// builder; +2: a timed trial (sub_lists_timed reports its device time).
// Restricted (multi-part) calls always take the subtree builder (it
// traverses only the part's subtrees). Otherwise the choice is measured:
// which builder is faster depends on the tree's shape (the subtree
// builder's blocks replay their ancestor paths; the global traversal pays
// grid-wide steps and read-backs) — on the BASELINE meshes it wins up to
// C2's size and loses at C4's, on the random cap it loses at 2^20 — so the
// first evaluations of a particle count alternate the two, timing each
// twice, and the faster one serves the next kSubRetrial calls.
int sub_lists_choice(Ctx& c, const ssum_config& cfg) {
  SubPlan& S = c.sub;
  const bool usable = S.valid && !S.disabled && S.thr == cfg.n_threshold && c.bins.n > 0 && c.bins.n_leaves > 0 &&
                      S.n_cut > 0 && c.nodes.max_level < kMaxChain - 1 && c.nodes.count < (1 << 30);
  if (!usable) return 0;
  if (S.forced) return 1;
  // a block outgrew its shared memory for this particle count (deep or
  // dense trees: long replayed paths): the global path from now on
  if (S.bad_n == c.bins.n) return 0;
  if (c.restrict_on) return 1;
  if (S.trial_n != c.bins.n || S.trial_calls >= kSubRetrial || S.trial_theta != cfg.theta) {
    S.trial_n = c.bins.n;
    S.trial_theta = cfg.theta;
    S.trial_calls = 0;
    S.trial_cnt[0] = S.trial_cnt[1] = 0;
    S.trial_ms[0] = S.trial_ms[1] = 0.0;
  }
  ++S.trial_calls;
  // one sample each decides when they differ by more than 25%; otherwise a
  // second (warm) sample each is compared
  const bool clear = S.trial_cnt[0] >= 1 && S.trial_cnt[1] >= 1 &&
                     (S.trial_ms[0] > 1.25 * S.trial_ms[1] || S.trial_ms[1] > 1.25 * S.trial_ms[0]);
  if (!clear && (S.trial_cnt[0] < 2 || S.trial_cnt[1] < 2)) return 2 + (S.trial_cnt[1] <= S.trial_cnt[0] ? 1 : 0);
  return S.trial_ms[1] <= S.trial_ms[0] ? 1 : 0;
}

// A trial's device time (lists + evaluation); the second sample of each
// builder is the one compared (the first may include buffer growth).
void sub_lists_timed(Ctx& c, int used_sub, double ms) {
  SubPlan& S = c.sub;
  S.trial_ms[used_sub] = ms;
  S.trial_cnt[used_sub]++;
  if (trace().on)
    std::fprintf(stderr, "[ssum sub] trial %s %.3f ms (global %.3f x%d, subtree %.3f x%d)\n",
                 used_sub ? "subtree" : "global", ms, S.trial_ms[0], S.trial_cnt[0], S.trial_ms[1], S.trial_cnt[1]);
}

// The lists of this call from the plan (see the file comment); no host
// read-back. The upward pass starts first, on the side stream.
void build_lists_subtree(Ctx& c, const ssum_config& cfg) {
  SubPlan& S = c.sub;
  Lists& L = c.lists;
  Binned& B = c.bins;
  TravScratch& TS = c.trav;
  const int64_t N = B.n;
  const int P = (cfg.degree + 1) * (cfg.degree + 2) / 2;
  const int nn = c.nodes.count;
  L.n_inter = 0;
  for (int k = 0; k < 4; ++k) L.counts[k] = L.evals[k] = 0;
  L.n_proxy = L.n_weight = S.n_big;
  L.n_fit = 0;
  L.n_fit_tiles = S.n_big;
  L.n_leaf_tiles = S.n_leaf_tiles;
  S.used = true;
  // restricted (multi-part) call: the upward pass only for the sources this
  // part's lists use, marked by the builder (it then follows the builder);
  // otherwise every big node's, beside the builder
  const bool lean_up = c.restrict_on;
  c.up_list = nullptr;
  c.up_count = nullptr;
  if (lean_up) {
    L.is_weight.ensure(size_t(nn));
    SSUM_CUDA_CHECK(cudaMemsetAsync(L.is_weight.p, 0, size_t(nn), c.stream));
  }

  const MacCtl* mac = reinterpret_cast<const MacCtl*>(mac_ctl_device(c));
  build_node_records(c, cfg.theta);
  TS.counters.ensure(24);
  SSUM_CUDA_CHECK(cudaMemsetAsync(TS.counters.p, 0, 21 * sizeof(unsigned long long), c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(TS.counters.p + 10, S.up_visits.p, 8, cudaMemcpyDeviceToDevice, c.stream));
  L.is_fit.ensure(size_t(nn));
  SSUM_CUDA_CHECK(cudaMemsetAsync(L.is_fit.p, 0, size_t(nn), c.stream));
  const size_t nfit = std::max(S.n_big, 1);
  L.fit_tiles.ensure(nfit);
  L.fit_cost.ensure(nfit);
  L.fit_nodes.ensure(nfit);
  SSUM_CUDA_CHECK(cudaMemsetAsync(L.fit_tiles.p, 0, nfit * sizeof(Tile), c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(L.fit_cost.p, 0, nfit * sizeof(ulonglong2), c.stream));
  if (S.n_big > 0)
    SSUM_CUDA_CHECK(cudaMemcpyAsync(L.fit_nodes.p, L.weight_nodes.p, size_t(S.n_big) * 4, cudaMemcpyDeviceToDevice,
                                    c.stream));
  const size_t ntl = std::max(S.n_leaf_tiles, 1);
  L.leaf_tiles.ensure(ntl);
  L.leaf_cost.ensure(ntl);
  // range buffers: the last call's use plus slack (first call: from N)
  if (S.leaf_cap == 0) {
    S.leaf_cap = std::max<int64_t>(64 * int64_t(B.n_leaves) + 65536, 1 << 20);
    S.fit_cap = std::max<int64_t>(64 * int64_t(S.n_big) + 65536, 1 << 18);
  }
  L.leaf_ranges.ensure(size_t(S.leaf_cap));
  L.fit_ranges.ensure(size_t(S.fit_cap));
  S.cursor.ensure(2);
  SSUM_CUDA_CHECK(cudaMemsetAsync(S.cursor.p, 0, 2 * sizeof(unsigned long long), c.stream));

  if (S.smem == 0) {
    S.smem = static_cast<int>(sizeof(SubSmem));
    SSUM_CUDA_CHECK(cudaFuncSetAttribute(k_sub_lists, cudaFuncAttributeMaxDynamicSharedMemorySize, S.smem));
  }
  SubArgs a;
  a.cnt = B.cnt.p;
  a.off = B.off.p;
  a.level = c.nodes.level.p;
  a.child_base = c.nodes.child_base.p;
  a.parent = c.nodes.parent.p;
  a.center = c.nodes.center.p;
  a.radius = c.nodes.radius.p;
  a.rec = c.trav.rec.p;
  a.pi_theta = kPi * cfg.theta * (1.0 - 1e-12);
  a.theta = cfg.theta;
  a.thr = cfg.n_threshold;
  a.max_depth = cfg.max_depth;
  a.pc_only = cfg.pc_only;
  a.mac = mac;
  a.cut = S.cut.p;
  a.leaves = B.d_leaves.p;
  a.leaf_pos = B.leaf_pos.p;
  a.nl = B.n_leaves;
  a.tile_off = S.tile_off.p;
  a.pslot = L.pslot.p;
  a.N = N;
  a.P = P;
  a.rp0 = c.restrict_on ? static_cast<int>(c.rp0) : 0;
  a.rp1 = c.restrict_on ? static_cast<int>(c.rp1) : 0x7fffffff;
  a.leaf_ranges = L.leaf_ranges.p;
  a.leaf_cap = S.leaf_cap;
  a.fit_ranges = L.fit_ranges.p;
  a.fit_cap = S.fit_cap;
  a.cursor = S.cursor.p;
  a.leaf_tiles = L.leaf_tiles.p;
  a.leaf_cost = L.leaf_cost.p;
  a.fit_tiles = L.fit_tiles.p;
  a.fit_cost = L.fit_cost.p;
  a.is_fit = L.is_fit.p;
  a.is_weight = lean_up ? L.is_weight.p : nullptr;
  a.counters = TS.counters.p;
  a.flags = c.d_flags.p;
  // the prep stream forks here (its inputs exist; buffers sized before), so
  // the proxy points + upward pass of every big node (low-priority stream)
  // run beside the list builder's latency-bound blocks
  if (c.early.xyz) size_eval_buffers(c, c.early.degree, c.early.dim, N);
  SSUM_CUDA_CHECK(cudaEventRecord(c.fork_ev, c.stream));
  // restricted call: the prep follows the builder (the upward pass needs its
  // marks; running the gather and proxy points beside it measured no faster)
  k_sub_lists<<<S.n_cut, kSubThreads, S.smem, c.stream>>>(a);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  if (lean_up) {
    // the marked sources, in node-id order, with their device count
    S.wsel.ensure(size_t(nn) + 1);
    cub::CountingInputIterator<int> ids(0);
    size_t tb = 0;
    SSUM_CUDA_CHECK(
        cub::DeviceSelect::Flagged(nullptr, tb, ids, L.is_weight.p, S.wsel.p + 1, S.wsel.p, nn, c.stream));
    c.cub_tmp.ensure(tb);
    SSUM_CUDA_CHECK(
        cub::DeviceSelect::Flagged(c.cub_tmp.p, tb, ids, L.is_weight.p, S.wsel.p + 1, S.wsel.p, nn, c.stream));
    c.launches += 2;
    c.up_list = S.wsel.p + 1;
    c.up_count = S.wsel.p;
    start_prep(c, false, 3);
  } else {
    start_prep(c, true, 3);
  }
  // counts, evaluations, visits and the range use: read back with the
  // evaluation's final sync (finalize_counts / sub_lists_check)
  SSUM_CUDA_CHECK(cudaMemcpyAsync(TS.h_small + 8, TS.counters.p, 21 * sizeof(unsigned long long),
                                  cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(TS.h_small + 29, S.cursor.p, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  c.stream));
  TS.h_small[31] = 0;
  SSUM_CUDA_CHECK(cudaMemcpyAsync(TS.h_small + 31, c.mac.amb_n.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  L.counts_pending = true;
  // this part's tiles
  if (c.restrict_on) {
    L.leaf_t0 = c.rt0;
    L.leaf_t1 = c.rt1;
  }
  partition_targets(c);
  if (c.restrict_on) {
    L.leaf_t0 = c.rt0;
    L.leaf_t1 = c.rt1;
  }
}

// After the evaluation's final sync: whether the subtree lists of this call
// were incomplete (a buffer outgrew; the MAC guard band met undecided
// pairs), in which case the caller redoes the evaluation on the global path.
// Also sizes the next call's range buffers and, after repeated block
// overflows, halves the cut size.
bool sub_lists_redo(Ctx& c, int flags) {
  SubPlan& S = c.sub;
  if (!S.used) return false;
  S.used = false;
  const unsigned long long* h = c.trav.h_small;
  const int64_t lu = static_cast<int64_t>(h[29]), fu = static_cast<int64_t>(h[30]);
  S.max_emit = static_cast<int64_t>(h[8 + 12]);
  S.max_front = static_cast<int64_t>(h[8 + 13]);
  c.lists.n_fit = static_cast<int>(h[8 + 8]);
  const bool ranges_out = lu > S.leaf_cap || fu > S.fit_cap;  // this call's capacities
  bool grown = false;  // a range buffer outgrew (or nearly): larger next time
  if (lu + lu / 4 > S.leaf_cap) S.leaf_cap = lu + lu / 2 + 65536, grown = true;
  if (fu + fu / 4 > S.fit_cap) S.fit_cap = fu + fu / 2 + 65536, grown = true;
  bool redo = (flags & kFlagListsRedo) != 0;
  // a block outgrew its shared memory: smaller subtrees next time
  if (redo && !ranges_out) {
    S.bad_n = c.bins.n;  // auto mode: the global path for this particle count
    if (S.forced) S.cmax = std::max(16, S.cmax / 2);  // forced: retry with smaller cuts
  }
  const int amb = *reinterpret_cast<const int*>(h + 31);  // undecided MAC pairs met
  if (amb > 0 && resolve_mac_host(c)) redo = true;
  if (trace().on)
    std::fprintf(stderr, "[ssum sub] cut %d big %d leaf tiles %d | max emissions %lld frontier %lld | ranges %lld/%lld "
                 "fit %lld/%lld | flags %d amb %d redo %d grown %d cmax %d | kcyc/block bfs %.1f sort %.1f leaf %.1f fit %.1f | per block steps %.1f rounds %.1f exact %.2f\n", S.n_cut, S.n_big, S.n_leaf_tiles,
                 (long long)S.max_emit, (long long)S.max_front, (long long)lu, (long long)S.leaf_cap, (long long)fu,
                 (long long)S.fit_cap, flags, amb, redo ? 1 : 0, grown ? 1 : 0, S.cmax, 1e-3 * h[22] / S.n_cut,
                 1e-3 * h[23] / S.n_cut, 1e-3 * h[24] / S.n_cut, 1e-3 * h[25] / S.n_cut, double(h[26]) / S.n_cut, double(h[27]) / S.n_cut,
                 double(h[28]) / S.n_cut);
  if (redo) S.redos++;
  return redo;
}

}  // namespace ssum
