// Dual tree traversal and interaction-list compaction on the device.
//
// dual_traversal / traverse / classify / mac_well_separated
// (treecode.cpp:22-77) are restated breadth-first: every step evaluates the
// whole frontier of (target, source) node pairs at once. A pair is dropped
// when either bin is empty (:42), emitted with classify()'s kind when
// (r_t + r_s)/R < theta with R > 0 (:22-25, :43-45), emitted as PP when both
// bins are <= N_T (:47-50), and otherwise the node with the larger bin (ties:
// source, :52) is refined into its 4 children, or the pair falls back to PP
// when that node has no children or sits at max_depth (:54-57). Each emitted
// pair carries a depth-first order key (root pair, then 2 bits per
// refinement) so the reference's emission order can be reproduced on export.
//
// The emitted list is then compacted into the evaluation layout:
//   * leaf tiles  (<= 256 target particles each) with a list of source ranges
//     gathered over the leaf's root-to-leaf path: PP ranges (particles of the
//     source bin, contiguous in tree order) and PC ranges (the source node's
//     proxy points) — treecode.cpp:366-396;
//   * fit tiles   (the p proxy points of a CP/CC target node) with CP ranges
//     (particles) and CC ranges (proxy points) — treecode.cpp:341-358;
//   * proxy slots for every node that needs proxy points (PC/CC sources carry
//     weights, CP/CC targets carry fit coefficients) — treecode.cpp:289-324.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "internal.cuh"
#include "travdev.cuh"

namespace ssum {

namespace {

// Emission / refinement of frontier entry p with action a at exclusive
// prefix pos = (emissions before << 32) | (children slots before).
__device__ __forceinline__ void pair_scatter(const PairEntry& p, int a, unsigned long long pos, long long e_base,
                                             const int* __restrict__ child_base, PairEntry* __restrict__ Fnext,
                                             int4* __restrict__ E, unsigned long long* __restrict__ K, int* flags) {
  if (a & 4) {
    const long long e = e_base + static_cast<long long>(pos >> 32);
    E[e] = int4{p.t, p.s, a & 3, 0};
    K[e] = p.key;
  } else {
    const int o = static_cast<int>(pos & 0xffffffffull);
    const bool rt = (a & 16) != 0;
    const int cb = child_base[rt ? p.t : p.s];
    const int step = p.step + 1;
    if (step > kKeyMaxSteps) atomicOr(flags, 4);  // order keys saturated (export only)
    const int shift = 54 - kKeyStepBits * min(step, kKeyMaxSteps);
    for (int q = 0; q < 4; ++q) {
      PairEntry c;
      c.t = rt ? cb + q : p.t;
      c.s = rt ? p.s : cb + q;
      c.key = p.key | (static_cast<unsigned long long>(q) << shift);
      c.step = step;
      c.pad = 0;
      Fnext[o + q] = c;
    }
  }
}
// One step of the breadth-first traversal, host-sized (bfs_synchronous):
// decide every frontier pair; packed[k] = (emits << 32) | child slots, and
// packed[m] = 0 so that the exclusive scan's entry m is the total.
__global__ void k_trav_eval(const PairEntry* __restrict__ F, int m, const int* __restrict__ cnt,
                            const int* __restrict__ off, int rlo, int rhi, const double* __restrict__ center,
                            const double* __restrict__ radius,
                            const int* __restrict__ level, const int* __restrict__ child_base, double theta, int thr,
                            int max_depth, int pc_only, const MacCtl* mac, int* __restrict__ action,
                            unsigned long long* __restrict__ packed, const NodeRec* __restrict__ rec, double pi_theta) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > m) return;
  if (k == m) {
    packed[k] = 0;
    return;
  }
  int cb, tl;
  const int a = pair_action_rec(F[k].t, F[k].s, rec, rlo, rhi, theta, pi_theta, thr, max_depth, pc_only, mac, &cb, &tl);
  action[k] = a;
  packed[k] = ((a & 4) ? (1ull << 32) : 0ull) | ((a & 8) ? 4ull : 0ull);
}

// ... and emit / refine at the scanned positions.
__global__ void k_trav_scatter(const PairEntry* __restrict__ F, int m, const int* __restrict__ action,
                               const unsigned long long* __restrict__ scan, const int* __restrict__ child_base,
                               PairEntry* __restrict__ Fnext, int4* __restrict__ E, unsigned long long* __restrict__ K,
                               long long e_base, int* flags) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int a = action[k];
  if (a) pair_scatter(F[k], a, scan[k], e_base, child_base, Fnext, E, K, flags);
}

__global__ void k_root_pairs(PairEntry* F) {
  const int k = threadIdx.x + blockIdx.x * blockDim.x;
  if (k >= 400) return;
  PairEntry p;
  p.t = k / 20;
  p.s = k % 20;
  p.key = static_cast<unsigned long long>(k) << 54;
  p.step = 0;
  p.pad = 0;
  F[k] = p;
}

// The whole breadth-first traversal in one cooperative launch (all blocks
// resident): per step, each block takes a contiguous slice of the frontier,
// decides every pair (pair_action) and scans its slice; after a grid barrier
// every block reads all block totals (its base = the totals of the blocks
// before it, so emissions and children keep frontier order exactly as the
// step-by-step version) and scatters; a second barrier hands the next
// frontier over. Capacities come from the previous call; a step that would
// exceed them stops the walk with out[1] = 1 (the caller then redoes the
// traversal step by step). out: [0] steps, [1] overflow, [2] largest frontier.
constexpr int kBfsThreads = 256;
#ifndef SSUM_BFS_MINB
#define SSUM_BFS_MINB 4
#endif
__global__ void __launch_bounds__(kBfsThreads, SSUM_BFS_MINB)
    k_bfs(const int* __restrict__ cnt, const int* __restrict__ off, int rlo, int rhi,
          const double* __restrict__ center, const double* __restrict__ radius,
          const int* __restrict__ level, const int* __restrict__ child_base, double theta, int thr, int max_depth,
          int pc_only, const MacCtl* mac, PairEntry* F0, PairEntry* F1, int fcap, int4* __restrict__ E,
          unsigned long long* __restrict__ K, long long ecap, int* __restrict__ action,
          unsigned long long* __restrict__ loc, unsigned long long* btot, int* out, long long* ne_out,
          int* flags, const NodeRec* __restrict__ rec, double pi_theta) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  typedef cub::BlockScan<unsigned long long, kBfsThreads> BS;
  typedef cub::BlockReduce<unsigned long long, kBfsThreads> BR;
  __shared__ union {
    typename BS::TempStorage scan;
    typename BR::TempStorage red;
  } tmp;
  const int nb = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
  PairEntry* Fc = F0;
  PairEntry* Fn = F1;
  int m = 400, fmax = 400;
  long long e_base = 0;
  for (int step = 0;; ++step) {
    const int per = (m + nb - 1) / nb;
    const int lo = min(m, b * per), hi = min(m, lo + per);
    unsigned long long run = 0;  // (emissions << 32) | child slots, this block so far
    // decide the whole slice first (no block-wide sync between pairs, so
    // each thread keeps several pairs' node loads in flight), then scan it
#pragma unroll 4
    for (int k = lo + tid; k < hi; k += kBfsThreads) {
      int cb, tl;
      action[k] = pair_action_rec(Fc[k].t, Fc[k].s, rec, rlo, rhi, theta, pi_theta, thr, max_depth, pc_only, mac, &cb,
                                  &tl);
    }
    for (int base = lo; base < hi; base += kBfsThreads) {
      const int k = base + tid;
      unsigned long long v = 0;
      if (k < hi) {
        const int a = action[k];  // this thread's own store
        v = ((a & 4) ? (1ull << 32) : 0ull) | ((a & 8) ? 4ull : 0ull);
      }
      unsigned long long ex, agg;
      BS(tmp.scan).ExclusiveSum(v, ex, agg);
      __syncthreads();
      if (k < hi) loc[k] = run + ex;
      run += agg;
    }
    if (tid == 0) btot[b] = run;
    grid.sync();
    unsigned long long below = 0, all = 0;
    for (int i = tid; i < nb; i += kBfsThreads) {
      const unsigned long long t = btot[i];
      all += t;
      if (i < b) below += t;
    }
    below = BR(tmp.red).Sum(below);
    __syncthreads();
    all = BR(tmp.red).Sum(all);
    __shared__ unsigned long long s_below, s_all;
    if (tid == 0) {
      s_below = below;
      s_all = all;
    }
    __syncthreads();
    below = s_below;
    all = s_all;
    const int next = static_cast<int>(all & 0xffffffffull);
    const long long emitted = static_cast<long long>(all >> 32);
    const bool ovf = next > fcap || e_base + emitted > ecap;
    if (!ovf)
      for (int k = lo + tid; k < hi; k += kBfsThreads) {
        const int a = action[k];
        if (a) pair_scatter(Fc[k], a, below + loc[k], e_base, child_base, Fn, E, K, flags);
      }
    e_base += emitted;
    if (ovf || next == 0) {
      if (b == 0 && tid == 0) {
        out[0] = step + 1;
        out[1] = ovf ? 1 : 0;
        out[2] = fmax;
        *ne_out = e_base;
      }
      break;
    }
    fmax = max(fmax, next);
    grid.sync();  // the next frontier is complete, and btot is free again
    PairEntry* t = Fc;
    Fc = Fn;
    Fn = t;
    m = next;
  }
}

// Upward / downward pass visits: bin sizes of the weight nodes and of the
// fit nodes (counters[0], counters[1]).
// is_fit (planned lists: fit_nodes lists every big node): only the fit
// nodes count, and their number goes to counters[-2].
__global__ void k_visits(const int* __restrict__ weight_nodes, int nw, const int* __restrict__ fit_nodes, int nf,
                         const int* __restrict__ cnt, unsigned long long* counters,
                         const unsigned char* __restrict__ is_fit) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long up = 0, down = 0, nfit = 0;
  if (k < nw) {
    up = static_cast<unsigned long long>(cnt[weight_nodes[k]]);
  } else if (k < nw + nf) {
    const int id = fit_nodes[k - nw];
    if (!is_fit || is_fit[id]) down = static_cast<unsigned long long>(cnt[id]), nfit = 1;
  }
  typedef cub::BlockReduce<unsigned long long, 256> BR;
  __shared__ typename BR::TempStorage tmp;
  up = BR(tmp).Sum(up);
  __syncthreads();
  down = BR(tmp).Sum(down);
  __syncthreads();
  nfit = BR(tmp).Sum(nfit);
  if (threadIdx.x == 0) {
    if (up) atomicAdd(&counters[0], up);
    if (down) atomicAdd(&counters[1], down);
    if (is_fit && nfit) atomicAdd(&counters[-2], nfit);
  }
}

// Node flags from the emitted list (treecode.cpp:295-317).
__global__ void k_mark(const int4* __restrict__ E, long long ne, unsigned char* is_weight, unsigned char* is_fit,
                       int* group_key, int* group_val, unsigned long long* kind_counts) {
  __shared__ unsigned int sc[4];
  if (threadIdx.x < 4) sc[threadIdx.x] = 0;
  __syncthreads();
  const long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  int kind = -1;
  if (e < ne) {
    const int4 it = E[e];
    kind = it.z;
    if (kind == 1 || kind == 3) is_weight[it.y] = 1;
    if (kind == 2 || kind == 3) is_fit[it.x] = 1;
    group_key[e] = 2 * it.x + ((kind >= 2) ? 1 : 0);
    group_val[e] = static_cast<int>(e);
  }
  // per-kind counts: warp ballots, one shared atomic per warp and kind
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const unsigned m = __ballot_sync(0xffffffffu, kind == k);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&sc[k], static_cast<unsigned>(__popc(m)));
  }
  __syncthreads();
  if (threadIdx.x < 4 && sc[threadIdx.x]) atomicAdd(&kind_counts[threadIdx.x], static_cast<unsigned long long>(sc[threadIdx.x]));
}

__global__ void k_slot_flags(const unsigned char* is_weight, const unsigned char* is_fit, int nn, int* flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nn) flag[k] = (is_weight[k] | is_fit[k]) ? 1 : 0;
}

__global__ void k_slots(const int* __restrict__ flag, const int* __restrict__ scan, int nn,
                        const unsigned char* is_weight, const unsigned char* is_fit, int* pslot,
                        int* slot_node) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nn) return;
  if (flag[k]) {
    pslot[k] = scan[k];
    slot_node[scan[k]] = k;
  } else {
    pslot[k] = -1;
  }
}

// Segment bounds of the sorted group keys (key = 2*node + class, class 1 = CP/CC):
// seg[key] = (begin, end) into the sorted emission order.
__global__ void k_seg_bounds(const int* __restrict__ keys, long long ne, int2* seg) {
  const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (i >= ne) return;
  const int k = keys[i];
  if (i == 0 || keys[i - 1] != k) seg[k].x = static_cast<int>(i);
  if (i == ne - 1 || keys[i + 1] != k) seg[k].y = static_cast<int>(i + 1);
}

// Per leaf: number of PP/PC ranges over its root-to-leaf path, and tiles.
__global__ void k_leaf_count(const int* __restrict__ leaves, int nl, const int* __restrict__ parent,
                             const int2* __restrict__ seg, const int* __restrict__ cnt, int* n_ranges,
                             int* n_tiles) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nl) return;
  const int leaf = leaves[k];
  int r = 0;
  for (int a = leaf; a >= 0; a = parent[a]) {
    const int2 sg = seg[2 * a];
    r += sg.y - sg.x;
  }
  n_ranges[k] = r;
  n_tiles[k] = (cnt[leaf] + kTileTargets - 1) / kTileTargets;
}

// Range list of one leaf, one warp per leaf: PP and PC entries of every node
// on its root-to-leaf path (treecode.cpp:379-396), near-possible PP ranges
// first, each pass in path order (root to leaf, segment order within a
// node). Lanes take 32 entries at a time; a ballot keeps the serial order and
// a warp scan gives each range its flattened-list prefix.
constexpr int kFillWarps = 4;
__global__ void __launch_bounds__(32 * kFillWarps)
    k_leaf_fill(const int* __restrict__ leaves, int nl, const int* __restrict__ parent,
                const int2* __restrict__ seg, const int* __restrict__ sorted_e, const int4* __restrict__ E,
                const int* __restrict__ cnt, const int* __restrict__ off, const int* __restrict__ pslot,
                const double* __restrict__ center, const double* __restrict__ radius,
                const int* __restrict__ range_off, const int* __restrict__ tile_off, int64_t N, int P,
                SrcRange* __restrict__ ranges, Tile* __restrict__ tiles, ulonglong2* __restrict__ tile_cost,
                unsigned long long* __restrict__ evals, const NodeRec* __restrict__ rec) {
  __shared__ int sseg[kFillWarps][48];  // first sorted entry of each path node's segment (root first)
  __shared__ int sbeg[kFillWarps][49];  // first flattened entry of each path node (root first)
  __shared__ int spl[kFillWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int k = blockIdx.x * kFillWarps + wid;
  unsigned long long pp = 0, pc = 0;
  if (k < nl) {  // warp-uniform
    const int leaf = leaves[k];
    if (lane == 0) {
      int tmp[48];
      int pl = 0;
      for (int a = leaf; a >= 0 && pl < 48; a = parent[a]) tmp[pl++] = a;
      int run = 0;
      for (int q = 0; q < pl; ++q) {
        const int node = tmp[pl - 1 - q];
        const int2 sg = seg[2 * node];
        sseg[wid][q] = sg.x;
        sbeg[wid][q] = run;
        run += sg.y - sg.x;
      }
      sbeg[wid][pl] = run;
      spl[wid] = pl;
    }
    __syncwarp();
    const int pl = spl[wid];
    const int T = sbeg[wid][pl];
    const NodeRec Lr = rec[leaf];
    const int offl = Lr.off;
    const int w0 = range_off[k];
    ListCursor cur;
    int src_pp = 0, src_pc = 0, near_total = 0, self_shift = 0, has_self = 0;
    for (int pass = 0; pass < 2; ++pass) {  // 0: near-possible PP ranges, 1: the rest
      for (int base = 0; base < T; base += 32) {
        const int idx = base + lane;
        bool sel = false, self = false;
        int cpp = 0, cpc = 0;
        SrcRange r{0, 0, 0, 0};
        if (idx < T) {
          int q = 0;
          while (sbeg[wid][q + 1] <= idx) ++q;
          const int4 it = E[sorted_e[sseg[wid][q] + (idx - sbeg[wid][q])]];
          const NodeRec Sr = rec[it.y];
          const bool nr = it.z == 0 && near_possible_rec(it.y == leaf, Lr, Sr);
          sel = nr == (pass == 0);
          if (sel) {
            if (it.z == 0) {
              r.begin = Sr.off;
              r.count = Sr.cnt;
              r.near = nr ? 1 : 0;
              self = r.begin <= offl && offl < r.begin + r.count;  // holds the leaf's own particles
              cpp = r.count;
            } else {
              r.begin = static_cast<int>(N + static_cast<int64_t>(pslot[it.y]) * P);
              r.count = P;
              cpc = P;
            }
          }
        }
        r.pad = append_ranges(sel, r, ranges + w0, cur, lane);  // flattened-list prefix
        const unsigned sb = __ballot_sync(0xffffffffu, self);
        if (sb) {
          const int sl = __ffs(sb) - 1;
          self_shift = __shfl_sync(0xffffffffu, r.pad - r.begin, sl);
          has_self = 1;
        }
        src_pp += __reduce_add_sync(0xffffffffu, cpp);
        src_pc += __reduce_add_sync(0xffffffffu, cpc);
      }
      if (pass == 0) near_total = cur.src;
    }
    const int w = cur.w;
    const int c = cnt[leaf];
    const int nt = (c + kTileTargets - 1) / kTileTargets;
    SSUM_DCHECK(w0 + w <= range_off[k + 1]);  // within the ranges k_leaf_count sized
    for (int j = lane; j < nt; j += 32) {
      Tile t;
      t.tgt_begin = offl + j * kTileTargets;
      t.tgt_count = min(kTileTargets, c - j * kTileTargets);
      t.list_begin = w0;
      t.list_end = w0 + w;
      t.near_total = near_total;
      t.self_shift = self_shift;
      // dense leaf: estimated point spacing sqrt(area / count), area ~ 1.3 r^2
      // of the leaf triangle in its circumcircle of angular radius r
      const double rl = Lr.r;
      const bool dense = near_total > 0 && 1.3 * rl * rl < kDenseSpacing * kDenseSpacing * double(c);
      t.has_self = has_self | (dense ? kTileDense : 0);
      t.total = cur.src;
      tiles[tile_off[k] + j] = t;
      const unsigned long long tc = static_cast<unsigned long long>(t.tgt_count);
      tile_cost[tile_off[k] + j] = make_ulonglong2(tc * src_pp - tc, tc * src_pc);  // self pairs excluded
    }
    if (lane == 0) {
      pp = static_cast<unsigned long long>(c) * src_pp - static_cast<unsigned long long>(c);  // self pairs excluded
      pc = static_cast<unsigned long long>(c) * src_pc;
    }
  }
  typedef cub::BlockReduce<unsigned long long, 32 * kFillWarps> BR;
  __shared__ typename BR::TempStorage tmp;
  const unsigned long long spp = BR(tmp).Sum(pp);
  __syncthreads();
  const unsigned long long spc = BR(tmp).Sum(pc);
  if (threadIdx.x == 0) {
    atomicAdd(&evals[0], spp);
    atomicAdd(&evals[1], spc);
  }
}

__global__ void k_fit_count(const int* __restrict__ fit_nodes, int nf, const int2* __restrict__ seg, int* n_ranges) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nf) return;
  const int2 sg = seg[2 * fit_nodes[k] + 1];
  n_ranges[k] = sg.y - sg.x;
}

// Range list of one fit node (its CP / CC entries in emission order,
// treecode.cpp:341-358), one warp per node as in k_leaf_fill.
__global__ void __launch_bounds__(32 * kFillWarps)
    k_fit_fill(const int* __restrict__ fit_nodes, int nf, const int2* __restrict__ seg,
               const int* __restrict__ sorted_e, const int4* __restrict__ E, const int* __restrict__ cnt,
               const int* __restrict__ off, const int* __restrict__ pslot, const int* __restrict__ range_off,
               int64_t N, int P, SrcRange* __restrict__ ranges, Tile* __restrict__ tiles,
               ulonglong2* __restrict__ tile_cost, unsigned long long* __restrict__ evals) {
  const int lane = threadIdx.x & 31;
  const int k = blockIdx.x * kFillWarps + (threadIdx.x >> 5);
  unsigned long long cp = 0, cc = 0;
  if (k < nf) {  // warp-uniform
    const int t = fit_nodes[k];
    const int2 sg = seg[2 * t + 1];
    const int w0 = range_off[k];
    ListCursor cur;
    int ncp = 0, ncc = 0;
    for (int base = sg.x; base < sg.y; base += 32) {
      const int i = base + lane;
      int is_cp = 0, is_cc = 0;
      SrcRange r{0, 0, 0, 0};
      if (i < sg.y) {
        const int4 it = E[sorted_e[i]];
        if (it.z == 2) {
          r.begin = off[it.y];
          r.count = cnt[it.y];
          is_cp = r.count;
        } else {
          r.begin = static_cast<int>(N + static_cast<int64_t>(pslot[it.y]) * P);
          r.count = P;
          is_cc = 1;
        }
      }
      append_ranges(i < sg.y, r, ranges + w0, cur, lane);
      ncp += __reduce_add_sync(0xffffffffu, is_cp);
      ncc += __reduce_add_sync(0xffffffffu, is_cc);
    }
    if (lane == 0) {
      Tile tl;
      tl.tgt_begin = static_cast<int>(N + static_cast<int64_t>(pslot[t]) * P);
      tl.tgt_count = P;
      tl.list_begin = w0;
      tl.list_end = w0 + cur.w;
      tl.near_total = 0;  // CP / CC pairs are well separated
      tl.self_shift = tl.has_self = 0;
      tl.total = cur.src;
      tiles[k] = tl;
      cp = static_cast<unsigned long long>(P) * static_cast<unsigned long long>(ncp);
      cc = static_cast<unsigned long long>(P) * static_cast<unsigned long long>(P) * static_cast<unsigned long long>(ncc);
      tile_cost[k] = make_ulonglong2(cp, cc);
    }
  }
  typedef cub::BlockReduce<unsigned long long, 32 * kFillWarps> BR;
  __shared__ typename BR::TempStorage tmp;
  const unsigned long long scp = BR(tmp).Sum(cp);
  __syncthreads();
  const unsigned long long scc = BR(tmp).Sum(cc);
  if (threadIdx.x == 0) {
    atomicAdd(&evals[2], scp);
    atomicAdd(&evals[3], scc);
  }
}

template <class T>
void exclusive_scan(Ctx& c, const T* in, T* out, int64_t n) {
  size_t tmp = 0;
  SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, static_cast<int>(n), c.stream));
  c.cub_tmp.ensure(tmp);
  SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, tmp, in, out, static_cast<int>(n), c.stream));
  c.launches += 2;
}

}  // namespace

static TravScratch& scratch(Ctx& c) { return c.trav; }

// Guard-band control for this traversal (see MacCtl); the undecided-pair
// counter is reset here, on the stream, before the traversal kernels.
static const MacCtl* mac_ctl(Ctx& c) {
  MacGuard& g = c.mac;
  g.amb.ensure(size_t(MacGuard::kAmbCap));
  g.amb_n.ensure(1);
  g.ctl.ensure(sizeof(MacCtl));
  if (!g.d_keys.p) g.d_keys.ensure(1);
  MacCtl m;
  m.keys = g.d_keys.p;
  m.n = static_cast<int>(g.keys.size());
  m.lo = g.theta * (1.0 - g.band);
  m.hi = g.theta * (1.0 + g.band);
  m.amb = g.amb.p;
  m.amb_n = g.amb_n.p;
  m.amb_cap = MacGuard::kAmbCap;
  m.screen = std::max(1e-9, 4.0 * g.band);
  // pageable source: staged before the call returns, so m may go out of scope
  SSUM_CUDA_CHECK(cudaMemcpyAsync(g.ctl.p, &m, sizeof(m), cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(g.amb_n.p, 0, sizeof(int), c.stream));
  return reinterpret_cast<const MacCtl*>(g.ctl.p);
}

// mac_well_separated (treecode.cpp:22-25) on the host, with the reference's
// expressions and glibc's atan2: great_circle_distance (geometry.cpp:55-57),
// radius = great_circle_distance(circumcenter, v1) (face_tree.hpp:23-24).
// Node geometry (circumcentre, v1) is bit-identical to the reference's.
static bool host_mac(const double* ct, const double* v1t, const double* cs, const double* v1s, double theta) {
  auto gcd = [](const double* a, const double* b) {
    const double cx = a[1] * b[2] - a[2] * b[1], cy = a[2] * b[0] - a[0] * b[2], cz = a[0] * b[1] - a[1] * b[0];
    return std::atan2(std::sqrt(cx * cx + cy * cy + cz * cz), a[0] * b[0] + a[1] * b[1] + a[2] * b[2]);
  };
  const double r = gcd(ct, cs);
  return r > 0.0 && (gcd(ct, v1t) + gcd(cs, v1s)) / r < theta;
}

// After a traversal: decide the pairs it met inside the guard band on the
// host, add them to the table and report whether the traversal must be
// redone (a provisional decision may have differed).
// known_namb >= 0: the undecided-pair count already read back (k_bfs's own
// read-back carries it: a separate copy into pageable memory stalled the host
// ~115 us per evaluation on the staged-copy path, CUPTI timeline).
static bool resolve_mac(Ctx& c, int known_namb = -1) {
  MacGuard& g = c.mac;
  int namb = known_namb;
  if (namb < 0) {
    TravScratch& S = c.trav;
    if (!S.h_small) SSUM_CUDA_CHECK(cudaMallocHost(&S.h_small, 32 * sizeof(unsigned long long)));
    int* h = reinterpret_cast<int*>(S.h_small + 30);
    SSUM_CUDA_CHECK(cudaMemcpyAsync(h, g.amb_n.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    namb = *h;
  }
  if (namb == 0) return false;
  const int m = std::min(namb, static_cast<int>(MacGuard::kAmbCap));
  std::vector<int2> pairs(static_cast<size_t>(m));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(pairs.data(), g.amb.p, size_t(m) * sizeof(int2), cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  // node geometry: a few pairs fetch their nodes one by one, many fetch the table
  std::vector<double> all_c, all_t;
  if (m > 64) {
    const size_t nn = size_t(c.nodes.count);
    all_c.resize(3 * nn);
    all_t.resize(9 * nn);
    SSUM_CUDA_CHECK(cudaMemcpy(all_c.data(), c.nodes.center.p, all_c.size() * 8, cudaMemcpyDeviceToHost));
    SSUM_CUDA_CHECK(cudaMemcpy(all_t.data(), c.nodes.tri.p, all_t.size() * 8, cudaMemcpyDeviceToHost));
  }
  auto geom = [&](int id, double* ctr, double* v1) {
    if (!all_c.empty()) {
      std::copy(all_c.begin() + 3 * size_t(id), all_c.begin() + 3 * size_t(id) + 3, ctr);
      std::copy(all_t.begin() + 9 * size_t(id), all_t.begin() + 9 * size_t(id) + 3, v1);
      return;
    }
    SSUM_CUDA_CHECK(cudaMemcpy(ctr, c.nodes.center.p + 3 * size_t(id), 24, cudaMemcpyDeviceToHost));
    SSUM_CUDA_CHECK(cudaMemcpy(v1, c.nodes.tri.p + 9 * size_t(id), 24, cudaMemcpyDeviceToHost));
  };
  for (const int2 p : pairs) {
    double ct[3], v1t[3], cs[3], v1s[3];
    geom(p.x, ct, v1t);
    geom(p.y, cs, v1s);
    const bool well = host_mac(ct, v1t, cs, v1s, g.theta);
    g.keys.push_back((static_cast<unsigned long long>(p.x) << 33) | (static_cast<unsigned long long>(p.y) << 1) |
                     (well ? 1ull : 0ull));
  }
  std::sort(g.keys.begin(), g.keys.end());
  g.keys.erase(std::unique(g.keys.begin(), g.keys.end(),
                           [](unsigned long long a, unsigned long long b) { return (a >> 1) == (b >> 1); }),
               g.keys.end());
  g.d_keys.ensure(g.keys.size());
  SSUM_CUDA_CHECK(cudaMemcpyAsync(g.d_keys.p, g.keys.data(), g.keys.size() * 8, cudaMemcpyHostToDevice, c.stream));
  g.resolved += m;
  return true;
}

const void* mac_ctl_device(Ctx& c) { return mac_ctl(c); }

namespace {
__global__ void k_node_records(int nn, const double* __restrict__ center, const double* __restrict__ radius,
                               const int* __restrict__ cnt, const int* __restrict__ off, const int* __restrict__ level,
                               const int* __restrict__ child_base, double half_inv_theta, NodeRec* __restrict__ rec) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  NodeRec r;
  r.cx = center[3 * i];
  r.cy = center[3 * i + 1];
  r.cz = center[3 * i + 2];
  r.r = radius[i];
  sincos(r.r * half_inv_theta, &r.sh, &r.ch);
  r.cnt = cnt[i];
  r.off = off[i];
  r.level = level[i];
  r.child_base = child_base[i];
  rec[i] = r;
}
}  // namespace

void build_node_records(Ctx& c, double theta) {
  const int nn = c.nodes.count;
  c.trav.rec.ensure(size_t(std::max(nn, 1)));
  k_node_records<<<grid_for(nn, 256), 256, 0, c.stream>>>(nn, c.nodes.center.p, c.nodes.radius.p, c.bins.cnt.p,
                                                          c.bins.off.p, c.nodes.level.p, c.nodes.child_base.p,
                                                          0.5 / theta, c.trav.rec.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
}
bool resolve_mac_host(Ctx& c) { return resolve_mac(c); }

// Breadth-first traversal with one host read per step (the frontier size
// sizes the next step). Records the step sizes as the plan for the next call.
static long long bfs_synchronous(Ctx& c, const ssum_config& cfg) {
  Lists& L = c.lists;
  Binned& B = c.bins;
  TravScratch& S = c.trav;
  const int bs = 256;
  S.F0.ensure(400);
  k_root_pairs<<<2, 256, 0, c.stream>>>(S.F0.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  const int rlo = c.restrict_on ? static_cast<int>(c.rp0) : 0;
  const int rhi = c.restrict_on ? static_cast<int>(c.rp1) : 0x7fffffff;
  int m = 400;
  long long ne = 0;
  L.inter.ensure(1 << 16);
  L.key.ensure(1 << 16);
  S.plan_m.clear();
  const MacCtl* mac = mac_ctl(c);
  while (m > 0) {
    S.plan_m.push_back(m);
    S.action.ensure(size_t(m) + 1);
    S.packed.ensure(size_t(m) + 1);
    S.scan.ensure(size_t(m) + 1);
    k_trav_eval<<<grid_for(m + 1, bs), bs, 0, c.stream>>>(S.F0.p, m, B.cnt.p, B.off.p, rlo, rhi, c.nodes.center.p,
                                                           c.nodes.radius.p,
                                                           c.nodes.level.p, c.nodes.child_base.p, cfg.theta,
                                                           cfg.n_threshold, cfg.max_depth, cfg.pc_only, mac,
                                                           S.action.p, S.packed.p, S.rec.p, kPi * cfg.theta * (1.0 - 1e-12));
    SSUM_LAUNCH_CHECK();
    c.launches++;
    exclusive_scan(c, S.packed.p, S.scan.p, m + 1);  // packed[m] = 0: totals at scan[m]
    SSUM_CUDA_CHECK(cudaMemcpyAsync(S.h_small, S.scan.p + m, 8, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    const unsigned long long tot = S.h_small[0];
    const int next = static_cast<int>(tot & 0xffffffffull);
    const long long emitted = static_cast<long long>(tot >> 32);
    L.inter.ensure(size_t(ne + emitted), true, c.stream);
    L.key.ensure(size_t(ne + emitted), true, c.stream);
    S.F1.ensure(size_t(std::max(next, 1)));
    k_trav_scatter<<<grid_for(m, bs), bs, 0, c.stream>>>(S.F0.p, m, S.action.p, S.scan.p, c.nodes.child_base.p,
                                                          S.F1.p, L.inter.p, L.key.p, ne, c.d_flags.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    ne += emitted;
    std::swap(S.F0, S.F1);
    m = next;
  }
  S.plan_ne = ne;
  S.plan_valid = true;
  return ne;
}

// The traversal as one cooperative kernel (k_bfs), sized from the previous
// call's largest frontier and emission count (plus slack); one read-back at
// the end. False (nothing committed) when there is no previous call, the
// launch is refused, or a step outgrew the capacities: the caller then runs
// the step-by-step traversal, which also refreshes the sizes.
template <class AfterLaunch>
static bool bfs_persistent(Ctx& c, const ssum_config& cfg, long long& ne_out, AfterLaunch&& after_launch) {
  Lists& L = c.lists;
  Binned& B = c.bins;
  TravScratch& S = c.trav;
  if (S.bfs_blocks == 0) {
    int per_sm = 0, sms = 0;
    SSUM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bfs, kBfsThreads, 0));
    SSUM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
#ifndef SSUM_BFS_PER_SM
#define SSUM_BFS_PER_SM 4
#endif
    int want = SSUM_BFS_PER_SM;
    if (const char* v = std::getenv("SSUM_BFS_PER_SM_RT")) want = std::max(1, std::atoi(v));
    S.bfs_blocks = sms * std::min(per_sm, want);
    if (S.bfs_blocks <= 0) S.bfs_blocks = -1;
  }
  if (S.bfs_blocks < 0) return false;
  const int nb = S.bfs_blocks;
  int fcap;
  long long ecap;
  if (S.plan_valid && !S.plan_m.empty()) {  // sized from the previous call
    const int fplan = *std::max_element(S.plan_m.begin(), S.plan_m.end());
    fcap = fplan + fplan / 8 + 1024;
    ecap = S.plan_ne + S.plan_ne / 8 + 4096;
  } else {  // first call: generous estimates from N (configs 1-5 emit 1.6-2.0 N pairs)
    const int64_t N = B.n;
    fcap = static_cast<int>(std::min<int64_t>(2 * N + 65536, 0x3fffffff));
    ecap = 3 * N + 65536;
  }
  S.F0.ensure(size_t(fcap));
  S.F1.ensure(size_t(fcap));
  S.action.ensure(size_t(fcap));
  S.packed.ensure(size_t(fcap));
  S.scan.ensure(size_t(nb));
  S.dm.ensure(4);
  S.debase.ensure(1);
  L.inter.ensure(size_t(ecap));
  L.key.ensure(size_t(ecap));
  if (!S.h_plan) SSUM_CUDA_CHECK(cudaMallocHost(&S.h_plan, 256 * sizeof(long long)));
  k_root_pairs<<<2, 256, 0, c.stream>>>(S.F0.p);
  SSUM_LAUNCH_CHECK();
  const int* cnt = B.cnt.p;
  const int* off = B.off.p;
  int rlo = c.restrict_on ? static_cast<int>(c.rp0) : 0;
  int rhi = c.restrict_on ? static_cast<int>(c.rp1) : 0x7fffffff;
  const double *center = c.nodes.center.p, *radius = c.nodes.radius.p;
  const int *level = c.nodes.level.p, *child_base = c.nodes.child_base.p;
  double theta = cfg.theta;
  int thr = cfg.n_threshold, max_depth = cfg.max_depth, pc_only = cfg.pc_only;
  const MacCtl* mac = mac_ctl(c);
  PairEntry *f0 = S.F0.p, *f1 = S.F1.p;
  int4* e = L.inter.p;
  unsigned long long* k = L.key.p;
  int* action = S.action.p;
  unsigned long long *loc = S.packed.p, *btot = S.scan.p;
  int* out = S.dm.p;
  long long* ne = S.debase.p;
  int* flags = c.d_flags.p;
  const NodeRec* rec = S.rec.p;
  double pi_theta = kPi * cfg.theta * (1.0 - 1e-12);
  void* args[] = {&cnt, &off, &rlo, &rhi, &center, &radius, &level, &child_base, &theta, &thr, &max_depth,
                  &pc_only, &mac, &f0, &f1,
                  &fcap, &e, &k, &ecap, &action, &loc, &btot, &out, &ne, &flags, &rec, &pi_theta};
  if (cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_bfs), dim3(nb), dim3(kBfsThreads), args, 0, c.stream) !=
      cudaSuccess) {
    (void)cudaGetLastError();
    S.bfs_blocks = -1;  // no cooperative launch here: step by step from now on
    return false;
  }
  c.launches += 2;
  after_launch();  // host work that need not precede the traversal (the prep stream's launches)
  int* h = reinterpret_cast<int*>(S.h_plan);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h, S.dm.p, 3 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(S.h_plan + 128, S.debase.p, sizeof(long long), cudaMemcpyDeviceToHost, c.stream));
  int* h_amb = reinterpret_cast<int*>(S.h_plan + 129);  // the MAC guard band's undecided pairs, same read-back
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h_amb, c.mac.amb_n.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  S.bfs_namb = *h_amb;
  if (h[1] != 0) return false;
  S.plan_m.assign(1, h[2]);
  S.plan_ne = S.h_plan[128];
  ne_out = S.plan_ne;
  return true;
}

void traverse_and_build_lists(Ctx& c, const ssum_config& cfg, bool keep_order_keys) {
  (void)keep_order_keys;
  Lists& L = c.lists;
  Binned& B = c.bins;
  TravScratch& S = scratch(c);
  const int64_t N = B.n;
  L.n_inter = 0;
  for (int k = 0; k < 4; ++k) L.counts[k] = L.evals[k] = 0;
  L.n_proxy = L.n_weight = L.n_fit = L.n_leaf_tiles = L.n_fit_tiles = 0;
  L.n_leaf_ranges = L.n_fit_ranges = 0;
  if (N == 0) return;

  // ---- breadth-first traversal
  long long ne = 0;
  if (!S.h_small) SSUM_CUDA_CHECK(cudaMallocHost(&S.h_small, 32 * sizeof(unsigned long long)));
  MacGuard& g = c.mac;
  if (g.theta != cfg.theta) {  // host decisions are per theta (node ids persist with the geometry)
    g.keys.clear();
    g.theta = cfg.theta;
  }
  build_node_records(c, cfg.theta);
  c.up_list = nullptr;  // the upward pass covers every weight node
  c.up_count = nullptr;
  // planned lists (the binning's subtree plan gave every big node a proxy
  // slot): the upward pass needs nothing from the traversal, so it starts
  // now and runs beside it; fit tiles are indexed by slot
  c.plan_lists = !keep_order_keys && c.sub.valid && c.sub.thr == cfg.n_threshold && c.sub.n_big > 0 &&
                 c.plan_lists_ok;
  // The prep stream forks here but its launches are queued behind k_bfs's:
  // nothing else starts while the cooperative kernel is resident anyway, and
  // queuing the prep's ~8 launches first kept the traversal waiting ~60 us
  // on the host (CUPTI timeline). SSUM_PREP_FIRST=1: the earlier order.
  static const bool prep_first = [] {
    const char* e = std::getenv("SSUM_PREP_FIRST");
    return e && *e == '1';
  }();
  bool prep_pending = false;
  if (c.plan_lists) {
    L.n_proxy = L.n_weight = c.sub.n_big;
    if (prep_first || !c.early.xyz || !c.early_prep) {
      start_prep(c);
    } else {
      size_eval_buffers(c, c.early.degree, c.early.dim, N);
      SSUM_CUDA_CHECK(cudaEventRecord(c.fork_ev, c.stream));
      prep_pending = true;
    }
  }
  auto prep_now = [&] {
    if (prep_pending) {
      prep_pending = false;
      start_prep(c, true);
    }
  };
  for (int round = 0;; ++round) {
    static const bool stepwise = [] {  // SSUM_BFS_STEPWISE=1: step by step, frontier sizes traced
      const char* e = std::getenv("SSUM_BFS_STEPWISE");
      return e && *e == '1';
    }();
    S.bfs_namb = -1;
    if (stepwise) prep_now();
    if (stepwise || !bfs_persistent(c, cfg, ne, prep_now)) {
      prep_now();
      ne = bfs_synchronous(c, cfg);
      S.bfs_namb = -1;  // the step-by-step traversal may have met other pairs
    }
    if (stepwise && trace().on) {
      std::fprintf(stderr, "[ssum bfs] %zu steps, frontier:", S.plan_m.size());
      for (const int m : S.plan_m) std::fprintf(stderr, " %d", m);
      std::fprintf(stderr, " emissions %lld\n", ne);
    }
    if (!resolve_mac(c, S.bfs_namb)) break;
    if (round > 64) throw Error(SSUM_INTERNAL, "dual traversal: MAC guard band did not settle");
  }
  L.n_inter = ne;
  trace().mark("trav.bfs");
  build_lists(c, cfg);
}

// From the emitted interactions (L.inter[0, L.n_inter)) to the evaluation
// layout: node flags, proxy slots, leaf tiles, fit tiles, target partition.
void build_lists(Ctx& c, const ssum_config& cfg) {
  Lists& L = c.lists;
  Binned& B = c.bins;
  TravScratch& S = scratch(c);
  const int nn = c.nodes.count;
  const int64_t N = B.n;
  const int P = (cfg.degree + 1) * (cfg.degree + 2) / 2;
  const int bs = 256;
  const long long ne = L.n_inter;
  for (int k = 0; k < 4; ++k) L.counts[k] = L.evals[k] = 0;
  L.n_proxy = L.n_weight = L.n_fit = L.n_leaf_tiles = L.n_fit_tiles = 0;
  L.n_leaf_ranges = L.n_fit_ranges = 0;
  if (N == 0) return;

  // ---- node flags, kind counts, grouping by (target, class)
  L.is_weight.ensure(size_t(nn));
  L.is_fit.ensure(size_t(nn));
  L.pslot.ensure(size_t(nn));
  SSUM_CUDA_CHECK(cudaMemsetAsync(L.is_weight.p, 0, size_t(nn), c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(L.is_fit.p, 0, size_t(nn), c.stream));
  S.counters.ensure(16);
  // [0..3] kinds, [4..7] kernel evals, [8] node-list selection counts, [10..11] pass visits
  SSUM_CUDA_CHECK(cudaMemsetAsync(S.counters.p, 0, 12 * sizeof(unsigned long long), c.stream));
  const size_t nes = size_t(std::max<long long>(ne, 1));
  S.gkey.ensure(nes);
  S.gkey2.ensure(nes);
  S.gval.ensure(nes);
  S.sorted_e.ensure(nes);
  if (ne > 0) {
    k_mark<<<grid_for(ne, bs), bs, 0, c.stream>>>(L.inter.p, ne, L.is_weight.p, L.is_fit.p, S.gkey.p, S.gval.p,
                                                   S.counters.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < 2 * int64_t(nn)) ++end_bit;
    size_t tmp = 0;
    SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, S.gkey.p, S.gkey2.p, S.gval.p, S.sorted_e.p,
                                                    static_cast<int>(ne), 0, end_bit, c.stream));
    c.cub_tmp.ensure(tmp);
    SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, tmp, S.gkey.p, S.gkey2.p, S.gval.p, S.sorted_e.p,
                                                    static_cast<int>(ne), 0, end_bit, c.stream));
    c.launches += 4;
  }
  S.seg.ensure(size_t(2) * nn);
  SSUM_CUDA_CHECK(cudaMemsetAsync(S.seg.p, 0, size_t(2) * nn * sizeof(int2), c.stream));
  if (ne > 0) {
    k_seg_bounds<<<grid_for(ne, bs), bs, 0, c.stream>>>(S.gkey2.p, ne, S.seg.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }

  const bool planned = c.plan_lists;
  if (planned) {
    // slots, weight nodes (every big node) from the plan; fit tiles for every
    // big node, indexed by slot (a node without CP/CC pairs gets an empty tile)
    L.n_proxy = L.n_weight = L.n_fit = c.sub.n_big;
    L.fit_nodes.ensure(size_t(std::max(c.sub.n_big, 1)));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(L.fit_nodes.p, L.weight_nodes.p, size_t(c.sub.n_big) * 4, cudaMemcpyDeviceToDevice,
                                    c.stream));
  } else {
  // ---- proxy slots (weight or fit nodes), slot-ordered node lists
  S.flag.ensure(size_t(nn));
  S.flag_scan.ensure(size_t(nn));
  S.slot_node.ensure(size_t(nn));
  k_slot_flags<<<grid_for(nn, bs), bs, 0, c.stream>>>(L.is_weight.p, L.is_fit.p, nn, S.flag.p);
  SSUM_LAUNCH_CHECK();
  exclusive_scan(c, S.flag.p, S.flag_scan.p, nn);
  k_slots<<<grid_for(nn, bs), bs, 0, c.stream>>>(S.flag.p, S.flag_scan.p, nn, L.is_weight.p, L.is_fit.p, L.pslot.p,
                                                  S.slot_node.p);
  SSUM_LAUNCH_CHECK();
  c.launches += 2;
  // weight / fit node lists in slot order (= node-id order): device compaction
  L.weight_nodes.ensure(size_t(nn));
  L.fit_nodes.ensure(size_t(nn));
  {
    int* nsel = reinterpret_cast<int*>(S.counters.p + 8);  // [0] weight nodes, [1] fit nodes
    cub::CountingInputIterator<int> ids(0);
    size_t t1 = 0, t2 = 0;
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, t1, ids, L.is_weight.p, L.weight_nodes.p,
                                               nsel, nn, c.stream));
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, t2, ids, L.is_fit.p, L.fit_nodes.p,
                                               nsel + 1, nn, c.stream));
    c.cub_tmp.ensure(std::max(t1, t2));
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(c.cub_tmp.p, t1, ids, L.is_weight.p, L.weight_nodes.p,
                                               nsel, nn, c.stream));
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(c.cub_tmp.p, t2, ids, L.is_fit.p, L.fit_nodes.p,
                                               nsel + 1, nn, c.stream));
    c.launches += 4;
    int tail[4];
    SSUM_CUDA_CHECK(cudaMemcpyAsync(&tail[0], S.flag_scan.p + (nn - 1), 4, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(&tail[1], S.flag.p + (nn - 1), 4, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(&tail[2], nsel, 8, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    L.n_proxy = tail[0] + tail[1];
    L.n_weight = tail[2];
    L.n_fit = tail[3];
  }
  start_prep(c);  // gather + proxies + upward on the prep stream, overlapping the rest
  }

  trace().mark("lists.group_slots");
  // ---- range and tile counts for leaves and fit nodes, one read-back
  // leaves to build tiles for: all of them, or this part's (restricted call)
  const int* leaves = B.d_leaves.p + (c.restrict_on ? c.rl0 : 0);
  const int nl = c.restrict_on ? c.rl1 - c.rl0 : B.n_leaves;
  const int nf = L.n_fit;
  S.nr.ensure(size_t(nl) + 1);
  S.nt.ensure(size_t(nl) + 1);
  S.nr_off.ensure(size_t(nl) + 1);
  S.nt_off.ensure(size_t(nl) + 1);
  S.fnr.ensure(size_t(nf) + 1);
  S.fnr_off.ensure(size_t(nf) + 1);
  SSUM_CUDA_CHECK(cudaMemsetAsync(S.nr.p + nl, 0, 4, c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(S.nt.p + nl, 0, 4, c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(S.fnr.p + nf, 0, 4, c.stream));
  k_leaf_count<<<grid_for(std::max(nl, 1), 128), 128, 0, c.stream>>>(leaves, nl, c.nodes.parent.p, S.seg.p, B.cnt.p,
                                                                      S.nr.p, S.nt.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  exclusive_scan(c, S.nr.p, S.nr_off.p, nl + 1);
  exclusive_scan(c, S.nt.p, S.nt_off.p, nl + 1);
  if (nf > 0) {
    k_fit_count<<<grid_for(nf, 128), 128, 0, c.stream>>>(L.fit_nodes.p, nf, S.seg.p, S.fnr.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    exclusive_scan(c, S.fnr.p, S.fnr_off.p, nf + 1);
  }
  if (!S.h_small) SSUM_CUDA_CHECK(cudaMallocHost(&S.h_small, 32 * sizeof(unsigned long long)));
  {
    int* tot = reinterpret_cast<int*>(S.h_small);
    SSUM_CUDA_CHECK(cudaMemcpyAsync(&tot[0], S.nr_off.p + nl, 4, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(&tot[1], S.nt_off.p + nl, 4, cudaMemcpyDeviceToHost, c.stream));
    tot[2] = 0;
    if (nf > 0) SSUM_CUDA_CHECK(cudaMemcpyAsync(&tot[2], S.fnr_off.p + nf, 4, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    L.n_leaf_ranges = tot[0];
    L.n_leaf_tiles = tot[1];
    L.n_fit_ranges = tot[2];
  }
  L.leaf_ranges.ensure(size_t(std::max<int64_t>(L.n_leaf_ranges, 1)));
  L.leaf_tiles.ensure(size_t(std::max(L.n_leaf_tiles, 1)));
  L.leaf_cost.ensure(size_t(std::max(L.n_leaf_tiles, 1)));
  k_leaf_fill<<<grid_for(std::max(nl, 1), kFillWarps), 32 * kFillWarps, 0, c.stream>>>(leaves, nl, c.nodes.parent.p, S.seg.p, S.sorted_e.p,
                                                        L.inter.p, B.cnt.p, B.off.p, L.pslot.p, c.nodes.center.p,
                                                        c.nodes.radius.p, S.nr_off.p, S.nt_off.p, N, P,
                                                        L.leaf_ranges.p, L.leaf_tiles.p, L.leaf_cost.p,
                                                        S.counters.p + 4, S.rec.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;

  // ---- fit tiles
  if (nf > 0) {
    L.fit_ranges.ensure(size_t(std::max<int64_t>(L.n_fit_ranges, 1)));
    L.fit_tiles.ensure(size_t(nf));
    L.fit_cost.ensure(size_t(nf));
    k_fit_fill<<<grid_for(nf, kFillWarps), 32 * kFillWarps, 0, c.stream>>>(L.fit_nodes.p, nf, S.seg.p, S.sorted_e.p, L.inter.p, B.cnt.p,
                                                         B.off.p, L.pslot.p, S.fnr_off.p, N, P, L.fit_ranges.p,
                                                         L.fit_tiles.p, L.fit_cost.p, S.counters.p + 4);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  L.n_fit_tiles = nf;
  // (particle, weight node) and (particle, fit node) visits of the upward /
  // downward passes
  if (L.n_weight + nf > 0) {
    k_visits<<<grid_for(L.n_weight + nf, 256), 256, 0, c.stream>>>(L.weight_nodes.p, L.n_weight, L.fit_nodes.p, nf,
                                                                  B.cnt.p, S.counters.p + 10,
                                                                  planned ? L.is_fit.p : nullptr);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  // interaction / evaluation / visit counts: read back with the evaluation's final sync
  SSUM_CUDA_CHECK(cudaMemcpyAsync(S.h_small + 8, S.counters.p, 12 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                                  c.stream));
  L.counts_pending = true;
  trace().mark("lists.tiles");
  partition_targets(c);
}

// L.counts / L.evals from the pinned read-back queued by build_lists (valid
// once the stream has been synchronised).
void finalize_counts(Ctx& c) {
  Lists& L = c.lists;
  if (!L.counts_pending) return;
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  const unsigned long long* h = c.trav.h_small + 8;
  for (int k = 0; k < 4; ++k) {
    L.counts[k] = h[k];
    L.evals[k] = h[4 + k];
  }
  L.visits[0] = h[10];
  L.visits[1] = h[11];
  if (c.plan_lists) L.n_fit = static_cast<int>(h[8]);  // fit nodes among the big nodes (k_visits)
  if (L.local_is_all)
    for (int k = 0; k < 4; ++k) L.local_evals[k] = L.evals[k];
  L.counts_pending = false;
}

// First leaf (depth-first index) starting at or after tree position x, for
// every cut position x = pos[r] (r = 0 .. m-1): out[r] its tree position,
// out[m + r] its leaf index.
__global__ void k_snap_cuts(const int* __restrict__ leaves, int nl, const int* __restrict__ off, long long n,
                            const long long* __restrict__ pos, int m, long long* out,
                            const int* __restrict__ tile_off, long long* tout) {
  const int r = threadIdx.x;
  if (r >= m) return;
  const long long x = pos[r];
  int lo = 0, hi = nl;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (off[leaves[mid]] < x)
      lo = mid + 1;
    else
      hi = mid;
  }
  out[r] = lo < nl ? off[leaves[lo]] : n;
  out[m + r] = lo;
  if (tile_off) tout[r] = tile_off[lo];  // subtree plan: the leaf's first tile
}

// Restricted multi-part call: once a full multi-part call has placed the
// cost-balanced cuts (partition_targets), later calls with the same N and
// part count snap those positions to leaf starts of the current binning and
// traverse / build lists for this part's targets only. The lists of a target
// are the same pairs in the same order as in the full traversal (dropping
// pairs keeps the relative emission order), so the union of the parts stays
// bitwise the single-part result. Every part's snapped range is kept
// (Ctx::part_pos): all ranks bin identically, so all agree on it.
bool plan_restriction(Ctx& c) {
  c.restrict_on = false;
  const Binned& B = c.bins;
  c.part_pos.assign({0, B.n});
  if (c.nparts <= 1 || c.cuts.n != B.n || c.cuts.nparts != c.nparts || B.n_leaves == 0) return false;
  const int m = c.nparts + 1;
  c.snap.ensure(size_t(4 * m));
  std::vector<long long> h(size_t(3 * m));
  for (int r = 0; r < m; ++r) h[size_t(r)] = c.cuts.pos[size_t(r)];
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.snap.p + 2 * m, h.data(), size_t(m) * 8, cudaMemcpyHostToDevice, c.stream));
  const int* tile_off = c.sub.valid ? c.sub.tile_off.p : nullptr;
  k_snap_cuts<<<1, ((m + 31) / 32) * 32, 0, c.stream>>>(B.d_leaves.p, B.n_leaves, B.off.p, B.n, c.snap.p + 2 * m, m,
                                                        c.snap.p, tile_off, c.snap.p + 3 * m);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h.data(), c.snap.p, size_t(2 * m) * 8, cudaMemcpyDeviceToHost, c.stream));
  if (tile_off)
    SSUM_CUDA_CHECK(cudaMemcpyAsync(h.data() + 2 * m, c.snap.p + 3 * m, size_t(m) * 8, cudaMemcpyDeviceToHost,
                                    c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  c.part_pos.assign(h.begin(), h.begin() + m);
  c.part_pos.front() = 0;
  c.rp0 = h[size_t(c.part)];
  c.rp1 = h[size_t(c.part) + 1];
  c.rl0 = static_cast<int>(h[size_t(m + c.part)]);
  c.rl1 = static_cast<int>(h[size_t(m + c.part) + 1]);
  if (tile_off) {
    c.rt0 = static_cast<int>(h[size_t(2 * m + c.part)]);
    c.rt1 = static_cast<int>(h[size_t(2 * m + c.part) + 1]);
  }
  c.restrict_on = true;
  return true;
}

// Multi-GPU target partition: leaf tiles are in depth-first
// order, so a contiguous tile range is a contiguous range [p0, p1) of tree
// positions. Cut points balance the tiles' PP + PC pair counts; a part keeps
// the fit nodes whose bins intersect its range (nodes straddling a cut are
// computed by both owners, identically). Each target is computed whole by
// one part with the same code, so the union of the parts is bitwise the
// single-part result. The tree build and upward pass are replicated.
void partition_targets(Ctx& c) {
  Lists& L = c.lists;
  const int64_t N = c.bins.n;
  L.leaf_t0 = 0;
  L.leaf_t1 = L.n_leaf_tiles;
  L.p0 = 0;
  L.p1 = N;
  L.n_fit_sel = L.n_fit_tiles;
  L.fit_sel_all = true;
  L.local_evals[0] = L.evals[0];
  L.local_evals[1] = L.evals[1];
  L.local_evals[2] = L.evals[2];
  L.local_evals[3] = L.evals[3];
  L.local_is_all = true;
  if (c.nparts <= 1) return;
  if (c.restrict_on) {  // the lists hold exactly this part's targets
    L.p0 = c.rp0;
    L.p1 = c.rp1;
    return;
  }
  L.local_is_all = false;
  if (L.n_leaf_tiles == 0) return;
  const int nt = L.n_leaf_tiles;
  std::vector<ulonglong2> cost(static_cast<size_t>(nt));
  std::vector<Tile> tiles(static_cast<size_t>(nt));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(cost.data(), L.leaf_cost.p, size_t(nt) * sizeof(ulonglong2), cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(tiles.data(), L.leaf_tiles.p, size_t(nt) * sizeof(Tile), cudaMemcpyDeviceToHost, c.stream));
  std::vector<ulonglong2> fcost(static_cast<size_t>(std::max(L.n_fit_tiles, 0)));
  if (L.n_fit_tiles > 0)
    SSUM_CUDA_CHECK(cudaMemcpyAsync(fcost.data(), L.fit_cost.p, fcost.size() * sizeof(ulonglong2), cudaMemcpyDeviceToHost, c.stream));
  std::vector<int> fit_nodes(static_cast<size_t>(L.n_fit_tiles));
  if (L.n_fit_tiles > 0)
    SSUM_CUDA_CHECK(cudaMemcpyAsync(fit_nodes.data(), L.fit_nodes.p, fit_nodes.size() * 4, cudaMemcpyDeviceToHost,
                                    c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  // Cost per tile, in pair evaluations (13 flop): its own PP + PC pairs, plus
  // a per-target share of every fit ancestor's work — the
  // node's CP + CC pairs and its 2 D P^2 fit epilogue spread evenly over its
  // bin, and the downward evaluation of its interpolant at each target
  // (~402 flop at d = 8, §8(d)) — through a difference array over tree
  // positions.
  const HostTree& ht = host_tree(c);
  const int D = c.early.dim > 0 ? c.early.dim : 3;
  const int deg = c.early.degree > 0 ? c.early.degree : 8;
  const int P = (deg + 1) * (deg + 2) / 2;
  const double down_pairs = (21.0 + 3.0 * (deg - 1) + (2.0 + 2.0 * D) * P) / 13.0;
  std::vector<double> dens(size_t(N) + 1, 0.0);
  for (int k = 0; k < L.n_fit_tiles; ++k) {
    const int id = fit_nodes[size_t(k)];
    const int64_t o = ht.off[size_t(id)], cn = ht.cnt[size_t(id)];
    if (cn <= 0) continue;
    const double node = double(fcost[size_t(k)].x + fcost[size_t(k)].y) + 2.0 * D * P * P / 13.0;
    const double per = node / double(cn) + down_pairs;
    dens[size_t(o)] += per;
    dens[size_t(o + cn)] -= per;
  }
  std::vector<double> pre(static_cast<size_t>(nt) + 1, 0.0);
  {
    double run = 0.0;  // density at position `at`
    int64_t at = 0;
    for (int t = 0; t < nt; ++t) {
      const int64_t b = tiles[size_t(t)].tgt_begin, e = b + tiles[size_t(t)].tgt_count;
      double share = 0.0;
      for (; at < e; ++at) {
        run += dens[size_t(at)];
        if (at >= b) share += run;
      }
      pre[size_t(t) + 1] = pre[size_t(t)] + double(cost[size_t(t)].x + cost[size_t(t)].y) + share + 1.0;
    }
  }
  const double total = pre[size_t(nt)];
  // cut before the first tile at or after the cost goal that starts a leaf
  // (a leaf's tiles share list_begin): parts never split a leaf, so the
  // positions are leaf starts, as restricted calls' snapped cuts are
  auto cut = [&](int r) {
    if (r <= 0) return 0;
    if (r >= c.nparts) return nt;
    const double goal = total * r / c.nparts;
    int t = static_cast<int>(std::lower_bound(pre.begin(), pre.end(), goal) - pre.begin());
    while (t > 0 && t < nt && tiles[size_t(t)].list_begin == tiles[size_t(t) - 1].list_begin) ++t;
    return std::min(t, nt);
  };
  const int t0 = std::min(cut(c.part), nt), t1 = std::max(std::min(cut(c.part + 1), nt), t0);
  L.leaf_t0 = t0;
  L.leaf_t1 = t1;
  L.local_evals[0] = L.local_evals[1] = L.local_evals[2] = L.local_evals[3] = 0;
  if (t1 > t0) {
    L.p0 = tiles[size_t(t0)].tgt_begin;
    L.p1 = tiles[size_t(t1) - 1].tgt_begin + tiles[size_t(t1) - 1].tgt_count;
  } else {
    L.p0 = L.p1 = (t0 < nt) ? tiles[size_t(t0)].tgt_begin : N;
  }
  for (int t = t0; t < t1; ++t) {
    L.local_evals[0] += cost[size_t(t)].x;
    L.local_evals[1] += cost[size_t(t)].y;
  }
  // the cut positions of every part, for the next (restricted) calls
  c.cuts.n = N;
  c.cuts.nparts = c.nparts;
  c.cuts.pos.assign(size_t(c.nparts) + 1, N);
  for (int r = 0; r <= c.nparts; ++r) {
    const int ct = std::min(cut(r), nt);
    c.cuts.pos[size_t(r)] = ct < nt ? tiles[size_t(ct)].tgt_begin : N;
  }
  c.cuts.pos.front() = 0;
  c.part_pos = c.cuts.pos;
  std::vector<int> sel;
  for (int k = 0; k < L.n_fit_tiles; ++k) {
    const int id = fit_nodes[size_t(k)];
    const int64_t o = ht.off[size_t(id)], e = o + ht.cnt[size_t(id)];
    if (o < L.p1 && e > L.p0) {
      sel.push_back(k);
      L.local_evals[2] += fcost[size_t(k)].x;
      L.local_evals[3] += fcost[size_t(k)].y;
    }
  }
  L.n_fit_sel = static_cast<int>(sel.size());
  L.fit_sel_all = false;
  L.fit_sel.ensure(std::max<size_t>(sel.size(), 1));
  if (!sel.empty())
    SSUM_CUDA_CHECK(cudaMemcpyAsync(L.fit_sel.p, sel.data(), sel.size() * 4, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// Export helper: the emitted list sorted into depth-first (reference) order.
void sorted_interactions(Ctx& c, std::vector<int4>& out) {
  Lists& L = c.lists;
  TravScratch& S = scratch(c);
  out.clear();
  const long long ne = L.n_inter;
  if (ne == 0) return;
  int fl = 0;
  SSUM_CUDA_CHECK(cudaMemcpyAsync(&fl, c.d_flags.p, 4, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  if (fl & 4) throw Error(SSUM_INTERNAL, "dual_traversal export: refinement depth exceeds the order-key width");
  DBuf<unsigned long long> k2;
  DBuf<int> v2;
  k2.ensure(size_t(ne));
  v2.ensure(size_t(ne));
  // values: emission index
  std::vector<int> idx(static_cast<size_t>(ne));
  for (long long e = 0; e < ne; ++e) idx[size_t(e)] = static_cast<int>(e);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(S.gval.p, idx.data(), size_t(ne) * 4, cudaMemcpyHostToDevice, c.stream));
  size_t tmp = 0;
  SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, L.key.p, k2.p, S.gval.p, v2.p, static_cast<int>(ne), 0,
                                                  64, c.stream));
  c.cub_tmp.ensure(tmp);
  SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, tmp, L.key.p, k2.p, S.gval.p, v2.p, static_cast<int>(ne),
                                                  0, 64, c.stream));
  std::vector<int4> E(static_cast<size_t>(ne));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(E.data(), L.inter.p, size_t(ne) * sizeof(int4), cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(idx.data(), v2.p, size_t(ne) * 4, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  k2.release();
  v2.release();
  out.resize(size_t(ne));
  for (long long e = 0; e < ne; ++e) out[size_t(e)] = E[size_t(idx[size_t(e)])];
}

}  // namespace ssum
