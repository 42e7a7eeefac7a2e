// Device helpers shared by the two list builders (traversal.cu: the
// breadth-first traversal + grouping; sublists.cu: the per-subtree build):
// the reference's pair decisions (treecode.cpp:22-65) with the exact-MAC
// guard band, the near-pair screen and the warp-cooperative range append.
#pragma once

#include "internal.cuh"

namespace ssum {
namespace {

constexpr int kKeyStepBits = 2;
constexpr int kKeyMaxSteps = 27;  // 9 bits root pair + 2 bits x 27 steps = 63 bits

// classify (treecode.cpp:29-36); pc_only remaps CP -> PP and CC -> PC.
__device__ __forceinline__ int classify_kind(int nt_, int ns_, int thr, int pc_only) {
  const bool tb = nt_ > thr, sb = ns_ > thr;
  int k = 0;
  if (tb && sb) k = 3;
  else if (sb) k = 1;
  else if (tb) k = 2;
  if (pc_only) {
    if (k == 2) k = 0;
    if (k == 3) k = 1;
  }
  return k;
}

// MAC decisions exact by construction. R and the radii come from CUDA's
// atan2 (<= 2 ulp) where the reference uses glibc's (< 1 ulp), so the
// quotient (r_t + r_s)/R may differ from the reference's by a few ulp
// (<= ~1e-15 relative). A decision can therefore differ only when the quotient
// lies that close to theta. Every pair whose device quotient falls in the
// guard band theta (1 +- band) (band = 1e-12 by default, ~5000 ulp) is looked
// up in a table of host-made decisions; a pair missing from it is recorded,
// takes the device decision provisionally, and the traversal is redone once
// the host (glibc atan2, the reference's expressions: great_circle_distance,
// triangle_radius, mac_well_separated, treecode.cpp:22-25) has decided it
// (resolve_mac below). Outside the band the device decision is the
// reference's; inside it the host's is.
struct MacCtl {
  const unsigned long long* keys;  // sorted (t << 33 | s << 1 | well)
  int n;
  double lo, hi;                   // theta (1 - band), theta (1 + band)
  int2* amb;                       // undecided pairs (first amb_cap)
  int* amb_n;
  int amb_cap;
  double screen;  // relative margin of the chord screen (pair_decide): max(1e-9, 4 band)
};

__device__ __noinline__ bool mac_lookup(const MacCtl& m, int t, int s, bool provisional) {
  const unsigned long long k = (static_cast<unsigned long long>(t) << 33) | (static_cast<unsigned long long>(s) << 1);
  int lo = 0, hi = m.n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if ((m.keys[mid] | 1ull) < k) lo = mid + 1;
    else hi = mid;
  }
  if (lo < m.n && (m.keys[lo] >> 1) == (k >> 1)) return (m.keys[lo] & 1ull) != 0;
  const int i = atomicAdd(m.amb_n, 1);
  if (i < m.amb_cap) m.amb[i] = make_int2(t, s);
  return provisional;
}

// Exact device MAC decision (the reference's expression with the guard
// band): (r_t + r_s) / R < theta with R = great_circle_distance > 0.
__device__ __noinline__ bool mac_exact(int t, int s, double tx, double ty, double tz, double tr, double sx, double sy,
                                       double sz, double sr, double theta, const MacCtl* __restrict__ mac) {
  const d3 a3{tx, ty, tz}, b3{sx, sy, sz};
  const double R = arc_dist(a3, b3);
  bool well = false;
  if (R > 0.0) {
    const double qv = div_rn(add_rn(tr, sr), R);
    well = qv < theta;
    if (qv > __ldg(&mac->lo) && qv < __ldg(&mac->hi)) well = mac_lookup(*mac, t, s, well);
  }
  return well;
}

// pair_action on packed node records (one 64-byte record per node: both
// nodes' data in two independent loads), with the MAC screened without
// atan2 or division: for unit centres the chord c = |a - b| = 2 sin(R/2) is
// monotonic in R on [0, pi], so R > X = (r_t + r_s)/theta <=> c^2 > 4
// sin^2(X/2), and sin(X/2) = sin(r_t/2theta) cos(r_s/2theta) + cos(r_t/2theta)
// sin(r_s/2theta) from per-node constants (no cancellation while X/2 <=
// pi/2). Decided only outside a 1e-9 relative margin — far wider than every
// rounding involved and than the exact path's 1e-12 guard band — so each
// screened decision is the one mac_exact (and the reference) makes; inside
// the margin, mac_exact decides. *cb: the refined node's first child.
__device__ __forceinline__ int pair_decide(int t, int s, const NodeRec& T, const NodeRec& S, int rlo, int rhi,
                                           double theta, double pi_theta, int thr, int max_depth, int pc_only,
                                           const MacCtl* __restrict__ mac, int* cb, int* n_exact = nullptr) {
  const int ct = T.cnt, cs = S.cnt;
  int a = 0;
  if (ct > 0 && cs > 0 && T.off < rhi && T.off + ct > rlo) {
    if (ct <= thr && cs <= thr) return 4;  // see pair_action
    const double dx = T.cx - S.cx, dy = T.cy - S.cy, dz = T.cz - S.cz;
    const double c2 = fma(dx, dx, fma(dy, dy, dz * dz));
    int dec = -1;
    if (T.r + S.r <= pi_theta) {
      // a relative margin mu on c^2 is at least mu/2 on R (d ln c^2 / d ln R
      // <= 2), so mu = 4 band keeps every screened pair outside the guard band
      const double mu = __ldg(&mac->screen);
      const double sh = fma(T.sh, S.ch, T.ch * S.sh);
      const double lim = 4.0 * sh * sh;
      if (c2 > lim * (1.0 + mu))
        dec = 1;
      else if (c2 < lim * (1.0 - mu))
        dec = 0;
    }
    if (dec < 0 && n_exact) ++*n_exact;
    const bool well = dec >= 0 ? dec == 1 : mac_exact(t, s, T.cx, T.cy, T.cz, T.r, S.cx, S.cy, S.cz, S.r, theta, mac);
    if (well) {
      a = 4 | classify_kind(ct, cs, thr, pc_only);
    } else {
      const bool rt = ct > cs;
      const NodeRec& Rn = rt ? T : S;
      if (Rn.child_base < 0 || Rn.level >= max_depth) {
        a = 4;  // PP fallback
      } else {
        a = 8 | (rt ? 16 : 0);
        *cb = Rn.child_base;
      }
    }
  }
  return a;
}
__device__ __forceinline__ int pair_action_rec(int t, int s, const NodeRec* __restrict__ rec, int rlo, int rhi,
                                               double theta, double pi_theta, int thr, int max_depth, int pc_only,
                                               const MacCtl* __restrict__ mac, int* cb, int* tlevel) {
  const NodeRec T = rec[t], S = rec[s];
  *tlevel = T.level;
  return pair_decide(t, s, T, S, rlo, rhi, theta, pi_theta, thr, max_depth, pc_only, mac, cb);
}
// near_possible on node records
__device__ __forceinline__ bool near_possible_rec(bool same, const NodeRec& L, const NodeRec& S) {
  if (same) return true;
  const double dx = L.cx - S.cx, dy = L.cy - S.cy, dz = L.cz - S.cz;
  const double lim = L.r + S.r + kNearArc;
  return fma(dx, dx, fma(dy, dy, dz * dz)) < lim * lim;
}

// action: bit0-1 kind, bit2 emit, bit3 refine, bit4 refine target
// [rlo, rhi): the tree-position range whose targets this call evaluates
// (restricted multi-part call; [0, INT_MAX) otherwise): a pair whose target
// bin misses it only feeds other parts' targets and is dropped.
__device__ __forceinline__ int pair_action(int t, int s, const int* __restrict__ cnt, const int* __restrict__ off,
                                           int rlo, int rhi, const double* __restrict__ center,
                                           const double* __restrict__ radius, const int* __restrict__ level,
                                           const int* __restrict__ child_base, double theta, int thr, int max_depth,
                                           int pc_only, const MacCtl* __restrict__ mac) {
  const int ct = cnt[t], cs = cnt[s];
  int a = 0;
  if (ct > 0 && cs > 0 && off[t] < rhi && off[t] + ct > rlo) {
    // two small bins interact directly whatever the MAC says: a
    // well-separated pair is emitted with classify()'s kind, which is PP for
    // two small bins (and stays PP in PC-only mode), the other case is the
    // both-small PP rule (treecode.cpp:43-50) — so the MAC (an atan2, a
    // square root, a division) is evaluated only where it can change the
    // outcome (at C4 the last BFS step alone holds 3.6M leaf pairs)
    if (ct <= thr && cs <= thr) return 4;
    const d3 a3{center[3 * t], center[3 * t + 1], center[3 * t + 2]};
    const d3 b3{center[3 * s], center[3 * s + 1], center[3 * s + 2]};
    const double R = arc_dist(a3, b3);
    bool well = false;
    if (R > 0.0) {
      const double qv = div_rn(add_rn(radius[t], radius[s]), R);
      well = qv < theta;
      if (qv > __ldg(&mac->lo) && qv < __ldg(&mac->hi)) well = mac_lookup(*mac, t, s, well);
    }
    if (well) {
      a = 4 | classify_kind(ct, cs, thr, pc_only);
    } else {
      const bool rt = ct > cs;
      const int r = rt ? t : s;
      if (child_base[r] < 0 || level[r] >= max_depth)
        a = 4;  // PP fallback
      else
        a = 8 | (rt ? 16 : 0);
    }
  }
  return a;
}

// May a pair (x in leaf, y in node s) have 1 - x.y < 2^-20? Only if the two
// circumcircles come within kNearArc of each other (every binned point lies
// in its node's circumcircle, up to the -1e-10 containment tolerance). The
// test is on the chord (<= the arc), so it errs only towards "near".
__device__ __forceinline__ bool near_possible(int leaf, int s, const double* __restrict__ center,
                                              const double* __restrict__ radius) {
  if (leaf == s) return true;
  const double dx = center[3 * leaf] - center[3 * s], dy = center[3 * leaf + 1] - center[3 * s + 1],
               dz = center[3 * leaf + 2] - center[3 * s + 2];
  const double lim = radius[leaf] + radius[s] + kNearArc;
  return fma(dx, dx, fma(dy, dy, dz * dz)) < lim * lim;
}

// Warp-cooperative append of one round of ranges (lane order = list order)
// to a tile's range list. A range that continues the previous one in memory
// with the same near flag is merged into it: the flattened source sequence
// is unchanged, the list (and the kernels' binary searches) shorter —
// sibling leaves' bins and sibling nodes' proxy blocks are contiguous.
// Returns this lane's flattened-list prefix (valid for selected lanes).
struct ListCursor {
  int w = 0;          // ranges written
  int src = 0;        // flattened sources so far
  int last_end = -1;  // end (begin + count) and near flag of the last range
  int last_near = -1;
};
__device__ __forceinline__ int append_ranges(bool sel, const SrcRange& r, SrcRange* __restrict__ out,
                                             ListCursor& cur, int lane) {
  const unsigned full = 0xffffffffu;
  const unsigned bal = __ballot_sync(full, sel);
  const int cnt = sel ? r.count : 0;
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(full, incl, o);
    if (lane >= o) incl += t;
  }
  const int excl = incl - cnt;
  const int total = __shfl_sync(full, incl, 31);
  const int end = r.begin + r.count;
  const unsigned below = bal & ((1u << lane) - 1u);
  const int pl = below ? 31 - __clz(below) : -1;  // previous selected lane
  const int pend = __shfl_sync(full, end, pl < 0 ? 0 : pl);
  const int pnear = __shfl_sync(full, r.near, pl < 0 ? 0 : pl);
  const int prev_end = pl < 0 ? cur.last_end : pend, prev_near = pl < 0 ? cur.last_near : pnear;
  const bool cont = sel && (pl >= 0 || cur.w > 0) && prev_end == r.begin && prev_near == r.near;
  const bool head = sel && !cont;
  const unsigned hb = __ballot_sync(full, head);
  const unsigned after = hb & ~((2u << lane) - 1u);  // heads after this lane (none for lane 31)
  const int nh = after ? __ffs(after) - 1 : -1;
  const int nh_excl = __shfl_sync(full, excl, nh < 0 ? 0 : nh);
  if (head) {
    SrcRange h = r;
    h.count = (nh < 0 ? total : nh_excl) - excl;  // this range and its continuations
    h.pad = cur.src + excl;
    out[cur.w + __popc(hb & ((1u << lane) - 1u))] = h;
  }
  // continuations before this round's first head extend the last range
  const int fh = hb ? __ffs(hb) - 1 : -1;
  const int lead = fh < 0 ? total : __shfl_sync(full, excl, fh);
  __syncwarp();
  if (lane == 0 && lead > 0) out[cur.w - 1].count += lead;
  __syncwarp();
  const int ls = bal ? 31 - __clz(bal) : -1;  // last selected lane
  if (ls >= 0) {
    cur.last_end = __shfl_sync(full, end, ls);
    cur.last_near = __shfl_sync(full, r.near, ls);
  }
  const int pad = cur.src + excl;
  cur.w += __popc(hb);
  cur.src += total;
  return pad;
}

}  // namespace
}  // namespace ssum
