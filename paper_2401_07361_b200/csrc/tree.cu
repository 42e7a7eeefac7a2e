// Face-tree binning on the device: FaceTree::bin_particles / distribute /
// ensure_children (face_tree.cpp:18-88) restated level-synchronously.
//
// The reference descends recursively, node by node. Here every level is a
// handful of device passes over the level's candidate nodes and the
// particles, with one small device->host read per level (how many nodes were
// split and how many candidates the next level has):
//   k_level_decide  per candidate: empty (distribute returns,
//                   face_tree.cpp:40), leaf (bin <= N_T or level >= max_depth,
//                   and no children yet, :42-45), descend into existing
//                   children, or split (ensure_children, :18-37);
//   scans           new node ids (4 per split, in candidate order) and the
//                   next level's candidate slots;
//   k_level_apply   child geometry (bit-exact midpoints, circumcentres,
//                   Cramer constants) and links for the splits, next
//                   candidates;
//   k_descend       every particle of a descending node moves to the first
//                   child whose barycentric min-score is >= -1e-10, else to
//                   the best-scoring child (face_tree.cpp:50-69); bin counts
//                   by warp-aggregated integer atomics.
// Bins end up as contiguous ranges of a tree-order permutation (depth-first,
// children in order, particles ascending by id inside each leaf): offsets are
// filled top-down level by level and one stable radix sort keyed by the
// leaf's offset orders the particles. Node ids are allocated breadth-first;
// the reference's depth-first numbering is reconstructed on export.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace ssum {

namespace {

enum : int { kActLeaf = 0, kActDescend = 1 };

__device__ __forceinline__ d3 load3(const double* p) { return {p[0], p[1], p[2]}; }

// A triangle's circumcap {x : x.centre >= cos R} holds the triangle; a point
// outside the cap by more than kCapMargin (in the cosine) is outside the
// triangle by far more than the containment tolerance (1e-10 in barycentric
// terms is ~1e-13 in distance), so its exact test can be skipped.
constexpr double kCapMargin = 1e-9;
__device__ __forceinline__ bool cap_excludes(const d3& p, const double* ctr, double cos_r_minus_margin) {
  return fma(p.z, ctr[2], fma(p.y, ctr[1], p.x * ctr[0])) < cos_r_minus_margin;
}

// First of the 20 roots whose triangle contains p (face_tree.cpp:77-85), or
// -1; st / skr: the roots' vertices and Cramer constants (shared memory).
__device__ __forceinline__ int find_root(const d3& p, const double* st, const double* skr, const double* sc) {
  for (int f = 0; f < 20; ++f) {
    const double* k = skr + 12 * f;
    if (cap_excludes(p, sc + 3 * f, k[11])) continue;
    const d3 v1 = load3(st + 9 * f), v2 = load3(st + 9 * f + 3), v3 = load3(st + 9 * f + 6);
    int in = contains_screen(v1, v2, v3, d3{k[0], k[1], k[2]}, k[3], k[10], p);
    if (in < 0) in = contains_rn(v1, v2, v3, p);
    if (in) return f;
  }
  return -1;
}

// distribute()'s child choice (face_tree.cpp:50-69): the first of the four
// children cb .. cb+3 whose barycentric min-score is >= -1e-10, else the one
// with the largest (least negative) exact score.
__device__ __forceinline__ int find_child(const d3& p, int cb, const double* __restrict__ tri,
                                          const double* __restrict__ cramer, const double* __restrict__ center) {
  for (int c = cb; c < cb + 4; ++c) {  // first containing child wins (face_tree.cpp:56-61)
    const double* k = cramer + 12 * c;
    if (cap_excludes(p, center + 3 * c, k[11])) continue;
    const double* t = tri + 9 * c;
    const d3 va = load3(t), vb = load3(t + 3), vc = load3(t + 6), bc{k[0], k[1], k[2]};
    int in = contains_screen(va, vb, vc, bc, k[3], k[10], p);
    if (in < 0) in = min_score_rn(va, vb, vc, bc, k[3], p) >= -1e-10;
    if (in) return c;
  }
  int best = cb;  // no child contains p: least-negative exact score (face_tree.cpp:62-69)
  double best_s = -1e300;
  for (int c = cb; c < cb + 4; ++c) {
    const double* t = tri + 9 * c;
    const double* k = cramer + 12 * c;
    const double sc = min_score_rn(load3(t), load3(t + 3), load3(t + 6), d3{k[0], k[1], k[2]}, k[3], p);
    if (sc > best_s) {
      best_s = sc;
      best = c;
    }
  }
  return best;
}

// Root-face assignment: first of the 20 roots with triangle_contains
// (face_tree.cpp:77-85). GeometryError when none contains the particle.
__global__ void k_bin_roots(const double* __restrict__ xyz, int64_t n, const double* __restrict__ tri,
                            const double* __restrict__ cramer, const double* __restrict__ center,
                            int* __restrict__ cur, int* __restrict__ cnt, int* __restrict__ flags) {
  __shared__ double st[20 * 9];
  __shared__ double skr[20 * 12];
  __shared__ double sc[20 * 3];
  __shared__ int scount[20];
  for (int k = threadIdx.x; k < 180; k += blockDim.x) st[k] = tri[k];
  for (int k = threadIdx.x; k < 240; k += blockDim.x) skr[k] = cramer[k];
  for (int k = threadIdx.x; k < 60; k += blockDim.x) sc[k] = center[k];
  if (threadIdx.x < 20) scount[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const int found = find_root(load3(xyz + 3 * i), st, skr, sc);
    cur[i] = found;
    if (found < 0)
      atomicOr(flags, kFlagGeometry);
    else
      atomicAdd(&scount[found], 1);
  }
  __syncthreads();
  if (threadIdx.x < 20 && scount[threadIdx.x]) atomicAdd(&cnt[threadIdx.x], scount[threadIdx.x]);
}

// Node geometry (TreeNode ctor, face_tree.hpp:22-25) plus the per-node
// constants the binning and the barycentric passes reuse:
// cramer = [v2 x v3, v1.(v2 x v3), v3 x v1, v1 x v2, 1 / det, 0].
__device__ void write_node(double* tri, double* center, double* radius, double* cramer, int id, d3 a,
                           d3 b, d3 c, int* flags) {
  int bad = 0;
  double* t = tri + 9 * id;
  t[0] = a.x; t[1] = a.y; t[2] = a.z;
  t[3] = b.x; t[4] = b.y; t[5] = b.z;
  t[6] = c.x; t[7] = c.y; t[8] = c.z;
  if (!triangle_ok(a, b, c)) bad = 1;
  const d3 cc = circumcenter_rn(a, b, c, &bad);
  center[3 * id] = cc.x;
  center[3 * id + 1] = cc.y;
  center[3 * id + 2] = cc.z;
  radius[id] = arc_dist(cc, a);
  const d3 bc = cross_rn(b, c);
  const d3 n2 = cross_rn(c, a);
  const d3 n3 = cross_rn(a, b);
  double* k = cramer + 12 * id;
  k[0] = bc.x; k[1] = bc.y; k[2] = bc.z;
  k[3] = dot_rn(a, bc);
  k[4] = n2.x; k[5] = n2.y; k[6] = n2.z;
  k[7] = n3.x; k[8] = n3.y; k[9] = n3.z;
  k[10] = 1.0 / k[3];  // screened containment (contains_screen)
  k[11] = cos(radius[id]) - kCapMargin;  // circumcap pre-filter (cap_excludes)
  if (bad) atomicOr(flags, kFlagGeometry);
}

// distribute()'s per-node decision (face_tree.cpp:40-47).
__global__ void k_level_decide(const int* __restrict__ cand, int m, const int* __restrict__ cnt,
                               const int* __restrict__ child_base, const int* __restrict__ level, int nt,
                               int max_depth, unsigned char* __restrict__ act, unsigned char* __restrict__ is_leaf,
                               int* __restrict__ split, int* __restrict__ nextc) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k > m) return;
  if (k == m) {  // sentinel for the exclusive scans (totals at index m)
    split[k] = 0;
    nextc[k] = 0;
    return;
  }
  const int id = cand[k];
  const int c = cnt[id];
  int s = 0, nx = 0;
  if (c > 0) {
    if (child_base[id] >= 0) {
      act[id] = kActDescend;
      nx = 4;
    } else if (c <= nt || level[id] >= max_depth) {
      act[id] = kActLeaf;
      is_leaf[id] = 1;
    } else {
      act[id] = kActDescend;
      s = 1;
      nx = 4;
    }
  }
  split[k] = s;
  nextc[k] = nx;
}

// ensure_children (face_tree.cpp:18-37) for the splits of this level —
// midpoints renormalised, children {v1,m12,m31}, {m12,v2,m23},
// {m31,m23,v3}, {m12,m23,m31} — and the next level's candidate list.
__global__ void k_level_apply(const int* __restrict__ cand, int m, const int* __restrict__ split,
                              const int* __restrict__ split_pos, const int* __restrict__ nextc,
                              const int* __restrict__ next_pos, int node_base, int call_index, double* tri,
                              double* center, double* radius, double* cramer, int* level, int* parent,
                              int* child_base, int* created_call, unsigned long long* key,
                              int* __restrict__ cand_next, int* flags) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int id = cand[k];
  int cb = child_base[id];
  if (split[k]) {
    cb = node_base + 4 * split_pos[k];
    const double* t = tri + 9 * id;
    const d3 v1 = load3(t), v2 = load3(t + 3), v3 = load3(t + 6);
    int bad = 0;
    const d3 m12 = unit_rn(add3(v1, v2), &bad);
    const d3 m23 = unit_rn(add3(v2, v3), &bad);
    const d3 m31 = unit_rn(add3(v3, v1), &bad);
    if (bad) atomicOr(flags, kFlagGeometry);
    write_node(tri, center, radius, cramer, cb + 0, v1, m12, m31, flags);
    write_node(tri, center, radius, cramer, cb + 1, m12, v2, m23, flags);
    write_node(tri, center, radius, cramer, cb + 2, m31, m23, v3, flags);
    write_node(tri, center, radius, cramer, cb + 3, m12, m23, m31, flags);
    const int lv = level[id] + 1;
    const int ks = kKeyRootShift - 2 * min(lv, kKeyMaxLevel);  // keys past kKeyMaxLevel are unused
    for (int q = 0; q < 4; ++q) {
      level[cb + q] = lv;
      parent[cb + q] = id;
      child_base[cb + q] = -1;
      created_call[cb + q] = call_index;
      key[cb + q] = key[id] | (static_cast<unsigned long long>(q) << ks);
    }
    child_base[id] = cb;
  }
  if (nextc[k])
    for (int q = 0; q < 4; ++q) cand_next[next_pos[k] + q] = cb + q;
}

// One level of distribute (face_tree.cpp:39-71) for every still-active particle.
__global__ void k_descend(const double* __restrict__ xyz, int64_t n, int* __restrict__ cur,
                          int* __restrict__ leaf_of, const unsigned char* __restrict__ act,
                          const int* __restrict__ child_base, const double* __restrict__ tri,
                          const double* __restrict__ cramer, const double* __restrict__ center,
                          int* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int node = cur[i];
  if (node < 0) return;
  if (act[node] == kActLeaf) {
    leaf_of[i] = node;
    cur[i] = -1;
    return;
  }
  const int placed = find_child(load3(xyz + 3 * i), child_base[node], tri, cramer, center);
  cur[i] = placed;
  // warp-aggregated bin count: one atomic per distinct child in the warp
  const unsigned peers = __match_any_sync(__activemask(), placed);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&cnt[placed], __popc(peers));
}

// ---- reuse path: every particle's path through the existing children ------
//
// Once the tree exists, distribute() descends into existing children
// whatever the bin size (face_tree.cpp:42-47), so a particle's path down to
// the first childless node is fixed by geometry alone. One kernel walks each
// particle down that path and emits the node's depth-first path key; one
// radix sort of (key, id) is the tree-order permutation; per-node bin ranges
// are two binary searches of the node's key range in the sorted keys. The
// binning is final unless a childless node must split (bin > N_T below
// max_depth) — then the level-synchronous build runs instead.
// Guessed leaf (the particle's leaf in the previous call): accepted when the
// node is childless and x lies inside its spherical triangle by at least
// kGuessMargin rad from each edge great circle. Nodes tile their parents
// exactly, so every sibling along the root-to-node path then lies >= that far
// from x, i.e. its barycentric score is <= ~ -kGuessMargin sin(alpha/2) / h
// (alpha >= ~50 deg the triangle angles, h <= ~1 the heights): below -4e-9,
// 40x beyond the -1e-10 containment tolerance and the 1e-13 guard band. The
// first-containing descent (face_tree.cpp:50-69) therefore ends at this
// node, and the shortcut returns exactly what the walk would. The same holds
// for any node x lies that deep inside (a node contains its descendants, so
// x is at least as deep inside every ancestor): when the guessed leaf fails
// the test — x moved, or sits on the leaf's boundary, as a third of the
// mesh vertices do — the walk resumes from the guess's deepest ancestor that
// passes it, descending from there with the ordinary child choice, and only
// falls back to the root when none does.
constexpr double kGuessMargin = 1e-8;
__device__ __forceinline__ bool deep_inside(const d3& p, const double* __restrict__ k) {
  const double sg = k[3] < 0.0 ? -1.0 : 1.0;  // inside: x . n_j has det's sign
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double* n = k + (j == 0 ? 0 : 1 + 3 * j);  // n1 = k[0..2], n2 = k[4..6], n3 = k[7..9]
    const double r = sg * fma(p.z, n[2], fma(p.y, n[1], p.x * n[0]));
    const double nn = fma(n[2], n[2], fma(n[1], n[1], n[0] * n[0]));
    if (!(r > 0.0 && r * r >= (kGuessMargin * kGuessMargin) * nn)) return false;
  }
  return true;
}

__global__ void k_iota(int* __restrict__ v, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) v[i] = static_cast<int>(i);
}

__global__ void k_walk(const double* __restrict__ xyz, int64_t i0, int64_t i1, const int* __restrict__ order,
                       const double* __restrict__ tri,
                       const double* __restrict__ cramer, const double* __restrict__ center,
                       const int* __restrict__ child_base, const int* __restrict__ parent,
                       const unsigned long long* __restrict__ nkey,
                       unsigned long long* __restrict__ key, int* __restrict__ ids, int* __restrict__ leaf_of,
                       int guess_nodes, int* __restrict__ flags) {
  __shared__ double st[20 * 9];
  __shared__ double skr[20 * 12];
  __shared__ double sc[20 * 3];
  for (int k = threadIdx.x; k < 180; k += blockDim.x) st[k] = tri[k];
  for (int k = threadIdx.x; k < 240; k += blockDim.x) skr[k] = cramer[k];
  for (int k = threadIdx.x; k < 60; k += blockDim.x) sc[k] = center[k];
  __syncthreads();
  const int64_t k = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= i1) return;
  // order: the previous call's tree order, so that a warp's particles are
  // neighbours and share their descent (results still land at index i)
  const int64_t i = order ? order[k] : k;
  const d3 p = load3(xyz + 3 * i);
  // guess_nodes > 0: leaf_of holds the previous call's leaves (node ids
  // below guess_nodes)
  int node = -1;
  if (guess_nodes > 0) {
    const int g = leaf_of[i];
    if (g >= 0 && g < guess_nodes) {
      if (child_base[g] < 0 && deep_inside(p, cramer + 12 * g)) {
        key[i] = nkey[g];
        ids[i] = static_cast<int>(i);
        return;  // leaf_of[i] stays g
      }
      for (int a = parent[g]; a >= 0; a = parent[a])
        if (deep_inside(p, cramer + 12 * a)) {
          node = a;
          break;
        }
    }
  }
  if (node < 0) node = find_root(p, st, skr, sc);
  if (node < 0) {
    atomicOr(flags, kFlagGeometry);
    key[i] = ~0ull;
    leaf_of[i] = -1;
  } else {
    for (int cb = child_base[node]; cb >= 0; cb = child_base[node]) node = find_child(p, cb, tri, cramer, center);
    key[i] = nkey[node];
    leaf_of[i] = node;
  }
  ids[i] = static_cast<int>(i);
}

// How many consecutive input particles share a leaf (input-order coherence).
__global__ void k_coherence(const int* __restrict__ leaf_of, int64_t n, int* count) {
  __shared__ int block_sum;
  if (threadIdx.x == 0) block_sum = 0;
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const bool same = i + 1 < n && leaf_of[i] == leaf_of[i + 1];
  const unsigned m = __ballot_sync(0xffffffffu, same);
  if ((threadIdx.x & 31) == 0 && m) atomicAdd(&block_sum, __popc(m));
  __syncthreads();
  if (threadIdx.x == 0 && block_sum) atomicAdd(count, block_sum);
}

__device__ __forceinline__ int lower_bound_u64(const unsigned long long* __restrict__ a, int n, unsigned long long v) {
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

// Bin range of every node: its key range [key, key + 4^(kKeyMaxLevel - level))
// in the sorted keys. Flags the leaves of this call (non-empty, childless)
// and counts the childless nodes that would have to split.
__global__ void k_node_ranges(int nn, const unsigned long long* __restrict__ nkey, const int* __restrict__ level,
                              const int* __restrict__ child_base, const unsigned long long* __restrict__ skey,
                              int n, int nt, int max_depth, int* __restrict__ cnt, int* __restrict__ off,
                              unsigned char* __restrict__ is_leaf, int* __restrict__ n_split) {
  const int id = blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= nn) return;
  const unsigned long long k0 = nkey[id];
  const unsigned long long k1 = k0 + (1ull << (kKeyRootShift - 2 * level[id]));
  const int b = lower_bound_u64(skey, n, k0);
  const int e = lower_bound_u64(skey, n, k1);
  cnt[id] = e - b;
  off[id] = b;
  const bool leaf = e > b && child_base[id] < 0;
  is_leaf[id] = leaf ? 1 : 0;
  if (leaf && e - b > nt && level[id] < max_depth) atomicAdd(n_split, 1);
}

// First tree position of each leaf: where the sorted key changes.
__global__ void k_leaf_starts(const unsigned long long* __restrict__ skey, int n, unsigned char* __restrict__ flag) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < n) flag[k] = (k == 0 || skey[k] != skey[k - 1]) ? 1 : 0;
}

__global__ void k_leaf_list(const int* __restrict__ start, const int* __restrict__ nl, const int* __restrict__ perm,
                            const int* __restrict__ leaf_of, int* __restrict__ leaves) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < *nl) leaves[r] = leaf_of[perm[start[r]]];
}

// Depth-first bin offsets, top-down: roots in face order ...
__global__ void k_root_offsets(const int* __restrict__ cnt, int* __restrict__ off) {
  if (threadIdx.x == 0) {
    int run = 0;
    for (int f = 0; f < 20; ++f) {
      off[f] = run;
      run += cnt[f];
    }
  }
}

// ... then each non-empty descending node hands out its range to its children.
__global__ void k_child_offsets(const int* __restrict__ nodes, int m, const int* __restrict__ cnt,
                                const int* __restrict__ child_base, const unsigned char* __restrict__ is_leaf,
                                int* __restrict__ off) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int id = nodes[k];
  if (cnt[id] == 0 || is_leaf[id]) return;
  const int cb = child_base[id];
  int o = off[id];
  for (int q = 0; q < 4; ++q) {
    off[cb + q] = o;
    o += cnt[cb + q];
  }
}

__global__ void k_leaf_keys(const int* __restrict__ leaves, int nl, const int* __restrict__ off, int* __restrict__ keys) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nl) keys[k] = off[leaves[k]];
}

__global__ void k_sort_keys(const int* __restrict__ leaf_of, int64_t n, const int* __restrict__ off,
                            int* __restrict__ keys, int* __restrict__ vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  keys[i] = off[leaf_of[i]];
  vals[i] = static_cast<int>(i);
}

__global__ void k_pos_leaf(const int* __restrict__ perm, int64_t n, const int* __restrict__ leaf_of,
                           int* __restrict__ pos_leaf) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) pos_leaf[k] = leaf_of[perm[k]];
}

template <class T>
void scan_excl(Ctx& c, const T* in, T* out, int n) {
  size_t tmp = 0;
  SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, in, out, n, c.stream));
  c.cub_tmp.ensure(tmp);
  SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(c.cub_tmp.p, tmp, in, out, n, c.stream));
  c.launches += 2;
}

}  // namespace

// Node arrays (geometry persists; `need` nodes).
static void grow_nodes(Ctx& c, int need) {
  NodeTable& t = c.nodes;
  t.tri.ensure(size_t(need) * 9, true, c.stream);
  t.center.ensure(size_t(need) * 3, true, c.stream);
  t.radius.ensure(size_t(need), true, c.stream);
  t.cramer.ensure(size_t(need) * 12, true, c.stream);
  t.child_base.ensure(size_t(need), true, c.stream);
  t.level.ensure(size_t(need), true, c.stream);
  t.parent.ensure(size_t(need), true, c.stream);
  t.created_call.ensure(size_t(need), true, c.stream);
  t.key.ensure(size_t(need), true, c.stream);
  c.bins.cnt.ensure(size_t(need), true, c.stream);
  c.bins.act.ensure(size_t(need), true, c.stream);
  c.bins.is_leaf.ensure(size_t(need), true, c.stream);
  c.bins.off.ensure(size_t(need), true, c.stream);
}

// The 20 roots, built with the host libm so their vertices are bit-identical
// to the reference's (IcosaMesh::base_icosahedron, icosa_mesh.cpp:10-35;
// latlon_to_unit, geometry.cpp:41-44; FaceTree ctor, face_tree.cpp:9-16).
void tree_init_roots(Ctx& c) {
  c.host = HostTree{};
  const double kPi = 3.14159265358979323846;  // M_PI
  int bad = 0;
  auto latlon = [&](double lat, double lon) {
    const double cl = std::cos(lat);
    return unit_rn(d3{cl * std::cos(lon), cl * std::sin(lon), std::sin(lat)}, &bad);
  };
  d3 v[12];
  v[0] = unit_rn(d3{0.0, 0.0, 1.0}, &bad);
  const double rl = std::atan(0.5);
  for (int k = 0; k < 5; ++k) v[1 + k] = latlon(rl, 2.0 * kPi * k / 5.0);
  for (int k = 0; k < 5; ++k) v[6 + k] = latlon(-rl, 2.0 * kPi * k / 5.0 + kPi / 5.0);
  v[11] = unit_rn(d3{0.0, 0.0, -1.0}, &bad);
  std::vector<double> tri(20 * 9), center(20 * 3), radius(20), cramer(20 * 12);
  int f = 0;
  for (int k = 0; k < 5; ++k) {
    const int u = 1 + k, un = 1 + (k + 1) % 5, l = 6 + k, ln = 6 + (k + 1) % 5;
    const int faces[4][3] = {{0, u, un}, {u, l, un}, {un, l, ln}, {11, ln, l}};
    for (int q = 0; q < 4; ++q, ++f) {
      const d3 a = v[faces[q][0]], b = v[faces[q][1]], cc = v[faces[q][2]];
      const d3 t3[3] = {a, b, cc};
      for (int z = 0; z < 3; ++z) {
        tri[9 * f + 3 * z] = t3[z].x;
        tri[9 * f + 3 * z + 1] = t3[z].y;
        tri[9 * f + 3 * z + 2] = t3[z].z;
      }
      if (!triangle_ok(a, b, cc)) bad = 1;
      const d3 ctr = circumcenter_rn(a, b, cc, &bad);
      center[3 * f] = ctr.x;
      center[3 * f + 1] = ctr.y;
      center[3 * f + 2] = ctr.z;
      radius[f] = arc_dist(ctr, a);
      const d3 bc = cross_rn(b, cc), n2 = cross_rn(cc, a), n3 = cross_rn(a, b);
      const double det = dot_rn(a, bc);
      const double kk[12] = {bc.x, bc.y, bc.z, det, n2.x, n2.y, n2.z, n3.x, n3.y, n3.z, 1.0 / det,
                             std::cos(radius[f]) - kCapMargin};
      std::copy(kk, kk + 12, cramer.begin() + 12 * f);
    }
  }
  if (bad) throw Error(SSUM_GEOMETRY, "degenerate base icosahedron");
  c.nodes.count = 20;
  c.nodes.max_level = 0;
  grow_nodes(c, 1024);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.tri.p, tri.data(), tri.size() * 8, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.center.p, center.data(), center.size() * 8, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.radius.p, radius.data(), radius.size() * 8, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.cramer.p, cramer.data(), cramer.size() * 8, cudaMemcpyHostToDevice, c.stream));
  const std::vector<int> zero(20, 0), minus(20, -1);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.level.p, zero.data(), 80, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.created_call.p, zero.data(), 80, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.parent.p, minus.data(), 80, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.child_base.p, minus.data(), 80, cudaMemcpyHostToDevice, c.stream));
  std::vector<unsigned long long> rkey(20);
  for (int q = 0; q < 20; ++q) rkey[q] = static_cast<unsigned long long>(q) << kKeyRootShift;
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.key.p, rkey.data(), 160, cudaMemcpyHostToDevice, c.stream));
  if (!c.bins.h_small) SSUM_CUDA_CHECK(cudaMallocHost(&c.bins.h_small, 64 * sizeof(int)));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// Binning through the existing tree (see k_walk). Returns false, with
// nothing of the call's state committed, when the tree cannot be reused as
// is: no children yet, deeper than the path keys reach, or a childless node
// whose bin now needs a split.
static bool bin_reuse(Ctx& c, const double* d_xyz, int64_t n, int nt, int max_depth, int64_t prev_perm_n) {
  NodeTable& T = c.nodes;
  Binned& B = c.bins;
  if (T.count <= 20 || T.max_level > kKeyMaxLevel || n > 0x3fffffff) return false;
  const int nn = T.count;
  const int ni = static_cast<int>(n);
  const int bs = 256;
  B.wkey.ensure(size_t(n));
  B.wkey2.ensure(size_t(n));
  B.sort_vals.ensure(std::max<size_t>(size_t(n), size_t(nn)));
  B.perm.ensure(size_t(n));
  B.pos_leaf.ensure(size_t(n));
  B.d_leaves.ensure(size_t(nn));
  B.leaf_pos.ensure(size_t(nn));
  B.leaf_flag.ensure(size_t(n));
  // [0] splits needed, [1] leaves, [2] input-order coherence, [3..5] the
  // subtree list plan's big nodes, cut nodes, leaf tiles
  int* d_cnt = c.d_flags.p + 16;
  SSUM_CUDA_CHECK(cudaMemsetAsync(d_cnt, 0, 6 * sizeof(int), c.stream));
  // Walk order: input order when the input is spatially coherent (the last
  // call found most consecutive particles in one leaf) — a host-pointer call
  // then walks each input piece as soon as it has landed — else the previous
  // call's tree order, so that a warp's particles are neighbours and share
  // their descent.
  const bool by_tree = prev_perm_n == n && !B.input_coherent;
  const int pieces = (c.io.active && !by_tree) ? Ctx::kIoChunks : 1;
  const int* order = by_tree ? B.perm.p : nullptr;
  // the previous call's leaf of each particle is the walk's first guess
  // (verified per particle, so any stale guess only costs the full walk)
  const int guess_nodes = prev_perm_n == n ? nn : 0;
  const bool walked = B.walked_n == n;  // every rank walked its shard, the keys were all-gathered
  B.walked_n = -1;
  if (walked) {
    k_iota<<<grid_for(n, bs), bs, 0, c.stream>>>(B.sort_vals.p, n);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  if (c.io.active && pieces == 1) SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.io.xyz[Ctx::kIoChunks - 1], 0));
  for (int j = 0; j < (walked ? 0 : pieces); ++j) {
    const int64_t a = pieces > 1 ? c.io.bounds[j] : 0, b = pieces > 1 ? c.io.bounds[j + 1] : n;
    if (pieces > 1) SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.io.xyz[j], 0));
    if (b <= a) continue;
    k_walk<<<grid_for(b - a, bs), bs, 0, c.stream>>>(d_xyz, a, b, order, T.tri.p, T.cramer.p, T.center.p,
                                                     T.child_base.p, T.parent.p, T.key.p, B.wkey.p, B.sort_vals.p,
                                                     B.leaf_of.p, guess_nodes, c.d_flags.p);
    SSUM_LAUNCH_CHECK();
  }
  const int begin_bit = kKeyRootShift - 2 * T.max_level;
  size_t tmp = 0;
  SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, B.wkey.p, B.wkey2.p, B.sort_vals.p, B.perm.p, ni,
                                                  begin_bit, 64, c.stream));
  c.cub_tmp.ensure(tmp);
  SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, tmp, B.wkey.p, B.wkey2.p, B.sort_vals.p, B.perm.p, ni,
                                                  begin_bit, 64, c.stream));
  k_node_ranges<<<grid_for(nn, bs), bs, 0, c.stream>>>(nn, T.key.p, T.level.p, T.child_base.p, B.wkey2.p, ni, nt,
                                                       max_depth, B.cnt.p, B.off.p, B.is_leaf.p, d_cnt);
  SSUM_LAUNCH_CHECK();
  k_leaf_starts<<<grid_for(n, bs), bs, 0, c.stream>>>(B.wkey2.p, ni, B.leaf_flag.p);
  SSUM_LAUNCH_CHECK();
  {
    cub::CountingInputIterator<int> pos(0);
    tmp = 0;
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, tmp, pos, B.leaf_flag.p, B.leaf_pos.p, d_cnt + 1, ni,
                                               c.stream));
    c.cub_tmp.ensure(tmp);
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(c.cub_tmp.p, tmp, pos, B.leaf_flag.p, B.leaf_pos.p, d_cnt + 1, ni,
                                               c.stream));
  }
  k_leaf_list<<<grid_for(n, bs), bs, 0, c.stream>>>(B.leaf_pos.p, d_cnt + 1, B.perm.p, B.leaf_of.p, B.d_leaves.p);
  SSUM_LAUNCH_CHECK();
  k_pos_leaf<<<grid_for(n, bs), bs, 0, c.stream>>>(B.perm.p, n, B.leaf_of.p, B.pos_leaf.p);
  SSUM_LAUNCH_CHECK();
  c.launches += 12;
  plan_subtrees(c, nt, d_cnt + 1, d_cnt + 3);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(B.h_small, c.d_flags.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  k_coherence<<<grid_for(n, 1024), 1024, 0, c.stream>>>(B.leaf_of.p, n, d_cnt + 2);
  SSUM_LAUNCH_CHECK();
  SSUM_CUDA_CHECK(cudaMemcpyAsync(B.h_small + 1, d_cnt, 6 * sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  if (B.h_small[0] & kFlagGeometry) check_flags(c, "bin_particles: particle contained in no root face");
  if (B.h_small[1] > 0) return false;
  B.n_leaves = B.h_small[2];
  B.input_coherent = 2 * int64_t(B.h_small[3]) > n;
  B.perm_n = n;
  plan_subtrees_done(c, B.h_small + 4);
  return true;
}

// Multi-GPU binning: rank r walks only particles
// [i0, i1) of the caller's order through the existing tree (the same k_walk,
// previous leaves as guesses); the caller all-gathers the keys and leaves of
// the other shards into this context's wkey / leaf_of (ssum_bin_walk_shard
// hands out the pointers, slots >= n rows each), and the next binning of the
// same n particles starts at the sort — bitwise the unsharded binning, with
// the walk (the binning's largest part) divided by the rank count.
bool tree_walk_shard(Ctx& c, const double* d_xyz, int64_t n, int64_t i0, int64_t i1, int64_t slots) {
  NodeTable& T = c.nodes;
  Binned& B = c.bins;
  B.walked_n = -1;
  if (T.count <= 20 || T.max_level > kKeyMaxLevel || n > 0x3fffffff || n <= 0) return false;
  B.wkey.ensure(size_t(std::max(slots, n)));
  B.leaf_of.ensure(size_t(std::max(slots, n)), true, c.stream);  // previous leaves: the guesses
  B.sort_vals.ensure(std::max<size_t>(size_t(n), size_t(T.count)));
  const int guess_nodes = B.perm_n == n ? T.count : 0;
  SSUM_CUDA_CHECK(cudaMemsetAsync(c.d_flags.p, 0, sizeof(int), c.stream));
  if (i1 > i0) {
    k_walk<<<grid_for(i1 - i0, 256), 256, 0, c.stream>>>(d_xyz, i0, i1, nullptr, T.tri.p, T.cramer.p, T.center.p,
                                                          T.child_base.p, T.parent.p, T.key.p, B.wkey.p, B.sort_vals.p,
                                                          B.leaf_of.p, guess_nodes, c.d_flags.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  B.walked_n = n;
  return true;
}

void tree_bin(Ctx& c, const double* d_xyz, int64_t n, int nt, int max_depth) {
  Binned& B = c.bins;
  // the previous permutation (a walk-order hint) is only trusted if that
  // binning completed; it is invalid until this one does
  const int64_t prev_perm_n = B.perm_n;
  B.perm_n = -1;
  c.call_index++;
  c.host.valid = false;
  c.sub.valid = false;
  B.n = n;
  B.n_leaves = 0;
  B.level_span.clear();
  const int bs = 256;

  // Fresh per-call counts and leaf flags; node geometry persists (face_tree.cpp:75).
  SSUM_CUDA_CHECK(cudaMemsetAsync(B.cnt.p, 0, size_t(c.nodes.count) * sizeof(int), c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(B.is_leaf.p, 0, size_t(c.nodes.count), c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(c.d_flags.p, 0, sizeof(int), c.stream));
  if (n == 0) return;
  B.cur.ensure(size_t(n));
  B.leaf_of.ensure(size_t(n));
  if (bin_reuse(c, d_xyz, n, nt, max_depth, prev_perm_n)) {
    trace().mark("bin.reuse");
    return;
  }
  // level-synchronous build from the roots (fresh counts again: the reuse
  // attempt may have filled them); needs the whole input
  if (c.io.active) SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.io.xyz[Ctx::kIoChunks - 1], 0));
  SSUM_CUDA_CHECK(cudaMemsetAsync(B.cnt.p, 0, size_t(c.nodes.count) * sizeof(int), c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(B.is_leaf.p, 0, size_t(c.nodes.count), c.stream));

  k_bin_roots<<<grid_for(n, bs), bs, 0, c.stream>>>(d_xyz, n, c.nodes.tri.p, c.nodes.cramer.p, c.nodes.center.p,
                                                     B.cur.p, B.cnt.p, c.d_flags.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  check_flags(c, "bin_particles: particle contained in no root face");
  trace().mark("bin.roots");

  // level 0 candidates: the 20 roots
  int m = 20;
  B.cand.ensure(1024);
  B.levels.ensure(1024);
  {
    int roots[20];
    for (int f = 0; f < 20; ++f) roots[f] = f;
    SSUM_CUDA_CHECK(cudaMemcpyAsync(B.cand.p, roots, sizeof(roots), cudaMemcpyHostToDevice, c.stream));
  }
  int levels_used = 0;
  while (m > 0) {
    // node table room for every candidate splitting (4 m new nodes)
    const int room = c.nodes.count + 4 * m;
    if (room > static_cast<int>(c.nodes.child_base.cap)) grow_nodes(c, room);
    SSUM_CUDA_CHECK(cudaMemsetAsync(B.cnt.p + c.nodes.count, 0, size_t(4) * m * sizeof(int), c.stream));
    SSUM_CUDA_CHECK(cudaMemsetAsync(B.is_leaf.p + c.nodes.count, 0, size_t(4) * m, c.stream));
    B.split.ensure(size_t(m) + 1);
    B.split_pos.ensure(size_t(m) + 1);
    B.nextc.ensure(size_t(m) + 1);
    B.next_pos.ensure(size_t(m) + 1);
    B.cand_next.ensure(size_t(4) * m);
    // keep this level's candidates for the offset pass
    B.levels.ensure(size_t(levels_used) + size_t(m), true, c.stream);
    SSUM_CUDA_CHECK(cudaMemcpyAsync(B.levels.p + levels_used, B.cand.p, size_t(m) * 4, cudaMemcpyDeviceToDevice,
                                    c.stream));
    B.level_span.emplace_back(levels_used, m);
    levels_used += m;

    k_level_decide<<<grid_for(m + 1, bs), bs, 0, c.stream>>>(B.cand.p, m, B.cnt.p, c.nodes.child_base.p,
                                                              c.nodes.level.p, nt, max_depth, B.act.p, B.is_leaf.p,
                                                              B.split.p, B.nextc.p);
    SSUM_LAUNCH_CHECK();
    scan_excl(c, B.split.p, B.split_pos.p, m + 1);
    scan_excl(c, B.nextc.p, B.next_pos.p, m + 1);
    k_level_apply<<<grid_for(m, 128), 128, 0, c.stream>>>(
        B.cand.p, m, B.split.p, B.split_pos.p, B.nextc.p, B.next_pos.p, c.nodes.count, c.call_index, c.nodes.tri.p,
        c.nodes.center.p, c.nodes.radius.p, c.nodes.cramer.p, c.nodes.level.p, c.nodes.parent.p,
        c.nodes.child_base.p, c.nodes.created_call.p, c.nodes.key.p, B.cand_next.p, c.d_flags.p);
    SSUM_LAUNCH_CHECK();
    k_descend<<<grid_for(n, bs), bs, 0, c.stream>>>(d_xyz, n, B.cur.p, B.leaf_of.p, B.act.p, c.nodes.child_base.p,
                                                     c.nodes.tri.p, c.nodes.cramer.p, c.nodes.center.p, B.cnt.p);
    SSUM_LAUNCH_CHECK();
    c.launches += 3;
    SSUM_CUDA_CHECK(cudaMemcpyAsync(B.h_small, B.split_pos.p + m, 4, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(B.h_small + 1, B.next_pos.p + m, 4, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    trace().mark("bin.level");
    c.nodes.count += 4 * B.h_small[0];
    if (B.h_small[0] > 0) c.nodes.max_level = std::max(c.nodes.max_level, static_cast<int>(B.level_span.size()));
    m = B.h_small[1];
    std::swap(B.cand, B.cand_next);
  }
  check_flags(c, "bin_particles: degenerate child triangle");

  // Depth-first bin offsets, top-down level by level.
  k_root_offsets<<<1, 32, 0, c.stream>>>(B.cnt.p, B.off.p);
  for (const auto& sp : B.level_span) {
    k_child_offsets<<<grid_for(sp.second, bs), bs, 0, c.stream>>>(B.levels.p + sp.first, sp.second, B.cnt.p,
                                                                  c.nodes.child_base.p, B.is_leaf.p, B.off.p);
    SSUM_LAUNCH_CHECK();
  }
  c.launches += 1 + static_cast<int64_t>(B.level_span.size());

  // Non-empty leaves in depth-first order: select, then sort by offset.
  const int nn = c.nodes.count;
  B.d_leaves.ensure(size_t(nn));
  B.leaf_keys.ensure(size_t(nn) * 2);
  B.sort_vals.ensure(std::max<size_t>(size_t(n), size_t(nn)));
  {
    cub::CountingInputIterator<int> ids(0);
    int* d_nsel = c.d_flags.p + 8;
    size_t tmp = 0;
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(nullptr, tmp, ids, B.is_leaf.p, B.sort_vals.p, d_nsel, nn, c.stream));
    c.cub_tmp.ensure(tmp);
    SSUM_CUDA_CHECK(cub::DeviceSelect::Flagged(c.cub_tmp.p, tmp, ids, B.is_leaf.p, B.sort_vals.p, d_nsel, nn,
                                               c.stream));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(B.h_small, d_nsel, 4, cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    B.n_leaves = B.h_small[0];
    const int nl = B.n_leaves;
    k_leaf_keys<<<grid_for(std::max(nl, 1), bs), bs, 0, c.stream>>>(B.sort_vals.p, nl, B.off.p, B.leaf_keys.p);
    int end_bit = 1;
    while ((int64_t(1) << end_bit) < n) ++end_bit;
    tmp = 0;
    SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, B.leaf_keys.p, B.leaf_keys.p + nn, B.sort_vals.p,
                                                    B.d_leaves.p, nl, 0, end_bit, c.stream));
    c.cub_tmp.ensure(tmp);
    SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, tmp, B.leaf_keys.p, B.leaf_keys.p + nn,
                                                    B.sort_vals.p, B.d_leaves.p, nl, 0, end_bit, c.stream));
    c.launches += 7;
  }
  trace().mark("bin.offsets_leaves");

  // Permutation: stable sort of particle ids by their leaf's offset.
  B.sort_keys.ensure(size_t(n));
  B.sort_keys2.ensure(size_t(n));
  B.perm.ensure(size_t(n));
  B.pos_leaf.ensure(size_t(n));
  k_sort_keys<<<grid_for(n, bs), bs, 0, c.stream>>>(B.leaf_of.p, n, B.off.p, B.sort_keys.p, B.sort_vals.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  int end_bit = 1;
  while ((int64_t(1) << end_bit) < n) ++end_bit;
  size_t tmp = 0;
  SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, B.sort_keys.p, B.sort_keys2.p, B.sort_vals.p, B.perm.p,
                                                  static_cast<int>(n), 0, end_bit, c.stream));
  c.cub_tmp.ensure(tmp);
  SSUM_CUDA_CHECK(cub::DeviceRadixSort::SortPairs(c.cub_tmp.p, tmp, B.sort_keys.p, B.sort_keys2.p, B.sort_vals.p,
                                                  B.perm.p, static_cast<int>(n), 0, end_bit, c.stream));
  c.launches += 4;
  k_pos_leaf<<<grid_for(n, bs), bs, 0, c.stream>>>(B.perm.p, n, B.leaf_of.p, B.pos_leaf.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  B.perm_n = n;
}

// Host snapshot of the node structure and this call's counts/offsets.
const HostTree& host_tree(Ctx& c) {
  HostTree& h = c.host;
  if (h.valid) return h;
  const size_t nn = size_t(c.nodes.count);
  h.level.resize(nn);
  h.parent.resize(nn);
  h.child_base.resize(nn);
  h.created_call.resize(nn);
  h.cnt.resize(nn);
  h.off.resize(nn);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h.level.data(), c.nodes.level.p, nn * 4, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h.parent.data(), c.nodes.parent.p, nn * 4, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h.child_base.data(), c.nodes.child_base.p, nn * 4, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h.created_call.data(), c.nodes.created_call.p, nn * 4, cudaMemcpyDeviceToHost,
                                  c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h.cnt.data(), c.bins.cnt.p, nn * 4, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(h.off.data(), c.bins.off.p, nn * 4, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  if (c.bins.n == 0) std::fill(h.cnt.begin(), h.cnt.end(), 0);
  h.valid = true;
  return h;
}

}  // namespace ssum
