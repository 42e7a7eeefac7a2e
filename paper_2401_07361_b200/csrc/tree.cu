// Face-tree binning on the device: FaceTree::bin_particles / distribute /
// ensure_children (face_tree.cpp:18-88) restated level-synchronously.
//
// The reference descends recursively, node by node. Here every level is one
// pass over the particles: the host decides per frontier node whether it is a
// leaf (bin <= N_T, or level >= max_depth, and no children yet), descends into
// existing children, or splits (face_tree.cpp:40-47); new children get their
// geometry on the device (k_make_children: bit-exact midpoints and Cramer
// constants); k_descend moves each particle into the first child whose
// barycentric min-score is >= -1e-10, else the best-scoring child
// (face_tree.cpp:50-69), and counts bins with integer atomics. Bins end up as
// contiguous ranges of a tree-order permutation (depth-first, children in
// order; particles ascending by id inside each leaf) from one stable radix
// sort keyed by the leaf's offset.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "internal.cuh"

namespace ssum {

namespace {

enum : int { kActLeaf = 0, kActDescend = 1 };

__device__ __forceinline__ d3 load3(const double* p) { return {p[0], p[1], p[2]}; }

// Root-face assignment: first of the 20 roots with triangle_contains
// (face_tree.cpp:77-85). GeometryError when none contains the particle.
__global__ void k_bin_roots(const double* __restrict__ xyz, int64_t n, const double* __restrict__ tri,
                            const double* __restrict__ cramer, int* __restrict__ cur, int* __restrict__ cnt,
                            int* __restrict__ flags) {
  __shared__ double st[20 * 9];
  __shared__ double skr[20 * 12];
  __shared__ int scount[20];
  for (int k = threadIdx.x; k < 180; k += blockDim.x) st[k] = tri[k];
  for (int k = threadIdx.x; k < 240; k += blockDim.x) skr[k] = cramer[k];
  if (threadIdx.x < 20) scount[threadIdx.x] = 0;
  __syncthreads();
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    const d3 p = load3(xyz + 3 * i);
    int found = -1;
    for (int f = 0; f < 20; ++f) {
      const d3 v1 = load3(st + 9 * f), v2 = load3(st + 9 * f + 3), v3 = load3(st + 9 * f + 6);
      const double* k = skr + 12 * f;
      int in = contains_screen(v1, v2, v3, d3{k[0], k[1], k[2]}, k[3], k[10], p);
      if (in < 0) in = contains_rn(v1, v2, v3, p);
      if (in) {
        found = f;
        break;
      }
    }
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
  k[11] = 0.0;
  if (bad) atomicOr(flags, kFlagGeometry);
}

// ensure_children (face_tree.cpp:18-37): midpoints renormalised, children
// {v1,m12,m31}, {m12,v2,m23}, {m31,m23,v3}, {m12,m23,m31}; links written here.
__global__ void k_make_children(const int2* __restrict__ splits, int ns, double* tri, double* center,
                                double* radius, double* cramer, int* level, int* parent, int* child_base,
                                int* flags) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= ns) return;
  const int par = splits[k].x, base = splits[k].y;
  const double* t = tri + 9 * par;
  const d3 v1 = load3(t), v2 = load3(t + 3), v3 = load3(t + 6);
  int bad = 0;
  const d3 m12 = unit_rn(add3(v1, v2), &bad);
  const d3 m23 = unit_rn(add3(v2, v3), &bad);
  const d3 m31 = unit_rn(add3(v3, v1), &bad);
  if (bad) atomicOr(flags, kFlagGeometry);
  write_node(tri, center, radius, cramer, base + 0, v1, m12, m31, flags);
  write_node(tri, center, radius, cramer, base + 1, m12, v2, m23, flags);
  write_node(tri, center, radius, cramer, base + 2, m31, m23, v3, flags);
  write_node(tri, center, radius, cramer, base + 3, m12, m23, m31, flags);
  const int lv = level[par] + 1;
  for (int q = 0; q < 4; ++q) {
    level[base + q] = lv;
    parent[base + q] = par;
    child_base[base + q] = -1;
  }
  child_base[par] = base;
}

__global__ void k_set_actions(const int2* __restrict__ fa, int nf, unsigned char* act) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nf) act[fa[k].x] = static_cast<unsigned char>(fa[k].y);
}

// One level of distribute (face_tree.cpp:39-71) for every still-active particle.
__global__ void k_descend(const double* __restrict__ xyz, int64_t n, int* __restrict__ cur,
                          int* __restrict__ leaf_of, const unsigned char* __restrict__ act,
                          const int* __restrict__ child_base, const double* __restrict__ tri,
                          const double* __restrict__ cramer, int* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int node = cur[i];
  if (node < 0) return;
  if (act[node] == kActLeaf) {
    leaf_of[i] = node;
    cur[i] = -1;
    return;
  }
  const d3 p = load3(xyz + 3 * i);
  const int cb = child_base[node];
  int placed = -1;
  for (int c = cb; c < cb + 4 && placed < 0; ++c) {  // first containing child wins (face_tree.cpp:56-61)
    const double* t = tri + 9 * c;
    const double* k = cramer + 12 * c;
    const d3 va = load3(t), vb = load3(t + 3), vc = load3(t + 6), bc{k[0], k[1], k[2]};
    int in = contains_screen(va, vb, vc, bc, k[3], k[10], p);
    if (in < 0) in = min_score_rn(va, vb, vc, bc, k[3], p) >= -1e-10;
    if (in) placed = c;
  }
  int best = cb;
  if (placed < 0) {  // no child contains p: least-negative exact score (face_tree.cpp:62-69)
    double best_s = -1e300;
    for (int c = cb; c < cb + 4; ++c) {
      const double* t = tri + 9 * c;
      const double* k = cramer + 12 * c;
      const double s = min_score_rn(load3(t), load3(t + 3), load3(t + 6), d3{k[0], k[1], k[2]}, k[3], p);
      if (s > best_s) {
        best_s = s;
        best = c;
      }
    }
  }
  if (placed < 0) placed = best;
  cur[i] = placed;
  // warp-aggregated bin count: one atomic per distinct child in the warp
  const unsigned peers = __match_any_sync(__activemask(), placed);
  if ((threadIdx.x & 31) == __ffs(peers) - 1) atomicAdd(&cnt[placed], __popc(peers));
}

__global__ void k_gather_counts(const int* __restrict__ ids, int m, const int* __restrict__ cnt, int* out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < m) out[k] = cnt[ids[k]];
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

}  // namespace

static void grow_nodes(Ctx& c, int need) {
  NodeTable& t = c.nodes;
  t.tri.ensure(size_t(need) * 9, true, c.stream);
  t.center.ensure(size_t(need) * 3, true, c.stream);
  t.radius.ensure(size_t(need), true, c.stream);
  t.cramer.ensure(size_t(need) * 12, true, c.stream);
  t.child_base.ensure(size_t(need), true, c.stream);
  t.level.ensure(size_t(need), true, c.stream);
  t.parent.ensure(size_t(need), true, c.stream);
  c.bins.cnt.ensure(size_t(need), true, c.stream);
  c.bins.act.ensure(size_t(need), true, c.stream);
}

// The 20 roots, built with the host libm so their vertices are bit-identical
// to the reference's (IcosaMesh::base_icosahedron, icosa_mesh.cpp:10-35;
// latlon_to_unit, geometry.cpp:41-44; FaceTree ctor, face_tree.cpp:9-16).
void tree_init_roots(Ctx& c) {
  HostTree& h = c.host;
  h = HostTree{};
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
      const double kk[12] = {bc.x, bc.y, bc.z, det, n2.x, n2.y, n2.z, n3.x, n3.y, n3.z, 1.0 / det, 0};
      std::copy(kk, kk + 12, cramer.begin() + 12 * f);
    }
  }
  if (bad) throw Error(SSUM_GEOMETRY, "degenerate base icosahedron");
  c.nodes.count = 20;
  grow_nodes(c, 1024);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.tri.p, tri.data(), tri.size() * 8, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.center.p, center.data(), center.size() * 8, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.radius.p, radius.data(), radius.size() * 8, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.cramer.p, cramer.data(), cramer.size() * 8, cudaMemcpyHostToDevice, c.stream));
  h.level.assign(20, 0);
  h.parent.assign(20, -1);
  h.child_base.assign(20, -1);
  h.created_call.assign(20, 0);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.level.p, h.level.data(), 80, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.parent.p, h.parent.data(), 80, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.nodes.child_base.p, h.child_base.data(), 80, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

void tree_bin(Ctx& c, const double* d_xyz, int64_t n, int nt, int max_depth) {
  HostTree& h = c.host;
  Binned& B = c.bins;
  c.call_index++;
  B.n = n;
  B.frontier.clear();
  B.leaves.clear();
  B.max_level = 0;
  const int bs = 256;

  // Fresh per-call counts; node geometry persists (face_tree.cpp:75).
  SSUM_CUDA_CHECK(cudaMemsetAsync(B.cnt.p, 0, B.cnt.cap * sizeof(int), c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(c.d_flags.p, 0, sizeof(int), c.stream));
  h.cnt.assign(h.level.size(), 0);
  h.off.assign(h.level.size(), 0);
  if (n == 0) return;
  B.cur.ensure(size_t(n));
  B.leaf_of.ensure(size_t(n));

  k_bin_roots<<<grid_for(n, bs), bs, 0, c.stream>>>(d_xyz, n, c.nodes.tri.p, c.nodes.cramer.p, B.cur.p, B.cnt.p,
                                                     c.d_flags.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  check_flags(c, "bin_particles: particle contained in no root face");
  trace().mark("bin.roots");

  std::vector<int> cand(20);
  for (int f = 0; f < 20; ++f) cand[f] = f;
  std::vector<int> counts;
  std::vector<int2> fa, splits;
  while (!cand.empty()) {
    const int m = static_cast<int>(cand.size());
    B.d_ids.ensure(size_t(m));
    B.d_cnt.ensure(size_t(m));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(B.d_ids.p, cand.data(), size_t(m) * 4, cudaMemcpyHostToDevice, c.stream));
    k_gather_counts<<<grid_for(m, bs), bs, 0, c.stream>>>(B.d_ids.p, m, B.cnt.p, B.d_cnt.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    counts.resize(size_t(m));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(counts.data(), B.d_cnt.p, size_t(m) * 4, cudaMemcpyDeviceToHost, c.stream));
    check_flags(c, "bin_particles: degenerate child triangle");  // synchronises
    trace().mark("bin.lvl_counts");

    std::vector<int> front;
    front.reserve(size_t(m));
    fa.clear();
    splits.clear();
    for (int k = 0; k < m; ++k) {
      const int id = cand[k];
      h.cnt[id] = counts[k];
      if (counts[k] == 0) continue;  // distribute returns on an empty bin (face_tree.cpp:40)
      front.push_back(id);
      int a = kActDescend;
      if (h.child_base[id] < 0) {
        if (counts[k] <= nt || h.level[id] >= max_depth) {
          a = kActLeaf;  // face_tree.cpp:42-45
        } else {
          const int base = static_cast<int>(h.level.size());
          h.child_base[id] = base;
          for (int q = 0; q < 4; ++q) {
            h.level.push_back(h.level[id] + 1);
            h.parent.push_back(id);
            h.child_base.push_back(-1);
            h.created_call.push_back(c.call_index);
            h.cnt.push_back(0);
            h.off.push_back(0);
          }
          splits.push_back(int2{id, base});
        }
      }
      if (a == kActLeaf) B.leaves.push_back(id);
      fa.push_back(int2{id, a});
    }
    trace().mark("bin.lvl_host");
    if (front.empty()) break;
    B.frontier.push_back(std::move(front));

    const int total = static_cast<int>(h.level.size());
    if (total > c.nodes.count) {
      const int first = c.nodes.count;
      grow_nodes(c, total);
      SSUM_CUDA_CHECK(cudaMemsetAsync(B.cnt.p + first, 0, size_t(total - first) * 4, c.stream));
      c.nodes.count = total;
    }
    B.d_pairs.ensure(splits.size() + fa.size());
    int2* d_splits = B.d_pairs.p;
    int2* d_fa = B.d_pairs.p + splits.size();
    if (!splits.empty()) {
      SSUM_CUDA_CHECK(cudaMemcpyAsync(d_splits, splits.data(), splits.size() * sizeof(int2), cudaMemcpyHostToDevice, c.stream));
      k_make_children<<<grid_for(int64_t(splits.size()), 128), 128, 0, c.stream>>>(
          d_splits, static_cast<int>(splits.size()), c.nodes.tri.p, c.nodes.center.p, c.nodes.radius.p,
          c.nodes.cramer.p, c.nodes.level.p, c.nodes.parent.p, c.nodes.child_base.p, c.d_flags.p);
      SSUM_LAUNCH_CHECK();
      c.launches++;
    }
    SSUM_CUDA_CHECK(cudaMemcpyAsync(d_fa, fa.data(), fa.size() * sizeof(int2), cudaMemcpyHostToDevice, c.stream));
    k_set_actions<<<grid_for(int64_t(fa.size()), bs), bs, 0, c.stream>>>(d_fa, static_cast<int>(fa.size()), B.act.p);
    SSUM_LAUNCH_CHECK();
    k_descend<<<grid_for(n, bs), bs, 0, c.stream>>>(d_xyz, n, B.cur.p, B.leaf_of.p, B.act.p, c.nodes.child_base.p,
                                                     c.nodes.tri.p, c.nodes.cramer.p, B.cnt.p);
    SSUM_LAUNCH_CHECK();
    c.launches += 2;

    trace().mark("bin.lvl_launch");
    cand.clear();
    for (const int2& p : fa)
      if (p.y == kActDescend)
        for (int q = 0; q < 4; ++q) cand.push_back(h.child_base[p.x] + q);
  }
  B.max_level = static_cast<int>(B.frontier.size()) - 1;

  // Bin offsets in depth-first order (roots in face order, children in
  // order) and the leaves in that order — one preorder walk over the
  // non-empty nodes. Leaf tiles then cover the tree-order particle array
  // left to right, which the target partition relies on.
  {
    std::vector<char> is_leaf(h.level.size(), 0);
    for (const int id : B.leaves) is_leaf[size_t(id)] = 1;
    B.leaves.clear();
    std::vector<int> stack;
    stack.reserve(256);
    for (int f = 19; f >= 0; --f) stack.push_back(f);
    int run = 0;
    while (!stack.empty()) {
      const int id = stack.back();
      stack.pop_back();
      if (h.cnt[size_t(id)] == 0) continue;
      h.off[size_t(id)] = run;
      if (is_leaf[size_t(id)]) {
        B.leaves.push_back(id);
        run += h.cnt[size_t(id)];
      } else {
        const int cb = h.child_base[size_t(id)];
        for (int q = 3; q >= 0; --q) stack.push_back(cb + q);
      }
    }
  }
  B.off.ensure(size_t(c.nodes.count));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(B.off.p, h.off.data(), size_t(c.nodes.count) * 4, cudaMemcpyHostToDevice, c.stream));
  B.d_leaves.ensure(std::max<size_t>(B.leaves.size(), 1));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(B.d_leaves.p, B.leaves.data(), B.leaves.size() * 4, cudaMemcpyHostToDevice, c.stream));

  // Permutation: stable sort of particle ids by their leaf's offset.
  trace().mark("bin.offsets");
  B.sort_keys.ensure(size_t(n));
  B.sort_keys2.ensure(size_t(n));
  B.sort_vals.ensure(size_t(n));
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
}

}  // namespace ssum
