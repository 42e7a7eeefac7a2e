// Evaluation passes of treecode_sum (treecode.cpp:326-404) on the device.
//
//   k_gather       particles into tree order, packed (x, y, z, q) — the
//                  unified point array's first N entries
//   k_proxy        Phase 1: lattice proxy points of every proxy node
//                  (proxy_points, sbb.cpp:46-66) — entries N + slot*p + m
//   k_up_partial   Phase 2: w_k = sum_j B_k(beta_s(x_j)) q_j over bin chunks
//   k_up_final     (compute_proxy_weights, treecode.cpp:79-91), then
//                  w_hat = V^-T w (solve_transposed, sbb.cpp:110-115) into
//                  the proxy entries' 4th component
//   k_tiles<fit>   Phase 3: CP/CC proxy potentials phi per fit node and the
//                  fit C = V^-1 phi (treecode.cpp:341-358, sbb.cpp:103-108)
//   k_tiles<leaf>  Phase 4 direct part: PP pairs and PC proxy pairs per leaf
//                  tile (treecode.cpp:386-396); also the direct sum
//   k_finish       Phase 4 downward part (add_fitted_value over the path,
//                  treecode.cpp:143-155,397-401), cross product, prefactor,
//                  scatter back to the caller's order (:402)
//
// Barycentrics use the per-node Cramer constants: beta_k = (x . n_k) / sum,
// with n_1 = v2 x v3, n_2 = v3 x v1, n_3 = v1 x v2 — algebraically the
// reference's spherical_barycentric (geometry.cpp:59-69: det cancels).
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "kernels.cuh"

namespace ssum {

namespace {

constexpr double kInv4Pi = 0.07957747154594767;  // 1 / (4 pi)

template <int DEG>
struct Sbb {
  static constexpr int P = (DEG + 1) * (DEG + 2) / 2;
};

__device__ __forceinline__ void bary(const double* k, double x0, double x1, double x2, double& b1, double& b2,
                                     double& b3) {
  const double r1 = fma(x2, k[2], fma(x1, k[1], x0 * k[0]));
  const double r2 = fma(x2, k[6], fma(x1, k[5], x0 * k[4]));
  const double r3 = fma(x2, k[9], fma(x1, k[8], x0 * k[7]));
  const double inv = 1.0 / ((r1 + r2) + r3);
  b1 = r1 * inv;
  b2 = r2 * inv;
  b3 = r3 * inv;
}

template <int DEG>
__device__ __forceinline__ void powers(double b1, double b2, double b3, double* p1, double* p2, double* p3) {
  p1[0] = p2[0] = p3[0] = 1.0;
#pragma unroll
  for (int n = 1; n <= DEG; ++n) {
    p1[n] = p1[n - 1] * b1;
    p2[n] = p2[n - 1] * b2;
    p3[n] = p3[n - 1] * b3;
  }
}

__global__ void k_gather(const double* __restrict__ xyz, const double* __restrict__ q, const int* __restrict__ perm,
                         int64_t n, double4* __restrict__ pts) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int i = perm ? perm[k] : static_cast<int>(k);
  pts[k] = make_double4(xyz[3 * i], xyz[3 * i + 1], xyz[3 * i + 2], q[i]);
}

// proxy_points (sbb.cpp:46-66): normalise(b1 v1 + b2 v2 + b3 v3), b = (i,j,k)/d
// in the SBB index order (sbb.cpp:19-23: k ascending, then j ascending).
__global__ void k_proxy(const int* __restrict__ slot_node, int nslots, int degree, const double* __restrict__ tri,
                        int64_t N, double4* __restrict__ pts) {
  const int P = (degree + 1) * (degree + 2) / 2;
  const int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (g >= int64_t(nslots) * P) return;
  const int slot = static_cast<int>(g / P), m = static_cast<int>(g % P);
  int kk = 0, jj = m;
  while (jj > degree - kk) {
    jj -= degree - kk + 1;
    ++kk;
  }
  const int ii = degree - kk - jj;
  const double d = static_cast<double>(degree);
  const double b1 = __ddiv_rn(static_cast<double>(ii), d), b2 = __ddiv_rn(static_cast<double>(jj), d),
               b3 = __ddiv_rn(static_cast<double>(kk), d);
  const double* t = tri + 9 * slot_node[slot];
  d3 v;
  v.x = add_rn(add_rn(mul_rn(t[0], b1), mul_rn(t[3], b2)), mul_rn(t[6], b3));
  v.y = add_rn(add_rn(mul_rn(t[1], b1), mul_rn(t[4], b2)), mul_rn(t[7], b3));
  v.z = add_rn(add_rn(mul_rn(t[2], b1), mul_rn(t[5], b2)), mul_rn(t[8], b3));
  int bad = 0;
  const d3 u = unit_rn(v, &bad);
  pts[N + g] = make_double4(u.x, u.y, u.z, 0.0);
}

// Partial proxy weights of one (weight node, particle chunk) per warp: each
// lane accumulates the P basis sums over its stride of the chunk, then the
// warp reduces them through a shared-memory transpose, 32 basis functions at
// a time (lane j sums row j: 32 loads + adds instead of 5 shuffle rounds per
// function).
constexpr int kUpWarps = 4;
template <int DEG>
#ifndef SSUM_UP_MINB
#define SSUM_UP_MINB 3  // measured: 3 resident blocks beat 1 (156 regs) and 4 (spills)
#endif
__global__ void __launch_bounds__(32 * kUpWarps, SSUM_UP_MINB) k_up_partial(const int4* __restrict__ chunks,
                                                             const int* __restrict__ nchunks,
                                                             const double4* __restrict__ pts,
                                                             const double* __restrict__ cramer,
                                                             double* __restrict__ wpart) {
  constexpr int P = Sbb<DEG>::P;
  __shared__ double tr[kUpWarps][32][33];
  const int lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  // grid-stride over the chunks: a small grid leaves room on every SM for
  // the latency-bound list kernels running beside the upward pass
  const int nch = *nchunks;
  for (int chunk = blockIdx.x * kUpWarps + wp; chunk < nch; chunk += gridDim.x * kUpWarps) {  // warp-uniform
  const int4 ch = chunks[chunk];  // node, begin, count
  const double* k = cramer + 12 * ch.x;
  double kc[10];
#pragma unroll
  for (int z = 0; z < 10; ++z) kc[z] = k[z];
  double w[P];
#pragma unroll
  for (int m = 0; m < P; ++m) w[m] = 0.0;
  const int end = ch.y + ch.z;
  double4 pn = ch.y + lane < end ? pts[ch.y + lane] : make_double4(0.0, 0.0, 0.0, 0.0);
  for (int i = ch.y + lane; i < end; i += 32) {
    const double4 p = pn;  // next particle's load in flight while this one is summed
    if (i + 32 < end) pn = pts[i + 32];
    double b1, b2, b3;
    bary(kc, p.x, p.y, p.z, b1, b2, b3);
    double p1[DEG + 1], p2[DEG + 1], p3[DEG + 1];
    powers<DEG>(b1, b2, b3, p1, p2, p3);
    int m = 0;
#pragma unroll
    for (int kk = 0; kk <= DEG; ++kk) {
      const double t3 = p3[kk] * p.w;
#pragma unroll
      for (int jj = 0; jj <= DEG - kk; ++jj, ++m) w[m] = fma(p1[DEG - kk - jj] * p2[jj], t3, w[m]);
    }
  }
  double (*t)[33] = tr[wp];
#pragma unroll
  for (int g = 0; g < P; g += 32) {
#pragma unroll
    for (int j = 0; j < 32; ++j)
      if (g + j < P) t[j][lane] = w[g + j];
    __syncwarp();
    if (g + lane < P) {
      double s = 0.0;
#pragma unroll 8
      for (int l = 0; l < 32; ++l) s += t[lane][l];
      wpart[size_t(chunk) * P + g + lane] = s;
    }
    __syncwarp();
  }
  }
}

#ifndef SSUM_UP_CHUNK
#define SSUM_UP_CHUNK 1024  // measured: 1024 = 2048 < 512 < 256 < 128 (0.31 vs 0.39 ms at C4 for 256)
#endif
constexpr int kUpChunk = SSUM_UP_CHUNK;  // particles per upward chunk (one warp each)

// d_nw (optional): the device-side weight-node count (<= the host bound nw,
// which sizes the grids); entries past it contribute nothing.
__global__ void k_up_nchunks(const int* __restrict__ weight_nodes, int nw, const int* __restrict__ cnt,
                             int* __restrict__ nch, const int* __restrict__ d_nw) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  const int nwe = d_nw ? min(*d_nw, nw) : nw;
  if (w < nwe) nch[w] = (cnt[weight_nodes[w]] + kUpChunk - 1) / kUpChunk;
  else if (w <= nw) nch[w] = 0;
}

__global__ void k_up_fill(const int* __restrict__ weight_nodes, int nw, const int* __restrict__ off,
                          const int* __restrict__ cnt, const int* __restrict__ chunk_off, int4* __restrict__ chunks,
                          int2* __restrict__ crange, const int* __restrict__ d_nw) {
  const int w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= (d_nw ? min(*d_nw, nw) : nw)) return;
  const int id = weight_nodes[w], o = off[id], cn = cnt[id];
  int k = chunk_off[w];
  crange[w] = make_int2(k, chunk_off[w + 1]);
  for (int b = 0; b < cn; b += kUpChunk, ++k) chunks[k] = make_int4(id, o + b, min(kUpChunk, cn - b), 0);
}

// w = sum of the node's chunk partials (in chunk order); w_hat = V^-T w.
// raw != nullptr: store w itself (compute_proxy_weights) and stop.
__global__ void k_up_final(const int* __restrict__ weight_nodes, int nw, const int2* __restrict__ chunk_range,
                           const double* __restrict__ wpart, const double* __restrict__ vinv, int P,
                           const int* __restrict__ pslot, int64_t N, double4* __restrict__ pts,
                           double* __restrict__ raw = nullptr, const int* __restrict__ d_nw = nullptr) {
  extern __shared__ double ws[];
  const int w = blockIdx.x;
  if (w >= (d_nw ? min(*d_nw, nw) : nw)) return;
  const int2 cr = chunk_range[w];
  for (int m = threadIdx.x; m < P; m += blockDim.x) {
    double s = 0.0;
    for (int c = cr.x; c < cr.y; ++c) s += wpart[size_t(c) * P + m];
    ws[m] = s;
    if (raw) raw[size_t(w) * P + m] = s;
  }
  if (raw) return;
  __syncthreads();
  const int64_t base = N + int64_t(pslot[weight_nodes[w]]) * P;
  for (int kk = threadIdx.x; kk < P; kk += blockDim.x) {
    double s = 0.0;
    for (int m = 0; m < P; ++m) s = fma(vinv[size_t(m) * P + kk], ws[m], s);  // (V^-1)^T row kk
    pts[base + kk].w = s;
  }
}

// Phase 4 downward part + finish.
template <int KER, int DEG>
__global__ void k_finish(int64_t p0, int64_t p1, const double4* __restrict__ pts, const double* __restrict__ S,
                         const int* __restrict__ pos_leaf, const int* __restrict__ parent,
                         const int* __restrict__ pslot, const unsigned char* __restrict__ is_fit,
                         const double* __restrict__ cramer, const double* __restrict__ coeff,
                         const int* __restrict__ perm, double* __restrict__ out, const int* __restrict__ inv,
                         int64_t i0, int64_t i1) {
  constexpr int D = KDim<KER>::D;
  constexpr int P = Sbb<DEG>::P;
  // thread -> tree position k (and original id o): in tree order over
  // [p0, p1), or, with inv, in original order over [i0, i1) (one piece of
  // the host result), skipping positions outside this part
  int64_t k, o;
  if (inv) {
    o = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (o >= i1) return;
    k = inv[o];
    if (k < p0 || k >= p1) return;
  } else {
    k = p0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (k >= p1) return;
    o = perm[k];
  }
  const double4 x = pts[k];
  double val[D];
#pragma unroll
  for (int d = 0; d < D; ++d) val[d] = 0.0;
  for (int a = pos_leaf[k]; a >= 0; a = parent[a]) {
    if (!is_fit[a]) continue;
    const double* c = coeff + size_t(pslot[a]) * D * P;
    double b1, b2, b3;
    bary(cramer + 12 * a, x.x, x.y, x.z, b1, b2, b3);
    double p1[DEG + 1], p2[DEG + 1], p3[DEG + 1];
    powers<DEG>(b1, b2, b3, p1, p2, p3);
    int m = 0;
#pragma unroll
    for (int kk = 0; kk <= DEG; ++kk) {
#pragma unroll
      for (int jj = 0; jj <= DEG - kk; ++jj, ++m) {
        const double B = p1[DEG - kk - jj] * p2[jj] * p3[kk];
#pragma unroll
        for (int d = 0; d < D; ++d) val[d] = fma(c[d * P + m], B, val[d]);
      }
    }
  }
  if constexpr (KER == kBS) {
    const double s0 = S[3 * k], s1 = S[3 * k + 1], s2 = S[3 * k + 2];
    const double pref = -kInv4Pi;  // BiotSavartKernel::prefactor (kernels.hpp:54)
    out[3 * size_t(o)] = pref * ((x.y * s2 - x.z * s1) + val[0]);
    out[3 * size_t(o) + 1] = pref * ((x.z * s0 - x.x * s2) + val[1]);
    out[3 * size_t(o) + 2] = pref * ((x.x * s1 - x.y * s0) + val[2]);
  } else {
    out[o] = -kInv4Pi * S[k] + val[0];
  }
}

// Phase 4 downward part + finish over tree positions [p0, p1) (one thread
// each, consecutive positions share their ancestors): the same arithmetic as
// k_finish, but each fit ancestor's D x P coefficients and Cramer constants
// are staged once per warp in shared memory and read back as warp-uniform
// (broadcast) shared loads — k_finish's per-lane global loads of them kept
// the L1 data pipe ~88% busy. Lanes walk their ancestor chains in lockstep;
// at each step the warp stages every distinct fit ancestor among its lanes in
// turn (normally one, two where the warp straddles a node boundary).
constexpr int kFinWarps = 4;
template <int KER, int DEG>
__global__ void __launch_bounds__(32 * kFinWarps) k_finish_tree(
    int64_t p0, int64_t p1, const double4* __restrict__ pts, const double* __restrict__ S,
    const int* __restrict__ pos_leaf, const int* __restrict__ parent, const int* __restrict__ pslot,
    const unsigned char* __restrict__ is_fit, const double* __restrict__ cramer, const double* __restrict__ coeff,
    const int* __restrict__ perm, double* __restrict__ out, int64_t obase) {
  constexpr int D = KDim<KER>::D;
  constexpr int P = Sbb<DEG>::P;
  // staged coefficients, packed (c_0, c_1, c_2) per basis function: a pair
  // of basis functions (m even, m + 1) is three LDS.128 (1.5 per function
  // instead of an LDS.128 + LDS.64 each — the kernel is LSU-bound)
  constexpr int DP = D == 3 ? 3 : 1;
  constexpr int kRow = (P * DP + 1) & ~1;  // even: every warp's row starts 16-byte aligned
  __shared__ __align__(16) double cs[kFinWarps][kRow];
  __shared__ __align__(16) double cr[kFinWarps][12];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu;
  const int64_t k = p0 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  const bool valid = k < p1;
  const double4 x = valid ? pts[k] : make_double4(0.0, 0.0, 0.0, 0.0);
  double val[D];
#pragma unroll
  for (int d = 0; d < D; ++d) val[d] = 0.0;
  int a = valid ? pos_leaf[k] : -1;
  while (__any_sync(full, a >= 0)) {
    const bool fit = a >= 0 && is_fit[a];
    unsigned pend = __ballot_sync(full, fit);
    while (pend) {
      const int an = __shfl_sync(full, a, __ffs(pend) - 1);
      const bool mine = fit && a == an;
      SSUM_DCHECK(pslot[an] >= 0);
      const double* c = coeff + size_t(pslot[an]) * D * P;
      // every load of the staging issued before its first store (one
      // latency per staged node, not one per 32 coefficients)
      constexpr int kIt = (D * P + 31) / 32;
      double tmp[kIt];
#pragma unroll
      for (int j = 0; j < kIt; ++j) tmp[j] = lane + 32 * j < D * P ? c[lane + 32 * j] : 0.0;
      const double crv = lane < 12 ? cramer[12 * an + lane] : 0.0;
#pragma unroll
      for (int j = 0; j < kIt; ++j) {
        const int i = lane + 32 * j;
        if (i < D * P) cs[w][(i % P) * DP + i / P] = tmp[j];
      }
      if (lane < 12) cr[w][lane] = crv;
      __syncwarp();
      if (mine) {
        double b1, b2, b3;
        bary(cr[w], x.x, x.y, x.z, b1, b2, b3);
        double q1[DEG + 1], q2[DEG + 1], q3[DEG + 1];
        powers<DEG>(b1, b2, b3, q1, q2, q3);
        int m = 0;
        double n0 = 0.0, n1 = 0.0, n2 = 0.0;  // basis m + 1's coefficients, loaded with m's
#pragma unroll
        for (int kk = 0; kk <= DEG; ++kk) {
#pragma unroll
          for (int jj = 0; jj <= DEG - kk; ++jj, ++m) {
            const double B = q1[DEG - kk - jj] * q2[jj] * q3[kk];
            if constexpr (D == 3) {
              double c0, c1, c2;
              if ((m & 1) == 0) {
                const double2* r = reinterpret_cast<const double2*>(&cs[w][m * 3]);
                const double2 a = r[0], b = r[1];
                c0 = a.x, c1 = a.y, c2 = b.x;
                if (m + 1 < P) {
                  const double2 e = r[2];
                  n0 = b.y, n1 = e.x, n2 = e.y;
                }
              } else {
                c0 = n0, c1 = n1, c2 = n2;
              }
              val[0] = fma(c0, B, val[0]);
              val[1] = fma(c1, B, val[1]);
              val[2] = fma(c2, B, val[2]);
            } else {
              val[0] = fma(cs[w][m], B, val[0]);
            }
          }
        }
      }
      __syncwarp();
      pend &= ~__ballot_sync(full, mine);
    }
    a = a >= 0 ? parent[a] : -1;
  }
  if (!valid) return;
  // no perm: tree order from obase (in place over S, obase 0, is safe: own row only)
  const int64_t o = perm ? perm[k] : k - obase;
  if constexpr (KER == kBS) {
    const double s0 = S[3 * k], s1 = S[3 * k + 1], s2 = S[3 * k + 2];
    const double pref = -kInv4Pi;  // BiotSavartKernel::prefactor (kernels.hpp:54)
    out[3 * size_t(o)] = pref * ((x.y * s2 - x.z * s1) + val[0]);
    out[3 * size_t(o) + 1] = pref * ((x.z * s0 - x.x * s2) + val[1]);
    out[3 * size_t(o) + 2] = pref * ((x.x * s1 - x.y * s0) + val[2]);
  } else {
    out[o] = -kInv4Pi * S[k] + val[0];
  }
}

// Caller-order rows [i0, i1) of a tree-order result (host pieces after a
// tree-order finish); rows outside this part's positions [p0, p1) are left
// as they are, like k_finish leaves them.
__global__ void k_gather_rows(const double* __restrict__ R, const int* __restrict__ inv, int64_t i0, int64_t i1,
                              int64_t p0, int64_t p1, int D, double* __restrict__ out) {
  const int64_t o = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (o >= i1) return;
  const int64_t k = inv[o];
  if (k < p0 || k >= p1) return;
  for (int d = 0; d < D; ++d) out[o * D + d] = R[k * D + d];
}

__global__ void k_inv_perm(const int* __restrict__ perm, int64_t n, int* __restrict__ inv) {
  const int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < n) inv[perm[k]] = static_cast<int>(k);
}

// inv: finish caller-order rows [i0, i1) (per-lane k_finish); otherwise the
// part's tree positions with k_finish_tree, written to d_out in caller order
// (perm) or, with tree_order, in tree order: position k to row k - obase.
template <int KER>
void launch_finish(Ctx& c, int degree, double* d_out, const int* inv = nullptr, int64_t i0 = 0, int64_t i1 = 0,
                   bool tree_order = false, int64_t obase = 0) {
  Lists& L = c.lists;
  Binned& B = c.bins;
  const int bs = 128;
  const int64_t n = inv ? i1 - i0 : L.p1 - L.p0;
  if (n <= 0) return;
#define SSUM_FINISH_CASE(DG)                                                                                   \
  case DG:                                                                                                    \
    if (inv)                                                                                                  \
      k_finish<KER, DG><<<grid_for(n, bs), bs, 0, c.stream>>>(L.p0, L.p1, c.pts.p, c.S.p, B.pos_leaf.p,        \
                                                               c.nodes.parent.p, L.pslot.p, L.is_fit.p,       \
                                                               c.nodes.cramer.p, c.coeff.p, B.perm.p, d_out,  \
                                                               inv, i0, i1);                                  \
    else                                                                                                      \
      k_finish_tree<KER, DG><<<grid_for(n, 32 * kFinWarps), 32 * kFinWarps, 0, c.stream>>>(                   \
          L.p0, L.p1, c.pts.p, c.S.p, B.pos_leaf.p, c.nodes.parent.p, L.pslot.p, L.is_fit.p, c.nodes.cramer.p, \
          c.coeff.p, tree_order ? nullptr : B.perm.p, d_out, obase);                                          \
    break;
  switch (degree) {
    SSUM_FINISH_CASE(1) SSUM_FINISH_CASE(2) SSUM_FINISH_CASE(3) SSUM_FINISH_CASE(4) SSUM_FINISH_CASE(5)
    SSUM_FINISH_CASE(6) SSUM_FINISH_CASE(7) SSUM_FINISH_CASE(8) SSUM_FINISH_CASE(9) SSUM_FINISH_CASE(10)
    SSUM_FINISH_CASE(11) SSUM_FINISH_CASE(12) SSUM_FINISH_CASE(13) SSUM_FINISH_CASE(14) SSUM_FINISH_CASE(15)
    SSUM_FINISH_CASE(16) SSUM_FINISH_CASE(17) SSUM_FINISH_CASE(18) SSUM_FINISH_CASE(19) SSUM_FINISH_CASE(20)
    default:
      throw Error(SSUM_CONFIG, "degree out of range");
  }
#undef SSUM_FINISH_CASE
  SSUM_LAUNCH_CHECK();
  c.launches++;
}

// nchunks: host upper bound (grid size); d_nchunks: the device-side count.
void launch_up_partial(Ctx& c, cudaStream_t stream, int degree, int nchunks, const int* d_nchunks) {
  unsigned grid = static_cast<unsigned>((nchunks + kUpWarps - 1) / kUpWarps);
  // at most SSUM_UP_GRID (default 3, its occupancy) blocks per SM, striding
  // over the chunks: one resident wave, no block-scheduling tail beside the
  // list kernels (C4: -40 us per evaluation); 0 = one block per 4 chunks
  static const int per_sm = [] {
    const char* v = std::getenv("SSUM_UP_GRID");
    return v ? std::atoi(v) : SSUM_UP_MINB;
  }();
  if (per_sm > 0) {
    int sms = 0;
    SSUM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device));
    grid = std::min<unsigned>(grid, static_cast<unsigned>(sms * per_sm));
  }
#define SSUM_UP_CASE(DG)                                                                                  \
  case DG:                                                                                                \
    k_up_partial<DG><<<grid, 32 * kUpWarps, 0, stream>>>(c.wchunks.p, d_nchunks, c.pts.p, c.nodes.cramer.p,   \
                                                           c.wpart.p);                                    \
    break;
  switch (degree) {
    SSUM_UP_CASE(1) SSUM_UP_CASE(2) SSUM_UP_CASE(3) SSUM_UP_CASE(4) SSUM_UP_CASE(5) SSUM_UP_CASE(6)
    SSUM_UP_CASE(7) SSUM_UP_CASE(8) SSUM_UP_CASE(9) SSUM_UP_CASE(10) SSUM_UP_CASE(11) SSUM_UP_CASE(12)
    SSUM_UP_CASE(13) SSUM_UP_CASE(14) SSUM_UP_CASE(15) SSUM_UP_CASE(16) SSUM_UP_CASE(17) SSUM_UP_CASE(18)
    SSUM_UP_CASE(19) SSUM_UP_CASE(20)
    default:
      throw Error(SSUM_CONFIG, "degree out of range");
  }
#undef SSUM_UP_CASE
  SSUM_LAUNCH_CHECK();
  c.launches++;
}

}  // namespace

// V[m][k] = B_k(b_m) on the lattice (sbb.cpp:80-85), LU with partial pivoting,
// explicit inverse, and the exact 1-norm reciprocal condition number
// (lattice_fit / ProxyFit, sbb.cpp:74-138; the reference's Eigen rcond() is
// an estimate of the same quantity). rcond = 0 for a singular matrix.
void lattice_inverse(int degree, std::vector<double>& inv, double& rcond) {
  const int P = (degree + 1) * (degree + 2) / 2;
  std::vector<int> I(static_cast<size_t>(P)), J(static_cast<size_t>(P)), K(static_cast<size_t>(P));
  {
    int m = 0;
    for (int k = 0; k <= degree; ++k)
      for (int j = 0; j <= degree - k; ++j, ++m) {
        I[m] = degree - k - j;
        J[m] = j;
        K[m] = k;
      }
  }
  const double d = static_cast<double>(degree);
  std::vector<double> V(size_t(P) * P), A;
  for (int r = 0; r < P; ++r) {
    const double b[3] = {I[r] / d, J[r] / d, K[r] / d};
    for (int col = 0; col < P; ++col) {
      double v = 1.0;
      for (int e = 0; e < I[col]; ++e) v *= b[0];
      double v2 = 1.0;
      for (int e = 0; e < J[col]; ++e) v2 *= b[1];
      double v3 = 1.0;
      for (int e = 0; e < K[col]; ++e) v3 *= b[2];
      V[size_t(r) * P + col] = v * v2 * v3;
    }
  }
  A = V;
  inv.assign(size_t(P) * P, 0.0);
  rcond = 0.0;
  std::vector<int> perm(static_cast<size_t>(P));
  for (int i = 0; i < P; ++i) perm[i] = i;
  for (int k = 0; k < P; ++k) {
    int piv = k;
    double best = std::fabs(A[size_t(k) * P + k]);
    for (int i = k + 1; i < P; ++i)
      if (std::fabs(A[size_t(i) * P + k]) > best) {
        best = std::fabs(A[size_t(i) * P + k]);
        piv = i;
      }
    if (best == 0.0) return;  // singular
    if (piv != k) {
      for (int j = 0; j < P; ++j) std::swap(A[size_t(k) * P + j], A[size_t(piv) * P + j]);
      std::swap(perm[k], perm[piv]);
    }
    for (int i = k + 1; i < P; ++i) {
      A[size_t(i) * P + k] /= A[size_t(k) * P + k];
      const double l = A[size_t(i) * P + k];
      for (int j = k + 1; j < P; ++j) A[size_t(i) * P + j] -= l * A[size_t(k) * P + j];
    }
  }
  std::vector<double> y(static_cast<size_t>(P));
  for (int col = 0; col < P; ++col) {
    for (int i = 0; i < P; ++i) y[i] = (perm[i] == col) ? 1.0 : 0.0;
    for (int i = 0; i < P; ++i)
      for (int k = 0; k < i; ++k) y[i] -= A[size_t(i) * P + k] * y[k];
    for (int i = P - 1; i >= 0; --i) {
      for (int k = i + 1; k < P; ++k) y[i] -= A[size_t(i) * P + k] * y[k];
      y[i] /= A[size_t(i) * P + i];
    }
    for (int i = 0; i < P; ++i) inv[size_t(i) * P + col] = y[i];
  }
  double an = 0.0, in = 0.0;
  for (int col = 0; col < P; ++col) {
    double s1 = 0.0, s2 = 0.0;
    for (int r = 0; r < P; ++r) {
      s1 += std::fabs(V[size_t(r) * P + col]);
      s2 += std::fabs(inv[size_t(r) * P + col]);
    }
    an = std::max(an, s1);
    in = std::max(in, s2);
  }
  rcond = (an > 0.0 && std::isfinite(in) && in > 0.0) ? 1.0 / (an * in) : 0.0;
}

// The far-pair log table (kernels.cuh log_tab): per bucket centre c_j a double
// r_j near 1 / c_j and L_j = RN(-log r_j). r_j is searched (Gal's accurate
// tables) outward from 1 / c_j in relative steps of 1e-9 for a double whose
// -log r_j lies within 2^-6 ulp of its double L_j (80-bit logl resolves
// ~2^-11 ulp). Steps of one ulp would not do: c_j has ~11 significant bits,
// so near 1 an ulp of r moves -log r by an integer number of L's ulps. ~35
// tries per bucket (tools/log_coeffs.py), at most 4096 (a 2e-6 relative move:
// inside the 2^-12 slack the polynomial range allows). c = 1: r = 1, L = 0.
void log_table(double2* tab) {
  for (int j = 0; j < kLogTabN; ++j) {
    const long double c = static_cast<long double>(log_tab_node(j));
    const long double r0 = 1.0L / c;
    double best_r = static_cast<double>(r0), best_e = 1.0;
    for (int i = 0; i < 4096 && best_e > 1.0 / 64; ++i) {
      const long double step = 1e-9L * static_cast<long double>((i & 1) ? -((i + 1) / 2) : i / 2);
      const double r = static_cast<double>(r0 * (1.0L + step));
      const long double L = -logl(static_cast<long double>(r));
      const double Ld = static_cast<double>(L);
      const long double u = Ld == 0.0 ? 1.0L : static_cast<long double>(std::nextafter(std::fabs(Ld), 1.0) - std::fabs(Ld));
      const double e = static_cast<double>(fabsl(L - static_cast<long double>(Ld)) / u);
      if (e < best_e) best_e = e, best_r = r;
    }
    tab[j] = make_double2(best_r, static_cast<double>(-logl(static_cast<long double>(best_r))));
  }
}

void ensure_log_table(Ctx& c) {
  if (c.logtab.p) return;
  std::vector<double2> h(static_cast<size_t>(kLogTabN));
  log_table(h.data());
  c.logtab.ensure(h.size());
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.logtab.p, h.data(), h.size() * sizeof(double2), cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

// ConditioningError when the reciprocal condition number is not > 1e-12
// (sbb.cpp:89-93); the value travels with the error (Ctx::last_rcond).
void ensure_vinv(Ctx& c, int degree) {
  if (c.vinv_degree == degree) return;
  std::vector<double> inv;
  double rcond = 0.0;
  lattice_inverse(degree, inv, rcond);
  if (!(rcond > 1e-12)) {
    c.last_rcond = rcond;
    throw Error(SSUM_CONDITIONING, "proxy Vandermonde too ill-conditioned (rcond " + std::to_string(rcond) + ")");
  }
  c.vinv.ensure(inv.size());
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.vinv.p, inv.data(), inv.size() * 8, cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  c.vinv_degree = degree;
}

// Particle gather, proxy points and the upward pass (Phases 1-2), on stream
// s: everything the tile kernels read from pts. tmp: cub scratch private to s.
// stages: bit 0 the gather + proxy points, bit 1 the upward pass.
void launch_prep(Ctx& c, cudaStream_t s, DBuf<unsigned char>& tmp, int degree, const double* d_xyz,
                 const double* d_q, int64_t n, int stages) {
  Lists& L = c.lists;
  Binned& B = c.bins;
  const int P = (degree + 1) * (degree + 2) / 2;
  const int bs = 256;
  if (stages & 1) {
    cudaEventRecord(c.ev[0], s);
    k_gather<<<grid_for(n, bs), bs, 0, s>>>(d_xyz, d_q, B.perm.p, n, c.pts.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    if (L.n_proxy > 0) {
      k_proxy<<<grid_for(int64_t(L.n_proxy) * P, bs), bs, 0, s>>>(c.trav.slot_node.p, L.n_proxy, degree,
                                                                    c.nodes.tri.p, n, c.pts.p);
      SSUM_LAUNCH_CHECK();
      c.launches++;
    }
    cudaEventRecord(c.ev[1], s);
  }
  if (!(stages & 2)) return;

  // ---- upward pass: chunk table (weight node bins cut into <= 1024-particle
  // chunks) built on the device
  // weight nodes: L.weight_nodes (host count), or the subtree builder's
  // marked subset (c.up_list with its device count c.up_count, <= n_weight)
  const int* wl = c.up_list ? c.up_list : L.weight_nodes.p;
  const int* d_nw = c.up_list ? c.up_count : nullptr;
  if (L.n_weight > 0) {
    const int nw = L.n_weight;
    c.wcount.ensure(size_t(nw) + 1, false, s);
    c.wcount_off.ensure(size_t(nw) + 1, false, s);
    k_up_nchunks<<<grid_for(nw + 1, 256), 256, 0, s>>>(wl, nw, B.cnt.p, c.wcount.p, d_nw);
    SSUM_LAUNCH_CHECK();
    size_t tb = 0;
    SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(nullptr, tb, c.wcount.p, c.wcount_off.p, nw + 1, s));
    tmp.ensure(tb, false, s);
    SSUM_CUDA_CHECK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, c.wcount.p, c.wcount_off.p, nw + 1, s));
    // chunk count without a read-back: a particle lies in at most one node
    // per level, so sum_w ceil(cnt_w / kUpChunk) <= nw + N (levels) / kUpChunk
    const int64_t nch_bound =
        int64_t(nw) + (int64_t(n) * (c.nodes.max_level + 1) + kUpChunk - 1) / kUpChunk;
    const int nch = static_cast<int>(nch_bound);
    c.wchunks.ensure(size_t(nch) + size_t(nw), false, s);
    c.wpart.ensure(size_t(nch) * P, false, s);
    int2* d_crange = reinterpret_cast<int2*>(c.wchunks.p + nch);
    k_up_fill<<<grid_for(nw, 256), 256, 0, s>>>(wl, nw, B.off.p, B.cnt.p, c.wcount_off.p, c.wchunks.p, d_crange,
                                                 d_nw);
    SSUM_LAUNCH_CHECK();
    c.launches += 4;
    if (nch > 0) launch_up_partial(c, s, degree, nch, c.wcount_off.p + nw);
    const int bt = ((P + 31) / 32) * 32;
    k_up_final<<<L.n_weight, bt, size_t(P) * 8, s>>>(wl, L.n_weight, d_crange, c.wpart.p, c.vinv.p, P, L.pslot.p, n,
                                                      c.pts.p, nullptr, d_nw);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  cudaEventRecord(c.ev[2], s);
}

void size_eval_buffers(Ctx& c, int degree, int D, int64_t n) {
  const int P = (degree + 1) * (degree + 2) / 2;
  ensure_vinv(c, degree);
  const int64_t npts = n + int64_t(c.lists.n_proxy) * P;
  if (npts > 0x7fffffff) throw Error(SSUM_INVALID, "point count exceeds int32 indexing");
  c.pts.ensure(size_t(npts));
  c.npts = npts;
  c.S.ensure(size_t(n) * D);
  c.coeff.ensure(std::max<size_t>(size_t(c.lists.n_proxy) * D * P, 1));
}

// Called by build_lists as soon as the proxy slots and weight nodes exist:
// the gather, proxy points and upward pass need nothing else from the lists,
// so they run on side_stream while the main stream builds the range lists
// and tiles (k_leaf_fill / k_fit_fill are latency-bound; the upward pass is
// FP64 work). evaluate() joins on prep_ev.
// stages: as launch_prep's (a call with stage 2 only follows one with stage
// 1 on the same evaluation).
void start_prep(Ctx& c, bool forked, int stages) {
  if (!c.early.xyz || !c.early_prep || c.bins.n == 0) return;
  const int64_t n = c.bins.n;
  size_eval_buffers(c, c.early.degree, c.early.dim, n);
  // forked: the caller recorded fork_ev (after sizing the buffers) before
  // launching work the prep stream need not wait for
  if (!forked) SSUM_CUDA_CHECK(cudaEventRecord(c.fork_ev, c.stream));
  SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.prep_stream, c.fork_ev, 0));
  if (c.io.active && (stages & 1))  // q of a host-pointer call
    SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.prep_stream, c.io.q, 0));
  launch_prep(c, c.prep_stream, c.cub_tmp_side, c.early.degree, c.early.xyz, c.early.q, n, stages);
  SSUM_CUDA_CHECK(cudaEventRecord(c.prep_ev, c.prep_stream));
  c.prep_started = true;
}

void evaluate(Ctx& c, int kernel, const ssum_config& cfg, const double* d_xyz, const double* d_q, int64_t n,
              double* d_out, ssum_stats* st) {
  Lists& L = c.lists;
  Binned& B = c.bins;
  const int degree = cfg.degree;
  const int P = (degree + 1) * (degree + 2) / 2;
  const int D = kernel == kBS ? 3 : 1;
  if (n == 0) return;
  if (!c.prep_started) size_eval_buffers(c, degree, D, n);
  const int bs = 256;

  if (c.prep_started) {
    // gather + proxy points + upward pass already running on side_stream
    // (start_prep, launched from build_lists once the slots were known)
    SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.prep_ev, 0));
    c.prep_started = false;
  } else {
    if (c.io.active) SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.io.q, 0));  // q of a host-pointer call
    launch_prep(c, c.stream, c.cub_tmp, degree, d_xyz, d_q, n, 3);
  }
  trace().mark("eval.upward_host");

  // ---- CP/CC + fit (side_stream, high priority) and PP + PC (this part's
  // contiguous tile range; c.stream). The two only read pts and write
  // disjoint buffers (coeff / S): the fit blocks (the larger tiles) are
  // dispatched first and the leaf blocks fill the SMs as the fit kernel's
  // tail drains.
  const int nfit = L.fit_sel_all ? L.n_fit_tiles : L.n_fit_sel;
  const int ntl = L.leaf_t1 - L.leaf_t0;
  const bool fork = c.overlap_tiles && nfit > 0 && ntl > 0;
  cudaStream_t fit_stream = fork ? c.side_stream : c.stream;
  cudaEventRecord(c.ev[3], c.stream);
  // the join below also runs when a launch check throws in between, so no
  // fit-tile work outlives this call unordered with the caller's stream
  struct Join {
    Ctx& c;
    bool on = false;
    void now() {
      if (!on) return;
      on = false;
      SSUM_CUDA_CHECK(cudaEventRecord(c.join_ev, c.side_stream));
      SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, c.join_ev, 0));
    }
    ~Join() {
      if (on) {
        cudaEventRecord(c.join_ev, c.side_stream);
        cudaStreamWaitEvent(c.stream, c.join_ev, 0);
      }
    }
  } join{c};
  if (fork) {
    SSUM_CUDA_CHECK(cudaEventRecord(c.fork_ev, c.stream));
    SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.side_stream, c.fork_ev, 0));
    join.on = true;
  }
  cudaEventRecord(c.side_ev[0], fit_stream);
  if (nfit > 0) {
    launch_fit_tiles(c, fit_stream, kernel, P, nfit, L.fit_sel_all ? nullptr : L.fit_sel.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  cudaEventRecord(c.side_ev[1], fit_stream);
  cudaEventRecord(c.leaf_ev[0], c.stream);
  if (ntl > 0) {
    launch_leaf_tiles(c, c.stream, kernel, L.leaf_tiles.p + L.leaf_t0, ntl, L.leaf_ranges.p, c.S.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  cudaEventRecord(c.leaf_ev[1], c.stream);
  join.now();
  cudaEventRecord(c.ev[4], c.stream);

  // ---- downward + finish
  if (c.io.active && c.io.h_out) {
    // host result: finish in original order, piece by piece, each piece's
    // copy to the host overlapping the next piece's finish
    c.inv_perm.ensure(size_t(n));
    k_inv_perm<<<grid_for(n, bs), bs, 0, c.stream>>>(B.perm.p, n, c.inv_perm.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    // Spatially coherent caller order (a warp's rows share ancestors): finish
    // each piece directly in caller order. Otherwise (e.g. random input) the
    // per-lane finish would walk unrelated ancestors in every lane: finish
    // in tree order in place over S, then gather each piece's rows.
    const bool gather = !B.input_coherent;
    if (gather) {
      if (kernel == kBS)
        launch_finish<kBS>(c, degree, c.S.p, nullptr, 0, 0, true);
      else
        launch_finish<kLOG>(c, degree, c.S.p, nullptr, 0, 0, true);
    }
    for (int j = 0; j < Ctx::kIoChunks; ++j) {
      const int64_t a = c.io.bounds[j], b = c.io.bounds[j + 1];
      if (gather) {
        if (b > a) {
          k_gather_rows<<<grid_for(b - a, bs), bs, 0, c.stream>>>(c.S.p, c.inv_perm.p, a, b, L.p0, L.p1, D, d_out);
          SSUM_LAUNCH_CHECK();
          c.launches++;
        }
      } else if (kernel == kBS) {
        launch_finish<kBS>(c, degree, d_out, c.inv_perm.p, a, b);
      } else {
        launch_finish<kLOG>(c, degree, d_out, c.inv_perm.p, a, b);
      }
      SSUM_CUDA_CHECK(cudaEventRecord(c.io.out[j], c.stream));
      SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, c.io.out[j], 0));
      if (j == 0) SSUM_CUDA_CHECK(cudaEventRecord(c.io.t0, c.copy_stream));
      if (b > a)
        SSUM_CUDA_CHECK(cudaMemcpyAsync(c.io.h_out + a * D, d_out + a * D, size_t(b - a) * D * sizeof(double),
                                        cudaMemcpyDeviceToHost, c.copy_stream));
    }
    SSUM_CUDA_CHECK(cudaEventRecord(c.io.t1, c.copy_stream));
  } else if (c.out_tree_order) {
    // this part's rows in tree order: position p0 + r -> row r (the rows
    // one multi-GPU all-gather exchanges, dist.py)
    if (kernel == kBS)
      launch_finish<kBS>(c, degree, d_out, nullptr, 0, 0, true, L.p0);
    else
      launch_finish<kLOG>(c, degree, d_out, nullptr, 0, 0, true, L.p0);
  } else if (kernel == kBS) {
    launch_finish<kBS>(c, degree, d_out);
  } else {
    launch_finish<kLOG>(c, degree, d_out);
  }
  cudaEventRecord(c.ev[5], c.stream);
  check_flags(c, "treecode_sum");
  if (st) {
    // upward: ev[0..2] (on side_stream when it started early); each tile
    // kernel's own span on its stream; tiles: both together
    auto span = [](cudaEvent_t e0, cudaEvent_t e1) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      return static_cast<double>(ms);
    };
    st->upward_ms = span(c.ev[0], c.ev[2]);
    st->cp_cc_fit_ms = span(c.side_ev[0], c.side_ev[1]);
    st->pp_pc_ms = span(c.leaf_ev[0], c.leaf_ev[1]);
    st->tiles_ms = span(c.ev[3], c.ev[4]);
    st->finish_ms = span(c.ev[4], c.ev[5]);
  }
}

void direct_sum_device(Ctx& c, int kernel, const double* d_xyz, const double* d_q, int64_t n, double* d_out) {
  if (n == 0) return;
  const int D = kernel == kBS ? 3 : 1;
  c.pts.ensure(size_t(n));
  c.S.ensure(size_t(n) * D);
  const int bs = 256;
  SSUM_CUDA_CHECK(cudaMemsetAsync(c.d_flags.p, 0, 4, c.stream));
  k_gather<<<grid_for(n, bs), bs, 0, c.stream>>>(d_xyz, d_q, nullptr, n, c.pts.p);
  SSUM_LAUNCH_CHECK();
  c.launches++;
  launch_direct(c, kernel, n, d_out);
  check_flags(c, "direct_sum");
}

// ---- per-interaction entry points -----------------------------------------
// eval_pp / eval_pc / eval_cp / eval_cc (treecode.cpp:170-244) and
// compute_proxy_weights (treecode.cpp:79-91) for one node pair of the last
// binning, in O(|t| |s| + (|t| + |s|) p + p^2) work: only the two bins'
// particles are packed (from the caller's arrays, through the binning's
// permutation) into a compact point array, followed by the source's and the
// target's proxy points, and the pairs run through the tree code's own
// kernels (k_tiles leaf / fit mode, k_up_partial / k_up_final, k_proxy).
namespace {

// Compact layout: bins are contiguous tree-position ranges and two bins are
// either nested or disjoint. Nested (incl. equal): the outer range is packed
// once, so a particle in both bins is one point (self pairs are excluded by
// index, as in the tree code). Disjoint: target bin, then source bin.
struct Compact {
  int64_t n = 0;
  int t0 = 0, nt = 0, s0 = 0, ns = 0;
  bool nested = false;
  std::vector<int> ids;  // caller index of each compact particle
};

Compact pack_bins(Ctx& c, const double* xyz, const double* q, int tdev, int sdev) {
  const HostTree& h = host_tree(c);
  Compact k;
  const int64_t a0 = h.off[size_t(tdev)], a1 = a0 + h.cnt[size_t(tdev)];
  const int64_t b0 = h.off[size_t(sdev)], b1 = b0 + h.cnt[size_t(sdev)];
  k.nt = static_cast<int>(a1 - a0);
  k.ns = static_cast<int>(b1 - b0);
  std::vector<std::pair<int64_t, int64_t>> runs;
  if (k.nt > 0 && k.ns > 0 && a0 < b1 && b0 < a1) {
    k.nested = true;
    const int64_t o0 = std::min(a0, b0), o1 = std::max(a1, b1);
    runs.push_back({o0, o1});
    k.t0 = static_cast<int>(a0 - o0);
    k.s0 = static_cast<int>(b0 - o0);
  } else {
    runs.push_back({a0, a1});
    runs.push_back({b0, b1});
    k.t0 = 0;
    k.s0 = k.nt;
  }
  for (const auto& r : runs) k.n += r.second - r.first;
  k.ids.resize(size_t(k.n));
  int64_t at = 0;
  for (const auto& r : runs) {
    if (r.second > r.first)
      SSUM_CUDA_CHECK(cudaMemcpyAsync(k.ids.data() + at, c.bins.perm.p + r.first, size_t(r.second - r.first) * 4,
                                      cudaMemcpyDeviceToHost, c.stream));
    at += r.second - r.first;
  }
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  std::vector<double4> hp(size_t(k.n));
  for (int64_t i = 0; i < k.n; ++i) {
    const size_t id = size_t(k.ids[size_t(i)]);
    hp[size_t(i)] = make_double4(xyz[3 * id], xyz[3 * id + 1], xyz[3 * id + 2], q[id]);
  }
  if (k.n) SSUM_CUDA_CHECK(cudaMemcpy(c.pts.p, hp.data(), hp.size() * sizeof(double4), cudaMemcpyHostToDevice));
  return k;
}

// fitted value sum_m C[m, d] B_m(beta_t(x)) at the compact targets (add_fitted_value,
// treecode.cpp:143-155); runtime degree (this is not the tree code's hot loop)
__global__ void k_ix_down(const double4* __restrict__ pts, int t0, int nt, const double* __restrict__ cramer_t,
                          const double* __restrict__ coeff, int degree, int D, double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nt) return;
  const int P = (degree + 1) * (degree + 2) / 2;
  const double4 x = pts[t0 + k];
  double b1, b2, b3;
  bary(cramer_t, x.x, x.y, x.z, b1, b2, b3);
  double p1[kMaxDegree + 1], p2[kMaxDegree + 1], p3[kMaxDegree + 1];
  p1[0] = p2[0] = p3[0] = 1.0;
  for (int e = 1; e <= degree; ++e) {
    p1[e] = p1[e - 1] * b1;
    p2[e] = p2[e - 1] * b2;
    p3[e] = p3[e - 1] * b3;
  }
  double val[3] = {0.0, 0.0, 0.0};
  int m = 0;
  for (int kk = 0; kk <= degree; ++kk)
    for (int jj = 0; jj <= degree - kk; ++jj, ++m) {
      const double B = p1[degree - kk - jj] * p2[jj] * p3[kk];
      for (int d = 0; d < D; ++d) val[d] = fma(coeff[d * P + m], B, val[d]);
    }
  for (int d = 0; d < D; ++d) out[size_t(k) * D + d] = val[d];
}

// raw PP / PC sums of the compact targets: x X S (Biot-Savart) or -S / (4 pi)
__global__ void k_ix_raw(const double4* __restrict__ pts, int t0, int nt, const double* __restrict__ S, int D,
                         double* __restrict__ out) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nt) return;
  const double* s = S + size_t(t0 + k) * D;
  if (D == 3) {
    const double4 x = pts[t0 + k];
    out[3 * size_t(k)] = x.y * s[2] - x.z * s[1];
    out[3 * size_t(k) + 1] = x.z * s[0] - x.x * s[2];
    out[3 * size_t(k) + 2] = x.x * s[1] - x.y * s[0];
  } else {
    out[k] = -kInv4Pi * s[0];
  }
}

// Upward pass of one node over compact [s0, s0 + ns): chunks, partial sums,
// then w_hat into the proxy points at pts[base ..) or, with raw, w into raw.
// ix_ints must hold [0] = 0 (weight node 0 -> slot 0).
void ix_upward(Ctx& c, int degree, int sdev, int s0, int ns, int64_t base, double* raw) {
  const int P = (degree + 1) * (degree + 2) / 2;
  std::vector<int4> ch;
  for (int b = 0; b < ns; b += kUpChunk) ch.push_back(make_int4(sdev, s0 + b, std::min(kUpChunk, ns - b), 0));
  const int nch = static_cast<int>(ch.size());
  c.wchunks.ensure(size_t(nch) + 2);
  c.wpart.ensure(size_t(std::max(nch, 1)) * P);
  // chunk table, then (count, pad, (0, count)) for launch_up_partial / k_up_final
  ch.push_back(make_int4(nch, 0, 0, nch));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.wchunks.p, ch.data(), ch.size() * sizeof(int4), cudaMemcpyHostToDevice, c.stream));
  const int* d_cnt = reinterpret_cast<const int*>(c.wchunks.p + nch);
  const int2* d_range = reinterpret_cast<const int2*>(reinterpret_cast<const int*>(c.wchunks.p + nch) + 2);
  if (nch > 0) launch_up_partial(c, c.stream, degree, nch, d_cnt);
  const int bt = ((P + 31) / 32) * 32;
  k_up_final<<<1, bt, size_t(P) * 8, c.stream>>>(c.ix_ints.p, 1, d_range, c.wpart.p, c.vinv.p, P, c.ix_ints.p, base,
                                                  c.pts.p, raw);
  SSUM_LAUNCH_CHECK();
  c.launches++;
}

}  // namespace

void eval_interaction(Ctx& c, int kernel, int degree, const double* xyz, const double* q, int target, int source,
                      int kind, double* field) {
  const int D = kernel == kBS ? 3 : 1;
  const int P = (degree + 1) * (degree + 2) / 2;
  if (kind != 0) ensure_vinv(c, degree);
  c.pts.ensure(size_t(c.bins.n) + 2 * size_t(P) + 1);
  const Compact k = pack_bins(c, xyz, q, target, source);
  if (k.nt == 0 || k.ns == 0) return;  // an empty bin contributes nothing
  const int64_t n = k.n;
  c.npts = n + 2 * P;
  c.S.ensure(size_t(n + 2 * P) * D);
  c.coeff.ensure(size_t(D) * P);
  c.ix_out.ensure(size_t(k.nt) * D);
  c.ix_ints.ensure(8);
  const int hi[8] = {0, source, target, 0, 0, 0, 0, 0};
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.ix_ints.p, hi, sizeof(hi), cudaMemcpyHostToDevice, c.stream));
  SSUM_CUDA_CHECK(cudaMemsetAsync(c.d_flags.p, 0, 4, c.stream));
  const int bs = 128;
  if (kind != 0) {  // proxy points of the source (slot 0) and the target (slot 1)
    k_proxy<<<grid_for(2 * P, bs), bs, 0, c.stream>>>(c.ix_ints.p + 1, 2, degree, c.nodes.tri.p, n, c.pts.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  }
  if (kind == 1 || kind == 3) ix_upward(c, degree, source, k.s0, k.ns, n, nullptr);  // w_hat at pts[n, n + P)
  // one range per interaction: PP / CP read the source bin, PC / CC its proxies
  const bool from_bin = kind == 0 || kind == 2;
  const SrcRange r{from_bin ? k.s0 : static_cast<int>(n), from_bin ? k.ns : P, kind == 0 ? 1 : 0, 0};
  c.ix_range.ensure(1);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.ix_range.p, &r, sizeof(r), cudaMemcpyHostToDevice, c.stream));
  if (kind == 0 || kind == 1) {
    const int ntile = (k.nt + kTileTargets - 1) / kTileTargets;
    std::vector<Tile> tl(static_cast<size_t>(ntile));
    for (int j = 0; j < ntile; ++j) {
      Tile& t = tl[size_t(j)];
      t.tgt_begin = k.t0 + j * kTileTargets;
      t.tgt_count = std::min(kTileTargets, k.nt - j * kTileTargets);
      t.list_begin = 0;
      t.list_end = 1;
      t.near_total = kind == 0 ? k.ns : 0;
      t.self_shift = -k.s0;  // point j of the bin sits at flattened position j - s0
      t.has_self = (kind == 0 && k.nested) ? 1 : 0;
      t.total = r.count;
    }
    c.ix_tiles.ensure(tl.size());
    SSUM_CUDA_CHECK(cudaMemcpyAsync(c.ix_tiles.p, tl.data(), tl.size() * sizeof(Tile), cudaMemcpyHostToDevice,
                                    c.stream));
    launch_leaf_tiles(c, c.stream, kernel, c.ix_tiles.p, ntile, c.ix_range.p, c.S.p);
    SSUM_LAUNCH_CHECK();
    k_ix_raw<<<grid_for(k.nt, bs), bs, 0, c.stream>>>(c.pts.p, k.t0, k.nt, c.S.p, D, c.ix_out.p);
    SSUM_LAUNCH_CHECK();
    c.launches += 2;
  } else {
    // phi at the target's proxy points (slot 1), C = V^-1 phi into coeff slot 0
    Tile t{static_cast<int>(n + P), P, 0, 1, 0, 0, 0, r.count};
    c.ix_tiles.ensure(1);
    SSUM_CUDA_CHECK(cudaMemcpyAsync(c.ix_tiles.p, &t, sizeof(t), cudaMemcpyHostToDevice, c.stream));
    launch_fit_tiles_on(c, c.stream, kernel, P, c.ix_tiles.p, 1, nullptr, c.ix_range.p, c.ix_ints.p, c.ix_ints.p,
                        c.coeff.p);
    SSUM_LAUNCH_CHECK();
    k_ix_down<<<grid_for(k.nt, bs), bs, 0, c.stream>>>(c.pts.p, k.t0, k.nt, c.nodes.cramer.p + 12 * size_t(target),
                                                        c.coeff.p, degree, D, c.ix_out.p);
    SSUM_LAUNCH_CHECK();
    c.launches += 2;
  }
  check_flags(c, "eval_interaction");
  std::vector<double> out(size_t(k.nt) * D);
  SSUM_CUDA_CHECK(cudaMemcpy(out.data(), c.ix_out.p, out.size() * 8, cudaMemcpyDeviceToHost));
  for (int i = 0; i < k.nt; ++i) {
    double* f = field + size_t(k.ids[size_t(k.t0 + i)]) * D;
    for (int d = 0; d < D; ++d) f[d] += out[size_t(i) * D + d];
  }
}

void proxy_weights(Ctx& c, int degree, const double* xyz, const double* q, int node, double* w) {
  const int P = (degree + 1) * (degree + 2) / 2;
  c.pts.ensure(size_t(c.bins.n) + 1);
  const Compact k = pack_bins(c, xyz, q, node, node);
  c.ix_out.ensure(size_t(P));
  c.ix_ints.ensure(8);
  const int hi[8] = {0, node, node, 0, 0, 0, 0, 0};
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.ix_ints.p, hi, sizeof(hi), cudaMemcpyHostToDevice, c.stream));
  ix_upward(c, degree, node, k.s0, k.ns, 0, c.ix_out.p);
  SSUM_CUDA_CHECK(cudaMemcpyAsync(w, c.ix_out.p, size_t(P) * 8, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
}

}  // namespace ssum
