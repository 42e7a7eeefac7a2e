// extern "C" boundary (include/spheresum_b200.h): context lifetime, the
// treecode/direct entry points, tree and list export in the reference's
// numbering, and the device-resident RK4 driver. Internal ssum::Error
// exceptions stop here and become status codes; nothing throws across the ABI.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "internal.cuh"

namespace ssum {

void sorted_interactions(Ctx& c, std::vector<int4>& out);

cudaStream_t& dbuf_stream() {
  thread_local cudaStream_t s = nullptr;
  return s;
}

double Trace::now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}
Trace& trace() {
  static Trace t = [] {
    Trace x;
    const char* e = std::getenv("SSUM_TRACE");
    x.on = e && *e && *e != '0';
    return x;
  }();
  return t;
}

void check_flags(Ctx& c, const char* where) {
  // pinned destination: a copy into pageable memory takes the driver's staged
  // path, which stalled the host ~0.1 ms per call (CUPTI timeline)
  if (!c.h_pinned) SSUM_CUDA_CHECK(cudaMallocHost(&c.h_pinned, 64 * sizeof(int)));
  SSUM_CUDA_CHECK(cudaMemcpyAsync(c.h_pinned, c.d_flags.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  const int f = c.h_pinned[0];
  c.last_flags = f;
  if (f & kFlagGeometry) throw Error(SSUM_GEOMETRY, std::string(where) + ": degenerate geometry");
  if (f & kFlagSingular)
    throw Error(SSUM_SINGULAR, std::string(where) + ": kernel evaluated at its singularity (1 - x.y <= 1e-14)");
}

namespace {

using clk = std::chrono::steady_clock;
double secs(clk::time_point a, clk::time_point b) { return std::chrono::duration<double>(b - a).count(); }

// TraversalConfig::validate (treecode.cpp:13-20)
void validate(const ssum_config* cfg) {
  if (!cfg) throw Error(SSUM_CONFIG, "null config");
  if (!(cfg->theta > 0.0 && cfg->theta <= 1.0)) throw Error(SSUM_CONFIG, "theta must be in (0, 1]");
  if (cfg->n_threshold < 1) throw Error(SSUM_CONFIG, "n_threshold must be >= 1");
  if (cfg->degree < 1 || cfg->degree > kMaxDegree) throw Error(SSUM_CONFIG, "degree must be in [1, 20]");
  if (cfg->max_depth < 1 || cfg->max_depth > 40) throw Error(SSUM_CONFIG, "max_depth must be in [1, 40]");
}

void check_kernel(int kernel) {
  if (kernel != SSUM_BIOT_SAVART && kernel != SSUM_LOG_POTENTIAL) throw Error(SSUM_INVALID, "unknown kernel id");
}

void check_n(int64_t n) {
  if (n < 0 || n > 0x3fffffff) throw Error(SSUM_INVALID, "particle count out of range");
}

template <class F>
int guarded(ssum_ctx* h, F&& f) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c) return SSUM_INVALID;
  try {
    cudaSetDevice(c->device);
    dbuf_stream() = c->stream;
    f(*c);
    return SSUM_OK;
  } catch (const Error& e) {
    c->last_error = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    c->last_error = "host allocation failed";
    return SSUM_NOMEM;
  } catch (const std::exception& e) {
    c->last_error = e.what();
    return SSUM_INTERNAL;
  }
}

// The full device path: bin, traverse, evaluate. Inputs/outputs on the device.
void treecode_device(Ctx& c, int kernel, const ssum_config& cfg, const double* d_xyz, const double* d_q, int64_t n,
                     double* d_out, ssum_stats* st) {
  const int64_t l0 = c.launches;
  Trace& tr = trace();
  if (tr.on) tr.start();
  const auto t0 = clk::now();
  tree_bin(c, d_xyz, n, cfg.n_threshold, cfg.max_depth);
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  tr.mark("bin.done");
  const auto t1 = clk::now();
  struct Unrestrict {  // the restriction is this evaluation's only (exports list everything)
    Ctx& c;
    ~Unrestrict() { c.restrict_on = false; }
  } unrestrict{c};
  plan_restriction(c);
  struct Early {  // build_lists starts the upward pass early (start_prep)
    Ctx& c;
    ~Early() {
      // evaluate() normally joins prep_ev; if anything threw in between, join
      // here so the side stream's gather / upward pass cannot overlap the
      // next call's binning
      if (c.prep_started) cudaStreamWaitEvent(c.stream, c.prep_ev, 0);
      c.early = Ctx::Early{};
      c.prep_started = false;
    }
  } early{c};
  // Lists per target subtree (sublists.cu) when the binning made a plan;
  // if they came out incomplete (a buffer outgrew, undecided MAC pairs) the
  // evaluation is redone on the global traversal path (traversal.cu).
  const int choice = sub_lists_choice(c, cfg);
  const bool sub = (choice & 1) != 0, trial = choice >= 2;
  if (trial) SSUM_CUDA_CHECK(cudaEventRecord(c.ev[6], c.stream));
  auto t2 = clk::now();
  for (int attempt = 0;; ++attempt) {
    c.early = Ctx::Early{d_xyz, d_q, cfg.degree, kernel == SSUM_BIOT_SAVART ? 3 : 1};
    if (sub && attempt == 0)
      build_lists_subtree(c, cfg);
    else
      traverse_and_build_lists(c, cfg, false);
    c.early = Ctx::Early{};
    tr.mark("lists.done");
    t2 = clk::now();
    evaluate(c, kernel, cfg, d_xyz, d_q, n, d_out, st);
    if (!sub_lists_redo(c, c.last_flags)) break;
    SSUM_CUDA_CHECK(cudaMemsetAsync(c.d_flags.p, 0, sizeof(int), c.stream));
  }
  if (trial) {  // the stream has drained (the evaluation's final check)
    SSUM_CUDA_CHECK(cudaEventRecord(c.ev[7], c.stream));
    SSUM_CUDA_CHECK(cudaEventSynchronize(c.ev[7]));
    float ms = 0.f;
    SSUM_CUDA_CHECK(cudaEventElapsedTime(&ms, c.ev[6], c.ev[7]));
    sub_lists_timed(c, sub ? 1 : 0, ms);
  }
  finalize_counts(c);
  tr.mark("eval.done");
  const auto t3 = clk::now();
  if (tr.on) {  // per label: total ms (count)
    double prev = tr.t0;
    std::vector<std::pair<std::string, std::pair<double, int>>> agg;
    for (const auto& m : tr.marks) {
      const double dt = (m.second - prev) * 1e3;
      prev = m.second;
      auto it = std::find_if(agg.begin(), agg.end(), [&](const auto& a) { return a.first == m.first; });
      if (it == agg.end())
        agg.push_back({m.first, {dt, 1}});
      else
        it->second.first += dt, it->second.second += 1;
    }
    std::fprintf(stderr, "[ssum trace]");
    for (const auto& a : agg) std::fprintf(stderr, " %s=%.3f(%d)", a.first.c_str(), a.second.first, a.second.second);
    std::fprintf(stderr, "\n");
  }
  if (st) {
    st->bin_seconds += secs(t0, t1);
    st->traversal_seconds += secs(t1, t2);
    st->eval_seconds += secs(t2, t3);
    for (int k = 0; k < 4; ++k) {
      st->interaction_counts[k] = c.lists.counts[k];
      st->kernel_evals[k] = c.lists.local_evals[k];  // this part's work (all of it when unpartitioned)
    }
    st->node_count = c.nodes.count;
    st->leaf_count = c.bins.n_leaves;
    st->weight_nodes = c.lists.n_weight;
    st->fit_nodes = c.lists.n_fit;
    st->up_visits = c.lists.visits[0];
    st->down_visits = c.lists.visits[1];
    st->gpu_launches = c.launches - l0;
    st->mac_host_decisions = c.mac.resolved;
  }
}

}  // namespace

// Reference node ids: roots 0..19; each bin_particles call appends the quads
// it creates in the order distribute() visits their parents (depth-first
// preorder, face_tree.cpp:39-71). Returns dev -> ref.
std::vector<int> reference_ids(const HostTree& h) {
  const int nn = static_cast<int>(h.level.size());
  std::vector<int> pre(size_t(nn), -1);
  int r = 0;
  std::vector<int> stack;
  for (int f = 19; f >= 0; --f) stack.push_back(f);
  while (!stack.empty()) {
    const int id = stack.back();
    stack.pop_back();
    pre[id] = r++;
    const int cb = h.child_base[id];
    if (cb >= 0)
      for (int q = 3; q >= 0; --q) stack.push_back(cb + q);
  }
  std::vector<int> quads;  // first child of every quad
  for (int id = 20; id < nn; id += 4) quads.push_back(id);
  std::stable_sort(quads.begin(), quads.end(), [&](int a, int b) {
    if (h.created_call[a] != h.created_call[b]) return h.created_call[a] < h.created_call[b];
    return pre[h.parent[a]] < pre[h.parent[b]];
  });
  std::vector<int> ref(static_cast<size_t>(nn));
  for (int f = 0; f < 20; ++f) ref[f] = f;
  int next = 20;
  for (const int q : quads)
    for (int k = 0; k < 4; ++k) ref[q + k] = next++;
  return ref;
}

namespace {

void upload(Ctx& c, DBuf<double>& buf, const double* h, size_t count, ssum_stats* st) {
  const auto t0 = clk::now();
  buf.ensure(std::max<size_t>(count, 1));
  if (count) SSUM_CUDA_CHECK(cudaMemcpyAsync(buf.p, h, count * 8, cudaMemcpyHostToDevice, c.stream));
  if (st) {
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
    st->h2d_seconds += secs(t0, clk::now());
  }
}

void download(Ctx& c, double* h, const double* d, size_t count, ssum_stats* st) {
  const auto t0 = clk::now();
  if (count) SSUM_CUDA_CHECK(cudaMemcpyAsync(h, d, count * 8, cudaMemcpyDeviceToHost, c.stream));
  SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  if (st) st->d2h_seconds += secs(t0, clk::now());
}

__global__ void k_add_scaled(double* __restrict__ y, const double* __restrict__ x, double a, int64_t n) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) y[i] += a * x[i];
}

void add_scaled(Ctx& c, double* y, const double* x, double a, int64_t n) {
  k_add_scaled<<<grid_for(n, 256), 256, 0, c.stream>>>(y, x, a, n);
  SSUM_LAUNCH_CHECK();
  c.launches++;
}

__global__ void k_rk4_stage(int64_t n, int stage, double cs, const double* __restrict__ x0,
                            const double* __restrict__ z0, const double* __restrict__ area,
                            const double* __restrict__ kprev, const double* __restrict__ kzprev,
                            double* __restrict__ xs, double* __restrict__ q, int* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double zs;
  if (stage == 0) {
    xs[3 * i] = x0[3 * i];
    xs[3 * i + 1] = x0[3 * i + 1];
    xs[3 * i + 2] = x0[3 * i + 2];
    zs = z0[i];
  } else {
    int bad = 0;
    const d3 v{add_rn(x0[3 * i], mul_rn(cs, kprev[3 * i])), add_rn(x0[3 * i + 1], mul_rn(cs, kprev[3 * i + 1])),
               add_rn(x0[3 * i + 2], mul_rn(cs, kprev[3 * i + 2]))};
    const d3 u = unit_rn(v, &bad);
    if (bad) atomicOr(flags, kFlagGeometry);
    xs[3 * i] = u.x;
    xs[3 * i + 1] = u.y;
    xs[3 * i + 2] = u.z;
    zs = add_rn(z0[i], mul_rn(cs, kzprev[i]));
  }
  q[i] = mul_rn(zs, area[i]);
}

// stage-0 strengths q = zeta A (k_rk4_stage's product) for the host-pointer RK4
__global__ void k_rk4_q(int64_t n, const double* __restrict__ z0, const double* __restrict__ area,
                        double* __restrict__ q) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) q[i] = mul_rn(z0[i], area[i]);
}

// k_s = u, kz_s = -2 Omega u_z; acc = ((k1 + 2 k2) + 2 k3) + k4 in that order.
__global__ void k_rk4_accum(int64_t n, int stage, double omega, const double* __restrict__ u, double* __restrict__ k,
                            double* __restrict__ kz, double* __restrict__ acc, double* __restrict__ accz) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double w = (stage == 1 || stage == 2) ? 2.0 : 1.0;
  const double kzv = mul_rn(mul_rn(-2.0, omega), u[3 * i + 2]);
  for (int d = 0; d < 3; ++d) {
    const double v = u[3 * i + d];
    k[3 * i + d] = v;
    acc[3 * i + d] = stage == 0 ? v : add_rn(acc[3 * i + d], mul_rn(w, v));
  }
  kz[i] = kzv;
  accz[i] = stage == 0 ? kzv : add_rn(accz[i], mul_rn(w, kzv));
}

// k_rk4_accum with u read from the all-gathered tree-order rows of every
// part (slot r of width W holds part r's positions [cuts[r], cuts[r+1]));
// one thread per tree position j, particle perm[j]. Same arithmetic, so a
// driver built on it reproduces ssum_rk4 bit for bit.
__global__ void k_rk4_accum_rows(int64_t n, int stage, double omega, const double* __restrict__ rows, int64_t W,
                                 const long long* __restrict__ cuts, int np, const int* __restrict__ perm,
                                 double* __restrict__ k, double* __restrict__ kz, double* __restrict__ acc,
                                 double* __restrict__ accz) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= n) return;
  int lo = 0, hi = np - 1;  // the part holding j: last r with cuts[r] <= j
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (cuts[mid] <= j)
      lo = mid;
    else
      hi = mid - 1;
  }
  const double* u = rows + 3 * (lo * W + (j - cuts[lo]));
  const int64_t i = perm[j];
  const double w = (stage == 1 || stage == 2) ? 2.0 : 1.0;
  const double kzv = mul_rn(mul_rn(-2.0, omega), u[2]);
  for (int d = 0; d < 3; ++d) {
    const double v = u[d];
    k[3 * i + d] = v;
    acc[3 * i + d] = stage == 0 ? v : add_rn(acc[3 * i + d], mul_rn(w, v));
  }
  kz[i] = kzv;
  accz[i] = stage == 0 ? kzv : add_rn(accz[i], mul_rn(w, kzv));
}

// k_rk4_accum_rows fused with the next stage's k_rk4_stage (cs >= 0): one
// thread per PARTICLE i, its row gathered from tree position inv[i] (one
// scattered 24-byte read instead of four scattered read-modify-writes), all
// other arrays coalesced; k / kz written only when given. Same arithmetic in
// the same order as the two kernels.
__global__ void k_rk4_advance_rows(int64_t n, int stage, double omega, double cs, const double* __restrict__ rows,
                                   int64_t W, const long long* __restrict__ cuts, int np, const int* __restrict__ inv,
                                   const double* __restrict__ x0, const double* __restrict__ z0,
                                   const double* __restrict__ area, double* __restrict__ acc,
                                   double* __restrict__ accz, double* __restrict__ k, double* __restrict__ kz,
                                   double* __restrict__ xs, double* __restrict__ q, int* flags) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double* u = rows + 3 * i;  // no inv: the velocities in the caller's order (ssum_rk4)
  if (inv) {
    const int64_t j = inv[i];
    int lo = 0, hi = np - 1;  // the part holding tree position j
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (cuts[mid] <= j)
        lo = mid;
      else
        hi = mid - 1;
    }
    u = rows + 3 * (lo * W + (j - cuts[lo]));
  }
  const double u0 = u[0], u1 = u[1], u2 = u[2];
  const double w = (stage == 1 || stage == 2) ? 2.0 : 1.0;
  const double kzv = mul_rn(mul_rn(-2.0, omega), u2);
  if (stage == 0) {
    acc[3 * i] = u0;
    acc[3 * i + 1] = u1;
    acc[3 * i + 2] = u2;
    accz[i] = kzv;
  } else {
    acc[3 * i] = add_rn(acc[3 * i], mul_rn(w, u0));
    acc[3 * i + 1] = add_rn(acc[3 * i + 1], mul_rn(w, u1));
    acc[3 * i + 2] = add_rn(acc[3 * i + 2], mul_rn(w, u2));
    accz[i] = add_rn(accz[i], mul_rn(w, kzv));
  }
  if (k) {
    k[3 * i] = u0;
    k[3 * i + 1] = u1;
    k[3 * i + 2] = u2;
    kz[i] = kzv;
  }
  if (cs >= 0.0) {  // k_rk4_stage of the next stage (stage + 1 >= 1)
    int bad = 0;
    const d3 v{add_rn(x0[3 * i], mul_rn(cs, u0)), add_rn(x0[3 * i + 1], mul_rn(cs, u1)),
               add_rn(x0[3 * i + 2], mul_rn(cs, u2))};
    const d3 un = unit_rn(v, &bad);
    if (bad) atomicOr(flags, kFlagGeometry);
    xs[3 * i] = un.x;
    xs[3 * i + 1] = un.y;
    xs[3 * i + 2] = un.z;
    q[i] = mul_rn(add_rn(z0[i], mul_rn(cs, kzv)), area[i]);
  }
}

__global__ void k_inv_of(const int* __restrict__ perm, int64_t n, int* __restrict__ inv) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j < n) inv[perm[j]] = static_cast<int>(j);
}

// particles [i0, i1)
__global__ void k_rk4_final(int64_t i0, int64_t i1, double h6, double* __restrict__ x0, double* __restrict__ z0,
                            const double* __restrict__ acc, const double* __restrict__ accz, int* flags) {
  const int64_t i = i0 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= i1) return;
  int bad = 0;
  const d3 v{add_rn(x0[3 * i], mul_rn(h6, acc[3 * i])), add_rn(x0[3 * i + 1], mul_rn(h6, acc[3 * i + 1])),
             add_rn(x0[3 * i + 2], mul_rn(h6, acc[3 * i + 2]))};
  const d3 u = unit_rn(v, &bad);
  if (bad) atomicOr(flags, kFlagGeometry);
  x0[3 * i] = u.x;
  x0[3 * i + 1] = u.y;
  x0[3 * i + 2] = u.z;
  z0[i] = add_rn(z0[i], mul_rn(h6, accz[i]));
}

// reference node id -> device node id of the context's tree
int dev_node(Ctx& c, int ref_id) {
  const std::vector<int> ref = reference_ids(host_tree(c));
  const int nn = static_cast<int>(ref.size());
  if (ref_id < 0 || ref_id >= nn) throw Error(SSUM_INVALID, "node id out of range");
  for (int d = 0; d < nn; ++d)
    if (ref[size_t(d)] == ref_id) return d;
  throw Error(SSUM_INTERNAL, "node id not found");
}

}  // namespace
}  // namespace ssum

using namespace ssum;

extern "C" {

int ssum_create(int device, ssum_ctx** out) {
  if (!out) return SSUM_INVALID;
  *out = nullptr;
  Ctx* c = nullptr;
  try {
    c = new Ctx();
    c->device = device;
    SSUM_CUDA_CHECK(cudaSetDevice(device));
    SSUM_CUDA_CHECK(cudaStreamCreateWithFlags(&c->own_stream, cudaStreamNonBlocking));
    c->stream = c->own_stream;
    dbuf_stream() = c->stream;
    {  // keep freed blocks in the device's pool between calls (ssum_destroy trims it)
      cudaMemPool_t pool;
      SSUM_CUDA_CHECK(cudaDeviceGetDefaultMemPool(&pool, device));
      uint64_t keep = ~0ull;
      SSUM_CUDA_CHECK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    for (auto& e : c->ev) SSUM_CUDA_CHECK(cudaEventCreate(&e));
    SSUM_CUDA_CHECK(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    int prio_lo = 0, prio_hi = 0;
    SSUM_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    SSUM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->side_stream, cudaStreamNonBlocking, prio_hi));
    {  // the upward pass (start_prep): lowest priority by default, so the list
       // builder's blocks are dispatched first and the FP64 work fills in
      const char* v = std::getenv("SSUM_PREP_PRIO");
      const int pr = (v && *v == 'h') ? prio_hi : prio_lo;
      SSUM_CUDA_CHECK(cudaStreamCreateWithPriority(&c->prep_stream, cudaStreamNonBlocking, pr));
    }
    SSUM_CUDA_CHECK(cudaEventCreateWithFlags(&c->fork_ev, cudaEventDisableTiming));
    SSUM_CUDA_CHECK(cudaEventCreateWithFlags(&c->join_ev, cudaEventDisableTiming));
    for (auto& e : c->side_ev) SSUM_CUDA_CHECK(cudaEventCreate(&e));
    for (auto& e : c->leaf_ev) SSUM_CUDA_CHECK(cudaEventCreate(&e));
    SSUM_CUDA_CHECK(cudaEventCreateWithFlags(&c->prep_ev, cudaEventDisableTiming));
    if (const char* v = std::getenv("SSUM_OVERLAP_TILES")) c->overlap_tiles = std::atoi(v) != 0;
    if (const char* v = std::getenv("SSUM_EARLY_PREP")) c->early_prep = std::atoi(v) != 0;
    if (const char* v = std::getenv("SSUM_PLAN_LISTS")) c->plan_lists_ok = std::atoi(v) != 0;
    if (const char* v = std::getenv("SSUM_MAC_BAND")) c->mac.band = std::atof(v);
    for (auto& e : c->io.xyz) SSUM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : c->io.out) SSUM_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SSUM_CUDA_CHECK(cudaEventCreateWithFlags(&c->io.q, cudaEventDisableTiming));
    SSUM_CUDA_CHECK(cudaEventCreate(&c->io.t0));
    SSUM_CUDA_CHECK(cudaEventCreate(&c->io.t1));
    c->d_flags.ensure(64);
    SSUM_CUDA_CHECK(cudaMemset(c->d_flags.p, 0, 64 * sizeof(int)));
    ensure_log_table(*c);
    tree_init_roots(*c);
  } catch (const Error& e) {
    delete c;
    return e.code;
  } catch (...) {
    delete c;
    return SSUM_INTERNAL;
  }
  *out = reinterpret_cast<ssum_ctx*>(c);
  return SSUM_OK;
}

void ssum_destroy(ssum_ctx* h) {
  Ctx* c = reinterpret_cast<Ctx*>(h);
  if (!c) return;
  const int dev = c->device;
  cudaSetDevice(dev);
  cudaDeviceSynchronize();
  // device buffers (DBuf) free themselves when the context is deleted below
  for (auto& e : c->ev) cudaEventDestroy(e);
  for (auto& e : c->io.xyz) if (e) cudaEventDestroy(e);
  for (auto& e : c->io.out) if (e) cudaEventDestroy(e);
  if (c->io.q) cudaEventDestroy(c->io.q);
  if (c->io.t0) cudaEventDestroy(c->io.t0);
  if (c->io.t1) cudaEventDestroy(c->io.t1);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->side_stream) cudaStreamDestroy(c->side_stream);
  if (c->prep_stream) cudaStreamDestroy(c->prep_stream);
  if (c->fork_ev) cudaEventDestroy(c->fork_ev);
  if (c->join_ev) cudaEventDestroy(c->join_ev);
  for (auto& e : c->side_ev) if (e) cudaEventDestroy(e);
  for (auto& e : c->leaf_ev) if (e) cudaEventDestroy(e);
  if (c->prep_ev) cudaEventDestroy(c->prep_ev);
  if (c->bins.h_small) cudaFreeHost(c->bins.h_small);
  if (c->trav.h_small) cudaFreeHost(c->trav.h_small);
  if (c->trav.h_plan) cudaFreeHost(c->trav.h_plan);
  if (c->h_pinned) cudaFreeHost(c->h_pinned);
  dbuf_stream() = nullptr;  // the buffers go back to the pool in legacy-stream order
  cudaStream_t own = c->own_stream;
  delete c;
  cudaDeviceSynchronize();
  if (own) cudaStreamDestroy(own);
  (void)dev;  // the blocks stay cached in the device pool for the next context (ssum_trim_memory)
}

int ssum_trim_memory(int device) {
  cudaMemPool_t pool;
  if (cudaSetDevice(device) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return SSUM_CUDA;
  if (cudaDeviceGetDefaultMemPool(&pool, device) != cudaSuccess) return SSUM_CUDA;
  return cudaMemPoolTrimTo(pool, 0) == cudaSuccess ? SSUM_OK : SSUM_CUDA;
}

const char* ssum_last_error(const ssum_ctx* h) {
  const Ctx* c = reinterpret_cast<const Ctx*>(h);
  return c ? c->last_error.c_str() : "null context";
}

int ssum_set_stream(ssum_ctx* h, void* stream) {
  return guarded(h, [&](Ctx& c) { c.stream = stream ? static_cast<cudaStream_t>(stream) : c.own_stream; });
}

int ssum_set_partition(ssum_ctx* h, int part, int nparts) {
  return guarded(h, [&](Ctx& c) {
    if (nparts < 1 || part < 0 || part >= nparts) throw Error(SSUM_INVALID, "partition out of range");
    c.part = part;
    c.nparts = nparts;
  });
}

int ssum_partition_range(ssum_ctx* h, int64_t* begin, int64_t* end) {
  return guarded(h, [&](Ctx& c) {
    *begin = c.lists.p0;
    *end = c.lists.p1;
  });
}

int ssum_tree_perm(ssum_ctx* h, int* dst, int on_device) {
  return guarded(h, [&](Ctx& c) {
    const int64_t n = c.bins.n;
    if (n == 0) return;
    SSUM_CUDA_CHECK(cudaMemcpyAsync(dst, c.bins.perm.p, size_t(n) * 4,
                                    on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c.stream));
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int ssum_tree_reset(ssum_ctx* h) {
  return guarded(h, [&](Ctx& c) {
    c.call_index = 0;
    c.mac.keys.clear();
    c.mac.theta = -1.0;
    tree_init_roots(c);
  });
}

int ssum_treecode_sum_device(ssum_ctx* h, int kernel, const ssum_config* cfg, const double* d_xyz,
                             const double* d_q, int64_t n, double* d_out, ssum_stats* st) {
  return guarded(h, [&](Ctx& c) {
    validate(cfg);
    check_kernel(kernel);
    check_n(n);
    treecode_device(c, kernel, *cfg, d_xyz, d_q, n, d_out, st);
  });
}

// Host buffers in and out, with the copies overlapped with the work: xyz
// travels in kIoChunks pieces on copy_stream (the tree walk starts on each as
// it lands), then q (waited for at the gather); the result comes back piece by
// piece behind the downward pass (eval.cu). h2d/d2h_seconds: device time from
// the first input byte to the last, and from the first result piece to the
// last.
int ssum_treecode_sum(ssum_ctx* h, int kernel, const ssum_config* cfg, const double* xyz, const double* q,
                      int64_t n, double* out, ssum_stats* st) {
  return guarded(h, [&](Ctx& c) {
    validate(cfg);
    check_kernel(kernel);
    check_n(n);
    const int D = kernel == SSUM_BIOT_SAVART ? 3 : 1;
    c.in_xyz.ensure(std::max<size_t>(size_t(n) * 3, 1));
    c.in_q.ensure(std::max<size_t>(size_t(n), 1));
    c.out_buf.ensure(std::max<size_t>(size_t(n) * D, 1));
    Ctx::HostIo& io = c.io;
    struct Reset {  // the staged mode, and copies into the caller's buffers, never outlive this call
      Ctx& c;
      ~Reset() {
        cudaStreamSynchronize(c.copy_stream);
        c.io.active = false, c.io.h_out = nullptr;
      }
    } reset{c};
    // the copy stream must not overwrite inputs still read by earlier work
    SSUM_CUDA_CHECK(cudaEventRecord(io.t0, c.stream));
    SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, io.t0, 0));
    for (int j = 0; j <= Ctx::kIoChunks; ++j) io.bounds[j] = n * j / Ctx::kIoChunks;
    for (int j = 0; j < Ctx::kIoChunks; ++j) {
      const int64_t a = io.bounds[j], b = io.bounds[j + 1];
      if (b > a)
        SSUM_CUDA_CHECK(cudaMemcpyAsync(c.in_xyz.p + 3 * a, xyz + 3 * a, size_t(b - a) * 24, cudaMemcpyHostToDevice,
                                        c.copy_stream));
      SSUM_CUDA_CHECK(cudaEventRecord(io.xyz[j], c.copy_stream));
    }
    if (n) SSUM_CUDA_CHECK(cudaMemcpyAsync(c.in_q.p, q, size_t(n) * 8, cudaMemcpyHostToDevice, c.copy_stream));
    SSUM_CUDA_CHECK(cudaEventRecord(io.q, c.copy_stream));
    // A partitioned call computes only its part's rows; the others must come
    // back as the caller had them, so the device result starts as a copy of
    // the caller's buffer (unpartitioned calls overwrite every row).
    if (c.nparts > 1 && n)
      SSUM_CUDA_CHECK(cudaMemcpyAsync(c.out_buf.p, out, size_t(n) * D * 8, cudaMemcpyHostToDevice, c.stream));
    io.active = true;
    io.h_out = out;
    io.dim = D;
    treecode_device(c, kernel, *cfg, c.in_xyz.p, c.in_q.p, n, c.out_buf.p, st);
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.copy_stream));
    if (st) {
      float ms = 0.0f;
      if (cudaEventElapsedTime(&ms, io.t0, io.t1) == cudaSuccess) st->d2h_seconds += ms * 1e-3;
    }
  });
}

int ssum_direct_sum_device(ssum_ctx* h, int kernel, const double* d_xyz, const double* d_q, int64_t n,
                           double* d_out) {
  return guarded(h, [&](Ctx& c) {
    check_kernel(kernel);
    check_n(n);
    direct_sum_device(c, kernel, d_xyz, d_q, n, d_out);
  });
}

int ssum_direct_sum(ssum_ctx* h, int kernel, const double* xyz, const double* q, int64_t n, double* out) {
  return guarded(h, [&](Ctx& c) {
    check_kernel(kernel);
    check_n(n);
    const int D = kernel == SSUM_BIOT_SAVART ? 3 : 1;
    upload(c, c.in_xyz, xyz, size_t(n) * 3, nullptr);
    upload(c, c.in_q, q, size_t(n), nullptr);
    c.out_buf.ensure(std::max<size_t>(size_t(n) * D, 1));
    direct_sum_device(c, kernel, c.in_xyz.p, c.in_q.p, n, c.out_buf.p);
    download(c, out, c.out_buf.p, size_t(n) * D, nullptr);
  });
}

int ssum_bin_particles(ssum_ctx* h, const double* xyz, int64_t n, int n_threshold, int max_depth) {
  return guarded(h, [&](Ctx& c) {
    check_n(n);
    if (n_threshold < 1) throw Error(SSUM_CONFIG, "n_threshold must be >= 1");
    if (max_depth < 1 || max_depth > 40) throw Error(SSUM_CONFIG, "max_depth must be in [1, 40]");
    upload(c, c.in_xyz, xyz, size_t(n) * 3, nullptr);
    tree_bin(c, c.in_xyz.p, n, n_threshold, max_depth);
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
  });
}

int ssum_tree_node_count(ssum_ctx* h, int* count) {
  return guarded(h, [&](Ctx& c) { *count = c.nodes.count; });
}

int ssum_tree_export(ssum_ctx* h, int* level, int* parent, int* child_base, double* tri, double* center,
                     double* radius, int64_t* bin_offsets, int* bin_ids, int* leaf_of) {
  return guarded(h, [&](Ctx& c) {
    const HostTree& t = host_tree(c);
    const int nn = c.nodes.count;
    const std::vector<int> ref = reference_ids(t);
    std::vector<int> dev_of(static_cast<size_t>(nn));
    for (int d = 0; d < nn; ++d) dev_of[ref[d]] = d;
    for (int r = 0; r < nn; ++r) {
      const int d = dev_of[r];
      if (level) level[r] = t.level[d];
      if (parent) parent[r] = t.parent[d] < 0 ? -1 : ref[t.parent[d]];
      if (child_base) child_base[r] = t.child_base[d] < 0 ? -1 : ref[t.child_base[d]];
    }
    auto fetch = [&](double* dst, const double* src, int w) {
      if (!dst) return;
      std::vector<double> tmp(size_t(nn) * w);
      SSUM_CUDA_CHECK(cudaMemcpyAsync(tmp.data(), src, tmp.size() * 8, cudaMemcpyDeviceToHost, c.stream));
      SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
      for (int r = 0; r < nn; ++r) std::memcpy(dst + size_t(r) * w, tmp.data() + size_t(dev_of[r]) * w, size_t(w) * 8);
    };
    fetch(tri, c.nodes.tri.p, 9);
    fetch(center, c.nodes.center.p, 3);
    fetch(radius, c.nodes.radius.p, 1);
    const int64_t n = c.bins.n;
    if (bin_offsets || bin_ids || leaf_of) {
      std::vector<int> perm(static_cast<size_t>(n)), lf(static_cast<size_t>(n));
      if (n) {
        SSUM_CUDA_CHECK(cudaMemcpyAsync(perm.data(), c.bins.perm.p, size_t(n) * 4, cudaMemcpyDeviceToHost, c.stream));
        SSUM_CUDA_CHECK(cudaMemcpyAsync(lf.data(), c.bins.leaf_of.p, size_t(n) * 4, cudaMemcpyDeviceToHost, c.stream));
      }
      SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
      if (leaf_of)
        for (int64_t i = 0; i < n; ++i) leaf_of[i] = ref[lf[size_t(i)]];
      int64_t o = 0;
      for (int r = 0; r < nn; ++r) {
        const int d = dev_of[r];
        const int cnt = d < static_cast<int>(t.cnt.size()) ? t.cnt[d] : 0;
        if (bin_offsets) bin_offsets[r] = o;
        if (bin_ids && cnt > 0) {
          std::copy(perm.begin() + t.off[d], perm.begin() + t.off[d] + cnt, bin_ids + o);
          std::sort(bin_ids + o, bin_ids + o + cnt);  // TreeNode::bin is ascending
        }
        o += cnt;
      }
      if (bin_offsets) bin_offsets[nn] = o;
    }
  });
}

int ssum_dual_traversal(ssum_ctx* h, const ssum_config* cfg, int* tsk, int64_t cap, int64_t* count) {
  return guarded(h, [&](Ctx& c) {
    validate(cfg);
    traverse_and_build_lists(c, *cfg, true);
    std::vector<int4> list;
    sorted_interactions(c, list);
    const std::vector<int> ref = reference_ids(host_tree(c));
    *count = static_cast<int64_t>(list.size());
    const int64_t m = std::min<int64_t>(cap, *count);
    for (int64_t e = 0; e < m; ++e) {
      tsk[3 * e] = ref[list[size_t(e)].x];
      tsk[3 * e + 1] = ref[list[size_t(e)].y];
      tsk[3 * e + 2] = list[size_t(e)].z;
    }
  });
}

// eval_pp / eval_pc / eval_cp / eval_cc: O(|t| |s|) on the device (eval.cu
// eval_interaction); only the two bins' rows of the caller's arrays are read
// and only the target bin's rows of field are updated.
int ssum_eval_interaction(ssum_ctx* h, int kernel, const ssum_config* cfg, const double* xyz, const double* q,
                          int64_t n, int target, int source, int kind, double* field) {
  return guarded(h, [&](Ctx& c) {
    validate(cfg);
    check_kernel(kernel);
    check_n(n);
    if (n != c.bins.n) throw Error(SSUM_INVALID, "eval_interaction: positions do not match the binned tree");
    if (kind < 0 || kind > 3) throw Error(SSUM_INVALID, "eval_interaction: unknown interaction kind");
    if (n == 0) return;
    const int tdev = dev_node(c, target), sdev = dev_node(c, source);
    eval_interaction(c, kernel, cfg->degree, xyz, q, tdev, sdev, kind, field);
  });
}

int ssum_compute_proxy_weights(ssum_ctx* h, int degree, const double* xyz, const double* q, int64_t n,
                               int source_node, double* w) {
  return guarded(h, [&](Ctx& c) {
    if (degree < 1 || degree > kMaxDegree) throw Error(SSUM_INVALID, "SBB degree must be in [1, 20]");
    check_n(n);
    if (n != c.bins.n) throw Error(SSUM_INVALID, "compute_proxy_weights: positions do not match the binned tree");
    const int P = (degree + 1) * (degree + 2) / 2;
    if (n == 0) {
      std::fill(w, w + P, 0.0);
      return;
    }
    proxy_weights(c, degree, xyz, q, dev_node(c, source_node), w);
  });
}

double ssum_last_rcond(const ssum_ctx* h) {
  const Ctx* c = reinterpret_cast<const Ctx*>(h);
  return c ? c->last_rcond : 0.0;
}

int ssum_lattice_fit(int degree, double* vinv, double* rcond) {
  try {
    if (degree < 1 || degree > kMaxDegree) return SSUM_INVALID;
    std::vector<double> inv;
    double rc = 0.0;
    lattice_inverse(degree, inv, rc);
    if (rcond) *rcond = rc;
    if (vinv) std::copy(inv.begin(), inv.end(), vinv);
    return rc > 1e-12 ? SSUM_OK : SSUM_CONDITIONING;
  } catch (...) {
    return SSUM_INTERNAL;
  }
}

int ssum_proxy_points(const double* tri, int degree, double* pts) {
  if (!tri || !pts || degree < 1 || degree > kMaxDegree) return SSUM_INVALID;
  const double d = static_cast<double>(degree);
  int m = 0;
  for (int kk = 0; kk <= degree; ++kk)
    for (int jj = 0; jj <= degree - kk; ++jj, ++m) {
      const int ii = degree - kk - jj;
      const double b1 = ii / d, b2 = jj / d, b3 = kk / d;
      const d3 v{add_rn(add_rn(mul_rn(tri[0], b1), mul_rn(tri[3], b2)), mul_rn(tri[6], b3)),
                 add_rn(add_rn(mul_rn(tri[1], b1), mul_rn(tri[4], b2)), mul_rn(tri[7], b3)),
                 add_rn(add_rn(mul_rn(tri[2], b1), mul_rn(tri[5], b2)), mul_rn(tri[8], b3))};
      int bad = 0;
      const d3 u = unit_rn(v, &bad);
      if (bad) return SSUM_GEOMETRY;
      pts[3 * m] = u.x;
      pts[3 * m + 1] = u.y;
      pts[3 * m + 2] = u.z;
    }
  return SSUM_OK;
}

int ssum_rk4(ssum_ctx* h, const ssum_config* cfg, double* xyz, double* zeta, const double* area, int64_t n,
             double dt, int steps, double omega, int direct, ssum_stats* st) {
  return guarded(h, [&](Ctx& c) {
    validate(cfg);
    check_n(n);
    if (n == 0 || steps <= 0) return;
    const size_t N = size_t(n);
    // state layout in rk_state: x0 3N | z0 N | area N | xs 3N | q N | u 3N | k 3N | kz N | acc 3N | accz N
    c.rk_state.ensure(N * 20);
    double* x0 = c.rk_state.p;
    double* z0 = x0 + 3 * N;
    double* ar = z0 + N;
    double* xs = ar + N;
    double* q = xs + 3 * N;
    double* u = q + N;
    double* k = u + 3 * N;
    double* kz = k + 3 * N;
    double* acc = kz + N;
    double* accz = acc + 3 * N;
    const double cs[4] = {0.0, 0.5 * dt, 0.5 * dt, dt};
    const int bs = 256;
    // Inputs on the copy stream, overlapped with the first evaluation as in
    // ssum_treecode_sum: x in kIoChunks pieces (the first stage's tree walk
    // starts on each as it lands), then zeta and A and, still on the copy
    // stream, the first stage's q = zeta A (waited for at the gather). The
    // first stage evaluates at x0 itself (its stage positions are x0 bit for
    // bit). The direct-sum driver takes the plain path.
    Ctx::HostIo& io = c.io;
    struct Reset {
      Ctx& c;
      ~Reset() {
        cudaStreamSynchronize(c.copy_stream);
        c.io.active = false, c.io.h_out = nullptr;
      }
    } reset{c};
    SSUM_CUDA_CHECK(cudaEventRecord(io.t0, c.stream));
    SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, io.t0, 0));
    for (int j = 0; j <= Ctx::kIoChunks; ++j) io.bounds[j] = n * j / Ctx::kIoChunks;
    for (int j = 0; j < Ctx::kIoChunks; ++j) {
      const int64_t a = io.bounds[j], b = io.bounds[j + 1];
      if (b > a)
        SSUM_CUDA_CHECK(cudaMemcpyAsync(x0 + 3 * a, xyz + 3 * a, size_t(b - a) * 24, cudaMemcpyHostToDevice,
                                        c.copy_stream));
      SSUM_CUDA_CHECK(cudaEventRecord(io.xyz[j], c.copy_stream));
    }
    SSUM_CUDA_CHECK(cudaMemcpyAsync(z0, zeta, N * 8, cudaMemcpyHostToDevice, c.copy_stream));
    SSUM_CUDA_CHECK(cudaMemcpyAsync(ar, area, N * 8, cudaMemcpyHostToDevice, c.copy_stream));
    k_rk4_q<<<grid_for(n, bs), bs, 0, c.copy_stream>>>(n, z0, ar, q);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    SSUM_CUDA_CHECK(cudaEventRecord(io.q, c.copy_stream));
    if (direct) {
      SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, io.q, 0));  // everything landed
    } else {
      io.active = true;
      io.h_out = nullptr;
      io.dim = 3;
    }
    for (int step = 0; step < steps; ++step) {
      // Each stage's accumulation is fused with the next stage's positions
      // and strengths (k_rk4_advance_rows on the caller-order velocities,
      // bitwise k_rk4_accum + k_rk4_stage); a geometry error it flags is
      // raised by the next evaluation's check (or the step's).
      for (int s = 0; s < 4; ++s) {
        if (s == 0) SSUM_CUDA_CHECK(cudaMemsetAsync(c.d_flags.p, 0, 4, c.stream));
        if (io.active) {  // first stage of the call: x0 and q as they land
          treecode_device(c, SSUM_BIOT_SAVART, *cfg, x0, q, n, u, st);
          SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.stream, io.q, 0));  // zeta and A for the next stages
          io.active = false;
        } else {
          if (s == 0) {  // stage 0 of a step: xs = x0, q = zeta A
            k_rk4_stage<<<grid_for(n, bs), bs, 0, c.stream>>>(n, 0, 0.0, x0, z0, ar, k, kz, xs, q, c.d_flags.p);
            SSUM_LAUNCH_CHECK();
            c.launches++;
          }
          if (direct)
            direct_sum_device(c, SSUM_BIOT_SAVART, xs, q, n, u);
          else
            treecode_device(c, SSUM_BIOT_SAVART, *cfg, xs, q, n, u, st);
        }
        k_rk4_advance_rows<<<grid_for(n, bs), bs, 0, c.stream>>>(n, s, omega, s < 3 ? cs[s + 1] : -1.0, u, 0,
                                                                 nullptr, 1, nullptr, x0, z0, ar, acc, accz,
                                                                 nullptr, nullptr, xs, q, c.d_flags.p);
        SSUM_LAUNCH_CHECK();
        c.launches++;
      }
      if (step + 1 < steps) {
        k_rk4_final<<<grid_for(n, bs), bs, 0, c.stream>>>(0, n, dt / 6.0, x0, z0, acc, accz, c.d_flags.p);
        SSUM_LAUNCH_CHECK();
        c.launches++;
        check_flags(c, "rk4");
        continue;
      }
      // last step: the final update in pieces, each piece's copy to the host
      // overlapping the next piece's update
      for (int j = 0; j < Ctx::kIoChunks; ++j) {
        const int64_t a = io.bounds[j], b = io.bounds[j + 1];
        if (b > a) {
          k_rk4_final<<<grid_for(b - a, bs), bs, 0, c.stream>>>(a, b, dt / 6.0, x0, z0, acc, accz, c.d_flags.p);
          SSUM_LAUNCH_CHECK();
          c.launches++;
        }
        SSUM_CUDA_CHECK(cudaEventRecord(io.out[j], c.stream));
        SSUM_CUDA_CHECK(cudaStreamWaitEvent(c.copy_stream, io.out[j], 0));
        if (b > a) {
          SSUM_CUDA_CHECK(cudaMemcpyAsync(xyz + 3 * a, x0 + 3 * a, size_t(b - a) * 24, cudaMemcpyDeviceToHost,
                                          c.copy_stream));
          SSUM_CUDA_CHECK(cudaMemcpyAsync(zeta + a, z0 + a, size_t(b - a) * 8, cudaMemcpyDeviceToHost,
                                          c.copy_stream));
        }
      }
      check_flags(c, "rk4");
    }
    SSUM_CUDA_CHECK(cudaStreamSynchronize(c.copy_stream));
  });
}

// The three pieces of ssum_rk4's step, for drivers that evaluate the stage
// velocities themselves (the multi-GPU driver: partitioned evaluation + one
// all-gather per stage). Same kernels, so a driver built from them matches
// ssum_rk4 bit for bit. Device pointers, the context's stream.
int ssum_rk4_stage_begin(ssum_ctx* h, int stage, double dt, int64_t n, const double* d_x0, const double* d_z0,
                         const double* d_area, const double* d_k, const double* d_kz, double* d_xs, double* d_q) {
  return guarded(h, [&](Ctx& c) {
    check_n(n);
    if (stage < 0 || stage > 3) throw Error(SSUM_INVALID, "RK4 stage must be 0..3");
    if (n == 0) return;
    const double cs[4] = {0.0, 0.5 * dt, 0.5 * dt, dt};
    k_rk4_stage<<<grid_for(n, 256), 256, 0, c.stream>>>(n, stage, cs[stage], d_x0, d_z0, d_area, d_k, d_kz, d_xs,
                                                        d_q, c.d_flags.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  });
}

int ssum_rk4_stage_end(ssum_ctx* h, int stage, double omega, int64_t n, const double* d_u, double* d_k, double* d_kz,
                       double* d_acc, double* d_accz) {
  return guarded(h, [&](Ctx& c) {
    check_n(n);
    if (stage < 0 || stage > 3) throw Error(SSUM_INVALID, "RK4 stage must be 0..3");
    if (n == 0) return;
    k_rk4_accum<<<grid_for(n, 256), 256, 0, c.stream>>>(n, stage, omega, d_u, d_k, d_kz, d_acc, d_accz);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  });
}

int ssum_bin_walk_shard(ssum_ctx* h, const double* d_xyz, int64_t n, int64_t i0, int64_t i1, int64_t slots,
                        void** keys, void** leaf_of, int* walked) {
  return guarded(h, [&](Ctx& c) {
    check_n(n);
    if (i0 < 0 || i1 < i0 || i1 > n || slots < n) throw Error(SSUM_INVALID, "bin_walk_shard: bad shard");
    *walked = tree_walk_shard(c, d_xyz, n, i0, i1, slots) ? 1 : 0;
    *keys = c.bins.wkey.p;
    *leaf_of = c.bins.leaf_of.p;
    if (*walked) {
      // a particle in no root face: the same GeometryError as the binning
      if (!c.h_pinned) SSUM_CUDA_CHECK(cudaMallocHost(&c.h_pinned, 64 * sizeof(int)));
      SSUM_CUDA_CHECK(cudaMemcpyAsync(c.h_pinned + 1, c.d_flags.p, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
      SSUM_CUDA_CHECK(cudaStreamSynchronize(c.stream));
      const int f = c.h_pinned[1];
      if (f & kFlagGeometry) {
        c.bins.walked_n = -1;
        throw Error(SSUM_GEOMETRY, "bin_particles: particle contained in no root face");
      }
    }
  });
}

int ssum_set_output_order(ssum_ctx* h, int tree_order) {
  return guarded(h, [&](Ctx& c) { c.out_tree_order = tree_order != 0; });
}

int ssum_partition_cuts(ssum_ctx* h, int64_t* cuts) {
  return guarded(h, [&](Ctx& c) {
    if (c.part_pos.empty()) throw Error(SSUM_INVALID, "partition_cuts: no evaluation yet");
    for (size_t r = 0; r < c.part_pos.size(); ++r) cuts[r] = c.part_pos[r];
  });
}

int ssum_rk4_stage_end_rows(ssum_ctx* h, int stage, double omega, int64_t n, const double* d_rows, int64_t width,
                            double* d_k, double* d_kz, double* d_acc, double* d_accz) {
  return guarded(h, [&](Ctx& c) {
    check_n(n);
    if (stage < 0 || stage > 3) throw Error(SSUM_INVALID, "RK4 stage must be 0..3");
    if (n == 0) return;
    if (n != c.bins.n || int64_t(c.part_pos.size()) != c.nparts + 1 || c.part_pos.back() != n)
      throw Error(SSUM_INVALID, "rk4_stage_end_rows: no partitioned evaluation of these particles");
    const int np = c.nparts;
    for (int r = 0; r < np; ++r)
      if (c.part_pos[size_t(r) + 1] - c.part_pos[size_t(r)] > width)
        throw Error(SSUM_INVALID, "rk4_stage_end_rows: a part has more rows than the slot width");
    c.cut_dev.ensure(size_t(np) + 1);
    SSUM_CUDA_CHECK(cudaMemcpyAsync(c.cut_dev.p, c.part_pos.data(), (size_t(np) + 1) * 8, cudaMemcpyHostToDevice,
                                    c.stream));
    k_rk4_accum_rows<<<grid_for(n, 256), 256, 0, c.stream>>>(n, stage, omega, d_rows, width, c.cut_dev.p, np,
                                                             c.bins.perm.p, d_k, d_kz, d_acc, d_accz);
    SSUM_LAUNCH_CHECK();
    c.launches++;
  });
}

int ssum_rk4_stage_advance_rows(ssum_ctx* h, int stage, double dt, double omega, int64_t n, const double* d_rows,
                                int64_t width, const double* d_x0, const double* d_z0, const double* d_area,
                                double* d_k, double* d_kz, double* d_acc, double* d_accz, double* d_xs, double* d_q) {
  return guarded(h, [&](Ctx& c) {
    check_n(n);
    if (stage < 0 || stage > 3) throw Error(SSUM_INVALID, "RK4 stage must be 0..3");
    if ((d_k == nullptr) != (d_kz == nullptr)) throw Error(SSUM_INVALID, "rk4_stage_advance_rows: k and kz together");
    if (stage < 3 && (!d_x0 || !d_z0 || !d_area || !d_xs || !d_q))
      throw Error(SSUM_INVALID, "rk4_stage_advance_rows: the next stage needs x0, z0, area, xs, q");
    if (n == 0) return;
    if (n != c.bins.n || c.bins.perm_n != n || int64_t(c.part_pos.size()) != c.nparts + 1 || c.part_pos.back() != n)
      throw Error(SSUM_INVALID, "rk4_stage_advance_rows: no partitioned evaluation of these particles");
    const int np = c.nparts;
    for (int r = 0; r < np; ++r)
      if (c.part_pos[size_t(r) + 1] - c.part_pos[size_t(r)] > width)
        throw Error(SSUM_INVALID, "rk4_stage_advance_rows: a part has more rows than the slot width");
    c.cut_dev.ensure(size_t(np) + 1);
    SSUM_CUDA_CHECK(cudaMemcpyAsync(c.cut_dev.p, c.part_pos.data(), (size_t(np) + 1) * 8, cudaMemcpyHostToDevice,
                                    c.stream));
    c.inv_perm.ensure(size_t(n));
    k_inv_of<<<grid_for(n, 256), 256, 0, c.stream>>>(c.bins.perm.p, n, c.inv_perm.p);
    SSUM_LAUNCH_CHECK();
    const double cs_next[4] = {0.5 * dt, 0.5 * dt, dt, -1.0};  // stage + 1's offset (none after stage 3)
    k_rk4_advance_rows<<<grid_for(n, 256), 256, 0, c.stream>>>(
        n, stage, omega, cs_next[stage], d_rows, width, c.cut_dev.p, np, c.inv_perm.p, d_x0, d_z0, d_area, d_acc,
        d_accz, d_k, d_kz, d_xs, d_q, c.d_flags.p);
    SSUM_LAUNCH_CHECK();
    c.launches += 2;
  });
}

int ssum_rk4_step_end(ssum_ctx* h, double dt, int64_t n, double* d_x0, double* d_z0, const double* d_acc,
                      const double* d_accz) {
  return guarded(h, [&](Ctx& c) {
    check_n(n);
    if (n == 0) return;
    k_rk4_final<<<grid_for(n, 256), 256, 0, c.stream>>>(0, n, dt / 6.0, d_x0, d_z0, d_acc, d_accz, c.d_flags.p);
    SSUM_LAUNCH_CHECK();
    c.launches++;
    check_flags(c, "rk4");
  });
}

}  // extern "C"
