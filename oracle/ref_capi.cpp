// ORACLE TEST INFRASTRUCTURE — not product code. Only tests/, smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load what this builds.
//
// extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj/src/*.cpp, compiled by oracle/Makefile into
// oracle/_ref/libspheresum_ref.so) so Python tests can call the reference's own
// treecode_sum / direct_sum / dual_traversal / FaceTree / make_icosa_mesh.
//
// Also holds the one piece of CPU driver logic the reference lacks but
// BASELINE config 4 needs: a classical RK4 stepper restated from
// SPEC.md:530-547 (+ design decisions SPEC.md:584,587) on top of the
// reference's own treecode_sum<BiotSavartKernel> (treecode.cpp:266-413).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "spheresum/errors.hpp"
#include "spheresum/face_tree.hpp"
#include "spheresum/geometry.hpp"
#include "spheresum/icosa_mesh.hpp"
#include "spheresum/kernels.hpp"
#include "spheresum/sbb.hpp"
#include "spheresum/treecode.hpp"

using namespace spheresum;

namespace {

thread_local std::string g_err;

enum RefStatus : int {
  kOk = 0,
  kConfig = 1,
  kGeometry = 2,
  kSingular = 3,
  kConditioning = 4,
  kInvalid = 5,
  kOther = 9,
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return kOk;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return kConfig;
  } catch (const GeometryError& e) {
    g_err = e.what();
    return kGeometry;
  } catch (const SingularKernelError& e) {
    g_err = e.what();
    return kSingular;
  } catch (const ConditioningError& e) {
    g_err = e.what();
    return kConditioning;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return kInvalid;
  } catch (const std::exception& e) {
    g_err = e.what();
    return kOther;
  }
}

// The caller's doubles ARE the UnitVector3 values (no renormalisation: a
// second normalisation is not bitwise idempotent). Callers pass unit vectors.
std::vector<UnitVector3> to_points(const double* xyz, int64_t n) {
  std::vector<UnitVector3> p(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    p[i].x = xyz[3 * i];
    p[i].y = xyz[3 * i + 1];
    p[i].z = xyz[3 * i + 2];
  }
  return p;
}

TraversalConfig make_cfg(double theta, int nt, int degree, int max_depth) {
  TraversalConfig c;
  c.theta = theta;
  c.n_threshold = nt;
  c.degree = degree;
  c.max_depth = max_depth;
  return c;
}

template <class K>
void run_treecode(const std::vector<UnitVector3>& pts, const std::vector<double>& q,
                  const TraversalConfig& cfg, FaceTree& tree, int workers, double* out,
                  double* stats) {
  TreecodeStats st;
  const auto f = treecode_sum<K>(pts, q, cfg, tree, workers, &st);
  for (size_t i = 0; i < f.size(); ++i)
    for (int d = 0; d < K::dim; ++d) out[i * K::dim + d] = f[i][d];
  if (stats) {
    stats[0] = st.bin_seconds;
    stats[1] = st.traversal_seconds;
    stats[2] = st.eval_seconds;
    for (int k = 0; k < 4; ++k) stats[3 + k] = static_cast<double>(st.interaction_counts[k]);
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- mesh fixtures (icosa_mesh.cpp:129-133, :75-106) -----------------------
int64_t ref_mesh_vertex_count(int level) { return 10 * (int64_t(1) << (2 * level)) + 2; }

int ref_make_mesh(int level, double* xyz, double* area) {
  return guarded([&] {
    const IcosaMesh m = make_icosa_mesh(level);
    const auto& v = m.vertices();
    for (size_t i = 0; i < v.size(); ++i) {
      xyz[3 * i] = v[i].x;
      xyz[3 * i + 1] = v[i].y;
      xyz[3 * i + 2] = v[i].z;
    }
    if (area) {
      const auto a = m.node_patch_areas();
      std::memcpy(area, a.data(), a.size() * sizeof(double));
    }
  });
}

// --- summation (treecode.cpp:246-264, :266-413) -----------------------------
// kernel: 0 = BiotSavartKernel (dim 3), 1 = LogPotentialKernel (dim 1)
int ref_direct_sum(int kernel, const double* xyz, const double* q, int64_t n, double* out) {
  return guarded([&] {
    const auto pts = to_points(xyz, n);
    const std::vector<double> s(q, q + n);
    if (kernel == 0) {
      const auto f = direct_sum<BiotSavartKernel>(pts, s);
      for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < 3; ++d) out[3 * i + d] = f[i][d];
    } else {
      const auto f = direct_sum<LogPotentialKernel>(pts, s);
      for (int64_t i = 0; i < n; ++i) out[i] = f[i][0];
    }
  });
}

int ref_treecode_sum(int kernel, const double* xyz, const double* q, int64_t n, double theta,
                     int nt, int degree, int max_depth, int workers, double* out,
                     double* stats) {
  return guarded([&] {
    const auto pts = to_points(xyz, n);
    const std::vector<double> s(q, q + n);
    const TraversalConfig cfg = make_cfg(theta, nt, degree, max_depth);
    FaceTree tree;
    if (kernel == 0)
      run_treecode<BiotSavartKernel>(pts, s, cfg, tree, workers, out, stats);
    else
      run_treecode<LogPotentialKernel>(pts, s, cfg, tree, workers, out, stats);
  });
}

// Reference velocity for a bounded subset of targets under the full tree code:
// used by bench.py's cpu_baseline leg is NOT this (it runs the whole
// treecode_sum); this helper only exists for tests that want the reference's
// proxy-fit constants.
int ref_lattice_fit_rcond(int degree, double* rcond) {
  return guarded([&] { *rcond = lattice_fit(degree).rcond(); });
}

// --- persistent FaceTree handle (face_tree.hpp:36-58) -----------------------
void* ref_tree_new() {
  try {
    return new FaceTree();
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void ref_tree_free(void* h) { delete static_cast<FaceTree*>(h); }

int ref_tree_bin(void* h, const double* xyz, int64_t n, int nt, int max_depth) {
  return guarded([&] {
    static_cast<FaceTree*>(h)->bin_particles(to_points(xyz, n), nt, max_depth);
  });
}

int ref_tree_node_count(void* h) { return static_cast<FaceTree*>(h)->node_count(); }

// Per node: level, parent, child_base, bin size, vertices (9), circumcenter (3),
// radius. Any output pointer may be null.
int ref_tree_nodes(void* h, int* level, int* parent, int* child_base, int* bin_size, double* tri,
                   double* center, double* radius) {
  return guarded([&] {
    const FaceTree& t = *static_cast<FaceTree*>(h);
    for (int id = 0; id < t.node_count(); ++id) {
      const TreeNode& nd = t.node(id);
      if (level) level[id] = nd.level;
      if (parent) parent[id] = nd.parent;
      if (child_base) child_base[id] = nd.child_base;
      if (bin_size) bin_size[id] = nd.size();
      if (tri) {
        const UnitVector3* v[3] = {&nd.triangle.v1, &nd.triangle.v2, &nd.triangle.v3};
        for (int k = 0; k < 3; ++k) {
          tri[9 * id + 3 * k] = v[k]->x;
          tri[9 * id + 3 * k + 1] = v[k]->y;
          tri[9 * id + 3 * k + 2] = v[k]->z;
        }
      }
      if (center) {
        center[3 * id] = nd.circumcenter.x;
        center[3 * id + 1] = nd.circumcenter.y;
        center[3 * id + 2] = nd.circumcenter.z;
      }
      if (radius) radius[id] = nd.radius;
    }
  });
}

// Concatenated bins (ascending ids per node) with offsets[node_count+1].
int ref_tree_bins(void* h, int64_t* offsets, int* ids) {
  return guarded([&] {
    const FaceTree& t = *static_cast<FaceTree*>(h);
    int64_t off = 0;
    for (int id = 0; id < t.node_count(); ++id) {
      offsets[id] = off;
      const auto& b = t.node(id).bin;
      if (ids) std::memcpy(ids + off, b.data(), b.size() * sizeof(int));
      off += static_cast<int64_t>(b.size());
    }
    offsets[t.node_count()] = off;
  });
}

int ref_tree_leaf_of(void* h, int64_t n, int* leaf) {
  return guarded([&] {
    const FaceTree& t = *static_cast<FaceTree*>(h);
    for (int64_t i = 0; i < n; ++i) leaf[i] = t.leaf_of_particle(static_cast<int>(i));
  });
}

// dual_traversal (treecode.cpp:69-77) on an already-binned tree. Writes up to
// `cap` (target, source, kind) triples; returns the total count via *count.
int ref_dual_traversal(void* h, double theta, int nt, int degree, int max_depth, int* tsk,
                       int64_t cap, int64_t* count) {
  return guarded([&] {
    const FaceTree& t = *static_cast<FaceTree*>(h);
    const auto list = dual_traversal(t, t, make_cfg(theta, nt, degree, max_depth));
    *count = static_cast<int64_t>(list.size());
    const int64_t m = std::min<int64_t>(cap, *count);
    for (int64_t i = 0; i < m; ++i) {
      tsk[3 * i] = list[i].target;
      tsk[3 * i + 1] = list[i].source;
      tsk[3 * i + 2] = static_cast<int>(list[i].kind);
    }
  });
}

// treecode_sum on a caller-held (possibly reused) FaceTree.
int ref_treecode_sum_tree(void* h, int kernel, const double* xyz, const double* q, int64_t n,
                          double theta, int nt, int degree, int max_depth, int workers,
                          double* out, double* stats) {
  return guarded([&] {
    const auto pts = to_points(xyz, n);
    const std::vector<double> s(q, q + n);
    const TraversalConfig cfg = make_cfg(theta, nt, degree, max_depth);
    FaceTree& tree = *static_cast<FaceTree*>(h);
    if (kernel == 0)
      run_treecode<BiotSavartKernel>(pts, s, cfg, tree, workers, out, stats);
    else
      run_treecode<LogPotentialKernel>(pts, s, cfg, tree, workers, out, stats);
  });
}

// eval_pp / eval_pc / eval_cp / eval_cc (treecode.cpp:170-244) on a binned
// reference tree: adds raw sums into field (N x D).
int ref_eval_interaction(void* h, int kernel, const double* xyz, const double* q, int64_t n, double theta, int nt,
                         int degree, int max_depth, int target, int source, int kind, double* field) {
  return guarded([&] {
    const FaceTree& tree = *static_cast<FaceTree*>(h);
    const auto pts = to_points(xyz, n);
    const std::vector<double> s(q, q + n);
    const TraversalConfig cfg = make_cfg(theta, nt, degree, max_depth);
    Interaction it;
    it.target = target;
    it.source = source;
    it.kind = static_cast<InteractionKind>(kind);
    auto run = [&](auto tag) {
      using K = decltype(tag);
      PotentialField<K::dim> f(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < K::dim; ++d) f[i][d] = field[i * K::dim + d];
      if (kind == 0)
        eval_pp<K>(tree, it, pts, s, f);
      else if (kind == 1)
        eval_pc<K>(tree, it, pts, s, cfg, f);
      else if (kind == 2)
        eval_cp<K>(tree, it, pts, s, cfg, f);
      else
        eval_cc<K>(tree, it, pts, s, cfg, f);
      for (int64_t i = 0; i < n; ++i)
        for (int d = 0; d < K::dim; ++d) field[i * K::dim + d] = f[i][d];
    };
    if (kernel == 0)
      run(BiotSavartKernel{});
    else
      run(LogPotentialKernel{});
  });
}

// compute_proxy_weights (treecode.cpp:79-91) of one node of a binned tree.
int ref_compute_proxy_weights(void* h, int degree, const double* xyz, const double* q, int64_t n, int node,
                              double* w) {
  return guarded([&] {
    const FaceTree& tree = *static_cast<FaceTree*>(h);
    const auto pts = to_points(xyz, n);
    const std::vector<double> s(q, q + n);
    const SBBBasis basis(degree);
    const std::vector<double> r = compute_proxy_weights(tree, node, basis, pts, s);
    std::memcpy(w, r.data(), r.size() * sizeof(double));
  });
}

// --- SBB / geometry probes used by the KAT tests ---------------------------
int ref_sbb_eval(int degree, double b1, double b2, double b3, double* out) {
  return guarded([&] { SBBBasis(degree).eval({b1, b2, b3}, out); });
}

int ref_proxy_points(const double* tri9, int degree, double* pts) {
  return guarded([&] {
    const SphericalTriangle t(UnitVector3(tri9[0], tri9[1], tri9[2]),
                              UnitVector3(tri9[3], tri9[4], tri9[5]),
                              UnitVector3(tri9[6], tri9[7], tri9[8]));
    const auto set = proxy_points(t, degree);
    for (size_t m = 0; m < set.points.size(); ++m) {
      pts[3 * m] = set.points[m].x;
      pts[3 * m + 1] = set.points[m].y;
      pts[3 * m + 2] = set.points[m].z;
    }
  });
}

// V^-1 applied to the identity (column-major p x p), through the reference's
// lattice_fit(d).solve (sbb.cpp:103-108,124-138).
int ref_lattice_inverse(int degree, double* inv) {
  return guarded([&] {
    const ProxyFit& f = lattice_fit(degree);
    const int p = f.size();
    std::vector<double> eye(static_cast<size_t>(p) * p, 0.0);
    for (int i = 0; i < p; ++i) eye[static_cast<size_t>(i) * p + i] = 1.0;
    f.solve(eye.data(), inv, p);
  });
}

int ref_kernel_eval(int kernel, const double* x, const double* y, double* out) {
  return guarded([&] {
    const UnitVector3 a(x[0], x[1], x[2]), b(y[0], y[1], y[2]);
    if (kernel == 0)
      BiotSavartKernel::eval(a, b, out);
    else
      LogPotentialKernel::eval(a, b, out);
  });
}

// --- RK4 (restated from SPEC.md:530-547; absent from the reference code) ----
// State: xyz (N x 3, unit vectors), zeta (N). Strengths q = zeta * area. Each
// stage calls the reference treecode_sum<BiotSavartKernel> on one FaceTree
// that is reused across stages (the reference re-bins per call,
// treecode.cpp:279). dzeta/dt = -2 Omega u_z. Stage
// positions and the final positions are renormalised through UnitVector3
// (SPEC.md:545, :587). Update order (shared with the device RK4):
//   stage s: x_s = normalise(x + c_s dt k_{s-1}), zeta_s = zeta + c_s dt kz_{s-1}
//   final:   x' = normalise(x + (dt/6) (((k1 + 2 k2) + 2 k3) + k4)), same for zeta.
int ref_rk4(double* xyz, double* zeta, const double* area, int64_t n, double theta, int nt,
            int degree, int max_depth, int workers, double dt, int steps, double omega,
            int direct) {
  return guarded([&] {
    const TraversalConfig cfg = make_cfg(theta, nt, degree, max_depth);
    FaceTree tree;
    const size_t N = static_cast<size_t>(n);
    std::vector<double> k[4];
    std::vector<double> kz[4];
    for (int s = 0; s < 4; ++s) {
      k[s].resize(3 * N);
      kz[s].resize(N);
    }
    std::vector<double> sx(3 * N), sz(N), q(N);
    std::vector<UnitVector3> pts(N);
    const double cs[4] = {0.0, 0.5 * dt, 0.5 * dt, dt};
    for (int step = 0; step < steps; ++step) {
      for (int s = 0; s < 4; ++s) {
        for (size_t i = 0; i < N; ++i) {
          if (s == 0) {  // the state is already unit (renormalised at the end of each step)
            pts[i].x = xyz[3 * i];
            pts[i].y = xyz[3 * i + 1];
            pts[i].z = xyz[3 * i + 2];
            sz[i] = zeta[i];
          } else {
            const double* kp = &k[s - 1][3 * i];
            pts[i] = UnitVector3(xyz[3 * i] + cs[s] * kp[0], xyz[3 * i + 1] + cs[s] * kp[1],
                                 xyz[3 * i + 2] + cs[s] * kp[2]);
            sz[i] = zeta[i] + cs[s] * kz[s - 1][i];
          }
          q[i] = sz[i] * area[i];
        }
        PotentialField<3> u = direct ? direct_sum<BiotSavartKernel>(pts, q)
                                     : treecode_sum<BiotSavartKernel>(pts, q, cfg, tree, workers);
        for (size_t i = 0; i < N; ++i) {
          k[s][3 * i] = u[i][0];
          k[s][3 * i + 1] = u[i][1];
          k[s][3 * i + 2] = u[i][2];
          kz[s][i] = -2.0 * omega * u[i][2];
        }
      }
      const double h6 = dt / 6.0;
      for (size_t i = 0; i < N; ++i) {
        double v[3];
        for (int d = 0; d < 3; ++d) {
          const double kk = ((k[0][3 * i + d] + 2.0 * k[1][3 * i + d]) + 2.0 * k[2][3 * i + d]) +
                            k[3][3 * i + d];
          v[d] = xyz[3 * i + d] + h6 * kk;
        }
        const UnitVector3 p(v[0], v[1], v[2]);
        xyz[3 * i] = p.x;
        xyz[3 * i + 1] = p.y;
        xyz[3 * i + 2] = p.z;
        const double kk = ((kz[0][i] + 2.0 * kz[1][i]) + 2.0 * kz[2][i]) + kz[3][i];
        zeta[i] = zeta[i] + h6 * kk;
      }
    }
  });
}

}  // extern "C"
