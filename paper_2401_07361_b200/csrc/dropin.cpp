// libspheresum_dropin.so: the reference-compatible C++ API
// (include/spheresum_b200/spheresum.hpp) implemented over the C-ABI. Only
// marshalling lives here; every computation runs in libspheresum_b200.so.
#include "../../include/spheresum_b200/spheresum.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>

#include "geom.cuh"  // the decision arithmetic shared with the device (host build)

namespace spheresum {

namespace {

[[noreturn]] void throw_status(int code, const char* msg, double rcond = 0.0) {
  const std::string m = msg ? msg : "";
  switch (code) {
    case SSUM_CONFIG:
      throw ConfigError(m);
    case SSUM_GEOMETRY:
      throw GeometryError(m);
    case SSUM_SINGULAR:
      throw SingularKernelError(m);
    case SSUM_CONDITIONING:
      throw ConditioningError(m, rcond);
    case SSUM_INVALID:
      throw std::invalid_argument(m);
    default:
      throw std::runtime_error("spheresum_b200: " + m);
  }
}

void check(ssum_ctx* c, int rc) {
  if (rc != SSUM_OK) throw_status(rc, c ? ssum_last_error(c) : "no context", c ? ssum_last_rcond(c) : 0.0);
}

ssum::d3 d3_of(const UnitVector3& u) { return {u.x, u.y, u.z}; }
UnitVector3 raw_unit(const ssum::d3& v) {  // already unit (computed with the reference's rounding)
  UnitVector3 u;
  u.x = v.x, u.y = v.y, u.z = v.z;
  return u;
}

ssum_config to_c(const TraversalConfig& cfg) {
  return ssum_config{cfg.theta, cfg.n_threshold, cfg.degree, cfg.max_depth, 0};
}

const double* xyz_of(const std::vector<UnitVector3>& p) { return p.empty() ? nullptr : &p[0].x; }

// Process-wide context for calls that take no tree (direct_sum).
ssum_ctx* default_ctx() {
  static std::mutex mu;
  static ssum_ctx* ctx = nullptr;
  std::lock_guard<std::mutex> lock(mu);
  if (!ctx) {
    const int rc = ssum_create(0, &ctx);
    if (rc != SSUM_OK) throw_status(rc, "ssum_create failed (no CUDA device?)");
  }
  return ctx;
}

template <int D>
PotentialField<D> unpack(const std::vector<double>& flat) {
  PotentialField<D> f(flat.size() / D);
  if (!flat.empty()) std::memcpy(f.data()->data(), flat.data(), flat.size() * sizeof(double));
  return f;
}

template <class K>
constexpr int kernel_id() {
  return K::dim == 3 ? SSUM_BIOT_SAVART : SSUM_LOG_POTENTIAL;
}

}  // namespace

UnitVector3::UnitVector3(double xr, double yr, double zr) {
  const double n = std::sqrt(xr * xr + yr * yr + zr * zr);
  if (!(n > 1e-300)) throw GeometryError("cannot normalize a zero vector onto the sphere");
  x = xr / n;
  y = yr / n;
  z = zr / n;
}

// ---- geometry.hpp (geometry.cpp), through the expressions of geom.cuh ------
SphericalTriangle::SphericalTriangle(const UnitVector3& a, const UnitVector3& b, const UnitVector3& c)
    : v1(a), v2(b), v3(c) {
  const ssum::d3 A = d3_of(a), B = d3_of(b), C = d3_of(c);
  if (ssum::arc_dist(A, B) <= 1e-12 || ssum::arc_dist(B, C) <= 1e-12 || ssum::arc_dist(C, A) <= 1e-12)
    throw GeometryError("spherical triangle has coincident vertices");
  if (ssum::dot_rn(A, ssum::cross_rn(B, C)) <= 0.0)
    throw GeometryError("spherical triangle vertices are not counterclockwise");
}

UnitVector3 latlon_to_unit(const LatLon& p) {
  const double cl = std::cos(p.lat);
  return UnitVector3(cl * std::cos(p.lon), cl * std::sin(p.lon), std::sin(p.lat));
}

LatLon unit_to_latlon(const UnitVector3& v) {
  LatLon o;
  o.lat = std::asin(std::min(1.0, std::max(-1.0, v.z)));
  o.lon = std::atan2(v.y, v.x);
  if (o.lon >= M_PI) o.lon -= 2.0 * M_PI;
  return o;
}

double great_circle_distance(const UnitVector3& a, const UnitVector3& b) { return ssum::arc_dist(d3_of(a), d3_of(b)); }

BarycentricCoords spherical_barycentric(const SphericalTriangle& t, const UnitVector3& p) {
  const ssum::d3 a = d3_of(t.v1), b = d3_of(t.v2), c = d3_of(t.v3), x = d3_of(p);
  const double det = ssum::dot_rn(a, ssum::cross_rn(b, c));
  if (std::fabs(det) < 1e-14) throw GeometryError("degenerate triangle in barycentric solve");
  const double r0 = ssum::dot_rn(x, ssum::cross_rn(b, c)) / det;
  const double r1 = ssum::dot_rn(a, ssum::cross_rn(x, c)) / det;
  const double r2 = ssum::dot_rn(a, ssum::cross_rn(b, x)) / det;
  const double sum = r0 + r1 + r2;
  if (std::fabs(sum) < 1e-14) throw GeometryError("point has no radial projection onto the triangle plane");
  return {r0 / sum, r1 / sum, r2 / sum};
}

UnitVector3 triangle_circumcenter(const SphericalTriangle& t) {
  int bad = 0;
  const ssum::d3 c = ssum::circumcenter_rn(d3_of(t.v1), d3_of(t.v2), d3_of(t.v3), &bad);
  if (bad) throw GeometryError("degenerate triangle in circumcenter");
  return raw_unit(c);
}

double triangle_radius(const SphericalTriangle& t) { return great_circle_distance(triangle_circumcenter(t), t.v1); }

bool triangle_contains(const SphericalTriangle& t, const UnitVector3& p) {
  return ssum::contains_rn(d3_of(t.v1), d3_of(t.v2), d3_of(t.v3), d3_of(p));
}

// spherical excess: interior angles (between the tangent directions towards
// the two neighbours) minus (n - 2) pi
double spherical_polygon_area(const std::vector<UnitVector3>& vs) {
  const size_t n = vs.size();
  if (n < 3) throw GeometryError("spherical polygon needs at least 3 vertices");
  double angles = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const UnitVector3& h = vs[i];
    const UnitVector3& a = vs[(i + n - 1) % n];
    const UnitVector3& b = vs[(i + 1) % n];
    const Vec3 ta = a.vec() - dot(a, h) * h.vec();
    const Vec3 tb = b.vec() - dot(b, h) * h.vec();
    angles += std::atan2(norm(cross(ta, tb)), dot(ta, tb));
  }
  return angles - (static_cast<double>(n) - 2.0) * M_PI;
}

double spherical_triangle_area(const SphericalTriangle& t) { return spherical_polygon_area({t.v1, t.v2, t.v3}); }

double barycentric_min_score(const UnitVector3& a, const UnitVector3& b, const UnitVector3& c, const UnitVector3& p) {
  const ssum::d3 A = d3_of(a), B = d3_of(b), C = d3_of(c);
  const ssum::d3 bc = ssum::cross_rn(B, C);
  return ssum::min_score_rn(A, B, C, bc, ssum::dot_rn(A, bc), d3_of(p));
}

// ---- sbb.hpp ------------------------------------------------------------------
SBBBasis::SBBBasis(int degree) : degree_(degree) {
  if (degree < 1 || degree > kMaxSbbDegree) throw std::invalid_argument("SBB degree must be in [1, 20]");
  for (int k = 0; k <= degree; ++k)
    for (int j = 0; j <= degree - k; ++j) index_set_.push_back({degree - k - j, j, k});
}

void SBBBasis::eval(const BarycentricCoords& b, double* out) const {
  double p1[kMaxSbbDegree + 1], p2[kMaxSbbDegree + 1], p3[kMaxSbbDegree + 1];
  p1[0] = p2[0] = p3[0] = 1.0;
  for (int e = 1; e <= degree_; ++e) {
    p1[e] = p1[e - 1] * b.b1;
    p2[e] = p2[e - 1] * b.b2;
    p3[e] = p3[e - 1] * b.b3;
  }
  for (size_t m = 0; m < index_set_.size(); ++m) {
    const std::array<int, 3>& e = index_set_[m];
    out[m] = p1[e[0]] * p2[e[1]] * p3[e[2]];
  }
}

std::vector<double> SBBBasis::eval(const BarycentricCoords& b) const {
  std::vector<double> v(index_set_.size());
  eval(b, v.data());
  return v;
}

ProxyPointSet proxy_points_from_barycentric(const SphericalTriangle& t, int degree,
                                            std::vector<BarycentricCoords> bary) {
  ProxyPointSet s{t, degree, {}, std::move(bary)};
  for (const BarycentricCoords& b : s.barycentric)
    s.points.push_back(UnitVector3(b.b1 * t.v1.vec() + b.b2 * t.v2.vec() + b.b3 * t.v3.vec()));
  return s;
}

ProxyPointSet proxy_points(const SphericalTriangle& t, int degree) {
  const SBBBasis basis(degree);
  lattice_fit(degree);  // the conditioning guard, as the reference trips it here
  const double d = static_cast<double>(degree);
  std::vector<BarycentricCoords> bary;
  for (const std::array<int, 3>& e : basis.index_set()) bary.push_back({e[0] / d, e[1] / d, e[2] / d});
  return proxy_points_from_barycentric(t, degree, std::move(bary));
}

// Row-major LU with partial pivoting (first largest pivot), P A = L U.
struct ProxyFit::Impl {
  int n = 0;
  std::vector<double> a;   // the matrix V
  std::vector<double> lu;  // packed L (unit diagonal) and U
  std::vector<int> piv;    // row of A at position i of P A
  double rcond = 0.0;
  void solve_col(const double* b, double* x) const {  // V x = b
    std::vector<double> y(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      double s = b[piv[size_t(i)]];
      for (int k = 0; k < i; ++k) s -= lu[size_t(i) * n + k] * y[size_t(k)];
      y[size_t(i)] = s;
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = y[size_t(i)];
      for (int k = i + 1; k < n; ++k) s -= lu[size_t(i) * n + k] * x[k];
      x[i] = s / lu[size_t(i) * n + i];
    }
  }
  void solve_col_t(const double* b, double* x) const {  // V^T x = b: U^T z = b, L^T w = z, x = P^T w
    std::vector<double> z(static_cast<size_t>(n));
    for (int i = 0; i < n; ++i) {
      double s = b[i];
      for (int k = 0; k < i; ++k) s -= lu[size_t(k) * n + i] * z[size_t(k)];
      z[size_t(i)] = s / lu[size_t(i) * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
      double s = z[size_t(i)];
      for (int k = i + 1; k < n; ++k) s -= lu[size_t(k) * n + i] * z[size_t(k)];
      z[size_t(i)] = s;
    }
    for (int i = 0; i < n; ++i) x[piv[size_t(i)]] = z[size_t(i)];
  }
};

ProxyFit::ProxyFit(const SBBBasis& basis, const std::vector<BarycentricCoords>& bary)
    : impl_(std::make_unique<Impl>()) {
  const int n = basis.size();
  if (static_cast<int>(bary.size()) != n) throw std::invalid_argument("proxy point count must equal the basis size");
  Impl& m = *impl_;
  m.n = n;
  m.a.resize(size_t(n) * n);
  for (int r = 0; r < n; ++r) basis.eval(bary[size_t(r)], &m.a[size_t(r) * n]);
  m.lu = m.a;
  m.piv.resize(size_t(n));
  for (int i = 0; i < n; ++i) m.piv[size_t(i)] = i;
  bool singular = false;
  for (int k = 0; k < n && !singular; ++k) {
    int p = k;
    for (int i = k + 1; i < n; ++i)
      if (std::fabs(m.lu[size_t(i) * n + k]) > std::fabs(m.lu[size_t(p) * n + k])) p = i;
    if (m.lu[size_t(p) * n + k] == 0.0) {
      singular = true;
      break;
    }
    if (p != k) {
      for (int j = 0; j < n; ++j) std::swap(m.lu[size_t(k) * n + j], m.lu[size_t(p) * n + j]);
      std::swap(m.piv[size_t(k)], m.piv[size_t(p)]);
    }
    for (int i = k + 1; i < n; ++i) {
      const double l = m.lu[size_t(i) * n + k] /= m.lu[size_t(k) * n + k];
      for (int j = k + 1; j < n; ++j) m.lu[size_t(i) * n + j] -= l * m.lu[size_t(k) * n + j];
    }
  }
  if (!singular) {  // exact 1-norm reciprocal condition number: ||V||_1 ||V^-1||_1
    double an = 0.0, in = 0.0;
    std::vector<double> e(static_cast<size_t>(n)), col(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j) {
      double s = 0.0;
      for (int i = 0; i < n; ++i) s += std::fabs(m.a[size_t(i) * n + j]);
      an = std::max(an, s);
      std::fill(e.begin(), e.end(), 0.0);
      e[size_t(j)] = 1.0;
      m.solve_col(e.data(), col.data());
      double t = 0.0;
      for (int i = 0; i < n; ++i) t += std::fabs(col[size_t(i)]);
      in = std::max(in, t);
    }
    m.rcond = (an > 0.0 && std::isfinite(in) && in > 0.0) ? 1.0 / (an * in) : 0.0;
  }
  if (!(m.rcond > 1e-12))
    throw ConditioningError("proxy Vandermonde too ill-conditioned (rcond " + std::to_string(m.rcond) + ")", m.rcond);
}

ProxyFit::~ProxyFit() = default;
ProxyFit::ProxyFit(ProxyFit&&) noexcept = default;
ProxyFit& ProxyFit::operator=(ProxyFit&&) noexcept = default;
int ProxyFit::size() const { return impl_->n; }
double ProxyFit::rcond() const { return impl_->rcond; }

void ProxyFit::solve(const double* rhs, double* out, int ncols) const {
  const int n = impl_->n;
  for (int c = 0; c < ncols; ++c) impl_->solve_col(rhs + size_t(c) * n, out + size_t(c) * n);
}

void ProxyFit::solve_transposed(const double* rhs, double* out, int ncols) const {
  const int n = impl_->n;
  for (int c = 0; c < ncols; ++c) impl_->solve_col_t(rhs + size_t(c) * n, out + size_t(c) * n);
}

double ProxyFit::residual(const double* rhs, const double* x) const {
  const int n = impl_->n;
  double worst = 0.0;
  for (int i = 0; i < n; ++i) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += impl_->a[size_t(i) * n + k] * x[k];
    worst = std::max(worst, std::fabs(s - rhs[i]));
  }
  return worst;
}

const ProxyFit& lattice_fit(int degree) {
  static std::mutex mu;
  static std::map<int, std::unique_ptr<ProxyFit>> fits;
  std::lock_guard<std::mutex> lock(mu);
  std::unique_ptr<ProxyFit>& f = fits[degree];
  if (!f) {
    const SBBBasis basis(degree);
    const double d = static_cast<double>(degree);
    std::vector<BarycentricCoords> bary;
    for (const std::array<int, 3>& e : basis.index_set()) bary.push_back({e[0] / d, e[1] / d, e[2] / d});
    f = std::make_unique<ProxyFit>(basis, bary);
  }
  return *f;
}

SBBInterpolant fit_coefficients(const ProxyPointSet& pts, const std::vector<double>& values, int dim) {
  const SBBBasis basis(pts.degree);
  if (static_cast<int>(values.size()) != basis.size() * dim)
    throw std::invalid_argument("value count must equal proxy point count times dim");
  const ProxyFit fit(basis, pts.barycentric);
  SBBInterpolant f{pts.triangle, pts.degree, dim, std::vector<double>(values.size())};
  fit.solve(values.data(), f.coefficients.data(), dim);
  return f;
}

void interpolant_eval(const SBBInterpolant& f, const UnitVector3& p, double* out) {
  const SBBBasis basis(f.degree);
  const int n = basis.size();
  double b[sbb_basis_size(kMaxSbbDegree)];
  basis.eval(spherical_barycentric(f.triangle, p), b);
  for (int d = 0; d < f.dim; ++d) {
    double s = 0.0;
    for (int k = 0; k < n; ++k) s += f.coefficients[size_t(d) * n + k] * b[k];
    out[d] = s;
  }
}

double interpolant_eval(const SBBInterpolant& f, const UnitVector3& p) {
  double v = 0.0;
  interpolant_eval(f, p, &v);
  return v;
}

void TraversalConfig::validate() const {
  if (!(theta > 0.0 && theta <= 1.0)) throw ConfigError("theta must be in (0, 1]");
  if (n_threshold < 1) throw ConfigError("n_threshold must be >= 1");
  if (degree < 1 || degree > 20) throw ConfigError("degree must be in [1, 20]");
  if (max_depth < 1 || max_depth > 40) throw ConfigError("max_depth must be in [1, 40]");
}

FaceTree::FaceTree(int device) { check(nullptr, ssum_create(device, &ctx_)); }
FaceTree::~FaceTree() {
  if (ctx_) ssum_destroy(ctx_);
}
FaceTree::FaceTree(FaceTree&& o) noexcept
    : ctx_(o.ctx_), stale_(o.stale_), nodes_(std::move(o.nodes_)), leaf_of_(std::move(o.leaf_of_)) {
  o.ctx_ = nullptr;
}
FaceTree& FaceTree::operator=(FaceTree&& o) noexcept {
  if (this != &o) {
    if (ctx_) ssum_destroy(ctx_);
    ctx_ = o.ctx_;
    stale_ = o.stale_;
    nodes_ = std::move(o.nodes_);
    leaf_of_ = std::move(o.leaf_of_);
    o.ctx_ = nullptr;
  }
  return *this;
}

void FaceTree::bin_particles(const std::vector<UnitVector3>& positions, int n_threshold, int max_depth) {
  check(ctx_, ssum_bin_particles(ctx_, xyz_of(positions), static_cast<int64_t>(positions.size()), n_threshold,
                                 max_depth));
  leaf_of_.assign(positions.size(), -1);
  stale_ = true;
}

void FaceTree::refresh() const {
  if (!stale_) return;
  int m = 0;
  check(ctx_, ssum_tree_node_count(ctx_, &m));
  std::vector<int> level(m), parent(m), child(m);
  std::vector<double> tri(size_t(m) * 9), center(size_t(m) * 3), radius(m);
  std::vector<int64_t> off(size_t(m) + 1);
  check(ctx_, ssum_tree_export(ctx_, level.data(), parent.data(), child.data(), tri.data(), center.data(),
                               radius.data(), off.data(), nullptr, nullptr));
  std::vector<int> ids(std::max<int64_t>(off[m], 1));
  std::vector<int> leaf(std::max<size_t>(leaf_of_.size(), 1));
  check(ctx_, ssum_tree_export(ctx_, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, off.data(), ids.data(),
                               leaf.data()));
  nodes_.assign(m, TreeNode{});
  for (int i = 0; i < m; ++i) {
    TreeNode& nd = nodes_[i];
    const double* t = &tri[size_t(i) * 9];
    nd.triangle = SphericalTriangle{};
    nd.triangle.v1.x = t[0], nd.triangle.v1.y = t[1], nd.triangle.v1.z = t[2];
    nd.triangle.v2.x = t[3], nd.triangle.v2.y = t[4], nd.triangle.v2.z = t[5];
    nd.triangle.v3.x = t[6], nd.triangle.v3.y = t[7], nd.triangle.v3.z = t[8];
    nd.circumcenter.x = center[size_t(i) * 3];
    nd.circumcenter.y = center[size_t(i) * 3 + 1];
    nd.circumcenter.z = center[size_t(i) * 3 + 2];
    nd.radius = radius[i];
    nd.level = level[i];
    nd.parent = parent[i];
    nd.child_base = child[i];
    nd.bin.assign(ids.begin() + off[i], ids.begin() + off[i + 1]);
  }
  for (int i = 0; i < m; ++i) {  // root face: walk up
    int r = i;
    while (nodes_[r].parent >= 0) r = nodes_[r].parent;
    nodes_[i].root_face = r;
  }
  std::copy(leaf.begin(), leaf.begin() + leaf_of_.size(), leaf_of_.begin());
  stale_ = false;
}

const TreeNode& FaceTree::node(int id) const {
  refresh();
  return nodes_.at(id);
}
int FaceTree::node_count() const {
  int m = 0;
  check(ctx_, ssum_tree_node_count(ctx_, &m));
  return m;
}
int FaceTree::leaf_of_particle(int i) const {
  refresh();
  return leaf_of_.at(i);
}
std::vector<int> FaceTree::path_of_particle(int i) const {
  refresh();
  std::vector<int> path;
  for (int id = leaf_of_.at(i); id >= 0; id = nodes_[id].parent) path.push_back(id);
  std::reverse(path.begin(), path.end());
  return path;
}

bool mac_well_separated(const TreeNode& tn, const TreeNode& sn, double theta) {
  const Vec3 c = cross(tn.circumcenter, sn.circumcenter);
  const double r = std::atan2(std::sqrt(c.x * c.x + c.y * c.y + c.z * c.z), dot(tn.circumcenter, sn.circumcenter));
  return r > 0.0 && (tn.radius + sn.radius) / r < theta;
}

InteractionList dual_traversal(const FaceTree& target_tree, const FaceTree& source_tree,
                               const TraversalConfig& cfg) {
  cfg.validate();
  if (&target_tree != &source_tree) throw std::invalid_argument("dual_traversal: trees must be the same FaceTree");
  const ssum_config c = to_c(cfg);
  int64_t count = 0;
  check(target_tree.context(), ssum_dual_traversal(target_tree.context(), &c, nullptr, 0, &count));
  std::vector<int> tsk(size_t(std::max<int64_t>(count, 1)) * 3);
  check(target_tree.context(), ssum_dual_traversal(target_tree.context(), &c, tsk.data(), count, &count));
  InteractionList out(static_cast<size_t>(count));
  for (int64_t e = 0; e < count; ++e)
    out[e] = Interaction{tsk[3 * e], tsk[3 * e + 1], static_cast<InteractionKind>(tsk[3 * e + 2])};
  return out;
}

std::vector<double> compute_proxy_weights(const FaceTree& tree, int source_node, const SBBBasis& basis,
                                          const std::vector<UnitVector3>& positions,
                                          const std::vector<double>& strengths) {
  if (positions.size() != strengths.size()) throw std::invalid_argument("compute_proxy_weights: size mismatch");
  std::vector<double> w(size_t(basis.size()));
  check(tree.context(), ssum_compute_proxy_weights(tree.context(), basis.degree(), xyz_of(positions),
                                                   strengths.data(), static_cast<int64_t>(positions.size()),
                                                   source_node, w.data()));
  return w;
}

namespace {
template <class K>
void eval_one(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
              const std::vector<double>& strengths, const TraversalConfig& cfg, PotentialField<K::dim>& field) {
  const ssum_config c = to_c(cfg);
  check(tree.context(), ssum_eval_interaction(tree.context(), kernel_id<K>(), &c, xyz_of(positions),
                                              strengths.data(), static_cast<int64_t>(positions.size()), it.target,
                                              it.source, static_cast<int>(it.kind),
                                              field.empty() ? nullptr : field.data()->data()));
}
}  // namespace

template <class K>
void eval_pp(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, PotentialField<K::dim>& field) {
  eval_one<K>(tree, it, positions, strengths, TraversalConfig{}, field);
}
template <class K>
void eval_pc(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, const TraversalConfig& cfg, PotentialField<K::dim>& field) {
  eval_one<K>(tree, it, positions, strengths, cfg, field);
}
template <class K>
void eval_cp(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, const TraversalConfig& cfg, PotentialField<K::dim>& field) {
  eval_one<K>(tree, it, positions, strengths, cfg, field);
}
template <class K>
void eval_cc(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, const TraversalConfig& cfg, PotentialField<K::dim>& field) {
  eval_one<K>(tree, it, positions, strengths, cfg, field);
}

template <class K>
PotentialField<K::dim> direct_sum(const std::vector<UnitVector3>& positions, const std::vector<double>& strengths) {
  if (positions.size() != strengths.size()) throw std::invalid_argument("direct_sum: size mismatch");
  std::vector<double> out(positions.size() * K::dim);
  ssum_ctx* c = default_ctx();
  check(c, ssum_direct_sum(c, kernel_id<K>(), xyz_of(positions), strengths.data(),
                           static_cast<int64_t>(positions.size()), out.data()));
  return unpack<K::dim>(out);
}

template <class K>
PotentialField<K::dim> treecode_sum(const std::vector<UnitVector3>& positions, const std::vector<double>& strengths,
                                    const TraversalConfig& cfg, FaceTree& tree, int workers, TreecodeStats* stats) {
  (void)workers;
  cfg.validate();
  if (positions.size() != strengths.size()) throw std::invalid_argument("treecode_sum: size mismatch");
  const ssum_config c = to_c(cfg);
  std::vector<double> out(positions.size() * K::dim);
  ssum_stats st{};
  check(tree.context(), ssum_treecode_sum(tree.context(), kernel_id<K>(), &c, xyz_of(positions), strengths.data(),
                                          static_cast<int64_t>(positions.size()), out.data(), &st));
  tree.invalidate(positions.size());
  if (stats) {  // accumulate like the reference (treecode.cpp:296,407-411)
    stats->bin_seconds += st.bin_seconds;
    stats->traversal_seconds += st.traversal_seconds;
    stats->eval_seconds += st.eval_seconds;
    for (int k = 0; k < 4; ++k) stats->interaction_counts[k] += st.interaction_counts[k];
  }
  return unpack<K::dim>(out);
}

void rk4_run(ParticleState& s, double dt, int steps, const TraversalConfig& cfg, FaceTree& tree, double omega,
             bool direct, TreecodeStats* stats) {
  cfg.validate();
  const size_t n = s.positions.size();
  if (s.zeta.size() != n || s.area.size() != n) throw std::invalid_argument("rk4_run: size mismatch");
  const ssum_config c = to_c(cfg);
  ssum_stats st{};
  check(tree.context(), ssum_rk4(tree.context(), &c, n ? &s.positions[0].x : nullptr, s.zeta.data(), s.area.data(),
                                 static_cast<int64_t>(n), dt, steps, omega, direct ? 1 : 0, &st));
  tree.invalidate(n);
  if (stats) {
    stats->bin_seconds += st.bin_seconds;
    stats->traversal_seconds += st.traversal_seconds;
    stats->eval_seconds += st.eval_seconds;
  }
}

void make_icosa_mesh(int level, std::vector<UnitVector3>& vertices, std::vector<double>* areas) {
  const int64_t n = ssum_mesh_vertex_count(level);
  if (n < 0) throw std::invalid_argument("make_icosa_mesh: level out of range");
  vertices.assign(static_cast<size_t>(n), UnitVector3{});
  if (areas) areas->assign(static_cast<size_t>(n), 0.0);
  const int rc = ssum_make_icosa_mesh(level, &vertices[0].x, areas ? areas->data() : nullptr);
  if (rc != SSUM_OK) throw_status(rc, "make_icosa_mesh failed");
}

// Explicit instantiations for the two reference kernels (treecode.cpp:415-436).
#define SPHERESUM_B200_INSTANTIATE(K)                                                                         \
  template void eval_pp<K>(const FaceTree&, const Interaction&, const std::vector<UnitVector3>&,              \
                           const std::vector<double>&, PotentialField<K::dim>&);                              \
  template void eval_pc<K>(const FaceTree&, const Interaction&, const std::vector<UnitVector3>&,              \
                           const std::vector<double>&, const TraversalConfig&, PotentialField<K::dim>&);      \
  template void eval_cp<K>(const FaceTree&, const Interaction&, const std::vector<UnitVector3>&,              \
                           const std::vector<double>&, const TraversalConfig&, PotentialField<K::dim>&);      \
  template void eval_cc<K>(const FaceTree&, const Interaction&, const std::vector<UnitVector3>&,              \
                           const std::vector<double>&, const TraversalConfig&, PotentialField<K::dim>&);      \
  template PotentialField<K::dim> direct_sum<K>(const std::vector<UnitVector3>&, const std::vector<double>&); \
  template PotentialField<K::dim> treecode_sum<K>(const std::vector<UnitVector3>&, const std::vector<double>&, \
                                                  const TraversalConfig&, FaceTree&, int, TreecodeStats*)
SPHERESUM_B200_INSTANTIATE(LogPotentialKernel);
SPHERESUM_B200_INSTANTIATE(BiotSavartKernel);
#undef SPHERESUM_B200_INSTANTIATE

}  // namespace spheresum
