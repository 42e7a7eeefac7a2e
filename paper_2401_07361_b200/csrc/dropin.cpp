// libspheresum_dropin.so: the reference-compatible C++ API
// (include/spheresum_b200/spheresum.hpp) implemented over the C-ABI. Only
// marshalling lives here; every computation runs in libspheresum_b200.so.
#include "../../include/spheresum_b200/spheresum.hpp"

#include <algorithm>
#include <cstring>
#include <mutex>

namespace spheresum {

namespace {

[[noreturn]] void throw_status(int code, const char* msg) {
  const std::string m = msg ? msg : "";
  switch (code) {
    case SSUM_CONFIG:
      throw ConfigError(m);
    case SSUM_GEOMETRY:
      throw GeometryError(m);
    case SSUM_SINGULAR:
      throw SingularKernelError(m);
    case SSUM_CONDITIONING:
      throw ConditioningError(m, 0.0);
    case SSUM_INVALID:
      throw std::invalid_argument(m);
    default:
      throw std::runtime_error("spheresum_b200: " + m);
  }
}

void check(ssum_ctx* c, int rc) {
  if (rc != SSUM_OK) throw_status(rc, c ? ssum_last_error(c) : "no context");
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
