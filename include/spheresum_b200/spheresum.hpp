// C++ drop-in for the reference's `spheresum` API on the B200 implementation.
//
// Same namespace, type names, signatures and exception types as the
// reference headers (proj/include/spheresum/{errors,geometry,face_tree,
// kernels,treecode}.hpp) for the velocity / stream-function path, written
// independently over the C-ABI (include/spheresum_b200.h). A caller of the
// reference recompiles against this header and links libspheresum_dropin.so
// (+ libspheresum_b200.so) instead of the reference library.
//
// Covered: errors.hpp, geometry.hpp, kernels.hpp (pointwise kernels),
// sbb.hpp, face_tree.hpp, treecode.hpp, plus the RK4 driver and the
// mesh fixture. Not covered (outside the velocity path): icosa_mesh.hpp's
// IcosaMesh class, test_cases.hpp, parallel.hpp, forcing.
//
// Differences a caller can observe:
//  * FaceTree is device-resident; node(id) / leaf_of_particle() return a host
//    snapshot refreshed lazily after each binning (ids are the reference's).
//  * `workers` is accepted and ignored (the GPU is the worker pool).
//  * Output agrees with the reference to ~1e-14 relative L2 (fp64 summation
//    order differs); trees and interaction lists are bit-identical.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../spheresum_b200.h"

namespace spheresum {

// ---- errors.hpp -----------------------------------------------------------
class GeometryError : public std::runtime_error {
 public:
  explicit GeometryError(const std::string& w) : std::runtime_error(w) {}
};
class SingularKernelError : public std::runtime_error {
 public:
  explicit SingularKernelError(const std::string& w) : std::runtime_error(w) {}
};
class ConditioningError : public std::runtime_error {
 public:
  ConditioningError(const std::string& w, double r) : std::runtime_error(w), rcond(r) {}
  double rcond;
};
class ConfigError : public std::runtime_error {
 public:
  explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};

// ---- geometry.hpp -------------------------------------------------------------
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
  Vec3& operator+=(const Vec3& o) {
    x += o.x, y += o.y, z += o.z;
    return *this;
  }
  Vec3& operator-=(const Vec3& o) {
    x -= o.x, y -= o.y, z -= o.z;
    return *this;
  }
  Vec3& operator*=(double s) {
    x *= s, y *= s, z *= s;
    return *this;
  }
};
inline Vec3 operator+(Vec3 a, const Vec3& b) { return a += b; }
inline Vec3 operator-(Vec3 a, const Vec3& b) { return a -= b; }
inline Vec3 operator*(Vec3 a, double s) { return a *= s; }
inline Vec3 operator*(double s, Vec3 a) { return a *= s; }
inline Vec3 operator-(const Vec3& a) { return {-a.x, -a.y, -a.z}; }
inline double dot(const Vec3& a, const Vec3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline Vec3 cross(const Vec3& a, const Vec3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline double norm(const Vec3& a) { return std::sqrt(dot(a, a)); }

// Point on the unit sphere; constructors renormalise (geometry.hpp:50-66).
struct UnitVector3 {
  double x = 1.0, y = 0.0, z = 0.0;
  UnitVector3() = default;
  UnitVector3(double xr, double yr, double zr);
  explicit UnitVector3(const Vec3& v) : UnitVector3(v.x, v.y, v.z) {}
  Vec3 vec() const { return {x, y, z}; }
};
static_assert(sizeof(UnitVector3) == 3 * sizeof(double), "UnitVector3 must be 3 packed doubles");

inline double dot(const UnitVector3& a, const UnitVector3& b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
inline Vec3 cross(const UnitVector3& a, const UnitVector3& b) {
  return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
}
inline Vec3 operator-(const UnitVector3& a, const UnitVector3& b) { return {a.x - b.x, a.y - b.y, a.z - b.z}; }

struct LatLon {
  double lat = 0.0;
  double lon = 0.0;
};
struct BarycentricCoords {
  double b1 = 0.0, b2 = 0.0, b3 = 0.0;
};
inline constexpr double kContainTol = -1e-10;

// Counterclockwise spherical triangle; the 3-vertex constructor validates
// like the reference's (GeometryError, geometry.cpp:27-39).
struct SphericalTriangle {
  UnitVector3 v1, v2, v3;
  SphericalTriangle() = default;
  SphericalTriangle(const UnitVector3& a, const UnitVector3& b, const UnitVector3& c);
};

UnitVector3 latlon_to_unit(const LatLon& p);
LatLon unit_to_latlon(const UnitVector3& v);
double great_circle_distance(const UnitVector3& a, const UnitVector3& b);
BarycentricCoords spherical_barycentric(const SphericalTriangle& t, const UnitVector3& p);
UnitVector3 triangle_circumcenter(const SphericalTriangle& t);
double triangle_radius(const SphericalTriangle& t);
bool triangle_contains(const SphericalTriangle& t, const UnitVector3& p);
double spherical_polygon_area(const std::vector<UnitVector3>& vs);
double spherical_triangle_area(const SphericalTriangle& t);
double barycentric_min_score(const UnitVector3& a, const UnitVector3& b, const UnitVector3& c, const UnitVector3& p);

// ---- kernels.hpp ------------------------------------------------------------
// Pointwise kernels for callers (kernels.hpp:13-61); the sums themselves run
// on the device.
inline constexpr double kSingularTol = 1e-14;
inline double greens_log(const UnitVector3& x, const UnitVector3& y) {
  const double den = 1.0 - dot(x, y);
  if (den <= kSingularTol) throw SingularKernelError("log kernel evaluated at its singularity");
  return -std::log(den) / (4.0 * M_PI);
}
inline Vec3 bve_velocity_kernel(const UnitVector3& x, const UnitVector3& y) {
  const double den = 1.0 - dot(x, y);
  if (den <= kSingularTol) throw SingularKernelError("velocity kernel evaluated at its singularity");
  return cross(x, y) * (1.0 / den);
}
struct LogPotentialKernel {
  static constexpr int dim = 1;
  static double prefactor() { return 1.0; }
  static void eval(const UnitVector3& x, const UnitVector3& y, double* out) { out[0] = greens_log(x, y); }
};
struct BiotSavartKernel {
  static constexpr int dim = 3;
  static double prefactor() { return -1.0 / (4.0 * M_PI); }
  static void eval(const UnitVector3& x, const UnitVector3& y, double* out) {
    const Vec3 v = bve_velocity_kernel(x, y);
    out[0] = v.x, out[1] = v.y, out[2] = v.z;
  }
};

// ---- sbb.hpp ------------------------------------------------------------------
inline constexpr int kMaxSbbDegree = 20;
inline constexpr int sbb_basis_size(int degree) { return (degree + 1) * (degree + 2) / 2; }

class SBBBasis {
 public:
  explicit SBBBasis(int degree);
  int degree() const { return degree_; }
  int size() const { return static_cast<int>(index_set_.size()); }
  const std::vector<std::array<int, 3>>& index_set() const { return index_set_; }
  void eval(const BarycentricCoords& b, double* out) const;
  std::vector<double> eval(const BarycentricCoords& b) const;

 private:
  int degree_;
  std::vector<std::array<int, 3>> index_set_;
};

struct ProxyPointSet {
  SphericalTriangle triangle;
  int degree;
  std::vector<UnitVector3> points;
  std::vector<BarycentricCoords> barycentric;
};
ProxyPointSet proxy_points(const SphericalTriangle& t, int degree);
ProxyPointSet proxy_points_from_barycentric(const SphericalTriangle& t, int degree,
                                            std::vector<BarycentricCoords> bary);

// LU of V[m][k] = B_k(b_m) with partial pivoting; ConditioningError (rcond)
// when the reciprocal condition number is not > 1e-12 (sbb.cpp:74-122).
class ProxyFit {
 public:
  ProxyFit(const SBBBasis& basis, const std::vector<BarycentricCoords>& bary);
  ~ProxyFit();
  ProxyFit(ProxyFit&&) noexcept;
  ProxyFit& operator=(ProxyFit&&) noexcept;
  int size() const;
  double rcond() const;
  void solve(const double* rhs, double* out, int ncols) const;
  void solve_transposed(const double* rhs, double* out, int ncols) const;
  double residual(const double* rhs, const double* x) const;

 private:
  struct Impl;
  std::unique_ptr<Impl> impl_;
};
const ProxyFit& lattice_fit(int degree);

struct SBBInterpolant {
  SphericalTriangle triangle;
  int degree;
  int dim;
  std::vector<double> coefficients;
};
SBBInterpolant fit_coefficients(const ProxyPointSet& pts, const std::vector<double>& values, int dim = 1);
double interpolant_eval(const SBBInterpolant& f, const UnitVector3& p);
void interpolant_eval(const SBBInterpolant& f, const UnitVector3& p, double* out);

// ---- treecode.hpp ----------------------------------------------------------
struct TraversalConfig {
  double theta = 0.7;
  int n_threshold = 32;
  int degree = 6;
  int max_depth = 10;
  void validate() const;
};

enum class InteractionKind : std::uint8_t { PP, PC, CP, CC };

struct Interaction {
  int target = -1;
  int source = -1;
  InteractionKind kind = InteractionKind::PP;
};
using InteractionList = std::vector<Interaction>;

template <int D>
using PotentialField = std::vector<std::array<double, D>>;

struct TreecodeStats {
  double bin_seconds = 0.0;
  double traversal_seconds = 0.0;
  double eval_seconds = 0.0;
  std::array<std::size_t, 4> interaction_counts{};
};

// ---- face_tree.hpp ---------------------------------------------------------
struct TreeNode {
  SphericalTriangle triangle;
  UnitVector3 circumcenter;
  double radius = 0.0;
  int level = 0;
  int parent = -1;
  int root_face = 0;
  int child_base = -1;
  std::vector<int> bin;
  bool has_children() const { return child_base >= 0; }
  int size() const { return static_cast<int>(bin.size()); }
};

// Device-resident face tree (one ssum_ctx per tree, on `device`).
class FaceTree {
 public:
  explicit FaceTree(int device = 0);
  ~FaceTree();
  FaceTree(const FaceTree&) = delete;
  FaceTree& operator=(const FaceTree&) = delete;
  FaceTree(FaceTree&&) noexcept;
  FaceTree& operator=(FaceTree&&) noexcept;

  void bin_particles(const std::vector<UnitVector3>& positions, int n_threshold, int max_depth);
  const TreeNode& node(int id) const;
  int node_count() const;
  int leaf_of_particle(int i) const;
  std::vector<int> path_of_particle(int i) const;

  ssum_ctx* context() const { return ctx_; }
  void invalidate(std::size_t n) {  // after any call that re-binned n particles
    leaf_of_.assign(n, -1);
    stale_ = true;
  }

 private:
  void refresh() const;
  ssum_ctx* ctx_ = nullptr;
  mutable bool stale_ = true;
  mutable std::vector<TreeNode> nodes_;
  mutable std::vector<int> leaf_of_;
};

bool mac_well_separated(const TreeNode& tn, const TreeNode& sn, double theta);

// target_tree and source_tree must be the same FaceTree (as in every reference call).
InteractionList dual_traversal(const FaceTree& target_tree, const FaceTree& source_tree, const TraversalConfig& cfg);

// Proxy weights of one source node (treecode.hpp:47-51), on the device. The
// tree must be binned on `positions` (bin_particles / treecode_sum).
std::vector<double> compute_proxy_weights(const FaceTree& tree, int source_node, const SBBBasis& basis,
                                          const std::vector<UnitVector3>& positions,
                                          const std::vector<double>& strengths);

template <class Kernel>
void eval_pp(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, PotentialField<Kernel::dim>& field);
template <class Kernel>
void eval_pc(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, const TraversalConfig& cfg, PotentialField<Kernel::dim>& field);
template <class Kernel>
void eval_cp(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, const TraversalConfig& cfg, PotentialField<Kernel::dim>& field);
template <class Kernel>
void eval_cc(const FaceTree& tree, const Interaction& it, const std::vector<UnitVector3>& positions,
             const std::vector<double>& strengths, const TraversalConfig& cfg, PotentialField<Kernel::dim>& field);

template <class Kernel>
PotentialField<Kernel::dim> direct_sum(const std::vector<UnitVector3>& positions,
                                       const std::vector<double>& strengths);

template <class Kernel>
PotentialField<Kernel::dim> treecode_sum(const std::vector<UnitVector3>& positions,
                                         const std::vector<double>& strengths, const TraversalConfig& cfg,
                                         FaceTree& tree, int workers = 1, TreecodeStats* stats = nullptr);

// ---- SPEC.md bve_solver: RK4 (absent from the reference code) --------------
inline constexpr double kOmega = 2.0 * M_PI;  // test_cases.hpp:11

// Lagrangian state: positions, relative vorticity, (fixed) areas.
struct ParticleState {
  std::vector<UnitVector3> positions;
  std::vector<double> zeta;
  std::vector<double> area;
};

// `steps` classical RK4 steps: u from treecode_sum (or
// direct_sum when direct), dzeta/dt = -2 omega u_z, positions renormalised
// after every stage; device-resident between stages.
void rk4_run(ParticleState& state, double dt, int steps, const TraversalConfig& cfg, FaceTree& tree,
             double omega = kOmega, bool direct = false, TreecodeStats* stats = nullptr);

// ---- fixtures ---------------------------------------------------------------
// make_icosa_mesh(level).vertices() and node_patch_areas() (icosa_mesh.cpp).
void make_icosa_mesh(int level, std::vector<UnitVector3>& vertices, std::vector<double>* areas);

}  // namespace spheresum
