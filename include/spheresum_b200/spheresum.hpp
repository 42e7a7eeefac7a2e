// C++ drop-in for the reference's `spheresum` API on the B200 implementation.
//
// Same namespace, type names, signatures and exception types as the
// reference headers (proj/include/spheresum/{errors,geometry,face_tree,
// kernels,treecode}.hpp) for the velocity / stream-function path, written
// independently over the C-ABI (include/spheresum_b200.h). A caller of the
// reference recompiles against this header and links libspheresum_dropin.so
// (+ libspheresum_b200.so) instead of the reference library.
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

// ---- geometry.hpp (the types the path's signatures use) --------------------
struct Vec3 {
  double x = 0.0, y = 0.0, z = 0.0;
};

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

struct SphericalTriangle {
  UnitVector3 v1, v2, v3;
};

// ---- kernels.hpp: kernel descriptors --------------------------------------
inline constexpr double kSingularTol = 1e-14;
struct LogPotentialKernel {
  static constexpr int dim = 1;
  static double prefactor() { return 1.0; }
};
struct BiotSavartKernel {
  static constexpr int dim = 3;
  static double prefactor() { return -1.0 / (4.0 * M_PI); }
};

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
