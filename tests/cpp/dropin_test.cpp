// Drives the C++ drop-in (include/spheresum_b200/spheresum.hpp) exactly as a
// reference caller would, on the level-3 mesh. Usage:
//   dropin_test <q.bin> <out.bin>
// q.bin: N float64 strengths (tests/golden l3_q). out.bin: u_tree (N x 3),
// psi_tree (N), u_direct (N x 3), list count + triples, node 0..19 bin sizes,
// eval_pp of the first PP interaction into zeros (N x 3), rk4 positions (N x 3)
// and zeta (N) after 2 steps — all float64. tests/test_gpu_dropin.py checks them.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <vector>

#include "spheresum_b200/spheresum.hpp"

using namespace spheresum;

template <class T>
void put(std::ofstream& f, const T* p, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    const double v = static_cast<double>(p[i]);
    f.write(reinterpret_cast<const char*>(&v), sizeof(double));
  }
}

int main(int argc, char** argv) {
  if (argc < 3) return 2;
  std::vector<UnitVector3> pts;
  std::vector<double> area;
  make_icosa_mesh(3, pts, &area);
  const size_t n = pts.size();
  std::vector<double> q(n);
  std::ifstream fq(argv[1], std::ios::binary);
  fq.read(reinterpret_cast<char*>(q.data()), std::streamsize(n * sizeof(double)));
  if (!fq) return 3;

  TraversalConfig cfg;
  cfg.theta = 0.7;
  cfg.n_threshold = 8;
  cfg.degree = 4;
  cfg.max_depth = 10;
  FaceTree tree;
  TreecodeStats stats;
  const auto u = treecode_sum<BiotSavartKernel>(pts, q, cfg, tree, 4, &stats);
  const auto psi = treecode_sum<LogPotentialKernel>(pts, q, cfg, tree, 4, &stats);
  const auto ud = direct_sum<BiotSavartKernel>(pts, q);
  const InteractionList list = dual_traversal(tree, tree, cfg);

  std::ofstream fo(argv[2], std::ios::binary);
  put(fo, u.data()->data(), n * 3);
  put(fo, psi.data()->data(), n);
  put(fo, ud.data()->data(), n * 3);
  const double cnt = double(list.size());
  put(fo, &cnt, 1);
  for (const Interaction& it : list) {
    const double t[3] = {double(it.target), double(it.source), double(static_cast<int>(it.kind))};
    put(fo, t, 3);
  }
  double sizes[20];
  for (int f = 0; f < 20; ++f) sizes[f] = tree.node(f).size();
  put(fo, sizes, 20);
  PotentialField<3> field(n, std::array<double, 3>{0.0, 0.0, 0.0});
  for (const Interaction& it : list)
    if (it.kind == InteractionKind::PP) {
      eval_pp<BiotSavartKernel>(tree, it, pts, q, field);
      break;
    }
  put(fo, field.data()->data(), n * 3);

  // compute_proxy_weights of root face 0 (degree 4) on the tree as binned by
  // the calls above; the SBB API: lattice_fit rcond, constant reproduction by
  // fit_coefficients / interpolant_eval, the degree-16 conditioning guard
  {
    const std::vector<double> w = compute_proxy_weights(tree, 0, SBBBasis(4), pts, q);
    put(fo, w.data(), w.size());
    const double rc8 = lattice_fit(8).rcond();
    put(fo, &rc8, 1);
    const TreeNode& nd = tree.node(0);
    const SphericalTriangle tri(nd.triangle.v1, nd.triangle.v2, nd.triangle.v3);
    const ProxyPointSet pp8 = proxy_points(tri, 8);
    const SBBInterpolant f = fit_coefficients(pp8, std::vector<double>(pp8.points.size(), 2.5));
    const double at = interpolant_eval(f, triangle_circumcenter(tri)) - 2.5;
    put(fo, &at, 1);
    double rc16 = -1.0;
    try {
      lattice_fit(16);
    } catch (const ConditioningError& e) {
      rc16 = e.rcond;
    }
    put(fo, &rc16, 1);
    const double geo[3] = {double(triangle_contains(tri, triangle_circumcenter(tri))),
                           triangle_radius(tri) - nd.radius, great_circle_distance(nd.circumcenter, tri.v1)};
    put(fo, geo, 3);
  }

  ParticleState st{pts, std::vector<double>(n), area};
  for (size_t i = 0; i < n; ++i) {  // RH4 vorticity from q = zeta * A
    st.zeta[i] = q[i] / area[i];
  }
  FaceTree rk_tree;
  rk4_run(st, 0.01, 2, cfg, rk_tree);
  put(fo, &st.positions[0].x, n * 3);
  put(fo, st.zeta.data(), n);

  bool threw = false;  // SingularKernelError mirrors kernels.hpp:27-29
  try {
    std::vector<UnitVector3> dup = pts;
    dup.push_back(pts[7]);
    std::vector<double> qd = q;
    qd.push_back(1.0);
    treecode_sum<BiotSavartKernel>(dup, qd, cfg, tree);
  } catch (const SingularKernelError&) {
    threw = true;
  }
  std::printf("dropin ok n=%zu list=%zu singular_threw=%d counts=%zu,%zu,%zu,%zu\n", n, list.size(), int(threw),
              stats.interaction_counts[0], stats.interaction_counts[1], stats.interaction_counts[2],
              stats.interaction_counts[3]);
  return threw ? 0 : 4;
}
