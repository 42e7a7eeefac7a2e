// Sphere geometry shared by host and device code.
//
// Tree-structure DECISIONS (root-face containment, child choice, node
// geometry) must match the reference bit for bit: a flipped decision changes
// the answer at the 1e-6 tree-error level, not at 1e-14.
// nvcc contracts `a*b + c` into DFMA by default, so every operation that
// feeds a decision is written with explicit round-to-nearest intrinsics
// (__dmul_rn / __dadd_rn / __dsub_rn / __ddiv_rn / __dsqrt_rn), which are never
// fused. On the host the same expressions compile with -ffp-contract=off.
// Each function cites the reference expression whose rounding it reproduces.
#pragma once

#include <cmath>

#if defined(__CUDACC__)
#define SSUM_HD __host__ __device__ __forceinline__
#else
#define SSUM_HD inline
#endif

namespace ssum {

struct d3 {
  double x, y, z;
};

SSUM_HD double mul_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dmul_rn(a, b);
#else
  return a * b;
#endif
}
SSUM_HD double add_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dadd_rn(a, b);
#else
  return a + b;
#endif
}
SSUM_HD double sub_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __dsub_rn(a, b);
#else
  return a - b;
#endif
}
SSUM_HD double div_rn(double a, double b) {
#if defined(__CUDA_ARCH__)
  return __ddiv_rn(a, b);
#else
  return a / b;
#endif
}
SSUM_HD double sqrt_rn(double a) {
#if defined(__CUDA_ARCH__)
  return __dsqrt_rn(a);
#else
  return std::sqrt(a);
#endif
}

SSUM_HD d3 add3(d3 a, d3 b) { return {add_rn(a.x, b.x), add_rn(a.y, b.y), add_rn(a.z, b.z)}; }
SSUM_HD d3 sub3(d3 a, d3 b) { return {sub_rn(a.x, b.x), sub_rn(a.y, b.y), sub_rn(a.z, b.z)}; }

// dot(a, b) = a.x*b.x + a.y*b.y + a.z*b.z, left to right (geometry.hpp:42,68-70)
SSUM_HD double dot_rn(d3 a, d3 b) {
  return add_rn(add_rn(mul_rn(a.x, b.x), mul_rn(a.y, b.y)), mul_rn(a.z, b.z));
}
// cross (geometry.hpp:43-45,71-73)
SSUM_HD d3 cross_rn(d3 a, d3 b) {
  return {sub_rn(mul_rn(a.y, b.z), mul_rn(a.z, b.y)), sub_rn(mul_rn(a.z, b.x), mul_rn(a.x, b.z)),
          sub_rn(mul_rn(a.x, b.y), mul_rn(a.y, b.x))};
}

// UnitVector3(x, y, z): n = sqrt(x*x + y*y + z*z); (x/n, y/n, z/n)
// (geometry.hpp:55-61). *bad is set when n <= 1e-300 (GeometryError).
SSUM_HD d3 unit_rn(d3 v, int* bad) {
  const double n = sqrt_rn(add_rn(add_rn(mul_rn(v.x, v.x), mul_rn(v.y, v.y)), mul_rn(v.z, v.z)));
  if (!(n > 1e-300)) {
    *bad = 1;
    return {1.0, 0.0, 0.0};
  }
  return {div_rn(v.x, n), div_rn(v.y, n), div_rn(v.z, n)};
}

// great_circle_distance = atan2(|a x b|, a.b) (geometry.cpp:55-57). The
// device atan2 is CUDA's (<= 2 ulp), not glibc's: node radii and MAC distances
// may differ from the reference in the last bits. A MAC decision could flip
// only if (r_t + r_s)/R lay within a few ulp of theta, so the traversal sends
// every pair within a 1e-12 relative band of theta to the host, which decides
// it with glibc and the reference's expressions (traversal.cu MacCtl /
// resolve_mac): decisions are the reference's by construction. Tests:
// tests/test_gpu_boundary.py (forced wide band), tests/test_gpu_parity.py and
// tests/test_gpu_fullsize.py (bit-identical lists up to C5).
SSUM_HD double arc_dist(d3 a, d3 b) {
  const d3 c = cross_rn(a, b);
  return atan2(sqrt_rn(dot_rn(c, c)), dot_rn(a, b));
}

// barycentric_min_score (geometry.cpp:114-125), bit-exact. bc = cross(b, c)
// and det = dot(a, bc) are per-triangle constants, passed precomputed (same
// expressions, same rounding).
SSUM_HD double min_score_rn(d3 a, d3 b, d3 c, d3 bc, double det, d3 p) {
  if (fabs(det) < 1e-14) return -1e30;
  const double b1 = div_rn(dot_rn(p, bc), det);
  const double b2 = div_rn(dot_rn(a, cross_rn(p, c)), det);
  const double b3 = div_rn(dot_rn(a, cross_rn(b, p)), det);
  const double s = add_rn(add_rn(b1, b2), b3);
  if (s <= 1e-14) return -1e30;
  const double s1 = div_rn(b1, s), s2 = div_rn(b2, s), s3 = div_rn(b3, s);
  double m = s1;
  if (s2 < m) m = s2;
  if (s3 < m) m = s3;
  return m;
}

// Divide-free screen for the containment DECISION min_score >= -1e-10.
// The three numerators d_k are the reference's exact expressions; only the
// divisions by det and by the sum are replaced by reciprocal multiplies. Each
// replaced division moves a quotient by <= 2 ulp, so the screened score is
// within ~2.5e-15 * max(|s|, 1) of the exact one; a guard band of 1e-13
// around the threshold (and around the sum <= 1e-14 test) sends every
// possibly-flipped case to the exact path. Returns 1 contained, 0 not,
// -1 undecided (caller evaluates min_score_rn).
SSUM_HD int contains_screen(d3 a, d3 b, d3 c, d3 bc, double det, double inv_det, d3 p) {
  if (fabs(det) < 1e-14) return 0;  // exact test, same operands as min_score_rn
  const double b1 = dot_rn(p, bc) * inv_det;
  const double b2 = dot_rn(a, cross_rn(p, c)) * inv_det;
  const double b3 = dot_rn(a, cross_rn(b, p)) * inv_det;
  const double s = (b1 + b2) + b3;
  if (fabs(s - 1e-14) <= 1e-13) return -1;
  if (s <= 1e-14) return 0;
  const double inv = 1.0 / s;
  double m = b1 * inv;
  const double m2 = b2 * inv, m3 = b3 * inv;
  if (m2 < m) m = m2;
  if (m3 < m) m = m3;
  if (fabs(m + 1e-10) <= 1e-13) return -1;
  return m >= -1e-10 ? 1 : 0;
}

// triangle_contains (geometry.cpp:85-92) via solve_vertex_basis
// (geometry.cpp:14-25): raw_k = triple(...) / det, normalised by their sum.
SSUM_HD bool contains_rn(d3 v1, d3 v2, d3 v3, d3 p) {
  const double det = dot_rn(v1, cross_rn(v2, v3));
  if (fabs(det) < 1e-14) return false;
  const double r0 = div_rn(dot_rn(p, cross_rn(v2, v3)), det);
  const double r1 = div_rn(dot_rn(v1, cross_rn(p, v3)), det);
  const double r2 = div_rn(dot_rn(v1, cross_rn(v2, p)), det);
  const double s = add_rn(add_rn(r0, r1), r2);
  if (s <= 1e-14) return false;
  return div_rn(r0, s) >= -1e-10 && div_rn(r1, s) >= -1e-10 && div_rn(r2, s) >= -1e-10;
}

// triangle_circumcenter (geometry.cpp:71-79)
SSUM_HD d3 circumcenter_rn(d3 v1, d3 v2, d3 v3, int* bad) {
  const d3 n = cross_rn(sub3(v2, v1), sub3(v3, v1));
  if (sqrt_rn(dot_rn(n, n)) < 1e-14) *bad = 1;
  d3 c = unit_rn(n, bad);
  const d3 cen = add3(add3(v1, v2), v3);
  if (dot_rn(c, cen) < 0.0) c = unit_rn(d3{-n.x, -n.y, -n.z}, bad);
  return c;
}

// SphericalTriangle ctor guards (geometry.cpp:27-39)
SSUM_HD bool triangle_ok(d3 a, d3 b, d3 c) {
  if (arc_dist(a, b) <= 1e-12 || arc_dist(b, c) <= 1e-12 || arc_dist(c, a) <= 1e-12) return false;
  return dot_rn(a, cross_rn(b, c)) > 0.0;
}

}  // namespace ssum
