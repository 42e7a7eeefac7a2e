// Host-side fixture generators for the BASELINE.json configs. These build the
// INPUTS of the hot path (they are not on it): icosahedral mesh vertices and
// their node-patch (spherical Voronoi) areas, the BASELINE Rossby-Haurwitz
// field, and the seeded random-cap point set of config 3.
//
// The mesh reproduces make_icosa_mesh(L).vertices() / node_patch_areas()
// (icosa_mesh.cpp:10-106) bit for bit — same vertex numbering, same
// arithmetic — with an adjacency-list midpoint table instead of a std::map and
// the per-vertex area loop spread over threads (results are independent of
// the thread count). Compiled with -ffp-contract=off.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <utility>
#include <vector>

#include "../../include/spheresum_b200.h"
#include "geom.cuh"

namespace {

using ssum::d3;

constexpr double kPi = 3.14159265358979323846;

d3 unit_of(double x, double y, double z) {
  int bad = 0;
  return ssum::unit_rn(d3{x, y, z}, &bad);
}

d3 latlon(double lat, double lon) {
  const double cl = std::cos(lat);
  return unit_of(cl * std::cos(lon), cl * std::sin(lon), std::sin(lat));
}

struct Mesh {
  std::vector<d3> v;
  std::vector<std::array<int, 3>> faces;  // finest level
};

// base_icosahedron + refine (icosa_mesh.cpp:10-64)
Mesh build_mesh(int level) {
  Mesh m;
  m.v.reserve(size_t(10) * (size_t(1) << (2 * level)) + 2);
  m.v.push_back(unit_of(0.0, 0.0, 1.0));
  const double rl = std::atan(0.5);
  for (int k = 0; k < 5; ++k) m.v.push_back(latlon(rl, 2.0 * kPi * k / 5.0));
  for (int k = 0; k < 5; ++k) m.v.push_back(latlon(-rl, 2.0 * kPi * k / 5.0 + kPi / 5.0));
  m.v.push_back(unit_of(0.0, 0.0, -1.0));
  for (int k = 0; k < 5; ++k) {
    const int u = 1 + k, un = 1 + (k + 1) % 5, l = 6 + k, ln = 6 + (k + 1) % 5;
    m.faces.push_back({0, u, un});
    m.faces.push_back({u, l, un});
    m.faces.push_back({un, l, ln});
    m.faces.push_back({11, ln, l});
  }
  for (int r = 0; r < level; ++r) {
    // midpoint table: per lower vertex id, (higher id, midpoint id), <= 6 entries
    std::vector<std::vector<std::pair<int, int>>> mid(m.v.size());
    auto midpoint = [&](int a, int b) {
      const int lo = std::min(a, b), hi = std::max(a, b);
      for (const auto& e : mid[size_t(lo)])
        if (e.first == hi) return e.second;
      const int id = static_cast<int>(m.v.size());
      const d3 pa = m.v[size_t(a)], pb = m.v[size_t(b)];
      m.v.push_back(unit_of(pa.x + pb.x, pa.y + pb.y, pa.z + pb.z));
      mid[size_t(lo)].emplace_back(hi, id);
      return id;
    };
    std::vector<std::array<int, 3>> kids(m.faces.size() * 4);
    for (size_t f = 0; f < m.faces.size(); ++f) {
      const auto p = m.faces[f];
      const int mab = midpoint(p[0], p[1]);
      const int mbc = midpoint(p[1], p[2]);
      const int mca = midpoint(p[2], p[0]);
      kids[4 * f + 0] = {p[0], mab, mca};
      kids[4 * f + 1] = {mab, p[1], mbc};
      kids[4 * f + 2] = {mca, mbc, p[2]};
      kids[4 * f + 3] = {mab, mbc, mca};
    }
    m.faces.swap(kids);
  }
  return m;
}

double dot(d3 a, d3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
d3 cross(d3 a, d3 b) { return {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x}; }
double norm(d3 a) { return std::sqrt(dot(a, a)); }

// node_patch_areas (icosa_mesh.cpp:75-106) with spherical_polygon_area
// (geometry.cpp:94-108)
std::vector<double> patch_areas(const Mesh& m) {
  const size_t nf = m.faces.size(), nv = m.v.size();
  std::vector<d3> centers(nf);
  int bad = 0;
  for (size_t f = 0; f < nf; ++f) {
    const auto& fc = m.faces[f];
    centers[f] = ssum::circumcenter_rn(m.v[size_t(fc[0])], m.v[size_t(fc[1])], m.v[size_t(fc[2])], &bad);
  }
  // incident faces per vertex in face order (the reference appends in face order)
  std::vector<int> deg(nv + 1, 0);
  for (const auto& fc : m.faces)
    for (int c : fc) deg[size_t(c) + 1]++;
  for (size_t i = 0; i < nv; ++i) deg[i + 1] += deg[i];
  std::vector<int> inc(static_cast<size_t>(deg[nv]));
  {
    std::vector<int> fill(deg.begin(), deg.end() - 1);
    for (size_t f = 0; f < nf; ++f)
      for (int c : m.faces[f]) inc[size_t(fill[size_t(c)]++)] = static_cast<int>(f);
  }
  std::vector<double> areas(nv, 0.0);
  auto work = [&](size_t lo, size_t hi) {
    std::vector<std::pair<double, int>> around;
    std::vector<d3> poly;
    for (size_t vi = lo; vi < hi; ++vi) {
      const d3 v = m.v[vi];
      around.clear();
      const d3 seed = std::abs(v.z) < 0.9 ? d3{0, 0, 1} : d3{1, 0, 0};
      const d3 c1 = cross(seed, v);
      const d3 e1 = unit_of(c1.x, c1.y, c1.z);
      const d3 e2 = cross(v, e1);
      for (int k = deg[vi]; k < deg[vi + 1]; ++k) {
        const int f = inc[size_t(k)];
        const d3 c = centers[size_t(f)];
        const double s = dot(c, v);
        const d3 d{c.x - v.x * s, c.y - v.y * s, c.z - v.z * s};
        around.emplace_back(std::atan2(dot(d, e2), dot(d, e1)), f);
      }
      std::sort(around.begin(), around.end());
      poly.clear();
      for (const auto& e : around) poly.push_back(centers[size_t(e.second)]);
      const size_t n = poly.size();
      double angle_sum = 0.0;
      for (size_t i = 0; i < n; ++i) {
        const d3 prev = poly[(i + n - 1) % n], here = poly[i], next = poly[(i + 1) % n];
        const double sp = dot(prev, here), sn = dot(next, here);
        const d3 tp{prev.x - here.x * sp, prev.y - here.y * sp, prev.z - here.z * sp};
        const d3 tn{next.x - here.x * sn, next.y - here.y * sn, next.z - here.z * sn};
        angle_sum += std::atan2(norm(cross(tp, tn)), dot(tp, tn));
      }
      areas[vi] = angle_sum - (static_cast<double>(n) - 2.0) * kPi;
    }
  };
  const size_t nt = std::max<size_t>(1, std::min<size_t>(std::thread::hardware_concurrency(), 32));
  std::vector<std::thread> pool;
  for (size_t t = 0; t < nt; ++t) pool.emplace_back(work, nv * t / nt, nv * (t + 1) / nt);
  for (auto& th : pool) th.join();
  return areas;
}

// Random numbers: splitmix64-seeded xoshiro256** (public-domain algorithms of
// Vigna / Blackman), uniform doubles from the top 53 bits.
struct Rng {
  uint64_t s[4];
  static uint64_t splitmix(uint64_t& x) {
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
  }
  explicit Rng(uint64_t seed) {
    for (auto& w : s) w = splitmix(seed);
  }
  static uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
  uint64_t next() {
    const uint64_t r = rotl(s[1] * 5, 7) * 9;
    const uint64_t t = s[1] << 17;
    s[2] ^= s[0];
    s[3] ^= s[1];
    s[1] ^= s[2];
    s[0] ^= s[3];
    s[2] ^= t;
    s[3] = rotl(s[3], 45);
    return r;
  }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }           // [0, 1)
  double uniform_open() { return (static_cast<double>(next() >> 11) + 0.5) * 0x1.0p-53; }  // (0, 1)
  double normal() {  // Box-Muller, one value per call
    const double u1 = uniform_open(), u2 = uniform();
    return std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
  }
};

d3 cap_center() { return latlon(40.0 * kPi / 180.0, 0.0); }

d3 draw_point(Rng& rng, bool in_cap) {
  if (!in_cap) {
    for (;;) {
      const double x = rng.normal(), y = rng.normal(), z = rng.normal();
      if (x * x + y * y + z * z > 1e-20) return unit_of(x, y, z);
    }
  }
  // uniform in area on the cap of angular radius 10 deg about x0
  const double c10 = std::cos(10.0 * kPi / 180.0);
  const double zp = c10 + (1.0 - c10) * rng.uniform();
  const double ph = 2.0 * kPi * rng.uniform();
  const double rp = std::sqrt(std::max(0.0, 1.0 - zp * zp));
  const double lat0 = 40.0 * kPi / 180.0;
  const d3 e3 = cap_center();
  const d3 e1{-std::sin(lat0), 0.0, std::cos(lat0)};  // north at x0
  const d3 e2{0.0, 1.0, 0.0};                          // east at x0
  const double a = rp * std::cos(ph), b = rp * std::sin(ph);
  return unit_of(a * e1.x + b * e2.x + zp * e3.x, a * e1.y + b * e2.y + zp * e3.y, a * e1.z + b * e2.z + zp * e3.z);
}

// Indices j > i with 1 - x_i.x_j <= 1e-12 (reference rounding) for some i < j.
std::vector<int64_t> near_duplicates(const std::vector<d3>& p) {
  const double h = 1.0 / (1 << 19);  // cell edge > chord sqrt(2e-12) ~ 1.414e-6
  const int64_t n = static_cast<int64_t>(p.size());
  auto cell = [&](double v) { return static_cast<int64_t>(std::floor((v + 1.0) / h)); };
  auto key = [&](int64_t a, int64_t b, int64_t c) { return (a << 42) | (b << 21) | c; };
  std::vector<std::pair<int64_t, int64_t>> ks(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) ks[size_t(i)] = {key(cell(p[size_t(i)].x), cell(p[size_t(i)].y), cell(p[size_t(i)].z)), i};
  std::sort(ks.begin(), ks.end());
  std::vector<char> bad(size_t(n), 0);
  for (int64_t i = 0; i < n; ++i) {
    const d3 x = p[size_t(i)];
    const int64_t cx = cell(x.x), cy = cell(x.y), cz = cell(x.z);
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const int64_t k = key(cx + dx, cy + dy, cz + dz);
          auto it = std::lower_bound(ks.begin(), ks.end(), std::make_pair(k, int64_t(-1)));
          for (; it != ks.end() && it->first == k; ++it) {
            const int64_t j = it->second;
            if (j <= i) continue;
            const d3 y = p[size_t(j)];
            const double den = 1.0 - ((x.x * y.x + x.y * y.y) + x.z * y.z);
            if (den <= 1e-12) bad[size_t(j)] = 1;
          }
        }
  }
  std::vector<int64_t> out;
  for (int64_t j = 0; j < n; ++j)
    if (bad[size_t(j)]) out.push_back(j);
  return out;
}

}  // namespace

extern "C" {

int64_t ssum_mesh_vertex_count(int level) {
  if (level < 0 || level > 12) return -1;
  return 10 * (int64_t(1) << (2 * level)) + 2;
}

int ssum_make_icosa_mesh(int level, double* xyz, double* area) {
  if (level < 0 || level > 12 || !xyz) return SSUM_INVALID;
  try {
    const Mesh m = build_mesh(level);
    for (size_t i = 0; i < m.v.size(); ++i) {
      xyz[3 * i] = m.v[i].x;
      xyz[3 * i + 1] = m.v[i].y;
      xyz[3 * i + 2] = m.v[i].z;
    }
    if (area) {
      const std::vector<double> a = patch_areas(m);
      std::memcpy(area, a.data(), a.size() * sizeof(double));
    }
  } catch (...) {
    return SSUM_NOMEM;
  }
  return SSUM_OK;
}

// lat = asin(clamp(z)), lon = atan2(y, x) with the [-pi, pi) convention
// (unit_to_latlon, geometry.cpp:46-53).
int ssum_rh4_vorticity(const double* xyz, int64_t n, double* zeta) {
  if (n < 0 || (n > 0 && (!xyz || !zeta))) return SSUM_INVALID;
  for (int64_t i = 0; i < n; ++i) {
    const double lat = std::asin(std::clamp(xyz[3 * i + 2], -1.0, 1.0));
    double lon = std::atan2(xyz[3 * i + 1], xyz[3 * i]);
    if (lon >= kPi) lon -= 2.0 * kPi;
    const double st = std::sin(lat), ct = std::cos(lat);
    zeta[i] = 2.0 * st - 30.0 * st * ct * ct * ct * ct * std::cos(4.0 * lon);
  }
  return SSUM_OK;
}

int ssum_make_random_cap(int64_t n, uint64_t seed, double* xyz, double* zeta, double* area) {
  if (n < 2 || !xyz || !zeta || !area) return SSUM_INVALID;
  try {
    Rng rng(seed);
    const int64_t half = n / 2;
    std::vector<d3> p(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) p[size_t(i)] = draw_point(rng, i >= half);
    for (int round = 0; round < 64; ++round) {
      const std::vector<int64_t> bad = near_duplicates(p);
      if (bad.empty()) break;
      for (const int64_t j : bad) p[size_t(j)] = draw_point(rng, j >= half);
      if (round == 63) return SSUM_GEOMETRY;
    }
    const d3 x0 = cap_center();
    const double a = 4.0 * kPi / static_cast<double>(n);
    double circ = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      const d3 x = p[size_t(i)];
      xyz[3 * i] = x.x;
      xyz[3 * i + 1] = x.y;
      xyz[3 * i + 2] = x.z;
      zeta[i] = std::exp(-16.0 * (1.0 - dot(x, x0)));
      area[i] = a;
      circ += zeta[i] * a;
    }
    const double mean = circ / (4.0 * kPi);
    for (int64_t i = 0; i < n; ++i) zeta[i] -= mean;
  } catch (...) {
    return SSUM_NOMEM;
  }
  return SSUM_OK;
}

}  // extern "C"
