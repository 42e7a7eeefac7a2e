/*
 * ORACLE TEST INFRASTRUCTURE — not product code.
 *
 * A plain-C restatement of the reference tree code's velocity / stream-function
 * path (arXiv 2401.07361 reference, /root/reference/proj). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it, and only
 * as a checker. It is pinned against the unmodified reference compiled into
 * oracle/_ref/ (tests/test_oracle_pin.py: identical trees, identical
 * interaction lists, velocities within 1e-14).
 *
 * It adds the one traversal mode BASELINE config 2 asks for that the reference
 * lacks: particle-cluster-only ("pc_only"), i.e. the reference recursion with
 * classify() remapping CP->PP and CC->PC.
 *
 * Build: oracle/Makefile, `-O2 -std=c11 -ffp-contract=off` so every product
 * and sum rounds separately, as the reference's do.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

enum { ORC_OK = 0, ORC_CONFIG = 1, ORC_GEOMETRY = 2, ORC_SINGULAR = 3, ORC_CONDITIONING = 4, ORC_NOMEM = 8 };
enum { KIND_PP = 0, KIND_PC = 1, KIND_CP = 2, KIND_CC = 3 };

static int g_status; /* first error raised in the current call */
static void raise_err(int code) {
  if (g_status == ORC_OK) g_status = code;
}

/* ------------------------------------------------------------------ geometry
 * geometry.hpp:13-76 / geometry.cpp:10-125 */
typedef struct {
  double x, y, z;
} v3;

static v3 v3add(v3 a, v3 b) { v3 r = {a.x + b.x, a.y + b.y, a.z + b.z}; return r; }
static v3 v3sub(v3 a, v3 b) { v3 r = {a.x - b.x, a.y - b.y, a.z - b.z}; return r; }
static v3 v3scale(double s, v3 a) { v3 r = {a.x * s, a.y * s, a.z * s}; return r; }
static double v3dot(v3 a, v3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
static v3 v3cross(v3 a, v3 b) {
  v3 r = {a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x};
  return r;
}
static double v3norm(v3 a) { return sqrt(v3dot(a, a)); }

/* UnitVector3 constructor (geometry.hpp:55-61): divide by the norm. */
static v3 unitv(double x, double y, double z) {
  const double n = sqrt(x * x + y * y + z * z);
  v3 r = {1.0, 0.0, 0.0};
  if (!(n > 1e-300)) {
    raise_err(ORC_GEOMETRY);
    return r;
  }
  r.x = x / n;
  r.y = y / n;
  r.z = z / n;
  return r;
}
static v3 unit_of(v3 a) { return unitv(a.x, a.y, a.z); }

static double triple3(v3 a, v3 b, v3 c) { return v3dot(a, v3cross(b, c)); }

/* geometry.cpp:55-57 */
static double arc_dist(v3 a, v3 b) { return atan2(v3norm(v3cross(a, b)), v3dot(a, b)); }

/* geometry.cpp:14-25 (Cramer), returns 0 when |det| < 1e-14 */
static int raw_bary(const v3* t, v3 p, double out[3]) {
  const double det = triple3(t[0], t[1], t[2]);
  if (fabs(det) < 1e-14) return 0;
  out[0] = triple3(p, t[1], t[2]) / det;
  out[1] = triple3(t[0], p, t[2]) / det;
  out[2] = triple3(t[0], t[1], p) / det;
  return 1;
}

/* geometry.cpp:59-69 */
static void sph_bary(const v3* t, v3 p, double b[3]) {
  double r[3];
  if (!raw_bary(t, p, r)) {
    raise_err(ORC_GEOMETRY);
    b[0] = b[1] = b[2] = 0.0;
    return;
  }
  const double s = r[0] + r[1] + r[2];
  if (fabs(s) < 1e-14) {
    raise_err(ORC_GEOMETRY);
    b[0] = b[1] = b[2] = 0.0;
    return;
  }
  b[0] = r[0] / s;
  b[1] = r[1] / s;
  b[2] = r[2] / s;
}

/* geometry.cpp:85-92 */
static int tri_contains(const v3* t, v3 p) {
  double r[3];
  if (!raw_bary(t, p, r)) return 0;
  const double s = r[0] + r[1] + r[2];
  if (s <= 1e-14) return 0;
  return r[0] / s >= -1e-10 && r[1] / s >= -1e-10 && r[2] / s >= -1e-10;
}

/* geometry.cpp:114-125 */
static double min_score(const v3* t, v3 p) {
  const v3 bc = v3cross(t[1], t[2]);
  const double det = v3dot(t[0], bc);
  if (fabs(det) < 1e-14) return -1e30;
  const double b1 = v3dot(p, bc) / det;
  const double b2 = v3dot(t[0], v3cross(p, t[2])) / det;
  const double b3 = v3dot(t[0], v3cross(t[1], p)) / det;
  const double s = b1 + b2 + b3;
  if (s <= 1e-14) return -1e30;
  double m = b1 / s;
  if (b2 / s < m) m = b2 / s;
  if (b3 / s < m) m = b3 / s;
  return m;
}

/* geometry.cpp:71-79 */
static v3 circumcenter(const v3* t) {
  const v3 n = v3cross(v3sub(t[1], t[0]), v3sub(t[2], t[0]));
  if (v3norm(n) < 1e-14) raise_err(ORC_GEOMETRY);
  v3 c = unit_of(n);
  const v3 cen = v3add(v3add(t[0], t[1]), t[2]);
  if (v3dot(c, cen) < 0.0) c = unitv(-n.x, -n.y, -n.z);
  return c;
}

/* SphericalTriangle ctor checks (geometry.cpp:27-39) */
static void check_triangle(const v3* t) {
  if (arc_dist(t[0], t[1]) <= 1e-12 || arc_dist(t[1], t[2]) <= 1e-12 || arc_dist(t[2], t[0]) <= 1e-12)
    raise_err(ORC_GEOMETRY);
  if (triple3(t[0], t[1], t[2]) <= 0.0) raise_err(ORC_GEOMETRY);
}

/* ------------------------------------------------------------- face tree
 * face_tree.hpp:12-58 / face_tree.cpp:9-95; base faces icosa_mesh.cpp:10-35 */
typedef struct {
  v3 tri[3];
  v3 center;
  double radius;
  int level, parent, child_base;
  int* bin;
  int nbin, capbin;
} node_t;

typedef struct {
  node_t* nodes;
  int count, cap;
  int* leaf_of;
  int64_t n;
} tree_t;

static int add_node(tree_t* T, v3 a, v3 b, v3 c) {
  if (T->count == T->cap) {
    T->cap = T->cap ? 2 * T->cap : 64;
    T->nodes = (node_t*)realloc(T->nodes, sizeof(node_t) * (size_t)T->cap);
  }
  node_t* nd = &T->nodes[T->count];
  memset(nd, 0, sizeof(*nd));
  nd->tri[0] = a;
  nd->tri[1] = b;
  nd->tri[2] = c;
  check_triangle(nd->tri);
  nd->center = circumcenter(nd->tri);
  nd->radius = arc_dist(nd->center, a);
  nd->parent = -1;
  nd->child_base = -1;
  return T->count++;
}

static void bin_push(node_t* nd, int id) {
  if (nd->nbin == nd->capbin) {
    nd->capbin = nd->capbin ? 2 * nd->capbin : 16;
    nd->bin = (int*)realloc(nd->bin, sizeof(int) * (size_t)nd->capbin);
  }
  nd->bin[nd->nbin++] = id;
}

static v3 latlon_unit(double lat, double lon) {
  const double cl = cos(lat);
  return unitv(cl * cos(lon), cl * sin(lon), sin(lat));
}

static void tree_init(tree_t* T) {
  memset(T, 0, sizeof(*T));
  v3 v[12];
  v[0] = unitv(0.0, 0.0, 1.0);
  const double rl = atan(0.5);
  for (int k = 0; k < 5; ++k) v[1 + k] = latlon_unit(rl, 2.0 * M_PI * k / 5.0);
  for (int k = 0; k < 5; ++k) v[6 + k] = latlon_unit(-rl, 2.0 * M_PI * k / 5.0 + M_PI / 5.0);
  v[11] = unitv(0.0, 0.0, -1.0);
  for (int k = 0; k < 5; ++k) {
    const int u = 1 + k, un = 1 + (k + 1) % 5, l = 6 + k, ln = 6 + (k + 1) % 5;
    add_node(T, v[0], v[u], v[un]);
    add_node(T, v[u], v[l], v[un]);
    add_node(T, v[un], v[l], v[ln]);
    add_node(T, v[11], v[ln], v[l]);
  }
}

static void tree_free(tree_t* T) {
  for (int i = 0; i < T->count; ++i) free(T->nodes[i].bin);
  free(T->nodes);
  free(T->leaf_of);
  memset(T, 0, sizeof(*T));
}

/* face_tree.cpp:18-37 */
static void make_children(tree_t* T, int id) {
  if (T->nodes[id].child_base >= 0) return;
  const v3 a = T->nodes[id].tri[0], b = T->nodes[id].tri[1], c = T->nodes[id].tri[2];
  const v3 m12 = unit_of(v3add(a, b)), m23 = unit_of(v3add(b, c)), m31 = unit_of(v3add(c, a));
  const int lvl = T->nodes[id].level + 1;
  const int base = add_node(T, a, m12, m31);
  add_node(T, m12, b, m23);
  add_node(T, m31, m23, c);
  add_node(T, m12, m23, m31);
  T->nodes[id].child_base = base;
  for (int k = base; k < base + 4; ++k) {
    T->nodes[k].level = lvl;
    T->nodes[k].parent = id;
  }
}

/* face_tree.cpp:39-71 */
static void distribute(tree_t* T, int id, const v3* pos, int nt, int max_depth) {
  if (T->nodes[id].nbin == 0) return;
  if (T->nodes[id].child_base < 0) {
    if (T->nodes[id].nbin <= nt || T->nodes[id].level >= max_depth) {
      for (int k = 0; k < T->nodes[id].nbin; ++k) T->leaf_of[T->nodes[id].bin[k]] = id;
      return;
    }
    make_children(T, id);
  }
  const int cb = T->nodes[id].child_base;
  for (int k = 0; k < T->nodes[id].nbin; ++k) {
    const int i = T->nodes[id].bin[k];
    int best = cb, placed = 0;
    double best_s = -1e300;
    for (int c = cb; c < cb + 4; ++c) {
      const double s = min_score(T->nodes[c].tri, pos[i]);
      if (s >= -1e-10) {
        bin_push(&T->nodes[c], i);
        placed = 1;
        break;
      }
      if (s > best_s) {
        best_s = s;
        best = c;
      }
    }
    if (!placed) bin_push(&T->nodes[best], i);
  }
  for (int c = cb; c < cb + 4; ++c) distribute(T, c, pos, nt, max_depth);
}

/* face_tree.cpp:73-88 */
static void bin_particles(tree_t* T, const v3* pos, int64_t n, int nt, int max_depth) {
  for (int i = 0; i < T->count; ++i) T->nodes[i].nbin = 0;
  free(T->leaf_of);
  T->leaf_of = (int*)malloc(sizeof(int) * (size_t)(n ? n : 1));
  T->n = n;
  for (int64_t i = 0; i < n; ++i) T->leaf_of[i] = -1;
  for (int64_t i = 0; i < n; ++i) {
    int placed = 0;
    for (int f = 0; f < 20 && !placed; ++f) {
      if (tri_contains(T->nodes[f].tri, pos[i])) {
        bin_push(&T->nodes[f], (int)i);
        placed = 1;
      }
    }
    if (!placed) {
      raise_err(ORC_GEOMETRY);
      return;
    }
  }
  for (int f = 0; f < 20; ++f) distribute(T, f, pos, nt, max_depth);
}

/* ------------------------------------------------------------- traversal
 * treecode.cpp:22-77 */
typedef struct {
  int* tsk;
  int64_t count, cap;
} ilist_t;

static void emit(ilist_t* L, int t, int s, int kind) {
  if (L->count == L->cap) {
    L->cap = L->cap ? 2 * L->cap : 1024;
    L->tsk = (int*)realloc(L->tsk, sizeof(int) * 3 * (size_t)L->cap);
  }
  L->tsk[3 * L->count] = t;
  L->tsk[3 * L->count + 1] = s;
  L->tsk[3 * L->count + 2] = kind;
  L->count++;
}

typedef struct {
  double theta;
  int nt, degree, max_depth, pc_only;
} cfg_t;

static int classify(int nt_, int ns_, const cfg_t* c) {
  const int tb = nt_ > c->nt, sb = ns_ > c->nt;
  int k = KIND_PP;
  if (tb && sb) k = KIND_CC;
  else if (sb) k = KIND_PC;
  else if (tb) k = KIND_CP;
  if (c->pc_only) { /* particle-cluster-only mode: targets are never clusters */
    if (k == KIND_CP) k = KIND_PP;
    if (k == KIND_CC) k = KIND_PC;
  }
  return k;
}

static void traverse(const tree_t* T, const cfg_t* c, int t, int s, ilist_t* L) {
  const node_t* tn = &T->nodes[t];
  const node_t* sn = &T->nodes[s];
  if (tn->nbin == 0 || sn->nbin == 0) return;
  const double R = arc_dist(tn->center, sn->center);
  if (R > 0.0 && (tn->radius + sn->radius) / R < c->theta) {
    emit(L, t, s, classify(tn->nbin, sn->nbin, c));
    return;
  }
  if (tn->nbin <= c->nt && sn->nbin <= c->nt) {
    emit(L, t, s, KIND_PP);
    return;
  }
  const int rt = tn->nbin > sn->nbin;
  const node_t* r = rt ? tn : sn;
  if (r->child_base < 0 || r->level >= c->max_depth) {
    emit(L, t, s, KIND_PP);
    return;
  }
  for (int k = r->child_base; k < r->child_base + 4; ++k) {
    if (rt) traverse(T, c, k, s, L);
    else traverse(T, c, t, k, L);
  }
}

static void dual_traversal(const tree_t* T, const cfg_t* c, ilist_t* L) {
  for (int t = 0; t < 20; ++t)
    for (int s = 0; s < 20; ++s) traverse(T, c, t, s, L);
}

/* ------------------------------------------------------------------ SBB
 * sbb.cpp:13-38 (basis, index order), :46-66 (lattice proxies), :68-138 (fit) */
typedef struct {
  int d, p;
  int (*ijk)[3];
  double* lu; /* p x p, row-major, packed L\U */
  int* perm;
} sbb_t;

static void sbb_eval(const sbb_t* B, const double b[3], double* out) {
  double p1[21], p2[21], p3[21];
  p1[0] = p2[0] = p3[0] = 1.0;
  for (int n = 1; n <= B->d; ++n) {
    p1[n] = p1[n - 1] * b[0];
    p2[n] = p2[n - 1] * b[1];
    p3[n] = p3[n - 1] * b[2];
  }
  for (int m = 0; m < B->p; ++m) out[m] = p1[B->ijk[m][0]] * p2[B->ijk[m][1]] * p3[B->ijk[m][2]];
}

static void lattice_bary(const sbb_t* B, int m, double b[3]) {
  const double d = (double)B->d;
  b[0] = B->ijk[m][0] / d;
  b[1] = B->ijk[m][1] / d;
  b[2] = B->ijk[m][2] / d;
}

static int sbb_init(sbb_t* B, int d) {
  B->d = d;
  B->p = (d + 1) * (d + 2) / 2;
  B->ijk = malloc(sizeof(int[3]) * (size_t)B->p);
  int m = 0;
  for (int k = 0; k <= d; ++k)
    for (int j = 0; j <= d - k; ++j) {
      B->ijk[m][0] = d - k - j;
      B->ijk[m][1] = j;
      B->ijk[m][2] = k;
      ++m;
    }
  const int p = B->p;
  B->lu = malloc(sizeof(double) * (size_t)p * p);
  B->perm = malloc(sizeof(int) * (size_t)p);
  double b[3];
  for (int r = 0; r < p; ++r) {
    lattice_bary(B, r, b);
    sbb_eval(B, b, B->lu + (size_t)r * p); /* V[r][k] = B_k(b_r) */
  }
  /* partial-pivot LU, first largest |a| in the column wins */
  for (int i = 0; i < p; ++i) B->perm[i] = i;
  for (int k = 0; k < p; ++k) {
    int piv = k;
    double best = fabs(B->lu[(size_t)k * p + k]);
    for (int i = k + 1; i < p; ++i)
      if (fabs(B->lu[(size_t)i * p + k]) > best) {
        best = fabs(B->lu[(size_t)i * p + k]);
        piv = i;
      }
    if (piv != k) {
      for (int j = 0; j < p; ++j) {
        const double t = B->lu[(size_t)k * p + j];
        B->lu[(size_t)k * p + j] = B->lu[(size_t)piv * p + j];
        B->lu[(size_t)piv * p + j] = t;
      }
      const int t = B->perm[k];
      B->perm[k] = B->perm[piv];
      B->perm[piv] = t;
    }
    const double dk = B->lu[(size_t)k * p + k];
    if (dk == 0.0) return ORC_CONDITIONING;
    for (int i = k + 1; i < p; ++i) {
      B->lu[(size_t)i * p + k] /= dk;
      const double l = B->lu[(size_t)i * p + k];
      for (int j = k + 1; j < p; ++j) B->lu[(size_t)i * p + j] -= l * B->lu[(size_t)k * p + j];
    }
  }
  return ORC_OK;
}

static void sbb_free(sbb_t* B) {
  free(B->ijk);
  free(B->lu);
  free(B->perm);
}

/* V x = rhs (ProxyFit::solve, sbb.cpp:103-108) */
static void fit_solve(const sbb_t* B, const double* rhs, double* x) {
  const int p = B->p;
  for (int i = 0; i < p; ++i) x[i] = rhs[B->perm[i]];
  for (int i = 0; i < p; ++i)
    for (int k = 0; k < i; ++k) x[i] -= B->lu[(size_t)i * p + k] * x[k];
  for (int i = p - 1; i >= 0; --i) {
    for (int k = i + 1; k < p; ++k) x[i] -= B->lu[(size_t)i * p + k] * x[k];
    x[i] /= B->lu[(size_t)i * p + i];
  }
}

/* V^T x = rhs (ProxyFit::solve_transposed, sbb.cpp:110-115) */
static void fit_solve_t(const sbb_t* B, const double* rhs, double* x) {
  const int p = B->p;
  double y[231];
  for (int i = 0; i < p; ++i) y[i] = rhs[i];
  for (int i = 0; i < p; ++i) {
    for (int k = 0; k < i; ++k) y[i] -= B->lu[(size_t)k * p + i] * y[k];
    y[i] /= B->lu[(size_t)i * p + i];
  }
  for (int i = p - 1; i >= 0; --i)
    for (int k = i + 1; k < p; ++k) y[i] -= B->lu[(size_t)k * p + i] * y[k];
  for (int i = 0; i < p; ++i) x[B->perm[i]] = y[i];
}

/* proxy_points (sbb.cpp:46-66): normalise(b1 v1 + b2 v2 + b3 v3) */
static void proxy_pts(const sbb_t* B, const v3* t, v3* out) {
  double b[3];
  for (int m = 0; m < B->p; ++m) {
    lattice_bary(B, m, b);
    out[m] = unit_of(v3add(v3add(v3scale(b[0], t[0]), v3scale(b[1], t[1])), v3scale(b[2], t[2])));
  }
}

/* --------------------------------------------------------------- kernels
 * kernels.hpp:13-61. kernel 0 = Biot-Savart (dim 3), 1 = log potential (dim 1) */
static void kern(int kernel, v3 x, v3 y, double* out) {
  const double den = 1.0 - v3dot(x, y);
  if (den <= 1e-14) {
    raise_err(ORC_SINGULAR);
    out[0] = out[1] = out[2] = 0.0;
    return;
  }
  if (kernel == 0) {
    const v3 c = v3cross(x, y);
    const double inv = 1.0 / den;
    out[0] = c.x * inv;
    out[1] = c.y * inv;
    out[2] = c.z * inv;
  } else {
    out[0] = -log(den) / (4.0 * M_PI);
  }
}

static double prefactor(int kernel) { return kernel == 0 ? -1.0 / (4.0 * M_PI) : 1.0; }

/* ------------------------------------------------------------------ sums */
static v3* load_pts(const double* xyz, int64_t n) {
  v3* p = malloc(sizeof(v3) * (size_t)(n ? n : 1));
  for (int64_t i = 0; i < n; ++i) { /* values taken as given unit vectors, not renormalised */
    p[i].x = xyz[3 * i];
    p[i].y = xyz[3 * i + 1];
    p[i].z = xyz[3 * i + 2];
  }
  return p;
}

/* direct_sum (treecode.cpp:246-264) */
int orc_direct_sum(int kernel, const double* xyz, const double* q, int64_t n, double* out) {
  g_status = ORC_OK;
  const int D = kernel == 0 ? 3 : 1;
  v3* P = load_pts(xyz, n);
  const double pref = prefactor(kernel);
  double term[3];
  for (int64_t i = 0; i < n; ++i) {
    double acc[3] = {0, 0, 0};
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      kern(kernel, P[i], P[j], term);
      for (int d = 0; d < D; ++d) acc[d] += term[d] * q[j];
    }
    for (int d = 0; d < D; ++d) out[i * D + d] = pref * acc[d];
  }
  free(P);
  return g_status;
}

static int cmp_int(const void* a, const void* b) {
  const int x = *(const int*)a, y = *(const int*)b;
  return (x > y) - (x < y);
}

typedef struct {
  int* v;
  int n, cap;
} ivec;
static void ivec_push(ivec* a, int x) {
  if (a->n == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 4;
    a->v = realloc(a->v, sizeof(int) * (size_t)a->cap);
  }
  a->v[a->n++] = x;
}

static int check_cfg(const cfg_t* c) {
  if (!(c->theta > 0.0 && c->theta <= 1.0)) return ORC_CONFIG;
  if (c->nt < 1) return ORC_CONFIG;
  if (c->degree < 1 || c->degree > 20) return ORC_CONFIG;
  if (c->max_depth < 1 || c->max_depth > 40) return ORC_CONFIG;
  return ORC_OK;
}

/* treecode_sum (treecode.cpp:266-413). counts4 (nullable) receives the
 * PP/PC/CP/CC interaction counts. */
int orc_treecode_sum(int kernel, const double* xyz, const double* q, int64_t n, double theta, int nt,
                     int degree, int max_depth, int pc_only, double* out, int64_t* counts4) {
  g_status = ORC_OK;
  const cfg_t c = {theta, nt, degree, max_depth, pc_only};
  if (check_cfg(&c) != ORC_OK) return ORC_CONFIG;
  const int D = kernel == 0 ? 3 : 1;
  v3* P = load_pts(xyz, n);
  tree_t T;
  tree_init(&T);
  bin_particles(&T, P, n, nt, max_depth);
  if (g_status != ORC_OK) {
    tree_free(&T);
    free(P);
    return g_status;
  }
  ilist_t L = {0};
  dual_traversal(&T, &c, &L);
  sbb_t B;
  if (sbb_init(&B, degree) != ORC_OK) return ORC_CONDITIONING;
  const int p = B.p, nn = T.count;

  /* bucketing (treecode.cpp:289-324) */
  ivec* pp = calloc((size_t)nn, sizeof(ivec));
  ivec* pc = calloc((size_t)nn, sizeof(ivec));
  ivec* ct = calloc((size_t)nn, sizeof(ivec)); /* encoded 2*s + (kind==CC) */
  char* need_proxy = calloc((size_t)nn, 1);
  char* need_w = calloc((size_t)nn, 1);
  if (counts4) memset(counts4, 0, 4 * sizeof(int64_t));
  for (int64_t k = 0; k < L.count; ++k) {
    const int t = L.tsk[3 * k], s = L.tsk[3 * k + 1], kind = L.tsk[3 * k + 2];
    if (counts4) counts4[kind]++;
    if (kind == KIND_PP) ivec_push(&pp[t], s);
    else if (kind == KIND_PC) {
      ivec_push(&pc[t], s);
      need_proxy[s] = need_w[s] = 1;
    } else if (kind == KIND_CP) {
      ivec_push(&ct[t], 2 * s);
      need_proxy[t] = 1;
    } else {
      ivec_push(&ct[t], 2 * s + 1);
      need_proxy[t] = need_proxy[s] = need_w[s] = 1;
    }
  }

  /* Phase 1: proxy points */
  v3** prox = calloc((size_t)nn, sizeof(v3*));
  for (int id = 0; id < nn; ++id)
    if (need_proxy[id]) {
      prox[id] = malloc(sizeof(v3) * (size_t)p);
      proxy_pts(&B, T.nodes[id].tri, prox[id]);
    }
  /* Phase 2: w_hat = V^-T sum_j B(beta_s(x_j)) q_j (treecode.cpp:79-91,157-166) */
  double** what = calloc((size_t)nn, sizeof(double*));
  double* bv = malloc(sizeof(double) * (size_t)p);
  double* w = malloc(sizeof(double) * (size_t)p);
  double b[3];
  for (int id = 0; id < nn; ++id)
    if (need_w[id]) {
      for (int k = 0; k < p; ++k) w[k] = 0.0;
      for (int k = 0; k < T.nodes[id].nbin; ++k) {
        const int j = T.nodes[id].bin[k];
        sph_bary(T.nodes[id].tri, P[j], b);
        sbb_eval(&B, b, bv);
        for (int m = 0; m < p; ++m) w[m] += bv[m] * q[j];
      }
      what[id] = malloc(sizeof(double) * (size_t)p);
      fit_solve_t(&B, w, what[id]);
    }
  /* Phase 3: CP / CC proxy potentials and the fit (treecode.cpp:341-358) */
  double** coeff = calloc((size_t)nn, sizeof(double*));
  double* phi = malloc(sizeof(double) * (size_t)p * 3);
  double term[3];
  for (int t = 0; t < nn; ++t) {
    if (ct[t].n == 0) continue;
    for (int k = 0; k < p * D; ++k) phi[k] = 0.0;
    for (int e = 0; e < ct[t].n; ++e) {
      const int s = ct[t].v[e] >> 1, is_cc = ct[t].v[e] & 1;
      for (int m = 0; m < p; ++m) {
        if (!is_cc) {
          for (int k = 0; k < T.nodes[s].nbin; ++k) {
            const int j = T.nodes[s].bin[k];
            kern(kernel, prox[t][m], P[j], term);
            for (int d = 0; d < D; ++d) phi[d * p + m] += term[d] * q[j];
          }
        } else {
          for (int k = 0; k < p; ++k) {
            kern(kernel, prox[t][m], prox[s][k], term);
            for (int d = 0; d < D; ++d) phi[d * p + m] += term[d] * what[s][k];
          }
        }
      }
    }
    coeff[t] = malloc(sizeof(double) * (size_t)p * D);
    for (int d = 0; d < D; ++d) fit_solve(&B, phi + d * p, coeff[t] + d * p);
  }
  /* Phase 4: per particle (treecode.cpp:360-404) */
  const double pref = prefactor(kernel);
  int* gather = NULL;
  size_t gcap = 0;
  for (int64_t i = 0; i < n; ++i) {
    int path[48], pl = 0;
    for (int id = T.leaf_of[i]; id >= 0; id = T.nodes[id].parent) path[pl++] = id;
    size_t g = 0;
    for (int r = pl - 1; r >= 0; --r)
      for (int e = 0; e < pp[path[r]].n; ++e) {
        const node_t* sn = &T.nodes[pp[path[r]].v[e]];
        if (g + (size_t)sn->nbin > gcap) {
          gcap = 2 * (g + (size_t)sn->nbin);
          gather = realloc(gather, sizeof(int) * gcap);
        }
        memcpy(gather + g, sn->bin, sizeof(int) * (size_t)sn->nbin);
        g += (size_t)sn->nbin;
      }
    qsort(gather, g, sizeof(int), cmp_int);
    double acc[3] = {0, 0, 0};
    for (size_t k = 0; k < g; ++k) {
      const int j = gather[k];
      if (j == i) continue;
      kern(kernel, P[i], P[j], term);
      for (int d = 0; d < D; ++d) acc[d] += term[d] * q[j];
    }
    for (int r = pl - 1; r >= 0; --r)
      for (int e = 0; e < pc[path[r]].n; ++e) {
        const int s = pc[path[r]].v[e];
        for (int m = 0; m < p; ++m) {
          kern(kernel, P[i], prox[s][m], term);
          for (int d = 0; d < D; ++d) acc[d] += term[d] * what[s][m];
        }
      }
    for (int r = pl - 1; r >= 0; --r) {
      const int t = path[r];
      if (!coeff[t]) continue;
      sph_bary(T.nodes[t].tri, P[i], b);
      sbb_eval(&B, b, bv);
      for (int d = 0; d < D; ++d) {
        double v = 0.0;
        for (int k = 0; k < p; ++k) v += coeff[t][d * p + k] * bv[k];
        acc[d] += v;
      }
    }
    for (int d = 0; d < D; ++d) out[i * D + d] = pref * acc[d];
  }

  free(gather);
  for (int id = 0; id < nn; ++id) {
    free(pp[id].v);
    free(pc[id].v);
    free(ct[id].v);
    free(prox[id]);
    free(what[id]);
    free(coeff[id]);
  }
  free(pp);
  free(pc);
  free(ct);
  free(prox);
  free(what);
  free(coeff);
  free(need_proxy);
  free(need_w);
  free(bv);
  free(w);
  free(phi);
  free(L.tsk);
  sbb_free(&B);
  tree_free(&T);
  free(P);
  return g_status;
}

/* Tree + list export for the pin tests. Nodes: level, parent, child_base,
 * bin size; leaf_of per particle; list triples (t, s, kind). Call with
 * null outputs first to size them (node_count, list_count). */
int orc_build_lists(const double* xyz, int64_t n, double theta, int nt, int max_depth, int pc_only,
                    int* node_count, int* level, int* parent, int* child_base, int* bin_size,
                    int* leaf_of, int64_t* list_count, int* tsk) {
  g_status = ORC_OK;
  const cfg_t c = {theta, nt, 1, max_depth, pc_only};
  if (check_cfg(&c) != ORC_OK) return ORC_CONFIG;
  v3* P = load_pts(xyz, n);
  tree_t T;
  tree_init(&T);
  bin_particles(&T, P, n, nt, max_depth);
  ilist_t L = {0};
  if (g_status == ORC_OK) dual_traversal(&T, &c, &L);
  *node_count = T.count;
  *list_count = L.count;
  for (int id = 0; id < T.count; ++id) {
    if (level) level[id] = T.nodes[id].level;
    if (parent) parent[id] = T.nodes[id].parent;
    if (child_base) child_base[id] = T.nodes[id].child_base;
    if (bin_size) bin_size[id] = T.nodes[id].nbin;
  }
  if (leaf_of) memcpy(leaf_of, T.leaf_of, sizeof(int) * (size_t)n);
  if (tsk) memcpy(tsk, L.tsk, sizeof(int) * 3 * (size_t)L.count);
  free(L.tsk);
  tree_free(&T);
  free(P);
  return g_status;
}

/* ------------------------------------------------------------------ fixtures
 * The BASELINE.json inputs for bench.py's reference arm, which must not load
 * the product library: the RH4 vorticity (config 1/2/4/5) and the config-3
 * random cap generator, restated here from their definitions in BASELINE.json
 * (the product's host generators, paper_2401_07361_b200/csrc/workloads.cpp,
 * implement the same definitions; tests/test_host.py checks the two agree bit
 * for bit). The mesh itself comes from the reference (ref_make_mesh). */

/* zeta = 2 sin(lat) - 30 sin(lat) cos^4(lat) cos(4 lon); lat = asin(clamp z),
 * lon = atan2(y, x) in [-pi, pi) (unit_to_latlon, geometry.cpp:46-53). */
int orc_rh4_vorticity(const double* xyz, int64_t n, double* zeta) {
  for (int64_t i = 0; i < n; ++i) {
    double z = xyz[3 * i + 2];
    if (z > 1.0) z = 1.0;
    if (z < -1.0) z = -1.0;
    const double lat = asin(z);
    double lon = atan2(xyz[3 * i + 1], xyz[3 * i]);
    if (lon >= M_PI) lon -= 2.0 * M_PI;
    const double st = sin(lat), ct = cos(lat);
    zeta[i] = 2.0 * st - 30.0 * st * ct * ct * ct * ct * cos(4.0 * lon);
  }
  return ORC_OK;
}

/* splitmix64 seeding of xoshiro256** (Vigna / Blackman, public domain);
 * doubles from the top 53 bits. */
typedef struct {
  uint64_t s[4];
} orc_rng;
static uint64_t orc_splitmix(uint64_t* x) {
  uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
static uint64_t orc_rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static uint64_t orc_next(orc_rng* r) {
  uint64_t* s = r->s;
  const uint64_t out = orc_rotl(s[1] * 5, 7) * 9;
  const uint64_t t = s[1] << 17;
  s[2] ^= s[0];
  s[3] ^= s[1];
  s[1] ^= s[2];
  s[0] ^= s[3];
  s[2] ^= t;
  s[3] = orc_rotl(s[3], 45);
  return out;
}
static double orc_u01(orc_rng* r) { return (double)(orc_next(r) >> 11) * 0x1.0p-53; }
static double orc_u01_open(orc_rng* r) { return ((double)(orc_next(r) >> 11) + 0.5) * 0x1.0p-53; }
static double orc_normal(orc_rng* r) { /* Box-Muller, one value per call */
  const double u1 = orc_u01_open(r), u2 = orc_u01(r);
  return sqrt(-2.0 * log(u1)) * cos(2.0 * M_PI * u2);
}

/* half the points: normalised i.i.d. N(0,1)^3; the other half uniform in area
 * on the 10-degree cap about x0 = (lat 40, lon 0): z' ~ U[cos 10, 1], azimuth
 * ~ U[0, 2 pi) in the frame (north, east, x0) at x0 */
static v3 orc_draw(orc_rng* r, int in_cap) {
  if (!in_cap) {
    for (;;) {
      const double x = orc_normal(r), y = orc_normal(r), z = orc_normal(r);
      if (x * x + y * y + z * z > 1e-20) return unitv(x, y, z);
    }
  }
  const double c10 = cos(10.0 * M_PI / 180.0);
  const double zp = c10 + (1.0 - c10) * orc_u01(r);
  const double ph = 2.0 * M_PI * orc_u01(r);
  const double q = 1.0 - zp * zp;
  const double rp = sqrt(q > 0.0 ? q : 0.0);
  const double lat0 = 40.0 * M_PI / 180.0;
  const v3 e3 = latlon_unit(lat0, 0.0);
  const v3 e1 = {-sin(lat0), 0.0, cos(lat0)};
  const v3 e2 = {0.0, 1.0, 0.0};
  const double a = rp * cos(ph), b = rp * sin(ph);
  return unitv(a * e1.x + b * e2.x + zp * e3.x, a * e1.y + b * e2.y + zp * e3.y, a * e1.z + b * e2.z + zp * e3.z);
}

typedef struct {
  int64_t key, idx;
} orc_cell;
static int orc_cell_cmp(const void* a, const void* b) {
  const orc_cell* x = (const orc_cell*)a;
  const orc_cell* y = (const orc_cell*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->idx < y->idx ? -1 : (x->idx > y->idx);
}

/* near-duplicate policy: flag every j with 1 - x_i.x_j <= 1e-12 (reference
 * rounding) against some i < j, found through a uniform grid of 2^-19 cells */
static int64_t orc_near_dups(const v3* p, int64_t n, char* bad) {
  const double h = 1.0 / (1 << 19);
  orc_cell* ks = (orc_cell*)malloc((size_t)n * sizeof(orc_cell));
  if (!ks) return -1;
#define ORC_CELL(v) ((int64_t)floor(((v) + 1.0) / h))
#define ORC_KEY(a, b, c) (((a) << 42) | ((b) << 21) | (c))
  for (int64_t i = 0; i < n; ++i) {
    ks[i].key = ORC_KEY(ORC_CELL(p[i].x), ORC_CELL(p[i].y), ORC_CELL(p[i].z));
    ks[i].idx = i;
  }
  qsort(ks, (size_t)n, sizeof(orc_cell), orc_cell_cmp);
  memset(bad, 0, (size_t)n);
  int64_t nbad = 0;
  for (int64_t i = 0; i < n; ++i) {
    const v3 x = p[i];
    const int64_t cx = ORC_CELL(x.x), cy = ORC_CELL(x.y), cz = ORC_CELL(x.z);
    for (int dx = -1; dx <= 1; ++dx)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dz = -1; dz <= 1; ++dz) {
          const int64_t k = ORC_KEY(cx + dx, cy + dy, cz + dz);
          int64_t lo = 0, hi = n;
          while (lo < hi) {
            const int64_t mid = (lo + hi) / 2;
            if (ks[mid].key < k) lo = mid + 1;
            else hi = mid;
          }
          for (; lo < n && ks[lo].key == k; ++lo) {
            const int64_t j = ks[lo].idx;
            if (j <= i) continue;
            const v3 y = p[j];
            const double den = 1.0 - ((x.x * y.x + x.y * y.y) + x.z * y.z);
            if (den <= 1e-12 && !bad[j]) {
              bad[j] = 1;
              ++nbad;
            }
          }
        }
  }
#undef ORC_CELL
#undef ORC_KEY
  free(ks);
  return nbad;
}

/* BASELINE config 3: xyz (n x 3), zeta = exp(-16 (1 - x.x0)) minus its
 * weighted mean, area = 4 pi / n. */
int orc_make_random_cap(int64_t n, uint64_t seed, double* xyz, double* zeta, double* area) {
  if (n < 2) return ORC_CONFIG;
  orc_rng r;
  for (int k = 0; k < 4; ++k) r.s[k] = orc_splitmix(&seed);
  const int64_t half = n / 2;
  v3* p = (v3*)malloc((size_t)n * sizeof(v3));
  char* bad = (char*)malloc((size_t)n);
  if (!p || !bad) {
    free(p);
    free(bad);
    return ORC_NOMEM;
  }
  for (int64_t i = 0; i < n; ++i) p[i] = orc_draw(&r, i >= half);
  int rc = ORC_OK;
  for (int round = 0; round < 64; ++round) {
    const int64_t nb = orc_near_dups(p, n, bad);
    if (nb < 0) {
      rc = ORC_NOMEM;
      break;
    }
    if (nb == 0) break;
    for (int64_t j = 0; j < n; ++j)
      if (bad[j]) p[j] = orc_draw(&r, j >= half);
    if (round == 63) rc = ORC_GEOMETRY;
  }
  if (rc == ORC_OK) {
    const v3 x0 = latlon_unit(40.0 * M_PI / 180.0, 0.0);
    const double a = 4.0 * M_PI / (double)n;
    double circ = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      xyz[3 * i] = p[i].x;
      xyz[3 * i + 1] = p[i].y;
      xyz[3 * i + 2] = p[i].z;
      zeta[i] = exp(-16.0 * (1.0 - v3dot(p[i], x0)));
      area[i] = a;
      circ += zeta[i] * a;
    }
    const double mean = circ / (4.0 * M_PI);
    for (int64_t i = 0; i < n; ++i) zeta[i] -= mean;
  }
  free(p);
  free(bad);
  return rc;
}
