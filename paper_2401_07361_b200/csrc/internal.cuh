// Internal declarations shared by the .cu translation units of
// libspheresum_b200.so: the context, device buffers, error plumbing, and the
// pass entry points (tree build, traversal, evaluation).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/spheresum_b200.h"
#include "geom.cuh"

namespace ssum {

// Internal failure carrying an ssum_status; converted to a return code at the
// C-ABI boundary (capi.cu). Never crosses extern "C".
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define SSUM_CUDA_CHECK(x)                                                                 \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      throw ::ssum::Error(SSUM_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_) +     \
                                         " (" __FILE__ ":" + std::to_string(__LINE__) + ")"); \
  } while (0)

#define SSUM_LAUNCH_CHECK() SSUM_CUDA_CHECK(cudaGetLastError())

// Device-side bounds checks of the index arithmetic (the checked build,
// `make -C paper_2401_07361_b200/csrc checked`, compiles with
// -DSSUM_DEVICE_CHECKS): a violated check prints its site and traps, so the
// test run fails at the first bad access. compute-sanitizer is not available
// on the GPU pool; this is the stand-in (tests run against the checked
// library with SSUM_LIBRARY=.../lib/checked/libspheresum_b200.so).
#ifdef SSUM_DEVICE_CHECKS
#define SSUM_DCHECK(cond)                                                                      \
  do {                                                                                         \
    if (!(cond)) {                                                                             \
      printf("SSUM_DCHECK failed %s:%d (block %d thread %d): %s\n", __FILE__, __LINE__,       \
             int(blockIdx.x), int(threadIdx.x), #cond);                                        \
      __trap();                                                                                \
    }                                                                                          \
  } while (0)
#else
#define SSUM_DCHECK(cond) \
  do {                    \
  } while (0)
#endif

constexpr int kMaxDegree = 20;  // kMaxSbbDegree (sbb.hpp:12)
constexpr int kWarp = 32;
constexpr double kSingularTol = 1e-14;  // kernels.hpp:13
constexpr double kPi = 3.141592653589793;

// Device error flags (bitmask in ctx.d_flags[0]).
// kFlagListsRedo: the subtree list builder (sublists.cu) ran out of room or
// met undecided MAC pairs; the evaluation is redone on the global path.
enum : int { kFlagGeometry = 1, kFlagSingular = 2, kFlagListsRedo = 8 };

// Stream the device allocations of the current C-ABI call are ordered on
// (the context's stream, set by the entry point): DBuf memory comes from the
// device's stream-ordered pool (cudaMallocAsync / cudaFreeAsync), so growing
// a buffer neither synchronises the device nor returns memory to the driver
// between calls, and a fresh context reuses what earlier ones released.
// Code that fills a buffer on another stream passes that stream explicitly.
cudaStream_t& dbuf_stream();

// Growable device array. Contents are NOT preserved on growth unless keep.
template <class T>
struct DBuf {
  T* p = nullptr;
  size_t cap = 0;
  DBuf() = default;
  DBuf(const DBuf&) = delete;  // owns device memory: freed once, by the owner
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), cap(o.cap) { o.p = nullptr, o.cap = 0; }
  DBuf& operator=(DBuf&& o) noexcept {
    if (this != &o) {
      release();
      p = o.p, cap = o.cap;
      o.p = nullptr, o.cap = 0;
    }
    return *this;
  }
  ~DBuf() { release(); }
  void ensure(size_t n, bool keep = false, cudaStream_t s = nullptr) {
    if (n <= cap) return;
    if (!s) s = dbuf_stream();
    size_t nc = cap ? cap : 1024;
    while (nc < n) nc *= 2;
    T* q = nullptr;
    SSUM_CUDA_CHECK(cudaMallocAsync(reinterpret_cast<void**>(&q), nc * sizeof(T), s));
    if (keep && p && cap) SSUM_CUDA_CHECK(cudaMemcpyAsync(q, p, cap * sizeof(T), cudaMemcpyDeviceToDevice, s));
    if (p) SSUM_CUDA_CHECK(cudaFreeAsync(p, s));  // after every earlier use on s (callers join other streams first)
    p = q;
    cap = nc;
  }
  void release() {
    if (p) cudaFreeAsync(p, dbuf_stream());
    p = nullptr;
    cap = 0;
  }
};

// Persistent node geometry (FaceTree::nodes_, face_tree.hpp:55). Index =
// device node id (breadth-first allocation); the reference's depth-first ids
// are reconstructed on export (tree_export in capi.cu).
struct NodeTable {
  int count = 0;            // nodes allocated
  DBuf<double> tri;         // 9 per node: v1, v2, v3
  DBuf<double> center;      // 3: circumcenter
  DBuf<double> radius;      // 1
  DBuf<double> cramer;      // 12: bc = v2 x v3 (3), det (1), n2 = v3 x v1, n3 = v1 x v2 (6), spare (2)
  DBuf<int> level, parent, child_base, created_call;
  // depth-first path key: root face << 58 | child index q << (58 - 2 level)
  // per step; key order = depth-first order (levels <= kKeyMaxLevel)
  DBuf<unsigned long long> key;
  int max_level = 0;        // deepest level allocated so far
};
constexpr int kKeyRootShift = 58;
constexpr int kKeyMaxLevel = 29;

// Host snapshot of the node structure (ids, levels, links, creating call)
// plus the last binning's counts/offsets. Downloaded on demand (exports,
// partitioning); the binning itself runs on the device.
struct HostTree {
  bool valid = false;
  std::vector<int> level, parent, child_base, created_call;
  std::vector<int> cnt, off;
};

// Per-call binned tree (bins as contiguous ranges of the tree-order permutation).
struct Binned {
  int64_t n = 0;
  int n_leaves = 0;
  DBuf<int> cnt;            // particles per node
  DBuf<int> off;            // first tree position of the node's bin
  DBuf<unsigned char> act;  // per candidate node: 0 leaf, 1 descend
  DBuf<unsigned char> is_leaf;  // node is a non-empty leaf of this call
  DBuf<int> cur;            // per particle: current node during the descent
  DBuf<int> leaf_of;        // per particle (original order)
  DBuf<int> perm;           // tree position -> original particle id
  int64_t perm_n = -1;      // particle count perm is complete for (-1: none)
  bool input_coherent = true;  // last reuse binning: most consecutive inputs in one leaf
  int64_t walked_n = -1;    // wkey / leaf_of of all walked_n particles filled by sharded walks
                            // (ssum_bin_walk_shard + the caller's all-gather): the next binning
                            // of walked_n particles skips its own walk
  DBuf<int> pos_leaf;       // tree position -> leaf node
  DBuf<int> sort_keys, sort_keys2, sort_vals;
  // level-synchronous descent: candidates of the current level, their split
  // flags / child counts and prefix sums, all candidates of all levels
  DBuf<int> cand, cand_next, split, split_pos, nextc, next_pos, levels;
  std::vector<std::pair<int, int>> level_span;  // (offset in levels, count) per level
  DBuf<unsigned long long> wkey, wkey2;  // reuse path: per-particle path keys, sorted
  DBuf<unsigned char> leaf_flag;
  DBuf<int> leaf_pos;       // reuse path: first tree position of each leaf
  DBuf<int> d_leaves;       // non-empty leaves in depth-first order
  DBuf<int> leaf_keys;
  int* h_small = nullptr;   // pinned host scratch
};

struct Ctx;

// One tile = up to kTileTargets targets against a list of source ranges. The
// list starts with the ranges that may hold near pairs (1 - x.y < 2^-20, or
// self pairs); near_total counts their sources. Beyond it every pair is
// well separated and the kernel runs its branch-free fast loop.
constexpr int kTileTargets = 256;
struct Tile {
  int tgt_begin;  // index into the unified point array
  int tgt_count;  // 1 .. kTileTargets
  int list_begin, list_end;  // into the range list
  int near_total;            // sources in the leading near-possible ranges
  int self_shift;  // self source of target i at flattened list position i + self_shift
  int has_self;    // bit 0: a range holds the targets themselves; bit 1 (kTileDense):
                   // dense leaf — near-possible ranges evaluated with reference rounding
  int total;       // sources in the flattened list (sum of the ranges' counts)
};
// Arc-length margin below which a (target leaf, source node) pair may hold a
// near pair: den = 2 sin^2(arc/2) < 2^-20 <=> arc < 2 asin(2^-10.5) =
// 1.38107e-3 rad. A binned point lies in its node's circumcircle up to the
// 1e-10 containment tolerance, so arc(x, y) >= arc(c_t, c_s) - r_t - r_s -
// 2e-10 >= chord(c_t, c_s) - r_t - r_s - 2e-10: a pair tested at or beyond
// 1.39e-3 (margin 9e-6 over every rounding involved) holds no near pair.
// (Round 1 used 2e-3; the tighter margin takes 7% of C3's leaf-tile time.)
#ifndef SSUM_NEAR_ARC
#define SSUM_NEAR_ARC 1.39e-3
#endif
constexpr double kNearArc = SSUM_NEAR_ARC;
// Leaf point spacing below which near pairs (den < 2^-20, arc < 1.38e-3)
// are common enough that masking and repairing them costs more than
// evaluating the near-possible ranges with reference rounding outright.
constexpr int kTileDense = 2;
#ifndef SSUM_DENSE_SPACING
#define SSUM_DENSE_SPACING 1.5e-3
#endif
constexpr double kDenseSpacing = SSUM_DENSE_SPACING;
// Source range in the unified point array. near != 0 marks a particle (PP)
// range, which may hold near-singular or self pairs; pad is the number of
// sources in the tile's list before this range (the flattened-list prefix).
struct SrcRange {
  int begin;
  int count;
  int near;
  int pad;
};

struct Lists {
  int64_t n_inter = 0;
  uint64_t counts[4] = {0, 0, 0, 0};
  DBuf<int4> inter;          // emissions: (t, s, kind, 0)
  DBuf<unsigned long long> key;  // depth-first order key of each emission
  int n_proxy = 0;           // nodes carrying proxy points (weight or fit nodes)
  int n_weight = 0, n_fit = 0;
  DBuf<int> pslot;           // node -> proxy slot or -1
  DBuf<unsigned char> is_weight, is_fit;
  DBuf<int> weight_nodes, fit_nodes;  // slot-ordered node lists
  int n_leaf_tiles = 0, n_fit_tiles = 0;
  DBuf<Tile> leaf_tiles, fit_tiles;
  int64_t n_leaf_ranges = 0, n_fit_ranges = 0;
  DBuf<SrcRange> leaf_ranges, fit_ranges;
  uint64_t evals[4] = {0, 0, 0, 0};
  uint64_t visits[2] = {0, 0};   // upward (particle, weight node), downward (particle, fit node)
  // per-tile work (PP, PC) / (CP, CC) pair counts and this part's share
  DBuf<ulonglong2> leaf_cost, fit_cost;
  int leaf_t0 = 0, leaf_t1 = 0;  // leaf tile range of this part
  int64_t p0 = 0, p1 = 0;        // tree-position range of this part
  DBuf<int> fit_sel;             // selected fit tiles (when !fit_sel_all)
  int n_fit_sel = 0;
  bool fit_sel_all = true;
  uint64_t local_evals[4] = {0, 0, 0, 0};
  bool counts_pending = false;   // counts/evals still in flight (finalize_counts)
  bool local_is_all = true;      // this part's work = all listed work (one part, or restricted lists)
};

// Breadth-first traversal frontier entry: node pair plus depth-first order key.
struct PairEntry {
  int t, s;
  unsigned long long key;
  int step, pad;
};

// Everything a pair decision reads about one node, packed per call (bin
// counts change, and sh / ch depend on theta): circumcentre, radius,
// sin / cos of radius / (2 theta) (the MAC screen, travdev.cuh), bin, level,
// first child. 64 bytes: one node is two aligned 32-byte sectors.
struct __align__(16) NodeRec {
  double cx, cy, cz, r, sh, ch;
  int cnt, off, level, child_base;
};
static_assert(sizeof(NodeRec) == 64, "NodeRec layout");

struct TravScratch {
  DBuf<NodeRec> rec;         // per call (build_node_records)
  double rec_theta = -1.0;
  DBuf<PairEntry> F0, F1;
  DBuf<int> action;
  DBuf<unsigned long long> packed, scan;
  DBuf<int> gkey, gkey2, gval, sorted_e;
  DBuf<int2> seg;
  DBuf<int> flag, flag_scan, slot_node;
  DBuf<int> nr, nt, nr_off, nt_off, fnr, fnr_off;
  DBuf<unsigned long long> counters;  // [0..3] kinds, [4..7] kernel evals
  unsigned long long* h_small = nullptr;  // pinned: [0..7] scratch, [8..15] counters read-back
  int bfs_namb = -1;  // k_bfs's read-back of the MAC guard band's undecided-pair count (-1: not read)
  // single-launch traversal (traversal.cu bfs_persistent): the last call's
  // frontier sizes and emission count size the next call's buffers
  std::vector<int> plan_m;
  long long plan_ne = 0;
  bool plan_valid = false;
  int bfs_blocks = 0;        // cooperative grid size (0: not queried, -1: unavailable)
  DBuf<int> dm;              // k_bfs results: steps, overflow, largest frontier
  DBuf<long long> debase;    // k_bfs result: emission count
  long long* h_plan = nullptr;  // pinned read-back
};

// Host-made MAC decisions for node pairs inside the guard band around theta
// (traversal.cu MacCtl / resolve_mac). Keys: t << 33 | s << 1 | well, sorted.
// Valid for one theta; node ids persist with the geometry (reset: cleared).
struct MacGuard {
  static constexpr int kAmbCap = 4096;
  double band = 1e-12;  // relative half-width (SSUM_MAC_BAND overrides, tests)
  double theta = -1.0;
  std::vector<unsigned long long> keys;
  DBuf<unsigned long long> d_keys;
  DBuf<int2> amb;
  DBuf<int> amb_n;
  DBuf<unsigned char> ctl;  // device copy of this traversal's MacCtl
  int64_t resolved = 0;  // pairs decided on the host so far
};

// Subtree list plan (sublists.cu): made by each reuse binning (tree.cu),
// consumed by build_lists_subtree.
struct SubPlan {
  bool valid = false;   // the last binning made the plan
  bool used = false;    // this call's lists came from the subtree builder
  int disabled = 0;     // SSUM_SUB_LISTS=0: global path only
  int forced = 0;       // SSUM_SUB_LISTS=1: whenever the plan applies (else by size / restriction)
  int thr = -1;         // N_T the big nodes were flagged with
  int cmax = 0;         // largest cut-node bin (0: not set yet)
  int n_big = 0, n_cut = 0, n_leaf_tiles = 0;
  int smem = 0;
  DBuf<unsigned char> big_flag, cut_flag;
  DBuf<int> cut, tpl, tile_off;
  DBuf<int> wsel;  // [0] count, [1..] marked weight nodes (restricted calls)
  DBuf<unsigned long long> up_visits, cursor;
  int64_t leaf_cap = 0, fit_cap = 0;  // range buffer sizes
  int64_t max_emit = 0, max_front = 0;  // last call's largest block emission count / frontier
  int64_t redos = 0;
  // measured choice between the two list builders (sub_lists_choice)
  int64_t bad_n = -1;  // particle count whose subtree blocks overflowed
  int64_t trial_n = -1;
  double trial_theta = -1.0;
  int trial_calls = 0;
  int trial_cnt[2] = {0, 0};      // [0] global, [1] subtree
  double trial_ms[2] = {0.0, 0.0};
};

struct Ctx {
  int device = 0;
  SubPlan sub;
  int last_flags = 0;  // device error flags read by the last check_flags
  int rt0 = 0, rt1 = 0;  // restricted call: this part's leaf tile range (subtree plan)
  TravScratch trav;
  MacGuard mac;
  cudaStream_t own_stream = nullptr;
  cudaStream_t stream = nullptr;
  std::string last_error;
  int call_index = 0;
  int part = 0, nparts = 1;  // target partition (multi-GPU)
  // Restricted multi-part evaluation (traversal.cu plan_restriction): the
  // cost-balanced cut positions of the last full multi-part call, and — once
  // they exist — this call's tree-position range and leaf-index range; the
  // traversal then only follows pairs whose target bin meets the range.
  struct Cuts {
    int64_t n = -1;
    int nparts = 0;
    std::vector<int64_t> pos;  // nparts + 1 tree positions
  } cuts;
  // every part's tree-position range in the last evaluation (nparts + 1
  // positions; {0, N} unpartitioned) — identical on every rank, so each rank
  // can place every other rank's rows without communication
  std::vector<int64_t> part_pos;
  DBuf<long long> snap;      // k_snap_cuts output
  DBuf<long long> cut_dev;   // part_pos on the device (ssum_rk4_stage_end_rows)
  bool out_tree_order = false;  // device results: this part's rows in tree order (ssum_set_output_order)
  bool restrict_on = false;
  int64_t rp0 = 0, rp1 = 0;
  int rl0 = 0, rl1 = 0;
  HostTree host;
  NodeTable nodes;
  Binned bins;
  Lists lists;
  int64_t launches = 0;

  // scratch
  DBuf<int> d_flags;                 // [0] error bits
  int* h_pinned = nullptr;           // small pinned host scratch (64 ints)
  DBuf<unsigned char> cub_tmp;
  DBuf<double4> pts;                 // unified points: N particles (tree order) + proxies
  int64_t npts = 0;                  // valid entries of pts (bounds checks)
  DBuf<double> S;                    // per tree position accumulated kernel sums (D doubles)
  DBuf<double> coeff;                // per proxy slot: D x P fit coefficients
  DBuf<double> wpart;                // upward partial sums
  DBuf<int4> wchunks;                // upward chunks (node, begin, count, 0) + per-node chunk ranges
  DBuf<int> wcount, wcount_off;      // chunks per weight node, and their prefix
  DBuf<double> vinv;                 // P x P inverse Vandermonde (row-major), per degree
  DBuf<double2> logtab;              // far-pair log table (kernels.cuh log_tab)
  int vinv_degree = -1;
  DBuf<double> in_xyz, in_q, out_buf;  // staging for host-pointer entry points
  DBuf<Tile> direct_tiles;
  DBuf<SrcRange> direct_range;
  DBuf<double> rk_state;             // RK4 scratch
  double last_rcond = 0.0;           // reciprocal condition of the last ConditioningError
  // per-interaction scratch (eval_interaction / proxy_weights)
  DBuf<Tile> ix_tiles;
  DBuf<SrcRange> ix_range;
  DBuf<int> ix_ints;
  DBuf<double> ix_out;
  cudaEvent_t ev[8];
  // The fit tiles (CP/CC+fit) run on side_stream (highest priority)
  // concurrently with the leaf tiles (PP+PC): both only read pts and write
  // disjoint buffers, and the leaf blocks fill the SMs the fit kernel's
  // tail leaves idle (eval.cu).
  cudaStream_t side_stream = nullptr;
  cudaStream_t prep_stream = nullptr;  // gather + proxies + upward pass (start_prep)
  cudaEvent_t fork_ev = nullptr, join_ev = nullptr, side_ev[2] = {}, leaf_ev[2] = {};
  bool overlap_tiles = true;
  // The gather + proxy points + upward pass start on side_stream from
  // build_lists (start_prep) when the treecode entry set `early` (the inputs
  // of the evaluation that follows); evaluate() waits on prep_ev.
  struct Early {
    const double* xyz = nullptr;
    const double* q = nullptr;
    int degree = 0, dim = 0;
  } early;
  bool prep_started = false;
  // global-path lists on the binning's plan (traversal.cu): proxy slots for
  // every big node, upward pass started before the traversal
  bool plan_lists = false;
  // upward pass on a subset of the weight nodes (subtree builder, restricted
  // call: only the sources this part's lists use): list + device count
  const int* up_list = nullptr;
  const int* up_count = nullptr;
  bool plan_lists_ok = true;  // SSUM_PLAN_LISTS=0: slots from the traversal's marks
  bool early_prep = true;
  cudaEvent_t prep_ev = nullptr;
  DBuf<unsigned char> cub_tmp_side;
  // Host-pointer entry (ssum_treecode_sum): the inputs travel on copy_stream
  // in kIoChunks pieces (the tree walk starts on each piece as it lands, q is
  // waited for only at the gather) and the result leaves in pieces as the
  // downward pass finishes them (eval.cu).
  static constexpr int kIoChunks = 4;
  cudaStream_t copy_stream = nullptr;
  struct HostIo {
    bool active = false;
    int64_t bounds[kIoChunks + 1] = {};  // particle ranges of the pieces
    cudaEvent_t xyz[kIoChunks] = {}, q = nullptr, out[kIoChunks] = {}, t0 = nullptr, t1 = nullptr;
    double* h_out = nullptr;           // result destination (original order), nullptr: none
    int dim = 0;
  } io;
  DBuf<int> inv_perm;                // original particle id -> tree position
};

// Host-side phase trace (SSUM_TRACE=1): wall time between marks, printed by
// the caller. Costs nothing when disabled.
struct Trace {
  bool on = false;
  std::vector<std::pair<const char*, double>> marks;
  double t0 = 0.0;
  static double now();
  void start() {
    marks.clear();
    t0 = now();
  }
  void mark(const char* what) {
    if (on) marks.emplace_back(what, now());
  }
};
Trace& trace();

// ---- passes (tree.cu / traversal.cu / eval.cu) ------------------------------
void tree_init_roots(Ctx& c);
void tree_bin(Ctx& c, const double* d_xyz, int64_t n, int nt, int max_depth);
// One rank's share [i0, i1) of the binning walk (multi-GPU); false when the
// tree cannot be walked yet (the next binning then builds it, replicated).
bool tree_walk_shard(Ctx& c, const double* d_xyz, int64_t n, int64_t i0, int64_t i1, int64_t slots);
void traverse_and_build_lists(Ctx& c, const ssum_config& cfg, bool keep_order_keys);
void partition_targets(Ctx& c);
bool plan_restriction(Ctx& c);  // multi-part: restrict this call's lists to the part's targets
void build_lists(Ctx& c, const ssum_config& cfg);
void finalize_counts(Ctx& c);
// subtree list builder (sublists.cu)
void plan_subtrees(Ctx& c, int thr, const int* d_nl, int* d_out);
void plan_subtrees_done(Ctx& c, const int* h);
int sub_lists_choice(Ctx& c, const ssum_config& cfg);  // 0 global, 1 subtree; +2: timed trial
void sub_lists_timed(Ctx& c, int used_sub, double ms);
void build_lists_subtree(Ctx& c, const ssum_config& cfg);
bool sub_lists_redo(Ctx& c, int flags);
// MAC guard band (traversal.cu): the device control block for a traversal
// (resets the undecided-pair count), and the host decision of undecided pairs
const void* mac_ctl_device(Ctx& c);
// NodeRec of every node for this call's bins and theta (c.trav.rec)
void build_node_records(Ctx& c, double theta);
bool resolve_mac_host(Ctx& c);
std::vector<int> reference_ids(const HostTree& h);
const HostTree& host_tree(Ctx& c);  // downloads the node structure when stale
void evaluate(Ctx& c, int kernel, const ssum_config& cfg, const double* d_xyz, const double* d_q,
              int64_t n, double* d_out, ssum_stats* st);
void direct_sum_device(Ctx& c, int kernel, const double* d_xyz, const double* d_q, int64_t n,
                       double* d_out);
void ensure_vinv(Ctx& c, int degree);
void ensure_log_table(Ctx& c);
void launch_fit_tiles(Ctx& c, cudaStream_t stream, int kernel, int P, int nfit, const int* sel);
// k_tiles<fit> over explicit tiles / ranges (fit node k -> coeff slot pslot[fit_nodes[k]])
void launch_fit_tiles_on(Ctx& c, cudaStream_t stream, int kernel, int P, const Tile* tiles, int nfit, const int* sel,
                        const SrcRange* ranges, const int* fit_nodes, const int* pslot, double* coeff);
// Per-interaction entry points (eval.cu): eval_pp/pc/cp/cc and
// compute_proxy_weights on the bins of the last binning, O(|t| |s|).
void eval_interaction(Ctx& c, int kernel, int degree, const double* xyz, const double* q, int target, int source,
                      int kind, double* field);
void proxy_weights(Ctx& c, int degree, const double* xyz, const double* q, int node, double* w);
// V^-1 of the degree-d lattice Vandermonde (row-major, P x P) and its exact
// 1-norm reciprocal condition number (no throw; eval.cu)
void lattice_inverse(int degree, std::vector<double>& inv, double& rcond);
// stages: bit 0 gather + proxy points, bit 1 upward pass
void start_prep(Ctx& c, bool forked = false, int stages = 3);
void size_eval_buffers(Ctx& c, int degree, int D, int64_t n);
void launch_leaf_tiles(Ctx& c, cudaStream_t stream, int kernel, const Tile* tiles, int ntl, const SrcRange* ranges, double* S,
                       bool direct = false);
void launch_direct(Ctx& c, int kernel, int64_t n, double* d_out);
void rk4_combine(Ctx& c, int stage, int64_t n, double dt, double omega, double* d_x0, double* d_z0,
                 const double* d_area, double* d_xs, double* d_q, const double* d_u, double* d_kacc,
                 double* d_kzacc);

// sync + read the device error flags; throws the mapped Error
void check_flags(Ctx& c, const char* where);

inline unsigned grid_for(int64_t n, int block) { return static_cast<unsigned>((n + block - 1) / block); }

}  // namespace ssum
