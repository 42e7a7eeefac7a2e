/*
 * spheresum_b200 — C-ABI of the B200-native spherical barycentric-Lagrange
 * tree code (arXiv 2401.07361). Plain pointers and sizes only; no exceptions
 * and no C++/torch types cross this boundary.
 *
 * Every entry point replaces one reference interface (namespace spheresum,
 * proj/include/spheresum/ in the reference). The mapping is given beside
 * each declaration. The C++ drop-in (see include/spheresum_b200/)
 * and the Python package (paper_2401_07361_b200) sit on top of this header.
 *
 * Layouts: positions are N x 3 fp64 AoS unit vectors (the bytes of
 * std::vector<UnitVector3>, geometry.hpp:50-66), strengths q_j = zeta_j A_j are
 * N fp64, outputs are N x D fp64 AoS (PotentialField<D>, treecode.hpp:32-33):
 * D = 3 for the Biot-Savart velocity, D = 1 for the log-kernel stream function.
 * All particle arrays are in the caller's (original) order.
 *
 * Error convention: every function returns an ssum_status. Non-zero codes
 * mirror the reference's exception taxonomy (errors.hpp:10-33), plus CUDA.
 * The message of the last failure is available from ssum_last_error().
 *
 * Threading: a context is not thread-safe; use one host thread per context.
 * A context owns one device, one CUDA stream and all device buffers, and it
 * holds the persistent face-tree geometry (FaceTree semantics: node geometry
 * survives across calls and only grows, face_tree.cpp:42,73-76).
 */
#ifndef SPHERESUM_B200_H_
#define SPHERESUM_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ssum_ctx ssum_ctx;

typedef enum {
  SSUM_OK = 0,
  SSUM_CONFIG = 1,       /* ConfigError           (treecode.cpp:13-20)            */
  SSUM_GEOMETRY = 2,     /* GeometryError         (face_tree.cpp:85, geometry.cpp) */
  SSUM_SINGULAR = 3,     /* SingularKernelError   (kernels.hpp:19,27-29)          */
  SSUM_CONDITIONING = 4, /* ConditioningError     (sbb.cpp:89-93)                 */
  SSUM_INVALID = 5,      /* std::invalid_argument (sbb.cpp:15,78,145)             */
  SSUM_CUDA = 6,         /* CUDA runtime failure (no reference equivalent)        */
  SSUM_NCCL = 7,         /* reserved for collective failures                      */
  SSUM_NOMEM = 8,        /* device or host allocation failure                     */
  SSUM_INTERNAL = 9
} ssum_status;

typedef enum {
  SSUM_BIOT_SAVART = 0,   /* BiotSavartKernel   (kernels.hpp:52-61), dim 3, prefactor -1/(4 pi) */
  SSUM_LOG_POTENTIAL = 1  /* LogPotentialKernel (kernels.hpp:44-50), dim 1, prefactor 1          */
} ssum_kernel;

/* TraversalConfig (treecode.hpp:13-20) with the same ranges (validate,
 * treecode.cpp:13-20). pc_only = 1 selects the particle-cluster-only traversal
 * (BASELINE config 2; not in the reference): CP -> PP and CC -> PC. */
typedef struct {
  double theta;    /* MAC, in (0, 1]                         */
  int n_threshold; /* bin size above which a node is a cluster */
  int degree;      /* SBB interpolation degree, [1, 20]       */
  int max_depth;   /* deepest tree level, [1, 40]             */
  int pc_only;     /* 0 = full dual traversal, 1 = PC-only    */
} ssum_config;

/* TreecodeStats (treecode.hpp:75-80) plus device-side detail. The three
 * *_seconds fields ACCUMULATE (+=) like the reference's; everything else is
 * overwritten by each call. */
typedef struct {
  double bin_seconds;
  double traversal_seconds;
  double eval_seconds;
  uint64_t interaction_counts[4]; /* indexed PP, PC, CP, CC (InteractionKind)      */
  double h2d_seconds, d2h_seconds;  /* host-pointer entry points only             */
  uint64_t kernel_evals[4];       /* PP pairs (excl. self), PC, CP, CC evaluations */
  int64_t node_count, leaf_count, weight_nodes, fit_nodes;
  int64_t gpu_launches;           /* kernels launched by the last call            */
  double pp_pc_ms, cp_cc_fit_ms, upward_ms, finish_ms; /* device time per pass     */
  uint64_t up_visits, down_visits; /* (particle, weight node) / (particle, fit node) pairs */
  double tiles_ms;                /* CP/CC+fit and PP+PC tiles together (they run
                                     concurrently on two streams: pp_pc_ms and
                                     cp_cc_fit_ms are each kernel's own span)   */
  int64_t mac_host_decisions;     /* node pairs whose MAC quotient fell inside the
                                     guard band around theta and were decided
                                     with the reference's host arithmetic
                                     (context total)          */
} ssum_stats;

/* ---- context ------------------------------------------------------------ */
int ssum_create(int device, ssum_ctx** out);
/* Device buffers come from the device's stream-ordered memory pool; blocks a
 * destroyed context released stay cached there for the next context (a fresh
 * FaceTree then allocates nothing from the driver). ssum_trim_memory returns
 * the cached, unused blocks of `device` to the driver. */
void ssum_destroy(ssum_ctx* ctx);
int ssum_trim_memory(int device);
const char* ssum_last_error(const ssum_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch's current stream); NULL restores the
 * context's own (non-blocking) stream. The legacy default stream has handle 0,
 * which reads as NULL here: pass cudaStreamLegacy ((void*)1) for it, so the
 * library's work stays ordered with work the caller queues there. */
int ssum_set_stream(ssum_ctx* ctx, void* cuda_stream);
/* Drop the persistent tree geometry (a freshly constructed FaceTree,
 * face_tree.cpp:9-16). */
int ssum_tree_reset(ssum_ctx* ctx);

/* ---- summation ---------------------------------------------------------- */
/* treecode_sum<K> (treecode.hpp:93-97, treecode.cpp:266-413): bins into the
 * context's tree, traverses, evaluates. Host pointers; copies are inside. */
int ssum_treecode_sum(ssum_ctx* ctx, int kernel, const ssum_config* cfg, const double* xyz,
                      const double* q, int64_t n, double* out, ssum_stats* stats);
/* Same, with DEVICE pointers (inputs already resident in HBM). Synchronous on
 * return unless stats == NULL and the stream is external (then only stream-ordered). */
int ssum_treecode_sum_device(ssum_ctx* ctx, int kernel, const ssum_config* cfg,
                             const double* d_xyz, const double* d_q, int64_t n, double* d_out,
                             ssum_stats* stats);
/* direct_sum<K> (treecode.hpp:84-86, treecode.cpp:246-264): exact O(N^2). */
int ssum_direct_sum(ssum_ctx* ctx, int kernel, const double* xyz, const double* q, int64_t n,
                    double* out);
int ssum_direct_sum_device(ssum_ctx* ctx, int kernel, const double* d_xyz, const double* d_q,
                           int64_t n, double* d_out);

/* ---- tree and interaction lists (host views, reference numbering) ------- */
/* FaceTree::bin_particles (face_tree.hpp:42, face_tree.cpp:73-88). */
int ssum_bin_particles(ssum_ctx* ctx, const double* xyz, int64_t n, int n_threshold,
                       int max_depth);
/* Node count of the context's tree (FaceTree::node_count, face_tree.hpp:47). */
int ssum_tree_node_count(ssum_ctx* ctx, int* count);
/* Export the binned tree with the reference's node ids. Any pointer may be
 * NULL. tri: 9 doubles per node (v1, v2, v3); center: 3; radius: 1;
 * bin_offsets: node_count + 1; bin_ids: ascending particle ids per node
 * (TreeNode::bin); leaf_of: n (FaceTree::leaf_of_particle). */
int ssum_tree_export(ssum_ctx* ctx, int* level, int* parent, int* child_base, double* tri,
                     double* center, double* radius, int64_t* bin_offsets, int* bin_ids,
                     int* leaf_of);
/* dual_traversal (treecode.hpp:44-45, treecode.cpp:69-77) on the binned tree:
 * (target, source, kind) triples in the reference's emission order and node
 * numbering. Writes min(count, cap) triples; *count receives the total. */
int ssum_dual_traversal(ssum_ctx* ctx, const ssum_config* cfg, int* tsk, int64_t cap,
                        int64_t* count);

/* eval_pp / eval_pc / eval_cp / eval_cc (treecode.hpp:55-73,
 * treecode.cpp:170-244): ADDS the raw kernel sums (no prefactor) of one
 * interaction (target, source: reference node ids of the tree as last binned
 * from these positions; kind: 0 PP, 1 PC, 2 CP, 3 CC) into field (host,
 * N x D, caller's order). Proxy weights and fits are computed for this
 * interaction alone, as the reference's per-interaction entry points do. */
int ssum_eval_interaction(ssum_ctx* ctx, int kernel, const ssum_config* cfg, const double* xyz,
                          const double* q, int64_t n, int target, int source, int kind,
                          double* field);

/* compute_proxy_weights (treecode.hpp:47-51, treecode.cpp:79-91): the raw
 * proxy weights w_k = sum_{j in bin(source_node)} B_k(beta(x_j)) q_j of one
 * node (reference id) of the tree as last binned from these positions;
 * w: (degree+1)(degree+2)/2 doubles, in SBBBasis index order. */
int ssum_compute_proxy_weights(ssum_ctx* ctx, int degree, const double* xyz, const double* q, int64_t n,
                               int source_node, double* w);
/* Reciprocal condition number carried by the context's last SSUM_CONDITIONING
 * failure (ConditioningError::rcond, errors.hpp:22-27). */
double ssum_last_rcond(const ssum_ctx* ctx);

/* ---- SBB interpolation (sbb.hpp; host) ------------------------------------ */
/* lattice_fit(degree) (sbb.hpp:74-78, sbb.cpp:124-138): V^-1 of the lattice
 * Vandermonde V[m][k] = B_k(b_m) (row-major P x P, may be NULL) and its
 * reciprocal condition number (exact 1-norm). Returns SSUM_CONDITIONING when
 * rcond <= 1e-12 (sbb.cpp:89-93), SSUM_INVALID for a degree outside [1, 20]. */
int ssum_lattice_fit(int degree, double* vinv, double* rcond);
/* proxy_points(t, degree).points (sbb.hpp:48, sbb.cpp:46-66): tri = v1, v2,
 * v3 (9 doubles); pts receives P x 3 doubles in SBBBasis index order, with the
 * reference's rounding (the tree code's device proxies are bit-identical). */
int ssum_proxy_points(const double* tri, int degree, double* pts);

/* ---- multi-GPU target partition (no reference equivalent) */
/* Subsequent treecode evaluations compute only part `part` of `nparts`
 * cost-balanced contiguous ranges of target leaves (tree order) and write only
 * those rows of the output; the tree build and upward pass are replicated.
 * The union over parts is bitwise the nparts = 1 result. */
int ssum_set_partition(ssum_ctx* ctx, int part, int nparts);
/* Tree-position range [begin, end) of the last evaluation's part. */
int ssum_partition_range(ssum_ctx* ctx, int64_t* begin, int64_t* end);
/* Copy the last binning's permutation (tree position -> caller's particle
 * index, N ints) into dst, a device pointer if on_device != 0. */
int ssum_tree_perm(ssum_ctx* ctx, int* dst, int on_device);
/* Every part's tree-position range in the last evaluation: nparts + 1
 * positions (part r = [cuts[r], cuts[r+1])). The ranks bin identically, so
 * every rank gets the same table without communicating. */
int ssum_partition_cuts(ssum_ctx* ctx, int64_t* cuts);
/* Sharded binning walk (multi-GPU): walks particles [i0, i1) of the caller's
 * order (device xyz, all n rows) through the context's existing tree and
 * returns device pointers to its per-particle leaf keys (uint64, n rows) and
 * leaves (int32, n rows), each with room for `slots` >= n rows. The caller
 * fills the other ranks' rows (one all-gather of equal slots per array); the
 * next binning of these n particles (e.g. ssum_treecode_sum_device) then
 * skips its walk and is bitwise the unsharded binning. *walked = 0 when the
 * tree cannot be walked yet (first call on a tree): nothing to exchange, the
 * next binning builds the tree itself. */
int ssum_bin_walk_shard(ssum_ctx* ctx, const double* d_xyz, int64_t n, int64_t i0, int64_t i1, int64_t slots,
                        void** keys, void** leaf_of, int* walked);
/* Device-pointer evaluations write this part's rows in tree order (position
 * p0 + r to row r, rows past p1 - p0 untouched) instead of the caller's order
 * over all N rows: the rows one all-gather exchanges (tree_order = 1). */
int ssum_set_output_order(ssum_ctx* ctx, int tree_order);

/* ---- Lagrangian RK4 (absent from the reference code) ---- */
/* In place on host arrays: xyz (N x 3), zeta (N); area (N) fixed. Each stage
 * evaluates u with treecode_sum<BiotSavartKernel> (direct_sum if direct != 0)
 * on the context's (reused) tree, dzeta/dt = -2 omega u_z, stage and final
 * positions renormalised. Device-resident between stages. */
int ssum_rk4(ssum_ctx* ctx, const ssum_config* cfg, double* xyz, double* zeta,
             const double* area, int64_t n, double dt, int steps, double omega, int direct,
             ssum_stats* stats);
/* The pieces of one ssum_rk4 step on device arrays, for drivers that
 * evaluate the stage velocities themselves (multi-GPU: partitioned
 * evaluation, then one all-gather of the rows per stage). Same kernels as
 * ssum_rk4, so such a driver reproduces it bit for bit. Per step:
 *   for stage in 0..3: stage_begin (xs, q from x0, z0, area and the previous
 *   stage's k, kz) -> evaluate u at (xs, q) -> stage_end (k, kz, acc, accz);
 *   then step_end (x0, z0 advanced, renormalised). */
int ssum_rk4_stage_begin(ssum_ctx* ctx, int stage, double dt, int64_t n, const double* d_x0,
                         const double* d_z0, const double* d_area, const double* d_k,
                         const double* d_kz, double* d_xs, double* d_q);
int ssum_rk4_stage_end(ssum_ctx* ctx, int stage, double omega, int64_t n, const double* d_u,
                       double* d_k, double* d_kz, double* d_acc, double* d_accz);
int ssum_rk4_step_end(ssum_ctx* ctx, double dt, int64_t n, double* d_x0, double* d_z0,
                      const double* d_acc, const double* d_accz);
/* stage_end on the all-gathered rows of a partitioned evaluation (SURVEY.md
 * §8(e)/(f) rank 2): d_rows holds nparts slots of `width` rows x 3, slot r =
 * part r's rows in tree order (ssum_set_output_order(ctx, 1)), exactly what one
 * ncclAllGather of equal slots leaves on every rank; the stage kernel reads
 * them through the binning's permutation. Bitwise ssum_rk4_stage_end on the
 * assembled field. */
int ssum_rk4_stage_end_rows(ssum_ctx* ctx, int stage, double omega, int64_t n, const double* d_rows,
                            int64_t width, double* d_k, double* d_kz, double* d_acc, double* d_accz);
/* ssum_rk4_stage_end_rows of `stage` fused with ssum_rk4_stage_begin of
 * stage + 1 (none after stage 3): per particle, its row gathered through the
 * inverse permutation, the accumulators advanced and the next stage's
 * positions / strengths formed; d_k / d_kz (both or neither) receive k and
 * kz when given. Bitwise the two calls. */
int ssum_rk4_stage_advance_rows(ssum_ctx* ctx, int stage, double dt, double omega, int64_t n, const double* d_rows,
                                int64_t width, const double* d_x0, const double* d_z0, const double* d_area,
                                double* d_k, double* d_kz, double* d_acc, double* d_accz, double* d_xs,
                                double* d_q);

/* ---- measurement --------------------------------------------------------- */
/* FP64 roofline denominator: DFMA-chain throughput of this device in TFLOP/s
 * (best of `reps` launches). MEASURED_PEAKS.json has no fp64 entry. */
int ssum_fp64_peak(ssum_ctx* ctx, int reps, double* tflops);
/* Accuracy probe of the log the tree code's far pairs use (log kernel,
 * kernels.cuh log_tab): out[i] = log(x[i]) for x[i] in [2^-20, 4]. Host arrays. */
int ssum_probe_log_far(ssum_ctx* ctx, const double* x, int64_t n, double* out);

/* ---- fixtures (BASELINE.json configs; host-side generators) -------------- */
/* make_icosa_mesh(level).vertices() / node_patch_areas() (icosa_mesh.cpp:37-133). */
int64_t ssum_mesh_vertex_count(int level);
int ssum_make_icosa_mesh(int level, double* xyz, double* area);
/* BASELINE Rossby-Haurwitz R=4 vorticity (omega = K = 1):
 * zeta = 2 sin(lat) - 30 sin(lat) cos^4(lat) cos(4 lon). */
int ssum_rh4_vorticity(const double* xyz, int64_t n, double* zeta);
/* BASELINE config 3: seeded points (half uniform, half in a 10 deg cap at lat
 * 40, lon 0), Gaussian vortex minus its weighted mean, A = 4 pi / N. The
 * near-duplicate policy resamples any point whose 1 - x.y <= 1e-12 against an
 * earlier point. */
int ssum_make_random_cap(int64_t n, uint64_t seed, double* xyz, double* zeta, double* area);

#ifdef __cplusplus
}
#endif

#endif /* SPHERESUM_B200_H_ */
