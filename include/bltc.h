/*
 * bltc.h -- C ABI of libbltc, the B200-native (sm_100a) BLTC evaluation path.
 *
 * Drop-in boundary: the reference exposes the path as Python functions
 *   bltc.engine.treecode_potentials(system, config, threads)   engine.py:350-372
 *   bltc.decomp.run_distributed(system, config, ranks, threads) decomp.py:483-593
 * plus the stage functions its tests call directly
 *   build_source_tree / build_target_batches                    tree.py:191-253
 *   build_interaction_lists / lists_against_root / count_pairs   engine.py:110-143
 *   compute_all_moments                                          moments.py:147-150
 *   compute_potentials                                           engine.py:315-335
 * The Python shim (paper_2003_01836_b200/engine.py, decomp.py) keeps those
 * signatures and binds the entry points below through ctypes; see
 * INTEGRATION.md for the binding a reference maintainer would add.
 *
 * Conventions: plain pointers and sizes, no torch types.  Every function
 * returns BLTC_OK (0) or a negative status; bltc_last_error() gives a
 * thread-local message.  Host-pointer arguments are borrowed for the call;
 * device-pointer arguments must live on the context's device.  A context
 * owns its device buffers and one CUDA stream; it is not thread-safe (one
 * context per host thread and device).  No C++ exception crosses this ABI.
 */
#ifndef BLTC_H
#define BLTC_H

#include <stdint.h>

#if defined(__GNUC__)
#define BLTC_API __attribute__((visibility("default")))
#else
#define BLTC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define BLTC_OK 0
#define BLTC_ERR_VALUE -1      /* maps to ValueError (engine.py:56-62, kernels.py:49-51, tree.py:182) */
#define BLTC_ERR_CUDA -2       /* CUDA runtime / launch failure */
#define BLTC_ERR_STATE -3      /* stage export without a preceding run */
#define BLTC_ERR_UNSUPPORTED -4

/* Evaluation modes.
 * PARITY: bit-faithful to the reference (IEEE sqrt/div, no FMA, the
 *         reference's per-target accumulation order incl. Neumaier).
 * FAST:   rsqrt + FMA, register-blocked tiles, load-balanced work items;
 *         validated against PARITY / the oracle within tolerances.
 * STRICT: the default of the Python shim.  Bitwise moments, the FAST
 *         interaction kernels, and a per-target certificate: every target
 *         whose FAST value cannot be shown to lie within 0.5e-10 (relative)
 *         of the reference's is recomputed in the reference's arithmetic
 *         and order (bitwise).  Result: every target within the north-star
 *         1e-10 of the reference at FAST speed. */
#define BLTC_MODE_PARITY 0
#define BLTC_MODE_FAST 1
#define BLTC_MODE_STRICT 2

typedef struct bltc_ctx bltc_ctx;

/* EvalConfig (engine.py:46-62) + KernelSpec (kernels.py:42-55) + mode. */
typedef struct {
  double theta;          /* MAC parameter, (0, 1] */
  int32_t degree;        /* interpolation degree n >= 0 */
  int32_t kernel_code;   /* 0 Coulomb, 1 Yukawa, 2 test constant (kernels.py:39) */
  int64_t leaf_size;     /* N_L >= 1 */
  int64_t batch_size;    /* N_B >= 1 */
  double kappa;          /* Yukawa screening, finite >= 0 */
  int32_t mode;          /* BLTC_MODE_* */
  int32_t all_moments;   /* 1: moments for every eligible cluster (compute_all_moments);
                            0: only clusters that some approximation list reads */
} bltc_params;

/* RunStats (engine.py:338-347) plus device-side detail.  Times are CUDA-event
 * times on the context stream, in seconds. */
typedef struct {
  int64_t n_clusters;
  int64_t n_batches;
  int64_t direct_pairs;
  int64_t approx_pairs;
  double setup_s;        /* tree + batches + lists */
  double precompute_s;   /* moments */
  double compute_s;      /* evaluation + un-permute */
  double total_s;        /* setup + precompute + compute (device) */
  double h2d_s;          /* host->device copies (host-pointer entry points) */
  double d2h_s;
  double far_s;          /* far-field kernel time (FAST mode: separate kernel) */
  double near_s;         /* near-field kernel time */
  int64_t n_moments;     /* clusters whose moments were computed */
  int64_t kernel_launches;
  int32_t tree_depth;
  int32_t batch_depth;
  int32_t packed;        /* FAST: 1 = packed multi-batch work items, 0 = per-batch chunks */
  int32_t reserved;
  int64_t n_recomputed;  /* STRICT: targets recomputed in the reference's arithmetic
                            (-1: evaluated as PARITY throughout) */
  double strict_s;       /* STRICT: certificate + recompute time */
} bltc_stats;

BLTC_API const char* bltc_last_error(void);
BLTC_API const char* bltc_version(void);

/* device < 0: current device.  stream: a cudaStream_t to run on, or NULL for
 * a context-owned non-blocking stream. */
BLTC_API int bltc_create(int device, void* stream, bltc_ctx** out);
BLTC_API int bltc_destroy(bltc_ctx* ctx);
/* Non-zero: record per-phase CUDA events (needs stream syncs between phases). */
BLTC_API int bltc_set_timing(bltc_ctx* ctx, int enable);

/* treecode_potentials (engine.py:350-372) on HOST buffers: copies inputs H2D
 * (pinned host memory is used as such), runs tree/batches/lists/moments/
 * evaluation on the device and copies phi (original target order) D2H.
 * coincident != 0 means targets are the sources (ParticleSystem.coincident,
 * particles.py:62-64); then t* may equal s* and are not read separately. */
BLTC_API int bltc_treecode(bltc_ctx* ctx, const bltc_params* p, const double* cheb_s, int64_t n_t,
                  const double* tx, const double* ty, const double* tz, int64_t n_s,
                  const double* sx, const double* sy, const double* sz, const double* q,
                  int32_t coincident, double* phi_out, bltc_stats* stats);

/* Same on DEVICE buffers (inputs resident in HBM; phi_out device pointer). */
BLTC_API int bltc_treecode_device(bltc_ctx* ctx, const bltc_params* p, const double* cheb_s, int64_t n_t,
                         const double* tx, const double* ty, const double* tz, int64_t n_s,
                         const double* sx, const double* sy, const double* sz,
                         const double* q, int32_t coincident, double* phi_out,
                         bltc_stats* stats);

/* Setup + precompute only: build_source_tree, build_target_batches,
 * build_interaction_lists and the moments (compute_all_moments with
 * all_moments = 1) on HOST buffers, no evaluation -- the structures are then
 * read with the bltc_export_* calls below (tree.py:191-253, engine.py:128-130,
 * moments.py:147-150).  stats: pair counts, setup / precompute times. */
BLTC_API int bltc_build(bltc_ctx* ctx, const bltc_params* p, const double* cheb_s, int64_t n_t,
                        const double* tx, const double* ty, const double* tz, int64_t n_s,
                        const double* sx, const double* sy, const double* sz, const double* q,
                        int32_t coincident, bltc_stats* stats);

/* ---- Stage introspection of the last run (bit-exact checks) ------------- */
typedef struct {
  int64_t n_sources, n_targets;
  int64_t n_clusters, n_batches;
  int64_t n_approx, n_direct;      /* CSR entries */
  int64_t n_moments;
  int32_t degree;
  int32_t tree_depth, batch_depth;
  int32_t n_groups;                /* source trees in the last evaluation (ranks) */
} bltc_sizes;

BLTC_API int bltc_get_sizes(bltc_ctx* ctx, bltc_sizes* out);
/* which: 0 source tree (clusters, BFS order), 1 target partition (all nodes).
 * Arrays sized n_nodes (lo/hi: 3*n_nodes), perm sized n_particles.  Any
 * pointer may be NULL. */
BLTC_API int bltc_export_tree(bltc_ctx* ctx, int which, int64_t* n_nodes_out, int64_t* perm,
                     int64_t* start, int64_t* stop, double* lo, double* hi,
                     int64_t* child_start, int64_t* child_count, int32_t* level);
/* Target batches in DFS (= ascending start) order. */
BLTC_API int bltc_export_batches(bltc_ctx* ctx, int64_t* start, int64_t* stop, double* center,
                        double* radius);
/* Interaction lists, CSR over (batch, group) segments, batch-major: ptr sized
 * n_batches*n_groups+1; entries are forest cluster ids. */
BLTC_API int bltc_export_lists(bltc_ctx* ctx, int64_t* a_ptr, int64_t* a_idx, int64_t* d_ptr,
                      int64_t* d_idx);
/* Moments: cluster ids [n_moments] and rows [n_moments][(n+1)^3]. */
BLTC_API int bltc_export_moments(bltc_ctx* ctx, int64_t* cluster_ids, double* rows);
/* STRICT certificate of the last single-device run, per target in the
 * ORIGINAL order: S_i = absum_i + farbound_b (the absolute mass of the pair
 * terms; the FAST-vs-reference difference is bounded by Kc eps S_i) -- for
 * calibration and tests.  Needs bltc_strict_keep_bounds(ctx, 1) before the
 * run; *kc_out: the Kc in use. */
BLTC_API int bltc_strict_keep_bounds(bltc_ctx* ctx, int32_t enable);
BLTC_API int bltc_export_strict_bounds(bltc_ctx* ctx, double* bounds_out, double* kc_out);

/* run_distributed (decomp.py:483-593) in one process: R ranks on the given
 * devices (rank r on devices[r % n_devices]), one host thread per rank; the
 * caller's RCB (rcb_order / rank_start, e.g. the reference's rcb_partition)
 * decides each rank's particles and their order.  Ranks evaluate against
 * every rank's published buffers across devices (peer access where
 * available) in the reference's owner order.  Host pointers; phi_out in the
 * original order; stats: sums of the pair counts, max of the times. */
BLTC_API int bltc_run_distributed(int32_t ranks, const int32_t* devices, int32_t n_devices,
                                  const bltc_params* p, const double* cheb_s, int64_t n,
                                  const double* x, const double* y, const double* z,
                                  const double* q, const int64_t* rcb_order,
                                  const int64_t* rank_start, double* phi_out,
                                  bltc_stats* stats);

/* ---- Stage calls with host-provided upstream structures -------------------
 * Each stage of the pipeline on structures the caller built (e.g. the
 * reference's own tree / batches / lists / moments, flattened), so a stage
 * can be swapped in alone and checked bit for bit.  Trees are BFS cluster
 * arrays as bltc_export_tree returns them (start/stop into the reordered
 * particles, lo/hi [n][3], child_start/child_count), batches as
 * bltc_export_batches.  Host pointers.
 *
 * bltc_stage_lists: build_interaction_lists (engine.py:128-130) of the batches
 * against the tree; the lists stay in the context -- read them with
 * bltc_export_lists (sizes in *n_approx / *n_direct). */
BLTC_API int bltc_stage_lists(bltc_ctx* ctx, const bltc_params* p, int64_t n_batches,
                              const int64_t* batch_start, const int64_t* batch_stop,
                              const double* batch_center, const double* batch_radius,
                              int64_t n_clusters, const int64_t* start, const int64_t* stop,
                              const double* lo, const double* hi, const int64_t* child_start,
                              const int64_t* child_count, int64_t* n_approx, int64_t* n_direct);
/* bltc_stage_moments: compute_modified_charges (moments.py:132-144) of the
 * clusters cluster_ids[0..n_list) of a tree whose sources (x, y, z, q) are in
 * cluster order; rows_out [n_list][(n+1)^3], k1-major. */
BLTC_API int bltc_stage_moments(bltc_ctx* ctx, const bltc_params* p, const double* cheb_s,
                                int64_t n_s, const double* sx, const double* sy,
                                const double* sz, const double* q, int64_t n_clusters,
                                const int64_t* start, const int64_t* stop, const double* lo,
                                const double* hi, int64_t n_list, const int64_t* cluster_ids,
                                double* rows_out);
/* bltc_stage_potentials: compute_potentials (engine.py:315-335).  Targets in
 * batch order, sources in cluster order; lists as CSR over batches (entries:
 * cluster ids); moment_row[c] = row of cluster c in rows ([n_rows][(n+1)^3]),
 * -1 if none (every approximated cluster needs one).  perm (original index ->
 * batch-order position) gives phi in the original order, NULL keeps batch
 * order. */
BLTC_API int bltc_stage_potentials(bltc_ctx* ctx, const bltc_params* p, const double* cheb_s,
                                   int64_t n_t, const double* tx, const double* ty,
                                   const double* tz, int64_t n_batches,
                                   const int64_t* batch_start, const int64_t* batch_stop,
                                   const double* batch_center, const double* batch_radius,
                                   int64_t n_s, const double* sx, const double* sy,
                                   const double* sz, const double* q, int64_t n_clusters,
                                   const int64_t* start, const int64_t* stop, const double* lo,
                                   const double* hi, const int64_t* a_ptr, const int64_t* a_idx,
                                   const int64_t* d_ptr, const int64_t* d_idx,
                                   const int64_t* moment_row, int64_t n_rows,
                                   const double* rows, const int64_t* perm, double* phi_out,
                                   bltc_stats* stats);

/* ---- Distributed (one rank per GPU; decomp.py:483-593) ------------------
 * Each rank: bltc_rank_build (local tree, batches, moments of every cluster
 * that may be approximated) -> bltc_rank_publish_sizes / bltc_rank_publish
 * (flattened TreeArray records, decomp.py:137-189, + particles + moment
 * rows into caller-provided DEVICE buffers) -> the caller all-gathers those
 * buffers (NCCL over NVLink) -> bltc_rank_evaluate against the gathered
 * forest in the reference's owner order (local first, then remote owners
 * ascending; decomp.py:437-454). */
typedef struct {
  int64_t n_clusters;
  int64_t n_particles;
  int64_t n_moment_rows;
  int64_t record_doubles;   /* doubles per cluster record */
} bltc_publish_sizes;

BLTC_API int bltc_rank_build(bltc_ctx* ctx, const bltc_params* p, const double* cheb_s, int64_t n,
                    const double* x, const double* y, const double* z, const double* q,
                    int32_t device_ptrs);
/* Optional, before bltc_rank_build: the bounding box of ALL ranks' targets
 * (lo[3], hi[3]).  The rank then computes and publishes moment rows only for
 * clusters some batch inside that box could accept (r_C / theta reachable,
 * engine.py:65-85); NULL restores "every cluster that passes the size test". */
BLTC_API int bltc_rank_set_domain(bltc_ctx* ctx, const double* lo, const double* hi);
/* The same with the domain as a union of n_boxes boxes, boxes[6k..6k+5] =
 * (lo xyz, hi xyz), every batch centre inside one of them (n_boxes = 0:
 * unset).  Host pointer; copied. */
BLTC_API int bltc_rank_set_domain_boxes(bltc_ctx* ctx, int64_t n_boxes, const double* boxes);
/* Host helper: the minimal bounding boxes of the occupied cells of a grid^3
 * grid over the points' bounding box (grid <= 64), in cell order; boxes
 * needs room for 6 grid^3 doubles.  The domain bltc_run_distributed passes
 * to its ranks (grid 16). */
BLTC_API int bltc_domain_cells(int64_t n, const double* x, const double* y, const double* z,
                               int32_t grid, double* boxes, int64_t* n_boxes);
BLTC_API int bltc_rank_publish_sizes(bltc_ctx* ctx, bltc_publish_sizes* out);
/* records: [n_clusters][record_doubles]; particles: [4][n_particles] (x,y,z,q);
 * moments: [n_moment_rows][(n+1)^3 rounded up to even].  All device pointers. */
BLTC_API int bltc_rank_publish(bltc_ctx* ctx, double* records, double* particles, double* moments);
/* Forest of R published trees (device pointers, one per owner rank, owner
 * order 0..R-1); my_rank's own entry is the local tree.  phi_out: host (or
 * device if device_ptrs) buffer in the rank's ORIGINAL particle order. */
BLTC_API int bltc_rank_evaluate(bltc_ctx* ctx, const bltc_params* p, int32_t ranks, int32_t my_rank,
                       const int64_t* n_clusters, const int64_t* n_particles,
                       const int64_t* n_moment_rows, const double* const* records,
                       const double* const* particles, const double* const* moments,
                       double* phi_out, int32_t device_ptrs, bltc_stats* stats);

/* LET step one (decomp.py:354-379, build_let): the interaction lists of this
 * rank's batches against every owner's published tree records (device
 * pointers, owner order 0..R-1; only the geometry / count / child fields are
 * read).  flags_out (device, int32, sum of n_clusters, owner order 0..R-1,
 * zeroed here): bit 0 = some batch approximates the cluster (its moment row
 * is needed), bit 1 = some batch sums it directly (its particles are
 * needed).  Step two (fetching exactly those rows and slices) is the
 * caller's exchange; the fetched data, with the records' particle ranges and
 * moment rows remapped into the fetched buffers, then go to
 * bltc_rank_evaluate unchanged. */
BLTC_API int bltc_rank_needs(bltc_ctx* ctx, const bltc_params* p, int32_t ranks, int32_t my_rank,
                             const int64_t* n_clusters, const double* const* records,
                             int32_t* flags_out);

/* ---- Verification oracle on the device (cli.py:73-149) --
 * Brute-force Neumaier direct sums at the targets idx[0..n_idx) (indices into
 * tx/ty/tz; NULL idx = all n_t targets) over all sources, singular pairs
 * skipped.  mode PARITY: sequential IEEE per target (bitwise the CPU oracle
 * for Coulomb); FAST: split sources, rsqrt.  Host pointers. */
BLTC_API int bltc_direct_sum(bltc_ctx* ctx, int32_t kernel_code, double kappa, int32_t mode,
                             int64_t n_idx, const int64_t* idx, int64_t n_t, const double* tx,
                             const double* ty, const double* tz, int64_t n_s, const double* sx,
                             const double* sy, const double* sz, const double* q,
                             double* out);

/* ---- Input generation on the device (cli.py:54-62) ----
 * numpy's Generator(Philox).uniform(low, high, (n, dims)) stream, bit for bit,
 * from the bit generator's key[2] and counter[4] (numpy state, read on the
 * host): draw j goes to out[j % dims][j / dims].  out: dims device pointers
 * of n doubles.  Runs on the default stream and synchronises. */
BLTC_API int bltc_philox_uniform(int device, const uint64_t* key, const uint64_t* counter,
                                 int64_t n, int32_t dims, double low, double high,
                                 double* const* out);

/* ---- Diagnostics --------------------------------------------------------
 * Sustained FP64 FMA throughput of the device (DFMA/s), measured for about
 * `seconds`: the denominator of the FP64 roofline fraction bench.py reports. */
BLTC_API int bltc_probe_fp64(int device, double seconds, double* dfma_per_s);
/* Kernels libbltc has launched in this process so far (all contexts): the
 * benchmark's count of its own launches inside a timed region. */
BLTC_API int bltc_launch_count(int64_t* out);
/* exp(x[i]) for i < n with the device port of the host libm exp the
 * reference's Yukawa tiles call (csrc/libm_exp.cuh); host pointers.  Lets a
 * test compare the device build with the host's exp bit for bit. */
BLTC_API int bltc_libm_exp_device(int device, int64_t n, const double* x, double* y);

#ifdef __cplusplus
}
#endif
#endif /* BLTC_H */
