/*
 * gosma_capi.h — the C ABI of the B200-native GOSMA bound-evaluation path.
 *
 * Plain C types only (pointers, sizes, doubles); no torch or CUDA types in the
 * signatures (streams are passed as void*). Each entry point names the
 * reference interface it replaces (paths relative to /root/reference/proj).
 *
 * Error behaviour mirrors the reference: invalid arguments return
 * GOSMA_EINVAL (reference: std::invalid_argument), an empty feasible domain
 * returns GOSMA_EINFEASIBLE (reference: InfeasiblePoseError), a solve that
 * stopped on a budget with an incumbent returns GOSMA_EBUDGET (reference CLI
 * exit code 3, tools/smalign_main.cpp:166); CUDA failures return >= 10. The
 * message of the last failure on the calling thread is gosma_last_error().
 * Infeasible branches are reported as {+inf, +inf}, not as errors
 * (core/src/bounds.cpp:277-279).
 */
#ifndef GOSMA_CAPI_H
#define GOSMA_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GOSMA_OK 0
#define GOSMA_EINVAL 1
#define GOSMA_EINFEASIBLE 2
#define GOSMA_EBUDGET 3
#define GOSMA_ECUDA 10
#define GOSMA_ENOMEM 11

typedef struct gosma_ctx gosma_ctx;

/* One semantic class: the model GMM and the image vMF mixture, as the
 * reference builds ObjectiveContext::ClassData from them
 * (core/include/smalign/objective.hpp:19-31, core/src/objective.cpp:28-68).
 * Arrays are caller-owned and deep-copied by gosma_ctx_create. */
typedef struct gosma_class_view {
  int n1;               /* model (GMM) components */
  int n2;               /* image (vMF) components */
  double class_weight;  /* SemanticClass::weight (mixtures.hpp:46-51) */
  const double* mu;     /* 3*n1, component means */
  const double* sigma2; /* n1, isotropic variances (> 0) */
  const double* phi1;   /* n1, weights (sum 1 within 1e-9) */
  const double* dir;    /* 3*n2, unit mean directions (|dir| within 1e-6 of 1) */
  const double* kappa2; /* n2, concentrations (> 0) */
  const double* phi2;   /* n2, weights (sum 1 within 1e-9) */
} gosma_class_view;

/* Search node: rotation cube x translation cuboid + inherited lower bound.
 * Replaces smalign::BranchRegion (core/include/smalign/se3.hpp:38-45); the
 * upper field of BranchRegion is output-only and not carried. 88 bytes. */
typedef struct gosma_node {
  double rc[3]; /* RotationCube::center (axis-angle) */
  double rhw;   /* RotationCube::half_width */
  double tc[3]; /* TranslationCuboid::center */
  double thw[3];/* TranslationCuboid::half_widths */
  double lower; /* BranchRegion::lower (parent floor; -inf for roots) */
} gosma_node;

/* Context flags. */
#define GOSMA_CTX_SINGLE_MIXTURE 1u /* ObjectiveContext(Gmm, Vmfmm, zeta): one class of
                                       weight 1, no class-weight closure check
                                       (objective.cpp:103-107) */

/* Replaces ObjectiveContext(const SemanticMixturePair&, double zeta)
 * (objective.hpp:33-34, objective.cpp:103-121). Validates like the reference
 * (zeta > 0, non-empty classes, weight closure 1e-9, sigma2 > 0, kappa > 0,
 * weights >= 0, unit directions within 1e-6) and uploads the mixtures to
 * `device` (FP64 master + FP32 working tables). */
int gosma_ctx_create(int device, const gosma_class_view* classes, int n_classes, double zeta,
                     unsigned flags, gosma_ctx** out);

/* Replaces ObjectiveContext::blurred (objective.hpp:36-43, objective.cpp:70-101). */
int gosma_ctx_blurred(const gosma_ctx* ctx, double w, double reference_distance,
                      gosma_ctx** out);

void gosma_ctx_destroy(gosma_ctx* ctx);

/* ObjectiveContext::image_self_energy (objective.hpp:50-52). */
double gosma_ctx_image_self_energy(const gosma_ctx* ctx);

/* ObjectiveContext::zeta (objective.hpp:46). */
double gosma_ctx_zeta(const gosma_ctx* ctx);

/* Lower-bound soundness margin. By default every lower
 * bound has subtracted (a) the kernel's per-term FP32 error estimate and (b)
 * rel_margin x the node's |term| mass (default 2e-7), so it never exceeds the
 * FP64 value. rel_margin < 0 selects the raw FP32 core (no margin at all),
 * for parity diagnostics only. */
int gosma_ctx_set_lb_margin(gosma_ctx* ctx, double rel_margin);

/* Branch + bound in one call (the solver's wave step): the 8 children of each
 * parent, subdivide_adaptive (se3.cpp:107-147) with the given split flags
 * (d_split[i] = 1 rotation, 0 translation: the flag gosma_eval_bounds returns
 * for the parent), are bounded; child c of parent i is slot 8i+c of d_lower /
 * d_upper / d_child_split. Rotation-split parents evaluate their cuboid's
 * prologue and self sums once for all 8 children. Children inherit the
 * parent's lower field as their floor. Device pointers, asynchronous on
 * `stream` (no host synchronisation: the rotation / translation split counts
 * stay on the device); the context's child scratch is reused, so calls on one
 * context must be ordered (one stream per context). Results equal
 * gosma_eval_bounds_device on the explicit children to 1e-12 of the |term|
 * mass. */
int gosma_eval_children_device(gosma_ctx* ctx, const gosma_node* d_parents, const int8_t* d_split,
                               size_t n, double skip_upper_at, double* d_lower, double* d_upper,
                               int8_t* d_child_split, void* stream);

/* Replaces evaluate_branch_batch(ctx, branches, threads, skip_upper_at)
 * (core/include/smalign/solver.hpp:87-95, core/src/solver.cpp:260-292) and,
 * per element, evaluate_bounds (core/src/bounds.cpp:275-284). Host buffers;
 * synchronous; results in input order and independent of launch geometry.
 * split_rot (optional, may be NULL) receives subdivide_adaptive's choice for
 * the node (1 rotation, 0 translation, -1 not splittable;
 * core/src/se3.cpp:107-121). */
int gosma_eval_bounds(gosma_ctx* ctx, const gosma_node* nodes, size_t n, double skip_upper_at,
                      double* lower, double* upper, int8_t* split_rot);

/* Same, with device-resident buffers, asynchronous on `stream`
 * (cudaStream_t; NULL = the context's stream). */
int gosma_eval_bounds_device(gosma_ctx* ctx, const gosma_node* d_nodes, size_t n,
                             double skip_upper_at, double* d_lower, double* d_upper,
                             int8_t* d_split_rot, void* stream);

/* Translation-cached variant: the translation-only (self) terms are computed
 * once per distinct translation cuboid (d_tindex[k] names node k's cuboid in
 * d_tboxes = {tc[3], thw[3]} records) and reused; the reference adds self
 * and cross terms separately (bounds.cpp:180) so results are identical up to
 * FP32 summation order. */
int gosma_eval_bounds_cached_device(gosma_ctx* ctx, const gosma_node* d_nodes, size_t n,
                                    const int32_t* d_tindex, const double* d_tboxes,
                                    size_t n_tboxes, double skip_upper_at, double* d_lower,
                                    double* d_upper, int8_t* d_split_rot, void* stream);

/* Host FP64 objective (objective.cpp:227-235); GOSMA_EINFEASIBLE when the
 * pose violates the standoff (objective.cpp:160-166). */
int gosma_objective_value(const gosma_ctx* ctx, const double r[3], const double t[3],
                          double* value);

/* Host FP64 analytic gradient d/dr, d/dt (objective.cpp:254-334). */
int gosma_objective_gradient(const gosma_ctx* ctx, const double r[3], const double t[3],
                             double g[6]);

/* Pose domain (se3.hpp:32-36): one rotation cube, n_boxes translation
 * cuboids as {center[3], half_widths[3]} records. */
typedef struct gosma_domain {
  double rot_center[3];
  double rot_half_width;
  const double* boxes;
  int n_boxes;
} gosma_domain;

/* Local refinement (SMA) — local_refine (solver.hpp:80-85, solver.cpp:164-258). */
int gosma_local_refine(const gosma_ctx* ctx, const double r0[3], const double t0[3],
                       const gosma_domain* domain, double r_out[3], double t_out[3],
                       double* value);

/* Batched local refinement on the GPU: n starts (r0, t0:
 * n*3 doubles each, row-major), each refined by one CTA running the same
 * L-BFGS / strong-Wolfe / projection loop as gosma_local_refine on the FP64
 * device objective. value[k] is the host FP64 objective at the returned pose
 * (never worse than the start unless the device and host objectives disagree
 * in the last bits). Replaces n calls of local_refine
 * (solver.hpp:80-85) as issued by the discovery dive (solver.cpp:560-595). */
int gosma_local_refine_batch(gosma_ctx* ctx, size_t n, const double* r0, const double* t0,
                             const gosma_domain* domain, double* r_out, double* t_out,
                             double* value);

/* Replaces SolverConfig (solver.hpp:14-37). Negative time_limit /
 * max_evaluations / queue_capacity mean "unset". */
typedef struct gosma_config {
  double epsilon;
  double zeta;
  int batch_size;          /* nodes expanded per wave = batch_size / 8 (solver.cpp:648-649) */
  double time_limit;
  long long max_evaluations;
  long long queue_capacity;
  int threads;             /* host threads for SMA; 0 = hardware concurrency */
  unsigned long long seed;
  int wave_nodes;          /* GPU frontier: max nodes expanded per wave (0 = auto) */
  int discovery_dive;      /* 1 = run the blurred-context dive (solver.cpp:449-595) */
} gosma_config;

#define GOSMA_STATUS_EPSILON_OPTIMAL 0
#define GOSMA_STATUS_TIME_LIMIT 1
#define GOSMA_STATUS_QUEUE_EXHAUSTED 2

/* Replaces SolverReport (solver.hpp:64-73). */
typedef struct gosma_report {
  double best_r[3];
  double best_t[3];
  double best_value;
  double global_lower;
  double gap;
  int status;
  unsigned long long branches_expanded;
  unsigned long long sma_invocations;
  unsigned long long bound_evaluations;
  double wall_time_seconds;
  unsigned long long waves;
} gosma_report;

/* Per-wave trace callback (TraceEntry, solver.hpp:45-55). May be NULL. */
typedef void (*gosma_trace_cb)(void* user, unsigned long long wave,
                               unsigned long long bound_evaluations, double best_upper,
                               double global_lower, unsigned long long queue_size,
                               double unexplored_fraction, double pruned_fraction,
                               double resolved_fraction);

/* Replaces solve(ctx, domain, config) (solver.hpp:97-103, solver.cpp:312-688):
 * GPU-resident best-first frontier, host SMA. */
int gosma_solve(gosma_ctx* ctx, const gosma_domain* domain, const gosma_config* config,
                gosma_report* report, gosma_trace_cb trace, void* user);

/* ---- Stepwise solver: the same branch-and-bound as gosma_solve, one wave per
 * call, so a driver can shard the frontier across GPUs (one rank per GPU) and
 * exchange the incumbent / frontier minimum between waves.
 * gosma_solve is exactly: create(rank 0, world 1); loop { status; certify;
 * stop rules; expand(d* - eps) }. */
typedef struct gosma_solver gosma_solver;

typedef struct gosma_wave_status {
  double best_value;       /* local incumbent d* (FP64 objective) */
  double frontier_min;     /* min lower bound over the local frontier (+inf if empty) */
  double floor_lower;      /* min lower bound of resolved / folded nodes */
  unsigned long long live_nodes;
  unsigned long long bound_evaluations;
  double pruned_volume, resolved_volume, total_volume;
  double elapsed_seconds;
} gosma_wave_status;

/* Every rank runs wave 0 and the discovery dive over all roots; with
 * world > 1 the roots are expanded deterministically to >= 8 x SMs nodes and
 * rank `rank` keeps nodes rank, rank + world, ... */
int gosma_solver_create(gosma_ctx* ctx, const gosma_domain* domain, const gosma_config* config,
                        int rank, int world, gosma_solver** out);
void gosma_solver_destroy(gosma_solver* solver);
/* Local statistics for the global certificate max(prev, min(d*, frontier_min,
 * floor)) (solver.cpp:626-627); applies capacity folding first. */
int gosma_solver_status(gosma_solver* solver, gosma_wave_status* status);
/* An incumbent value found elsewhere (another rank): prunes, carries no pose. */
int gosma_solver_set_incumbent(gosma_solver* solver, double value);
/* One wave: expand the best nodes with lower < limit (normally d* - eps),
 * bound the children, update the incumbent (+SMA), route. Children whose
 * lower bound is >= min(limit, d*) are finished: they join the certificate's
 * floor instead of the frontier, so later calls must not raise the limit
 * (d* - eps never rises). max_evals > 0 caps the children evaluated. */
int gosma_solver_expand(gosma_solver* solver, double limit, unsigned long long max_evals);
/* Frontier rebalancing: remove up to max_nodes of the best live nodes into
 * host buffers / add nodes received from another rank. */
int gosma_solver_export(gosma_solver* solver, size_t max_nodes, gosma_node* nodes, int8_t* split,
                        double* volume, size_t* n_out);
int gosma_solver_import(gosma_solver* solver, const gosma_node* nodes, const int8_t* split,
                        const double* volume, size_t n);
/* Device-buffer variants (rebalancing over NCCL without host staging): the
 * same records in device memory; export's buffers hold at least max_nodes. */
int gosma_solver_export_device(gosma_solver* solver, size_t max_nodes, gosma_node* d_nodes,
                               int8_t* d_split, double* d_vol, size_t* n_out);
int gosma_solver_import_device(gosma_solver* solver, const gosma_node* d_nodes,
                               const int8_t* d_split, const double* d_vol, size_t n);
/* Local incumbent pose / value and counters (global_lower, gap, status are
 * the driver's). */
int gosma_solver_result(gosma_solver* solver, gosma_report* report);
/* Volume still held by the live frontier (a full pass over the pool; for the
 * ledger check total = pruned + resolved + live, solver.cpp:597-608). */
int gosma_solver_live_volume(gosma_solver* solver, double* volume);

const char* gosma_last_error(void);

/* Build / device introspection for benches and tests. */
int gosma_device_info(int device, int* sm_count, int* sm_clock_khz, int* cc_major,
                      int* cc_minor);
/* A finished solver's device buffers are kept per device for the next solve
 * instead of being freed (the frontier pool when >= 16M nodes; every other
 * frontier block, up to 8 GB, in an exact-size cache): cudaMalloc / cudaFree
 * of large blocks cost milliseconds to tenths of a second. This frees what is
 * kept for `device`. */
int gosma_release_cached_memory(int device);

/* Batched objective_value + objective_gradient (objective.cpp:175-334) on the
 * GPU in FP64 (kernel K6, the local refiner's evaluator): poses = n x {r[3],
 * t[3]}; f[n] (+inf where the pose is within zeta of a mean) and g[6n]
 * ({d/dr, d/dt}, zero where infeasible). Synchronous. */
int gosma_objective_batch(gosma_ctx* ctx, const double* poses, size_t n, double* f, double* g);

/* ---- Mixture construction (host C++; mixtures.hpp:55-98) ------------------
 * Replaces smalign::build_semantic_mixtures (mixtures.cpp:269-362) and the
 * DP-means clusterers it uses (mixtures.cpp:49-182); bit-identical results. */
typedef struct gosma_mixtures gosma_mixtures;

/* points: 3*n_points doubles; bearings: 3*n_bearings doubles, each within 1e-6
 * of unit length (UnitVector3, renormalised). point_labels / bearing_labels:
 * one C string per element, or both NULL (a single class "all"). weight_labels
 * / weights: n_weights class weights (LabeledPointSet class_weights), or NULL
 * for uniform weights. Invalid input -> GOSMA_EINVAL with the reference's
 * message. */
int gosma_mixtures_build(const double* points, const char* const* point_labels,
                         size_t n_points, const double* bearings,
                         const char* const* bearing_labels, size_t n_bearings, double lambda_p,
                         double lambda_f, const char* const* weight_labels,
                         const double* weights, size_t n_weights, gosma_mixtures** out);
int gosma_mixtures_class_count(const gosma_mixtures* m);
/* Class k (in the reference's order: sorted class ids) as a view usable with
 * gosma_ctx_create; the arrays are owned by m. */
int gosma_mixtures_class(const gosma_mixtures* m, int k, gosma_class_view* view,
                         const char** id);
int gosma_mixtures_warning_count(const gosma_mixtures* m);
const char* gosma_mixtures_warning(const gosma_mixtures* m, int k);
void gosma_mixtures_destroy(gosma_mixtures* m);

/* dp_means / dp_vmf_means (mixtures.cpp:49-182). assignment: n ints; centers:
 * 3*centers_cap doubles; shuffle (0/1) + seed = the optional shuffle seed;
 * *iterations = length of the objective history. */
int gosma_dp_means(const double* points, size_t n, double lambda_p, int shuffle,
                   unsigned long long seed, int* assignment, double* centers, size_t centers_cap,
                   size_t* n_centers, int* iterations);
int gosma_dp_vmf_means(const double* bearings, size_t n, double lambda_f, int shuffle,
                       unsigned long long seed, int* assignment, double* centers,
                       size_t centers_cap, size_t* n_centers, int* iterations);

/* Pipe-throughput microbenchmarks (roofline denominators): MUFU (SFU/XU)
 * ops/s and FP32 FMA flop/s measured on `device` at its current clocks. */
int gosma_calibrate_pipes(int device, double* mufu_ops_per_s, double* fma_flops_per_s);
/* Number of bound-kernel launches issued by this process so far. */
unsigned long long gosma_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* GOSMA_CAPI_H */
