// Internal types shared by the CUDA kernels and the host runtime.
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "gosma_capi.h"

namespace gosma {

// log2(e): exponents are carried in log2 units so every exp is one MUFU.EX2.
constexpr float kL2E = 1.4426950408889634f;
// Margin below which a pair is dropped from the objective
// (objective.cpp:17 kNegligibleExponentMargin).
constexpr double kNegligibleMargin = 64.0;
// log(phi) stand-in for zero weights: keeps 2^(e) exactly 0 without inf-inf.
constexpr float kLogZeroWeight = -1.0e30f;

// Per-class span of the pooled component tables.
struct ClassSpan {
  int o1, n1, o2, n2;
};

// Device view of an ObjectiveContext (objective.hpp:19-31), passed by value.
// FP64 master copies feed the per-node prep (feasibility, kappa intervals,
// projections); FP32 tables feed the pair loops.
struct DevCtx {
  int n_classes;
  int n1_total;
  int n2_total;
  int max_n1;            // largest class n1 (self-loop sizing)
  const ClassSpan* cls;  // n_classes
  const double* cls_w;   // n_classes
  const double* mu;      // 3*N1 component means
  const double* inv_s2;  // N1, 1/sigma^2
  const double* phi1;    // N1
  const float* log_phi1; // N1 (kLogZeroWeight for 0)
  const double* m;       // 3*N2, b_j / kappa_j (bounds.cpp:100)
  const float* kappa2;   // N2
  const float* g2;       // N2, phi2 / W(kappa2), W(k) = (1 - e^{-2k}) / k
  double zeta;
  double lb_margin;      // relative soundness floor (x |term| mass)
  double lb_err_scale;   // 1: subtract the FP32 error estimate; 0: raw core (diagnostics)
  int tail_chunks;       // some class has a last row chunk of <= 16 of 32 rows
  int max_n2;            // largest class n2
  int stream_classes;    // full mode keeps one class's table at a time (n_classes > 1)
  int precise;           // precise fix-up for nodes whose FP32 error estimate is large
  double redo_rel;       // fix-up threshold: amplified estimate / cross mass
  float min_k2;          // smallest image concentration (K1's exact-path gate)
};

// Host-side master copy of one class (ClassData, objective.hpp:19-31).
struct HostClass {
  double weight = 1.0;
  std::vector<double> mu;      // 3*n1
  std::vector<double> sigma2;  // n1
  std::vector<double> phi1;    // n1
  std::vector<double> b;       // 3*n2, kappa * unit direction
  std::vector<double> kappa2;  // n2
  std::vector<double> log_z2;  // n2
  std::vector<double> phi2;    // n2
  double self_energy = 0.0;
  int n1() const { return static_cast<int>(sigma2.size()); }
  int n2() const { return static_cast<int>(kappa2.size()); }
};

// Kernel entry points (bounds_kernel.cu).
struct EvalArgs {
  const double* nodes;   // 11 doubles per node (gosma_node)
  long long n;
  double skip_upper_at;
  double* lower;
  double* upper;
  int8_t* split_rot;     // may be null
  unsigned int* work;    // dynamic work counter (zeroed before launch)
  // translation-cached modes: per-cuboid {lb_self, ub_self, lb_err, flag}
  double* self_out = nullptr;
  const int32_t* tindex = nullptr;  // node -> cuboid (cross-cached mode)
  const int* item_index = nullptr;  // optional work list: item -> node slot (or selection k)
  const unsigned int* sel = nullptr;  // siblings mode: selection k -> pool slot
  const long long* n_dev = nullptr;   // item count in device memory (<= n, which sizes the grid)
  // precise fix-up: nodes whose cross-term error estimate has a
  // large theta/B-amplified part are appended here by the main pass (node
  // record + output slot) and re-evaluated by a second launch with the
  // alignment angle's numerator in FP64; null: no fix-up
  unsigned long long* redo_count = nullptr;
  double* redo_nodes = nullptr;      // 11 doubles per entry
  long long* redo_slot = nullptr;    // output slot of each entry
  long long redo_cap = 0;
  const long long* out_slot = nullptr;  // fix-up launches: item -> output slot
};

cudaError_t launch_eval_bounds(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                               cudaStream_t stream);
// Translation-cached evaluation: self sums once per cuboid (a.nodes are the
// cuboids as nodes, a.self_out receives 4 doubles each), then cross terms per
// node with a.tindex mapping nodes to cuboids.
// Rotation-split parents (item_index = selection indices k, sel = pool slots):
// writes the bounds and split flags of children 8k .. 8k+7.
cudaError_t launch_eval_siblings(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                                 cudaStream_t stream);
cudaError_t launch_eval_self(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                             cudaStream_t stream);
cudaError_t launch_eval_cross_cached(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                                     cudaStream_t stream);
// Shared-memory table bytes per lane group: every class's rows and columns
// (mode < 0: the largest over the modes), or one class's at a time for the
// class-streamed full mode of a multi-class context (mode 4).
size_t eval_smem_per_warp(const DevCtx& ctx, int mode = -1);
cudaError_t make_children(const gosma_node* d_parents, const int8_t* d_split, size_t n,
                          gosma_node* d_kids, int* d_rot, int* d_trans,
                          unsigned long long* d_counts, unsigned int* d_sel,
                          cudaStream_t stream);
cudaError_t boxes_as_nodes(const double* d_boxes, size_t n, gosma_node* d_out,
                           cudaStream_t stream);
unsigned long long bound_kernel_launch_count();

// Host FP64 math (host_math.cpp) shared by SMA, the solver and the C ABI.
double log_z_eval(double kappa);
double log_z_deriv(double kappa);

}  // namespace gosma
