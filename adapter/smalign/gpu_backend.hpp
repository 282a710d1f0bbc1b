// smalign/gpu_backend.hpp — the B200 backend of the reference's solver API.
//
// The header a maintainer adds next to core/include/smalign/solver.hpp in the
// reference tree. It keeps the reference's types
// (ObjectiveContext, BranchRegion, BoundPair, PoseDomain, SolverConfig,
// SolverReport, TraceEntry, the exception taxonomy of errors.hpp) and routes
// the two hot entry points through the C ABI of include/gosma_capi.h:
//
//   smalign::evaluate_branch_batch(ctx, branches, threads, skip)
//       (solver.hpp:87-95, solver.cpp:260-292)
//     -> smalign::gpu::evaluate_branch_batch(gctx, branches, threads, skip)
//   smalign::solve(ctx, domain, config)   (solver.hpp:97-103, solver.cpp:312-688)
//     -> smalign::gpu::solve(gctx, domain, config)
//
// where gctx = smalign::gpu::Context(ctx) uploads the context's flattened
// per-class data (ObjectiveContext::ClassData, objective.hpp:19-31) once.
// Build: -I<repo>/include, link <repo>/paper_1812_01232_b200/libgosma.so.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

#include "gosma_capi.h"
#include "smalign/errors.hpp"
#include "smalign/solver.hpp"

namespace smalign::gpu {

// Maps the C ABI's error codes onto the reference's exceptions
// (errors.hpp:10-27; CLI codes smalign_main.cpp:5-6).
inline void check(int rc) {
  if (rc == GOSMA_OK || rc == GOSMA_EBUDGET) return;
  const std::string msg = gosma_last_error();
  if (rc == GOSMA_EINVAL) throw std::invalid_argument(msg);
  if (rc == GOSMA_EINFEASIBLE) throw InfeasiblePoseError(msg);
  throw std::runtime_error("gosma: " + msg);
}

// The device copy of an ObjectiveContext (deep copy; the reference context may
// be destroyed afterwards). One context per (host thread, device).
class Context {
 public:
  explicit Context(const ObjectiveContext& ctx, int device = 0) {
    const auto& cls = ctx.classes();
    std::vector<std::vector<double>> buf;
    buf.reserve(6 * cls.size());
    std::vector<gosma_class_view> views;
    for (const auto& c : cls) {
      auto& mu = buf.emplace_back();
      auto& dir = buf.emplace_back();
      for (const auto& m : c.mu) mu.insert(mu.end(), {m.x(), m.y(), m.z()});
      for (std::size_t j = 0; j < c.b.size(); ++j) {
        const Eigen::Vector3d d = c.b[j] / c.kappa2[j];  // b = kappa * direction
        dir.insert(dir.end(), {d.x(), d.y(), d.z()});
      }
      views.push_back({static_cast<int>(c.sigma2.size()), static_cast<int>(c.kappa2.size()),
                       c.class_weight, mu.data(), c.sigma2.data(), c.phi1.data(), dir.data(),
                       c.kappa2.data(), c.phi2.data()});
    }
    const unsigned flags =
        (cls.size() == 1 && cls[0].class_weight == 1.0) ? GOSMA_CTX_SINGLE_MIXTURE : 0u;
    check(gosma_ctx_create(device, views.data(), static_cast<int>(views.size()), ctx.zeta(),
                           flags, &ctx_));
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ~Context() { gosma_ctx_destroy(ctx_); }
  gosma_ctx* get() const { return ctx_; }

 private:
  gosma_ctx* ctx_ = nullptr;
};

inline gosma_node to_node(const BranchRegion& b) {
  gosma_node n;
  for (int a = 0; a < 3; ++a) {
    n.rc[a] = b.rotation.center[a];
    n.tc[a] = b.translation.center[a];
    n.thw[a] = b.translation.half_widths[a];
  }
  n.rhw = b.rotation.half_width;
  n.lower = b.lower;
  return n;
}

// evaluate_branch_batch (solver.hpp:87-95): bounds in input order, the
// reference's {+inf, +inf} for infeasible branches; `threads` is accepted for
// signature compatibility (the GPU result does not depend on it). Lower bounds
// are certified (never above the FP64 reference value).
inline std::vector<BoundPair> evaluate_branch_batch(
    const Context& ctx, const std::vector<BranchRegion>& branches, int /*threads*/ = 0,
    double skip_upper_at = std::numeric_limits<double>::infinity()) {
  std::vector<BoundPair> out(branches.size());
  if (branches.empty()) return out;
  std::vector<gosma_node> nodes(branches.size());
  for (std::size_t k = 0; k < branches.size(); ++k) nodes[k] = to_node(branches[k]);
  std::vector<double> lo(nodes.size()), up(nodes.size());
  check(gosma_eval_bounds(ctx.get(), nodes.data(), nodes.size(), skip_upper_at, lo.data(),
                          up.data(), nullptr));
  for (std::size_t k = 0; k < out.size(); ++k) {
    out[k].lower = lo[k];
    out[k].upper = up[k];
  }
  return out;
}

// solve (solver.hpp:97-103): the GPU-resident branch-and-bound. Same
// validation (std::invalid_argument / InfeasiblePoseError), stop rules,
// report fields and per-wave trace.
inline SolverReport solve(const Context& ctx, const PoseDomain& domain,
                          const SolverConfig& config) {
  std::vector<double> boxes;
  for (const auto& b : domain.translations)
    boxes.insert(boxes.end(), {b.center.x(), b.center.y(), b.center.z(), b.half_widths.x(),
                               b.half_widths.y(), b.half_widths.z()});
  gosma_domain d;
  for (int a = 0; a < 3; ++a) d.rot_center[a] = domain.rotation.center[a];
  d.rot_half_width = domain.rotation.half_width;
  d.boxes = boxes.data();
  d.n_boxes = static_cast<int>(domain.translations.size());
  gosma_config c;
  c.epsilon = config.epsilon;
  c.zeta = config.zeta;
  c.batch_size = config.batch_size;
  c.time_limit = config.time_limit ? *config.time_limit : -1.0;
  c.max_evaluations =
      config.max_evaluations ? static_cast<long long>(*config.max_evaluations) : -1;
  c.queue_capacity = config.queue_capacity ? static_cast<long long>(*config.queue_capacity) : -1;
  c.threads = config.threads;
  c.seed = config.seed;
  c.wave_nodes = 0;
  c.discovery_dive = 1;
  SolverReport r;
  auto cb = [](void* user, unsigned long long wave, unsigned long long evals, double ub,
               double lb, unsigned long long q, double fu, double fp, double fr) {
    TraceEntry t;
    t.wave = wave;
    t.bound_evaluations = evals;
    t.best_upper = ub;
    t.global_lower = lb;
    t.queue_size = static_cast<std::size_t>(q);
    t.unexplored_volume_fraction = fu;
    t.pruned_volume_fraction = fp;
    t.resolved_volume_fraction = fr;
    static_cast<SolverReport*>(user)->trace.push_back(t);
  };
  gosma_report rep;
  check(gosma_solve(ctx.get(), &d, &c, &rep, cb, &r));
  r.best_pose.r = Eigen::Vector3d(rep.best_r[0], rep.best_r[1], rep.best_r[2]);
  r.best_pose.t = Eigen::Vector3d(rep.best_t[0], rep.best_t[1], rep.best_t[2]);
  r.best_value = rep.best_value;
  r.global_lower = rep.global_lower;
  r.gap = rep.gap;
  r.status = rep.status == GOSMA_STATUS_EPSILON_OPTIMAL ? SolverStatus::epsilon_optimal
             : rep.status == GOSMA_STATUS_TIME_LIMIT    ? SolverStatus::time_limit
                                                         : SolverStatus::queue_exhausted;
  r.epsilon_interpretation = "absolute gap on the objective (GPU backend)";
  r.stats.branches_expanded = rep.branches_expanded;
  r.stats.sma_invocations = rep.sma_invocations;
  r.stats.bound_evaluations = rep.bound_evaluations;
  r.stats.wall_time_seconds = rep.wall_time_seconds;
  return r;
}

}  // namespace smalign::gpu
