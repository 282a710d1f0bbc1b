// TEST INFRASTRUCTURE ONLY — flat C entry points over the UNMODIFIED reference
// C++ library (compiled in place from /root/reference/proj/core/src by
// oracle/Makefile against the Eigen/doctest shims). Loaded with ctypes by
// tests/ (golden generation, parity checks) and by bench.py's cpu_baseline /
// --impl reference leg only. Never linked into the product.
//
// Node records use the product ABI layout (include/gosma_capi.h gosma_node):
//   {rc[3], rhw, tc[3], thw[3], lower}  (11 doubles)
#include <chrono>
#include <cstdio>
#include <map>
#include <optional>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <limits>
#include <string>
#include <vector>

#include "smalign/bench.hpp"
#include "smalign/bounds.hpp"
#include "smalign/errors.hpp"
#include "smalign/mixtures.hpp"
#include "smalign/objective.hpp"
#include "smalign/se3.hpp"
#include "smalign/solver.hpp"
#include "smalign/sphere_stats.hpp"

using namespace smalign;

namespace {

thread_local std::string g_err;

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

BranchRegion node_to_branch(const double* n) {
  BranchRegion b;
  b.rotation.center = Eigen::Vector3d(n[0], n[1], n[2]);
  b.rotation.half_width = n[3];
  b.translation.center = Eigen::Vector3d(n[4], n[5], n[6]);
  b.translation.half_widths = Eigen::Vector3d(n[7], n[8], n[9]);
  b.lower = n[10];
  return b;
}

void branch_to_node(const BranchRegion& b, double* n) {
  n[0] = b.rotation.center.x();
  n[1] = b.rotation.center.y();
  n[2] = b.rotation.center.z();
  n[3] = b.rotation.half_width;
  n[4] = b.translation.center.x();
  n[5] = b.translation.center.y();
  n[6] = b.translation.center.z();
  n[7] = b.translation.half_widths.x();
  n[8] = b.translation.half_widths.y();
  n[9] = b.translation.half_widths.z();
  n[10] = b.lower;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// classes: for class c, n1[c] model comps and n2[c] image comps, laid out
// consecutively in mu (3 per comp), sigma2, phi1, dir (3 per comp), kappa2,
// phi2; class_weight[c]. Mirrors ObjectiveContext(SemanticMixturePair, zeta)
// (objective.cpp:109-121) — or (Gmm, Vmfmm, zeta) when n_classes == 1 and
// single_ctor != 0 (objective.cpp:103-107).
int ref_ctx_create(int n_classes, const int* n1, const int* n2, const double* class_weight,
                   const double* mu, const double* sigma2, const double* phi1,
                   const double* dir, const double* kappa2, const double* phi2, double zeta,
                   int single_ctor, void** out) {
  try {
    SemanticMixturePair pair;
    std::size_t o1 = 0, o2 = 0;
    for (int c = 0; c < n_classes; ++c) {
      SemanticClass cls;
      cls.id = "c" + std::to_string(c);
      cls.weight = class_weight[c];
      for (int i = 0; i < n1[c]; ++i, ++o1) {
        cls.gmm.components.emplace_back(
            Eigen::Vector3d(mu[3 * o1], mu[3 * o1 + 1], mu[3 * o1 + 2]), sigma2[o1], phi1[o1]);
      }
      for (int j = 0; j < n2[c]; ++j, ++o2) {
        cls.vmfmm.components.emplace_back(
            UnitVector3(Eigen::Vector3d(dir[3 * o2], dir[3 * o2 + 1], dir[3 * o2 + 2])),
            kappa2[o2], phi2[o2]);
      }
      pair.classes.push_back(std::move(cls));
    }
    ObjectiveContext* ctx;
    if (single_ctor && n_classes == 1) {
      ctx = new ObjectiveContext(pair.classes[0].gmm, pair.classes[0].vmfmm, zeta);
    } else {
      ctx = new ObjectiveContext(pair, zeta);
    }
    *out = ctx;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_ctx_blurred(void* ctx, double w, double ref_dist, void** out) {
  try {
    *out = new ObjectiveContext(
        ObjectiveContext::blurred(*static_cast<ObjectiveContext*>(ctx), w, ref_dist));
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

void ref_ctx_destroy(void* ctx) { delete static_cast<ObjectiveContext*>(ctx); }

double ref_ctx_self_energy(void* ctx) {
  return static_cast<ObjectiveContext*>(ctx)->image_self_energy();
}

// Derived per-class arrays (b = kappa * dir, log_z2), to pin the product's
// context construction. Writes n2_total * 3 into b and n2_total into log_z2.
void ref_ctx_image_cache(void* ctx, double* b, double* log_z2) {
  const auto& classes = static_cast<ObjectiveContext*>(ctx)->classes();
  std::size_t o = 0;
  for (const auto& cls : classes) {
    for (std::size_t j = 0; j < cls.kappa2.size(); ++j, ++o) {
      b[3 * o] = cls.b[j].x();
      b[3 * o + 1] = cls.b[j].y();
      b[3 * o + 2] = cls.b[j].z();
      log_z2[o] = cls.log_z2[j];
    }
  }
}

// evaluate_branch_batch (solver.cpp:260-292).
int ref_eval_bounds(void* ctx, const double* nodes, long n, int threads, double skip,
                    double* lower, double* upper) {
  try {
    std::vector<BranchRegion> branches(static_cast<std::size_t>(n));
    for (long k = 0; k < n; ++k) branches[k] = node_to_branch(nodes + 11 * k);
    const auto res = evaluate_branch_batch(*static_cast<ObjectiveContext*>(ctx), branches,
                                           threads, skip);
    for (long k = 0; k < n; ++k) {
      lower[k] = res[k].lower;
      upper[k] = res[k].upper;
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// objective_value (objective.cpp:227-235); +inf when infeasible.
double ref_objective_value(void* ctx, const double* r, const double* t) {
  Pose p;
  p.r = Eigen::Vector3d(r[0], r[1], r[2]);
  p.t = Eigen::Vector3d(t[0], t[1], t[2]);
  try {
    return objective_value(*static_cast<ObjectiveContext*>(ctx), p);
  } catch (const InfeasiblePoseError&) {
    return std::numeric_limits<double>::infinity();
  }
}

int ref_objective_gradient(void* ctx, const double* r, const double* t, double* g6) {
  Pose p;
  p.r = Eigen::Vector3d(r[0], r[1], r[2]);
  p.t = Eigen::Vector3d(t[0], t[1], t[2]);
  try {
    const auto g = objective_gradient(*static_cast<ObjectiveContext*>(ctx), p);
    for (int k = 0; k < 6; ++k) g6[k] = g[k];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 2);
  }
}

// upper_bound_pose (bounds.cpp:262-271): writes t*, returns 0 or 2 (none).
int ref_upper_bound_pose(void* ctx, const double* node, double* t_out) {
  const auto pose = upper_bound_pose(*static_cast<ObjectiveContext*>(ctx), node_to_branch(node));
  if (!pose) return 2;
  t_out[0] = pose->t.x();
  t_out[1] = pose->t.y();
  t_out[2] = pose->t.z();
  return 0;
}

// subdivide_adaptive (se3.cpp:107-147): 8 children, returns split-rotation
// flag (1/0), or -1 if not splittable.
int ref_subdivide(void* ctx, const double* node, double* children) {
  const BranchRegion b = node_to_branch(node);
  if (!is_splittable(b)) return -1;
  const auto& c = *static_cast<ObjectiveContext*>(ctx);
  const auto kids = subdivide_adaptive(b, c.all_means());
  for (int k = 0; k < 8; ++k) branch_to_node(kids[k], children + 11 * k);
  return kids[0].rotation.half_width < b.rotation.half_width ? 1 : 0;
}

double ref_psi_trans(const double* tc, const double* thw, const double* p) {
  TranslationCuboid box;
  box.center = Eigen::Vector3d(tc[0], tc[1], tc[2]);
  box.half_widths = Eigen::Vector3d(thw[0], thw[1], thw[2]);
  return psi_trans(box, Eigen::Vector3d(p[0], p[1], p[2]));
}

double ref_log_z(double k) { return log_z_eval(k); }

// local_refine (solver.cpp:164-258) over a domain {rot cube, boxes}.
int ref_local_refine(void* ctx, const double* r0, const double* t0, const double* rot_c,
                     double rot_hw, const double* boxes, int n_boxes, double* r_out,
                     double* t_out, double* value) {
  try {
    PoseDomain d;
    d.rotation.center = Eigen::Vector3d(rot_c[0], rot_c[1], rot_c[2]);
    d.rotation.half_width = rot_hw;
    for (int k = 0; k < n_boxes; ++k) {
      TranslationCuboid b;
      b.center = Eigen::Vector3d(boxes[6 * k], boxes[6 * k + 1], boxes[6 * k + 2]);
      b.half_widths = Eigen::Vector3d(boxes[6 * k + 3], boxes[6 * k + 4], boxes[6 * k + 5]);
      d.translations.push_back(b);
    }
    Pose s;
    s.r = Eigen::Vector3d(r0[0], r0[1], r0[2]);
    s.t = Eigen::Vector3d(t0[0], t0[1], t0[2]);
    const RefineResult rr = local_refine(*static_cast<ObjectiveContext*>(ctx), s, d);
    for (int k = 0; k < 3; ++k) {
      r_out[k] = rr.pose.r[k];
      t_out[k] = rr.pose.t[k];
    }
    *value = rr.value;
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// solve (solver.cpp:312-688). report: [best_value, global_lower, gap, status,
// branches_expanded, sma_invocations, bound_evaluations, wall_time, r[3], t[3]]
int ref_solve(void* ctx, const double* rot_c, double rot_hw, const double* boxes, int n_boxes,
              double epsilon, double zeta, int batch_size, double time_limit,
              long long max_evaluations, long long queue_capacity, int threads,
              double* report, long* n_trace, double* trace /* 8 per wave, may be null */,
              long trace_cap) {
  try {
    PoseDomain d;
    d.rotation.center = Eigen::Vector3d(rot_c[0], rot_c[1], rot_c[2]);
    d.rotation.half_width = rot_hw;
    for (int k = 0; k < n_boxes; ++k) {
      TranslationCuboid b;
      b.center = Eigen::Vector3d(boxes[6 * k], boxes[6 * k + 1], boxes[6 * k + 2]);
      b.half_widths = Eigen::Vector3d(boxes[6 * k + 3], boxes[6 * k + 4], boxes[6 * k + 5]);
      d.translations.push_back(b);
    }
    SolverConfig cfg;
    cfg.epsilon = epsilon;
    cfg.zeta = zeta;
    cfg.batch_size = batch_size;
    if (time_limit >= 0.0) cfg.time_limit = time_limit;
    if (max_evaluations >= 0) cfg.max_evaluations = static_cast<std::uint64_t>(max_evaluations);
    if (queue_capacity >= 0) cfg.queue_capacity = static_cast<std::size_t>(queue_capacity);
    cfg.threads = threads;
    const SolverReport r = solve(*static_cast<ObjectiveContext*>(ctx), d, cfg);
    report[0] = r.best_value;
    report[1] = r.global_lower;
    report[2] = r.gap;
    report[3] = static_cast<double>(static_cast<int>(r.status));
    report[4] = static_cast<double>(r.stats.branches_expanded);
    report[5] = static_cast<double>(r.stats.sma_invocations);
    report[6] = static_cast<double>(r.stats.bound_evaluations);
    report[7] = r.stats.wall_time_seconds;
    for (int k = 0; k < 3; ++k) {
      report[8 + k] = r.best_pose.r[k];
      report[11 + k] = r.best_pose.t[k];
    }
    *n_trace = static_cast<long>(r.trace.size());
    if (trace) {
      for (long w = 0; w < static_cast<long>(r.trace.size()) && w < trace_cap; ++w) {
        const TraceEntry& e = r.trace[w];
        double* o = trace + 8 * w;
        o[0] = static_cast<double>(e.wave);
        o[1] = static_cast<double>(e.bound_evaluations);
        o[2] = e.best_upper;
        o[3] = e.global_lower;
        o[4] = static_cast<double>(e.queue_size);
        o[5] = e.unexplored_volume_fraction;
        o[6] = e.pruned_volume_fraction;
        o[7] = e.resolved_volume_fraction;
      }
    }
    return 0;
  } catch (const InfeasiblePoseError& e) {
    return fail(e, 2);
  } catch (const std::invalid_argument& e) {
    return fail(e, 1);
  } catch (const std::exception& e) {
    return fail(e, 9);
  }
}

// generate_scene (bench.cpp:59-142) + pixel_to_bearing + build_semantic_mixtures
// (mixtures.cpp:269-362), unlabeled. Outputs the single class mixture. Sizes
// are returned in n1_out/n2_out; arrays must hold cap entries.
int ref_scene_mixtures(int n_inliers, double omega_3d, double omega_2d, double noise_px,
                       unsigned long long seed, double lambda_p, double lambda_f, int cap,
                       int* n1_out, int* n2_out, double* mu, double* sigma2, double* phi1,
                       double* dir, double* kappa2, double* phi2, double* true_r,
                       double* true_t, int* n_points, double* points, int* n_pixels,
                       double* pixels) {
  try {
    const SyntheticScene scene = generate_scene(n_inliers, omega_3d, omega_2d, noise_px, seed);
    LabeledPointSet pts;
    pts.points = scene.points_3d;
    LabeledBearingSet brg;
    for (const auto& px : scene.pixels_2d) brg.bearings.push_back(pixel_to_bearing(scene.intrinsics, px));
    const SemanticMixturePair pair = build_semantic_mixtures(pts, brg, lambda_p, lambda_f);
    const auto& cls = pair.classes.at(0);
    const int n1 = static_cast<int>(cls.gmm.components.size());
    const int n2 = static_cast<int>(cls.vmfmm.components.size());
    if (n1 > cap || n2 > cap) {
      g_err = "capacity";
      return 1;
    }
    *n1_out = n1;
    *n2_out = n2;
    for (int i = 0; i < n1; ++i) {
      const auto& g = cls.gmm.components[i];
      for (int k = 0; k < 3; ++k) mu[3 * i + k] = g.mean[k];
      sigma2[i] = g.variance;
      phi1[i] = g.weight;
    }
    for (int j = 0; j < n2; ++j) {
      const auto& v = cls.vmfmm.components[j];
      for (int k = 0; k < 3; ++k) dir[3 * j + k] = v.mean_direction.vec()[k];
      kappa2[j] = v.concentration;
      phi2[j] = v.weight;
    }
    for (int k = 0; k < 3; ++k) {
      true_r[k] = scene.true_pose.r[k];
      true_t[k] = scene.true_pose.t[k];
    }
    *n_points = static_cast<int>(scene.points_3d.size());
    *n_pixels = static_cast<int>(scene.pixels_2d.size());
    if (points) {
      for (std::size_t i = 0; i < scene.points_3d.size(); ++i)
        for (int k = 0; k < 3; ++k) points[3 * i + k] = scene.points_3d[i][k];
    }
    if (pixels) {
      for (std::size_t i = 0; i < scene.pixels_2d.size(); ++i) {
        pixels[2 * i] = scene.pixels_2d[i].x();
        pixels[2 * i + 1] = scene.pixels_2d[i].y();
      }
    }
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// torus_cover (se3.cpp:155-175): writes n boxes (6 doubles each) up to cap.
int ref_torus_cover(double major, double minor, double* boxes, int cap) {
  try {
    const PoseDomain d = torus_cover(major, minor);
    const int n = static_cast<int>(d.translations.size());
    for (int k = 0; k < n && k < cap; ++k) {
      for (int a = 0; a < 3; ++a) {
        boxes[6 * k + a] = d.translations[k].center[a];
        boxes[6 * k + 3 + a] = d.translations[k].half_widths[a];
      }
    }
    return n;
  } catch (const std::exception& e) {
    return -fail(e, 1);
  }
}

// dp_means / dp_vmf_means (mixtures.cpp:49-182) of the reference.
int ref_dp_means(const double* pts, long n, double lambda, int shuffle, unsigned long long seed,
                 int* assignment, double* centers, long cap, long* n_centers, int* iters) {
  try {
    std::vector<Eigen::Vector3d> p(n);
    for (long i = 0; i < n; ++i) p[i] = Eigen::Vector3d(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    const Clustering c = dp_means(p, lambda, shuffle ? std::optional<std::uint64_t>(seed)
                                                     : std::nullopt);
    *n_centers = static_cast<long>(c.centers.size());
    *iters = static_cast<int>(c.objective_history.size());
    for (long i = 0; i < n; ++i) assignment[i] = c.assignment[i];
    for (long k = 0; k < *n_centers && k < cap; ++k)
      for (int a = 0; a < 3; ++a) centers[3 * k + a] = c.centers[k][a];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

int ref_dp_vmf_means(const double* dirs, long n, double lambda, int shuffle,
                     unsigned long long seed, int* assignment, double* centers, long cap,
                     long* n_centers, int* iters) {
  try {
    std::vector<UnitVector3> b;
    for (long i = 0; i < n; ++i)
      b.emplace_back(Eigen::Vector3d(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]));
    const Clustering c = dp_vmf_means(b, lambda, shuffle ? std::optional<std::uint64_t>(seed)
                                                         : std::nullopt);
    *n_centers = static_cast<long>(c.centers.size());
    *iters = static_cast<int>(c.objective_history.size());
    for (long i = 0; i < n; ++i) assignment[i] = c.assignment[i];
    for (long k = 0; k < *n_centers && k < cap; ++k)
      for (int a = 0; a < 3; ++a) centers[3 * k + a] = c.centers[k][a];
    return 0;
  } catch (const std::exception& e) {
    return fail(e, 1);
  }
}

// build_semantic_mixtures (mixtures.cpp:269-362) with string labels (NULL:
// unlabeled) and optional class weights. Outputs are flattened over classes in
// result order; per class: n1, n2, weight, id (into ids, '\n'-separated), then
// warnings ('\n'-separated). Returns the class count (or -1 on error).
int ref_build_mixtures(const double* pts, const char* const* plab, long np, const double* dirs,
                       const char* const* blab, long nb, double lambda_p, double lambda_f,
                       const char* const* wlab, const double* w, long nw, int cap_classes,
                       int cap_comp, int* n1, int* n2, double* cls_w, double* mu, double* sigma2,
                       double* phi1, double* dir, double* kappa2, double* phi2, char* ids,
                       long ids_cap, char* warnings, long warn_cap) {
  try {
    LabeledPointSet ps;
    LabeledBearingSet bs;
    for (long i = 0; i < np; ++i)
      ps.points.emplace_back(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    for (long i = 0; i < nb; ++i)
      bs.bearings.emplace_back(Eigen::Vector3d(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2]));
    if (plab)
      for (long i = 0; i < np; ++i) ps.labels.emplace_back(plab[i]);
    if (blab)
      for (long i = 0; i < nb; ++i) bs.labels.emplace_back(blab[i]);
    std::optional<std::map<std::string, double>> cw;
    if (w) {
      cw.emplace();
      for (long k = 0; k < nw; ++k) (*cw)[wlab[k]] = w[k];
    }
    const SemanticMixturePair pair = build_semantic_mixtures(ps, bs, lambda_p, lambda_f, cw);
    const int nc = static_cast<int>(pair.classes.size());
    if (nc > cap_classes) {
      g_err = "capacity";
      return -1;
    }
    std::string idcat, wcat;
    long o1 = 0, o2 = 0;
    for (int c = 0; c < nc; ++c) {
      const auto& cls = pair.classes[c];
      n1[c] = static_cast<int>(cls.gmm.components.size());
      n2[c] = static_cast<int>(cls.vmfmm.components.size());
      cls_w[c] = cls.weight;
      if (o1 + n1[c] > cap_comp || o2 + n2[c] > cap_comp) {
        g_err = "capacity";
        return -1;
      }
      for (const auto& g : cls.gmm.components) {
        for (int a = 0; a < 3; ++a) mu[3 * o1 + a] = g.mean[a];
        sigma2[o1] = g.variance;
        phi1[o1] = g.weight;
        ++o1;
      }
      for (const auto& v : cls.vmfmm.components) {
        for (int a = 0; a < 3; ++a) dir[3 * o2 + a] = v.mean_direction.vec()[a];
        kappa2[o2] = v.concentration;
        phi2[o2] = v.weight;
        ++o2;
      }
      idcat += cls.id + "\n";
    }
    for (const auto& s : pair.warnings) wcat += s + "\n";
    std::snprintf(ids, ids_cap, "%s", idcat.c_str());
    std::snprintf(warnings, warn_cap, "%s", wcat.c_str());
    return nc;
  } catch (const std::exception& e) {
    fail(e, 1);
    return -1;
  }
}

}  // extern "C"
