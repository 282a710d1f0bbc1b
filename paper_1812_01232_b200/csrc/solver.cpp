// gosma_solve: globally-optimal alignment by branch-and-bound with the
// frontier resident on the GPU (frontier.cu) and every bound evaluated by the
// fused kernel (bounds_kernel.cu). Follows solve() (core/src/solver.cpp:312-688):
// feasible roots (339-368), wave 0 + discovery dive (449-621), the certified
// lower bound max(prev, min(d*, frontier min, resolved floor)) (626-627), the
// stop rules (629-645), routing (396-405), capacity folding (433-447) and the
// volume ledger (597-608). Differences by design: a wave expands the W best
// live nodes (not batch_size/8), and a wave's incumbent update happens once,
// after the whole wave is bounded (the d* used to route is then the wave's
// best, which only prunes more, soundly).
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <limits>
#include <mutex>
#include <thread>
#include <vector>

#include "capi_internal.hpp"
#include "frontier.hpp"
#include "sma.hpp"

using namespace gosma;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr double kFloor = 1e-9;  // is_splittable floor (se3.cpp:102-105)

Domain make_domain(const gosma_domain* d) {
  Domain dom;
  dom.rot_center = Vec3(d->rot_center[0], d->rot_center[1], d->rot_center[2]);
  dom.rot_hw = d->rot_half_width;
  for (int b = 0; b < d->n_boxes; ++b) {
    const double* x = d->boxes + 6 * b;
    dom.boxes.push_back({Vec3(x[0], x[1], x[2]), Vec3(x[3], x[4], x[5])});
  }
  return dom;
}

double volume_of(const gosma_node& n) {
  const double w = 2.0 * n.rhw;
  return w * w * w * (2.0 * n.thw[0]) * (2.0 * n.thw[1]) * (2.0 * n.thw[2]);
}

bool splittable(const gosma_node& n) {
  return n.rhw > kFloor || std::max(std::max(n.thw[0], n.thw[1]), n.thw[2]) > kFloor;
}

bool feasible_box(const HostModel& m, const Vec3& c, const Vec3& h) {
  for (const Vec3& mu : m.all_means)
    if (point_box_hi(mu, c, h) < m.zeta) return false;
  return true;
}

// ObjectiveContext::blurred on the host model only (objective.cpp:70-101):
// the SMA ladder needs the value/gradient, not device tables.
HostModel blurred_model(const HostModel& src, double w, double dist) {
  HostModel hm = src;
  const double var_add = (w * dist) * (w * dist);
  for (HostClass& c : hm.classes) {
    for (double& s2 : c.sigma2) s2 += var_add;
    for (int j = 0; j < c.n2(); ++j) {
      const Vec3 dir = Vec3(c.b[3 * j], c.b[3 * j + 1], c.b[3 * j + 2]) / c.kappa2[j];
      const double k = c.kappa2[j] / (1.0 + c.kappa2[j] * w * w);
      c.kappa2[j] = k;
      for (int a = 0; a < 3; ++a) c.b[3 * j + a] = k * dir[a];
      c.log_z2[j] = log_z_eval(k);
    }
  }
  return hm;
}

struct Incumbent {
  double value = kInf;
  Vec3 r, t;
  unsigned long long sma = 0;
};

// process_wave's incumbent update (solver.cpp:409-431) for one improving
// branch: FP64 objective at the feasible centre, then SMA from there.
void improve(const HostModel& m, const Domain& dom, const gosma_node& b, Incumbent* inc) {
  Vec3 t;
  if (!feasible_center(m, Vec3(b.tc[0], b.tc[1], b.tc[2]), Vec3(b.thw[0], b.thw[1], b.thw[2]),
                       &t))
    return;
  const Vec3 r(b.rc[0], b.rc[1], b.rc[2]);
  const double f = objective_value(m, r, t);
  if (!(f < inc->value)) return;
  inc->value = f;
  inc->r = r;
  inc->t = t;
  const RefineResult rr = local_refine(m, r, t, dom);
  ++inc->sma;
  if (rr.value < inc->value) {
    inc->value = rr.value;
    inc->r = rr.r;
    inc->t = rr.t;
  }
}

int eval_host(gosma_ctx* ctx, const std::vector<gosma_node>& nodes, double skip,
              std::vector<double>* lo, std::vector<double>* up, std::vector<int8_t>* sp) {
  lo->resize(nodes.size());
  up->resize(nodes.size());
  sp->resize(nodes.size());
  if (nodes.empty()) return GOSMA_OK;
  return gosma_eval_bounds(ctx, nodes.data(), nodes.size(), skip, lo->data(), up->data(),
                           sp->data());
}

gosma_node child_of(const gosma_node& p, int split_rot, int c) {
  // subdivide_adaptive child order (se3.cpp:124-145): sx, sy, sz in {-1, +1}
  const int sx = (c & 4) ? 1 : -1, sy = (c & 2) ? 1 : -1, sz = (c & 1) ? 1 : -1;
  gosma_node k = p;
  if (split_rot == 1) {
    const double h = 0.5 * p.rhw;
    k.rc[0] = p.rc[0] + h * sx;
    k.rc[1] = p.rc[1] + h * sy;
    k.rc[2] = p.rc[2] + h * sz;
    k.rhw = h;
  } else {
    for (int a = 0; a < 3; ++a) {
      const double h = 0.5 * p.thw[a];
      k.tc[a] = p.tc[a] + h * (a == 0 ? sx : (a == 1 ? sy : sz));
      k.thw[a] = h;
    }
  }
  return k;
}

// Discovery dive (solver.cpp:449-595): beam search on a blurred copy of the
// problem (bounds on the GPU), then the SMA annealing ladder per sector on
// host threads. Improves the incumbent only.
int discovery_dive(gosma_ctx* ctx, const Domain& dom, const std::vector<gosma_node>& roots,
                   const gosma_config& cfg, Incumbent* inc, unsigned long long* evals,
                   double t0_unused) {
  (void)t0_unused;
  const HostModel& m = ctx->model;
  const unsigned long long cap = 100000;
  const unsigned long long budget =
      cfg.max_evaluations >= 0 ? std::min<unsigned long long>(cap, cfg.max_evaluations / 4) : cap;
  if (budget < 8 * roots.size()) return GOSMA_OK;
  const size_t kQuota = 12;
  const int kMaxIt = 40;
  const double kCoarse = 0.1;
  Vec3 centroid;
  for (const Vec3& mu : m.all_means) centroid = centroid + mu;
  centroid = centroid / static_cast<double>(m.all_means.size());
  double dbar = 0.0;
  for (const Box& b : dom.boxes) dbar += (b.c - centroid).norm();
  dbar /= static_cast<double>(dom.boxes.size());
  gosma_ctx* coarse = nullptr;
  int rc = gosma_ctx_blurred(ctx, kCoarse, dbar, &coarse);
  if (rc != GOSMA_OK) return rc;
  struct Cand {
    double value = kInf;
    gosma_node b{};
  };
  std::vector<Cand> best(roots.size());
  auto offer = [&](double v, const gosma_node& b, size_t s) {
    if (std::isfinite(v) && v < best[s].value) best[s] = {v, b};
  };
  struct Beam {
    gosma_node b;
    int8_t split;
    unsigned sector;
  };
  std::vector<Beam> beam;
  std::vector<double> lo, up;
  std::vector<int8_t> sp;
  unsigned long long used = 0;
  rc = eval_host(coarse, roots, kInf, &lo, &up, &sp);
  if (rc != GOSMA_OK) {
    gosma_ctx_destroy(coarse);
    return rc;
  }
  used += roots.size();
  for (size_t i = 0; i < roots.size(); ++i) {
    offer(up[i], roots[i], i);
    if (splittable(roots[i])) {
      Beam e{roots[i], sp[i], static_cast<unsigned>(i)};
      e.b.lower = lo[i];
      beam.push_back(e);
    }
  }
  std::vector<gosma_node> kids;
  std::vector<unsigned> ksec;
  for (int it = 0; it < kMaxIt && !beam.empty() && used + beam.size() * 8 <= budget; ++it) {
    kids.clear();
    ksec.clear();
    for (const Beam& e : beam) {
      for (int c = 0; c < 8; ++c) {
        gosma_node k = child_of(e.b, e.split, c);
        kids.push_back(k);
        ksec.push_back(e.sector);
      }
    }
    double skip = -kInf;  // worst sector candidate (kInf until all seeded)
    for (const Cand& c : best) skip = std::max(skip, c.value);
    rc = eval_host(coarse, kids, skip, &lo, &up, &sp);
    if (rc != GOSMA_OK) break;
    used += kids.size();
    beam.clear();
    for (size_t i = 0; i < kids.size(); ++i) {
      offer(up[i], kids[i], ksec[i]);
      if (splittable(kids[i])) {
        Beam e{kids[i], sp[i], ksec[i]};
        e.b.lower = lo[i];
        beam.push_back(e);
      }
    }
    std::stable_sort(beam.begin(), beam.end(), [](const Beam& a, const Beam& b) {
      if (a.sector != b.sector) return a.sector < b.sector;
      return a.b.lower < b.b.lower;
    });
    size_t out = 0, run = 0;
    for (size_t i = 0; i < beam.size(); ++i) {
      run = (i > 0 && beam[i].sector == beam[i - 1].sector) ? run + 1 : 0;
      if (run < kQuota) beam[out++] = beam[i];
    }
    beam.resize(out);
  }
  *evals += used;
  // annealing ladder per sector: coarse -> 0.03 -> 0.01 -> exact
  const HostModel hc = blurred_model(m, kCoarse, dbar);
  const HostModel h3 = blurred_model(m, 0.03, dbar);
  const HostModel h1 = blurred_model(m, 0.01, dbar);
  std::vector<RefineResult> res(best.size());
  std::vector<char> ok(best.size(), 0);
  std::atomic<size_t> next{0};
  unsigned nthreads = cfg.threads > 0 ? cfg.threads : std::max(1u, std::thread::hardware_concurrency());
  nthreads = std::min<unsigned>(nthreads, static_cast<unsigned>(best.size()));
  auto work = [&] {
    for (;;) {
      const size_t s = next.fetch_add(1);
      if (s >= best.size()) return;
      if (!std::isfinite(best[s].value)) continue;
      Vec3 t;
      const gosma_node& b = best[s].b;
      if (!feasible_center(hc, Vec3(b.tc[0], b.tc[1], b.tc[2]), Vec3(b.thw[0], b.thw[1], b.thw[2]),
                           &t))
        continue;
      RefineResult r = local_refine(hc, Vec3(b.rc[0], b.rc[1], b.rc[2]), t, dom);
      r = local_refine(h3, r.r, r.t, dom);
      r = local_refine(h1, r.r, r.t, dom);
      res[s] = local_refine(m, r.r, r.t, dom);
      ok[s] = 1;
    }
  };
  std::vector<std::thread> pool;
  for (unsigned k = 0; k + 1 < nthreads; ++k) pool.emplace_back(work);
  work();
  for (auto& th : pool) th.join();
  for (size_t s = 0; s < best.size(); ++s) {
    if (!ok[s]) continue;
    inc->sma += 4;
    if (res[s].value < inc->value) {
      inc->value = res[s].value;
      inc->r = res[s].r;
      inc->t = res[s].t;
    }
  }
  gosma_ctx_destroy(coarse);
  return GOSMA_OK;
}

}  // namespace

extern "C" {

int gosma_local_refine(const gosma_ctx* ctx, const double* r0, const double* t0,
                       const gosma_domain* domain, double* r_out, double* t_out, double* value) {
  if (!ctx || !r0 || !t0 || !domain || !r_out || !t_out || !value)
    return set_error(GOSMA_EINVAL, "null argument");
  const Domain dom = make_domain(domain);
  const RefineResult rr =
      local_refine(ctx->model, Vec3(r0[0], r0[1], r0[2]), Vec3(t0[0], t0[1], t0[2]), dom);
  for (int k = 0; k < 3; ++k) {
    r_out[k] = rr.r[k];
    t_out[k] = rr.t[k];
  }
  *value = rr.value;
  return GOSMA_OK;
}

int gosma_solve(gosma_ctx* ctx, const gosma_domain* domain, const gosma_config* config,
                gosma_report* report, gosma_trace_cb trace, void* user) {
  using Clock = std::chrono::steady_clock;
  const auto t_start = Clock::now();
  auto elapsed = [&] { return std::chrono::duration<double>(Clock::now() - t_start).count(); };
  if (!ctx || !domain || !config || !report) return set_error(GOSMA_EINVAL, "null argument");
  const gosma_config& cfg = *config;
  // solver.cpp:320-329
  if (!(cfg.epsilon > 0.0)) return set_error(GOSMA_EINVAL, "solve: epsilon must be > 0");
  if (cfg.batch_size < 1) return set_error(GOSMA_EINVAL, "solve: batch_size must be >= 1");
  if (cfg.zeta != ctx->model.zeta)
    return set_error(GOSMA_EINVAL, "solve: config.zeta differs from the context's standoff radius");
  if (domain->n_boxes < 1 || !domain->boxes)
    return set_error(GOSMA_EINVAL, "solve: empty translation domain");
  *report = gosma_report{};
  const HostModel& m = ctx->model;
  const Domain dom = make_domain(domain);
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;

  // Roots and the measure (solver.cpp:339-368).
  double total_volume = 0.0;
  for (const Box& b : dom.boxes) {
    gosma_node n{};
    n.rhw = dom.rot_hw;
    for (int a = 0; a < 3; ++a) n.thw[a] = b.h[a];
    total_volume += volume_of(n);
  }
  const bool unit_measure = !(total_volume > 0.0);
  if (unit_measure) total_volume = static_cast<double>(dom.boxes.size());
  double pruned_volume = 0.0, resolved_volume = 0.0, queue_volume = 0.0;
  double floor_lower = kInf;
  std::vector<gosma_node> roots;
  std::vector<double> root_vol;
  for (const Box& b : dom.boxes) {
    gosma_node n{};
    for (int a = 0; a < 3; ++a) {
      n.rc[a] = dom.rot_center[a];
      n.tc[a] = b.c[a];
      n.thw[a] = b.h[a];
    }
    n.rhw = dom.rot_hw;
    n.lower = -kInf;
    const double v = unit_measure ? 1.0 : volume_of(n);
    if (feasible_box(m, b.c, b.h)) {
      roots.push_back(n);
      root_vol.push_back(v);
    } else {
      pruned_volume += v;
    }
  }
  if (roots.empty())
    return set_error(GOSMA_EINFEASIBLE, "solve: no feasible camera center in the domain");

  Incumbent inc;
  unsigned long long evals = 0, expanded = 0, wave = 0;
  double certified = -kInf;
  auto emit = [&](unsigned long long w, size_t qsize) {
    if (trace)
      trace(user, w, evals, inc.value, certified, qsize, queue_volume / total_volume,
            pruned_volume / total_volume, resolved_volume / total_volume);
  };

  // Wave 0: the roots (solver.cpp:611-621).
  std::vector<double> lo, up;
  std::vector<int8_t> sp;
  int rc = eval_host(ctx, roots, kInf, &lo, &up, &sp);
  if (rc != GOSMA_OK) return rc;
  evals += roots.size();
  if (cfg.discovery_dive) {
    rc = discovery_dive(ctx, dom, roots, cfg, &inc, &evals, 0.0);
    if (rc != GOSMA_OK) return rc;
  }
  for (size_t i = 0; i < roots.size(); ++i) {
    if (up[i] < inc.value) improve(m, dom, roots[i], &inc);
  }
  Frontier F;
  // Wave size: enough children to keep the bound kernel busy for a few ms
  // (pair terms per wave ~1e9), but never more than the caller asks for.
  size_t pairs = 0;
  for (const HostClass& c : m.classes)
    pairs += static_cast<size_t>(c.n1()) * c.n2() + static_cast<size_t>(c.n1()) * (c.n1() - 1) / 2;
  size_t wave_nodes = cfg.wave_nodes > 0
                          ? static_cast<size_t>(cfg.wave_nodes)
                          : std::min<size_t>(std::max<size_t>(120000000 / std::max<size_t>(pairs, 1), 1024),
                                             1u << 19);
  cudaError_t e = F.reserve(std::max<size_t>(8 * wave_nodes, roots.size() * 2), wave_nodes);
  if (e != cudaSuccess) return cuda_error(e, "frontier reserve");
  struct Guard {
    Frontier* f;
    ~Guard() { f->release(); }
  } guard{&F};
  {
    std::vector<gosma_node> keep;
    std::vector<int8_t> ks;
    std::vector<double> kv;
    for (size_t i = 0; i < roots.size(); ++i) {
      gosma_node b = roots[i];
      b.lower = lo[i];
      if (!(b.lower < inc.value)) {
        pruned_volume += root_vol[i];
      } else if (!splittable(b)) {
        // resolved: FP64 bound, so zero-size domains certify exactly
        const double l64 = lower_bound_fp64(m, Vec3(b.rc[0], b.rc[1], b.rc[2]), b.rhw,
                                            Vec3(b.tc[0], b.tc[1], b.tc[2]),
                                            Vec3(b.thw[0], b.thw[1], b.thw[2]), -kInf);
        resolved_volume += root_vol[i];
        floor_lower = std::min(floor_lower, std::max(l64, b.lower));
      } else {
        keep.push_back(b);
        ks.push_back(sp[i]);
        kv.push_back(root_vol[i]);
      }
    }
    if (!keep.empty() &&
        (e = F.upload(keep.data(), ks.data(), kv.data(), keep.size(), s)) != cudaSuccess)
      return cuda_error(e, "frontier upload");
  }

  // Device memory budget for the pool: beyond it the worst nodes are folded
  // into the resolved set (sound; the reference's queue_capacity mechanism).
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t per_node = sizeof(gosma_node) + 1 + 8 + 8;
  const size_t mem_cap = std::max<size_t>(free_b / 4 / per_node, 16 * wave_nodes);
  const size_t qcap = cfg.queue_capacity >= 0
                          ? std::min<size_t>(static_cast<size_t>(cfg.queue_capacity), mem_cap)
                          : mem_cap;
  int status = GOSMA_STATUS_QUEUE_EXHAUSTED;
  for (;;) {
    // capacity folding (solver.cpp:433-447); the memory budget folds to 3/4
    if (F.live_upper_bound() > qcap ||
        F.size + 8 * wave_nodes > (cfg.queue_capacity >= 0 ? ~size_t{0} : mem_cap)) {
      const size_t target = cfg.queue_capacity >= 0 && static_cast<size_t>(cfg.queue_capacity) <= mem_cap
                                ? static_cast<size_t>(cfg.queue_capacity)
                                : mem_cap * 3 / 4 - 8 * wave_nodes;
      double fv = 0.0, fmin = kInf;
      if ((e = F.fold_to(target, s, &fv, &fmin)) != cudaSuccess)
        return cuda_error(e, "fold");
      resolved_volume += fv;
      floor_lower = std::min(floor_lower, fmin);
    }
    unsigned long long kmin = kHoleKey;
    if ((e = F.min_key(s, &kmin)) != cudaSuccess) return cuda_error(e, "frontier min");
    const bool empty = (kmin == kHoleKey);
    const double front_min = empty ? kInf : key_to_double(kmin);
    queue_volume = std::max(0.0, total_volume - pruned_volume - resolved_volume);
    certified = std::max(certified, std::min(std::min(inc.value, front_min), floor_lower));
    emit(wave, F.live_upper_bound());
    if (inc.value - certified <= cfg.epsilon) {
      status = GOSMA_STATUS_EPSILON_OPTIMAL;
      break;
    }
    if (empty) {
      status = GOSMA_STATUS_QUEUE_EXHAUSTED;
      break;
    }
    if (cfg.time_limit >= 0.0 && elapsed() >= cfg.time_limit) {
      status = GOSMA_STATUS_TIME_LIMIT;
      break;
    }
    if (cfg.max_evaluations >= 0 && evals >= static_cast<unsigned long long>(cfg.max_evaluations)) {
      status = GOSMA_STATUS_TIME_LIMIT;
      break;
    }
    // Expand only nodes that can still matter: lower < d* - eps (the stop rule
    // never needs the others expanded).
    const double limit = inc.value - cfg.epsilon;
    size_t want = wave_nodes;
    if (cfg.max_evaluations >= 0) {  // keep within the evaluation budget
      const unsigned long long left =
          static_cast<unsigned long long>(cfg.max_evaluations) > evals
              ? static_cast<unsigned long long>(cfg.max_evaluations) - evals
              : 0;
      want = std::min<size_t>(want, std::max<unsigned long long>(1, (left + 7) / 8));
    }
    size_t n_sel = 0;
    if ((e = F.select_smallest(want, host_order_key(limit), s, &n_sel)) != cudaSuccess)
      return cuda_error(e, "select");
    if (n_sel == 0) {
      // Nothing below d* - eps, yet the gap is open (a resolved floor holds the
      // certified bound down): keep refining the live nodes, as the
      // reference's heap would, until the queue runs dry.
      if ((e = F.select_smallest(want, host_order_key(inc.value), s, &n_sel)) != cudaSuccess)
        return cuda_error(e, "select");
      if (n_sel == 0) {  // only stale nodes remain
        double dropped = 0.0;
        if ((e = F.compact(host_order_key(inc.value), s, &dropped)) != cudaSuccess)
          return cuda_error(e, "compact");
        pruned_volume += dropped;
        continue;
      }
    }
    const size_t n_kids = n_sel * 8;
    if ((e = F.expand_selected(n_sel, s)) != cudaSuccess) return cuda_error(e, "expand");
    EvalArgs a;
    a.nodes = reinterpret_cast<const double*>(F.kids);
    a.n = static_cast<long long>(n_kids);
    a.skip_upper_at = inc.value;
    a.lower = F.kid_lower;
    a.upper = F.kid_upper;
    a.split_rot = F.kid_split;
    a.work = static_cast<unsigned int*>(ctx->d_work);
    if ((e = launch_eval_bounds(ctx->dev, a, ctx->sm_count, s)) != cudaSuccess)
      return cuda_error(e, "eval children");
    evals += n_kids;
    expanded += n_sel;
    int bi = -1;
    double bu = kInf;
    if ((e = F.best_child(n_kids, s, &bi, &bu)) != cudaSuccess) return cuda_error(e, "argmin");
    if (bi >= 0 && bu < inc.value) {
      gosma_node b;
      cudaMemcpy(&b, F.kids + bi, sizeof(gosma_node), cudaMemcpyDeviceToHost);
      improve(m, dom, b, &inc);
    }
    RouteStats rs;
    if ((e = F.route_append(n_kids, inc.value, s, &rs)) != cudaSuccess)
      return cuda_error(e, "route");
    pruned_volume += rs.pruned_volume;
    resolved_volume += rs.resolved_volume;
    if (rs.floor_key != ~0ull) floor_lower = std::min(floor_lower, key_to_double(rs.floor_key));
    // amortised compaction: drop holes and stale nodes (lower >= d*,
    // solver.cpp:660-663) once they fill half the pool
    if (F.holes * 2 > F.size) {
      double dropped = 0.0;
      if ((e = F.compact(host_order_key(inc.value), s, &dropped)) != cudaSuccess)
        return cuda_error(e, "compact");
      pruned_volume += dropped;
    }
    ++wave;
  }
  report->best_value = inc.value;
  for (int k = 0; k < 3; ++k) {
    report->best_r[k] = inc.r[k];
    report->best_t[k] = inc.t[k];
  }
  report->global_lower = certified;
  report->gap = inc.value - certified;
  report->status = status;
  report->branches_expanded = expanded;
  report->sma_invocations = inc.sma;
  report->bound_evaluations = evals;
  report->wall_time_seconds = elapsed();
  report->waves = wave;
  return status == GOSMA_STATUS_TIME_LIMIT ? GOSMA_EBUDGET : GOSMA_OK;
}

int gosma_eval_bounds_cached_device(gosma_ctx*, const gosma_node*, size_t, const int32_t*,
                                    const double*, size_t, double, double*, double*, int8_t*,
                                    void*) {
  return set_error(GOSMA_EINVAL, "gosma_eval_bounds_cached_device: not built yet");
}

}  // extern "C"
