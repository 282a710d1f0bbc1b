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
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <cmath>
#include <limits>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "capi_internal.hpp"
#include "frontier.hpp"
#include "objective_device.hpp"
#include "dive.hpp"
#include "sma.hpp"

using namespace gosma;

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();
constexpr size_t kDfsWaveFactor = 4;
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

// Pair terms of a model (the refiner's cost per evaluation).
size_t model_pairs(const HostModel& m) {
  size_t p = 0;
  for (const HostClass& c : m.classes)
    p += static_cast<size_t>(c.n1()) * c.n2() + static_cast<size_t>(c.n1()) * (c.n1() - 1) / 2;
  return p;
}

// Refinements run their objective on the GPU (batched FP64 kernel K6) once a
// host evaluation gets expensive; GOSMA_SMA=host|gpu overrides.
bool gpu_sma(const HostModel& m) {
  static const int forced = [] {
    const char* e = std::getenv("GOSMA_SMA");
    if (!e) return -1;
    return std::string(e) == "gpu" ? 1 : (std::string(e) == "host" ? 0 : -1);
  }();
  if (forced >= 0) return forced == 1;
  return model_pairs(m) >= 500;  // measured dive ladders: 20x16 GPU 0.15 s vs host 0.17 s, 12x12 0.70 vs 0.09
}

// Runs refinement jobs on the GPU (refine_kernel: one CTA per start runs the
// whole L-BFGS ladder, no host round trips per evaluation).
cudaError_t refine_device(DeviceObjective* dev, const Domain& dom,
                          const std::vector<RefineJob>& jobs, std::vector<RefineOut>* out) {
  std::vector<double> boxes;
  for (const Box& b : dom.boxes)
    for (const Vec3* v : {&b.c, &b.h})
      for (int a = 0; a < 3; ++a) boxes.push_back((*v)[a]);
  const double rc[3] = {dom.rot_center[0], dom.rot_center[1], dom.rot_center[2]};
  return dev->refine(jobs, rc, dom.rot_hw, boxes, out);
}

// process_wave's incumbent update (solver.cpp:409-431) for one improving
// branch: FP64 objective at the feasible centre, then SMA from there (on the
// GPU when dev is set; the incumbent value is always the host FP64 d*).
int improve(const HostModel& m, const Domain& dom, const gosma_node& b, Incumbent* inc,
            DeviceObjective* dev = nullptr) {
  Vec3 t;
  if (!feasible_center(m, Vec3(b.tc[0], b.tc[1], b.tc[2]), Vec3(b.thw[0], b.thw[1], b.thw[2]),
                       &t))
    return GOSMA_OK;
  const Vec3 r(b.rc[0], b.rc[1], b.rc[2]);
  const double f = objective_value(m, r, t);
  if (!(f < inc->value)) return GOSMA_OK;
  inc->value = f;
  inc->r = r;
  inc->t = t;
  RefineResult rr;
  std::vector<RefineOut> out;
  if (dev) {
    const cudaError_t e =
        refine_device(dev, dom, {RefineJob{{r[0], r[1], r[2], t[0], t[1], t[2]}, 1, {0}}}, &out);
    if (e != cudaSuccess) return cuda_error(e, "refine kernel");
    rr.r = Vec3(out[0].x[0], out[0].x[1], out[0].x[2]);
    rr.t = Vec3(out[0].x[3], out[0].x[4], out[0].x[5]);
    rr.value = objective_value(m, rr.r, rr.t);
  } else {
    rr = local_refine(m, r, t, dom);
  }
  ++inc->sma;
  if (rr.value < inc->value) {
    inc->value = rr.value;
    inc->r = rr.r;
    inc->t = rr.t;
  }
  return GOSMA_OK;
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
  const auto t_dive = std::chrono::steady_clock::now();
  double t_eval = 0.0;
  int beam_its = 0;
  // the blurred context is cached on ctx (same width and reference distance
  // on the next solve of this problem); the dive holds its lock throughout
  std::lock_guard<std::mutex> dive_lock(ctx->dive_mu);
  int rc = GOSMA_OK;
  if (!ctx->dive_ctx || ctx->dive_w != kCoarse || ctx->dive_dist != dbar ||
      ctx->dive_ctx->lb_margin != ctx->lb_margin ||
      ctx->dive_ctx->dev.lb_err_scale != ctx->dev.lb_err_scale) {
    gosma_ctx_destroy(ctx->dive_ctx);
    ctx->dive_ctx = nullptr;
    if ((rc = gosma_ctx_blurred(ctx, kCoarse, dbar, &ctx->dive_ctx)) != GOSMA_OK) return rc;
    ctx->dive_w = kCoarse;
    ctx->dive_dist = dbar;
  }
  gosma_ctx* const coarse = ctx->dive_ctx;
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
  if (rc != GOSMA_OK) return rc;
  used += roots.size();
  for (size_t i = 0; i < roots.size(); ++i) {
    offer(up[i], roots[i], i);
    if (splittable(roots[i])) {
      Beam e{roots[i], sp[i], static_cast<unsigned>(i)};
      e.b.lower = lo[i];
      beam.push_back(e);
    }
  }
  // the beam loop runs on the device (dive.cu: no host round trip per
  // iteration); GOSMA_DIVE=host runs the same loop here (A/B, tests)
  static const bool device_beam = [] {
    const char* e = std::getenv("GOSMA_DIVE");
    return !(e && std::string(e) == "host");
  }();
  if (device_beam) {
    std::vector<DiveEntry> db;
    db.reserve(beam.size());
    for (const Beam& e : beam) db.push_back(DiveEntry{e.b, e.split, e.sector});
    std::vector<DiveBest> b0(best.size());
    for (size_t k = 0; k < best.size(); ++k) b0[k] = DiveBest{best[k].value, best[k].b};
    DiveBeamResult res;
    rc = dive_beam_device(coarse, db, b0, used, budget, kMaxIt, static_cast<int>(kQuota), kFloor,
                          &res);
    if (rc != GOSMA_OK) return rc;
    for (size_t k = 0; k < best.size(); ++k) best[k] = Cand{res.best[k].value, res.best[k].node};
    used = res.used;
    beam.clear();
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
    const auto te = std::chrono::steady_clock::now();
    rc = eval_host(coarse, kids, skip, &lo, &up, &sp);
    t_eval += std::chrono::duration<double>(std::chrono::steady_clock::now() - te).count();
    ++beam_its;
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
  const auto t_beam = std::chrono::steady_clock::now();
  if (std::getenv("GOSMA_PROFILE"))
    std::fprintf(stderr,
                 "[gosma profile] dive: beam %.3fs (%s: %d host iterations, bounds %.3fs, %llu "
                 "evals)\n",
                 std::chrono::duration<double>(t_beam - t_dive).count(),
                 device_beam ? "device" : "host", beam_its, t_eval, used);
  // annealing ladder per sector: coarse -> 0.03 -> 0.01 -> exact
  const HostModel hc = blurred_model(m, kCoarse, dbar);
  const HostModel h3 = blurred_model(m, 0.03, dbar);
  const HostModel h1 = blurred_model(m, 0.01, dbar);
  std::vector<RefineResult> res(best.size());
  std::vector<char> ok(best.size(), 0);
  // start of each sector's ladder: the coarse model's feasible centre
  std::vector<RefineJob> jobs(best.size());
  for (size_t s = 0; s < best.size(); ++s) {
    if (!std::isfinite(best[s].value)) continue;
    const gosma_node& b = best[s].b;
    Vec3 t;
    if (!feasible_center(hc, Vec3(b.tc[0], b.tc[1], b.tc[2]), Vec3(b.thw[0], b.thw[1], b.thw[2]),
                         &t))
      continue;
    jobs[s] = RefineJob{{b.rc[0], b.rc[1], b.rc[2], t[0], t[1], t[2]}, 4, {0, 1, 2, 3}};
    ok[s] = 1;
  }
  std::unique_ptr<DeviceObjective> dobj;
  if (gpu_sma(m)) {
    dobj = std::make_unique<DeviceObjective>(ctx->device,
                                             std::vector<const HostModel*>{&hc, &h3, &h1, &m});
    if (!dobj->ok()) dobj.reset();
  }
  std::vector<RefineOut> out;
  if (dobj) {
    std::vector<RefineJob> run;
    for (size_t s = 0; s < best.size(); ++s)
      if (ok[s]) run.push_back(jobs[s]);
    const cudaError_t e = refine_device(dobj.get(), dom, run, &out);
    if (e != cudaSuccess) return cuda_error(e, "refine kernel");
  }
  if (dobj) {
    // incumbents are host FP64 values
    size_t k = 0;
    for (size_t s = 0; s < best.size(); ++s) {
      if (!ok[s]) continue;
      RefineResult& r = res[s];
      r.r = Vec3(out[k].x[0], out[k].x[1], out[k].x[2]);
      r.t = Vec3(out[k].x[3], out[k].x[4], out[k].x[5]);
      r.value = objective_value(m, r.r, r.t);
      ++k;
    }
  } else {
    const HostModel* stage[4] = {&hc, &h3, &h1, &m};
    std::atomic<size_t> next{0};
    unsigned nthreads =
        cfg.threads > 0 ? cfg.threads : std::max(1u, std::thread::hardware_concurrency());
    nthreads = std::min<unsigned>(nthreads, static_cast<unsigned>(best.size()));
    auto work = [&] {
      for (;;) {
        const size_t s = next.fetch_add(1);
        if (s >= best.size()) return;
        if (!ok[s]) continue;
        RefineResult r;
        r.r = Vec3(jobs[s].x[0], jobs[s].x[1], jobs[s].x[2]);
        r.t = Vec3(jobs[s].x[3], jobs[s].x[4], jobs[s].x[5]);
        for (int k = 0; k < 4; ++k) r = local_refine(*stage[k], r.r, r.t, dom);
        res[s] = r;
      }
    };
    std::vector<std::thread> pool;
    for (unsigned k = 0; k + 1 < nthreads; ++k) pool.emplace_back(work);
    work();
    for (auto& th : pool) th.join();
  }
  if (std::getenv("GOSMA_PROFILE"))
    std::fprintf(stderr, "[gosma profile] dive: ladder %.3fs (%s SMA), %zu starts\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - t_beam).count(),
                 dobj ? "GPU" : "host", best.size());
  for (size_t s = 0; s < best.size(); ++s) {
    if (!ok[s]) continue;
    inc->sma += 4;
    if (res[s].value < inc->value) {
      inc->value = res[s].value;
      inc->r = res[s].r;
      inc->t = res[s].t;
    }
  }
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

int gosma_local_refine_batch(gosma_ctx* ctx, size_t n, const double* r0, const double* t0,
                             const gosma_domain* domain, double* r_out, double* t_out,
                             double* value) {
  if (!ctx || !domain || (n && (!r0 || !t0 || !r_out || !t_out || !value)))
    return set_error(GOSMA_EINVAL, "null argument");
  if (n == 0) return GOSMA_OK;
  const Domain dom = make_domain(domain);
  DeviceObjective dev(ctx->device, {&ctx->model});
  if (!dev.ok()) return set_error(GOSMA_ECUDA, "device objective unavailable");
  std::vector<RefineJob> jobs(n);
  for (size_t k = 0; k < n; ++k)
    jobs[k] = RefineJob{{r0[3 * k], r0[3 * k + 1], r0[3 * k + 2], t0[3 * k], t0[3 * k + 1],
                         t0[3 * k + 2]},
                        1,
                        {0}};
  std::vector<RefineOut> out;
  const cudaError_t e = refine_device(&dev, dom, jobs, &out);
  if (e != cudaSuccess)
    return set_error(GOSMA_ECUDA, std::string("refine kernel: ") + cudaGetErrorString(e));
  for (size_t k = 0; k < n; ++k) {
    for (int a = 0; a < 3; ++a) {
      r_out[3 * k + a] = out[k].x[a];
      t_out[3 * k + a] = out[k].x[3 + a];
    }
    value[k] = objective_value(ctx->model, Vec3(out[k].x[0], out[k].x[1], out[k].x[2]),
                               Vec3(out[k].x[3], out[k].x[4], out[k].x[5]));
  }
  return GOSMA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Stepwise solver (one object per rank): the single-GPU gosma_solve and the
// sharded multi-GPU driver (paper_1812_01232_b200/distributed.py) both run
// status() -> [global exchange] -> expand() waves on it.
struct gosma_solver {
  gosma_ctx* ctx = nullptr;
  Domain dom;
  gosma_config cfg{};
  int rank = 0, world = 1;
  Incumbent inc;
  double external = kInf;  // best value found by other ranks (prunes, no pose)
  Frontier F;
  double total_volume = 0.0, pruned_volume = 0.0, resolved_volume = 0.0;
  double floor_lower = kInf;
  // depth-first order (Frontier::select_deepest) while the pool is above its
  // high-water mark; folding (enforce_capacity) only as a last resort
  bool drain = false;
  unsigned long long drain_waves = 0, folds = 0;
  unsigned long long evals = 0, expanded = 0, wave = 0;
  size_t wave_nodes = 0, qcap = 0, mem_cap = 0;
  // child bounds per wave: 2 = siblings (a rotation-split parent's cuboid
  // prologue + self sums once, cross sums per child; translation-split
  // children with the full kernel), 1 = translation-cached (self kernel per
  // distinct cuboid + cross kernel per child), 0 = full kernel per child.
  // GOSMA_WAVE_MODE=full|cached|siblings selects (A/B measurements).
  int wave_mode = [] {
    const char* e = std::getenv("GOSMA_WAVE_MODE");
    if (!e) return 2;
    const std::string m(e);
    return m == "full" ? 0 : (m == "cached" ? 1 : 2);
  }();
  bool cached = wave_mode == 1;
  // GPU objective for incumbent refinements (large mixtures, see gpu_sma)
  std::unique_ptr<DeviceObjective> sma_dev;
  std::vector<ImprovingChild> improving;
  unsigned long long cuboid_evals = 0;
  // GOSMA_PROFILE=1: synchronising per-phase wall times, printed on destroy
  bool profile = std::getenv("GOSMA_PROFILE") != nullptr;
  double phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  std::chrono::steady_clock::time_point lap_t;
  void lap(int k, cudaStream_t s) {
    if (!profile) return;
    cudaStreamSynchronize(s);
    const auto now = std::chrono::steady_clock::now();
    if (k >= 0) phase[k] += std::chrono::duration<double>(now - lap_t).count();
    lap_t = now;
  }
  std::chrono::steady_clock::time_point t_start;
  double elapsed() const {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count();
  }
  double dstar() const { return std::min(inc.value, external); }
};

namespace {

// Free device memory, re-read at most every 0.5 s per device: cudaMemGetInfo
// costs ~1 ms, a tenth of a short solve. The pool budget derived from it only
// decides when to fold (sound either way).
void free_device_memory(int device, size_t* free_b) {
  static std::mutex mu;
  static std::vector<std::pair<std::chrono::steady_clock::time_point, size_t>> seen(64);
  const auto now = std::chrono::steady_clock::now();
  std::lock_guard<std::mutex> lk(mu);
  auto& slot = seen[device & 63];
  if (slot.second == 0 || now - slot.first > std::chrono::milliseconds(500)) {
    size_t total = 0;
    cudaMemGetInfo(&slot.second, &total);
    slot.first = now;
  }
  *free_b = slot.second;
}

int solver_init(gosma_solver* S) {
  gosma_ctx* ctx = S->ctx;
  S->F.prof = S->profile;
  // GOSMA_PROFILE: wall time of the init steps
  auto t_last = std::chrono::steady_clock::now();
  std::string init_prof;
  auto mark = [&](const char* what) {
    if (!S->profile) return;
    const auto now = std::chrono::steady_clock::now();
    char buf[64];
    std::snprintf(buf, sizeof buf, " %s %.2fms", what,
                  1e3 * std::chrono::duration<double>(now - t_last).count());
    init_prof += buf;
    t_last = now;
  };
  if (gpu_sma(ctx->model)) {
    S->sma_dev = std::make_unique<DeviceObjective>(
        ctx->device, std::vector<const HostModel*>{&ctx->model});
    if (!S->sma_dev->ok()) S->sma_dev.reset();
  }
  const HostModel& m = ctx->model;
  const gosma_config& cfg = S->cfg;
  cudaStream_t s = ctx->stream;
  // Roots and the measure (solver.cpp:339-368); rank r owns roots r, r+W, ...
  double total_volume = 0.0;
  for (const Box& b : S->dom.boxes) {
    gosma_node n{};
    n.rhw = S->dom.rot_hw;
    for (int a = 0; a < 3; ++a) n.thw[a] = b.h[a];
    total_volume += volume_of(n);
  }
  const bool unit_measure = !(total_volume > 0.0);
  if (unit_measure) total_volume = static_cast<double>(S->dom.boxes.size());
  S->total_volume = total_volume;
  // Every rank evaluates all feasible roots and runs the full discovery dive
  // (identical, deterministic work: every rank starts from the same d*);
  // with world > 1 the roots are then expanded deterministically to >= 8 x SMs
  // nodes and rank r keeps nodes r, r + world, .... Volumes and
  // evaluations of the replicated work are booked on rank 0 only.
  const bool book = S->rank == 0;
  std::vector<gosma_node> roots;
  std::vector<double> root_vol;
  bool any_feasible = false;
  for (size_t k = 0; k < S->dom.boxes.size(); ++k) {
    const Box& b = S->dom.boxes[k];
    gosma_node n{};
    for (int a = 0; a < 3; ++a) {
      n.rc[a] = S->dom.rot_center[a];
      n.tc[a] = b.c[a];
      n.thw[a] = b.h[a];
    }
    n.rhw = S->dom.rot_hw;
    n.lower = -kInf;
    const double v = unit_measure ? 1.0 : volume_of(n);
    const bool feas = feasible_box(m, b.c, b.h);
    any_feasible = any_feasible || feas;
    if (feas) {
      roots.push_back(n);
      root_vol.push_back(v);
    } else if (book) {
      S->pruned_volume += v;
    }
  }
  if (!any_feasible)
    return set_error(GOSMA_EINFEASIBLE, "solve: no feasible camera center in the domain");
  // Wave size: enough children to keep the bound kernel busy for a few ms
  // (~1.2e8 pair terms per wave), or what the caller asks for.
  size_t pairs = 0;
  for (const HostClass& c : m.classes)
    pairs += static_cast<size_t>(c.n1()) * c.n2() + static_cast<size_t>(c.n1()) * (c.n1() - 1) / 2;
  S->wave_nodes =
      cfg.wave_nodes > 0
          ? static_cast<size_t>(cfg.wave_nodes)
          : std::min<size_t>(std::max<size_t>(300000000 / std::max<size_t>(pairs, 1), 1024),
                             1u << 21);
  // selection arrays for depth-first waves of kDfsWaveFactor x wave_nodes
  cudaError_t e = S->F.reserve(std::max<size_t>(size_t(1) << 20, roots.size() * 2 + 16),
                               kDfsWaveFactor * S->wave_nodes);
  if (e != cudaSuccess) return cuda_error(e, "frontier reserve");
  mark("reserve");
  // Device memory budget for the pool: beyond it the worst nodes fold into the
  // resolved set (sound; the reference's queue_capacity mechanism).
  size_t free_b = 0;
  free_device_memory(ctx->device, &free_b);
  // pool record + key + candidate/compaction indices; the pool may take
  // GOSMA_POOL_FRAC (default 0.5) of the free memory (growth copies need the
  // old arrays alongside the new ones once)
  const size_t per_node = sizeof(gosma_node) + 1 + 8 + 8 + 12;
  static const double pool_frac = [] {
    const char* e = std::getenv("GOSMA_POOL_FRAC");
    const double f = e ? std::atof(e) : 0.5;
    return f > 0.0 && f < 0.9 ? f : 0.5;
  }();
  // (at least 64 waves' parents: a depth-first wave needs room for 32 W
  // children, twice over for the fold target below)
  S->mem_cap = std::max<size_t>(static_cast<size_t>(pool_frac * static_cast<double>(free_b)) /
                                    per_node,
                                64 * S->wave_nodes);
  S->F.cap_limit = S->mem_cap;
  S->qcap = cfg.queue_capacity >= 0
                ? std::min<size_t>(static_cast<size_t>(cfg.queue_capacity), S->mem_cap)
                : S->mem_cap;
  mark("meminfo");
  if (roots.empty()) return GOSMA_OK;
  // Wave 0: the roots (solver.cpp:611-621) + discovery dive.
  std::vector<double> lo, up;
  std::vector<int8_t> sp;
  int rc = eval_host(ctx, roots, kInf, &lo, &up, &sp);
  if (rc != GOSMA_OK) return rc;
  mark("roots");
  unsigned long long evals = roots.size();
  if (cfg.discovery_dive) {
    const auto t0 = std::chrono::steady_clock::now();
    rc = discovery_dive(ctx, S->dom, roots, cfg, &S->inc, &evals, 0.0);
    if (rc != GOSMA_OK) return rc;
    S->phase[7] += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
  mark("dive");
  for (size_t i = 0; i < roots.size(); ++i)
    if (up[i] < S->inc.value && (rc = improve(m, S->dom, roots[i], &S->inc, S->sma_dev.get())) !=
                                    GOSMA_OK)
      return rc;
  mark("improve");
  // route the wave's nodes (solver.cpp:396-405); returns the ones to keep
  std::vector<gosma_node> keep;
  std::vector<int8_t> ks;
  std::vector<double> kv;
  auto route_host = [&](const std::vector<gosma_node>& nodes, const std::vector<double>& vols) {
    keep.clear();
    ks.clear();
    kv.clear();
    for (size_t i = 0; i < nodes.size(); ++i) {
      gosma_node b = nodes[i];
      b.lower = lo[i];
      if (!(b.lower < S->dstar())) {
        if (book) S->pruned_volume += vols[i];
      } else if (!splittable(b)) {
        // resolved: FP64 bound, so zero-size domains certify exactly
        const double l64 = lower_bound_fp64(m, Vec3(b.rc[0], b.rc[1], b.rc[2]), b.rhw,
                                            Vec3(b.tc[0], b.tc[1], b.tc[2]),
                                            Vec3(b.thw[0], b.thw[1], b.thw[2]), -kInf);
        if (book) S->resolved_volume += vols[i];
        S->floor_lower = std::min(S->floor_lower, std::max(l64, b.lower));
      } else {
        keep.push_back(b);
        ks.push_back(sp[i]);
        kv.push_back(vols[i]);
      }
    }
  };
  route_host(roots, root_vol);
  if (S->world > 1) {
    // deterministic breadth-first expansion (subdivide_adaptive with the
    // kernel's split flags) until every rank gets a share, then stripe
    const size_t target = std::max<size_t>(8 * static_cast<size_t>(ctx->sm_count),
                                           256 * static_cast<size_t>(S->world));
    while (!keep.empty() && keep.size() < target) {
      std::vector<gosma_node> kids;
      std::vector<double> kvol;
      kids.reserve(8 * keep.size());
      for (size_t i = 0; i < keep.size(); ++i)
        for (int c = 0; c < 8; ++c) {
          gosma_node k = child_of(keep[i], ks[i], c);
          k.lower = keep[i].lower;
          kids.push_back(k);
          kvol.push_back(kv[i] / 8.0);
        }
      if ((rc = eval_host(ctx, kids, S->dstar(), &lo, &up, &sp)) != GOSMA_OK) return rc;
      evals += kids.size();
      for (size_t i = 0; i < kids.size(); ++i)
        if (up[i] < S->inc.value &&
            (rc = improve(m, S->dom, kids[i], &S->inc, S->sma_dev.get())) != GOSMA_OK)
          return rc;
      route_host(kids, kvol);
    }
    size_t out = 0;
    for (size_t i = 0; i < keep.size(); ++i)
      if (static_cast<int>(i % S->world) == S->rank) {
        keep[out] = keep[i];
        ks[out] = ks[i];
        kv[out] = kv[i];
        ++out;
      }
    keep.resize(out);
    ks.resize(out);
    kv.resize(out);
  }
  if (book) S->evals += evals;
  if (!keep.empty() &&
      (e = S->F.upload(keep.data(), ks.data(), kv.data(), keep.size(), s)) != cudaSuccess)
    return cuda_error(e, "frontier upload");
  mark("upload");
  if (S->profile) std::fprintf(stderr, "[gosma profile] init:%s\n", init_prof.c_str());
  return GOSMA_OK;
}

}  // namespace

extern "C" {

int gosma_solver_create(gosma_ctx* ctx, const gosma_domain* domain, const gosma_config* config,
                        int rank, int world, gosma_solver** out) {
  if (!ctx || !domain || !config || !out) return set_error(GOSMA_EINVAL, "null argument");
  *out = nullptr;
  const gosma_config& cfg = *config;
  // solver.cpp:320-329
  if (!(cfg.epsilon > 0.0)) return set_error(GOSMA_EINVAL, "solve: epsilon must be > 0");
  if (cfg.batch_size < 1) return set_error(GOSMA_EINVAL, "solve: batch_size must be >= 1");
  if (cfg.zeta != ctx->model.zeta)
    return set_error(GOSMA_EINVAL, "solve: config.zeta differs from the context's standoff radius");
  if (domain->n_boxes < 1 || !domain->boxes)
    return set_error(GOSMA_EINVAL, "solve: empty translation domain");
  if (world < 1 || rank < 0 || rank >= world) return set_error(GOSMA_EINVAL, "bad rank/world");
  auto* S = new gosma_solver();
  S->ctx = ctx;
  S->dom = make_domain(domain);
  S->cfg = cfg;
  S->rank = rank;
  S->world = world;
  S->t_start = std::chrono::steady_clock::now();
  DeviceGuard g(ctx->device);
  const int rc = solver_init(S);
  if (rc != GOSMA_OK) {
    S->F.release();
    delete S;
    return rc;
  }
  *out = S;
  return GOSMA_OK;
}

void gosma_solver_destroy(gosma_solver* S) {
  if (!S) return;
  if (S->profile) {
    static const char* kName[8] = {"status", "select", "expand+self", "eval", "best+improve",
                                   "route", "compact", "dive"};
    std::fprintf(stderr,
                 "[gosma profile] waves %llu (drain %llu, folds %llu, budget %zu nodes) evals %llu "
                 "cuboids %llu rebuilds %llu pool %zu:",
                 S->wave, S->drain_waves, S->folds, S->mem_cap, S->evals, S->cuboid_evals,
                 S->F.rebuilds, S->F.size);
    for (int k = 0; k < 8; ++k) std::fprintf(stderr, " %s %.3fs", kName[k], S->phase[k]);
    std::fprintf(stderr,
                 " | select: rebuild %.3fs descend %.3fs pick %.3fs list %.3fs (max bin %zu, "
                 "max list %zu) | route: grow %.3fs rest %.3fs | kept %.3f of children\n",
                 S->F.t_sub[0], S->F.t_sub[1], S->F.t_sub[2], S->F.t_sub[3], S->F.max_bin,
                 S->F.max_cand, S->F.t_sub[4], S->F.t_sub[5],
                 S->F.kids_total ? double(S->F.kids_kept) / double(S->F.kids_total) : 0.0);
  }
  DeviceGuard g(S->ctx->device);
  S->F.release();
  delete S;
}

int gosma_solver_status(gosma_solver* S, gosma_wave_status* st) {
  if (!S || !st) return set_error(GOSMA_EINVAL, "null argument");
  DeviceGuard g(S->ctx->device);
  cudaStream_t s = S->ctx->stream;
  cudaError_t e;
  S->lap(-1, s);
  struct LapAtExit {
    gosma_solver* S;
    cudaStream_t s;
    ~LapAtExit() { S->lap(0, s); }
  } lap_at_exit{S, s};
  // capacity folding (solver.cpp:433-447) at the caller's queue_capacity
  const bool user_cap = S->cfg.queue_capacity >= 0 &&
                        static_cast<size_t>(S->cfg.queue_capacity) <= S->mem_cap;
  const size_t wave_room =
      8 * std::max(S->wave_nodes, std::min(kDfsWaveFactor * S->wave_nodes, size_t(1) << 20));
  if (user_cap && S->F.live_upper_bound() > S->qcap) {
    double fv = 0.0, fmin = kInf;
    if ((e = S->F.fold_to(S->qcap, s, &fv, &fmin)) != cudaSuccess) return cuda_error(e, "fold");
    S->resolved_volume += fv;
    S->floor_lower = std::min(S->floor_lower, fmin);
  } else if (!user_cap) {
    // The device memory budget: above the high-water mark the waves take the
    // deepest nodes below the limit (depth-first: the open set stays ~8 W per
    // level), which bounds the pool without changing the work or the
    // certificate; below the low-water mark best-first resumes. Folding (it
    // caps the certified bound) happens only if the pool still overflows.
    static const bool drain_on = [] {
      const char* e = std::getenv("GOSMA_DRAIN");
      return !(e && std::string(e) == "0");
    }();
    const size_t live = S->F.live_upper_bound();
    if (drain_on && !S->drain && live + wave_room > S->mem_cap * 3 / 4) S->drain = true;
    if (S->drain && live + wave_room < S->mem_cap * 9 / 20) S->drain = false;
    if (S->F.size + wave_room > S->mem_cap) {
      double dropped = 0.0;  // holes and stale nodes first
      if ((e = S->F.compact(host_order_key(S->dstar()), s, &dropped)) != cudaSuccess)
        return cuda_error(e, "compact");
      S->pruned_volume += dropped;
    }
    if (S->F.size + wave_room > S->mem_cap) {
      const size_t target = drain_on && S->mem_cap > 4 * wave_room
                                ? S->mem_cap - 2 * wave_room
                                : (S->mem_cap * 3 / 4 > 2 * wave_room ? S->mem_cap * 3 / 4 - wave_room
                                                                      : S->mem_cap / 2);
      double fv = 0.0, fmin = kInf;
      if ((e = S->F.fold_to(target, s, &fv, &fmin)) != cudaSuccess) return cuda_error(e, "fold");
      S->resolved_volume += fv;
      S->floor_lower = std::min(S->floor_lower, fmin);
      ++S->folds;
    }
  }
  unsigned long long kmin = kHoleKey;
  if ((e = S->F.min_key(s, &kmin)) != cudaSuccess) return cuda_error(e, "frontier min");
  st->best_value = S->inc.value;
  st->frontier_min = kmin == kHoleKey ? kInf : key_to_double(kmin);
  st->floor_lower = S->floor_lower;
  st->live_nodes = kmin == kHoleKey ? 0 : S->F.live_upper_bound();
  st->bound_evaluations = S->evals;
  st->pruned_volume = S->pruned_volume;
  st->resolved_volume = S->resolved_volume;
  st->total_volume = S->total_volume;
  st->elapsed_seconds = S->elapsed();
  return GOSMA_OK;
}

int gosma_solver_set_incumbent(gosma_solver* S, double value) {
  if (!S) return set_error(GOSMA_EINVAL, "null argument");
  S->external = std::min(S->external, value);
  return GOSMA_OK;
}

int gosma_solver_expand(gosma_solver* S, double limit, unsigned long long max_evals) {
  if (!S) return set_error(GOSMA_EINVAL, "null argument");
  gosma_ctx* ctx = S->ctx;
  DeviceGuard g(ctx->device);
  cudaStream_t s = ctx->stream;
  cudaError_t e;
  // depth-first waves take kDfsWaveFactor x as many parents: their selection
  // scans the whole pool, which a larger wave amortises
  size_t want = S->drain ? std::max(S->wave_nodes,
                                    std::min(kDfsWaveFactor * S->wave_nodes, size_t(1) << 20))
                         : S->wave_nodes;
  if (max_evals > 0) want = std::min<size_t>(want, std::max<unsigned long long>(1, (max_evals + 7) / 8));
  size_t n_sel = 0;
  S->lap(-1, s);
  // Expand only nodes that can still matter: lower < limit (= d* - eps).
  if ((e = S->drain ? S->F.select_deepest(want, host_order_key(limit), s, &n_sel)
                    : S->F.select_smallest(want, host_order_key(limit), s, &n_sel)) !=
      cudaSuccess)
    return cuda_error(e, "select");
  if (S->drain) ++S->drain_waves;
  if (n_sel == 0) {
    // Nothing below the limit yet the gap is open (a resolved floor holds the
    // bound down): keep refining the live nodes, as the reference's heap would.
    if ((e = S->F.select_smallest(want, host_order_key(S->dstar()), s, &n_sel)) != cudaSuccess)
      return cuda_error(e, "select");
    if (n_sel == 0) {  // only stale nodes remain
      double dropped = 0.0;
      if ((e = S->F.compact(host_order_key(S->dstar()), s, &dropped)) != cudaSuccess)
        return cuda_error(e, "compact");
      S->pruned_volume += dropped;
      ++S->wave;
      return GOSMA_OK;
    }
  }
  const size_t n_kids = n_sel * 8;
  if ((e = S->F.ensure_kids(n_sel)) != cudaSuccess) return cuda_error(e, "child buffers");
  S->lap(1, s);
  EvalArgs a;
  a.work = work_counter(ctx, s);
  if ((e = attach_redo(ctx, s, static_cast<long long>(n_kids), &a)) != cudaSuccess)
    return cuda_error(e, "redo list");
  a.skip_upper_at = S->dstar();
  if (S->cached) {
    // Translation-cached bounds: the self sums once per distinct cuboid
    // (rotation-split siblings share theirs), then the cross sums per child.
    size_t n_cub = 0;
    if ((e = S->F.expand_selected_cached(n_sel, s, &n_cub)) != cudaSuccess)
      return cuda_error(e, "expand");
    a.nodes = reinterpret_cast<const double*>(S->F.tnodes);
    a.n = static_cast<long long>(n_cub);
    a.self_out = S->F.tself;
    if ((e = launch_eval_self(ctx->dev, a, ctx->sm_count, s)) != cudaSuccess)
      return cuda_error(e, "eval cuboids");
    a.tindex = S->F.tidx;
    S->cuboid_evals += n_cub;
    S->lap(2, s);
  } else if ((e = S->F.expand_selected(n_sel, s)) != cudaSuccess) {
    return cuda_error(e, "expand");
  }
  a.nodes = reinterpret_cast<const double*>(S->F.kids);
  a.n = static_cast<long long>(n_kids);
  a.lower = S->F.kid_lower;
  a.upper = S->F.kid_upper;
  a.split_rot = S->F.kid_split;
  if (S->wave_mode == 2) {
    // the split of the selection into rotation parents / translation children
    // stays on the device: the kernels read their item counts there (grids
    // sized for the upper bounds), no host round trip
    if ((e = S->F.wave_lists(n_sel, s)) != cudaSuccess) return cuda_error(e, "wave lists");
    S->lap(2, s);
    EvalArgs b = a;
    b.nodes = reinterpret_cast<const double*>(S->F.nodes);  // the parents, in the pool
    b.n = static_cast<long long>(n_sel);
    b.n_dev = reinterpret_cast<const long long*>(S->F.list_counts);
    b.item_index = S->F.rot_list;
    b.sel = S->F.sel;
    if ((e = launch_eval_siblings(ctx->dev, b, ctx->sm_count, s)) != cudaSuccess)
      return cuda_error(e, "eval siblings");
    EvalArgs c = a;
    c.n = static_cast<long long>(n_kids);
    c.n_dev = reinterpret_cast<const long long*>(S->F.list_counts + 1);
    c.item_index = S->F.trans_list;
    if ((e = launch_eval_bounds(ctx->dev, c, ctx->sm_count, s)) != cudaSuccess)
      return cuda_error(e, "eval children");
    S->cuboid_evals += n_sel;
  } else if ((e = (S->cached ? launch_eval_cross_cached(ctx->dev, a, ctx->sm_count, s)
                             : launch_eval_bounds(ctx->dev, a, ctx->sm_count, s))) !=
             cudaSuccess) {
    return cuda_error(e, "eval children");
  }
  S->lap(3, s);
  S->evals += n_kids;
  S->expanded += n_sel;
  // process_wave (solver.cpp:409-431): in child order, every branch whose
  // upper bound beats the incumbent at that moment is refined; the device
  // hands over the prefix-minimum records below the incumbent, the host
  // replays them against the incumbent as the refinements lower it
  if ((e = S->F.improving_children(n_kids, S->inc.value, s, &S->improving)) != cudaSuccess)
    return cuda_error(e, "improving children");
  for (const ImprovingChild& c : S->improving) {
    if (!(c.upper < S->inc.value)) continue;
    const int rc = improve(ctx->model, S->dom, c.node, &S->inc, S->sma_dev.get());
    if (rc != GOSMA_OK) return rc;
  }
  S->lap(4, s);
  RouteStats rs;
  // children already finished for the certificate (bound >= limit = d* - eps)
  // go to the floor instead of the pool (GOSMA_FINISH=0: keep them, A/B)
  static const bool finish_on = [] {
    const char* v = std::getenv("GOSMA_FINISH");
    return !(v && std::string(v) == "0");
  }();
  const double finish = finish_on ? std::min(limit, S->dstar()) : kInf;
  if ((e = S->F.route_append(n_kids, S->dstar(), finish, s, &rs)) != cudaSuccess)
    return cuda_error(e, "route");
  S->pruned_volume += rs.pruned_volume;
  S->resolved_volume += rs.resolved_volume;
  if (rs.floor_key != ~0ull) S->floor_lower = std::min(S->floor_lower, key_to_double(rs.floor_key));
  S->lap(5, s);
  // amortised compaction: drop holes and stale nodes (lower >= d*,
  // solver.cpp:660-663) once they fill half the pool
  if (S->F.holes * 2 > S->F.size) {
    double dropped = 0.0;
    if ((e = S->F.compact(host_order_key(S->dstar()), s, &dropped)) != cudaSuccess)
      return cuda_error(e, "compact");
    S->pruned_volume += dropped;
  }
  S->lap(6, s);
  ++S->wave;
  return GOSMA_OK;
}

namespace {
// Selects the best live nodes (they are the next to expand) and gathers them
// into the wave's child buffers; returns the count.
int export_select(gosma_solver* S, size_t max_nodes, size_t* n) {
  cudaStream_t s = S->ctx->stream;
  cudaError_t e;
  *n = 0;
  max_nodes = std::min(max_nodes, S->F.sel_cap);
  if ((e = S->F.select_smallest(max_nodes, host_order_key(S->dstar()), s, n)) != cudaSuccess)
    return cuda_error(e, "export select");
  if ((e = S->F.ensure_kids((*n + 7) / 8)) != cudaSuccess) return cuda_error(e, "export buffers");
  if ((e = S->F.gather_selected(*n, s, S->F.kids, S->F.kid_split, S->F.kid_vol)) != cudaSuccess)
    return cuda_error(e, "export gather");
  return GOSMA_OK;
}
}  // namespace

int gosma_solver_export(gosma_solver* S, size_t max_nodes, gosma_node* nodes, int8_t* split,
                        double* vol, size_t* n_out) {
  if (!S || !n_out) return set_error(GOSMA_EINVAL, "null argument");
  *n_out = 0;
  if (max_nodes == 0) return GOSMA_OK;
  DeviceGuard g(S->ctx->device);
  cudaStream_t s = S->ctx->stream;
  size_t n = 0;
  int rc = export_select(S, max_nodes, &n);
  if (rc != GOSMA_OK) return rc;
  cudaError_t e = cudaSuccess;
  if (n) {
    e = cudaMemcpyAsync(nodes, S->F.kids, n * sizeof(gosma_node), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(split, S->F.kid_split, n, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(vol, S->F.kid_vol, n * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (e != cudaSuccess) return cuda_error(e, "export copy");
  *n_out = n;
  return GOSMA_OK;
}

int gosma_solver_export_device(gosma_solver* S, size_t max_nodes, gosma_node* d_nodes,
                               int8_t* d_split, double* d_vol, size_t* n_out) {
  if (!S || !n_out) return set_error(GOSMA_EINVAL, "null argument");
  *n_out = 0;
  if (max_nodes == 0) return GOSMA_OK;
  DeviceGuard g(S->ctx->device);
  cudaStream_t s = S->ctx->stream;
  size_t n = 0;
  int rc = export_select(S, max_nodes, &n);
  if (rc != GOSMA_OK) return rc;
  cudaError_t e = cudaSuccess;
  if (n) {
    e = cudaMemcpyAsync(d_nodes, S->F.kids, n * sizeof(gosma_node), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_split, S->F.kid_split, n, cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d_vol, S->F.kid_vol, n * sizeof(double), cudaMemcpyDeviceToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  if (e != cudaSuccess) return cuda_error(e, "export copy");
  *n_out = n;
  return GOSMA_OK;
}

int gosma_solver_import_device(gosma_solver* S, const gosma_node* d_nodes, const int8_t* d_split,
                               const double* d_vol, size_t n) {
  if (!S) return set_error(GOSMA_EINVAL, "null argument");
  if (n == 0) return GOSMA_OK;
  DeviceGuard g(S->ctx->device);
  const cudaError_t e = S->F.upload_device(d_nodes, d_split, d_vol, n, S->ctx->stream);
  if (e != cudaSuccess) return cuda_error(e, "import");
  return GOSMA_OK;
}

int gosma_solver_import(gosma_solver* S, const gosma_node* nodes, const int8_t* split,
                        const double* vol, size_t n) {
  if (!S) return set_error(GOSMA_EINVAL, "null argument");
  if (n == 0) return GOSMA_OK;
  DeviceGuard g(S->ctx->device);
  const cudaError_t e = S->F.upload(nodes, split, vol, n, S->ctx->stream);
  if (e != cudaSuccess) return cuda_error(e, "import");
  return GOSMA_OK;
}

int gosma_objective_batch(gosma_ctx* ctx, const double* poses, size_t n, double* f, double* g) {
  if (!ctx) return set_error(GOSMA_EINVAL, "null context");
  if (n == 0) return GOSMA_OK;
  if (!poses || !f || !g) return set_error(GOSMA_EINVAL, "null buffer");
  DeviceObjective dev(ctx->device, {&ctx->model});
  if (!dev.ok()) return set_error(GOSMA_ECUDA, "objective kernel setup failed");
  std::vector<ObjRequest> req(n);
  for (size_t k = 0; k < n; ++k) {
    for (int a = 0; a < 6; ++a) req[k].x[a] = poses[6 * k + a];
    req[k].model = 0;
  }
  std::vector<double> fv, gv;
  const cudaError_t e = dev.evaluate(req, &fv, &gv);
  if (e != cudaSuccess) return cuda_error(e, "objective batch");
  std::copy(fv.begin(), fv.end(), f);
  std::copy(gv.begin(), gv.end(), g);
  return GOSMA_OK;
}

int gosma_solver_live_volume(gosma_solver* S, double* volume) {
  if (!S || !volume) return set_error(GOSMA_EINVAL, "null argument");
  DeviceGuard g(S->ctx->device);
  const cudaError_t e = S->F.live_volume(S->ctx->stream, volume);
  if (e != cudaSuccess) return cuda_error(e, "live volume");
  return GOSMA_OK;
}

int gosma_solver_result(gosma_solver* S, gosma_report* report) {
  if (!S || !report) return set_error(GOSMA_EINVAL, "null argument");
  *report = gosma_report{};
  report->best_value = S->inc.value;
  for (int k = 0; k < 3; ++k) {
    report->best_r[k] = S->inc.r[k];
    report->best_t[k] = S->inc.t[k];
  }
  report->branches_expanded = S->expanded;
  report->sma_invocations = S->inc.sma;
  report->bound_evaluations = S->evals;
  report->wall_time_seconds = S->elapsed();
  report->waves = S->wave;
  return GOSMA_OK;
}

// solve() (solver.cpp:312-688) on one GPU: status -> stop rules -> expand.
int gosma_solve(gosma_ctx* ctx, const gosma_domain* domain, const gosma_config* config,
                gosma_report* report, gosma_trace_cb trace, void* user) {
  if (!report) return set_error(GOSMA_EINVAL, "null argument");
  gosma_solver* S = nullptr;
  const auto tc0 = std::chrono::steady_clock::now();
  int rc = gosma_solver_create(ctx, domain, config, 0, 1, &S);
  if (rc != GOSMA_OK) return rc;
  if (S->profile)
    std::fprintf(stderr, "[gosma profile] create %.3fs\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - tc0).count());
  const gosma_config& cfg = *config;
  double certified = -kInf;
  int status = GOSMA_STATUS_QUEUE_EXHAUSTED;
  for (;;) {
    gosma_wave_status st;
    if ((rc = gosma_solver_status(S, &st)) != GOSMA_OK) break;
    const double dstar = st.best_value;
    // certified lower bound (solver.cpp:626-627)
    certified = std::max(certified, std::min(std::min(dstar, st.frontier_min), st.floor_lower));
    if (trace) {
      const double queue_volume =
          std::max(0.0, st.total_volume - st.pruned_volume - st.resolved_volume);
      trace(user, S->wave, st.bound_evaluations, dstar, certified, st.live_nodes,
            queue_volume / st.total_volume, st.pruned_volume / st.total_volume,
            st.resolved_volume / st.total_volume);
    }
    // stop rules (solver.cpp:629-645)
    if (dstar - certified <= cfg.epsilon) {
      status = GOSMA_STATUS_EPSILON_OPTIMAL;
      break;
    }
    if (st.live_nodes == 0) {
      status = GOSMA_STATUS_QUEUE_EXHAUSTED;
      break;
    }
    if (cfg.time_limit >= 0.0 && st.elapsed_seconds >= cfg.time_limit) {
      status = GOSMA_STATUS_TIME_LIMIT;
      break;
    }
    unsigned long long left = 0;
    if (cfg.max_evaluations >= 0) {
      if (st.bound_evaluations >= static_cast<unsigned long long>(cfg.max_evaluations)) {
        status = GOSMA_STATUS_TIME_LIMIT;
        break;
      }
      left = static_cast<unsigned long long>(cfg.max_evaluations) - st.bound_evaluations;
    }
    if ((rc = gosma_solver_expand(S, dstar - cfg.epsilon, left)) != GOSMA_OK) break;
  }
  if (rc != GOSMA_OK) {
    gosma_solver_destroy(S);
    return rc;
  }
  gosma_solver_result(S, report);
  report->global_lower = certified;
  report->gap = report->best_value - certified;
  report->status = status;
  const auto td0 = std::chrono::steady_clock::now();
  const bool prof = S->profile;
  gosma_solver_destroy(S);
  if (prof)
    std::fprintf(stderr, "[gosma profile] destroy %.3fs\n",
                 std::chrono::duration<double>(std::chrono::steady_clock::now() - td0).count());
  return status == GOSMA_STATUS_TIME_LIMIT ? GOSMA_EBUDGET : GOSMA_OK;
}


}  // extern "C"
