// C ABI (include/gosma_capi.h): context construction, bound evaluation entry
// points, host objective. The solver entry point lives in solver.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "capi_internal.hpp"
#include "gosma_capi.h"

namespace gosma {

thread_local std::string g_last_error;

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_error(cudaError_t e, const char* where) {
  return set_error(GOSMA_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

namespace {
gosma_ctx::StreamScratch* stream_scratch(gosma_ctx* ctx, cudaStream_t s) {
  for (auto& ws : ctx->work_slots)
    if (ws.stream == s) return &ws;
  gosma_ctx::StreamScratch ws;
  ws.stream = s;
  if (cudaMalloc(&ws.work, sizeof(unsigned int)) != cudaSuccess) return nullptr;
  ctx->work_slots.push_back(ws);
  return &ctx->work_slots.back();
}
}  // namespace

unsigned int* work_counter(gosma_ctx* ctx, cudaStream_t s) {
  if (s == ctx->stream || s == nullptr) return static_cast<unsigned int*>(ctx->d_work);
  std::lock_guard<std::mutex> lk(ctx->work_mu);
  gosma_ctx::StreamScratch* ws = stream_scratch(ctx, s);
  return ws ? static_cast<unsigned int*>(ws->work) : nullptr;
}

cudaError_t attach_redo(gosma_ctx* ctx, cudaStream_t s, long long n_out, EvalArgs* a) {
  if (s == nullptr) s = ctx->stream;
  std::lock_guard<std::mutex> lk(ctx->work_mu);
  gosma_ctx::StreamScratch* ws = stream_scratch(ctx, s);
  if (!ws) return cudaErrorMemoryAllocation;
  if (n_out > ws->redo_cap) {
    cudaFree(ws->redo_count);
    cudaFree(ws->redo_nodes);
    cudaFree(ws->redo_slot);
    ws->redo_count = nullptr;
    ws->redo_nodes = nullptr;
    ws->redo_slot = nullptr;
    ws->redo_cap = 0;
    const long long cap = std::max<long long>(n_out, 1024);
    cudaError_t e;
    if ((e = cudaMalloc(&ws->redo_count, sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMalloc(&ws->redo_nodes, cap * 11 * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&ws->redo_slot, cap * sizeof(long long))) != cudaSuccess)
      return e;
    ws->redo_cap = cap;
  }
  a->redo_count = ws->redo_count;
  a->redo_nodes = ws->redo_nodes;
  a->redo_slot = ws->redo_slot;
  a->redo_cap = ws->redo_cap;
  return cudaSuccess;
}

namespace {

bool weights_close(double sum) { return std::fabs(sum - 1.0) <= 1e-9; }

template <typename T>
cudaError_t upload(const std::vector<T>& h, T** d) {
  *d = nullptr;
  if (h.empty()) return cudaSuccess;
  cudaError_t e = cudaMalloc(reinterpret_cast<void**>(d), h.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  return cudaMemcpy(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
}

double class_self_energy(const HostClass& c) {
  // objective.cpp:55-64
  double c2 = 0.0;
  for (int j = 0; j < c.n2(); ++j)
    for (int k = 0; k < c.n2(); ++k) {
      const Vec3 s(c.b[3 * j] + c.b[3 * k], c.b[3 * j + 1] + c.b[3 * k + 1],
                   c.b[3 * j + 2] + c.b[3 * k + 2]);
      c2 += c.phi2[j] * c.phi2[k] * std::exp(log_z_eval(s.norm()) - c.log_z2[j] - c.log_z2[k]);
    }
  return c2;
}

double logw_host(double x) {
  if (x > 30.0) return -std::log(x);
  return log_z_eval(x) - x;
}

}  // namespace

// Builds the device tables from the host model.
int ctx_upload(gosma_ctx* ctx) {
  const HostModel& hm = ctx->model;
  std::vector<ClassSpan> spans;
  std::vector<double> cls_w, mu, inv_s2, phi1, m;
  std::vector<float> log_phi1, kappa2, e2;
  int o1 = 0, o2 = 0, max_n1 = 0;
  for (const HostClass& c : hm.classes) {
    spans.push_back({o1, c.n1(), o2, c.n2()});
    cls_w.push_back(c.weight);
    max_n1 = std::max(max_n1, c.n1());
    for (int i = 0; i < c.n1(); ++i) {
      for (int a = 0; a < 3; ++a) mu.push_back(c.mu[3 * i + a]);
      inv_s2.push_back(1.0 / c.sigma2[i]);
      phi1.push_back(c.phi1[i]);
      log_phi1.push_back(c.phi1[i] > 0.0 ? static_cast<float>(std::log(c.phi1[i]))
                                         : kLogZeroWeight);
    }
    for (int j = 0; j < c.n2(); ++j) {
      for (int a = 0; a < 3; ++a) m.push_back(c.b[3 * j + a] / c.kappa2[j]);
      kappa2.push_back(static_cast<float>(c.kappa2[j]));
      const double k = c.kappa2[j];
      e2.push_back(static_cast<float>(c.phi2[j] * k / -std::expm1(-2.0 * k)));  // phi2 / W(k)
    }
    o1 += c.n1();
    o2 += c.n2();
  }
  cudaError_t e;
  DevCtx& d = ctx->dev;
  d.n_classes = static_cast<int>(hm.classes.size());
  d.n1_total = o1;
  d.n2_total = o2;
  d.max_n1 = max_n1;
  d.max_n2 = 0;
  for (const HostClass& c : hm.classes) d.max_n2 = std::max(d.max_n2, c.n2());
  // GOSMA_STREAM_CLASSES=0: keep every class's table (A/B measurements)
  static const bool no_stream = [] {
    const char* e = std::getenv("GOSMA_STREAM_CLASSES");
    return e && std::string(e) == "0";
  }();
  d.stream_classes = hm.classes.size() > 1 && !no_stream ? 1 : 0;
  d.zeta = hm.zeta;
  d.lb_margin = ctx->lb_margin;
  d.lb_err_scale = 1.0;
  d.tail_chunks = 0;
  static const bool precise_off = [] {  // GOSMA_PRECISE=0: FP32 pass only (A/B)
    const char* e = std::getenv("GOSMA_PRECISE");
    return e && std::string(e) == "0";
  }();
  d.precise = precise_off ? 0 : 1;
  static const double redo_rel = [] {  // GOSMA_REDO_REL: fix-up threshold (A/B)
    const char* e = std::getenv("GOSMA_REDO_REL");
    const double v = e ? std::atof(e) : 0.0;
    return v > 0.0 ? v : 1.2e-4;
  }();
  d.redo_rel = redo_rel;
  d.min_k2 = INFINITY;  // K1's exact-path gate (exact_needed_row)
  for (const HostClass& c : hm.classes)
    for (double k : c.kappa2) d.min_k2 = std::min(d.min_k2, static_cast<float>(k));
  for (const ClassSpan& cs : spans)
    if (cs.n1 % 32 != 0 && cs.n1 % 32 <= 16) d.tail_chunks = 1;
  ClassSpan* dspans;
  if ((e = upload(spans, &dspans)) != cudaSuccess) return cuda_error(e, "ctx upload");
  d.cls = dspans;
  double *dw, *dmu, *dis2, *dphi, *dm;
  float *dlp, *dk2, *de2;
  if ((e = upload(cls_w, &dw)) != cudaSuccess || (e = upload(mu, &dmu)) != cudaSuccess ||
      (e = upload(inv_s2, &dis2)) != cudaSuccess || (e = upload(phi1, &dphi)) != cudaSuccess ||
      (e = upload(m, &dm)) != cudaSuccess || (e = upload(log_phi1, &dlp)) != cudaSuccess ||
      (e = upload(kappa2, &dk2)) != cudaSuccess || (e = upload(e2, &de2)) != cudaSuccess)
    return cuda_error(e, "ctx upload");
  d.cls_w = dw;
  d.mu = dmu;
  d.inv_s2 = dis2;
  d.phi1 = dphi;
  d.m = dm;
  d.log_phi1 = dlp;
  d.kappa2 = dk2;
  d.g2 = de2;
  ctx->owned = {dspans, dw, dmu, dis2, dphi, dm, dlp, dk2, de2};
  if ((e = cudaMalloc(&ctx->d_work, sizeof(unsigned int))) != cudaSuccess)
    return cuda_error(e, "ctx upload");
  // one node's tables must fit a CTA (launches shrink the CTA, down to one
  // table per CTA, as tables grow)
  const size_t smem = eval_smem_per_warp(d) + 256;
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device);
  if (smem > static_cast<size_t>(max_optin)) {
    return set_error(GOSMA_EINVAL, "mixtures too large for the shared-memory tables (" +
                                       std::to_string(smem) + " B per node)");
  }
  return GOSMA_OK;
}

void ctx_free_device(gosma_ctx* ctx) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(ctx->device);
  for (void* p : ctx->owned) cudaFree(p);
  ctx->owned.clear();
  if (ctx->d_work) cudaFree(ctx->d_work);
  ctx->d_work = nullptr;
  {
    std::lock_guard<std::mutex> lk(ctx->work_mu);
    for (auto& ws : ctx->work_slots) {
      cudaFree(ws.work);
      cudaFree(ws.redo_count);
      cudaFree(ws.redo_nodes);
      cudaFree(ws.redo_slot);
    }
    ctx->work_slots.clear();
  }
  cudaFree(ctx->d_cache_nodes);
  cudaFree(ctx->d_cache_self);
  ctx->d_cache_nodes = nullptr;
  ctx->d_cache_self = nullptr;
  ctx->cache_cap = 0;
  cudaFree(ctx->d_child_kids);
  cudaFree(ctx->d_child_lists);
  cudaFree(ctx->d_child_sel);
  ctx->d_child_kids = nullptr;
  ctx->d_child_lists = nullptr;
  ctx->d_child_sel = nullptr;
  ctx->child_cap = 0;
  ctx->scratch.release();
  if (ctx->dive_graph) cudaGraphExecDestroy(ctx->dive_graph);
  ctx->dive_graph = nullptr;
  cudaFree(ctx->dive_buf);
  ctx->dive_buf = nullptr;
  ctx->dive_bytes = 0;
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->h2d_stream) cudaStreamDestroy(ctx->h2d_stream);
  if (ctx->d2h_stream) cudaStreamDestroy(ctx->d2h_stream);
  for (cudaEvent_t& ev : ctx->pipe_ev) {
    if (ev) cudaEventDestroy(ev);
    ev = nullptr;
  }
  ctx->h2d_stream = ctx->d2h_stream = nullptr;
  ctx->stream = nullptr;
  cudaSetDevice(cur);
}

void Scratch::release() {
  if (d_nodes) cudaFree(d_nodes);
  if (d_lower) cudaFree(d_lower);
  if (d_upper) cudaFree(d_upper);
  if (d_split) cudaFree(d_split);
  if (h_pinned) cudaFreeHost(h_pinned);
  d_nodes = nullptr;
  d_lower = d_upper = nullptr;
  d_split = nullptr;
  h_pinned = nullptr;
  cap = 0;
}

cudaError_t Scratch::reserve(size_t n) {
  if (n <= cap) return cudaSuccess;
  release();
  size_t c = std::max<size_t>(n, 1024);
  cudaError_t e;
  if ((e = cudaMalloc(&d_nodes, c * sizeof(gosma_node))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&d_lower, c * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&d_upper, c * sizeof(double))) != cudaSuccess) return e;
  if ((e = cudaMalloc(&d_split, c * sizeof(int8_t))) != cudaSuccess) return e;
  cap = c;
  return cudaSuccess;
}

int validate_and_build(const gosma_class_view* classes, int n_classes, double zeta,
                       unsigned flags, HostModel* out) {
  // ObjectiveContext constructors (objective.cpp:28-68, 103-121) and the
  // component invariants (sphere_stats.cpp:10-35, unit_vector.hpp:17-24).
  if (!(zeta > 0.0)) return set_error(GOSMA_EINVAL, "ObjectiveContext: zeta must be > 0");
  if (n_classes < 1 || classes == nullptr)
    return set_error(GOSMA_EINVAL, "ObjectiveContext: no semantic classes");
  const bool single = (flags & GOSMA_CTX_SINGLE_MIXTURE) != 0;
  if (single && n_classes != 1)
    return set_error(GOSMA_EINVAL, "GOSMA_CTX_SINGLE_MIXTURE needs exactly one class");
  if (!single) {
    double wsum = 0.0;
    for (int c = 0; c < n_classes; ++c) wsum += classes[c].class_weight;
    if (!weights_close(wsum))
      return set_error(GOSMA_EINVAL, "ObjectiveContext class weights: weights sum to " +
                                         std::to_string(wsum) + ", expected 1");
  }
  HostModel hm;
  hm.zeta = zeta;
  for (int c = 0; c < n_classes; ++c) {
    const gosma_class_view& v = classes[c];
    if (v.n1 < 1 || v.n2 < 1)
      return set_error(GOSMA_EINVAL, "ObjectiveContext: class with empty mixture");
    HostClass hc;
    hc.weight = single ? 1.0 : v.class_weight;
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < v.n1; ++i) {
      if (!(v.sigma2[i] > 0.0) || !std::isfinite(v.sigma2[i]))
        return set_error(GOSMA_EINVAL, "IsotropicGaussian: variance must be positive");
      if (!(v.phi1[i] >= 0.0) || !std::isfinite(v.phi1[i]))
        return set_error(GOSMA_EINVAL, "IsotropicGaussian: weight must be non-negative");
      for (int a = 0; a < 3; ++a) hc.mu.push_back(v.mu[3 * i + a]);
      hc.sigma2.push_back(v.sigma2[i]);
      hc.phi1.push_back(v.phi1[i]);
      hm.all_means.emplace_back(v.mu[3 * i], v.mu[3 * i + 1], v.mu[3 * i + 2]);
      s1 += v.phi1[i];
    }
    for (int j = 0; j < v.n2; ++j) {
      const Vec3 d(v.dir[3 * j], v.dir[3 * j + 1], v.dir[3 * j + 2]);
      const double n = d.norm();
      if (!(std::fabs(n - 1.0) <= 1e-6))
        return set_error(GOSMA_EINVAL, "UnitVector3: input norm deviates from 1 by more than 1e-6");
      if (!(v.kappa2[j] > 0.0) || !std::isfinite(v.kappa2[j]))
        return set_error(GOSMA_EINVAL, "VmfComponent: concentration must be positive");
      if (!(v.phi2[j] >= 0.0) || !std::isfinite(v.phi2[j]))
        return set_error(GOSMA_EINVAL, "VmfComponent: weight must be non-negative");
      const Vec3 u = d / n;  // UnitVector3 renormalises (unit_vector.hpp:23)
      for (int a = 0; a < 3; ++a) hc.b.push_back(v.kappa2[j] * u[a]);
      hc.kappa2.push_back(v.kappa2[j]);
      hc.log_z2.push_back(log_z_eval(v.kappa2[j]));
      hc.phi2.push_back(v.phi2[j]);
      s2 += v.phi2[j];
    }
    if (!weights_close(s1))
      return set_error(GOSMA_EINVAL, "ObjectiveContext model: weights sum to " +
                                         std::to_string(s1) + ", expected 1");
    if (!weights_close(s2))
      return set_error(GOSMA_EINVAL, "ObjectiveContext image: weights sum to " +
                                         std::to_string(s2) + ", expected 1");
    hc.self_energy = class_self_energy(hc);
    hm.image_self_energy += hc.weight * hc.self_energy;
    hm.classes.push_back(std::move(hc));
  }
  *out = std::move(hm);
  return GOSMA_OK;
}

int ctx_from_model(int device, HostModel&& hm, gosma_ctx** out) {
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess) return cuda_error(e, "cudaGetDeviceCount");
  if (device < 0 || device >= ndev)
    return set_error(GOSMA_EINVAL, "device index " + std::to_string(device) + " out of range");
  auto* ctx = new gosma_ctx();
  ctx->device = device;
  ctx->model = std::move(hm);
  DeviceGuard g(device);
  cudaDeviceProp prop;
  if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) {
    delete ctx;
    return cuda_error(e, "cudaGetDeviceProperties");
  }
  ctx->sm_count = prop.multiProcessorCount;
  if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess) {
    delete ctx;
    return cuda_error(e, "cudaStreamCreate");
  }
  const int rc = ctx_upload(ctx);
  if (rc != GOSMA_OK) {
    ctx_free_device(ctx);
    delete ctx;
    return rc;
  }
  *out = ctx;
  return GOSMA_OK;
}

}  // namespace gosma

using namespace gosma;

extern "C" {

const char* gosma_last_error(void) { return g_last_error.c_str(); }

int gosma_ctx_create(int device, const gosma_class_view* classes, int n_classes, double zeta,
                     unsigned flags, gosma_ctx** out) {
  if (!out) return set_error(GOSMA_EINVAL, "out is null");
  *out = nullptr;
  HostModel hm;
  const int rc = validate_and_build(classes, n_classes, zeta, flags, &hm);
  if (rc != GOSMA_OK) return rc;
  return ctx_from_model(device, std::move(hm), out);
}

int gosma_ctx_blurred(const gosma_ctx* src, double w, double reference_distance,
                      gosma_ctx** out) {
  // ObjectiveContext::blurred (objective.cpp:70-101)
  if (!src || !out) return set_error(GOSMA_EINVAL, "null argument");
  if (!(w >= 0.0) || !(reference_distance >= 0.0))
    return set_error(GOSMA_EINVAL, "ObjectiveContext::blurred: negative width");
  HostModel hm = src->model;
  hm.image_self_energy = 0.0;
  const double var_add = (w * reference_distance) * (w * reference_distance);
  const double w2 = w * w;
  for (HostClass& c : hm.classes) {
    for (double& s2 : c.sigma2) s2 += var_add;
    for (int j = 0; j < c.n2(); ++j) {
      const Vec3 dir = Vec3(c.b[3 * j], c.b[3 * j + 1], c.b[3 * j + 2]) / c.kappa2[j];
      const double k = c.kappa2[j] / (1.0 + c.kappa2[j] * w2);
      c.kappa2[j] = k;
      for (int a = 0; a < 3; ++a) c.b[3 * j + a] = k * dir[a];
      c.log_z2[j] = log_z_eval(k);
    }
    c.self_energy = class_self_energy(c);
    hm.image_self_energy += c.weight * c.self_energy;
  }
  const int rc = ctx_from_model(src->device, std::move(hm), out);
  if (rc == GOSMA_OK) {
    (*out)->lb_margin = src->lb_margin;
    (*out)->dev.lb_margin = src->lb_margin;
    (*out)->dev.lb_err_scale = src->dev.lb_err_scale;
  }
  return rc;
}

void gosma_ctx_destroy(gosma_ctx* ctx) {
  if (!ctx) return;
  gosma_ctx_destroy(ctx->dive_ctx);
  ctx_free_device(ctx);
  delete ctx;
}

double gosma_ctx_image_self_energy(const gosma_ctx* ctx) {
  return ctx ? ctx->model.image_self_energy : NAN;
}

double gosma_ctx_zeta(const gosma_ctx* ctx) { return ctx ? ctx->model.zeta : NAN; }

int gosma_ctx_set_lb_margin(gosma_ctx* ctx, double rel) {
  if (!ctx || !(rel < 1e-2)) return set_error(GOSMA_EINVAL, "lb margin must be below 1e-2");
  if (rel < 0.0) {  // raw FP32 core: no error estimate, no floor (parity diagnostics)
    ctx->lb_margin = 0.0;
    ctx->dev.lb_margin = 0.0;
    ctx->dev.lb_err_scale = 0.0;
    return GOSMA_OK;
  }
  ctx->lb_margin = rel;
  ctx->dev.lb_margin = rel;
  ctx->dev.lb_err_scale = 1.0;
  return GOSMA_OK;
}

int gosma_eval_bounds_device(gosma_ctx* ctx, const gosma_node* d_nodes, size_t n, double skip,
                             double* d_lower, double* d_upper, int8_t* d_split, void* stream) {
  if (!ctx) return set_error(GOSMA_EINVAL, "null context");
  if (n == 0) return GOSMA_OK;
  if (!d_nodes || !d_lower || !d_upper) return set_error(GOSMA_EINVAL, "null buffer");
  DeviceGuard g(ctx->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  EvalArgs a;
  a.nodes = reinterpret_cast<const double*>(d_nodes);
  a.n = static_cast<long long>(n);
  a.skip_upper_at = skip;
  a.lower = d_lower;
  a.upper = d_upper;
  a.split_rot = d_split;
  a.work = work_counter(ctx, s);
  cudaError_t e = attach_redo(ctx, s, static_cast<long long>(n), &a);
  if (e == cudaSuccess) e = launch_eval_bounds(ctx->dev, a, ctx->sm_count, s);
  if (e != cudaSuccess) return cuda_error(e, "eval_bounds launch");
  return GOSMA_OK;
}

int gosma_eval_children_device(gosma_ctx* ctx, const gosma_node* d_parents, const int8_t* d_split,
                               size_t n, double skip, double* d_lower, double* d_upper,
                               int8_t* d_child_split, void* stream) {
  if (!ctx) return set_error(GOSMA_EINVAL, "null context");
  if (n == 0) return GOSMA_OK;
  if (!d_parents || !d_split || !d_lower || !d_upper) return set_error(GOSMA_EINVAL, "null buffer");
  DeviceGuard g(ctx->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  cudaError_t e;
  if (n > ctx->child_cap) {
    cudaFree(ctx->d_child_kids);
    cudaFree(ctx->d_child_lists);
    cudaFree(ctx->d_child_sel);
    ctx->d_child_kids = nullptr;
    ctx->d_child_lists = nullptr;
    ctx->d_child_sel = nullptr;
    ctx->child_cap = 0;  // stays 0 unless every allocation below succeeds
    if ((e = cudaMalloc(&ctx->d_child_kids, 8 * n * sizeof(gosma_node))) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_child_lists, 9 * n * sizeof(int) + 32)) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_child_sel, n * sizeof(unsigned int))) != cudaSuccess)
      return cuda_error(e, "children alloc");
    ctx->child_cap = n;
  }
  int* rot = ctx->d_child_lists;
  int* trans = rot + n;
  // the two counts (8-byte aligned after the lists) stay on the device: the
  // kernels read them (grids sized for the upper bounds), no host round trip
  auto* counts = reinterpret_cast<unsigned long long*>(
      (reinterpret_cast<uintptr_t>(trans + 8 * n) + 7) & ~uintptr_t(7));
  if ((e = make_children(d_parents, d_split, n, ctx->d_child_kids, rot, trans, counts,
                         ctx->d_child_sel, s)) != cudaSuccess)
    return cuda_error(e, "children");
  EvalArgs a;
  a.skip_upper_at = skip;
  a.lower = d_lower;
  a.upper = d_upper;
  a.split_rot = d_child_split;
  a.work = work_counter(ctx, s);
  if ((e = attach_redo(ctx, s, static_cast<long long>(8 * n), &a)) != cudaSuccess)
    return cuda_error(e, "redo list");
  EvalArgs b = a;
  b.nodes = reinterpret_cast<const double*>(d_parents);
  b.n = static_cast<long long>(n);
  b.n_dev = reinterpret_cast<const long long*>(counts);
  b.item_index = rot;
  b.sel = ctx->d_child_sel;
  if ((e = launch_eval_siblings(ctx->dev, b, ctx->sm_count, s)) != cudaSuccess)
    return cuda_error(e, "siblings kernel");
  EvalArgs c = a;
  c.nodes = reinterpret_cast<const double*>(ctx->d_child_kids);
  c.n = static_cast<long long>(8 * n);
  c.n_dev = reinterpret_cast<const long long*>(counts + 1);
  c.item_index = trans;
  if ((e = launch_eval_bounds(ctx->dev, c, ctx->sm_count, s)) != cudaSuccess)
    return cuda_error(e, "children kernel");
  return GOSMA_OK;
}

int gosma_eval_bounds_cached_device(gosma_ctx* ctx, const gosma_node* d_nodes, size_t n,
                                    const int32_t* d_tindex, const double* d_tboxes,
                                    size_t n_tboxes, double skip, double* d_lower,
                                    double* d_upper, int8_t* d_split, void* stream) {
  if (!ctx) return set_error(GOSMA_EINVAL, "null context");
  if (n == 0) return GOSMA_OK;
  if (!d_nodes || !d_tindex || !d_tboxes || !d_lower || !d_upper || n_tboxes == 0)
    return set_error(GOSMA_EINVAL, "null buffer");
  DeviceGuard g(ctx->device);
  cudaStream_t s = stream ? static_cast<cudaStream_t>(stream) : ctx->stream;
  cudaError_t e;
  if (n_tboxes > ctx->cache_cap) {
    cudaFree(ctx->d_cache_nodes);
    cudaFree(ctx->d_cache_self);
    ctx->d_cache_nodes = nullptr;
    ctx->d_cache_self = nullptr;
    ctx->cache_cap = 0;  // stays 0 unless both allocations below succeed
    if ((e = cudaMalloc(&ctx->d_cache_nodes, n_tboxes * sizeof(gosma_node))) != cudaSuccess ||
        (e = cudaMalloc(&ctx->d_cache_self, n_tboxes * 4 * sizeof(double))) != cudaSuccess)
      return cuda_error(e, "cache alloc");
    ctx->cache_cap = n_tboxes;
  }
  if ((e = boxes_as_nodes(d_tboxes, n_tboxes, ctx->d_cache_nodes, s)) != cudaSuccess)
    return cuda_error(e, "boxes");
  EvalArgs a;
  a.nodes = reinterpret_cast<const double*>(ctx->d_cache_nodes);
  a.n = static_cast<long long>(n_tboxes);
  a.skip_upper_at = skip;
  a.lower = nullptr;
  a.upper = nullptr;
  a.split_rot = nullptr;
  a.work = work_counter(ctx, s);
  a.self_out = ctx->d_cache_self;
  if ((e = launch_eval_self(ctx->dev, a, ctx->sm_count, s)) != cudaSuccess)
    return cuda_error(e, "self kernel");
  a.nodes = reinterpret_cast<const double*>(d_nodes);
  a.n = static_cast<long long>(n);
  a.lower = d_lower;
  a.upper = d_upper;
  a.split_rot = d_split;
  a.tindex = d_tindex;
  if ((e = attach_redo(ctx, s, static_cast<long long>(n), &a)) != cudaSuccess)
    return cuda_error(e, "redo list");
  if ((e = launch_eval_cross_cached(ctx->dev, a, ctx->sm_count, s)) != cudaSuccess)
    return cuda_error(e, "cross kernel");
  return GOSMA_OK;
}

int gosma_eval_bounds(gosma_ctx* ctx, const gosma_node* nodes, size_t n, double skip,
                      double* lower, double* upper, int8_t* split_rot) {
  if (!ctx) return set_error(GOSMA_EINVAL, "null context");
  if (n == 0) return GOSMA_OK;
  if (!nodes || !lower || !upper) return set_error(GOSMA_EINVAL, "null buffer");
  DeviceGuard g(ctx->device);
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaError_t e;
  // Three-stream pipeline over two device slots: H2D of chunk k+1 (copy-in
  // stream) and D2H of chunk k-1 (copy-out stream) overlap the bound kernel on
  // chunk k (compute stream). Overlap needs pinned host buffers; pageable ones
  // still work (the copies then serialise).
  // chunk of 2^19 nodes (46 MB of nodes per slot): 1M-node batches run
  // 64k, 128k, 256k, 512k chunks; e2e 8.22e7 (2^17) -> 8.40e7 (2^19) ->
  // 8.33e7 (2^20) bounds/s on the configs[1] batch. GOSMA_CHUNK_LOG2 (A/B).
  static const int chunk_log2 = [] {
    const char* e = std::getenv("GOSMA_CHUNK_LOG2");
    const int v = e ? std::atoi(e) : 19;
    return v >= 12 && v <= 24 ? v : 19;
  }();
  const size_t chunk = std::min<size_t>(n, static_cast<size_t>(1) << chunk_log2);
  if ((e = ctx->scratch.reserve(2 * chunk)) != cudaSuccess) return cuda_error(e, "scratch");
  constexpr size_t kSmall = 8192;
  if (n <= kSmall) {
    // a small batch (the discovery dive's beam): one stream, no cross-stream
    // events (their latency would dominate), staged through pinned memory
    // (pageable copies go through the driver's own staging, ~10 us each)
    constexpr size_t kRec = sizeof(gosma_node) + 2 * sizeof(double) + 1;
    if (!ctx->scratch.h_pinned &&
        (e = cudaMallocHost(&ctx->scratch.h_pinned, kSmall * kRec)) != cudaSuccess)
      return cuda_error(e, "pinned staging");
    auto* hn = static_cast<gosma_node*>(ctx->scratch.h_pinned);
    auto* hl = reinterpret_cast<double*>(hn + kSmall);
    double* hu = hl + kSmall;
    auto* hs = reinterpret_cast<int8_t*>(hu + kSmall);
    std::memcpy(hn, nodes, n * sizeof(gosma_node));
    cudaStream_t ks = ctx->stream;
    if ((e = cudaMemcpyAsync(ctx->scratch.d_nodes, hn, n * sizeof(gosma_node),
                             cudaMemcpyHostToDevice, ks)) != cudaSuccess)
      return cuda_error(e, "H2D nodes");
    int8_t* dsp = split_rot ? ctx->scratch.d_split : nullptr;
    const int rc = gosma_eval_bounds_device(ctx, ctx->scratch.d_nodes, n, skip,
                                            ctx->scratch.d_lower, ctx->scratch.d_upper, dsp, ks);
    if (rc != GOSMA_OK) return rc;
    if ((e = cudaMemcpyAsync(hl, ctx->scratch.d_lower, n * sizeof(double),
                             cudaMemcpyDeviceToHost, ks)) != cudaSuccess ||
        (e = cudaMemcpyAsync(hu, ctx->scratch.d_upper, n * sizeof(double),
                             cudaMemcpyDeviceToHost, ks)) != cudaSuccess ||
        (split_rot && (e = cudaMemcpyAsync(hs, dsp, n * sizeof(int8_t), cudaMemcpyDeviceToHost,
                                           ks)) != cudaSuccess))
      return cuda_error(e, "D2H bounds");
    if ((e = cudaStreamSynchronize(ks)) != cudaSuccess) return cuda_error(e, "eval_bounds");
    std::memcpy(lower, hl, n * sizeof(double));
    std::memcpy(upper, hu, n * sizeof(double));
    if (split_rot) std::memcpy(split_rot, hs, n * sizeof(int8_t));
    return GOSMA_OK;
  }
  if (!ctx->h2d_stream) {
    if ((e = cudaStreamCreateWithFlags(&ctx->h2d_stream, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->d2h_stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_error(e, "pipeline streams");
    for (cudaEvent_t& ev : ctx->pipe_ev)
      if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess)
        return cuda_error(e, "pipeline events");
  }
  cudaStream_t ks = ctx->stream, hs = ctx->h2d_stream, ds = ctx->d2h_stream;
  cudaEvent_t* h2d_done = ctx->pipe_ev;      // [slot]
  cudaEvent_t* k_done = ctx->pipe_ev + 2;    // [slot]
  cudaEvent_t* d2h_done = ctx->pipe_ev + 4;  // [slot]
  // the compute stream may hold earlier work on these slots
  if ((e = cudaEventRecord(k_done[0], ks)) != cudaSuccess) return cuda_error(e, "event");
  cudaEventRecord(k_done[1], ks);
  cudaEventRecord(d2h_done[0], ks);
  cudaEventRecord(d2h_done[1], ks);
  // chunk k covers [off[k], off[k+1]); the first chunks ramp up (chunk/8,
  // chunk/4, chunk/2) so the kernel starts after a short copy instead of a
  // full 11 MB one, then full chunks
  std::vector<size_t> offs{0};
  for (size_t c = std::max<size_t>(chunk / 8, 1); offs.back() < n; c = std::min(2 * c, chunk))
    offs.push_back(std::min(n, offs.back() + c));
  const size_t nchunks = offs.size() - 1;
  auto h2d = [&](size_t k) -> cudaError_t {
    const size_t off = offs[k], m = offs[k + 1] - offs[k], slot = k & 1;
    cudaStreamWaitEvent(hs, k_done[slot], 0);  // the kernel of chunk k-2 has read the slot
    cudaError_t err = cudaMemcpyAsync(ctx->scratch.d_nodes + slot * chunk, nodes + off,
                                      m * sizeof(gosma_node), cudaMemcpyHostToDevice, hs);
    if (err == cudaSuccess) err = cudaEventRecord(h2d_done[slot], hs);
    return err;
  };
  if ((e = h2d(0)) != cudaSuccess) return cuda_error(e, "H2D nodes");
  for (size_t k = 0; k < nchunks; ++k) {
    const size_t off = offs[k], m = offs[k + 1] - offs[k], slot = k & 1;
    if (k + 1 < nchunks && (e = h2d(k + 1)) != cudaSuccess) return cuda_error(e, "H2D nodes");
    cudaStreamWaitEvent(ks, h2d_done[slot], 0);
    cudaStreamWaitEvent(ks, d2h_done[slot], 0);  // chunk k-2's bounds have left the slot
    double* dl = ctx->scratch.d_lower + slot * chunk;
    double* du = ctx->scratch.d_upper + slot * chunk;
    int8_t* dsp = split_rot ? ctx->scratch.d_split + slot * chunk : nullptr;
    const int rc = gosma_eval_bounds_device(ctx, ctx->scratch.d_nodes + slot * chunk, m, skip,
                                            dl, du, dsp, ks);
    if (rc != GOSMA_OK) return rc;
    cudaEventRecord(k_done[slot], ks);
    cudaStreamWaitEvent(ds, k_done[slot], 0);
    if ((e = cudaMemcpyAsync(lower + off, dl, m * sizeof(double), cudaMemcpyDeviceToHost, ds)) !=
            cudaSuccess ||
        (e = cudaMemcpyAsync(upper + off, du, m * sizeof(double), cudaMemcpyDeviceToHost, ds)) !=
            cudaSuccess)
      return cuda_error(e, "D2H bounds");
    if (split_rot && (e = cudaMemcpyAsync(split_rot + off, dsp, m * sizeof(int8_t),
                                          cudaMemcpyDeviceToHost, ds)) != cudaSuccess)
      return cuda_error(e, "D2H split");
    cudaEventRecord(d2h_done[slot], ds);
  }
  if ((e = cudaStreamSynchronize(ds)) != cudaSuccess) return cuda_error(e, "eval_bounds");
  if ((e = cudaStreamSynchronize(ks)) != cudaSuccess) return cuda_error(e, "eval_bounds");
  return GOSMA_OK;
}

int gosma_objective_value(const gosma_ctx* ctx, const double r[3], const double t[3],
                          double* value) {
  if (!ctx || !r || !t || !value) return set_error(GOSMA_EINVAL, "null argument");
  const Vec3 tv(t[0], t[1], t[2]);
  if (!pose_feasible(ctx->model, tv))
    return set_error(GOSMA_EINFEASIBLE, "pose within zeta of a component mean");
  *value = objective_value(ctx->model, Vec3(r[0], r[1], r[2]), tv);
  return GOSMA_OK;
}

int gosma_objective_gradient(const gosma_ctx* ctx, const double r[3], const double t[3],
                             double g[6]) {
  if (!ctx || !r || !t || !g) return set_error(GOSMA_EINVAL, "null argument");
  if (!objective_gradient(ctx->model, Vec3(r[0], r[1], r[2]), Vec3(t[0], t[1], t[2]), g))
    return set_error(GOSMA_EINFEASIBLE, "pose within zeta of a component mean");
  return GOSMA_OK;
}

int gosma_device_info(int device, int* sm_count, int* sm_clock_khz, int* cc_major,
                      int* cc_minor) {
  cudaDeviceProp p;
  const cudaError_t e = cudaGetDeviceProperties(&p, device);
  if (e != cudaSuccess) return cuda_error(e, "cudaGetDeviceProperties");
  if (sm_count) *sm_count = p.multiProcessorCount;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
  if (sm_clock_khz) *sm_clock_khz = clk;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return GOSMA_OK;
}

unsigned long long gosma_kernel_launches(void) { return bound_kernel_launch_count(); }

}  // extern "C"
