// Host side of the batched FP64 objective (objective_device.hpp).
#include "objective_device.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace gosma {

namespace {

template <typename T>
cudaError_t upload_vec(const std::vector<T>& h, const T** d, std::vector<void*>* owned) {
  *d = nullptr;
  if (h.empty()) return cudaSuccess;
  T* p = nullptr;
  cudaError_t e = cudaMalloc(&p, h.size() * sizeof(T));
  if (e != cudaSuccess) return e;
  owned->push_back(p);
  *d = p;
  return cudaMemcpy(p, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice);
}

}  // namespace

DeviceObjective::DeviceObjective(int device, const std::vector<const HostModel*>& models)
    : device_(device) {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device_);
  cudaDeviceGetAttribute(&sm_count_, cudaDevAttrMultiProcessorCount, device_);
  std::vector<DevModel64> dm;
  cudaError_t e = cudaSuccess;
  for (const HostModel* hm : models) {
    std::vector<ClassSpan> spans;
    std::vector<double> cw, mu, s2, p1, b, k2, lz2, p2, all;
    int o1 = 0, o2 = 0, mx = 1, mp = 1;
    size_t pairs = 0;
    for (const HostClass& c : hm->classes) {
      spans.push_back({o1, c.n1(), o2, c.n2()});
      cw.push_back(c.weight);
      mx = std::max(mx, c.n1());
      mp = std::max(mp, c.n1() + c.n2());
      pairs += static_cast<size_t>(c.n1()) * (c.n1() + c.n2());
      mu.insert(mu.end(), c.mu.begin(), c.mu.end());
      s2.insert(s2.end(), c.sigma2.begin(), c.sigma2.end());
      p1.insert(p1.end(), c.phi1.begin(), c.phi1.end());
      b.insert(b.end(), c.b.begin(), c.b.end());
      k2.insert(k2.end(), c.kappa2.begin(), c.kappa2.end());
      lz2.insert(lz2.end(), c.log_z2.begin(), c.log_z2.end());
      p2.insert(p2.end(), c.phi2.begin(), c.phi2.end());
      o1 += c.n1();
      o2 += c.n2();
    }
    for (const Vec3& v : hm->all_means)
      for (int a = 0; a < 3; ++a) all.push_back(v[a]);
    DevModel64 d{};
    d.n_classes = static_cast<int>(spans.size());
    d.n_all = static_cast<int>(hm->all_means.size());
    d.max_n1 = mx;
    d.zeta = hm->zeta;
    max_n1_ = std::max(max_n1_, mx);
    max_pairs_ = std::max(max_pairs_, pairs);
    slices_ = std::max(slices_, objgrad_slices(mp));
    const ClassSpan* dspans = nullptr;
    if (e == cudaSuccess) e = upload_vec(spans, &dspans, &owned_);
    d.cls = dspans;
    if (e == cudaSuccess) e = upload_vec(cw, &d.cls_w, &owned_);
    if (e == cudaSuccess) e = upload_vec(mu, &d.mu, &owned_);
    if (e == cudaSuccess) e = upload_vec(s2, &d.sigma2, &owned_);
    if (e == cudaSuccess) e = upload_vec(p1, &d.phi1, &owned_);
    if (e == cudaSuccess) e = upload_vec(b, &d.b, &owned_);
    if (e == cudaSuccess) e = upload_vec(k2, &d.kappa2, &owned_);
    if (e == cudaSuccess) e = upload_vec(lz2, &d.log_z2, &owned_);
    if (e == cudaSuccess) e = upload_vec(p2, &d.phi2, &owned_);
    if (e == cudaSuccess) e = upload_vec(all, &d.all_means, &owned_);
    dm.push_back(d);
  }
  const DevModel64* dmp = nullptr;
  if (e == cudaSuccess) e = upload_vec(dm, &dmp, &owned_);
  d_models_ = const_cast<DevModel64*>(dmp);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking);
  int max_optin = 0;
  cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device_);
  ok_ = e == cudaSuccess && objgrad_smem_bytes(max_n1_) <= static_cast<size_t>(max_optin);
  cudaSetDevice(cur);
}

DeviceObjective::~DeviceObjective() {
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device_);
  for (void* p : owned_) cudaFree(p);
  cudaFree(d_req_);
  cudaFree(d_part_);
  cudaFree(d_jobs_);
  cudaFree(d_out_);
  cudaFree(d_boxes_);
  if (stream_) cudaStreamDestroy(stream_);
  cudaSetDevice(cur);
}

cudaError_t DeviceObjective::evaluate(const std::vector<ObjRequest>& requests,
                                      std::vector<double>* f, std::vector<double>* g) {
  const size_t n = requests.size();
  f->assign(n, INFINITY);
  g->assign(6 * n, 0.0);
  if (n == 0) return cudaSuccess;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device_);
  cudaError_t e = cudaSuccess;
  if (n > cap_) {
    cudaFree(d_req_);
    cudaFree(d_part_);
    d_req_ = nullptr;
    d_part_ = nullptr;
    const size_t c = std::max<size_t>(n, 64);
    if ((e = cudaMalloc(&d_req_, c * sizeof(ObjRequest))) == cudaSuccess)
      e = cudaMalloc(&d_part_, c * slices_ * 7 * sizeof(double));
    cap_ = e == cudaSuccess ? c : 0;
  }
  std::vector<double> part(n * slices_ * 7);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_req_, requests.data(), n * sizeof(ObjRequest), cudaMemcpyHostToDevice,
                        stream_);
  if (e == cudaSuccess)
    e = launch_objgrad(d_models_, d_req_, static_cast<int>(n), slices_, d_part_, max_n1_,
                       stream_);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(part.data(), d_part_, part.size() * sizeof(double),
                        cudaMemcpyDeviceToHost, stream_);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream_);
  if (e == cudaSuccess) {
    // ordered sum over the slices (deterministic)
    for (size_t k = 0; k < n; ++k) {
      double acc[7] = {0, 0, 0, 0, 0, 0, 0};
      for (int sl = 0; sl < slices_; ++sl)
        for (int a = 0; a < 7; ++a) acc[a] += part[(k * slices_ + sl) * 7 + a];
      (*f)[k] = acc[0];
      for (int a = 0; a < 6; ++a) (*g)[6 * k + a] = std::isinf(acc[0]) ? 0.0 : acc[1 + a];
    }
  }
  if (e != cudaSuccess) {
    f->assign(n, INFINITY);
    g->assign(6 * n, 0.0);
  }
  cudaSetDevice(cur);
  return e;
}

cudaError_t DeviceObjective::refine(const std::vector<RefineJob>& jobs, const double rc[3],
                                    double rhw, const std::vector<double>& boxes,
                                    std::vector<RefineOut>* out) {
  out->assign(jobs.size(), RefineOut{INFINITY, {0, 0, 0, 0, 0, 0}, 0});
  if (jobs.empty()) return cudaSuccess;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(device_);
  // persistent buffers (grown on demand): refinements run once per improving
  // wave, so per-call cudaMalloc / cudaFree (a device sync each) would show
  cudaError_t e = cudaSuccess;
  if (jobs.size() > job_cap_) {
    cudaFree(d_jobs_);
    cudaFree(d_out_);
    d_jobs_ = nullptr;
    d_out_ = nullptr;
    const size_t c = std::max<size_t>(jobs.size(), 64);
    if ((e = cudaMalloc(&d_jobs_, c * sizeof(RefineJob))) == cudaSuccess)
      e = cudaMalloc(&d_out_, c * sizeof(RefineOut));
    job_cap_ = e == cudaSuccess ? c : 0;
  }
  if (e == cudaSuccess && boxes.size() > box_cap_) {
    cudaFree(d_boxes_);
    d_boxes_ = nullptr;
    if ((e = cudaMalloc(&d_boxes_, boxes.size() * sizeof(double))) == cudaSuccess)
      box_cap_ = boxes.size();
    else
      box_cap_ = 0;
  }
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_jobs_, jobs.data(), jobs.size() * sizeof(RefineJob),
                        cudaMemcpyHostToDevice, stream_);
  if (e == cudaSuccess && !boxes.empty())
    e = cudaMemcpyAsync(d_boxes_, boxes.data(), boxes.size() * 8, cudaMemcpyHostToDevice,
                        stream_);
  RefineDomain dom{{rc[0], rc[1], rc[2]}, rhw, static_cast<int>(boxes.size() / 6), d_boxes_};
  // spread each start over a cluster of CTAs when the GPU has SMs to spare
  // and an evaluation is big enough to amortise the cluster exchange
  const int n = static_cast<int>(jobs.size());
  // (GOSMA_REFINE_CLUSTER=c forces c, for A/B measurements)
  static const int forced = [] {
    const char* v = std::getenv("GOSMA_REFINE_CLUSTER");
    return v ? std::atoi(v) : 0;
  }();
  const int cluster = forced > 0 ? forced
                                 : (max_pairs_ >= 8192 ? std::max(1, std::min(8, sm_count_ / n)) : 1);
  cudaEvent_t ev[2] = {nullptr, nullptr};
  const bool prof = n > 1 && std::getenv("GOSMA_PROFILE") != nullptr;  // batches only
  if (prof) {
    cudaEventCreate(&ev[0]);
    cudaEventCreate(&ev[1]);
    cudaEventRecord(ev[0], stream_);
  }
  if (e == cudaSuccess)
    e = launch_refine(d_models_, d_jobs_, n, dom, d_out_, max_n1_, cluster, stream_);
  if (prof) cudaEventRecord(ev[1], stream_);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(out->data(), d_out_, jobs.size() * sizeof(RefineOut),
                        cudaMemcpyDeviceToHost, stream_);
  if (e == cudaSuccess) e = cudaStreamSynchronize(stream_);
  if (prof) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev[0], ev[1]);
    long long tot = 0, mx = 0;
    for (const RefineOut& o : *out) {
      tot += o.evals;
      mx = std::max(mx, o.evals);
    }
    std::fprintf(stderr,
                 "[gosma profile] refine kernel: %d jobs x %d CTAs %.3f ms, evals %lld (max %lld "
                 "per job, %.2f us each)\n",
                 n, cluster, ms, tot, mx, mx ? 1e3 * ms / mx : 0.0);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
  }
  cudaSetDevice(cur);
  return e;
}

}  // namespace gosma
