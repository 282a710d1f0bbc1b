// Batched FP64 objective / gradient on the GPU for the local refiner (K6,
// objective_kernel.cu) and the host-side batcher that lets many L-BFGS starts
// (one host thread each) share kernel launches.
#pragma once

#include <cuda_runtime.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "gosma_internal.hpp"
#include "host_math.hpp"

namespace gosma {

// Device copy of one HostModel (FP64; pooled classes, objective.hpp:19-31).
struct DevModel64 {
  int n_classes, n_all, max_n1;
  const ClassSpan* cls;
  const double* cls_w;
  const double* mu;      // 3*N1
  const double* sigma2;  // N1
  const double* phi1;    // N1
  const double* b;       // 3*N2, kappa * direction
  const double* kappa2;  // N2
  const double* log_z2;  // N2
  const double* phi2;    // N2
  const double* all_means;  // 3*n_all (check_feasible)
  double zeta;
};

struct ObjRequest {
  double x[6];  // r[3], t[3]
  int model;    // index into the model table
  int pad;
};

size_t objgrad_smem_bytes(int max_n1);
int objgrad_slices(int max_pairs_per_row);
// partial: n * slices * 7 doubles ({f, g[6]} per request and partner slice)
cudaError_t launch_objgrad(const DevModel64* models, const ObjRequest* req, int n, int slices,
                           double* partial, int max_n1, cudaStream_t s);

// Owns device copies of a set of models and evaluates batches of requests.
// evaluate() is synchronous; BatchGate lets host threads pool their requests.
class DeviceObjective {
 public:
  DeviceObjective(int device, const std::vector<const HostModel*>& models);
  ~DeviceObjective();
  bool ok() const { return ok_; }
  // f[k], g[6k] for requests[k]; f = +inf and g = 0 for infeasible poses.
  cudaError_t evaluate(const std::vector<ObjRequest>& requests, std::vector<double>* f,
                       std::vector<double>* g);

 private:
  int device_ = 0, sm_count_ = 1, max_n1_ = 1, slices_ = 1;
  bool ok_ = false;
  std::vector<void*> owned_;
  DevModel64* d_models_ = nullptr;
  ObjRequest* d_req_ = nullptr;
  double* d_part_ = nullptr;
  size_t cap_ = 0;
  cudaStream_t stream_ = nullptr;
};

// Collects one request per participating thread and launches when every
// active participant is waiting (deterministic per request: results depend
// only on the pose and the model).
class BatchGate {
 public:
  explicit BatchGate(DeviceObjective* dev, int participants)
      : dev_(dev), active_(participants) {}
  // Blocks until the batch containing this request has been evaluated.
  void eval(const ObjRequest& r, double* f, double g[6]);
  // A participant that will make no more requests.
  void leave();

 private:
  void launch_locked(std::unique_lock<std::mutex>& lk);
  DeviceObjective* dev_;
  std::mutex mu_;
  std::condition_variable cv_;
  int active_;
  unsigned long long generation_ = 0;
  std::vector<ObjRequest> pending_;
  std::vector<double*> f_out_;
  std::vector<double*> g_out_;
};

}  // namespace gosma
