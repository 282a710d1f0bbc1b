// Batched FP64 objective / gradient on the GPU (K6, objective_kernel.cu) and
// the GPU-resident local refiner built on it (one CTA per L-BFGS start).
#pragma once

#include <cuda_runtime.h>

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

// GPU-resident local refinement: one CTA per job runs the L-BFGS ladder
// (up to 4 stages, each on its own model) from x; the domain's boxes are a
// device array of 6 doubles per box.
struct RefineJob {
  double x[6];
  int stages;
  int model[4];
};
struct RefineDomain {
  double rc[3];
  double rhw;
  int n_boxes;
  const double* boxes;
};
struct RefineOut {
  double value;
  double x[6];
  long long evals;  // objective + gradient evaluations the job made
};
// cluster: CTAs per job (1..8), each taking a slice of every evaluation's
// partners (results depend on it in the last bits, deterministically).
cudaError_t launch_refine(const DevModel64* models, const RefineJob* jobs, int n,
                          const RefineDomain& dom, RefineOut* out, int max_n1, int cluster,
                          cudaStream_t s);

size_t objgrad_smem_bytes(int max_n1);
int objgrad_slices(int max_pairs_per_row);
// partial: n * slices * 7 doubles ({f, g[6]} per request and partner slice)
cudaError_t launch_objgrad(const DevModel64* models, const ObjRequest* req, int n, int slices,
                           double* partial, int max_n1, cudaStream_t s);

// Owns device copies of a set of models and evaluates batches of requests.
// evaluate() and refine() are synchronous.
class DeviceObjective {
 public:
  DeviceObjective(int device, const std::vector<const HostModel*>& models);
  ~DeviceObjective();
  bool ok() const { return ok_; }
  // f[k], g[6k] for requests[k]; f = +inf and g = 0 for infeasible poses.
  cudaError_t evaluate(const std::vector<ObjRequest>& requests, std::vector<double>* f,
                       std::vector<double>* g);
  // runs the refinement jobs on the GPU (one CTA each); boxes: 6 doubles per box
  cudaError_t refine(const std::vector<RefineJob>& jobs, const double rc[3], double rhw,
                     const std::vector<double>& boxes, std::vector<RefineOut>* out);

 private:
  int device_ = 0, sm_count_ = 1, max_n1_ = 1, slices_ = 1;
  size_t max_pairs_ = 0;  // largest model's pair terms per evaluation
  bool ok_ = false;
  std::vector<void*> owned_;
  DevModel64* d_models_ = nullptr;
  ObjRequest* d_req_ = nullptr;
  double* d_part_ = nullptr;
  size_t cap_ = 0;
  RefineJob* d_jobs_ = nullptr;
  RefineOut* d_out_ = nullptr;
  double* d_boxes_ = nullptr;
  size_t job_cap_ = 0, box_cap_ = 0;
  cudaStream_t stream_ = nullptr;
};

}  // namespace gosma
