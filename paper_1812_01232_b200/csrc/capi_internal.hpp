// The opaque gosma_ctx and helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "gosma_capi.h"
#include "gosma_internal.hpp"
#include "host_math.hpp"

namespace gosma {

// Reusable device buffers for the host-buffer entry point.
struct Scratch {
  gosma_node* d_nodes = nullptr;
  double* d_lower = nullptr;
  double* d_upper = nullptr;
  int8_t* d_split = nullptr;
  void* h_pinned = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t n);
  void release();
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// Default relative LB soundness margin (x |term| mass); see DESIGN.md.
constexpr double kDefaultLbMargin = 2e-7;

}  // namespace gosma

struct gosma_ctx {
  int device = 0;
  int sm_count = 0;
  gosma::HostModel model;
  gosma::DevCtx dev{};
  double lb_margin = gosma::kDefaultLbMargin;
  std::vector<void*> owned;
  void* d_work = nullptr;  // persistent-warp node counter of launches on `stream`
  // per caller stream: a node counter (the kernels' persistent warps claim
  // nodes from it; two launches in flight on different streams must not share
  // one) and the precise fix-up's redo list; work_counter() / attach_redo()
  // hand them out, ctx_free_device releases them
  struct StreamScratch {
    cudaStream_t stream = nullptr;
    void* work = nullptr;
    unsigned long long* redo_count = nullptr;
    double* redo_nodes = nullptr;
    long long* redo_slot = nullptr;
    long long redo_cap = 0;
  };
  std::vector<StreamScratch> work_slots;
  std::mutex work_mu;
  gosma_node* d_cache_nodes = nullptr;  // translation-cached mode scratch
  double* d_cache_self = nullptr;
  size_t cache_cap = 0;
  gosma_node* d_child_kids = nullptr;  // gosma_eval_children_device scratch
  int* d_child_lists = nullptr;
  unsigned int* d_child_sel = nullptr;
  size_t child_cap = 0;
  cudaStream_t stream = nullptr;
  // host-buffer pipeline (gosma_eval_bounds): copy-in / copy-out streams and
  // per-slot events (H2D done, kernel done, D2H done) x 2 slots
  cudaStream_t h2d_stream = nullptr, d2h_stream = nullptr;
  cudaEvent_t pipe_ev[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  gosma::Scratch scratch;
  std::mutex mu;
  // the discovery dive's blurred copy (solver.cpp:449-457), kept for the
  // next solve on this context (creating one costs device allocations)
  gosma_ctx* dive_ctx = nullptr;
  double dive_w = -1.0, dive_dist = -1.0;
  std::mutex dive_mu;
  // device beam of the dive run on this (blurred) context: one device block
  // and the captured two-iteration graph, reused while the sizes match
  void* dive_buf = nullptr;
  size_t dive_bytes = 0;
  int dive_sectors = 0, dive_quota = 0;
  cudaGraphExec_t dive_graph = nullptr;
};

namespace gosma {
// The node counter of bound-kernel launches on stream s (launches on one
// stream are ordered, so they may share it; other streams get their own).
unsigned int* work_counter(gosma_ctx* ctx, cudaStream_t s);
// Points a's redo list (precise fix-up) at the stream's buffers, grown to hold
// n_out entries (one per output slot, so it never overflows). Not during
// stream capture (it may allocate): captured callers leave it unset.
cudaError_t attach_redo(gosma_ctx* ctx, cudaStream_t s, long long n_out, EvalArgs* a);
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* where);
}  // namespace gosma
