// GPU scoring for DP-means / DP-vMF-means at scale (the
// paper's 100k-point real-data setting).
//
// The reference's assignment sweep (core/src/mixtures.cpp:68-88, 132-152)
// visits points in order and may open a new centre at any point, so the
// sweep looks sequential. Its cost is not: every point scans all centres
// (O(n k) distances per sweep) and every centre that existed when the sweep
// began is fixed for the whole sweep (means move only after it). The engine
// in mixtures.cpp therefore splits a sweep into
//   (1) a GPU pass scoring every point against the centres fixed at the
//       sweep's start (this file: exact FP64, the reference's operation order,
//       first-minimum tie rule), and
//   (2) an admission pass in visit order that only scores the centres opened
//       during this sweep; it runs in blocks of visit order, each block's
//       points first scored on the GPU against the centres opened before the
//       block, so the host only compares against centres opened inside the
//       block.
// The result is bit-identical to the sequential sweep.
#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "dp_cluster.hpp"

namespace gosma {
namespace mix {

namespace {

constexpr int kTile = 512;  // centres per shared-memory tile

// score of point p against centre c: squared distance (metric 0) or negated
// cosine (metric 1) - lower is better; the reference's operation order
// (Vector3d subtraction then x*x + y*y + z*z; dot = x*x' + y*y' + z*z'),
// no FMA contraction.
__device__ __forceinline__ double score(int metric, double px, double py, double pz, double cx,
                                        double cy, double cz) {
  if (metric == 0) {
    const double dx = __dsub_rn(px, cx), dy = __dsub_rn(py, cy), dz = __dsub_rn(pz, cz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  }
  return -__dadd_rn(__dadd_rn(__dmul_rn(px, cx), __dmul_rn(py, cy)), __dmul_rn(pz, cz));
}

// Points idx[0..m) (all points when idx is null) against centres [c0, c1):
// the first strictly-lower score wins, continuing the running best when
// `merge` (centres c0.. come after every centre already scored).
__global__ void score_kernel(const double* __restrict__ pts, const int* __restrict__ idx,
                             int m, const double* __restrict__ centres, int c0, int c1,
                             int metric, bool merge, double* best_score, int* best_idx) {
  __shared__ double sc[3 * kTile];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < m;
  const int p = live ? (idx ? idx[t] : t) : 0;
  double px = 0.0, py = 0.0, pz = 0.0;
  if (live) {
    px = pts[3 * p];
    py = pts[3 * p + 1];
    pz = pts[3 * p + 2];
  }
  double best = INFINITY;
  int bi = -1;
  if (live && merge) {
    best = best_score[t];
    bi = best_idx[t];
  }
  for (int base = c0; base < c1; base += kTile) {
    const int nt = min(kTile, c1 - base);
    __syncthreads();
    for (int k = threadIdx.x; k < 3 * nt; k += blockDim.x) sc[k] = centres[3 * base + k];
    __syncthreads();
    if (!live) continue;
    for (int k = 0; k < nt; ++k) {
      const double s = score(metric, px, py, pz, sc[3 * k], sc[3 * k + 1], sc[3 * k + 2]);
      if (bi < 0 || s < best) {
        best = s;
        bi = base + k;
      }
    }
  }
  if (live) {
    best_score[t] = best;
    best_idx[t] = bi;
  }
}

template <typename T>
cudaError_t grow(T** p, size_t* cap, size_t need) {
  if (need <= *cap) return cudaSuccess;
  cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  const size_t c = need + need / 2;
  const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), c * sizeof(T));
  if (e == cudaSuccess) *cap = c;
  return e;
}

}  // namespace

struct DeviceScorer::Impl {
  int device = 0;
  cudaStream_t s = nullptr;
  double* pts = nullptr;
  double* centres = nullptr;
  double* best = nullptr;
  int* bidx = nullptr;
  int* idx = nullptr;
  size_t n = 0, cap_c = 0, cap_b = 0, cap_i = 0, cap_i2 = 0;
};

DeviceScorer::DeviceScorer() = default;

DeviceScorer::~DeviceScorer() {
  if (!d_) return;
  int cur = 0;
  cudaGetDevice(&cur);
  cudaSetDevice(d_->device);
  cudaFree(d_->pts);
  cudaFree(d_->centres);
  cudaFree(d_->best);
  cudaFree(d_->bidx);
  cudaFree(d_->idx);
  if (d_->s) cudaStreamDestroy(d_->s);
  cudaSetDevice(cur);
}

bool DeviceScorer::open(const std::vector<Vec3>& points, int device) {
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) return false;
  d_ = std::make_unique<Impl>();
  d_->device = device;
  d_->n = points.size();
  cudaSetDevice(device);
  if (cudaStreamCreateWithFlags(&d_->s, cudaStreamNonBlocking) != cudaSuccess) return false;
  std::vector<double> flat(3 * points.size());
  for (size_t i = 0; i < points.size(); ++i)
    for (int a = 0; a < 3; ++a) flat[3 * i + a] = points[i][a];
  if (cudaMalloc(&d_->pts, flat.size() * sizeof(double)) != cudaSuccess) return false;
  return cudaMemcpy(d_->pts, flat.data(), flat.size() * sizeof(double),
                    cudaMemcpyHostToDevice) == cudaSuccess;
}

bool DeviceScorer::score(const std::vector<Vec3>& centres, size_t c0, size_t c1,
                         const std::vector<int>* subset, int metric, bool merge,
                         std::vector<double>* best, std::vector<int>* best_idx) {
  Impl& d = *d_;
  cudaSetDevice(d.device);
  const size_t m = subset ? subset->size() : d.n;
  if (m == 0) return true;
  std::vector<double> flat(3 * (c1 - c0));
  for (size_t c = c0; c < c1; ++c)
    for (int a = 0; a < 3; ++a) flat[3 * (c - c0) + a] = centres[c][a];
  if (grow(&d.centres, &d.cap_c, 3 * c1) != cudaSuccess || grow(&d.best, &d.cap_b, m) != cudaSuccess ||
      grow(&d.bidx, &d.cap_i, m) != cudaSuccess)
    return false;
  cudaError_t e = cudaSuccess;
  if (c1 > c0)
    e = cudaMemcpyAsync(d.centres + 3 * c0, flat.data(), flat.size() * sizeof(double),
                        cudaMemcpyHostToDevice, d.s);
  int* didx = nullptr;
  if (e == cudaSuccess && subset) {
    if (grow(&d.idx, &d.cap_i2, m) != cudaSuccess) return false;
    didx = d.idx;
    e = cudaMemcpyAsync(didx, subset->data(), m * sizeof(int), cudaMemcpyHostToDevice, d.s);
  }
  if (e == cudaSuccess && merge) {
    e = cudaMemcpyAsync(d.best, best->data(), m * sizeof(double), cudaMemcpyHostToDevice, d.s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(d.bidx, best_idx->data(), m * sizeof(int), cudaMemcpyHostToDevice, d.s);
  }
  if (e != cudaSuccess) return false;
  const int threads = 256;
  score_kernel<<<static_cast<unsigned>((m + threads - 1) / threads), threads, 0, d.s>>>(
      d.pts, didx, static_cast<int>(m), d.centres, static_cast<int>(c0), static_cast<int>(c1),
      metric, merge, d.best, d.bidx);
  best->resize(m);
  best_idx->resize(m);
  e = cudaMemcpyAsync(best->data(), d.best, m * sizeof(double), cudaMemcpyDeviceToHost, d.s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(best_idx->data(), d.bidx, m * sizeof(int), cudaMemcpyDeviceToHost, d.s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(d.s);
  return e == cudaSuccess && cudaGetLastError() == cudaSuccess;
}

}  // namespace mix
}  // namespace gosma
