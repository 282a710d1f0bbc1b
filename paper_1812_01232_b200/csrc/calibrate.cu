// On-box pipe-throughput microbenchmarks for the roofline denominators that
// MEASURED_PEAKS.json does not carry (it has HBM and bf16 tensor only):
// the SFU/XU pipe (MUFU ex2/rsqrt/rcp, the bound kernel's limiter) and the
// FP32 FMA pipe. Timed with CUDA events at whatever clock the GPU runs.
#include <cuda_runtime.h>

#include "capi_internal.hpp"

namespace {

__global__ void mufu_loop(float* out, int iters, float seed) {
  float a0 = seed + threadIdx.x * 1e-7f, a1 = a0 + 0.1f, a2 = a0 + 0.2f, a3 = a0 + 0.3f;
  float a4 = a0 + 0.4f, a5 = a0 + 0.5f, a6 = a0 + 0.6f, a7 = a0 + 0.7f;
  for (int k = 0; k < iters; ++k) {
#define STEP(a) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a));
    STEP(a0) STEP(a1) STEP(a2) STEP(a3) STEP(a4) STEP(a5) STEP(a6) STEP(a7)
#undef STEP
  }
  if (a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7 == 12345.f) out[threadIdx.x] = a0;
}

__global__ void fma_loop(float* out, int iters, float seed) {
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = seed + i * 1e-3f + threadIdx.x * 1e-7f;
  const float m = 0.9999f, c = 1e-5f;
  for (int k = 0; k < iters; ++k) {
#pragma unroll
    for (int i = 0; i < 16; ++i) a[i] = fmaf(a[i], m, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  if (s == 12345.f) out[threadIdx.x] = s;
}

}  // namespace

extern "C" int gosma_calibrate_pipes(int device, double* mufu_ops_per_s,
                                     double* fma_flops_per_s) {
  using namespace gosma;
  DeviceGuard g(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  cudaError_t e = cudaMalloc(&out, 1024 * sizeof(float));
  if (e != cudaSuccess) return cuda_error(e, "calibrate");
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int threads = 256, blocks = sms * 8;
  // MUFU: 8 ops per iteration per thread.
  const int it_m = 4096;
  mufu_loop<<<blocks, threads>>>(out, 64, 0.5f);
  cudaEventRecord(e0);
  mufu_loop<<<blocks, threads>>>(out, it_m, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  if (mufu_ops_per_s)
    *mufu_ops_per_s = static_cast<double>(blocks) * threads * it_m * 8.0 / (ms * 1e-3);
  const int it_f = 8192;
  fma_loop<<<blocks, threads>>>(out, 64, 0.5f);
  cudaEventRecord(e0);
  fma_loop<<<blocks, threads>>>(out, it_f, 0.5f);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  if (fma_flops_per_s)
    *fma_flops_per_s = static_cast<double>(blocks) * threads * it_f * 16.0 * 2.0 / (ms * 1e-3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_error(e, "calibrate");
  return GOSMA_OK;
}
