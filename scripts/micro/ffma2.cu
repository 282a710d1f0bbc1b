// FFMA vs FFMA2 issue/throughput microbenchmark (sm_100a).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, float a, float b, int iters) {
  float x[8];
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fmaf(x[k], a, b);
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, float a, float b, int iters) {
  float2 x[8];
  for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], a2, b2);
  float s = 0; for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed: per iteration 8 FFMA2 (16 flops) + 2 MUFU vs 16 FFMA + 2 MUFU
__global__ void k_mix1(float* out, float a, float b, int iters) {
  float x[16];
  for (int k = 0; k < 16; ++k) x[k] = threadIdx.x * 1e-3f + k;
  float m = 1.0f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 16; ++k) x[k] = fmaf(x[k], a, b);
    float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[0] * 1e-9f)); m += y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[3] + 2.0f)); m += y;
  }
  float s = m; for (int k = 0; k < 16; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix2(float* out, float a, float b, int iters) {
  float2 x[8];
  for (int k = 0; k < 8; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
  const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
  float m = 1.0f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = __ffma2_rn(x[k], a2, b2);
    float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[0].x * 1e-9f)); m += y;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[1].y + 2.0f)); m += y;
  }
  float s = m; for (int k = 0; k < 8; ++k) s += x[k].x + x[k].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000; dim3 g(148 * 8), b(256);
  auto run = [&](const char* name, void (*k)(float*, float, float, int), double flops_per_iter) {
    k<<<g, b>>>(d, 0.999f, 0.001f, 100);
    cudaEventRecord(e0);
    k<<<g, b>>>(d, 0.999f, 0.001f, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double thr = (double)g.x * b.x * iters;
    printf("%-8s %8.3f ms  %.2f TFLOP/s  %.3e iters/s\n", name, ms, thr * flops_per_iter / ms / 1e9, thr / ms * 1e3);
  };
  run("ffma", k_ffma, 16); run("ffma2", k_ffma2, 32); run("mix1", k_mix1, 32); run("mix2", k_mix2, 32);
  return 0;
}
