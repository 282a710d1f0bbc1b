// Issue-bound mix (FP32 arithmetic + MUFU + compares/selects): scalar vs
// float2-packed (FFMA2/FADD2/FMUL2) arithmetic, same work per "pair".
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float ex2f(float x) { float y; asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rsqf(float x) { float y; asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float rcpf(float x) { float y; asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
struct P { float a, b, c, d; };
__device__ __forceinline__ float pair1(float4 r, float4 q, float& acc) {
  float dx = r.x - q.x, dy = r.y - q.y, dz = r.z - q.z;
  float px = r.x + q.x, py = r.y + q.y, pz = r.z + q.z;
  float x = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  float y = fmaf(px, px, fmaf(py, py, pz * pz));
  float m = rsqf(x * y + 1.0f) * r.w;
  float num = (x > y) ? (q.w - y) : (x - r.w);
  bool bz = !(num > 0.0f);
  num = bz ? 0.0f : num;
  float den = fmaf(x, r.w, fmaf(y, q.w, m));
  float c2 = fmaf(y, q.w, fmaf(x, r.w, m));
  float k = fmaf(r.w - q.w, r.w - q.w, r.w * q.w * c2);
  float rk = rsqf(k);
  float K = k * rk;
  float D = K + r.w + q.w;
  float inv = rcpf(D * den + 1.0f);
  float e = r.w * q.w * num * num * inv * -1.4427f;
  float t = ex2f(e) * rk;
  acc = fmaf(q.w, t, acc);
  return fabsf(e) * t;
}
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, f2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ void pair2(float4 r, float4 q0, float4 q1, float& acc, float& me) {
  const float2 rx = f2(r.x, r.x), ry = f2(r.y, r.y), rz = f2(r.z, r.z), rw = f2(r.w, r.w);
  const float2 qx = f2(q0.x, q1.x), qy = f2(q0.y, q1.y), qz = f2(q0.z, q1.z), qw = f2(q0.w, q1.w);
  float2 dx = sub2(rx, qx), dy = sub2(ry, qy), dz = sub2(rz, qz);
  float2 px = add2(rx, qx), py = add2(ry, qy), pz = add2(rz, qz);
  float2 x = fma2(dx, dx, fma2(dy, dy, mul2(dz, dz)));
  float2 y = fma2(px, px, fma2(py, py, mul2(pz, pz)));
  float2 xy = fma2(x, y, f2(1.f, 1.f));
  float2 m = mul2(f2(rsqf(xy.x), rsqf(xy.y)), rw);
  float2 num = f2((x.x > y.x) ? (q0.w - y.x) : (x.x - r.w), (x.y > y.y) ? (q1.w - y.y) : (x.y - r.w));
  num.x = (num.x > 0.f) ? num.x : 0.f;
  num.y = (num.y > 0.f) ? num.y : 0.f;
  float2 den = fma2(x, rw, fma2(y, qw, m));
  float2 c2 = fma2(y, qw, fma2(x, rw, m));
  float2 dd = sub2(rw, qw);
  float2 k = fma2(dd, dd, mul2(mul2(rw, qw), c2));
  float2 rk = f2(rsqf(k.x), rsqf(k.y));
  float2 K = mul2(k, rk);
  float2 D = add2(add2(K, rw), qw);
  float2 dn = fma2(D, den, f2(1.f, 1.f));
  float2 inv = f2(rcpf(dn.x), rcpf(dn.y));
  float2 e = mul2(mul2(mul2(mul2(rw, qw), mul2(num, num)), inv), f2(-1.4427f, -1.4427f));
  float2 t = mul2(f2(ex2f(e.x), ex2f(e.y)), rk);
  float2 a2 = mul2(qw, t);
  acc += a2.x + a2.y;
  me += fabsf(e.x) * t.x + fabsf(e.y) * t.y;
}
__global__ void k1(const float4* __restrict__ q, float* out, int iters) {
  __shared__ float4 sq[64];
  if (threadIdx.x < 64) sq[threadIdx.x] = q[threadIdx.x];
  __syncthreads();
  float4 r = make_float4(threadIdx.x * 1e-3f, 0.3f, 0.5f, 2.0f);
  float acc = 0, me = 0;
  for (int it = 0; it < iters; ++it)
#pragma unroll 2
    for (int j = 0; j < 64; ++j) me += pair1(r, sq[j], acc);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + me;
}
__global__ void k2(const float4* __restrict__ q, float* out, int iters) {
  __shared__ float4 sq[64];
  if (threadIdx.x < 64) sq[threadIdx.x] = q[threadIdx.x];
  __syncthreads();
  float4 r = make_float4(threadIdx.x * 1e-3f, 0.3f, 0.5f, 2.0f);
  float acc = 0, me = 0;
  for (int it = 0; it < iters; ++it)
    for (int j = 0; j < 64; j += 2) pair2(r, sq[j], sq[j + 1], acc, me);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + me;
}
int main() {
  float4 h[64];
  for (int i = 0; i < 64; ++i) h[i] = make_float4(0.01f * i, 0.2f, 0.7f, 1.0f + 0.1f * i);
  float4* dq; float* d; cudaMalloc(&dq, sizeof(h)); cudaMemcpy(dq, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&d, 148 * 24 * 128 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 200;
  for (int v = 0; v < 2; ++v) {
    auto k = v ? k2 : k1;
    k<<<148 * 6, 128>>>(dq, d, 2);
    cudaEventRecord(e0);
    k<<<148 * 6, 128>>>(dq, d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double pairs = 148.0 * 6 * 128 * iters * 64;
    printf("%s: %.3f ms  %.3e pairs/s\n", v ? "float2" : "scalar", ms, pairs / ms * 1e3);
  }
  return 0;
}
