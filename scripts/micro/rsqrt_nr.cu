// Accuracy of K1's rsqrt_nr (MUFU.RSQ64H estimate + two Newton steps) against
// the correctly rounded 1/sqrt over 1e-300 .. 1e300 (max error in ulps).
#include <cmath>
#include <cstdio>
#include <cuda_runtime.h>
__device__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}
__global__ void k(const double* x, double* a, double* b, double* e0, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  a[i] = rsqrt_nr(x[i]);
  b[i] = 1.0 / sqrt(x[i]);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x[i]));
  e0[i] = y;
}
int main() {
  const int n = 1 << 20;
  double *x, *a, *b, *e0;
  cudaMallocManaged(&x, n * 8); cudaMallocManaged(&a, n * 8); cudaMallocManaged(&b, n * 8);
  cudaMallocManaged(&e0, n * 8);
  unsigned long long s = 88172645463325252ull;
  for (int i = 0; i < n; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    double u = (s >> 11) * (1.0 / 9007199254740992.0);
    x[i] = pow(10.0, -300.0 + 600.0 * u);
  }
  k<<<n / 256, 256>>>(x, a, b, e0, n);
  cudaDeviceSynchronize();
  double worst = 0, worst0 = 0;
  for (int i = 0; i < n; ++i) {
    double ulp = nextafter(b[i], INFINITY) - b[i];
    worst = fmax(worst, fabs(a[i] - b[i]) / ulp);
    worst0 = fmax(worst0, fabs(e0[i] - b[i]) / b[i]);
  }
  printf("rsqrt_nr max error %.2f ulp; MUFU estimate max rel error %.3e (2^%.1f)\n", worst,
         worst0, log2(worst0));
  return 0;
}
