// K6 — batched FP64 objective value + gradient for the local refiner (SMA):
// objective_value / objective_gradient (core/src/objective.cpp:175-334) for
// many poses at once, so the L-BFGS starts of the discovery dive and the
// incumbent refinements evaluate on the GPU. A request is
// spread over a grid row of CTAs (threads = model rows, CTAs = slices of the
// pair partners) so a batch of a few dozen starts still fills the GPU; model
// rows live in shared memory; FP64 throughout (the refiner tests |g| < 1e-6). Pair terms below the reference's margin
// (K < a + b - 64, objective.cpp:17) are skipped exactly as on the host.
//
// Gradient algebra (objective.cpp:254-334), rearranged so no 3x3 matrix is
// stored: J_i v = u_i (u_i.v)(-2 d_i / s2_i) - (v - u_i (u_i.v)) (k_i / d_i)
// is linear in v, so every J_i / R^T / Jl^T product is applied once per row
// (or once per pose) to an accumulated vector. Self pairs are visited as
// ordered pairs (i != j), each side adding its own half of the gradient.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "objective_device.hpp"

namespace gosma {

namespace {

constexpr unsigned kFullMask = 0xffffffffu;
constexpr double kMarginObj = 64.0;  // objective.cpp:17

__device__ __forceinline__ double log_z_d(double k) {
  // sphere_stats.cpp:47-56
  if (k < 1e-4) return 0.69314718055994531 + log1p(k * k / 6.0);
  return k + log1p(-exp(-2.0 * k)) - log(k);
}

__device__ __forceinline__ double log_z_deriv_d(double k) {
  // sphere_stats.cpp:58-69
  if (k < 1e-4) return k / 3.0 - k * k * k / 45.0;
  if (k > 350.0) return 1.0 - 1.0 / k;
  const double e2 = exp(-2.0 * k);
  return (1.0 + e2) / (1.0 - e2) - 1.0 / k;
}

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFullMask, v, o);
  return v;
}

// Per-row record in shared memory (FP64).
struct RowD {
  double ux, uy, uz;  // unit direction of mu_i - t
  double d, k, lz, zl, is2, phi;
};

__device__ __forceinline__ void jv(const RowD& r, double vx, double vy, double vz, double& ox,
                                   double& oy, double& oz) {
  const double p = r.ux * vx + r.uy * vy + r.uz * vz;
  const double a = -2.0 * r.d * r.is2, b = r.k / r.d;
  ox = r.ux * p * a - (vx - r.ux * p) * b;
  oy = r.uy * p * a - (vy - r.uy * p) * b;
  oz = r.uz * p * a - (vz - r.uz * p) * b;
}

// Block-wide deterministic sum (fixed tree over the warps).
__device__ __forceinline__ double block_sum(double v, double* red) {
  v = wsum(v);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = 0.0;
  for (int k = 0; k < nw; ++k) t += red[k];
  return t;
}

// Grid: x = partner slice, y = request. Thread = model row (strided), the
// slice = a contiguous range of partners (self rows j != i, then image
// columns). Per-slice partial {f, g[6]} go to out[(q * S + s) * 7]; the host
// sums slices in order (deterministic).
__global__ void __launch_bounds__(256)
    objgrad_kernel(const DevModel64* models, const ObjRequest* req, double* out, int max_n1) {
  extern __shared__ double smem_d[];
  RowD* rows = reinterpret_cast<RowD*>(smem_d);
  double* red = smem_d + static_cast<size_t>(max_n1) * (sizeof(RowD) / sizeof(double));
  const int q = blockIdx.y, slice = blockIdx.x, S = gridDim.x;
  const ObjRequest rq = req[q];
  const DevModel64 m = models[rq.model];
  const double r0 = rq.x[0], r1 = rq.x[1], r2 = rq.x[2];
  const double t0 = rq.x[3], t1 = rq.x[4], t2 = rq.x[5];
  double* o = out + (static_cast<size_t>(q) * S + slice) * 7;
  // check_feasible (objective.cpp:160-166)
  int hit = 0;
  for (int i = threadIdx.x; i < m.n_all; i += blockDim.x) {
    const double dx = m.all_means[3 * i] - t0, dy = m.all_means[3 * i + 1] - t1,
                 dz = m.all_means[3 * i + 2] - t2;
    hit |= sqrt(dx * dx + dy * dy + dz * dz) < m.zeta;
  }
  if (__syncthreads_or(hit)) {
    if (threadIdx.x == 0) {
      o[0] = slice == 0 ? INFINITY : 0.0;
      for (int k = 1; k < 7; ++k) o[k] = 0.0;
    }
    return;
  }
  // Rodrigues R (se3.cpp:21-31) and the left Jacobian (objective.cpp:240-250)
  double R[9], Jl[9];
  {
    const double th2 = r0 * r0 + r1 * r1 + r2 * r2;
    const double K[9] = {0.0, -r2, r1, r2, 0.0, -r0, -r1, r0, 0.0};
    double K2[9];
    for (int a = 0; a < 3; ++a)
      for (int c = 0; c < 3; ++c)
        K2[3 * a + c] = K[3 * a] * K[c] + K[3 * a + 1] * K[3 + c] + K[3 * a + 2] * K[6 + c];
    double ra, rc, ja, jb;
    if (th2 < 1e-16) {
      ra = 1.0;
      rc = 0.5;
    } else {
      const double th = sqrt(th2);
      ra = sin(th) / th;
      rc = (1.0 - cos(th)) / th2;
    }
    if (th2 < 1e-12) {
      ja = 0.5;
      jb = 1.0 / 6.0;
    } else {
      const double th = sqrt(th2);
      ja = (1.0 - cos(th)) / th2;
      jb = (th - sin(th)) / (th2 * th);
    }
    for (int e = 0; e < 9; ++e) {
      const double id = (e % 4 == 0) ? 1.0 : 0.0;
      R[e] = (id + ra * K[e]) + rc * K2[e];
      Jl[e] = id + K[e] * ja + K2[e] * jb;
    }
  }
  double fval = 0.0, gt0 = 0.0, gt1 = 0.0, gt2 = 0.0, cr0 = 0.0, cr1 = 0.0, cr2 = 0.0;
  for (int c = 0; c < m.n_classes; ++c) {
    const ClassSpan cs = m.cls[c];
    const double w = m.cls_w[c];
    __syncthreads();
    for (int il = threadIdx.x; il < cs.n1; il += blockDim.x) {
      const int i = cs.o1 + il;
      const double ux = m.mu[3 * i] - t0, uy = m.mu[3 * i + 1] - t1, uz = m.mu[3 * i + 2] - t2;
      const double d2 = ux * ux + uy * uy + uz * uz;
      const double d = sqrt(d2);
      RowD r;
      r.ux = ux * (1.0 / d);
      r.uy = uy * (1.0 / d);
      r.uz = uz * (1.0 / d);
      r.d = d;
      r.is2 = 1.0 / m.sigma2[i];
      r.k = d2 / m.sigma2[i] + 1.0;
      r.lz = log_z_d(r.k);
      r.zl = log_z_deriv_d(r.k);
      r.phi = m.phi1[i];
      rows[il] = r;
    }
    __syncthreads();
    // this slice's partners: [p0, p1) over self rows (0..n1-1) then columns
    const int np = cs.n1 + cs.n2;
    const int p0 = static_cast<int>(static_cast<long long>(np) * slice / S);
    const int p1 = static_cast<int>(static_cast<long long>(np) * (slice + 1) / S);
    for (int il = threadIdx.x; il < cs.n1; il += blockDim.x) {
      const RowD a = rows[il];
      const double uix = a.ux * a.d, uiy = a.uy * a.d, uiz = a.uz * a.d;  // u_i
      const double cu = 2.0 * a.zl * a.is2;
      double fself = 0.0, fcross = 0.0;
      if (slice == 0) {  // diagonal (objective.cpp:201-203, 268-274)
        const double term = 0.5 * a.k / tanh(a.k);
        fself += a.phi * a.phi * term;
        const double dlog = 2.0 * (log_z_deriv_d(2.0 * a.k) - a.zl);
        const double sd = a.phi * a.phi * term * dlog * (-2.0 * a.is2);
        gt0 += w * uix * sd;
        gt1 += w * uiy * sd;
        gt2 += w * uiz * sd;
      }
      const double vix = a.ux * a.k, viy = a.uy * a.k, viz = a.uz * a.k;
      // self pairs, ordered (i != j): this row's half of each pair
      double sx = 0.0, sy = 0.0, sz = 0.0, su = 0.0;
      const int s_end = min(p1, cs.n1);
      for (int jl = p0; jl < s_end; ++jl) {
        if (jl == il) continue;
        const RowD b = rows[jl];
        const double ex = vix + b.ux * b.k, ey = viy + b.uy * b.k, ez = viz + b.uz * b.k;
        const double K = sqrt(ex * ex + ey * ey + ez * ez);
        if (K < a.k + b.k - kMarginObj) continue;
        const double term = 2.0 * a.phi * b.phi * exp(log_z_d(K) - a.lz - b.lz);
        fself += 0.5 * term;
        if (K > 1e-12) {
          const double s = log_z_deriv_d(K) * term / K;
          sx += ex * s;
          sy += ey * s;
          sz += ez * s;
        }
        su += term;
      }
      // cross pairs (objective.cpp:212-220, 300-326)
      const double wx = R[0] * vix + R[1] * viy + R[2] * viz;
      const double wy = R[3] * vix + R[4] * viy + R[5] * viz;
      const double wz = R[6] * vix + R[7] * viy + R[8] * viz;
      double hx = 0.0, hy = 0.0, hz = 0.0, hu = 0.0;
      for (int jp = max(p0, cs.n1); jp < p1; ++jp) {
        const int j = cs.o2 + (jp - cs.n1);
        const double ex = wx + m.b[3 * j], ey = wy + m.b[3 * j + 1], ez = wz + m.b[3 * j + 2];
        const double K = sqrt(ex * ex + ey * ey + ez * ez);
        if (K < a.k + m.kappa2[j] - kMarginObj) continue;
        const double term = a.phi * m.phi2[j] * exp(log_z_d(K) - a.lz - m.log_z2[j]);
        fcross += term;
        double qx = 0.0, qy = 0.0, qz = 0.0;
        if (K > 1e-12) {
          qx = ex / K;
          qy = ey / K;
          qz = ez / K;
        }
        const double s = log_z_deriv_d(K) * (-2.0 * term);
        hx += qx * s;
        hy += qy * s;
        hz += qz * s;
        hu += -2.0 * term;
        // (w x what) for the rotation gradient (Jl^T applied per pose)
        cr0 += w * (wy * qz - wz * qy) * s;
        cr1 += w * (wz * qx - wx * qz) * s;
        cr2 += w * (wx * qy - wy * qx) * s;
      }
      double ox, oy, oz;
      jv(a, sx, sy, sz, ox, oy, oz);  // self: J_i (sum/K) zl(K) term + u_i (2 zl_i/s2_i) term
      gt0 += w * (ox + uix * cu * su);
      gt1 += w * (oy + uiy * cu * su);
      gt2 += w * (oz + uiz * cu * su);
      const double px = R[0] * hx + R[3] * hy + R[6] * hz;  // R^T what
      const double py = R[1] * hx + R[4] * hy + R[7] * hz;
      const double pz = R[2] * hx + R[5] * hy + R[8] * hz;
      jv(a, px, py, pz, ox, oy, oz);
      gt0 += w * (ox + uix * cu * hu);
      gt1 += w * (oy + uiy * cu * hu);
      gt2 += w * (oz + uiz * cu * hu);
      fval += w * (fself - 2.0 * fcross);
    }
  }
  fval = block_sum(fval, red);
  gt0 = block_sum(gt0, red);
  gt1 = block_sum(gt1, red);
  gt2 = block_sum(gt2, red);
  cr0 = block_sum(cr0, red);
  cr1 = block_sum(cr1, red);
  cr2 = block_sum(cr2, red);
  if (threadIdx.x == 0) {
    o[0] = fval;
    o[1] = Jl[0] * cr0 + Jl[3] * cr1 + Jl[6] * cr2;
    o[2] = Jl[1] * cr0 + Jl[4] * cr1 + Jl[7] * cr2;
    o[3] = Jl[2] * cr0 + Jl[5] * cr1 + Jl[8] * cr2;
    o[4] = gt0;
    o[5] = gt1;
    o[6] = gt2;
  }
}

}  // namespace

size_t objgrad_smem_bytes(int max_n1) {
  return static_cast<size_t>(max_n1) * sizeof(RowD) + 8 * sizeof(double);
}

int objgrad_slices(int max_pairs_per_row) {
  // ~16 partners per thread and slice, at most 32 slices
  return std::max(1, std::min(32, max_pairs_per_row / 16));
}

cudaError_t launch_objgrad(const DevModel64* models, const ObjRequest* req, int n, int slices,
                           double* partial, int max_n1, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const size_t smem = objgrad_smem_bytes(max_n1);
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    const cudaError_t e = cudaFuncSetAttribute(
        objgrad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  const int threads = std::min(256, std::max(32, (max_n1 + 31) / 32 * 32));
  objgrad_kernel<<<dim3(slices, n), threads, smem, s>>>(models, req, partial, max_n1);
  return cudaGetLastError();
}

}  // namespace gosma
