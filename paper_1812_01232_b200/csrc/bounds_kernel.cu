// K1 — fused lower + upper bound evaluation of rotation x translation
// sub-cubes (GOSMA hot path), hand-written for sm_100a.
//
// Reference semantics: evaluate_bounds (core/src/bounds.cpp:275-284) =
//   feasibility scan (se3.cpp:94-100)
//   + branch_lower_core (bounds.cpp:46-183)   -> lower (max'd with parent floor)
//   + objective_value at feasible_center      -> upper (bounds.cpp:187-214,
//     objective.cpp:175-235), skipped when lower >= skip_upper_at.
// plus subdivide_adaptive's split decision (se3.cpp:107-121), fused because
// it reuses psi_trans.
//
// Work decomposition: one warp per node (persistent warps, dynamic node
// counter). Lanes first build per-component tables for the node in shared
// memory (FP64 prep, FP32 results), then sweep the pair terms:
//   cross  (i, j): lane owns model row i, image column j is a smem broadcast;
//   self   (i, j): circulant schedule (i, i+d mod n), conflict-free smem rows.
// LB and UB contributions of a pair share the geometry and one reciprocal.
//
// Numerics: every pair ratio is evaluated in the
// coupled log form the reference uses for its lower bound,
//   log[Z(K)/(Z(a)Z(b))] = (K-a-b) + log W(K) - log W(a) - log W(b),
// with the excess K-a-b = -2ab(1-cos)/(K+a+b) and 1-cos / 1+cos taken from
// half-angle sines and cosines (|u-v|/2, |u+v|/2), which keeps FP32 accurate
// at concentrations of 1e4-1e5 where log Z(K)-log Z(a)-log Z(b) would cancel
// catastrophically. Terms are FP32 (MUFU ex2/rsqrt/rcp); per-lane partial sums
// are flushed to FP64 every row; per-node sums are FP64 warp reductions.
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>

#include "gosma_internal.hpp"

namespace gosma {

namespace {

std::atomic<unsigned long long> g_launches{0};

constexpr int kWarpsPerCta = 4;
constexpr unsigned kFull = 0xffffffffu;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcpf(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rsqf(float x) {
  float y;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// log W(x) in log2 units, for x <= 15 (W(x) = (1 - e^{-2x})/x, bounds.cpp:18-37).
// Series below 0.25 keeps relative accuracy where 1 - e^{-2x} cancels.
__device__ __noinline__ float log2w_small(float x) {
  float w;
  if (x < 0.25f) {
    // W/2 = 1 - x + 2x^2/3 - x^3/3 + 2x^4/15 - 2x^5/45 + 4x^6/315 - x^7/315 + 2x^8/2835
    float p = 2.0f / 2835.0f;
    p = fmaf(p, x, -1.0f / 315.0f);
    p = fmaf(p, x, 4.0f / 315.0f);
    p = fmaf(p, x, -2.0f / 45.0f);
    p = fmaf(p, x, 2.0f / 15.0f);
    p = fmaf(p, x, -1.0f / 3.0f);
    p = fmaf(p, x, 2.0f / 3.0f);
    p = fmaf(p, x, -1.0f);
    p = fmaf(p, x, 1.0f);
    w = 2.0f * p;
    return lg2f(w);
  }
  const float e = ex2f(-2.0f * kL2E * x);
  return lg2f(1.0f - e) - lg2f(x);
}

// FP64 log W(x) = log_z_eval(x) - x, or -log x past 30 (bounds.cpp:34-37,
// sphere_stats.cpp:47-56).
__device__ double logw_d(double x) {
  if (x > 30.0) return -log(x);
  double lz;
  if (x < 1e-4) {
    lz = log(2.0) + log1p(x * x / 6.0);
  } else {
    lz = x + log1p(-exp(-2.0 * x)) - log(x);
  }
  return lz - x;
}

// Half-angle coth term of the diagonal pair: phi^2 * k/2 * coth k
// (bounds.cpp:104-106, objective.cpp:201-203). k >= 1 always.
__device__ __forceinline__ double diag_term(double phi, double k) {
  double c;
  if (k > 20.0) {
    c = 1.0;  // coth(20) = 1 + 8.5e-18, below double resolution
  } else {
    const double e = exp(-2.0 * k);
    c = (1.0 + e) / (1.0 - e);
  }
  return phi * phi * 0.5 * k * c;
}

__device__ __forceinline__ double dnorm3(double x, double y, double z) {
  // Same evaluation order as the reference (x*x + y*y) + z*z, no FMA.
  return sqrt(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
}

__device__ __forceinline__ double shfl_d(double v, int src) {
  return __shfl_sync(kFull, v, src);
}

__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
  return v;
}

// Per-warp shared-memory tables.
struct WarpTables {
  float4* r0;  // (ux, uy, uz, klo)           uhat at the cuboid centre
  float4* r1;  // (khi, eLo, st, ct)          eLo = (log phi - lw(klo)) log2e; psi_t half-angle
  float4* r2;  // (kst, eUb, sp, cp)          UB kappa at t*, its exponent, half-angle of psi_t+psi_r
  float4* r3;  // (usx, usy, usz, eHi)        uhat at t*, eHi = (log phi - lw(khi)) log2e
  float4* c0;  // (qx, qy, qz, k2)            q_j = R0^T m_j
  float* c1;   // e2 = (log phi2 - lw(k2)) log2e
};

// Cross terms of one model row against the image columns of its class.
// Returns (LB cross sum, UB cross sum) in FP32 (caller flushes to FP64).
template <bool kSame>
__device__ __forceinline__ void cross_row(const WarpTables& T, int i, int o2, int n2, float& acc_lb,
                                          float& acc_ub) {
  const float4 a0 = T.r0[i];
  const float4 a1 = T.r1[i];
  const float4 a2 = T.r2[i];
  const float4 a3 = T.r3[i];
  const float ux = a0.x, uy = a0.y, uz = a0.z, klo = a0.w;
  const float khi = a1.x;
  const float kst = a2.x, eUb = a2.y, sp = a2.z, cp = a2.w;
  const float eHi = a3.w;
  float lb = 0.0f, ub = 0.0f;
#pragma unroll 2
  for (int j = o2; j < o2 + n2; ++j) {
    const float4 q = T.c0[j];
    const float ej = T.c1[j];
    const float k2 = q.w;
    // --- geometry at the cuboid centre
    const float dx = ux - q.x, dy = uy - q.y, dz = uz - q.z;
    const float x = fminf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)), 4.0f);  // |u - q|^2
    const float y = 4.0f - x;                                          // |u + q|^2
    const float rx = rsqf(fmaxf(x, 1e-30f));
    const float ry = rsqf(fmaxf(y, 1e-30f));
    const float sth = 0.5f * x * rx;  // sin(theta/2)
    const float cth = 0.5f * y * ry;  // cos(theta/2)
    // B = max(0, theta - psi_t - psi_r) (alignment_angle_B, bounds.cpp:143-156)
    const float sb = fmaf(sth, cp, -cth * sp);
    const float cb = fmaf(cth, cp, sth * sp);
    const bool bzero = !(sb > 0.0f);
    const float omc = bzero ? 0.0f : 2.0f * sb * sb;  // 1 - cos B
    const float opc = bzero ? 2.0f : 2.0f * cb * cb;  // 1 + cos B
    // --- LB: excess at the low kappa endpoint, W(K) at K's minimum
    const float ab = klo * k2;
    const float amb = klo - k2;
    const float K2lo = fmaf(amb, amb, 2.0f * ab * opc);
    const float rKlo = rsqf(fmaxf(K2lo, 1e-30f));
    const float Klo = K2lo * rKlo;
    const float D1 = Klo + klo + k2;
    const float num1 = -2.0f * kL2E * ab * omc;
    // --- UB: objective at (r0, t*) (class_objective cross loop)
    float xs, ys;
    if (kSame) {
      xs = x;
      ys = y;
    } else {
      const float ex = a3.x - q.x, ey = a3.y - q.y, ez = a3.z - q.z;
      xs = fminf(fmaf(ex, ex, fmaf(ey, ey, ez * ez)), 4.0f);
      ys = 4.0f - xs;
    }
    const float ab2 = kst * k2;
    const float amb2 = kst - k2;
    const float K2u = fmaf(amb2, amb2, ab2 * ys);
    const float rKu = rsqf(fmaxf(K2u, 1e-30f));
    const float Ku = K2u * rKu;
    const float D2 = Ku + kst + k2;
    const float num2 = -kL2E * ab2 * xs;
    const float inv = rcpf(D1 * D2);
    const float ex1 = num1 * D2 * inv;  // (K - a - b) log2e, LB
    const float ex2 = num2 * D1 * inv;  // (K - a - b) log2e, UB
    // K's minimum over the kappa interval (vertex case, bounds.cpp:163-173)
    const float vertex = (omc - 1.0f) * k2;  // -cos B * k2
    float t1;
    if (vertex <= klo && Klo > 15.0f) {
      t1 = ex2f(ex1 + eHi + ej) * rKlo;
    } else {
      float kmin;
      if (vertex <= klo) {
        kmin = Klo;
      } else if (vertex >= khi) {
        const float d = khi - k2;
        const float kk = fmaf(d, d, 2.0f * khi * k2 * opc);
        kmin = kk * rsqf(fmaxf(kk, 1e-30f));
      } else {
        const float s = omc * opc;
        kmin = k2 * (s * rsqf(fmaxf(s, 1e-30f)));
      }
      const float lw = kmin > 15.0f ? -lg2f(kmin) : log2w_small(kmin);
      t1 = ex2f(ex1 + lw + eHi + ej);
    }
    float t2;
    if (Ku > 15.0f) {
      t2 = ex2f(ex2 + eUb + ej) * rKu;
    } else {
      t2 = ex2f(ex2 + log2w_small(Ku) + eUb + ej);
    }
    // Reference drops pairs with K < a + b - 64 from the objective.
    t2 = (ex2 < -64.0f * kL2E) ? 0.0f : t2;
    lb += t1;
    ub += t2;
  }
  acc_lb = lb;
  acc_ub = ub;
}

// One self pair (i < j logically) with row i held in registers.
template <bool kSame>
__device__ __forceinline__ void self_pair(const float4& a0, const float4& a1, const float4& a2,
                                          const float4& a3, const float4& b0, const float4& b1,
                                          const float4& b2, const float4& b3, float& lb,
                                          float& ub) {
  // --- spread angle A = min(pi, theta + psi_i + psi_j) (bounds.cpp:108-124)
  const float dx = a0.x - b0.x, dy = a0.y - b0.y, dz = a0.z - b0.z;
  const float x = fminf(fmaf(dx, dx, fmaf(dy, dy, dz * dz)), 4.0f);
  const float y = 4.0f - x;
  const float rx = rsqf(fmaxf(x, 1e-30f));
  const float ry = rsqf(fmaxf(y, 1e-30f));
  const float sth = 0.5f * x * rx;
  const float cth = 0.5f * y * ry;
  const float sij = fmaf(a1.z, b1.w, a1.w * b1.z);   // sin((psi_i+psi_j)/2)
  const float cij = fmaf(a1.w, b1.w, -a1.z * b1.z);  // cos((psi_i+psi_j)/2)
  const float S = fmaf(sth, cij, cth * sij);
  const float Cc = fmaf(cth, cij, -sth * sij);
  const bool api = !(cij > 0.0f) || !(Cc > 0.0f);
  const float omc = api ? 2.0f : 2.0f * S * S;   // 1 - cos A
  const float opc = api ? 0.0f : 2.0f * Cc * Cc; // 1 + cos A
  // --- LB: excess at the high corner, W(K) at K's corner maximum
  const float alo = a0.w, ahi = a1.x, blo = b0.w, bhi = b1.x;
  const float hh = ahi * bhi;
  const float dhh = ahi - bhi;
  const float K2hh = fmaf(dhh, dhh, 2.0f * hh * opc);
  const float rKhh = rsqf(fmaxf(K2hh, 1e-30f));
  const float Khh = K2hh * rKhh;
  float K2cm = K2hh;
  float rKcm = rKhh;
  if (opc < 1.0f) {  // cos A < 0: K^2 need not be monotone in each kappa
    const float dll = alo - blo, dlh = alo - bhi, dhl = ahi - blo;
    const float K2ll = fmaf(dll, dll, 2.0f * alo * blo * opc);
    const float K2lh = fmaf(dlh, dlh, 2.0f * alo * bhi * opc);
    const float K2hl = fmaf(dhl, dhl, 2.0f * ahi * blo * opc);
    const float m = fmaxf(fmaxf(K2ll, K2lh), K2hl);
    if (m > K2hh) {
      K2cm = m;
      rKcm = rsqf(fmaxf(m, 1e-30f));
    }
  }
  const float D1 = Khh + ahi + bhi;
  const float num1 = -2.0f * kL2E * hh * omc;
  // --- UB: objective self pair at t* (objective.cpp:204-209)
  float xs, ys;
  if (kSame) {
    xs = x;
    ys = y;
  } else {
    const float ex = a3.x - b3.x, ey = a3.y - b3.y, ez = a3.z - b3.z;
    xs = fminf(fmaf(ex, ex, fmaf(ey, ey, ez * ez)), 4.0f);
    ys = 4.0f - xs;
  }
  const float ka = a2.x, kb = b2.x;
  const float ab2 = ka * kb;
  const float d2 = ka - kb;
  const float K2u = fmaf(d2, d2, ab2 * ys);
  const float rKu = rsqf(fmaxf(K2u, 1e-30f));
  const float Ku = K2u * rKu;
  const float D2 = Ku + ka + kb;
  const float num2 = -kL2E * ab2 * xs;
  const float inv = rcpf(D1 * D2);
  const float ex1 = num1 * D2 * inv;
  const float ex2 = num2 * D1 * inv;
  const float Kcm = K2cm * rKcm;
  float t1;
  if (Kcm > 15.0f) {
    t1 = ex2f(ex1 + a1.y + b1.y + 1.0f) * rKcm;  // +1: factor 2 (bounds.cpp:138)
  } else {
    t1 = ex2f(ex1 + log2w_small(Kcm) + a1.y + b1.y + 1.0f);
  }
  float t2;
  if (Ku > 15.0f) {
    t2 = ex2f(ex2 + a2.y + b2.y + 1.0f) * rKu;
  } else {
    t2 = ex2f(ex2 + log2w_small(Ku) + a2.y + b2.y + 1.0f);
  }
  t2 = (ex2 < -64.0f * kL2E) ? 0.0f : t2;
  lb += t1;
  ub += t2;
}

template <bool kSame>
__device__ __forceinline__ void class_pairs(const WarpTables& T, const ClassSpan cs, int lane,
                                            double w, double& lb_self, double& lb_cross,
                                            double& ub_self, double& ub_cross) {
  const int n = cs.n1;
  // Cross terms: rows over lanes, columns broadcast.
  for (int base = 0; base < n; base += 32) {
    const int il = base + lane;
    if (il < n) {
      float l, u;
      cross_row<kSame>(T, cs.o1 + il, cs.o2, cs.n2, l, u);
      lb_cross += w * static_cast<double>(l);
      ub_cross += w * static_cast<double>(u);
    }
  }
  // Self terms i<j via the circulant schedule: every unordered pair once as
  // (i, i+d mod n), d = 1..(n-1)/2, plus d = n/2 for i < n/2 when n is even.
  const int dfull = (n - 1) / 2;
  const bool even = (n % 2) == 0;
  for (int base = 0; base < n; base += 32) {
    const int il = base + lane;
    if (il < n) {
      const int i = cs.o1 + il;
      const float4 a0 = T.r0[i], a1 = T.r1[i], a2 = T.r2[i];
      const float4 a3 = kSame ? make_float4(0.f, 0.f, 0.f, 0.f) : T.r3[i];
      float l = 0.0f, u = 0.0f;
      int jl = il;
#pragma unroll 2
      for (int d = 1; d <= dfull; ++d) {
        jl = (jl + 1 == n) ? 0 : jl + 1;
        const int j = cs.o1 + jl;
        const float4 b0 = T.r0[j], b1 = T.r1[j], b2 = T.r2[j];
        const float4 b3 = kSame ? make_float4(0.f, 0.f, 0.f, 0.f) : T.r3[j];
        self_pair<kSame>(a0, a1, a2, a3, b0, b1, b2, b3, l, u);
      }
      if (even && il < n / 2) {
        const int j = cs.o1 + il + n / 2;
        const float4 b0 = T.r0[j], b1 = T.r1[j], b2 = T.r2[j];
        const float4 b3 = kSame ? make_float4(0.f, 0.f, 0.f, 0.f) : T.r3[j];
        self_pair<kSame>(a0, a1, a2, a3, b0, b1, b2, b3, l, u);
      }
      lb_self += w * static_cast<double>(l);
      ub_self += w * static_cast<double>(u);
    }
  }
}

__global__ void __launch_bounds__(kWarpsPerCta * 32)
    eval_bounds_kernel(const DevCtx ctx, const EvalArgs args) {
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int N1 = ctx.n1_total, N2 = ctx.n2_total;
  // Per-warp table carve-out.
  const size_t per_warp_f4 = static_cast<size_t>(4 * N1 + N2) + (N2 + 3) / 4;
  float4* base = smem4 + warp * per_warp_f4;
  WarpTables T;
  T.r0 = base;
  T.r1 = T.r0 + N1;
  T.r2 = T.r1 + N1;
  T.r3 = T.r2 + N1;
  T.c0 = T.r3 + N1;
  T.c1 = reinterpret_cast<float*>(T.c0 + N2);

  const double zeta = ctx.zeta;
  for (;;) {
    long long node = 0;
    if (lane == 0) node = static_cast<long long>(atomicAdd(args.work, 1u));
    node = __shfl_sync(kFull, node, 0);
    if (node >= args.n) break;

    // ---- node fetch (gosma_node: rc[3], rhw, tc[3], thw[3], lower)
    double v = 0.0;
    if (lane < 11) v = args.nodes[node * 11 + lane];
    const double rc0 = shfl_d(v, 0), rc1 = shfl_d(v, 1), rc2 = shfl_d(v, 2);
    const double rhw = shfl_d(v, 3);
    const double tc0 = shfl_d(v, 4), tc1 = shfl_d(v, 5), tc2 = shfl_d(v, 6);
    const double h0 = shfl_d(v, 7), h1 = shfl_d(v, 8), h2 = shfl_d(v, 9);
    const double parent_lower = shfl_d(v, 10);

    // ---- feasibility scan (feasible_wrt_zeta, se3.cpp:94-100)
    bool infeasible = false;
    for (int mb = 0; mb < N1; mb += 32) {
      const int mi = mb + lane;
      bool hit = false;
      if (mi < N1) {
        const double* mu = ctx.mu + 3 * mi;
        const double f0 = __dadd_rn(fabs(__dsub_rn(mu[0], tc0)), h0);
        const double f1 = __dadd_rn(fabs(__dsub_rn(mu[1], tc1)), h1);
        const double f2 = __dadd_rn(fabs(__dsub_rn(mu[2], tc2)), h2);
        hit = dnorm3(f0, f1, f2) < zeta;
      }
      if (__any_sync(kFull, hit)) {
        infeasible = true;
        break;
      }
    }

    // ---- rotation: R0 = rotation_matrix(rc) (se3.cpp:21-31), psi_r (se3.cpp:68-70)
    double R[9];
    {
      const double th2 = rc0 * rc0 + rc1 * rc1 + rc2 * rc2;
      double a, c;
      if (th2 < 1e-16) {
        a = 1.0;
        c = 0.5;
      } else {
        const double th = sqrt(th2);
        double s, co;
        sincos(th, &s, &co);
        a = s / th;
        c = (1.0 - co) / th2;
      }
      const double K[9] = {0.0, -rc2, rc1, rc2, 0.0, -rc0, -rc1, rc0, 0.0};
#pragma unroll
      for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int cix = 0; cix < 3; ++cix) {
          const double k2 = K[3 * r] * K[cix] + K[3 * r + 1] * K[3 + cix] + K[3 * r + 2] * K[6 + cix];
          R[3 * r + cix] = ((r == cix ? 1.0 : 0.0) + a * K[3 * r + cix]) + c * k2;
        }
    }
    const double psi_r = fmin(sqrt(3.0) * rhw, M_PI);
    float s_r, c_r;
    {
      double s, c;
      sincos(0.5 * psi_r, &s, &c);
      s_r = static_cast<float>(s);
      c_r = static_cast<float>(c);
    }

    // ---- feasible_center (bounds.cpp:187-214): t*, warp-cooperative scan
    double ts0 = tc0, ts1 = tc1, ts2 = tc2;
    bool have_center = false;
    if (!infeasible) {
      for (int proj = 0; proj <= 8; ++proj) {
        int off = -1;
        for (int mb = 0; mb < N1; mb += 32) {
          const int mi = mb + lane;
          bool hit = false;
          if (mi < N1) {
            const double* mu = ctx.mu + 3 * mi;
            hit = dnorm3(__dsub_rn(mu[0], ts0), __dsub_rn(mu[1], ts1), __dsub_rn(mu[2], ts2)) < zeta;
          }
          const unsigned bal = __ballot_sync(kFull, hit);
          if (bal) {
            off = mb + __ffs(bal) - 1;
            break;
          }
        }
        if (off < 0) {
          have_center = true;
          break;
        }
        if (proj == 8) break;
        const double* mu = ctx.mu + 3 * off;
        double d0 = __dsub_rn(ts0, mu[0]), d1 = __dsub_rn(ts1, mu[1]), d2 = __dsub_rn(ts2, mu[2]);
        const double nn = dnorm3(d0, d1, d2);
        if (nn > 1e-12) {
          d0 = __ddiv_rn(d0, nn);
          d1 = __ddiv_rn(d1, nn);
          d2 = __ddiv_rn(d2, nn);
        } else {
          d0 = 1.0;
          d1 = 0.0;
          d2 = 0.0;
        }
        const double rad = __dmul_rn(zeta, 1.0 + 1e-9);
        ts0 = fmin(fmax(__dadd_rn(mu[0], __dmul_rn(d0, rad)), __dsub_rn(tc0, h0)), __dadd_rn(tc0, h0));
        ts1 = fmin(fmax(__dadd_rn(mu[1], __dmul_rn(d1, rad)), __dsub_rn(tc1, h1)), __dadd_rn(tc1, h1));
        ts2 = fmin(fmax(__dadd_rn(mu[2], __dmul_rn(d2, rad)), __dsub_rn(tc2, h2)), __dadd_rn(tc2, h2));
      }
    }
    const bool same = (ts0 == tc0) && (ts1 == tc1) && (ts2 == tc2);

    // ---- per-row prep (all classes): kappa interval, psi_t, projections
    double lb_self = 0.0, lb_cross = 0.0, ub_self = 0.0, ub_cross = 0.0;
    float st_max = 0.0f;
    for (int c = 0; c < ctx.n_classes; ++c) {
      const ClassSpan cs = ctx.cls[c];
      const double w = ctx.cls_w[c];
      for (int il = lane; il < cs.n1; il += 32) {
        const int i = cs.o1 + il;
        const double m0 = ctx.mu[3 * i], m1 = ctx.mu[3 * i + 1], m2 = ctx.mu[3 * i + 2];
        const double is2 = ctx.inv_s2[i];
        const double u0 = m0 - tc0, u1 = m1 - tc1, u2 = m2 - tc2;
        const double a0 = fabs(u0), a1 = fabs(u1), a2 = fabs(u2);
        // point_cuboid_distance (se3.cpp:60-66)
        const double o0 = fmax(a0 - h0, 0.0), o1 = fmax(a1 - h1, 0.0), o2 = fmax(a2 - h2, 0.0);
        const double dlo = fmax(sqrt(o0 * o0 + o1 * o1 + o2 * o2), zeta);
        const double dhi2 = (a0 + h0) * (a0 + h0) + (a1 + h1) * (a1 + h1) + (a2 + h2) * (a2 + h2);
        const double klo = dlo * dlo * is2 + 1.0;
        const double khi = dhi2 * is2 + 1.0;
        const double lphi = static_cast<double>(ctx.log_phi1[i]);
        const double nrm = sqrt(u0 * u0 + u1 * u1 + u2 * u2);
        float ux = 1.0f, uy = 0.0f, uz = 0.0f;
        if (nrm > 1e-12) {
          const double inv = 1.0 / nrm;
          ux = static_cast<float>(u0 * inv);
          uy = static_cast<float>(u1 * inv);
          uz = static_cast<float>(u2 * inv);
        }
        // psi_trans (se3.cpp:72-92) as a half-angle: max over the 8 vertices
        // of |c_hat - v_hat| / 2 = sin(angle / 2).
        float st, ct;
        if (a0 <= h0 && a1 <= h1 && a2 <= h2) {
          st = 1.0f;  // psi_t = pi
          ct = 0.0f;
        } else {
          const float fu0 = static_cast<float>(u0), fu1 = static_cast<float>(u1),
                      fu2 = static_cast<float>(u2);
          const float fh0 = static_cast<float>(h0), fh1 = static_cast<float>(h1),
                      fh2 = static_cast<float>(h2);
          float best = -1.0f, bx = 0.f, by = 0.f, bz = 0.f;
#pragma unroll
          for (int s = 0; s < 8; ++s) {
            const float vx = fu0 - ((s & 4) ? fh0 : -fh0);
            const float vy = fu1 - ((s & 2) ? fh1 : -fh1);
            const float vz = fu2 - ((s & 1) ? fh2 : -fh2);
            const float rv = rsqf(fmaxf(fmaf(vx, vx, fmaf(vy, vy, vz * vz)), 1e-37f));
            const float wx = vx * rv, wy = vy * rv, wz = vz * rv;
            const float ex = ux - wx, ey = uy - wy, ez = uz - wz;
            const float d2 = fmaf(ex, ex, fmaf(ey, ey, ez * ez));
            if (d2 > best) {
              best = d2;
              bx = wx;
              by = wy;
              bz = wz;
            }
          }
          const float px = ux + bx, py = uy + by, pz = uz + bz;
          const float e2 = fmaf(px, px, fmaf(py, py, pz * pz));
          st = 0.5f * sqrtf(fmaxf(best, 0.0f));
          ct = 0.5f * sqrtf(e2);
        }
        st_max = fmaxf(st_max, st);
        // half-angle of psi_t + psi_r; B = 0 when the sum reaches pi
        float sp = fmaf(st, c_r, ct * s_r);
        float cp = fmaf(ct, c_r, -st * s_r);
        if (!(cp > 0.0f)) {
          sp = 1.0f;
          cp = 0.0f;
        }
        // UB projection at t* (project_model, objective.cpp:175-192)
        const double v0 = m0 - ts0, v1 = m1 - ts1, v2 = m2 - ts2;
        const double dd2 = v0 * v0 + v1 * v1 + v2 * v2;
        const double dd = sqrt(dd2);
        const double kst = dd2 * is2 + 1.0;
        const double id = 1.0 / dd;
        const double phi = ctx.phi1[i];
        if (!infeasible) {
          lb_self += w * diag_term(phi, klo);
          ub_self += w * diag_term(phi, kst);
        }
        const float eLo = static_cast<float>((lphi - logw_d(klo)) * kL2E);
        const float eHi = static_cast<float>((lphi - logw_d(khi)) * kL2E);
        const float eUb = static_cast<float>((lphi - logw_d(kst)) * kL2E);
        T.r0[i] = make_float4(ux, uy, uz, static_cast<float>(klo));
        T.r1[i] = make_float4(static_cast<float>(khi), eLo, st, ct);
        T.r2[i] = make_float4(static_cast<float>(kst), eUb, sp, cp);
        T.r3[i] = make_float4(static_cast<float>(v0 * id), static_cast<float>(v1 * id),
                              static_cast<float>(v2 * id), eHi);
      }
    }
    // split decision (subdivide_adaptive, se3.cpp:107-121)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) st_max = fmaxf(st_max, __shfl_xor_sync(kFull, st_max, o));
    if (lane == 0 && args.split_rot) {
      const bool rot_ok = rhw > 1e-9;
      const bool trans_ok = fmax(fmax(h0, h1), h2) > 1e-9;
      int8_t sr;
      if (!rot_ok && !trans_ok) {
        sr = -1;
      } else {
        sr = (rot_ok && (!trans_ok || s_r >= st_max)) ? 1 : 0;
      }
      args.split_rot[node] = sr;
    }
    if (infeasible) {
      if (lane == 0) {
        args.lower[node] = INFINITY;
        args.upper[node] = INFINITY;
      }
      __syncwarp();
      continue;
    }
    // ---- per-column prep: q_j = R0^T m_j (bounds.cpp:97-102)
    for (int j = lane; j < N2; j += 32) {
      const double x0 = ctx.m[3 * j], x1 = ctx.m[3 * j + 1], x2 = ctx.m[3 * j + 2];
      const float q0 = static_cast<float>(R[0] * x0 + R[3] * x1 + R[6] * x2);
      const float q1 = static_cast<float>(R[1] * x0 + R[4] * x1 + R[7] * x2);
      const float q2 = static_cast<float>(R[2] * x0 + R[5] * x1 + R[8] * x2);
      T.c0[j] = make_float4(q0, q1, q2, ctx.kappa2[j]);
      T.c1[j] = ctx.e2[j];
    }
    __syncwarp();

    // ---- pair sweeps
    for (int c = 0; c < ctx.n_classes; ++c) {
      const ClassSpan cs = ctx.cls[c];
      const double w = ctx.cls_w[c];
      if (same) {
        class_pairs<true>(T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross);
      } else {
        class_pairs<false>(T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross);
      }
    }
    lb_self = warp_sum_d(lb_self);
    lb_cross = warp_sum_d(lb_cross);
    ub_self = warp_sum_d(ub_self);
    ub_cross = warp_sum_d(ub_cross);
    if (lane == 0) {
      // Soundness margin proportional to the |term| mass (all terms >= 0).
      const double mass = lb_self + 2.0 * lb_cross;
      const double core = (lb_self - 2.0 * lb_cross) - ctx.lb_margin * mass;
      const double lo = core < parent_lower ? parent_lower : core;  // std::max(core, lower)
      double up = INFINITY;
      if (!(lo >= args.skip_upper_at) && have_center) up = ub_self - 2.0 * ub_cross;
      args.lower[node] = lo;
      args.upper[node] = up;
    }
    __syncwarp();
  }
}

}  // namespace

size_t eval_smem_per_warp(const DevCtx& ctx) {
  const size_t f4 = static_cast<size_t>(4 * ctx.n1_total + ctx.n2_total) + (ctx.n2_total + 3) / 4;
  return f4 * sizeof(float4);
}

cudaError_t launch_eval_bounds(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                               cudaStream_t stream) {
  if (a.n <= 0) return cudaSuccess;
  const size_t smem = eval_smem_per_warp(ctx) * kWarpsPerCta;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(eval_bounds_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, eval_bounds_kernel,
                                                                kWarpsPerCta * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  long long grid = static_cast<long long>(per_sm) * sm_count;
  const long long need = (a.n + kWarpsPerCta - 1) / kWarpsPerCta;
  if (grid > need) grid = need;
  e = cudaMemsetAsync(a.work, 0, sizeof(unsigned int), stream);
  if (e != cudaSuccess) return e;
  eval_bounds_kernel<<<static_cast<unsigned>(grid), kWarpsPerCta * 32, smem, stream>>>(ctx, a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

unsigned long long bound_kernel_launch_count() { return g_launches.load(); }

}  // namespace gosma
