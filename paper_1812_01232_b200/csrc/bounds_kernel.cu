// K1 — fused lower + upper bound evaluation of rotation x translation
// sub-cubes (GOSMA hot path), hand-written for sm_100a.
//
// Reference semantics: evaluate_bounds (core/src/bounds.cpp:275-284) =
//   feasibility scan (se3.cpp:94-100)
//   + branch_lower_core (bounds.cpp:46-183)   -> lower (max'd with parent floor)
//   + objective_value at feasible_center      -> upper (bounds.cpp:187-214,
//     objective.cpp:175-235), +inf when lower >= skip_upper_at.
// plus subdivide_adaptive's split decision (se3.cpp:107-121), fused because
// it reuses psi_trans.
//
// Work decomposition: one lane group per node (1, 8 or 32 lanes, or a whole
// CTA for large mixtures; persistent groups, dynamic node counter). Lanes
// first build per-component tables for the node in shared memory, then sweep
// the pair terms:
//   cross (i, j): the lane owns model row i (registers), the image column j
//                 is a shared-memory broadcast;
//   self  (i, j): circulant schedule (i, i+d mod n) — every unordered pair
//                 once, lanes read consecutive rows (conflict-free).
// The LB and UB contributions of a pair share the geometry and one MUFU.RCP.
//
// Numerics: every pair ratio is evaluated in the
// coupled log form the reference uses for its lower bound,
//   log[Z(K)/(Z(a)Z(b))] = (K-a-b) + log W(K) - log W(a) - log W(b),
// with the excess K-a-b = -2ab(1-cos)/(K+a+b) and 1-cos, 1+cos taken from
// half-angle sines/cosines (|u-v|/2, |u+v|/2 and their angle-addition
// formulas). This keeps FP32 accurate at concentrations of 1e4-1e5, where
// log Z(K) - log Z(a) - log Z(b) would cancel catastrophically. For K > 15,
// W(K) = 1/K to FP32 precision, so exp(... + log W(K)) = 2^(...) * rsqrt(K^2):
// a pair costs 6 MUFU ops (1 sqrt, 2 rsqrt, 1 rcp, 2 ex2). The rare exact
// paths (K <= 15, the interior K minimum of the cross LB, the corner maximum
// of the self LB when cos A < 0) run only for terms that survive FP32
// underflow, and only in the exact loop copies: per node, group votes over
// per-row scores send the cross and self loops to copies without them
// (FastScore). Terms are FP32; per-row partial sums flush to FP64; per-node
// sums are FP64 group reductions; a precise fix-up launch re-evaluates the
// few nodes whose FP32 error estimate is large (kFixFull / kFixStream).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "gosma_internal.hpp"

// Unroll factor of the pair loops (A/B builds: -DGOSMA_UNROLL=n).
#ifndef GOSMA_UNROLL
#define GOSMA_UNROLL 1
#endif

namespace gosma {

namespace {

std::atomic<unsigned long long> g_launches{0};

constexpr int kWarpsPerCta = 4;
constexpr int kUnrollPairs = GOSMA_UNROLL;
constexpr unsigned kFull = 0xffffffffu;
// Pair exponents (log2) below this leave the term under 2^-45 of its F_i G_j
// prefactor (<= ~2^34): the exact W paths are skipped for them.
constexpr float kNegligibleLog2 = -80.0f;
// FP32 error model of a pair term (relative; unit roundoff u = 2^-24, safety
// factor 2): exponent error from the B = theta - psi cancellation
// (kErrAmp * |e/num| * max(x, y)), from the exponent's own operations
// (kErrExp * |e|), and the term's MUFU/rounding error (kErrTerm). Summed into
// a per-node margin subtracted from the lower bound.
constexpr float kU = 5.9604645e-8f;
constexpr float kErrAmp = 2.0f * 8.0f * kU * 0.6931472f;
constexpr float kErrExp = 2.0f * 10.0f * kU * 0.6931472f;
constexpr float kErrTerm = 2.0f * 6.0f * kU;

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
__device__ __forceinline__ float sqf(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float lg2f(float x) {
  float y;
  asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// log2 W(x) for any x >= 0 (W(x) = (1 - e^{-2x})/x, bounds.cpp:18-37;
// log W = log_z_eval(x) - x, sphere_stats.cpp:47-56). Past 15 the e^{-2x}
// correction is below FP32 resolution. The series below 0.25 keeps relative
// accuracy where 1 - e^{-2x} cancels.
__device__ __noinline__ float log2w(float x) {
  if (x > 15.0f) return -lg2f(x);
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
    return 1.0f + lg2f(p);
  }
  const float e = ex2f(-2.0f * kL2E * x);
  return lg2f(1.0f - e) - lg2f(x);
}

// Diagonal pair in closed form: phi^2 * (k/2) coth k (bounds.cpp:104-106,
// objective.cpp:201-203); k >= 1 always, so 1 - e^{-2k} >= 0.86.
__device__ __forceinline__ float diag_term(float phi, float k) {
  const float e = ex2f(-2.0f * kL2E * k);
  return phi * phi * 0.5f * k * (1.0f + e) * rcpf(1.0f - e);
}

// Lane groups: a group of kG lanes evaluates one node. kG = 32 is a warp;
// small mixtures (max class n1 <= 16 / 8) run 2 or 4 nodes per warp (kG =
// 16 / 8) so the row lanes stay busy; large mixtures (kG = 128) give one node
// to a whole CTA, so 4 warps share one set of tables and residency is not
// capped by shared memory. Group collectives below cover all three shapes.
constexpr int kCtaGroup = 128;

struct GroupScratch {  // static shared memory of a CTA-wide group
  double d[4];
  long long ll;
  int i[4];
  double node[11];
};

template <int kG>
struct Group {
  unsigned gm;   // lane mask (warp groups)
  int gbase;     // first lane of the group in its warp
  GroupScratch* sh;
  __device__ __forceinline__ void sync() const {
    if constexpr (kG == 1) {
      // a one-lane group needs no synchronisation
    } else if constexpr (kG <= 32) {
      __syncwarp(gm);
    } else {
      __syncthreads();
    }
  }
  __device__ __forceinline__ bool any(bool b) const {
    if constexpr (kG == 1) {
      return b;
    } else if constexpr (kG <= 32) {
      return __any_sync(gm, b);
    } else {
      return __syncthreads_or(b) != 0;
    }
  }
  // OR of 3-bit flags over the group (one vote per bit: __reduce_or_sync
  // with a partial mask serialises the groups of a warp)
  __device__ __forceinline__ unsigned bor3(unsigned v) const {
    return (any((v & 1u) != 0u) ? 1u : 0u) | (any((v & 2u) != 0u) ? 2u : 0u) |
           (any((v & 4u) != 0u) ? 4u : 0u);
  }
  __device__ __forceinline__ double sum(double v) const {
    if constexpr (kG <= 32) {
#pragma unroll
      for (int o = kG / 2; o > 0; o >>= 1) v += __shfl_xor_sync(gm, v, o, kG);
      return v;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
      __syncthreads();
      if ((threadIdx.x & 31) == 0) sh->d[threadIdx.x >> 5] = v;
      __syncthreads();
      return (sh->d[0] + sh->d[1]) + (sh->d[2] + sh->d[3]);
    }
  }
  __device__ __forceinline__ double max(double v) const {
    if constexpr (kG <= 32) {
#pragma unroll
      for (int o = kG / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(gm, v, o, kG));
      return v;
    } else {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(kFull, v, o));
      __syncthreads();
      if ((threadIdx.x & 31) == 0) sh->d[threadIdx.x >> 5] = v;
      __syncthreads();
      return fmax(fmax(sh->d[0], sh->d[1]), fmax(sh->d[2], sh->d[3]));
    }
  }
  // value of lane k of this warp's part of the group (kG > 32: of this warp)
  __device__ __forceinline__ double shfl(double v, int k) const {
    if constexpr (kG == 1) {
      return v;
    } else if constexpr (kG <= 32) {
      return __shfl_sync(gm, v, k, kG);
    } else {
      return __shfl_sync(kFull, v, k);
    }
  }
  // value of group lane 0
  __device__ __forceinline__ long long bcast0(long long v) const {
    if constexpr (kG == 1) {
      return v;
    } else if constexpr (kG <= 32) {
      return __shfl_sync(gm, v, 0, kG);
    } else {
      __syncthreads();
      if (threadIdx.x == 0) sh->ll = v;
      __syncthreads();
      return sh->ll;
    }
  }
  // first group lane with b set (-1: none)
  __device__ __forceinline__ int first(bool b) const {
    if constexpr (kG == 1) {
      return b ? 0 : -1;
    } else if constexpr (kG <= 32) {
      const unsigned bal = __ballot_sync(gm, b) >> gbase;
      return bal ? __ffs(bal) - 1 : -1;
    } else {
      const unsigned bal = __ballot_sync(kFull, b);
      __syncthreads();
      if ((threadIdx.x & 31) == 0) sh->i[threadIdx.x >> 5] = bal ? __ffs(bal) - 1 : -1;
      __syncthreads();
      for (int w = 0; w < 4; ++w)
        if (sh->i[w] >= 0) return 32 * w + sh->i[w];
      return -1;
    }
  }
};

// sqrt(s) < z with the reference's rounding (Eigen norm() = sqrt of the
// squared norm): the squared comparison decides unless s is within a relative
// 1e-12 of z^2, where the correctly rounded sqrt decides.
__device__ __forceinline__ bool norm_below(double s, double z, double z2) {
  const double d = s - z2;
  if (fabs(d) > 1e-12 * z2) return d < 0.0;
  return sqrt(s) < z;
}

// Per-warp shared-memory tables: one record of kRowF4 float4 per model row
// (80 B: conflict-free when lanes read consecutive rows) and kColF4 float4 per
// image column (broadcast), so a row or column costs one address.
struct WarpTables {
  float4* row;  // [0] (uhx, uhy, uhz, Fst)   uhat at the cuboid centre (FP32 high part), phi/W(kst)
                // [1] (khi, Flo, st, ct)     Flo = phi / W(klo); psi_t half-angle
                // [2] (ulx, uly, ulz, kst)   uhat low part (double-float), kappa at t*
                // [3] (usx, usy, usz, s4)    uhat at t*, s4 = 4 sin^2((psi_t + psi_r)/2)
                // [4] (klo, sp, cp, Fhi)     kappa_lo, half-angle of psi_t + psi_r, phi/W(khi)
                // (a self pair reads [0..2] of its partner row: whole 128-bit loads)
  float4* col;  // [0] (qhx, qhy, qhz, k2)    q_j = R0^T m_j, FP32 high part
                // [1] (qlx, qly, qlz, G)     q_j low part, G = phi2 / W(k2)
  float4* rowp; // fix-up launches: per model row (s4 hi, s4 lo, c4 hi, c4 lo),
                // 4 sin^2(psi/2) and 4 cos^2(psi/2) as double-floats
};
// Pair terms are F_i G_j 2^(excess log2e) W(K) (the log W(a), log W(b) and
// log phi pieces of the reference's log_term, bounds.cpp:136/176, as linear
// factors): the exponent then only carries the small excess, so FP32 keeps
// ~1e-7 relative accuracy on the terms that matter. F_i multiplies row sums.

constexpr int kRowF4 = 5;  // float4 per model row
constexpr int kColF4 = 2;  // float4 per image column
constexpr int kRowPF4 = 1;  // float4 per model row, fix-up launches only

// Precise fix-up: a node (or child) whose cross terms carry a
// theta/B-amplified FP32 error estimate above kRedoRel of its cross mass is
// appended to a redo list by the main pass and re-evaluated by a second
// launch (kFixFull / kFixStream) whose cross pass forms the alignment angle's
// numerator x - 4 sin^2(psi/2) in FP64 from the double-float directions and a
// double-float 4 sin^2(psi/2). The main kernel only accumulates the estimate's
// amplified part (one multiply-add per row) and appends; nodes that never
// reach the threshold pay nothing else.
// kRedoRel: the threshold (DevCtx::redo_rel, default 1.2e-4 of the cross mass;
// profiles/r02_k1_variants.md)

struct Row {
  float uhx, uhy, uhz, ulx, uly, ulz, klo, khi, kst, Fhi, Fst, cp2, sp2, csp2, s4, c4, usx, usy,
      usz, klo2;
};

// Cross LB exact path: K minimum over the kappa interval (vertex case,
// bounds.cpp:160-175) with the exact W factor. s2 = 2(1 - cos B),
// c2 = 2(1 + cos B).
__device__ __noinline__ float cross_lb_exact(float klo, float khi, float k2, float s2, float c2,
                                             float K1, float e1) {
  const float cosb = 1.0f - 0.5f * s2;
  const float vertex = -cosb * k2;
  float kmin;
  if (vertex <= klo) {
    kmin = K1;
  } else if (vertex >= khi) {
    const float d = khi - k2;
    kmin = sqf(fmaxf(fmaf(d, d, khi * k2 * c2), 0.0f));
  } else {
    kmin = k2 * sqf(0.25f * s2 * c2);  // k2 sin B
  }
  return ex2f(e1 + log2w(kmin));
}

#ifndef GOSMA_SIGNSEL
#define GOSMA_SIGNSEL 1
#endif
// x = |u - v|^2 = 4 sin^2(theta/2) and y = |u + v|^2 = 4 cos^2(theta/2) of two
// double-float unit vectors (high parts h, low parts l). Only the smaller one
// is formed from the double-float difference (u - v when u.v >= 0, u + v
// otherwise) and the other is 4 minus it (|u|^2 + |v|^2 = 2 to FP64 precision;
// the complement is >= 2, so it keeps ~1e-7 relative error): 3% fewer
// instructions per pair than forming both (GOSMA_SIGNSEL=0, kept for A/B).
__device__ __forceinline__ void sincos_sq(float hx, float hy, float hz, float lx, float ly,
                                          float lz, float gx, float gy, float gz, float mx,
                                          float my, float mz, float& x, float& y) {
#if GOSMA_SIGNSEL
  const bool near = fmaf(hx, gx, fmaf(hy, gy, hz * gz)) >= 0.0f;
  const float sg = near ? -1.0f : 1.0f;
  const float vx = fmaf(sg, gx, hx) + fmaf(sg, mx, lx);
  const float vy = fmaf(sg, gy, hy) + fmaf(sg, my, ly);
  const float vz = fmaf(sg, gz, hz) + fmaf(sg, mz, lz);
  const float w = fmaf(vx, vx, fmaf(vy, vy, vz * vz));
  x = near ? w : 4.0f - w;
  y = near ? 4.0f - w : w;
#else
  const float dx = (hx - gx) + (lx - mx), dy = (hy - gy) + (ly - my), dz = (hz - gz) + (lz - mz);
  const float px = (hx + gx) + (lx + mx), py = (hy + gy) + (ly + my), pz = (hz + gz) + (lz + mz);
  x = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  y = fmaf(px, px, fmaf(py, py, pz * pz));
#endif
}

// x = |u - v|^2 alone, from the double-float difference, and y = 4 - x: the
// fast loop copies (kExact = false), whose nodes have every psi <= pi/2 and
// concentrations that make the theta-near-pi terms negligible, so y's
// absolute (not relative) precision never reaches a non-negligible term.
#ifndef GOSMA_XONLY
#define GOSMA_XONLY 1
#endif
__device__ __forceinline__ void sin_sq(float hx, float hy, float hz, float lx, float ly, float lz,
                                       float gx, float gy, float gz, float mx, float my,
                                       float mz, float& x, float& y) {
  const float dx = (hx - gx) + (lx - mx), dy = (hy - gy) + (ly - my), dz = (hz - gz) + (lz - mz);
  x = fmaf(dx, dx, fmaf(dy, dy, dz * dz));
  y = fmaxf(4.0f - x, 0.0f);  // x may round past 4 for antipodal directions
}

// One cross pair (model row i x image column j). The alignment angle
// B = max(0, theta - psi_t - psi_r) (alignment_angle_B, bounds.cpp:143-156)
// enters as 2 sin(B/2) = (x - s4) / (2 sin(theta/2) cos(psi/2) + 2 cos(theta/2) sin(psi/2))
// with x = |u - q|^2 = 4 sin^2(theta/2) from double-float directions and
// s4 = 4 sin^2(psi/2) from FP64 per-row prep: the theta ~ psi cancellation
// happens in x - s4, where both operands carry ~1e-7 relative error, instead
// of in sin/cos products.
template <bool kSame, bool kPrecise = false, bool kExact = true, bool kXo = !kExact>
__device__ __forceinline__ void cross_pair(const Row& r, const float4 qa, const float4 qb, float& l,
                                           float& u, float& ma, float& mb,
                                           const float4 rp = float4{}) {
  const float k2 = qa.w;
  // x = |u - q|^2 = 4 sin^2(theta/2), y = |u + q|^2 = 4 cos^2(theta/2), each
  // without cancellation (sincos_sq)
  constexpr bool kX = kXo && GOSMA_XONLY;
  float x, y;
  if constexpr (kX)
    sin_sq(r.uhx, r.uhy, r.uhz, r.ulx, r.uly, r.ulz, qa.x, qa.y, qa.z, qb.x, qb.y, qb.z, x, y);
  else
    sincos_sq(r.uhx, r.uhy, r.uhz, r.ulx, r.uly, r.ulz, qa.x, qa.y, qa.z, qb.x, qb.y, qb.z, x, y);
  // With sg = 2 sin(theta/2) = sqrt(x), gm = 2 cos(theta/2) = sqrt(y):
  //   den^2 = (sg cp + gm sp)^2 = x cp^2 + y sp^2 + 2 sg gm cp sp
  //   c2    = (gm cp + sg sp)^2 = y cp^2 + x sp^2 + 2 sg gm cp sp = 2(1 + cos B)
  // so one MUFU sqrt (of x*y) serves both.
  const float m = sqf(x * y) * r.csp2;
  // 2 sin(B/2) * den = x - 4 sin^2(psi/2) = 4 cos^2(psi/2) - y: take the form
  // whose operands are small (theta below / above 90 degrees).
  float num;
  if constexpr (kPrecise) {
    // the same difference in FP64 (fix-up launches): |u -+ q|^2 from the
    // double-float directions minus the double-float 4 sin^2 (4 cos^2) of psi/2
    const bool obtuse = x > y;
    const double sg = obtuse ? 1.0 : -1.0;
    const double vx = (static_cast<double>(r.uhx) + r.ulx) + sg * (static_cast<double>(qa.x) + qb.x);
    const double vy = (static_cast<double>(r.uhy) + r.uly) + sg * (static_cast<double>(qa.y) + qb.y);
    const double vz = (static_cast<double>(r.uhz) + r.ulz) + sg * (static_cast<double>(qa.z) + qb.z);
    const double w = fma(vx, vx, fma(vy, vy, vz * vz));
    num = static_cast<float>(obtuse ? (static_cast<double>(rp.z) + rp.w) - w
                                    : w - (static_cast<double>(rp.x) + rp.y));
  } else if constexpr (kX) {
    num = x - r.s4;  // x carries its relative precision on both sides of 90 deg
  } else {
    num = (x > y) ? (r.c4 - y) : (x - r.s4);
  }
  const bool bz = !(num > 0.0f);                        // theta <= psi: B = 0
  num = bz ? 0.0f : num;
  const float den2 = bz ? 1.0f : fmaf(x, r.cp2, fmaf(y, r.sp2, m));
  const float c2 = bz ? 4.0f : fmaf(y, r.cp2, fmaf(x, r.sp2, m));
  // LB: excess at the low kappa endpoint, W(K) at K's minimum
  const float ab = r.klo * k2;
  const float amb = r.klo - k2;
  const float K2lo = fmaf(amb, amb, ab * c2);
  const float rK1 = rsqf(K2lo);
  const float K1 = K2lo * rK1;
  const float D1 = K1 + r.klo + k2;
  // UB: objective at (r0, t*) (class_objective cross loop, objective.cpp:212-220)
  float xs, ys;
  if (kSame) {
    xs = x;
    ys = y;
  } else {
    const float ex = r.usx - qa.x, ey = r.usy - qa.y, ez = r.usz - qa.z;
    const float fx = r.usx + qa.x, fy = r.usy + qa.y, fz = r.usz + qa.z;
    xs = fmaf(ex, ex, fmaf(ey, ey, ez * ez));
    ys = fmaf(fx, fx, fmaf(fy, fy, fz * fz));
  }
  const float ab2 = r.kst * k2;
  const float amb2 = r.kst - k2;
  const float K2u = fmaf(amb2, amb2, ab2 * ys);
  const float rK2 = rsqf(K2u);
  const float K2 = K2u * rK2;
  const float D2 = K2 + r.kst + k2;
  // excess_LB = -ab (num/den)^2 / D1,  excess_UB = -ab2 xs / D2, one reciprocal
  const float inv = rcpf(D1 * D2 * den2) * -kL2E;
  const float g = ab * num * D2 * inv;          // e1 / num
  const float e1 = g * num;                     // (K - a - b) log2e, LB
  const float e2 = ab2 * xs * D1 * den2 * inv;  // (K - a - b) log2e, UB
  float t1 = ex2f(e1) * rK1;
  float t2 = ex2f(e2) * rK2;
  // exact paths (one rarely-taken branch): K's interior minimum
  // (cos B < -klo/k2, i.e. c2 k2 + 2 klo < 2 k2) or small K
  // (kExact = false: the node's concentrations exclude every case below
  // from non-negligible terms, see exact_needed)
  if constexpr (kExact) {
    const bool s1 = e1 > kNegligibleLog2 && (fmaf(c2, k2, r.klo2) < k2 + k2 || !(K1 > 15.0f));
    const bool s2 = e2 > kNegligibleLog2 && !(K2 > 15.0f);
    if (s1 | s2) {
      if (s1) t1 = cross_lb_exact(r.klo, r.khi, k2, 4.0f - c2, c2, K1, e1);
      if (s2) t2 = ex2f(e2 + log2w(K2));
    }
  }
  // FP32 error estimate of the LB term: B = theta - psi
  // carries ~u theta absolute error, amplified in e1 by min(x, y)/num (the
  // operand used); accumulated as sum t |e1/num| min(x,y) and sum t |e1|.
  // (the fix-up's FP64 numerator leaves only the exponent's own error)
  const float gt1 = qb.w * t1;  // G_j; F_i is applied to the row sum
  l += gt1;
  if constexpr (!kPrecise) ma = fmaf(gt1, fabsf(g) * (kX ? x : fminf(x, y)), ma);
  mb = fmaf(gt1, fabsf(e1), mb);
  u = fmaf(qb.w, t2, u);
}

// Self LB exact path: K's corner maximum (bounds.cpp:124-137) when cos A < 0
// or K small.
__device__ __noinline__ float self_lb_exact(float alo, float ahi, float blo, float bhi, float c2,
                                            float K2hh, float e1) {
  const float dll = alo - blo, dlh = alo - bhi, dhl = ahi - blo;
  const float K2ll = fmaf(dll, dll, alo * blo * c2);
  const float K2lh = fmaf(dlh, dlh, alo * bhi * c2);
  const float K2hl = fmaf(dhl, dhl, ahi * blo * c2);
  const float m = fmaxf(fmaxf(K2ll, K2lh), fmaxf(K2hl, K2hh));
  return ex2f(e1 + log2w(sqf(fmaxf(m, 0.0f))));
}

template <bool kSame, bool kExact = true>
__device__ __forceinline__ void self_pair(const float4& a0, const float4& a1, const float4& a2,
                                          const float4& a3, const float4* pa, const float4* pb,
                                          float& l, float& u, float& me) {
  // records (kRowF4 float4 per row): [0] (uh, Fst) [1] (khi, Flo, st, ct)
  // [2] (ul, kst) [3] (us, s4) [4] (klo, sp, cp, Fhi); a self pair reads
  // [0..2] of row j as three conflict-free 128-bit loads ([3] only off-centre).
  const float4 b0 = pb[0], b1 = pb[1], b2 = pb[2];
  // spread angle A = min(pi, theta + psi_i + psi_j) (bounds.cpp:108-124);
  // directions are double-float (high part in [0], low part in [2])
  float x, y;  // |u_i - u_j|^2, |u_i + u_j|^2
  if constexpr (!kExact && GOSMA_XONLY)
    sin_sq(a0.x, a0.y, a0.z, a2.x, a2.y, a2.z, b0.x, b0.y, b0.z, b2.x, b2.y, b2.z, x, y);
  else
    sincos_sq(a0.x, a0.y, a0.z, a2.x, a2.y, a2.z, b0.x, b0.y, b0.z, b2.x, b2.y, b2.z, x, y);
  const float sij = fmaf(a1.z, b1.w, a1.w * b1.z);   // sin((psi_i+psi_j)/2)
  const float cij = fmaf(a1.w, b1.w, -a1.z * b1.z);  // cos((psi_i+psi_j)/2)
  // With sg = sqrt(x) = 2 sin(theta/2), gm = sqrt(y) = 2 cos(theta/2):
  //   s2 = (sg cij + gm sij)^2 = 2(1 - cos A),  c2 = (gm cij - sg sij)^2 = 2(1 + cos A);
  // the cross products need only sg gm = sqrt(x y). A = pi once gm cij <= sg sij.
  const float cij2 = cij * cij, sij2 = sij * sij;
  const float m = 2.0f * cij * sij * sqf(x * y);
  const float gc2 = y * cij2;
  const bool api = !(cij > 0.0f) || !(gc2 > x * sij2);
  const float s2 = api ? 4.0f : fmaf(x, cij2, fmaf(y, sij2, m));
  const float c2 = api ? 0.0f : fmaf(x, sij2, gc2 - m);
  // LB: excess at the high corner, W(K) at K's corner maximum
  const float ahi = a1.x, bhi = b1.x;
  const float hh = ahi * bhi;
  const float dhh = ahi - bhi;
  const float K2hh = fmaf(dhh, dhh, hh * c2);
  const float rKhh = rsqf(K2hh);
  const float Khh = K2hh * rKhh;
  const float D1 = Khh + ahi + bhi;
  const float n1 = hh * s2;
  // UB: objective self pair at t* (objective.cpp:204-209)
  float xs, ys;
  if (kSame) {
    xs = x;
    ys = y;
  } else {
    const float4 b3 = pb[3];
    const float ex = a3.x - b3.x, ey = a3.y - b3.y, ez = a3.z - b3.z;
    const float fx = a3.x + b3.x, fy = a3.y + b3.y, fz = a3.z + b3.z;
    xs = fmaf(ex, ex, fmaf(ey, ey, ez * ez));
    ys = fmaf(fx, fx, fmaf(fy, fy, fz * fz));
  }
  const float ka = a2.w, kb = b2.w;
  const float ab2 = ka * kb;
  const float d2 = ka - kb;
  const float K2u = fmaf(d2, d2, ab2 * ys);
  const float rK2 = rsqf(K2u);
  const float K2 = K2u * rK2;
  const float D2 = K2 + ka + kb;
  const float n2 = ab2 * xs;
  const float inv = rcpf(D1 * D2) * -kL2E;
  const float e1 = n1 * D2 * inv;
  const float e2 = n2 * D1 * inv;
  float t1 = ex2f(e1) * rKhh;
  float t2 = ex2f(e2) * rK2;
  // exact paths (one rarely-taken branch, as in cross_pair)
  if constexpr (kExact) {
    const bool x1 = e1 > kNegligibleLog2 && (c2 < 2.0f || !(Khh > 15.0f));
    const bool x2 = e2 > kNegligibleLog2 && !(K2 > 15.0f);
    if (x1 | x2) {
      if (x1) t1 = self_lb_exact(pa[4].x, ahi, pb[4].x, bhi, c2, K2hh, e1);
      if (x2) t2 = ex2f(e2 + log2w(K2));
    }
  }
  const float ft1 = b1.y * t1;  // F_j (Flo); 2 F_i is applied to the row sum
  l += ft1;
  me = fmaf(ft1, fabsf(e1), me);
  u = fmaf(b0.w, t2, u);  // F_j (Fst)
}

__device__ __forceinline__ Row load_row(const WarpTables& T, int i) {
  const float4* p = T.row + i * kRowF4;
  const float4 a0 = p[0], a1 = p[1], a2 = p[2], a3 = p[3], a4 = p[4];
  Row r;
  r.uhx = a0.x;
  r.uhy = a0.y;
  r.uhz = a0.z;
  r.Fst = a0.w;
  r.khi = a1.x;
  r.ulx = a2.x;
  r.uly = a2.y;
  r.ulz = a2.z;
  r.kst = a2.w;
  r.usx = a3.x;
  r.usy = a3.y;
  r.usz = a3.z;
  r.s4 = a3.w;
  r.klo = a4.x;
  r.klo2 = 2.0f * a4.x;
  r.sp2 = a4.y * a4.y;
  r.cp2 = a4.z * a4.z;
  r.csp2 = 2.0f * a4.y * a4.z;
  r.c4 = 4.0f * r.cp2;
  r.Fhi = a4.w;
  return r;
}

template <int kG, bool kSame, bool kCross, bool kSelf, bool kPrecise, bool kExact,
          bool kXo = !kExact>
__device__ __forceinline__ void class_pairs_rows(const WarpTables& T, const ClassSpan cs, int lane,
                                            float w, double& lb_self, double& lb_cross,
                                            double& ub_self, double& ub_cross, double& lb_err,
                                            float& lb_amp) {
  const int n = cs.n1;
  // Cross terms: rows over lanes, columns broadcast.
  for (int base = 0; kCross && base < n; base += kG) {
    const int il = base + lane;
    if (il < n) {
      const Row r = load_row(T, cs.o1 + il);
      float4 rp{};
      if constexpr (kPrecise) rp = T.rowp[cs.o1 + il];
      float l = 0.0f, u = 0.0f, ma = 0.0f, mb = 0.0f;
      const float4* cp = T.col + cs.o2 * kColF4;  // pointer walk: no index math per pair
      const float4* const ce = cp + cs.n2 * kColF4;
#pragma unroll kUnrollPairs
      for (; cp < ce; cp += kColF4) cross_pair<kSame, kPrecise, kExact, kXo>(r, cp[0], cp[1], l, u, ma, mb, rp);
      lb_cross += static_cast<double>(w * r.Fhi * l);
      const float amp = 2.0f * w * r.Fhi * ma * kErrAmp;
      lb_err += static_cast<double>(
          fmaf(2.0f * w * r.Fhi, fmaf(mb, kErrExp, l * kErrTerm), amp));
#ifndef GOSMA_NO_AMP
      lb_amp += amp;
#endif
      ub_cross += static_cast<double>(w * r.Fst * u);
    }
  }
  // Self terms i<j via the circulant schedule: every unordered pair once as
  // (i, i+d mod n), d = 1..(n-1)/2, plus d = n/2 for i < n/2 when n is even.
  const int dfull = (n - 1) / 2;
  const bool even = (n % 2) == 0;
  for (int base = 0; kSelf && base < n; base += kG) {
    const int il = base + lane;
    if (il < n) {
      const int i = cs.o1 + il;
      const float4* pa = T.row + i * kRowF4;
      const float4 a0 = pa[0], a1 = pa[1], a2 = pa[2];
      const float4 a3 = kSame ? make_float4(0.f, 0.f, 0.f, 0.f) : pa[3];
      float l = 0.0f, u = 0.0f, me = 0.0f;
      const float4* const rbeg = T.row + cs.o1 * kRowF4;
      const float4* const rend = rbeg + n * kRowF4;
      const float4* pb = pa;  // partner row i + d (mod n)
#pragma unroll kUnrollPairs
      for (int d = dfull; d > 0; --d) {
        pb += kRowF4;
        pb = pb == rend ? rbeg : pb;
        self_pair<kSame, kExact>(a0, a1, a2, a3, pa, pb, l, u, me);
      }
      if (even && il < n / 2) {
        const int j = i + n / 2;
        self_pair<kSame, kExact>(a0, a1, a2, a3, pa, T.row + j * kRowF4, l, u, me);
      }
      lb_self += static_cast<double>(2.0f * w * a1.y * l);
      lb_err += static_cast<double>(2.0f * w * a1.y * fmaf(me, kErrExp, l * kErrTerm));
      ub_self += static_cast<double>(2.0f * w * a0.w * u);
    }
  }
}

// Variant for classes whose last row chunk is partial: that chunk of r rows
// gives each row k = kG / r lanes ("slots") sharing its partners round-robin
// (the node sums are sums over pairs, so any pair -> lane assignment is
// exact). Separate instantiation: the plain loops stay tighter for full chunks.
template <int kG, bool kSame, bool kCross, bool kSelf, bool kPrecise, bool kExact,
          bool kXo = !kExact>
__device__ __forceinline__ void class_pairs_tail(const WarpTables& T, const ClassSpan cs,
                                                 int lane, float w, double& lb_self,
                                                 double& lb_cross, double& ub_self,
                                                 double& ub_cross, double& lb_err,
                                                 float& lb_amp) {
  const int n = cs.n1;
  // cross terms: columns broadcast (slot s takes columns s, s+k, ...)
  for (int base = 0; kCross && base < n; base += kG) {
    const int r = min(kG, n - base), k = kG / r;
    const int il = base + lane % r, slot = lane / r;
    if (lane < r * k) {
      const Row rw = load_row(T, cs.o1 + il);
      float4 rp{};
      if constexpr (kPrecise) rp = T.rowp[cs.o1 + il];
      float l = 0.0f, u = 0.0f, ma = 0.0f, mb = 0.0f;
      const float4* cp = T.col + (cs.o2 + slot) * kColF4;
      const float4* const ce = T.col + (cs.o2 + cs.n2) * kColF4;
      const int cstep = k * kColF4;
#pragma unroll kUnrollPairs
      for (; cp < ce; cp += cstep)
        cross_pair<kSame, kPrecise, kExact, kXo>(rw, cp[0], cp[1], l, u, ma, mb, rp);
      lb_cross += static_cast<double>(w * rw.Fhi * l);
      const float amp = 2.0f * w * rw.Fhi * ma * kErrAmp;
      lb_err += static_cast<double>(
          fmaf(2.0f * w * rw.Fhi, fmaf(mb, kErrExp, l * kErrTerm), amp));
#ifndef GOSMA_NO_AMP
      lb_amp += amp;
#endif
      ub_cross += static_cast<double>(w * rw.Fst * u);
    }
  }
  // self terms: circulant (i, i+d mod n); slot s takes d = 1+s, 1+s+k, ...,
  // slot 0 the half-way pair of an even n
  const int dfull = (n - 1) / 2;
  const bool even = (n % 2) == 0;
  for (int base = 0; kSelf && base < n; base += kG) {
    const int r = min(kG, n - base), k = kG / r;
    const int il = base + lane % r, slot = lane / r;
    if (lane < r * k) {
      const int i = cs.o1 + il;
      const float4* pa = T.row + i * kRowF4;
      const float4 a0 = pa[0], a1 = pa[1], a2 = pa[2];
      const float4 a3 = kSame ? make_float4(0.f, 0.f, 0.f, 0.f) : pa[3];
      float l = 0.0f, u = 0.0f, me = 0.0f;
      // partner row il + d (mod n), walked as a pointer
      const float4* const rbeg = T.row + cs.o1 * kRowF4;
      const float4* const rend = rbeg + n * kRowF4;
      const int step = k * kRowF4;
      const float4* pb = pa + (1 + slot - k) * kRowF4;
#pragma unroll kUnrollPairs
      for (int d = 1 + slot; d <= dfull; d += k) {
        pb += step;
        pb = pb >= rend ? pb - n * kRowF4 : pb;
        self_pair<kSame, kExact>(a0, a1, a2, a3, pa, pb, l, u, me);
      }
      if (even && slot == 0 && il < n / 2) {
        const int j = i + n / 2;
        self_pair<kSame, kExact>(a0, a1, a2, a3, pa, T.row + j * kRowF4, l, u, me);
      }
      lb_self += static_cast<double>(2.0f * w * a1.y * l);
      lb_err += static_cast<double>(2.0f * w * a1.y * fmaf(me, kErrExp, l * kErrTerm));
      ub_self += static_cast<double>(2.0f * w * a0.w * u);
    }
  }
}

#ifndef GOSMA_FAST_MIN_G
#define GOSMA_FAST_MIN_G 16
#endif
constexpr int kFastMinG = GOSMA_FAST_MIN_G;
constexpr int kSibFastMinG = 8;  // the class-streamed siblings mode (semantic solves)
#ifndef GOSMA_STREAM_FAST_MIN_G
#define GOSMA_STREAM_FAST_MIN_G 16
#endif
constexpr int kStreamFastMinG = GOSMA_STREAM_FAST_MIN_G;  // class-streamed full mode

template <int kG, bool kSame, bool kCross, bool kSelf, bool kTail, bool kPrecise, bool kExact,
          bool kXo = !kExact>
__device__ __forceinline__ void class_pairs_part(const WarpTables& T, const ClassSpan cs, int lane,
                                                 float w, double& lb_self, double& lb_cross,
                                                 double& ub_self, double& ub_cross,
                                                 double& lb_err, float& lb_amp) {
  if constexpr (kTail)
    class_pairs_tail<kG, kSame, kCross, kSelf, kPrecise, kExact, kXo>(
        T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross, lb_err, lb_amp);
  else
    class_pairs_rows<kG, kSame, kCross, kSelf, kPrecise, kExact, kXo>(
        T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross, lb_err, lb_amp);
}

// exact: bit 0 the cross loop needs the exact-path copy, bit 1 the self loop,
// bit 2 the cross loop's fast copy must keep the sign-selected angles (a row's
// psi too large for x-only; FastScore); the cross sums come first, as in
// class_pairs_rows.
template <int kG, bool kSame, bool kCross, bool kSelf, bool kTail, bool kPrecise,
          int kMinG = kFastMinG>
__device__ __forceinline__ void class_pairs(const WarpTables& T, const ClassSpan cs, int lane,
                                            float w, double& lb_self, double& lb_cross,
                                            double& ub_self, double& ub_cross, double& lb_err,
                                            float& lb_amp, unsigned exact) {
  // the fast loop copies only for groups of >= kMinG lanes (classes of > 24
  // rows in the full modes): short loops gain nothing from them and lose to
  // the larger code; the class-streamed siblings mode gains at 8 lanes too
  if (kG < kMinG) exact = 7u;
  if constexpr (kCross) {
    // (8-lane groups: no sign-selected fast copy; its code cost the
    // class-streamed siblings mode 3% there)
    if (exact & 1u || (kG < 16 && (exact & 4u))) {
      class_pairs_part<kG, kSame, true, false, kTail, kPrecise, true>(
          T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross, lb_err, lb_amp);
    } else if (exact & 4u) {
      if constexpr (kG >= 16)
        class_pairs_part<kG, kSame, true, false, kTail, kPrecise, false, false>(
            T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross, lb_err, lb_amp);
    } else {
      class_pairs_part<kG, kSame, true, false, kTail, kPrecise, false>(
          T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross, lb_err, lb_amp);
    }
  }
  if constexpr (kSelf) {
    if (exact & 2u)
      class_pairs_part<kG, kSame, false, true, kTail, kPrecise, true>(
          T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross, lb_err, lb_amp);
    else
      class_pairs_part<kG, kSame, false, true, kTail, kPrecise, false>(
          T, cs, lane, w, lb_self, lb_cross, ub_self, ub_cross, lb_err, lb_amp);
  }
}

// Whether a node's terms can skip the rare exact paths (small K, the cross
// LB's interior K minimum, the self LB's corner maximum past 90 degrees) and
// take the fast loop copies (no exact branches, x-only angles via sin_sq).
// Every skipped case is shown to leave the pair's log2 exponent below -64,
// i.e. the term at most 2^-64 of its F_i G_j W(K) prefactor (below 1e-13 of
// the node's |term| mass even for kappa2 / kappa1 ratios of 1e5), so skipping
// it moves the bound by far less than the 2e-7 mass margin. With
// |excess| = ab (1 - cos) 2 / (K + a + b) >= ab (1 - cos) / (a + b) and
// L = log2 e:
//  * cross LB interior K minimum (cos B < -kappa_lo / k2):
//    |e| > L ab (1 + a/b) / (a + b) = L kappa_lo, so kappa_lo >= 45;
//  * K <= 15 (cross LB / UB, self LB / UB): |a - b| <= 15 and ab c <= 225
//    force 1 - cos >= 2 - 113/ab and |e| >= L (4ab - 225) / (15 + a + b),
//    above 64 once both concentrations are >= 30 (kappa_lo, kappa_hi,
//    kappa at t* >= 45 here, the partner within 15 of it);
//  * self LB corner maximum (cos A < 0): |e| >= L H(kappa_hi_i, kappa_hi_j),
//    so kappa_hi >= 90 (H = ab / (a + b));
//  * sin_sq's y = 4 - x has absolute, not relative, precision: it matters only
//    for theta near pi, where B >= pi - psi gives |e| >= L H(kappa_lo, k2)
//    (1 + cos psi) = L H 2 cos^2(psi/2) (and the UB / self terms at
//    theta ~ pi have |e| >= 2 L H): H(kappa_lo, min k2) min(1, 2 cp^2) >= 45,
//    with cp = 0 exempt (psi clamped at pi: every cross pair has B = 0).
// Per row three scores, >= 1 when the cross loop may skip the exact paths
// (kappa_lo, kappa at t* >= 45), when its fast copy may use x-only angles
// (H(kappa_lo, min k2) min(1, 2 cos^2(psi/2)) >= 45), and when the self loop
// may take its fast copy (kappa_hi >= 90, kappa at t* >= 45); the node
// decisions are one vote each over its rows (group-uniform: the loops never
// diverge inside a group). Nodes failing only the x-only score (psi near pi,
// e.g. rotation-level-1 cubes) run the fast cross copy with sign-selected
// angles.
// GOSMA_FAST_SCALE scales the thresholds (A/B builds).
#ifndef GOSMA_FAST_SCALE
#define GOSMA_FAST_SCALE 1.0f
#endif
struct FastScore {
  float cross = INFINITY, self = INFINITY, xonly = INFINITY;
  __device__ __forceinline__ void add(float klo, float khi, float kst, float k2_min, double cp) {
    constexpr float kA = 1.0f / (45.0f * GOSMA_FAST_SCALE), kB = 1.0f / (90.0f * GOSMA_FAST_SCALE);
    const float h = klo * k2_min / (klo + k2_min);
    const float c = cp > 0.0 ? fminf(1.0f, static_cast<float>(2.0 * cp * cp)) : 1.0f;
    cross = fminf(cross, fminf(klo, kst) * kA);
    xonly = fminf(xonly, h * c * kA);
    self = fminf(self, fminf(kst * kA, khi * kB));
  }
  __device__ __forceinline__ void reset() { cross = self = xonly = INFINITY; }
  // this lane's rows: bit 0 the cross loop needs the exact copy, bit 1 the
  // self loop, bit 2 the cross loop's fast copy needs the sign-selected angles
  __device__ __forceinline__ unsigned need() const {
    return (cross >= 1.0f ? 0u : 1u) | (self >= 1.0f ? 0u : 2u) | (xonly >= 1.0f ? 0u : 4u);
  }
};

// 1/sqrt(x) in FP64 for normal x > 0: the MUFU FP64 estimate
// (rsqrt.approx.f64, full exponent range) and two branch-free Newton steps.
// The libdevice rsqrt carries a special-case branch whose reconvergence
// points stalled the prologue's warps (profiles/r02_k1_variants.md).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double hx = 0.5 * x;
  y = y * fma(-hx * y, y, 1.5);
  y = y * fma(-hx * y, y, 1.5);
  return y;
}

// Half-angle of psi_trans (se3.cpp:72-92) for a mean outside the cuboid: the
// vertex with the largest angle to the centre direction has the smallest
// cosine c_hat . v_hat. FP32 ranks the vertices, FP64 evaluates the FP32 best
// and (rarely) every other vertex within 1e-6 of it, keeping the largest
// FP64 angle (first vertex on exact ties): returns sin and cos of half the
// angle as |c_hat - v_hat|/2 and |c_hat + v_hat|/2. The best vertex is
// evaluated with its signs as data, so lanes with different best vertices
// share one FP64 evaluation instead of diverging over all eight.
__device__ __forceinline__ void psi_trans_half(double u0, double u1, double u2, double h0,
                                               double h1, double h2, double c0, double c1,
                                               double c2, double& st, double& ct) {
  const float fu0 = static_cast<float>(u0), fu1 = static_cast<float>(u1),
              fu2 = static_cast<float>(u2);
  const float fh0 = static_cast<float>(h0), fh1 = static_cast<float>(h1),
              fh2 = static_cast<float>(h2);
  const float fc0 = static_cast<float>(c0), fc1 = static_cast<float>(c1),
              fc2 = static_cast<float>(c2);
  float cosv[8];
  float best = 2.0f;
  int sb = 0;
#pragma unroll
  for (int s = 0; s < 8; ++s) {
    const float vx = fu0 - ((s & 4) ? fh0 : -fh0);
    const float vy = fu1 - ((s & 2) ? fh1 : -fh1);
    const float vz = fu2 - ((s & 1) ? fh2 : -fh2);
    const float rv = rsqf(fmaf(vx, vx, fmaf(vy, vy, vz * vz)));
    cosv[s] = fmaf(fc0, vx, fmaf(fc1, vy, fc2 * vz)) * rv;
    if (cosv[s] < best) {
      best = cosv[s];
      sb = s;
    }
  }
  // FP64 squared half-chords |c - w|^2, |c + w|^2 of vertex s
  auto chord = [&](int s, double& sd, double& pd) {
    const double vx = u0 - ((s & 4) ? h0 : -h0);
    const double vy = u1 - ((s & 2) ? h1 : -h1);
    const double vz = u2 - ((s & 1) ? h2 : -h2);
    const double iv = rsqrt_nr(vx * vx + vy * vy + vz * vz);
    const double wx = vx * iv, wy = vy * iv, wz = vz * iv;
    const double ex = c0 - wx, ey = c1 - wy, ez = c2 - wz;
    sd = ex * ex + ey * ey + ez * ez;
    const double px = c0 + wx, py = c1 + wy, pz = c2 + wz;
    pd = px * px + py * py + pz * pz;
  };
  double bs, bc;
  chord(sb, bs, bc);
  bool tie = false;
#pragma unroll
  for (int s = 0; s < 8; ++s) tie |= (s != sb) & (cosv[s] <= best + 1e-6f);
  if (tie) {  // FP32 near-ties (rare): decide in FP64, one branch for all
    int bsi = sb;
#pragma unroll
    for (int s = 0; s < 8; ++s) {
      if (s != sb && cosv[s] <= best + 1e-6f) {
        double sd, pd;
        chord(s, sd, pd);
        if (sd > bs || (sd == bs && s < bsi)) {
          bs = sd;
          bc = pd;
          bsi = s;
        }
      }
    }
  }
  st = bs > 0.0 ? 0.5 * bs * rsqrt_nr(bs) : 0.0;
  ct = bc > 0.0 ? 0.5 * bc * rsqrt_nr(bc) : 0.0;
}

// kMode: kModeFull = every term per node; kSelfOnly = per distinct translation
// cuboid, the translation-only (self + diagonal) sums; kCrossCached = per node,
// the cross terms plus the cached self sums of the node's cuboid; kSiblings =
// per rotation-split parent: the cuboid prologue and self sums once, then the
// cross sums of its 8 children (subdivide_adaptive, se3.cpp:124-131).
// kModeStream = the full mode for multi-class contexts, one class's table at
// a time (a separate instantiation: the single-class kernel is unchanged).
enum {
  kModeFull = 0,
  kSelfOnly = 1,
  kCrossCached = 2,
  kSiblings = 3,
  kModeStream = 4,
  kSiblingsStream = 5,  // siblings mode of a multi-class context, one class's table at a time
  kFixFull = 6,         // precise fix-up of redo-list entries (single class)
  kFixStream = 7        // precise fix-up, multi-class context
};
// per-group extra shared memory of the siblings modes: the 8 children's R
// (72 doubles, computed by 8 lanes at once) and (streamed) their {lb, ub,
// err, amplified err} cross sums (32 doubles)
constexpr int kSibStreamExtraF4 = (72 + 32) * 8 / 16;

// Rodrigues R0 = rotation_matrix(rc) (se3.cpp:21-31), FP64, from sin and
// cos of theta = |rc| (unused when theta^2 < 1e-16).
__device__ __forceinline__ void rodrigues_sc(double rc0, double rc1, double rc2, double th2,
                                             double s, double co, double R[9]) {
  double a, c;
  if (th2 < 1e-16) {
    a = 1.0;
    c = 0.5;
  } else {
    const double ith = rsqrt_nr(th2);  // 1 / theta
    a = s * ith;
    c = (1.0 - co) * (ith * ith);
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

__device__ __forceinline__ void rodrigues(double rc0, double rc1, double rc2, double R[9]) {
  const double th2 = rc0 * rc0 + rc1 * rc1 + rc2 * rc2;
  double s = 0.0, co = 1.0;
  if (!(th2 < 1e-16)) sincos(th2 * rsqrt_nr(th2), &s, &co);
  rodrigues_sc(rc0, rc1, rc2, th2, s, co, R);
}

// Half-angle of psi_t + psi_r per row (B = 0 once the sum reaches pi) from the
// FP64 psi_t half-angles: the rotation-dependent row fields.
__device__ __forceinline__ void half_angles(double st, double ct, double s_r, double c_r,
                                            double& sp, double& cp) {
  sp = st * c_r + ct * s_r;
  cp = ct * c_r - st * s_r;
  if (!(cp > 0.0)) {
    sp = 1.0;
    cp = 0.0;
  }
}

// q_j = R0^T m_j (bounds.cpp:97-102), double-float columns.
__device__ __forceinline__ void column_prep(const WarpTables& T, const DevCtx& ctx, int lane,
                                            int step, const double R[9]) {
  for (int j = lane; j < ctx.n2_total; j += step) {
    const double x0 = ctx.m[3 * j], x1 = ctx.m[3 * j + 1], x2 = ctx.m[3 * j + 2];
    const double q0 = R[0] * x0 + R[3] * x1 + R[6] * x2;
    const double q1 = R[1] * x0 + R[4] * x1 + R[7] * x2;
    const double q2 = R[2] * x0 + R[5] * x1 + R[8] * x2;
    const float f0 = static_cast<float>(q0), f1 = static_cast<float>(q1),
                f2 = static_cast<float>(q2);
    T.col[j * kColF4] = make_float4(f0, f1, f2, ctx.kappa2[j]);
    T.col[j * kColF4 + 1] = make_float4(static_cast<float>(q0 - f0), static_cast<float>(q1 - f1),
                                        static_cast<float>(q2 - f2), ctx.g2[j]);
  }
}

// Columns [o2, o2 + n2) of the context into table slots 0..n2-1.
__device__ __forceinline__ void column_prep_span(const WarpTables& T, const DevCtx& ctx, int lane,
                                                 int step, const double R[9], int o2, int n2) {
  for (int jl = lane; jl < n2; jl += step) {
    const int j = o2 + jl;
    const double x0 = ctx.m[3 * j], x1 = ctx.m[3 * j + 1], x2 = ctx.m[3 * j + 2];
    const double q0 = R[0] * x0 + R[3] * x1 + R[6] * x2;
    const double q1 = R[1] * x0 + R[4] * x1 + R[7] * x2;
    const double q2 = R[2] * x0 + R[5] * x1 + R[8] * x2;
    const float f0 = static_cast<float>(q0), f1 = static_cast<float>(q1),
                f2 = static_cast<float>(q2);
    T.col[jl * kColF4] = make_float4(f0, f1, f2, ctx.kappa2[j]);
    T.col[jl * kColF4 + 1] = make_float4(static_cast<float>(q0 - f0), static_cast<float>(q1 - f1),
                                         static_cast<float>(q2 - f2), ctx.g2[j]);
  }
}

#ifndef GOSMA_MIN_BLOCKS
#define GOSMA_MIN_BLOCKS 7
#endif
// CTAs per SM the register allocation targets (72 registers at 7). The
// class-streamed siblings mode (semantic solves) runs best at 5 (96
// registers: its per-class / per-child loops otherwise rematerialise the
// table addresses; 8 x (8x4) siblings 2.04 -> 1.93 ms, 8 x (32x16) 15.6 ->
// 14.6 ms); every other mode loses at 5 or 6 (profiles/r02_k1_variants.md).
#ifndef GOSMA_SIB_MIN_BLOCKS
#define GOSMA_SIB_MIN_BLOCKS 5
#endif
constexpr int min_blocks_for(int mode) {
  return mode == kSiblingsStream ? GOSMA_SIB_MIN_BLOCKS : GOSMA_MIN_BLOCKS;
}
template <int kMode, int kG, bool kTail>
__global__ void __launch_bounds__(kWarpsPerCta * 32, min_blocks_for(kMode))
    eval_bounds_kernel(const DevCtx ctx, const EvalArgs args) {
  extern __shared__ float4 smem4[];
  __shared__ GroupScratch gscratch;
  const int wl = threadIdx.x & 31;
  const int lane = kG <= 32 ? (wl & (kG - 1)) : static_cast<int>(threadIdx.x);  // in the group
  const int gbase = kG <= 32 ? (wl & ~(kG - 1)) : 0;
  const unsigned gm = kG >= 32 ? kFull : (((1u << kG) - 1u) << gbase);
  const int group = static_cast<int>(threadIdx.x) / kG;
  const Group<kG> G{gm, gbase, &gscratch};
  // class-streamed full mode (multi-class contexts): the table holds one
  // class's rows and columns at a time, so it is sized by the largest class
  // fix-up launches run the full (or class-streamed) mode on redo-list
  // entries with the FP64-numerator cross pass
  constexpr bool kFix = kMode == kFixFull || kMode == kFixStream;
  constexpr bool streamed =
      kMode == kModeStream || kMode == kSiblingsStream || kMode == kFixStream;
  constexpr bool kSib = kMode == kSiblings || kMode == kSiblingsStream;
  const int N1 = ctx.n1_total;  // every model mean (feasibility scans)
  const int TN1 = streamed ? ctx.max_n1 : N1, TN2 = streamed ? ctx.max_n2 : ctx.n2_total;
  const size_t table_f4 =
      static_cast<size_t>(kRowF4 * TN1 + kColF4 * TN2 + (kFix ? kRowPF4 * TN1 : 0));
  const size_t per_warp_f4 = table_f4 + (kSib ? kSibStreamExtraF4 : 0);
  float4* base = smem4 + group * per_warp_f4;
  WarpTables T;
  T.row = base;
  T.col = base + kRowF4 * TN1;
  T.rowp = kFix ? T.col + kColF4 * TN2 : nullptr;  // (a constant outside the fix-up)
  // redo-list append (main launches): the evaluated node's record, re-read
  // from memory so no node coordinate stays live through the pair loops;
  // child >= 0: rotation child `child` of the (parent) record
  auto redo = [&](long long rec, int child, long long slot) {
    const unsigned long long k = atomicAdd(args.redo_count, 1ull);
    if (static_cast<long long>(k) >= args.redo_cap) return;
    const double* in = args.nodes + 11 * rec;
    double* o = args.redo_nodes + 11 * k;
    for (int q = 0; q < 11; ++q) o[q] = in[q];
    if (child >= 0) {  // subdivide_adaptive's rotation child (se3.cpp:124-131)
      const double h = 0.5 * in[3];
      o[0] = in[0] + h * ((child & 4) ? 1 : -1);
      o[1] = in[1] + h * ((child & 2) ? 1 : -1);
      o[2] = in[2] + h * ((child & 1) ? 1 : -1);
      o[3] = h;
    }
    args.redo_slot[k] = slot;
  };
  const double zeta = ctx.zeta;
  const double zeta2 = zeta * zeta;
  // fix-up launches: the count stays on the device (it may exceed the list's
  // capacity, whose overflow keeps its FP32 bounds); an empty list exits
  // before any work-counter traffic
  const long long n_items = args.n_dev ? min(*args.n_dev, args.n) : args.n;
  if (n_items <= 0) return;
  for (;;) {
    long long node = 0;
    if (lane == 0) node = static_cast<long long>(atomicAdd(args.work, 1u));
    node = G.bcast0(node);
    if (node >= n_items) break;
    // item lists: full mode over a subset (node = slot); siblings: the item
    // is a selection index k, the parent the pool slot sel[k], the outputs
    // are children 8k .. 8k+7
    long long item = node;
    if (args.item_index) node = args.item_index[node];
    if (kSib) {
      item = node;
      node = args.sel[node];
    }

    // ---- node fetch (gosma_node: rc[3], rhw, tc[3], thw[3], lower)
    double v = 0.0, v2 = 0.0;
    double nv[kG == 1 ? 11 : 1];  // one-lane groups: the lane reads its node itself
    if constexpr (kG == 1) {
      for (int k = 0; k < 11; ++k) nv[k] = args.nodes[node * 11 + k];
    } else {
      if (lane < 11) v = args.nodes[node * 11 + lane];
      if (kG < 11 && lane < 11 - kG) v2 = args.nodes[node * 11 + kG + lane];
    }
    if constexpr (kG > 32) {
      if (lane < 11) gscratch.node[lane] = v;
      __syncthreads();
    }
    auto fetch = [&](int k) -> double {
      if constexpr (kG == 1) {
        return nv[k];
      } else if constexpr (kG > 32) {
        return gscratch.node[k];
      } else {
        if (kG < 11 && k >= kG) return __shfl_sync(gm, v2, k - kG, kG);
        return __shfl_sync(gm, v, k, kG);
      }
    };
    const double rc0 = fetch(0), rc1 = fetch(1), rc2 = fetch(2);
    const double rhw = fetch(3);
    const double tc0 = fetch(4), tc1 = fetch(5), tc2 = fetch(6);
    const double h0 = fetch(7), h1 = fetch(8), h2 = fetch(9);
    const double parent_lower = fetch(10);

    // ---- feasibility scan (feasible_wrt_zeta, se3.cpp:94-100)
    bool infeasible = false;
    for (int mb = 0; mb < N1; mb += kG) {
      const int mi = mb + lane;
      bool hit = false;
      if (mi < N1) {
        const double* mu = ctx.mu + 3 * mi;
        const double f0 = fabs(mu[0] - tc0) + h0;
        const double f1 = fabs(mu[1] - tc1) + h1;
        const double f2 = fabs(mu[2] - tc2) + h2;
        hit = norm_below(__dadd_rn(__dadd_rn(__dmul_rn(f0, f0), __dmul_rn(f1, f1)),
                                   __dmul_rn(f2, f2)),
                         zeta, zeta2);
      }
      if (G.any(hit)) {
        infeasible = true;
        break;
      }
    }

    // ---- rotation: R0 = rotation_matrix(rc) (se3.cpp:21-31), psi_r (se3.cpp:68-70)
    double R[9];
    double s_r = 0.0, c_r = 1.0;
    if (!kSib) {
      const double psi_r = fmin(sqrt(3.0) * rhw, M_PI);
      const double th2 = rc0 * rc0 + rc1 * rc1 + rc2 * rc2;
      if constexpr (kG == 1) {
        rodrigues(rc0, rc1, rc2, R);
        sincos(0.5 * psi_r, &s_r, &c_r);
      } else {
        // one FP64 sincos for both angles: even lanes theta = |rc| (Rodrigues),
        // odd lanes psi_r / 2, exchanged with a shuffle
        const bool odd = (lane & 1) != 0;
        double s1, c1;
        sincos(odd ? 0.5 * psi_r : (th2 < 1e-16 ? 0.0 : th2 * rsqrt_nr(th2)), &s1, &c1);
        const double sr0 = G.shfl(s1, 0), cr0 = G.shfl(c1, 0);
        s_r = G.shfl(s1, 1);
        c_r = G.shfl(c1, 1);
        rodrigues_sc(rc0, rc1, rc2, th2, sr0, cr0, R);
      }
    } else {
      // the 8 rotation children share psi_r (their half-width 0.5 rhw): the
      // rows are prepared once with it (psi_t + psi_r half-angles)
      const double psi_c = fmin(sqrt(3.0) * (0.5 * rhw), M_PI);
      sincos(0.5 * psi_c, &s_r, &c_r);
    }

    // ---- feasible_center (bounds.cpp:187-214): t*, warp-cooperative scan
    double ts0 = tc0, ts1 = tc1, ts2 = tc2;
    bool have_center = false;
    if (!infeasible) {
      for (int proj = 0; proj <= 8; ++proj) {
        int off = -1;
        for (int mb = 0; mb < N1; mb += kG) {
          const int mi = mb + lane;
          bool hit = false;
          if (mi < N1) {
            const double* mu = ctx.mu + 3 * mi;
            const double d0 = __dsub_rn(mu[0], ts0), d1 = __dsub_rn(mu[1], ts1),
                         d2 = __dsub_rn(mu[2], ts2);
            hit = norm_below(
                __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)),
                zeta, zeta2);
          }
          const int f = G.first(hit);
          if (f >= 0) {
            off = mb + f;
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
        const double nn =
            sqrt(__dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2)));
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
        ts0 = fmin(fmax(__dadd_rn(mu[0], __dmul_rn(d0, rad)), __dsub_rn(tc0, h0)),
                   __dadd_rn(tc0, h0));
        ts1 = fmin(fmax(__dadd_rn(mu[1], __dmul_rn(d1, rad)), __dsub_rn(tc1, h1)),
                   __dadd_rn(tc1, h1));
        ts2 = fmin(fmax(__dadd_rn(mu[2], __dmul_rn(d2, rad)), __dsub_rn(tc2, h2)),
                   __dadd_rn(tc2, h2));
      }
    }
    const bool same = (ts0 == tc0) && (ts1 == tc1) && (ts2 == tc2);

    // ---- per-row prep: kappa interval, psi_t, projections; row i of the
    // context into table slot `slot`
    double lb_self = 0.0, lb_cross = 0.0, ub_self = 0.0, ub_cross = 0.0, lb_err = 0.0;
    float lb_amp = 0.0f;  // the theta/B-amplified part of the cross terms' error estimate
    double st_max = 0.0;
    FastScore fs;  // fast-loop eligibility of this lane's rows
    auto prep_row = [&](int i, int slot, float& dsl, float& dsu) {
      const double m0 = ctx.mu[3 * i], m1 = ctx.mu[3 * i + 1], m2 = ctx.mu[3 * i + 2];
      const double is2 = ctx.inv_s2[i];
      const double u0 = m0 - tc0, u1 = m1 - tc1, u2 = m2 - tc2;
      const double a0 = fabs(u0), a1 = fabs(u1), a2 = fabs(u2);
      // point_cuboid_distance (se3.cpp:60-66); dlo floored at zeta
      const double o0 = fmax(a0 - h0, 0.0), o1 = fmax(a1 - h1, 0.0), o2 = fmax(a2 - h2, 0.0);
      const double dlo2 = fmax(o0 * o0 + o1 * o1 + o2 * o2, zeta2);
      const double dhi2 = (a0 + h0) * (a0 + h0) + (a1 + h1) * (a1 + h1) + (a2 + h2) * (a2 + h2);
      const float klo = static_cast<float>(dlo2 * is2 + 1.0);
      const float khi = static_cast<float>(dhi2 * is2 + 1.0);
      const double un2 = u0 * u0 + u1 * u1 + u2 * u2;
      double c0 = 1.0, c1 = 0.0, c2 = 0.0;  // UnitX when the mean is at the centre
      if (un2 > 1e-24) {
        const double inv = rsqrt_nr(un2);
        c0 = u0 * inv;
        c1 = u1 * inv;
        c2 = u2 * inv;
      }
      double st, ct;
      if (a0 <= h0 && a1 <= h1 && a2 <= h2) {
        st = 1.0;  // psi_t = pi
        ct = 0.0;
      } else {
        psi_trans_half(u0, u1, u2, h0, h1, h2, c0, c1, c2, st, ct);
      }
      st_max = fmax(st_max, st);
      double sp, cp;
      half_angles(st, ct, s_r, c_r, sp, cp);
      // UB projection at t* (project_model, objective.cpp:175-192)
      const double v0 = m0 - ts0, v1 = m1 - ts1, v2 = m2 - ts2;
      const double vn2 = v0 * v0 + v1 * v1 + v2 * v2;
      const float kst = static_cast<float>(vn2 * is2 + 1.0);
      fs.add(klo, khi, kst, ctx.min_k2, cp);
      const double iv = rsqrt_nr(vn2);
      const float phi = static_cast<float>(ctx.phi1[i]);
      dsl += diag_term(phi, klo);
      dsu += diag_term(phi, kst);
      // phi / W(k) = phi * k / (1 - e^{-2k}) (k >= 1)
      const float Flo = phi * klo * rcpf(1.0f - ex2f(-2.0f * kL2E * klo));
      const float Fhi = phi * khi * rcpf(1.0f - ex2f(-2.0f * kL2E * khi));
      const float Fst = phi * kst * rcpf(1.0f - ex2f(-2.0f * kL2E * kst));
      const float uhx = static_cast<float>(c0), uhy = static_cast<float>(c1),
                  uhz = static_cast<float>(c2);
      float4* pr = T.row + slot * kRowF4;
      pr[0] = make_float4(uhx, uhy, uhz, Fst);
      pr[1] = make_float4(khi, Flo, static_cast<float>(st), static_cast<float>(ct));
      pr[2] = make_float4(static_cast<float>(c0 - uhx), static_cast<float>(c1 - uhy),
                          static_cast<float>(c2 - uhz), kst);
      pr[3] = make_float4(static_cast<float>(v0 * iv), static_cast<float>(v1 * iv),
                          static_cast<float>(v2 * iv), static_cast<float>(4.0 * sp * sp));
      pr[4] = make_float4(klo, static_cast<float>(sp), static_cast<float>(cp), Fhi);
      if constexpr (kFix) {
        const double s4 = 4.0 * sp * sp, c4 = 4.0 * cp * cp;
        const float s4h = static_cast<float>(s4), c4h = static_cast<float>(c4);
        T.rowp[slot] = make_float4(s4h, static_cast<float>(s4 - s4h), c4h,
                                   static_cast<float>(c4 - c4h));
      }
    };
    if constexpr (!streamed) {
      for (int c = 0; c < ctx.n_classes; ++c) {
        const ClassSpan cs = ctx.cls[c];
        const float w = static_cast<float>(ctx.cls_w[c]);
        float dsl = 0.0f, dsu = 0.0f;
        for (int il = lane; il < cs.n1; il += kG) prep_row(cs.o1 + il, cs.o1 + il, dsl, dsu);
        if (!infeasible && kMode != kCrossCached) {
          lb_self += static_cast<double>(w * dsl);
          lb_err += static_cast<double>(w * dsl * kErrTerm);
          ub_self += static_cast<double>(w * dsu);
        }
      }
    } else if constexpr (kMode == kModeStream || kMode == kFixStream) {
      // one class at a time: rows, columns, then its pairs
      for (int c = 0; c < ctx.n_classes; ++c) {
        const ClassSpan cs = ctx.cls[c];
        const float w = static_cast<float>(ctx.cls_w[c]);
        float dsl = 0.0f, dsu = 0.0f;
        G.sync();  // the previous class's pairs are done with the table
        fs.reset();
        for (int il = lane; il < cs.n1; il += kG) prep_row(cs.o1 + il, il, dsl, dsu);
        if (infeasible) continue;  // (rows still feed the split decision)
        const unsigned exact = kG < kStreamFastMinG ? 7u : G.bor3(fs.need());
        lb_self += static_cast<double>(w * dsl);
        lb_err += static_cast<double>(w * dsl * kErrTerm);
        ub_self += static_cast<double>(w * dsu);
        column_prep_span(T, ctx, lane, kG, R, cs.o2, cs.n2);
        G.sync();
#ifndef GOSMA_PREP_ONLY
        const ClassSpan loc{0, cs.n1, 0, cs.n2};
        if (same) {
          class_pairs<kG, true, true, true, kTail, kFix, kStreamFastMinG>(T, loc, lane, w, lb_self, lb_cross,
                                                         ub_self, ub_cross, lb_err, lb_amp, exact);
        } else {
          class_pairs<kG, false, true, true, kTail, kFix, kStreamFastMinG>(T, loc, lane, w, lb_self, lb_cross,
                                                          ub_self, ub_cross, lb_err, lb_amp, exact);
        }
#endif
      }
    }
    if constexpr (kMode == kSiblingsStream) {
      // one cuboid, 8 rotation children, one class at a time: the class's
      // rows (with the children's shared psi_r) and self sums, then per child
      // its columns and cross sums, accumulated per child in shared memory
      double* const Rcs = reinterpret_cast<double*>(base + table_f4);  // [8][9]
      double* const acc = Rcs + 72;                                      // [8][4]
      const double hr = 0.5 * rhw;
      for (int ch = lane; ch < 8; ch += kG) {
        const int sx = (ch & 4) ? 1 : -1, sy = (ch & 2) ? 1 : -1, sz = (ch & 1) ? 1 : -1;
        rodrigues(rc0 + hr * sx, rc1 + hr * sy, rc2 + hr * sz, Rcs + 9 * ch);
      }
      for (int k = lane; k < 32; k += kG) acc[k] = 0.0;
      double sl_self = 0.0, su_self = 0.0, se_self = 0.0;
      for (int c = 0; c < ctx.n_classes; ++c) {
        const ClassSpan cs = ctx.cls[c];
        const float w = static_cast<float>(ctx.cls_w[c]);
        float dsl = 0.0f, dsu = 0.0f;
        G.sync();  // the previous class's pairs are done with the table
        fs.reset();
        for (int il = lane; il < cs.n1; il += kG) prep_row(cs.o1 + il, il, dsl, dsu);
        if (infeasible) continue;  // (rows still feed the split decision)
        const unsigned exact = kG < kSibFastMinG ? 7u : G.bor3(fs.need());
        sl_self += static_cast<double>(w * dsl);
        se_self += static_cast<double>(w * dsl * kErrTerm);
        su_self += static_cast<double>(w * dsu);
        G.sync();
        const ClassSpan loc{0, cs.n1, 0, cs.n2};
        double dl = 0.0, du = 0.0;
#ifndef GOSMA_PREP_ONLY
        if (same) {
          class_pairs<kG, true, false, true, kTail, false, kSibFastMinG>(T, loc, lane, w, sl_self, dl, su_self,
                                                           du, se_self, lb_amp, exact);
        } else {
          class_pairs<kG, false, false, true, kTail, false, kSibFastMinG>(T, loc, lane, w, sl_self, dl, su_self,
                                                            du, se_self, lb_amp, exact);
        }
#endif
        for (int ch = 0; ch < 8; ++ch) {
          G.sync();  // the previous child's pairs are done with the columns
          column_prep_span(T, ctx, lane, kG, Rcs + 9 * ch, cs.o2, cs.n2);
          G.sync();
          double lcr = 0.0, ucr = 0.0, ecr = 0.0;
          float acr = 0.0f;
#ifndef GOSMA_PREP_ONLY
          if (same) {
            class_pairs<kG, true, true, false, kTail, false, kSibFastMinG>(T, loc, lane, w, dl, lcr, du, ucr,
                                                             ecr, acr, exact);
          } else {
            class_pairs<kG, false, true, false, kTail, false, kSibFastMinG>(T, loc, lane, w, dl, lcr, du, ucr,
                                                              ecr, acr, exact);
          }
#endif
          lcr = G.sum(lcr);
          ucr = G.sum(ucr);
          ecr = G.sum(ecr);
          const double acr_sum = G.sum(static_cast<double>(acr));
          if (lane == 0) {
            acc[4 * ch] += lcr;
            acc[4 * ch + 1] += ucr;
            acc[4 * ch + 2] += ecr;
            acc[4 * ch + 3] += acr_sum;
          }
        }
      }
      st_max = G.max(st_max);
      sl_self = G.sum(sl_self);
      su_self = G.sum(su_self);
      se_self = G.sum(se_self);
      G.sync();
      const bool trans_ok = fmax(fmax(h0, h1), h2) > 1e-9;
      for (int ch = lane; ch < 8; ch += kG) {
        const long long slot = 8 * item + ch;
        if (args.split_rot) {
          const bool rot_ok = hr > 1e-9;
          int8_t sr;
          if (!rot_ok && !trans_ok) {
            sr = -1;
          } else {
            sr = (rot_ok && (!trans_ok || s_r >= st_max)) ? 1 : 0;
          }
          args.split_rot[slot] = sr;
        }
        if (infeasible) {
          args.lower[slot] = INFINITY;
          args.upper[slot] = INFINITY;
        } else {
          const double lcr = acc[4 * ch], ucr = acc[4 * ch + 1], ecr = acc[4 * ch + 2];
          const double mass = sl_self + 2.0 * lcr;
          const double core = (sl_self - 2.0 * lcr) - ctx.lb_err_scale * (se_self + ecr) -
                              ctx.lb_margin * mass;
          const double lo = core < parent_lower ? parent_lower : core;
          double up = INFINITY;
          if (!(lo >= args.skip_upper_at) && have_center) up = su_self - 2.0 * ucr;
          args.lower[slot] = lo;
          args.upper[slot] = up;
          if (args.redo_count && acc[4 * ch + 3] > ctx.redo_rel * 2.0 * lcr) redo(node, ch, slot);
        }
      }
      G.sync();
      continue;
    }
    // split decision (subdivide_adaptive, se3.cpp:107-121)
    st_max = G.max(st_max);
    // whole-table modes: every row is prepared, one decision for the node
    const unsigned exact = (streamed || kG < kFastMinG) ? 7u : G.bor3(fs.need());
    if constexpr (kMode == kSiblings) {
      // one cuboid, 8 rotation children: self sums once, then per child
      const double hr = 0.5 * rhw;
      const bool trans_ok = fmax(fmax(h0, h1), h2) > 1e-9;
      double sl_self = lb_self, su_self = ub_self, se_self = lb_err;
      // the children's rotations, 8 lanes at once (each child exactly as the
      // expand kernel builds it: k.rc[a] += h * s)
      double* const Rcs = reinterpret_cast<double*>(base + table_f4);  // [8][9]
      for (int ch = lane; ch < 8; ch += kG) {
        const int sx = (ch & 4) ? 1 : -1, sy = (ch & 2) ? 1 : -1, sz = (ch & 1) ? 1 : -1;
        rodrigues(rc0 + hr * sx, rc1 + hr * sy, rc2 + hr * sz, Rcs + 9 * ch);
      }
      if (!infeasible) {
        G.sync();
        for (int c = 0; c < ctx.n_classes; ++c) {
          const ClassSpan cs = ctx.cls[c];
          const float w = static_cast<float>(ctx.cls_w[c]);
          double dl = 0.0, du = 0.0;
          if (same) {
            class_pairs<kG, true, false, true, kTail, false>(T, cs, lane, w, sl_self, dl, su_self,
                                                             du, se_self, lb_amp, exact);
          } else {
            class_pairs<kG, false, false, true, kTail, false>(T, cs, lane, w, sl_self, dl,
                                                              su_self, du, se_self, lb_amp, exact);
          }
        }
        sl_self = G.sum(sl_self);
        su_self = G.sum(su_self);
        se_self = G.sum(se_self);
      }
      for (int ch = 0; ch < 8; ++ch) {
        const long long slot = 8 * item + ch;
        const double cs_r = s_r;  // sin(psi_c / 2), shared by the children
        if (lane == 0 && args.split_rot) {
          const bool rot_ok = hr > 1e-9;
          int8_t sr;
          if (!rot_ok && !trans_ok) {
            sr = -1;
          } else {
            sr = (rot_ok && (!trans_ok || cs_r >= st_max)) ? 1 : 0;
          }
          args.split_rot[slot] = sr;
        }
        if (infeasible) {
          if (lane == 0) {
            args.lower[slot] = INFINITY;
            args.upper[slot] = INFINITY;
          }
          continue;
        }
        G.sync();
        column_prep(T, ctx, lane, kG, Rcs + 9 * ch);
        G.sync();
        double lcr = 0.0, ucr = 0.0, ecr = 0.0, dl = 0.0, du = 0.0;
        float acr = 0.0f;
        for (int c = 0; c < ctx.n_classes; ++c) {
          const ClassSpan cs = ctx.cls[c];
          const float w = static_cast<float>(ctx.cls_w[c]);
          if (same) {
            class_pairs<kG, true, true, false, kTail, false>(T, cs, lane, w, dl, lcr, du, ucr, ecr,
                                                             acr, exact);
          } else {
            class_pairs<kG, false, true, false, kTail, false>(T, cs, lane, w, dl, lcr, du, ucr,
                                                              ecr, acr, exact);
          }
        }
        lcr = G.sum(lcr);
        ucr = G.sum(ucr);
        ecr = G.sum(ecr);
        const double acr_sum = G.sum(static_cast<double>(acr));
        if (lane == 0) {
          const double mass = sl_self + 2.0 * lcr;
          const double core = (sl_self - 2.0 * lcr) - ctx.lb_err_scale * (se_self + ecr) -
                              ctx.lb_margin * mass;
          const double lo = core < parent_lower ? parent_lower : core;
          double up = INFINITY;
          if (!(lo >= args.skip_upper_at) && have_center) up = su_self - 2.0 * ucr;
          args.lower[slot] = lo;
          args.upper[slot] = up;
          if (args.redo_count && acr_sum > ctx.redo_rel * 2.0 * lcr) redo(node, ch, slot);
        }
        G.sync();
      }
      G.sync();
      continue;
    }
    if (kMode != kSelfOnly && lane == 0 && args.split_rot) {
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
        if (kMode == kSelfOnly) {
          double* o = args.self_out + 4 * node;
          o[0] = o[1] = o[2] = 0.0;
          o[3] = 1.0;  // infeasible
        } else {
          const long long out = kFix ? args.out_slot[node] : node;
          args.lower[out] = INFINITY;
          args.upper[out] = INFINITY;
        }
      }
      G.sync();
      continue;
    }
    // ---- per-column prep: q_j = R0^T m_j (bounds.cpp:97-102), double-float
    if (kMode != kSelfOnly && !streamed) column_prep(T, ctx, lane, kG, R);
    G.sync();

    // ---- pair sweeps (GOSMA_PREP_ONLY: times the per-node prep alone)
#ifndef GOSMA_PREP_ONLY
    for (int c = 0; !streamed && c < ctx.n_classes; ++c) {
      const ClassSpan cs = ctx.cls[c];
      const float w = static_cast<float>(ctx.cls_w[c]);
      constexpr bool kC = kMode != kSelfOnly, kS = kMode != kCrossCached;
      if (same) {
        class_pairs<kG, true, kC, kS, kTail, kFix>(T, cs, lane, w, lb_self, lb_cross, ub_self,
                                                   ub_cross, lb_err, lb_amp, exact);
      } else {
        class_pairs<kG, false, kC, kS, kTail, kFix>(T, cs, lane, w, lb_self, lb_cross, ub_self,
                                                    ub_cross, lb_err, lb_amp, exact);
      }
    }
#endif
    lb_self = G.sum(lb_self);
    lb_cross = G.sum(lb_cross);
    ub_self = G.sum(ub_self);
    ub_cross = G.sum(ub_cross);
    lb_err = G.sum(lb_err);
    double amp_sum = 0.0;
    if constexpr (!kFix && kMode != kSelfOnly) amp_sum = G.sum(static_cast<double>(lb_amp));
    if (kMode == kSelfOnly) {
      if (lane == 0) {
        double* o = args.self_out + 4 * node;
        o[0] = lb_self;
        o[1] = ub_self;
        o[2] = lb_err;
        o[3] = have_center ? 0.0 : 2.0;  // 2: no feasible centre (upper = +inf)
      }
      G.sync();
      continue;
    }
    if (kMode == kCrossCached) {  // the cuboid's translation-only sums
      const double* o = args.self_out + 4 * static_cast<long long>(args.tindex[node]);
      lb_self = o[0];
      ub_self = o[1];
      lb_err += o[2];
    }
    if (lane == 0) {
      // Soundness margin: the FP32 error estimate of the terms plus a relative
      // floor on the |term| mass (all terms >= 0).
      const double mass = lb_self + 2.0 * lb_cross;
      const double core =
          (lb_self - 2.0 * lb_cross) - ctx.lb_err_scale * lb_err - ctx.lb_margin * mass;
      const double lo = core < parent_lower ? parent_lower : core;  // std::max(core, lower)
      double up = INFINITY;
      if (!(lo >= args.skip_upper_at) && have_center) up = ub_self - 2.0 * ub_cross;
      const long long out = kFix ? args.out_slot[node] : node;
      args.lower[out] = lo;
      args.upper[out] = up;
      if constexpr (!kFix) {
        if (args.redo_count && amp_sum > ctx.redo_rel * 2.0 * lb_cross) redo(node, -1, node);
      }
    }
    G.sync();
  }
}

}  // namespace

size_t eval_smem_per_warp(const DevCtx& ctx, int mode) {
  const bool streamed = mode == kModeStream || mode == kSiblingsStream || mode == kFixStream;
  const int n1 = streamed ? ctx.max_n1 : ctx.n1_total, n2 = streamed ? ctx.max_n2 : ctx.n2_total;
  size_t f4 = static_cast<size_t>(kRowF4 * n1 + kColF4 * n2);
  if (mode == kFixFull || mode == kFixStream) f4 += static_cast<size_t>(kRowPF4 * n1);
  if (mode == kSiblings || mode == kSiblingsStream) f4 += kSibStreamExtraF4;
  return f4 * sizeof(float4);
}

namespace {

// Lanes per node, from measured sweeps (scripts/kernel_timing.py, B200):
//  1  tiny mixtures (5 n1 + 2 n2 <= 48 table float4, e.g. up to 6x6): one lane
//     runs a whole node - 4.8x at 2x2, 2x at 4x4 over 8-lane groups;
//  8  up to 24 rows per class (8x8 .. 24x20: 1.2-2x over 16 / 32 lanes);
//  32 beyond (since the fast loop copies, 32 beats 16 lanes at 25-32 rows:
//     32x32 5.85 -> 5.33 ms, 8 x (32x16) 32.7 -> 28.0 ms; 16 stays
//     selectable); a whole CTA (4 warps sharing one node's tables) for large
//     mixtures whose tables would cap residency.
// Each choice also keeps the CTA's tables within a shared-memory budget.
// GOSMA_GROUP forces a size (A/B runs).
int group_lanes(const DevCtx& ctx, int mode) {
  static const int forced = [] {
    const char* e = std::getenv("GOSMA_GROUP");
    return e ? std::atoi(e) : 0;
  }();
  if (forced == 1 || forced == 8 || forced == 16 || forced == 32) return forced;
  if (forced == 128) return kCtaGroup;
  const size_t table = eval_smem_per_warp(ctx, mode);  // per group, incl. the siblings' extras
  const size_t core =
      table - ((mode == kSiblings || mode == kSiblingsStream) ? kSibStreamExtraF4 * 16 : 0);
  const int groups_per_cta = kWarpsPerCta * 32;
  const long long n1 = ctx.n1_total, n2 = ctx.n2_total;
  const long long pairs_bound = n1 * (n1 - 1) / 2 + n1 * n2;  // exact for one class
  if (core <= 48 * 16 && pairs_bound <= 64 && table * groups_per_cta <= 160 * 1024) return 1;
  if (ctx.max_n1 <= 24 && table * kWarpsPerCta * 4 <= 64 * 1024) return 8;
  if (ctx.max_n1 >= 64 && table > 10 * 1024) return kCtaGroup;
  return 32;
}

template <int kMode, int kG, bool kTail>
cudaError_t launch_group(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                         cudaStream_t stream) {
  // Warps per CTA: 4, or fewer when large mixtures' per-group tables would
  // leave few CTAs resident (e.g. 256x128: 1 CTA of 4 warps vs 7 of 1 warp).
  // The choice depends only on the device and the table size: cached, since
  // the occupancy queries cost microseconds per launch (short solves launch
  // thousands of small batches).
  struct Choice {
    int device;
    size_t per_warp;
    int warps, per_sm;
    size_t smem;
  };
  static std::mutex mu;
  static std::vector<Choice> cache;
  static int limit_on[64] = {};  // dynamic smem limit set on this kernel, per device
  auto limit_of = [](int dev) -> int& { return limit_on[dev & 63]; };
  int device = 0;
  cudaGetDevice(&device);
  const size_t per_warp = eval_smem_per_warp(ctx, kMode);
  int best_warps = kWarpsPerCta, best_per_sm = 0;
  size_t best_smem = 0;
  bool hit = false;
  {
    std::lock_guard<std::mutex> lk(mu);
    for (const Choice& c : cache)
      if (c.device == device && c.per_warp == per_warp) {
        best_warps = c.warps;
        best_per_sm = c.per_sm;
        best_smem = c.smem;
        hit = true;
        break;
      }
  }
  for (int warps = kWarpsPerCta, best_resident = -1;
       !hit && warps >= (kG > 32 ? kWarpsPerCta : 1); warps /= 2) {
    const int groups = kG > 32 ? 1 : warps * (32 / kG);
    const size_t smem = per_warp * groups;
    if (smem > 48 * 1024) {
      // the occupancy query needs the limit to cover smem; never lower it
      std::lock_guard<std::mutex> lk(mu);
      int& lim = limit_of(device);
      if (static_cast<int>(smem) > lim) {
        if (cudaFuncSetAttribute(eval_bounds_kernel<kMode, kG, kTail>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)) != cudaSuccess)
          continue;
        lim = static_cast<int>(smem);
      }
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(
            &per_sm, eval_bounds_kernel<kMode, kG, kTail>, warps * 32, smem) != cudaSuccess)
      continue;
    if (per_sm * warps > best_resident) {
      best_resident = per_sm * warps;
      best_warps = warps;
      best_per_sm = per_sm;
      best_smem = smem;
    }
  }
  if (!hit && best_per_sm >= 1) {
    std::lock_guard<std::mutex> lk(mu);
    cache.push_back(Choice{device, per_warp, best_warps, best_per_sm, best_smem});
  }
  // the kernel's dynamic shared-memory limit on this device only ever grows
  // (another context may have chosen a larger table): raise it when needed
  if (best_smem > 48 * 1024) {
    std::lock_guard<std::mutex> lk(mu);
    int& lim = limit_of(device);
    if (static_cast<int>(best_smem) > lim) {
      const cudaError_t e = cudaFuncSetAttribute(eval_bounds_kernel<kMode, kG, kTail>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(best_smem));
      if (e != cudaSuccess) return e;
      lim = static_cast<int>(best_smem);
    }
  }
  if (best_per_sm < 1) return cudaErrorInvalidConfiguration;
  const int groups_per_cta = kG > 32 ? 1 : best_warps * (32 / kG);
  long long grid = static_cast<long long>(best_per_sm) * sm_count;
  const long long need = (a.n + groups_per_cta - 1) / groups_per_cta;
  if (grid > need) grid = need;
  cudaError_t e = cudaMemsetAsync(a.work, 0, sizeof(unsigned int), stream);
  if (e != cudaSuccess) return e;
  eval_bounds_kernel<kMode, kG, kTail>
      <<<static_cast<unsigned>(grid), best_warps * 32, best_smem, stream>>>(ctx, a);
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaGetLastError();
}

template <int kMode>
cudaError_t launch_dispatch(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                            cudaStream_t stream, int lanes) {
  switch (lanes) {
    case kCtaGroup:
      return launch_group<kMode, kCtaGroup, false>(ctx, a, sm_count, stream);
    case 1:
      return launch_group<kMode, 1, false>(ctx, a, sm_count, stream);
    case 8:
      return launch_group<kMode, 8, false>(ctx, a, sm_count, stream);
    case 16:
      return launch_group<kMode, 16, false>(ctx, a, sm_count, stream);
    default:
      return ctx.tail_chunks ? launch_group<kMode, 32, true>(ctx, a, sm_count, stream)
                             : launch_group<kMode, 32, false>(ctx, a, sm_count, stream);
  }
}

template <int kMode>
cudaError_t launch_mode(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                        cudaStream_t stream) {
  if (a.n <= 0) return cudaSuccess;
  if (!a.work) return cudaErrorMemoryAllocation;  // no node counter for this stream
  const bool fix = kMode != kSelfOnly && a.redo_count && ctx.precise;
  EvalArgs m = a;
  if (!fix) {
    m.redo_count = nullptr;
  } else {
    const cudaError_t e = cudaMemsetAsync(a.redo_count, 0, sizeof(unsigned long long), stream);
    if (e != cudaSuccess) return e;
  }
  cudaError_t e = launch_dispatch<kMode>(ctx, m, sm_count, stream, group_lanes(ctx, kMode));
  if (e != cudaSuccess || !fix) return e;
  static const bool stats = std::getenv("GOSMA_REDO_STATS") != nullptr;
  if (stats) {  // diagnostics: how many items the fix-up re-evaluates
    unsigned long long k = 0;
    cudaMemcpyAsync(&k, a.redo_count, sizeof(k), cudaMemcpyDeviceToHost, stream);
    cudaStreamSynchronize(stream);
    std::fprintf(stderr, "[gosma] mode %d: %llu of %lld items to the precise fix-up\n", kMode, k,
                 a.n);
  }
  // the redo list, re-evaluated with the FP64 numerator (its count stays on
  // the device: the grid is sized for the capacity, idle groups exit at once)
  EvalArgs f{};
  f.nodes = a.redo_nodes;
  f.n = a.redo_cap;
  f.n_dev = reinterpret_cast<const long long*>(a.redo_count);
  f.out_slot = a.redo_slot;
  f.skip_upper_at = a.skip_upper_at;
  f.lower = a.lower;
  f.upper = a.upper;
  f.split_rot = nullptr;
  f.work = a.work;
  return ctx.stream_classes ? launch_dispatch<kFixStream>(ctx, f, sm_count, stream,
                                              group_lanes(ctx, kFixStream))
                : launch_dispatch<kFixFull>(ctx, f, sm_count, stream, group_lanes(ctx, kFixFull));
}

}  // namespace

cudaError_t launch_eval_bounds(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                               cudaStream_t stream) {
  return ctx.stream_classes ? launch_mode<kModeStream>(ctx, a, sm_count, stream)
                            : launch_mode<kModeFull>(ctx, a, sm_count, stream);
}

cudaError_t launch_eval_self(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                             cudaStream_t stream) {
  return launch_mode<kSelfOnly>(ctx, a, sm_count, stream);
}

cudaError_t launch_eval_cross_cached(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                                     cudaStream_t stream) {
  return launch_mode<kCrossCached>(ctx, a, sm_count, stream);
}

cudaError_t launch_eval_siblings(const DevCtx& ctx, const EvalArgs& a, int sm_count,
                                 cudaStream_t stream) {
  return ctx.stream_classes ? launch_mode<kSiblingsStream>(ctx, a, sm_count, stream)
                            : launch_mode<kSiblings>(ctx, a, sm_count, stream);
}


unsigned long long bound_kernel_launch_count() { return g_launches.load(); }

namespace {
// {tc[3], thw[3]} cuboid records -> node records for the self kernel (the
// rotation part does not enter the translation-only sums).
__global__ void boxes_to_nodes(const double* boxes, size_t n, gosma_node* out) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  gosma_node b{};
  for (int a = 0; a < 3; ++a) {
    b.tc[a] = boxes[6 * i + a];
    b.thw[a] = boxes[6 * i + 3 + a];
  }
  b.lower = -INFINITY;
  out[i] = b;
}
}  // namespace

namespace {
// subdivide_adaptive children (se3.cpp:107-147) of n parents with the given
// split flags (1 rotation, 0 translation, -1 none: children = copies), and the
// work lists of the siblings / full kernels (order irrelevant).
__global__ void children_of(const gosma_node* parents, const int8_t* split, size_t n,
                            gosma_node* kids, int* rot, int* trans_kids,
                            unsigned long long* counts) {
  const size_t t = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (t >= 8 * n) return;
  const size_t p = t / 8;
  const int c = static_cast<int>(t % 8);
  const int sx = (c & 4) ? 1 : -1, sy = (c & 2) ? 1 : -1, sz = (c & 1) ? 1 : -1;
  gosma_node k = parents[p];
  if (split[p] == 1) {
    const double h = 0.5 * k.rhw;
    k.rc[0] += h * sx;
    k.rc[1] += h * sy;
    k.rc[2] += h * sz;
    k.rhw = h;
    if (c == 0) rot[atomicAdd(&counts[0], 1ull)] = static_cast<int>(p);
  } else {
    if (split[p] == 0) {
      const double h0 = 0.5 * k.thw[0], h1 = 0.5 * k.thw[1], h2 = 0.5 * k.thw[2];
      k.tc[0] += h0 * sx;
      k.tc[1] += h1 * sy;
      k.tc[2] += h2 * sz;
      k.thw[0] = h0;
      k.thw[1] = h1;
      k.thw[2] = h2;
    }
    trans_kids[atomicAdd(&counts[1], 1ull)] = static_cast<int>(t);
  }
  kids[t] = k;
}

__global__ void identity_sel(unsigned int* sel, size_t n) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) sel[i] = static_cast<unsigned int>(i);
}
}  // namespace

cudaError_t make_children(const gosma_node* d_parents, const int8_t* d_split, size_t n,
                          gosma_node* d_kids, int* d_rot, int* d_trans,
                          unsigned long long* d_counts, unsigned int* d_sel,
                          cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  cudaError_t e = cudaMemsetAsync(d_counts, 0, 2 * sizeof(unsigned long long), stream);
  if (e != cudaSuccess) return e;
  children_of<<<static_cast<unsigned>((8 * n + 255) / 256), 256, 0, stream>>>(
      d_parents, d_split, n, d_kids, d_rot, d_trans, d_counts);
  identity_sel<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(d_sel, n);
  return cudaGetLastError();
}

cudaError_t boxes_as_nodes(const double* d_boxes, size_t n, gosma_node* d_out,
                           cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  boxes_to_nodes<<<static_cast<unsigned>((n + 255) / 256), 256, 0, stream>>>(d_boxes, n, d_out);
  return cudaGetLastError();
}

}  // namespace gosma
