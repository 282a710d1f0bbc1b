// FP64 pieces of the objective and its gradient shared by the GPU evaluator
// (objective_kernel.cu: objgrad_block, one CTA per pose) and the host
// evaluator (host_math.cpp): the same formulation on both sides.
//
//   log Z(k)  = k + log1p(-e^{-2k}) - log k, its derivative (the reference's
//               log_z_eval / log_z_deriv, sphere_stats.cpp:47-69);
//   pair term = exp(log Z(K) - c) = e^{K-c} (1 - e^{-2K}) / K with one
//               exponential shared with log Z'(K);
//   J_i v     = u_i (u_i.v)(-2 d_i / s2_i) - (v - u_i (u_i.v)) (k_i / d_i), the
//               Jacobian of v_i = k_i u_i with respect to t applied to a
//               vector, so no 3x3 matrix is formed.
#pragma once

#include <cmath>

#include "refine_core.hpp"  // GOSMA_HD

namespace gosma {
namespace objmath {

constexpr double kNegligible = 64.0;  // pair skip margin (objective.cpp:17)

GOSMA_HD inline double log_z_d(double k) {
  if (k < 1e-4) return 0.69314718055994531 + log1p(k * k / 6.0);
  // above 19, exp(-2k) < 2^-54: k + log1p(-exp(-2k)) rounds to k (bit-identical)
  if (k > 19.0) return k - log(k);
  return k + log1p(-exp(-2.0 * k)) - log(k);
}

GOSMA_HD inline double log_z_deriv_d(double k) {
  if (k < 1e-4) return k / 3.0 - k * k * k / 45.0;
  if (k > 19.0) return 1.0 - 1.0 / k;  // (1 + e2) / (1 - e2) == 1 exactly above 19
  const double e2 = exp(-2.0 * k);
  return (1.0 + e2) / (1.0 - e2) - 1.0 / k;
}

// A pair's exp(log_z(K) - c) and log_z'(K) from one exp(-2K).
GOSMA_HD inline void pair_terms(double K, double c, double& ez, double& zl) {
  if (K < 1e-4) {
    ez = exp(log_z_d(K) - c);
    zl = log_z_deriv_d(K);
    return;
  }
  const double iK = 1.0 / K;
  // 1 - e2; above K = 19, e2 = exp(-2K) < 2^-54 and 1 - e2 rounds to 1.0 in
  // FP64, so the exp is skipped with bit-identical results (realistic K ~ 1e2-1e5)
  const double om = K < 0.5 ? -expm1(-2.0 * K) : (K > 19.0 ? 1.0 : 1.0 - exp(-2.0 * K));
  ez = exp(K - c) * om * iK;
  zl = K > 350.0 ? 1.0 - iK : (2.0 - om) / om - iK;
}

// Per-row record of a pose evaluation.
struct RowD {
  double ux, uy, uz;  // unit direction of mu_i - t
  double d, k, lz, zl, is2, phi;
};

GOSMA_HD inline RowD make_row(double mx, double my, double mz, double sigma2, double phi,
                              double t0, double t1, double t2) {
  const double ux = mx - t0, uy = my - t1, uz = mz - t2;
  const double d2 = ux * ux + uy * uy + uz * uz;
  const double d = sqrt(d2);
  RowD r;
  r.ux = ux * (1.0 / d);
  r.uy = uy * (1.0 / d);
  r.uz = uz * (1.0 / d);
  r.d = d;
  r.is2 = 1.0 / sigma2;
  r.k = d2 / sigma2 + 1.0;
  r.lz = log_z_d(r.k);
  r.zl = log_z_deriv_d(r.k);
  r.phi = phi;
  return r;
}

GOSMA_HD inline void jv(const RowD& r, double vx, double vy, double vz, double& ox, double& oy,
                        double& oz) {
  const double p = r.ux * vx + r.uy * vy + r.uz * vz;
  const double a = -2.0 * r.d * r.is2, b = r.k / r.d;
  ox = r.ux * p * a - (vx - r.ux * p) * b;
  oy = r.uy * p * a - (vy - r.uy * p) * b;
  oz = r.uz * p * a - (vz - r.uz * p) * b;
}

// Rotation R = exp([r]x) and the left Jacobian Jl of SO(3) at r, row-major,
// from one sin / cos of |r| (series below 1e-8 / 1e-6 rad).
GOSMA_HD inline void rotation_and_jacobian(double r0, double r1, double r2, double* R,
                                           double* Jl) {
  const double th2 = r0 * r0 + r1 * r1 + r2 * r2;
  const double K[9] = {0.0, -r2, r1, r2, 0.0, -r0, -r1, r0, 0.0};
  double K2[9];
  for (int a = 0; a < 3; ++a)
    for (int c = 0; c < 3; ++c)
      K2[3 * a + c] = K[3 * a] * K[c] + K[3 * a + 1] * K[3 + c] + K[3 * a + 2] * K[6 + c];
  double th = 0.0, sth = 0.0, cth = 1.0;
  if (th2 >= 1e-16) {
    th = sqrt(th2);
    sth = sin(th);
    cth = cos(th);
  }
  double ra, rc, ja, jb;
  if (th2 < 1e-16) {
    ra = 1.0;
    rc = 0.5;
  } else {
    ra = sth / th;
    rc = (1.0 - cth) / th2;
  }
  if (th2 < 1e-12) {
    ja = 0.5;
    jb = 1.0 / 6.0;
  } else {
    ja = (1.0 - cth) / th2;
    jb = (th - sth) / (th2 * th);
  }
  for (int e = 0; e < 9; ++e) {
    const double id = (e % 4 == 0) ? 1.0 : 0.0;
    R[e] = (id + ra * K[e]) + rc * K2[e];
    if (Jl) Jl[e] = id + K[e] * ja + K2[e] * jb;
  }
}

}  // namespace objmath
}  // namespace gosma
