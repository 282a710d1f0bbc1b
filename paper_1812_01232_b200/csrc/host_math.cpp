// Host FP64 objective, gradient and geometry: the thin host side of the
// path (north star (4)) used by the local refiner (SMA), the incumbent
// re-evaluation and gosma_objective_value. Follows the reference formulas:
// sphere_stats.cpp:47-69 (log Z, its derivative), se3.cpp:21-31 (Rodrigues),
// objective.cpp:160-334 (value, gradient).
#include "host_math.hpp"

#include <algorithm>
#include <cmath>

namespace gosma {

double log_z_eval(double kappa) {
  // sphere_stats.cpp:47-56
  if (kappa < 1e-4) return std::log(2.0) + std::log1p(kappa * kappa / 6.0);
  return kappa + std::log1p(-std::exp(-2.0 * kappa)) - std::log(kappa);
}

double log_z_deriv(double kappa) {
  // sphere_stats.cpp:58-69
  if (kappa < 1e-4) return kappa / 3.0 - kappa * kappa * kappa / 45.0;
  if (kappa > 350.0) return 1.0 - 1.0 / kappa;
  const double e2 = std::exp(-2.0 * kappa);
  return (1.0 + e2) / (1.0 - e2) - 1.0 / kappa;
}

Mat3 rotation_matrix(const Vec3& r) {
  // se3.cpp:21-31
  const double theta2 = r.dot(r);
  const Mat3 K = Mat3::skew(r);
  const Mat3 K2 = K * K;
  double a, c;
  if (theta2 < 1e-16) {
    a = 1.0;
    c = 0.5;
  } else {
    const double theta = std::sqrt(theta2);
    a = std::sin(theta) / theta;
    c = (1.0 - std::cos(theta)) / theta2;
  }
  Mat3 R;
  for (int i = 0; i < 9; ++i) R.m[i] = ((i % 4 == 0 ? 1.0 : 0.0) + a * K.m[i]) + c * K2.m[i];
  return R;
}

Vec3 wrap_rotation_vector(const Vec3& r) {
  // se3.cpp:50-58
  Vec3 w = r;
  double n = w.norm();
  while (n > M_PI) {
    w = w * (1.0 - 2.0 * M_PI / n);
    n = w.norm();
  }
  return w;
}

bool pose_feasible(const HostModel& model, const Vec3& t) {
  // check_feasible, objective.cpp:160-166
  for (const Vec3& mu : model.all_means) {
    if ((mu - t).norm() < model.zeta) return false;
  }
  return true;
}

namespace {

constexpr double kMargin = 64.0;  // objective.cpp:17

double class_objective(const HostClass& cls, const Mat3& R, const Vec3& t) {
  // class_objective + project_model, objective.cpp:175-223
  const int n1 = cls.n1(), n2 = cls.n2();
  std::vector<Vec3> v(n1);
  std::vector<double> kap(n1), lz(n1);
  for (int i = 0; i < n1; ++i) {
    const Vec3 u = Vec3(cls.mu[3 * i], cls.mu[3 * i + 1], cls.mu[3 * i + 2]) - t;
    const double d2 = u.dot(u);
    const double d = std::sqrt(d2);
    kap[i] = d2 / cls.sigma2[i] + 1.0;
    v[i] = u * (kap[i] / d);
    lz[i] = log_z_eval(kap[i]);
  }
  double self_sum = 0.0;
  for (int i = 0; i < n1; ++i) {
    self_sum += cls.phi1[i] * cls.phi1[i] * 0.5 * kap[i] / std::tanh(kap[i]);
    for (int j = i + 1; j < n1; ++j) {
      const double K = (v[i] + v[j]).norm();
      if (K < kap[i] + kap[j] - kMargin) continue;
      self_sum += 2.0 * cls.phi1[i] * cls.phi1[j] * std::exp(log_z_eval(K) - lz[i] - lz[j]);
    }
  }
  double cross_sum = 0.0;
  for (int i = 0; i < n1; ++i) {
    const Vec3 w = R * v[i];
    for (int j = 0; j < n2; ++j) {
      const double K = (w + Vec3(cls.b[3 * j], cls.b[3 * j + 1], cls.b[3 * j + 2])).norm();
      if (K < kap[i] + cls.kappa2[j] - kMargin) continue;
      cross_sum +=
          cls.phi1[i] * cls.phi2[j] * std::exp(log_z_eval(K) - lz[i] - cls.log_z2[j]);
    }
  }
  return self_sum - 2.0 * cross_sum;
}

Mat3 left_jacobian(const Vec3& r) {
  // objective.cpp:240-250
  const double theta2 = r.dot(r);
  const Mat3 K = Mat3::skew(r);
  const Mat3 K2 = K * K;
  if (theta2 < 1e-12) return Mat3::identity() + K * 0.5 + K2 * (1.0 / 6.0);
  const double theta = std::sqrt(theta2);
  return Mat3::identity() + K * ((1.0 - std::cos(theta)) / theta2) +
         K2 * ((theta - std::sin(theta)) / (theta2 * theta));
}

}  // namespace

double objective_value(const HostModel& model, const Vec3& r, const Vec3& t) {
  // objective.cpp:227-235 (+inf in place of InfeasiblePoseError)
  if (!pose_feasible(model, t)) return INFINITY;
  const Mat3 R = rotation_matrix(r);
  double f = 0.0;
  for (const HostClass& cls : model.classes) f += cls.weight * class_objective(cls, R, t);
  return f;
}

bool objective_gradient(const HostModel& model, const Vec3& r, const Vec3& t, double g[6]) {
  // objective.cpp:254-334
  if (!pose_feasible(model, t)) return false;
  const Mat3 R = rotation_matrix(r);
  const Mat3 Jl = left_jacobian(r);
  Vec3 grad_r, grad_t;
  for (const HostClass& cls : model.classes) {
    const int n1 = cls.n1(), n2 = cls.n2();
    std::vector<Vec3> u(n1), uhat(n1);
    std::vector<double> kappa(n1), lz(n1), zl(n1), d(n1);
    std::vector<Mat3> J(n1);
    for (int i = 0; i < n1; ++i) {
      u[i] = Vec3(cls.mu[3 * i], cls.mu[3 * i + 1], cls.mu[3 * i + 2]) - t;
      const double d2 = u[i].dot(u[i]);
      d[i] = std::sqrt(d2);
      uhat[i] = u[i] * (1.0 / d[i]);
      kappa[i] = d2 / cls.sigma2[i] + 1.0;
      lz[i] = log_z_eval(kappa[i]);
      zl[i] = log_z_deriv(kappa[i]);
      const Mat3 outer = Mat3::outer(uhat[i], uhat[i]);
      J[i] = outer * (-(2.0 * d[i] / cls.sigma2[i])) -
             (Mat3::identity() - outer) * (kappa[i] / d[i]);
    }
    Vec3 cgr, cgt;
    for (int i = 0; i < n1; ++i) {
      const Vec3 vi = uhat[i] * kappa[i];
      {
        const double term = 0.5 * kappa[i] / std::tanh(kappa[i]);
        const double dlog = 2.0 * (log_z_deriv(2.0 * kappa[i]) - zl[i]);
        cgt = cgt + u[i] * (cls.phi1[i] * cls.phi1[i] * term * dlog * (-2.0 / cls.sigma2[i]));
      }
      for (int j = i + 1; j < n1; ++j) {
        const Vec3 sum = vi + uhat[j] * kappa[j];
        const double K = sum.norm();
        if (K < kappa[i] + kappa[j] - kMargin) continue;
        const double term =
            2.0 * cls.phi1[i] * cls.phi1[j] * std::exp(log_z_eval(K) - lz[i] - lz[j]);
        Vec3 dK;
        if (K > 1e-12) dK = (J[i] + J[j]) * (sum * (1.0 / K));
        cgt = cgt + (dK * log_z_deriv(K) + u[i] * (2.0 * zl[i] / cls.sigma2[i]) +
                     u[j] * (2.0 * zl[j] / cls.sigma2[j])) *
                        term;
      }
      const Vec3 w = R * vi;
      for (int j = 0; j < n2; ++j) {
        const Vec3 sum = w + Vec3(cls.b[3 * j], cls.b[3 * j + 1], cls.b[3 * j + 2]);
        const double K = sum.norm();
        if (K < kappa[i] + cls.kappa2[j] - kMargin) continue;
        const double term =
            cls.phi1[i] * cls.phi2[j] * std::exp(log_z_eval(K) - lz[i] - cls.log_z2[j]);
        Vec3 what;
        if (K > 1e-12) what = sum * (1.0 / K);
        const double zlK = log_z_deriv(K);
        const Vec3 dt_part = (J[i] * (R.transpose() * what)) * zlK + u[i] * (2.0 * zl[i] / cls.sigma2[i]);
        const Vec3 dr_part = (Jl.transpose() * w.cross(what)) * zlK;
        cgt = cgt + dt_part * (-2.0 * term);
        cgr = cgr + dr_part * (-2.0 * term);
      }
    }
    grad_r = grad_r + cgr * cls.weight;
    grad_t = grad_t + cgt * cls.weight;
  }
  for (int k = 0; k < 3; ++k) {
    g[k] = grad_r[k];
    g[3 + k] = grad_t[k];
  }
  return true;
}

bool feasible_center(const HostModel& model, const Vec3& c, const Vec3& h, Vec3* t_out) {
  // bounds.cpp:187-214
  Vec3 t = c;
  for (int projection = 0; projection <= 8; ++projection) {
    const Vec3* offender = nullptr;
    for (const Vec3& mu : model.all_means) {
      if ((mu - t).norm() < model.zeta) {
        offender = &mu;
        break;
      }
    }
    if (!offender) {
      *t_out = t;
      return true;
    }
    if (projection == 8) break;
    Vec3 dir = t - *offender;
    const double n = dir.norm();
    dir = n > 1e-12 ? dir / n : Vec3(1.0, 0.0, 0.0);
    t =*offender + dir * (model.zeta * (1.0 + 1e-9));
    for (int k = 0; k < 3; ++k) t[k] = std::clamp(t[k], c[k] - h[k], c[k] + h[k]);
  }
  return false;
}

double point_box_lo(const Vec3& p, const Vec3& c, const Vec3& h) {
  Vec3 o;
  for (int k = 0; k < 3; ++k) o[k] = std::max(std::fabs(p[k] - c[k]) - h[k], 0.0);
  return o.norm();
}

double point_box_hi(const Vec3& p, const Vec3& c, const Vec3& h) {
  Vec3 f;
  for (int k = 0; k < 3; ++k) f[k] = std::fabs(p[k] - c[k]) + h[k];
  return f.norm();
}

double psi_trans(const Vec3& c, const Vec3& h, const Vec3& p) {
  // se3.cpp:72-92
  const Vec3 cdir = p - c;
  if (std::fabs(cdir[0]) <= h[0] && std::fabs(cdir[1]) <= h[1] && std::fabs(cdir[2]) <= h[2])
    return M_PI;
  double worst = 0.0;
  for (int sx = -1; sx <= 1; sx += 2)
    for (int sy = -1; sy <= 1; sy += 2)
      for (int sz = -1; sz <= 1; sz += 2) {
        const Vec3 vertex(c[0] + sx * h[0], c[1] + sy * h[1], c[2] + sz * h[2]);
        const Vec3 v = p - vertex;
        worst = std::max(worst, std::atan2(cdir.cross(v).norm(), cdir.dot(v)));
      }
  return worst;
}

}  // namespace gosma

namespace gosma {

namespace {
double logw_fp64(double x) { return x > 30.0 ? -std::log(x) : log_z_eval(x) - x; }
double pair_k64(double a, double b, double c) {
  return std::sqrt(std::max(0.0, a * a + b * b + 2.0 * c * a * b));
}
}  // namespace

double lower_bound_fp64(const HostModel& model, const Vec3& rc, double rhw, const Vec3& tc,
                        const Vec3& th, double parent_lower) {
  // FP64 evaluate_bounds lower part (bounds.cpp:46-183, 270-273): used by the
  // solver for resolved (unsplittable) branches, where the certified floor
  // should carry no FP32 slack.
  for (const Vec3& mu : model.all_means)
    if (point_box_hi(mu, tc, th) < model.zeta) return INFINITY;
  const Mat3 R0t = rotation_matrix(rc).transpose();
  const double psi_r = std::min(std::sqrt(3.0) * rhw, M_PI);
  double total = 0.0;
  for (const HostClass& c : model.classes) {
    const int n1 = c.n1(), n2 = c.n2();
    std::vector<double> klo(n1), khi(n1), lwlo(n1), lwhi(n1), pt(n1), cpt(n1), spt(n1), cps(n1),
        sps(n1);
    std::vector<Vec3> uh(n1), q(n2);
    std::vector<char> bz(n1);
    for (int i = 0; i < n1; ++i) {
      const Vec3 mu(c.mu[3 * i], c.mu[3 * i + 1], c.mu[3 * i + 2]);
      const double dlo = std::max(point_box_lo(mu, tc, th), model.zeta);
      const double dhi = point_box_hi(mu, tc, th);
      klo[i] = dlo * dlo / c.sigma2[i] + 1.0;
      khi[i] = dhi * dhi / c.sigma2[i] + 1.0;
      lwlo[i] = logw_fp64(klo[i]);
      lwhi[i] = logw_fp64(khi[i]);
      const Vec3 u = mu - tc;
      const double n = u.norm();
      uh[i] = n > 1e-12 ? u / n : Vec3(1.0, 0.0, 0.0);
      pt[i] = psi_trans(tc, th, mu);
      cpt[i] = std::cos(pt[i]);
      spt[i] = std::sin(pt[i]);
      const double ps = pt[i] + psi_r;
      bz[i] = ps >= M_PI;
      cps[i] = bz[i] ? -1.0 : std::cos(ps);
      sps[i] = bz[i] ? 0.0 : std::sin(ps);
    }
    for (int j = 0; j < n2; ++j)
      q[j] = R0t * (Vec3(c.b[3 * j], c.b[3 * j + 1], c.b[3 * j + 2]) / c.kappa2[j]);
    double self_lo = 0.0;
    for (int i = 0; i < n1; ++i) {
      self_lo += c.phi1[i] * c.phi1[i] * 0.5 * klo[i] / std::tanh(klo[i]);
      for (int j = i + 1; j < n1; ++j) {
        double ca;
        if (pt[i] + pt[j] >= M_PI) {
          ca = -1.0;
        } else {
          const double cth = std::clamp(uh[i].dot(uh[j]), -1.0, 1.0);
          const double cpp = cpt[i] * cpt[j] - spt[i] * spt[j];
          if (cth <= -cpp) {
            ca = -1.0;
          } else {
            const double spp = spt[i] * cpt[j] + cpt[i] * spt[j];
            ca = cth * cpp - std::sqrt(std::max(0.0, 1.0 - cth * cth)) * spp;
          }
        }
        const double khh = pair_k64(khi[i], khi[j], ca);
        const double ex = 2.0 * khi[i] * khi[j] * (ca - 1.0) / (khh + khi[i] + khi[j]);
        const double kcm = std::max(std::max(pair_k64(klo[i], klo[j], ca), pair_k64(klo[i], khi[j], ca)),
                                    std::max(pair_k64(khi[i], klo[j], ca), khh));
        self_lo += 2.0 * c.phi1[i] * c.phi1[j] * std::exp(ex + logw_fp64(kcm) - lwlo[i] - lwlo[j]);
      }
    }
    double cross_hi = 0.0;
    for (int i = 0; i < n1; ++i)
      for (int j = 0; j < n2; ++j) {
        double cb;
        if (bz[i]) {
          cb = 1.0;
        } else {
          const double cth = std::clamp(uh[i].dot(q[j]), -1.0, 1.0);
          cb = cth >= cps[i] ? 1.0
                             : cth * cps[i] + std::sqrt(std::max(0.0, 1.0 - cth * cth)) * sps[i];
        }
        const double k2 = c.kappa2[j];
        const double kl = pair_k64(klo[i], k2, cb);
        const double ex = 2.0 * klo[i] * k2 * (cb - 1.0) / (kl + klo[i] + k2);
        const double vx = -cb * k2;
        const double kmin = vx <= klo[i] ? kl
                                         : (vx >= khi[i] ? pair_k64(khi[i], k2, cb)
                                                         : k2 * std::sqrt(std::max(0.0, (1.0 - cb) * (1.0 + cb))));
        cross_hi += c.phi1[i] * c.phi2[j] *
                    std::exp(ex + logw_fp64(kmin) - lwhi[i] - (c.log_z2[j] - k2));
      }
    total += c.weight * (self_lo - 2.0 * cross_hi);
  }
  return std::max(total, parent_lower);
}

}  // namespace gosma
