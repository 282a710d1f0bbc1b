// Host FP64 objective, gradient and geometry: the thin host side of the
// path (north star (4)) used by the host refiner, the incumbent
// re-evaluation and gosma_objective_value. The objective and gradient are the
// GPU evaluator's formulation (objective_math.hpp) run serially, so host and
// device agree to FP64 summation order.
#include "host_math.hpp"

#include "objective_math.hpp"

#include <algorithm>
#include <cmath>

namespace gosma {

double log_z_eval(double kappa) { return objmath::log_z_d(kappa); }

double log_z_deriv(double kappa) { return objmath::log_z_deriv_d(kappa); }

Mat3 rotation_matrix(const Vec3& r) {
  Mat3 R;
  objmath::rotation_and_jacobian(r[0], r[1], r[2], R.m, nullptr);
  return R;
}

Vec3 wrap_rotation_vector(const Vec3& r) {
  // the same rotation with |r| <= pi
  Vec3 w = r;
  for (double n = w.norm(); n > M_PI; n = w.norm()) w = w * (1.0 - 2.0 * M_PI / n);
  return w;
}

bool pose_feasible(const HostModel& model, const Vec3& t) {
  // camera centre outside every standoff ball (objective.cpp:160-166)
  for (const Vec3& mu : model.all_means)
    if ((mu - t).norm() < model.zeta) return false;
  return true;
}

namespace {

// The objective (and optionally its gradient) at x = (r, t) in the GPU
// evaluator's formulation (objective_math.hpp; objgrad_block in
// objective_kernel.cu with one partner slice): per class, rows of
// (u_i, d_i, k_i, log Z, log Z'), the closed-form diagonal, ordered self pairs
// i != j each adding half of the pair, cross pairs against the rotated rows;
// gradients accumulated as vectors and mapped by J_i (jv) and Jl^T.
double evaluate(const HostModel& model, const Vec3& r, const Vec3& t, double* grad) {
  double R[9], Jl[9];
  objmath::rotation_and_jacobian(r[0], r[1], r[2], R, grad ? Jl : nullptr);
  double f = 0.0, gt[3] = {0.0, 0.0, 0.0}, cr[3] = {0.0, 0.0, 0.0};
  std::vector<objmath::RowD> rows;
  for (const HostClass& cls : model.classes) {
    const double w = cls.weight;
    const int n1 = cls.n1(), n2 = cls.n2();
    rows.resize(n1);
    for (int i = 0; i < n1; ++i)
      rows[i] = objmath::make_row(cls.mu[3 * i], cls.mu[3 * i + 1], cls.mu[3 * i + 2],
                                  cls.sigma2[i], cls.phi1[i], t[0], t[1], t[2]);
    for (int i = 0; i < n1; ++i) {
      const objmath::RowD& a = rows[i];
      const double ui[3] = {a.ux * a.d, a.uy * a.d, a.uz * a.d};
      const double vi[3] = {a.ux * a.k, a.uy * a.k, a.uz * a.k};
      const double cu = 2.0 * a.zl * a.is2;
      const double diag = 0.5 * a.k / std::tanh(a.k);
      double fself = a.phi * a.phi * diag, fcross = 0.0;
      double s[3] = {0.0, 0.0, 0.0}, su = 0.0, h[3] = {0.0, 0.0, 0.0}, hu = 0.0;
      if (grad) {
        const double sd = a.phi * a.phi * diag * 2.0 * (objmath::log_z_deriv_d(2.0 * a.k) - a.zl) *
                          (-2.0 * a.is2);
        for (int k = 0; k < 3; ++k) gt[k] += w * ui[k] * sd;
      }
      for (int j = 0; j < n1; ++j) {  // self pairs, this row's half
        if (j == i) continue;
        const objmath::RowD& b = rows[j];
        const double e[3] = {vi[0] + b.ux * b.k, vi[1] + b.uy * b.k, vi[2] + b.uz * b.k};
        const double K = std::sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
        if (K < a.k + b.k - objmath::kNegligible) continue;
        double eK, zl;
        objmath::pair_terms(K, a.lz + b.lz, eK, zl);
        const double term = 2.0 * a.phi * b.phi * eK;
        fself += 0.5 * term;
        if (grad) {
          if (K > 1e-12)
            for (int k = 0; k < 3; ++k) s[k] += e[k] * (zl * term / K);
          su += term;
        }
      }
      const double wv[3] = {R[0] * vi[0] + R[1] * vi[1] + R[2] * vi[2],
                            R[3] * vi[0] + R[4] * vi[1] + R[5] * vi[2],
                            R[6] * vi[0] + R[7] * vi[1] + R[8] * vi[2]};
      for (int j = 0; j < n2; ++j) {  // cross pairs
        const double e[3] = {wv[0] + cls.b[3 * j], wv[1] + cls.b[3 * j + 1],
                             wv[2] + cls.b[3 * j + 2]};
        const double K = std::sqrt(e[0] * e[0] + e[1] * e[1] + e[2] * e[2]);
        if (K < a.k + cls.kappa2[j] - objmath::kNegligible) continue;
        double eK, zl;
        objmath::pair_terms(K, a.lz + cls.log_z2[j], eK, zl);
        const double term = a.phi * cls.phi2[j] * eK;
        fcross += term;
        if (grad) {
          double q[3] = {0.0, 0.0, 0.0};
          if (K > 1e-12)
            for (int k = 0; k < 3; ++k) q[k] = e[k] / K;
          const double sc = zl * (-2.0 * term);
          for (int k = 0; k < 3; ++k) h[k] += q[k] * sc;
          hu += -2.0 * term;
          cr[0] += w * (wv[1] * q[2] - wv[2] * q[1]) * sc;
          cr[1] += w * (wv[2] * q[0] - wv[0] * q[2]) * sc;
          cr[2] += w * (wv[0] * q[1] - wv[1] * q[0]) * sc;
        }
      }
      if (grad) {
        double o[3];
        objmath::jv(a, s[0], s[1], s[2], o[0], o[1], o[2]);
        for (int k = 0; k < 3; ++k) gt[k] += w * (o[k] + ui[k] * cu * su);
        const double p[3] = {R[0] * h[0] + R[3] * h[1] + R[6] * h[2],  // R^T h
                             R[1] * h[0] + R[4] * h[1] + R[7] * h[2],
                             R[2] * h[0] + R[5] * h[1] + R[8] * h[2]};
        objmath::jv(a, p[0], p[1], p[2], o[0], o[1], o[2]);
        for (int k = 0; k < 3; ++k) gt[k] += w * (o[k] + ui[k] * cu * hu);
      }
      f += w * (fself - 2.0 * fcross);
    }
  }
  if (grad) {
    for (int k = 0; k < 3; ++k) grad[k] = Jl[k] * cr[0] + Jl[3 + k] * cr[1] + Jl[6 + k] * cr[2];
    for (int k = 0; k < 3; ++k) grad[3 + k] = gt[k];
  }
  return f;
}

}  // namespace

double objective_value(const HostModel& model, const Vec3& r, const Vec3& t) {
  // +inf in place of the reference's InfeasiblePoseError
  if (!pose_feasible(model, t)) return INFINITY;
  return evaluate(model, r, t, nullptr);
}

bool objective_gradient(const HostModel& model, const Vec3& r, const Vec3& t, double g[6]) {
  if (!pose_feasible(model, t)) return false;
  evaluate(model, r, t, g);
  return true;
}

double objective_and_gradient(const HostModel& model, const Vec3& r, const Vec3& t,
                              double g[6]) {
  if (!pose_feasible(model, t)) {
    for (int k = 0; k < 6; ++k) g[k] = 0.0;
    return INFINITY;
  }
  return evaluate(model, r, t, g);
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
