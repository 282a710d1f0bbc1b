// Local refinement ("SMA"): limited-memory quasi-Newton descent of the FP64
// host objective with a strong-Wolfe line search, projected into the domain
// and out of the standoff balls. Thin host C++ off the hot path (north star
// (4)); follows local_refine / wolfe_search / clamp_to_domain
// (core/src/solver.cpp:37-258): memory 10, <= 200 iterations, |g| < 1e-6,
// c1 = 1e-4, c2 = 0.9, <= 20 bracket + 30 zoom steps, never worse than the
// start.
#include "sma.hpp"


#include <algorithm>
#include <cmath>
#include <deque>
#include <limits>
#include <vector>

namespace gosma {

namespace {

constexpr double kInf = std::numeric_limits<double>::infinity();

using V6 = std::array<double, 6>;

double dot6(const V6& a, const V6& b) {
  double s = 0.0;
  for (int k = 0; k < 6; ++k) s += a[k] * b[k];
  return s;
}
double norm6(const V6& a) { return std::sqrt(dot6(a, a)); }
V6 axpy(const V6& x, double a, const V6& d) {
  V6 r;
  for (int k = 0; k < 6; ++k) r[k] = x[k] + a * d[k];
  return r;
}

Vec3 head(const V6& x) { return Vec3(x[0], x[1], x[2]); }
Vec3 tail(const V6& x) { return Vec3(x[3], x[4], x[5]); }

// Objective with infeasible poses mapped to +inf (solver.cpp:37-43) and its
// gradient (zero when infeasible).
class Objective {
 public:
  explicit Objective(const HostModel& m) : m_(m) {}
  const HostModel& model() const { return m_; }
  double value(const V6& x) { return objective_value(m_, head(x), tail(x)); }
  V6 grad(const V6& x) {
    V6 g;
    double gg[6];
    if (!objective_gradient(m_, head(x), tail(x), gg)) {
      g.fill(0.0);
      return g;
    }
    for (int k = 0; k < 6; ++k) g[k] = gg[k];
    return g;
  }

 private:
  const HostModel& m_;
};

// clamp_to_domain (solver.cpp:48-95)
bool clamp_to_domain(const HostModel& m, const Domain& dom, V6* x) {
  V6& v = *x;
  for (int k = 0; k < 3; ++k)
    v[k] = std::clamp(v[k], dom.rot_center[k] - dom.rot_hw, dom.rot_center[k] + dom.rot_hw);
  const Vec3 t(v[3], v[4], v[5]);
  int best = -1;
  double best_d = kInf;
  for (size_t b = 0; b < dom.boxes.size(); ++b) {
    const double d = point_box_lo(t, dom.boxes[b].c, dom.boxes[b].h);
    if (d < best_d) {
      best_d = d;
      best = static_cast<int>(b);
    }
  }
  if (best < 0) return false;
  const Vec3 c = dom.boxes[best].c, h = dom.boxes[best].h;
  Vec3 p = t;
  for (int k = 0; k < 3; ++k) p[k] = std::clamp(p[k], c[k] - h[k], c[k] + h[k]);
  for (int projection = 0; projection <= 8; ++projection) {
    const Vec3* off = nullptr;
    for (const Vec3& mu : m.all_means) {
      if ((mu - p).norm() < m.zeta) {
        off = &mu;
        break;
      }
    }
    if (!off) {
      v[3] = p[0];
      v[4] = p[1];
      v[5] = p[2];
      return true;
    }
    if (projection == 8) break;
    Vec3 dir = p - *off;
    const double n = dir.norm();
    dir = n > 1e-12 ? dir / n : Vec3(1.0, 0.0, 0.0);
    p = *off + dir * (m.zeta * (1.0 + 1e-9));
    for (int k = 0; k < 3; ++k) p[k] = std::clamp(p[k], c[k] - h[k], c[k] + h[k]);
  }
  return false;
}

struct LineSearch {
  double alpha = 0.0;
  double value = kInf;
  bool wolfe = false;
};

// wolfe_search (solver.cpp:105-160)
LineSearch wolfe(Objective& m, const V6& x, const V6& d, double f0, double g0) {
  const double c1 = 1e-4, c2 = 0.9, alpha_max = 1e3;
  auto phi = [&](double a) { return m.value(axpy(x, a, d)); };
  auto dphi = [&](double a) { return dot6(m.grad(axpy(x, a, d)), d); };
  LineSearch best;
  auto consider = [&](double a, double v) {
    if (v <= f0 + c1 * a * g0 && v < best.value) {
      best.alpha = a;
      best.value = v;
    }
  };
  auto zoom = [&](double lo, double flo, double hi) -> LineSearch {
    for (int it = 0; it < 30; ++it) {
      const double a = 0.5 * (lo + hi);
      const double v = phi(a);
      consider(a, v);
      if (v > f0 + c1 * a * g0 || v >= flo) {
        hi = a;
        continue;
      }
      const double g = dphi(a);
      if (std::fabs(g) <= -c2 * g0) return {a, v, true};
      if (g * (hi - lo) >= 0.0) hi = lo;
      lo = a;
      flo = v;
    }
    return best;
  };
  double a_prev = 0.0, f_prev = f0, a = 1.0;
  for (int it = 0; it < 20; ++it) {
    const double v = phi(a);
    consider(a, v);
    if (v > f0 + c1 * a * g0 || (it > 0 && v >= f_prev)) return zoom(a_prev, f_prev, a);
    const double g = dphi(a);
    if (std::fabs(g) <= -c2 * g0) return {a, v, true};
    if (g >= 0.0) return zoom(a, v, a_prev);
    a_prev = a;
    f_prev = v;
    a = std::min(2.0 * a, alpha_max);
    if (a_prev >= alpha_max) break;
  }
  return best;
}

}  // namespace

RefineResult local_refine(const HostModel& hm, const Vec3& r0, const Vec3& t0, const Domain& dom) {
  Objective m(hm);
  const int kMaxIt = 200, kMem = 10;
  const double kGradTol = 1e-6;
  RefineResult best;
  V6 x = {r0[0], r0[1], r0[2], t0[0], t0[1], t0[2]};
  best.value = m.value(x);
  best.r = r0;
  best.t = t0;
  if (!std::isfinite(best.value)) return best;
  auto offer = [&](const V6& xx, double fx) {
    V6 p = xx;
    if (!clamp_to_domain(m.model(), dom, &p)) return;
    const double fp = (p == xx) ? fx : m.value(p);
    if (fp < best.value) {
      best.value = fp;
      best.r = head(p);
      best.t = tail(p);
    }
  };
  double fx = best.value;
  offer(x, fx);
  V6 g = m.grad(x);
  std::deque<V6> S, Y;
  std::deque<double> Rho;
  for (int it = 0; it < kMaxIt; ++it) {
    if (norm6(g) < kGradTol) break;
    // two-loop recursion
    V6 q = g;
    std::vector<double> alpha(S.size());
    for (int i = static_cast<int>(S.size()) - 1; i >= 0; --i) {
      alpha[i] = Rho[i] * dot6(S[i], q);
      q = axpy(q, -alpha[i], Y[i]);
    }
    if (!S.empty()) {
      const double sc = dot6(S.back(), Y.back()) / dot6(Y.back(), Y.back());
      for (double& v : q) v *= sc;
    }
    for (size_t i = 0; i < S.size(); ++i) {
      const double beta = Rho[i] * dot6(Y[i], q);
      q = axpy(q, alpha[i] - beta, S[i]);
    }
    V6 d;
    for (int k = 0; k < 6; ++k) d[k] = -q[k];
    double dg = dot6(d, g);
    if (!(dg < -1e-14 * norm6(d) * norm6(g))) {  // not a descent direction
      S.clear();
      Y.clear();
      Rho.clear();
      for (int k = 0; k < 6; ++k) d[k] = -g[k];
      dg = -dot6(g, g);
    }
    const LineSearch ls = wolfe(m, x, d, fx, dg);
    if (!(ls.alpha > 0.0) || !std::isfinite(ls.value)) break;
    const V6 xn = axpy(x, ls.alpha, d);
    const V6 gn = m.grad(xn);
    V6 s, y;
    for (int k = 0; k < 6; ++k) {
      s[k] = xn[k] - x[k];
      y[k] = gn[k] - g[k];
    }
    const double sy = dot6(s, y);
    if (sy > 1e-10 * norm6(s) * norm6(y)) {
      S.push_back(s);
      Y.push_back(y);
      Rho.push_back(1.0 / sy);
      if (static_cast<int>(S.size()) > kMem) {
        S.pop_front();
        Y.pop_front();
        Rho.pop_front();
      }
    }
    x = xn;
    fx = ls.value;
    g = gn;
    offer(x, fx);
    // re-express past pi (solver.cpp:249-255)
    if (head(x).norm() > M_PI) {
      const Vec3 w = wrap_rotation_vector(head(x));
      x[0] = w[0];
      x[1] = w[1];
      x[2] = w[2];
      g = m.grad(x);
      S.clear();
      Y.clear();
      Rho.clear();
    }
  }
  return best;
}

}  // namespace gosma
