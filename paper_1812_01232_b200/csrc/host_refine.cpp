// Host local refinement: the shared L-BFGS controller (refine_core.hpp, the
// same code the GPU refiner runs per CTA) over the host FP64 evaluator
// (host_math.cpp). Used for small mixtures, where one host thread per start
// beats a CTA's latency (solver.cpp: gpu_sma).
#include <cmath>
#include <limits>

#include "refine_core.hpp"
#include "sma.hpp"

namespace gosma {

namespace {

// Objective with a one-pose cache (the controller evaluates each accepted
// step's gradient once more), and the domain projection.
struct HostObjective {
  const HostModel& m;
  const Domain& dom;
  bool have = false;
  double x[6] = {0, 0, 0, 0, 0, 0}, f = 0.0, g[6] = {0, 0, 0, 0, 0, 0};

  void eval(const double* xx) {
    bool same = have;
    for (int k = 0; k < 6; ++k) same = same && xx[k] == x[k];
    if (same) return;
    f = objective_and_gradient(m, Vec3(xx[0], xx[1], xx[2]), Vec3(xx[3], xx[4], xx[5]), g);
    for (int k = 0; k < 6; ++k) x[k] = xx[k];
    have = true;
  }
  double value(const double* xx) {
    eval(xx);
    return f;
  }
  const double* grad() const { return g; }

  // Clamp r into the rotation cube and t into the nearest translation box
  // (smallest distance, then lowest index), then push t out of standoff balls
  // (first offending mean, up to 8 times, staying in the box); false when no
  // feasible point is reached.
  bool project(double* p) const {
    for (int k = 0; k < 3; ++k)
      p[k] = std::fmin(std::fmax(p[k], dom.rot_center[k] - dom.rot_hw),
                       dom.rot_center[k] + dom.rot_hw);
    const Box* box = nullptr;
    double best = std::numeric_limits<double>::infinity();
    for (const Box& b : dom.boxes) {
      double s2 = 0.0;
      for (int k = 0; k < 3; ++k) {
        const double o = std::fmax(std::fabs(p[3 + k] - b.c[k]) - b.h[k], 0.0);
        s2 += o * o;
      }
      const double d = std::sqrt(s2);
      if (d < best) {
        best = d;
        box = &b;
      }
    }
    if (!box) return false;
    double q[3];
    for (int k = 0; k < 3; ++k)
      q[k] = std::fmin(std::fmax(p[3 + k], box->c[k] - box->h[k]), box->c[k] + box->h[k]);
    for (int pass = 0; pass <= 8; ++pass) {
      const Vec3* hit = nullptr;
      for (const Vec3& mu : m.all_means) {
        const double dx = mu[0] - q[0], dy = mu[1] - q[1], dz = mu[2] - q[2];
        if (std::sqrt(dx * dx + dy * dy + dz * dz) < m.zeta) {
          hit = &mu;
          break;
        }
      }
      if (!hit) {
        for (int k = 0; k < 3; ++k) p[3 + k] = q[k];
        return true;
      }
      if (pass == 8) break;
      double dir[3] = {q[0] - (*hit)[0], q[1] - (*hit)[1], q[2] - (*hit)[2]};
      const double n = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
      if (n > 1e-12) {
        for (double& c : dir) c /= n;
      } else {
        dir[0] = 1.0;
        dir[1] = dir[2] = 0.0;
      }
      for (int k = 0; k < 3; ++k)
        q[k] = std::fmin(std::fmax((*hit)[k] + dir[k] * (m.zeta * (1.0 + 1e-9)),
                                   box->c[k] - box->h[k]),
                         box->c[k] + box->h[k]);
    }
    return false;
  }
};

struct HostHistory {
  double S[refine::kMem][6], Y[refine::kMem][6], Rho[refine::kMem];
  void put(int slot, const double* s, const double* y, double rho) {
    for (int k = 0; k < 6; ++k) {
      S[slot][k] = s[k];
      Y[slot][k] = y[k];
    }
    Rho[slot] = rho;
  }
};

}  // namespace

RefineResult local_refine(const HostModel& m, const Vec3& r0, const Vec3& t0, const Domain& dom) {
  HostObjective ob{m, dom};
  HostHistory h;
  double x[6] = {r0[0], r0[1], r0[2], t0[0], t0[1], t0[2]}, f = 0.0;
  refine::lbfgs_refine(ob, h, x, &f);
  RefineResult r;
  r.value = f;
  r.r = Vec3(x[0], x[1], x[2]);
  r.t = Vec3(x[3], x[4], x[5]);
  return r;
}

}  // namespace gosma
