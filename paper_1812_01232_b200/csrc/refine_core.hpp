// One L-BFGS local-refinement controller for both sides of the path: the
// GPU-resident refiner (objective_kernel.cu, one CTA / cluster per start,
// every thread running this code on identical values) and the host refiner
// (host_refine.cpp). The objective supplies the evaluations, the domain
// projection and the storage of the curvature pairs, so the search itself is
// written once.
//
// Behaviour (the reference's SMA contract, core/include/smalign/solver.hpp:
// 75-85, core/src/solver.cpp:105-258): quasi-Newton steps with memory 10
// from a feasible start, strong-Wolfe line search (c1 = 1e-4, c2 = 0.9,
// doubling bracket up to 1e3 in <= 20 trials, bisection zoom in <= 30),
// stop at |g| < 1e-6 or 200 iterations, every iterate offered to the domain
// projection and the best projected point returned (never worse than the
// start), rotation vectors re-expressed inside the pi-ball with the history
// reset.
//
//   Obj:  double value(const double x[6]);   f (+inf outside the standoff)
//         void   eval(const double x[6]);    f and gradient at x (cached)
//         const double* grad() const;        gradient of the last eval
//         bool   project(double p[6]);       clamp into the domain (false: no
//                                            feasible point)
//   Hist: double (&S)[kMem][6], (&Y)[kMem][6], (&Rho)[kMem] readable by all;
//         void put(int slot, const double s[6], const double y[6], double rho)
#pragma once

#include <cmath>

#ifdef __CUDACC__
#define GOSMA_HD __host__ __device__
#else
#define GOSMA_HD
#endif

namespace gosma {
namespace refine {

constexpr int kMem = 10;
constexpr int kMaxIterations = 200;
constexpr double kGradTol = 1e-6;

GOSMA_HD inline double dot6(const double* a, const double* b) {
  double s = 0.0;
  for (int k = 0; k < 6; ++k) s += a[k] * b[k];
  return s;
}

struct Step {
  double alpha = 0.0, value = INFINITY;
};

// Strong-Wolfe search along d from x (value f0, slope g0 < 0): doubling
// bracket, then bisection; returns the best sufficient-decrease point seen
// when neither phase meets the curvature condition.
template <class Obj>
GOSMA_HD Step wolfe_step(Obj& ob, const double* x, const double* d, double f0, double g0) {
  constexpr double c1 = 1e-4, c2 = 0.9, kAlphaMax = 1e3;
  double xt[6];
  Step best;
  auto trial = [&](double a) -> double {
    for (int k = 0; k < 6; ++k) xt[k] = x[k] + a * d[k];
    const double v = ob.value(xt);
    if (v <= f0 + c1 * a * g0 && v < best.value) {
      best.alpha = a;
      best.value = v;
    }
    return v;
  };
  double lo = 0.0, flo = f0, hi = 0.0;
  bool bracketed = false;
  double a = 1.0;
  for (int it = 0; it < 20 && !bracketed; ++it) {
    const double v = trial(a);
    if (v > f0 + c1 * a * g0 || (it > 0 && v >= flo)) {
      hi = a;  // the minimum lies between the previous trial and this one
      bracketed = true;
      break;
    }
    const double g = dot6(ob.grad(), d);
    if (fabs(g) <= -c2 * g0) return Step{a, v};
    if (g >= 0.0) {  // overshot the minimum: bracket [a, previous]
      hi = lo;
      lo = a;
      flo = v;
      bracketed = true;
      break;
    }
    lo = a;
    flo = v;
    a = fmin(2.0 * a, kAlphaMax);
    if (lo >= kAlphaMax) return best;
  }
  if (!bracketed) return best;
  for (int it = 0; it < 30; ++it) {
    const double m = 0.5 * (lo + hi);
    const double v = trial(m);
    if (v > f0 + c1 * m * g0 || v >= flo) {
      hi = m;
      continue;
    }
    const double g = dot6(ob.grad(), d);
    if (fabs(g) <= -c2 * g0) return Step{m, v};
    if (g * (hi - lo) >= 0.0) hi = lo;
    lo = m;
    flo = v;
  }
  return best;
}

// Refines x[6] = (r, t) in place to the best projected point found; *fout
// receives its value (the start's when nothing better is found; +inf starts
// are returned unchanged).
template <class Obj, class Hist>
GOSMA_HD void lbfgs_refine(Obj& ob, Hist& H, double* x_io, double* fout) {
  double x[6], bx[6];
  for (int k = 0; k < 6; ++k) x[k] = bx[k] = x_io[k];
  double bf = ob.value(x);
  if (!(bf < INFINITY)) {
    *fout = bf;
    return;
  }
  auto offer = [&](const double* xx, double fx) {
    double p[6];
    for (int k = 0; k < 6; ++k) p[k] = xx[k];
    if (!ob.project(p)) return;
    bool moved = false;
    for (int k = 0; k < 6; ++k) moved = moved || p[k] != xx[k];
    const double fp = moved ? ob.value(p) : fx;
    if (fp < bf) {
      bf = fp;
      for (int k = 0; k < 6; ++k) bx[k] = p[k];
    }
  };
  double fx = bf;
  offer(x, fx);
  ob.eval(x);
  double g[6];
  for (int k = 0; k < 6; ++k) g[k] = ob.grad()[k];
  int nh = 0, h0 = 0;  // ring of the last nh curvature pairs, oldest at h0
  for (int it = 0; it < kMaxIterations; ++it) {
    if (sqrt(dot6(g, g)) < kGradTol) break;
    // two-loop recursion: d = -H g
    double q[6], alpha[kMem];
    for (int k = 0; k < 6; ++k) q[k] = g[k];
    for (int i = nh - 1; i >= 0; --i) {
      const int s = (h0 + i) % kMem;
      alpha[i] = H.Rho[s] * dot6(H.S[s], q);
      for (int k = 0; k < 6; ++k) q[k] -= alpha[i] * H.Y[s][k];
    }
    if (nh > 0) {
      const int s = (h0 + nh - 1) % kMem;
      const double scale = dot6(H.S[s], H.Y[s]) / dot6(H.Y[s], H.Y[s]);
      for (int k = 0; k < 6; ++k) q[k] *= scale;
    }
    for (int i = 0; i < nh; ++i) {
      const int s = (h0 + i) % kMem;
      const double beta = H.Rho[s] * dot6(H.Y[s], q);
      for (int k = 0; k < 6; ++k) q[k] += (alpha[i] - beta) * H.S[s][k];
    }
    double d[6];
    for (int k = 0; k < 6; ++k) d[k] = -q[k];
    double dg = dot6(d, g);
    if (!(dg < -1e-14 * sqrt(dot6(d, d)) * sqrt(dot6(g, g)))) {
      // not a descent direction: forget the history, steepest descent
      nh = h0 = 0;
      for (int k = 0; k < 6; ++k) d[k] = -g[k];
      dg = -dot6(g, g);
    }
    const Step st = wolfe_step(ob, x, d, fx, dg);
    if (!(st.alpha > 0.0) || !(st.value < INFINITY)) break;
    double xn[6], s[6], y[6];
    for (int k = 0; k < 6; ++k) xn[k] = x[k] + st.alpha * d[k];
    ob.eval(xn);
    for (int k = 0; k < 6; ++k) {
      s[k] = xn[k] - x[k];
      y[k] = ob.grad()[k] - g[k];
    }
    const double sy = dot6(s, y);
    if (sy > 1e-10 * sqrt(dot6(s, s)) * sqrt(dot6(y, y))) {  // curvature pair kept
      int slot;
      if (nh < kMem) {
        slot = (h0 + nh) % kMem;
        ++nh;
      } else {
        slot = h0;
        h0 = (h0 + 1) % kMem;
      }
      H.put(slot, s, y, 1.0 / sy);
    }
    for (int k = 0; k < 6; ++k) {
      x[k] = xn[k];
      g[k] = ob.grad()[k];
    }
    fx = st.value;
    offer(x, fx);
    // keep the rotation vector inside the pi-ball (same rotation)
    const double rn = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
    if (rn > M_PI) {
      double n = rn;
      while (n > M_PI) {
        const double f = 1.0 - 2.0 * M_PI / n;
        for (int k = 0; k < 3; ++k) x[k] *= f;
        n = sqrt(x[0] * x[0] + x[1] * x[1] + x[2] * x[2]);
      }
      ob.eval(x);
      for (int k = 0; k < 6; ++k) g[k] = ob.grad()[k];
      nh = h0 = 0;
    }
  }
  for (int k = 0; k < 6; ++k) x_io[k] = bx[k];
  *fout = bf;
}

}  // namespace refine
}  // namespace gosma
