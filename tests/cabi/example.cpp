// Plain C++ use of the C ABI (include/gosma_capi.h): the binding a reference
// maintainer adds. Built and run by tests/test_cabi_gpu.py.
#include <cmath>
#include <cstdio>
#include <vector>

#include "gosma_capi.h"

static int fail(const char* what) {
  std::fprintf(stderr, "FAIL %s: %s\n", what, gosma_last_error());
  return 1;
}

int main() {
  // test_solver.cpp:112-117: one Gaussian at (0,0,2), var 4; vMF +z, kappa 2.
  const double mu[3] = {0, 0, 2}, s2[1] = {4.0}, p1[1] = {1.0};
  const double dir[3] = {0, 0, 1}, k2[1] = {2.0}, p2[1] = {1.0};
  gosma_class_view v{1, 1, 1.0, mu, s2, p1, dir, k2, p2};
  gosma_ctx* ctx = nullptr;
  if (gosma_ctx_create(0, &v, 1, 0.5, GOSMA_CTX_SINGLE_MIXTURE, &ctx)) return fail("ctx");
  // invalid arguments map to GOSMA_EINVAL
  gosma_ctx* bad = nullptr;
  if (gosma_ctx_create(0, &v, 1, 0.0, GOSMA_CTX_SINGLE_MIXTURE, &bad) != GOSMA_EINVAL)
    return fail("zeta validation");
  // f* = -Z(4)/Z(2)^2 at the identity
  const double z2 = (std::exp(2.0) - std::exp(-2.0)) / 2.0;
  const double z4 = (std::exp(4.0) - std::exp(-4.0)) / 4.0;
  const double fstar = -z4 / (z2 * z2);
  const double r0[3] = {0, 0, 0}, t0[3] = {0, 0, 0};
  double f = 0.0;
  if (gosma_objective_value(ctx, r0, t0, &f)) return fail("objective");
  if (std::fabs(f - fstar) > 1e-12) return fail("objective value");
  const double tin[3] = {0, 0, 1.8};
  if (gosma_objective_value(ctx, r0, tin, &f) != GOSMA_EINFEASIBLE) return fail("standoff");
  // bounds of a few branches around the optimum
  std::vector<gosma_node> nodes;
  for (int k = 0; k < 16; ++k) {
    const double h = 0.4 / (1 << (k % 4));
    nodes.push_back({{0.01 * k, 0, 0}, h, {0.05, -0.03, 0.02}, {h, h, h}, -INFINITY});
  }
  std::vector<double> lo(nodes.size()), up(nodes.size());
  std::vector<int8_t> sp(nodes.size());
  if (gosma_eval_bounds(ctx, nodes.data(), nodes.size(), INFINITY, lo.data(), up.data(),
                        sp.data()))
    return fail("eval");
  for (size_t k = 0; k < nodes.size(); ++k) {
    if (!(lo[k] <= up[k]) || !(lo[k] <= fstar + 1e-9)) return fail("bound order");
    if (sp[k] < -1 || sp[k] > 1) return fail("split flag");
  }
  // full solve (test_solver.cpp:105-140): certified within eps = 0.3
  const double boxes[6] = {0.05, -0.03, 0.02, 0.4, 0.4, 0.4};
  gosma_domain dom{{0, 0, 0}, 0.4, boxes, 1};
  gosma_config cfg{0.3, 0.5, 1024, -1.0, 3000000, -1, 0, 0, 0, 1};
  gosma_report rep{};
  if (gosma_solve(ctx, &dom, &cfg, &rep, nullptr, nullptr)) return fail("solve");
  if (rep.status != GOSMA_STATUS_EPSILON_OPTIMAL) return fail("solve status");
  if (std::fabs(rep.best_value - fstar) > 1e-6) return fail("solve optimum");
  if (!(rep.global_lower <= fstar + 1e-9)) return fail("certified bound");
  gosma_ctx_destroy(ctx);
  std::printf("cabi example ok: f*=%.12f d*=%.12f lower=%.6f evals=%llu\n", fstar,
              rep.best_value, rep.global_lower, rep.bound_evaluations);
  return 0;
}
