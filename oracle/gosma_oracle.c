/*
 * TEST INFRASTRUCTURE ONLY — plain-C, FP64, scalar restatement of the GOSMA
 * bound-evaluation hot path of the reference (/root/reference/proj/core/src).
 * It is the checker for the CUDA product path: only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg may load it. Every function cites the
 * reference file:line it follows. Pinned against (a) the reference's own
 * known-answer values (tests/test_oracle_kats.py) and (b) golden vectors
 * produced by the unmodified reference compiled in place (oracle/_ref,
 * tests/golden/make_golden.py).
 *
 * Arithmetic is kept in the reference's evaluation order (no FMA contraction:
 * built with -ffp-contract=off), so agreement with oracle/_ref is to a few ulp.
 */
#include "gosma_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#ifndef M_PI
#define M_PI 3.14159265358979323846
#endif

static __thread char g_err[256];

const char* oracle_last_error(void) { return g_err; }

typedef struct {
  int n1, n2;
  double weight;
  double* mu;     /* 3*n1 */
  double* sigma2; /* n1 */
  double* phi1;   /* n1 */
  double* b;      /* 3*n2, kappa * unit direction (objective.cpp:51) */
  double* kappa2; /* n2 */
  double* log_z2; /* n2 */
  double* phi2;   /* n2 */
} oclass;

struct oracle_ctx {
  int n_classes;
  oclass* cls;
  int n_means;
  double* means; /* pooled 3*n_means (objective.hpp:48) */
  double zeta;
  double self_energy;
};

/* ---------------------------------------------------------------- L1 math */

/* log_z_eval, sphere_stats.cpp:47-56. */
double oracle_log_z(double kappa) {
  if (kappa < 1e-4) return log(2.0) + log1p(kappa * kappa / 6.0);
  return kappa + log1p(-exp(-2.0 * kappa)) - log(kappa);
}

/* log_w, bounds.cpp:34-37. */
static double log_w(double x) {
  if (x > 30.0) return -log(x);
  return oracle_log_z(x) - x;
}

/* pair_k, bounds.cpp:40-42. */
static double pair_k(double a, double b, double c) {
  const double v = a * a + b * b + 2.0 * c * a * b;
  return sqrt(v > 0.0 ? v : 0.0);
}

static double norm3(const double* v) { return sqrt(v[0] * v[0] + v[1] * v[1] + v[2] * v[2]); }
static double dot3(const double* a, const double* b) {
  return a[0] * b[0] + a[1] * b[1] + a[2] * b[2];
}
static double clampd(double x, double lo, double hi) { return x < lo ? lo : (hi < x ? hi : x); }

/* rotation_matrix (Rodrigues), se3.cpp:21-31. R row-major R[3*i+j]. */
static void rotation_matrix(const double* r, double* R) {
  const double theta2 = r[0] * r[0] + r[1] * r[1] + r[2] * r[2];
  const double K[9] = {0.0, -r[2], r[1], r[2], 0.0, -r[0], -r[1], r[0], 0.0};
  double K2[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      K2[3 * i + j] = K[3 * i] * K[j] + K[3 * i + 1] * K[3 + j] + K[3 * i + 2] * K[6 + j];
  double a, c;
  if (theta2 < 1e-16) {
    a = 1.0;
    c = 0.5;
  } else {
    const double theta = sqrt(theta2);
    a = sin(theta) / theta;
    c = (1.0 - cos(theta)) / theta2;
  }
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      R[3 * i + j] = ((i == j ? 1.0 : 0.0) + a * K[3 * i + j]) + c * K2[3 * i + j];
}

/* point_cuboid_distance, se3.cpp:60-66. */
static void point_cuboid_distance(const double* tc, const double* thw, const double* p,
                                  double* lo, double* hi) {
  double o[3], f[3];
  for (int k = 0; k < 3; ++k) {
    const double d = fabs(p[k] - tc[k]);
    const double out = d - thw[k];
    o[k] = out > 0.0 ? out : 0.0;
    f[k] = d + thw[k];
  }
  *lo = norm3(o);
  *hi = norm3(f);
}

/* psi_rot, se3.cpp:68-70. */
static double psi_rot(double hw) {
  const double v = sqrt(3.0) * hw;
  return v < M_PI ? v : M_PI;
}

/* psi_trans, se3.cpp:72-92. */
double oracle_psi_trans(const double* tc, const double* thw, const double* p) {
  double d[3], cdir[3];
  int inside = 1;
  for (int k = 0; k < 3; ++k) {
    cdir[k] = p[k] - tc[k];
    d[k] = fabs(cdir[k]);
    if (!(d[k] <= thw[k])) inside = 0;
  }
  if (inside) return M_PI;
  double worst = 0.0;
  for (int sx = -1; sx <= 1; sx += 2)
    for (int sy = -1; sy <= 1; sy += 2)
      for (int sz = -1; sz <= 1; sz += 2) {
        const double vert[3] = {tc[0] + sx * thw[0], tc[1] + sy * thw[1], tc[2] + sz * thw[2]};
        const double v[3] = {p[0] - vert[0], p[1] - vert[1], p[2] - vert[2]};
        const double cr[3] = {cdir[1] * v[2] - cdir[2] * v[1], cdir[2] * v[0] - cdir[0] * v[2],
                              cdir[0] * v[1] - cdir[1] * v[0]};
        const double angle = atan2(norm3(cr), dot3(cdir, v));
        if (angle > worst) worst = angle;
      }
  return worst;
}

/* feasible_wrt_zeta, se3.cpp:94-100. */
static int feasible_wrt_zeta(const oracle_ctx* ctx, const double* tc, const double* thw) {
  for (int m = 0; m < ctx->n_means; ++m) {
    double lo, hi;
    point_cuboid_distance(tc, thw, ctx->means + 3 * m, &lo, &hi);
    if (hi < ctx->zeta) return 0;
  }
  return 1;
}

/* ------------------------------------------------------------ L3 context */

static int check_closure(double sum, const char* what) {
  if (fabs(sum - 1.0) > 1e-9) {
    snprintf(g_err, sizeof g_err, "%s: weights sum to %g, expected 1", what, sum);
    return 0;
  }
  return 1;
}

/* Image self-energy C2, objective.cpp:55-64. */
static double class_self_energy(const oclass* c) {
  double c2 = 0.0;
  for (int j = 0; j < c->n2; ++j)
    for (int k = 0; k < c->n2; ++k) {
      const double s[3] = {c->b[3 * j] + c->b[3 * k], c->b[3 * j + 1] + c->b[3 * k + 1],
                           c->b[3 * j + 2] + c->b[3 * k + 2]};
      const double K = norm3(s);
      c2 += c->phi2[j] * c->phi2[k] * exp(oracle_log_z(K) - c->log_z2[j] - c->log_z2[k]);
    }
  return c2;
}

/* ObjectiveContext constructors + add_class, objective.cpp:28-68, 103-121;
 * component invariants from sphere_stats.cpp:10-35 and unit_vector.hpp:17-24. */
oracle_ctx* oracle_ctx_create(int n_classes, const int* n1, const int* n2,
                              const double* class_weight, const double* mu,
                              const double* sigma2, const double* phi1, const double* dir,
                              const double* kappa2, const double* phi2, double zeta) {
  g_err[0] = 0;
  if (!(zeta > 0.0)) {
    snprintf(g_err, sizeof g_err, "ObjectiveContext: zeta must be > 0");
    return NULL;
  }
  if (n_classes < 1) {
    snprintf(g_err, sizeof g_err, "ObjectiveContext: no semantic classes");
    return NULL;
  }
  double wsum = 0.0;
  for (int c = 0; c < n_classes; ++c) wsum += class_weight[c];
  if (n_classes > 1 && !check_closure(wsum, "ObjectiveContext class weights")) return NULL;

  oracle_ctx* ctx = (oracle_ctx*)calloc(1, sizeof(oracle_ctx));
  ctx->n_classes = n_classes;
  ctx->zeta = zeta;
  ctx->cls = (oclass*)calloc((size_t)n_classes, sizeof(oclass));
  int total1 = 0;
  for (int c = 0; c < n_classes; ++c) total1 += n1[c];
  ctx->means = (double*)malloc(sizeof(double) * 3 * (size_t)(total1 > 0 ? total1 : 1));
  ctx->n_means = 0;
  long o1 = 0, o2 = 0;
  for (int c = 0; c < n_classes; ++c) {
    oclass* k = &ctx->cls[c];
    k->n1 = n1[c];
    k->n2 = n2[c];
    k->weight = class_weight[c];
    if (k->n1 < 1 || k->n2 < 1) {
      snprintf(g_err, sizeof g_err, "ObjectiveContext: class with empty mixture");
      oracle_ctx_destroy(ctx);
      return NULL;
    }
    k->mu = (double*)malloc(sizeof(double) * 3 * (size_t)k->n1);
    k->sigma2 = (double*)malloc(sizeof(double) * (size_t)k->n1);
    k->phi1 = (double*)malloc(sizeof(double) * (size_t)k->n1);
    k->b = (double*)malloc(sizeof(double) * 3 * (size_t)k->n2);
    k->kappa2 = (double*)malloc(sizeof(double) * (size_t)k->n2);
    k->log_z2 = (double*)malloc(sizeof(double) * (size_t)k->n2);
    k->phi2 = (double*)malloc(sizeof(double) * (size_t)k->n2);
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < k->n1; ++i, ++o1) {
      if (!(sigma2[o1] > 0.0) || !isfinite(sigma2[o1]) || !(phi1[o1] >= 0.0)) {
        snprintf(g_err, sizeof g_err, "IsotropicGaussian: invalid variance or weight");
        oracle_ctx_destroy(ctx);
        return NULL;
      }
      for (int a = 0; a < 3; ++a) {
        k->mu[3 * i + a] = mu[3 * o1 + a];
        ctx->means[3 * ctx->n_means + a] = mu[3 * o1 + a];
      }
      ctx->n_means++;
      k->sigma2[i] = sigma2[o1];
      k->phi1[i] = phi1[o1];
      s1 += phi1[o1];
    }
    for (int j = 0; j < k->n2; ++j, ++o2) {
      const double* d = dir + 3 * o2;
      const double n = norm3(d);
      if (!(fabs(n - 1.0) <= 1e-6) || !(kappa2[o2] > 0.0) || !isfinite(kappa2[o2]) ||
          !(phi2[o2] >= 0.0)) {
        snprintf(g_err, sizeof g_err, "VmfComponent: invalid direction, concentration or weight");
        oracle_ctx_destroy(ctx);
        return NULL;
      }
      for (int a = 0; a < 3; ++a) k->b[3 * j + a] = kappa2[o2] * (d[a] / n);
      k->kappa2[j] = kappa2[o2];
      k->log_z2[j] = oracle_log_z(kappa2[o2]);
      k->phi2[j] = phi2[o2];
      s2 += phi2[o2];
    }
    if (!check_closure(s1, "ObjectiveContext model") ||
        !check_closure(s2, "ObjectiveContext image")) {
      oracle_ctx_destroy(ctx);
      return NULL;
    }
    ctx->self_energy += k->weight * class_self_energy(k);
  }
  return ctx;
}

oracle_ctx* oracle_ctx_blurred(const oracle_ctx* src, double w, double reference_distance) {
  if (!(w >= 0.0) || !(reference_distance >= 0.0)) {
    snprintf(g_err, sizeof g_err, "ObjectiveContext::blurred: negative width");
    return NULL;
  }
  oracle_ctx* ctx = (oracle_ctx*)calloc(1, sizeof(oracle_ctx));
  *ctx = *src;
  ctx->cls = (oclass*)calloc((size_t)src->n_classes, sizeof(oclass));
  ctx->means = (double*)malloc(sizeof(double) * 3 * (size_t)src->n_means);
  memcpy(ctx->means, src->means, sizeof(double) * 3 * (size_t)src->n_means);
  ctx->self_energy = 0.0;
  const double var_add = (w * reference_distance) * (w * reference_distance);
  const double w2 = w * w;
  for (int c = 0; c < src->n_classes; ++c) {
    const oclass* s = &src->cls[c];
    oclass* k = &ctx->cls[c];
    *k = *s;
    k->mu = (double*)malloc(sizeof(double) * 3 * (size_t)s->n1);
    k->sigma2 = (double*)malloc(sizeof(double) * (size_t)s->n1);
    k->phi1 = (double*)malloc(sizeof(double) * (size_t)s->n1);
    k->b = (double*)malloc(sizeof(double) * 3 * (size_t)s->n2);
    k->kappa2 = (double*)malloc(sizeof(double) * (size_t)s->n2);
    k->log_z2 = (double*)malloc(sizeof(double) * (size_t)s->n2);
    k->phi2 = (double*)malloc(sizeof(double) * (size_t)s->n2);
    memcpy(k->mu, s->mu, sizeof(double) * 3 * (size_t)s->n1);
    memcpy(k->phi1, s->phi1, sizeof(double) * (size_t)s->n1);
    memcpy(k->phi2, s->phi2, sizeof(double) * (size_t)s->n2);
    for (int i = 0; i < s->n1; ++i) k->sigma2[i] = s->sigma2[i] + var_add;
    for (int j = 0; j < s->n2; ++j) {
      const double dir[3] = {s->b[3 * j] / s->kappa2[j], s->b[3 * j + 1] / s->kappa2[j],
                             s->b[3 * j + 2] / s->kappa2[j]};
      const double kk = s->kappa2[j] / (1.0 + s->kappa2[j] * w2);
      k->kappa2[j] = kk;
      for (int a = 0; a < 3; ++a) k->b[3 * j + a] = kk * dir[a];
      k->log_z2[j] = oracle_log_z(kk);
    }
    ctx->self_energy += k->weight * class_self_energy(k);
  }
  return ctx;
}

void oracle_ctx_destroy(oracle_ctx* ctx) {
  if (!ctx) return;
  for (int c = 0; c < ctx->n_classes; ++c) {
    oclass* k = &ctx->cls[c];
    free(k->mu);
    free(k->sigma2);
    free(k->phi1);
    free(k->b);
    free(k->kappa2);
    free(k->log_z2);
    free(k->phi2);
  }
  free(ctx->cls);
  free(ctx->means);
  free(ctx);
}

double oracle_ctx_self_energy(const oracle_ctx* ctx) { return ctx->self_energy; }

/* --------------------------------------------------------- L3 objective */

#define NEGLIGIBLE_MARGIN 64.0 /* objective.cpp:17 */

/* class_objective + project_model, objective.cpp:175-223. mass accumulates
 * |term| contributions (tolerance scale only). */
static double class_objective(const oclass* c, const double* R, const double* t, double* mass) {
  const int n1 = c->n1, n2 = c->n2;
  double* v = (double*)malloc(sizeof(double) * 3 * (size_t)n1);
  double* kap = (double*)malloc(sizeof(double) * (size_t)n1);
  double* lz = (double*)malloc(sizeof(double) * (size_t)n1);
  for (int i = 0; i < n1; ++i) {
    const double u[3] = {c->mu[3 * i] - t[0], c->mu[3 * i + 1] - t[1], c->mu[3 * i + 2] - t[2]};
    const double d2 = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    const double d = sqrt(d2);
    const double kappa = d2 / c->sigma2[i] + 1.0;
    for (int a = 0; a < 3; ++a) v[3 * i + a] = (kappa / d) * u[a];
    kap[i] = kappa;
    lz[i] = oracle_log_z(kappa);
  }
  double self_sum = 0.0, m = 0.0;
  for (int i = 0; i < n1; ++i) {
    const double diag = c->phi1[i] * c->phi1[i] * 0.5 * kap[i] / tanh(kap[i]);
    self_sum += diag;
    m += fabs(diag);
    for (int j = i + 1; j < n1; ++j) {
      const double s[3] = {v[3 * i] + v[3 * j], v[3 * i + 1] + v[3 * j + 1],
                           v[3 * i + 2] + v[3 * j + 2]};
      const double K = norm3(s);
      if (K < kap[i] + kap[j] - NEGLIGIBLE_MARGIN) continue;
      const double term = 2.0 * c->phi1[i] * c->phi1[j] * exp(oracle_log_z(K) - lz[i] - lz[j]);
      self_sum += term;
      m += fabs(term);
    }
  }
  double cross_sum = 0.0;
  for (int i = 0; i < n1; ++i) {
    const double* vi = v + 3 * i;
    double w[3];
    for (int a = 0; a < 3; ++a) w[a] = R[3 * a] * vi[0] + R[3 * a + 1] * vi[1] + R[3 * a + 2] * vi[2];
    for (int j = 0; j < n2; ++j) {
      const double s[3] = {w[0] + c->b[3 * j], w[1] + c->b[3 * j + 1], w[2] + c->b[3 * j + 2]};
      const double K = norm3(s);
      if (K < kap[i] + c->kappa2[j] - NEGLIGIBLE_MARGIN) continue;
      const double term = c->phi1[i] * c->phi2[j] * exp(oracle_log_z(K) - lz[i] - c->log_z2[j]);
      cross_sum += term;
      m += 2.0 * fabs(term);
    }
  }
  free(v);
  free(kap);
  free(lz);
  if (mass) *mass += c->weight * m;
  return self_sum - 2.0 * cross_sum;
}

static int pose_feasible(const oracle_ctx* ctx, const double* t) {
  /* check_feasible, objective.cpp:160-166 */
  for (int m = 0; m < ctx->n_means; ++m) {
    const double* mu = ctx->means + 3 * m;
    const double u[3] = {mu[0] - t[0], mu[1] - t[1], mu[2] - t[2]};
    if (norm3(u) < ctx->zeta) return 0;
  }
  return 1;
}

static double objective_value_mass(const oracle_ctx* ctx, const double* r, const double* t,
                                   double* mass) {
  /* objective_value, objective.cpp:227-235 (+inf in place of the throw). */
  if (!pose_feasible(ctx, t)) return INFINITY;
  double R[9];
  rotation_matrix(r, R);
  double f = 0.0;
  for (int c = 0; c < ctx->n_classes; ++c)
    f += ctx->cls[c].weight * class_objective(&ctx->cls[c], R, t, mass);
  return f;
}

double oracle_objective_value(const oracle_ctx* ctx, const double* r, const double* t) {
  return objective_value_mass(ctx, r, t, NULL);
}

/* ------------------------------------------------------------ L4 bounds */

/* branch_lower_core, bounds.cpp:46-183. */
static double branch_lower_core(const oracle_ctx* ctx, const double* node, double* mass) {
  const double* rc = node;
  const double rhw = node[3];
  const double* tc = node + 4;
  const double* thw = node + 7;
  double R[9];
  rotation_matrix(rc, R); /* R0t = R^T: q = R^T x → q_a = sum_b R[b][a] x_b */
  const double psi_r = psi_rot(rhw);
  const double zeta = ctx->zeta;
  double total = 0.0, tmass = 0.0;
  for (int c = 0; c < ctx->n_classes; ++c) {
    const oclass* k = &ctx->cls[c];
    const int n1 = k->n1, n2 = k->n2;
    double* buf = (double*)malloc(sizeof(double) * (size_t)(13 * n1 + 4 * n2));
    double *klo = buf, *khi = klo + n1, *lw_lo = khi + n1, *lw_hi = lw_lo + n1,
           *pt = lw_hi + n1, *cpt = pt + n1, *spt = cpt + n1, *cps = spt + n1,
           *sps = cps + n1, *uhat = sps + n1 /* 3*n1 */, *bz = uhat + 3 * n1,
           *q = bz + n1 /* 3*n2 */, *lw2 = q + 3 * n2;
    for (int i = 0; i < n1; ++i) {
      const double* mu = k->mu + 3 * i;
      double dlo0, dhi;
      point_cuboid_distance(tc, thw, mu, &dlo0, &dhi);
      const double dlo = dlo0 < zeta ? zeta : dlo0; /* std::max(d.lo, zeta) */
      klo[i] = dlo * dlo / k->sigma2[i] + 1.0;
      khi[i] = dhi * dhi / k->sigma2[i] + 1.0;
      lw_lo[i] = log_w(klo[i]);
      lw_hi[i] = log_w(khi[i]);
      const double u[3] = {mu[0] - tc[0], mu[1] - tc[1], mu[2] - tc[2]};
      const double n = norm3(u);
      if (n > 1e-12) {
        for (int a = 0; a < 3; ++a) uhat[3 * i + a] = u[a] / n;
      } else {
        uhat[3 * i] = 1.0;
        uhat[3 * i + 1] = 0.0;
        uhat[3 * i + 2] = 0.0;
      }
      pt[i] = oracle_psi_trans(tc, thw, mu);
      cpt[i] = cos(pt[i]);
      spt[i] = sin(pt[i]);
      const double ps = pt[i] + psi_r;
      bz[i] = ps >= M_PI ? 1.0 : 0.0;
      if (bz[i] == 0.0) {
        cps[i] = cos(ps);
        sps[i] = sin(ps);
      } else {
        cps[i] = -1.0;
        sps[i] = 0.0;
      }
    }
    for (int j = 0; j < n2; ++j) {
      const double x[3] = {k->b[3 * j] / k->kappa2[j], k->b[3 * j + 1] / k->kappa2[j],
                           k->b[3 * j + 2] / k->kappa2[j]};
      for (int a = 0; a < 3; ++a) q[3 * j + a] = R[a] * x[0] + R[3 + a] * x[1] + R[6 + a] * x[2];
      lw2[j] = k->log_z2[j] - k->kappa2[j];
    }

    double self_lo = 0.0, m = 0.0;
    for (int i = 0; i < n1; ++i) {
      const double diag = k->phi1[i] * k->phi1[i] * 0.5 * klo[i] / tanh(klo[i]);
      self_lo += diag;
      m += fabs(diag);
      for (int j = i + 1; j < n1; ++j) {
        double cos_a;
        if (pt[i] + pt[j] >= M_PI) {
          cos_a = -1.0;
        } else {
          const double cth = clampd(dot3(uhat + 3 * i, uhat + 3 * j), -1.0, 1.0);
          const double cpp = cpt[i] * cpt[j] - spt[i] * spt[j];
          if (cth <= -cpp) {
            cos_a = -1.0;
          } else {
            const double spp = spt[i] * cpt[j] + cpt[i] * spt[j];
            const double s2 = 1.0 - cth * cth;
            const double sth = sqrt(s2 > 0.0 ? s2 : 0.0);
            cos_a = cth * cpp - sth * spp;
          }
        }
        const double k_hh = pair_k(khi[i], khi[j], cos_a);
        const double excess_min = 2.0 * khi[i] * khi[j] * (cos_a - 1.0) / (k_hh + khi[i] + khi[j]);
        const double a1 = pair_k(klo[i], klo[j], cos_a), a2 = pair_k(klo[i], khi[j], cos_a);
        const double a3 = pair_k(khi[i], klo[j], cos_a);
        const double m12 = a1 < a2 ? a2 : a1; /* std::max */
        const double m34 = a3 < k_hh ? k_hh : a3;
        const double k_corner_max = m12 < m34 ? m34 : m12;
        const double log_term = excess_min + log_w(k_corner_max) - lw_lo[i] - lw_lo[j];
        const double term = 2.0 * k->phi1[i] * k->phi1[j] * exp(log_term);
        self_lo += term;
        m += fabs(term);
      }
    }

    double cross_hi = 0.0;
    for (int i = 0; i < n1; ++i) {
      for (int j = 0; j < n2; ++j) {
        double cos_b;
        if (bz[i] != 0.0) {
          cos_b = 1.0;
        } else {
          const double cth = clampd(dot3(uhat + 3 * i, q + 3 * j), -1.0, 1.0);
          if (cth >= cps[i]) {
            cos_b = 1.0;
          } else {
            const double s2 = 1.0 - cth * cth;
            const double sth = sqrt(s2 > 0.0 ? s2 : 0.0);
            cos_b = cth * cps[i] + sth * sps[i];
          }
        }
        const double k2 = k->kappa2[j];
        const double k_at_lo = pair_k(klo[i], k2, cos_b);
        const double excess_max = 2.0 * klo[i] * k2 * (cos_b - 1.0) / (k_at_lo + klo[i] + k2);
        const double vertex = -cos_b * k2;
        double k_min;
        if (vertex <= klo[i]) {
          k_min = k_at_lo;
        } else if (vertex >= khi[i]) {
          k_min = pair_k(khi[i], k2, cos_b);
        } else {
          const double s = (1.0 - cos_b) * (1.0 + cos_b);
          k_min = k2 * sqrt(s > 0.0 ? s : 0.0);
        }
        const double log_term = excess_max + log_w(k_min) - lw_hi[i] - lw2[j];
        const double term = k->phi1[i] * k->phi2[j] * exp(log_term);
        cross_hi += term;
        m += 2.0 * fabs(term);
      }
    }
    free(buf);
    total += k->weight * (self_lo - 2.0 * cross_hi);
    tmass += k->weight * m;
  }
  if (mass) *mass = tmass;
  return total;
}

/* feasible_center, bounds.cpp:187-214. */
int oracle_feasible_center(const oracle_ctx* ctx, const double* node, double* t_out) {
  const double zeta = ctx->zeta;
  const double* c = node + 4;
  const double* h = node + 7;
  double t[3] = {c[0], c[1], c[2]};
  for (int projection = 0; projection <= 8; ++projection) {
    const double* off = NULL;
    for (int m = 0; m < ctx->n_means; ++m) {
      const double* mu = ctx->means + 3 * m;
      const double u[3] = {mu[0] - t[0], mu[1] - t[1], mu[2] - t[2]};
      if (norm3(u) < zeta) {
        off = mu;
        break;
      }
    }
    if (!off) {
      t_out[0] = t[0];
      t_out[1] = t[1];
      t_out[2] = t[2];
      return 0;
    }
    if (projection == 8) break;
    double dir[3] = {t[0] - off[0], t[1] - off[1], t[2] - off[2]};
    const double n = norm3(dir);
    if (n > 1e-12) {
      for (int a = 0; a < 3; ++a) dir[a] = dir[a] / n;
    } else {
      dir[0] = 1.0;
      dir[1] = 0.0;
      dir[2] = 0.0;
    }
    for (int a = 0; a < 3; ++a) {
      t[a] = off[a] + dir[a] * (zeta * (1.0 + 1e-9));
      t[a] = clampd(t[a], c[a] - h[a], c[a] + h[a]);
    }
  }
  return 2;
}

/* subdivide_adaptive, se3.cpp:102-147. */
static int split_decision(const oracle_ctx* ctx, const double* node) {
  const double kFloor = 1e-9;
  const double* thw = node + 7;
  const int rot_ok = node[3] > kFloor;
  const double tmax = fmax(fmax(thw[0], thw[1]), thw[2]);
  const int trans_ok = tmax > kFloor;
  if (!rot_ok && !trans_ok) return -1;
  double psi_t = 0.0;
  for (int m = 0; m < ctx->n_means; ++m) {
    const double p = oracle_psi_trans(node + 4, thw, ctx->means + 3 * m);
    if (p > psi_t) psi_t = p;
  }
  return (rot_ok && (!trans_ok || psi_rot(node[3]) >= psi_t)) ? 1 : 0;
}

int oracle_subdivide(const oracle_ctx* ctx, const double* node, double* children) {
  const int split_rot = split_decision(ctx, node);
  if (split_rot < 0) return -1;
  int idx = 0;
  for (int sx = -1; sx <= 1; sx += 2)
    for (int sy = -1; sy <= 1; sy += 2)
      for (int sz = -1; sz <= 1; sz += 2) {
        double* ch = children + 11 * idx++;
        memcpy(ch, node, sizeof(double) * 11);
        const double sign[3] = {(double)sx, (double)sy, (double)sz};
        if (split_rot) {
          const double h = 0.5 * node[3];
          for (int a = 0; a < 3; ++a) ch[a] = node[a] + h * sign[a];
          ch[3] = h;
        } else {
          for (int a = 0; a < 3; ++a) {
            const double h = 0.5 * node[7 + a];
            ch[4 + a] = node[4 + a] + h * sign[a];
            ch[7 + a] = h;
          }
        }
        ch[10] = node[10];
      }
  return split_rot;
}

/* evaluate_bounds, bounds.cpp:275-284. */
static void eval_one(const oracle_ctx* ctx, const double* node, double skip, double* lower,
                     double* upper, double* lb_mass, double* ub_mass, int* split_rot) {
  if (split_rot) *split_rot = split_decision(ctx, node);
  if (!feasible_wrt_zeta(ctx, node + 4, node + 7)) {
    *lower = INFINITY;
    *upper = INFINITY;
    if (lb_mass) *lb_mass = 0.0;
    if (ub_mass) *ub_mass = 0.0;
    return;
  }
  double lm = 0.0, um = 0.0;
  const double core = branch_lower_core(ctx, node, &lm);
  const double lo = core < node[10] ? node[10] : core; /* std::max(core, branch.lower) */
  double up = INFINITY;
  if (!(lo >= skip)) {
    double t[3];
    if (oracle_feasible_center(ctx, node, t) == 0) up = objective_value_mass(ctx, node, t, &um);
  }
  *lower = lo;
  *upper = up;
  if (lb_mass) *lb_mass = lm;
  if (ub_mass) *ub_mass = um;
}

typedef struct {
  const oracle_ctx* ctx;
  const double* nodes;
  long n;
  double skip;
  double *lower, *upper, *lb_mass, *ub_mass;
  int* split_rot;
  long next;
  pthread_mutex_t mu;
} batch_job;

static void* batch_worker(void* arg) {
  batch_job* job = (batch_job*)arg;
  for (;;) {
    pthread_mutex_lock(&job->mu);
    const long i = job->next++;
    pthread_mutex_unlock(&job->mu);
    if (i >= job->n) return NULL;
    eval_one(job->ctx, job->nodes + 11 * i, job->skip, job->lower + i, job->upper + i,
             job->lb_mass ? job->lb_mass + i : NULL, job->ub_mass ? job->ub_mass + i : NULL,
             job->split_rot ? job->split_rot + i : NULL);
  }
}

/* evaluate_branch_batch, solver.cpp:260-292 (order-preserving fan-out). */
void oracle_eval_bounds(const oracle_ctx* ctx, const double* nodes, long n, double skip,
                        double* lower, double* upper, double* lb_mass, double* ub_mass,
                        int* split_rot, int threads) {
  if (threads <= 1 || n <= 1) {
    for (long i = 0; i < n; ++i)
      eval_one(ctx, nodes + 11 * i, skip, lower + i, upper + i, lb_mass ? lb_mass + i : NULL,
               ub_mass ? ub_mass + i : NULL, split_rot ? split_rot + i : NULL);
    return;
  }
  batch_job job = {ctx, nodes, n, skip, lower, upper, lb_mass, ub_mass, split_rot, 0};
  pthread_mutex_init(&job.mu, NULL);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)threads);
  for (int k = 0; k < threads; ++k) pthread_create(&th[k], NULL, batch_worker, &job);
  for (int k = 0; k < threads; ++k) pthread_join(th[k], NULL);
  free(th);
  pthread_mutex_destroy(&job.mu);
}
