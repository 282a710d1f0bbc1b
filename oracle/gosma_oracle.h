/* TEST INFRASTRUCTURE ONLY — see gosma_oracle.c. */
#ifndef GOSMA_ORACLE_H
#define GOSMA_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

typedef struct oracle_ctx oracle_ctx;

/* Mirrors ObjectiveContext(SemanticMixturePair, zeta) (objective.cpp:28-68,
 * 109-121): per-class model means/variances/weights and image
 * directions/concentrations/weights, concatenated over classes. Returns NULL
 * on invalid input (message via oracle_last_error). */
oracle_ctx* oracle_ctx_create(int n_classes, const int* n1, const int* n2,
                              const double* class_weight, const double* mu,
                              const double* sigma2, const double* phi1, const double* dir,
                              const double* kappa2, const double* phi2, double zeta);
/* ObjectiveContext::blurred (objective.cpp:70-101). */
oracle_ctx* oracle_ctx_blurred(const oracle_ctx* ctx, double w, double reference_distance);
void oracle_ctx_destroy(oracle_ctx* ctx);
const char* oracle_last_error(void);
double oracle_ctx_self_energy(const oracle_ctx* ctx);

double oracle_log_z(double kappa);
double oracle_psi_trans(const double* tc, const double* thw, const double* p);

/* node = {rc[3], rhw, tc[3], thw[3], lower} (11 doubles). */
/* evaluate_bounds (bounds.cpp:275-284) plus diagnostics: lb_mass/ub_mass =
 * sum of |pair-term contributions| (the parity tolerance scale), split_rot =
 * subdivide_adaptive's decision (se3.cpp:107-121) or -1 if not splittable. */
void oracle_eval_bounds(const oracle_ctx* ctx, const double* nodes, long n, double skip,
                        double* lower, double* upper, double* lb_mass, double* ub_mass,
                        int* split_rot, int threads);
double oracle_objective_value(const oracle_ctx* ctx, const double* r, const double* t);
/* feasible_center (bounds.cpp:187-214): 0 ok (t_out written), 2 none. */
int oracle_feasible_center(const oracle_ctx* ctx, const double* node, double* t_out);
/* subdivide_adaptive (se3.cpp:107-147): returns split-rotation flag, -1 if
 * not splittable. */
int oracle_subdivide(const oracle_ctx* ctx, const double* node, double* children);

#ifdef __cplusplus
}
#endif
#endif
