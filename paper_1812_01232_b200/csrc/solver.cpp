// Placeholder entry points, replaced by the GPU-resident solver.
#include "capi_internal.hpp"

using namespace gosma;

extern "C" {

int gosma_local_refine(const gosma_ctx*, const double*, const double*, const gosma_domain*,
                       double*, double*, double*) {
  return set_error(GOSMA_EINVAL, "gosma_local_refine: not built yet");
}

int gosma_solve(gosma_ctx*, const gosma_domain*, const gosma_config*, gosma_report*,
                gosma_trace_cb, void*) {
  return set_error(GOSMA_EINVAL, "gosma_solve: not built yet");
}

int gosma_eval_bounds_cached_device(gosma_ctx*, const gosma_node*, size_t, const int32_t*,
                                    const double*, size_t, double, double*, double*, int8_t*,
                                    void*) {
  return set_error(GOSMA_EINVAL, "gosma_eval_bounds_cached_device: not built yet");
}
}
