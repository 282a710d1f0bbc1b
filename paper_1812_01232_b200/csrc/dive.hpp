// Discovery-dive beam search on the device: the beam
// loop of discovery_dive (core/src/solver.cpp:459-568) - expand every beam
// node into its 8 children, bound them (K1 on the blurred context), offer
// their upper bounds to their sector's best candidate, keep the kQuota
// lowest-LB splittable children per sector - with no host round trip per
// iteration (one CUDA graph per two iterations, a device-side stop flag).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "gosma_capi.h"
#include "gosma_internal.hpp"

namespace gosma {

struct DiveBest {
  double value;  // +inf until the sector has a finite candidate
  gosma_node node;
};

// One beam entry (the host beam's Beam{b, split, sector}).
struct DiveEntry {
  gosma_node node;  // node.lower = its own lower bound
  int split;
  unsigned sector;
};

struct DiveBeamResult {
  std::vector<DiveBest> best;   // per sector
  unsigned long long used = 0;  // children bounded
};

// Runs up to max_it beam iterations from `beam` (sorted by sector) and the
// sectors' current best candidates; children are bounded with `ctx` (the
// blurred context). budget: children-evaluation budget, counted together
// with `used0` as in the host loop.
int dive_beam_device(gosma_ctx* ctx, const std::vector<DiveEntry>& beam,
                     const std::vector<DiveBest>& best0, unsigned long long used0,
                     unsigned long long budget, int max_it, int quota, double floor,
                     DiveBeamResult* out);

}  // namespace gosma
