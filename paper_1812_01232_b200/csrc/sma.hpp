// Host local refinement (host_refine.cpp: the shared L-BFGS controller over
// the host FP64 evaluator) and the pose-domain type shared by the solver.
#pragma once

#include <array>
#include <vector>

#include "host_math.hpp"

namespace gosma {

struct Box {
  Vec3 c, h;
};

// PoseDomain (se3.hpp:32-36).
struct Domain {
  Vec3 rot_center;
  double rot_hw = 0.0;
  std::vector<Box> boxes;
};

struct RefineResult {
  double value = 0.0;
  Vec3 r, t;
};

// local_refine (solver.hpp:80-85, solver.cpp:164-258).
RefineResult local_refine(const HostModel& m, const Vec3& r0, const Vec3& t0, const Domain& dom);

}  // namespace gosma
