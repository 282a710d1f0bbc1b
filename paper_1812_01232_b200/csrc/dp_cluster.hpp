// GPU scoring of points against cluster centres (dp_cluster.cu): the
// data-parallel half of a DP-means / DP-vMF-means assignment sweep.
#pragma once

#include <memory>
#include <vector>

#include "host_math.hpp"

namespace gosma {
namespace mix {

class DeviceScorer {
 public:
  DeviceScorer();
  ~DeviceScorer();
  // uploads the points once; false when no CUDA device is usable
  bool open(const std::vector<Vec3>& points, int device = 0);
  // best (lowest) score and its centre index over centres [c0, c1) for every
  // point (or the points `subset`, in that order); metric 0 = squared
  // distance, 1 = negated cosine. With `merge` the running best in
  // best / best_idx is continued (centres c0.. come after those already
  // scored; ties keep the earlier centre). Exact FP64, the reference's order.
  bool score(const std::vector<Vec3>& centres, size_t c0, size_t c1,
             const std::vector<int>* subset, int metric, bool merge, std::vector<double>* best,
             std::vector<int>* best_idx);

 private:
  struct Impl;
  std::unique_ptr<Impl> d_;
};

}  // namespace mix
}  // namespace gosma
