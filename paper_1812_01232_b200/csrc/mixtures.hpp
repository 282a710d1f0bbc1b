// Mixture construction (off the hot path per the north star): DP-means /
// DP-vMF-means clustering (one engine; fixed centres scored on the GPU at
// scale, dp_cluster.cu) and the semantic mixture pair, with every floating
// point sum in the reference's order (core/src/mixtures.cpp:49-362), so
// results are bit-identical.
#pragma once

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "host_math.hpp"

namespace gosma {
namespace mix {

struct Clustering {
  std::vector<int> assignment;
  std::vector<Vec3> centers;
  std::vector<double> objective_history;
};

struct Gaussian {
  Vec3 mean;
  double variance;
  double weight;
};

struct Vmf {
  Vec3 direction;
  double concentration;
  double weight;
};

struct SemanticClass {
  std::string id;
  double weight = 1.0;
  std::vector<Gaussian> gmm;
  std::vector<Vmf> vmfmm;
};

struct SemanticMixturePair {
  std::vector<SemanticClass> classes;
  std::vector<std::string> warnings;
};

// UnitVector3(v) (unit_vector.hpp:16-23): accepts |v| within 1e-6 of 1 and
// renormalises; throws std::invalid_argument otherwise.
Vec3 unit_vector(const Vec3& v);

Clustering dp_means(const std::vector<Vec3>& points, double lambda_p,
                    std::optional<std::uint64_t> shuffle_seed = std::nullopt);
Clustering dp_vmf_means(const std::vector<Vec3>& bearings, double lambda_f,
                        std::optional<std::uint64_t> shuffle_seed = std::nullopt);
// component fits from a clustering of x (fit_gaussian_components /
// fit_vmf_components, mixtures.cpp:204-267)
std::vector<Gaussian> fit_gaussians(const std::vector<Vec3>& x, const Clustering& c,
                                    double sigma2_min);
std::vector<Vmf> fit_vmfs(const std::vector<Vec3>& x, const Clustering& c,
                          double kappa_min = 1e-3, double kappa_max = 1e5);
SemanticMixturePair build_semantic_mixtures(
    const std::vector<Vec3>& points, const std::vector<std::string>& point_labels,
    const std::vector<Vec3>& bearings, const std::vector<std::string>& bearing_labels,
    double lambda_p, double lambda_f,
    const std::optional<std::map<std::string, double>>& class_weights = std::nullopt);

}  // namespace mix
}  // namespace gosma
