// C ABI of the host mixture construction (include/gosma_capi.h).
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "capi_internal.hpp"
#include "gosma_capi.h"
#include "mixtures.hpp"

struct gosma_mixtures {
  gosma::mix::SemanticMixturePair pair;
  // flattened per-class arrays behind the views
  struct Flat {
    std::vector<double> mu, sigma2, phi1, dir, kappa2, phi2;
  };
  std::vector<Flat> flat;
};

namespace {

std::vector<gosma::Vec3> vec3s(const double* p, size_t n) {
  std::vector<gosma::Vec3> v(n);
  for (size_t i = 0; i < n; ++i) v[i] = gosma::Vec3(p[3 * i], p[3 * i + 1], p[3 * i + 2]);
  return v;
}

std::vector<std::string> labels(const char* const* l, size_t n) {
  std::vector<std::string> out;
  if (!l) return out;
  out.reserve(n);
  for (size_t i = 0; i < n; ++i) {
    if (!l[i]) throw std::invalid_argument("null label");
    out.emplace_back(l[i]);
  }
  return out;
}

int clustering_out(const gosma::mix::Clustering& c, int* assignment, double* centers,
                   size_t cap, size_t* n_centers, int* iterations) {
  if (n_centers) *n_centers = c.centers.size();
  if (iterations) *iterations = static_cast<int>(c.objective_history.size());
  if (assignment) std::memcpy(assignment, c.assignment.data(), c.assignment.size() * sizeof(int));
  if (centers) {
    if (c.centers.size() > cap) return gosma::set_error(GOSMA_EINVAL, "centers_cap too small");
    for (size_t k = 0; k < c.centers.size(); ++k)
      for (int a = 0; a < 3; ++a) centers[3 * k + a] = c.centers[k][a];
  }
  return GOSMA_OK;
}

}  // namespace

extern "C" {

int gosma_mixtures_build(const double* points, const char* const* point_labels,
                         size_t n_points, const double* bearings,
                         const char* const* bearing_labels, size_t n_bearings, double lambda_p,
                         double lambda_f, const char* const* weight_labels,
                         const double* weights, size_t n_weights, gosma_mixtures** out) {
  if (!out) return gosma::set_error(GOSMA_EINVAL, "null output");
  *out = nullptr;
  if ((n_points && !points) || (n_bearings && !bearings))
    return gosma::set_error(GOSMA_EINVAL, "null buffer");
  try {
    std::vector<gosma::Vec3> b = vec3s(bearings, n_bearings);
    for (gosma::Vec3& v : b) v = gosma::mix::unit_vector(v);
    std::optional<std::map<std::string, double>> cw;
    if (weights) {
      if (!weight_labels) throw std::invalid_argument("class weights need labels");
      cw.emplace();
      for (size_t k = 0; k < n_weights; ++k) (*cw)[weight_labels[k]] = weights[k];
    }
    auto* m = new gosma_mixtures();
    try {
      m->pair = gosma::mix::build_semantic_mixtures(
          vec3s(points, n_points), labels(point_labels, n_points), b,
          labels(bearing_labels, n_bearings), lambda_p, lambda_f, cw);
    } catch (...) {
      delete m;
      throw;
    }
    for (const auto& cls : m->pair.classes) {
      gosma_mixtures::Flat f;
      for (const auto& g : cls.gmm) {
        for (int a = 0; a < 3; ++a) f.mu.push_back(g.mean[a]);
        f.sigma2.push_back(g.variance);
        f.phi1.push_back(g.weight);
      }
      for (const auto& v : cls.vmfmm) {
        for (int a = 0; a < 3; ++a) f.dir.push_back(v.direction[a]);
        f.kappa2.push_back(v.concentration);
        f.phi2.push_back(v.weight);
      }
      m->flat.push_back(std::move(f));
    }
    *out = m;
    return GOSMA_OK;
  } catch (const std::invalid_argument& e) {
    return gosma::set_error(GOSMA_EINVAL, e.what());
  } catch (const std::exception& e) {
    return gosma::set_error(GOSMA_EINVAL, e.what());
  }
}

int gosma_mixtures_class_count(const gosma_mixtures* m) {
  return m ? static_cast<int>(m->pair.classes.size()) : 0;
}

int gosma_mixtures_class(const gosma_mixtures* m, int k, gosma_class_view* view,
                         const char** id) {
  if (!m || !view || k < 0 || k >= static_cast<int>(m->pair.classes.size()))
    return gosma::set_error(GOSMA_EINVAL, "bad class index");
  const auto& cls = m->pair.classes[k];
  const auto& f = m->flat[k];
  view->n1 = static_cast<int>(cls.gmm.size());
  view->n2 = static_cast<int>(cls.vmfmm.size());
  view->class_weight = cls.weight;
  view->mu = f.mu.data();
  view->sigma2 = f.sigma2.data();
  view->phi1 = f.phi1.data();
  view->dir = f.dir.data();
  view->kappa2 = f.kappa2.data();
  view->phi2 = f.phi2.data();
  if (id) *id = cls.id.c_str();
  return GOSMA_OK;
}

int gosma_mixtures_warning_count(const gosma_mixtures* m) {
  return m ? static_cast<int>(m->pair.warnings.size()) : 0;
}

const char* gosma_mixtures_warning(const gosma_mixtures* m, int k) {
  if (!m || k < 0 || k >= static_cast<int>(m->pair.warnings.size())) return nullptr;
  return m->pair.warnings[k].c_str();
}

void gosma_mixtures_destroy(gosma_mixtures* m) { delete m; }

int gosma_dp_means(const double* points, size_t n, double lambda_p, int shuffle,
                   unsigned long long seed, int* assignment, double* centers, size_t centers_cap,
                   size_t* n_centers, int* iterations) {
  if (n && !points) return gosma::set_error(GOSMA_EINVAL, "null buffer");
  try {
    const auto c = gosma::mix::dp_means(vec3s(points, n), lambda_p,
                                        shuffle ? std::optional<std::uint64_t>(seed)
                                                : std::nullopt);
    return clustering_out(c, assignment, centers, centers_cap, n_centers, iterations);
  } catch (const std::exception& e) {
    return gosma::set_error(GOSMA_EINVAL, e.what());
  }
}

int gosma_dp_vmf_means(const double* bearings, size_t n, double lambda_f, int shuffle,
                       unsigned long long seed, int* assignment, double* centers,
                       size_t centers_cap, size_t* n_centers, int* iterations) {
  if (n && !bearings) return gosma::set_error(GOSMA_EINVAL, "null buffer");
  try {
    std::vector<gosma::Vec3> b = vec3s(bearings, n);
    for (gosma::Vec3& v : b) v = gosma::mix::unit_vector(v);
    const auto c = gosma::mix::dp_vmf_means(b, lambda_f,
                                            shuffle ? std::optional<std::uint64_t>(seed)
                                                    : std::nullopt);
    return clustering_out(c, assignment, centers, centers_cap, n_centers, iterations);
  } catch (const std::exception& e) {
    return gosma::set_error(GOSMA_EINVAL, e.what());
  }
}

}  // extern "C"
