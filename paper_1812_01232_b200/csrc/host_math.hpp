// Small fixed-size FP64 linear algebra and the host model (the FP64 master
// copy of an ObjectiveContext) for the host-side solver pieces.
#pragma once

#include <cmath>
#include <vector>

#include "gosma_internal.hpp"

namespace gosma {

struct Vec3 {
  double v[3] = {0.0, 0.0, 0.0};
  Vec3() = default;
  Vec3(double x, double y, double z) : v{x, y, z} {}
  double& operator[](int k) { return v[k]; }
  double operator[](int k) const { return v[k]; }
  Vec3 operator+(const Vec3& o) const { return {v[0] + o.v[0], v[1] + o.v[1], v[2] + o.v[2]}; }
  Vec3 operator-(const Vec3& o) const { return {v[0] - o.v[0], v[1] - o.v[1], v[2] - o.v[2]}; }
  Vec3 operator*(double s) const { return {v[0] * s, v[1] * s, v[2] * s}; }
  Vec3 operator/(double s) const { return {v[0] / s, v[1] / s, v[2] / s}; }
  bool operator==(const Vec3& o) const {
    return v[0] == o.v[0] && v[1] == o.v[1] && v[2] == o.v[2];
  }
  double dot(const Vec3& o) const { return v[0] * o.v[0] + v[1] * o.v[1] + v[2] * o.v[2]; }
  double norm() const { return std::sqrt(dot(*this)); }
  Vec3 cross(const Vec3& o) const {
    return {v[1] * o.v[2] - v[2] * o.v[1], v[2] * o.v[0] - v[0] * o.v[2],
            v[0] * o.v[1] - v[1] * o.v[0]};
  }
};

struct Mat3 {
  double m[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};  // row-major
  static Mat3 identity() {
    Mat3 r;
    r.m[0] = r.m[4] = r.m[8] = 1.0;
    return r;
  }
  static Mat3 skew(const Vec3& r) {
    Mat3 k;
    k.m[1] = -r[2];
    k.m[2] = r[1];
    k.m[3] = r[2];
    k.m[5] = -r[0];
    k.m[6] = -r[1];
    k.m[7] = r[0];
    return k;
  }
  static Mat3 outer(const Vec3& a, const Vec3& b) {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[3 * i + j] = a[i] * b[j];
    return r;
  }
  Mat3 operator*(const Mat3& o) const {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        r.m[3 * i + j] =
            m[3 * i] * o.m[j] + m[3 * i + 1] * o.m[3 + j] + m[3 * i + 2] * o.m[6 + j];
    return r;
  }
  Vec3 operator*(const Vec3& x) const {
    return {m[0] * x[0] + m[1] * x[1] + m[2] * x[2], m[3] * x[0] + m[4] * x[1] + m[5] * x[2],
            m[6] * x[0] + m[7] * x[1] + m[8] * x[2]};
  }
  Mat3 operator*(double s) const {
    Mat3 r;
    for (int i = 0; i < 9; ++i) r.m[i] = m[i] * s;
    return r;
  }
  Mat3 operator+(const Mat3& o) const {
    Mat3 r;
    for (int i = 0; i < 9; ++i) r.m[i] = m[i] + o.m[i];
    return r;
  }
  Mat3 operator-(const Mat3& o) const {
    Mat3 r;
    for (int i = 0; i < 9; ++i) r.m[i] = m[i] - o.m[i];
    return r;
  }
  Mat3 transpose() const {
    Mat3 r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r.m[3 * j + i] = m[3 * i + j];
    return r;
  }
};

// FP64 master copy of an ObjectiveContext (objective.hpp:17-62).
struct HostModel {
  std::vector<HostClass> classes;
  std::vector<Vec3> all_means;
  double zeta = 0.5;
  double image_self_energy = 0.0;
};

Mat3 rotation_matrix(const Vec3& r);
Vec3 wrap_rotation_vector(const Vec3& r);
bool pose_feasible(const HostModel& model, const Vec3& t);
double objective_value(const HostModel& model, const Vec3& r, const Vec3& t);
bool objective_gradient(const HostModel& model, const Vec3& r, const Vec3& t, double g[6]);
// value and gradient in one pass (+inf and a zero gradient when infeasible)
double objective_and_gradient(const HostModel& model, const Vec3& r, const Vec3& t, double g[6]);
bool feasible_center(const HostModel& model, const Vec3& c, const Vec3& h, Vec3* t_out);
double point_box_lo(const Vec3& p, const Vec3& c, const Vec3& h);
double point_box_hi(const Vec3& p, const Vec3& c, const Vec3& h);
double psi_trans(const Vec3& c, const Vec3& h, const Vec3& p);

}  // namespace gosma

namespace gosma {
// FP64 lower bound of one branch (bounds.cpp:46-183, 270-273); +inf if infeasible.
double lower_bound_fp64(const HostModel& model, const Vec3& rc, double rhw, const Vec3& tc,
                        const Vec3& th, double parent_lower);
}  // namespace gosma
