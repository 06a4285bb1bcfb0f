// pot/registration.hpp — drop-in mirror of the reference's rigid point-cloud
// registration (/root/reference/proj/include/pot/registration.hpp), backed by
// potgpu_register_point_clouds / potgpu_fit_rigid (include/potgpu.h).
// Matrix3d / Vector3d stand in for Eigen's fixed-size types with the subset
// of their interface the reference API exposes.
#pragma once

#include <array>
#include <cmath>
#include <vector>

#include "pot.hpp"

namespace pot {

struct Vector3d {
  std::array<double, 3> v{0, 0, 0};
  Vector3d() = default;
  Vector3d(double a, double b, double c) : v{a, b, c} {}
  static Vector3d Zero() { return Vector3d(); }
  double& operator()(int i) { return v[size_t(i)]; }
  double operator()(int i) const { return v[size_t(i)]; }
  Vector3d operator+(const Vector3d& o) const { return Vector3d(v[0] + o.v[0], v[1] + o.v[1], v[2] + o.v[2]); }
  Vector3d operator-(const Vector3d& o) const { return Vector3d(v[0] - o.v[0], v[1] - o.v[1], v[2] - o.v[2]); }
  Vector3d operator-() const { return Vector3d(-v[0], -v[1], -v[2]); }
  double norm() const { return std::sqrt((v[0] * v[0] + v[1] * v[1]) + v[2] * v[2]); }
};

struct Matrix3d {  // row-major storage, (i, j) indexing
  std::array<double, 9> a{0, 0, 0, 0, 0, 0, 0, 0, 0};
  static Matrix3d Identity() { Matrix3d m; m.a = {1, 0, 0, 0, 1, 0, 0, 0, 1}; return m; }
  static Matrix3d Zero() { return Matrix3d(); }
  double& operator()(int i, int j) { return a[size_t(3 * i + j)]; }
  double operator()(int i, int j) const { return a[size_t(3 * i + j)]; }
  Matrix3d operator*(const Matrix3d& o) const {
    Matrix3d r;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) r(i, j) = ((*this)(i, 0) * o(0, j) + (*this)(i, 1) * o(1, j)) + (*this)(i, 2) * o(2, j);
    return r;
  }
  Vector3d operator*(const Vector3d& x) const {
    Vector3d r;
    for (int i = 0; i < 3; ++i) r(i) = ((*this)(i, 0) * x(0) + (*this)(i, 1) * x(1)) + (*this)(i, 2) * x(2);
    return r;
  }
  Matrix3d operator-(const Matrix3d& o) const { Matrix3d r; for (int k = 0; k < 9; ++k) r.a[size_t(k)] = a[size_t(k)] - o.a[size_t(k)]; return r; }
  Matrix3d transpose() const { Matrix3d r; for (int i = 0; i < 3; ++i) for (int j = 0; j < 3; ++j) r(i, j) = (*this)(j, i); return r; }
  double trace() const { return ((*this)(0, 0) + (*this)(1, 1)) + (*this)(2, 2); }
  double determinant() const {
    const Matrix3d& m = *this;
    return m(0, 0) * (m(1, 1) * m(2, 2) - m(1, 2) * m(2, 1)) - m(0, 1) * (m(1, 0) * m(2, 2) - m(1, 2) * m(2, 0)) +
           m(0, 2) * (m(1, 0) * m(2, 1) - m(1, 1) * m(2, 0));
  }
  double norm() const { double s = 0.0; for (double x : a) s += x * x; return std::sqrt(s); }
};

// Proper rigid motion y -> R y + t (registration.hpp:13-33).
struct RigidTransform {
  Matrix3d R = Matrix3d::Identity();
  Vector3d t = Vector3d::Zero();
  Vector3d apply(const Vector3d& y) const { return R * y + t; }
  Matrix apply_all(const Matrix& pts) const {
    if (pts.cols() != 3) throw PotError(ErrorCode::DimensionMismatch, "point cloud must be N x 3");
    Matrix out(pts.rows(), 3);
    for (long j = 0; j < pts.rows(); ++j) {
      const Vector3d q = apply(Vector3d(pts(j, 0), pts(j, 1), pts(j, 2)));
      for (int d = 0; d < 3; ++d) out(j, d) = q(d);
    }
    return out;
  }
  static RigidTransform compose(const RigidTransform& a, const RigidTransform& b) {
    RigidTransform out;
    out.R = a.R * b.R;
    out.t = a.R * b.t + a.t;
    return out;
  }
};

namespace detail {
inline std::vector<double> rows3(const Matrix& m) {  // N x 3 column-major -> row-major
  std::vector<double> o(static_cast<size_t>(3 * m.rows()));
  for (long i = 0; i < m.rows(); ++i)
    for (int d = 0; d < 3; ++d) o[size_t(3 * i + d)] = m(i, d);
  return o;
}
inline RigidTransform from_c(const double* R, const double* t) {
  RigidTransform T;
  for (int k = 0; k < 9; ++k) T.R.a[size_t(k)] = R[k];
  for (int k = 0; k < 3; ++k) T.t(k) = t[k];
  return T;
}
}  // namespace detail

// fit_rigid (registration.hpp:40-71): coupling reductions on the device.
inline RigidTransform fit_rigid(const Matrix& pi, const Matrix& x_pts, const Matrix& y_pts) {
  if (x_pts.cols() != 3 || y_pts.cols() != 3) throw PotError(ErrorCode::DimensionMismatch, "point clouds must be N x 3");
  if (pi.rows() != x_pts.rows() || pi.cols() != y_pts.rows())
    throw PotError(ErrorCode::DimensionMismatch, "coupling shape does not match the clouds");
  std::vector<double> prm(static_cast<size_t>(pi.size()));
  for (long i = 0; i < pi.rows(); ++i)
    for (long j = 0; j < pi.cols(); ++j) prm[size_t(i * pi.cols() + j)] = pi(i, j);
  const std::vector<double> x = detail::rows3(x_pts), y = detail::rows3(y_pts);
  double R[9], t[3];
  if (int rc = potgpu_fit_rigid(detail::context(), prm.data(), pi.rows(), pi.cols(), x.data(), y.data(), R, t))
    detail::rethrow(rc);
  return detail::from_c(R, t);
}

struct RegistrationConfig {  // registration.hpp:75-100
  double alpha = 0.4;
  double gamma0 = 4.4e-3;
  double anneal_rate = 0.83;
  double transform_threshold = 1e-5;
  int max_registrations = 60;
  SolverConfig solve;
  void check() const {
    if (!(alpha > 0) || !(alpha <= 1)) throw PotError(ErrorCode::InvalidArgument, "alpha must lie in (0, 1]");
    if (!(gamma0 > 0)) throw PotError(ErrorCode::InvalidArgument, "gamma0 must be positive");
    if (!(anneal_rate > 0) || !(anneal_rate < 1)) throw PotError(ErrorCode::InvalidArgument, "anneal rate must lie in (0, 1)");
    if (!(transform_threshold > 0)) throw PotError(ErrorCode::InvalidArgument, "threshold must be positive");
    if (max_registrations < 1) throw PotError(ErrorCode::InvalidArgument, "max_registrations must be >= 1");
    solve.check();
  }
};

struct RegistrationRecord {  // registration.hpp:102-109
  int round = 0;
  long inner_iterations = 0;
  long accumulated_iterations = 0;
  double cost = 0.0;
  double increment = 0.0;
  double gamma = 0.0;
};

struct RegistrationResult {  // registration.hpp:111-115
  RigidTransform transform;
  bool converged = false;
  std::vector<RegistrationRecord> rounds;
};

// register_point_clouds (registration.hpp:127-199) on the device.
inline RegistrationResult register_point_clouds(const Matrix& reference, const Matrix& moving,
                                                const RegistrationConfig& config, SolverKind kind) {
  if (reference.cols() != 3 || moving.cols() != 3) throw PotError(ErrorCode::DimensionMismatch, "point clouds must be N x 3");
  if (reference.rows() < 3 || moving.rows() < 3) throw PotError(ErrorCode::EmptyInput, "need at least 3 points per cloud");
  config.check();
  potgpu_reg_config rc{config.alpha, config.gamma0, config.anneal_rate, config.transform_threshold,
                       config.max_registrations};
  const potgpu_config sc = detail::to_cconfig(config.solve, config.solve.epsilon, config.solve.tuning_exponent_p);
  const std::vector<double> ref = detail::rows3(reference), mov = detail::rows3(moving);
  potgpu_reg_result res{};
  std::vector<potgpu_reg_record> recs(static_cast<size_t>(config.max_registrations));
  if (int rc2 = potgpu_register_point_clouds(detail::context(), int(kind), ref.data(), reference.rows(), mov.data(),
                                             moving.rows(), &rc, &sc, POTGPU_F64, &res, recs.data(),
                                             int64_t(recs.size())))
    detail::rethrow(rc2);
  RegistrationResult out;
  out.transform = detail::from_c(res.R, res.t);
  out.converged = res.converged != 0;
  for (int64_t k = 0; k < std::min<int64_t>(res.rounds, int64_t(recs.size())); ++k) {
    const potgpu_reg_record& q = recs[size_t(k)];
    out.rounds.push_back(RegistrationRecord{q.round, long(q.inner_iterations), long(q.accumulated_iterations), q.cost,
                                            q.increment, q.gamma});
  }
  return out;
}

}  // namespace pot
