// pot/pot.hpp — drop-in C++ mirror of the reference's `namespace pot` solver
// API (/root/reference/proj/include/pot/{core,dual,solvers,extend,rounding,
// synthetic}.hpp), backed by libpotgpu.so (include/potgpu.h) on a B200.
//
// Same names, argument meaning and error behaviour: a reference user replaces
// `-I proj/include` with `-I <repo>/include` and links `-lpotgpu`. Eigen is not
// required: pot::Vector / pot::Matrix are small owning dense types with the
// subset of Eigen's interface the reference API exposes (column-major Matrix,
// (i, j) indexing). Solves run on the GPU; validation, plan metrics and the
// small helpers (entropy, theta_next, rho, theory_bounds) are host code.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "../potgpu.h"

namespace pot {

// ------------------------------------------------------------- dense types --
class Vector {
 public:
  Vector() = default;
  explicit Vector(long n) : d_(static_cast<size_t>(n), 0.0) {}
  static Vector Zero(long n) { return Vector(n); }
  static Vector Constant(long n, double x) { Vector v(n); std::fill(v.d_.begin(), v.d_.end(), x); return v; }
  long size() const { return long(d_.size()); }
  double& operator()(long i) { return d_[size_t(i)]; }
  double operator()(long i) const { return d_[size_t(i)]; }
  double& operator[](long i) { return d_[size_t(i)]; }
  double operator[](long i) const { return d_[size_t(i)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double sum() const { double s = 0.0; for (double x : d_) s += x; return s; }
  double minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
  double maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
  bool allFinite() const { for (double x : d_) if (!std::isfinite(x)) return false; return true; }
  void resize(long n) { d_.resize(size_t(n)); }

 private:
  std::vector<double> d_;
};

class Matrix {  // column-major like Eigen::MatrixXd
 public:
  Matrix() = default;
  Matrix(long r, long c) : r_(r), c_(c), d_(static_cast<size_t>(r * c), 0.0) {}
  static Matrix Zero(long r, long c) { return Matrix(r, c); }
  static Matrix Constant(long r, long c, double x) { Matrix m(r, c); std::fill(m.d_.begin(), m.d_.end(), x); return m; }
  static Matrix Ones(long r, long c) { return Constant(r, c, 1.0); }
  long rows() const { return r_; }
  long cols() const { return c_; }
  long size() const { return r_ * c_; }
  double& operator()(long i, long j) { return d_[size_t(i + j * r_)]; }
  double operator()(long i, long j) const { return d_[size_t(i + j * r_)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  double sum() const { double s = 0.0; for (double x : d_) s += x; return s; }
  double maxCoeff() const { return *std::max_element(d_.begin(), d_.end()); }
  double minCoeff() const { return *std::min_element(d_.begin(), d_.end()); }
  bool allFinite() const { for (double x : d_) if (!std::isfinite(x)) return false; return true; }
  Vector rowSums() const { Vector v(r_); for (long j = 0; j < c_; ++j) for (long i = 0; i < r_; ++i) v(i) += (*this)(i, j); return v; }
  Vector colSums() const { Vector v(c_); for (long j = 0; j < c_; ++j) for (long i = 0; i < r_; ++i) v(j) += (*this)(i, j); return v; }

 private:
  long r_ = 0, c_ = 0;
  std::vector<double> d_;
};

// ------------------------------------------------------------ core.hpp --
enum class ErrorCode {  // core.hpp:21-39 (order is the C-ABI contract)
  DimensionMismatch, NegativeEntry, NonFiniteEntry, BudgetExceedsMass, Overflow, NonPositiveArgument,
  DegenerateInstance, PenaltyTooSmall, UnbalancedMarginals, ZeroEntropy, Infeasible, SizeLimitExceeded,
  ZeroMassPlan, DegenerateSvd, EmptyInput, InvalidArgument, IoFailure,
};

inline const char* error_code_name(ErrorCode code) {
  static const char* names[] = {"DimensionMismatch", "NegativeEntry", "NonFiniteEntry", "BudgetExceedsMass", "Overflow",
                                "NonPositiveArgument", "DegenerateInstance", "PenaltyTooSmall", "UnbalancedMarginals",
                                "ZeroEntropy", "Infeasible", "SizeLimitExceeded", "ZeroMassPlan", "DegenerateSvd",
                                "EmptyInput", "InvalidArgument", "IoFailure"};
  const int k = int(code);
  return k >= 0 && k < 17 ? names[k] : "Unknown";
}

class PotError : public std::runtime_error {  // core.hpp:64-74
 public:
  PotError(ErrorCode code, const std::string& message)
      : std::runtime_error(std::string(error_code_name(code)) + ": " + message), code_(code) {}
  ErrorCode code() const { return code_; }

 private:
  ErrorCode code_;
};

// Device-side failures with no reference counterpart (CUDA / NCCL errors).
class DeviceError : public std::runtime_error {
 public:
  DeviceError(int code, const std::string& m) : std::runtime_error(m), code_(code) {}
  int code() const { return code_; }

 private:
  int code_;
};

struct Instance {  // core.hpp:108-118
  Vector r;
  Vector c;
  Matrix C;
  double s = 0.0;
  long size() const { return r.size(); }
  double source_mass() const { return r.sum(); }
  double target_mass() const { return c.sum(); }
  double max_cost() const { return C.size() > 0 ? C.maxCoeff() : 0.0; }
};

inline constexpr double kBudgetSlack = 1e-12;  // core.hpp:129

struct TransportPlan {  // core.hpp:179-197
  Matrix X;
  Vector row_slack;
  Vector col_slack;
  double mass = 0.0;
};

inline double transport_cost(const Matrix& C, const Matrix& X) {  // core.hpp:199-204
  if (C.rows() != X.rows() || C.cols() != X.cols()) throw PotError(ErrorCode::DimensionMismatch, "cost/plan shape mismatch");
  double s = 0.0;
  for (long k = 0; k < C.size(); ++k) s += C.data()[k] * X.data()[k];
  return s;
}

inline double plan_feasibility_gap(const TransportPlan& p, const Instance& in) {  // core.hpp:207-219
  if (p.X.rows() != in.size() || p.X.cols() != in.size())
    throw PotError(ErrorCode::DimensionMismatch, "plan shape does not match the instance");
  const Vector rs = p.X.rowSums(), cs = p.X.colSums();
  double rg = 0.0, cg = 0.0;
  for (long i = 0; i < rs.size(); ++i) rg = std::max(rg, std::max(rs(i) - in.r(i), 0.0));
  for (long j = 0; j < cs.size(); ++j) cg = std::max(cg, std::max(cs(j) - in.c(j), 0.0));
  return std::max({rg, cg, std::fabs(p.X.sum() - in.s)});
}

enum class BlockRule { Greedy, RoundRobin };
enum class SolverKind { Aspot, FeasibleSinkhorn, TunedSinkhorn };
enum class SolveStatus { Converged, MaxIterationsExceeded, StepSizeUnderflow };

inline std::optional<SolverKind> solver_kind_from_name(const std::string& name) {  // core.hpp:234-239
  if (name == "aspot") return SolverKind::Aspot;
  if (name == "sinkhorn") return SolverKind::FeasibleSinkhorn;
  if (name == "tuned-sinkhorn") return SolverKind::TunedSinkhorn;
  return std::nullopt;
}

inline const char* solver_kind_name(SolverKind k) {
  switch (k) {
    case SolverKind::Aspot: return "aspot";
    case SolverKind::FeasibleSinkhorn: return "sinkhorn";
    case SolverKind::TunedSinkhorn: return "tuned-sinkhorn";
  }
  return "unknown";
}

inline const char* solve_status_name(SolveStatus s) {
  switch (s) {
    case SolveStatus::Converged: return "converged";
    case SolveStatus::MaxIterationsExceeded: return "max-iterations-exceeded";
    case SolveStatus::StepSizeUnderflow: return "step-size-underflow";
  }
  return "unknown";
}

struct SolverConfig {  // core.hpp:241-267
  double epsilon = 0.1;
  std::optional<double> gamma_override;
  long max_iterations = 50000;
  BlockRule block_rule = BlockRule::Greedy;
  double tuning_exponent_p = 1.0;
  bool deterministic = true;
  long log_every = 1;
  void check() const {
    if (!(epsilon > 0) || !std::isfinite(epsilon)) throw PotError(ErrorCode::InvalidArgument, "epsilon must be positive");
    if (max_iterations < 1) throw PotError(ErrorCode::InvalidArgument, "max_iterations must be >= 1");
    if (!(tuning_exponent_p >= 1)) throw PotError(ErrorCode::InvalidArgument, "tuning exponent p must be >= 1");
    if (log_every < 1) throw PotError(ErrorCode::InvalidArgument, "log_every must be >= 1");
    if (gamma_override && !(*gamma_override > 0)) throw PotError(ErrorCode::InvalidArgument, "gamma override must be positive");
  }
};

struct TraceRecord {  // core.hpp:269-275
  long t = 0;
  double error = 0.0;
  double phi = 0.0;
  std::optional<double> rounded_cost;
  double elapsed_s = 0.0;
};

struct ConvergenceTrace {
  std::vector<TraceRecord> records;
  std::string stopping_iterate;
};

// ---------------------------------------------------------- solvers.hpp --
struct TheoryBounds {  // solvers.hpp:139-144
  double R = 0.0, L = 0.0, mu_f = 0.0, iteration_bound = 0.0;
};

struct SolveResult {  // solvers.hpp:176-186
  TransportPlan plan;
  ConvergenceTrace trace;
  SolveStatus status = SolveStatus::Converged;
  long iterations = 0;
  double gamma = 0.0;
  double tolerance = 0.0;
  double final_error = 0.0;
  double wall_seconds = 0.0;
  std::optional<TheoryBounds> bounds;
};

inline double entropy(const Vector& x) {  // solvers.hpp:19-28
  for (long i = 0; i < x.size(); ++i)
    if (x(i) < 0) throw PotError(ErrorCode::NegativeEntry, "entropy requires x >= 0");
  double h = 0.0;
  for (long i = 0; i < x.size(); ++i)
    if (x(i) > 0) h -= x(i) * std::log(x(i));
  return h;
}

inline double theta_next(double theta) {  // solvers.hpp:32-37
  if (!(theta > 0) || !(theta <= 1)) throw PotError(ErrorCode::InvalidArgument, "theta must lie in (0, 1]");
  return theta * (std::sqrt(theta * theta + 4.0) - theta) / 2.0;
}

inline double rho(double a, double b) {  // dual.hpp:144-149
  if (!(a > 0) || !(b > 0)) throw PotError(ErrorCode::NonPositiveArgument, "rho requires a, b > 0");
  return b - a + a * std::log(a / b);
}

namespace detail {

inline potgpu_ctx* context() {
  // one context per thread: distinct solves may run concurrently (README.md:132-133)
  struct Holder {
    potgpu_ctx* c = nullptr;
    ~Holder() { if (c) potgpu_destroy(c); }
  };
  thread_local Holder h;
  if (!h.c) {
    if (int rc = potgpu_create(0, &h.c)) throw DeviceError(rc, potgpu_last_error());
  }
  return h.c;
}

[[noreturn]] inline void rethrow(int rc) {
  const std::string msg = potgpu_last_error();
  if (rc >= 1 && rc <= 17) throw PotError(ErrorCode(rc - 1), msg);
  throw DeviceError(rc, msg);
}

inline potgpu_config to_cconfig(const SolverConfig& config, double epsilon, double p) {
  potgpu_config cfg;
  potgpu_config_default(&cfg);
  cfg.epsilon = epsilon;
  cfg.gamma_override = config.gamma_override.value_or(0.0);
  cfg.max_iterations = config.max_iterations;
  cfg.block_rule = config.block_rule == BlockRule::Greedy ? POTGPU_GREEDY : POTGPU_ROUND_ROBIN;
  cfg.tuning_exponent_p = p;
  cfg.deterministic = config.deterministic ? 1 : 0;
  cfg.log_every = config.log_every;
  return cfg;
}

// step_cb (optional): the solve runs through the session C-ABI one accepted
// iteration at a time and step_cb(session) is called after each one.
inline SolveResult run(int kind, const Instance& in, const SolverConfig& config, double epsilon, double p,
                       const std::function<void(potgpu_session*)>& step_cb = {}) {
  config.check();
  const long n = in.size();
  potgpu_problem pr{};
  pr.n = n;
  pr.dtype = POTGPU_F64;
  pr.cost_kind = POTGPU_COST_DENSE;
  pr.C = in.C.data();
  pr.ldc = in.C.rows();
  pr.row_major = 0;  // Eigen layout
  pr.r = in.r.data();
  pr.c = in.c.data();
  pr.s = in.s;
  if (in.c.size() != n || in.C.rows() != n || in.C.cols() != n)
    throw PotError(ErrorCode::DimensionMismatch, "instance shapes differ");
  potgpu_config cfg = to_cconfig(config, epsilon, p);
  const int64_t cap = std::min<int64_t>(config.max_iterations / config.log_every + 4, 1 << 20);
  std::vector<potgpu_trace_record> trace(static_cast<size_t>(cap));
  SolveResult res;
  res.plan.X = Matrix(n, n);
  std::vector<double> Xrm(static_cast<size_t>(n * n));
  res.plan.row_slack = Vector(n);
  res.plan.col_slack = Vector(n);
  potgpu_outputs out{};
  out.X = Xrm.data();
  out.row_slack = res.plan.row_slack.data();
  out.col_slack = res.plan.col_slack.data();
  out.trace = trace.data();
  out.trace_cap = cap;
  potgpu_summary sm{};
  if (!step_cb) {
    if (int rc = potgpu_solve(context(), kind, &pr, &cfg, &sm, &out)) rethrow(rc);
  } else {
    potgpu_session* ses = nullptr;
    if (int rc = potgpu_session_begin(context(), kind, &pr, &cfg, cap, 0, &ses)) rethrow(rc);
    struct Guard { potgpu_session* s; ~Guard() { potgpu_session_destroy(s); } } guard{ses};
    while (true) {
      double ms = 0.0;
      int64_t it = 0;
      int fin = 0;
      if (int rc = potgpu_session_iterate(ses, 1, &ms, &it, &fin)) rethrow(rc);
      if (it > 0) step_cb(ses);
      if (fin) break;
    }
    if (int rc = potgpu_session_finish(ses, &sm, &out)) rethrow(rc);
  }
  for (long i = 0; i < n; ++i)
    for (long j = 0; j < n; ++j) res.plan.X(i, j) = Xrm[size_t(i * n + j)];
  res.plan.mass = sm.mass;
  res.status = SolveStatus(sm.status);
  res.iterations = sm.iterations;
  res.gamma = sm.gamma;
  res.tolerance = sm.tolerance;
  res.final_error = sm.final_error;
  res.wall_seconds = sm.wall_seconds;
  if (sm.has_bounds) res.bounds = TheoryBounds{sm.bound_R, sm.bound_L, sm.bound_mu_f, sm.iteration_bound};
  res.trace.stopping_iterate = sm.stopping_iterate;
  for (int64_t k = 0; k < std::min<int64_t>(sm.trace_len, cap); ++k) {
    TraceRecord r;
    r.t = trace[size_t(k)].t;
    r.error = trace[size_t(k)].error;
    r.phi = trace[size_t(k)].phi;
    if (!std::isnan(trace[size_t(k)].rounded_cost)) r.rounded_cost = trace[size_t(k)].rounded_cost;
    r.elapsed_s = trace[size_t(k)].elapsed_s;
    res.trace.records.push_back(r);
  }
  return res;
}

}  // namespace detail

// The AspotObserver overload is below (after the dual types).
inline SolveResult aspot_solve(const Instance& in, const SolverConfig& config) {  // solvers.hpp:265
  return detail::run(POTGPU_ASPOT, in, config, config.epsilon, config.tuning_exponent_p);
}

inline SolveResult feasible_sinkhorn_solve(const Instance& in, const SolverConfig& config) {  // solvers.hpp:516
  return detail::run(POTGPU_FEASIBLE_SINKHORN, in, config, config.epsilon, config.tuning_exponent_p);
}

inline SolveResult tuned_sinkhorn_solve(const Instance& in, double epsilon, double p,
                                        const SolverConfig& config = {}) {  // solvers.hpp:547
  if (!(epsilon > 0) || !std::isfinite(epsilon)) throw PotError(ErrorCode::InvalidArgument, "epsilon must be positive");
  if (!(p >= 1)) throw PotError(ErrorCode::InvalidArgument, "tuning exponent p must be >= 1");
  return detail::run(POTGPU_TUNED_SINKHORN, in, config, epsilon, p);
}

inline SolveResult tuned_sinkhorn_solve(const Instance& in, const SolverConfig& config) {  // solvers.hpp:586
  return tuned_sinkhorn_solve(in, config.epsilon, config.tuning_exponent_p, config);
}

inline SolveResult solve(const Instance& in, SolverKind kind, const SolverConfig& config) {  // solvers.hpp:591
  switch (kind) {
    case SolverKind::Aspot: return aspot_solve(in, config);
    case SolverKind::FeasibleSinkhorn: return feasible_sinkhorn_solve(in, config);
    case SolverKind::TunedSinkhorn: return tuned_sinkhorn_solve(in, config);
  }
  throw PotError(ErrorCode::InvalidArgument, "unknown solver kind");
}

// -------------------------------------------------------- synthetic.hpp --
inline Instance make_synthetic_instance(long n, std::uint64_t seed, double mass_r, double mass_c, double s_frac) {
  Instance in;
  in.r = Vector(n);
  in.c = Vector(n);
  std::vector<double> Crm(static_cast<size_t>(n * n));
  double s = 0.0;
  if (int rc = potgpu_make_synthetic(n, seed, mass_r, mass_c, s_frac, in.r.data(), in.c.data(), Crm.data(), &s))
    throw PotError(ErrorCode::InvalidArgument, "invalid synthetic instance parameters (rc " + std::to_string(rc) + ")");
  in.C = Matrix(n, n);
  for (long i = 0; i < n; ++i)
    for (long j = 0; j < n; ++j) in.C(i, j) = Crm[size_t(i * n + j)];
  in.s = s;
  return in;
}

inline Instance make_scaling_instance(long n, std::uint64_t seed) {  // synthetic.hpp:58-60
  return make_synthetic_instance(n, seed, 5.0, 3.0, 0.2);
}


// ------------------------------------------------- rounding.hpp / extend.hpp --
struct Violation {  // core.hpp:76-79
  ErrorCode code;
  std::string detail;
};

// Thrown by validate(); carries every violated invariant (core.hpp:82-104).
class ValidationError : public PotError {
 public:
  explicit ValidationError(std::vector<Violation> violations)
      : PotError(violations.empty() ? ErrorCode::InvalidArgument : violations.front().code, describe(violations)),
        violations_(std::move(violations)) {}
  const std::vector<Violation>& violations() const { return violations_; }

 private:
  static std::string describe(const std::vector<Violation>& vs) {
    std::string msg = "invalid instance";
    for (const auto& v : vs) {
      msg += "; ";
      msg += error_code_name(v.code);
      msg += " (" + v.detail + ")";
    }
    return msg;
  }
  std::vector<Violation> violations_;
};

inline std::vector<Violation> validation_report(const Instance& in) {  // core.hpp:131-162
  std::vector<Violation> out;
  const long n = in.r.size();
  if (n == 0) {
    out.push_back({ErrorCode::EmptyInput, "marginals are empty"});
    return out;
  }
  if (in.c.size() != n)
    out.push_back({ErrorCode::DimensionMismatch, "r has " + std::to_string(n) + " entries, c has " + std::to_string(in.c.size())});
  if (in.C.rows() != n || in.C.cols() != n)
    out.push_back({ErrorCode::DimensionMismatch, "cost matrix is " + std::to_string(in.C.rows()) + "x" +
                                                     std::to_string(in.C.cols()) + ", expected " + std::to_string(n) + "x" +
                                                     std::to_string(n)});
  if (!in.r.allFinite() || !in.c.allFinite() || !in.C.allFinite() || !std::isfinite(in.s)) {
    out.push_back({ErrorCode::NonFiniteEntry, "non-finite entry in r, c, C or s"});
  } else {
    if ((in.r.size() && in.r.minCoeff() < 0) || (in.c.size() && in.c.minCoeff() < 0))
      out.push_back({ErrorCode::NegativeEntry, "negative marginal entry"});
    if (in.C.size() > 0 && in.C.minCoeff() < 0) out.push_back({ErrorCode::NegativeEntry, "negative cost entry"});
    if (in.s < 0) out.push_back({ErrorCode::NegativeEntry, "negative budget"});
    if (in.c.size() == n && in.s > std::min(in.r.sum(), in.c.sum()) + kBudgetSlack)
      out.push_back({ErrorCode::BudgetExceedsMass, "budget " + std::to_string(in.s) + " exceeds min marginal mass " +
                                                       std::to_string(std::min(in.r.sum(), in.c.sum()))});
  }
  return out;
}

// Returns the instance unchanged when every invariant holds (core.hpp:164-169).
inline const Instance& validate(const Instance& in) {
  auto violations = validation_report(in);
  if (!violations.empty()) throw ValidationError(std::move(violations));
  return in;
}

// TransportPlan::from (core.hpp:185-197): mass and marginal slacks of X.
inline TransportPlan plan_from(Matrix X, const Instance& in) {
  TransportPlan p;
  const Vector rs = X.rowSums(), cs = X.colSums();
  p.row_slack = Vector(in.size());
  p.col_slack = Vector(in.size());
  for (long i = 0; i < in.size(); ++i) { p.row_slack(i) = in.r(i) - rs(i); p.col_slack(i) = in.c(i) - cs(i); }
  p.mass = X.sum();
  p.X = std::move(X);
  return p;
}

namespace detail {
inline std::vector<double> to_rows(const Matrix& m) {
  std::vector<double> o(static_cast<size_t>(m.size()));
  for (long i = 0; i < m.rows(); ++i)
    for (long j = 0; j < m.cols(); ++j) o[size_t(i * m.cols() + j)] = m(i, j);
  return o;
}
inline Matrix from_rows(const std::vector<double>& v, long rows, long cols) {
  Matrix m(rows, cols);
  for (long i = 0; i < rows; ++i)
    for (long j = 0; j < cols; ++j) m(i, j) = v[size_t(i * cols + j)];
  return m;
}
}  // namespace detail

// round_pot (rounding.hpp:46-77) on the device.
inline TransportPlan round_pot(const Matrix& X, const Instance& in) {
  validate(in);
  if (X.rows() != in.size() || X.cols() != in.size())
    throw PotError(ErrorCode::DimensionMismatch, "plan shape does not match the instance");
  const std::vector<double> xr = detail::to_rows(X);
  std::vector<double> out(xr.size());
  if (int rc = potgpu_round_pot(detail::context(), in.size(), xr.data(), in.r.data(), in.c.data(), in.s, out.data()))
    detail::rethrow(rc);
  return plan_from(detail::from_rows(out, X.rows(), X.cols()), in);
}

// round_balanced (rounding.hpp:14-39) on the device.
inline Matrix round_balanced(const Matrix& X, const Vector& r, const Vector& c) {
  if (X.rows() != r.size() || X.cols() != c.size()) throw PotError(ErrorCode::DimensionMismatch, "plan/marginal shape mismatch");
  const std::vector<double> xr = detail::to_rows(X);
  std::vector<double> out(xr.size());
  if (int rc = potgpu_round_balanced(detail::context(), X.rows(), X.cols(), xr.data(), r.data(), c.data(), out.data()))
    detail::rethrow(rc);
  return detail::from_rows(out, X.rows(), X.cols());
}

struct ExtendedOtInstance {  // extend.hpp:11-18
  Matrix C_ext;
  Vector r_ext;
  Vector c_ext;
  double penalty_A = 0.0;
  long original_size() const { return r_ext.size() - 1; }
};

inline ExtendedOtInstance extend(const Instance& in, double penalty_A) {  // extend.hpp:22-39
  validate(in);
  if (!(penalty_A > in.max_cost()))
    throw PotError(ErrorCode::PenaltyTooSmall, "penalty must exceed max cost " + std::to_string(in.max_cost()));
  const long n = in.size();
  ExtendedOtInstance ext;
  ext.penalty_A = penalty_A;
  ext.C_ext = Matrix::Zero(n + 1, n + 1);
  for (long j = 0; j < n; ++j)
    for (long i = 0; i < n; ++i) ext.C_ext(i, j) = in.C(i, j);
  ext.C_ext(n, n) = penalty_A;
  ext.r_ext = Vector(n + 1);
  ext.c_ext = Vector(n + 1);
  for (long i = 0; i < n; ++i) { ext.r_ext(i) = in.r(i); ext.c_ext(i) = in.c(i); }
  ext.r_ext(n) = std::max(in.c.sum() - in.s, 0.0);
  ext.c_ext(n) = std::max(in.r.sum() - in.s, 0.0);
  return ext;
}

struct BlockDecomposition {  // extend.hpp:41-46
  Matrix block;
  Vector dummy_col;
  Vector dummy_row;
  double corner = 0.0;
};

inline BlockDecomposition extract_block(const Matrix& X_ext) {  // extend.hpp:48-60
  if (X_ext.rows() != X_ext.cols() || X_ext.rows() < 2)
    throw PotError(ErrorCode::DimensionMismatch, "extended plan must be square with side >= 2");
  const long n = X_ext.rows() - 1;
  BlockDecomposition out;
  out.block = Matrix(n, n);
  out.dummy_col = Vector(n);
  out.dummy_row = Vector(n);
  for (long j = 0; j < n; ++j)
    for (long i = 0; i < n; ++i) out.block(i, j) = X_ext(i, j);
  for (long i = 0; i < n; ++i) { out.dummy_col(i) = X_ext(i, n); out.dummy_row(i) = X_ext(n, i); }
  out.corner = X_ext(n, n);
  return out;
}


// ---------------------------------------------------------------- dual.hpp --
struct DualPoint {  // dual.hpp:15-31
  Vector u;
  Vector v;
  double w = 0.0;
  static DualPoint zero(long n) { return DualPoint{Vector::Zero(n), Vector::Zero(n), 0.0}; }
  bool all_finite() const { return u.allFinite() && v.allFinite() && std::isfinite(w); }
};

inline DualPoint operator*(double a, const DualPoint& z) {  // dual.hpp:33-43
  DualPoint o{Vector(z.u.size()), Vector(z.v.size()), a * z.w};
  for (long i = 0; i < z.u.size(); ++i) o.u(i) = a * z.u(i);
  for (long i = 0; i < z.v.size(); ++i) o.v(i) = a * z.v(i);
  return o;
}
inline DualPoint operator+(const DualPoint& a, const DualPoint& b) {
  DualPoint o{Vector(a.u.size()), Vector(a.v.size()), a.w + b.w};
  for (long i = 0; i < a.u.size(); ++i) o.u(i) = a.u(i) + b.u(i);
  for (long i = 0; i < a.v.size(); ++i) o.v(i) = a.v(i) + b.v(i);
  return o;
}
inline DualPoint operator-(const DualPoint& a, const DualPoint& b) {
  DualPoint o{Vector(a.u.size()), Vector(a.v.size()), a.w - b.w};
  for (long i = 0; i < a.u.size(); ++i) o.u(i) = a.u(i) - b.u(i);
  for (long i = 0; i < a.v.size(); ++i) o.v(i) = a.v(i) - b.v(i);
  return o;
}

inline constexpr double kMaxExponent = 700.0;  // dual.hpp:47

// dual.hpp:52-75. logK is materialised on the host like the reference's
// member; the reductions run on the device from C.
struct EntropicContext {
  double gamma = 0.0;
  Matrix logK;
  Vector r;
  Vector c;
  double s = 0.0;
  Matrix C;  // kept for the device evaluations
  EntropicContext(const Matrix& C_, double gamma_, Vector r_, Vector c_, double s_)
      : gamma(gamma_), r(std::move(r_)), c(std::move(c_)), s(s_), C(C_) {
    if (!(gamma > 0) || !std::isfinite(gamma)) throw PotError(ErrorCode::InvalidArgument, "gamma must be positive");
    if (C.rows() != r.size() || C.cols() != c.size())
      throw PotError(ErrorCode::DimensionMismatch, "cost/marginal shape mismatch");
    logK = Matrix(C.rows(), C.cols());
    for (long k = 0; k < C.size(); ++k) logK.data()[k] = -C.data()[k] / gamma;
  }
  static EntropicContext from_instance(const Instance& in, double gamma) {
    return EntropicContext(in.C, gamma, in.r, in.c, in.s);
  }
  long size() const { return r.size(); }
};

namespace detail {
inline void check_dual_shape(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:79-83
  if (z.u.size() != ctx.size() || z.v.size() != ctx.size())
    throw PotError(ErrorCode::DimensionMismatch, "dual point shape mismatch");
}
inline void check_exp_range(double max_exponent, const char* what) {  // dual.hpp:85-90
  if (!(max_exponent <= kMaxExponent))
    throw PotError(ErrorCode::Overflow, std::string(what) + " exponent exceeds representable range");
}
inline double eexp(double x) {  // Eigen's packet exp (clamped argument)
  if (std::isnan(x) || x == std::numeric_limits<double>::infinity()) return std::exp(x);
  return std::exp(std::min(std::max(x, -709.784), 709.784));
}
inline potgpu_problem dense_problem(const EntropicContext& ctx) {
  potgpu_problem pr{};
  pr.n = ctx.size();
  pr.dtype = POTGPU_F64;
  pr.cost_kind = POTGPU_COST_DENSE;
  pr.C = ctx.C.data();
  pr.ldc = ctx.C.rows();
  pr.row_major = 0;
  pr.r = ctx.r.data();
  pr.c = ctx.c.data();
  pr.s = ctx.s;
  return pr;
}
inline double max_of(const Vector& x) {
  double m = -std::numeric_limits<double>::infinity();
  for (long i = 0; i < x.size(); ++i) { if (std::isnan(x(i))) return x(i); m = std::max(m, x(i)); }
  return m;
}
// B 1, B^T 1, B.sum() at z on the device (potgpu_dual_eval).
struct BSums { Vector row, col; double total = 0.0; };
inline BSums b_sums(const EntropicContext& ctx, const DualPoint& z) {
  const potgpu_problem pr = dense_problem(ctx);
  BSums b{Vector(ctx.size()), Vector(ctx.size()), 0.0};
  double sc[6];
  if (int rc = potgpu_dual_eval(context(), &pr, ctx.gamma, z.u.data(), z.v.data(), z.w, b.row.data(), b.col.data(), sc))
    rethrow(rc);
  b.total = sc[0];
  return b;
}
inline Matrix dual_matrix(const EntropicContext& ctx, const DualPoint& z, int which) {
  const potgpu_problem pr = dense_problem(ctx);
  const long n = ctx.size();
  std::vector<double> o(static_cast<size_t>(n * n));
  if (int rc = potgpu_dual_matrix(context(), &pr, ctx.gamma, z.u.data(), z.v.data(), z.w, which, o.data())) rethrow(rc);
  return from_rows(o, n, n);
}
inline Matrix exponent_matrix(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:92-99
  check_dual_shape(ctx, z);
  return dual_matrix(ctx, z, 0);
}
inline double rho_limit(double a, double b);
}  // namespace detail

inline Matrix b_matrix(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:103-109
  detail::check_dual_shape(ctx, z);
  return detail::dual_matrix(ctx, z, 1);
}

inline DualPoint dual_gradient(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:122-133
  detail::check_dual_shape(ctx, z);
  detail::check_exp_range(detail::max_of(z.u), "exp(u)");
  detail::check_exp_range(detail::max_of(z.v), "exp(v)");
  const detail::BSums b = detail::b_sums(ctx, z);
  DualPoint g{Vector(ctx.size()), Vector(ctx.size()), b.total - ctx.s};
  for (long i = 0; i < ctx.size(); ++i) {
    g.u(i) = (b.row(i) + detail::eexp(z.u(i))) - ctx.r(i);
    g.v(i) = (b.col(i) + detail::eexp(z.v(i))) - ctx.c(i);
  }
  return g;
}

inline double dual_objective(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:111-120
  detail::check_dual_shape(ctx, z);
  detail::check_exp_range(detail::max_of(z.u), "exp(u)");
  detail::check_exp_range(detail::max_of(z.v), "exp(v)");
  const detail::BSums b = detail::b_sums(ctx, z);
  double eu = 0.0, ev = 0.0, ur = 0.0, vc = 0.0;
  for (long i = 0; i < ctx.size(); ++i) {
    eu += detail::eexp(z.u(i));
    ev += detail::eexp(z.v(i));
    ur += z.u(i) * ctx.r(i);
    vc += z.v(i) * ctx.c(i);
  }
  return ((((b.total + eu) + ev) - ur) - vc) - z.w * ctx.s;
}

inline double feasibility_error(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:135-139
  const DualPoint g = dual_gradient(ctx, z);
  double e = 0.0;
  for (long i = 0; i < g.u.size(); ++i) e += std::fabs(g.u(i));
  for (long i = 0; i < g.v.size(); ++i) e += std::fabs(g.v(i));
  return e + std::fabs(g.w);
}

namespace detail {
inline double rho_limit(double a, double b) {  // dual.hpp:150-158
  if (!(a > 0)) return b;
  if (!(b > 0)) return std::numeric_limits<double>::infinity();
  return rho(a, b);
}
}  // namespace detail

// greenkhorn_step (solvers.hpp:43-89): the sums on the device, the block
// choice and update on the host in the reference's order.
inline DualPoint greenkhorn_step(const EntropicContext& ctx, const DualPoint& z, BlockRule rule, long t) {
  detail::check_dual_shape(ctx, z);
  detail::check_exp_range(detail::max_of(z.u), "exp(u)");
  detail::check_exp_range(detail::max_of(z.v), "exp(v)");
  const detail::BSums b = detail::b_sums(ctx, z);
  const long n = ctx.size();
  Vector row(n), col(n);
  for (long i = 0; i < n; ++i) {
    row(i) = b.row(i) + detail::eexp(z.u(i));
    col(i) = b.col(i) + detail::eexp(z.v(i));
  }
  int block = 0;
  if (rule == BlockRule::RoundRobin) {
    block = int(t % 3);
  } else {
    double su = 0.0, sv = 0.0;
    for (long i = 0; i < n; ++i) {
      su += detail::rho_limit(ctx.r(i), row(i));
      sv += detail::rho_limit(ctx.c(i), col(i));
    }
    const double sw = detail::rho_limit(ctx.s, b.total);
    double best = su;
    if (sv > best) { block = 1; best = sv; }
    if (sw > best) block = 2;
  }
  DualPoint out = z;
  if (block == 0) for (long i = 0; i < n; ++i) out.u(i) += std::log(ctx.r(i)) - std::log(row(i));
  else if (block == 1) for (long i = 0; i < n; ++i) out.v(i) += std::log(ctx.c(i)) - std::log(col(i));
  else out.w += std::log(ctx.s) - std::log(b.total);
  if (!out.all_finite()) throw PotError(ErrorCode::Overflow, "block update left the exp range");
  return out;
}

struct AspotSetup {  // solvers.hpp:94-99
  double gamma = 0.0;
  double eps_tilde = 0.0;
  Vector mixed_r;
  Vector mixed_c;
};

inline AspotSetup aspot_setup(const Instance& in, double epsilon) {  // solvers.hpp:100-133
  validate(in);
  if (!(epsilon > 0) || !std::isfinite(epsilon)) throw PotError(ErrorCode::InvalidArgument, "epsilon must be positive");
  const long n = in.size();
  if (n < 2) throw PotError(ErrorCode::DegenerateInstance, "accelerated setup needs n >= 2 (log n vanishes)");
  AspotSetup st;
  st.gamma = epsilon / (4.0 * std::log(double(n)));
  const double cmax = in.max_cost();
  st.eps_tilde = cmax > 0 ? epsilon / (8.0 * cmax) : std::numeric_limits<double>::infinity();
  const double sr = in.r.sum(), sc = in.c.sum();
  if (sr > 1) st.eps_tilde = std::min(st.eps_tilde, 8.0 * (sr - in.s) / (sr - 1.0));
  if (sc > 1) st.eps_tilde = std::min(st.eps_tilde, 8.0 * (sc - in.s) / (sc - 1.0));
  if (!(st.gamma > 0) || !std::isfinite(st.gamma)) throw PotError(ErrorCode::DegenerateInstance, "derived gamma is not positive");
  if (!(st.eps_tilde > 0))
    throw PotError(ErrorCode::DegenerateInstance, "stopping tolerance collapsed to zero (budget equals mass)");
  const double lambda = std::min(st.eps_tilde / 8.0, 0.5);
  st.mixed_r = Vector(n);
  st.mixed_c = Vector(n);
  for (long i = 0; i < n; ++i) {
    st.mixed_r(i) = (1.0 - lambda) * in.r(i) + lambda / double(n);
    st.mixed_c(i) = (1.0 - lambda) * in.c(i) + lambda / double(n);
  }
  return st;
}

// Per-iteration snapshot of the accelerated solver (solvers.hpp:188-202);
// references valid only inside the callback.
struct AspotIterate {
  long t = 0;
  double theta = 0.0;
  double error = 0.0;
  const EntropicContext& ctx;
  const DualPoint& z_grave;
  const DualPoint& z_hat;
  const DualPoint& z_best;
  const DualPoint& z_check;
  double phi_hat = 0.0;
  double phi_best = 0.0;
  double phi_check = 0.0;
};

using AspotObserver = std::function<void(const AspotIterate&)>;

// aspot_solve with an observer (solvers.hpp:265-266, 364-367): the device
// loop advances one accepted iteration at a time and the four points are
// copied to the host for the callback (a diagnostic slow path).
inline SolveResult aspot_solve(const Instance& in, const SolverConfig& config, const AspotObserver& observer) {
  if (!observer) return aspot_solve(in, config);
  config.check();
  validate(in);
  if (in.s == 0 || in.size() < 2) return aspot_solve(in, config);  // trivial / degenerate: no iterations
  const AspotSetup st = aspot_setup(in, config.epsilon);
  const EntropicContext ectx(in.C, config.gamma_override.value_or(st.gamma), st.mixed_r, st.mixed_c, in.s);
  const long n = in.size();
  return detail::run(POTGPU_ASPOT, in, config, config.epsilon, config.tuning_exponent_p, [&](potgpu_session* ses) {
    DualPoint pts[4];
    double sc[6];
    for (int k = 0; k < 4; ++k) {
      pts[k] = DualPoint{Vector(n), Vector(n), 0.0};
      if (int rc = potgpu_session_read_state(ses, k, pts[k].u.data(), pts[k].v.data(), &pts[k].w, sc)) detail::rethrow(rc);
    }
    observer(AspotIterate{long(sc[0]), sc[1], sc[2], ectx, pts[3], pts[2], pts[0], pts[1], sc[3], sc[4], sc[5]});
  });
}

}  // namespace pot
