// pot_oracle.hpp — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
//
// A plain C++20 restatement of the reference's entropic-POT hot path
// (/root/reference/proj/include/pot/{core,dual,solvers,extend,rounding,
// synthetic}.hpp), used ONLY by tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py, and only as the checker.
// The product (paper_2601_17196_b200/libpotgpu.so) never links or calls it.
//
// The reference itself cannot be built in this image (it needs Eigen >= 3.3,
// which is absent — see DESIGN.md §Oracle), so this restatement is the parity
// anchor. It is pinned against every known-answer test the reference's own
// suites hold for this path (tests/test_oracle_kat.py runs oracle/kat_main.cpp,
// a GTest-free port of proj/tests/test_{dual,solvers,extend_rounding,core}.cpp
// hand values). There are no golden vectors in the reference.
//
// Deviations from the reference, all arithmetic-order only:
//   * Eigen's vectorised reductions are replaced by Neumaier-compensated
//     sums (deterministic, <= 1 ulp-class error), so the oracle is closer to
//     the exact sums than either Eigen or the GPU tree reductions.
//   * B(z) is streamed instead of materialised; the values and the
//     exponent association ((logK + u_i) + v_j) + w are identical
//     (dual.hpp:93-99).
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <thread>

namespace pot_oracle {

// ---------------------------------------------------------------------------
// core.hpp:21-39 — the enum order is part of the C-ABI error contract.
enum class ErrorCode {
  DimensionMismatch, NegativeEntry, NonFiniteEntry, BudgetExceedsMass, Overflow,
  NonPositiveArgument, DegenerateInstance, PenaltyTooSmall, UnbalancedMarginals,
  ZeroEntropy, Infeasible, SizeLimitExceeded, ZeroMassPlan, DegenerateSvd,
  EmptyInput, InvalidArgument, IoFailure,
};

struct PotError : std::runtime_error {
  ErrorCode code;
  PotError(ErrorCode c, const std::string& m) : std::runtime_error(m), code(c) {}
};

using Vec = std::vector<double>;

// Column-major dense matrix, (i, j) indexing like Eigen::MatrixXd.
struct Mat {
  long rows = 0, cols = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(long r, long c, double fill = 0.0) : rows(r), cols(c), a(size_t(r) * size_t(c), fill) {}
  double& operator()(long i, long j) { return a[size_t(i) + size_t(j) * size_t(rows)]; }
  double operator()(long i, long j) const { return a[size_t(i) + size_t(j) * size_t(rows)]; }
  long size() const { return rows * cols; }
};

// Neumaier compensated accumulator (stands in for Eigen's redux; see header).
struct KSum {
  double s = 0.0, c = 0.0;
  inline void add(double x) {
    const double t = s + x;
    if (std::fabs(s) >= std::fabs(x)) c += (s - t) + x; else c += (x - t) + s;
    s = t;
  }
  double get() const { return s + c; }
};

inline double vsum(const Vec& x) { KSum k; for (double e : x) k.add(e); return k.get(); }
inline double vdot(const Vec& x, const Vec& y) { KSum k; for (size_t i = 0; i < x.size(); ++i) k.add(x[i] * y[i]); return k.get(); }
inline double vl1(const Vec& x) { KSum k; for (double e : x) k.add(std::fabs(e)); return k.get(); }
inline double vmax(const Vec& x) { double m = -std::numeric_limits<double>::infinity(); for (double e : x) { if (e != e) return e; if (e > m) m = e; } return m; }
inline double vmin(const Vec& x) { double m = std::numeric_limits<double>::infinity(); for (double e : x) m = std::min(m, e); return m; }
inline bool vfinite(const Vec& x) { for (double e : x) if (!std::isfinite(e)) return false; return true; }
inline double msum(const Mat& m) { KSum k; for (double e : m.a) k.add(e); return k.get(); }
inline Vec mrowsum(const Mat& m) {
  std::vector<KSum> acc(size_t(m.rows));
  for (long j = 0; j < m.cols; ++j) for (long i = 0; i < m.rows; ++i) acc[size_t(i)].add(m(i, j));
  Vec out(size_t(m.rows)); for (long i = 0; i < m.rows; ++i) out[size_t(i)] = acc[size_t(i)].get();
  return out;
}
inline Vec mcolsum(const Mat& m) {
  Vec out(size_t(m.cols));
  for (long j = 0; j < m.cols; ++j) { KSum k; for (long i = 0; i < m.rows; ++i) k.add(m(i, j)); out[size_t(j)] = k.get(); }
  return out;
}
inline double mmax(const Mat& m) { double x = -std::numeric_limits<double>::infinity(); for (double e : m.a) { if (e != e) return e; if (e > x) x = e; } return x; }

// ---------------------------------------------------------------------------
// Instance / validation — core.hpp:108-176.
struct Instance {
  Vec r, c;
  Mat C;
  double s = 0.0;
  // Oracle-only: points mode (C never materialised, config C4). The cost
  // is then C_ij = scale*|x_i - y_j|^2 with known max `cmax_hint`.
  bool points_mode = false;
  double cmax_hint = 0.0;
  long size() const { return long(r.size()); }
  double source_mass() const { return vsum(r); }
  double target_mass() const { return vsum(c); }
  double max_cost() const { return points_mode ? cmax_hint : (C.size() > 0 ? mmax(C) : 0.0); }
};

inline constexpr double kBudgetSlack = 1e-12;  // core.hpp:129

struct Violation { ErrorCode code; std::string detail; };

inline std::vector<Violation> validation_report(const Instance& in) {  // core.hpp:131-169
  std::vector<Violation> out;
  const long n = long(in.r.size());
  if (n == 0) { out.push_back({ErrorCode::EmptyInput, "marginals are empty"}); return out; }
  if (long(in.c.size()) != n) out.push_back({ErrorCode::DimensionMismatch, "r/c size"});
  if (!in.points_mode && (in.C.rows != n || in.C.cols != n)) out.push_back({ErrorCode::DimensionMismatch, "cost shape"});
  bool finite = vfinite(in.r) && vfinite(in.c) && std::isfinite(in.s);
  for (double e : in.C.a) if (!std::isfinite(e)) { finite = false; break; }
  if (!finite) {
    out.push_back({ErrorCode::NonFiniteEntry, "non-finite entry in r, c, C or s"});
  } else {
    bool neg = false;
    for (double e : in.r) neg |= e < 0;
    for (double e : in.c) neg |= e < 0;
    if (neg) out.push_back({ErrorCode::NegativeEntry, "negative marginal entry"});
    bool negc = false;
    for (double e : in.C.a) negc |= e < 0;
    if (in.C.size() > 0 && negc) out.push_back({ErrorCode::NegativeEntry, "negative cost entry"});
    if (in.s < 0) out.push_back({ErrorCode::NegativeEntry, "negative budget"});
    if (long(in.c.size()) == n && in.s > std::min(vsum(in.r), vsum(in.c)) + kBudgetSlack)
      out.push_back({ErrorCode::BudgetExceedsMass, "budget exceeds min marginal mass"});
  }
  return out;
}

inline const Instance& validate(const Instance& in) {  // core.hpp:172-176
  auto v = validation_report(in);
  if (!v.empty()) throw PotError(v.front().code, "invalid instance: " + v.front().detail);
  return in;
}

struct TransportPlan {  // core.hpp:179-197
  Mat X;
  Vec row_slack, col_slack;
  double mass = 0.0;
  static TransportPlan from(Mat X, const Instance& in) {
    if (X.rows != in.size() || X.cols != in.size())
      throw PotError(ErrorCode::DimensionMismatch, "plan shape does not match the instance");
    TransportPlan p;
    const Vec rs = mrowsum(X), cs = mcolsum(X);
    p.row_slack.resize(rs.size()); p.col_slack.resize(cs.size());
    for (size_t i = 0; i < rs.size(); ++i) p.row_slack[i] = in.r[i] - rs[i];
    for (size_t j = 0; j < cs.size(); ++j) p.col_slack[j] = in.c[j] - cs[j];
    p.mass = msum(X);
    p.X = std::move(X);
    return p;
  }
};

inline double transport_cost(const Mat& C, const Mat& X) {  // core.hpp:199-204
  if (C.rows != X.rows || C.cols != X.cols) throw PotError(ErrorCode::DimensionMismatch, "cost/plan shape mismatch");
  KSum k; for (size_t e = 0; e < C.a.size(); ++e) k.add(C.a[e] * X.a[e]); return k.get();
}

inline double plan_feasibility_gap(const TransportPlan& p, const Instance& in) {  // core.hpp:207-219
  if (p.X.rows != in.size() || p.X.cols != in.size()) throw PotError(ErrorCode::DimensionMismatch, "plan shape");
  const Vec rs = mrowsum(p.X), cs = mcolsum(p.X);
  double rg = 0.0, cg = 0.0;
  for (size_t i = 0; i < rs.size(); ++i) rg = std::max(rg, std::max(rs[i] - in.r[i], 0.0));
  for (size_t j = 0; j < cs.size(); ++j) cg = std::max(cg, std::max(cs[j] - in.c[j], 0.0));
  return std::max({rg, cg, std::fabs(msum(p.X) - in.s)});
}

enum class BlockRule { Greedy = 0, RoundRobin = 1 };
enum class SolverKind { Aspot = 0, FeasibleSinkhorn = 1, TunedSinkhorn = 2 };
enum class SolveStatus { Converged = 0, MaxIterationsExceeded = 1, StepSizeUnderflow = 2 };

struct SolverConfig {  // core.hpp:241-267
  double epsilon = 0.1;
  std::optional<double> gamma_override;
  long max_iterations = 50000;
  BlockRule block_rule = BlockRule::Greedy;
  double tuning_exponent_p = 1.0;
  bool deterministic = true;
  long log_every = 1;
  bool record_rounded_cost = true;  // oracle-only switch: skip round_pot in trace records
  void check() const {
    if (!(epsilon > 0) || !std::isfinite(epsilon)) throw PotError(ErrorCode::InvalidArgument, "epsilon must be positive");
    if (max_iterations < 1) throw PotError(ErrorCode::InvalidArgument, "max_iterations must be >= 1");
    if (!(tuning_exponent_p >= 1)) throw PotError(ErrorCode::InvalidArgument, "tuning exponent p must be >= 1");
    if (log_every < 1) throw PotError(ErrorCode::InvalidArgument, "log_every must be >= 1");
    if (gamma_override && !(*gamma_override > 0)) throw PotError(ErrorCode::InvalidArgument, "gamma override must be positive");
  }
};

struct TraceRecord { long t = 0; double error = 0.0, phi = 0.0; std::optional<double> rounded_cost; double elapsed_s = 0.0; };
struct ConvergenceTrace { std::vector<TraceRecord> records; std::string stopping_iterate; };

// ---------------------------------------------------------------------------
// dual.hpp:15-159
struct DualPoint {
  Vec u, v;
  double w = 0.0;
  static DualPoint zero(long n) { DualPoint z; z.u.assign(size_t(n), 0.0); z.v.assign(size_t(n), 0.0); return z; }
  bool all_finite() const { return vfinite(u) && vfinite(v) && std::isfinite(w); }
};
inline DualPoint operator*(double a, const DualPoint& z) {
  DualPoint o; o.u.resize(z.u.size()); o.v.resize(z.v.size());
  for (size_t i = 0; i < z.u.size(); ++i) o.u[i] = a * z.u[i];
  for (size_t i = 0; i < z.v.size(); ++i) o.v[i] = a * z.v[i];
  o.w = a * z.w; return o;
}
inline DualPoint operator+(const DualPoint& a, const DualPoint& b) {
  DualPoint o; o.u.resize(a.u.size()); o.v.resize(a.v.size());
  for (size_t i = 0; i < a.u.size(); ++i) o.u[i] = a.u[i] + b.u[i];
  for (size_t i = 0; i < a.v.size(); ++i) o.v[i] = a.v[i] + b.v[i];
  o.w = a.w + b.w; return o;
}
inline DualPoint operator-(const DualPoint& a, const DualPoint& b) {
  DualPoint o; o.u.resize(a.u.size()); o.v.resize(a.v.size());
  for (size_t i = 0; i < a.u.size(); ++i) o.u[i] = a.u[i] - b.u[i];
  for (size_t i = 0; i < a.v.size(); ++i) o.v[i] = a.v[i] - b.v[i];
  o.w = a.w - b.w; return o;
}

inline constexpr double kMaxExponent = 700.0;  // dual.hpp:47

// Coefficient-wise exp as the reference evaluates it. Every exp on the path
// is an Eigen array expression (dual.hpp:108, 117, 129-130; solvers.hpp:49-51,
// 225-226, 400, 430), which Eigen 3.4 evaluates with its packet pexp: the
// argument is clamped to [-709.784, 709.784] before the polynomial and the
// result is max(result, x) (so NaN/+inf propagate). Consequence that the
// reference's own tests rely on (test_solvers.cpp:292-303): exp of a very
// negative exponent is ~5.6e-309, never 0, so B sums never vanish exactly.
inline constexpr double kExpLo = -709.784;
inline constexpr double kExpHi = 709.784;
inline double eexp(double x) {
  if (x != x) return x;
  if (x == std::numeric_limits<double>::infinity()) return x;
  return std::exp(std::min(std::max(x, kExpLo), kExpHi));
}

// Source of logK_ij = -C_ij / gamma. Dense: the reference materialises it
// (dual.hpp:67). Points: the same value recomputed per entry from fp64
// coordinates (C_ij = scale * |x_i - y_j|^2), for sizes where a dense copy
// does not fit host RAM (config C4).
struct LogK {
  long n = 0;
  double gamma = 0.0;
  Mat dense;                       // column-major -C/gamma, when materialised
  const double* X = nullptr;       // points mode: n x d row-major
  const double* Y = nullptr;
  int d = 0;
  double scale = 1.0;
  bool points() const { return X != nullptr; }
  inline double cost(long i, long j) const {
    double acc = 0.0;
    for (int k = 0; k < d; ++k) { const double t = X[i * d + k] - Y[j * d + k]; acc += t * t; }
    return acc * scale;
  }
  inline double at(long i, long j) const { return points() ? -cost(i, j) / gamma : dense(i, j); }
};

struct EntropicContext {  // dual.hpp:52-75
  double gamma = 0.0;
  LogK logK;
  Vec r, c;
  double s = 0.0;
  EntropicContext() = default;
  EntropicContext(const Mat& C, double g, Vec r_, Vec c_, double s_) : gamma(g), r(std::move(r_)), c(std::move(c_)), s(s_) {
    if (!(gamma > 0) || !std::isfinite(gamma)) throw PotError(ErrorCode::InvalidArgument, "gamma must be positive");
    if (C.rows != long(r.size()) || C.cols != long(c.size())) throw PotError(ErrorCode::DimensionMismatch, "cost/marginal shape mismatch");
    logK.n = C.rows; logK.gamma = gamma;
    logK.dense = Mat(C.rows, C.cols);
    for (size_t e = 0; e < C.a.size(); ++e) logK.dense.a[e] = -C.a[e] / gamma;
  }
  long size() const { return long(r.size()); }
};

inline void check_exp_range(double m, const char* what) {  // dual.hpp:85-90
  if (!(m <= kMaxExponent)) throw PotError(ErrorCode::Overflow, std::string(what) + " exponent exceeds representable range");
}

// One streamed pass over B(z) = exp(((logK + u_i) + v_j) + w): the
// reductions every caller of b_matrix takes (dual.hpp:104-109, 127-131;
// solvers.hpp:46-52, 224-232). Throws Overflow exactly when
// b_matrix's maxCoeff check would (NaN included).
struct BSums { Vec row, col; double total = 0.0; double max_e = 0.0; };

// Host threads for the oracle's n^2 passes: 1 (default) is the reference's
// single-threaded semantics used by every parity test; >1 is only for the
// CPU-baseline timing (bench.py), splitting columns into contiguous chunks.
inline int& oracle_threads() { static int t = 1; return t; }

// f(k) for k in [0, count) on oracle_threads() host threads (contiguous
// chunks). Every index is computed independently, so results do not depend
// on the thread count.
template <class F>
inline void parallel_for(long count, F f) {
  const int T = std::max(1, std::min<int>(oracle_threads(), int(std::max<long>(count, 1))));
  if (T == 1) { for (long k = 0; k < count; ++k) f(k); return; }
  std::vector<std::thread> pool;
  for (int t = 0; t < T; ++t)
    pool.emplace_back([&, t] { for (long k = count * t / T; k < count * (t + 1) / T; ++k) f(k); });
  for (auto& th : pool) th.join();
}

// Row i's sum runs over j in order, column j's over i in order, the total
// is the compensated sum of the column sums: the same bits for any number of
// oracle threads (the threaded form recomputes the exponentials per pass).
inline BSums sweep(const EntropicContext& ctx, const DualPoint& z, bool want_rows = true, bool want_cols = true) {
  (void)want_rows; (void)want_cols;
  const long n = ctx.size();
  BSums out;
  out.row.assign(static_cast<size_t>(n), 0.0);
  out.col.assign(static_cast<size_t>(n), 0.0);
  const auto expo = [&](long i, long j) { return ((ctx.logK.at(i, j) + z.u[size_t(i)]) + z.v[size_t(j)]) + z.w; };
  double mx = -std::numeric_limits<double>::infinity();
  bool nan = false;
  if (oracle_threads() <= 1) {
    std::vector<KSum> racc(static_cast<size_t>(n));
    for (long j = 0; j < n; ++j) {
      KSum cacc;
      for (long i = 0; i < n; ++i) {
        const double e = expo(i, j);
        if (e != e) nan = true; else if (e > mx) mx = e;
        const double b = eexp(e);
        racc[size_t(i)].add(b);
        cacc.add(b);
      }
      out.col[size_t(j)] = cacc.get();
    }
    for (long i = 0; i < n; ++i) out.row[size_t(i)] = racc[size_t(i)].get();
  } else {
    std::vector<double> cmx(static_cast<size_t>(n), -std::numeric_limits<double>::infinity());
    std::vector<char> cnan(static_cast<size_t>(n), 0);
    parallel_for(n, [&](long i) {
      KSum r; for (long j = 0; j < n; ++j) r.add(eexp(expo(i, j)));
      out.row[size_t(i)] = r.get();
    });
    parallel_for(n, [&](long j) {
      KSum c; double m = -std::numeric_limits<double>::infinity(); char nn = 0;
      for (long i = 0; i < n; ++i) { const double e = expo(i, j); if (e != e) nn = 1; else if (e > m) m = e; c.add(eexp(e)); }
      out.col[size_t(j)] = c.get(); cmx[size_t(j)] = m; cnan[size_t(j)] = nn;
    });
    for (long j = 0; j < n; ++j) { mx = std::max(mx, cmx[size_t(j)]); nan = nan || cnan[size_t(j)]; }
  }
  out.max_e = nan ? std::numeric_limits<double>::quiet_NaN() : mx;
  check_exp_range(out.max_e, "B(z)");
  out.total = vsum(out.col);
  return out;
}

inline Mat b_matrix(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:104-109
  const long n = ctx.size();
  Mat M(n, n);
  for (long j = 0; j < n; ++j) for (long i = 0; i < n; ++i) M(i, j) = ((ctx.logK.at(i, j) + z.u[size_t(i)]) + z.v[size_t(j)]) + z.w;
  check_exp_range(mmax(M), "B(z)");
  for (double& e : M.a) e = eexp(e);
  return M;
}

inline double sum_exp(const Vec& x) { KSum k; for (double e : x) k.add(eexp(e)); return k.get(); }

inline double phi_from(const EntropicContext& ctx, const DualPoint& z, double btotal) {
  // dual.hpp:117-118 / solvers.hpp:228-229
  return btotal + sum_exp(z.u) + sum_exp(z.v) - vdot(z.u, ctx.r) - vdot(z.v, ctx.c) - z.w * ctx.s;
}

inline double dual_objective(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:112-119
  check_exp_range(vmax(z.u), "exp(u)");
  check_exp_range(vmax(z.v), "exp(v)");
  const BSums b = sweep(ctx, z, false, false);
  return phi_from(ctx, z, b.total);
}

inline DualPoint grad_from(const EntropicContext& ctx, const DualPoint& z, const BSums& b) {  // dual.hpp:129-131
  DualPoint g; const size_t n = z.u.size();
  g.u.resize(n); g.v.resize(n);
  for (size_t i = 0; i < n; ++i) g.u[i] = (b.row[i] + eexp(z.u[i])) - ctx.r[i];
  for (size_t j = 0; j < n; ++j) g.v[j] = (b.col[j] + eexp(z.v[j])) - ctx.c[j];
  g.w = b.total - ctx.s;
  return g;
}

inline DualPoint dual_gradient(const EntropicContext& ctx, const DualPoint& z) {  // dual.hpp:123-133
  check_exp_range(vmax(z.u), "exp(u)");
  check_exp_range(vmax(z.v), "exp(v)");
  return grad_from(ctx, z, sweep(ctx, z));
}

inline double grad_l1(const DualPoint& g) { return vl1(g.u) + vl1(g.v) + std::fabs(g.w); }  // dual.hpp:138-141
inline double feasibility_error(const EntropicContext& ctx, const DualPoint& z) { return grad_l1(dual_gradient(ctx, z)); }

inline double rho(double a, double b) {  // dual.hpp:144-149
  if (!(a > 0) || !(b > 0)) throw PotError(ErrorCode::NonPositiveArgument, "rho requires a, b > 0");
  return b - a + a * std::log(a / b);
}
inline double rho_limit(double a, double b) {  // dual.hpp:155-159
  if (!(a > 0)) return b;
  if (!(b > 0)) return std::numeric_limits<double>::infinity();
  return rho(a, b);
}

// ---------------------------------------------------------------------------
// solvers.hpp
inline double entropy(const Vec& x) {  // solvers.hpp:19-28
  for (double e : x) if (e < 0) throw PotError(ErrorCode::NegativeEntry, "entropy requires x >= 0");
  double h = 0.0;
  for (double e : x) if (e > 0) h -= e * std::log(e);
  return h;
}

inline double theta_next(double theta) {  // solvers.hpp:32-37
  if (!(theta > 0) || !(theta <= 1)) throw PotError(ErrorCode::InvalidArgument, "theta must lie in (0, 1]");
  return theta * (std::sqrt(theta * theta + 4.0) - theta) / 2.0;
}

struct GkOut { DualPoint z; int block = 0; };

// Block choice + update from the sums of B at z (solvers.hpp:54-88).
inline GkOut greenkhorn_from(const EntropicContext& ctx, const DualPoint& z, const BSums& b, BlockRule rule, long t) {
  const size_t n = z.u.size();
  Vec row(n), col(n);
  for (size_t i = 0; i < n; ++i) row[i] = b.row[i] + eexp(z.u[i]);
  for (size_t j = 0; j < n; ++j) col[j] = b.col[j] + eexp(z.v[j]);
  const double total = b.total;
  int block = 0;
  if (rule == BlockRule::RoundRobin) {
    block = int(t % 3);
  } else {
    // The reference accumulates the scores sequentially (solvers.hpp:60-63).
    double su = 0.0, sv = 0.0;
    for (size_t i = 0; i < n; ++i) { su += rho_limit(ctx.r[i], row[i]); sv += rho_limit(ctx.c[i], col[i]); }
    const double sw = rho_limit(ctx.s, total);
    double best = su;
    if (sv > best) { block = 1; best = sv; }
    if (sw > best) block = 2;
  }
  GkOut o{z, block};
  if (block == 0) for (size_t i = 0; i < n; ++i) o.z.u[i] += std::log(ctx.r[i]) - std::log(row[i]);
  else if (block == 1) for (size_t j = 0; j < n; ++j) o.z.v[j] += std::log(ctx.c[j]) - std::log(col[j]);
  else o.z.w += std::log(ctx.s) - std::log(total);
  if (!o.z.all_finite()) throw PotError(ErrorCode::Overflow, "block update left the exp range");
  return o;
}

inline GkOut greenkhorn_step_ex(const EntropicContext& ctx, const DualPoint& z, BlockRule rule, long t) {  // solvers.hpp:43-89
  const BSums b = sweep(ctx, z);
  check_exp_range(vmax(z.u), "exp(u)");
  check_exp_range(vmax(z.v), "exp(v)");
  return greenkhorn_from(ctx, z, b, rule, t);
}
inline DualPoint greenkhorn_step(const EntropicContext& ctx, const DualPoint& z, BlockRule rule, long t) {
  return greenkhorn_step_ex(ctx, z, rule, t).z;
}

struct AspotSetup { double gamma = 0.0, eps_tilde = 0.0; Vec mixed_r, mixed_c; };

inline AspotSetup aspot_setup(const Instance& in, double epsilon) {  // solvers.hpp:100-133
  validate(in);
  if (!(epsilon > 0) || !std::isfinite(epsilon)) throw PotError(ErrorCode::InvalidArgument, "epsilon must be positive");
  const long n = in.size();
  if (n < 2) throw PotError(ErrorCode::DegenerateInstance, "accelerated setup needs n >= 2 (log n vanishes)");
  AspotSetup s;
  s.gamma = epsilon / (4.0 * std::log(double(n)));
  const double cmax = in.max_cost();
  s.eps_tilde = cmax > 0 ? epsilon / (8.0 * cmax) : std::numeric_limits<double>::infinity();
  const double sr = in.source_mass(), sc = in.target_mass();
  if (sr > 1) s.eps_tilde = std::min(s.eps_tilde, 8.0 * (sr - in.s) / (sr - 1.0));
  if (sc > 1) s.eps_tilde = std::min(s.eps_tilde, 8.0 * (sc - in.s) / (sc - 1.0));
  if (!(s.gamma > 0) || !std::isfinite(s.gamma)) throw PotError(ErrorCode::DegenerateInstance, "derived gamma is not positive");
  if (!(s.eps_tilde > 0)) throw PotError(ErrorCode::DegenerateInstance, "stopping tolerance collapsed to zero (budget equals mass)");
  const double lambda = std::min(s.eps_tilde / 8.0, 0.5);
  const double nd = double(n);
  s.mixed_r.resize(static_cast<size_t>(n)); s.mixed_c.resize(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) {
    s.mixed_r[size_t(i)] = (1.0 - lambda) * in.r[size_t(i)] + lambda / nd;
    s.mixed_c[size_t(i)] = (1.0 - lambda) * in.c[size_t(i)] + lambda / nd;
  }
  return s;
}

struct TheoryBounds { double R = 0.0, L = 0.0, mu_f = 0.0, iteration_bound = 0.0; };

inline TheoryBounds theory_bounds(const Instance& in, double gamma, double eps_prime) {  // solvers.hpp:146-174
  if (!(gamma > 0) || !std::isfinite(gamma)) throw PotError(ErrorCode::InvalidArgument, "gamma must be positive");
  if (!(eps_prime > 0) || !std::isfinite(eps_prime)) throw PotError(ErrorCode::InvalidArgument, "eps_prime must be positive");
  const double sr = in.source_mass(), sc = in.target_mass();
  const double M = std::max(sr, sc);
  if (!(M > in.s)) throw PotError(ErrorCode::DegenerateInstance, "dual radius is infinite when budget equals max mass");
  const double me = std::min(vmin(in.r), vmin(in.c));
  if (!(me > 0)) throw PotError(ErrorCode::DegenerateInstance, "dual radius needs strictly positive marginals");
  TheoryBounds tb;
  tb.R = in.max_cost() * M / (gamma * (M - in.s)) - std::log(me);
  tb.mu_f = gamma / (sr + sc - in.s);
  tb.L = 3.0 / tb.mu_f;
  const double n = double(in.size());
  tb.iteration_bound = 1.0 + std::pow(12.0 * std::sqrt(14.0 * n * tb.L) * tb.R / eps_prime, 2.0 / 3.0);
  return tb;
}

// rounding.hpp:14-39
inline Mat round_balanced(const Mat& X, const Vec& r, const Vec& c) {
  if (X.rows != long(r.size()) || X.cols != long(c.size())) throw PotError(ErrorCode::DimensionMismatch, "plan/marginal shape mismatch");
  const double sr = vsum(r), sc = vsum(c);
  if (std::fabs(sr - sc) > 1e-12 * std::max({1.0, sr, sc})) throw PotError(ErrorCode::UnbalancedMarginals, "marginal masses differ");
  Mat out = X;
  const Vec row = mrowsum(out);
  for (long i = 0; i < out.rows; ++i) if (row[size_t(i)] > 0) { const double f = std::min(1.0, r[size_t(i)] / row[size_t(i)]); for (long j = 0; j < out.cols; ++j) out(i, j) *= f; }
  const Vec col = mcolsum(out);
  for (long j = 0; j < out.cols; ++j) if (col[size_t(j)] > 0) { const double f = std::min(1.0, c[size_t(j)] / col[size_t(j)]); for (long i = 0; i < out.rows; ++i) out(i, j) *= f; }
  const Vec rs = mrowsum(out), cs = mcolsum(out);
  Vec er(rs.size()), ec(cs.size());
  for (size_t i = 0; i < rs.size(); ++i) er[i] = r[i] - rs[i];
  for (size_t j = 0; j < cs.size(); ++j) ec[j] = c[j] - cs[j];
  const double total = vsum(er);
  if (total > 0) for (long j = 0; j < out.cols; ++j) for (long i = 0; i < out.rows; ++i) out(i, j) += (er[size_t(i)] * ec[size_t(j)]) / total;
  return out;
}

// rounding.hpp:46-77
inline TransportPlan round_pot(const Mat& X, const Instance& in) {
  validate(in);
  if (X.rows != in.size() || X.cols != in.size()) throw PotError(ErrorCode::DimensionMismatch, "plan shape does not match the instance");
  Mat out = X;
  const double mass = msum(out);
  if (mass > 0) { const double f = std::min(1.0, in.s / mass); for (double& e : out.a) e *= f; }
  const Vec row = mrowsum(out);
  for (long i = 0; i < out.rows; ++i) if (row[size_t(i)] > 0) { const double f = std::min(1.0, in.r[size_t(i)] / row[size_t(i)]); for (long j = 0; j < out.cols; ++j) out(i, j) *= f; }
  const Vec col = mcolsum(out);
  for (long j = 0; j < out.cols; ++j) if (col[size_t(j)] > 0) { const double f = std::min(1.0, in.c[size_t(j)] / col[size_t(j)]); for (long i = 0; i < out.rows; ++i) out(i, j) *= f; }
  const double deficit = in.s - msum(out);
  if (deficit > 0) {
    const Vec rs = mrowsum(out), cs = mcolsum(out);
    Vec a(rs.size()), b(cs.size());
    for (size_t i = 0; i < rs.size(); ++i) a[i] = std::max(in.r[i] - rs[i], 0.0);
    for (size_t j = 0; j < cs.size(); ++j) b[j] = std::max(in.c[j] - cs[j], 0.0);
    const double na = vsum(a), nb = vsum(b);
    if (na <= 0 || nb <= 0) throw PotError(ErrorCode::Infeasible, "deficit fill has no slack mass");
    const double f = deficit / (na * nb);
    for (long j = 0; j < out.cols; ++j) for (long i = 0; i < out.rows; ++i) out(i, j) += f * (a[size_t(i)] * b[size_t(j)]);
  }
  return TransportPlan::from(std::move(out), in);
}

// extend.hpp:11-60
struct ExtendedOtInstance { Mat C_ext; Vec r_ext, c_ext; double penalty_A = 0.0; };

inline ExtendedOtInstance extend(const Instance& in, double A) {
  validate(in);
  if (!(A > in.max_cost())) throw PotError(ErrorCode::PenaltyTooSmall, "penalty must exceed max cost");
  const long n = in.size();
  ExtendedOtInstance e;
  e.penalty_A = A;
  e.C_ext = Mat(n + 1, n + 1, 0.0);
  for (long j = 0; j < n; ++j) for (long i = 0; i < n; ++i) e.C_ext(i, j) = in.C(i, j);
  e.C_ext(n, n) = A;
  e.r_ext = in.r; e.r_ext.push_back(std::max(vsum(in.c) - in.s, 0.0));
  e.c_ext = in.c; e.c_ext.push_back(std::max(vsum(in.r) - in.s, 0.0));
  return e;
}

struct BlockDecomposition { Mat block; Vec dummy_col, dummy_row; double corner = 0.0; };

inline BlockDecomposition extract_block(const Mat& Xe) {
  if (Xe.rows != Xe.cols || Xe.rows < 2) throw PotError(ErrorCode::DimensionMismatch, "extended plan must be square with side >= 2");
  const long n = Xe.rows - 1;
  BlockDecomposition o;
  o.block = Mat(n, n);
  for (long j = 0; j < n; ++j) for (long i = 0; i < n; ++i) o.block(i, j) = Xe(i, j);
  o.dummy_col.resize(static_cast<size_t>(n)); o.dummy_row.resize(static_cast<size_t>(n));
  for (long i = 0; i < n; ++i) { o.dummy_col[size_t(i)] = Xe(i, n); o.dummy_row[size_t(i)] = Xe(n, i); }
  o.corner = Xe(n, n);
  return o;
}

struct SolveResult {  // solvers.hpp:176-186
  TransportPlan plan;
  ConvergenceTrace trace;
  SolveStatus status = SolveStatus::Converged;
  long iterations = 0;
  double gamma = 0.0, tolerance = 0.0, final_error = 0.0, wall_seconds = 0.0;
  std::optional<TheoryBounds> bounds;
  double phi = 0.0;  // dual value at the stopping iterate (not in the reference struct; for parity)
};

// Decision log per accepted ASPOT iteration (oracle + GPU both emit it).
struct IterLog {
  long t = 0;
  int halvings = 0;
  int block_hat = 0;       // GK block chosen at z_grave
  int zbest_is_check = 0;  // 1 when phi(z_check) <= phi_hat
  int block_check = 0;     // GK block chosen at z_best
  double error = 0.0, phi_check = 0.0, phi_hat = 0.0, theta = 0.0;
};

struct AspotIterate {  // solvers.hpp:190-202
  long t; double theta, error;
  const EntropicContext& ctx;
  const DualPoint &z_grave, &z_hat, &z_best, &z_check;
  double phi_hat, phi_best, phi_check;
};
using AspotObserver = std::function<void(const AspotIterate&)>;

using Clock = std::chrono::steady_clock;
inline double seconds_since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

inline SolveResult trivial_result(const Instance& in, Mat X, double gamma, double tol) {  // solvers.hpp:240-255
  SolveResult o;
  o.plan = TransportPlan::from(std::move(X), in);
  o.gamma = gamma; o.tolerance = tol;
  TraceRecord rec; rec.rounded_cost = transport_cost(in.C, o.plan.X);
  o.trace.records.push_back(rec);
  o.trace.stopping_iterate = "trivial";
  return o;
}

struct PhiGrad { double phi = 0.0; DualPoint grad; BSums sums; };

inline PhiGrad phi_and_gradient(const EntropicContext& ctx, const DualPoint& z) {  // solvers.hpp:220-234
  check_exp_range(vmax(z.u), "exp(u)");
  check_exp_range(vmax(z.v), "exp(v)");
  PhiGrad o;
  o.sums = sweep(ctx, z);
  o.phi = phi_from(ctx, z, o.sums.total);
  o.grad = grad_from(ctx, z, o.sums);
  return o;
}

// Optional hooks so the oracle can run with a points-based logK (config C4)
// and skip dense plan materialisation for the CPU-baseline timing.
struct RunOptions {
  const double* X = nullptr; const double* Y = nullptr; int d = 0; double scale = 1.0;  // points mode
  bool skip_plan = false;      // do not round/materialise the final plan (timing only)
  std::vector<IterLog>* log = nullptr;
};

// solvers.hpp:265-385
inline SolveResult aspot_solve(const Instance& in, const SolverConfig& config, const AspotObserver& observer = {},
                               const RunOptions& ro = {}) {
  validate(in);
  config.check();
  if (in.size() < 2) throw PotError(ErrorCode::DegenerateInstance, "accelerated solver needs n >= 2");
  const auto start = Clock::now();
  if (in.s == 0) return trivial_result(in, Mat(in.size(), in.size(), 0.0), 0.0, 0.0);
  const AspotSetup setup = aspot_setup(in, config.epsilon);
  const double gamma = config.gamma_override.value_or(setup.gamma);
  if (!(gamma > 0) || !std::isfinite(gamma)) throw PotError(ErrorCode::InvalidArgument, "gamma must be positive");
  EntropicContext ctx;
  if (ro.X) {
    ctx.gamma = gamma; ctx.r = setup.mixed_r; ctx.c = setup.mixed_c; ctx.s = in.s;
    ctx.logK.n = in.size(); ctx.logK.gamma = gamma; ctx.logK.X = ro.X; ctx.logK.Y = ro.Y; ctx.logK.d = ro.d; ctx.logK.scale = ro.scale;
  } else {
    ctx = EntropicContext(in.C, gamma, setup.mixed_r, setup.mixed_c, in.s);
  }
  SolveResult result;
  result.gamma = gamma;
  result.tolerance = setup.eps_tilde;
  result.trace.stopping_iterate = "z_check";
  try {
    Instance mixed{setup.mixed_r, setup.mixed_c, in.C, in.s, in.points_mode, in.cmax_hint};
    result.bounds = theory_bounds(mixed, gamma, setup.eps_tilde);
  } catch (const PotError&) { result.bounds.reset(); }

  const long n = in.size();
  const double step_denom = 3.0 * (vsum(setup.mixed_r) + vsum(setup.mixed_c) - in.s);
  DualPoint z = DualPoint::zero(n), z_check = DualPoint::zero(n);
  double theta = 1.0;
  long t = 0, gk_calls = 0;
  PhiGrad check_eval = phi_and_gradient(ctx, z_check);
  double error = grad_l1(check_eval.grad);

  const auto record = [&](long iter, double err, double phi) {
    if (iter % config.log_every != 0 && err > setup.eps_tilde) return;
    TraceRecord rec; rec.t = iter; rec.error = err; rec.phi = phi;
    if (config.record_rounded_cost && !ro.X) rec.rounded_cost = transport_cost(in.C, round_pot(b_matrix(ctx, z_check), in).X);
    rec.elapsed_s = seconds_since(start);
    result.trace.records.push_back(rec);
  };
  record(0, error, check_eval.phi);
  result.status = SolveStatus::Converged;

  while (error > setup.eps_tilde) {
    if (t >= config.max_iterations) { result.status = SolveStatus::MaxIterationsExceeded; break; }
    double step = gamma / (step_denom * theta);
    DualPoint z_grave, z_hat, z_best, next_check;
    PhiGrad next_eval;
    double phi_hat = 0.0, phi_best = 0.0;
    bool stepped = false;
    IterLog lg;
    for (int halvings = 0; halvings <= 60; ++halvings) {
      try {
        const DualPoint z_bar = (1.0 - theta) * z_check + theta * z;
        const DualPoint grad = dual_gradient(ctx, z_bar);
        const DualPoint z_next = z_bar - step * grad;
        z_grave = z_bar + theta * (z_next - z);
        const GkOut gh = greenkhorn_step_ex(ctx, z_grave, config.block_rule, gk_calls);
        z_hat = gh.z;
        phi_hat = dual_objective(ctx, z_hat);
        const bool keep_check = check_eval.phi <= phi_hat;
        z_best = keep_check ? z_check : z_hat;
        phi_best = std::min(check_eval.phi, phi_hat);
        // GK at z_best: when z_best == z_check its B sums are the ones
        // check_eval already holds (identical values, solvers.hpp:46).
        GkOut gc;
        if (keep_check) {
          check_exp_range(vmax(z_best.u), "exp(u)"); check_exp_range(vmax(z_best.v), "exp(v)");
          gc = greenkhorn_from(ctx, z_best, check_eval.sums, config.block_rule, gk_calls + 1);
        } else {
          gc = greenkhorn_step_ex(ctx, z_best, config.block_rule, gk_calls + 1);
        }
        next_check = gc.z;
        next_eval = phi_and_gradient(ctx, next_check);
        lg.halvings = halvings; lg.block_hat = gh.block; lg.zbest_is_check = keep_check ? 1 : 0; lg.block_check = gc.block;
        stepped = true;
        break;
      } catch (const PotError& e) {
        if (e.code != ErrorCode::Overflow) throw;
        step *= 0.5;
      }
    }
    if (!stepped) { result.status = SolveStatus::StepSizeUnderflow; break; }
    gk_calls += 2;
    z = std::move(z_best);
    z_check = std::move(next_check);
    check_eval = std::move(next_eval);
    error = grad_l1(check_eval.grad);
    theta = theta_next(theta);
    ++t;
    if (ro.log) { lg.t = t; lg.error = error; lg.phi_check = check_eval.phi; lg.phi_hat = phi_hat; lg.theta = theta; ro.log->push_back(lg); }
    if (observer) observer(AspotIterate{t, theta, error, ctx, z_grave, z_hat, z, z_check, phi_hat, phi_best, check_eval.phi});
    record(t, error, check_eval.phi);
  }
  if (!ro.skip_plan && !ro.X) result.plan = round_pot(b_matrix(ctx, z_check), in);
  result.iterations = t;
  result.final_error = error;
  result.phi = check_eval.phi;
  result.wall_seconds = seconds_since(start);
  if (result.trace.records.empty() || result.trace.records.back().t != t) {
    TraceRecord rec; rec.t = t; rec.error = error; rec.phi = check_eval.phi;
    if (!ro.skip_plan && !ro.X) rec.rounded_cost = transport_cost(in.C, result.plan.X);
    rec.elapsed_s = result.wall_seconds;
    result.trace.records.push_back(rec);
  }
  return result;
}

// ---------------------------------------------------------------------------
// Extended (dummy-node) log-domain Sinkhorn — solvers.hpp:387-481.
inline double masked_dot(const Vec& p, const Vec& w) {  // solvers.hpp:389-395
  double t = 0.0;
  for (size_t i = 0; i < w.size(); ++i) if (w[i] > 0) t += p[i] * w[i];
  return t;
}

// logK over the (n+1)^2 extension without materialising C_ext: the top-left
// block is the base logK, the dummy row/column hold -0/gamma and the corner
// -A/gamma (extend.hpp:31-33 then solvers.hpp:420).
struct ExtLogK {
  const LogK* base; long n; double corner;
  inline double at(long i, long j) const {
    if (i < n && j < n) return base->at(i, j);
    if (i == n && j == n) return corner;
    return -0.0 / base->gamma;
  }
};

struct ExtendedSinkhornRun { Mat B; Vec u, v; long iterations = 0; SolveStatus status = SolveStatus::Converged; double final_error = 0.0; double phi = 0.0; };

inline double seq_max(double m, double x) { return (x > m || m != m) ? x : m; }



inline ExtendedSinkhornRun extended_sinkhorn(const ExtendedOtInstance& ext, const ExtLogK& K, double tol, const SolverConfig& config,
                                             const Instance& original, ConvergenceTrace& trace, Clock::time_point start,
                                             bool materialise_B) {
  const long m = long(ext.r_ext.size());
  Vec log_r(static_cast<size_t>(m)), log_c(static_cast<size_t>(m));
  for (long i = 0; i < m; ++i) { log_r[size_t(i)] = std::log(ext.r_ext[size_t(i)]); log_c[size_t(i)] = std::log(ext.c_ext[size_t(i)]); }
  Vec u(static_cast<size_t>(m), 0.0), v(static_cast<size_t>(m), 0.0);
  // B = exp((logK + u_i) + v_j) (solvers.hpp:426-431) and its row/col sums.
  const auto kernel_sums = [&](Vec& rs, Vec& cs, double& tot) {
    // row sums (each over j in order) and column sums (each over i in order)
    rs.assign(static_cast<size_t>(m), 0.0);
    cs.assign(static_cast<size_t>(m), 0.0);
    parallel_for(m, [&](long i) {
      KSum r; for (long j = 0; j < m; ++j) r.add(eexp((K.at(i, j) + u[size_t(i)]) + v[size_t(j)]));
      rs[size_t(i)] = r.get();
    });
    parallel_for(m, [&](long j) {
      KSum c; for (long i = 0; i < m; ++i) c.add(eexp((K.at(i, j) + u[size_t(i)]) + v[size_t(j)]));
      cs[size_t(j)] = c.get();
    });
    tot = vsum(cs);
  };
  const auto marginal_error = [&](const Vec& rs, const Vec& cs) {  // solvers.hpp:432-435
    Vec a(static_cast<size_t>(m)), b(static_cast<size_t>(m));
    for (long i = 0; i < m; ++i) { a[size_t(i)] = rs[size_t(i)] - ext.r_ext[size_t(i)]; b[size_t(i)] = cs[size_t(i)] - ext.c_ext[size_t(i)]; }
    return vl1(a) + vl1(b);
  };
  const auto full_B = [&]() {
    Mat B(m, m);
    for (long j = 0; j < m; ++j) for (long i = 0; i < m; ++i) B(i, j) = eexp((K.at(i, j) + u[size_t(i)]) + v[size_t(j)]);
    return B;
  };
  ExtendedSinkhornRun run;
  Vec rs, cs; double tot = 0.0;
  kernel_sums(rs, cs, tot);
  run.final_error = marginal_error(rs, cs);
  const auto dual_value = [&]() { return tot - masked_dot(u, ext.r_ext) - masked_dot(v, ext.c_ext); };  // solvers.hpp:436-438
  const auto record = [&](long iter, double err) {  // solvers.hpp:444-455
    if (iter % config.log_every != 0 && err > tol) return;
    TraceRecord rec; rec.t = iter; rec.error = err; rec.phi = dual_value();
    if (config.record_rounded_cost && original.C.size() > 0) {
      const Mat bal = round_balanced(full_B(), ext.r_ext, ext.c_ext);
      rec.rounded_cost = transport_cost(original.C, round_pot(extract_block(bal).block, original).X);
    }
    rec.elapsed_s = seconds_since(start);
    trace.records.push_back(rec);
  };
  record(0, run.final_error);
  while (run.final_error > tol) {
    if (run.iterations >= config.max_iterations) { run.status = SolveStatus::MaxIterationsExceeded; break; }
    // u = log r - lse_rows(logK + 1 v^T)  (solvers.hpp:463-467, lse_rows :397-401)
    Vec nu(static_cast<size_t>(m));
    parallel_for(m, [&](long i) {
      double mx = -std::numeric_limits<double>::infinity();
      for (long j = 0; j < m; ++j) mx = seq_max(mx, K.at(i, j) + v[size_t(j)]);
      KSum s; for (long j = 0; j < m; ++j) s.add(eexp((K.at(i, j) + v[size_t(j)]) - mx));
      nu[size_t(i)] = log_r[size_t(i)] - (mx + std::log(s.get()));
    });
    u = std::move(nu);
    // v = log c - lse_rows(logK^T + 1 u^T)  (solvers.hpp:468-472)
    Vec nv(static_cast<size_t>(m));
    parallel_for(m, [&](long j) {
      double mx = -std::numeric_limits<double>::infinity();
      for (long i = 0; i < m; ++i) mx = seq_max(mx, K.at(i, j) + u[size_t(i)]);
      KSum s; for (long i = 0; i < m; ++i) s.add(eexp((K.at(i, j) + u[size_t(i)]) - mx));
      nv[size_t(j)] = log_c[size_t(j)] - (mx + std::log(s.get()));
    });
    v = std::move(nv);
    kernel_sums(rs, cs, tot);
    run.final_error = marginal_error(rs, cs);
    ++run.iterations;
    record(run.iterations, run.final_error);
  }
  run.phi = dual_value();
  run.u = u; run.v = v;
  if (materialise_B) run.B = full_B();
  return run;
}

inline double dummy_penalty(const Instance& in, double epsilon) {  // solvers.hpp:485-490
  const double cmax = in.max_cost();
  double A = cmax > 0 ? 8.0 * cmax / epsilon : 0.0;
  if (!(A > cmax) || !std::isfinite(A)) A = cmax > 0 ? 2.0 * cmax : 1.0;
  return A;
}

inline SolveResult finish_extended_solve(const Instance& in, const ExtendedOtInstance& ext, ExtendedSinkhornRun run, double gamma,
                                         double tol, ConvergenceTrace trace, Clock::time_point start, bool skip_plan) {  // :492-509
  SolveResult r;
  if (!skip_plan) {
    const Mat bal = round_balanced(run.B, ext.r_ext, ext.c_ext);
    r.plan = round_pot(extract_block(bal).block, in);
  }
  r.trace = std::move(trace);
  r.trace.stopping_iterate = "extended-marginals";
  r.status = run.status; r.iterations = run.iterations; r.gamma = gamma; r.tolerance = tol;
  r.final_error = run.final_error; r.phi = run.phi;
  r.wall_seconds = seconds_since(start);
  return r;
}

inline ExtendedOtInstance extend_lite(const Instance& in, double A) {
  // extend() without the (n+1)^2 copy: marginals only (extend.hpp:35-37).
  if (!(A > in.max_cost())) throw PotError(ErrorCode::PenaltyTooSmall, "penalty must exceed max cost");
  ExtendedOtInstance e; e.penalty_A = A;
  e.r_ext = in.r; e.r_ext.push_back(std::max(vsum(in.c) - in.s, 0.0));
  e.c_ext = in.c; e.c_ext.push_back(std::max(vsum(in.r) - in.s, 0.0));
  return e;
}

inline SolveResult feasible_sinkhorn_solve(const Instance& in, const SolverConfig& config, const RunOptions& ro = {}) {  // :516-542
  validate(in);
  config.check();
  const auto start = Clock::now();
  if (in.s == 0) return trivial_result(in, Mat(in.size(), in.size(), 0.0), 0.0, 0.0);
  if (in.size() == 1) return trivial_result(in, Mat(1, 1, in.s), config.gamma_override.value_or(0.0), 0.0);
  const AspotSetup setup = aspot_setup(in, config.epsilon);
  const double gamma = config.gamma_override.value_or(setup.gamma);
  if (!(gamma > 0) || !std::isfinite(gamma)) throw PotError(ErrorCode::InvalidArgument, "gamma must be positive");
  const double A = dummy_penalty(in, config.epsilon);
  const Instance mixed{setup.mixed_r, setup.mixed_c, in.C, in.s, in.points_mode, in.cmax_hint};
  const ExtendedOtInstance ext = extend_lite(mixed, A);
  LogK base;
  if (ro.X) { base.n = in.size(); base.gamma = gamma; base.X = ro.X; base.Y = ro.Y; base.d = ro.d; base.scale = ro.scale; }
  else { base.n = in.size(); base.gamma = gamma; base.dense = Mat(in.size(), in.size()); for (size_t e = 0; e < in.C.a.size(); ++e) base.dense.a[e] = -in.C.a[e] / gamma; }
  const ExtLogK K{&base, in.size(), -A / gamma};
  ConvergenceTrace trace;
  SolverConfig cfg = config; if (ro.X) cfg.record_rounded_cost = false;
  auto run = extended_sinkhorn(ext, K, setup.eps_tilde, cfg, in, trace, start, !(ro.skip_plan || ro.X));
  return finish_extended_solve(in, ext, std::move(run), gamma, setup.eps_tilde, std::move(trace), start, ro.skip_plan || ro.X);
}

inline SolveResult tuned_sinkhorn_solve(const Instance& in, double epsilon, double p, const SolverConfig& config = {}, const RunOptions& ro = {}) {  // :547-584
  validate(in);
  config.check();
  if (!(epsilon > 0) || !std::isfinite(epsilon)) throw PotError(ErrorCode::InvalidArgument, "epsilon must be positive");
  if (!(p >= 1)) throw PotError(ErrorCode::InvalidArgument, "tuning exponent p must be >= 1");
  const auto start = Clock::now();
  if (in.s == 0) return trivial_result(in, Mat(in.size(), in.size(), 0.0), 0.0, 0.0);
  const double h_min = std::min(entropy(in.r), entropy(in.c));
  if (!(h_min > 0)) throw PotError(ErrorCode::ZeroEntropy, "tuned gamma needs positive marginal entropy");
  if (in.size() == 1) return trivial_result(in, Mat(1, 1, in.s), config.gamma_override.value_or(0.0), 0.0);
  const double gamma = config.gamma_override.value_or(std::pow(2.0 * epsilon / (49.0 * h_min), 1.0 / p));
  if (!(gamma > 0) || !std::isfinite(gamma)) throw PotError(ErrorCode::InvalidArgument, "gamma must be positive");
  const double eps_prime = h_min * std::pow(gamma, p);
  const double A = dummy_penalty(in, epsilon);
  const ExtendedOtInstance ext = extend_lite(in, A);
  LogK base;
  if (ro.X) { base.n = in.size(); base.gamma = gamma; base.X = ro.X; base.Y = ro.Y; base.d = ro.d; base.scale = ro.scale; }
  else { base.n = in.size(); base.gamma = gamma; base.dense = Mat(in.size(), in.size()); for (size_t e = 0; e < in.C.a.size(); ++e) base.dense.a[e] = -in.C.a[e] / gamma; }
  const ExtLogK K{&base, in.size(), -A / gamma};
  ConvergenceTrace trace;
  SolverConfig cfg = config; if (ro.X) cfg.record_rounded_cost = false;
  auto run = extended_sinkhorn(ext, K, eps_prime, cfg, in, trace, start, !(ro.skip_plan || ro.X));
  return finish_extended_solve(in, ext, std::move(run), gamma, eps_prime, std::move(trace), start, ro.skip_plan || ro.X);
}

inline SolveResult tuned_sinkhorn_solve(const Instance& in, const SolverConfig& config) {  // :586-589
  return tuned_sinkhorn_solve(in, config.epsilon, config.tuning_exponent_p, config);
}

inline SolveResult solve(const Instance& in, SolverKind kind, const SolverConfig& config) {  // :591-599
  switch (kind) {
    case SolverKind::Aspot: return aspot_solve(in, config);
    case SolverKind::FeasibleSinkhorn: return feasible_sinkhorn_solve(in, config);
    case SolverKind::TunedSinkhorn: return tuned_sinkhorn_solve(in, config);
  }
  throw PotError(ErrorCode::InvalidArgument, "unknown solver kind");
}

// synthetic.hpp:15-60 (draw order r, c, src(2), tgt(2) interleaved per i).
inline Instance make_synthetic_instance(long n, std::uint64_t seed, double mass_r, double mass_c, double s_frac) {
  if (n < 1) throw PotError(ErrorCode::InvalidArgument, "n must be >= 1");
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0), weight(0.2, 1.0);
  Instance in;
  in.r.resize(static_cast<size_t>(n)); in.c.resize(static_cast<size_t>(n));
  std::vector<double> src(size_t(2 * n)), tgt(size_t(2 * n));
  for (long i = 0; i < n; ++i) {
    in.r[size_t(i)] = weight(rng);
    in.c[size_t(i)] = weight(rng);
    src[size_t(2 * i)] = unit(rng); src[size_t(2 * i + 1)] = unit(rng);
    tgt[size_t(2 * i)] = unit(rng); tgt[size_t(2 * i + 1)] = unit(rng);
  }
  // Eigen's `r *= a / r.sum()` (synthetic.hpp:42-43)
  { const double f = mass_r / vsum(in.r); for (double& e : in.r) e *= f; }
  { const double f = mass_c / vsum(in.c); for (double& e : in.c) e *= f; }
  in.C = Mat(n, n);
  for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) {
    const double dx = src[size_t(2 * i)] - tgt[size_t(2 * j)], dy = src[size_t(2 * i + 1)] - tgt[size_t(2 * j + 1)];
    in.C(i, j) = dx * dx + dy * dy;
  }
  const double cmax = mmax(in.C);
  if (cmax > 0) for (double& e : in.C.a) e /= cmax;
  in.s = s_frac * std::min(vsum(in.r), vsum(in.c));
  return in;
}
inline Instance make_scaling_instance(long n, std::uint64_t seed) { return make_synthetic_instance(n, seed, 5.0, 3.0, 0.2); }

// proj/tests/test_util.hpp:12-30 (the reference's randomized fixture).
inline Instance random_instance(std::mt19937_64& rng, long n) {
  std::uniform_real_distribution<double> unit(0.0, 1.0), weight(0.2, 1.0);
  Instance in;
  in.r.resize(static_cast<size_t>(n)); in.c.resize(static_cast<size_t>(n)); in.C = Mat(n, n);
  for (long i = 0; i < n; ++i) {
    in.r[size_t(i)] = weight(rng);
    in.c[size_t(i)] = weight(rng);
    for (long j = 0; j < n; ++j) in.C(i, j) = unit(rng);
  }
  { const double f = (0.7 + 0.6 * unit(rng)) / vsum(in.r); for (double& e : in.r) e *= f; }
  { const double f = (0.7 + 0.6 * unit(rng)) / vsum(in.c); for (double& e : in.c) e *= f; }
  const double cmax = mmax(in.C);
  if (cmax > 0) for (double& e : in.C.a) e /= cmax;
  in.s = (0.3 + 0.5 * unit(rng)) * std::min(vsum(in.r), vsum(in.c));
  return in;
}

inline DualPoint random_dual_point(std::mt19937_64& rng, long n, double scale = 1.0) {  // test_util.hpp:33-43
  std::uniform_real_distribution<double> sym(-scale, scale);
  DualPoint z = DualPoint::zero(n);
  for (long i = 0; i < n; ++i) { z.u[size_t(i)] = sym(rng); z.v[size_t(i)] = sym(rng); }
  z.w = sym(rng);
  return z;
}

}  // namespace pot_oracle
