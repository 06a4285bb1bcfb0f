// oracle_capi.cpp — C-ABI over the CPU oracle for the Python test harness
// and bench.py's cpu_baseline / --impl reference legs. TEST INFRASTRUCTURE.
//
// Matrices cross this boundary ROW-MAJOR (numpy default); the oracle keeps
// the reference's column-major layout internally.
#include <algorithm>
#include <random>
#include <cstring>

#include "pot_oracle.hpp"

using namespace pot_oracle;

namespace {

Instance make_instance(long n, const double* C, const double* r, const double* c, double s) {
  Instance in;
  in.r.assign(r, r + n);
  in.c.assign(c, c + n);
  in.s = s;
  if (C) {
    in.C = Mat(n, n);
    for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) in.C(i, j) = C[i * n + j];
  }
  return in;
}

int fail(const PotError& e, char* err, int errlen) {
  if (err && errlen > 0) { std::strncpy(err, e.what(), size_t(errlen - 1)); err[errlen - 1] = 0; }
  return 1 + int(e.code);
}

}  // namespace

extern "C" {

// cfg layout (doubles): [0] epsilon, [1] gamma_override (<= 0: none),
// [2] max_iterations, [3] block_rule, [4] tuning p, [5] log_every,
// [6] record_rounded_cost.
// summary layout (doubles, 16): status, iterations, gamma, tolerance,
// final_error, wall_seconds, cost, feasibility_gap, mass, phi, has_bounds,
// R, L, mu_f, iteration_bound, trace_len.
// log rows (9 doubles): t, halvings, block_hat, zbest_is_check, block_check,
// error, phi_check, phi_hat, theta.
// trace rows (5 doubles): t, error, phi, rounded_cost (NaN if none), elapsed.
int oracle_solve(int kind, long n, const double* C, const double* r, const double* c, double s, const double* cfg,
                 const double* X, const double* Y, int d, double scale, int skip_plan, double* summary,
                 double* plan_out, double* log_out, long log_cap, long* log_len, double* trace_out, long trace_cap,
                 char* err, int errlen) {
  try {
    Instance in = make_instance(n, X ? nullptr : C, r, c, s);
    if (X) {
      // Points mode: C is never materialised. max_cost (core.hpp:117) is the
      // max of the fp64 costs scale * |x_i - y_j|^2 themselves (one pass;
      // with scale = 1 / max d^2 it can be 1 + 1 ulp).
      in.points_mode = true;
      LogK lk;
      lk.n = n; lk.X = X; lk.Y = Y; lk.d = d; lk.scale = scale;
      std::vector<double> rowmax(static_cast<size_t>(n), 0.0);
      parallel_for(n, [&](long i) {
        double m = 0.0;
        for (long j = 0; j < n; ++j) m = std::max(m, lk.cost(i, j));
        rowmax[size_t(i)] = m;
      });
      in.cmax_hint = n > 0 ? *std::max_element(rowmax.begin(), rowmax.end()) : 0.0;
    }
    SolverConfig sc;
    sc.epsilon = cfg[0];
    if (cfg[1] > 0) sc.gamma_override = cfg[1];
    sc.max_iterations = long(cfg[2]);
    sc.block_rule = BlockRule(int(cfg[3]));
    sc.tuning_exponent_p = cfg[4];
    sc.log_every = long(cfg[5]);
    sc.record_rounded_cost = cfg[6] != 0;
    std::vector<IterLog> lg;
    RunOptions ro;
    ro.X = X; ro.Y = Y; ro.d = d; ro.scale = scale; ro.skip_plan = skip_plan != 0; ro.log = &lg;
    SolveResult res;
    if (kind == 0) {
      res = aspot_solve(in, sc, {}, ro);
    } else if (kind == 1) {
      res = feasible_sinkhorn_solve(in, sc, ro);
    } else {
      res = tuned_sinkhorn_solve(in, sc.epsilon, sc.tuning_exponent_p, sc, ro);
    }
    const bool have_plan = res.plan.X.size() > 0;
    summary[0] = double(int(res.status));
    summary[1] = double(res.iterations);
    summary[2] = res.gamma;
    summary[3] = res.tolerance;
    summary[4] = res.final_error;
    summary[5] = res.wall_seconds;
    summary[6] = have_plan && !X ? transport_cost(in.C, res.plan.X) : std::nan("");
    summary[7] = have_plan && !X ? plan_feasibility_gap(res.plan, in) : std::nan("");
    summary[8] = have_plan ? res.plan.mass : std::nan("");
    summary[9] = res.phi;
    summary[10] = res.bounds ? 1.0 : 0.0;
    summary[11] = res.bounds ? res.bounds->R : 0.0;
    summary[12] = res.bounds ? res.bounds->L : 0.0;
    summary[13] = res.bounds ? res.bounds->mu_f : 0.0;
    summary[14] = res.bounds ? res.bounds->iteration_bound : 0.0;
    summary[15] = double(res.trace.records.size());
    if (plan_out && have_plan) for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) plan_out[i * n + j] = res.plan.X(i, j);
    if (log_len) *log_len = long(lg.size());
    if (log_out) {
      for (long k = 0; k < long(lg.size()) && k < log_cap; ++k) {
        double* o = log_out + 9 * k;
        o[0] = double(lg[size_t(k)].t); o[1] = lg[size_t(k)].halvings; o[2] = lg[size_t(k)].block_hat;
        o[3] = lg[size_t(k)].zbest_is_check; o[4] = lg[size_t(k)].block_check; o[5] = lg[size_t(k)].error;
        o[6] = lg[size_t(k)].phi_check; o[7] = lg[size_t(k)].phi_hat; o[8] = lg[size_t(k)].theta;
      }
    }
    if (trace_out) {
      for (long k = 0; k < long(res.trace.records.size()) && k < trace_cap; ++k) {
        const auto& rc = res.trace.records[size_t(k)];
        double* o = trace_out + 5 * k;
        o[0] = double(rc.t); o[1] = rc.error; o[2] = rc.phi; o[3] = rc.rounded_cost ? *rc.rounded_cost : std::nan(""); o[4] = rc.elapsed_s;
      }
    }
    return 0;
  } catch (const PotError& e) {
    return fail(e, err, errlen);
  }
}

// One B(z) pass: row/col sums, total and max exponent at logK = -C/gamma.
// Returns 1 + Overflow when the reference's b_matrix would throw.
int oracle_sweep(long n, const double* C, double gamma, const double* u, const double* v, double w, double* row,
                 double* col, double* total, double* max_e, char* err, int errlen) {
  try {
    Mat Cm(n, n);
    for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) Cm(i, j) = C[i * n + j];
    Vec r(size_t(n), 1.0), c(size_t(n), 1.0);
    EntropicContext ctx(Cm, gamma, r, c, 0.0);
    DualPoint z; z.u.assign(u, u + n); z.v.assign(v, v + n); z.w = w;
    BSums b;
    // report max even when it overflows: compute without the throw first
    double mx = -std::numeric_limits<double>::infinity();
    for (long j = 0; j < n; ++j) for (long i = 0; i < n; ++i) mx = std::max(mx, ((ctx.logK.at(i, j) + z.u[size_t(i)]) + z.v[size_t(j)]) + z.w);
    *max_e = mx;
    b = sweep(ctx, z);
    for (long i = 0; i < n; ++i) { row[i] = b.row[size_t(i)]; col[i] = b.col[size_t(i)]; }
    *total = b.total;
    return 0;
  } catch (const PotError& e) {
    return fail(e, err, errlen);
  }
}

// round_pot (rounding.hpp:46-77) on a row-major X; writes the row-major plan.
int oracle_round_pot(long n, const double* Xin, const double* C, const double* r, const double* c, double s, double* Xout,
                     double* cost_gap_mass, char* err, int errlen) {
  try {
    Instance in = make_instance(n, C, r, c, s);
    Mat X(n, n);
    for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) X(i, j) = Xin[i * n + j];
    TransportPlan p = round_pot(X, in);
    for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) Xout[i * n + j] = p.X(i, j);
    cost_gap_mass[0] = transport_cost(in.C, p.X);
    cost_gap_mass[1] = plan_feasibility_gap(p, in);
    cost_gap_mass[2] = p.mass;
    return 0;
  } catch (const PotError& e) {
    return fail(e, err, errlen);
  }
}

// round_balanced (rounding.hpp:14-39), row-major, rows x cols.
int oracle_round_balanced(long rows, long cols, const double* Xin, const double* r, const double* c, double* Xout, char* err,
                          int errlen) {
  try {
    Mat X(rows, cols);
    for (long i = 0; i < rows; ++i) for (long j = 0; j < cols; ++j) X(i, j) = Xin[i * cols + j];
    Vec rv(r, r + rows), cv(c, c + cols);
    Mat o = round_balanced(X, rv, cv);
    for (long i = 0; i < rows; ++i) for (long j = 0; j < cols; ++j) Xout[i * cols + j] = o(i, j);
    return 0;
  } catch (const PotError& e) {
    return fail(e, err, errlen);
  }
}

// make_synthetic_instance (synthetic.hpp:15-54); C written row-major.
int oracle_make_synthetic(long n, unsigned long long seed, double mass_r, double mass_c, double s_frac, double* r, double* c,
                          double* C, double* s) {
  try {
    Instance in = make_synthetic_instance(n, seed, mass_r, mass_c, s_frac);
    for (long i = 0; i < n; ++i) { r[i] = in.r[size_t(i)]; c[i] = in.c[size_t(i)]; }
    for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) C[i * n + j] = in.C(i, j);
    *s = in.s;
    return 0;
  } catch (const PotError& e) {
    return 1 + int(e.code);
  }
}

// test_util.hpp:12-30 random_instance draws from an mt19937_64(seed) stream;
// `skip` earlier instances of sizes `sizes[k]` are drawn first so a test can
// reproduce the k-th instance of a reference test loop.
int oracle_random_instance(unsigned long long seed, long n, double* r, double* c, double* C, double* s) {
  std::mt19937_64 rng(seed);
  Instance in = random_instance(rng, n);
  for (long i = 0; i < n; ++i) { r[i] = in.r[size_t(i)]; c[i] = in.c[size_t(i)]; }
  for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) C[i * n + j] = in.C(i, j);
  *s = in.s;
  return 0;
}

// aspot_setup (solvers.hpp:100-133): out = gamma, eps_tilde; mixed r/c.
int oracle_aspot_setup(long n, const double* C, const double* r, const double* c, double s, double epsilon, double* out,
                       double* mixed_r, double* mixed_c, char* err, int errlen) {
  try {
    Instance in = make_instance(n, C, r, c, s);
    AspotSetup st = aspot_setup(in, epsilon);
    out[0] = st.gamma; out[1] = st.eps_tilde;
    for (long i = 0; i < n; ++i) { mixed_r[i] = st.mixed_r[size_t(i)]; mixed_c[i] = st.mixed_c[size_t(i)]; }
    return 0;
  } catch (const PotError& e) {
    return fail(e, err, errlen);
  }
}

// kmeans_quantize (color_transfer.hpp:34-118): k-means++ seeding with the
// reference's draws (std::mt19937_64, uniform_int / uniform_real
// distributions), Lloyd rounds with sequential cluster sums, final
// assignment. points: n x 3 row-major. Sums follow the reference's
// sequential order except dist2.sum(), which Eigen reduces with packets
// (here: sequential; the pick can differ only on an exact boundary tie).
int oracle_kmeans(long n, const double* pts, int k, unsigned long long seed, double* centroids, double* weights,
                  int* assign_out, int* rounds_out, char* err, int errlen) {
  try {
    if (n == 0) throw PotError(ErrorCode::EmptyInput, "no points to quantize");
    if (k < 1 || k > n) throw PotError(ErrorCode::InvalidArgument, "k must lie in [1, N]");
    auto d2 = [&](long i, const double* c) {
      const double dx = pts[3 * i] - c[0], dy = pts[3 * i + 1] - c[1], dz = pts[3 * i + 2] - c[2];
      return (dx * dx + dy * dy) + dz * dz;
    };
    std::mt19937_64 rng(seed);
    std::vector<double> C(static_cast<size_t>(3 * k));
    std::uniform_int_distribution<long> first(0, n - 1);
    const long f0 = first(rng);
    for (int d = 0; d < 3; ++d) C[size_t(d)] = pts[3 * f0 + d];
    std::vector<double> dist2(static_cast<size_t>(n));
    for (long i = 0; i < n; ++i) dist2[size_t(i)] = d2(i, C.data());
    std::uniform_real_distribution<double> unit(0.0, 1.0);
    for (int j = 1; j < k; ++j) {
      double total = 0.0;
      for (long i = 0; i < n; ++i) total += dist2[size_t(i)];
      long pick = 0;
      if (total > 0) {
        double target = unit(rng) * total;
        for (long i = 0; i < n; ++i) {
          target -= dist2[size_t(i)];
          if (target <= 0) { pick = i; break; }
        }
      } else {
        pick = first(rng);
      }
      for (int d = 0; d < 3; ++d) C[size_t(3 * j + d)] = pts[3 * pick + d];
      for (long i = 0; i < n; ++i) dist2[size_t(i)] = std::min(dist2[size_t(i)], d2(i, &C[size_t(3 * j)]));
    }
    std::vector<int> assign(static_cast<size_t>(n), 0);
    auto nearest = [&](long i) {
      int best = 0;
      double bd = d2(i, C.data());
      for (int j = 1; j < k; ++j) {
        const double dd = d2(i, &C[size_t(3 * j)]);
        if (dd < bd) { best = j; bd = dd; }
      }
      return best;
    };
    int rounds = 0;
    for (int round = 0; round < 100; ++round) {
      ++rounds;
      for (long i = 0; i < n; ++i) assign[size_t(i)] = nearest(i);
      std::vector<double> sums(static_cast<size_t>(3 * k), 0.0);
      std::vector<long> counts(static_cast<size_t>(k), 0);
      for (long i = 0; i < n; ++i) {
        const int a = assign[size_t(i)];
        for (int d = 0; d < 3; ++d) sums[size_t(3 * a + d)] += pts[3 * i + d];
        counts[size_t(a)] += 1;
      }
      double moved = 0.0;
      for (int j = 0; j < k; ++j) {
        if (counts[size_t(j)] == 0) continue;
        double nx[3], m2 = 0.0;
        for (int d = 0; d < 3; ++d) {
          nx[d] = sums[size_t(3 * j + d)] / double(counts[size_t(j)]);
          const double e = nx[d] - C[size_t(3 * j + d)];
          m2 += e * e;
        }
        moved = std::max(moved, std::sqrt(m2));
        for (int d = 0; d < 3; ++d) C[size_t(3 * j + d)] = nx[d];
      }
      if (moved < 1e-6) break;
    }
    std::vector<long> counts(static_cast<size_t>(k), 0);
    for (long i = 0; i < n; ++i) {
      assign[size_t(i)] = nearest(i);
      counts[size_t(assign[size_t(i)])] += 1;
    }
    for (int q = 0; q < 3 * k; ++q) centroids[q] = C[size_t(q)];
    for (int j = 0; j < k; ++j) weights[j] = double(counts[size_t(j)]) / double(n);
    for (long i = 0; i < n; ++i) assign_out[i] = assign[size_t(i)];
    if (rounds_out) *rounds_out = rounds;
    return 0;
  } catch (const PotError& e) {
    return fail(e, err, errlen);
  }
}

// Host threads for the n^2 passes (1 = the reference's single-threaded
// semantics; >1 only for CPU-baseline timing).
int oracle_set_threads(int t) {
  oracle_threads() = t < 1 ? 1 : t;
  return oracle_threads();
}

}  // extern "C"
