// kat_main.cpp — pins the CPU oracle against the reference's own known-answer
// tests. TEST INFRASTRUCTURE. A GTest-free port of the hand-valued cases in
// /root/reference/proj/tests/test_{dual,solvers,extend_rounding,core}.cpp
// (GoogleTest is absent from this image). Each case cites its source lines.
// Exit status = number of failed checks. Run by tests/test_oracle_kat.py.
#include <cstdio>
#include <functional>

#include "pot_oracle.hpp"

using namespace pot_oracle;

static int g_fail = 0, g_checks = 0;
static const char* g_case = "";

#define CHECK(cond)                                                                 \
  do {                                                                              \
    ++g_checks;                                                                     \
    if (!(cond)) { ++g_fail; std::printf("FAIL %s: %s (line %d)\n", g_case, #cond, __LINE__); } \
  } while (0)
#define CHECK_NEAR(a, b, tol) CHECK(std::fabs(double(a) - double(b)) <= (tol))
#define CHECK_THROWS(expr, ecode)                                                   \
  do {                                                                              \
    ++g_checks;                                                                     \
    bool ok_ = false;                                                               \
    try { (void)(expr); } catch (const PotError& e_) { ok_ = e_.code == (ecode); }  \
    if (!ok_) { ++g_fail; std::printf("FAIL %s: %s did not throw %s (line %d)\n", g_case, #expr, #ecode, __LINE__); } \
  } while (0)

static void run(const char* name, const std::function<void()>& f) {
  g_case = name;
  const int before = g_fail;
  try { f(); } catch (const std::exception& e) { ++g_fail; std::printf("FAIL %s: unexpected exception %s\n", name, e.what()); }
  std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", name);
}

static Instance scalar_instance(double r, double c, double cost, double s) {
  Instance in; in.r = {r}; in.c = {c}; in.C = Mat(1, 1, cost); in.s = s; return in;
}
static DualPoint scalar_dual(double u, double v, double w) { DualPoint z; z.u = {u}; z.v = {v}; z.w = w; return z; }
static EntropicContext ctx_of(const Instance& in, double g) { return EntropicContext(in.C, g, in.r, in.c, in.s); }
static Instance uniform_instance(long n, double mass, double s) {  // test_solvers.cpp:24-32
  Instance in; in.r.assign(size_t(n), mass / double(n)); in.c = in.r;
  in.C = Mat(n, n, 1.0); for (long i = 0; i < n; ++i) in.C(i, i) = 0.0; in.s = s; return in;
}
static Instance two_point_instance() {  // test_extend_rounding.cpp:14-24
  Instance in; in.r = {0.3, 0.2}; in.c = {0.4, 0.1}; in.C = Mat(2, 2);
  in.C(0, 0) = 0.2; in.C(0, 1) = 0.9; in.C(1, 0) = 0.7; in.C(1, 1) = 0.1; in.s = 0.1; return in;
}

int main() {
  // ---------------- test_dual.cpp ----------------
  run("BMatrix.ZeroEverything (test_dual.cpp:33-37)", [] {
    const auto ctx = ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0);
    CHECK(b_matrix(ctx, DualPoint::zero(1))(0, 0) == 1.0);
  });
  run("BMatrix.PotentialsMultiply (:39-43)", [] {
    const auto ctx = ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0);
    CHECK_NEAR(b_matrix(ctx, scalar_dual(std::log(2.0), 0.0, std::log(3.0)))(0, 0), 6.0, 1e-14);
  });
  run("BMatrix.CostAttenuates (:45-52)", [] {
    for (double g : {0.5, 1.0, 3.0}) {
      const auto ctx = ctx_of(scalar_instance(1, 1, g * std::log(4.0), 0.5), g);
      CHECK_NEAR(b_matrix(ctx, DualPoint::zero(1))(0, 0), 0.25, 1e-14);
    }
  });
  run("BMatrix.OverflowIsStructuredError (:54-62)", [] {
    const auto ctx = ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0);
    CHECK_THROWS(b_matrix(ctx, scalar_dual(400.0, 400.0, 0.0)), ErrorCode::Overflow);
    CHECK_THROWS(sweep(ctx, scalar_dual(400.0, 400.0, 0.0)), ErrorCode::Overflow);
  });
  run("EntropicContext.LogKernelIsRecomputable (:64-71)", [] {
    std::mt19937_64 rng(11);
    const Instance in = random_instance(rng, 4);
    const auto ctx = ctx_of(in, 0.3);
    double worst = 0.0;
    for (long i = 0; i < 4; ++i) for (long j = 0; j < 4; ++j) worst = std::max(worst, std::fabs(ctx.logK.dense(i, j) * (-0.3) - in.C(i, j)));
    CHECK(worst <= 1e-15);
    CHECK_THROWS(ctx_of(in, 0.0), ErrorCode::InvalidArgument);
  });
  run("DualObjective.ScalarHandEvaluation (:73-76)", [] {
    CHECK(dual_objective(ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0), DualPoint::zero(1)) == 3.0);
  });
  run("DualObjective.ZeroPotentialsKillLinearTerms (:78-86)", [] {
    std::mt19937_64 rng(12);
    for (int rep = 0; rep < 5; ++rep) {
      Instance in = random_instance(rng, 2);
      for (double& e : in.C.a) e = 0.0;
      CHECK(dual_objective(ctx_of(in, 1.0), DualPoint::zero(2)) == 8.0);
    }
  });
  run("DualObjective.ConvergedSolverPointIsMinimal (:88-109)", [] {
    std::mt19937_64 rng(13);
    const Instance in = random_instance(rng, 4);
    SolverConfig cfg; cfg.epsilon = 0.02; cfg.max_iterations = 100000; cfg.log_every = 1000000;
    DualPoint zs = DualPoint::zero(4); double g = 0.0;
    const auto res = aspot_solve(in, cfg, [&](const AspotIterate& it) { zs = it.z_check; g = it.ctx.gamma; });
    CHECK(res.status == SolveStatus::Converged);
    const AspotSetup st = aspot_setup(in, cfg.epsilon);
    const EntropicContext ctx(in.C, g, st.mixed_r, st.mixed_c, in.s);
    const double phis = dual_objective(ctx, zs);
    for (int rep = 0; rep < 50; ++rep) CHECK(phis <= dual_objective(ctx, random_dual_point(rng, 4, 2.0)) + 1e-9);
  });
  run("DualGradient.ScalarHandEvaluation (:111-117)", [] {
    const DualPoint g = dual_gradient(ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0), DualPoint::zero(1));
    CHECK(g.u[0] == 1.0); CHECK(g.v[0] == 1.0); CHECK(g.w == 0.5);
  });
  run("DualGradient.ExactBlockUpdateZeroesGradientBlock (:119-130)", [] {
    std::mt19937_64 rng(14);
    for (int rep = 0; rep < 20; ++rep) {
      const Instance in = random_instance(rng, 3);
      const auto ctx = ctx_of(in, 0.7);
      const DualPoint z = random_dual_point(rng, 3, 0.5);
      const DualPoint g = dual_gradient(ctx, greenkhorn_step(ctx, z, BlockRule::RoundRobin, 0));
      double m = 0.0; for (double e : g.u) m = std::max(m, std::fabs(e));
      CHECK(m <= 1e-12);
    }
  });
  run("DualGradient.MatchesCentralDifferences (:132-155)", [] {
    std::mt19937_64 rng(15);
    const double h = 1e-6;
    for (int rep = 0; rep < 20; ++rep) {
      const long n = 2 + (rep % 5);
      const Instance in = random_instance(rng, n);
      const auto ctx = ctx_of(in, 0.5);
      DualPoint z = random_dual_point(rng, n, 1.0);
      const DualPoint g = dual_gradient(ctx, z);
      auto chk = [&](double an, double* slot) {
        const double sv = *slot; *slot = sv + h; const double hi = dual_objective(ctx, z);
        *slot = sv - h; const double lo = dual_objective(ctx, z); *slot = sv;
        const double fd = (hi - lo) / (2.0 * h);
        CHECK_NEAR(an, fd, 1e-5 * std::max(1e-2, std::fabs(fd)));
      };
      for (long i = 0; i < n; ++i) chk(g.u[size_t(i)], &z.u[size_t(i)]);
      for (long j = 0; j < n; ++j) chk(g.v[size_t(j)], &z.v[size_t(j)]);
      chk(g.w, &z.w);
    }
  });
  run("FeasibilityError.ScalarHandEvaluation (:157-160)", [] {
    CHECK(feasibility_error(ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0), DualPoint::zero(1)) == 2.5);
  });
  run("FeasibilityError.VanishesAtStationarity (:162-167)", [] {
    CHECK_NEAR(feasibility_error(ctx_of(scalar_instance(1.5, 1.5, 0, 0.5), 1.0), scalar_dual(0, 0, std::log(0.5))), 0.0, 1e-15);
  });
  run("FeasibilityError.EqualsGradientNormsExactly (:169-180)", [] {
    std::mt19937_64 rng(16);
    for (int rep = 0; rep < 200; ++rep) {
      const long n = 2 + (rep % 4);
      const Instance in = random_instance(rng, n);
      const auto ctx = ctx_of(in, 0.4);
      const DualPoint z = random_dual_point(rng, n, 1.5);
      CHECK(feasibility_error(ctx, z) == grad_l1(dual_gradient(ctx, z)));
    }
  });
  run("DualObjective.ConvexityWitness (:182-197)", [] {
    std::mt19937_64 rng(17);
    std::uniform_real_distribution<double> unit(0.01, 0.99);
    for (int rep = 0; rep < 200; ++rep) {
      const long n = 2 + (rep % 4);
      const Instance in = random_instance(rng, n);
      const auto ctx = ctx_of(in, 0.6);
      const DualPoint z1 = random_dual_point(rng, n, 1.0), z2 = random_dual_point(rng, n, 1.0);
      const double l = unit(rng);
      CHECK(dual_objective(ctx, l * z1 + (1.0 - l) * z2) <= l * dual_objective(ctx, z1) + (1.0 - l) * dual_objective(ctx, z2) + 1e-10);
    }
  });
  run("Rho.HandValues (:199-203)", [] {
    CHECK(rho(1.0, 1.0) == 0.0);
    CHECK_NEAR(rho(1.0, std::exp(1.0)), std::exp(1.0) - 2.0, 1e-15);
    CHECK_NEAR(rho(2.0, 1.0), 1.0 - 2.0 + 2.0 * std::log(2.0), 1e-15);
  });
  run("Rho.NonnegativeAndZeroOnDiagonal (:205-216)", [] {
    std::mt19937_64 rng(18);
    std::uniform_real_distribution<double> pos(1e-6, 100.0);
    for (int rep = 0; rep < 10000; ++rep) { const double a = pos(rng), b = pos(rng); CHECK(rho(a, b) >= 0.0); }
    for (int rep = 0; rep < 100; ++rep) { const double a = pos(rng); CHECK(std::fabs(rho(a, a)) <= 1e-15); }
  });
  run("Rho.RejectsNonPositiveArguments (:218-227)", [] {
    CHECK_THROWS(rho(0.0, 1.0), ErrorCode::NonPositiveArgument);
    CHECK_THROWS(rho(1.0, -1.0), ErrorCode::NonPositiveArgument);
  });

  // ---------------- test_solvers.cpp ----------------
  run("Entropy.HandValues (test_solvers.cpp:36-43)", [] {
    CHECK(entropy({1.0}) == 0.0);
    CHECK_NEAR(entropy({0.5, 0.5}), std::log(2.0), 1e-15);
    CHECK_NEAR(entropy({0.5, 0.5, 0.0}), std::log(2.0), 1e-15);
    CHECK_THROWS(entropy({-0.1}), ErrorCode::NegativeEntry);
  });
  run("ThetaSchedule (:45-67)", [] {
    CHECK_NEAR(theta_next(1.0), (std::sqrt(5.0) - 1.0) / 2.0, 1e-15);
    for (double th : {1.0, 0.5, 0.1}) { const double nx = theta_next(th); CHECK_NEAR(nx / th - std::sqrt(1.0 - nx), 0.0, 1e-14); }
    double th = 1.0;
    for (long t = 0; t <= 10000; ++t) { CHECK(th <= 2.0 / double(t + 2) + 1e-15); th = theta_next(th); }
    CHECK_THROWS(theta_next(0.0), ErrorCode::InvalidArgument);
    CHECK_THROWS(theta_next(1.5), ErrorCode::InvalidArgument);
  });
  run("GreenkhornStep.ScalarUBlock (:69-75)", [] {
    const DualPoint z2 = greenkhorn_step(ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0), DualPoint::zero(1), BlockRule::RoundRobin, 0);
    CHECK_NEAR(z2.u[0], -std::log(2.0), 1e-15); CHECK(z2.v[0] == 0.0); CHECK(z2.w == 0.0);
  });
  run("GreenkhornStep.StationaryBlockUnchanged (:77-84)", [] {
    DualPoint z = DualPoint::zero(1); z.w = std::log(0.5);
    CHECK_NEAR(greenkhorn_step(ctx_of(scalar_instance(1.5, 1.5, 0, 0.5), 1.0), z, BlockRule::RoundRobin, 0).u[0], 0.0, 1e-15);
  });
  run("GreenkhornStep.ScalarWBlock (:86-91)", [] {
    const DualPoint z2 = greenkhorn_step(ctx_of(scalar_instance(1, 1, 0, 0.5), 1.0), DualPoint::zero(1), BlockRule::RoundRobin, 2);
    CHECK_NEAR(z2.w, -std::log(2.0), 1e-15); CHECK(z2.u[0] == 0.0);
  });
  run("GreenkhornStep.MonotoneDescent (:93-106)", [] {
    std::mt19937_64 rng(21);
    for (int rep = 0; rep < 10000; ++rep) {
      const long n = 2 + (rep % 4);
      const Instance in = random_instance(rng, n);
      const auto ctx = ctx_of(in, 0.5);
      const DualPoint z = random_dual_point(rng, n, 1.5);
      const double before = dual_objective(ctx, z);
      const BlockRule rule = rep % 2 == 0 ? BlockRule::Greedy : BlockRule::RoundRobin;
      CHECK(dual_objective(ctx, greenkhorn_step(ctx, z, rule, rep)) <= before + 1e-12 * std::fabs(before));
    }
  });
  run("AspotSetup.DerivedConstantsWithoutClamps (:108-114)", [] {
    const AspotSetup st = aspot_setup(uniform_instance(100, 1.0, 0.5), 0.1);
    CHECK_NEAR(st.gamma, 0.1 / (4.0 * std::log(100.0)), 1e-15);
    CHECK_NEAR(st.gamma, 0.005429, 1e-6);
    CHECK(st.eps_tilde == 0.0125);
  });
  run("AspotSetup.UniformMarginalIsMixingFixedPoint (:116-121)", [] {
    const Instance in = uniform_instance(8, 1.0, 0.25);
    const AspotSetup st = aspot_setup(in, 0.1);
    for (long i = 0; i < 8; ++i) { CHECK_NEAR(st.mixed_r[size_t(i)], in.r[size_t(i)], 1e-16); CHECK_NEAR(st.mixed_c[size_t(i)], in.c[size_t(i)], 1e-16); }
  });
  run("AspotSetup.ClampFormula (:123-137)", [] {
    Instance in = uniform_instance(4, 5.0, 0.6);
    in.c.assign(4, 5.0 / 4.0);
    CHECK(aspot_setup(in, 0.1).eps_tilde == 0.0125);
    CHECK(aspot_setup(in, 100.0).eps_tilde == 8.8);
  });
  run("AspotSetup.MixedMarginalsStrictlyPositive (:139-151)", [] {
    std::mt19937_64 rng(22);
    for (int rep = 0; rep < 20; ++rep) {
      Instance in = random_instance(rng, 5);
      in.r[0] = 0.0;
      in.s = 0.2 * std::min(vsum(in.r), vsum(in.c));
      const AspotSetup st = aspot_setup(in, 0.1);
      CHECK(vmin(st.mixed_r) > 0.0); CHECK(vmin(st.mixed_c) > 0.0);
      CHECK(vsum(st.mixed_r) >= in.s - 1e-12); CHECK(vsum(st.mixed_c) >= in.s - 1e-12);
    }
  });
  run("AspotSetup.RejectsTinyProblems (:153-155)", [] {
    CHECK_THROWS(aspot_setup(scalar_instance(1, 1, 0, 0.5), 0.1), ErrorCode::DegenerateInstance);
  });
  run("AspotSetup.BudgetAtMassWithLargeMarginalsDegenerates (:157-165)", [] {
    CHECK_THROWS(aspot_setup(uniform_instance(4, 5.0, 5.0), 0.1), ErrorCode::DegenerateInstance);
  });
  run("TheoryBounds.MatchesDerivedLipschitzConstant (:167-176)", [] {
    std::mt19937_64 rng(23);
    const Instance in = random_instance(rng, 6);
    const double eps = 0.2, g = eps / (4.0 * std::log(6.0));
    const TheoryBounds tb = theory_bounds(in, g, eps / 8.0);
    const double L = 12.0 * std::log(6.0) * (vsum(in.r) + vsum(in.c) - in.s) / eps;
    CHECK_NEAR(tb.L, L, 1e-9 * L);
  });
  run("TheoryBounds.HandComputedRadius (:178-187)", [] {
    Instance in; in.r = {0.5, 0.5}; in.c = {0.25, 0.75}; in.C = Mat(2, 2, 1.0); in.s = 0.5;
    CHECK_NEAR(theory_bounds(in, 1.0, 0.1).R, 2.0 + std::log(4.0), 1e-12);
  });
  run("TheoryBounds.DegenerateWhenBudgetEqualsMaxMass (:189-192)", [] {
    CHECK_THROWS(theory_bounds(uniform_instance(3, 1.0, 1.0), 0.5, 0.1), ErrorCode::DegenerateInstance);
  });
  run("AspotSolve.ZeroCostInstance (:194-203)", [] {
    Instance in = uniform_instance(2, 1.0, 0.5);
    for (double& e : in.C.a) e = 0.0;
    SolverConfig cfg; cfg.epsilon = 0.1;
    const SolveResult res = aspot_solve(in, cfg);
    CHECK(res.status == SolveStatus::Converged);
    CHECK_NEAR(transport_cost(in.C, res.plan.X), 0.0, 1e-15);
    CHECK(plan_feasibility_gap(res.plan, in) <= 1e-9);
  });
  run("AspotSolve.RejectsSinglePoint (:205-207)", [] {
    CHECK_THROWS(aspot_solve(scalar_instance(1, 1, 0, 0.5), SolverConfig{}), ErrorCode::DegenerateInstance);
  });
  run("AspotSolve.PaperStyleOverrides (:225-237)", [] {
    const Instance in = make_scaling_instance(40, 5);
    SolverConfig cfg; cfg.epsilon = 8e-7; cfg.gamma_override = 1e-3; cfg.max_iterations = 1500; cfg.log_every = 1000000;
    const SolveResult res = aspot_solve(in, cfg);
    CHECK(res.gamma == 1e-3);
    CHECK_NEAR(res.tolerance, 1e-7, 1e-20);
    CHECK(res.status == SolveStatus::Converged);
    CHECK(res.final_error <= res.tolerance);
  });
  run("AspotSolve.StoppingIterateRecordedAndTraceMonotoneIndices (:239-250)", [] {
    std::mt19937_64 rng(25);
    const Instance in = random_instance(rng, 6);
    SolverConfig cfg; cfg.epsilon = 0.05;
    const SolveResult res = aspot_solve(in, cfg);
    CHECK(res.trace.stopping_iterate == "z_check");
    for (size_t i = 1; i < res.trace.records.size(); ++i) CHECK(res.trace.records[i - 1].t < res.trace.records[i].t);
    CHECK(res.final_error <= res.tolerance);
  });
  run("AspotSolve.DescentChainHoldsEveryIteration (:252-270)", [] {
    std::mt19937_64 rng(26);
    for (int rep = 0; rep < 3; ++rep) {
      const Instance in = random_instance(rng, 5);
      SolverConfig cfg; cfg.epsilon = 0.05; cfg.log_every = 1000000;
      long checked = 0;
      aspot_solve(in, cfg, [&](const AspotIterate& it) {
        const double pg = dual_objective(it.ctx, it.z_grave);
        const double slack = 1e-10 * std::max(1.0, std::fabs(pg));
        CHECK(it.phi_hat <= pg + slack); CHECK(it.phi_best <= it.phi_hat + slack); CHECK(it.phi_check <= it.phi_best + slack);
        ++checked;
      });
      CHECK(checked > 0);
    }
  });
  run("AspotSolve.OverflowTriggersStepHalvingAndStillSolves (:272-290)", [] {
    Instance in; in.r = {50.0, 50.0}; in.c = {50.0, 50.0}; in.C = Mat(2, 2, 1.0); in.C(0, 0) = 0; in.C(1, 1) = 0; in.s = 1.0;
    SolverConfig cfg; cfg.epsilon = 0.1; cfg.gamma_override = 1e5; cfg.max_iterations = 20000; cfg.log_every = 1000000;
    const SolveResult res = aspot_solve(in, cfg);
    CHECK(plan_feasibility_gap(res.plan, in) <= 1e-9 * vsum(in.r));
    CHECK(res.status != SolveStatus::StepSizeUnderflow);
  });
  run("AspotSolve.MaxIterationsStillReturnsTraceAndFeasiblePlan (:292-303)", [] {
    std::mt19937_64 rng(27);
    const Instance in = random_instance(rng, 6);
    SolverConfig cfg; cfg.epsilon = 1e-4; cfg.max_iterations = 2;
    const SolveResult res = aspot_solve(in, cfg);
    CHECK(res.status == SolveStatus::MaxIterationsExceeded);
    CHECK(res.iterations == 2);
    CHECK(!res.trace.records.empty());
    CHECK(plan_feasibility_gap(res.plan, in) <= 1e-9);
  });
  run("AspotSolve.ObservedIterationsWithinTheoryBound (:305-316)", [] {
    std::mt19937_64 rng(28);
    SolverConfig cfg; cfg.epsilon = 0.1; cfg.log_every = 1000000;
    for (int rep = 0; rep < 5; ++rep) {
      const Instance in = random_instance(rng, 6);
      const SolveResult res = aspot_solve(in, cfg);
      CHECK(res.bounds.has_value());
      if (res.bounds) CHECK(double(res.iterations) <= res.bounds->iteration_bound);
    }
  });
  run("ExtendedSinkhornEngine.StationaryStartExitsImmediately (:318-335)", [] {
    ExtendedOtInstance ext; ext.r_ext = {2.0, 2.0}; ext.c_ext = {2.0, 2.0};
    LogK base; base.n = 1; base.gamma = 1.0; base.dense = Mat(1, 1, 0.0);
    const ExtLogK K{&base, 1, -0.0 / 1.0};
    Instance original = scalar_instance(2.0, 2.0, 0.0, 0.5);
    SolverConfig cfg; ConvergenceTrace tr;
    const auto run = extended_sinkhorn(ext, K, 0.1, cfg, original, tr, Clock::now(), true);
    CHECK(run.iterations == 0); CHECK(run.status == SolveStatus::Converged); CHECK_NEAR(run.final_error, 0.0, 1e-12);
  });
  run("ExtendedSinkhornEngine.FirstUpdateMatchesHandComputation (:337-354)", [] {
    const Instance original = scalar_instance(1.0, 1.0, 0.5, 0.4);
    const ExtendedOtInstance ext = extend(original, 2.0);
    const double g = 0.8;
    LogK base; base.n = 1; base.gamma = g; base.dense = Mat(1, 1, -0.5 / g);
    const ExtLogK K{&base, 1, -2.0 / g};
    SolverConfig cfg; cfg.max_iterations = 1; ConvergenceTrace tr;
    const auto run = extended_sinkhorn(ext, K, 0.0, cfg, original, tr, Clock::now(), true);
    // K = exp(-C_ext/gamma); expected u = log r_ext - log(K 1)
    const double k00 = std::exp(-0.5 / g), k01 = std::exp(-0.0 / g), k10 = std::exp(-0.0 / g), k11 = std::exp(-2.0 / g);
    CHECK(run.iterations == 1);
    CHECK_NEAR(run.u[0], std::log(ext.r_ext[0]) - std::log(k00 + k01), 1e-13);
    CHECK_NEAR(run.u[1], std::log(ext.r_ext[1]) - std::log(k10 + k11), 1e-13);
  });
  run("FeasibleSinkhorn.SinglePointIsExact (:373-378)", [] {
    const SolveResult res = feasible_sinkhorn_solve(scalar_instance(1.0, 0.8, 3.0, 0.5), SolverConfig{});
    CHECK(res.plan.X(0, 0) == 0.5); CHECK(res.status == SolveStatus::Converged);
  });
  run("TunedSinkhorn.GammaAndTolerancePrescription (:380-392)", [] {
    std::mt19937_64 rng(30);
    const Instance in = random_instance(rng, 5);
    const double h = std::min(entropy(in.r), entropy(in.c));
    SolverConfig cfg; cfg.max_iterations = 1;
    for (double p : {1.0, 2.0, 4.0}) {
      const SolveResult res = tuned_sinkhorn_solve(in, 0.098, p, cfg);
      CHECK_NEAR(res.gamma, std::pow(2.0 * 0.098 / (49.0 * h), 1.0 / p), 1e-14);
      CHECK_NEAR(res.tolerance, 2.0 * 0.098 / 49.0, 1e-14);
    }
  });
  run("TunedSinkhorn.UnitEntropyGivesHandComputedGamma (:394-415)", [] {
    double lo = 0.3, hi = 1.0;
    for (int it = 0; it < 200; ++it) { const double mid = 0.5 * (lo + hi); (entropy(Vec(3, mid / 3.0)) < 1.0 ? lo : hi) = mid; }
    const double a = 0.5 * (lo + hi);
    Instance in; in.r.assign(3, a / 3.0); in.c = in.r; in.C = Mat(3, 3, 1.0); for (long i = 0; i < 3; ++i) in.C(i, i) = 0; in.s = 0.25 * a;
    CHECK_NEAR(entropy(in.r), 1.0, 1e-12);
    SolverConfig cfg; cfg.max_iterations = 1;
    const SolveResult res = tuned_sinkhorn_solve(in, 0.098, 1.0, cfg);
    CHECK_NEAR(res.gamma, 0.004, 1e-12); CHECK_NEAR(res.tolerance, 0.004, 1e-12);
  });
  run("TunedSinkhorn.GammaApproachesOneFromBelow (:417-429)", [] {
    std::mt19937_64 rng(31);
    const Instance in = random_instance(rng, 5);
    SolverConfig cfg; cfg.max_iterations = 1;
    double prev = 0.0;
    for (double p : {1.0, 2.0, 4.0, 8.0, 16.0, 64.0}) { const SolveResult r = tuned_sinkhorn_solve(in, 0.05, p, cfg); CHECK(r.gamma > prev); CHECK(r.gamma < 1.0); prev = r.gamma; }
  });
  run("TunedSinkhorn.RejectsNonPositiveEntropy (:446-461)", [] {
    Instance in; in.r = {3.0, 2.0}; in.c = {2.5, 2.5}; in.C = Mat(2, 2, 1.0); in.s = 1.0;
    CHECK_THROWS(tuned_sinkhorn_solve(in, 0.1, 1.0), ErrorCode::ZeroEntropy);
  });
  run("Solvers.ZeroBudgetReturnsEmptyPlan (:480-490)", [] {
    std::mt19937_64 rng(34);
    Instance in = random_instance(rng, 4);
    in.s = 0.0;
    for (SolverKind k : {SolverKind::Aspot, SolverKind::FeasibleSinkhorn, SolverKind::TunedSinkhorn}) {
      const SolveResult res = solve(in, k, SolverConfig{});
      double m = 0.0; for (double e : res.plan.X.a) m = std::max(m, std::fabs(e));
      CHECK(m == 0.0); CHECK(res.status == SolveStatus::Converged);
    }
  });

  // ---------------- test_extend_rounding.cpp ----------------
  run("Extend.HandComputedMarginals (test_extend_rounding.cpp:28-38)", [] {
    const ExtendedOtInstance e = extend(two_point_instance(), 2.0);
    const double er[3] = {0.3, 0.2, 0.4}, ec[3] = {0.4, 0.1, 0.4};
    for (int i = 0; i < 3; ++i) { CHECK_NEAR(e.r_ext[size_t(i)], er[i], 1e-15); CHECK_NEAR(e.c_ext[size_t(i)], ec[i], 1e-15); }
    CHECK_NEAR(vsum(e.r_ext), 0.9, 1e-15); CHECK_NEAR(vsum(e.c_ext), 0.9, 1e-15);
  });
  run("Extend.FullBudgetGivesZeroDummyMass (:40-50)", [] {
    Instance in; in.r = {0.5, 0.5}; in.c = {0.5, 0.5}; in.C = Mat(2, 2, 1.0); in.s = 1.0;
    const ExtendedOtInstance e = extend(in, 2.0);
    CHECK(e.r_ext[2] == 0.0); CHECK(e.c_ext[2] == 0.0);
  });
  run("Extend.BlockStructure (:52-61)", [] {
    const Instance in = two_point_instance();
    const ExtendedOtInstance e = extend(in, 5.0);
    for (long i = 0; i < 2; ++i) for (long j = 0; j < 2; ++j) CHECK(e.C_ext(i, j) == in.C(i, j));
    CHECK(e.C_ext(2, 2) == 5.0); CHECK(e.C_ext(0, 2) == 0.0); CHECK(e.C_ext(2, 1) == 0.0);
  });
  run("Extend.MassConservation (:63-70)", [] {
    std::mt19937_64 rng(41);
    for (int rep = 0; rep < 100; ++rep) {
      const Instance in = random_instance(rng, 3 + (rep % 4));
      const ExtendedOtInstance e = extend(in, in.max_cost() + 1.0);
      CHECK(std::fabs(vsum(e.r_ext) - vsum(e.c_ext)) <= 1e-12);
    }
  });
  run("Extend.RejectsSmallPenalty (:72-79)", [] { CHECK_THROWS(extend(two_point_instance(), 0.5), ErrorCode::PenaltyTooSmall); });
  run("ExtractBlock.CornerOnlyPlanGivesZeroBlock (:81-87)", [] {
    Mat X(3, 3, 0.0); X(2, 2) = 0.7;
    const BlockDecomposition d = extract_block(X);
    double m = 0.0; for (double e : d.block.a) m = std::max(m, std::fabs(e));
    CHECK(m == 0.0); CHECK(d.corner == 0.7);
  });
  run("ExtractBlock.IdentityBlockPassesThrough (:89-98)", [] {
    Mat X(3, 3, 0.0); X(0, 0) = 0.25; X(1, 1) = 0.25;
    const BlockDecomposition d = extract_block(X);
    CHECK(d.block(0, 0) == 0.25); CHECK(d.block(1, 1) == 0.25);
    CHECK(vmax(d.dummy_col) == 0.0); CHECK(vmax(d.dummy_row) == 0.0);
  });
  run("ExtractBlock.FeasibleExtendedPlansDecompose (:100-118)", [] {
    std::mt19937_64 rng(42);
    for (int rep = 0; rep < 50; ++rep) {
      const Instance in = random_instance(rng, 4);
      const ExtendedOtInstance e = extend(in, in.max_cost() + 0.5);
      std::uniform_real_distribution<double> unit(0.0, 1.0);
      Mat raw(5, 5); for (long i = 0; i < 5; ++i) for (long j = 0; j < 5; ++j) raw(i, j) = unit(rng);
      const BlockDecomposition d = extract_block(round_balanced(raw, e.r_ext, e.c_ext));
      const Vec rs = mrowsum(d.block), cs = mcolsum(d.block);
      for (long i = 0; i < 4; ++i) { CHECK(rs[size_t(i)] - in.r[size_t(i)] <= 1e-9); CHECK(cs[size_t(i)] - in.c[size_t(i)] <= 1e-9); }
      CHECK_NEAR(msum(d.block), in.s + d.corner, 1e-9);
      CHECK(plan_feasibility_gap(round_pot(d.block, in), in) <= 1e-9 * std::max(1.0, vsum(in.r)));
    }
  });
  run("RoundBalanced.FeasibleInputUnchanged (:133-140)", [] {
    Mat X(2, 2, 0.25);
    const Mat o = round_balanced(X, {0.5, 0.5}, {0.5, 0.5});
    for (size_t e = 0; e < 4; ++e) CHECK(o.a[e] == X.a[e]);
  });
  run("RoundBalanced.ScalarScaling (:142-147)", [] { CHECK(round_balanced(Mat(1, 1, 1.0), {0.5}, {0.5})(0, 0) == 0.5); });
  run("RoundBalanced.RandomMatricesGetExactMarginals (:149-170)", [] {
    std::mt19937_64 rng(44);
    std::uniform_real_distribution<double> weight(0.1, 1.0);
    for (int rep = 0; rep < 200; ++rep) {
      Vec r(4), c(4);
      for (int i = 0; i < 4; ++i) { r[size_t(i)] = weight(rng); c[size_t(i)] = weight(rng); }
      { const double f = vsum(r) / vsum(c); for (double& e : c) e *= f; }
      std::uniform_real_distribution<double> unit(0.0, 1.0);
      Mat X(4, 4); for (long i = 0; i < 4; ++i) for (long j = 0; j < 4; ++j) X(i, j) = unit(rng);
      const Mat o = round_balanced(X, r, c);
      const Vec rs = mrowsum(o), cs = mcolsum(o);
      for (int i = 0; i < 4; ++i) { CHECK(std::fabs(rs[size_t(i)] - r[size_t(i)]) <= 1e-12); CHECK(std::fabs(cs[size_t(i)] - c[size_t(i)]) <= 1e-12); }
      double mn = 1e300; for (double e : o.a) mn = std::min(mn, e);
      CHECK(mn >= 0.0);
    }
  });
  run("RoundBalanced.RejectsUnbalancedMarginals (:172-179)", [] {
    CHECK_THROWS(round_balanced(Mat(2, 2, 1.0), {1.0, 1.0}, {0.6, 0.6}), ErrorCode::UnbalancedMarginals);
  });
  run("RoundPot.FeasibleInputUnchanged (:181-189)", [] {
    Instance in = scalar_instance(1.0, 1.0, 0.0, 0.5);
    CHECK(round_pot(Mat(1, 1, 0.5), in).X(0, 0) == 0.5);
  });
  run("RoundPot.MassScalingOnly (:191-199)", [] {
    CHECK(round_pot(Mat(1, 1, 2.0), scalar_instance(1.0, 1.0, 0.0, 0.5)).X(0, 0) == 0.5);
  });
  run("RoundPot.DeficitFillFromZero (:201-214)", [] {
    Instance in; in.r = {0.6, 0.4}; in.c = {0.5, 0.5}; in.C = Mat(2, 2, 1.0); in.s = 0.5;
    const TransportPlan p = round_pot(Mat(2, 2, 0.0), in);
    for (long i = 0; i < 2; ++i) for (long j = 0; j < 2; ++j) CHECK_NEAR(p.X(i, j), 0.5 * in.r[size_t(i)] * in.c[size_t(j)], 1e-15);
    CHECK_NEAR(p.mass, 0.5, 1e-15);
  });
  run("RoundPot.ExactFeasibilityAndIdempotence (:216-231)", [] {
    std::mt19937_64 rng(45);
    for (int rep = 0; rep < 2000; ++rep) {
      const long n = 2 + (rep % 5);
      const Instance in = random_instance(rng, n);
      std::uniform_real_distribution<double> unit(0.0, 2.0);
      Mat X(n, n); for (long i = 0; i < n; ++i) for (long j = 0; j < n; ++j) X(i, j) = unit(rng);
      const TransportPlan p = round_pot(X, in);
      CHECK(plan_feasibility_gap(p, in) <= 1e-9 * std::max(1.0, vsum(in.r)));
      const TransportPlan again = round_pot(p.X, in);
      double d = 0.0; for (size_t e = 0; e < p.X.a.size(); ++e) d = std::max(d, std::fabs(again.X.a[e] - p.X.a[e]));
      CHECK(d <= 1e-12);
    }
  });

  // ---------------- test_core.cpp ----------------
  run("Validate (test_core.cpp:24-87)", [] {
    validate(scalar_instance(1.0, 1.0, 0.0, 0.5));
    CHECK_THROWS(validate(scalar_instance(1.0, 1.0, 0.0, 2.0)), ErrorCode::BudgetExceedsMass);
    validate(scalar_instance(0.7, 0.9, 1.0, 0.7));
    Instance bad; bad.r = {-1.0, 0.5}; bad.c = {0.5, 0.5}; bad.C = Mat(1, 1, -2.0); bad.s = 5.0;
    CHECK(validation_report(bad).size() >= 3u);
    Instance nf = scalar_instance(1.0, 1.0, 0.0, 0.5); nf.C(0, 0) = std::numeric_limits<double>::infinity();
    CHECK_THROWS(validate(nf), ErrorCode::NonFiniteEntry);
  });
  run("FeasibilityGap (test_core.cpp:89-120)", [] {
    const Instance in = scalar_instance(1.0, 1.0, 0.0, 0.5);
    CHECK(plan_feasibility_gap(TransportPlan::from(Mat(1, 1, 0.5), in), in) == 0.0);
    CHECK_NEAR(plan_feasibility_gap(TransportPlan::from(Mat(1, 1, 1.2), in), in), 0.7, 1e-15);
    std::mt19937_64 rng(3);
    for (int rep = 0; rep < 10; ++rep) { const Instance r4 = random_instance(rng, 4); CHECK_NEAR(plan_feasibility_gap(TransportPlan::from(Mat(4, 4, 0.0), r4), r4), r4.s, 1e-15); }
  });

  std::printf("%d checks, %d failures\n", g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
