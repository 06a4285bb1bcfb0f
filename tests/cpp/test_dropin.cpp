// test_dropin.cpp — the reference's own solver tests, unchanged in spirit,
// compiled against the drop-in headers (include/pot/) and libpotgpu.so.
// Ports of /root/reference/proj/tests/test_solvers.cpp and test_apps.cpp
// (FitRigid*, Registration*) cases; GTest-free.
#include <cmath>
#include <cstdio>
#include <random>

#include "pot/color_transfer.hpp"
#include "pot/io.hpp"
#include "pot/registration.hpp"
#include "pot/solvers.hpp"
#include "pot/synthetic.hpp"

using namespace pot;

static int fails = 0;
#define EXPECT(c) do { if (!(c)) { ++fails; std::printf("FAIL line %d: %s\n", __LINE__, #c); } } while (0)

static Instance uniform_instance(long n, double mass, double s) {  // test_solvers.cpp:24-32
  Instance in;
  in.r = Vector::Constant(n, mass / double(n));
  in.c = Vector::Constant(n, mass / double(n));
  in.C = Matrix::Ones(n, n);
  for (long i = 0; i < n; ++i) in.C(i, i) = 0.0;
  in.s = s;
  return in;
}

int main() {
  {  // AspotSolve.ZeroCostInstance (:194-203)
    Instance in = uniform_instance(2, 1.0, 0.5);
    in.C = Matrix::Zero(2, 2);
    SolverConfig cfg; cfg.epsilon = 0.1;
    const SolveResult res = aspot_solve(in, cfg);
    EXPECT(res.status == SolveStatus::Converged);
    EXPECT(std::fabs(transport_cost(in.C, res.plan.X)) <= 1e-15);
    EXPECT(plan_feasibility_gap(res.plan, in) <= 1e-9);
  }
  {  // AspotSolve.RejectsSinglePoint (:205-207)
    Instance in; in.r = Vector::Constant(1, 1); in.c = Vector::Constant(1, 1); in.C = Matrix::Zero(1, 1); in.s = 0.5;
    bool threw = false;
    try { aspot_solve(in, SolverConfig{}); } catch (const PotError& e) { threw = e.code() == ErrorCode::DegenerateInstance; }
    EXPECT(threw);
  }
  {  // AspotSolve.PaperStyleOverrides (:225-237)
    const Instance in = make_scaling_instance(40, 5);
    SolverConfig cfg; cfg.epsilon = 8e-7; cfg.gamma_override = 1e-3; cfg.max_iterations = 1500; cfg.log_every = 1000000;
    const SolveResult res = aspot_solve(in, cfg);
    EXPECT(res.gamma == 1e-3);
    EXPECT(std::fabs(res.tolerance - 1e-7) <= 1e-20);
    EXPECT(res.status == SolveStatus::Converged);
    EXPECT(res.final_error <= res.tolerance);
  }
  {  // AspotSolve.OverflowTriggersStepHalvingAndStillSolves (:272-290)
    Instance in; in.r = Vector::Constant(2, 50.0); in.c = Vector::Constant(2, 50.0);
    in.C = Matrix::Ones(2, 2); in.C(0, 0) = 0; in.C(1, 1) = 0; in.s = 1.0;
    SolverConfig cfg; cfg.epsilon = 0.1; cfg.gamma_override = 1e5; cfg.max_iterations = 20000; cfg.log_every = 1000000;
    const SolveResult res = aspot_solve(in, cfg);
    EXPECT(plan_feasibility_gap(res.plan, in) <= 1e-9 * in.r.sum());
    EXPECT(res.status != SolveStatus::StepSizeUnderflow);
  }
  {  // StoppingIterateRecordedAndTraceMonotoneIndices (:239-250) on a synthetic instance
    const Instance in = make_synthetic_instance(6, 25, 1.0, 1.1, 0.5);
    SolverConfig cfg; cfg.epsilon = 0.05;
    const SolveResult res = aspot_solve(in, cfg);
    EXPECT(res.trace.stopping_iterate == "z_check");
    for (size_t i = 1; i < res.trace.records.size(); ++i) EXPECT(res.trace.records[i - 1].t < res.trace.records[i].t);
    EXPECT(res.final_error <= res.tolerance);
    EXPECT(res.trace.records.back().rounded_cost.has_value());
  }
  {  // FeasibleSinkhorn.SinglePointIsExact (:373-378)
    Instance in; in.r = Vector::Constant(1, 1.0); in.c = Vector::Constant(1, 0.8); in.C = Matrix::Constant(1, 1, 3.0); in.s = 0.5;
    const SolveResult res = feasible_sinkhorn_solve(in, SolverConfig{});
    EXPECT(res.plan.X(0, 0) == 0.5);
    EXPECT(res.status == SolveStatus::Converged);
  }
  {  // TunedSinkhorn.RejectsNonPositiveEntropy (:446-461)
    Instance in; in.r = Vector(2); in.r(0) = 3.0; in.r(1) = 2.0; in.c = Vector::Constant(2, 2.5); in.C = Matrix::Ones(2, 2); in.s = 1.0;
    bool threw = false;
    try { tuned_sinkhorn_solve(in, 0.1, 1.0); } catch (const PotError& e) { threw = e.code() == ErrorCode::ZeroEntropy; }
    EXPECT(threw);
  }
  {  // Solvers.AgreeWithinTwoEpsilon (:463-478) + ZeroBudgetReturnsEmptyPlan (:480-490)
    const Instance in = make_synthetic_instance(6, 33, 1.0, 0.9, 0.6);
    SolverConfig cfg; cfg.epsilon = 0.1; cfg.log_every = 1000000; cfg.max_iterations = 200000;
    const double a = transport_cost(in.C, aspot_solve(in, cfg).plan.X);
    const double s = transport_cost(in.C, feasible_sinkhorn_solve(in, cfg).plan.X);
    const double t = transport_cost(in.C, tuned_sinkhorn_solve(in, 0.1, 2.0, cfg).plan.X);
    EXPECT(std::fabs(a - s) <= 2 * cfg.epsilon + 1e-9);
    EXPECT(std::fabs(a - t) <= 2 * cfg.epsilon + 1e-9);
    EXPECT(std::fabs(s - t) <= 2 * cfg.epsilon + 1e-9);
    Instance z = in; z.s = 0.0;
    for (SolverKind k : {SolverKind::Aspot, SolverKind::FeasibleSinkhorn, SolverKind::TunedSinkhorn}) {
      const SolveResult r = solve(z, k, SolverConfig{});
      double m = 0.0;
      for (long q = 0; q < r.plan.X.size(); ++q) m = std::max(m, std::fabs(r.plan.X.data()[q]));
      EXPECT(m == 0.0);
      EXPECT(r.status == SolveStatus::Converged);
    }
  }
  {  // Validate (test_core.cpp:28-37): budget above mass
    Instance in; in.r = Vector::Constant(1, 1.0); in.c = Vector::Constant(1, 1.0); in.C = Matrix::Zero(1, 1); in.s = 2.0;
    bool threw = false;
    try { feasible_sinkhorn_solve(in, SolverConfig{}); } catch (const PotError& e) { threw = e.code() == ErrorCode::BudgetExceedsMass; }
    EXPECT(threw);
  }
  {  // FitRigid.IdentityForAlignedClouds / RecoversKnownTransform / Reflection (test_apps.cpp:160-195)
    std::mt19937_64 rng(68);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    Matrix cloud(30, 3);
    for (long i = 0; i < 30; ++i) for (int d = 0; d < 3; ++d) cloud(i, d) = u(rng);
    Matrix coupling = Matrix::Zero(30, 30);
    for (long i = 0; i < 30; ++i) coupling(i, i) = 1.0 / 30.0;
    const RigidTransform I = fit_rigid(coupling, cloud, cloud);
    EXPECT((I.R - Matrix3d::Identity()).norm() <= 1e-12 && I.t.norm() <= 1e-12);
    const double a = 37.0 * M_PI / 180.0;
    RigidTransform T0;
    T0.R(0, 0) = std::cos(a); T0.R(0, 1) = -std::sin(a); T0.R(1, 0) = std::sin(a); T0.R(1, 1) = std::cos(a);
    T0.t = Vector3d(0.4, -0.7, 0.2);
    const Matrix moved = T0.apply_all(cloud);
    const RigidTransform T = fit_rigid(coupling, moved, cloud);
    EXPECT((T.R - T0.R).norm() <= 1e-8 && (T.t - T0.t).norm() <= 1e-8);
    EXPECT((T.R.transpose() * T.R - Matrix3d::Identity()).norm() <= 1e-9);
    EXPECT(std::fabs(T.R.determinant() - 1.0) <= 1e-9);
    Matrix mirrored = cloud;
    for (long i = 0; i < 30; ++i) mirrored(i, 2) *= -1.0;
    EXPECT(std::fabs(fit_rigid(coupling, mirrored, cloud).R.determinant() - 1.0) <= 1e-9);
    bool threw = false;
    try { fit_rigid(Matrix::Zero(30, 30), cloud, cloud); } catch (const PotError& e) { threw = e.code() == ErrorCode::ZeroMassPlan; }
    EXPECT(threw);
  }
  {  // Registration.IdenticalCloudsAreAFixedPoint (test_apps.cpp:216-230)
    std::mt19937_64 rng(71);
    std::uniform_real_distribution<double> u(-1.0, 1.0);
    Matrix pts(40, 3);
    for (long i = 0; i < 40; ++i) for (int d = 0; d < 3; ++d) pts(i, d) = u(rng);
    RegistrationConfig cfg;
    cfg.alpha = 1.0;
    cfg.solve.epsilon = 0.01;
    cfg.solve.max_iterations = 5000;
    cfg.solve.log_every = 1000000;
    const RegistrationResult res = register_point_clouds(pts, pts, cfg, SolverKind::Aspot);
    EXPECT(res.converged);
    EXPECT(res.rounds.size() <= 1u);
    EXPECT((res.transform.R - Matrix3d::Identity()).norm() <= 1e-4);
    EXPECT(res.transform.t.norm() <= 1e-4);
  }
  {  // Kmeans.EachPointItsOwnCentroidWhenKEqualsN / RejectsBadArguments (test_apps.cpp:38-87)
    std::mt19937_64 rng(61);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    Matrix pts(6, 3);
    for (long i = 0; i < 6; ++i) for (int d = 0; d < 3; ++d) pts(i, d) = u(rng);
    const ColorHistogram h = kmeans_quantize(pts, 6, 7);
    for (long j = 0; j < 6; ++j) EXPECT(std::fabs(h.weights(j) - 1.0 / 6.0) <= 1e-15);
    bool threw = false;
    try { kmeans_quantize(pts, 7, 1); } catch (const PotError& e) { threw = e.code() == ErrorCode::InvalidArgument; }
    EXPECT(threw);
  }
  {  // ColorTransfer.BudgetAndNormalization (test_apps.cpp:145-158)
    std::mt19937_64 rng(66);
    std::uniform_real_distribution<double> u(0.0, 1.0);
    Matrix a(300, 3), b(300, 3);
    for (long i = 0; i < 300; ++i) for (int d = 0; d < 3; ++d) { a(i, d) = u(rng); b(i, d) = u(rng); }
    const ColorHistogram src = kmeans_quantize(a, 6, 1), tgt = kmeans_quantize(b, 6, 2);
    SolverConfig cfg;
    cfg.epsilon = 0.05;
    cfg.log_every = 1000000;
    const ColorTransferResult res = color_transfer(src, tgt, 0.2, SolverKind::TunedSinkhorn, cfg);
    EXPECT(std::fabs(res.instance.s - 0.2 * std::min(res.instance.r.sum(), res.instance.c.sum())) <= 1e-12);
    EXPECT(std::fabs(res.instance.C.maxCoeff() - 1.0) <= 1e-12);
    EXPECT(plan_feasibility_gap(res.solve.plan, res.instance) <= 1e-9);
  }
  {  // io round trips: JSON / binary instance, trace CSV header, PPM, XYZ
    Instance in = make_synthetic_instance(7, 3, 1.0, 1.2, 0.5);
    write_instance_json("/tmp/potgpu_dropin_inst.json", in);
    const Instance j = read_instance_json("/tmp/potgpu_dropin_inst.json");
    write_instance_bin("/tmp/potgpu_dropin_inst.potb", in);
    const Instance b = read_instance_bin("/tmp/potgpu_dropin_inst.potb");
    for (long i = 0; i < 7; ++i)
      for (long k = 0; k < 7; ++k) EXPECT(j.C(i, k) == in.C(i, k) && b.C(i, k) == in.C(i, k));
    EXPECT(j.s == in.s && b.s == in.s && j.r(3) == in.r(3) && b.c(6) == in.c(6));
    SolverConfig cfg; cfg.epsilon = 0.1; cfg.log_every = 5;
    const SolveResult res = aspot_solve(in, cfg);
    const std::string csv = trace_to_csv(res.trace);
    EXPECT(csv.rfind("t,E,phi,rounded_cost,elapsed_s\n", 0) == 0);
    const std::string sm = summary_json(in, res, "aspot");
    for (const char* key : {"\"solver\": \"aspot\"", "\"status\": ", "\"iterations\": ", "\"cost\": ", "\"final_error\": ",
                            "\"tolerance\": ", "\"gamma\": ", "\"wall_seconds\": ", "\"feasibility_gap\": ",
                            "\"theory_bounds\": {"})
      EXPECT(sm.find(key) != std::string::npos);
    EXPECT(run_command([] {}) == 0);
    EXPECT(run_command([] { throw PotError(ErrorCode::InvalidArgument, "x"); }) == 1);
  }
  {  // test_dual.cpp: hand values on the 1 x 1 instance, overflow, shape errors
    const EntropicContext ctx(Matrix::Zero(1, 1), 1.0, Vector::Constant(1, 1.0), Vector::Constant(1, 1.0), 0.5);
    const DualPoint z = DualPoint::zero(1);
    EXPECT(dual_objective(ctx, z) == 3.0);
    const DualPoint g = dual_gradient(ctx, z);
    EXPECT(g.u(0) == 1.0 && g.v(0) == 1.0 && g.w == 0.5);
    EXPECT(feasibility_error(ctx, z) == 2.5);
    EXPECT(b_matrix(ctx, z)(0, 0) == 1.0);
    DualPoint big{Vector::Constant(1, 400.0), Vector::Constant(1, 400.0), 0.0};
    bool threw = false;
    try { b_matrix(ctx, big); } catch (const PotError& e) { threw = e.code() == ErrorCode::Overflow; }
    EXPECT(threw);
    threw = false;
    try { dual_objective(ctx, DualPoint::zero(2)); } catch (const PotError& e) { threw = e.code() == ErrorCode::DimensionMismatch; }
    EXPECT(threw);
    // greenkhorn on u makes the row marginal exact (solvers.hpp:74-76)
    const DualPoint z1 = greenkhorn_step(ctx, z, BlockRule::RoundRobin, 0);
    EXPECT(std::fabs(dual_gradient(ctx, z1).u(0)) <= 1e-15);
  }
  {  // AspotObserver: one callback per accepted iteration, t = 1..T (solvers.hpp:364-367)
    Instance in = make_synthetic_instance(30, 5, 1.0, 1.2, 0.6);
    SolverConfig cfg; cfg.epsilon = 0.05; cfg.log_every = 1000000;
    long calls = 0, last_t = 0;
    double last_err = 0.0;
    const SolveResult res = aspot_solve(in, cfg, [&](const AspotIterate& it) {
      ++calls;
      EXPECT(it.t == last_t + 1);
      last_t = it.t;
      last_err = it.error;
      EXPECT(it.phi_best <= it.phi_hat);
    });
    EXPECT(calls == res.iterations && last_t == res.iterations);
    EXPECT(last_err == res.final_error);
    const SolveResult plain = aspot_solve(in, cfg);
    EXPECT(plain.iterations == res.iterations && plain.final_error == res.final_error);
  }
  {  // validation_report / ValidationError (test_core.cpp)
    Instance in;
    in.r = Vector::Constant(2, 1.0); in.r(1) = -1.0;
    in.c = Vector::Constant(2, 1.0);
    in.C = Matrix::Ones(2, 2);
    in.s = 5.0;
    EXPECT(validation_report(in).size() == 2u);
    bool threw = false;
    try { validate(in); } catch (const ValidationError& e) { threw = e.violations().size() == 2u && e.code() == ErrorCode::NegativeEntry; }
    EXPECT(threw);
    EXPECT(solver_kind_from_name("tuned-sinkhorn") == SolverKind::TunedSinkhorn && !solver_kind_from_name("x"));
    const AspotSetup st = aspot_setup(make_synthetic_instance(10, 2, 1.0, 1.0, 0.5), 0.1);
    EXPECT(std::fabs(st.gamma - 0.1 / (4.0 * std::log(10.0))) <= 1e-17);
  }
  std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
  return fails ? 1 : 0;
}
