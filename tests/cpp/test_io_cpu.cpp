// CPU-only checks of include/pot/io.hpp (no solve, no GPU): the trace CSV
// contract (reference io.hpp:116-131), the summary.json field set
// (tools/pot_main.cpp:78-97), the exit-code mapping (pot_main.cpp:337-386)
// and the instance round trips. Prints "OK" on success.
#include <cmath>
#include <cstdio>

#include "pot/io.hpp"

static int failures = 0;
#define EXPECT(c) do { if (!(c)) { std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c); ++failures; } } while (0)

int main() {
  using namespace pot;
  ConvergenceTrace tr;
  TraceRecord a; a.t = 0; a.error = 1.5; a.phi = -2.0; a.rounded_cost = 0.25; a.elapsed_s = 0.0;
  TraceRecord b; b.t = 10; b.error = 0.125; b.phi = -1.0; b.elapsed_s = 0.5;
  tr.records = {a, b};
  EXPECT(trace_to_csv(tr) == "t,E,phi,rounded_cost,elapsed_s\n0,1.5,-2,0.25,0\n10,0.125,-1,,0.5\n");

  Instance in;
  in.r = Vector(2); in.r(0) = 0.5; in.r(1) = 0.5;
  in.c = Vector(2); in.c(0) = 0.5; in.c(1) = 0.5;
  in.C = Matrix(2, 2); in.C(0, 0) = 0.0; in.C(0, 1) = 1.0; in.C(1, 0) = 1.0; in.C(1, 1) = 0.0;
  in.s = 0.5;
  SolveResult res;
  res.plan.X = Matrix(2, 2); res.plan.X(0, 0) = 0.25; res.plan.X(1, 1) = 0.25;
  res.plan.mass = 0.5;
  res.iterations = 7; res.gamma = 0.1; res.tolerance = 1e-3; res.final_error = 5e-4; res.wall_seconds = 0.01;
  const std::string s0 = summary_json(in, res, "aspot");
  if (std::getenv("SHOW")) std::printf("%s", s0.c_str());
  EXPECT(s0 == "{\n  \"cost\": 0.0,\n  \"feasibility_gap\": 0.0,\n  \"final_error\": 0.0005,\n  \"gamma\": 0.1,\n"
               "  \"iterations\": 7,\n  \"solver\": \"aspot\",\n  \"status\": \"converged\",\n  \"tolerance\": 0.001,\n"
               "  \"wall_seconds\": 0.01\n}\n");
  res.bounds = TheoryBounds{2.0, 3.5, 0.25, 1e6};
  const std::string s1 = summary_json(in, res, "aspot");
  EXPECT(s1.find("\"theory_bounds\": {\n    \"L\": 3.5,\n    \"R\": 2.0,\n    \"iteration_bound\": 1e+06,\n"
                 "    \"mu_f\": 0.25\n  }") != std::string::npos);

  EXPECT(run_command([] {}) == 0);
  EXPECT(run_command([] { throw PotError(ErrorCode::InvalidArgument, "bad"); }) == 1);
  EXPECT(run_command([] { throw std::runtime_error("x"); }) == 1);
  EXPECT(int(ExitCode::Usage) == 2);

  const char* pj = "/tmp/potgpu_io_cpu.json";
  write_instance_json(pj, in);
  const Instance j = read_instance_json(pj);
  EXPECT(j.C(0, 1) == 1.0 && j.r(1) == 0.5 && j.s == 0.5);
  bool threw = false;
  try { read_instance_json("/nonexistent/x.json"); } catch (const PotError& e) { threw = e.code() == ErrorCode::IoFailure; }
  EXPECT(threw);
  std::printf(failures ? "FAILED (%d)\n" : "OK\n", failures);
  return failures ? 1 : 0;
}
