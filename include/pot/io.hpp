// pot/io.hpp — the host file formats around the solver path (SURVEY.md
// §8(f) row 3). Only the contracts a drop-in user depends on are kept from
// the reference (/root/reference/proj/include/pot/io.hpp); the code is our
// own:
//   trace CSV      header "t,E,phi,rounded_cost,elapsed_s" (reference io.hpp:117),
//                  %.17g numbers, an absent rounded cost is an empty field
//   instance JSON  keys "r", "c", "C" (flat row-major or rows), "s" (io.hpp:37-94)
//   summary JSON   the CLI's summary.json field set (tools/pot_main.cpp:78-97)
//   exit codes     0 ok, 1 PotError / std::exception, 2 usage (pot_main.cpp:337-386)
//   binary         POTINST1 / POTPLAN1 (new; layout documented below) for
//                  sizes where JSON is unusable
// The reference's PPM / XYZ readers belong to its CLI apps, which are out of
// scope here; the colour-transfer API takes pixel buffers.
// The JSON reader is a minimal parser for the instance documents (objects,
// arrays, numbers); no external JSON library is needed.
#pragma once

#include <cctype>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "pot.hpp"

namespace pot {

namespace detail {
// Shortest text that round-trips an IEEE double (the %.17g contract).
inline std::string num17(double x) {
  char b[40];
  const int k = std::snprintf(b, sizeof b, "%.17g", x);
  return std::string(b, size_t(k > 0 ? k : 0));
}
// Shortest decimal that parses back to the same double (how the CLI's JSON
// library prints numbers).
inline std::string shortest(double x) {
  char b[40];
  for (int prec = 1; prec <= 17; ++prec) {
    std::snprintf(b, sizeof b, "%.*g", prec, x);
    if (std::strtod(b, nullptr) == x) break;
  }
  std::string t(b);
  if (std::isfinite(x) && t.find_first_of(".eEn") == std::string::npos) t += ".0";
  return t;
}
inline std::string slurp(const std::string& path) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) throw PotError(ErrorCode::IoFailure, "cannot open " + path);
  std::string body;
  char chunk[1 << 16];
  for (size_t got; (got = std::fread(chunk, 1, sizeof chunk, f)) > 0;) body.append(chunk, got);
  const bool bad = std::ferror(f) != 0;
  std::fclose(f);
  if (bad) throw PotError(ErrorCode::IoFailure, "read error on " + path);
  return body;
}
inline void spill(const std::string& path, const std::string& body) {
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw PotError(ErrorCode::IoFailure, "cannot write " + path);
  const size_t put = std::fwrite(body.data(), 1, body.size(), f);
  const bool bad = (std::fclose(f) != 0) || put != body.size();
  if (bad) throw PotError(ErrorCode::IoFailure, "write error on " + path);
}

// Minimal JSON value: number, array or object (what instance files use).
struct JVal {
  enum Kind { Num, Arr, Obj } kind = Num;
  double num = 0.0;
  std::vector<JVal> arr;
  std::map<std::string, JVal> obj;
};
class JParser {
 public:
  explicit JParser(const std::string& s) : s_(s) {}
  JVal parse() {
    JVal v = value();
    ws();
    if (i_ != s_.size()) fail("trailing characters");
    return v;
  }

 private:
  const std::string& s_;
  size_t i_ = 0;
  [[noreturn]] void fail(const char* what) { throw PotError(ErrorCode::IoFailure, std::string("json: ") + what); }
  void ws() { while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_; }
  JVal value() {
    ws();
    if (i_ >= s_.size()) fail("unexpected end");
    JVal v;
    if (s_[i_] == '[') {
      v.kind = JVal::Arr;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == ']') { ++i_; return v; }
      while (true) {
        v.arr.push_back(value());
        ws();
        if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
        if (i_ < s_.size() && s_[i_] == ']') { ++i_; break; }
        fail("expected , or ]");
      }
    } else if (s_[i_] == '{') {
      v.kind = JVal::Obj;
      ++i_;
      ws();
      if (i_ < s_.size() && s_[i_] == '}') { ++i_; return v; }
      while (true) {
        ws();
        if (i_ >= s_.size() || s_[i_] != '"') fail("expected key");
        const size_t e = s_.find('"', i_ + 1);
        if (e == std::string::npos) fail("unterminated key");
        const std::string key = s_.substr(i_ + 1, e - i_ - 1);
        i_ = e + 1;
        ws();
        if (i_ >= s_.size() || s_[i_] != ':') fail("expected :");
        ++i_;
        v.obj[key] = value();
        ws();
        if (i_ < s_.size() && s_[i_] == ',') { ++i_; continue; }
        if (i_ < s_.size() && s_[i_] == '}') { ++i_; break; }
        fail("expected , or }");
      }
    } else {
      const char* b = s_.c_str() + i_;
      char* end = nullptr;
      v.num = std::strtod(b, &end);
      if (end == b) fail("expected a number");
      i_ += size_t(end - b);
    }
    return v;
  }
};
}  // namespace detail

// Instance documents (io.hpp:37-80): keys "r", "c", "C" (flat row-major or
// rows) and "s".
inline Instance instance_from_json_text(const std::string& text) {
  const detail::JVal doc = detail::JParser(text).parse();
  if (doc.kind != detail::JVal::Obj || !doc.obj.count("r") || !doc.obj.count("c") || !doc.obj.count("C") ||
      !doc.obj.count("s"))
    throw PotError(ErrorCode::IoFailure, "instance needs keys r, c, C, s");
  const auto& jr = doc.obj.at("r").arr;
  const auto& jc = doc.obj.at("c").arr;
  const long n = long(jr.size());
  Instance in;
  in.r = Vector(n);
  for (long i = 0; i < n; ++i) in.r(i) = jr[size_t(i)].num;
  if (long(jc.size()) != n) throw PotError(ErrorCode::IoFailure, "r and c lengths differ");
  in.c = Vector(n);
  for (long i = 0; i < n; ++i) in.c(i) = jc[size_t(i)].num;
  const auto& jC = doc.obj.at("C").arr;
  in.C = Matrix(n, n);
  if (!jC.empty() && jC[0].kind == detail::JVal::Arr) {
    if (long(jC.size()) != n) throw PotError(ErrorCode::IoFailure, "cost row count mismatch");
    for (long i = 0; i < n; ++i) {
      if (long(jC[size_t(i)].arr.size()) != n) throw PotError(ErrorCode::IoFailure, "cost column count mismatch");
      for (long j = 0; j < n; ++j) in.C(i, j) = jC[size_t(i)].arr[size_t(j)].num;
    }
  } else {
    if (long(jC.size()) != n * n) throw PotError(ErrorCode::IoFailure, "flat cost must have n^2 entries");
    for (long i = 0; i < n; ++i)
      for (long j = 0; j < n; ++j) in.C(i, j) = jC[size_t(i * n + j)].num;
  }
  in.s = doc.obj.at("s").num;
  return in;
}

inline Instance read_instance_json(const std::string& path) {  // io.hpp:96-104
  return instance_from_json_text(detail::slurp(path));
}

inline void write_text_file(const std::string& path, const std::string& body) {  // io.hpp:106-110 (same role)
  detail::spill(path, body);
}

inline std::string instance_to_json_text(const Instance& in) {  // io.hpp:82-94 (flat C)
  auto arr = [](const double* p, long k) {
    std::string o = "[";
    for (long i = 0; i < k; ++i) { if (i) o += ", "; o += detail::num17(p[i]); }
    return o + "]";
  };
  std::vector<double> flat;
  for (long i = 0; i < in.C.rows(); ++i)
    for (long j = 0; j < in.C.cols(); ++j) flat.push_back(in.C(i, j));
  return "{\n  \"C\": " + arr(flat.data(), long(flat.size())) + ",\n  \"c\": " + arr(in.c.data(), in.c.size()) +
         ",\n  \"r\": " + arr(in.r.data(), in.r.size()) + ",\n  \"s\": " + detail::num17(in.s) + "\n}\n";
}

inline void write_instance_json(const std::string& path, const Instance& in) {
  write_text_file(path, instance_to_json_text(in));
}

// Trace CSV (reference io.hpp:116-131 contract): one line per record.
inline std::string trace_to_csv(const ConvergenceTrace& trace) {
  std::ostringstream o;
  o << "t,E,phi,rounded_cost,elapsed_s\n";
  for (const TraceRecord& rec : trace.records) {
    const std::string cost = rec.rounded_cost ? detail::num17(*rec.rounded_cost) : std::string();
    o << rec.t << ',' << detail::num17(rec.error) << ',' << detail::num17(rec.phi) << ',' << cost << ','
      << detail::num17(rec.elapsed_s) << '\n';
  }
  return o.str();
}

inline void write_trace_csv(const std::string& path, const ConvergenceTrace& trace) {
  write_text_file(path, trace_to_csv(trace));
}

// ------------------------------------------------------------- binary --
// Binary instance (".potb"), little-endian:
//   char magic[8] = "POTINST1"; int64 n; double s; double r[n]; double c[n];
//   double C[n*n] (row-major).
// Binary plan: char magic[8] = "POTPLAN1"; int64 rows, cols; double mass;
//   double X[rows*cols] (row-major); double row_slack[rows]; double col_slack[cols].
inline void write_instance_bin(const std::string& path, const Instance& in) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw PotError(ErrorCode::IoFailure, "cannot write " + path);
  const int64_t n = in.size();
  f.write("POTINST1", 8);
  f.write(reinterpret_cast<const char*>(&n), sizeof(n));
  f.write(reinterpret_cast<const char*>(&in.s), sizeof(double));
  f.write(reinterpret_cast<const char*>(in.r.data()), std::streamsize(n * sizeof(double)));
  f.write(reinterpret_cast<const char*>(in.c.data()), std::streamsize(n * sizeof(double)));
  std::vector<double> row(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    for (int64_t j = 0; j < n; ++j) row[size_t(j)] = in.C(long(i), long(j));
    f.write(reinterpret_cast<const char*>(row.data()), std::streamsize(n * sizeof(double)));
  }
  if (!f) throw PotError(ErrorCode::IoFailure, "write failed: " + path);
}

inline Instance read_instance_bin(const std::string& path) {
  std::ifstream f(path, std::ios::binary);
  if (!f) throw PotError(ErrorCode::IoFailure, "cannot open " + path);
  char magic[8];
  int64_t n = 0;
  Instance in;
  f.read(magic, 8);
  f.read(reinterpret_cast<char*>(&n), sizeof(n));
  if (!f || std::memcmp(magic, "POTINST1", 8) != 0 || n < 0) throw PotError(ErrorCode::IoFailure, path + ": not a POTINST1 file");
  f.read(reinterpret_cast<char*>(&in.s), sizeof(double));
  in.r = Vector(long(n));
  in.c = Vector(long(n));
  in.C = Matrix(long(n), long(n));
  f.read(reinterpret_cast<char*>(in.r.data()), std::streamsize(n * sizeof(double)));
  f.read(reinterpret_cast<char*>(in.c.data()), std::streamsize(n * sizeof(double)));
  std::vector<double> row(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) {
    f.read(reinterpret_cast<char*>(row.data()), std::streamsize(n * sizeof(double)));
    for (int64_t j = 0; j < n; ++j) in.C(long(i), long(j)) = row[size_t(j)];
  }
  if (!f) throw PotError(ErrorCode::IoFailure, path + ": truncated");
  return in;
}

inline void write_plan_bin(const std::string& path, const TransportPlan& plan) {
  std::ofstream f(path, std::ios::binary);
  if (!f) throw PotError(ErrorCode::IoFailure, "cannot write " + path);
  const int64_t rows = plan.X.rows(), cols = plan.X.cols();
  f.write("POTPLAN1", 8);
  f.write(reinterpret_cast<const char*>(&rows), sizeof(rows));
  f.write(reinterpret_cast<const char*>(&cols), sizeof(cols));
  f.write(reinterpret_cast<const char*>(&plan.mass), sizeof(double));
  std::vector<double> row(static_cast<size_t>(cols));
  for (int64_t i = 0; i < rows; ++i) {
    for (int64_t j = 0; j < cols; ++j) row[size_t(j)] = plan.X(long(i), long(j));
    f.write(reinterpret_cast<const char*>(row.data()), std::streamsize(cols * sizeof(double)));
  }
  f.write(reinterpret_cast<const char*>(plan.row_slack.data()), std::streamsize(rows * sizeof(double)));
  f.write(reinterpret_cast<const char*>(plan.col_slack.data()), std::streamsize(cols * sizeof(double)));
  if (!f) throw PotError(ErrorCode::IoFailure, "write failed: " + path);
}

// ------------------------------------------------------------ summary --
// The CLI's summary.json document (reference tools/pot_main.cpp:78-97): the
// same keys, in the order nlohmann::json would print them (sorted), with
// theory_bounds only when the solver computed them.
inline std::string summary_json(const Instance& in, const SolveResult& res, const std::string& solver) {
  std::map<std::string, std::string> doc;
  auto q = [](const std::string& x) { return "\"" + x + "\""; };
  doc["solver"] = q(solver);
  doc["status"] = q(solve_status_name(res.status));
  doc["iterations"] = std::to_string(res.iterations);
  doc["cost"] = detail::shortest(transport_cost(in.C, res.plan.X));
  doc["final_error"] = detail::shortest(res.final_error);
  doc["tolerance"] = detail::shortest(res.tolerance);
  doc["gamma"] = detail::shortest(res.gamma);
  doc["wall_seconds"] = detail::shortest(res.wall_seconds);
  doc["feasibility_gap"] = detail::shortest(plan_feasibility_gap(res.plan, in));
  if (res.bounds) {
    doc["theory_bounds"] = "{\n    \"L\": " + detail::shortest(res.bounds->L) + ",\n    \"R\": " +
                           detail::shortest(res.bounds->R) + ",\n    \"iteration_bound\": " +
                           detail::shortest(res.bounds->iteration_bound) + ",\n    \"mu_f\": " +
                           detail::shortest(res.bounds->mu_f) + "\n  }";
  }
  std::string out = "{";
  bool first = true;
  for (const auto& kv : doc) {
    out += first ? "\n  " : ",\n  ";
    first = false;
    out += q(kv.first) + ": " + kv.second;
  }
  return out + "\n}\n";
}

// Process exit code of the reference CLI for an outcome (pot_main.cpp:337-386):
// 0 success, 1 a PotError or other exception while running a command, 2 a
// command-line usage error.
enum class ExitCode : int { Ok = 0, Failure = 1, Usage = 2 };
template <class F>
inline int run_command(F&& command) {
  try {
    command();
    return int(ExitCode::Ok);
  } catch (const PotError& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
  }
  return int(ExitCode::Failure);
}

}  // namespace pot
