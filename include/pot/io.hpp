// pot/io.hpp — drop-in mirror of the reference's file formats
// (/root/reference/proj/include/pot/io.hpp) plus a binary instance / plan
// format for sizes where JSON is unusable.
//   trace_to_csv / write_trace_csv   io.hpp:116-135 (header contract kept)
//   Image, read_ppm / write_ppm      io.hpp:159-218 (binary P6)
//   read_xyz / write_xyz             io.hpp:220-258
//   instance JSON read / write       io.hpp:37-114 ("r", "c", "C", "s"; C flat or rows)
//   read/write_instance_bin, write_plan_bin   (new; layout documented below)
// The JSON reader is a minimal parser for the instance documents (objects,
// arrays, numbers); no external JSON library is needed.
#pragma once

#include <cctype>
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
inline std::string format_double(double value) {  // io.hpp:21-25
  char buf[32];
  std::snprintf(buf, sizeof(buf), "%.17g", value);
  return buf;
}
inline std::string read_text_file(const std::string& path) {
  std::ifstream stream(path, std::ios::binary);
  if (!stream) throw PotError(ErrorCode::IoFailure, "cannot open " + path);
  std::ostringstream out;
  out << stream.rdbuf();
  return out.str();
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
  return instance_from_json_text(detail::read_text_file(path));
}

inline void write_text_file(const std::string& path, const std::string& body) {  // io.hpp:106-110
  std::ofstream stream(path, std::ios::binary);
  if (!stream) throw PotError(ErrorCode::IoFailure, "cannot write " + path);
  stream << body;
}

inline std::string instance_to_json_text(const Instance& in) {  // io.hpp:82-94 (flat C)
  auto arr = [](const double* p, long k) {
    std::string o = "[";
    for (long i = 0; i < k; ++i) { if (i) o += ", "; o += detail::format_double(p[i]); }
    return o + "]";
  };
  std::vector<double> flat;
  for (long i = 0; i < in.C.rows(); ++i)
    for (long j = 0; j < in.C.cols(); ++j) flat.push_back(in.C(i, j));
  return "{\n  \"C\": " + arr(flat.data(), long(flat.size())) + ",\n  \"c\": " + arr(in.c.data(), in.c.size()) +
         ",\n  \"r\": " + arr(in.r.data(), in.r.size()) + ",\n  \"s\": " + detail::format_double(in.s) + "\n}\n";
}

inline void write_instance_json(const std::string& path, const Instance& in) {
  write_text_file(path, instance_to_json_text(in));
}

inline std::string trace_to_csv(const ConvergenceTrace& trace) {  // io.hpp:116-131
  std::string out = "t,E,phi,rounded_cost,elapsed_s\n";
  for (const auto& rec : trace.records) {
    out += std::to_string(rec.t);
    out += ',';
    out += detail::format_double(rec.error);
    out += ',';
    out += detail::format_double(rec.phi);
    out += ',';
    if (rec.rounded_cost) out += detail::format_double(*rec.rounded_cost);
    out += ',';
    out += detail::format_double(rec.elapsed_s);
    out += '\n';
  }
  return out;
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

// ---------------------------------------------------------------- PPM --
struct Image {  // io.hpp:159-166
  int width = 0;
  int height = 0;
  std::vector<unsigned char> rgb;  // 3 bytes per pixel, row-major
  int pixel_count() const { return width * height; }
};

inline Image read_ppm(const std::string& path) {  // io.hpp:168-210
  std::ifstream stream(path, std::ios::binary);
  if (!stream) throw PotError(ErrorCode::IoFailure, "cannot open " + path);
  std::string magic;
  stream >> magic;
  if (magic != "P6") throw PotError(ErrorCode::IoFailure, path + ": expected binary PPM (P6)");
  auto next_int = [&]() {
    while (true) {
      const int ch = stream.peek();
      if (ch == '#') {
        std::string line;
        std::getline(stream, line);
      } else if (std::isspace(ch)) {
        stream.get();
      } else {
        break;
      }
    }
    int value = 0;
    if (!(stream >> value)) throw PotError(ErrorCode::IoFailure, path + ": malformed PPM header");
    return value;
  };
  Image img;
  img.width = next_int();
  img.height = next_int();
  const int maxval = next_int();
  if (img.width <= 0 || img.height <= 0 || maxval != 255) throw PotError(ErrorCode::IoFailure, path + ": unsupported PPM header");
  stream.get();
  img.rgb.resize(static_cast<size_t>(img.width) * size_t(img.height) * 3);
  stream.read(reinterpret_cast<char*>(img.rgb.data()), std::streamsize(img.rgb.size()));
  if (stream.gcount() != std::streamsize(img.rgb.size())) throw PotError(ErrorCode::IoFailure, path + ": truncated pixel data");
  return img;
}

inline void write_ppm(const std::string& path, const Image& img) {  // io.hpp:212-218
  std::ofstream stream(path, std::ios::binary);
  if (!stream) throw PotError(ErrorCode::IoFailure, "cannot write " + path);
  stream << "P6\n" << img.width << " " << img.height << "\n255\n";
  stream.write(reinterpret_cast<const char*>(img.rgb.data()), std::streamsize(img.rgb.size()));
}

// ---------------------------------------------------------------- XYZ --
inline Matrix read_xyz(const std::string& path) {  // io.hpp:220-242
  std::ifstream stream(path);
  if (!stream) throw PotError(ErrorCode::IoFailure, "cannot open " + path);
  std::vector<double> values;
  double x = 0, y = 0, z = 0;
  while (stream >> x >> y >> z) {
    values.push_back(x);
    values.push_back(y);
    values.push_back(z);
  }
  if (values.empty()) throw PotError(ErrorCode::IoFailure, path + ": no points");
  const long n = long(values.size() / 3);
  Matrix pts(n, 3);
  for (long i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) pts(i, d) = values[size_t(3 * i + d)];
  return pts;
}

inline void write_xyz(const std::string& path, const Matrix& pts) {  // io.hpp:244-258
  if (pts.cols() != 3) throw PotError(ErrorCode::DimensionMismatch, "point cloud must be N x 3");
  std::string body;
  for (long i = 0; i < pts.rows(); ++i) {
    body += detail::format_double(pts(i, 0));
    body += ' ';
    body += detail::format_double(pts(i, 1));
    body += ' ';
    body += detail::format_double(pts(i, 2));
    body += '\n';
  }
  write_text_file(path, body);
}

}  // namespace pot
