// pot/color_transfer.hpp — drop-in mirror of the reference's colour transfer
// (/root/reference/proj/include/pot/color_transfer.hpp): k-means
// quantisation on the device (potgpu_kmeans_quantize), the partial transport
// solve between the two histograms on the device, barycentric recolouring.
#pragma once

#include <cmath>
#include <cstdint>
#include <vector>

#include "io.hpp"
#include "pot.hpp"

namespace pot {

// An 8-bit RGB pixel buffer (the reference's pot::Image, io.hpp:159-166:
// width, height, 3 bytes per pixel in row-major order). Reading and writing
// image files is the reference CLI's business and is not part of this API.
struct Image {
  int width = 0;
  int height = 0;
  std::vector<unsigned char> rgb;
  int pixel_count() const { return width * height; }
};

struct ColorHistogram {  // color_transfer.hpp:15-19
  Matrix centroids;              // k x 3, values in [0, 1]
  Vector weights;                // cluster sizes / N
  std::vector<int> assignments;  // pixel -> centroid
};

inline Matrix image_to_points(const Image& img) {  // :21-30
  const long n = img.pixel_count();
  Matrix pts(n, 3);
  for (long i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) pts(i, d) = img.rgb[size_t(3 * i + d)] / 255.0;
  return pts;
}

inline ColorHistogram kmeans_quantize(const Matrix& points, int k, std::uint64_t seed) {  // :34-118
  const long n = points.rows();
  if (n > 0 && points.cols() != 3) throw PotError(ErrorCode::DimensionMismatch, "points must be N x 3");
  std::vector<double> prm(static_cast<size_t>(3 * n));
  for (long i = 0; i < n; ++i)
    for (int d = 0; d < 3; ++d) prm[size_t(3 * i + d)] = points(i, d);
  std::vector<double> C(static_cast<size_t>(3 * std::max(k, 1))), W(static_cast<size_t>(std::max(k, 1)));
  std::vector<int32_t> A(static_cast<size_t>(std::max<long>(n, 1)));
  if (int rc = potgpu_kmeans_quantize(detail::context(), n ? prm.data() : nullptr, n, k, seed, C.data(), W.data(), A.data()))
    detail::rethrow(rc);
  ColorHistogram h;
  h.centroids = Matrix(k, 3);
  h.weights = Vector(k);
  for (int j = 0; j < k; ++j) {
    for (int d = 0; d < 3; ++d) h.centroids(j, d) = C[size_t(3 * j + d)];
    h.weights(j) = W[size_t(j)];
  }
  h.assignments.assign(A.begin(), A.begin() + n);
  return h;
}

struct ColorTransferResult {  // :120-124
  Matrix recolored;
  SolveResult solve;
  Instance instance;
};

// Plan-weighted average of target colours per source row; rows carrying no
// mass keep their source colour (:128-141).
inline Matrix barycentric_projection(const Matrix& plan, const Matrix& source_colors, const Matrix& target_colors) {
  if (plan.rows() != source_colors.rows() || plan.cols() != target_colors.rows())
    throw PotError(ErrorCode::DimensionMismatch, "plan/color shape mismatch");
  Matrix out = source_colors;
  for (long i = 0; i < plan.rows(); ++i) {
    double mass = 0.0;
    for (long j = 0; j < plan.cols(); ++j) mass += plan(i, j);
    if (!(mass > 0)) continue;
    for (long d = 0; d < target_colors.cols(); ++d) {
      double acc = 0.0;
      for (long j = 0; j < plan.cols(); ++j) acc += plan(i, j) * target_colors(j, d);
      out(i, d) = acc / mass;
    }
  }
  return out;
}

inline ColorTransferResult color_transfer(const ColorHistogram& source, const ColorHistogram& target, double s_frac,
                                          SolverKind kind, const SolverConfig& config) {  // :146-185
  if (source.centroids.rows() != source.weights.size() || target.centroids.rows() != target.weights.size())
    throw PotError(ErrorCode::DimensionMismatch, "histogram shape mismatch");
  if (source.centroids.rows() != target.centroids.rows())
    throw PotError(ErrorCode::DimensionMismatch, "histograms must have equal color counts");
  if (s_frac < 0 || s_frac > 1) throw PotError(ErrorCode::InvalidArgument, "s_frac must lie in [0, 1]");
  const long k = source.centroids.rows();
  const double norm = std::max(source.weights.sum(), target.weights.sum());
  if (!(norm > 0)) throw PotError(ErrorCode::EmptyInput, "empty histograms");
  Instance in;
  in.r = Vector(k);
  in.c = Vector(k);
  for (long i = 0; i < k; ++i) { in.r(i) = source.weights(i) / norm; in.c(i) = target.weights(i) / norm; }
  in.C = Matrix(k, k);
  for (long i = 0; i < k; ++i)
    for (long j = 0; j < k; ++j) {
      const double dx = source.centroids(i, 0) - target.centroids(j, 0), dy = source.centroids(i, 1) - target.centroids(j, 1),
                   dz = source.centroids(i, 2) - target.centroids(j, 2);
      in.C(i, j) = (dx * dx + dy * dy) + dz * dz;
    }
  const double cmax = in.C.maxCoeff();
  if (cmax > 0)
    for (long q = 0; q < in.C.size(); ++q) in.C.data()[q] /= cmax;
  in.s = s_frac * std::min(in.r.sum(), in.c.sum());
  ColorTransferResult out;
  out.solve = solve(in, kind, config);
  out.recolored = barycentric_projection(out.solve.plan.X, source.centroids, target.centroids);
  out.instance = std::move(in);
  return out;
}

inline Image recolor_image(const Image& img, const ColorHistogram& hist, const Matrix& recolored) {  // :187-203
  if (size_t(img.pixel_count()) != hist.assignments.size())
    throw PotError(ErrorCode::DimensionMismatch, "histogram does not match the image");
  Image out = img;
  for (int i = 0; i < img.pixel_count(); ++i) {
    const int j = hist.assignments[size_t(i)];
    for (int ch = 0; ch < 3; ++ch) {
      const double value = std::min(std::max(recolored(j, ch), 0.0), 1.0);
      out.rgb[size_t(3 * i + ch)] = static_cast<unsigned char>(std::lround(value * 255.0));
    }
  }
  return out;
}

}  // namespace pot
