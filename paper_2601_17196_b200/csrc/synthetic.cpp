// synthetic.cpp — seeded fixtures: the reference's make_synthetic_instance
// (synthetic.hpp:15-54) and the five BASELINE.json workload recipes
// (DESIGN.md §Workloads). Host code; deterministic with libstdc++'s
// mt19937_64 / uniform_real_distribution / normal_distribution.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <vector>

#include "../../include/potgpu.h"

namespace {

double ksum(const double* x, int64_t n) {
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double t = s + x[i];
    if (std::fabs(s) >= std::fabs(x[i])) c += (s - t) + x[i]; else c += (x[i] - t) + s;
    s = t;
  }
  return s + c;
}

void normalize(double* x, int64_t n, double mass) {
  const double f = mass / ksum(x, n);
  for (int64_t i = 0; i < n; ++i) x[i] *= f;
}

double max_d2(const double* X, const double* Y, int64_t n, int d) {
  double m = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      double acc = 0.0;
      for (int k = 0; k < d; ++k) { const double t = X[i * d + k] - Y[j * d + k]; acc += t * t; }
      m = std::max(m, acc);
    }
  return m;
}

}  // namespace

extern "C" {

int potgpu_make_synthetic(int64_t n, uint64_t seed, double mass_r, double mass_c, double s_frac, double* r, double* c,
                          double* C, double* s) {
  if (n < 1) return POTGPU_INVALID_ARGUMENT;
  if (!(mass_r > 0) || !(mass_c > 0)) return POTGPU_INVALID_ARGUMENT;
  if (s_frac < 0 || s_frac > 1) return POTGPU_INVALID_ARGUMENT;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0), weight(0.2, 1.0);
  std::vector<double> src(size_t(2 * n)), tgt(size_t(2 * n));
  for (int64_t i = 0; i < n; ++i) {  // synthetic.hpp:34-41 draw order
    r[i] = weight(rng);
    c[i] = weight(rng);
    src[size_t(2 * i)] = unit(rng); src[size_t(2 * i + 1)] = unit(rng);
    tgt[size_t(2 * i)] = unit(rng); tgt[size_t(2 * i + 1)] = unit(rng);
  }
  normalize(r, n, mass_r);
  normalize(c, n, mass_c);
  double cmax = 0.0;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t j = 0; j < n; ++j) {
      const double dx = src[size_t(2 * i)] - tgt[size_t(2 * j)], dy = src[size_t(2 * i + 1)] - tgt[size_t(2 * j + 1)];
      const double v = dx * dx + dy * dy;
      C[i * n + j] = v;
      cmax = std::max(cmax, v);
    }
  if (cmax > 0)
    for (int64_t k = 0; k < n * n; ++k) C[k] /= cmax;
  *s = s_frac * std::min(ksum(r, n), ksum(c, n));
  return 0;
}

// config_id 1..5 as in BASELINE.json configs[0..4]; points are n x d
// row-major (X: rows / sources, Y: columns / targets); cost_scale = 1/max
// |x - y|^2 (computed here for n <= 20000, else 0 = "derive on the device").
int potgpu_make_config(int config_id, int64_t n, uint64_t seed, double* r, double* c, double* X, double* Y, int* d,
                       double* s, double* cost_scale) {
  if (n < 2) return POTGPU_INVALID_ARGUMENT;
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  std::normal_distribution<double> normal(0.0, 1.0);
  switch (config_id) {
    case 1: {  // X, Y ~ U[0,1]^2; r, c ~ U(0.1, 1) -> masses 1.0 / 1.2; s = 0.8
      *d = 2;
      for (int64_t i = 0; i < 2 * n; ++i) X[i] = unit(rng);
      for (int64_t i = 0; i < 2 * n; ++i) Y[i] = unit(rng);
      std::uniform_real_distribution<double> w(0.1, 1.0);
      for (int64_t i = 0; i < n; ++i) r[i] = w(rng);
      for (int64_t i = 0; i < n; ++i) c[i] = w(rng);
      normalize(r, n, 1.0);
      normalize(c, n, 1.2);
      *s = 0.8;
      break;
    }
    case 2: {  // colours: 8-component GMMs in [0,1]^3 (sigma 0.08, clipped); masses 1.0 / 1.1; s = 0.9
      *d = 3;
      std::uniform_real_distribution<double> mu(0.15, 0.85);
      std::uniform_int_distribution<int> comp(0, 7);
      for (double* P : {X, Y}) {
        double means[8][3];
        for (auto& m : means) for (double& e : m) e = mu(rng);
        for (int64_t i = 0; i < n; ++i) {
          const int k = comp(rng);
          for (int q = 0; q < 3; ++q) P[i * 3 + q] = std::min(1.0, std::max(0.0, means[k][q] + 0.08 * normal(rng)));
        }
      }
      for (int64_t i = 0; i < n; ++i) { r[i] = 1.0 / double(n); c[i] = 1.1 / double(n); }
      *s = 0.9;
      break;
    }
    case 3: {  // registration: T ~ U[-1,1]^3 (rows); source = R T + t + N(0, 0.01^2), 10% outliers in [-2,2]^3
      *d = 3;
      for (int64_t i = 0; i < 3 * n; ++i) X[i] = 2.0 * unit(rng) - 1.0;
      double q[4];
      double qn = 0.0;
      for (double& e : q) { e = normal(rng); qn += e * e; }
      qn = std::sqrt(qn);
      for (double& e : q) e /= qn;
      const double a = q[0], b = q[1], cq = q[2], dq = q[3];
      const double R[3][3] = {{a * a + b * b - cq * cq - dq * dq, 2 * (b * cq - a * dq), 2 * (b * dq + a * cq)},
                              {2 * (b * cq + a * dq), a * a - b * b + cq * cq - dq * dq, 2 * (cq * dq - a * b)},
                              {2 * (b * dq - a * cq), 2 * (cq * dq + a * b), a * a - b * b - cq * cq + dq * dq}};
      double t[3], tn = 0.0;
      for (double& e : t) { e = normal(rng); tn += e * e; }
      tn = std::sqrt(tn);
      const double rad = 0.2 * std::cbrt(unit(rng));
      for (double& e : t) e = e / tn * rad;
      for (int64_t i = 0; i < n; ++i)
        for (int k = 0; k < 3; ++k) {
          double v = t[k];
          for (int m = 0; m < 3; ++m) v += R[k][m] * X[i * 3 + m];
          Y[i * 3 + k] = v + 0.01 * normal(rng);
        }
      std::vector<int64_t> idx(static_cast<size_t>(n));
      for (int64_t i = 0; i < n; ++i) idx[size_t(i)] = i;
      const int64_t n_out = n / 10;
      for (int64_t k = 0; k < n_out; ++k) {  // partial Fisher-Yates
        std::uniform_int_distribution<int64_t> pick(k, n - 1);
        std::swap(idx[size_t(k)], idx[size_t(pick(rng))]);
        for (int m = 0; m < 3; ++m) Y[idx[size_t(k)] * 3 + m] = 4.0 * unit(rng) - 2.0;
      }
      for (int64_t i = 0; i < n; ++i) { r[i] = 1.0 / double(n); c[i] = 1.0 / double(n); }
      *s = 0.9;
      break;
    }
    case 4: {  // X, Y ~ N(0, I3), Y += 0.5 e1; r, c ~ Dirichlet(1) -> masses 1.0 / 1.3; s = 0.95
      *d = 3;
      for (int64_t i = 0; i < 3 * n; ++i) X[i] = normal(rng);
      for (int64_t i = 0; i < 3 * n; ++i) Y[i] = normal(rng) + ((i % 3) == 0 ? 0.5 : 0.0);
      for (int64_t i = 0; i < n; ++i) r[i] = -std::log(1.0 - unit(rng));
      for (int64_t i = 0; i < n; ++i) c[i] = -std::log(1.0 - unit(rng));
      normalize(r, n, 1.0);
      normalize(c, n, 1.3);
      *s = 0.95;
      break;
    }
    case 5: {  // one batched problem: U[0,1]^3 points, U(0.2,1) weights, masses U(1.0, 1.5), s = 0.9 min mass
      *d = 3;
      std::uniform_real_distribution<double> weight(0.2, 1.0), mass(1.0, 1.5);
      for (int64_t i = 0; i < 3 * n; ++i) X[i] = unit(rng);
      for (int64_t i = 0; i < 3 * n; ++i) Y[i] = unit(rng);
      for (int64_t i = 0; i < n; ++i) { r[i] = weight(rng); c[i] = weight(rng); }
      const double mr = mass(rng), mc = mass(rng);
      normalize(r, n, mr);
      normalize(c, n, mc);
      *s = 0.9 * std::min(ksum(r, n), ksum(c, n));
      break;
    }
    default:
      return POTGPU_INVALID_ARGUMENT;
  }
  *cost_scale = 0.0;
  if (n <= 20000) {
    const double m = max_d2(X, Y, n, *d);
    *cost_scale = m > 0 ? 1.0 / m : 1.0;
  }
  return 0;
}

}  // extern "C"
