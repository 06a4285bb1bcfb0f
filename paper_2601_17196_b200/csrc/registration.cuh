// registration.cuh — rigid point-cloud registration driven by partial
// transport (reference registration.hpp:13-199).
//
// Per round (register_point_clouds, registration.hpp:127-199):
//   current = T(moving)                             host, O(n)
//   C = |ref_i - current_j|^2 / cmax, padded = 1    device kernels (fp64
//                                                   coordinates, side x side)
//   solve(C, gamma_override = gamma)                the device sessions
//   fit_rigid(plan block, ref, current)             plan row / column sums
//       from the rounding, z_j = sum_i X_ij xh_i    device pass over the
//       implicit plan (plan.cuh k_plan_moments); 3x3 cross-covariance and
//       its SVD on the host
//   compose, delta, record, anneal gamma
// The dense plan is never materialised.
#pragma once

#include <array>

namespace potgpu {

using Mat3 = std::array<double, 9>;  // row-major
using Vec3 = std::array<double, 3>;

inline Mat3 mat3_identity() { return Mat3{1, 0, 0, 0, 1, 0, 0, 0, 1}; }

inline Mat3 mat3_mul(const Mat3& a, const Mat3& b) {  // (a b)_ij = sum_k a_ik b_kj, k in order
  Mat3 o{};
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) o[3 * i + j] = (a[3 * i] * b[j] + a[3 * i + 1] * b[3 + j]) + a[3 * i + 2] * b[6 + j];
  return o;
}

inline Vec3 mat3_apply(const Mat3& a, const Vec3& x) {
  Vec3 o{};
  for (int i = 0; i < 3; ++i) o[i] = (a[3 * i] * x[0] + a[3 * i + 1] * x[1]) + a[3 * i + 2] * x[2];
  return o;
}

inline double mat3_det(const Mat3& a) {
  return a[0] * (a[4] * a[8] - a[5] * a[7]) - a[1] * (a[3] * a[8] - a[5] * a[6]) + a[2] * (a[3] * a[7] - a[4] * a[6]);
}

// SVD of a 3x3 matrix by one-sided (Hestenes) Jacobi: A V = U diag(sigma),
// sigma descending. U's third column is completed as u0 x u1 when sigma_2
// vanishes (the determinant-corrected polar factor below does not depend on
// that choice).
inline void svd3(const Mat3& A, Mat3& U, Vec3& sigma, Mat3& V) {
  double b[3][3], v[3][3];  // columns
  for (int k = 0; k < 3; ++k)
    for (int r = 0; r < 3; ++r) {
      b[k][r] = A[3 * r + k];
      v[k][r] = r == k ? 1.0 : 0.0;
    }
  for (int sweep = 0; sweep < 60; ++sweep) {
    double off = 0.0;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        double al = 0, be = 0, ga = 0;
        for (int r = 0; r < 3; ++r) {
          al += b[p][r] * b[p][r];
          be += b[q][r] * b[q][r];
          ga += b[p][r] * b[q][r];
        }
        if (ga == 0.0 || std::fabs(ga) <= 1e-300) continue;
        off = std::max(off, std::fabs(ga) / std::sqrt(std::max(al * be, 1e-300)));
        const double zeta = (be - al) / (2.0 * ga);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        for (int r = 0; r < 3; ++r) {
          const double bp = b[p][r], bq = b[q][r];
          b[p][r] = c * bp - s * bq;
          b[q][r] = s * bp + c * bq;
          const double vp = v[p][r], vq = v[q][r];
          v[p][r] = c * vp - s * vq;
          v[q][r] = s * vp + c * vq;
        }
      }
    if (off < 1e-15) break;
  }
  double sg[3];
  for (int k = 0; k < 3; ++k) sg[k] = std::sqrt((b[k][0] * b[k][0] + b[k][1] * b[k][1]) + b[k][2] * b[k][2]);
  int ord[3] = {0, 1, 2};
  std::sort(ord, ord + 3, [&](int x, int y) { return sg[x] > sg[y]; });
  double u[3][3];
  for (int k = 0; k < 3; ++k) {
    const int o = ord[k];
    sigma[k] = sg[o];
    for (int r = 0; r < 3; ++r) {
      V[3 * r + k] = v[o][r];
      u[k][r] = sg[o] > 0 ? b[o][r] / sg[o] : 0.0;
    }
  }
  if (!(sigma[2] > 1e-14 * std::max(sigma[0], 1e-300))) {  // complete a proper basis
    u[2][0] = u[0][1] * u[1][2] - u[0][2] * u[1][1];
    u[2][1] = u[0][2] * u[1][0] - u[0][0] * u[1][2];
    u[2][2] = u[0][0] * u[1][1] - u[0][1] * u[1][0];
  }
  for (int k = 0; k < 3; ++k)
    for (int r = 0; r < 3; ++r) U[3 * r + k] = u[k][r];
}

struct Rigid {
  Mat3 R = mat3_identity();
  Vec3 t{0, 0, 0};
};

// RigidTransform::compose (registration.hpp:27-32): (a o b)(y) = a(b(y)).
inline Rigid rigid_compose(const Rigid& a, const Rigid& b) {
  Rigid o;
  o.R = mat3_mul(a.R, b.R);
  const Vec3 rt = mat3_apply(a.R, b.t);
  for (int k = 0; k < 3; ++k) o.t[k] = rt[k] + a.t[k];
  return o;
}

// fit_rigid's tail (registration.hpp:52-70) from the plan-weighted means and
// the centred cross-covariance.
inline Rigid rigid_from_cov(const Mat3& cov, const Vec3& mean_x, const Vec3& mean_y) {
  Mat3 U, V;
  Vec3 sg;
  svd3(cov, U, sg, V);
  if (!(sg[1] > 1e-12 * std::max(sg[0], 1e-300)))
    throw Error(POTGPU_DEGENERATE_SVD, "cross-covariance has rank < 2; rotation is not determined");
  Mat3 Vt;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Vt[3 * i + j] = V[3 * j + i];
  const double orient = mat3_det(mat3_mul(U, Vt)) > 0 ? 1.0 : -1.0;
  Mat3 UD = U;
  for (int r = 0; r < 3; ++r) UD[3 * r + 2] *= orient;
  Rigid out;
  out.R = mat3_mul(UD, Vt);
  const Vec3 rm = mat3_apply(out.R, mean_y);
  for (int k = 0; k < 3; ++k) out.t[k] = mean_x[k] - rm[k];
  return out;
}

// fit_rigid from row sums a (m), column sums b (n) and moments z_j = sum_i
// pi_ij xh_i (n x 3) of the coupling.
inline Rigid fit_rigid_from(const HVec& a, const HVec& b, const double* x, int64_t m, const double* y, int64_t n,
                            const std::function<HVec(const HVec& xh)>& moments) {
  const double mass = hsum(a);
  if (!(mass > 0)) throw Error(POTGPU_ZERO_MASS_PLAN, "coupling carries no mass");
  Vec3 mx{0, 0, 0}, my{0, 0, 0};
  for (int d = 0; d < 3; ++d) {
    HVec t1(static_cast<size_t>(m)), t2(static_cast<size_t>(n));
    for (int64_t i = 0; i < m; ++i) t1[size_t(i)] = x[3 * i + d] * a[size_t(i)];
    for (int64_t j = 0; j < n; ++j) t2[size_t(j)] = y[3 * j + d] * b[size_t(j)];
    mx[d] = hsum(t1) / mass;
    my[d] = hsum(t2) / mass;
  }
  HVec xh(static_cast<size_t>(3 * m));
  for (int64_t i = 0; i < m; ++i)
    for (int d = 0; d < 3; ++d) xh[size_t(3 * i + d)] = x[3 * i + d] - mx[d];
  const HVec z = moments(xh);  // n x 3
  Mat3 cov{};
  for (int d = 0; d < 3; ++d)
    for (int e = 0; e < 3; ++e) {
      HVec t(static_cast<size_t>(n));
      for (int64_t j = 0; j < n; ++j) t[size_t(j)] = z[size_t(3 * j + d)] * (y[3 * j + e] - my[e]);
      cov[3 * d + e] = hsum(t);
    }
  return rigid_from_cov(cov, mx, my);
}

// ------------------------------------------------------------- kernels --
__global__ void k_reg_d2max(const double* ref, const double* cur, int64_t m, int64_t n, unsigned long long* out) {
  unsigned long long mx = 0;
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x)
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
      const double dx = ref[3 * i] - cur[3 * j], dy = ref[3 * i + 1] - cur[3 * j + 1], dz = ref[3 * i + 2] - cur[3 * j + 2];
      const double d2 = ((dx * dx) + dy * dy) + dz * dz;
      mx = max(mx, (unsigned long long)__double_as_longlong(d2));
    }
  atomicMax(out, mx);
}

// C_ij = |ref_i - cur_j|^2 / cmax on the m x n block, 1 on the padding
// (registration.hpp:156-166), 0 in the row-pitch padding columns.
__global__ void k_reg_cost(const double* ref, const double* cur, int64_t m, int64_t n, int64_t side, int64_t ld, double cmax,
                           double* C64, float* C32) {
  const int64_t total = side * ld;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = k / ld, j = k % ld;
    double c = 0.0;
    if (j < side) {
      c = 1.0;
      if (i < m && j < n) {
        const double dx = ref[3 * i] - cur[3 * j], dy = ref[3 * i + 1] - cur[3 * j + 1], dz = ref[3 * i + 2] - cur[3 * j + 2];
        c = (((dx * dx) + dy * dy) + dz * dz) / cmax;
      }
    }
    if (C64) C64[k] = c;
    if (C32) C32[k] = float(c);
  }
}

// Dense coupling reductions for fit_rigid on a user matrix: row sums, column
// sums and z_j = sum_i pi_ij xh_i, thread per column (fixed order).
__global__ void k_dense_colmoments(const double* pi, int64_t m, int64_t n, const double* xh, double* colsum, double* z) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
    double s = 0, z0 = 0, z1 = 0, z2 = 0;
    for (int64_t i = 0; i < m; ++i) {
      const double p = pi[i * n + j];
      s += p;
      if (xh) {
        z0 += p * xh[3 * i];
        z1 += p * xh[3 * i + 1];
        z2 += p * xh[3 * i + 2];
      }
    }
    if (colsum) colsum[j] = s;
    if (z) { z[3 * j] = z0; z[3 * j + 1] = z1; z[3 * j + 2] = z2; }
  }
}

__global__ void k_dense_rowsums(const double* pi, int64_t m, int64_t n, double* rowsum) {
  for (int64_t i = blockIdx.x; i < m; i += gridDim.x) {
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s += pi[i * n + j];
    s = warp_sum(s);
    __shared__ double sh[32];
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) t += sh[w];
      rowsum[i] = t;
    }
    __syncthreads();
  }
}

struct RegRecord {
  int round;
  int64_t inner, accumulated;
  double cost, increment, gamma;
};

}  // namespace potgpu
