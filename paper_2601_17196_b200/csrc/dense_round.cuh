// dense_round.cuh — the reference's rounding operators on a user-supplied
// dense plan (rounding.hpp:14-77): round_pot (onto U(r, c, s)) and
// round_balanced (onto the balanced polytope). The solvers never need these
// (their plans are implicit, plan.cuh); they serve the public API.
// Row-major X; every n^2 pass is a device kernel (row sums, column sums,
// one apply pass in the reference's multiplication order
// ((X alpha) rho_i) kappa_j + coef (a_i b_j)); the O(n) scalars are host code.
#pragma once

namespace potgpu {

// row sums of ((X alpha) rs_i) cs_j (rs / cs may be null = 1)
__global__ void k_dr_rowsums(const double* X, int64_t rows, int64_t cols, double alpha, const double* rs, const double* cs,
                             double* out) {
  __shared__ double sh[32];
  for (int64_t i = blockIdx.x; i < rows; i += gridDim.x) {
    const double ri = rs ? rs[i] : 1.0;
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) {
      double x = X[i * cols + j] * alpha;
      x = x * ri;
      if (cs) x = x * cs[j];
      s += x;
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < int(blockDim.x >> 5); ++w) t += sh[w];
      out[i] = t;
    }
    __syncthreads();
  }
}

// column sums of ((X alpha) rs_i) cs_j, thread per column (coalesced rows)
__global__ void k_dr_colsums(const double* X, int64_t rows, int64_t cols, double alpha, const double* rs, const double* cs,
                             double* out) {
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < cols; j += int64_t(gridDim.x) * blockDim.x) {
    const double cj = cs ? cs[j] : 1.0;
    double s = 0.0;
    for (int64_t i = 0; i < rows; ++i) {
      double x = X[i * cols + j] * alpha;
      if (rs) x = x * rs[i];
      s += x * cj;
    }
    out[j] = s;
  }
}

// Y_ij = ((X_ij alpha) rs_i) cs_j + coef (a_i b_j)   [den != 0: + (a_i b_j) / den]
__global__ void k_dr_apply(const double* X, int64_t rows, int64_t cols, double alpha, const double* rs, const double* cs,
                           double coef, double den, const double* a, const double* b, double* Y) {
  const int64_t total = rows * cols;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = k / cols, j = k % cols;
    double x = X[k] * alpha;
    if (rs) x = x * rs[i];
    if (cs) x = x * cs[j];
    if (a) x = den != 0.0 ? x + (a[i] * b[j]) / den : x + coef * (a[i] * b[j]);
    Y[k] = x;
  }
}

struct DenseRounder {
  Context& cx;
  int64_t rows, cols;
  DevBuf<double> X, Y, v;  // v: rs, cs, a, b, rowout, colout
  DenseRounder(Context& c, int64_t r, int64_t k) : cx(c), rows(r), cols(k) {
    X.alloc(size_t(r * k));
    Y.alloc(size_t(r * k));
    v.alloc(size_t(3 * (r + k)));
  }
  ~DenseRounder() { cudaStreamSynchronize(cx.stream); }
  double* rs() { return v.p; }
  double* cs() { return v.p + rows; }
  double* a() { return v.p + rows + cols; }
  double* b() { return v.p + 2 * rows + cols; }
  double* ro() { return v.p + 2 * (rows + cols); }
  double* co() { return v.p + 2 * (rows + cols) + rows; }
  void up(double* d, const HVec& h) {
    PG_CK(cudaMemcpyAsync(d, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  }
  HVec down(const double* d, int64_t k) {
    HVec h(static_cast<size_t>(k));
    PG_CK(cudaMemcpyAsync(h.data(), d, size_t(k) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
    return h;
  }
  HVec rowsums(double alpha, bool use_rs, bool use_cs) {
    k_dr_rowsums<<<int(std::min<int64_t>(rows, 8 * cx.num_sms)), 256, 0, cx.stream>>>(X.p, rows, cols, alpha,
                                                                                     use_rs ? rs() : nullptr,
                                                                                     use_cs ? cs() : nullptr, ro());
    PG_CK(cudaGetLastError());
    return down(ro(), rows);
  }
  HVec colsums(double alpha, bool use_rs, bool use_cs) {
    k_dr_colsums<<<int(std::max<int64_t>(1, std::min<int64_t>(ceil_div(cols, 128), 8 * cx.num_sms))), 128, 0, cx.stream>>>(
        X.p, rows, cols, alpha, use_rs ? rs() : nullptr, use_cs ? cs() : nullptr, co());
    PG_CK(cudaGetLastError());
    return down(co(), cols);
  }
  void apply(double alpha, bool use_rs, bool use_cs, double coef, double den, bool use_ab) {
    k_dr_apply<<<cx.num_sms * 8, 256, 0, cx.stream>>>(X.p, rows, cols, alpha, use_rs ? rs() : nullptr,
                                                     use_cs ? cs() : nullptr, coef, den, use_ab ? a() : nullptr,
                                                     use_ab ? b() : nullptr, Y.p);
    PG_CK(cudaGetLastError());
  }
};

// round_pot (rounding.hpp:46-77); X, Y host row-major n x n.
inline void round_pot_dense(Context& cx, int64_t n, const double* Xh, const HVec& r, const HVec& c, double s, double* Yh) {
  DenseRounder d(cx, n, n);
  PG_CK(cudaMemcpyAsync(d.X.p, Xh, size_t(n * n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  const double mass = hsum(d.rowsums(1.0, false, false));
  const double alpha = mass > 0 ? std::min(1.0, s / mass) : 1.0;
  const HVec row = d.rowsums(alpha, false, false);
  HVec rho(static_cast<size_t>(n), 1.0);
  for (int64_t i = 0; i < n; ++i)
    if (row[size_t(i)] > 0) rho[size_t(i)] = std::min(1.0, r[size_t(i)] / row[size_t(i)]);
  d.up(d.rs(), rho);
  const HVec col = d.colsums(alpha, true, false);
  HVec kap(static_cast<size_t>(n), 1.0);
  for (int64_t j = 0; j < n; ++j)
    if (col[size_t(j)] > 0) kap[size_t(j)] = std::min(1.0, c[size_t(j)] / col[size_t(j)]);
  d.up(d.cs(), kap);
  const HVec rows3 = d.rowsums(alpha, true, true);
  const HVec cols3 = d.colsums(alpha, true, true);
  const double deficit = s - hsum(rows3);
  double coef = 0.0;
  bool fill = false;
  if (deficit > 0) {
    HVec a(static_cast<size_t>(n)), b(static_cast<size_t>(n));
    for (int64_t i = 0; i < n; ++i) a[size_t(i)] = std::max(r[size_t(i)] - rows3[size_t(i)], 0.0);
    for (int64_t j = 0; j < n; ++j) b[size_t(j)] = std::max(c[size_t(j)] - cols3[size_t(j)], 0.0);
    const double na = hsum(a), nb = hsum(b);
    if (na <= 0 || nb <= 0) throw Error(POTGPU_INFEASIBLE, "deficit fill has no slack mass");
    coef = deficit / (na * nb);
    d.up(d.a(), a);
    d.up(d.b(), b);
    fill = true;
  }
  d.apply(alpha, true, true, coef, 0.0, fill);
  PG_CK(cudaMemcpyAsync(Yh, d.Y.p, size_t(n * n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
  PG_CK(cudaStreamSynchronize(cx.stream));
}

// round_balanced (rounding.hpp:14-39); X, Y host row-major rows x cols.
inline void round_balanced_dense(Context& cx, int64_t rows, int64_t cols, const double* Xh, const HVec& r, const HVec& c,
                                 double* Yh) {
  const double sr = hsum(r), sc = hsum(c);
  if (std::fabs(sr - sc) > 1e-12 * std::max({1.0, sr, sc}))
    throw Error(POTGPU_UNBALANCED_MARGINALS, "marginal masses differ: " + std::to_string(sr) + " vs " + std::to_string(sc));
  DenseRounder d(cx, rows, cols);
  PG_CK(cudaMemcpyAsync(d.X.p, Xh, size_t(rows * cols) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  const HVec row = d.rowsums(1.0, false, false);
  HVec rho(static_cast<size_t>(rows), 1.0);
  for (int64_t i = 0; i < rows; ++i)
    if (row[size_t(i)] > 0) rho[size_t(i)] = std::min(1.0, r[size_t(i)] / row[size_t(i)]);
  d.up(d.rs(), rho);
  const HVec col = d.colsums(1.0, true, false);
  HVec kap(static_cast<size_t>(cols), 1.0);
  for (int64_t j = 0; j < cols; ++j)
    if (col[size_t(j)] > 0) kap[size_t(j)] = std::min(1.0, c[size_t(j)] / col[size_t(j)]);
  d.up(d.cs(), kap);
  const HVec rows2 = d.rowsums(1.0, true, true);
  const HVec cols2 = d.colsums(1.0, true, true);
  HVec er(static_cast<size_t>(rows)), ec(static_cast<size_t>(cols));
  for (int64_t i = 0; i < rows; ++i) er[size_t(i)] = r[size_t(i)] - rows2[size_t(i)];
  for (int64_t j = 0; j < cols; ++j) ec[size_t(j)] = c[size_t(j)] - cols2[size_t(j)];
  const double total = hsum(er);
  bool fill = false;
  if (total > 0) {  // (err_r err_c^T) / total, coefficient-wise (er_i ec_j) / total
    d.up(d.a(), er);
    d.up(d.b(), ec);
    fill = true;
  }
  d.apply(1.0, true, true, 0.0, fill ? total : 0.0, fill);
  PG_CK(cudaMemcpyAsync(Yh, d.Y.p, size_t(rows * cols) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
  PG_CK(cudaStreamSynchronize(cx.stream));
}

}  // namespace potgpu
