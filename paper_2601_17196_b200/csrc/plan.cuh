// plan.cuh — the output stage without materialising the plan.
//
// Every plan the reference returns is a rounding of B(z) (rounding.hpp:14-77,
// extend.hpp:48-60), which keeps the form
//     X = diag(P) B(z) diag(Q) + sum_k a_k b_k^T        (K <= 2 rank-1 terms)
// over the n x n block. The O(n) scaling logic of round_pot / round_balanced
// runs on the host in the reference's order; every n^2 reduction it needs
// (row / column sums of diag(P) B diag(Q), <C, X>, the dense X on request)
// is a weighted sweep on the device.
#pragma once

#include "engine.cuh"

namespace potgpu {

// Row sums (rows) and column sums (cols) of the fp64/fp32 sweep partials,
// with the fp32 row-partial offset (u_i + lu_i + w) log2 e.
__global__ void __launch_bounds__(kVecThreads) k_sum_partials(const double* rowp, int64_t nstrips, const double* colp,
                                                             int64_t nrb, int pfmt, Slot z, const double* lu,
                                                             const double* rowshift, double* row, double* col,
                                                             const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int64_t n = z.n;
  const double w = *z.w();
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double a2 = ((z.u()[i] + (lu ? lu[i] : 0.0)) + w) * kLog2e;
    if (rowshift) a2 = a2 + rowshift[i];
    double rr = 0.0, cc = 0.0;
    for (int64_t s = 0; s < nstrips; ++s) rr += partial_value(rowp, i * nstrips + s, pfmt, a2);
    for (int64_t s = 0; s < nrb; ++s) cc += partial_value(colp, i * nrb + s, pfmt);
    row[i] = rr;  // (output stage only: fp64 exp2 per partial is fine here)
    col[i] = cc;
  }
}

struct PlanTermsDev {
  const double* P; const double* Q;
  const double* a0; const double* b0;  // may be null
  const double* a1; const double* b1;  // may be null
};

// <C, X> (core.hpp:199-204) with X_ij = (B_ij P_i) Q_j + a0_i b0_j + a1_i b1_j,
// B_ij = exp(((logK_ij + u_i) + v_j) + w) with the Eigen clamp; optionally
// writes X (row-major, n x n).
template <class E, bool MATERIALIZE>
__global__ void __launch_bounds__(kThreads) k_plan_cost(E el, Slot z, PlanTermsDev t, int64_t row_lo, int64_t row_hi,
                                                        int rows_per_cta, double* partial, double* Xout) {
  const int64_t n = z.n;
  const int64_t j = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  const double w = *z.w();
  double acc = 0.0;
  if (j < n) {
    const double vj = z.v()[j], qj = t.Q[j];
    const double b0 = t.b0 ? t.b0[j] : 0.0, b1 = t.b1 ? t.b1[j] : 0.0;
    const int64_t r0 = row_lo + int64_t(blockIdx.y) * rows_per_cta, r1 = min(row_hi, r0 + rows_per_cta);
    for (int64_t i = r0; i < r1; ++i) {
      const double e = ((el.logk(i, j) + z.u()[i]) + vj) + w;
      const double B = exp(fmin(fmax(e, kExpLo), kExpHi));
      double x = (B * t.P[i]) * qj;
      if (t.a0) x += t.a0[i] * b0;
      if (t.a1) x += t.a1[i] * b1;
      acc += el.cost(i, j) * x;
      if (MATERIALIZE) Xout[i * n + j] = x;
    }
  }
  __shared__ double sh[kThreads];
  sh[threadIdx.x] = acc;
  __syncthreads();
  for (int stride = kThreads / 2; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride) sh[threadIdx.x] += sh[threadIdx.x + stride];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = sh[0];
}

// Plan moments for the weighted Procrustes fit (registration.hpp:40-58):
// z_j = sum_i X_ij xh_i (3-vectors, xh = centred first-cloud points, 0 on
// padded rows), thread per column, fixed-order partials per row block.
template <class E>
__global__ void __launch_bounds__(kThreads) k_plan_moments(E el, Slot z, PlanTermsDev t, const double* xh, int rows_per_cta,
                                                           double* part) {
  const int64_t n = z.n;
  const int64_t j = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  if (j >= n) return;
  const double w = *z.w();
  const double vj = z.v()[j], qj = t.Q[j];
  const double b0 = t.b0 ? t.b0[j] : 0.0, b1 = t.b1 ? t.b1[j] : 0.0;
  const int64_t r0 = int64_t(blockIdx.y) * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
  double m0 = 0.0, m1 = 0.0, m2 = 0.0;
  for (int64_t i = r0; i < r1; ++i) {
    const double e = ((el.logk(i, j) + z.u()[i]) + vj) + w;
    const double B = exp(fmin(fmax(e, kExpLo), kExpHi));
    double x = (B * t.P[i]) * qj;
    if (t.a0) x += t.a0[i] * b0;
    if (t.a1) x += t.a1[i] * b1;
    m0 += x * xh[3 * i];
    m1 += x * xh[3 * i + 1];
    m2 += x * xh[3 * i + 2];
  }
  double* o = part + (int64_t(blockIdx.y) * n + j) * 3;
  o[0] = m0; o[1] = m1; o[2] = m2;
}

__global__ void k_sum_moment_parts(const double* part, int64_t nrb, int64_t n, double* out) {
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < 3 * n; k += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int64_t b = 0; b < nrb; ++b) s += part[b * 3 * n + k];
    out[k] = s;
  }
}

// ------------------------------------------------------------------------
// fp32 output stage: round_pot's final row sums and <C, X> in ONE pass over
// the plan (rounding.hpp:57-77 + core.hpp:199-204). For the final plan
//   X = diag(Pf) B diag(Qf) + a0 b0^T + a1 b1^T,  Pf = (alpha rho) P0, Qf = Q0 kap
// every n^2 quantity the output stage needs is a per-row sum over the
// weights known before the pass (lu = log P0, lv = log(Q0 kap), b0, b1):
//   R_i  = sum_j P0_i B_ij Qf_j          (the final row sums)
//   W_i  = sum_j C_ij P0_i B_ij Qf_j     (<C, X> = sum_i alpha rho_i W_i + ...)
//   K0_i = sum_j C_ij b0_j,  K1_i = sum_j C_ij b1_j   (the rank-1 terms)
// Exponents as the fp32 sweeps (log2 units relative to each row segment's
// exact max, the row potential added back in fp64 by k_rowcost_reduce), the
// cost c_ij in fp32: the stored C, or |x_i - y_j|^2 of the raw coordinates
// (cost_scale applied in fp64 by the reduce). The dense plan (materialize)
// and fp64 problems keep k_plan_cost.
struct RowCostArgs {
  int64_t n, row_lo, row_hi;
  int rows_per_cta;
  const double* u; const double* v; const double* w;
  const double* lv;                  // log column weights (may be null)
  const double* b0; const double* b1;  // rank-1 column factors (may be null)
  float g;                           // log2 e / gamma (dense C) or log2 e cost_scale / gamma (points)
  float4* part;                      // [row][strip]: (R, W) relative to 2^m, (K0, K1)
  float* pm;                         // [row][strip]: m
  const int* gate;                   // null: always
};

template <bool POINTS>
__global__ void __launch_bounds__(kThreads, 2) k_rowcost_f32(const float* __restrict__ C, int64_t ld,
                                                             const float4* __restrict__ X, const float4* __restrict__ Y,
                                                             RowCostArgs a) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStripCols32;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  // the rank-1 column factors in shared memory (registers hold B_j and y_j)
  __shared__ float2 s_c0[kStripCols32 / 2], s_c1[kStripCols32 / 2];
  for (int k = threadIdx.x; k < kStripCols32; k += kThreads) {
    const int64_t j = j0 + k;
    reinterpret_cast<float*>(s_c0)[k] = (j < n && a.b0) ? float(a.b0[j]) : 0.f;
    reinterpret_cast<float*>(s_c1)[k] = (j < n && a.b1) ? float(a.b1[j]) : 0.f;
  }
  float2 Bj[kPairs];
  float2 yx[kPairs], yy[kPairs], yz[kPairs];
#pragma unroll
  for (int q = 0; q < kPairs; ++q) {
    float b[2];
    float4 y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;  // padding column: exp2(-inf) = 0
      y[h] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
        vv = vv * kLog2e;
        if (POINTS) y[h] = Y[j];
      }
      b[h] = float(vv);
    }
    Bj[q] = make_float2(b[0], b[1]);
    yx[q] = make_float2(y[0].x, y[1].x);
    yy[q] = make_float2(y[0].y, y[1].y);
    yz[q] = make_float2(y[0].z, y[1].z);
  }
  __syncthreads();
  const bool has_b1 = a.b1 != nullptr;
  const float2 G = make_float2(-a.g, -a.g);
  const int64_t ldp = gridDim.x;
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    float2 c[kPairs];
    if constexpr (POINTS) {
      const float4 xi = X[i];
      const float2 px = make_float2(-xi.x, -xi.x), py = make_float2(-xi.y, -xi.y), pz = make_float2(-xi.z, -xi.z);
#pragma unroll
      for (int q = 0; q < kPairs; ++q) {
        const float2 dx = __fadd2_rn(yx[q], px), dy = __fadd2_rn(yy[q], py), dz = __fadd2_rn(yz[q], pz);
        c[q] = __ffma2_rn(dz, dz, __ffma2_rn(dy, dy, __fmul2_rn(dx, dx)));
      }
    } else {
      const float4* rowp = reinterpret_cast<const float4*>(C + i * ld + j0) + lane;
#pragma unroll
      for (int k = 0; k < kPairs / 2; ++k) {
        const float4 f = __ldcs(rowp + 32 * k);
        c[2 * k] = make_float2(f.x, f.y);
        c[2 * k + 1] = make_float2(f.z, f.w);
      }
    }
    float2 t[kPairs];
#pragma unroll
    for (int q = 0; q < kPairs; ++q) t[q] = __ffma2_rn(G, c[q], Bj[q]);
    float m = tree_max2<kPairs>(t);
    m = warp_maxf(m);
    const float ms = (m == -INFINITY) ? 0.f : m;
    const float2 M2 = make_float2(-ms, -ms);
    float2 R = make_float2(0.f, 0.f), Wc = R, K0 = R, K1 = R;
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      const float2 d = __fadd2_rn(t[q], M2);
      const float2 p = make_float2(ex2f(d.x), ex2f(d.y));
      R = __fadd2_rn(R, p);
      Wc = __ffma2_rn(c[q], p, Wc);
      const int cc = 2 * lane + 64 * (q >> 1) + (q & 1);  // float2 index of f32_col(0, lane, q, 0)
      K0 = __ffma2_rn(c[q], s_c0[cc], K0);
      if (has_b1) K1 = __ffma2_rn(c[q], s_c1[cc], K1);
    }
    float4 o = make_float4(R.x + R.y, Wc.x + Wc.y, K0.x + K0.y, K1.x + K1.y);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      o.x += __shfl_xor_sync(0xffffffffu, o.x, off);
      o.y += __shfl_xor_sync(0xffffffffu, o.y, off);
      o.z += __shfl_xor_sync(0xffffffffu, o.z, off);
      o.w += __shfl_xor_sync(0xffffffffu, o.w, off);
    }
    if (lane == 0) {
      a.part[i * ldp + blockIdx.x] = o;
      a.pm[i * ldp + blockIdx.x] = ms;
    }
  }
}

// The same pass for on-the-fly points with the exponent formed in fp64:
// c_ij = |x_i - y_j|^2 is exact-ish in fp64 from the fp32 coordinates and
// t = (v_j + lv_j) log2 e - g c_ij rounds once, near the row max, when it
// goes to fp32 — the fp32 difference form loses ~g c eps (1e-5 relative
// per entry at C3) in c alone. 8 columns per lane (256 per warp), fp64
// column coordinates and constants in registers; the cost weights, sums and
// exponentials in fp32 (B200 runs FP64 at half the FP32 FMA rate: ~7 DFMA
// per entry keep this an output-stage pass of ~0.2 ms at n = 16384).
constexpr int kRcCols = 8;  // columns per lane
constexpr int kRcStrip = 32 * kRcCols;

template <bool B1>  // a second rank-1 column factor (Sinkhorn plans); without it one sum fewer per row
__global__ void __launch_bounds__(kThreads, 2) k_rowcost_pts64(const float4* __restrict__ X, const float4* __restrict__ Y,
                                                               double g, RowCostArgs a) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kRcStrip;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  // expanded fp64 exponent: t = (v_j log2e - g |y_j|^2) + (2 g y_j) . x_i - g |x_i|^2,
  // every term exact to ~1e-16 of its magnitude, so t rounds once (to fp32)
  // near the row max; the fp32 cost weight from the fp32 coordinates in smem
  __shared__ float s_c0[kRcStrip], s_c1[kRcStrip];
  __shared__ float4 s_y[kRcStrip];
  for (int k = threadIdx.x; k < kRcStrip; k += kThreads) {
    const int64_t j = j0 + k;
    s_c0[k] = (j < n && a.b0) ? float(a.b0[j]) : 0.f;
    s_c1[k] = (j < n && a.b1) ? float(a.b1[j]) : 0.f;
    s_y[k] = j < n ? Y[j] : make_float4(0.f, 0.f, 0.f, 0.f);
  }
  double Bq[kRcCols], gx[kRcCols], gy[kRcCols], gz[kRcCols];
#pragma unroll
  for (int k = 0; k < kRcCols; ++k) {
    const int64_t j = j0 + lane + 32 * k;
    double vv = -INFINITY;  // padding column: exp2(-inf) = 0
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < n) {
      vv = a.v[j];
      if (a.lv) vv = vv + a.lv[j];
      vv = vv * kLog2e;
      y = Y[j];
    }
    const double yx = y.x, yy = y.y, yz = y.z;
    Bq[k] = vv - g * fma(yz, yz, fma(yy, yy, yx * yx));
    gx[k] = 2.0 * g * yx; gy[k] = 2.0 * g * yy; gz[k] = 2.0 * g * yz;
  }
  __syncthreads();
  const int64_t ldp = gridDim.x;
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    const float4 xi = X[i];
    const double xx = xi.x, xy = xi.y, xz = xi.z;
    const double ax = g * fma(xz, xz, fma(xy, xy, xx * xx));
    float t[kRcCols], cf[kRcCols];
#pragma unroll
    for (int k = 0; k < kRcCols; ++k) {
      t[k] = __double2float_rn(fma(xz, gz[k], fma(xy, gy[k], fma(xx, gx[k], Bq[k]))) - ax);
      const float4 y = s_y[lane + 32 * k];
      const float dx = xi.x - y.x, dy = xi.y - y.y, dz = xi.z - y.z;
      cf[k] = fmaf(dz, dz, fmaf(dy, dy, dx * dx));
    }
    float m = t[0];
#pragma unroll
    for (int k = 1; k < kRcCols; ++k) m = fmaxf(m, t[k]);
    m = warp_maxf(m);
    const float ms = (m == -INFINITY) ? 0.f : m;
    float R = 0.f, Wc = 0.f, K0 = 0.f, K1 = 0.f;
#pragma unroll
    for (int k = 0; k < kRcCols; ++k) {
      const float p = ex2f(t[k] - ms);
      R += p;
      Wc = fmaf(cf[k], p, Wc);
      K0 = fmaf(cf[k], s_c0[lane + 32 * k], K0);
      if (B1) K1 = fmaf(cf[k], s_c1[lane + 32 * k], K1);
    }
    float4 o = make_float4(R, Wc, K0, K1);
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      o.x += __shfl_xor_sync(0xffffffffu, o.x, off);
      o.y += __shfl_xor_sync(0xffffffffu, o.y, off);
      o.z += __shfl_xor_sync(0xffffffffu, o.z, off);
      if (B1) o.w += __shfl_xor_sync(0xffffffffu, o.w, off);
    }
    if (lane == 0) {
      a.part[i * ldp + blockIdx.x] = o;
      a.pm[i * ldp + blockIdx.x] = ms;
    }
  }
}

// Per row: R_i, W_i (x cost_scale) with the fp64 row offset ((u_i + lu_i) + w) log2 e,
// K0_i, K1_i (x cost_scale); fixed strip order.
__global__ void __launch_bounds__(kVecThreads) k_rowcost_reduce(const float4* part, const float* pm, int64_t nstrips,
                                                               int64_t row_lo, int64_t row_hi, const double* u,
                                                               const double* lu, const double* w, double wscale,
                                                               double* R, double* W, double* K0, double* K1,
                                                               const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const double ww = *w;
  for (int64_t i = row_lo + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < row_hi;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double a2 = ((u[i] + (lu ? lu[i] : 0.0)) + ww) * kLog2e;
    double r = 0.0, wc = 0.0, k0 = 0.0, k1 = 0.0;
    for (int64_t s = 0; s < nstrips; ++s) {
      const float4 o = part[i * nstrips + s];
      if (o.x != 0.f) {
        const double sc = exp2(double(pm[i * nstrips + s]) + a2);
        r += double(o.x) * sc;
        wc += double(o.y) * sc;
      }
      k0 += double(o.z);
      k1 += double(o.w);
    }
    R[i] = r;
    W[i] = wc * wscale;
    K0[i] = k0 * wscale;
    K1[i] = k1 * wscale;
  }
}

using HVec = std::vector<double>;

inline double hsum(const HVec& x) { return ksum(x.data(), int64_t(x.size())); }

struct PlanEngine {
  Context& cx;
  const DevProblem& P;
  Workspace& ws;
  double gamma;
  DevBuf<double> buf;  // 8 n-vectors: lu, lv, row, col, P, Q, a0, b0 (+ a1, b1)
  PlanEngine(Context& c, const DevProblem& p, Workspace& w, double g) : cx(c), P(p), ws(w), gamma(g) {
    buf.alloc(size_t(10 * P.n));
  }
  ~PlanEngine() { cudaStreamSynchronize(cx.stream); }
  double* d(int k) { return buf.p + k * P.n; }
  void up(int k, const HVec& h) {
    PG_CK(cudaMemcpyAsync(d(k), h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  }

  // rows / cols of diag(exp(lu)) B(z) diag(exp(lv)) over the n x n block
  void block_sums(Slot z, const HVec* lu, const HVec* lv, HVec& row, HVec& col) {
    const int64_t n = P.n;
    if (lu) up(0, *lu);
    if (lv) up(1, *lv);
    const SweepOut so = sweep_point(cx, P, ws, z, lu ? d(0) : nullptr, lv ? d(1) : nullptr, nullptr, false, gamma);
    k_sum_partials<<<ws.nblk, kVecThreads, 0, cx.stream>>>(so.rowp, so.nstrips, so.colp, so.nrb, so.pfmt, z,
                                                           lu ? d(0) : nullptr, so.rowshift, d(2), d(3), nullptr);
    PG_CK(cudaGetLastError());
    row.resize(size_t(n));
    col.resize(size_t(n));
    PG_CK(cudaMemcpyAsync(row.data(), d(2), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(col.data(), d(3), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
  }

  // The fused fp32 pass (k_rowcost_f32) serves unsharded fp32 problems when
  // no dense plan is requested.
  bool fused_ok(const double* Xdev) const {
    return Xdev == nullptr && P.dtype == POTGPU_F32 && !cx.comm.sharded() && !fused_disabled() &&
           (P.kind == POTGPU_COST_DENSE || P.kind == POTGPU_COST_SQEUCLIDEAN || P.kind == POTGPU_COST_SQEUCLIDEAN_STORED);
  }
  static bool fused_disabled() {
    static const bool off = [] {
      const char* e = std::getenv("POTGPU_FUSED_ROUND");
      return e && e[0] == '0';
    }();
    return off;
  }

  // Per-row R, W, K0, K1 of the final plan (see RowCostArgs) in one pass.
  void row_cost_sums(Slot z, const HVec& lu, const HVec& lv, const HVec* b0, const HVec* b1, HVec& R, HVec& W,
                     HVec& K0, HVec& K1) {
    const int64_t n = P.n;
    up(0, lu);
    up(1, lv);
    if (b0) up(6, *b0);
    if (b1) up(7, *b1);
    const bool pts = P.kind == POTGPU_COST_SQEUCLIDEAN;
    const int64_t strips = ceil_div(n, pts ? int64_t(kRcStrip) : int64_t(kStripCols32));
    const int64_t target_rb = std::max<int64_t>(1, ceil_div(int64_t(cx.num_sms) * 4, strips));
    const int rpc = int(std::max<int64_t>(8, ceil_div(n, target_rb)));
    const dim3 g(unsigned(strips), unsigned(ceil_div(n, rpc)));
    if (rc_part.count < size_t(n * strips)) {
      rc_part.alloc(size_t(n * strips));
      rc_pm.alloc(size_t(n * strips));
    }
    RowCostArgs a{};
    a.n = n;
    a.row_lo = 0;
    a.row_hi = n;
    a.rows_per_cta = rpc;
    a.u = z.u(); a.v = z.v(); a.w = z.w();
    a.lv = d(1);
    a.b0 = b0 ? d(6) : nullptr;
    a.b1 = b1 ? d(7) : nullptr;
    a.part = rc_part.p;
    a.pm = rc_pm.p;
    double wscale = 1.0;
    if (pts) {
      wscale = P.cost_scale;
      if (b1) k_rowcost_pts64<true><<<g, kThreads, 0, cx.stream>>>(P.X4.p, P.Y4.p, kLog2e * P.cost_scale / gamma, a);
      else k_rowcost_pts64<false><<<g, kThreads, 0, cx.stream>>>(P.X4.p, P.Y4.p, kLog2e * P.cost_scale / gamma, a);
    } else {
      a.g = float(kLog2e / gamma);
      k_rowcost_f32<false><<<g, kThreads, 0, cx.stream>>>(P.C32.p, P.ld, nullptr, nullptr, a);
    }
    // R, W, K0, K1 land in d(2), d(3), d(8), d(9)
    k_rowcost_reduce<<<ws.nblk, kVecThreads, 0, cx.stream>>>(rc_part.p, rc_pm.p, strips, 0, n, z.u(), d(0), z.w(),
                                                             wscale, d(2), d(3), d(8), d(9), nullptr);
    PG_CK(cudaGetLastError());
    for (HVec* h : {&R, &W, &K0, &K1}) h->resize(size_t(n));
    PG_CK(cudaMemcpyAsync(R.data(), d(2), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(W.data(), d(3), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(K0.data(), d(8), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(K1.data(), d(9), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
  }
  DevBuf<float4> rc_part;
  DevBuf<float> rc_pm;

  // <C, X> for X = diag(Pv) B diag(Qv) + a0 b0^T + a1 b1^T; Xdev optional.
  double cost(Slot z, const HVec& Pv, const HVec& Qv, const HVec* a0, const HVec* b0, const HVec* a1, const HVec* b1,
              double* Xdev) {
    const int64_t n = P.n;
    up(4, Pv);
    up(5, Qv);
    PlanTermsDev t{d(4), d(5), nullptr, nullptr, nullptr, nullptr};
    if (a0) { up(6, *a0); up(7, *b0); t.a0 = d(6); t.b0 = d(7); }
    if (a1) { up(8, *a1); up(9, *b1); t.a1 = d(8); t.b1 = d(9); }
    const int rows = cost_sweep_rows(n);
    const bool mat = Xdev != nullptr;
    // this process's row ranges (all rows on one GPU); a sharded job's
    // materialised plan holds the process's own rows (the rest stays 0)
    std::vector<std::pair<int64_t, int64_t>> ranges;
    if (!cx.comm.sharded()) ranges.push_back({0, n});
    else for (const ShardGrid& sh : ws.shards) ranges.push_back({sh.lo, sh.hi});
    if (mat && cx.comm.world > 1) PG_CK(cudaMemsetAsync(Xdev, 0, size_t(n * n) * sizeof(double), cx.stream));
    int64_t np = 0;
    for (const auto& rg : ranges) {
      const int64_t nrows = rg.second - rg.first;
      if (nrows <= 0) continue;
      dim3 g(unsigned(ceil_div(n, kThreads)), unsigned(ceil_div(nrows, rows)));
      double* part = ws.partial.p + np;
      np += int64_t(g.x) * g.y;
      if (P.dtype == POTGPU_F64) {
        ElemDenseF64 el{P.L64.p, P.ld, gamma};
        if (mat) k_plan_cost<ElemDenseF64, true><<<g, kThreads, 0, cx.stream>>>(el, z, t, rg.first, rg.second, rows, part, Xdev);
        else k_plan_cost<ElemDenseF64, false><<<g, kThreads, 0, cx.stream>>>(el, z, t, rg.first, rg.second, rows, part, Xdev);
      } else if (P.kind == POTGPU_COST_DENSE) {
        ElemDenseF32 el{P.C32.p, P.ld, gamma};
        if (mat) k_plan_cost<ElemDenseF32, true><<<g, kThreads, 0, cx.stream>>>(el, z, t, rg.first, rg.second, rows, part, Xdev);
        else k_plan_cost<ElemDenseF32, false><<<g, kThreads, 0, cx.stream>>>(el, z, t, rg.first, rg.second, rows, part, Xdev);
      } else {
        ElemPointsF32 el{P.X4.p, P.Y4.p, P.cost_scale, gamma};
        if (mat) k_plan_cost<ElemPointsF32, true><<<g, kThreads, 0, cx.stream>>>(el, z, t, rg.first, rg.second, rows, part, Xdev);
        else k_plan_cost<ElemPointsF32, false><<<g, kThreads, 0, cx.stream>>>(el, z, t, rg.first, rg.second, rows, part, Xdev);
      }
      PG_CK(cudaGetLastError());
    }
    HVec part(static_cast<size_t>(np));
    PG_CK(cudaMemcpyAsync(part.data(), ws.partial.p, size_t(np) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
    return allreduce_host_sum(cx, ws, hsum(part));
  }

  // z_j = sum_i X_ij xh_i for the final plan terms (xh: n x 3 host, row-major);
  // one process's rows (the caller sums over ranks when sharded).
  HVec moments(Slot z, const HVec& Pv, const HVec& Qv, const HVec* a0, const HVec* b0, const HVec* a1, const HVec* b1,
               const HVec& xh) {
    const int64_t n = P.n;
    up(4, Pv);
    up(5, Qv);
    PlanTermsDev t{d(4), d(5), nullptr, nullptr, nullptr, nullptr};
    if (a0) { up(6, *a0); up(7, *b0); t.a0 = d(6); t.b0 = d(7); }
    if (a1) { up(8, *a1); up(9, *b1); t.a1 = d(8); t.b1 = d(9); }
    DevBuf<double> xhd, part, zd;
    xhd.alloc(size_t(3 * n));
    PG_CK(cudaMemcpyAsync(xhd.p, xh.data(), size_t(3 * n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    const int rows = cost_sweep_rows(n);
    dim3 g(unsigned(ceil_div(n, kThreads)), unsigned(ceil_div(n, rows)));
    part.alloc(size_t(g.y) * size_t(3 * n));
    zd.alloc(size_t(3 * n));
    if (P.dtype == POTGPU_F64) {
      ElemDenseF64 el{P.L64.p, P.ld, gamma};
      k_plan_moments<ElemDenseF64><<<g, kThreads, 0, cx.stream>>>(el, z, t, xhd.p, rows, part.p);
    } else if (P.kind == POTGPU_COST_DENSE) {
      ElemDenseF32 el{P.C32.p, P.ld, gamma};
      k_plan_moments<ElemDenseF32><<<g, kThreads, 0, cx.stream>>>(el, z, t, xhd.p, rows, part.p);
    } else {
      ElemPointsF32 el{P.X4.p, P.Y4.p, P.cost_scale, gamma};
      k_plan_moments<ElemPointsF32><<<g, kThreads, 0, cx.stream>>>(el, z, t, xhd.p, rows, part.p);
    }
    k_sum_moment_parts<<<cx.num_sms * 2, kVecThreads, 0, cx.stream>>>(part.p, g.y, n, zd.p);
    PG_CK(cudaGetLastError());
    HVec out(static_cast<size_t>(3 * n));
    PG_CK(cudaMemcpyAsync(out.data(), zd.p, size_t(3 * n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
    return out;
  }
};

struct PlanResult {
  double cost = 0, mass = 0, gap = 0;
  HVec row_slack, col_slack;
  HVec rowx, colx;  // X 1, X^T 1
  // the final plan X = diag(Pf) B(z) diag(Qf) + a0 b0^T (+ a1 b1^T)
  HVec Pf, Qf, a0, b0, a1, b1;
};

inline HVec vlog(const HVec& x) {
  HVec o(x.size());
  for (size_t i = 0; i < x.size(); ++i) o[i] = std::log(x[i]);
  return o;
}

// round_pot (rounding.hpp:46-77) of X1 = diag(P0) B diag(Q0) + a b^T (a, b
// optional), given the block row sums of diag(P0) B diag(Q0) (row0). Writes
// the final plan terms and metrics; the rank-1 term a b^T is the extracted
// balanced fill of the Sinkhorn path (extend.hpp:55).
inline PlanResult round_pot_implicit(PlanEngine& pe, Slot z, const HVec& P0, const HVec& Q0, const HVec& row0,
                                     const HVec* a, const HVec* b, const HVec& r, const HVec& c, double s,
                                     double* Xdev) {
  const size_t n = r.size();
  const double sa = a ? hsum(*a) : 0.0, sb = b ? hsum(*b) : 0.0;
  // out *= min(1, s / mass)
  const double mass1 = hsum(row0) + sa * sb;
  const double alpha = mass1 > 0 ? std::min(1.0, s / mass1) : 1.0;
  // row clip
  HVec rho(n, 1.0);
  for (size_t i = 0; i < n; ++i) {
    const double row = alpha * (row0[i] + (a ? (*a)[i] * sb : 0.0));
    if (row > 0) rho[i] = std::min(1.0, r[i] / row);
  }
  // column clip: columns of diag(alpha rho) X1
  HVec lrp(n), lq = vlog(Q0);
  for (size_t i = 0; i < n; ++i) lrp[i] = std::log(rho[i] * P0[i]);
  PhaseTimer pt(pe.cx.stream);
  HVec rr, cc;
  pe.block_sums(z, &lrp, &lq, rr, cc);
  pt.mark("round: column clip sums");
  double sra = 0.0;
  if (a) { HVec t(n); for (size_t i = 0; i < n; ++i) t[i] = rho[i] * (*a)[i]; sra = hsum(t); }
  HVec kap(n, 1.0), col3(n);
  for (size_t j = 0; j < n; ++j) {
    col3[j] = alpha * (cc[j] + (b ? (*b)[j] * sra : 0.0));
    if (col3[j] > 0) kap[j] = std::min(1.0, c[j] / col3[j]);
  }
  // rows / cols after both clips
  HVec lp = vlog(P0), lqk(n);
  for (size_t j = 0; j < n; ++j) lqk[j] = std::log(Q0[j] * kap[j]);
  HVec colX3(n), fb(n), kb0;
  for (size_t j = 0; j < n; ++j) colX3[j] = kap[j] * col3[j];
  for (size_t j = 0; j < n; ++j) fb[j] = std::max(c[j] - colX3[j], 0.0);
  if (b) { kb0.resize(n); for (size_t j = 0; j < n; ++j) kb0[j] = (*b)[j] * kap[j]; }
  // fused fp32 pass: final row sums + the cost's per-row terms (RowCostArgs);
  // the column factors of both rank-1 terms (fb, b kap) are known already
  const bool fused = pe.fused_ok(Xdev);
  HVec Wr, K0r, K1r;
  if (fused) pe.row_cost_sums(z, lp, lqk, &fb, b ? &kb0 : nullptr, rr, Wr, K0r, K1r);
  else pe.block_sums(z, &lp, &lqk, rr, cc);
  pt.mark("round: final sums");
  const double sbk = b ? hsum(kb0) : 0.0;
  HVec rowX3(n);
  for (size_t i = 0; i < n; ++i) rowX3[i] = alpha * rho[i] * (rr[i] + (a ? (*a)[i] * sbk : 0.0));
  // deficit fill (rounding.hpp:63-75)
  const double mass3 = hsum(rowX3);
  const double deficit = s - mass3;
  HVec fa(n);
  for (size_t i = 0; i < n; ++i) fa[i] = std::max(r[i] - rowX3[i], 0.0);
  const double na = hsum(fa), nb = hsum(fb);
  double f = 0.0;
  if (deficit > 0) {
    if (na <= 0 || nb <= 0) throw Error(POTGPU_INFEASIBLE, "Infeasible: deficit fill has no slack mass");
    f = deficit / (na * nb);
  }
  PlanResult out;
  out.mass = mass3 + f * na * nb;
  out.row_slack.resize(n);
  out.col_slack.resize(n);
  out.rowx.resize(n);
  out.colx.resize(n);
  double rg = 0.0, cg = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const double rx = rowX3[i] + f * fa[i] * nb;
    out.rowx[i] = rx;
    out.row_slack[i] = r[i] - rx;
    rg = std::max(rg, std::max(rx - r[i], 0.0));
  }
  for (size_t j = 0; j < n; ++j) {
    const double cx = colX3[j] + f * na * fb[j];
    out.colx[j] = cx;
    out.col_slack[j] = c[j] - cx;
    cg = std::max(cg, std::max(cx - c[j], 0.0));
  }
  out.gap = std::max({rg, cg, std::fabs(out.mass - s)});  // core.hpp:207-219
  // final plan terms
  HVec Pf(n), Qf(n), fa2(n);
  for (size_t i = 0; i < n; ++i) Pf[i] = (alpha * rho[i]) * P0[i];
  for (size_t j = 0; j < n; ++j) Qf[j] = Q0[j] * kap[j];
  for (size_t i = 0; i < n; ++i) fa2[i] = f * fa[i];
  HVec ra, kb;
  if (a) {
    ra.resize(n);
    kb.resize(n);
    for (size_t i = 0; i < n; ++i) ra[i] = alpha * rho[i] * (*a)[i];
    for (size_t j = 0; j < n; ++j) kb[j] = (*b)[j] * kap[j];
  }
  pt.mark("round: host O(n)");
  if (fused) {
    // <C, X> = sum_i (alpha rho_i) W_i + f fa_i K0_i + alpha rho_i a_i K1_i
    HVec terms(3 * n, 0.0);
    for (size_t i = 0; i < n; ++i) {
      terms[i] = (alpha * rho[i]) * Wr[i];
      terms[n + i] = fa2[i] * K0r[i];
      if (a) terms[2 * n + i] = ra[i] * K1r[i];
    }
    out.cost = hsum(terms);
  } else {
    out.cost = pe.cost(z, Pf, Qf, &fa2, &fb, a ? &ra : nullptr, a ? &kb : nullptr, Xdev);
  }
  pt.mark("round: plan cost");
  out.Pf = std::move(Pf);
  out.Qf = std::move(Qf);
  out.a0 = std::move(fa2);
  out.b0 = std::move(fb);
  if (a) {
    out.a1 = std::move(ra);
    out.b1 = std::move(kb);
  }
  return out;
}

// ------------------------------------------------------------------------
// round_pot (rounding.hpp:46-77) of B(z) ON THE DEVICE for the ASPOT plan
// (P0 = Q0 = 1, no rank-1 input term): the same arithmetic as
// round_pot_implicit with the O(n) scaling logic in three single-block
// kernels around the two sweeps (column-clip column sums; fused final row
// sums + <C, X>), no host round trip in between. Capturable: the per-record
// rounding of record_rounded_cost runs inside the attempt graph (gate).
//
// ro vectors (Workspace::rv): 0 log rho, 1 log kappa, 2 alpha rho, 3 colX3,
// 4 fb = max(c - colX3, 0), 5 R (final row sums of B diag(kappa)), 6 W, 7 K,
// 8 row slack, 9 col slack; + the column sums of the clip sweep in 3.
constexpr int kDrThreads = 1024;

__device__ __forceinline__ double dr_block_sum(double x, double* sh) {  // fixed order, all threads get it
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  __syncthreads();
  if (lane == 0) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    x = lane < (blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if (lane == 0) sh[32] = x;
  }
  __syncthreads();
  return sh[32];
}
__device__ __forceinline__ double dr_block_max(double x, double* sh) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  __syncthreads();
  if (lane == 0) sh[wid] = x;
  __syncthreads();
  if (wid == 0) {
    x = lane < (blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sh[32] = x;
  }
  __syncthreads();
  return sh[32];
}

struct DevRoundArgs {
  int64_t n;
  const double* row0;  // B(z) 1
  const double* r;     // original marginals
  const double* c;
  double s;
  double* v;           // 10 n ro vectors
  RoundOut* ro;
  const int* gate;     // null: always
  // record rounding: the last appended trace record gets the cost
  const AspotCtl* ctl;
  TraceDev* trace;
  int* clear;          // set to 0 at the end (the record gate), may be null
};

// The O(n) steps run on kDrBlocks blocks: a first pass writes per-block
// partials, the next kernel reduces them in block order (every block alike,
// fixed order) and goes on element-wise.
constexpr int kDrBlocks = 32;

// block partials of the mass of B(z): part[b]
__global__ void __launch_bounds__(kDrThreads) k_dr_mass(DevRoundArgs a, double* part) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  __shared__ double sh[33];
  double m = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.n; i += int64_t(gridDim.x) * blockDim.x)
    m += a.row0[i];
  m = dr_block_sum(m, sh);
  if (threadIdx.x == 0) part[blockIdx.x] = m;
}

// out *= min(1, s / mass); row clip rho (rounding.hpp:52-56)
__global__ void __launch_bounds__(kDrThreads) k_dr_rowclip(DevRoundArgs a, const double* part) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  const int64_t n = a.n;
  double mass1 = 0.0;
  for (int b = 0; b < kDrBlocks; ++b) mass1 += part[b];
  const double alpha = mass1 > 0 ? fmin(1.0, a.s / mass1) : 1.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double row = alpha * a.row0[i];
    const double rh = row > 0 ? fmin(1.0, a.r[i] / row) : 1.0;
    a.v[i] = log(rh);
    a.v[2 * n + i] = alpha * rh;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.ro->alpha = alpha;
}

// column clip kappa (rounding.hpp:57-61) from the column sums cc of diag(rho) B
__global__ void __launch_bounds__(kDrThreads) k_dr_colclip(DevRoundArgs a, const double* cc) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  const int64_t n = a.n;
  const double alpha = a.ro->alpha;
  for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
    const double col3 = alpha * cc[j];
    const double kp = col3 > 0 ? fmin(1.0, a.c[j] / col3) : 1.0;
    const double cx3 = kp * col3;
    a.v[n + j] = log(kp);
    a.v[3 * n + j] = cx3;
    a.v[4 * n + j] = fmax(a.c[j] - cx3, 0.0);
  }
}

// block partials of the deficit fill's sums: part[5 b + (mass3, na, nb, sum arho W, sum fa K)]
__global__ void __launch_bounds__(kDrThreads) k_dr_sums(DevRoundArgs a, double* part) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  __shared__ double sh[33];
  const int64_t n = a.n;
  const double* arho = a.v + 2 * n;
  const double* fb = a.v + 4 * n;
  const double* R = a.v + 5 * n;
  const double* W = a.v + 6 * n;
  const double* K = a.v + 7 * n;
  double m3 = 0.0, na = 0.0, nb = 0.0, saw = 0.0, sfk = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double x3 = arho[i] * R[i];
    const double fa = fmax(a.r[i] - x3, 0.0);
    m3 += x3;
    na += fa;
    nb += fb[i];
    saw += arho[i] * W[i];
    sfk += fa * K[i];
  }
  m3 = dr_block_sum(m3, sh);
  na = dr_block_sum(na, sh);
  nb = dr_block_sum(nb, sh);
  saw = dr_block_sum(saw, sh);
  sfk = dr_block_sum(sfk, sh);
  if (threadIdx.x == 0) {
    double* o = part + 5 * blockIdx.x;
    o[0] = m3; o[1] = na; o[2] = nb; o[3] = saw; o[4] = sfk;
  }
}

// deficit fill (rounding.hpp:63-75), <C, X> (core.hpp:199-204), slacks and
// plan_feasibility_gap (core.hpp:207-219); the gap maxima as block partials
__global__ void __launch_bounds__(kDrThreads) k_dr_slacks(DevRoundArgs a, const double* part, double* gpart) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  __shared__ double sh[33];
  const int64_t n = a.n;
  const double* arho = a.v + 2 * n;
  const double* cx3 = a.v + 3 * n;
  const double* fb = a.v + 4 * n;
  const double* R = a.v + 5 * n;
  double m3 = 0.0, na = 0.0, nb = 0.0, saw = 0.0, sfk = 0.0;
  for (int b = 0; b < kDrBlocks; ++b) {
    const double* o = part + 5 * b;
    m3 += o[0]; na += o[1]; nb += o[2]; saw += o[3]; sfk += o[4];
  }
  const double deficit = a.s - m3;
  double f = 0.0;
  int infeasible = 0;
  if (deficit > 0) {
    if (na <= 0 || nb <= 0) infeasible = 1;
    else f = deficit / (na * nb);
  }
  double rg = 0.0, cg = 0.0;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double x3 = arho[i] * R[i];
    const double fa = fmax(a.r[i] - x3, 0.0);
    const double rx = x3 + f * fa * nb;
    const double cx = cx3[i] + f * na * fb[i];
    a.v[8 * n + i] = a.r[i] - rx;
    a.v[9 * n + i] = a.c[i] - cx;
    rg = fmax(rg, fmax(rx - a.r[i], 0.0));
    cg = fmax(cg, fmax(cx - a.c[i], 0.0));
  }
  rg = dr_block_max(rg, sh);
  cg = dr_block_max(cg, sh);
  if (threadIdx.x == 0) {
    gpart[2 * blockIdx.x] = rg;
    gpart[2 * blockIdx.x + 1] = cg;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    RoundOut& o = *a.ro;
    o.mass3 = m3; o.na = na; o.nb = nb; o.f = f;
    o.mass = m3 + f * na * nb;
    o.cost = saw + f * sfk;
    o.infeasible = infeasible;
  }
}

__global__ void k_dr_finish(DevRoundArgs a, const double* gpart) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  if (threadIdx.x == 0) {
    double rg = 0.0, cg = 0.0;
    for (int b = 0; b < kDrBlocks; ++b) {
      rg = fmax(rg, gpart[2 * b]);
      cg = fmax(cg, gpart[2 * b + 1]);
    }
    RoundOut& o = *a.ro;
    o.row_gap = rg; o.col_gap = cg;
    o.gap = fmax(fmax(rg, cg), fabs(o.mass - a.s));
    if (a.trace && a.ctl && a.ctl->trace_len >= 1 && a.ctl->trace_len <= a.ctl->trace_cap)
      a.trace[a.ctl->trace_len - 1].rounded_cost = o.cost;
    if (a.clear) *a.clear = 0;
  }
}

// fp64 stored logK: the fused final pass (rows of B diag(kappa), W, K) with
// the reference's exponent association and clamp (k_plan_cost), cost
// C_ij = -logK_ij gamma (ElemDenseF64). Partials [row][strip] x 3 (fp64).
__global__ void __launch_bounds__(kThreads, 2) k_rowcost_f64(const double* __restrict__ L, int64_t ld, double gamma,
                                                             RowCostArgs a, double* part) {
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStripCols;
  double vj[8], fbj[8];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t j = j0 + 2 * lane + 64 * k + e;
      double vv = -INFINITY, ff = 0.0;
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
        if (a.b0) ff = a.b0[j];
      }
      vj[2 * k + e] = vv;
      fbj[2 * k + e] = ff;
    }
  const double w = *a.w;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    const double ui = a.u[i];
    const double2* row = reinterpret_cast<const double2*>(L + i * ld + j0) + lane;
    double R = 0.0, Wc = 0.0, K = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 x = __ldcs(row + 32 * k);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const double lk = e ? x.y : x.x;
        const double ee = ((lk + ui) + vj[2 * k + e]) + w;
        const double B = vj[2 * k + e] == -INFINITY ? 0.0 : exp(fmin(fmax(ee, kExpLo), kExpHi));
        const double cst = vj[2 * k + e] == -INFINITY ? 0.0 : -lk * gamma;
        R += B;
        Wc += cst * B;
        K += cst * fbj[2 * k + e];
      }
    }
    R = warp_sum(R);
    Wc = warp_sum(Wc);
    K = warp_sum(K);
    if (lane == 0) {
      double* o = part + (i * gridDim.x + blockIdx.x) * 3;
      o[0] = R; o[1] = Wc; o[2] = K;
    }
  }
}

__global__ void __launch_bounds__(kVecThreads) k_rowcost_reduce64(const double* part, int64_t nstrips, int64_t n,
                                                                 const int* gate, double* R, double* W, double* K) {
  pdl_wait();
  if (gate && *gate == 0) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double r = 0.0, wc = 0.0, k = 0.0;
    for (int64_t s = 0; s < nstrips; ++s) {
      const double* o = part + (i * nstrips + s) * 3;
      r += o[0]; wc += o[1]; k += o[2];
    }
    R[i] = r; W[i] = wc; K[i] = k;
  }
}

__global__ void k_gate_copy(const int* gate, int* dst) {  // a kernel-side copy of a gate for kernels without one
  pdl_wait();
  *dst = gate ? *gate : 1;
}

// The device rounding of the ASPOT plan: enqueue (capturable) ...
inline bool device_round_ok(const Context& cx, const DevProblem& P, const Workspace& ws) {
  static const bool on = [] {
    const char* e = std::getenv("POTGPU_DEVICE_ROUND");
    return !(e && e[0] == '0');
  }();
  if (!on || cx.comm.sharded()) return false;
  if (P.dtype == POTGPU_F64) return P.kind == POTGPU_COST_DENSE && ws.rc_part64.p;
  return ws.rc_part.p != nullptr;
}

inline void enqueue_round_device(Context& cx, const DevProblem& P, Workspace& ws, double gamma, Slot z,
                                 const double* row0, RoundOut* ro, const int* gate, const AspotCtl* ctl,
                                 TraceDev* trace) {
  const int64_t n = P.n;
  DevRoundArgs a{n, row0, ws.ro_r.p, ws.ro_c.p, P.s, ws.rv(0), ro, gate, ctl, trace, const_cast<int*>(gate)};
  double* drp = ws.rc_scratch.p;  // [kDrBlocks * 5] sums, then [kDrBlocks * 2] gap maxima
  launch_k(k_dr_mass, dim3(kDrBlocks), dim3(kDrThreads), 0, cx.stream, a, drp);
  launch_k(k_dr_rowclip, dim3(kDrBlocks), dim3(kDrThreads), 0, cx.stream, a, static_cast<const double*>(drp));
  // column clip: column sums of diag(rho) B (plain exp, the reference's b_matrix of the rounding input)
  launch_sweep(cx, P, ws, z, ws.rv(0), nullptr, gate, false, gamma);
  launch_k(k_sum_partials, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream, static_cast<const double*>(ws.rowp.p),
           ws.nstrips, static_cast<const double*>(ws.colp.p), ws.nrb, ws.pfmt, z, static_cast<const double*>(ws.rv(0)),
           P.rowshift(), ws.rv(5), ws.rv(3), gate);
  launch_k(k_dr_colclip, dim3(kDrBlocks), dim3(kDrThreads), 0, cx.stream, a, static_cast<const double*>(ws.rv(3)));
  // final row sums of B diag(kappa) + the cost's per-row terms
  RowCostArgs ra{};
  ra.n = n;
  ra.row_lo = 0;
  ra.row_hi = n;
  ra.u = z.u(); ra.v = z.v(); ra.w = z.w();
  ra.lv = ws.rv(1);
  ra.b0 = ws.rv(4);
  ra.b1 = nullptr;
  ra.gate = gate;
  if (P.dtype == POTGPU_F64) {
    const int64_t strips = ceil_div(n, int64_t(kStripCols));
    const int64_t target_rb = std::max<int64_t>(1, ceil_div(int64_t(cx.num_sms) * 4, strips));
    ra.rows_per_cta = int(std::max<int64_t>(8, ceil_div(n, target_rb)));
    const dim3 g(unsigned(strips), unsigned(ceil_div(n, ra.rows_per_cta)));
    launch_k(k_rowcost_f64, g, dim3(kThreads), 0, cx.stream, static_cast<const double*>(P.L64.p), P.ld, gamma, ra,
             ws.rc_part64.p);
    launch_k(k_rowcost_reduce64, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream,
             static_cast<const double*>(ws.rc_part64.p), strips, n, gate, ws.rv(5), ws.rv(6), ws.rv(7));
  } else {
    const bool pts = P.kind == POTGPU_COST_SQEUCLIDEAN;
    const int64_t strips = ceil_div(n, pts ? int64_t(kRcStrip) : int64_t(kStripCols32));
    const int64_t target_rb = std::max<int64_t>(1, ceil_div(int64_t(cx.num_sms) * 4, strips));
    ra.rows_per_cta = int(std::max<int64_t>(8, ceil_div(n, target_rb)));
    const dim3 g(unsigned(strips), unsigned(ceil_div(n, ra.rows_per_cta)));
    ra.part = ws.rc_part.p;
    ra.pm = ws.rc_pm.p;
    double wscale = 1.0;
    if (pts) {
      wscale = P.cost_scale;
      launch_k(k_rowcost_pts64<false>, g, dim3(kThreads), 0, cx.stream, static_cast<const float4*>(P.X4.p),
               static_cast<const float4*>(P.Y4.p), kLog2e * P.cost_scale / gamma, ra);
    } else {
      ra.g = float(kLog2e / gamma);
      launch_k(k_rowcost_f32<false>, g, dim3(kThreads), 0, cx.stream, static_cast<const float*>(P.C32.p), P.ld,
               static_cast<const float4*>(nullptr), static_cast<const float4*>(nullptr), ra);
    }
    launch_k(k_rowcost_reduce, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream, static_cast<const float4*>(ws.rc_part.p),
             static_cast<const float*>(ws.rc_pm.p), strips, int64_t(0), n, z.u(), static_cast<const double*>(nullptr),
             z.w(), wscale, ws.rv(5), ws.rv(6), ws.rv(7), ws.rv(8) /* K1 = 0 (no rank-1 input); slack slot, rewritten */, gate);
  }
  launch_k(k_dr_sums, dim3(kDrBlocks), dim3(kDrThreads), 0, cx.stream, a, drp);
  launch_k(k_dr_slacks, dim3(kDrBlocks), dim3(kDrThreads), 0, cx.stream, a, static_cast<const double*>(drp),
           drp + 5 * kDrBlocks);
  launch_k(k_dr_finish, dim3(1), dim3(32), 0, cx.stream, a, static_cast<const double*>(drp + 5 * kDrBlocks));
  PG_CK(cudaGetLastError());
}

// ... and collect: the PlanResult of round_pot_implicit (plan terms only when `full`).
inline PlanResult collect_round_device(Context& cx, const DevProblem& P, Workspace& ws, const RoundOut& ro, bool full) {
  const int64_t n = P.n;
  if (ro.infeasible) throw Error(POTGPU_INFEASIBLE, "Infeasible: deficit fill has no slack mass");
  PlanResult out;
  out.cost = ro.cost;
  out.mass = ro.mass;
  out.gap = ro.gap;
  out.row_slack.resize(size_t(n));
  out.col_slack.resize(size_t(n));
  PG_CK(cudaMemcpyAsync(out.row_slack.data(), ws.rv(8), size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
  PG_CK(cudaMemcpyAsync(out.col_slack.data(), ws.rv(9), size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
  HVec lk, arho, cx3, fb, R;
  if (full) {
    for (HVec* h : {&lk, &arho, &cx3, &fb, &R}) h->resize(size_t(n));
    PG_CK(cudaMemcpyAsync(lk.data(), ws.rv(1), size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(arho.data(), ws.rv(2), size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(cx3.data(), ws.rv(3), size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(fb.data(), ws.rv(4), size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(R.data(), ws.rv(5), size_t(n) * 8, cudaMemcpyDeviceToHost, cx.stream));
  }
  PG_CK(cudaStreamSynchronize(cx.stream));
  if (full) {
    out.Pf = arho;
    out.Qf.resize(size_t(n));
    out.a0.resize(size_t(n));
    out.rowx.resize(size_t(n));
    out.colx.resize(size_t(n));
    for (int64_t i = 0; i < n; ++i) {
      const double x3 = arho[size_t(i)] * R[size_t(i)];
      const double fa = std::max(P.r[size_t(i)] - x3, 0.0);
      out.Qf[size_t(i)] = std::exp(lk[size_t(i)]);
      out.a0[size_t(i)] = ro.f * fa;
      out.rowx[size_t(i)] = x3 + ro.f * fa * ro.nb;
      out.colx[size_t(i)] = cx3[size_t(i)] + ro.f * ro.na * fb[size_t(i)];
    }
    out.b0 = std::move(fb);
  }
  return out;
}

}  // namespace potgpu
