// rounding.cuh — the output stage on the device without materialising the
// plan: round_pot(B(z), in) (rounding.hpp:46-77) held implicitly as
//   X = diag(alpha rho) B diag(kappa) + f a b^T
// with its row/column sums, mass, feasibility gap (core.hpp:207-219) and
// cost <C, X> (core.hpp:199-204) computed by weighted sweeps; the dense plan
// is written only on request (n <= a few thousand).
#pragma once

#include "aspot_kernels.cuh"
#include "sweep.cuh"

namespace potgpu {

// Per-element views of the cost for the (non-hot) cost/materialise sweeps.
struct ElemDenseF64 {
  const double* L; int64_t ld; double gamma;
  __device__ __forceinline__ double logk(int64_t i, int64_t j) const { return L[i * ld + j]; }
  __device__ __forceinline__ double cost(int64_t i, int64_t j) const { return -L[i * ld + j] * gamma; }
};
struct ElemDenseF32 {
  const float* C; int64_t ld; double gamma;
  __device__ __forceinline__ double cost(int64_t i, int64_t j) const { return double(C[i * ld + j]); }
  __device__ __forceinline__ double logk(int64_t i, int64_t j) const { return -cost(i, j) / gamma; }
};
struct ElemPointsF32 {
  const float4* X; const float4* Y; double scale; double gamma;
  __device__ __forceinline__ double cost(int64_t i, int64_t j) const {
    const float4 a = X[i], b = Y[j];
    const double dx = double(a.x) - double(b.x), dy = double(a.y) - double(b.y), dz = double(a.z) - double(b.z);
    return (((dx * dx) + dy * dy) + dz * dz) * scale;
  }
  __device__ __forceinline__ double logk(int64_t i, int64_t j) const { return -cost(i, j) / gamma; }
};

struct RoundArgs {
  int64_t n;
  Slot z;                  // point whose B is rounded
  const double* rowb;      // B 1 at z
  const double* r; const double* c; double s;  // ORIGINAL instance (solvers.hpp:371)
  double* rho; double* kappa; double* lu; double* lv;
  double* rowx; double* colx; double* a; double* b;
  double* row_slack; double* col_slack;
  double* scratch;
  const int* gate;
  const double* total_ptr;  // 1^T B 1 at z
};

// alpha = min(1, s/mass); rho_i = min(1, r_i / (alpha B1)_i)  (rounding.hpp:53-58)
__global__ void k_round_a(AspotCtl* ctl, RoundArgs a) {
  if (a.gate && *a.gate == 0) return;
  const double mass = *a.total_ptr;
  const double alpha = mass > 0 ? fmin(1.0, a.s / mass) : 1.0;
  if (blockIdx.x == 0 && threadIdx.x == 0) ctl->ro.alpha = alpha;
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += int64_t(gridDim.x) * blockDim.x) {
    const double row = alpha * a.rowb[i];
    const double rh = row > 0 ? fmin(1.0, a.r[i] / row) : 1.0;
    a.rho[i] = rh;
    a.lu[i] = log(alpha * rh);
  }
}

// kappa_j = min(1, c_j / col_j) of the row-scaled plan (rounding.hpp:59-62)
__global__ void k_round_b(RoundArgs a, const double* colp, int64_t nrb, int pfmt) {
  if (a.gate && *a.gate == 0) return;
  const int64_t n = a.n;
  for (int64_t j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += int64_t(gridDim.x) * blockDim.x) {
    double col = 0.0;
    for (int64_t s = 0; s < nrb; ++s) col += partial_value(colp, s * n + j, pfmt);
    const double k = col > 0 ? fmin(1.0, a.c[j] / col) : 1.0;
    a.kappa[j] = k;
    a.lv[j] = log(k);
  }
}

template <int K>
__device__ void block_reduce_store(double (&acc)[K], double* out, const bool* is_max) {
  __shared__ double sh[K][kVecThreads];
  for (int k = 0; k < K; ++k) sh[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int stride = kVecThreads / 2; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride)
      for (int k = 0; k < K; ++k)
        sh[k][threadIdx.x] = is_max[k] ? fmax(sh[k][threadIdx.x], sh[k][threadIdx.x + stride]) : sh[k][threadIdx.x] + sh[k][threadIdx.x + stride];
    __syncthreads();
  }
  if (threadIdx.x < K) out[blockIdx.x * K + threadIdx.x] = sh[threadIdx.x][0];
}

// Row/col sums of the scaled plan, slacks a, b (rounding.hpp:63-67)
__global__ void __launch_bounds__(kVecThreads) k_round_c(RoundArgs a, const double* rowp, int64_t nstrips, const double* colp,
                                                         int64_t nrb, int pfmt) {
  if (a.gate && *a.gate == 0) return;
  const int64_t n = a.n;
  double acc[3] = {0.0, 0.0, 0.0};  // mass3, na, nb
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double row = 0.0, col = 0.0;
    const double a2 = ((a.z.u()[i] + a.lu[i]) + *a.z.w()) * kLog2e;  // fp32 row-partial offset
    for (int64_t s = 0; s < nstrips; ++s) row += partial_value(rowp, s * n + i, pfmt, a2);
    for (int64_t s = 0; s < nrb; ++s) col += partial_value(colp, s * n + i, pfmt);
    a.rowx[i] = row;
    a.colx[i] = col;
    const double ai = fmax(a.r[i] - row, 0.0), bi = fmax(a.c[i] - col, 0.0);
    a.a[i] = ai;
    a.b[i] = bi;
    acc[0] += row; acc[1] += ai; acc[2] += bi;
  }
  const bool ismax[3] = {false, false, false};
  block_reduce_store<3>(acc, a.scratch, ismax);
}

// Deficit fill coefficient (rounding.hpp:63-75)
__global__ void k_round_d(AspotCtl* ctl, RoundArgs a, int nblk) {
  if (a.gate && *a.gate == 0) return;
  if (threadIdx.x || blockIdx.x) return;
  double mass3 = 0, na = 0, nb = 0;
  for (int b = 0; b < nblk; ++b) { mass3 += a.scratch[3 * b]; na += a.scratch[3 * b + 1]; nb += a.scratch[3 * b + 2]; }
  RoundOut& ro = ctl->ro;
  ro.mass3 = mass3; ro.na = na; ro.nb = nb; ro.f = 0.0; ro.infeasible = 0;
  const double deficit = a.s - mass3;
  if (deficit > 0) {
    if (na <= 0 || nb <= 0) { ro.infeasible = 1; ctl->fatal = POTGPU_INFEASIBLE; }
    else ro.f = deficit / (na * nb);
  }
  ro.mass = mass3 + ro.f * na * nb;
}

// Final marginals, slacks and gap terms (core.hpp:185-196, 207-219)
__global__ void __launch_bounds__(kVecThreads) k_round_e(AspotCtl* ctl, RoundArgs a) {
  if (a.gate && *a.gate == 0) return;
  const double f = ctl->ro.f, na = ctl->ro.na, nb = ctl->ro.nb;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += int64_t(gridDim.x) * blockDim.x) {
    const double rx = a.rowx[i] + f * a.a[i] * nb;
    const double cx = a.colx[i] + f * na * a.b[i];
    if (a.row_slack) a.row_slack[i] = a.r[i] - rx;
    if (a.col_slack) a.col_slack[i] = a.c[i] - cx;
    acc[0] = fmax(acc[0], fmax(rx - a.r[i], 0.0));
    acc[1] = fmax(acc[1], fmax(cx - a.c[i], 0.0));
  }
  const bool ismax[2] = {true, true};
  block_reduce_store<2>(acc, a.scratch + 4096, ismax);
}

// <C, X> with X_ij = ((B_ij alpha) rho_i) kappa_j + f (a_i b_j)  (core.hpp:203)
template <class E, bool MATERIALIZE>
__global__ void __launch_bounds__(kThreads) k_cost_sweep(AspotCtl* ctl, E el, RoundArgs a, int rows_per_cta, double* partial,
                                                         double* Xout, bool floor_exp) {
  if (a.gate && *a.gate == 0) return;
  const int64_t n = a.n;
  const int64_t j = int64_t(blockIdx.x) * kThreads + threadIdx.x;
  const double alpha = ctl->ro.alpha, f = ctl->ro.f;
  const double w = *a.z.w();
  double acc = 0.0;
  if (j < n) {
    const double vj = a.z.v()[j], kj = a.kappa[j], bj = a.b[j];
    const int64_t r0 = int64_t(blockIdx.y) * rows_per_cta, r1 = min(n, r0 + rows_per_cta);
    for (int64_t i = r0; i < r1; ++i) {
      const double e = ((el.logk(i, j) + a.z.u()[i]) + vj) + w;
      const double B = floor_exp ? exp(fmax(e, kExpLo)) : exp(e);
      const double x = ((B * alpha) * a.rho[i]) * kj + f * (a.a[i] * bj);
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

__global__ void k_round_f(AspotCtl* ctl, RoundArgs a, const double* partial, int64_t npart, int nblk_e, TraceDev* trace,
                          int is_record) {
  if (a.gate && *a.gate == 0) return;
  if (threadIdx.x || blockIdx.x) return;
  double cost = 0.0;
  for (int64_t k = 0; k < npart; ++k) cost += partial[k];
  double rg = 0.0, cg = 0.0;
  for (int b = 0; b < nblk_e; ++b) { rg = fmax(rg, a.scratch[4096 + 2 * b]); cg = fmax(cg, a.scratch[4096 + 2 * b + 1]); }
  RoundOut& ro = ctl->ro;
  ro.cost = cost; ro.row_gap = rg; ro.col_gap = cg;
  ro.gap = fmax(fmax(rg, cg), fabs(ro.mass - a.s));
  if (is_record) {
    if (trace && ctl->trace_len >= 1 && ctl->trace_len <= ctl->trace_cap) trace[ctl->trace_len - 1].rounded_cost = cost;
    ctl->g_record = 0;
  }
}

}  // namespace potgpu
