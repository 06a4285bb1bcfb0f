// sinkhorn_kernels.cuh — log-domain Sinkhorn on the dummy-node extension
// (solvers.hpp:415-481) without materialising the (n+1)^2 extension or
// transposing C (the reference copies logK^T every iteration, :469).
//
// Per iteration two n^2 sweeps:
//   column LSE at u_{k+1}:  v_j = log c_j - LSE_i(logK_ij + u_i)
//   row LSE at v_{k+1}:     LSE_i(logK_ij + v_j) -> row sums of B(u, v) for
//                           the marginal error and the next u update.
// The column sums of B(u_{k+1}, v_{k+1}) are exp(v_j + LSE_j) (no extra
// pass). The dummy row/column (logK = -0/gamma, corner -A/gamma) are O(n)
// terms. LSE partials are (max, sum) pairs with an exact per-row (warp max)
// or per-column (chunked running max) shift, so arbitrarily small rows or
// columns never flush — the reference's max-shifted lse_rows (:397-401).
#pragma once

#include "sweep.cuh"

namespace potgpu {

// double2 (m, S) natural log | float2 (S, m) log2 | split: m at p[k], S at p[split + k]
enum LsePartialFormat { LP_F64 = 0, LP_F32 = 1, LP_SPLIT = 2 };

__device__ __forceinline__ void lse_part(const double* p, int64_t idx, int fmt, double& m, double& S) {
  if (fmt == LP_F64) {
    const double2 q = reinterpret_cast<const double2*>(p)[idx];
    m = q.x;
    S = q.y;
  } else {
    const float2 q = reinterpret_cast<const float2*>(p)[idx];
    m = q.x == 0.f ? -INFINITY : double(q.y) * kLn2;
    S = double(q.x);
  }
}

// (m, S) <- (m, S) (+) (m2, S2)
__device__ __forceinline__ void lse_merge(double& m, double& S, double m2, double S2) {
  if (m2 == -INFINITY || S2 == 0.0) return;
  if (m == -INFINITY) { m = m2; S = S2; return; }
  if (m2 > m) { S = S * exp(m - m2) + S2; m = m2; }
  else S = S + S2 * exp(m2 - m);
}

// ---------------------------------------------------------------- fp64 --
// Row LSE: x_ij = logK_ij + v_j (solvers.hpp:464-466).
__global__ void __launch_bounds__(kThreads, 2) sweep_rowlse_f64(const double* __restrict__ L, int64_t ld, int64_t n,
                                                               const double* __restrict__ v, int64_t row_lo, int64_t row_hi, int rows_per_cta,
                                                               double2* rowp, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j0 = int64_t(blockIdx.x) * kStripCols;
  double vj[8];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t j = j0 + 2 * lane + 64 * k + e;
      vj[2 * k + e] = j < n ? v[j] : 0.0;  // padding columns of L hold -inf
    }
  const int64_t r0 = row_lo + int64_t(blockIdx.y) * rows_per_cta, r1 = min(row_hi, r0 + rows_per_cta);
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    const double2* row = reinterpret_cast<const double2*>(L + i * ld + j0) + lane;
    double x[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double2 c = __ldcs(row + 32 * k);
      x[2 * k] = c.x + vj[2 * k];
      x[2 * k + 1] = c.y + vj[2 * k + 1];
    }
    double m = x[0];
#pragma unroll
    for (int k = 1; k < 8; ++k) m = fmax(m, x[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    double S = 0.0;
    if (m != -INFINITY) {
#pragma unroll
      for (int k = 0; k < 8; ++k) S += exp(x[k] - m);
    }
    S = warp_sum(S);
    if (lane == 0) rowp[i * gridDim.x + blockIdx.x] = make_double2(m, S);
  }
}

// Column LSE: x_ij = logK_ij + u_i (solvers.hpp:469-471), rows in chunks of
// 4 with a per-column running max.
__global__ void __launch_bounds__(kThreads, 2) sweep_collse_f64(const double* __restrict__ L, int64_t ld, int64_t n,
                                                               const double* __restrict__ u, int64_t row_lo, int64_t row_hi, int rows_per_cta,
                                                               double2* colp, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j0 = int64_t(blockIdx.x) * kStripCols;
  double m[8], S[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) { m[k] = -INFINITY; S[k] = 0.0; }
  const int64_t r0 = row_lo + int64_t(blockIdx.y) * rows_per_cta, r1 = min(row_hi, r0 + rows_per_cta);
  constexpr int R = 2;  // rows per chunk (register budget: no spills)
  for (int64_t base = r0 + R * warp; base < r1; base += R * kWarps) {
    double x[R][8];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t i = base + q;
      if (i < r1) {
        const double ui = u[i];
        const double2* row = reinterpret_cast<const double2*>(L + i * ld + j0) + lane;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const double2 c = __ldcs(row + 32 * k);
          x[q][2 * k] = c.x + ui;
          x[q][2 * k + 1] = c.y + ui;
        }
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) x[q][k] = -INFINITY;
      }
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const double cm = fmax(x[0][k], x[1][k]);
      if (cm == -INFINITY) continue;
      if (cm > m[k]) {
        S[k] = (m[k] == -INFINITY) ? 0.0 : S[k] * exp(m[k] - cm);
        m[k] = cm;
      }
#pragma unroll
      for (int q = 0; q < R; ++q) S[k] += exp(x[q][k] - m[k]);
    }
  }
  __shared__ double sm[kWarps][kStripCols];
  __shared__ double sS[kWarps][kStripCols];
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      sm[warp][2 * lane + 64 * k + e] = m[2 * k + e];
      sS[warp][2 * lane + 64 * k + e] = S[2 * k + e];
    }
  __syncthreads();
  const int t = threadIdx.x;
  double M = -INFINITY, SS = 0.0;
  for (int w = 0; w < kWarps; ++w) lse_merge(M, SS, sm[w][t], sS[w][t]);
  if (j0 + t < n) colp[(j0 + t) * gridDim.y + blockIdx.y] = make_double2(M, SS);
}

// ---------------------------------------------------------------- fp32 --
// Column LSE in log2 units: t_ij = U_i - kappa_ij with U_i = u_i log2 e,
// 16 columns per lane, rows in chunks of 4 with a per-column running max;
// partial = float2 (S, m) meaning S 2^m.
template <class Src>
__global__ void __launch_bounds__(kThreads, 2) sweep_collse_f32(Src src, int64_t n, const double* __restrict__ u,
                                                               int64_t row_lo, int64_t row_hi, int rows_per_cta,
                                                               float2* colp, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t j0 = int64_t(blockIdx.x) * kStripCols32;
  typename Src::Col cols[kPairs];
  bool ok[2 * kPairs];
#pragma unroll
  for (int q = 0; q < kPairs; ++q) {
    ok[2 * q] = f32_col(j0, lane, q, 0) < n;
    ok[2 * q + 1] = f32_col(j0, lane, q, 1) < n;
  }
  if constexpr (Src::kHasCols) {
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      float4 y0 = make_float4(0, 0, 0, 0), y1 = make_float4(0, 0, 0, 0);
      const int64_t ja = f32_col(j0, lane, q, 0), jb = f32_col(j0, lane, q, 1);
      if (ja < n) y0 = src.Ys[ja];
      if (jb < n) y1 = src.Ys[jb];
      cols[q].x = make_float2(y0.x, y1.x);
      cols[q].y = make_float2(y0.y, y1.y);
      cols[q].z = make_float2(y0.z, y1.z);
    }
  }
  float m[2 * kPairs], S[2 * kPairs];
#pragma unroll
  for (int k = 0; k < 2 * kPairs; ++k) { m[k] = -INFINITY; S[k] = 0.f; }
  const int64_t r0 = row_lo + int64_t(blockIdx.y) * rows_per_cta, r1 = min(row_hi, r0 + rows_per_cta);
  constexpr int R = 2;
  for (int64_t base = r0 + R * warp; base < r1; base += R * kWarps) {
    float2 t[R][kPairs];
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int64_t i = base + q;
      if (i < r1) {
        const float Ui = float(u[i] * kLog2e);
        float2 U2[kPairs];
#pragma unroll
        for (int p = 0; p < kPairs; ++p) U2[p] = make_float2(Ui, Ui);
        src.expo(src.load(i, j0, lane), cols, U2, t[q]);
      } else {
#pragma unroll
        for (int p = 0; p < kPairs; ++p) t[q][p] = make_float2(-INFINITY, -INFINITY);
      }
    }
#pragma unroll
    for (int p = 0; p < kPairs; ++p) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int k = 2 * p + h;
        float cm = -INFINITY;
#pragma unroll
        for (int q = 0; q < R; ++q) cm = fmaxf(cm, h ? t[q][p].y : t[q][p].x);
        if (!ok[k] || cm == -INFINITY) continue;
        if (cm > m[k]) {
          S[k] = (m[k] == -INFINITY) ? 0.f : S[k] * ex2f(m[k] - cm);
          m[k] = cm;
        }
#pragma unroll
        for (int q = 0; q < R; ++q) S[k] += ex2f((h ? t[q][p].y : t[q][p].x) - m[k]);
      }
    }
  }
  __shared__ float sm[kWarps][kStripCols32];
  __shared__ float sS[kWarps][kStripCols32];
#pragma unroll
  for (int p = 0; p < kPairs; ++p) {
    const int c = 4 * lane + 128 * (p >> 1) + 2 * (p & 1);
    sm[warp][c] = m[2 * p];
    sS[warp][c] = S[2 * p];
    sm[warp][c + 1] = m[2 * p + 1];
    sS[warp][c + 1] = S[2 * p + 1];
  }
  __syncthreads();
  for (int c = threadIdx.x; c < kStripCols32; c += kThreads) {
    float M = -INFINITY;
    for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm[w][c]);
    float SS = 0.f;
    if (M != -INFINITY)
      for (int w = 0; w < kWarps; ++w)
        if (sm[w][c] != -INFINITY) SS += sS[w][c] * ex2f(sm[w][c] - M);
    if (j0 + c < n) colp[(j0 + c) * gridDim.y + blockIdx.y] = make_float2(M == -INFINITY ? 0.f : SS, M == -INFINITY ? 0.f : M);
  }
}

// Sharded Sinkhorn (shard.cuh): one shard's LSE partials -> its slice of
// the all-reduce vector. ROWS: (M_i, S_i) pairs (LP_F64 layout) for the
// shard's rows, exact (0, 0) elsewhere (SUM-reduced). COLS: m_j at out[j],
// S_j at out[n + j] (MAX-reduced, rescaled, SUM-reduced).
template <bool ROWS>
__global__ void k_shard_gather_lse(const double* p, int64_t cnt, int fmt, int64_t n, int64_t lo, int64_t hi,
                                   const double* rowshift, double* out, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double M = -INFINITY, S = 0.0;
    if (!ROWS || (i >= lo && i < hi))
      for (int64_t k = 0; k < cnt; ++k) {
        double m2, S2;
        lse_part(p, i * cnt + k, fmt, m2, S2);
        lse_merge(M, S, m2, S2);
      }
    if (ROWS && rowshift && M != -INFINITY) M = M + rowshift[i] * kLn2;
    if (ROWS) {
      const bool own = i >= lo && i < hi;
      out[2 * i] = own ? M : 0.0;
      out[2 * i + 1] = own ? S : 0.0;
    } else {
      out[i] = M;
      out[n + i] = S;
    }
  }
}

// ------------------------------------------------------------ control --
struct SinkCtl {
  int g_active, paused, status, fatal;
  int64_t n, it, max_iterations, pause_at, log_every, trace_len, trace_cap;
  double tol, error, phi, corner;  // corner = -A/gamma (solvers.hpp:420 on C_ext(n, n) = A)
  double row_lse_n, col_lse_n;     // dummy row / column LSEs
  uint64_t t0_ns, loop_end_ns;
  int64_t sweeps;
  int col_flush;  // fast column pass lost a column (fp32 flush): run the exact pass
  int pad;
  int64_t col_flush_count;  // iterations that needed the exact column pass
};

struct SinkVec {  // device vectors of the extended problem (length n + 1)
  double* u; double* u_next; double* v;
  double* log_r; double* log_c; double* r; double* c;
  double* zv_v;    // v[0..n) mirrored into the fp32 row-sweep point slot (0, v, 0)
  double* zuv_u;   // u[0..n), v[0..n) mirrored into the point slot (u, v, 0) of the
  double* zuv_v;   // fp32 fast column pass (null: no fast pass)
  double* scratch; // block partials: [nblk][4] rows, [nblk][4] cols
};

// log-sum-exp of x_k = (-0 + a_k) (k < n) and corner + a_n (the dummy
// row/column of the extension): block partials (max, sum relative to it),
// merged in block order by the last block to finish (atomic ticket).
constexpr int kSkDummyBlocks = 148;
__global__ void k_sk_dummy(SinkCtl* ctl, const double* a, int which, double* part, unsigned* ticket, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int64_t n = ctl->n;
  __shared__ double sh[kVecThreads];
  __shared__ bool last;
  const int64_t chunk = (n + gridDim.x - 1) / gridDim.x;
  const int64_t k0 = int64_t(blockIdx.x) * chunk, k1 = min(n, k0 + chunk);
  double m = -INFINITY;
  for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) m = fmax(m, -0.0 + a[k]);
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int s = kVecThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
    __syncthreads();
  }
  const double M = sh[0];
  __syncthreads();
  double S = 0.0;
  if (M != -INFINITY)
    for (int64_t k = k0 + threadIdx.x; k < k1; k += blockDim.x) S += exp((-0.0 + a[k]) - M);
  sh[threadIdx.x] = S;
  __syncthreads();
  for (int s = kVecThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) sh[threadIdx.x] += sh[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    part[2 * blockIdx.x] = M;
    part[2 * blockIdx.x + 1] = sh[0];
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  *ticket = 0u;
  const volatile double* vp = part;
  double Mt = -INFINITY, St = 0.0;
  for (int b = 0; b < int(gridDim.x); ++b) lse_merge(Mt, St, vp[2 * b], vp[2 * b + 1]);
  lse_merge(Mt, St, ctl->corner + a[n], 1.0);
  const double lse = Mt + log(St);
  if (which == 0) ctl->row_lse_n = lse; else ctl->col_lse_n = lse;
}

template <int K, int T>
__device__ void sk_block_store(double (&acc)[K], double* out) {
  __shared__ double sh[K][T];
  for (int k = 0; k < K; ++k) sh[k][threadIdx.x] = acc[k];
  __syncthreads();
  for (int s = T / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int k = 0; k < K; ++k) sh[k][threadIdx.x] += sh[k][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x < K) out[blockIdx.x * K + threadIdx.x] = sh[threadIdx.x][0];
}

constexpr int kSkThreads = 128;
constexpr int kSkTPI = 4;  // threads per index

// log-sum-exp of the cnt (max, sum) partials at p[base..] of one index,
// split over a group of kSkTPI threads (max pass, then sum pass); result as
// (M, S) in natural-log units, replicated in the group.
__device__ __forceinline__ void group_lse(const double* p, int64_t base, int64_t cnt, int fmt, int q, double& M, double& S,
                                          int64_t split = 0) {
  if (fmt == LP_SPLIT) {  // one (m, S) per index (all-reduced shards)
    M = p[base];
    S = p[split + base];
    if (S == 0.0) M = -INFINITY;
    return;
  }
  M = -INFINITY;
  for (int64_t k = q; k < cnt; k += kSkTPI) {
    double m2, S2;
    lse_part(p, base + k, fmt, m2, S2);
    if (S2 != 0.0) M = fmax(M, m2);
  }
#pragma unroll
  for (int o = kSkTPI / 2; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
  S = 0.0;
  if (M != -INFINITY) {
    if (fmt == LP_F32) {
      const float Ml2 = float(M * kLog2e);
      float Sf = 0.f;
      const float2* f = reinterpret_cast<const float2*>(p) + base;
      for (int64_t k = q; k < cnt; k += kSkTPI) {
        const float2 x = f[k];
        if (x.x != 0.f) Sf += x.x * ex2f(x.y - Ml2);
      }
      S = double(Sf);
      M = double(Ml2) * kLn2;
    } else {
      for (int64_t k = q; k < cnt; k += kSkTPI) {
        double m2, S2;
        lse_part(p, base + k, fmt, m2, S2);
        if (S2 != 0.0) S += S2 * exp(m2 - M);
      }
    }
  }
#pragma unroll
  for (int o = kSkTPI / 2; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
}

// Rows (a thread group per row; the row's strip partials are contiguous):
// LSE_i + the dummy column (logK_in = -0, x = v_n); row sums of B(u, v) =
// exp(u_i + LSE_i); next u = log r - LSE.
__global__ void __launch_bounds__(kSkThreads) k_sk_rows(SinkCtl* ctl, SinkVec sv, const double* rowp, int64_t nstrips,
                                                        int fmt, const double* rowshift, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int64_t n = ctl->n;
  const double vn = sv.v[n];
  const int q = threadIdx.x % kSkTPI;
  const int64_t per_block = kSkThreads / kSkTPI, span = int64_t(gridDim.x) * per_block;
  double acc[4] = {0, 0, 0, 0};  // |row - r|, sum row, masked u.r
  for (int64_t i0 = int64_t(blockIdx.x) * per_block; i0 < n; i0 += span) {
    const int64_t i = i0 + threadIdx.x / kSkTPI;
    const bool live = i < n;
    const int64_t ii = live ? i : n - 1;
    double M, S;
    group_lse(rowp, ii * nstrips, nstrips, fmt, q, M, S);
    if (!live || q != 0) continue;
    if (rowshift && M != -INFINITY) M = M + rowshift[i] * kLn2;  // the source's row term (log2 -> natural)
    lse_merge(M, S, -0.0 + vn, 1.0);
    const double lse = M + log(S);
    const double row = exp(sv.u[i] + lse);
    acc[0] += fabs(row - sv.r[i]);
    acc[1] += row;
    if (sv.r[i] > 0) acc[2] += sv.u[i] * sv.r[i];  // masked_dot (solvers.hpp:389-395)
    sv.u_next[i] = sv.log_r[i] - lse;
  }
  sk_block_store<4, kSkThreads>(acc, sv.scratch);
}

// Columns (a thread group per column): LSE_j + the dummy row (logK_nj =
// -0, x = u_n). update: v_j = log c_j - LSE_j; the column sums of B(u, v)
// are exp(v_j + LSE_j) with the (updated or current) v.
// vshift (fast pass): the partials are column sums of B(u, v_old), i.e. the
// LSE in the frame shifted by v_old_j, removed here in fp64; a column whose
// combined fp32 sum is below 2^-64 of its scale may have flushed and sets
// ctl->col_flush (the exact pass then redoes every column).
constexpr double kColFlushRel = 5.421010862427522e-20;  // 2^-64
__global__ void __launch_bounds__(kSkThreads) k_sk_cols(SinkCtl* ctl, SinkVec sv, const double* colp, int64_t nrb, int fmt,
                                                        int update, int nblk_rows, const double* vshift, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int64_t n = ctl->n;
  const double un = sv.u[n];
  const int q = threadIdx.x % kSkTPI;
  const int64_t per_block = kSkThreads / kSkTPI, span = int64_t(gridDim.x) * per_block;
  double acc[4] = {0, 0, 0, 0};  // |col - c|, masked v.c
  bool flushed = false;
  for (int64_t j0 = int64_t(blockIdx.x) * per_block; j0 < n; j0 += span) {
    const int64_t j = j0 + threadIdx.x / kSkTPI;
    const bool live = j < n;
    const int64_t jj = live ? j : n - 1;
    double M, S;
    group_lse(colp, jj * nrb, nrb, fmt, q, M, S, n);
    if (!live || q != 0) continue;
    double lse;
    if (vshift) {
      const double vo = vshift[j];
      if (vo == -INFINITY) {
        lse = 0.0;  // c_j = 0: B's column is 0 whatever the LSE (v stays -inf)
      } else {
        if (!(S >= kColFlushRel)) flushed = true;
        lse_merge(M, S, (-0.0 + un) + vo, 1.0);
        lse = (M + log(S)) - vo;
      }
    } else {
      lse_merge(M, S, -0.0 + un, 1.0);
      lse = M + log(S);
    }
    double vj = sv.v[j];
    if (update) {
      vj = sv.log_c[j] - lse;
      sv.v[j] = vj;
      sv.zv_v[j] = vj;
      if (sv.zuv_v) sv.zuv_v[j] = vj;
    }
    const double col = exp(vj + lse);
    acc[0] += fabs(col - sv.c[j]);
    if (sv.c[j] > 0) acc[1] += vj * sv.c[j];
  }
  if (flushed) ctl->col_flush = 1;
  if (update && blockIdx.x == 0 && threadIdx.x == 0) sv.v[n] = sv.log_c[n] - ctl->col_lse_n;
  sk_block_store<4, kSkThreads>(acc, sv.scratch + 4 * nblk_rows);
}

__global__ void k_sk_commit_u(SinkCtl* ctl, SinkVec sv) {
  pdl_wait();
  if (!ctl->g_active) return;
  for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= ctl->n; i += int64_t(gridDim.x) * blockDim.x) {
    sv.u[i] = sv.u_next[i];
    if (sv.zuv_u && i < ctl->n) sv.zuv_u[i] = sv.u_next[i];
  }
}

__device__ void sk_loop_head(SinkCtl* ctl) {  // solvers.hpp:458-462
  if (!(ctl->error > ctl->tol)) { ctl->status = POTGPU_CONVERGED; ctl->g_active = 0; ctl->loop_end_ns = globaltimer_ns(); return; }
  if (ctl->it >= ctl->max_iterations) {
    ctl->status = POTGPU_MAX_ITERATIONS_EXCEEDED; ctl->g_active = 0; ctl->loop_end_ns = globaltimer_ns(); return;
  }
  if (ctl->it >= ctl->pause_at) { ctl->paused = 1; ctl->g_active = 0; ctl->loop_end_ns = globaltimer_ns(); return; }
  ctl->g_active = 1;
}

// E = |B1 - r|_1 + |B^T 1 - c|_1 (solvers.hpp:432-435), the trace's dual
// value (:436-438), record rule (:445) and the loop head.
__global__ void __launch_bounds__(kVecThreads) k_sk_scalars(SinkCtl* ctl, SinkVec sv, int nblk, int init, TraceDev* trace,
                                                            const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  double part[5] = {0, 0, 0, 0, 0};  // rerr, rsum, ur, cerr, vc
  for (int b = threadIdx.x; b < nblk; b += blockDim.x) {
    part[0] += sv.scratch[4 * b]; part[1] += sv.scratch[4 * b + 1]; part[2] += sv.scratch[4 * b + 2];
    part[3] += sv.scratch[4 * nblk + 4 * b]; part[4] += sv.scratch[4 * nblk + 4 * b + 1];
  }
  __shared__ double sh[5][kVecThreads];
  for (int q = 0; q < 5; ++q) sh[q][threadIdx.x] = part[q];
  __syncthreads();
  for (int s = kVecThreads / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s)
      for (int q = 0; q < 5; ++q) sh[q][threadIdx.x] += sh[q][threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x) return;
  const int64_t n = ctl->n;
  double rerr = sh[0][0], rsum = sh[1][0], ur = sh[2][0], cerr = sh[3][0], vc = sh[4][0];
  // dummy row n and column n
  const double rown = exp(sv.u[n] + ctl->row_lse_n);
  const double coln = exp(sv.v[n] + ctl->col_lse_n);
  rerr += fabs(rown - sv.r[n]);
  rsum += rown;
  if (sv.r[n] > 0) ur += sv.u[n] * sv.r[n];
  cerr += fabs(coln - sv.c[n]);
  if (sv.c[n] > 0) vc += sv.v[n] * sv.c[n];
  ctl->error = rerr + cerr;
  ctl->phi = (rsum - ur) - vc;
  sv.u_next[n] = sv.log_r[n] - ctl->row_lse_n;  // dummy row's u update
  ctl->sweeps += 2 + ctl->col_flush;  // + the exact column pass after a flush
  ctl->col_flush_count += ctl->col_flush;
  ctl->col_flush = 0;
  if (!init) ctl->it += 1;
  const int64_t it = ctl->it;
  if (init || it % ctl->log_every == 0 || !(ctl->error > ctl->tol)) {
    if (ctl->trace_len < ctl->trace_cap) {
      TraceDev& r = trace[ctl->trace_len];
      r.t = it; r.error = ctl->error; r.phi = ctl->phi;
      r.rounded_cost = __longlong_as_double(0x7ff8000000000000ULL);
      r.elapsed_s = double(globaltimer_ns() - ctl->t0_ns) * 1e-9;
    }
    ctl->trace_len += 1;
  }
  sk_loop_head(ctl);
}

__global__ void k_sk_resume(SinkCtl* ctl, int64_t pause_at) {
  pdl_wait();
  ctl->pause_at = pause_at;
  if (!ctl->paused) return;
  ctl->paused = 0;
  sk_loop_head(ctl);
}

__global__ void k_sk_stamp(SinkCtl* ctl) { ctl->t0_ns = globaltimer_ns(); }

}  // namespace potgpu
