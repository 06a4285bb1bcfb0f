// sweep.cuh — the n^2 hot path: one pass over B(z) = exp(-C/gamma + u_i + v_j + w)
// producing per-strip row partials, per-rowblock column partials and the
// max exponent, without ever transposing or materialising B.
//
// Reference counterpart: exponent_matrix + b_matrix + rowwise()/colwise()/
// sum() reductions (dual.hpp:93-133; solvers.hpp:46-52, 224-232).
//
// Tiling (sm_100a, 148 SMs): a warp owns a 256-column strip of one row per
// step (8 columns per lane, 128-bit coalesced loads), a CTA's 8 warps share
// the strip and interleave over the CTA's row range. Row sums are warp
// shuffles; column sums stay in registers across the CTA's rows and are
// combined across warps in shared memory, so the matrix is read once, in
// row order, and never transposed. All reductions are fixed-order
// (deterministic run to run).
#pragma once

#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"

namespace potgpu {

struct SweepArgs {
  int64_t n;            // plan side
  int64_t row_lo, row_hi;  // the row shard this launch covers ([0, n) unsharded)
  int rows_per_cta;
  const double* u;      // point (fp64 potentials)
  const double* v;
  const double* w;
  const double* lu;     // optional additive row log-weights (rounding), may be null
  const double* lv;     // optional additive column log-weights
  const double* rowshift;  // optional per-row / per-column exponent terms (log2 units) of the
  const double* colshift;  // source (expanded-norm points: -|x'_i|^2, -|y'_j|^2); may be null
  double* rowp;         // [n][gridDim.x]: row partials, one per strip (contiguous per row)
  double* colp;         // [n][gridDim.y]: column partials, one per row block
  double* maxp;         // [gridDim.y][gridDim.x]: max exponent (natural log units)
  const int* gate;      // kernel runs iff *gate != 0 (null: always)
  double gamma;         // for fp32 sources: exponent scale log2(e)/gamma folded in src
  // carried shifts of the points sweep (sweep_pts2_f32; null: exact path only)
  float* carry;             // [strip][n]: c_i of the last launch (log2 units, t' frame)
  float* carry_b;           // [n]: that launch's column constants B_j (one array per row shard)
  unsigned* carry_ticket;   // [strips]: last-CTA tickets (one array per row shard)
  unsigned long long* carry_stats;  // [2]: CTAs that took the carried / the exact path
  int tc_debug;  // timing experiments of sweep_tc_f32 ($POTGPU_TC_DEBUG; 0 = normal)
};

// ------------------------------------------------------------------------
// fp64, stored logK = -C/gamma (the reference's EntropicContext::logK,
// dual.hpp:67, computed once by IEEE division). Exponent association
// ((logK + u_i) + v_j) + w exactly as dual.hpp:94-97; exp with the Eigen
// packet clamp when FLOOR (the reference's B), plain exp for rounding
// sweeps. Padding columns of L hold -inf.
template <bool FLOOR>
__global__ void __launch_bounds__(kThreads, 2) sweep_f64_dense(const double* __restrict__ L, int64_t ld, SweepArgs a) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStripCols;
  double vj[8];
  bool ok[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t j = j0 + 2 * lane + 64 * k + e;
      ok[2 * k + e] = j < n;
      double vv = 0.0;
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
      }
      vj[2 * k + e] = vv;
    }
  }
  const double w = *a.w;
  double cacc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) cacc[k] = 0.0;
  double mx = -INFINITY;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    double ui = a.u[i];
    if (a.lu) ui = ui + a.lu[i];
    const double2* row = reinterpret_cast<const double2*>(L + i * ld + j0) + lane;
    double2 x[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) x[k] = __ldcs(row + 32 * k);
    double rs = 0.0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double e0 = ((x[k].x + ui) + vj[2 * k]) + w;
      const double e1 = ((x[k].y + ui) + vj[2 * k + 1]) + w;
      mx = fmax(mx, fmax(e0, e1));
      double b0 = exp(FLOOR ? fmax(e0, kExpLo) : e0);
      double b1 = exp(FLOOR ? fmax(e1, kExpLo) : e1);
      b0 = ok[2 * k] ? b0 : 0.0;
      b1 = ok[2 * k + 1] ? b1 : 0.0;
      rs += b0;
      rs += b1;
      cacc[2 * k] += b0;
      cacc[2 * k + 1] += b1;
    }
    rs = warp_sum(rs);
    if (lane == 0) a.rowp[i * gridDim.x + blockIdx.x] = rs;  // [row][strip]
  }
  __shared__ double cs[kWarps][kStripCols];
  __shared__ double ms[kWarps];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    cs[warp][2 * lane + 64 * k] = cacc[2 * k];
    cs[warp][2 * lane + 64 * k + 1] = cacc[2 * k + 1];
  }
  mx = warp_nanmax(mx);
  if (lane == 0) ms[warp] = mx;
  __syncthreads();
  const int t = threadIdx.x;
  double s = 0.0;
#pragma unroll
  for (int ww = 0; ww < kWarps; ++ww) s += cs[ww][t];
  if (j0 + t < n) a.colp[(j0 + t) * gridDim.y + blockIdx.y] = s;  // [col][row block]
  if (t == 0) {
    double m = ms[0];
    for (int ww = 1; ww < kWarps; ++ww) m = nan_max(m, ms[ww]);
    a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = m;
  }
}

// ------------------------------------------------------------------------
// fp32 sweeps. Exponent in log2 units t_ij = A_i + B_j - kappa_ij with
// A_i = (u_i + w) log2 e and B_j = v_j log2 e (fp32, from the fp64
// potentials) and kappa_ij = g2 C_ij (stored fp32 C) or |x'_i - y'_j|^2 with
// coordinates pre-scaled by sqrt(log2 e * scale / gamma) (on-the-fly).
//
// Each row segment of a warp (512 columns, 16 per lane) is exponentiated
// once with MUFU.EX2 at its exact max m_i, so the row's mass never over- or
// underflows; column accumulators carry a per-warp running scale sigma and
// take p_ij 2^(m_i - sigma). Partials leave as fp32 (sum, log2 scale) pairs
// and are turned into fp64 values by the reduce kernels, so the hot loop has
// no fp64 work at all.
constexpr int kPairs = 8;  // columns per lane / 2 (float2 pairs)
constexpr int kStripCols32 = 64 * kPairs;  // columns per warp strip

// Lane column map: pair q (0..7), half h: j = j0 + 4*lane + 128*(q>>1) + 2*(q&1) + h.
__device__ __forceinline__ int64_t f32_col(int64_t j0, int lane, int q, int h) {
  return j0 + 4 * lane + 128 * (q >> 1) + 2 * (q & 1) + h;
}

struct SrcDenseF32 {
  const float* C;
  int64_t ld;
  float g2;  // log2(e) / gamma
  struct Col {};
  struct RowData { float4 c[kPairs / 2]; };  // the lane's 2*kPairs entries of one row
  static constexpr bool kHasCols = false;
  __device__ __forceinline__ RowData load(int64_t i, int64_t j0, int lane) const {
    const float4* p = reinterpret_cast<const float4*>(C + i * ld + j0) + lane;
    RowData d;
#pragma unroll
    for (int k = 0; k < kPairs / 2; ++k) d.c[k] = __ldcs(p + 32 * k);
    return d;
  }
  // t' = B_j - g2 * C for the lane's 16 columns (the row potential is
  // added back in fp64 by the reduce kernels)
  __device__ __forceinline__ void expo(const RowData& d, const Col*, const float2 (&B)[kPairs], float2 (&t)[kPairs]) const {
    const float2 g = make_float2(-g2, -g2);
#pragma unroll
    for (int k = 0; k < kPairs / 2; ++k) {
      t[2 * k] = __ffma2_rn(g, make_float2(d.c[k].x, d.c[k].y), B[2 * k]);
      t[2 * k + 1] = __ffma2_rn(g, make_float2(d.c[k].z, d.c[k].w), B[2 * k + 1]);
    }
  }
};

struct SrcPointsF32 {
  const float4* Xs;  // pre-scaled coordinates (x, y, z, 0)
  const float4* Ys;
  struct Col { float2 x, y, z; };  // 2 columns per pair
  struct RowData { float4 p; };
  static constexpr bool kHasCols = true;
  __device__ __forceinline__ RowData load(int64_t i, int64_t, int) const { return RowData{Xs[i]}; }
  // t' = B_j - |x'_i - y'_j|^2 as an FFMA2 chain on d = y' - x'
  __device__ __forceinline__ void expo(const RowData& d, const Col* c, const float2 (&B)[kPairs], float2 (&t)[kPairs]) const {
    const float2 rx = make_float2(-d.p.x, -d.p.x), ry = make_float2(-d.p.y, -d.p.y), rz = make_float2(-d.p.z, -d.p.z);
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      const float2 dx = __fadd2_rn(rx, c[q].x);
      const float2 dy = __fadd2_rn(ry, c[q].y);
      const float2 dz = __fadd2_rn(rz, c[q].z);
      float2 tt = __ffma2_rn(make_float2(-dx.x, -dx.y), dx, B[q]);
      tt = __ffma2_rn(make_float2(-dy.x, -dy.y), dy, tt);
      t[q] = __ffma2_rn(make_float2(-dz.x, -dz.y), dz, tt);
    }
  }
};

// On-the-fly squared-Euclidean cost in expanded form: kappa = |x'|^2 +
// |y'|^2 - 2 x'.y'. The norms are exact fp64 terms folded into the row offset
// (rowshift = -|x'_i|^2) and the column constant (colshift = -|y'_j|^2), so
// the per-entry exponent is one 3-deep FFMA2 chain on (2 x'_i) . y'_j —
// half the FP32-pipe work of the difference form. Rounding happens at the
// magnitude of B_j, as in the difference form.
struct SrcPointsDotF32 {
  const float4* X2;  // 2 x'_i (exact doubling of the pre-scaled coordinates)
  const float4* Ys;  // y'_j
  struct Col { float2 x, y, z; };
  struct RowData { float4 p; };
  static constexpr bool kHasCols = true;
  __device__ __forceinline__ RowData load(int64_t i, int64_t, int) const { return RowData{X2[i]}; }
  __device__ __forceinline__ void expo(const RowData& d, const Col* c, const float2 (&B)[kPairs], float2 (&t)[kPairs]) const {
    const float2 px = make_float2(d.p.x, d.p.x), py = make_float2(d.p.y, d.p.y), pz = make_float2(d.p.z, d.p.z);
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      float2 tt = __ffma2_rn(px, c[q].x, B[q]);
      tt = __ffma2_rn(py, c[q].y, tt);
      t[q] = __ffma2_rn(pz, c[q].z, tt);
    }
  }
};

// Dynamic shared memory of the fp32 sweep: row potentials (rows_per_cta
// floats, padded to 16 B) then 8 per-warp 32x33 row-sum tiles.
__host__ __device__ constexpr int kRowTileOffset(int rows_per_cta) { return (rows_per_cta + 3) & ~3; }
__host__ __device__ constexpr size_t sweep_f32_smem(int rows_per_cta) {
  return size_t(kRowTileOffset(rows_per_cta) + kWarps * 32 * 33) * sizeof(float);
}

// Partial formats understood by the reduce kernels: fp64 values, or fp32
// (sum, log2 scale) pairs whose scale is relative to a per-row fp64 offset
// (rows: A_i = (u_i + lu_i + w) log2 e; columns: 0).
enum PartialFormat { PF_F64 = 0, PF_F32_SCALED = 1 };

__device__ __forceinline__ double partial_value(const double* p, int64_t idx, int fmt, double log2_offset = 0.0) {
  if (fmt == PF_F64) return p[idx];
  const float2 f = reinterpret_cast<const float2*>(p)[idx];
  return f.x == 0.f ? 0.0 : double(f.x) * exp2(double(f.y) + log2_offset);
}

template <class Src>
__global__ void __launch_bounds__(kThreads, 2) sweep_f32(Src src, SweepArgs a) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStripCols32;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  const double w = *a.w;
  // row potentials of this CTA's rows, once, into shared memory
  extern __shared__ float s_A[];
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
    double ud = a.u[i];
    if (a.lu) ud = ud + a.lu[i];
    double A = (ud + w) * kLog2e;
    if (a.rowshift) A = A + a.rowshift[i];
    s_A[i - r0] = float(A);
  }
  float2 Bj[kPairs];  // v_j log2 e (+ lv_j) (+ colshift_j)
  typename Src::Col cols[kPairs];
#pragma unroll
  for (int q = 0; q < kPairs; ++q) {
    float b[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;  // padding column: exp2(-inf) = 0, ignored by max
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
        vv = vv * kLog2e;
        if (a.colshift) vv = vv + a.colshift[j];
      }
      b[h] = float(vv);
    }
    Bj[q] = make_float2(b[0], b[1]);
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
  __syncthreads();
  float2 cacc[kPairs];
#pragma unroll
  for (int q = 0; q < kPairs; ++q) cacc[q] = make_float2(0.f, 0.f);
  float sigma = -INFINITY;  // running column scale (log2) of this warp
  float mmax = -INFINITY;
  float2* rowp = reinterpret_cast<float2*>(a.rowp);  // [row][strip]
  (void)rowp;
  // one-row-ahead software pipeline: the next row's data is in flight while
  // this row is exponentiated
  typename Src::RowData nxt{};
  if (r0 + warp < r1) nxt = src.load(r0 + warp, j0, lane);
  // Row sums: each lane parks its lane-local sum of a row in a per-warp
  // shared tile (32 rows x 33, conflict-free); every 32 rows lane L reduces
  // row L of the tile. No shuffle chain inside the row loop.
  float* tile = s_A + kRowTileOffset(a.rows_per_cta) + warp * (32 * 33);
  float* tslot = tile + lane;  // &tile[slot][lane]
  float my_ms = 0.f;  // max of tile row `lane`
  int slot = 0;
  int64_t ib = r0 + warp;  // first row of the tile
  const int64_t ldp = gridDim.x;
  auto flush = [&](int cnt) {
    __syncwarp();
    if (lane < cnt) {
      const float* rowv = tile + lane * 33;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; k += 4) { s0 += rowv[k]; s1 += rowv[k + 1]; s2 += rowv[k + 2]; s3 += rowv[k + 3]; }
      // value = sum 2^(ms + A_i); A_i is added in fp64 by the reduce kernels
      rowp[(ib + int64_t(kWarps) * lane) * ldp + blockIdx.x] = make_float2((s0 + s1) + (s2 + s3), my_ms);
    }
    __syncwarp();
  };
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    const typename Src::RowData cur = nxt;
    if (i + kWarps < r1) nxt = src.load(i + kWarps, j0, lane);
    const float Ai = s_A[i - r0];
    float2 t[kPairs];
    src.expo(cur, cols, Bj, t);  // t' = t - A_i
    float m = fmaxf(fmaxf(fmaxf(t[0].x, t[0].y), fmaxf(t[1].x, t[1].y)), fmaxf(fmaxf(t[2].x, t[2].y), fmaxf(t[3].x, t[3].y)));
#pragma unroll
    for (int q = 4; q < kPairs; q += 4)
      m = fmaxf(m, fmaxf(fmaxf(fmaxf(t[q].x, t[q].y), fmaxf(t[q + 1].x, t[q + 1].y)), fmaxf(fmaxf(t[q + 2].x, t[q + 2].y), fmaxf(t[q + 3].x, t[q + 3].y))));
    m = warp_maxf(m);
    // m == -inf only if the whole row segment is padding / -inf potentials
    const float ms = (m == -INFINITY) ? 0.f : m;
    const float2 M2 = make_float2(-ms, -ms);
    float2 p[kPairs];
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      const float2 d = __fadd2_rn(t[q], M2);
      p[q] = make_float2(ex2f(d.x), ex2f(d.y));
    }
    float2 rs = __fadd2_rn(__fadd2_rn(p[0], p[1]), __fadd2_rn(p[2], p[3]));
#pragma unroll
    for (int q = 4; q < kPairs; q += 4) rs = __fadd2_rn(rs, __fadd2_rn(__fadd2_rn(p[q], p[q + 1]), __fadd2_rn(p[q + 2], p[q + 3])));
    *tslot = rs.x + rs.y;
    tslot += 33;
    if (lane == slot) my_ms = ms;
    if (++slot == 32) {
      flush(32);
      slot = 0;
      tslot = tile + lane;
      ib = i + kWarps;
    }
    const float mA = (m == -INFINITY) ? -INFINITY : m + Ai;  // row max of t (log2)
    if (mA > sigma) {  // warp-uniform
      const float sc = ex2f(sigma - mA);
#pragma unroll
      for (int q = 0; q < kPairs; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
      sigma = mA;
    }
    mmax = fmaxf(mmax, mA);
    const float f = (mA == -INFINITY) ? 0.f : ex2f(mA - sigma);
    const float2 F2 = make_float2(f, f);
#pragma unroll
    for (int q = 0; q < kPairs; ++q) cacc[q] = __ffma2_rn(p[q], F2, cacc[q]);
  }
  if (slot > 0) flush(slot);
  // CTA combine of the 8 warps' column accumulators (each with its sigma)
  __shared__ float cs[kWarps][kStripCols32];
  __shared__ float ss[kWarps];
  __shared__ float mm[kWarps];
  if (lane == 0) {
    ss[warp] = sigma;
    mm[warp] = mmax;
  }
  __syncthreads();
  float sig = ss[0];
  for (int ww = 1; ww < kWarps; ++ww) sig = fmaxf(sig, ss[ww]);
  const float fw = (sigma == -INFINITY) ? 0.f : ex2f(sigma - sig);
#pragma unroll
  for (int q = 0; q < kPairs; ++q) {
    const int c = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
    cs[warp][c] = cacc[q].x * fw;
    cs[warp][c + 1] = cacc[q].y * fw;
  }
  __syncthreads();
  float2* colp = reinterpret_cast<float2*>(a.colp);  // [col][row block]
  for (int c = threadIdx.x; c < kStripCols32; c += kThreads) {
    float s = 0.f;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) s += cs[ww][c];
    if (j0 + c < n) colp[(j0 + c) * gridDim.y + blockIdx.y] = make_float2(sig == -INFINITY ? 0.f : s, sig == -INFINITY ? 0.f : sig);
  }
  if (threadIdx.x == 0) {
    float m = mm[0];
    for (int ww = 1; ww < kWarps; ++ww) m = fmaxf(m, mm[ww]);
    a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m) * kLn2;
  }
}

// ------------------------------------------------------------------------
// On-the-fly points sweep (C3, C4), software-pipelined on the row max.
// The warp max of a row segment (CREDUX.MAX) has a long latency; here row
// i+1's exponents are formed only to issue its max, and row i's exponents
// are recomputed (24 FFMA2) and exponentiated with the max issued one
// iteration earlier, so the reduction's latency hides behind a whole row of
// work without holding a second row of exponents in registers. The CTA's
// rows live in shared memory as (2 x'_i, A_i) float4s (no global loads in
// the row loop). Epilogue and partial formats as sweep_f32.
__host__ __device__ constexpr size_t sweep_pts_smem(int rows_per_cta, bool cluster_merge = false) {
  // (2x', A_i) rows, the per-warp row-sum tiles (+ the row partials of the cluster merge)
  return size_t(rows_per_cta) * sizeof(float4) + size_t(kWarps * 32 * 33) * sizeof(float) +
         (cluster_merge ? size_t(rows_per_cta) * sizeof(float2) : 0);
}

// Balanced reductions over a lane's KP column pairs (depth log2(2 KP)
// instead of a 2 KP-long dependency chain).
template <int KP>
__device__ __forceinline__ float tree_max2(const float2 (&t)[KP]) {
  float m[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) m[q] = fmaxf(t[q].x, t[q].y);
#pragma unroll
  for (int w = 1; w < KP; w *= 2)
#pragma unroll
    for (int q = 0; q + w < KP; q += 2 * w) m[q] = fmaxf(m[q], m[q + w]);
  return m[0];
}

template <int KP>
__device__ __forceinline__ float tree_sum2(const float2 (&t)[KP]) {
  float2 m[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) m[q] = t[q];
#pragma unroll
  for (int w = 1; w < KP; w *= 2)
#pragma unroll
    for (int q = 0; q + w < KP; q += 2 * w) m[q] = __fadd2_rn(m[q], m[q + w]);
  return m[0].x + m[0].y;
}

// sum_q (t_q . g_q) over a lane's KP column pairs as two FFMA2 chains
// (KP + 2 operations instead of the 2 KP of a product array + sum tree).
template <int KP>
__device__ __forceinline__ float wsum2(const float2 (&t)[KP], const float2 (&g)[KP]) {
  static_assert(KP % 2 == 0, "pairs in two chains");
  float2 a0 = __fmul2_rn(t[0], g[0]), a1 = __fmul2_rn(t[1], g[1]);
#pragma unroll
  for (int q = 2; q < KP; q += 2) {
    a0 = __ffma2_rn(t[q], g[q], a0);
    a1 = __ffma2_rn(t[q + 1], g[q + 1], a1);
  }
  const float2 s = __fadd2_rn(a0, a1);
  return s.x + s.y;
}

// KP column pairs per lane (2 KP columns, a 64 KP-column warp strip); KP = 8
// matches sweep_f32's map. Fewer pairs -> fewer registers -> more resident
// warps to cover the per-row dependency chain (profiles/pts_variants.sh).
template <int KP>
__global__ void __launch_bounds__(kThreads, (KP <= 4 ? 3 : 2)) sweep_pts_f32(SrcPointsDotF32 src, SweepArgs a) {
  pdl_wait();
  constexpr int kStrip = 64 * KP;
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStrip;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  const double w = *a.w;
  extern __shared__ float4 s_R[];  // [rows_per_cta]: (2x', A_i), then the row-sum tiles
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
    double ud = a.u[i];
    if (a.lu) ud = ud + a.lu[i];
    double A = (ud + w) * kLog2e;
    if (a.rowshift) A = A + a.rowshift[i];
    const float4 x2 = src.X2[i];
    s_R[i - r0] = make_float4(x2.x, x2.y, x2.z, float(A));
  }
  float2 Bj[KP], cx[KP], cy[KP], cz[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    float b[2];
    float4 y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;  // padding column: exp2(-inf) = 0, ignored by max
      y[h] = make_float4(0, 0, 0, 0);
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
        vv = vv * kLog2e;
        if (a.colshift) vv = vv + a.colshift[j];
        y[h] = src.Ys[j];
      }
      b[h] = float(vv);
    }
    Bj[q] = make_float2(b[0], b[1]);
    cx[q] = make_float2(y[0].x, y[1].x);
    cy[q] = make_float2(y[0].y, y[1].y);
    cz[q] = make_float2(y[0].z, y[1].z);
  }
  __syncthreads();
  float2 cacc[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) cacc[q] = make_float2(0.f, 0.f);
  float sigma = -INFINITY;
  float mmax = -INFINITY;
  float2* rowp = reinterpret_cast<float2*>(a.rowp);  // [row][strip]
  float* tile = reinterpret_cast<float*>(s_R + a.rows_per_cta) + warp * (32 * 33);
  float* tslot = tile + lane;
  float my_ms = 0.f;
  int slot = 0;
  int64_t ib = r0 + warp;
  const int64_t ldp = gridDim.x;
  auto flush = [&](int cnt) {
    __syncwarp();
    if (lane < cnt) {
      const float* rowv = tile + lane * 33;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; k += 4) { s0 += rowv[k]; s1 += rowv[k + 1]; s2 += rowv[k + 2]; s3 += rowv[k + 3]; }
      rowp[(ib + int64_t(kWarps) * lane) * ldp + blockIdx.x] = make_float2((s0 + s1) + (s2 + s3), my_ms);
    }
    __syncwarp();
  };
  for (int64_t i = r0 + warp; i < r1; i += kWarps) {
    const float4 dc = s_R[i - r0];
    const float2 px = make_float2(dc.x, dc.x), py = make_float2(dc.y, dc.y), pz = make_float2(dc.z, dc.z);
    float2 t[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      float2 tt = __ffma2_rn(px, cx[q], Bj[q]);
      tt = __ffma2_rn(py, cy[q], tt);
      t[q] = __ffma2_rn(pz, cz[q], tt);
    }
    float m = fmaxf(t[0].x, t[0].y);
#pragma unroll
    for (int q = 1; q < KP; ++q) m = fmaxf(m, fmaxf(t[q].x, t[q].y));
    m = warp_maxf(m);
    const float Ai = dc.w;
    const float ms = (m == -INFINITY) ? 0.f : m;
    const float2 M2 = make_float2(-ms, -ms);
    float2 p[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float2 d = __fadd2_rn(t[q], M2);
      p[q] = make_float2(ex2f(d.x), ex2f(d.y));
    }
    *tslot = tree_sum2<KP>(p);
    tslot += 33;
    if (lane == slot) my_ms = ms;
    if (++slot == 32) {
      flush(32);
      slot = 0;
      tslot = tile + lane;
      ib = i + kWarps;
    }
    const float mA = (m == -INFINITY) ? -INFINITY : m + Ai;
    if (mA > sigma) {  // warp-uniform
      const float sc = ex2f(sigma - mA);
#pragma unroll
      for (int q = 0; q < KP; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
      sigma = mA;
    }
    mmax = fmaxf(mmax, mA);
    const float f = (mA == -INFINITY) ? 0.f : ex2f(mA - sigma);
    const float2 F2 = make_float2(f, f);
#pragma unroll
    for (int q = 0; q < KP; ++q) cacc[q] = __ffma2_rn(p[q], F2, cacc[q]);
  }
  if (slot > 0) flush(slot);
  __shared__ float cs[kWarps][kStrip];
  __shared__ float ss[kWarps];
  __shared__ float mm[kWarps];
  if (lane == 0) {
    ss[warp] = sigma;
    mm[warp] = mmax;
  }
  __syncthreads();
  float sig = ss[0];
  for (int ww = 1; ww < kWarps; ++ww) sig = fmaxf(sig, ss[ww]);
  const float fw = (sigma == -INFINITY) ? 0.f : ex2f(sigma - sig);
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int c = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
    cs[warp][c] = cacc[q].x * fw;
    cs[warp][c + 1] = cacc[q].y * fw;
  }
  __syncthreads();
  float2* colp = reinterpret_cast<float2*>(a.colp);
  for (int c = threadIdx.x; c < kStrip; c += kThreads) {
    float s = 0.f;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) s += cs[ww][c];
    if (j0 + c < n) colp[(j0 + c) * gridDim.y + blockIdx.y] = make_float2(sig == -INFINITY ? 0.f : s, sig == -INFINITY ? 0.f : sig);
  }
  if (threadIdx.x == 0) {
    float m = mm[0];
    for (int ww = 1; ww < kWarps; ++ww) m = fmaxf(m, mm[ww]);
    a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m) * kLn2;
  }
}

// Two-row variant of sweep_pts_f32<8>: a warp exponentiates rows i and
// i + 8 in one iteration (two independent max / CREDUX / MUFU chains in
// flight). The column constants B'_j live in shared memory ([pair][lane]
// float2, conflict-free) so the second row's exponents fit in registers.
// CS > 1: launched in clusters of CS CTAs along the strips; the row partials
// of the cluster's CS strips are merged through distributed shared memory
// before they are written (one partial per row per cluster: CS x fewer for
// the evaluation to read).
//
// Carried shifts (a.carry != null, CS == 1). The exact path above serialises
// every row: segment max -> CREDUX -> shift -> 32-wide MUFU burst, and the
// warps of a scheduler fall into lock step (all in their FMA phase with the
// MUFU idle, then all in the MUFU burst). The shift only has to be an upper
// bound of the row segment's max within ~60 log2 units (fp32 keeps its
// relative precision at any magnitude; only over- and underflow matter), and
// one is known before the sweep starts:
//   t'_ij = B_j + 2 x'_i . y'_j   (the row offset A_i is not in t'),
//   max_j t'_new <= max_j t'_old + max_j (B_new - B_old)_j  over the strip,
// and the previous launch left c_i = s_i + log2(sum_j 2^(t'_old - s_i)), which
// lies in [max t'_old, max t'_old + log2(512)]. So s_i = c_i + dB_max bounds
// the new max from above with slack <= 9 + (dB_max - dB_min). A CTA whose
// strip moved by at most kCarrySpread takes this path: no max tree, no
// CREDUX, no per-row column-scale MUFU (one CTA-wide column scale sigma,
// f_i = 2^(s_i + A_i - sigma) formed in the prologue), and each pair's MUFU
// depends only on its own 3-FFMA2 chain, so the MUFU work interleaves freely
// with the FMA work. Row partials are (sum, s_i): the same format. The max
// exponent of the CTA (the reference's 700 overflow test, dual.hpp:85-90) is
// reported as the bound max_i (c_i^new + A_i) (exact to within 9 log2 units)
// and recomputed exactly when that bound is within 10 of the threshold.
// Every launch (either path) writes its carries c_i and its column constants
// (the latter by the strip's last CTA, by ticket), so the state stays
// consistent whichever launch ran last.
constexpr float kCarrySpread = 48.f;
__host__ __device__ constexpr size_t sweep_pts2_smem(int rows_per_cta, bool cluster_merge = false) {
  // + (f_i, A_i) per row for the carried path
  return sweep_pts_smem(rows_per_cta, cluster_merge) + size_t(rows_per_cta) * sizeof(float2);
}

template <int CS>
__global__ void __launch_bounds__(kThreads, 2) sweep_pts2_f32(SrcPointsDotF32 src, SweepArgs a) {
  pdl_wait();
  constexpr int KP = kPairs;
  constexpr int kStrip = 64 * KP;
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStrip;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  const int nrows = int(r1 - r0);
  const double w = *a.w;
  const bool use_carry = CS == 1 && a.carry != nullptr;
  extern __shared__ float4 s_R[];  // [rows_per_cta]: (2x', A_i) or (2x', s_i), then the row-sum tiles, then (f_i, A_i)
  // column constants B'_j of the strip, two column pairs per 16-byte word (one LDS.128 per two pairs)
  __shared__ float4 s_B4[KP / 2][32];
  auto Bof = [&](int q, int l) -> float2 {
    const float4 v = s_B4[q >> 1][l];
    return (q & 1) ? make_float2(v.z, v.w) : make_float2(v.x, v.y);
  };
  __shared__ float s_red[3][kWarps];
  float2* s_FA = reinterpret_cast<float2*>(reinterpret_cast<float*>(s_R + a.rows_per_cta) + kWarps * 32 * 33 +
                                           (CS > 1 ? 2 * a.rows_per_cta : 0));
  float2 cx[KP], cy[KP], cz[KP];
  float dmax = -INFINITY, dmin = INFINITY;
  int dbad = 0;
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    float b[2];
    float4 y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;
      y[h] = make_float4(0, 0, 0, 0);
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
        vv = vv * kLog2e;
        if (a.colshift) vv = vv + a.colshift[j];
        y[h] = src.Ys[j];
      }
      b[h] = float(vv);
      if (use_carry && j < n) {
        const float bo = a.carry_b[j];
        if (!(b[h] == -INFINITY && bo == -INFINITY)) {  // a column masked before and after moves nothing
          const float d = b[h] - bo;
          dbad |= !(fabsf(d) < 1e30f);  // NaN, +-inf: a column appeared, vanished or is not finite
          dmax = fmaxf(dmax, d);
          dmin = fminf(dmin, d);
        }
      }
    }
    if (warp == 0) reinterpret_cast<float2*>(&s_B4[q >> 1][lane])[q & 1] = make_float2(b[0], b[1]);
    cx[q] = make_float2(y[0].x, y[1].x);
    cy[q] = make_float2(y[0].y, y[1].y);
    cz[q] = make_float2(y[0].z, y[1].z);
  }
  bool carried = false;
  float dBmax = 0.f;
  if (use_carry) {
    dbad = __any_sync(0xffffffffu, dbad);
    dmax = warp_maxf(dmax);
    dmin = -warp_maxf(-dmin);
    if (lane == 0) { s_red[0][warp] = dmax; s_red[1][warp] = dmin; s_red[2][warp] = dbad ? 1.f : 0.f; }
    __syncthreads();
    float dx = -INFINITY, dn = INFINITY, bad = 0.f;
    for (int ww = 0; ww < kWarps; ++ww) { dx = fmaxf(dx, s_red[0][ww]); dn = fminf(dn, s_red[1][ww]); bad += s_red[2][ww]; }
    carried = bad == 0.f && dx > -INFINITY && dx - dn <= kCarrySpread;
    dBmax = dx;
    __syncthreads();  // s_red is reused below
  }
  // rows: (2x', A_i), or for the carried path (2x', s_i) and (f_i, A_i)
  float lsig = -INFINITY;
  int rbad = 0;
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
    double ud = a.u[i];
    if (a.lu) ud = ud + a.lu[i];
    double A = (ud + w) * kLog2e;
    if (a.rowshift) A = A + a.rowshift[i];
    const float4 x2 = src.X2[i];
    const float Af = float(A);
    if (carried) {
      const float si = a.carry[int64_t(blockIdx.x) * n + i] + dBmax;
      rbad |= !(fabsf(si) < 1e30f) || !(fabsf(Af) < 1e30f);
      lsig = fmaxf(lsig, si + Af);
      s_R[i - r0] = make_float4(x2.x, x2.y, x2.z, si);
      s_FA[i - r0] = make_float2(0.f, Af);
    } else {
      s_R[i - r0] = make_float4(x2.x, x2.y, x2.z, Af);
      if (use_carry) s_FA[i - r0] = make_float2(0.f, Af);
    }
  }
  float sigma_c = -INFINITY;
  if (carried) {
    rbad = __syncthreads_or(rbad);
    lsig = warp_maxf(lsig);
    if (lane == 0) s_red[0][warp] = lsig;
    __syncthreads();
    for (int ww = 0; ww < kWarps; ++ww) sigma_c = fmaxf(sigma_c, s_red[0][ww]);
    if (rbad || !(sigma_c > -INFINITY)) {
      carried = false;  // CTA-uniform: back to the exact path, rows as (2x', A_i)
      for (int k = threadIdx.x; k < nrows; k += kThreads) s_R[k].w = s_FA[k].y;
    } else {
      for (int k = threadIdx.x; k < nrows; k += kThreads) s_FA[k].x = ex2f(s_R[k].w + s_FA[k].y - sigma_c);
    }
  }
  __syncthreads();
  if (use_carry && a.carry_stats && threadIdx.x == 0) atomicAdd(a.carry_stats + (carried ? 0 : 1), 1ull);
  float2 cacc[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) cacc[q] = make_float2(0.f, 0.f);
  float sigma = carried ? sigma_c : -INFINITY;
  float mmax = -INFINITY;
  float ubmax = -INFINITY;  // carried: max over flushed rows of c_i + A_i
  int ubnan = 0;
  float2* rowp = reinterpret_cast<float2*>(a.rowp);
  float* tile = reinterpret_cast<float*>(s_R + a.rows_per_cta) + warp * (32 * 33);
  float2* s_rp = reinterpret_cast<float2*>(reinterpret_cast<float*>(s_R + a.rows_per_cta) + kWarps * 32 * 33);  // [rows]
  float* tslot = tile + lane;
  float my_ms = 0.f;
  int slot = 0;
  int64_t ib = r0 + warp;
  const int64_t ldp = gridDim.x;
  auto flush = [&](int cnt) {
    __syncwarp();
    if (lane < cnt) {
      const float* rowv = tile + lane * 33;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; k += 4) { s0 += rowv[k]; s1 += rowv[k + 1]; s2 += rowv[k + 2]; s3 += rowv[k + 3]; }
      const float sum = (s0 + s1) + (s2 + s3);
      const int64_t row = ib + int64_t(kWarps) * lane;
      const float2 part = make_float2(sum, my_ms);
      if constexpr (CS > 1) s_rp[row - r0] = part;
      else rowp[row * ldp + blockIdx.x] = part;
      if (use_carry) {
        float lg;
        asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(sum));
        const float c = my_ms + lg;  // -inf for an empty segment
        a.carry[int64_t(blockIdx.x) * n + row] = c;
        const float ub = c + s_FA[row - r0].y;
        ubnan |= ub != ub;
        ubmax = fmaxf(ubmax, ub);
      }
    }
    __syncwarp();
  };
  auto next_slot = [&](float ms, int64_t i) {
    tslot += 33;
    if (lane == slot) my_ms = ms;
    if (++slot == 32) {
      flush(32);
      slot = 0;
      tslot = tile + lane;
      ib = i + kWarps;
    }
  };
  // exact path: one row's tile slot, column scale update and accumulation
  auto finish_row = [&](float m, float Ai, const float2 (&p)[KP], int64_t i) {
    const float ms = (m == -INFINITY) ? 0.f : m;
    *tslot = tree_sum2<KP>(p);
    next_slot(ms, i);
    const float mA = (m == -INFINITY) ? -INFINITY : m + Ai;
    if (mA > sigma) {
      const float sc = ex2f(sigma - mA);
#pragma unroll
      for (int q = 0; q < KP; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
      sigma = mA;
    }
    mmax = fmaxf(mmax, mA);
    const float f = (mA == -INFINITY) ? 0.f : ex2f(mA - sigma);
    const float2 F2 = make_float2(f, f);
#pragma unroll
    for (int q = 0; q < KP; ++q) cacc[q] = __ffma2_rn(p[q], F2, cacc[q]);
  };
  // carried path: exponents at the carried shift, column scale f_i precomputed
  auto finish_row_c = [&](float si, float fi, const float2 (&p)[KP], int64_t i) {
    *tslot = tree_sum2<KP>(p);
    next_slot(si, i);
    const float2 F2 = make_float2(fi, fi);
#pragma unroll
    for (int q = 0; q < KP; ++q) cacc[q] = __ffma2_rn(p[q], F2, cacc[q]);
  };
  int64_t i = r0 + warp;
  if (carried) {
    for (; i + kWarps < r1; i += 2 * kWarps) {  // rows i and i + 8
      const float4 da = s_R[i - r0], db = s_R[i + kWarps - r0];
      const float fa = s_FA[i - r0].x, fb = s_FA[i + kWarps - r0].x;
      float2 ta[KP], tb[KP];
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 B = Bof(q, lane);
        float2 xa = __ffma2_rn(make_float2(da.x, da.x), cx[q], B);
        float2 xb = __ffma2_rn(make_float2(db.x, db.x), cx[q], B);
        xa = __ffma2_rn(make_float2(da.y, da.y), cy[q], xa);
        xb = __ffma2_rn(make_float2(db.y, db.y), cy[q], xb);
        xa = __ffma2_rn(make_float2(da.z, da.z), cz[q], xa);
        xb = __ffma2_rn(make_float2(db.z, db.z), cz[q], xb);
        const float2 d = __fadd2_rn(xa, make_float2(-da.w, -da.w));
        const float2 e = __fadd2_rn(xb, make_float2(-db.w, -db.w));
        ta[q] = make_float2(ex2f(d.x), ex2f(d.y));
        tb[q] = make_float2(ex2f(e.x), ex2f(e.y));
      }
      finish_row_c(da.w, fa, ta, i);
      finish_row_c(db.w, fb, tb, i + kWarps);
    }
    if (i < r1) {
      const float4 da = s_R[i - r0];
      const float fa = s_FA[i - r0].x;
      float2 ta[KP];
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 B = Bof(q, lane);
        float2 xa = __ffma2_rn(make_float2(da.x, da.x), cx[q], B);
        xa = __ffma2_rn(make_float2(da.y, da.y), cy[q], xa);
        xa = __ffma2_rn(make_float2(da.z, da.z), cz[q], xa);
        const float2 d = __fadd2_rn(xa, make_float2(-da.w, -da.w));
        ta[q] = make_float2(ex2f(d.x), ex2f(d.y));
      }
      finish_row_c(da.w, fa, ta, i);
    }
  } else {
    for (; i + kWarps < r1; i += 2 * kWarps) {  // rows i and i + 8
      const float4 da = s_R[i - r0], db = s_R[i + kWarps - r0];
      float2 ta[KP], tb[KP];
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 B = Bof(q, lane);
        float2 xa = __ffma2_rn(make_float2(da.x, da.x), cx[q], B);
        float2 xb = __ffma2_rn(make_float2(db.x, db.x), cx[q], B);
        xa = __ffma2_rn(make_float2(da.y, da.y), cy[q], xa);
        xb = __ffma2_rn(make_float2(db.y, db.y), cy[q], xb);
        ta[q] = __ffma2_rn(make_float2(da.z, da.z), cz[q], xa);
        tb[q] = __ffma2_rn(make_float2(db.z, db.z), cz[q], xb);
      }
      float ma = tree_max2<KP>(ta), mb = tree_max2<KP>(tb);
      ma = warp_maxf(ma);
      mb = warp_maxf(mb);
      const float msa = (ma == -INFINITY) ? 0.f : ma, msb = (mb == -INFINITY) ? 0.f : mb;
      // The column scale of both rows needs the maxima only: it is formed
      // BEFORE the 32 exponentials, so each pair's column accumulation and
      // the row-sum trees issue in the gaps of the MUFU burst (ptxas paces
      // MUFU.EX2 at one per 8 cycles per warp) instead of after it. Measured
      // on B200: C3 sweep 0.1072 -> 0.1054 ms, C4 1.512 -> 1.473 ms.
      const float mAa = (ma == -INFINITY) ? -INFINITY : ma + da.w;
      const float mAb = (mb == -INFINITY) ? -INFINITY : mb + db.w;
      const float mAx = fmaxf(mAa, mAb);
      if (mAx > sigma) {
        const float sc = ex2f(sigma - mAx);
#pragma unroll
        for (int q = 0; q < KP; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
        sigma = mAx;
      }
      mmax = fmaxf(mmax, mAx);
      const float fa = (mAa == -INFINITY) ? 0.f : ex2f(mAa - sigma);
      const float fb = (mAb == -INFINITY) ? 0.f : ex2f(mAb - sigma);
      const float2 Fa = make_float2(fa, fa), Fb = make_float2(fb, fb);
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 d = __fadd2_rn(ta[q], make_float2(-msa, -msa));
        ta[q] = make_float2(ex2f(d.x), ex2f(d.y));
        cacc[q] = __ffma2_rn(ta[q], Fa, cacc[q]);
      }
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 e = __fadd2_rn(tb[q], make_float2(-msb, -msb));
        tb[q] = make_float2(ex2f(e.x), ex2f(e.y));
        cacc[q] = __ffma2_rn(tb[q], Fb, cacc[q]);
      }
      // both rows' tile slots in one step (the slot count is even here: only two-row steps precede)
      tslot[0] = tree_sum2<KP>(ta);
      tslot[33] = tree_sum2<KP>(tb);
      tslot += 66;
      if (lane == slot) my_ms = msa;
      if (lane == slot + 1) my_ms = msb;
      slot += 2;
      if (slot == 32) {
        flush(32);
        slot = 0;
        tslot = tile + lane;
        ib = i + 2 * kWarps;
      }
    }
    if (i < r1) {  // a last single row
      const float4 da = s_R[i - r0];
      float2 ta[KP];
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 B = Bof(q, lane);
        float2 xa = __ffma2_rn(make_float2(da.x, da.x), cx[q], B);
        xa = __ffma2_rn(make_float2(da.y, da.y), cy[q], xa);
        ta[q] = __ffma2_rn(make_float2(da.z, da.z), cz[q], xa);
      }
      float ma = fmaxf(ta[0].x, ta[0].y);
#pragma unroll
      for (int q = 1; q < KP; ++q) ma = fmaxf(ma, fmaxf(ta[q].x, ta[q].y));
      ma = warp_maxf(ma);
      const float msa = (ma == -INFINITY) ? 0.f : ma;
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 d = __fadd2_rn(ta[q], make_float2(-msa, -msa));
        ta[q] = make_float2(ex2f(d.x), ex2f(d.y));
      }
      finish_row(ma, da.w, ta, i);
    }
  }
  if (slot > 0) flush(slot);
  __shared__ float cs[kWarps][kStrip];
  __shared__ float ss[kWarps];
  __shared__ float mm[kWarps];
  if (carried) {
    // the bound of the CTA's max exponent; exact when it is near the
    // reference's overflow threshold (kMaxExponent, natural log units)
    ubnan = __any_sync(0xffffffffu, ubnan);
    float ub = ubnan ? NAN : warp_maxf(ubmax);
    if (lane == 0) s_red[0][warp] = ub;
    __syncthreads();
    float cub = s_red[0][0];
    for (int ww = 1; ww < kWarps; ++ww) cub = (cub != cub || s_red[0][ww] != s_red[0][ww]) ? NAN : fmaxf(cub, s_red[0][ww]);
    mmax = cub;
    if (double(cub) * kLn2 > kMaxExponent - 10.0) {  // CTA-uniform, rare: the exact max of t' + A_i
      mmax = -INFINITY;
      for (int64_t k = r0 + warp; k < r1; k += kWarps) {
        const float4 d = s_R[k - r0];
        float2 t[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 B = Bof(q, lane);
          float2 x = __ffma2_rn(make_float2(d.x, d.x), cx[q], B);
          x = __ffma2_rn(make_float2(d.y, d.y), cy[q], x);
          t[q] = __ffma2_rn(make_float2(d.z, d.z), cz[q], x);
        }
        const float m = warp_maxf(tree_max2<KP>(t));
        if (m != -INFINITY) mmax = fmaxf(mmax, m + s_FA[k - r0].y);
      }
    }
  }
  if (lane == 0) {
    ss[warp] = sigma;
    mm[warp] = mmax;
  }
  __syncthreads();
  float sig = ss[0];
  for (int ww = 1; ww < kWarps; ++ww) sig = fmaxf(sig, ss[ww]);
  const float fw = (sigma == -INFINITY) ? 0.f : ex2f(sigma - sig);
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int c = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
    cs[warp][c] = cacc[q].x * fw;
    cs[warp][c + 1] = cacc[q].y * fw;
  }
  __syncthreads();
  float2* colp = reinterpret_cast<float2*>(a.colp);
  for (int c = threadIdx.x; c < kStrip; c += kThreads) {
    float s = 0.f;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) s += cs[ww][c];
    if (j0 + c < n) colp[(j0 + c) * gridDim.y + blockIdx.y] = make_float2(sig == -INFINITY ? 0.f : s, sig == -INFINITY ? 0.f : sig);
  }
  if constexpr (CS > 1) {
    // merge the cluster's row partials (sum, log2 scale) per row through DSMEM
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    cl.sync();
    const int rank = int(cl.block_rank());
    const int64_t ldc = gridDim.x / CS;
    const int64_t col = blockIdx.x / CS;
    for (int lr = rank * kThreads + threadIdx.x; lr < nrows; lr += CS * kThreads) {
      float2 q[CS];
#pragma unroll
      for (int c = 0; c < CS; ++c) q[c] = cl.map_shared_rank(s_rp, c)[lr];
      float M = -INFINITY;
#pragma unroll
      for (int c = 0; c < CS; ++c)
        if (q[c].x != 0.f) M = fmaxf(M, q[c].y);
      float S = 0.f;
      if (M != -INFINITY)
#pragma unroll
        for (int c = 0; c < CS; ++c)
          if (q[c].x != 0.f) S += q[c].x * ex2f(q[c].y - M);
      rowp[(r0 + lr) * ldc + col] = M == -INFINITY ? make_float2(0.f, 0.f) : make_float2(S, M);
    }
    cl.sync();  // keep this CTA's shared memory until every remote read is done
  }
  if (threadIdx.x == 0) {
    float m = mm[0];
    for (int ww = 1; ww < kWarps; ++ww) m = (m != m || mm[ww] != mm[ww]) ? NAN : fmaxf(m, mm[ww]);
    a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m) * kLn2;
  }
  if (use_carry) {
    // the strip's column constants for the next launch: written by the last
    // CTA of the strip, after every CTA of it has read the previous ones
    __shared__ int s_last;
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(a.carry_ticket + blockIdx.x, 1u) == gridDim.y - 1;
    }
    __syncthreads();
    if (s_last) {
      for (int k = threadIdx.x; k < kStrip; k += kThreads) {
        const int q = k >> 5, l = k & 31;
        const float2 b = Bof(q, l);
        const int64_t jj = f32_col(j0, l, q, 0);
        if (jj < n) a.carry_b[jj] = b.x;
        if (jj + 1 < n) a.carry_b[jj + 1] = b.y;
      }
      if (threadIdx.x == 0) a.carry_ticket[blockIdx.x] = 0u;
    }
  }
}

// sweep_pts2_f32 with the column constants in shared memory instead of
// registers ($POTGPU_PTS_PAIRS=3): ~48 fewer registers for 3 CTAs (24
// warps) per SM to cover the per-row dependency chain, at the cost of two
// LDS.128 per column pair and warp step. Rows per CTA are capped at
// kMaxRowsPerCtaS so three CTAs' shared memory fits; the epilogue's column
// combine reuses the row-sum tiles.
constexpr int64_t kMaxRowsPerCtaS = 1280;
__global__ void __launch_bounds__(kThreads, 3) sweep_pts2s_f32(SrcPointsDotF32 src, SweepArgs a) {
  pdl_wait();
  constexpr int KP = kPairs;
  constexpr int kStrip = 64 * KP;
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStrip;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  const double w = *a.w;
  extern __shared__ float4 s_R[];  // [rows_per_cta]: (2x', A_i), then the row-sum tiles
  // the lane's column constants: (cx, cy) and (cz, B') per pair, read per warp step
  __shared__ float4 s_XY[KP][32], s_ZB[KP][32];
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
    double ud = a.u[i];
    if (a.lu) ud = ud + a.lu[i];
    double A = (ud + w) * kLog2e;
    if (a.rowshift) A = A + a.rowshift[i];
    const float4 x2 = src.X2[i];
    s_R[i - r0] = make_float4(x2.x, x2.y, x2.z, float(A));
  }
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    if (warp != 0) break;
    float b[2];
    float4 y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;
      y[h] = make_float4(0, 0, 0, 0);
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
        vv = vv * kLog2e;
        if (a.colshift) vv = vv + a.colshift[j];
        y[h] = src.Ys[j];
      }
      b[h] = float(vv);
    }
    s_XY[q][lane] = make_float4(y[0].x, y[1].x, y[0].y, y[1].y);
    s_ZB[q][lane] = make_float4(y[0].z, y[1].z, b[0], b[1]);
  }
  __syncthreads();
  float2 cacc[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) cacc[q] = make_float2(0.f, 0.f);
  float sigma = -INFINITY;
  float mmax = -INFINITY;
  float2* rowp = reinterpret_cast<float2*>(a.rowp);
  float* tile = reinterpret_cast<float*>(s_R + a.rows_per_cta) + warp * (32 * 33);
  float* tslot = tile + lane;
  float my_ms = 0.f;
  int slot = 0;
  int64_t ib = r0 + warp;
  const int64_t ldp = gridDim.x;
  auto flush = [&](int cnt) {
    __syncwarp();
    if (lane < cnt) {
      const float* rowv = tile + lane * 33;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; k += 4) { s0 += rowv[k]; s1 += rowv[k + 1]; s2 += rowv[k + 2]; s3 += rowv[k + 3]; }
      const float2 part = make_float2((s0 + s1) + (s2 + s3), my_ms);
      rowp[(ib + int64_t(kWarps) * lane) * ldp + blockIdx.x] = part;
    }
    __syncwarp();
  };
  // one row's tile slot, column scale update and accumulation
  auto finish_row = [&](float m, float Ai, const float2 (&p)[KP], int64_t i) {
    const float ms = (m == -INFINITY) ? 0.f : m;
    *tslot = tree_sum2<KP>(p);
    tslot += 33;
    if (lane == slot) my_ms = ms;
    if (++slot == 32) {
      flush(32);
      slot = 0;
      tslot = tile + lane;
      ib = i + kWarps;
    }
    const float mA = (m == -INFINITY) ? -INFINITY : m + Ai;
    if (mA > sigma) {
      const float sc = ex2f(sigma - mA);
#pragma unroll
      for (int q = 0; q < KP; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
      sigma = mA;
    }
    mmax = fmaxf(mmax, mA);
    const float f = (mA == -INFINITY) ? 0.f : ex2f(mA - sigma);
    const float2 F2 = make_float2(f, f);
#pragma unroll
    for (int q = 0; q < KP; ++q) cacc[q] = __ffma2_rn(p[q], F2, cacc[q]);
  };
  int64_t i = r0 + warp;
  for (; i + kWarps < r1; i += 2 * kWarps) {  // rows i and i + 8
    const float4 da = s_R[i - r0], db = s_R[i + kWarps - r0];
    float2 ta[KP], tb[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float4 xy = s_XY[q][lane], zb = s_ZB[q][lane];
      const float2 cxq = make_float2(xy.x, xy.y), cyq = make_float2(xy.z, xy.w), czq = make_float2(zb.x, zb.y);
      const float2 B = make_float2(zb.z, zb.w);
      float2 xa = __ffma2_rn(make_float2(da.x, da.x), cxq, B);
      float2 xb = __ffma2_rn(make_float2(db.x, db.x), cxq, B);
      xa = __ffma2_rn(make_float2(da.y, da.y), cyq, xa);
      xb = __ffma2_rn(make_float2(db.y, db.y), cyq, xb);
      ta[q] = __ffma2_rn(make_float2(da.z, da.z), czq, xa);
      tb[q] = __ffma2_rn(make_float2(db.z, db.z), czq, xb);
    }
    float ma = tree_max2<KP>(ta), mb = tree_max2<KP>(tb);
    ma = warp_maxf(ma);
    mb = warp_maxf(mb);
    const float msa = (ma == -INFINITY) ? 0.f : ma, msb = (mb == -INFINITY) ? 0.f : mb;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float2 d = __fadd2_rn(ta[q], make_float2(-msa, -msa));
      ta[q] = make_float2(ex2f(d.x), ex2f(d.y));
      const float2 e = __fadd2_rn(tb[q], make_float2(-msb, -msb));
      tb[q] = make_float2(ex2f(e.x), ex2f(e.y));
    }
    finish_row(ma, da.w, ta, i);
    finish_row(mb, db.w, tb, i + kWarps);
  }
  if (i < r1) {  // a last single row
    const float4 da = s_R[i - r0];
    float2 ta[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float4 xy = s_XY[q][lane], zb = s_ZB[q][lane];
      float2 xa = __ffma2_rn(make_float2(da.x, da.x), make_float2(xy.x, xy.y), make_float2(zb.z, zb.w));
      xa = __ffma2_rn(make_float2(da.y, da.y), make_float2(xy.z, xy.w), xa);
      ta[q] = __ffma2_rn(make_float2(da.z, da.z), make_float2(zb.x, zb.y), xa);
    }
    float ma = fmaxf(ta[0].x, ta[0].y);
#pragma unroll
    for (int q = 1; q < KP; ++q) ma = fmaxf(ma, fmaxf(ta[q].x, ta[q].y));
    ma = warp_maxf(ma);
    const float msa = (ma == -INFINITY) ? 0.f : ma;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float2 d = __fadd2_rn(ta[q], make_float2(-msa, -msa));
      ta[q] = make_float2(ex2f(d.x), ex2f(d.y));
    }
    finish_row(ma, da.w, ta, i);
  }
  if (slot > 0) flush(slot);
  float (*cs)[kStrip] = reinterpret_cast<float (*)[kStrip]>(reinterpret_cast<float*>(s_R + a.rows_per_cta));  // the tiles, done
  __shared__ float ss[kWarps];
  __shared__ float mm[kWarps];
  if (lane == 0) {
    ss[warp] = sigma;
    mm[warp] = mmax;
  }
  __syncthreads();
  float sig = ss[0];
  for (int ww = 1; ww < kWarps; ++ww) sig = fmaxf(sig, ss[ww]);
  const float fw = (sigma == -INFINITY) ? 0.f : ex2f(sigma - sig);
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int c = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
    cs[warp][c] = cacc[q].x * fw;
    cs[warp][c + 1] = cacc[q].y * fw;
  }
  __syncthreads();
  float2* colp = reinterpret_cast<float2*>(a.colp);
  for (int c = threadIdx.x; c < kStrip; c += kThreads) {
    float s = 0.f;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) s += cs[ww][c];
    if (j0 + c < n) colp[(j0 + c) * gridDim.y + blockIdx.y] = make_float2(sig == -INFINITY ? 0.f : s, sig == -INFINITY ? 0.f : sig);
  }
  if (threadIdx.x == 0) {
    float m = mm[0];
    for (int ww = 1; ww < kWarps; ++ww) m = fmaxf(m, mm[ww]);
    a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m) * kLn2;
  }
}

// R rows per warp step with the column constants in shared memory
// ($POTGPU_PTS_PAIRS=5: R = 4): R independent max / CREDUX / MUFU chains in
// flight per warp. Same partial formats and epilogue as sweep_pts2s_f32.
template <int R>
__global__ void __launch_bounds__(kThreads, 2) sweep_ptsR_f32(SrcPointsDotF32 src, SweepArgs a) {
  pdl_wait();
  constexpr int KP = kPairs;
  constexpr int kStrip = 64 * KP;
  if (a.gate && *a.gate == 0) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStrip;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  const double w = *a.w;
  extern __shared__ float4 s_R[];  // [rows_per_cta]: (2x', A_i), then the row-sum tiles
  // the lane's column constants: (cx, cy) and (cz, B') per pair, read per warp step
  __shared__ float4 s_XY[KP][32], s_ZB[KP][32];
  for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) {
    double ud = a.u[i];
    if (a.lu) ud = ud + a.lu[i];
    double A = (ud + w) * kLog2e;
    if (a.rowshift) A = A + a.rowshift[i];
    const float4 x2 = src.X2[i];
    s_R[i - r0] = make_float4(x2.x, x2.y, x2.z, float(A));
  }
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    if (warp != 0) break;
    float b[2];
    float4 y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;
      y[h] = make_float4(0, 0, 0, 0);
      if (j < n) {
        vv = a.v[j];
        if (a.lv) vv = vv + a.lv[j];
        vv = vv * kLog2e;
        if (a.colshift) vv = vv + a.colshift[j];
        y[h] = src.Ys[j];
      }
      b[h] = float(vv);
    }
    s_XY[q][lane] = make_float4(y[0].x, y[1].x, y[0].y, y[1].y);
    s_ZB[q][lane] = make_float4(y[0].z, y[1].z, b[0], b[1]);
  }
  __syncthreads();
  float2 cacc[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q) cacc[q] = make_float2(0.f, 0.f);
  float sigma = -INFINITY;
  float mmax = -INFINITY;
  float2* rowp = reinterpret_cast<float2*>(a.rowp);
  float* tile = reinterpret_cast<float*>(s_R + a.rows_per_cta) + warp * (32 * 33);
  float* tslot = tile + lane;
  float my_ms = 0.f;
  int slot = 0;
  int64_t ib = r0 + warp;
  const int64_t ldp = gridDim.x;
  auto flush = [&](int cnt) {
    __syncwarp();
    if (lane < cnt) {
      const float* rowv = tile + lane * 33;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; k += 4) { s0 += rowv[k]; s1 += rowv[k + 1]; s2 += rowv[k + 2]; s3 += rowv[k + 3]; }
      const float2 part = make_float2((s0 + s1) + (s2 + s3), my_ms);
      rowp[(ib + int64_t(kWarps) * lane) * ldp + blockIdx.x] = part;
    }
    __syncwarp();
  };
  // one row's tile slot, column scale update and accumulation
  auto finish_row = [&](float m, float Ai, const float2 (&p)[KP], int64_t i) {
    const float ms = (m == -INFINITY) ? 0.f : m;
    *tslot = tree_sum2<KP>(p);
    tslot += 33;
    if (lane == slot) my_ms = ms;
    if (++slot == 32) {
      flush(32);
      slot = 0;
      tslot = tile + lane;
      ib = i + kWarps;
    }
    const float mA = (m == -INFINITY) ? -INFINITY : m + Ai;
    if (mA > sigma) {
      const float sc = ex2f(sigma - mA);
#pragma unroll
      for (int q = 0; q < KP; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
      sigma = mA;
    }
    mmax = fmaxf(mmax, mA);
    const float f = (mA == -INFINITY) ? 0.f : ex2f(mA - sigma);
    const float2 F2 = make_float2(f, f);
#pragma unroll
    for (int q = 0; q < KP; ++q) cacc[q] = __ffma2_rn(p[q], F2, cacc[q]);
  };
  int64_t i = r0 + warp;
  for (; i + (R - 1) * kWarps < r1; i += R * kWarps) {  // rows i, i + 8, ..., i + 8 (R - 1)
    float4 d[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) d[rr] = s_R[i + rr * kWarps - r0];
    float2 t[R][KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float4 xy = s_XY[q][lane], zb = s_ZB[q][lane];
      const float2 cxq = make_float2(xy.x, xy.y), cyq = make_float2(xy.z, xy.w), czq = make_float2(zb.x, zb.y);
      const float2 B = make_float2(zb.z, zb.w);
#pragma unroll
      for (int rr = 0; rr < R; ++rr) {
        float2 x = __ffma2_rn(make_float2(d[rr].x, d[rr].x), cxq, B);
        x = __ffma2_rn(make_float2(d[rr].y, d[rr].y), cyq, x);
        t[rr][q] = __ffma2_rn(make_float2(d[rr].z, d[rr].z), czq, x);
      }
    }
    float m[R];
#pragma unroll
    for (int rr = 0; rr < R; ++rr) m[rr] = warp_maxf(tree_max2<KP>(t[rr]));
#pragma unroll
    for (int rr = 0; rr < R; ++rr) {
      const float ms = (m[rr] == -INFINITY) ? 0.f : m[rr];
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 e = __fadd2_rn(t[rr][q], make_float2(-ms, -ms));
        t[rr][q] = make_float2(ex2f(e.x), ex2f(e.y));
      }
    }
#pragma unroll
    for (int rr = 0; rr < R; ++rr) finish_row(m[rr], d[rr].w, t[rr], i + rr * kWarps);
  }
  for (; i < r1; i += kWarps) {  // the last rows, one at a time
    const float4 da = s_R[i - r0];
    float2 ta[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float4 xy = s_XY[q][lane], zb = s_ZB[q][lane];
      float2 xa = __ffma2_rn(make_float2(da.x, da.x), make_float2(xy.x, xy.y), make_float2(zb.z, zb.w));
      xa = __ffma2_rn(make_float2(da.y, da.y), make_float2(xy.z, xy.w), xa);
      ta[q] = __ffma2_rn(make_float2(da.z, da.z), make_float2(zb.x, zb.y), xa);
    }
    float ma = warp_maxf(tree_max2<KP>(ta));
    const float msa = (ma == -INFINITY) ? 0.f : ma;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float2 e = __fadd2_rn(ta[q], make_float2(-msa, -msa));
      ta[q] = make_float2(ex2f(e.x), ex2f(e.y));
    }
    finish_row(ma, da.w, ta, i);
  }
  if (slot > 0) flush(slot);
  float (*cs)[kStrip] = reinterpret_cast<float (*)[kStrip]>(reinterpret_cast<float*>(s_R + a.rows_per_cta));  // the tiles, done
  __shared__ float ss[kWarps];
  __shared__ float mm[kWarps];
  if (lane == 0) {
    ss[warp] = sigma;
    mm[warp] = mmax;
  }
  __syncthreads();
  float sig = ss[0];
  for (int ww = 1; ww < kWarps; ++ww) sig = fmaxf(sig, ss[ww]);
  const float fw = (sigma == -INFINITY) ? 0.f : ex2f(sigma - sig);
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    const int c = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
    cs[warp][c] = cacc[q].x * fw;
    cs[warp][c + 1] = cacc[q].y * fw;
  }
  __syncthreads();
  float2* colp = reinterpret_cast<float2*>(a.colp);
  for (int c = threadIdx.x; c < kStrip; c += kThreads) {
    float s = 0.f;
#pragma unroll
    for (int ww = 0; ww < kWarps; ++ww) s += cs[ww][c];
    if (j0 + c < n) colp[(j0 + c) * gridDim.y + blockIdx.y] = make_float2(sig == -INFINITY ? 0.f : s, sig == -INFINITY ? 0.f : sig);
  }
  if (threadIdx.x == 0) {
    float m = mm[0];
    for (int ww = 1; ww < kWarps; ++ww) m = fmaxf(m, mm[ww]);
    a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m) * kLn2;
  }
}


// One-sided points sweep of z_check' (ASPOT) when its Greenkhorn block is u
// or v and z_best = z_hat: one side of B(z_check') is an O(n) rescale of
// z_hat's sums (k_gk_update writes it to krow / kcol), the other needs one
// pass, and the row shifts need no max: u enters the fp64 row offset A_i,
// not t, so for block u each row segment's max is exactly the one z_hat's
// sweep (or z_grave's, when z_hat differs only in w) left in rowp; for block
// v it is that max plus at most the strip's largest change of B'_j (exact up
// to the strip's spread of changes; a wider spread takes the exact warp max).
// The known side is written into the partials in the reduce kernels' format
// (one nonzero partial per index: S 2^(M + offset) = the known sum), so the
// evaluation is the same kernel. block (device): 0 = u (columns swept),
// 1 = v (rows swept).
//
// K1'' (reference: the z_bar of the next iteration,
// solvers.hpp:336, evaluated at :337). The next iteration's
//   z_bar' = (1 - theta') z_check' + theta' z_best = z_best + (1 - theta') D
// differs from z_best, like z_check' = z_best + D, only in the Greenkhorn
// block, so B(z_bar') is the same row (block u) or column (block v)
// rescaling of the entries this pass already exponentiates. With rowp2 set,
// the pass also forms z_bar''s unknown side from those entries (block u: a
// second column accumulator with row factors 2^(m_i + A''_i); block v: a
// second row sum with column weights 2^(d_j - dmax), d_j = B''_j - B'_j) and
// writes z_bar''s partials (known side encoded from kbar_row / kbar_col) to
// rowp2 / colp2 / maxp2, so the next iteration's z_bar needs no sweep. The
// block-v max exponent of z_bar' is an upper bound; a bound near the
// overflow threshold, a spread of d_j wider than kOneSidedSpread or a
// non-finite d_j raise *bad and the next iteration sweeps z_bar as before.
struct OneSidedArgs {
  const double* krow;  // B' 1 (block u)
  const double* kcol;  // B'^T 1 (block v)
  const double* vsrc;  // v of the source point (block v)
  const int* block;
  // K1'' (null rowp2: off)
  const double* u2; const double* v2; const double* w2;  // z_bar'
  const double* kbar_row;  // B(z_bar') 1 (block u)
  const double* kbar_col;  // B(z_bar')^T 1 (block v)
  double* rowp2; double* colp2; double* maxp2;
  int* bad;
};
constexpr float kOneSidedSpread = 40.f;
__host__ __device__ constexpr size_t sweep_pts1_smem(int rows_per_cta) {
  // + source segment maxima, + z_bar''s row offsets
  return sweep_pts_smem(rows_per_cta) + 2 * size_t((rows_per_cta + 3) & ~3) * sizeof(float);
}
__device__ __forceinline__ float2 encode_sum(double R, double off) {  // (S, M): S 2^(M + off) = R
  if (!(R > 0.0)) return make_float2(0.f, 0.f);
  const double M = floor(log2(R) - off);
  return make_float2(float(R * exp2(-(M + off))), float(M));
}

// TWO: rows i and i + 8 per warp step, as sweep_pts2_f32 (both rows' dot
// products share each column operand, two independent MUFU bursts in flight).
template <int TWO>
__global__ void __launch_bounds__(kThreads, 2) sweep_pts1_f32(SrcPointsDotF32 src, SweepArgs a, OneSidedArgs o) {
  pdl_wait();
  constexpr int KP = kPairs;
  constexpr int kStrip = 64 * KP;
  if (a.gate && *a.gate == 0) return;
  const int mode = *o.block;
  const bool fuse = o.rowp2 != nullptr;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kStrip;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  const double w = *a.w;
  const double w2 = fuse ? *o.w2 : 0.0;
  const int64_t ldp = gridDim.x;
  extern __shared__ float4 s_R[];  // rows (2x', A_i), the row-sum tiles, [rows] source segment maxima, [rows] A''_i
  float* s_tiles = reinterpret_cast<float*>(s_R + a.rows_per_cta);
  float* s_M = s_tiles + kWarps * 32 * 33;
  float* s_A2 = s_M + ((a.rows_per_cta + 3) & ~3);
  // column constants B'_j of the strip, two column pairs per 16-byte word (one LDS.128 per two pairs)
  __shared__ float4 s_B4[KP / 2][32];
  auto Bof = [&](int q, int l) -> float2 {
    const float4 v = s_B4[q >> 1][l];
    return (q & 1) ? make_float2(v.z, v.w) : make_float2(v.x, v.y);
  };
  __shared__ float s_dv[5][kWarps];
  float2* rowp = reinterpret_cast<float2*>(a.rowp);
  float2* colp = reinterpret_cast<float2*>(a.colp);
  float2* rowp2 = reinterpret_cast<float2*>(o.rowp2);
  float2* colp2 = reinterpret_cast<float2*>(o.colp2);
  // rows in batches of 4 per thread: all of a batch's loads (the source's partial is a scattered
  // 8-byte read per row) are issued before its stores, which the compiler could not hoist them over
  float rbnd = -INFINITY;  // max over this thread's rows of (source segment max + row offset): bounds the exponents
  for (int64_t ib0 = r0 + threadIdx.x; ib0 < r1; ib0 += 4 * kThreads) {
    double uu[4], rs[4], u2[4];
    float4 x2[4];
    float2 pp[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = ib0 + int64_t(k) * kThreads;
      if (i < r1) {
        uu[k] = a.u[i];
        rs[k] = a.rowshift ? a.rowshift[i] : 0.0;
        x2[k] = src.X2[i];
        pp[k] = rowp[i * ldp + blockIdx.x];  // read before this thread overwrites it
        u2[k] = fuse ? o.u2[i] : 0.0;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = ib0 + int64_t(k) * kThreads;
      if (i < r1) {
        double A = (uu[k] + w) * kLog2e;
        if (a.rowshift) A = A + rs[k];
        s_R[i - r0] = make_float4(x2[k].x, x2[k].y, x2[k].z, float(A));
        const float smk = pp[k].x != 0.f ? pp[k].y : -INFINITY;
        s_M[i - r0] = smk;
        rbnd = fmaxf(rbnd, smk + float(A));
        if (mode == 0) rowp[i * ldp + blockIdx.x] = blockIdx.x == 0 ? encode_sum(o.krow[i], A) : make_float2(0.f, 0.f);
        if (fuse) {
          double A2 = (u2[k] + w2) * kLog2e;
          if (a.rowshift) A2 = A2 + rs[k];
          s_A2[i - r0] = float(A2);
          rbnd = fmaxf(rbnd, smk + float(A2));
          if (mode == 0) rowp2[i * ldp + blockIdx.x] = blockIdx.x == 0 ? encode_sum(o.kbar_row[i], A2) : make_float2(0.f, 0.f);
        }
      }
    }
  }
  float2 cx[KP], cy[KP], cz[KP];
  float2 dd[KP];  // block v, K1'': d_j = B''_j - B'_j of the lane's columns
  float dmax = -INFINITY, dmin = INFINITY, emax = -INFINITY, emin = INFINITY;
  int ebad = 0;
#pragma unroll
  for (int q = 0; q < KP; ++q) {
    float b[2], e[2] = {0.f, 0.f};
    float4 y[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;
      y[h] = make_float4(0, 0, 0, 0);
      if (j < n) {
        vv = a.v[j] * kLog2e;
        if (a.colshift) vv = vv + a.colshift[j];
        y[h] = src.Ys[j];
        if (mode == 1) {
          double vs = o.vsrc[j] * kLog2e;
          if (a.colshift) vs = vs + a.colshift[j];
          const float d = float(vv) - float(vs);
          dmax = fmaxf(dmax, d);
          dmin = fminf(dmin, d);
          if (fuse) {
            double v2 = o.v2[j] * kLog2e;
            if (a.colshift) v2 = v2 + a.colshift[j];
            e[h] = float(v2) - float(vv);
            ebad |= !(fabsf(e[h]) < 1e30f);
            emax = fmaxf(emax, e[h]);
            emin = fminf(emin, e[h]);
          }
        }
      }
      b[h] = float(vv);
    }
    if (warp == 0) reinterpret_cast<float2*>(&s_B4[q >> 1][lane])[q & 1] = make_float2(b[0], b[1]);
    cx[q] = make_float2(y[0].x, y[1].x);
    cy[q] = make_float2(y[0].y, y[1].y);
    cz[q] = make_float2(y[0].z, y[1].z);
    dd[q] = make_float2(e[0], e[1]);
  }
  if (mode == 1) {
    dmax = warp_maxf(dmax);
    dmin = -warp_maxf(-dmin);
    if (fuse) {
      emax = warp_maxf(emax);
      emin = -warp_maxf(-emin);
      ebad = __any_sync(0xffffffffu, ebad);
    }
    rbnd = warp_maxf(rbnd);
    if (lane == 0) {
      s_dv[0][warp] = dmax; s_dv[1][warp] = dmin;
      s_dv[2][warp] = ebad ? NAN : emax; s_dv[3][warp] = emin;
      s_dv[4][warp] = rbnd;
    }
    for (int c = threadIdx.x; c < kStrip; c += kThreads)  // the known column sums
      if (j0 + c < n) {
        colp[(j0 + c) * gridDim.y + blockIdx.y] = blockIdx.y == 0 ? encode_sum(o.kcol[j0 + c], 0.0) : make_float2(0.f, 0.f);
        if (fuse)
          colp2[(j0 + c) * gridDim.y + blockIdx.y] =
              blockIdx.y == 0 ? encode_sum(o.kbar_col[j0 + c], 0.0) : make_float2(0.f, 0.f);
      }
  }
  __syncthreads();
  float dvmax = -INFINITY, dvmin = INFINITY, evmax = -INFINITY, evmin = INFINITY;
  bool fuse_bad = false;
  if (mode == 1) {
    for (int ww = 0; ww < kWarps; ++ww) {
      dvmax = fmaxf(dvmax, s_dv[0][ww]);
      dvmin = fminf(dvmin, s_dv[1][ww]);
      if (fuse) {
        fuse_bad = fuse_bad || s_dv[2][ww] != s_dv[2][ww];
        evmax = fmaxf(evmax, s_dv[2][ww]);
        evmin = fminf(evmin, s_dv[3][ww]);
      }
    }
    // an all-masked strip (evmax = -inf) has no entries: weights are unused
    if (fuse && evmax > -INFINITY && !(evmax - evmin <= kOneSidedSpread)) fuse_bad = true;
    if (!(evmax > -INFINITY)) evmax = 0.f;
  }
  const bool exact = mode == 1 && !(dvmax - dvmin <= kOneSidedSpread);  // CTA-uniform
  // Block v: the max exponent of a row segment (the reference's overflow test, dual.hpp:85-90) is
  // bounded by its shift m_i = (source segment max) + dvmax. Far below the threshold the bound
  // decides the test like the exact value, and the per-row max tree is skipped; a CTA whose bound
  // comes within a few units of it (or takes the exact shifts anyway) computes the exact maxima.
  bool need_lm = exact;
  if (mode == 1) {
    float bcta = -INFINITY;
    for (int ww = 0; ww < kWarps; ++ww) bcta = fmaxf(bcta, s_dv[4][ww]);
    const float ub = bcta + dvmax + (fuse ? fmaxf(evmax, 0.f) : 0.f);
    if (!(double(ub) * kLn2 <= kMaxExponent - 20.0)) need_lm = true;  // also NaN
  }
  float mmax = -INFINITY, mmax2 = -INFINITY;
  auto dots = [&](const float4& d, float2 (&t)[KP]) {
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float2 B = Bof(q, lane);
      float2 x = __ffma2_rn(make_float2(d.x, d.x), cx[q], B);
      x = __ffma2_rn(make_float2(d.y, d.y), cy[q], x);
      t[q] = __ffma2_rn(make_float2(d.z, d.z), cz[q], x);
    }
  };
  if (mode == 0) {  // block u: column sums of B' (and of B(z_bar')) at the source's row-segment maxima
    float2 cacc[KP], cacc2[KP];
#pragma unroll
    for (int q = 0; q < KP; ++q) cacc[q] = cacc2[q] = make_float2(0.f, 0.f);
    float sigma = -INFINITY, sigma2 = -INFINITY;
    int64_t i = r0 + warp;
    if constexpr ((TWO & 1) != 0) {
      for (; i + kWarps < r1; i += 2 * kWarps) {  // rows i and i + 8
        const float4 da = s_R[i - r0], db = s_R[i + kWarps - r0];
        const float ma = s_M[i - r0], mb = s_M[i + kWarps - r0];
        const bool la = ma != -INFINITY, lb = mb != -INFINITY;  // an empty segment has t = -inf throughout: exact zeros
        if (!la && !lb) continue;
        float2 ta[KP], tb[KP];
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 B = Bof(q, lane);
          float2 xa = __ffma2_rn(make_float2(da.x, da.x), cx[q], B);
          float2 xb = __ffma2_rn(make_float2(db.x, db.x), cx[q], B);
          xa = __ffma2_rn(make_float2(da.y, da.y), cy[q], xa);
          xb = __ffma2_rn(make_float2(db.y, db.y), cy[q], xb);
          ta[q] = __ffma2_rn(make_float2(da.z, da.z), cz[q], xa);
          tb[q] = __ffma2_rn(make_float2(db.z, db.z), cz[q], xb);
        }
        const float msa = la ? ma : 0.f, msb = lb ? mb : 0.f;
        const float mAa = ma + da.w, mAb = mb + db.w;
        const float mAx = fmaxf(mAa, mAb);
        mmax = fmaxf(mmax, mAx);
        if (mAx > sigma) {
          const float sc = ex2f(sigma - mAx);
#pragma unroll
          for (int q = 0; q < KP; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
          sigma = mAx;
        }
        const float fa = la ? ex2f(mAa - sigma) : 0.f, fb = lb ? ex2f(mAb - sigma) : 0.f;
        const float2 Fa = make_float2(fa, fa), Fb = make_float2(fb, fb);
        float2 Ga = make_float2(0.f, 0.f), Gb = Ga;
        if (fuse) {
          const float mA2a = ma + s_A2[i - r0], mA2b = mb + s_A2[i + kWarps - r0];
          const float mA2x = fmaxf(mA2a, mA2b);
          mmax2 = fmaxf(mmax2, mA2x);
          if (mA2x > sigma2) {
            const float sc = ex2f(sigma2 - mA2x);
#pragma unroll
            for (int q = 0; q < KP; ++q) cacc2[q] = __fmul2_rn(cacc2[q], make_float2(sc, sc));
            sigma2 = mA2x;
          }
          const float ga = la ? ex2f(mA2a - sigma2) : 0.f, gb = lb ? ex2f(mA2b - sigma2) : 0.f;
          Ga = make_float2(ga, ga);
          Gb = make_float2(gb, gb);
        }
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 e = __fadd2_rn(ta[q], make_float2(-msa, -msa));
          const float2 x = make_float2(ex2f(e.x), ex2f(e.y));
          cacc[q] = __ffma2_rn(x, Fa, cacc[q]);
          if (fuse) cacc2[q] = __ffma2_rn(x, Ga, cacc2[q]);
        }
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 e = __fadd2_rn(tb[q], make_float2(-msb, -msb));
          const float2 x = make_float2(ex2f(e.x), ex2f(e.y));
          cacc[q] = __ffma2_rn(x, Fb, cacc[q]);
          if (fuse) cacc2[q] = __ffma2_rn(x, Gb, cacc2[q]);
        }
      }
    }
    for (; i < r1; i += kWarps) {
      const float4 d = s_R[i - r0];
      const float m = s_M[i - r0];
      if (m == -INFINITY) continue;  // empty segment (warp-uniform)
      float2 t[KP];
      dots(d, t);
      const float mA = m + d.w;
      mmax = fmaxf(mmax, mA);
      if (mA > sigma) {
        const float sc = ex2f(sigma - mA);
#pragma unroll
        for (int q = 0; q < KP; ++q) cacc[q] = __fmul2_rn(cacc[q], make_float2(sc, sc));
        sigma = mA;
      }
      const float f = ex2f(mA - sigma);
      const float2 F2 = make_float2(f, f);
      if (fuse) {
        const float mA2 = m + s_A2[i - r0];
        mmax2 = fmaxf(mmax2, mA2);
        if (mA2 > sigma2) {
          const float sc = ex2f(sigma2 - mA2);
#pragma unroll
          for (int q = 0; q < KP; ++q) cacc2[q] = __fmul2_rn(cacc2[q], make_float2(sc, sc));
          sigma2 = mA2;
        }
        const float f2 = ex2f(mA2 - sigma2);
        const float2 G2 = make_float2(f2, f2);
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 e = __fadd2_rn(t[q], make_float2(-m, -m));
          const float2 x = make_float2(ex2f(e.x), ex2f(e.y));
          cacc[q] = __ffma2_rn(x, F2, cacc[q]);
          cacc2[q] = __ffma2_rn(x, G2, cacc2[q]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < KP; ++q) {
          const float2 e = __fadd2_rn(t[q], make_float2(-m, -m));
          cacc[q] = __ffma2_rn(make_float2(ex2f(e.x), ex2f(e.y)), F2, cacc[q]);
        }
      }
    }
    // per-warp column sums: [2][kWarps][kStrip] floats in the (unused) row-sum tile area
    float* cs = s_tiles;
    float* cs2 = s_tiles + kWarps * kStrip;
    __shared__ float ss[2][kWarps], mm[2][kWarps];
    if (lane == 0) { ss[0][warp] = sigma; mm[0][warp] = mmax; ss[1][warp] = sigma2; mm[1][warp] = mmax2; }
    __syncthreads();
    float sig = ss[0][0], sig2 = ss[1][0];
    for (int ww = 1; ww < kWarps; ++ww) { sig = fmaxf(sig, ss[0][ww]); sig2 = fmaxf(sig2, ss[1][ww]); }
    const float fw = (sigma == -INFINITY) ? 0.f : ex2f(sigma - sig);
    const float fw2 = (sigma2 == -INFINITY) ? 0.f : ex2f(sigma2 - sig2);
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const int c = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
      cs[warp * kStrip + c] = cacc[q].x * fw;
      cs[warp * kStrip + c + 1] = cacc[q].y * fw;
      if (fuse) {
        cs2[warp * kStrip + c] = cacc2[q].x * fw2;
        cs2[warp * kStrip + c + 1] = cacc2[q].y * fw2;
      }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < kStrip; c += kThreads) {
      float sc = 0.f, sc2 = 0.f;
#pragma unroll
      for (int ww = 0; ww < kWarps; ++ww) { sc += cs[ww * kStrip + c]; sc2 += cs2[ww * kStrip + c]; }
      if (j0 + c < n) {
        colp[(j0 + c) * gridDim.y + blockIdx.y] = make_float2(sig == -INFINITY ? 0.f : sc, sig == -INFINITY ? 0.f : sig);
        if (fuse)
          colp2[(j0 + c) * gridDim.y + blockIdx.y] =
              make_float2(sig2 == -INFINITY ? 0.f : sc2, sig2 == -INFINITY ? 0.f : sig2);
      }
    }
    if (threadIdx.x == 0) {
      float m = mm[0][0], m2 = mm[1][0];
      for (int ww = 1; ww < kWarps; ++ww) { m = fmaxf(m, mm[0][ww]); m2 = fmaxf(m2, mm[1][ww]); }
      a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m) * kLn2;
      if (fuse) o.maxp2[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m2) * kLn2;  // exact
    }
    return;
  }
  // block v: row sums of B' at the source's segment maxima + the strip's largest change;
  // K1'': row sums of B(z_bar') = sum_j B'_ij 2^(d_j), weights 2^(d_j - dmax) <= 1.
  // Rows are flushed every 16: the tile holds [sum][16 rows][33] per warp, lane l < 16
  // reduces row l of B', lane 16 + l row l of B(z_bar').
  float2 gw[KP];
#pragma unroll
  for (int q = 0; q < KP; ++q)
    gw[q] = fuse ? make_float2(ex2f(dd[q].x - evmax), ex2f(dd[q].y - evmax)) : make_float2(0.f, 0.f);
  float* tile = s_tiles + warp * (32 * 33);
  constexpr int kSlotRows = 16;
  int slot = 0;
  float my_ms = 0.f;
  int64_t ib = r0 + warp;
  auto flush = [&](int cnt) {
    __syncwarp();
    const int h = lane >> 4, r = lane & 15;
    if (r < cnt && (h == 0 || fuse)) {
      const float* rowv = tile + (h * kSlotRows + r) * 33;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int k = 0; k < 32; k += 4) { s0 += rowv[k]; s1 += rowv[k + 1]; s2 += rowv[k + 2]; s3 += rowv[k + 3]; }
      const int64_t row = ib + int64_t(kWarps) * r;
      const float S = (s0 + s1) + (s2 + s3);
      if (h == 0) rowp[row * ldp + blockIdx.x] = make_float2(S, my_ms);
      else rowp2[row * ldp + blockIdx.x] = make_float2(S, my_ms + evmax);
    }
    __syncwarp();
  };
  int64_t i = r0 + warp;
  if constexpr ((TWO & 2) != 0) {
    for (; i + kWarps < r1; i += 2 * kWarps) {  // rows i and i + 8 (slots slot and slot + 1)
      const float4 da = s_R[i - r0], db = s_R[i + kWarps - r0];
      float2 ta[KP], tb[KP];
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 B = Bof(q, lane);
        float2 xa = __ffma2_rn(make_float2(da.x, da.x), cx[q], B);
        float2 xb = __ffma2_rn(make_float2(db.x, db.x), cx[q], B);
        xa = __ffma2_rn(make_float2(da.y, da.y), cy[q], xa);
        xb = __ffma2_rn(make_float2(db.y, db.y), cy[q], xb);
        ta[q] = __ffma2_rn(make_float2(da.z, da.z), cz[q], xa);
        tb[q] = __ffma2_rn(make_float2(db.z, db.z), cz[q], xb);
      }
      float lma = -INFINITY, lmb = -INFINITY;
      if (need_lm) { lma = tree_max2<KP>(ta); lmb = tree_max2<KP>(tb); }
      const float sma = s_M[i - r0], smb = s_M[i + kWarps - r0];
      const float ma = exact ? warp_maxf(lma) : (sma == -INFINITY ? -INFINITY : sma + dvmax);
      const float mb = exact ? warp_maxf(lmb) : (smb == -INFINITY ? -INFINITY : smb + dvmax);
      if (!need_lm) { lma = ma; lmb = mb; }  // the shifts bound the segment maxima
      mmax = fmaxf(mmax, fmaxf(lma + da.w, lmb + db.w));
      const float msa = (ma == -INFINITY) ? 0.f : ma, msb = (mb == -INFINITY) ? 0.f : mb;
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 e = __fadd2_rn(ta[q], make_float2(-msa, -msa));
        ta[q] = make_float2(ex2f(e.x), ex2f(e.y));
      }
#pragma unroll
      for (int q = 0; q < KP; ++q) {
        const float2 e = __fadd2_rn(tb[q], make_float2(-msb, -msb));
        tb[q] = make_float2(ex2f(e.x), ex2f(e.y));
      }
      tile[slot * 33 + lane] = tree_sum2<KP>(ta);
      tile[(slot + 1) * 33 + lane] = tree_sum2<KP>(tb);
      if (fuse) {
        mmax2 = fmaxf(mmax2, fmaxf(lma + s_A2[i - r0], lmb + s_A2[i + kWarps - r0]));
        tile[(kSlotRows + slot) * 33 + lane] = wsum2<KP>(ta, gw);
        tile[(kSlotRows + slot + 1) * 33 + lane] = wsum2<KP>(tb, gw);
      }
      if ((lane & 15) == slot) my_ms = msa;
      if ((lane & 15) == slot + 1) my_ms = msb;
      slot += 2;
      if (slot == kSlotRows) {
        flush(kSlotRows);
        slot = 0;
        ib = i + 2 * kWarps;
      }
    }
    // an odd slot count before the single-row tail: the tail keeps filling the same batch
  }
  for (; i < r1; i += kWarps) {
    const float4 d = s_R[i - r0];
    float2 t[KP];
    dots(d, t);
    float lm = need_lm ? tree_max2<KP>(t) : -INFINITY;
    const float sm = s_M[i - r0];
    const float m = exact ? warp_maxf(lm) : (sm == -INFINITY ? -INFINITY : sm + dvmax);
    if (!need_lm) lm = m;  // the shift bounds the segment maximum
    mmax = fmaxf(mmax, lm + d.w);
    const float ms = (m == -INFINITY) ? 0.f : m;
#pragma unroll
    for (int q = 0; q < KP; ++q) {
      const float2 e = __fadd2_rn(t[q], make_float2(-ms, -ms));
      t[q] = make_float2(ex2f(e.x), ex2f(e.y));
    }
    tile[slot * 33 + lane] = tree_sum2<KP>(t);
    if (fuse) {
      mmax2 = fmaxf(mmax2, lm + s_A2[i - r0]);
      float2 p[KP];
#pragma unroll
      for (int q = 0; q < KP; ++q) p[q] = __fmul2_rn(t[q], gw[q]);
      tile[(kSlotRows + slot) * 33 + lane] = tree_sum2<KP>(p);
    }
    if ((lane & 15) == slot) my_ms = ms;
    if (++slot == kSlotRows) {
      flush(kSlotRows);
      slot = 0;
      ib = i + kWarps;
    }
  }
  if (slot > 0) flush(slot);
  mmax = warp_maxf(mmax);
  if (fuse) mmax2 = warp_maxf(mmax2);
  __shared__ float mm1[2][kWarps];
  if (lane == 0) { mm1[0][warp] = mmax; mm1[1][warp] = mmax2; }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = mm1[0][0], m2 = mm1[1][0];
    for (int ww = 1; ww < kWarps; ++ww) { m = fmaxf(m, mm1[0][ww]); m2 = fmaxf(m2, mm1[1][ww]); }
    a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(m) * kLn2;
    if (fuse) {
      // upper bound of z_bar''s max exponent (natural units); the exact one
      // only matters at the overflow threshold: near it, z_bar is re-swept
      const double ub = (double(m2) + double(evmax)) * kLn2;
      if (fuse_bad || ub != ub || ub > kMaxExponent - 16.0) *o.bad = 1;
      o.maxp2[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = ub;
    }
  } else if (fuse_bad && threadIdx.x == 32) {
    *o.bad = 1;
  }
}

// ------------------------------------------------------------------------
// Grid shape: strips x row blocks, the row-block count chosen so the CTA
// count fills the resident capacity (SMs x occupancy) as evenly as possible.
struct SweepGrid {
  dim3 grid;
  int rows_per_cta;
};

// Target waves of resident CTAs per sweep ($POTGPU_SWEEP_WAVES, default 1:
// measured on B200 at n = 16384, one wave of long-lived CTAs beats 8 waves
// by 17% (per-CTA prologue/epilogue and fewer column partials); see
// profiles/waves.sh).
inline int sweep_waves() {
  static const int w = [] {
    const char* e = std::getenv("POTGPU_SWEEP_WAVES");
    const int v = e ? std::atoi(e) : 0;
    return v > 0 ? v : 1;
  }();
  return w;
}

// Points-sweep kernel ($POTGPU_PTS_PAIRS): 2 = sweep_pts2_f32 (8 pairs per
// lane, two rows per iteration; default, fastest measured), 4 / 6 / 8 =
// sweep_pts_f32<KP> (profiles/pts_variants.sh).
inline int pts_pairs() {
  static const int v = [] {
    const char* e = std::getenv("POTGPU_PTS_PAIRS");
    const int k = e ? std::atoi(e) : 0;
    return (k == 2 || k == 3 || k == 4 || k == 5 || k == 6 || k == 8) ? k : 2;  // 2: the two-row 8-pair variant (default); 3: its smem-column form
  }();
  return v;
}

// $POTGPU_PTS1_TWO: two rows per warp step in the one-sided pass
// (sweep_pts1_f32<TWO>): bit 0 = its block-u loop, bit 1 = its block-v loop.
// Default 3. Measured on B200 (tools/one_sided_times.py,
// profiles/r02/pts1_two_rows_ab.jsonl): C3 block u 0.1302 -> 0.1204 ms, block v
// 0.1331 -> 0.1257 ms, 3417 -> 3509 it/s; C4 1.60 -> 1.44 / 1.83 -> 1.68 ms,
// 283.4 -> 296.5 it/s.
inline int pts1_two() {
  static const int v = [] {
    const char* e = std::getenv("POTGPU_PTS1_TWO");
    const int k = e ? std::atoi(e) : 3;
    return (k >= 0 && k <= 3) ? k : 3;
  }();
  return v;
}

// Cluster size of the points sweep's row-partial merge ($POTGPU_PTS_CLUSTER:
// 1, 2, 4, 8): the largest allowed power of two dividing the strips.
// Default 1 (off): measured on B200 (profiles/cluster_sizes.sh), clusters of
// 8 / 4 / 2 slow the C3 sweep from 0.106 to 0.168 / 0.161 / 0.110 ms — the
// one-wave grid no longer fits the GPCs in one wave of co-scheduled clusters
// — more than the smaller evaluation saves.
inline int pts_cluster(int64_t strips) {
  static const int cap = [] {
    const char* e = std::getenv("POTGPU_PTS_CLUSTER");
    const int k = e ? std::atoi(e) : 0;
    return (k == 1 || k == 2 || k == 4 || k == 8) ? k : 1;
  }();
  int c = cap;
  while (c > 1 && strips % c != 0) c >>= 1;
  return c;
}

constexpr int64_t kMaxRowsPerCta = 2048;

// Grid of the tensor-core points sweep (sweep_tc.cuh): strips of 512
// columns, row blocks of 128 x tiles rows; tiles (1..4) chosen for the
// fullest last wave of `cap` resident CTAs, preferring more rows per CTA
// (the column sums' cross-lane combine is paid once per tile group).
inline SweepGrid choose_grid_tc(int64_t ncols, int64_t nrows, int64_t cap, int max_tiles = 4) {
  const int64_t strips = ceil_div(ncols, 512);
  int best_t = max_tiles;
  double best = -1.0;
  for (int t = max_tiles; t >= 2; --t) {
    const int64_t ctas = strips * ceil_div(std::max<int64_t>(nrows, 1), 128 * t);
    const double eff = double(ctas) / double(ceil_div(ctas, cap) * cap);
    if (eff > best + 0.02) { best = eff; best_t = t; }
  }
  SweepGrid g;
  g.rows_per_cta = 128 * best_t;
  g.grid = dim3(unsigned(strips), unsigned(ceil_div(std::max<int64_t>(nrows, 1), g.rows_per_cta)), 1);
  return g;
}

inline SweepGrid choose_grid(int64_t ncols, int64_t nrows, int num_sms, int occupancy, int strip_cols,
                             int64_t max_rows = kMaxRowsPerCta) {
  const int64_t strips = ceil_div(ncols, strip_cols);
  const int64_t cap = int64_t(num_sms) * occupancy;  // resident CTAs
  const int64_t max_rb = std::max<int64_t>(1, nrows / 8);
  // row blocks: about sweep_waves() waves of resident CTAs, the count whose
  // last wave is fullest (exact multiples of the capacity when possible)
  // at most kMaxRowsPerCta rows per CTA: the fp32 sweep keeps the CTA's row
  // potentials in shared memory (8 KB), which must not cost occupancy
  const int64_t min_rb = std::min<int64_t>(max_rb, ceil_div(nrows, max_rows));
  const int64_t target =
      std::max<int64_t>(min_rb, std::max<int64_t>(1, std::min<int64_t>(max_rb, (sweep_waves() * cap) / strips)));
  int64_t rb = target;
  double best = -1.0;
  for (int64_t k = std::max<int64_t>(min_rb, target / 2); k <= std::min<int64_t>(max_rb, target + target / 2 + 1); ++k) {
    const int64_t ctas = strips * k;
    const double eff = double(ctas) / double(ceil_div(ctas, cap) * cap);
    const double score = eff - 0.01 * double(std::llabs(k - target)) / double(target);
    if (score > best) { best = score; rb = k; }
  }
  SweepGrid g;
  g.rows_per_cta = int(ceil_div(std::max<int64_t>(nrows, 1), rb));
  rb = ceil_div(std::max<int64_t>(nrows, 1), g.rows_per_cta);
  g.grid = dim3(unsigned(strips), unsigned(rb), 1);
  return g;
}

}  // namespace potgpu
