// batch_cluster.cuh — BASELINE configs[4]: many independent small fp32
// stored-cost ASPOT problems, ONE PROBLEM PER THREAD-BLOCK CLUSTER.
//
// The per-problem path (AspotSession) runs an attempt as 12 kernels; for a
// 2048-point problem each of them is a few microseconds, so a batch of
// problems is bound by the rate at which the GPU starts kernels (DESIGN.md
// §9). Here ONE persistent launch solves the whole batch: each cluster of
// kBcCta CTAs (one per SM) takes problems from a queue and runs aspot_solve
// (solvers.hpp:265-385) to its stop and round_pot (rounding.hpp:46-77) of
// the stopping iterate inside the launch, with cluster barriers where the
// kernel sequence had launch boundaries.
//
// Work split inside a cluster: CTA k owns the index slice [lo_k, hi_k) —
// rows lo_k..hi_k of every sweep (whole rows: row sums are CTA-local) and
// the same columns for every O(n) step (column sums, the functionals'
// per-index terms, the dual-point updates). A sweep leaves each CTA's column
// partials of all n columns in global memory (L2); after a cluster barrier
// CTA k combines its slice's columns over the cluster. Scalars (the 14
// functional accumulators + a non-finite flag) are exchanged the same way
// and every CTA reduces them in the same fixed order, so every CTA's copy
// of the control block (AspotCtl in shared memory) takes the same
// decisions with the same device code as the per-problem path (apply_role,
// commit_state, loop_head: aspot_kernels.cuh) — no broadcast needed.
//
// Sweep numerics = sweep_f32<SrcDenseF32> (sweep.cuh): t' = v_j log2 e -
// g2 C_ij in fp32, exponentiated relative to each 512-column row segment's
// exact max, row partials (sum, max) combined in fp64 with the fp64 row
// offset, column accumulators with a per-warp running scale.
#pragma once

#include <cooperative_groups.h>

#include "aspot_kernels.cuh"

namespace potgpu {

namespace cgx = cooperative_groups;

constexpr int kBcThreads = 512;  // 16 warps per CTA, one CTA per SM
constexpr int kBcWarps = kBcThreads / 32;
constexpr int kBcStrip = 512;     // columns per warp segment (16 per lane)
constexpr int kBcMaxStrips = 8;   // n <= 4096
constexpr int kBcMaxN = kBcStrip * kBcMaxStrips;
constexpr int kBcX = kNumAcc + 2; // exchanged scalars per CTA: accumulators, flag, spare

// One problem of the batch (host-filled, device array).
struct BcProblem {
  const float* C;      // n x ld row-major fp32 cost (padding columns 0)
  int64_t ld;
  const double* rt;    // mixed marginals (the dual targets, aspot_setup)
  const double* ct;
  const double* r;     // original marginals (rounding)
  const double* c;
  float g2;            // log2 e / gamma
  AspotCtl ctl0;       // initial control block (as AspotSession::begin)
  TraceDev* trace;     // [ctl0.trace_cap]
  IterLogDev* iterlog; // [ctl0.log_cap]
  double* zc_out;      // [2n + 1]: the stopping iterate z_check (u | v | w)
  double* row_slack;   // [n]
  double* col_slack;   // [n]
};

// Per-problem result written by the cluster's rank-0 CTA.
struct BcResult {
  AspotCtl ctl;   // final control block (status, t, error, phi, sweeps, ...)
  double cost, mass, gap;
  int infeasible;
  int done;
  uint64_t sweep_ns, total_ns;  // rank 0's device time inside the solve's sweeps / the whole problem
};

// Global workspace of one cluster (reused by every problem it takes).
struct BcWs {
  double* slots;     // kBcSlots x stride
  double* sums;      // kRoles x 2 x n (rows | cols per role)
  double* vec;       // 8 x n scratch (rounding)
  float2* colpart;   // [cluster rank][n]
  float2* colpart2;  // [cluster rank][n]: the fused sweep's second point
  double* xch;       // [2][cluster rank][kBcX]
  int64_t stride;    // slot stride
  int cur;           // problem being solved (set by rank 0)
  int skip;          // that problem failed its upload / never arrived (set by rank 0)
};

// Fixed part of the CTA's shared memory; the row-sized arrays follow it
// (bc_smem_layout): A[rows] (fp32 row offsets), rowpart[rows][S] (segment
// (sum, max) per row and strip), then a region used either as the per-warp
// column accumulators [16][512] or, in the cost pass, as wk[rows][S]
// (segment sums of C p and C fb). rows = ceil(n_max / cluster size).
struct BcShared {
  uint32_t ctl[kCtlWords];
  float colsig[kBcWarps];
  float wmax[kBcWarps];
  double red[kBcX][kBcWarps];
  double tot[kBcX];
  double stash[kNumAcc];  // z_bar's functional totals from the fused sweep (K1'')
  int stash_valid;
  int flag;
};

// The fused two-point sweep (K1'') also uses A2[rows] (the second point's
// row offsets), the union region for the second point's row partials, and
// Bs[2][s_cap * 512] (both points' column constants).
struct BcLayout {
  int rows_cap, s_cap;
  __host__ __device__ size_t off_A() const { return (sizeof(BcShared) + 15) & ~size_t(15); }
  __host__ __device__ size_t off_A2() const { return (off_A() + size_t(rows_cap) * 4 + 15) & ~size_t(15); }
  __host__ __device__ size_t off_rowpart() const { return (off_A2() + size_t(rows_cap) * 4 + 15) & ~size_t(15); }
  __host__ __device__ size_t off_u() const { return off_rowpart() + size_t(rows_cap) * s_cap * 8; }
  __host__ __device__ size_t off_B() const {
    const size_t u = size_t(rows_cap) * s_cap * 8, c = size_t(kBcWarps) * kBcStrip * 4;
    return (off_u() + (u > c ? u : c) + 15) & ~size_t(15);
  }
  int nst;  // stages of each warp's row ring (cp.async)
  __host__ __device__ size_t off_ring() const { return (off_B() + size_t(2) * s_cap * kBcStrip * 4 + 127) & ~size_t(127); }
  __host__ __device__ size_t bytes() const { return off_ring() + size_t(kBcWarps) * nst * kBcStrip * 4; }
};

// Per-lane cp.async (LDGSTS) ring of row segments: each lane streams ITS 4 x
// 16 B of every row segment into its own slots of the warp's ring, so the
// lane's wait_group is the only synchronisation; nst - 1 rows are in flight
// per warp while one is exponentiated (a register double buffer holds one;
// ncu: the sweep was long_scoreboard-bound on C at 2.4 TB/s).
struct BcRowStream {
  float4* ring;       // warp ring + lane: slot (k % nst) at ring + (k % nst) * 128
  const float4* g;    // P.C + j0 (as float4) + lane
  int64_t ld4, i0, step, cnt;
  int nst;
  __device__ __forceinline__ void issue(int64_t k) const {
    if (k < cnt) {
      const float4* src = g + (i0 + k * step) * ld4;
      float4* dst = ring + (k % nst) * (kBcStrip / 4);
#pragma unroll
      for (int q4 = 0; q4 < 4; ++q4)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst + 32 * q4)), "l"(src + 32 * q4)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  __device__ __forceinline__ void wait() const {  // all but the nst - 1 newest groups done
    switch (nst) {
      case 2: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
      case 3: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
      case 4: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
      case 5: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
      default: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    }
  }
  __device__ __forceinline__ void get(int64_t k, float4 (&v)[4]) const {
    const float4* src = ring + (k % nst) * (kBcStrip / 4);
#pragma unroll
    for (int q4 = 0; q4 < 4; ++q4) v[q4] = src[32 * q4];
  }
};
constexpr int kBcSlots = kSlots + 1;  // + the provisional next z_bar of the fused sweep
constexpr int S_ZB2 = kSlots;

struct BcCtx {
  const BcProblem* P;
  BcWs* W;
  BcShared* sm;
  float* A;         // [rows_cap]
  float* A2;        // [rows_cap]: second point of the fused sweep
  float* Bs;        // [2][s_cap * kBcStrip]: column constants of the fused sweep
  float4* ring;     // [kBcWarps][nst][kBcStrip / 4]
  int nst;
  float2* rowpart;  // [rows_cap][s_cap]
  float* colacc;    // [kBcWarps][kBcStrip] (sweep) ...
  float2* wk;       // ... or [rows_cap][s_cap] (cost pass)
  int s_cap;
  AspotCtl* c;     // == sm->ctl
  int64_t n;
  int rank, cs;
  int64_t lo, hi;  // the CTA's index slice
  int xphase;      // exchange buffer parity (uniform over the cluster)
  uint64_t sweep_ns;  // time spent in sweeps (thread 0)
  bool fuse;          // K1'' fused z_check' + next z_bar sweep
  __device__ double* slot(int k) const { return W->slots + k * W->stride; }
  __device__ double* rows(int role) const { return W->sums + int64_t(2 * role) * n; }
  __device__ double* cols(int role) const { return W->sums + int64_t(2 * role + 1) * n; }
};

__device__ __forceinline__ void bc_sync() { cgx::this_cluster().sync(); }

// Fixed-order cluster reduction of kBcX scalars (acc_join semantics for the
// first kNumAcc, max for the flag): every CTA writes its row, one barrier,
// every CTA reduces all rows in rank order -> identical totals in sm->tot.
// SUMS: every slot below kNumAcc is a plain sum, kNumAcc and kNumAcc + 1 are maxima.
__device__ __forceinline__ double bc_join(bool sums, int k, double a, double b) {
  if (k >= kNumAcc) return (sums || k == kNumAcc) ? fmax(a, b) : a + b;
  return sums ? a + b : acc_join(k, a, b);
}
__device__ __forceinline__ double bc_init(bool sums, int k) {
  if (sums) return k >= kNumAcc ? -INFINITY : 0.0;
  return k < kNumAcc ? acc_init(k) : 0.0;
}

// Publishes the CTA's totals (sm->red[k][0], from bc_block_acc).
template <bool SUMS = false>
__device__ void bc_exchange(BcCtx& X) {
  double* buf = X.W->xch + int64_t(X.xphase & 1) * X.cs * kBcX;
  X.xphase += 1;
  if (threadIdx.x < kBcX) buf[X.rank * kBcX + threadIdx.x] = X.sm->red[threadIdx.x][0];
  bc_sync();
  if (threadIdx.x < kBcX) {
    const int k = threadIdx.x;
    double a = bc_init(SUMS, k);
    for (int r = 0; r < X.cs; ++r) a = bc_join(SUMS, k, a, __ldcg(buf + r * kBcX + k));
    X.sm->tot[k] = a;
  }
  __syncthreads();
}

// Block reduction of kBcX accumulators; the CTA's totals land in
// sm->red[k][0] (what bc_exchange publishes).
template <bool SUMS = false>
__device__ void bc_block_acc(BcCtx& X, double (&acc)[kBcX]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < kBcX; ++k) {
    double x = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = bc_join(SUMS, k, x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) X.sm->red[k][wid] = x;
  }
  __syncthreads();
  if (threadIdx.x < kBcX) {
    const int k = threadIdx.x;
    double x = X.sm->red[k][0];
    for (int w2 = 1; w2 < kBcWarps; ++w2) x = bc_join(SUMS, k, x, X.sm->red[k][w2]);
    X.sm->red[k][0] = x;
  }
  __syncthreads();
}

// One sweep over the CTA's rows of the point (u + lu, v + lv, w):
//   rows_out[i] (fp64 row sums of the CTA's rows), X.W->colpart[rank][j]
//   (fp32 (sum, log2 scale) column partials of all columns), returns the
//   CTA's max exponent (natural units). COST: also W_out[i] = sum_j C_ij
//   B'_ij and K_out[i] = sum_j C_ij fb_j (no column partials).
template <bool COST>
__device__ __noinline__ double bc_sweep(BcCtx& X, const double* z, const double* lu, const double* lv, const double* fb,
                           double* rows_out, double* W_out, double* K_out) {
  BcShared& sm = *X.sm;
  const BcProblem& P = *X.P;
  const int64_t n = X.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* u = z;
  const double* v = z + n;
  const double w = __ldcg(z + 2 * n);
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    double a = __ldcg(u + i);
    if (lu) a = a + __ldcg(lu + i);
    X.A[i - X.lo] = float((a + w) * kLog2e);
  }
  const int S = int((n + kBcStrip - 1) / kBcStrip);
  const int PH = kBcWarps / S;
  const int strip = warp % S, ph = warp / S;
  const bool active = ph < PH;
  const int64_t j0 = int64_t(strip) * kBcStrip;
  float2 Bj[kPairs], Fb[kPairs];
#pragma unroll
  for (int q = 0; q < kPairs; ++q) {
    float b[2], f[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int64_t j = f32_col(j0, lane, q, h);
      double vv = -INFINITY;
      f[h] = 0.f;
      if (j < n) {
        vv = __ldcg(v + j);
        if (lv) vv = vv + __ldcg(lv + j);
        vv = vv * kLog2e;
        if (COST) f[h] = float(__ldcg(fb + j));
      }
      b[h] = float(vv);
    }
    Bj[q] = make_float2(b[0], b[1]);
    Fb[q] = make_float2(f[0], f[1]);
  }
  __syncthreads();
  float2 cacc[kPairs];
#pragma unroll
  for (int q = 0; q < kPairs; ++q) cacc[q] = make_float2(0.f, 0.f);
  float sigma = -INFINITY, mmax = -INFINITY;
  const float2 G = make_float2(-P.g2, -P.g2);
  if (active) {
    const int64_t cnt = X.hi > X.lo + ph ? (X.hi - X.lo - ph + PH - 1) / PH : 0;
    const BcRowStream rsm{X.ring + warp * X.nst * (kBcStrip / 4) + lane,
                          reinterpret_cast<const float4*>(P.C + j0) + lane, P.ld / 4, X.lo + ph, PH, cnt, X.nst};
    for (int k = 0; k < X.nst - 1; ++k) rsm.issue(k);
    for (int64_t kk = 0; kk < cnt; ++kk) {
      const int64_t i = X.lo + ph + kk * PH;
      rsm.issue(kk + X.nst - 1);  // into the slot of row kk - 1, consumed last step
      rsm.wait();
      float4 cur[4];
      rsm.get(kk, cur);
      float2 cc[kPairs], t[kPairs];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cc[2 * k] = make_float2(cur[k].x, cur[k].y);
        cc[2 * k + 1] = make_float2(cur[k].z, cur[k].w);
      }
#pragma unroll
      for (int q = 0; q < kPairs; ++q) t[q] = __ffma2_rn(G, cc[q], Bj[q]);
      float m = warp_maxf(tree_max2<kPairs>(t));
      const float ms = (m == -INFINITY) ? 0.f : m;
      const float2 M2 = make_float2(-ms, -ms);
      float2 p[kPairs];
#pragma unroll
      for (int q = 0; q < kPairs; ++q) {
        const float2 d = __fadd2_rn(t[q], M2);
        p[q] = make_float2(ex2f(d.x), ex2f(d.y));
      }
      float rs = tree_sum2<kPairs>(p);
      float ws = 0.f, ks = 0.f;
      if (COST) {
        float2 W2 = make_float2(0.f, 0.f), K2 = W2;
#pragma unroll
        for (int q = 0; q < kPairs; ++q) {
          W2 = __ffma2_rn(cc[q], p[q], W2);
          K2 = __ffma2_rn(cc[q], Fb[q], K2);
        }
        ws = W2.x + W2.y;
        ks = K2.x + K2.y;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        rs += __shfl_xor_sync(0xffffffffu, rs, o);
        if (COST) {
          ws += __shfl_xor_sync(0xffffffffu, ws, o);
          ks += __shfl_xor_sync(0xffffffffu, ks, o);
        }
      }
      const int64_t il = i - X.lo;
      if (lane == 0) {
        X.rowpart[il * X.s_cap + strip] = make_float2(rs, ms);
        if (COST) X.wk[il * X.s_cap + strip] = make_float2(ws, ks);
      }
      if (!COST) {
        const float mA = (m == -INFINITY) ? -INFINITY : m + X.A[il];
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
    }
  }
  if (!COST) {
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      const int cidx = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
      X.colacc[warp * kBcStrip + cidx] = cacc[q].x;
      X.colacc[warp * kBcStrip + cidx + 1] = cacc[q].y;
    }
    if (lane == 0) {
      sm.colsig[warp] = sigma;
      sm.wmax[warp] = mmax;
    }
  }
  __syncthreads();
  // row sums of the CTA's rows (fp64, the row offset added back exactly)
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    const int64_t il = i - X.lo;
    double a = __ldcg(u + i);
    if (lu) a = a + __ldcg(lu + i);
    const double a2 = (a + w) * kLog2e;
    double rr = 0.0, wc = 0.0, kk = 0.0;
    for (int s = 0; s < S; ++s) {
      const float2 rp = X.rowpart[il * X.s_cap + s];
      const float2 wkp = COST ? X.wk[il * X.s_cap + s] : make_float2(0.f, 0.f);
      if (rp.x != 0.f) {
        const double sc = exp2(double(rp.y) + a2);
        rr += double(rp.x) * sc;
        if (COST) wc += double(wkp.x) * sc;
      }
      if (COST) kk += double(wkp.y);
    }
    rows_out[i] = rr;
    if (COST) {
      W_out[i] = wc;
      K_out[i] = kk;
    }
  }
  if (COST) {
    __syncthreads();
    return -INFINITY;
  }
  // CTA column partials: combine the PH warps of each strip
  float2* cp = X.W->colpart + int64_t(X.rank) * n;
  for (int k = threadIdx.x; k < S * kBcStrip; k += kBcThreads) {
    const int s = k / kBcStrip, cidx = k % kBcStrip;
    const int64_t j = int64_t(s) * kBcStrip + cidx;
    if (j >= n) continue;
    float SIG = -INFINITY;
    for (int p2 = 0; p2 < PH; ++p2) SIG = fmaxf(SIG, sm.colsig[p2 * S + s]);
    float acc = 0.f;
    if (SIG != -INFINITY)
      for (int p2 = 0; p2 < PH; ++p2) {
        const float sg = sm.colsig[p2 * S + s];
        if (sg != -INFINITY) acc += X.colacc[(p2 * S + s) * kBcStrip + cidx] * ex2f(sg - SIG);
      }
    cp[j] = (SIG == -INFINITY) ? make_float2(0.f, 0.f) : make_float2(acc, SIG);
  }
  float mx = -INFINITY;
  for (int ww = 0; ww < S * PH; ++ww) mx = fmaxf(mx, sm.wmax[ww]);
  __syncthreads();
  return double(mx) * kLn2;
}

// Column sums of the CTA's slice over the cluster's partials (after a barrier).
__device__ __forceinline__ double bc_col_sum(const BcCtx& X, int64_t j, const float2* cp) {
  float M = -INFINITY;
  for (int r = 0; r < X.cs; ++r) {
    const float2 x = __ldcg(cp + int64_t(r) * X.n + j);
    if (x.x != 0.f) M = fmaxf(M, x.y);
  }
  if (M == -INFINITY) return 0.0;
  float S = 0.f;
  for (int r = 0; r < X.cs; ++r) {
    const float2 x = __ldcg(cp + int64_t(r) * X.n + j);
    if (x.x != 0.f) S += x.x * ex2f(x.y - M);
  }
  return double(S) * exp2(double(M));
}

// Sweep + evaluation + decision of a point (k_point_eval + decide_pending).
__device__ __noinline__ void bc_eval_swept(BcCtx& X, int slot, int role) {
  bc_sync();  // the point's slices (every CTA's writes) are complete
  const double* z = X.slot(slot);
  const uint64_t ts = globaltimer_ns();
  const double maxe = bc_sweep<false>(X, z, nullptr, nullptr, nullptr, X.rows(role), nullptr, nullptr);
  bc_sync();  // column partials of every CTA
  X.sweep_ns += globaltimer_ns() - ts;
  double acc[kBcX];
#pragma unroll
  for (int k = 0; k < kBcX; ++k) acc[k] = k < kNumAcc ? acc_init(k) : 0.0;
  const double* P_rt = X.P->rt;
  const double* P_ct = X.P->ct;
  double* rb = X.rows(role);
  double* cb = X.cols(role);
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    const double c = bc_col_sum(X, i, X.W->colpart);
    cb[i] = c;
    add_index_terms(acc, __ldcg(rb + i), c, __ldcg(z + i), __ldcg(z + X.n + i), P_rt[i], P_ct[i]);
  }
  bc_block_acc(X, acc);
  if (threadIdx.x == 0) X.sm->red[11][0] = nan_max(X.sm->red[11][0], maxe);
  __syncthreads();
  bc_exchange(X);
  if (threadIdx.x == 0) {
    double tot[kNumAcc];
#pragma unroll
    for (int k = 0; k < kNumAcc; ++k) tot[k] = X.sm->tot[k];
    apply_role(X.c, role, tot, __ldcg(z + 2 * X.n), true);
  }
  __syncthreads();
}

// K1'': ONE pass over the CTA's rows of C for two points (z_check' and the
// provisional next z_bar): each loaded entry is exponentiated
// for both, with the numerics of bc_sweep per point. Row sums -> rowsA /
// rowsB, column partials -> colpart / colpart2, max exponents -> maxe[2].
__device__ __noinline__ void bc_sweep2(BcCtx& X, const double* zA, const double* zB, double* rowsA, double* rowsB,
                                       double (&maxe)[2]) {
  const BcProblem& P = *X.P;
  const int64_t n = X.n;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double wA = __ldcg(zA + 2 * n), wB = __ldcg(zB + 2 * n);
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    X.A[i - X.lo] = float((__ldcg(zA + i) + wA) * kLog2e);
    X.A2[i - X.lo] = float((__ldcg(zB + i) + wB) * kLog2e);
  }
  const int S = int((n + kBcStrip - 1) / kBcStrip);
  const int PH = kBcWarps / S;
  const int strip = warp % S, ph = warp / S;
  const bool active = ph < PH;
  const int64_t j0 = int64_t(strip) * kBcStrip;
  float* BsA = X.Bs;
  float* BsB = X.Bs + int64_t(X.s_cap) * kBcStrip;
  for (int64_t j = threadIdx.x; j < int64_t(S) * kBcStrip; j += kBcThreads) {
    BsA[j] = j < n ? float(__ldcg(zA + n + j) * kLog2e) : -INFINITY;
    BsB[j] = j < n ? float(__ldcg(zB + n + j) * kLog2e) : -INFINITY;
  }
  __syncthreads();
  float2 caA[kPairs], caB[kPairs];
#pragma unroll
  for (int q = 0; q < kPairs; ++q) caA[q] = caB[q] = make_float2(0.f, 0.f);
  float sigA = -INFINITY, sigB = -INFINITY, mmA = -INFINITY, mmB = -INFINITY;
  const float2 G = make_float2(-P.g2, -P.g2);
  float2* rpB = X.wk;  // the union region holds the second point's row partials during the loop
  if (active) {
    const int64_t cnt = X.hi > X.lo + ph ? (X.hi - X.lo - ph + PH - 1) / PH : 0;
    const BcRowStream rsm{X.ring + warp * X.nst * (kBcStrip / 4) + lane,
                          reinterpret_cast<const float4*>(P.C + j0) + lane, P.ld / 4, X.lo + ph, PH, cnt, X.nst};
    for (int k = 0; k < X.nst - 1; ++k) rsm.issue(k);
    for (int64_t kk = 0; kk < cnt; ++kk) {
      const int64_t i = X.lo + ph + kk * PH;
      rsm.issue(kk + X.nst - 1);
      rsm.wait();
      float4 cur[4];
      rsm.get(kk, cur);
      float2 cc[kPairs];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        cc[2 * k] = make_float2(cur[k].x, cur[k].y);
        cc[2 * k + 1] = make_float2(cur[k].z, cur[k].w);
      }
      const int64_t il = i - X.lo;
      // each point: exact segment max, MUFU burst, row partial, column update
      // (unrolled over the two points, so every select below is static)
#pragma unroll
      for (int pt = 0; pt < 2; ++pt) {
        float2 p[kPairs];
        const float4* b4 = reinterpret_cast<const float4*>((pt ? BsB : BsA) + j0) + lane;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const float4 b = b4[32 * q4];
          p[2 * q4] = __ffma2_rn(G, cc[2 * q4], make_float2(b.x, b.y));
          p[2 * q4 + 1] = __ffma2_rn(G, cc[2 * q4 + 1], make_float2(b.z, b.w));
        }
        const float m = warp_maxf(tree_max2<kPairs>(p));
        const float ms = (m == -INFINITY) ? 0.f : m;
        const float2 M2 = make_float2(-ms, -ms);
#pragma unroll
        for (int q = 0; q < kPairs; ++q) {
          const float2 d = __fadd2_rn(p[q], M2);
          p[q] = make_float2(ex2f(d.x), ex2f(d.y));
        }
        float rs = tree_sum2<kPairs>(p);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
        if (lane == 0) (pt ? rpB : X.rowpart)[il * X.s_cap + strip] = make_float2(rs, ms);
        const float mA = (m == -INFINITY) ? -INFINITY : m + (pt ? X.A2 : X.A)[il];
        float sg = pt ? sigB : sigA;
        if (mA > sg) {  // warp-uniform
          const float sc = ex2f(sg - mA);
#pragma unroll
          for (int q = 0; q < kPairs; ++q) {
            if (pt) caB[q] = __fmul2_rn(caB[q], make_float2(sc, sc));
            else caA[q] = __fmul2_rn(caA[q], make_float2(sc, sc));
          }
          sg = mA;
        }
        if (pt) { sigB = sg; mmB = fmaxf(mmB, mA); } else { sigA = sg; mmA = fmaxf(mmA, mA); }
        const float f = (mA == -INFINITY) ? 0.f : ex2f(mA - sg);
        const float2 F2 = make_float2(f, f);
#pragma unroll
        for (int q = 0; q < kPairs; ++q) {
          if (pt) caB[q] = __ffma2_rn(p[q], F2, caB[q]);
          else caA[q] = __ffma2_rn(p[q], F2, caA[q]);
        }
      }
    }
  }
  __syncthreads();
  // row sums of both points (fp64 row offsets)
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    const int64_t il = i - X.lo;
    const double a2A = (__ldcg(zA + i) + wA) * kLog2e, a2B = (__ldcg(zB + i) + wB) * kLog2e;
    double ra = 0.0, rb = 0.0;
    for (int s2 = 0; s2 < S; ++s2) {
      const float2 pa = X.rowpart[il * X.s_cap + s2], pb = rpB[il * X.s_cap + s2];
      if (pa.x != 0.f) ra += double(pa.x) * exp2(double(pa.y) + a2A);
      if (pb.x != 0.f) rb += double(pb.x) * exp2(double(pb.y) + a2B);
    }
    rowsA[i] = ra;
    rowsB[i] = rb;
  }
  __syncthreads();  // rpB is dead: the region takes the column accumulators
  // column partials, one point at a time through the per-warp accumulators
  // (explicit per point: selecting between two register arrays by pointer
  // would put them in local memory)
#pragma unroll
  for (int pt = 0; pt < 2; ++pt) {
#pragma unroll
    for (int q = 0; q < kPairs; ++q) {
      const int cidx = 4 * lane + 128 * (q >> 1) + 2 * (q & 1);
      const float2 v = pt == 0 ? caA[q] : caB[q];
      X.colacc[warp * kBcStrip + cidx] = v.x;
      X.colacc[warp * kBcStrip + cidx + 1] = v.y;
    }
    if (lane == 0) {
      X.sm->colsig[warp] = pt == 0 ? sigA : sigB;
      X.sm->wmax[warp] = pt == 0 ? mmA : mmB;
    }
    __syncthreads();
    float2* cp = (pt == 0 ? X.W->colpart : X.W->colpart2) + int64_t(X.rank) * n;
    for (int k = threadIdx.x; k < S * kBcStrip; k += kBcThreads) {
      const int s2 = k / kBcStrip, cidx = k % kBcStrip;
      const int64_t j = int64_t(s2) * kBcStrip + cidx;
      if (j >= n) continue;
      float SIG = -INFINITY;
      for (int p2 = 0; p2 < PH; ++p2) SIG = fmaxf(SIG, X.sm->colsig[p2 * S + s2]);
      float acc = 0.f;
      if (SIG != -INFINITY)
        for (int p2 = 0; p2 < PH; ++p2) {
          const float sg = X.sm->colsig[p2 * S + s2];
          if (sg != -INFINITY) acc += X.colacc[(p2 * S + s2) * kBcStrip + cidx] * ex2f(sg - SIG);
        }
      cp[j] = (SIG == -INFINITY) ? make_float2(0.f, 0.f) : make_float2(acc, SIG);
    }
    float mx = -INFINITY;
    for (int ww = 0; ww < S * PH; ++ww) mx = fmaxf(mx, X.sm->wmax[ww]);
    maxe[pt] = double(mx) * kLn2;
    __syncthreads();
  }
}

// Fused evaluation of z_check' (R_NEW, decided now) and the provisional next
// z_bar (S_ZB2: its sums go to R_BAR, its totals are stashed for the next
// iteration's z_bar decision, which then needs no sweep).
__device__ __noinline__ void bc_eval2_swept(BcCtx& X) {
  bc_sync();
  const double* zA = X.slot(S_ZN);
  const double* zB = X.slot(S_ZB2);
  const uint64_t ts = globaltimer_ns();
  double maxe[2];
  bc_sweep2(X, zA, zB, X.rows(R_NEW), X.rows(R_BAR), maxe);
  bc_sync();
  X.sweep_ns += globaltimer_ns() - ts;
  const double* rt = X.P->rt;
  const double* ct = X.P->ct;
#pragma unroll 1
  for (int pt = 0; pt < 2; ++pt) {
    const double* z = pt == 0 ? zA : zB;
    const int role = pt == 0 ? R_NEW : R_BAR;
    const float2* cp = pt == 0 ? X.W->colpart : X.W->colpart2;
    double acc[kBcX];
#pragma unroll
    for (int k = 0; k < kBcX; ++k) acc[k] = k < kNumAcc ? acc_init(k) : 0.0;
    double* rb = X.rows(role);
    double* cb = X.cols(role);
    for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
      const double c = bc_col_sum(X, i, cp);
      cb[i] = c;
      add_index_terms(acc, __ldcg(rb + i), c, __ldcg(z + i), __ldcg(z + X.n + i), rt[i], ct[i]);
    }
    bc_block_acc(X, acc);
    if (threadIdx.x == 0) X.sm->red[11][0] = nan_max(X.sm->red[11][0], maxe[pt]);
    __syncthreads();
    bc_exchange(X);
    if (threadIdx.x == 0) {
      double tot[kNumAcc];
#pragma unroll
      for (int k = 0; k < kNumAcc; ++k) tot[k] = X.sm->tot[k];
      if (pt == 0) {
        apply_role(X.c, R_NEW, tot, __ldcg(z + 2 * X.n), true);
      } else {
        for (int k = 0; k < kNumAcc; ++k) X.sm->stash[k] = tot[k];
        X.sm->stash_valid = 1;
      }
    }
    __syncthreads();
  }
}

__device__ void bc_kill_gates(AspotCtl* c) {  // ctl_finish's non-finite fold (solvers.hpp:83-87)
  c->g_alive = 0;
  c->g_hat_sweep = c->g_hat_scaled = c->g_new_sweep = c->g_new_scaled = 0;
  c->g_new_one = c->g_new_eval = 0;
}

// Exact block update (k_gk_update) of the slice, then the exchange of the
// non-finite flag and, for a w-block point, of its scaled functionals;
// the decision at the new point when it was scaled.
__device__ __noinline__ void bc_gk_update(BcCtx& X, int which) {
  AspotCtl* c = X.c;
  const int64_t n = X.n;
  int block, role;
  int src_slot, dst_slot, dst_role;
  if (which == 0) {
    block = c->block_hat; src_slot = S_ZG; role = R_GRAVE; dst_slot = S_ZH; dst_role = R_HAT;
  } else {
    block = c->block_check;
    const bool keep = c->keep_check;
    src_slot = keep ? S_ZC : S_ZH; role = keep ? R_CHECK : R_HAT; dst_slot = S_ZN; dst_role = R_NEW;
  }
  const double* src = X.slot(src_slot);
  double* dst = X.slot(dst_slot);
  const double* rowb = X.rows(role);
  const double* colb = X.cols(role);
  const double* rt = X.P->rt;
  const double* ct = X.P->ct;
  bool finite = true;
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    double x = __ldcg(src + i);
    if (block == 0) x = x + (log(rt[i]) - log(__ldcg(rowb + i) + eexp(x)));
    dst[i] = x;
    finite = finite && isfinite(x);
    double y = __ldcg(src + n + i);
    if (block == 1) y = y + (log(ct[i]) - log(__ldcg(colb + i) + eexp(y)));
    dst[n + i] = y;
    finite = finite && isfinite(y);
  }
  const double ws = __ldcg(src + 2 * n);
  const double wd = block == 2 ? ws + (log(c->s) - log(c->ps[role].total)) : ws;
  if (X.rank == 0 && threadIdx.x == 0) dst[2 * n] = wd;
  finite = finite && isfinite(wd);
  const bool scaled = which == 0 ? c->g_hat_scaled : c->g_new_scaled;
  double acc[kBcX];
#pragma unroll
  for (int k = 0; k < kBcX; ++k) acc[k] = k < kNumAcc ? acc_init(k) : 0.0;
  acc[kNumAcc] = finite ? 0.0 : 1.0;
  const double dw = wd - ws;
  if (scaled) {
    const double fs = exp(dw);
    double* dr = X.rows(dst_role);
    double* dc = X.cols(dst_role);
    for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
      const double rb = __ldcg(rowb + i) * fs, cb = __ldcg(colb + i) * fs;
      dr[i] = rb;
      dc[i] = cb;
      add_index_terms(acc, rb, cb, __ldcg(src + i), __ldcg(src + n + i), rt[i], ct[i]);
    }
  }
  bc_block_acc(X, acc);
  bc_exchange(X);
  if (threadIdx.x == 0) {
    if (X.sm->tot[kNumAcc] != 0.0) {
      bc_kill_gates(c);
    } else if (scaled) {
      double tot[kNumAcc];
#pragma unroll
      for (int k = 0; k < kNumAcc; ++k) tot[k] = X.sm->tot[k];
      tot[11] = c->ps[role].maxe + dw;
      apply_role(c, dst_role, tot, wd, false);
    }
  }
  __syncthreads();
}

// Round_pot (rounding.hpp:46-77) of B(z_check), the implicit-plan form of
// plan.cuh round_pot_implicit with P0 = Q0 = 1 and no rank-1 input term
// (two sweeps: the column clip's column sums, then the final row sums fused
// with <C, X>, as k_rowcost_f32). Rank 0 writes the metrics.
__device__ __noinline__ double bc_round(BcCtx& X, BcResult* res) {
  const int64_t n = X.n;
  const BcProblem& P = *X.P;
  const double s = X.c->s;
  double* lrho = X.W->vec;         // log rho (row clip)
  double* lkap = X.W->vec + n;     // log kappa (column clip)
  double* fbv = X.W->vec + 2 * n;  // deficit column factors max(c - colX3, 0)
  double* rx = X.W->vec + 3 * n;   // rowX3
  double* arho = X.W->vec + 4 * n; // alpha rho
  double* cx3 = X.W->vec + 5 * n;  // colX3
  const double* zc = X.slot(S_ZC);
  const double* row0 = X.rows(R_CHECK);
  double acc[kBcX];
  // out *= min(1, s / mass)
#pragma unroll
  for (int k = 0; k < kBcX; ++k) acc[k] = bc_init(true, k);
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) acc[0] += __ldcg(row0 + i);
  bc_block_acc<true>(X, acc);
  bc_exchange<true>(X);
  const double mass1 = X.sm->tot[0];
  const double alpha = mass1 > 0 ? fmin(1.0, s / mass1) : 1.0;
  // row clip
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    const double row = alpha * __ldcg(row0 + i);
    const double rh = row > 0 ? fmin(1.0, P.r[i] / row) : 1.0;
    lrho[i] = log(rh);
    arho[i] = alpha * rh;
  }
  bc_sync();
  // column clip: column sums of diag(rho) B
  (void)bc_sweep<false>(X, zc, lrho, nullptr, nullptr, X.rows(R_EVAL), nullptr, nullptr);
  bc_sync();
  for (int64_t j = X.lo + threadIdx.x; j < X.hi; j += kBcThreads) {
    const double col3 = alpha * bc_col_sum(X, j, X.W->colpart);
    const double kp = col3 > 0 ? fmin(1.0, P.c[j] / col3) : 1.0;
    const double c3 = kp * col3;
    lkap[j] = log(kp);
    cx3[j] = c3;
    fbv[j] = fmax(P.c[j] - c3, 0.0);
  }
  bc_sync();
  // final row sums of B diag(kappa) and the cost's per-row terms
  double* rr = X.rows(R_EVAL);
  double* Wv = X.W->vec + 6 * n;  // (not R_BAR's sums: a record rounding runs between the fused
  double* Kv = X.W->vec + 7 * n;  //  sweep that wrote the next z_bar's sums and their use)
  (void)bc_sweep<true>(X, zc, nullptr, lkap, fbv, rr, Wv, Kv);
#pragma unroll
  for (int k = 0; k < kBcX; ++k) acc[k] = bc_init(true, k);
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    const double x3 = __ldcg(arho + i) * __ldcg(rr + i);
    rx[i] = x3;
    acc[0] += x3;                                // mass3
    acc[1] += fmax(P.r[i] - x3, 0.0);            // na
    acc[2] += __ldcg(fbv + i);                   // nb (the slice's columns)
  }
  bc_block_acc<true>(X, acc);
  bc_exchange<true>(X);
  const double mass3 = X.sm->tot[0], na = X.sm->tot[1], nb = X.sm->tot[2];
  const double deficit = s - mass3;
  double f = 0.0;
  int infeasible = 0;
  if (deficit > 0) {  // deficit fill (rounding.hpp:63-75)
    if (na <= 0 || nb <= 0) infeasible = 1;
    else f = deficit / (na * nb);
  }
  // <C, X> = sum_i alpha rho_i W_i + f fa_i K_i ; slacks ; gap (core.hpp:199-219)
#pragma unroll
  for (int k = 0; k < kBcX; ++k) acc[k] = bc_init(true, k);
  for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
    const double x3 = __ldcg(rx + i);
    const double fa = fmax(P.r[i] - x3, 0.0);
    acc[0] += __ldcg(arho + i) * __ldcg(Wv + i) + (f * fa) * __ldcg(Kv + i);
    const double rxi = x3 + f * fa * nb;
    const double cxj = __ldcg(cx3 + i) + f * na * __ldcg(fbv + i);
    P.row_slack[i] = P.r[i] - rxi;
    P.col_slack[i] = P.c[i] - cxj;
    acc[kNumAcc] = fmax(acc[kNumAcc], fmax(rxi - P.r[i], 0.0));
    acc[kNumAcc + 1] = fmax(acc[kNumAcc + 1], fmax(cxj - P.c[i], 0.0));
  }
  bc_block_acc<true>(X, acc);
  bc_exchange<true>(X);
  const double cost = X.sm->tot[0];
  if (res && X.rank == 0 && threadIdx.x == 0) {
    const double mass = mass3 + f * na * nb;
    res->cost = cost;
    res->mass = mass;
    res->gap = fmax(fmax(fmax(X.sm->tot[kNumAcc], 0.0), fmax(X.sm->tot[kNumAcc + 1], 0.0)), fabs(mass - s));
    res->infeasible = infeasible;
  }
  return cost;
}

// record_rounded_cost: the record just appended (record(t), solvers.hpp:
// 309-318) gets the cost of round_pot(B(z_check)) at that t.
__device__ void bc_record_cost(BcCtx& X, int64_t len_before, TraceDev* trace) {
  const AspotCtl* c = X.c;
  if (!c->record_rounded_cost || c->trace_len == len_before || c->trace_len > c->trace_cap) return;
  const double cost = bc_round(X, nullptr);
  if (trace && threadIdx.x == 0) trace[c->trace_len - 1].rounded_cost = cost;
}

// The persistent batch kernel: grid = cs x clusters, cluster = (cs, 1, 1).
__global__ void __launch_bounds__(kBcThreads, 1) k_batch_aspot(const BcProblem* probs, int count, BcWs* wss,
                                                              BcResult* results, int* queue, BcLayout lay, int fuse,
                                                              const int* ready) {
  extern __shared__ __align__(16) unsigned char bc_smem_raw[];
  BcShared* sm = reinterpret_cast<BcShared*>(bc_smem_raw);
  cgx::cluster_group cl = cgx::this_cluster();
  const int cs = int(cl.num_blocks());
  const int rank = int(cl.block_rank());
  const int cid = int(blockIdx.x) / cs;
  BcWs* W = wss + cid;
  for (;;) {
    if (rank == 0 && threadIdx.x == 0) {
      const int q = atomicAdd(queue, 1);
      W->cur = q;
      // the host uploads problems while the launch runs: wait for this one
      // (1 = ready, 2 = its upload failed; bounded so a lost flag cannot hang the GPU)
      int st = 1;
      if (ready && q < count) {
        const uint64_t t0 = globaltimer_ns();
        for (;;) {
          asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(st) : "l"(ready + q) : "memory");
          if (st != 0) break;
          if (globaltimer_ns() - t0 > 60000000000ull) { st = 3; break; }
          __nanosleep(200);
        }
      }
      W->skip = st != 1;
    }
    bc_sync();
    const int p = *reinterpret_cast<volatile int*>(&W->cur);
    if (p >= count) break;
    if (*reinterpret_cast<volatile int*>(&W->skip)) {  // uniform over the cluster
      bc_sync();
      continue;
    }
    BcCtx X;
    X.P = probs + p;
    X.W = W;
    X.sm = sm;
    X.c = reinterpret_cast<AspotCtl*>(sm->ctl);
    X.A2 = reinterpret_cast<float*>(bc_smem_raw + lay.off_A2());
    X.Bs = reinterpret_cast<float*>(bc_smem_raw + lay.off_B());
    X.fuse = fuse != 0;
    X.ring = reinterpret_cast<float4*>(bc_smem_raw + lay.off_ring());
    X.nst = lay.nst;
    X.A = reinterpret_cast<float*>(bc_smem_raw + lay.off_A());
    X.rowpart = reinterpret_cast<float2*>(bc_smem_raw + lay.off_rowpart());
    X.colacc = reinterpret_cast<float*>(bc_smem_raw + lay.off_u());
    X.wk = reinterpret_cast<float2*>(bc_smem_raw + lay.off_u());
    X.s_cap = lay.s_cap;
    X.n = X.P->ctl0.n;
    X.rank = rank;
    X.cs = cs;
    X.lo = X.n * rank / cs;
    X.hi = X.n * (rank + 1) / cs;
    X.xphase = 0;
    X.sweep_ns = 0;
    const uint64_t t_problem = globaltimer_ns();
    {  // control block copy, zero dual points (z = z_check = z_bar = 0)
      const uint32_t* src = reinterpret_cast<const uint32_t*>(&X.P->ctl0);
      for (int k = threadIdx.x; k < kCtlWords; k += kBcThreads) sm->ctl[k] = src[k];
      const int64_t n = X.n;
      if (threadIdx.x == 0) sm->stash_valid = 0;
      for (int s2 = 0; s2 < kBcSlots; ++s2) {
        double* zz = X.slot(s2);
        for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
          zz[i] = 0.0;
          zz[n + i] = 0.0;
        }
        if (rank == 0 && threadIdx.x == 0) zz[2 * n] = 0.0;
      }
      __syncthreads();
      if (threadIdx.x == 0) X.c->t0_ns = globaltimer_ns();
    }
    AspotCtl* c = X.c;
    TraceDev* trace = rank == 0 ? X.P->trace : nullptr;
    IterLogDev* lg = rank == 0 ? X.P->iterlog : nullptr;
    // phi_and_gradient(z_check = 0) (solvers.hpp:305), record(0) (:320)
    bc_eval_swept(X, S_ZC, R_CHECK);
    int64_t len0 = c->trace_len;
    if (threadIdx.x == 0 && !c->fatal) {
      c->error = c->ps[R_CHECK].err;
      c->phi_check = c->ps[R_CHECK].phi;
      c->g_active = 1;
      append_trace(c, trace, 0, c->error, c->phi_check);
      loop_head(c);
    }
    __syncthreads();
    bc_record_cost(X, len0, trace);
    const int64_t n = X.n;
    while (c->g_active) {  // identical on every CTA of the cluster
      // z_bar: range check and gradient of a new iteration (solvers.hpp:336-337)
      if (c->g_new) {
        const int stashed = X.sm->stash_valid;
        __syncthreads();  // every thread has read the flag before thread 0 clears it
        if (stashed) {  // z_bar was swept with the last z_check' (K1'')
          if (threadIdx.x == 0) {
            apply_role(c, R_BAR, X.sm->stash, __ldcg(X.slot(S_ZB) + 2 * n), false);
            X.sm->stash_valid = 0;
          }
          __syncthreads();
        } else {
          bc_eval_swept(X, S_ZB, R_BAR);
        }
      }
      if (c->g_alive) {  // z_next = z_bar - step grad; z_grave = z_bar + theta (z_next - z) (:338-339)
        const bool fresh = c->g_new;
        const double step = c->step, th = c->theta;
        const double* zb = X.slot(S_ZB);
        const double* z = X.slot(S_Z);
        double* g = X.slot(S_G);
        double* zg = X.slot(S_ZG);
        const double* rb = X.rows(R_BAR);
        const double* cb = X.cols(R_BAR);
        for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            const int64_t k = side * n + i;
            double gk;
            if (fresh) {
              gk = side == 0 ? (__ldcg(rb + i) + eexp(__ldcg(zb + k))) - X.P->rt[i]
                             : (__ldcg(cb + i) + eexp(__ldcg(zb + k))) - X.P->ct[i];
              g[k] = gk;
            } else {
              gk = __ldcg(g + k);
            }
            const double zn = __ldcg(zb + k) - step * gk;
            zg[k] = __ldcg(zb + k) + th * (zn - __ldcg(z + k));
          }
        }
        if (rank == 0 && threadIdx.x == 0) {
          const int64_t k = 2 * n;
          double gk;
          if (fresh) { gk = c->ps[R_BAR].total - c->s; g[k] = gk; } else { gk = __ldcg(g + k); }
          const double zn = __ldcg(zb + k) - step * gk;
          zg[k] = __ldcg(zb + k) + th * (zn - __ldcg(z + k));
        }
        bc_eval_swept(X, S_ZG, R_GRAVE);
      }
      if (c->g_alive) bc_gk_update(X, 0);                 // z_hat (solvers.hpp:340)
      if (c->g_hat_sweep) bc_eval_swept(X, S_ZH, R_HAT);  // phi(z_hat), z_best (:341-343)
      if (c->g_alive) bc_gk_update(X, 1);                 // z_check' = GK(z_best) (:344)
      if (c->g_new_sweep) {  // phi, grad at z_check' (:345), fused with the next z_bar
        if (X.fuse) {
          const bool keep = c->keep_check;
          const double th = theta_next_d(c->theta), om = 1.0 - th;
          const double* zc = X.slot(S_ZC);
          const double* zh = X.slot(S_ZH);
          const double* zn = X.slot(S_ZN);
          double* zb2 = X.slot(S_ZB2);
          for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads)
#pragma unroll
            for (int side = 0; side < 2; ++side) {
              const int64_t k = side * n + i;
              zb2[k] = om * __ldcg(zn + k) + th * (keep ? __ldcg(zc + k) : __ldcg(zh + k));
            }
          if (rank == 0 && threadIdx.x == 0) {
            const int64_t k = 2 * n;
            zb2[k] = om * __ldcg(zn + k) + th * (keep ? __ldcg(zc + k) : __ldcg(zh + k));
          }
          bc_eval2_swept(X);
        } else {
          bc_eval_swept(X, S_ZN, R_NEW);
        }
      }
      if (c->attempt_ok) {  // commit (k_commit)
        const bool keep = c->keep_check;
        const double th = theta_next_d(c->theta), om = 1.0 - th;
        double* z = X.slot(S_Z);
        double* zc = X.slot(S_ZC);
        const double* zh = X.slot(S_ZH);
        const double* zn = X.slot(S_ZN);
        double* zb = X.slot(S_ZB);
        double* rc = X.rows(R_CHECK);
        double* cc = X.cols(R_CHECK);
        const double* rn = X.rows(R_NEW);
        const double* cn = X.cols(R_NEW);
        for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
#pragma unroll
          for (int side = 0; side < 2; ++side) {
            const int64_t k = side * n + i;
            const double zbst = keep ? __ldcg(zc + k) : __ldcg(zh + k);
            const double zcn = __ldcg(zn + k);
            z[k] = zbst;
            zc[k] = zcn;
            zb[k] = om * zcn + th * zbst;
          }
          rc[i] = __ldcg(rn + i);
          cc[i] = __ldcg(cn + i);
        }
        if (rank == 0 && threadIdx.x == 0) {  // w (index 2n) has one writer
          const int64_t k = 2 * n;
          const double zbst = keep ? __ldcg(zc + k) : __ldcg(zh + k);
          const double zcn = __ldcg(zn + k);
          z[k] = zbst;
          zc[k] = zcn;
          zb[k] = om * zcn + th * zbst;
        }
      }
      __syncthreads();
      if (threadIdx.x == 0 && !c->attempt_ok) X.sm->stash_valid = 0;  // a retry keeps z_bar (no stash)
      len0 = c->trace_len;
      __syncthreads();
      if (threadIdx.x == 0) commit_state(c, trace, lg);
      __syncthreads();
      bc_sync();  // every slice of the committed points before the next attempt reads them
      bc_record_cost(X, len0, trace);
    }
    bc_round(X, results + p);
    if (rank == 0 && threadIdx.x == 0) {
      c->loop_end_ns = c->loop_end_ns ? c->loop_end_ns : globaltimer_ns();
      results[p].ctl = *c;
      results[p].done = 1;
      results[p].sweep_ns = X.sweep_ns;
      results[p].total_ns = globaltimer_ns() - t_problem;
      double* zo = X.P->zc_out;
      if (zo) zo[2 * n] = __ldcg(X.slot(S_ZC) + 2 * n);
    }
    {
      double* zo = X.P->zc_out;
      const double* zc = X.slot(S_ZC);
      if (zo)
        for (int64_t i = X.lo + threadIdx.x; i < X.hi; i += kBcThreads) {
          zo[i] = __ldcg(zc + i);
          zo[n + i] = __ldcg(zc + n + i);
        }
    }
    bc_sync();  // the workspace is free for the next problem
  }
}

}  // namespace potgpu
