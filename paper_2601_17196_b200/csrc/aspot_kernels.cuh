// aspot_kernels.cuh — device-resident control of the accelerated solver
// (reference: aspot_solve, solvers.hpp:265-385; Alg. 2 of PAPER.md:108-134).
//
// One step attempt is a fixed sequence of kernels; every decision the
// reference takes on the host (overflow -> halve the step, Greenkhorn block
// choice, z_best selection, stopping) is taken on the device by single-thread
// "scalar" kernels that write gate flags. Later kernels read the gates and
// become no-ops, so the whole attempt is replayable as one CUDA graph with no
// host round trip; the host only polls the state every few attempts.
#pragma once

#include <cstdlib>

#include "common.cuh"
#include "sweep.cuh"

namespace potgpu {

enum PointRole { R_BAR = 0, R_GRAVE = 1, R_HAT = 2, R_CHECK = 3, R_NEW = 4, R_EVAL = 5, kRoles = 6 };

enum CtlStatus { ST_RUNNING = -1 };

struct TraceDev {  // mirrors potgpu_trace_record
  int64_t t;
  double error, phi, rounded_cost, elapsed_s;
};
struct IterLogDev {  // mirrors potgpu_iter_log
  int64_t t;
  int32_t halvings, block_hat, zbest_is_check, block_check;
  double error, phi_check, phi_hat, theta;
};

struct RoundOut {
  double alpha, mass3, na, nb, f, mass, cost, row_gap, col_gap, gap;
  int infeasible, pad;
};

struct AspotCtl {
  // gates (read by kernels)
  int g_active;   // solve not finished
  int g_new;      // this attempt starts a new iteration (z_bar, grad recomputed)
  int g_alive;    // no range failure so far in this attempt
  int g_record;   // trace record rounding pending
  int g_round;    // rounding pipeline gate (set by the caller of the pipeline)
  int attempt_ok;
  int zbar_failed;
  int keep_check;
  int block_hat, block_check;
  int block_rule;
  int status;
  int halvings;
  int fatal;      // potgpu error code raised on the device (0 = none)
  int record_rounded_cost;
  int paused;     // loop stopped at pause_at (session API), not finished
  // sweep-vs-scale gates of z_hat and z_check' (block w: B scales by e^dw)
  int g_hat_sweep, g_hat_scaled, g_new_sweep, g_new_scaled;
  // z_check' by the one-sided sweep (block u or v from z_best = z_hat; sweep_pts1_f32)
  // and the gate of its evaluation (g_new_sweep | g_new_one); one_sided_ok: problem allows it
  int g_new_one, g_new_eval, one_sided_ok;
  int clamp_guard;  // fp64 (Eigen-clamped exp) problems: scale only far above the clamp floor
  // K1'' (sweep.cuh sweep_pts1_f32): the one-sided pass of z_check' also formed
  // the next z_bar's partials (g_bar_stash = 1), or z_check''s block was w and
  // z_bar's sums are z_best's scaled (= 2, sums in kbar, max exponent bar_maxe);
  // fuse_ok: the problem allows it; g_bar_sweep: this attempt sweeps z_bar
  // (= g_new unless stashed)
  int fuse_ok, g_bar_stash, g_bar_sweep, pad_k1;
  double bar_maxe;
  int64_t pause_at;
  int64_t loop_budget;  // attempts the device loop (graph WHILE node) may still run in this launch
  int64_t n, t, gk_calls, max_iterations, log_every, attempts, sweeps;
  int64_t trace_len, trace_cap, log_len, log_cap;
  double theta, step, gamma, eps_tilde, step_denom, s;
  double error, phi_check, phi_hat, phi_best;
  uint64_t t0_ns, loop_end_ns;
  PointScalars ps[kRoles];
  RoundOut ro;
};

// The scalar decisions (apply_role, commit_state) are single-thread code
// with many dependent reads and writes of the control block; on global
// memory each is an L2 round trip (measured: ~10 us of a 15 us evaluation
// with the SMs idle). The deciding block stages the block in shared memory,
// decides there, and writes it back (same arithmetic, same bits). Only that
// block touches the control block at that point of the launch.
constexpr int kCtlWords = int(sizeof(AspotCtl) / sizeof(uint32_t));
static_assert(sizeof(AspotCtl) % sizeof(uint32_t) == 0, "control block is copied as 32-bit words");

__device__ __forceinline__ void ctl_stage_in(uint32_t* sm, const AspotCtl* ctl) {
  const uint32_t* g = reinterpret_cast<const uint32_t*>(ctl);
  for (int k = threadIdx.x; k < kCtlWords; k += blockDim.x) sm[k] = __ldcg(g + k);
}

__device__ __forceinline__ void ctl_stage_out(AspotCtl* ctl, const uint32_t* sm) {
  uint32_t* g = reinterpret_cast<uint32_t*>(ctl);
  for (int k = threadIdx.x; k < kCtlWords; k += blockDim.x) g[k] = sm[k];
}

__device__ __forceinline__ double theta_next_d(double th) {  // solvers.hpp:32-37
  return th * (sqrt(th * th + 4.0) - th) / 2.0;
}

// Per-point reduction of the sweep partials into B 1, B^T 1 and the scalar
// partials of every functional the reference evaluates at that point.
// One launch per point (k_point_eval).
struct ReduceArgs {
  Slot z;
  const double* rowp; int64_t nstrips;
  const double* colp; int64_t nrowblocks;
  const double* maxp; int64_t nmax;
  double* row_out; double* col_out;
  const double* rt; const double* ct;  // marginals the dual targets (mixed r~, c~)
  double* scratch;                      // [gridDim.x][kNumAcc]
  const int* gate;
  int pfmt;                             // PartialFormat of rowp/colp
  const double* rowshift;               // source row term of the fp32 row offset (log2), may be null
  // mode 1: no sweep; the point differs from a source point only in w, so
  // B = B(src) e^(w - w_src): sums are scaled (source b when *select_b).
  int mode;
  const double* src_row_a; const double* src_col_a; const double* src_w_a; int src_role_a;
  const double* src_row_b; const double* src_col_b; const double* src_w_b; int src_role_b;
  const int* select_b;
  // K1'': when *alt_sel == 1, the partials come from the stash the previous
  // attempt's one-sided pass wrote (same layout); == 2: the sums themselves
  // (direct_row / direct_col) and the max exponent (ctl->bar_maxe)
  const int* alt_sel;
  const double* rowp_alt; const double* colp_alt; const double* maxp_alt;
  const double* direct_row; const double* direct_col;
  // deferred decision: write this launch's block partials to scratch and
  // stop; the next O(n) kernel of the attempt reduces them and decides
  // (decide_pending), so no block waits on a ticket here
  int defer;
};

__device__ __forceinline__ bool is_max_slot(int k) { return k == 1 || k == 2 || k == 11; }
__device__ __forceinline__ bool is_min_slot(int k) { return k == 12 || k == 13; }
__device__ __forceinline__ double acc_init(int k) { return is_max_slot(k) ? -INFINITY : (is_min_slot(k) ? INFINITY : 0.0); }
__device__ __forceinline__ double acc_join(int k, double x, double y) {
  return is_max_slot(k) ? nan_max(x, y) : (is_min_slot(k) ? fmin(x, y) : x + y);
}

// Scaling shortcut guard (fp64 only): B(z + dw e_w) = B(z) e^dw holds
// entry-wise only while no exponent meets the Eigen clamp (kExpLo); sums far
// above the clamp floor on both sides make the clamp's contribution
// negligible. The fp32 sweeps have no clamp: a column flushed to 0 relative
// to its rows' maxima stays flushed after a shift of w, so scaling matches a
// fresh sweep.
constexpr double kScaleSafeFloor = 1e-250;
__device__ __forceinline__ bool scale_safe(const PointScalars& src, double s) {
  const double m = fmin(src.minrow, src.mincol);
  return m >= kScaleSafeFloor && m * (s / src.total) >= kScaleSafeFloor && src.total > 0;
}

__device__ __forceinline__ int greedy_block(const PointScalars& ps, double s) {  // solvers.hpp:58-68
  const double su = ps.score_u, sv = ps.score_v, sw = rho_limit(s, ps.total);
  int block = 0;
  double best = su;
  if (sv > best) { block = 1; best = sv; }
  if (sw > best) block = 2;
  return block;
}

// Scalar finalisation + the decision the reference takes at that point.
__device__ void apply_role(AspotCtl* ctl, int role, const double (&acc)[kNumAcc], double w, bool swept) {
  PointScalars ps;
  ps.total = acc[0]; ps.maxu = acc[1]; ps.maxv = acc[2]; ps.seu = acc[3]; ps.sev = acc[4];
  ps.ur = acc[5]; ps.vc = acc[6]; ps.score_u = acc[7]; ps.score_v = acc[8]; ps.gl1u = acc[9]; ps.gl1v = acc[10];
  ps.maxe = acc[11];
  ps.minrow = acc[12];
  ps.mincol = acc[13];
  // phi (dual.hpp:117-118): B.sum() + eu.sum() + ev.sum() - u.r - v.c - w s
  ps.phi = ((((ps.total + ps.seu) + ps.sev) - ps.ur) - ps.vc) - w * ctl->s;
  ps.err = (ps.gl1u + ps.gl1v) + fabs(ps.total - ctl->s);  // dual.hpp:138-141
  ps.overflow = !(ps.maxe <= kMaxExponent) || !(ps.maxu <= kMaxExponent) || !(ps.maxv <= kMaxExponent) || (w != w);
  ps.pad = 0;
  ctl->ps[role] = ps;
  if (swept) ctl->sweeps += 1;
  switch (role) {
    case R_BAR:
      if (ps.overflow) { ctl->zbar_failed = 1; ctl->g_alive = 0; }
      break;
    case R_GRAVE:
      if (ps.overflow) { ctl->g_alive = 0; break; }
      ctl->block_hat = ctl->block_rule == POTGPU_ROUND_ROBIN ? int(ctl->gk_calls % 3) : greedy_block(ps, ctl->s);
      ctl->g_hat_scaled = ctl->block_hat == 2 && (!ctl->clamp_guard || scale_safe(ps, ctl->s));
      ctl->g_hat_sweep = !ctl->g_hat_scaled;
      break;
    case R_HAT: {
      if (ps.overflow) { ctl->g_alive = 0; break; }
      ctl->phi_hat = ps.phi;
      const int keep = ctl->phi_check <= ps.phi;  // solvers.hpp:342
      ctl->keep_check = keep;
      ctl->phi_best = fmin(ctl->phi_check, ps.phi);
      const PointScalars& pb = keep ? ctl->ps[R_CHECK] : ps;
      ctl->block_check = ctl->block_rule == POTGPU_ROUND_ROBIN ? int((ctl->gk_calls + 1) % 3) : greedy_block(pb, ctl->s);
      ctl->g_new_scaled = ctl->block_check == 2 && (!ctl->clamp_guard || scale_safe(pb, ctl->s));
      // one side of B(z_check') is an O(n) rescale of z_hat's; the other one
      // sweep with the row shifts z_hat's sweep left in rowp
      ctl->g_new_one = ctl->one_sided_ok && !keep && !ctl->g_new_scaled && ctl->block_check != 2;
      ctl->g_new_sweep = !ctl->g_new_scaled && !ctl->g_new_one;
      ctl->g_new_eval = ctl->g_new_sweep | ctl->g_new_one;
      break;
    }
    case R_NEW:
      if (ps.overflow) { ctl->g_alive = 0; break; }
      ctl->attempt_ok = 1;
      break;
    case R_CHECK:  // initial evaluation at z_check = 0 (solvers.hpp:305)
      if (ps.overflow) { ctl->fatal = POTGPU_OVERFLOW; ctl->g_active = 0; ctl->g_new = 0; ctl->g_bar_sweep = 0; ctl->g_alive = 0; }
      break;
    default:
      break;
  }
}

constexpr int kEvalThreads = 128;
// threads per index of k_point_eval ($POTGPU_EVAL_TPI: 1, 2, 4, 8; default:
// 4, or 8 when an index's partial list would not fit the register path of
// 4 threads (more than 4 kGroupRegs strips: C4, 128 strips). Measured: C3
// (32 strips) 2693 / 2624 it/s with 4 / 8, C4 214.9 / 216.8 it/s.
constexpr int kGroupRegsDecl = 16;
inline int eval_tpi(int64_t nstrips = 0) {
  static const int v = [] {
    const char* e = std::getenv("POTGPU_EVAL_TPI");
    const int k = e ? std::atoi(e) : 0;
    return (k == 1 || k == 2 || k == 4 || k == 8) ? k : 0;
  }();
  if (v) return v;
  return nstrips > 4 * kGroupRegsDecl ? 8 : 4;
}

// Per-index terms of every functional the reference evaluates at a point
// (dual.hpp:112-141, solvers.hpp:49-52): B 1 = rb, B^T 1 = cb at z = (u, v, w).
template <int N>
__device__ __forceinline__ void add_index_terms(double (&acc)[N], double rb, double cb, double ui, double vi,
                                                double rti, double cti) {
  static_assert(N >= kNumAcc, "accumulator array too short");
  const double eu = eexp(ui), ev = eexp(vi);
  acc[0] += rb;
  acc[1] = nan_max(acc[1], ui);
  acc[2] = nan_max(acc[2], vi);
  acc[3] += eu;
  acc[4] += ev;
  acc[5] += ui * rti;
  acc[6] += vi * cti;
  const double rowf = rb + eu, colf = cb + ev;
  acc[7] += rho_limit(rti, rowf);
  acc[8] += rho_limit(cti, colf);
  acc[9] += fabs(rowf - rti);
  acc[10] += fabs(colf - cti);
  acc[12] = fmin(acc[12], rb);
  acc[13] = fmin(acc[13], cb);
}

// Grid cap of k_point_eval: $POTGPU_EVAL_BLOCKS_PER_SM (default 4) x SMs
// (and at most 2 kVecThreads blocks, engine.cuh). Measured with deferred
// decisions, C3 back-to-back: 2 / 3 / 4 per SM 2663 / 2653 / 2691 it/s.
inline int64_t eval_blocks_cap(int num_sms) {
  static const int v = [] {
    const char* e = std::getenv("POTGPU_EVAL_BLOCKS_PER_SM");
    return e ? std::atoi(e) : 0;
  }();
  return int64_t(v > 0 ? v : 4) * num_sms;
}

// Sum of the partials p[base .. base + cnt) of one index, split over the
// kTPI threads of a group (thread q takes s = q, q + kTPI, ...). fp32
// (sum, log2 scale) partials are combined relative to their max with MUFU
// ex2 and turned into fp64 once: S 2^(M + offset).
// Lists of up to kTPI * kGroupRegs partials are loaded into registers
// before the max / sum passes (one L2 round trip instead of one per
// partial); longer lists stream. Same M, per-thread order and shuffle tree
// either way -> identical bits.
constexpr int kGroupRegs = kGroupRegsDecl;

template <int kTPI>
__device__ __forceinline__ double group_partial_sum(const double* p, int64_t base, int64_t cnt, int fmt, double offset,
                                                    int q) {
  const bool regs = cnt <= int64_t(kTPI) * kGroupRegs;
  if (fmt == PF_F64) {
    double s = 0.0;
    if (regs) {
      double x[kGroupRegs];
#pragma unroll
      for (int r = 0; r < kGroupRegs; ++r) {
        const int64_t k = q + int64_t(r) * kTPI;
        x[r] = k < cnt ? p[base + k] : 0.0;
      }
#pragma unroll
      for (int r = 0; r < kGroupRegs; ++r)
        if (q + int64_t(r) * kTPI < cnt) s += x[r];
    } else {
      for (int64_t k = q; k < cnt; k += kTPI) s += p[base + k];
    }
#pragma unroll
    for (int o = kTPI / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
  }
  const float2* f = reinterpret_cast<const float2*>(p) + base;
  float M = -INFINITY, S = 0.f;
  if (regs) {
    float2 x[kGroupRegs];
#pragma unroll
    for (int r = 0; r < kGroupRegs; ++r) {
      const int64_t k = q + int64_t(r) * kTPI;
      x[r] = k < cnt ? f[k] : make_float2(0.f, 0.f);
    }
#pragma unroll
    for (int r = 0; r < kGroupRegs; ++r)
      if (x[r].x != 0.f) M = fmaxf(M, x[r].y);
#pragma unroll
    for (int o = kTPI / 2; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (M != -INFINITY)
#pragma unroll
      for (int r = 0; r < kGroupRegs; ++r)
        if (x[r].x != 0.f) S += x[r].x * ex2f(x[r].y - M);
  } else {
    for (int64_t k = q; k < cnt; k += kTPI) {
      const float2 x = f[k];
      if (x.x != 0.f) M = fmaxf(M, x.y);
    }
#pragma unroll
    for (int o = kTPI / 2; o > 0; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
    if (M != -INFINITY)
      for (int64_t k = q; k < cnt; k += kTPI) {
        const float2 x = f[k];
        if (x.x != 0.f) S += x.x * ex2f(x.y - M);
      }
  }
#pragma unroll
  for (int o = kTPI / 2; o > 0; o >>= 1) S += __shfl_xor_sync(0xffffffffu, S, o);
  return M == -INFINITY ? 0.0 : double(S) * exp2(double(M) + offset);
}

// One kernel per evaluated point: a group of kTPI threads per index i
// combines the sweep's strip / row-block partials (contiguous per index)
// into (B 1)_i and (B^T 1)_i and forms the per-element terms of every
// functional the reference evaluates there; blocks reduce them to
// fixed-order partials, and the last block to finish (atomic ticket)
// reduces all partials in a fixed order and takes the decision
// (apply_role). Deterministic, one launch.
template <int kTPI>
__global__ void __launch_bounds__(kEvalThreads) k_point_eval(AspotCtl* ctl, int role, ReduceArgs a, unsigned* ticket) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  const int64_t n = a.z.n;
  double acc[kNumAcc];
#pragma unroll
  for (int k = 0; k < kNumAcc; ++k) acc[k] = acc_init(k);
  const double* u = a.z.u();
  const double* v = a.z.v();
  const double w = *a.z.w();
  const int q = threadIdx.x % kTPI;
  const int64_t per_block = kEvalThreads / kTPI;
  const int64_t span = int64_t(gridDim.x) * per_block;
  const bool useb = a.mode == 1 && a.select_b && *a.select_b;
  const double* srow = useb ? a.src_row_b : a.src_row_a;
  const double* scol = useb ? a.src_col_b : a.src_col_a;
  const double dw = a.mode == 1 ? w - *(useb ? a.src_w_b : a.src_w_a) : 0.0;
  const double fs = a.mode == 1 ? exp(dw) : 1.0;
  const int alt_mode = a.alt_sel ? *a.alt_sel : 0;
  const bool alt = alt_mode == 1, direct = alt_mode == 2;
  const double* rowp = alt ? a.rowp_alt : a.rowp;
  const double* colp = alt ? a.colp_alt : a.colp;
  const double* maxp = alt ? a.maxp_alt : a.maxp;
  // all threads iterate the same number of times (the shuffles need the full warp)
  for (int64_t i0 = int64_t(blockIdx.x) * per_block; i0 < n; i0 += span) {
    const int64_t i = i0 + threadIdx.x / kTPI;
    const bool live = i < n;
    const int64_t ii = live ? i : n - 1;
    const double ui = u[ii], vi = v[ii];
    double rb, cb;
    if (direct) {
      rb = a.direct_row[ii];
      cb = a.direct_col[ii];
    } else if (a.mode == 0) {
      double off = (ui + w) * kLog2e;
      if (a.rowshift) off = off + a.rowshift[ii];
      rb = group_partial_sum<kTPI>(rowp, ii * a.nstrips, a.nstrips, a.pfmt, off, q);
      cb = group_partial_sum<kTPI>(colp, ii * a.nrowblocks, a.nrowblocks, a.pfmt, 0.0, q);
    } else {
      rb = srow[ii] * fs;
      cb = scol[ii] * fs;
    }
    if (!live || q != 0) continue;
    a.row_out[i] = rb;
    a.col_out[i] = cb;
    add_index_terms(acc, rb, cb, ui, vi, a.rt[i], a.ct[i]);
  }
  if (direct) {
    if (blockIdx.x == 0 && threadIdx.x == 0) acc[11] = __ldcg(&ctl->bar_maxe);
  } else if (a.mode == 0) {
    for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < a.nmax; k += int64_t(gridDim.x) * blockDim.x)
      acc[11] = nan_max(acc[11], maxp[k]);
  }
  // block reduction: warp shuffles, then the kEvalThreads / 32 warp results
  __shared__ double sh[kNumAcc][kEvalThreads / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  auto block_reduce = [&]() {
#pragma unroll
    for (int k = 0; k < kNumAcc; ++k) {
      double x = acc[k];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x = acc_join(k, x, __shfl_xor_sync(0xffffffffu, x, o));
      if (lane == 0) sh[k][wid] = x;
    }
    __syncthreads();
    if (threadIdx.x < kNumAcc) {
      double x = sh[threadIdx.x][0];
      for (int w2 = 1; w2 < kEvalThreads / 32; ++w2) x = acc_join(threadIdx.x, x, sh[threadIdx.x][w2]);
      sh[threadIdx.x][0] = x;
    }
    __syncthreads();
  };
  block_reduce();
  if (threadIdx.x < kNumAcc) a.scratch[blockIdx.x * (kNumAcc) + threadIdx.x] = sh[threadIdx.x][0];
  if (a.defer) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ __align__(16) uint32_t ctl_sm[kCtlWords];
  ctl_stage_in(ctl_sm, ctl);
  const double* sc = a.scratch;
#pragma unroll
  for (int k = 0; k < kNumAcc; ++k) acc[k] = acc_init(k);
  for (int b = threadIdx.x; b < int(gridDim.x); b += blockDim.x)
#pragma unroll
    for (int k = 0; k < kNumAcc; ++k) acc[k] = acc_join(k, acc[k], __ldcg(sc + b * (kNumAcc) + k));
  __syncthreads();
  block_reduce();
  if (threadIdx.x == 0) {
    AspotCtl* sctl = reinterpret_cast<AspotCtl*>(ctl_sm);
    double tot[kNumAcc];
#pragma unroll
    for (int k = 0; k < kNumAcc; ++k) tot[k] = sh[k][0];
    *ticket = 0u;  // ready for the next launch
    if (a.mode == 1) tot[11] = sctl->ps[useb ? a.src_role_b : a.src_role_a].maxe + dw;  // max exponent shifts by dw
    apply_role(sctl, role, tot, w, a.mode == 0);
  }
  __syncthreads();
  ctl_stage_out(ctl, ctl_sm);
}

// ---------------------------------------------------------------------------
// Deferred decisions. The per-point evaluations of an attempt (launch_eval
// with defer = 1) only write their block partials; the O(n) kernel that
// consumes the point (k_zgrave, k_gk_update, k_commit) reduces them in
// every block in one fixed order (reduce_partials_wide), and takes the reference's decision at that point (apply_role) on a
// shared-memory copy of the control block. All blocks see identical inputs,
// so all copies agree; the block that finishes last (ticket) writes its copy
// back. No block of an evaluation waits on a ticket, and the decision costs
// no serial tail.
struct Pending {
  const double* eval_part; int eval_nb;  // k_point_eval block partials [eval_nb][kNumAcc]
  double* gk_part; int gk_nb;            // k_gk_update partials of a w-block point [gridDim.x][kNumAcc]
  int* flag;                             // non-finite block update seen by some block (solvers.hpp:83-87)
  unsigned* ticket;
};

// Fixed-order reduction of [nb][kNumAcc] partials over all threads of the
// calling block (blockDim.x a multiple of 32): thread t takes rows t and
// t + blockDim.x (all loads issued before the first join; nb <= 2
// blockDim.x), then warp trees and warps in order. Result in sh[k][0].
__device__ void reduce_partials_wide(const double* sc, int nb, double (&sh)[kNumAcc][32]) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
  double x0[kNumAcc], x1[kNumAcc];
  const int b0 = t, b1 = t + blockDim.x;
#pragma unroll
  for (int k = 0; k < kNumAcc; ++k) {
    x0[k] = b0 < nb ? __ldg(sc + b0 * kNumAcc + k) : acc_init(k);  // written by an earlier kernel
    x1[k] = b1 < nb ? __ldg(sc + b1 * kNumAcc + k) : acc_init(k);
  }
#pragma unroll
  for (int k = 0; k < kNumAcc; ++k) {
    double x = acc_join(k, x0[k], x1[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = acc_join(k, x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sh[k][wid] = x;
  }
  __syncthreads();
  if (t < kNumAcc) {
    double x = sh[t][0];
    for (int w2 = 1; w2 < nw; ++w2) x = acc_join(t, x, sh[t][w2]);
    sh[t][0] = x;
  }
  __syncthreads();
}

__device__ void decide_pending(AspotCtl* c, int role, const double* sc, int nb, double w, bool swept) {
  __shared__ double sh[kNumAcc][32];
  reduce_partials_wide(sc, nb, sh);
  if (threadIdx.x == 0) {
    double tot[kNumAcc];
#pragma unroll
    for (int k = 0; k < kNumAcc; ++k) tot[k] = sh[k][0];
    apply_role(c, role, tot, w, swept);
  }
  __syncthreads();
}

// Block tree of kNumAcc accumulators over blockDim.x (a multiple of 32,
// at most 1024) threads; result in sh[k][0].
__device__ void block_reduce_acc(double (&acc)[kNumAcc], double (&sh)[kNumAcc][32]) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int k = 0; k < kNumAcc; ++k) {
    double x = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = acc_join(k, x, __shfl_xor_sync(0xffffffffu, x, o));
    if (lane == 0) sh[k][wid] = x;
  }
  __syncthreads();
  if (t < kNumAcc) {
    double x = sh[t][0];
    for (int w2 = 1; w2 < nw; ++w2) x = acc_join(t, x, sh[t][w2]);
    sh[t][0] = x;
  }
  __syncthreads();
}

// End of a consuming kernel: the last block (ticket) folds in the
// non-finite flag, runs `last_fn` on its copy and writes the copy back.
// Every block staged its copy in (and used it) before taking its ticket, so
// the write-back cannot overtake a read; the only cross-block data is the
// flag, whose writer fences (k_gk_update). Everything else a consumer writes
// is read by later kernels only. (Measured: dropping the per-block fence
// took k_zgrave 11.5 -> 7.9 us, C3 2594 -> 2664 it/s back-to-back.)
template <class F>
__device__ void ctl_finish(AspotCtl* ctl, uint32_t* ctl_sm, const Pending& pd, F last_fn) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(pd.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x == 0) {
    AspotCtl* c = reinterpret_cast<AspotCtl*>(ctl_sm);
    *pd.ticket = 0u;
    if (pd.flag && __ldcg(pd.flag)) {  // solvers.hpp:83-87: non-finite update -> Overflow
      c->g_alive = 0;
      c->g_hat_sweep = c->g_hat_scaled = c->g_new_sweep = c->g_new_scaled = 0;
      c->g_new_one = c->g_new_eval = 0;
      *pd.flag = 0;
    }
    last_fn(c);
  }
  __syncthreads();
  ctl_stage_out(ctl, ctl_sm);
}

__device__ __forceinline__ AspotCtl* ctl_stage(uint32_t* ctl_sm, const AspotCtl* ctl) {
  ctl_stage_in(ctl_sm, ctl);
  __syncthreads();
  return reinterpret_cast<AspotCtl*>(ctl_sm);
}

// z_next = z_bar - step grad ; z_grave = z_bar + theta (z_next - z)
// (solvers.hpp:337-339). On a new iteration the decision at z_bar (range
// check) is taken first and the gradient of z_bar formed (dual.hpp:129-131)
// and kept for the retries (halving keeps z_bar).
__global__ void k_zgrave(AspotCtl* ctl, Slot zb, Slot z, Slot g, Slot zg, const double* rowb, const double* colb,
                         const double* rt, const double* ct, Pending pd) {
  pdl_wait();
  __shared__ __align__(16) uint32_t ctl_sm[kCtlWords];
  AspotCtl* c = ctl_stage(ctl_sm, ctl);
  const int fresh = c->g_new;
  if (!fresh && !c->g_alive) return;  // uniform: nothing to decide or update
  if (fresh) decide_pending(c, R_BAR, pd.eval_part, pd.eval_nb, *zb.w(), !c->g_bar_stash);
  if (c->g_alive) {
    const int64_t n = zb.n;
    const double step = c->step, th = c->theta;
    for (int64_t k = blockIdx.x * blockDim.x + threadIdx.x; k < 2 * n + 1; k += int64_t(gridDim.x) * blockDim.x) {
      double gk;
      if (fresh) {
        if (k < n) gk = (rowb[k] + eexp(zb.base[k])) - rt[k];
        else if (k < 2 * n) gk = (colb[k - n] + eexp(zb.base[k])) - ct[k - n];
        else gk = c->ps[R_BAR].total - c->s;
        g.base[k] = gk;
      } else {
        gk = g.base[k];
      }
      const double zn = zb.base[k] - step * gk;
      zg.base[k] = zb.base[k] + th * (zn - z.base[k]);
    }
  }
  ctl_finish(ctl, ctl_sm, pd, [](AspotCtl*) {});
}

// Exact block minimisation (solvers.hpp:71-88) of src with the B sums of
// src; dst = src with the chosen block replaced. `which` selects the source:
// 0 = (src_a, rows_a, ps_a) [z_grave], 1 = z_best (z_check if keep_check
// else z_hat). First the pending decision at the source point (which = 0:
// z_grave's Greenkhorn block; which = 1: z_hat's phi, z_best and its block).
// When the new point is to be scaled rather than swept (block w: B scales
// by e^dw), its sums (dst_row, dst_col) and the block partials of its
// functionals are formed here (pd.gk_part), for the next kernel to decide on.
// K1'' (which = 1, one-sided z_check'): also the next iteration's z_bar' =
// (1 - theta') z_check' + theta' z_best (k_commit's arithmetic, same bits)
// and the side of B(z_bar') that only rescales, for the fused pass.
struct BarStash {
  Slot zbn;
  double* row;  // B(z_bar') 1 (block u)
  double* col;  // B(z_bar')^T 1 (block v)
};
__global__ void k_gk_update(AspotCtl* ctl, int which, Slot src_a, const double* row_a, const double* col_a, int role_a,
                            Slot src_b, const double* row_b, const double* col_b, int role_b, Slot dst,
                            const double* rt, const double* ct, double* dst_row, double* dst_col, Pending pd,
                            BarStash bs) {
  pdl_wait();
  __shared__ __align__(16) uint32_t ctl_sm[kCtlWords];
  AspotCtl* c = ctl_stage(ctl_sm, ctl);
  if (which == 0) {
    if (!c->g_alive) return;  // uniform: z_grave was not evaluated
    decide_pending(c, R_GRAVE, pd.eval_part, pd.eval_nb, *src_a.w(), true);
  } else {
    const bool swept = c->g_hat_sweep, scaled = c->g_hat_scaled;
    if (!swept && !scaled) return;  // uniform: z_hat was not evaluated
    decide_pending(c, R_HAT, swept ? pd.eval_part : pd.gk_part, swept ? pd.eval_nb : pd.gk_nb, *src_a.w(), swept);
  }
  if (c->g_alive) {
    int block;
    Slot src;
    const double *rowb, *colb;
    int role;
    if (which == 0) {
      block = c->block_hat; src = src_a; rowb = row_a; colb = col_a; role = role_a;
    } else {
      block = c->block_check;
      const bool keep = c->keep_check;
      src = keep ? src_b : src_a; rowb = keep ? row_b : row_a; colb = keep ? col_b : col_a; role = keep ? role_b : role_a;
    }
    const int64_t n = src.n;
    bool finite = true;
    const double th = theta_next_d(c->theta), om = 1.0 - th;
    const bool k1 = which == 1 && c->g_new_one && c->fuse_ok && bs.zbn.base;
    // block w: B(z_bar') = B(z_best) e^(w' - w_best), z_bar's sums without any pass
    const bool k1w = which == 1 && c->g_new_scaled && c->fuse_ok && bs.zbn.base;
    double fbar = 0.0;
    if (k1w) {
      const double ws = *src.w();
      const double wd = ws + (log(c->s) - log(c->ps[role].total));  // = dst.w
      const double za = om * wd;
      const double zb2 = th * ws;
      const double dwb = (za + zb2) - ws;  // k_commit's z_bar w
      fbar = exp(dwb);
      if (threadIdx.x == 0) c->bar_maxe = c->ps[role].maxe + dwb;  // every block's copy agrees
    }
    for (int64_t k = blockIdx.x * blockDim.x + threadIdx.x; k < 2 * n + 1; k += int64_t(gridDim.x) * blockDim.x) {
      double x = src.base[k];
      if (k < n) {
        if (block == 0) x = x + (log(rt[k]) - log(rowb[k] + eexp(x)));
      } else if (k < 2 * n) {
        if (block == 1) x = x + (log(ct[k - n]) - log(colb[k - n] + eexp(x)));
      } else {
        if (block == 2) x = x + (log(c->s) - log(c->ps[role].total));
      }
      dst.base[k] = x;
      finite = finite && isfinite(x);
      if (which == 1 && c->g_new_one) {  // the side of z_check' that only rescales: B' = B e^(x' - x)
        if (k < n && block == 0) dst_row[k] = rowb[k] * exp(x - src.base[k]);
        else if (k >= n && k < 2 * n && block == 1) dst_col[k - n] = colb[k - n] * exp(x - src.base[k]);
      }
      if (k1w) {
        if (k < n) bs.row[k] = rowb[k] * fbar;
        else if (k < 2 * n) bs.col[k - n] = colb[k - n] * fbar;
      }
      if (k1) {  // z_bar' and its rescaled side (k_commit: a = om z_check', b = th z_best, z_bar = a + b)
        const double za = om * x;
        const double zb2 = th * src.base[k];
        const double zbar = za + zb2;
        bs.zbn.base[k] = zbar;
        if (k < n && block == 0) bs.row[k] = rowb[k] * exp(zbar - src.base[k]);
        else if (k >= n && k < 2 * n && block == 1) bs.col[k - n] = colb[k - n] * exp(zbar - src.base[k]);
      }
    }
    if (!finite) {
      *pd.flag = 1;
      __threadfence();  // visible to the deciding block before this block's ticket
    }
    const bool scaled = which == 0 ? c->g_hat_scaled : c->g_new_scaled;
    if (scaled) {  // block w: B(dst) = B(src) e^dw, the point's sums and functionals without a sweep
      const double ws = *src.w();
      const double wd = ws + (log(c->s) - log(c->ps[role].total));  // = dst.w (same arithmetic as the update)
      const double dw = wd - ws;
      const double fs = exp(dw);
      double acc[kNumAcc];
#pragma unroll
      for (int k = 0; k < kNumAcc; ++k) acc[k] = acc_init(k);
      const double* u = src.u();
      const double* v = src.v();
      for (int64_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
        const double rb = rowb[i] * fs, cb = colb[i] * fs;
        dst_row[i] = rb;
        dst_col[i] = cb;
        add_index_terms(acc, rb, cb, u[i], v[i], rt[i], ct[i]);
      }
      acc[11] = c->ps[role].maxe + dw;  // the max exponent shifts by dw
      __shared__ double sh[kNumAcc][32];
      block_reduce_acc(acc, sh);
      if (threadIdx.x < kNumAcc) pd.gk_part[blockIdx.x * kNumAcc + threadIdx.x] = sh[threadIdx.x][0];
    }
  }
  ctl_finish(ctl, ctl_sm, pd, [](AspotCtl*) {});
}

// Commit of an accepted attempt: z <- z_best, z_check <- z_check', sums of
// z_check <- sums of z_check' (solvers.hpp:357-360). Element-parallel.
__device__ void append_trace(AspotCtl* ctl, TraceDev* trace, int64_t t, double err, double phi) {
  if (trace && ctl->trace_len < ctl->trace_cap) {  // null: a cluster rank that only counts
    TraceDev& r = trace[ctl->trace_len];
    r.t = t; r.error = err; r.phi = phi;
    r.rounded_cost = __longlong_as_double(0x7ff8000000000000ULL);
    r.elapsed_s = double(globaltimer_ns() - ctl->t0_ns) * 1e-9;
  }
  ctl->trace_len += 1;
}

__device__ void reset_point_gates(AspotCtl* ctl) {
  ctl->g_hat_sweep = ctl->g_hat_scaled = ctl->g_new_sweep = ctl->g_new_scaled = 0;
  ctl->g_new_one = ctl->g_new_eval = 0;
  ctl->g_bar_sweep = 0;
}

__device__ void begin_iteration(AspotCtl* ctl) {
  reset_point_gates(ctl);
  ctl->halvings = 0;
  ctl->step = ctl->gamma / (ctl->step_denom * ctl->theta);  // solvers.hpp:328
  ctl->g_new = 1;
  ctl->g_bar_sweep = !ctl->g_bar_stash;
  ctl->g_alive = 1;
  ctl->attempt_ok = 0;
  ctl->zbar_failed = 0;
}

__device__ void finish(AspotCtl* ctl, int status) {
  ctl->status = status;
  ctl->g_active = 0;
  ctl->g_new = 0;
  ctl->g_alive = 0;
  reset_point_gates(ctl);  // attempt graphs still queued after the stop must do nothing
  ctl->loop_end_ns = globaltimer_ns();
}

// Loop-head test of the reference (solvers.hpp:323-327), plus the session
// pause point (no reference counterpart: lets a caller run k iterations).
__device__ void loop_head(AspotCtl* ctl) {
  if (!(ctl->error > ctl->eps_tilde)) { finish(ctl, POTGPU_CONVERGED); return; }
  if (ctl->t >= ctl->max_iterations) { finish(ctl, POTGPU_MAX_ITERATIONS_EXCEEDED); return; }
  if (ctl->t >= ctl->pause_at) {
    ctl->paused = 1;
    ctl->g_active = 0;
    ctl->g_new = 0;
    ctl->g_alive = 0;
    reset_point_gates(ctl);
    ctl->loop_end_ns = globaltimer_ns();
    return;
  }
  begin_iteration(ctl);
}

__device__ __forceinline__ void resume(AspotCtl* ctl, int64_t pause_at, int64_t budget) {
  ctl->pause_at = pause_at;
  ctl->loop_budget = budget;
  if (!ctl->paused) return;
  ctl->paused = 0;
  ctl->g_active = 1;
  loop_head(ctl);
}

__global__ void k_resume(AspotCtl* ctl, int64_t pause_at, int64_t budget) {
  pdl_wait();
  resume(ctl, pause_at, budget);
}

// Resume as the first node of a captured "resume + attempt" graph: the
// arguments come from pinned host memory written before the launch (read
// through UVA), so a run starts with ONE host launch and the GPU does not
// idle between a separate resume kernel and the graph.
struct ResumeArgs {
  int64_t pause_at, budget;
};
__global__ void k_resume_pinned(AspotCtl* ctl, const ResumeArgs* args) {
  pdl_wait();
  const volatile ResumeArgs* va = args;
  resume(ctl, va->pause_at, va->budget);
}

__device__ void commit_state(AspotCtl* ctl, TraceDev* trace, IterLogDev* lg) {
  if (!ctl->g_active) return;
  ctl->attempts += 1;
  if (!ctl->attempt_ok) {
    // halving loop (solvers.hpp:334-356): z_bar/grad failures repeat on every
    // retry, so they exhaust the 61 tries immediately.
    if (ctl->zbar_failed || ctl->halvings >= 60) { finish(ctl, POTGPU_STEP_SIZE_UNDERFLOW); return; }
    reset_point_gates(ctl);
    ctl->halvings += 1;
    ctl->step *= 0.5;
    ctl->g_new = 0;
    ctl->g_alive = 1;
    ctl->attempt_ok = 0;
    return;
  }
  ctl->ps[R_CHECK] = ctl->ps[R_NEW];
  ctl->gk_calls += 2;
  ctl->error = ctl->ps[R_NEW].err;
  ctl->phi_check = ctl->ps[R_NEW].phi;
  ctl->theta = theta_next_d(ctl->theta);
  ctl->t += 1;
  if (lg && ctl->log_len < ctl->log_cap) {
    IterLogDev& e = lg[ctl->log_len];
    e.t = ctl->t; e.halvings = ctl->halvings; e.block_hat = ctl->block_hat; e.zbest_is_check = ctl->keep_check;
    e.block_check = ctl->block_check; e.error = ctl->error; e.phi_check = ctl->phi_check; e.phi_hat = ctl->phi_hat;
    e.theta = ctl->theta;
  }
  ctl->log_len += 1;
  if (ctl->t % ctl->log_every == 0 || !(ctl->error > ctl->eps_tilde)) {  // solvers.hpp:309
    append_trace(ctl, trace, ctl->t, ctl->error, ctl->phi_check);
    // the record's rounded cost (solvers.hpp:314-315): the attempt graph's
    // device-rounding tail runs when this is set (and clears it)
    ctl->g_record = ctl->record_rounded_cost && ctl->trace_len <= ctl->trace_cap;
  }
  loop_head(ctl);
}

// End of a step attempt, one launch: on success z <- z_best, z_check <-
// z_check', their sums, and already the next iteration's
// z_bar = (1 - theta') z_check + theta' z (solvers.hpp:336 with theta' =
// theta_next(theta), DualPoint ops dual.hpp:33-43); then the last block to finish takes the scalar
// decisions of commit_state (halving / record / loop head).
// In the device loop (a CUDA-graph WHILE node around the attempt, `loop`
// = its condition handle) the deciding block also tells the graph whether
// to run another attempt: while the solve is active and the launch's
// attempt budget lasts.
__global__ void k_commit(AspotCtl* ctl, Slot z, Slot zc, Slot zh, Slot zn, Slot zb, double* rowc, double* colc,
                         const double* rown, const double* coln, TraceDev* trace, IterLogDev* lg, Pending pd,
                         cudaGraphConditionalHandle loop, int in_loop, int* stash_bad) {
  pdl_wait();
  __shared__ __align__(16) uint32_t ctl_sm[kCtlWords];
  AspotCtl* c = ctl_stage(ctl_sm, ctl);
  if (!c->g_active) {  // uniform over the grid
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (in_loop) cudaGraphSetConditional(loop, 0u);
      if (stash_bad) *stash_bad = 0;
    }
    return;
  }
  const bool swept = c->g_new_sweep || c->g_new_one, scaled = c->g_new_scaled;
  if (swept || scaled)  // decision at z_check' (solvers.hpp:345-352)
    decide_pending(c, R_NEW, swept ? pd.eval_part : pd.gk_part, swept ? pd.eval_nb : pd.gk_nb, *zn.w(), swept);
  if (c->attempt_ok) {
    const bool keep = c->keep_check;
    const double th = theta_next_d(c->theta), om = 1.0 - th;
    const int64_t n = z.n;
    for (int64_t k = blockIdx.x * blockDim.x + threadIdx.x; k < 2 * n + 1; k += int64_t(gridDim.x) * blockDim.x) {
      const double zbst = keep ? zc.base[k] : zh.base[k];
      const double zcn = zn.base[k];
      z.base[k] = zbst;
      zc.base[k] = zcn;
      const double a = om * zcn;
      const double b = th * zbst;
      zb.base[k] = a + b;
      if (k < n) {
        rowc[k] = rown[k];
        colc[k] = coln[k];
      }
    }
  }
  ctl_finish(ctl, ctl_sm, pd, [&](AspotCtl* cc) {
    // K1'': the fused pass of this attempt's z_check' left the next z_bar's partials
    const int bad = stash_bad ? __ldcg(stash_bad) : 1;
    if (stash_bad) *stash_bad = 0;
    cc->g_bar_stash = !(cc->attempt_ok && cc->fuse_ok) ? 0 : (cc->g_new_one && !bad) ? 1 : cc->g_new_scaled ? 2 : 0;
    commit_state(cc, trace, lg);
    if (in_loop) {
      cc->loop_budget -= 1;
      cudaGraphSetConditional(loop, (cc->g_active && cc->loop_budget > 0) ? 1u : 0u);
    }
  });
}

// Initial state after the first phi/grad evaluation at z_check = 0.
__global__ void k_init_state(AspotCtl* ctl, TraceDev* trace) {
  if (ctl->fatal) return;
  ctl->error = ctl->ps[R_CHECK].err;
  ctl->phi_check = ctl->ps[R_CHECK].phi;
  ctl->g_active = 1;
  append_trace(ctl, trace, 0, ctl->error, ctl->phi_check);  // record(0) (solvers.hpp:320)
  loop_head(ctl);
}

__global__ void k_stamp_t0(AspotCtl* ctl) { ctl->t0_ns = globaltimer_ns(); }

}  // namespace potgpu
