// engine.cuh — host-side engine: device problem, workspaces, sweep dispatch.
#pragma once

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <limits>
#include <memory>

#include "aspot_kernels.cuh"
#include "rounding.cuh"
#include "shard.cuh"
#include "sweep.cuh"
#include "sweep_tc.cuh"

namespace potgpu {

// Neumaier sum on the host: the same accumulator as the oracle, so setup
// scalars (masses, gamma, eps~, mixing weight, step denominator) are bitwise
// those of the CPU reference restatement.
inline double ksum(const double* x, int64_t n) {
  double s = 0.0, c = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double t = s + x[i];
    if (std::fabs(s) >= std::fabs(x[i])) c += (s - t) + x[i]; else c += (x[i] - t) + s;
    s = t;
  }
  return s + c;
}

using HostClock = std::chrono::steady_clock;
inline double secs(HostClock::time_point a) { return std::chrono::duration<double>(HostClock::now() - a).count(); }

// $POTGPU_TRACE_SETUP=1: host wall time of the setup / output phases on
// stderr (after a stream sync), for the e2e breakdown.
struct PhaseTimer {
  bool on;
  cudaStream_t st;
  HostClock::time_point t;
  explicit PhaseTimer(cudaStream_t s) : on(std::getenv("POTGPU_TRACE_SETUP") != nullptr), st(s), t(HostClock::now()) {}
  void mark(const char* what) {
    if (!on) return;
    cudaStreamSynchronize(st);
    std::fprintf(stderr, "[potgpu] %-24s %8.3f ms\n", what, secs(t) * 1e3);
    t = HostClock::now();
  }
};

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  Comm comm;  // row sharding (potgpu_comm_init / potgpu_comm_init_local)
};

// Device-resident problem: one of three cost representations.
struct DevProblem {
  int64_t n = 0;
  int dtype = POTGPU_F64;
  int kind = POTGPU_COST_DENSE;
  int64_t ld = 0;          // padded row pitch (elements), multiple of kStripCols
  DevBuf<double> C64;      // fp64 dense C (n x ld), 0-padded
  DevBuf<double> L64;      // fp64 dense logK = -C/gamma (n x ld), -inf padded
  double L_gamma = -1.0;   // gamma L64 was built for
  DevBuf<float> C32;       // fp32 dense C (n x ld), 0-padded
  DevBuf<float4> X4, Y4;   // fp32 points
  DevBuf<float4> XS4, YS4; // points pre-scaled by sqrt(log2 e * scale / gamma) for the fp32 sweeps
  DevBuf<float4> XD4;      // 2 x' (expanded-norm sweep, SrcPointsDotF32)
  DevBuf<double> xshift, yshift;  // -|x'_i|^2, -|y'_j|^2 (fp64, log2 units)
  double XS_gamma = -1.0;
  bool dot_form() const { return kind == POTGPU_COST_SQEUCLIDEAN && dtype == POTGPU_F32; }
  const double* rowshift() const { return dot_form() ? xshift.p : nullptr; }
  double cost_scale = 1.0;
  double cmax = 0.0;
  std::vector<double> r, c;  // host copies (original marginals)
  double s = 0.0;
};

// The tensor-core points sweep (sweep_tc.cuh), opt-in with $POTGPU_TC=1.
// Measured on B200 at C3: 0.131 ms per sweep against 0.108
// for sweep_pts2_f32 — reading S back from TMEM (32x32b loads) is paced at
// about the MUFU rate, so the two do not overlap enough.
inline bool tc_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("POTGPU_TC");
    return e && e[0] == '1';
  }();
  return on;
}

// Carried shifts for the fp32 points sweep (sweep.cuh, sweep_tc.cuh):
// $POTGPU_CARRY=1, or implied by $POTGPU_TC=1. Off by default: on the CUDA-
// core sweep they measured neutral (C3 0.1106 vs 0.1078 ms per sweep; the
// per-row max/CREDUX chain was not the binding limit).
inline bool carry_supported(const DevProblem& P) {
  static const bool on = [] {
    const char* e = std::getenv("POTGPU_CARRY");
    return (e && e[0] == '1') || tc_enabled();
  }();
  return on && P.dot_form() && pts_pairs() == 2;
}

struct ShardGrid {
  int64_t lo = 0, hi = 0;  // rows [lo, hi)
  int index = 0;           // global shard index
  SweepGrid g{};
};

struct Workspace {
  int64_t n = 0;
  SweepGrid g{};
  std::vector<ShardGrid> shards;  // this process's row shards (sharded contexts only)
  int nshards = 1;                // all shards of the job
  int64_t xstride = 0;            // per-shard length of the all-reduce vector
  DevBuf<double> xsend, xrecv;
  int64_t nstrips = 0, nrb = 0;  // row partials per row, column partials per column
  int64_t nmax = 0;               // max-exponent slots (CTAs of a full sweep)
  int pts_cs = 1;                 // cluster size of the points sweep's row-partial merge
  int nblk = 0;  // O(n) kernel grid
  int gv = 0;    // grid of the ASPOT attempt's O(n) kernels (one element of 2n + 1 per thread, <= 2 per SM)
  int eval_blocks = 0;  // k_point_eval grid
  int eval_tpi = 4;     // k_point_eval threads per index
  int pfmt = 0;  // PartialFormat of rowp/colp written by the sweep
  bool use_tc = false;  // fp32 points sweeps run sweep_tc_f32 (tensor-core exponents)
  int strip = 256;
  size_t sweep_smem = 0;
  size_t one_smem = 0;  // sweep_pts1_f32 (one-sided z_check' sweep)
  DevBuf<double> slots;     // 7 dual points
  DevBuf<double> sums;      // 6 x (row, col)
  DevBuf<double> rowp, colp, maxp, scratch, partial;
  DevBuf<float> carry, carry_b;  // carried shifts of the points sweep (sweep_pts2_f32): [strip][n], [vshard][n]
  DevBuf<unsigned> carry_ticket; // [vshard][strip]
  DevBuf<unsigned long long> carry_stats;  // CTAs of sweep_pts2_f32 launches: carried, exact
  DevBuf<double> dpart, gpart;  // deferred-decision partials: k_point_eval (defer) / k_gk_update (scaled point)
  DevBuf<int> gflag;            // non-finite Greenkhorn update seen (k_gk_update)
  // K1'' stash: the next z_bar's partials from the fused one-sided pass
  // (sweep_pts1_f32), its rescaled side (kbar: [row | col]) and the pass's veto
  DevBuf<double> rowp2, colp2, maxp2, kbar;
  DevBuf<int> stash_bad;
  DevBuf<double> rt, ct;    // marginals the dual targets
  DevBuf<double> ro_buf;    // rounding vectors: rho, kappa, lu, lv, rowx, colx, a, b, row_slack, col_slack
  DevBuf<double> ro_r, ro_c;  // original marginals for rounding
  DevBuf<float4> rc_part;     // fused final pass of the device rounding (plan.cuh): fp32 [row][strip] partials
  DevBuf<float> rc_pm;
  DevBuf<double> rc_part64;   // fp64 problems: [row][strip][3]
  DevBuf<double> rc_scratch;  // device rounding's block partials
  DevBuf<AspotCtl> ctl;
  DevBuf<unsigned> ticket;
  PinnedObj<AspotCtl> host_ctl_buf;
  AspotCtl* host_ctl = nullptr;  // pinned mirror
  cudaStream_t stream = nullptr;  // the stream every kernel on these buffers runs on
  DevBuf<TraceDev> trace;
  DevBuf<IterLogDev> iterlog;
  int64_t slot_stride = 0;
  ~Workspace() {
    // blocks return to the cache only once nothing can still use them
    if (stream) cudaStreamSynchronize(stream);
  }
  Slot slot(int k) const { return Slot{slots.p + k * slot_stride, n}; }
  double* row(int k) const { return sums.p + (2 * k) * n; }
  double* col(int k) const { return sums.p + (2 * k + 1) * n; }
  double* rv(int k) const { return ro_buf.p + k * n; }
};

// Cost-sweep grid (the rounding output stage): 256 columns x `rows` rows.
inline int cost_sweep_rows(int64_t n) { return int(std::max<int64_t>(16, ceil_div(n, 64))); }
inline int64_t cost_sweep_parts(int64_t n) { return ceil_div(n, kThreads) * ceil_div(n, cost_sweep_rows(n)); }

enum SlotId { S_Z = 0, S_ZC = 1, S_ZB = 2, S_G = 3, S_ZG = 4, S_ZH = 5, S_ZN = 6, kSlots = 7 };
constexpr int S_ZBN = kSlots;           // K1'': the next z_bar, formed with z_check' (k_gk_update)
constexpr int kSlotsWs = kSlots + 1;

// One-sided points sweep of z_check' (sweep_pts1_f32): the same grid and
// partial buffers as launch_sweep, unsharded fp32 points problems only.
inline bool one_sided_supported(const Context& cx, const DevProblem& P) {
  static const bool on = [] {
    const char* e = std::getenv("POTGPU_ONE_SIDED");
    return !(e && e[0] == '0');
  }();
  return on && P.dtype == POTGPU_F32 && P.dot_form() && !cx.comm.sharded() && pts_pairs() == 2;
}

// K1'' on the one-sided pass ($POTGPU_K1PP, default on): the pass also forms
// the next iteration's z_bar (sweep.cuh sweep_pts1_f32).
inline bool k1pp_supported(const Context& cx, const DevProblem& P) {
  static const bool on = [] {
    const char* e = std::getenv("POTGPU_K1PP");
    return !(e && e[0] == '0');
  }();
  return on && one_sided_supported(cx, P);
}

inline void prepare_workspace(Context& cx, const DevProblem& P, Workspace& ws, int64_t trace_cap, int64_t log_cap) {
  const int64_t n = P.n;
  ws.n = n;
  ws.stream = cx.stream;
  int occ = 2;
  if (P.dtype == POTGPU_F64) {
    PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_f64_dense<true>, kThreads, 0));
  } else if (P.kind == POTGPU_COST_DENSE) {
    PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_f32<SrcDenseF32>, kThreads, 0));
  } else {
    const size_t sm_est = sweep_pts_smem(int(std::min<int64_t>(n, kMaxRowsPerCta)));
    switch (pts_pairs()) {
      case 2:
        raise_dyn_smem(sweep_pts2_f32<1>, size_t(int(sweep_pts2_smem(int(kMaxRowsPerCta)))));
        PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_pts2_f32<1>, kThreads,
                                                            sweep_pts2_smem(int(std::min<int64_t>(n, kMaxRowsPerCta)))));
        break;
      case 5:
        raise_dyn_smem(sweep_ptsR_f32<4>, size_t(int(sweep_pts_smem(int(kMaxRowsPerCta)))));
        PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_ptsR_f32<4>, kThreads, sm_est));
        break;
      case 3:
        raise_dyn_smem(sweep_pts2s_f32, size_t(int(sweep_pts_smem(int(kMaxRowsPerCtaS)))));
        PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_pts2s_f32, kThreads,
                                                            sweep_pts_smem(int(std::min<int64_t>(n, kMaxRowsPerCtaS)))));
        break;
      case 4: PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_pts_f32<4>, kThreads, sm_est)); break;
      case 6: PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_pts_f32<6>, kThreads, sm_est)); break;
      default: PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_pts_f32<8>, kThreads, sm_est)); break;
    }
  }
  occ = std::max(occ, 1);
  const bool use_tc = carry_supported(P) && tc_enabled();
  ws.use_tc = use_tc;
  ws.strip = P.dtype == POTGPU_F64 ? kStripCols : (P.dot_form() ? 64 * ((pts_pairs() == 2 || pts_pairs() == 3 || pts_pairs() == 5) ? kPairs : pts_pairs()) : kStripCols32);
  const int64_t max_rows = (P.dot_form() && pts_pairs() == 3) ? kMaxRowsPerCtaS : kMaxRowsPerCta;
  ws.pfmt = P.dtype == POTGPU_F64 ? PF_F64 : PF_F32_SCALED;
  const int64_t tc_cap = int64_t(cx.num_sms) * 4;
  if (use_tc) {
    raise_dyn_smem(sweep_tc_f32, size_t(int(sweep_tc_smem())));
  }
  ws.g = use_tc ? choose_grid_tc(n, n, tc_cap) : choose_grid(n, n, cx.num_sms, occ, ws.strip, max_rows);
  int64_t max_rb = ws.g.grid.y;
  int max_rpc = ws.g.rows_per_cta;
  ws.shards.clear();
  ws.nshards = cx.comm.total();
  if (cx.comm.sharded()) {
    for (int p = 0; p < cx.comm.vshards; ++p) {
      ShardGrid sg;
      sg.index = cx.comm.shard_index(p);
      sg.lo = cx.comm.lo(n, sg.index);
      sg.hi = cx.comm.hi(n, sg.index);
      sg.g = use_tc ? choose_grid_tc(n, sg.hi - sg.lo, tc_cap) : choose_grid(n, sg.hi - sg.lo, cx.num_sms, occ, ws.strip, max_rows);
      max_rb = std::max<int64_t>(max_rb, sg.g.grid.y);
      max_rpc = std::max(max_rpc, sg.g.rows_per_cta);
      ws.shards.push_back(sg);
    }
    ws.xstride = round_up(2 * n + ws.nshards + 2, 32);
    ws.xsend.alloc(size_t(cx.comm.vshards * ws.xstride));
    ws.xrecv.alloc(size_t(ws.xstride));
  }
  ws.pts_cs = (P.dot_form() && pts_pairs() == 2 && !use_tc) ? pts_cluster(ws.g.grid.x) : 1;
  for (const ShardGrid& sh : ws.shards) ws.pts_cs = std::min(ws.pts_cs, pts_cluster(sh.g.grid.x));
  ws.sweep_smem = P.dtype == POTGPU_F64 ? 0 : std::max(sweep_pts2_smem(max_rpc, ws.pts_cs > 1), sweep_f32_smem(max_rpc));
  if (P.dtype != POTGPU_F64) {
    raise_dyn_smem(sweep_f32<SrcDenseF32>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts2_f32<1>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts2s_f32, size_t(int(ws.sweep_smem)));
    {
      const int sm1 = int(std::max(ws.sweep_smem, sweep_pts1_smem(max_rpc)));
      raise_dyn_smem(sweep_pts1_f32<0>, size_t(sm1));
      raise_dyn_smem(sweep_pts1_f32<1>, size_t(sm1));
      raise_dyn_smem(sweep_pts1_f32<2>, size_t(sm1));
      raise_dyn_smem(sweep_pts1_f32<3>, size_t(sm1));
    }
    ws.one_smem = std::max(ws.sweep_smem, sweep_pts1_smem(max_rpc));
    raise_dyn_smem(sweep_ptsR_f32<4>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts2_f32<2>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts2_f32<4>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts2_f32<8>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts_f32<4>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts_f32<6>, size_t(int(ws.sweep_smem)));
    raise_dyn_smem(sweep_pts_f32<8>, size_t(int(ws.sweep_smem)));
  }
  ws.nstrips = ws.g.grid.x / ws.pts_cs;
  if (carry_supported(P) && ws.pts_cs == 1) {
    // -inf carries: the first launch of a row segment takes the exact path
    const int vsh = std::max(1, cx.comm.sharded() ? cx.comm.vshards : 1);
    ws.carry.alloc(size_t(ws.g.grid.x) * size_t(n));
    ws.carry_b.alloc(size_t(vsh) * size_t(n));
    ws.carry_ticket.alloc(size_t(vsh) * ws.g.grid.x);
    launch_k(k_fill_f32, dim3(cx.num_sms), dim3(kVecThreads), 0, cx.stream, ws.carry.p, int64_t(ws.g.grid.x) * n,
             -INFINITY);
    launch_k(k_fill_f32, dim3(cx.num_sms), dim3(kVecThreads), 0, cx.stream, ws.carry_b.p, int64_t(vsh) * n, NAN);
    ws.carry_ticket.zero(cx.stream);
    ws.carry_stats.alloc(2);
    ws.carry_stats.zero(cx.stream);
  }
  ws.nrb = ws.g.grid.y;
  ws.nmax = int64_t(ws.g.grid.x) * ws.g.grid.y;
  ws.nblk = int(std::min<int64_t>(cx.num_sms, std::max<int64_t>(1, ceil_div(n, kVecThreads))));
  ws.slot_stride = round_up(2 * n + 1, 32);
  ws.slots.alloc(size_t(kSlotsWs * ws.slot_stride));
  ws.sums.alloc(size_t(2 * kRoles * n));
  ws.rowp.alloc(size_t(2 * ws.g.grid.x * n));  // x2: (max, sum) LSE partials
  ws.colp.alloc(size_t(2 * max_rb * n));
  ws.maxp.alloc(size_t(ws.g.grid.x * max_rb));
  // <= 2 kVecThreads: the deferred decisions reduce at most two partial rows per thread
  ws.eval_tpi = eval_tpi(ws.nstrips);
  ws.eval_blocks = int(std::min<int64_t>(std::min<int64_t>(ceil_div(n * ws.eval_tpi, kEvalThreads), eval_blocks_cap(cx.num_sms)),
                                         2 * kVecThreads));
  ws.scratch.alloc(size_t(std::max(8192, kNumAcc * ws.eval_blocks)));
  ws.ticket.alloc(2);  // [0] k_point_eval, [1] the attempt's O(n) kernels (k_zgrave, k_gk_update, k_commit)
  ws.ticket.zero(cx.stream);
  ws.dpart.alloc(size_t(kNumAcc * ws.eval_blocks));
  ws.gv = int(std::min<int64_t>(2 * cx.num_sms, ceil_div(2 * n + 1, kVecThreads)));
  ws.gpart.alloc(size_t(kNumAcc * ws.gv));
  ws.gflag.alloc(1);
  ws.gflag.zero(cx.stream);
  if (k1pp_supported(cx, P)) {
    ws.rowp2.alloc(size_t(ws.g.grid.x * n));
    ws.colp2.alloc(size_t(ws.g.grid.y * n));
    ws.maxp2.alloc(size_t(ws.g.grid.x * ws.g.grid.y));
    ws.kbar.alloc(size_t(2 * n));
    ws.stash_bad.alloc(1);
    ws.stash_bad.zero(cx.stream);
  }
  ws.partial.alloc(size_t(std::max<int64_t>(4096, cost_sweep_parts(n) + ws.nshards * ceil_div(n, kThreads))));
  ws.rt.alloc(size_t(n));
  ws.ct.alloc(size_t(n));
  ws.ro_buf.alloc(size_t(10 * n));
  ws.ro_r.alloc(size_t(n));
  ws.ro_c.alloc(size_t(n));
  PG_CK(cudaMemcpyAsync(ws.ro_r.p, P.r.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  PG_CK(cudaMemcpyAsync(ws.ro_c.p, P.c.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  ws.rc_scratch.alloc(size_t(8 * 32));
  if (!cx.comm.sharded()) {  // the device rounding's fused pass (plan.cuh round_device)
    if (P.dtype == POTGPU_F64) {
      if (P.kind == POTGPU_COST_DENSE) ws.rc_part64.alloc(size_t(3 * n * ceil_div(n, kStripCols)));
    } else {
      const int64_t strips = ceil_div(n, P.kind == POTGPU_COST_SQEUCLIDEAN ? int64_t(256) : int64_t(512));
      ws.rc_part.alloc(size_t(n * strips));
      ws.rc_pm.alloc(size_t(n * strips));
    }
  }
  ws.ctl.alloc(1);
  if (!ws.host_ctl) ws.host_ctl = ws.host_ctl_buf.get();
  ws.trace.alloc(size_t(std::max<int64_t>(trace_cap, 1)));
  ws.iterlog.alloc(size_t(std::max<int64_t>(log_cap, 1)));
}

// --------------------------------------------------------------------------

// Sweep dispatch (one launch over the rows of `sh`, or all rows).
inline void launch_sweep(Context& cx, const DevProblem& P, Workspace& ws, Slot z, const double* lu, const double* lv,
                         const int* gate, bool floor_exp, double gamma, const ShardGrid* sh = nullptr) {
  const SweepGrid& g = sh ? sh->g : ws.g;
  SweepArgs a{};
  a.n = P.n;
  a.row_lo = sh ? sh->lo : 0;
  a.row_hi = sh ? sh->hi : P.n;
  a.rows_per_cta = g.rows_per_cta;
  a.u = z.u(); a.v = z.v(); a.w = z.w();
  a.lu = lu; a.lv = lv;
  a.rowshift = P.rowshift();
  a.colshift = P.dot_form() ? P.yshift.p : nullptr;
  a.rowp = ws.rowp.p; a.colp = ws.colp.p; a.maxp = ws.maxp.p;
  a.gate = gate;
  a.gamma = gamma;
  if (ws.carry.p && pts_pairs() == 2 && ws.pts_cs == 1 && P.dot_form()) {
    const int64_t k = sh ? int64_t(sh - ws.shards.data()) : 0;
    a.carry = ws.carry.p;
    a.carry_b = ws.carry_b.p + k * P.n;
    a.carry_ticket = ws.carry_ticket.p + k * g.grid.x;
    a.carry_stats = ws.carry_stats.p;
    static const int dbg = [] { const char* e = std::getenv("POTGPU_TC_DEBUG"); return e ? std::atoi(e) : 0; }();
    a.tc_debug = dbg;
  }
  if (P.dtype == POTGPU_F64) {
    if (floor_exp) launch_k(sweep_f64_dense<true>, dim3(g.grid), dim3(kThreads), 0, cx.stream, P.L64.p, P.ld, a);
    else launch_k(sweep_f64_dense<false>, dim3(g.grid), dim3(kThreads), 0, cx.stream, P.L64.p, P.ld, a);
  } else if (P.kind == POTGPU_COST_DENSE) {
    SrcDenseF32 s{P.C32.p, P.ld, float(kLog2e / gamma)};
    launch_k(sweep_f32<SrcDenseF32>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, s, a);
  } else {
    if (P.XS_gamma != gamma) throw Error(POTGPU_ERR_CUDA, "internal: scaled coordinates not prepared for this gamma");
    SrcPointsDotF32 s{P.XD4.p, P.YS4.p};
    switch (pts_pairs()) {
      case 3: launch_k(sweep_pts2s_f32, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, s, a); break;
      case 5: launch_k(sweep_ptsR_f32<4>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, s, a); break;
      case 2:  // two-row variant, row partials merged over a cluster of ws.pts_cs strips
        switch (ws.pts_cs) {
          case 8: launch_kc(sweep_pts2_f32<8>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, 8, s, a); break;
          case 4: launch_kc(sweep_pts2_f32<4>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, 4, s, a); break;
          case 2: launch_kc(sweep_pts2_f32<2>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, 2, s, a); break;
          default:
            if (ws.use_tc && a.carry) launch_k(sweep_tc_f32, dim3(g.grid), dim3(kTcThreads), sweep_tc_smem(), cx.stream, s, a);
            else launch_k(sweep_pts2_f32<1>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, s, a);
            break;
        }
        break;
      case 4: launch_k(sweep_pts_f32<4>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, s, a); break;
      case 6: launch_k(sweep_pts_f32<6>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, s, a); break;
      default: launch_k(sweep_pts_f32<8>, dim3(g.grid), dim3(kThreads), ws.sweep_smem, cx.stream, s, a); break;
    }
  }
  PG_CK(cudaGetLastError());
}

// Where the reductions of one swept point live: the raw per-strip /
// per-row-block partials (one GPU), or the all-reduced fp64 vector
// [rows | cols | per-shard max] (sharded).
struct SweepOut {
  const double* rowp; int64_t nstrips;
  const double* colp; int64_t nrb;
  const double* maxp; int64_t nmax;
  int pfmt;
  const double* rowshift;  // source row term of the fp32 row offsets (raw partials only)
};

// The hot path of every evaluation: sweep B(z) (own rows) and, when sharded,
// gather + all-reduce (shard.cuh).
inline SweepOut sweep_point(Context& cx, const DevProblem& P, Workspace& ws, Slot z, const double* lu, const double* lv,
                            const int* gate, bool floor_exp, double gamma) {
  const int64_t n = P.n;
  if (!cx.comm.sharded()) {
    launch_sweep(cx, P, ws, z, lu, lv, gate, floor_exp, gamma);
    return SweepOut{ws.rowp.p, ws.nstrips, ws.colp.p, ws.nrb, ws.maxp.p, ws.nmax, ws.pfmt, P.rowshift()};
  }
  for (size_t p = 0; p < ws.shards.size(); ++p) {
    const ShardGrid& sh = ws.shards[p];
    launch_sweep(cx, P, ws, z, lu, lv, gate, floor_exp, gamma, &sh);
    launch_k(k_shard_gather, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream, ws.rowp.p, ws.nstrips, ws.colp.p, sh.g.grid.y, ws.maxp.p,
                                                          int64_t(sh.g.grid.x) * sh.g.grid.y, ws.pfmt, z, lu, P.rowshift(),
                                                          sh.lo, sh.hi,
                                                          sh.index, ws.nshards, ws.xsend.p + p * ws.xstride, gate);
    PG_CK(cudaGetLastError());
  }
  shard_allreduce(cx.comm, cx.stream, cx.num_sms, ws.xsend.p, ws.xstride, 2 * n + ws.nshards, NcclApi::kSum, ws.xrecv.p,
                  gate);
  return SweepOut{ws.xrecv.p, 1, ws.xrecv.p + n, 1, ws.xrecv.p + 2 * n, ws.nshards, PF_F64, nullptr};
}

// Device time of the hot-path sweeps alone (no reduction) over this
// process's rows; the rows that costs.
inline int64_t launch_local_sweeps(Context& cx, const DevProblem& P, Workspace& ws, Slot z, double gamma) {
  if (!cx.comm.sharded()) {
    launch_sweep(cx, P, ws, z, nullptr, nullptr, nullptr, true, gamma);
    return P.n;
  }
  int64_t rows = 0;
  for (const ShardGrid& sh : ws.shards) {
    launch_sweep(cx, P, ws, z, nullptr, nullptr, nullptr, true, gamma, &sh);
    rows += sh.hi - sh.lo;
  }
  return rows;
}

// Sum of a host scalar over the processes of a sharded job.
inline double allreduce_host_sum(Context& cx, Workspace& ws, double x) {
  if (cx.comm.host_fn) {
    PG_CK(cudaStreamSynchronize(cx.stream));
    cx.comm.host_fn(&x, 1, NcclApi::kSum, cx.comm.host_user);
    return x;
  }
  if (!cx.comm.nccl) return x;
  PG_CK(cudaMemcpyAsync(ws.xsend.p, &x, sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  nccl_check(nccl_api().AllReduce(ws.xsend.p, ws.xrecv.p, 1, NcclApi::kFloat64, NcclApi::kSum, cx.comm.nccl, cx.stream),
             "ncclAllReduce");
  double y = 0.0;
  PG_CK(cudaMemcpyAsync(&y, ws.xrecv.p, sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
  PG_CK(cudaStreamSynchronize(cx.stream));
  return y;
}

// The per-point evaluation (partials -> B 1, B^T 1, scalars, decision).
inline void launch_eval(Context& cx, Workspace& ws, const SweepOut& so, Slot z, int role, const int* gate,
                        const ReduceArgs* scaled = nullptr, bool defer = false, const int* alt_sel = nullptr) {
  ReduceArgs r{};
  if (scaled) r = *scaled;
  r.z = z;
  r.rowp = so.rowp; r.nstrips = so.nstrips;
  r.colp = so.colp; r.nrowblocks = so.nrb;
  r.maxp = so.maxp; r.nmax = so.nmax;
  r.row_out = ws.row(role); r.col_out = ws.col(role);
  r.rt = ws.rt.p; r.ct = ws.ct.p;
  r.scratch = defer ? ws.dpart.p : ws.scratch.p;
  r.defer = defer ? 1 : 0;
  r.gate = gate;
  r.pfmt = so.pfmt;
  r.rowshift = so.rowshift;
  r.mode = scaled ? 1 : 0;
  if (alt_sel && ws.rowp2.p) {  // K1'' stash (same grid and layout as the sweep's partials)
    r.alt_sel = alt_sel;
    r.rowp_alt = ws.rowp2.p;
    r.colp_alt = ws.colp2.p;
    r.maxp_alt = ws.maxp2.p;
    r.direct_row = ws.kbar.p;
    r.direct_col = ws.kbar.p + ws.n;
  }
  switch (ws.eval_tpi) {
    case 1: launch_k(k_point_eval<1>, dim3(ws.eval_blocks), dim3(kEvalThreads), 0, cx.stream, ws.ctl.p, role, r, ws.ticket.p); break;
    case 2: launch_k(k_point_eval<2>, dim3(ws.eval_blocks), dim3(kEvalThreads), 0, cx.stream, ws.ctl.p, role, r, ws.ticket.p); break;
    case 8: launch_k(k_point_eval<8>, dim3(ws.eval_blocks), dim3(kEvalThreads), 0, cx.stream, ws.ctl.p, role, r, ws.ticket.p); break;
    default: launch_k(k_point_eval<4>, dim3(ws.eval_blocks), dim3(kEvalThreads), 0, cx.stream, ws.ctl.p, role, r, ws.ticket.p); break;
  }
  PG_CK(cudaGetLastError());
}

inline void launch_one_sided(Context& cx, const DevProblem& P, Workspace& ws, Slot z, const int* gate, const OneSidedArgs& o) {
  const SweepGrid& g = ws.g;
  SweepArgs a{};
  a.n = P.n;
  a.row_lo = 0;
  a.row_hi = P.n;
  a.rows_per_cta = g.rows_per_cta;
  a.u = z.u(); a.v = z.v(); a.w = z.w();
  a.lu = nullptr; a.lv = nullptr;
  a.rowshift = P.rowshift();
  a.colshift = P.yshift.p;
  a.rowp = ws.rowp.p; a.colp = ws.colp.p; a.maxp = ws.maxp.p;
  a.gate = gate;
  a.gamma = 0.0;
  SrcPointsDotF32 s{P.XD4.p, P.YS4.p};
  switch (pts1_two()) {
    case 1: launch_k(sweep_pts1_f32<1>, dim3(g.grid), dim3(kThreads), ws.one_smem, cx.stream, s, a, o); break;
    case 2: launch_k(sweep_pts1_f32<2>, dim3(g.grid), dim3(kThreads), ws.one_smem, cx.stream, s, a, o); break;
    case 3: launch_k(sweep_pts1_f32<3>, dim3(g.grid), dim3(kThreads), ws.one_smem, cx.stream, s, a, o); break;
    default: launch_k(sweep_pts1_f32<0>, dim3(g.grid), dim3(kThreads), ws.one_smem, cx.stream, s, a, o); break;
  }
}

// Where an attempt's deferred decisions find their partials (aspot_kernels.cuh Pending).
inline Pending pending_of(Workspace& ws) {
  Pending pd;
  pd.eval_part = ws.dpart.p;
  pd.eval_nb = ws.eval_blocks;
  pd.gk_part = ws.gpart.p;
  pd.gk_nb = ws.gv;
  pd.flag = ws.gflag.p;
  pd.ticket = ws.ticket.p + 1;
  return pd;
}

}  // namespace potgpu
