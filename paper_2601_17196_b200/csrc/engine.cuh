// engine.cuh — host-side engine: device problem, workspaces, sweep dispatch.
#pragma once

#include <algorithm>
#include <limits>
#include <memory>

#include "aspot_kernels.cuh"
#include "rounding.cuh"
#include "sweep.cuh"

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

struct Context {
  int device = 0;
  cudaStream_t stream = nullptr;
  int num_sms = 148;
  // multi-GPU row sharding (filled by potgpu_comm_init)
  int rank = 0, world = 1;
  void* nccl_comm = nullptr;
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
  DevBuf<float4> XS4, YS4; // points pre-scaled by sqrt(log2 e * scale / gamma) for the fp32 sweep
  double XS_gamma = -1.0;
  double cost_scale = 1.0;
  double cmax = 0.0;
  std::vector<double> r, c;  // host copies (original marginals)
  double s = 0.0;
};

struct Workspace {
  int64_t n = 0;
  SweepGrid g{};
  int64_t nstrips = 0, nrb = 0;
  int nblk = 0;  // O(n) kernel grid
  int eval_blocks = 0;  // k_point_eval grid (8 indices per block)
  int pfmt = 0;  // PartialFormat of rowp/colp written by the sweep
  int strip = 256;
  size_t sweep_smem = 0;
  DevBuf<double> slots;     // 7 dual points
  DevBuf<double> sums;      // 6 x (row, col)
  DevBuf<double> rowp, colp, maxp, scratch, partial;
  DevBuf<double> rt, ct;    // marginals the dual targets
  DevBuf<double> ro_buf;    // rounding vectors: rho, kappa, lu, lv, rowx, colx, a, b, row_slack, col_slack
  DevBuf<double> ro_r, ro_c;  // original marginals for rounding
  DevBuf<AspotCtl> ctl;
  DevBuf<unsigned> ticket;
  AspotCtl* host_ctl = nullptr;  // pinned mirror
  DevBuf<TraceDev> trace;
  DevBuf<IterLogDev> iterlog;
  int64_t slot_stride = 0;
  ~Workspace() {
    if (host_ctl) cudaFreeHost(host_ctl);
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

inline void prepare_workspace(Context& cx, const DevProblem& P, Workspace& ws, int64_t trace_cap, int64_t log_cap) {
  const int64_t n = P.n;
  ws.n = n;
  int occ = 2;
  if (P.dtype == POTGPU_F64) {
    PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_f64_dense<true>, kThreads, 0));
  } else if (P.kind == POTGPU_COST_DENSE) {
    PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_f32<SrcDenseF32>, kThreads, 0));
  } else {
    PG_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sweep_f32<SrcPointsF32>, kThreads, 0));
  }
  occ = std::max(occ, 1);
  ws.strip = P.dtype == POTGPU_F64 ? kStripCols : kStripCols32;
  ws.pfmt = P.dtype == POTGPU_F64 ? PF_F64 : PF_F32_SCALED;
  ws.g = choose_grid(n, cx.num_sms, occ, ws.strip);
  ws.sweep_smem = P.dtype == POTGPU_F64 ? 0 : sweep_f32_smem(ws.g.rows_per_cta);
  if (P.dtype != POTGPU_F64) {
    PG_CK(cudaFuncSetAttribute(sweep_f32<SrcDenseF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ws.sweep_smem)));
    PG_CK(cudaFuncSetAttribute(sweep_f32<SrcPointsF32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(ws.sweep_smem)));
  }
  ws.nstrips = ws.g.grid.x;
  ws.nrb = ws.g.grid.y;
  ws.nblk = int(std::min<int64_t>(cx.num_sms, std::max<int64_t>(1, ceil_div(n, kVecThreads))));
  ws.slot_stride = round_up(2 * n + 1, 32);
  ws.slots.alloc(size_t(kSlots * ws.slot_stride));
  ws.sums.alloc(size_t(2 * kRoles * n));
  ws.rowp.alloc(size_t(2 * ws.nstrips * n));  // x2: (max, sum) LSE partials
  ws.colp.alloc(size_t(2 * ws.nrb * n));
  ws.maxp.alloc(size_t(ws.nstrips * ws.nrb));
  ws.eval_blocks = int(std::min<int64_t>(ceil_div(n * kTPI, kEvalThreads), 4096));
  ws.scratch.alloc(size_t(std::max(8192, kNumAcc * ws.eval_blocks)));
  ws.ticket.alloc(1);
  ws.ticket.zero(cx.stream);
  ws.partial.alloc(size_t(std::max<int64_t>(4096, cost_sweep_parts(n))));
  ws.rt.alloc(size_t(n));
  ws.ct.alloc(size_t(n));
  ws.ro_buf.alloc(size_t(10 * n));
  ws.ro_r.alloc(size_t(n));
  ws.ro_c.alloc(size_t(n));
  ws.ctl.alloc(1);
  if (!ws.host_ctl) PG_CK(cudaMallocHost(&ws.host_ctl, sizeof(AspotCtl)));
  ws.trace.alloc(size_t(std::max<int64_t>(trace_cap, 1)));
  ws.iterlog.alloc(size_t(std::max<int64_t>(log_cap, 1)));
}

// --------------------------------------------------------------------------
// Sweep dispatch.
inline void launch_sweep(Context& cx, const DevProblem& P, Workspace& ws, Slot z, const double* lu, const double* lv,
                         const int* gate, bool floor_exp, double gamma) {
  SweepArgs a;
  a.n = P.n;
  a.rows_per_cta = ws.g.rows_per_cta;
  a.u = z.u(); a.v = z.v(); a.w = z.w();
  a.lu = lu; a.lv = lv;
  a.rowp = ws.rowp.p; a.colp = ws.colp.p; a.maxp = ws.maxp.p;
  a.gate = gate;
  a.gamma = gamma;
  if (P.dtype == POTGPU_F64) {
    if (floor_exp) sweep_f64_dense<true><<<ws.g.grid, kThreads, 0, cx.stream>>>(P.L64.p, P.ld, a);
    else sweep_f64_dense<false><<<ws.g.grid, kThreads, 0, cx.stream>>>(P.L64.p, P.ld, a);
  } else if (P.kind == POTGPU_COST_DENSE) {
    SrcDenseF32 s{P.C32.p, P.ld, float(kLog2e / gamma)};
    sweep_f32<SrcDenseF32><<<ws.g.grid, kThreads, ws.sweep_smem, cx.stream>>>(s, a);
  } else {
    if (P.XS_gamma != gamma) throw Error(POTGPU_ERR_CUDA, "internal: scaled coordinates not prepared for this gamma");
    SrcPointsF32 s{P.XS4.p, P.YS4.p};
    sweep_f32<SrcPointsF32><<<ws.g.grid, kThreads, ws.sweep_smem, cx.stream>>>(s, a);
  }
  PG_CK(cudaGetLastError());
}

// The per-point evaluation (partials -> B 1, B^T 1, scalars, decision).
inline void launch_eval(Context& cx, Workspace& ws, Slot z, int role, const int* gate, const ReduceArgs* scaled = nullptr) {
  ReduceArgs r{};
  if (scaled) r = *scaled;
  r.z = z;
  r.rowp = ws.rowp.p; r.nstrips = ws.nstrips;
  r.colp = ws.colp.p; r.nrowblocks = ws.nrb;
  r.maxp = ws.maxp.p; r.nmax = ws.nstrips * ws.nrb;
  r.row_out = ws.row(role); r.col_out = ws.col(role);
  r.rt = ws.rt.p; r.ct = ws.ct.p;
  r.scratch = ws.scratch.p;
  r.gate = gate;
  r.pfmt = ws.pfmt;
  r.mode = scaled ? 1 : 0;
  k_point_eval<<<ws.eval_blocks, kEvalThreads, 0, cx.stream>>>(ws.ctl.p, role, r, ws.ticket.p);
  PG_CK(cudaGetLastError());
}

}  // namespace potgpu
