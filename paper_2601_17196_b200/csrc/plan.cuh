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
                                                             const double* rowshift, double* row, double* col) {
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
                                                           lu ? d(0) : nullptr, so.rowshift, d(2), d(3));
    PG_CK(cudaGetLastError());
    row.resize(size_t(n));
    col.resize(size_t(n));
    PG_CK(cudaMemcpyAsync(row.data(), d(2), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(col.data(), d(3), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
  }

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
  pe.block_sums(z, &lp, &lqk, rr, cc);
  pt.mark("round: final sums");
  double sbk = 0.0;
  if (b) { HVec t(n); for (size_t j = 0; j < n; ++j) t[j] = (*b)[j] * kap[j]; sbk = hsum(t); }
  HVec rowX3(n), colX3(n);
  for (size_t i = 0; i < n; ++i) rowX3[i] = alpha * rho[i] * (rr[i] + (a ? (*a)[i] * sbk : 0.0));
  for (size_t j = 0; j < n; ++j) colX3[j] = kap[j] * col3[j];
  // deficit fill (rounding.hpp:63-75)
  const double mass3 = hsum(rowX3);
  const double deficit = s - mass3;
  HVec fa(n), fb(n);
  for (size_t i = 0; i < n; ++i) fa[i] = std::max(r[i] - rowX3[i], 0.0);
  for (size_t j = 0; j < n; ++j) fb[j] = std::max(c[j] - colX3[j], 0.0);
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
  out.cost = pe.cost(z, Pf, Qf, &fa2, &fb, a ? &ra : nullptr, a ? &kb : nullptr, Xdev);
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

}  // namespace potgpu
