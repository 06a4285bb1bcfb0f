// sinkhorn.cuh — feasible / tuned Sinkhorn sessions (solvers.hpp:483-589)
// over the kernels of sinkhorn_kernels.cuh. Included by capi.cu after the
// Session base and the setup helpers.
#pragma once

#include "sinkhorn_kernels.cuh"

namespace potgpu {

// entropy H(x) = -sum x log x, 0 log 0 = 0 (solvers.hpp:19-28)
inline double entropy_h(const HVec& x) {
  double h = 0.0;
  for (double e : x)
    if (e > 0) h -= e * std::log(e);
  return h;
}

// dummy_penalty (solvers.hpp:485-490)
inline double dummy_penalty(double cmax, double epsilon) {
  double A = cmax > 0 ? 8.0 * cmax / epsilon : 0.0;
  if (!(A > cmax) || !std::isfinite(A)) A = cmax > 0 ? 2.0 * cmax : 1.0;
  return A;
}

struct SinkhornSession : Session {
  int kind;
  Workspace ws;
  double gamma = 0, tol = 0, A = 0;
  HVec r_ext, c_ext;
  DevBuf<double> vec;     // u, u_next, v, log_r, log_c, r, c (each n+1), scratch
  DevBuf<double> zv;      // point (0, v[0..n), 0) for the fp32 row-LSE sweep
  DevBuf<double> zf;      // point (u[0..n), v[0..n), 0) for the output stage
  DevBuf<double> zuv;     // point (u[0..n), v[0..n), 0) of the fast column pass (fp32)
  DevBuf<double> dummy;   // k_sk_dummy block partials
  DevBuf<unsigned> dummy_ticket;
  DevBuf<SinkCtl> ctl;
  PinnedObj<SinkCtl> hctl_buf;
  SinkCtl* hctl = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t trace_cap = 1;
  int64_t graph_nodes = 8;
  SinkVec sv{};

  SinkhornSession(Context& c, int k) : Session(c), kind(k) {}
  ~SinkhornSession() override {
    cudaStreamSynchronize(cx.stream);  // before any buffer returns to the cache
    if (exec) cudaGraphExecDestroy(exec);
  }

  // k_sk_dummy grid: >= 2048 values per block (the last block merges the
  // block partials sequentially)
  int dummy_blocks() const { return int(std::max<int64_t>(1, std::min<int64_t>(kSkDummyBlocks, P.n / 2048))); }
  int sk_blocks() const { return int(std::min<int64_t>(ceil_div(P.n * kSkTPI, kSkThreads), 4096)); }
  Slot zv_slot() const { return Slot{zv.p, P.n}; }
  Slot zf_slot() const { return Slot{zf.p, P.n}; }

  void sync_ctl() {
    PG_CK(cudaMemcpyAsync(hctl, ctl.p, sizeof(SinkCtl), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
  }

  // one n^2 row-LSE sweep over rows [lo, hi) (grid g) at the current v
  void row_sweep(const int* gate, const ShardGrid* sh) {
    const int64_t n = P.n;
    const SweepGrid& g = sh ? sh->g : ws.g;
    if (P.dtype == POTGPU_F64) {
      launch_k(sweep_rowlse_f64, dim3(g.grid), dim3(kThreads), 0, cx.stream, P.L64.p, P.ld, n, sv.v, sh ? sh->lo : 0, sh ? sh->hi : n,
                                                           g.rows_per_cta, reinterpret_cast<double2*>(ws.rowp.p), gate);
    } else {
      launch_sweep(cx, P, ws, zv_slot(), nullptr, nullptr, gate, false, gamma, sh);  // rows of (0, v, 0)
    }
  }

  // one n^2 column-LSE sweep over rows [lo, hi) at the current u
  void col_sweep(const int* gate, const ShardGrid* sh) {
    const int64_t n = P.n;
    const SweepGrid& g = sh ? sh->g : ws.g;
    const int64_t lo = sh ? sh->lo : 0, hi = sh ? sh->hi : n;
    if (P.dtype == POTGPU_F64) {
      launch_k(sweep_collse_f64, dim3(g.grid), dim3(kThreads), 0, cx.stream, P.L64.p, P.ld, n, sv.u, lo, hi, g.rows_per_cta,
                                                           reinterpret_cast<double2*>(ws.colp.p), gate);
    } else if (P.kind == POTGPU_COST_DENSE) {
      SrcDenseF32 s{P.C32.p, P.ld, float(kLog2e / gamma)};
      launch_k(sweep_collse_f32<SrcDenseF32>, dim3(g.grid), dim3(kThreads), 0, cx.stream, s, n, sv.u, lo, hi, g.rows_per_cta,
                                                                        reinterpret_cast<float2*>(ws.colp.p), gate);
    } else {
      SrcPointsF32 s{P.XS4.p, P.YS4.p};
      launch_k(sweep_collse_f32<SrcPointsF32>, dim3(g.grid), dim3(kThreads), 0, cx.stream, s, n, sv.u, lo, hi, g.rows_per_cta,
                                                                         reinterpret_cast<float2*>(ws.colp.p), gate);
    }
  }

  int lse_fmt() const { return P.dtype == POTGPU_F64 ? LP_F64 : LP_F32; }

  void row_lse(const int* gate) {  // at the current v
    const int64_t n = P.n;
    const double* rowp = ws.rowp.p;
    int64_t nstrips = ws.nstrips;
    int fmt = lse_fmt();
    if (!cx.comm.sharded()) {
      row_sweep(gate, nullptr);
    } else {  // rows are whole in a shard: gather (M, S) of own rows, SUM
      for (size_t p = 0; p < ws.shards.size(); ++p) {
        const ShardGrid& sh = ws.shards[p];
        row_sweep(gate, &sh);
        launch_k(k_shard_gather_lse<true>, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream, ws.rowp.p, ws.nstrips, fmt, n, sh.lo, sh.hi,
                                                                        P.rowshift(), ws.xsend.p + p * ws.xstride, gate);
      }
      shard_allreduce(cx.comm, cx.stream, cx.num_sms, ws.xsend.p, ws.xstride, 2 * n, NcclApi::kSum, ws.xrecv.p, gate);
      rowp = ws.xrecv.p;
      nstrips = 1;
      fmt = LP_F64;
    }
    launch_k(k_sk_dummy, dim3(dummy_blocks()), dim3(kVecThreads), 0, cx.stream, ctl.p, sv.v, 0, dummy.p, dummy_ticket.p, gate);
    launch_k(k_sk_rows, dim3(sk_blocks()), dim3(kSkThreads), 0, cx.stream, ctl.p, sv, rowp, nstrips, fmt,
                                                      cx.comm.sharded() ? nullptr : P.rowshift(), gate);
  }

  // fp32: the column LSE comes from the fast row-shifted sweep at (u, v_old, 0)
  // (sweep_f32, the production kernel) with v_old removed in fp64; the exact
  // per-column-max pass runs only when that flags a flushed column.
  bool fast_cols() const { return P.dtype == POTGPU_F32; }
  Slot zuv_slot() const { return Slot{zuv.p, P.n}; }

  void col_lse(int update, const int* gate) {  // at the current u
    launch_k(k_sk_dummy, dim3(dummy_blocks()), dim3(kVecThreads), 0, cx.stream, ctl.p, sv.u, 1, dummy.p, dummy_ticket.p, gate);
    if (fast_cols()) {
      col_pass(update, gate, true);
      col_pass(update, &ctl.p->col_flush, false);  // gated: only after a flush
    } else {
      col_pass(update, gate, false);
    }
  }

  void col_pass(int update, const int* gate, bool fast) {
    const int64_t n = P.n;
    const double* colp = ws.colp.p;
    int64_t nrb = ws.nrb;
    int fmt = lse_fmt();
    if (!cx.comm.sharded()) {
      if (fast) launch_sweep(cx, P, ws, zuv_slot(), nullptr, nullptr, gate, false, gamma);
      else col_sweep(gate, nullptr);
    } else {  // column LSE over shards: MAX of the shard maxima, rescale, SUM
      for (size_t p = 0; p < ws.shards.size(); ++p) {
        const ShardGrid& sh = ws.shards[p];
        if (fast) launch_sweep(cx, P, ws, zuv_slot(), nullptr, nullptr, gate, false, gamma, &sh);
        else col_sweep(gate, &sh);
        launch_k(k_shard_gather_lse<false>, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream, ws.colp.p, sh.g.grid.y, fmt, n, sh.lo, sh.hi,
                                                                         nullptr, ws.xsend.p + p * ws.xstride, gate);
      }
      shard_allreduce(cx.comm, cx.stream, cx.num_sms, ws.xsend.p, ws.xstride, n, NcclApi::kMax, ws.xrecv.p, gate);
      launch_k(k_shard_lse_rescale, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream, ws.xsend.p, int(ws.shards.size()), ws.xstride, n,
                                                                  ws.xrecv.p, gate);
      shard_allreduce(cx.comm, cx.stream, cx.num_sms, ws.xsend.p + n, ws.xstride, n, NcclApi::kSum, ws.xrecv.p + n, gate);
      colp = ws.xrecv.p;
      nrb = 1;
      fmt = LP_SPLIT;
    }
    launch_k(k_sk_cols, dim3(sk_blocks()), dim3(kSkThreads), 0, cx.stream, ctl.p, sv, colp, nrb, fmt, update, sk_blocks(),
                                                      fast ? sv.zuv_v : nullptr, gate);
  }

  // solvers.hpp:463-476: u update, v update, B, E, ++iterations, record
  void enqueue_iteration() {
    const int* gate = &ctl.p->g_active;
    launch_k(k_sk_commit_u, dim3(ws.nblk), dim3(kVecThreads), 0, cx.stream, ctl.p, sv);
    col_lse(1, gate);
    row_lse(gate);
    launch_k(k_sk_scalars, dim3(1), dim3(kVecThreads), 0, cx.stream, ctl.p, sv, sk_blocks(), 0, ws.trace.p, gate);
    PG_CK(cudaGetLastError());
  }

  void begin() override {
    const int64_t n = P.n;
    if (kind == POTGPU_TUNED_SINKHORN) {  // solvers.hpp:552-557
      if (!(cfg.epsilon > 0) || !std::isfinite(cfg.epsilon)) throw Error(POTGPU_INVALID_ARGUMENT, "epsilon must be positive");
      if (!(cfg.tuning_exponent_p >= 1)) throw Error(POTGPU_INVALID_ARGUMENT, "tuning exponent p must be >= 1");
    }
    if (P.s == 0) {  // solvers.hpp:521-523, 559-561
      trivial = true;
      trivial_plan = 0.0;
      trivial_gamma = 0.0;
      return;
    }
    double h_min = 0.0;
    if (kind == POTGPU_TUNED_SINKHORN) {
      h_min = std::min(entropy_h(P.r), entropy_h(P.c));
      if (!(h_min > 0)) throw Error(POTGPU_ZERO_ENTROPY, "ZeroEntropy: tuned gamma needs positive marginal entropy");
    }
    if (n == 1) {  // one support point: the budget pins the only entry
      trivial = true;
      trivial_plan = P.s;
      trivial_gamma = cfg.gamma_override > 0 ? cfg.gamma_override : 0.0;
      return;
    }
    HVec rr, cc;
    if (kind == POTGPU_FEASIBLE_SINKHORN) {  // solvers.hpp:529-538
      const Setup st = aspot_setup(P, cfg.epsilon);
      gamma = cfg.gamma_override > 0 ? cfg.gamma_override : st.gamma;
      tol = st.eps_tilde;
      rr = st.mr;
      cc = st.mc;
      // extend(mixed, A) validates the mixed instance (extend.hpp:23)
      if (P.s > std::min(hsum(rr), hsum(cc)) + 1e-12)
        throw Error(POTGPU_BUDGET_EXCEEDS_MASS, "invalid instance: budget exceeds min mixed marginal mass");
    } else {  // solvers.hpp:571-578
      gamma = cfg.gamma_override > 0 ? cfg.gamma_override : std::pow(2.0 * cfg.epsilon / (49.0 * h_min), 1.0 / cfg.tuning_exponent_p);
      tol = h_min * std::pow(gamma, cfg.tuning_exponent_p);
      rr = P.r;
      cc = P.c;
    }
    if (!(gamma > 0) || !std::isfinite(gamma)) throw Error(POTGPU_INVALID_ARGUMENT, "gamma must be positive");
    A = dummy_penalty(P.cmax, cfg.epsilon);
    if (!(A > P.cmax)) throw Error(POTGPU_PENALTY_TOO_SMALL, "penalty must exceed max cost");
    // extend.hpp:35-37
    r_ext = rr;
    r_ext.push_back(std::max(hsum(cc) - P.s, 0.0));
    c_ext = cc;
    c_ext.push_back(std::max(hsum(rr) - P.s, 0.0));
    build_logk(cx, P, gamma);
    prepare_workspace(cx, P, ws, trace_cap, 0);
    const size_t m = size_t(n + 1);
    vec.alloc(7 * m + 8 * size_t(sk_blocks()) + 64);
    sv.u = vec.p; sv.u_next = vec.p + m; sv.v = vec.p + 2 * m; sv.log_r = vec.p + 3 * m; sv.log_c = vec.p + 4 * m;
    sv.r = vec.p + 5 * m; sv.c = vec.p + 6 * m; sv.scratch = vec.p + 7 * m;
    zv.alloc(size_t(ws.slot_stride));
    zf.alloc(size_t(ws.slot_stride));
    dummy.alloc(size_t(2 * kSkDummyBlocks));
    dummy_ticket.alloc(1);
    dummy_ticket.zero(cx.stream);
    sv.zv_v = zv.p + n;
    if (fast_cols()) {
      zuv.alloc(size_t(ws.slot_stride));
      zuv.zero(cx.stream);
      sv.zuv_u = zuv.p;
      sv.zuv_v = zuv.p + n;
    }
    HVec lr(m), lc(m);
    for (size_t i = 0; i < m; ++i) { lr[i] = std::log(r_ext[i]); lc[i] = std::log(c_ext[i]); }  // solvers.hpp:421-422
    vec.zero(cx.stream);
    zv.zero(cx.stream);
    PG_CK(cudaMemcpyAsync(sv.log_r, lr.data(), m * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    PG_CK(cudaMemcpyAsync(sv.log_c, lc.data(), m * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    PG_CK(cudaMemcpyAsync(sv.r, r_ext.data(), m * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    PG_CK(cudaMemcpyAsync(sv.c, c_ext.data(), m * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    ctl.alloc(1);
    if (!hctl) hctl = hctl_buf.get();
    std::memset(hctl, 0, sizeof(SinkCtl));
    hctl->n = n;
    hctl->max_iterations = cfg.max_iterations;
    hctl->pause_at = INT64_MAX;
    hctl->log_every = cfg.log_every;
    hctl->trace_cap = trace_cap;
    hctl->tol = tol;
    hctl->corner = -A / gamma;
    hctl->status = ST_RUNNING;
    hctl->g_active = 1;
    PG_CK(cudaMemcpyAsync(ctl.p, hctl, sizeof(SinkCtl), cudaMemcpyHostToDevice, cx.stream));
    k_sk_stamp<<<1, 1, 0, cx.stream>>>(ctl.p);
    // B at u = v = 0 and E (solvers.hpp:441-442), record(0)
    row_lse(nullptr);
    col_lse(0, nullptr);
    launch_k(k_sk_scalars, dim3(1), dim3(kVecThreads), 0, cx.stream, ctl.p, sv, sk_blocks(), 1, ws.trace.p, nullptr);
    PG_CK(cudaGetLastError());
    sync_ctl();
    if (cfg.record_rounded_cost) fill_last_record_cost(round_now(nullptr).cost);
    if (cfg.use_graphs) {
      cudaGraph_t graph;
      PG_CK(cudaStreamBeginCapture(cx.stream, cudaStreamCaptureModeThreadLocal));
      enqueue_iteration();
      PG_CK(cudaStreamEndCapture(cx.stream, &graph));
      size_t nodes = 0;
      PG_CK(cudaGraphGetNodes(graph, nullptr, &nodes));
      graph_nodes = int64_t(nodes);
      PG_CK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
    }
  }

  void launch_iterations(int64_t k) {
    for (int64_t i = 0; i < k; ++i) {
      if (exec) PG_CK(cudaGraphLaunch(exec, cx.stream));
      else enqueue_iteration();
      launches += graph_nodes;
    }
  }

  void run_until(int64_t stop) {
    launch_k(k_sk_resume, dim3(1), dim3(1), 0, cx.stream, ctl.p, stop);
    launches += 1;
    int64_t burst = (stop == INT64_MAX || stop - hctl->it > 4096) ? std::max(1, cfg.sync_every)
                                                                   : std::max<int64_t>(1, stop - hctl->it);
    while (true) {
      launch_iterations(burst);
      PG_CK(cudaEventRecord(ev1, cx.stream));
      sync_ctl();
      if (!hctl->g_active || hctl->fatal) break;
      burst = std::max(1, cfg.sync_every);
      if (stop != INT64_MAX) burst = std::max<int64_t>(1, std::min<int64_t>(burst, stop - hctl->it));
    }
  }

  void fill_last_record_cost(double cost) {
    const int64_t k = std::min(hctl->trace_len, hctl->trace_cap) - 1;
    if (k < 0) return;
    TraceDev last;
    PG_CK(cudaMemcpy(&last, ws.trace.p + k, sizeof(TraceDev), cudaMemcpyDeviceToHost));
    if (last.t != hctl->it || !std::isnan(last.rounded_cost)) return;
    last.rounded_cost = cost;
    PG_CK(cudaMemcpy(ws.trace.p + k, &last, sizeof(TraceDev), cudaMemcpyHostToDevice));
  }

  void iterate(int64_t k, double* ms, int64_t* iters, int* finished) override {
    if (trivial || (!hctl->g_active && !hctl->paused)) {
      if (ms) *ms = 0.0;
      if (iters) *iters = 0;
      if (finished) *finished = 1;
      return;
    }
    const int64_t t0 = hctl->it;
    const int64_t target = k < 0 ? INT64_MAX : t0 + k;
    PG_CK(cudaEventRecord(ev0, cx.stream));
    while (true) {
      int64_t stop = target;
      if (cfg.record_rounded_cost) stop = std::min(stop, (hctl->it / cfg.log_every + 1) * cfg.log_every);
      run_until(stop);
      if (hctl->fatal) break;
      if (cfg.record_rounded_cost && hctl->paused) fill_last_record_cost(round_now(nullptr).cost);
      if (!hctl->paused || hctl->it >= target) break;
    }
    PG_CK(cudaEventSynchronize(ev1));
    float f = 0.f;
    PG_CK(cudaEventElapsedTime(&f, ev0, ev1));
    if (ms) *ms = double(f);
    if (iters) *iters = hctl->it - t0;
    if (finished) *finished = hctl->paused ? 0 : 1;
  }

  // finish_extended_solve (solvers.hpp:492-509): round_balanced(B, r_ext,
  // c_ext) -> extract_block -> round_pot(block, in), all on the implicit plan.
  PlanResult round_now(double* Xdev) {
    const int64_t n = P.n;
    const size_t m = size_t(n + 1), nn = size_t(n);
    HVec u(m), v(m);
    PG_CK(cudaMemcpy(u.data(), sv.u, m * sizeof(double), cudaMemcpyDeviceToHost));
    PG_CK(cudaMemcpy(v.data(), sv.v, m * sizeof(double), cudaMemcpyDeviceToHost));
    // the block point (u[0..n), v[0..n), 0)
    PG_CK(cudaMemsetAsync(zf.p, 0, size_t(ws.slot_stride) * sizeof(double), cx.stream));
    PG_CK(cudaMemcpyAsync(zf.p, u.data(), nn * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    PG_CK(cudaMemcpyAsync(zf.p + n, v.data(), nn * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    const auto eex = [](double x) { return std::exp(std::min(std::max(x, kExpLo), kExpHi)); };
    // dummy entries of B = exp((logK + u_i) + v_j): logK = -0 off the corner
    HVec D(nn), R(nn);
    for (size_t i = 0; i < nn; ++i) D[i] = eex((-0.0 + u[i]) + v[n]);
    for (size_t j = 0; j < nn; ++j) R[j] = eex((-0.0 + u[n]) + v[j]);
    const double c0 = eex((-A / gamma + u[n]) + v[n]);
    PlanEngine pe(cx, P, ws, gamma);
    const Slot z = zf_slot();
    // round_balanced (rounding.hpp:14-39)
    HVec rb, cb;
    pe.block_sums(z, nullptr, nullptr, rb, cb);
    HVec rowE(m), f(m, 1.0);
    for (size_t i = 0; i < nn; ++i) rowE[i] = rb[i] + D[i];
    rowE[nn] = hsum(R) + c0;
    for (size_t i = 0; i < m; ++i)
      if (rowE[i] > 0) f[i] = std::min(1.0, r_ext[i] / rowE[i]);
    HVec lf(nn);
    for (size_t i = 0; i < nn; ++i) lf[i] = std::log(f[i]);
    HVec rr, cc;
    pe.block_sums(z, &lf, nullptr, rr, cc);
    HVec colE(m), g(m, 1.0), fD(nn);
    for (size_t j = 0; j < nn; ++j) colE[j] = cc[j] + f[nn] * R[j];
    for (size_t i = 0; i < nn; ++i) fD[i] = f[i] * D[i];
    colE[nn] = hsum(fD) + f[nn] * c0;
    for (size_t j = 0; j < m; ++j)
      if (colE[j] > 0) g[j] = std::min(1.0, c_ext[j] / colE[j]);
    HVec lg(nn);
    for (size_t j = 0; j < nn; ++j) lg[j] = std::log(g[j]);
    HVec rfg, cfg2;
    pe.block_sums(z, &lf, &lg, rfg, cfg2);
    HVec err_r(m), err_c(m), fRg(nn);
    for (size_t i = 0; i < nn; ++i) err_r[i] = r_ext[i] - (rfg[i] + f[i] * D[i] * g[nn]);
    for (size_t j = 0; j < nn; ++j) fRg[j] = f[nn] * R[j] * g[j];
    err_r[nn] = r_ext[nn] - (hsum(fRg) + f[nn] * c0 * g[nn]);
    for (size_t j = 0; j < m; ++j) err_c[j] = c_ext[j] - g[j] * colE[j];
    const double total = hsum(err_r);
    // extract_block (extend.hpp:55) + round_pot(block, in) (solvers.hpp:499)
    HVec P0(f.begin(), f.begin() + long(nn)), Q0(g.begin(), g.begin() + long(nn));
    if (total > 0) {
      HVec a(nn), b(nn);
      for (size_t i = 0; i < nn; ++i) a[i] = err_r[i];
      for (size_t j = 0; j < nn; ++j) b[j] = err_c[j] / total;
      return round_pot_implicit(pe, z, P0, Q0, rfg, &a, &b, P.r, P.c, P.s, Xdev);
    }
    return round_pot_implicit(pe, z, P0, Q0, rfg, nullptr, nullptr, P.r, P.c, P.s, Xdev);
  }

  void stats(int64_t* attempts, int64_t* sweeps) override {
    if (trivial) { *attempts = 0; *sweeps = 0; return; }
    sync_ctl();
    *attempts = hctl->it;
    *sweeps = hctl->sweeps;
  }

  PlanResult final_plan(double* Xdev) override {
    if (trivial) throw Error(POTGPU_ERR_UNSUPPORTED, "trivial solve has no device plan");
    return round_now(Xdev);
  }
  Slot plan_point() override { return zf_slot(); }
  Workspace& workspace() override { return ws; }
  double gamma_value() const override { return gamma; }
  int64_t iterations_done() override {
    if (trivial) return 0;
    sync_ctl();
    return hctl->it;
  }
  int status_code() override {
    if (trivial) return POTGPU_CONVERGED;
    sync_ctl();
    return hctl->status;
  }

  double time_sweep(int reps, double* elems, double* bytes) override {
    if (trivial) throw Error(POTGPU_INVALID_ARGUMENT, "trivial solve has no sweep");
    col_lse(0, nullptr);
    int64_t rows = 0;
    auto sweeps = [&] {
      rows = 0;
      const bool fast = fast_cols();
      if (!cx.comm.sharded()) {
        if (fast) launch_sweep(cx, P, ws, zuv_slot(), nullptr, nullptr, nullptr, false, gamma);
        else col_sweep(nullptr, nullptr);
        rows = P.n;
        return;
      }
      for (const ShardGrid& sh : ws.shards) {
        if (fast) launch_sweep(cx, P, ws, zuv_slot(), nullptr, nullptr, nullptr, false, gamma, &sh);
        else col_sweep(nullptr, &sh);
        rows += sh.hi - sh.lo;
      }
    };
    PG_CK(cudaEventRecord(ev0, cx.stream));
    for (int k = 0; k < reps; ++k) sweeps();
    PG_CK(cudaEventRecord(ev1, cx.stream));
    PG_CK(cudaEventSynchronize(ev1));
    float fms = 0.f;
    PG_CK(cudaEventElapsedTime(&fms, ev0, ev1));
    const double n = double(P.n);
    if (elems) *elems = double(rows) * n;
    if (bytes) *bytes = double(rows) * n * stream_bytes_per_elem(P);
    return double(fms) / reps;
  }

  void finish(potgpu_summary* sm, potgpu_outputs* out) override {
    const int64_t n = P.n;
    if (trivial) {
      fill_trivial(P, trivial_gamma, trivial_plan, sm, out, cfg);
      return;
    }
    const bool stopped_early = hctl->paused != 0;  // as a solve with max_iterations = it
    DevBuf<double> Xd;
    const bool mat = cfg.materialize_plan && out && out->X;
    if (mat) Xd.alloc(size_t(n * n));
    const PlanResult pr = round_now(mat ? Xd.p : nullptr);
    sync_ctl();
    const double wall = secs(t_start);
    sm->status = stopped_early ? POTGPU_MAX_ITERATIONS_EXCEEDED : hctl->status;
    sm->iterations = hctl->it;
    sm->gamma = gamma;
    sm->tolerance = tol;
    sm->final_error = hctl->error;
    sm->wall_seconds = wall;
    sm->loop_seconds = hctl->loop_end_ns > hctl->t0_ns ? double(hctl->loop_end_ns - hctl->t0_ns) * 1e-9 : 0.0;
    sm->has_bounds = 0;
    sm->cost = pr.cost;
    sm->feasibility_gap = pr.gap;
    sm->mass = pr.mass;
    sm->phi = hctl->phi;
    sm->iter_log_len = 0;
    sm->sweeps = hctl->sweeps;
    sm->attempts = hctl->it;
    std::strncpy(sm->stopping_iterate, "extended-marginals", sizeof(sm->stopping_iterate));
    if (cfg.record_rounded_cost) fill_last_record_cost(pr.cost);
    const int64_t tl = std::min(hctl->trace_len, hctl->trace_cap);
    if (out && out->trace && out->trace_cap > 0) {
      const int64_t k = std::min(tl, out->trace_cap);
      std::vector<TraceDev> tr(size_t(std::max<int64_t>(k, 1)));
      if (k > 0) PG_CK(cudaMemcpy(tr.data(), ws.trace.p, size_t(k) * sizeof(TraceDev), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < k; ++i)
        out->trace[i] = potgpu_trace_record{tr[size_t(i)].t, tr[size_t(i)].error, tr[size_t(i)].phi, tr[size_t(i)].rounded_cost,
                                            tr[size_t(i)].elapsed_s};
    }
    sm->trace_len = tl;
    if (out) {
      if (out->row_slack) std::memcpy(out->row_slack, pr.row_slack.data(), size_t(n) * sizeof(double));
      if (out->col_slack) std::memcpy(out->col_slack, pr.col_slack.data(), size_t(n) * sizeof(double));
      if (out->u) PG_CK(cudaMemcpy(out->u, sv.u, size_t(n + 1) * sizeof(double), cudaMemcpyDeviceToHost));
      if (out->v) PG_CK(cudaMemcpy(out->v, sv.v, size_t(n + 1) * sizeof(double), cudaMemcpyDeviceToHost));
      if (out->w) *out->w = 0.0;
      if (mat) PG_CK(cudaMemcpy(out->X, Xd.p, size_t(n * n) * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
};

inline std::unique_ptr<Session> make_sinkhorn_session(Context& c, int kind, int64_t trace_cap) {
  auto s = std::make_unique<SinkhornSession>(c, kind);
  s->trace_cap = std::max<int64_t>(trace_cap, 0) + 1;
  return s;
}

}  // namespace potgpu
