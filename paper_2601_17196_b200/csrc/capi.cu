// capi.cu — the C-ABI (include/potgpu.h): context, problem upload and
// validation, the accelerated solver driver, dual evaluation.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <functional>
#include <mutex>
#include <thread>
#include <type_traits>

#include "engine.cuh"
#include "plan.cuh"
#include "batch_cluster.cuh"

namespace potgpu {

thread_local std::string g_last_error;

// ------------------------------------------------------------------ setup --
template <class S>
__global__ void k_dense_prepare(const S* __restrict__ src, int64_t n, int64_t ldc, int row_major, int64_t ld,
                                double* C64, float* C32, unsigned long long* flags) {
  // flags[0]: non-finite, flags[1]: negative, flags[2]: max (bit pattern, >= 0 values)
  const int64_t total = n * ld;
  unsigned long long nf = 0, neg = 0, mx = 0;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = k / ld, j = k % ld;
    double x = 0.0;
    if (j < n) {
      if (!src) x = double(C32[k]);  // rescan of an already stored fp32 matrix
      else x = double(row_major ? src[i * ldc + j] : src[i + j * ldc]);
      if (C32) x = double(float(x));  // fp32 instances: every semantic on the rounded value
      if (!isfinite(x)) nf = 1;
      else if (x < 0) neg = 1;
      else mx = max(mx, (unsigned long long)__double_as_longlong(x));
    }
    if (C64) C64[k] = x;
    if (C32) C32[k] = float(x);
  }
  if (nf) atomicOr(&flags[0], 1ULL);
  if (neg) atomicOr(&flags[1], 1ULL);
  if (mx) atomicMax(&flags[2], mx);
}

// logK = -C / gamma (dual.hpp:67, IEEE division); padding columns -inf.
__global__ void k_build_logk(const double* __restrict__ C64, int64_t n, int64_t ld, double gamma, double* L) {
  const int64_t total = n * ld;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t j = k % ld;
    L[k] = j < n ? (-C64[k]) / gamma : -INFINITY;
  }
}

// max_ij |x_i - y_j|^2 under the fp64 formula of the cost views
// (ElemPointsF32::cost), in two fp32 passes instead of one fp64 pass over
// the n^2 pairs (the fp64 pass was bound by the F2F conversions: 0.74 ms at
// n = 16384). Pass 1 takes the fp32 maximum M of the same difference-square
// sums (nonnegative terms: relative error below 12 * 2^-24 of the fp64 value);
// pass 2 re-evaluates in fp64 only the pairs whose fp32 value reaches
// M (1 - 2^-18), a set that contains every maximising pair (only rows whose
// fp32 maximum reaches it are rescanned). Result: the
// exact fp64 maximum (bit pattern, atomicMax over nonnegative doubles).
// Grid: (row blocks of 256, column slices); Y staged in shared memory.
constexpr int kPmaxCols = 256;
__device__ __forceinline__ float d2_f32(const float4& a, const float4& b) {
  const float dx = __fsub_rn(a.x, b.x), dy = __fsub_rn(a.y, b.y), dz = __fsub_rn(a.z, b.z);
  return __fadd_rn(__fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy)), __fmul_rn(dz, dz));
}

__device__ __noinline__ unsigned long long d2_f64_bits(const float4* X, const float4* Y, int64_t i, int64_t j) {
  const ElemPointsF32 el{X, Y, 1.0, 1.0};
  return (unsigned long long)__double_as_longlong(el.cost(i, j));
}

// EXACT = false: fp32 maxima per row (rowmax, bit patterns of nonnegative
// floats) and overall (out32). EXACT = true: only rows whose fp32 maximum
// reaches the threshold are rescanned; their candidate pairs in fp64.
template <bool EXACT>
__global__ void __launch_bounds__(256) k_points_max2(const float4* X, const float4* Y, int64_t n, unsigned* rowmax,
                                                     unsigned* out32, unsigned long long* out64) {
  __shared__ float4 sY[kPmaxCols];
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t per = (n + gridDim.y - 1) / gridDim.y;
  const int64_t c0 = int64_t(blockIdx.y) * per, c1 = min(n, c0 + per);
  const float4 a = i < n ? X[i] : make_float4(0.f, 0.f, 0.f, 0.f);
  const float thr = EXACT ? __uint_as_float(*out32) * (1.0f - 0x1p-18f) : 0.f;
  const bool active = i < n && (!EXACT || __uint_as_float(rowmax[i]) >= thr);
  if (EXACT && !__syncthreads_or(active)) return;  // no candidate row in this block
  float m = 0.f;
  unsigned long long mx = 0;
  for (int64_t j0 = c0; j0 < c1; j0 += kPmaxCols) {
    const int cnt = c1 - j0 < kPmaxCols ? int(c1 - j0) : kPmaxCols;
    __syncthreads();
    if (threadIdx.x < cnt) sY[threadIdx.x] = Y[j0 + threadIdx.x];
    __syncthreads();
    if (active) {
      for (int k = 0; k < cnt; ++k) {
        const float d = d2_f32(a, sY[k]);
        if (!EXACT) m = fmaxf(m, d);
        else if (d >= thr) mx = max(mx, d2_f64_bits(X, Y, i, j0 + k));
      }
    }
  }
  if (!EXACT) {
    if (i < n && m > 0.f) atomicMax(rowmax + i, __float_as_uint(m));
    m = warp_maxf(m);
    if ((threadIdx.x & 31) == 0 && m > 0.f) atomicMax(out32, __float_as_uint(m));
  } else if (mx) {
    atomicMax(out64, mx);
  }
}

__global__ void k_points_store(const float4* X, const float4* Y, int64_t n, int64_t ld, double scale, double* C64,
                               float* C32) {
  ElemPointsF32 el{X, Y, scale, 1.0};
  const int64_t total = n * ld;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = k / ld, j = k % ld;
    const double c = j < n ? el.cost(i, j) : 0.0;
    if (C64) C64[k] = c;
    if (C32) C32[k] = float(c);
  }
}

// Host dense cost -> device through two pinned staging chunks (the copy of
// chunk k + 1 into pinned memory overlaps the DMA of chunk k). fp32
// instances are rounded to float on the host (every semantic of an fp32
// instance is on the rounded value, k_dense_prepare), halving the bytes over
// the link. Each batched worker stages its own problems, so uploads proceed
// in parallel instead of through the driver's pageable-copy path one at a
// time (configs[4]: 256 x 33.5 MB).
template <class T>
static void upload_dense_host(Context& cx, const double* C, int64_t count, T* dst) {
  constexpr int64_t kChunk = int64_t(1) << 20;  // elements per staging chunk
  void* stage[2] = {BlockCache::get().alloc(kChunk * sizeof(T), true), BlockCache::get().alloc(kChunk * sizeof(T), true)};
  cudaEvent_t ev[2];
  PG_CK(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
  PG_CK(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
  for (int64_t off = 0, k = 0; off < count; off += kChunk, ++k) {
    const int b = int(k & 1);
    const int64_t m = std::min(kChunk, count - off);
    if (k >= 2) PG_CK(cudaEventSynchronize(ev[b]));
    T* h = static_cast<T*>(stage[b]);
    if constexpr (std::is_same<T, double>::value) std::memcpy(h, C + off, size_t(m) * sizeof(double));
    else for (int64_t e = 0; e < m; ++e) h[e] = float(C[off + e]);
    PG_CK(cudaMemcpyAsync(dst + off, h, size_t(m) * sizeof(T), cudaMemcpyHostToDevice, cx.stream));
    PG_CK(cudaEventRecord(ev[b], cx.stream));
  }
  PG_CK(cudaEventSynchronize(ev[0]));
  PG_CK(cudaEventSynchronize(ev[1]));
  cudaEventDestroy(ev[0]);
  cudaEventDestroy(ev[1]);
  BlockCache::get().free(stage[0], kChunk * sizeof(T), true);
  BlockCache::get().free(stage[1], kChunk * sizeof(T), true);
}

// device_ptrs inputs: order the context stream (non-blocking) after the
// producer's writes (potgpu_problem.producer_stream, CAI v3 convention).
static void wait_for_producer(Context& cx, int64_t ps) {
  if (ps == -1) return;
  if (ps == 0) {
    PG_CK(cudaDeviceSynchronize());
    return;
  }
  cudaStream_t s = ps == 1 ? cudaStreamLegacy : ps == 2 ? cudaStreamPerThread : reinterpret_cast<cudaStream_t>(ps);
  cudaEvent_t ev;
  PG_CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  PG_CK(cudaEventRecord(ev, s));
  PG_CK(cudaStreamWaitEvent(cx.stream, ev, 0));
  PG_CK(cudaEventDestroy(ev));
}

static void upload_problem(Context& cx, const potgpu_problem* pr, DevProblem& P) {
  if (!pr) throw Error(POTGPU_INVALID_ARGUMENT, "null problem");
  const int64_t n = pr->n;
  const bool dev = pr->device_ptrs != 0;  // r, c, C, X, Y are device pointers (e.g. CUDA tensors)
  if (dev) wait_for_producer(cx, pr->producer_stream);
  // validation_report (core.hpp:131-169): report the FIRST violation's code.
  if (n <= 0) throw Error(POTGPU_EMPTY_INPUT, "invalid instance: marginals are empty");
  if (!pr->r || !pr->c) throw Error(POTGPU_INVALID_ARGUMENT, "null marginals");
  if (pr->dtype != POTGPU_F64 && pr->dtype != POTGPU_F32) throw Error(POTGPU_INVALID_ARGUMENT, "unknown dtype");
  P.n = n;
  P.dtype = pr->dtype;
  P.kind = pr->cost_kind;
  P.ld = round_up(n, kStripCols32);  // covers both strip widths
  if (dev) {  // the O(n) marginals are needed on the host (setup, rounding logic)
    P.r.resize(size_t(n));
    P.c.resize(size_t(n));
    PG_CK(cudaMemcpyAsync(P.r.data(), pr->r, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(P.c.data(), pr->c, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
  } else {
    P.r.assign(pr->r, pr->r + n);
    P.c.assign(pr->c, pr->c + n);
  }
  P.s = pr->s;
  bool finite = std::isfinite(pr->s);
  for (int64_t i = 0; i < n; ++i) finite = finite && std::isfinite(P.r[i]) && std::isfinite(P.c[i]);
  bool cnf = false, cneg = false;
  if (pr->cost_kind == POTGPU_COST_DENSE) {
    if (!pr->C) throw Error(POTGPU_DIMENSION_MISMATCH, "invalid instance: cost matrix missing");
    const int64_t ldc = pr->ldc > 0 ? pr->ldc : n;
    DevBuf<double> raw;
    DevBuf<float> raw32;
    DevBuf<unsigned long long> flags;
    flags.alloc(3);
    flags.zero(cx.stream);
    if (pr->dtype == POTGPU_F64) P.C64.alloc(size_t(n * P.ld)); else P.C32.alloc(size_t(n * P.ld));
    double* c64 = pr->dtype == POTGPU_F64 ? P.C64.p : nullptr;
    float* c32 = pr->dtype == POTGPU_F32 ? P.C32.p : nullptr;
    if (dev) {  // device_ptrs: read in place
      k_dense_prepare<double><<<cx.num_sms * 8, 256, 0, cx.stream>>>(pr->C, n, ldc, pr->row_major, P.ld, c64, c32, flags.p);
    } else if (pr->dtype == POTGPU_F32) {
      // the last row / column ends at (n - 1) ldc + n: nothing past it is read
      raw32.alloc(size_t(n * ldc));
      upload_dense_host<float>(cx, pr->C, (n - 1) * ldc + n, raw32.p);
      k_dense_prepare<float><<<cx.num_sms * 8, 256, 0, cx.stream>>>(raw32.p, n, ldc, pr->row_major, P.ld, c64, c32, flags.p);
    } else {
      raw.alloc(size_t(n * ldc));
      upload_dense_host<double>(cx, pr->C, (n - 1) * ldc + n, raw.p);
      k_dense_prepare<double><<<cx.num_sms * 8, 256, 0, cx.stream>>>(raw.p, n, ldc, pr->row_major, P.ld, c64, c32, flags.p);
    }
    PG_CK(cudaGetLastError());
    unsigned long long hf[3];
    PG_CK(cudaMemcpyAsync(hf, flags.p, sizeof(hf), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
    cnf = hf[0] != 0;
    cneg = hf[1] != 0;
    double mx;
    std::memcpy(&mx, &hf[2], sizeof(double));
    P.cmax = mx;
  } else if (pr->cost_kind == POTGPU_COST_SQEUCLIDEAN || pr->cost_kind == POTGPU_COST_SQEUCLIDEAN_STORED) {
    if (pr->cost_kind == POTGPU_COST_SQEUCLIDEAN && pr->dtype != POTGPU_F32)
      throw Error(POTGPU_ERR_UNSUPPORTED, "on-the-fly costs run in fp32 (dtype=F32)");
    if (!pr->X || !pr->Y || pr->d < 1 || pr->d > 3) throw Error(POTGPU_INVALID_ARGUMENT, "points need X, Y and 1 <= d <= 3");
    std::vector<float4> hx(static_cast<size_t>(n)), hy(static_cast<size_t>(n));
    std::vector<double> xd, yd;
    const double* Xs = pr->X;
    const double* Ys = pr->Y;
    if (dev) {  // n x d coordinates: small, staged through the host
      xd.resize(size_t(n * pr->d));
      yd.resize(size_t(n * pr->d));
      PG_CK(cudaMemcpyAsync(xd.data(), pr->X, xd.size() * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
      PG_CK(cudaMemcpyAsync(yd.data(), pr->Y, yd.size() * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
      PG_CK(cudaStreamSynchronize(cx.stream));
      Xs = xd.data();
      Ys = yd.data();
    }
    for (int64_t i = 0; i < n; ++i) {
      float a[3] = {0, 0, 0}, b[3] = {0, 0, 0};
      for (int k = 0; k < pr->d; ++k) {
        a[k] = float(Xs[i * pr->d + k]);
        b[k] = float(Ys[i * pr->d + k]);
        finite = finite && std::isfinite(a[k]) && std::isfinite(b[k]);
      }
      hx[size_t(i)] = make_float4(a[0], a[1], a[2], 0.f);
      hy[size_t(i)] = make_float4(b[0], b[1], b[2], 0.f);
    }
    P.X4.alloc(size_t(n));
    P.Y4.alloc(size_t(n));
    PG_CK(cudaMemcpyAsync(P.X4.p, hx.data(), size_t(n) * sizeof(float4), cudaMemcpyHostToDevice, cx.stream));
    PG_CK(cudaMemcpyAsync(P.Y4.p, hy.data(), size_t(n) * sizeof(float4), cudaMemcpyHostToDevice, cx.stream));
    DevBuf<unsigned long long> mx;
    DevBuf<unsigned> m32, rowmax;
    mx.alloc(1);
    mx.zero(cx.stream);
    m32.alloc(1);
    m32.zero(cx.stream);
    rowmax.alloc(size_t(n));
    rowmax.zero(cx.stream);
    {
      const unsigned rb = unsigned(ceil_div(n, int64_t(256)));
      const unsigned cs = unsigned(std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, int64_t(kPmaxCols)),
                                                                           ceil_div(int64_t(cx.num_sms) * 4, int64_t(rb)))));
      k_points_max2<false><<<dim3(rb, cs), 256, 0, cx.stream>>>(P.X4.p, P.Y4.p, n, rowmax.p, m32.p, nullptr);
      // rescan in column slices of one staging chunk: a block holding a
      // candidate row does little serial work; the others exit at once
      const unsigned cs2 = unsigned(ceil_div(n, int64_t(kPmaxCols)));
      k_points_max2<true><<<dim3(rb, cs2), 256, 0, cx.stream>>>(P.X4.p, P.Y4.p, n, rowmax.p, m32.p, mx.p);
      PG_CK(cudaGetLastError());
    }
    unsigned long long hm = 0;
    PG_CK(cudaMemcpyAsync(&hm, mx.p, sizeof(hm), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
    double maxd2;
    std::memcpy(&maxd2, &hm, sizeof(double));
    P.cost_scale = pr->cost_scale > 0 ? pr->cost_scale : (maxd2 > 0 ? 1.0 / maxd2 : 1.0);
    // max C under the fp64 formula of the cost views, max_ij (d2_ij * scale):
    // rounded multiplication by a positive scale is monotone, so it is
    // exactly (max_ij d2_ij) * scale — no second pass over the n^2 pairs
    P.cmax = maxd2 * P.cost_scale;
    if (pr->cost_kind == POTGPU_COST_SQEUCLIDEAN_STORED) {
      // materialise C = scale |x - y|^2 once (fp64 formula of the cost views)
      if (P.dtype == POTGPU_F64) P.C64.alloc(size_t(n * P.ld)); else P.C32.alloc(size_t(n * P.ld));
      k_points_store<<<cx.num_sms * 8, 256, 0, cx.stream>>>(P.X4.p, P.Y4.p, n, P.ld, P.cost_scale,
                                                            P.dtype == POTGPU_F64 ? P.C64.p : nullptr,
                                                            P.dtype == POTGPU_F32 ? P.C32.p : nullptr);
      PG_CK(cudaGetLastError());
      P.kind = POTGPU_COST_DENSE;
      if (P.dtype == POTGPU_F32) {  // every semantic on the stored (rounded) value
        DevBuf<unsigned long long> m2;
        m2.alloc(3);
        m2.zero(cx.stream);
        k_dense_prepare<float><<<cx.num_sms * 8, 256, 0, cx.stream>>>(static_cast<const float*>(nullptr), n, P.ld, 2, P.ld, nullptr, P.C32.p, m2.p);
        unsigned long long hf[3];
        PG_CK(cudaMemcpyAsync(hf, m2.p, sizeof(hf), cudaMemcpyDeviceToHost, cx.stream));
        PG_CK(cudaStreamSynchronize(cx.stream));
        std::memcpy(&P.cmax, &hf[2], sizeof(double));
      }
    }
  } else {
    throw Error(POTGPU_INVALID_ARGUMENT, "unknown cost kind");
  }
  if (!finite || cnf) throw Error(POTGPU_NON_FINITE_ENTRY, "invalid instance: non-finite entry in r, c, C or s");
  bool neg = false;
  for (int64_t i = 0; i < n; ++i) neg = neg || P.r[i] < 0 || P.c[i] < 0;
  if (neg) throw Error(POTGPU_NEGATIVE_ENTRY, "invalid instance: negative marginal entry");
  if (cneg) throw Error(POTGPU_NEGATIVE_ENTRY, "invalid instance: negative cost entry");
  if (P.s < 0) throw Error(POTGPU_NEGATIVE_ENTRY, "invalid instance: negative budget");
  if (P.s > std::min(ksum(P.r.data(), n), ksum(P.c.data(), n)) + 1e-12)
    throw Error(POTGPU_BUDGET_EXCEEDS_MASS, "invalid instance: budget exceeds min marginal mass");
}

__global__ void k_scale_points(const float4* X, int64_t n, float sc, float4* out) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 p = X[i];
    out[i] = make_float4(p.x * sc, p.y * sc, p.z * sc, 0.f);
  }
}

// 2 x' and the exact (fp64) squared norms -|x'|^2, -|y'|^2 of the scaled
// coordinates for the expanded-norm sweep (SrcPointsDotF32).
__global__ void k_dot_prep(const float4* XS, const float4* YS, int64_t n, float4* XD, double* xshift, double* yshift) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 a = XS[i], b = YS[i];
    XD[i] = make_float4(2.f * a.x, 2.f * a.y, 2.f * a.z, 0.f);
    xshift[i] = -((double(a.x) * a.x + double(a.y) * a.y) + double(a.z) * a.z);
    yshift[i] = -((double(b.x) * b.x + double(b.y) * b.y) + double(b.z) * b.z);
  }
}

// Coordinates pre-scaled by sqrt(log2 e * scale / gamma): the fp32 sweeps'
// kappa is then |x' - y'|^2 in log2 units.
void prepare_points(Context& cx, DevProblem& P, double gamma) {
  if (P.kind != POTGPU_COST_SQEUCLIDEAN || P.XS_gamma == gamma) return;
  P.XS4.alloc(size_t(P.n));
  P.YS4.alloc(size_t(P.n));
  P.XD4.alloc(size_t(P.n));
  P.xshift.alloc(size_t(P.n));
  P.yshift.alloc(size_t(P.n));
  const float sc = float(std::sqrt(kLog2e * P.cost_scale / gamma));
  k_scale_points<<<cx.num_sms * 4, 256, 0, cx.stream>>>(P.X4.p, P.n, sc, P.XS4.p);
  k_scale_points<<<cx.num_sms * 4, 256, 0, cx.stream>>>(P.Y4.p, P.n, sc, P.YS4.p);
  k_dot_prep<<<cx.num_sms * 4, 256, 0, cx.stream>>>(P.XS4.p, P.YS4.p, P.n, P.XD4.p, P.xshift.p, P.yshift.p);
  PG_CK(cudaGetLastError());
  P.XS_gamma = gamma;
}

void build_logk(Context& cx, DevProblem& P, double gamma) {
  prepare_points(cx, P, gamma);
  if (P.dtype != POTGPU_F64 || P.kind != POTGPU_COST_DENSE) return;
  if (P.L_gamma == gamma && P.L64.p) return;
  P.L64.alloc(size_t(P.n * P.ld));
  k_build_logk<<<cx.num_sms * 8, 256, 0, cx.stream>>>(P.C64.p, P.n, P.ld, gamma, P.L64.p);
  PG_CK(cudaGetLastError());
  P.L_gamma = gamma;
}

// ------------------------------------------------------- aspot_setup etc. --
struct Setup {
  double gamma = 0, eps_tilde = 0;
  std::vector<double> mr, mc;
};

// solvers.hpp:100-133
Setup aspot_setup(const DevProblem& P, double epsilon) {
  if (!(epsilon > 0) || !std::isfinite(epsilon)) throw Error(POTGPU_INVALID_ARGUMENT, "epsilon must be positive");
  const int64_t n = P.n;
  if (n < 2) throw Error(POTGPU_DEGENERATE_INSTANCE, "accelerated setup needs n >= 2 (log n vanishes)");
  Setup st;
  st.gamma = epsilon / (4.0 * std::log(double(n)));
  const double cmax = P.cmax;
  st.eps_tilde = cmax > 0 ? epsilon / (8.0 * cmax) : std::numeric_limits<double>::infinity();
  const double sr = ksum(P.r.data(), n), sc = ksum(P.c.data(), n);
  if (sr > 1) st.eps_tilde = std::min(st.eps_tilde, 8.0 * (sr - P.s) / (sr - 1.0));
  if (sc > 1) st.eps_tilde = std::min(st.eps_tilde, 8.0 * (sc - P.s) / (sc - 1.0));
  if (!(st.gamma > 0) || !std::isfinite(st.gamma)) throw Error(POTGPU_DEGENERATE_INSTANCE, "derived gamma is not positive");
  if (!(st.eps_tilde > 0))
    throw Error(POTGPU_DEGENERATE_INSTANCE, "stopping tolerance collapsed to zero (budget equals mass)");
  const double lambda = std::min(st.eps_tilde / 8.0, 0.5);
  const double nd = double(n);
  st.mr.resize(size_t(n));
  st.mc.resize(size_t(n));
  for (int64_t i = 0; i < n; ++i) {
    st.mr[size_t(i)] = (1.0 - lambda) * P.r[size_t(i)] + lambda / nd;
    st.mc[size_t(i)] = (1.0 - lambda) * P.c[size_t(i)] + lambda / nd;
  }
  return st;
}

// solvers.hpp:146-174 on the mixed marginals; returns false when undefined.
bool theory_bounds(const std::vector<double>& r, const std::vector<double>& c, double s, double cmax, double gamma,
                   double eps_prime, double* out4) {
  if (!(gamma > 0) || !std::isfinite(gamma) || !(eps_prime > 0) || !std::isfinite(eps_prime)) return false;
  const int64_t n = int64_t(r.size());
  const double sr = ksum(r.data(), n), sc = ksum(c.data(), n);
  const double M = std::max(sr, sc);
  if (!(M > s)) return false;
  double me = std::numeric_limits<double>::infinity();
  for (int64_t i = 0; i < n; ++i) me = std::min(me, std::min(r[size_t(i)], c[size_t(i)]));
  if (!(me > 0)) return false;
  const double R = cmax * M / (gamma * (M - s)) - std::log(me);
  const double mu = gamma / (sr + sc - s);
  const double L = 3.0 / mu;
  out4[0] = R; out4[1] = L; out4[2] = mu;
  out4[3] = 1.0 + std::pow(12.0 * std::sqrt(14.0 * double(n) * L) * R / eps_prime, 2.0 / 3.0);
  return true;
}



void fill_trivial(const DevProblem& P, double gamma, double plan_value, potgpu_summary* sm, potgpu_outputs* out,
                  const potgpu_config& cfg) {
  // trivial_result (solvers.hpp:240-255): plan 0 (s == 0) or [[s]] (n == 1)
  const int64_t n = P.n;
  sm->status = POTGPU_CONVERGED;
  sm->iterations = 0;
  sm->gamma = gamma;
  sm->tolerance = 0.0;
  sm->final_error = 0.0;
  sm->wall_seconds = 0.0;
  sm->loop_seconds = 0.0;
  sm->has_bounds = 0;
  sm->mass = plan_value;  // n == 1 plan [[s]] or zero plan
  double cost = 0.0;
  if (n == 1 && plan_value != 0.0) {
    // cost = C_00 * s; C_00 from the device copy
    double c00 = 0.0;
    if (P.kind == POTGPU_COST_DENSE) {
      if (P.dtype == POTGPU_F64) PG_CK(cudaMemcpy(&c00, P.C64.p, sizeof(double), cudaMemcpyDeviceToHost));
      else { float f; PG_CK(cudaMemcpy(&f, P.C32.p, sizeof(float), cudaMemcpyDeviceToHost)); c00 = f; }
    }
    cost = c00 * plan_value;
  }
  sm->cost = cost;
  sm->phi = 0.0;
  double gap = 0.0;
  for (int64_t i = 0; i < n; ++i) {
    const double rowx = n == 1 ? plan_value : 0.0;
    gap = std::max(gap, std::max(rowx - P.r[size_t(i)], 0.0));
    gap = std::max(gap, std::max(rowx - P.c[size_t(i)], 0.0));
    if (out && out->row_slack) out->row_slack[i] = P.r[size_t(i)] - rowx;
    if (out && out->col_slack) out->col_slack[i] = P.c[size_t(i)] - rowx;
  }
  sm->feasibility_gap = std::max(gap, std::fabs(plan_value - P.s));
  sm->trace_len = 1;
  sm->iter_log_len = 0;
  sm->sweeps = 0;
  sm->attempts = 0;
  std::strncpy(sm->stopping_iterate, "trivial", sizeof(sm->stopping_iterate));
  if (out && out->X && cfg.materialize_plan)
    for (int64_t k = 0; k < n * n; ++k) out->X[k] = (n == 1) ? plan_value : 0.0;
  if (out && out->trace && out->trace_cap > 0) {
    out->trace[0] = potgpu_trace_record{0, 0.0, 0.0, cost, 0.0};
  }
}

void copy_trace_and_log(Workspace& ws, const AspotCtl& hc, potgpu_outputs* out) {
  if (!out) return;
  if (out->trace && out->trace_cap > 0) {
    const int64_t k = std::min<int64_t>(std::min<int64_t>(hc.trace_len, hc.trace_cap), out->trace_cap);
    std::vector<TraceDev> tr(size_t(std::max<int64_t>(k, 1)));
    if (k > 0) PG_CK(cudaMemcpy(tr.data(), ws.trace.p, size_t(k) * sizeof(TraceDev), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < k; ++i)
      out->trace[i] = potgpu_trace_record{tr[size_t(i)].t, tr[size_t(i)].error, tr[size_t(i)].phi, tr[size_t(i)].rounded_cost,
                                          tr[size_t(i)].elapsed_s};
  }
  if (out->iter_log && out->iter_log_cap > 0) {
    const int64_t k = std::min<int64_t>(std::min<int64_t>(hc.log_len, hc.log_cap), out->iter_log_cap);
    std::vector<IterLogDev> lg(size_t(std::max<int64_t>(k, 1)));
    if (k > 0) PG_CK(cudaMemcpy(lg.data(), ws.iterlog.p, size_t(k) * sizeof(IterLogDev), cudaMemcpyDeviceToHost));
    for (int64_t i = 0; i < k; ++i) {
      const IterLogDev& e = lg[size_t(i)];
      out->iter_log[i] = potgpu_iter_log{e.t, e.halvings, e.block_hat, e.zbest_is_check, e.block_check, e.error,
                                         e.phi_check, e.phi_hat, e.theta};
    }
  }
}

// ------------------------------------------------------------ sessions --
// A solve = begin (validate, setup, first evaluation, record(0)) ->
// iterate(k) any number of times (device-resident loop, CUDA-graph replay)
// -> finish (final rounding, outputs). potgpu_solve runs all three.
struct Session {
  Context& cx;
  DevProblem P;
  potgpu_config cfg{};
  HostClock::time_point t_start;
  bool trivial = false;
  double trivial_plan = 0.0, trivial_gamma = 0.0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  explicit Session(Context& c) : cx(c) {
    PG_CK(cudaEventCreate(&ev0));
    PG_CK(cudaEventCreate(&ev1));
  }
  virtual ~Session() {
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
  }
  virtual void begin() = 0;
  virtual void iterate(int64_t k, double* ms, int64_t* iters, int* finished) = 0;
  virtual void finish(potgpu_summary* sm, potgpu_outputs* out) = 0;
  // average device time (ms) of one hot-path sweep launch; algorithmic
  // elements and HBM bytes that launch must touch
  virtual double time_sweep(int reps, double* elems, double* bytes) = 0;
  // average device time (ms) of one one-sided pass (block 0 = u, 1 = v) at the current z_check
  virtual double time_one_sided(int, int) {
    throw Error(POTGPU_ERR_UNSUPPORTED, "the one-sided pass exists for fp32 on-the-fly ASPOT only");
  }
  virtual void stats(int64_t* attempts, int64_t* sweeps) = 0;
  // for drivers that consume the plan themselves (registration): the
  // rounding of the stopping iterate, the point its implicit plan is built
  // on, the workspace / gamma of the sweeps, iterations and status
  virtual PlanResult final_plan(double* Xdev) = 0;
  virtual Slot plan_point() = 0;
  virtual Workspace& workspace() = 0;
  virtual double gamma_value() const = 0;
  virtual int64_t iterations_done() = 0;
  virtual int status_code() = 0;
  // ASPOT observer support: a dual point of the last accepted iteration and
  // its scalars (t, theta, error, phi_hat, phi_best, phi_check)
  virtual void read_state(int, double*, double*, double*, double*) {
    throw Error(POTGPU_ERR_UNSUPPORTED, "iterate state is available for the accelerated solver only");
  }
  int64_t launches = 0;  // kernels this session launched inside iterate()
};

inline double stream_bytes_per_elem(const DevProblem& P) {
  if (P.kind != POTGPU_COST_DENSE) return 0.0;
  return P.dtype == POTGPU_F64 ? 8.0 : 4.0;
}

// aspot_solve (solvers.hpp:265-385).
struct AspotSession : Session {
  Workspace ws;
  double gamma = 0;
  Setup st;
  cudaGraphExec_t exec = nullptr;       // one step attempt (host-launched per attempt)
  cudaGraphExec_t exec_first = nullptr; // resume (k_resume_pinned) + one step attempt: the first launch of a run
  PinnedObj<ResumeArgs> resume_args;
  bool one_sided = false;  // z_check' by sweep_pts1_f32 when its block is u or v (fp32 points)
  bool k1pp = false;       // ... which also forms the next z_bar (K1'')
  bool round_tail = false; // per-record rounding inside the attempt graph (record_rounded_cost)
  cudaGraphExec_t loop_exec = nullptr;  // the attempt inside a WHILE node: the whole loop in one launch
  int64_t trace_cap = 1, log_cap = 0;
  static constexpr int64_t kKernelsPerAttempt = 12;
  int64_t graph_nodes = kKernelsPerAttempt;
  explicit AspotSession(Context& c) : Session(c) {}
  ~AspotSession() override {
    cudaStreamSynchronize(cx.stream);  // before any buffer returns to the cache
    if (exec) cudaGraphExecDestroy(exec);
    if (exec_first) cudaGraphExecDestroy(exec_first);
    if (loop_exec) cudaGraphExecDestroy(loop_exec);
  }

  // The device loop: a graph whose WHILE node runs the attempt until
  // k_commit clears the condition (solve stopped or paused, or the
  // launch's attempt budget spent). One host launch per run instead of one
  // per attempt (the host launch rate bounds small problems, and batched
  // solves whose workers share the driver). Returns false (no loop graph)
  // when the driver refuses conditional nodes.
  bool build_loop_graph() {
    cudaGraph_t g = nullptr;
    if (cudaGraphCreate(&g, 0) != cudaSuccess) { cudaGetLastError(); return false; }
    cudaGraphConditionalHandle h;
    cudaGraphNodeParams cp = {};
    cudaGraphNode_t node;
    bool ok = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
    if (ok) {
      cp.type = cudaGraphNodeTypeConditional;
      cp.conditional.handle = h;
      cp.conditional.type = cudaGraphCondTypeWhile;
      cp.conditional.size = 1;
      ok = cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
    }
    if (ok) {
      cudaGraph_t body = cp.conditional.phGraph_out[0];
      ok = cudaStreamBeginCaptureToGraph(cx.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
           cudaSuccess;
      if (ok) {
        enqueue_attempt(h, 1);
        ok = cudaStreamEndCapture(cx.stream, &body) == cudaSuccess;
        size_t nodes = 0;
        if (ok && cudaGraphGetNodes(body, nullptr, &nodes) == cudaSuccess) graph_nodes = int64_t(nodes);
      }
    }
    if (ok) ok = cudaGraphInstantiate(&loop_exec, g, 0) == cudaSuccess;
    cudaGraphDestroy(g);
    if (!ok) {
      cudaGetLastError();
      loop_exec = nullptr;
    }
    return ok;
  }

  // One step attempt of the halving loop (solvers.hpp:334-352) + commit.
  void enqueue_attempt(cudaGraphConditionalHandle loop = 0, int in_loop = 0) {
    AspotCtl* ctl = ws.ctl.p;
    const Slot Z = ws.slot(S_Z), ZC = ws.slot(S_ZC), ZB = ws.slot(S_ZB), G = ws.slot(S_G), ZG = ws.slot(S_ZG),
               ZH = ws.slot(S_ZH), ZN = ws.slot(S_ZN);
    const int gv = ws.gv;
    // z_bar of a new iteration was formed by the previous attempt's k_commit
    // (0 at the start: z = z_check = 0). Each evaluation defers its decision
    // to the O(n) kernel that follows it (Pending, aspot_kernels.cuh).
    const Pending pd = pending_of(ws);
    // (K1'': no sweep when the previous attempt's fused pass left z_bar's partials)
    launch_eval(cx, ws, sweep_point(cx, P, ws, ZB, nullptr, nullptr, &ctl->g_bar_sweep, true, gamma), ZB, R_BAR,
                &ctl->g_new, nullptr, true, &ctl->g_bar_stash);
    launch_k(k_zgrave, dim3(gv), dim3(kVecThreads), 0, cx.stream, ctl, ZB, Z, G, ZG, ws.row(R_BAR), ws.col(R_BAR), ws.rt.p,
             ws.ct.p, pd);
    launch_eval(cx, ws, sweep_point(cx, P, ws, ZG, nullptr, nullptr, &ctl->g_alive, true, gamma), ZG, R_GRAVE,
                &ctl->g_alive, nullptr, true);
    // decides z_grave's block; forms z_hat, and when z_hat only differs in w
    // (~all iterations) also its scaled sums B(z_grave) e^dw and functionals
    launch_k(k_gk_update, dim3(gv), dim3(kVecThreads), 0, cx.stream, ctl, 0, ZG, ws.row(R_GRAVE), ws.col(R_GRAVE), R_GRAVE,
             ZG, ws.row(R_GRAVE), ws.col(R_GRAVE), R_GRAVE, ZH, ws.rt.p, ws.ct.p, ws.row(R_HAT), ws.col(R_HAT), pd,
             BarStash{});
    launch_eval(cx, ws, sweep_point(cx, P, ws, ZH, nullptr, nullptr, &ctl->g_hat_sweep, true, gamma), ZH, R_HAT,
                &ctl->g_hat_sweep, nullptr, true);
    // decides z_hat (phi, z_best, its block); forms z_check' = GK(z_best)
    // (scaled sums and functionals when its block is w)
    launch_k(k_gk_update, dim3(gv), dim3(kVecThreads), 0, cx.stream, ctl, 1, ZH, ws.row(R_HAT), ws.col(R_HAT), R_HAT, ZC,
             ws.row(R_CHECK), ws.col(R_CHECK), R_CHECK, ZN, ws.rt.p, ws.ct.p, ws.row(R_NEW), ws.col(R_NEW), pd,
             k1pp ? BarStash{ws.slot(S_ZBN), ws.kbar.p, ws.kbar.p + P.n} : BarStash{});
    const SweepOut so_n = sweep_point(cx, P, ws, ZN, nullptr, nullptr, &ctl->g_new_sweep, true, gamma);
    if (one_sided) {
      OneSidedArgs o{ws.row(R_NEW), ws.col(R_NEW), ZH.v(), &ctl->block_check};
      if (k1pp) {  // K1'': the pass also forms the next z_bar's partials
        const Slot ZBN = ws.slot(S_ZBN);
        o.u2 = ZBN.u(); o.v2 = ZBN.v(); o.w2 = ZBN.w();
        o.kbar_row = ws.kbar.p; o.kbar_col = ws.kbar.p + P.n;
        o.rowp2 = ws.rowp2.p; o.colp2 = ws.colp2.p; o.maxp2 = ws.maxp2.p;
        o.bad = ws.stash_bad.p;
      }
      launch_one_sided(cx, P, ws, ZN, &ctl->g_new_one, o);
    }
    launch_eval(cx, ws, so_n, ZN, R_NEW, &ctl->g_new_eval, nullptr, true);
    // decides z_check' and commits the attempt
    launch_k(k_commit, dim3(gv), dim3(kVecThreads), 0, cx.stream, ctl, Z, ZC, ZH, ZN, ZB, ws.row(R_CHECK), ws.col(R_CHECK),
             ws.row(R_NEW), ws.col(R_NEW), ws.trace.p, ws.iterlog.p, pd, loop, in_loop, k1pp ? ws.stash_bad.p : nullptr);
    PG_CK(cudaGetLastError());
    // record_rounded_cost with records inside the loop: the record's rounding
    // (round_pot of B(z_check), solvers.hpp:314-315) as a gated device tail
    // of the attempt, instead of pausing the loop for a host rounding
    if (round_tail)
      enqueue_round_device(cx, P, ws, gamma, ZC, ws.row(R_CHECK), &ctl->ro, &ctl->g_record, ctl, ws.trace.p);
  }

  void sync_ctl() {
    PG_CK(cudaMemcpyAsync(ws.host_ctl, ws.ctl.p, sizeof(AspotCtl), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
  }

  // round_pot(b_matrix(ctx, z_check), in) (solvers.hpp:315, :371): on the
  // device (plan.cuh enqueue_round_device) unless a dense plan is wanted or
  // the job is sharded; `full` also returns the plan terms (registration).
  PlanResult round_now(double* Xdev, bool full = false) {
    const int64_t n = P.n;
    if (!Xdev && device_round_ok(cx, P, ws)) {
      enqueue_round_device(cx, P, ws, gamma, ws.slot(S_ZC), ws.row(R_CHECK), &ws.ctl.p->ro, nullptr, nullptr, nullptr);
      sync_ctl();
      return collect_round_device(cx, P, ws, ws.host_ctl->ro, full);
    }
    PlanEngine pe(cx, P, ws, gamma);
    HVec row0(static_cast<size_t>(n)), ones(static_cast<size_t>(n), 1.0);
    PG_CK(cudaMemcpy(row0.data(), ws.row(R_CHECK), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost));
    return round_pot_implicit(pe, ws.slot(S_ZC), ones, ones, row0, nullptr, nullptr, P.r, P.c, P.s, Xdev);
  }

  // The record appended at the current t gets its rounded cost (solvers.hpp:314-315).
  void fill_last_record_cost(double cost) {
    const AspotCtl& h = *ws.host_ctl;
    const int64_t k = std::min(h.trace_len, h.trace_cap) - 1;
    if (k < 0) return;
    TraceDev last;
    PG_CK(cudaMemcpy(&last, ws.trace.p + k, sizeof(TraceDev), cudaMemcpyDeviceToHost));
    if (last.t != h.t || !std::isnan(last.rounded_cost)) return;
    last.rounded_cost = cost;
    PG_CK(cudaMemcpy(ws.trace.p + k, &last, sizeof(TraceDev), cudaMemcpyHostToDevice));
  }

  void begin() override {
    const int64_t n = P.n;
    if (n < 2) throw Error(POTGPU_DEGENERATE_INSTANCE, "accelerated solver needs n >= 2");
    if (P.s == 0) {  // solvers.hpp:274-276
      trivial = true;
      return;
    }
    PhaseTimer pt(cx.stream);
    st = aspot_setup(P, cfg.epsilon);
    gamma = cfg.gamma_override > 0 ? cfg.gamma_override : st.gamma;
    if (!(gamma > 0) || !std::isfinite(gamma)) throw Error(POTGPU_INVALID_ARGUMENT, "gamma must be positive");
    const double step_denom = 3.0 * (ksum(st.mr.data(), n) + ksum(st.mc.data(), n) - P.s);
    pt.mark("aspot_setup (host)");
    build_logk(cx, P, gamma);
    pt.mark("build_logk / points");
    prepare_workspace(cx, P, ws, trace_cap, log_cap);
    pt.mark("prepare_workspace");
    PG_CK(cudaMemcpyAsync(ws.rt.p, st.mr.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    PG_CK(cudaMemcpyAsync(ws.ct.p, st.mc.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    ws.slots.zero(cx.stream);
    AspotCtl& h = *ws.host_ctl;
    std::memset(&h, 0, sizeof(AspotCtl));
    h.n = n;
    h.max_iterations = cfg.max_iterations;
    h.pause_at = INT64_MAX;
    h.log_every = cfg.log_every;
    h.block_rule = cfg.block_rule;
    h.trace_cap = trace_cap;
    h.log_cap = log_cap;
    h.theta = 1.0;
    h.gamma = gamma;
    h.eps_tilde = st.eps_tilde;
    h.step_denom = step_denom;
    h.s = P.s;
    h.status = ST_RUNNING;
    h.clamp_guard = P.dtype == POTGPU_F64 ? 1 : 0;
    one_sided = one_sided_supported(cx, P) && ws.pts_cs == 1;
    h.one_sided_ok = one_sided ? 1 : 0;
    k1pp = one_sided && k1pp_supported(cx, P) && ws.rowp2.p;
    h.fuse_ok = k1pp ? 1 : 0;
    h.record_rounded_cost = cfg.record_rounded_cost ? 1 : 0;
    round_tail = cfg.record_rounded_cost && cfg.use_graphs && cfg.log_every < cfg.max_iterations &&
                 device_round_ok(cx, P, ws) && !std::getenv("POTGPU_NO_ROUND_TAIL");
    PG_CK(cudaMemcpyAsync(ws.ctl.p, &h, sizeof(AspotCtl), cudaMemcpyHostToDevice, cx.stream));
    AspotCtl* ctl = ws.ctl.p;
    k_stamp_t0<<<1, 1, 0, cx.stream>>>(ctl);
    // phi_and_gradient(z_check = 0) (solvers.hpp:305) and record(0) (:320)
    const Slot ZC = ws.slot(S_ZC);
    launch_eval(cx, ws, sweep_point(cx, P, ws, ZC, nullptr, nullptr, nullptr, true, gamma), ZC, R_CHECK, nullptr);
    k_init_state<<<1, 1, 0, cx.stream>>>(ctl, ws.trace.p);
    sync_ctl();
    pt.mark("first evaluation");
    if (h.fatal) throw Error(h.fatal, "Overflow: B(z) exponent exceeds representable range at z = 0");
    if (cfg.record_rounded_cost && h.g_active) fill_last_record_cost(round_now(nullptr).cost);
    pt.mark("record(0) rounding");
    if (cfg.use_graphs && graph_loop_enabled()) build_loop_graph();
    if (cfg.use_graphs && !loop_exec) {
      cudaGraph_t graph;
      PG_CK(cudaStreamBeginCapture(cx.stream, cudaStreamCaptureModeThreadLocal));
      enqueue_attempt();
      PG_CK(cudaStreamEndCapture(cx.stream, &graph));
      size_t nodes = 0;
      PG_CK(cudaGraphGetNodes(graph, nullptr, &nodes));
      graph_nodes = int64_t(nodes);
      PG_CK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      const ResumeArgs* ra = resume_args.get();  // pinned allocation outside the capture
      PG_CK(cudaStreamBeginCapture(cx.stream, cudaStreamCaptureModeThreadLocal));
      launch_k(k_resume_pinned, dim3(1), dim3(1), 0, cx.stream, ws.ctl.p, ra);
      enqueue_attempt();
      PG_CK(cudaStreamEndCapture(cx.stream, &graph));
      PG_CK(cudaGraphInstantiate(&exec_first, graph, 0));
      cudaGraphDestroy(graph);
    }
    pt.mark("graph capture");
  }

  void launch_attempts(int64_t k) {
    for (int64_t i = 0; i < k; ++i) {
      if (exec) PG_CK(cudaGraphLaunch(exec, cx.stream));
      else enqueue_attempt();
      launches += graph_nodes;
    }
  }

  // Device loop until it pauses at `stop` or the solve stops.
  void run_until(int64_t stop) {
    AspotCtl& h = *ws.host_ctl;
    if (loop_exec) {
      while (true) {
        // an accepted iteration takes at most 61 attempts (solvers.hpp:334):
        // the budget only bounds a launch, the solve stops the loop first
        const int64_t left = std::max<int64_t>(1, std::min(stop, h.max_iterations) - h.t);
        const int64_t budget = left > (int64_t(1) << 34) ? (int64_t(1) << 40) : 64 * left + 64;
        const int64_t a0 = h.attempts;
        launch_k(k_resume, dim3(1), dim3(1), 0, cx.stream, ws.ctl.p, stop, budget);
        PG_CK(cudaGraphLaunch(loop_exec, cx.stream));
        PG_CK(cudaEventRecord(ev1, cx.stream));  // device end of the loop (before the host poll)
        sync_ctl();
        launches += 1 + (h.attempts - a0) * graph_nodes;
        if (!h.g_active || h.fatal) break;
      }
      return;
    }
    bool resumed = false;
    if (exec_first) {  // the resume travels inside the first graph launch (nothing of this session in flight)
      resume_args.get()->pause_at = stop;
      resume_args.get()->budget = 0;
    } else {
      launch_k(k_resume, dim3(1), dim3(1), 0, cx.stream, ws.ctl.p, stop, int64_t(0));
      resumed = true;
    }
    launches += 1;
    // first burst: exactly the iterations asked for (1 attempt each unless a
    // step is halved), then poll every sync_every attempts
    // (a distant stop, e.g. the next record of a large log_every, polls every
    // sync_every attempts like an unbounded run)
    int64_t burst = (stop == INT64_MAX || stop - h.t > 4096) ? std::max(1, cfg.sync_every)
                                                              : std::max<int64_t>(1, stop - h.t);
    while (true) {
      if (!resumed) {
        PG_CK(cudaGraphLaunch(exec_first, cx.stream));
        launches += graph_nodes;
        resumed = true;
        if (burst > 1) launch_attempts(burst - 1);
      } else {
        launch_attempts(burst);
      }
      PG_CK(cudaEventRecord(ev1, cx.stream));  // device end of the loop (before the host poll)
      sync_ctl();
      if (!h.g_active || h.fatal) break;
      burst = std::max(1, cfg.sync_every);
      if (stop != INT64_MAX) burst = std::max<int64_t>(1, std::min<int64_t>(burst, stop - h.t));
    }
  }

  void iterate(int64_t k, double* ms, int64_t* iters, int* finished) override {
    AspotCtl& h = *ws.host_ctl;
    if (probed) throw Error(POTGPU_INVALID_ARGUMENT, "time_one_sided clobbered the pass buffers: no iterate() after it");
    if (trivial || (!h.g_active && !h.paused)) {
      if (ms) *ms = 0.0;
      if (iters) *iters = 0;
      if (finished) *finished = 1;
      return;
    }
    const int64_t t0 = h.t;
    const int64_t target = k < 0 ? INT64_MAX : t0 + k;
    PG_CK(cudaEventRecord(ev0, cx.stream));
    while (true) {
      int64_t stop = target;
      if (cfg.record_rounded_cost && !round_tail) stop = std::min(stop, (h.t / cfg.log_every + 1) * cfg.log_every);
      run_until(stop);
      if (h.fatal) break;
      if (cfg.record_rounded_cost && !round_tail && h.paused) fill_last_record_cost(round_now(nullptr).cost);
      if (!h.paused || h.t >= target) break;
    }
    PG_CK(cudaEventSynchronize(ev1));
    float f = 0.f;
    PG_CK(cudaEventElapsedTime(&f, ev0, ev1));
    if (ms) *ms = double(f);
    if (iters) *iters = h.t - t0;
    if (finished) *finished = h.paused ? 0 : 1;
    if (h.fatal) throw Error(h.fatal, "device reported an error in the solve loop");
  }

  void stats(int64_t* attempts, int64_t* sweeps) override {
    if (trivial) { *attempts = 0; *sweeps = 0; return; }
    sync_ctl();
    *attempts = ws.host_ctl->attempts;
    *sweeps = ws.host_ctl->sweeps;
  }

  PlanResult final_plan(double* Xdev) override {
    if (trivial) throw Error(POTGPU_ERR_UNSUPPORTED, "trivial solve has no device plan");
    return round_now(Xdev, true);
  }
  Slot plan_point() override { return ws.slot(S_ZC); }
  void read_state(int which, double* u, double* v, double* w, double* scalars) override {
    if (trivial) throw Error(POTGPU_ERR_UNSUPPORTED, "trivial solve has no iterates");
    static const int slot_of[4] = {S_Z, S_ZC, S_ZH, S_ZG};  // z_best (= z), z_check, z_hat, z_grave
    if (which < 0 || which > 3) throw Error(POTGPU_INVALID_ARGUMENT, "point index must be 0..3");
    const Slot z = ws.slot(slot_of[which]);
    const int64_t n = P.n;
    if (u) PG_CK(cudaMemcpyAsync(u, z.u(), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    if (v) PG_CK(cudaMemcpyAsync(v, z.v(), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    if (w) PG_CK(cudaMemcpyAsync(w, z.w(), sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    sync_ctl();
    const AspotCtl& h = *ws.host_ctl;
    if (scalars) {
      scalars[0] = double(h.t);
      scalars[1] = h.theta;
      scalars[2] = h.error;
      scalars[3] = h.phi_hat;
      scalars[4] = h.phi_best;
      scalars[5] = h.phi_check;
    }
  }
  Workspace& workspace() override { return ws; }
  double gamma_value() const override { return gamma; }
  int64_t iterations_done() override {
    if (trivial) return 0;
    sync_ctl();
    return ws.host_ctl->t;
  }
  int status_code() override {
    if (trivial) return POTGPU_CONVERGED;
    sync_ctl();
    return ws.host_ctl->status;
  }

  double time_sweep(int reps, double* elems, double* bytes) override {
    if (trivial) throw Error(POTGPU_INVALID_ARGUMENT, "trivial solve has no sweep");
    const Slot ZC = ws.slot(S_ZC);
    int64_t rows = launch_local_sweeps(cx, P, ws, ZC, gamma);  // warm
    PG_CK(cudaEventRecord(ev0, cx.stream));
    for (int k = 0; k < reps; ++k) rows = launch_local_sweeps(cx, P, ws, ZC, gamma);
    PG_CK(cudaEventRecord(ev1, cx.stream));
    PG_CK(cudaEventSynchronize(ev1));
    float f = 0.f;
    PG_CK(cudaEventElapsedTime(&f, ev0, ev1));
    const double n = double(P.n);
    if (elems) *elems = double(rows) * n;
    if (bytes) *bytes = double(rows) * n * stream_bytes_per_elem(P);
    return double(f) / reps;
  }

  // Roofline probe of the one-sided pass (sweep_pts1_f32, with the K1''
  // accumulation when the session runs it): z_check' := z_check, source :=
  // z_check. Each timed launch follows an untimed full sweep of z_check, which
  // leaves the row-segment maxima the pass shifts by (the pass overwrites
  // them). The stash and partial buffers are clobbered: no iterate() after.
  bool probed = false;
  double time_one_sided(int reps, int block) override {
    if (trivial || !one_sided || (block != 0 && block != 1))
      throw Error(POTGPU_ERR_UNSUPPORTED, "the one-sided pass exists for fp32 on-the-fly ASPOT only (block 0 or 1)");
    probed = true;
    const Slot ZC = ws.slot(S_ZC);
    DevBuf<int> blk;
    blk.alloc(1);
    PG_CK(cudaMemcpyAsync(blk.p, &block, sizeof(int), cudaMemcpyHostToDevice, cx.stream));
    OneSidedArgs o{ws.row(R_CHECK), ws.col(R_CHECK), ZC.v(), blk.p};
    if (k1pp) {
      o.u2 = ZC.u(); o.v2 = ZC.v(); o.w2 = ZC.w();
      o.kbar_row = ws.row(R_CHECK); o.kbar_col = ws.col(R_CHECK);
      o.rowp2 = ws.rowp2.p; o.colp2 = ws.colp2.p; o.maxp2 = ws.maxp2.p;
      o.bad = ws.stash_bad.p;
    }
    double total = 0.0;
    for (int k = 0; k <= reps; ++k) {  // k = 0: warm
      launch_local_sweeps(cx, P, ws, ZC, gamma);
      PG_CK(cudaEventRecord(ev0, cx.stream));
      launch_one_sided(cx, P, ws, ZC, nullptr, o);
      PG_CK(cudaEventRecord(ev1, cx.stream));
      PG_CK(cudaEventSynchronize(ev1));
      float f = 0.f;
      PG_CK(cudaEventElapsedTime(&f, ev0, ev1));
      if (k > 0) total += double(f);
    }
    return total / reps;
  }

  void finish(potgpu_summary* sm, potgpu_outputs* out) override {
    const int64_t n = P.n;
    if (trivial) {
      fill_trivial(P, 0.0, 0.0, sm, out, cfg);
      return;
    }
    AspotCtl& h = *ws.host_ctl;
    // a session paused by iterate(k) finishes like a solve with
    // max_iterations = t: the loop head stopped there (MaxIterationsExceeded)
    const bool stopped_early = h.paused != 0;
    double tb[4];
    sm->has_bounds = theory_bounds(st.mr, st.mc, P.s, P.cmax, gamma, st.eps_tilde, tb) ? 1 : 0;
    if (sm->has_bounds) { sm->bound_R = tb[0]; sm->bound_L = tb[1]; sm->bound_mu_f = tb[2]; sm->iteration_bound = tb[3]; }
    // result.plan = round_pot(b_matrix(ctx, z_check), in)  (solvers.hpp:371)
    const Slot ZC = ws.slot(S_ZC);
    DevBuf<double> Xd;
    const bool mat = cfg.materialize_plan && out && out->X;
    if (mat) Xd.alloc(size_t(n * n));
    PhaseTimer pt(cx.stream);
    const PlanResult pr = round_now(mat ? Xd.p : nullptr);
    sync_ctl();
    pt.mark("final rounding");
    const double wall = secs(t_start);
    sm->status = stopped_early ? POTGPU_MAX_ITERATIONS_EXCEEDED : h.status;
    sm->iterations = h.t;
    sm->gamma = gamma;
    sm->tolerance = st.eps_tilde;
    sm->final_error = h.error;
    sm->wall_seconds = wall;
    sm->loop_seconds = h.loop_end_ns > h.t0_ns ? double(h.loop_end_ns - h.t0_ns) * 1e-9 : 0.0;
    sm->cost = pr.cost;
    sm->feasibility_gap = pr.gap;
    sm->mass = pr.mass;
    sm->phi = h.phi_check;
    sm->iter_log_len = h.log_len;
    sm->sweeps = h.sweeps;
    sm->attempts = h.attempts;
    std::strncpy(sm->stopping_iterate, "z_check", sizeof(sm->stopping_iterate));
    if (cfg.record_rounded_cost) fill_last_record_cost(pr.cost);  // record at the stopping t
    copy_trace_and_log(ws, h, out);
    int64_t tl = std::min<int64_t>(h.trace_len, h.trace_cap);
    int64_t last_t = -1;
    if (tl > 0) {
      TraceDev last;
      PG_CK(cudaMemcpy(&last, ws.trace.p + (tl - 1), sizeof(TraceDev), cudaMemcpyDeviceToHost));
      last_t = last.t;
    }
    // final record if the last one is not at t (solvers.hpp:375-383)
    if (h.trace_len == 0 || last_t != h.t) {
      if (out && out->trace && tl < out->trace_cap) out->trace[tl] = potgpu_trace_record{h.t, h.error, h.phi_check, pr.cost, wall};
      tl += 1;
    }
    sm->trace_len = tl;
    if (out) {
      if (out->row_slack) std::memcpy(out->row_slack, pr.row_slack.data(), size_t(n) * sizeof(double));
      if (out->col_slack) std::memcpy(out->col_slack, pr.col_slack.data(), size_t(n) * sizeof(double));
      if (out->u) PG_CK(cudaMemcpy(out->u, ZC.u(), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost));
      if (out->v) PG_CK(cudaMemcpy(out->v, ZC.v(), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost));
      if (out->w) PG_CK(cudaMemcpy(out->w, ZC.w(), sizeof(double), cudaMemcpyDeviceToHost));
      if (mat) PG_CK(cudaMemcpy(out->X, Xd.p, size_t(n * n) * sizeof(double), cudaMemcpyDeviceToHost));
    }
  }
};

}  // namespace potgpu

#include "sinkhorn.cuh"
#include "registration.cuh"
#include "kmeans.cuh"
#include "dense_round.cuh"

namespace potgpu {
}  // namespace potgpu

using namespace potgpu;

struct potgpu_ctx {
  Context cx;
};

template <class F>
static int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const Error& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return POTGPU_ERR_CUDA;
  }
}

extern "C" {

int potgpu_abi_version(void) { return POTGPU_ABI_VERSION; }
const char* potgpu_last_error(void) { return g_last_error.c_str(); }

void potgpu_config_default(potgpu_config* c) {
  std::memset(c, 0, sizeof(*c));
  c->epsilon = 0.1;
  c->gamma_override = 0.0;
  c->max_iterations = 50000;
  c->block_rule = POTGPU_GREEDY;
  c->tuning_exponent_p = 1.0;
  c->deterministic = 1;
  c->log_every = 1;
  c->record_rounded_cost = 1;
  c->materialize_plan = 1;
  c->collect_iter_log = 0;
  c->use_graphs = 1;
  c->sync_every = 8;
}

int potgpu_create(int device, potgpu_ctx** out) {
  return guarded([&] {
    if (!out) throw Error(POTGPU_INVALID_ARGUMENT, "null out");
    int count = 0;
    PG_CK(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) throw Error(POTGPU_ERR_CUDA, "no such CUDA device");
    PG_CK(cudaSetDevice(device));
    auto* c = new potgpu_ctx();
    c->cx.device = device;
    PG_CK(cudaStreamCreateWithFlags(&c->cx.stream, cudaStreamNonBlocking));
    PG_CK(cudaDeviceGetAttribute(&c->cx.num_sms, cudaDevAttrMultiProcessorCount, device));
    *out = c;
  });
}

int potgpu_destroy(potgpu_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->cx.device);
    if (c->cx.comm.nccl) nccl_api().CommDestroy(c->cx.comm.nccl);
    if (c->cx.stream) cudaStreamDestroy(c->cx.stream);
    delete c;
  });
}

static void check_config(const potgpu_config& c) {  // core.hpp:250-266
  if (!(c.epsilon > 0) || !std::isfinite(c.epsilon)) throw Error(POTGPU_INVALID_ARGUMENT, "epsilon must be positive");
  if (c.max_iterations < 1) throw Error(POTGPU_INVALID_ARGUMENT, "max_iterations must be >= 1");
  if (!(c.tuning_exponent_p >= 1)) throw Error(POTGPU_INVALID_ARGUMENT, "tuning exponent p must be >= 1");
  if (c.log_every < 1) throw Error(POTGPU_INVALID_ARGUMENT, "log_every must be >= 1");
  if (c.gamma_override != 0 && !(c.gamma_override > 0)) throw Error(POTGPU_INVALID_ARGUMENT, "gamma override must be positive");
}

static std::unique_ptr<Session> make_session_cx(Context& cx, int kind, const potgpu_problem* pr,
                                                const potgpu_config* cfg_in, int64_t trace_cap, int64_t log_cap) {
  PG_CK(cudaSetDevice(cx.device));
  potgpu_config cfg;
  if (cfg_in) cfg = *cfg_in; else potgpu_config_default(&cfg);
  const auto t_start = HostClock::now();
  std::unique_ptr<Session> s;
  if (kind == POTGPU_ASPOT) {
    auto a = std::make_unique<AspotSession>(cx);
    a->trace_cap = std::max<int64_t>(trace_cap, 0) + 1;
    a->log_cap = cfg.collect_iter_log ? std::max<int64_t>(log_cap, 0) : 0;
    s = std::move(a);
  } else if (kind == POTGPU_FEASIBLE_SINKHORN || kind == POTGPU_TUNED_SINKHORN) {
    s = make_sinkhorn_session(cx, kind, trace_cap);
  } else {
    throw Error(POTGPU_INVALID_ARGUMENT, "unknown solver kind");
  }
  s->cfg = cfg;
  s->t_start = t_start;
  PhaseTimer pt(cx.stream);
  if (pr) {
    upload_problem(cx, pr, s->P);
    pt.mark("upload + validation");
  }
  check_config(cfg);
  if (pr) s->begin();  // otherwise the caller fills s->P and calls begin()
  return s;
}

static std::unique_ptr<Session> make_session(potgpu_ctx* c, int kind, const potgpu_problem* pr,
                                             const potgpu_config* cfg_in, int64_t trace_cap, int64_t log_cap) {
  if (!c) throw Error(POTGPU_INVALID_ARGUMENT, "null context");
  if (!pr) throw Error(POTGPU_INVALID_ARGUMENT, "null problem");
  return make_session_cx(c->cx, kind, pr, cfg_in, trace_cap, log_cap);
}

// ------------------------------------------------ one problem per cluster --
// BASELINE configs[4] through batch_cluster.cuh: every problem uploaded and
// set up on the host side (validation, aspot_setup, control block), then ONE
// persistent launch solves and rounds the whole batch, one problem per
// thread-block cluster. Used by potgpu_solve_batched for ASPOT on fp32
// stored costs of n <= kBcMaxN ($POTGPU_BATCH_CLUSTER=0 turns it off;
// $POTGPU_BC_CS = cluster size, default 8; $POTGPU_BC_CLUSTERS caps the
// resident clusters).
static int env_int(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e && *e ? std::atoi(e) : dflt;
}

static bool bc_wanted(int kind, const potgpu_problem* problems, int64_t count, const potgpu_config& cfg,
                      const potgpu_outputs* outputs) {
  if (env_int("POTGPU_BATCH_CLUSTER", 1) == 0 || kind != POTGPU_ASPOT || count < 1) return false;
  if (cfg.gamma_override != 0 && !(cfg.gamma_override > 0)) return false;
  for (int64_t k = 0; k < count; ++k) {
    const potgpu_problem& p = problems[k];
    if (p.dtype != POTGPU_F32 || !(p.cost_kind == POTGPU_COST_DENSE || p.cost_kind == POTGPU_COST_SQEUCLIDEAN_STORED))
      return false;
    if (p.n < 2 || p.n > kBcMaxN || !(p.s > 0)) return false;  // trivial / degenerate: the session path
    if (cfg.materialize_plan && outputs && outputs[k].X) return false;
  }
  return true;
}

struct BcHostProblem {
  DevProblem P;
  Setup st;
  double gamma = 0;
  DevBuf<double> marg;   // rt | ct | r | c
  DevBuf<double> outv;   // z_check (2n + 1) | row slack | col slack
  DevBuf<TraceDev> trace;
  DevBuf<IterLogDev> lg;
  int64_t trace_cap = 1, log_cap = 0;
  std::string err;
  int code = 0;
};

static void bc_solve_batched(Context& base, const potgpu_problem* problems, int64_t count, const potgpu_config& cfg,
                             potgpu_summary* summaries, potgpu_outputs* outputs, int concurrency) {
  const auto t_start = HostClock::now();
  check_config(cfg);
  std::vector<std::unique_ptr<BcHostProblem>> hp(static_cast<size_t>(count));
  std::vector<BcProblem> dp(static_cast<size_t>(count));
  int64_t nmax = 0;
  bool dev_inputs = false;
  for (int64_t k = 0; k < count; ++k) {
    nmax = std::max(nmax, problems[k].n);
    dev_inputs = dev_inputs || problems[k].device_ptrs != 0;
  }
  // launch geometry
  // cluster size: $POTGPU_BC_CS, else the smallest whose per-CTA rows fit
  // shared memory (every problem's CTAs stream at the per-SM rate and share
  // HBM, so more, smaller clusters win: measured C5, kernel 0.90 / 1.20 /
  // 1.96 s with 4 / 8 / 16 CTAs per cluster)
  const int64_t scap = ceil_div(nmax, int64_t(kBcStrip));
  // (measured alternatives: a per-warp cp.async.bulk ring of
  // 4 row segments streamed faster per SM with few SMs busy but was slower
  // at full load, 1.06 vs 0.84 s; two rows per warp step did not help)
  constexpr size_t kSmemMax = size_t(227) * 1024;
  const int want_nst = std::max(2, std::min(5, env_int("POTGPU_BC_STAGES", 3)));  // measured: 2-3 stages 0.90 s, 4 (225 KB smem) 1.26 s
  auto layout_of = [&](int c) {  // the deepest ring (<= want_nst, >= 2) that fits
    BcLayout l{int(ceil_div(nmax, int64_t(c))), int(scap), want_nst};
    while (l.nst > 2 && l.bytes() > kSmemMax) --l.nst;
    return l;
  };
  int cs = env_int("POTGPU_BC_CS", 0);
  if (cs <= 0) {
    cs = 16;
    for (int c : {2, 4, 8, 16})
      if (layout_of(c).bytes() <= kSmemMax && layout_of(c).nst >= std::min(want_nst, 3)) { cs = c; break; }
  }
  cs = std::max(1, std::min(16, cs));
  const BcLayout lay = layout_of(cs);
  const size_t smem = lay.bytes();
  if (smem > kSmemMax) throw Error(POTGPU_ERR_UNSUPPORTED, "cluster too small for n");
  raise_dyn_smem(k_batch_aspot, size_t(int(smem)));
  if (cs > 8) PG_CK(cudaFuncSetAttribute(k_batch_aspot, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = unsigned(cs);
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.blockDim = dim3(kBcThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = base.stream;
  lc.attrs = at;
  lc.numAttrs = 1;
  lc.gridDim = dim3(unsigned(cs * 64));
  int maxc = 0;
  PG_CK(cudaOccupancyMaxActiveClusters(&maxc, k_batch_aspot, &lc));
  if (maxc < 1) throw Error(POTGPU_ERR_UNSUPPORTED, "no resident cluster of this size");
  int nc = int(std::min<int64_t>(maxc, count));
  // $POTGPU_BC_OVERLAP=1: the uploads overlap the launch (off by default:
  // measured 2.65 s vs 1.17 s for configs[4], the upload path's device work
  // confined to the free SMs is slower than running it first); keep
  // SMs free for the upload path's own kernels (validation, layout), which
  // the resident clusters would otherwise block while waiting for them;
  // device-resident inputs may need a device synchronise: never overlapped
  const bool overlap = !dev_inputs && env_int("POTGPU_BC_OVERLAP", 0) != 0;
  if (overlap) nc = std::max(1, std::min(nc, (base.num_sms - 8) / cs));
  const int cap = env_int("POTGPU_BC_CLUSTERS", 0);
  if (cap > 0) nc = std::min(nc, cap);
  lc.gridDim = dim3(unsigned(cs * nc));
  // per-cluster workspaces
  const int64_t stride = round_up(2 * nmax + 1, 32);
  const int64_t per = kBcSlots * stride + 2 * kRoles * nmax + 8 * nmax + 2 * int64_t(cs) * kBcX;
  DevBuf<double> wsd;
  wsd.alloc(size_t(per * nc));
  DevBuf<float2> colpart;
  colpart.alloc(size_t(2 * int64_t(cs) * nmax * nc));
  std::vector<BcWs> hw(static_cast<size_t>(nc));
  for (int k = 0; k < nc; ++k) {
    double* b = wsd.p + int64_t(k) * per;
    BcWs& h = hw[size_t(k)];
    h.slots = b;
    h.sums = b + kBcSlots * stride;
    h.vec = h.sums + 2 * kRoles * nmax;
    h.xch = h.vec + 8 * nmax;
    h.colpart = colpart.p + int64_t(2 * k) * cs * nmax;
    h.colpart2 = h.colpart + int64_t(cs) * nmax;
    h.stride = stride;
    h.cur = 0;
    h.skip = 0;
  }
  // K1'': z_check' and the next z_bar in one pass over C ($POTGPU_BC_FUSE=0: separate)
  const int fuse = env_int("POTGPU_BC_FUSE", 1) != 0 ? 1 : 0;
  DevBuf<BcWs> dws;
  dws.alloc(size_t(nc));
  DevBuf<BcProblem> dprob;
  dprob.alloc(size_t(count));
  DevBuf<BcResult> dres;
  dres.alloc(size_t(count));
  DevBuf<int> queue, ready;
  queue.alloc(1);
  ready.alloc(size_t(count));
  PG_CK(cudaMemsetAsync(ready.p, 0, size_t(count) * sizeof(int), base.stream));
  cudaStream_t st = base.stream;
  PG_CK(cudaMemcpyAsync(dws.p, hw.data(), hw.size() * sizeof(BcWs), cudaMemcpyHostToDevice, st));

  PG_CK(cudaMemsetAsync(dres.p, 0, size_t(count) * sizeof(BcResult), st));
  queue.zero(st);
  auto run_uploads = [&] {
  // upload + validation + setup, `concurrency` host threads with own streams
    const int workers = int(std::max<int64_t>(1, std::min<int64_t>(concurrency > 0 ? concurrency : 8, count)));
    std::atomic<int64_t> next{0};
    std::vector<std::thread> pool;
    for (int t = 0; t < workers; ++t) {
      pool.emplace_back([&] {
        Context cx = base;
        cx.comm = Comm{};
        PG_CK(cudaSetDevice(cx.device));
        PG_CK(cudaStreamCreateWithFlags(&cx.stream, cudaStreamNonBlocking));
        int64_t k;
        while ((k = next.fetch_add(1)) < count) {
          auto h = std::make_unique<BcHostProblem>();
          try {
            upload_problem(cx, &problems[k], h->P);
            const int64_t n = h->P.n;
            h->st = aspot_setup(h->P, cfg.epsilon);
            h->gamma = cfg.gamma_override > 0 ? cfg.gamma_override : h->st.gamma;
            if (!(h->gamma > 0) || !std::isfinite(h->gamma)) throw Error(POTGPU_INVALID_ARGUMENT, "gamma must be positive");
            build_logk(cx, h->P, h->gamma);
            if (!h->P.C32.p) throw Error(POTGPU_ERR_UNSUPPORTED, "internal: no fp32 stored cost");
            h->marg.alloc(size_t(4 * n));
            PG_CK(cudaMemcpyAsync(h->marg.p, h->st.mr.data(), size_t(n) * 8, cudaMemcpyHostToDevice, cx.stream));
            PG_CK(cudaMemcpyAsync(h->marg.p + n, h->st.mc.data(), size_t(n) * 8, cudaMemcpyHostToDevice, cx.stream));
            PG_CK(cudaMemcpyAsync(h->marg.p + 2 * n, h->P.r.data(), size_t(n) * 8, cudaMemcpyHostToDevice, cx.stream));
            PG_CK(cudaMemcpyAsync(h->marg.p + 3 * n, h->P.c.data(), size_t(n) * 8, cudaMemcpyHostToDevice, cx.stream));
            h->outv.alloc(size_t(4 * n + 1));
            const potgpu_outputs* out = outputs ? &outputs[k] : nullptr;
            h->trace_cap = std::max<int64_t>(out ? out->trace_cap : 0, 0) + 1;
            h->log_cap = cfg.collect_iter_log ? std::max<int64_t>(out ? out->iter_log_cap : 0, 0) : 0;
            h->trace.alloc(size_t(h->trace_cap));
            h->lg.alloc(size_t(std::max<int64_t>(h->log_cap, 1)));
            BcProblem& b = dp[size_t(k)];
            std::memset(&b, 0, sizeof(b));
            b.C = h->P.C32.p;
            b.ld = h->P.ld;
            b.rt = h->marg.p;
            b.ct = h->marg.p + n;
            b.r = h->marg.p + 2 * n;
            b.c = h->marg.p + 3 * n;
            b.g2 = float(kLog2e / h->gamma);
            AspotCtl& c = b.ctl0;  // AspotSession::begin's control block
            c.n = n;
            c.max_iterations = cfg.max_iterations;
            c.pause_at = INT64_MAX;
            c.log_every = cfg.log_every;
            c.block_rule = cfg.block_rule;
            c.trace_cap = h->trace_cap;
            c.log_cap = h->log_cap;
            c.theta = 1.0;
            c.gamma = h->gamma;
            c.eps_tilde = h->st.eps_tilde;
            c.step_denom = 3.0 * (ksum(h->st.mr.data(), n) + ksum(h->st.mc.data(), n) - h->P.s);
            c.s = h->P.s;
            c.status = ST_RUNNING;
            c.record_rounded_cost = cfg.record_rounded_cost ? 1 : 0;
            b.trace = h->trace.p;
            b.iterlog = h->log_cap > 0 ? h->lg.p : nullptr;
            b.zc_out = h->outv.p;
            b.row_slack = h->outv.p + 2 * n + 1;
            b.col_slack = h->outv.p + 3 * n + 1;
            PG_CK(cudaStreamSynchronize(cx.stream));
            if (overlap) {  // publish: the problem record, then its ready flag (same stream: ordered)
              static const int kReady = 1;
              PG_CK(cudaMemcpyAsync(dprob.p + k, &b, sizeof(BcProblem), cudaMemcpyHostToDevice, cx.stream));
              PG_CK(cudaMemcpyAsync(ready.p + k, &kReady, sizeof(int), cudaMemcpyHostToDevice, cx.stream));
              PG_CK(cudaStreamSynchronize(cx.stream));
            }
          } catch (const Error& e) {
            h->code = e.code;
            h->err = e.what();
            if (overlap) {
              static const int kFailed = 2;
              cudaMemcpyAsync(ready.p + k, &kFailed, sizeof(int), cudaMemcpyHostToDevice, cx.stream);
              cudaStreamSynchronize(cx.stream);
            }
          }
          hp[size_t(k)] = std::move(h);
        }
        cudaStreamSynchronize(cx.stream);
        cudaStreamDestroy(cx.stream);
      });
    }
    for (auto& th : pool) th.join();
  };
  if (overlap) {
    // load the upload path's kernels now: with lazy module loading (the CUDA 12
    // default) a kernel's first launch waits for the device, here for the
    // resident clusters that are themselves waiting for that upload
    cudaFuncAttributes fa;
    PG_CK(cudaFuncGetAttributes(&fa, k_dense_prepare<double>));
    PG_CK(cudaFuncGetAttributes(&fa, k_dense_prepare<float>));
    PG_CK(cudaFuncGetAttributes(&fa, k_points_max2<false>));
    PG_CK(cudaFuncGetAttributes(&fa, k_points_max2<true>));
    PG_CK(cudaFuncGetAttributes(&fa, k_points_store));
    PG_CK(cudaFuncGetAttributes(&fa, k_scale_points));
    PG_CK(cudaFuncGetAttributes(&fa, k_dot_prep));
    PG_CK(cudaFuncGetAttributes(&fa, k_build_logk));
  } else {
    run_uploads();
  }
  const auto t_launch = HostClock::now();
  cudaEvent_t e0, e1;
  PG_CK(cudaEventCreate(&e0));
  PG_CK(cudaEventCreate(&e1));
  PG_CK(cudaEventRecord(e0, st));
  if (!overlap) {
    for (int64_t k = 0; k < count; ++k)
      if (hp[size_t(k)]->code) throw Error(hp[size_t(k)]->code, "problem " + std::to_string(k) + ": " + hp[size_t(k)]->err);
    PG_CK(cudaMemcpyAsync(dprob.p, dp.data(), dp.size() * sizeof(BcProblem), cudaMemcpyHostToDevice, st));
  }
  PG_CK(cudaLaunchKernelEx(&lc, k_batch_aspot, static_cast<const BcProblem*>(dprob.p), int(count), dws.p, dres.p,
                           queue.p, lay, fuse, overlap ? static_cast<const int*>(ready.p) : nullptr));
  PG_CK(cudaGetLastError());
  PG_CK(cudaEventRecord(e1, st));
  if (overlap) {
    run_uploads();
    for (int64_t k = 0; k < count; ++k)
      if (hp[size_t(k)]->code) {
        cudaStreamSynchronize(st);  // the launch skips the failed problem and finishes
        throw Error(hp[size_t(k)]->code, "problem " + std::to_string(k) + ": " + hp[size_t(k)]->err);
      }
  }
  std::vector<BcResult> res(static_cast<size_t>(count));
  PG_CK(cudaMemcpyAsync(res.data(), dres.p, res.size() * sizeof(BcResult), cudaMemcpyDeviceToHost, st));
  PG_CK(cudaStreamSynchronize(st));
  float kms = 0.f;
  PG_CK(cudaEventElapsedTime(&kms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (std::getenv("POTGPU_TRACE_SETUP")) {
    double sw = 0, tot = 0;
    for (const BcResult& r : res) { sw += double(r.sweep_ns); tot += double(r.total_ns); }
    std::fprintf(stderr, "[potgpu] batch cluster: per problem %.3f ms on its cluster, %.1f %% in sweeps (rank 0)\n",
                 tot / double(count) * 1e-6, tot > 0 ? 100.0 * sw / tot : 0.0);
  }
  if (std::getenv("POTGPU_TRACE_SETUP"))
    std::fprintf(stderr, "[potgpu] batch cluster: %lld problems, upload+setup %.3f ms, kernel %.3f ms (%d clusters of %d, %d-stage rings, %zu B smem)\n",
                 (long long)count, std::chrono::duration<double, std::milli>(t_launch - t_start).count(), double(kms), nc, cs,
                 lay.nst, smem);
  const double wall = secs(t_start);
  for (int64_t k = 0; k < count; ++k) {
    BcHostProblem& h = *hp[size_t(k)];
    const BcResult& r = res[size_t(k)];
    const AspotCtl& c = r.ctl;
    const int64_t n = h.P.n;
    if (!r.done) throw Error(POTGPU_ERR_CUDA, "problem " + std::to_string(k) + ": not solved by the batch kernel");
    if (c.fatal) throw Error(c.fatal, "problem " + std::to_string(k) + ": Overflow: B(z) exponent exceeds representable range at z = 0");
    if (r.infeasible) throw Error(POTGPU_INFEASIBLE, "problem " + std::to_string(k) + ": Infeasible: deficit fill has no slack mass");
    potgpu_summary* sm = &summaries[k];
    std::memset(sm, 0, sizeof(*sm));
    double tb[4];
    sm->has_bounds = theory_bounds(h.st.mr, h.st.mc, h.P.s, h.P.cmax, h.gamma, h.st.eps_tilde, tb) ? 1 : 0;
    if (sm->has_bounds) { sm->bound_R = tb[0]; sm->bound_L = tb[1]; sm->bound_mu_f = tb[2]; sm->iteration_bound = tb[3]; }
    sm->status = c.status;
    sm->iterations = c.t;
    sm->gamma = h.gamma;
    sm->tolerance = h.st.eps_tilde;
    sm->final_error = c.error;
    sm->wall_seconds = wall;  // the batch call: every problem finishes inside it
    sm->loop_seconds = c.loop_end_ns > c.t0_ns ? double(c.loop_end_ns - c.t0_ns) * 1e-9 : 0.0;
    sm->cost = r.cost;
    sm->feasibility_gap = r.gap;
    sm->mass = r.mass;
    sm->phi = c.phi_check;
    sm->iter_log_len = c.log_len;
    sm->sweeps = c.sweeps;
    sm->attempts = c.attempts;
    std::strncpy(sm->stopping_iterate, "z_check", sizeof(sm->stopping_iterate));
    potgpu_outputs* out = outputs ? &outputs[k] : nullptr;
    // trace records (+ the final record at t, solvers.hpp:375-383), iteration log
    const int64_t tl0 = std::min(c.trace_len, c.trace_cap);
    std::vector<TraceDev> tr(size_t(std::max<int64_t>(tl0, 1)));
    if (tl0 > 0) PG_CK(cudaMemcpy(tr.data(), h.trace.p, size_t(tl0) * sizeof(TraceDev), cudaMemcpyDeviceToHost));
    int64_t tl = tl0;
    const bool have_last = c.trace_len > 0 && tl0 > 0 && tr[size_t(tl0 - 1)].t == c.t;
    if (have_last && cfg.record_rounded_cost) tr[size_t(tl0 - 1)].rounded_cost = r.cost;
    if (out && out->trace)
      for (int64_t i = 0; i < std::min(tl0, out->trace_cap); ++i)
        out->trace[i] = potgpu_trace_record{tr[size_t(i)].t, tr[size_t(i)].error, tr[size_t(i)].phi,
                                            tr[size_t(i)].rounded_cost, tr[size_t(i)].elapsed_s};
    if (!have_last) {
      if (out && out->trace && tl < out->trace_cap) out->trace[tl] = potgpu_trace_record{c.t, c.error, c.phi_check, r.cost, wall};
      tl += 1;
    }
    sm->trace_len = tl;
    if (out && out->iter_log && out->iter_log_cap > 0 && h.log_cap > 0) {
      const int64_t m = std::min(std::min(c.log_len, c.log_cap), out->iter_log_cap);
      std::vector<IterLogDev> lg(size_t(std::max<int64_t>(m, 1)));
      if (m > 0) PG_CK(cudaMemcpy(lg.data(), h.lg.p, size_t(m) * sizeof(IterLogDev), cudaMemcpyDeviceToHost));
      for (int64_t i = 0; i < m; ++i) {
        const IterLogDev& e = lg[size_t(i)];
        out->iter_log[i] = potgpu_iter_log{e.t, e.halvings, e.block_hat, e.zbest_is_check, e.block_check, e.error,
                                           e.phi_check, e.phi_hat, e.theta};
      }
    }
    if (out) {
      if (out->row_slack) PG_CK(cudaMemcpy(out->row_slack, h.outv.p + 2 * n + 1, size_t(n) * 8, cudaMemcpyDeviceToHost));
      if (out->col_slack) PG_CK(cudaMemcpy(out->col_slack, h.outv.p + 3 * n + 1, size_t(n) * 8, cudaMemcpyDeviceToHost));
      if (out->u) PG_CK(cudaMemcpy(out->u, h.outv.p, size_t(n) * 8, cudaMemcpyDeviceToHost));
      if (out->v) PG_CK(cudaMemcpy(out->v, h.outv.p + n, size_t(n) * 8, cudaMemcpyDeviceToHost));
      if (out->w) PG_CK(cudaMemcpy(out->w, h.outv.p + 2 * n, 8, cudaMemcpyDeviceToHost));
    }
  }
}

// Batched independent problems (BASELINE configs[4]): `concurrency` host
// workers, each with its own CUDA stream, pull problems from a shared
// counter and run complete device-resident solves; the GPU overlaps the
// streams' kernels. No reference counterpart (the reference solves one
// instance per call).
int potgpu_solve_batched(potgpu_ctx* c, int kind, const potgpu_problem* problems, int64_t count,
                         const potgpu_config* cfg_in, potgpu_summary* summaries, potgpu_outputs* outputs, int concurrency) {
  const potgpu_config* cfg = cfg_in;
  return guarded([&] {
    if (!c || !problems || !summaries || count < 0) throw Error(POTGPU_INVALID_ARGUMENT, "null argument");
    {
      potgpu_config cfg;
      if (cfg_in) cfg = *cfg_in; else potgpu_config_default(&cfg);
      if (!c->cx.comm.sharded() && bc_wanted(kind, problems, count, cfg, outputs)) {
        PG_CK(cudaSetDevice(c->cx.device));
        bc_solve_batched(c->cx, problems, count, cfg, summaries, outputs, concurrency);
        return;
      }
    }
    const int workers = int(std::max<int64_t>(1, std::min<int64_t>(concurrency > 0 ? concurrency : 8, count)));
    std::atomic<int64_t> next{0};
    std::mutex mu;
    int first_code = 0;
    std::string first_msg;
    std::vector<std::thread> pool;
    for (int t = 0; t < workers; ++t) {
      pool.emplace_back([&] {
        Context cx = c->cx;
        // each worker plans its grids for its share of the SMs, so the
        // workers' sweeps run side by side instead of each filling the GPU
        // for a few microseconds in turn (profiles/c5_batched.py)
        cx.num_sms = std::max(1, c->cx.num_sms / workers);
        tl_no_pdl = true;
        try {
          PG_CK(cudaSetDevice(cx.device));
          PG_CK(cudaStreamCreateWithFlags(&cx.stream, cudaStreamNonBlocking));
        } catch (const Error& e) {
          std::lock_guard<std::mutex> lk(mu);
          if (!first_code) { first_code = e.code; first_msg = e.what(); }
          return;
        }
        int64_t k;
        while ((k = next.fetch_add(1)) < count) {
          try {
            potgpu_summary* sm = &summaries[k];
            std::memset(sm, 0, sizeof(*sm));
            potgpu_outputs* out = outputs ? &outputs[k] : nullptr;
            auto s = make_session_cx(cx, kind, &problems[k], cfg, out ? out->trace_cap : 0, out ? out->iter_log_cap : 0);
            s->iterate(-1, nullptr, nullptr, nullptr);
            s->finish(sm, out);
          } catch (const std::exception& e) {
            std::lock_guard<std::mutex> lk(mu);
            if (!first_code) {
              const Error* pe = dynamic_cast<const Error*>(&e);
              first_code = pe ? pe->code : POTGPU_ERR_CUDA;
              first_msg = "problem " + std::to_string(k) + ": " + e.what();
            }
          }
        }
        cudaStreamSynchronize(cx.stream);
        cudaStreamDestroy(cx.stream);
      });
    }
    for (auto& th : pool) th.join();
    if (first_code) throw Error(first_code, first_msg);
  });
}

int potgpu_solve(potgpu_ctx* c, int kind, const potgpu_problem* pr, const potgpu_config* cfg_in, potgpu_summary* sm,
                 potgpu_outputs* out) {
  return guarded([&] {
    if (!sm) throw Error(POTGPU_INVALID_ARGUMENT, "null summary");
    std::memset(sm, 0, sizeof(*sm));
    auto s = make_session(c, kind, pr, cfg_in, out ? out->trace_cap : 0, out ? out->iter_log_cap : 0);
    s->iterate(-1, nullptr, nullptr, nullptr);
    s->finish(sm, out);
  });
}

int potgpu_session_begin(potgpu_ctx* c, int kind, const potgpu_problem* pr, const potgpu_config* cfg,
                         int64_t trace_cap, int64_t iter_log_cap, potgpu_session** out) {
  return guarded([&] {
    if (!out) throw Error(POTGPU_INVALID_ARGUMENT, "null out");
    auto s = make_session(c, kind, pr, cfg, trace_cap, iter_log_cap);
    *out = reinterpret_cast<potgpu_session*>(s.release());
  });
}

int potgpu_session_iterate(potgpu_session* s, int64_t k, double* device_ms, int64_t* iterations, int* finished) {
  return guarded([&] {
    if (!s) throw Error(POTGPU_INVALID_ARGUMENT, "null session");
    reinterpret_cast<Session*>(s)->iterate(k, device_ms, iterations, finished);
  });
}

int potgpu_session_finish(potgpu_session* s, potgpu_summary* sm, potgpu_outputs* out) {
  return guarded([&] {
    if (!s || !sm) throw Error(POTGPU_INVALID_ARGUMENT, "null session or summary");
    std::memset(sm, 0, sizeof(*sm));
    reinterpret_cast<Session*>(s)->finish(sm, out);
  });
}

int potgpu_session_destroy(potgpu_session* s) {
  return guarded([&] { delete reinterpret_cast<Session*>(s); });
}

int potgpu_session_read_state(potgpu_session* s, int which, double* u, double* v, double* w, double scalars[6]) {
  return guarded([&] {
    if (!s) throw Error(POTGPU_INVALID_ARGUMENT, "null session");
    reinterpret_cast<Session*>(s)->read_state(which, u, v, w, scalars);
  });
}

int potgpu_session_time_sweep(potgpu_session* s, int reps, double* ms_per_sweep, double* elements, double* bytes) {
  return guarded([&] {
    if (!s || reps < 1) throw Error(POTGPU_INVALID_ARGUMENT, "null session or reps < 1");
    const double ms = reinterpret_cast<Session*>(s)->time_sweep(reps, elements, bytes);
    if (ms_per_sweep) *ms_per_sweep = ms;
  });
}

int potgpu_session_time_one_sided(potgpu_session* s, int reps, int block, double* ms_per_pass) {
  return guarded([&] {
    if (!s || reps < 1) throw Error(POTGPU_INVALID_ARGUMENT, "null session or reps < 1");
    const double ms = reinterpret_cast<Session*>(s)->time_one_sided(reps, block);
    if (ms_per_pass) *ms_per_pass = ms;
  });
}

int potgpu_session_stats(potgpu_session* s, int64_t* kernel_launches, int64_t* attempts, int64_t* sweeps) {
  return guarded([&] {
    if (!s) throw Error(POTGPU_INVALID_ARGUMENT, "null session");
    Session* se = reinterpret_cast<Session*>(s);
    int64_t a = 0, w = 0;
    se->stats(&a, &w);
    if (kernel_launches) *kernel_launches = se->launches;
    if (attempts) *attempts = a;
    if (sweeps) *sweeps = w;
  });
}

int potgpu_session_carry_stats(potgpu_session* s, int64_t* carried, int64_t* exact) {
  return guarded([&] {
    if (!s) throw Error(POTGPU_INVALID_ARGUMENT, "null session");
    Workspace& ws = reinterpret_cast<Session*>(s)->workspace();
    unsigned long long h[2] = {0, 0};
    if (ws.carry_stats.p) {
      PG_CK(cudaMemcpyAsync(h, ws.carry_stats.p, sizeof h, cudaMemcpyDeviceToHost, ws.stream));
      PG_CK(cudaStreamSynchronize(ws.stream));
    }
    if (carried) *carried = int64_t(h[0]);
    if (exact) *exact = int64_t(h[1]);
  });
}

void* potgpu_ctx_stream(potgpu_ctx* c) { return c ? reinterpret_cast<void*>(c->cx.stream) : nullptr; }

int potgpu_dual_eval(potgpu_ctx* c, const potgpu_problem* pr, double gamma, const double* u, const double* v, double w,
                     double* row, double* col, double* scalars) {
  int overflow = 0;
  const int rc = guarded([&] {
    if (!c) throw Error(POTGPU_INVALID_ARGUMENT, "null context");
    if (!(gamma > 0) || !std::isfinite(gamma)) throw Error(POTGPU_INVALID_ARGUMENT, "gamma must be positive");
    PG_CK(cudaSetDevice(c->cx.device));
    DevProblem P;
    upload_problem(c->cx, pr, P);
    build_logk(c->cx, P, gamma);
    Workspace ws;
    prepare_workspace(c->cx, P, ws, 1, 0);
    const int64_t n = P.n;
    const Slot Z = ws.slot(S_ZB);
    ws.slots.zero(c->cx.stream);
    PG_CK(cudaMemcpyAsync(Z.u(), u, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    PG_CK(cudaMemcpyAsync(Z.v(), v, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    PG_CK(cudaMemcpyAsync(Z.w(), &w, sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    PG_CK(cudaMemcpyAsync(ws.rt.p, P.r.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    PG_CK(cudaMemcpyAsync(ws.ct.p, P.c.data(), size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    AspotCtl& h = *ws.host_ctl;
    std::memset(&h, 0, sizeof(h));
    h.n = n;
    h.s = P.s;
    PG_CK(cudaMemcpyAsync(ws.ctl.p, &h, sizeof(h), cudaMemcpyHostToDevice, c->cx.stream));
    launch_eval(c->cx, ws, sweep_point(c->cx, P, ws, Z, nullptr, nullptr, nullptr, true, gamma), Z, R_EVAL, nullptr);
    PG_CK(cudaMemcpyAsync(&h, ws.ctl.p, sizeof(h), cudaMemcpyDeviceToHost, c->cx.stream));
    if (row) PG_CK(cudaMemcpyAsync(row, ws.row(R_EVAL), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c->cx.stream));
    if (col) PG_CK(cudaMemcpyAsync(col, ws.col(R_EVAL), size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, c->cx.stream));
    PG_CK(cudaStreamSynchronize(c->cx.stream));
    const PointScalars& ps = h.ps[R_EVAL];
    if (scalars) {
      scalars[0] = ps.total;
      scalars[1] = ps.maxe;
      scalars[2] = ps.phi;
      scalars[3] = ps.err;
      scalars[4] = ps.total - P.s;
      scalars[5] = ps.overflow;
    }
    overflow = ps.overflow;
  });
  if (rc) return rc;
  if (overflow) {
    g_last_error = "B(z) exponent exceeds representable range";
    return POTGPU_OVERFLOW;
  }
  return 0;
}

int potgpu_comm_unique_id(unsigned char id_out[128]) {
  return guarded([&] {
    if (!id_out) throw Error(POTGPU_INVALID_ARGUMENT, "null id");
    NcclUid id;
    nccl_check(nccl_api().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(id_out, id.internal, sizeof(id.internal));
  });
}

int potgpu_comm_init(potgpu_ctx* c, int rank, int world_size, const unsigned char id[128]) {
  return guarded([&] {
    if (!c || !id) throw Error(POTGPU_INVALID_ARGUMENT, "null context or id");
    if (world_size < 1 || rank < 0 || rank >= world_size) throw Error(POTGPU_INVALID_ARGUMENT, "bad rank / world size");
    if (c->cx.comm.multi()) throw Error(POTGPU_INVALID_ARGUMENT, "communicator already initialised");
    PG_CK(cudaSetDevice(c->cx.device));
    NcclUid uid;
    std::memcpy(uid.internal, id, sizeof(uid.internal));
    void* comm = nullptr;
    nccl_check(nccl_api().CommInitRank(&comm, world_size, uid, rank), "ncclCommInitRank");
    c->cx.comm.nccl = comm;
    c->cx.comm.rank = rank;
    c->cx.comm.world = world_size;
  });
}

int potgpu_comm_init_host(potgpu_ctx* c, int rank, int world_size, potgpu_host_allreduce_fn allreduce, void* user) {
  return guarded([&] {
    if (!c || !allreduce) throw Error(POTGPU_INVALID_ARGUMENT, "null context or all-reduce function");
    if (world_size < 1 || rank < 0 || rank >= world_size) throw Error(POTGPU_INVALID_ARGUMENT, "bad rank / world size");
    if (c->cx.comm.multi()) throw Error(POTGPU_INVALID_ARGUMENT, "communicator already initialised");
    c->cx.comm.host_fn = allreduce;
    c->cx.comm.host_user = user;
    c->cx.comm.rank = rank;
    c->cx.comm.world = world_size;
  });
}

int potgpu_comm_init_local(potgpu_ctx* c, int shards) {
  return guarded([&] {
    if (!c) throw Error(POTGPU_INVALID_ARGUMENT, "null context");
    if (shards < 1 || shards > 1024) throw Error(POTGPU_INVALID_ARGUMENT, "shards must be in [1, 1024]");
    c->cx.comm.vshards = shards;
  });
}

int potgpu_comm_info(potgpu_ctx* c, int* rank, int* world_size, int* shards_per_rank) {
  return guarded([&] {
    if (!c) throw Error(POTGPU_INVALID_ARGUMENT, "null context");
    if (rank) *rank = c->cx.comm.rank;
    if (world_size) *world_size = c->cx.comm.world;
    if (shards_per_rank) *shards_per_rank = c->cx.comm.vshards;
  });
}

void potgpu_release_cached_memory(void) { BlockCache::get().release_all(); }

void potgpu_reg_config_default(potgpu_reg_config* c) {  // registration.hpp:75-80
  std::memset(c, 0, sizeof(*c));
  c->alpha = 0.4;
  c->gamma0 = 4.4e-3;
  c->anneal_rate = 0.83;
  c->transform_threshold = 1e-5;
  c->max_registrations = 60;
}

static void check_reg_config(const potgpu_reg_config& c) {  // registration.hpp:83-99
  if (!(c.alpha > 0) || !(c.alpha <= 1)) throw Error(POTGPU_INVALID_ARGUMENT, "alpha must lie in (0, 1]");
  if (!(c.gamma0 > 0)) throw Error(POTGPU_INVALID_ARGUMENT, "gamma0 must be positive");
  if (!(c.anneal_rate > 0) || !(c.anneal_rate < 1)) throw Error(POTGPU_INVALID_ARGUMENT, "anneal rate must lie in (0, 1)");
  if (!(c.transform_threshold > 0)) throw Error(POTGPU_INVALID_ARGUMENT, "threshold must be positive");
  if (c.max_registrations < 1) throw Error(POTGPU_INVALID_ARGUMENT, "max_registrations must be >= 1");
}

// register_point_clouds (registration.hpp:127-199).
int potgpu_register_point_clouds(potgpu_ctx* c, int kind, const double* reference, int64_t m, const double* moving,
                                 int64_t n, const potgpu_reg_config* reg_in, const potgpu_config* solve_in, int dtype,
                                 potgpu_reg_result* res, potgpu_reg_record* records, int64_t records_cap) {
  return guarded([&] {
    if (!c || !res) throw Error(POTGPU_INVALID_ARGUMENT, "null context or result");
    if (!reference || !moving) throw Error(POTGPU_DIMENSION_MISMATCH, "point clouds must be N x 3");
    if (m < 3 || n < 3) throw Error(POTGPU_EMPTY_INPUT, "need at least 3 points per cloud");
    potgpu_reg_config rc;
    if (reg_in) rc = *reg_in; else potgpu_reg_config_default(&rc);
    check_reg_config(rc);
    potgpu_config cfg;
    if (solve_in) cfg = *solve_in; else potgpu_config_default(&cfg);
    check_config(cfg);
    if (dtype != POTGPU_F64 && dtype != POTGPU_F32) throw Error(POTGPU_INVALID_ARGUMENT, "unknown dtype");
    Context& cx = c->cx;
    PG_CK(cudaSetDevice(cx.device));
    const int64_t side = std::max(m, n);
    const double denom = double(side);
    HVec r(static_cast<size_t>(side), 0.0), cc(static_cast<size_t>(side), 0.0);
    for (int64_t i = 0; i < m; ++i) r[size_t(i)] = 1.0 / denom;
    for (int64_t j = 0; j < n; ++j) cc[size_t(j)] = 1.0 / denom;
    const double budget = rc.alpha * double(std::min(m, n)) / denom;
    DevBuf<double> refd, curd;
    DevBuf<unsigned long long> mxd;
    refd.alloc(size_t(3 * m));
    curd.alloc(size_t(3 * n));
    mxd.alloc(1);
    PG_CK(cudaMemcpyAsync(refd.p, reference, size_t(3 * m) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    Rigid T;
    double gamma = rc.gamma0;
    int64_t accumulated = 0;
    bool converged = false;
    std::vector<RegRecord> recs;
    HVec cur(static_cast<size_t>(3 * n));
    for (int round = 1; round <= rc.max_registrations; ++round) {
      // current = T.apply_all(moving) (registration.hpp:21-25)
      for (int64_t j = 0; j < n; ++j) {
        const Vec3 y{moving[3 * j], moving[3 * j + 1], moving[3 * j + 2]};
        const Vec3 ry = mat3_apply(T.R, y);
        for (int d = 0; d < 3; ++d) cur[size_t(3 * j + d)] = ry[d] + T.t[d];
      }
      PG_CK(cudaMemcpyAsync(curd.p, cur.data(), size_t(3 * n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
      mxd.zero(cx.stream);
      k_reg_d2max<<<int(std::min<int64_t>(m, 4096)), 256, 0, cx.stream>>>(refd.p, curd.p, m, n, mxd.p);
      PG_CK(cudaGetLastError());
      unsigned long long hb = 0;
      PG_CK(cudaMemcpyAsync(&hb, mxd.p, sizeof(hb), cudaMemcpyDeviceToHost, cx.stream));
      PG_CK(cudaStreamSynchronize(cx.stream));
      double cmax;
      std::memcpy(&cmax, &hb, sizeof(double));
      if (!(cmax > 0)) {  // clouds coincide (registration.hpp:160-167)
        converged = true;
        break;
      }
      if (!std::isfinite(cmax)) throw Error(POTGPU_NON_FINITE_ENTRY, "invalid instance: non-finite point coordinates");
      potgpu_config rcfg = cfg;
      rcfg.gamma_override = gamma;
      auto s = make_session_cx(cx, kind, nullptr, &rcfg, 0, 0);
      DevProblem& P = s->P;  // the padded instance, built on the device
      P.n = side;
      P.dtype = dtype;
      P.kind = POTGPU_COST_DENSE;
      P.ld = round_up(side, kStripCols32);
      P.r = r;
      P.c = cc;
      P.s = budget;
      P.cmax = 1.0;  // block max = cmax / cmax, padding = 1
      if (dtype == POTGPU_F64) P.C64.alloc(size_t(side * P.ld)); else P.C32.alloc(size_t(side * P.ld));
      k_reg_cost<<<cx.num_sms * 8, 256, 0, cx.stream>>>(refd.p, curd.p, m, n, side, P.ld, cmax,
                                                       dtype == POTGPU_F64 ? P.C64.p : nullptr,
                                                       dtype == POTGPU_F32 ? P.C32.p : nullptr);
      PG_CK(cudaGetLastError());
      s->begin();
      s->iterate(-1, nullptr, nullptr, nullptr);
      const PlanResult pr = s->final_plan(nullptr);
      const int64_t inner = s->iterations_done();
      // fit_rigid(plan.X.topLeftCorner(m, n), reference, current)
      HVec a(pr.rowx.begin(), pr.rowx.begin() + long(m)), b(pr.colx.begin(), pr.colx.begin() + long(n));
      Session* sp = s.get();
      const Rigid inc = fit_rigid_from(a, b, reference, m, cur.data(), n, [&](const HVec& xh) {
        HVec xf(static_cast<size_t>(3 * side), 0.0);
        std::copy(xh.begin(), xh.end(), xf.begin());
        PlanEngine pe(cx, sp->P, sp->workspace(), sp->gamma_value());
        HVec z = pe.moments(sp->plan_point(), pr.Pf, pr.Qf, &pr.a0, &pr.b0, pr.a1.empty() ? nullptr : &pr.a1,
                            pr.a1.empty() ? nullptr : &pr.b1, xf);
        z.resize(size_t(3 * n));
        return z;
      });
      const Rigid next = rigid_compose(inc, T);
      double dR = 0.0, dt = 0.0;
      for (int k = 0; k < 9; ++k) dR += (next.R[k] - T.R[k]) * (next.R[k] - T.R[k]);
      for (int k = 0; k < 3; ++k) dt += (next.t[k] - T.t[k]) * (next.t[k] - T.t[k]);
      const double delta = std::sqrt(dR) + std::sqrt(dt);
      T = next;
      accumulated += inner;
      recs.push_back(RegRecord{round, inner, accumulated, pr.cost, delta, gamma});
      gamma *= rc.anneal_rate;
      if (delta < rc.transform_threshold) {
        converged = true;
        break;
      }
    }
    std::memcpy(res->R, T.R.data(), sizeof(res->R));
    std::memcpy(res->t, T.t.data(), sizeof(res->t));
    res->converged = converged ? 1 : 0;
    res->rounds = int64_t(recs.size());
    if (records)
      for (int64_t k = 0; k < std::min<int64_t>(records_cap, int64_t(recs.size())); ++k) {
        const RegRecord& q = recs[size_t(k)];
        records[k] = potgpu_reg_record{q.round, q.inner, q.accumulated, q.cost, q.increment, q.gamma};
      }
  });
}

// kmeans_quantize (color_transfer.hpp:34-118).
int potgpu_kmeans_quantize(potgpu_ctx* c, const double* points, int64_t n, int k, uint64_t seed, double* centroids,
                           double* weights, int32_t* assignments) {
  return guarded([&] {
    if (!c || !centroids || !weights) throw Error(POTGPU_INVALID_ARGUMENT, "null argument");
    if (n > 0 && !points) throw Error(POTGPU_INVALID_ARGUMENT, "null points");
    PG_CK(cudaSetDevice(c->cx.device));
    kmeans_quantize(c->cx, points, n, k, seed, centroids, weights, assignments);
  });
}

// fit_rigid (registration.hpp:40-71) on a dense row-major m x n coupling.
int potgpu_fit_rigid(potgpu_ctx* c, const double* pi, int64_t m, int64_t n, const double* x, const double* y, double R[9],
                     double t[3]) {
  return guarded([&] {
    if (!c || !R || !t) throw Error(POTGPU_INVALID_ARGUMENT, "null argument");
    if (!pi || !x || !y || m < 1 || n < 1) throw Error(POTGPU_DIMENSION_MISMATCH, "coupling shape does not match the clouds");
    Context& cx = c->cx;
    PG_CK(cudaSetDevice(cx.device));
    DevBuf<double> pid, rows, cols, xhd, zd;
    pid.alloc(size_t(m * n));
    rows.alloc(size_t(m));
    cols.alloc(size_t(n));
    xhd.alloc(size_t(3 * m));
    zd.alloc(size_t(3 * n));
    PG_CK(cudaMemcpyAsync(pid.p, pi, size_t(m * n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    k_dense_rowsums<<<int(std::min<int64_t>(m, 4096)), 256, 0, cx.stream>>>(pid.p, m, n, rows.p);
    k_dense_colmoments<<<cx.num_sms, 256, 0, cx.stream>>>(pid.p, m, n, nullptr, cols.p, nullptr);
    PG_CK(cudaGetLastError());
    HVec a(static_cast<size_t>(m)), b(static_cast<size_t>(n));
    PG_CK(cudaMemcpyAsync(a.data(), rows.p, size_t(m) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaMemcpyAsync(b.data(), cols.p, size_t(n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
    const Rigid T = fit_rigid_from(a, b, x, m, y, n, [&](const HVec& xh) {
      PG_CK(cudaMemcpyAsync(xhd.p, xh.data(), size_t(3 * m) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
      k_dense_colmoments<<<cx.num_sms, 256, 0, cx.stream>>>(pid.p, m, n, xhd.p, nullptr, zd.p);
      PG_CK(cudaGetLastError());
      HVec z(static_cast<size_t>(3 * n));
      PG_CK(cudaMemcpyAsync(z.data(), zd.p, size_t(3 * n) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
      PG_CK(cudaStreamSynchronize(cx.stream));
      return z;
    });
    std::memcpy(R, T.R.data(), 9 * sizeof(double));
    std::memcpy(t, T.t.data(), 3 * sizeof(double));
  });
}

static void check_marginals(int64_t n, const double* r, const double* c, double s) {  // validate (core.hpp:131-169) on r, c, s
  if (n <= 0) throw Error(POTGPU_EMPTY_INPUT, "invalid instance: marginals are empty");
  if (!r || !c) throw Error(POTGPU_INVALID_ARGUMENT, "null marginals");
  bool finite = std::isfinite(s), neg = s < 0;
  for (int64_t i = 0; i < n; ++i) {
    finite = finite && std::isfinite(r[i]) && std::isfinite(c[i]);
    neg = neg || r[i] < 0 || c[i] < 0;
  }
  if (!finite) throw Error(POTGPU_NON_FINITE_ENTRY, "invalid instance: non-finite entry in r, c or s");
  if (neg) throw Error(POTGPU_NEGATIVE_ENTRY, "invalid instance: negative entry");
  if (s > std::min(ksum(r, n), ksum(c, n)) + 1e-12)
    throw Error(POTGPU_BUDGET_EXCEEDS_MASS, "invalid instance: budget exceeds min marginal mass");
}

// round_pot (rounding.hpp:46-77) on a dense row-major plan.
// exponent_matrix / b_matrix (dual.hpp:93-109): e_ij = ((logK_ij + u_i) + v_j) + w,
// B = exp(e) (POTGPU_OVERFLOW when max e > 700, as check_exp_range).
__global__ void k_dual_matrix(Slot z, const double* L, int64_t ld, int64_t n, int which, double* out, unsigned long long* mx) {
  unsigned long long m = 0;
  bool nan = false;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n * n; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = k / n, j = k % n;
    const double e = ((L[i * ld + j] + z.u()[i]) + z.v()[j]) + *z.w();
    out[k] = which == 0 ? e : eexp(e);
    if (e != e) nan = true;
    // order-preserving key of the double (max over signed values)
    const unsigned long long b = (unsigned long long)__double_as_longlong(e);
    const unsigned long long key = (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
    m = max(m, key);
  }
  if (nan) m = ~0ULL;
  atomicMax(mx, m);
}

int potgpu_dual_matrix(potgpu_ctx* c, const potgpu_problem* pr, double gamma, const double* u, const double* v, double w,
                       int which, double* out) {
  int overflow = 0;
  const int rc = guarded([&] {
    if (!c || !out || !u || !v) throw Error(POTGPU_INVALID_ARGUMENT, "null argument");
    if (!(gamma > 0) || !std::isfinite(gamma)) throw Error(POTGPU_INVALID_ARGUMENT, "gamma must be positive");
    if (which != 0 && which != 1) throw Error(POTGPU_INVALID_ARGUMENT, "which: 0 exponent, 1 B");
    PG_CK(cudaSetDevice(c->cx.device));
    potgpu_problem p64 = *pr;
    p64.dtype = POTGPU_F64;  // the reference's semantics
    if (p64.cost_kind == POTGPU_COST_SQEUCLIDEAN) p64.cost_kind = POTGPU_COST_SQEUCLIDEAN_STORED;
    DevProblem P;
    upload_problem(c->cx, &p64, P);
    build_logk(c->cx, P, gamma);
    const int64_t n = P.n;
    DevBuf<double> zb, ob;
    DevBuf<unsigned long long> mx;
    zb.alloc(size_t(2 * n + 1));
    ob.alloc(size_t(n * n));
    mx.alloc(1);
    mx.zero(c->cx.stream);
    PG_CK(cudaMemcpyAsync(zb.p, u, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    PG_CK(cudaMemcpyAsync(zb.p + n, v, size_t(n) * sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    PG_CK(cudaMemcpyAsync(zb.p + 2 * n, &w, sizeof(double), cudaMemcpyHostToDevice, c->cx.stream));
    k_dual_matrix<<<c->cx.num_sms * 8, 256, 0, c->cx.stream>>>(Slot{zb.p, n}, P.L64.p, P.ld, n, which, ob.p, mx.p);
    PG_CK(cudaGetLastError());
    unsigned long long key = 0;
    PG_CK(cudaMemcpyAsync(&key, mx.p, sizeof(key), cudaMemcpyDeviceToHost, c->cx.stream));
    PG_CK(cudaMemcpyAsync(out, ob.p, size_t(n * n) * sizeof(double), cudaMemcpyDeviceToHost, c->cx.stream));
    PG_CK(cudaStreamSynchronize(c->cx.stream));
    double maxe;
    if (key == ~0ULL) {
      maxe = std::numeric_limits<double>::quiet_NaN();
    } else {
      const unsigned long long b = (key >> 63) ? (key & 0x7fffffffffffffffULL) : ~key;
      std::memcpy(&maxe, &b, sizeof(double));
    }
    overflow = which == 1 && !(maxe <= kMaxExponent);
  });
  if (rc) return rc;
  if (overflow) {
    g_last_error = "Overflow: B(z) exponent exceeds representable range";
    return POTGPU_OVERFLOW;
  }
  return 0;
}

int potgpu_round_pot(potgpu_ctx* c, int64_t n, const double* X, const double* r, const double* cm, double s,
                     double* X_out) {
  return guarded([&] {
    if (!c || !X || !X_out) throw Error(POTGPU_INVALID_ARGUMENT, "null argument");
    check_marginals(n, r, cm, s);
    PG_CK(cudaSetDevice(c->cx.device));
    round_pot_dense(c->cx, n, X, HVec(r, r + n), HVec(cm, cm + n), s, X_out);
  });
}

// round_balanced (rounding.hpp:14-39) on a dense row-major rows x cols plan.
int potgpu_round_balanced(potgpu_ctx* c, int64_t rows, int64_t cols, const double* X, const double* r, const double* cm,
                          double* X_out) {
  return guarded([&] {
    if (!c || !X || !X_out || !r || !cm) throw Error(POTGPU_INVALID_ARGUMENT, "null argument");
    if (rows <= 0 || cols <= 0) throw Error(POTGPU_DIMENSION_MISMATCH, "plan/marginal shape mismatch");
    PG_CK(cudaSetDevice(c->cx.device));
    round_balanced_dense(c->cx, rows, cols, X, HVec(r, r + rows), HVec(cm, cm + cols), X_out);
  });
}

}  // extern "C"
