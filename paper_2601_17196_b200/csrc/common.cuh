// common.cuh — shared device/host internals of libpotgpu (sm_100a).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <utility>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/potgpu.h"

namespace potgpu {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

#define PG_CK(x)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (x);                                                                     \
    if (e_ != cudaSuccess)                                                                    \
      throw ::potgpu::Error(POTGPU_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// dual.hpp:47 and the Eigen packet-exp clamp (see oracle/pot_oracle.hpp eexp).
constexpr double kMaxExponent = 700.0;
constexpr double kExpLo = -709.784;
constexpr double kExpHi = 709.784;
constexpr double kLog2e = 1.4426950408889634074;
constexpr double kLn2 = 0.69314718055994530942;

// Sweep geometry: a warp owns 256 consecutive columns of a row (8 per lane),
// a CTA's 8 warps share that column strip and split the CTA's row range.
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * 32;
constexpr int kStripCols = 256;
constexpr int kVecThreads = 256;  // O(n) kernels

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t round_up(int64_t a, int64_t b) { return ceil_div(a, b) * b; }

// A dual point z = (u, v, w) lives in one slot: [u (n) | v (n) | w | pad].
struct Slot {
  double* base = nullptr;
  int64_t n = 0;
  __host__ __device__ double* u() const { return base; }
  __host__ __device__ double* v() const { return base + n; }
  __host__ __device__ double* w() const { return base + 2 * n; }
};

// Reductions of B at a point that every caller needs (dual.hpp:117-131,
// solvers.hpp:49-69, 224-232), produced by finalize kernels.
struct PointScalars {
  double total;    // 1^T B 1
  double maxe;     // max_ij exponent (NaN-propagating)
  double maxu, maxv;
  double seu, sev; // sum exp(u), sum exp(v)
  double ur, vc;   // <u, r~>, <v, c~>
  double score_u, score_v;  // sum rho(r~_i, row_i), sum rho(c~_j, col_j)
  double gl1u, gl1v;        // |grad_u|_1, |grad_v|_1
  double phi, err;
  double minrow, mincol;  // smallest entry of B 1 and B^T 1 (scaling shortcut guard)
  int overflow;
  int pad;
};
constexpr int kNumPartials = 11;  // total, maxu, maxv, seu, sev, ur, vc, score_u, score_v, gl1u, gl1v
constexpr int kNumAcc = kNumPartials + 3;  // + maxe (11), minrow (12), mincol (13)

// Process-wide caching allocator for device and pinned host blocks: a freed
// block is kept (per device, per size class) and handed to the next request
// of that class, so repeated solves pay neither cudaMalloc / cudaMallocHost
// (milliseconds each) nor cudaFree (which synchronises the device and would
// serialise the batched workers). Callers return a block only after the
// stream that used it has been synchronised (sessions do so in their
// destructors). potgpu_release_cached_memory() hands everything back.
class BlockCache {
 public:
  static BlockCache& get() {
    static BlockCache* c = new BlockCache();  // never destroyed: outlives static DevBufs
    return *c;
  }
  static size_t size_class(size_t bytes) {
    if (bytes <= (size_t(1) << 20)) {
      size_t c = 256;
      while (c < bytes) c <<= 1;
      return c;
    }
    return (bytes + (size_t(1) << 20) - 1) & ~((size_t(1) << 20) - 1);
  }
  void* alloc(size_t bytes, bool host) {
    const size_t cls = size_class(bytes);
    int dev = -1;
    if (!host) cudaGetDevice(&dev);
    {
      std::lock_guard<std::mutex> lk(mu_);
      auto it = free_.find(Key{dev, cls});
      if (it != free_.end()) {
        void* p = it->second;
        free_.erase(it);
        return p;
      }
    }
    void* p = nullptr;
    cudaError_t e = host ? cudaMallocHost(&p, cls) : cudaMalloc(&p, cls);
    if (e != cudaSuccess) {  // out of memory: drop the cache and retry once
      cudaGetLastError();
      release_all();
      e = host ? cudaMallocHost(&p, cls) : cudaMalloc(&p, cls);
    }
    if (e != cudaSuccess)
      throw Error(POTGPU_ERR_CUDA, std::string(host ? "cudaMallocHost: " : "cudaMalloc: ") + cudaGetErrorString(e));
    return p;
  }
  void free(void* p, size_t bytes, bool host) {
    if (!p) return;
    int dev = -1;
    if (!host) cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu_);
    free_.emplace(Key{dev, size_class(bytes)}, p);
  }
  void release_all() {
    std::lock_guard<std::mutex> lk(mu_);
    int cur = 0;
    cudaGetDevice(&cur);
    for (auto& kv : free_) {
      if (kv.first.dev < 0) {
        cudaFreeHost(kv.second);
      } else {
        cudaSetDevice(kv.first.dev);
        cudaFree(kv.second);
      }
    }
    free_.clear();
    cudaSetDevice(cur);
  }

 private:
  struct Key {
    int dev;
    size_t cls;
    bool operator<(const Key& o) const { return dev != o.dev ? dev < o.dev : cls < o.cls; }
  };
  std::mutex mu_;
  std::multimap<Key, void*> free_;
};

// $POTGPU_PDL (default on): launch the per-iteration kernels with
// programmatic stream serialization (captured as programmatic edges in the
// CUDA graphs), hiding the launch latency between dependent kernels.
// Worker threads of a batched solve turn PDL off for their launches: with
// several streams in flight, early-launched dependents hold SM slots while
// they wait and the streams' kernels overlap worse (measured at configs[4]:
// 118 vs 70 problems/s at 8 workers, profiles/c5_batched.py).
inline thread_local bool tl_no_pdl = false;
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("POTGPU_PDL");
    return !(e && e[0] == '0');
  }();
  return on && !tl_no_pdl;
}

// $POTGPU_GRAPH_LOOP=1: run the ASPOT loop as a CUDA-graph WHILE node (one
// host launch per run) instead of one graph launch per attempt. Off by
// default: measured equal on one stream (C3 2584 vs 2592 it/s; the host
// launches run ahead of the GPU) and slower with concurrent batched workers
// (54-59 vs 118 problems/s at configs[4]).
inline bool graph_loop_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("POTGPU_GRAPH_LOOP");
    return e && e[0] == '1';
  }();
  return on;
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is one process-wide value per
// kernel (and device), while sessions of different sizes are prepared
// concurrently (batched workers): the limit is only ever RAISED, under a
// lock, so a concurrent smaller session cannot lower it below what another
// session is about to launch with.
template <typename K>
inline void raise_dyn_smem(K kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<int, const void*>, size_t> cur;
  int dev = 0;
  PG_CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  size_t& v = cur[{dev, reinterpret_cast<const void*>(kernel)}];
  if (bytes > v) {
    PG_CK(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes)));
    v = bytes;
  }
}

template <typename... KArgs, typename... Args>
inline void launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PG_CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

// launch_k with a thread-block cluster of cx CTAs along x (cx = 1: plain).
template <typename... KArgs, typename... Args>
inline void launch_kc(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, int cx,
                      Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (pdl_enabled()) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (cx > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = unsigned(cx);
    at[na].val.clusterDim.y = 1;
    at[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = at;
  cfg.numAttrs = unsigned(na);
  PG_CK(cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...));
}

template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t count = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) BlockCache::get().free(p, count * sizeof(T), false);
    p = nullptr;
    count = 0;
  }
  void alloc(size_t k) {
    if (k <= count && p) return;
    release();
    if (k == 0) return;
    p = static_cast<T*>(BlockCache::get().alloc(k * sizeof(T), false));
    count = k;
  }
  void zero(cudaStream_t st) {
    if (p) PG_CK(cudaMemsetAsync(p, 0, count * sizeof(T), st));
  }
};

// A pinned host object from the cache (control-block mirrors).
template <class T>
struct PinnedObj {
  T* p = nullptr;
  PinnedObj() = default;
  PinnedObj(const PinnedObj&) = delete;
  PinnedObj& operator=(const PinnedObj&) = delete;
  ~PinnedObj() {
    if (p) BlockCache::get().free(p, sizeof(T), true);
  }
  T* get() {
    if (!p) p = static_cast<T*>(BlockCache::get().alloc(sizeof(T), true));
    return p;
  }
};

// ---------------------------------------------------------------- device --
__device__ __forceinline__ double nan_max(double a, double b) {
  // NaN-propagating max, the reference's !(max <= 700) sees NaN as overflow.
  return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000ULL) : (a > b ? a : b);
}

// Eigen packet exp semantics (pot_oracle.hpp eexp).
__device__ __forceinline__ double eexp(double x) {
  if (x != x) return x;
  if (x == __longlong_as_double(0x7ff0000000000000ULL)) return x;
  return exp(fmin(fmax(x, kExpLo), kExpHi));
}

// rho extended by its limits (dual.hpp:144-159).
__device__ __forceinline__ double rho_limit(double a, double b) {
  if (!(a > 0)) return b;
  if (!(b > 0)) return __longlong_as_double(0x7ff0000000000000ULL);
  return b - a + a * log(a / b);
}

// Programmatic dependent launch: a kernel launched with the PDL attribute
// may start while its predecessor drains; it waits here before touching
// anything the predecessor writes (a no-op for ordinary launches).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

template <class T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
// sm_100a: one CREDUX.MAX.F32 instead of a 5-step shuffle tree.
__device__ __forceinline__ float warp_maxf(float x) {
  float r;
  asm volatile("redux.sync.max.f32 %0, %1, 0xffffffff;" : "=f"(r) : "f"(x));
  return r;
}
__device__ __forceinline__ double warp_nanmax(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = nan_max(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

__global__ void k_fill_f32(float* p, int64_t count, float value) {
  pdl_wait();
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < count; k += int64_t(gridDim.x) * blockDim.x)
    p[k] = value;
}

}  // namespace potgpu
