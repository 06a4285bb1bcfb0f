// shard.cuh — multi-GPU row-block sharding.
//
// The problem is split into S = world x vshards contiguous row shards
// [lo_s, hi_s). A process (one per GPU) owns `vshards` of them (normally 1;
// more only to run the sharded arithmetic on one GPU, see
// potgpu_comm_init_local). Every n^2 sweep runs over the owned rows only;
// a gather kernel folds the shard's partials into one fp64 vector
//     [ row sums (own rows; 0 elsewhere) | column sums | max slots (S) ]
// and ONE SUM all-reduce (NCCL over NVLink/NVSwitch; plus a fixed-order
// device sum over the process's own shards) makes it global. Because every
// non-owned entry is an exact zero, the sum reproduces the owned row sums and
// the per-shard max exponents bit for bit; only column sums are reassociated.
// Everything after the reduction (per-index functionals, Greenkhorn block,
// z-updates, stopping) runs redundantly and identically on every rank, so
// no further exchange is needed and all ranks take the same decisions.
//
// Sinkhorn's row LSE is local to a shard (rows are whole); its column LSE is
// combined with a MAX all-reduce of the shard maxima followed by a SUM
// all-reduce of the rescaled shard sums.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2", or $POTGPU_NCCL_LIB):
// the library has no link-time dependency on it and single-GPU use never
// touches it. Collectives are enqueued on the context stream, so they are
// captured into the per-iteration CUDA graphs like the kernels around them.
#pragma once

#include <dlfcn.h>

#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <tuple>
#include <memory>
#include <vector>

#include "sweep.cuh"

namespace potgpu {

struct NcclUid {
  char internal[128];
};

// The subset of the NCCL C API used here (nccl.h; enum values are ABI).
struct NcclApi {
  void* lib = nullptr;
  int (*GetUniqueId)(NcclUid*) = nullptr;
  int (*CommInitRank)(void**, int, NcclUid, int) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*CommDestroy)(void*) = nullptr;
  const char* (*GetErrorString)(int) = nullptr;
  static constexpr int kFloat64 = 8;
  static constexpr int kSum = 0;
  static constexpr int kMax = 2;
};

inline NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (!tried) {
    tried = true;
    const char* env = std::getenv("POTGPU_NCCL_LIB");
    const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      if (!nm || !*nm) continue;
      api.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.lib) break;
    }
    if (api.lib) {
      api.GetUniqueId = reinterpret_cast<int (*)(NcclUid*)>(dlsym(api.lib, "ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<int (*)(void**, int, NcclUid, int)>(dlsym(api.lib, "ncclCommInitRank"));
      api.AllReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
          dlsym(api.lib, "ncclAllReduce"));
      api.CommDestroy = reinterpret_cast<int (*)(void*)>(dlsym(api.lib, "ncclCommDestroy"));
      api.GetErrorString = reinterpret_cast<const char* (*)(int)>(dlsym(api.lib, "ncclGetErrorString"));
      if (!api.GetUniqueId || !api.CommInitRank || !api.AllReduce || !api.CommDestroy) api.lib = nullptr;
    }
  }
  if (!api.lib) throw Error(POTGPU_ERR_NCCL, "NCCL runtime (libnccl.so.2) not found; set POTGPU_NCCL_LIB");
  return api;
}

inline void nccl_check(int rc, const char* what) {
  if (rc != 0) {
    const NcclApi& a = nccl_api();
    throw Error(POTGPU_ERR_NCCL, std::string(what) + ": " + (a.GetErrorString ? a.GetErrorString(rc) : "error"));
  }
}

// One cross-process reduction of the host backend: captured into the
// per-iteration graphs as D2H copy -> host node -> H2D copy, so its record
// must outlive them (owned by the Comm, stable addresses).
struct HostReduceCall {
  potgpu_host_allreduce_fn fn = nullptr;
  void* user = nullptr;
  double* buf = nullptr;  // pinned
  int64_t count = 0;
  int op = 0;
};

struct PinnedArr {
  double* p = nullptr;
  size_t bytes = 0;
  PinnedArr() = default;
  PinnedArr(const PinnedArr&) = delete;
  PinnedArr& operator=(const PinnedArr&) = delete;
  ~PinnedArr() {
    if (p) BlockCache::get().free(p, bytes, true);
  }
};

// Records of the host backend's reductions, one per (device vector, count,
// op) call site: reused by every capture and eager call of that site.
struct HostReduceSites {
  std::deque<HostReduceCall> calls;
  std::deque<PinnedArr> bufs;
  std::map<std::tuple<const double*, int64_t, int>, HostReduceCall*> index;
};

inline void CUDART_CB host_reduce_trampoline(void* p) {
  const HostReduceCall* c = static_cast<const HostReduceCall*>(p);
  c->fn(c->buf, c->count, c->op, c->user);
}

struct Comm {
  int rank = 0, world = 1;  // processes (one per GPU)
  int vshards = 1;          // row shards computed by this process
  void* nccl = nullptr;     // ncclComm_t when world > 1
  potgpu_host_allreduce_fn host_fn = nullptr;  // host collective backend (potgpu_comm_init_host)
  void* host_user = nullptr;
  std::shared_ptr<HostReduceSites> host_sites = std::make_shared<HostReduceSites>();
  int total() const { return world * vshards; }
  // a cross-process backend (NCCL, even of one rank, or host callbacks)
  // routes every reduction through it, so the multi-GPU plumbing is
  // exercised on one GPU too
  bool multi() const { return nccl != nullptr || host_fn != nullptr; }
  bool sharded() const { return total() > 1 || multi(); }
  int shard_index(int p) const { return rank * vshards + p; }
  // balanced contiguous row ranges
  int64_t lo(int64_t n, int s) const { return (n * s) / total(); }
  int64_t hi(int64_t n, int s) const { return (n * (s + 1)) / total(); }
  int64_t local_lo(int64_t n) const { return lo(n, shard_index(0)); }
  int64_t local_hi(int64_t n) const { return hi(n, shard_index(vshards - 1)); }
};

// ------------------------------------------------------------ kernels --
// recv[k] = op over p of send[p * stride + k] in shard order (SUM / NaN-max).
__global__ void k_shard_reduce(const double* send, int nsend, int64_t stride, int64_t count, int op, double* recv,
                               const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count; k += int64_t(gridDim.x) * blockDim.x) {
    double a = send[k];
    for (int p = 1; p < nsend; ++p) {
      const double b = send[p * stride + k];
      a = op == NcclApi::kSum ? a + b : nan_max(a, b);
    }
    recv[k] = a;
  }
}

// One shard's sweep partials -> its slice of the all-reduce vector:
// out[i] (rows, own rows only), out[n + j] (columns), out[2n + s] (max
// exponent of shard s; 0 in the other shards' slots).
__global__ void k_shard_gather(const double* rowp, int64_t nstrips, const double* colp, int64_t nrb, const double* maxp,
                               int64_t nmax, int pfmt, Slot z, const double* lu, const double* rowshift, int64_t lo,
                               int64_t hi, int shard, int nshards, double* out, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  const int64_t n = z.n;
  const double w = *z.w();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double rr = 0.0;
    if (i >= lo && i < hi) {
      double a2 = ((z.u()[i] + (lu ? lu[i] : 0.0)) + w) * kLog2e;
      if (rowshift) a2 = a2 + rowshift[i];
      for (int64_t s = 0; s < nstrips; ++s) rr += partial_value(rowp, i * nstrips + s, pfmt, a2);
    }
    double cc = 0.0;
    for (int64_t s = 0; s < nrb; ++s) cc += partial_value(colp, i * nrb + s, pfmt);
    out[i] = rr;
    out[n + i] = cc;
  }
  if (blockIdx.x == 0) {
    __shared__ double sh[kVecThreads];
    double m = -INFINITY;
    for (int64_t k = threadIdx.x; k < nmax; k += blockDim.x) m = nan_max(m, maxp[k]);
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int st = kVecThreads / 2; st > 0; st >>= 1) {
      if (threadIdx.x < st) sh[threadIdx.x] = nan_max(sh[threadIdx.x], sh[threadIdx.x + st]);
      __syncthreads();
    }
    for (int s = threadIdx.x; s < nshards; s += blockDim.x) out[2 * n + s] = s == shard ? sh[0] : 0.0;
  }
}

// A shard's per-column LSE pair (m, S) -> rescaled to the global max M:
// S' = S e^(m - M) (in place).
__global__ void k_shard_lse_rescale(double* send, int nsend, int64_t stride, int64_t n, const double* M, const int* gate) {
  pdl_wait();
  if (gate && *gate == 0) return;
  for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
    const double Mk = M[k];
    for (int p = 0; p < nsend; ++p) {
      const double m = send[p * stride + k];
      double& S = send[p * stride + n + k];
      S = (S == 0.0 || m == -INFINITY) ? 0.0 : S * exp(m - Mk);
    }
  }
}

// Reduction of `count` doubles: the process's own shards (fixed order), then
// across processes.
// Host backend: recv (device) -> pinned -> the caller's all-reduce -> recv.
inline void host_allreduce(const Comm& cm, cudaStream_t st, double* recv, int64_t count, int op) {
  HostReduceSites& hs = *cm.host_sites;
  HostReduceCall*& site = hs.index[std::make_tuple(static_cast<const double*>(recv), count, op)];
  if (!site) {
    PinnedArr& b = hs.bufs.emplace_back();
    b.bytes = size_t(std::max<int64_t>(count, 1)) * sizeof(double);
    b.p = static_cast<double*>(BlockCache::get().alloc(b.bytes, true));
    HostReduceCall& c = hs.calls.emplace_back();
    c.buf = b.p;
    c.count = count;
    c.op = op;
    site = &c;
  }
  site->fn = cm.host_fn;
  site->user = cm.host_user;
  PG_CK(cudaMemcpyAsync(site->buf, recv, size_t(count) * sizeof(double), cudaMemcpyDeviceToHost, st));
  PG_CK(cudaLaunchHostFunc(st, host_reduce_trampoline, site));
  PG_CK(cudaMemcpyAsync(recv, site->buf, size_t(count) * sizeof(double), cudaMemcpyHostToDevice, st));
}

inline void shard_allreduce(const Comm& cm, cudaStream_t st, int num_sms, double* send, int64_t stride, int64_t count,
                            int op, double* recv, const int* gate) {
  if (cm.host_fn) {
    // the device sum over this process's shards (a copy for one), then the
    // host round trip; every rank issues it whatever the gate (same order)
    const int blocks = int(std::min<int64_t>(num_sms * 4, std::max<int64_t>(1, ceil_div(count, kVecThreads))));
    launch_k(k_shard_reduce, dim3(blocks), dim3(kVecThreads), 0, st, send, cm.vshards, stride, count, op, recv, nullptr);
    PG_CK(cudaGetLastError());
    host_allreduce(cm, st, recv, count, op);
    return;
  }
  const bool multi = cm.nccl != nullptr;
  if (cm.vshards > 1 || !multi) {
    const int blocks = int(std::min<int64_t>(num_sms * 4, std::max<int64_t>(1, ceil_div(count, kVecThreads))));
    launch_k(k_shard_reduce, dim3(blocks), dim3(kVecThreads), 0, st, send, cm.vshards, stride, count, op, recv, gate);
    PG_CK(cudaGetLastError());
    if (multi) nccl_check(nccl_api().AllReduce(recv, recv, size_t(count), NcclApi::kFloat64, op, cm.nccl, st), "ncclAllReduce");
  } else {
    nccl_check(nccl_api().AllReduce(send, recv, size_t(count), NcclApi::kFloat64, op, cm.nccl, st), "ncclAllReduce");
  }
}

}  // namespace potgpu
