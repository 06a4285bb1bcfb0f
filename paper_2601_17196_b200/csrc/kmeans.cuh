// kmeans.cuh — colour quantisation for colour transfer (SURVEY.md §8(f)
// row 4; reference color_transfer.hpp:34-118 kmeans_quantize).
//
// k-means++ seeding is sequential by definition (each pick scans the
// running distances with the reference's std::mt19937_64 draws) and runs on
// the host exactly as the reference; the Lloyd rounds — N x k distance
// evaluations per round — run on the device: nearest-centroid assignment
// with the centroids in shared memory, and deterministic cluster sums (a
// block owns a contiguous chunk of points, thread j accumulates cluster j
// over it in order, block partials are reduced in block order).
#pragma once

#include <random>

namespace potgpu {

__device__ __forceinline__ double km_d2(const double* p, const double* c) {
  const double dx = p[0] - c[0], dy = p[1] - c[1], dz = p[2] - c[2];
  return (dx * dx + dy * dy) + dz * dz;
}

// assign[i] = argmin_j |p_i - c_j|^2 (first minimum, strict <).
__global__ void k_km_assign(const double* pts, int64_t n, const double* C, int k, int* assign) {
  extern __shared__ double sC[];
  for (int q = threadIdx.x; q < 3 * k; q += blockDim.x) sC[q] = C[q];
  __syncthreads();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const double p[3] = {pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]};
    int best = 0;
    double bd = km_d2(p, sC);
    for (int j = 1; j < k; ++j) {
      const double d = km_d2(p, sC + 3 * j);
      if (d < bd) { best = j; bd = d; }
    }
    assign[i] = best;
  }
}

constexpr int kKmChunk = 1024;  // points per block in the cluster-sum pass (28 KB smem)

// part[b][j] = (sum x, sum y, sum z, count) of cluster j over block b's chunk.
__global__ void k_km_partial(const double* pts, const int* assign, int64_t n, int k, double* part) {
  __shared__ int sa[kKmChunk];
  __shared__ double sp[kKmChunk * 3];
  const int64_t c0 = int64_t(blockIdx.x) * kKmChunk;
  const int cnt = int(n - c0 < int64_t(kKmChunk) ? n - c0 : int64_t(kKmChunk));
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
    sa[q] = assign[c0 + q];
    sp[3 * q] = pts[3 * (c0 + q)];
    sp[3 * q + 1] = pts[3 * (c0 + q) + 1];
    sp[3 * q + 2] = pts[3 * (c0 + q) + 2];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < k; j += blockDim.x) {
    double sx = 0, sy = 0, sz = 0, c = 0;
    for (int q = 0; q < cnt; ++q)
      if (sa[q] == j) { sx += sp[3 * q]; sy += sp[3 * q + 1]; sz += sp[3 * q + 2]; c += 1.0; }
    double* o = part + (int64_t(blockIdx.x) * k + j) * 4;
    o[0] = sx; o[1] = sy; o[2] = sz; o[3] = c;
  }
}

__global__ void k_km_reduce(const double* part, int nblocks, int k, double* out) {
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < 4 * k; q += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < nblocks; ++b) s += part[int64_t(b) * 4 * k + q];
    out[q] = s;
  }
}

// kmeans_quantize: centroids (k x 3), weights (k), assignments (n).
inline int kmeans_quantize(Context& cx, const double* pts_h, int64_t n, int k, uint64_t seed, double* centroids,
                           double* weights, int* assignments) {
  if (n == 0) throw Error(POTGPU_EMPTY_INPUT, "no points to quantize");
  if (k < 1 || int64_t(k) > n)
    throw Error(POTGPU_INVALID_ARGUMENT, "k must lie in [1, N] (k=" + std::to_string(k) + ", N=" + std::to_string(n) + ")");
  if (k > 4096) throw Error(POTGPU_ERR_UNSUPPORTED, "k > 4096 centroids");
  auto d2h = [&](int64_t i, const double* c) {
    const double dx = pts_h[3 * i] - c[0], dy = pts_h[3 * i + 1] - c[1], dz = pts_h[3 * i + 2] - c[2];
    return (dx * dx + dy * dy) + dz * dz;
  };
  // k-means++ seeding (color_transfer.hpp:47-73), the reference's draws
  std::mt19937_64 rng(seed);
  std::vector<double> C(static_cast<size_t>(3 * k));
  std::uniform_int_distribution<long> first(0, long(n) - 1);
  const long f0 = first(rng);
  for (int d = 0; d < 3; ++d) C[size_t(d)] = pts_h[3 * f0 + d];
  std::vector<double> dist2(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) dist2[size_t(i)] = d2h(i, C.data());
  std::uniform_real_distribution<double> unit(0.0, 1.0);
  for (int j = 1; j < k; ++j) {
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) total += dist2[size_t(i)];
    long pick = 0;
    if (total > 0) {
      double target = unit(rng) * total;
      for (int64_t i = 0; i < n; ++i) {
        target -= dist2[size_t(i)];
        if (target <= 0) { pick = long(i); break; }
      }
    } else {
      pick = first(rng);
    }
    for (int d = 0; d < 3; ++d) C[size_t(3 * j + d)] = pts_h[3 * pick + d];
    for (int64_t i = 0; i < n; ++i) dist2[size_t(i)] = std::min(dist2[size_t(i)], d2h(i, &C[size_t(3 * j)]));
  }
  // Lloyd rounds on the device (color_transfer.hpp:75-97)
  DevBuf<double> pts, Cd, part, red;
  DevBuf<int> asg;
  pts.alloc(size_t(3 * n));
  Cd.alloc(size_t(3 * k));
  asg.alloc(size_t(n));
  const int nblocks = int(ceil_div(n, kKmChunk));
  part.alloc(size_t(nblocks) * size_t(4 * k));
  red.alloc(size_t(4 * k));
  PG_CK(cudaMemcpyAsync(pts.p, pts_h, size_t(3 * n) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
  const int ablocks = int(std::min<int64_t>(ceil_div(n, 256), int64_t(cx.num_sms) * 8));
  const size_t csmem = size_t(3 * k) * sizeof(double);
  if (csmem > 48 * 1024) raise_dyn_smem(k_km_assign, size_t(int(csmem)));
  std::vector<double> R(static_cast<size_t>(4 * k));
  auto cluster_sums = [&]() {
    PG_CK(cudaMemcpyAsync(Cd.p, C.data(), size_t(3 * k) * sizeof(double), cudaMemcpyHostToDevice, cx.stream));
    k_km_assign<<<ablocks, 256, csmem, cx.stream>>>(pts.p, n, Cd.p, k, asg.p);
    k_km_partial<<<nblocks, 256, 0, cx.stream>>>(pts.p, asg.p, n, k, part.p);
    k_km_reduce<<<int(std::min<int64_t>(ceil_div(4 * k, 256), 64)), 256, 0, cx.stream>>>(part.p, nblocks, k, red.p);
    PG_CK(cudaGetLastError());
    PG_CK(cudaMemcpyAsync(R.data(), red.p, size_t(4 * k) * sizeof(double), cudaMemcpyDeviceToHost, cx.stream));
    PG_CK(cudaStreamSynchronize(cx.stream));
  };
  for (int round = 0; round < 100; ++round) {
    cluster_sums();
    double moved = 0.0;
    for (int j = 0; j < k; ++j) {
      const double cnt = R[size_t(4 * j + 3)];
      if (cnt == 0) continue;  // empty cluster keeps its centroid
      double nx[3], m2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        nx[d] = R[size_t(4 * j + d)] / cnt;
        const double e = nx[d] - C[size_t(3 * j + d)];
        m2 += e * e;
      }
      moved = std::max(moved, std::sqrt(m2));
      for (int d = 0; d < 3; ++d) C[size_t(3 * j + d)] = nx[d];
    }
    if (moved < 1e-6) break;
  }
  cluster_sums();  // final assignment and counts (color_transfer.hpp:99-117)
  for (int q = 0; q < 3 * k; ++q) centroids[q] = C[size_t(q)];
  for (int j = 0; j < k; ++j) weights[j] = R[size_t(4 * j + 3)] / double(n);
  if (assignments) PG_CK(cudaMemcpy(assignments, asg.p, size_t(n) * sizeof(int), cudaMemcpyDeviceToHost));
  return 0;
}

}  // namespace potgpu
