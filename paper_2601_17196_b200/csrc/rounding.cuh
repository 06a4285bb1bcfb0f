// rounding.cuh — per-element fp64 views of the cost (C_ij and logK_ij) used
// by the output-stage kernels (plan.cuh): <C, X> and the dense plan.
#pragma once

#include "sweep.cuh"

namespace potgpu {

// Per-element views of the cost for the (non-hot) cost/materialise sweeps.
struct ElemDenseF64 {
  const double* L; int64_t ld; double gamma;
  __device__ __forceinline__ double logk(int64_t i, int64_t j) const { return L[i * ld + j]; }
  __device__ __forceinline__ double cost(int64_t i, int64_t j) const { return -L[i * ld + j] * gamma; }
};
struct ElemDenseF32 {
  const float* C; int64_t ld; double gamma;
  __device__ __forceinline__ double cost(int64_t i, int64_t j) const { return double(C[i * ld + j]); }
  __device__ __forceinline__ double logk(int64_t i, int64_t j) const { return -cost(i, j) / gamma; }
};
struct ElemPointsF32 {
  const float4* X; const float4* Y; double scale; double gamma;
  __device__ __forceinline__ double cost(int64_t i, int64_t j) const {
    const float4 a = X[i], b = Y[j];
    const double dx = double(a.x) - double(b.x), dy = double(a.y) - double(b.y), dz = double(a.z) - double(b.z);
    return (((dx * dx) + dy * dy) + dz * dz) * scale;
  }
  __device__ __forceinline__ double logk(int64_t i, int64_t j) const { return -cost(i, j) / gamma; }
};

}  // namespace potgpu
