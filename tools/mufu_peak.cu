// MUFU.EX2 throughput microbenchmark (B200): the denominator of the on-the-fly
// sweep's roofline. Each thread runs K independent chains x <- ex2(x) * a + b
// (one MUFU.EX2 + one FFMA per element, the FFMA keeps the chain in range),
// with 2..32 warps per SM; reports ex2/clk/SM against the nominal 16.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mufu_peak mufu_peak.cu && ./mufu_peak
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void k_ex2(float* out, int iters, float a, float b) {
  float x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = -0.001f * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x[k]));
      x[k] = fmaf(y, a, b);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  if (s == 123.456f) out[0] = s;
}

// The sweep's mix: per ex2, 5 more FP32-pipe ops (3 FFMA of the exponent,
// a max, the subtraction of the shift), K independent chains per thread.
template <int K>
__global__ void k_mix(float* out, int iters, float a, float b) {
  float x[K], m[K];
#pragma unroll
  for (int k = 0; k < K; ++k) { x[k] = -0.001f * (threadIdx.x + k); m[k] = 0.f; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float t = fmaf(x[k], a, b);
      t = fmaf(t, a, b);
      t = fmaf(t, a, b);
      m[k] = fmaxf(m[k], t);
      float y;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(t - 0.125f));
      x[k] = y;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k] + m[k];
  if (s == 123.456f) out[0] = s;
}

// The sweep's per-pair work with paired FP32 ops, independent chains, no
// cross-lane work: per 2 ex2: 3 FFMA2 (exponent), 1 max, 1 FADD2 (shift),
// 2 MUFU.EX2, 1 FADD2 (row sum), 1 FFMA2 (column accumulator).
template <int K>
__global__ void k_mix2(float* out, int iters, float a, float b) {
  float2 x[K], acc[K], rs[K];
  float m[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    x[k] = make_float2(-0.001f * (threadIdx.x + k), -0.002f * k);
    acc[k] = make_float2(0.f, 0.f);
    rs[k] = make_float2(0.f, 0.f);
    m[k] = 0.f;
  }
  const float2 A = make_float2(a, a), B = make_float2(b, b);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      float2 t = __ffma2_rn(x[k], A, B);
      t = __ffma2_rn(t, A, B);
      t = __ffma2_rn(t, A, B);
      m[k] = fmaxf(m[k], fmaxf(t.x, t.y));
      const float2 d = __fadd2_rn(t, make_float2(-0.125f, -0.125f));
      float2 p;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p.x) : "f"(d.x));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p.y) : "f"(d.y));
      rs[k] = __fadd2_rn(rs[k], p);
      acc[k] = __ffma2_rn(p, A, acc[k]);
      x[k] = p;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k].x + acc[k].y + rs[k].x + m[k];
  if (s == 123.456f) out[0] = s;
}

// mix_pairs plus one LDS.64 per pair (the sweep's column constant B'_j
// read from shared memory each row): MUFU and LDS share the MIO queue.
template <int K>
__global__ void k_mix2_lds(float* out, int iters, float a, float b) {
  __shared__ float2 sB[K][32];
  const int lane = threadIdx.x & 31;
  for (int k = 0; k < K; ++k) if (threadIdx.x < 32) sB[k][lane] = make_float2(0.001f * k, -0.002f * lane);
  __syncthreads();
  float2 x[K], acc[K], rs[K];
  float m[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    x[k] = make_float2(-0.001f * (threadIdx.x + k), -0.002f * k);
    acc[k] = make_float2(0.f, 0.f);
    rs[k] = make_float2(0.f, 0.f);
    m[k] = 0.f;
  }
  const float2 A = make_float2(a, a);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
      const float2 B = sB[k][lane];
      float2 t = __ffma2_rn(x[k], A, B);
      t = __ffma2_rn(t, A, B);
      t = __ffma2_rn(t, A, B);
      m[k] = fmaxf(m[k], fmaxf(t.x, t.y));
      const float2 d = __fadd2_rn(t, make_float2(-0.125f, -0.125f));
      float2 p;
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p.x) : "f"(d.x));
      asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(p.y) : "f"(d.y));
      rs[k] = __fadd2_rn(rs[k], p);
      acc[k] = __ffma2_rn(p, A, acc[k]);
      x[k] = p;
    }
  }
  float s = 0.f;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k].x + acc[k].y + rs[k].x + m[k];
  if (s == 123.456f) out[0] = s;
}

int main() {
  int dev = 0, sms = 0, clk_khz = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  float* out;
  cudaMalloc(&out, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  printf("{\"sms\": %d, \"attr_clock_mhz\": %.0f, \"runs\": [", sms, clk_khz / 1e3);
  bool first = true;
  for (int warps = 4; warps <= 32; warps *= 2) {
    const int threads = 256, blocks = sms * warps * 32 / threads;
    k_ex2<8><<<blocks, threads>>>(out, 64, 0.5f, -0.25f);
    cudaEventRecord(e0);
    k_ex2<8><<<blocks, threads>>>(out, iters, 0.5f, -0.25f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ex2 = double(blocks) * threads * iters * 8;
    printf("%s{\"warps_per_sm\": %d, \"ms\": %.4f, \"gex2_s\": %.1f}", first ? "" : ", ", warps, ms, ex2 / (ms * 1e-3) / 1e9);
    first = false;
  }
  printf("], \"mix5\": [");
  first = true;
  for (int warps = 8; warps <= 32; warps *= 2) {
    const int threads = 256, blocks = sms * warps * 32 / threads;
    k_mix<8><<<blocks, threads>>>(out, 64, 0.5f, -0.25f);
    cudaEventRecord(e0);
    k_mix<8><<<blocks, threads>>>(out, iters, 0.5f, -0.25f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ex2 = double(blocks) * threads * iters * 8;
    printf("%s{\"warps_per_sm\": %d, \"ms\": %.4f, \"gex2_s\": %.1f}", first ? "" : ", ", warps, ms, ex2 / (ms * 1e-3) / 1e9);
    first = false;
  }
  printf("], \"mix_pairs\": [");
  first = true;
  for (int warps = 8; warps <= 32; warps *= 2) {
    const int threads = 256, blocks = sms * warps * 32 / threads;
    k_mix2<4><<<blocks, threads>>>(out, 64, 0.5f, -0.25f);
    cudaEventRecord(e0);
    k_mix2<4><<<blocks, threads>>>(out, iters, 0.5f, -0.25f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ex2 = double(blocks) * threads * iters * 8;
    printf("%s{\"warps_per_sm\": %d, \"ms\": %.4f, \"gex2_s\": %.1f}", first ? "" : ", ", warps, ms, ex2 / (ms * 1e-3) / 1e9);
    first = false;
  }
  printf("], \"mix_pairs_lds\": [");
  first = true;
  for (int warps = 8; warps <= 32; warps *= 2) {
    const int threads = 256, blocks = sms * warps * 32 / threads;
    k_mix2_lds<4><<<blocks, threads>>>(out, 64, 0.5f, -0.25f);
    cudaEventRecord(e0);
    k_mix2_lds<4><<<blocks, threads>>>(out, iters, 0.5f, -0.25f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ex2 = double(blocks) * threads * iters * 8;
    printf("%s{\"warps_per_sm\": %d, \"ms\": %.4f, \"gex2_s\": %.1f}", first ? "" : ", ", warps, ms, ex2 / (ms * 1e-3) / 1e9);
    first = false;
  }
  printf("]}\n");
  return 0;
}
