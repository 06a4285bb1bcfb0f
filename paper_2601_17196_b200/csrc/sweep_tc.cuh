// sweep_tc.cuh — the fp32 on-the-fly points sweep with its exponents formed
// on the 5th-generation tensor cores (tcgen05.mma, accumulators in TMEM).
//
// Why: sweep_pts2_f32 spends ~6 FP32-pipe operations per plan entry (a
// 3-term dot product, the row shift, the row sum, the column accumulation)
// beside its one MUFU.EX2, and at 4 warps per scheduler the two pipes do not
// overlap well enough: it runs at ~55 % of the MUFU roof (ncu: XU 60 %, FMA
// 46 %, issue 48 %). Here the log2 exponent of every entry
//   S_ij = t'_ij - s_i = B_j + 2 x'_i . y'_j - s_i
// (reference: exponent_matrix, dual.hpp:93-99, in the fp32 sweeps' log2
// frame, sweep.cuh) is one K = 32 bf16 GEMM tile: each of the 5 row terms
// (2x'_1, 2x'_2, 2x'_3, -s_i, 1) and column terms (y'_1, y'_2, y'_3, 1, B_j)
// is split into three bf16 pieces (hi + mid + lo = the fp32 value, 24
// significant bits), and the six products hi.hi, hi.mid, mid.hi, hi.lo,
// lo.hi, mid.mid are laid out along K, so the fp32-accumulated product is
// the fp32 exponent to ~2^-24 of the largest term (the FFMA2 chain of
// sweep_pts2_f32 rounds at the same magnitude). The CUDA cores then only do
// tcgen05.ld -> MUFU.EX2 -> row sum (thread-local: TMEM lane = row) ->
// column accumulation; per entry 2 FP32-pipe operations instead of 6.
//
// Layout: one CTA = one warpgroup (4 warps, TMEM lanes 0..127) owns a
// 512-column strip (the points sweep's strip, so carries and partial formats
// are shared with sweep_pts2_f32) and up to 4 x 128 rows. Per 32-column
// chunk and 128-row tile one elected thread issues 2 MMAs (K = 16 each) into
// a ring of kTcStages TMEM buffers and commits each to an mbarrier; MMAs run
// up to 3 tiles ahead of the warps reading them. The warps never meet at a
// CTA barrier inside a pass: the column operand of chunk c + kTcBRing is
// rebuilt by each warp (its 8-element K piece) as soon as it has consumed
// chunk c, and published through an mbarrier the issuing thread waits on.
// Row sums accumulate in registers across the strip (thread = row); column
// sums accumulate across the CTA's row tiles, are combined across lanes by a
// butterfly at the end of each chunk (lane l keeps column l) and across the
// 4 warps once per pass, in a fixed order (deterministic).
//
// Shifts: the carried bound of sweep_pts2_f32 (s_i = c_i + max dB over the
// strip). A CTA without a valid carry first runs the same tile loop without
// exponentials to get each row's exact segment max (s_i = that max), then
// the exponential pass. Output formats, carries, maxp semantics: as
// sweep_pts2_f32 (carried path).
#pragma once

#include <cuda_bf16.h>

#include "sweep.cuh"

namespace potgpu {

constexpr int kTcTilesMax = 4;             // 128-row tiles per CTA (<= 512 rows)
constexpr int kTcN = 32;                   // columns per MMA tile (chunk)
constexpr int kTcStrip = 512;              // columns per CTA
constexpr int kTcChunks = kTcStrip / kTcN;
constexpr int kTcThreads = 128;

constexpr int kTcStages = 4;               // S ring in TMEM (MMAs run up to 3 tiles ahead)
constexpr int kTcBRing = 4;                // column-operand ring (chunks)
constexpr uint32_t kTcTmemCols = kTcStages * kTcN;

struct TcSmem {
  uint4 A[kTcTilesMax][4 * 16 * 8];   // per tile: [kchunk 4][row group 16][row 8] x 8 bf16 (8 KB); reused for the
                                      // per-warp column sums at the end of a pass
  uint4 B[kTcBRing][4 * 4 * 8];       // per chunk: [kchunk 4][col group 4][col 8] x 8 bf16 (2 KB)
  uint2 pc[kTcStrip][3];              // bf16 pieces of the column terms (y'_1, y'_2, y'_3, B_j): [piece][term]
  float colB[kTcStrip];               // B_j (fp32) of the strip
  unsigned long long mma_done[kTcStages];
  unsigned long long s_free[kTcStages];
  unsigned long long b_full[kTcBRing];
  uint32_t tmem_base;
  int last;
  float red[3][4];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// bf16 hi / mid / lo pieces of an fp32 value (their sum is the value to
// 2^-24 relative; each difference is exact in fp32)
__device__ __forceinline__ void split3(float v, __nv_bfloat16 (&o)[3]) {
  o[0] = __float2bfloat16_rn(v);
  const float r1 = __fsub_rn(v, __bfloat162float(o[0]));
  o[1] = __float2bfloat16_rn(r1);
  const float r2 = __fsub_rn(r1, __bfloat162float(o[1]));
  o[2] = __float2bfloat16_rn(r2);
}

// The K = 32 operand vector of a row: 6 blocks of its 5 terms with piece
// indices 0,0,1,0,2,1 (the columns use 0,1,0,2,0,1: the six products hi.hi,
// hi.mid, mid.hi, hi.lo, lo.hi, mid.mid), then 2 zeros; as 4 K pieces.
__device__ __forceinline__ void tc_row_kvector(const float (&v)[5], uint4 (&out)[4]) {
  constexpr int prow[6] = {0, 0, 1, 0, 2, 1};
  __nv_bfloat16 pc[5][3];
#pragma unroll
  for (int t = 0; t < 5; ++t) split3(v[t], pc[t]);
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t h[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int k = 8 * c + 2 * q + e;
        h[e] = k < 30 ? uint32_t(__bfloat16_as_ushort(pc[k % 5][prow[k / 5]])) : 0u;
      }
      w[q] = h[0] | (h[1] << 16);
    }
    out[c] = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// The 12 bf16 pieces of a column's varying terms (y'_1, y'_2, y'_3, B_j),
// [piece][term]; the constant term 1 is (1, 0, 0).
__device__ __forceinline__ void tc_col_pieces(const float (&v)[4], uint2 (&out)[3]) {
  __nv_bfloat16 pc[4][3];
#pragma unroll
  for (int t = 0; t < 4; ++t) split3(v[t], pc[t]);
  uint32_t w[6];
#pragma unroll
  for (int q = 0; q < 6; ++q) {
    const int e0 = 2 * q, e1 = 2 * q + 1;  // index = piece * 4 + term
    w[q] = uint32_t(__bfloat16_as_ushort(pc[e0 % 4][e0 / 4])) | (uint32_t(__bfloat16_as_ushort(pc[e1 % 4][e1 / 4])) << 16);
  }
  out[0] = make_uint2(w[0], w[1]);
  out[1] = make_uint2(w[2], w[3]);
  out[2] = make_uint2(w[4], w[5]);
}
// K piece C (8 elements) of a column's operand vector, from its pieces
template <int C>
__device__ __forceinline__ uint4 tc_col_kchunk(const uint2 (&p)[3]) {
  constexpr int pcol[6] = {0, 1, 0, 2, 0, 1};
  const uint32_t w[6] = {p[0].x, p[0].y, p[1].x, p[1].y, p[2].x, p[2].y};
  uint32_t o[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t h[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int k = 8 * C + 2 * q + e;
      const int term = k % 5, piece = pcol[k / 5 < 6 ? k / 5 : 0];
      if (k >= 30) {
        h[e] = 0u;
      } else if (term == 3) {  // the constant 1: hi = 1, mid = lo = 0
        h[e] = piece == 0 ? 0x3F80u : 0u;
      } else {
        const int idx = piece * 4 + (term < 3 ? term : 3);
        h[e] = (w[idx >> 1] >> (16 * (idx & 1))) & 0xFFFFu;
      }
    }
    o[q] = h[0] | (h[1] << 16);
  }
  return make_uint4(o[0], o[1], o[2], o[3]);
}

// UMMA shared-memory descriptor, K-major, no swizzle (core matrices of 8
// rows x 16 bytes): LBO = byte stride between the two 8-element K halves of
// one K = 16 step, SBO = byte stride between 8-row groups; version 1.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return uint64_t((saddr >> 4) & 0x3FFFu) | (uint64_t((lbo >> 4) & 0x3FFFu) << 16) |
         (uint64_t((sbo >> 4) & 0x3FFFu) << 32) | (uint64_t(1) << 46);
}
// instruction descriptor: D fp32, A/B bf16, both K-major, N = kTcN, M = 128
constexpr uint32_t kTcIdesc = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(kTcN >> 3) << 17) | (uint32_t(128 >> 4) << 24);

__device__ __forceinline__ void mbar_init(unsigned long long* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// bounded wait: a lost arrival traps (a kernel error) instead of hanging the GPU
__device__ __forceinline__ void mbar_wait(unsigned long long* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  for (uint32_t spin = 0;; ++spin) {
    uint32_t done;
    asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\tselp.b32 %0, 1, 0, P1;\n\t}"
                 : "=r"(done) : "r"(a), "r"(parity) : "memory");
    if (done) return;
    if (spin > (1u << 26)) __trap();
  }
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accumulate) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(tmem_d), "l"(adesc), "l"(bdesc), "r"(kTcIdesc), "r"(accumulate) : "memory");
}
__device__ __forceinline__ void tc_commit(unsigned long long* b) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void tc_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
               "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                 "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
                 "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
                 "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(r[k]);
}

__host__ __device__ constexpr size_t sweep_tc_smem() { return sizeof(TcSmem) + 16; }

// rows_per_cta = tiles * 128 (tiles in 1..kTcTilesMax); grid = (strips of
// 512 columns, row blocks). a.carry / carry_b / carry_ticket must be set.
__global__ void __launch_bounds__(kTcThreads, 4) sweep_tc_f32(SrcPointsDotF32 src, SweepArgs a) {
  pdl_wait();
  if (a.gate && *a.gate == 0) return;
  extern __shared__ uint8_t tc_raw[];
  TcSmem& S = *reinterpret_cast<TcSmem*>((reinterpret_cast<uintptr_t>(tc_raw) + 15) & ~uintptr_t(15));
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t n = a.n;
  const int64_t j0 = int64_t(blockIdx.x) * kTcStrip;
  const int64_t r0 = a.row_lo + int64_t(blockIdx.y) * a.rows_per_cta;
  const int64_t r1 = min(a.row_hi, r0 + a.rows_per_cta);
  const int nrows = int(r1 - r0);
  const int tiles = (nrows + 127) >> 7;
  const double w = *a.w;
  const int dbg = a.tc_debug;

  if (warp == 0) {  // TMEM: the ring of kTcStages 32-column S buffers
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&S.tmem_base)),
                 "r"(kTcTmemCols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int b = 0; b < kTcStages; ++b) {
      mbar_init(&S.mma_done[b], 1);
      mbar_init(&S.s_free[b], 4);
    }
    for (int b = 0; b < kTcBRing; ++b) mbar_init(&S.b_full[b], 4);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // columns: pieces of (y', B_j) and the strip's change since the carry was written
  float dmax = -INFINITY, dmin = INFINITY;
  int dbad = 0;
  for (int jj = tid; jj < kTcStrip; jj += kTcThreads) {
    const int64_t j = j0 + jj;
    float b = -1e30f;  // masked column: exponent ~ -1e30 -> exp 0
    float4 y = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < n) {
      double vv = a.v[j];
      if (a.lv) vv = vv + a.lv[j];
      vv = vv * kLog2e;
      if (a.colshift) vv = vv + a.colshift[j];
      y = src.Ys[j];
      b = float(vv);
      const float bo = a.carry_b[j];
      if (!(b == -INFINITY && bo == -INFINITY)) {
        const float d = b - bo;
        dbad |= !(fabsf(d) < 1e30f);
        dmax = fmaxf(dmax, d);
        dmin = fminf(dmin, d);
      }
      if (!(fabsf(b) < 1e30f)) { dbad = 1; b = (b == -INFINITY) ? -1e30f : b; }
    }
    const float cv[4] = {y.x, y.y, y.z, b};
    tc_col_pieces(cv, S.pc[jj]);
    S.colB[jj] = b;
  }
  dbad = __any_sync(0xffffffffu, dbad);
  dmax = warp_maxf(dmax);
  dmin = -warp_maxf(-dmin);
  if (lane == 0) { S.red[0][warp] = dmax; S.red[1][warp] = dmin; S.red[2][warp] = dbad ? 1.f : 0.f; }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = S.tmem_base;
  float dx = -INFINITY, dn = INFINITY, bad = 0.f;
  for (int ww = 0; ww < 4; ++ww) { dx = fmaxf(dx, S.red[0][ww]); dn = fminf(dn, S.red[1][ww]); bad += S.red[2][ww]; }
  bool carried = bad == 0.f && dx > -INFINITY && dx - dn <= kCarrySpread;
  // rows: thread tid owns the rows r0 + 128 k + tid (TMEM lane tid of tile k)
  float Ar[kTcTilesMax], sr[kTcTilesMax];
  int rbad = 0;
#pragma unroll
  for (int k = 0; k < kTcTilesMax; ++k) {
    const int64_t i = r0 + 128 * k + tid;
    float A = -INFINITY, s = 1e30f;
    if (k < tiles && i < r1) {
      double ud = a.u[i];
      if (a.lu) ud = ud + a.lu[i];
      double Ad = (ud + w) * kLog2e;
      if (a.rowshift) Ad = Ad + a.rowshift[i];
      A = float(Ad);
      s = a.carry[int64_t(blockIdx.x) * n + i] + dx;
      rbad |= !(fabsf(s) < 1e30f) || !(fabsf(A) < 1e30f);
    }
    Ar[k] = A;
    sr[k] = s;
  }
  carried = carried && !__syncthreads_or(rbad);

  // A operand of every row tile at the shifts sh (dead rows: 1e30 -> exponent ~ -1e30)
  auto build_a = [&](const float (&sh)[kTcTilesMax]) {
#pragma unroll
    for (int k = 0; k < kTcTilesMax; ++k) {
      if (k >= tiles) break;
      const int64_t i = r0 + 128 * k + tid;
      const float4 x = i < r1 ? src.X2[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      const float v[5] = {x.x, x.y, x.z, -sh[k], 1.f};
      uint4 kv[4];
      tc_row_kvector(v, kv);
      const int g = tid >> 3, rin = tid & 7;
#pragma unroll
      for (int c = 0; c < 4; ++c) S.A[k][(c * 16 + g) * 8 + rin] = kv[c];
    }
  };
  // this warp's K piece of chunk `chunk`'s column operand, then publish it
  auto build_b = [&](int chunk, int cglob) {
    const uint2 (&p)[3] = S.pc[chunk * kTcN + lane];
    uint4 q;
    switch (warp) {
      case 0: q = tc_col_kchunk<0>(p); break;
      case 1: q = tc_col_kchunk<1>(p); break;
      case 2: q = tc_col_kchunk<2>(p); break;
      default: q = tc_col_kchunk<3>(p); break;
    }
    S.B[cglob % kTcBRing][(warp * 4 + (lane >> 3)) * 8 + (lane & 7)] = q;
    fence_async_smem();
    __syncwarp();
    if (lane == 0 && dbg != 2) mbar_arrive(&S.b_full[cglob % kTcBRing]);
  };
  int tg = 0, cg = 0;  // tiles and chunks of earlier passes (mbarrier phases continue across passes)
  const int T = kTcChunks * tiles;
  // One pass over the strip. kExp: rsum[k] += sum 2^S, column sums; else rmax[k] = max S.
  float rsum[kTcTilesMax], rmax[kTcTilesMax], fr[kTcTilesMax];
  auto run = [&](bool kExp) {
    int issued = 0, ic = 0, ik = 0;  // thread 0: next tile to issue (chunk, row tile)
    // issue every tile < limit: its TMEM stage free (the tile kTcStages back
    // consumed), its column operand published
    auto issue_upto = [&](int limit) {
      for (; issued < limit; ++issued) {
        const int u = tg + issued;  // tg is a multiple of 16: stages / parities continue
        const int st = u & (kTcStages - 1);
        if (u >= kTcStages) mbar_wait(&S.s_free[st], uint32_t(((u - kTcStages) / kTcStages) & 1));
        if (ik == 0) {
          const int cgl = cg + ic;
          mbar_wait(&S.b_full[cgl % kTcBRing], uint32_t((cgl / kTcBRing) & 1));
        }
        tc_fence_after();
        const uint32_t a0 = smem_u32(&S.A[ik][0]), b0 = smem_u32(&S.B[(cg + ic) % kTcBRing][0]);
        const uint32_t d = tmem + uint32_t(st * kTcN);
#pragma unroll
        for (int s = 0; s < 2; ++s)  // K = 16 steps: kchunks 2s, 2s + 1
          tc_mma(d, umma_desc(a0 + s * 4096, 2048, 128), umma_desc(b0 + s * 1024, 512, 128), s);
        tc_commit(&S.mma_done[st]);
        if (++ik == tiles) { ik = 0; ++ic; }
      }
    };
    for (int c = 0; c < kTcBRing; ++c) build_b(c, cg + c);
    fence_async_smem();
    __syncthreads();  // the A operand (built before the call) is complete
    if (tid == 0 && dbg != 2) issue_upto(min(T, kTcStages - 1));
    for (int k = 0; k < kTcTilesMax; ++k) { rsum[k] = 0.f; rmax[k] = -INFINITY; }
    float colsum[kTcChunks];  // lane l: this warp's sum of column l of each chunk (local memory: one store per chunk)
#pragma unroll 1
    for (int c = 0; c < kTcChunks; ++c) {  // not unrolled: the tile loop body is large (instruction cache)
      float2 cacc[kTcN / 2];
#pragma unroll
      for (int q = 0; q < kTcN / 2; ++q) cacc[q] = make_float2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < kTcTilesMax; ++k) {  // unrolled: the per-tile registers stay registers
        if (k >= tiles) break;
        const int t = c * tiles + k;  // tile of this pass
        const int tgl = tg + t;       // global tile index (barrier phases)
        if (tid == 0 && dbg != 2) issue_upto(min(T, t + kTcStages));
        __syncwarp();
        const int st = tgl & (kTcStages - 1);
        if (dbg != 2) mbar_wait(&S.mma_done[st], uint32_t((tgl / kTcStages) & 1));
        tc_fence_after();
        float v[32];
        tc_ld32(tmem + (uint32_t(warp * 32) << 16) + uint32_t(st * kTcN), v);
        tc_fence_before();
        __syncwarp();
        if (lane == 0 && dbg != 2) mbar_arrive(&S.s_free[st]);
        if (kExp && dbg == 3) {
          float2 r2 = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < kTcN / 2; ++q) {
            const float2 p = make_float2(v[2 * q], v[2 * q + 1]);
            r2 = __fadd2_rn(r2, p);
            cacc[q] = __ffma2_rn(p, make_float2(fr[k], fr[k]), cacc[q]);
          }
          rsum[k] += r2.x + r2.y;
        } else if (kExp) {
          const float f = fr[k];
          const float2 F = make_float2(f, f);
          float2 r2 = make_float2(0.f, 0.f), r3 = make_float2(0.f, 0.f);
#pragma unroll
          for (int q = 0; q < kTcN / 2; ++q) {
            const float2 p = make_float2(ex2f(v[2 * q]), ex2f(v[2 * q + 1]));
            if (q & 1) r3 = __fadd2_rn(r3, p); else r2 = __fadd2_rn(r2, p);
            cacc[q] = __ffma2_rn(p, F, cacc[q]);
          }
          const float2 r = __fadd2_rn(r2, r3);
          rsum[k] += r.x + r.y;
        } else {
          float m = v[0];
#pragma unroll
          for (int q = 1; q < 32; ++q) m = fmaxf(m, v[q]);
          rmax[k] = fmaxf(rmax[k], m);
        }
      }
      // every MMA of chunk c has completed (this warp consumed its tiles):
      // its operand buffer can take chunk c + kTcBRing
      if (c + kTcBRing < kTcChunks) build_b(c + kTcBRing, cg + c + kTcBRing);
      if (kExp) {  // butterfly reduce-scatter: lane l ends with the warp's sum of column l
        float x[kTcN];
#pragma unroll
        for (int q = 0; q < kTcN / 2; ++q) { x[2 * q] = cacc[q].x; x[2 * q + 1] = cacc[q].y; }
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
          const bool up = (lane & off) != 0;
#pragma unroll
          for (int q = 0; q < off; ++q) {
            const float send = up ? x[q] : x[q + off];
            const float keep = up ? x[q + off] : x[q];
            x[q] = keep + __shfl_xor_sync(0xffffffffu, send, off);
          }
        }
        colsum[c] = x[0];
      }
    }
    tg += T;
    cg += kTcChunks;
    __syncthreads();  // every MMA of the pass has completed: the A buffer is free
    if (kExp) {  // combine the 4 warps' column sums in a fixed order
      float* cw = reinterpret_cast<float*>(&S.A[0][0]);  // [warp][512]
#pragma unroll
      for (int c = 0; c < kTcChunks; ++c) cw[warp * kTcStrip + c * kTcN + lane] = colsum[c];
      __syncthreads();
      const float sig = S.red[0][0];
      for (int jj = tid; jj < kTcStrip; jj += kTcThreads) {
        const float sum = (cw[jj] + cw[kTcStrip + jj]) + (cw[2 * kTcStrip + jj] + cw[3 * kTcStrip + jj]);
        if (j0 + jj < n) reinterpret_cast<float2*>(a.colp)[(j0 + jj) * gridDim.y + blockIdx.y] = make_float2(sum, sig);
      }
      __syncthreads();  // before the A buffer is rebuilt
    }
  };
  auto set_scale = [&]() {  // CTA column scale sigma and f_i = 2^(s_i + A_i - sigma)
    float ls = -INFINITY;
#pragma unroll
    for (int k = 0; k < kTcTilesMax; ++k)
      if (k < tiles && r0 + 128 * k + tid < r1 && sr[k] < 1e29f) ls = fmaxf(ls, sr[k] + Ar[k]);
    ls = warp_maxf(ls);
    __syncthreads();
    if (lane == 0) S.red[1][warp] = ls;
    __syncthreads();
    float sig = -INFINITY;
    for (int ww = 0; ww < 4; ++ww) sig = fmaxf(sig, S.red[1][ww]);
#pragma unroll
    for (int k = 0; k < kTcTilesMax; ++k)
      fr[k] = (sig > -INFINITY && sr[k] < 1e29f && Ar[k] > -INFINITY) ? ex2f(sr[k] + Ar[k] - sig) : 0.f;
    if (tid == 0) S.red[0][0] = sig == -INFINITY ? 0.f : sig;  // read by the column-partial writers after a barrier
  };
  if (!carried) {
    // exact shifts: a pass without exponentials gives each row's segment max
    float zero[kTcTilesMax];
#pragma unroll
    for (int k = 0; k < kTcTilesMax; ++k) zero[k] = 0.f;
    build_a(zero);
    run(false);
#pragma unroll
    for (int k = 0; k < kTcTilesMax; ++k) {
      const bool live = k < tiles && r0 + 128 * k + tid < r1;
      // a row with no finite entry in the strip (or non-finite potentials,
      // caught by the evaluation's potential checks) is left out: partial 0
      sr[k] = (!live || !(rmax[k] > -1e29f)) ? 1e30f : rmax[k];
    }
  }
  set_scale();
  build_a(sr);
  run(dbg != 1);
  // row partials, carries, the bound of the max exponent
  float ub = -INFINITY;
  int ubnan = 0;
  const int64_t ldp = gridDim.x;
  float2* rowp = reinterpret_cast<float2*>(a.rowp);
#pragma unroll
  for (int k = 0; k < kTcTilesMax; ++k) {
    const int64_t i = r0 + 128 * k + tid;
    if (k < tiles && i < r1) {
      const bool empty = !(sr[k] < 1e29f) || rsum[k] == 0.f;
      const float ms = empty ? 0.f : sr[k];
      rowp[i * ldp + blockIdx.x] = make_float2(empty ? 0.f : rsum[k], ms);
      float lg;
      asm("lg2.approx.ftz.f32 %0, %1;" : "=f"(lg) : "f"(rsum[k]));
      const float c = empty ? -INFINITY : ms + lg;
      a.carry[int64_t(blockIdx.x) * n + i] = c;
      const float u = c + Ar[k];
      ubnan |= u != u;
      ub = fmaxf(ub, u);
    }
  }
  ubnan = __syncthreads_or(ubnan);
  ub = warp_maxf(ub);
  if (lane == 0) S.red[2][warp] = ub;
  __syncthreads();
  float cub = S.red[2][0];
  for (int ww = 1; ww < 4; ++ww) cub = fmaxf(cub, S.red[2][ww]);
  if (ubnan) cub = NAN;
  if (double(cub) * kLn2 > kMaxExponent - 10.0) {  // near the overflow threshold: the exact max
    build_a(sr);
    run(false);
    float m = -INFINITY;
#pragma unroll
    for (int k = 0; k < kTcTilesMax; ++k)
      if (k < tiles && r0 + 128 * k + tid < r1 && sr[k] < 1e29f && rmax[k] > -1e29f) m = fmaxf(m, rmax[k] + sr[k] + Ar[k]);
    m = warp_maxf(m);
    __syncthreads();
    if (lane == 0) S.red[2][warp] = m;
    __syncthreads();
    cub = S.red[2][0];
    for (int ww = 1; ww < 4; ++ww) cub = fmaxf(cub, S.red[2][ww]);
  }
  if (tid == 0) a.maxp[int64_t(blockIdx.y) * gridDim.x + blockIdx.x] = double(cub) * kLn2;
  if (a.carry_stats && tid == 0) atomicAdd(a.carry_stats + (carried ? 0 : 1), 1ull);
  // the strip's column constants for the next launch (last CTA of the strip, by ticket)
  if (tid == 0) {
    __threadfence();
    S.last = atomicAdd(a.carry_ticket + blockIdx.x, 1u) == gridDim.y - 1;
  }
  tc_fence_before();
  __syncthreads();
  if (S.last) {
    for (int jj = tid; jj < kTcStrip; jj += kTcThreads) {
      const float b = S.colB[jj];
      if (j0 + jj < n) a.carry_b[j0 + jj] = b <= -1e30f ? -INFINITY : b;
    }
    if (tid == 0) a.carry_ticket[blockIdx.x] = 0u;
  }
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTcTmemCols) : "memory");
  }
}

}  // namespace potgpu
