// SIMT fp32 kernel ladder: one sm_100a kernel per ELEVATE/TVM schedule.
//
// Each kernel is the B200 lowering of the low-level patterns the schedule's
// rewrite leaves in the `mm` term (reference rules.py:391-456, 516-549):
//   mapSeq/reduceSeq           -> per-thread loops             (K0)
//   tile(32,32) (split+interchange) -> 32x32 CTA tile in SMEM  (K1, K2)
//   split(4) + reorder (liftReduce, absorbReduceInit) -> k loop outside the
//                                 in-tile loops, sequential fold per element
//   mapVec (vectorize(32) of yi) -> 128-bit loads/stores       (K2..K6)
//   reorder (loopPerm)         -> register outer-product tiles (K3..K6)
//   packB / toMem(packed)      -> packedB[N/32][K][32] panels  (K4..K6)
//   toMem(acc) + unroll        -> 8x8 register accumulators    (K5, K6)
//   mapPar (outer row blocks)  -> persistent grid over all SMs (K6)
// Everything computes in fp32 with FFMA; the f64 reference (interp.py:145-148)
// is matched within the sqrt(K)-scaled bound of SURVEY.md §8(d).
//
// All kernels take arbitrary M, N, K >= 1 (predicated tails, SURVEY.md §7
// hard part 2) and any leading dimensions; 128-bit paths are used only when
// the operand is 16-byte aligned, otherwise the same kernel loads scalars.

#include "elv_common.cuh"

#include <stdlib.h>

namespace elv {
namespace {

__device__ __forceinline__ bool aligned16(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) & 15u) == 0;
}

// sm_100 packed FP32: FFMA2 does two IEEE fp32 FMAs (each rounded exactly
// like fmaf, so results are bitwise those of the scalar kernels) per issue
// slot.  The A value is broadcast into both halves -- ptxas folds the
// {a, a} pack into the FFMA2's .F32 scalar-operand form -- and B / the
// accumulators are adjacent column pairs.  Halving the FMA instruction
// count relieves the issue / register-bank dispatch stalls that hold the
// scalar 8x16 kernel at ~71 % of the FFMA peak.
__device__ __forceinline__ unsigned long long pack2(float lo, float hi) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
__device__ __forceinline__ float2 unpack2(unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}


// ---------------------------------------------------------------------------
// K0 baseline: mapSeq(arow => mapSeq(bcol => reduceSeq(acc + a*b)(0)(zip)))
// One thread per C(i,j); `transpose(b)` is a strided view (column reads of B
// are coalesced across the warp's j), the k loop is the reduceSeq.
__global__ void __launch_bounds__(256)
k0_baseline(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
            int M, int N, int K, int lda, int ldb, int ldc) {
  const int j = blockIdx.x * 32 + threadIdx.x;
  const int i = blockIdx.y * 8 + threadIdx.y;
  if (i >= M || j >= N) return;
  const float* a = A + (size_t)i * lda;
  const float* b = B + j;
  float acc = 0.f;
  for (int k = 0; k < K; ++k) acc = fmaf(__ldg(a + k), __ldg(b + (size_t)k * ldb), acc);
  C[(size_t)i * ldc + j] = acc;
}

// ---------------------------------------------------------------------------
// K1 blocking: TVM order (xo, yo, ko, ki, xi, yi).  (xo, yo) -> one 32x32 C
// tile per CTA with A/B tiles staged in SMEM; (ko, ki) -> the k loop, chunks
// of 4, outside the in-tile loops; (xi, yi) -> the CTA's threads.  Each
// element accumulates sequentially in k, the lowered term's fold
// (absorbReduceInit makes it acc + p0 + p1 + ..., not per-chunk sums).
constexpr int K1_BK = 32;
__global__ void __launch_bounds__(256)
k1_blocking(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
            int M, int N, int K, int lda, int ldb, int ldc) {
  __shared__ float As[32][K1_BK + 1];
  __shared__ float Bs[K1_BK][32];
  const int tx = threadIdx.x, ty = threadIdx.y;    // 32 x 8
  const int row0 = blockIdx.y * 32, col0 = blockIdx.x * 32;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < K; k0 += K1_BK) {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      const int rr = ty + 8 * r;
      const int gi = row0 + rr, gk = k0 + tx;
      As[rr][tx] = (gi < M && gk < K) ? __ldg(A + (size_t)gi * lda + gk) : 0.f;
      const int bk = k0 + rr, bj = col0 + tx;
      Bs[rr][tx] = (bk < K && bj < N) ? __ldg(B + (size_t)bk * ldb + bj) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kc = 0; kc < K1_BK; kc += 4) {          // ko: chunks of split(4)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)                   // ki
#pragma unroll
        for (int r = 0; r < 4; ++r)                    // xi (this thread's rows); yi = tx
          acc[r] = fmaf(As[ty + 8 * r][kc + kk], Bs[kc + kk][tx], acc[r]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int gi = row0 + ty + 8 * r, gj = col0 + tx;
    if (gi < M && gj < N) C[(size_t)gi * ldc + gj] = acc[r];
  }
}

// ---------------------------------------------------------------------------
// K2 vectorized: K1 plus vectorize(yi) -> 128-bit (float4) global loads and
// stores and float4 SMEM reads of B; each thread owns 1 row x 4 columns.
__global__ void __launch_bounds__(256)
k2_vectorized(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
              int M, int N, int K, int lda, int ldb, int ldc) {
  __shared__ float As[32][K1_BK + 1];
  __shared__ __align__(16) float Bs[K1_BK][32];
  const int tid = threadIdx.x;
  const int r = tid >> 3, c4 = (tid & 7) * 4;
  const int row0 = blockIdx.y * 32, col0 = blockIdx.x * 32;
  const bool vecA = aligned16(A) && (lda & 3) == 0;
  const bool vecB = aligned16(B) && (ldb & 3) == 0;
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (int k0 = 0; k0 < K; k0 += K1_BK) {
    {  // A tile: row r, k = k0 + c4 .. +3
      const int gi = row0 + r, gk = k0 + c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gi < M) {
        const float* p = A + (size_t)gi * lda + gk;
        if (vecA && gk + 3 < K) v = __ldg(reinterpret_cast<const float4*>(p));
        else {
          if (gk + 0 < K) v.x = __ldg(p + 0);
          if (gk + 1 < K) v.y = __ldg(p + 1);
          if (gk + 2 < K) v.z = __ldg(p + 2);
          if (gk + 3 < K) v.w = __ldg(p + 3);
        }
      }
      As[r][c4 + 0] = v.x; As[r][c4 + 1] = v.y; As[r][c4 + 2] = v.z; As[r][c4 + 3] = v.w;
    }
    {  // B tile: k row r, columns col0 + c4 .. +3
      const int gk = k0 + r, gj = col0 + c4;
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (gk < K) {
        const float* p = B + (size_t)gk * ldb + gj;
        if (vecB && gj + 3 < N) v = __ldg(reinterpret_cast<const float4*>(p));
        else {
          if (gj + 0 < N) v.x = __ldg(p + 0);
          if (gj + 1 < N) v.y = __ldg(p + 1);
          if (gj + 2 < N) v.z = __ldg(p + 2);
          if (gj + 3 < N) v.w = __ldg(p + 3);
        }
      }
      *reinterpret_cast<float4*>(&Bs[r][c4]) = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K1_BK; ++k) {                // ko, ki
      const float a = As[r][k];
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][c4]);   // yi, vectorised
      acc[0] = fmaf(a, b.x, acc[0]); acc[1] = fmaf(a, b.y, acc[1]);
      acc[2] = fmaf(a, b.z, acc[2]); acc[3] = fmaf(a, b.w, acc[3]);
    }
    __syncthreads();
  }
  const int gi = row0 + r, gj = col0 + c4;
  if (gi < M) {
    float* p = C + (size_t)gi * ldc + gj;
    if (aligned16(C) && (ldc & 3) == 0 && gj + 3 < N) {
      *reinterpret_cast<float4*>(p) = make_float4(acc[0], acc[1], acc[2], acc[3]);
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) if (gj + q < N) p[q] = acc[q];
    }
  }
}

// ---------------------------------------------------------------------------
// Shared loaders for the register-tiled kernels.
// A tile (BM rows x BK k) is stored transposed in SMEM: As[k][m].
template <int BM, int BK>
__device__ __forceinline__ float4 load_a4(const float* __restrict__ A, int M, int K, int lda,
                                          bool vecA, int gi, int gk) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (gi < M) {
    const float* p = A + (size_t)gi * lda + gk;
    if (vecA && gk + 3 < K) v = __ldg(reinterpret_cast<const float4*>(p));
    else {
      if (gk + 0 < K) v.x = __ldg(p + 0);
      if (gk + 1 < K) v.y = __ldg(p + 1);
      if (gk + 2 < K) v.z = __ldg(p + 2);
      if (gk + 3 < K) v.w = __ldg(p + 3);
    }
  }
  return v;
}

__device__ __forceinline__ float4 load_b4_rowmajor(const float* __restrict__ B, int N, int K, int ldb,
                                                   bool vecB, int gk, int gj) {
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (gk < K) {
    const float* p = B + (size_t)gk * ldb + gj;
    if (vecB && gj + 3 < N) v = __ldg(reinterpret_cast<const float4*>(p));
    else {
      if (gj + 0 < N) v.x = __ldg(p + 0);
      if (gj + 1 < N) v.y = __ldg(p + 1);
      if (gj + 2 < N) v.z = __ldg(p + 2);
      if (gj + 3 < N) v.w = __ldg(p + 3);
    }
  }
  return v;
}

// packedB[p][k][c]: rows of 32 floats; always 16B-aligned, zero past N
__device__ __forceinline__ float4 load_b4_packed(const float* __restrict__ P, int K, int gk, int gj) {
  if (gk >= K) return make_float4(0.f, 0.f, 0.f, 0.f);
  const int p = gj >> 5, c = gj & 31;
  return __ldg(reinterpret_cast<const float4*>(P + ((size_t)p * K + gk) * kPanel + c));
}

// ---------------------------------------------------------------------------
// K3 loopPerm / K4 arrayPacking: TVM order (xo, yo, ko, xi, ki, yi): 64x64
// CTA tile, 16x16 threads, each thread a 4x4 register outer product per k
// (xi outside ki: a thread's rows of A stay in registers while k sweeps,
// yi vectorised in float4).
// PACKED selects packedB panels (arrayPacking's toMem) over row-major B.
#ifndef ELV_K34_FFMA2
#define ELV_K34_FFMA2 1
#endif
template <bool PACKED>
__global__ void __launch_bounds__(256)
k34_outer4x4(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ C,
             int M, int N, int K, int lda, int ldb, int ldc) {
  constexpr int BM = 64, BN = 64, BK = 8;
  __shared__ __align__(16) float As[BK][BM + 4];
  __shared__ __align__(16) float Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int row0 = blockIdx.y * BM, col0 = blockIdx.x * BN;
  const bool vecA = aligned16(A) && (lda & 3) == 0;
  const bool vecB = PACKED || (aligned16(B) && (ldb & 3) == 0);
#if ELV_K34_FFMA2
  unsigned long long acc2[4][2];                   // column pairs, FFMA2 (bitwise = fmaf)
#pragma unroll
  for (int i = 0; i < 4; ++i) acc2[i][0] = acc2[i][1] = 0ull;
#else
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
#endif

  // A: 64 rows x 8 k = 128 float4 (threads 0..127); B: 8 x 64 = 128 float4 (threads 128..255)
  for (int k0 = 0; k0 < K; k0 += BK) {
    if (tid < 128) {
      const int r = tid >> 1, kq = (tid & 1) * 4;
      const float4 v = load_a4<BM, BK>(A, M, K, lda, vecA, row0 + r, k0 + kq);
      As[kq + 0][r] = v.x; As[kq + 1][r] = v.y; As[kq + 2][r] = v.z; As[kq + 3][r] = v.w;
    } else {
      const int t = tid - 128;
      const int kr = t >> 4, c4 = (t & 15) * 4;
      float4 v;
      if (PACKED) v = load_b4_packed(B, K, k0 + kr, col0 + c4);
      else v = load_b4_rowmajor(B, N, K, ldb, vecB, k0 + kr, col0 + c4);
      *reinterpret_cast<float4*>(&Bs[kr][c4]) = v;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      const float4 a = *reinterpret_cast<const float4*>(&As[k][ty * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[k][tx * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
#if ELV_K34_FFMA2
      const unsigned long long b01 = pack2(b.x, b.y), b23 = pack2(b.z, b.w);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const unsigned long long ai = pack2(av[i], av[i]);
        ffma2(acc2[i][0], ai, b01);
        ffma2(acc2[i][1], ai, b23);
      }
#else
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
#endif
    }
    __syncthreads();
  }
  const bool vecC = aligned16(C) && (ldc & 3) == 0;
#if ELV_K34_FFMA2
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 lo = unpack2(acc2[i][0]), hi = unpack2(acc2[i][1]);
    acc[i][0] = lo.x; acc[i][1] = lo.y; acc[i][2] = hi.x; acc[i][3] = hi.y;
  }
#endif
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gi = row0 + ty * 4 + i, gj = col0 + tx * 4;
    if (gi >= M) continue;
    float* p = C + (size_t)gi * ldc + gj;
    if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    else
#pragma unroll
      for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = acc[i][j];
  }
}

// ---------------------------------------------------------------------------
// K5 cacheBlocks / K6 parallel: 128x128 CTA tile over packedB, 8 warps laid
// out 2 (M) x 4 (N), warp tile 64x32, lane grid 8 x 4, each thread an 8x8
// register accumulator block (the toMem'd block accumulator of cache_write),
// k unrolled by BK=8 (reduceSeqUnroll).
//   K5: one tile per CTA, single-buffered SMEM.
//   K6: mapPar -> persistent CTAs (2 per SM) sweeping an L2-grouped tile
//       order, SMEM double-buffered with register prefetch of the next
//       k-block so global latency overlaps the FFMA stream.
constexpr int G_BM = 128, G_BN = 128, G_BK = 8, G_APAD = 4;

struct TileCoord { int m, n; };

__device__ __forceinline__ TileCoord tile_of(int t, int tiles_m, int tiles_n) {
  constexpr int GROUP = 8;                        // row-tiles per L2 group
  const int per_group = GROUP * tiles_n;
  const int g = t / per_group;
  const int first_m = g * GROUP;
  const int gm = min(tiles_m - first_m, GROUP);
  const int in = t - g * per_group;
  return {first_m + in % gm, in / gm};
}

// TBM = 128 (256 threads) or 64 (128 threads, small problems): the same
// 8x8 register accumulators per thread, half the rows per CTA.
#ifndef ELV_K56_FFMA2
#define ELV_K56_FFMA2 1
#endif
// Tuning build only (-DELV_K56_SHFL=1): the north star's
// "register tiles with warp-shuffle reuse" for cache_write -- each lane reads
// one value per operand row / column from SMEM and the 8 + 8 fragment values
// of its 8x8 tile come by __shfl_sync (16 shuffles + 3 LDS.32 per k instead
// of 4 LDS.128); the same values, so the same bits.
#ifndef ELV_K56_SHFL
#define ELV_K56_SHFL 0
#endif
#ifndef ELV_K56_MINB
#define ELV_K56_MINB 2
#endif
template <bool PARALLEL, int TBM = G_BM>
__global__ void __launch_bounds__(TBM * 2, ELV_K56_MINB)
k56_packed_8x8(const float* __restrict__ A, const float* __restrict__ P, float* __restrict__ C,
               int M, int N, int K, int lda, int ldc) {
  constexpr int NBUF = PARALLEL ? 2 : 1;
  constexpr int G_BM = TBM;
  constexpr int NT = TBM * 2;
  __shared__ __align__(16) float As[NBUF][G_BK][G_BM + G_APAD];
  __shared__ __align__(16) float Bs[NBUF][G_BK][G_BN];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;         // 2 x 4 warps
  const int lm = lane >> 2, ln = lane & 3;         // 8 x 4 lanes
  const int trow = wm * 64 + lm * 4;               // + {0..3} and +32
  const int tcol = wn * 32 + ln * 4;               // + {0..3} and +16
  const bool vecA = aligned16(A) && (lda & 3) == 0;
  const bool vecC = aligned16(C) && (ldc & 3) == 0;

  // loader roles: A float4 (row = tid/2, k = (tid&1)*4); B float4 from panel tid/64
  const int a_r = tid >> 1, a_k = (tid & 1) * 4;
  constexpr int BLD = 256 / NT;                    // float4 of B per thread per k-block

  const int tiles_m = (M + G_BM - 1) / G_BM, tiles_n = (N + G_BN - 1) / G_BN;
  const int num_tiles = tiles_m * tiles_n;
  const int first = PARALLEL ? (int)blockIdx.x : (int)(blockIdx.y * gridDim.x + blockIdx.x);
  const int stride = PARALLEL ? (int)gridDim.x : num_tiles;

  for (int t = first; t < num_tiles; t += stride) {
    TileCoord tc = PARALLEL ? tile_of(t, tiles_m, tiles_n) : TileCoord{(int)blockIdx.y, (int)blockIdx.x};
    const int row0 = tc.m * G_BM, col0 = tc.n * G_BN;
#if ELV_K56_FFMA2
    unsigned long long acc2[8][4];                 // column pairs, FFMA2 (bitwise = fmaf)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc2[i][j] = 0ull;
#else
    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;
#endif

    struct VB { float4 v[BLD]; };
    auto ldA = [&](int k0) { return load_a4<G_BM, G_BK>(A, M, K, lda, vecA, row0 + a_r, k0 + a_k); };
    auto ldB = [&](int k0) {
      VB r;
#pragma unroll
      for (int i = 0; i < BLD; ++i) {
        const int q = tid + i * NT;
        const int b_p = q >> 6, b_in = q & 63, b_k = b_in >> 3, b_c = (b_in & 7) * 4;
        const int gk = k0 + b_k;
        r.v[i] = gk < K ? __ldg(reinterpret_cast<const float4*>(P + ((size_t)((col0 >> 5) + b_p) * K + gk) * kPanel
                                                                + b_c))
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      return r;
    };
    auto stage = [&](int buf, float4 va, const VB& vb) {
      As[buf][a_k + 0][a_r] = va.x; As[buf][a_k + 1][a_r] = va.y;
      As[buf][a_k + 2][a_r] = va.z; As[buf][a_k + 3][a_r] = va.w;
#pragma unroll
      for (int i = 0; i < BLD; ++i) {
        const int q = tid + i * NT;
        const int b_p = q >> 6, b_in = q & 63, b_k = b_in >> 3, b_c = (b_in & 7) * 4;
        *reinterpret_cast<float4*>(&Bs[buf][b_k][b_p * 32 + b_c]) = vb.v[i];
      }
    };
    auto compute = [&](int buf) {
#pragma unroll
      for (int k = 0; k < G_BK; ++k) {
#if ELV_K56_SHFL
        const float a_lo = As[buf][k][wm * 64 + lane], a_hi = As[buf][k][wm * 64 + 32 + lane];
        const float b_l = Bs[buf][k][wn * 32 + lane];
        float av[8];
        float4 b0, b1;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          av[i] = __shfl_sync(0xffffffffu, a_lo, lm * 4 + i);
          av[4 + i] = __shfl_sync(0xffffffffu, a_hi, lm * 4 + i);
        }
        b0.x = __shfl_sync(0xffffffffu, b_l, ln * 4 + 0); b0.y = __shfl_sync(0xffffffffu, b_l, ln * 4 + 1);
        b0.z = __shfl_sync(0xffffffffu, b_l, ln * 4 + 2); b0.w = __shfl_sync(0xffffffffu, b_l, ln * 4 + 3);
        b1.x = __shfl_sync(0xffffffffu, b_l, 16 + ln * 4 + 0); b1.y = __shfl_sync(0xffffffffu, b_l, 16 + ln * 4 + 1);
        b1.z = __shfl_sync(0xffffffffu, b_l, 16 + ln * 4 + 2); b1.w = __shfl_sync(0xffffffffu, b_l, 16 + ln * 4 + 3);
#else
        const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][trow]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][trow + 32]);
        const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tcol]);
        const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][tcol + 16]);
        const float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#endif
#if ELV_K56_FFMA2
        const unsigned long long bp[4] = {pack2(b0.x, b0.y), pack2(b0.z, b0.w), pack2(b1.x, b1.y),
                                          pack2(b1.z, b1.w)};
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const unsigned long long ai = pack2(av[i], av[i]);
#pragma unroll
          for (int j = 0; j < 4; ++j) ffma2(acc2[i][j], ai, bp[j]);
        }
#else
        const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
#endif
      }
    };

    if (PARALLEL) {
      float4 va = ldA(0);
      VB vb = ldB(0);
      stage(0, va, vb);
      __syncthreads();
      int buf = 0;
      for (int k0 = 0; k0 < K; k0 += G_BK) {
        const bool more = k0 + G_BK < K;
        if (more) { va = ldA(k0 + G_BK); vb = ldB(k0 + G_BK); }
        compute(buf);
        if (more) stage(buf ^ 1, va, vb);
        __syncthreads();
        buf ^= 1;
      }
    } else {
      for (int k0 = 0; k0 < K; k0 += G_BK) {
        stage(0, ldA(k0), ldB(k0));
        __syncthreads();
        compute(0);
        __syncthreads();
      }
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gi = row0 + trow + (i & 3) + (i >> 2) * 32;
      if (gi >= M) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = col0 + tcol + h * 16;
        float* p = C + (size_t)gi * ldc + gj;
#if ELV_K56_FFMA2
        const float2 lo = unpack2(acc2[i][2 * h]), hi = unpack2(acc2[i][2 * h + 1]);
        const float v[4] = {lo.x, lo.y, hi.x, hi.y};
#else
        const float* v = &acc[i][h * 4];
#endif
        if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = v[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K6 parallel (tuned): 128x128 CTA tile over packedB, 8x8 per thread, SMEM
// double buffer with the next k-block prefetched into registers, and the
// next k-step's A/B fragments prefetched from SMEM while the current 64
// FFMAs issue (hides LDS latency -- the short_scoreboard stall of the plain
// K5 loop).  BK and blocks/SM are template parameters; ELV_SGEMM_CFG selects
// among the instantiations for tuning (default: the measured best).
template <int BK, int MINB>
__global__ void __launch_bounds__(256, MINB)
k6_sgemm_db(const float* __restrict__ A, const float* __restrict__ P, float* __restrict__ C,
            int M, int N, int K, int lda, int ldc) {
  constexpr int LA = BK / 8;                      // float4 loads of A per thread per k-block
  constexpr int LB = BK / 8;                      // float4 loads of B per thread per k-block
  __shared__ __align__(16) float As[2][BK][G_BM + G_APAD];
  __shared__ __align__(16) float Bs[2][BK][G_BN];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int lm = lane >> 2, ln = lane & 3;
  const int trow = wm * 64 + lm * 4;
  const int tcol = wn * 32 + ln * 4;
  const bool vecA = aligned16(A) && (lda & 3) == 0;
  const bool vecC = aligned16(C) && (ldc & 3) == 0;

  // A loader: float4 index q = tid + i*256 over (row, k4) with k4 fastest
  constexpr int K4 = BK / 4;
  // B loader: float4 index q = tid + i*256 over (panel, k, c4) with c4 fastest
  constexpr int PANEL4 = BK * 8;                  // float4 per panel per k-block

  const int tiles_m = (M + G_BM - 1) / G_BM, tiles_n = (N + G_BN - 1) / G_BN;
  const int num_tiles = tiles_m * tiles_n;

  for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    const TileCoord tc = tile_of(t, tiles_m, tiles_n);
    const int row0 = tc.m * G_BM, col0 = tc.n * G_BN;
    const float* Pbase = P + (size_t)(col0 >> 5) * K * kPanel;

    float4 ra[LA], rb[LB];
    auto gload = [&](int k0) {
#pragma unroll
      for (int i = 0; i < LA; ++i) {
        const int q = tid + i * 256;
        const int r = q / K4, kq = (q % K4) * 4;
        ra[i] = load_a4<G_BM, BK>(A, M, K, lda, vecA, row0 + r, k0 + kq);
      }
#pragma unroll
      for (int i = 0; i < LB; ++i) {
        const int q = tid + i * 256;
        const int pnl = q / PANEL4, w = q % PANEL4;
        const int kk = w >> 3, c4 = (w & 7) * 4;
        const int gk = k0 + kk;
        rb[i] = gk < K ? __ldg(reinterpret_cast<const float4*>(Pbase + ((size_t)pnl * K + gk) * kPanel + c4))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto sstore = [&](int buf) {
#pragma unroll
      for (int i = 0; i < LA; ++i) {
        const int q = tid + i * 256;
        const int r = q / K4, kq = (q % K4) * 4;
        As[buf][kq + 0][r] = ra[i].x; As[buf][kq + 1][r] = ra[i].y;
        As[buf][kq + 2][r] = ra[i].z; As[buf][kq + 3][r] = ra[i].w;
      }
#pragma unroll
      for (int i = 0; i < LB; ++i) {
        const int q = tid + i * 256;
        const int pnl = q / PANEL4, w = q % PANEL4;
        *reinterpret_cast<float4*>(&Bs[buf][w >> 3][pnl * 32 + (w & 7) * 4]) = rb[i];
      }
    };

    float acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

    gload(0);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += BK) {
      const bool more = k0 + BK < K;
      if (more) gload(k0 + BK);
      float a[2][8], b[2][8];
      auto lfrag = [&](int slot, int k) {
        const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][trow]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][trow + 32]);
        const float4 b0 = *reinterpret_cast<const float4*>(&Bs[buf][k][tcol]);
        const float4 b1 = *reinterpret_cast<const float4*>(&Bs[buf][k][tcol + 16]);
        a[slot][0] = a0.x; a[slot][1] = a0.y; a[slot][2] = a0.z; a[slot][3] = a0.w;
        a[slot][4] = a1.x; a[slot][5] = a1.y; a[slot][6] = a1.z; a[slot][7] = a1.w;
        b[slot][0] = b0.x; b[slot][1] = b0.y; b[slot][2] = b0.z; b[slot][3] = b0.w;
        b[slot][4] = b1.x; b[slot][5] = b1.y; b[slot][6] = b1.z; b[slot][7] = b1.w;
      };
      lfrag(0, 0);
#pragma unroll
      for (int k = 0; k < BK; ++k) {
        if (k + 1 < BK) lfrag((k + 1) & 1, k + 1);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[k & 1][i], b[k & 1][j], acc[i][j]);
      }
      if (more) sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gi = row0 + trow + (i & 3) + (i >> 2) * 32;
      if (gi >= M) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gj = col0 + tcol + h * 16;
        float* p = C + (size_t)gi * ldc + gj;
        const float* v = &acc[i][h * 4];
        if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = v[j];
      }
    }
  }
}

// 128x256 CTA tile, 8x16 per thread (128 accumulators, 1 CTA of 8 warps per
// SM): 128 FFMA per 6 LDS.128 per k-step instead of 64 per 4.
template <int BK>
__global__ void __launch_bounds__(256, 1)
k6_sgemm_8x16(const float* __restrict__ A, const float* __restrict__ P, float* __restrict__ C,
              int M, int N, int K, int lda, int ldc) {
  constexpr int BM = 128, BN = 256;
  constexpr int LA = BM * BK / 4 / 256;           // float4 of A per thread per k-block
  constexpr int LB = BN * BK / 4 / 256;           // float4 of B per thread per k-block
  constexpr int K4 = BK / 4;
  constexpr int PANEL4 = BK * 8;
  __shared__ __align__(16) float As[2][BK][BM + G_APAD];
  __shared__ __align__(16) float Bs[2][BK][BN];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;         // 2 x 4 warps, warp tile 64 x 64
  const int lm = lane >> 2, ln = lane & 3;         // 8 x 4 lanes
  const int trow = wm * 64 + lm * 4;               // rows +{0..3}, +32+{0..3}
  const int tcol = wn * 64 + ln * 4;               // cols +{0..3} +16h
  const bool vecA = aligned16(A) && (lda & 3) == 0;
  const bool vecC = aligned16(C) && (ldc & 3) == 0;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;

  for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    const TileCoord tc = tile_of(t, tiles_m, tiles_n);
    const int row0 = tc.m * BM, col0 = tc.n * BN;
    const float* Pbase = P + (size_t)(col0 >> 5) * K * kPanel;
    float4 ra[LA], rb[LB];
    auto gload = [&](int k0) {
#pragma unroll
      for (int i = 0; i < LA; ++i) {
        const int q = tid + i * 256;
        ra[i] = load_a4<BM, BK>(A, M, K, lda, vecA, row0 + q / K4, k0 + (q % K4) * 4);
      }
#pragma unroll
      for (int i = 0; i < LB; ++i) {
        const int q = tid + i * 256;
        const int pnl = q / PANEL4, w = q % PANEL4;
        const int gk = k0 + (w >> 3);
        rb[i] = gk < K ? __ldg(reinterpret_cast<const float4*>(Pbase + ((size_t)pnl * K + gk) * kPanel + (w & 7) * 4))
                       : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    };
    auto sstore = [&](int buf) {
#pragma unroll
      for (int i = 0; i < LA; ++i) {
        const int q = tid + i * 256;
        const int r = q / K4, kq = (q % K4) * 4;
        As[buf][kq + 0][r] = ra[i].x; As[buf][kq + 1][r] = ra[i].y;
        As[buf][kq + 2][r] = ra[i].z; As[buf][kq + 3][r] = ra[i].w;
      }
#pragma unroll
      for (int i = 0; i < LB; ++i) {
        const int q = tid + i * 256;
        const int pnl = q / PANEL4, w = q % PANEL4;
        *reinterpret_cast<float4*>(&Bs[buf][w >> 3][pnl * 32 + (w & 7) * 4]) = rb[i];
      }
    };
    unsigned long long acc[8][8];                  // [row][column pair], FFMA2
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;
    gload(0);
    sstore(0);
    __syncthreads();
    int buf = 0;
    for (int k0 = 0; k0 < K; k0 += BK) {
      const bool more = k0 + BK < K;
      if (more) gload(k0 + BK);
#pragma unroll
      for (int k = 0; k < BK; ++k) {
        float a[8];
        unsigned long long b[8];
        const float4 a0 = *reinterpret_cast<const float4*>(&As[buf][k][trow]);
        const float4 a1 = *reinterpret_cast<const float4*>(&As[buf][k][trow + 32]);
        a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
        a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float4 bv = *reinterpret_cast<const float4*>(&Bs[buf][k][tcol + 16 * h]);
          b[2 * h] = pack2(bv.x, bv.y);
          b[2 * h + 1] = pack2(bv.z, bv.w);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const unsigned long long ai = pack2(a[i], a[i]);
#pragma unroll
          for (int j = 0; j < 8; ++j) ffma2(acc[i][j], ai, b[j]);
        }
      }
      if (more) sstore(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gi = row0 + trow + (i & 3) + (i >> 2) * 32;
      if (gi >= M) continue;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int gj = col0 + tcol + h * 16;
        float* p = C + (size_t)gi * ldc + gj;
        const float2 lo = unpack2(acc[i][2 * h]), hi = unpack2(acc[i][2 * h + 1]);
        const float v[4] = {lo.x, lo.y, hi.x, hi.y};
        if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = v[j];
      }
    }
  }
}

// ---------------------------------------------------------------------------
// K6 on packed operands (the default `parallel` path of elv_gemm): A is
// packed by the prepass like B (packedA[M/128][K][128], the "packB" treatment
// applied to the other operand), so every k-block of both tiles is a
// contiguous run of 16-byte chunks.  The main loop is then a multi-stage
// cp.async (LDGSTS) pipeline with no register staging and no transposing
// stores, and the registers that frees hold a second A/B fragment set so the
// next k-step's LDS overlap the current 128 FFMAs.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// k-block depth x ring stages of the cp.async SIMT kernels: 32 x 3 (144 KB)
// measured +1.5 % over 16 x 4 at the bench shape (60.4 -> 61.2 TF; one
// barrier per 32 k instead of 16); 32 x 4 +0.7 %, 16 x 6 -1 %
// (profiles/r1/small/k6_bk_stages.jsonl)
#ifndef ELV_CP_BK
#define ELV_CP_BK 32
#endif
#ifndef ELV_CP_STAGES
#define ELV_CP_STAGES 3
#endif
constexpr int CP_BK = ELV_CP_BK, CP_STAGES = ELV_CP_STAGES;
constexpr int CP_SMEM = CP_STAGES * CP_BK * (128 + 256) * 4;    // 144 KB at 32 x 3

template <int ORDER>
__global__ void __launch_bounds__(256, 1)
k6_sgemm_cp(const float* __restrict__ PA, const float* __restrict__ PB, float* __restrict__ C,
            int M, int N, int K, int ldc) {
  extern __shared__ __align__(16) float smem_f[];
  float* As = smem_f;                               // [STAGES][BK][128]
  float* Bs = smem_f + CP_STAGES * CP_BK * 128;     // [STAGES][BK][256]
  constexpr int BM = 128, BN = 256;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int lm = lane >> 2, ln = lane & 3;
  const int trow = wm * 64 + lm * 4;
  const int tcol = wn * 64 + ln * 4;
  const bool vecC = aligned16(C) && (ldc & 3) == 0;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int nkb = (K + CP_BK - 1) / CP_BK;

  griddep_wait();                                   // packed operands from k_pack_ab
  for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    const TileCoord tc = tile_of(t, tiles_m, tiles_n);
    const int row0 = tc.m * BM, col0 = tc.n * BN;
    const float* pa = PA + (size_t)tc.m * K * BM;
    const float* pb = PB + (size_t)(col0 >> 5) * K * kPanel;
    auto issue = [&](int kb, int slot) {
      const int k0 = kb * CP_BK;
#pragma unroll
      for (int i = 0; i < CP_BK * 32 / 256; ++i) {          // A: BK rows of 128 floats
        const int q = tid + i * 256;
        const int kk = q >> 5, c4 = (q & 31) * 4;
        const int gk = k0 + kk;
        cp_async16(&As[(slot * CP_BK + kk) * BM + c4], pa + (size_t)min(gk, K - 1) * BM + c4, gk < K ? 16 : 0);
      }
#pragma unroll
      for (int i = 0; i < CP_BK * 64 / 256; ++i) {          // B: 8 panels x BK rows x 32 floats
        const int q = tid + i * 256;
        const int pnl = q / (CP_BK * 8), w = q % (CP_BK * 8);
        const int kk = w >> 3, c4 = (w & 7) * 4;
        const int gk = k0 + kk;
        cp_async16(&Bs[(slot * CP_BK + kk) * BN + pnl * 32 + c4],
                   pb + ((size_t)pnl * K + min(gk, K - 1)) * kPanel + c4, gk < K ? 16 : 0);
      }
    };

    float acc[8][16];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 16; ++j) acc[i][j] = 0.f;

#pragma unroll
    for (int st = 0; st < CP_STAGES - 1; ++st) {
      if (st < nkb) issue(st, st);
      cp_async_commit();
    }
    for (int kb = 0; kb < nkb; ++kb) {
      cp_async_wait<CP_STAGES - 2>();
      __syncthreads();
      const int nk = kb + CP_STAGES - 1;
      if (nk < nkb) issue(nk, nk % CP_STAGES);
      cp_async_commit();
      const float* as = As + (kb % CP_STAGES) * CP_BK * BM;
      const float* bs = Bs + (kb % CP_STAGES) * CP_BK * BN;
      float a[2][8], b[2][16];
      auto lfrag = [&](int slot, int k) {
        const float4 a0 = *reinterpret_cast<const float4*>(as + k * BM + trow);
        const float4 a1 = *reinterpret_cast<const float4*>(as + k * BM + trow + 32);
        a[slot][0] = a0.x; a[slot][1] = a0.y; a[slot][2] = a0.z; a[slot][3] = a0.w;
        a[slot][4] = a1.x; a[slot][5] = a1.y; a[slot][6] = a1.z; a[slot][7] = a1.w;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float4 bv = *reinterpret_cast<const float4*>(bs + k * BN + tcol + 16 * h);
          b[slot][4 * h] = bv.x; b[slot][4 * h + 1] = bv.y; b[slot][4 * h + 2] = bv.z; b[slot][4 * h + 3] = bv.w;
        }
      };
      lfrag(0, 0);
#pragma unroll
      for (int k = 0; k < CP_BK; ++k) {
        if (k + 1 < CP_BK) lfrag((k + 1) & 1, k + 1);
        if (ORDER == 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[i][j] = fmaf(a[k & 1][i], b[k & 1][j], acc[i][j]);
        } else if (ORDER == 1) {
#pragma unroll
          for (int j = 0; j < 16; ++j)
#pragma unroll
            for (int i = 0; i < 8; ++i) acc[i][j] = fmaf(a[k & 1][i], b[k & 1][j], acc[i][j]);
        } else {                                   // 2x2 blocks: both operands reused in pairs
#pragma unroll
          for (int i = 0; i < 8; i += 2)
#pragma unroll
            for (int j = 0; j < 16; j += 2) {
              acc[i][j] = fmaf(a[k & 1][i], b[k & 1][j], acc[i][j]);
              acc[i][j + 1] = fmaf(a[k & 1][i], b[k & 1][j + 1], acc[i][j + 1]);
              acc[i + 1][j + 1] = fmaf(a[k & 1][i + 1], b[k & 1][j + 1], acc[i + 1][j + 1]);
              acc[i + 1][j] = fmaf(a[k & 1][i + 1], b[k & 1][j], acc[i + 1][j]);
            }
        }
      }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gi = row0 + trow + (i & 3) + (i >> 2) * 32;
      if (gi >= M) continue;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int gj = col0 + tcol + h * 16;
        float* p = C + (size_t)gi * ldc + gj;
        const float* v = &acc[i][h * 4];
        if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = v[j];
      }
    }
    __syncthreads();                               // smem slots are reused by the next tile
  }
}

__global__ void __launch_bounds__(256, 1)
k6_sgemm_ffma2(const float* __restrict__ PA, const float* __restrict__ PB, float* __restrict__ C,
               int M, int N, int K, int ldc) {
  extern __shared__ __align__(16) float smem_f2[];
  float* As = smem_f2;                              // [STAGES][BK][128]
  float* Bs = smem_f2 + CP_STAGES * CP_BK * 128;    // [STAGES][BK][256]
  constexpr int BM = 128, BN = 256;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int lm = lane >> 2, ln = lane & 3;
  const int trow = wm * 64 + lm * 4;
  const int tcol = wn * 64 + ln * 4;
  const bool vecC = aligned16(C) && (ldc & 3) == 0;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int nkb = (K + CP_BK - 1) / CP_BK;

  griddep_wait();                                   // packed operands from k_pack_ab
  for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    const TileCoord tc = tile_of(t, tiles_m, tiles_n);
    const int row0 = tc.m * BM, col0 = tc.n * BN;
    const float* pa = PA + (size_t)tc.m * K * BM;
    const float* pb = PB + (size_t)(col0 >> 5) * K * kPanel;
    auto issue = [&](int kb, int slot) {
      const int k0 = kb * CP_BK;
#pragma unroll
      for (int i = 0; i < CP_BK * 32 / 256; ++i) {
        const int q = tid + i * 256;
        const int kk = q >> 5, c4 = (q & 31) * 4;
        const int gk = k0 + kk;
        cp_async16(&As[(slot * CP_BK + kk) * BM + c4], pa + (size_t)min(gk, K - 1) * BM + c4, gk < K ? 16 : 0);
      }
#pragma unroll
      for (int i = 0; i < CP_BK * 64 / 256; ++i) {
        const int q = tid + i * 256;
        const int pnl = q / (CP_BK * 8), w = q % (CP_BK * 8);
        const int kk = w >> 3, c4 = (w & 7) * 4;
        const int gk = k0 + kk;
        cp_async16(&Bs[(slot * CP_BK + kk) * BN + pnl * 32 + c4],
                   pb + ((size_t)pnl * K + min(gk, K - 1)) * kPanel + c4, gk < K ? 16 : 0);
      }
    };

    unsigned long long acc[8][8];                  // [row i][column pair]
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;

#pragma unroll
    for (int st = 0; st < CP_STAGES - 1; ++st) {
      if (st < nkb) issue(st, st);
      cp_async_commit();
    }
    for (int kb = 0; kb < nkb; ++kb) {
      cp_async_wait<CP_STAGES - 2>();
      __syncthreads();
      const int nk = kb + CP_STAGES - 1;
      if (nk < nkb) issue(nk, nk % CP_STAGES);
      cp_async_commit();
      const float* as = As + (kb % CP_STAGES) * CP_BK * BM;
      const float* bs = Bs + (kb % CP_STAGES) * CP_BK * BN;
      float a[2][8];
      unsigned long long b[2][8];
      auto lfrag = [&](int slot, int k) {
        const float4 a0 = *reinterpret_cast<const float4*>(as + k * BM + trow);
        const float4 a1 = *reinterpret_cast<const float4*>(as + k * BM + trow + 32);
        a[slot][0] = a0.x; a[slot][1] = a0.y; a[slot][2] = a0.z; a[slot][3] = a0.w;
        a[slot][4] = a1.x; a[slot][5] = a1.y; a[slot][6] = a1.z; a[slot][7] = a1.w;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const float4 bv = *reinterpret_cast<const float4*>(bs + k * BN + tcol + 16 * h);
          b[slot][2 * h] = pack2(bv.x, bv.y);
          b[slot][2 * h + 1] = pack2(bv.z, bv.w);
        }
      };
      lfrag(0, 0);
#pragma unroll
      for (int k = 0; k < CP_BK; ++k) {
        if (k + 1 < CP_BK) lfrag((k + 1) & 1, k + 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const unsigned long long ai = pack2(a[k & 1][i], a[k & 1][i]);
#pragma unroll
          for (int j = 0; j < 8; ++j) ffma2(acc[i][j], ai, b[k & 1][j]);
        }
      }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gi = row0 + trow + (i & 3) + (i >> 2) * 32;
      if (gi >= M) continue;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int gj = col0 + tcol + h * 16;
        float* p = C + (size_t)gi * ldc + gj;
        const float2 lo = unpack2(acc[i][2 * h]), hi = unpack2(acc[i][2 * h + 1]);
        const float v[4] = {lo.x, lo.y, hi.x, hi.y};
        if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = v[j];
      }
    }
    __syncthreads();
  }
}

// The same kernel with the tiles staged by the TMA engine (ELV_K6_BULK=1;
// K % 32 == 0): the packed panels are contiguous, so one thread issues a
// 1-D bulk copy (cp.async.bulk) per operand panel and k-block -- 16 KB of A,
// 8 x 4 KB of B, B staged panel-major [8][BK][32] -- onto the stage's
// mbarrier (complete_tx), consumers wait on it instead of cp.async groups +
// __syncthreads, and each warp releases the stage on an "empty" mbarrier.
// Same fragments, same FFMA2 sequence: bitwise k6_sgemm_ffma2.
__device__ __forceinline__ uint32_t s_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(s_u32(b)), "r"(n));
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t parity) {
  asm volatile("{\n.reg .pred p;\nBW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra BW_%=;\n}\n" ::"r"(
                   s_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   s_u32(dst)), "l"(src), "r"(bytes), "r"(s_u32(bar)) : "memory");
}

__global__ void __launch_bounds__(256, 1)
k6_sgemm_bulk(const float* __restrict__ PA, const float* __restrict__ PB, float* __restrict__ C,
              int M, int N, int K, int ldc) {
  extern __shared__ __align__(128) float smem_b[];
  float* As = smem_b;                               // [STAGES][BK][128]
  float* Bs = smem_b + CP_STAGES * CP_BK * 128;     // [STAGES][8 panels][BK][32]
  __shared__ __align__(8) uint64_t full[CP_STAGES], empty[CP_STAGES];
  constexpr int BM = 128, BN = 256;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int wm = warp >> 2, wn = warp & 3;
  const int lm = lane >> 2, ln = lane & 3;
  const int trow = wm * 64 + lm * 4;
  const int tcol = wn * 64 + ln * 4;
  const bool vecC = aligned16(C) && (ldc & 3) == 0;
  const int tiles_m = (M + BM - 1) / BM, tiles_n = (N + BN - 1) / BN;
  const int num_tiles = tiles_m * tiles_n;
  const int nkb = K / CP_BK;
  if (tid == 0) {
    for (int i = 0; i < CP_STAGES; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 8); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  griddep_wait();                                   // packed operands from k_pack_ab
  uint32_t g0 = 0;                                  // global stage counter (across tiles)
  for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, g0 += nkb) {
    const TileCoord tc = tile_of(t, tiles_m, tiles_n);
    const int row0 = tc.m * BM, col0 = tc.n * BN;
    const float* pa = PA + (size_t)tc.m * K * BM;
    const float* pb = PB + (size_t)(col0 >> 5) * K * kPanel;
    auto issue = [&](uint32_t g, int kb) {          // thread 0
      const int slot = g % CP_STAGES;
      if (g >= CP_STAGES) bar_wait(&empty[slot], ((g / CP_STAGES) & 1) ^ 1);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_u32(&full[slot])),
                   "r"((uint32_t)(CP_BK * (BM + BN) * 4)) : "memory");
      bulk_g2s(As + slot * CP_BK * BM, pa + (size_t)kb * CP_BK * BM, CP_BK * BM * 4, &full[slot]);
#pragma unroll
      for (int p = 0; p < 8; ++p)
        bulk_g2s(Bs + (slot * 8 + p) * CP_BK * kPanel, pb + ((size_t)p * K + (size_t)kb * CP_BK) * kPanel,
                 CP_BK * kPanel * 4, &full[slot]);
    };

    unsigned long long acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) acc[i][j] = 0ull;

    if (tid == 0)
      for (int st = 0; st < CP_STAGES - 1 && st < nkb; ++st) issue(g0 + st, st);
    for (int kb = 0; kb < nkb; ++kb) {
      const uint32_t g = g0 + kb;
      const int slot = g % CP_STAGES;
      if (tid == 0 && kb + CP_STAGES - 1 < nkb) issue(g + CP_STAGES - 1, kb + CP_STAGES - 1);
      bar_wait(&full[slot], (g / CP_STAGES) & 1);
      const float* as = As + slot * CP_BK * BM;
      const float* bs = Bs + slot * 8 * CP_BK * kPanel;
      float a[2][8];
      unsigned long long b[2][8];
      auto lfrag = [&](int sl, int k) {
        const float4 a0 = *reinterpret_cast<const float4*>(as + k * BM + trow);
        const float4 a1 = *reinterpret_cast<const float4*>(as + k * BM + trow + 32);
        a[sl][0] = a0.x; a[sl][1] = a0.y; a[sl][2] = a0.z; a[sl][3] = a0.w;
        a[sl][4] = a1.x; a[sl][5] = a1.y; a[sl][6] = a1.z; a[sl][7] = a1.w;
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int c = tcol + 16 * h;              // column within the 256-wide tile -> panel c / 32
          const float4 bv = *reinterpret_cast<const float4*>(bs + ((c >> 5) * CP_BK + k) * kPanel + (c & 31));
          b[sl][2 * h] = pack2(bv.x, bv.y);
          b[sl][2 * h + 1] = pack2(bv.z, bv.w);
        }
      };
      lfrag(0, 0);
#pragma unroll
      for (int k = 0; k < CP_BK; ++k) {
        if (k + 1 < CP_BK) lfrag((k + 1) & 1, k + 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const unsigned long long ai = pack2(a[k & 1][i], a[k & 1][i]);
#pragma unroll
          for (int j = 0; j < 8; ++j) ffma2(acc[i][j], ai, b[k & 1][j]);
        }
      }
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_u32(&empty[slot])) : "memory");
    }

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gi = row0 + trow + (i & 3) + (i >> 2) * 32;
      if (gi >= M) continue;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const int gj = col0 + tcol + h * 16;
        float* p = C + (size_t)gi * ldc + gj;
        const float2 lo = unpack2(acc[i][2 * h]), hi = unpack2(acc[i][2 * h + 1]);
        const float v[4] = {lo.x, lo.y, hi.x, hi.y};
        if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = v[j];
      }
    }
  }
}

// Small problems (fewer 128x256 tiles than SMs, e.g. 1024^3 -> 32): 64x64
// tiles so every SM gets work, 64 threads x 8x8 outputs (4 LDS.128 per 32
// FFMA2, so SMEM bandwidth is not the bound), the same packed operands and
// cp.async ring structure as k6_sgemm_cp.  A 64-row tile is one half of a
// 128-row packedA panel.  Same sequential fmaf chain per element.
// 32 x 3 (48 KB, 4 CTAs per SM): 1024^3 51.4 vs 55.3 us (16 x 4), +1 % at
// 2048^3 / 4096^3 (profiles/r1/small/k6_small_bk_stages.jsonl)
#ifndef ELV_SM_BK
#define ELV_SM_BK 32
#endif
#ifndef ELV_SM_STAGES
#define ELV_SM_STAGES 3
#endif
constexpr int SM_BM = 64, SM_BN = 64, SM_BK = ELV_SM_BK, SM_STAGES = ELV_SM_STAGES;
constexpr int SM_SMEM = SM_STAGES * SM_BK * (SM_BM + SM_BN) * 4;   // 48 KB at 32 x 3

// NT = 64: 8x8 outputs per thread; NT = 128 (tuning: ELV_K6_SMALL_NT=128):
// the 64x64 tile split into two column halves, 8x4 outputs per thread --
// twice the warps per SM for the same tiles; measured slower (the extra
// fragment loads cost more than the latency they hide).  Each output keeps
// the same fmaf chain either way.
template <int NT>
__global__ void __launch_bounds__(NT, 4)
k6_sgemm_small(const float* __restrict__ PA, const float* __restrict__ PB, float* __restrict__ C,
               int M, int N, int K, int ldc) {
  constexpr int NCP = NT == 64 ? 4 : 2;               // column pairs per thread (FFMA2 accumulators)
  extern __shared__ __align__(16) float smem_s[];
  float* As = smem_s;                                  // [STAGES][BK][64]
  float* Bs = smem_s + SM_STAGES * SM_BK * SM_BM;      // [STAGES][BK][64]
  const int tid = threadIdx.x;
  const int tl = tid & 63, half = tid >> 6;              // NT = 128: column half
  const int trow = (tl >> 3) * 4, tcol = (tl & 7) * 4 + 32 * half;   // rows + {0..3, 32..35}; cols + {0..3} (+32 at NT = 64)
  const bool vecC = aligned16(C) && (ldc & 3) == 0;
  const int tiles_m = (M + SM_BM - 1) / SM_BM, tiles_n = (N + SM_BN - 1) / SM_BN;
  const int num_tiles = tiles_m * tiles_n;
  const int nkb = (K + SM_BK - 1) / SM_BK;

  griddep_wait();                                   // packed operands from k_pack_ab
  for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
    const int tm = t % tiles_m, tn = t / tiles_m;      // column-major: neighbours share B panels
    const int row0 = tm * SM_BM, col0 = tn * SM_BN;
    const float* pa = PA + (size_t)(row0 >> 7) * K * 128 + (row0 & 127);
    const float* pb = PB + (size_t)(col0 >> 5) * K * kPanel;
    auto issue = [&](int kb, int slot) {
      const int k0 = kb * SM_BK;
#pragma unroll
      for (int i = 0; i < SM_BK * 16 / NT; ++i) {      // A: BK rows x 64 floats = 256 float4
        const int q = tid + i * NT;
        const int kk = q >> 4, c4 = (q & 15) * 4;
        const int gk = k0 + kk;
        cp_async16(&As[(slot * SM_BK + kk) * SM_BM + c4], pa + (size_t)min(gk, K - 1) * 128 + c4,
                   gk < K ? 16 : 0);
      }
#pragma unroll
      for (int i = 0; i < SM_BK * 16 / NT; ++i) {      // B: 2 panels x BK rows x 32 floats
        const int q = tid + i * NT;
        const int pnl = q / (SM_BK * 8), w = q % (SM_BK * 8);
        const int kk = w >> 3, c4 = (w & 7) * 4;
        const int gk = k0 + kk;
        cp_async16(&Bs[(slot * SM_BK + kk) * SM_BN + pnl * 32 + c4],
                   pb + ((size_t)pnl * K + min(gk, K - 1)) * kPanel + c4, gk < K ? 16 : 0);
      }
    };

    unsigned long long acc[8][NCP];                // [row][column pair], FFMA2 (see k6_sgemm_ffma2)
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < NCP; ++j) acc[i][j] = 0ull;

#pragma unroll
    for (int st = 0; st < SM_STAGES - 1; ++st) {
      if (st < nkb) issue(st, st);
      cp_async_commit();
    }
    for (int kb = 0; kb < nkb; ++kb) {
      cp_async_wait<SM_STAGES - 2>();
      __syncthreads();
      const int nk = kb + SM_STAGES - 1;
      if (nk < nkb) issue(nk, nk % SM_STAGES);
      cp_async_commit();
      const float* as = As + (kb % SM_STAGES) * SM_BK * SM_BM;
      const float* bs = Bs + (kb % SM_STAGES) * SM_BK * SM_BN;
      float a[2][8];
      unsigned long long b[2][NCP];
      auto lfrag = [&](int slot, int k) {
        const float4 a0 = *reinterpret_cast<const float4*>(as + k * SM_BM + trow);
        const float4 a1 = *reinterpret_cast<const float4*>(as + k * SM_BM + trow + 32);
        const float4 b0 = *reinterpret_cast<const float4*>(bs + k * SM_BN + tcol);
        a[slot][0] = a0.x; a[slot][1] = a0.y; a[slot][2] = a0.z; a[slot][3] = a0.w;
        a[slot][4] = a1.x; a[slot][5] = a1.y; a[slot][6] = a1.z; a[slot][7] = a1.w;
        b[slot][0] = pack2(b0.x, b0.y); b[slot][1] = pack2(b0.z, b0.w);
        if (NT == 64) {
          const float4 b1 = *reinterpret_cast<const float4*>(bs + k * SM_BN + tcol + 32);
          b[slot][NCP - 2] = pack2(b1.x, b1.y); b[slot][NCP - 1] = pack2(b1.z, b1.w);
        }
      };
      lfrag(0, 0);
#pragma unroll
      for (int k = 0; k < SM_BK; ++k) {
        if (k + 1 < SM_BK) lfrag((k + 1) & 1, k + 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const unsigned long long ai = pack2(a[k & 1][i], a[k & 1][i]);
#pragma unroll
          for (int j = 0; j < NCP; ++j) ffma2(acc[i][j], ai, b[k & 1][j]);
        }
      }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int gi = row0 + trow + (i & 3) + (i >> 2) * 32;
      if (gi >= M) continue;
#pragma unroll
      for (int h = 0; h < NCP / 2; ++h) {
        const int gj = col0 + tcol + h * 32;
        float* p = C + (size_t)gi * ldc + gj;
        const float2 lo = unpack2(acc[i][2 * h]), hi = unpack2(acc[i][2 * h + 1]);
        const float v[4] = {lo.x, lo.y, hi.x, hi.y};
        if (vecC && gj + 3 < N) *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
        else
#pragma unroll
          for (int j = 0; j < 4; ++j) if (gj + j < N) p[j] = v[j];
      }
    }
    __syncthreads();
  }
}

// packA: packedA[p][k][r] = A[128p + r][k], zero past M.  32x32 tiles through
// SMEM so both the row reads of A and the panel-row writes coalesce.
__device__ __forceinline__ void pack_a_block(const float* __restrict__ A, float* __restrict__ PA, int M, int K,
                                             int lda, int bx, int by) {
  __shared__ float tt[32][33];
  const int k0 = bx * 32, r0 = by * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = r0 + ty + 8 * i, k = k0 + tx;
    tt[ty + 8 * i][tx] = (r < M && k < K) ? __ldg(A + (size_t)r * lda + k) : 0.f;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int k = k0 + ty + 8 * i, r = r0 + tx;
    if (k < K) PA[((size_t)(r >> 7) * K + k) * 128 + (r & 127)] = tt[tx][ty + 8 * i];
  }
}
__global__ void __launch_bounds__(256)
k_pack_a(const float* __restrict__ A, float* __restrict__ PA, int M, int K, int lda) {
  pack_a_block(A, PA, M, K, lda, blockIdx.x, blockIdx.y);
}

struct SgemmCfg { void (*fn)(const float*, const float*, float*, int, int, int, int, int); int minb, bm, bn; };
static const SgemmCfg kSgemmCfgs[] = {
    {k6_sgemm_db<8, 2>, 2, 128, 128}, {k6_sgemm_db<8, 1>, 1, 128, 128}, {k6_sgemm_db<16, 2>, 2, 128, 128},
    {k6_sgemm_db<16, 1>, 1, 128, 128}, {k6_sgemm_8x16<8>, 1, 128, 256},
};

static int sgemm_cfg() {
  static int cfg = -2;
  if (cfg == -2) {
    const char* e = getenv("ELV_SGEMM_CFG");
    cfg = e ? atoi(e) : -2;   // -2: choose by problem size (below)
    if (cfg < -3 || cfg >= (int)(sizeof(kSgemmCfgs) / sizeof(kSgemmCfgs[0]))) cfg = -2;
  }
  return cfg;
}

// ---------------------------------------------------------------------------
// packB: packedB[p][k][c] = B[k][32p + c], zero-filled past N (rules.py:516-549,
// TVM packedB PAPER.md:49-50).  Pure layout transform, HBM-bound: every
// thread moves one float4; reads are coalesced along B's rows, writes along
// the panel rows.
__device__ __forceinline__ void pack_b_part(const float* __restrict__ B, float* __restrict__ P, int K, int N,
                                            int ldb, int panels, bool vecB, int bx, int gx) {
  const long long total4 = (long long)panels * K * (kPanel / 4);
  for (long long q = bx * (long long)blockDim.x + threadIdx.x; q < total4;
       q += (long long)gx * blockDim.x) {
    // q enumerates (k, p, c4) with c4 fastest so reads of a B row coalesce
    const int c4 = (int)(q & 7) * 4;
    const long long kp = q >> 3;
    const int p = (int)(kp % panels);
    const int k = (int)(kp / panels);
    const int j = p * kPanel + c4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    const float* src = B + (size_t)k * ldb + j;
    if (vecB && j + 3 < N) v = __ldg(reinterpret_cast<const float4*>(src));
    else {
      if (j + 0 < N) v.x = __ldg(src + 0);
      if (j + 1 < N) v.y = __ldg(src + 1);
      if (j + 2 < N) v.z = __ldg(src + 2);
      if (j + 3 < N) v.w = __ldg(src + 3);
    }
    *reinterpret_cast<float4*>(P + ((size_t)p * K + k) * kPanel + c4) = v;
  }
}
__global__ void __launch_bounds__(256)
k_pack_b(const float* __restrict__ B, float* __restrict__ P, int K, int N, int ldb,
         int panels, bool vecB) {
  pack_b_part(B, P, K, N, ldb, panels, vecB, blockIdx.x, gridDim.x);
}

// the parallel variant's prepare in one launch: blocks [0, gb) pack B
// (grid-stride), the rest pack A in 32x32 tiles (independent work)
__global__ void __launch_bounds__(256)
k_pack_ab(const float* __restrict__ B, float* __restrict__ P, int K, int N, int ldb, int panels, bool vecB,
          int gb, const float* __restrict__ A, float* __restrict__ PA, int M, int lda, int gxa) {
  griddep_launch_dependents();
  const int b = blockIdx.x;
  if (b < gb) pack_b_part(B, P, K, N, ldb, panels, vecB, b, gb);
  else pack_a_block(A, PA, M, K, lda, (b - gb) % gxa, (b - gb) / gxa);
}

}  // namespace

int launch_pack_b(const float* B, float* packedB, int K, int N, int ldb, cudaStream_t st) {
  const int panels = (int)(packed_cols(N) / kPanel);
  const bool vecB = ((reinterpret_cast<uintptr_t>(B) & 15u) == 0) && (ldb & 3) == 0;
  const long long total4 = (long long)panels * K * (kPanel / 4);
  long long blocks = (total4 + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  ELV_PREFER_MAX_SMEM(k_pack_b);
  k_pack_b<<<(unsigned)blocks, 256, 0, st>>>(B, packedB, K, N, ldb, panels, vecB);
  return check_launch("pack_b");
}

// the packed-A cp.async kernel serves the large-problem regime of the
// parallel schedule (the same regime as the 8x16 kernel); ELV_SGEMM_CP=0
// falls back to the raw-A kernels for tuning comparisons.
// tuning hook: ELV_K6_PATH=1 small 64x64 kernel, 2 cp.async 128x256 kernel
// (packed A), 3 the unpacked 128x128 kernel; unset = by problem size
static int k6_path_forced() {
  static int v = -2;
  if (v == -2) {
    const char* e = getenv("ELV_K6_PATH");
    v = e ? atoi(e) : 0;
  }
  return v;
}
// The 128x256 cp.async kernel runs whole waves of one tile per SM; where its
// last wave would be <95 % full, the 64x64-tile kernel (4 resident per SM,
// 16x finer tiles) wins.  Measured (profiles/r1/small/k6_paths.jsonl, TF):
// 2048^3 48.7 vs 39.7 (old 128x128 mid kernel), 4096^3 57.2 vs 51.2,
// 5120^3 57.1 vs 53.6; cp ahead at 3072^3 (57.1 vs 55.6), 6144^3 (58.1 vs
// 56.7), 8192^3 (59.2 vs 57.8), 4096x8192x2048 (58.6 vs 57.2).
static bool parallel_small(int M, int N) {
  const int f = k6_path_forced();
  if (f != 0) return f == 1;
  const long long tiles = (long long)((M + 127) / 128) * ((N + 255) / 256);
  const long long sms = num_sms();
  const long long waves = (tiles + sms - 1) / sms;
  return tiles < 0.95 * (double)(waves * sms);
}

bool parallel_uses_packed_a(int M, int N) {
  static int enabled = -1;
  if (enabled < 0) {
    const char* e = getenv("ELV_SGEMM_CP");
    enabled = e ? (atoi(e) != 0) : 1;
  }
  if (!enabled) return false;
  const int f = k6_path_forced();
  if (f != 0) return f == 1 || f == 2;
  (void)M;
  (void)N;
  return true;            // both the small and the cp.async kernel read packed A
}

size_t pack_a_bytes(int M, int K) { return (size_t)((M + 127) / 128) * 128 * (size_t)K * sizeof(float); }

int launch_pack_ab(const float* B, float* packedB, int K, int N, int ldb, const float* A, float* packedA, int M,
                   int lda, cudaStream_t st) {
  const int panels = (int)(packed_cols(N) / kPanel);
  const bool vecB = ((reinterpret_cast<uintptr_t>(B) & 15u) == 0) && (ldb & 3) == 0;
  const long long total4 = (long long)panels * K * (kPanel / 4);
  long long gb = (total4 + 255) / 256;
  const long long cap = (long long)num_sms() * 16;
  if (gb > cap) gb = cap;
  if (gb < 1) gb = 1;
  const int gxa = (K + 31) / 32, gya = (M + 127) / 128 * 4;
  const long long blocks = gb + (long long)gxa * gya;
  if (blocks > 0x7fffffffLL) return set_error(ELV_EINVAL, "pack_ab: problem too large for one launch");
  ELV_PREFER_MAX_SMEM(k_pack_ab);
  k_pack_ab<<<(unsigned)blocks, 256, 0, st>>>(B, packedB, K, N, ldb, panels, vecB, (int)gb, A, packedA, M, lda, gxa);
  return check_launch("pack_ab");
}

int launch_pack_a(const float* A, float* packedA, int M, int K, int lda, cudaStream_t st) {
  dim3 grid((K + 31) / 32, (M + 127) / 128 * 4);
  k_pack_a<<<grid, 256, 0, st>>>(A, packedA, M, K, lda);
  return check_launch("pack_a");
}

int launch_parallel_packed(const float* packedA, const float* packedB, float* C, int M, int N, int K, int ldc,
                           cudaStream_t st) {
  if (parallel_small(M, N)) {
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      cudaError_t e = cudaFuncSetAttribute(k6_sgemm_small<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_SMEM);
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k6_sgemm_small<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, SM_SMEM);
      if (e != cudaSuccess) return set_error(ELV_ECUDA, "sgemm_small smem attribute: %s", cudaGetErrorString(e));
      attr_dev = dev;
    }
    const long long tiles = (long long)((M + SM_BM - 1) / SM_BM) * ((N + SM_BN - 1) / SM_BN);
    long long grid = (long long)num_sms() * 4;
    if (grid > tiles) grid = tiles;
    // no PDL here: with back-to-back calls at 1024^3 the early-resident
    // GEMM CTAs cost 92 vs 55 us per call (scripts/small_timing.py, ELV_PDL)
    static int pdl = -1;
    if (pdl < 0) pdl = getenv("ELV_K6_SMALL_PDL") ? atoi(getenv("ELV_K6_SMALL_PDL")) != 0 : 0;
    // 64 threads per 64x64 tile (8x8 each); ELV_K6_SMALL_NT=128 (8x4 each, two
    // warps per SMSP) measured slower: 1024^3 62.4 vs 60.4 us, 2048^3 378 vs 361 us
    static int nt = -1;
    if (nt < 0) nt = getenv("ELV_K6_SMALL_NT") && atoi(getenv("ELV_K6_SMALL_NT")) == 128 ? 128 : 64;
    cudaError_t e = launch_pdl_if(pdl != 0, nt == 64 ? k6_sgemm_small<64> : k6_sgemm_small<128>, dim3((unsigned)grid),
                                  dim3(nt), (size_t)SM_SMEM, st,
                                  packedA, packedB, C, M, N, K, ldc);
    if (e != cudaSuccess) return set_error(ELV_ECUDA, "gemm_parallel_small: %s", cudaGetErrorString(e));
    return check_launch("gemm_parallel_small");
  }
  static int order = -1;
  if (order < 0) {
    const char* e = getenv("ELV_SGEMM_ORDER");
    order = e ? atoi(e) : 3;   // measured at 32768x32768x8192: FFMA2 60.5 TF; scalar 2x2 FFMA blocks 52.6
    if (order < 0 || order > 3) order = 2;
  }
  static int bulk = -1;                     // ELV_K6_BULK=1: TMA bulk-copy staging (K % 32 == 0)
  if (bulk < 0) bulk = getenv("ELV_K6_BULK") ? atoi(getenv("ELV_K6_BULK")) != 0 : 0;
  if (bulk && order == 3 && K % CP_BK == 0) {
    static int battr = -1;
    int bdev = 0;
    cudaGetDevice(&bdev);
    if (battr != bdev) {
      cudaError_t e = cudaFuncSetAttribute(k6_sgemm_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, CP_SMEM);
      if (e != cudaSuccess) return set_error(ELV_ECUDA, "sgemm_bulk smem attribute: %s", cudaGetErrorString(e));
      battr = bdev;
    }
    const long long tiles = (long long)((M + 127) / 128) * ((N + 255) / 256);
    long long grid = num_sms();
    if (grid > tiles) grid = tiles;
    cudaError_t e = launch_pdl(k6_sgemm_bulk, dim3((unsigned)grid), dim3(256), (size_t)CP_SMEM, st, packedA, packedB,
                               C, M, N, K, ldc);
    if (e != cudaSuccess) return set_error(ELV_ECUDA, "gemm_parallel_bulk: %s", cudaGetErrorString(e));
    return check_launch("gemm_parallel_bulk");
  }
  auto fn = order == 0 ? k6_sgemm_cp<0> : order == 1 ? k6_sgemm_cp<1> : order == 2 ? k6_sgemm_cp<2>
                                                                                      : k6_sgemm_ffma2;
  static int attr_dev[4] = {-1, -1, -1, -1};
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev[order] != dev) {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, CP_SMEM);
    if (e != cudaSuccess) return set_error(ELV_ECUDA, "sgemm_cp smem attribute: %s", cudaGetErrorString(e));
    attr_dev[order] = dev;
  }
  const long long tiles = (long long)((M + 127) / 128) * ((N + 255) / 256);
  long long grid = num_sms();
  if (grid > tiles) grid = tiles;
  cudaError_t e = launch_pdl(fn, dim3((unsigned)grid), dim3(256), (size_t)CP_SMEM, st, packedA, packedB, C, M, N, K,
                             ldc);
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "gemm_parallel: %s", cudaGetErrorString(e));
  return check_launch("gemm_parallel");
}

int launch_simt(int variant, const float* A, const float* B, const float* packedB,
                float* C, int M, int N, int K, int lda, int ldb, int ldc, cudaStream_t st) {
  switch (variant) {
    case ELV_BASELINE: {
      dim3 grid((N + 31) / 32, (M + 7) / 8);
      k0_baseline<<<grid, dim3(32, 8), 0, st>>>(A, B, C, M, N, K, lda, ldb, ldc);
      return check_launch("gemm_baseline");
    }
    case ELV_BLOCKING: {
      dim3 grid((N + 31) / 32, (M + 31) / 32);
      k1_blocking<<<grid, dim3(32, 8), 0, st>>>(A, B, C, M, N, K, lda, ldb, ldc);
      return check_launch("gemm_blocking");
    }
    case ELV_VECTORIZED: {
      dim3 grid((N + 31) / 32, (M + 31) / 32);
      k2_vectorized<<<grid, 256, 0, st>>>(A, B, C, M, N, K, lda, ldb, ldc);
      return check_launch("gemm_vectorized");
    }
    case ELV_LOOPPERM: {
      dim3 grid((N + 63) / 64, (M + 63) / 64);
      k34_outer4x4<false><<<grid, 256, 0, st>>>(A, B, C, M, N, K, lda, ldb, ldc);
      return check_launch("gemm_loopperm");
    }
    case ELV_ARRAYPACKING: {
      dim3 grid((N + 63) / 64, (M + 63) / 64);
      k34_outer4x4<true><<<grid, 256, 0, st>>>(A, packedB, C, M, N, K, lda, 0, ldc);
      return check_launch("gemm_arraypacking");
    }
    case ELV_CACHEBLOCKS: {
      // fewer 128x128 tiles than SMs (e.g. 1024^3: 64): 64-row tiles, 128 threads
      if ((long long)((M + G_BM - 1) / G_BM) * ((N + G_BN - 1) / G_BN) < num_sms()) {
        dim3 grid((N + G_BN - 1) / G_BN, (M + 63) / 64);
        k56_packed_8x8<false, 64><<<grid, 128, 0, st>>>(A, packedB, C, M, N, K, lda, ldc);
        return check_launch("gemm_cacheblocks");
      }
      dim3 grid((N + G_BN - 1) / G_BN, (M + G_BM - 1) / G_BM);
      k56_packed_8x8<false><<<grid, 256, 0, st>>>(A, packedB, C, M, N, K, lda, ldc);
      return check_launch("gemm_cacheblocks");
    }
    case ELV_PARALLEL: {
      // mapPar -> a grid covering all SMs.  Large problems: the 8x16-per-thread
      // 128x256 persistent kernel (measured best, 51.9 TF at 32768x32768x8192);
      // mid-size: 128x128 tiles at 2 CTAs/SM; small (fewer 128x128 tiles than
      // SMs, e.g. 1024^3): 64x64 tiles so every SM gets work.
      auto tiles_of = [&](int bm, int bn) {
        return (long long)((M + bm - 1) / bm) * ((N + bn - 1) / bn);
      };
      int cfg = sgemm_cfg();
      if (cfg == -2) {
        if (tiles_of(128, 256) >= 2LL * num_sms()) cfg = 4;
        else if (tiles_of(128, 128) >= num_sms()) cfg = 0;
        else cfg = -3;
      }
      if (cfg == -3) {
        dim3 grid((N + 63) / 64, (M + 63) / 64);
        k34_outer4x4<true><<<grid, 256, 0, st>>>(A, packedB, C, M, N, K, lda, 0, ldc);
        return check_launch("gemm_parallel");
      }
      if (cfg >= 0) {
        const long long tiles = tiles_of(kSgemmCfgs[cfg].bm, kSgemmCfgs[cfg].bn);
        long long grid = (long long)num_sms() * kSgemmCfgs[cfg].minb;
        if (grid > tiles) grid = tiles;
        kSgemmCfgs[cfg].fn<<<(unsigned)grid, 256, 0, st>>>(A, packedB, C, M, N, K, lda, ldc);
        return check_launch("gemm_parallel");
      }
      const long long tiles = (long long)((M + G_BM - 1) / G_BM) * ((N + G_BN - 1) / G_BN);
      long long grid = (long long)num_sms() * 2;
      if (grid > tiles) grid = tiles;
      k56_packed_8x8<true><<<(unsigned)grid, 256, 0, st>>>(A, packedB, C, M, N, K, lda, ldc);
      return check_launch("gemm_parallel");
    }
    default:
      return set_error(ELV_EVARIANT, "launch_simt: variant %d is not a SIMT variant", variant);
  }
}

}  // namespace elv
