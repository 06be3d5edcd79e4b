// K7: the parallel schedule's dense contraction on the 5th-generation tensor
// cores, in fp32-accurate 3xTF32 form (and K8, the same kernels on scaled
// fp16 planes, below).
//
//   x = hi + lo,  hi = rna_tf32(x), lo = rna_tf32(x - hi)
//   C = A_hi.B_hi + A_hi.B_lo + A_lo.B_hi       (A_lo.B_lo ~ 2^-22, added for K < 512)
//
// Pipeline (one persistent CTA -- or CTA pair -- per SM, 10 warps):
//   warp 0      TMA producer: A_hi/A_lo (BM x BK) and Bt_hi/Bt_lo (BN x BK)
//               tiles into a STAGES-deep SMEM ring, mbarrier complete_tx.
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer.
//   warps 2..9  epilogue: two warps per TMEM lane group (one per column half).
// Accumulation in chunks: the tensor core rounds every accumulate toward
// zero, and on one long chain that bias grows like K (measured on B200,
// scripts/tc_numerics_r2.py: 10.9x the tau=1 bound at K=8192 on non-negative
// inputs, profiles/r2/tc_numerics_before_chunked.jsonl).  So every k-block
// is one chunk accumulated into a FRESH TMEM buffer (two buffers, ping-pong):
// the correction products first (they build up at their own, 2^-11 smaller
// scale), then hi.hi -- only KSUB truncations per chunk land on the chunk's
// magnitude -- and the epilogue warps add the chunks into fp32 registers
// with round-to-nearest (a blocked summation, like the SIMT kernels' RN fold
// but over K/BK partial sums).  Draining 128 KB of TMEM per chunk and CTA
// costs ~300 of the chunk's ~1500 MMA cycles at the measured ~420 B/clk
// (profiles/r2/tmem_ld_bw.jsonl), overlapped with the next chunk's MMAs.
// The split prepass (split_a / split_transpose_b below) is the packB of this
// variant: it writes the hi/lo planes K-major, zero-padded to BK, so TMA
// boxes and UMMA K-major descriptors apply to both operands.

#include "elv_common.cuh"

#include <cuda.h>
#include <cuda_fp16.h>
#include <map>
#include <mutex>
#include <utility>
#include <stdlib.h>

namespace elv {
namespace {

constexpr int BM = 128, BK = 16;                  // BK fp32 = 64 B rows (SWIZZLE_64B)
constexpr int NUM_THREADS = 320;                  // 1-CTA kernel: producer, MMA, 8 epilogue warps
constexpr int EPI_WARPS = 8;
constexpr int TMEM_COLS = 512;                    // pair kernel: two 256-column chunk buffers

// The 1-CTA kernel is templated on its N tile (256, 128 or 64): narrow tiles
// give small problems (e.g. 1024^3: 32 tiles of 128x256 for 148 SMs) more
// CTAs.  Per-element arithmetic does not depend on the tile shape.
template <int TBN, int TBK = BK, bool F16 = false> struct OneCfg {
  static constexpr int EB = F16 ? 2 : 4;               // bytes per operand element
  static constexpr int ROW_BYTES = TBK * EB;            // 64 or 128 (swizzle width)
  static constexpr int A_TILE = BM * ROW_BYTES;
  static constexpr int B_TILE = TBN * ROW_BYTES;
  static constexpr int STAGE = 2 * A_TILE + 2 * B_TILE;
  static constexpr int NST = (192 * 1024) / STAGE > 8 ? 8 : (192 * 1024) / STAGE;
  // chunk buffers: all 512 TMEM columns (one CTA per SM), so narrow tiles
  // keep the MMA up to NBUF - 1 chunks ahead of the epilogue's drain (a
  // 64-column chunk is only ~400 MMA cycles, shorter than one drain's latency)
  static constexpr int NBUF = 512 / TBN > 8 ? 8 : 512 / TBN;
  static constexpr int TMEM = 512;
  static constexpr int SMEM = NST * STAGE + 512 + 1024;
  static constexpr int KSUB = TBK / (F16 ? 16 : 8);     // MMAs per product per stage
  static constexpr uint32_t IDESC = (1u << 4) | ((F16 ? 0u : 2u) << 7) | ((F16 ? 0u : 2u) << 10) |
                                    ((uint32_t)(TBN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
};
inline long long round_up(long long v, long long m) { return (v + m - 1) / m * m; }

// ----------------------------------------------------------------------------
// PTX wrappers (sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
template <bool F16>
__device__ __forceinline__ void tc_mma_one(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
  if (F16) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
__device__ __forceinline__ void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor: K-major, 64B swizzle, 8-row atoms of 512 B.
__device__ __forceinline__ uint64_t umma_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);        // start address
  d |= (uint64_t)1 << 16;                         // LBO (ignored for swizzled K-major)
  d |= (uint64_t)(512 >> 4) << 32;                // SBO: 8 rows x 64 B
  d |= (uint64_t)1 << 46;                         // descriptor version (sm_100)
  d |= (uint64_t)4 << 61;                         // SWIZZLE_64B
  return d;
}

// K-major descriptor for 128B swizzle: 8-row atoms of 1024 B.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;                         // SWIZZLE_128B
  return d;
}
template <int BKT>
__device__ __forceinline__ uint64_t umma_desc_k(uint32_t saddr) {
  return BKT == 32 ? umma_desc_sw128(saddr) : umma_desc_sw64(saddr);
}

// instruction descriptor: D=f32, A=B=tf32, both K-major, N=256, M=128

// Wave synchronisation of the persistent CTAs' producers: before loading its
// (w+1)-th tile a producer waits until every CTA has issued the loads of its
// w-th tile.  Tiles that run concurrently share A rows / B columns through L2
// only while their k positions stay close; unsynchronised, per-tile timing
// noise lets the CTAs drift apart over hundreds of tiles and the operands
// are re-read from HBM (measured: 222-260 GB of DRAM reads per 32768^2 x 8192
// launch against ~64-83 GB for lock-step waves).  The wait is bounded
// (~20 us) so a CTA that is not resident (e.g. SMs busy with an NCCL kernel)
// never stalls the others for long.
__device__ __forceinline__ void wave_sync_wait(unsigned int* ctr, unsigned int target) {
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  while (true) {
    unsigned int v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    if (v >= target) break;
    uint64_t t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (t1 - t0 > 20000) break;
    __nanosleep(64);
  }
}

struct TileSched {
  int tiles_m, tiles_n, group, bn;
  __device__ void coords(int t, int& m0, int& n0) const {
    const int GROUP = group;                        // row-tiles per L2 group
    const int per_group = GROUP * tiles_n;
    const int g = t / per_group;
    const int first_m = g * GROUP;
    const int gm = min(tiles_m - first_m, GROUP);
    const int in = t - g * per_group;
    m0 = (first_m + in % gm) * BM;
    n0 = (in / gm) * bn;
  }
};

// Scaled MMA: D = A.B + D * 2^-11 (scale-input-d; kind::f16 / kind::tf32,
// sm_100a).  Used once per chunk to bring the fp16 encoding's correction
// partial (lo planes carry 2^11) to the scale of hi.hi.
template <bool F16>
__device__ __forceinline__ void tc_mma_one_sc11(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                uint32_t idesc) {
  if (F16)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p, 11;\n}\n" ::"r"(d_tmem), "l"(a_desc),
                 "l"(b_desc), "r"(idesc), "r"(1u)
                 : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p, 11;\n}\n" ::"r"(d_tmem), "l"(a_desc),
                 "l"(b_desc), "r"(idesc), "r"(1u)
                 : "memory");
}

// Exact power-of-two unscaling of the fp16 encoding: v * 2^(e_row + e_col)
// as two factors of the same sign of exponent, so an intermediate overflows
// or underflows only when the result does (e_row, e_col in [-115, 113]).
__device__ __forceinline__ int pow2_exp(float p) { return (int)((__float_as_uint(p) >> 23) & 0xffu) - 127; }
__device__ __forceinline__ float unscale2(float v, int e) {
  const int e1 = e >> 1, e2 = e - e1;
  return v * __int_as_float((e1 + 127) << 23) * __int_as_float((e2 + 127) << 23);
}

// Unscale one 32-column chunk of a row (fp16 encoding): lane j holds the
// column scale 1/t of column j (one coalesced load per warp), broadcast by
// shuffles -- no per-element loads, few live registers.
__device__ __forceinline__ void unscale_chunk(float* v, int er, float inv_t_lane) {
  const int ec_lane = pow2_exp(inv_t_lane);
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = unscale2(v[j], er + __shfl_sync(0xffffffffu, ec_lane, j));
}

// Epilogue drain of one chunk: this warp's NC x 32 accumulator columns added
// (RN) into the register-resident running sums.
template <int NC>
__device__ __forceinline__ void drain_add(uint32_t taddr, float (&acc)[NC * 32]) {
#pragma unroll
  for (int c = 0; c < NC; ++c) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(taddr + (uint32_t)(c * 32), r);
#pragma unroll
    for (int q = 0; q < 32; ++q) acc[c * 32 + q] += __uint_as_float(r[q]);
  }
}

// Accumulation chunk length in k: 32 (tf32) / 64 (fp16) -- one stage of the
// default pair kernels; kernels with shallower stages take CH = CHUNK_K / BK
// stages per chunk.  The per-element operation sequence then depends only on
// the chunk's k range, never on the stage depth or the tile shape, so every
// kernel configuration of an encoding produces the same bits.
template <bool F16> struct ChunkK { static constexpr int value = F16 ? 64 : 32; };

template <bool PAIR, bool F16>
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc);
template <bool F16>
__device__ __forceinline__ void tc_mma_pair_sc11(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc);

// The MMAs of one chunk (CH stages of KSUB k-steps) into a fresh accumulator
// d: the correction products first (hi.lo for every k-step, then lo.hi, then
// lo.lo when requested) -- they build up at their own, 2^-11 smaller scale --
// then hi.hi, whose first MMA rescales the fp16 corrections by 2^-11
// (scale-input-d), so only CH * KSUB truncations fall on the chunk's magnitude.
template <bool PAIR, bool F16, int KSUB, int CH>
__device__ __forceinline__ void mma_chunk(uint32_t d, const uint64_t (&ahi)[CH], const uint64_t (&alo)[CH],
                                          const uint64_t (&bhi)[CH], const uint64_t (&blo)[CH], uint32_t idesc,
                                          int lolo) {
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int k = 0; k < KSUB; ++k) tc_mma<PAIR, F16>(d, ahi[j] + 2 * k, blo[j] + 2 * k, idesc, (j | k) != 0);
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int k = 0; k < KSUB; ++k) tc_mma<PAIR, F16>(d, alo[j] + 2 * k, bhi[j] + 2 * k, idesc, 1u);
  if (!F16 && lolo) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
#pragma unroll
      for (int k = 0; k < KSUB; ++k) tc_mma<PAIR, F16>(d, alo[j] + 2 * k, blo[j] + 2 * k, idesc, 1u);
  }
#pragma unroll
  for (int j = 0; j < CH; ++j)
#pragma unroll
    for (int k = 0; k < KSUB; ++k) {
      if (F16 && j == 0 && k == 0) {
        if (PAIR) tc_mma_pair_sc11<F16>(d, ahi[0], bhi[0], idesc);
        else tc_mma_one_sc11<F16>(d, ahi[0], bhi[0], idesc);
      } else {
        tc_mma<PAIR, F16>(d, ahi[j] + 2 * k, bhi[j] + 2 * k, idesc, 1u);
      }
    }
}

#ifdef ELV_K7_PROF
// cycle accounting for tuning builds only (scripts/k7_prof.sh):
// [0] MMA: waiting tempty  [1] MMA: waiting full  [2] MMA: total
// [3] producer: waiting empty  [4] producer: wave sync  [5] epilogue: waiting tfull
// [6] epilogue: drain  [7] tiles
// [5] epilogue: waiting tfull  [6] epilogue: store per tile  [8] epilogue: TMEM drain (ld + add)
// [9] epilogue: chunks  [10] epilogue: arrive  [11] (1-CTA kernel) entry -> after griddepcontrol.wait
constexpr int K7_PROF_SLOTS = 12;
__device__ unsigned long long g_k7_prof[512][K7_PROF_SLOTS];
#define PROF_T(x) const long long x = clock64()
#define PROF_ADD(i, v) prof[i] += (unsigned long long)(v)
#else
#define PROF_T(x)
#define PROF_ADD(i, v)
#endif

template <int TBN, int TBK, bool F16>
__global__ void __launch_bounds__(NUM_THREADS, 1)
k7_tf32x3(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
          const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
          float* __restrict__ C, int M, int N, int ldc, int num_kb, int with_lolo, int group,
          unsigned int* __restrict__ wave_ctr, const float* __restrict__ inv_s,
          const float* __restrict__ inv_t, const FixArgs fix, int K) {
  using Cfg = OneCfg<TBN, TBK, F16>;
  constexpr int STAGES = Cfg::NST;
  constexpr int STAGE_BYTES = Cfg::STAGE;
  constexpr int B_TILE_BYTES = Cfg::B_TILE;
  constexpr int A_TILE_BYTES = Cfg::A_TILE;
  constexpr int BN = TBN;
  constexpr int NC = TBN / 64;                       // 32-column groups per epilogue warp
  constexpr int CH = ChunkK<F16>::value / TBK;           // stages per accumulation chunk
  static_assert(CH >= 1 && CH * TBK == ChunkK<F16>::value, "chunk length");
  constexpr uint32_t kIdesc = Cfg::IDESC;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  constexpr int NBUF = Cfg::NBUF;
  uint64_t* tfull = empty + STAGES;                  // [NBUF]: chunk in TMEM buffer b complete
  uint64_t* tempty = tfull + NBUF;                   // [NBUF]: buffer b drained by the epilogue
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + NBUF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef ELV_K7_PROF
  unsigned long long prof[K7_PROF_SLOTS] = {};
#endif
  PROF_T(k_entry);
  const TileSched sched{(M + BM - 1) / BM, (N + BN - 1) / BN, group, BN};
  const int num_tiles = sched.tiles_m * sched.tiles_n;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_ahi); tma_prefetch_desc(&map_alo);
    tma_prefetch_desc(&map_bhi); tma_prefetch_desc(&map_blo);
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < NBUF; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)), "r"(Cfg::TMEM));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  griddep_wait();                                   // operand planes from the preceding split kernel
  griddep_launch_dependents();                      // the range-guard fix-up may be scheduled (it waits for us)
  PROF_T(k_ready);
  PROF_ADD(11, k_ready - k_entry);

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer ----------------
      int s = 0; uint32_t ph = 0;
      int wave = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++wave) {
        int m0, n0;
        sched.coords(t, m0, n0);
        if (wave_ctr != nullptr && wave > 0) wave_sync_wait(wave_ctr, (unsigned)(wave * gridDim.x));
        for (int kb = 0; kb < num_kb; ++kb) {
          PROF_T(e0);
          mbar_wait(&empty[s], ph ^ 1);
          PROF_T(e1);
          PROF_ADD(3, e1 - e0);
          uint8_t* st = smem + s * STAGE_BYTES;
          mbar_expect_tx(&full[s], STAGE_BYTES);
          const int k0 = kb * TBK;
          tma_load_2d(&map_ahi, &full[s], st, k0, m0);
          tma_load_2d(&map_alo, &full[s], st + A_TILE_BYTES, k0, m0);
          tma_load_2d(&map_bhi, &full[s], st + 2 * A_TILE_BYTES, k0, n0);
          tma_load_2d(&map_blo, &full[s], st + 2 * A_TILE_BYTES + B_TILE_BYTES, k0, n0);
          if (++s == STAGES) { s = 0; ph ^= 1; }
        }
        if (wave_ctr != nullptr) atomicAdd(wave_ctr, 1u);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer: one accumulation chunk per CH stages ----------------
      int s = 0; uint32_t ph = 0;
      uint32_t q = 0;                                  // chunk counter (TMEM buffer q % NBUF)
      PROF_T(m_start);
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        PROF_ADD(7, 1);
        for (int kb = 0; kb < num_kb; kb += CH, ++q) {
          const uint32_t b = q % NBUF;
          PROF_T(q0);
          mbar_wait(&tempty[b], ((q / NBUF) & 1) ^ 1);
          PROF_T(f0);
          PROF_ADD(0, f0 - q0);
          uint64_t ahi[CH], alo[CH], bhi[CH], blo[CH];
          int ss[CH];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            mbar_wait(&full[s], ph);
            const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
            ahi[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st);
            alo[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st + A_TILE_BYTES);
            bhi[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st + 2 * A_TILE_BYTES);
            blo[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st + 2 * A_TILE_BYTES + B_TILE_BYTES);
            ss[j] = s;
            if (++s == STAGES) { s = 0; ph ^= 1; }
          }
          PROF_T(f1);
          PROF_ADD(1, f1 - f0);
          tc_fence_after();
          mma_chunk<false, F16, Cfg::KSUB, CH>(tmem_base + b * (uint32_t)BN, ahi, alo, bhi, blo, kIdesc, with_lolo);
#pragma unroll
          for (int j = 0; j < CH; ++j) tc_commit(&empty[ss[j]]);   // frees the slots when these MMAs finish
          tc_commit(&tfull[b]);                                    // chunk complete in buffer b
        }
      }
      PROF_T(m_end);
      PROF_ADD(2, m_end - m_start);
    }
  } else {
    // ---------------- epilogue (warps 2..9): C = RN-sum of the chunks ----------------
    const int g = warp & 3;                      // TMEM lane group this warp may access
    const int h = (warp - 2) >> 2;               // column half
    const bool vecC = ((reinterpret_cast<uintptr_t>(C) & 15u) == 0) && (ldc & 3) == 0;
    uint32_t q = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int m0, n0;
      sched.coords(t, m0, n0);
      const int row = m0 + g * 32 + lane;
      const uint32_t lane_base = tmem_base + ((uint32_t)(g * 32) << 16) + (uint32_t)(h * (BN / 2));
      // the tile's unscaling exponents / factors and range-guard flags are
      // final (griddep_wait above): load them before the chunk loop, so their
      // latency hides behind the MMAs instead of the tile's tail (1024^3 fp16:
      // the store phase was ~2.8K cycles against ~0.6K for tf32)
      const int er = (F16 && row < M) ? pow2_exp(__ldg(inv_s + row)) : 0;
      const bool frow = fix.A != nullptr && row < M && __ldg(fix.flag_a + row) != 0u;
      float it[NC];
      unsigned int fb[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int col = n0 + h * (BN / 2) + c * 32;
        it[c] = (F16 && col < N - lane) ? __ldg(inv_t + col + lane) : 1.f;
        fb[c] = (fix.A != nullptr && col + lane < N) ? __ldg(fix.flag_b + col + lane) : 0u;
      }
      float acc[NC * 32];
#pragma unroll
      for (int i = 0; i < NC * 32; ++i) acc[i] = 0.f;
#pragma unroll 1
      for (int kb = 0; kb < num_kb; kb += CH, ++q) {
        const uint32_t b = q % NBUF;
        PROF_T(c0);
        mbar_wait(&tfull[b], (q / NBUF) & 1);
        tc_fence_after();
        PROF_T(c1);
        PROF_ADD(5, c1 - c0);
        PROF_ADD(9, 1);
        drain_add<NC>(lane_base + b * (uint32_t)BN, acc);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
      PROF_T(d1);
      float* crow = C + (size_t)row * ldc;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int col = n0 + h * (BN / 2) + c * 32;
        float* v = acc + c * 32;
        if (F16) unscale_chunk(v, er, it[c]);
        if (row < M && col < N) {
          if (vecC && col + 31 < N) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(crow + col + 4 * j) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < N) crow[col + j] = v[j];
          }
        }
      }
      if (fix.A != nullptr) {
        // range-guard fix-up of this thread's outputs (its row x its columns):
        // flagged rows / columns are recomputed with the SIMT arithmetic of
        // k_tc_fixup -- an fmaf chain over k ascending from 0 -- after the
        // thread's own stores above (program order; flags are complete: the
        // split finished before griddepcontrol.wait returned)
        unsigned int fcols[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) fcols[c] = __ballot_sync(0xffffffffu, fb[c] != 0u);
#pragma unroll 1
        for (int c = 0; c < NC; ++c) {
          const int col0 = n0 + h * (BN / 2) + c * 32;
          unsigned int fcol = fcols[0];
#pragma unroll
          for (int i = 1; i < NC; ++i) fcol = c == i ? fcols[i] : fcol;   // register select (no local array)
          if (row >= M || (!frow && fcol == 0u)) continue;
          for (int j = 0; j < 32 && col0 + j < N; ++j) {
            if (!frow && !((fcol >> j) & 1u)) continue;
            const float* a = fix.A + (size_t)row * fix.lda;
            const float* b = fix.B + col0 + j;
            float acc = 0.f;
            for (int k = 0; k < K; ++k) acc = fmaf(__ldg(a + k), __ldg(b + (size_t)k * fix.ldb), acc);
            crow[col0 + j] = acc;
          }
        }
      }
      PROF_T(d2);
      PROF_ADD(6, d2 - d1);
    }
  }
#ifdef ELV_K7_PROF
  if (lane == 0 && warp <= 2 && blockIdx.x < 512)
    for (int i = 0; i < K7_PROF_SLOTS; ++i) if (prof[i]) atomicAdd(&g_k7_prof[blockIdx.x][i], prof[i]);
#endif

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM));
  }
}

// ----------------------------------------------------------------------------
// K7 on a CTA pair (cta_group::2): the same 3xTF32 math on 256x256 tiles.
// Each CTA of a 2-CTA cluster stages its own 128 rows of A and its own 128
// columns of B (as Bt rows); the leader CTA issues tcgen05.mma.cta_group::2
// (M=256, N=256), which reads A halves from both CTAs' SMEM and B halves
// from both, and writes each CTA's 128 accumulator rows into its own TMEM.
// Per SM this halves the B operand's SMEM reads and L2->SMEM fills relative
// to the 1-CTA kernel (the 1-CTA kernel measured L1/SMEM throughput 88 %,
// its limiter), for the same MMA work.

constexpr int P_BM = 128;                          // rows per CTA (pair: 256)
// warps: 0 TMA producer, 1 MMA issuer, 2..9 epilogue (two per TMEM lane
// group, one per 128-column half, so the accumulators drain twice as fast)
constexpr int P_NUM_THREADS = 320;
constexpr int P_EPI_WARPS = 8;
constexpr int P_BN = 256;                          // columns per pair tile (128 per CTA staged)
// BKT = K elements per stage; F16: operands are scaled fp16 hi/lo planes
// (2 B per element, kind::f16, 16 K per MMA) instead of tf32 (4 B, 8 K).
// PBN: columns per pair tile -- 256 for large problems; 128 / 64 for small
// ones, where wide tiles would leave SMs idle (the narrow pair still reads
// half of B per SM and issues M = 256 MMAs, unlike the 1-CTA kernel).
template <int BKT, bool F16 = false, int PBN = P_BN> struct PairCfg {
  static constexpr int EB = F16 ? 2 : 4;                   // bytes per element
  static constexpr int ROW_BYTES = BKT * EB;                // 64 or 128 (swizzle width)
  static constexpr int A_TILE = P_BM * ROW_BYTES;           // 8 / 16 KB
  static constexpr int B_TILE = (PBN / 2) * ROW_BYTES;      // this CTA's half of Bt
  static constexpr int STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;
  static constexpr int STAGES = PBN == 256 ? (ROW_BYTES == 128 ? 3 : 6)
                                           : ((192 * 1024) / STAGE_BYTES > 8 ? 8 : (192 * 1024) / STAGE_BYTES);
  static constexpr int NBUF = 512 / PBN;                     // TMEM chunk buffers
  // epilogue staging for TMA stores of C: one 32 x 32 fp32 tile (4 KB) per epilogue warp
  static constexpr int EPI_BYTES = 8 * 32 * 32 * 4;
  static constexpr int BAR_BYTES = PBN == 256 ? 256 : 512;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES + 1024;
  static constexpr int KSUB = BKT / (F16 ? 16 : 8);         // MMAs per product per stage
  // idesc: D f32; A/B type tf32 (2) or f16 (0); K-major both; N, M
  static constexpr uint32_t IDESC = (1u << 4) | ((F16 ? 0u : 2u) << 7) | ((F16 ? 0u : 2u) << 10) |
                                    ((uint32_t)(PBN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
};

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// Arrive on a (possibly remote) CTA's mbarrier.  Default .release.cta
// semantics: an explicit .release.cluster costs a GPU-scope MEMBAR per call,
// which the chunked epilogue would pay on every k-block; ordering of the
// TMEM reads it publishes comes from tcgen05.wait::ld + fence::before_thread_sync.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// With an L2 cache policy (createpolicy): the pair kernel keeps the A panels
// of its current m-group resident (evict_last) while B streams (evict_first).
__device__ __forceinline__ void tma_load_2d_pair_hint(const CUtensorMap* map, uint32_t leader_bar, void* dst, int c0,
                                                      int c1, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* map, uint32_t leader_bar, void* dst,
                                                 int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
template <bool F16>
__device__ __forceinline__ void tc_mma_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                            uint32_t idesc, uint32_t accumulate) {
  if (F16) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  } else {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n"
        "}\n" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
  }
}
template <bool PAIR, bool F16>
__device__ __forceinline__ void tc_mma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  if (PAIR) tc_mma_pair<F16>(d, a, b, idesc, acc);
  else tc_mma_one<F16>(d, a, b, idesc, acc);
}
__device__ __forceinline__ void tc_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)), "h"((uint16_t)3)
      : "memory");
}

template <bool F16>
__device__ __forceinline__ void tc_mma_pair_sc11(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                                 uint32_t idesc) {
  if (F16)
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p, 11;\n}\n" ::"r"(d_tmem), "l"(a_desc),
                 "l"(b_desc), "r"(idesc), "r"(1u)
                 : "memory");
  else
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p, 11;\n}\n" ::"r"(d_tmem), "l"(a_desc),
                 "l"(b_desc), "r"(idesc), "r"(1u)
                 : "memory");
}

template <int BKT, bool F16, bool TMA_C, int PBN = P_BN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(P_NUM_THREADS, 1)
k7_tf32x3_pair(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
               const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
               const __grid_constant__ CUtensorMap map_c,
               float* __restrict__ C, int M, int N, int ldc, int num_kb, int with_lolo, int group,
               unsigned int* __restrict__ wave_ctr, const float* __restrict__ inv_s,
               const float* __restrict__ inv_t, int l2_hints, const FixArgs fix, int K) {
  using Cfg = PairCfg<BKT, F16, PBN>;
  constexpr int NBUF = Cfg::NBUF;
  constexpr int P_STAGES = Cfg::STAGES;
  constexpr int P_A_TILE = Cfg::A_TILE;
  constexpr int P_B_TILE = Cfg::B_TILE;
  constexpr int P_STAGE_BYTES = Cfg::STAGE_BYTES;
  constexpr uint32_t kIdescPair = Cfg::IDESC;
  constexpr int NC = PBN / 2 / 32;                   // 32-column groups per epilogue warp (its half)
  constexpr int CH = ChunkK<F16>::value / BKT;           // stages per accumulation chunk
  static_assert(CH >= 1 && CH * BKT == ChunkK<F16>::value, "chunk length");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_stage = smem + P_STAGES * P_STAGE_BYTES;      // 1 KB-aligned (stages are)
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_stage + Cfg::EPI_BYTES);
  uint64_t* empty = full + P_STAGES;
  uint64_t* tfull = empty + P_STAGES;                // [NBUF]
  uint64_t* tempty = tfull + NBUF;                   // [NBUF] (leader's copy counts both CTAs' warps)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + NBUF);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#ifdef ELV_K7_PROF
  unsigned long long prof[K7_PROF_SLOTS] = {};
#endif
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int tiles_m = (M + 2 * P_BM - 1) / (2 * P_BM), tiles_n = (N + PBN - 1) / PBN;
  const int num_tiles = tiles_m * tiles_n;
  const int cluster_id = blockIdx.x >> 1, num_clusters = gridDim.x >> 1;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_ahi); tma_prefetch_desc(&map_alo);
    tma_prefetch_desc(&map_bhi); tma_prefetch_desc(&map_blo);
    if (TMA_C) tma_prefetch_desc(&map_c);
    for (int s = 0; s < P_STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < NBUF; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 2 * P_EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  griddep_wait();                                   // operand planes from the preceding split kernel
  griddep_launch_dependents();                      // the range-guard fix-up may be scheduled (it waits for us)

  // tile t: rows [mt*256, +256) (this CTA: + rank*128), cols [nt*256, +256) (this CTA stages + rank*128)
  auto coords = [&](int t, int& m0, int& n0) {
    const int GROUP = group;
    const int per_group = GROUP * tiles_n;
    const int g = t / per_group;
    const int first_m = g * GROUP;
    const int gm = min(tiles_m - first_m, GROUP);
    const int in = t - g * per_group;
    m0 = (first_m + in % gm) * 2 * P_BM;
    n0 = (in / gm) * PBN;
  };

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs) ----------------
      const uint32_t full0 = mapa_rank(smem_u32(&full[0]), 0);
      const uint64_t pol_a = l2_policy_evict_last();
      const uint64_t pol_b = (l2_hints & 3) >= 2 ? l2_policy_evict_first() : l2_policy_evict_normal();
      // bit 2 (ELV_SERPENTINE=1, an experiment): odd waves walk the k-blocks
      // backwards, so they start on the slabs of the m-group's A panels the
      // previous wave left in L2.  Each element's chunk sums then run in the
      // order of its wave's parity: within the tolerance, but no longer
      // bitwise the 1-CTA kernel / other tilings, hence off by default.
      const bool serp = (l2_hints & 4) != 0;
      int s = 0; uint32_t ph = 0;
      int wave = 0;
      for (int t = cluster_id; t < num_tiles; t += num_clusters, ++wave) {
        int m0, n0;
        coords(t, m0, n0);
        PROF_T(w0);
        if (wave_ctr != nullptr && wave > 0) wave_sync_wait(wave_ctr, (unsigned)(wave * gridDim.x));
        PROF_T(w1);
        PROF_ADD(4, w1 - w0);
        const int ma = m0 + (int)rank * P_BM, nb = n0 + (int)rank * (PBN / 2);
        for (int kb = 0; kb < num_kb; ++kb) {
          PROF_T(e0);
          mbar_wait(&empty[s], ph ^ 1);
          PROF_T(e1);
          PROF_ADD(3, e1 - e0);
          uint8_t* st = smem + s * P_STAGE_BYTES;
          const uint32_t bar = full0 + (uint32_t)(s * 8);
          const int k0 = (serp && (wave & 1)) ? (num_kb - 1 - kb) * BKT : kb * BKT;
          if (leader) mbar_expect_tx(&full[s], 2 * P_STAGE_BYTES);   // both CTAs' bytes
          if (l2_hints & 3) {
            tma_load_2d_pair_hint(&map_ahi, bar, st, k0, ma, pol_a);
            tma_load_2d_pair_hint(&map_alo, bar, st + P_A_TILE, k0, ma, pol_a);
            tma_load_2d_pair_hint(&map_bhi, bar, st + 2 * P_A_TILE, k0, nb, pol_b);
            tma_load_2d_pair_hint(&map_blo, bar, st + 2 * P_A_TILE + P_B_TILE, k0, nb, pol_b);
          } else {
            tma_load_2d_pair(&map_ahi, bar, st, k0, ma);
            tma_load_2d_pair(&map_alo, bar, st + P_A_TILE, k0, ma);
            tma_load_2d_pair(&map_bhi, bar, st + 2 * P_A_TILE, k0, nb);
            tma_load_2d_pair(&map_blo, bar, st + 2 * P_A_TILE + P_B_TILE, k0, nb);
          }
          if (++s == P_STAGES) { s = 0; ph ^= 1; }
        }
        if (wave_ctr != nullptr) atomicAdd(wave_ctr, 1u);
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader CTA only): one chunk per k-block ----------------
      // Each k-block accumulates into a FRESH TMEM buffer (ping-pong, 2 x 256
      // columns) that the epilogue drains into fp32 registers with
      // round-to-nearest adds.  The tensor core rounds every accumulate
      // toward zero; over one long chain that bias grows with K (measured:
      // 10.9x the tau=1 bound at K=8192 on non-negative inputs,
      // profiles/r2/tc_numerics_before_chunked.jsonl).  Within a chunk the
      // correction products go first, so they accumulate at their own (small)
      // scale, and the hi.hi products last: only KSUB truncations per chunk
      // fall on the chunk's magnitude.  fp16: the lo planes carry 2^11, and
      // the first hi.hi MMA rescales the correction partial by 2^-11
      // (scale-input-d), so one accumulator holds the whole chunk.
      int s = 0; uint32_t ph = 0;
      uint32_t q = 0;
      PROF_T(m_start);
      for (int t = cluster_id; t < num_tiles; t += num_clusters) {
        PROF_ADD(7, 1);
        for (int kb = 0; kb < num_kb; kb += CH, ++q) {
          const uint32_t b = q % NBUF;
          PROF_T(q0);
          mbar_wait(&tempty[b], ((q / NBUF) & 1) ^ 1);
          PROF_T(f0);
          PROF_ADD(0, f0 - q0);
          uint64_t ahi[CH], alo[CH], bhi[CH], blo[CH];
          int ss[CH];
#pragma unroll
          for (int j = 0; j < CH; ++j) {
            mbar_wait(&full[s], ph);
            const uint32_t st = smem_u32(smem + s * P_STAGE_BYTES);
            // 128 B rows (tf32 BK=32 / f16 BK=64): 128B swizzle; 64 B rows: 64B
            ahi[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st);
            alo[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st + P_A_TILE);
            bhi[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st + 2 * P_A_TILE);
            blo[j] = umma_desc_k<Cfg::ROW_BYTES / 4>(st + 2 * P_A_TILE + P_B_TILE);
            ss[j] = s;
            if (++s == P_STAGES) { s = 0; ph ^= 1; }
          }
          PROF_T(f1);
          PROF_ADD(1, f1 - f0);
          tc_fence_after();
          mma_chunk<true, F16, Cfg::KSUB, CH>(tmem_base + b * (uint32_t)PBN, ahi, alo, bhi, blo, kIdescPair,
                                              with_lolo);
#pragma unroll
          for (int j = 0; j < CH; ++j) tc_commit_pair(&empty[ss[j]]);   // frees the slots in both CTAs
          tc_commit_pair(&tfull[b]);            // chunk ready in both CTAs
        }
      }
      PROF_T(m_end);
      PROF_ADD(2, m_end - m_start);
    }
  } else {
    // ---------------- epilogue (warps 2..9, both CTAs) ----------------
    // warp -> TMEM lane group g (rows), column half h; each thread owns one
    // row's 128 columns as register running sums across the chunks
    const int g = warp & 3;
    const int h = (warp - 2) >> 2;
    const bool vecC = ((reinterpret_cast<uintptr_t>(C) & 15u) == 0) && (ldc & 3) == 0;
    const uint32_t tempty0 = mapa_rank(smem_u32(&tempty[0]), 0);
    uint32_t q = 0;
    for (int t = cluster_id; t < num_tiles; t += num_clusters) {
      int m0, n0;
      coords(t, m0, n0);
      const int row = m0 + (int)rank * P_BM + g * 32 + lane;
      const uint32_t lane_base = tmem_base + ((uint32_t)(g * 32) << 16) + (uint32_t)(h * (PBN / 2));
      float acc[NC * 32];
#pragma unroll
      for (int i = 0; i < NC * 32; ++i) acc[i] = 0.f;
#pragma unroll 1
      for (int kb = 0; kb < num_kb; kb += CH, ++q) {
        const uint32_t b = q % NBUF;
        PROF_T(c0);
        mbar_wait(&tfull[b], (q / NBUF) & 1);
        tc_fence_after();
        PROF_T(c1);
        drain_add<NC>(lane_base + b * (uint32_t)PBN, acc);
        tc_fence_before();
        __syncwarp();
        PROF_T(c2);
        if (lane == 0) mbar_arrive_cluster(tempty0 + b * 8);
        PROF_T(c3);
        PROF_ADD(5, c1 - c0);
        PROF_ADD(8, c2 - c1);
        PROF_ADD(10, c3 - c2);
        PROF_ADD(9, 1);
      }
      PROF_T(d1);
      float* crow = C + (size_t)row * ldc;
      const int er = (F16 && row < M) ? pow2_exp(__ldg(inv_s + row)) : 0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int col = n0 + h * (PBN / 2) + c * 32;
        float* v = acc + c * 32;
        if (F16) unscale_chunk(v, er, col < N - lane ? __ldg(inv_t + col + lane) : 1.f);
        if (TMA_C) {
          // 32 x 32 chunk -> this warp's SMEM tile in the 128B-swizzled layout
          // the tensor map expects -> one bulk tensor store (clipped at M, N)
          uint8_t* tile = epi_stage + (warp - 2) * 4096;
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            *reinterpret_cast<float4*>(tile + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&map_c)),
                "r"(col), "r"(row - lane), "r"(smem_u32(tile))
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else if (row < M && col < N) {
          if (vecC && col + 31 < N) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(crow + col + 4 * j) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < N) crow[col + j] = v[j];
          }
        }
      }
      PROF_T(d2);
      PROF_ADD(6, d2 - d1);
      if (PBN != P_BN && fix.A != nullptr) {
        // range-guard fix-up of this thread's outputs (the narrow small-problem pairs; see k7_tf32x3):
        // after this warp's C stores have completed (TMA bulk stores are async)
        if (TMA_C) {
          if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
          __syncwarp();
        }
        const bool frow = row < M && __ldg(fix.flag_a + row) != 0u;
#pragma unroll 1
        for (int c = 0; c < NC; ++c) {
          const int col0 = n0 + h * (PBN / 2) + c * 32;
          const unsigned int fcol =
              __ballot_sync(0xffffffffu, col0 + lane < N && __ldg(fix.flag_b + col0 + lane) != 0u);
          if (row >= M || (!frow && fcol == 0u)) continue;
          for (int j = 0; j < 32 && col0 + j < N; ++j) {
            if (!frow && !((fcol >> j) & 1u)) continue;
            const float* a = fix.A + (size_t)row * fix.lda;
            const float* bb = fix.B + col0 + j;
            float sacc = 0.f;
            for (int k = 0; k < K; ++k) sacc = fmaf(__ldg(a + k), __ldg(bb + (size_t)k * fix.ldb), sacc);
            C[(size_t)row * ldc + col0 + j] = sacc;
          }
        }
      }
    }
  }
#ifdef ELV_K7_PROF
  if (lane == 0 && warp <= 2 && blockIdx.x < 512)
    for (int i = 0; i < K7_PROF_SLOTS; ++i) if (prof[i]) atomicAdd(&g_k7_prof[blockIdx.x][i], prof[i]);
#endif

  if (TMA_C && warp >= 2 && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ----------------------------------------------------------------------------
// split prepass: A -> A_hi, A_lo (M x Kp, K-major);  B -> Bt_hi, Bt_lo (N x Kp)
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Range guard.  The 3-product split is exact to 2^-22 only for finite
// elements inside the encoding's window: tf32 keeps fp32's exponent range,
// so only |x| < 2^-100 (lo would leave the normal range) and non-finite x
// fall outside; the scaled fp16 encoding keeps an element only if its scaled
// value is >= 2^-14 (fp16's normal range; below it hi and lo lose relative
// precision), i.e. within 2^29 of its row / column maximum.  The split
// kernels mark every row of A / column of B holding such an element
// (flag = 1; zeroed first, see the callers), and k_tc_fixup recomputes the
// marked rows and columns of C with the SIMT fp32 FMA chain.
__device__ __forceinline__ bool tf32_out_of_window(float x) {
  const float a = fabsf(x);
  return !(a <= 3.402823466e38f) || (a != 0.f && a < 0x1p-100f);
}
__device__ __forceinline__ bool f16_out_of_window(float x, float y) {
  const float b = fabsf(y);
  return !(fabsf(x) <= 3.402823466e38f) || (b != 0.f && b < 0x1p-14f);
}

// One row segment of 4 k's per thread: float4 in, two float4 out (rows of A
// are K-major already, so the planes are a padded elementwise map).  2D grid:
// x over Kp/4, y-stride over rows -- no 64-bit division per element.
__device__ __forceinline__ void split_a_block(const float* __restrict__ A, float* __restrict__ hi,
                                              float* __restrict__ lo, int M, int K, int lda, int Kp, bool vec,
                                              int bx, int by, int gy, unsigned int* __restrict__ flag) {
  const int k = (bx * 256 + threadIdx.x) * 4;
  if (k >= Kp) return;
  for (int r = by; r < M; r += gy) {
    const float* src = A + (size_t)r * lda + k;
    float4 x;
    if (vec && k + 3 < K) {
      x = __ldg(reinterpret_cast<const float4*>(src));
    } else {
      x.x = k + 0 < K ? __ldg(src + 0) : 0.f;
      x.y = k + 1 < K ? __ldg(src + 1) : 0.f;
      x.z = k + 2 < K ? __ldg(src + 2) : 0.f;
      x.w = k + 3 < K ? __ldg(src + 3) : 0.f;
    }
    if (tf32_out_of_window(x.x) || tf32_out_of_window(x.y) || tf32_out_of_window(x.z) || tf32_out_of_window(x.w)) {
      griddep_wait();                             // flags zeroed by k_zero_u32 (PDL launch; no-op otherwise)
      flag[r] = 1u;
    }
    const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(x.z), tf32_rna(x.w));
    const float4 l = make_float4(tf32_rna(x.x - h.x), tf32_rna(x.y - h.y), tf32_rna(x.z - h.z),
                                 tf32_rna(x.w - h.w));
    const size_t o = (size_t)r * Kp + k;
    *reinterpret_cast<float4*>(hi + o) = h;
    *reinterpret_cast<float4*>(lo + o) = l;
  }
}
__global__ void __launch_bounds__(256)
k_split_a(const float* __restrict__ A, float* __restrict__ hi, float* __restrict__ lo, int M, int K,
          int lda, int Kp, bool vec, unsigned int* __restrict__ flag) {
  split_a_block(A, hi, lo, M, K, lda, Kp, vec, blockIdx.x, blockIdx.y, gridDim.y, flag);
}

// 32x32 tiles through SMEM: reads of B rows and writes of Bt rows coalesce.
// PACKED: the source is packedB panels [N/32][K][32] (the packB layout the
// row-shard driver broadcasts) instead of row-major B.
template <bool PACKED>
__device__ __forceinline__ void split_transpose_b_block(const float* __restrict__ B, float* __restrict__ hi,
                                                        float* __restrict__ lo, int K, int N, int ldb, int Kp,
                                                        int bx, int by, unsigned int* __restrict__ flag) {
  __shared__ float t[32][33];
  const int k0 = by * 32, n0 = bx * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int k = k0 + ty + 8 * r, n = n0 + tx;
    float v = 0.f;
    if (k < K && n < N)
      v = PACKED ? __ldg(B + ((size_t)(n >> 5) * K + k) * 32 + (n & 31)) : __ldg(B + (size_t)k * ldb + n);
    t[ty + 8 * r][tx] = v;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int n = n0 + ty + 8 * r, k = k0 + tx;
    if (n < N && k < Kp) {
      const float x = t[tx][ty + 8 * r];
      if (tf32_out_of_window(x)) {
        griddep_wait();                           // flags zeroed by k_zero_u32 (PDL launch; no-op otherwise)
        flag[n] = 1u;
      }
      const float h = tf32_rna(x);
      hi[(size_t)n * Kp + k] = h;
      lo[(size_t)n * Kp + k] = tf32_rna(x - h);
    }
  }
}
template <bool PACKED>
__global__ void __launch_bounds__(256)
k_split_transpose_b(const float* __restrict__ B, float* __restrict__ hi, float* __restrict__ lo,
                    int K, int N, int ldb, int Kp, unsigned int* __restrict__ flag) {
  split_transpose_b_block<PACKED>(B, hi, lo, K, N, ldb, Kp, blockIdx.x, blockIdx.y, flag);
}

// elv_gemm's prepare for variant 7 in one launch: blocks [0, ga) split A,
// the rest split-transpose B (the two are independent).
__global__ void __launch_bounds__(256)
k_split_ab(const float* __restrict__ A, float* __restrict__ ahi, float* __restrict__ alo, int M, int lda,
           bool vecA, int gxa, int gya, const float* __restrict__ B, float* __restrict__ bhi,
           float* __restrict__ blo, int N, int ldb, int gxb, int K, int Kp, unsigned int* __restrict__ flag_a,
           unsigned int* __restrict__ flag_b) {
  griddep_launch_dependents();
  const int b = blockIdx.x, ga = gxa * gya;
  if (b < ga) split_a_block(A, ahi, alo, M, K, lda, Kp, vecA, b % gxa, b / gxa, gya, flag_a);
  else split_transpose_b_block<false>(B, bhi, blo, K, N, ldb, Kp, (b - ga) % gxb, (b - ga) / gxb, flag_b);
  // PDL-launched behind k_zero_u32 (elv_gemm's prepare): our completion must
  // imply the flags' zeroing is done, since the GEMM / fix-up that wait for
  // us read them -- blocks that set no flag wait here, after their split
  griddep_wait();
}

// Zeroes n words and lets its PDL dependent start at once: replaces a
// cudaMemsetAsync before the prepare kernels (a memset node serialises the
// chain; the dependents overlap their loads with it and wait
// (griddepcontrol.wait) only before touching the zeroed words).
__global__ void __launch_bounds__(256) k_zero_u32(unsigned int* __restrict__ p, size_t n) {
  griddep_launch_dependents();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = 0u;
}
static int zero_words(unsigned int* p, size_t n, cudaStream_t st) {
  if (n == 0) return ELV_OK;
  const size_t want = (n + 1023) / 1024;
  const unsigned blocks = (unsigned)(want < 148 ? want : 148);
  k_zero_u32<<<blocks, 256, 0, st>>>(p, n);
  return cudaPeekAtLastError() == cudaSuccess ? ELV_OK : check_launch("zero_words");
}

// ----------------------------------------------------------------------------
// Range-guard fix-up: the rows of A / columns of B that a split marked
// (tf32_out_of_window / f16_out_of_window) are recomputed after the tensor-
// core GEMM with the SIMT kernels' arithmetic -- C_ij = fmaf chain over k
// ascending from 0, the parallel schedule's sequential fold
// (reference interp.py:84-89, 145-148) in fp32.  One block per 64-row segment
// of A (blocks [0, gm)) or 64-column segment of B (the rest): a segment
// without marks returns after reading its 64 flags, so with nothing marked
// the call is one short launch.  Marked segments work in groups of 16 rows
// (x 256 columns per pass, 16 FMAs per B load) or 16 columns (x 256 rows,
// A staged through SMEM so its rows are read coalesced).
constexpr int FIX_SEG = 64, FIX_GRP = 16, FIX_T = 256, FIX_KT = 32;

__device__ __forceinline__ float fix_ld_b(const float* __restrict__ B, int ldb, int packed, int K, int k, int n) {
  return packed ? __ldg(B + ((size_t)(n >> 5) * K + k) * 32 + (n & 31)) : __ldg(B + (size_t)k * ldb + n);
}

__global__ void __launch_bounds__(FIX_T)
k_tc_fixup(const float* __restrict__ A, int lda, const float* __restrict__ B, int ldb, int b_packed,
           float* __restrict__ C, int ldc, int M, int N, int K, const unsigned int* __restrict__ flag_a,
           const unsigned int* __restrict__ flag_b) {
  __shared__ int list[FIX_SEG];
  __shared__ int cnt;
  __shared__ float As[FIX_T][FIX_KT + 1];
  __shared__ float Bs[FIX_KT][FIX_GRP + 1];
  griddep_wait();                                   // the GEMM's C (and the splits' flags) are complete
  const int gm = (M + FIX_SEG - 1) / FIX_SEG;
  const bool rowmode = (int)blockIdx.x < gm;
  const int seg0 = (rowmode ? (int)blockIdx.x : (int)blockIdx.x - gm) * FIX_SEG;
  const int lim = rowmode ? M : N;
  const unsigned int* flag = rowmode ? flag_a : flag_b;
  const int tid = threadIdx.x;
  if (tid == 0) cnt = 0;
  __syncthreads();
  if (tid < FIX_SEG && seg0 + tid < lim && __ldcg(flag + seg0 + tid) != 0u) list[atomicAdd(&cnt, 1)] = seg0 + tid;
  __syncthreads();
  const int n = cnt;
  if (n == 0) return;
  for (int g0 = 0; g0 < n; g0 += FIX_GRP) {
    const int gn = min(FIX_GRP, n - g0);
    if (rowmode) {
      // rows list[g0 .. g0+gn) x all N columns, 256 columns per pass
      for (int c0 = 0; c0 < N; c0 += FIX_T) {
        const int col = c0 + tid;
        float acc[FIX_GRP];
#pragma unroll
        for (int r = 0; r < FIX_GRP; ++r) acc[r] = 0.f;
        for (int k0 = 0; k0 < K; k0 += FIX_KT) {
          const int kn = min(FIX_KT, K - k0);
#pragma unroll
          for (int i = 0; i < FIX_GRP * FIX_KT / FIX_T; ++i) {
            const int idx = tid + i * FIX_T, r = idx / FIX_KT, kk = idx % FIX_KT;
            As[r][kk] = (r < gn && kk < kn) ? __ldg(A + (size_t)list[g0 + r] * lda + k0 + kk) : 0.f;
          }
          __syncthreads();
          if (col < N) {
            for (int kk = 0; kk < kn; ++kk) {
              const float b = fix_ld_b(B, ldb, b_packed, K, k0 + kk, col);
#pragma unroll
              for (int r = 0; r < FIX_GRP; ++r) acc[r] = fmaf(As[r][kk], b, acc[r]);
            }
          }
          __syncthreads();
        }
        if (col < N)
          for (int r = 0; r < gn; ++r) C[(size_t)list[g0 + r] * ldc + col] = acc[r];
      }
    } else {
      // all M rows x columns list[g0 .. g0+gn), 256 rows per pass
      const int warp = tid >> 5, lane = tid & 31;
      for (int r0 = 0; r0 < M; r0 += FIX_T) {
        const int row = r0 + tid;
        float acc[FIX_GRP];
#pragma unroll
        for (int c = 0; c < FIX_GRP; ++c) acc[c] = 0.f;
        for (int k0 = 0; k0 < K; k0 += FIX_KT) {
          const int kn = min(FIX_KT, K - k0);
          for (int rr = 0; rr < 32; ++rr) {           // warp w stages rows w*32 .. w*32+31, lane = k
            const int ar = r0 + warp * 32 + rr;
            As[warp * 32 + rr][lane] = (ar < M && lane < kn) ? __ldg(A + (size_t)ar * lda + k0 + lane) : 0.f;
          }
#pragma unroll
          for (int i = 0; i < FIX_GRP * FIX_KT / FIX_T; ++i) {
            const int idx = tid + i * FIX_T, kk = idx / FIX_GRP, c = idx % FIX_GRP;
            Bs[kk][c] = (c < gn && kk < kn) ? fix_ld_b(B, ldb, b_packed, K, k0 + kk, list[g0 + c]) : 0.f;
          }
          __syncthreads();
          for (int kk = 0; kk < kn; ++kk) {
            const float a = As[tid][kk];
#pragma unroll
            for (int c = 0; c < FIX_GRP; ++c) acc[c] = fmaf(a, Bs[kk][c], acc[c]);
          }
          __syncthreads();
        }
        if (row < M)
          for (int c = 0; c < gn; ++c) C[(size_t)row * ldc + list[g0 + c]] = acc[c];
      }
    }
  }
}

// ----------------------------------------------------------------------------
// K7F: 3xTF32 with the operand split fused into the pair kernel -- no
// preparation pass.  The producers TMA the RAW fp32 tiles: A (K-major, as
// the planes kernel's A_hi box) into the A_hi slot, B (row-major K x N, four
// [32 k][32 n] boxes, 128B swizzle) into the B_lo slot.  Dedicated converter
// warps split each landed stage -- A in place (hi over the raw tile, lo into
// A_lo, same swizzled offsets), B transposed into the K-major B_hi / B_lo
// rows the MMA reads (kind::tf32 takes K-major operands only: an MN-major B
// descriptor produced no result, scripts/probes/tf32_mn_probe.cu) -- with the
// planes split's arithmetic, so the result is bitwise the planes path's.
// The range guard (tf32_out_of_window) is applied to the converted elements
// (every tile sees the full K of its rows and columns).  Barriers per stage:
// full[s] (local TMA), conv[s] (leader: its converters + the peer's
// converted stage, relayed by the peer's warp 2 with a cluster release),
// empty[s] (MMA done, multicast commit).
// Measured: the conversion sits between TMA landing
// and the MMA with only three 64 KB stages of slack in 227 KB of SMEM, and
// the pipeline has none to spare -- the same kernel with the conversion
// skipped runs at 261 TF (planes path 250 TF) but converting A alone costs
// ~17 % and A and B ~30-45 % at 32768^2 x 8192 -- so variant 7 keeps the
// planes path by default (ELV_TF32X3_FUSED=1 selects this one).
constexpr int F_STAGES = 3;
constexpr int F_A_TILE = P_BM * 128;                       // 128 rows x 32 k fp32 (128 B rows)
constexpr int F_B_TILE = (P_BN / 2) * 128;                 // this CTA's 128 columns x 32 k
constexpr int F_STAGE = 2 * F_A_TILE + 2 * F_B_TILE;       // [A_hi | A_lo | B_hi | B_lo]
constexpr int F_EPI = 8 * 32 * 32 * 4;
constexpr int F_SMEM = F_STAGES * F_STAGE + F_EPI + 256 + 1024;
constexpr uint32_t F_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(P_BN >> 3) << 17) |
                             ((uint32_t)(256 >> 4) << 24);


__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAITC_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAITC_%=;\n"
      "}\n" ::"r"(a), "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_release_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

// 16 warps: warpgroup 0 = TMA producer (w0), MMA issuer (w1, leader), the
// cross-CTA relay (w2), a converter (w3); warpgroups 1-2 = epilogue (w4..w11,
// TMEM lane group w & 3, column half (w - 4) >> 2); warpgroup 3 = converters
// (w12..w15).  setmaxnreg gives the epilogue 168 registers (128 running sums
// per thread) and the other warpgroups 88.
constexpr int F_NUM_THREADS = 512;
constexpr int F_CONV_WARPS = 5;
constexpr int F_EPI_W0 = 4;

__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, float x, float y, float z, float w) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(x), "f"(y), "f"(z), "f"(w) : "memory");
}
// the planes split (split_a_block): hi = rna_tf32(x), lo = rna_tf32(x - hi).
// (A truncated hi -- what kind::tf32 MMAs read from a raw fp32 operand,
// scripts/probes/tf32_mn_probe.cu -- would let the raw TMA tile serve as the
// hi operand without a write, but leaves |x - hi - lo| up to 2^-21 |x| instead
// of 2^-23: 3.5x the tau = 2 bound at K = 1, tests/test_gpu_parity.py.)
// Range-guard accumulators over a group of elements: `tiny` = min over
// (2|x| bits - 2) (wraps for zeros, so only 0 < |x| < 2^-100 can land below
// 2 * 0x0d800000 - 2), `fin` = sum of the lo parts (NaN iff some element is
// inf / NaN: inf - trunc(inf) = NaN; finite lo sums cannot overflow).
struct Guard {
  uint32_t tiny = 0xffffffffu;
  float fin = 0.f;
  __device__ __forceinline__ void add(float x, float lo) {
    tiny = min(tiny, (__float_as_uint(x) << 1) - 2u);
    fin += lo;
  }
  __device__ __forceinline__ bool bad() const { return tiny < 2u * 0x0d800000u - 2u || !(fabsf(fin) <= 3.402823466e38f); }
};

// One launch per GEMM.  FUSE_B: B is split (and transposed) in the kernel
// from raw row-major B; otherwise ("A-fused") B arrives as tf32 hi/lo planes
// (map_b, map_b2: the planes kernel's K-major Bt boxes, e.g. a broadcast
// chunk split on arrival) and only A is split here.
template <bool TMA_C, bool FUSE_B>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(F_NUM_THREADS, 1)
k7f_tf32x3_fused(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                 const __grid_constant__ CUtensorMap map_b2, const __grid_constant__ CUtensorMap map_c,
                 float* __restrict__ C, int M, int N, int ldc, int num_kb, int with_lolo, int group,
                 unsigned int* __restrict__ wave_ctr, unsigned int* __restrict__ flag_a,
                 unsigned int* __restrict__ flag_b, int dbg) {
  constexpr int NC = P_BN / 2 / 32;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* epi_stage = smem + F_STAGES * F_STAGE;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_stage + F_EPI);   // this CTA's TMA landed
  uint64_t* conv = full + F_STAGES;                  // converted (leader: + the peer's relayed arrival)
  uint64_t* empty = conv + F_STAGES;
  uint64_t* tfull = empty + F_STAGES;                // [2]
  uint64_t* tempty = tfull + 2;                      // [2]
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int tiles_m = (M + 2 * P_BM - 1) / (2 * P_BM), tiles_n = (N + P_BN - 1) / P_BN;
  const int num_tiles = tiles_m * tiles_n;
  const int cluster_id = blockIdx.x >> 1, num_clusters = gridDim.x >> 1;
  constexpr int TX = F_A_TILE + (FUSE_B ? 1 : 2) * F_B_TILE;   // bytes per full[s] phase

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&map_a); tma_prefetch_desc(&map_b);
    if (!FUSE_B) tma_prefetch_desc(&map_b2);
    if (TMA_C) tma_prefetch_desc(&map_c);
    for (int s = 0; s < F_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], F_CONV_WARPS + (leader ? 1 : 0));
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 2 * P_EPI_WARPS); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_holder)), "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  griddep_wait();                                   // flags zeroed / operands written by preceding work
  griddep_launch_dependents();                      // the range-guard fix-up may be scheduled (it waits for us)

  auto coords = [&](int t, int& m0, int& n0) {
    const int per_group = group * tiles_n;
    const int g = t / per_group;
    const int first_m = g * group;
    const int gm = min(tiles_m - first_m, group);
    const int in = t - g * per_group;
    m0 = (first_m + in % gm) * 2 * P_BM;
    n0 = (in / gm) * P_BN;
  };

  if (warp >= F_EPI_W0 && warp < F_EPI_W0 + P_EPI_WARPS) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 168;\n" ::: "memory");
    // ---------------- epilogue (w4..w11, both CTAs): as k7_tf32x3_pair ----------------
    const int g = warp & 3;
    const int h = (warp - F_EPI_W0) >> 2;
    const bool vecC = ((reinterpret_cast<uintptr_t>(C) & 15u) == 0) && (ldc & 3) == 0;
    const uint32_t tempty0 = mapa_rank(smem_u32(&tempty[0]), 0);
    uint32_t q = 0;
    for (int t = cluster_id; t < num_tiles; t += num_clusters) {
      int m0, n0;
      coords(t, m0, n0);
      const int row = m0 + (int)rank * P_BM + g * 32 + lane;
      const uint32_t lane_base = tmem_base + ((uint32_t)(g * 32) << 16) + (uint32_t)(h * (P_BN / 2));
      float acc[NC * 32];
#pragma unroll
      for (int i = 0; i < NC * 32; ++i) acc[i] = 0.f;
#pragma unroll 1
      for (int kb = 0; kb < num_kb; ++kb, ++q) {
        const uint32_t b = q & 1;
        mbar_wait(&tfull[b], (q >> 1) & 1);
        tc_fence_after();
        drain_add<NC>(lane_base + b * (uint32_t)P_BN, acc);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(tempty0 + b * 8);
      }
      float* crow = C + (size_t)row * ldc;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        const int col = n0 + h * (P_BN / 2) + c * 32;
        float* v = acc + c * 32;
        if (TMA_C) {
          const uint32_t tile = smem_u32(epi_stage + (warp - F_EPI_W0) * 4096);
          if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j)
            sts128(tile + (uint32_t)(lane * 128 + ((j ^ (lane & 7)) << 4)), v[4 * j], v[4 * j + 1], v[4 * j + 2],
                   v[4 * j + 3]);
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            asm volatile(
                "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(
                    reinterpret_cast<uint64_t>(&map_c)),
                "r"(col), "r"(row - lane), "r"(tile)
                : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        } else if (row < M && col < N) {
          if (vecC && col + 31 < N) {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(crow + col + 4 * j) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (col + j < N) crow[col + j] = v[j];
          }
        }
      }
    }
    if (TMA_C && lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;\n" ::: "memory");
    if (warp == 0) {
      if (lane == 0) {
        // ---------------- TMA producer (both CTAs) ----------------
        // raw A -> A_hi slot; FUSE_B: raw B (4 boxes [32 k][32 n], 128B swizzle)
        // -> B_lo slot, else the B planes -> B_hi / B_lo; on this CTA's barrier
        int s = 0; uint32_t ph = 0;
        int wave = 0;
        for (int t = cluster_id; t < num_tiles; t += num_clusters, ++wave) {
          int m0, n0;
          coords(t, m0, n0);
          if (wave_ctr != nullptr && wave > 0) wave_sync_wait(wave_ctr, (unsigned)(wave * gridDim.x));
          const int ma = m0 + (int)rank * P_BM, nb = n0 + (int)rank * (P_BN / 2);
          for (int kb = 0; kb < num_kb; ++kb) {
            mbar_wait(&empty[s], ph ^ 1);
            uint8_t* st = smem + s * F_STAGE;
            const int k0 = kb * 32;
            mbar_expect_tx(&full[s], TX);
            tma_load_2d(&map_a, &full[s], st, k0, ma);
            if (FUSE_B) {
#pragma unroll
              for (int j = 0; j < 4; ++j)
                tma_load_2d(&map_b, &full[s], st + 2 * F_A_TILE + F_B_TILE + j * 4096, nb + 32 * j, k0);
            } else {
              tma_load_2d(&map_b, &full[s], st + 2 * F_A_TILE, k0, nb);
              tma_load_2d(&map_b2, &full[s], st + 2 * F_A_TILE + F_B_TILE, k0, nb);
            }
            if (++s == F_STAGES) { s = 0; ph ^= 1; }
          }
          if (wave_ctr != nullptr) atomicAdd(wave_ctr, 1u);
        }
      }
    } else if (warp == 1) {
      if (leader && lane == 0) {
        // ---------------- MMA issuer (leader CTA): one chunk per k-block ----------------
        // the k7_tf32x3_pair chunk (hi.lo, lo.hi, [lo.lo], hi.hi; same order, same bits)
        int s = 0; uint32_t ph = 0;
        uint32_t q = 0;
        for (int t = cluster_id; t < num_tiles; t += num_clusters) {
          for (int kb = 0; kb < num_kb; ++kb, ++q) {
            const uint32_t b = q & 1, d = tmem_base + b * (uint32_t)P_BN;
            mbar_wait(&tempty[b], ((q >> 1) & 1) ^ 1);
            const uint32_t st = smem_u32(smem + s * F_STAGE);
            const uint64_t ahi = umma_desc_sw128(st), alo = umma_desc_sw128(st + F_A_TILE);
            const uint64_t bhi = umma_desc_sw128(st + 2 * F_A_TILE);
            const uint64_t blo = umma_desc_sw128(st + 2 * F_A_TILE + F_B_TILE);
            mbar_wait_cluster(&conv[s], ph);     // both CTAs' stages converted
            tc_fence_after();
#pragma unroll
            for (int k = 0; k < 4; ++k) tc_mma_pair<false>(d, ahi + 2 * k, blo + 2 * k, F_IDESC, k != 0);
#pragma unroll
            for (int k = 0; k < 4; ++k) tc_mma_pair<false>(d, alo + 2 * k, bhi + 2 * k, F_IDESC, 1u);
            if (with_lolo) {
#pragma unroll
              for (int k = 0; k < 4; ++k) tc_mma_pair<false>(d, alo + 2 * k, blo + 2 * k, F_IDESC, 1u);
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) tc_mma_pair<false>(d, ahi + 2 * k, bhi + 2 * k, F_IDESC, 1u);
            tc_commit_pair(&empty[s]);
            tc_commit_pair(&tfull[b]);
            if (++s == F_STAGES) { s = 0; ph ^= 1; }
          }
        }
      }
    } else if (warp == 2) {
      if (lane == 0) {
        // ---------------- cross-CTA relay (peer): "my stage is converted" ----------------
        // -> the leader's conv[s] with cluster release (one thread pays the
        // release fence, off the converters' path)
        int s = 0; uint32_t ph = 0;
        const uint32_t conv0 = mapa_rank(smem_u32(&conv[0]), 0);
        if (!leader) {
          for (int t = cluster_id; t < num_tiles; t += num_clusters)
            for (int kb = 0; kb < num_kb; ++kb) {
              mbar_wait(&conv[s], ph);
              mbar_arrive_release_cluster(conv0 + (uint32_t)(s * 8));
              if (++s == F_STAGES) { s = 0; ph ^= 1; }
            }
        }
      }
    } else {
      // ---------------- converters (w3, w12..w15; both CTAs) ----------------
      // Work per stage: B = 8 items of 32 lanes x (4 n x 4 k) (FUSE_B), A = 32
      // items of 32 float4.  Converter c takes B items {c, c + 5} and A items
      // [start[c], start[c + 1]) -- ~52 elements per lane each (A-fused: 6-7 A
      // items).  All loads of a stage are issued before any arithmetic.
      const int cw = warp == 3 ? 0 : warp - 11;            // 0..4
      constexpr uint64_t kAStart = 0ull | (5ull << 6) | (10ull << 12) | (15ull << 18) | (23ull << 24) |
                                   (32ull << 30);
      const int a_lo = FUSE_B ? (int)((kAStart >> (6 * cw)) & 63) : (32 * cw) / F_CONV_WARPS;
      const int a_hi = FUSE_B ? (int)((kAStart >> (6 * cw + 6)) & 63) : (32 * (cw + 1)) / F_CONV_WARPS;
      // B lane mapping (lane = 8 Q + e): k chunk kc = 4 (Q & 1) + (e >> 1), column
      // group cg (n = 4 cg .. 4 cg + 3) from e & 1, (e >> 2) ^ (item >> 2), Q >> 1,
      // item & 3.  Every quarter-warp of a 128-bit access then touches 8
      // distinct 16-byte bank groups both in the raw tile (128B-swizzled TMA
      // boxes) and in the K-major hi/lo rows: conflict-free reads and writes.
      const int Q = lane >> 3, e = lane & 7;
      const int kc = 4 * (Q & 1) + (e >> 1);
      int s = 0; uint32_t ph = 0;
      for (int t = cluster_id; t < num_tiles; t += num_clusters) {
        int m0, n0;
        coords(t, m0, n0);
        const int ma = m0 + (int)rank * P_BM, nb = n0 + (int)rank * (P_BN / 2);
        for (int kb = 0; kb < num_kb; ++kb) {
          mbar_wait(&full[s], ph);
          const uint32_t st = smem_u32(smem + s * F_STAGE);
          const uint32_t b_raw = st + 2 * F_A_TILE + F_B_TILE;
          float4 r[2][4];
          if (FUSE_B && !(dbg & 2)) {
#pragma unroll
            for (int u = 0; u < 2; ++u) {
              const int item = cw + 5 * u;
              if (item < 8) {
                const int cg = (e & 1) | ((((e >> 2) ^ (item >> 2)) & 1) << 1) | ((Q >> 1) << 2) | ((item & 3) << 3);
                const uint32_t box = b_raw + (uint32_t)((cg >> 3) * 4096);
#pragma unroll
                for (int qq = 0; qq < 4; ++qq) {
                  const int k = 4 * kc + qq;
                  r[u][qq] = lds128(box + (uint32_t)(k * 128 + (((cg & 7) ^ (k & 7)) << 4)));
                }
              }
            }
          }
          // A: hi (in place) and lo from the raw tile at the same (swizzled) offsets
          if (!(dbg & 1)) {
            constexpr int AMAX = FUSE_B ? 9 : 7;           // most A items of one converter
            float4 xa[AMAX];
#pragma unroll
            for (int j = 0; j < AMAX; ++j)
              if (a_lo + j < a_hi) xa[j] = lds128(st + (uint32_t)(((a_lo + j) * 32 + lane) * 16));
#pragma unroll
            for (int j = 0; j < AMAX; ++j) {
              if (a_lo + j < a_hi) {
                const int i = (a_lo + j) * 32 + lane;             // float4 index; tile row i / 8
                const float4 x = xa[j];
                const float h0 = tf32_rna(x.x), h1 = tf32_rna(x.y), h2 = tf32_rna(x.z), h3 = tf32_rna(x.w);
                const float l0 = tf32_rna(x.x - h0), l1 = tf32_rna(x.y - h1), l2 = tf32_rna(x.z - h2),
                            l3 = tf32_rna(x.w - h3);
                sts128(st + (uint32_t)(i * 16), h0, h1, h2, h3);
                sts128(st + F_A_TILE + (uint32_t)(i * 16), l0, l1, l2, l3);
                Guard gd;
                gd.add(x.x, l0); gd.add(x.y, l1); gd.add(x.z, l2); gd.add(x.w, l3);
                if (gd.bad()) flag_a[ma + (i >> 3)] = 1u;
              }
            }
          }
          if (FUSE_B) {
            asm volatile("bar.sync 1, 160;" ::: "memory");   // every raw B element read before the slot is overwritten
            if (!(dbg & 2)) {
#pragma unroll
              for (int u = 0; u < 2; ++u) {
                const int item = cw + 5 * u;
                if (item < 8) {
                  const int cg = (e & 1) | ((((e >> 2) ^ (item >> 2)) & 1) << 1) | ((Q >> 1) << 2) | ((item & 3) << 3);
#pragma unroll
                  for (int i = 0; i < 4; ++i) {
                    const int n = 4 * cg + i;
                    const float x0 = (&r[u][0].x)[i], x1 = (&r[u][1].x)[i], x2 = (&r[u][2].x)[i], x3 = (&r[u][3].x)[i];
                    const float h0 = tf32_rna(x0), h1 = tf32_rna(x1), h2 = tf32_rna(x2), h3 = tf32_rna(x3);
                    const float l0 = tf32_rna(x0 - h0), l1 = tf32_rna(x1 - h1), l2 = tf32_rna(x2 - h2),
                                l3 = tf32_rna(x3 - h3);
                    const uint32_t off = st + 2 * F_A_TILE + (uint32_t)(n * 128 + ((kc ^ (n & 7)) << 4));
                    sts128(off, h0, h1, h2, h3);
                    sts128(off + F_B_TILE, l0, l1, l2, l3);
                    Guard gd;
                    gd.add(x0, l0); gd.add(x1, l1); gd.add(x2, l2); gd.add(x3, l3);
                    if (gd.bad()) flag_b[nb + n] = 1u;
                  }
                }
              }
            }
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic writes -> tensor-core reads
          __syncwarp();
          if (lane == 0) mbar_arrive(&conv[s]);
          if (++s == F_STAGES) { s = 0; ph ^= 1; }
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS));
  }
}

// ----------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

int make_map(CUtensorMap* map, const void* base, int rows, int kp, int box_rows, int box_k = BK,
             bool f16 = false) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(ELV_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const size_t eb = f16 ? 2 : 4;
  const cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)kp * eb};
  const cuuint32_t box[2] = {(cuuint32_t)box_k, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, f16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   box_k * eb == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ELV_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ELV_OK;
}

}  // namespace

static inline long long kpad(int K) { return round_up(K, 32); }   // both BK=16 and BK=32 kernels

// lo.lo (a 4th MMA per k-step) is added for short reductions, where the
// missing ~2^-22 |a b| term is not averaged out over K (measured: without it
// the worst err/bound is 3.4 at K=1 even with exact accumulation).
// ELV_TF32X3_LOLO=0/1 forces it off/on (diagnostics).
static int with_lolo(int K) {
  static int force = -2;
  if (force == -2) {
    const char* e = getenv("ELV_TF32X3_LOLO");
    force = e ? (atoi(e) != 0) : -1;
  }
  if (force >= 0) return force;
  return K < 512 ? 1 : 0;
}

static int env_int(const char* name, int dflt) {
  const char* e = getenv(name);
  return e ? atoi(e) : dflt;
}
static int one_cta_bn(int M, int N);
static int one_cta_bn_model(int M, int N, long long sms);

// Mainloop cycles per accumulation chunk (64 k fp16 / 32 k tf32: 12 MMAs of
// k16 / k8) of one CTA whose MMAs are n_mma wide and whose SMEM holds
// n_smem columns of B: max(tensor pipe, 12 x 128 n / 256 = 6 n; shared
// memory, the TMA writes of the hi/lo planes plus the three products'
// operand reads, 10 B per row or column and k (fp16; tf32 20 B over half
// the k) = 640 B per chunk at 128 B/clk = 5 (128 + n_smem)).  The MMA-rate
// probe (scripts/probes/mma_rate.cu, profiles/r2/small/mma_rate_probe.jsonl)
// measured SMEM-operand MMAs at 48 / 64 / 128 cycles for N = 64 / 128 / 256.
static double chunk_cycles(int n_mma, int n_smem) {
  const double mma = 6.0 * n_mma, smem = 5.0 * (128 + n_smem);
  return mma > smem ? mma : smem;
}

// The default kernel choice (no environment overrides) for `sms` SMs, given
// the 1-CTA kernel's N tile: pair when there is at least one 256x256 pair
// tile per SM or its modelled mainloop is shorter (see pair_mode).
static bool pair_model(int M, int N, long long sms, int bn) {
  const long long pair_tiles = (long long)((M + 255) / 256) * ((N + 255) / 256);
  if (pair_tiles >= sms) return true;
  const double pair = (double)((pair_tiles + sms / 2 - 1) / (sms / 2)) * chunk_cycles(256, 128);
  const long long tiles = (long long)((M + BM - 1) / BM) * ((N + bn - 1) / bn);
  const double one = (double)((tiles + sms - 1) / sms) * chunk_cycles(bn, bn);
  return pair < one;
}

// Kernel choice.  Default: the cta_group::2 kernel with BK=32 (128B swizzle)
// when there are at least as many 256x256 pair tiles as SMs (measured at
// 32768^2 x 8192 under the power cap: 251-256 TF vs 244-245 TF for the 1-CTA
// kernel, scripts/gpu_pairws.sh) or when its modelled mainloop is shorter
// than the 1-CTA kernel's: a pair's CTA holds half of B, so it streams
// 5 (128 + 128) SMEM cycles per 1536 MMA cycles, where a 1-CTA 128 x 256 tile
// needs 1920 (mid-size problems, e.g. 2048^3 fp16 55.3 -> 48.2 us, 3072^3
// 151.6 -> 122.9 us, bitwise the same; profiles/r2/small/mid_pair.jsonl);
// else the 1-CTA kernel (more, narrower tiles for small problems: 1024^3,
// 1536^3).  ELV_TF32X3_PAIR=0 / 16 / 32 forces a choice.
static int pair_mode(int M, int N) {
  static int forced = -2;
  if (forced == -2) {
    forced = env_int("ELV_TF32X3_PAIR", -1);
    if (forced == 1) forced = 16;
    if (forced != -1 && forced != 0 && forced != 16 && forced != 32) forced = -1;
  }
  if (forced >= 0) return forced;
  return pair_model(M, N, num_sms(), one_cta_bn(M, N)) ? 32 : 0;
}
// Wave counter (library-internal scratch, 4 bytes) zeroed on the launch
// stream before every launch; ELV_WAVE_SYNC=0 disables the sync.  One counter
// per (device, stream): launches on one stream run in order, so the zeroing
// never races a running kernel; a counter shared across streams could be
// zeroed under a concurrently running GEMM whose producers then wait for
// increments that never come.  The first launch on a stream allocates (not
// allowed under graph capture: that launch simply runs without the sync).
static unsigned int* wave_counter(int dev, cudaStream_t st) {
  static int enabled = -1;
  if (enabled < 0) enabled = env_int("ELV_WAVE_SYNC", 1) != 0;
  if (!enabled) return nullptr;
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, unsigned int*> ctrs;
  unsigned int* c = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = ctrs.find({dev, st});
    if (it != ctrs.end()) {
      c = it->second;
    } else {
      if (ctrs.size() >= 4096) return nullptr;
      cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone) {
        cudaGetLastError();
        return nullptr;
      }
      if (cudaMalloc(&c, 256) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
      }
      ctrs[{dev, st}] = c;
    }
  }
  if (cudaMemsetAsync(c, 0, sizeof(unsigned int), st) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return c;
}

// L2 residency hints in the pair kernel (ELV_L2_HINTS, default off: 1 = the
// m-group's A panels evict_last, 2 = also B evict_first), plus bit 2 for the
// serpentine k order of odd waves (ELV_SERPENTINE=1, default off; see the
// producer).  One flags word, read once per process.
static int l2_hints() {
  static int v = -2;
  if (v == -2) v = (env_int("ELV_L2_HINTS", 0) & 3) | (env_int("ELV_SERPENTINE", 0) ? 4 : 0);
  return v;
}

static int tile_group(int dflt) {
  static int v = -2;
  if (v == -2) v = env_int("ELV_TILE_GROUP", -1);
  return v > 0 ? v : dflt;
}

// ELV_TMA_STORE_C=0 selects the register-store epilogue (A/B measurements)
static bool c_store_tma() {
  static int v = -2;
  if (v == -2) v = env_int("ELV_TMA_STORE_C", 1);
  return v != 0;
}

// m-tiles per L2 raster group of the pair kernel: with L2 hints the group's A
// panels (group x 256 rows x K of hi+lo planes) stay resident -- 64 MB at
// K = 8192 for 8 fp16 / 4 tf32 m-tiles, half the 126 MB L2
template <bool F16> static int pair_group() { return (!F16 && (l2_hints() & 3)) ? 4 : 8; }

template <int BKT, bool F16 = false, int PBN = P_BN>
static int launch_pair(const void* a_hi, const void* a_lo, const void* b_hi, const void* b_lo, float* C, int M,
                       int N, int K, int Kp, int ldc, int dev, cudaStream_t st, const float* inv_s = nullptr,
                       const float* inv_t = nullptr, FixArgs* fix = nullptr) {
  using Cfg = PairCfg<BKT, F16, PBN>;
  CUtensorMap ma_hi, ma_lo, mb_hi, mb_lo;
  int rc = make_map(&ma_hi, a_hi, M, Kp, P_BM, BKT, F16);
  if (!rc) rc = make_map(&ma_lo, a_lo, M, Kp, P_BM, BKT, F16);
  if (!rc) rc = make_map(&mb_hi, b_hi, N, Kp, PBN / 2, BKT, F16);
  if (!rc) rc = make_map(&mb_lo, b_lo, N, Kp, PBN / 2, BKT, F16);
  if (rc) return rc;
  // C through TMA bulk stores when it can be described by a tensor map
  // (16 B-aligned base and pitch); otherwise the register-store epilogue
  CUtensorMap mc{};
  bool tma_c = c_store_tma() && (reinterpret_cast<uintptr_t>(C) & 15u) == 0 && (ldc & 3) == 0;
  if (tma_c) {
    EncodeTiledFn enc = get_encode();
    const cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)M};
    const cuuint64_t strides[1] = {(cuuint64_t)ldc * 4};
    const cuuint32_t box[2] = {32, 32}, estr[2] = {1, 1};
    tma_c = enc && enc(&mc, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, C, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  auto kern = tma_c ? k7_tf32x3_pair<BKT, F16, true, PBN> : k7_tf32x3_pair<BKT, F16, false, PBN>;
  static int attr_dev[2] = {-1, -1};
  if (attr_dev[tma_c] != dev) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return set_error(ELV_ECUDA, "tf32x3 pair smem attribute: %s", cudaGetErrorString(e));
    attr_dev[tma_c] = dev;
  }
  const int tiles = ((M + 255) / 256) * ((N + PBN - 1) / PBN);
  int clusters = num_sms() / 2;
  if (clusters > tiles) clusters = tiles;
  unsigned int* ctr = tiles > clusters ? wave_counter(dev, st) : nullptr;   // one wave: nothing to sync
  cudaError_t e = launch_pdl(kern, dim3(2 * clusters), dim3(P_NUM_THREADS),
                             (size_t)Cfg::SMEM_BYTES, st, ma_hi, ma_lo, mb_hi, mb_lo, mc, C, M, N, ldc, Kp / BKT,
                             F16 ? 0 : with_lolo(K), tile_group(pair_group<F16>()), ctr, inv_s, inv_t, l2_hints(),
                             fix != nullptr ? *fix : FixArgs{}, K);
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "gemm_parallel_tf32x3_pair: %s", cudaGetErrorString(e));
  if (fix != nullptr) fix->applied = 1;
  return check_launch("gemm_parallel_tf32x3_pair");
}
// K7F (the split fused into the GEMM, one launch) is bitwise the planes path
// (split prepass + pair kernel) but measured slower at every shape it applies
// to (>= 148 pair tiles: 32768^2 x 8192 138-181 TF vs 250 TF, DESIGN.md
// section 12), so variant 7 uses it only with ELV_TF32X3_FUSED=1 (read per
// call); elv_tf32x3_gemm_fused / _fused_a call it directly.
static bool fused_enabled() { return env_int("ELV_TF32X3_FUSED", 0) != 0; }
static bool fused_shape_ok(const float* A, int lda, const float* B, int ldb, int M, int N) {
  const bool al = ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B)) & 15u) == 0 &&
                  (lda & 3) == 0 && (ldb & 3) == 0;
  return al && pair_mode(M, N) == 32;
}
bool tf32x3_fused_ok(const float* A, int lda, const float* B, int ldb, int M, int N) {
  return fused_shape_ok(A, lda, B, ldb, M, N);
}
// the A-fused kernel reads only A raw (B comes as planes)
bool tf32x3_fused_a_ok(const float* A, int lda, int M, int N) {
  return (reinterpret_cast<uintptr_t>(A) & 15u) == 0 && (lda & 3) == 0 && pair_mode(M, N) == 32;
}

static int make_map_2d(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
                       uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_error(ELV_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  const cuuint64_t strides[1] = {(cuuint64_t)pitch_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer}, estr[2] = {1, 1};
  const CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box, estr,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(ELV_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ELV_OK;
}

// C = A B on raw fp32 operands (A row-major M x K, B row-major K x N) in one
// launch; flag_a[M], flag_b[N] must be zero (the caller's memset) and are
// read by the range-guard fix-up that follows.
static inline float* align128(const void* p);
// b_planes == nullptr: B is split inside the kernel (K7F, one launch);
// otherwise b_planes holds tf32x3_split_b's planes of B (the columns
// [c0, c0 + N) of b_total) and the kernel splits only A.
int tf32x3_gemm_fused(const float* A, int lda, const float* B, int ldb, float* C, int ldc, int M, int N, int K,
                      unsigned int* flag_a, unsigned int* flag_b, cudaStream_t st, const void* b_planes, int b_total,
                      int c0) {
  CUtensorMap ma, mb, mb2{}, mc{};
  const bool fuse_b = b_planes == nullptr;
  int rc = make_map_2d(&ma, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda * 4, 32, P_BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (!rc) {
    if (fuse_b) {
      rc = make_map_2d(&mb, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb * 4, 32, 32, CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
      const int Kp = (int)kpad(K);
      if (b_total <= 0) b_total = N;
      const float* b_hi = align128(b_planes) + (size_t)c0 * Kp;
      rc = make_map(&mb, b_hi, N, Kp, P_BN / 2, 32);
      if (!rc) rc = make_map(&mb2, b_hi + (size_t)b_total * Kp, N, Kp, P_BN / 2, 32);
    }
  }
  if (rc) return rc;
  bool tma_c = c_store_tma() && (reinterpret_cast<uintptr_t>(C) & 15u) == 0 && (ldc & 3) == 0;
  if (tma_c) tma_c = make_map_2d(&mc, C, (uint64_t)N, (uint64_t)M, (uint64_t)ldc * 4, 32, 32,
                                 CU_TENSOR_MAP_SWIZZLE_128B) == ELV_OK;
  if (!tma_c) cudaGetLastError();
  int dev = 0;
  cudaGetDevice(&dev);
  auto kern = tma_c ? (fuse_b ? k7f_tf32x3_fused<true, true> : k7f_tf32x3_fused<true, false>)
                    : (fuse_b ? k7f_tf32x3_fused<false, true> : k7f_tf32x3_fused<false, false>);
  const int ki = (tma_c ? 2 : 0) + (fuse_b ? 1 : 0);
  static int attr_dev[4] = {-1, -1, -1, -1};
  if (attr_dev[ki] != dev) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, F_SMEM);
    if (e != cudaSuccess) return set_error(ELV_ECUDA, "tf32x3 fused smem attribute: %s", cudaGetErrorString(e));
    attr_dev[ki] = dev;
  }
  const int tiles = ((M + 255) / 256) * ((N + P_BN - 1) / P_BN);
  int clusters = num_sms() / 2;
  if (clusters > tiles) clusters = tiles;
  unsigned int* ctr = tiles > clusters ? wave_counter(dev, st) : nullptr;
  const int num_kb = (K + 31) / 32;
  cudaError_t e = launch_pdl(kern, dim3(2 * clusters), dim3(F_NUM_THREADS), (size_t)F_SMEM, st, ma, mb, mb2, mc, C, M,
                             N, ldc, num_kb, with_lolo(K), tile_group(pair_group<false>()), ctr, flag_a, flag_b,
                             env_int("ELV_K7F_DBG", 0));
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "gemm_parallel_tf32x3_fused: %s", cudaGetErrorString(e));
  return check_launch("gemm_parallel_tf32x3_fused");
}

// tf32 plane buffers: [hi rows x Kp | lo rows x Kp] fp32 | range-guard flags (rows u32)
static inline size_t up128(size_t x) { return (x + 127) / 128 * 128; }
static inline size_t planes_bytes(int rows, int K) {
  return (size_t)(2 * (long long)rows * kpad(K)) * sizeof(float) + 128 + up128((size_t)rows * 4);
}
static inline float* align128(const void* p) {
  return reinterpret_cast<float*>((reinterpret_cast<uintptr_t>(p) + 127) & ~uintptr_t(127));
}
static inline unsigned int* planes_flags(const void* buf, int total, int K) {
  return reinterpret_cast<unsigned int*>(align128(buf) + 2 * (size_t)total * kpad(K));
}

size_t tf32x3_a_planes_bytes(int M, int K) { return planes_bytes(M, K); }
const unsigned int* tf32x3_b_planes_flags(const void* b_planes, int N, int K) { return planes_flags(b_planes, N, K); }
size_t tf32x3_b_planes_bytes(int N, int K) { return planes_bytes(N, K); }

// elv_gemm workspace for variant 7 = [A planes | B planes | flags A (M) | flags B (N)]:
// the tail keeps both operands' range-guard flags contiguous (one memset)
size_t tf32x3_workspace_bytes(int M, int N, int K) {
  return tf32x3_a_planes_bytes(M, K) + tf32x3_b_planes_bytes(N, K) + 128 + up128((size_t)(M + N) * 4);
}
static unsigned int* ws_tail_flags(void* ws, int M, int N, int K) {
  return reinterpret_cast<unsigned int*>(
      align128(static_cast<uint8_t*>(ws) + tf32x3_a_planes_bytes(M, K) + tf32x3_b_planes_bytes(N, K)));
}

bool tc_fixup_enabled() {
  static int enabled = -1;                          // ELV_TC_FIXUP=0: tuning measurements only (unguarded)
  if (enabled < 0) enabled = env_int("ELV_TC_FIXUP", 1) != 0;
  return enabled != 0;
}

// elv_gemm hands the fix-up to the 1-CTA GEMM (ELV_TC_FIXUP_INKERNEL=0, read
// per call: always the separate k_tc_fixup launch -- same bits, tested)
static bool fix_in_kernel() { return tc_fixup_enabled() && env_int("ELV_TC_FIXUP_INKERNEL", 1) != 0; }

// The fix-up after a tensor-core GEMM of a row window of A planes (flags
// flag_a[0, M)) and a column window of B planes (flag_b[0, N)); A, B are the
// fp32 operands of the same windows (B row-major, or packedB panels).
int tc_fixup(const float* A, int lda, const float* B, int ldb, bool b_packed, float* C, int ldc, int M, int N, int K,
             const unsigned int* flag_a, const unsigned int* flag_b, cudaStream_t st) {
  if (!tc_fixup_enabled()) return ELV_OK;
  const long long blocks = (long long)(M + FIX_SEG - 1) / FIX_SEG + (N + FIX_SEG - 1) / FIX_SEG;
  if (blocks <= 0) return ELV_OK;
  if (blocks > 0x7fffffffLL) return set_error(ELV_EINVAL, "tc_fixup: problem too large");
  ELV_PREFER_MAX_SMEM(k_tc_fixup);
  const cudaError_t e = launch_pdl(k_tc_fixup, dim3((unsigned)blocks), dim3(FIX_T), 0, st, A, lda, B, ldb,
                                   (int)b_packed, C, ldc, M, N, K, flag_a, flag_b);
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "tc_fixup: %s", cudaGetErrorString(e));
  return check_launch("tc_fixup");
}


static void split_a_grid(int M, int Kp, int* gx, int* gy) {
  *gx = (Kp / 4 + 255) / 256;
  int y = num_sms() * 16 / *gx;
  if (y < 1) y = 1;
  if (y > M) y = M;
  if (y > 65535) y = 65535;
  *gy = y;
}

// Plane buffers hold `total` rows (0: just these M); the split writes rows
// [r0, r0 + M) of them, so strips prepared one by one form one operand that a
// later GEMM can read across strips (the host pipeline's growing schedule).
int tf32x3_split_a(const float* A, int M, int K, int lda, void* a_planes, cudaStream_t st, int total, int r0) {
  const int Kp = (int)kpad(K);
  if (total <= 0) total = M;
  float* hi = align128(a_planes) + (size_t)r0 * Kp;
  float* lo = hi + (size_t)total * Kp;
  unsigned int* flag = planes_flags(a_planes, total, K) + r0;
  if (cudaMemsetAsync(flag, 0, (size_t)M * 4, st) != cudaSuccess) return set_error(ELV_ECUDA, "tf32x3: memset");
  int gx, gy;
  split_a_grid(M, Kp, &gx, &gy);
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15u) == 0) && (lda & 3) == 0;
  k_split_a<<<dim3(gx, gy), 256, 0, st>>>(A, hi, lo, M, K, lda, Kp, vec, flag);
  return check_launch("tf32x3_split_a");
}

int tf32x3_split_b(const float* B, int K, int N, int ldb, bool packed, void* b_planes, cudaStream_t st, int total,
                   int c0) {
  const int Kp = (int)kpad(K);
  if (total <= 0) total = N;
  float* hi = align128(b_planes) + (size_t)c0 * Kp;
  float* lo = hi + (size_t)total * Kp;
  unsigned int* flag = planes_flags(b_planes, total, K) + c0;
  if (cudaMemsetAsync(flag, 0, (size_t)N * 4, st) != cudaSuccess) return set_error(ELV_ECUDA, "tf32x3: memset");
  dim3 grid((N + 31) / 32, (Kp + 31) / 32);
  if (packed) k_split_transpose_b<true><<<grid, 256, 0, st>>>(B, hi, lo, K, N, 0, Kp, flag);
  else k_split_transpose_b<false><<<grid, 256, 0, st>>>(B, hi, lo, K, N, ldb, Kp, flag);
  return check_launch("tf32x3_split_b");
}

// N tile of the 1-CTA kernel: minimise waves x tile work / efficiency, with
// the narrow tiles' SMEM-operand-bandwidth penalty (measured-order estimate:
// 128 ~ 0.95, 64 ~ 0.67 of the 256-wide MMA rate).  ELV_TF32X3_BN forces one.
static int one_cta_bn(int M, int N) {
  static int forced = -2;
  if (forced == -2) {
    forced = env_int("ELV_TF32X3_BN", -1);
    if (forced != 64 && forced != 128 && forced != 256) forced = -1;
  }
  if (forced > 0) return forced;
  return one_cta_bn_model(M, N, num_sms());
}
static int one_cta_bn_model(int M, int N, long long sms) {
  const int bns[3] = {256, 128, 64};
  const double eff[3] = {1.0, 0.95, 0.67};
  int best = 256;
  double best_cost = 1e30;
  for (int i = 0; i < 3; ++i) {
    const long long tiles = (long long)((M + BM - 1) / BM) * ((N + bns[i] - 1) / bns[i]);
    const long long waves = (tiles + sms - 1) / sms;
    const double cost = (double)waves * bns[i] / eff[i];
    if (cost < best_cost * 0.999) { best_cost = cost; best = bns[i]; }
  }
  return best;
}

// elv_tc_kernel_choice: the default choice as data, for callers that count
// launches (interp.GemmCall.count_launches mirrors it; tests compare the two)
int tc_kernel_choice(int M, int N, int sms, int* bn) {
  const int b = one_cta_bn_model(M, N, sms);
  if (bn != nullptr) *bn = b;
  return pair_model(M, N, sms, b) ? 1 : 0;
}

template <int TBN, int TBK, bool F16 = false>
static int launch_one(const void* a_hi, const void* a_lo, const void* b_hi, const void* b_lo, float* C,
                      int M, int N, int K, int Kp, int ldc, int dev, cudaStream_t st,
                      const float* inv_s = nullptr, const float* inv_t = nullptr, FixArgs* fix = nullptr) {
  using Cfg = OneCfg<TBN, TBK, F16>;
  CUtensorMap m_ahi, m_alo, m_bhi, m_blo;
  int rc = make_map(&m_ahi, a_hi, M, Kp, BM, TBK, F16);
  if (!rc) rc = make_map(&m_alo, a_lo, M, Kp, BM, TBK, F16);
  if (!rc) rc = make_map(&m_bhi, b_hi, N, Kp, TBN, TBK, F16);
  if (!rc) rc = make_map(&m_blo, b_lo, N, Kp, TBN, TBK, F16);
  if (rc) return rc;
  static int attr_dev = -1;
  if (attr_dev != dev) {
    cudaError_t e = cudaFuncSetAttribute(k7_tf32x3<TBN, TBK, F16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return set_error(ELV_ECUDA, "tf32x3 smem attribute: %s", cudaGetErrorString(e));
    attr_dev = dev;
  }
  const int tiles = ((M + BM - 1) / BM) * ((N + TBN - 1) / TBN);
  const int grid = tiles < num_sms() ? tiles : num_sms();
  unsigned int* ctr = tiles > grid ? wave_counter(dev, st) : nullptr;
  cudaError_t e = launch_pdl(k7_tf32x3<TBN, TBK, F16>, dim3(grid), dim3(NUM_THREADS), (size_t)Cfg::SMEM, st, m_ahi,
                             m_alo, m_bhi, m_blo, C, M, N, ldc, Kp / TBK, F16 ? 0 : with_lolo(K), tile_group(16), ctr, inv_s,
                             inv_t, fix != nullptr ? *fix : FixArgs{}, K);
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "gemm_parallel_tf32x3: %s", cudaGetErrorString(e));
  if (fix != nullptr) fix->applied = 1;
  return check_launch("gemm_parallel_tf32x3");
}

// K depth of a stage: 32 (128 B rows, 128B swizzle) for the narrow tiles --
// measured 1024^3 BN=64: 26.6 us vs 30.7 us at BK=16 -- but 16 for BN=256,
// whose 96 KB BK=32 stage would leave only two stages.  ELV_TF32X3_BK forces.
static int one_cta_bk(int bn) {
  static int forced = -2;
  if (forced == -2) {
    forced = env_int("ELV_TF32X3_BK", -1);
    if (forced != 16 && forced != 32) forced = -1;
  }
  if (forced > 0) return forced;
  return bn == 256 ? 16 : 32;
}

// Small problems (pair_mode 0): the narrow CTA-pair
// kernel (PBN = 128 / 64 columns per pair) instead of the 1-CTA kernel when
// ELV_SMALL_PAIR=128 / 64 (read per call; 0 = the 1-CTA kernel)
static int small_pair_bn(int M, int N) {
  (void)M;
  (void)N;
  const int v = env_int("ELV_SMALL_PAIR", 0);
  return (v == 64 || v == 128) ? v : 0;
}

int tf32x3_gemm_planes(const void* a_planes, const void* b_planes, float* C, int M, int N, int K, int ldc,
                       cudaStream_t st, int a_total, int r0, int b_total, int c0, FixArgs* fix) {
  const int Kp = (int)kpad(K);
  if (a_total <= 0) a_total = M;
  if (b_total <= 0) b_total = N;
  const float* a_hi = align128(a_planes) + (size_t)r0 * Kp;
  const float* a_lo = a_hi + (size_t)a_total * Kp;
  const float* b_hi = align128(b_planes) + (size_t)c0 * Kp;
  const float* b_lo = b_hi + (size_t)b_total * Kp;
  int dev = 0;
  cudaGetDevice(&dev);
  const int pm = pair_mode(M, N);
  if (pm == 16) return launch_pair<16>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st);
  if (pm == 32) return launch_pair<32>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st);
  const int spb = small_pair_bn(M, N);
  if (spb == 64) return launch_pair<32, false, 64>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
  if (spb == 128)
    return launch_pair<32, false, 128>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
  const int bn = one_cta_bn(M, N);
  if (one_cta_bk(bn) == 32) {
    if (bn == 64) return launch_one<64, 32>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
    if (bn == 128)
      return launch_one<128, 32>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
    return launch_one<256, 32>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
  }
  if (bn == 64) return launch_one<64, 16>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
  if (bn == 128) return launch_one<128, 16>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
  return launch_one<256, 16>(a_hi, a_lo, b_hi, b_lo, C, M, N, K, Kp, ldc, dev, st, nullptr, nullptr, fix);
}

// elv_gemm workspace for variant 7 = [A planes | B planes]
int tf32x3_prepare(const float* A, const float* B, int M, int N, int K, int lda, int ldb, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (ws == nullptr || ws_bytes < tf32x3_workspace_bytes(M, N, K))
    return set_error(ELV_EWORKSPACE, "tf32x3: workspace too small");
  if (fused_enabled() && tf32x3_fused_ok(A, lda, B, ldb, M, N)) return ELV_OK;   // K7F splits inside the GEMM
  const int Kp = (int)kpad(K);
  float* ahi = align128(ws);
  float* alo = ahi + (size_t)M * Kp;
  float* bhi = align128(static_cast<uint8_t*>(ws) + tf32x3_a_planes_bytes(M, K));
  float* blo = bhi + (size_t)N * Kp;
  int gxa, gya;
  split_a_grid(M, Kp, &gxa, &gya);
  const int gxb = (N + 31) / 32, gyb = (Kp + 31) / 32;
  const long long blocks = (long long)gxa * gya + (long long)gxb * gyb;
  if (blocks > 0x7fffffffLL) return set_error(ELV_EINVAL, "tf32x3: problem too large for one split launch");
  const bool vec = ((reinterpret_cast<uintptr_t>(A) & 15u) == 0) && (lda & 3) == 0;
  unsigned int* flags = ws_tail_flags(ws, M, N, K);
  // flags zeroed by a kernel the split follows with PDL (it overlaps the
  // split's loads; the split waits only before setting a flag and at its end)
  int rc = zero_words(flags, (size_t)(M + N), st);
  if (rc) return rc;
  ELV_PREFER_MAX_SMEM(k_split_ab);
  const cudaError_t e = launch_pdl(k_split_ab, dim3((unsigned)blocks), dim3(256), 0, st, A, ahi, alo, M, lda, vec, gxa,
                                   gya, B, bhi, blo, N, ldb, gxb, K, Kp, flags, flags + M);
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "tf32x3_split_ab: %s", cudaGetErrorString(e));
  return check_launch("tf32x3_split_ab");
}

int tf32x3_compute(const float* A, const float* B, int lda, int ldb, float* C, int M, int N, int K, int ldc, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (ws == nullptr || ws_bytes < tf32x3_workspace_bytes(M, N, K))
    return set_error(ELV_EWORKSPACE, "tf32x3: workspace too small");
  if (fused_enabled() && tf32x3_fused_ok(A, lda, B, ldb, M, N)) {
    unsigned int* flags = ws_tail_flags(ws, M, N, K);
    if (cudaMemsetAsync(flags, 0, (size_t)(M + N) * 4, st) != cudaSuccess)
      return set_error(ELV_ECUDA, "tf32x3: memset");
    const int rc = tf32x3_gemm_fused(A, lda, B, ldb, C, ldc, M, N, K, flags, flags + M, st);
    if (rc) return rc;
    return tc_fixup(A, lda, B, ldb, false, C, ldc, M, N, K, flags, flags + M, st);
  }
  const unsigned int* flags = ws_tail_flags(ws, M, N, K);
  FixArgs fx{A, lda, B, ldb, flags, flags + M, 0};
  const int rc = tf32x3_gemm_planes(ws, static_cast<uint8_t*>(ws) + tf32x3_a_planes_bytes(M, K), C, M, N, K, ldc, st,
                                    0, 0, 0, 0, fix_in_kernel() ? &fx : nullptr);
  if (rc || fx.applied) return rc;
  return tc_fixup(A, lda, B, ldb, false, C, ldc, M, N, K, flags, flags + M, st);
}

// The fix-up of a planes-API GEMM (row window [r0, r0+M) of A planes holding
// a_total rows, column window [c0, c0+N) of B planes holding b_total)
int tc_fixup_planes(bool f16, const void* a_planes, const void* b_planes, const float* A, int lda, const float* B,
                    int ldb, bool b_packed, float* C, int ldc, int M, int N, int K, cudaStream_t st, int a_total,
                    int r0, int b_total, int c0) {
  if (a_total <= 0) a_total = M;
  if (b_total <= 0) b_total = N;
  const unsigned int* fa = (f16 ? fp16x3_planes_flags(a_planes, a_total, K) : planes_flags(a_planes, a_total, K)) + r0;
  const unsigned int* fb = (f16 ? fp16x3_planes_flags(b_planes, b_total, K) : planes_flags(b_planes, b_total, K)) + c0;
  return tc_fixup(A, lda, B, ldb, b_packed, C, ldc, M, N, K, fa, fb, st);
}

// ---------------------------------------------------------------------------
// 3xFP16 encoding (variant 8): the same three-product scheme as 3xTF32 with
// fp16 hi/lo planes -- fp16 keeps 11 significant bits like tf32, so the
// split is exact to 2^-22 -- at half the bytes per element and twice the
// tensor rate (kind::f16).  fp16's exponent range is restored by power-of-two
// scaling (Ootomo & Yokota's FP16 error correction with exponent handling):
// row i of A by s_i and column j of B by t_j so each row / column maximum
// lands in [2^14, 2^15), and lo by 2^11 so it does not underflow:
//   a s_i = hi + lo / 2^11 (+ 2^-22 |a s_i|),  hi, lo in fp16
//   C_ij = (hi.hi + 2^-11 (hi.lo + lo.hi)) / (s_i t_j)       (exact scalings)
// Elements more than 2^29 below their row / column maximum would lose
// relative precision to fp16 subnormals; the range guard (f16_out_of_window)
// marks their rows / columns for the SIMT fix-up.  The scale's exponent is
// clamped only on the low side (rows with a maximum below 2^-101 keep a
// finite 2^115 scale; their small elements are then guarded): s and 1/s stay
// normal powers of two for every finite maximum, up to 2^128.
constexpr int K16_ALIGN = 64;                     // 128 B rows of fp16 per stage
static inline long long kpad16(int K) { return round_up(K, K16_ALIGN); }

__device__ __forceinline__ void pow2_scale(float m, float* s, float* inv) {
  if (!(m > 0.f) || !isfinite(m)) { *s = 1.f; *inv = 1.f; return; }
  int e;
  frexpf(m, &e);                                  // m = f 2^e, f in [0.5, 1)
  e = max(-100, e);                               // e <= 128 for finite m
  *s = ldexpf(1.f, 15 - e);                        // m s in [2^14, 2^15)
  *inv = ldexpf(1.f, e - 15);
}

// column maxima of B (K x N row-major): a 64-row slab per block, one column
// per thread, combined with an integer atomicMax on the (non-negative) bits
constexpr int COLMAX_SLAB = 64;
// B element (k, n): row-major with ldb, or (PACKED) packedB panels
// [N/32][K][32] (elv_pack_b layout: the multi-GPU broadcast unit)
template <bool PACKED>
__device__ __forceinline__ float ld_b_elem(const float* __restrict__ B, int K, int ldb, int k, int n) {
  return PACKED ? __ldg(B + ((size_t)(n >> 5) * K + k) * 32 + (n & 31)) : __ldg(B + (size_t)k * ldb + n);
}
template <bool PACKED = false>
__device__ __forceinline__ void col_max_slab(const float* __restrict__ B, int K, int N, int ldb, int bx, int by,
                                             unsigned int* __restrict__ maxbits, unsigned int* __restrict__ flag,
                                             int slab = COLMAX_SLAB) {
  const int j = bx * 256 + threadIdx.x;
  if (j >= N) return;
  if (by == 0) flag[j] = 0u;                      // range-guard flags, set by the split-transpose that follows
  const int k0 = by * slab, k1 = min(K, k0 + slab);
  float m = 0.f;
  for (int k = k0; k < k1; ++k) m = fmaxf(m, fabsf(ld_b_elem<PACKED>(B, K, ldb, k, j)));
  griddep_wait();                                 // maxima zeroed by k_zero_u32 (PDL launch; no-op otherwise)
  atomicMax(maxbits + j, __float_as_uint(m));
}
template <bool PACKED>
__global__ void __launch_bounds__(256)
k16_col_max(const float* __restrict__ B, int K, int N, int ldb, unsigned int* __restrict__ maxbits,
            unsigned int* __restrict__ flag) {
  col_max_slab<PACKED>(B, K, N, ldb, blockIdx.x, blockIdx.y, maxbits, flag);
}

__device__ __forceinline__ void split16(float x, __half* hi, __half* lo) {
  const __half h = __float2half_rn(x);
  *hi = h;
  *lo = __float2half_rn((x - __half2float(h)) * 2048.f);
}

// A planes: [M][Kp] hi and lo, K-major (A is already K-major).  One CTA per
// row: the row is read once into registers, its maximum reduced across the
// block, then scaled and split (row scale fused with the split).
__device__ __forceinline__ void split_a_row(const float* __restrict__ A, int K, int lda, int Kp, int r,
                                            float* __restrict__ s, float* __restrict__ inv, __half* __restrict__ hi,
                                            __half* __restrict__ lo, unsigned int* __restrict__ flag) {
  __shared__ float red[8];
  const float* row = A + (size_t)r * lda;
  float m = 0.f;
  for (int k = threadIdx.x; k < K; k += 256) m = fmaxf(m, fabsf(__ldg(row + k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  m = red[0];
#pragma unroll
  for (int w = 1; w < 8; ++w) m = fmaxf(m, red[w]);
  float sc, iv;
  pow2_scale(m, &sc, &iv);
  if (threadIdx.x == 0) { s[r] = sc; inv[r] = iv; }
  __half2* h2 = reinterpret_cast<__half2*>(hi + (size_t)r * Kp);
  __half2* l2 = reinterpret_cast<__half2*>(lo + (size_t)r * Kp);
  bool bad = false;
  for (int k2 = threadIdx.x; k2 < Kp / 2; k2 += 256) {       // second read hits L1/L2
    const int k = 2 * k2;
    const float x0 = k < K ? __ldg(row + k) : 0.f, x1 = k + 1 < K ? __ldg(row + k + 1) : 0.f;
    const float y0 = x0 * sc, y1 = x1 * sc;
    bad |= f16_out_of_window(x0, y0) || f16_out_of_window(x1, y1);
    __half a0, a1, b0, b1;
    split16(y0, &a0, &b0);
    split16(y1, &a1, &b1);
    h2[k2] = __halves2half2(a0, a1);
    l2[k2] = __halves2half2(b0, b1);
  }
  bad = __syncthreads_or(bad);
  if (threadIdx.x == 0) flag[r] = bad ? 1u : 0u;
}
__global__ void __launch_bounds__(256)
k16_split_a_rows(const float* __restrict__ A, int M, int K, int lda, int Kp, float* __restrict__ s,
                 float* __restrict__ inv, __half* __restrict__ hi, __half* __restrict__ lo,
                 unsigned int* __restrict__ flag) {
  split_a_row(A, K, lda, Kp, blockIdx.x, s, inv, hi, lo, flag);
}

// Short rows (K <= K16_WARP_ROW_K): one WARP per row -- the maximum is a
// shuffle reduction with no block barrier, and a block covers 8 rows, so a
// 1024^3 prepare launches 128 A blocks instead of 1024 one-row blocks (the
// one-row blocks were latency-bound there).  Same scales and bits.
constexpr int K16_WARP_ROW_K = 2048;
__device__ __forceinline__ void split_a_row_warp(const float* __restrict__ A, int M, int K, int lda, int Kp, int r,
                                                 float* __restrict__ s, float* __restrict__ inv,
                                                 __half* __restrict__ hi, __half* __restrict__ lo,
                                                 unsigned int* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  if (r >= M) return;
  const float* row = A + (size_t)r * lda;
  float m = 0.f;
  for (int k = lane; k < K; k += 32) m = fmaxf(m, fabsf(__ldg(row + k)));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float sc, iv;
  pow2_scale(m, &sc, &iv);
  if (lane == 0) { s[r] = sc; inv[r] = iv; }
  __half2* h2 = reinterpret_cast<__half2*>(hi + (size_t)r * Kp);
  __half2* l2 = reinterpret_cast<__half2*>(lo + (size_t)r * Kp);
  bool bad = false;
  for (int k2 = lane; k2 < Kp / 2; k2 += 32) {
    const int k = 2 * k2;
    const float x0 = k < K ? __ldg(row + k) : 0.f, x1 = k + 1 < K ? __ldg(row + k + 1) : 0.f;
    const float y0 = x0 * sc, y1 = x1 * sc;
    bad |= f16_out_of_window(x0, y0) || f16_out_of_window(x1, y1);
    __half a0, a1, b0, b1;
    split16(y0, &a0, &b0);
    split16(y1, &a1, &b1);
    h2[k2] = __halves2half2(a0, a1);
    l2[k2] = __halves2half2(b0, b1);
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) flag[r] = bad ? 1u : 0u;
}

// The same warp-per-row split with the row held in registers: each lane
// loads its float4 chunks once (all loads in flight together), reduces the
// maximum and splits from registers -- no second pass over the row and no
// dependent load chain.  Needs K % 4 == 0, lda % 4 == 0 and a 16 B aligned A;
// identical scales and bits (max is order-free, the split is per element).
constexpr int K16_VEC_CHUNKS = K16_WARP_ROW_K / 128;
__device__ __forceinline__ void split_a_row_warp_vec(const float* __restrict__ A, int M, int K, int lda, int Kp,
                                                     int r, float* __restrict__ s, float* __restrict__ inv,
                                                     __half* __restrict__ hi, __half* __restrict__ lo,
                                                     unsigned int* __restrict__ flag) {
  const int lane = threadIdx.x & 31;
  if (r >= M) return;
  const float4* row = reinterpret_cast<const float4*>(A + (size_t)r * lda);
  float4 v[K16_VEC_CHUNKS];
  float m = 0.f;
#pragma unroll
  for (int c = 0; c < K16_VEC_CHUNKS; ++c) {
    const int k = c * 128 + lane * 4;
    v[c] = k < K ? __ldg(row + c * 32 + lane) : make_float4(0.f, 0.f, 0.f, 0.f);
    m = fmaxf(m, fmaxf(fmaxf(fabsf(v[c].x), fabsf(v[c].y)), fmaxf(fabsf(v[c].z), fabsf(v[c].w))));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  float sc, iv;
  pow2_scale(m, &sc, &iv);
  if (lane == 0) { s[r] = sc; inv[r] = iv; }
  bool bad = false;
#pragma unroll
  for (int c = 0; c < K16_VEC_CHUNKS; ++c) {
    const int k = c * 128 + lane * 4;
    if (k < Kp) {
      const float4 y = make_float4(v[c].x * sc, v[c].y * sc, v[c].z * sc, v[c].w * sc);
      bad |= f16_out_of_window(v[c].x, y.x) || f16_out_of_window(v[c].y, y.y) ||
             f16_out_of_window(v[c].z, y.z) || f16_out_of_window(v[c].w, y.w);
      __half h[4], l[4];
      split16(y.x, &h[0], &l[0]);
      split16(y.y, &h[1], &l[1]);
      split16(y.z, &h[2], &l[2]);
      split16(y.w, &h[3], &l[3]);
      const __half2 h01 = __halves2half2(h[0], h[1]), h23 = __halves2half2(h[2], h[3]);
      const __half2 l01 = __halves2half2(l[0], l[1]), l23 = __halves2half2(l[2], l[3]);
      *reinterpret_cast<uint2*>(hi + (size_t)r * Kp + k) =
          make_uint2(*reinterpret_cast<const unsigned int*>(&h01), *reinterpret_cast<const unsigned int*>(&h23));
      *reinterpret_cast<uint2*>(lo + (size_t)r * Kp + k) =
          make_uint2(*reinterpret_cast<const unsigned int*>(&l01), *reinterpret_cast<const unsigned int*>(&l23));
    }
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) flag[r] = bad ? 1u : 0u;
}

// elv_gemm's variant-8 prepare in one launch: blocks [0, ga) scale and split
// the rows of A (one row per block, or 8 rows per block with warp_rows), the
// rest take column-maximum slabs of B (independent work)
__global__ void __launch_bounds__(256)
k16_prep_ab(const float* __restrict__ A, int M, int K, int lda, int Kp, float* __restrict__ s,
            float* __restrict__ inv, __half* __restrict__ hi, __half* __restrict__ lo, const float* __restrict__ B,
            int N, int ldb, int gxb, unsigned int* __restrict__ maxbits, int warp_rows, int slab,
            unsigned int* __restrict__ flag_a, unsigned int* __restrict__ flag_b) {
  griddep_launch_dependents();                    // the split-transpose may stage its B tiles meanwhile
  const int b = blockIdx.x;
  const int ga = warp_rows ? (M + 7) / 8 : M;
  if (b < ga) {
    const int r = b * 8 + (threadIdx.x >> 5);
    if (warp_rows == 2) split_a_row_warp_vec(A, M, K, lda, Kp, r, s, inv, hi, lo, flag_a);
    else if (warp_rows) split_a_row_warp(A, M, K, lda, Kp, r, s, inv, hi, lo, flag_a);
    else split_a_row(A, K, lda, Kp, b, s, inv, hi, lo, flag_a);
  } else {
    col_max_slab(B, K, N, ldb, (b - ga) % gxb, (b - ga) / gxb, maxbits, flag_b, slab);
  }
}

// Short reductions (K <= K16_FUSED_PREP_K), ELV_FP16X3_FUSED_PREP=1 (read per
// call): the whole variant-8 prepare in ONE launch and no memset -- A rows as
// k16_prep_ab, and B in slabs of 16 columns x all K held in shared memory, so
// each block takes its columns' maxima and splits / transposes them without a
// grid-wide pass between.  Same scales, planes, maxima and flags as
// k16_prep_ab + k16_split_transpose_b (tested bitwise).  Not the default:
// measured slower at 1024^3 (single call 32.8 vs 29.7 us) -- the 64 slab
// blocks each stream 64 KB in and 64 KB out and set the time, while the two
// PDL-chained kernels spread the same bytes over 640 + 512 blocks.
constexpr int K16_FUSED_PREP_K = 1024;
constexpr int K16_SLAB_N = 16;
__global__ void __launch_bounds__(256)
k16_prep_fused(const float* __restrict__ A, int M, int K, int lda, int Kp, float* __restrict__ s,
               float* __restrict__ inv, __half* __restrict__ hi, __half* __restrict__ lo,
               const float* __restrict__ B, int N, int ldb, unsigned int* __restrict__ maxbits,
               float* __restrict__ inv_t, __half* __restrict__ bhi, __half* __restrict__ blo, int warp_rows,
               unsigned int* __restrict__ flag_a, unsigned int* __restrict__ flag_b, int vec_b) {
  extern __shared__ float slab[];                 // [K][K16_SLAB_N + 1]
  __shared__ float red[K16_SLAB_N][17];
  __shared__ float scale[K16_SLAB_N];
  griddep_launch_dependents();                    // the GEMM waits (griddepcontrol.wait) for our completion
  const int ga = (M + 7) / 8;
  const int b = blockIdx.x;
  if (b < ga) {
    const int r = b * 8 + (threadIdx.x >> 5);
    if (warp_rows == 2) split_a_row_warp_vec(A, M, K, lda, Kp, r, s, inv, hi, lo, flag_a);
    else split_a_row_warp(A, M, K, lda, Kp, r, s, inv, hi, lo, flag_a);
    return;
  }
  constexpr int W = K16_SLAB_N + 1;
  const int n0 = (b - ga) * K16_SLAB_N;
  const int tid = threadIdx.x;
  // stage B[0:K][n0:n0+16] (rows of 64 B: 4 threads x float4 per row when
  // aligned, every load of the slab in flight at once)
  if (vec_b && n0 + K16_SLAB_N <= N) {
    constexpr int PER = K16_FUSED_PREP_K * K16_SLAB_N / 4 / 256;       // float4 per thread (K = 1024)
    float4 v[PER];
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = tid + 256 * j, k = i >> 2, c = (i & 3) * 4;
      v[j] = k < K ? __ldg(reinterpret_cast<const float4*>(B + (size_t)k * ldb + n0 + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int j = 0; j < PER; ++j) {
      const int i = tid + 256 * j, k = i >> 2, c = (i & 3) * 4;
      if (k < K) {
        slab[k * W + c] = v[j].x; slab[k * W + c + 1] = v[j].y;
        slab[k * W + c + 2] = v[j].z; slab[k * W + c + 3] = v[j].w;
      }
    }
  } else {
#pragma unroll 8
    for (int i = tid; i < K * K16_SLAB_N; i += 256) {
      const int k = i / K16_SLAB_N, c = i % K16_SLAB_N;
      slab[k * W + c] = n0 + c < N ? __ldg(B + (size_t)k * ldb + n0 + c) : 0.f;
    }
  }
  __syncthreads();
  // column maxima: 16 threads per column
  {
    const int c = tid >> 4, part = tid & 15;
    float m = 0.f;
    for (int k = part; k < K; k += 16) m = fmaxf(m, fabsf(slab[k * W + c]));
    red[c][part] = m;
  }
  __syncthreads();
  if (tid < K16_SLAB_N) {
    float m = red[tid][0];
#pragma unroll
    for (int q = 1; q < 16; ++q) m = fmaxf(m, red[tid][q]);
    float sc, iv;
    pow2_scale(m, &sc, &iv);
    scale[tid] = sc;
    if (n0 + tid < N) {
      maxbits[n0 + tid] = __float_as_uint(m);
      inv_t[n0 + tid] = iv;
    }
  }
  __syncthreads();
  // split + transpose: warp w takes columns w and w + 8; lane j the k pairs 2j + 64 i
  const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
  for (int cc = 0; cc < 2; ++cc) {
    const int c = warp + 8 * cc, n = n0 + c;
    if (n >= N) continue;
    const float sc = scale[c];
    bool bad = false;
    __half2* h2 = reinterpret_cast<__half2*>(bhi + (size_t)n * Kp);
    __half2* l2 = reinterpret_cast<__half2*>(blo + (size_t)n * Kp);
    for (int k2 = lane; k2 < Kp / 2; k2 += 32) {
      const int k = 2 * k2;
      const float x0 = k < K ? slab[k * W + c] : 0.f, x1 = k + 1 < K ? slab[(k + 1) * W + c] : 0.f;
      const float y0 = x0 * sc, y1 = x1 * sc;
      bad |= f16_out_of_window(x0, y0) || f16_out_of_window(x1, y1);
      __half a0, a1, b0, b1;
      split16(y0, &a0, &b0);
      split16(y1, &a1, &b1);
      h2[k2] = __halves2half2(a0, a1);
      l2[k2] = __halves2half2(b0, b1);
    }
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) flag_b[n] = bad ? 1u : 0u;
  }
}

// B planes: [N][Kp] (B transposed to K-major) through 64(k) x 32(n) SMEM
// tiles: coalesced 128 B reads along B's rows, 128 B half2 writes along the
// planes' rows.  Each block turns its 32 columns' maxima (k16_col_max) into
// scales once; the blocks of the first k-tile publish 1/t_j.
template <bool PACKED>
__global__ void __launch_bounds__(256)
k16_split_transpose_b(const float* __restrict__ B, int K, int N, int ldb, int Kp,
                      const unsigned int* __restrict__ maxbits, __half* __restrict__ hi, __half* __restrict__ lo,
                      float* __restrict__ inv_t, unsigned int* __restrict__ flag) {
  __shared__ float tile[64][33];
  __shared__ float scale[32];
  griddep_launch_dependents();                    // the GEMM waits (griddepcontrol.wait) for our completion
  const int k0 = blockIdx.y * 64, n0 = blockIdx.x * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
#pragma unroll
  for (int r = 0; r < 8; ++r) {                   // B is an input: staged before the maxima are ready
    const int k = k0 + ty + 8 * r, n = n0 + tx;
    tile[ty + 8 * r][tx] = (k < K && n < N) ? ld_b_elem<PACKED>(B, K, ldb, k, n) : 0.f;
  }
  griddep_wait();                                 // column maxima from k16_prep_ab (PDL launch)
  if (ty == 0) {
    float sc = 1.f, iv = 1.f;
    if (n0 + tx < N) pow2_scale(__uint_as_float(__ldcg(maxbits + n0 + tx)), &sc, &iv);
    scale[tx] = sc;
    if (blockIdx.y == 0 && n0 + tx < N) inv_t[n0 + tx] = iv;
  }
  __syncthreads();
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const int nl = ty + 8 * r, n = n0 + nl, k = k0 + 2 * tx;
    if (n < N && k < Kp) {
      const float sc = scale[nl];
      const float x0 = tile[2 * tx][nl], x1 = tile[2 * tx + 1][nl];
      const float y0 = x0 * sc, y1 = x1 * sc;
      if (f16_out_of_window(x0, y0) || f16_out_of_window(x1, y1)) flag[n] = 1u;   // zeroed by the maxima pass
      __half a0, a1, b0, b1;
      split16(y0, &a0, &b0);
      split16(y1, &a1, &b1);
      *reinterpret_cast<__half2*>(hi + (size_t)n * Kp + k) = __halves2half2(a0, a1);
      *reinterpret_cast<__half2*>(lo + (size_t)n * Kp + k) = __halves2half2(b0, b1);
    }
  }
}

// Plane buffers of the fp16 encoding (the unit the C ABI, the row-shard
// broadcast and the host pipeline move around):
//   A planes = [hi M x Kp | lo M x Kp] fp16 | s (M f32) | 1/s (M f32) | guard flags (M u32)
//   B planes = [hi N x Kp | lo N x Kp] fp16 | t (N f32; max bits first) | 1/t (N f32) | flags (N u32)
size_t fp16x3_a_planes_bytes(int M, int K) {
  return 128 + up128((size_t)M * kpad16(K) * 2) * 2 + up128((size_t)M * 4) * 3;
}
size_t fp16x3_b_planes_bytes(int N, int K) { return fp16x3_a_planes_bytes(N, K); }
struct Planes16 {
  __half *hi, *lo;
  float* s;            // A: s_i ; B: max bits (as u32)
  float* inv;          // 1/s_i or 1/t_j
  unsigned int* flag;  // range guard
};
static Planes16 planes16(const void* buf, int rows, int K) {
  uint8_t* b = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(buf) + 127) & ~uintptr_t(127));
  const size_t plane = up128((size_t)rows * kpad16(K) * 2), vec = up128((size_t)rows * 4);
  return {reinterpret_cast<__half*>(b), reinterpret_cast<__half*>(b + plane),
          reinterpret_cast<float*>(b + 2 * plane), reinterpret_cast<float*>(b + 2 * plane + vec),
          reinterpret_cast<unsigned int*>(b + 2 * plane + 2 * vec)};
}
unsigned int* fp16x3_planes_flags(const void* buf, int total, int K) { return planes16(buf, total, K).flag; }

// rows [r0, r0 + n) of plane buffers that hold `total` rows (see tf32x3_split_a)
static Planes16 planes16_at(const void* buf, int n, int K, int total, int r0) {
  Planes16 P = planes16(buf, total > 0 ? total : n, K);
  const size_t off = (size_t)r0 * kpad16(K);
  return {P.hi + off, P.lo + off, P.s + r0, P.inv + r0, P.flag + r0};
}

int fp16x3_split_a(const float* A, int M, int K, int lda, void* a_planes, cudaStream_t st, int total, int r0) {
  const Planes16 P = planes16_at(a_planes, M, K, total, r0);
  const int Kp = (int)kpad16(K);
  k16_split_a_rows<<<M, 256, 0, st>>>(A, M, K, lda, Kp, P.s, P.inv, P.hi, P.lo, P.flag);
  return check_launch("fp16x3_split_a");
}

int fp16x3_split_b(const float* B, int K, int N, int ldb, void* b_planes, cudaStream_t st, int total, int c0,
                   bool packed) {
  const Planes16 P = planes16_at(b_planes, N, K, total, c0);
  const int Kp = (int)kpad16(K);
  unsigned int* tmax = reinterpret_cast<unsigned int*>(P.s);
  if (cudaMemsetAsync(tmax, 0, (size_t)N * 4, st) != cudaSuccess) return set_error(ELV_ECUDA, "fp16x3: memset");
  const dim3 gm((N + 255) / 256, (K + COLMAX_SLAB - 1) / COLMAX_SLAB), gs((N + 31) / 32, (Kp + 63) / 64);
  if (packed) {
    k16_col_max<true><<<gm, 256, 0, st>>>(B, K, N, 0, tmax, P.flag);
    k16_split_transpose_b<true><<<gs, 256, 0, st>>>(B, K, N, 0, Kp, tmax, P.hi, P.lo, P.inv, P.flag);
  } else {
    k16_col_max<false><<<gm, 256, 0, st>>>(B, K, N, ldb, tmax, P.flag);
    k16_split_transpose_b<false><<<gs, 256, 0, st>>>(B, K, N, ldb, Kp, tmax, P.hi, P.lo, P.inv, P.flag);
  }
  return check_launch("fp16x3_split_b");
}

int fp16x3_gemm_planes(const void* a_planes, const void* b_planes, float* C, int M, int N, int K, int ldc,
                       cudaStream_t st, int a_total, int r0, int b_total, int c0, FixArgs* fix) {
  if (!fp16x3_applicable(M, N, K))
    return set_error(ELV_EINVAL, "fp16x3: needs K >= 512 (got %dx%dx%d)", M, N, K);
  const Planes16 A = planes16_at(a_planes, M, K, a_total, r0), B = planes16_at(b_planes, N, K, b_total, c0);
  const int Kp = (int)kpad16(K);
  int dev = 0;
  cudaGetDevice(&dev);
  if (pair_mode(M, N) != 0)
    return launch_pair<64, true>(A.hi, A.lo, B.hi, B.lo, C, M, N, K, Kp, ldc, dev, st, A.inv, B.inv);
  const int spb = small_pair_bn(M, N);
  if (spb == 64) return launch_pair<64, true, 64>(A.hi, A.lo, B.hi, B.lo, C, M, N, K, Kp, ldc, dev, st, A.inv, B.inv, fix);
  if (spb == 128)
    return launch_pair<64, true, 128>(A.hi, A.lo, B.hi, B.lo, C, M, N, K, Kp, ldc, dev, st, A.inv, B.inv, fix);
  // pair_mode 0 (small problems): the 1-CTA kernel, 128 B stage rows for the
  // narrow N tiles, 64 B for N = 256 (keeps 4 stages)
  const int bn = one_cta_bn(M, N);
  if (bn == 64)
    return launch_one<64, 64, true>(A.hi, A.lo, B.hi, B.lo, C, M, N, K, Kp, ldc, dev, st, A.inv, B.inv, fix);
  if (bn == 128)
    return launch_one<128, 64, true>(A.hi, A.lo, B.hi, B.lo, C, M, N, K, Kp, ldc, dev, st, A.inv, B.inv, fix);
  return launch_one<256, 32, true>(A.hi, A.lo, B.hi, B.lo, C, M, N, K, Kp, ldc, dev, st, A.inv, B.inv, fix);
}

// The fp16 encoding has no lo.lo term (lo is pre-scaled by 2^11, so lo.lo
// would need a third accumulator scale): it serves K >= 512, where that
// term is below the bound; shorter reductions use the tf32 encoding.
bool fp16x3_applicable(int M, int N, int K) {
  (void)M;
  (void)N;
  return K >= 512;
}

// elv_gemm workspace for variant 8 = [A planes | B planes] (or variant 7's)
size_t fp16x3_workspace_bytes(int M, int N, int K) {
  return fp16x3_applicable(M, N, K) ? fp16x3_a_planes_bytes(M, K) + fp16x3_b_planes_bytes(N, K)
                                    : tf32x3_workspace_bytes(M, N, K);
}

int fp16x3_prepare(const float* A, const float* B, int M, int N, int K, int lda, int ldb, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (!fp16x3_applicable(M, N, K)) return tf32x3_prepare(A, B, M, N, K, lda, ldb, ws, ws_bytes, st);
  if (ws == nullptr || ws_bytes < fp16x3_workspace_bytes(M, N, K))
    return set_error(ELV_EWORKSPACE, "fp16x3: workspace too small");
  // memset + [A rows | B column maxima] + B split-transpose: two launches
  // (K <= K16_FUSED_PREP_K: one, k16_prep_fused)
  const Planes16 PA = planes16(ws, M, K);
  const Planes16 PB = planes16(static_cast<uint8_t*>(ws) + fp16x3_a_planes_bytes(M, K), N, K);
  const int Kp = (int)kpad16(K);
  unsigned int* tmax = reinterpret_cast<unsigned int*>(PB.s);
  const bool vec_ok0 = K % 4 == 0 && lda % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  if (K <= K16_FUSED_PREP_K && env_int("ELV_FP16X3_FUSED_PREP", 0) != 0) {
    const int warp_rows = min(env_int("ELV_FP16X3_WARP_ROWS", 2), vec_ok0 ? 2 : 1) == 2 ? 2 : 1;
    const size_t smem = (size_t)K * (K16_SLAB_N + 1) * sizeof(float);
    static int attr_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (attr_dev != dev) {
      const cudaError_t ea = cudaFuncSetAttribute(k16_prep_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                  (int)((size_t)K16_FUSED_PREP_K * (K16_SLAB_N + 1) * sizeof(float)));
      if (ea != cudaSuccess) return set_error(ELV_ECUDA, "fp16x3 prepare smem attribute: %s", cudaGetErrorString(ea));
      attr_dev = dev;
    }
    const unsigned blocks = (unsigned)((M + 7) / 8 + (N + K16_SLAB_N - 1) / K16_SLAB_N);
    k16_prep_fused<<<blocks, 256, smem, st>>>(A, M, K, lda, Kp, PA.s, PA.inv, PA.hi, PA.lo, B, N, ldb, tmax, PB.inv,
                                              PB.hi, PB.lo, warp_rows, PA.flag, PB.flag,
                                              (int)(ldb % 4 == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0));
    return check_launch("fp16x3_prepare_fused");
  }
  // the column maxima are zeroed by a kernel that k16_prep_ab follows with
  // PDL: its A rows and B slab loads overlap the zeroing, the B blocks wait
  // (griddepcontrol.wait) only before their atomicMax
  int zrc = zero_words(tmax, (size_t)N, st);
  if (zrc) return zrc;
  // Short rows: one warp per A row (2: row in registers, when float4 loads
  // are legal; 1: two scalar passes); ELV_FP16X3_WARP_ROWS caps the mode
  // (0 = one block per row).  Column-maximum slabs shrink from 64 rows
  // until the B part has >= 4 blocks per SM (1024^3: 64 -> 512 blocks of
  // 8 rows) -- with few, long slabs the dependent load chain set the time.
  const int gxb = (N + 255) / 256;
  const bool vec_ok = K % 4 == 0 && lda % 4 == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0;
  const int warp_rows = K <= K16_WARP_ROW_K ? min(env_int("ELV_FP16X3_WARP_ROWS", 2), vec_ok ? 2 : 1) : 0;
  int slab = env_int("ELV_FP16X3_COLMAX_SLAB", 0);
  if (slab <= 0) {
    slab = COLMAX_SLAB;
    while (slab > 8 && (long long)gxb * ((K + slab - 1) / slab) < 4LL * 148) slab /= 2;
  }
  const int gyb = (K + slab - 1) / slab;
  const long long ga = warp_rows ? (M + 7) / 8 : M;
  const long long blocks = ga + (long long)gxb * gyb;
  if (blocks > 0x7fffffffLL) return set_error(ELV_EINVAL, "fp16x3: problem too large for one prepare launch");
  ELV_PREFER_MAX_SMEM(k16_prep_ab);
  ELV_PREFER_MAX_SMEM(k16_split_transpose_b<false>);
  const cudaError_t ep = launch_pdl(k16_prep_ab, dim3((unsigned)blocks), dim3(256), 0, st, A, M, K, lda, Kp, PA.s,
                                    PA.inv, PA.hi, PA.lo, B, N, ldb, gxb, tmax, warp_rows, slab, PA.flag, PB.flag);
  if (ep != cudaSuccess) return set_error(ELV_ECUDA, "fp16x3_prepare: %s", cudaGetErrorString(ep));
  const cudaError_t e = launch_pdl(k16_split_transpose_b<false>, dim3((N + 31) / 32, (Kp + 63) / 64), dim3(256), 0, st, B, K,
                                   N, ldb, Kp, (const unsigned int*)tmax, PB.hi, PB.lo, PB.inv, PB.flag);
  if (e != cudaSuccess) return set_error(ELV_ECUDA, "fp16x3_prepare: %s", cudaGetErrorString(e));
  return check_launch("fp16x3_prepare");
}

int fp16x3_compute(const float* A, const float* B, int lda, int ldb, float* C, int M, int N, int K, int ldc, void* ws,
                   size_t ws_bytes, cudaStream_t st) {
  if (!fp16x3_applicable(M, N, K)) return tf32x3_compute(A, B, lda, ldb, C, M, N, K, ldc, ws, ws_bytes, st);
  if (ws == nullptr || ws_bytes < fp16x3_workspace_bytes(M, N, K))
    return set_error(ELV_EWORKSPACE, "fp16x3: workspace too small");
  void* bp = static_cast<uint8_t*>(ws) + fp16x3_a_planes_bytes(M, K);
  const unsigned int *fa = planes16(ws, M, K).flag, *fb = planes16(bp, N, K).flag;
  FixArgs fx{A, lda, B, ldb, fa, fb, 0};
  const int rc = fp16x3_gemm_planes(ws, bp, C, M, N, K, ldc, st, 0, 0, 0, 0, fix_in_kernel() ? &fx : nullptr);
  if (rc || fx.applied) return rc;
  return tc_fixup(A, lda, B, ldb, false, C, ldc, M, N, K, fa, fb, st);
}

}  // namespace elv

#ifdef ELV_K7_PROF
extern "C" int elv_debug_k7_prof(unsigned long long* host, int reset) {   // host: [512][K7_PROF_SLOTS]
  cudaMemcpyFromSymbol(host, elv::g_k7_prof, sizeof(elv::g_k7_prof));
  if (reset) {
    static unsigned long long zeros[512][elv::K7_PROF_SLOTS];
    cudaMemcpyToSymbol(elv::g_k7_prof, zeros, sizeof(zeros));
  }
  return (int)cudaGetLastError();
}
#endif
