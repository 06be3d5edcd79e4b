// TMEM read-throughput probe (tuning evidence, not product code).
// One CTA per SM allocates 512 TMEM columns; W warps (W % 4 == 0, warp w reads
// lane group w % 4) repeatedly tcgen05.ld 32x32b.x32 chunks of their columns
// and accumulate them with FADD (as a chunked-flush epilogue would).  Prints
// bytes per SM-clock.  Also assembles tcgen05.mma ... scale-input-d.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
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
}

template <int W, int COLS_PER_WARP>
__global__ void __launch_bounds__(W * 32, 1) k_tmem_bw(int iters, float* out, unsigned long long* cyc) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = holder;
  const int g = warp & 3;
  const int col0 = (warp >> 2) * COLS_PER_WARP;
  float acc[COLS_PER_WARP];
#pragma unroll
  for (int i = 0; i < COLS_PER_WARP; ++i) acc[i] = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < COLS_PER_WARP / 32; ++c) {
      uint32_t r[32];
      tmem_ld32(base + ((uint32_t)(g * 32) << 16) + (uint32_t)(col0 + c * 32), r);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
      for (int q = 0; q < 32; ++q) acc[c * 32 + q] += __uint_as_float(r[q]);
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < COLS_PER_WARP; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = (unsigned long long)(t1 - t0);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

// scale-input-d assembles for the pair MMA (never launched)
__global__ void k_scale_d_asm(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, int acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p, 11;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p, 11;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}

template <int W, int CPW>
void run(int sms) {
  const int iters = 2000;
  float* out; unsigned long long* cyc;
  cudaMalloc(&out, sms * W * 32 * 4);
  cudaMalloc(&cyc, sms * 8);
  k_tmem_bw<W, CPW><<<sms, W * 32>>>(10, out, cyc);
  k_tmem_bw<W, CPW><<<sms, W * 32>>>(iters, out, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[256];
  cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (int i = 0; i < sms; ++i) mean += h[i];
  mean /= sms;
  const double bytes = (double)iters * W * 32 * CPW * 4;   // per CTA
  printf("{\"probe\": \"tmem_ld_bw\", \"warps\": %d, \"cols_per_warp\": %d, \"err\": \"%s\", \"cycles\": %.0f, "
         "\"bytes_per_clk_per_sm\": %.1f}\n", W, CPW, cudaGetErrorString(e), mean, bytes / mean);
  cudaFree(out); cudaFree(cyc);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<4, 128>(sms);
  run<8, 64>(sms);
  run<8, 128>(sms);
  run<16, 64>(sms);
  run<16, 32>(sms);
  return 0;
}
