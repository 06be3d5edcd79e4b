// Probe (tuning evidence, not product code): what does kind::tf32 tcgen05.mma
// do with raw fp32 operands (truncate / round the low 13 mantissa bits?), and
// is an MN-major, 128B-swizzled B operand -- B[k][n] row-major loaded by TMA
// in {32 n, 32 k} boxes -- described by LBO = 4096 B (next 32-n block),
// SBO = 1024 B (next 8-k group)?  One CTA, M = N = 128, K = 32 (4 MMAs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -o tf32_mn_probe tf32_mn_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(128, 1) k_probe(const __grid_constant__ CUtensorMap ma,
                                                  const __grid_constant__ CUtensorMap mb, float* D,
                                                  uint32_t lbo, uint32_t sbo, uint32_t bmaj) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = sm;               // 128 rows x 128 B (K-major, SW128)
  uint8_t* sB = sm + 16384;       // 4 boxes of 32 k x 128 B (MN-major, SW128)
  __shared__ uint64_t bar, done;
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(sa(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = holder;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(32768) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            sa(sA)), "l"((uint64_t)&ma), "r"(sa(&bar)), "r"(0), "r"(0) : "memory");
    for (int j = 0; j < (bmaj ? 4 : 1); ++j)
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
              sa(sB + j * 4096)), "l"((uint64_t)&mb), "r"(sa(&bar)), "r"(32 * j), "r"(0) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(
                     sa(&bar)) : "memory");
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (0) printf("tmem %u sA %u sB %u A[0..1] %g %g B[0] %g\n", tmem, sa(sA), sa(sB), ((float*)sA)[0], ((float*)sA)[1], ((float*)sB)[0]);
    // D f32, A tf32 K-major, B tf32 MN-major, N = 128, M = 128
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (bmaj << 16) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
    for (int ks = 0; ks < 4; ++ks) {
      const uint64_t ad = desc(sa(sA) + ks * 32, 16, 1024);
      const uint64_t bd = bmaj ? desc(sa(sB) + ks * 1024, lbo, sbo) : desc(sa(sB) + ks * 32, 16, 1024);
      asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(
                       tmem), "l"(ad), "l"(bd), "r"(idesc), "r"((uint32_t)(ks > 0)) : "memory");
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(sa(&done)) : "memory");
  }
  __syncwarp();
  asm volatile("{\n.reg .pred p;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W2;\n}\n" ::"r"(
                   sa(&done)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int row = warp * 32 + lane;
  if (threadIdx.x == 0) if (0) printf("done waited\n");
  for (int c = 0; c < 128; ++c) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem + ((uint32_t)(warp * 32) << 16) + c));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    D[row * 128 + c] = __uint_as_float(v);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

static float trunc_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }
static float rna_tf32(float x) { uint32_t u; memcpy(&u, &x, 4); u += 0x1000u; u &= 0xffffe000u; memcpy(&x, &u, 4); return x; }
static float rne_tf32(float x) {
  uint32_t u; memcpy(&u, &x, 4); u += 0xfffu + ((u >> 13) & 1u); u &= 0xffffe000u; memcpy(&x, &u, 4); return x;
}

int main() {
  void* fp = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fp;
  const int M = 128, N = 128, K = 32;
  float *hA = new float[M * K], *hB = new float[K * N], *hD = new float[M * N];
  float *dA, *dB, *dD, *dBt;
  float* hBt = new float[K * N];
  cudaMalloc(&dA, M * K * 4); cudaMalloc(&dB, K * N * 4); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dBt, K * N * 4);
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (float)rand() / RAND_MAX * 2.f - 1.f;
  CUtensorMap ma, mb, mbt;
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)N}, str[1] = {(cuuint64_t)K * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    enc(&mbt, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dBt, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)M}, str[1] = {(cuuint64_t)K * 4};
    cuuint32_t box[2] = {32, 128}, es[2] = {1, 1};
    int r = enc(&ma, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dA, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc A %d\n", r);
  }
  {
    cuuint64_t dims[2] = {(cuuint64_t)N, (cuuint64_t)K}, str[1] = {(cuuint64_t)N * 4};
    cuuint32_t box[2] = {32, 32}, es[2] = {1, 1};
    int r = enc(&mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("enc B %d\n", r);
  }
  printf("attr %d\n", (int)cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40 * 1024));
  const uint32_t lbos[8] = {4096, 1024, 1024, 4096, 128, 128, 16, 8192}, sbos[8] = {1024, 4096, 1024, 4096, 1024, 4096, 1024, 1024};
  for (int test = 0; test < 2; ++test) {
    // test 0: B[k][n] = (k == n % 32) -> D[m][n] = hw_tf32(A[m][n % 32]) exactly
    // test 1: random B -> compare with f64 products of trunc / rna / rne operands
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n)
        hB[k * N + n] = test == 0 ? (k == n % 32 ? 1.f : 0.f) : (float)rand() / RAND_MAX * 2.f - 1.f;
    cudaMemcpy(dA, hA, M * K * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, K * N * 4, cudaMemcpyHostToDevice);
    for (int k = 0; k < K; ++k) for (int n = 0; n < N; ++n) hBt[n * K + k] = hB[k * N + n];
    cudaMemcpy(dBt, hBt, K * N * 4, cudaMemcpyHostToDevice);
    for (int v = 0; v < 8; ++v) {
      cudaMemset(dD, 0, M * N * 4);
      k_probe<<<1, 128, 40 * 1024>>>(ma, mb, dD, lbos[v], sbos[v], 1u);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaDeviceSynchronize();
      cudaMemcpy(hD, dD, M * N * 4, cudaMemcpyDeviceToHost);
      double err[4] = {0, 0, 0, 0};  // raw fp32, trunc, rna, rne models
      int nz = 0;
      for (int i = 0; i < M * N; ++i) nz += hD[i] != 0.f;
      for (int m = 0; m < M; ++m)
        for (int n = 0; n < N; ++n) {
          double s[4] = {0, 0, 0, 0};
          for (int k = 0; k < K; ++k) {
            const float a = hA[m * K + k], b = hB[k * N + n];
            s[0] += (double)a * b;
            s[1] += (double)trunc_tf32(a) * trunc_tf32(b);
            s[2] += (double)rna_tf32(a) * rna_tf32(b);
            s[3] += (double)rne_tf32(a) * rne_tf32(b);
          }
          for (int i = 0; i < 4; ++i) err[i] = fmax(err[i], fabs(hD[m * N + n] - s[i]));
        }
      printf("{\"test\": \"%s\", \"b\": \"%s\", \"lbo\": %u, \"sbo\": %u, \"cuda\": \"%s\", \"max_abs_err\": {\"raw\": %.3g, \"trunc\": %.3g, "
             "\"rna\": %.3g, \"rne\": %.3g}, \"D00\": %.9g, \"D01\": %.9g, \"D0_32\": %.9g, \"nz\": %d, \"A00\": %.9g}\n",
             test == 0 ? "identity_B" : "random_B", "MN-major B", lbos[v], sbos[v], cudaGetErrorString(e), err[0], err[1], err[2],
             err[3], hD[0], hD[1], hD[32], nz, hA[0]);
    }
  }
  return 0;
}
