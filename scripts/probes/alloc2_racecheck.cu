// Probe (tooling evidence, not product code): does compute-sanitizer
// racecheck report a hazard on the minimal, documented TMEM allocation
// pattern for a CTA pair -- one warp per CTA runs tcgen05.alloc.cta_group::2
// into a shared word, tcgen05.fence::before_thread_sync, bar.sync, cluster
// barrier, tcgen05.fence::after_thread_sync, every thread reads the word
// (the pattern of /opt/skills/guides/blackwell_cuda_programming.md and of
// k7_tf32x3_pair)?  Mode 1 is the same with cta_group::1 (no cluster).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -o alloc2_racecheck alloc2_racecheck.cu
// Run:   compute-sanitizer --tool racecheck ./alloc2_racecheck 2   (and 1)
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_pair(unsigned* out) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = holder;
  out[blockIdx.x * blockDim.x + threadIdx.x] = base;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(base));
  }
}

__global__ void __launch_bounds__(128, 1) k_one(unsigned* out) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x >> 5;
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(sa(&holder)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t base = holder;
  out[blockIdx.x * blockDim.x + threadIdx.x] = base;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
  }
}

int main(int argc, char** argv) {
  const int mode = argc > 1 ? atoi(argv[1]) : 2;
  unsigned* d;
  cudaMalloc(&d, 8 * 128 * sizeof(unsigned));
  if (mode == 2) k_pair<<<8, 128>>>(d);
  else k_one<<<8, 128>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned h[8 * 128];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  unsigned mx = 0;
  for (int i = 0; i < 8 * 128; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("{\"mode\": \"cta_group::%d\", \"cuda\": \"%s\", \"max_tmem_base\": %u}\n", mode, cudaGetErrorString(e), mx);
  return 0;
}
