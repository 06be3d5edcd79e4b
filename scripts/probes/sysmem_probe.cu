// PCIe probe: SM-initiated stores into pinned host memory (zero-copy) vs the
// copy engines, alone and under a concurrent H2D copy.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_fill_host(float4* __restrict__ dst, size_t n4, float v) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    dst[i] = make_float4(v, v, v, v);
}

extern "C" int probe_fill_host(void* host_ptr, size_t bytes, int blocks, void* stream) {
  void* dptr = nullptr;
  if (cudaHostGetDevicePointer(&dptr, host_ptr, 0) != cudaSuccess) return -1;
  k_fill_host<<<blocks, 256, 0, (cudaStream_t)stream>>>((float4*)dptr, bytes / 16, 1.0f);
  return (int)cudaGetLastError();
}
