// How many CTAs of an (one-CTA-per-SM, ~200 KB SMEM) kernel can be resident
// at once for cluster sizes 1, 2, 4, 8 on this GPU: the GPC topology decides
// whether a 4-CTA cluster (TMA multicast of an operand between two CTA pairs)
// can still cover all SMs.   nvcc -arch=sm_100a -o /tmp/cluster_occ scripts/cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (p) p[0] = s[threadIdx.x]; }
int main() {
  int dev = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  printf("{\"sms\": %d, \"clusters\": [", sms);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64); cfg.blockDim = dim3(320); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a; a.id = cudaLaunchAttributeClusterDimension;
    a.val.clusterDim.x = cs; a.val.clusterDim.y = 1; a.val.clusterDim.z = 1;
    cfg.attrs = &a; cfg.numAttrs = 1;
    int n = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("%s{\"size\": %d, \"max_active_clusters\": %d, \"resident_ctas\": %d, \"err\": \"%s\"}",
           cs == 1 ? "" : ", ", cs, n, n * cs, cudaGetErrorString(e));
  }
  printf("]}\n");
}
