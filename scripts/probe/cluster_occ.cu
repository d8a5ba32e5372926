// Probe: how many clusters of size Q (1 CTA/SM, ~200 KB smem, 416 threads) are co-resident on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  extern __shared__ int s[];
  s[threadIdx.x] = threadIdx.x;
  if (threadIdx.x == 0 && out) out[blockIdx.x] = s[0];
}
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int q : {1, 2, 4, 8, 12, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(q * 8);
    cfg.blockDim = dim3(416);
    cfg.dynamicSmemBytes = 200 * 1024;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = q; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d CTAs (%s)\n", q, n, n * q, cudaGetErrorString(e));
  }
  return 0;
}
