// How many thread-block clusters of C CTAs (one CTA per SM: ~200 KB dynamic
// SMEM) fit on the GPU at once, C = 1..16 -- the GPC structure as the
// cluster scheduler sees it.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* p) { extern __shared__ int s[]; if (threadIdx.x == 0 && p) p[blockIdx.x] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int C = 1; C <= 16; ++C) {
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = C; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    lc.gridDim = dim3(C); lc.blockDim = dim3(256); lc.dynamicSmemBytes = 200 * 1024; lc.attrs = a; lc.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &lc);
    printf("C=%2d max_active_clusters=%3d SMs=%3d %s\n", C, n, n * C, e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  return 0;
}
