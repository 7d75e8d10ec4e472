// How many clusters of size 2/4/8 (one 196 KB CTA per SM) can be co-resident:
// multicast across CTA pairs only pays if no SM is left idle.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int *x) { extern __shared__ int s[]; if (x) x[0] = s[0]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 199680);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int c : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * 64); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = 199680;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension;
    a[0].val.clusterDim.x = c; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d -> %d SMs of %d (%s)\n", c, n, n * c, sms, cudaGetErrorString(e));
  }
  return 0;
}
