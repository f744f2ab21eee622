// Max co-resident clusters of a 512-thread CTA with the fused sparse kernel's
// shared memory, per cluster size (decides whether 16-CTA clusters fit one wave).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) dummy() {
  extern __shared__ char sm[];
  sm[threadIdx.x] = 0;
}
int main() {
  for (int smem : {199264, 225888, 227424, 110000}) {
    cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cs : {4, 6, 7, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs, 8);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
      printf("smem %d cluster %d: max active clusters %d (%s)\n", smem, cs, n, cudaGetErrorString(e));
    }
  }
  return 0;
}
