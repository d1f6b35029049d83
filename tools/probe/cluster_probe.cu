// How many thread-block clusters of a given size fit at once for a kernel
// shaped like the persistent 2D kernel (512 threads, ~110 KB smem, 1 CTA/SM).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(512, 1) dummy(double* p) {
  extern __shared__ double sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (p) p[threadIdx.x] = sm[511 - threadIdx.x];
}
int main() {
  cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, 112 * 1024);
  cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smemkb : {64, 110}) {
    for (int cs : {1, 2, 4, 8, 12, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(cs * 8, 1, 1);
      cfg.blockDim = dim3(512, 1, 1);
      cfg.dynamicSmemBytes = smemkb * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cs;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)dummy, &cfg);
      printf("smem %3d KB cluster %2d: max active clusters %d (%d CTAs) %s\n", smemkb, cs, n,
             n * cs, cudaGetErrorString(e));
    }
  }
  return 0;
}
