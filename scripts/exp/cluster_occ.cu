// Max co-resident clusters (1 CTA per SM: ~200 KB dynamic shared memory) per cluster size.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(float *o) { extern __shared__ float s[]; s[threadIdx.x] = 1.f; __syncthreads(); if (o) o[0] = s[5]; }
int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(512);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, n, n * cs, cudaGetErrorString(e));
  }
  // cooperative + cluster launch accepted?
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(8 * 16); cfg.blockDim = dim3(512); cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 8; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative; at[1].val.cooperative = 1;
  cfg.attrs = at; cfg.numAttrs = 2;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, (float *)nullptr);
  cudaError_t e2 = cudaDeviceSynchronize();
  printf("cooperative + cluster 8 x 16: %s / %s\n", cudaGetErrorString(e), cudaGetErrorString(e2));
  for (int ncl : {17, 18}) {
    cfg.gridDim = dim3(8 * ncl);
    e = cudaLaunchKernelEx(&cfg, k, (float *)nullptr);
    e2 = cudaDeviceSynchronize();
    printf("cooperative + cluster 8 x %d: %s / %s\n", ncl, cudaGetErrorString(e), cudaGetErrorString(e2));
    cudaGetLastError();
  }
  return 0;
}
