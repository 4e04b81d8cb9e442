// Grid-barrier latency of a cooperative cluster launch (33 clusters x 4 CTAs x 512
// threads, ~215 KB shared memory: the fused low-rank step's geometry): flat (every CTA
// arrives on one counter) vs hierarchical (cluster barrier, one arrival per cluster).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int MODE>
__global__ void __launch_bounds__(512, 1) k(unsigned *ctl, int iters, int ncl, int sleep_ns) {
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double sm[];
  const int q = cluster.block_rank();
  const unsigned G = gridDim.x;
  for (int i = 1; i <= iters; ++i) {
    if (MODE == 0) {  // flat
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctl, 1u);
        while (ld_acquire(ctl) < i * G) if (sleep_ns) __nanosleep(sleep_ns);
        __threadfence();
      }
      __syncthreads();
    } else if (MODE == 1) {  // hierarchical
      cluster.sync();
      if (q == 0 && threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctl, 1u);
        while (ld_acquire(ctl) < (unsigned)(i * ncl)) if (sleep_ns) __nanosleep(sleep_ns);
        __threadfence();
      }
      cluster.sync();
    } else {  // hierarchical, red.release arrival + acquire poll without fences
      cluster.sync();
      if (q == 0 && threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctl) : "memory");
        while (ld_acquire(ctl) < (unsigned)(i * ncl)) if (sleep_ns) __nanosleep(sleep_ns);
      }
      cluster.sync();
    }
  }
  if (sm[threadIdx.x] == 12345.0) ctl[1] = 1;
}
int main() {
  const int ncl = 33, smem = 215 * 1024, iters = 1000;
  unsigned *ctl;
  cudaMalloc(&ctl, 256);
  void *kerns[3] = {(void *)k<0>, (void *)k<1>, (void *)k<2>};
  const char *names[3] = {"flat (132 arrivals)", "hierarchical (33 arrivals)", "hierarchical, red.release"};
  for (int m = 0; m < 3; ++m) {
    cudaFuncSetAttribute(kerns[m], cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int sl : {0, 16, 64}) {
      cudaMemset(ctl, 0, 256);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(ncl * 4);
      cfg.blockDim = dim3(512);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[2];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 4; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      at[1].id = cudaLaunchAttributeCooperative;
      at[1].val.cooperative = 1;
      cfg.attrs = at;
      cfg.numAttrs = 2;
      int it = iters;
      int nc = ncl;
      void *args[] = {&ctl, &it, &nc, &sl};
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      cudaError_t e = cudaLaunchKernelExC(&cfg, kerns[m], args);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("%-30s sleep %2d ns: %.3f us per barrier (%s)\n", names[m], sl, ms * 1000 / iters, cudaGetErrorString(e));
    }
  }
  return 0;
}
