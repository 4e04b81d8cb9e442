// FP64 vs FP32 add / FMA throughput on this GPU (independent chains, all SMs).
#include <cstdio>
#include <cuda_runtime.h>
template <typename T, bool FMA>
__global__ void k(T *out, int iters, T a, T b) {
  T x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
    if (FMA) {
      x0 = x0 * a + b; x1 = x1 * a + b; x2 = x2 * a + b; x3 = x3 * a + b;
      x4 = x4 * a + b; x5 = x5 * a + b; x6 = x6 * a + b; x7 = x7 * a + b;
    } else {
      x0 += a; x1 += a; x2 += a; x3 += a; x4 += a; x5 += a; x6 += a; x7 += a;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
template <typename T, bool FMA>
void run(const char *name) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512, iters = 4096;
  T *out;
  cudaMalloc(&out, sizeof(T) * blocks * threads);
  k<T, FMA><<<blocks, threads>>>(out, 16, (T)1.0000001, (T)0.5);
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  k<T, FMA><<<blocks, threads>>>(out, iters, (T)1.0000001, (T)0.5);
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  const double ops = (double)blocks * threads * iters * 8;
  printf("%-10s %8.3f ms  %9.1f Gop/s  %6.1f op/clk/SM (at 1.965 GHz)\n", name, ms, ops / ms / 1e6,
         ops / (ms * 1e-3) / sms / 1.965e9);
  cudaFree(out);
}
int main() {
  run<float, false>("FADD");
  run<float, true>("FFMA");
  run<double, false>("DADD");
  run<double, true>("DFMA");
  return 0;
}
