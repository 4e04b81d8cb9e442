// Throughput of the f32 -> f64 conversion (F2F.F64.F32) and of DMMA m8n8k4 (independent
// chains, all SMs): sizes the f64 projection kernels of the fused low-rank step.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_cvt(double *out, int iters, float a) {
  float f[8];
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    f[u] = threadIdx.x + u;
    acc[u] = 0.0;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[u] += (double)f[u];  // F2F + DADD
      f[u] = __fadd_rn(f[u], a);
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += acc[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_add_only(double *out, int iters, float a) {  // same loop without the conversion
  float f[8];
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    f[u] = threadIdx.x + u;
    acc[u] = 0.0;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      acc[u] += 1.0000001;
      f[u] = __fadd_rn(f[u], a);
    }
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += acc[u] + f[u];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k_dmma(double *out, int iters) {
  double d[8][2];
  const double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
#pragma unroll
  for (int u = 0; u < 8; ++u) d[u][0] = d[u][1] = 0.0;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) dmma884(d[u][0], d[u][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s += d[u][0] + d[u][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
float timeit(F f) {
  f();
  cudaEvent_t s, e;
  cudaEventCreate(&s);
  cudaEventCreate(&e);
  cudaEventRecord(s);
  f();
  cudaEventRecord(e);
  cudaEventSynchronize(e);
  float ms;
  cudaEventElapsedTime(&ms, s, e);
  return ms;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms * 4, threads = 512, iters = 4096;
  double *out;
  cudaMalloc(&out, sizeof(double) * blocks * threads);
  const double n = (double)blocks * threads * iters * 8;
  const double clk = sms * 1.965e9;
  float ms = timeit([&] { k_cvt<<<blocks, threads>>>(out, iters, 1.0f); });
  printf("F2F.F64.F32+DADD+FADD  %8.3f ms  %6.1f cvt/clk/SM\n", ms, n / (ms * 1e-3) / clk);
  ms = timeit([&] { k_add_only<<<blocks, threads>>>(out, iters, 1.0f); });
  printf("DADD+FADD (no cvt)     %8.3f ms  %6.1f op/clk/SM\n", ms, n / (ms * 1e-3) / clk);
  ms = timeit([&] { k_dmma<<<blocks, threads>>>(out, iters); });
  const double dm = n / 32 / (ms * 1e-3) / clk;  // warp-level DMMAs per clk per SM
  printf("DMMA m8n8k4            %8.3f ms  %6.1f FMA/clk/SM (%.2f clk per DMMA per SMSP)\n", ms, dm * 256, 4 / dm);
  cudaFree(out);
  return 0;
}
