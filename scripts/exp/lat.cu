// Dependent-chain latencies (cycles) of a few instructions on this GPU, one warp.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double *out, long long *cyc, int n, double a, double b) {
  double x = threadIdx.x * 1e-3 + 1.0;
  float f = (float)x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) f = fmaf(f, (float)a, (float)b);
  long long t2 = clock64();
  double y = x;
  for (int i = 0; i < n; ++i) y = rsqrt(y + 2.0);
  long long t3 = clock64();
  double z = x;
  for (int i = 0; i < n; ++i) z = __shfl_sync(0xffffffffu, z, (threadIdx.x + 1) & 31) + 1.0;
  long long t4 = clock64();
  double d0 = x, d1 = y;
  for (int i = 0; i < n; ++i)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
  long long t5 = clock64();
  double q = x;
  for (int i = 0; i < n; ++i) q = 1.0 / (q + 3.0);
  long long t6 = clock64();
  out[threadIdx.x] = x + f + y + z + d0 + d1 + q;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
}
int main() {
  double *o; long long *c, h[6];
  cudaMalloc(&o, 32 * 8); cudaMalloc(&c, 6 * 8);
  const int n = 1000;
  k<<<1, 32>>>(o, c, n, 0.999, 1e-3);
  k<<<1, 32>>>(o, c, n, 0.999, 1e-3);
  cudaMemcpy(h, c, 48, cudaMemcpyDeviceToHost);
  const char *nm[6] = {"DFMA", "FFMA", "rsqrt(f64)+DADD", "SHFL(f64)+DADD", "DMMA m8n8k4", "f64 div+DADD"};
  for (int i = 0; i < 6; ++i) printf("%-18s %7.1f cycles per dependent op\n", nm[i], (double)h[i] / n);
  return 0;
}
