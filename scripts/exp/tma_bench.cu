// Experiment: read-streaming rate of K1 phase A's structure on B200 —
// 1-D TMA (cp.async.bulk) rings fed by one loader warp, consumers that only
// release stages — against plain LDG streaming, over the same 126 MB
// (x bf16 + base f32 + fb f32 of a [4096, 3072] layer, 8 layers rotated).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../../paper_2507_17511_b200/csrc/cc_async.cuh"

using namespace cc;

struct P {
  const uint8_t *x, *b, *f;
  int64_t rows, C;
  int R, S, W;
  unsigned long long *ctr;
  int dynamic;
};

__global__ void k_tma(P p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t xb = p.R * p.C * 2, fb = p.R * p.C * 4, sb = xb + 2 * fb;
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (size_t)p.S * sb);
  uint64_t *empty = full + p.S;
  long long *tid = reinterpret_cast<long long *>(empty + p.S);
  if (threadIdx.x == 0) {
    for (int s = 0; s < p.S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], p.W);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const int64_t nT = p.rows / p.R;
  if (warp == p.W) {
    int k = 0, s = 0;
    uint32_t ph = 0;
    const uint64_t pol = l2_policy_evict_first();
    for (int64_t it = 0;; ++it) {
      if (k >= p.S) mbar_wait(&empty[s], ph ^ 1u);
      long long t;
      if (p.dynamic) {
        t = 0;
        if (lane == 0) t = (long long)atomicAdd(p.ctr, 1ull);
        t = __shfl_sync(0xffffffffu, t, 0);
      } else {
        t = blockIdx.x + it * gridDim.x;
      }
      if (t >= nT) t = -1;
      if (lane == 0) {
        tid[s] = t;
        if (t < 0) {
          mbar_arrive(&full[s]);
        } else {
          uint8_t *st = smem + (size_t)s * sb;
          mbar_expect_tx(&full[s], sb);
          bulk_g2s(st, p.x + t * xb, xb, &full[s], pol);
          bulk_g2s(st + xb, p.b + t * fb, fb, &full[s], pol);
          bulk_g2s(st + xb + fb, p.f + t * fb, fb, &full[s], pol);
        }
      }
      __syncwarp();
      if (t < 0) break;
      ++k;
      if (++s == p.S) {
        s = 0;
        ph ^= 1u;
      }
    }
  } else if (warp < p.W) {
    int s = 0;
    uint32_t ph = 0;
    for (;;) {
      mbar_wait(&full[s], ph);
      const long long t = tid[s];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (t < 0) break;
      if (++s == p.S) {
        s = 0;
        ph ^= 1u;
      }
    }
  }
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const uint4 *__restrict__ x, const uint4 *__restrict__ b,
                                             const uint4 *__restrict__ f, int64_t n16x, float *out) {
  // x has n16x 16-B vectors, b and f 2*n16x each
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * 256 * U;
  for (int64_t i0 = (int64_t)blockIdx.x * 256 * U + threadIdx.x; i0 < n16x; i0 += stride) {
    uint4 v[3 * U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * 256;
      if (i < n16x) {
        v[3 * u] = __ldcs(x + i);
        v[3 * u + 1] = __ldcs(b + 2 * i);
        v[3 * u + 2] = __ldcs(f + 2 * i + 1);
      }
    }
#pragma unroll
    for (int u = 0; u < 3 * U; ++u) acc ^= v[u].x ^ v[u].w;
    // second halves of b / f
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * 256;
      if (i < n16x) {
        v[3 * u + 1] = __ldcs(b + 2 * i + 1);
        v[3 * u + 2] = __ldcs(f + 2 * i);
      }
    }
#pragma unroll
    for (int u = 0; u < 3 * U; ++u) acc ^= v[u].y;
  }
  if (acc == 0x12345678u) out[0] = 1.f;
}

__global__ void k_fill(uint32_t *p, int64_t n, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u ^ seed;
    h ^= h >> 15; h *= 2246822519u; h ^= h >> 13; h *= 3266489917u; h ^= h >> 16;
    p[i] = h;
  }
}

int main(int argc, char **argv) {
  const bool random = argc > 1;
  const int64_t rows = 4096, C = 3072, n = rows * C;
  const int L = 8;
  uint8_t *x[L], *b[L], *f[L];
  for (int l = 0; l < L; ++l) {
    cudaMalloc(&x[l], n * 2);
    cudaMalloc(&b[l], n * 4);
    cudaMalloc(&f[l], n * 4);
    cudaMemset(x[l], 1, n * 2);
    cudaMemset(b[l], 1, n * 4);
    cudaMemset(f[l], 1, n * 4);
    if (random) {
      k_fill<<<1024, 256>>>((uint32_t *)x[l], n / 2, 11 + l);
      k_fill<<<1024, 256>>>((uint32_t *)b[l], n, 23 + l);
      k_fill<<<1024, 256>>>((uint32_t *)f[l], n, 37 + l);
    }
  }
  printf("data: %s\n", random ? "random" : "memset 0x01");
  unsigned long long *ctr;
  cudaMalloc(&ctr, 8 * 64);
  float *o;
  cudaMalloc(&o, 64);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const double bytes = n * 10.0;
  auto run = [&](const char *name, auto launch) {
    for (int i = 0; i < 2 * L; ++i) launch(i % L, i);
    cudaEventRecord(e0);
    const int reps = 4 * L;
    for (int i = 0; i < reps; ++i) launch(i % L, i);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1000 / reps;
    printf("%-44s %8.2f us  %7.1f GB/s  %s\n", name, us, bytes / us / 1e3, cudaGetErrorString(cudaGetLastError()));
  };
  char nm[96];
  // K1 phase-A look-alikes: 12 consumer warps, ~220 KB smem, cooperative launch
  for (int coop : {0, 1})
    for (int W : {4, 12})
      for (int pad : {0, 1}) {
        const int R = 2, S = 3;
        const size_t sb = (size_t)R * C * 10;
        size_t smem = S * sb + 2 * S * 8 + S * 8 + 64;
        if (pad) smem = 220 * 1024;
        snprintf(nm, 96, "tma dyn R=2 S=3 W=%d smem=%zuKB coop=%d", W, smem >> 10, coop);
        run(nm, [&](int l, int i) {
          P p{x[l], b[l], f[l], rows, C, R, S, W, ctr + (i % 32), 1};
          cudaMemsetAsync(ctr + (i % 32), 0, 8);
          if (coop) {
            void *args[] = {&p};
            cudaLaunchCooperativeKernel((const void *)k_tma, dim3(sms), dim3((W + 1) * 32), args, smem, 0);
          } else {
            k_tma<<<sms, (W + 1) * 32, smem>>>(p);
          }
        });
      }
  for (int dyn : {0, 1})
    for (int per : {1, 2})
      for (int R : {1, 2, 4})
        for (int S : {2, 3, 4, 6}) {
          const size_t sb = (size_t)R * C * 10;
          const size_t smem = S * sb + 2 * S * 8 + S * 8 + 64;
          if (smem * per > 227 * 1024) continue;
          snprintf(nm, 96, "tma %s R=%d S=%d ctas/SM=%d (%zu KB)", dyn ? "dyn" : "static", R, S, per, smem >> 10);
          run(nm, [&](int l, int i) {
            P p{x[l], b[l], f[l], rows, C, R, S, 4, ctr + (i % 32), dyn};
            if (dyn) cudaMemsetAsync(ctr + (i % 32), 0, 8);
            k_tma<<<sms * per, 5 * 32, smem>>>(p);
          });
        }
  const int64_t n16x = n * 2 / 16;
  for (int g : {1, 2, 4, 8}) {
    snprintf(nm, 96, "ldg U2 grid=%dxSM", g);
    run(nm, [&](int l, int) {
      k_ldg<2><<<sms * g, 256>>>((const uint4 *)x[l], (const uint4 *)b[l], (const uint4 *)f[l], n16x, o);
    });
    snprintf(nm, 96, "ldg U4 grid=%dxSM", g);
    run(nm, [&](int l, int) {
      k_ldg<4><<<sms * g, 256>>>((const uint4 *)x[l], (const uint4 *)b[l], (const uint4 *)f[l], n16x, o);
    });
  }
  return 0;
}
