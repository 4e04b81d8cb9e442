// Device helpers shared by the low-rank kernels (lowrank.cu, lr_step.cu): the f64
// tensor-pipe MMA, the register Cholesky / R^-1 of an r x r Gram, and the single-CTA
// CGS2 with random replacement columns (the rank-deficient fallback, la:77-112).
#pragma once
#include "cc_common.cuh"

#include <curand_kernel.h>

namespace cc {
namespace lr {

constexpr double kDegenerate = 1e-12;  // la:13
constexpr int kMaxRank = 32;

__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// one warp, registers: G = R^T R (lane c holds column c of G / R) by RP compile-time
// pivot steps with one rsqrt each (no division chain), then R^-1 by back
// substitution with the reciprocal diagonal.  Rm / Ri in shared memory for the apply.
template <int RP, int LD>
__device__ __forceinline__ void chol_rinv_regs(const double (*G)[LD], double (*Rm)[LD], double (*Ri)[LD], int r,
                                               int *bad) {
  const int c = threadIdx.x & 31;
  double g[RP];
#pragma unroll
  for (int a = 0; a < RP; ++a) g[a] = (c < r && a < r) ? G[a][c] : 0.0;
  double invd[RP];
#pragma unroll
  for (int j = 0; j < RP; ++j) {
    if (j >= r) break;
    double piv = __shfl_sync(0xffffffffu, g[j], j);  // G[j][j] (Schur complement) from lane j
    if (!(piv >= kDegenerate)) {
      if (c == 0) *bad = 1;
      piv = 1.0;
    }
    const double inv = rsqrt(piv);
    invd[j] = inv;
    const double rjc = c == j ? piv * inv : (c > j && c < r ? g[j] * inv : 0.0);  // R[j][c]
    if (c < r) Rm[j][c] = rjc;
#pragma unroll
    for (int a = j + 1; a < RP; ++a) {
      const double rja = __shfl_sync(0xffffffffu, rjc, a);  // R[j][a]
      if (a < r && c >= a && c < r) g[a] -= rja * rjc;
    }
  }
  __syncwarp();
  if (c < r) {  // column c of R^-1: x[i] = (delta_ic - sum_{k>i} R[i][k] x[k]) / R[i][i]
    double x[RP];
#pragma unroll
    for (int i = RP - 1; i >= 0; --i) {
      double sacc = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = i + 1; k < RP; ++k)
        if (k <= c) sacc -= Rm[i][k] * x[k];
      x[i] = (i > c || i >= r) ? 0.0 : sacc * invd[i];
    }
#pragma unroll
    for (int i = 0; i < RP; ++i) Ri[i][c] = x[i];
  }
}

// r = 8: every lane of the warp factors the WHOLE 8x8 Gram in registers (the same
// arithmetic in every lane, no shuffles, no shared-memory round trips in the
// pivot chain); lane c < 8 then back-substitutes column c of R^-1.  The pivot
// chain is 8 x (rsqrt + one multiply + an independent rank-1 update).
__device__ __forceinline__ void chol8_regs(const double (*G)[17], double (*Rm)[17], double (*Ri)[17], int *bad) {
  const int c = threadIdx.x & 31;
  double g[8][8];
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = a; b < 8; ++b) g[a][b] = G[a][b];
  double invd[8];
  bool degenerate = false;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    double piv = g[j][j];
    if (!(piv >= kDegenerate)) {
      degenerate = true;
      piv = 1.0;
    }
    const double inv = rsqrt(piv);
    invd[j] = inv;
    g[j][j] = piv * inv;  // R[j][j]
#pragma unroll
    for (int b = j + 1; b < 8; ++b) g[j][b] *= inv;  // R[j][b]
#pragma unroll
    for (int a = j + 1; a < 8; ++a)
#pragma unroll
      for (int b = a; b < 8; ++b) g[a][b] -= g[j][a] * g[j][b];
  }
  if (degenerate && c == 0) *bad = 1;
  if (c < 8) {
#pragma unroll
    for (int a = 0; a < 8; ++a)  // row a of R by lane a (compile-time indices: g stays in registers)
      if (a == c)
#pragma unroll
        for (int b = 0; b < 8; ++b) Rm[a][b] = b >= a ? g[a][b] : 0.0;
    double x[8];  // column c of R^-1
#pragma unroll
    for (int i = 7; i >= 0; --i) {
      double sacc = (i == c) ? 1.0 : 0.0;
#pragma unroll
      for (int k = i + 1; k < 8; ++k)
        if (k <= c) sacc -= g[i][k] * x[k];
      x[i] = i > c ? 0.0 : sacc * invd[i];
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) Ri[i][c] = x[i];
  }
}

// INT4 factor code / value (cx:556-572): per-column symmetric 16 levels, np.rint half-even
__device__ __forceinline__ uint32_t int4_code(float f, float range) {
  if (!(range > 0.0f)) return 0u;  // zero column: code 0 (cx:561-562)
  const double rg = (double)range;
  const double step = 2.0 * rg / 15.0;
  double c = rint(((double)f + rg) / step);  // half-even like np.rint
  c = c < 0.0 ? 0.0 : (c > 15.0 ? 15.0 : c);
  return (uint32_t)c;
}
__device__ __forceinline__ double int4_value(uint32_t code, float range) {
  return -(double)range + (double)code * (2.0 * (double)range / 15.0);  // cx:569-572, as factor_at
}

static __device__ __noinline__ void cgs2_block(const float *__restrict__ orig, double *__restrict__ M, float *__restrict__ out,
                           int64_t m, int r, unsigned long long seed, double *red, double *coef) {
  auto block_sum = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
    __syncthreads();
    return s;
  };
  curandStatePhilox4_32_10_t rng;
  curand_init(seed, threadIdx.x, 0, &rng);
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) M[e] = (double)orig[e];
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    for (int attempt = 0;; ++attempt) {
      for (int pass = 0; pass < 2; ++pass) {
        for (int k = 0; k < j; ++k) {
          double part = 0.0;
          for (int64_t i = threadIdx.x; i < m; i += blockDim.x) part += M[i * r + k] * M[i * r + j];
          const double s = block_sum(part);
          if (threadIdx.x == 0) coef[k] = s;
        }
        __syncthreads();
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) {
          double v = M[i * r + j];
          for (int k = 0; k < j; ++k) v -= M[i * r + k] * coef[k];
          M[i * r + j] = v;
        }
        __syncthreads();
      }
      double part = 0.0;
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) part += M[i * r + j] * M[i * r + j];
      const double nsq = block_sum(part);
      if (nsq >= kDegenerate || attempt > 16) {
        const double inv = 1.0 / sqrt(nsq);
        for (int64_t i = threadIdx.x; i < m; i += blockDim.x) M[i * r + j] *= inv;
        __syncthreads();
        break;
      }
      for (int64_t i = threadIdx.x; i < m; i += blockDim.x) M[i * r + j] = (double)curand_normal(&rng);
      __syncthreads();
    }
  }
  for (int64_t e = threadIdx.x; e < m * r; e += blockDim.x) out[e] = (float)M[e];
}

}  // namespace lr
}  // namespace cc
