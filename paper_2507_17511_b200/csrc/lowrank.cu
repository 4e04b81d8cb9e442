// K3: low-rank residual compressor (compressors.py:394-426, linalg.py:49-112).
//
//   Q0 = orth(G)                      G ~ N(0,1)[C, r] drawn on the host (cx:407)
//   T x { Z = A^T (A Q);  Q = orth(Z) }
//   U = orth(A Q);  W = A^T U         payload: U, W as column-major f16, or INT4
//                                     per-column codes + f32 ranges (cx:556-566)
//   decode: A_hat = U W^T             (cx:286-288), accumulated into the base
//
// The projections are skinny GEMMs (N = r <= 32) that stream A once per pass;
// they accumulate in f64 like the reference's la.matmul (la:49-58).  orth() is
// CholQR2 in f64: two passes of  G = M^T M (multi-CTA partial Grams, fixed-order
// reduction) -> Cholesky -> M <- M R^-1.  That computes the same Q as the
// reference's CGS2 (QR with positive diagonal) up to rounding; if a pivot falls
// below the reference's degeneracy tolerance (la:13, 1e-12) a single-CTA CGS2
// with random replacement columns takes over (rank-deficient inputs).
// Parity is tolerance-based (f64 summation order), see tests/test_gpu_lowrank.py.
#include "cc_common.cuh"
#include "cc_internal.h"
#include "lr_dev.cuh"
#include "cc_async.cuh"

#include <algorithm>
#include <cooperative_groups.h>
#include <mutex>
#include <unordered_map>
#include <curand_kernel.h>

namespace cc {
int64_t tc_partial_floats(int64_t n, int64_t C, int r);
int tc_project(int mode, const float *A, const float *S, float *D, float *Dpart, int64_t n, int64_t C, int r,
               cudaStream_t st, __half *d16 = nullptr);
int lowrank_backend();

namespace lr {

constexpr int kMaxR = 32;
constexpr int kThreads = 256;
constexpr int kRowsAQ = 32;    // rows per CTA in Y = A Q
constexpr int kKChunk = 96;    // K chunk staged in shared memory
constexpr int kColsATY = 32;   // columns of A per CTA in Z = A^T Y
constexpr int kSplitATY = 4;   // row splits (partial Z, fixed-order reduction)
constexpr int kGramRows = 128; // rows per CTA in the Gram partials

// ---------------------------------------------------------------------------
// Y[n, r] = A[n, C] Q[C, r]   (f64 accumulate, f32 store: la.matmul)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_aq(const float *__restrict__ A, const float *__restrict__ Q,
                                                  float *__restrict__ Y, int64_t n, int64_t C, int r) {
  __shared__ double qs[kKChunk][kMaxR + 1];
  __shared__ float as[kRowsAQ][kKChunk + 1];
  const int64_t i0 = (int64_t)blockIdx.x * kRowsAQ;
  // thread -> (row ii, output column pair)
  const int outs = kRowsAQ * r;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t k0 = 0; k0 < C; k0 += kKChunk) {
    const int kc = (int)min64(kKChunk, C - k0);
    for (int e = threadIdx.x; e < kc * r; e += kThreads) {
      const int kk = e / r, j = e % r;
      qs[kk][j] = (double)Q[(k0 + kk) * r + j];
    }
    for (int e = threadIdx.x; e < kRowsAQ * kc; e += kThreads) {
      const int ii = e / kc, kk = e % kc;
      as[ii][kk] = (i0 + ii < n) ? A[(i0 + ii) * C + k0 + kk] : 0.0f;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int o = threadIdx.x + s * kThreads;
      if (o < outs) {
        const int ii = o / r, j = o % r;
        double a = acc[s];
        for (int kk = 0; kk < kc; ++kk) a += (double)as[ii][kk] * qs[kk][j];
        acc[s] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int o = threadIdx.x + s * kThreads;
    if (o < outs) {
      const int ii = o / r, j = o % r;
      if (i0 + ii < n) Y[(i0 + ii) * r + j] = (float)acc[s];
    }
  }
}

// ---------------------------------------------------------------------------
// Zpart[split][C, r] = A[rows of split, :]^T Y[rows of split, :]
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_aty(const float *__restrict__ A, const float *__restrict__ Y,
                                                   double *__restrict__ Zpart, int64_t n, int64_t C, int r) {
  __shared__ float as[64][kColsATY + 1];
  __shared__ double ys[64][kMaxR + 1];
  const int64_t c0 = (int64_t)blockIdx.x * kColsATY;
  const int split = blockIdx.y;
  const int64_t rows_per = (n + kSplitATY - 1) / kSplitATY;
  const int64_t rlo = split * rows_per, rhi = min64(n, rlo + rows_per);
  const int outs = kColsATY * r;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t i0 = rlo; i0 < rhi; i0 += 64) {
    const int rc = (int)min64(64, rhi - i0);
    for (int e = threadIdx.x; e < rc * kColsATY; e += kThreads) {
      const int ii = e / kColsATY, cc = e % kColsATY;
      as[ii][cc] = (c0 + cc < C) ? A[(i0 + ii) * C + c0 + cc] : 0.0f;
    }
    for (int e = threadIdx.x; e < rc * r; e += kThreads) {
      const int ii = e / r, j = e % r;
      ys[ii][j] = (double)Y[(i0 + ii) * r + j];
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      const int o = threadIdx.x + s * kThreads;
      if (o < outs) {
        const int cc = o % kColsATY, j = o / kColsATY;
        double a = acc[s];
        for (int ii = 0; ii < rc; ++ii) a += (double)as[ii][cc] * ys[ii][j];
        acc[s] = a;
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int s = 0; s < 4; ++s) {
    const int o = threadIdx.x + s * kThreads;
    if (o < outs) {
      const int cc = o % kColsATY, j = o / kColsATY;
      if (c0 + cc < C) Zpart[((int64_t)split * C + c0 + cc) * r + j] = acc[s];
    }
  }
}

// Z[C, r] (f32) = sum over splits in order
__global__ void k_zsum(const double *__restrict__ Zpart, float *__restrict__ Z, int64_t C, int r) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= C * r) return;
  double s = 0.0;
  for (int sp = 0; sp < kSplitATY; ++sp) s += Zpart[sp * C * r + e];
  Z[e] = (float)s;
}

// ---------------------------------------------------------------------------
// CholQR2 (f64): M[m, r] -> orthonormal columns, positive R diagonal
// ---------------------------------------------------------------------------
__global__ void k_to64(const float *__restrict__ in, double *__restrict__ out, int64_t cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < cnt) out[e] = (double)in[e];
}

__global__ void __launch_bounds__(kThreads) k_gram(const double *__restrict__ M, double *__restrict__ Gpart,
                                                    int64_t m, int r) {
  __shared__ double ms[kGramRows][kMaxR + 1];
  const int64_t i0 = (int64_t)blockIdx.x * kGramRows;
  const int rc = (int)min64(kGramRows, m - i0);
  for (int e = threadIdx.x; e < rc * r; e += kThreads) ms[e / r][e % r] = M[(i0 + e / r) * r + e % r];
  __syncthreads();
  for (int o = threadIdx.x; o < r * r; o += kThreads) {
    const int a = o / r, b = o % r;
    double s = 0.0;
    for (int i = 0; i < rc; ++i) s += ms[i][a] * ms[i][b];
    Gpart[(int64_t)blockIdx.x * r * r + o] = s;
  }
}

// one CTA (1024 threads): G = sum of partials (fixed order); Cholesky G = R^T R
// (right-looking, one column per step, trailing update in parallel); Rinv = R^-1
// (one column per thread, back substitution); flag = 1 if any pivot^2 < tol
// (degenerate column -> CGS2 fallback)
__global__ void __launch_bounds__(1024) k_chol(const double *__restrict__ Gpart, int nblk, int r,
                                               double *__restrict__ Rinv, int *__restrict__ flag, int pass) {
  __shared__ double G[kMaxR][kMaxR + 1];
  __shared__ double R[kMaxR][kMaxR + 1];
  __shared__ int bad;
  const int t = threadIdx.x;
  const int a = t / kMaxR, c = t % kMaxR;  // (row, column) owned by this thread
  if (a < r && c < r) {
    // fixed-order sum of the block partials; 8 independent loads in flight per step
    double s = 0.0;
    int b = 0;
    for (; b + 8 <= nblk; b += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = Gpart[(int64_t)(b + q) * r * r + a * r + c];
#pragma unroll
      for (int q = 0; q < 8; ++q) s += v[q];
    }
    for (; b < nblk; ++b) s += Gpart[(int64_t)b * r * r + a * r + c];
    G[a][c] = s;
    R[a][c] = 0.0;
  }
  if (t == 0) bad = 0;
  __syncthreads();
  for (int j = 0; j < r; ++j) {
    // G now holds the Schur complement for rows/cols >= j
    if (t == 0) {
      double piv = G[j][j];
      if (!(piv >= kDegenerate)) {
        bad = 1;
        piv = 1.0;
      }
      R[j][j] = sqrt(piv);
    }
    __syncthreads();
    if (t > j && t < r) R[j][t] = G[j][t] / R[j][j];
    __syncthreads();
    if (a > j && a < r && c >= a && c < r) G[a][c] -= R[j][a] * R[j][c];
    if (a > j && a < r && c > j && c < a) G[a][c] -= R[j][a] * R[j][c];  // keep the lower half consistent
    __syncthreads();
  }
  if (t < r) {  // column t of Rinv (upper triangular)
    double x[kMaxR];
    for (int i = r - 1; i >= 0; --i) {
      double s = (i == t) ? 1.0 : 0.0;
      for (int k = i + 1; k <= t; ++k) s -= R[i][k] * x[k];
      x[i] = (i > t) ? 0.0 : s / R[i][i];
    }
    for (int i = 0; i < r; ++i) Rinv[i * r + t] = x[i];
  }
  if (t == 0) {
    if (pass == 0) *flag = bad;
    else *flag |= bad;
  }
}

// M <- M Rinv (row-wise, f64)
__global__ void __launch_bounds__(kThreads) k_apply_rinv(double *__restrict__ M, const double *__restrict__ Rinv,
                                                          int64_t m, int r) {
  __shared__ double rs[kMaxR * kMaxR];
  for (int e = threadIdx.x; e < r * r; e += kThreads) rs[e] = Rinv[e];
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (i >= m) return;
  double row[kMaxR];
  for (int k = 0; k < r; ++k) row[k] = M[i * r + k];
  for (int c = 0; c < r; ++c) {
    double s = 0.0;
    for (int k = 0; k <= c; ++k) s += row[k] * rs[k * r + c];
    M[i * r + c] = s;
  }
}

// Fallback (rank-deficient input): CGS2 with two projection passes, degenerate
// columns replaced by N(0,1) draws (la:77-112).  One CTA, only when flagged.
__global__ void __launch_bounds__(1024) k_cgs2_fallback(const float *__restrict__ orig, double *__restrict__ M,
                                                         int64_t m, int r, const int *__restrict__ flag,
                                                         unsigned long long seed) {
  if (*flag == 0) return;
  __shared__ double red[32];
  __shared__ double coef[kMaxR];
  auto block_sum = [&](double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += red[w];
      red[0] = s;
    }
    __syncthreads();
    s = red[0];
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
}

// ---------------------------------------------------------------------------
// CholQR2 in ONE cooperative launch (the production orth): nb = ceil(m / 128)
// CTAs x 256 threads, CTA b keeps rows [128 b, 128 b + 128) of M in shared
// memory (f64).  Per pass: partial Gram of the CTA's rows -> grid sync -> every
// CTA sums the partials in the same fixed order, factors G = R^T R and forms
// R^-1 (identical in every CTA) -> M <- M R^-1 on its rows.  Same arithmetic as
// k_gram / k_chol / k_apply_rinv (so the same Q bit for bit), without the eight
// dependent launches.  A degenerate pivot (la:13) in either pass hands the whole
// matrix to CTA 0's CGS2 with random replacement columns (la:77-112).
// ---------------------------------------------------------------------------
constexpr int kOrthThreads = 256;


// one warp: right-looking Cholesky of G (as k_chol) and R^-1 into Ri, lane c owns column c
template <int LD = kMaxR + 1>
__device__ __forceinline__ void chol_rinv_warp(double (*G)[LD], double (*R)[LD], double (*Ri)[LD], int r, int *bad) {
  const int c = threadIdx.x & 31;
  for (int j = 0; j < r; ++j) {
    double piv = G[j][j];  // every lane reads the same pivot
    if (!(piv >= kDegenerate)) {
      if (c == 0) *bad = 1;
      piv = 1.0;
    }
    const double rjj = sqrt(piv);
    if (c == j) R[j][j] = rjj;
    if (c > j && c < r) R[j][c] = G[j][c] / rjj;
    __syncwarp();
    if (c > j && c < r)
      for (int a = j + 1; a < r; ++a) G[a][c] -= R[j][a] * R[j][c];
    __syncwarp();
  }
  if (c < r) {  // column c of R^-1 (upper triangular), back substitution into shared memory
    for (int i = r - 1; i >= 0; --i) {
      double sacc = (i == c) ? 1.0 : 0.0;
      for (int k = i + 1; k <= c; ++k) sacc -= R[i][k] * Ri[k][c];
      Ri[i][c] = (i > c) ? 0.0 : sacc / R[i][i];
    }
  }
}

__global__ void __launch_bounds__(kOrthThreads) k_orth(const float *__restrict__ Min, float *__restrict__ out,
                                                        int64_t m, int r, double *__restrict__ Gpart,
                                                        double *__restrict__ scratch, unsigned long long seed) {
  extern __shared__ double osm[];
  double(*ms)[kMaxR + 1] = reinterpret_cast<double(*)[kMaxR + 1]>(osm);           // [kGramRows][33]
  double(*G)[kMaxR + 1] = reinterpret_cast<double(*)[kMaxR + 1]>(osm + kGramRows * (kMaxR + 1));
  double(*R)[kMaxR + 1] = G + kMaxR;
  double(*Ri)[kMaxR + 1] = R + kMaxR;
  __shared__ int bad;
  __shared__ double red[kOrthThreads / 32], coef[kMaxR];
  cooperative_groups::grid_group grid = cooperative_groups::this_grid();
  const int tid = threadIdx.x, b = blockIdx.x, nb = gridDim.x;
  const int64_t i0 = (int64_t)b * kGramRows;
  const int rc = (int)min64(kGramRows, m - i0);
  for (int e = tid; e < rc * r; e += kOrthThreads) ms[e / r][e % r] = (double)Min[(i0 + e / r) * r + e % r];
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    double *gp = Gpart + (size_t)pass * nb * r * r;
    for (int o = tid; o < r * r; o += kOrthThreads) {  // partial Gram of this CTA's rows (as k_gram)
      const int a = o / r, c = o % r;
      double acc = 0.0;
      for (int i = 0; i < rc; ++i) acc += ms[i][a] * ms[i][c];
      gp[(size_t)b * r * r + o] = acc;
    }
    grid.sync();
    for (int o = tid; o < r * r; o += kOrthThreads) {  // fixed-order sum of the partials (as k_chol)
      const int a = o / r, c = o % r;
      double acc = 0.0;
      int bb = 0;
      for (; bb + 8 <= nb; bb += 8) {
        double v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) v[q] = __ldcg(gp + (size_t)(bb + q) * r * r + o);
#pragma unroll
        for (int q = 0; q < 8; ++q) acc += v[q];
      }
      for (; bb < nb; ++bb) acc += __ldcg(gp + (size_t)bb * r * r + o);
      G[a][c] = acc;
      R[a][c] = 0.0;
    }
    __syncthreads();
    if (tid < 32) chol_rinv_warp(G, R, Ri, r, &bad);
    __syncthreads();
    for (int i = tid; i < rc; i += kOrthThreads) {  // M <- M R^-1 (as k_apply_rinv)
      double row[kMaxR];
      for (int k = 0; k < r; ++k) row[k] = ms[i][k];
      for (int c = 0; c < r; ++c) {
        double acc = 0.0;
        for (int k = 0; k <= c; ++k) acc += row[k] * Ri[k][c];
        ms[i][c] = acc;
      }
    }
    __syncthreads();
  }
  if (!bad) {
    for (int e = tid; e < rc * r; e += kOrthThreads) out[(i0 + e / r) * r + e % r] = (float)ms[e / r][e % r];
  } else if (b == 0) {  // every CTA saw the same pivots: CTA 0 alone re-orthogonalizes with CGS2
    cgs2_block(Min, scratch, out, m, r, seed, red, coef);
  }
}

// ---------------------------------------------------------------------------
// CholQR2 in ONE CTA for r <= 16 when the [m, r] block fits in shared memory (no
// grid-wide synchronisation), with the two r-wide products on the f64 tensor
// pipe (DMMA, mma.sync m8n8k4 f64: exact products, f64 accumulation):
//   Gram   G = M^T M: warp w takes rows 4k.. of its share; per k-step ONE shared
//          load per lane feeds both operands (A = M^T chunk, B = M chunk: the
//          same element for a lane); the 16 warps' 8x8 tiles summed in order
//   apply  M <- M R^-1 row tile by row tile (8 rows x r, k-steps of 4)
// The block is kept column-major in f64 (odd column stride), padded to RP = 8 or
// 16 columns with zeros; the warp Cholesky / R^-1 as in k_orth.  Same CholQR2
// mathematics as k_orth, a different (fixed) summation order.
// ---------------------------------------------------------------------------
constexpr int kOrth1Threads = 512;


__device__ unsigned long long *g_orth1_stamps = nullptr;  // profiling: [16] clock64 stamps of block 0

template <int RP>
__global__ void __launch_bounds__(kOrth1Threads, 1) k_orth1(const float *__restrict__ Min, float *__restrict__ out,
                                                             int64_t m, int r, double *__restrict__ scratch,
                                                             unsigned long long seed) {
  constexpr int W = kOrth1Threads / 32, RB = RP / 8;
  extern __shared__ __align__(16) uint8_t o1sm[];
  double *M = reinterpret_cast<double *>(o1sm);  // column-major [RP][mp], rows padded to a multiple of 8
  const int64_t m8 = (m + 7) & ~int64_t(7);
  const int64_t mp = m8 | 1;                     // odd stride: the rows of a column map to distinct banks
  constexpr int LD = 17;  // r <= 16
  __shared__ double G[16][LD], Rm[16][LD], Ri[16][LD];
  __shared__ double part[W][RB * RB][64];
  __shared__ double red[kOrth1Threads / 32], coef[kMaxR];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;  // MMA fragment coordinates
  unsigned long long *stp = g_orth1_stamps;
  auto stamp = [&](int i) {
    if (stp && tid == 0) stp[i] = clock64();
  };
  stamp(0);
  if (r == RP && (reinterpret_cast<uintptr_t>(Min) & 15) == 0) {  // float4 loads, 4 in flight per thread
    const int64_t nq = m8 * RP / 4;
    for (int64_t q0 = tid; q0 < nq; q0 += 4 * kOrth1Threads) {
      float4 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + u * kOrth1Threads;
        v[u] = (q < nq && 4 * q < m * RP) ? __ldg(reinterpret_cast<const float4 *>(Min) + q)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t q = q0 + u * kOrth1Threads;
        if (q < nq) {
          const int64_t i = 4 * q / RP;
          const int k = (int)(4 * q % RP);
          M[(k + 0) * mp + i] = v[u].x;
          M[(k + 1) * mp + i] = v[u].y;
          M[(k + 2) * mp + i] = v[u].z;
          M[(k + 3) * mp + i] = v[u].w;
        }
      }
    }
  } else {
    for (int64_t e = tid; e < m8 * RP; e += kOrth1Threads) {
      const int64_t i = e / RP;
      const int k = (int)(e % RP);
      M[k * mp + i] = (i < m && k < r) ? (double)Min[i * r + k] : 0.0;
    }
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  stamp(1);
  const int64_t nks = m8 / 4;  // Gram k-steps of 4 rows
  for (int pass = 0; pass < 2; ++pass) {
    // ---- Gram on the tensor pipe: tiles (ra, rc) with ra <= rc ----
    double acc[RB * RB][2];
#pragma unroll
    for (int t = 0; t < RB * RB; ++t) acc[t][0] = acc[t][1] = 0.0;
    double acc2[RB * RB][2];  // second accumulator chain (odd k-step pairs)
#pragma unroll
    for (int t = 0; t < RB * RB; ++t) acc2[t][0] = acc2[t][1] = 0.0;
    for (int64_t ks = warp; ks < nks; ks += 2 * W) {
      const bool two = ks + W < nks;
      double v[RB], v2[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b) {
        v[b] = M[(8 * b + gq) * mp + 4 * ks + tq];  // M[i][8b + gq]
        v2[b] = two ? M[(8 * b + gq) * mp + 4 * (ks + W) + tq] : 0.0;
      }
#pragma unroll
      for (int ra = 0; ra < RB; ++ra)
#pragma unroll
        for (int rc = ra; rc < RB; ++rc) {
          dmma884(acc[ra * RB + rc][0], acc[ra * RB + rc][1], v[ra], v[rc]);
          dmma884(acc2[ra * RB + rc][0], acc2[ra * RB + rc][1], v2[ra], v2[rc]);
        }
    }
#pragma unroll
    for (int t = 0; t < RB * RB; ++t) {
      acc[t][0] += acc2[t][0];
      acc[t][1] += acc2[t][1];
    }
#pragma unroll
    for (int t = 0; t < RB * RB; ++t) {
      part[warp][t][gq * 8 + 2 * tq] = acc[t][0];
      part[warp][t][gq * 8 + 2 * tq + 1] = acc[t][1];
    }
    __syncthreads();
    stamp(2 + 4 * pass);
    for (int o = tid; o < RP * RP; o += kOrth1Threads) {  // G entry (a, c), a <= c: warps summed in order
      const int a = o / RP, c = o % RP;
      if (a <= c && c < r) {
        const int t = (a / 8) * RB + c / 8;
        double v = 0.0;
        for (int w = 0; w < W; ++w) v += part[w][t][(a % 8) * 8 + (c % 8)];
        G[a][c] = v;
        G[c][a] = v;
      }
    }
    for (int e = tid; e < 16 * LD; e += kOrth1Threads) {
      Rm[e / LD][e % LD] = 0.0;
      Ri[e / LD][e % LD] = 0.0;
    }
    __syncthreads();
    stamp(3 + 4 * pass);
    if (warp == 0) {
      if (RP == 8 && r == 8) chol8_regs(G, Rm, Ri, &bad);
      else chol_rinv_regs<RP, LD>(G, Rm, Ri, r, &bad);
    }
    __syncthreads();
    stamp(4 + 4 * pass);
    // ---- apply: M <- M R^-1 (8-row tiles; Ri zero beyond r) ----
    double bfr[RB][RP / 4];  // B fragments: Ri[4 ks + tq][8 cb + gq]
#pragma unroll
    for (int cb = 0; cb < RB; ++cb)
#pragma unroll
      for (int ks = 0; ks < RP / 4; ++ks) bfr[cb][ks] = Ri[4 * ks + tq][8 * cb + gq];
    const int64_t ntile = m8 / 8;
    for (int64_t tile = warp; tile < ntile; tile += 2 * W) {  // two row tiles in flight
      const bool two = tile + W < ntile;
      const int64_t i = 8 * tile + gq, i2 = 8 * (tile + W) + gq;
      double afr[RP / 4], afr2[RP / 4];
#pragma unroll
      for (int ks = 0; ks < RP / 4; ++ks) {
        afr[ks] = M[(4 * ks + tq) * mp + i];  // A = M[i][4 ks + tq]
        afr2[ks] = two ? M[(4 * ks + tq) * mp + i2] : 0.0;
      }
      __syncwarp();
#pragma unroll
      for (int cb = 0; cb < RB; ++cb) {
        double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < RP / 4; ++ks) {
          dmma884(d0, d1, afr[ks], bfr[cb][ks]);
          dmma884(e0, e1, afr2[ks], bfr[cb][ks]);
        }
        M[(8 * cb + 2 * tq) * mp + i] = d0;  // D[gq][2 tq], D[gq][2 tq + 1]
        M[(8 * cb + 2 * tq + 1) * mp + i] = d1;
        if (two) {
          M[(8 * cb + 2 * tq) * mp + i2] = e0;
          M[(8 * cb + 2 * tq + 1) * mp + i2] = e1;
        }
      }
    }
    __syncthreads();
    stamp(5 + 4 * pass);
  }
  if (!bad) {
    if (r == RP && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
      const int64_t nq = m * RP / 4;
      for (int64_t q = tid; q < nq; q += kOrth1Threads) {
        const int64_t i = 4 * q / RP;
        const int k = (int)(4 * q % RP);
        reinterpret_cast<float4 *>(out)[q] = make_float4((float)M[(k + 0) * mp + i], (float)M[(k + 1) * mp + i],
                                                         (float)M[(k + 2) * mp + i], (float)M[(k + 3) * mp + i]);
      }
    } else {
      for (int64_t e = tid; e < m * r; e += kOrth1Threads) out[e] = (float)M[(e % r) * mp + e / r];
    }
  } else {  // rank-deficient: CGS2 with random replacement columns (la:77-112)
    cgs2_block(Min, scratch, out, m, r, seed, red, coef);
  }
  __syncthreads();
  stamp(10);
  if (stp && tid == 0) stp[11] = bad;
}

// ---------------------------------------------------------------------------
// CholQR2 on a thread-block CLUSTER of kOrthCl CTAs (distributed shared memory):
// CTA q keeps rows [q m8 / kOrthCl, ...) of the block (f64, column-major), so the
// f64 tensor-pipe work (Gram, M R^-1) and the loads / stores are split kOrthCl
// ways; per pass the CTAs' 8x8 Gram partials are exchanged through DSMEM (one
// cluster barrier) and summed in the same order by every CTA, which then factors
// the Gram redundantly (identical R^-1 everywhere, no broadcast).  r <= 16.
// ---------------------------------------------------------------------------
constexpr int kOrthCl = 8;
constexpr int kOrthClThreads = 256;

template <int RP>
__global__ void __launch_bounds__(kOrthClThreads, 1) k_orth_cl(const float *__restrict__ Min, float *__restrict__ out,
                                                                int64_t m, int r, double *__restrict__ scratch,
                                                                unsigned long long seed, __half *__restrict__ out16) {
  namespace cg = cooperative_groups;
  constexpr int W = kOrthClThreads / 32, RB = RP / 8, LD = 17;
  cg::cluster_group cluster = cg::this_cluster();
  const int q = (int)cluster.block_rank();
  extern __shared__ __align__(16) uint8_t ocsm[];
  const int64_t m8 = (m + 7) & ~int64_t(7);
  const int64_t t0 = (int64_t)q * (m8 / 8) / kOrthCl, t1 = (int64_t)(q + 1) * (m8 / 8) / kOrthCl;  // 8-row tiles
  const int64_t r0 = 8 * t0, nr = 8 * (t1 - t0);  // this CTA's rows [r0, r0 + nr)
  const int64_t mp = nr | 1;
  double *M = reinterpret_cast<double *>(ocsm);  // [RP][mp]
  __shared__ double G[16][LD], Rm[16][LD], Ri[16][LD];
  __shared__ double part[W][RB * RB][64];
  __shared__ double cpart[2][RB * RB][64];  // this CTA's Gram partial per pass (read by the cluster)
  __shared__ double red[kOrthClThreads / 32], coef[kMaxR];
  __shared__ int bad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  for (int64_t e = tid; e < nr * RP; e += kOrthClThreads) {
    const int64_t i = e / RP;
    const int k = (int)(e % RP);
    const int64_t gi = r0 + i;
    M[k * mp + i] = (gi < m && k < r) ? (double)Min[gi * r + k] : 0.0;
  }
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int pass = 0; pass < 2; ++pass) {
    double acc[RB * RB][2];
#pragma unroll
    for (int t = 0; t < RB * RB; ++t) acc[t][0] = acc[t][1] = 0.0;
    for (int64_t ks = warp; ks < nr / 4; ks += W) {
      double v[RB];
#pragma unroll
      for (int b = 0; b < RB; ++b) v[b] = M[(8 * b + gq) * mp + 4 * ks + tq];
#pragma unroll
      for (int ra = 0; ra < RB; ++ra)
#pragma unroll
        for (int rc = ra; rc < RB; ++rc) dmma884(acc[ra * RB + rc][0], acc[ra * RB + rc][1], v[ra], v[rc]);
    }
#pragma unroll
    for (int t = 0; t < RB * RB; ++t) {
      part[warp][t][gq * 8 + 2 * tq] = acc[t][0];
      part[warp][t][gq * 8 + 2 * tq + 1] = acc[t][1];
    }
    __syncthreads();
    for (int o = tid; o < RB * RB * 64; o += kOrthClThreads) {  // CTA partial: warps in order
      double v = 0.0;
      for (int w = 0; w < W; ++w) v += part[w][o / 64][o % 64];
      cpart[pass][o / 64][o % 64] = v;
    }
    cluster.sync();  // every CTA's partial of this pass is published
    for (int o = tid; o < RP * RP; o += kOrthClThreads) {  // G entry (a, c): CTAs summed in rank order
      const int a = o / RP, c = o % RP;
      if (a <= c && c < r) {
        const int t = (a / 8) * RB + c / 8, idx = (a % 8) * 8 + (c % 8);
        double v = 0.0;
        for (int cq = 0; cq < kOrthCl; ++cq) {
          const double *rp = cluster.map_shared_rank(&cpart[pass][0][0], cq);
          v += rp[t * 64 + idx];
        }
        G[a][c] = v;
        G[c][a] = v;
      }
    }
    for (int e = tid; e < 16 * LD; e += kOrthClThreads) {
      Rm[e / LD][e % LD] = 0.0;
      Ri[e / LD][e % LD] = 0.0;
    }
    __syncthreads();
    if (warp == 0) {
      if (RP == 8 && r == 8) chol8_regs(G, Rm, Ri, &bad);
      else chol_rinv_regs<RP, LD>(G, Rm, Ri, r, &bad);
    }
    __syncthreads();
    double bfr[RB][RP / 4];
#pragma unroll
    for (int cb = 0; cb < RB; ++cb)
#pragma unroll
      for (int ks = 0; ks < RP / 4; ++ks) bfr[cb][ks] = Ri[4 * ks + tq][8 * cb + gq];
    for (int64_t tile = warp; tile < nr / 8; tile += W) {
      const int64_t i = 8 * tile + gq;
      double afr[RP / 4];
#pragma unroll
      for (int ks = 0; ks < RP / 4; ++ks) afr[ks] = M[(4 * ks + tq) * mp + i];
      __syncwarp();
#pragma unroll
      for (int cb = 0; cb < RB; ++cb) {
        double d0 = 0.0, d1 = 0.0;
#pragma unroll
        for (int ks = 0; ks < RP / 4; ++ks) dmma884(d0, d1, afr[ks], bfr[cb][ks]);
        M[(8 * cb + 2 * tq) * mp + i] = d0;
        M[(8 * cb + 2 * tq + 1) * mp + i] = d1;
      }
    }
    __syncthreads();
  }
  if (!bad) {
    for (int64_t e = tid; e < nr * r; e += kOrthClThreads) {
      const int64_t i = e / r;
      if (r0 + i < m) out[(r0 + i) * r + e % r] = (float)M[(e % r) * mp + i];
    }
    if (out16) {  // the f16 body factor, column-major (cx:425): f16(f32(q)) as k_pack_f16
      for (int64_t e = tid; e < nr * r; e += kOrthClThreads) {
        const int k = (int)(e / nr);
        const int64_t i = e % nr;
        if (r0 + i < m) out16[(int64_t)k * m + r0 + i] = __float2half_rn((float)M[k * mp + i]);
      }
    }
  } else if (q == 0) {  // every CTA saw the same pivots: CTA 0 alone runs CGS2 (la:77-112)
    cgs2_block(Min, scratch, out, m, r, seed, red, coef);
  }
  cluster.sync();  // no CTA exits while another may still read its partials
}

__global__ void k_to32(const double *__restrict__ in, float *__restrict__ out, int64_t cnt) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < cnt) out[e] = (float)in[e];
}

// ---------------------------------------------------------------------------
// packing (cx:415-426, 556-566, 589-595)
// ---------------------------------------------------------------------------
// f16 body: U column-major [n, r] then W column-major [C, r]
__global__ void k_pack_f16(const float *__restrict__ F, int64_t m, int r, __half *__restrict__ out) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // column-major index
  if (e >= m * r) return;
  const int64_t j = e / m, i = e % m;
  out[e] = __float2half_rn(F[i * r + j]);
}

// per-column max |f| -> ranges (f32); one CTA per column
__global__ void k_colmax(const float *__restrict__ F, int64_t m, int r, float *__restrict__ ranges) {
  const int j = blockIdx.x;
  float mx = 0.0f;
  for (int64_t i = threadIdx.x; i < m; i += blockDim.x) mx = fmaxf(mx, fabsf(F[i * r + j]));
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  __shared__ float sm[32];
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    float v = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v = fmaxf(v, sm[w]);
    ranges[j] = v;
  }
}


// nibble stream: U column-major then W column-major, low nibble first
__global__ void k_pack_int4(const float *__restrict__ U, const float *__restrict__ W, int64_t n, int64_t C, int r,
                            const float *__restrict__ ur, const float *__restrict__ wr, uint8_t *__restrict__ nib) {
  const int64_t total = (n + C) * r;
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // output byte
  if (2 * b >= total) return;
  uint32_t byte = 0;
  for (int h = 0; h < 2; ++h) {
    const int64_t e = 2 * b + h;
    if (e >= total) break;
    uint32_t code;
    if (e < n * r) {
      const int64_t j = e / n, i = e % n;
      code = int4_code(U[i * r + j], ur[j]);
    } else {
      const int64_t e2 = e - n * r;
      const int64_t j = e2 / C, i = e2 % C;
      code = int4_code(W[i * r + j], wr[j]);
    }
    byte |= code << (4 * h);
  }
  nib[b] = (uint8_t)byte;
}

// ---------------------------------------------------------------------------
// decode: base (+)= U W^T from a body (f16 or INT4 factors), f64 accumulate
// ---------------------------------------------------------------------------
__device__ __forceinline__ double factor_at(const uint8_t *body, int int4, int64_t n, int64_t C, int r, int which,
                                            int64_t i, int j) {
  if (!int4) {
    const __half *h = reinterpret_cast<const __half *>(body);
    const int64_t off = which == 0 ? (int64_t)j * n + i : n * r + (int64_t)j * C + i;
    return (double)__half2float(h[off]);
  }
  const float *rg = reinterpret_cast<const float *>(body);
  const double range = (double)(which == 0 ? rg[j] : rg[r + j]);
  const int64_t e = which == 0 ? (int64_t)j * n + i : n * r + (int64_t)j * C + i;
  const uint8_t *nib = body + 8 * r;
  const uint32_t code = (nib[e >> 1] >> (4 * (e & 1))) & 15u;
  return -range + (double)code * (2.0 * range / 15.0);  // cx:569-572
}

// Sender-side state update of a low-rank step with the decode fused in: the
// reconstruction d = f32(sum_k U[i,k] W[j,k]) in f64 from the body's factors (the
// receiver's k_lr_decode arithmetic, same summation order, so sender and receiver
// bases stay bit-identical) applied directly: base' = base + d (naive: d),
// feedback' = t - d, ref' = x (pipeline.py:107-113); StepRecord partials per CTA
// (||d - t||^2, ||t||^2, pipeline.py:115-120).  No decoded tensor is materialised.
// Thread = one column j (W's column from the transposed factor WfT [r][C]:
// coalesced), kOARows rows per CTA with every row's loads in flight together.
constexpr int kOARows = 16;
// The factors come straight from the body (f16 / INT4 -> f64 exactly as the
// receiver's k_unpack_factors does) and the last CTA (ticket on a zeroed slab
// word) reduces the record partials in CTA order: one launch for decode + update +
// record.
template <int MODE, typename XT, int RM>
__global__ void __launch_bounds__(kThreads) k_outer_apply(const uint8_t *__restrict__ body, int int4, int64_t n,
                                                           int64_t C, int r, const XT *__restrict__ x,
                                                           const float *__restrict__ t, float *__restrict__ base,
                                                           float *__restrict__ aux, double *__restrict__ part,
                                                           unsigned int *ticket, double *__restrict__ record) {
  __shared__ double us[kOARows][kMaxR];
  __shared__ double se[kThreads / 32], st2[kThreads / 32];
  __shared__ unsigned last;
  const int64_t i0 = (int64_t)blockIdx.y * kOARows;
  const int nr = (int)min64(kOARows, n - i0);
  for (int e = threadIdx.x; e < kOARows * r; e += kThreads) {
    const int ii = e / r, k = e % r;
    us[ii][k] = ii < nr ? factor_at(body, int4, n, C, r, 0, i0 + ii, k) : 0.0;
  }
  __syncthreads();
  const int64_t j = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  double err = 0.0, tsq = 0.0;
  if (j < C) {
    double w[RM];  // RM >= r, compile-time: W's column stays in registers
#pragma unroll
    for (int k = 0; k < RM; ++k) w[k] = k < r ? factor_at(body, int4, n, C, r, 1, j, k) : 0.0;
    float tt[kOARows], bb[kOARows], xx[kOARows];
#pragma unroll
    for (int ii = 0; ii < kOARows; ++ii) {  // every row's loads in flight together
      const int64_t e = (i0 + ii) * C + j;
      tt[ii] = ii < nr ? t[e] : 0.0f;
      bb[ii] = (MODE != CC_NAIVE && ii < nr) ? base[e] : 0.0f;
      xx[ii] = (MODE == CC_NO_FEEDBACK && ii < nr) ? Act<XT>::load1(x + e) : 0.0f;
    }
#pragma unroll
    for (int ii = 0; ii < kOARows; ++ii) {
      if (ii >= nr) break;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < RM; ++k)
        if (k < r) s += us[ii][k] * w[k];
      const float d = (float)s;
      const int64_t e = (i0 + ii) * C + j;
      const double df = (double)d - (double)tt[ii];
      err += df * df;
      tsq += (double)tt[ii] * (double)tt[ii];
      if constexpr (MODE == CC_NAIVE) {
        base[e] = d;
      } else {
        base[e] = __fadd_rn(bb[ii], d);
        if constexpr (MODE == CC_WITH_FEEDBACK) aux[e] = __fsub_rn(tt[ii], d);
        else aux[e] = xx[ii];
      }
    }
  }
  err = warp_sum(err);
  tsq = warp_sum(tsq);
  if ((threadIdx.x & 31) == 0) {
    se[threadIdx.x >> 5] = err;
    st2[threadIdx.x >> 5] = tsq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) {
      a += se[i];
      b += st2[i];
    }
    const int64_t blk = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
    part[2 * blk] = a;
    part[2 * blk + 1] = b;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
  }
  __syncthreads();
  if (last) {  // fixed-order sum of every CTA's partials (as k_sum_parts)
    __threadfence();
    const int nparts = (int)(gridDim.x * gridDim.y);
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kThreads) {
      a += __ldcg(part + 2 * i);
      b += __ldcg(part + 2 * i + 1);
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if ((threadIdx.x & 31) == 0) {
      se[threadIdx.x >> 5] = a;
      st2[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double x0 = 0.0, y0 = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) {
        x0 += se[w];
        y0 += st2[w];
      }
      record[0] = x0;
      record[1] = y0;
      *ticket = 0u;  // the slab word is zero again for the next launch
    }
  }
}

struct Work {
  float *Q, *Y, *Z, *U, *W, *TCpart;
  double *Zpart, *M64, *Gpart, *Rinv, *Uf, *Wf;
  float *ur, *wr;
  int *flag;
};

static Work carve(void *ws, int64_t n, int64_t C, int64_t r, size_t *bytes) {
  Work w{};
  uint8_t *b = reinterpret_cast<uint8_t *>(ws);
  size_t off = 0;
  auto take = [&](size_t sz) {
    uint8_t *q = b ? b + off : nullptr;
    off = align_up(off + sz, 256);
    return q;
  };
  const int64_t m = std::max(n, C);
  w.Q = reinterpret_cast<float *>(take(4 * C * r));
  w.Y = reinterpret_cast<float *>(take(4 * n * r));
  w.Z = reinterpret_cast<float *>(take(4 * C * r));
  w.U = reinterpret_cast<float *>(take(4 * n * r));
  w.W = reinterpret_cast<float *>(take(4 * C * r));
  w.Zpart = reinterpret_cast<double *>(take(8 * kSplitATY * C * r));
  w.M64 = reinterpret_cast<double *>(take(8 * m * r));
  w.Gpart = reinterpret_cast<double *>(take(8 * 2 * cdiv(m, kGramRows) * r * r));
  w.Rinv = reinterpret_cast<double *>(take(8 * r * r));
  w.Uf = reinterpret_cast<double *>(take(8 * n * r));
  w.Wf = reinterpret_cast<double *>(take(8 * C * r));
  w.ur = reinterpret_cast<float *>(take(4 * r));
  w.wr = reinterpret_cast<float *>(take(4 * r));
  w.flag = reinterpret_cast<int *>(take(256));
  w.TCpart = reinterpret_cast<float *>(take(4 * (size_t)tc_partial_floats(n, C, (int)r)));
  if (bytes) *bytes = off;
  return w;
}

}  // namespace lr

int64_t lowrank_workspace_bytes(int64_t n, int64_t C, int64_t r) {
  size_t b = 0;
  lr::carve(nullptr, n, C, r, &b);
  return (int64_t)b;
}

static unsigned long long g_lr_seed = 0x5eed5eedULL;
static int g_orth_cluster = 1;  // 1: cluster CholQR2 (k_orth_cl), 0: single CTA / grid forms (A/B)
void set_orth_cluster(int on) { g_orth_cluster = on; }

void set_orth1_stamps(void *buf) {
  unsigned long long *p = reinterpret_cast<unsigned long long *>(buf);
  cudaMemcpyToSymbol(lr::g_orth1_stamps, &p, sizeof(p));
}

// M (f32 [m, r]) -> orthonormal f32 columns written to out (may alias M)
// returns true when the f16 column-major copy (out16, optional) was written too
static bool orth(const float *M, float *out, int64_t m, int r, const lr::Work &w, cudaStream_t st,
                 __half *out16 = nullptr) {
  using namespace lr;
  const int rp = r <= 8 ? 8 : 16;
  if (r <= 16 && g_orth_cluster) {  // cluster of kOrthCl CTAs (DSMEM Gram exchange)
    const int64_t m8 = (m + 7) & ~int64_t(7);
    const int64_t rows_max = 8 * cdiv(m8 / 8, kOrthCl);
    const size_t need = (size_t)(rows_max | 1) * rp * 8;
    const void *kern = rp == 8 ? (const void *)k_orth_cl<8> : (const void *)k_orth_cl<16>;
    static size_t max_dyn[2] = {0, 0};
    size_t &md = max_dyn[rp == 16];
    if (md == 0) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      md = 227 * 1024 - fa.sharedSizeBytes - 1024;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)md);
    }
    if (need <= md && m >= 8 * kOrthCl) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(kOrthCl);
      cfg.blockDim = dim3(kOrthClThreads);
      cfg.dynamicSmemBytes = need;
      cfg.stream = st;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = kOrthCl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      unsigned long long seed = g_lr_seed++;
      double *scratch = w.M64;
      __half *o16 = out16;
      const cudaError_t e = rp == 8 ? cudaLaunchKernelEx(&cfg, k_orth_cl<8>, M, out, m, r, scratch, seed, o16)
                                    : cudaLaunchKernelEx(&cfg, k_orth_cl<16>, M, out, m, r, scratch, seed, o16);
      if (e == cudaSuccess) {
        count_launch();
        return true;
      }
      cudaGetLastError();
    }
  }
  const size_t need = (size_t)(((m + 7) & ~int64_t(7)) | 1) * rp * 8;
  if (r <= 16) {  // one CTA (no cluster launch available): same mathematics, no grid sync
    const void *kern = rp == 8 ? (const void *)k_orth1<8> : (const void *)k_orth1<16>;
    static size_t max_dyn[2] = {0, 0};
    size_t &md = max_dyn[rp == 16];
    if (md == 0) {
      cudaFuncAttributes fa{};
      cudaFuncGetAttributes(&fa, kern);
      md = 227 * 1024 - fa.sharedSizeBytes - 1024;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)md);
    }
    if (need <= md) {
      unsigned long long seed = g_lr_seed++;
      double *scratch = w.M64;
      void *args[] = {&M, &out, &m, &r, &scratch, &seed};
      if (cudaLaunchKernel(kern, dim3(1), dim3(kOrth1Threads), args, need, st) == cudaSuccess) {
        count_launch();
        return false;
      }
      cudaGetLastError();
    }
  }
  {
    const int nb = (int)cdiv(m, kGramRows);
    const size_t smem = sizeof(double) * (size_t)(kGramRows + 3 * kMaxR) * (kMaxR + 1);
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_orth, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      attr = true;
    }
    unsigned long long seed = g_lr_seed++;
    double *gp = w.Gpart, *scratch = w.M64;
    void *args[] = {&M, &out, &m, &r, &gp, &scratch, &seed};
    if (cudaLaunchCooperativeKernel((const void *)k_orth, dim3(nb), dim3(kOrthThreads), args, smem, st) ==
        cudaSuccess) {
      count_launch();
      return false;
    }
    cudaGetLastError();  // fall through to the multi-kernel CholQR2
  }
  const int64_t cnt = m * r;
  const unsigned b1 = (unsigned)cdiv(cnt, 256);
  k_to64<<<b1, 256, 0, st>>>(M, w.M64, cnt);
  const int nblk = (int)cdiv(m, kGramRows);
  for (int pass = 0; pass < 2; ++pass) {
    k_gram<<<nblk, kThreads, 0, st>>>(w.M64, w.Gpart, m, r);
    k_chol<<<1, 1024, 0, st>>>(w.Gpart, nblk, r, w.Rinv, w.flag, pass);
    k_apply_rinv<<<(unsigned)cdiv(m, kThreads), kThreads, 0, st>>>(w.M64, w.Rinv, m, r);
  }
  k_cgs2_fallback<<<1, 1024, 0, st>>>(M, w.M64, m, r, w.flag, g_lr_seed++);
  k_to32<<<b1, 256, 0, st>>>(w.M64, out, cnt);
  count_launch(4 + 6);
  return false;
}

static void aq(const float *A, const float *Q, float *Y, const lr::Work &w, int64_t n, int64_t C, int r,
               cudaStream_t st) {
  if (lowrank_backend() == 1) {
    tc_project(0, A, Q, Y, w.TCpart, n, C, r, st);
    return;
  }
  lr::k_aq<<<(unsigned)cdiv(n, lr::kRowsAQ), lr::kThreads, 0, st>>>(A, Q, Y, n, C, r);
  count_launch();
}

// returns true when the f16 column-major copy (z16, optional) was written too
static bool aty(const float *A, const float *Y, float *Z, const lr::Work &w, int64_t n, int64_t C, int r,
                cudaStream_t st, __half *z16 = nullptr) {
  if (lowrank_backend() == 1) {
    tc_project(1, A, Y, Z, w.TCpart, n, C, r, st, z16);
    return z16 != nullptr;
  }
  dim3 g((unsigned)cdiv(C, lr::kColsATY), lr::kSplitATY);
  lr::k_aty<<<g, lr::kThreads, 0, st>>>(A, Y, w.Zpart, n, C, r);
  lr::k_zsum<<<(unsigned)cdiv(C * r, 256), 256, 0, st>>>(w.Zpart, Z, C, r);
  count_launch(2);
  return false;
}

namespace lr {
// ---------------------------------------------------------------------------
// Batched receiver decode (cx:286-288 for every peer of the step in one launch):
// base (+)= f32(U W^T), the factors read straight from each body (f16 / INT4 ->
// f64 as factor_at), f64 accumulation in k order (the sender's k_outer_apply /
// lr_step.cu arithmetic: bases stay bit-identical).  Block = kDecRows rows x
// kDecThreads x CPT columns of one peer (blockIdx.z); W's columns stay in
// registers, U's rows in shared memory; 4 rows of base loads in flight.
// ---------------------------------------------------------------------------
constexpr int kDecRows = 16;
constexpr int kDecThreads = 128;
constexpr int kDecMax = 16;  // peers per launch
constexpr int kDecBatch = 4; // rows of base loads in flight per thread (8: measured slower)
struct DecBatch {
  const uint8_t *body[kDecMax];
  float *base[kDecMax];
  int64_t rows[kDecMax];
};

template <int RM, int CPT>
__global__ void __launch_bounds__(kDecThreads) k_lr_decode(const DecBatch B, int int4, int64_t C, int r, int acc) {
  const int pi = (int)blockIdx.z;
  const int64_t n = B.rows[pi];
  const int64_t i0 = (int64_t)blockIdx.y * kDecRows;
  if (i0 >= n) return;
  const uint8_t *body = B.body[pi];
  __shared__ double us[kDecRows][RM];
  const int nr = (int)min64(kDecRows, n - i0);
  for (int e = threadIdx.x; e < kDecRows * RM; e += kDecThreads) {
    const int ii = e / RM, k = e % RM;
    us[ii][k] = (ii < nr && k < r) ? factor_at(body, int4, n, C, r, 0, i0 + ii, k) : 0.0;
  }
  __syncthreads();
  const int64_t j0 = ((int64_t)blockIdx.x * kDecThreads + threadIdx.x) * CPT;
  if (j0 >= C) return;
  double w[CPT][RM];
#pragma unroll
  for (int jj = 0; jj < CPT; ++jj)
#pragma unroll
    for (int k = 0; k < RM; ++k) w[jj][k] = (j0 + jj < C && k < r) ? factor_at(body, int4, n, C, r, 1, j0 + jj, k) : 0.0;
  float *out = B.base[pi];
  const bool vec = CPT == 4 && j0 + 4 <= C && ((reinterpret_cast<uintptr_t>(out + j0) | (uintptr_t)(C * 4)) & 15) == 0;
  for (int ib = 0; ib < nr; ib += kDecBatch) {
    float o[kDecBatch][CPT];
#pragma unroll
    for (int u = 0; u < kDecBatch; ++u) {  // the base rows' loads in flight together
      const int ii = ib + u;
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) o[u][jj] = 0.f;
      if (acc && ii < nr) {
        const float *src = out + (i0 + ii) * C + j0;
        if (vec) {
          const float4 v = *reinterpret_cast<const float4 *>(src);
          o[u][0] = v.x;
          o[u][1] = v.y;
          o[u][2] = v.z;
          o[u][3] = v.w;
        } else {
#pragma unroll
          for (int jj = 0; jj < CPT; ++jj)
            if (j0 + jj < C) o[u][jj] = src[jj];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < kDecBatch; ++u) {
      const int ii = ib + u;
      if (ii >= nr) break;
#pragma unroll
      for (int jj = 0; jj < CPT; ++jj) {
        double sacc = 0.0;  // k_lr_decode's order: k = 0 .. r-1
#pragma unroll
        for (int k = 0; k < RM; ++k)
          if (k < r) sacc += us[ii][k] * w[jj][k];
        const float d = (float)sacc;
        o[u][jj] = acc ? __fadd_rn(o[u][jj], d) : d;
      }
      float *dst = out + (i0 + ii) * C + j0;
      if (vec) {
        *reinterpret_cast<float4 *>(dst) = make_float4(o[u][0], o[u][1], o[u][2], o[u][3]);
      } else {
#pragma unroll
        for (int jj = 0; jj < CPT; ++jj)
          if (j0 + jj < C) dst[jj] = o[u][jj];
      }
    }
  }
}

// TMA form (r <= 8, accumulate): the CTA's tile of every base row (16 rows x 512
// columns, 32 KB) arrives by 1-D bulk copies on one mbarrier while the factors load,
// so the base reads are in flight without holding registers; thread = 2 columns.
constexpr int kDtRows = 16, kDtCols = 512, kDtThreads = 256;
__global__ void __launch_bounds__(kDtThreads) k_lr_decode_tma(const DecBatch B, int int4, int64_t C, int r) {
  const int pi = (int)blockIdx.z;
  const int64_t n = B.rows[pi];
  const int64_t i0 = (int64_t)blockIdx.y * kDtRows;
  if (i0 >= n) return;
  const int64_t jb = (int64_t)blockIdx.x * kDtCols;
  const uint8_t *body = B.body[pi];
  float *out = B.base[pi];
  __shared__ __align__(128) float tile[kDtRows][kDtCols];
  __shared__ double us[kDtRows][8];
  __shared__ __align__(8) uint64_t bar;
  const int nr = (int)min64(kDtRows, n - i0);
  const int nc = (int)min64(kDtCols, C - jb);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_fence_init();
    mbar_expect_tx(&bar, (uint32_t)(nr * nc * 4));
    for (int i = 0; i < nr; ++i) bulk_g2s(&tile[i][0], out + (i0 + i) * C + jb, (uint32_t)(nc * 4), &bar,
                                          l2_policy_evict_first());
  }
  for (int e = threadIdx.x; e < kDtRows * 8; e += kDtThreads) {
    const int ii = e >> 3, k = e & 7;
    us[ii][k] = (ii < nr && k < r) ? factor_at(body, int4, n, C, r, 0, i0 + ii, k) : 0.0;
  }
  const int j0 = 2 * threadIdx.x;
  double w[2][8];
#pragma unroll
  for (int jj = 0; jj < 2; ++jj)
#pragma unroll
    for (int k = 0; k < 8; ++k) w[jj][k] = (j0 + jj < nc && k < r) ? factor_at(body, int4, n, C, r, 1, jb + j0 + jj, k) : 0.0;
  __syncthreads();  // us, and the barrier's initialisation
  mbar_wait(&bar, 0);
  if (j0 < nc) {
    for (int ii = 0; ii < nr; ++ii) {
      float o[2];
#pragma unroll
      for (int jj = 0; jj < 2; ++jj) {
        double sacc = 0.0;  // k_lr_decode's order: k = 0 .. r-1
#pragma unroll
        for (int k = 0; k < 8; ++k)
          if (k < r) sacc += us[ii][k] * w[jj][k];
        o[jj] = __fadd_rn(tile[ii][j0 + jj], (float)sacc);
      }
      float *dst = out + (i0 + ii) * C + jb + j0;
      if (j0 + 2 <= nc) __stcs(reinterpret_cast<float2 *>(dst), make_float2(o[0], o[1]));
      else dst[0] = o[0];
    }
  }
}
}  // namespace lr

static int g_dec_tma = [] {
  const char *e = getenv("CC_LR_DECODE_TMA");  // A/B: 0 = the register-staged decode
  return e ? atoi(e) : 1;
}();
// every body of the step (same C, r) decoded into its base in one launch per kDecMax
static void decode_batch(const uint8_t *const *bodies, float *const *bases, const int64_t *rows, int count, int int4,
                         int64_t C, int r, int acc, cudaStream_t st) {
  for (int b0 = 0; b0 < count; b0 += lr::kDecMax) {
    const int m = std::min(count - b0, lr::kDecMax);
    lr::DecBatch B{};
    int64_t maxn = 0;
    for (int i = 0; i < m; ++i) {
      B.body[i] = bodies[b0 + i];
      B.base[i] = bases[b0 + i];
      B.rows[i] = rows[b0 + i];
      maxn = std::max(maxn, rows[b0 + i]);
    }
    const dim3 blk(lr::kDecThreads);
    bool tma_ok = acc && r <= 8 && (C % 4) == 0 && g_dec_tma;
    for (int i = 0; i < m && tma_ok; ++i)
      tma_ok = (reinterpret_cast<uintptr_t>(B.base[i]) & 15) == 0;
    if (tma_ok) {
      const dim3 g((unsigned)cdiv(C, lr::kDtCols), (unsigned)cdiv(maxn, lr::kDtRows), (unsigned)m);
      lr::k_lr_decode_tma<<<g, lr::kDtThreads, 0, st>>>(B, int4, C, r);
    } else if (r <= 8) {
      const dim3 g((unsigned)cdiv(C, lr::kDecThreads * 4), (unsigned)cdiv(maxn, lr::kDecRows), (unsigned)m);
      lr::k_lr_decode<8, 4><<<g, blk, 0, st>>>(B, int4, C, r, acc);
    } else if (r <= 16) {
      const dim3 g((unsigned)cdiv(C, lr::kDecThreads * 2), (unsigned)cdiv(maxn, lr::kDecRows), (unsigned)m);
      lr::k_lr_decode<16, 2><<<g, blk, 0, st>>>(B, int4, C, r, acc);
    } else {
      const dim3 g((unsigned)cdiv(C, lr::kDecThreads), (unsigned)cdiv(maxn, lr::kDecRows), (unsigned)m);
      lr::k_lr_decode<32, 1><<<g, blk, 0, st>>>(B, int4, C, r, acc);
    }
    count_launch();
  }
}

static void decode_into(const uint8_t *body, int int4, int64_t n, int64_t C, int r, float *out, int acc,
                        const lr::Work &, cudaStream_t st) {
  decode_batch(&body, &out, &n, 1, int4, C, r, acc, st);
}

int lowrank_encode(int int4, int64_t n, int64_t C, int64_t r64, int iters, const float *t, const float *q0,
                   uint8_t *body, float *decoded, void *ws, int64_t ws_bytes, cudaStream_t st) {
  const int r = (int)r64;
  if (r > lr::kMaxR) {
    set_error("low-rank: rank > 32 not supported on device");
    return CC_ERR_UNSUPPORTED;
  }
  size_t need = 0;
  lr::carve(nullptr, n, C, r, &need);
  if ((int64_t)need > ws_bytes) {
    set_error("low-rank workspace too small");
    return CC_ERR_ARG;
  }
  const lr::Work w = lr::carve(ws, n, C, r, nullptr);
  orth(q0, w.Q, C, r, w, st);                  // Q0 = orth(G)        (cx:407)
  for (int it = 0; it < iters; ++it) {         // (cx:408-410)
    aq(t, w.Q, w.Y, w, n, C, r, st);
    aty(t, w.Y, w.Z, w, n, C, r, st);
    orth(w.Z, w.Q, C, r, w, st);
  }
  aq(t, w.Q, w.Y, w, n, C, r, st);
  // f16 bodies: U and W are written into the body by the last orth / projection
  // themselves when those paths can (column-major f16, cx:425), else packed here
  __half *h = int4 ? nullptr : reinterpret_cast<__half *>(body);
  const bool u_packed = orth(w.Y, w.U, n, r, w, st, h);       // U = orth(A Q)  (cx:411)
  const bool w_packed = aty(t, w.U, w.W, w, n, C, r, st, h ? h + n * r : nullptr);  // W = A^T U (cx:419)
  if (!int4) {
    if (!u_packed) {
      lr::k_pack_f16<<<(unsigned)cdiv(n * r, 256), 256, 0, st>>>(w.U, n, r, h);
      count_launch();
    }
    if (!w_packed) {
      lr::k_pack_f16<<<(unsigned)cdiv(C * r, 256), 256, 0, st>>>(w.W, C, r, h + n * r);
      count_launch();
    }
  } else {
    float *ranges = reinterpret_cast<float *>(body);  // 2r f32: U ranges then W ranges
    lr::k_colmax<<<r, 256, 0, st>>>(w.U, n, r, ranges);
    lr::k_colmax<<<r, 256, 0, st>>>(w.W, C, r, ranges + r);
    lr::k_pack_int4<<<(unsigned)cdiv(cdiv((n + C) * r, 2), 256), 256, 0, st>>>(w.U, w.W, n, C, r, ranges,
                                                                              ranges + r, body + 8 * r);
    count_launch(3);
  }
  if (decoded) decode_into(body, int4, n, C, r, decoded, 0, w, st);
  return cuda_status("lowrank_encode");
}

int residual_target(int mode, int64_t n, int64_t C, const void *x, int x_dtype, const float *base, const float *aux,
                    float *t, cudaStream_t st);
int gaussian_keyed(int64_t rows, int64_t cols, uint32_t *key, int nwords, int step_word, float *out, void *ws,
                   int64_t ws_bytes, cudaStream_t st);
int64_t gaussian_workspace_bytes(int64_t rows, int64_t cols);
int sum_parts(int nparts, const double *part, double *record, cudaStream_t st);
uint8_t *stream_zero_slab(cudaStream_t st, size_t bytes);
// low-rank words in the per-stream zeroed slab (after the top-k kernel's ~34 KB)
constexpr size_t kLrTicketOff = 40 * 1024;
constexpr size_t kSlabBytesNeeded = kLrTicketOff + 128;  // (lr_step.cu's words follow at +256)

// A library-owned side stream + fork / join events per (device, caller stream),
// created on first use outside a capture (null otherwise: no fork).
struct SideStream {
  cudaStream_t s;
  cudaEvent_t fork, join;
};
static SideStream *side_stream(cudaStream_t st) {
  static std::mutex mu;
  static std::unordered_map<uint64_t, SideStream> m;
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t k = (uint64_t)reinterpret_cast<uintptr_t>(st) * 64 + (uint64_t)dev;
  std::lock_guard<std::mutex> lock(mu);
  auto it = m.find(k);
  if (it != m.end()) return &it->second;
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return nullptr;
  }
  SideStream ss{};
  if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return &m.emplace(k, ss).first->second;
}

int64_t lowrank_fused_workspace_bytes(int64_t n, int64_t C, int64_t r);
bool lowrank_fused_may_run(int64_t n, int64_t C, int64_t r, int iters, int int4);
int lowrank_step_fused(int mode, int64_t n, int64_t C, int64_t r, int iters, int int4, const void *x, int x_dtype,
                       float *base, float *aux, const float *q0, uint8_t *body, void *ws, int64_t ws_bytes,
                       double *record, cudaStream_t st);

// encode_step workspace: t [n, C] | Q0 [C, r] | gaussian scratch | encode workspace |
// f64 factors [n + C, r] | record partials | fused-step workspace
static size_t lr_step_layout(int64_t n, int64_t C, int64_t r, uint8_t *w, float **t, float **q0, void **gws,
                             size_t *gbytes, void **ews, size_t *ebytes, double **Uf, double **part,
                             void **fws = nullptr, size_t *fbytes = nullptr) {
  size_t off = 0;
  auto take = [&](size_t b) {
    uint8_t *q = w ? w + off : nullptr;
    off = align_up(off + b, 256);
    return q;
  };
  const size_t gb = (size_t)gaussian_workspace_bytes(C, r);
  const size_t eb = (size_t)lowrank_workspace_bytes(n, C, r);
  const int64_t nblk = cdiv(C, lr::kThreads) * cdiv(n, lr::kOARows);
  uint8_t *pt = take(4 * (size_t)n * C), *pq = take(4 * (size_t)C * r), *pg = take(gb), *pe = take(eb);
  uint8_t *pu = take(8 * (size_t)(n + C) * r), *pp = take(16 * (size_t)nblk);
  const size_t fb = (size_t)lowrank_fused_workspace_bytes(n, C, r);
  uint8_t *pf = take(fb);
  if (w && fws) {
    *fws = pf;
    *fbytes = fb;
  }
  if (w) {
    *t = reinterpret_cast<float *>(pt);
    *q0 = reinterpret_cast<float *>(pq);
    *gws = pg;
    *gbytes = gb;
    *ews = pe;
    *ebytes = eb;
    *Uf = reinterpret_cast<double *>(pu);
    *part = reinterpret_cast<double *>(pp);
  }
  return off;
}

int64_t lowrank_step_workspace_bytes(int64_t n, int64_t C, int64_t r) {
  return (int64_t)lr_step_layout(n, C, r, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                                 nullptr);
}

// One low-rank encode_step (pipeline.py:84-121 with cx:394-426): t = target ->
// Q0 (host-drawn q0, or drawn on the device from `key`) -> subspace iteration ->
// body -> fused decode + state update + record.  Every launch is stream-ordered
// device work, so the step can be captured in a CUDA graph (with a device key).
int lowrank_encode_step(int mode, int64_t n, int64_t C, int64_t r, int iters, int int4, const void *x, int x_dtype,
                        float *base, float *aux, const float *q0_in, uint32_t *key, int nwords, int step_word,
                        uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st) {
  if ((int64_t)lr_step_layout(n, C, r, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                              nullptr) > ws_bytes) {
    set_error("low-rank step workspace too small");
    return CC_ERR_ARG;
  }
  float *t, *q0;
  void *gws, *ews, *fws;
  size_t gb, eb, fb;
  double *Uf, *part;
  lr_step_layout(n, C, r, reinterpret_cast<uint8_t *>(ws), &t, &q0, &gws, &gb, &ews, &eb, &Uf, &part, &fws, &fb);
  int rc;
  // the whole step as one persistent cluster launch (lr_step.cu) when it covers the shape
  bool drawn = false;
  if (lowrank_fused_may_run(n, C, r, iters, int4)) {
    const float *qs = q0_in;
    if (key) {
      rc = gaussian_keyed(C, r, key, nwords, step_word, q0, gws, (int64_t)gb, st);
      if (rc) return rc;
      qs = q0;
      drawn = true;
    }
    rc = lowrank_step_fused(mode, n, C, r, iters, int4, x, x_dtype, base, aux, qs, body, fws, (int64_t)fb, record, st);
    if (rc == CC_OK) return cuda_status("lowrank_encode_step (fused)");
    if (rc != 1) return rc;
  }
  // the start block depends only on the key: draw it on a side stream while the
  // target is formed (fork / join through events: also inside a graph capture)
  SideStream *ss = (key && !drawn) ? side_stream(st) : nullptr;
  if (key && ss) {
    cudaEventRecord(ss->fork, st);
    cudaStreamWaitEvent(ss->s, ss->fork, 0);
    rc = gaussian_keyed(C, r, key, nwords, step_word, q0, gws, (int64_t)gb, ss->s);
    if (rc) return rc;
    cudaEventRecord(ss->join, ss->s);
  }
  rc = residual_target(mode, n, C, x, x_dtype, base, aux, t, st);
  if (rc) return rc;
  if (key && ss) {
    cudaStreamWaitEvent(st, ss->join, 0);
  } else if (key && drawn) {
  } else if (key) {
    rc = gaussian_keyed(C, r, key, nwords, step_word, q0, gws, (int64_t)gb, st);
    if (rc) return rc;
  } else {
    q0 = const_cast<float *>(q0_in);
  }
  rc = lowrank_encode(int4, n, C, r, iters, t, q0, body, nullptr, ews, (int64_t)eb, st);
  if (rc) return rc;
  (void)Uf;
  uint8_t *slab = stream_zero_slab(st, kSlabBytesNeeded);
  unsigned int *ticket = slab ? reinterpret_cast<unsigned int *>(slab + kLrTicketOff) : nullptr;
  if (!ticket) {
    set_error("low-rank step: no control slab (first use inside a capture)");
    return CC_ERR_UNSUPPORTED;
  }
  dim3 g((unsigned)cdiv(C, lr::kThreads), (unsigned)cdiv(n, lr::kOARows));
#define CC_LA3(MODE, XT, RM)                                                                                    \
  lr::k_outer_apply<MODE, XT, RM><<<g, lr::kThreads, 0, st>>>(body, int4, n, C, (int)r, (const XT *)x, t, base, \
                                                              aux, part, ticket, record)
#define CC_LA(MODE, XT)                   \
  do {                                    \
    if (r <= 8) CC_LA3(MODE, XT, 8);      \
    else if (r <= 16) CC_LA3(MODE, XT, 16); \
    else CC_LA3(MODE, XT, 32);            \
  } while (0)
  if (x_dtype == CC_F32) {
    if (mode == CC_WITH_FEEDBACK) CC_LA(CC_WITH_FEEDBACK, float);
    else if (mode == CC_NO_FEEDBACK) CC_LA(CC_NO_FEEDBACK, float);
    else CC_LA(CC_NAIVE, float);
  } else {
    if (mode == CC_WITH_FEEDBACK) CC_LA(CC_WITH_FEEDBACK, __nv_bfloat16);
    else if (mode == CC_NO_FEEDBACK) CC_LA(CC_NO_FEEDBACK, __nv_bfloat16);
    else CC_LA(CC_NAIVE, __nv_bfloat16);
  }
#undef CC_LA
#undef CC_LA3
  count_launch();
  return cuda_status("lowrank_encode_step");
}

int lowrank_decode(int int4, int count, const int64_t *rows, int64_t C, int64_t r, const uint8_t *const *bodies,
                   int accumulate, float *const *bases, cudaStream_t st) {
  decode_batch(bodies, bases, rows, count, int4, C, (int)r, accumulate ? 1 : 0, st);
  return cuda_status("lowrank_decode");
}

}  // namespace cc
