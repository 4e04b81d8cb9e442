// K3 fused: one low-rank encode_step (pipeline.py:84-121 with compressors.py:394-426)
// as ONE persistent cooperative launch of thread-block clusters, the residual kept
// on chip from the target to the state update.
//
//   t = target(x, base, feedback)                     (pipeline.py:98-105)
//   Q = orth(Q0);  T x { Z = A^T (A Q); Q = orth(Z) }  (cx:407-410)
//   U = orth(A Q);  W = A^T U;  body = f16(U), f16(W)  (cx:411, 419, 425)
//   d = U W^T;  base' = base + d, feedback' = t - d;  record = (||d - t||^2, ||t||^2)
//
// Geometry: clusters of kCL = 4 CTAs, one CTA per SM (the co-resident cluster count
// of a ~220 KB CTA: 33 on a B200).  Cluster c owns row band [c n / ncl, (c+1) n / ncl)
// of the shard, its CTA q the column slice [q C/4, (q+1) C/4): the CTA's block of the
// residual A = t (<= 32 rows x 768 columns at [1024, 3072]) is formed once from
// x / base / feedback and stays in shared memory in f64 for the whole step.
//   * A Q: the CTA's 16 warps split the slice's k-steps and run the f64 tensor-pipe
//     MMA (DMMA m8n8k4: exact products, f64 accumulation, like la.matmul,
//     la:49-58); the warps' partials are summed in a fixed tree, the cluster's four
//     column-slice partials through distributed shared memory, then rounded to f32
//     (la.matmul stores f32): every CTA of the cluster holds the band's rows of A Q.
//   * A^T Y: DMMA over the band's rows; each cluster writes an f64 partial of the
//     [C, r] product; the owner CTA of each block of rows sums the ncl partials in
//     cluster order and rounds to f32.
//   * orth: CholQR2 in f64 on the owners' rows (Q side: C / G rows per CTA; U side: the
//     band's rows, computed redundantly by the cluster's CTAs, each contributing a
//     quarter of the Gram): Gram partials -> grid barrier -> fixed-order sum in every
//     CTA (identical R) -> register Cholesky -> M <- M R^-1.  A degenerate pivot
//     (la:13) in any CTA is seen by all of them (same sums): CTA 0 then runs CGS2
//     with random replacement columns on the whole block (la:77-112).
// Grid barriers are flag barriers on a zeroed per-stream slab counter (cumulative
// targets, reset by the last CTA to exit, which also reduces the StepRecord).
// Same mathematics as the multi-kernel path (lowrank.cu); the projections are
// exact-product f64 here instead of 3xTF32, so the bodies agree with it and with the
// reference to the same tolerance (tests/test_gpu_lowrank.py).
#include "cc_common.cuh"
#include "cc_internal.h"
#include "lr_dev.cuh"

#include <cooperative_groups.h>
#include <cstdlib>

namespace cc {

namespace lrs {

constexpr int kCL = 4;          // CTAs per cluster = column slices of a band
constexpr int kThreads = 512;   // 16 warps
constexpr int kWarps = kThreads / 32;
constexpr int kMaxBand = 32;    // rows per band (4 MMA row tiles)
constexpr int kMaxVec = 32;     // vector rows (of Q / Z / W) owned per CTA
constexpr int kMaxKW = 16;      // k-steps per warp in A Q (C <= 4096)
constexpr int LD = 17;          // chol8_regs / chol_rinv_regs leading dimension
constexpr int kGsChunks = 14;   // Gram-partial sum: 14 x 36 threads, <= kGsPer CTAs each
constexpr int kGsPer = 12;      // (G <= 168)
constexpr double kOnePass = 100.0;  // CholQR: single pass when max R_jj < 100 min R_jj
constexpr int kTh = 3;          // quads per register half of the target pipeline
constexpr int kZPer = 20;       // clusters per half in the A^T Y reduction (ncl <= 40)

struct Params {
  int64_t n, C;
  int r, iters, ncl, nbm;  // nbm: rows of the shared-memory block (max band, multiple of 8)
  int int4;                // INT4 factors (per-column ranges, cx:556-566) instead of f16
  const void *x;
  float *base, *aux;
  const float *q0;
  uint8_t *body;
  double *record;
  double *Z64;   // [C][8] f64: the Q-side basis Z (f32-rounded values, zero beyond r)
  double *W64;   // [C][8] f64: W rows (f32-rounded values)
  float *Zg;     // [C][r] reduced Z / W (f32): CGS2 fallback input
  float *Qf;     // [C][r] CGS2 fallback output (Q side)
  float *Yg;     // [n][r] Y = A Q (f32): CGS2 fallback input (U side)
  float *Uf;     // [n][r] CGS2 fallback output (U side)
  double *Zp;    // [ncl][C][8] per-cluster partials of A^T Y
  double *Gp;    // [2][G][36] Gram partials (alternating)
  double *Rp;    // [G][2] StepRecord partials
  float *Mx;     // [2][G][8] per-CTA column maxima of |U| / |W| (INT4 ranges)
  double *M64;   // [max(n, C)][r] CGS2 scratch
  unsigned *ctl; // zeroed slab: [0] barrier counter, [32] exit counter
  unsigned long long seed;
  unsigned long long *stamps;  // profiling: [32] %globaltimer stamps of CTA 0 (may be null)
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// upper-triangle entry e (0..35) of an 8x8 symmetric matrix -> (a, b), a <= b
__device__ __forceinline__ void tri8(int e, int &a, int &b) {
  a = 0;
  int rowlen = 8;
  while (e >= rowlen) {
    e -= rowlen;
    ++a;
    --rowlen;
  }
  b = a + e;
}

// one warp, lane c < r holds column c of the Gram: right-looking Cholesky with one rsqrt
// per pivot and shuffles for row j of R (16 live registers: the kernel runs at 128);
// writes R (upper, zero elsewhere) and 1 / diag(R).  No R^-1: M R^-1 is a row-wise
// forward substitution (solve_row).
__device__ __forceinline__ void chol8_lane(const double (*G)[LD], double (*R)[LD], double *invd, int r, int *bad) {
  const int c = threadIdx.x & 31;
  double g[8];
#pragma unroll
  for (int a = 0; a < 8; ++a) g[a] = (c < r && a < r) ? G[a][c] : 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (j >= r) break;  // uniform
    double piv = __shfl_sync(0xffffffffu, g[j], j);  // Schur complement G[j][j] from lane j
    if (!(piv >= lr::kDegenerate)) {
      if (c == 0) *bad = 1;
      piv = 1.0;
    }
    const double inv = rsqrt(piv);
    const double rjc = c == j ? piv * inv : (c > j && c < r ? g[j] * inv : 0.0);  // R[j][c]
    if (c < 8) R[j][c] = rjc;
    if (c == j) invd[j] = inv;
#pragma unroll
    for (int a = j + 1; a < 8; ++a) {
      const double rja = __shfl_sync(0xffffffffu, rjc, a);  // R[j][a]
      if (a < r && c >= a && c < r) g[a] -= rja * rjc;
    }
  }
}

// x <- x R^-1 for one row (forward substitution, columns beyond r zero)
__device__ __forceinline__ void solve_row(double (&x)[8], const double (*R)[LD], const double *invd, int r) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    double s = x[c];
#pragma unroll
    for (int k = 0; k < c; ++k) s -= x[k] * R[k][c];
    x[c] = c < r ? s * invd[c] : 0.0;
  }
}

template <int MODE, typename XT>
__global__ void __launch_bounds__(kThreads, 1) k_lr_step(const Params p) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) uint8_t sm[];
  __shared__ double Gm[8][LD], Rf[2][8][LD], Rinvd[2][8];  // Gram; R and 1/diag(R) of the passes
  __shared__ double red[kWarps], coef[lr::kMaxRank], rsum[2][kWarps];
  __shared__ int bad_s, one_s, qpass;
  __shared__ float rng_s[16];  // INT4 ranges: U columns, then W columns  // qpass: CholQR passes the Q side's next product applies
  __shared__ unsigned last_s;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gq = lane >> 2, tq = lane & 3;
  const int G = (int)gridDim.x, b = (int)blockIdx.x, q = (int)cluster.block_rank(), c = b / kCL;
  const int64_t n = p.n, C = p.C;
  const int r = p.r;
  const int CS = (int)(C / kCL), S = CS + 4;  // S = 4 mod 16 doubles: conflict-free MMA fragments
  const int64_t cs0 = (int64_t)q * CS;
  // row partitions on even boundaries (the last part takes an odd remainder): an INT4
  // body byte (two consecutive rows of a factor column) is always written by one CTA
  auto even_split = [](int64_t total, int parts, int i) -> int64_t {
    return i >= parts ? total : 2 * ((int64_t)i * (total / 2) / parts);
  };
  const int64_t rb0 = even_split(n, p.ncl, c), rb1 = even_split(n, p.ncl, c + 1);
  const int nb = (int)(rb1 - rb0);
  const int64_t v0 = even_split(C, G, b), v1 = even_split(C, G, b + 1);
  const int nv = (int)(v1 - v0);
  const int u0 = (int)even_split(nb, kCL, q), u1 = (int)even_split(nb, kCL, q + 1);

  double *T = reinterpret_cast<double *>(sm);      // [nbm][S]  the residual block (f64)
  double *ysc = T + (size_t)p.nbm * S;             // [8][4][32][2] warp-tree partials
  double *yp = ysc + 8 * 4 * 64;                   // [32][8] CTA partial of A Z (read by the cluster)
  double *yb = yp + kMaxBand * 8;                  // [32][8] the band's rows of A Q / U
  double *Mv = yb + kMaxBand * 8;                  // [kMaxVec][8] owned rows of Z / W
  // scratch of the Gram sum and the A^T Y reduction: the warp-tree area (never live together)
  double(*gs)[36] = reinterpret_cast<double(*)[36]>(ysc);                       // [kGsChunks][36]
  double(*zr)[kMaxVec * 8] = reinterpret_cast<double(*)[kMaxVec * 8]>(ysc + 1024);  // [2][256]

  // grid barrier: one arrival per CTA on the slab counter (cumulative targets)
  unsigned nbar = 0;
  auto gbar = [&]() {  // (measured 1.3 us; a cluster-level arrival tree is slower: 2.0 us)
    ++nbar;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicAdd(p.ctl, 1u);
      const unsigned tgt = nbar * (unsigned)G;
      while (ld_acquire(p.ctl) < tgt) __nanosleep(16);
      __threadfence();
    }
    __syncthreads();
  };
  int nst = 0;
  auto stamp = [&]() {
    if (p.stamps && b == 0 && tid == 0 && nst < 48) p.stamps[nst] = gtimer();
    ++nst;
  };
  stamp();

  if (tid == 0 && (reinterpret_cast<uintptr_t>(p.q0 + cs0 * r) & 15) == 0)
    prefetch_l2(p.q0 + cs0 * r, (uint32_t)(CS * r * 4));  // the first A Q's B operand
  for (int e = tid; e < kMaxBand * 8; e += kThreads) yb[e] = 0.0;
  for (int64_t e = (int64_t)nb * S + tid; e < (int64_t)p.nbm * S; e += kThreads) T[e] = 0.0;

  // B fragments of the next A Z (the warp's k-steps of the slice's rows of Z64): loaded
  // right after the first Gram barrier of the Q-side orth (Z64 is complete then), so their
  // L2 round trip overlaps the Gram sum and the Cholesky
  const int KS = CS / 4, KW = KS / kWarps;  // k-steps of 4 columns: per slice, per warp
  const int ks0 = warp * KW;
  double bpre[kMaxKW];
  bool have_pre = false;
  auto preload_b = [&]() {
#pragma unroll
    for (int u = 0; u < kMaxKW; ++u) bpre[u] = u < KW ? __ldcg(p.Z64 + (cs0 + 4 * (ks0 + u) + tq) * 8 + gq) : 0.0;
    have_pre = true;
  };

  // ---- CholQR of rows M[0, nrows) x 8 (f64, row-major), Gram over rows [g0, g1): pass
  // 1 always, pass 2 when R's diagonal spread is >= kOnePass.  Leaves R (Rf[pass]) and
  // 1 / diag(R) for the passes taken (their count in np_s); returns the (grid-uniform)
  // degenerate flag.
  int gpar = 0;
  __shared__ int np_s;
  auto orth_rows = [&](double *M, int nrows, int g0, int g1, bool pre) -> bool {
    if (tid == 0) bad_s = 0;
    for (int pass = 0; pass < 2; ++pass) {
      double *gp = p.Gp + (size_t)(gpar & 1) * G * 36;
      ++gpar;
      if (tid < 36) {
        int a, bb;
        tri8(tid, a, bb);
        double s = 0.0;
        for (int i = g0; i < g1; ++i) s += M[i * 8 + a] * M[i * 8 + bb];
        gp[(size_t)b * 36 + tid] = s;
      }
      gbar();
      stamp();
      if (pre && pass == 0) preload_b();
      if (tid < kGsChunks * 36) {  // fixed-order sum of the G partials: chunks of CTAs, then the chunks
        const int e = tid % 36, h = tid / 36;
        const int k0 = h * G / kGsChunks, k1 = (h + 1) * G / kGsChunks;
        double v[kGsPer];
#pragma unroll
        for (int u = 0; u < kGsPer; ++u) v[u] = k0 + u < k1 ? __ldcg(gp + (size_t)(k0 + u) * 36 + e) : 0.0;
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < kGsPer; ++u) s += v[u];
        gs[h][e] = s;
      }
      for (int e = tid; e < 8 * LD; e += kThreads) Rf[pass][e / LD][e % LD] = 0.0;
      __syncthreads();
      if (tid < 36) {
        double s = 0.0;
#pragma unroll
        for (int h = 0; h < kGsChunks; ++h) s += gs[h][tid];
        int a, bb;
        tri8(tid, a, bb);
        Gm[a][bb] = s;
        Gm[bb][a] = s;
      }
      __syncthreads();
      if (warp == 0) {
        chol8_lane(Gm, Rf[pass], Rinvd[pass], r, &bad_s);
        __syncwarp();
        if (pass == 0 && lane == 0) {  // R's diagonal spread bounds kappa: CholQR's loss of
          double mx = 0.0, mn = 1e300;  // orthogonality ~ eps kappa^2 is below f32 rounding for a
          for (int j = 0; j < r; ++j) {  // spread < kOnePass: the second pass is skipped (uniform)
            mx = fmax(mx, Rf[0][j][j]);
            mn = fmin(mn, Rf[0][j][j]);
          }
          one_s = mx < kOnePass * mn;
          np_s = one_s ? 1 : 2;
        }
      }
      __syncthreads();
      stamp();
      if (tid < nrows) {  // M <- M R^-1, one row per thread
        double x[8];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const double2 v = *reinterpret_cast<const double2 *>(M + tid * 8 + k);
          x[k] = v.x;
          x[k + 1] = v.y;
        }
        solve_row(x, Rf[pass], Rinvd[pass], r);
#pragma unroll
        for (int k = 0; k < 8; k += 2) *reinterpret_cast<double2 *>(M + tid * 8 + k) = make_double2(x[k], x[k + 1]);
      }
      __syncthreads();
      if (pass == 0 && one_s) break;  // uniform
    }
    return bad_s != 0;
  };

  // ---- Q side: Q = Z R1^-1 [R2^-1] is never materialised: the owners factor the Gram of
  // their rows of Z (Z64 / Zg already published), every CTA holds the same R's and the
  // next A Q is computed as (A Z) R1^-1 [R2^-1] row by row.  Fallback: CTA 0's CGS2
  // replaces Z64 by the orthonormal Q (from src, the f32 matrix), no solve.
  int salt = 0;
  auto orth_q = [&](const float *src) {
    const bool bad = orth_rows(Mv, nv, 0, nv, true);
    if (tid == 0) qpass = bad ? 0 : np_s;
    if (bad) {  // uniform (Z64 is rewritten: the preloaded fragments are stale)
      have_pre = false;
      if (b == 0) {
        lr::cgs2_block(src, p.M64, p.Qf, C, r, p.seed + 7919ull * (unsigned)salt, red, coef);
        __syncthreads();
        for (int64_t e = tid; e < C * 8; e += kThreads) {
          const int k = (int)(e & 7);
          p.Z64[e] = k < r ? (double)p.Qf[(e >> 3) * r + k] : 0.0;
        }
      }
      gbar();
    }
    ++salt;
    __syncthreads();
  };

  // ---- yb <- f32((A Z) R1^-1 [R2^-1]) for the band (rows < nb), every CTA of the cluster
  const int MT = (nb + 7) / 8;
  auto y_phase = [&](bool from_q0) {
    double acc[4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m) acc[m][0] = acc[m][1] = 0.0;
    double bq[kMaxKW];  // the warp's B fragments (Z rows of its k-steps), all loads in flight
    if (have_pre && !from_q0) {  // loaded during the orth (the fallback rewrote Z64: reload)
#pragma unroll
      for (int u = 0; u < kMaxKW; ++u) bq[u] = bpre[u];
    } else if (from_q0) {
#pragma unroll
      for (int u = 0; u < kMaxKW; ++u)
        bq[u] = (u < KW && gq < r) ? (double)__ldg(p.q0 + (cs0 + 4 * (ks0 + u) + tq) * r + gq) : 0.0;
    } else {
#pragma unroll
      for (int u = 0; u < kMaxKW; ++u) bq[u] = u < KW ? __ldcg(p.Z64 + (cs0 + 4 * (ks0 + u) + tq) * 8 + gq) : 0.0;
    }
    have_pre = false;
#pragma unroll
    for (int u = 0; u < kMaxKW; ++u) {
      if (u >= KW) break;
      const int col = 4 * (ks0 + u) + tq;
#pragma unroll
      for (int m = 0; m < 4; ++m)
        if (m < MT) lr::dmma884(acc[m][0], acc[m][1], T[(size_t)(8 * m + gq) * S + col], bq[u]);
    }
    // warp tree: 16 -> 8 -> 4 -> 2 -> 1 (fixed order)
    for (int half = kWarps / 2; half >= 1; half >>= 1) {
      if (warp >= half && warp < 2 * half) {
        double *o = ysc + (size_t)(warp - half) * 256;
#pragma unroll
        for (int m = 0; m < 4; ++m)
          *reinterpret_cast<double2 *>(o + m * 64 + 2 * lane) = make_double2(acc[m][0], acc[m][1]);
      }
      __syncthreads();
      if (warp < half) {
        const double *o = ysc + (size_t)warp * 256;
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const double2 v = *reinterpret_cast<const double2 *>(o + m * 64 + 2 * lane);
          acc[m][0] += v.x;
          acc[m][1] += v.y;
        }
      }
      if (half > 1) __syncthreads();
    }
    if (warp == 0) {
#pragma unroll
      for (int m = 0; m < 4; ++m) {
        const int row = 8 * m + gq;
        *reinterpret_cast<double2 *>(yp + row * 8 + 2 * tq) = make_double2(acc[m][0], acc[m][1]);
      }
    }
    cluster.sync();  // the four column-slice partials of the band are published
    if (tid < nb * 8) {
      double yz = 0.0;
#pragma unroll
      for (int qq = 0; qq < kCL; ++qq) yz += cluster.map_shared_rank(yp, qq)[tid];
      yb[tid] = yz;
    }
    __syncthreads();
    if (tid < nb) {  // (A Z) R1^-1 [R2^-1], rounded to f32 (la.matmul stores f32)
      double x[8];
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const double2 v = *reinterpret_cast<const double2 *>(yb + tid * 8 + k);
        x[k] = v.x;
        x[k + 1] = v.y;
      }
      if (qpass >= 1) solve_row(x, Rf[0], Rinvd[0], r);
      if (qpass >= 2) solve_row(x, Rf[1], Rinvd[1], r);
#pragma unroll
      for (int k = 0; k < 8; k += 2)
        *reinterpret_cast<double2 *>(yb + tid * 8 + k) = make_double2((double)(float)x[k], (double)(float)x[k + 1]);
    }
    __syncthreads();
  };

  // ---- Zp[c][cs0 + j][k] = sum over the band's rows of A[row][j] * yb[row][k]
  auto z_phase = [&]() {
    const int KR = (nb + 3) / 4;
    double bfr[8];
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) bfr[ks] = ks < KR ? yb[(4 * ks + tq) * 8 + gq] : 0.0;
    double *zp = p.Zp + ((size_t)c * C + cs0) * 8;
    const int MTZ = CS / 8;
    for (int mt = warp; mt < MTZ; mt += 2 * kWarps) {  // two column tiles in flight
      const bool two = mt + kWarps < MTZ;
      double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        if (ks >= KR) break;
        const double *tr = T + (size_t)(4 * ks + tq) * S + gq;
        lr::dmma884(d0, d1, tr[8 * mt], bfr[ks]);
        if (two) lr::dmma884(e0, e1, tr[8 * (mt + kWarps)], bfr[ks]);
      }
      *reinterpret_cast<double2 *>(zp + (size_t)(8 * mt + gq) * 8 + 2 * tq) = make_double2(d0, d1);
      if (two) *reinterpret_cast<double2 *>(zp + (size_t)(8 * (mt + kWarps) + gq) * 8 + 2 * tq) = make_double2(e0, e1);
    }
  };

  // ---- owners: Mv = f32(sum over clusters of Zp) for rows [v0, v1) (two halves of the
  // clusters per value, all loads in flight); published as Z64 (f64) and Zg (f32)
  auto z_reduce = [&](double *out64) {
    {
      const int e = tid & 255, h = tid >> 8;
      const int c0 = h * p.ncl / 2, c1 = (h + 1) * p.ncl / 2;
      double s = 0.0;
      if (e < nv * 8) {
        const double *zp = p.Zp + (v0 + (e >> 3)) * 8 + (e & 7);
        double v[kZPer];
#pragma unroll
        for (int u = 0; u < kZPer; ++u) v[u] = c0 + u < c1 ? __ldcg(zp + (size_t)(c0 + u) * C * 8) : 0.0;
#pragma unroll
        for (int u = 0; u < kZPer; ++u) s += v[u];
      }
      zr[h][e] = s;
    }
    __syncthreads();
    if (tid < nv * 8) {
      const int k = tid & 7;
      const int64_t i = v0 + (tid >> 3);
      const float f = (float)(zr[0][tid] + zr[1][tid]);
      Mv[tid] = (double)f;
      out64[i * 8 + k] = (double)f;
      if (k < r) p.Zg[i * r + k] = f;
    }
    __syncthreads();
  };

  // ---- orth(Q0) (cx:407) is not formed: QR is invariant under a right factor that is
  // upper triangular (orth(M R^-1) = orth(M)), so orth(A^T A orth(Q0)) = orth(A^T A Q0)
  // and the first product reads the Gaussian block itself (no solve).  Q0 is well
  // conditioned (never degenerate), so the only difference is rounding.
  if (tid == 0) qpass = 0;

  // ---- the residual block: t = target(x, base, feedback) -> f64 in shared memory.
  // Software-pipelined in register halves of kTh quads: the loads of one half are in
  // flight while the other half is converted and stored.
  double tsq = 0.0;
  {
    const int QR = CS / 4;  // quads per row
    const int nq = nb * QR;
    struct Half {
      float4 x[kTh], b[kTh], a[kTh];
    } hv[2];
    auto load = [&](Half &H, int e0) {
#pragma unroll
      for (int u = 0; u < kTh; ++u) {
        const int e = e0 + u * kThreads;
        H.x[u] = H.b[u] = H.a[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e < nq) {
          const int64_t g = (rb0 + e / QR) * C + cs0 + 4 * (e % QR);
          H.x[u] = Act<XT>::load4(reinterpret_cast<const XT *>(p.x) + g);
          if (MODE == CC_WITH_FEEDBACK) H.b[u] = __ldcs(reinterpret_cast<const float4 *>(p.base + g));
          if (MODE != CC_NAIVE) H.a[u] = __ldcs(reinterpret_cast<const float4 *>(p.aux + g));
        }
      }
    };
    auto store = [&](const Half &H, int e0) {
#pragma unroll
      for (int u = 0; u < kTh; ++u) {
        const int e = e0 + u * kThreads;
        if (e < nq) {
          const double t0 = target_of<MODE>(H.x[u].x, H.b[u].x, H.a[u].x);
          const double t1 = target_of<MODE>(H.x[u].y, H.b[u].y, H.a[u].y);
          const double t2 = target_of<MODE>(H.x[u].z, H.b[u].z, H.a[u].z);
          const double t3 = target_of<MODE>(H.x[u].w, H.b[u].w, H.a[u].w);
          double *d = T + (size_t)(e / QR) * S + 4 * (e % QR);
          *reinterpret_cast<double2 *>(d) = make_double2(t0, t1);
          *reinterpret_cast<double2 *>(d + 2) = make_double2(t2, t3);
          tsq += t0 * t0 + t1 * t1 + t2 * t2 + t3 * t3;
        }
      }
    };
    const int step = kTh * kThreads;
    load(hv[0], tid);
    load(hv[1], tid + step);
    for (int e0 = tid; e0 < nq; e0 += 2 * step) {
      store(hv[0], e0);
      if (e0 + 2 * step < nq) load(hv[0], e0 + 2 * step);
      store(hv[1], e0 + step);
      if (e0 + 3 * step < nq) load(hv[1], e0 + 3 * step);
    }
  }
  __syncthreads();
  stamp();

  // ---- subspace iteration
  for (int it = 0; it < p.iters; ++it) {
    y_phase(it == 0);
    stamp();
    z_phase();
    stamp();
    gbar();  // every cluster's partial of A^T (A Q)
    stamp();
    z_reduce(p.Z64);
    stamp();
    orth_q(p.Zg);
    stamp();
  }

  // ---- U = orth(A Q) on the band (Gram quarter per CTA), body U
  y_phase(false);
  if (MODE != CC_NAIVE && tid < nb) {  // the state update's rows: into L2 while U / W form
    const int64_t e = (rb0 + tid) * C + cs0;
    prefetch_l2(p.base + e, (uint32_t)(CS * 4));
    if (MODE == CC_NO_FEEDBACK) prefetch_l2(reinterpret_cast<const XT *>(p.x) + e, (uint32_t)(CS * sizeof(XT)));
  }
  for (int e = tid; e < (u1 - u0) * 8; e += kThreads) {  // Y rows for the fallback
    const int i = u0 + (e >> 3), k = e & 7;
    if (k < r) p.Yg[(rb0 + i) * r + k] = (float)yb[i * 8 + k];
  }
  // the last reads of the cluster peers' shared memory are done: no CTA of the cluster
  // may exit before every peer has passed this point (waited on at the end)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  const bool ubad = orth_rows(yb, nb, u0, u1, false);
  if (ubad) {  // uniform: every CTA factored the same Gram
    if (b == 0) lr::cgs2_block(p.Yg, p.M64, p.Uf, n, r, p.seed + 104729ull, red, coef);
    gbar();
    if (tid < nb * 8) {
      const int i = tid >> 3, k = tid & 7;
      yb[tid] = k < r ? (double)__ldcg(p.Uf + (rb0 + i) * r + k) : 0.0;
    }
    __syncthreads();
  } else if (tid < nb * 8) {
    yb[tid] = (double)(float)yb[tid];  // U is f32 (la:112)
  }
  __syncthreads();
  __half *h = reinterpret_cast<__half *>(p.body);
  if (!p.int4) {
    for (int e = tid; e < (u1 - u0) * r; e += kThreads) {  // body U: column-major f16 (cx:425)
      const int k = e / (u1 - u0), i = u0 + e % (u1 - u0);
      h[(int64_t)k * n + rb0 + i] = __float2half_rn((float)yb[i * 8 + k]);
    }
  } else if (tid < 8) {  // |U| column maxima of this CTA's quarter of the band (cx:559)
    float mx = 0.0f;
    for (int i = u0; i < u1; ++i) mx = fmaxf(mx, fabsf((float)yb[i * 8 + tid]));
    p.Mx[(size_t)b * 8 + tid] = mx;
  }
  stamp();

  // ---- W = A^T U -> body W; published for the state update
  z_phase();
  gbar();
  z_reduce(p.W64);
  if (!p.int4) {
    for (int e = tid; e < nv * r; e += kThreads) {
      const int i = e % nv, k = e / nv;
      h[n * r + (int64_t)k * C + v0 + i] = __float2half_rn((float)Mv[i * 8 + k]);
    }
    for (int e = tid; e < nb * 8; e += kThreads) yb[e] = (double)__double2half(yb[e]);
  } else if (tid < 8) {  // |W| column maxima of the owned rows
    float mx = 0.0f;
    for (int i = 0; i < nv; ++i) mx = fmaxf(mx, fabsf((float)Mv[i * 8 + tid]));
    p.Mx[(size_t)(G + b) * 8 + tid] = mx;
  }
  gbar();  // W (and the INT4 column maxima) visible
  if (p.int4) {
    // ranges = max over every CTA's maxima (order-free: identical in every CTA)
    if (tid < 16) {
      const float *mx = p.Mx + (size_t)(tid >> 3) * G * 8 + (tid & 7);
      float v = 0.0f;
      for (int i = 0; i < G; ++i) v = fmaxf(v, __ldcg(mx + (size_t)i * 8));
      rng_s[tid] = v;
      if (b == 0 && (tid & 7) < r) reinterpret_cast<float *>(p.body)[(tid >> 3) * r + (tid & 7)] = v;
    }
    __syncthreads();
    uint8_t *nib = p.body + 8 * r;
    for (int e = tid; e < ((u1 - u0 + 1) >> 1) * r; e += kThreads) {  // U codes, two rows per byte
      const int pr = (u1 - u0 + 1) >> 1;
      const int k = e / pr, i = u0 + 2 * (e % pr);
      uint32_t byte = lr::int4_code((float)yb[i * 8 + k], rng_s[k]);
      if (i + 1 < u1) byte |= lr::int4_code((float)yb[(i + 1) * 8 + k], rng_s[k]) << 4;
      nib[((int64_t)k * n + rb0 + i) >> 1] = (uint8_t)byte;
    }
    for (int e = tid; e < ((nv + 1) >> 1) * r; e += kThreads) {  // W codes of the owned rows
      const int pr = (nv + 1) >> 1;
      const int k = e / pr, i = 2 * (e % pr);
      uint32_t byte = lr::int4_code((float)Mv[i * 8 + k], rng_s[8 + k]);
      if (i + 1 < nv) byte |= lr::int4_code((float)Mv[(i + 1) * 8 + k], rng_s[8 + k]) << 4;
      nib[(n * r + (int64_t)k * C + v0 + i) >> 1] = (uint8_t)byte;
    }
    __syncthreads();  // the U codes above read yb
    for (int e = tid; e < nb * 8; e += kThreads) {  // the band's U as the receiver decodes it
      const int k = e & 7;
      yb[e] = k < r ? lr::int4_value(lr::int4_code((float)yb[e], rng_s[k]), rng_s[k]) : 0.0;
    }
    __syncthreads();
  }
  stamp();

  // ---- state update from the body's factors (the receiver's k_lr_decode arithmetic):
  // thread = 2 columns of the slice, every row of the band
  double err = 0.0;
  if (tid < CS / 2) {
    const int j0 = 2 * tid;
    double w[2][8];  // f16(W) of the two columns, as the receiver decodes them
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double *wr = p.W64 + (cs0 + j0 + j) * 8;
#pragma unroll
      for (int k = 0; k < 8; k += 2) {
        const double2 v = __ldcg(reinterpret_cast<const double2 *>(wr + k));
        if (p.int4) {
          w[j][k] = k < r ? lr::int4_value(lr::int4_code((float)v.x, rng_s[8 + k]), rng_s[8 + k]) : 0.0;
          w[j][k + 1] = k + 1 < r ? lr::int4_value(lr::int4_code((float)v.y, rng_s[9 + k]), rng_s[9 + k]) : 0.0;
        } else {
          w[j][k] = (double)__double2half(v.x);
          w[j][k + 1] = (double)__double2half(v.y);
        }
      }
    }
    for (int row0 = 0; row0 < nb; row0 += 4) {
      float2 bbv[4], xxv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {  // the loads of 4 rows in flight
        const int row = row0 + u;
        bbv[u] = xxv[u] = make_float2(0.f, 0.f);
        if (row < nb) {
          const int64_t g = (rb0 + row) * C + cs0 + j0;
          if (MODE != CC_NAIVE) bbv[u] = __ldcs(reinterpret_cast<const float2 *>(p.base + g));
          if (MODE == CC_NO_FEEDBACK) {
            const XT *xp = reinterpret_cast<const XT *>(p.x) + g;
            xxv[u] = make_float2(Act<XT>::load1(xp), Act<XT>::load1(xp + 1));
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int row = row0 + u;
        if (row >= nb) break;
        const int64_t g = (rb0 + row) * C + cs0 + j0;
        double uu[8];
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
          const double2 v = *reinterpret_cast<const double2 *>(yb + row * 8 + k);
          uu[k] = v.x;
          uu[k + 1] = v.y;
        }
        const double2 tv = *reinterpret_cast<const double2 *>(T + (size_t)row * S + j0);
        float dd[2], tt[2];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          double s = 0.0;  // k_lr_decode's order: k = 0 .. r-1
#pragma unroll
          for (int k = 0; k < 8; ++k)
            if (k < r) s += uu[k] * w[j][k];
          dd[j] = (float)s;
          const double t64 = j == 0 ? tv.x : tv.y;
          tt[j] = (float)t64;
          const double df = (double)dd[j] - t64;
          err += df * df;
        }
        if (MODE == CC_NAIVE) {
          __stcs(reinterpret_cast<float2 *>(p.base + g), make_float2(dd[0], dd[1]));
        } else {
          const float2 bb = bbv[u];
          __stcs(reinterpret_cast<float2 *>(p.base + g), make_float2(__fadd_rn(bb.x, dd[0]), __fadd_rn(bb.y, dd[1])));
          const float2 naux = MODE == CC_WITH_FEEDBACK ? make_float2(__fsub_rn(tt[0], dd[0]), __fsub_rn(tt[1], dd[1]))
                                                       : xxv[u];
          __stcs(reinterpret_cast<float2 *>(p.aux + g), naux);
        }
      }
    }
  }
  stamp();
  // ---- StepRecord: CTA partials, the last CTA to leave sums them in CTA order
  err = warp_sum(err);
  tsq = warp_sum(tsq);
  if (lane == 0) {
    rsum[0][warp] = err;
    rsum[1][warp] = tsq;
  }
  __syncthreads();
  if (tid == 0) {
    double a = 0.0, bb = 0.0;
    for (int w = 0; w < kWarps; ++w) {
      a += rsum[0][w];
      bb += rsum[1][w];
    }
    p.Rp[2 * b] = a;
    p.Rp[2 * b + 1] = bb;
    __threadfence();
    last_s = atomicAdd(p.ctl + 32, 1u) == (unsigned)G - 1;
  }
  __syncthreads();
  if (last_s) {
    __threadfence();
    double a = 0.0, bb = 0.0;
    for (int i = tid; i < G; i += kThreads) {
      a += __ldcg(p.Rp + 2 * i);
      bb += __ldcg(p.Rp + 2 * i + 1);
    }
    a = warp_sum(a);
    bb = warp_sum(bb);
    if (lane == 0) {
      rsum[0][warp] = a;
      rsum[1][warp] = bb;
    }
    __syncthreads();
    if (tid == 0) {
      double x0 = 0.0, y0 = 0.0;
      for (int w = 0; w < kWarps; ++w) {
        x0 += rsum[0][w];
        y0 += rsum[1][w];
      }
      p.record[0] = x0;
      p.record[1] = y0;
      p.ctl[0] = 0u;  // every CTA has passed its last barrier: the slab words are zero again
      p.ctl[32] = 0u;
    }
  }
  stamp();
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

size_t smem_bytes(int nbm, int64_t C) {
  const int S = (int)(C / kCL) + 4;
  return sizeof(double) * ((size_t)nbm * S + 8 * 4 * 64 + 2 * kMaxBand * 8 + kMaxVec * 8);
}

}  // namespace lrs

uint8_t *stream_zero_slab(cudaStream_t st, size_t bytes);
constexpr size_t kLrsCtlOff = 40 * 1024 + 256;  // after the low-rank ticket (40 KB), before the Gaussian's (44 KB)

static int g_lrs_enable = 1;
static int64_t g_lrs_launches = 0;
static unsigned long long *g_lrs_stamps = nullptr;
void set_lowrank_fused(int on) { g_lrs_enable = on; }
int64_t lowrank_fused_launches() { return g_lrs_launches; }
void set_lowrank_fused_stamps(void *buf) { g_lrs_stamps = reinterpret_cast<unsigned long long *>(buf); }

static size_t lrs_layout(int64_t n, int64_t C, int64_t r, int ncl, uint8_t *w, lrs::Params *p) {
  size_t off = 0;
  auto take = [&](size_t sz) {
    uint8_t *q = w ? w + off : nullptr;
    off = align_up(off + sz, 256);
    return q;
  };
  const int G = ncl * lrs::kCL;
  const int64_t m = std::max(n, C);
  uint8_t *qg = take(8 * C * 8), *wg = take(8 * C * 8), *zg = take(4 * C * r), *qf = take(4 * C * r), *yg = take(4 * n * r),
          *uf = take(4 * n * r), *zp = take(8 * (size_t)ncl * C * 8), *gp = take(8 * 2 * (size_t)G * 36),
          *rp = take(16 * (size_t)G), *m64 = take(8 * m * r), *mx = take(4 * 2 * (size_t)G * 8);
  if (w && p) {
    p->Z64 = reinterpret_cast<double *>(qg);
    p->W64 = reinterpret_cast<double *>(wg);
    p->Zg = reinterpret_cast<float *>(zg);
    p->Qf = reinterpret_cast<float *>(qf);
    p->Yg = reinterpret_cast<float *>(yg);
    p->Uf = reinterpret_cast<float *>(uf);
    p->Zp = reinterpret_cast<double *>(zp);
    p->Gp = reinterpret_cast<double *>(gp);
    p->Rp = reinterpret_cast<double *>(rp);
    p->M64 = reinterpret_cast<double *>(m64);
    p->Mx = reinterpret_cast<float *>(mx);
  }
  return off;
}

constexpr int kLrsMaxClusters = 40;
int64_t lowrank_fused_workspace_bytes(int64_t n, int64_t C, int64_t r) {
  return (int64_t)lrs_layout(n, C, r, kLrsMaxClusters, nullptr, nullptr);
}

template <int MODE, typename XT>
static const void *lrs_kernel() {
  return (const void *)lrs::k_lr_step<MODE, XT>;
}

static const void *lrs_pick(int mode, int x_dtype) {
  if (x_dtype == CC_F32) {
    if (mode == CC_WITH_FEEDBACK) return lrs_kernel<CC_WITH_FEEDBACK, float>();
    if (mode == CC_NO_FEEDBACK) return lrs_kernel<CC_NO_FEEDBACK, float>();
    return lrs_kernel<CC_NAIVE, float>();
  }
  if (mode == CC_WITH_FEEDBACK) return lrs_kernel<CC_WITH_FEEDBACK, __nv_bfloat16>();
  if (mode == CC_NO_FEEDBACK) return lrs_kernel<CC_NO_FEEDBACK, __nv_bfloat16>();
  return lrs_kernel<CC_NAIVE, __nv_bfloat16>();
}

bool lowrank_fused_may_run(int64_t n, int64_t C, int64_t r, int iters, int int4) {
  // INT4 bodies pack two consecutive entries of a factor column per byte: with n even every
  // byte stays inside one CTA's rows (odd n: the multi-kernel step)
  return g_lrs_enable && r >= 1 && r <= 8 && iters >= 1 && C % (lrs::kCL * 64) == 0 && n >= 8 &&
         !(int4 && (n & 1));
}

// Returns CC_OK after launching the fused step, 1 when the shape / options are not
// covered (the caller runs the multi-kernel step), or an error code.
int lowrank_step_fused(int mode, int64_t n, int64_t C, int64_t r, int iters, int int4, const void *x, int x_dtype,
                       float *base, float *aux, const float *q0, uint8_t *body, void *ws, int64_t ws_bytes,
                       double *record, cudaStream_t st) {
  if (!lowrank_fused_may_run(n, C, r, iters, int4) || (x_dtype != CC_F32 && x_dtype != CC_BF16)) return 1;
  const uintptr_t al = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(base) |
                       reinterpret_cast<uintptr_t>(aux) | reinterpret_cast<uintptr_t>(body);
  if (al & 15) return 1;
  const void *kern = lrs_pick(mode, x_dtype);
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return 1;
  // co-resident clusters at the largest block (kMaxBand rows); smaller bands only use less
  // (per kernel instance and shared-memory size: a narrower slice fits more CTAs per SM)
  static int ncl_cache[64][8] = {};
  static size_t ncl_smem[64][8] = {};
  const size_t smax = lrs::smem_bytes(lrs::kMaxBand, C);
  if (smax > 227 * 1024 - 10 * 1024) return 1;
  const int slot = (mode & 3) * 2 + (x_dtype == CC_F32);
  if (ncl_smem[dev][slot] != smax) {
    ncl_cache[dev][slot] = 0;
    ncl_smem[dev][slot] = smax;
  }
  int &ncl = ncl_cache[dev][slot];
  if (ncl == 0) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smax) != cudaSuccess) {
      cudaGetLastError();
      ncl = -1;
      return 1;
    }
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = lrs::kCL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(lrs::kThreads);
    cfg.gridDim = dim3(lrs::kCL * 8);
    cfg.dynamicSmemBytes = smax;
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      mc = -1;
    }
    ncl = mc > 0 ? std::min(mc, kLrsMaxClusters) : -1;
  }
  if (ncl < 1) return 1;
  const int G = ncl * lrs::kCL;
  // the kernel's even row partitions (bands of n over the clusters, vector rows of C over the CTAs)
  auto max_part = [](int64_t total, int parts) {
    int64_t mx = 0;
    for (int i = 0; i < parts; ++i) {
      const int64_t a = i >= parts ? total : 2 * ((int64_t)i * (total / 2) / parts);
      const int64_t b = i + 1 >= parts ? total : 2 * ((int64_t)(i + 1) * (total / 2) / parts);
      mx = std::max(mx, b - a);
    }
    return mx;
  };
  const int64_t band = max_part(n, ncl);
  const int nbm = (int)(8 * cdiv(band, 8));
  if (nbm > lrs::kMaxBand || n < (int64_t)ncl * 8 || max_part(C, G) > lrs::kMaxVec) return 1;
  const size_t smem = lrs::smem_bytes(nbm, C);
  if ((int64_t)lrs_layout(n, C, r, ncl, nullptr, nullptr) > ws_bytes) return 1;
  uint8_t *slab = stream_zero_slab(st, kLrsCtlOff + 256);
  if (!slab) return 1;
  lrs::Params p{};
  p.n = n;
  p.C = C;
  p.r = (int)r;
  p.iters = iters;
  p.int4 = int4;
  p.ncl = ncl;
  p.nbm = nbm;
  p.x = x;
  p.base = base;
  p.aux = aux;
  p.q0 = q0;
  p.body = body;
  p.record = record;
  lrs_layout(n, C, r, ncl, reinterpret_cast<uint8_t *>(ws), &p);
  p.ctl = reinterpret_cast<unsigned *>(slab + kLrsCtlOff);
  static unsigned long long seed = 0x1a2b3c4dULL;
  p.seed = seed++;
  p.stamps = g_lrs_stamps;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(lrs::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = lrs::kCL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  // CC_LRS_NONCOOP=1 (profiling only: ncu cannot replay a cooperative cluster launch):
  // the same grid without the co-residency check (it fits an otherwise idle GPU)
  static const bool noncoop = getenv("CC_LRS_NONCOOP") && atoi(getenv("CC_LRS_NONCOOP")) == 1;
  cfg.numAttrs = noncoop ? 1 : 2;
  void *args[] = {&p};
  const cudaError_t e = cudaLaunchKernelExC(&cfg, kern, args);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return 1;
  }
  count_launch();
  ++g_lrs_launches;
  return CC_OK;
}

}  // namespace cc
