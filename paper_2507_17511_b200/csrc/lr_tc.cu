// K3 projections on the 5th-generation tensor cores (tcgen05, kind::tf32).
//
//   mode AQ : Y[n, r]  = A[n, C] Q[C, r]        (cx:409, la:49-58)
//   mode ATY: Z[C, r]  = A[n, C]^T Y[n, r]      (cx:409, cx:419)
//
// Both are skinny (r <= 32) and stream A once, so they are HBM/L2-bound; the tensor
// cores keep the f32-accurate product off the CUDA cores.  Precision: the reference
// accumulates in f64 BLAS, so each operand is split x = hi + lo (hi = RNA-tf32(x),
// lo = tf32(x - hi)) and D += Ahi*Bhi + Ahi*Blo + Alo*Bhi ("3xTF32"), f32 accumulate
// in TMEM: ~1e-6 relative, far below the tolerance of the low-rank parity tests.
//
// CTA = 128 threads (4 warps) owning a 128-row M tile and a K range (split-K for
// parallelism; partial D tiles reduced in a fixed order).  Per 32-wide K chunk the
// warps stage hi/lo operand tiles into shared memory in the canonical K-major
// SWIZZLE_128B layout (8 rows x 128 B atoms, 16-byte chunk index XOR row), thread 0
// issues 12 tcgen05.mma (4 K-steps x 3 products) and commits to an mbarrier; two
// stage buffers let the next chunk's staging overlap the tensor-core work.  The
// epilogue moves D from TMEM with tcgen05.ld (warp w owns TMEM lanes 32w..32w+31).
#include "cc_async.cuh"
#include "cc_common.cuh"
#include "cc_internal.h"

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>

namespace cc {
namespace tc {

constexpr int kM = 128;     // UMMA M (one CTA)
constexpr int kKC = 32;     // K chunk: 32 f32 = one 128-byte swizzle row
constexpr int kThreads = 128;
constexpr int kTmemCols = 32;

// ---- tcgen05 / UMMA helpers ------------------------------------------------
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  // K-major SWIZZLE_128B: start>>4 [0,14), LBO>>4 = 1 [16,30), SBO>>4 = 1024>>4 [32,46),
  // version 1 [46,48), layout type 2 (SWIZZLE_128B) [61,64)
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFFu) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
  // c_format F32 [4,6)=1, a_format TF32 [7,10)=2, b_format TF32 [10,13)=2,
  // a/b K-major, n_dim = N>>3 [17,23), m_dim = M>>4 [24,29)
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t *dst_smem, int cols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(cols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, int cols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(cols) : "memory");
}

__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// byte offset of element (row, k) inside a K-major SWIZZLE_128B tile of 32-f32 rows
__device__ __forceinline__ uint32_t sw128(int row, int k) {
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((((k >> 2) ^ (row & 7)) & 7) << 4) + (k & 3) * 4);
}

struct Stage {
  // hi / lo operand tiles, each 1024-byte aligned
  uint8_t *a_hi, *a_lo, *b_hi, *b_lo;
};

// MODE 0 (AQ): P[m][k] = A[i0+m][k0+k], S[j][k] = Q[k0+k][j]   (K = C)
// MODE 1 (ATY): P[m][k] = A[k0+k][c0+m], S[j][k] = Y[k0+k][j]  (K = n)
//
// Software pipeline: the raw f32 operands of chunk c+1 are loaded into registers
// (8 x 128-bit A loads + NP/4 S loads per thread) right after chunk c has been
// split into hi/lo shared tiles, so the global loads fly while chunk c's sync,
// MMA issue and the wait for stage reuse go on.
constexpr int kAItems = kM * kKC / 4 / kThreads;  // 8 float4 per thread per chunk
template <int MODE, int NP>
struct Raw {
  float4 a[kAItems];
  float s[NP * kKC / kThreads];
};

// item i of thread tid -> (m, k) of its 4-element group
template <int MODE>
__device__ __forceinline__ void a_item(int tid, int i, int &m, int &k) {
  const int e = tid + i * kThreads;
  if constexpr (MODE == 0) {  // 4 consecutive k of one row: a warp reads 4 rows x 128 B
    m = e >> 3;
    k = (e & 7) * 4;
  } else {  // 4 consecutive m of one k: a warp covers 8 k x 4 m-quads (2-way smem conflicts)
    k = (e & 7) | (((e >> 5) & 3) << 3);
    m = (((e >> 3) & 3) | ((e >> 7) << 2)) * 4;
  }
}

template <int MODE, int NP>
__device__ __forceinline__ void load_raw(Raw<MODE, NP> &rw, const float *__restrict__ A, const float *__restrict__ S,
                                         int64_t m0, int64_t k0, int64_t khi, int64_t Mdim, int64_t C, int r,
                                         bool vec) {
  const int tid = threadIdx.x;
  const int kc = (int)min64(kKC, khi - k0);
#pragma unroll
  for (int i = 0; i < kAItems; ++i) {
    int m, k;
    a_item<MODE>(tid, i, m, k);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if constexpr (MODE == 0) {
      if (m0 + m < Mdim && k < kc) {
        const float *src = A + (m0 + m) * C + k0 + k;
        if (vec && k + 4 <= kc) {
          v = __ldg(reinterpret_cast<const float4 *>(src));
        } else {
          v.x = src[0];
          if (k + 1 < kc) v.y = src[1];
          if (k + 2 < kc) v.z = src[2];
          if (k + 3 < kc) v.w = src[3];
        }
      }
    } else {
      if (k < kc && m0 + m < Mdim) {
        const float *src = A + (k0 + k) * C + m0 + m;
        if (vec && m0 + m + 4 <= Mdim) {
          v = __ldg(reinterpret_cast<const float4 *>(src));
        } else {
          v.x = src[0];
          if (m0 + m + 1 < Mdim) v.y = src[1];
          if (m0 + m + 2 < Mdim) v.z = src[2];
          if (m0 + m + 3 < Mdim) v.w = src[3];
        }
      }
    }
    rw.a[i] = v;
  }
#pragma unroll
  for (int i = 0; i < NP * kKC / kThreads; ++i) {
    const int e = tid + i * kThreads;
    const int j = e / kKC, kk = e % kKC;
    rw.s[i] = (j < r && kk < kc) ? __ldg(S + (k0 + kk) * r + j) : 0.0f;
  }
}

template <int MODE, int NP>
__device__ __forceinline__ void store_split(const Raw<MODE, NP> &rw, const Stage &sg) {
  const int tid = threadIdx.x;
#pragma unroll
  for (int i = 0; i < kAItems; ++i) {
    int m, k;
    a_item<MODE>(tid, i, m, k);
    const float4 v = rw.a[i];
    const float h0 = tf32_rna(v.x), h1 = tf32_rna(v.y), h2 = tf32_rna(v.z), h3 = tf32_rna(v.w);
    const float l0 = tf32_rna(v.x - h0), l1 = tf32_rna(v.y - h1), l2 = tf32_rna(v.z - h2), l3 = tf32_rna(v.w - h3);
    if constexpr (MODE == 0) {
      const uint32_t off = sw128(m, k);
      *reinterpret_cast<float4 *>(sg.a_hi + off) = make_float4(h0, h1, h2, h3);
      *reinterpret_cast<float4 *>(sg.a_lo + off) = make_float4(l0, l1, l2, l3);
    } else {
      const float hh[4] = {h0, h1, h2, h3}, ll[4] = {l0, l1, l2, l3};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t off = sw128(m + q, k);
        *reinterpret_cast<float *>(sg.a_hi + off) = hh[q];
        *reinterpret_cast<float *>(sg.a_lo + off) = ll[q];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < NP * kKC / kThreads; ++i) {
    const int e = tid + i * kThreads;
    const int j = e / kKC, kk = e % kKC;
    const float v = rw.s[i], h = tf32_rna(v);
    const uint32_t off = sw128(j, kk);
    *reinterpret_cast<float *>(sg.b_hi + off) = h;
    *reinterpret_cast<float *>(sg.b_lo + off) = tf32_rna(v - h);
  }
  fence_proxy_async_smem();
}

template <int MODE, int NP>
__global__ void __launch_bounds__(kThreads) k_tc_gemm(const float *__restrict__ A, const float *__restrict__ S,
                                                       float *__restrict__ Dpart, int64_t n, int64_t C, int r,
                                                       int64_t kper, int vec) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-align the tile area
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t Mdim = MODE == 0 ? n : C;
  const int64_t Kdim = MODE == 0 ? C : n;
  const int64_t m0 = (int64_t)blockIdx.x * kM;
  const int split = blockIdx.y;
  const int64_t klo = split * kper, khi = min64(Kdim, klo + kper);
  constexpr uint32_t a_bytes = kM * kKC * 4;  // 16 KB
  constexpr uint32_t b_round = ((uint32_t)NP * kKC * 4 + 1023) & ~1023u;
  auto stage = [&](int s) {  // computed, not indexed: keeps the stage table out of local memory
    uint8_t *b = smem + (uint32_t)s * (2 * a_bytes + 2 * b_round);
    return Stage{b, b + a_bytes, b + 2 * a_bytes, b + 2 * a_bytes + b_round};
  };
  uint64_t *bar = reinterpret_cast<uint64_t *>(smem + 2 * (2 * a_bytes + 2 * b_round));
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 2);
  const int64_t nchunks = (khi - klo + kKC - 1) / kKC;
  Raw<MODE, NP> rw;
  if (nchunks > 0) load_raw<MODE, NP>(rw, A, S, m0, klo, khi, Mdim, C, r, vec != 0);  // overlaps the setup
  if (warp == 0) tmem_alloc(tmem_slot, kTmemCols);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = idesc_tf32(kM, NP);

  uint32_t ph = 0u;  // bit s = parity of stage s's barrier
  for (int64_t c = 0; c < nchunks; ++c) {
    const int s = (int)(c & 1);
    if (c >= 2) {  // the MMAs that read this stage two chunks ago must be done
      mbar_wait(&bar[s], (ph >> s) & 1u);
      ph ^= 1u << s;
    }
    const Stage sg = stage(s);
    store_split<MODE, NP>(rw, sg);
    if (c + 1 < nchunks) load_raw<MODE, NP>(rw, A, S, m0, klo + (c + 1) * kKC, khi, Mdim, C, r, vec != 0);
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      const uint64_t ah = umma_desc_sw128(smem_u32(sg.a_hi)), al = umma_desc_sw128(smem_u32(sg.a_lo));
      const uint64_t bh = umma_desc_sw128(smem_u32(sg.b_hi)), bl = umma_desc_sw128(smem_u32(sg.b_lo));
#pragma unroll
      for (int ks = 0; ks < kKC / 8; ++ks) {  // K = 8 tf32 (32 bytes) per instruction
        const uint64_t dk = (uint64_t)((ks * 32) >> 4);
        const uint32_t acc0 = (c > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, ah + dk, bh + dk, idesc, acc0);
        mma_tf32(tmem, ah + dk, bl + dk, idesc, 1u);
        mma_tf32(tmem, al + dk, bh + dk, idesc, 1u);
      }
      mma_commit(&bar[s]);
    }
    __syncwarp();
  }
  // drain: wait for the last (up to two) commits
  for (int64_t c = std::max<int64_t>(0, nchunks - 2); c < nchunks; ++c) {
    const int s = (int)(c & 1);
    mbar_wait(&bar[s], (ph >> s) & 1u);
    ph ^= 1u << s;
  }
  tc_fence_after();
  // epilogue: warp w reads TMEM lanes 32w..32w+31 (rows m0 + 32w + lane)
  const int64_t m = m0 + warp * 32 + lane;
  float *out = Dpart + (int64_t)split * Mdim * r;
#pragma unroll
  for (int cb = 0; cb < NP; cb += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cb, v);
    if (m < Mdim) {
#pragma unroll
      for (int q = 0; q < 16; ++q)
        if (cb + q < r) out[m * r + cb + q] = nchunks > 0 ? v[q] : 0.0f;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// ---------------------------------------------------------------------------
// TMA-staged variant (the production kernel when K % 32 == 0 and A is 16-byte
// aligned): a fifth warp streams each K chunk's raw f32 operands with 1-D bulk
// copies (cp.async.bulk, one per A row segment + one for the S rows) into a
// kRawStages-deep mbarrier ring; the four consumer warps split raw -> hi/lo into
// the SW128 MMA stages and thread 0 issues the tcgen05.mma chain as above.  The
// ring keeps ~kRawStages x 20 KB per SM in flight independent of the split work.
// ---------------------------------------------------------------------------
constexpr int kRawStages = 3;
constexpr int kMmaStages = 1;  // one hi/lo MMA stage: ~100 KB of smem, two CTAs per SM overlap each other
constexpr int kTThreads = kThreads + 32;  // + the TMA producer warp
constexpr uint32_t kRawA = kM * kKC * 4;  // 16 KB
constexpr uint32_t kRawS = 32 * kKC * 4;  // S rows of the chunk (NP <= 32)

__device__ __forceinline__ void cons_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kThreads) : "memory"); }

__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, int c0, int c1, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

template <int MODE, int NP>
__global__ void __launch_bounds__(kTThreads) k_tc_gemm_tma(const __grid_constant__ CUtensorMap amap,
                                                           const float *__restrict__ S, float *__restrict__ Dpart,
                                                           int64_t n, int64_t C, int r, int64_t kper) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t Mdim = MODE == 0 ? n : C;
  const int64_t Kdim = MODE == 0 ? C : n;
  const int64_t m0 = (int64_t)blockIdx.x * kM;
  const int split = blockIdx.y;
  const int64_t klo = split * kper, khi = min64(Kdim, klo + kper);
  constexpr uint32_t a_bytes = kM * kKC * 4;
  constexpr uint32_t b_round = ((uint32_t)NP * kKC * 4 + 1023) & ~1023u;
  auto stage = [&](int st_) {
    uint8_t *b = smem + (uint32_t)st_ * (2 * a_bytes + 2 * b_round);
    return Stage{b, b + a_bytes, b + 2 * a_bytes, b + 2 * a_bytes + b_round};
  };
  uint8_t *raw = smem + kMmaStages * (2 * a_bytes + 2 * b_round);  // [kRawStages][kRawA + kRawS]
  uint64_t *bar = reinterpret_cast<uint64_t *>(raw + kRawStages * (kRawA + kRawS));
  uint64_t *rfull = bar + 2, *rempty = rfull + kRawStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(rempty + kRawStages);
  const int64_t nchunks = (khi - klo + kKC - 1) / kKC;
  const int64_t mc = min64(kM, Mdim - m0);  // valid rows of this M tile
  if (warp == 0) tmem_alloc(tmem_slot, kTmemCols);
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    for (int q = 0; q < kRawStages; ++q) {
      mbar_init(&rfull[q], 1);
      mbar_init(&rempty[q], kThreads / 32);
    }
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == kThreads / 32) {  // ---- TMA producer warp ----
    const uint64_t pol = l2_policy_evict_first();
    for (int64_t c = 0; c < nchunks; ++c) {
      const int q = (int)(c % kRawStages);
      if (c >= kRawStages) mbar_wait(&rempty[q], (uint32_t)((c / kRawStages - 1) & 1));
      const int64_t k0 = klo + c * kKC;
      const int kc = (int)min64(kKC, khi - k0);
      uint8_t *ra = raw + (size_t)q * (kRawA + kRawS);
      // one 2-D TMA per chunk: the full box always lands (out-of-range rows zero-filled)
      if (lane == 0) {
        mbar_expect_tx(&rfull[q], kRawA + (uint32_t)(kc * r * 4));
        if constexpr (MODE == 0) tma_load_2d(ra, &amap, (int)k0, (int)m0, &rfull[q]);  // box {32 cols, 128 rows}
        else tma_load_2d(ra, &amap, (int)m0, (int)k0, &rfull[q]);                       // box {128 cols, 32 rows}
        bulk_g2s(ra + kRawA, S + k0 * r, (uint32_t)(kc * r * 4), &rfull[q], pol);
      }
    }
    return;
  }
  // ---- consumer warps 0-3 ----
  const uint32_t tmem = *tmem_slot;
  constexpr uint32_t idesc = idesc_tf32(kM, NP);
  uint32_t ph = 0u;
  for (int64_t c = 0; c < nchunks; ++c) {
    const int q = (int)(c % kRawStages);
    mbar_wait(&rfull[q], (uint32_t)((c / kRawStages) & 1));
    const int64_t k0 = klo + c * kKC;
    const int kc = (int)min64(kKC, khi - k0);
    const float *ra = reinterpret_cast<const float *>(raw + (size_t)q * (kRawA + kRawS));
    const float *rs = reinterpret_cast<const float *>(raw + (size_t)q * (kRawA + kRawS) + kRawA);
    Raw<MODE, NP> rw;
#pragma unroll
    for (int i = 0; i < kAItems; ++i) {  // raw tile -> registers (masked at the tile edges)
      int m, k;
      a_item<MODE>(tid, i, m, k);
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if constexpr (MODE == 0) {
        if (m < mc && k < kc) v = *reinterpret_cast<const float4 *>(ra + m * kKC + k);  // kc % 4 == 0
      } else {
        if (k < kc && m < mc) {  // mc % 4 == 0
          v = *reinterpret_cast<const float4 *>(ra + k * kM + m);
        }
      }
      rw.a[i] = v;
    }
#pragma unroll
    for (int i = 0; i < NP * kKC / kThreads; ++i) {
      const int e = tid + i * kThreads;
      const int j = e / kKC, kk = e % kKC;
      rw.s[i] = (j < r && kk < kc) ? rs[kk * r + j] : 0.0f;
    }
    const int st_ = (int)(c % kMmaStages);
    if (c >= kMmaStages) {  // the MMAs that read this MMA stage kMmaStages chunks ago must be done
      mbar_wait(&bar[st_], (ph >> st_) & 1u);
      ph ^= 1u << st_;
    }
    const Stage sg = stage(st_);
    store_split<MODE, NP>(rw, sg);
    __syncwarp();
    if (lane == 0) mbar_arrive(&rempty[q]);  // raw chunk consumed: the producer may refill the stage
    cons_sync();
    if (tid == 0) {
      tc_fence_after();
      const uint64_t ah = umma_desc_sw128(smem_u32(sg.a_hi)), al = umma_desc_sw128(smem_u32(sg.a_lo));
      const uint64_t bh = umma_desc_sw128(smem_u32(sg.b_hi)), bl = umma_desc_sw128(smem_u32(sg.b_lo));
#pragma unroll
      for (int ks = 0; ks < kKC / 8; ++ks) {
        const uint64_t dk = (uint64_t)((ks * 32) >> 4);
        const uint32_t acc0 = (c > 0 || ks > 0) ? 1u : 0u;
        mma_tf32(tmem, ah + dk, bh + dk, idesc, acc0);
        mma_tf32(tmem, ah + dk, bl + dk, idesc, 1u);
        mma_tf32(tmem, al + dk, bh + dk, idesc, 1u);
      }
      mma_commit(&bar[st_]);
    }
    __syncwarp();
  }
  for (int64_t c = std::max<int64_t>(0, nchunks - kMmaStages); c < nchunks; ++c) {
    const int st_ = (int)(c % kMmaStages);
    mbar_wait(&bar[st_], (ph >> st_) & 1u);
    ph ^= 1u << st_;
  }
  tc_fence_after();
  const int64_t m = m0 + warp * 32 + lane;
  float *out = Dpart + (int64_t)split * Mdim * r;
#pragma unroll
  for (int cb = 0; cb < NP; cb += 16) {
    float v[16];
    tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)cb, v);
    if (m < Mdim) {
#pragma unroll
      for (int q2 = 0; q2 < 16; ++q2)
        if (cb + q2 < r) out[m * r + cb + q2] = nchunks > 0 ? v[q2] : 0.0f;
    }
  }
  tc_fence_before();
  cons_sync();
  if (warp == 0) tmem_dealloc(tmem, kTmemCols);
}

// fixed-order split reduction -> f32 result
// (+ optionally the f16 column-major copy of D [M, r], the body factor layout cx:425)
__global__ void k_tc_reduce(const float *__restrict__ Dpart, float *__restrict__ D, int64_t cnt, int splits,
                            __half *__restrict__ d16, int r) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cnt) return;
  float s = 0.0f;
  for (int sp = 0; sp < splits; ++sp) s += Dpart[(int64_t)sp * cnt + e];
  D[e] = s;
  if (d16) d16[(e % r) * (cnt / r) + e / r] = __float2half_rn(s);
}

}  // namespace tc

static int g_lr_backend = 1;  // 1 = tcgen05 3xTF32 projections, 0 = f64 CUDA-core projections
void set_lowrank_backend(int v) { g_lr_backend = v; }
int lowrank_backend() { return g_lr_backend; }

static size_t tc_smem_bytes(int NP) {
  const size_t a = tc::kM * tc::kKC * 4;
  const size_t b = ((size_t)NP * tc::kKC * 4 + 1023) & ~size_t(1023);
  return 1024 + 2 * (2 * a + 2 * b) + 64;
}

// split-K plan: ~4 CTAs per SM (2 resident x 2 waves), >= 4 K chunks per CTA
static int tc_ctas_per_sm() {
  static const int v = [] {
    const char *e = getenv("CC_TC_CTAS_PER_SM");  // experiments
    return e ? std::max(1, atoi(e)) : 4;
  }();
  return v;
}

static void tc_plan(int64_t M, int64_t K, int64_t *splits, int64_t *kper) {
  const int64_t tiles = cdiv(M, tc::kM);
  int64_t sp = std::max<int64_t>(1, std::min<int64_t>(cdiv(tc_ctas_per_sm() * sm_count(), tiles), cdiv(K, 4 * tc::kKC)));
  *kper = cdiv(cdiv(K, sp), tc::kKC) * tc::kKC;
  *splits = cdiv(K, *kper);
}

int64_t tc_partial_floats(int64_t n, int64_t C, int r) {
  int64_t s0, s1, kp;
  tc_plan(n, C, &s0, &kp);
  tc_plan(C, n, &s1, &kp);
  return std::max(s0 * n, s1 * C) * r;
}

static size_t tc_tma_smem_bytes(int NP) {
  const size_t a = tc::kM * tc::kKC * 4;
  const size_t b = ((size_t)NP * tc::kKC * 4 + 1023) & ~size_t(1023);
  return 1024 + tc::kMmaStages * (2 * a + 2 * b) + (size_t)tc::kRawStages * (tc::kRawA + tc::kRawS) +
         8 * (2 + 2 * tc::kRawStages) + 64;
}

// 2-D tensor map over A [n, C] f32 (row-major); box {32, 128} (mode 0: K-chunk x M-tile)
// or {128, 32} (mode 1), no swizzle: the raw staging layout the consumer warps read.
// The driver entry point is fetched through the runtime (no libcuda link).
static bool make_amap(CUtensorMap *map, const float *A, int64_t n, int64_t C, int mode) {
  static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
  if (!encode) {
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void **>(&encode), cudaEnableDefault,
                                &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !encode) {
      cudaGetLastError();
      encode = nullptr;
      return false;
    }
  }
  const cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)n};
  const cuuint64_t strides[1] = {(cuuint64_t)C * 4};
  const cuuint32_t box[2] = {mode == 0 ? (cuuint32_t)tc::kKC : (cuuint32_t)tc::kM,
                             mode == 0 ? (cuuint32_t)tc::kM : (cuuint32_t)tc::kKC};
  const cuuint32_t estr[2] = {1, 1};
  return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(A), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int MODE, int NP>
static bool tc_launch_tma(dim3 grid, cudaStream_t st, const float *A, const float *S, float *Dpart, int64_t n,
                          int64_t C, int r, int64_t kper) {
  CUtensorMap map;
  if (!make_amap(&map, A, n, C, MODE)) return false;
  const size_t smem = tc_tma_smem_bytes(NP);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(tc::k_tc_gemm_tma<MODE, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr = true;
  }
  tc::k_tc_gemm_tma<MODE, NP><<<grid, tc::kTThreads, smem, st>>>(map, S, Dpart, n, C, r, kper);
  return true;
}

// 2 (default): A Q with TMA-staged raw tiles (2-D tensor map, 3-deep raw ring, one hi/lo MMA
//    stage, ~100 KB smem -> 2 CTAs per SM), A^T Y register-staged — measured 10% faster than
//    all register-staged at [1024 | 4096, 3072] r = 8 (A Q: 14.0 -> 11.3 us, 30.7 -> 24.7 us);
// 1: both TMA-staged (A^T Y 1.35x slower: its transposing split dominates); 0: both register-
//    staged.  All variants give identical results (same split-K plan).
static int g_tc_tma = 2;
void set_tc_tma(int v, int waves) {
  (void)waves;
  g_tc_tma = v;
}

template <int MODE, int NP>
static void tc_launch(dim3 grid, size_t smem, cudaStream_t st, const float *A, const float *S, float *Dpart,
                      int64_t n, int64_t C, int r, int64_t kper, int vec) {
  static int smem_set = 0;
  if ((int)smem > smem_set) {
    cudaFuncSetAttribute(tc::k_tc_gemm<MODE, NP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smem_set = (int)smem;
  }
  tc::k_tc_gemm<MODE, NP><<<grid, tc::kThreads, smem, st>>>(A, S, Dpart, n, C, r, kper, vec);
}

// D = A Q (mode 0) or A^T Y (mode 1) on the tensor cores; Dpart = scratch of tc_partial_floats()
int tc_project(int mode, const float *A, const float *S, float *D, float *Dpart, int64_t n, int64_t C, int r,
               cudaStream_t st, __half *d16) {
  const int NP = r <= 16 ? 16 : 32;
  const int64_t M = mode == 0 ? n : C, K = mode == 0 ? C : n;
  int64_t nsplit, kper;
  tc_plan(M, K, &nsplit, &kper);
  const size_t smem = tc_smem_bytes(NP);
  const int vec = (reinterpret_cast<uintptr_t>(A) & 15) == 0 && C % 4 == 0;
  // TMA path: K chunks of exactly 32 (1-D bulk copies need 16-byte sizes), aligned rows
  // TMA staging wins for A Q (row tiles, K-major already); A^T Y keeps the register path
  // (its transposing split dominates and the deeper TMA ring costs occupancy)
  const bool tma = (g_tc_tma == 1 || (g_tc_tma == 2 && mode == 0)) && vec && n % tc::kKC == 0 &&
                   C % tc::kKC == 0 && (reinterpret_cast<uintptr_t>(S) & 15) == 0;
  // (the TMA path uses the same split-K plan as the register-staged one, so both give
  // the same f32 partial sums; with one CTA resident per SM it runs in several waves)
  dim3 grid((unsigned)cdiv(M, tc::kM), (unsigned)nsplit);
  bool done = false;
  if (tma) {
    if (mode == 0) {
      done = NP == 16 ? tc_launch_tma<0, 16>(grid, st, A, S, Dpart, n, C, r, kper)
                      : tc_launch_tma<0, 32>(grid, st, A, S, Dpart, n, C, r, kper);
    } else {
      done = NP == 16 ? tc_launch_tma<1, 16>(grid, st, A, S, Dpart, n, C, r, kper)
                      : tc_launch_tma<1, 32>(grid, st, A, S, Dpart, n, C, r, kper);
    }
  }
  if (done) {
  } else if (mode == 0) {
    if (NP == 16) tc_launch<0, 16>(grid, smem, st, A, S, Dpart, n, C, r, kper, vec);
    else tc_launch<0, 32>(grid, smem, st, A, S, Dpart, n, C, r, kper, vec);
  } else {
    if (NP == 16) tc_launch<1, 16>(grid, smem, st, A, S, Dpart, n, C, r, kper, vec);
    else tc_launch<1, 32>(grid, smem, st, A, S, Dpart, n, C, r, kper, vec);
  }
  const int64_t cnt = M * r;
  tc::k_tc_reduce<<<(unsigned)cdiv(cnt, 256), 256, 0, st>>>(Dpart, D, cnt, (int)nsplit, d16, r);
  count_launch(2);
  return cuda_status("tc_project");
}

}  // namespace cc
