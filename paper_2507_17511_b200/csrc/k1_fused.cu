// K1, persistent form: ONE cooperative kernel per encode_step for the 1/2/4-bit
// codecs on row strips of 1024 columns (C % 1024 == 0, e.g. FLUX's 3072).
//
//   phase A  stream (x, base, aux) tiles global->smem with cp.async.bulk (1-D TMA)
//            on a multi-stage mbarrier ring fed by a producer warp; 8 consumer
//            warps form t = target(x, base, aux) (pipeline.py:99-104) and
//            accumulate |t| in f64: column partials in registers (each CTA owns
//            a fixed strip), row partials per tile through shared memory.
//   grid.sync
//   phase F1 column sums -> v_j = colmean (f32), row sums, per-CTA row-sum partials
//   grid.sync
//   phase F2 g = mean|t| (identical fixed-order tree in every CTA),
//            u_i = max(rowmean_i / g, 1e-30) (compressors.py:135-149)
//   grid.sync
//   phase B  stream the SAME tiles in reverse order (the tail of phase A is
//            still L2-resident; phase-A loads carry L2::evict_last, phase-B loads
//            evict_first), quantize (compressors.py:373-391), pack codes, write
//            base' / feedback' / ref' with streaming stores (pipeline.py:107-113),
//            StepRecord partials -> last-CTA ticket reduction (pipeline.py:115-120).
//
// Results are bit-identical to the multi-kernel path in quant.cu (same f64
// reduction trees per element group, same code/decode arithmetic); the parity
// tests run both.
#include <cooperative_groups.h>

#include "cc_async.cuh"
#include "cc_common.cuh"
#include "cc_internal.h"

#include <algorithm>

namespace cg = cooperative_groups;

namespace cc {
namespace fused {

constexpr int kGroupThreads = 256;  // one row group: 8 warps x 32 lanes x 4 columns = 1024-column strip
constexpr int kGroups = 2;          // row groups (alternate rows of a tile) -> 16 consumer warps
constexpr int kGWarps = kGroupThreads / 32;
constexpr int kConsumers = kGroups * kGroupThreads;
constexpr int kCWarps = kConsumers / 32;
constexpr int kThreads = kConsumers + 32;  // + producer warp
constexpr int kStrip = 4 * kGroupThreads;
constexpr int kRowsBuffered = 16;  // stages * rows-per-tile

struct Params {
  const void *x;
  float *base, *aux;
  int64_t n, C;
  int nStrips, R, S, G;
  int64_t nTiles;
  double *colpart, *rowpart, *rowsum, *blkpart, *recpart, *record;
  float *u, *v;
  uint8_t *codes, *body_u, *body_v;
  unsigned int *ticket;
  int scale_mode;
  int stop_after;  // profiling: 1 = phase A only, 2 = A + scales, 0 = full
  unsigned long long *timer;  // profiling: [G][8] globaltimer stamps, or null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

constexpr int kUCache = 512;  // cached u_i per CTA for phase B

// f32 state arrays staged per tile: base + aux (feedback or ref); naive mode none
template <int MODE>
constexpr int n_f32_arrays() {
  return MODE == CC_NAIVE ? 0 : 2;
}

// deterministic block sum over all kThreads threads (fixed pairing)
__device__ __forceinline__ double block_sum(double v, double *red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kThreads / 32; ++i) s += red[i];
    red[kThreads / 32] = s;
  }
  __syncthreads();
  s = red[kThreads / 32];
  __syncthreads();
  return s;
}

struct CodeVal {
  uint32_t code;
  float d;
};

// exact path for one element (f64 scale math, identical to quant.cu)
template <int CODEC>
__device__ __noinline__ CodeVal quantize1_exact(float t, double ud, double vd) {
  const double s = ud * vd;
  CodeVal r;
  if constexpr (CODEC == CC_SIGN1) {
    r.code = t < 0.0f ? 1u : 0u;
    r.d = (float)(r.code ? -s : s);
  } else if constexpr (CODEC == CC_QUANT2) {
    r.code = quant2_code(t, s, ud * (1.25 * vd));
    r.d = (float)(quant2_level(r.code) * s);
  } else {
    r.code = quant4_code(t, s);
    r.d = (float)(quant4_level(r.code) * s);
  }
  return r;
}

// Per-column constants of the fast 2-bit path: v, and 1.25 v scaled by
// (1 +- 2^-20) and rounded outward, so that for |u| in range
//   RN(u * vhi) > 1.25 u v  and  RN(u * vlo) < 1.25 u v  (exactly),
// i.e. |t| > RN(u vhi) proves code 0/3 and |t| < RN(u vlo) proves code 1/2.
struct ColConst {
  float v[4], vhi[4], vlo[4];
  bool ok;  // all 4 columns have |v| in [2^-50, 2^50] (and v != 0)
};

__device__ __forceinline__ bool scale_in_range(float a) { return a >= 0x1p-50f && a <= 0x1p+50f; }

// 4 elements of one row.  Fast path: pure f32 (p = RN32(u v) == f32(u64 v64);
// d = level * p exact for power-of-two levels while u, v are in range);
// elements inside the 2^-20 guard band around the thresholds, and rows/columns
// with extreme scales, take the exact f64 path.
template <int CODEC>
__device__ __forceinline__ uint32_t quantize4(const float (&t)[4], float uf, bool row_ok, const ColConst &cc,
                                              float (&d)[4]) {
  constexpr int bits = CODEC == CC_SIGN1 ? 1 : (CODEC == CC_QUANT2 ? 2 : 4);
  uint32_t packed = 0;
  if constexpr (CODEC == CC_SIGN1) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float p = __fmul_rn(uf, cc.v[q]);
      const uint32_t neg = t[q] < 0.0f;
      d[q] = neg ? -p : p;
      packed |= neg << q;
    }
    return packed;
  } else if constexpr (CODEC == CC_QUANT2) {
    bool ambiguous = !(row_ok && cc.ok);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float p = __fmul_rn(uf, cc.v[q]);
      const float ax = fabsf(t[q]);
      const bool big = ax > __fmul_rn(uf, cc.vhi[q]);
      ambiguous |= !big && !(ax < __fmul_rn(uf, cc.vlo[q]));
      const bool neg = t[q] < 0.0f;
      // code: big -> (neg ? 0 : 3), else (neg ? 1 : 2)
      const uint32_t code = big ? (neg ? 0u : 3u) : (neg ? 1u : 2u);
      const float lv = big ? 2.0f : 0.5f;
      d[q] = __fmul_rn(neg ? -lv : lv, p);
      packed |= code << (2 * q);
    }
    if (__builtin_expect(ambiguous, 0)) {
      packed = 0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const CodeVal r = quantize1_exact<CODEC>(t[q], (double)uf, (double)cc.v[q]);
        d[q] = r.d;
        packed |= r.code << (2 * q);
      }
    }
    return packed;
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const CodeVal r = quantize1_exact<CODEC>(t[q], (double)uf, (double)cc.v[q]);
      d[q] = r.d;
      packed |= r.code << (bits * q);
    }
    return packed;
  }
}

// ||d - t||^2 and ||t||^2 of 4 elements: f32 quad sums (rel. err < 2^-21)
// added in f64; quads that overflow f32 are redone in f64
__device__ __forceinline__ void record4(const float (&t)[4], const float (&e)[4], double &err, double &tsq) {
  float e2 = e[0] * e[0], t2 = t[0] * t[0];
#pragma unroll
  for (int q = 1; q < 4; ++q) {
    e2 = __fmaf_rn(e[q], e[q], e2);
    t2 = __fmaf_rn(t[q], t[q], t2);
  }
  if (__builtin_expect(!(e2 + t2 <= 3.0e38f), 0)) {
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      a += (double)e[q] * (double)e[q];
      b += (double)t[q] * (double)t[q];
    }
    err += a;
    tsq += b;
  } else {
    err += (double)e2;
    tsq += (double)t2;
  }
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

template <int MODE, int CODEC, typename XT>
__global__ void __launch_bounds__(kThreads, 1) k1_fused(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  constexpr int NF = n_f32_arrays<MODE>();
  const int R = p.R, S = p.S, G = p.G;
  const int64_t n = p.n, C = p.C;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  const int strip = cta % p.nStrips;
  const int64_t c0 = (int64_t)strip * kStrip;
  const int width = (int)min64(kStrip, C - c0);
  const bool producer = warp == kCWarps;
  const int grp = producer ? 0 : tid / kGroupThreads;  // consumer row group
  const int gtid = tid % kGroupThreads;
  const int gwarp = gtid >> 5;

  // ---- shared memory carve-up ----
  const size_t xs_bytes = (size_t)R * kStrip * sizeof(XT);
  const size_t fs_bytes = (size_t)R * kStrip * sizeof(float);
  const size_t stage_bytes = xs_bytes + NF * fs_bytes;
  uint8_t *tiles = smem;
  double *rp = reinterpret_cast<double *>(smem + (size_t)S * stage_bytes);  // [S][R][kGWarps]
  double *red = rp + (size_t)S * R * kGWarps;                               // block-sum scratch
  float *ucache = reinterpret_cast<float *>(red + 64);                        // [kUCache]
  uint64_t *full = reinterpret_cast<uint64_t *>(ucache + kUCache);
  uint64_t *empty = full + S;

  auto stamp = [&](int i) {
    if (p.timer && tid == 0) p.timer[(size_t)cta * 8 + i] = gtimer();
  };
  stamp(0);
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCWarps);
    }
    mbar_fence_init();
  }
  __syncthreads();

  // tiles of this CTA: T_k = cta + k*G, k < K (strip fixed because G % nStrips == 0)
  const int64_t K = p.nTiles > cta ? (p.nTiles - 1 - cta) / G + 1 : 0;
  auto tile_r0 = [&](int64_t k) -> int64_t { return ((cta + k * G) / p.nStrips) * (int64_t)R; };
  auto stage_x = [&](int s) { return reinterpret_cast<XT *>(tiles + (size_t)s * stage_bytes); };
  auto stage_b = [&](int s) { return reinterpret_cast<float *>(tiles + (size_t)s * stage_bytes + xs_bytes); };
  auto stage_a = [&](int s) {
    return reinterpret_cast<float *>(tiles + (size_t)s * stage_bytes + xs_bytes + fs_bytes);
  };
  double cta_total = 0.0;  // producer lanes: running sum of this CTA's row partials
  auto finish_rows = [&](int s, int64_t k) {  // producer lanes: per-row sums over the 8 warps of a group
    const int64_t r0p = tile_r0(k);
    if (lane < R && r0p + lane < n) {
      double acc = 0.0;
      for (int w = 0; w < kGWarps; ++w) acc += rp[((size_t)s * R + lane) * kGWarps + w];
      p.rowpart[(int64_t)strip * n + r0p + lane] = acc;
      cta_total += acc;
    }
  };

  const XT *X = reinterpret_cast<const XT *>(p.x);
  // ---------------- producer warp ----------------
  // phaseB: stage base too in no-feedback mode (t only needs x - ref, the update needs base)
  auto produce = [&](int64_t seq0, bool phaseB, uint64_t policy) {
    for (int64_t k = 0; k < K; ++k) {
      const int64_t seq = seq0 + k;
      const int s = (int)(seq % S);
      const int64_t use = seq / S;
      if (use > 0) {
        mbar_wait(&empty[s], (uint32_t)((use - 1) & 1));
        if (!phaseB && k >= S) finish_rows(s, k - S);
      }
      if (lane == 0) {
        const int64_t kk = phaseB ? (K - 1 - k) : k;
        const int64_t r0 = tile_r0(kk);
        const int nrows = (int)min64(R, n - r0);
        const bool need_base = MODE == CC_WITH_FEEDBACK || (MODE == CC_NO_FEEDBACK && phaseB);
        const uint32_t xrow = (uint32_t)(width * sizeof(XT)), frow = (uint32_t)(width * sizeof(float));
        const uint32_t per = xrow + (need_base ? frow : 0u) + (NF ? frow : 0u);
        mbar_expect_tx(&full[s], (uint32_t)nrows * per);
        for (int r = 0; r < nrows; ++r) {
          const int64_t e = (r0 + r) * C + c0;
          bulk_g2s(stage_x(s) + (size_t)r * kStrip, X + e, xrow, &full[s], policy);
          if (need_base) bulk_g2s(stage_b(s) + (size_t)r * kStrip, p.base + e, frow, &full[s], policy);
          if constexpr (NF) bulk_g2s(stage_a(s) + (size_t)r * kStrip, p.aux + e, frow, &full[s], policy);
        }
      }
      __syncwarp();
    }
  };

  const int col = 4 * gtid;  // consumer's first column inside the strip
  const bool active = !producer && col < width;
  auto load_row = [&](int s, int r, float (&xx)[4], float (&bb)[4], float (&aa)[4], bool with_base) {
    if constexpr (sizeof(XT) == 2) {
      const uint2 raw = *reinterpret_cast<const uint2 *>(stage_x(s) + (size_t)r * kStrip + col);
      xx[0] = __uint_as_float(raw.x << 16);
      xx[1] = __uint_as_float(raw.x & 0xffff0000u);
      xx[2] = __uint_as_float(raw.y << 16);
      xx[3] = __uint_as_float(raw.y & 0xffff0000u);
    } else {
      const float4 v = lds4(reinterpret_cast<const float *>(stage_x(s)) + (size_t)r * kStrip + col);
      xx[0] = v.x; xx[1] = v.y; xx[2] = v.z; xx[3] = v.w;
    }
    if (NF && with_base) {
      const float4 v = lds4(stage_b(s) + (size_t)r * kStrip + col);
      bb[0] = v.x; bb[1] = v.y; bb[2] = v.z; bb[3] = v.w;
    }
    if constexpr (NF) {
      const float4 v = lds4(stage_a(s) + (size_t)r * kStrip + col);
      aa[0] = v.x; aa[1] = v.y; aa[2] = v.z; aa[3] = v.w;
    }
  };

  // ================= phase A: |t| partial sums =================
  if (producer) {
    produce(0, false, l2_policy_evict_last());
    for (int64_t k = K - min64(S, K); k < K; ++k) {  // drain the last tiles' row sums
      const int s = (int)(k % S);
      mbar_wait(&empty[s], (uint32_t)((k / S) & 1));
      finish_rows(s, k);
    }
  } else {
    double cs[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t k = 0; k < K; ++k) {
      const int s = (int)(k % S);
      mbar_wait(&full[s], (uint32_t)((k / S) & 1));
      const int64_t r0 = tile_r0(k);
      const int nrows = (int)min64(R, n - r0);
      for (int r = grp; r < nrows; r += kGroups) {
        float xx[4] = {0.f, 0.f, 0.f, 0.f}, bb[4] = {0.f, 0.f, 0.f, 0.f}, aa[4] = {0.f, 0.f, 0.f, 0.f};
        double a[4] = {0.0, 0.0, 0.0, 0.0};
        if (active) {
          load_row(s, r, xx, bb, aa, MODE == CC_WITH_FEEDBACK);
#pragma unroll
          for (int q = 0; q < 4; ++q) a[q] = fabs((double)target_of<MODE>(xx[q], bb[q], aa[q]));
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) cs[q] += a[q];
        double rs = ((a[0] + a[1]) + a[2]) + a[3];
        rs = warp_sum(rs);
        if (lane == 0) rp[((size_t)s * R + r) * kGWarps + gwarp] = rs;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // merge the two row groups' column partials (fixed order g0 + g1) through smem
    double *xchg = reinterpret_cast<double *>(tiles);
    named_sync(1, kConsumers);  // all consumers done with the last stage
    if (grp == 1) {
#pragma unroll
      for (int q = 0; q < 4; ++q) xchg[4 * gtid + q] = cs[q];
    }
    named_sync(1, kConsumers);
    if (grp == 0 && active) {
      double *cp = p.colpart + (int64_t)(cta / p.nStrips) * C + c0 + col;
#pragma unroll
      for (int q = 0; q < 4; ++q) cp[q] = cs[q] + xchg[4 * gtid + q];
    }
  }

  // per-CTA |t| total (deterministic: fixed lane order) -> blkpart
  {
    const double b = block_sum(producer ? cta_total : 0.0, red);
    if (tid == 0) p.blkpart[cta] = b;
  }
  stamp(1);
  cg::grid_group grid = cg::this_grid();
  grid.sync();
  stamp(2);
  if (p.stop_after == 1) return;

  // ================= phase F: v_j (column means), g, u_i =================
  const int slots = G / p.nStrips;
  if (cta == 0 && tid == 0) *p.ticket = 0u;
  {
    // 8 lanes per column, fixed split of the slots, fixed butterfly combine
    const int64_t gid = (int64_t)cta * kThreads + tid;
    const int64_t nthr = (int64_t)G * kThreads;
    for (int64_t base_id = gid - (gid & 7); base_id < C * 8; base_id += nthr - (nthr & 7)) {
      const int64_t j = base_id / 8;
      const int part = (int)(gid & 7);
      double sacc = 0.0;
      for (int q = part; q < slots; q += 8) sacc += __ldcg(p.colpart + (int64_t)q * C + j);
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 1);
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 2);
      sacc += __shfl_xor_sync(0xffffffffu, sacc, 4);
      if (part == 0) {
        float v = (float)(sacc / (double)n);  // colmean (cx:148)
        if (p.scale_mode == CC_SCALE_PER_TOKEN) v = 1.0f;
        p.v[j] = v;
        store_f32_bytes(p.body_v + 4 * j, v);
      }
    }
  }
  {
    const double part = tid < G ? __ldcg(p.blkpart + tid) : 0.0;  // G <= kThreads (launcher)
    const double tot = block_sum(part, red);
    const double g = tot / (double)(n * C);  // mean|t| (cx:142)
    const int64_t ch = (n + G - 1) / G;
    const int64_t i0 = (int64_t)cta * ch, i1 = min64(n, i0 + ch);
    for (int64_t i = i0 + tid; i < i1; i += kThreads) {
      double rs = 0.0;
      for (int s = 0; s < p.nStrips; ++s) rs += __ldcg(p.rowpart + (int64_t)s * n + i);
      float u;
      if (p.scale_mode == CC_SCALE_PER_CHANNEL) u = 1.0f;
      else if (p.scale_mode == CC_SCALE_PER_TOKEN) u = (float)(rs / (double)C);
      else if (g == 0.0) u = 1.0f;
      else u = (float)fmax((rs / (double)C) / g, kRowScaleFloor);  // cx:147
      p.u[i] = u;
      store_f32_bytes(p.body_u + 4 * i, u);
    }
  }
  stamp(3);
  grid.sync();
  stamp(4);
  if (p.stop_after == 2) return;

  // u_i of every row this CTA quantizes, in phase-B order
  const bool ucached = K * R <= kUCache;
  if (ucached) {
    for (int i = tid; i < K * R; i += kThreads) {
      const int64_t row = tile_r0(K - 1 - i / R) + i % R;
      ucache[i] = row < n ? __ldcg(p.u + row) : 0.0f;
    }
  }
  __syncthreads();

  // ================= phase B: quantize, pack, update state =================
  double err = 0.0, tsq = 0.0;
  if (producer) {
    produce(K, true, l2_policy_evict_first());
  } else {
    ColConst cc;
    cc.ok = true;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float v = active ? __ldcg(p.v + c0 + col + q) : 1.0f;
      cc.v[q] = v;
      cc.vhi[q] = __fmul_ru(__fmul_ru(v, 1.25f), 1.00000095367431640625f);  // (1 + 2^-20)
      cc.vlo[q] = __fmul_rd(__fmul_rd(v, 1.25f), 0.99999904632568359375f);  // (1 - 2^-20)
      cc.ok = cc.ok && scale_in_range(fabsf(v));
    }
    for (int64_t k = 0; k < K; ++k) {
      const int64_t seq = K + k;
      const int s = (int)(seq % S);
      mbar_wait(&full[s], (uint32_t)((seq / S) & 1));
      const int64_t r0 = tile_r0(K - 1 - k);
      const int nrows = (int)min64(R, n - r0);
      for (int r = grp; r < nrows; r += kGroups) {
        const int64_t row = r0 + r;
        const float uf = ucached ? ucache[k * R + r] : __ldcg(p.u + row);
        float xx[4] = {0.f, 0.f, 0.f, 0.f}, bb[4] = {0.f, 0.f, 0.f, 0.f}, aa[4] = {0.f, 0.f, 0.f, 0.f};
        if (active) load_row(s, r, xx, bb, aa, true);
        float t[4], d[4], e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = target_of<MODE>(xx[q], bb[q], aa[q]);
        const uint32_t packed = quantize4<CODEC>(t, uf, scale_in_range(fabsf(uf)), cc, d);
#pragma unroll
        for (int q = 0; q < 4; ++q) e[q] = __fsub_rn(t[q], d[q]);
        if (active) {
          record4(t, e, err, tsq);
          const int64_t eo = row * C + c0 + col;
          if constexpr (MODE == CC_NAIVE) {
            stg_cs4(p.base + eo, make_float4(d[0], d[1], d[2], d[3]));
          } else {
            stg_cs4(p.base + eo, make_float4(__fadd_rn(bb[0], d[0]), __fadd_rn(bb[1], d[1]), __fadd_rn(bb[2], d[2]),
                                             __fadd_rn(bb[3], d[3])));
            if constexpr (MODE == CC_WITH_FEEDBACK)
              stg_cs4(p.aux + eo, make_float4(e[0], e[1], e[2], e[3]));
            else
              stg_cs4(p.aux + eo, make_float4(xx[0], xx[1], xx[2], xx[3]));
          }
        }
        if constexpr (CODEC == CC_SIGN1) {
          const uint32_t other = __shfl_down_sync(0xffffffffu, packed, 1);
          if (active && (lane & 1) == 0) p.codes[(row * C + c0 + col) >> 3] = (uint8_t)(packed | (other << 4));
        } else if constexpr (CODEC == CC_QUANT2) {
          if (active) p.codes[(row * C + c0 + col) >> 2] = (uint8_t)packed;
        } else {
          if (active) *reinterpret_cast<uint16_t *>(p.codes + ((row * C + c0 + col) >> 1)) = (uint16_t)packed;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  stamp(5);
  {
    const double es = block_sum(err, red);
    const double ts = block_sum(tsq, red);
    if (tid == 0) {
      p.recpart[2 * cta] = es;
      p.recpart[2 * cta + 1] = ts;
      __threadfence();
      const unsigned prev = atomicAdd(p.ticket, 1u);
      if (prev == (unsigned)G - 1) {
        __threadfence();
        double a = 0.0, b = 0.0;
        for (int c = 0; c < G; ++c) {
          a += __ldcg(p.recpart + 2 * c);
          b += __ldcg(p.recpart + 2 * c + 1);
        }
        p.record[0] = a;
        p.record[1] = b;
      }
    }
  }
  stamp(6);
}

}  // namespace fused

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static size_t fused_smem(int mode, int xsize, int R, int S) {
  const int NF = mode == CC_NAIVE ? 0 : 2;
  const size_t stage = (size_t)R * fused::kStrip * (xsize + 4 * NF);
  const size_t rp = (size_t)S * R * fused::kGWarps * sizeof(double);
  const size_t red = 64 * sizeof(double) + fused::kUCache * sizeof(float);  // block-sum scratch + u cache
  return (size_t)S * stage + rp + red + 2 * S * sizeof(uint64_t) + 256;
}

template <int MODE, int CODEC, typename XT>
static int launch_fused(fused::Params &p, cudaStream_t st) {
  auto kern = fused::k1_fused<MODE, CODEC, XT>;
  const size_t smem = fused_smem(MODE, sizeof(XT), p.R, p.S);
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return cuda_status("k1_fused attr");
  void *args[] = {&p};
  cudaError_t e = cudaLaunchCooperativeKernel((const void *)kern, dim3(p.G), dim3(fused::kThreads), args, smem, st);
  if (e != cudaSuccess) {
    set_error(std::string("k1_fused launch: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return CC_ERR_CUDA;
  }
  count_launch();
  return CC_OK;
}

static int g_fused_stop = 0;
static unsigned long long *g_fused_timer = nullptr;
void set_fused_stop(int v) { g_fused_stop = v; }
void set_fused_timer(void *buf) { g_fused_timer = reinterpret_cast<unsigned long long *>(buf); }

bool fused_supported(int64_t n, int64_t C, const void *x, int x_dtype, const float *base, const float *aux,
                     const uint8_t *body) {
  (void)n;
  if (C % fused::kStrip != 0) return false;
  if (!aligned(x, 16) || !aligned(base, 16) || (aux && !aligned(aux, 16)) || !aligned(body, 2)) return false;
  (void)x_dtype;
  return true;
}

int64_t fused_workspace_bytes(int64_t n, int64_t C) {
  const int G = fused::kThreads;  // upper bound on the grid
  size_t b = 0;
  auto add = [&](size_t x) { b += align_up(x, 256); };
  add(sizeof(double) * (size_t)G * fused::kGroups * C);  // colpart (slots <= G * groups)
  add(sizeof(double) * (size_t)cdiv(C, fused::kStrip) * n);
  add(sizeof(double) * n);
  add(sizeof(double) * G);
  add(sizeof(double) * 2 * G);
  add(sizeof(float) * n);
  add(sizeof(float) * C);
  add(256);
  return (int64_t)b;
}

int fused_encode(int codec, int mode, int scale_mode, int64_t n, int64_t C, const void *x, int x_dtype, float *base,
                 float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st) {
  fused::Params p{};
  p.x = x;
  p.base = base;
  p.aux = aux;
  p.n = n;
  p.C = C;
  p.nStrips = (int)(C / fused::kStrip);
  // rows per tile: keep >= ~8 tiles per CTA so the ring reaches steady state
  int G = sm_count();
  G -= G % p.nStrips;
  if (G > fused::kThreads) G = fused::kThreads - (fused::kThreads % p.nStrips);
  const int64_t per1 = cdiv(n * p.nStrips, G);
  p.R = per1 >= 32 ? 4 : 2;
  p.S = fused::kRowsBuffered / p.R;
  p.G = G;
  p.nTiles = cdiv(n, p.R) * p.nStrips;
  p.scale_mode = scale_mode;
  p.stop_after = g_fused_stop;
  p.timer = g_fused_timer;
  const int bits = codec == CC_SIGN1 ? 1 : (codec == CC_QUANT2 ? 2 : 4);
  const int64_t cbytes = cdiv(n * C * bits, 8);
  p.codes = body;
  p.body_u = body + cbytes;
  p.body_v = p.body_u + 4 * n;
  p.record = record;
  // workspace
  uint8_t *w = reinterpret_cast<uint8_t *>(ws);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    uint8_t *q = w + off;
    off = align_up(off + bytes, 256);
    return q;
  };
  const int slots = G / p.nStrips;
  p.colpart = reinterpret_cast<double *>(take(sizeof(double) * (size_t)slots * C));
  p.rowpart = reinterpret_cast<double *>(take(sizeof(double) * (size_t)p.nStrips * n));
  p.rowsum = reinterpret_cast<double *>(take(sizeof(double) * n));
  p.blkpart = reinterpret_cast<double *>(take(sizeof(double) * G));
  p.recpart = reinterpret_cast<double *>(take(sizeof(double) * 2 * G));
  p.u = reinterpret_cast<float *>(take(sizeof(float) * n));
  p.v = reinterpret_cast<float *>(take(sizeof(float) * C));
  p.ticket = reinterpret_cast<unsigned int *>(take(256));
  if ((int64_t)off > ws_bytes) {
    set_error("fused workspace too small");
    return CC_ERR_ARG;
  }
#define CC_FUSED(MODE, XT)                                                          \
  do {                                                                              \
    if (codec == CC_SIGN1) return launch_fused<MODE, CC_SIGN1, XT>(p, st);          \
    if (codec == CC_QUANT2) return launch_fused<MODE, CC_QUANT2, XT>(p, st);        \
    return launch_fused<MODE, CC_QUANT4, XT>(p, st);                                \
  } while (0)
  if (x_dtype == CC_BF16) {
    if (mode == CC_WITH_FEEDBACK) CC_FUSED(CC_WITH_FEEDBACK, __nv_bfloat16);
    if (mode == CC_NO_FEEDBACK) CC_FUSED(CC_NO_FEEDBACK, __nv_bfloat16);
    CC_FUSED(CC_NAIVE, __nv_bfloat16);
  } else {
    if (mode == CC_WITH_FEEDBACK) CC_FUSED(CC_WITH_FEEDBACK, float);
    if (mode == CC_NO_FEEDBACK) CC_FUSED(CC_NO_FEEDBACK, float);
    CC_FUSED(CC_NAIVE, float);
  }
#undef CC_FUSED
}

}  // namespace cc
