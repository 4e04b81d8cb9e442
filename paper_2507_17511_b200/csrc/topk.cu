// K4: global top-k residual sparsifier (compressors.py:446-456) on sm_100a.
//
// Reference order: |v| descending, then flat index ascending (np.lexsort);
// k = min(size, ceil(f * size)); indices emitted ascending as u32, values as
// f16 (RNE, overflow -> inf).  Decode = dense zero + scatter (cx:358-361).
//
// Device algorithm (radix select on the f32 magnitude bits, key = bits & 0x7fffffff,
// which orders exactly like |v| for finite values, +0 and -0 alike):
//   pass H1  t = target(x, base, aux) written once (into the feedback buffer in
//            residual_with_feedback mode, else into scratch), 4096-bin histogram
//            of key[30:19] in shared memory -> global; ||t||^2 partials.
//   find     the pass's last CTA (ticket): suffix scan of the histogram -> bin b1,
//            remaining need (no separate launch)
//   pass H2  keys in bin b1: 4096-bin histogram of key[18:7]; last CTA -> b2
//   pass H3  keys with key[30:7] == (b1, b2): 128-bin histogram of key[6:0]; last
//            CTA -> threshold key T and the number of ties at T to take (lowest
//            indices first)
//   pass C   per-chunk counts of key > T and key == T
//   scan     exclusive scans -> each chunk's output offset and tie offset
//   pass W   in index order: selected = key > T || (key == T && tie-rank < ties);
//            block scans give each selected element its output slot, so indices
//            come out ascending with no sort; f16 values; sparse state update
//            base[e] += d, fb[e] = t - d (pipeline.py:107-112).
// Every pass streams t once (4 B/elem) with 128-bit loads.
#include "cc_common.cuh"
#include "cc_internal.h"

#include <algorithm>

namespace cc {
namespace topk {

constexpr int kBins = 4096;
constexpr int kBins3 = 128;
constexpr int kThreads = 256;
constexpr int64_t kChunk = 8192;  // elements per CTA in passes C and W

struct State {
  uint32_t need;        // remaining elements to take at the current level
  uint32_t b1, b2;      // selected bins
  uint32_t T;           // threshold key
  uint32_t ties;        // elements with key == T to take
  uint32_t pad[3];      // pad[0]: k_write's record ticket
  uint32_t tk[4];       // last-CTA tickets of the histogram passes (zeroed with the state)
};

// The histogram passes end with a last-CTA selection step (no separate 1-CTA
// launch): every CTA adds its shared histogram into the global one, takes a
// ticket, and the last CTA scans the complete histogram from the top bin.
template <int NB>
__device__ __forceinline__ void block_find(const uint32_t *__restrict__ hist, uint32_t need, uint32_t &bin,
                                           uint32_t &rem, uint32_t *sm);
template <int NB>
__device__ __forceinline__ bool last_cta_find(const uint32_t *__restrict__ hist, unsigned int *ticket,
                                              uint32_t need, uint32_t &bin, uint32_t &rem, uint32_t *sm) {
  __shared__ unsigned last;
  __syncthreads();  // every thread's global histogram adds are issued
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return false;
  __threadfence();
  block_find<NB>(hist, need, bin, rem, sm);
  return true;
}

struct Work {
  uint32_t *hist1, *hist2, *hist3;
  State *st;
  uint32_t *cnt_gt, *cnt_eq, *sel_pref, *eq_pref;
  double *part;  // [nH1 + nChunks][2]
  float *tscratch;
  int nH1;
  int64_t nChunks;
};

__device__ __forceinline__ uint32_t key_of(float t) { return __float_as_uint(t) & 0x7fffffffu; }

// shared-memory histogram increment.  Plain shared atomics: measured on B200 with
// activation residuals (~28 distinct bins per 32 keys) they run at ~70% of the
// streaming rate, while __match_any_sync warp aggregation is 4x slower
// (scripts/exp/hist_bench.cu).
__device__ __forceinline__ void hist_add(uint32_t *h, uint32_t bin, bool valid) {
  if (valid) atomicAdd(&h[bin], 1u);
}

// ---- pass H1 ---------------------------------------------------------------
// 4 consecutive elements per item (128-bit loads when `vec`), 2 items in flight per
// thread per iteration: the warp-synchronous histogram update would otherwise leave
// one load in flight per thread and the pass latency bound.
constexpr int kH1Unroll = 2;
template <int MODE, typename XT, bool FROM_T>
__device__ __forceinline__ void h1_item(const XT *__restrict__ x, float *__restrict__ base, float *__restrict__ aux,
                                        const float *__restrict__ tin, float *__restrict__ tout,
                                        float *__restrict__ decoded, int64_t e, int64_t total, bool vec,
                                        float (&t)[4]) {
  if (vec && e + 4 <= total) {
    float4 tv;
    if constexpr (FROM_T) {
      tv = __ldcs(reinterpret_cast<const float4 *>(tin + e));
    } else {
      const float4 xx = Act<XT>::load4(x + e);
      float4 bb = make_float4(0.f, 0.f, 0.f, 0.f), aa = bb;
      if constexpr (MODE != CC_NAIVE) {
        bb = *reinterpret_cast<const float4 *>(base + e);
        aa = *reinterpret_cast<const float4 *>(aux + e);
        const bool neg0 = __float_as_uint(bb.x) == 0x80000000u || __float_as_uint(bb.y) == 0x80000000u ||
                          __float_as_uint(bb.z) == 0x80000000u || __float_as_uint(bb.w) == 0x80000000u;
        if (neg0) {  // dense base + 0.0 semantics
          float4 c = bb;
          if (__float_as_uint(c.x) == 0x80000000u) c.x = 0.0f;
          if (__float_as_uint(c.y) == 0x80000000u) c.y = 0.0f;
          if (__float_as_uint(c.z) == 0x80000000u) c.z = 0.0f;
          if (__float_as_uint(c.w) == 0x80000000u) c.w = 0.0f;
          *reinterpret_cast<float4 *>(base + e) = c;
        }
      }
      tv = make_float4(target_of<MODE>(xx.x, bb.x, aa.x), target_of<MODE>(xx.y, bb.y, aa.y),
                       target_of<MODE>(xx.z, bb.z, aa.z), target_of<MODE>(xx.w, bb.w, aa.w));
      *reinterpret_cast<float4 *>(tout + e) = tv;
      if constexpr (MODE == CC_NO_FEEDBACK) *reinterpret_cast<float4 *>(aux + e) = xx;  // ref' = a*
      if constexpr (MODE == CC_NAIVE) *reinterpret_cast<float4 *>(base + e) = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    if (decoded) *reinterpret_cast<float4 *>(decoded + e) = make_float4(0.f, 0.f, 0.f, 0.f);
    t[0] = tv.x; t[1] = tv.y; t[2] = tv.z; t[3] = tv.w;
    return;
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t ee = e + q;
    t[q] = 0.0f;
    if (ee >= total) continue;
    float tq;
    if constexpr (FROM_T) {
      tq = tin[ee];
    } else {
      const float xx = Act<XT>::load1(x + ee);
      float bb = 0.f, aa = 0.f;
      if constexpr (MODE != CC_NAIVE) {
        bb = base[ee];
        if (__float_as_uint(bb) == 0x80000000u) base[ee] = 0.0f;
        aa = aux[ee];
      }
      tq = target_of<MODE>(xx, bb, aa);
      tout[ee] = tq;
      if constexpr (MODE == CC_NO_FEEDBACK) aux[ee] = xx;
      if constexpr (MODE == CC_NAIVE) base[ee] = 0.0f;
    }
    if (decoded) decoded[ee] = 0.0f;
    t[q] = tq;
  }
}

template <int MODE, typename XT, bool FROM_T>
__global__ void __launch_bounds__(kThreads) k_h1(const XT *__restrict__ x, float *__restrict__ base,
                                                  float *__restrict__ aux, const float *__restrict__ tin,
                                                  float *__restrict__ tout, float *__restrict__ decoded,
                                                  int64_t total, int vec, uint32_t *__restrict__ hist1,
                                                  double *__restrict__ part, State *st, uint32_t k,
                                                  int fuse_find) {
  __shared__ uint32_t h[kBins];
  __shared__ double red[kThreads / 32];
  for (int i = threadIdx.x; i < kBins; i += kThreads) h[i] = 0;
  __syncthreads();
  double tsq = 0.0;
  const int64_t nitems = (total + 3) / 4;
  const int64_t stride = (int64_t)gridDim.x * kThreads * kH1Unroll;
  for (int64_t i0 = (int64_t)blockIdx.x * kThreads * kH1Unroll; i0 < nitems; i0 += stride) {
    float t[kH1Unroll][4];
#pragma unroll
    for (int u = 0; u < kH1Unroll; ++u)
      h1_item<MODE, XT, FROM_T>(x, base, aux, tin, tout, decoded, (i0 + u * kThreads + threadIdx.x) * 4, total,
                                vec != 0, t[u]);
#pragma unroll
    for (int u = 0; u < kH1Unroll; ++u) {
      const int64_t e = (i0 + u * kThreads + threadIdx.x) * 4;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const bool ok = e + q < total;
        tsq += (double)t[u][q] * (double)t[u][q];
        hist_add(h, key_of(t[u][q]) >> 19, ok);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < kBins; i += kThreads)
    if (h[i]) atomicAdd(&hist1[i], h[i]);
  tsq = warp_sum(tsq);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = tsq;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += red[i];
    part[2 * blockIdx.x] = 0.0;
    part[2 * blockIdx.x + 1] = s;
  }
  __shared__ uint32_t fsm[kThreads / 32 + 2];
  uint32_t bin, rem;
  if (fuse_find && last_cta_find<kBins>(hist1, &st->tk[0], k, bin, rem, fsm) && threadIdx.x == 0) {  // level 1
    st->b1 = bin;
    st->need = rem;
  }
}

// inclusive scan of one value per thread over a CTA of NT threads (warp shuffles, warp
// totals through `wsum` [NT/32]); `total` = the CTA-wide sum
template <int NT>
__device__ __forceinline__ uint32_t block_incl_scan(uint32_t v, uint32_t *wsum, uint32_t &total) {
  static_assert(NT % 32 == 0 && NT <= 1024, "block size");
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  if (w == 0) {
    uint32_t s = lane < NT / 32 ? wsum[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < NT / 32) wsum[lane] = s;
  }
  __syncthreads();
  if (w > 0) incl += wsum[w - 1];
  total = wsum[NT / 32 - 1];
  __syncthreads();  // wsum is reused by the next call
  return incl;
}

// suffix scan of a histogram from the top bin by one CTA (kThreads threads): the bin
// holding the need-th largest key, and how many are still needed inside it
template <int NB>
__device__ __forceinline__ void block_find(const uint32_t *__restrict__ hist, uint32_t need, uint32_t &bin,
                                           uint32_t &rem, uint32_t *sm) {
  constexpr int PER = (NB + kThreads - 1) / kThreads;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t v[PER], local = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {  // thread t owns bins NB-1-t*PER-q (descending)
    const int b = NB - 1 - (t * PER + q);
    v[q] = b >= 0 ? __ldcg(hist + b) : 0u;
    local += v[q];
  }
  uint32_t incl = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) sm[w] = incl;
  __syncthreads();
  uint32_t wpre = 0;
  for (int i = 0; i < w; ++i) wpre += sm[i];
  incl += wpre;
  uint32_t before = incl - local;
  if (before < need && incl >= need) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = NB - 1 - (t * PER + q);
      if (b < 0) break;
      if (before + v[q] >= need) {
        sm[kThreads / 32] = (uint32_t)b;
        sm[kThreads / 32 + 1] = need - before;
        break;
      }
      before += v[q];
    }
  }
  __syncthreads();
  bin = sm[kThreads / 32];
  rem = sm[kThreads / 32 + 1];
  __syncthreads();
}

// ---- find: suffix scan of a histogram from the top bin ---------------------
template <int NB>
__global__ void __launch_bounds__(1024) k_find(const uint32_t *__restrict__ hist, State *st, int level, uint32_t k) {
  constexpr int PER = (NB + 1023) / 1024;
  __shared__ uint32_t tot[32];
  const int t = threadIdx.x;
  // thread t owns bins [NB-1-t*PER ... NB-PER-t*PER] (descending order)
  uint32_t local = 0;
  uint32_t v[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int b = NB - 1 - (t * PER + q);
    v[q] = b >= 0 ? hist[b] : 0u;
    local += v[q];
  }
  uint32_t total;
  const uint32_t incl = block_incl_scan<1024>(local, tot, total);
  const uint32_t need = level == 1 ? k : st->need;
  uint32_t before = incl - local;
  if (before < need && incl >= need) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = NB - 1 - (t * PER + q);
      if (b < 0) break;
      if (before + v[q] >= need) {
        const uint32_t rem = need - before;
        if (level == 1) {
          st->b1 = (uint32_t)b;
        } else if (level == 2) {
          st->b2 = (uint32_t)b;
        } else {
          st->T = (st->b1 << 19) | (st->b2 << 7) | (uint32_t)b;
          st->ties = rem;
        }
        st->need = rem;
        break;
      }
      before += v[q];
    }
  }
}

// ---- passes H2 / H3: histograms of the keys inside the selected prefix ---------
// H2: key[18:7] of keys with key[30:19] == b1;  H3: key[6:0] of keys with
// key[30:7] == (b1, b2).  Both re-stream t (8 keys per thread per iteration).
template <int LEVEL, bool FUSE>  // FUSE: the last CTA selects the next level (compiled out otherwise)
__global__ void __launch_bounds__(kThreads) k_hsub(const float *__restrict__ t, int64_t total, int vec,
                                                    State *st_w, uint32_t *__restrict__ hist) {
  const State *st = st_w;
  constexpr int NB = LEVEL == 2 ? kBins : kBins3;
  __shared__ uint32_t h[NB];
  for (int i = threadIdx.x; i < NB; i += kThreads) h[i] = 0;
  __syncthreads();
  const uint32_t prefix = LEVEL == 2 ? st->b1 : ((st->b1 << 12) | st->b2);
  constexpr int shift = LEVEL == 2 ? 19 : 7;
  const int64_t nitems = (total + 3) / 4;
  constexpr int kU = 4;  // float4 loads in flight per thread
  const int64_t stride = (int64_t)gridDim.x * kThreads * kU;
  for (int64_t i0 = (int64_t)blockIdx.x * kThreads * kU; i0 < nitems; i0 += stride) {
    uint32_t key[4 * kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t e = (i0 + u * kThreads + threadIdx.x) * 4;
      if (vec && e + 4 <= total) {
        const float4 v = __ldcg(reinterpret_cast<const float4 *>(t + e));  // t is re-read: keep it in L2
        key[4 * u] = key_of(v.x); key[4 * u + 1] = key_of(v.y);
        key[4 * u + 2] = key_of(v.z); key[4 * u + 3] = key_of(v.w);
      } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) key[4 * u + q] = e + q < total ? key_of(t[e + q]) : 0xffffffffu;
      }
    }
#pragma unroll
    for (int j = 0; j < 4 * kU; ++j) {
      const bool in = key[j] != 0xffffffffu && (key[j] >> shift) == prefix;
      hist_add(h, LEVEL == 2 ? (key[j] >> 7) & 0xfffu : key[j] & 127u, in);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < NB; i += kThreads)
    if (h[i]) atomicAdd(&hist[i], h[i]);
  if constexpr (FUSE) {
  __shared__ uint32_t fsm[kThreads / 32 + 2];
  uint32_t bin, rem;
  if (last_cta_find<NB>(hist, &st_w->tk[LEVEL - 1], st_w->need, bin, rem, fsm) && threadIdx.x == 0) {
    if (LEVEL == 2) {
      st_w->b2 = bin;
    } else {
      st_w->T = (st_w->b1 << 19) | (st_w->b2 << 7) | bin;  // exact threshold key
      st_w->ties = rem;                                    // keys equal to T to take (lowest indices)
    }
    st_w->need = rem;
  }
  }
}

// chunk offsets: exclusive scans of the per-chunk tie counts and selected counts (the
// first `ties` keys equal to T, in index order, are taken), NT threads of one CTA
template <int NT>
__device__ __forceinline__ void scan_chunks(int64_t nch, uint32_t ties, const uint32_t *__restrict__ cnt_gt,
                                            const uint32_t *__restrict__ cnt_eq, uint32_t *__restrict__ sel_pref,
                                            uint32_t *__restrict__ eq_pref, uint32_t *s_eq, uint32_t *s_sel,
                                            uint32_t *carry) {
  (void)carry;
  uint32_t carry_eq = 0, carry_sel = 0;  // identical in every thread
  for (int64_t base = 0; base < nch; base += NT) {
    const int64_t i = base + threadIdx.x;
    const uint32_t eq = i < nch ? __ldcg(cnt_eq + i) : 0u;
    const uint32_t gt = i < nch ? __ldcg(cnt_gt + i) : 0u;
    uint32_t tot_eq, tot_sel;
    const uint32_t eq_before = carry_eq + block_incl_scan<NT>(eq, s_eq, tot_eq) - eq;
    uint32_t take = 0;
    if (eq_before < ties) take = min(eq, ties - eq_before);
    const uint32_t sel = gt + take;
    const uint32_t sel_incl = block_incl_scan<NT>(sel, s_sel, tot_sel);
    if (i < nch) {
      eq_pref[i] = eq_before;
      sel_pref[i] = carry_sel + sel_incl - sel;
    }
    carry_eq += tot_eq;
    carry_sel += tot_sel;
  }
}

// ---- pass C: per-chunk counts ------------------------------------------------
template <bool FUSE>  // FUSE: the last CTA also computes the chunk offsets (replaces k_scan)
__global__ void __launch_bounds__(kThreads) k_count(const float *__restrict__ t, int64_t total, State *st,
                                                     uint32_t *__restrict__ cnt_gt, uint32_t *__restrict__ cnt_eq,
                                                     uint32_t *__restrict__ sel_pref, uint32_t *__restrict__ eq_pref) {
  __shared__ uint32_t sg[kThreads / 32], se[kThreads / 32];
  const uint32_t T = st->T;
  const int64_t c0 = (int64_t)blockIdx.x * kChunk;
  const int64_t c1 = min64(total, c0 + kChunk);
  uint32_t gt = 0, eq = 0;
  if (((c1 - c0) & 3) == 0 && (reinterpret_cast<uintptr_t>(t) & 15) == 0) {
    // kChunk / 4 float4 per CTA: all of a thread's loads in flight together
    constexpr int kV = kChunk / 4 / kThreads;  // 8
    float4 v[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t e = c0 + 4 * ((int64_t)u * kThreads + threadIdx.x);
      v[u] = e < c1 ? __ldcg(reinterpret_cast<const float4 *>(t + e)) : make_float4(-0.f, -0.f, -0.f, -0.f);
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t e = c0 + 4 * ((int64_t)u * kThreads + threadIdx.x);
      if (e >= c1) continue;
      const uint32_t k4[4] = {key_of(v[u].x), key_of(v[u].y), key_of(v[u].z), key_of(v[u].w)};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        gt += k4[q] > T;
        eq += k4[q] == T;
      }
    }
  } else {
    for (int64_t e = c0 + threadIdx.x; e < c1; e += kThreads) {
      const uint32_t key = key_of(__ldcg(t + e));
      gt += key > T;
      eq += key == T;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    gt += __shfl_xor_sync(0xffffffffu, gt, o);
    eq += __shfl_xor_sync(0xffffffffu, eq, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sg[threadIdx.x >> 5] = gt;
    se[threadIdx.x >> 5] = eq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t a = 0, b = 0;
    for (int i = 0; i < kThreads / 32; ++i) {
      a += sg[i];
      b += se[i];
    }
    cnt_gt[blockIdx.x] = a;
    cnt_eq[blockIdx.x] = b;
  }
  if constexpr (FUSE) {
    __shared__ unsigned last;
    __shared__ uint32_t s_eq[kThreads], s_sel[kThreads], carry[2];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      last = atomicAdd(&st->tk[3], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      scan_chunks<kThreads>((int64_t)gridDim.x, st->ties, cnt_gt, cnt_eq, sel_pref, eq_pref, s_eq, s_sel, carry);
    }
  }
}

// ---- scan: chunk offsets --------------------------------------------------------
__global__ void __launch_bounds__(1024) k_scan(int64_t nch, const State *st, const uint32_t *__restrict__ cnt_gt,
                                               const uint32_t *__restrict__ cnt_eq, uint32_t *__restrict__ sel_pref,
                                               uint32_t *__restrict__ eq_pref) {
  __shared__ uint32_t s_eq[1024], s_sel[1024], carry[2];
  scan_chunks<1024>(nch, st->ties, cnt_gt, cnt_eq, sel_pref, eq_pref, s_eq, s_sel, carry);
}

// block-wide exclusive scan of a per-thread count; returns the block total
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t &excl, uint32_t *sm) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += y;
  }
  if (lane == 31) sm[w] = inc;
  __syncthreads();
  uint32_t wpre = 0, tot = 0;
  for (int i = 0; i < kThreads / 32; ++i) {
    if (i < w) wpre += sm[i];
    tot += sm[i];
  }
  __syncthreads();
  excl = wpre + inc - v;
  return tot;
}

// ---- pass W: ordered write + sparse state update ------------------------------
// Each CTA stages its 8192-element chunk in shared memory (coalesced), every
// thread owns a run of 32 consecutive elements: two block scans per chunk give the
// tie ranks and the output slots, then each thread emits its selected elements in
// index order.  (Run index i of thread r lives at smem[33 r + i]: conflict-free.)
constexpr int kRun = kChunk / kThreads;  // 32
template <int MODE, typename XT>
__global__ void __launch_bounds__(kThreads) k_write(const float *__restrict__ t, const XT *__restrict__ x,
                                                     float *__restrict__ base, float *__restrict__ aux,
                                                     float *__restrict__ decoded, int64_t total, int64_t k,
                                                     const State *st, const uint32_t *__restrict__ sel_pref,
                                                     const uint32_t *__restrict__ eq_pref, uint8_t *__restrict__ body,
                                                     double *__restrict__ part, int stateful,
                                                     const double *__restrict__ allpart, int nparts,
                                                     unsigned int *__restrict__ ticket, double *__restrict__ record) {
  __shared__ float tv_s[kThreads * (kRun + 1)];
  __shared__ uint32_t sm[kThreads / 32];
  __shared__ double red[kThreads / 32];
  const uint32_t T = st->T, ties = st->ties;
  const int64_t c0 = (int64_t)blockIdx.x * kChunk;
  const int64_t c1 = min64(total, c0 + kChunk);
  if ((reinterpret_cast<uintptr_t>(t) & 15) == 0) {
    constexpr int kV = kChunk / 4 / kThreads;  // 8 float4 per thread, all in flight together
    float4 v[kV];
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int64_t e = c0 + 4 * ((int64_t)u * kThreads + threadIdx.x);
      if (e + 4 <= c1) {
        v[u] = __ldcs(reinterpret_cast<const float4 *>(t + e));
      } else {
        v[u].x = e < c1 ? __ldcs(t + e) : 0.0f;
        v[u].y = e + 1 < c1 ? __ldcs(t + e + 1) : 0.0f;
        v[u].z = e + 2 < c1 ? __ldcs(t + e + 2) : 0.0f;
        v[u].w = e + 3 < c1 ? __ldcs(t + e + 3) : 0.0f;
      }
    }
#pragma unroll
    for (int u = 0; u < kV; ++u) {
      const int i = 4 * (u * kThreads + threadIdx.x);
      const float vv[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
      for (int q = 0; q < 4; ++q) tv_s[((i + q) / kRun) * (kRun + 1) + (i + q) % kRun] = vv[q];
    }
  } else {
    for (int64_t e = c0 + threadIdx.x; e < c0 + kChunk; e += kThreads) {
      const int i = (int)(e - c0);
      tv_s[(i / kRun) * (kRun + 1) + i % kRun] = e < c1 ? __ldcs(t + e) : 0.0f;
    }
  }
  __syncthreads();
  const float *run = tv_s + threadIdx.x * (kRun + 1);
  const int64_t e_run = c0 + (int64_t)threadIdx.x * kRun;
  const int64_t rem = c1 - e_run;
  const int valid = rem <= 0 ? 0 : (int)min64(kRun, rem);
  uint32_t m_gt = 0, m_eq = 0;  // bit i of the run: key > T / key == T
  for (int i = 0; i < valid; ++i) {
    const uint32_t key = key_of(run[i]);
    m_gt |= (uint32_t)(key > T) << i;
    m_eq |= (uint32_t)(key == T) << i;
  }
  const uint32_t n_eq = __popc(m_eq), n_gt = __popc(m_gt);
  uint32_t eq_ex;
  block_excl_scan(n_eq, eq_ex, sm);
  const uint32_t tie_rank = eq_pref[blockIdx.x] + eq_ex;  // ties before this run
  const uint32_t ties_here = tie_rank < ties ? min(n_eq, ties - tie_rank) : 0u;
  uint32_t sel_ex;
  block_excl_scan(n_gt + ties_here, sel_ex, sm);
  uint32_t pos = sel_pref[blockIdx.x] + sel_ex;
  uint32_t *idx_out = reinterpret_cast<uint32_t *>(body);
  __half *val_out = reinterpret_cast<__half *>(body + 4 * k);
  // the run's selected elements: every key > T plus its first `ties_here` keys == T
  // (ties go to the lowest index); visited in index order through the bit mask, so a
  // thread loops over its selections only, not over all 32 elements
  uint32_t msel = m_gt;
  for (uint32_t take = ties_here, mm = m_eq; take; --take) {
    const uint32_t b = mm & (0u - mm);
    msel |= b;
    mm ^= b;
  }
  double adj = 0.0;  // sum over selected of (d - t)^2 - t^2
  while (msel) {
    const int i = __ffs(msel) - 1;
    msel &= msel - 1;
    const float tv = run[i];
    const int64_t e = e_run + i;
    idx_out[pos] = (uint32_t)e;
    const __half h = __float2half_rn(tv);
    val_out[pos] = h;
    ++pos;
    const float d = __half2float(h);
    const double df = (double)d - (double)tv;
    adj += df * df - (double)tv * (double)tv;
    if (decoded) decoded[e] = d;
    if (stateful) {
      if constexpr (MODE == CC_NAIVE) {
        base[e] = d;
      } else {
        base[e] = __fadd_rn(base[e], d);
        if constexpr (MODE == CC_WITH_FEEDBACK) aux[e] = __fsub_rn(tv, d);
      }
    }
  }
  adj = warp_sum(adj);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = adj;
  __syncthreads();
  __shared__ unsigned last;
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) s += red[i];
    part[2 * blockIdx.x] = s;
    part[2 * blockIdx.x + 1] = 0.0;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last) {  // the last CTA reduces every (adj, ||t||^2) partial in a fixed order (pl:115-120)
    __threadfence();
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < nparts; i += kThreads) {
      a += __ldcg(allpart + 2 * i);
      b += __ldcg(allpart + 2 * i + 1);
    }
    a = warp_sum(a);
    b = warp_sum(b);
    __shared__ double ra[kThreads / 32], rb[kThreads / 32];
    if ((threadIdx.x & 31) == 0) {
      ra[threadIdx.x >> 5] = a;
      rb[threadIdx.x >> 5] = b;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double sa = 0.0, sb = 0.0;
      for (int i = 0; i < kThreads / 32; ++i) {
        sa += ra[i];
        sb += rb[i];
      }
      record[0] = sb + sa;  // ||d - t||^2 = ||t||^2 + sum over kept of ((d - t)^2 - t^2)
      record[1] = sb;
    }
  }
  (void)x;
}

// ---- receiver: sparse scatter (and -0.0 canonicalisation) ------------------------
constexpr int kMaxPeers = 64;
struct Peers {
  const uint8_t *body[kMaxPeers];
  float *base[kMaxPeers];
  int64_t total[kMaxPeers];
  int64_t k[kMaxPeers];
};

__global__ void __launch_bounds__(kThreads) k_canon(const __grid_constant__ Peers pp, int replace) {
  const int peer = blockIdx.y;
  float *base = pp.base[peer];
  const int64_t total = pp.total[peer];
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += stride) {
    if (replace) base[e] = 0.0f;
    else if (__float_as_uint(base[e]) == 0x80000000u) base[e] = 0.0f;
  }
}

__global__ void __launch_bounds__(kThreads) k_scatter(const __grid_constant__ Peers pp, int replace) {
  const int peer = blockIdx.y;
  const int64_t k = pp.k[peer];
  const uint32_t *idx = reinterpret_cast<const uint32_t *>(pp.body[peer]);
  const __half *val = reinterpret_cast<const __half *>(pp.body[peer] + 4 * k);
  float *base = pp.base[peer];
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < k; i += stride) {
    const uint32_t e = idx[i];
    const float d = __half2float(val[i]);
    base[e] = replace ? d : __fadd_rn(base[e], d);
  }
}

}  // namespace topk

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static topk::Work carve_topk(void *ws, int64_t total, bool need_t, int nH1, size_t *bytes) {
  topk::Work w{};
  uint8_t *b = reinterpret_cast<uint8_t *>(ws);
  size_t off = 0;
  auto take = [&](size_t n) {
    uint8_t *q = b ? b + off : nullptr;
    off = align_up(off + n, 256);
    return q;
  };
  w.nH1 = nH1;
  w.nChunks = cdiv(total, topk::kChunk);
  // zeroed region first: hist1, hist2, hist3, state
  w.hist1 = reinterpret_cast<uint32_t *>(take(4 * topk::kBins));
  w.hist2 = reinterpret_cast<uint32_t *>(take(4 * topk::kBins));
  w.hist3 = reinterpret_cast<uint32_t *>(take(4 * topk::kBins3));
  w.st = reinterpret_cast<topk::State *>(take(sizeof(topk::State)));
  w.cnt_gt = reinterpret_cast<uint32_t *>(take(4 * w.nChunks));
  w.cnt_eq = reinterpret_cast<uint32_t *>(take(4 * w.nChunks));
  w.sel_pref = reinterpret_cast<uint32_t *>(take(4 * w.nChunks));
  w.eq_pref = reinterpret_cast<uint32_t *>(take(4 * w.nChunks));
  w.part = reinterpret_cast<double *>(take(16 * (size_t)(nH1 + w.nChunks)));
  w.tscratch = need_t ? reinterpret_cast<float *>(take(4 * (size_t)total)) : nullptr;
  if (bytes) *bytes = off;
  return w;
}

static bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// histogram passes: few, fat CTAs (each zeroes / flushes a 4096-bin shared histogram)
// measured: the last-CTA selection wins below ~4M elements (512 x 3072: 97 -> 86 us per
// encode_step), the separate 1-CTA launches above (4096 x 3072: 121.6 vs 127.5 us)
static int fuse_find(int64_t total) {
  static const int64_t lim = [] {
    const char *e = getenv("CC_TOPK_FUSE_MAX");  // experiment knob: largest fused-find size
    return e ? (int64_t)atoll(e) : (int64_t)4 << 20;
  }();
  return total <= lim;
}

static int h1_blocks(int64_t total) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), sm_count() * 2)); }

int64_t topk_resident_workspace_bytes();

int64_t topk_workspace_bytes(int64_t n, int64_t C, int64_t) {
  size_t b = 0;
  carve_topk(nullptr, n * C, true, h1_blocks(n * C), &b);
  return std::max<int64_t>((int64_t)b, topk_resident_workspace_bytes());
}

static const size_t kZeroBytes = 2 * 4 * topk::kBins + 4 * topk::kBins3 + 3 * 256;

// common tail after the H1 pass: select T, count, scan, write
template <int MODE, typename XT>
static void select_and_write(const topk::Work &w, const float *t, const XT *x, float *base, float *aux,
                             float *decoded, int64_t total, int64_t k, uint8_t *body, double *record, int stateful,
                             cudaStream_t st) {
  using namespace topk;
  const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 4 * kThreads), sm_count() * 8));
  const int vec = al16(t);
  // small problems: each histogram pass's last CTA selects the next level (no 1-CTA
  // launches); large ones: the ticket adds would serialise, keep the k_find launches
  const int fuse = fuse_find(total);
  if (fuse) {
    k_hsub<2, true><<<nb, kThreads, 0, st>>>(t, total, vec, w.st, w.hist2);
    k_hsub<3, true><<<nb, kThreads, 0, st>>>(t, total, vec, w.st, w.hist3);
  } else {
    k_find<kBins><<<1, 1024, 0, st>>>(w.hist1, w.st, 1, (uint32_t)k);
    k_hsub<2, false><<<nb, kThreads, 0, st>>>(t, total, vec, w.st, w.hist2);
    k_find<kBins><<<1, 1024, 0, st>>>(w.hist2, w.st, 2, 0);
    k_hsub<3, false><<<nb, kThreads, 0, st>>>(t, total, vec, w.st, w.hist3);
    k_find<kBins3><<<1, 1024, 0, st>>>(w.hist3, w.st, 3, 0);
  }
  if (fuse) {
    k_count<true><<<(unsigned)w.nChunks, kThreads, 0, st>>>(t, total, w.st, w.cnt_gt, w.cnt_eq, w.sel_pref,
                                                           w.eq_pref);
  } else {
    k_count<false><<<(unsigned)w.nChunks, kThreads, 0, st>>>(t, total, w.st, w.cnt_gt, w.cnt_eq, nullptr, nullptr);
    k_scan<<<1, 1024, 0, st>>>(w.nChunks, w.st, w.cnt_gt, w.cnt_eq, w.sel_pref, w.eq_pref);
  }
  // k_write's last CTA also reduces the StepRecord partials (no separate launch)
  k_write<MODE, XT><<<(unsigned)w.nChunks, kThreads, 0, st>>>(t, x, base, aux, decoded, total, k, w.st, w.sel_pref,
                                                             w.eq_pref, body, w.part + 2 * w.nH1, stateful, w.part,
                                                             (int)(w.nH1 + w.nChunks), &w.st->pad[0], record);
  count_launch(fuse ? 4 : 8);
}

int topk_encode(int64_t n, int64_t C, int64_t k, const float *t, uint8_t *body, float *decoded, void *ws,
                int64_t ws_bytes, cudaStream_t st) {
  const int64_t total = n * C;
  size_t need = 0;
  const int nH1 = h1_blocks(total);
  carve_topk(nullptr, total, false, nH1, &need);
  if ((int64_t)need + 256 > ws_bytes) {
    set_error("top-k workspace too small");
    return CC_ERR_ARG;
  }
  topk::Work w = carve_topk(ws, total, false, nH1, nullptr);
  double *record = reinterpret_cast<double *>(reinterpret_cast<uint8_t *>(ws) + need);
  cudaMemsetAsync(ws, 0, kZeroBytes, st);
  topk::k_h1<CC_NAIVE, float, true><<<nH1, topk::kThreads, 0, st>>>(nullptr, nullptr, nullptr, t, nullptr, decoded,
                                                                    total, al16(t) && al16(decoded), w.hist1, w.part,
                                                                    w.st, (uint32_t)k, fuse_find(total));
  count_launch();
  select_and_write<CC_NAIVE, float>(w, t, nullptr, nullptr, nullptr, decoded, total, k, body, record, 0, st);
  return cuda_status("topk_encode");
}

int topk_resident_encode_step(int mode, int64_t n, int64_t C, int64_t k, const void *x, int x_dtype, float *base,
                              float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record,
                              cudaStream_t st);

int topk_encode_step(int mode, int64_t n, int64_t C, int64_t k, const void *x, int x_dtype, float *base, float *aux,
                     uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st) {
  {  // one persistent launch when the grid can be co-resident (topk_resident.cu)
    const int rc = topk_resident_encode_step(mode, n, C, k, x, x_dtype, base, aux, body, ws, ws_bytes, record, st);
    if (rc != CC_ERR_UNSUPPORTED) return rc;
  }
  const int64_t total = n * C;
  size_t need = 0;
  const int nH1 = h1_blocks(total);
  const bool need_t = mode != CC_WITH_FEEDBACK;
  carve_topk(nullptr, total, need_t, nH1, &need);
  if ((int64_t)need > ws_bytes) {
    set_error("top-k workspace too small");
    return CC_ERR_ARG;
  }
  topk::Work w = carve_topk(ws, total, need_t, nH1, nullptr);
  float *t = mode == CC_WITH_FEEDBACK ? aux : w.tscratch;
  const int vec = al16(t) && al16(base) && al16(aux) &&
                  (reinterpret_cast<uintptr_t>(x) & (x_dtype == CC_BF16 ? 7 : 15)) == 0;
  cudaMemsetAsync(ws, 0, kZeroBytes, st);
#define CC_TK(MODE, XT)                                                                                      \
  do {                                                                                                       \
    topk::k_h1<MODE, XT, false><<<nH1, topk::kThreads, 0, st>>>((const XT *)x, base, aux, nullptr, t, nullptr, \
                                                                total, vec, w.hist1, w.part, w.st, (uint32_t)k, \
                                                                fuse_find(total));                          \
    count_launch();                                                                                          \
    select_and_write<MODE, XT>(w, t, (const XT *)x, base, aux, nullptr, total, k, body, record, 1, st);      \
  } while (0)
  if (x_dtype == CC_BF16) {
    if (mode == CC_WITH_FEEDBACK) CC_TK(CC_WITH_FEEDBACK, __nv_bfloat16);
    else if (mode == CC_NO_FEEDBACK) CC_TK(CC_NO_FEEDBACK, __nv_bfloat16);
    else CC_TK(CC_NAIVE, __nv_bfloat16);
  } else {
    if (mode == CC_WITH_FEEDBACK) CC_TK(CC_WITH_FEEDBACK, float);
    else if (mode == CC_NO_FEEDBACK) CC_TK(CC_NO_FEEDBACK, float);
    else CC_TK(CC_NAIVE, float);
  }
#undef CC_TK
  return cuda_status("topk_encode_step");
}

// accumulate: 0 replace (zero + scatter), 1 sparse add, 2 canonicalise -0.0 then sparse add
int topk_decode(int count, const int64_t *rows, int64_t C, int64_t k, const uint8_t *const *bodies, int accumulate,
                float *const *bases, cudaStream_t st) {
  for (int c0 = 0; c0 < count; c0 += topk::kMaxPeers) {
    const int cnt = std::min(topk::kMaxPeers, count - c0);
    topk::Peers pp{};
    int64_t maxk = 0, maxt = 0;
    for (int i = 0; i < cnt; ++i) {
      pp.body[i] = bodies[c0 + i];
      pp.base[i] = bases[c0 + i];
      pp.total[i] = rows[c0 + i] * C;
      pp.k[i] = k;
      maxk = std::max(maxk, k);
      maxt = std::max(maxt, pp.total[i]);
    }
    if (accumulate != 1) {
      dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(maxt, topk::kThreads), sm_count() * 4)), cnt);
      topk::k_canon<<<g, topk::kThreads, 0, st>>>(pp, accumulate == 0);
      count_launch();
    }
    if (maxk > 0) {
      dim3 g((unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(maxk, topk::kThreads), sm_count() * 4)), cnt);
      topk::k_scatter<<<g, topk::kThreads, 0, st>>>(pp, accumulate == 0);
      count_launch();
    }
  }
  return cuda_status("topk_decode");
}

}  // namespace cc
