// K4, shard-resident form: the whole top-k encode_step (compressors.py:446-456,
// pipeline.py:99-120) in ONE persistent cooperative kernel with the shard's
// residual t kept in shared memory across the grid-wide selection.
//
// Reference semantics (restated in oracle/cc_oracle.py): k = min(s, ceil(f s));
// order |t| descending, flat index ascending (np.lexsort); indices emitted
// ascending as u32, values as f16 (RNE, overflow -> inf); decode = dense zero +
// scatter, so base' = base + decoded is base + 0.0 (-0.0 -> +0.0) off the
// selection and feedback' = t - decoded is t there.
//
// Selection = exact radix select on key = bits(t) & 0x7fffffff (orders like |t|
// for finite t, +0 and -0 alike).  CTA c owns the contiguous elements
// [e0_c, e1_c) (multiples of 8, the last CTA takes the tail):
//   phase A   x / aux / base of the CTA's range -> shared memory by three 1-D TMA
//             bulk copies (when they fit; else 128-bit register loads, t only);
//             t = target(x, base, aux) (pipeline.py:99-104) kept in shared memory and
//             written where the step needs it (feedback' = t off the selection);
//             base -0.0 -> +0.0 (naive: base = 0, no-feedback: ref = x); ||t||^2
//   level 1   4096-bin histogram of key[30:19] -> the CTAs' non-empty bins added
//             into a global histogram -> grid barrier -> every CTA scans it the same
//             way: bin b1 holding the k-th largest key, and how many are still needed
//   candidates (when bin b1 holds <= kCandCap keys in total): every CTA appends its
//             keys in b1 (19-bit suffix, tagged with the CTA) to a global list and
//             publishes its count of keys above b1 -> grid barrier -> every CTA
//             selects the exact threshold key T and the tie count from the list (two
//             radix levels over it) and, from the same list, the number of selected
//             elements of the CTAs below it: no further barrier
//   fallback  (bin b1 too full) two more global histogram levels key[18:7], key[6:0]
//             and a count barrier, as in the multi-kernel select (topk.cu)
//   write     warps own contiguous segments: warp scans give every selected element
//             its slot in index order (no sort); f16 values; sparse state update
//             base[e] += d, feedback[e] = t - d (pipeline.py:107-112), base read from
//             shared memory when it is resident
//   record    last-CTA ticket: ||d - t||^2 = ||t||^2 + sum_sel((d - t)^2 - t^2)
// HBM bytes per element: x 2 + base 4 + aux 4 read, feedback 4 written (+ the
// selection's O(f) bytes): 14 B, one pass.  Histograms, list counter and barrier
// words live in a library-owned per-stream slab that every launch leaves zeroed.
#include <cstdlib>
#include "cc_async.cuh"
#include "cc_common.cuh"
#include "cc_internal.h"

#include <algorithm>

namespace cc {
namespace k4r {

constexpr int kThreads = 512, kWarps = kThreads / 32;
constexpr int kBins = 4096, kBins3 = 128;
constexpr int kU = 4;                 // quads in flight per thread (register phase A)
constexpr uint32_t kCandCap = 32768;  // largest bin-b1 population for the list path
constexpr size_t kSmemMax = 227 * 1024;
constexpr int kLB = 8;                // candidate-list loads in flight per thread

struct Slab {  // zero between launches
  uint32_t hist1[kBins], hist2[kBins], hist3[kBins3];
  uint32_t bar[4][32];  // one 128-byte line per barrier counter
  uint32_t ticket[32];
  uint32_t cand_count[32];
};

struct Params {
  const void *x;
  float *base, *aux, *tout;
  int64_t total, k, noct;
  int G, fit, nsm, write_t;  // fit: x / aux / base of every CTA in shared memory; else t of nsm quads
  uint32_t off_t, off_b;     // shared-memory offsets (the staging / histogram area U is at 0)
  uint32_t off_l, lcap;      // shared-memory copy of the candidate list (lcap entries; 0 = read it from L2)
  uint8_t *body;
  double *record, *recpart;  // [2], [G][2]
  uint32_t *cnt;             // [G][2]: key > T, key == T (fallback) / [G]: keys above b1 (list)
  uint32_t *cand;            // [kCandCap] (cta << 19 | key[18:0]) of the keys in bin b1
  Slab *slab;
  unsigned long long *timer;  // profiling: [G][16] %globaltimer stamps, or null
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t key_of(float t) { return __float_as_uint(t) & 0x7fffffffu; }

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// grid-wide barrier over the G co-resident CTAs (cooperative launch)
__device__ __forceinline__ void grid_barrier(unsigned *ctr, unsigned G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    while (ld_acquire(ctr) < G) {
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t warp_incl(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

__device__ __forceinline__ uint32_t block_sum(uint32_t v, uint32_t *sm) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) sm[threadIdx.x >> 5] = v;
  __syncthreads();
  uint32_t s = 0;
  for (int i = 0; i < kWarps; ++i) s += sm[i];
  __syncthreads();
  return s;
}

// Suffix scan of a histogram from the top bin (global: __ldcg; shared: plain), done
// identically by every CTA: the bin holding the need-th largest key and how many are
// still needed inside it.
template <int NB, bool GLOBAL>
__device__ __forceinline__ void find_bin(const uint32_t *hist, uint32_t need, uint32_t &bin, uint32_t &rem,
                                         uint32_t *sm /* [kWarps + 2] */) {
  constexpr int PER = (NB + kThreads - 1) / kThreads;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t v[PER], local = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {  // thread t owns bins NB-1-t*PER-q (descending)
    const int b = NB - 1 - (t * PER + q);
    v[q] = b >= 0 ? (GLOBAL ? __ldcg(hist + b) : hist[b]) : 0u;
    local += v[q];
  }
  uint32_t incl = warp_incl(local);
  if (lane == 31) sm[w] = incl;
  __syncthreads();
  if (w == 0) {  // exclusive prefix of the warp totals, in place
    const uint32_t v = lane < kWarps ? sm[lane] : 0u;
    const uint32_t vi = warp_incl(v);
    if (lane < kWarps) sm[lane] = vi - v;
  }
  __syncthreads();
  incl += sm[w];
  uint32_t before = incl - local;
  if (before < need && incl >= need) {
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = NB - 1 - (t * PER + q);
      if (b < 0) break;
      if (before + v[q] >= need) {
        sm[kWarps] = (uint32_t)b;
        sm[kWarps + 1] = need - before;
        break;
      }
      before += v[q];
    }
  }
  __syncthreads();
  bin = sm[kWarps];
  rem = sm[kWarps + 1];
  __syncthreads();
}

// candidate list entry: shared-memory copy or L2 (generic pointer; __ldcg only for global)
__device__ __forceinline__ uint32_t ld_list(const uint32_t *l, uint32_t i) {
  return __isShared(l) ? l[i] : __ldcg(l + i);
}

__device__ __forceinline__ void quad_vals(const float4 &v, float (&t)[4]) {
  t[0] = v.x;
  t[1] = v.y;
  t[2] = v.z;
  t[3] = v.w;
}

// register-capped (112) so the previous layer's sparse decode (a small scatter kernel on
// the decode stream) can share the SMs while this kernel waits at its barriers
template <int MODE, typename XT>
__global__ void __maxnreg__(112) k4_resident(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint32_t *h = reinterpret_cast<uint32_t *>(smem);  // area U: x staging (fit), then histograms
  float *tS = reinterpret_cast<float *>(smem + p.off_t);
  float *bS = reinterpret_cast<float *>(smem + p.off_b);
  __shared__ uint32_t sm[kWarps + 2];
  __shared__ uint32_t wgt[kWarps], weq[kWarps], wsel_base[kWarps], weq_base[kWarps];
  __shared__ double red[kWarps][2];
  __shared__ uint32_t s_pre[4];
  __shared__ unsigned last;
  __shared__ __align__(8) uint64_t mb;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = blockIdx.x, G = p.G;
  const int64_t e0 = 8 * ((int64_t)cta * p.noct / G);
  const int64_t e1 = cta == G - 1 ? p.total : 8 * ((int64_t)(cta + 1) * p.noct / G);
  const int ne = (int)(e1 - e0);  // elements of this CTA
  const int nqc = (ne + 3) >> 2;  // quads (the last may be partial)
  Slab *S = p.slab;
  const XT *X = reinterpret_cast<const XT *>(p.x);
  constexpr bool kAux = MODE != CC_NAIVE;
  const bool fit = p.fit != 0;
  auto stamp = [&](int i) {
    if (p.timer && tid == 0) p.timer[(size_t)cta * 16 + i] = gtimer();
  };
  stamp(0);

  if (tid == 0) {
    mbar_init(&mb, 1);
    mbar_fence_init();
  }
  __syncthreads();

  // ---------------- phase A ----------------
  double tsq = 0.0;
  uint32_t a_phases = 0;  // completed phases of mb
  if (fit) {
    XT *xS = reinterpret_cast<XT *>(smem);
    const int nb = ne & ~7;  // bulk part (16-byte multiples for every array)
    if (tid == 0 && nb > 0) {
      const uint64_t pol = l2_policy_evict_first();
      const uint32_t bx = (uint32_t)(nb * sizeof(XT)), bf = (uint32_t)(nb * 4);
      mbar_expect_tx(&mb, bx + (kAux ? 2 * bf : 0));
      bulk_g2s(xS, X + e0, bx, &mb, pol);
      if constexpr (kAux) {
        bulk_g2s(tS, p.aux + e0, bf, &mb, pol);
        bulk_g2s(bS, p.base + e0, bf, &mb, l2_policy_evict_last());  // written back at the selection
      }
    }
    if (tid < ne - nb) {  // the last CTA's tail (< 8 elements)
      const int i = nb + tid;
      xS[i] = X[e0 + i];
      if constexpr (kAux) {
        tS[i] = p.aux[e0 + i];
        bS[i] = p.base[e0 + i];
      }
    }
    if (nb > 0) {
      mbar_wait(&mb, 0);
      a_phases = 1;
    }
    __syncthreads();
    for (int q = tid; q < nqc; q += kThreads) {
      const int i = 4 * q;
      const int nv = min(4, ne - i);
      const int64_t e = e0 + i;
      float x[4] = {0.f, 0.f, 0.f, 0.f}, b[4] = {0.f, 0.f, 0.f, 0.f}, a[4] = {0.f, 0.f, 0.f, 0.f}, t[4];
      if (nv == 4) {
        if constexpr (sizeof(XT) == 2) {
          const uint2 r = *reinterpret_cast<const uint2 *>(xS + i);
          x[0] = __uint_as_float(r.x << 16);
          x[1] = __uint_as_float(r.x & 0xffff0000u);
          x[2] = __uint_as_float(r.y << 16);
          x[3] = __uint_as_float(r.y & 0xffff0000u);
        } else {
          quad_vals(*reinterpret_cast<const float4 *>(xS + i), x);
        }
        if constexpr (kAux) {
          quad_vals(*reinterpret_cast<const float4 *>(bS + i), b);
          quad_vals(*reinterpret_cast<const float4 *>(tS + i), a);
        }
      } else {
        for (int j = 0; j < nv; ++j) {
          x[j] = Act<XT>::load1(xS + i + j);
          if constexpr (kAux) {
            b[j] = bS[i + j];
            a[j] = tS[i + j];
          }
        }
      }
      bool neg0 = false;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        t[j] = target_of<MODE>(x[j], b[j], a[j]);
        if constexpr (kAux) {
          if (__float_as_uint(b[j]) == 0x80000000u) {  // dense base + 0.0 (pipeline.py:110)
            b[j] = 0.0f;
            neg0 = true;
          }
        }
        if (j < nv) tsq += (double)t[j] * (double)t[j];
      }
      if (nv == 4) {
        *reinterpret_cast<float4 *>(tS + i) = make_float4(t[0], t[1], t[2], t[3]);
        if (p.write_t) *reinterpret_cast<float4 *>(p.tout + e) = make_float4(t[0], t[1], t[2], t[3]);
        if constexpr (MODE == CC_NAIVE) {
          __stcs(reinterpret_cast<float4 *>(p.base + e), make_float4(0.f, 0.f, 0.f, 0.f));  // base' = decoded
        } else if (neg0) {
          *reinterpret_cast<float4 *>(bS + i) = make_float4(b[0], b[1], b[2], b[3]);
          *reinterpret_cast<float4 *>(p.base + e) = make_float4(b[0], b[1], b[2], b[3]);
        }
        if constexpr (MODE == CC_NO_FEEDBACK)
          __stcs(reinterpret_cast<float4 *>(p.aux + e), make_float4(x[0], x[1], x[2], x[3]));  // ref' = a*
      } else {
        for (int j = 0; j < nv; ++j) {
          tS[i + j] = t[j];
          if (p.write_t) p.tout[e + j] = t[j];
          if constexpr (MODE == CC_NAIVE) {
            p.base[e + j] = 0.0f;
          } else if (neg0) {
            bS[i + j] = b[j];
            p.base[e + j] = b[j];
          }
          if constexpr (MODE == CC_NO_FEEDBACK) p.aux[e + j] = x[j];
        }
      }
    }
    __syncthreads();  // x staging is dead: area U becomes the histogram
    for (int b = tid; b < kBins; b += kThreads) h[b] = 0u;
    __syncthreads();
    for (int i = tid; i < ne; i += kThreads) atomicAdd(&h[key_of(tS[i]) >> 19], 1u);
  } else {
    for (int b = tid; b < kBins; b += kThreads) h[b] = 0u;
    __syncthreads();
    for (int i0 = 0; i0 < nqc; i0 += kThreads * kU) {
      float4 xv[kU], bv[kU], av[kU];
      int nv[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {  // every load of the thread in flight together
        const int i = i0 + u * kThreads + tid;
        const int64_t e = e0 + 4 * (int64_t)i;
        nv[u] = i < nqc ? min(4, ne - 4 * i) : 0;
        xv[u] = bv[u] = av[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (nv[u] == 4) {
          xv[u] = Act<XT>::load4(X + e);
          if constexpr (kAux) {
            bv[u] = *reinterpret_cast<const float4 *>(p.base + e);
            av[u] = __ldcs(reinterpret_cast<const float4 *>(p.aux + e));
          }
        } else if (nv[u] > 0) {
          float xs[4] = {0.f, 0.f, 0.f, 0.f}, bs[4] = {0.f, 0.f, 0.f, 0.f}, as[4] = {0.f, 0.f, 0.f, 0.f};
          for (int j = 0; j < nv[u]; ++j) {
            xs[j] = Act<XT>::load1(X + e + j);
            if constexpr (kAux) {
              bs[j] = p.base[e + j];
              as[j] = p.aux[e + j];
            }
          }
          xv[u] = make_float4(xs[0], xs[1], xs[2], xs[3]);
          bv[u] = make_float4(bs[0], bs[1], bs[2], bs[3]);
          av[u] = make_float4(as[0], as[1], as[2], as[3]);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        if (nv[u] == 0) continue;
        const int i = i0 + u * kThreads + tid;
        const int64_t e = e0 + 4 * (int64_t)i;
        float x[4], b[4], a[4], t[4];
        quad_vals(xv[u], x);
        quad_vals(bv[u], b);
        quad_vals(av[u], a);
        bool neg0 = false;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          t[j] = target_of<MODE>(x[j], b[j], a[j]);
          if constexpr (kAux) neg0 |= __float_as_uint(b[j]) == 0x80000000u;
        }
        const float4 tv = make_float4(t[0], t[1], t[2], t[3]);
        if (i < p.nsm) reinterpret_cast<float4 *>(tS)[i] = tv;
        if (nv[u] == 4) {
          if (p.write_t) *reinterpret_cast<float4 *>(p.tout + e) = tv;
          if constexpr (MODE == CC_NAIVE) {
            __stcs(reinterpret_cast<float4 *>(p.base + e), make_float4(0.f, 0.f, 0.f, 0.f));
          } else if (neg0) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
              if (__float_as_uint(b[j]) == 0x80000000u) b[j] = 0.0f;
            *reinterpret_cast<float4 *>(p.base + e) = make_float4(b[0], b[1], b[2], b[3]);
          }
          if constexpr (MODE == CC_NO_FEEDBACK) __stcs(reinterpret_cast<float4 *>(p.aux + e), xv[u]);
        } else {
          for (int j = 0; j < nv[u]; ++j) {
            if (p.write_t) p.tout[e + j] = t[j];
            if constexpr (MODE == CC_NAIVE) p.base[e + j] = 0.0f;
            else if (__float_as_uint(b[j]) == 0x80000000u) p.base[e + j] = 0.0f;
            if constexpr (MODE == CC_NO_FEEDBACK) p.aux[e + j] = x[j];
          }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j < nv[u]) {
            tsq += (double)t[j] * (double)t[j];
            atomicAdd(&h[key_of(t[j]) >> 19], 1u);
          }
        }
      }
    }
  }
  // one quad of t: shared memory when resident, else the t buffer (written above)
  auto t_quad = [&](int q, float (&t)[4], int &nv) {
    nv = min(4, ne - 4 * q);
    if (fit) {
      if (nv == 4) {
        quad_vals(*reinterpret_cast<const float4 *>(tS + 4 * q), t);
      } else {
        for (int j = 0; j < 4; ++j) t[j] = j < nv ? tS[4 * q + j] : 0.0f;
      }
    } else if (q < p.nsm) {
      quad_vals(reinterpret_cast<const float4 *>(tS)[q], t);
    } else if (nv == 4) {
      quad_vals(__ldcg(reinterpret_cast<const float4 *>(p.tout + e0) + q), t);
    } else {
      for (int j = 0; j < 4; ++j) t[j] = j < nv ? __ldcg(p.tout + e0 + 4 * q + j) : 0.0f;
    }
  };
  __syncthreads();
  stamp(1);
  for (int b = tid; b < kBins; b += kThreads) {
    const uint32_t c = h[b];
    if (c) atomicAdd(&S->hist1[b], c);
  }
  grid_barrier(&S->bar[0][0], (unsigned)G);
  stamp(2);
  uint32_t b1, need;
  find_bin<kBins, true>(S->hist1, (uint32_t)p.k, b1, need, sm);
  const uint32_t in_b1 = __ldcg(&S->hist1[b1]);
  stamp(3);
  if (p.timer && tid == 0) {  // profiling: bin-b1 population and the path taken
    p.timer[(size_t)cta * 16 + 12] = in_b1;
    p.timer[(size_t)cta * 16 + 13] = in_b1 <= kCandCap;
  }

  uint32_t T, ties;
  if (in_b1 <= kCandCap) {
    // ---- candidates: keys in bin b1 to the global list; keys above b1 counted ----
    uint32_t above = 0, nc = 0;
    for (int q = tid; q < nqc; q += kThreads) {
      float t[4];
      int nv;
      t_quad(q, t, nv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t hb = key_of(t[j]) >> 19;
        above += (j < nv) & (hb > b1);
        nc += (j < nv) & (hb == b1);
      }
    }
    const uint32_t nc_cta = block_sum(nc, sm);
    const uint32_t above_cta = block_sum(above, sm);
    if (tid == 0) {
      s_pre[0] = nc_cta ? atomicAdd(&S->cand_count[0], nc_cta) : 0u;
      p.cnt[cta] = above_cta;
    }
    {
      // slots in thread order: exclusive scan of the per-thread counts
      const uint32_t incl = warp_incl(nc);
      if (lane == 31) wgt[warp] = incl;
      __syncthreads();
      uint32_t off = s_pre[0] + incl - nc;
      for (int w = 0; w < warp; ++w) off += wgt[w];
      if (nc) {
        for (int q = tid; q < nqc; q += kThreads) {
          float t[4];
          int nv;
          t_quad(q, t, nv);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t key = key_of(t[j]);
            if (j < nv && (key >> 19) == b1) p.cand[off++] = ((uint32_t)cta << 19) | (key & 0x7ffffu);
          }
        }
      }
    }
    grid_barrier(&S->bar[1][0], (unsigned)G);
    stamp(4);
    const uint32_t L = in_b1;
    // the list in shared memory when there is room: one bulk copy, then on-chip passes
    const uint32_t *cl = p.cand;
    if (L <= p.lcap) {
      uint32_t *ls = reinterpret_cast<uint32_t *>(smem + p.off_l);
      const uint32_t lb = (L + 3) & ~3u;  // 16-byte multiple (the list buffer has the capacity)
      if (tid == 0) {
        asm volatile("fence.proxy.async.global;" ::: "memory");  // generic-proxy list writes -> bulk copy
        mbar_expect_tx(&mb, 4 * lb);
        bulk_g2s(ls, p.cand, 4 * lb, &mb, l2_policy_evict_first());
      }
      mbar_wait(&mb, a_phases);  // phases completed so far by phase A's copy
      cl = ls;
    }
    // hist1 was read by every CTA before barrier 2: clear it for the next launch
    for (int i = cta * kThreads + tid; i < kBins; i += G * kThreads) S->hist1[i] = 0u;
    stamp(5);
    // ---- exact threshold from the list: suffix[18:9], then suffix[8:0] ----
    for (int b = tid; b < 1024; b += kThreads) h[b] = 0u;
    __syncthreads();
    // list passes: kLB loads of a thread in flight together (the list lives in L2)
    for (uint32_t i0 = tid; i0 < L; i0 += kLB * kThreads) {
      uint32_t c[kLB];
#pragma unroll
      for (int u = 0; u < kLB; ++u) c[u] = i0 + u * kThreads < L ? ld_list(cl, i0 + u * kThreads) : ~0u;
#pragma unroll
      for (int u = 0; u < kLB; ++u)
        if (c[u] != ~0u) atomicAdd(&h[(c[u] >> 9) & 1023u], 1u);
    }
    __syncthreads();
    uint32_t ba, needa;
    find_bin<1024, false>(h, need, ba, needa, sm);
    stamp(7);
    for (int b = tid; b < 512; b += kThreads) h[b] = 0u;
    __syncthreads();
    for (uint32_t i0 = tid; i0 < L; i0 += kLB * kThreads) {
      uint32_t c[kLB];
#pragma unroll
      for (int u = 0; u < kLB; ++u) c[u] = i0 + u * kThreads < L ? ld_list(cl, i0 + u * kThreads) : ~0u;
#pragma unroll
      for (int u = 0; u < kLB; ++u)
        if (c[u] != ~0u && ((c[u] >> 9) & 1023u) == ba) atomicAdd(&h[c[u] & 511u], 1u);
    }
    __syncthreads();
    uint32_t bb;
    find_bin<512, false>(h, needa, bb, ties, sm);
    stamp(8);
    const uint32_t ts = (ba << 9) | bb;
    T = (b1 << 19) | ts;
    // ---- selected / tie totals of the CTAs below this one ----
    uint32_t gt = 0, eq = 0;
    for (uint32_t i0 = tid; i0 < L; i0 += kLB * kThreads) {
      uint32_t c[kLB];
#pragma unroll
      for (int u = 0; u < kLB; ++u) c[u] = i0 + u * kThreads < L ? ld_list(cl, i0 + u * kThreads) : ~0u;
#pragma unroll
      for (int u = 0; u < kLB; ++u)
        if (c[u] != ~0u && (int)(c[u] >> 19) < cta) {
          gt += (c[u] & 0x7ffffu) > ts;
          eq += (c[u] & 0x7ffffu) == ts;
        }
    }
    for (int c = tid; c < cta; c += kThreads) gt += __ldcg(p.cnt + c);
    gt = block_sum(gt, sm);
    eq = block_sum(eq, sm);
    if (tid == 0) {
      s_pre[0] = eq;                            // ties below (index order)
      s_pre[1] = gt + (eq < ties ? eq : ties);  // selected below
    }
  } else {
    // ---- fallback: two more histogram levels and a count barrier ----
    for (int b = tid; b < kBins; b += kThreads) h[b] = 0u;
    __syncthreads();
    for (int q = tid; q < nqc; q += kThreads) {
      float t[4];
      int nv;
      t_quad(q, t, nv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = key_of(t[j]);
        if (j < nv && (key >> 19) == b1) atomicAdd(&h[(key >> 7) & 0xfffu], 1u);
      }
    }
    __syncthreads();
    for (int b = tid; b < kBins; b += kThreads) {
      const uint32_t c = h[b];
      if (c) atomicAdd(&S->hist2[b], c);
      h[b] = 0u;
    }
    grid_barrier(&S->bar[1][0], (unsigned)G);
    stamp(4);
    for (int i = cta * kThreads + tid; i < kBins; i += G * kThreads) S->hist1[i] = 0u;
    uint32_t b2;
    find_bin<kBins, true>(S->hist2, need, b2, need, sm);
    const uint32_t pre24 = (b1 << 12) | b2;
    for (int q = tid; q < nqc; q += kThreads) {
      float t[4];
      int nv;
      t_quad(q, t, nv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = key_of(t[j]);
        if (j < nv && (key >> 7) == pre24) atomicAdd(&h[key & 127u], 1u);
      }
    }
    __syncthreads();
    for (int b = tid; b < kBins3; b += kThreads) {
      const uint32_t c = h[b];
      if (c) atomicAdd(&S->hist3[b], c);
    }
    grid_barrier(&S->bar[2][0], (unsigned)G);
    uint32_t b3;
    find_bin<kBins3, true>(S->hist3, need, b3, ties, sm);
    T = (pre24 << 7) | b3;
    uint32_t gt = 0, eq = 0;
    for (int q = tid; q < nqc; q += kThreads) {
      float t[4];
      int nv;
      t_quad(q, t, nv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = key_of(t[j]);
        gt += (j < nv) & (key > T);
        eq += (j < nv) & (key == T);
      }
    }
    gt = block_sum(gt, sm);
    eq = block_sum(eq, sm);
    if (tid == 0) {
      p.cnt[2 * cta] = gt;
      p.cnt[2 * cta + 1] = eq;
    }
    grid_barrier(&S->bar[3][0], (unsigned)G);
    for (int i = cta * kThreads + tid; i < kBins + kBins3; i += G * kThreads) S->hist2[i] = 0u;  // hist2 | hist3
    if (warp == 0) {
      uint32_t eq_carry = 0, sel_carry = 0;
      for (int c0 = 0; c0 < cta; c0 += 32) {
        const int c = c0 + lane;
        const uint32_t g = c < cta ? __ldcg(p.cnt + 2 * c) : 0u;
        const uint32_t q = c < cta ? __ldcg(p.cnt + 2 * c + 1) : 0u;
        const uint32_t incl = warp_incl(q);
        const uint32_t before = eq_carry + incl - q;
        const uint32_t taken = before < ties ? min(q, ties - before) : 0u;
        uint32_t sel = g + taken;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) sel += __shfl_xor_sync(0xffffffffu, sel, o);
        eq_carry += __shfl_sync(0xffffffffu, incl, 31);
        sel_carry += sel;
      }
      if (lane == 0) {
        s_pre[0] = eq_carry;
        s_pre[1] = sel_carry;
      }
    }
  }
  stamp(9);

  // ---------------- per-warp counts of this CTA, warp bases ----------------
  const int wq0 = warp * nqc / kWarps, wq1 = (warp + 1) * nqc / kWarps;
  {
    uint32_t gt = 0, eq = 0;
    for (int q = wq0 + lane; q < wq1; q += 32) {
      float t[4];
      int nv;
      t_quad(q, t, nv);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = key_of(t[j]);
        gt += (j < nv) & (key > T);
        eq += (j < nv) & (key == T);
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      gt += __shfl_xor_sync(0xffffffffu, gt, o);
      eq += __shfl_xor_sync(0xffffffffu, eq, o);
    }
    if (lane == 0) {
      wgt[warp] = gt;
      weq[warp] = eq;
    }
  }
  __syncthreads();
  stamp(6);
  if (tid == 0) {
    uint32_t eqb = s_pre[0], selb = s_pre[1];
    for (int w = 0; w < kWarps; ++w) {
      weq_base[w] = eqb;
      wsel_base[w] = selb;
      const uint32_t taken = eqb < ties ? min(weq[w], ties - eqb) : 0u;
      eqb += weq[w];
      selb += wgt[w] + taken;
    }
  }
  __syncthreads();

  // ---------------- ordered write + sparse state update ----------------
  double adj = 0.0;  // sum over selected of (d - t)^2 - t^2
  {
    uint32_t eq_run = weq_base[warp], pos_run = wsel_base[warp];
    uint32_t *idx_out = reinterpret_cast<uint32_t *>(p.body);
    __half *val_out = reinterpret_cast<__half *>(p.body + 4 * p.k);
    for (int c0 = wq0; c0 < wq1; c0 += 32) {
      const int q = c0 + lane;
      float t[4] = {0.f, 0.f, 0.f, 0.f};
      int nv = 0;
      if (q < wq1) t_quad(q, t, nv);
      uint32_t mgt = 0, meq = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = key_of(t[j]);
        mgt |= (uint32_t)((j < nv) & (key > T)) << j;
        meq |= (uint32_t)((j < nv) & (key == T)) << j;
      }
      uint32_t msel = mgt;
      if (__any_sync(0xffffffffu, meq != 0u)) {  // ties in this chunk: their ranks (lowest index first)
        const uint32_t neq = __popc(meq);
        const uint32_t ie = warp_incl(neq);
        uint32_t er = eq_run + ie - neq;  // tie rank of this lane's first tie
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if ((meq >> j) & 1u) {
            if (er < ties) msel |= 1u << j;
            ++er;
          }
        eq_run += __shfl_sync(0xffffffffu, ie, 31);
      }
      const uint32_t ns = __popc(msel);
      const uint32_t is = warp_incl(ns);
      uint32_t pos = pos_run + is - ns;
      pos_run += __shfl_sync(0xffffffffu, is, 31);
      if (msel) {
        float bb[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (MODE != CC_NAIVE) {  // all of this lane's base reads in flight together
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if ((msel >> j) & 1u) bb[j] = fit ? bS[4 * q + j] : p.base[e0 + 4 * q + j];
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (!((msel >> j) & 1u)) continue;
          const int64_t e = e0 + 4 * q + j;
          const float tv = t[j];
          const __half hv = __float2half_rn(tv);
          idx_out[pos] = (uint32_t)e;
          val_out[pos] = hv;
          ++pos;
          const float d = __half2float(hv);
          const double df = (double)d - (double)tv;
          adj += df * df - (double)tv * (double)tv;
          if constexpr (MODE == CC_NAIVE) {
            p.base[e] = d;
          } else {
            p.base[e] = __fadd_rn(bb[j], d);
            if constexpr (MODE == CC_WITH_FEEDBACK) p.aux[e] = __fsub_rn(tv, d);
          }
        }
      }
    }
  }
  stamp(10);

  // ---------------- StepRecord: last-CTA ticket ----------------
  {
    const double a = warp_sum(adj), b = warp_sum(tsq);
    if (lane == 0) {
      red[warp][0] = a;
      red[warp][1] = b;
    }
    __syncthreads();
    if (tid == 0) {
      double sa = 0.0, sb = 0.0;
      for (int w = 0; w < kWarps; ++w) {
        sa += red[w][0];
        sb += red[w][1];
      }
      p.recpart[2 * cta] = sa;
      p.recpart[2 * cta + 1] = sb;
      __threadfence();
      last = atomicAdd(&S->ticket[0], 1u) == (unsigned)G - 1;
    }
    __syncthreads();
    if (last) {
      __threadfence();
      double sa = 0.0, sb = 0.0;
      for (int c = tid; c < G; c += kThreads) {
        sa += __ldcg(p.recpart + 2 * c);
        sb += __ldcg(p.recpart + 2 * c + 1);
      }
      sa = warp_sum(sa);
      sb = warp_sum(sb);
      __syncthreads();
      if (lane == 0) {
        red[warp][0] = sa;
        red[warp][1] = sb;
      }
      __syncthreads();
      if (tid == 0) {
        double ta = 0.0, tb = 0.0;
        for (int w = 0; w < kWarps; ++w) {
          ta += red[w][0];
          tb += red[w][1];
        }
        p.record[0] = tb + ta;  // ||d - t||^2 (pipeline.py:117)
        p.record[1] = tb;       // ||t||^2
        // every CTA is past every barrier: leave the slab's words zeroed
        S->bar[0][0] = S->bar[1][0] = S->bar[2][0] = S->bar[3][0] = 0u;
        S->ticket[0] = 0u;
        S->cand_count[0] = 0u;
      }
    }
  }
  stamp(11);
}

}  // namespace k4r

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
uint8_t *stream_zero_slab(cudaStream_t st, size_t bytes);

static int g_topk_resident = 1;  // 0 off, 1 when t fits on chip, 2 also when it does not (A/B)
static unsigned long long *g_topk_timer = nullptr;
void set_topk_timer(void *buf) { g_topk_timer = reinterpret_cast<unsigned long long *>(buf); }
void set_topk_resident_enabled(int on) { g_topk_resident = on; }
std::atomic<int64_t> g_topk_resident_launches{0};
int64_t topk_resident_launches() { return g_topk_resident_launches.load(); }

// per-CTA counts, record partials and the candidate list
int64_t topk_resident_workspace_bytes() {
  return (int64_t)(align_up(8 * 256, 256) + align_up(16 * 256, 256) + align_up(4 * (size_t)k4r::kCandCap, 256));
}

int topk_resident_encode_step(int mode, int64_t n, int64_t C, int64_t k, const void *x, int x_dtype, float *base,
                              float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record,
                              cudaStream_t st) {
  using namespace k4r;
  if (!g_topk_resident) return CC_ERR_UNSUPPORTED;
  const int64_t total = n * C;
  if (total >= (int64_t)1 << 32 || k < 1) return CC_ERR_UNSUPPORTED;
  if (!aligned(x, 16) || !aligned(base, 16) || (aux && !aligned(aux, 16)) || !aligned(body, 4))
    return CC_ERR_UNSUPPORTED;
  Params p{};
  p.x = x;
  p.base = base;
  p.aux = aux;
  p.total = total;
  p.k = k;
  p.noct = total / 8;
  // SMs left to the sparse decode running beside this kernel on the decode stream (the
  // previous layer's peers): it only overlaps on SMs this kernel leaves empty.  Worth it
  // for heavy decodes: per-rank P = 8 [512, 3072] 10 %: 47.9 -> 41.8 us per layer with 16
  // SMs free; 1 %: 32.7 -> 33.1 (kept at 0).  CC_TOPK_RESIDENT_RESERVE overrides.
  static const int reserve_env = [] {
    const char *e = std::getenv("CC_TOPK_RESIDENT_RESERVE");
    return e ? std::atoi(e) : -1;
  }();
  const int reserve = reserve_env >= 0 ? reserve_env : (k * 20 >= total ? 16 : 0);
  p.G = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, sm_count() - reserve), cdiv(total, 2048)));
  if (p.G > 255) return CC_ERR_UNSUPPORTED;  // the candidate tag is 8 bits
  // largest CTA range (the last one takes the tail)
  const int64_t ne_max = 8 * cdiv(p.noct, p.G) + 8;
  const size_t xb = x_dtype == CC_BF16 ? 2 : 4;
  const bool aux_mode = mode != CC_NAIVE;
  const size_t budget = kSmemMax - 2048;
  auto al = [](size_t v) { return align_up(v, 128); };
  // fit: area U = max(histogram, x staging), then t and base (aux modes)
  const size_t areaU = al(std::max<size_t>(4 * kBins, xb * ne_max));
  const size_t fit_bytes = areaU + al(4 * ne_max) + (aux_mode ? al(4 * ne_max) : 0);
  size_t smem;
  if (fit_bytes <= budget) {
    p.fit = 1;
    p.off_t = (uint32_t)areaU;
    p.off_b = (uint32_t)(areaU + al(4 * ne_max));
    p.nsm = 0;
    smem = fit_bytes;
  } else {
    p.fit = 0;
    p.off_t = (uint32_t)al(4 * kBins);
    p.off_b = 0;
    p.nsm = (int)std::min<int64_t>(cdiv(ne_max, 4), (int64_t)((budget - p.off_t) / 16));
    smem = p.off_t + 16 * (size_t)p.nsm;
  }
  // the rest of shared memory holds a copy of the candidate list when it is short enough
  smem = al(smem);
  p.off_l = (uint32_t)smem;
  p.lcap = smem + 4096 <= budget ? (uint32_t)std::min<size_t>(kCandCap, (budget - smem) / 4) & ~3u : 0u;
  smem += 4 * (size_t)p.lcap;
  const bool t_on_chip = p.fit || (int64_t)p.nsm * 4 >= ne_max;
  // shards whose residual stays off chip: the multi-kernel select is faster there
  if (!t_on_chip && g_topk_resident < 2) return CC_ERR_UNSUPPORTED;
  Slab *slab = reinterpret_cast<Slab *>(stream_zero_slab(st, sizeof(Slab)));
  if (!slab) return CC_ERR_UNSUPPORTED;
  uint8_t *w = reinterpret_cast<uint8_t *>(ws);
  size_t off = 0;
  auto take = [&](size_t b) {
    uint8_t *q = w + off;
    off = align_up(off + b, 256);
    return q;
  };
  p.cnt = reinterpret_cast<uint32_t *>(take(8 * (size_t)p.G));
  p.recpart = reinterpret_cast<double *>(take(16 * (size_t)p.G));
  p.cand = reinterpret_cast<uint32_t *>(take(4 * (size_t)kCandCap));
  if (mode == CC_WITH_FEEDBACK) {  // feedback' = t off the selection
    p.tout = aux;
    p.write_t = 1;
  } else {  // t kept nowhere else: scratch when it does not fit on chip
    p.tout = t_on_chip ? nullptr : reinterpret_cast<float *>(take(4 * (size_t)total));
    p.write_t = t_on_chip ? 0 : 1;
  }
  if ((int64_t)off > ws_bytes) return CC_ERR_UNSUPPORTED;
  p.body = body;
  p.record = record;
  p.slab = slab;
  p.timer = g_topk_timer;
  void *args[] = {&p};
  auto go = [&](const void *kern) -> int {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      cudaGetLastError();
      return CC_ERR_UNSUPPORTED;
    }
    const cudaError_t e = cudaLaunchCooperativeKernel(kern, dim3(p.G), dim3(kThreads), args, smem, st);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return CC_ERR_UNSUPPORTED;  // e.g. not enough co-resident CTAs now: the multi-kernel path
    }
    count_launch();
    g_topk_resident_launches.fetch_add(1, std::memory_order_relaxed);
    return CC_OK;
  };
#define CC_K4(MODE, XT) return go((const void *)k4_resident<MODE, XT>)
  if (x_dtype == CC_BF16) {
    if (mode == CC_WITH_FEEDBACK) CC_K4(CC_WITH_FEEDBACK, __nv_bfloat16);
    if (mode == CC_NO_FEEDBACK) CC_K4(CC_NO_FEEDBACK, __nv_bfloat16);
    CC_K4(CC_NAIVE, __nv_bfloat16);
  } else {
    if (mode == CC_WITH_FEEDBACK) CC_K4(CC_WITH_FEEDBACK, float);
    if (mode == CC_NO_FEEDBACK) CC_K4(CC_NO_FEEDBACK, float);
    CC_K4(CC_NAIVE, float);
  }
#undef CC_K4
}

}  // namespace cc
