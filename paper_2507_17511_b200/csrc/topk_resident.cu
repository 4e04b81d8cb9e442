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
// Radix select on key = bits(t) & 0x7fffffff (orders like |t| for finite t,
// +0 and -0 alike), three levels of 12 / 12 / 7 bits as in topk.cu, but with the
// levels' histograms reduced through global atomics of the CTAs' non-empty bins
// and a flag barrier between levels instead of separate launches:
//   phase A   t = target(x, base, aux) (pipeline.py:99-104) of the CTA's
//             contiguous quads -> shared memory (the part that fits) and, where
//             the step needs it, the feedback / scratch buffer; base -0.0 -> +0.0
//             (naive: base = 0, no-feedback: ref = x); ||t||^2; level-1 histogram
//   barrier   every CTA finds (b1, need) from the global histogram (same scan in
//             every CTA, so no broadcast step)
//   level 2   keys in b1: histogram of key[18:7] -> barrier -> (b2, need)
//   level 3   keys in (b1, b2): histogram of key[6:0] -> barrier -> threshold key
//             T and the number of ties at T to take (lowest indices first)
//   count     per-warp counts of key > T and key == T -> per-CTA totals -> barrier
//   write     each CTA's output offset from the totals of the CTAs below it; warps
//             own contiguous segments, so warp scans give every selected element
//             its slot in index order (no sort); f16 values; sparse state update
//             base[e] += d, feedback[e] = t - d (pipeline.py:107-112)
//   record    last-CTA ticket: ||d - t||^2 = ||t||^2 + sum_sel((d - t)^2 - t^2)
// Bytes: x 2 + base 4 + aux 4 read, feedback 4 written per element, plus the
// selection (14 + O(f) B/elem): one HBM pass.  Histograms / barrier words live in
// a library-owned per-stream slab that every launch leaves zeroed.
#include "cc_common.cuh"
#include "cc_internal.h"

#include <algorithm>

namespace cc {
namespace k4r {

constexpr int kThreads = 512, kWarps = kThreads / 32;
constexpr int kBins = 4096, kBins3 = 128;
constexpr int kU = 4;  // quads in flight per thread in phase A
constexpr size_t kSmemMax = 227 * 1024;

struct Slab {  // zero between launches
  uint32_t hist1[kBins], hist2[kBins], hist3[kBins3];
  uint32_t bar[4][32];  // one 128-byte line per barrier counter
  uint32_t ticket[32];
};

struct Params {
  const void *x;
  float *base, *aux, *tout;
  int64_t total, k, nq;
  int G, nsm, write_t;
  uint8_t *body;
  double *record, *recpart;  // [2], [G][2]
  uint32_t *cnt;             // [G][2]: key > T, key == T
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

// warp-inclusive scan (shuffles)
__device__ __forceinline__ uint32_t warp_incl(uint32_t v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += y;
  }
  return v;
}

// Suffix scan of a global histogram from the top bin, done identically by every
// CTA: the bin holding the need-th largest key and how many are still needed in it.
template <int NB>
__device__ __forceinline__ void find_bin(const uint32_t *__restrict__ hist, uint32_t need, uint32_t &bin,
                                         uint32_t &rem, uint32_t *sm /* [kWarps + 2] */) {
  constexpr int PER = (NB + kThreads - 1) / kThreads;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  uint32_t v[PER], local = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {  // thread t owns bins NB-1-t*PER-q (descending)
    const int b = NB - 1 - (t * PER + q);
    v[q] = b >= 0 ? __ldcg(hist + b) : 0u;
    local += v[q];
  }
  uint32_t incl = warp_incl(local);
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

// one quad of t: shared memory for the CTA's first nsm quads, else the t buffer
__device__ __forceinline__ float4 t_quad(const Params &p, const float4 *tS, int i, int64_t q) {
  return i < p.nsm ? tS[i] : __ldcg(reinterpret_cast<const float4 *>(p.tout) + q);
}

__device__ __forceinline__ void quad_vals(const float4 &v, float (&t)[4]) {
  t[0] = v.x;
  t[1] = v.y;
  t[2] = v.z;
  t[3] = v.w;
}

template <int MODE, typename XT>
__global__ void __launch_bounds__(kThreads, 1) k4_resident(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint32_t *h = reinterpret_cast<uint32_t *>(smem);          // [kBins] level histogram
  float4 *tS = reinterpret_cast<float4 *>(smem + 4 * kBins);  // [nsm] resident t quads
  __shared__ uint32_t sm[kWarps + 2];
  __shared__ uint32_t wgt[kWarps], weq[kWarps], wsel_base[kWarps], weq_base[kWarps];
  __shared__ double red[kWarps][2];
  __shared__ uint32_t s_pre[2];
  __shared__ unsigned last;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cta = blockIdx.x, G = p.G;
  const int64_t q0 = (int64_t)cta * p.nq / G, q1 = (int64_t)(cta + 1) * p.nq / G;
  const int nqc = (int)(q1 - q0);
  const int64_t total = p.total;
  Slab *S = p.slab;
  const XT *X = reinterpret_cast<const XT *>(p.x);
  constexpr bool kAux = MODE != CC_NAIVE;
  auto stamp = [&](int i) {
    if (p.timer && tid == 0) p.timer[(size_t)cta * 16 + i] = gtimer();
  };
  stamp(0);

  for (int b = tid; b < kBins; b += kThreads) h[b] = 0u;
  __syncthreads();

  // ---------------- phase A: target, residency, level-1 histogram ----------------
  double tsq = 0.0;
  for (int i0 = 0; i0 < nqc; i0 += kThreads * kU) {
    float4 xv[kU], bv[kU], av[kU];
    int nv[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {  // every load of the thread in flight together
      const int i = i0 + u * kThreads + tid;
      const int64_t e = 4 * (q0 + i);
      nv[u] = i < nqc ? (int)min64(4, total - e) : 0;
      xv[u] = bv[u] = av[u] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (nv[u] == 4) {
        xv[u] = Act<XT>::load4(X + e);
        if constexpr (kAux) {
          if constexpr (MODE == CC_WITH_FEEDBACK) bv[u] = *reinterpret_cast<const float4 *>(p.base + e);
          else bv[u] = __ldcs(reinterpret_cast<const float4 *>(p.base + e));
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
      const int64_t e = 4 * (q0 + i);
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
      if (i < p.nsm) tS[i] = tv;
      if (nv[u] == 4) {
        if (p.write_t) *reinterpret_cast<float4 *>(p.tout + e) = tv;
        if constexpr (MODE == CC_NAIVE) {
          __stcs(reinterpret_cast<float4 *>(p.base + e), make_float4(0.f, 0.f, 0.f, 0.f));  // base' = decoded
        } else if (neg0) {  // dense base + 0.0 (pipeline.py:110): -0.0 -> +0.0
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (__float_as_uint(b[j]) == 0x80000000u) b[j] = 0.0f;
          *reinterpret_cast<float4 *>(p.base + e) = make_float4(b[0], b[1], b[2], b[3]);
        }
        if constexpr (MODE == CC_NO_FEEDBACK) __stcs(reinterpret_cast<float4 *>(p.aux + e), xv[u]);  // ref' = a*
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
  __syncthreads();
  stamp(1);
  for (int b = tid; b < kBins; b += kThreads) {
    const uint32_t c = h[b];
    if (c) atomicAdd(&S->hist1[b], c);
    h[b] = 0u;
  }
  grid_barrier(&S->bar[0][0], (unsigned)G);
  stamp(2);
  uint32_t b1, need;
  find_bin<kBins>(S->hist1, (uint32_t)p.k, b1, need, sm);
  stamp(3);

  // ---------------- level 2: key[18:7] of the keys in bin b1 ----------------
  for (int i = tid; i < nqc; i += kThreads) {
    const int64_t q = q0 + i;
    float t[4];
    quad_vals(t_quad(p, tS, i, q), t);
    const int nv = (int)min64(4, total - 4 * q);
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
  stamp(4);
  grid_barrier(&S->bar[1][0], (unsigned)G);
  stamp(5);
  uint32_t b2;
  find_bin<kBins>(S->hist2, need, b2, need, sm);

  // ---------------- level 3: key[6:0] of the keys in (b1, b2) ----------------
  const uint32_t pre24 = (b1 << 12) | b2;
  for (int i = tid; i < nqc; i += kThreads) {
    const int64_t q = q0 + i;
    float t[4];
    quad_vals(t_quad(p, tS, i, q), t);
    const int nv = (int)min64(4, total - 4 * q);
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
  stamp(6);
  grid_barrier(&S->bar[2][0], (unsigned)G);
  stamp(7);
  uint32_t b3, ties;
  find_bin<kBins3>(S->hist3, need, b3, ties, sm);
  const uint32_t T = (pre24 << 7) | b3;

  // ---------------- count: per-warp segments ----------------
  const int wq0 = warp * nqc / kWarps, wq1 = (warp + 1) * nqc / kWarps;
  {
    uint32_t gt = 0, eq = 0;
    for (int i = wq0 + lane; i < wq1; i += 32) {
      const int64_t q = q0 + i;
      float t[4];
      quad_vals(t_quad(p, tS, i, q), t);
      const int nv = (int)min64(4, total - 4 * q);
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
  if (tid == 0) {
    uint32_t a = 0, b = 0;
    for (int w = 0; w < kWarps; ++w) {
      a += wgt[w];
      b += weq[w];
    }
    p.cnt[2 * cta] = a;
    p.cnt[2 * cta + 1] = b;
  }
  stamp(8);
  grid_barrier(&S->bar[3][0], (unsigned)G);
  stamp(9);
  // every CTA is past level 3: the histograms can be cleared for the next launch
  {
    uint32_t *hz = reinterpret_cast<uint32_t *>(S);  // hist1 | hist2 | hist3, contiguous
    for (int i = cta * kThreads + tid; i < 2 * kBins + kBins3; i += G * kThreads) hz[i] = 0u;
  }

  // selected / tie totals of the CTAs below this one (ties go to the lowest indices)
  if (warp == 0) {
    uint32_t eq_carry = 0, sel_carry = 0;
    for (int c0 = 0; c0 < cta; c0 += 32) {
      const int c = c0 + lane;
      const uint32_t gt = c < cta ? __ldcg(p.cnt + 2 * c) : 0u;
      const uint32_t eq = c < cta ? __ldcg(p.cnt + 2 * c + 1) : 0u;
      const uint32_t incl = warp_incl(eq);
      const uint32_t before = eq_carry + incl - eq;
      const uint32_t taken = before < ties ? min(eq, ties - before) : 0u;
      uint32_t sel = gt + taken;
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
  __syncthreads();
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
      const int i = c0 + lane;
      const int64_t q = q0 + i;
      float t[4] = {0.f, 0.f, 0.f, 0.f};
      int nv = 0;
      if (i < wq1) {
        quad_vals(t_quad(p, tS, i, q), t);
        nv = (int)min64(4, total - 4 * q);
      }
      uint32_t mgt = 0, meq = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t key = key_of(t[j]);
        mgt |= (uint32_t)((j < nv) & (key > T)) << j;
        meq |= (uint32_t)((j < nv) & (key == T)) << j;
      }
      const uint32_t ne = __popc(meq);
      const uint32_t ie = warp_incl(ne);
      uint32_t er = eq_run + ie - ne;  // tie rank of this lane's first tie
      uint32_t msel = mgt;
#pragma unroll
      for (int j = 0; j < 4; ++j)
        if ((meq >> j) & 1u) {
          if (er < ties) msel |= 1u << j;
          ++er;
        }
      const uint32_t ns = __popc(msel);
      const uint32_t is = warp_incl(ns);
      uint32_t pos = pos_run + is - ns;
      eq_run += __shfl_sync(0xffffffffu, ie, 31);
      pos_run += __shfl_sync(0xffffffffu, is, 31);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (!((msel >> j) & 1u)) continue;
        const int64_t e = 4 * q + j;
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
          p.base[e] = __fadd_rn(p.base[e], d);
          if constexpr (MODE == CC_WITH_FEEDBACK) p.aux[e] = __fsub_rn(tv, d);
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

static bool g_topk_resident = true;
static unsigned long long *g_topk_timer = nullptr;
void set_topk_timer(void *buf) { g_topk_timer = reinterpret_cast<unsigned long long *>(buf); }
void set_topk_resident_enabled(int on) { g_topk_resident = on != 0; }
std::atomic<int64_t> g_topk_resident_launches{0};
int64_t topk_resident_launches() { return g_topk_resident_launches.load(); }

// workspace of the resident path: per-CTA counts and record partials (+ the t
// scratch when the mode keeps t nowhere else and it does not fit on chip)
int64_t topk_resident_workspace_bytes(int64_t total) {
  return (int64_t)(align_up(8 * 1024, 256) + align_up(16 * 1024, 256) + align_up(4 * (size_t)total, 256));
}

int topk_resident_encode_step(int mode, int64_t n, int64_t C, int64_t k, const void *x, int x_dtype, float *base,
                              float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record,
                              cudaStream_t st) {
  using namespace k4r;
  if (!g_topk_resident) return CC_ERR_UNSUPPORTED;
  const int64_t total = n * C;
  if (total >= (int64_t)1 << 32 || k < 1) return CC_ERR_UNSUPPORTED;
  if (!aligned(x, x_dtype == CC_BF16 ? 8 : 16) || !aligned(base, 16) || (aux && !aligned(aux, 16)) ||
      !aligned(body, 4))
    return CC_ERR_UNSUPPORTED;
  Slab *slab = reinterpret_cast<Slab *>(stream_zero_slab(st, sizeof(Slab)));
  if (!slab) return CC_ERR_UNSUPPORTED;
  Params p{};
  p.x = x;
  p.base = base;
  p.aux = aux;
  p.total = total;
  p.k = k;
  p.nq = cdiv(total, 4);
  p.G = (int)std::max<int64_t>(1, std::min<int64_t>(sm_count(), cdiv(p.nq, 256)));
  if (p.G > 1024) return CC_ERR_UNSUPPORTED;
  const int64_t per = cdiv(p.nq, p.G);
  const size_t budget = kSmemMax - 4 * kBins - 2048;
  p.nsm = (int)std::min<int64_t>(per, (int64_t)(budget / 16));
  const bool fits = p.nsm >= per;
  // t outside shared memory: the feedback buffer (it becomes feedback' = t off the
  // selection anyway) or, in the other modes, workspace scratch
  uint8_t *w = reinterpret_cast<uint8_t *>(ws);
  size_t off = 0;
  auto take = [&](size_t b) {
    uint8_t *q = w + off;
    off = align_up(off + b, 256);
    return q;
  };
  p.cnt = reinterpret_cast<uint32_t *>(take(8 * (size_t)p.G));
  p.recpart = reinterpret_cast<double *>(take(16 * (size_t)p.G));
  if (mode == CC_WITH_FEEDBACK) {
    p.tout = aux;
    p.write_t = 1;
  } else {
    p.tout = fits ? nullptr : reinterpret_cast<float *>(take(4 * (size_t)total));
    p.write_t = fits ? 0 : 1;
  }
  if ((int64_t)off > ws_bytes) return CC_ERR_UNSUPPORTED;
  p.body = body;
  p.record = record;
  p.slab = slab;
  p.timer = g_topk_timer;
  const size_t smem = 4 * kBins + 16 * (size_t)p.nsm;
  void *args[] = {&p};
  auto go = [&](const void *kern) -> int {
    static int attr_set[16] = {0};
    (void)attr_set;
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
