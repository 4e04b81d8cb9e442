// K5: N:M block sparsifier (compressors.py:429-443 encode, :291-329 payload) on sm_100a.
//
// Reference semantics: columns are zero-padded to a multiple of m; every 1 x m
// block of the padded row-major matrix keeps the n entries of largest |v|, ties to
// the lowest index (stable argsort of -|v|); mask = m bits per block, little bit
// order, over the flat padded matrix (np.packbits(bitorder="little")); values = n
// f16 (RNE) per block in ascending index order, block-major.  Body = mask bytes
// (ceil(blocks*m/8)) immediately followed by the f16 values (cx:442-443, cx:596).
//
// The selection is local to a block, so encode_step is ONE pass over the shard:
// target t = f(x, base, aux) -> select -> emit mask/values -> state update ->
// record partials.  Ranking: rank_j = #{i < j : |t_i| >= |t_j|} + #{i > j : |t_i| >
// |t_j|} on the magnitude bits (key = bits & 0x7fffffff orders like |v| for finite
// values, +0 and -0 alike); entry j is kept iff rank_j < n, which is exactly the
// stable-argsort choice.
//
//   fast path  m in {2, 4, 8, 16, 32}: one thread per block, keys in registers;
//              the m-bit masks of 32/m consecutive lanes form one u32 word (warp
//              shuffle OR), written directly.
//   generic    any other m (<= 65535): one warp per block; t staged in a scratch
//              [n, C], mask bits atomically OR-ed into a zeroed scratch, then copied to the
//              body.
#include "cc_common.cuh"
#include "cc_internal.h"

#include <algorithm>

namespace cc {
namespace nm {

constexpr int kThreads = 256;

struct Geo {
  int64_t C;           // real columns
  int64_t bpr;         // blocks per row = ceil(C / m)
  int64_t nblocks;     // rows * bpr
  int64_t mask_bytes;  // ceil(nblocks * m / 8)
  int N, M;
};

__device__ __forceinline__ uint32_t key_of(float t) { return __float_as_uint(t) & 0x7fffffffu; }

// record partials: per-CTA (||d - t||^2, ||t||^2), last CTA reduces in fixed order
__device__ __forceinline__ void record_tail(double err, double tsq, double *part, unsigned *ticket, double *record) {
  __shared__ double se[kThreads / 32], st[kThreads / 32];
  __shared__ bool last;
  err = warp_sum(err);
  tsq = warp_sum(tsq);
  if ((threadIdx.x & 31) == 0) {
    se[threadIdx.x >> 5] = err;
    st[threadIdx.x >> 5] = tsq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < kThreads / 32; ++i) {
      a += se[i];
      b += st[i];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double a = 0.0, b = 0.0;
    for (unsigned i = 0; i < gridDim.x; ++i) {
      a += __ldcg(part + 2 * i);
      b += __ldcg(part + 2 * i + 1);
    }
    record[0] = a;
    record[1] = b;
    *ticket = 0u;
  }
}

template <int MODE, typename XT, bool STEP>
__device__ __forceinline__ float target1(const XT *x, const float *base, const float *aux, const float *tin, int64_t e) {
  if constexpr (!STEP) {
    return tin[e];
  } else {
    const float xx = Act<XT>::load1(x + e);
    float bb = 0.f, aa = 0.f;
    if constexpr (MODE == CC_WITH_FEEDBACK) bb = base[e];
    if constexpr (MODE != CC_NAIVE) aa = aux[e];
    return target_of<MODE>(xx, bb, aa);
  }
}

// state update of one real element (pipeline.py:105-112); d = 0 for dropped entries
template <int MODE, typename XT, bool STEP>
__device__ __forceinline__ void update1(const XT *x, float *base, float *aux, float *decoded, int64_t e, float t,
                                        float d) {
  if constexpr (STEP) {
    if constexpr (MODE == CC_NAIVE) {
      base[e] = d;
    } else {
      base[e] = __fadd_rn(base[e], d);  // -0.0 + 0.0 = +0.0, as the dense reference add
      if constexpr (MODE == CC_WITH_FEEDBACK) aux[e] = __fsub_rn(t, d);
      else aux[e] = Act<XT>::load1(x + e);  // ref' = a*
    }
  } else {
    if (decoded) decoded[e] = d;
  }
}

// write `nb` bytes of a little-endian word at body[byte0 ...], clipped to `limit`
__device__ __forceinline__ void put_word(uint8_t *body, int64_t byte0, uint32_t w, int64_t limit) {
  if (byte0 + 4 <= limit && (reinterpret_cast<uintptr_t>(body + byte0) & 3) == 0) {
    *reinterpret_cast<uint32_t *>(body + byte0) = w;
  } else {
    for (int b = 0; b < 4; ++b)
      if (byte0 + b < limit) body[byte0 + b] = (uint8_t)(w >> (8 * b));
  }
}

__device__ __forceinline__ void put_half(uint8_t *p, __half h) {
  const uint16_t u = __half_as_ushort(h);
  if ((reinterpret_cast<uintptr_t>(p) & 1) == 0) {
    *reinterpret_cast<uint16_t *>(p) = u;
  } else {
    p[0] = (uint8_t)(u & 0xff);
    p[1] = (uint8_t)(u >> 8);
  }
}

__device__ __forceinline__ float get_half(const uint8_t *p) {
  uint16_t u;
  if ((reinterpret_cast<uintptr_t>(p) & 1) == 0) u = *reinterpret_cast<const uint16_t *>(p);
  else u = (uint16_t)p[0] | (uint16_t)((uint16_t)p[1] << 8);
  return __half2float(__ushort_as_half(u));
}

// ---- fast encode: m in {2,4,8,16,32}, one thread per block ---------------------
template <int MODE, typename XT, bool STEP, int M>
__global__ void __launch_bounds__(kThreads) k_nm_fast(const XT *__restrict__ x, float *__restrict__ base,
                                                       float *__restrict__ aux, const float *__restrict__ tin,
                                                       float *__restrict__ decoded, Geo g, uint8_t *__restrict__ body,
                                                       int vec, double *__restrict__ part, unsigned *ticket,
                                                       double *__restrict__ record) {
  constexpr int L = 32 / M;  // lanes per mask word
  const int lane = threadIdx.x & 31;
  uint8_t *vals = body + g.mask_bytes;
  double err = 0.0, tsq = 0.0;
  for (int64_t gb0 = (int64_t)blockIdx.x * kThreads; gb0 < g.nblocks; gb0 += (int64_t)gridDim.x * kThreads) {
    const int64_t gb = gb0 + threadIdx.x;
    uint32_t mask = 0;
    if (gb < g.nblocks) {
      const int64_t row = gb / g.bpr;
      const int64_t c0 = (gb - row * g.bpr) * M;
      const int64_t e0 = row * g.C + c0;
      const int nreal = (int)min64(M, g.C - c0);
      float t[M];
      if constexpr (M >= 4) {
        if (vec) {  // C % 4 == 0 and 16-byte aligned rows: whole float4 groups are in or out
#pragma unroll
          for (int q = 0; q < M / 4; ++q) {
            if (4 * q < nreal) {
              float4 v;
              if constexpr (!STEP) {
                v = __ldcs(reinterpret_cast<const float4 *>(tin + e0 + 4 * q));
              } else {
                const float4 xx = Act<XT>::load4(x + e0 + 4 * q);
                float4 bb = make_float4(0.f, 0.f, 0.f, 0.f), aa = bb;
                if constexpr (MODE == CC_WITH_FEEDBACK) bb = *reinterpret_cast<const float4 *>(base + e0 + 4 * q);
                if constexpr (MODE != CC_NAIVE) aa = *reinterpret_cast<const float4 *>(aux + e0 + 4 * q);
                v = make_float4(target_of<MODE>(xx.x, bb.x, aa.x), target_of<MODE>(xx.y, bb.y, aa.y),
                                target_of<MODE>(xx.z, bb.z, aa.z), target_of<MODE>(xx.w, bb.w, aa.w));
              }
              t[4 * q] = v.x; t[4 * q + 1] = v.y; t[4 * q + 2] = v.z; t[4 * q + 3] = v.w;
            } else {
              t[4 * q] = t[4 * q + 1] = t[4 * q + 2] = t[4 * q + 3] = 0.0f;
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < M; ++j) t[j] = j < nreal ? target1<MODE, XT, STEP>(x, base, aux, tin, e0 + j) : 0.0f;
        }
      } else {
#pragma unroll
        for (int j = 0; j < M; ++j) t[j] = j < nreal ? target1<MODE, XT, STEP>(x, base, aux, tin, e0 + j) : 0.0f;
      }
      uint32_t k[M];
#pragma unroll
      for (int j = 0; j < M; ++j) k[j] = key_of(t[j]);
#pragma unroll
      for (int j = 0; j < M; ++j) {
        int rank = 0;
#pragma unroll
        for (int i = 0; i < M; ++i) {
          if (i < j) rank += k[i] >= k[j];
          else if (i > j) rank += k[i] > k[j];
        }
        if (rank < g.N) mask |= 1u << j;
      }
      // values + state update, ascending index order
      uint8_t *vp = vals + 2 * gb * g.N;
      int slot = 0;
      float d[M];
#pragma unroll
      for (int j = 0; j < M; ++j) {
        d[j] = 0.0f;
        if (mask & (1u << j)) {
          const __half h = __float2half_rn(t[j]);
          put_half(vp + 2 * slot, h);
          ++slot;
          d[j] = __half2float(h);
        }
      }
#pragma unroll
      for (int j = 0; j < M; ++j) {
        if (j < nreal) {
          const double df = (double)d[j] - (double)t[j];
          err += df * df;
          tsq += (double)t[j] * (double)t[j];
        }
      }
      bool done = false;
      if constexpr (M >= 4) {
        if (vec) {
#pragma unroll
          for (int q = 0; q < M / 4; ++q) {
            if (4 * q >= nreal) continue;
            const int64_t e = e0 + 4 * q;
            const float4 dv = make_float4(d[4 * q], d[4 * q + 1], d[4 * q + 2], d[4 * q + 3]);
            if constexpr (STEP) {
              if constexpr (MODE == CC_NAIVE) {
                *reinterpret_cast<float4 *>(base + e) = dv;
              } else {
                const float4 bb = *reinterpret_cast<const float4 *>(base + e);
                *reinterpret_cast<float4 *>(base + e) = make_float4(
                    __fadd_rn(bb.x, dv.x), __fadd_rn(bb.y, dv.y), __fadd_rn(bb.z, dv.z), __fadd_rn(bb.w, dv.w));
                if constexpr (MODE == CC_WITH_FEEDBACK) {
                  *reinterpret_cast<float4 *>(aux + e) =
                      make_float4(__fsub_rn(t[4 * q], dv.x), __fsub_rn(t[4 * q + 1], dv.y),
                                  __fsub_rn(t[4 * q + 2], dv.z), __fsub_rn(t[4 * q + 3], dv.w));
                } else {
                  *reinterpret_cast<float4 *>(aux + e) = Act<XT>::load4(x + e);
                }
              }
            } else if (decoded) {
              *reinterpret_cast<float4 *>(decoded + e) = dv;
            }
          }
          done = true;
        }
      }
      if (!done) {
#pragma unroll
        for (int j = 0; j < M; ++j)
          if (j < nreal) update1<MODE, XT, STEP>(x, base, aux, decoded, e0 + j, t[j], d[j]);
      }
    }
    // assemble the mask words of L consecutive lanes
    uint32_t w = mask << ((lane % L) * M);
#pragma unroll
    for (int o = 1; o < L; o <<= 1) w |= __shfl_xor_sync(0xffffffffu, w, o);
    if (lane % L == 0 && gb < g.nblocks) put_word(body, (gb / L) * 4, w, g.mask_bytes);
  }
  if (record) record_tail(err, tsq, part, ticket, record);
}

// ---- generic encode: any m, one warp per block -------------------------------
// pass 1 (STEP only): t -> tstage;
// NO_FEEDBACK: ref' = a* is written after t is formed.
template <int MODE, typename XT>
__global__ void __launch_bounds__(kThreads) k_nm_target(const XT *__restrict__ x, const float *__restrict__ base,
                                                         float *__restrict__ aux, float *__restrict__ tstage,
                                                         int64_t total) {
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t e = (int64_t)blockIdx.x * kThreads + threadIdx.x; e < total; e += stride) {
    const float xx = Act<XT>::load1(x + e);
    float bb = 0.f, aa = 0.f;
    if constexpr (MODE == CC_WITH_FEEDBACK) bb = base[e];
    if constexpr (MODE != CC_NAIVE) aa = aux[e];
    tstage[e] = target_of<MODE>(xx, bb, aa);
    if constexpr (MODE == CC_NO_FEEDBACK) aux[e] = xx;
  }
}

template <int MODE, bool STEP>
__global__ void __launch_bounds__(kThreads) k_nm_generic(const float *__restrict__ t, float *__restrict__ base,
                                                          float *__restrict__ aux, float *__restrict__ decoded, Geo g,
                                                          uint8_t *__restrict__ body, uint32_t *__restrict__ mwords,
                                                          double *__restrict__ part, unsigned *ticket,
                                                          double *__restrict__ record) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
  uint8_t *vals = body + g.mask_bytes;
  double err = 0.0, tsq = 0.0;
  for (int64_t gb = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); gb < g.nblocks; gb += warps) {
    const int64_t row = gb / g.bpr;
    const int64_t c0 = (gb - row * g.bpr) * g.M;
    const int64_t e0 = row * g.C + c0;
    const int nreal = (int)min64(g.M, g.C - c0);
    int taken = 0;
    for (int j0 = 0; j0 < g.M; j0 += 32) {
      const int j = j0 + lane;
      const bool inb = j < g.M;
      const float tj = (inb && j < nreal) ? t[e0 + j] : 0.0f;
      const uint32_t kj = key_of(tj);
      int rank = 0;
      if (inb) {
        for (int i = 0; i < nreal && rank < g.N; ++i) {
          const uint32_t ki = key_of(t[e0 + i]);
          rank += i < j ? (ki >= kj) : (i > j && ki > kj);
        }
        // padded entries (t = 0) beat j only if j's key is 0 and they come first
        if (rank < g.N && kj == 0u && j > nreal) rank += j - nreal;
      }
      const bool sel = inb && rank < g.N;
      const unsigned bal = __ballot_sync(0xffffffffu, sel);
      float d = 0.0f;
      if (sel) {
        const int slot = taken + __popc(bal & ((1u << lane) - 1u));
        const __half h = __float2half_rn(tj);
        put_half(vals + 2 * (gb * g.N + slot), h);
        d = __half2float(h);
        const int64_t bit = gb * g.M + j;
        atomicOr(&mwords[bit >> 5], 1u << (bit & 31));
      }
      taken += __popc(bal);
      if (inb && j < nreal) {
        const int64_t e = e0 + j;
        const double df = (double)d - (double)tj;
        err += df * df;
        tsq += (double)tj * (double)tj;
        if constexpr (STEP) {
          if constexpr (MODE == CC_NAIVE) {
            base[e] = d;
          } else {
            base[e] = __fadd_rn(base[e], d);
            if constexpr (MODE == CC_WITH_FEEDBACK) aux[e] = __fsub_rn(tj, d);
          }
        } else if (decoded) {
          decoded[e] = d;
        }
      }
    }
  }
  if (record) record_tail(err, tsq, part, ticket, record);
}

// ---- decode (+ accumulate into base), batched over peers -----------------------
constexpr int kMaxPeers = 16;
struct Peers {
  const uint8_t *body[kMaxPeers];
  float *base[kMaxPeers];
  int64_t nblocks[kMaxPeers];
};

__device__ __forceinline__ uint32_t get_bits(const uint8_t *mask, int64_t bit0, int nbits) {
  // nbits <= 32 bits starting at bit0 (little bit order)
  const int64_t byte0 = bit0 >> 3;
  const int sh = (int)(bit0 & 7);
  const int nbytes = (sh + nbits + 7) >> 3;
  uint64_t w = 0;
  for (int b = 0; b < nbytes; ++b) w |= (uint64_t)mask[byte0 + b] << (8 * b);
  w >>= sh;
  return nbits == 32 ? (uint32_t)w : (uint32_t)(w & ((1ull << nbits) - 1ull));
}

template <int M>
__global__ void __launch_bounds__(kThreads) k_nm_decode_fast(const __grid_constant__ Peers pp, int64_t C, int64_t bpr,
                                                              int N, int accumulate) {
  const int peer = blockIdx.y;
  const int64_t nb = pp.nblocks[peer];
  const uint8_t *body = pp.body[peer];
  float *base = pp.base[peer];
  const int64_t mask_bytes = (nb * M + 7) / 8;
  const uint8_t *vals = body + mask_bytes;
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  for (int64_t gb = (int64_t)blockIdx.x * kThreads + threadIdx.x; gb < nb; gb += stride) {
    const uint32_t mask = get_bits(body, gb * M, M);
    const int64_t row = gb / bpr;
    const int64_t c0 = (gb - row * bpr) * M;
    const int64_t e0 = row * C + c0;
    const int nreal = (int)min64(M, C - c0);
    const uint8_t *vp = vals + 2 * gb * N;
    int slot = 0;
#pragma unroll
    for (int j = 0; j < M; ++j) {
      float d = 0.0f;
      if (mask & (1u << j)) d = get_half(vp + 2 * slot++);
      if (j < nreal) base[e0 + j] = accumulate ? __fadd_rn(base[e0 + j], d) : d;
    }
  }
}

__global__ void __launch_bounds__(kThreads) k_nm_decode_generic(const __grid_constant__ Peers pp, int64_t C,
                                                                 int64_t bpr, int N, int M, int accumulate) {
  const int peer = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int64_t nb = pp.nblocks[peer];
  const uint8_t *body = pp.body[peer];
  float *base = pp.base[peer];
  const int64_t mask_bytes = (nb * M + 7) / 8;
  const uint8_t *vals = body + mask_bytes;
  const int64_t warps = (int64_t)gridDim.x * (kThreads / 32);
  for (int64_t gb = (int64_t)blockIdx.x * (kThreads / 32) + (threadIdx.x >> 5); gb < nb; gb += warps) {
    const int64_t row = gb / bpr;
    const int64_t c0 = (gb - row * bpr) * M;
    const int64_t e0 = row * C + c0;
    const int nreal = (int)min64(M, C - c0);
    int taken = 0;
    for (int j0 = 0; j0 < M; j0 += 32) {
      const int j = j0 + lane;
      const bool bit = j < M && get_bits(body, gb * M + j, 1);
      const unsigned bal = __ballot_sync(0xffffffffu, bit);
      float d = 0.0f;
      if (bit) d = get_half(vals + 2 * (gb * N + taken + __popc(bal & ((1u << lane) - 1u))));
      taken += __popc(bal);
      if (j < nreal) base[e0 + j] = accumulate ? __fadd_rn(base[e0 + j], d) : d;
    }
  }
}

}  // namespace nm

// ---------------------------------------------------------------------------
// host
// ---------------------------------------------------------------------------
static bool nm_fast(int m) { return m == 2 || m == 4 || m == 8 || m == 16 || m == 32; }

static nm::Geo nm_geo(int64_t rows, int64_t C, int n, int m) {
  nm::Geo g;
  g.C = C;
  g.bpr = cdiv(C, m);
  g.nblocks = rows * g.bpr;
  g.mask_bytes = cdiv(g.nblocks * m, 8);
  g.N = n;
  g.M = m;
  return g;
}

int64_t nm_body_bytes(int64_t rows, int64_t C, int n, int m) {
  const nm::Geo g = nm_geo(rows, C, n, m);
  return g.mask_bytes + 2 * g.nblocks * n;
}

static unsigned nm_grid(int64_t work_items) {
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(work_items, nm::kThreads), sm_count() * 8));
}

struct NmWork {
  double *part;
  unsigned *ticket;
  double *rec;       // record scratch for the stateless encode
  uint32_t *mwords;  // generic path: mask scratch
  float *tstage;     // generic path: staged target
  size_t bytes;
};

static NmWork nm_carve(void *ws, int64_t rows, int64_t C, int n, int m, bool need_t) {
  NmWork w{};
  uint8_t *b = reinterpret_cast<uint8_t *>(ws);
  size_t off = 0;
  auto take = [&](size_t sz) {
    uint8_t *q = b ? b + off : nullptr;
    off = align_up(off + sz, 256);
    return q;
  };
  const nm::Geo g = nm_geo(rows, C, n, m);
  w.ticket = reinterpret_cast<unsigned *>(take(16));
  w.rec = reinterpret_cast<double *>(take(16));
  w.part = reinterpret_cast<double *>(take(16 * (size_t)sm_count() * 8 + 16));
  if (!nm_fast(m)) {
    w.mwords = reinterpret_cast<uint32_t *>(take(4 * (size_t)cdiv(g.nblocks * m, 32)));
    if (need_t) w.tstage = reinterpret_cast<float *>(take(4 * (size_t)(rows * C)));
  }
  w.bytes = off;
  return w;
}

int64_t nm_workspace_bytes(int64_t rows, int64_t C, int n, int m) {
  return (int64_t)nm_carve(nullptr, rows, C, n, m, true).bytes;
}

template <int MODE, typename XT, bool STEP>
static int nm_run(const nm::Geo &g, int64_t rows, const XT *x, float *base, float *aux, const float *tin,
                  float *decoded, uint8_t *body, const NmWork &w, double *record, cudaStream_t st) {
  using namespace nm;
  const int64_t total = rows * g.C;
  if (nm_fast(g.M)) {
    const unsigned grid = nm_grid(g.nblocks);
    auto al = [](const void *p) { return p == nullptr || (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    const int vec = g.C % 4 == 0 && al(base) && al(aux) && al(tin) && al(decoded) &&
                    (x == nullptr || (reinterpret_cast<uintptr_t>(x) & (sizeof(XT) == 2 ? 7 : 15)) == 0);
#define NM_L(MM) k_nm_fast<MODE, XT, STEP, MM><<<grid, kThreads, 0, st>>>(x, base, aux, tin, decoded, g, body, vec, \
                                                                          w.part, w.ticket, record)
    switch (g.M) {
      case 2: NM_L(2); break;
      case 4: NM_L(4); break;
      case 8: NM_L(8); break;
      case 16: NM_L(16); break;
      default: NM_L(32); break;
    }
#undef NM_L
    count_launch();
    return CC_OK;
  }
  // generic path
  const float *t = tin;
  if constexpr (STEP) {
    // staged separately from the feedback buffer: a warp ranks a whole block before
    // its later 32-wide chunks are updated, so t must not be overwritten in place
    float *ts = w.tstage;
    k_nm_target<MODE, XT><<<nm_grid(total), kThreads, 0, st>>>(x, base, aux, ts, total);
    count_launch();
    t = ts;
  }
  cudaMemsetAsync(w.mwords, 0, 4 * (size_t)cdiv(g.nblocks * g.M, 32), st);
  const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(g.nblocks, kThreads / 32), sm_count() * 8));
  k_nm_generic<MODE, STEP><<<grid, kThreads, 0, st>>>(t, base, aux, decoded, g, body, w.mwords, w.part, w.ticket,
                                                      record);
  count_launch();
  cudaMemcpyAsync(body, w.mwords, (size_t)g.mask_bytes, cudaMemcpyDeviceToDevice, st);
  return CC_OK;
}

int nm_encode(int64_t rows, int64_t C, int n, int m, const float *t, uint8_t *body, float *decoded, void *ws,
              int64_t ws_bytes, cudaStream_t st) {
  const NmWork need = nm_carve(nullptr, rows, C, n, m, false);
  if ((int64_t)need.bytes > ws_bytes) {
    set_error("N:M workspace too small");
    return CC_ERR_ARG;
  }
  const NmWork w = nm_carve(ws, rows, C, n, m, false);
  const nm::Geo g = nm_geo(rows, C, n, m);
  cudaMemsetAsync(w.ticket, 0, 16, st);
  nm_run<CC_NAIVE, float, false>(g, rows, nullptr, nullptr, nullptr, t, decoded, body, w, nullptr, st);
  return cuda_status("nm_encode");
}

int nm_encode_step(int mode, int64_t rows, int64_t C, int n, int m, const void *x, int x_dtype, float *base,
                   float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st) {
  const NmWork need = nm_carve(nullptr, rows, C, n, m, true);
  if ((int64_t)need.bytes > ws_bytes) {
    set_error("N:M workspace too small");
    return CC_ERR_ARG;
  }
  const NmWork w = nm_carve(ws, rows, C, n, m, true);
  const nm::Geo g = nm_geo(rows, C, n, m);
  cudaMemsetAsync(w.ticket, 0, 16, st);
#define NM_S(MODE, XT) nm_run<MODE, XT, true>(g, rows, (const XT *)x, base, aux, nullptr, nullptr, body, w, record, st)
  if (x_dtype == CC_BF16) {
    if (mode == CC_WITH_FEEDBACK) NM_S(CC_WITH_FEEDBACK, __nv_bfloat16);
    else if (mode == CC_NO_FEEDBACK) NM_S(CC_NO_FEEDBACK, __nv_bfloat16);
    else NM_S(CC_NAIVE, __nv_bfloat16);
  } else {
    if (mode == CC_WITH_FEEDBACK) NM_S(CC_WITH_FEEDBACK, float);
    else if (mode == CC_NO_FEEDBACK) NM_S(CC_NO_FEEDBACK, float);
    else NM_S(CC_NAIVE, float);
  }
#undef NM_S
  return cuda_status("nm_encode_step");
}

// accumulate: 0 replace (base = decode), else base = base + decode (dense add)
int nm_decode(int count, const int64_t *rows, int64_t C, int n, int m, const uint8_t *const *bodies, int accumulate,
              float *const *bases, cudaStream_t st) {
  const int64_t bpr = cdiv(C, m);
  for (int c0 = 0; c0 < count; c0 += nm::kMaxPeers) {
    const int cnt = std::min(nm::kMaxPeers, count - c0);
    nm::Peers pp{};
    int64_t maxb = 0;
    for (int i = 0; i < cnt; ++i) {
      pp.body[i] = bodies[c0 + i];
      pp.base[i] = bases[c0 + i];
      pp.nblocks[i] = rows[c0 + i] * bpr;
      maxb = std::max(maxb, pp.nblocks[i]);
    }
    const int acc = accumulate != 0;
    if (nm_fast(m)) {
      dim3 grid(nm_grid(maxb), cnt);
      switch (m) {
        case 2: nm::k_nm_decode_fast<2><<<grid, nm::kThreads, 0, st>>>(pp, C, bpr, n, acc); break;
        case 4: nm::k_nm_decode_fast<4><<<grid, nm::kThreads, 0, st>>>(pp, C, bpr, n, acc); break;
        case 8: nm::k_nm_decode_fast<8><<<grid, nm::kThreads, 0, st>>>(pp, C, bpr, n, acc); break;
        case 16: nm::k_nm_decode_fast<16><<<grid, nm::kThreads, 0, st>>>(pp, C, bpr, n, acc); break;
        default: nm::k_nm_decode_fast<32><<<grid, nm::kThreads, 0, st>>>(pp, C, bpr, n, acc); break;
      }
    } else {
      dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(maxb, nm::kThreads / 32), sm_count() * 8)), cnt);
      nm::k_nm_decode_generic<<<grid, nm::kThreads, 0, st>>>(pp, C, bpr, n, m, acc);
    }
    count_launch();
  }
  return cuda_status("nm_decode");
}

}  // namespace cc
