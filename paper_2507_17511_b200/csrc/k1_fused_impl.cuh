// K1 persistent kernel + its launch template, shared by the two translation
// units that instantiate it (k1_fused.cu: plain steps, k1_fused_seg.cu: column
// segments) so they compile in parallel.
#pragma once
// K1, persistent form: ONE cooperative kernel per encode_step for the 1/2/4-bit
// codecs (C % 128 == 0 and C <= 3072, e.g. FLUX's 3072 or a Ulysses chunk of 384),
// 148 CTAs x (12 consumer warps + TMA load warp + TMA store warp).
//
// Tiles are R FULL rows, so every array of a tile is one contiguous range and
// moves with a single cp.async.bulk (1-D TMA) per array:
//   phase A  the load warp streams (x, base, aux) tiles into an mbarrier ring
//            (dynamic tile claims, one ahead); the consumers form
//            t = target(x, base, aux) (pipeline.py:99-104) and accumulate |t| in
//            f64: column partials in registers, row partials per 128-column block
//            through shared memory (summed per segment by the load-warp lanes).
//   hand-off 1  flag barrier (release arrivals, one acquire poller per CTA)
//   phase F  consumers: v_j = colmean (32-column groups per CTA, 148 partials in
//            one L2 round trip); store warp: g = mean|t|, u_i = max(rowmean_i / g,
//            1e-30) (compressors.py:135-149); u, v straight into the body.  The load
//            warp is already streaming phase B's first tiles.
//   hand-off 2  flag barrier
//   phase B  the SAME rows in reverse order (the last ~40 MB of phase A is still
//            L2-resident): consumers quantize (compressors.py:373-391) into an
//            output ring: base' / feedback' / ref' (pipeline.py:107-113) and the
//            packed codes, drained to HBM by the store warp with TMA bulk stores.
//            StepRecord partials -> last-CTA ticket reduction (pipeline.py:115-120).
//
// Column segments (SEG): the same pass over full-width rows serves P independent
// column-slice channels (Ulysses (src, dst) chunks): per-segment row
// sums, g, u, bodies and records; v is per column anyway.
//
// Results are bit-identical to the multi-kernel path in quant.cu (same f64 element
// arithmetic; f64 reductions), pinned by the parity tests that run both paths
// against the oracle.

#include "cc_async.cuh"
#include "cc_common.cuh"
#include "cc_internal.h"

#include <algorithm>
#include <string>


namespace cc {
namespace fused {

constexpr int kCons = 384;             // consumer threads (12 warps)
constexpr int kCW = kCons / 32;
constexpr int kThreads = kCons + 64;   // + TMA load warp + TMA store warp
constexpr int kMaxC = 2 * 4 * kCons;   // 3072 columns: two column quads per consumer thread
constexpr int kNB = kMaxC / 128;       // 128-column blocks per row (one warp-quad span each)
constexpr int kMaxSeg = 16;            // column segments with independent scales (Ulysses chunks)
constexpr size_t kSmemBudget = 224 * 1024;

struct Params {
  const void *x;
  float *base, *aux;
  int64_t n, C;
  int G4, groups, wpg;  // column quads, row groups, warps per group
  int R, S, G;          // phase A: rows per tile, stages; grid size
  int S_in, S_out;      // phase B ring depths
  uint32_t ring_bytes;  // shared bytes of the tile rings
  int cb_row;           // code bytes per row
  int64_t nTiles;
  double *colpart, *rowpart, *blkpart, *recpart, *record;  // rowpart [nseg][n], blkpart [G][nseg],
                                                           // recpart [G][nseg][2], record [nseg][2]
  float *u, *v;                                            // u [nseg][un], v [C]
  // Column segments: nseg column slices of width cw (multiple of 128), each an
  // independent channel with its own scales and body (segment d = columns
  // [d cw, (d+1) cw), body at body + d * body_stride: codes [n][cbs] | u[n] | v[cw]).
  // nseg = 1 is the plain encode_step.
  uint8_t *body;
  int64_t body_stride, cbytes_seg, un;
  int nseg, cw, cbs, bps;  // segments, width, code bytes per segment row, 128-col blocks per segment
  unsigned int *ticket;     // control words: zero on entry, left zero on exit
  unsigned int *bar;        // grid hand-off counters bar1 = bar[0], bar2 = bar[32] (control words)
  unsigned long long *ctr;  // dynamic tile counters [phase A, phase B], zeroed before launch
  int scale_mode;
  int stop_after;             // profiling: 1 = phase A only, 2 = A + scales, 3 = A w/o sync, 0 = full
  int ctl_in_ws;              // control words live in the workspace (memset before launch)
  long long early_tiles;      // phase-A tiles loaded L2::evict_first (the rest evict_last)
  int tail_mult, tail_keep;   // phase-B end-game: < tail_mult * G tiles left -> <= tail_keep tiles ahead
  int static_sched;           // 0: static rounds then dynamic tail, 1: all static, 2: static prologue only
  unsigned long long *timer;  // profiling: [G][16] globaltimer stamps, or null
  int policy;  // experiment bits: 1 = phase-B stores without L2 hint, 2 = phase-B loads evict_first,
               // 4 = phase-A loads evict_normal, 8 = phase-A consumers skip the math (timing only),
               // 16 = skip phase-A row finishing (timing only), 32 = control words in the workspace,
               // 64 = phase-B consumers skip loads/math/results (timing only), 128 = phase-B results
               // stored directly from registers (no output ring / TMA stores)
};

// Params::policy experiment bits (L2 hints, skipped math / stores for movement-only
// timings) are compiled in only with -DCC_K1_EXPERIMENTS=1: in production builds every
// K1_XP(p) test is a compile-time 0 and the branches vanish from the kernels.
#ifndef CC_K1_EXPERIMENTS
#define CC_K1_EXPERIMENTS 0
#endif
#define K1_XP(p) (CC_K1_EXPERIMENTS ? (p).policy : 0)

__device__ __forceinline__ uint64_t l2_policy_normal() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
  return p;
}

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
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
  bool ok;  // all 4 columns have |v| in [2^-50, 2^50]
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
      const uint32_t code = (big ? 3u : 2u) - (neg ? (big ? 3u : 1u) : 0u);
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

// deterministic sums of two values over the kCons consumer threads (named
// barrier 1): fixed butterfly per warp, then warps in order; all consumers get them
__device__ __forceinline__ void cons_sum2(double a, double b, double *red, double &sa, double &sb) {
  a = warp_sum(a);
  b = warp_sum(b);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    red[2 * w] = a;
    red[2 * w + 1] = b;
  }
  named_sync(1, kCons);
  sa = 0.0;
  sb = 0.0;
  for (int i = 0; i < kCW; ++i) {
    sa += red[2 * i];
    sb += red[2 * i + 1];
  }
  named_sync(1, kCons);
}

__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned *p) {
  unsigned old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

// grid hand-off wait: spin until *p >= target (acquire)
__device__ __forceinline__ void spin_until(const unsigned *p, unsigned target) {
  for (;;) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    if (v >= target) break;
  }
}

// grid hand-off arrival: release-ordered add (cumulative over the CTA's writes
// ordered before it by a barrier)
__device__ __forceinline__ void arrive_release(unsigned *p) {
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(p) : "memory");
}

__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int MODE>
constexpr bool has_aux() {
  return MODE != CC_NAIVE;
}

// byte offsets of the arrays of one ring stage holding R rows
struct InStage {
  uint32_t x, base, aux, bytes;
};
struct OutStage {
  uint32_t base, aux, codes, bytes;
};
__host__ __device__ inline uint32_t al128(uint64_t v) { return (uint32_t)((v + 127u) & ~127ull); }

template <int MODE, typename XT>
__host__ __device__ inline InStage in_stage(int R, int64_t C, bool with_base) {
  InStage L;
  L.x = 0;
  L.base = al128((uint64_t)R * C * sizeof(XT));
  L.aux = with_base ? al128(L.base + (uint64_t)R * C * 4) : L.base;
  L.bytes = has_aux<MODE>() ? al128(L.aux + (uint64_t)R * C * 4) : L.aux;
  return L;
}
template <int MODE>
__host__ __device__ inline OutStage out_stage(int R, int64_t C, int cb_row) {
  OutStage L;
  L.base = 0;
  L.aux = al128((uint64_t)R * C * 4);
  L.codes = has_aux<MODE>() ? al128(L.aux + (uint64_t)R * C * 4) : L.aux;
  L.bytes = al128(L.codes + (uint64_t)R * cb_row);
  return L;
}

__device__ __forceinline__ void unpack_x(const __nv_bfloat16 *p, float (&xx)[4]) {
  const uint2 raw = *reinterpret_cast<const uint2 *>(p);
  xx[0] = __uint_as_float(raw.x << 16);
  xx[1] = __uint_as_float(raw.x & 0xffff0000u);
  xx[2] = __uint_as_float(raw.y << 16);
  xx[3] = __uint_as_float(raw.y & 0xffff0000u);
}
__device__ __forceinline__ void unpack_x(const float *p, float (&xx)[4]) {
  const float4 v = lds4(p);
  xx[0] = v.x; xx[1] = v.y; xx[2] = v.z; xx[3] = v.w;
}
__device__ __forceinline__ void unpack_f(const float *p, float (&v)[4]) {
  const float4 w = lds4(p);
  v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
}

// Q = column quads per consumer thread (1: C <= 1536 with row groups; 2: C <= 3072);
// SEG = column segments (cc_encode_step_segmented); false compiles the plain step
template <int MODE, int CODEC, typename XT, int Q, bool SEG>
__global__ void __launch_bounds__(kThreads, 1) k1_fused(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int RA = p.R, SA = p.S, G = p.G;
  const int RB = p.groups, SI = p.S_in, SO = p.S_out;
  const int64_t n = p.n, C = p.C;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x;
  const bool loader = warp == kCW, storer = warp == kCW + 1, consumer = warp < kCW;
  int grp = 0, quad0 = tid, wig = warp;
  if constexpr (Q == 1) {
    grp = tid / p.G4;
    quad0 = tid % p.G4;
    wig = quad0 >> 5;
  }
  const bool in_group = consumer && grp < p.groups;
  bool qact[Q];
  int qcol[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    const int qd = quad0 + j * kCons;
    qact[j] = in_group && qd < p.G4;
    qcol[j] = 4 * qd;
  }

  // ---- shared memory: [ring area][rp][red][ucache][barriers] ----
  uint8_t *ring = smem;
  double *rp = reinterpret_cast<double *>(smem + p.ring_bytes);  // [2 use parities][SA][RA][kNB blocks]
  double *red = rp + (size_t)2 * SA * RA * kNB;                  // [512]: reductions scratch
  uint64_t *fullA = reinterpret_cast<uint64_t *>(red + 512);
  uint64_t *emptyA = fullA + SA;
  uint64_t *fullB = emptyA + SA;
  uint64_t *emptyB = fullB + SI;
  uint64_t *outFull = emptyB + SI;
  uint64_t *outFree = outFull + SO;
  uint64_t *handA = outFree + SO;  // CTA-local relays of the grid hand-offs (bar1, bar2)
  volatile long long *tileA = reinterpret_cast<volatile long long *>(handA + 2);  // [SA]
  volatile long long *tileB = tileA + SA;                                           // [SI]
  volatile long long *tileO = tileB + SI;                                           // [SO]
  float *ustage = reinterpret_cast<float *>(
      (reinterpret_cast<uintptr_t>(const_cast<long long *>(tileO + SO)) + 15) & ~uintptr_t(15));  // [SI][nseg][16]
  const int nseg = SEG ? p.nseg : 1, bps = p.bps;
  // the 128-column block (and so the segment) each of this thread's column quads lies in
  // (nseg == 1: one combined partial per warp, "block" = the warp's index in its row)
  int qblk[Q], qseg[Q];
#pragma unroll
  for (int j = 0; j < Q; ++j) {
    qblk[j] = Q == 2 ? j * kCW + warp : wig;
    qseg[j] = nseg == 1 ? 0 : min(qblk[j] / bps, nseg - 1);
  }

  auto stamp = [&](int i) {
    if (p.timer && tid == 0) p.timer[(size_t)cta * 16 + i] = gtimer();
  };
  stamp(0);
  if (tid == 0) {
    for (int s = 0; s < SA; ++s) {
      mbar_init(&fullA[s], 1);
      mbar_init(&emptyA[s], kCW);
    }
    for (int s = 0; s < SI; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], kCW);
    }
    for (int s = 0; s < SO; ++s) {
      mbar_init(&outFull[s], kCW);
      mbar_init(&outFree[s], 1);
    }
    mbar_init(&handA[0], 1);
    mbar_init(&handA[1], 1);
    mbar_fence_init();
  }
  __syncthreads();
  pdl_wait();  // PDL launches only: our inputs may come from the previous kernel
  const XT *X = reinterpret_cast<const XT *>(p.x);

  // ================= phase A: |t| partial sums over tiles of RA rows =================
  const InStage LA = in_stage<MODE, XT>(RA, C, MODE == CC_WITH_FEEDBACK);
  double cta_total = 0.0;
  // producer lanes: row sums of a finished tile (stage s, use parity par)
  // lane = d * RA + r owns (row r of the tile, segment d): RA * nseg <= 32 (launcher)
  auto finish_rows = [&](int s, long long tile, uint32_t par) {
    const int64_t r0 = (int64_t)tile * RA;
    const int r = lane % RA, d = lane / RA;
    if (d < nseg && r0 + r < n) {
      double acc = 0.0;
      const double *q = rp + (((size_t)par * SA + s) * RA + r) * kNB + d * bps;
      for (int b = 0; b < bps; ++b) acc += q[b];
      p.rowpart[(int64_t)d * n + r0 + r] = acc;
      cta_total += acc;
    }
  };
  // ---- phase-B ring geometry (shared by every role) ----
  // Phase-B tiles are RB (= row groups) rows, visited in REVERSE order (phase A's
  // tail is L2-resident); a load ring (S_in) and a separate output ring (S_out)
  // drained by the store warp with TMA bulk stores, so loads never wait for stores.
  const InStage LI = in_stage<MODE, XT>(RB, C, has_aux<MODE>());
  const OutStage LO = out_stage<MODE>(RB, C, p.cb_row);
  uint8_t *in_ring = ring;
  uint8_t *out_ring = ring + (size_t)SI * LI.bytes;
  const int64_t nTB = (n + RB - 1) / RB;
  unsigned int *bar1 = p.bar, *bar2 = p.bar + 32;  // separate 128-byte lines
  double err[Q], tsq[Q];  // StepRecord partials per column quad (its block's segment)
#pragma unroll
  for (int j = 0; j < Q; ++j) err[j] = tsq[j] = 0.0;

  // Grid-wide hand-offs are flag barriers (arrive = fence + atomicAdd, wait = one
  // thread spinning on ld.acquire, then a CTA-local named barrier) instead of
  // grid.sync, so the loader never stalls with the rest of the grid:
  //   bar1 (2 arrivals per CTA: loader rows + consumer columns) = phase A done;
  //   bar2 (2 arrivals per CTA: consumers v, store warp u) = scales published.
  // While the consumers run the scale pass, the loader already streams phase B's
  // first S_in tiles (only their u windows wait for bar2).
  //
  // Phase A uses a dynamic tile scheduler: the loader claims tiles with an atomic
  // counter one tile AHEAD (the claim's L2 round trip hides behind the ring wait)
  // and publishes the tile id with the stage (-1 = no more work).  Row sums of the
  // tile a stage held are finished after its refill is issued (rp is
  // double-buffered by use parity, so the new tile's partials cannot collide).
  if (loader) {
   {  // phase A
    const uint64_t pol_late = (K1_XP(p) & 4) ? l2_policy_normal() : l2_policy_evict_last();
    const uint64_t pol_early = l2_policy_evict_first();
    // Only the last ~kL2KeepBytes of phase A stay L2-resident (evict_last) for the
    // reverse-order phase B; earlier tiles are loaded evict_first so they do not
    // compete (measured at [4096, 3072]: 70 % evict_first is ~2 us faster than 0 %).
    const long long early = p.early_tiles;
    int k = 0, s = 0;
    uint32_t ph = 0;  // phase parity of stage s's current use
    // The first proA claims of every CTA are static (cta + k G): the ring fills
    // without a chain of atomic round trips (what bounds small shards); the rest
    // come from the counter, offset past the static ones.
    // (all but the last ~2 rounds static; the tail is claimed dynamically, which keeps
    // CTAs that share their SM with other kernels from holding up the grid)
    const int proA = p.static_sched == 1   ? 0x7fffffff
                     : p.static_sched == 2 ? (int)min64(SA, p.nTiles / G)
                                           : (int)max64(min64(SA, p.nTiles / G), p.nTiles / G - 2);
    int kcA = 0;
    auto claimA = [&]() -> unsigned long long {  // lane 0
      const unsigned long long v = kcA < proA ? (unsigned long long)(cta + (long long)kcA * G)
                                              : (unsigned long long)proA * G + atomicAdd(p.ctr, 1ull);
      ++kcA;
      return v;
    };
    unsigned long long nxt = 0;
    if (lane == 0) nxt = claimA();
    for (;;) {
      long long old = -1;
      if (k >= SA) {
        mbar_wait(&emptyA[s], ph ^ 1u);
        old = tileA[s];
      }
      long long tile = (long long)__shfl_sync(0xffffffffu, nxt, 0);
      if (tile >= p.nTiles) tile = -1;
      if (lane == 0) {
        if (tile >= 0) nxt = claimA();
        tileA[s] = tile;
        if (tile < 0) {
          mbar_arrive(&fullA[s]);
        } else {
          uint8_t *st = ring + (size_t)s * LA.bytes;
          const int64_t r0 = (int64_t)tile * RA;
          const uint64_t pol = tile < early ? pol_early : pol_late;
          const int nrows = (int)min64(RA, n - r0);
          const uint32_t xb = (uint32_t)(nrows * C * sizeof(XT)), fb = (uint32_t)(nrows * C * 4);
          const bool wb = MODE == CC_WITH_FEEDBACK;
          mbar_expect_tx(&fullA[s], xb + (wb ? fb : 0u) + (has_aux<MODE>() ? fb : 0u));
          bulk_g2s(st + LA.x, X + r0 * C, xb, &fullA[s], pol);
          if (wb) bulk_g2s(st + LA.base, p.base + r0 * C, fb, &fullA[s], pol);
          if (has_aux<MODE>()) bulk_g2s(st + LA.aux, p.aux + r0 * C, fb, &fullA[s], pol);
        }
      }
      __syncwarp();
      if (old >= 0 && !(K1_XP(p) & 16)) finish_rows(s, old, ph ^ 1u);
      if (tile < 0) break;
      ++k;
      if (++s == SA) {
        s = 0;
        ph ^= 1u;
      }
    }
    // drain: the stages still in use are the last min(SA, k+1) (sentinel included)
    const int used = min(SA, k + 1);
    for (int q = 0; q < used; ++q) {  // walk backwards from the sentinel stage
      const int sq = (s - q + SA) % SA;
      const uint32_t pq = (q <= s) ? ph : (ph ^ 1u);
      mbar_wait(&emptyA[sq], pq);
      if (q > 0 && tileA[sq] >= 0) finish_rows(sq, tileA[sq], pq);
    }
    if (p.timer && lane == 0) p.timer[(size_t)cta * 16 + 10] = gtimer();
   }
    // CTA |t| total per segment: lanes d*RA .. d*RA+RA-1 hold segment d's row sums
    {
      double tot = cta_total;
      for (int o = 1; o < RA; ++o) {
        const double v = __shfl_down_sync(0xffffffffu, cta_total, o);
        if (lane % RA == 0) tot += v;
      }
      if (lane % RA == 0 && lane / RA < nseg) p.blkpart[(size_t)cta * nseg + lane / RA] = tot;
      __syncwarp();
      if (lane == 0) arrive_release(bar1);
    }
    if (p.stop_after) return;
    // Phase B.  The first S_in tiles are loaded while the consumers still run
    // the scale pass; their u windows follow once bar2 publishes u.
    // phase-B loads: evict_normal (measured ~1 us better than evict_first at [4096, 3072])
    const uint64_t pol = (K1_XP(p) & 2) ? l2_policy_evict_first() : l2_policy_normal();
    // k = stage uses issued (stage k % SI), w = uses whose release has been awaited.
    // Claims run one tile ahead while plenty of work is left; in the end-game
    // (fewer than tail_mult x G tiles unclaimed) a CTA claims only when at most
    // tail_keep of its tiles are still unconsumed, so the last tiles spread over
    // the grid instead of queueing behind a few full rings.
    int k = 0, w = 0;
    bool u_ready = false, have_nxt = true, near_end = false;
    const long long tail = (long long)p.tail_mult * G;
    const int proB = p.static_sched == 1   ? 0x7fffffff  // static first claims, as in phase A
                     : p.static_sched == 2 ? (int)min64(SI, nTB / G)
                                           : (int)max64(min64(SI, nTB / G), nTB / G - 2);
    int kcB = 0;
    auto claimB = [&]() -> unsigned long long {  // lane 0
      const unsigned long long v = kcB < proB ? (unsigned long long)(cta + (long long)kcB * G)
                                              : (unsigned long long)proB * G + atomicAdd(p.ctr + 16, 1ull);
      ++kcB;
      return v;
    };
    unsigned long long nxt = 0;
    if (lane == 0) nxt = claimB();
    auto load_u = [&](int st_, long long tile) {  // lane 0: 16B-aligned windows of u_d for the tile's rows
      const int64_t r0 = (int64_t)tile * RB;
      const int nrows = (int)min64(RB, n - r0);
      const uint32_t ub = (uint32_t)(((r0 & 3) + nrows + 3) / 4 * 16);
      for (int d = 0; d < nseg; ++d)
        bulk_g2s(ustage + ((size_t)st_ * nseg + d) * 16, p.u + d * p.un + (r0 & ~3LL), ub, &fullB[st_], pol);
    };
    auto publish_u = [&](int nst) {
      if (lane == 0) {
        mbar_wait(&handA[1], 0);  // relayed by consumer thread 0, the CTA's only poller
        fence_proxy_async_global();  // u was written through the generic proxy; TMA reads it
        for (int q = 0; q < nst; ++q)
          if (tileB[q] >= 0) load_u(q, tileB[q]);
      }
      __syncwarp();
      u_ready = true;
    };
    for (;;) {
      int req = k - SI + 1;  // stage k % SI must be free
      if (near_end) req = max(req, k - p.tail_keep);
      if (w < req && !u_ready) publish_u(min(k, SI));  // consumers need u before any release
      for (; w < req; ++w) mbar_wait(&emptyB[w % SI], (uint32_t)(w / SI) & 1u);
      if (!have_nxt && lane == 0) nxt = claimB();
      const long long t = (long long)__shfl_sync(0xffffffffu, nxt, 0);
      const long long tile = t < nTB ? nTB - 1 - t : -1;
      near_end = tail > 0 && t + tail >= nTB;
      have_nxt = tile >= 0 && !near_end;
      const int s = k % SI;
      if (lane == 0) {
        if (have_nxt) nxt = claimB();
        tileB[s] = tile;
        if (tile < 0) {
          mbar_arrive(&fullB[s]);
        } else {
          uint8_t *st = in_ring + (size_t)s * LI.bytes;
          const int64_t r0 = (int64_t)tile * RB;
          const int nrows = (int)min64(RB, n - r0);
          const uint32_t xb = (uint32_t)(nrows * C * sizeof(XT)), fb = (uint32_t)(nrows * C * 4);
          const uint32_t ub = (uint32_t)(((r0 & 3) + nrows + 3) / 4 * 16);
          mbar_expect_tx(&fullB[s], xb + (has_aux<MODE>() ? 2 * fb : 0u) + ub * nseg);
          if (u_ready) load_u(s, tile);
          bulk_g2s(st + LI.x, X + r0 * C, xb, &fullB[s], pol);
          if (has_aux<MODE>()) {
            bulk_g2s(st + LI.base, p.base + r0 * C, fb, &fullB[s], pol);
            bulk_g2s(st + LI.aux, p.aux + r0 * C, fb, &fullB[s], pol);
          }
        }
      }
      __syncwarp();
      if (tile < 0) break;
      ++k;
    }
    if (!u_ready) publish_u(min(k + 1, SI));  // stages 0..k (the last one holds the sentinel)
  } else if (storer) {
    if (p.stop_after == 1 || p.stop_after == 3) return;
    // ---- scale pass, row half (the consumers do the columns): g_d, u_{d,i} ----
    {
      __shared__ double gseg[kMaxSeg];
      mbar_wait(&handA[0], 0);  // bar1, relayed by consumer thread 0
      for (int d = 0; d < nseg; ++d) {  // g_d = mean |t| over segment d (cx:142), same order in every CTA
        double part = 0.0;
        for (int i = lane; i < G; i += 32) part += __ldcg(p.blkpart + (size_t)i * nseg + d);
        part = warp_sum(part);
        if (lane == 0) gseg[d] = part / ((double)n * (double)p.cw);
      }
      __syncwarp();
      const int64_t uch = (n + G - 1) / G;
      const int64_t ui0 = (int64_t)cta * uch, ui1 = min64(n, ui0 + uch);
      for (int d = 0; d < nseg; ++d) {
        const double g = gseg[d];
        for (int64_t i0 = ui0; i0 < ui1; i0 += 32 * 4) {
          double rs[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {  // loads first, then the math
            const int64_t i = i0 + lane + 32 * q;
            rs[q] = i < ui1 ? __ldcg(p.rowpart + d * n + i) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int64_t i = i0 + lane + 32 * q;
            if (i >= ui1) continue;
            float u;
            if (p.scale_mode == CC_SCALE_PER_CHANNEL) u = 1.0f;
            else if (p.scale_mode == CC_SCALE_PER_TOKEN) u = (float)(rs[q] / (double)p.cw);
            else if (g == 0.0) u = 1.0f;
            else u = (float)fmax((rs[q] / (double)p.cw) / g, kRowScaleFloor);  // cx:147
            p.u[d * p.un + i] = u;
            store_f32_bytes(p.body + d * p.body_stride + p.cbytes_seg + 4 * i, u);
          }
        }
      }
      __syncwarp();
      if (lane == 0) arrive_release(bar2);
    }
    if (p.stop_after) return;
    int o = 0;
    uint32_t ph = 0;
    const bool hint = !(K1_XP(p) & 1);  // results are not re-read in this launch: evict_first
    const uint64_t spol = l2_policy_evict_first();
    for (;; o = (o + 1 == SO) ? 0 : o + 1, ph ^= (o == 0)) {
      mbar_wait(&outFull[o], ph);
      const long long tile = tileO[o];
      if (tile < 0) break;
      if (lane == 0 && !(K1_XP(p) & 128)) {
        const uint8_t *so = out_ring + (size_t)o * LO.bytes;
        const int64_t r0 = (int64_t)tile * RB;
        const int nrows = (int)min64(RB, n - r0);
        if (hint) {
          bulk_s2g_hint(p.base + r0 * C, so + LO.base, (uint32_t)(nrows * C * 4), spol);
          if constexpr (has_aux<MODE>()) bulk_s2g_hint(p.aux + r0 * C, so + LO.aux, (uint32_t)(nrows * C * 4), spol);
        } else {
          bulk_s2g(p.base + r0 * C, so + LO.base, (uint32_t)(nrows * C * 4));
          if constexpr (has_aux<MODE>()) bulk_s2g(p.aux + r0 * C, so + LO.aux, (uint32_t)(nrows * C * 4));
        }
        if (nseg == 1) {
          bulk_s2g(p.body + r0 * p.cb_row, so + LO.codes, (uint32_t)(nrows * p.cb_row));
        } else {  // segment d's code row lives in its own body
          for (int rr = 0; rr < nrows; ++rr)
            for (int d = 0; d < nseg; ++d)
              bulk_s2g(p.body + d * p.body_stride + (r0 + rr) * p.cbs, so + LO.codes + rr * p.cb_row + d * p.cbs,
                       (uint32_t)p.cbs);
        }
        bulk_commit();
        bulk_wait_read<0>();  // smem source consumed -> the slot may be rewritten
      }
      if (lane == 0) mbar_arrive(&outFree[o]);
      __syncwarp();
    }
    if (lane == 0) bulk_wait_read<0>();  // smem sources consumed; the global writes complete on their own
    __syncwarp();
  } else {
    double cs[Q][4];
#pragma unroll
    for (int j = 0; j < Q; ++j) cs[j][0] = cs[j][1] = cs[j][2] = cs[j][3] = 0.0;
   {  // phase A
    int s = 0;
    uint32_t ph = 0;
    bool first = true;
    for (;; s = (s + 1 == SA) ? 0 : s + 1, ph ^= (s == 0)) {
      mbar_wait(&fullA[s], ph);
      if (first) {
        stamp(8);
        first = false;
      }
      const long long tile = tileA[s];
      if (tile < 0) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyA[s]);
        break;
      }
      const uint8_t *st = ring + (size_t)s * LA.bytes;
      const int nrows = (int)min64(RA, n - (int64_t)tile * RA);
      if (grp < p.groups && !(K1_XP(p) & 8)) {
        for (int r = grp; r < nrows; r += p.groups) {
          double rs[Q];
#pragma unroll
          for (int j = 0; j < Q; ++j) {
            rs[j] = 0.0;
            if (!qact[j]) continue;
            const size_t o = (size_t)r * C + qcol[j];
            float xx[4], bb[4] = {0.f, 0.f, 0.f, 0.f}, aa[4] = {0.f, 0.f, 0.f, 0.f};
            unpack_x(reinterpret_cast<const XT *>(st + LA.x) + o, xx);
            if constexpr (MODE == CC_WITH_FEEDBACK) unpack_f(reinterpret_cast<const float *>(st + LA.base) + o, bb);
            if constexpr (has_aux<MODE>()) unpack_f(reinterpret_cast<const float *>(st + LA.aux) + o, aa);
            double a[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              a[q] = fabs((double)target_of<MODE>(xx[q], bb[q], aa[q]));
              cs[j][q] += a[q];
            }
            rs[j] = ((a[0] + a[1]) + a[2]) + a[3];
          }
          if (nseg == 1) {  // one partial per warp
            double v = rs[0];
#pragma unroll
            for (int j = 1; j < Q; ++j) v += rs[j];
            v = warp_sum(v);
            if (lane == 0) rp[(((size_t)ph * SA + s) * RA + r) * kNB + wig] = v;
          } else {
#pragma unroll
            for (int j = 0; j < Q; ++j) {  // one partial per 128-column block
              const double v = warp_sum(rs[j]);
              if (lane == 0 && qblk[j] < kNB) rp[(((size_t)ph * SA + s) * RA + r) * kNB + qblk[j]] = v;
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyA[s]);
    }
   }
    stamp(9);
    if constexpr (Q == 1) {  // merge row groups' column partials in a fixed order
      double *xchg = reinterpret_cast<double *>(out_ring);  // in_ring is being refilled by the loader
      named_sync(1, kCons);
      if (in_group && qact[0]) {
#pragma unroll
        for (int q = 0; q < 4; ++q) xchg[((size_t)grp * p.G4 + quad0) * 4 + q] = cs[0][q];
      }
      named_sync(1, kCons);
      if (in_group && grp == 0 && qact[0]) {
        double *cp = p.colpart + (int64_t)cta * C + qcol[0];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          double v = cs[0][q];
          for (int g2 = 1; g2 < p.groups; ++g2) v += xchg[((size_t)g2 * p.G4 + quad0) * 4 + q];
          cp[q] = v;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        if (!qact[j]) continue;
        double *cp = p.colpart + (int64_t)cta * C + qcol[j];
        cp[0] = cs[j][0]; cp[1] = cs[j][1]; cp[2] = cs[j][2]; cp[3] = cs[j][3];
      }
    }
    // ---- hand-off 1: column partials published, wait for every CTA's phase A ----
    named_sync(1, kCons);
    if (tid == 0) arrive_release(bar1);
    if (p.stop_after == 3) return;
    stamp(1);
    if (tid == 0) {
      spin_until(bar1, 2u * G);
      mbar_arrive(&handA[0]);  // relay to the store warp
    }
    named_sync(1, kCons);
    stamp(2);
    if (p.stop_after == 1) return;

    // ================= phase F: v_j (consumers); g, u_i (store warp) =================
    if (cta == 0 && tid == 0) p.ctr[0] = 0ull;  // every phase-A claim happened before bar1
    {
      // column sums: one CTA per 32-column group; warp w sums CTA slots w, w + kCW, ...
      // (8 loads in flight per lane), then warp 0 adds the per-warp partials in order
      double *wpart = red + 16;  // [kCW][32] doubles after the reduction scratch
      for (int64_t grp32 = cta; grp32 * 32 < C; grp32 += G) {
        const int64_t j = grp32 * 32 + lane;
        double acc = 0.0;
        if (j < C) {
          constexpr int kB = 16;  // >= ceil(148 / kCW): one L2 round trip on B200
          for (int s0 = warp; s0 < G; s0 += kB * kCW) {
            double vals[kB];
#pragma unroll
            for (int q = 0; q < kB; ++q) {
              const int slot = s0 + q * kCW;
              vals[q] = slot < G ? __ldcg(p.colpart + (int64_t)slot * C + j) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kB; ++q) acc += vals[q];
          }
        }
        wpart[warp * 32 + lane] = acc;
        named_sync(1, kCons);
        if (warp == 0 && j < C) {
          double sacc = 0.0;
          for (int w = 0; w < kCW; ++w) sacc += wpart[w * 32 + lane];
          float v = (float)(sacc / (double)n);  // colmean (cx:148)
          if (p.scale_mode == CC_SCALE_PER_TOKEN) v = 1.0f;
          p.v[j] = v;
          const int d = (int)(j / p.cw);
          store_f32_bytes(p.body + d * p.body_stride + p.cbytes_seg + 4 * n + 4 * (j - (int64_t)d * p.cw), v);
        }
        named_sync(1, kCons);
      }
    }
    stamp(7);
    stamp(3);
    // ---- hand-off 2: v (consumers) and u (store warp) published ----
    named_sync(1, kCons);
    if (tid == 0) {
      arrive_release(bar2);
      spin_until(bar2, 2u * G);
      mbar_arrive(&handA[1]);  // relay to the loader
    }
    named_sync(1, kCons);
    stamp(4);
    if (p.stop_after == 2) return;

    // ================= phase B (consumers): quantize, pack, update state =================
    ColConst cc[Q];
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      cc[j].ok = true;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float v = qact[j] ? __ldcg(p.v + qcol[j] + q) : 1.0f;
        cc[j].v[q] = v;
        cc[j].vhi[q] = __fmul_ru(__fmul_ru(v, 1.25f), 1.00000095367431640625f);  // (1 + 2^-20)
        cc[j].vlo[q] = __fmul_rd(__fmul_rd(v, 1.25f), 0.99999904632568359375f);  // (1 - 2^-20)
        cc[j].ok = cc[j].ok && scale_in_range(fabsf(v));  // zero / extreme scales: exact path
      }
    }
    const int r = grp;  // this thread's row inside a phase-B tile
    int s = 0, o = 0, k = 0;
    uint32_t phs = 0, pho = 0;
    for (;; ++k, s = (s + 1 == SI) ? 0 : s + 1, phs ^= (s == 0), o = (o + 1 == SO) ? 0 : o + 1, pho ^= (o == 0)) {
      mbar_wait(&fullB[s], phs);
      const long long tile = tileB[s];
      if (tile < 0) {  // forward the end-of-work marker to the store warp
        __syncwarp();
        if (lane == 0) mbar_arrive(&emptyB[s]);
        if (k >= SO) mbar_wait(&outFree[o], pho ^ 1u);
        if (tid == 0) tileO[o] = -1;
        __syncwarp();
        if (lane == 0) mbar_arrive(&outFull[o]);
        break;
      }
      const uint8_t *st = in_ring + (size_t)s * LI.bytes;
      const int64_t r0 = (int64_t)tile * RB;
      const bool row_live = in_group && r0 + r < n && !(K1_XP(p) & 64);
      float xx[Q][4], bb[Q][4], aa[Q][4];
#pragma unroll
      for (int j = 0; j < Q; ++j) {
#pragma unroll
        for (int q = 0; q < 4; ++q) xx[j][q] = bb[j][q] = aa[j][q] = 0.f;
        if (row_live && qact[j]) {
          const size_t oo = (size_t)r * C + qcol[j];
          unpack_x(reinterpret_cast<const XT *>(st + LI.x) + oo, xx[j]);
          if constexpr (has_aux<MODE>()) {
            unpack_f(reinterpret_cast<const float *>(st + LI.base) + oo, bb[j]);
            unpack_f(reinterpret_cast<const float *>(st + LI.aux) + oo, aa[j]);
          }
        }
      }
      float ufj[Q];
#pragma unroll
      for (int j = 0; j < Q; ++j)
        ufj[j] = row_live ? ustage[((size_t)s * nseg + (SEG ? qseg[j] : 0)) * 16 + (r0 & 3) + r] : 1.0f;
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyB[s]);  // inputs are in registers: the loader may refill
      if (k >= SO) mbar_wait(&outFree[o], pho ^ 1u);
      uint8_t *so = out_ring + (size_t)o * LO.bytes;
      const bool direct = K1_XP(p) & 128;  // experiment: results straight to HBM (generic stores)
      float *obase = direct ? p.base + r0 * C : reinterpret_cast<float *>(so + LO.base);
      float *oaux = direct ? p.aux + r0 * C : reinterpret_cast<float *>(so + LO.aux);
      uint8_t *ocode = direct && nseg == 1 ? p.body + r0 * p.cb_row : so + LO.codes;
#pragma unroll
      for (int j = 0; j < Q; ++j) {
        float t[4], d[4], e[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) t[q] = target_of<MODE>(xx[j][q], bb[j][q], aa[j][q]);
        const uint32_t packed = quantize4<CODEC>(t, ufj[j], scale_in_range(fabsf(ufj[j])), cc[j], d);
#pragma unroll
        for (int q = 0; q < 4; ++q) e[q] = __fsub_rn(t[q], d[q]);
        const bool live = row_live && qact[j];
        const size_t oo = (size_t)r * C + qcol[j];
        if (live) {
          record4(t, e, err[SEG ? j : 0], tsq[SEG ? j : 0]);
          float4 nb;
          if constexpr (MODE == CC_NAIVE) {
            nb = make_float4(d[0], d[1], d[2], d[3]);
          } else {
            nb = make_float4(__fadd_rn(bb[j][0], d[0]), __fadd_rn(bb[j][1], d[1]), __fadd_rn(bb[j][2], d[2]),
                             __fadd_rn(bb[j][3], d[3]));
            *reinterpret_cast<float4 *>(oaux + oo) =
                MODE == CC_WITH_FEEDBACK ? make_float4(e[0], e[1], e[2], e[3])
                                         : make_float4(xx[j][0], xx[j][1], xx[j][2], xx[j][3]);
          }
          *reinterpret_cast<float4 *>(obase + oo) = nb;
        }
        uint8_t *crow = ocode + (size_t)r * p.cb_row;
        if constexpr (CODEC == CC_SIGN1) {
          const uint32_t other = __shfl_down_sync(0xffffffffu, packed, 1);
          if (live && (lane & 1) == 0) crow[qcol[j] >> 3] = (uint8_t)(packed | (other << 4));
        } else if constexpr (CODEC == CC_QUANT2) {
          if (live) crow[qcol[j] >> 2] = (uint8_t)packed;
        } else {
          if (live) *reinterpret_cast<uint16_t *>(crow + (qcol[j] >> 1)) = (uint16_t)packed;
        }
      }
      if (tid == 0) tileO[o] = tile;
      fence_proxy_async_smem();  // results -> visible to the TMA store engine
      __syncwarp();
      if (lane == 0) mbar_arrive(&outFull[o]);
    }
  }
  // ---- StepRecord: consumer warps only (the store warp drains its last stages
  // meanwhile; the loader made its last claim before publishing the sentinel) ----
  if (!consumer) return;
  pdl_launch_dependents();  // phase B done: the next kernel may launch during the record tail
  stamp(5);
  {
    __shared__ unsigned last;
    // per (warp, quad slot) partials, then per segment in a fixed (warp, slot) order
#pragma unroll
    for (int j = 0; j < Q; ++j) {
      const double a = warp_sum(err[j]), b = warp_sum(tsq[j]);
      if (lane == 0) {
        red[(warp * Q + j) * 2] = a;
        red[(warp * Q + j) * 2 + 1] = b;
      }
    }
    named_sync(1, kCons);
    if (tid < nseg) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < kCW; ++w)
        for (int j = 0; j < Q; ++j) {
          const int blk = Q == 2 ? j * kCW + w : (w % (int)(p.G4 / 32));
          if (nseg == 1 || (blk < kNB && blk / bps == tid)) {
            a += red[(w * Q + j) * 2];
            b += red[(w * Q + j) * 2 + 1];
          }
        }
      p.recpart[((size_t)cta * nseg + tid) * 2] = a;
      p.recpart[((size_t)cta * nseg + tid) * 2 + 1] = b;
    }
    named_sync(1, kCons);
    if (tid == 0) last = atom_add_acq_rel(p.ticket) == (unsigned)G - 1;  // release: partials; acquire: others'
    named_sync(1, kCons);
    if (last) {  // the last CTA reduces the per-CTA partials in a fixed order
      double vals[2 * kMaxSeg];
#pragma unroll
      for (int k = 0; k < 2 * kMaxSeg; ++k)  // every load in flight before the sums
        vals[k] = (k < 2 * nseg && tid < G) ? __ldcg(p.recpart + (size_t)tid * nseg * 2 + k) : 0.0;
      named_sync(1, kCons);  // red is reused below
#pragma unroll
      for (int k = 0; k < 2 * kMaxSeg; ++k) {
        if (k >= 2 * nseg) break;
        const double v = warp_sum(vals[k]);
        if (lane == 0) red[warp * 2 * kMaxSeg + k] = v;
      }
      named_sync(1, kCons);
      if (tid < 2 * nseg) {
        double a = 0.0;
        for (int w = 0; w < kCW; ++w) a += red[w * 2 * kMaxSeg + tid];
        p.record[tid] = a;  // record[2d] = ||d - t||^2, record[2d+1] = ||t||^2 of segment d
      }
      if (tid == 0) {
        // every CTA passed both hand-offs and finished claiming before taking its
        // ticket: leave the control words zeroed for the next launch
        p.ctr[16] = 0ull;
        *p.ticket = 0u;
        p.bar[0] = 0u;
        p.bar[32] = 0u;
      }
    }
  }
  stamp(6);
}

}  // namespace fused

// ---------------------------------------------------------------------------
// host-side launch (ring sizing from the shared-memory budget)
// ---------------------------------------------------------------------------
extern int g_fused_si, g_fused_so, g_fused_sa;  // debug ring overrides (k1_fused.cu)

template <int MODE, int CODEC, typename XT, int Q, bool SEG>
inline int launch_fused(fused::Params &p, cudaStream_t st) {
  using namespace fused;
  auto kern = k1_fused<MODE, CODEC, XT, Q, SEG>;
  const size_t ustage_bytes = (size_t)8 * p.nseg * 64;  // [S_in <= 8][nseg][16] floats
  const size_t fixed_tail = 512 * 8 + 3 * 8 * 8 * 3 + 8 * 64 + 256 + ustage_bytes;
  const size_t budget = kSmemBudget;
  // phase B rings (tiles of `groups` rows): loads S_in, outputs S_out
  const InStage LI = in_stage<MODE, XT>(p.groups, p.C, has_aux<MODE>());
  const OutStage LO = out_stage<MODE>(p.groups, p.C, p.cb_row);
  const InStage LA = in_stage<MODE, XT>(p.R, p.C, MODE == CC_WITH_FEEDBACK);
  // phase A ring + its row-partial scratch (2 use parities x SA stages)
  // full-width rows (> 1536 columns): 2-row tiles, 2 stages measured best at every shard height
  // (512..4096 rows: -0.8 .. -2.2 us vs 8 stages, scripts/microbench.py phase-A sweep)
  const int sa_default = p.G4 > kCons ? 2 : 8;
  int SA = (int)std::min<size_t>(g_fused_sa > 0 ? g_fused_sa : sa_default,
                                  (budget - fixed_tail) / (LA.bytes + (size_t)2 * p.R * kNB * 8));
  if (SA < 2) {
    set_error("k1_fused: phase-A stages do not fit shared memory");
    return CC_ERR_UNSUPPORTED;
  }
  const size_t rp_bytes = (size_t)2 * SA * p.R * kNB * 8;
  // phase B rings share the ring area: loads S_in, outputs S_out
  int SO = g_fused_so > 0 ? g_fused_so : 2, SI = 0;
  for (;;) {
    const size_t avail = budget - fixed_tail - rp_bytes;
    if ((size_t)SO * LO.bytes + 2 * (size_t)LI.bytes <= avail) {
      SI = (int)std::min<size_t>(g_fused_si > 0 ? g_fused_si : 8, (avail - (size_t)SO * LO.bytes) / LI.bytes);
      break;
    }
    if (SO == 1) break;
    --SO;
  }
  if (SI < 2) {
    set_error("k1_fused: phase-B stages do not fit shared memory");
    return CC_ERR_UNSUPPORTED;
  }
  const size_t ringB = (size_t)SI * LI.bytes + (size_t)SO * LO.bytes;
  const size_t ringA = (size_t)SA * LA.bytes;
  p.S = SA;
  p.S_in = SI;
  p.S_out = SO;
  p.ring_bytes = (uint32_t)align_up(std::max(ringA, ringB), 128);
  const size_t smem = p.ring_bytes + rp_bytes + 512 * 8 + (size_t)(3 * SA + 3 * SI + 3 * SO + 2) * 8 + 16 +
                      (size_t)SI * p.nseg * 64 + 128;
  static int smem_set = 0;  // per instantiation: raise the opt-in limit only when a launch needs more
  if ((int)smem > smem_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return cuda_status("k1_fused attr");
    smem_set = (int)smem;
  }
  void *args[] = {&p};
  if (p.ctl_in_ws) cudaMemsetAsync(p.ctr, 0, 512, st);  // control words
  cudaError_t e;
  if (pdl_enabled()) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(p.G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelExC(&cfg, (const void *)kern, args);
  } else {
    e = cudaLaunchCooperativeKernel((const void *)kern, dim3(p.G), dim3(kThreads), args, smem, st);
  }
  if (e != cudaSuccess) {
    set_error(std::string("k1_fused launch: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return CC_ERR_CUDA;
  }
  count_launch();
  return CC_OK;
}


// SEG = true instantiations live in k1_fused_seg.cu
int fused_dispatch_seg(fused::Params &p, int codec, int mode, int x_dtype, int Q, cudaStream_t st);

}  // namespace cc
