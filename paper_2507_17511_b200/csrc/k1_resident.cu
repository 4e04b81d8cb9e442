// K1, shard-resident form: ONE persistent cooperative kernel per encode_step that
// keeps the shard's residual t (and, when it fits, its base) in shared memory
// across the grid-wide scale dependency, so every byte of x / base / feedback is
// read from HBM exactly once and every result written once: 18 + b/8 B per
// element, the algorithmic traffic of SURVEY §8(d).
//
// Used when the CTA's residual rows fit on chip.  t lives in shared memory and,
// for rows beyond what shared memory holds, in TENSOR MEMORY (256 KB per SM,
// otherwise idle in this kernel): every thread parks its 8 values of such a row in
// its warp's TMEM lane quarter with tcgen05.st and takes them back with tcgen05.ld.
// Shared + tensor memory hold ~58 MB of t across 148 SMs, so even the P = 1 shard
// [4096, 3072] (50 MB) stays on chip: phase B re-reads only base (L2-resident,
// loaded evict_last in phase A).  Per shape:
//   [512 / 1024, 3072]  t + base in shared memory (no re-read at all);
//   [2048, 3072]        t in shared memory, base re-read;
//   [4096, 3072]        t in shared + tensor memory, base re-read.
// Larger shards take the streaming two-pass kernel (k1_fused_impl.cuh).
//
// CTA c owns the contiguous rows [c n / G, (c + 1) n / G) (static: every CTA moves
// the same bytes, so the phases end together without a tile scheduler).
//   phase A  a producer warp TMA-loads every row: x into a small ring, aux (feedback
//            / ref) straight into the row's resident t slot, base into its
//            resident slot (or through the ring when only t stays on chip); the 12
//            consumer warps form t = target(x, base, aux) in place (pipeline.py:99-104)
//            and accumulate |t| in f64: 8 column sums per thread in registers and one
//            partial per (row, 128-column block) in shared memory.
//   hand-off 1  flag barrier: column partials [G][C] published.
//   phase F  v_j = colmean over the G partials (one CTA per 32-column group);
//            g = mean|t| from the G CTA totals (same order in every CTA) and u_i of
//            the CTA's OWN rows from its on-chip row sums — u never leaves the CTA
//            except into the body (compressors.py:135-149).
//   hand-off 2  flag barrier: v published.
//   phase B  quantize from shared memory (compressors.py:373-391), base' / feedback'
//            / codes stored straight to HBM (pipeline.py:107-113), StepRecord partials
//            -> last-CTA ticket reduction (pipeline.py:115-120).
// Column segments (Ulysses (src, dst) chunks) exactly as in the
// streaming kernel: per-segment row sums, g, u, bodies and records.
//
// Arithmetic is element-for-element the streaming kernel's (same target, same f64
// scale formulas, same quantize4 / record4), so the bodies and states are
// bit-identical to it and to the multi-kernel path (tests/test_gpu_k1_resident.py).

#include "k1_fused_impl.cuh"

namespace cc {
namespace k1r {

using fused::ColConst;
constexpr int kNQ = 1;                // column quads per consumer thread (see Geo)
constexpr int kNB = fused::kNB;       // 128-column blocks per row (24 at C = 3072)
constexpr int kMaxSlots = 148;        // column-partial slots read per column in phase F (grid <= SMs)
constexpr int kMaxSeg = fused::kMaxSeg;
constexpr int kMaxStages = 8;
constexpr size_t kSmemMax = 227 * 1024;

struct Params {
  const void *x;
  float *base, *aux;
  int64_t n, C;
  int G4, G;
  int R;          // max rows per CTA (ceil(n / G))
  int nsm;        // rows whose t lives in shared memory; rows nsm.. live in tensor memory
  int keep_base;  // base rows resident (else streamed through the ring in both phases)
  int S;          // phase-A ring stages
  int SB;         // phase-B base slots (carved from the phase-A ring area)
  uint32_t stage_bytes, st_base, st_fb;                     // ring stage: x at 0, base, feedback (TMEM rows)
  uint32_t off_t, off_b, off_ring, off_rp, off_rs, off_u;   // shared-memory layout
  uint32_t off_bar, off_red;
  double *colpart, *blkpart, *recpart, *record;  // [G][C], [G][nseg], [G][nseg][2], [nseg][2]
  float *v;                                      // [C]
  uint8_t *body;
  int64_t body_stride, cbytes_seg;
  int nseg, cw, cbs, bps, cb_row;
  unsigned int *bar1, *bar2, *ticket;
  // row assignment: CTA c first takes the static rows [c stat, (c + 1) stat); with
  // dyn, the rows from G stat on are claimed one at a time from *claim (faster SMs
  // take more: balances the phases' ends) up to R rows per CTA in total
  int dyn, stat;
  unsigned int *claim;
  uint32_t off_rows;  // shared-memory row list [R + 1]
  int scale_mode;
  unsigned long long *timer;  // profiling: [G][16] %globaltimer stamps, or null
  int policy;                 // experiments: L2 hints of the phase-A loads (0 = production)
};

template <typename XT>
__device__ __forceinline__ void ld_x4(const XT *p, float (&v)[4]) {
  fused::unpack_x(p, v);
}

// ---- tensor memory (tcgen05) as a residual store --------------------------------
__device__ __forceinline__ void tmem_alloc512(uint32_t *dst_smem) {  // warp-collective
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(dst_smem))
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc512(uint32_t taddr) {  // warp-collective
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(taddr) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// each lane writes / reads 4 NQ consecutive 32-bit columns of its own TMEM lane
template <int NQ>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const float (&v)[NQ][4]) {
  if constexpr (NQ == 1) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0][0])), "r"(__float_as_uint(v[0][1])), "r"(__float_as_uint(v[0][2])),
                 "r"(__float_as_uint(v[0][3]))
                 : "memory");
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(__float_as_uint(v[0][0])), "r"(__float_as_uint(v[0][1])), "r"(__float_as_uint(v[0][2])),
                 "r"(__float_as_uint(v[0][3])), "r"(__float_as_uint(v[NQ - 1][0])), "r"(__float_as_uint(v[NQ - 1][1])),
                 "r"(__float_as_uint(v[NQ - 1][2])), "r"(__float_as_uint(v[NQ - 1][3]))
                 : "memory");
  }
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
template <int NQ>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[NQ][4]) {
  uint32_t r[8];
  if constexpr (NQ == 1) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr)
                 : "memory");
  } else {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr)
                 : "memory");
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int j = 0; j < NQ; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) v[j][q] = __uint_as_float(r[4 * j + q]);
}

__device__ __forceinline__ void stcs4(float *p, const float (&v)[4]) {
  __stcs(reinterpret_cast<float4 *>(p), make_float4(v[0], v[1], v[2], v[3]));
}

// The 2-bit fast path of fused::quantize4<CC_QUANT2> with fewer instructions (same
// decisions and values, bit for bit): code bit 1 = !neg, bit 0 = big ^ neg, and
// d = (+-2 | +-0.5) * RN(u v); elements in the guard band, and rows / columns with
// extreme scales, take the exact f64 path (compressors.py:379-391).
__device__ __forceinline__ uint32_t quant2_lean(const float (&t)[4], float uf, const fused::ColConst &cc,
                                                float (&d)[4]) {
  uint32_t packed = 0;
  bool ambiguous = !(cc.ok && fused::scale_in_range(fabsf(uf)));
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const float ax = fabsf(t[q]);
    const bool big = ax > __fmul_rn(uf, cc.vhi[q]);
    ambiguous |= !big && !(ax < __fmul_rn(uf, cc.vlo[q]));
    const bool neg = t[q] < 0.0f;
    const float lv = big ? 2.0f : 0.5f;
    d[q] = __fmul_rn(neg ? -lv : lv, __fmul_rn(uf, cc.v[q]));
    packed |= ((neg ? 0u : 2u) | ((uint32_t)big ^ (uint32_t)neg)) << (2 * q);
  }
  if (__builtin_expect(ambiguous, 0)) {
    packed = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const fused::CodeVal r = fused::quantize1_exact<CC_QUANT2>(t[q], (double)uf, (double)cc.v[q]);
      d[q] = r.d;
      packed |= r.code << (2 * q);
    }
  }
  return packed;
}

// A ring position: stage index and the parity of its current use, advanced
// incrementally (no runtime division in the loops).
struct RingPos {
  int s = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next(int S) {
    if (++s == S) {
      s = 0;
      ph ^= 1u;
    }
  }
};

// NQ column quads per consumer thread: 768 / NQ consumer threads cover the 3072
// columns of a full row (quad j of thread tid = quad tid + j CONS).  NQ = 1 (24
// consumer warps) hides latency best; NQ = 2 (12 warps) is the register-light form.
template <int NQ>
struct Geo {
  static constexpr int CONS = 768 / NQ;
  static constexpr int CW = CONS / 32;
  static constexpr int THREADS = CONS + 32;  // + producer warp
};

// TMEM address of a consumer warp's 4 NQ columns of tensor-memory row m: warp w
// reaches lanes 32 (w % 4) .. + 31; the CW / 4 warps sharing a lane quarter take 4 NQ
// columns each, so a row uses 24 of the 512 columns (<= 21 rows).
template <int NQ>
__device__ __forceinline__ uint32_t tmem_off(int warp, int m) {
  return ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(m * 24 + (warp >> 2) * 4 * NQ);
}

template <int MODE, int CODEC, typename XT, int NQ>
// NQ = 2 is register-capped (two CTAs' worth) so a decode kernel on another stream
// can share the SM during the hand-offs (overlap experiments at small shards)
__global__ void __launch_bounds__(Geo<NQ>::THREADS, NQ == 2 ? 2 : 1) k1_resident(const __grid_constant__ Params p) {
  constexpr int CONS = Geo<NQ>::CONS, CW = Geo<NQ>::CW;
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x, G = p.G, S = p.S, SB = p.SB;
  const int64_t n = p.n, C = p.C;
  const int nseg = p.nseg;
  int *rowS = reinterpret_cast<int *>(smem + p.off_rows);  // [R + 1]: row of each slot, -1 ends
  constexpr bool kAux = MODE != CC_NAIVE;
  constexpr bool kWB = MODE == CC_WITH_FEEDBACK;
  const bool keep_base = kAux && p.keep_base;
  const bool ring_base = kAux && !p.keep_base;  // base through the ring (phase A if kWB, phase B always)

  float *tS = reinterpret_cast<float *>(smem + p.off_t);   // [nsm][C]
  float *bS = reinterpret_cast<float *>(smem + p.off_b);   // [R][C] (keep_base)
  uint8_t *ring = smem + p.off_ring;                        // [S][stage_bytes] / [SB][4 C]
  double *rp = reinterpret_cast<double *>(smem + p.off_rp); // [R][kNB]
  double *rs = reinterpret_cast<double *>(smem + p.off_rs); // [R][nseg] row sums
  float *uS = reinterpret_cast<float *>(smem + p.off_u);    // [R][nseg]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *empty = full + kMaxStages;
  uint64_t *fullB = empty + kMaxStages;  // phase-B base slots
  uint64_t *emptyB = fullB + kMaxStages;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(emptyB + kMaxStages);
  double *red = reinterpret_cast<double *>(smem + p.off_red);  // [CW][32]
  const bool use_tmem = p.nsm < p.R;

  auto stamp = [&](int i) {
    if (p.timer && tid == 0) p.timer[(size_t)cta * 16 + i] = fused::gtimer();
  };
  stamp(0);
  if (p.timer && tid == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    p.timer[(size_t)cta * 16 + 8] = smid;
  }
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CW);
    }
    for (int s = 0; s < SB; ++s) {
      mbar_init(&fullB[s], 1);
      mbar_init(&emptyB[s], CW);
    }
    mbar_fence_init();
  }
  if (use_tmem && warp == 0) tmem_alloc512(tmem_slot);  // the whole TMEM: one CTA per SM
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = use_tmem ? *tmem_slot : 0u;
  const XT *X = reinterpret_cast<const XT *>(p.x);

  if (warp == CW) {  // ===================== producer warp =====================
    if (lane == 0) {
      const uint64_t pol_once = (K1_XP(p) & 4) ? fused::l2_policy_normal() : l2_policy_evict_first();
      // base rows are re-read in phase B, but keeping them L2-resident (evict_last)
      // slows phase A more than the re-read costs: [4096, 3072] 62.6 us with
      // evict_last, 60.5 us with evict_first (scripts/k1_ab.py --policies)
      const uint64_t pol_again = (K1_XP(p) & 1)   ? fused::l2_policy_normal()
                                 : (K1_XP(p) & 2) ? l2_policy_evict_last()
                                                  : l2_policy_evict_first();
      const uint64_t pol_b = (K1_XP(p) & 8) ? fused::l2_policy_normal() : l2_policy_evict_first();
      const uint32_t xb = (uint32_t)(C * sizeof(XT)), fb = (uint32_t)(C * 4);
      uint32_t bytes = xb;
      if (kAux) bytes += fb;
      if (kWB || keep_base) bytes += fb;
      // phase A: one ring use per row.  Rows with t in shared memory take their aux
      // straight into the t slot; rows with t in tensor memory stage it in the ring.
      RingPos w;
      const int64_t s0 = (int64_t)cta * p.stat;
      const int nstat = p.dyn ? p.stat : (int)((int64_t)(cta + 1) * n / G - (int64_t)cta * n / G);
      const int64_t rbase = p.dyn ? s0 : (int64_t)cta * n / G;
      int k = 0;
      for (;; ++k, w.next(S)) {
        int64_t row;
        if (k < nstat) {
          row = rbase + k;
        } else {
          if (!p.dyn || k >= p.R) break;
          row = (int64_t)G * p.stat + atomicAdd(p.claim, 1u);
          if (row >= n) break;
        }
        if (k >= S) mbar_wait(&empty[w.s], w.ph ^ 1u);
        rowS[k] = (int)row;
        const int64_t off = row * C;
        uint8_t *st = ring + (size_t)w.s * p.stage_bytes;
        mbar_expect_tx(&full[w.s], bytes);
        bulk_g2s(st, X + off, xb, &full[w.s], pol_once);
        if (kAux) {
          float *dst = k < p.nsm ? tS + (size_t)k * C : reinterpret_cast<float *>(st + p.st_fb);
          bulk_g2s(dst, p.aux + off, fb, &full[w.s], pol_once);
        }
        if (keep_base) {
          bulk_g2s(bS + (size_t)k * C, p.base + off, fb, &full[w.s], pol_once);
        } else if (kWB) {
          bulk_g2s(st + p.st_base, p.base + off, fb, &full[w.s], pol_again);
        }
      }
      const int nr = k;
      // end of phase A: a ring use with no data (row -1)
      if (k >= S) mbar_wait(&empty[w.s], w.ph ^ 1u);
      rowS[k] = -1;
      mbar_arrive(&full[w.s]);
      w.next(S);
      // phase B: base rows through SB slots carved from the ring area, newest first
      // (the most recently loaded base rows are the likeliest L2 hits), loaded while
      // the consumers wait on the hand-offs
      if (ring_base) {
        // the ring area is free once phase A's last min(S, nr + 1) uses are released
        RingPos q = w;
        for (int i = 0; i < min(S, nr + 1); ++i) {
          if (--q.s < 0) {
            q.s = S - 1;
            q.ph ^= 1u;
          }
          mbar_wait(&empty[q.s], q.ph);
        }
        RingPos b;
        for (int i = 0; i < nr; ++i, b.next(SB)) {
          const int k = nr - 1 - i;
          if (i >= SB) mbar_wait(&emptyB[b.s], b.ph ^ 1u);
          mbar_expect_tx(&fullB[b.s], fb);
          bulk_g2s(ring + (size_t)b.s * fb, p.base + (int64_t)rowS[k] * C, fb, &fullB[b.s], pol_b);
        }
      }
    }
    return;
  }

  // ===================== consumer warps =====================
  bool qact[NQ];
  int qcol[NQ], qblk[NQ], qseg[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    const int qd = tid + j * CONS;
    qact[j] = qd < p.G4;
    qcol[j] = 4 * qd;
    qblk[j] = j * CW + warp;  // 128-column block of the quad
    qseg[j] = nseg == 1 ? 0 : min(qblk[j] / p.bps, nseg - 1);
  }
  double cs[NQ][4];
#pragma unroll
  for (int j = 0; j < NQ; ++j) cs[j][0] = cs[j][1] = cs[j][2] = cs[j][3] = 0.0;

  // ---------------- phase A ----------------
  int nr = 0;
  {
    RingPos w;
    for (int k = 0;; ++k, w.next(S)) {
      mbar_wait(&full[w.s], w.ph);
      if (k == 0) stamp(1);
      const int rowk = rowS[k];
      if (rowk < 0) {  // end of the CTA's rows
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[w.s]);
        nr = k;
        break;
      }
      const uint8_t *st = ring + (size_t)w.s * p.stage_bytes;
      const XT *xs = reinterpret_cast<const XT *>(st);
      const bool in_smem = k < p.nsm;
      float *trow = tS + (size_t)k * C;
      const float *arow = in_smem ? trow : reinterpret_cast<const float *>(st + p.st_fb);
      const float *brow = keep_base ? bS + (size_t)k * C : reinterpret_cast<const float *>(st + p.st_base);
      float *refrow = p.aux + (int64_t)rowk * C;
      double rsum[NQ];
      float tt[NQ][4];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        rsum[j] = 0.0;
        tt[j][0] = tt[j][1] = tt[j][2] = tt[j][3] = 0.f;
        if (!qact[j]) continue;
        const int o = qcol[j];
        float xx[4], bb[4] = {0.f, 0.f, 0.f, 0.f}, aa[4] = {0.f, 0.f, 0.f, 0.f};
        ld_x4(xs + o, xx);
        if constexpr (kWB) fused::unpack_f(brow + o, bb);
        if constexpr (kAux) fused::unpack_f(arow + o, aa);
        double a[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          tt[j][q] = target_of<MODE>(xx[q], bb[q], aa[q]);
          a[q] = fabs((double)tt[j][q]);
          cs[j][q] += a[q];
        }
        rsum[j] = ((a[0] + a[1]) + a[2]) + a[3];
        if (in_smem) *reinterpret_cast<float4 *>(trow + o) = make_float4(tt[j][0], tt[j][1], tt[j][2], tt[j][3]);
        if constexpr (MODE == CC_NO_FEEDBACK) stcs4(refrow + o, xx);  // ref' = a* (pl:113)
      }
      if (!in_smem) tmem_st<NQ>(tmem + tmem_off<NQ>(warp, k - p.nsm), tt);  // warp-collective
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        const double v = warp_sum(rsum[j]);
        if (lane == 0 && qblk[j] < kNB) rp[(size_t)k * kNB + qblk[j]] = v;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[w.s]);
    }
  }
  if (use_tmem) tmem_wait_st();
  stamp(2);
  // column partials of this CTA
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    if (!qact[j]) continue;
    double *cp = p.colpart + (int64_t)cta * C + qcol[j];
    cp[0] = cs[j][0]; cp[1] = cs[j][1]; cp[2] = cs[j][2]; cp[3] = cs[j][3];
  }
  stamp(9);
  // the CTA's |t| total(s) for g: with one segment straight from the column sums in
  // registers (warp butterflies, warps in order) so the arrival does not wait for the
  // row sums; those (needed only for u) are formed while the barrier completes
  auto row_sums = [&]() {  // per segment (blocks of the segment in order)
    for (int i = tid; i < nr * nseg; i += CONS) {
      const int k = i / nseg, d = i - k * nseg;
      double acc = 0.0;
      for (int b = 0; b < p.bps; ++b) acc += rp[(size_t)k * kNB + d * p.bps + b];
      rs[i] = acc;
    }
  };
  if (nseg == 1) {
    double tsum = 0.0;
#pragma unroll
    for (int j = 0; j < NQ; ++j)
      if (qact[j]) tsum += ((cs[j][0] + cs[j][1]) + cs[j][2]) + cs[j][3];
    tsum = warp_sum(tsum);
    if (lane == 0) red[warp * 32] = tsum;
    fused::named_sync(1, CONS);
    if (tid == 0) {
      double tot = 0.0;
      for (int w = 0; w < CW; ++w) tot += red[w * 32];
      p.blkpart[cta] = tot;
    }
  } else {
    fused::named_sync(1, CONS);
    row_sums();
    fused::named_sync(1, CONS);
    if (tid < nseg) {
      double tot = 0.0;
      for (int k = 0; k < nr; ++k) tot += rs[k * nseg + tid];
      p.blkpart[(size_t)cta * nseg + tid] = tot;
    }
  }
  // ---- hand-off 1 ----
  fused::named_sync(1, CONS);
  stamp(10);
  if (tid == 0) fused::arrive_release(p.bar1);
  stamp(11);
  if (nseg == 1) row_sums();  // overlaps the barrier
  if (tid == 0) fused::spin_until(p.bar1, (unsigned)G);
  fused::named_sync(1, CONS);
  stamp(3);

  // ---------------- phase F ----------------
  {
    double *wpart = red;  // [CW][32]
    for (int64_t grp32 = cta; grp32 * 32 < C; grp32 += G) {
      const int64_t j = grp32 * 32 + lane;
      double acc = 0.0;
      if (j < C) {
        constexpr int kB = (kMaxSlots + CW - 1) / CW;  // one L2 round trip for all G slots
        for (int s0 = warp; s0 < G; s0 += kB * CW) {
          double vals[kB];
#pragma unroll
          for (int q = 0; q < kB; ++q) {
            const int slot = s0 + q * CW;
            vals[q] = slot < G ? __ldcg(p.colpart + (int64_t)slot * C + j) : 0.0;
          }
#pragma unroll
          for (int q = 0; q < kB; ++q) acc += vals[q];
        }
      }
      wpart[warp * 32 + lane] = acc;
      fused::named_sync(1, CONS);
      if (warp == 0 && j < C) {
        double sacc = 0.0;
        for (int w = 0; w < CW; ++w) sacc += wpart[w * 32 + lane];
        float v = (float)(sacc / (double)n);  // colmean (cx:148)
        if (p.scale_mode == CC_SCALE_PER_TOKEN) v = 1.0f;
        p.v[j] = v;
        const int d = (int)(j / p.cw);
        store_f32_bytes(p.body + d * p.body_stride + p.cbytes_seg + 4 * n + 4 * (j - (int64_t)d * p.cw), v);
      }
      fused::named_sync(1, CONS);
    }
  }
  // v published: arrive now, compute g / u of the own rows while the others finish
  fused::named_sync(1, CONS);
  stamp(4);
  if (tid == 0) fused::arrive_release(p.bar2);
  {
    __shared__ double gseg[kMaxSeg];
    for (int d = warp; d < nseg; d += CW) {  // g_d = mean |t| over segment d, same order in every CTA
      double part = 0.0;
      for (int i = lane; i < G; i += 32) part += __ldcg(p.blkpart + (size_t)i * nseg + d);
      part = warp_sum(part);
      if (lane == 0) gseg[d] = part / ((double)n * (double)p.cw);
    }
    fused::named_sync(1, CONS);
    for (int i = tid; i < nr * nseg; i += CONS) {
      const int k = i / nseg, d = i - k * nseg;
      const double g = gseg[d], rsum = rs[i];
      float u;
      if (p.scale_mode == CC_SCALE_PER_CHANNEL) u = 1.0f;
      else if (p.scale_mode == CC_SCALE_PER_TOKEN) u = (float)(rsum / (double)p.cw);
      else if (g == 0.0) u = 1.0f;  // all-zero segment (cx:143-146)
      else u = (float)fmax((rsum / (double)p.cw) / g, kRowScaleFloor);  // cx:147
      uS[i] = u;
      store_f32_bytes(p.body + d * p.body_stride + p.cbytes_seg + 4 * (int64_t)rowS[k], u);
    }
  }
  // ---- hand-off 2: every CTA's v ----
  if (tid == 0) fused::spin_until(p.bar2, (unsigned)G);
  fused::named_sync(1, CONS);
  stamp(5);

  // ---------------- phase B ----------------
  ColConst cc[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    cc[j].ok = true;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float v = qact[j] ? __ldcg(p.v + qcol[j] + q) : 1.0f;
      cc[j].v[q] = v;
      cc[j].vhi[q] = __fmul_ru(__fmul_ru(v, 1.25f), 1.00000095367431640625f);  // (1 + 2^-20)
      cc[j].vlo[q] = __fmul_rd(__fmul_rd(v, 1.25f), 0.99999904632568359375f);  // (1 - 2^-20)
      cc[j].ok = cc[j].ok && fused::scale_in_range(fabsf(v));
    }
    // keep the column constants in registers: left to itself the compiler re-derives
    // vhi / vlo (4 directed-rounding multiplies per element) in every row
#pragma unroll
    for (int q = 0; q < 4; ++q) asm volatile("" : "+f"(cc[j].v[q]), "+f"(cc[j].vhi[q]), "+f"(cc[j].vlo[q]));
  }
  // code byte offset of each quad inside its segment's code row
  int ccol[NQ];
  uint8_t *cbase[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) {
    const int sg = qseg[j];
    ccol[j] = (qcol[j] - sg * p.cw) * (CODEC == CC_SIGN1 ? 1 : CODEC == CC_QUANT2 ? 2 : 4) / 8;
    cbase[j] = p.body + sg * p.body_stride;
  }
  double err[NQ], tsq[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) err[j] = tsq[j] = 0.0;
  RingPos bpos;
  for (int i = 0; i < nr; ++i) {
    const int k = nr - 1 - i;  // newest rows first (matches the producer's base order)
    const int64_t row = rowS[k];
    const float *brow = bS + (size_t)k * C;
    if (ring_base) {
      mbar_wait(&fullB[bpos.s], bpos.ph);
      brow = reinterpret_cast<const float *>(ring + (size_t)bpos.s * C * 4);
    }
    const bool in_smem = k < p.nsm;
    const float *trow = tS + (size_t)k * C;
    float tt[NQ][4];
    if (!in_smem) tmem_ld<NQ>(tmem + tmem_off<NQ>(warp, k - p.nsm), tt);  // warp-collective
    // 32-bit offsets: a resident shard holds < 2^31 elements (it fits on chip)
    const uint32_t ro = (uint32_t)row * (uint32_t)C;
    float *obase = p.base + ro, *oaux = p.aux + ro;
    const uint32_t crow = (uint32_t)row * (uint32_t)p.cbs;
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const int o = qcol[j];
      float t[4], bb[4] = {0.f, 0.f, 0.f, 0.f}, d[4], e[4];
      if (qact[j]) {
        if (in_smem) {
          fused::unpack_f(trow + o, t);
        } else {
          t[0] = tt[j][0]; t[1] = tt[j][1]; t[2] = tt[j][2]; t[3] = tt[j][3];
        }
        if constexpr (kAux) fused::unpack_f(brow + o, bb);
      } else {
        t[0] = t[1] = t[2] = t[3] = 0.f;
      }
      const float uf = uS[k * nseg + qseg[j]];
      uint32_t packed;
      if constexpr (CODEC == CC_QUANT2) packed = quant2_lean(t, uf, cc[j], d);
      else packed = fused::quantize4<CODEC>(t, uf, fused::scale_in_range(fabsf(uf)), cc[j], d);
#pragma unroll
      for (int q = 0; q < 4; ++q) e[q] = __fsub_rn(t[q], d[q]);
      if (qact[j]) {
        fused::record4(t, e, err[j], tsq[j]);
        float nb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) nb[q] = MODE == CC_NAIVE ? d[q] : __fadd_rn(bb[q], d[q]);
        stcs4(obase + o, nb);
        if constexpr (kWB) stcs4(oaux + o, e);
      }
      // codes: segment d's code row lives in its own body
      uint8_t *cp = cbase[j] + (crow + (uint32_t)ccol[j]);
      if constexpr (CODEC == CC_SIGN1) {
        const uint32_t other = __shfl_down_sync(0xffffffffu, packed, 1);
        if (qact[j] && (lane & 1) == 0) *cp = (uint8_t)(packed | (other << 4));
      } else if constexpr (CODEC == CC_QUANT2) {
        if (qact[j]) *cp = (uint8_t)packed;
      } else {
        if (qact[j]) *reinterpret_cast<uint16_t *>(cp) = (uint16_t)packed;
      }
    }
    if (ring_base) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&emptyB[bpos.s]);
      bpos.next(SB);
    }
  }
  if (use_tmem) {  // every consumer warp is done with tensor memory before it is freed
    tc_fence_before();
    fused::named_sync(1, CONS);
    tc_fence_after();
    if (warp == 0) tmem_dealloc512(tmem);
  }
  stamp(6);

  // ---------------- StepRecord ----------------
  {
    __shared__ unsigned last;
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      const double a = warp_sum(err[j]), b = warp_sum(tsq[j]);
      if (lane == 0) {
        red[(warp * NQ + j) * 2] = a;
        red[(warp * NQ + j) * 2 + 1] = b;
      }
    }
    fused::named_sync(1, CONS);
    if (tid < nseg) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < CW; ++w)
        for (int j = 0; j < NQ; ++j) {
          const int blk = j * CW + w;
          if (nseg == 1 || (blk < kNB && blk / p.bps == tid)) {
            a += red[(w * NQ + j) * 2];
            b += red[(w * NQ + j) * 2 + 1];
          }
        }
      p.recpart[((size_t)cta * nseg + tid) * 2] = a;
      p.recpart[((size_t)cta * nseg + tid) * 2 + 1] = b;
    }
    fused::named_sync(1, CONS);
    stamp(12);
    if (tid == 0) last = fused::atom_add_acq_rel(p.ticket) == (unsigned)G - 1;
    fused::named_sync(1, CONS);
    stamp(13);
    if (last) {
      // thread i < G holds CTA i's partials; warps sum them in a fixed order
      double vals[2 * kMaxSeg];
#pragma unroll
      for (int q = 0; q < 2 * kMaxSeg; ++q)
        vals[q] = (q < 2 * nseg && tid < G) ? __ldcg(p.recpart + (size_t)tid * nseg * 2 + q) : 0.0;
      fused::named_sync(1, CONS);
#pragma unroll
      for (int q = 0; q < 2 * kMaxSeg; ++q) {
        if (q >= 2 * nseg) break;
        const double v = warp_sum(vals[q]);
        if (lane == 0) red[warp * 2 * kMaxSeg + q] = v;
      }
      fused::named_sync(1, CONS);
      if (tid < 2 * nseg) {
        double a = 0.0;
        for (int w = 0; w < CW; ++w) a += red[w * 2 * kMaxSeg + tid];
        p.record[tid] = a;
      }
      if (tid == 0) {  // every CTA is past both hand-offs: leave the control words zeroed
        *p.ticket = 0u;
        *p.bar1 = 0u;
        *p.bar2 = 0u;
        *p.claim = 0u;
      }
    }
  }
  stamp(7);
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static bool g_resident_enabled = true;
// shared memory the 12-warp form leaves free for kernels sharing its SMs (the decode
// needs none; an NCCL kernel at N > 1 may): measured on the per-rank sims, 0 / 48 /
// 96 KB free: [2048, 3072] 45.9 / 44.5 / 43.7 us, [1024, 3072] 32.5 / 36.2 / 33.8 us
// (the base rows stop fitting on chip), [512, 3072] 28.5 in all three: default 0
static size_t g_share_smem = [] {
  const char *e = std::getenv("CC_K1_SHARE_SMEM_KB");
  return (size_t)(e ? std::atoi(e) : 0) * 1024;
}();
// consumer quads per thread: 1 (24 warps) or 2 (12 register-capped warps); 0 = by shape
static int g_resident_nq = [] {
  const char *e = std::getenv("CC_K1_RESIDENT_NQ");  // experiments
  return e ? std::atoi(e) : 0;
}();
static int g_resident_grid = [] {  // persistent grid size: 0 = by shape (below), -1 = every SM
  const char *e = std::getenv("CC_K1_RESIDENT_GRID");
  return e ? std::atoi(e) : 0;
}();
std::atomic<int64_t> g_resident_launches{0};

template <int MODE, int CODEC, typename XT, int NQ>
static int launch(Params &p, size_t smem, cudaStream_t st) {
  auto kern = k1_resident<MODE, CODEC, XT, NQ>;
  static int smem_set = 0;
  if ((int)smem > smem_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return cuda_status("k1_resident attr");
    smem_set = (int)smem;
  }
  void *args[] = {&p};
  const cudaError_t e =
      cudaLaunchCooperativeKernel((const void *)kern, dim3(p.G), dim3(Geo<NQ>::THREADS), args, smem, st);
  if (e != cudaSuccess) {
    set_error(std::string("k1_resident launch: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return CC_ERR_CUDA;
  }
  count_launch();
  g_resident_launches.fetch_add(1, std::memory_order_relaxed);
  return CC_OK;
}

}  // namespace k1r

int64_t resident_launches() { return k1r::g_resident_launches.load(); }

void set_resident_enabled(int on) { k1r::g_resident_enabled = on != 0; }
void set_resident_nq(int nq) { k1r::g_resident_nq = nq == 2 ? 2 : nq == 1 ? 1 : 0; }

// Shared / tensor-memory plan for a shard; false when the CTA's rows do not fit.
static bool resident_plan(k1r::Params &q, int mode, int x_dtype, int nq) {
  using namespace k1r;
  const int64_t C = q.C;
  const size_t xb = (size_t)C * (x_dtype == CC_BF16 ? 2 : 4), fb = (size_t)C * 4;
  const bool aux = mode != CC_NAIVE;
  constexpr int kTmemRows = 512 / 24;  // tensor-memory rows per CTA (tmem_off)
  // returns the shared bytes of a layout with `nsm` shared-memory t rows
  auto layout = [&](int keep_base, int S, int nsm) -> size_t {
    const size_t R = (size_t)q.R;
    size_t off = 0;
    auto take = [&](size_t b) {
      const size_t o = off;
      off = align_up(off + b, 128);
      return (uint32_t)o;
    };
    q.keep_base = keep_base;
    q.S = S;
    q.nsm = nsm;
    const bool ring_base = aux && !keep_base;
    const bool tmem_rows = nsm < q.R;
    // ring stage: x | base (feedback mode, base streamed) | aux (tensor-memory rows)
    size_t st = align_up(xb, 128);
    q.st_base = (uint32_t)st;
    if (mode == CC_WITH_FEEDBACK && ring_base) st = align_up(st + fb, 128);
    q.st_fb = (uint32_t)st;
    if (aux && tmem_rows) st = align_up(st + fb, 128);
    q.stage_bytes = (uint32_t)st;
    size_t ring = (size_t)S * q.stage_bytes;
    q.SB = 0;
    if (ring_base) {  // phase-B base slots in the ring area (at least 2)
      ring = std::max(ring, 2 * fb);
      q.SB = (int)std::min<size_t>(kMaxStages, ring / fb);
    }
    q.off_t = take((size_t)nsm * fb);
    q.off_b = take(keep_base ? R * fb : 0);
    q.off_ring = take(ring);
    q.off_rp = take(R * kNB * 8);
    q.off_rs = take(R * q.nseg * 8);
    q.off_u = take(R * q.nseg * 4);
    q.off_bar = take(4 * kMaxStages * 8 + 16);
    q.off_rows = take(4 * (R + 1));
    q.off_red = take((size_t)(nq == 2 ? Geo<2>::CW : Geo<1>::CW) * 32 * 8);
    return off + 16 * 8 + 64;  // + static shared (gseg, last)
  };
  // the register-capped form shares its SMs (the previous layer's decode, NCCL's
  // collective kernels at N > 1): it leaves kShareSmem of shared memory free
  const size_t budget = kSmemMax - 1024 - (nq == 2 ? g_share_smem : 0);
  // 1. every row in shared memory (t, and base when it fits too)
  for (int keep_base : {aux ? 1 : 0, 0}) {
    for (int S = kMaxStages; S >= 2; --S)
      if (layout(keep_base, S, q.R) <= budget) return true;
    if (!aux) break;
  }
  // 2. overflow rows in tensor memory (base streamed): the deepest ring that leaves
  //    with the most shared t rows for it.  Experiment (policy bit 4096): a few rows
  //    of headroom per CTA, ~80 % of the rows assigned statically and the rest claimed
  //    one at a time, so faster SMs take more — phase A then ends together, but the
  //    producer's claim round trips stall its ring and the step got slower ([4096,
  //    3072] 59.3 -> 61.5-63.9 us, scripts/k1_ab.py): static rows are the default
  const int s_force = (q.policy >> 16) & 15;  // experiments: ring depth override
  const int R0 = q.R;
  const bool no_dyn = (q.policy & 4096) == 0;
  for (int extra : {6, 4, 2, 0}) {
    if (no_dyn && extra) continue;
    q.R = R0 + extra;
    for (int S = s_force ? s_force : kMaxStages; S >= 2; --S) {
      for (int nsm = q.R - 1; nsm >= std::max(0, q.R - kTmemRows); --nsm) {
        if (layout(0, S, nsm) <= budget) {
          q.dyn = extra > 0;
          q.stat = extra > 0 ? (int)(0.8 * (double)q.n / q.G) : 0;
          return true;
        }
      }
    }
  }
  q.R = R0;
  return false;
}

// Try the shard-resident K1; CC_ERR_UNSUPPORTED when the shard does not fit (the
// caller then launches the streaming kernel).  `fp` carries the workspace and
// control-word pointers set up by fused_encode_segments.
int resident_encode(const fused::Params &fp, int codec, int mode, int x_dtype, cudaStream_t st) {
  using namespace k1r;
  if (!g_resident_enabled) return CC_ERR_UNSUPPORTED;
  if (fp.C > fused::kMaxC || fp.C % 128 != 0 || fp.G4 <= fused::kCons) return CC_ERR_UNSUPPORTED;  // wide rows only
  Params q{};
  q.x = fp.x;
  q.base = fp.base;
  q.aux = fp.aux;
  q.n = fp.n;
  q.C = fp.C;
  q.G4 = fp.G4;
  // Grid: leave SMs free for the receiver decode that runs beside this K1 on the
  // decode stream (the previous layer's K2, or the peers' at N > 1) — a K1 CTA holds
  // ~all of an SM's shared memory, so the decode can only overlap on SMs K1 leaves
  // empty.  Measured (graph-replayed steps, scripts/exp/k2cap_ab.py and bench.py):
  // P = 1 [4096, 3072] 148 -> 136 CTAs: 76.6 -> 73.5 us per layer-step (K1 alone
  // 60.8 -> 62.4 us); per-rank P = 2 / 4 / 8 at 128 CTAs: 49.0 -> 42.3, 33.7 -> 33.4,
  // 27.1 -> 25.7 us.  CC_K1_RESIDENT_GRID overrides (-1 = every SM).
  int G = fp.G;
  if (g_resident_grid > 0) G = std::min(g_resident_grid, fp.G);
  else if (g_resident_grid == 0 && fp.G >= 128) G = fp.G - (cdiv(fp.n, fp.G) >= 20 ? 12 : 20);
  q.G = (int)std::min<int64_t>(G, fp.n);
  q.R = (int)cdiv(fp.n, q.G);
  q.nseg = fp.nseg;
  q.cw = fp.cw;
  q.cbs = fp.cbs;
  q.bps = fp.C / 128 / fp.nseg;
  q.cb_row = fp.cb_row;
  q.cbytes_seg = fp.cbytes_seg;
  q.body = fp.body;
  q.body_stride = fp.nseg > 1 ? fp.body_stride : 0;
  q.colpart = fp.colpart;
  q.blkpart = fp.blkpart;
  q.recpart = fp.recpart;
  q.record = fp.record;
  q.v = fp.v;
  q.bar1 = fp.bar;
  q.bar2 = fp.bar + 32;
  q.ticket = fp.ticket;
  q.claim = reinterpret_cast<unsigned int *>(fp.ctr);  // control word 0 (left zero on exit)
  q.dyn = 0;
  q.stat = 0;
  q.scale_mode = fp.scale_mode;
  q.timer = fp.timer;
  q.policy = fp.policy;
  if (fp.ctl_in_ws) return CC_ERR_UNSUPPORTED;  // needs the stream's zeroed control slot
  // 24 consumer warps hide latency best when the kernel has the SMs to itself; at the
  // small per-rank shards (<= 14 rows per CTA) the register-capped 12-warp form lets
  // the previous layer's decode share the SMs during the hand-offs (measured per-rank
  // step: [1024, 3072] 44.5 -> 37.0 us, [512, 3072] 40.2 -> 32.9 us, scripts/exp/nq_ab.py)
  int nq = g_resident_nq ? g_resident_nq : (q.R <= 14 ? 2 : 1);
  if (!resident_plan(q, mode, x_dtype, nq)) {
    // the reduced grid's rows do not fit on chip: every SM (more room per row)
    if (q.G >= (int)std::min<int64_t>(fp.G, fp.n) || g_resident_grid > 0) return CC_ERR_UNSUPPORTED;
    q.G = (int)std::min<int64_t>(fp.G, fp.n);
    q.R = (int)cdiv(fp.n, q.G);
    nq = g_resident_nq ? g_resident_nq : (q.R <= 14 ? 2 : 1);
    if (!resident_plan(q, mode, x_dtype, nq)) return CC_ERR_UNSUPPORTED;
  }
  size_t smem = 0;
  {
    // recompute the total from the chosen layout
    smem = (size_t)q.off_red + (size_t)(nq == 2 ? Geo<2>::CW : Geo<1>::CW) * 32 * 8;
  }
#define CC_RESQ(MODE, CODEC, XT) \
  return nq == 2 ? launch<MODE, CODEC, XT, 2>(q, smem, st) : launch<MODE, CODEC, XT, 1>(q, smem, st)
#define CC_RES(MODE, XT)                                \
  do {                                                  \
    if (codec == CC_SIGN1) CC_RESQ(MODE, CC_SIGN1, XT);   \
    if (codec == CC_QUANT2) CC_RESQ(MODE, CC_QUANT2, XT); \
    CC_RESQ(MODE, CC_QUANT4, XT);                       \
  } while (0)
  if (x_dtype == CC_BF16) {
    if (mode == CC_WITH_FEEDBACK) CC_RES(CC_WITH_FEEDBACK, __nv_bfloat16);
    if (mode == CC_NO_FEEDBACK) CC_RES(CC_NO_FEEDBACK, __nv_bfloat16);
    CC_RES(CC_NAIVE, __nv_bfloat16);
  } else {
    if (mode == CC_WITH_FEEDBACK) CC_RES(CC_WITH_FEEDBACK, float);
    if (mode == CC_NO_FEEDBACK) CC_RES(CC_NO_FEEDBACK, float);
    CC_RES(CC_NAIVE, float);
  }
#undef CC_RES
#undef CC_RESQ
}

}  // namespace cc
