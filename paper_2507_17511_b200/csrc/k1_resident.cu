// K1, shard-resident form: ONE persistent cooperative kernel per encode_step that
// keeps the shard's residual t (and, when it fits, its base) in shared memory
// across the grid-wide scale dependency, so every byte of x / base / feedback is
// read from HBM exactly once and every result written once: 18 + b/8 B per
// element, the algorithmic traffic of SURVEY §8(d).
//
// Used when the CTA's rows fit on chip: ceil(n / G) rows x (4 C [+ 4 C]) B next to
// the input ring, e.g. the per-rank shards of patch parallelism at P >= 2
// ([2048, 3072] t-resident, [1024 / 512, 3072] t + base resident) and the
// Ulysses senders ([512, 3072] in 8 column segments).  Larger shards take the
// streaming two-pass kernel (k1_fused_impl.cuh).
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
using fused::kCons;
using fused::kCW;
constexpr int kThreads = kCons + 32;  // 12 consumer warps + 1 producer warp
constexpr int kNB = fused::kNB;       // 128-column blocks per row (24 at C = 3072)
constexpr int kMaxSeg = fused::kMaxSeg;
constexpr int kMaxStages = 8;
constexpr size_t kSmemMax = 227 * 1024;

struct Params {
  const void *x;
  float *base, *aux;
  int64_t n, C;
  int G4, G;
  int R;          // max rows per CTA (ceil(n / G))
  int keep_base;  // base rows resident (else streamed through the ring in both phases)
  int S;          // ring stages
  uint32_t stage_bytes, st_base;                            // ring stage: x at 0, base at st_base
  uint32_t off_t, off_b, off_ring, off_rp, off_rs, off_u;   // shared-memory layout
  uint32_t off_bar, off_red;
  double *colpart, *blkpart, *recpart, *record;  // [G][C], [G][nseg], [G][nseg][2], [nseg][2]
  float *v;                                      // [C]
  uint8_t *body;
  int64_t body_stride, cbytes_seg;
  int nseg, cw, cbs, bps, cb_row;
  unsigned int *bar1, *bar2, *ticket;
  int scale_mode;
};

template <typename XT>
__device__ __forceinline__ void ld_x4(const XT *p, float (&v)[4]) {
  fused::unpack_x(p, v);
}

__device__ __forceinline__ void stcs4(float *p, const float (&v)[4]) {
  __stcs(reinterpret_cast<float4 *>(p), make_float4(v[0], v[1], v[2], v[3]));
}

template <int MODE, int CODEC, typename XT>
__global__ void __launch_bounds__(kThreads, 1) k1_resident(const __grid_constant__ Params p) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int cta = blockIdx.x, G = p.G, S = p.S;
  const int64_t n = p.n, C = p.C;
  const int64_t r0 = (int64_t)cta * n / G, r1 = (int64_t)(cta + 1) * n / G;
  const int nr = (int)(r1 - r0);
  const int nseg = p.nseg;
  constexpr bool kAux = MODE != CC_NAIVE;
  constexpr bool kWB = MODE == CC_WITH_FEEDBACK;
  const bool keep_base = kAux && p.keep_base;
  const bool ring_base = kAux && !p.keep_base;  // base through the ring (phase A if kWB, phase B always)

  float *tS = reinterpret_cast<float *>(smem + p.off_t);   // [R][C]
  float *bS = reinterpret_cast<float *>(smem + p.off_b);   // [R][C] (keep_base)
  uint8_t *ring = smem + p.off_ring;                        // [S][stage_bytes]
  double *rp = reinterpret_cast<double *>(smem + p.off_rp); // [R][kNB]
  double *rs = reinterpret_cast<double *>(smem + p.off_rs); // [R][nseg] row sums
  float *uS = reinterpret_cast<float *>(smem + p.off_u);    // [R][nseg]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + p.off_bar);
  uint64_t *empty = full + kMaxStages;
  double *red = reinterpret_cast<double *>(smem + p.off_red);  // [kCW * 2 * 2 * kMaxSeg]

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCW);
    }
    mbar_fence_init();
  }
  __syncthreads();
  const XT *X = reinterpret_cast<const XT *>(p.x);

  if (warp == kCW) {  // ===================== producer warp =====================
    if (lane == 0) {
      const uint64_t pol_once = l2_policy_evict_first();
      const uint64_t pol_again = l2_policy_evict_last();  // base rows re-read in phase B
      const uint32_t xb = (uint32_t)(C * sizeof(XT)), fb = (uint32_t)(C * 4);
      // phase A: one ring use per row
      for (int k = 0; k < nr; ++k) {
        const int s = k % S;
        if (k >= S) mbar_wait(&empty[s], (uint32_t)((k / S) - 1) & 1u);
        const int64_t row = r0 + k;
        uint8_t *st = ring + (size_t)s * p.stage_bytes;
        uint32_t bytes = xb;
        if (kAux) bytes += fb;
        if (kWB || keep_base) bytes += fb;
        mbar_expect_tx(&full[s], bytes);
        bulk_g2s(st, X + row * C, xb, &full[s], pol_once);
        if (kAux) bulk_g2s(tS + (size_t)k * C, p.aux + row * C, fb, &full[s], pol_once);
        if (keep_base) {
          bulk_g2s(bS + (size_t)k * C, p.base + row * C, fb, &full[s], pol_once);
        } else if (kWB) {
          bulk_g2s(st + p.st_base, p.base + row * C, fb, &full[s], pol_again);
        }
      }
      // phase B: base rows through the ring (uses nr .. 2 nr - 1), loaded while the
      // consumers wait on the hand-offs
      if (ring_base) {
        for (int k = 0; k < nr; ++k) {
          const int u = nr + k, s = u % S;
          if (u >= S) mbar_wait(&empty[s], (uint32_t)((u / S) - 1) & 1u);
          mbar_expect_tx(&full[s], fb);
          bulk_g2s(ring + (size_t)s * p.stage_bytes, p.base + (r0 + k) * C, fb, &full[s], pol_once);
        }
      }
    }
    return;
  }

  // ===================== consumer warps =====================
  // column quads: thread tid owns quads tid and tid + kCons (columns 4 q .. 4 q + 3)
  bool qact[2];
  int qcol[2], qblk[2], qseg[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    const int qd = tid + j * kCons;
    qact[j] = qd < p.G4;
    qcol[j] = 4 * qd;
    qblk[j] = j * kCW + warp;  // 128-column block of the quad
    qseg[j] = nseg == 1 ? 0 : min(qblk[j] / p.bps, nseg - 1);
  }
  double cs[2][4];
#pragma unroll
  for (int j = 0; j < 2; ++j) cs[j][0] = cs[j][1] = cs[j][2] = cs[j][3] = 0.0;

  // ---------------- phase A ----------------
  for (int k = 0; k < nr; ++k) {
    const int s = k % S;
    mbar_wait(&full[s], (uint32_t)(k / S) & 1u);
    const uint8_t *st = ring + (size_t)s * p.stage_bytes;
    const XT *xs = reinterpret_cast<const XT *>(st);
    float *trow = tS + (size_t)k * C;
    const float *brow = keep_base ? bS + (size_t)k * C : reinterpret_cast<const float *>(st + p.st_base);
    double rsum[2] = {0.0, 0.0};
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      if (!qact[j]) continue;
      const int o = qcol[j];
      float xx[4], bb[4] = {0.f, 0.f, 0.f, 0.f}, aa[4] = {0.f, 0.f, 0.f, 0.f}, t[4];
      ld_x4(xs + o, xx);
      if constexpr (kWB) fused::unpack_f(brow + o, bb);
      if constexpr (kAux) fused::unpack_f(trow + o, aa);
      double a[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        t[q] = target_of<MODE>(xx[q], bb[q], aa[q]);
        a[q] = fabs((double)t[q]);
        cs[j][q] += a[q];
      }
      rsum[j] = ((a[0] + a[1]) + a[2]) + a[3];
      *reinterpret_cast<float4 *>(trow + o) = make_float4(t[0], t[1], t[2], t[3]);
      if constexpr (MODE == CC_NO_FEEDBACK) stcs4(p.aux + (r0 + k) * C + o, xx);  // ref' = a* (pl:113)
    }
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double v = warp_sum(rsum[j]);
      if (lane == 0 && qblk[j] < kNB) rp[(size_t)k * kNB + qblk[j]] = v;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
  // column partials of this CTA
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    if (!qact[j]) continue;
    double *cp = p.colpart + (int64_t)cta * C + qcol[j];
    cp[0] = cs[j][0]; cp[1] = cs[j][1]; cp[2] = cs[j][2]; cp[3] = cs[j][3];
  }
  fused::named_sync(1, kCons);
  // row sums per segment (blocks of the segment in order), then CTA totals
  for (int i = tid; i < nr * nseg; i += kCons) {
    const int k = i / nseg, d = i % nseg;
    double acc = 0.0;
    for (int b = 0; b < p.bps; ++b) acc += rp[(size_t)k * kNB + d * p.bps + b];
    rs[i] = acc;
  }
  fused::named_sync(1, kCons);
  if (tid < nseg) {
    double tot = 0.0;
    for (int k = 0; k < nr; ++k) tot += rs[k * nseg + tid];
    p.blkpart[(size_t)cta * nseg + tid] = tot;
  }
  // ---- hand-off 1 ----
  fused::named_sync(1, kCons);
  if (tid == 0) {
    fused::arrive_release(p.bar1);
    fused::spin_until(p.bar1, (unsigned)G);
  }
  fused::named_sync(1, kCons);

  // ---------------- phase F ----------------
  {
    double *wpart = red;  // [kCW][32]
    for (int64_t grp32 = cta; grp32 * 32 < C; grp32 += G) {
      const int64_t j = grp32 * 32 + lane;
      double acc = 0.0;
      if (j < C) {
        constexpr int kB = 16;
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
      fused::named_sync(1, kCons);
      if (warp == 0 && j < C) {
        double sacc = 0.0;
        for (int w = 0; w < kCW; ++w) sacc += wpart[w * 32 + lane];
        float v = (float)(sacc / (double)n);  // colmean (cx:148)
        if (p.scale_mode == CC_SCALE_PER_TOKEN) v = 1.0f;
        p.v[j] = v;
        const int d = (int)(j / p.cw);
        store_f32_bytes(p.body + d * p.body_stride + p.cbytes_seg + 4 * n + 4 * (j - (int64_t)d * p.cw), v);
      }
      fused::named_sync(1, kCons);
    }
  }
  // v published: arrive now, compute g / u of the own rows while the others finish
  fused::named_sync(1, kCons);
  if (tid == 0) fused::arrive_release(p.bar2);
  {
    __shared__ double gseg[kMaxSeg];
    for (int d = warp; d < nseg; d += kCW) {  // g_d = mean |t| over segment d, same order in every CTA
      double part = 0.0;
      for (int i = lane; i < G; i += 32) part += __ldcg(p.blkpart + (size_t)i * nseg + d);
      part = warp_sum(part);
      if (lane == 0) gseg[d] = part / ((double)n * (double)p.cw);
    }
    fused::named_sync(1, kCons);
    for (int i = tid; i < nr * nseg; i += kCons) {
      const int k = i / nseg, d = i % nseg;
      const double g = gseg[d], rsum = rs[i];
      float u;
      if (p.scale_mode == CC_SCALE_PER_CHANNEL) u = 1.0f;
      else if (p.scale_mode == CC_SCALE_PER_TOKEN) u = (float)(rsum / (double)p.cw);
      else if (g == 0.0) u = 1.0f;  // all-zero segment (cx:143-146)
      else u = (float)fmax((rsum / (double)p.cw) / g, kRowScaleFloor);  // cx:147
      uS[i] = u;
      store_f32_bytes(p.body + d * p.body_stride + p.cbytes_seg + 4 * (r0 + k), u);
    }
  }
  // ---- hand-off 2: every CTA's v ----
  if (tid == 0) fused::spin_until(p.bar2, (unsigned)G);
  fused::named_sync(1, kCons);

  // ---------------- phase B ----------------
  ColConst cc[2];
#pragma unroll
  for (int j = 0; j < 2; ++j) {
    cc[j].ok = true;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float v = qact[j] ? __ldcg(p.v + qcol[j] + q) : 1.0f;
      cc[j].v[q] = v;
      cc[j].vhi[q] = __fmul_ru(__fmul_ru(v, 1.25f), 1.00000095367431640625f);  // (1 + 2^-20)
      cc[j].vlo[q] = __fmul_rd(__fmul_rd(v, 1.25f), 0.99999904632568359375f);  // (1 - 2^-20)
      cc[j].ok = cc[j].ok && fused::scale_in_range(fabsf(v));
    }
  }
  constexpr int bits = CODEC == CC_SIGN1 ? 1 : (CODEC == CC_QUANT2 ? 2 : 4);
  double err[2] = {0.0, 0.0}, tsq[2] = {0.0, 0.0};
  for (int k = 0; k < nr; ++k) {
    const int64_t row = r0 + k;
    const float *brow = bS + (size_t)k * C;
    int s = 0;
    if (ring_base) {
      const int u = nr + k;
      s = u % S;
      mbar_wait(&full[s], (uint32_t)(u / S) & 1u);
      brow = reinterpret_cast<const float *>(ring + (size_t)s * p.stage_bytes);
    }
    const float *trow = tS + (size_t)k * C;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int o = qcol[j];
      float t[4], bb[4] = {0.f, 0.f, 0.f, 0.f}, d[4], e[4];
      if (qact[j]) {
        fused::unpack_f(trow + o, t);
        if constexpr (kAux) fused::unpack_f(brow + o, bb);
      } else {
        t[0] = t[1] = t[2] = t[3] = 0.f;
      }
      const float uf = uS[k * nseg + qseg[j]];
      const uint32_t packed = fused::quantize4<CODEC>(t, uf, fused::scale_in_range(fabsf(uf)), cc[j], d);
#pragma unroll
      for (int q = 0; q < 4; ++q) e[q] = __fsub_rn(t[q], d[q]);
      if (qact[j]) {
        fused::record4(t, e, err[j], tsq[j]);
        float nb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) nb[q] = MODE == CC_NAIVE ? d[q] : __fadd_rn(bb[q], d[q]);
        stcs4(p.base + row * C + o, nb);
        if constexpr (kWB) stcs4(p.aux + row * C + o, e);
      }
      // codes: segment d's code row lives in its own body
      const int sg = qseg[j];
      uint8_t *crow = p.body + sg * p.body_stride + row * p.cbs;
      const int cl = o - sg * p.cw;  // column inside the segment
      if constexpr (CODEC == CC_SIGN1) {
        const uint32_t other = __shfl_down_sync(0xffffffffu, packed, 1);
        if (qact[j] && (lane & 1) == 0) crow[cl >> 3] = (uint8_t)(packed | (other << 4));
      } else if constexpr (CODEC == CC_QUANT2) {
        if (qact[j]) crow[cl >> 2] = (uint8_t)packed;
      } else {
        if (qact[j]) *reinterpret_cast<uint16_t *>(crow + (cl >> 1)) = (uint16_t)packed;
      }
    }
    if (ring_base) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  (void)bits;

  // ---------------- StepRecord ----------------
  {
    __shared__ unsigned last;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const double a = warp_sum(err[j]), b = warp_sum(tsq[j]);
      if (lane == 0) {
        red[(warp * 2 + j) * 2] = a;
        red[(warp * 2 + j) * 2 + 1] = b;
      }
    }
    fused::named_sync(1, kCons);
    if (tid < nseg) {
      double a = 0.0, b = 0.0;
      for (int w = 0; w < kCW; ++w)
        for (int j = 0; j < 2; ++j) {
          const int blk = j * kCW + w;
          if (nseg == 1 || (blk < kNB && blk / p.bps == tid)) {
            a += red[(w * 2 + j) * 2];
            b += red[(w * 2 + j) * 2 + 1];
          }
        }
      p.recpart[((size_t)cta * nseg + tid) * 2] = a;
      p.recpart[((size_t)cta * nseg + tid) * 2 + 1] = b;
    }
    fused::named_sync(1, kCons);
    if (tid == 0) last = fused::atom_add_acq_rel(p.ticket) == (unsigned)G - 1;
    fused::named_sync(1, kCons);
    if (last) {
      double vals[2 * kMaxSeg];
#pragma unroll
      for (int q = 0; q < 2 * kMaxSeg; ++q)
        vals[q] = (q < 2 * nseg && tid < G) ? __ldcg(p.recpart + (size_t)tid * nseg * 2 + q) : 0.0;
      fused::named_sync(1, kCons);
#pragma unroll
      for (int q = 0; q < 2 * kMaxSeg; ++q) {
        if (q >= 2 * nseg) break;
        const double v = warp_sum(vals[q]);
        if (lane == 0) red[warp * 2 * kMaxSeg + q] = v;
      }
      fused::named_sync(1, kCons);
      if (tid < 2 * nseg) {
        double a = 0.0;
        for (int w = 0; w < kCW; ++w) a += red[w * 2 * kMaxSeg + tid];
        p.record[tid] = a;
      }
      if (tid == 0) {  // every CTA is past both hand-offs: leave the control words zeroed
        *p.ticket = 0u;
        *p.bar1 = 0u;
        *p.bar2 = 0u;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static bool g_resident_enabled = true;
std::atomic<int64_t> g_resident_launches{0};

template <int MODE, int CODEC, typename XT>
static int launch(Params &p, size_t smem, cudaStream_t st) {
  auto kern = k1_resident<MODE, CODEC, XT>;
  static int smem_set = 0;
  if ((int)smem > smem_set) {
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
      return cuda_status("k1_resident attr");
    smem_set = (int)smem;
  }
  void *args[] = {&p};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void *)kern, dim3(p.G), dim3(kThreads), args, smem, st);
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

// Shared-memory plan for a shard; false when the CTA's rows do not fit.
static bool resident_plan(k1r::Params &q, int mode, int x_dtype) {
  using namespace k1r;
  const int64_t C = q.C;
  const size_t xb = (size_t)C * (x_dtype == CC_BF16 ? 2 : 4), fb = (size_t)C * 4;
  const bool aux = mode != CC_NAIVE;
  auto layout = [&](int keep_base, int S) -> size_t {
    const size_t R = (size_t)q.R;
    size_t off = 0;
    auto take = [&](size_t b) {
      const size_t o = off;
      off = align_up(off + b, 128);
      return (uint32_t)o;
    };
    q.keep_base = keep_base;
    q.S = S;
    // ring stage: x, plus base when base is streamed (phase A for feedback mode;
    // phase B reuses stage starts for base rows)
    const bool ring_base = aux && !keep_base;
    q.st_base = (uint32_t)align_up(xb, 128);
    const size_t stage_a = (mode == CC_WITH_FEEDBACK && ring_base) ? q.st_base + fb : xb;
    q.stage_bytes = (uint32_t)align_up(std::max(stage_a, ring_base ? fb : (size_t)0), 128);
    q.off_t = take(R * fb);
    q.off_b = take(keep_base ? R * fb : 0);
    q.off_ring = take((size_t)S * q.stage_bytes);
    q.off_rp = take(R * kNB * 8);
    q.off_rs = take(R * q.nseg * 8);
    q.off_u = take(R * q.nseg * 4);
    q.off_bar = take(2 * kMaxStages * 8);
    q.off_red = take((size_t)kCW * 32 * 8);
    return off + 16 * 8 + 64;  // + static shared (gseg, last)
  };
  for (int keep_base : {aux ? 1 : 0, 0}) {
    for (int S = kMaxStages; S >= 2; --S) {
      const size_t bytes = layout(keep_base, S);
      if (bytes <= kSmemMax - 1024) return true;
    }
    if (!aux) break;
  }
  return false;
}

// Try the shard-resident K1; CC_ERR_UNSUPPORTED when the shard does not fit (the
// caller then launches the streaming kernel).  `fp` carries the workspace and
// control-word pointers set up by fused_encode_segments.
int resident_encode(const fused::Params &fp, int codec, int mode, int x_dtype, cudaStream_t st) {
  using namespace k1r;
  if (!g_resident_enabled) return CC_ERR_UNSUPPORTED;
  if (fp.C > fused::kMaxC || fp.C % 128 != 0 || fp.G4 <= kCons) return CC_ERR_UNSUPPORTED;  // full-width rows only
  Params q{};
  q.x = fp.x;
  q.base = fp.base;
  q.aux = fp.aux;
  q.n = fp.n;
  q.C = fp.C;
  q.G4 = fp.G4;
  q.G = (int)std::min<int64_t>(fp.G, fp.n);
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
  q.scale_mode = fp.scale_mode;
  if (fp.ctl_in_ws) return CC_ERR_UNSUPPORTED;  // needs the stream's zeroed control slot
  if (!resident_plan(q, mode, x_dtype)) return CC_ERR_UNSUPPORTED;
  size_t smem = 0;
  {
    // recompute the total from the chosen layout
    smem = (size_t)q.off_red + (size_t)kCW * 32 * 8;
  }
#define CC_RES(MODE, XT)                                                                     \
  do {                                                                                       \
    if (codec == CC_SIGN1) return launch<MODE, CC_SIGN1, XT>(q, smem, st);                   \
    if (codec == CC_QUANT2) return launch<MODE, CC_QUANT2, XT>(q, smem, st);                 \
    return launch<MODE, CC_QUANT4, XT>(q, smem, st);                                         \
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
}

}  // namespace cc
