// K1, host side: debug knobs, workspace layout, parameter set-up and the
// plain-step (one segment) instantiations.  The kernel is in k1_fused_impl.cuh.
#include "k1_fused_impl.cuh"

namespace cc {

int resident_encode(const fused::Params &fp, int codec, int mode, int x_dtype, cudaStream_t st);

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static int g_fused_stop = 0;
static int g_fused_policy = 0;
int g_fused_si = 0, g_fused_so = 0, g_fused_sa = 0;
static int g_fused_ra = 0;
void set_fused_phase_a(int rows_per_tile, int stages) {
  g_fused_ra = rows_per_tile;
  g_fused_sa = stages;
}
static int g_fused_tail_mult = 0, g_fused_tail_keep = 0;
void set_fused_tail(int mult, int keep) {
  g_fused_tail_mult = mult;
  g_fused_tail_keep = keep;
}
void set_fused_rings(int si, int so) {
  g_fused_si = si;
  g_fused_so = so;
}
static unsigned long long *g_fused_timer = nullptr;
void set_fused_policy(int v) { g_fused_policy = v; }
void set_fused_stop(int v) { g_fused_stop = v; }
void set_fused_timer(void *buf) { g_fused_timer = reinterpret_cast<unsigned long long *>(buf); }

bool fused_supported(int64_t n, int64_t C, const void *x, int x_dtype, const float *base, const float *aux,
                     const uint8_t *body) {
  (void)n;
  (void)x_dtype;
  if (C % 128 != 0 || C > fused::kMaxC) return false;
  if (!aligned(x, 16) || !aligned(base, 16) || (aux && !aligned(aux, 16)) || !aligned(body, 16)) return false;
  return true;
}

// workspace layout (any segment count up to kMaxSeg)
static size_t fused_ws_layout(int64_t n, int64_t C, int G, int nseg, uint8_t *w, fused::Params *p) {
  size_t off = 0;
  const int64_t un = (n + 3) & ~int64_t(3);
  auto take = [&](size_t bytes) {
    uint8_t *q = w ? w + off : nullptr;
    off = align_up(off + bytes, 256);
    return q;
  };
  uint8_t *colpart = take(sizeof(double) * (size_t)G * C);
  uint8_t *rowpart = take(sizeof(double) * nseg * n);
  uint8_t *blkpart = take(sizeof(double) * (size_t)G * nseg);
  uint8_t *recpart = take(sizeof(double) * 2 * (size_t)G * nseg);
  uint8_t *u = take(sizeof(float) * nseg * un);
  uint8_t *v = take(sizeof(float) * C);
  uint8_t *ctl = take(512);
  if (p) {
    p->colpart = reinterpret_cast<double *>(colpart);
    p->rowpart = reinterpret_cast<double *>(rowpart);
    p->blkpart = reinterpret_cast<double *>(blkpart);
    p->recpart = reinterpret_cast<double *>(recpart);
    p->u = reinterpret_cast<float *>(u);
    p->v = reinterpret_cast<float *>(v);
    p->un = un;
    p->ctr = reinterpret_cast<unsigned long long *>(ctl);
  }
  return off;
}

int64_t fused_workspace_bytes(int64_t n, int64_t C) {
  return (int64_t)fused_ws_layout(n, C, fused::kCons, fused::kMaxSeg, nullptr, nullptr);
}

// nseg column segments of width C / nseg (see Params): segment d is an independent
// encode_step channel over columns [d cw, (d+1) cw) with its body at body + d *
// body_stride and its record at record + 2 d.  nseg = 1: the plain encode_step.
bool fused_segments_supported(int64_t n, int64_t C, int nseg, int64_t body_stride, int codec) {
  using namespace fused;
  if (nseg < 1 || nseg > kMaxSeg || C % nseg != 0) return false;
  const int64_t cw = C / nseg;
  if (nseg > 1) {
    const int bits = codec == CC_SIGN1 ? 1 : (codec == CC_QUANT2 ? 2 : 4);
    if (cw % 128 != 0 || (cw * bits / 8) % 16 != 0 || body_stride % 16 != 0) return false;
    const int64_t body = cdiv(n * cw * bits, 8) + 4 * (n + cw);
    if (body_stride < body) return false;
    // rows per phase-A tile x segments must fit one warp (finish_rows lanes)
    const int groups = C / 4 > kCons ? 1 : kCons / (int)(C / 4);
    if (2 * groups * nseg > 32) return false;
  }
  return true;
}

int fused_encode_segments(int codec, int mode, int scale_mode, int64_t n, int64_t C, int nseg, const void *x,
                          int x_dtype, float *base, float *aux, uint8_t *body, int64_t body_stride, void *ws,
                          int64_t ws_bytes, double *record, cudaStream_t st) {
  using namespace fused;
  Params p{};
  p.x = x;
  p.base = base;
  p.aux = aux;
  p.n = n;
  p.C = C;
  p.G4 = (int)(C / 4);
  const int Q = p.G4 > kCons ? 2 : 1;
  p.groups = Q == 2 ? 1 : kCons / p.G4;
  p.wpg = Q == 2 ? kCW : p.G4 / 32;
  int G = std::min(sm_count(), kCons);  // the record / scale reductions assume G <= kCons
  // rows per tile: a multiple of the row groups; two per group when each CTA has plenty of rows
  const int64_t rows_per_cta = cdiv(n, G);
  constexpr double kL2KeepBytes = 40e6;
  p.R = p.groups * ((Q == 2 || rows_per_cta >= 16 * p.groups) ? 2 : 1);
  if (g_fused_ra > 0) p.R = p.groups * g_fused_ra;
  p.G = G;
  p.nTiles = cdiv(n, p.R);
  {
    const int pf = (g_fused_policy >> 8) & 15;  // debug override: 1..10 -> tenths, 15 -> none
    const double tile_bytes = (double)p.R * C * (x_dtype == CC_BF16 ? 10.0 : 12.0);
    const long long keep = (long long)(kL2KeepBytes / tile_bytes);
    p.early_tiles = pf == 15 ? 0 : pf ? p.nTiles * pf / 10 : std::max(0LL, (long long)p.nTiles - keep);
  }
  p.scale_mode = scale_mode;
  p.stop_after = g_fused_stop;
  p.tail_mult = g_fused_tail_mult > 0 ? g_fused_tail_mult : g_fused_tail_mult < 0 ? 0 : 2;
  p.tail_keep = g_fused_tail_keep > 0 ? g_fused_tail_keep : 2;
  p.static_sched = (g_fused_policy & 16384) ? 1 : (g_fused_policy & 32768) ? 2 : 0;
  p.timer = g_fused_timer;
  p.policy = g_fused_policy;
  const int bits = codec == CC_SIGN1 ? 1 : (codec == CC_QUANT2 ? 2 : 4);
  p.cb_row = (int)(C * bits / 8);
  p.nseg = nseg;
  p.cw = (int)(C / nseg);
  p.cbs = (int)(p.cw * bits / 8);
  // 128-column blocks per segment; with one segment phase A keeps one partial per warp
  p.bps = nseg == 1 ? (Q == 2 ? kCW : (int)(C / 128)) : p.cw / 128;
  p.cbytes_seg = cdiv(n * p.cw * bits, 8);
  p.body = body;
  p.body_stride = nseg > 1 ? body_stride : 0;
  p.record = record;
  const size_t off = fused_ws_layout(n, C, G, nseg, reinterpret_cast<uint8_t *>(ws), &p);
  uint8_t *ctl_ws = reinterpret_cast<uint8_t *>(p.ctr);
  // control words, one 128-byte line each (pollers and atomics never share a line):
  // ctr0 @0, ctr1 @128, bar1 @256 (+ ticket @260), bar2 @384.  The stream's
  // library-owned slot (kept zero by every launch), or the workspace + a memset
  // when there is none / a debug stop exits early
  uint8_t *ctl = (g_fused_stop == 0 && !(g_fused_policy & 32)) ? stream_control_block(st) : nullptr;
  p.ctl_in_ws = ctl == nullptr;
  if (!ctl) ctl = ctl_ws;
  p.ctr = reinterpret_cast<unsigned long long *>(ctl);
  p.ticket = reinterpret_cast<unsigned int *>(ctl + 260);
  p.bar = reinterpret_cast<unsigned int *>(ctl + 256);
  if ((int64_t)off > ws_bytes) {
    set_error("fused workspace too small");
    return CC_ERR_ARG;
  }
  {  // shards whose rows fit on chip: the single-pass resident kernel (k1_resident.cu)
    const int rc = resident_encode(p, codec, mode, x_dtype, st);
    if (rc != CC_ERR_UNSUPPORTED) return rc;
  }
  if (nseg > 1) return fused_dispatch_seg(p, codec, mode, x_dtype, Q, st);
#define CC_FUSED_Q(MODE, CODEC, XT) \
  return Q == 2 ? launch_fused<MODE, CODEC, XT, 2, false>(p, st) : launch_fused<MODE, CODEC, XT, 1, false>(p, st)
#define CC_FUSED(MODE, XT)                                          \
  do {                                                              \
    if (codec == CC_SIGN1) CC_FUSED_Q(MODE, CC_SIGN1, XT);          \
    if (codec == CC_QUANT2) CC_FUSED_Q(MODE, CC_QUANT2, XT);        \
    CC_FUSED_Q(MODE, CC_QUANT4, XT);                                \
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
#undef CC_FUSED_Q
}

}  // namespace cc

namespace cc {
int fused_encode(int codec, int mode, int scale_mode, int64_t n, int64_t C, const void *x, int x_dtype, float *base,
                 float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st) {
  return fused_encode_segments(codec, mode, scale_mode, n, C, 1, x, x_dtype, base, aux, body, 0, ws, ws_bytes, record,
                               st);
}
}  // namespace cc
