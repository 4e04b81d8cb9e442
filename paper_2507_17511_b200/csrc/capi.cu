// extern "C" entry points (include/compactcomm.h).  Host-side argument and
// shape validation happens here, before any launch, so a rejected call never
// touches device state (reference pipeline.py:146-151 semantics).
#include <cuda_runtime.h>

#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <unordered_map>

#include "../../include/compactcomm.h"
#include "cc_debug.h"
#include "cc_internal.h"

namespace cc {

std::atomic<int64_t> g_launches{0};
static thread_local std::string g_err;

void set_error(const std::string &msg) { g_err = msg; }

int cuda_status(const char *where) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error(std::string(where) + ": " + cudaGetErrorString(e));
    return CC_ERR_CUDA;
  }
  return CC_OK;
}

int sm_count() {
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) dev = 0;
  if (cached[dev] == 0) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cached[dev] = v;
  }
  return cached[dev];
}

// Library-owned control words (tile counters, tickets) of the persistent
// kernels: one zero-initialised 512-byte slot per (device, stream).  Every launch
// leaves its slot zeroed on exit, so no per-launch memset node is needed;
// launches on one stream are ordered, launches on different streams use
// different slots.  Returns null (caller falls back to a memset'd workspace
// word) if the pool cannot be created now, e.g. during a stream capture.
static int g_pdl = [] {  // default off; CC_PDL=1 in the environment turns it on (tests / benchmarks)
  const char *e = std::getenv("CC_PDL");
  return e && e[0] == '1' ? 1 : 0;
}();
int pdl_enabled() { return g_pdl; }

uint8_t *stream_control_block(cudaStream_t st) {
  constexpr int kSlots = 1024, kSlotBytes = 512;
  struct Pool {
    uint8_t *base = nullptr;
    int used = 0;
    std::unordered_map<cudaStream_t, int> slot;
  };
  static std::mutex mu;
  static Pool pools[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  Pool &P = pools[dev];
  if (!P.base) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    void *b = nullptr;
    if (cudaMalloc(&b, (size_t)kSlots * kSlotBytes) != cudaSuccess || cudaMemset(b, 0, (size_t)kSlots * kSlotBytes) !=
                                                                           cudaSuccess) {
      cudaGetLastError();
      if (b) cudaFree(b);
      return nullptr;
    }
    P.base = static_cast<uint8_t *>(b);
  }
  auto it = P.slot.find(st);
  if (it != P.slot.end()) return P.base + (size_t)it->second * kSlotBytes;
  if (P.used == kSlots) return nullptr;
  P.slot.emplace(st, P.used);
  return P.base + (size_t)(P.used++) * kSlotBytes;
}

// Library-owned zero-initialised scratch slabs of the persistent kernels that need
// more than a control slot (top-k histograms): one 48 KB slab per (device,
// stream) from a pool allocated on first use, left zeroed by every launch.  A
// stream first seen during a capture still gets a slab as long as the pool
// exists; null when it cannot be created (first use inside a capture).
uint8_t *stream_zero_slab(cudaStream_t st, size_t bytes) {
  constexpr size_t kSlabBytes = 48 * 1024;
  constexpr int kSlabs = 128;
  if (bytes > kSlabBytes) return nullptr;
  struct Pool {
    uint8_t *base = nullptr;
    int used = 0;
    std::unordered_map<cudaStream_t, int> slot;
  };
  static std::mutex mu;
  static Pool pools[64];
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  Pool &P = pools[dev];
  if (!P.base) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
      cudaGetLastError();
      return nullptr;
    }
    void *b = nullptr;
    if (cudaMalloc(&b, kSlabBytes * kSlabs) != cudaSuccess || cudaMemset(b, 0, kSlabBytes * kSlabs) != cudaSuccess) {
      cudaGetLastError();
      if (b) cudaFree(b);
      return nullptr;
    }
    P.base = static_cast<uint8_t *>(b);
  }
  auto it = P.slot.find(st);
  if (it != P.slot.end()) return P.base + (size_t)it->second * kSlabBytes;
  if (P.used == kSlabs) return nullptr;
  P.slot.emplace(st, P.used);
  return P.base + (size_t)(P.used++) * kSlabBytes;
}

int64_t topk_workspace_bytes(int64_t n, int64_t C, int64_t k);
void set_topk_resident_enabled(int on);
void set_topk_timer(void *buf);
void set_orth1_stamps(void *buf);
void set_orth_cluster(int on);
void set_lowrank_fused(int on);
int64_t lowrank_fused_launches();
void set_lowrank_fused_stamps(void *buf);
namespace rng {
void set_gauss_stamps(void *buf);
}
int64_t topk_resident_launches();
int topk_encode(int64_t n, int64_t C, int64_t k, const float *t, uint8_t *body, float *decoded, void *ws,
                int64_t ws_bytes, cudaStream_t st);
int topk_encode_step(int mode, int64_t n, int64_t C, int64_t k, const void *x, int x_dtype, float *base, float *aux,
                     uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st);
int topk_decode(int count, const int64_t *rows, int64_t C, int64_t k, const uint8_t *const *bodies, int accumulate,
                float *const *bases, cudaStream_t st);
int64_t lowrank_workspace_bytes(int64_t n, int64_t C, int64_t r);
int64_t lowrank_step_workspace_bytes(int64_t n, int64_t C, int64_t r);
int lowrank_encode_step(int mode, int64_t n, int64_t C, int64_t r, int iters, int int4, const void *x, int x_dtype,
                        float *base, float *aux, const float *q0_in, uint32_t *key, int nwords, int step_word,
                        uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st);
int lowrank_encode(int int4, int64_t n, int64_t C, int64_t r, int iters, const float *t, const float *q0,
                   uint8_t *body, float *decoded, void *ws, int64_t ws_bytes, cudaStream_t st);
int lowrank_decode(int int4, int count, const int64_t *rows, int64_t C, int64_t r, const uint8_t *const *bodies,
                   int accumulate, float *const *bases, cudaStream_t st);
int64_t nm_body_bytes(int64_t rows, int64_t C, int n, int m);
int64_t nm_workspace_bytes(int64_t rows, int64_t C, int n, int m);
int nm_encode(int64_t rows, int64_t C, int n, int m, const float *t, uint8_t *body, float *decoded, void *ws,
              int64_t ws_bytes, cudaStream_t st);
int nm_encode_step(int mode, int64_t rows, int64_t C, int n, int m, const void *x, int x_dtype, float *base,
                   float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record, cudaStream_t st);
int nm_decode(int count, const int64_t *rows, int64_t C, int n, int m, const uint8_t *const *bodies, int accumulate,
              float *const *bases, cudaStream_t st);
void set_quant_path(int v);
bool fused_supported(int64_t n, int64_t C, const void *x, int x_dtype, const float *base, const float *aux,
                     const uint8_t *body);
bool fused_segments_supported(int64_t n, int64_t C, int nseg, int64_t body_stride, int codec);
int fused_encode_segments(int codec, int mode, int scale_mode, int64_t n, int64_t C, int nseg, const void *x,
                          int x_dtype, float *base, float *aux, uint8_t *body, int64_t body_stride, void *ws,
                          int64_t ws_bytes, double *record, cudaStream_t st);
void set_fused_stop(int v);
void set_fused_timer(void *buf);
void set_fused_policy(int v);
void set_fused_rings(int si, int so);
void set_fused_tail(int mult, int keep);
void set_fused_phase_a(int rows_per_tile, int stages);
void set_lowrank_backend(int v);
void set_tc_tma(int v, int waves);
void set_resident_enabled(int on);
void set_resident_nq(int nq);
int64_t resident_launches();
int residual_target(int mode, int64_t n, int64_t C, const void *x, int x_dtype, const float *base, const float *aux,
                    float *t, cudaStream_t st);
int apply_decoded(int mode, int64_t n, int64_t C, const void *x, int x_dtype, const float *t, const float *dec,
                  float *base, float *aux, double *record, void *ws, int64_t ws_bytes, cudaStream_t st);

int64_t gaussian_workspace_bytes(int64_t rows, int64_t cols);
int gaussian_keyed(int64_t rows, int64_t cols, uint32_t *key, int nwords, int step_word, float *out, void *ws,
                   int64_t ws_bytes, cudaStream_t st);
}  // namespace cc

using namespace cc;

static bool quant_codec(int c) { return c == CC_SIGN1 || c == CC_QUANT2 || c == CC_QUANT4; }
static bool nm_split(int64_t param, int *n, int *m) {
  *n = (int)(param >> 16);
  *m = (int)(param & 0xffff);
  return param >= 0 && (param >> 32) == 0 && *n >= 1 && *n <= *m;
}
static bool valid_mode(int m) { return m == CC_NAIVE || m == CC_NO_FEEDBACK || m == CC_WITH_FEEDBACK; }

extern "C" {

CC_API const char *cc_last_error(void) { return g_err.c_str(); }
CC_API int cc_version(void) { return 1; }
CC_API int64_t cc_launch_count(void) { return g_launches.load(); }
CC_API void cc_set_quant_path(int path) { set_quant_path(path); }
CC_API void cc_debug_fused_stop(int phase) { set_fused_stop(phase); }
CC_API void cc_debug_fused_timer(void *dev_buf) { set_fused_timer(dev_buf); }
CC_API void cc_debug_fused_policy(int policy) { set_fused_policy(policy); }
CC_API void cc_debug_fused_rings(int s_in, int s_out) { set_fused_rings(s_in, s_out); }
CC_API void cc_debug_fused_tail(int mult, int keep) { set_fused_tail(mult, keep); }
CC_API void cc_set_pdl(int enable) { g_pdl = enable ? 1 : 0; }
CC_API void cc_debug_fused_phase_a(int rows_per_group, int stages) { set_fused_phase_a(rows_per_group, stages); }
CC_API void cc_set_lowrank_backend(int backend) { set_lowrank_backend(backend); }
CC_API void cc_debug_lowrank_tma(int enable, int waves) { set_tc_tma(enable, waves); }
CC_API void cc_debug_k1_resident(int enable) { set_resident_enabled(enable); }
CC_API int64_t cc_debug_k1_resident_count(void) { return resident_launches(); }
CC_API void cc_debug_k1_resident_nq(int nq) { set_resident_nq(nq); }
CC_API void cc_debug_topk_resident(int enable) { set_topk_resident_enabled(enable); }
CC_API int64_t cc_debug_topk_resident_count(void) { return topk_resident_launches(); }
CC_API void cc_debug_topk_timer(void *dev_buf) { set_topk_timer(dev_buf); }
CC_API void cc_debug_orth_stamps(void *dev_buf) { set_orth1_stamps(dev_buf); }
CC_API void cc_debug_orth_cluster(int enable) { set_orth_cluster(enable); }
CC_API void cc_debug_lowrank_fused(int enable) { set_lowrank_fused(enable); }
CC_API int64_t cc_debug_lowrank_fused_count(void) { return lowrank_fused_launches(); }
CC_API void cc_debug_lowrank_fused_stamps(void *dev_buf) { set_lowrank_fused_stamps(dev_buf); }
CC_API void cc_debug_gauss_stamps(void *dev_buf) { rng::set_gauss_stamps(dev_buf); }

CC_API int64_t cc_topk_count(int64_t rows, int64_t cols, double keep_fraction) {
  if (rows < 1 || cols < 1 || !(keep_fraction > 0.0 && keep_fraction <= 1.0)) return CC_ERR_ARG;
  const int64_t size = rows * cols;
  // k = min(size, int(np.ceil(keep_fraction * size)))  (cx:451) — f64 product as numpy
  const double prod = keep_fraction * (double)size;
  const int64_t k = (int64_t)std::ceil(prod);
  return k < size ? k : size;
}

CC_API int64_t cc_body_bytes(int codec, int64_t rows, int64_t cols, int64_t param) {
  if (rows < 1 || cols < 1) return CC_ERR_SHAPE;
  const int64_t s = rows * cols;
  switch (codec) {
    case CC_RAW: return 4 * s;
    case CC_SIGN1: return (s + 7) / 8 + 4 * (rows + cols);
    case CC_QUANT2: return (2 * s + 7) / 8 + 4 * (rows + cols);
    case CC_QUANT4: return (4 * s + 7) / 8 + 4 * (rows + cols);
    case CC_LOWRANK: return param < 1 ? CC_ERR_ARG : 2 * param * (rows + cols);
    case CC_LOWRANK4: return param < 1 ? CC_ERR_ARG : (4 * param * (rows + cols) + 7) / 8 + 8 * param;
    case CC_TOPK: return param < 0 ? CC_ERR_ARG : 6 * param;
    case CC_NMBLOCK: {
      int n, m;
      return nm_split(param, &n, &m) ? nm_body_bytes(rows, cols, n, m) : CC_ERR_ARG;
    }
    default: return CC_ERR_ARG;
  }
}

CC_API int64_t cc_workspace_bytes(int codec, int64_t rows, int64_t cols, int64_t param) {
  if (rows < 1 || cols < 1) return CC_ERR_SHAPE;
  if (quant_codec(codec)) return quant_workspace_bytes(rows, cols) + 256;
  if (codec == CC_TOPK) return topk_workspace_bytes(rows, cols, param);
  if (codec == CC_LOWRANK || codec == CC_LOWRANK4) return lowrank_workspace_bytes(rows, cols, param);
  if (codec == CC_NMBLOCK) {
    int n, m;
    return nm_split(param, &n, &m) ? nm_workspace_bytes(rows, cols, n, m) : CC_ERR_ARG;
  }
  if (codec == CC_RAW) return 0;
  return CC_ERR_ARG;
}

CC_API int cc_encode_step(int codec, int mode, int scale_mode, int64_t rows, int64_t cols, const void *x,
                          int x_dtype, float *base, float *aux, uint8_t *body, void *workspace,
                          int64_t workspace_bytes, double *record, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || (x_dtype != CC_F32 && x_dtype != CC_BF16)) { set_error("bad mode/dtype"); return CC_ERR_ARG; }
  if (!x || !base || !body || !record || (mode != CC_NAIVE && !aux)) { set_error("null pointer"); return CC_ERR_ARG; }
  if (scale_mode < CC_SCALE_RANK1 || scale_mode > CC_SCALE_PER_CHANNEL) { set_error("bad scale mode"); return CC_ERR_ARG; }
  if (!quant_codec(codec)) { set_error("cc_encode_step: codec must be sign1/quant2/quant4"); return CC_ERR_UNSUPPORTED; }
  return quant_encode_step(codec, mode, scale_mode, rows, cols, x, x_dtype, base, aux, body, workspace,
                           workspace_bytes, record, (cudaStream_t)stream);
}

CC_API int cc_encode_step_segmented(int codec, int mode, int scale_mode, int64_t rows, int64_t cols, int segments,
                                    const void *x, int x_dtype, float *base, float *aux, uint8_t *body,
                                    int64_t body_stride, void *workspace, int64_t workspace_bytes, double *record,
                                    void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || (x_dtype != CC_F32 && x_dtype != CC_BF16)) { set_error("bad mode/dtype"); return CC_ERR_ARG; }
  if (!x || !base || !body || !record || (mode != CC_NAIVE && !aux)) { set_error("null pointer"); return CC_ERR_ARG; }
  if (scale_mode < CC_SCALE_RANK1 || scale_mode > CC_SCALE_PER_CHANNEL) { set_error("bad scale mode"); return CC_ERR_ARG; }
  if (!quant_codec(codec)) { set_error("cc_encode_step_segmented: codec must be sign1/quant2/quant4"); return CC_ERR_UNSUPPORTED; }
  if (segments < 1 || cols % segments != 0) { set_error("segments must divide cols"); return CC_ERR_SHAPE; }
  if (segments == 1)
    return quant_encode_step(codec, mode, scale_mode, rows, cols, x, x_dtype, base, aux, body, workspace,
                             workspace_bytes, record, (cudaStream_t)stream);
  if (!fused_supported(rows, cols, x, x_dtype, base, aux, body) ||
      !fused_segments_supported(rows, cols, segments, body_stride, codec)) {
    set_error("cc_encode_step_segmented: shape / alignment not supported by the fused kernel "
              "(needs cols % 128 == 0, cols <= 3072, (cols/segments) % 128 == 0, 16-byte aligned buffers)");
    return CC_ERR_UNSUPPORTED;
  }
  return fused_encode_segments(codec, mode, scale_mode, rows, cols, segments, x, x_dtype, base, aux, body,
                               body_stride, workspace, workspace_bytes, record, (cudaStream_t)stream);
}

CC_API int cc_warmup_step(int mode, int64_t rows, int64_t cols, const void *x, int x_dtype, float *base, float *aux,
                          void *body, int body_dtype, double *record, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || (x_dtype != CC_F32 && x_dtype != CC_BF16)) { set_error("bad mode/dtype"); return CC_ERR_ARG; }
  if (body_dtype == CC_BF16 && x_dtype != CC_BF16) { set_error("bf16 raw body needs bf16 input (lossless only)"); return CC_ERR_ARG; }
  if (!x || !base || !body || (mode != CC_NAIVE && !aux)) { set_error("null pointer"); return CC_ERR_ARG; }
  return raw_warmup(mode, rows, cols, x, x_dtype, base, aux, body, body_dtype, record, (cudaStream_t)stream);
}

CC_API int cc_decode_batched(int codec, int accumulate, int count, const int64_t *rows, int64_t cols, int64_t param,
                             const uint8_t *const *bodies, int body_dtype, float *const *bases, void *stream) {
  if (count < 0 || cols < 1 || (count > 0 && (!rows || !bodies || !bases))) { set_error("bad batch"); return CC_ERR_ARG; }
  for (int i = 0; i < count; ++i) {
    if (rows[i] < 1) { set_error("empty shard"); return CC_ERR_SHAPE; }
    if (!bodies[i] || !bases[i]) { set_error("null pointer"); return CC_ERR_ARG; }
  }
  if (count == 0) return CC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (codec == CC_RAW) return raw_decode(count, rows, cols, reinterpret_cast<const void *const *>(bodies), body_dtype, bases, st);
  if (quant_codec(codec)) return quant_decode(codec, accumulate, count, rows, cols, bodies, bases, st);
  if (codec == CC_TOPK) return topk_decode(count, rows, cols, param, bodies, accumulate, bases, st);
  if (codec == CC_NMBLOCK) {
    int n, m;
    if (!nm_split(param, &n, &m)) { set_error("bad n:m"); return CC_ERR_ARG; }
    return nm_decode(count, rows, cols, n, m, bodies, accumulate, bases, st);
  }
  if (codec == CC_LOWRANK || codec == CC_LOWRANK4)
    return lowrank_decode(codec == CC_LOWRANK4, count, rows, cols, param, bodies, accumulate, bases, st);
  set_error("unsupported codec");
  return CC_ERR_UNSUPPORTED;
}

CC_API int cc_decode_step(int codec, int accumulate, int64_t rows, int64_t cols, int64_t param, const uint8_t *body,
                          int body_dtype, float *base, void *stream) {
  return cc_decode_batched(codec, accumulate, 1, &rows, cols, param, &body, body_dtype, &base, stream);
}

CC_API int cc_residual_target(int mode, int64_t rows, int64_t cols, const void *x, int x_dtype, const float *base,
                              const float *aux, float *t, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || !x || !t || (mode == CC_WITH_FEEDBACK && !base) || (mode != CC_NAIVE && !aux)) {
    set_error("bad residual_target args");
    return CC_ERR_ARG;
  }
  return residual_target(mode, rows, cols, x, x_dtype, base, aux, t, (cudaStream_t)stream);
}

CC_API int cc_apply_decoded(int mode, int64_t rows, int64_t cols, const void *x, int x_dtype, const float *t,
                            const float *decoded, float *base, float *aux, double *record, void *workspace,
                            int64_t workspace_bytes, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || !x || !t || !decoded || !base || !record || (mode != CC_NAIVE && !aux)) {
    set_error("bad apply_decoded args");
    return CC_ERR_ARG;
  }
  return apply_decoded(mode, rows, cols, x, x_dtype, t, decoded, base, aux, record, workspace, workspace_bytes,
                       (cudaStream_t)stream);
}

CC_API int cc_topk_encode(int64_t rows, int64_t cols, int64_t k, const float *t, uint8_t *body, float *decoded,
                          void *workspace, int64_t workspace_bytes, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (k < 0 || k > rows * cols || !t || !body) { set_error("bad top-k args"); return CC_ERR_ARG; }
  if (rows * cols > (int64_t)UINT32_MAX) { set_error("top-k indices are u32"); return CC_ERR_SHAPE; }
  return topk_encode(rows, cols, k, t, body, decoded, workspace, workspace_bytes, (cudaStream_t)stream);
}

CC_API int cc_topk_encode_step(int mode, int64_t rows, int64_t cols, int64_t k, const void *x, int x_dtype,
                               float *base, float *aux, uint8_t *body, void *workspace, int64_t workspace_bytes,
                               double *record, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || (x_dtype != CC_F32 && x_dtype != CC_BF16)) { set_error("bad mode/dtype"); return CC_ERR_ARG; }
  if (k < 1 || k > rows * cols || !x || !base || !body || !record || (mode != CC_NAIVE && !aux)) {
    set_error("bad top-k step args");
    return CC_ERR_ARG;
  }
  if (rows * cols > (int64_t)UINT32_MAX) { set_error("top-k indices are u32"); return CC_ERR_SHAPE; }
  return topk_encode_step(mode, rows, cols, k, x, x_dtype, base, aux, body, workspace, workspace_bytes, record,
                          (cudaStream_t)stream);
}

CC_API int cc_nm_encode(int64_t rows, int64_t cols, int n, int m, const float *t, uint8_t *body, float *decoded,
                        void *workspace, int64_t workspace_bytes, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!(1 <= n && n <= m && m <= 65535) || !t || !body) { set_error("need 1 <= n <= m <= 65535"); return CC_ERR_ARG; }
  return nm_encode(rows, cols, n, m, t, body, decoded, workspace, workspace_bytes, (cudaStream_t)stream);
}

CC_API int cc_nm_encode_step(int mode, int64_t rows, int64_t cols, int n, int m, const void *x, int x_dtype,
                             float *base, float *aux, uint8_t *body, void *workspace, int64_t workspace_bytes,
                             double *record, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || (x_dtype != CC_F32 && x_dtype != CC_BF16)) { set_error("bad mode/dtype"); return CC_ERR_ARG; }
  if (!(1 <= n && n <= m && m <= 65535)) { set_error("need 1 <= n <= m <= 65535"); return CC_ERR_ARG; }
  if (!x || !base || !body || !record || (mode != CC_NAIVE && !aux)) { set_error("null pointer"); return CC_ERR_ARG; }
  return nm_encode_step(mode, rows, cols, n, m, x, x_dtype, base, aux, body, workspace, workspace_bytes, record,
                        (cudaStream_t)stream);
}

CC_API int64_t cc_lowrank_workspace_bytes(int64_t rows, int64_t cols, int64_t rank) {
  if (rows < 1 || cols < 1) return CC_ERR_SHAPE;
  if (rank < 1 || rank > (rows < cols ? rows : cols)) return CC_ERR_SHAPE;
  return lowrank_workspace_bytes(rows, cols, rank);
}

CC_API int cc_lowrank_encode(int int4, int64_t rows, int64_t cols, int64_t rank, int iterations, const float *t,
                             const float *q0, uint8_t *body, float *decoded, void *workspace,
                             int64_t workspace_bytes, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (rank < 1 || rank > (rows < cols ? rows : cols)) { set_error("rank out of range"); return CC_ERR_SHAPE; }
  if (iterations < 1 || !t || !q0 || !body) { set_error("bad low-rank args"); return CC_ERR_ARG; }
  return lowrank_encode(int4, rows, cols, rank, iterations, t, q0, body, decoded, workspace, workspace_bytes,
                        (cudaStream_t)stream);
}

CC_API int64_t cc_gaussian_workspace_bytes(int64_t rows, int64_t cols) {
  if (rows < 1 || cols < 1) return CC_ERR_SHAPE;
  return cc::gaussian_workspace_bytes(rows, cols);
}

CC_API int cc_gaussian_keyed(int64_t rows, int64_t cols, uint32_t *key, int nwords, int step_word, float *out,
                             void *workspace, int64_t workspace_bytes, void *stream) {
  return cc::gaussian_keyed(rows, cols, key, nwords, step_word, out, workspace, workspace_bytes, (cudaStream_t)stream);
}

CC_API int64_t cc_lowrank_step_workspace_bytes(int64_t rows, int64_t cols, int64_t rank) {
  if (rows < 1 || cols < 1) return CC_ERR_SHAPE;
  if (rank < 1 || rank > (rows < cols ? rows : cols)) return CC_ERR_SHAPE;
  return lowrank_step_workspace_bytes(rows, cols, rank);
}

CC_API int cc_lowrank_encode_step(int mode, int64_t rows, int64_t cols, int64_t rank, int iterations, int int4,
                                  const void *x, int x_dtype, float *base, float *aux, const float *q0,
                                  uint32_t *key, int nwords, int step_word, uint8_t *body, void *workspace,
                                  int64_t workspace_bytes, double *record, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (rank < 1 || rank > (rows < cols ? rows : cols)) { set_error("rank out of range"); return CC_ERR_SHAPE; }
  if (!valid_mode(mode) || (x_dtype != CC_F32 && x_dtype != CC_BF16)) { set_error("bad mode/dtype"); return CC_ERR_ARG; }
  if (iterations < 1 || !x || !base || !body || !record || (mode != CC_NAIVE && !aux) || (!q0 == !key)) {
    set_error("bad low-rank step args (exactly one of q0 / key)");
    return CC_ERR_ARG;
  }
  if (key && (nwords < 1 || nwords > 16 || step_word >= nwords)) { set_error("bad key"); return CC_ERR_ARG; }
  return lowrank_encode_step(mode, rows, cols, rank, iterations, int4, x, x_dtype, base, aux, q0, key, nwords,
                             step_word, body, workspace, workspace_bytes, record, (cudaStream_t)stream);
}

CC_API int cc_encode(int codec, int scale_mode, int64_t rows, int64_t cols, int64_t param, const float *t,
                     uint8_t *body, float *decoded, void *workspace, int64_t workspace_bytes, void *stream) {
  if (rows < 1 || cols < 1) { set_error("empty shape"); return CC_ERR_SHAPE; }
  if (!t || !body) { set_error("null pointer"); return CC_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  if (quant_codec(codec)) {
    // stateless encode = naive-mode step on a scratch base: base <- decode(body)
    if (!decoded) { set_error("cc_encode(quant) needs a decoded buffer"); return CC_ERR_ARG; }
    int64_t wsq = quant_workspace_bytes(rows, cols);
    if (workspace_bytes < wsq + 256) { set_error("workspace too small"); return CC_ERR_ARG; }
    double *rec = reinterpret_cast<double *>(reinterpret_cast<uint8_t *>(workspace) + wsq);
    return quant_encode_step(codec, CC_NAIVE, scale_mode, rows, cols, t, CC_F32, decoded, nullptr, body,
                             workspace, wsq, rec, st);
  }
  if (codec == CC_TOPK) return topk_encode(rows, cols, param, t, body, decoded, workspace, workspace_bytes, st);
  if (codec == CC_NMBLOCK) {
    int n, m;
    if (!nm_split(param, &n, &m)) { set_error("bad n:m"); return CC_ERR_ARG; }
    return nm_encode(rows, cols, n, m, t, body, decoded, workspace, workspace_bytes, st);
  }
  set_error("cc_encode: use cc_lowrank_encode for low-rank");
  return CC_ERR_UNSUPPORTED;
}

}  // extern "C"
