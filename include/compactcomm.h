/*
 * compactcomm.h — C ABI of the B200 (sm_100a) residual-compression path.
 *
 * Drop-in boundary for the reference package `compactcomm` (arXiv 2507.17511,
 * /root/reference/pkg/src/compactcomm).  Every entry point is extern "C", takes
 * plain device pointers, sizes and a cudaStream_t (passed as void*), never
 * throws, and returns CC_OK or a negative status.  The Python host mirror
 * (paper_2507_17511_b200/) binds these with ctypes and raises the reference's
 * exception classes for the status codes.
 *
 * All work is stream-ordered: nothing here synchronizes the device.  State
 * buffers (base, feedback, ref) are owned by the caller and updated in place;
 * shape/step validation happens host-side BEFORE any launch, so a failing call
 * leaves state untouched (reference pipeline.py:146-151).
 *
 * Body layout = the reference's codec body byte-for-byte (compressors.py:580-603,
 * i.e. the frame minus its 9-byte <BII header and meta ints):
 *   CC_SIGN1   ceil(n*C/8) B sign bitmap (little bit order, 1 = negative),
 *              then u f32[n], v f32[C]                          (cx:373-376, 586)
 *   CC_QUANT2  ceil(2*n*C/8) B codes (4/byte, first code in low bits,
 *              0:-2 1:-0.5 2:+0.5 3:+2), then u f32[n], v f32[C] (cx:379-391, 588)
 *   CC_QUANT4  extension (no reference; parity unpinned): ceil(4*n*C/8) B
 *              codes (2/byte, low nibble first, level (k-7.5)/2), then u, v
 *   CC_TOPK    k x u32 ascending flat indices, then k x f16 values (cx:446-456, 601)
 *   CC_LOWRANK U [n,r] then W [C,r], column-major f16           (cx:415-426, 591)
 *   CC_LOWRANK4 2r f32 ranges, then one nibble stream U then W col-major (cx:592-595)
 *   CC_NMBLOCK ceil(blocks*m/8) B keep-mask (m bits per 1 x m block of the
 *              column-padded matrix, little bit order), then n f16 values per
 *              block in index order                            (cx:429-443, 596)
 *   CC_RAW     n*C f32 (wire may carry bf16 when inputs are bf16: lossless)
 */
#ifndef COMPACTCOMM_H
#define COMPACTCOMM_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CC_API __attribute__((visibility("default")))

/* status codes (reference exception classes in brackets) */
#define CC_OK 0
#define CC_ERR_ARG (-1)        /* ValueError (cx:90-100)                       */
#define CC_ERR_SHAPE (-2)      /* linalg.ShapeError (la:16)                    */
#define CC_ERR_PAYLOAD (-3)    /* compressors.PayloadError (cx:67)             */
#define CC_ERR_PROTOCOL (-4)   /* pipeline.ProtocolError (pl:36)               */
#define CC_ERR_CUDA (-5)       /* launch / runtime failure                      */
#define CC_ERR_UNSUPPORTED (-6)
#define CC_ERR_NCCL (-7)       /* transport.TransportError (tr:22)             */

/* codec tags: identical numbering to compressors.py:56-62 */
#define CC_RAW 0
#define CC_SIGN1 1
#define CC_QUANT2 2
#define CC_LOWRANK 3
#define CC_LOWRANK4 4
#define CC_NMBLOCK 5
#define CC_TOPK 6
#define CC_QUANT4 16 /* extension: 4-bit element quantizer (north_star), no reference */

/* pipeline modes: pipeline.py:40-43 */
#define CC_NAIVE 0
#define CC_NO_FEEDBACK 1
#define CC_WITH_FEEDBACK 2

/* element types of activations / raw wire bodies */
#define CC_F32 0
#define CC_BF16 1

/* scale modes for the quantizers: CC_SCALE_RANK1 is the reference's u v^T
 * (cx:135-149); the other two are north_star extensions (parity unpinned). */
#define CC_SCALE_RANK1 0
#define CC_SCALE_PER_TOKEN 1
#define CC_SCALE_PER_CHANNEL 2

/* `param` of the N:M codec: n (kept per block) and m (block width), 1 <= n <= m
 * <= 65535 — the frame meta <HH n, m> of cx:596-597. */
#define CC_NM_PARAM(n, m) ((((int64_t)(n)) << 16) | (int64_t)(m))

/* ---- sizes -------------------------------------------------------------- */

/* Exact body size in bytes: ceil(bit_size/8) (cx:195-348). param = rank for
 * low-rank, k for top-k, CC_NM_PARAM(n, m) for N:M, ignored otherwise.
 * Returns <0 on bad arguments. */
CC_API int64_t cc_body_bytes(int codec, int64_t rows, int64_t cols, int64_t param);

/* Device scratch bytes needed by cc_encode_step for this codec/shape. */
CC_API int64_t cc_workspace_bytes(int codec, int64_t rows, int64_t cols, int64_t param);

/* ---- sender step: pipeline.encode_step (pl:84-121) ------------------------
 * One fused residual -> scale -> quantize -> pack -> state-update pass for
 * the 1/2/4-bit codecs.
 *   x        [rows, cols] activation (x_dtype), borrowed
 *   base     [rows, cols] f32 shared base, updated in place
 *   aux      [rows, cols] f32: feedback (CC_WITH_FEEDBACK), previous input
 *            `ref` (CC_NO_FEEDBACK), unused (CC_NAIVE, may be NULL)
 *   body     cc_body_bytes() device bytes, written
 *   scales   optional f32 [rows+cols] aligned copy of (u, v) (may be NULL)
 *   record   2 f64 on device: ||decode - target||^2, ||target||^2  (pl:115-120)
 */
CC_API int cc_encode_step(int codec, int mode, int scale_mode, int64_t rows, int64_t cols,
                          const void *x, int x_dtype, float *base, float *aux,
                          uint8_t *body, void *workspace, int64_t workspace_bytes,
                          double *record, void *stream);

/* Segmented sender step for Ulysses sequence parallelism (every
 * directed (src, dst) chunk is its own LayerState channel).  Equivalent to
 * `segments` independent cc_encode_step calls on the column slices
 * x[:, d*cw:(d+1)*cw] (cw = cols / segments) with states base/aux[:, slice],
 * bodies at body + d * body_stride (each the reference body of an [rows, cw]
 * channel) and records at record + 2 d — in ONE persistent launch over the
 * full-width rows (no chunk copies).  base / aux / x stay [rows, cols] row-major.
 * Needs the fused kernel's shapes: cols % 128 == 0, cols <= 3072, cw % 128 == 0,
 * segments <= 16, 16-byte aligned buffers and body_stride; CC_ERR_UNSUPPORTED
 * otherwise (the caller then encodes chunk by chunk). */
CC_API int cc_encode_step_segmented(int codec, int mode, int scale_mode, int64_t rows, int64_t cols,
                                    int segments, const void *x, int x_dtype, float *base, float *aux,
                                    uint8_t *body, int64_t body_stride, void *workspace,
                                    int64_t workspace_bytes, double *record, void *stream);

/* Warmup / identity step (pl:89-97): base = x, feedback = 0, ref = x,
 * body = raw x as body_dtype (CC_F32 = the reference wire, CC_BF16 lossless
 * for bf16 inputs), record = {0, 0}: compression_error = 0, so delta_hat = 1
 * (pl:76-81) and the target norm is not computed on warmup steps. */
CC_API int cc_warmup_step(int mode, int64_t rows, int64_t cols, const void *x, int x_dtype,
                          float *base, float *aux, void *body, int body_dtype, double *record,
                          void *stream);

/* ---- receiver step: pipeline.decode_step (pl:146-165) ----------------------
 * base = decode(body) when !accumulate (warmup / raw / naive), else
 * base += decode(body).  param as in cc_body_bytes. */
CC_API int cc_decode_step(int codec, int accumulate, int64_t rows, int64_t cols, int64_t param,
                          const uint8_t *body, int body_dtype, float *base, void *stream);

/* Batched receiver step for P-1 peers of one all-gather (mesh:232-236): one
 * launch decodes `count` bodies into their bases.  rows[i] may differ (last
 * shard takes the remainder, mesh:125-135); the arrays are HOST arrays of
 * device pointers.  count <= 64. */
CC_API int cc_decode_batched(int codec, int accumulate, int count, const int64_t *rows, int64_t cols,
                             int64_t param, const uint8_t *const *bodies, int body_dtype,
                             float *const *bases, void *stream);

/* ---- generic protocol halves (for codecs that need the materialized target:
 * top-k, low-rank) ------------------------------------------------------------
 * cc_residual_target: t = (x - base) + fb | x - ref | x   (pl:99-104)
 * cc_apply_decoded:   fb' = t - d, base' = base + d | d, ref' = x, and the
 *                     record {||d - t||^2, ||t||^2} (pl:107-120); workspace
 *                     >= 16 KiB of device scratch. */
CC_API int cc_residual_target(int mode, int64_t rows, int64_t cols, const void *x, int x_dtype,
                              const float *base, const float *aux, float *t, void *stream);
CC_API int cc_apply_decoded(int mode, int64_t rows, int64_t cols, const void *x, int x_dtype,
                            const float *t, const float *decoded, float *base, float *aux,
                            double *record, void *workspace, int64_t workspace_bytes, void *stream);

/* ---- standalone codec (compressors.encode / decode, cx:459-481) ---------- */

/* encode target t (f32 [rows, cols]) into body; decoded (optional, f32) gets
 * decode(body) — the stateless codec entry used by compressors.encode. */
CC_API int cc_encode(int codec, int scale_mode, int64_t rows, int64_t cols, int64_t param,
                     const float *t, uint8_t *body, float *decoded, void *workspace,
                     int64_t workspace_bytes, void *stream);

/* ---- top-k (cx:446-456) ---------------------------------------------------
 * Radix-select the k largest |t| (ties -> lowest flat index), emit ascending
 * u32 indices + f16 values.  Used by cc_encode_step with codec CC_TOPK; k is
 * cc_topk_count(rows, cols, keep_fraction). */
CC_API int64_t cc_topk_count(int64_t rows, int64_t cols, double keep_fraction);
CC_API int cc_topk_encode(int64_t rows, int64_t cols, int64_t k, const float *t, uint8_t *body,
                          float *decoded, void *workspace, int64_t workspace_bytes, void *stream);
/* Fused top-k sender step: target -> radix select -> ordered body -> sparse
 * state update + record, straight from (x, base, aux).  Receivers decode with
 * cc_decode_step(CC_TOPK, accumulate, ..., param = k): accumulate 0 = replace
 * (zero + scatter), 1 = sparse add, 2 = dense `base + 0.0` (-0.0 -> +0.0, the
 * reference's dense add, pl:163) then sparse add. */
CC_API int cc_topk_encode_step(int mode, int64_t rows, int64_t cols, int64_t k, const void *x, int x_dtype,
                               float *base, float *aux, uint8_t *body, void *workspace,
                               int64_t workspace_bytes, double *record, void *stream);

/* ---- N:M block sparsifier (cx:429-443) ----------------------------------------
 * Keep the n largest-|t| entries of every 1 x m column block (ties -> lowest
 * index), columns zero-padded to a multiple of m.  One pass: the selection is
 * block-local.  cc_nm_encode_step fuses target -> select -> body -> state update
 * + record (pl:99-120); receivers decode with cc_decode_step(CC_NMBLOCK,
 * accumulate, ..., CC_NM_PARAM(n, m)) (accumulate = dense base + decode). */
CC_API int cc_nm_encode(int64_t rows, int64_t cols, int n, int m, const float *t, uint8_t *body,
                        float *decoded, void *workspace, int64_t workspace_bytes, void *stream);
CC_API int cc_nm_encode_step(int mode, int64_t rows, int64_t cols, int n, int m, const void *x, int x_dtype,
                             float *base, float *aux, uint8_t *body, void *workspace,
                             int64_t workspace_bytes, double *record, void *stream);

/* ---- low-rank (cx:394-426) -------------------------------------------------
 * q0: [cols, r] f32 initial Gaussian block (drawn host-side from the same
 * PCG64 stream as la.gaussian_matrix, cx:407); iterations = T. */
CC_API int cc_lowrank_encode(int int4, int64_t rows, int64_t cols, int64_t rank, int iterations,
                             const float *t, const float *q0, uint8_t *body, float *decoded,
                             void *workspace, int64_t workspace_bytes, void *stream);
CC_API int64_t cc_lowrank_workspace_bytes(int64_t rows, int64_t cols, int64_t rank);

/* One low-rank encode_step (pl:84-121 with cx:394-426): t = target(x, base, aux)
 * -> Q0 -> subspace iteration -> body -> base' / aux' and record (the decode is
 * fused into the state update, bit-identical to the receiver's decode).  Q0 is
 * either q0 (a host draw, la.gaussian_matrix(rng, cols, rank)) or drawn on the
 * device from key (cc_gaussian_keyed below); exactly one of q0 / key is non-null.
 * With a key every launch is stream-ordered device work (CUDA-graph capturable). */
CC_API int64_t cc_lowrank_step_workspace_bytes(int64_t rows, int64_t cols, int64_t rank);
CC_API int cc_lowrank_encode_step(int mode, int64_t rows, int64_t cols, int64_t rank, int iterations, int int4,
                                  const void *x, int x_dtype, float *base, float *aux, const float *q0,
                                  uint32_t *key, int nwords, int step_word, uint8_t *body, void *workspace,
                                  int64_t workspace_bytes, double *record, void *stream);

/* ---- the low-rank start block drawn on the device (cx:407, la:67-74) --------
 * out [rows, cols] f32 = float32(numpy Generator(PCG64(SeedSequence(entropy,
 * spawn_key))).standard_normal((rows, cols))), bit for bit (la:25-27 spawn_rng;
 * keys of pl:190 / mesh:193).  key: DEVICE array of nwords (<= 16) uint32 =
 * SeedSequence's assembled entropy: the entropy's little-endian 32-bit words,
 * zero-padded to 4 words when a spawn key follows, then one word per spawn-key
 * element (< 2^32).  step_word >= 0: key[step_word] += 1 after the draw
 * (stream-ordered), so a step captured in a CUDA graph draws the next step's
 * block on every replay; -1 leaves the key unchanged. */
CC_API int64_t cc_gaussian_workspace_bytes(int64_t rows, int64_t cols);
CC_API int cc_gaussian_keyed(int64_t rows, int64_t cols, uint32_t *key, int nwords, int step_word, float *out,
                             void *workspace, int64_t workspace_bytes, void *stream);

/* ---- exchanges: K1 encode -> NCCL collective -> K2 decode, from C -----------
 * The reference's seam is mesh._Device._run (mesh.py:188-236) over
 * Transport.send/recv (transport.py:36-43); here one call runs one layer step of
 * the patch-parallel all-gather or the Ulysses all-to-all on `stream`.
 *
 * Communicator: cc_comm_wrap() adopts an existing ncclComm_t (e.g. PyTorch's
 * ProcessGroupNCCL._comm_ptr(); not destroyed by cc_comm_destroy), or
 * cc_comm_get_unique_id() on one rank + cc_comm_init_rank() on every rank builds
 * one (NCCL is loaded at run time: libnccl.so.2).  A NULL comm means world size 1.
 *
 * Layer objects own every device buffer of the step: the [rows, cols] f32
 * reconstruction (this rank's row shard = the sender base, mesh:233), the
 * sender's feedback / ref, the codec workspace, the StepRecord and the send /
 * receive wire buffers (ncclCommRegister'd when NCCL offers it).  x is borrowed.
 * Shards are contiguous row ranges, the last rank takes the remainder
 * (mesh:125-135); warmup and identity steps move the raw activation in its own
 * dtype (bf16 stays bf16: lossless).  Codecs: identity (CC_RAW), sign1 / quant2 /
 * quant4 (any scale mode), top-k and N:M for the all-gather; the quantizers for
 * the all-to-all (segmented K1: cols % 128 == 0, cols <= 3072, (cols/P) % 128 == 0). */
typedef struct cc_comm cc_comm;
typedef struct cc_allgather_layer cc_allgather_layer;
typedef struct cc_alltoall_layer cc_alltoall_layer;
typedef struct {
  int codec;            /* CC_RAW (identity), CC_SIGN1, CC_QUANT2, CC_QUANT4, CC_TOPK, CC_NMBLOCK */
  int scale_mode;       /* CC_SCALE_* (quantizers) */
  double keep_fraction; /* top-k (cx:446-451) */
  int nm_n, nm_m;       /* N:M block sparsifier (cx:429-443) */
} cc_codec_spec;

CC_API int cc_comm_get_unique_id(uint8_t *id_out /* 128 bytes */);
CC_API int cc_comm_init_rank(const uint8_t *id, int nranks, int rank, cc_comm **out);
CC_API int cc_comm_wrap(void *nccl_comm, cc_comm **out);
CC_API int cc_comm_rank(const cc_comm *c);
CC_API int cc_comm_size(const cc_comm *c);
CC_API int cc_comm_destroy(cc_comm *c);

/* patch parallelism (mesh.py:188-237): x_shard is this rank's [hi - lo, cols]
 * rows (cc_allgather_shard).  After a step, cc_allgather_reconstruction() is the
 * [rows, cols] f32 activation every rank agrees on bit for bit (mesh:237). */
CC_API int cc_allgather_create(cc_comm *c, const cc_codec_spec *spec, int mode, int64_t rows, int64_t cols,
                               int warmup, int x_dtype, cc_allgather_layer **out);
CC_API int cc_allgather_step(cc_allgather_layer *layer, const void *x_shard, void *stream);
CC_API float *cc_allgather_reconstruction(cc_allgather_layer *layer);
CC_API float *cc_allgather_sender_base(cc_allgather_layer *layer);
CC_API float *cc_allgather_sender_aux(cc_allgather_layer *layer);
CC_API const uint8_t *cc_allgather_body(cc_allgather_layer *layer, int64_t *nbytes);
CC_API const double *cc_allgather_record(cc_allgather_layer *layer);
CC_API int cc_allgather_shard(cc_allgather_layer *layer, int64_t *lo, int64_t *hi);
CC_API int cc_allgather_destroy(cc_allgather_layer *layer);

/* Ulysses sequence parallelism: x_local [n_local, cols]; output
 * [P * n_local, cols / P] = the full sequence for this rank's heads. */
CC_API int cc_alltoall_create(cc_comm *c, const cc_codec_spec *spec, int mode, int64_t n_local, int64_t cols,
                              int warmup, int x_dtype, cc_alltoall_layer **out);
CC_API int cc_alltoall_step(cc_alltoall_layer *layer, const void *x_local, void *stream);
CC_API float *cc_alltoall_output(cc_alltoall_layer *layer);
CC_API float *cc_alltoall_sender_base(cc_alltoall_layer *layer);
CC_API int cc_alltoall_destroy(cc_alltoall_layer *layer);

/* ---- diagnostics ----------------------------------------------------------- */
CC_API const char *cc_last_error(void);
CC_API int cc_version(void);
/* number of kernels this library launched since load (evidence counter) */
CC_API int64_t cc_launch_count(void);
/* Test / profiling knobs (encode-path selection, K1 experiment switches, PDL,
 * low-rank backends) are NOT part of this ABI: they are declared in the private
 * header paper_2507_17511_b200/csrc/cc_debug.h. */

#ifdef __cplusplus
}
#endif
#endif /* COMPACTCOMM_H */
