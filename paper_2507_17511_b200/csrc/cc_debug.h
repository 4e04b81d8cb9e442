/*
 * cc_debug.h — PRIVATE test / profiling knobs of libcompactcomm_b200.so.
 *
 * Not part of the drop-in ABI (include/compactcomm.h): the symbols are exported
 * so the parity tests and the experiment scripts can pin a code path or stamp a
 * kernel timeline, but no production caller should use them.  Every knob's
 * default is the production behaviour.
 */
#ifndef CC_DEBUG_H
#define CC_DEBUG_H

#include "compactcomm.h"

#ifdef __cplusplus
extern "C" {
#endif

/* encode-path selection for tests/benchmarks: -1 auto (persistent fused K1
 * when C % 1024 == 0 and aligned), 0 force the multi-kernel K1, 1 prefer fused */
CC_API void cc_set_quant_path(int path);
/* profiling only: stop the persistent K1 after phase 1 (scale partials) or
 * 2 (scales); 0 = full step.  Results are incomplete when != 0. */
CC_API void cc_debug_fused_stop(int phase);
/* profiling only: device buffer of [grid][8] u64 %globaltimer stamps written by
 * every CTA of the persistent K1 at its phase boundaries (NULL disables). */
CC_API void cc_debug_fused_timer(void *dev_buf);
/* profiling only (effective in builds with -DCC_K1_EXPERIMENTS=1): experiment bits of the persistent K1 (0 = production path; see
 * k1_fused.cu Params::policy: L2 hints, skipped math / stores, workspace control words,
 * forced phase-A evict_first fraction in bits 8..11) */
CC_API void cc_debug_fused_policy(int policy);
/* profiling only: phase-B end-game of the persistent K1: when fewer than mult x grid
 * tiles remain, a CTA keeps at most `keep` loaded tiles ahead of its consumers
 * (0, 0 = automatic) */
CC_API void cc_debug_fused_tail(int mult, int keep);
/* programmatic dependent launch for the encode (K1) / decode (K2) kernels: each
 * launches with programmatic stream serialization and waits for its predecessor's
 * completion (griddepcontrol.wait) before touching memory, so launch and prologue
 * overlap the previous kernel's tail.  Results are unchanged.  0 = off (default: measured
 * 2% slower in bench.py's graph replay at [4096, 3072]). */
CC_API void cc_set_pdl(int enable);
/* profiling only: phase-B ring depths of the persistent K1 (0 = automatic) */
CC_API void cc_debug_fused_rings(int s_in, int s_out);
/* profiling only: phase-A tile height (rows per row group) and ring depth of the
 * persistent K1 (0 = automatic) */
CC_API void cc_debug_fused_phase_a(int rows_per_group, int stages);
/* low-rank projections: 1 = tcgen05 tensor cores, 3xTF32 split (default),
 * 0 = f64-accumulating CUDA-core GEMMs (cross-check) */
CC_API void cc_set_lowrank_backend(int backend);
/* low-rank tcgen05 projections: operand staging — 2 (default) A Q TMA-staged (2-D tensor map)
 * and A^T Y register-staged, 1 both TMA-staged, 0 both register-staged; identical results.
 * waves: unused */
CC_API void cc_debug_lowrank_tma(int enable, int waves);

/* K1 shard-resident kernel (k1_resident.cu): 1 = use it whenever the shard fits
 * on chip (default), 0 = always the streaming kernel (A/B and parity tests). */
CC_API void cc_debug_k1_resident(int enable);
/* launches of the shard-resident K1 since load (tests check which kernel ran) */
CC_API int64_t cc_debug_k1_resident_count(void);
/* K1 shard-resident kernel geometry: 1 = 24 consumer warps (default), 2 = 12
 * register-capped warps (lets a decode on another stream share the SMs) */
CC_API void cc_debug_k1_resident_nq(int nq);

/* K4 shard-resident top-k kernel (topk_resident.cu): 1 = use it for encode steps
 * whenever it can launch (default), 0 = always the multi-kernel radix select. */
CC_API void cc_debug_topk_resident(int enable);
/* launches of the shard-resident top-k kernel since load */
CC_API int64_t cc_debug_topk_resident_count(void);
/* profiling only: device buffer of [grid][16] u64 %globaltimer stamps of the
 * resident top-k kernel's phases (NULL disables) */
CC_API void cc_debug_topk_timer(void *dev_buf);
/* profiling only: device buffer of 16 u64 clock64 stamps of the single-CTA
 * CholQR2 (k_orth1) phases (NULL disables) */
CC_API void cc_debug_orth_stamps(void *dev_buf);
/* low-rank orthogonalisation: 1 = thread-block-cluster CholQR2 (default),
 * 0 = the single-CTA / cooperative-grid forms (A/B and cross-checks) */
CC_API void cc_debug_orth_cluster(int enable);
/* profiling only: device buffer of 16 u64 %globaltimer stamps of the device Gaussian
 * draw's phases (NULL disables) */
CC_API void cc_debug_gauss_stamps(void *dev_buf);

/* low-rank encode_step as one persistent cluster launch (lr_step.cu): 1 = whenever it
 * covers the shape (default), 0 = always the multi-kernel step (A/B and cross-checks) */
CC_API void cc_debug_lowrank_fused(int enable);
/* launches of the fused low-rank step since load */
CC_API int64_t cc_debug_lowrank_fused_count(void);
/* profiling only: device buffer of 32 u64 %globaltimer stamps of the fused low-rank
 * step's phases (CTA 0; NULL disables) */
CC_API void cc_debug_lowrank_fused_stamps(void *dev_buf);

#ifdef __cplusplus
}
#endif
#endif /* CC_DEBUG_H */
