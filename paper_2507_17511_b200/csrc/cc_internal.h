// Internal host-side declarations shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <string>

namespace cc {

extern std::atomic<int64_t> g_launches;
void set_error(const std::string &msg);
int cuda_status(const char *where);  // checks cudaGetLastError, returns CC_OK / CC_ERR_CUDA

inline void count_launch(int k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

inline bool aligned(const void *p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }
inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// number of SMs of the current device (cached)
int sm_count();

// programmatic dependent launch (PDL) for the K1 / K2 chain: kernels launch with
// programmatic stream serialization, trigger their dependents at entry and wait
// (griddepcontrol.wait) before touching memory, so a kernel's launch and prologue
// overlap its predecessor's tail.  1 = on.
int pdl_enabled();
// zero-initialised 512-byte control slot of `st` on the current device (see capi.cu);
// persistent kernels must leave it zeroed on exit.  Null when unavailable.
uint8_t *stream_control_block(cudaStream_t st);

// --- quantizer family (quant.cu) ------------------------------------------
int64_t quant_workspace_bytes(int64_t n, int64_t C);
int quant_encode_step(int codec, int mode, int scale_mode, int64_t n, int64_t C, const void *x, int x_dtype,
                      float *base, float *aux, uint8_t *body, void *ws, int64_t ws_bytes, double *record,
                      cudaStream_t st);
int quant_decode(int codec, int accumulate, int count, const int64_t *rows, int64_t C,
                 const uint8_t *const *bodies, float *const *bases, cudaStream_t st);
int raw_warmup(int mode, int64_t n, int64_t C, const void *x, int x_dtype, float *base, float *aux, void *body,
               int body_dtype, double *record, cudaStream_t st);
int raw_decode(int count, const int64_t *rows, int64_t C, const void *const *bodies, int body_dtype,
               float *const *bases, cudaStream_t st);

}  // namespace cc
