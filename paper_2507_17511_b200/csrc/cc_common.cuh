// Shared device helpers for the sm_100a residual-compression kernels.
//
// Floating-point discipline (needed for bit parity with the numpy reference):
//   * no fast-math, no FTZ (nvcc defaults: -ftz=false -prec-div=true)
//   * every f32 op the reference performs element-wise is written with an
//     explicit round-to-nearest intrinsic (__fadd_rn / __fsub_rn) so ptxas can
//     never contract it into an FMA
//   * scale math is done in f64 where the reference does it in f64
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <stdint.h>

#include "../../include/compactcomm.h"

namespace cc {

constexpr double kRowScaleFloor = 1e-30;  // compressors.py:52

__host__ __device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }
// PDL: let the next kernel in the stream launch now / wait for the previous one to
// complete (no-ops when the launch carried no programmatic dependency)
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__host__ __device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ __forceinline__ int64_t cdiv_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// activation loads: f32 or bf16 (bf16 -> f32 is exact: bits << 16)
// ---------------------------------------------------------------------------
template <typename XT>
struct Act;

template <>
struct Act<float> {
  static __device__ __forceinline__ float4 load4(const float *p) {
    return __ldcs(reinterpret_cast<const float4 *>(p));
  }
  static __device__ __forceinline__ float load1(const float *p) { return *p; }
};

template <>
struct Act<__nv_bfloat16> {
  static __device__ __forceinline__ float4 load4(const __nv_bfloat16 *p) {
    uint2 r = __ldcs(reinterpret_cast<const uint2 *>(p));
    float4 o;
    o.x = __uint_as_float(r.x << 16);
    o.y = __uint_as_float(r.x & 0xffff0000u);
    o.z = __uint_as_float(r.y << 16);
    o.w = __uint_as_float(r.y & 0xffff0000u);
    return o;
  }
  static __device__ __forceinline__ float load1(const __nv_bfloat16 *p) {
    return __uint_as_float(((uint32_t)(*reinterpret_cast<const uint16_t *>(p))) << 16);
  }
};

__device__ __forceinline__ float f4get(const float4 &v, int k) {
  return k == 0 ? v.x : (k == 1 ? v.y : (k == 2 ? v.z : v.w));
}
__device__ __forceinline__ void f4set(float4 &v, int k, float x) {
  if (k == 0) v.x = x; else if (k == 1) v.y = x; else if (k == 2) v.z = x; else v.w = x;
}

// ---------------------------------------------------------------------------
// residual target (pipeline.py:99-104); aux = feedback or ref
// ---------------------------------------------------------------------------
template <int MODE>
__device__ __forceinline__ float target_of(float x, float base, float aux) {
  if constexpr (MODE == CC_WITH_FEEDBACK) {
    return __fadd_rn(__fsub_rn(x, base), aux);  // (a* - base) + feedback
  } else if constexpr (MODE == CC_NO_FEEDBACK) {
    return __fsub_rn(x, aux);  // a* - ref
  } else {
    return x;  // naive
  }
}

// ---------------------------------------------------------------------------
// code assignment.  s = u_i * v_j exactly in f64 (24b x 24b mantissas),
// thr = u_i * (1.25 v_j) exactly (24b x 27b).  For f32 x the comparisons
// x > thr etc. are equivalent to the reference's rounded f64 x/s > 1.25
// (compressors.py:383-390) — see DESIGN.md §parity.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t quant2_code(float t, double s, double thr) {
  const double x = (double)t;
  if (s == 0.0) return 2u;  // zero scale -> +0.5 code (cx:387)
  if (x > thr) return 3u;
  if (x < -thr) return 0u;
  return x < 0.0 ? 1u : 2u;
}

__device__ __forceinline__ double quant2_level(uint32_t c) {
  // QUANT2_LEVELS (cx:54)
  return c == 0 ? -2.0 : (c == 1 ? -0.5 : (c == 2 ? 0.5 : 2.0));
}

// 4-bit extension: levels (k - 7.5)/2, k = 0..15; nearest with ties toward
// the smaller magnitude; -0.0 and zero scale map to +0.25 (code 8), mirroring
// the 2-bit tie rules.  m = #{k in 1..7 : |x| > k*s/2} (exact: k*s/2 needs
// <= 51 mantissa bits).
__device__ __forceinline__ uint32_t quant4_code(float t, double s) {
  if (s == 0.0) return 8u;
  const double ax = fabs((double)t);
  const double hs = 0.5 * s;
  // estimate then correct with exact compares
  double q = ax / hs;  // ~ 2|x|/s
  int m = (int)ceil(q) - 1;
  m = m < 0 ? 0 : (m > 7 ? 7 : m);
  if (m < 7 && ax > (double)(m + 1) * hs) ++m;
  if (m < 7 && ax > (double)(m + 1) * hs) ++m;
  if (m > 0 && !(ax > (double)m * hs)) --m;
  if (m > 0 && !(ax > (double)m * hs)) --m;
  return t < 0.0f ? (uint32_t)(7 - m) : (uint32_t)(8 + m);
}

__device__ __forceinline__ double quant4_level(uint32_t c) { return ((double)c - 7.5) * 0.5; }

// ---------------------------------------------------------------------------
// reductions
// ---------------------------------------------------------------------------
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// unaligned-safe f32 store / load inside a byte body
__device__ __forceinline__ void store_f32_bytes(uint8_t *p, float v) {
  uint32_t b = __float_as_uint(v);
  if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) {
    *reinterpret_cast<uint32_t *>(p) = b;
  } else {
    p[0] = b & 0xff; p[1] = (b >> 8) & 0xff; p[2] = (b >> 16) & 0xff; p[3] = b >> 24;
  }
}
__device__ __forceinline__ float load_f32_bytes(const uint8_t *p) {
  if ((reinterpret_cast<uintptr_t>(p) & 3) == 0) return *reinterpret_cast<const float *>(p);
  uint32_t b = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
  return __uint_as_float(b);
}

}  // namespace cc
