// Generic protocol kernels used by the codecs whose encode needs the
// materialized target (top-k, low-rank): t = target(x, base, aux) and the
// state update base' / feedback' / ref' + StepRecord reductions
// (pipeline.py:99-120).  The 1/2/4-bit path never uses these: it fuses the
// same arithmetic into k_scale_vec / k_quant_vec.
#include "cc_common.cuh"
#include "cc_internal.h"

#include <algorithm>

namespace cc {

constexpr int kApplyBlocks = 592;  // fixed grid -> fixed reduction order

template <int MODE, typename XT>
__global__ void __launch_bounds__(256) k_target(const XT *__restrict__ x, const float *__restrict__ base,
                                                const float *__restrict__ aux, float *__restrict__ t, int64_t total) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const bool vec = ((reinterpret_cast<uintptr_t>(x) & (sizeof(XT) == 2 ? 7 : 15)) |
                    (reinterpret_cast<uintptr_t>(base) & 15) | (reinterpret_cast<uintptr_t>(aux) & 15) |
                    (reinterpret_cast<uintptr_t>(t) & 15)) == 0;
  if (vec) {  // 128-bit accesses, two quads per thread in flight
    const int64_t nq = total / 4;
    for (int64_t q0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q0 < nq; q0 += 2 * stride) {
      float4 xx[2], bb[2], aa[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t q = q0 + u * stride;
        xx[u] = bb[u] = aa[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (q < nq) {
          xx[u] = Act<XT>::load4(x + 4 * q);
          if constexpr (MODE == CC_WITH_FEEDBACK) bb[u] = *reinterpret_cast<const float4 *>(base + 4 * q);
          if constexpr (MODE != CC_NAIVE) aa[u] = *reinterpret_cast<const float4 *>(aux + 4 * q);
        }
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int64_t q = q0 + u * stride;
        if (q < nq)
          *reinterpret_cast<float4 *>(t + 4 * q) =
              make_float4(target_of<MODE>(xx[u].x, bb[u].x, aa[u].x), target_of<MODE>(xx[u].y, bb[u].y, aa[u].y),
                          target_of<MODE>(xx[u].z, bb[u].z, aa[u].z), target_of<MODE>(xx[u].w, bb[u].w, aa[u].w));
      }
    }
    for (int64_t e = 4 * nq + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
      const float xx = Act<XT>::load1(x + e);
      float bb = 0.f, aa = 0.f;
      if constexpr (MODE == CC_WITH_FEEDBACK) bb = base[e];
      if constexpr (MODE != CC_NAIVE) aa = aux[e];
      t[e] = target_of<MODE>(xx, bb, aa);
    }
    return;
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const float xx = Act<XT>::load1(x + e);
    float bb = 0.f, aa = 0.f;
    if constexpr (MODE == CC_WITH_FEEDBACK) bb = base[e];
    if constexpr (MODE != CC_NAIVE) aa = aux[e];
    t[e] = target_of<MODE>(xx, bb, aa);
  }
}

template <int MODE, typename XT>
__global__ void __launch_bounds__(256) k_apply(const XT *__restrict__ x, const float *__restrict__ t,
                                               const float *__restrict__ dec, float *__restrict__ base,
                                               float *__restrict__ aux, int64_t total, double *__restrict__ part) {
  __shared__ double se[8], st[8];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  double err = 0.0, tsq = 0.0;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += stride) {
    const float tt = t[e], d = dec[e];
    const double df = (double)d - (double)tt;
    err += df * df;
    tsq += (double)tt * (double)tt;
    if constexpr (MODE == CC_NAIVE) {
      base[e] = d;
    } else {
      base[e] = __fadd_rn(base[e], d);
      if constexpr (MODE == CC_WITH_FEEDBACK) aux[e] = __fsub_rn(tt, d);
      else aux[e] = Act<XT>::load1(x + e);
    }
  }
  err = warp_sum(err);
  tsq = warp_sum(tsq);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { se[w] = err; st[w] = tsq; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) { a += se[i]; b += st[i]; }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

// fixed-order parallel sum of the per-block partials (256 threads: strided
// per-thread sums, warp butterflies, warps in order)
__global__ void __launch_bounds__(256) k_sum_parts(int nparts, const double *__restrict__ part,
                                                   double *__restrict__ record) {
  __shared__ double sa[8], sb[8];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nparts; i += 256) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  a = warp_sum(a);
  b = warp_sum(b);
  if ((threadIdx.x & 31) == 0) {
    sa[threadIdx.x >> 5] = a;
    sb[threadIdx.x >> 5] = b;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double x = 0.0, y = 0.0;
    for (int w = 0; w < 8; ++w) {
      x += sa[w];
      y += sb[w];
    }
    record[0] = x;
    record[1] = y;
  }
}

int sum_parts(int nparts, const double *part, double *record, cudaStream_t st) {
  k_sum_parts<<<1, 256, 0, st>>>(nparts, part, record);
  count_launch();
  return cuda_status("sum_parts");
}

int residual_target(int mode, int64_t n, int64_t C, const void *x, int x_dtype, const float *base, const float *aux,
                    float *t, cudaStream_t st) {
  const int64_t total = n * C;
  const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), sm_count() * 8));
#define CC_T(MODE, XT) k_target<MODE, XT><<<blocks, 256, 0, st>>>((const XT *)x, base, aux, t, total)
  if (x_dtype == CC_F32) {
    if (mode == CC_WITH_FEEDBACK) CC_T(CC_WITH_FEEDBACK, float);
    else if (mode == CC_NO_FEEDBACK) CC_T(CC_NO_FEEDBACK, float);
    else CC_T(CC_NAIVE, float);
  } else {
    if (mode == CC_WITH_FEEDBACK) CC_T(CC_WITH_FEEDBACK, __nv_bfloat16);
    else if (mode == CC_NO_FEEDBACK) CC_T(CC_NO_FEEDBACK, __nv_bfloat16);
    else CC_T(CC_NAIVE, __nv_bfloat16);
  }
#undef CC_T
  count_launch();
  return cuda_status("residual_target");
}

int apply_decoded(int mode, int64_t n, int64_t C, const void *x, int x_dtype, const float *t, const float *dec,
                  float *base, float *aux, double *record, void *ws, int64_t ws_bytes, cudaStream_t st) {
  if (!ws || ws_bytes < (int64_t)(2 * sizeof(double) * kApplyBlocks)) {
    set_error("apply_decoded: workspace too small");
    return CC_ERR_ARG;
  }
  double *part = reinterpret_cast<double *>(ws);
  const int64_t total = n * C;
#define CC_A(MODE, XT) \
  k_apply<MODE, XT><<<kApplyBlocks, 256, 0, st>>>((const XT *)x, t, dec, base, aux, total, part)
  if (x_dtype == CC_F32) {
    if (mode == CC_WITH_FEEDBACK) CC_A(CC_WITH_FEEDBACK, float);
    else if (mode == CC_NO_FEEDBACK) CC_A(CC_NO_FEEDBACK, float);
    else CC_A(CC_NAIVE, float);
  } else {
    if (mode == CC_WITH_FEEDBACK) CC_A(CC_WITH_FEEDBACK, __nv_bfloat16);
    else if (mode == CC_NO_FEEDBACK) CC_A(CC_NO_FEEDBACK, __nv_bfloat16);
    else CC_A(CC_NAIVE, __nv_bfloat16);
  }
#undef CC_A
  k_sum_parts<<<1, 256, 0, st>>>(kApplyBlocks, part, record);
  count_launch(2);
  return cuda_status("apply_decoded");
}

}  // namespace cc
