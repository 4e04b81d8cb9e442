// Temporary: codecs not yet implemented on device report CC_ERR_UNSUPPORTED.
#include "cc_common.cuh"
#include "cc_internal.h"

namespace cc {


int64_t lowrank_workspace_bytes(int64_t, int64_t, int64_t) { return 0; }
int lowrank_encode(int, int64_t, int64_t, int64_t, int, const float *, const float *, uint8_t *, float *, void *,
                   int64_t, cudaStream_t) {
  set_error("low-rank not built");
  return CC_ERR_UNSUPPORTED;
}
int lowrank_decode(int, int, const int64_t *, int64_t, int64_t, const uint8_t *const *, int, float *const *,
                   cudaStream_t) {
  set_error("low-rank not built");
  return CC_ERR_UNSUPPORTED;
}

}  // namespace cc
