// K1 column-segment instantiations (cc_encode_step_segmented, the Ulysses sender):
// compiled separately from k1_fused.cu so the two halves build in parallel.
#include "k1_fused_impl.cuh"

namespace cc {

int fused_dispatch_seg(fused::Params &p, int codec, int mode, int x_dtype, int Q, cudaStream_t st) {
#define CC_FUSED_Q(MODE, CODEC, XT) \
  return Q == 2 ? launch_fused<MODE, CODEC, XT, 2, true>(p, st) : launch_fused<MODE, CODEC, XT, 1, true>(p, st)
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
