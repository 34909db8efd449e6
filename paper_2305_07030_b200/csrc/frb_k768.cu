// Relaxation kernels of 768-thread CTAs (see frb_relax.cuh).
#include "frb_relax.cuh"

namespace frb_tu {
int dispatch_768(const frb_batch* b, const frb_config* c, const frb_group& g, int32_t* q, cudaStream_t s, int k) {
  return dispatch_k<768>(b, c, g, q, s, k);
}
}  // namespace frb_tu
