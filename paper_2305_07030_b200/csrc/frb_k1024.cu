// Relaxation kernels of 1024-thread CTAs (see frb_relax.cuh).
#include "frb_relax.cuh"

namespace frb_tu {
int dispatch_1024(const frb_batch* b, const frb_config* c, const frb_group& g, int32_t* q, cudaStream_t s, int k) {
  return dispatch_k<1024>(b, c, g, q, s, k);
}
}  // namespace frb_tu
