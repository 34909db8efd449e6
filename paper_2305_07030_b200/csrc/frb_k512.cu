// Relaxation kernels of 512-thread CTAs (see frb_relax.cuh).
#include "frb_relax.cuh"

namespace frb_tu {
int dispatch_512(const frb_batch* b, const frb_config* c, const frb_group& g, int32_t* q, cudaStream_t s, int k) {
  return dispatch_k<512>(b, c, g, q, s, k);
}
}  // namespace frb_tu
