// Work-ledger relaxation kernels (energy_check_interval > 0; see frb_relax.cuh).
#include "frb_relax.cuh"

namespace frb_tu {
int dispatch_energy(const frb_batch* batch, const frb_config* cfg, const frb_group& g, int32_t* q, cudaStream_t s,
                    int T, int ke) {
  if (g.fprv_global) {
    return ke <= 4   ? launch_group<4, 512, true, true>(batch, cfg, g, q, s, T)
           : ke <= 8 ? launch_group<8, 512, true, true>(batch, cfg, g, q, s, T)
                     : launch_group<16, 512, true, true>(batch, cfg, g, q, s, T);
  }
  return ke <= 4   ? launch_group<4, 512, false, true>(batch, cfg, g, q, s, T)
         : ke <= 8 ? launch_group<8, 512, false, true>(batch, cfg, g, q, s, T)
                   : launch_group<16, 512, false, true>(batch, cfg, g, q, s, T);
}
}  // namespace frb_tu
