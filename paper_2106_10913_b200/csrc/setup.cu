// GPU setup pipeline (placeholder until the batched setup kernels land).
#include "awg_internal.cuh"

namespace awgb {
void run_setup(Ctx& c, const awg_config& cfg) {
  (void)cfg;
  c.fail(AWG_E_STATE, "setup: device setup not built yet; use awg_load_factors");
}
}  // namespace awgb
