// Instantiates the sparse (SELL) engine with storage __half, arithmetic float.
#include "gadi_host.cuh"

namespace gadi_host {
GADI_ENGINE_FACTORY(make_engine_csr_h32) {
  return new Engine<Sell<__half>, __half, float>(h, sp, a, om, ur, acc);
}
}  // namespace gadi_host
