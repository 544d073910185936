// Instantiates the sparse (SELL) engine with storage float, arithmetic float.
#include "gadi_host.cuh"

namespace gadi_host {
GADI_ENGINE_FACTORY(make_engine_csr_f32) {
  return new Engine<Sell<float>, float, float>(h, sp, a, om, ur, acc);
}
}  // namespace gadi_host
