// Instantiates the sparse (SELL) engine with storage __half, arithmetic __half.
#include "gadi_host.cuh"

namespace gadi_host {
GADI_ENGINE_FACTORY(make_engine_csr_h16) {
  return new Engine<Sell<__half>, __half, __half>(h, sp, a, om, ur, acc);
}
}  // namespace gadi_host
