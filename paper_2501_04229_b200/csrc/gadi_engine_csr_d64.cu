// Instantiates the sparse (SELL) engine with storage double, arithmetic double.
#include "gadi_host.cuh"

namespace gadi_host {
GADI_ENGINE_FACTORY(make_engine_csr_d64) {
  return new Engine<Sell<double>, double, double>(h, sp, a, om, ur, acc);
}
}  // namespace gadi_host
