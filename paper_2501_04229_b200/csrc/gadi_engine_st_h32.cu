// Instantiates the Stencil7 engine with storage __half, arithmetic float.
#include "gadi_host.cuh"

namespace gadi_host {
GADI_ENGINE_FACTORY(make_engine_st_h32) {
  return new Engine<Stencil7<float>, __half, float>(h, sp, a, om, ur, acc);
}
}  // namespace gadi_host
