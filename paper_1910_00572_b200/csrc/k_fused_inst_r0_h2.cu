// One (R, H) instantiation of the fused step kernels (see k_fused.cuh).
#include "k_fused.cuh"

namespace glb {
namespace fk {
template void launch_rh<0, 2>(gl_context*, const CUtensorMap* const*, FusedParams&, bool, bool, bool);
}  // namespace fk
}  // namespace glb
