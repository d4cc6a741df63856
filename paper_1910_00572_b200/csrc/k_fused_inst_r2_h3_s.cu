// One (R, H, parameter block) instantiation of the fused step kernels
// (see k_fused.cuh): compiled as its own translation unit so the build runs
// them in parallel.
#include "k_fused.cuh"

namespace glb {
namespace fk {
template void launch_rh<2, 3, FusedParamsSmall>(gl_context*, const CUtensorMap* const*, FusedParamsSmall&, bool, bool, bool);
}  // namespace fk
}  // namespace glb
