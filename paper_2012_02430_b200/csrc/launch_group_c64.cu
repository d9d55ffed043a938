// launch_group_c64.cu -- k_group_t instantiations for float2 (see launch.cuh)
#include "launch_group.inl"

namespace tnb {
template bool try_launch_group<float2>(const GDesc&, cudaStream_t);
}  // namespace tnb
