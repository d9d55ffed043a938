// launch_group_c128.cu -- k_group_t instantiations for double2 (see launch.cuh)
#include "launch_group.inl"

namespace tnb {
template bool try_launch_group<double2>(const GDesc&, cudaStream_t);
}  // namespace tnb
