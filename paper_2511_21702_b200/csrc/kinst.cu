// Explicit instantiations of the step kernel, one weight dtype / row plan per
// translation unit (compiled in parallel by build.py with -DKI_ET, -DKI_CPL,
// -DKI_Q); csvd_b200.cu declares them `extern template`.
#include "headstep.cuh"

#if KI_CPL > 0
template __global__ void k_step<KI_ET, KI_CPL, KI_Q, KI_CPL, KI_Q>(const __grid_constant__ Dev);
#endif
template __global__ void k_step<KI_ET, KI_CPL, KI_Q, 0, 0>(const __grid_constant__ Dev);
#if KI_CPL > 0
template __global__ void k_dense_gemv<KI_ET, KI_CPL, KI_Q>(const __grid_constant__ Dev);
template __global__ void k_step<KI_ET, KI_CPL, KI_Q, KI_CPL, KI_Q, true>(const __grid_constant__ Dev);  // grouped batch lanes
#endif
#if KI_CPL == 8
template __global__ void k_head<KI_ET, KI_Q>(const __grid_constant__ Dev);  // the head step
template __global__ void k_head_lanes<KI_ET, KI_Q>(const __grid_constant__ Dev);  // head step per batch lane
#endif
