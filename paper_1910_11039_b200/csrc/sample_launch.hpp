// Entry points of the separately compiled sampling-kernel instantiations (sample_launch.cu).
#pragma once

#include <cuda_runtime.h>

#include "device_types.cuh"

namespace ebc {

// launch_sample_b<BLOCK>(items, ...): launches sample_kernel<BLOCK, items, bitmap?>; false if `items` is not one
// of 1, 2, 4 (a graph with fixed-stride rows, p.ell, gets the kernel written for them).
// sample_occupancy_b<BLOCK>(items, fixed_rows): resident CTAs per SM, -1 for unknown items, -2 on a CUDA error.
#define EBC_DECLARE_SHAPE_GROUP(B)                                                                        \
    bool launch_sample_b##B(u32 items, const SamplerParams &p, u32 grid, cudaStream_t stream);           \
    int sample_occupancy_b##B(u32 items, bool fixed_rows);
EBC_DECLARE_SHAPE_GROUP(32)
EBC_DECLARE_SHAPE_GROUP(64)
EBC_DECLARE_SHAPE_GROUP(128)
EBC_DECLARE_SHAPE_GROUP(256)
EBC_DECLARE_SHAPE_GROUP(512)
#undef EBC_DECLARE_SHAPE_GROUP

} // namespace ebc
