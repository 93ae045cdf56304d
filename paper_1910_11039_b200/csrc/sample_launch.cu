// Instantiations of the sampling kernel for ONE block size (EBC_SHAPE_BLOCK, set by the build) and 1, 2 or 4
// adjacency slots per thread, with and without visited bitmaps.  Compiled once per block size so that the
// fifteen shapes build in parallel; nothing here but the launches.
#include "sample_launch.hpp"
// the kernels twice: with the statistics (work counters, records, paths, state dumps) and without (see the header)
#define EBC_STATS 1
#include "sampler_kernels.cuh"
#undef EBC_STATS
#define EBC_STATS 0
#include "sampler_kernels.cuh"
#undef EBC_STATS

#ifndef EBC_SHAPE_BLOCK
#error "compile with -DEBC_SHAPE_BLOCK=32|64|128|256|512"
#endif

namespace ebc {

#define EBC_CAT2(a, b) a##b
#define EBC_CAT(a, b) EBC_CAT2(a, b)

// Graphs with fixed-stride rows (SamplerParams::ell) have a kernel of their own: one per block size up to 128 threads
// (the adjacency slots per thread of the general expansion mean nothing there).
#if EBC_SHAPE_BLOCK <= 128
#define EBC_HAVE_FIXED 1
#else
#define EBC_HAVE_FIXED 0
#endif

template <int ITEMS> static void launch_one(const SamplerParams &p, u32 grid, cudaStream_t stream) {
    const bool stats = (p.flags & kFlagStats) != 0;
#if EBC_HAVE_FIXED
    if (p.ell) { // (rows of eight or of four entries: SamplerParams::ell_width)
        if (p.ell_width == kEllNarrow) {
            if (stats)
                with_stats::sample_kernel<EBC_SHAPE_BLOCK, 2, false, kEllNarrow><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
            else
                lean::sample_kernel<EBC_SHAPE_BLOCK, 2, false, kEllNarrow><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
        } else {
            if (stats)
                with_stats::sample_kernel<EBC_SHAPE_BLOCK, 2, false, kEllWidth><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
            else
                lean::sample_kernel<EBC_SHAPE_BLOCK, 2, false, kEllWidth><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
        }
        return;
    }
#endif
    if (p.flags & kFlagUseBitmap) {
        if (stats)
            with_stats::sample_kernel<EBC_SHAPE_BLOCK, ITEMS, true><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
        else
            lean::sample_kernel<EBC_SHAPE_BLOCK, ITEMS, true><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
    } else {
        if (stats)
            with_stats::sample_kernel<EBC_SHAPE_BLOCK, ITEMS, false><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
        else
            lean::sample_kernel<EBC_SHAPE_BLOCK, ITEMS, false><<<grid, EBC_SHAPE_BLOCK, 0, stream>>>(p);
    }
}

bool EBC_CAT(launch_sample_b, EBC_SHAPE_BLOCK)(u32 items, const SamplerParams &p, u32 grid, cudaStream_t stream) {
    switch (items) {
    case 1: launch_one<1>(p, grid, stream); return true;
    case 2: launch_one<2>(p, grid, stream); return true;
    case 4: launch_one<4>(p, grid, stream); return true;
    default: return false;
    }
}

template <int ITEMS> static int occupancy_one() {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, with_stats::sample_kernel<EBC_SHAPE_BLOCK, ITEMS, true>, EBC_SHAPE_BLOCK, 0) !=
        cudaSuccess)
        return -2;
    return per_sm;
}

int EBC_CAT(sample_occupancy_b, EBC_SHAPE_BLOCK)(u32 items, bool fixed_rows) {
    if (fixed_rows) {
#if EBC_HAVE_FIXED
        int per_sm = 0;
        int narrow = 0; // (both row widths must fit: the width is known only once the rows are built)
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, with_stats::sample_kernel<EBC_SHAPE_BLOCK, 2, false, kEllWidth>,
                                                          EBC_SHAPE_BLOCK, 0) != cudaSuccess ||
            cudaOccupancyMaxActiveBlocksPerMultiprocessor(&narrow, with_stats::sample_kernel<EBC_SHAPE_BLOCK, 2, false, kEllNarrow>,
                                                          EBC_SHAPE_BLOCK, 0) != cudaSuccess)
            return -2;
        return per_sm < narrow ? per_sm : narrow;
#else
        return -1;
#endif
    }
    switch (items) {
    case 1: return occupancy_one<1>();
    case 2: return occupancy_one<2>();
    case 4: return occupancy_one<4>();
    default: return -1;
    }
}

} // namespace ebc
