// Counter-based random stream of the sampling path (host + device).
//
// Replaces the reference's per-worker std::mt19937_64 (include/epochbc/rng.hpp:30-52)
// by Philox-4x32-10 so that a sample's draws depend only on
// (seed, phase tag, global sample index, draw number) and are identical on any
// number of GPUs.  Interface mirrors Rng: next_u64,
// next_below, next_double.
//
//   key     = (seed lo32, seed hi32)
//   counter = (draw, tag, index lo32, index hi32)
//   next_u64   = word0 | word1 << 32 of that block, then draw += 1
//   next_below = Lemire multiply-shift with rejection (unbiased)
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define EBC_HD __host__ __device__ __forceinline__
#else
#define EBC_HD inline
#endif

namespace ebc {

enum : std::uint32_t {
    kTagAdaptive = 0,    // adaptive-phase samples
    kTagCalibration = 1, // calibration samples (engine.cpp:46 kCalibrationSalt)
    kTagGenErdosRenyi = 0x1001,
    kTagGenRmat = 0x1002,
    kTagGenGridDelete = 0x1003,
    kTagGenGridShortcut = 0x1004,
};

EBC_HD std::uint32_t mulhi32(std::uint32_t a, std::uint32_t b) {
#if defined(__CUDA_ARCH__)
    return __umulhi(a, b);
#else
    return static_cast<std::uint32_t>((static_cast<std::uint64_t>(a) * b) >> 32);
#endif
}

struct Philox4 {
    std::uint32_t x, y, z, w;
};

EBC_HD Philox4 philox4x32_10(Philox4 c, std::uint32_t k0, std::uint32_t k1) {
    constexpr std::uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    constexpr std::uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int round = 0; round < 10; ++round) {
        const std::uint32_t hi0 = mulhi32(M0, c.x), lo0 = M0 * c.x;
        const std::uint32_t hi1 = mulhi32(M1, c.z), lo1 = M1 * c.z;
        c = Philox4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += W0;
        k1 += W1;
    }
    return c;
}

#if defined(__CUDACC__)
// Device code keeps ONE copy of the ten rounds per kernel: a sample makes a handful of draws, while the
// sampling kernel's instruction footprint is a measured bottleneck (profiles/r01_icache.txt).
__device__ __noinline__ static std::uint64_t philox_draw_device(std::uint32_t draw, std::uint32_t tag, std::uint32_t i0,
                                                                std::uint32_t i1, std::uint32_t k0, std::uint32_t k1) {
    const Philox4 r = philox4x32_10(Philox4{draw, tag, i0, i1}, k0, k1);
    return static_cast<std::uint64_t>(r.x) | (static_cast<std::uint64_t>(r.y) << 32);
}
// (0 - bound) % bound, the rejection threshold of next_below, out of line and compact.
// Restoring division, one bit per iteration: the threshold is needed with probability bound / 2^64.
__device__ __noinline__ static std::uint64_t lemire_threshold_device(std::uint64_t bound) {
    const std::uint64_t a = 0 - bound;
    std::uint64_t r = 0;
#pragma unroll 1
    for (int i = 63; i >= 0; --i) {
        const bool top = (r >> 63) != 0;
        r = (r << 1) | ((a >> i) & 1);
        if (top || r >= bound)
            r -= bound;
    }
    return r;
}
#endif

class SampleStream {
public:
    EBC_HD SampleStream(std::uint64_t seed, std::uint32_t tag, std::uint64_t index)
        : k0_(static_cast<std::uint32_t>(seed)), k1_(static_cast<std::uint32_t>(seed >> 32)), tag_(tag),
          i0_(static_cast<std::uint32_t>(index)), i1_(static_cast<std::uint32_t>(index >> 32)), draw_(0) {}

    EBC_HD std::uint64_t next_u64() {
#if defined(__CUDA_ARCH__)
        return philox_draw_device(draw_++, tag_, i0_, i1_, k0_, k1_);
#else
        const Philox4 r = philox4x32_10(Philox4{draw_, tag_, i0_, i1_}, k0_, k1_);
        ++draw_;
        return static_cast<std::uint64_t>(r.x) | (static_cast<std::uint64_t>(r.y) << 32);
#endif
    }

    // Both 64-bit halves of one block (generators only; counts as one draw).
    EBC_HD void next_u64x2(std::uint64_t &a, std::uint64_t &b) {
        const Philox4 r = philox4x32_10(Philox4{draw_, tag_, i0_, i1_}, k0_, k1_);
        ++draw_;
        a = static_cast<std::uint64_t>(r.x) | (static_cast<std::uint64_t>(r.y) << 32);
        b = static_cast<std::uint64_t>(r.z) | (static_cast<std::uint64_t>(r.w) << 32);
    }

    EBC_HD std::uint64_t next_below(std::uint64_t bound) {
        std::uint64_t x = next_u64();
        std::uint64_t hi = mul64hi(x, bound), lo = x * bound;
        if (lo < bound) {
#if defined(__CUDA_ARCH__)
            const std::uint64_t threshold = lemire_threshold_device(bound);
#else
            const std::uint64_t threshold = (0 - bound) % bound;
#endif
            while (lo < threshold) {
                x = next_u64();
                hi = mul64hi(x, bound);
                lo = x * bound;
            }
        }
        return hi;
    }

    EBC_HD double next_double() { return static_cast<double>(next_u64() >> 11) * (1.0 / 9007199254740992.0); }

    EBC_HD std::uint32_t draws() const { return draw_; }

    static EBC_HD std::uint64_t mul64hi(std::uint64_t a, std::uint64_t b) {
#if defined(__CUDA_ARCH__)
        return __umul64hi(a, b);
#else
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(a) * b) >> 64);
#endif
    }

private:
    std::uint32_t k0_, k1_, tag_, i0_, i1_, draw_;
};

} // namespace ebc
