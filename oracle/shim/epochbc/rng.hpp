// TEST INFRASTRUCTURE (oracle side) -- not part of the shipped product.
//
// Stream shim: this header SHADOWS /root/reference/proj/include/epochbc/rng.hpp
// when oracle/shim is placed before the reference include directory on the
// compiler command line (every reference include is "epochbc/rng.hpp", so the
// first -I wins).  It supplies an epochbc::Rng with the same interface as the
// reference class (rng.hpp:30-52: ctor(seed), stream(), next_u64, next_below,
// next_double) but backed by the counter-based Philox stream of
// oracle/ebc_philox.h, so the UNMODIFIED reference sampler.cpp can be driven
// by the same random stream as the CUDA kernels.
//
// Never link objects compiled against this header together with objects
// compiled against the real rng.hpp (two different epochbc::Rng => ODR).
#pragma once

#include <cstdint>

#include "epochbc/types.hpp"
#include "../../ebc_philox.h"

namespace epochbc {

// Kept so reference translation units that call them still compile; these two
// are pure integer functions restated from the published splitmix64 scheme.
inline std::uint64_t splitmix64(std::uint64_t &state) {
    state += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

class Rng {
public:
    explicit Rng(std::uint64_t seed) { ebc_stream_init(&s_, seed, 0, 0); }

    // (master, rank, thread) -> a distinct (tag, index) lane of the same key.
    static Rng stream(std::uint64_t master, std::uint64_t rank, std::uint64_t thread) {
        Rng r(master);
        r.rekey(master, static_cast<std::uint32_t>(0x80000000u | (rank & 0xffff)), thread);
        return r;
    }

    // Shim-only: position the stream at draw 0 of (seed, tag, sample index).
    void rekey(std::uint64_t seed, std::uint32_t tag, std::uint64_t index) {
        ebc_stream_init(&s_, seed, tag, index);
    }
    std::uint32_t draws() const { return s_.draw; }

    std::uint64_t next_u64() { return ebc_stream_u64(&s_); }

    std::uint64_t next_below(std::uint64_t bound) {
        require(bound > 0, "Rng::next_below: bound must be positive");
        return ebc_stream_below(&s_, bound);
    }

    double next_double() { return ebc_stream_double(&s_); }

private:
    ebc_stream s_;
};

} // namespace epochbc
