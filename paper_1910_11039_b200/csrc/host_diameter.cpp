// Host side of the diameter phase (phase 1 of run_pipeline,
// /root/reference/proj/src/engine.cpp:298-311): queue BFS with the reference's
// farthest-vertex tie-break (bfs.cpp:9-34) and the mt19937_64 stream its
// random restarts are drawn from (bfs.cpp:46,61-65 via rng.hpp:19-46).  The
// sweep loop itself is the template in host_common.hpp so the device BFS can
// be plugged in.
#include "host_common.hpp"

namespace ebc {

BfsSummary host_bfs(const HostGraph &g, std::uint32_t source, std::uint32_t *dist_out) {
    require(source < g.n, "bfs: source out of range");
    constexpr std::uint32_t kFar = 0xffffffffu;
    std::vector<std::uint32_t> local;
    std::uint32_t *dist = dist_out;
    if (!dist) {
        local.resize(g.n);
        dist = local.data();
    }
    std::fill(dist, dist + g.n, kFar);
    std::vector<std::uint32_t> level{source}, next;
    dist[source] = 0;
    BfsSummary r;
    r.farthest = source;
    r.reached = 1;
    std::uint32_t depth = 0;
    // Level-synchronous; the farthest vertex with the lowest id equals the
    // reference's queue-order rule (max distance, lowest id on ties).
    while (!level.empty()) {
        next.clear();
        for (std::uint32_t u : level)
            for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i) {
                const std::uint32_t v = g.targets[i];
                if (dist[v] == kFar) {
                    dist[v] = depth + 1;
                    next.push_back(v);
                }
            }
        if (next.empty())
            break;
        ++depth;
        r.reached += next.size();
        r.eccentricity = depth;
        r.farthest = *std::min_element(next.begin(), next.end());
        level.swap(next);
    }
    return r;
}

DiameterBounds diameter_upper_bound_host(const HostGraph &g, int sweeps, std::uint64_t seed) {
    return diameter_upper_bound(g, sweeps, seed,
                                [&](std::uint32_t v) { return host_bfs(g, v, nullptr); });
}

// ---- mt19937_64 (Matsumoto & Nishimura 2000), the engine behind the reference Rng ----
namespace {
std::uint64_t splitmix_step(std::uint64_t &state) {
    state += 0x9e3779b97f4a7c15ULL;
    std::uint64_t z = state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
} // namespace

RefMtStream::RefMtStream(std::uint64_t master, std::uint64_t rank, std::uint64_t thread) {
    // mix_seed (rng.hpp:19-27)
    std::uint64_t s = master;
    std::uint64_t h = splitmix_step(s);
    s ^= rank * 0x2545f4914f6cdd1dULL;
    h ^= splitmix_step(s);
    s ^= thread * 0x9e3779b97f4a7c15ULL;
    h ^= splitmix_step(s);
    mt_[0] = h;
    for (int i = 1; i < 312; ++i)
        mt_[i] = 6364136223846793005ULL * (mt_[i - 1] ^ (mt_[i - 1] >> 62)) + static_cast<std::uint64_t>(i);
    idx_ = 312;
}

std::uint64_t RefMtStream::next_u64() {
    if (idx_ >= 312) {
        constexpr std::uint64_t kUpper = 0xFFFFFFFF80000000ULL, kLower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            const std::uint64_t x = (mt_[i] & kUpper) | (mt_[(i + 1) % 312] & kLower);
            mt_[i] = mt_[(i + 156) % 312] ^ (x >> 1) ^ ((x & 1) ? 0xB5026F5AA96619E9ULL : 0);
        }
        idx_ = 0;
    }
    std::uint64_t y = mt_[idx_++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

// std::uniform_int_distribution<uint64_t>(0, bound-1) over a full-range 64-bit
// engine in libstdc++ >= 11: Lemire's multiply-shift with rejection.
std::uint64_t RefMtStream::next_below(std::uint64_t bound) {
    require(bound > 0, "Rng::next_below: bound must be positive");
    unsigned __int128 m = static_cast<unsigned __int128>(next_u64()) * bound;
    std::uint64_t low = static_cast<std::uint64_t>(m);
    if (low < bound) {
        const std::uint64_t threshold = (0 - bound) % bound;
        while (low < threshold) {
            m = static_cast<unsigned __int128>(next_u64()) * bound;
            low = static_cast<std::uint64_t>(m);
        }
    }
    return static_cast<std::uint64_t>(m >> 64);
}

} // namespace ebc
