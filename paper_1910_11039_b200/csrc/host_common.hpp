// Host-side common types of the B200 KADABRA hot path: error classes mapped to
// ebc_status at the C ABI, and the immutable CSR graph (u64 offsets, u32
// targets) that is uploaded unchanged into HBM.
#pragma once

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace ebc {

// Same four classes as the reference (include/epochbc/types.hpp:15-36) plus CUDA.
struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ConfigError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct BackendFault : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct ContractViolation : std::logic_error {
    using std::logic_error::logic_error;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void require(bool cond, const char *what) {
    if (!cond)
        throw ContractViolation(what);
}

// Immutable undirected CSR; rows sorted ascending, symmetric, no loops or
// duplicates (the invariants of epochbc::Graph, graph.hpp:14-20).
// std::vector whose resize() leaves trivially constructible elements uninitialised, so large arrays
// can be filled (and their pages first touched) by several threads instead of being zeroed by one.
// Large graph arrays live in page-locked host memory when a CUDA device is present (pinned_pool.cpp):
// the CSR upload then runs at PCIe speed instead of through the driver's staging copies (config 2:
// 12 -> 4 ms of a 55 ms run).  Blocks are pooled per process, because cudaHostAlloc / cudaFreeHost are
// slow.  Both functions have weak no-op definitions in host_graph.cpp, so host-only builds (the CPU
// test harness) simply use the heap.
void *pinned_alloc(std::size_t bytes); // nullptr: use the heap
bool pinned_free(void *p);             // false: p did not come from pinned_alloc
void pinned_release_idle();            // frees the cached blocks (ebc_release_device_cache)
constexpr std::size_t kPinnedMinBytes = std::size_t{1} << 20;

template <class T> struct DefaultInitAllocator : std::allocator<T> {
    template <class U> struct rebind {
        using other = DefaultInitAllocator<U>;
    };
    DefaultInitAllocator() = default;
    template <class U> DefaultInitAllocator(const DefaultInitAllocator<U> &) noexcept {}
    T *allocate(std::size_t n) {
        const std::size_t bytes = n * sizeof(T);
        if (bytes >= kPinnedMinBytes)
            if (void *p = pinned_alloc(bytes))
                return static_cast<T *>(p);
        return static_cast<T *>(::operator new(bytes));
    }
    void deallocate(T *p, std::size_t n) noexcept {
        if (n * sizeof(T) >= kPinnedMinBytes && pinned_free(p))
            return;
        ::operator delete(p);
    }
    template <class U> void construct(U *p) noexcept { ::new (static_cast<void *>(p)) U; }
    template <class U, class... Args> void construct(U *p, Args &&...args) {
        ::new (static_cast<void *>(p)) U(std::forward<Args>(args)...);
    }
};
template <class T> using RawVector = std::vector<T, DefaultInitAllocator<T>>;

struct HostGraph {
    std::uint64_t n = 0;
    std::uint64_t m = 0; // undirected edges
    RawVector<std::uint64_t> offsets; // n+1
    RawVector<std::uint32_t> targets; // 2m
    RawVector<std::uint64_t> original_ids; // n

    std::uint64_t degree(std::uint64_t v) const { return offsets[v + 1] - offsets[v]; }
};

// host_graph.cpp
HostGraph graph_from_csr(std::uint64_t n, const std::uint64_t *offsets, const std::uint32_t *targets,
                         const std::uint64_t *original_ids, bool validate);
HostGraph graph_from_edges(std::uint64_t n, const std::uint64_t *src, const std::uint64_t *dst,
                           std::uint64_t count);
HostGraph graph_from_arc_keys(std::uint64_t n, std::vector<std::uint64_t> &&keys); // (u<<32|v), any order
HostGraph graph_load(const std::string &path);
void graph_save(const HostGraph &g, const std::string &path, bool binary);
HostGraph graph_lcc(const HostGraph &g);
HostGraph gen_erdos_renyi(std::uint64_t n, std::uint64_t m, std::uint64_t seed);
HostGraph gen_rmat(int scale, int edge_factor, double a, double b, double c, double d,
                   std::uint64_t seed);
HostGraph gen_grid(std::uint64_t w, std::uint64_t h, double delete_prob, double shortcut_fraction,
                   std::uint64_t seed);

// host_stopping.cpp
std::uint64_t compute_omega(std::uint64_t vd, double eps, double delta);
std::uint64_t epoch_length(int ranks, int threads, double base, double exponent);
void calibrate(const std::uint64_t *calib_words, std::uint64_t n, double delta, int allocator,
               double *delta_lower, double *delta_upper);
// ln(1/delta_v) (Hoeffding) or ln(2/delta_v) (empirical Bernstein), evaluated with the host libm.
void bound_log_terms(const double *delta_v, std::uint64_t n, int bound, double *out);
// Per-vertex, per-side failure probability of the uniform allocator (what calibrate() writes n times).
double calibrate_uniform_value(std::uint64_t n, double delta);

// host_diameter.cpp
struct BfsSummary {
    std::uint32_t farthest = 0;
    std::uint32_t eccentricity = 0;
    std::uint64_t reached = 0;
};
BfsSummary host_bfs(const HostGraph &g, std::uint32_t source, std::uint32_t *dist_or_null);
struct DiameterBounds {
    std::uint64_t upper = 0, lower = 0, vertex_diameter = 0;
};
// bfs_fn lets the device BFS be plugged in; it must return what host_bfs returns.
template <typename BfsFn> DiameterBounds diameter_upper_bound(const HostGraph &g, int sweeps, std::uint64_t seed, BfsFn &&bfs_fn);
DiameterBounds diameter_upper_bound_host(const HostGraph &g, int sweeps, std::uint64_t seed);

// mt19937_64 stream of the reference's Rng::stream(master, rank, thread)
// (rng.hpp:19-46), needed so the diameter phase's random restarts (bfs.cpp:46,
// 61-65) pick the same vertices as the reference.
class RefMtStream {
public:
    RefMtStream(std::uint64_t master, std::uint64_t rank, std::uint64_t thread);
    std::uint64_t next_u64();
    std::uint64_t next_below(std::uint64_t bound);

private:
    std::uint64_t mt_[312];
    int idx_;
};

void shard_range(std::uint64_t first, std::uint64_t count, int rank, int world,
                 std::uint64_t *shard_first, std::uint64_t *shard_count);

template <typename BfsFn>
DiameterBounds diameter_upper_bound(const HostGraph &g, int sweeps, std::uint64_t seed, BfsFn &&bfs_fn) {
    // Follows bfs.cpp:36-76.
    const std::uint64_t n = g.n;
    require(n >= 1, "diameter_upper_bound: empty graph");
    require(sweeps >= 1, "diameter_upper_bound: need at least one sweep");
    std::uint32_t start = 0;
    for (std::uint64_t v = 1; v < n; ++v)
        if (g.degree(v) > g.degree(start))
            start = static_cast<std::uint32_t>(v);
    RefMtStream rng(seed, 0, 0x00d1a0ULL);
    std::uint64_t upper = UINT64_MAX, lower = 0;
    std::vector<char> used(n, 0);
    std::uint32_t v = start;
    for (int i = 0; i < sweeps; ++i) {
        BfsSummary r = bfs_fn(v);
        if (r.reached != n)
            throw ConfigError("diameter_upper_bound: graph is disconnected");
        upper = std::min<std::uint64_t>(upper, 2ULL * r.eccentricity);
        lower = std::max<std::uint64_t>(lower, r.eccentricity);
        used[v] = 1;
        if (n == 1)
            break;
        v = r.farthest;
        for (int tries = 0; used[v] && tries < 16; ++tries)
            v = static_cast<std::uint32_t>(rng.next_below(n));
        if (used[v])
            break;
    }
    require(lower <= upper, "diameter bound: lower exceeds upper");
    DiameterBounds b;
    b.upper = upper;
    b.lower = lower;
    b.vertex_diameter = upper + 1;
    return b;
}

} // namespace ebc
