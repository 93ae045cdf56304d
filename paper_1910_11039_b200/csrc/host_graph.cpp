// Host-side graph ingestion for the B200 KADABRA hot path: canonical CSR
// construction, largest connected component, the reference's two on-disk
// formats, and the seeded synthetic inputs of BASELINE.json's configs.
//
// Behavioural contract (what, not how) follows the reference:
//   Graph::from_edges            /root/reference/proj/src/graph.cpp:14-46
//   load_edge_list               graph.cpp:71-126
//   write_edge_list              graph.cpp:128-136
//   write_binary / load_binary   graph.cpp:166-202 ("EBCG" v1)
//   load_graph_file              graph.cpp:204-215
//   largest_connected_component  graph.cpp:229-290
//   gen_rmat quadrant convention rmat.cpp:24-42
// The implementation is different by design: arcs are packed into 64-bit keys
// (u << 32 | v) and sorted by a multi-threaded merge sort, rows are emitted
// straight from the sorted keys, and ids are 32-bit.
#include "host_common.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <sstream>
#include <thread>
#include <unordered_set>

#include "philox.cuh"

namespace ebc {

namespace {

unsigned worker_count(std::uint64_t items, std::uint64_t min_per_worker) {
    unsigned hw = std::thread::hardware_concurrency();
    if (hw == 0)
        hw = 1;
    hw = std::min(hw, 64u);
    std::uint64_t by_size = std::max<std::uint64_t>(1, items / std::max<std::uint64_t>(1, min_per_worker));
    return static_cast<unsigned>(std::min<std::uint64_t>(hw, by_size));
}

template <typename Fn> void parallel_blocks(std::uint64_t items, unsigned workers, Fn &&fn) {
    if (workers <= 1) {
        fn(0u, std::uint64_t{0}, items);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(workers);
    for (unsigned w = 0; w < workers; ++w) {
        std::uint64_t b = items * w / workers, e = items * (w + 1) / workers;
        pool.emplace_back([&fn, w, b, e] { fn(w, b, e); });
    }
    for (auto &t : pool)
        t.join();
}

// Chunked std::sort followed by rounds of pairwise merges.
void parallel_sort(std::vector<std::uint64_t> &keys) {
    const std::uint64_t count = keys.size();
    unsigned workers = worker_count(count, 1u << 16);
    if (workers <= 1) {
        std::sort(keys.begin(), keys.end());
        return;
    }
    std::vector<std::uint64_t> bounds(workers + 1);
    for (unsigned w = 0; w <= workers; ++w)
        bounds[w] = count * w / workers;
    parallel_blocks(count, workers, [&](unsigned, std::uint64_t b, std::uint64_t e) {
        std::sort(keys.begin() + b, keys.begin() + e);
    });
    std::vector<std::uint64_t> scratch(count);
    std::vector<std::uint64_t> *src = &keys, *dst = &scratch;
    while (bounds.size() > 2) {
        std::vector<std::uint64_t> next_bounds;
        std::vector<std::thread> pool;
        for (std::size_t i = 0; i + 1 < bounds.size(); i += 2) {
            std::uint64_t lo = bounds[i], mid = bounds[i + 1];
            std::uint64_t hi = i + 2 < bounds.size() ? bounds[i + 2] : mid;
            next_bounds.push_back(lo);
            pool.emplace_back([src, dst, lo, mid, hi] {
                std::merge(src->begin() + lo, src->begin() + mid, src->begin() + mid, src->begin() + hi,
                           dst->begin() + lo);
            });
        }
        next_bounds.push_back(count);
        for (auto &t : pool)
            t.join();
        std::swap(src, dst);
        bounds.swap(next_bounds);
    }
    if (src != &keys)
        keys.swap(scratch);
}

inline std::uint64_t arc_key(std::uint64_t u, std::uint64_t v) { return (u << 32) | v; }

} // namespace

// Host-only builds: no pinned memory (the product library links the strong definitions of pinned_pool.cpp).
__attribute__((weak)) void *pinned_alloc(std::size_t) { return nullptr; }
__attribute__((weak)) bool pinned_free(void *) { return false; }
__attribute__((weak)) void pinned_release_idle() {}

// Sorted unique arc keys -> CSR.  Because keys sort by (u, v), rows come out
// ascending with no further work.
HostGraph graph_from_arc_keys(std::uint64_t n, std::vector<std::uint64_t> &&keys_in) {
    if (n > (std::uint64_t{1} << 32))
        throw ConfigError("graph: more than 2^32 vertices are not supported (32-bit vertex ids)");
    std::vector<std::uint64_t> keys = std::move(keys_in);
    parallel_sort(keys);
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());

    HostGraph g;
    g.n = n;
    g.m = keys.size() / 2;
    g.offsets.assign(n + 1, 0);
    g.targets.resize(keys.size());
    unsigned workers = worker_count(keys.size(), 1u << 18);
    parallel_blocks(keys.size(), workers, [&](unsigned, std::uint64_t b, std::uint64_t e) {
        for (std::uint64_t i = b; i < e; ++i)
            g.targets[i] = static_cast<std::uint32_t>(keys[i]);
    });
    // offsets[u] = first key index with source >= u.
    std::uint64_t pos = 0;
    for (std::uint64_t u = 0; u <= n; ++u) {
        while (pos < keys.size() && (keys[pos] >> 32) < u)
            ++pos;
        g.offsets[u] = pos;
    }
    g.original_ids.resize(n);
    for (std::uint64_t v = 0; v < n; ++v)
        g.original_ids[v] = v;
    return g;
}

HostGraph graph_from_edges(std::uint64_t n, const std::uint64_t *src, const std::uint64_t *dst,
                           std::uint64_t count) {
    if (n > (std::uint64_t{1} << 32))
        throw ConfigError("graph: more than 2^32 vertices are not supported (32-bit vertex ids)");
    std::vector<std::uint64_t> keys;
    keys.reserve(count * 2);
    for (std::uint64_t i = 0; i < count; ++i) {
        const std::uint64_t u = src[i], v = dst[i];
        require(u < n && v < n, "from_edges: endpoint out of range");
        if (u == v)
            continue;
        keys.push_back(arc_key(u, v));
        keys.push_back(arc_key(v, u));
    }
    return graph_from_arc_keys(n, std::move(keys));
}

HostGraph graph_from_csr(std::uint64_t n, const std::uint64_t *offsets, const std::uint32_t *targets,
                         const std::uint64_t *original_ids, bool validate) {
    if (n > (std::uint64_t{1} << 32))
        throw ConfigError("graph: more than 2^32 vertices are not supported (32-bit vertex ids)");
    require(offsets != nullptr, "graph_from_csr: null offsets");
    require(offsets[0] == 0, "graph_from_csr: offsets[0] must be 0");
    HostGraph g;
    g.n = n;
    const std::uint64_t arcs = offsets[n];
    require(arcs % 2 == 0, "graph_from_csr: odd arc count (graph not symmetric)");
    require(arcs == 0 || targets != nullptr, "graph_from_csr: null targets");
    g.m = arcs / 2;
    // Copies run in parallel: for ~100 MB inputs the first-touch page faults of the destination dominate.
    g.offsets.resize(n + 1);
    g.targets.resize(arcs);
    g.original_ids.resize(n);
    parallel_blocks(n + 1, worker_count(n + 1, 1u << 18), [&](unsigned, std::uint64_t b, std::uint64_t e) {
        std::memcpy(g.offsets.data() + b, offsets + b, (e - b) * 8);
    });
    parallel_blocks(arcs, worker_count(arcs, 1u << 19), [&](unsigned, std::uint64_t b, std::uint64_t e) {
        std::memcpy(g.targets.data() + b, targets + b, (e - b) * 4);
    });
    parallel_blocks(n, worker_count(n, 1u << 18), [&](unsigned, std::uint64_t b, std::uint64_t e) {
        if (original_ids)
            std::memcpy(g.original_ids.data() + b, original_ids + b, (e - b) * 8);
        else
            for (std::uint64_t v = b; v < e; ++v)
                g.original_ids[v] = v;
    });
    if (validate) {
        // Offsets first, all of them: nothing below may index targets (or offsets[v]) through an unchecked value.
        for (std::uint64_t u = 0; u < n; ++u)
            if (g.offsets[u + 1] < g.offsets[u] || g.offsets[u + 1] > arcs)
                throw ConfigError("graph_from_csr: offsets not monotone or beyond offsets[n]");
        for (std::uint64_t u = 0; u < n; ++u) {
            for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i) {
                const std::uint32_t v = g.targets[i];
                if (v >= n)
                    throw ConfigError("graph_from_csr: target out of range");
                if (v == u)
                    throw ConfigError("graph_from_csr: self-loop");
                if (i > g.offsets[u] && g.targets[i - 1] >= v)
                    throw ConfigError("graph_from_csr: row not strictly ascending");
            }
        }
        for (std::uint64_t u = 0; u < n; ++u)
            for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i) {
                const std::uint32_t v = g.targets[i];
                auto b = g.targets.begin() + g.offsets[v], e = g.targets.begin() + g.offsets[v + 1];
                if (!std::binary_search(b, e, static_cast<std::uint32_t>(u)))
                    throw ConfigError("graph_from_csr: graph not symmetric");
            }
    }
    return g;
}

// ---------------------------------------------------------------- components ---
HostGraph graph_lcc(const HostGraph &g) {
    const std::uint64_t n = g.n;
    constexpr std::uint32_t kNone = 0xffffffffu;
    std::vector<std::uint32_t> comp(n, kNone);
    std::vector<std::uint32_t> stack;
    std::vector<std::uint64_t> size, min_orig;
    for (std::uint64_t s = 0; s < n; ++s) {
        if (comp[s] != kNone)
            continue;
        const std::uint32_t c = static_cast<std::uint32_t>(size.size());
        size.push_back(0);
        min_orig.push_back(UINT64_MAX);
        stack.clear();
        stack.push_back(static_cast<std::uint32_t>(s));
        comp[s] = c;
        while (!stack.empty()) {
            const std::uint32_t u = stack.back();
            stack.pop_back();
            ++size[c];
            min_orig[c] = std::min(min_orig[c], g.original_ids[u]);
            for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i) {
                const std::uint32_t v = g.targets[i];
                if (comp[v] == kNone) {
                    comp[v] = c;
                    stack.push_back(v);
                }
            }
        }
    }
    // Largest; ties toward the component holding the smallest original id (graph.cpp:262-267).
    std::uint32_t best = 0;
    for (std::uint32_t c = 1; c < size.size(); ++c)
        if (size[c] > size[best] || (size[c] == size[best] && min_orig[c] < min_orig[best]))
            best = c;

    HostGraph out;
    if (n == 0)
        return out;
    std::vector<std::uint32_t> dense(n, 0);
    std::uint64_t kept = 0;
    for (std::uint64_t v = 0; v < n; ++v)
        if (comp[v] == best) {
            dense[v] = static_cast<std::uint32_t>(kept++);
            out.original_ids.push_back(g.original_ids[v]);
        }
    // The remap is monotone, so rows stay sorted and the CSR can be emitted directly.
    out.n = kept;
    out.offsets.assign(kept + 1, 0);
    std::uint64_t arcs = 0;
    for (std::uint64_t v = 0; v < n; ++v)
        if (comp[v] == best) {
            arcs += g.degree(v);
            out.offsets[dense[v] + 1] = arcs;
        }
    out.targets.resize(arcs);
    out.m = arcs / 2;
    for (std::uint64_t v = 0; v < n; ++v)
        if (comp[v] == best) {
            std::uint64_t o = out.offsets[dense[v]];
            for (std::uint64_t i = g.offsets[v]; i < g.offsets[v + 1]; ++i)
                out.targets[o++] = dense[g.targets[i]];
        }
    return out;
}

// ------------------------------------------------------------------- file I/O ---
namespace {

constexpr char kMagic[4] = {'E', 'B', 'C', 'G'};
constexpr std::uint32_t kBinaryVersion = 1;

bool blank_or_comment(const std::string &line) {
    for (char c : line) {
        if (c == ' ' || c == '\t' || c == '\r')
            continue;
        return c == '#' || c == '%';
    }
    return true;
}

HostGraph load_text(std::istream &in) {
    std::vector<std::uint64_t> a, b;
    std::string line;
    std::uint64_t lineno = 0;
    while (std::getline(in, line)) {
        ++lineno;
        if (blank_or_comment(line))
            continue;
        std::istringstream ls(line);
        std::uint64_t u, v;
        if (!(ls >> u >> v))
            throw ParseError("edge list: malformed line " + std::to_string(lineno) + ": '" + line + "'");
        std::string weight;
        ls >> weight;
        if (!weight.empty()) {
            std::string extra;
            if (ls >> extra)
                throw ParseError("edge list: too many fields on line " + std::to_string(lineno));
            for (char c : weight) {
                const bool numeric = (c >= '0' && c <= '9') || c == '.' || c == '-' || c == '+' ||
                                     c == 'e' || c == 'E';
                if (!numeric)
                    throw ParseError("edge list: malformed token on line " + std::to_string(lineno) +
                                     ": '" + weight + "'");
            }
        }
        a.push_back(u);
        b.push_back(v);
    }
    if (a.empty())
        throw ParseError("edge list: no edges in input");
    std::vector<std::uint64_t> ids;
    ids.reserve(a.size() * 2);
    ids.insert(ids.end(), a.begin(), a.end());
    ids.insert(ids.end(), b.begin(), b.end());
    std::sort(ids.begin(), ids.end());
    ids.erase(std::unique(ids.begin(), ids.end()), ids.end());
    for (std::size_t i = 0; i < a.size(); ++i) {
        a[i] = static_cast<std::uint64_t>(std::lower_bound(ids.begin(), ids.end(), a[i]) - ids.begin());
        b[i] = static_cast<std::uint64_t>(std::lower_bound(ids.begin(), ids.end(), b[i]) - ids.begin());
    }
    HostGraph g = graph_from_edges(ids.size(), a.data(), b.data(), a.size());
    if (g.m == 0)
        throw ParseError("edge list: graph has no edges after removing self-loops");
    g.original_ids.assign(ids.begin(), ids.end());
    return g;
}

template <typename T> T read_pod(std::istream &in, const char *what) {
    T v{};
    in.read(reinterpret_cast<char *>(&v), sizeof(T));
    if (!in)
        throw ParseError(what);
    return v;
}

std::vector<std::uint64_t> read_u64_array(std::istream &in) {
    const std::uint64_t len = read_pod<std::uint64_t>(in, "binary graph: truncated input");
    std::vector<std::uint64_t> v;
    try {
        v.resize(len);
    } catch (const std::exception &) {
        throw ParseError("binary graph: truncated array");
    }
    in.read(reinterpret_cast<char *>(v.data()), static_cast<std::streamsize>(8 * len));
    if (!in)
        throw ParseError("binary graph: truncated array");
    return v;
}

HostGraph load_ebcg(std::istream &in) {
    char magic[4] = {0, 0, 0, 0};
    in.read(magic, 4);
    if (!in || std::memcmp(magic, kMagic, 4) != 0)
        throw ParseError("binary graph: bad magic");
    const auto version = read_pod<std::uint32_t>(in, "binary graph: truncated input");
    if (version != kBinaryVersion)
        throw ParseError("binary graph: unsupported version " + std::to_string(version));
    const auto n = read_pod<std::uint64_t>(in, "binary graph: truncated input");
    const auto m = read_pod<std::uint64_t>(in, "binary graph: truncated input");
    std::vector<std::uint64_t> offsets = read_u64_array(in);
    std::vector<std::uint64_t> targets = read_u64_array(in);
    std::vector<std::uint64_t> ids = read_u64_array(in);
    if (offsets.size() != n + 1 || targets.size() != 2 * m || ids.size() != n)
        throw ParseError("binary graph: inconsistent array sizes");
    // Re-establish every invariant from the arcs, as the reference does (graph.cpp:190-201).
    std::vector<std::uint64_t> keys;
    keys.reserve(targets.size());
    for (std::uint64_t u = 0; u < n; ++u) {
        if (offsets[u + 1] < offsets[u] || offsets[u + 1] > targets.size())
            throw ParseError("binary graph: inconsistent array sizes");
        for (std::uint64_t i = offsets[u]; i < offsets[u + 1]; ++i) {
            const std::uint64_t v = targets[i];
            require(v < n, "from_edges: endpoint out of range");
            if (u < v) {
                keys.push_back(arc_key(u, v));
                keys.push_back(arc_key(v, u));
            }
        }
    }
    HostGraph g = graph_from_arc_keys(n, std::move(keys));
    g.original_ids.assign(ids.begin(), ids.end());
    return g;
}

} // namespace

HostGraph graph_load(const std::string &path) {
    std::ifstream in(path, std::ios::binary);
    if (!in)
        throw ParseError("cannot open graph file: " + path);
    char magic[4] = {0, 0, 0, 0};
    in.read(magic, 4);
    const bool binary = in && std::memcmp(magic, kMagic, 4) == 0;
    in.clear();
    in.seekg(0);
    return binary ? load_ebcg(in) : load_text(in);
}

void graph_save(const HostGraph &g, const std::string &path, bool binary) {
    std::ofstream out(path, std::ios::binary);
    if (!out)
        throw ParseError("cannot open output file: " + path);
    if (binary) {
        auto put_u64 = [&](std::uint64_t v) { out.write(reinterpret_cast<const char *>(&v), 8); };
        out.write(kMagic, 4);
        out.write(reinterpret_cast<const char *>(&kBinaryVersion), 4);
        put_u64(g.n);
        put_u64(g.m);
        put_u64(g.offsets.size());
        out.write(reinterpret_cast<const char *>(g.offsets.data()),
                  static_cast<std::streamsize>(8 * g.offsets.size()));
        put_u64(g.targets.size()); // on disk targets are u64 (graph.cpp:166-174)
        std::vector<std::uint64_t> wide(1u << 16);
        for (std::uint64_t i = 0; i < g.targets.size(); i += wide.size()) {
            const std::uint64_t k = std::min<std::uint64_t>(wide.size(), g.targets.size() - i);
            for (std::uint64_t j = 0; j < k; ++j)
                wide[j] = g.targets[i + j];
            out.write(reinterpret_cast<const char *>(wide.data()), static_cast<std::streamsize>(8 * k));
        }
        put_u64(g.original_ids.size());
        out.write(reinterpret_cast<const char *>(g.original_ids.data()),
                  static_cast<std::streamsize>(8 * g.original_ids.size()));
    } else {
        for (std::uint64_t u = 0; u < g.n; ++u)
            for (std::uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i)
                if (u < g.targets[i])
                    out << g.original_ids[u] << ' ' << g.original_ids[g.targets[i]] << '\n';
    }
    if (!out)
        throw ParseError("failed writing graph file: " + path);
}

// ----------------------------------------------------------------- generators ---
// G(n, m): the first m distinct non-loop unordered pairs of the candidate
// stream i = 0, 1, 2, ...; candidate i = (below(n), below(n)) of stream
// (seed, kTagGenErdosRenyi, i).
HostGraph gen_erdos_renyi(std::uint64_t n, std::uint64_t m, std::uint64_t seed) {
    if (n < 2)
        throw ConfigError("gen_erdos_renyi: need at least two vertices");
    if (n > (std::uint64_t{1} << 32))
        throw ConfigError("gen_erdos_renyi: n too large");
    const long double max_edges = static_cast<long double>(n) * (n - 1) / 2;
    if (static_cast<long double>(m) > max_edges)
        throw ConfigError("gen_erdos_renyi: more edges requested than the complete graph has");
    std::unordered_set<std::uint64_t> seen;
    seen.reserve(m * 2);
    std::vector<std::uint64_t> keys;
    keys.reserve(m * 2);
    for (std::uint64_t i = 0; seen.size() < m; ++i) {
        SampleStream st(seed, kTagGenErdosRenyi, i);
        std::uint64_t u = st.next_below(n), v = st.next_below(n);
        if (u == v)
            continue;
        if (u > v)
            std::swap(u, v);
        if (!seen.insert(arc_key(u, v)).second)
            continue;
        keys.push_back(arc_key(u, v));
        keys.push_back(arc_key(v, u));
    }
    return graph_from_arc_keys(n, std::move(keys));
}

// R-MAT: edge i descends `scale` quadrant levels; level b uses the b-th
// 53-bit uniform of stream (seed, kTagGenRmat, i) (two per Philox block).
// r < a: neither bit; r < a+b: target bit; r < a+b+c: source bit; else both.
HostGraph gen_rmat(int scale, int edge_factor, double a, double b, double c, double d,
                   std::uint64_t seed) {
    if (scale < 1 || scale > 30)
        throw ConfigError("gen_rmat: scale must be in [1, 30]");
    if (edge_factor < 1)
        throw ConfigError("gen_rmat: edge_factor must be positive");
    if (a < 0 || b < 0 || c < 0 || d < 0 || std::abs(a + b + c + d - 1.0) > 1e-9)
        throw ConfigError("gen_rmat: quadrant probabilities must be nonnegative and sum to 1");
    const std::uint64_t n = std::uint64_t{1} << scale;
    const std::uint64_t samples = static_cast<std::uint64_t>(edge_factor) * n;
    std::vector<std::uint64_t> keys(samples * 2);
    const double ab = a + b, abc = a + b + c;
    const double inv53 = 1.0 / 9007199254740992.0;
    parallel_blocks(samples, worker_count(samples, 1u << 14), [&](unsigned, std::uint64_t lo, std::uint64_t hi) {
        for (std::uint64_t i = lo; i < hi; ++i) {
            SampleStream st(seed, kTagGenRmat, i);
            std::uint64_t u = 0, v = 0, w0 = 0, w1 = 0;
            for (int bit = 0; bit < scale; ++bit) {
                if ((bit & 1) == 0)
                    st.next_u64x2(w0, w1);
                const double r = static_cast<double>(((bit & 1) ? w1 : w0) >> 11) * inv53;
                u <<= 1;
                v <<= 1;
                if (r < a) {
                } else if (r < ab) {
                    v |= 1;
                } else if (r < abc) {
                    u |= 1;
                } else {
                    u |= 1;
                    v |= 1;
                }
            }
            // Self-loops are filtered after generation (graph.cpp:20-21 drops them).
            keys[2 * i] = arc_key(u, v);
            keys[2 * i + 1] = arc_key(v, u);
        }
    });
    keys.erase(std::remove_if(keys.begin(), keys.end(),
                              [](std::uint64_t k) { return (k >> 32) == (k & 0xffffffffu); }),
               keys.end());
    return graph_from_arc_keys(n, std::move(keys));
}

// width x height 4-neighbour grid (vertex id = y*width + x).  Grid edge e is
// kept iff the first uniform of stream (seed, kTagGenGridDelete, e) >= delete_prob
// (edge ids: horizontal edges first in row-major order, then vertical).
// Then round(shortcut_fraction * #grid_edges) shortcut edges are added:
// shortcut j = first non-loop candidate pair of stream (seed, kTagGenGridShortcut, j).
HostGraph gen_grid(std::uint64_t w, std::uint64_t h, double delete_prob, double shortcut_fraction,
                   std::uint64_t seed) {
    if (w < 1 || h < 1 || w * h < 2)
        throw ConfigError("gen_grid: need at least two vertices");
    if (w * h > (std::uint64_t{1} << 32))
        throw ConfigError("gen_grid: too many vertices");
    if (!(delete_prob >= 0.0 && delete_prob < 1.0) || shortcut_fraction < 0.0)
        throw ConfigError("gen_grid: bad probabilities");
    const std::uint64_t n = w * h;
    const std::uint64_t horiz = (w - 1) * h, vert = w * (h - 1), grid_edges = horiz + vert;
    const std::uint64_t shortcuts = static_cast<std::uint64_t>(std::llround(shortcut_fraction * static_cast<double>(grid_edges)));
    std::vector<std::uint64_t> keys((grid_edges + shortcuts) * 2, UINT64_MAX);
    parallel_blocks(grid_edges, worker_count(grid_edges, 1u << 16), [&](unsigned, std::uint64_t lo, std::uint64_t hi) {
        for (std::uint64_t e = lo; e < hi; ++e) {
            SampleStream st(seed, kTagGenGridDelete, e);
            if (st.next_double() < delete_prob)
                continue;
            std::uint64_t u, v;
            if (e < horiz) {
                const std::uint64_t y = e / (w - 1), x = e % (w - 1);
                u = y * w + x;
                v = u + 1;
            } else {
                const std::uint64_t k = e - horiz;
                u = k;
                v = k + w;
            }
            keys[2 * e] = arc_key(u, v);
            keys[2 * e + 1] = arc_key(v, u);
        }
    });
    for (std::uint64_t j = 0; j < shortcuts; ++j) {
        SampleStream st(seed, kTagGenGridShortcut, j);
        std::uint64_t u, v;
        do {
            u = st.next_below(n);
            v = st.next_below(n);
        } while (u == v);
        keys[2 * (grid_edges + j)] = arc_key(u, v);
        keys[2 * (grid_edges + j) + 1] = arc_key(v, u);
    }
    keys.erase(std::remove(keys.begin(), keys.end(), UINT64_MAX), keys.end());
    return graph_from_arc_keys(n, std::move(keys));
}

void shard_range(std::uint64_t first, std::uint64_t count, int rank, int world,
                 std::uint64_t *shard_first, std::uint64_t *shard_count) {
    const std::uint64_t W = static_cast<std::uint64_t>(world < 1 ? 1 : world);
    const std::uint64_t r = static_cast<std::uint64_t>(rank < 0 ? 0 : rank);
    const std::uint64_t base = count / W, extra = count % W;
    const std::uint64_t lo = r * base + std::min(r, extra);
    *shard_first = first + lo;
    *shard_count = base + (r < extra ? 1 : 0);
}

} // namespace ebc
