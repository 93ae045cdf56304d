// TEST INFRASTRUCTURE (oracle side) -- not part of the shipped product.
//
// C wrapper around the UNMODIFIED reference sources
//   /root/reference/proj/src/{sampler,stopping,graph}.cpp
// compiled against oracle/shim/epochbc/rng.hpp (Philox stream instead of
// mt19937_64).  Built by oracle/Makefile into oracle/_ref/libebc_ref_shim.so;
// no reference source is copied into this repository.
//
// The wrapper re-keys the stream per sample exactly as SURVEY.md section 8c
// prescribes: draw 0 = below(n) (s), draw 1.. = below(n-1) (t), then the
// draws sample_shortest_path makes (sampler.cpp:124,142).
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

// Read-only peek at SearchScratch internals (dist / sigma / stamp dumps for
// the parity tests).  Layout is unaffected by access specifiers.
#define private public
#include "epochbc/sampler.hpp"
#undef private
#include "epochbc/graph.hpp"
#include "epochbc/stopping.hpp"

using namespace epochbc;

namespace {
struct ShimGraph {
    Graph g;
    std::unique_ptr<SearchScratch> scratch;
    PathSample sample;
};
thread_local char g_err[512];
void set_err(const char *what) {
    std::strncpy(g_err, what, sizeof(g_err) - 1);
    g_err[sizeof(g_err) - 1] = 0;
}
} // namespace

#pragma GCC visibility push(default)
extern "C" {

const char *refshim_last_error() { return g_err; }

// Builds the reference Graph through Graph::from_edges (graph.cpp:14-46) from a
// symmetric CSR; returns nullptr on failure.
void *refshim_graph_from_csr(std::uint64_t n, const std::uint64_t *offsets,
                             const std::uint32_t *targets) {
    try {
        std::vector<std::pair<Vertex, Vertex>> edges;
        edges.reserve(offsets[n] / 2);
        for (std::uint64_t u = 0; u < n; ++u)
            for (std::uint64_t i = offsets[u]; i < offsets[u + 1]; ++i)
                if (u < targets[i])
                    edges.emplace_back(u, targets[i]);
        auto *h = new ShimGraph;
        h->g = Graph::from_edges(n, std::move(edges));
        h->scratch = std::make_unique<SearchScratch>(n);
        return h;
    } catch (const std::exception &e) {
        set_err(e.what());
        return nullptr;
    }
}

void refshim_graph_free(void *h) { delete static_cast<ShimGraph *>(h); }

std::uint64_t refshim_graph_n(void *h) { return static_cast<ShimGraph *>(h)->g.num_vertices(); }
std::uint64_t refshim_graph_m(void *h) { return static_cast<ShimGraph *>(h)->g.num_edges(); }

// Exports the reference CSR (rows sorted ascending) so tests can check the
// product's canonicalisation against Graph::from_edges.
void refshim_graph_csr(void *h, std::uint64_t *offsets, std::uint64_t *targets) {
    auto *sg = static_cast<ShimGraph *>(h);
    std::memcpy(offsets, sg->g.offsets().data(), sizeof(std::uint64_t) * sg->g.offsets().size());
    std::memcpy(targets, sg->g.targets().data(), sizeof(std::uint64_t) * sg->g.targets().size());
}

// One sample with the stream keyed (seed, tag, index).  If explicit_pair != 0
// the given (s,t) are used and NO pair draws are consumed (test hook: draws
// start at 0 inside sample_shortest_path); otherwise sample_pair runs first.
// path_out must hold path_cap vertices; returns the internal length, or -1.
// info_out (may be null): [0]=s [1]=t [2]=draws consumed.
std::int64_t refshim_sample(void *h, std::uint64_t seed, std::uint32_t tag, std::uint64_t index,
                            int explicit_pair, std::uint64_t s, std::uint64_t t,
                            std::uint32_t *path_out, std::uint64_t path_cap,
                            std::uint64_t *info_out) {
    auto *sg = static_cast<ShimGraph *>(h);
    try {
        Rng rng(seed);
        rng.rekey(seed, tag, index);
        if (!explicit_pair) {
            auto p = sample_pair(sg->g.num_vertices(), rng);
            s = p.first;
            t = p.second;
        }
        sample_shortest_path(sg->g, s, t, *sg->scratch, rng, sg->sample);
        const auto &in = sg->sample.internal;
        if (in.size() > path_cap) {
            set_err("refshim_sample: path buffer too small");
            return -1;
        }
        for (std::size_t i = 0; i < in.size(); ++i)
            path_out[i] = static_cast<std::uint32_t>(in[i]);
        if (info_out) {
            info_out[0] = s;
            info_out[1] = t;
            info_out[2] = rng.draws();
        }
        return static_cast<std::int64_t>(in.size());
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

// State of the LAST sample: per-side dist (0xffffffff where not visited in
// that sample) and sigma (0 where not visited).  side 0 = from s, 1 = from t.
void refshim_last_search_state(void *h, int side, std::uint32_t *dist_out,
                               std::uint64_t *sigma_out) {
    auto *sg = static_cast<ShimGraph *>(h);
    const auto &sd = side == 0 ? sg->scratch->fwd_ : sg->scratch->bwd_;
    const std::uint32_t cur = sg->scratch->round_;
    const std::uint64_t n = sg->g.num_vertices();
    for (std::uint64_t v = 0; v < n; ++v) {
        bool vis = sd.stamp[v] == cur;
        dist_out[v] = vis ? sd.dist[v] : 0xffffffffu;
        sigma_out[v] = vis ? sd.sigma[v] : 0;
    }
}

// Meet set of the last sample in the reference's order (sampler.cpp:109-113).
std::uint64_t refshim_last_meet(void *h, std::uint32_t *meet_out, std::uint64_t cap) {
    auto *sg = static_cast<ShimGraph *>(h);
    const auto &m = sg->scratch->meet_;
    for (std::size_t i = 0; i < m.size() && i < cap; ++i)
        meet_out[i] = static_cast<std::uint32_t>(m[i]);
    return m.size();
}

// Samples [first, first+count) applied with apply_sample (sampler.hpp:74-78)
// into a StateFrame (state_frame.hpp:14-42); frame_words has n+1 u64 and is
// ACCUMULATED into (StateFrame::add).
int refshim_accumulate(void *h, std::uint64_t seed, std::uint32_t tag, std::uint64_t first,
                       std::uint64_t count, std::uint64_t *frame_words) {
    auto *sg = static_cast<ShimGraph *>(h);
    try {
        const Vertex n = sg->g.num_vertices();
        StateFrame frame(n);
        Rng rng(seed);
        for (std::uint64_t i = 0; i < count; ++i) {
            rng.rekey(seed, tag, first + i);
            auto p = sample_pair(n, rng);
            sample_shortest_path(sg->g, p.first, p.second, *sg->scratch, rng, sg->sample);
            apply_sample(frame, sg->sample);
        }
        auto w = frame.words();
        for (std::size_t i = 0; i < w.size(); ++i)
            frame_words[i] += w[i];
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

std::uint64_t refshim_compute_omega(std::uint64_t vd, double eps, double delta) {
    return compute_omega(vd, eps, delta);
}

// calibrate (stopping.cpp:43-92); kind 0 = uniform, 1 = weighted.
int refshim_calibrate(const std::uint64_t *calib_words, std::uint64_t n, double delta, int kind,
                      double *delta_lower, double *delta_upper) {
    try {
        StateFrame f(n);
        auto w = f.words();
        for (std::size_t i = 0; i < w.size(); ++i)
            w[i] = calib_words[i];
        StoppingParams p;
        calibrate(f, delta, n, kind == 0 ? AllocatorKind::kUniform : AllocatorKind::kWeighted, p);
        std::memcpy(delta_lower, p.delta_lower.data(), sizeof(double) * n);
        std::memcpy(delta_upper, p.delta_upper.data(), sizeof(double) * n);
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

// check_stop (stopping.cpp:125-142); bound 0 = Hoeffding, 1 = empirical Bernstein.
// Returns 0/1, or -1 on a contract violation.
int refshim_check_stop(const std::uint64_t *words, std::uint64_t n, double eps, std::uint64_t omega,
                       const double *delta_lower, const double *delta_upper, int bound) {
    try {
        StateFrame f(n);
        auto w = f.words();
        for (std::size_t i = 0; i < w.size(); ++i)
            w[i] = words[i];
        StoppingParams p;
        p.eps = eps;
        p.omega = omega;
        p.delta_lower.assign(delta_lower, delta_lower + n);
        p.delta_upper.assign(delta_upper, delta_upper + n);
        return check_stop(f, p, bound == 0 ? BoundKind::kHoeffding : BoundKind::kEmpiricalBernstein)
                   ? 1
                   : 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

double refshim_bound(double b, double delta_v, std::uint64_t tau, int bound) {
    return f_bound(b, delta_v, 0, tau,
                   bound == 0 ? BoundKind::kHoeffding : BoundKind::kEmpiricalBernstein);
}

} // extern "C"
#pragma GCC visibility pop
