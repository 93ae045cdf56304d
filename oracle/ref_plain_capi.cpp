// TEST INFRASTRUCTURE (oracle side) -- not part of the shipped product.
//
// C wrapper around the UNMODIFIED reference library objects
//   /root/reference/proj/src/{graph,bfs,rmat,oracle,sampler,stopping,epoch,sim_comm,engine,score_io}.cpp
// with the reference's own rng.hpp (std::mt19937_64).  Built by oracle/Makefile
// into oracle/_ref/libebc_ref_plain.so.  Used for
//   * pipeline-level / statistical parity (run_simulated, engine.cpp:405-434),
//   * exact betweenness on config 1 (brandes_exact, oracle.cpp:61-102),
//   * the diameter phase known answers (bfs.cpp:36-76),
//   * pinning the product's mt19937_64 + libstdc++ next_below restatement,
//   * the CPU baseline timed by bench.py (cpu_baseline.kind = "reference").
#include <cstdint>
#include <cstring>
#include <fstream>
#include <vector>

#include "epochbc/bfs.hpp"
#include "epochbc/engine.hpp"
#include "epochbc/graph.hpp"
#include "epochbc/oracle.hpp"
#include "epochbc/rmat.hpp"
#include "epochbc/rng.hpp"
#include "epochbc/sampler.hpp"
#include "epochbc/score_io.hpp"
#include "epochbc/stopping.hpp"

using namespace epochbc;

namespace {
thread_local char g_err[512];
void set_err(const char *what) {
    std::strncpy(g_err, what, sizeof(g_err) - 1);
    g_err[sizeof(g_err) - 1] = 0;
}
} // namespace

#pragma GCC visibility push(default)
extern "C" {

const char *refplain_last_error() { return g_err; }

void *refplain_graph_from_csr(std::uint64_t n, const std::uint64_t *offsets,
                              const std::uint32_t *targets) {
    try {
        std::vector<std::pair<Vertex, Vertex>> edges;
        edges.reserve(offsets[n] / 2);
        for (std::uint64_t u = 0; u < n; ++u)
            for (std::uint64_t i = offsets[u]; i < offsets[u + 1]; ++i)
                if (u < targets[i])
                    edges.emplace_back(u, targets[i]);
        return new Graph(Graph::from_edges(n, std::move(edges)));
    } catch (const std::exception &e) {
        set_err(e.what());
        return nullptr;
    }
}

// Graph::from_edges on a raw (possibly dirty) edge list: loops, duplicates and
// both orientations allowed (graph.cpp:14-46).
void *refplain_graph_from_edges(std::uint64_t n, const std::uint64_t *src, const std::uint64_t *dst,
                                std::uint64_t count) {
    try {
        std::vector<std::pair<Vertex, Vertex>> edges(count);
        for (std::uint64_t i = 0; i < count; ++i)
            edges[i] = {src[i], dst[i]};
        return new Graph(Graph::from_edges(n, std::move(edges)));
    } catch (const std::exception &e) {
        set_err(e.what());
        return nullptr;
    }
}

void *refplain_graph_load(const char *path) {
    try {
        return new Graph(load_graph_file(path));
    } catch (const std::exception &e) {
        set_err(e.what());
        return nullptr;
    }
}

int refplain_graph_save(void *g, const char *path, int binary) {
    try {
        save_graph_file(*static_cast<Graph *>(g), path, binary != 0);
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

void *refplain_lcc(void *g) {
    try {
        return new Graph(largest_connected_component(*static_cast<Graph *>(g)));
    } catch (const std::exception &e) {
        set_err(e.what());
        return nullptr;
    }
}

void refplain_graph_free(void *g) { delete static_cast<Graph *>(g); }
std::uint64_t refplain_graph_n(void *g) { return static_cast<Graph *>(g)->num_vertices(); }
std::uint64_t refplain_graph_m(void *g) { return static_cast<Graph *>(g)->num_edges(); }

void refplain_graph_csr(void *g, std::uint64_t *offsets, std::uint64_t *targets,
                        std::uint64_t *original_ids) {
    auto *gr = static_cast<Graph *>(g);
    std::memcpy(offsets, gr->offsets().data(), 8 * gr->offsets().size());
    std::memcpy(targets, gr->targets().data(), 8 * gr->targets().size());
    if (original_ids)
        std::memcpy(original_ids, gr->original_ids().data(), 8 * gr->original_ids().size());
}

// diameter_upper_bound (bfs.cpp:36-76): out = {upper, lower, vertex_diameter_bound}.
int refplain_diameter(void *g, int sweeps, std::uint64_t seed, std::uint64_t *out) {
    try {
        GraphStats st = diameter_upper_bound(*static_cast<Graph *>(g), sweeps, seed);
        out[0] = st.diameter_upper_bound;
        out[1] = st.diameter_lower_bound;
        out[2] = st.vertex_diameter_bound;
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

// bfs (bfs.cpp:9-34): dist_out[n]; out = {farthest, eccentricity, reached}.
int refplain_bfs(void *g, std::uint64_t source, std::uint32_t *dist_out, std::uint64_t *out) {
    try {
        BfsResult r = bfs(*static_cast<Graph *>(g), source);
        std::memcpy(dist_out, r.dist.data(), 4 * r.dist.size());
        out[0] = r.farthest;
        out[1] = r.eccentricity;
        out[2] = r.reached;
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

int refplain_brandes(void *g, int workers, double *scores_out) {
    try {
        ExactScores s = brandes_exact(*static_cast<Graph *>(g), workers);
        std::memcpy(scores_out, s.data(), 8 * s.size());
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

std::uint64_t refplain_compute_omega(std::uint64_t vd, double eps, double delta) {
    return compute_omega(vd, eps, delta);
}

std::uint64_t refplain_epoch_length(int ranks, int threads, double base, double exponent) {
    return epoch_length(ranks, threads, base, exponent);
}

// Rng::stream(master, rank, thread) (rng.hpp:19-36) -> count draws of
// next_below(bounds[i]) (bound 0 => next_u64).  Pins the product's
// restatement of mt19937_64 + libstdc++ uniform_int_distribution.
void refplain_rng_draws(std::uint64_t master, std::uint64_t rank, std::uint64_t thread,
                        const std::uint64_t *bounds, std::uint64_t count, std::uint64_t *out) {
    Rng rng = Rng::stream(master, rank, thread);
    for (std::uint64_t i = 0; i < count; ++i)
        out[i] = bounds[i] == 0 ? rng.next_u64() : rng.next_below(bounds[i]);
}

struct refplain_run_args {
    double eps, delta;
    std::uint64_t seed;
    int ranks, threads;
    int algo;      // 1 | 2
    int bound;     // 0 hoeffding | 1 eb
    int allocator; // 0 uniform | 1 weighted
    int real_clock;
    std::uint64_t omega_override;
    std::uint64_t calib_samples_per_worker;
    int diameter_sweeps;
    double sample_cost_ms;
};

struct refplain_run_stats {
    std::uint64_t epochs, samples, tau, omega, calibration_samples, discarded_samples, n0;
    std::uint64_t diameter_upper_bound, vertex_diameter_bound;
    double adaptive_s, diameter_s, calibration_s, transition_s, reduce_s, check_s, wall_s;
    double wall_ms;
};

// run_simulated (engine.cpp:405-434).  scores_out has n doubles.
int refplain_run(void *g, const refplain_run_args *a, double *scores_out,
                 refplain_run_stats *st) {
    try {
        RunConfig cfg;
        cfg.eps = a->eps;
        cfg.delta = a->delta;
        cfg.seed = a->seed;
        cfg.ranks = a->ranks;
        cfg.threads = a->threads;
        cfg.algo = a->algo == 1 ? Algo::kRankOnly : Algo::kEpochBased;
        cfg.bound = a->bound == 0 ? BoundKind::kHoeffding : BoundKind::kEmpiricalBernstein;
        cfg.allocator = a->allocator == 0 ? AllocatorKind::kUniform : AllocatorKind::kWeighted;
        cfg.omega_override = a->omega_override;
        if (a->calib_samples_per_worker)
            cfg.calib_samples_per_worker = a->calib_samples_per_worker;
        if (a->diameter_sweeps)
            cfg.diameter_sweeps = a->diameter_sweeps;
        cfg.sample_cost_ms = a->sample_cost_ms;
        SimOptions opts;
        opts.clock_mode = a->real_clock ? SimClockMode::kReal : SimClockMode::kVirtual;
        SimRunOutcome o = run_simulated(*static_cast<Graph *>(g), cfg, opts);
        std::memcpy(scores_out, o.result.scores.data(), 8 * o.result.scores.size());
        const RunStats &s = o.stats;
        st->epochs = s.epochs;
        st->samples = s.samples;
        st->tau = s.tau;
        st->omega = s.omega;
        st->calibration_samples = s.calibration_samples;
        st->discarded_samples = s.discarded_samples;
        st->n0 = s.n0;
        st->diameter_upper_bound = s.diameter_upper_bound;
        st->vertex_diameter_bound = s.vertex_diameter_bound;
        st->adaptive_s = s.adaptive_s;
        st->diameter_s = s.diameter_s;
        st->calibration_s = s.calibration_s;
        st->transition_s = s.transition_s;
        st->reduce_s = s.reduce_s;
        st->check_s = s.check_s;
        st->wall_s = s.wall_s;
        st->wall_ms = o.wall_ms;
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

// write_scores (score_io.cpp:12-21) with an explicit meta map.
int refplain_write_scores(const char *path, const std::uint64_t *ids, const double *scores, std::uint64_t n,
                          const char *const *keys, const char *const *values, std::uint64_t meta_count) {
    try {
        ScoreFile f;
        for (std::uint64_t i = 0; i < meta_count; ++i)
            f.meta[keys[i]] = values[i];
        f.vertex_ids.assign(ids, ids + n);
        f.scores.assign(scores, scores + n);
        std::ofstream out(path, std::ios::binary);
        write_scores(out, f);
        return out ? 0 : -1;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

// read_scores + compare_scores (score_io.cpp:23-52, 98-122): out = {max_abs_error, top10, top100},
// counts = {vertices_above_eps, vertices}.
int refplain_compare_files(const char *approx, const char *exact, double eps, double *out, std::uint64_t *counts) {
    try {
        std::ifstream a(approx, std::ios::binary), b(exact, std::ios::binary);
        if (!a || !b)
            throw std::runtime_error("cannot open score file");
        CompareReport r = compare_scores(read_scores(a), read_scores(b), eps);
        out[0] = r.max_abs_error;
        out[1] = r.top10_overlap;
        out[2] = r.top100_overlap;
        counts[0] = r.vertices_above_eps;
        counts[1] = r.vertices;
        return 0;
    } catch (const std::exception &e) {
        set_err(e.what());
        return -1;
    }
}

} // extern "C"
#pragma GCC visibility pop
