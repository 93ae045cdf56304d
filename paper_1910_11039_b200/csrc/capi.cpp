// C ABI of the B200 KADABRA hot path (include/ebc_b200.h).  Thin: argument
// checks, exception -> status mapping, handle ownership.  All sampling work is
// done by CudaSampler's kernels; nothing here computes on the CPU what the
// header says runs on the GPU.
#include "../../include/ebc_b200.h"

#include <dlfcn.h>

#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "cuda_sampler.hpp"
#include "device_graph.hpp"
#include "epoch_driver.hpp"
#include "host_common.hpp"
#include "host_scores.hpp"

using namespace ebc;

struct ebc_graph {
    HostGraph g;
};

struct ebc_result {
    RunOutput out;
};

struct ebc_scores {
    ScoreTable t;
};

struct ebc_sampler {
    std::unique_ptr<CudaSampler> s;
    ebc_allreduce_fn allreduce = nullptr;
    void *allreduce_user = nullptr;
};

namespace {

thread_local std::string g_last_error;

template <typename Fn> ebc_status guarded(Fn &&fn) {
    try {
        fn();
        return EBC_OK;
    } catch (const CudaError &e) {
        g_last_error = e.what();
        return EBC_ERR_CUDA;
    } catch (const BackendFault &e) {
        g_last_error = e.what();
        return EBC_ERR_BACKEND;
    } catch (const ParseError &e) {
        g_last_error = e.what();
        return EBC_ERR_PARSE;
    } catch (const ConfigError &e) {
        g_last_error = e.what();
        return EBC_ERR_CONFIG;
    } catch (const ContractViolation &e) {
        g_last_error = e.what();
        return EBC_ERR_CONFIG;
    } catch (const std::bad_alloc &) {
        g_last_error = "out of host memory";
        return EBC_ERR_PARSE;
    } catch (const std::exception &e) { // "other" maps to 3 like the reference CLI (epochbc.cpp:398-402)
        g_last_error = e.what();
        return EBC_ERR_PARSE;
    }
}

void need(const void *p, const char *what) {
    if (!p)
        throw ContractViolation(what);
}

SamplerOptions sampler_options(const ebc_run_config *cfg) {
    SamplerOptions o;
    if (cfg) {
        o.device = cfg->device;
        o.block_threads = cfg->block_threads;
        o.slots = cfg->slots;
        o.slot_capacity = cfg->slot_capacity;
        o.items_per_thread = cfg->items_per_thread;
        o.materialize_final_level = cfg->materialize_final_level != 0;
        o.renumber = cfg->renumber;
        o.work_counters = cfg->work_counters != 0;
        // the frame all-reduce of epoch e runs beside the sampling of epoch e+1 (see ebc_b200.h)
        o.reserved_sms = cfg->reserved_sms > 0 ? static_cast<std::uint32_t>(cfg->reserved_sms)
                         : cfg->reserved_sms == 0 && cfg->world_size > 1 && cfg->overlap ? 4u : 0u;
    }
    return o;
}

// SamplerBackend over the CUDA sampler: the only backend the product ships.
class CudaBackend final : public SamplerBackend {
public:
    explicit CudaBackend(CudaSampler &s) : s_(s) {}
    BfsSummary bfs(std::uint32_t source) override { return s_.bfs(source, nullptr); }
    void sample(std::uint64_t seed, std::uint32_t tag, std::uint64_t first, std::uint64_t count,
                int frame) override {
        s_.sample(seed, tag, first, count, frame);
    }
    void set_stopping(double eps, std::uint64_t omega, const double *dl, const double *du,
                      int bound) override {
        s_.set_stopping(eps, omega, dl, du, bound);
    }
    void set_stopping_uniform(double eps, std::uint64_t omega, double delta_each, std::uint64_t, int bound) override {
        s_.set_stopping_uniform(eps, omega, delta_each, bound);
    }
    void fold_async(int frame, AllreduceHook allreduce, void *user) override {
        s_.fold_and_check_async(frame, allreduce, user);
    }
    bool wait_fold(int frame, std::uint64_t *tau_out) override { return s_.wait_fold(frame, tau_out); }
    void discard_frame(int frame) override { s_.discard_frame(frame); }
    void read_state(std::uint64_t *words_out) override { s_.read_frame(2, words_out); }
    void clear() override { s_.clear(); }
    void finish(RunStats &st) override {
        s_.work(st.work, false);
        st.overflow_samples = s_.overflow_samples();
    }

private:
    CudaSampler &s_;
};

} // namespace

extern "C" {

const char *ebc_last_error(void) { return g_last_error.c_str(); }
const char *ebc_version(void) { return "ebc_b200 0.1 (sm_100a)"; }

// ------------------------------------------------------------------ graph ---
ebc_status ebc_graph_from_csr(uint64_t n, const uint64_t *offsets, const uint32_t *targets,
                              const uint64_t *original_ids, int validate, ebc_graph **out) {
    return guarded([&] {
        need(out, "ebc_graph_from_csr: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = graph_from_csr(n, offsets, targets, original_ids, validate != 0);
        *out = h.release();
    });
}

ebc_status ebc_graph_from_edges(uint64_t n, const uint64_t *src, const uint64_t *dst, uint64_t count,
                                ebc_graph **out) {
    return guarded([&] {
        need(out, "ebc_graph_from_edges: null out");
        if (count) {
            need(src, "ebc_graph_from_edges: null src");
            need(dst, "ebc_graph_from_edges: null dst");
        }
        auto h = std::make_unique<ebc_graph>();
        h->g = graph_from_edges(n, src, dst, count);
        *out = h.release();
    });
}

ebc_status ebc_graph_load(const char *path, int take_lcc, ebc_graph **out) {
    return guarded([&] {
        need(path, "ebc_graph_load: null path");
        need(out, "ebc_graph_load: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = graph_load(path);
        if (take_lcc)
            h->g = graph_lcc(h->g);
        *out = h.release();
    });
}

ebc_status ebc_graph_save(const ebc_graph *g, const char *path, int binary) {
    return guarded([&] {
        need(g, "ebc_graph_save: null graph");
        need(path, "ebc_graph_save: null path");
        graph_save(g->g, path, binary != 0);
    });
}

ebc_status ebc_graph_lcc(const ebc_graph *g, ebc_graph **out) {
    return guarded([&] {
        need(g, "ebc_graph_lcc: null graph");
        need(out, "ebc_graph_lcc: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = graph_lcc(g->g);
        *out = h.release();
    });
}

uint64_t ebc_graph_num_vertices(const ebc_graph *g) { return g ? g->g.n : 0; }
uint64_t ebc_graph_num_edges(const ebc_graph *g) { return g ? g->g.m : 0; }
const uint64_t *ebc_graph_offsets(const ebc_graph *g) { return g ? g->g.offsets.data() : nullptr; }
const uint32_t *ebc_graph_targets(const ebc_graph *g) { return g ? g->g.targets.data() : nullptr; }
const uint64_t *ebc_graph_original_ids(const ebc_graph *g) { return g ? g->g.original_ids.data() : nullptr; }
void ebc_graph_free(ebc_graph *g) { delete g; }

ebc_status ebc_gen_erdos_renyi(uint64_t n, uint64_t m, uint64_t seed, ebc_graph **out) {
    return guarded([&] {
        need(out, "ebc_gen_erdos_renyi: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = gen_erdos_renyi(n, m, seed);
        *out = h.release();
    });
}

ebc_status ebc_gen_rmat(int scale, int edge_factor, double a, double b, double c, double d, uint64_t seed,
                        ebc_graph **out) {
    return guarded([&] {
        need(out, "ebc_gen_rmat: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = gen_rmat(scale, edge_factor, a, b, c, d, seed);
        *out = h.release();
    });
}

ebc_status ebc_gen_rmat_device(int scale, int edge_factor, double a, double b, double c, double d, uint64_t seed,
                               int take_lcc, int device, ebc_graph **out) {
    return guarded([&] {
        need(out, "ebc_gen_rmat_device: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = device_gen_rmat(scale, edge_factor, a, b, c, d, seed, take_lcc != 0, device);
        *out = h.release();
    });
}

ebc_status ebc_graph_from_edges_device(uint64_t n, const uint64_t *src, const uint64_t *dst, uint64_t count,
                                       int take_lcc, int device, ebc_graph **out) {
    return guarded([&] {
        need(out, "ebc_graph_from_edges_device: null out");
        if (count) {
            need(src, "ebc_graph_from_edges_device: null src");
            need(dst, "ebc_graph_from_edges_device: null dst");
        }
        auto h = std::make_unique<ebc_graph>();
        h->g = device_graph_from_edges(n, src, dst, count, take_lcc != 0, device);
        *out = h.release();
    });
}

ebc_status ebc_graph_lcc_device(const ebc_graph *g, int device, ebc_graph **out) {
    return guarded([&] {
        need(g, "ebc_graph_lcc_device: null graph");
        need(out, "ebc_graph_lcc_device: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = device_graph_lcc(g->g, device);
        *out = h.release();
    });
}

ebc_status ebc_gen_grid(uint64_t width, uint64_t height, double delete_prob, double shortcut_fraction,
                        uint64_t seed, ebc_graph **out) {
    return guarded([&] {
        need(out, "ebc_gen_grid: null out");
        auto h = std::make_unique<ebc_graph>();
        h->g = gen_grid(width, height, delete_prob, shortcut_fraction, seed);
        *out = h.release();
    });
}

// ------------------------------------------------- host-side run parameters ---
ebc_status ebc_compute_omega(uint64_t vd, double eps, double delta, uint64_t *omega_out) {
    return guarded([&] {
        need(omega_out, "ebc_compute_omega: null out");
        *omega_out = compute_omega(vd, eps, delta);
    });
}

ebc_status ebc_epoch_length(int ranks, int threads, double base, double exponent, uint64_t *n0_out) {
    return guarded([&] {
        need(n0_out, "ebc_epoch_length: null out");
        *n0_out = epoch_length(ranks, threads, base, exponent);
    });
}

ebc_status ebc_calibrate(const uint64_t *calib_words, uint64_t n, double delta, int allocator,
                         double *delta_lower, double *delta_upper) {
    return guarded([&] {
        need(calib_words, "ebc_calibrate: null frame");
        need(delta_lower, "ebc_calibrate: null delta_lower");
        need(delta_upper, "ebc_calibrate: null delta_upper");
        if (allocator != 0 && allocator != 1)
            throw ConfigError("unknown allocator kind");
        calibrate(calib_words, n, delta, allocator, delta_lower, delta_upper);
    });
}

ebc_status ebc_diameter_upper_bound(const ebc_graph *g, int sweeps, uint64_t seed, uint64_t out[3]) {
    return guarded([&] {
        need(g, "ebc_diameter_upper_bound: null graph");
        need(out, "ebc_diameter_upper_bound: null out");
        // GPU BFS sweeps; the host only drives the restart logic.
        CudaSampler s(g->g, SamplerOptions{-1, 32, 1, 2, 1});
        DiameterBounds b = diameter_upper_bound(g->g, sweeps, seed,
                                                [&](std::uint32_t v) { return s.bfs(v, nullptr); });
        out[0] = b.upper;
        out[1] = b.lower;
        out[2] = b.vertex_diameter;
    });
}

void ebc_shard_range(uint64_t first, uint64_t count, int rank, int world, uint64_t *shard_first,
                     uint64_t *shard_count) {
    uint64_t a = 0, b = 0;
    shard_range(first, count, rank, world, &a, &b);
    if (shard_first)
        *shard_first = a;
    if (shard_count)
        *shard_count = b;
}

// -------------------------------------------------------------------- run ---
void ebc_run_config_default(ebc_run_config *cfg) {
    if (!cfg)
        return;
    std::memset(cfg, 0, sizeof(*cfg));
    RunConfig d;
    cfg->eps = d.eps;
    cfg->delta = d.delta;
    cfg->seed = d.seed;
    cfg->calib_samples = d.calib_samples;
    cfg->diameter_sweeps = d.diameter_sweeps;
    cfg->device = -1;
    cfg->rank = 0;
    cfg->world_size = 1;
    cfg->overlap = 1;
    cfg->work_counters = 1;
}

ebc_status ebc_run(const ebc_graph *g, const ebc_run_config *cfg, ebc_result **out) {
    return guarded([&] {
        need(g, "ebc_run: null graph");
        need(cfg, "ebc_run: null config");
        need(out, "ebc_run: null out");
        RunConfig rc;
        rc.eps = cfg->eps;
        rc.delta = cfg->delta;
        rc.seed = cfg->seed;
        rc.bound = cfg->bound;
        rc.allocator = cfg->allocator;
        rc.omega_override = cfg->omega_override;
        rc.calib_samples = cfg->calib_samples;
        rc.diameter_sweeps = cfg->diameter_sweeps;
        rc.vertex_diameter_override = cfg->vertex_diameter_override;
        rc.epoch_samples = cfg->epoch_samples;
        rc.max_epochs = cfg->max_epochs;
        rc.rank = cfg->rank;
        rc.world_size = cfg->world_size;
        rc.allreduce = cfg->allreduce;
        rc.allreduce_user = cfg->allreduce_user;
        rc.overlap = cfg->overlap;
        rc.validate();
        if (g->g.n < 2)
            throw ContractViolation("run_pipeline: need at least two vertices");
        const auto t0 = std::chrono::steady_clock::now();
        SamplerOptions so = sampler_options(cfg);
        so.short_launches = true; // epochs of some 10^4 samples
        CudaSampler sampler(g->g, so);
        const double upload_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        CudaBackend backend(sampler);
        auto h = std::make_unique<ebc_result>();
        h->out = run_pipeline(g->g, rc, backend);
        h->out.stats.upload_s = upload_s;
        h->out.stats.wall_s += upload_s;
        *out = h.release();
    });
}

ebc_status ebc_result_scores(const ebc_result *r, const double **scores, uint64_t *n) {
    return guarded([&] {
        need(r, "ebc_result_scores: null result");
        if (scores)
            *scores = r->out.scores.data();
        if (n)
            *n = r->out.scores.size();
    });
}

ebc_status ebc_result_counts(const ebc_result *r, const uint64_t **counts, uint64_t *n) {
    return guarded([&] {
        need(r, "ebc_result_counts: null result");
        if (counts)
            *counts = r->out.counts.data();
        if (n)
            *n = r->out.counts.size();
    });
}

uint64_t ebc_result_tau(const ebc_result *r) { return r ? r->out.tau_total : 0; }

ebc_status ebc_result_original_ids(const ebc_result *r, const uint64_t **ids, uint64_t *n) {
    return guarded([&] {
        need(r, "ebc_result_original_ids: null result");
        if (ids)
            *ids = r->out.original_ids.data();
        if (n)
            *n = r->out.original_ids.size();
    });
}

ebc_status ebc_result_stats(const ebc_result *r, ebc_run_stats *stats) {
    return guarded([&] {
        need(r, "ebc_result_stats: null result");
        need(stats, "ebc_result_stats: null stats");
        const RunStats &s = r->out.stats;
        stats->epochs = s.epochs;
        stats->samples = s.samples;
        stats->tau = s.tau;
        stats->omega = s.omega;
        stats->calibration_samples = s.calibration_samples;
        stats->discarded_samples = s.discarded_samples;
        stats->n0 = s.n0;
        stats->n = s.n;
        stats->m = s.m;
        stats->diameter_upper_bound = s.diameter_upper_bound;
        stats->vertex_diameter_bound = s.vertex_diameter_bound;
        stats->adaptive_s = s.adaptive_s;
        stats->diameter_s = s.diameter_s;
        stats->calibration_s = s.calibration_s;
        stats->reduce_s = s.reduce_s;
        stats->check_s = s.check_s;
        stats->upload_s = s.upload_s;
        stats->wall_s = s.wall_s;
        stats->overflow_samples = s.overflow_samples;
        std::memcpy(stats->work, s.work, sizeof(stats->work));
    });
}

void ebc_result_free(ebc_result *r) { delete r; }

// ------------------------------------------------------------ score files ---
ebc_status ebc_scores_write(const char *path, const uint64_t *vertex_ids, const double *scores, uint64_t n,
                            const char *const *meta_keys, const char *const *meta_values, uint64_t meta_count) {
    return guarded([&] {
        need(path, "ebc_scores_write: null path");
        if (n) {
            need(vertex_ids, "ebc_scores_write: null ids");
            need(scores, "ebc_scores_write: null scores");
        }
        ScoreTable t;
        for (uint64_t i = 0; i < meta_count; ++i) {
            if (!(meta_keys && meta_keys[i] && meta_values && meta_values[i]))
                throw ContractViolation("ebc_scores_write: null meta entry");
            t.meta[meta_keys[i]] = meta_values[i];
        }
        t.vertex_ids.assign(vertex_ids, vertex_ids + n);
        t.scores.assign(scores, scores + n);
        write_scores(path, t);
    });
}

ebc_status ebc_result_write_scores(const ebc_result *r, const ebc_run_config *cfg, const char *path) {
    return guarded([&] {
        need(r, "ebc_result_write_scores: null result");
        need(cfg, "ebc_result_write_scores: null config");
        need(path, "ebc_result_write_scores: null path");
        ScoreTable t;
        t.meta = run_meta(cfg->eps, cfg->delta, cfg->seed, r->out.tau_total);
        t.vertex_ids.assign(r->out.original_ids.begin(), r->out.original_ids.end());
        t.scores.assign(r->out.scores.begin(), r->out.scores.end());
        write_scores(path, t);
    });
}

ebc_status ebc_scores_read(const char *path, ebc_scores **out) {
    return guarded([&] {
        need(path, "ebc_scores_read: null path");
        need(out, "ebc_scores_read: null out");
        auto h = std::make_unique<ebc_scores>();
        h->t = read_scores(path);
        *out = h.release();
    });
}

ebc_status ebc_scores_data(const ebc_scores *s, const uint64_t **vertex_ids, const double **scores, uint64_t *n) {
    return guarded([&] {
        need(s, "ebc_scores_data: null scores");
        if (vertex_ids)
            *vertex_ids = s->t.vertex_ids.data();
        if (scores)
            *scores = s->t.scores.data();
        if (n)
            *n = s->t.vertex_ids.size();
    });
}

const char *ebc_scores_meta(const ebc_scores *s, const char *key) {
    if (!s || !key)
        return nullptr;
    auto it = s->t.meta.find(key);
    return it == s->t.meta.end() ? nullptr : it->second.c_str();
}

void ebc_scores_free(ebc_scores *s) { delete s; }

ebc_status ebc_scores_compare(const ebc_scores *approx, const ebc_scores *exact, double eps,
                              ebc_compare_report *out) {
    return guarded([&] {
        need(approx, "ebc_scores_compare: null approx");
        need(exact, "ebc_scores_compare: null exact");
        need(out, "ebc_scores_compare: null out");
        CompareReport r = compare_scores(approx->t, exact->t, eps);
        out->max_abs_error = r.max_abs_error;
        out->vertices_above_eps = r.vertices_above_eps;
        out->top10_overlap = r.top10_overlap;
        out->top100_overlap = r.top100_overlap;
        out->vertices = r.vertices;
    });
}

ebc_status ebc_result_stats_json(const ebc_result *r, const ebc_run_config *cfg, char *buf, uint64_t cap,
                                 uint64_t *needed) {
    return guarded([&] {
        need(r, "ebc_result_stats_json: null result");
        need(cfg, "ebc_result_stats_json: null config");
        const std::string j = stats_json(r->out.stats, cfg->eps, cfg->delta, cfg->seed, cfg->bound, cfg->allocator,
                                         cfg->world_size);
        if (needed)
            *needed = j.size() + 1;
        if (buf && cap) {
            const std::size_t k = std::min<std::size_t>(cap - 1, j.size());
            std::memcpy(buf, j.data(), k);
            buf[k] = 0;
        }
    });
}

// --------------------------------------------------------- device sampler ---
ebc_status ebc_sampler_create(const ebc_graph *g, const ebc_run_config *cfg, ebc_sampler **out) {
    return guarded([&] {
        need(g, "ebc_sampler_create: null graph");
        need(out, "ebc_sampler_create: null out");
        auto h = std::make_unique<ebc_sampler>();
        h->s = std::make_unique<CudaSampler>(g->g, sampler_options(cfg));
        if (cfg && cfg->world_size > 1 && !cfg->allreduce)
            throw ConfigError("run config: world_size > 1 needs an allreduce hook");
        if (cfg && cfg->allreduce) { // also honoured for world_size == 1 (a 1-rank communicator)
            h->allreduce = cfg->allreduce;
            h->allreduce_user = cfg->allreduce_user;
        }
        *out = h.release();
    });
}

void ebc_sampler_free(ebc_sampler *s) { delete s; }

ebc_status ebc_sampler_sample(ebc_sampler *s, uint64_t seed, uint32_t tag, uint64_t first, uint64_t count,
                              int frame) {
    return guarded([&] {
        need(s, "ebc_sampler_sample: null sampler");
        s->s->sample(seed, tag, first, count, frame);
    });
}

ebc_status ebc_sampler_sample_debug(ebc_sampler *s, uint64_t seed, uint32_t tag, uint64_t first,
                                    uint64_t count, const uint32_t *pairs_or_null, int frame,
                                    ebc_sample_record *records, uint32_t *paths, uint64_t path_stride) {
    static_assert(sizeof(ebc_sample_record) == sizeof(SampleRecordHost), "record layouts must match");
    return guarded([&] {
        need(s, "ebc_sampler_sample_debug: null sampler");
        if (pairs_or_null) {
            const std::uint64_t n = s->s->n();
            for (std::uint64_t i = 0; i < count; ++i) {
                const std::uint32_t a = pairs_or_null[2 * i], b = pairs_or_null[2 * i + 1];
                if (a >= n || b >= n)
                    throw ContractViolation("sample_shortest_path: endpoint out of range");
                if (a == b) // sampler.cpp:56
                    throw ContractViolation("sample_shortest_path: endpoints must differ");
            }
        }
        s->s->sample_debug(seed, tag, first, count, pairs_or_null, frame,
                           reinterpret_cast<SampleRecordHost *>(records), paths, path_stride);
    });
}

ebc_status ebc_sampler_last_state(ebc_sampler *s, int side, uint32_t *dist_out, uint64_t *sigma_out) {
    return guarded([&] {
        need(s, "ebc_sampler_last_state: null sampler");
        need(dist_out, "ebc_sampler_last_state: null dist_out");
        need(sigma_out, "ebc_sampler_last_state: null sigma_out");
        s->s->last_state(side, dist_out, sigma_out);
    });
}

ebc_status ebc_sampler_set_stopping(ebc_sampler *s, double eps, uint64_t omega, const double *delta_lower,
                                    const double *delta_upper, int bound) {
    return guarded([&] {
        need(s, "ebc_sampler_set_stopping: null sampler");
        need(delta_lower, "check_stop: calibration missing");
        need(delta_upper, "check_stop: calibration missing");
        s->s->set_stopping(eps, omega, delta_lower, delta_upper, bound);
    });
}

ebc_status ebc_sampler_fold_and_check(ebc_sampler *s, int frame, int *stop_out) {
    return guarded([&] {
        need(s, "ebc_sampler_fold_and_check: null sampler");
        const bool stop = s->s->fold_and_check(frame, s->allreduce, s->allreduce_user);
        if (stop_out)
            *stop_out = stop ? 1 : 0;
    });
}

ebc_status ebc_sampler_read_frame(ebc_sampler *s, int which, uint64_t *words_out) {
    return guarded([&] {
        need(s, "ebc_sampler_read_frame: null sampler");
        need(words_out, "ebc_sampler_read_frame: null out");
        s->s->read_frame(which, words_out);
    });
}

ebc_status ebc_sampler_write_state(ebc_sampler *s, const uint64_t *words) {
    return guarded([&] {
        need(s, "ebc_sampler_write_state: null sampler");
        need(words, "ebc_sampler_write_state: null words");
        s->s->write_state(words);
    });
}

ebc_status ebc_sampler_clear(ebc_sampler *s) {
    return guarded([&] {
        need(s, "ebc_sampler_clear: null sampler");
        s->s->clear();
    });
}

ebc_status ebc_sampler_work(ebc_sampler *s, uint64_t work_out[12], int reset) {
    return guarded([&] {
        need(s, "ebc_sampler_work: null sampler");
        need(work_out, "ebc_sampler_work: null out");
        s->s->work(work_out, reset != 0);
    });
}

ebc_status ebc_sampler_mark(ebc_sampler *s, int event) {
    return guarded([&] {
        need(s, "ebc_sampler_mark: null sampler");
        s->s->mark(event);
    });
}

ebc_status ebc_sampler_elapsed_ms(ebc_sampler *s, int from_event, int to_event, float *ms) {
    return guarded([&] {
        need(s, "ebc_sampler_elapsed_ms: null sampler");
        need(ms, "ebc_sampler_elapsed_ms: null out");
        *ms = s->s->elapsed_ms(from_event, to_event);
    });
}

ebc_status ebc_sampler_sync(ebc_sampler *s) {
    return guarded([&] {
        need(s, "ebc_sampler_sync: null sampler");
        s->s->sync();
    });
}

ebc_status ebc_sampler_info(ebc_sampler *s, uint64_t info_out[6]) {
    return guarded([&] {
        need(s, "ebc_sampler_info: null sampler");
        need(info_out, "ebc_sampler_info: null out");
        s->s->info(info_out);
    });
}

ebc_status ebc_sampler_stream(ebc_sampler *s, void **cuda_stream_out) {
    return guarded([&] {
        need(s, "ebc_sampler_stream: null sampler");
        need(cuda_stream_out, "ebc_sampler_stream: null out");
        *cuda_stream_out = s->s->stream_handle();
    });
}

ebc_status ebc_sampler_frame_ptr(ebc_sampler *s, int frame, void **dev_ptr_out, uint64_t *words_out) {
    return guarded([&] {
        need(s, "ebc_sampler_frame_ptr: null sampler");
        need(dev_ptr_out, "ebc_sampler_frame_ptr: null out");
        std::uint64_t words = 0;
        s->s->frame_ptr(frame, dev_ptr_out, &words);
        if (words_out)
            *words_out = words;
    });
}

ebc_status ebc_sampler_bfs(ebc_sampler *s, uint32_t source, uint32_t *dist_out, uint64_t out[3]) {
    return guarded([&] {
        need(s, "ebc_sampler_bfs: null sampler");
        need(out, "ebc_sampler_bfs: null out");
        BfsSummary r = s->s->bfs(source, dist_out);
        out[0] = r.farthest;
        out[1] = r.eccentricity;
        out[2] = r.reached;
    });
}

void ebc_release_device_cache(void) {
    try {
        release_device_cache();
    } catch (...) {
    }
}

ebc_status ebc_sampler_flush_l2(ebc_sampler *s) {
    return guarded([&] {
        need(s, "ebc_sampler_flush_l2: null sampler");
        s->s->flush_l2();
    });
}

} // extern "C"

// ---------------------------------------------------------------- native NCCL hook ----
// The five NCCL entry points are bound at run time; the handful of types below is NCCL's stable C ABI
// (nccl.h: ncclUniqueId is 128 opaque bytes, ncclUint32 = 3, ncclSum = 0, ncclSuccess = 0).
namespace {
struct NcclApi {
    struct UniqueId {
        char internal[EBC_NCCL_UNIQUE_ID_BYTES];
    };
    int (*GetUniqueId)(UniqueId *) = nullptr;
    int (*CommInitRank)(void **, int, UniqueId, int) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, void *, void *) = nullptr;
    int (*CommDestroy)(void *) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
    std::string why;
};

const NcclApi &nccl_api() {
    static const NcclApi api = [] {
        NcclApi a;
        void *h = nullptr;
        for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
            h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (h)
                break;
        }
        if (!h) {
            const char *err = dlerror(); // (a second call would return null: the first one clears the state)
            a.why = std::string("libnccl.so.2 not found: ") + (err ? err : "");
            return a;
        }
        a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
        a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(dlsym(h, "ncclGetErrorString"));
        if (!a.GetUniqueId || !a.CommInitRank || !a.AllReduce || !a.CommDestroy || !a.GetErrorString)
            a.why = "libnccl.so.2 lacks an expected entry point";
        return a;
    }();
    if (!api.why.empty())
        throw BackendFault(api.why);
    return api;
}

void nccl_check(const NcclApi &a, int rc, const char *what) {
    if (rc != 0)
        throw BackendFault(std::string(what) + ": " + a.GetErrorString(rc));
}
} // namespace

struct ebc_nccl_comm {
    void *comm = nullptr;
    int rank = 0, world = 1;
};

extern "C" {

ebc_status ebc_nccl_unique_id(void *id_out) {
    return guarded([&] {
        need(id_out, "ebc_nccl_unique_id: null id");
        const NcclApi &a = nccl_api();
        NcclApi::UniqueId id;
        nccl_check(a, a.GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(id_out, id.internal, sizeof id.internal);
    });
}

ebc_status ebc_nccl_comm_create(const void *id, int rank, int world_size, int device, ebc_nccl_comm **out) {
    return guarded([&] {
        need(id, "ebc_nccl_comm_create: null id");
        need(out, "ebc_nccl_comm_create: null out");
        if (world_size < 1 || rank < 0 || rank >= world_size)
            throw ConfigError("ebc_nccl_comm_create: need 0 <= rank < world_size");
        // The all-reduce runs beside the sampling kernel on the SMs that kernel leaves empty (ebc_run_config.reserved_sms):
        // keep NCCL's kernel to as many CTAs, unless the caller has chosen otherwise.
        setenv("NCCL_MAX_CTAS", "4", /*overwrite=*/0);
        const NcclApi &a = nccl_api();
        set_device_or_throw(device);
        NcclApi::UniqueId uid;
        std::memcpy(uid.internal, id, sizeof uid.internal);
        auto c = std::make_unique<ebc_nccl_comm>();
        c->rank = rank;
        c->world = world_size;
        nccl_check(a, a.CommInitRank(&c->comm, world_size, uid, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

int ebc_nccl_allreduce(void *user, void *buf, uint64_t count, void *cuda_stream) {
    const ebc_status st = guarded([&] {
        need(user, "ebc_nccl_allreduce: null communicator");
        need(buf, "ebc_nccl_allreduce: null buffer");
        const NcclApi &a = nccl_api();
        auto *c = static_cast<ebc_nccl_comm *>(user);
        nccl_check(a, a.AllReduce(buf, buf, static_cast<size_t>(count), /*ncclUint32*/ 3, /*ncclSum*/ 0, c->comm, cuda_stream),
                   "ncclAllReduce");
    });
    return st == EBC_OK ? 0 : 1;
}

void ebc_nccl_comm_free(ebc_nccl_comm *c) {
    if (!c)
        return;
    try {
        if (c->comm)
            nccl_api().CommDestroy(c->comm);
    } catch (...) {
    }
    delete c;
}

} // extern "C"
