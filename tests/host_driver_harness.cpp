// TEST-ONLY harness: the product's host-side epoch driver (paper_1910_11039_b200/csrc/epoch_driver.cpp,
// CUDA-free) instantiated over a SamplerBackend that calls the CPU oracle.  It exists so the multi-rank
// orchestration (sharding, epoch schedule, allreduce hook, discard semantics, conservation checks) can
// be exercised on CPU with gloo, world_size 2.  It is compiled by tests/test_multi_rank_gloo.py into
// tests/_build/ and is never part of libebc_b200.so.
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../paper_1910_11039_b200/csrc/epoch_driver.hpp"

extern "C" {
struct ebc_oracle;
ebc_oracle *ebc_oracle_create(uint64_t n, const uint64_t *offsets, const uint32_t *targets);
void ebc_oracle_destroy(ebc_oracle *o);
void ebc_oracle_accumulate(ebc_oracle *o, uint64_t seed, uint32_t tag, uint64_t first, uint64_t count,
                           uint64_t *frame_words);
int ebc_oracle_check_stop(const uint64_t *words, uint64_t n, double eps, uint64_t omega, const double *dl,
                          const double *du, int bound);
void ebc_oracle_bfs(const ebc_oracle *o, uint32_t source, uint32_t *dist, uint32_t *queue, uint64_t *out);
}

namespace {
using namespace ebc;

class OracleBackend final : public SamplerBackend {
public:
    explicit OracleBackend(const HostGraph &g) : n_(g.n), S_(g.n + 1, 0) {
        o_ = ebc_oracle_create(g.n, g.offsets.data(), g.targets.data());
        frame_[0].assign(g.n + 1, 0);
        frame_[1].assign(g.n + 1, 0);
    }
    ~OracleBackend() override { ebc_oracle_destroy(o_); }
    BfsSummary bfs(std::uint32_t source) override {
        std::vector<std::uint32_t> d(n_), q(n_);
        std::uint64_t out[3];
        ebc_oracle_bfs(o_, source, d.data(), q.data(), out);
        BfsSummary r;
        r.farthest = static_cast<std::uint32_t>(out[0]);
        r.eccentricity = static_cast<std::uint32_t>(out[1]);
        r.reached = out[2];
        return r;
    }
    void sample(std::uint64_t seed, std::uint32_t tag, std::uint64_t first, std::uint64_t count, int frame) override {
        std::vector<std::uint64_t> w(n_ + 1, 0);
        ebc_oracle_accumulate(o_, seed, tag, first, count, w.data());
        for (std::uint64_t i = 0; i <= n_; ++i)
            frame_[frame][i] += static_cast<std::uint32_t>(w[i]);
    }
    void set_stopping(double eps, std::uint64_t omega, const double *dl, const double *du, int bound) override {
        eps_ = eps;
        omega_ = omega;
        dl_.assign(dl, dl + n_);
        du_.assign(du, du + n_);
        bound_ = bound;
        have_ = true;
    }
    void fold_async(int frame, AllreduceHook allreduce, void *user) override {
        if (allreduce && allreduce(user, frame_[frame].data(), n_ + 1, nullptr) != 0)
            throw BackendFault("allreduce callback failed");
        for (std::uint64_t i = 0; i <= n_; ++i) {
            S_[i] += frame_[frame][i];
            frame_[frame][i] = 0;
        }
        stop_[frame] = have_ && ebc_oracle_check_stop(S_.data(), n_, eps_, omega_, dl_.data(), du_.data(), bound_);
    }
    bool wait_fold(int frame, std::uint64_t *tau_out) override {
        if (tau_out)
            *tau_out = S_[0];
        return stop_[frame];
    }
    void discard_frame(int frame) override { std::fill(frame_[frame].begin(), frame_[frame].end(), 0u); }
    void read_state(std::uint64_t *words_out) override { std::memcpy(words_out, S_.data(), 8 * (n_ + 1)); }
    void clear() override {
        std::fill(S_.begin(), S_.end(), 0);
        discard_frame(0);
        discard_frame(1);
    }
    void finish(RunStats &) override {}

private:
    std::uint64_t n_;
    ebc_oracle *o_;
    std::vector<std::uint32_t> frame_[2];
    std::vector<std::uint64_t> S_;
    std::vector<double> dl_, du_;
    double eps_ = 0;
    std::uint64_t omega_ = 0;
    int bound_ = 0;
    bool have_ = false;
    bool stop_[2] = {false, false};
};

std::string g_err;
} // namespace

extern "C" __attribute__((visibility("default"))) const char *harness_last_error() { return g_err.c_str(); }

// Runs the product's run_pipeline over the oracle backend.  out_counts: n u64; out_stats: 8 u64
// {epochs, samples, tau, omega, calibration_samples, discarded_samples, n0, vertex_diameter_bound}.
extern "C" __attribute__((visibility("default"))) int
harness_run(uint64_t n, const uint64_t *offsets, const uint32_t *targets, double eps, double delta, uint64_t seed,
            int bound, int allocator, uint64_t epoch_samples, uint64_t calib_samples, int overlap, int rank,
            int world, AllreduceHook hook, uint64_t *out_counts, uint64_t *out_stats) {
    try {
        HostGraph g = graph_from_csr(n, offsets, targets, nullptr, true);
        RunConfig cfg;
        cfg.eps = eps;
        cfg.delta = delta;
        cfg.seed = seed;
        cfg.bound = bound;
        cfg.allocator = allocator;
        cfg.epoch_samples = epoch_samples;
        cfg.calib_samples = calib_samples;
        cfg.overlap = overlap;
        cfg.rank = rank;
        cfg.world_size = world;
        cfg.allreduce = hook;
        OracleBackend be(g);
        RunOutput out = run_pipeline(g, cfg, be);
        std::memcpy(out_counts, out.counts.data(), 8 * n);
        const RunStats &s = out.stats;
        const uint64_t st[8] = {s.epochs, s.samples, s.tau, s.omega, s.calibration_samples, s.discarded_samples,
                                s.n0, s.vertex_diameter_bound};
        std::memcpy(out_stats, st, sizeof(st));
        return 0;
    } catch (const std::exception &e) {
        g_err = e.what();
        return 1;
    }
}
