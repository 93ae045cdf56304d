// Host-side orchestration of one run: diameter -> omega -> calibration ->
// adaptive epochs -> scores.  Mirrors the phase sequence and the epoch /
// overshoot / discard semantics of the reference's run_pipeline and
// AdaptiveDriver (/root/reference/proj/src/engine.cpp:124-167, 281-403) with
// GPUs in place of ranks/threads:
//   * epoch e covers the global sample indices [e*B, (e+1)*B) for a B that does
//     not depend on the number of GPUs, each rank takes a contiguous shard;
//   * epoch frames are double buffered; while epoch e is reduced, folded and
//     checked on the aggregation stream, epoch e+1 is already being sampled
//     (the paper's overlap of aggregation with sampling);
//   * every rank evaluates the same stop predicate on identical integers, so no
//     broadcast is needed; samples of an epoch in flight at the stop are
//     discarded (engine.cpp:166,276).
// This file is CUDA-free: the device work sits behind SamplerBackend.
#pragma once

#include <cstdint>
#include <vector>

#include "host_common.hpp"

namespace ebc {

using AllreduceHook = int (*)(void *user, void *buf, std::uint64_t count, void *cuda_stream);

struct RunConfig { // replaces epochbc::RunConfig (engine.hpp:59-81)
    double eps = 0.001;
    double delta = 0.1;
    std::uint64_t seed = 1;
    int bound = 0;
    int allocator = 0;
    std::uint64_t omega_override = 0;
    std::uint64_t calib_samples = 800; // reference: 100 per worker (engine.hpp:73); 8 workers
    int diameter_sweeps = 4;
    std::uint64_t vertex_diameter_override = 0;
    std::uint64_t epoch_samples = 0;
    std::uint64_t max_epochs = 0;
    int rank = 0, world_size = 1;
    AllreduceHook allreduce = nullptr;
    void *allreduce_user = nullptr;
    int overlap = 1;

    void validate() const; // RunConfig::validate (engine.cpp:13-24)
};

struct RunStats { // replaces epochbc::RunStats (engine.hpp:89-110)
    std::uint64_t epochs = 0, samples = 0, tau = 0, omega = 0, calibration_samples = 0,
                  discarded_samples = 0, n0 = 0;
    std::uint64_t n = 0, m = 0, diameter_upper_bound = 0, vertex_diameter_bound = 0;
    double adaptive_s = 0, diameter_s = 0, calibration_s = 0, reduce_s = 0, check_s = 0, upload_s = 0,
           wall_s = 0;
    std::uint64_t overflow_samples = 0;
    std::uint64_t work[12] = {0};
};

struct RunOutput { // ApproxResult (engine.hpp:83-87) + stats
    RawVector<double> scores; // (RawVector: pooled page-locked memory, no zero fill -- see host_common.hpp)
    RawVector<std::uint64_t> counts;
    std::uint64_t tau_total = 0;
    RawVector<std::uint64_t> original_ids;
    RunStats stats;
};

class SamplerBackend {
public:
    virtual ~SamplerBackend() = default;
    virtual BfsSummary bfs(std::uint32_t source) = 0;
    // Asynchronous: samples [first, first+count) of (seed, tag) into epoch frame `frame`.
    virtual void sample(std::uint64_t seed, std::uint32_t tag, std::uint64_t first, std::uint64_t count,
                        int frame) = 0;
    virtual void set_stopping(double eps, std::uint64_t omega, const double *delta_lower,
                              const double *delta_upper, int bound) = 0;
    // Same with delta_lower[v] == delta_upper[v] == delta_each for every vertex (uniform allocator);
    // a backend may override it to skip the per-vertex arrays.
    virtual void set_stopping_uniform(double eps, std::uint64_t omega, double delta_each, std::uint64_t n, int bound) {
        const std::vector<double> each(n, delta_each);
        set_stopping(eps, omega, each.data(), each.data(), bound);
    }
    // Asynchronous: (allreduce) -> S += frame, frame := 0 -> check_stop(S).
    virtual void fold_async(int frame, AllreduceHook allreduce, void *user) = 0;
    // Completes the fold of `frame`; returns the stop decision and tau of S.
    virtual bool wait_fold(int frame, std::uint64_t *tau_out) = 0;
    // Waits for the sampling into `frame` and zeroes it without folding (discarded epoch).
    virtual void discard_frame(int frame) = 0;
    virtual void read_state(std::uint64_t *words_out) = 0; // S, n+1 words
    virtual void clear() = 0;                              // frames and S := 0
    virtual void finish(RunStats &stats) = 0;              // work counters, overflow count
};

// Samples per epoch derived from omega and the stopping rule only (never from the GPU count).
std::uint64_t default_epoch_samples(std::uint64_t omega, bool adaptive_rule);

RunOutput run_pipeline(const HostGraph &g, const RunConfig &cfg, SamplerBackend &backend);

} // namespace ebc
