// Host-side handle of the device sampler: replicated CSR in HBM, per-slot
// search state, two epoch frames (double buffer, as ThreadSlot::frames[2] in
// /root/reference/proj/include/epochbc/epoch.hpp:80-84) and the accumulated
// state S.  All compute happens in the kernels of cuda_sampler.cu; there is no
// CPU path.
#pragma once

#include <cstdint>
#include <memory>
#include <vector>

#include "host_common.hpp"

namespace ebc {

struct SamplerOptions {
    int device = -1;
    std::uint32_t block_threads = 0; // 0 = auto
    std::uint32_t slots = 0;         // 0 = auto
    std::uint64_t slot_capacity = 0; // 0 = auto
    std::uint32_t items_per_thread = 0; // 0 = auto
    bool materialize_final_level = false; // settle the final level of every sample (see ebc_b200.h)
    int renumber = 0; // device-side numbering: 0 = auto, -1 = never, 1 = degree classes, 2 = neighbourhood clusters
    std::uint32_t reserved_sms = 0; // SMs the main sampling pass leaves empty (for a collective running beside it)
    bool work_counters = true; // false: kernels without statistics (see ebc_run_config.work_counters)
    bool short_launches = false; // launches of a few samples per slot (the epochs of a pipeline run): prefer fewer, larger CTAs
};

struct SampleRecordHost { // == ebc_sample_record
    std::uint32_t s, t, dist, meet, meet_count, draws, path_len, flags;
    std::uint64_t weight_lo, weight_hi;
};

using AllreduceFn = int (*)(void *user, void *buf, std::uint64_t count, void *cuda_stream);

// Frees the device buffers cached from destroyed samplers (see DevicePool in cuda_sampler.cu).
void release_device_cache();
// Makes `device` (>= 0) the calling thread's CUDA device; throws CudaError when there is no device at all.
void set_device_or_throw(int device);

class CudaSampler {
public:
    CudaSampler(const HostGraph &g, const SamplerOptions &opt);
    ~CudaSampler();
    CudaSampler(const CudaSampler &) = delete;
    CudaSampler &operator=(const CudaSampler &) = delete;

    std::uint64_t n() const;
    // Asynchronous: samples [first, first+count) of stream (seed, tag) into epoch frame `frame`.
    void sample(std::uint64_t seed, std::uint32_t tag, std::uint64_t first, std::uint64_t count, int frame);
    // Synchronous test hook.
    void sample_debug(std::uint64_t seed, std::uint32_t tag, std::uint64_t first, std::uint64_t count,
                      const std::uint32_t *pairs, int frame, SampleRecordHost *records,
                      std::uint32_t *paths, std::uint64_t path_stride);
    void last_state(int side, std::uint32_t *dist_out, std::uint64_t *sigma_out);

    void set_stopping(double eps, std::uint64_t omega, const double *delta_lower,
                      const double *delta_upper, int bound);
    // delta_lower[v] == delta_upper[v] == delta_each for all v: the log terms are filled on the device.
    void set_stopping_uniform(double eps, std::uint64_t omega, double delta_each, int bound);
    // Asynchronous part of fold+check on the aggregation stream; wait_fold() returns the decision.
    void fold_and_check_async(int frame, AllreduceFn allreduce, void *user);
    bool wait_fold(int frame, std::uint64_t *tau_out = nullptr);
    bool fold_and_check(int frame, AllreduceFn allreduce, void *user) {
        fold_and_check_async(frame, allreduce, user);
        return wait_fold(frame);
    }
    // Waits for the sampling into `frame`, then zeroes it without folding (discarded epoch).
    void discard_frame(int frame);
    void read_frame(int which, std::uint64_t *words_out);
    void write_state(const std::uint64_t *words);
    void clear();
    void work(std::uint64_t *out, bool reset);
    void mark(int event);
    float elapsed_ms(int from, int to);
    void sync();
    void info(std::uint64_t *out6);
    void *stream_handle();
    void frame_ptr(int frame, void **ptr, std::uint64_t *words);
    BfsSummary bfs(std::uint32_t source, std::uint32_t *dist_out);
    void flush_l2();
    std::uint64_t overflow_samples() const;
    std::uint64_t kernel_launches() const;

private:
    struct Impl;
    std::unique_ptr<Impl> impl_;
};

} // namespace ebc
