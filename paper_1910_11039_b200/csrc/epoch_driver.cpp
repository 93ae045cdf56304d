// See epoch_driver.hpp.  Phase structure follows run_pipeline
// (/root/reference/proj/src/engine.cpp:281-403); the epoch loop follows
// AdaptiveDriver::run_algorithm1 (engine.cpp:124-167) with the reduce-to-root +
// flag broadcast replaced by one sum-allreduce of the epoch frame.
#include "epoch_driver.hpp"

#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>

#include "philox.cuh"

namespace ebc {

namespace {
double now_s() {
    using clock = std::chrono::steady_clock;
    return std::chrono::duration<double>(clock::now().time_since_epoch()).count();
}
} // namespace

void RunConfig::validate() const {
    if (!(eps > 0 && eps < 1) || !(delta > 0 && delta < 1))
        throw ConfigError("run config: eps and delta must lie in (0,1)");
    if (world_size < 1 || rank < 0 || rank >= world_size)
        throw ConfigError("run config: rank must lie in [0, world_size)");
    if (world_size > 1 && allreduce == nullptr)
        throw ConfigError("run config: world_size > 1 needs an allreduce hook");
    if (bound != 0 && bound != 1)
        throw ConfigError("unknown bound kind");
    if (allocator != 0 && allocator != 1)
        throw ConfigError("unknown allocator kind");
    if (diameter_sweeps < 1)
        throw ConfigError("run config: need at least one diameter sweep");
    // Epoch frames are u32 (word 0 = the epoch's tau, hub counters <= tau): an epoch or a calibration batch
    // must stay below 2^32 samples or the words wrap.
    if (epoch_samples >= (std::uint64_t{1} << 32) || calib_samples >= (std::uint64_t{1} << 32))
        throw ConfigError("run config: epoch_samples and calib_samples must be below 2^32 (epoch frames are 32-bit)");
}

std::uint64_t default_epoch_samples(std::uint64_t omega, bool adaptive_rule) {
    // k epochs of equal size.  Under the Hoeffding bound the width does not depend on the counters and
    // the static budget omega fires first, so k = clamp(round(omega / 32768), 2, 16): an epoch keeps every
    // resident CTA busy for many samples (the tail of a launch costs about one sample time).  With the
    // empirical-Bernstein bound the run can stop long before omega, and the epoch in flight at the stop is
    // discarded, so epochs are half as long there (k = clamp(round(omega / 16384), 3, 32); config 2 with
    // the weighted allocator then stops at tau = 55 296 instead of 71 680; 8192-sample epochs stop a
    // little earlier still but sample 30 % slower).  B is rounded up to 1024 so that k * B overshoots
    // omega by less than k * 1024 samples.  Depends on omega and the rule only, never on the GPU count.
    const std::uint64_t unit = adaptive_rule ? 16384 : 32768;
    const std::uint64_t k_min = adaptive_rule ? 3 : 2, k_max = adaptive_rule ? 32 : 16;
    std::uint64_t k = (omega + unit / 2) / unit;
    k = k < k_min ? k_min : (k > k_max ? k_max : k);
    std::uint64_t b = (omega + k - 1) / k;
    b = (b + 1023) / 1024 * 1024;
    if (b < 1024)
        b = 1024;
    if (b > (std::uint64_t{1} << 20))
        b = std::uint64_t{1} << 20;
    return b;
}

RunOutput run_pipeline(const HostGraph &g, const RunConfig &cfg, SamplerBackend &be) {
    cfg.validate();
    require(g.n >= 2, "run_pipeline: need at least two vertices");
    const std::uint64_t n = g.n;
    RunOutput out;
    RunStats &st = out.stats;
    st.n = n;
    st.m = g.m;
    const double run_start = now_s();
    const AllreduceHook hook = cfg.allreduce; // also honoured for world_size == 1 (a 1-rank communicator)

    // Phase 1: vertex-diameter bound (engine.cpp:298-311).  Deterministic, so
    // every rank computes it locally instead of receiving a broadcast.
    std::uint64_t vd = cfg.vertex_diameter_override;
    {
        const double t0 = now_s();
        if (vd == 0) {
            DiameterBounds b = diameter_upper_bound(g, cfg.diameter_sweeps, cfg.seed,
                                                    [&](std::uint32_t v) { return be.bfs(v); });
            st.diameter_upper_bound = b.upper;
            vd = b.vertex_diameter;
        }
        st.vertex_diameter_bound = vd;
        st.diameter_s = now_s() - t0;
    }

    // Phase 2: static sample budget (engine.cpp:313-319).
    const std::uint64_t omega = cfg.omega_override ? cfg.omega_override : compute_omega(vd, cfg.eps, cfg.delta);
    st.omega = omega;

    // Phase 3: calibration (engine.cpp:321-357): non-adaptive samples from an
    // independent stream, blocking aggregation, failure-probability allocation.
    {
        const double t0 = now_s();
        // the uniform allocator uses no calibration counts (stopping.cpp:50,72-78): no arrays needed
        const bool uniform = cfg.allocator == 0;
        std::vector<std::uint64_t> calib(uniform ? 1 : n + 1, 0);
        double uniform_each = 0.0;
        if (cfg.calib_samples > 0) {
            std::uint64_t lo, cnt;
            shard_range(0, cfg.calib_samples, cfg.rank, cfg.world_size, &lo, &cnt);
            be.sample(cfg.seed, kTagCalibration, lo, cnt, 0);
            be.fold_async(0, hook, cfg.allreduce_user);
            if (uniform) // a serial long-double sum over n: done while the GPU takes the calibration samples
                uniform_each = calibrate_uniform_value(n, cfg.delta);
            std::uint64_t tau = 0;
            be.wait_fold(0, &tau);
            if (uniform)
                calib[0] = tau;
            else
                be.read_state(calib.data());
            be.clear();
        }
        st.calibration_samples = calib[0];
        if (uniform) {
            if (uniform_each == 0.0)
                uniform_each = calibrate_uniform_value(n, cfg.delta);
            be.set_stopping_uniform(cfg.eps, omega, uniform_each, n, cfg.bound);
        } else {
            std::vector<double> delta_lower(n), delta_upper(n);
            calibrate(calib.data(), n, cfg.delta, cfg.allocator, delta_lower.data(), delta_upper.data());
            be.set_stopping(cfg.eps, omega, delta_lower.data(), delta_upper.data(), cfg.bound);
        }
        st.calibration_s = now_s() - t0;
    }

    // Phase 4: adaptive sampling in epochs.
    const std::uint64_t B = cfg.epoch_samples ? cfg.epoch_samples : default_epoch_samples(omega, cfg.bound != 0);
    st.n0 = B;
    std::uint64_t applied = 0, discarded = 0, tau = 0;
    {
        const double t0 = now_s();
        // tau after epoch e is (e+1)*B exactly, so the omega rule fires at this epoch at the latest.
        const std::uint64_t last_epoch = (omega + B - 1) / B - (omega > 0 ? 1 : 0);
        auto launch = [&](std::uint64_t e) {
            std::uint64_t lo, cnt;
            shard_range(e * B, B, cfg.rank, cfg.world_size, &lo, &cnt);
            be.sample(cfg.seed, kTagAdaptive, lo, cnt, static_cast<int>(e & 1));
            applied += B;
        };
        std::uint64_t launched = 0; // epochs launched so far
        launch(0);
        launched = 1;
        for (std::uint64_t e = 0;; ++e) {
            const int frame = static_cast<int>(e & 1);
            be.fold_async(frame, hook, cfg.allreduce_user);
            if (cfg.overlap && e < last_epoch && launched == e + 1 &&
                (cfg.max_epochs == 0 || e + 1 < cfg.max_epochs)) {
                launch(e + 1); // overlapped with the reduce + check of epoch e
                launched = e + 2;
            }
            const double t1 = now_s();
            const bool stop = be.wait_fold(frame, &tau);
            st.check_s += now_s() - t1;
            ++st.epochs;
            const bool capped = cfg.max_epochs != 0 && st.epochs >= cfg.max_epochs;
            if (stop || capped) {
                if (launched > e + 1) { // an epoch is in flight: its samples are discarded
                    be.discard_frame(static_cast<int>((e + 1) & 1));
                    discarded += B;
                }
                break;
            }
            if (launched == e + 1) {
                launch(e + 1);
                launched = e + 2;
            }
        }
        st.adaptive_s = now_s() - t0;
    }

    // Sample accounting (engine.cpp:371-386): exact integers.
    st.samples = st.calibration_samples + applied;
    st.discarded_samples = discarded;
    st.tau = tau;
    require(tau == applied - discarded, "sample conservation violated: tau != applied - discarded");

    // Result assembly (engine.cpp:391-401).
    RawVector<std::uint64_t> words(n + 1);
    be.read_state(words.data());
    require(words[0] == tau, "sample conservation violated: tau of S differs from the checked tau");
    out.tau_total = tau;
    out.original_ids.resize(n);
    out.counts.resize(n);
    out.scores.resize(n);
    std::memcpy(out.original_ids.data(), g.original_ids.data(), n * sizeof(std::uint64_t));
    std::memcpy(out.counts.data(), words.data() + 1, n * sizeof(std::uint64_t));
    for (std::uint64_t v = 0; v < n; ++v)
        out.scores[v] = tau > 0 ? static_cast<double>(out.counts[v]) / static_cast<double>(tau) : 0.0;
    be.finish(st);
    st.wall_s = now_s() - run_start;
    if (std::getenv("EBC_TRACE"))
        std::fprintf(stderr, "[ebc] run_pipeline: diameter %.3f ms, calibration %.3f ms, adaptive %.3f ms, total %.3f ms\n",
                     st.diameter_s * 1e3, st.calibration_s * 1e3, st.adaptive_s * 1e3, st.wall_s * 1e3);
    return out;
}

} // namespace ebc
