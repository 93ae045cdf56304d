// Host-side pieces of the stopping rule that run once per run: the static
// sample budget, the epoch length and the per-vertex failure-probability
// allocation.  FP64 with the same operation order as the reference so the
// values (and therefore the device-side stop decision) are identical:
//   compute_omega  /root/reference/proj/src/stopping.cpp:31-41
//   calibrate      stopping.cpp:43-92
//   epoch_length   /root/reference/proj/src/engine.cpp:26-31
//   log terms of bound_width  stopping.cpp:103,106
#include "host_common.hpp"

#include <cmath>

namespace ebc {

std::uint64_t compute_omega(std::uint64_t vd, double eps, double delta) {
    require(vd >= 2, "compute_omega: vertex diameter bound below 2");
    require(eps > 0 && delta > 0 && delta < 1, "compute_omega: bad eps/delta");
    const double levels = vd > 2 ? std::floor(std::log2(static_cast<double>(vd - 2))) : 0.0;
    const double budget = (0.5 / (eps * eps)) * (levels + 1.0 + std::log(1.0 / delta));
    return static_cast<std::uint64_t>(std::ceil(budget));
}

std::uint64_t epoch_length(int ranks, int threads, double base, double exponent) {
    require(ranks >= 1 && threads >= 1, "epoch_length: bad worker counts");
    const double workers = static_cast<double>(ranks) * threads;
    const long long n0 = std::llround(base / std::pow(workers, exponent));
    return n0 < 1 ? 1 : static_cast<std::uint64_t>(n0);
}

void calibrate(const std::uint64_t *calib, std::uint64_t n, double delta, int allocator,
               double *lower, double *upper) {
    require(n >= 1, "calibrate: empty graph");
    require(delta > 0 && delta < 1, "calibrate: bad delta");
    const std::uint64_t tau = calib ? calib[0] : 0;
    bool weighted = allocator == 1 && tau != 0;
    if (weighted) {
        const double t = static_cast<double>(tau);
        double weight_sum = 0.0;
        for (std::uint64_t v = 0; v < n; ++v)
            weight_sum += std::sqrt(static_cast<double>(calib[v + 1]) / t);
        if (weight_sum == 0.0) {
            weighted = false; // no signal to redistribute
        } else {
            const double budget = delta * (1.0 - 1e-6);
            const double floor_per_vertex = delta / (2.0 * static_cast<double>(n));
            const double spare = budget - floor_per_vertex * static_cast<double>(n);
            for (std::uint64_t v = 0; v < n; ++v) {
                const double w = std::sqrt(static_cast<double>(calib[v + 1]) / t);
                const double both_sides = floor_per_vertex + spare * (w / weight_sum);
                lower[v] = both_sides / 2.0;
                upper[v] = both_sides / 2.0;
            }
        }
    }
    if (!weighted) {
        const double per_side = delta / (2.0 * static_cast<double>(n));
        for (std::uint64_t v = 0; v < n; ++v)
            lower[v] = upper[v] = per_side;
    }
    // Union-bound budget must hold exactly after rounding (stopping.cpp:82-91).
    long double total = 0.0L;
    for (std::uint64_t v = 0; v < n; ++v)
        total += static_cast<long double>(lower[v]) + upper[v];
    if (total > static_cast<long double>(delta)) {
        const double scale =
            static_cast<double>(static_cast<long double>(delta) / total) * (1.0 - 1e-12);
        for (std::uint64_t v = 0; v < n; ++v) {
            lower[v] *= scale;
            upper[v] *= scale;
        }
    }
}

// The value every entry of lower[] and upper[] gets from calibrate() under the uniform allocator,
// including the budget guard (same operations in the same order, without the two arrays).
double calibrate_uniform_value(std::uint64_t n, double delta) {
    require(n >= 1, "calibrate: empty graph");
    require(delta > 0 && delta < 1, "calibrate: bad delta");
    double per_side = delta / (2.0 * static_cast<double>(n));
    long double total = 0.0L;
    for (std::uint64_t v = 0; v < n; ++v)
        total += static_cast<long double>(per_side) + per_side;
    if (total > static_cast<long double>(delta)) {
        const double scale = static_cast<double>(static_cast<long double>(delta) / total) * (1.0 - 1e-12);
        per_side *= scale;
    }
    return per_side;
}

void bound_log_terms(const double *delta_v, std::uint64_t n, int bound, double *out) {
    // Equal inputs give equal outputs, so the last (input, output) pair is reused: under the uniform
    // allocator all n values are identical and this is one log() instead of n.
    double last_in = -1.0, last_out = 0.0;
    for (std::uint64_t v = 0; v < n; ++v) {
        const double d = delta_v[v];
        if (d != last_in) {
            if (!(d > 0.0 && d < 1.0))
                throw ContractViolation("bound: bad per-vertex delta");
            last_in = d;
            last_out = bound == 0 ? std::log(1.0 / d) : std::log(2.0 / d);
        }
        out[v] = last_out;
    }
}

} // namespace ebc
