// proj/src/b200_backend.cpp -- the adapter INTEGRATION.md section 2 describes, as real code.
// Reference interfaces it stands in for: run_simulated (include/epochbc/engine.hpp:153-156), called by cmd_run at
// tools/epochbc.cpp:218; error classes include/epochbc/types.hpp:15-36.
#include "b200_backend.hpp"

#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#include "ebc_b200.h" // this repository, include/
#include "epochbc/types.hpp"

namespace epochbc {

namespace {

[[noreturn]] void throw_status(ebc_status st) { // ebc_status -> the reference's exception classes
    const std::string msg = ebc_last_error();
    switch (st) {
    case EBC_ERR_CONFIG: throw ConfigError(msg);                  // also ContractViolation; CLI exit 2 (tools/epochbc.cpp:26-30)
    case EBC_ERR_PARSE: throw ParseError(msg);                    // CLI exit 3
    case EBC_ERR_BACKEND: throw BackendFault(msg);                // CLI exit 4
    default: throw BackendFault("b200 backend: " + msg);          // CUDA / NCCL failures, no GPU
    }
}

struct GraphHandle { // frees the C handle on every exit path
    ebc_graph *g = nullptr;
    ~GraphHandle() { ebc_graph_free(g); }
};
struct ResultHandle {
    ebc_result *r = nullptr;
    ~ResultHandle() { ebc_result_free(r); }
};

} // namespace

SimRunOutcome run_b200(const Graph &g, const RunConfig &cfg, int device) {
    cfg.validate(); // the reference's own checks (engine.cpp), same messages
    // Graph -> CSR with 32-bit ids (graph.hpp:57-58 exposes offsets()/targets(); Vertex is 64-bit there)
    if (g.num_vertices() > std::numeric_limits<std::uint32_t>::max())
        throw ConfigError("b200 backend: vertex ids must fit 32 bits");
    std::vector<std::uint32_t> targets(g.targets().begin(), g.targets().end());
    GraphHandle gh;
    ebc_status st = ebc_graph_from_csr(g.num_vertices(), g.offsets().data(), targets.data(), g.original_ids().data(),
                                       /*validate=*/0, &gh.g);
    if (st != EBC_OK)
        throw_status(st);
    targets = {};

    ebc_run_config rc;
    ebc_run_config_default(&rc);
    rc.eps = cfg.eps;
    rc.delta = cfg.delta;
    rc.seed = cfg.seed;
    rc.bound = cfg.bound == BoundKind::kHoeffding ? 0 : 1;
    rc.allocator = cfg.allocator == AllocatorKind::kUniform ? 0 : 1;
    rc.omega_override = cfg.omega_override;
    rc.calib_samples = cfg.calib_samples_per_worker * static_cast<std::uint64_t>(cfg.ranks) *
                       static_cast<std::uint64_t>(cfg.threads); // engine.cpp:330-344
    rc.diameter_sweeps = cfg.diameter_sweeps;
    rc.device = device;

    ResultHandle rh;
    st = ebc_run(gh.g, &rc, &rh.r);
    if (st != EBC_OK)
        throw_status(st);

    SimRunOutcome out;
    const double *scores = nullptr;
    std::uint64_t n = 0;
    st = ebc_result_scores(rh.r, &scores, &n);
    if (st != EBC_OK)
        throw_status(st);
    out.result.scores.assign(scores, scores + n);
    out.result.tau_total = ebc_result_tau(rh.r);
    out.result.original_ids = g.original_ids();
    ebc_run_stats s;
    st = ebc_result_stats(rh.r, &s);
    if (st != EBC_OK)
        throw_status(st);
    out.stats.epochs = s.epochs;
    out.stats.samples = s.samples;
    out.stats.tau = s.tau;
    out.stats.omega = s.omega;
    out.stats.n0 = s.n0;
    out.stats.calibration_samples = s.calibration_samples;
    out.stats.discarded_samples = s.discarded_samples;
    out.stats.adaptive_s = s.adaptive_s;
    out.stats.diameter_s = s.diameter_s;
    out.stats.calibration_s = s.calibration_s;
    out.stats.check_s = s.check_s;
    out.stats.wall_s = s.wall_s;
    out.stats.n = s.n;
    out.stats.m = s.m;
    out.stats.diameter_upper_bound = s.diameter_upper_bound;
    out.stats.vertex_diameter_bound = s.vertex_diameter_bound;
    out.debug.resize(1);
    out.debug[0].applied_adaptive = s.tau + s.discarded_samples;
    out.debug[0].applied_calibration = s.calibration_samples;
    out.debug[0].discarded = s.discarded_samples;
    out.wall_ms = s.wall_s * 1e3;
    return out;
}

} // namespace epochbc
