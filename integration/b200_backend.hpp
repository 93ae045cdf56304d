// Reference-side binding of libebc_b200.so: the ONE translation unit (b200_backend.cpp) a maintainer of the
// reference adds to proj/src, declared here.  Compiled in this repository against the reference's unmodified
// headers (integration/Makefile) so that it is known to build and to give the reference's results.
#pragma once

#include "epochbc/engine.hpp" // reference: RunConfig, SimRunOutcome (engine.hpp:59-81, 145-151)
#include "epochbc/graph.hpp"

namespace epochbc {

// Drop-in for run_simulated(g, cfg, opts) (engine.hpp:153-156, engine.cpp:405-434; call site
// tools/epochbc.cpp:218) on one B200: same inputs, same SimRunOutcome, the reference's exception classes.
// cfg.ranks / cfg.threads only scale the calibration sample count (engine.cpp:330-344), as in the reference.
SimRunOutcome run_b200(const Graph &g, const RunConfig &cfg, int device = 0);

} // namespace epochbc
