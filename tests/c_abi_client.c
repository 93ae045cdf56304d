/* A plain-C client of include/ebc_b200.h -- what the reference-side adapter of INTEGRATION.md compiles to:
 * graph -> run(eps, delta, seed) -> scores / tau / stats, no Python, no C++ types.
 * usage: c_abi_client <scale> <eps>      prints one line "n m tau epochs checksum" or "status <code>: <message>" */
#include <inttypes.h>
#include <stdio.h>
#include <stdlib.h>

#include "ebc_b200.h"

static int fail(const char *what, ebc_status st) {
    printf("status %d: %s: %s\n", (int)st, what, ebc_last_error());
    return (int)st;
}

int main(int argc, char **argv) {
    const int scale = argc > 1 ? atoi(argv[1]) : 12;
    const double eps = argc > 2 ? atof(argv[2]) : 0.05;
    ebc_graph *full = NULL, *g = NULL;
    ebc_status st = ebc_gen_rmat(scale, 16, 0.57, 0.19, 0.19, 0.05, 2, &full);
    if (st != EBC_OK)
        return fail("ebc_gen_rmat", st);
    st = ebc_graph_lcc(full, &g);
    ebc_graph_free(full);
    if (st != EBC_OK)
        return fail("ebc_graph_lcc", st);

    ebc_run_config cfg;
    ebc_run_config_default(&cfg);
    cfg.eps = eps;
    cfg.delta = 0.1;
    cfg.seed = 7;
    ebc_result *res = NULL;
    st = ebc_run(g, &cfg, &res);
    if (st != EBC_OK) {
        ebc_graph_free(g);
        return fail("ebc_run", st);
    }
    const double *scores = NULL;
    uint64_t n = 0;
    ebc_result_scores(res, &scores, &n);
    ebc_run_stats stats;
    ebc_result_stats(res, &stats);
    double checksum = 0.0;
    for (uint64_t v = 0; v < n; ++v)
        checksum += scores[v];
    printf("%" PRIu64 " %" PRIu64 " %" PRIu64 " %" PRIu64 " %.12g\n", ebc_graph_num_vertices(g), ebc_graph_num_edges(g),
           ebc_result_tau(res), stats.epochs, checksum);
    ebc_result_free(res);
    ebc_graph_free(g);
    return 0;
}
