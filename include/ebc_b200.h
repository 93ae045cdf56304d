/*
 * ebc_b200.h -- C ABI of the B200-native KADABRA sampling hot path.
 *
 * Drop-in boundary for ONE path of the reference C++ library `epochbc_core`
 * (arxiv/paper_1910_11039, /root/reference/proj): graph load -> run(eps, delta,
 * seed) -> per-vertex score vector + sample count.  The reference has no FFI
 * of its own: its boundary is the C++ API in
 * the headers under proj/include/epochbc/.  Each entry point below names the reference
 * interface it replaces; INTEGRATION.md shows the binding a maintainer adds
 * on the reference side.
 *
 * Conventions
 *   - plain pointers and sizes only; opaque handles are freed by the caller
 *     with the matching *_free; pointers returned by accessors are borrowed
 *     from the handle and stay valid until it is freed.
 *   - vertex ids are 32-bit, row offsets 64-bit (the reference stores both as
 *     u64: include/epochbc/types.hpp:11-12, graph.hpp:49-50).
 *   - no exceptions cross the boundary: every call returns an ebc_status whose
 *     classes mirror the reference's exception classes and CLI exit codes
 *     (types.hpp:15-36, tools/epochbc.cpp:26-30); the message of the last
 *     failure on the calling thread is ebc_last_error().
 *   - everything that computes on the sampling path runs on the GPU.  There is
 *     NO CPU fallback: without a CUDA device those calls fail with
 *     EBC_ERR_CUDA.  Host-only calls (graph ingestion, generators, omega,
 *     calibration) work without a GPU.
 */
#ifndef EBC_B200_H
#define EBC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define EBC_API __attribute__((visibility("default")))
#else
#define EBC_API
#endif

typedef enum ebc_status {
    EBC_OK = 0,
    EBC_ERR_CONFIG = 2,  /* ConfigError / ContractViolation (types.hpp:22-36), CLI exit 2 */
    EBC_ERR_PARSE = 3,   /* ParseError / I/O failure (types.hpp:15-19), CLI exit 3        */
    EBC_ERR_BACKEND = 4, /* BackendFault: collective failure (types.hpp:27-30), CLI exit 4 */
    EBC_ERR_CUDA = 5     /* CUDA runtime failure or no device (no CPU fallback)           */
} ebc_status;

/* Message of the last failed call on this thread ("" if none). */
EBC_API const char *ebc_last_error(void);
EBC_API const char *ebc_version(void);

/* ------------------------------------------------------------------ graph --- */
/* Host-side immutable undirected CSR: replaces epochbc::Graph (graph.hpp:21-52). */
typedef struct ebc_graph ebc_graph;

/* Adopts (copies) an already canonical CSR: rows sorted ascending, symmetric,
 * no loops / duplicates, targets < n.  original_ids may be NULL (identity).
 * validate != 0 checks those invariants and fails with EBC_ERR_CONFIG.
 * Replaces Graph construction + set_original_ids (graph.hpp:27,40). */
EBC_API ebc_status ebc_graph_from_csr(uint64_t n, const uint64_t *offsets, const uint32_t *targets,
                                      const uint64_t *original_ids, int validate, ebc_graph **out);

/* Canonicalises a raw edge list (drops self-loops, deduplicates, symmetrises,
 * sorts rows).  Replaces Graph::from_edges (graph.hpp:27, graph.cpp:14-46). */
EBC_API ebc_status ebc_graph_from_edges(uint64_t n, const uint64_t *src, const uint64_t *dst,
                                        uint64_t count, ebc_graph **out);

/* Text edge list or "EBCG" v1 binary, sniffed by magic; take_lcc != 0 applies
 * largest_connected_component afterwards as the reference CLI always does.
 * Replaces load_graph_file (graph.hpp:74, graph.cpp:204-215) and
 * tools/epochbc.cpp:72-88. */
EBC_API ebc_status ebc_graph_load(const char *path, int take_lcc, ebc_graph **out);

/* Replaces save_graph_file (graph.hpp:75, graph.cpp:217-227). */
EBC_API ebc_status ebc_graph_save(const ebc_graph *g, const char *path, int binary);

/* Replaces largest_connected_component (graph.hpp:80, graph.cpp:229-290). */
EBC_API ebc_status ebc_graph_lcc(const ebc_graph *g, ebc_graph **out);

EBC_API uint64_t ebc_graph_num_vertices(const ebc_graph *g); /* Graph::num_vertices */
EBC_API uint64_t ebc_graph_num_edges(const ebc_graph *g);    /* Graph::num_edges (undirected) */
EBC_API const uint64_t *ebc_graph_offsets(const ebc_graph *g);      /* n+1 */
EBC_API const uint32_t *ebc_graph_targets(const ebc_graph *g);      /* 2m  */
EBC_API const uint64_t *ebc_graph_original_ids(const ebc_graph *g); /* n   */
EBC_API void ebc_graph_free(ebc_graph *g);

/* Seeded synthetic inputs of BASELINE.json's five configs.
 * Counter-based (Philox keyed by (seed, edge index)), so generation is
 * reproducible and independent of thread count.  All return the canonical
 * graph on the full vertex range; apply ebc_graph_lcc afterwards.
 * ebc_gen_rmat follows the quadrant convention of gen_rmat (rmat.cpp:24-42). */
EBC_API ebc_status ebc_gen_erdos_renyi(uint64_t n, uint64_t m, uint64_t seed, ebc_graph **out);
EBC_API ebc_status ebc_gen_rmat(int scale, int edge_factor, double a, double b, double c, double d,
                                uint64_t seed, ebc_graph **out);
EBC_API ebc_status ebc_gen_grid(uint64_t width, uint64_t height, double delete_prob,
                                double shortcut_fraction, uint64_t seed, ebc_graph **out);

/* The same ingestion steps computed on the GPU (`device` = CUDA ordinal, -1 = current device): arcs are
 * sorted and deduplicated with device radix sort, components are found by lock-free hooking, R-MAT arcs
 * are generated in place.  Results equal those of ebc_gen_rmat / ebc_graph_from_edges / ebc_graph_lcc
 * array for array (tie-break of graph.cpp:262-267 and the order-preserving renumbering of :269-289
 * included); `take_lcc` != 0 keeps the data on the device between the two steps.  At R-MAT scale 26
 * the host path takes about 100 s, the device path a few seconds.  They fail with EBC_ERR_CUDA when no
 * device is present. */
EBC_API ebc_status ebc_gen_rmat_device(int scale, int edge_factor, double a, double b, double c, double d,
                                       uint64_t seed, int take_lcc, int device, ebc_graph **out);
EBC_API ebc_status ebc_graph_from_edges_device(uint64_t n, const uint64_t *src, const uint64_t *dst,
                                               uint64_t count, int take_lcc, int device, ebc_graph **out);
EBC_API ebc_status ebc_graph_lcc_device(const ebc_graph *g, int device, ebc_graph **out);

/* ------------------------------------------------- host-side run parameters --- */
/* compute_omega (stopping.hpp:42, stopping.cpp:31-41). */
EBC_API ebc_status ebc_compute_omega(uint64_t vertex_diameter_bound, double eps, double delta,
                                     uint64_t *omega_out);
/* epoch_length (engine.hpp:119-120, engine.cpp:26-31). */
EBC_API ebc_status ebc_epoch_length(int ranks, int threads, double base, double exponent,
                                    uint64_t *n0_out);
/* calibrate (stopping.hpp:49-50, stopping.cpp:43-92).  calib_words = n+1 u64
 * (word 0 tau); allocator 0 = uniform, 1 = weighted; outputs n doubles each. */
EBC_API ebc_status ebc_calibrate(const uint64_t *calib_words, uint64_t n, double delta, int allocator,
                                 double *delta_lower, double *delta_upper);
/* diameter_upper_bound (bfs.hpp:35, bfs.cpp:36-76): out = {upper, lower, vertex_diameter_bound}. */
EBC_API ebc_status ebc_diameter_upper_bound(const ebc_graph *g, int sweeps, uint64_t seed,
                                            uint64_t out[3]);
/* Contiguous shard of the global sample index range [first, first+count) owned by
 * `rank` of `world`.  Pure host arithmetic. */
EBC_API void ebc_shard_range(uint64_t first, uint64_t count, int rank, int world,
                             uint64_t *shard_first, uint64_t *shard_count);

/* -------------------------------------------------------------------- run --- */
/* Sum-allreduce hook for multi-GPU runs: must sum `count` u32 words in place
 * across all ranks.  `buf` is DEVICE memory and the reduction must be enqueued
 * on `cuda_stream` (a cudaStream_t) without blocking the host.
 * Replaces Communicator::ireduce_sum + ibroadcast (comm.hpp:38-51) as used at
 * engine.cpp:149,160,232-262.  Return 0 on success. */
typedef int (*ebc_allreduce_fn)(void *user, void *buf, uint64_t count, void *cuda_stream);

/* Replaces RunConfig (engine.hpp:59-81).  Initialise with ebc_run_config_default. */
typedef struct ebc_run_config {
    double eps;                /* RunConfig::eps   (default 0.001) */
    double delta;              /* RunConfig::delta (default 0.1)   */
    uint64_t seed;             /* RunConfig::seed  (default 1)     */
    int bound;                 /* 0 Hoeffding | 1 empirical Bernstein (stopping.hpp:18-21) */
    int allocator;             /* 0 uniform | 1 weighted (stopping.hpp:23-26)              */
    uint64_t omega_override;   /* RunConfig::omega_override; 0 = formula                   */
    uint64_t calib_samples;    /* total calibration samples (reference: 100 per worker); < 2^32 */
    int diameter_sweeps;       /* RunConfig::diameter_sweeps (default 4)                   */
    uint64_t vertex_diameter_override; /* 0 = run the diameter phase                      */
    uint64_t epoch_samples;    /* samples per epoch over ALL ranks; 0 = derive from omega and the rule; < 2^32
                                  (epoch frames are 32-bit words), else EBC_ERR_CONFIG */
    uint64_t max_epochs;       /* safety cap; 0 = unlimited                                */
    int device;                /* CUDA device ordinal; -1 = current device                 */
    int rank, world_size;      /* this process' shard of every epoch (one process per GPU) */
    ebc_allreduce_fn allreduce; /* required when world_size > 1                            */
    void *allreduce_user;
    uint32_t block_threads;    /* threads cooperating on one sample: 0 = auto              */
    uint32_t slots;            /* concurrent samples (resident CTAs): 0 = auto             */
    uint64_t slot_capacity;    /* settled vertices per side per slot: 0 = auto             */
    int overlap;               /* 1 = sample epoch e+1 while epoch e is reduced/checked    */
    uint32_t items_per_thread; /* adjacency slots per thread per tile (1|2|4): 0 = auto    */
    int materialize_final_level; /* 1 = also settle (label, sigma) every vertex of a sample's LAST level.
                                  * By default a large last level is only scanned: its contact edges give
                                  * the meet set, sigma and order the reference derives (bit-identical
                                  * paths, counters, tau), but vertices that cannot lie on the sampled path
                                  * are not labelled.  Needed for ebc_sampler_last_state and for work
                                  * counters V_set / F_chk / E_lvl that equal the reference algorithm's. */
    int renumber;              /* device-side vertex numbering of the search state: 0 = auto, -1 = never,
                                * 1 = by descending degree class, 2 = by neighbourhood cluster.
                                * On graphs with hubs (max degree >= 1024) the sampler keeps a copy of the graph
                                * renumbered by descending degree, so probes of hub vertices share cache lines; on
                                * large graphs without hubs (grids, road networks) one numbered by clusters of
                                * neighbouring vertices, so the surface of a search ball covers few cache lines.
                                * Purely internal: row order, discovery order, samples, counters and every id
                                * that crosses this interface stay those of the caller's graph. */
    int reserved_sms;          /* SMs the sampling kernel leaves empty so that the frame all-reduce of epoch e (NCCL's
                                * kernel) finds room BESIDE the sampling of epoch e+1 at once -- the overlap of
                                * aggregation with sampling (engine.cpp:145-163).  0 = auto: 4 when world_size > 1 and
                                * overlap != 0 (ebc_nccl_comm_create keeps NCCL to as many CTAs), else none;
                                * -1 = none; k > 0 = k SMs.  Costs k/148 of the sampling rate; without it a kernel
                                * of NCCL's footprint waited 40 us for room at the epoch switch
                                * (tools/overlap_timeline.py, profiles/r02_overlap_timeline.txt). */
    int work_counters;         /* 1 (ebc_run_config_default) = the sampling kernels maintain the device work counters
                                * (ebc_sampler_work, ebc_run_stats.work) and the bookkeeping behind
                                * ebc_sampler_last_state; 0 = production kernels without them: the counters read 0,
                                * results are the same, sampling is 3-10 % faster (the statistics are code every
                                * sample runs through once, and instruction fetch is the kernel's largest stall).
                                * Launches that return records or paths, or materialize_final_level, always use the
                                * kernels with statistics. */
} ebc_run_config;

EBC_API void ebc_run_config_default(ebc_run_config *cfg);

/* Replaces RunStats (engine.hpp:89-110). */
typedef struct ebc_run_stats {
    uint64_t epochs, samples, tau, omega, calibration_samples, discarded_samples, n0;
    uint64_t n, m, diameter_upper_bound, vertex_diameter_bound;
    double adaptive_s, diameter_s, calibration_s, reduce_s, check_s, upload_s, wall_s;
    uint64_t overflow_samples; /* samples re-run in large slots (capacity overflow)        */
    uint64_t work[12];         /* device work counters, see ebc_sampler_work               */
} ebc_run_stats;

typedef struct ebc_result ebc_result;

/* Full pipeline on this process' GPU: diameter -> omega -> calibration ->
 * adaptive epochs -> scores.  Blocking.  Replaces run_pipeline / run_simulated
 * (engine.hpp:142-156, engine.cpp:281-434). */
EBC_API ebc_status ebc_run(const ebc_graph *g, const ebc_run_config *cfg, ebc_result **out);

/* ApproxResult (engine.hpp:83-87): scores[v] = count(v)/tau in dense-id order. */
EBC_API ebc_status ebc_result_scores(const ebc_result *r, const double **scores, uint64_t *n);
EBC_API ebc_status ebc_result_counts(const ebc_result *r, const uint64_t **counts, uint64_t *n);
EBC_API uint64_t ebc_result_tau(const ebc_result *r);
EBC_API ebc_status ebc_result_original_ids(const ebc_result *r, const uint64_t **ids, uint64_t *n);
EBC_API ebc_status ebc_result_stats(const ebc_result *r, ebc_run_stats *stats);
EBC_API void ebc_result_free(ebc_result *r);

/* ------------------------------------------------------------ score files --- */
/* The result / score path of the reference CLI. */
typedef struct ebc_scores ebc_scores;
typedef struct ebc_compare_report { /* CompareReport (score_io.hpp:31-37) */
    double max_abs_error;
    uint64_t vertices_above_eps;
    double top10_overlap, top100_overlap;
    uint64_t vertices;
} ebc_compare_report;

/* write_scores (score_io.cpp:12-21): "# key=value" lines sorted by key, then "id<TAB>%.12g". */
EBC_API ebc_status ebc_scores_write(const char *path, const uint64_t *vertex_ids, const double *scores,
                                    uint64_t n, const char *const *meta_keys, const char *const *meta_values,
                                    uint64_t meta_count);
/* scores_from_result + run_meta + write_scores as cmd_run does (tools/epochbc.cpp:179-190,219-222):
 * header eps, delta, tau, seed, algo; one line per vertex in original-id order of the graph. */
EBC_API ebc_status ebc_result_write_scores(const ebc_result *r, const ebc_run_config *cfg, const char *path);
/* read_scores (score_io.cpp:23-52). */
EBC_API ebc_status ebc_scores_read(const char *path, ebc_scores **out);
EBC_API ebc_status ebc_scores_data(const ebc_scores *s, const uint64_t **vertex_ids, const double **scores,
                                   uint64_t *n);
/* Value of a "# key=value" header entry, or NULL. */
EBC_API const char *ebc_scores_meta(const ebc_scores *s, const char *key);
EBC_API void ebc_scores_free(ebc_scores *s);
/* compare_scores (score_io.cpp:98-122); the reference CLI exits 1 iff max_abs_error > eps. */
EBC_API ebc_status ebc_scores_compare(const ebc_scores *approx, const ebc_scores *exact, double eps,
                                      ebc_compare_report *out);
/* stats_to_json (stats.cpp:7-40): same keys in the same order; fields that have no GPU counterpart
 * (barrier_s, transition_s, bcast_s) are 0.  Writes at most cap bytes incl. NUL; *needed = full size. */
EBC_API ebc_status ebc_result_stats_json(const ebc_result *r, const ebc_run_config *cfg, char *buf, uint64_t cap,
                                         uint64_t *needed);

/* --------------------------------------------------------- device sampler --- */
/* The device-resident pieces ebc_run is built from, exposed for parity tests
 * and benchmarks: replicated CSR + per-slot search state + two epoch frames +
 * the accumulated state S.  Replaces SearchScratch / WorkerState / EpochClock
 * frames (sampler.hpp:26-60, engine.cpp:48-60, epoch.hpp:80-84). */
typedef struct ebc_sampler ebc_sampler;

EBC_API ebc_status ebc_sampler_create(const ebc_graph *g, const ebc_run_config *cfg,
                                      ebc_sampler **out);
EBC_API void ebc_sampler_free(ebc_sampler *s);

/* take_sample + apply_sample (engine.cpp:57-60, sampler.hpp:74-78) for global
 * sample indices [first, first+count) of stream (seed, tag) into epoch frame
 * `frame` (0|1).  Asynchronous on the sampler's stream. */
EBC_API ebc_status ebc_sampler_sample(ebc_sampler *s, uint64_t seed, uint32_t tag, uint64_t first,
                                      uint64_t count, int frame);

/* Per-sample record written by ebc_sampler_sample_debug. */
typedef struct ebc_sample_record {
    uint32_t s, t;
    uint32_t dist;        /* d(s,t), 0xffffffff if unreachable            */
    uint32_t meet;        /* chosen meeting vertex, 0xffffffff if none    */
    uint32_t meet_count;  /* |meet set|                                   */
    uint32_t draws;       /* random draws consumed                        */
    uint32_t path_len;    /* internal vertices                            */
    uint32_t flags;       /* bit0: capacity overflow (re-run in big slot); bit1: the final level was resolved by the
                           * read-only probe (not settled); bit2: a probe found contact edges it could not resolve
                           * (buffer or scratch too small) and the level was expanded instead; bit3: the probed
                           * level had more contact edges than the shared-memory meet path holds (resolved in the
                           * slot's global arrays: config 2 12-20 % of the samples, tools/probe_stats.py);
                           * bit4: at most 32 contact edges, the meet vertex was chosen in registers */
    uint64_t weight_lo, weight_hi; /* total meet weight (saturating u128) */
} ebc_sample_record;

/* Test hook: sample_pair + sample_shortest_path (sampler.cpp:45-52, 54-164)
 * for `count` samples; pairs_or_null = 2*count u32 explicit (s,t) (then no
 * pair draws are consumed).  Host outputs: records[count]; paths holds
 * path_stride u32 per sample (internal vertices in s..t order).  Also applies
 * the samples to epoch frame `frame`.  Synchronous. */
EBC_API ebc_status ebc_sampler_sample_debug(ebc_sampler *s, uint64_t seed, uint32_t tag,
                                            uint64_t first, uint64_t count,
                                            const uint32_t *pairs_or_null, int frame,
                                            ebc_sample_record *records, uint32_t *paths,
                                            uint64_t path_stride);

/* Per-side search state of the LAST sample of a 1-sample debug call made with
 * slots == 1: dist (0xffffffff unvisited) and sigma (0 unvisited), n entries. */
EBC_API ebc_status ebc_sampler_last_state(ebc_sampler *s, int side, uint32_t *dist_out,
                                          uint64_t *sigma_out);

/* Installs the stopping parameters (StoppingParams, stopping.hpp:30-36).
 * delta_lower/upper: n doubles (host).  ln(1/delta_v) resp. ln(2/delta_v) are
 * evaluated on the host once (glibc, as the reference does per call at
 * stopping.cpp:103,106) so the device test uses only correctly rounded
 * IEEE operations. */
EBC_API ebc_status ebc_sampler_set_stopping(ebc_sampler *s, double eps, uint64_t omega,
                                            const double *delta_lower, const double *delta_upper,
                                            int bound);

/* S += frame (StateFrame::add, state_frame.hpp:29-33), frame := 0
 * (collect_epoch, epoch.cpp:66-81), then check_stop(S) (stopping.cpp:125-142)
 * on the device.  If allreduce != NULL the frame is summed across ranks first.
 * stop_out receives 0/1.  Synchronous. */
EBC_API ebc_status ebc_sampler_fold_and_check(ebc_sampler *s, int frame, int *stop_out);

/* Copies frames to the host: which = 0|1 epoch frame (n+1 u32 widened to u64),
 * 2 = accumulated S.  words_out has n+1 u64 (word 0 = tau). */
EBC_API ebc_status ebc_sampler_read_frame(ebc_sampler *s, int which, uint64_t *words_out);
/* Overwrites S from host words (test hook for check_stop parity). */
EBC_API ebc_status ebc_sampler_write_state(ebc_sampler *s, const uint64_t *words);
EBC_API ebc_status ebc_sampler_clear(ebc_sampler *s); /* zero frames and S */

/* Device-side work counters accumulated since creation / last reset
 * (SURVEY.md section 8d): E_bfs, E_lvl, V_exp, V_set, F_chk, M, S_walk, E_walk,
 * P_walk, L, levels, samples. */
EBC_API ebc_status ebc_sampler_work(ebc_sampler *s, uint64_t work_out[12], int reset);

/* Timing on the sampler's stream with CUDA events: mark(i) records event i
 * (0..7); elapsed(i,j) synchronises event j and returns milliseconds. */
EBC_API ebc_status ebc_sampler_mark(ebc_sampler *s, int event);
EBC_API ebc_status ebc_sampler_elapsed_ms(ebc_sampler *s, int from_event, int to_event, float *ms);
EBC_API ebc_status ebc_sampler_sync(ebc_sampler *s);
/* slots, block_threads, slot_capacity, device bytes in use, SM count,
 * launches (bits 0-47) | renumbered (bits 48-51) | fixed-stride rows in use (bit 52), of four entries (bit 53),
 * of eight with a 16-byte copy for the expansion (bit 54) | items_per_thread (bits 56-63). */
EBC_API ebc_status ebc_sampler_info(ebc_sampler *s, uint64_t info_out[6]);
/* The sampler's cudaStream_t and the device address of epoch frame 0|1
 * (for callers that aggregate frames themselves, e.g. NCCL in bench.py). */
EBC_API ebc_status ebc_sampler_stream(ebc_sampler *s, void **cuda_stream_out);
EBC_API ebc_status ebc_sampler_frame_ptr(ebc_sampler *s, int frame, void **dev_ptr_out,
                                         uint64_t *words_out);

/* GPU level-synchronous BFS used by the diameter phase (bfs.hpp:19, bfs.cpp:9-34):
 * dist_out may be NULL; out = {farthest (lowest id on ties), eccentricity, reached}. */
EBC_API ebc_status ebc_sampler_bfs(ebc_sampler *s, uint32_t source, uint32_t *dist_out,
                                   uint64_t out[3]);

/* Device buffers of destroyed samplers / finished runs are cached per process and reused by the next
 * run (cudaMalloc/cudaFree of ~10 GB costs more than sampling a small input); this releases them. */
EBC_API void ebc_release_device_cache(void);

/* L2 flush helper for benchmarks: writes a buffer larger than L2 on the sampler's stream. */
EBC_API ebc_status ebc_sampler_flush_l2(ebc_sampler *s);

/* ------------------------------------------------------- native NCCL hook --- */
/* A ready-made ebc_allreduce_fn over NCCL (NVLink 5 / NVSwitch), so that a C or C++ host (one process
 * per GPU) needs nothing but this library on the data path: no callback into another runtime per epoch.
 * Replaces the reduce + broadcast of Communicator (comm.hpp:38-51; MpiCommunicator, mpi_comm.cpp) for the
 * epoch frames.  libnccl.so.2 is resolved at run time (dlopen; a copy already loaded by the process, e.g.
 * torch's, is reused), so the library itself has no link-time NCCL dependency.
 *
 *   rank 0: ebc_nccl_unique_id(id);  send the 128 bytes to every rank (MPI_Bcast, a file, a socket ...)
 *   all   : ebc_nccl_comm_create(id, rank, world, device, &comm);
 *           cfg.allreduce = ebc_nccl_allreduce;  cfg.allreduce_user = comm;  cfg.rank / world_size = ...
 *           ebc_run(g, &cfg, &res);   ...   ebc_nccl_comm_free(comm);
 */
typedef struct ebc_nccl_comm ebc_nccl_comm;
#define EBC_NCCL_UNIQUE_ID_BYTES 128
EBC_API ebc_status ebc_nccl_unique_id(void *id_out /* EBC_NCCL_UNIQUE_ID_BYTES */);
/* Collective over all `world_size` ranks (ncclCommInitRank).  device = CUDA ordinal, -1 = current. */
EBC_API ebc_status ebc_nccl_comm_create(const void *id, int rank, int world_size, int device,
                                        ebc_nccl_comm **out);
/* ebc_allreduce_fn: in-place ncclAllReduce(sum, u32) of `count` words at device address `buf`, enqueued
 * on `cuda_stream`; `user` is the ebc_nccl_comm.  Returns 0 on success (message: ebc_last_error()). */
EBC_API int ebc_nccl_allreduce(void *user, void *buf, uint64_t count, void *cuda_stream);
EBC_API void ebc_nccl_comm_free(ebc_nccl_comm *c);

#ifdef __cplusplus
}
#endif
#endif /* EBC_B200_H */
