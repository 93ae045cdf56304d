/*
 * TEST INFRASTRUCTURE -- CPU oracle for the KADABRA sampling hot path.
 *
 * Plain-C restatement of the reference algorithm (arxiv/paper_1910_11039,
 * /root/reference/proj), operating directly on the product's CSR layout
 * (u64 offsets, u32 targets, rows sorted ascending).  It exists so that
 *   (1) the CUDA path can be checked bit-for-bit on machines where
 *       /root/reference is absent (the GPU box), and
 *   (2) inputs the unmodified reference cannot ingest (u64 targets + 16-byte
 *       pair lists) still have a checker.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library; the shipped product never does.
 *
 * PARITY PIN: this file is validated against the UNMODIFIED reference
 * sampler.cpp / stopping.cpp compiled with the Philox stream shim
 * (oracle/_ref/libebc_ref_shim.so, built by oracle/Makefile from the sources
 * under /root/reference) on >= 10^4 random (graph, s, t, stream) cases by
 * tests/test_oracle_vs_reference.py, and against golden vectors generated
 * from that same build (tests/golden/, generator tests/golden/make_golden.py).
 * The reference ships no tests of its own; its SPEC.md
 * worked examples are checked in tests/test_spec_examples.py.
 *
 * Every function cites the reference lines it follows.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "ebc_philox.h"

typedef unsigned __int128 u128;

#define EBC_UNREACHED 0xffffffffu

/* ---- work counters (algorithmic bytes per sample) ---- */
enum {
    EBC_W_E_BFS = 0, /* adjacency entries scanned by the BFS            */
    EBC_W_E_LVL,     /* ... of which dist[v]==next_depth (sigma RMW)     */
    EBC_W_V_EXP,     /* expanded frontier vertices                       */
    EBC_W_V_SET,     /* settled vertices incl. s and t                   */
    EBC_W_F_CHK,     /* new-frontier vertices tested against other side  */
    EBC_W_M,         /* meet-set size                                    */
    EBC_W_S_WALK,    /* walk steps                                       */
    EBC_W_E_WALK,    /* sum of deg over walk vertices (one fused pass)   */
    EBC_W_P_WALK,    /* predecessor hits during the walk                 */
    EBC_W_L,         /* internal vertices                                */
    EBC_W_LEVELS,    /* BFS levels expanded                              */
    EBC_W_COUNT
};

typedef struct {
    uint32_t *dist;
    uint64_t *sigma;
    uint32_t *stamp;
    uint32_t *frontier, *next;
    uint64_t fsize, nsize;
    uint64_t pending_edges;
    uint32_t depth;
} ebc_side;

typedef struct {
    uint64_t n;
    const uint64_t *offsets;
    const uint32_t *targets;
    ebc_side side[2];
    uint32_t *meet;
    uint64_t meet_size;
    uint32_t round;
    uint64_t work[EBC_W_COUNT];
    uint32_t last_dist; /* d(s,t) of the last sample, EBC_UNREACHED if none */
    uint32_t last_meet;
} ebc_oracle;

/* ------------------------------------------------------------------------- */
/* sampler.cpp:11-13 */
static uint64_t sat_add_u64(uint64_t a, uint64_t b) { return a > UINT64_MAX - b ? UINT64_MAX : a + b; }

/* sampler.cpp:15-18 */
static u128 sat_add_u128(u128 a, u128 b) {
    u128 s = a + b;
    return s < a ? ~(u128)0 : s;
}

/* sampler.cpp:21-30: one next_below when the bound fits 64 bits, otherwise
 * 128-bit rejection sampling on (hi = next_u64) << 64 | (lo = next_u64). */
static u128 uniform_below_u128(ebc_stream *rng, u128 bound) {
    if (bound <= (u128)UINT64_MAX)
        return ebc_stream_below(rng, (uint64_t)bound);
    const u128 all = ~(u128)0;
    const u128 reject_from = all - (all % bound);
    for (;;) {
        u128 hi = ebc_stream_u64(rng);
        u128 lo = ebc_stream_u64(rng);
        u128 r = (hi << 64) | lo;
        if (r < reject_from)
            return r % bound;
    }
}

/* sampler.cpp:34-43 (SearchScratch ctor) */
ebc_oracle *ebc_oracle_create(uint64_t n, const uint64_t *offsets, const uint32_t *targets) {
    ebc_oracle *o = (ebc_oracle *)calloc(1, sizeof(ebc_oracle));
    if (!o)
        return NULL;
    o->n = n;
    o->offsets = offsets;
    o->targets = targets;
    for (int k = 0; k < 2; ++k) {
        ebc_side *sd = &o->side[k];
        sd->dist = (uint32_t *)calloc(n ? n : 1, 4);
        sd->sigma = (uint64_t *)calloc(n ? n : 1, 8);
        sd->stamp = (uint32_t *)calloc(n ? n : 1, 4);
        sd->frontier = (uint32_t *)malloc((n ? n : 1) * 4);
        sd->next = (uint32_t *)malloc((n ? n : 1) * 4);
    }
    o->meet = (uint32_t *)malloc((n ? n : 1) * 4);
    o->last_dist = EBC_UNREACHED;
    return o;
}

void ebc_oracle_destroy(ebc_oracle *o) {
    if (!o)
        return;
    for (int k = 0; k < 2; ++k) {
        free(o->side[k].dist);
        free(o->side[k].sigma);
        free(o->side[k].stamp);
        free(o->side[k].frontier);
        free(o->side[k].next);
    }
    free(o->meet);
    free(o);
}

void ebc_oracle_work(const ebc_oracle *o, uint64_t *out) { memcpy(out, o->work, sizeof(o->work)); }
void ebc_oracle_work_reset(ebc_oracle *o) { memset(o->work, 0, sizeof(o->work)); }
int ebc_oracle_work_count(void) { return EBC_W_COUNT; }

static inline uint64_t deg(const ebc_oracle *o, uint32_t v) { return o->offsets[v + 1] - o->offsets[v]; }

/* sampler.hpp:49-53 */
static inline void settle(ebc_side *sd, uint32_t v, uint32_t d, uint32_t cur) {
    sd->stamp[v] = cur;
    sd->dist[v] = d;
    sd->sigma[v] = 0;
}

/* sampler.cpp:45-52 */
void ebc_oracle_sample_pair(uint64_t n, ebc_stream *rng, uint32_t *s, uint32_t *t) {
    uint64_t a = ebc_stream_below(rng, n);
    uint64_t b = ebc_stream_below(rng, n - 1);
    if (b >= a)
        ++b;
    *s = (uint32_t)a;
    *t = (uint32_t)b;
}

/* sampler.cpp:135-155: sigma-weighted walk from `from` toward the side's root.
 * Emits the vertices strictly between (in walk order) into out[*len..]. */
static void walk(ebc_oracle *o, const ebc_side *sd, uint32_t cur, uint32_t from, ebc_stream *rng,
                 uint32_t *out, uint64_t *len) {
    uint32_t u = from;
    while (sd->dist[u] > 0) {
        const uint64_t b = o->offsets[u], e = o->offsets[u + 1];
        u128 total = 0;
        for (uint64_t i = b; i < e; ++i) { /* :139-141 */
            uint32_t w = o->targets[i];
            if (sd->stamp[w] == cur && sd->dist[w] + 1 == sd->dist[u]) {
                total += sd->sigma[w];
                o->work[EBC_W_P_WALK]++;
            }
        }
        o->work[EBC_W_S_WALK]++;
        o->work[EBC_W_E_WALK] += e - b;
        u128 r = uniform_below_u128(rng, total); /* :142 */
        for (uint64_t i = b; i < e; ++i) {       /* :143-151 */
            uint32_t w = o->targets[i];
            if (sd->stamp[w] == cur && sd->dist[w] + 1 == sd->dist[u]) {
                if (r < sd->sigma[w]) {
                    u = w;
                    break;
                }
                r -= sd->sigma[w];
            }
        }
        if (sd->dist[u] > 0) /* :152-153 */
            out[(*len)++] = u;
    }
}

/* sampler.cpp:54-164.  Returns the number of internal vertices written to
 * path_out (path order s..t, endpoints excluded).  path_out needs room for n. */
uint64_t ebc_oracle_sample_path(ebc_oracle *o, uint32_t s, uint32_t t, ebc_stream *rng,
                                uint32_t *path_out) {
    ebc_side *fwd = &o->side[0], *bwd = &o->side[1];
    const uint32_t cur = ++o->round; /* :63 */
    o->last_dist = EBC_UNREACHED;
    o->last_meet = EBC_UNREACHED;
    o->meet_size = 0;

    /* :65-76 */
    settle(fwd, s, 0, cur);
    fwd->sigma[s] = 1;
    fwd->frontier[0] = s;
    fwd->fsize = 1;
    fwd->pending_edges = deg(o, s);
    fwd->depth = 0;
    settle(bwd, t, 0, cur);
    bwd->sigma[t] = 1;
    bwd->frontier[0] = t;
    bwd->fsize = 1;
    bwd->pending_edges = deg(o, t);
    bwd->depth = 0;
    o->work[EBC_W_V_SET] += 2;

    int found = 0;
    while (!found) { /* :81 */
        if (fwd->fsize == 0 || bwd->fsize == 0)
            return 0; /* :82-83 unreachable: empty sample, still counts */
        ebc_side *ex = fwd->pending_edges <= bwd->pending_edges ? fwd : bwd; /* :84, tie -> fwd */
        ebc_side *ot = ex == fwd ? bwd : fwd;

        ex->nsize = 0;
        uint64_t next_pending = 0;
        const uint32_t next_depth = ex->depth + 1;
        o->work[EBC_W_LEVELS]++;
        for (uint64_t fi = 0; fi < ex->fsize; ++fi) { /* :90-100 */
            const uint32_t u = ex->frontier[fi];
            const uint64_t b = o->offsets[u], e = o->offsets[u + 1];
            o->work[EBC_W_V_EXP]++;
            o->work[EBC_W_E_BFS] += e - b;
            for (uint64_t i = b; i < e; ++i) {
                const uint32_t v = o->targets[i];
                if (ex->stamp[v] != cur) {
                    settle(ex, v, next_depth, cur);
                    ex->next[ex->nsize++] = v;
                    next_pending += deg(o, v);
                    o->work[EBC_W_V_SET]++;
                }
                if (ex->dist[v] == next_depth) {
                    ex->sigma[v] = sat_add_u64(ex->sigma[v], ex->sigma[u]);
                    o->work[EBC_W_E_LVL]++;
                }
            }
        }
        { /* :101-103 */
            uint32_t *tmp = ex->frontier;
            ex->frontier = ex->next;
            ex->next = tmp;
            ex->fsize = ex->nsize;
            ex->pending_edges = next_pending;
            ex->depth = next_depth;
        }

        uint32_t best = EBC_UNREACHED; /* :105-108 */
        for (uint64_t fi = 0; fi < ex->fsize; ++fi) {
            uint32_t v = ex->frontier[fi];
            if (ot->stamp[v] == cur && ot->dist[v] < best)
                best = ot->dist[v];
        }
        o->work[EBC_W_F_CHK] += ex->fsize;
        if (best != EBC_UNREACHED) { /* :109-115 */
            o->meet_size = 0;
            for (uint64_t fi = 0; fi < ex->fsize; ++fi) {
                uint32_t v = ex->frontier[fi];
                if (ot->stamp[v] == cur && ot->dist[v] == best)
                    o->meet[o->meet_size++] = v;
            }
            found = 1;
            o->last_dist = ex->depth + best;
        }
    }
    o->work[EBC_W_M] += o->meet_size;

    /* :121-133 meet vertex proportional to sigma_s * sigma_t */
    u128 total_weight = 0;
    for (uint64_t i = 0; i < o->meet_size; ++i) {
        uint32_t v = o->meet[i];
        total_weight = sat_add_u128(total_weight, (u128)fwd->sigma[v] * bwd->sigma[v]);
    }
    u128 pick = uniform_below_u128(rng, total_weight);
    uint32_t meet = o->meet[o->meet_size - 1];
    for (uint64_t i = 0; i < o->meet_size; ++i) {
        uint32_t v = o->meet[i];
        u128 w = (u128)fwd->sigma[v] * bwd->sigma[v];
        if (pick < w) {
            meet = v;
            break;
        }
        pick -= w;
    }
    o->last_meet = meet;

    /* :157-163 path order s .. meet .. t */
    uint64_t len = 0;
    walk(o, fwd, cur, meet, rng, path_out, &len);
    for (uint64_t i = 0; i < len / 2; ++i) {
        uint32_t tmp = path_out[i];
        path_out[i] = path_out[len - 1 - i];
        path_out[len - 1 - i] = tmp;
    }
    if (meet != s && meet != t)
        path_out[len++] = meet;
    walk(o, bwd, cur, meet, rng, path_out, &len);
    o->work[EBC_W_L] += len;
    return len;
}

/* One keyed sample: stream (seed, tag, index); draws 0.. = pair, then path
 * (engine.cpp:57-60 take_sample).  info_out: s, t, d(s,t) or 0xffffffff, meet
 * vertex or 0xffffffff, draws consumed. */
uint64_t ebc_oracle_sample(ebc_oracle *o, uint64_t seed, uint32_t tag, uint64_t index,
                           int explicit_pair, uint32_t s, uint32_t t, uint32_t *path_out,
                           uint64_t *info_out) {
    ebc_stream rng;
    ebc_stream_init(&rng, seed, tag, index);
    if (!explicit_pair)
        ebc_oracle_sample_pair(o->n, &rng, &s, &t);
    uint64_t len = ebc_oracle_sample_path(o, s, t, &rng, path_out);
    if (info_out) {
        info_out[0] = s;
        info_out[1] = t;
        info_out[2] = o->last_dist;
        info_out[3] = o->last_meet;
        info_out[4] = rng.draw;
    }
    return len;
}

/* Per-side dist / sigma of the last sample (0xffffffff / 0 where unvisited). */
void ebc_oracle_last_state(const ebc_oracle *o, int side, uint32_t *dist_out, uint64_t *sigma_out) {
    const ebc_side *sd = &o->side[side];
    for (uint64_t v = 0; v < o->n; ++v) {
        int vis = sd->stamp[v] == o->round;
        dist_out[v] = vis ? sd->dist[v] : EBC_UNREACHED;
        sigma_out[v] = vis ? sd->sigma[v] : 0;
    }
}

uint64_t ebc_oracle_last_meet_set(const ebc_oracle *o, uint32_t *out, uint64_t cap) {
    for (uint64_t i = 0; i < o->meet_size && i < cap; ++i)
        out[i] = o->meet[i];
    return o->meet_size;
}

/* apply_sample (sampler.hpp:74-78) over samples [first, first+count) into a
 * frame of n+1 u64 words (state_frame.hpp:21-25: word 0 = tau, word v+1 = c[v]);
 * the frame is accumulated into (StateFrame::add, state_frame.hpp:29-33). */
void ebc_oracle_accumulate(ebc_oracle *o, uint64_t seed, uint32_t tag, uint64_t first,
                           uint64_t count, uint64_t *frame_words) {
    uint32_t *path = (uint32_t *)malloc((o->n ? o->n : 1) * 4);
    for (uint64_t i = 0; i < count; ++i) {
        uint64_t len = ebc_oracle_sample(o, seed, tag, first + i, 0, 0, 0, path, NULL);
        frame_words[0] += 1;
        for (uint64_t k = 0; k < len; ++k)
            frame_words[(uint64_t)path[k] + 1] += 1;
    }
    free(path);
}

/* ------------------------------------------------------------------------- */
/* stopping.cpp:31-41 */
uint64_t ebc_oracle_compute_omega(uint64_t vd, double eps, double delta) {
    double log_term = 0.0;
    if (vd > 2)
        log_term = floor(log2((double)(vd - 2)));
    double omega = (0.5 / (eps * eps)) * (log_term + 1.0 + log(1.0 / delta));
    return (uint64_t)ceil(omega);
}

/* engine.cpp:26-31 */
uint64_t ebc_oracle_epoch_length(int ranks, int threads, double base, double exponent) {
    double workers = (double)ranks * threads;
    long long n0 = llround(base / pow(workers, exponent));
    return n0 < 1 ? 1 : (uint64_t)n0;
}

/* stopping.cpp:43-92; kind 0 uniform, 1 weighted. */
void ebc_oracle_calibrate(const uint64_t *calib_words, uint64_t n, double delta, int kind,
                          double *dl, double *du) {
    const uint64_t tau = calib_words[0];
    int uniform = kind == 0 || tau == 0;
    if (!uniform) {
        double weight_sum = 0.0;
        for (uint64_t v = 0; v < n; ++v)
            weight_sum += sqrt((double)calib_words[v + 1] / (double)tau);
        if (weight_sum == 0.0) {
            uniform = 1;
        } else {
            const double budget = delta * (1.0 - 1e-6);
            const double floor_per_vertex = delta / (2.0 * (double)n);
            const double spare = budget - floor_per_vertex * (double)n;
            for (uint64_t v = 0; v < n; ++v) {
                double w = sqrt((double)calib_words[v + 1] / (double)tau);
                double combined = floor_per_vertex + spare * (w / weight_sum);
                dl[v] = combined / 2.0;
                du[v] = combined / 2.0;
            }
        }
    }
    if (uniform) {
        const double per_side = delta / (2.0 * (double)n);
        for (uint64_t v = 0; v < n; ++v) {
            dl[v] = per_side;
            du[v] = per_side;
        }
    }
    long double total = 0.0L; /* :82-91 rounding guard */
    for (uint64_t v = 0; v < n; ++v)
        total += (long double)dl[v] + du[v];
    if (total > (long double)delta) {
        double scale = (double)((long double)delta / total) * (1.0 - 1e-12);
        for (uint64_t v = 0; v < n; ++v) {
            dl[v] *= scale;
            du[v] *= scale;
        }
    }
}

/* stopping.cpp:96-111; bound 0 Hoeffding, 1 empirical Bernstein. */
double ebc_oracle_bound_width(double b, double delta_v, uint64_t tau, int bound) {
    const double t = (double)tau;
    if (bound == 0)
        return sqrt(log(1.0 / delta_v) / (2.0 * t));
    const double var = b * (1.0 - b);
    const double l = log(2.0 / delta_v);
    return sqrt(2.0 * var * l / t) + 7.0 * l / (3.0 * (t - 1.0));
}

/* stopping.cpp:125-142 */
int ebc_oracle_check_stop(const uint64_t *words, uint64_t n, double eps, uint64_t omega,
                          const double *dl, const double *du, int bound) {
    const uint64_t tau = words[0];
    if (tau >= omega)
        return 1;
    if (tau < 2)
        return 0;
    for (uint64_t v = 0; v < n; ++v) {
        double b = (double)words[v + 1] / (double)tau;
        if (ebc_oracle_bound_width(b, dl[v], tau, bound) >= eps)
            return 0;
        if (ebc_oracle_bound_width(b, du[v], tau, bound) >= eps)
            return 0;
    }
    return 1;
}

/* Epoch replay of the adaptive phase as the GPU build schedules it (SURVEY.md
 * section 8e; semantics of engine.cpp:124-167): epoch e covers global sample
 * indices [e*B, (e+1)*B); after each epoch S += S_epoch and check_stop(S).
 * Returns the number of epochs folded into S at the stop (stop epoch + 1);
 * S_words (n+1 u64, zero on entry) holds the final aggregate. */
uint64_t ebc_oracle_run_epochs(ebc_oracle *o, uint64_t seed, uint32_t tag, uint64_t epoch_samples,
                               uint64_t max_epochs, double eps, uint64_t omega, const double *dl,
                               const double *du, int bound, uint64_t *S_words) {
    uint64_t e = 0;
    for (; e < max_epochs; ++e) {
        ebc_oracle_accumulate(o, seed, tag, e * epoch_samples, epoch_samples, S_words);
        if (ebc_oracle_check_stop(S_words, o->n, eps, omega, dl, du, bound))
            return e + 1;
    }
    return e;
}

/* ------------------------------------------------------------------------- */
/* bfs.cpp:9-34.  out = {farthest, eccentricity, reached}. */
void ebc_oracle_bfs(const ebc_oracle *o, uint32_t source, uint32_t *dist, uint32_t *queue,
                    uint64_t *out) {
    const uint64_t n = o->n;
    for (uint64_t v = 0; v < n; ++v)
        dist[v] = EBC_UNREACHED;
    uint64_t head = 0, tail = 0;
    queue[tail++] = source;
    dist[source] = 0;
    uint32_t far = source, ecc = 0;
    for (; head < tail; ++head) {
        uint32_t u = queue[head];
        uint32_t du = dist[u];
        if (du > ecc || (du == ecc && u < far)) {
            ecc = du;
            far = u;
        }
        for (uint64_t i = o->offsets[u]; i < o->offsets[u + 1]; ++i) {
            uint32_t v = o->targets[i];
            if (dist[v] == EBC_UNREACHED) {
                dist[v] = du + 1;
                queue[tail++] = v;
            }
        }
    }
    out[0] = far;
    out[1] = ecc;
    out[2] = tail;
}

/* mt19937_64 (Matsumoto & Nishimura) restated from the published recurrence;
 * the reference reaches it through std::mt19937_64 (rng.hpp:32,52). */
typedef struct {
    uint64_t mt[312];
    int idx;
} ebc_mt64;

static void mt64_seed(ebc_mt64 *g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(ebc_mt64 *g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t y = g->mt[(i + 156) % 312] ^ (x >> 1);
            if (x & 1)
                y ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = y;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* libstdc++ (GCC >= 11) uniform_int_distribution<uint64_t>(0, bound-1) on a
 * full-range 64-bit engine: Lemire's nearly-divisionless method on a 128-bit
 * product; this is what rng.hpp:41-44 evaluates to with the toolchain the
 * reference was measured with (g++ 13.3). */
static uint64_t mt64_below(ebc_mt64 *g, uint64_t bound) {
    u128 m = (u128)mt64_next(g) * bound;
    uint64_t lo = (uint64_t)m;
    if (lo < bound) {
        uint64_t t = (0 - bound) % bound;
        while (lo < t) {
            m = (u128)mt64_next(g) * bound;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* rng.hpp:12-27 */
static uint64_t splitmix64(uint64_t *state) {
    uint64_t z = (*state += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

uint64_t ebc_oracle_mix_seed(uint64_t master, uint64_t rank, uint64_t thread) {
    uint64_t s = master;
    uint64_t h = splitmix64(&s);
    s ^= rank * 0x2545f4914f6cdd1dULL;
    h ^= splitmix64(&s);
    s ^= thread * 0x9e3779b97f4a7c15ULL;
    h ^= splitmix64(&s);
    return h;
}

/* Draws from Rng::stream(master, rank, thread) (rng.hpp:34-46): bound 0 =>
 * next_u64, else next_below(bound). */
void ebc_oracle_mt_draws(uint64_t master, uint64_t rank, uint64_t thread, const uint64_t *bounds,
                         uint64_t count, uint64_t *out) {
    ebc_mt64 g;
    mt64_seed(&g, ebc_oracle_mix_seed(master, rank, thread));
    for (uint64_t i = 0; i < count; ++i)
        out[i] = bounds[i] == 0 ? mt64_next(&g) : mt64_below(&g, bounds[i]);
}

/* bfs.cpp:36-76.  out = {upper, lower, vertex_diameter_bound}; returns -1 if
 * the graph is disconnected (the reference throws ConfigError). */
int ebc_oracle_diameter(const ebc_oracle *o, int sweeps, uint64_t seed, uint64_t *out) {
    const uint64_t n = o->n;
    uint32_t start = 0;
    for (uint64_t v = 1; v < n; ++v)
        if (deg(o, (uint32_t)v) > deg(o, start))
            start = (uint32_t)v;
    ebc_mt64 g;
    mt64_seed(&g, ebc_oracle_mix_seed(seed, 0, 0x00d1a0ULL));
    uint64_t upper = UINT64_MAX, lower = 0;
    char *used = (char *)calloc(n ? n : 1, 1);
    uint32_t *dist = (uint32_t *)malloc((n ? n : 1) * 4);
    uint32_t *queue = (uint32_t *)malloc((n ? n : 1) * 4);
    uint32_t v = start;
    int rc = 0;
    for (int i = 0; i < sweeps; ++i) {
        uint64_t r[3];
        ebc_oracle_bfs(o, v, dist, queue, r);
        if (r[2] != n) {
            rc = -1;
            break;
        }
        if (2 * r[1] < upper)
            upper = 2 * r[1];
        if (r[1] > lower)
            lower = r[1];
        used[v] = 1;
        if (n == 1)
            break;
        v = (uint32_t)r[0];
        for (int tries = 0; used[v] && tries < 16; ++tries)
            v = (uint32_t)mt64_below(&g, n);
        if (used[v])
            break;
    }
    free(used);
    free(dist);
    free(queue);
    out[0] = upper;
    out[1] = lower;
    out[2] = upper + 1;
    return rc;
}

/* Known-answer hook for the Philox block function itself. */
void ebc_oracle_philox_block(const uint32_t *ctr, const uint32_t *key, uint32_t *out) {
    ebc_philox4x32_10(ctr, key, out);
}

void ebc_oracle_stream_draws(uint64_t seed, uint32_t tag, uint64_t index, const uint64_t *bounds,
                             uint64_t count, uint64_t *out) {
    ebc_stream s;
    ebc_stream_init(&s, seed, tag, index);
    for (uint64_t i = 0; i < count; ++i)
        out[i] = bounds[i] == 0 ? ebc_stream_u64(&s) : ebc_stream_below(&s, bounds[i]);
}

/* Exact betweenness by Brandes' dependency accumulation, normalised as the
 * reference does (oracle.hpp:10-11: b(x) = 1/(n(n-1)) * sum over ordered pairs
 * s != t of sigma_st(x)/sigma_st, endpoints excluded).  Restated from the
 * published algorithm (Brandes 2001); checked against brandes_exact
 * (oracle.cpp:61-102) in tests/test_oracle_vs_reference.py.  Sources
 * [src_begin, src_end) are accumulated into scores_out (caller zeroes and,
 * after all blocks, divides by n(n-1) via ebc_oracle_brandes_finish). */
void ebc_oracle_brandes_block(const ebc_oracle *o, uint64_t src_begin, uint64_t src_end,
                              double *scores_out) {
    const uint64_t n = o->n;
    uint32_t *dist = (uint32_t *)malloc((n ? n : 1) * 4);
    uint32_t *order = (uint32_t *)malloc((n ? n : 1) * 4);
    double *sigma = (double *)malloc((n ? n : 1) * 8);
    double *dep = (double *)malloc((n ? n : 1) * 8);
    for (uint64_t s = src_begin; s < src_end; ++s) {
        for (uint64_t v = 0; v < n; ++v) {
            dist[v] = EBC_UNREACHED;
            sigma[v] = 0.0;
            dep[v] = 0.0;
        }
        uint64_t head = 0, tail = 0;
        order[tail++] = (uint32_t)s;
        dist[s] = 0;
        sigma[s] = 1.0;
        for (; head < tail; ++head) {
            uint32_t u = order[head];
            for (uint64_t i = o->offsets[u]; i < o->offsets[u + 1]; ++i) {
                uint32_t v = o->targets[i];
                if (dist[v] == EBC_UNREACHED) {
                    dist[v] = dist[u] + 1;
                    order[tail++] = v;
                }
                if (dist[v] == dist[u] + 1)
                    sigma[v] += sigma[u];
            }
        }
        for (uint64_t k = tail; k-- > 1;) {
            uint32_t w = order[k];
            for (uint64_t i = o->offsets[w]; i < o->offsets[w + 1]; ++i) {
                uint32_t v = o->targets[i];
                if (dist[v] + 1 == dist[w])
                    dep[v] += sigma[v] / sigma[w] * (1.0 + dep[w]);
            }
            scores_out[w] += dep[w];
        }
    }
    free(dist);
    free(order);
    free(sigma);
    free(dep);
}

void ebc_oracle_brandes_finish(uint64_t n, double *scores) {
    const double norm = (double)n * (double)(n - 1);
    for (uint64_t v = 0; v < n; ++v)
        scores[v] /= norm;
}
