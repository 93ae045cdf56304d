// Device side of the B200 KADABRA hot path: graph upload, slot allocation,
// kernel launches (sampling, frame fold + stopping check, BFS) and the small
// amount of host bookkeeping around them.  sm_100a only; no CPU fallback.
#include "cuda_sampler.hpp"

#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <chrono>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "device_types.cuh"
#include "sample_launch.hpp"

namespace ebc {

namespace {

void cuda_check(cudaError_t e, const char *what, const char *file, int line) {
    if (e != cudaSuccess) {
        char buf[512];
        std::snprintf(buf, sizeof(buf), "CUDA failure: %s: %s (%s:%d)", what, cudaGetErrorString(e), file, line);
        throw CudaError(buf);
    }
}
#define EBC_CUDA(expr) cuda_check((expr), #expr, __FILE__, __LINE__)

// Process-wide cache of device allocations.  A run allocates ~10 GB of slot state; cudaMalloc/cudaFree of
// that size costs far more than the sampling itself on small inputs, so buffers released by one sampler
// are kept (per device, keyed by size) and handed to the next one.  ebc_release_device_cache() frees them.
class DevicePool {
public:
    void *alloc(std::size_t bytes) {
        bytes = std::max<std::size_t>(bytes, 256);
        int dev = 0;
        EBC_CUDA(cudaGetDevice(&dev));
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto it = idle_.find({dev, bytes});
            if (it != idle_.end()) {
                void *p = it->second;
                idle_.erase(it);
                idle_bytes_ -= bytes;
                live_[p] = {dev, bytes};
                live_bytes_ += bytes;
                return p;
            }
        }
        void *p = nullptr;
        ++mallocs_;
        malloc_bytes_ += bytes;
        cudaError_t e = cudaMalloc(&p, bytes);
        if (e == cudaErrorMemoryAllocation) { // make room and retry once
            cudaGetLastError();
            release_idle();
            e = cudaMalloc(&p, bytes);
        }
        cuda_check(e, "cudaMalloc", __FILE__, __LINE__);
        std::lock_guard<std::mutex> lk(mu_);
        live_[p] = {dev, bytes};
        live_bytes_ += bytes;
        return p;
    }
    void free(void *p) {
        if (!p)
            return;
        std::lock_guard<std::mutex> lk(mu_);
        auto it = live_.find(p);
        if (it == live_.end()) {
            cudaFree(p);
            return;
        }
        const auto key = it->second;
        live_.erase(it);
        live_bytes_ -= key.second;
        if (idle_bytes_ + key.second > kMaxIdleBytes) {
            ++frees_;
            cudaFree(p);
            return;
        }
        idle_.emplace(key, p);
        idle_bytes_ += key.second;
    }
    void stats(const char *where) {
        std::lock_guard<std::mutex> lk(mu_);
        std::fprintf(stderr, "[ebc] pool %s: %zu cudaMalloc (%.1f MB), %zu cudaFree, idle %.1f MB in %zu buffers, live %zu\n", where,
                     mallocs_, malloc_bytes_ / 1e6, frees_, idle_bytes_ / 1e6, idle_.size(), live_.size());
    }
    std::size_t live_bytes() {
        std::lock_guard<std::mutex> lk(mu_);
        return live_bytes_;
    }
    // Device memory this process can use = free + everything the pool holds.  cudaMemGetInfo was measured
    // at 8-90 ms per call with ~14 GB allocated -- a sixth of a whole run on a small input -- so the
    // figure is cached per device and refreshed every few seconds (an allocation that fails because
    // somebody else took the memory still frees the idle buffers and retries, see alloc()).
    std::size_t capacity() {
        int dev = 0;
        EBC_CUDA(cudaGetDevice(&dev));
        const auto now = std::chrono::steady_clock::now();
        std::lock_guard<std::mutex> lk(mu_);
        auto it = capacity_.find(dev);
        if (it != capacity_.end() && now - it->second.first < std::chrono::seconds(5))
            return it->second.second;
        size_t free_b = 0, total_b = 0;
        EBC_CUDA(cudaMemGetInfo(&free_b, &total_b));
        const std::size_t cap = free_b + idle_bytes_ + live_bytes_;
        capacity_[dev] = {now, cap};
        return cap;
    }
    void release_idle() {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto &kv : idle_)
            cudaFree(kv.second);
        idle_.clear();
        idle_bytes_ = 0;
    }

private:
    static constexpr std::size_t kMaxIdleBytes = std::size_t{96} << 30;
    std::mutex mu_;
    std::map<void *, std::pair<int, std::size_t>> live_;
    std::multimap<std::pair<int, std::size_t>, void *> idle_;
    std::size_t idle_bytes_ = 0, live_bytes_ = 0;
    std::map<int, std::pair<std::chrono::steady_clock::time_point, std::size_t>> capacity_;
    std::size_t mallocs_ = 0, malloc_bytes_ = 0, frees_ = 0;
};

DevicePool &pool() {
    static DevicePool *p = new DevicePool; // intentionally leaked: must outlive every sampler at exit
    return *p;
}

// Streams, events and the pinned result words are cached the same way: creating and, above all,
// destroying them (cudaFreeHost, cudaStreamDestroy) sporadically blocks for 10^2 ms in the driver, which
// is longer than a whole run on a small input.
class HandleCache {
public:
    cudaStream_t take_stream() {
        int dev = device();
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto &v = streams_[dev];
            if (!v.empty()) {
                cudaStream_t s = v.back();
                v.pop_back();
                return s;
            }
        }
        cudaStream_t s = nullptr;
        EBC_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        return s;
    }
    void give_stream(cudaStream_t s) {
        if (!s)
            return;
        std::lock_guard<std::mutex> lk(mu_);
        streams_[device()].push_back(s);
    }
    cudaEvent_t take_event(bool timing) {
        int dev = device();
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto &v = events_[{dev, timing}];
            if (!v.empty()) {
                cudaEvent_t e = v.back();
                v.pop_back();
                return e;
            }
        }
        cudaEvent_t e = nullptr;
        EBC_CUDA(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming));
        return e;
    }
    void give_event(cudaEvent_t e, bool timing) {
        if (!e)
            return;
        std::lock_guard<std::mutex> lk(mu_);
        events_[{device(), timing}].push_back(e);
    }
    // two u64 of pinned, mapped host memory
    u64 *take_words() {
        int dev = device();
        {
            std::lock_guard<std::mutex> lk(mu_);
            auto &v = words_[dev];
            if (!v.empty()) {
                u64 *w = v.back();
                v.pop_back();
                return w;
            }
        }
        u64 *w = nullptr;
        EBC_CUDA(cudaHostAlloc(reinterpret_cast<void **>(&w), 2 * sizeof(u64), cudaHostAllocMapped));
        return w;
    }
    void give_words(u64 *w) {
        if (!w)
            return;
        std::lock_guard<std::mutex> lk(mu_);
        words_[device()].push_back(w);
    }
    void release_idle() {
        std::lock_guard<std::mutex> lk(mu_);
        for (auto &kv : streams_)
            for (cudaStream_t s : kv.second)
                cudaStreamDestroy(s);
        for (auto &kv : events_)
            for (cudaEvent_t e : kv.second)
                cudaEventDestroy(e);
        for (auto &kv : words_)
            for (u64 *w : kv.second)
                cudaFreeHost(w);
        streams_.clear();
        events_.clear();
        words_.clear();
    }

private:
    static int device() {
        int dev = 0;
        cudaGetDevice(&dev);
        return dev;
    }
    std::mutex mu_;
    std::map<int, std::vector<cudaStream_t>> streams_;
    std::map<std::pair<int, bool>, std::vector<cudaEvent_t>> events_;
    std::map<int, std::vector<u64 *>> words_;
};

HandleCache &handles() {
    static HandleCache *h = new HandleCache; // leaked on purpose, like the pool
    return *h;
}

template <typename T> T *dev_alloc(std::uint64_t count) {
    return static_cast<T *>(pool().alloc(std::max<std::uint64_t>(count, 1) * sizeof(T)));
}
void dev_free(void *p) { pool().free(p); }

// ------------------------------------------------------------------------------------
// Frame fold + stopping check.
//   fold:   S[i] += frame[i]; frame[i] = 0 for i in 1..n        (StateFrame::add,
//           state_frame.hpp:29-33; collect_epoch's sum-then-zero, epoch.cpp:66-81)
//   check:  any vertex whose f or g width >= eps clears the "all below" flag
//           (check_stop, stopping.cpp:125-142; bound_width, stopping.cpp:96-111)
// tau (word 0) is read by every thread before anyone writes it: word 0 is folded
// by finish_fold_kernel afterwards.  FP64 uses explicit round-to-nearest
// intrinsics in the reference's operation order so no FMA contraction can
// change a comparison.
struct StopParams {
    double eps;
    u64 omega;
    const double *log_lower; // ln(1/delta_L) or ln(2/delta_L)
    const double *log_upper;
    int bound; // 0 Hoeffding, 1 empirical Bernstein
    int have;
};

__device__ __forceinline__ double bound_width_dev(double b, double logterm, double t, int bound) {
    if (bound == 0) // sqrt(log(1/delta_v) / (2 t))
        return __dsqrt_rn(__ddiv_rn(logterm, __dmul_rn(2.0, t)));
    // sqrt(2 var l / t) + 7 l / (3 (t - 1))
    const double var = __dmul_rn(b, __dsub_rn(1.0, b));
    const double first = __dsqrt_rn(__ddiv_rn(__dmul_rn(__dmul_rn(2.0, var), logterm), t));
    const double second = __ddiv_rn(__dmul_rn(7.0, logterm), __dmul_rn(3.0, __dsub_rn(t, 1.0)));
    return __dadd_rn(first, second);
}

__global__ void __launch_bounds__(256) fold_check_kernel(u32 *frame, u64 *S, u64 n, StopParams sp, u32 *fail_flag) {
    const u64 tau = S[0] + frame[0];
    const bool evaluate = sp.have && tau < sp.omega && tau >= 2;
    const double t = static_cast<double>(tau);
    bool fail = false;
    for (u64 i = 1 + blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i <= n;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 f = frame[i];
        u64 c = S[i];
        if (f != 0) {
            c += f;
            S[i] = c;
            frame[i] = 0;
        }
        if (evaluate) {
            const double b = __ddiv_rn(static_cast<double>(c), t);
            if (bound_width_dev(b, sp.log_lower[i - 1], t, sp.bound) >= sp.eps)
                fail = true;
            if (bound_width_dev(b, sp.log_upper[i - 1], t, sp.bound) >= sp.eps)
                fail = true;
        }
    }
    if (__syncthreads_or(fail ? 1 : 0) && threadIdx.x == 0)
        atomicOr(fail_flag, 1u);
}

// Folds word 0 (tau) and publishes the stop decision: result[0] = stop (0|1), result[1] = tau.
__global__ void finish_fold_kernel(u32 *frame, u64 *S, StopParams sp, u32 *fail_flag, volatile u64 *result) {
    const u64 tau = S[0] + frame[0];
    S[0] = tau;
    frame[0] = 0;
    u64 stop;
    if (!sp.have)
        stop = 0;
    else if (tau >= sp.omega)
        stop = 1; // stopping.cpp:127
    else if (tau < 2)
        stop = 0; // stopping.cpp:129
    else
        stop = *fail_flag ? 0 : 1;
    *fail_flag = 0;
    result[1] = tau;
    __threadfence_system();
    result[0] = stop;
}

__global__ void widen_kernel(const u32 *in, u64 *out, u64 words) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < words;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        out[i] = in[i];
}

// ------------------------------------------------------------------------------------
// Level-synchronous BFS for the diameter phase (bfs.cpp:9-34).  One warp per
// frontier vertex, lanes stride the row; the level loop runs on the device
// stream without host round trips (each launch reads the queue size written by
// the previous one and exits when it is empty).
constexpr u32 kBfsBigRow = 8192;  // adjacency entries
constexpr u32 kBfsBigCap = 2048;  // set-aside rows per level (further ones are expanded in place)

struct BfsState {
    u32 queue_size[2];
    u32 depth;
    u32 done;
    u64 reached;
    // direction optimisation (Beamer et al.): a level whose frontier carries more than 1/16 of the arcs is
    // expanded bottom-up (every unvisited vertex looks for one parent in the frontier and stops at the first)
    u64 frontier_arcs[2]; // sum of the degrees of the frontier being built, by level parity
    u32 bottom_up;        // mode of the level about to run
    u32 have_queue;       // the frontier of the level about to run exists as a queue
    u32 bu_found;         // vertices settled by the bottom-up pass of this level
    // top-down levels: frontier vertices whose row is too long for one warp are set aside and expanded
    // by the whole grid (bfs_big_rows_kernel) -- a sweep that starts at a hub is otherwise one warp's work
    u32 big_count;
    u32 big[kBfsBigCap];
};

__global__ void __launch_bounds__(256) bfs_level_kernel(const u64 *offsets, const u32 *targets, u32 *dist,
                                                        u32 *queue0, u32 *queue1, BfsState *st, u32 level) {
    if (st->done || st->bottom_up)
        return;
    const u32 *in = (level & 1) ? queue1 : queue0;
    u32 *out = (level & 1) ? queue0 : queue1;
    const u32 count = st->queue_size[level & 1];
    const u32 warps = (gridDim.x * blockDim.x) >> 5;
    const u32 warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const u32 lane = threadIdx.x & 31;
    u64 arcs = 0;
    for (u32 i = warp; i < count; i += warps) {
        const u32 u = in[i];
        const u64 beg = offsets[u], end = offsets[u + 1];
        if (end - beg > kBfsBigRow) {
            u32 slot = 0;
            if (lane == 0)
                slot = atomicAdd(&st->big_count, 1u);
            slot = __shfl_sync(0xffffffffu, slot, 0);
            if (slot < kBfsBigCap) {
                if (lane == 0)
                    st->big[slot] = u;
                continue;
            }
        }
        for (u64 k = beg + lane; k < end; k += 32) {
            const u32 v = targets[k];
            if (dist[v] == 0xffffffffu && atomicCAS(dist + v, 0xffffffffu, level + 1) == 0xffffffffu) {
                const u32 pos = atomicAdd(&st->queue_size[(level + 1) & 1], 1u);
                out[pos] = v;
                arcs += offsets[v + 1] - offsets[v];
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        arcs += __shfl_xor_sync(0xffffffffu, arcs, o);
    if (lane == 0 && arcs)
        atomicAdd(reinterpret_cast<unsigned long long *>(&st->frontier_arcs[(level + 1) & 1]), static_cast<unsigned long long>(arcs));
}

// Second half of a top-down level: the rows set aside by bfs_level_kernel, each spread over the whole grid.
__global__ void __launch_bounds__(256) bfs_big_rows_kernel(const u64 *offsets, const u32 *targets, u32 *dist,
                                                           u32 *queue0, u32 *queue1, BfsState *st, u32 level) {
    if (st->done || st->bottom_up)
        return;
    const u32 rows = st->big_count < kBfsBigCap ? st->big_count : kBfsBigCap;
    if (rows == 0)
        return;
    u32 *out = (level & 1) ? queue0 : queue1;
    const u64 threads = static_cast<u64>(gridDim.x) * blockDim.x;
    const u64 me = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x;
    u64 arcs = 0;
    for (u32 r = 0; r < rows; ++r) {
        const u32 u = st->big[r];
        const u64 beg = offsets[u], end = offsets[u + 1];
        for (u64 k = beg + me; k < end; k += threads) {
            const u32 v = targets[k];
            if (dist[v] == 0xffffffffu && atomicCAS(dist + v, 0xffffffffu, level + 1) == 0xffffffffu) {
                const u32 pos = atomicAdd(&st->queue_size[(level + 1) & 1], 1u);
                out[pos] = v;
                arcs += offsets[v + 1] - offsets[v];
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1)
        arcs += __shfl_xor_sync(0xffffffffu, arcs, o);
    if ((threadIdx.x & 31) == 0 && arcs)
        atomicAdd(reinterpret_cast<unsigned long long *>(&st->frontier_arcs[(level + 1) & 1]), static_cast<unsigned long long>(arcs));
}

// Bottom-up level: one thread per vertex; an unvisited vertex scans its row until it meets the frontier.
__global__ void __launch_bounds__(256) bfs_bottom_up_kernel(const u64 *offsets, const u32 *targets, u32 *dist, u64 n,
                                                            BfsState *st, u32 level) {
    if (st->done || !st->bottom_up)
        return;
    u32 found = 0;
    u64 arcs = 0;
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        if (dist[v] != 0xffffffffu)
            continue;
        const u64 beg = offsets[v], end = offsets[v + 1];
        for (u64 k = beg; k < end; ++k)
            if (dist[targets[k]] == level) {
                dist[v] = level + 1; // only this thread writes dist[v]; readers compare with `level`
                ++found;
                arcs += end - beg;
                break;
            }
    }
    for (int o = 16; o > 0; o >>= 1) {
        found += __shfl_xor_sync(0xffffffffu, found, o);
        arcs += __shfl_xor_sync(0xffffffffu, arcs, o);
    }
    if ((threadIdx.x & 31) == 0 && found) {
        atomicAdd(&st->bu_found, found);
        atomicAdd(reinterpret_cast<unsigned long long *>(&st->frontier_arcs[(level + 1) & 1]), static_cast<unsigned long long>(arcs));
    }
}

// After a bottom-up level the next frontier exists only as dist == level + 1; a top-down level needs it
// as a queue.
__global__ void __launch_bounds__(256) bfs_rebuild_queue_kernel(const u32 *dist, u64 n, u32 *queue0, u32 *queue1,
                                                                BfsState *st, u32 level) {
    if (st->done || st->bottom_up || st->have_queue)
        return;
    u32 *out = (level & 1) ? queue1 : queue0;
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x)
        if (dist[v] == level)
            out[atomicAdd(&st->queue_size[level & 1], 1u)] = static_cast<u32>(v);
}

// Runs as one thread between levels: closes level `level`, opens level + 1 and picks its direction.
__global__ void bfs_advance_kernel(BfsState *st, u32 level, u64 arcs_total, u32 allow_bottom_up) {
    if (st->done)
        return;
    const u32 next = st->bottom_up ? st->bu_found : st->queue_size[(level + 1) & 1];
    const bool next_is_queue = !st->bottom_up;
    st->queue_size[level & 1] = 0;
    st->bu_found = 0;
    st->big_count = 0;
    st->frontier_arcs[level & 1] = 0;
    if (next == 0) {
        st->done = 1;
        st->depth = level;
        return;
    }
    st->reached += next;
    const u64 next_arcs = st->frontier_arcs[(level + 1) & 1];
    st->bottom_up = allow_bottom_up && next_arcs > arcs_total / 16 ? 1u : 0u;
    st->have_queue = next_is_queue ? 1u : 0u;
    if (!next_is_queue)
        st->queue_size[(level + 1) & 1] = 0; // rebuilt on demand by bfs_rebuild_queue_kernel
}

// farthest = max distance, lowest id on ties (bfs.cpp:21-24): key = dist << 32 | ~v.
__global__ void __launch_bounds__(256) bfs_farthest_kernel(const u32 *dist, u64 n, unsigned long long *best) {
    unsigned long long local = 0;
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 d = dist[v];
        if (d != 0xffffffffu) {
            const unsigned long long key = (static_cast<unsigned long long>(d) << 32) | (0xffffffffu - static_cast<u32>(v));
            local = key > local ? key : local;
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, local, o);
        local = other > local ? other : local;
    }
    if ((threadIdx.x & 31) == 0)
        atomicMax(best, local);
}

// ---- dense (hub-clustered) numbering, see SamplerParams::to_dense ----
__global__ void __launch_bounds__(256) degree_kernel(const u64 *offsets, u64 n, u32 *deg, u32 *ids) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        // Sort key = bit length of the degree.  Coarse on purpose: the sort is stable, so vertices of one
        // class keep their external order and a row (ascending external ids) still walks every class in
        // ascending dense order -- hub entries land in a small, ascending id range.
        // (finer classes were measured 0..3 % slower on R-MAT-20: profiles/r01_numbering.txt)
        deg[v] = 64u - static_cast<u32>(__clzll(offsets[v + 1] - offsets[v]));
        ids[v] = static_cast<u32>(v);
    }
}

// ---- neighbourhood-clustered numbering for graphs without hubs ----
// On a hub-free graph (grid, road network) a search settles a connected ball, and every label / offsets /
// row access of a level goes to the ball's surface.  If vertices that are close in the graph are close in the
// numbering, those accesses share 128-byte lines and the surface of a ball is a few lines instead of one per
// vertex.  Clusters: every vertex whose hashed id falls into a 1/kClusterSize slice is a centre; centres grow
// breadth-first in lock step and a vertex joins the smallest centre id among its assigned neighbours (a
// graph Voronoi partition, deterministic because each round reads the previous round's array).  Vertices are
// then sorted by (centre id, own id).
constexpr u32 kClusterSize = 32; // vertices per 128-byte line of labels
constexpr u32 kNoCluster = 0xffffffffu;
__global__ void __launch_bounds__(256) cluster_seed_kernel(u64 n, u32 *center, u32 *ids) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 h = (static_cast<u32>(v) * 2654435761u) >> 12;
        center[v] = h % kClusterSize == 0 ? static_cast<u32>(v) : kNoCluster;
        ids[v] = static_cast<u32>(v);
    }
}
__global__ void __launch_bounds__(256) cluster_grow_kernel(const u64 *offsets, const u32 *targets, u64 n, const u32 *in,
                                                           u32 *out, u32 *unassigned) {
    u32 open = 0;
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        u32 c = in[v];
        if (c == kNoCluster) {
            for (u64 k = offsets[v]; k < offsets[v + 1]; ++k) {
                const u32 cw = in[targets[k]];
                c = cw < c ? cw : c;
            }
            open += c == kNoCluster ? 1u : 0u;
        }
        out[v] = c;
    }
    if (__syncthreads_or(open != 0 ? 1 : 0) && threadIdx.x == 0)
        atomicOr(unassigned, 1u);
}
// vertices no centre reached within the round limit are their own cluster
__global__ void __launch_bounds__(256) cluster_finish_kernel(u64 n, u32 *center) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x)
        if (center[v] == kNoCluster)
            center[v] = static_cast<u32>(v);
}

// to_dense = inverse of to_ext; dense_offsets[i] = degree of dense vertex i (scanned afterwards)
__global__ void __launch_bounds__(256) invert_kernel(const u32 *to_ext, const u64 *ext_offsets, u64 n, u32 *to_dense,
                                                     u64 *dense_offsets) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i <= n;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        if (i < n) {
            const u32 v = to_ext[i];
            to_dense[v] = static_cast<u32>(i);
            dense_offsets[i] = ext_offsets[v + 1] - ext_offsets[v];
        } else {
            dense_offsets[i] = 0;
        }
    }
}

// Dense rows: row i holds the entries of the external row to_ext[i] in their original order, renamed.
// One CTA per chunk of kDenseChunk arcs; the rows a chunk touches are bracketed once per CTA.
constexpr u64 kDenseChunk = 2048;
__global__ void __launch_bounds__(256) dense_rows_kernel(const u64 *ext_offsets, const u32 *ext_targets, const u64 *offsets,
                                                         const u32 *to_ext, const u32 *to_dense, u32 *targets, u64 n,
                                                         u64 arcs) {
    __shared__ u64 bracket[2];
    const u64 chunks = (arcs + kDenseChunk - 1) / kDenseChunk;
    for (u64 c = blockIdx.x; c < chunks; c += gridDim.x) {
        const u64 c0 = c * kDenseChunk, c1 = c0 + kDenseChunk < arcs ? c0 + kDenseChunk : arcs;
        __syncthreads();
        if (threadIdx.x < 2) { // last row r with offsets[r] <= j for j = c0 and j = c1 - 1
            const u64 j = threadIdx.x == 0 ? c0 : c1 - 1;
            u64 lo = 0, hi = n;
            while (hi - lo > 1) {
                const u64 mid = (lo + hi) >> 1;
                if (offsets[mid] <= j)
                    lo = mid;
                else
                    hi = mid;
            }
            bracket[threadIdx.x] = lo;
        }
        __syncthreads();
        for (u64 j = c0 + threadIdx.x; j < c1; j += blockDim.x) {
            u64 lo = bracket[0], hi = bracket[1] + 1;
            while (hi - lo > 1) {
                const u64 mid = (lo + hi) >> 1;
                if (__ldg(offsets + mid) <= j)
                    lo = mid;
                else
                    hi = mid;
            }
            const u64 src = __ldg(ext_offsets + __ldg(to_ext + lo)) + (j - __ldg(offsets + lo));
            targets[j] = __ldg(to_dense + __ldg(ext_targets + src));
        }
    }
}

// Fixed-stride rows (SamplerParams::ell): row v = its entries in row order, each with the position of the reverse arc
// and the target's degree - 1 in the upper bits, padded with kEllEmpty.  *bad is raised if that does not work out (a
// row above kEllWidth entries, or an arc without its reverse -- an asymmetric input); the sampler then runs without them.
// `width` = entries stored per row: kEllWidth, or kEllNarrow when the caller knows that no row is longer.
__global__ void __launch_bounds__(256) ell_rows_kernel(const u64 *offsets, const u32 *targets, u64 n, u32 width, u32 *ell, u32 *ell4,
                                                       u32 *bad) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 beg = offsets[v], deg = offsets[v + 1] - beg;
        u32 row[kEllWidth];
#pragma unroll
        for (u32 k = 0; k < kEllWidth; ++k) {
            row[k] = kEllEmpty;
            if (k < deg) {
                const u32 w = targets[beg + k];
                const u64 wb = offsets[w], dw = offsets[w + 1] - wb;
                u32 rev = kEllWidth; // position of v in the row of w
                for (u32 j = 0; j < kEllWidth && j < dw; ++j)
                    if (targets[wb + j] == v)
                        rev = j;
                if (dw < 1 || dw > width || rev == kEllWidth)
                    *bad = 1;
                row[k] = w | ((rev & (kEllWidth - 1)) << kEllRevShift) | (static_cast<u32>(dw - 1) << kEllDegShift);
            }
        }
        if (deg > width)
            *bad = 1;
        uint4 *out = reinterpret_cast<uint4 *>(ell) + (width / 4) * v;
        out[0] = make_uint4(row[0], row[1], row[2], row[3]);
        if (width == kEllWidth)
            out[1] = make_uint4(row[4], row[5], row[6], row[7]);
        if (ell4) // the 16-byte copy: rows of more than four entries refer to `ell`
            reinterpret_cast<uint4 *>(ell4)[v] = make_uint4(deg > kEllNarrow ? kEllEscape : row[0], row[1], row[2], row[3]);
    }
}

__global__ void __launch_bounds__(256) fill_two_kernel(double *a, double *b, u64 count, double value) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        a[i] = value;
        b[i] = value;
    }
}

__global__ void flush_kernel(u32 *buf, u64 count, u32 salt) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        buf[i] = static_cast<u32>(i) ^ salt;
}

// The (BLOCK, ITEMS) instantiations of the sampling kernel are compiled in their own translation units, one per
// block size (sample_launch.cu, built five times with -DEBC_SHAPE_BLOCK=...), so that they compile in parallel.
void launch_sample_dispatch(u32 block, u32 items, const SamplerParams &p, u32 grid, cudaStream_t stream) {
    bool done = false;
    switch (block) {
    case 32: done = launch_sample_b32(items, p, grid, stream); break;
    case 64: done = launch_sample_b64(items, p, grid, stream); break;
    case 128: done = launch_sample_b128(items, p, grid, stream); break;
    case 256: done = launch_sample_b256(items, p, grid, stream); break;
    case 512: done = launch_sample_b512(items, p, grid, stream); break;
    default: break;
    }
    if (!done)
        throw ConfigError("block_threads must be one of 32, 64, 128, 256, 512 and items_per_thread one of 1, 2, 4");
    EBC_CUDA(cudaGetLastError());
}

int occupancy_for(u32 block, u32 items, bool fixed_rows) {
    int per_sm = -1;
    switch (block) {
    case 32: per_sm = sample_occupancy_b32(items, fixed_rows); break;
    case 64: per_sm = sample_occupancy_b64(items, fixed_rows); break;
    case 128: per_sm = sample_occupancy_b128(items, fixed_rows); break;
    case 256: per_sm = sample_occupancy_b256(items, fixed_rows); break;
    case 512: per_sm = sample_occupancy_b512(items, fixed_rows); break;
    default: break;
    }
    if (per_sm == -1)
        throw ConfigError("block_threads must be one of 32, 64, 128, 256, 512 and items_per_thread one of 1, 2, 4");
    if (per_sm < -1)
        throw CudaError("cudaOccupancyMaxActiveBlocksPerMultiprocessor failed for the sampling kernel");
    return per_sm;
}

// 8-byte bitmap words per slot (one word = 32 vertices x 2 sides), padded to whole 32-byte sectors: the
// kernel clears a settled vertex's bits by zeroing its sector with one 32-byte store.
static u64 bit_words_of(u64 n) { return ((n + 31) / 32 + 3) & ~u64{3}; }

struct SlotArrays {
    u32 *lab = nullptr, *list = nullptr, *lvl = nullptr, *contact = nullptr, *hdr = nullptr, *bits = nullptr, *pm = nullptr;
    u64 *sig = nullptr;
    u64 slots = 0, cap = 0, aux_cap = 0;
    u64 bytes = 0;

    static u64 pm_words_of(u64 cap) { return (cap + 3) / 4 + 1; }

    void allocate(u64 slots_, u64 cap_, u64 n, bool fixed_rows, cudaStream_t stream) {
        slots = slots_;
        cap = cap_;
        aux_cap = aux_cap_of(cap_, n);
        if (fixed_rows)
            pm = dev_alloc<u32>(slots * 2 * pm_words_of(cap));
        lab = dev_alloc<u32>(slots * n);
        list = dev_alloc<u32>(slots * 2 * cap);
        sig = dev_alloc<u64>(slots * 2 * cap);
        lvl = dev_alloc<u32>(slots * 2 * (aux_cap + 2));
        contact = dev_alloc<u32>(slots * 6 * aux_cap);
        bits = dev_alloc<u32>(slots * 2 * bit_words_of(n));
        EBC_CUDA(cudaMemsetAsync(bits, 0, slots * 2 * bit_words_of(n) * 4, stream));
        hdr = dev_alloc<u32>(slots * kHdrWords);
        bytes = slots * bytes_per_slot(n, cap, fixed_rows);
        EBC_CUDA(cudaMemsetAsync(lab, 0, slots * n * 4, stream));
        std::vector<u32> h(slots * kHdrWords, 0);
        for (u64 s = 0; s < slots; ++s)
            h[s * kHdrWords + kHdrBase0] = h[s * kHdrWords + kHdrBase1] = 1; // label 0 == never visited
        if (const char *env = std::getenv("EBC_TEST_LABEL_BASE")) { // test hook: start close to the label-space reset
            const u32 base = static_cast<u32>(std::strtoul(env, nullptr, 0));
            for (u64 s = 0; s < slots; ++s) {
                h[s * kHdrWords + kHdrBase0] = base;
                h[s * kHdrWords + kHdrBase1] = base;
            }
        }
        EBC_CUDA(cudaMemcpyAsync(hdr, h.data(), h.size() * 4, cudaMemcpyHostToDevice, stream));
        EBC_CUDA(cudaStreamSynchronize(stream));
    }
    void release() {
        dev_free(lab);
        dev_free(pm);
        dev_free(list);
        dev_free(sig);
        dev_free(lvl);
        dev_free(contact);
        dev_free(bits);
        dev_free(hdr);
    }
    // Level table and contact list are far smaller than the settle lists in practice: 2^16 entries unless
    // the slot is a full-capacity one (cap == n), which must never overflow.
    static u64 aux_cap_of(u64 cap, u64 n) { return cap >= n ? n : std::min<u64>(cap, u64{1} << 16); }
    static u64 bytes_per_slot(u64 n, u64 cap, bool fixed_rows) {
        const u64 aux = aux_cap_of(cap, n);
        return (fixed_rows ? 2 * pm_words_of(cap) * 4 : 0) + n * 4 + 2 * bit_words_of(n) * 4 + 2 * cap * (4 + 8) + 2 * (aux + 2) * 4 + 6 * aux * 4 + kHdrWords * 4;
    }
};

constexpr u32 kOverflowCap = 1u << 20; // also the largest number of samples per launch
constexpr int kEvents = 8;
constexpr u64 kLargeSlots = 8; // full-capacity slots of the re-run pass

} // namespace

void set_device_or_throw(int device) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw CudaError(std::string("no CUDA device available (this library has no CPU fallback): ") +
                        (e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e)));
    if (device >= count)
        throw ConfigError("device ordinal out of range");
    if (device >= 0)
        EBC_CUDA(cudaSetDevice(device));
}

void release_device_cache() {
    pool().release_idle();
    handles().release_idle();
    pinned_release_idle();
}

struct CudaSampler::Impl {
    ~Impl();
    int device = 0;
    int sm_count = 0;
    u64 n = 0, arcs = 0;
    u64 *d_offsets = nullptr; // the graph as uploaded (external ids): BFS, row searches of the walk
    u32 *d_targets = nullptr;
    u64 *d_dense_offsets = nullptr; // hub-clustered copy the sampling kernel searches on (null: not renumbered)
    u32 *d_dense_targets = nullptr;
    u32 *d_to_dense = nullptr, *d_to_ext = nullptr;
    u32 *d_ell = nullptr; // fixed-stride rows of the graph the kernel searches on (null: maximum degree above kEllWidth)
    u32 ell_width = kEllWidth; // entries per row: kEllNarrow when the maximum degree allows
    u32 *d_ell4 = nullptr;     // 16-byte copy of 32-byte rows for the expansion (SamplerParams::ell4)
    bool want_ell4 = false;
    std::vector<u32> h_to_ext; // fetched on demand (last_state)
    u32 block = 128;
    u32 items = 4;
    u32 flags = 0;
    u64 probe_min_slots = 512;
    u64 probe_growth_x4 = 8; // the frontier's pending edges at least doubled
    bool hub_graph = false; // max degree >= 1024: visited bitmaps, direction-optimising BFS
    u32 reserved_sms = 0;   // SMs the main pass leaves empty (SamplerOptions::reserved_sms)
    int per_sm = 0;         // resident CTAs per SM of the sampling kernel
    u32 *d_started = nullptr; // [lane] see SamplerParams::started
    int numbering = 0;      // 0 none, 1 degree classes, 2 neighbourhood clusters
    SlotArrays small, big;
    u32 *d_frame[2] = {nullptr, nullptr};
    u64 *d_S = nullptr;
    u64 *d_wide = nullptr; // scratch for read_frame
    unsigned long long *d_ticket = nullptr; // [lane][2]: main pass, re-run pass
    u32 *d_ring = nullptr;                  // free slots (see acquire_slot in sampler_kernels.cuh)
    unsigned long long *d_ring_pos = nullptr; // {head, tail}
    unsigned long long *d_work = nullptr;
    u32 *d_overflow_list = nullptr, *d_overflow_count = nullptr; // per lane: list[kOverflowCap], count{main, re-run}
    u32 *d_fail = nullptr;
    double *d_log_lower = nullptr, *d_log_upper = nullptr;
    StopParams stop{};
    u64 *h_result[2] = {nullptr, nullptr}; // pinned, mapped: {stop, tau} per frame
    unsigned long long *d_ovf_total = nullptr; // [2]: abandoned samples in the main / re-run pass
    // Two sampling lanes (one per epoch frame): consecutive epochs run on different streams, so the CTAs
    // of epoch e+1 start on SMs that epoch e's tail has already left; slots are handed out dynamically.
    cudaStream_t s_sample = nullptr, s_sample2 = nullptr, s_agg = nullptr;
    cudaEvent_t ev_rerun[2]{}, ev_lane{};
    cudaEvent_t ev_sampled[2]{}, ev_folded[2]{}, ev_user[kEvents]{};
    bool folded_pending[2] = {false, false};
    u64 overflow_seen = 0;
    u64 launches = 0;
    // bfs
    u32 *d_dist = nullptr, *d_queue[2] = {nullptr, nullptr};
    BfsState *d_bfs = nullptr;
    unsigned long long *d_best = nullptr;
    // flush
    u32 *d_flush = nullptr;
    u64 flush_words = 0;
    u64 graph_bytes = 0;

    SamplerParams base_params(const SlotArrays &a) const {
        SamplerParams p{};
        p.n = n;
        p.offsets = d_dense_offsets ? d_dense_offsets : d_offsets;
        p.targets = d_dense_targets ? d_dense_targets : d_targets;
        p.to_dense = d_to_dense;
        p.to_ext = d_to_ext;
        p.ext_offsets = d_offsets;
        p.ext_targets = d_targets;
        p.ell = d_ell;
        p.ell_width = ell_width;
        p.ell4 = d_ell4;
        p.lab = a.lab;
        p.list = a.list;
        p.sig = a.sig;
        p.lvl = a.lvl;
        p.contact = a.contact;
        p.hdr = a.hdr;
        p.bits = a.bits;
        p.pm = a.pm;
        p.pm_words = SlotArrays::pm_words_of(a.cap);
        p.bit_words = bit_words_of(n);
        p.probe_min_slots = probe_min_slots;
        p.probe_growth_x4 = probe_growth_x4;
        p.cap = a.cap;
        p.aux_cap = a.aux_cap;
        p.work = d_work;
        p.overflow_cap = kOverflowCap;
        p.flags = flags;
        return p;
    }

    cudaStream_t lane_stream(int lane) const { return lane == 0 ? s_sample : s_sample2; }

    // Builds to_ext, its inverse and the dense CSR on the device from the uploaded graph.  to_ext lists the
    // vertices by descending degree class (hub graphs) or by neighbourhood cluster (`clusters`), ties by
    // ascending id.
    void build_dense_graph(bool clusters) {
        cudaStream_t st = s_sample;
        u32 *deg = dev_alloc<u32>(n), *ids = dev_alloc<u32>(n), *deg_sorted = dev_alloc<u32>(n);
        d_to_ext = dev_alloc<u32>(n);
        d_to_dense = dev_alloc<u32>(n);
        d_dense_offsets = dev_alloc<u64>(n + 1);
        d_dense_targets = dev_alloc<u32>(arcs + 4); // (+4: the probe reads whole 16-byte groups)
        const u32 grid = static_cast<u32>(std::min<u64>((n + 255) / 256, static_cast<u64>(sm_count) * 8));
        size_t sort_bytes = 0, sort2_bytes = 0, scan_bytes = 0;
        EBC_CUDA(cub::DeviceRadixSort::SortPairsDescending(nullptr, sort_bytes, deg, deg_sorted, ids, d_to_ext,
                                                           static_cast<int>(n), 0, 7, st));
        EBC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, sort2_bytes, deg, deg_sorted, ids, d_to_ext,
                                                 static_cast<int>(n), 0, 32, st));
        EBC_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, d_dense_offsets, d_dense_offsets,
                                               static_cast<int>(n + 1), st));
        unsigned char *tmp = dev_alloc<unsigned char>(std::max(std::max(sort_bytes, sort2_bytes), scan_bytes) + 16);
        if (clusters) {
            // `deg` / `deg_sorted` double as the two centre arrays of the growth rounds
            u32 *cur = deg, *nxt = deg_sorted;
            cluster_seed_kernel<<<grid, 256, 0, st>>>(n, cur, ids);
            u32 *flag = reinterpret_cast<u32 *>(tmp);
            u32 open = 1;
            for (int round = 0; round < 64 && open; round += 4) {
                EBC_CUDA(cudaMemsetAsync(flag, 0, 4, st));
                for (int k = 0; k < 4; ++k) { // the flag reports the last of four rounds
                    if (k == 3)
                        EBC_CUDA(cudaMemsetAsync(flag, 0, 4, st));
                    cluster_grow_kernel<<<grid, 256, 0, st>>>(d_offsets, d_targets, n, cur, nxt, flag);
                    std::swap(cur, nxt);
                }
                EBC_CUDA(cudaGetLastError());
                EBC_CUDA(cudaMemcpyAsync(&open, flag, 4, cudaMemcpyDeviceToHost, st));
                EBC_CUDA(cudaStreamSynchronize(st));
            }
            cluster_finish_kernel<<<grid, 256, 0, st>>>(n, cur);
            EBC_CUDA(cub::DeviceRadixSort::SortPairs(tmp, sort2_bytes, cur, nxt, ids, d_to_ext, static_cast<int>(n), 0, 32,
                                                     st)); // stable: a cluster keeps its external order
        } else {
            degree_kernel<<<grid, 256, 0, st>>>(d_offsets, n, deg, ids);
            EBC_CUDA(cudaGetLastError());
            EBC_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, sort_bytes, deg, deg_sorted, ids, d_to_ext,
                                                               static_cast<int>(n), 0, 7, st)); // stable
        }
        invert_kernel<<<grid, 256, 0, st>>>(d_to_ext, d_offsets, n, d_to_dense, d_dense_offsets);
        EBC_CUDA(cudaGetLastError());
        EBC_CUDA(cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, d_dense_offsets, d_dense_offsets,
                                               static_cast<int>(n + 1), st));
        const u64 chunks = (arcs + kDenseChunk - 1) / kDenseChunk;
        const u32 grid2 = static_cast<u32>(std::min<u64>(chunks, static_cast<u64>(sm_count) * 16));
        dense_rows_kernel<<<grid2, 256, 0, st>>>(d_offsets, d_targets, d_dense_offsets, d_to_ext, d_to_dense,
                                                 d_dense_targets, n, arcs);
        EBC_CUDA(cudaGetLastError());
        EBC_CUDA(cudaStreamSynchronize(st));
        dev_free(deg);
        dev_free(ids);
        dev_free(deg_sorted);
        dev_free(tmp);
        graph_bytes += (n + 1) * 8 + arcs * 4 + n * 8;
    }

    // Fixed-stride rows of the graph the kernel searches on (the dense copy if there is one).
    void build_fixed_rows() {
        cudaStream_t st = s_sample;
        d_ell = dev_alloc<u32>(n * ell_width);
        if (want_ell4)
            d_ell4 = dev_alloc<u32>(n * kEllNarrow);
        u32 *bad = dev_alloc<u32>(1);
        EBC_CUDA(cudaMemsetAsync(bad, 0, 4, st));
        const u32 grid = static_cast<u32>(std::min<u64>((n + 255) / 256, static_cast<u64>(sm_count) * 8));
        ell_rows_kernel<<<grid, 256, 0, st>>>(d_dense_offsets ? d_dense_offsets : d_offsets,
                                              d_dense_targets ? d_dense_targets : d_targets, n, ell_width, d_ell, d_ell4, bad);
        EBC_CUDA(cudaGetLastError());
        u32 h_bad = 0;
        EBC_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, st));
        EBC_CUDA(cudaStreamSynchronize(st));
        dev_free(bad);
        if (h_bad) {
            dev_free(d_ell);
            dev_free(d_ell4);
            d_ell = d_ell4 = nullptr;
        } else {
            graph_bytes += n * ell_width * 4 + (d_ell4 ? n * kEllNarrow * 4 : 0);
        }
    }

    // Launches the main pass and the re-run pass for [first, first+count), count <= kOverflowCap, on the
    // sampling lane of `frame`.
    void launch(u64 seed, u32 tag, u64 first, u64 count, int frame, const u32 *d_pairs,
                SampleRecordDev *d_records, u32 *d_paths, u64 path_stride) {
        const int lane = frame;
        cudaStream_t st = lane_stream(lane);
        unsigned long long *ticket = d_ticket + 2 * lane;
        u32 *ovf_count = d_overflow_count + 2 * lane;
        u32 *ovf_list = d_overflow_list + static_cast<u64>(lane) * kOverflowCap;
        EBC_CUDA(cudaMemsetAsync(ticket, 0, 2 * sizeof(unsigned long long), st));
        EBC_CUDA(cudaMemsetAsync(ovf_count, 0, 2 * sizeof(u32), st));
        SamplerParams p = base_params(small);
        if (d_records || d_paths)
            p.flags |= kFlagStats; // (only the kernels with statistics fill records and paths)
        p.seed = seed;
        p.tag = tag;
        p.first = first;
        p.count = count;
        p.ticket = ticket;
        p.frame = d_frame[frame];
        p.pairs = d_pairs;
        p.records = d_records;
        p.paths = d_paths;
        p.path_stride = path_stride;
        p.overflow_list = ovf_list;
        p.overflow_count = ovf_count;
        p.overflow_total = d_ovf_total;
        p.ring = d_ring;
        p.ring_size = static_cast<u32>(small.slots);
        p.ring_pos = d_ring_pos;
        const u32 grid = static_cast<u32>(std::min<u64>(small.slots, count));
        const u32 held = reserved_sms * static_cast<u32>(per_sm); // CTAs the reserved SMs hold
        if (reserved_sms && grid > 2 * held) { // (a launch that small leaves room anyway)
            p.reserved_sms = reserved_sms;
            p.reserve_target = grid - held;
            p.started = d_started + lane;
            EBC_CUDA(cudaMemsetAsync(p.started, 0, sizeof(u32), st));
        }
        launch_sample_dispatch(block, items, p, grid, st);
        ++launches;
        if (small.cap < n) { // capacity overflow is impossible when cap == n
            // the large slots are bound to blockIdx: re-run passes of the two lanes must not overlap
            EBC_CUDA(cudaStreamWaitEvent(st, ev_rerun[1 - lane], 0));
            SamplerParams q = base_params(big);
            q.flags = p.flags;
            q.seed = seed;
            q.tag = tag;
            q.first = first;
            q.count = count;
            q.ticket = ticket + 1;
            q.frame = d_frame[frame];
            q.pairs = d_pairs;
            q.records = d_records;
            q.paths = d_paths;
            q.path_stride = path_stride;
            q.overflow_list = ovf_list;
            q.overflow_count = ovf_count + 1;
            q.overflow_total = d_ovf_total + 1;
            q.relist = ovf_list;
            q.count_ptr = ovf_count;
            launch_sample_dispatch(block, items, q, static_cast<u32>(big.slots), st);
            EBC_CUDA(cudaEventRecord(ev_rerun[lane], st));
            ++launches;
        }
    }

    void sync_sampling() {
        EBC_CUDA(cudaStreamSynchronize(s_sample));
        EBC_CUDA(cudaStreamSynchronize(s_sample2));
    }

    // Synchronises the sampling stream and returns {abandoned in small slots, abandoned in large slots}.
    void read_overflow(unsigned long long out[2]) {
        sync_sampling();
        EBC_CUDA(cudaMemcpy(out, d_ovf_total, 16, cudaMemcpyDeviceToHost));
        if (out[1] != 0)
            throw CudaError("internal: capacity overflow in a full-capacity slot");
    }
};

CudaSampler::CudaSampler(const HostGraph &g, const SamplerOptions &opt) : impl_(new Impl) {
    Impl &m = *impl_;
    const bool trace = std::getenv("EBC_TRACE") != nullptr;
    const auto c0 = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        if (trace) {
            cudaDeviceSynchronize();
            std::fprintf(stderr, "[ebc] CudaSampler ctor: %-22s at %.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count());
        }
    };
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw CudaError(std::string("no CUDA device available (this library has no CPU fallback): ") +
                        (e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e)));
    if (opt.device >= 0) {
        if (opt.device >= count)
            throw ConfigError("device ordinal out of range");
        EBC_CUDA(cudaSetDevice(opt.device));
    }
    EBC_CUDA(cudaGetDevice(&m.device));
    int cc_major = 0, cc_minor = 0; // (cudaGetDeviceProperties costs milliseconds; three attributes do not)
    EBC_CUDA(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, m.device));
    EBC_CUDA(cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, m.device));
    EBC_CUDA(cudaDeviceGetAttribute(&m.sm_count, cudaDevAttrMultiProcessorCount, m.device));
    if (cc_major < 10)
        throw CudaError("this build targets sm_100a (B200); found compute capability " +
                        std::to_string(cc_major) + "." + std::to_string(cc_minor));
    lap("device query");
    {
        // Experiment hook: cudaLimitMaxL2FetchGranularity.  The path is dominated by random 4..8-byte
        // probes, each of which pulls a 128-byte line from HBM; the limit was measured to change neither
        // the DRAM bytes nor the probe rate on B200 (profiles/r01_microbench_random_gather.txt), and
        // cudaDeviceSetLimit is not free, so it is only applied on request.
        if (const char *env = std::getenv("EBC_L2_FETCH_GRANULARITY")) {
            const size_t granularity = static_cast<size_t>(std::atoi(env));
            if (granularity == 32 || granularity == 64 || granularity == 128)
                cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, granularity);
        }
        cudaGetLastError();
    }
    require(g.n >= 2, "sampler: need at least two vertices");
    m.n = g.n;
    m.arcs = g.targets.size();

    m.s_sample = handles().take_stream();
    m.s_sample2 = handles().take_stream();
    m.s_agg = handles().take_stream();
    for (int i = 0; i < 2; ++i) {
        m.ev_sampled[i] = handles().take_event(false);
        m.ev_folded[i] = handles().take_event(false);
        m.ev_rerun[i] = handles().take_event(false);
    }
    m.ev_lane = handles().take_event(false);
    for (int i = 0; i < kEvents; ++i)
        m.ev_user[i] = handles().take_event(true);
    lap("streams and events");

    // ---- graph: replicated CSR, u64 offsets + u32 targets ----
    m.d_offsets = dev_alloc<u64>(g.n + 1);
    m.d_targets = dev_alloc<u32>(m.arcs + 4); // (+4: the probe reads whole 16-byte groups)
    // (a staged copy through pinned buffers was measured slower than the driver's pageable path here)
    EBC_CUDA(cudaMemcpyAsync(m.d_offsets, g.offsets.data(), (g.n + 1) * 8, cudaMemcpyHostToDevice, m.s_sample));
    if (m.arcs)
        EBC_CUDA(cudaMemcpyAsync(m.d_targets, g.targets.data(), m.arcs * 4, cudaMemcpyHostToDevice, m.s_sample));
    m.graph_bytes = (g.n + 1) * 8 + m.arcs * 4;
    lap("graph upload");

    // ---- launch shape ----
    m.flags = opt.materialize_final_level ? kFlagMaterializeFinal : 0u;
    if (opt.work_counters || opt.materialize_final_level)
        m.flags |= kFlagStats;
    if (const char *env = std::getenv("EBC_RESERVED_SMS")) // test / tuning hook
        m.reserved_sms = static_cast<u32>(std::atoi(env));
    else
        m.reserved_sms = opt.reserved_sms;
    m.reserved_sms = std::min<u32>(m.reserved_sms, m.sm_count > 1 ? static_cast<u32>(m.sm_count) - 1 : 0);
    std::uint64_t max_degree = 0;
    {
        // Visited bitmaps pay off when single rows are long enough to be probed (hub graphs); on
        // low-degree graphs they would only add an atomic per settled vertex.
        for (std::uint64_t v = 0; v < g.n; ++v)
            max_degree = std::max<std::uint64_t>(max_degree, g.degree(v));
        const char *env = std::getenv("EBC_BITMAP");
        m.hub_graph = max_degree >= 1024;
        // Launch shape (threads cooperating on one sample, adjacency slots per thread per tile), from
        // sweeps over R-MAT 14/17/20/24, Erdos-Renyi 10^4 and 10^6 and grids 300^2 / 2000^2
        // (profiles/r01_shapes.txt).  Small graphs mean little work per sample: more, smaller CTAs win
        // (config 1: 20.0 M samples/s at 128 threads, 27.6 M at 64, 34.4 M at 32).  Four slots per thread
        // pay once levels are long (R-MAT-20: 4.92 M vs 4.78 M; grid 2000^2: 170 k vs 150 k); on smaller
        // inputs two are faster (R-MAT-17: 13.7 M vs 11.4 M).
        // Hub graphs (profiles/r01_shapes.txt, second table): since every large final level is resolved by the
        // probe, no sample is much heavier than the rest and more, smaller CTAs win again -- up to the point
        // where the slot state (8 bytes of labels per vertex and slot) no longer fits: R-MAT-14/17 32x2
        // (42.7 / 22.3 M samples/s; 64x2 29.4 / 18.4 M), R-MAT-20 64x2 (9.0 M; 128x4 8.1 M), R-MAT-22 128x4,
        // R-MAT-24 256x4 (2.03 M; 512x2 1.55 M), R-MAT-26 512x4 (742 k; 256x4 614 k, 263 slots either way).
        if (m.hub_graph) {
            // (one warp per sample is the fastest shape up to 2^25 arcs when a launch holds many samples per slot --
            // config 2, 524 288-sample launches: 13.1 M samples/s against 10.9 M with two warps -- but not on the
            // 35 840-sample epochs of its pipeline run: 13.4 ms against 12.0 ms of adaptive phase)
            const u64 one_warp_below = opt.short_launches ? (u64{1} << 23) : (u64{1} << 25);
            const int lg = m.arcs < one_warp_below ? 0 : m.arcs < (u64{1} << 26) ? 1 : m.arcs < (u64{1} << 28) ? 2
                           : m.arcs < (u64{1} << 32) ? 3 : 4;
            static const u32 kBlock[5] = {32, 64, 128, 256, 512}, kItems[5] = {2, 2, 2, 4, 4}; // (R-MAT-22: 128x2 6.90 M, 128x4 6.60 M)
            m.block = opt.block_threads ? opt.block_threads : kBlock[lg];
            m.items = opt.items_per_thread ? opt.items_per_thread : kItems[lg];
        } else if (max_degree <= kEllWidth && m.arcs >= (u64{1} << 18) && !opt.block_threads) {
            // fixed-stride rows (expand_level_ell): two warps per sample (config 3: 64 threads 481 k samples/s,
            // 32 threads 473 k, 128 threads 443 k); the adjacency slots per thread mean nothing there
            m.block = 64;
            m.items = 2;
        } else {
            m.block = opt.block_threads ? opt.block_threads
                                        : (m.arcs < (u64{1} << 18) ? 32 : m.arcs < (u64{1} << 21) ? 64 : 128);
            m.items = opt.items_per_thread ? opt.items_per_thread : (m.arcs >= (u64{1} << 22) ? 4 : 2);
        }
        // Probe threshold (profiles/r01_probe_threshold.txt): with visited bitmaps a probe is cheap enough to pay
        // from 256 adjacency slots on (R-MAT-14 +13 %, R-MAT-20 +5 % over 2048); probing through labels, from 512.
        m.probe_min_slots = m.hub_graph ? 256 : 512;
        if (const char *pe = std::getenv("EBC_PROBE_MIN_SLOTS")) // tuning hook (tools/sweep_probe_min.py)
            m.probe_min_slots = std::strtoull(pe, nullptr, 0);
        if (const char *pe = std::getenv("EBC_PROBE_GROWTH_X4")) // tuning hook
            m.probe_growth_x4 = std::strtoull(pe, nullptr, 0);
        const bool want = env ? std::atoi(env) != 0 : m.hub_graph;
        if (want && !opt.materialize_final_level)
            m.flags |= kFlagUseBitmap;
    }
    // Hub-clustered numbering: on graphs with hubs most adjacency entries name a few high-degree
    // vertices; numbering by descending degree puts their labels / visited bits next to each other
    // (measured on R-MAT: +11 % at scale 20, +26 % at scale 24; +30..65 % when the input ids are
    // arbitrary).  Low-degree graphs keep their own numbering, which usually is spatially coherent.
    // Hub-free graphs too large for their labels to stay in L2 (grids, road networks) are numbered by
    // neighbourhood clusters instead (cluster_*_kernel above): config 3, see DESIGN.md section 3.
    int numbering = opt.renumber > 0 ? opt.renumber : opt.renumber < 0 ? 0 : m.hub_graph ? 1 : m.n >= (u64{1} << 18) ? 2 : 0;
    if (const char *env = std::getenv("EBC_RENUMBER"))
        numbering = std::atoi(env);
    if (numbering < 0 || numbering > 2)
        throw ConfigError("renumber must be -1 (never), 0 (auto), 1 (degree classes) or 2 (neighbourhood clusters)");
    const bool want_dense = numbering != 0 && m.arcs && m.n < (u64{1} << 31); // (the CUB passes take 32-bit counts)
    // Fixed-stride rows (expand_level_ell): lattice-like graphs, where a sample is a long chain of small levels.
    bool want_ell = !m.hub_graph && max_degree <= kEllWidth && m.arcs && m.n < kEllIdMask && m.block <= 128;
    if (const char *env = std::getenv("EBC_ELL"))
        want_ell = want_ell && std::atoi(env) != 0;
    // 16-byte rows when no row has more than four entries (EBC_ELL_WIDTH=8: the wide rows all the same)
    m.ell_width = max_degree <= kEllNarrow ? kEllNarrow : kEllWidth;
    if (const char *env = std::getenv("EBC_ELL_WIDTH"))
        if (std::atoi(env) == static_cast<int>(kEllWidth))
            m.ell_width = kEllWidth;
    // ... and, on request (EBC_ELL4=1), a 16-byte copy of 32-byte rows for the expansion (SamplerParams::ell4).  Not a
    // default: on config 3 (0.2 % of the rows longer than four entries) it halves the row bytes and changes the rate by
    // +0.5 % -- that kernel is bound by the number of random sector accesses, not by their bytes.
    m.want_ell4 = false;
    if (const char *env = std::getenv("EBC_ELL4"))
        m.want_ell4 = want_ell && m.ell_width == kEllWidth && std::atoi(env) != 0;
    const int per_sm = occupancy_for(m.block, m.items, want_ell);
    m.per_sm = per_sm;
    lap("occupancy query");
    if (per_sm < 1)
        throw CudaError("sampling kernel does not fit on an SM");
    // (hub graphs: the probe never settles a large final level, a side rarely holds 10^5 vertices, and with n/32
    // config 5 fits 592 slots of 256 threads: 1.71 M samples/s, n/16 1.58 M, n/8 with the 515 slots that fit 1.47 M)
    u64 cap = opt.slot_capacity ? std::min<u64>(opt.slot_capacity, g.n)
                                : std::min<u64>(g.n, std::max<u64>(u64{1} << 17, m.hub_graph ? g.n / 32 : g.n / 8));
    // (While large final levels were still settled, n/6 instead of n/4 cost 10x throughput through the re-run
    // path on R-MAT graphs; now that they are only scanned, n/16 runs as fast as n/4 on R-MAT-20/24/26 --
    // profiles/r01_capacity_sweep.txt.  n/8 lets config 5 keep two 512-thread CTAs per SM.)
    cap = std::max<u64>(cap, 2);
    u64 slots = opt.slots ? opt.slots : static_cast<u64>(per_sm) * m.sm_count;
    const u64 capacity = pool().capacity();
    const u64 live = pool().live_bytes();
    lap("memory query");
    const u64 fixed = (g.n + 1) * (4 * 2 + 8 + 8 + 16 + 12) + (u64{256} << 20) + kOverflowCap * 4 +
                      (cap < g.n ? kLargeSlots * SlotArrays::bytes_per_slot(g.n, g.n, want_ell) : 0) +
                      (want_dense ? g.n * 40 + m.arcs * 4 + (u64{16} << 20) : 0) + // the dense copy is built below
                      (want_ell ? g.n * (kEllWidth + kEllNarrow) * 4 : 0);
    // Buffers cached by the pool are reusable (or released on demand), so they count as free.
    const u64 avail = capacity > live ? capacity - live : 0;
    const u64 budget = avail > fixed ? (avail - fixed) / 10 * 8 : 0;
    const u64 per_slot = SlotArrays::bytes_per_slot(g.n, cap, want_ell);
    if (!opt.slots && slots * per_slot > budget)
        slots = budget / per_slot;
    if (slots < 1)
        throw CudaError("not enough device memory for a single sampling slot");
    // The slot arrays are cleared on the aggregation stream while the graph is still crossing PCIe on the
    // sampling stream (the numbering below waits for it).
    m.small.allocate(slots, cap, g.n, want_ell, m.s_agg);
    if (cap < g.n)
        m.big.allocate(kLargeSlots, g.n, g.n, want_ell, m.s_agg);
    lap("slot arrays");
    if (want_dense) {
        m.build_dense_graph(numbering == 2);
        m.numbering = numbering;
    }
    lap("dense numbering");
    if (want_ell)
        m.build_fixed_rows();
    lap("fixed-stride rows");

    // ---- frames, state, bookkeeping ----
    for (int i = 0; i < 2; ++i) {
        m.d_frame[i] = dev_alloc<u32>(g.n + 1);
        EBC_CUDA(cudaMemsetAsync(m.d_frame[i], 0, (g.n + 1) * 4, m.s_sample));
        m.h_result[i] = handles().take_words();
        m.h_result[i][0] = m.h_result[i][1] = 0;
    }
    m.d_ovf_total = dev_alloc<unsigned long long>(2);
    EBC_CUDA(cudaMemsetAsync(m.d_ovf_total, 0, 16, m.s_sample));
    m.d_S = dev_alloc<u64>(g.n + 1);
    m.d_wide = dev_alloc<u64>(g.n + 1);
    EBC_CUDA(cudaMemsetAsync(m.d_S, 0, (g.n + 1) * 8, m.s_sample));
    m.d_ticket = dev_alloc<unsigned long long>(4);
    m.d_started = dev_alloc<u32>(2);
    {
        m.d_ring = dev_alloc<u32>(m.small.slots);
        std::vector<u32> ids(m.small.slots);
        for (u64 i = 0; i < m.small.slots; ++i)
            ids[i] = static_cast<u32>(i);
        EBC_CUDA(cudaMemcpyAsync(m.d_ring, ids.data(), ids.size() * 4, cudaMemcpyHostToDevice, m.s_sample));
        m.d_ring_pos = dev_alloc<unsigned long long>(2);
        EBC_CUDA(cudaMemsetAsync(m.d_ring_pos, 0, 16, m.s_sample));
        EBC_CUDA(cudaStreamSynchronize(m.s_sample)); // ids goes out of scope
    }
    m.d_work = dev_alloc<unsigned long long>(kWorkCounters);
    EBC_CUDA(cudaMemsetAsync(m.d_work, 0, kWorkCounters * 8, m.s_sample));
    m.d_overflow_list = dev_alloc<u32>(2 * static_cast<u64>(kOverflowCap));
    m.d_overflow_count = dev_alloc<u32>(4);
    m.d_fail = dev_alloc<u32>(1);
    EBC_CUDA(cudaMemsetAsync(m.d_fail, 0, 4, m.s_sample));
    m.d_log_lower = dev_alloc<double>(g.n);
    m.d_log_upper = dev_alloc<double>(g.n);
    m.stop.have = 0;
    EBC_CUDA(cudaStreamSynchronize(m.s_sample));
    lap("frames and bookkeeping");
    if (trace)
        pool().stats("after ctor");
}

// Everything the sampler holds goes back to the process-wide caches here, in the destructor of Impl, so that a
// constructor that throws half way (out of memory, kernel does not fit, ...) returns what it had taken:
// impl_ is a complete member by then and is destroyed during unwinding.  Null handles are skipped.
CudaSampler::Impl::~Impl() {
    Impl &m = *this;
    const bool trace = std::getenv("EBC_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    cudaDeviceSynchronize();
    if (trace)
        std::fprintf(stderr, "[ebc] ~CudaSampler: device sync %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
    m.small.release();
    m.big.release();
    dev_free(m.d_offsets);
    dev_free(m.d_targets);
    dev_free(m.d_dense_offsets);
    dev_free(m.d_dense_targets);
    dev_free(m.d_to_dense);
    dev_free(m.d_to_ext);
    dev_free(m.d_ell);
    dev_free(m.d_ell4);
    for (int i = 0; i < 2; ++i) {
        dev_free(m.d_frame[i]);
        handles().give_words(m.h_result[i]);
        handles().give_event(m.ev_sampled[i], false);
        handles().give_event(m.ev_folded[i], false);
        handles().give_event(m.ev_rerun[i], false);
    }
    handles().give_event(m.ev_lane, false);
    for (int i = 0; i < kEvents; ++i)
        handles().give_event(m.ev_user[i], true);
    dev_free(m.d_ovf_total);
    dev_free(m.d_S);
    dev_free(m.d_wide);
    dev_free(m.d_ticket);
    dev_free(m.d_started);
    dev_free(m.d_ring);
    dev_free(m.d_ring_pos);
    dev_free(m.d_work);
    dev_free(m.d_overflow_list);
    dev_free(m.d_overflow_count);
    dev_free(m.d_fail);
    dev_free(m.d_log_lower);
    dev_free(m.d_log_upper);
    dev_free(m.d_dist);
    dev_free(m.d_queue[0]);
    dev_free(m.d_queue[1]);
    dev_free(m.d_bfs);
    dev_free(m.d_best);
    dev_free(m.d_flush);
    handles().give_stream(m.s_sample);
    handles().give_stream(m.s_sample2);
    handles().give_stream(m.s_agg);
    if (trace)
        pool().stats("after dtor");
    if (trace)
        std::fprintf(stderr, "[ebc] ~CudaSampler: total %.3f ms\n",
                     std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
}

CudaSampler::~CudaSampler() = default;

std::uint64_t CudaSampler::n() const { return impl_->n; }
std::uint64_t CudaSampler::overflow_samples() const {
    unsigned long long o[2];
    impl_->read_overflow(o);
    return o[0];
}
std::uint64_t CudaSampler::kernel_launches() const { return impl_->launches; }

void CudaSampler::sample(std::uint64_t seed, std::uint32_t tag, std::uint64_t first, std::uint64_t count, int frame) {
    Impl &m = *impl_;
    require(frame == 0 || frame == 1, "sample: frame must be 0 or 1");
    // The frame is being reused: the fold that zeroes it must have finished (epoch.hpp:24-30).
    cudaStream_t st = m.lane_stream(frame);
    EBC_CUDA(cudaStreamWaitEvent(st, m.ev_folded[frame], 0));
    for (u64 done = 0; done < count; done += kOverflowCap) {
        const u64 chunk = std::min<u64>(kOverflowCap, count - done);
        m.launch(seed, tag, first + done, chunk, frame, nullptr, nullptr, nullptr, 0);
    }
    EBC_CUDA(cudaEventRecord(m.ev_sampled[frame], st));
}

void CudaSampler::sample_debug(std::uint64_t seed, std::uint32_t tag, std::uint64_t first, std::uint64_t count,
                               const std::uint32_t *pairs, int frame, SampleRecordHost *records,
                               std::uint32_t *paths, std::uint64_t path_stride) {
    Impl &m = *impl_;
    require(frame == 0 || frame == 1, "sample_debug: frame must be 0 or 1");
    require(count <= kOverflowCap, "sample_debug: at most 2^20 samples per call");
    static_assert(sizeof(SampleRecordHost) == sizeof(SampleRecordDev), "record layouts must match");
    u32 *d_pairs = nullptr, *d_paths = nullptr;
    SampleRecordDev *d_rec = nullptr;
    if (count == 0)
        return;
    cudaStream_t st = m.lane_stream(frame);
    try {
        EBC_CUDA(cudaStreamWaitEvent(st, m.ev_folded[frame], 0));
        if (pairs) {
            d_pairs = dev_alloc<u32>(2 * count);
            EBC_CUDA(cudaMemcpyAsync(d_pairs, pairs, 2 * count * 4, cudaMemcpyHostToDevice, st));
        }
        if (records)
            d_rec = dev_alloc<SampleRecordDev>(count);
        if (paths && path_stride) {
            d_paths = dev_alloc<u32>(count * path_stride);
            EBC_CUDA(cudaMemsetAsync(d_paths, 0xff, count * path_stride * 4, st));
        }
        m.launch(seed, tag, first, count, frame, d_pairs, d_rec, d_paths, d_paths ? path_stride : 0);
        EBC_CUDA(cudaEventRecord(m.ev_sampled[frame], st));
        if (records)
            EBC_CUDA(cudaMemcpyAsync(records, d_rec, count * sizeof(SampleRecordDev), cudaMemcpyDeviceToHost, st));
        if (d_paths)
            EBC_CUDA(cudaMemcpyAsync(paths, d_paths, count * path_stride * 4, cudaMemcpyDeviceToHost, st));
        unsigned long long ovf[2];
        m.read_overflow(ovf);
    } catch (...) {
        dev_free(d_pairs);
        dev_free(d_rec);
        dev_free(d_paths);
        throw;
    }
    dev_free(d_pairs);
    dev_free(d_rec);
    dev_free(d_paths);
}

// Decodes the label / list / sigma / level arrays of the slot that ran the last
// sample of a single-slot sampler into per-vertex dist and sigma.
void CudaSampler::last_state(int side, std::uint32_t *dist_out, std::uint64_t *sigma_out) {
    Impl &m = *impl_;
    require(side == 0 || side == 1, "last_state: side must be 0 or 1");
    require(m.small.slots == 1, "last_state: needs a sampler created with slots == 1");
    unsigned long long ovf[2];
    m.read_overflow(ovf);
    // If the last sample overflowed it was re-run in large slot 0.
    const bool rerun = m.small.cap < m.n && ovf[0] != m.overflow_seen;
    m.overflow_seen = ovf[0];
    const SlotArrays &a = rerun ? m.big : m.small;
    std::vector<u32> hdr(kHdrWords);
    EBC_CUDA(cudaMemcpy(hdr.data(), a.hdr, kHdrWords * 4, cudaMemcpyDeviceToHost));
    const u32 cnt = hdr[kHdrLastCnt0 + side], depth = hdr[kHdrLastDepth0 + side];
    std::vector<u32> list(cnt), lvl(depth + 2);
    std::vector<u64> sig(cnt);
    EBC_CUDA(cudaMemcpy(list.data(), a.list + static_cast<u64>(side) * a.cap, cnt * 4ull, cudaMemcpyDeviceToHost));
    EBC_CUDA(cudaMemcpy(sig.data(), a.sig + static_cast<u64>(side) * a.cap, cnt * 8ull, cudaMemcpyDeviceToHost));
    EBC_CUDA(cudaMemcpy(lvl.data(), a.lvl + static_cast<u64>(side) * (a.aux_cap + 2), (depth + 1) * 4ull, cudaMemcpyDeviceToHost));
    lvl[depth + 1] = cnt;
    for (u64 v = 0; v < m.n; ++v) {
        dist_out[v] = 0xffffffffu;
        sigma_out[v] = 0;
    }
    if (m.d_to_ext && m.h_to_ext.empty()) {
        m.h_to_ext.resize(m.n);
        EBC_CUDA(cudaMemcpy(m.h_to_ext.data(), m.d_to_ext, m.n * 4, cudaMemcpyDeviceToHost));
    }
    for (u32 d = 0; d <= depth; ++d)
        for (u32 i = lvl[d]; i < lvl[d + 1]; ++i) {
            const u32 v = m.d_to_ext ? m.h_to_ext[list[i]] : list[i]; // the slot lists hold dense ids
            dist_out[v] = d;
            sigma_out[v] = sig[i];
        }
}

void CudaSampler::set_stopping(double eps, std::uint64_t omega, const double *delta_lower,
                               const double *delta_upper, int bound) {
    Impl &m = *impl_;
    require(bound == 0 || bound == 1, "set_stopping: unknown bound kind");
    std::vector<double> lo(m.n), up(m.n);
    bound_log_terms(delta_lower, m.n, bound, lo.data());
    bound_log_terms(delta_upper, m.n, bound, up.data());
    // (on the stream that reads them; a pageable cudaMemcpy only orders against the legacy stream, which the
    // sampler's non-blocking streams do not synchronise with)
    EBC_CUDA(cudaMemcpyAsync(m.d_log_lower, lo.data(), m.n * 8, cudaMemcpyHostToDevice, m.s_agg));
    EBC_CUDA(cudaMemcpyAsync(m.d_log_upper, up.data(), m.n * 8, cudaMemcpyHostToDevice, m.s_agg));
    EBC_CUDA(cudaStreamSynchronize(m.s_agg)); // lo / up go out of scope
    m.stop.eps = eps;
    m.stop.omega = omega;
    m.stop.log_lower = m.d_log_lower;
    m.stop.log_upper = m.d_log_upper;
    m.stop.bound = bound;
    m.stop.have = 1;
}

void CudaSampler::set_stopping_uniform(double eps, std::uint64_t omega, double delta_each, int bound) {
    Impl &m = *impl_;
    require(bound == 0 || bound == 1, "set_stopping: unknown bound kind");
    double term = 0.0;
    bound_log_terms(&delta_each, 1, bound, &term); // the host libm's log, as for per-vertex values
    fill_two_kernel<<<static_cast<u32>(m.sm_count) * 4, 256, 0, m.s_agg>>>(m.d_log_lower, m.d_log_upper, m.n, term);
    EBC_CUDA(cudaGetLastError());
    m.stop.eps = eps;
    m.stop.omega = omega;
    m.stop.log_lower = m.d_log_lower;
    m.stop.log_upper = m.d_log_upper;
    m.stop.bound = bound;
    m.stop.have = 1;
}

void CudaSampler::fold_and_check_async(int frame, AllreduceFn allreduce, void *user) {
    Impl &m = *impl_;
    require(frame == 0 || frame == 1, "fold_and_check: frame must be 0 or 1");
    EBC_CUDA(cudaStreamWaitEvent(m.s_agg, m.ev_sampled[frame], 0));
    if (allreduce) {
        if (allreduce(user, m.d_frame[frame], m.n + 1, m.s_agg) != 0)
            throw BackendFault("allreduce callback failed");
    }
    m.h_result[frame][0] = ~u64{0};
    u64 *d_result = nullptr;
    EBC_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void **>(&d_result), m.h_result[frame], 0));
    const u32 grid = static_cast<u32>(std::min<u64>((m.n + 255) / 256, static_cast<u64>(m.sm_count) * 8));
    fold_check_kernel<<<grid, 256, 0, m.s_agg>>>(m.d_frame[frame], m.d_S, m.n, m.stop, m.d_fail);
    finish_fold_kernel<<<1, 1, 0, m.s_agg>>>(m.d_frame[frame], m.d_S, m.stop, m.d_fail, d_result);
    EBC_CUDA(cudaGetLastError());
    m.launches += 2;
    EBC_CUDA(cudaEventRecord(m.ev_folded[frame], m.s_agg));
    m.folded_pending[frame] = true;
}

bool CudaSampler::wait_fold(int frame, std::uint64_t *tau_out) {
    Impl &m = *impl_;
    require(frame == 0 || frame == 1, "wait_fold: frame must be 0 or 1");
    require(m.folded_pending[frame], "wait_fold: no fold in flight for this frame");
    EBC_CUDA(cudaEventSynchronize(m.ev_folded[frame]));
    m.folded_pending[frame] = false;
    if (tau_out)
        *tau_out = m.h_result[frame][1];
    return m.h_result[frame][0] == 1;
}

void CudaSampler::discard_frame(int frame) {
    Impl &m = *impl_;
    require(frame == 0 || frame == 1, "discard_frame: frame must be 0 or 1");
    EBC_CUDA(cudaStreamWaitEvent(m.s_agg, m.ev_sampled[frame], 0));
    EBC_CUDA(cudaMemsetAsync(m.d_frame[frame], 0, (m.n + 1) * 4, m.s_agg));
    EBC_CUDA(cudaEventRecord(m.ev_folded[frame], m.s_agg));
    EBC_CUDA(cudaStreamSynchronize(m.s_agg));
}

void CudaSampler::read_frame(int which, std::uint64_t *words_out) {
    Impl &m = *impl_;
    require(which >= 0 && which <= 2, "read_frame: which must be 0, 1 or 2");
    m.sync_sampling();
    EBC_CUDA(cudaStreamSynchronize(m.s_agg));
    if (which == 2) {
        EBC_CUDA(cudaMemcpy(words_out, m.d_S, (m.n + 1) * 8, cudaMemcpyDeviceToHost));
        return;
    }
    widen_kernel<<<static_cast<u32>(m.sm_count) * 4, 256, 0, m.s_sample>>>(m.d_frame[which], m.d_wide, m.n + 1);
    EBC_CUDA(cudaGetLastError());
    EBC_CUDA(cudaMemcpyAsync(words_out, m.d_wide, (m.n + 1) * 8, cudaMemcpyDeviceToHost, m.s_sample));
    EBC_CUDA(cudaStreamSynchronize(m.s_sample));
}

void CudaSampler::write_state(const std::uint64_t *words) {
    Impl &m = *impl_;
    m.sync_sampling();
    EBC_CUDA(cudaMemcpyAsync(m.d_S, words, (m.n + 1) * 8, cudaMemcpyHostToDevice, m.s_agg));
    EBC_CUDA(cudaStreamSynchronize(m.s_agg));
}

void CudaSampler::clear() {
    Impl &m = *impl_;
    m.sync_sampling();
    // All streams are idle here; the memsets run on the aggregation stream and are complete on return, so
    // whatever the caller launches next (on any of the sampler's streams) is ordered behind them.
    for (int i = 0; i < 2; ++i)
        EBC_CUDA(cudaMemsetAsync(m.d_frame[i], 0, (m.n + 1) * 4, m.s_agg));
    EBC_CUDA(cudaMemsetAsync(m.d_S, 0, (m.n + 1) * 8, m.s_agg));
    EBC_CUDA(cudaStreamSynchronize(m.s_agg));
}

void CudaSampler::work(std::uint64_t *out, bool reset) {
    Impl &m = *impl_;
    m.sync_sampling();
    EBC_CUDA(cudaMemcpyAsync(out, m.d_work, kWorkCounters * 8, cudaMemcpyDeviceToHost, m.s_sample));
    if (reset)
        EBC_CUDA(cudaMemsetAsync(m.d_work, 0, kWorkCounters * 8, m.s_sample));
    EBC_CUDA(cudaStreamSynchronize(m.s_sample)); // both lanes are idle: the next launch on either sees the reset
}

void CudaSampler::mark(int event) {
    require(event >= 0 && event < kEvents, "mark: event index out of range");
    // The mark completes when BOTH sampling lanes have reached this point.
    Impl &m = *impl_;
    EBC_CUDA(cudaEventRecord(m.ev_lane, m.s_sample2));
    EBC_CUDA(cudaStreamWaitEvent(m.s_sample, m.ev_lane, 0));
    EBC_CUDA(cudaEventRecord(m.ev_user[event], m.s_sample));
    EBC_CUDA(cudaStreamWaitEvent(m.s_sample2, m.ev_user[event], 0));
}

float CudaSampler::elapsed_ms(int from, int to) {
    require(from >= 0 && from < kEvents && to >= 0 && to < kEvents, "elapsed_ms: event index out of range");
    EBC_CUDA(cudaEventSynchronize(impl_->ev_user[to]));
    float ms = 0.f;
    EBC_CUDA(cudaEventElapsedTime(&ms, impl_->ev_user[from], impl_->ev_user[to]));
    return ms;
}

void CudaSampler::sync() {
    impl_->sync_sampling();
    EBC_CUDA(cudaStreamSynchronize(impl_->s_agg));
}

void CudaSampler::info(std::uint64_t *out) {
    Impl &m = *impl_;
    out[0] = m.small.slots;
    out[1] = m.block;
    out[2] = m.small.cap;
    out[3] = m.small.bytes + m.big.bytes + m.graph_bytes + (m.n + 1) * (4 * 2 + 8 + 8 + 16);
    out[4] = static_cast<std::uint64_t>(m.sm_count);
    out[5] = (m.launches & ((std::uint64_t{1} << 48) - 1)) | (static_cast<std::uint64_t>(m.numbering) << 48) |
             (static_cast<std::uint64_t>(m.d_ell ? 1 : 0) << 52) |
             (static_cast<std::uint64_t>(m.d_ell && m.ell_width == kEllNarrow ? 1 : 0) << 53) |
             (static_cast<std::uint64_t>(m.d_ell4 ? 1 : 0) << 54) | (static_cast<std::uint64_t>(m.items) << 56);
}

void *CudaSampler::stream_handle() { return impl_->s_sample; }

void CudaSampler::frame_ptr(int frame, void **ptr, std::uint64_t *words) {
    require(frame == 0 || frame == 1, "frame_ptr: frame must be 0 or 1");
    *ptr = impl_->d_frame[frame];
    *words = impl_->n + 1;
}

BfsSummary CudaSampler::bfs(std::uint32_t source, std::uint32_t *dist_out) {
    Impl &m = *impl_;
    require(source < m.n, "bfs: source out of range");
    if (!m.d_dist) {
        m.d_dist = dev_alloc<u32>(m.n);
        m.d_queue[0] = dev_alloc<u32>(m.n);
        m.d_queue[1] = dev_alloc<u32>(m.n);
        m.d_bfs = dev_alloc<BfsState>(1);
        m.d_best = dev_alloc<unsigned long long>(1);
    }
    cudaStream_t st = m.s_sample;
    EBC_CUDA(cudaMemsetAsync(m.d_dist, 0xff, m.n * 4, st));
    BfsState init{};
    init.queue_size[0] = 1;
    init.reached = 1;
    init.have_queue = 1;
    EBC_CUDA(cudaMemcpyAsync(m.d_bfs, &init, sizeof(init), cudaMemcpyHostToDevice, st));
    const u32 zero = 0;
    EBC_CUDA(cudaMemcpyAsync(m.d_dist + source, &zero, 4, cudaMemcpyHostToDevice, st));
    EBC_CUDA(cudaMemcpyAsync(m.d_queue[0], &source, 4, cudaMemcpyHostToDevice, st));
    EBC_CUDA(cudaMemsetAsync(m.d_best, 0, 8, st));
    const u32 grid = static_cast<u32>(m.sm_count) * 8;
    const u32 allow_bu = m.hub_graph ? 1u : 0u; // low-degree graphs stay top-down (2 launches per level)
    // Only the head of the state (done, reached) comes back per round trip; levels are enqueued in
    // batches of 8, 16, 32, 32 ...: launches after the search is done are no-ops, but not free.
    struct { u32 queue_size[2]; u32 depth; u32 done; u64 reached; } host{};
    static_assert(offsetof(BfsState, reached) == 16, "BfsState head layout");
    int batch = 8;
    for (u32 level = 0;;) {
        for (int k = 0; k < batch; ++k, ++level) {
            if (allow_bu) {
                bfs_rebuild_queue_kernel<<<grid, 256, 0, st>>>(m.d_dist, m.n, m.d_queue[0], m.d_queue[1], m.d_bfs, level);
                bfs_bottom_up_kernel<<<grid, 256, 0, st>>>(m.d_offsets, m.d_targets, m.d_dist, m.n, m.d_bfs, level);
                m.launches += 2;
            }
            bfs_level_kernel<<<grid, 256, 0, st>>>(m.d_offsets, m.d_targets, m.d_dist, m.d_queue[0], m.d_queue[1], m.d_bfs, level);
            if (m.hub_graph) { // rows above kBfsBigRow exist only there
                bfs_big_rows_kernel<<<grid, 256, 0, st>>>(m.d_offsets, m.d_targets, m.d_dist, m.d_queue[0], m.d_queue[1], m.d_bfs, level);
                ++m.launches;
            }
            bfs_advance_kernel<<<1, 1, 0, st>>>(m.d_bfs, level, m.arcs, allow_bu);
            m.launches += 2;
        }
        EBC_CUDA(cudaGetLastError());
        EBC_CUDA(cudaMemcpyAsync(&host, m.d_bfs, sizeof(host), cudaMemcpyDeviceToHost, st));
        EBC_CUDA(cudaStreamSynchronize(st));
        if (host.done)
            break;
        batch = batch < 32 ? batch * 2 : 32;
    }
    bfs_farthest_kernel<<<grid, 256, 0, st>>>(m.d_dist, m.n, m.d_best);
    ++m.launches;
    unsigned long long best = 0;
    EBC_CUDA(cudaMemcpyAsync(&best, m.d_best, 8, cudaMemcpyDeviceToHost, st));
    if (dist_out)
        EBC_CUDA(cudaMemcpyAsync(dist_out, m.d_dist, m.n * 4, cudaMemcpyDeviceToHost, st));
    EBC_CUDA(cudaStreamSynchronize(st));
    BfsSummary r;
    r.eccentricity = static_cast<u32>(best >> 32);
    r.farthest = 0xffffffffu - static_cast<u32>(best & 0xffffffffu);
    r.reached = host.reached;
    return r;
}

void CudaSampler::flush_l2() {
    Impl &m = *impl_;
    if (!m.d_flush) {
        m.flush_words = (u64{192} << 20) / 4; // 192 MiB > 126 MB L2
        m.d_flush = dev_alloc<u32>(m.flush_words);
    }
    static u32 salt = 0;
    flush_kernel<<<static_cast<u32>(m.sm_count) * 8, 256, 0, m.s_sample>>>(m.d_flush, m.flush_words, ++salt);
    EBC_CUDA(cudaGetLastError());
}

} // namespace ebc
