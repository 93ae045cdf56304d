// Graph ingestion on the GPU (SURVEY.md section 8f, N3, and the generator half of N4): canonical CSR from
// arcs, largest connected component, and the R-MAT generator, for inputs where the host versions in
// host_graph.cpp take minutes (scale 26: 70 s to generate, 30 s for the component).
//
// Behavioural contract as in host_graph.cpp (what, not how):
//   Graph::from_edges            /root/reference/proj/src/graph.cpp:14-46   symmetrise, drop loops and duplicates,
//                                                                           rows ascending
//   largest_connected_component  graph.cpp:229-290   largest component, ties toward the smallest minimum original
//                                                     id (:262-267), order-preserving dense renumbering (:269-289)
//   gen_rmat quadrant convention rmat.cpp:24-42      (stream: Philox, see host_graph.cpp gen_rmat)
// Every function returns exactly the HostGraph its host counterpart returns (tested array for array);
// nothing here is a fallback for anything -- without a CUDA device these functions throw.
#include <cuda_runtime.h>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>

#include <cmath>
#include <cstdio>
#include <string>

#include "cuda_sampler.hpp"
#include "device_graph.hpp"
#include "philox.cuh"

namespace ebc {
namespace {

using u32 = std::uint32_t;
using u64 = std::uint64_t;

void check(cudaError_t e, const char *what, int line) {
    if (e != cudaSuccess) {
        char buf[384];
        std::snprintf(buf, sizeof(buf), "CUDA failure: %s: %s (device_graph.cu:%d)", what, cudaGetErrorString(e), line);
        throw CudaError(buf);
    }
}
#define DG_CUDA(expr) check((expr), #expr, __LINE__)

template <typename T> struct DevBuf {
    T *p = nullptr;
    u64 count = 0;
    DevBuf() = default;
    explicit DevBuf(u64 n) { alloc(n); }
    DevBuf(const DevBuf &) = delete;
    DevBuf &operator=(const DevBuf &) = delete;
    DevBuf(DevBuf &&o) noexcept : p(o.p), count(o.count) {
        o.p = nullptr;
        o.count = 0;
    }
    DevBuf &operator=(DevBuf &&o) noexcept {
        if (this != &o) {
            release();
            p = o.p;
            count = o.count;
            o.p = nullptr;
            o.count = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(u64 n) {
        release();
        count = n;
        const size_t bytes = std::max<u64>(n, 1) * sizeof(T);
        cudaError_t e = cudaMalloc(reinterpret_cast<void **>(&p), bytes);
        if (e == cudaErrorMemoryAllocation) { // the samplers' buffer cache may be holding the memory
            cudaGetLastError();
            release_device_cache();
            e = cudaMalloc(reinterpret_cast<void **>(&p), bytes);
        }
        check(e, "cudaMalloc", __LINE__);
    }
    void release() {
        if (p)
            cudaFree(p);
        p = nullptr;
        count = 0;
    }
    void swap(DevBuf &o) {
        std::swap(p, o.p);
        std::swap(count, o.count);
    }
};

void select_device(int device) {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        throw CudaError(std::string("no CUDA device available for device-side graph ingestion: ") +
                        (e == cudaSuccess ? "device count is 0" : cudaGetErrorString(e)));
    if (device >= 0) {
        if (device >= count)
            throw ConfigError("device ordinal out of range");
        DG_CUDA(cudaSetDevice(device));
    }
}

constexpr u64 kLoopKey = ~u64{0}; // marks a dropped arc; sorts behind every real key

inline u32 grid_for(u64 items, u32 block = 256) {
    const u64 blocks = (items + block - 1) / block;
    return static_cast<u32>(std::min<u64>(std::max<u64>(blocks, 1), u64{148} * 32));
}

// ---- R-MAT arcs: same stream and quadrant rule as gen_rmat in host_graph.cpp ----
__global__ void __launch_bounds__(256) rmat_keys_kernel(u64 *keys, u64 samples, int scale, double a, double ab, double abc,
                                                        u64 seed) {
    const double inv53 = 1.0 / 9007199254740992.0;
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < samples;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        SampleStream st(seed, kTagGenRmat, i);
        u64 u = 0, v = 0, w0 = 0, w1 = 0;
        for (int bit = 0; bit < scale; ++bit) {
            if ((bit & 1) == 0)
                st.next_u64x2(w0, w1);
            const double r = static_cast<double>(((bit & 1) ? w1 : w0) >> 11) * inv53;
            u <<= 1;
            v <<= 1;
            if (r < a) {
            } else if (r < ab) {
                v |= 1;
            } else if (r < abc) {
                u |= 1;
            } else {
                u |= 1;
                v |= 1;
            }
        }
        const bool loop = u == v; // graph.cpp:20-21 drops self-loops
        keys[2 * i] = loop ? kLoopKey : ((u << 32) | v);
        keys[2 * i + 1] = loop ? kLoopKey : ((v << 32) | u);
    }
}

__global__ void __launch_bounds__(256) edge_keys_kernel(const u64 *src, const u64 *dst, u64 count, u64 n, u64 *keys,
                                                        u32 *bad) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 u = src[i], v = dst[i];
        if (u >= n || v >= n) {
            *bad = 1;
            keys[2 * i] = keys[2 * i + 1] = kLoopKey;
            continue;
        }
        const bool loop = u == v;
        keys[2 * i] = loop ? kLoopKey : ((u << 32) | v);
        keys[2 * i + 1] = loop ? kLoopKey : ((v << 32) | u);
    }
}

// offsets[u] = first index of a key with source >= u (keys sorted, unique, `count` of them)
__global__ void __launch_bounds__(256) row_offsets_kernel(const u64 *keys, u64 count, u64 n, u64 *offsets) {
    for (u64 u = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; u <= n;
         u += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u64 want = u << 32;
        u64 lo = 0, hi = count; // first index with keys[idx] >= want
        while (lo < hi) {
            const u64 mid = (lo + hi) >> 1;
            if (keys[mid] < want)
                lo = mid + 1;
            else
                hi = mid;
        }
        offsets[u] = u == n ? count : lo;
    }
}

__global__ void __launch_bounds__(256) low_words_kernel(const u64 *keys, u64 count, u32 *targets) {
    for (u64 i = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<u64>(gridDim.x) * blockDim.x)
        targets[i] = static_cast<u32>(keys[i]);
}

struct DeviceCsr {
    u64 n = 0, arcs = 0;
    DevBuf<u64> offsets;
    DevBuf<u32> targets;
};

// keys: `count` arc keys in any order, kLoopKey = dropped.  Consumes (frees) the key buffer.
DeviceCsr csr_from_keys(u64 n, DevBuf<u64> &keys, u64 count) {
    DeviceCsr g;
    g.n = n;
    if (n > (u64{1} << 32))
        throw ConfigError("graph: more than 2^32 vertices are not supported (32-bit vertex ids)");
    g.offsets.alloc(n + 1);
    if (count == 0) {
        DG_CUDA(cudaMemset(g.offsets.p, 0, (n + 1) * 8));
        g.targets.alloc(0);
        keys.release();
        return g;
    }
    DevBuf<u64> alt(count);
    const ::cuda::std::int64_t items = static_cast<::cuda::std::int64_t>(count);
    {
        size_t bytes = 0;
        DG_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys.p, alt.p, items, 0, 64));
        DevBuf<unsigned char> tmp(bytes);
        DG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, keys.p, alt.p, items, 0, 64));
    }
    DevBuf<u64> selected(1);
    {
        size_t bytes = 0;
        DG_CUDA(cub::DeviceSelect::Unique(nullptr, bytes, alt.p, keys.p, selected.p, items));
        DevBuf<unsigned char> tmp(bytes);
        DG_CUDA(cub::DeviceSelect::Unique(tmp.p, bytes, alt.p, keys.p, selected.p, items));
    }
    alt.release();
    u64 unique = 0;
    DG_CUDA(cudaMemcpy(&unique, selected.p, 8, cudaMemcpyDeviceToHost));
    u64 last = 0;
    DG_CUDA(cudaMemcpy(&last, keys.p + (unique - 1), 8, cudaMemcpyDeviceToHost));
    if (last == kLoopKey) // all dropped arcs collapsed into one trailing key
        --unique;
    g.arcs = unique;
    g.targets.alloc(unique);
    if (unique)
        low_words_kernel<<<grid_for(unique), 256>>>(keys.p, unique, g.targets.p);
    row_offsets_kernel<<<grid_for(n + 1), 256>>>(keys.p, unique, n, g.offsets.p);
    DG_CUDA(cudaGetLastError());
    DG_CUDA(cudaDeviceSynchronize());
    keys.release();
    return g;
}

// ---- connected components: hook the larger root under the smaller, then compress; the root of a
// ---- component ends up being its smallest vertex id
__global__ void __launch_bounds__(256) cc_init_kernel(u32 *comp, u64 n) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x)
        comp[v] = static_cast<u32>(v);
}

__global__ void __launch_bounds__(256) cc_hook_kernel(const u64 *offsets, const u32 *targets, u32 *comp, u64 n, u32 *changed) {
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const u64 warp = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5;
    const u32 lane = threadIdx.x & 31;
    bool any = false;
    for (u64 u = warp; u < n; u += warps) {
        const u64 beg = offsets[u], end = offsets[u + 1];
        for (u64 k = beg + lane; k < end; k += 32) {
            const u32 v = targets[k];
            if (v > u)
                continue; // every edge is seen from its larger endpoint
            u32 a = comp[u], b = comp[v];
            // find the current roots (paths are short after every compress)
            while (a != comp[a])
                a = comp[a];
            while (b != comp[b])
                b = comp[b];
            while (a != b) {
                const u32 hi = a > b ? a : b, lo = a > b ? b : a;
                const u32 old = atomicMin(comp + hi, lo);
                any = true;
                if (old == hi) // hooked a root
                    break;
                // somebody else hooked `hi` meanwhile: continue from its new parent
                a = old < lo ? old : lo;
                b = old < lo ? lo : old;
                while (a != comp[a])
                    a = comp[a];
                while (b != comp[b])
                    b = comp[b];
            }
        }
    }
    if (any)
        *changed = 1;
}

__global__ void __launch_bounds__(256) cc_compress_kernel(u32 *comp, u64 n) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        u32 r = comp[v];
        while (r != comp[r])
            r = comp[r];
        comp[v] = r;
    }
}

__global__ void __launch_bounds__(256) cc_sizes_kernel(const u32 *comp, const u64 *orig, u64 n, u32 *size,
                                                       unsigned long long *min_orig) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 c = comp[v];
        atomicAdd(size + c, 1u);
        atomicMin(min_orig + c, static_cast<unsigned long long>(orig ? orig[v] : v));
    }
}

// best root: largest size, then smallest minimum original id.  Two keyed atomic passes.
__global__ void __launch_bounds__(256) cc_best_size_kernel(const u32 *comp, const u32 *size, u64 n, u32 *best_size) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x)
        if (comp[v] == v)
            atomicMax(best_size, size[v]);
}
__global__ void __launch_bounds__(256) cc_best_root_kernel(const u32 *comp, const u32 *size, const unsigned long long *min_orig,
                                                           u64 n, const u32 *best_size, unsigned long long *best_key) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x)
        if (comp[v] == v && size[v] == *best_size)
            atomicMin(best_key, min_orig[v]); // minimum original ids of distinct components differ
}
__global__ void __launch_bounds__(256) cc_keep_kernel(const u32 *comp, const unsigned long long *min_orig, u64 n,
                                                      const unsigned long long *best_key, const u32 *size,
                                                      const u32 *best_size, u32 *keep) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x) {
        const u32 c = comp[v];
        keep[v] = (size[c] == *best_size && min_orig[c] == *best_key) ? 1u : 0u;
    }
}

__global__ void __launch_bounds__(256) lcc_degrees_kernel(const u64 *offsets, const u32 *keep, const u32 *dense, const u64 *orig,
                                                          u64 n, u64 *new_offsets, u64 *new_orig) {
    for (u64 v = blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x; v < n;
         v += static_cast<u64>(gridDim.x) * blockDim.x)
        if (keep[v]) {
            new_offsets[dense[v]] = offsets[v + 1] - offsets[v];
            new_orig[dense[v]] = orig ? orig[v] : v;
        }
}

// one warp per kept vertex copies and renames its row (the renaming is monotone: rows stay ascending)
__global__ void __launch_bounds__(256) lcc_rows_kernel(const u64 *offsets, const u32 *targets, const u32 *keep, const u32 *dense,
                                                       u64 n, const u64 *new_offsets, u32 *new_targets) {
    const u64 warps = (static_cast<u64>(gridDim.x) * blockDim.x) >> 5;
    const u64 warp = (blockIdx.x * static_cast<u64>(blockDim.x) + threadIdx.x) >> 5;
    const u32 lane = threadIdx.x & 31;
    for (u64 v = warp; v < n; v += warps) {
        if (!keep[v])
            continue;
        const u64 beg = offsets[v], end = offsets[v + 1], out = new_offsets[dense[v]];
        for (u64 k = lane; k < end - beg; k += 32)
            new_targets[out + k] = dense[targets[beg + k]];
    }
}

struct DeviceLcc {
    DeviceCsr g;
    DevBuf<u64> original_ids;
};

DeviceLcc lcc_on_device(const DeviceCsr &in, const u64 *d_orig) {
    const u64 n = in.n;
    DeviceLcc out;
    if (n == 0)
        return out;
    DevBuf<u32> comp(n), flag(1);
    cc_init_kernel<<<grid_for(n), 256>>>(comp.p, n);
    for (int round = 0; round < 64; ++round) { // one round suffices unless hooks raced; bounded for safety
        DG_CUDA(cudaMemset(flag.p, 0, 4));
        cc_hook_kernel<<<grid_for(n * 32), 256>>>(in.offsets.p, in.targets.p, comp.p, n, flag.p);
        cc_compress_kernel<<<grid_for(n), 256>>>(comp.p, n);
        u32 changed = 0;
        DG_CUDA(cudaMemcpy(&changed, flag.p, 4, cudaMemcpyDeviceToHost));
        if (!changed)
            break;
    }
    DevBuf<u32> size(n), best_size(1), keep(n), dense(n + 1);
    DevBuf<unsigned long long> min_orig(n), best_key(1);
    DG_CUDA(cudaMemset(size.p, 0, n * 4));
    DG_CUDA(cudaMemset(min_orig.p, 0xff, n * 8));
    DG_CUDA(cudaMemset(best_size.p, 0, 4));
    DG_CUDA(cudaMemset(best_key.p, 0xff, 8));
    cc_sizes_kernel<<<grid_for(n), 256>>>(comp.p, d_orig, n, size.p, min_orig.p);
    cc_best_size_kernel<<<grid_for(n), 256>>>(comp.p, size.p, n, best_size.p);
    cc_best_root_kernel<<<grid_for(n), 256>>>(comp.p, size.p, min_orig.p, n, best_size.p, best_key.p);
    cc_keep_kernel<<<grid_for(n), 256>>>(comp.p, min_orig.p, n, best_key.p, size.p, best_size.p, keep.p);
    DG_CUDA(cudaGetLastError());
    {
        size_t bytes = 0;
        DG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, keep.p, dense.p, static_cast<::cuda::std::int64_t>(n)));
        DevBuf<unsigned char> tmp(bytes);
        DG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, keep.p, dense.p, static_cast<::cuda::std::int64_t>(n)));
    }
    u32 kept = 0;
    DG_CUDA(cudaMemcpy(&kept, best_size.p, 4, cudaMemcpyDeviceToHost));
    out.g.n = kept;
    out.g.offsets.alloc(static_cast<u64>(kept) + 1);
    out.original_ids.alloc(kept);
    DG_CUDA(cudaMemset(out.g.offsets.p, 0, (static_cast<u64>(kept) + 1) * 8));
    lcc_degrees_kernel<<<grid_for(n), 256>>>(in.offsets.p, keep.p, dense.p, d_orig, n, out.g.offsets.p, out.original_ids.p);
    {
        size_t bytes = 0;
        const ::cuda::std::int64_t items = static_cast<::cuda::std::int64_t>(kept) + 1;
        DG_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, out.g.offsets.p, out.g.offsets.p, items));
        DevBuf<unsigned char> tmp(bytes);
        DG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, out.g.offsets.p, out.g.offsets.p, items));
    }
    u64 arcs = 0;
    DG_CUDA(cudaMemcpy(&arcs, out.g.offsets.p + kept, 8, cudaMemcpyDeviceToHost));
    out.g.arcs = arcs;
    out.g.targets.alloc(arcs);
    lcc_rows_kernel<<<grid_for(n * 32), 256>>>(in.offsets.p, in.targets.p, keep.p, dense.p, n, out.g.offsets.p, out.g.targets.p);
    DG_CUDA(cudaGetLastError());
    DG_CUDA(cudaDeviceSynchronize());
    return out;
}

HostGraph download(const DeviceCsr &g, const u64 *d_orig) {
    HostGraph h;
    h.n = g.n;
    h.m = g.arcs / 2;
    h.offsets.resize(g.n + 1);
    h.targets.resize(g.arcs);
    h.original_ids.resize(g.n);
    DG_CUDA(cudaMemcpy(h.offsets.data(), g.offsets.p, (g.n + 1) * 8, cudaMemcpyDeviceToHost));
    if (g.arcs)
        DG_CUDA(cudaMemcpy(h.targets.data(), g.targets.p, g.arcs * 4, cudaMemcpyDeviceToHost));
    if (d_orig) {
        if (g.n)
            DG_CUDA(cudaMemcpy(h.original_ids.data(), d_orig, g.n * 8, cudaMemcpyDeviceToHost));
    } else {
        for (u64 v = 0; v < g.n; ++v)
            h.original_ids[v] = v;
    }
    return h;
}

HostGraph finish(DeviceCsr &g, bool take_lcc) {
    if (!take_lcc)
        return download(g, nullptr);
    DeviceLcc l = lcc_on_device(g, nullptr);
    g.offsets.release();
    g.targets.release();
    return download(l.g, l.original_ids.p);
}

} // namespace

HostGraph device_gen_rmat(int scale, int edge_factor, double a, double b, double c, double d, std::uint64_t seed,
                          bool take_lcc, int device) {
    if (scale < 1 || scale > 30)
        throw ConfigError("gen_rmat: scale must be in [1, 30]");
    if (edge_factor < 1)
        throw ConfigError("gen_rmat: edge_factor must be positive");
    if (a < 0 || b < 0 || c < 0 || d < 0 || std::abs(a + b + c + d - 1.0) > 1e-9)
        throw ConfigError("gen_rmat: quadrant probabilities must be nonnegative and sum to 1");
    select_device(device);
    const u64 n = u64{1} << scale;
    const u64 samples = static_cast<u64>(edge_factor) * n;
    DevBuf<u64> keys(samples * 2);
    rmat_keys_kernel<<<grid_for(samples), 256>>>(keys.p, samples, scale, a, a + b, a + b + c, seed);
    DG_CUDA(cudaGetLastError());
    DeviceCsr g = csr_from_keys(n, keys, samples * 2);
    return finish(g, take_lcc);
}

HostGraph device_graph_from_edges(std::uint64_t n, const std::uint64_t *src, const std::uint64_t *dst,
                                  std::uint64_t count, bool take_lcc, int device) {
    if (n > (u64{1} << 32))
        throw ConfigError("graph: more than 2^32 vertices are not supported (32-bit vertex ids)");
    select_device(device);
    DevBuf<u64> keys(count * 2);
    {
        DevBuf<u64> d_src(count), d_dst(count);
        DevBuf<u32> bad(1);
        DG_CUDA(cudaMemset(bad.p, 0, 4));
        if (count) {
            DG_CUDA(cudaMemcpy(d_src.p, src, count * 8, cudaMemcpyHostToDevice));
            DG_CUDA(cudaMemcpy(d_dst.p, dst, count * 8, cudaMemcpyHostToDevice));
            edge_keys_kernel<<<grid_for(count), 256>>>(d_src.p, d_dst.p, count, n, keys.p, bad.p);
            DG_CUDA(cudaGetLastError());
        }
        u32 any_bad = 0;
        DG_CUDA(cudaMemcpy(&any_bad, bad.p, 4, cudaMemcpyDeviceToHost));
        require(any_bad == 0, "from_edges: endpoint out of range");
    }
    DeviceCsr g = csr_from_keys(n, keys, count * 2);
    return finish(g, take_lcc);
}

HostGraph device_graph_lcc(const HostGraph &h, int device) {
    select_device(device);
    DeviceCsr g;
    g.n = h.n;
    g.arcs = h.targets.size();
    g.offsets.alloc(h.n + 1);
    g.targets.alloc(g.arcs);
    DevBuf<u64> orig(h.n);
    DG_CUDA(cudaMemcpy(g.offsets.p, h.offsets.data(), (h.n + 1) * 8, cudaMemcpyHostToDevice));
    if (g.arcs)
        DG_CUDA(cudaMemcpy(g.targets.p, h.targets.data(), g.arcs * 4, cudaMemcpyHostToDevice));
    if (h.n)
        DG_CUDA(cudaMemcpy(orig.p, h.original_ids.data(), h.n * 8, cudaMemcpyHostToDevice));
    if (h.n == 0)
        return HostGraph{};
    DeviceLcc l = lcc_on_device(g, orig.p);
    return download(l.g, l.original_ids.p);
}

} // namespace ebc
