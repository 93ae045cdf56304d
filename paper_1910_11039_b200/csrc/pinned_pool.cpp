// Page-locked host memory for the graph arrays (see host_common.hpp, DefaultInitAllocator).
//
// cudaHostAlloc costs about a millisecond per 10 MB and cudaFreeHost can block for 10^2 ms, so blocks are
// kept per process, keyed by size, and handed to the next graph of the same shape; at most
// kMaxIdleBytes stay cached.  Without a CUDA device every request returns nullptr (the heap is used).
#include <cuda_runtime.h>

#include <cstddef>
#include <map>
#include <mutex>

#include "host_common.hpp"

namespace ebc {
namespace {

constexpr std::size_t kMaxIdleBytes = std::size_t{24} << 30;

struct PinnedPool {
    std::mutex mu;
    std::map<void *, std::size_t> live;
    std::multimap<std::size_t, void *> idle;
    std::size_t idle_bytes = 0;
    int usable = -1; // -1 unknown, 0 no device, 1 yes
};

PinnedPool &pinned() {
    static PinnedPool *p = new PinnedPool; // leaked on purpose: graphs may outlive static destruction
    return *p;
}

} // namespace

void *pinned_alloc(std::size_t bytes) {
    PinnedPool &pp = pinned();
    {
        std::lock_guard<std::mutex> lk(pp.mu);
        if (pp.usable == 0)
            return nullptr;
        auto it = pp.idle.find(bytes);
        if (it != pp.idle.end()) {
            void *p = it->second;
            pp.idle.erase(it);
            pp.idle_bytes -= bytes;
            pp.live[p] = bytes;
            return p;
        }
        if (pp.usable < 0) {
            int count = 0;
            pp.usable = cudaGetDeviceCount(&count) == cudaSuccess && count > 0 ? 1 : 0;
            cudaGetLastError();
            if (pp.usable == 0)
                return nullptr;
        }
    }
    void *p = nullptr;
    if (cudaHostAlloc(&p, bytes, cudaHostAllocDefault) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(pp.mu);
    pp.live[p] = bytes;
    return p;
}

bool pinned_free(void *p) {
    PinnedPool &pp = pinned();
    std::size_t bytes = 0;
    {
        std::lock_guard<std::mutex> lk(pp.mu);
        auto it = pp.live.find(p);
        if (it == pp.live.end())
            return false;
        bytes = it->second;
        pp.live.erase(it);
        if (pp.idle_bytes + bytes <= kMaxIdleBytes) {
            pp.idle.emplace(bytes, p);
            pp.idle_bytes += bytes;
            return true;
        }
    }
    cudaFreeHost(p);
    return true;
}

void pinned_release_idle() {
    PinnedPool &pp = pinned();
    std::lock_guard<std::mutex> lk(pp.mu);
    for (auto &kv : pp.idle)
        cudaFreeHost(kv.second);
    pp.idle.clear();
    pp.idle_bytes = 0;
}

} // namespace ebc
