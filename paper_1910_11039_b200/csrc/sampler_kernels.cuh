// Batched KADABRA sampling kernel for sm_100a.
//
// One CTA = one sample at a time (persistent CTAs pull sample indices from a
// ticket counter).  A sample is: draw (s,t) -> balanced bidirectional BFS with
// sigma counting -> sigma-weighted meet vertex -> sigma-weighted walks to both
// endpoints -> counter increments.  Results are bit-identical to the
// reference's sample_pair + sample_shortest_path + apply_sample
//   /root/reference/proj/src/sampler.cpp:45-52, 54-164
//   /root/reference/proj/include/epochbc/sampler.hpp:74-78
// under the shared Philox stream (philox.cuh).
//
// How order-dependent reference semantics survive a parallel expansion
// (hard part 1): the reference picks the meet vertex by a
// prefix walk over the new frontier in DISCOVERY order (sampler.cpp:111-113,
// 126-133), and discovery order is (position of first parent in the frontier,
// index in that parent's sorted row).  Here a level's adjacency slots are
// enumerated in exactly that order and processed in tiles of BLOCK*ITEMS slots.
//   * A tile that lies inside ONE row cannot contain duplicate targets (rows
//     are strictly ascending), so every unvisited target is a winner at once.
//   * In a tile spanning several rows every unvisited target is claimed with
//     atomicMax(label, TOP - slot): the LOWEST slot wins.
// Winners are ranked by an ordered ballot/popc block scan and receive
// idx = cnt + rank.  Earlier tiles are final before later tiles start, hence
// idx == the reference's position in `next` (sampler.cpp:92-95).  Sigma sums,
// pending edge counts and counters are order independent.
//
// This file is included TWICE by sample_launch.cu (no include guard): once with EBC_STATS 1 -> namespace
// ebc::with_stats, the kernels that maintain the work counters, sample records, paths and state-dump bookkeeping;
// once with EBC_STATS 0 -> namespace ebc::lean, the same kernels without any of it (EBC_STAT(...) expands to
// nothing).  A warp runs through some 3000 instructions once per sample, sixteen to thirty-two CTAs per SM each at a
// different place of them, and instruction fetch is the largest stall of the hub kernels
// (profiles/r02_instruction_supply.txt): the statistics cost config 2 a tenth of its rate.
#include <cstddef>
#include <type_traits>
#include <cuda_runtime.h>

#include "device_types.cuh"
#include "philox.cuh"

#if EBC_STATS
#define EBC_VARIANT with_stats
#define EBC_STAT(...) { __VA_ARGS__ }
#else
#define EBC_VARIANT lean
#define EBC_STAT(...) {}
#endif

namespace ebc {
namespace EBC_VARIANT {

using u128 = unsigned __int128;

// Zeroes the 32-byte sector at `p` (32-byte aligned) with one 256-bit store: a whole-sector write needs
// no fill read from DRAM, unlike an 8-byte one.
__device__ __forceinline__ void st_zero_sector(u64 *p) {
#ifdef EBC_CLEAR_8B
    __stcg(reinterpret_cast<unsigned long long *>(p), 0ull);
    __stcg(reinterpret_cast<unsigned long long *>(p) + 1, 0ull);
    __stcg(reinterpret_cast<unsigned long long *>(p) + 2, 0ull);
    __stcg(reinterpret_cast<unsigned long long *>(p) + 3, 0ull);
#else
    const unsigned long long z = 0;
    asm volatile("st.global.cg.v4.u64 [%0], {%1, %1, %1, %1};" ::"l"(p), "l"(z) : "memory");
#endif
}
__device__ __forceinline__ u32 ld_cg(const u32 *p) { return __ldcg(p); }
__device__ __forceinline__ u64 ld_cg(const u64 *p) { return __ldcg(reinterpret_cast<const unsigned long long *>(p)); }
__device__ __forceinline__ void st_cg(u32 *p, u32 v) { __stcg(p, v); }
__device__ __forceinline__ void st_cg(u64 *p, u64 v) { __stcg(reinterpret_cast<unsigned long long *>(p), v); }

// Atomics on the slot arrays, spelled as .global PTX.  The slot pointers are read back from shared
// memory, so the compiler only knows them as generic addresses, and a generic 64-bit atomicAdd expands
// to a run-time address-space test plus a shared-memory CAS loop next to the real instruction (21
// instructions per call site, 16 call sites in the 4-item kernel).  None of the results is needed
// except the old value of the saturating add, so the rest are fire-and-forget reductions.
__device__ __forceinline__ void red_add_u64(u64 *p, u64 v) {
    asm volatile("red.global.add.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}
__device__ __forceinline__ u64 atom_add_u64(u64 *p, u64 v) {
    u64 old;
    asm volatile("atom.global.add.u64 %0, [%1], %2;" : "=l"(old) : "l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_max_u64(u64 *p, u64 v) {
    asm volatile("red.global.max.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}
__device__ __forceinline__ u64 atom_min_u64(u64 *p, u64 v) {
    u64 old;
    asm volatile("atom.global.min.u64 %0, [%1], %2;" : "=l"(old) : "l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
    return old;
}
__device__ __forceinline__ void red_min_u64(u64 *p, u64 v) {
    asm volatile("red.global.min.u64 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "l"(v) : "memory");
}
__device__ __forceinline__ void red_max_u32(u32 *p, u32 v) {
    asm volatile("red.global.max.u32 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void red_or_u32(u32 *p, u32 v) {
    asm volatile("red.global.or.b32 [%0], %1;" ::"l"(__cvta_generic_to_global(p)), "r"(v) : "memory");
}

// Shared-memory accesses by shared-window address (see expand_level_ell).
__device__ __forceinline__ u32 smem_addr(const void *p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ u32 lds_u32(u32 a) {
    u32 v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts_u32(u32 a, u32 v) { asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ u32 atoms_cas_u32(u32 a, u32 cmp, u32 v) {
    u32 old;
    asm volatile("atom.shared.cas.b32 %0, [%1], %2, %3;" : "=r"(old) : "r"(a), "r"(cmp), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ void reds_min_u32(u32 a, u32 v) { asm volatile("red.shared.min.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }
__device__ __forceinline__ void reds_or_u32(u32 a, u32 v) { asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory"); }

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31u; }
__device__ __forceinline__ u32 lanemask_lt() {
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// External (caller-visible) id of a dense vertex id (see SamplerParams::to_ext).
__device__ __forceinline__ u32 ext_id(const SamplerParams &p, u32 v) { return p.to_ext ? __ldg(p.to_ext + v) : v; }

// sigma[idx] = sat_add_u64(sigma[idx], add)  (sampler.cpp:11-13,98) with atomics:
// a wrapped add is always followed by the same thread's atomicMax(.., 2^64-1),
// so the value after the level barrier is 2^64-1 iff the true sum overflowed.
// `small`: the sum of sigma over the whole frontier fits 64 bits (see sum_frontier_degrees), so no
// sum can wrap and the add needs no return value (a fire-and-forget reduction).
__device__ __forceinline__ void sat_atomic_add(u64 *p, u64 add, bool small) {
    if (small) {
        red_add_u64(p, add);
        return;
    }
    const u64 old = atom_add_u64(p, add);
    if (old + add < old)
        red_max_u64(p, ~0ull);
}

// uniform_below_u128 (sampler.cpp:21-30).  Executed redundantly by every thread
// of the CTA (the stream state is uniform), so no broadcast is needed.
// a % b for b >= 2^64 by restoring division, one bit per iteration.  Only the wide rejection sampler
// below uses it (total weights >= 2^64); the compiler's inline 128-bit division is ~100 instructions
// per use, and the kernel's instruction footprint is what it is short of (profiles/r01_icache.txt).
static __device__ __noinline__ u128 umod128_compact(u128 a, u128 b) {
    u128 r = 0;
#pragma unroll 1
    for (int i = 127; i >= 0; --i) {
        const bool top = static_cast<u64>(r >> 127) != 0;
        r = (r << 1) | ((a >> i) & 1);
        if (top || r >= b)
            r -= b;
    }
    return r;
}
static __device__ __noinline__ u128 uniform_below_wide(SampleStream &rng, u128 bound) {
    const u128 all = ~static_cast<u128>(0);
    const u128 reject_from = all - umod128_compact(all, bound);
    for (;;) {
        const u128 hi = rng.next_u64();
        const u128 lo = rng.next_u64();
        const u128 r = (hi << 64) | lo;
        if (r < reject_from)
            return umod128_compact(r, bound);
    }
}
__device__ __forceinline__ u128 uniform_below_u128(SampleStream &rng, u128 bound) {
    if (static_cast<u64>(bound >> 64) == 0)
        return rng.next_below(static_cast<u64>(bound));
    return uniform_below_wide(rng, bound);
}

// The slot's array addresses live in shared memory (BlockShared::sp), not in registers: the kernel
// is compiled for 64 registers and every pointer kept live across a sample is a spill elsewhere.
struct SidePtrs {
    u32 *list;
    u64 *sig;
    u32 *lvl;
    u32 *pm; // fixed-stride rows: parent masks, one byte per settled vertex (SamplerParams::pm)
};

constexpr int kPredCache = 32;

// Final-level probe (see probe_level): a level with at least SamplerParams::probe_min_slots adjacency
// slots (256 with visited bitmaps, else 512; set by the host) is first scanned read-only; if it touches
// the other side, the meet vertex is chosen from the contact edges and the level is never settled: up to
// 32 edges in registers (pick_meet_warp), up to FinalEdgeCap<BLOCK>::value in shared memory (meet_from_edges),
// more -- as many as the slot's contact buffer holds -- in the slot's global arrays (pick_meet_large).
#ifndef EBC_EDGE_CAP_MAX
#define EBC_EDGE_CAP_MAX 512
#endif
template <int BLOCK> struct FinalEdgeCap {
    static constexpr int value = 4 * BLOCK < EBC_EDGE_CAP_MAX ? 4 * BLOCK : EBC_EDGE_CAP_MAX;
};

template <int BLOCK, int ITEMS> struct BlockShared {
    static constexpr int WARPS = BLOCK / 32;
    u64 f_key[FinalEdgeCap<BLOCK>::value]; // contact edges of a probed final level: discovery key,
    u64 f_s[FinalEdgeCap<BLOCK>::value];   //   sigma of the parent,
    u32 f_v[FinalEdgeCap<BLOCK>::value];   //   target vertex,
    u32 f_o[FinalEdgeCap<BLOCK>::value];   //   its idx on the other side
    // (f_key .. c_sig are contiguous: expand_level_ell keeps its tables there)
    u64 c_beg[BLOCK];      // row start of each frontier-chunk vertex
    u64 c_scan[BLOCK + 1]; // exclusive prefix of the chunk's degrees
    u64 c_sig[BLOCK];      // sigma of each chunk vertex
    u32 edge_cnt;
    SidePtrs sp[2];
    u64 prev_pending[2]; // per side: pending edges of the level expanded last (0 before the first)
    u32 sigma_small[2]; // per side: the frontier's sigma values sum to < 2^63 (no add of the next level can wrap)
    u32 last[6]; // base / cnt / depth of both sides of the last finished sample (state dumps)
    u32 *lab, *bits, *contact, *meetbuf; // the slot's label / bitmap / contact arrays
    SampleRecordDev rec; // record of the sample in flight (thread 0)
    u64 red64[WARPS * 3];  // block reductions
    u32 warp_cnt[ITEMS * WARPS];
    u32 warp_cnt2[ITEMS * WARPS];
    unsigned long long ticket;
    u32 min_contact;       // min other-side idx over contact vertices of this level
    u32 found_lane;        // ordered-search result
    u32 pred_cnt;
    u32 pred_pos[kPredCache];
    u64 pred_sig[kPredCache];
    u32 pred_vtx[kPredCache];
    u32 bcast[4];
    u64 ws[kWorkCounters]; // work counters of the sample in flight (thread 0)
    u64 wk[kWorkCounters]; // committed work counters of this CTA
};

// Ordered ranks for ITEMS flags per thread, slot order = (item, warp, lane).
// rank[k] = number of set flags before slot (k, tid); returns the total.
// One __syncthreads; `cnt` (ITEMS*WARPS words) must not be reused before the next barrier.
template <int BLOCK, int ITEMS>
__device__ __forceinline__ u32 block_ranks(const bool (&flag)[ITEMS], u32 (&rank)[ITEMS], u32 *cnt) {
    constexpr int WARPS = BLOCK / 32;
    const u32 warp = threadIdx.x >> 5;
    u32 in_warp[ITEMS];
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
        const u32 ballot = __ballot_sync(0xffffffffu, flag[k]);
        in_warp[k] = __popc(ballot & lanemask_lt());
        if (lane_id() == 0)
            cnt[k * WARPS + warp] = __popc(ballot);
    }
    __syncthreads();
    if (ITEMS * WARPS <= 32) {
        // every warp scans the ITEMS * WARPS counts with shuffles (far fewer instructions than the
        // unrolled ITEMS x WARPS walk; this code is instantiated in every tile loop)
        const u32 mine = lane_id() < static_cast<u32>(ITEMS * WARPS) ? cnt[lane_id()] : 0u;
        u32 incl = mine;
#pragma unroll
        for (int o = 1; o < ITEMS * WARPS; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane_id() >= static_cast<u32>(o))
                incl += t;
        }
        const u32 excl = incl - mine;
#pragma unroll
        for (int k = 0; k < ITEMS; ++k)
            rank[k] = __shfl_sync(0xffffffffu, excl, k * WARPS + static_cast<int>(warp)) + in_warp[k];
        return __shfl_sync(0xffffffffu, incl, ITEMS * WARPS - 1);
    }
    u32 running = 0;
#pragma unroll
    for (int k = 0; k < ITEMS; ++k) {
#pragma unroll
        for (int w = 0; w < WARPS; ++w) {
            if (static_cast<u32>(w) == warp)
                rank[k] = running + in_warp[k];
            running += cnt[k * WARPS + w];
        }
    }
    return running;
}

template <int BLOCK> __device__ __forceinline__ u64 block_sum_u64(u64 v, u64 *red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
        v += __shfl_xor_sync(0xffffffffu, v, o);
    if (BLOCK == 32)
        return v;
    __syncthreads();
    if (lane_id() == 0)
        red[threadIdx.x >> 5] = v;
    __syncthreads();
    u64 s = 0;
#pragma unroll
    for (int w = 0; w < BLOCK / 32; ++w)
        s += red[w];
    return s;
}

// 192-bit sum (lo, hi, carry-out count) of per-thread 128-bit values.
template <int BLOCK>
__device__ __noinline__ void block_sum_u128(u128 v, u64 &lo, u64 &hi, u64 &ovf, u64 *red) {
    u64 a = static_cast<u64>(v), b = static_cast<u64>(v >> 64), c = 0;
#pragma unroll 1 // (called a few times per sample: compact beats fast)
    for (int o = 16; o > 0; o >>= 1) {
        const u64 a2 = __shfl_xor_sync(0xffffffffu, a, o);
        const u64 b2 = __shfl_xor_sync(0xffffffffu, b, o);
        const u64 c2 = __shfl_xor_sync(0xffffffffu, c, o);
        const u128 x = (static_cast<u128>(b) << 64) | a, y = (static_cast<u128>(b2) << 64) | a2;
        const u128 s = x + y;
        c += c2 + (s < x ? 1 : 0);
        a = static_cast<u64>(s);
        b = static_cast<u64>(s >> 64);
    }
    if (BLOCK > 32) {
        __syncthreads();
        if (lane_id() == 0) {
            red[(threadIdx.x >> 5) * 3 + 0] = a;
            red[(threadIdx.x >> 5) * 3 + 1] = b;
            red[(threadIdx.x >> 5) * 3 + 2] = c;
        }
        __syncthreads();
        u128 s = 0;
        c = 0;
#pragma unroll 1
        for (int w = 0; w < BLOCK / 32; ++w) {
            const u128 y = (static_cast<u128>(red[w * 3 + 1]) << 64) | red[w * 3 + 0];
            const u128 t = s + y;
            c += red[w * 3 + 2] + (t < s ? 1 : 0);
            s = t;
        }
        a = static_cast<u64>(s);
        b = static_cast<u64>(s >> 64);
        __syncthreads();
    }
    lo = a;
    hi = b;
    ovf = c;
}

// Ordered search: first thread (in thread order) whose inclusive 128-bit prefix
// of `w`, added to `running`, exceeds `pick`.  Returns the thread index or BLOCK
// if none; `running` is advanced by the block total when nothing is found.
// Values that overflow 128 bits compare as "exceeds".
template <int BLOCK>
__device__ __noinline__ u32 block_first_exceeding(u128 w, u128 &running, bool &running_ovf, u128 pick,
                                                  u64 *red64, u32 *found_lane) {
    u64 a = static_cast<u64>(w), b = static_cast<u64>(w >> 64);
    u32 of = 0;
#pragma unroll 1
    for (int o = 1; o < 32; o <<= 1) {
        const u64 a2 = __shfl_up_sync(0xffffffffu, a, o);
        const u64 b2 = __shfl_up_sync(0xffffffffu, b, o);
        const u32 of2 = __shfl_up_sync(0xffffffffu, of, o);
        if (lane_id() >= static_cast<u32>(o)) {
            const u128 x = (static_cast<u128>(b) << 64) | a, y = (static_cast<u128>(b2) << 64) | a2;
            const u128 s = x + y;
            of |= of2 | (s < x ? 1u : 0u);
            a = static_cast<u64>(s);
            b = static_cast<u64>(s >> 64);
        }
    }
    u128 incl = (static_cast<u128>(b) << 64) | a;
    bool incl_of = of != 0;
    const u32 warp = threadIdx.x >> 5;
    if (BLOCK > 32) {
        __syncthreads();
        if (lane_id() == 31) {
            red64[warp * 3 + 0] = a;
            red64[warp * 3 + 1] = b;
            red64[warp * 3 + 2] = of;
        }
        __syncthreads();
        u128 before = 0;
        bool before_of = false;
#pragma unroll 1
        for (u32 k = 0; k < warp; ++k) {
            const u128 y = (static_cast<u128>(red64[k * 3 + 1]) << 64) | red64[k * 3 + 0];
            const u128 t = before + y;
            before_of = before_of || red64[k * 3 + 2] != 0 || t < before;
            before = t;
        }
        const u128 t = incl + before;
        incl_of = incl_of || before_of || t < incl;
        incl = t;
    }
    const u128 tot = incl + running;
    const bool tot_of = incl_of || running_ovf || tot < incl;
    const bool hit = (w != 0) && (tot_of || tot > pick);
    const u32 ballot = __ballot_sync(0xffffffffu, hit);
    if (threadIdx.x == 0)
        *found_lane = BLOCK;
    __syncthreads();
    if (ballot != 0 && lane_id() == 0)
        atomicMin(found_lane, (warp << 5) + (__ffs(ballot) - 1));
    if (threadIdx.x == BLOCK - 1) {
        red64[0] = static_cast<u64>(tot);
        red64[1] = static_cast<u64>(tot >> 64);
        red64[2] = tot_of ? 1 : 0;
    }
    __syncthreads();
    const u32 found = *found_lane;
    if (found == BLOCK) {
        running = (static_cast<u128>(red64[1]) << 64) | red64[0];
        running_ovf = red64[2] != 0;
    }
    __syncthreads();
    return found;
}

// One 4-byte label per vertex serves BOTH sides: lab[v] = base + 2 * idx + side, where idx is the
// vertex' position in that side's settle list.  That is enough because, until the search ends, a vertex
// is settled by at most one side: the first level that touches the other side's settled set is the last
// one (sampler.cpp:105-115).  A contact vertex of that last level is settled on the expanding side like
// any other (its label is overwritten), and its other-side idx -- read from the old label before the
// overwrite -- travels in the contact record; the walks only look at levels below the contact level on
// their own side, whose labels are never overwritten.  One load answers "visited on the expanding side?"
// and "visited on the other side?" (contact test, sampler.cpp:107), and a 32-byte sector covers eight
// vertices.  `base` is the same for both sides and advances by 2 * max(settled counts) per sample.
struct SideRegs {
    const SidePtrs *pp;
    u32 base;  // label base of this sample (same value on both sides)
    u32 cnt;   // settled vertices so far
    u32 fb;    // frontier = list[fb .. cnt)
    u32 depth; // depth of the frontier
    u64 pending;
};

// Per-thread partial work counters of the sample in flight (the thread-0-only
// counters live in BlockShared::ws).
struct WorkRegs {
    u64 e_lvl = 0, p_walk = 0;
};

// idx on side `s` encoded in `label`, or a value >= 2^31 (never below a settled count) if the label belongs to
// the other side, to an earlier sample (label < base wraps) or is a transient claim value.
__device__ __forceinline__ u32 label_idx(u32 label, u32 base, int s) {
    const u32 r = label - base - static_cast<u32>(s);
    return (r & 1u) ? 0xffffffffu : (r >> 1);
}
__device__ __forceinline__ u32 make_label(u32 base, u32 idx, int s) { return base + 2u * idx + static_cast<u32>(s); }

// Visited filter (hub graphs, BITS kernels): an approximate copy of the visited set of BOTH sides together in
// shared memory, one bit per position h = v mod kPositions.  A clear bit means "certainly not visited by either
// side": the probe of a final level, whose targets are overwhelmingly unvisited, then needs no global access
// for that slot at all.  A set bit (a visited vertex, or another one that shares its position) is looked up
// in the global bitmap.  Under the degree-class numbering small ids are the hubs, so the hubs -- the vertices
// most often visited -- have positions of their own.  Set when a vertex is settled, cleared once per sample.
template <int BLOCK> struct VisitedFilter {
    // 64 bytes of filter per thread, at most 16 KB; 1 KB for one-warp CTAs (32 of them share an SM's shared memory)
    static constexpr u32 kPositions = BLOCK <= 32 ? 8192u : 512u * (BLOCK < 256 ? BLOCK : 256);
    static constexpr u32 kWords = kPositions / 32;
};
template <int BLOCK> __device__ __forceinline__ void filter_insert(u32 *vf, u32 v) {
    const u32 h = v & (VisitedFilter<BLOCK>::kPositions - 1);
    atomicOr(vf + (h >> 5), 1u << (h & 31));
}

// 16-byte load of four consecutive adjacency entries (SASS: LDG.E.128 through the read-only path).
__device__ __forceinline__ uint4 ldg_targets4(const u32 *p) { return __ldg(reinterpret_cast<const uint4 *>(p)); }

// Loads the chunk of BLOCK frontier vertices at list positions [c0, c0 + BLOCK) (clipped to fe): row
// start and sigma of each into c_beg / c_sig, the exclusive prefix of their degrees into
// c_scan[0..BLOCK]; returns the chunk's number of adjacency slots.  Starts with a barrier (the previous
// chunk's readers of c_* are done) and ends with one.  Inline in expand_level and probe_level (out of line
// it cost config 4 1.5 % and config 1 3 %: a call per BLOCK frontier vertices).
template <int BLOCK>
__device__ __forceinline__ u64 load_chunk(const SamplerParams &p, const SidePtrs *pp, u32 c0, u32 fe, u64 *c_beg, u64 *c_scan,
                                       u64 *c_sig, u64 *red64) {
    const u32 tid = threadIdx.x;
    const u32 i = c0 + tid;
    u64 beg = 0, deg = 0, su = 0;
    if (i < fe) {
        const u32 u = ld_cg(pp->list + i);
        beg = __ldg(p.offsets + u);
        deg = __ldg(p.offsets + u + 1) - beg;
        su = ld_cg(pp->sig + i);
    }
    u64 inc = deg;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u64 t = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane_id() >= static_cast<u32>(o))
            inc += t;
    }
    __syncthreads();
    if (BLOCK > 32 && lane_id() == 31)
        red64[tid >> 5] = inc;
    c_beg[tid] = beg;
    c_sig[tid] = su;
    if (BLOCK > 32)
        __syncthreads();
    u64 before = 0;
    if (BLOCK > 32)
        for (u32 w = 0; w < (tid >> 5); ++w)
            before += red64[w];
    c_scan[tid + 1] = before + inc;
    if (tid == 0)
        c_scan[0] = 0;
    __syncthreads();
    return c_scan[BLOCK];
}

// Expands the frontier of side `e` by one level (sampler.cpp:86-103) and
// records contacts with the other side (sampler.cpp:105-108).  ex.pending is NOT
// updated here (see sum_frontier_degrees).  Returns false on
// slot-capacity overflow (the sample is then re-run in a large slot).
// contact_n returns the number of contact vertices appended to `contact`.
template <int BLOCK, int ITEMS, bool BITS>
__device__ bool expand_level(const SamplerParams &p, u32 *lab, u32 *bits, u32 *vf, int e, SideRegs &ex, const SideRegs &ot,
                             u32 *contact, u32 &contact_n, BlockShared<BLOCK, ITEMS> &sh, WorkRegs &wk) {
    constexpr int TILE = BLOCK * ITEMS;
    const u32 tid = threadIdx.x;
    const u32 fb = ex.fb, fe = ex.cnt;
    const u32 level_start = fe;
    const u32 next_depth = ex.depth + 1;
    u32 cnt = fe;
    contact_n = 0;
    const bool sigma_small = sh.sigma_small[e] != 0; // uniform; written behind a barrier
    if (static_cast<u64>(next_depth) + 1 > p.aux_cap) // more levels than the slot's level table holds
        return false;
    if (tid == 0) {
        st_cg(ex.pp->lvl + next_depth, level_start);
        sh.min_contact = 0xffffffffu;
        EBC_STAT(sh.ws[kW_V_exp] += fe - fb;)
        EBC_STAT(sh.ws[kW_levels] += 1;)
    }
    for (u32 c0 = fb; c0 < fe; c0 += BLOCK) {
        // ---- load a chunk of BLOCK frontier vertices, scan their degrees ----
        // (the loader's first barrier: the previous chunk's tiles are done with c_*, their label stores visible)
        const u64 T = load_chunk<BLOCK>(p, ex.pp, c0, fe, sh.c_beg, sh.c_scan, sh.c_sig, sh.red64);
        if (tid == 0)
            EBC_STAT(sh.ws[kW_E_bfs] += T;)

        // ---- ordered tiles of TILE adjacency slots ----
        int prev_row = -1;
        int row_lo = 0; // owner of the tile's first slot; non-decreasing over the tiles of a chunk
        for (u64 t0 = 0; t0 < T; t0 += TILE) {
            const u64 t_last = (t0 + TILE < T ? t0 + TILE : T) - 1;
            // owner rows of the first and last slot (uniform): last r with c_scan[r] <= j
            while (sh.c_scan[row_lo + 1] <= t0)
                ++row_lo;
            int row_hi = row_lo;
            {
                int hi = BLOCK;
                while (hi - row_hi > 1) {
                    const int mid = (row_hi + hi) >> 1;
                    if (sh.c_scan[mid] <= t_last)
                        row_hi = mid;
                    else
                        hi = mid;
                }
            }
            u32 v[ITEMS], idx[ITEMS];
            bool win[ITEMS], at_level[ITEMS], is_contact[ITEMS];
            u32 other_idx[ITEMS];
            u32 rank[ITEMS];
            if (row_lo == row_hi) {
                // ================= single-row tile: no duplicate targets possible =================
                if (prev_row != row_lo && prev_row != -1)
                    __syncthreads(); // label stores of the previous row's tiles must be visible
                prev_row = row_lo;
                const u32 *row = p.targets + (sh.c_beg[row_lo] - sh.c_scan[row_lo]);
                const u64 sig_u = sh.c_sig[row_lo];
                bool act[ITEMS];
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    const u64 j = t0 + static_cast<u64>(k) * BLOCK + tid;
                    act[k] = j <= t_last;
                    v[k] = act[k] ? __ldg(row + j) : 0u;
                }
                u32 lbl[ITEMS];
#pragma unroll
                for (int k = 0; k < ITEMS; ++k)
                    lbl[k] = act[k] ? ld_cg(lab + v[k]) : 0u;
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    const u32 rel = label_idx(lbl[k], ex.base, e);
                    const bool visited = rel < cnt;
                    win[k] = act[k] && !visited;
                    at_level[k] = act[k] && visited && rel >= level_start; // dist[v] == next_depth (sampler.cpp:97)
                    idx[k] = rel;
                    other_idx[k] = label_idx(lbl[k], ex.base, 1 - e);
                    is_contact[k] = win[k] && other_idx[k] < ot.cnt; // other.visited(v) (sampler.cpp:107)
                }
                const u32 winners = block_ranks<BLOCK, ITEMS>(win, rank, sh.warp_cnt);
                if (static_cast<u64>(cnt) + winners > p.cap) {
                    ex.cnt = cnt; // nothing of this tile was written; the caller retires labels < cnt
                    return false;
                }
                bool any_contact_local = false;
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    if (win[k]) { // settle (sampler.cpp:93-95) and the discovering edge's sigma (sampler.cpp:98)
                        idx[k] = cnt + rank[k];
                        st_cg(lab + v[k], make_label(ex.base, idx[k], e));
                        st_cg(ex.pp->list + idx[k], v[k]);
                        st_cg(ex.pp->sig + idx[k], sig_u);
                        if (BITS) {
                            red_or_u32(bits + 2 * static_cast<u64>(v[k] >> 5) + e, 1u << (v[k] & 31));
                            filter_insert<BLOCK>(vf, v[k]);
                        }
                        if (is_contact[k]) {
                            atomicMin(&sh.min_contact, other_idx[k]);
                            any_contact_local = true;
                        }
                        EBC_STAT(wk.e_lvl += 1;)
                    } else if (at_level[k]) {
                        sat_atomic_add(ex.pp->sig + idx[k], sig_u, sigma_small);
                        EBC_STAT(wk.e_lvl += 1;)
                    }
                }
                if (__syncthreads_or(any_contact_local ? 1 : 0)) {
                    u32 crank[ITEMS];
                    const u32 ctot = block_ranks<BLOCK, ITEMS>(is_contact, crank, sh.warp_cnt2);
                    if (static_cast<u64>(contact_n) + ctot > p.aux_cap) { // contact list full: re-run in a large slot
                        ex.cnt = cnt + winners;
                        return false;
                    }
#pragma unroll
                    for (int k = 0; k < ITEMS; ++k)
                        if (is_contact[k]) {
                            st_cg(contact + 2 * static_cast<u64>(contact_n + crank[k]), idx[k]);
                            st_cg(contact + 2 * static_cast<u64>(contact_n + crank[k]) + 1, other_idx[k]);
                        }
                    contact_n += ctot;
                }
                cnt += winners;
            } else {
                // ================= tile spanning several rows: claim, lowest slot wins =================
                if (prev_row != -1)
                    __syncthreads();
                prev_row = -2;
                u64 sig_u[ITEMS];
                bool candidate[ITEMS];
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    const u64 j = t0 + static_cast<u64>(k) * BLOCK + tid;
                    const bool act = j <= t_last;
                    v[k] = 0;
                    idx[k] = 0;
                    sig_u[k] = 0;
                    candidate[k] = false;
                    at_level[k] = false;
                    other_idx[k] = 0xffffffffu;
                    if (act) {
                        int lo = row_lo, hi = row_hi + 1; // owner row: last r with c_scan[r] <= j
                        while (hi - lo > 1) {
                            const int mid = (lo + hi) >> 1;
                            if (sh.c_scan[mid] <= j)
                                lo = mid;
                            else
                                hi = mid;
                        }
                        v[k] = __ldg(p.targets + sh.c_beg[lo] + (j - sh.c_scan[lo]));
                        sig_u[k] = sh.c_sig[lo];
                    }
                }
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    const u64 j = t0 + static_cast<u64>(k) * BLOCK + tid;
                    if (j <= t_last) {
                        const u32 lbl = ld_cg(lab + v[k]);
                        const u32 rel = label_idx(lbl, ex.base, e);
                        other_idx[k] = label_idx(lbl, ex.base, 1 - e);
                        if (rel < cnt) {
                            idx[k] = rel;
                            at_level[k] = rel >= level_start;
                        } else {
                            candidate[k] = true;
                        }
                    }
                }
                // Every label of the tile is read before any is claimed: a claim replaces the label, and the
                // winner of a contact vertex needs the other side's idx that was in it.
                __syncthreads();
                // claim: the lowest slot of every distinct unvisited target wins (see the header comment)
#pragma unroll
                for (int k = 0; k < ITEMS; ++k)
                    if (candidate[k])
                        red_max_u32(lab + v[k], kClaimTop - (k * BLOCK + tid));
                __syncthreads(); // claims visible
                // A candidate reads back the claim that won its target: its own (winner) or the winning slot's,
                // through which it later finds the winner's idx in shared memory (no second look at the label).
                static_assert(sizeof(u32) * TILE <= sizeof(sh.f_key) + sizeof(sh.f_s), "tile idx table aliases f_key/f_s");
                u32 *tile_idx = reinterpret_cast<u32 *>(sh.f_key); // (f_key, f_s are only live in the meet phase)
                u32 won_by[ITEMS];
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    won_by[k] = candidate[k] ? kClaimTop - ld_cg(lab + v[k]) : 0u;
                    win[k] = candidate[k] && won_by[k] == static_cast<u32>(k * BLOCK + tid);
                    is_contact[k] = win[k] && other_idx[k] < ot.cnt;
                }
                const u32 winners = block_ranks<BLOCK, ITEMS>(win, rank, sh.warp_cnt);
                const bool overflow = static_cast<u64>(cnt) + winners > p.cap;
                bool any_contact_local = false;
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    if (win[k]) {
                        if (overflow) {
                            st_cg(lab + v[k], 0u); // undo the claim (the sample is abandoned and re-run)
                        } else {
                            idx[k] = cnt + rank[k];
                            tile_idx[k * BLOCK + tid] = idx[k];
                            st_cg(lab + v[k], make_label(ex.base, idx[k], e));
                            st_cg(ex.pp->list + idx[k], v[k]);
                            st_cg(ex.pp->sig + idx[k], static_cast<u64>(0));
                            if (BITS) {
                                red_or_u32(bits + 2 * static_cast<u64>(v[k] >> 5) + e, 1u << (v[k] & 31));
                                filter_insert<BLOCK>(vf, v[k]);
                            }
                            if (is_contact[k]) {
                                atomicMin(&sh.min_contact, other_idx[k]);
                                any_contact_local = true;
                            }
                        }
                    }
                }
                const int any_contact = __syncthreads_or(any_contact_local ? 1 : 0); // finals visible
                if (overflow) {
                    ex.cnt = cnt;
                    return false;
                }
#pragma unroll
                for (int k = 0; k < ITEMS; ++k) {
                    if (candidate[k] && !win[k])
                        idx[k] = tile_idx[won_by[k]]; // the winner's idx
                    if (candidate[k] || at_level[k]) {
                        sat_atomic_add(ex.pp->sig + idx[k], sig_u[k], sigma_small); // sampler.cpp:97-98
                        EBC_STAT(wk.e_lvl += 1;)
                    }
                }
                if (any_contact) {
                    u32 crank[ITEMS];
                    const u32 ctot = block_ranks<BLOCK, ITEMS>(is_contact, crank, sh.warp_cnt2);
                    if (static_cast<u64>(contact_n) + ctot > p.aux_cap) {
                        ex.cnt = cnt + winners;
                        return false;
                    }
#pragma unroll
                    for (int k = 0; k < ITEMS; ++k)
                        if (is_contact[k]) {
                            st_cg(contact + 2 * static_cast<u64>(contact_n + crank[k]), idx[k]);
                            st_cg(contact + 2 * static_cast<u64>(contact_n + crank[k]) + 1, other_idx[k]);
                        }
                    contact_n += ctot;
                }
                cnt += winners;
            }
        }
    }
    __syncthreads();
    if (tid == 0) {
        EBC_STAT(sh.ws[kW_V_set] += cnt - level_start;)
        EBC_STAT(sh.ws[kW_F_chk] += cnt - level_start;)
    }
    ex.fb = level_start; // sampler.cpp:101-103
    ex.cnt = cnt;
    ex.depth = next_depth;
    return true;
}

// next_pending (sampler.cpp:95,102): the sum of the degrees of the new frontier.
// Only needed when the search continues, so it is evaluated after the level,
// not per settled vertex (the last level of a sample never needs it).
template <int BLOCK>
__device__ __forceinline__ u64 sum_frontier_degrees(const SamplerParams &p, const SideRegs &sd, u64 *red,
                                                    u32 *sigma_small) {
    u64 s = 0, g = 0;
    for (u32 i = sd.fb + threadIdx.x; i < sd.cnt; i += BLOCK) {
        const u32 v = ld_cg(sd.pp->list + i);
        s += __ldg(p.offsets + v + 1) - __ldg(p.offsets + v);
        const u64 sg = ld_cg(sd.pp->sig + i);
        g = g > ~0ull - sg ? ~0ull : g + sg;
    }
    const u64 r = block_sum_u64<BLOCK>(s, red);
    // The graph is simple, so sigma of a vertex of the next level is a sum over DISTINCT frontier
    // vertices and cannot exceed the frontier's total; every thread's share below 2^63 / BLOCK bounds it.
    const int big = __syncthreads_or(g >= (1ull << 63) / BLOCK ? 1 : 0);
    if (threadIdx.x == 0)
        *sigma_small = big ? 0u : 1u;
    return r;
}

// expand_level for graphs with fixed-stride rows (SamplerParams::ell: maximum degree <= kEllWidth -- grids, road
// networks).  Such searches are long chains of small levels (config 3: 86 levels of ~450 vertices per sample): what
// a level costs is its number of DEPENDENT memory round trips and the instructions issued around them, not its
// bytes.  Per chunk of BLOCK frontier vertices there are three trips: list/sigma of the chunk (coalesced) -> the rows
// (one 32-byte sector each, no offsets look-up) -> the labels of their targets.  Everything else stays on the SM:
//  * thread t owns frontier vertex c0 + t and its (at most eight) entries, key = 8 t + k = discovery order
//    (sampler.cpp:90-95: frontier order, then row order).  Entries are handled in two groups of four, the second
//    only by warps that hold a row of more than four entries.  The chunk's vertex is loaded two chunks ahead and
//    its row one chunk ahead, so only the label trip stays on the critical path;
//  * entries that lead back to the vertices this one was discovered from are skipped (parent mask pm[idx], one
//    bit per row entry): every discoverer of a vertex -- the winner with a byte store, the others with a
//    red.or next to their sigma add -- leaves the position of its arc's reverse in the vertex' row, which every
//    entry carries;
//  * the unvisited targets of the chunk are deduplicated in a shared-memory hash set instead of being claimed in
//    their labels: a candidate inserts its vertex with linear probing (atomicCAS(hv[slot], empty, v) until the
//    slot is empty or already holds v -- slots are never emptied while a chunk inserts, so all candidates of a
//    vertex end in the same slot) and then does atomicMin(hk[slot], key).  After one barrier the candidate whose
//    key is in hk[slot] has won the vertex, the others have lost to that key (first version: lock-step rounds
//    of atomicMin(table[h(v) + round], key) with two barriers per round -- three to five rounds per chunk,
//    as many as the longest probe sequence);
//  * winners are ranked by a scan over the threads (keys ascend with the thread index, then k), settle their
//    vertex (label, list, sigma = sigma[u]: sampler.cpp:93-98) and publish idx in kv[key]; the other discoverers
//    keep their winner's key in kv[own key] and add their sigma[u] after the barrier (sampler.cpp:97-98).  A
//    chunk costs three barriers;
//  * the degree of a settled vertex travels in the upper bits of the entry that discovered it, so the next
//    frontier's pending edges (sampler.cpp:95,102) and the bound behind `sigma_small` are sums over registers:
//    sum_frontier_degrees -- two more dependent round trips per level -- is not needed.
// Sets ex.pending, sh.prev_pending[e] and sh.sigma_small[e] itself.
// RW = entries per row (SamplerParams::ell_width): 8, or 4 -- one 16-byte load per row, half the tables, no second
// entry group.
template <int BLOCK, int ITEMS, int RW>
__device__ bool expand_level_ell(const SamplerParams &p, u32 *lab, int e, SideRegs &ex, const SideRegs &ot, u32 *contact,
                                 u32 &contact_n, BlockShared<BLOCK, ITEMS> &sh, WorkRegs &wk) {
    constexpr u32 W = RW;
    constexpr u32 KEYS = BLOCK * W; // candidates per chunk, at most; also the number of hash slots
    constexpr u32 HBITS = (BLOCK == 32 ? 5 : BLOCK == 64 ? 6 : 7) + (W == 8 ? 3 : 2);
    constexpr int WARPS = BLOCK / 32;
    static_assert((1u << HBITS) == KEYS && (W == 8 || W == 4), "hash table size; a row is one or two 16-byte loads");
    using Shared = BlockShared<BLOCK, ITEMS>;
    static_assert(sizeof(u32) * 3 * KEYS <= offsetof(Shared, c_sig) + sizeof(sh.c_sig) - offsetof(Shared, f_key) &&
                      offsetof(Shared, c_sig) + sizeof(sh.c_sig) - offsetof(Shared, f_key) ==
                          sizeof(sh.f_key) + sizeof(sh.f_s) + sizeof(sh.f_v) + sizeof(sh.f_o) + sizeof(sh.c_beg) +
                              sizeof(sh.c_scan) + sizeof(sh.c_sig),
                  "dedup tables alias the contact-edge and chunk arrays (live in the meet phase / the general expansion only)");
    // Tables, as shared-window byte addresses (ld/st/atom.shared: no generic-address arithmetic per access):
    u32 *tab = reinterpret_cast<u32 *>(sh.f_key);
    const u32 kv_base = smem_addr(tab);          // [W][BLOCK] by key 8 t + k at [k][t] (no bank conflicts): the candidate's slot;
    const u32 kv = kv_base + 4 * threadIdx.x;    //   then a loser's winner key / a winner's idx
    const u32 hv = kv_base + 4 * KEYS;           // [KEYS] hash set: the slot's vertex ...
    const u32 hk = hv + 4 * KEYS;                // [KEYS] ... and the lowest key that brought it
    const u32 tid = threadIdx.x;
    const u32 fb = ex.fb, fe = ex.cnt;
    const u32 level_start = fe;
    const u32 next_depth = ex.depth + 1;
    const u32 base = ex.base, ot_cnt = ot.cnt; // (side[] is indexed at run time and lives in local memory)
    u32 cnt = fe;
    contact_n = 0;
    const bool sigma_small = sh.sigma_small[e] != 0;
    if (static_cast<u64>(next_depth) + 1 > p.aux_cap)
        return false;
    if (tid == 0) {
        st_cg(ex.pp->lvl + next_depth, level_start);
        sh.min_contact = 0xffffffffu;
        EBC_STAT(sh.ws[kW_V_exp] += fe - fb;)
        EBC_STAT(sh.ws[kW_levels] += 1;)
        EBC_STAT(sh.ws[kW_E_bfs] += ex.pending;) // the frontier's adjacency entries
    }
    const uint4 empty4 = make_uint4(kEllEmpty, kEllEmpty, kEllEmpty, kEllEmpty);
    uint4 *h_mine = reinterpret_cast<uint4 *>(tab + KEYS) + tid; // this thread clears h_mine[0], [BLOCK], ... [(W/2 - 1) BLOCK] (hv and hk)
#pragma unroll
    for (int q = 0; q < static_cast<int>(W / 2); ++q)
        h_mine[q * BLOCK] = empty4;
    __syncthreads();
    const u32 key0 = tid * W;
    u32 pend = 0;  // degrees of the vertices this thread settled
    u64 gsum = 0;  // saturating sum of sigma[u] over this thread's level edges (= its share of the new sigmas)
    u32 n_lvl = 0;
    // The frontier is known when the level starts, so a chunk's vertex is loaded two chunks ahead and its row one
    // chunk ahead: of the three trips only the labels' stays on a chunk's critical path.
    const uint4 *rows = reinterpret_cast<const uint4 *>(p.ell);
    const uint4 *rows4 = W == 8 ? reinterpret_cast<const uint4 *>(p.ell4) : nullptr; // (uniform)
    auto load_row = [&](u32 u, uint4 &a, uint4 &b) {
        if constexpr (W == 8) {
            if (rows4) { // 16 bytes unless the row has more than four entries
                a = __ldg(rows4 + u);
                if (a.x != kEllEscape)
                    return;
            }
            a = __ldg(rows + 2 * static_cast<u64>(u));
            b = __ldg(rows + 2 * static_cast<u64>(u) + 1);
        } else {
            a = __ldg(rows + u);
        }
    };
    uint4 a_nxt = empty4, b_nxt = empty4;
    if (fb + tid < fe)
        load_row(ld_cg(ex.pp->list + fb + tid), a_nxt, b_nxt);
    u32 u_nxt = fb + BLOCK + tid < fe ? ld_cg(ex.pp->list + fb + BLOCK + tid) : 0u;
    const unsigned char *pm_in = reinterpret_cast<const unsigned char *>(ex.pp->pm);
    for (u32 c0 = fb; c0 < fe; c0 += BLOCK) {
        // ---- trips 1 and 2 (of the next chunks): vertices, rows ----
        const u32 i = c0 + tid;
        const uint4 a = a_nxt, b = b_nxt;
        const u64 sig_u = i < fe ? ld_cg(ex.pp->sig + i) : 0;
        // Entries that lead back to the vertices this one was discovered from: their targets sit one level down,
        // visited, and a look at their labels -- two levels after they were written, long evicted from L2 -- would
        // change nothing (sampler.cpp:92,97 both fail).  On a grid that is every second entry.
        const u32 parents = i < fe ? __ldcg(pm_in + i) : 0u;
        a_nxt = empty4, b_nxt = empty4;
        if (i + BLOCK < fe)
            load_row(u_nxt, a_nxt, b_nxt);
        u_nxt = i + 2 * BLOCK < fe ? ld_cg(ex.pp->list + i + 2 * BLOCK) : 0u;
        // Entries are handled in two groups of four; the second one exists in few warps (a row of more than four
        // entries), and its code is a copy of the first with other constants -- executed rarely, it costs no
        // instruction-cache space worth mentioning, while a loop over the groups costs every access a run-time
        // shift or select.
        const bool two = W == 8 && __any_sync(0xffffffffu, b.x != kEllEmpty);
        // ---- trip 3: labels; candidates enter the hash set ----
        u32 cand = 0, ccand = 0; // bit k: entry k is unvisited on this side / and visited on the other one
        u32 n_edges = 0;         // level edges of this thread in this chunk
        auto classify = [&](auto G, const uint4 &r) {
            constexpr int g = decltype(G)::value;
            const u32 en[4] = {r.x, r.y, r.z, r.w};
            u32 lb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
                lb[q] = en[q] != kEllEmpty && !(parents & (1u << (4 * g + q))) ? ld_cg(lab + (en[q] & kEllIdMask)) : 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (en[q] == kEllEmpty || (parents & (1u << (4 * g + q))))
                    continue;
                const u32 v = en[q] & kEllIdMask;
                const u32 d = lb[q] - base, idx = d >> 1; // label = base + 2 idx + side (stale labels: idx >= 2^30)
                const bool here = ((d ^ static_cast<u32>(e)) & 1u) == 0;
                const u32 rev_bit = 1u << ((en[q] >> kEllRevShift) & (W - 1));
                if (here && idx < cnt) {
                    if (idx >= level_start) { // dist[v] == next_depth (sampler.cpp:97), settled by an earlier chunk
                        sat_atomic_add(ex.pp->sig + idx, sig_u, sigma_small);
                        red_or_u32(ex.pp->pm + (idx >> 2), rev_bit << (8 * (idx & 3)));
                        ++n_edges;
                    }
                    continue;
                }
                cand |= 1u << (4 * g + q);
                u32 slot = (v * 2654435761u) >> (32 - HBITS);
                for (;;) { // (a chunk has at most KEYS distinct candidates: there is a slot for each)
                    const u32 prev = atoms_cas_u32(hv + 4 * slot, kEllEmpty, v);
                    if (prev == kEllEmpty || prev == v)
                        break;
                    slot = (slot + 1) & (KEYS - 1);
                }
                reds_min_u32(hk + 4 * slot, key0 + 4 * g + q);
                sts_u32(kv + 4 * ((4 * g + q) * BLOCK), slot);
                if (!here && idx < ot_cnt) // other.visited(v) (sampler.cpp:107)
                    ccand |= 1u << (4 * g + q);
            }
        };
        classify(std::integral_constant<int, 0>{}, a);
        if constexpr (W == 8)
            if (two)
                classify(std::integral_constant<int, 1>{}, b);
        n_edges += __popc(cand);
        n_lvl += n_edges;
        {
            u64 add = sig_u * n_edges;
            if (__umul64hi(sig_u, n_edges))
                add = ~0ull;
            gsum = gsum > ~0ull - add ? ~0ull : gsum + add;
        }
        // ---- winners; rank them: inclusive scan over the threads of (winners, contact winners) ----
        __syncthreads(); // the hash set is complete
        u32 win = 0;
        auto resolve = [&](auto G) {
            constexpr int g = decltype(G)::value;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (cand & (1u << (4 * g + q))) {
                    const u32 mine = kv + 4 * ((4 * g + q) * BLOCK);
                    const u32 slot = lds_u32(mine);
                    const u32 w = lds_u32(hk + 4 * slot);
                    if (w == key0 + 4 * g + q)
                        win |= 1u << (4 * g + q);
                    else
                        sts_u32(mine, w);
                }
        };
        if (cand & 0x0fu)
            resolve(std::integral_constant<int, 0>{});
        if constexpr (W == 8)
            if (cand & 0xf0u)
                resolve(std::integral_constant<int, 1>{});
        const u32 packed = __popc(win) | (__popc(win & ccand) << 16);
        u32 incl = packed;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane_id() >= static_cast<u32>(o))
                incl += t;
        }
        if (WARPS > 1) {
            if (lane_id() == 31)
                sh.warp_cnt[tid >> 5] = incl;
            __syncthreads();
        }
        u32 totals = WARPS > 1 ? 0u : __shfl_sync(0xffffffffu, incl, 31);
        if (WARPS > 1) {
#pragma unroll
            for (int w = 0; w < WARPS; ++w) {
                const u32 c = sh.warp_cnt[w];
                totals += c;
                if (static_cast<u32>(w) < (tid >> 5))
                    incl += c;
            }
        }
        const u32 winners = totals & 0xffffu, ctot = totals >> 16;
        if (static_cast<u64>(cnt) + winners > p.cap || (ctot && static_cast<u64>(contact_n) + ctot > p.aux_cap)) {
            ex.cnt = cnt; // nothing of this chunk was written
            return false;
        }
        u32 my_idx = cnt + ((incl - packed) & 0xffffu), my_c = contact_n + ((incl - packed) >> 16);
        auto settle = [&](auto G, const uint4 &r) {
            constexpr int g = decltype(G)::value;
            const u32 en[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (win & (1u << (4 * g + q))) {
                    const u32 v = en[q] & kEllIdMask;
                    if (ccand & (1u << (4 * g + q))) { // contact (sampler.cpp:105-108); the label still holds the other side's idx
                        const u32 oi = (ld_cg(lab + v) - base) >> 1;
                        atomicMin(&sh.min_contact, oi);
                        st_cg(contact + 2 * static_cast<u64>(my_c), my_idx);
                        st_cg(contact + 2 * static_cast<u64>(my_c) + 1, oi);
                        ++my_c;
                    }
                    const u32 mine = kv + 4 * ((4 * g + q) * BLOCK);
                    st_cg(lab + v, make_label(base, my_idx, e)); // settle (sampler.cpp:93-95)
                    st_cg(ex.pp->list + my_idx, v);
                    st_cg(ex.pp->sig + my_idx, sig_u); // the discovering edge's sigma (sampler.cpp:98)
                    __stcg(reinterpret_cast<unsigned char *>(ex.pp->pm) + my_idx,
                           static_cast<unsigned char>(1u << ((en[q] >> kEllRevShift) & (W - 1))));
                    sts_u32(mine, my_idx);
                    pend += (en[q] >> kEllDegShift) + 1;
                    ++my_idx;
                }
        };
        if (win & 0x0fu)
            settle(std::integral_constant<int, 0>{}, a);
        if constexpr (W == 8)
            if (win & 0xf0u)
                settle(std::integral_constant<int, 1>{}, b);
#pragma unroll
        for (int q = 0; q < static_cast<int>(W / 2); ++q) // (every thread read the hash set before the scan's barrier / shuffles)
            h_mine[q * BLOCK] = empty4;
        __syncthreads(); // settled vertices, kv and the cleared hash set are visible
        auto add_sigma = [&](auto G, const uint4 &r) { // later discoverers of a vertex settled in this chunk (sampler.cpp:97-98)
            constexpr int g = decltype(G)::value;
            const u32 en[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (cand & ~win & (1u << (4 * g + q))) {
                    const u32 w = lds_u32(kv + 4 * ((4 * g + q) * BLOCK)); // the winner's key
                    const u32 idx = lds_u32(kv_base + 4 * ((w & (W - 1)) * BLOCK + w / W));
                    sat_atomic_add(ex.pp->sig + idx, sig_u, sigma_small);
                    red_or_u32(ex.pp->pm + (idx >> 2), (1u << ((en[q] >> kEllRevShift) & (W - 1))) << (8 * (idx & 3)));
                }
        };
        if (cand & ~win & 0x0fu)
            add_sigma(std::integral_constant<int, 0>{}, a);
        if constexpr (W == 8)
            if (cand & ~win & 0xf0u)
                add_sigma(std::integral_constant<int, 1>{}, b);
        cnt += winners;
        contact_n += ctot;
    }
    EBC_STAT(wk.e_lvl += n_lvl;)
    const u64 pending = block_sum_u64<BLOCK>(pend, sh.red64);
    const int big = __syncthreads_or(gsum >= (1ull << 63) / BLOCK ? 1 : 0);
    if (tid == 0) {
        EBC_STAT(sh.ws[kW_V_set] += cnt - level_start;)
        EBC_STAT(sh.ws[kW_F_chk] += cnt - level_start;)
        sh.prev_pending[e] = ex.pending;
        sh.sigma_small[e] = big ? 0u : 1u;
    }
    ex.pending = pending;
    ex.fb = level_start; // sampler.cpp:101-103
    ex.cnt = cnt;
    ex.depth = next_depth;
    __syncthreads();
    return true;
}

// Read-only scan of the level that is about to be expanded on side `e`: every
// adjacency slot is visited (its target is tested exactly as in expand_level)
// but nothing is written.  Each slot whose target is unvisited on
// this side and visited on the other side is a CONTACT EDGE; it is appended
// (unordered) to `edges` as 6 words {frontier position, index in row, target,
// other-side idx, sigma[u] lo, hi}.  If the level has at least one contact edge
// the search ends with this level (sampler.cpp:105-115), and everything the
// reference derives from it -- the meet set in discovery order and
// sigma_ex[v] = sat-sum of sigma[u] over the parents u of v (sampler.cpp:97-98)
// -- can be recomputed from the contact edges alone (meet_from_edges), so the
// ~10^4 label / list / sigma writes of settling a level whose other vertices
// are never looked at again are skipped.  Returns the number of contact edges
// (possibly > edge_cap, in which case the caller falls back to expand_level).
// new_slots counts (per thread) the slots whose target is unvisited on this
// side (= the level's E_lvl, sampler.cpp:97).
//
// The scan is unordered (a contact edge carries its own discovery key), so the rows are streamed: a row is
// cut into items of G lanes x 4 consecutive entries, aligned to 16 bytes; a group of G lanes takes item after
// item (one 128-bit load per lane, the next item's entries requested before the current one's are tested) and
// finds an item's row with one search per group instead of one per slot.  G = 32 on hub graphs (rows of 10^3..10^5
// entries), 4 otherwise.  Entries a 16-byte group shares with the neighbouring rows are masked out.
#ifndef EBC_PROBE_G
#define EBC_PROBE_G 8
#endif
// Appends one contact edge (see probe_level); out of line, it runs a few dozen times per sample.
static __device__ __forceinline__ void record_contact_edge(u32 *edges, u32 pos, u32 frontier_pos, u32 index_in_row, u32 v, u32 oi,
                                                        u64 sg) {
    u64 *w = reinterpret_cast<u64 *>(edges) + 3 * static_cast<u64>(pos); // (24-byte records in an 8-byte aligned array)
    st_cg(w + 0, static_cast<u64>(frontier_pos) | (static_cast<u64>(index_in_row) << 32));
    st_cg(w + 1, static_cast<u64>(v) | (static_cast<u64>(oi) << 32));
    st_cg(w + 2, sg);
}

template <int BLOCK, int ITEMS, bool BITS>
__device__ u32 probe_level(const SamplerParams &p, const u32 *lab, const u32 *bits, const u32 *vf, int e, const SideRegs &ex,
                           const SideRegs &ot, u32 *edges, u32 edge_cap, BlockShared<BLOCK, ITEMS> &sh, u64 &new_slots,
                           u64 &total_slots, u64 *scr_first, u64 *scr_sum) {
    constexpr u32 G = BITS ? EBC_PROBE_G : 4; // lanes per item
    constexpr u32 NG = BLOCK / G;             // groups per CTA
    constexpr u32 kItemLen = 4 * G;           // adjacency entries per item
#ifndef EBC_LONG_ENTRIES
#define EBC_LONG_ENTRIES 1
#endif
    constexpr u32 kLongEntries = EBC_LONG_ENTRIES * BLOCK; // a long row: at least one entry per thread (profiles/r02_probe.txt)
    const u32 tid = threadIdx.x;
    const u32 gid = tid / G, q = tid % G;
    const u32 fb = ex.fb, fe = ex.cnt;
    // The side as a value of its own (the compiler otherwise re-derives it from the two 64-bit pending counts at
    // every use in the scan), the filter by its shared-window address (no generic-address arithmetic per look-up).
    int e_opaque = e;
    asm volatile("" : "+r"(e_opaque));
    const bool backward = e_opaque != 0;
    const u32 vf_base = smem_addr(vf);
    if (tid == 0) {
        sh.edge_cnt = 0;
        sh.min_contact = 0xffffffffu;
    }
    u64 t_total = 0;
    u32 fresh = 0; // slots whose target is unvisited on this side (< 2^32 per thread and level)
    for (u32 c0 = fb; c0 < fe; c0 += BLOCK) {
        t_total += load_chunk<BLOCK>(p, ex.pp, c0, fe, sh.c_beg, sh.c_scan, sh.c_sig, sh.red64);
        // items per row (thread tid owns row tid of the chunk), exclusive prefix -> l_scan[0..BLOCK]
        // (in f_key, which is only live in the meet phase and in expand_level's multi-row tiles)
        static_assert(2 * FinalEdgeCap<BLOCK>::value >= BLOCK + 1, "l_scan aliases f_key");
        u32 *l_scan = reinterpret_cast<u32 *>(sh.f_key);
        {
            const u64 deg = sh.c_scan[tid + 1] - sh.c_scan[tid];
            // Long rows are streamed by the whole CTA, one after the other, below; only the others are cut into items.
            const bool is_long = (sh.c_beg[tid] & 3) + deg >= kLongEntries;
            const u32 long_ballot = __ballot_sync(0xffffffffu, is_long);
            if (lane_id() == 0)
                sh.warp_cnt2[tid >> 5] = long_ballot;
            const u32 items = deg && !is_long ? static_cast<u32>(((sh.c_beg[tid] & 3) + deg + kItemLen - 1) / kItemLen) : 0u;
            u32 inc = items;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const u32 t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane_id() >= static_cast<u32>(o))
                    inc += t;
            }
            if (BLOCK > 32) {
                if (lane_id() == 31)
                    sh.warp_cnt[tid >> 5] = inc;
                __syncthreads();
                u32 before = 0;
                for (u32 w = 0; w < (tid >> 5); ++w)
                    before += sh.warp_cnt[w];
                inc += before;
            }
            l_scan[tid + 1] = inc;
            if (tid == 0)
                l_scan[0] = 0;
            __syncthreads();
        }
        // Tests the four entries `cur` (bit k of `valid`: entry k belongs to the row) of row `row_c` of the chunk;
        // rel0_c = index in the row of the first of the four (negative where the 16-byte group starts before the row).
        auto test_quad = [&](const uint4 &cur, u32 valid, u32 row_c, int rel0_c) {
            const u32 vv[4] = {cur.x, cur.y, cur.z, cur.w};
            u32 need = 0; // bit k: entry k must be looked up in global memory
            if (BITS) {
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    // (word (v mod kPositions) / 32 by its shared-window address; the shift takes v mod 32 by itself)
                    const u32 word = lds_u32(vf_base + ((vv[k] >> 3) & (4 * VisitedFilter<BLOCK>::kWords - 4)));
                    need |= ((word >> (vv[k] & 31)) & 1u) << k; // clear: certainly unvisited on both sides
                }
                need &= valid;
                fresh += __popc(valid & ~need);
            } else {
                need = valid;
            }
            if (need) {
                u64 both[4]; // bitmap word of both sides, or (labels) the 4-byte label
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    both[k] = 0;
                    if ((need >> k) & 1u)
                        both[k] = BITS ? ld_cg(reinterpret_cast<const u64 *>(bits) + (vv[k] >> 5))
                                       : static_cast<u64>(ld_cg(lab + vv[k]));
                }
                u32 cmask = 0;   // bit k: entry k is a contact edge
                u32 ois[4] = {0, 0, 0, 0};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if (!((need >> k) & 1u))
                        continue;
                    u32 oi;
                    if (BITS) {
                        const u32 lo = static_cast<u32>(both[k]), hi = static_cast<u32>(both[k] >> 32);
                        if (((backward ? hi : lo) >> (vv[k] & 31)) & 1u)
                            continue; // visited before this level
                        fresh += 1;
                        if (!(((backward ? lo : hi) >> (vv[k] & 31)) & 1u))
                            continue; // not a contact
                        // The other side's bit already says "contact"; its idx is only needed for the record
                        // and is fetched for all contact edges at once after the scan.
                        oi = 0;
                    } else {
                        const u32 lbl = static_cast<u32>(both[k]);
                        if (label_idx(lbl, ex.base, e) < ex.cnt)
                            continue; // visited before this level
                        fresh += 1;
                        oi = label_idx(lbl, ex.base, 1 - e);
                        ois[k] = oi;
                    }
                    if (oi < ot.cnt) {
                        if (!BITS)
                            atomicMin(&sh.min_contact, oi);
                        cmask |= 1u << k;
                    }
                }
                if (cmask) { // rare: one counter update per quad, one copy of the record code
                    u32 pos = atomicAdd(&sh.edge_cnt, static_cast<u32>(__popc(cmask)));
                    const u64 sg = sh.c_sig[row_c];
#pragma unroll 1
                    for (; cmask; cmask &= cmask - 1, ++pos) {
                        const int k = __ffs(cmask) - 1;
                        if (pos < edge_cap)
                            record_contact_edge(edges, pos, (c0 - fb) + row_c, static_cast<u32>(rel0_c + k),
                                                k == 0 ? vv[0] : k == 1 ? vv[1] : k == 2 ? vv[2] : vv[3],
                                                BITS ? 0u : k == 0 ? ois[0] : k == 1 ? ois[1] : k == 2 ? ois[2] : ois[3], sg);
                    }
                }
            }
        };
        // ---- long rows: thread t takes the 16-byte groups t, t + BLOCK, ... of the row; no search, and only the
        // row's first and last group are partial ----
#pragma unroll 1
        for (int w = 0; w < BLOCK / 32; ++w) {
            u32 mask = sh.warp_cnt2[w];
            while (mask) {
                const u32 r = 32u * w + (__ffs(mask) - 1);
                mask &= mask - 1;
                const u64 beg = sh.c_beg[r];
                const u32 head = static_cast<u32>(beg & 3);
                const u32 span = head + static_cast<u32>(sh.c_scan[r + 1] - sh.c_scan[r]); // (a row has < 2^32 entries)
                const u32 nq = (span + 3) >> 2;
                const uint4 *quads = reinterpret_cast<const uint4 *>(p.targets + (beg - head));
                u32 qi = tid;
                uint4 cur = make_uint4(0, 0, 0, 0);
                if (qi < nq)
                    cur = __ldg(quads + qi);
                while (qi < nq) {
                    const u32 qn = qi + BLOCK;
                    uint4 nxt = make_uint4(0, 0, 0, 0);
                    if (qn < nq)
                        nxt = __ldg(quads + qn);
                    // the row is a stream from DRAM: ask L2 for the sector three rounds ahead (config 4 +5 %; six
                    // rounds ahead +4 %; config 2, whose rows mostly sit in L2, +0)
                    if (qi + 3 * BLOCK < nq && (qi & 1) == 0) // (one request per 32-byte sector; qi = tid mod 2)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(quads + qi + 3 * BLOCK));
                    u32 valid = 0xfu;
                    if (qi == 0)
                        valid = (0xfu << head) & 0xfu;
                    if (qi == nq - 1)
                        valid &= 0xfu >> (4 * nq - span);
                    test_quad(cur, valid, r, static_cast<int>(4 * qi) - static_cast<int>(head));
                    cur = nxt;
                    qi = qn;
                }
            }
        }
        const u32 n_items = l_scan[BLOCK];
        // Iteration i requests the entries of item i and tests those requested by iteration i - 1 (nothing in
        // the first one); written as one loop so that the request code exists once.
        int row = 0;              // row of the item requested last (items ascend per group)
        u32 row_c = 0, deg_c = 0; // ... of the item under test: row, its degree,
        int rel0_c = 0;           //     index in the row of the item's first entry (negative: 16-byte alignment)
        bool have_c = false;
        uint4 cur = make_uint4(0, 0, 0, 0);
        for (u32 item = gid;; item += NG) {
            const bool have_n = item < n_items;
            uint4 nxt = make_uint4(0, 0, 0, 0);
            u32 deg_n = 0;
            int rel0_n = 0;
            if (have_n) {
                // row = last r with l_scan[r] <= item: gallop upwards from the previous item's row, then bisect
                int lo = row, hi = lo + 1, step = 1;
                while (hi < BLOCK && l_scan[hi] <= item) {
                    lo = hi;
                    hi = hi + step < BLOCK ? hi + step : BLOCK;
                    step <<= 1;
                }
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (l_scan[mid] <= item)
                        lo = mid;
                    else
                        hi = mid;
                }
                row = lo;
                const u64 beg = sh.c_beg[lo];
                const u64 first = (beg & ~u64{3}) + static_cast<u64>(item - l_scan[lo]) * kItemLen + 4 * q; // 16-byte aligned
                rel0_n = static_cast<int>(static_cast<long long>(first) - static_cast<long long>(beg));
                deg_n = static_cast<u32>(sh.c_scan[lo + 1] - sh.c_scan[lo]);
                nxt = ldg_targets4(p.targets + first);
            }
            if (have_c) {
                // entries [lo_k, hi_k) of the four belong to the row
                const int lo_k = rel0_c < 0 ? -rel0_c : 0;
                const int left = static_cast<int>(deg_c) - rel0_c;
                const int hi_k = left < 4 ? left : 4;
                if (hi_k > lo_k)
                    test_quad(cur, ((1u << hi_k) - 1u) & ~((1u << lo_k) - 1u), row_c, rel0_c);
            }
            if (!have_n)
                break;
            cur = nxt;
            row_c = static_cast<u32>(row);
            deg_c = deg_n;
            rel0_c = rel0_n;
            have_c = true;
        }
    }
    new_slots += fresh;
    __syncthreads();
    total_slots = t_total;
    const u32 found = sh.edge_cnt;
    if (BITS && found > 0 && found <= edge_cap) { // other-side idx of every contact edge, and their minimum
        // (four edges per thread at a time: the two dependent trips of each overlap.)  More edges than
        // meet_from_edges takes: the scratch entries pick_meet_large indexes by oi - ot.fb are cleared on the way
        // (its pass A) -- a contact vertex always sits in the other side's LAST level: had it been expanded there,
        // its neighbour on this side's frontier would have been a contact one level earlier.
        const bool clear = scr_first != nullptr && found > static_cast<u32>(FinalEdgeCap<BLOCK>::value);
        u32 lowest = 0xffffffffu;
#pragma unroll 1
        for (u32 i0 = 0; i0 < found; i0 += 4 * BLOCK) {
            u32 v[4], oi[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const u32 i = i0 + k * BLOCK + tid;
                v[k] = i < found ? ld_cg(edges + 6 * static_cast<u64>(i) + 2) : 0xffffffffu;
            }
#pragma unroll
            for (int k = 0; k < 4; ++k)
                oi[k] = v[k] != 0xffffffffu ? label_idx(ld_cg(lab + v[k]), ot.base, 1 - e) : 0xffffffffu;
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (v[k] != 0xffffffffu) {
                    st_cg(edges + 6 * static_cast<u64>(i0 + k * BLOCK + tid) + 3, oi[k]);
                    lowest = oi[k] < lowest ? oi[k] : lowest;
                    if (clear && oi[k] - ot.fb < ot.cnt - ot.fb) {
                        st_cg(scr_first + (oi[k] - ot.fb), ~0ull);
                        st_cg(scr_sum + (oi[k] - ot.fb), static_cast<u64>(0));
                    }
                }
        }
        if (lowest != 0xffffffffu)
            atomicMin(&sh.min_contact, lowest);
        __syncthreads();
    }
    return found;
}

// Meet set of a probed final level from its m <= final_edge_cap contact edges:
// groups the edges by target, sigma_ex[v] = saturating sum of the parents' sigma
// (order independent), discovery key of v = smallest (frontier position, index
// in row) among its edges -- exactly the order in which the reference would
// have appended v to `next` -- and writes the members whose other-side idx lies
// in [olo, ohi) to meetbuf in that order as {v, other idx, sigma lo, sigma hi}.
template <int BLOCK, int ITEMS>
__device__ u32 meet_from_edges(const u32 *edges, u32 m, u32 olo, u32 ohi, u32 *meetbuf,
                               BlockShared<BLOCK, ITEMS> &sh) {
    constexpr int CAP = FinalEdgeCap<BLOCK>::value;
    constexpr int PER = CAP / BLOCK > 0 ? CAP / BLOCK : 1;
    // Edges of one vertex find each other through hash buckets (a chained table over the edge indices: head[] by
    // bucket, next[] by edge), members rank themselves against the dense list of members only: both passes used to
    // walk all m edges per edge -- 2 m^2 / BLOCK steps per thread, a fifth of a sample on hub graphs.  The tables
    // live in the chunk arrays, which nobody uses between the level loop and the next sample.
    using Shared = BlockShared<BLOCK, ITEMS>;
    static_assert(CAP <= 0xffff && sizeof(u32) * CAP + sizeof(unsigned short) * CAP <=
                                       sizeof(sh.c_beg) + sizeof(sh.c_scan) + sizeof(sh.c_sig) &&
                      offsetof(Shared, c_sig) + sizeof(sh.c_sig) - offsetof(Shared, c_beg) ==
                          sizeof(sh.c_beg) + sizeof(sh.c_scan) + sizeof(sh.c_sig),
                  "bucket heads and chains alias the chunk arrays");
    u32 *head = reinterpret_cast<u32 *>(sh.c_beg);                        // [CAP] first edge of the bucket, or kNone
    unsigned short *next = reinterpret_cast<unsigned short *>(head + CAP); // [CAP] next edge of the same bucket
    unsigned short *dense = reinterpret_cast<unsigned short *>(sh.c_beg); // [CAP] afterwards: the members' edge indices
    constexpr u32 kNone = 0xffffu;
    const u32 tid = threadIdx.x;
    for (u32 i = tid; i < static_cast<u32>(CAP); i += BLOCK)
        head[i] = kNone;
    for (u32 i = tid; i < m; i += BLOCK) {
        const u32 *w = edges + 6 * static_cast<u64>(i);
        sh.f_key[i] = (static_cast<u64>(ld_cg(w)) << 32) | ld_cg(w + 1);
        sh.f_v[i] = ld_cg(w + 2);
        sh.f_o[i] = ld_cg(w + 3);
        sh.f_s[i] = static_cast<u64>(ld_cg(w + 4)) | (static_cast<u64>(ld_cg(w + 5)) << 32);
    }
    __syncthreads();
    u32 vi[PER];
    u64 ki[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const u32 i = tid + q * BLOCK;
        vi[q] = i < m ? sh.f_v[i] : 0u;
        ki[q] = i < m ? sh.f_key[i] : 0ull;
        if (i < m)
            next[i] = static_cast<unsigned short>(atomicExch(head + ((vi[q] * 2654435761u) >> 16) % CAP, i));
    }
    __syncthreads();
    // sigma_ex[v] = sat-sum over v's edges (sampler.cpp:11-13,97-98); the edge with the smallest key represents v
    u64 sum[PER];
    bool first[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const u32 i = tid + q * BLOCK;
        sum[q] = 0;
        first[q] = i < m;
        if (i < m)
            for (u32 j = head[((vi[q] * 2654435761u) >> 16) % CAP]; j != kNone; j = next[j])
                if (sh.f_v[j] == vi[q]) {
                    const u64 sj = sh.f_s[j];
                    sum[q] = sum[q] > ~0ull - sj ? ~0ull : sum[q] + sj;
                    if (sh.f_key[j] < ki[q])
                        first[q] = false;
                }
    }
    __syncthreads(); // every thread has read f_s, head and next
    bool member[PER];
    u32 before = 0; // members in slots below this thread's (ranking them all needs an order, any order)
    {
        u32 mine = 0;
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const u32 i = tid + q * BLOCK;
            member[q] = first[q] && sh.f_o[i] - olo < ohi - olo;
            if (first[q])
                sh.f_s[i] = sum[q];
            mine += member[q] ? 1u : 0u;
        }
        u32 incl = mine;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane_id() >= static_cast<u32>(o))
                incl += t;
        }
        if (BLOCK > 32) {
            if (lane_id() == 31)
                sh.warp_cnt[tid >> 5] = incl;
            __syncthreads();
            for (u32 w = 0; w < (tid >> 5); ++w)
                incl += sh.warp_cnt[w];
        }
        before = incl - mine;
        if (tid == BLOCK - 1)
            sh.bcast[1] = incl;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q)
        if (member[q])
            dense[before++] = static_cast<unsigned short>(tid + q * BLOCK);
    __syncthreads();
    const u32 members = sh.bcast[1];
    // position in discovery order = number of members with a smaller key (sampler.cpp:92-95: order of `next`)
    u32 rank[PER];
#pragma unroll
    for (int q = 0; q < PER; ++q)
        rank[q] = 0;
#pragma unroll 1
    for (u32 jj = 0; jj < members; ++jj) {
        const u64 kj = sh.f_key[dense[jj]];
#pragma unroll
        for (int q = 0; q < PER; ++q)
            rank[q] += kj < ki[q] ? 1u : 0u;
    }
#pragma unroll
    for (int q = 0; q < PER; ++q) {
        const u32 i = tid + q * BLOCK;
        if (member[q]) {
            u32 *w = meetbuf + 4 * static_cast<u64>(rank[q]);
            st_cg(w + 0, vi[q]);
            st_cg(w + 1, sh.f_o[i]);
            st_cg(w + 2, static_cast<u32>(sh.f_s[i]));
            st_cg(w + 3, static_cast<u32>(sh.f_s[i] >> 32));
        }
    }
    __syncthreads();
    return members;
}

// Lanes 0 .. n-1 of a warp hold one candidate each (discovery key, 128-bit weight; weight 0 = not a candidate):
// the lane of the first candidate in key order whose inclusive prefix of weights, on top of `acc`, exceeds `pick`
// (sampler.cpp:126-132), or 32.  A prefix that leaves 128 bits exceeds.  acc <= pick.
static __device__ __forceinline__ u32 warp_first_exceeding(u64 key, u64 wl, u64 wh, u32 n, u128 acc, u128 pick) {
    u128 excl = acc;
    bool excl_ovf = false;
#pragma unroll 1
    for (u32 j = 0; j < n; ++j) {
        const u64 kj = __shfl_sync(0xffffffffu, key, j), lj = __shfl_sync(0xffffffffu, wl, j), hj = __shfl_sync(0xffffffffu, wh, j);
        if (kj < key) {
            const u128 t = excl + ((static_cast<u128>(hj) << 64) | lj);
            excl_ovf = excl_ovf || t < excl;
            excl = t;
        }
    }
    const u128 incl = excl + ((static_cast<u128>(wh) << 64) | wl);
    const bool hit = (wl | wh) != 0 && !excl_ovf && excl <= pick && (incl < excl || incl > pick);
    const u32 found = __ballot_sync(0xffffffffu, hit);
    return found ? __ffs(found) - 1 : 32u;
}

// A probed final level with at most 32 contact edges -- more than half of the samples on R-MAT graphs: lane i of every
// warp takes edge i and the whole choice of the meet vertex happens in registers (the warps of a CTA compute it
// redundantly: no shared memory, no barrier).  Two round trips (the edges, sigma on the other side) instead of the
// dozen of meet_from_edges + the prefix search over its global meet set, and a fraction of the instructions.
//  * edges of one vertex find each other with match.any on the other-side idx; sigma_ex = saturating sum of their
//    parents' sigma (sampler.cpp:11-13,97-98), the edge with the smallest discovery key represents the vertex;
//  * weight = sigma_ex * sigma_other (sampler.cpp:121-123), total by a 5-step butterfly with carry count;
//  * a member's exclusive prefix in discovery order = sum of the weights of the members with a smaller key, the
//    chosen one is the member with exclusive <= pick < inclusive (sampler.cpp:126-132).
// Returns the meet vertex; meet_count and total_weight as the reference would see them.
static __device__ __noinline__ u32 pick_meet_warp(const u32 *contact, u32 m, u32 olo, u32 ohi, const u64 *ot_sig, SampleStream &rng,
                                           u32 &meet_count, u128 &total_weight) {
    constexpr u32 kAll = 0xffffffffu;
    const u32 lane = lane_id();
    const u64 *w = reinterpret_cast<const u64 *>(contact) + 3 * lane; // {position | index << 32, v | oi << 32, sigma}
    u64 key = ~0ull, sg = 0;
    u32 v = 0, oi = kAll - lane; // (lanes without an edge of the level `best`: alone in their group)
    bool in = false;
    if (lane < m) {
        const u64 q0 = ld_cg(w), q1 = ld_cg(w + 1);
        sg = ld_cg(w + 2);
        if (static_cast<u32>(q1 >> 32) - olo < ohi - olo) {
            in = true;
            key = (q0 << 32) | (q0 >> 32);
            v = static_cast<u32>(q1);
            oi = static_cast<u32>(q1 >> 32);
        }
    }
    const u64 so = in ? ld_cg(ot_sig + oi) : 0ull;
    u32 rest = __match_any_sync(kAll, oi);
    u64 sx = 0, kmin = ~0ull;
    while (__any_sync(kAll, rest != 0)) { // as many rounds as the largest group has edges
        const int src = rest ? __ffs(rest) - 1 : static_cast<int>(lane);
        const u64 s2 = __shfl_sync(kAll, sg, src), k2 = __shfl_sync(kAll, key, src);
        if (rest) {
            sx = sx > ~0ull - s2 ? ~0ull : sx + s2;
            kmin = k2 < kmin ? k2 : kmin;
            rest &= rest - 1;
        }
    }
    const bool member = in && key == kmin;
    const u128 wt = member ? static_cast<u128>(sx) * so : static_cast<u128>(0);
    const u64 wl = static_cast<u64>(wt), wh = static_cast<u64>(wt >> 64);
    meet_count = __popc(__ballot_sync(kAll, member));
    {
        u64 a = wl, b = wh;
        u32 c = 0;
#pragma unroll 1
        for (int o = 16; o > 0; o >>= 1) {
            const u64 a2 = __shfl_xor_sync(kAll, a, o), b2 = __shfl_xor_sync(kAll, b, o);
            const u32 c2 = __shfl_xor_sync(kAll, c, o);
            const u128 x = (static_cast<u128>(b) << 64) | a, y = (static_cast<u128>(b2) << 64) | a2;
            const u128 t = x + y;
            c += c2 + (t < x ? 1u : 0u);
            a = static_cast<u64>(t);
            b = static_cast<u64>(t >> 64);
        }
        total_weight = c ? ~static_cast<u128>(0) : ((static_cast<u128>(b) << 64) | a);
    }
    const u128 pick = uniform_below_u128(rng, total_weight); // sampler.cpp:124
    u32 chosen = warp_first_exceeding(key, wl, wh, m, 0, pick); // (an edge that does not represent a member carries weight 0)
    if (chosen == 32u) { // cannot happen (pick < total); the reference's default is the last member (sampler.cpp:125)
        u64 kmax = member ? key : 0ull;
#pragma unroll 1
        for (int o = 16; o > 0; o >>= 1) {
            const u64 k2 = __shfl_xor_sync(kAll, kmax, o);
            kmax = k2 > kmax ? k2 : kmax;
        }
        chosen = __ffs(__ballot_sync(kAll, member && key == kmax)) - 1;
    }
    return __shfl_sync(kAll, v, chosen);
}

// A probed final level with more contact edges than meet_from_edges holds in shared memory (R-MAT-20: a fifth of
// the samples at one warp per sample, R-MAT-24: 16 % -- the ones with the largest final levels, which would otherwise
// be expanded and settled in full; a hub on the other side's frontier alone brings thousands of contact edges).
// The reference orders the meet set only to turn `pick` into a vertex (sampler.cpp:124-133: the first member whose
// inclusive prefix of weights exceeds pick), so the set is not sorted here: it is SEARCHED, a weighted quickselect on
// the discovery keys.  Everything lives in the slot's global arrays and every pass keeps several independent loads
// per thread in flight (a pass costs its dependent round trips, not its bytes):
//  * a member's other-side idx oi is unique and lies in [olo, ohi), so oi - olo indexes two scratch arrays (unused
//    tails of the two sides' sigma arrays): first[] = smallest discovery key among the vertex' contact edges
//    (= its place in the reference's `next`), sum[] = saturating sum of the parents' sigma (sampler.cpp:97-98);
//  * pass A clears first[] / sum[] where an edge points; pass B does atom.min(first[], key) and adds sigma -- the one
//    edge of a vertex that still finds ~0 in first[] enters the vertex in the member list;
//  * pass C turns the member list into records {key, weight = sum * sigma_other (sampler.cpp:121-123), oi} and
//    totals the weights; pick is drawn;
//  * select: pivot = a record of the active list; S = total weight of the active records with a smaller key.
//    acc + S > pick: the answer is among those; else acc + S + w(pivot) > pick: it is the pivot; else acc takes
//    both and the records with a larger key stay.  Both candidate lists are written in the same pass (front and
//    back of the other buffer).  Contact edges arrive roughly in key order, so the middle of the list is a good
//    pivot: ~log2(members) passes over geometrically shrinking lists.  Sums that leave 128 bits compare as
//    "exceeds", exactly like the reference's running subtraction.
// (Rounds 1-2 sorted the representatives with a one-CTA bitonic network through shared-memory chunks and walked the
// edges one dependent load at a time: 3.3 10^5 cycles per such sample on a one-warp CTA.)
// `contact`: the 6-word edge records at [0, 6 m) of the slot's 6 aux_cap >= 18 m words; the rest is scratch here.
// Returns the chosen member's other-side idx; meet_count and total_weight as the reference would see them.
template <int BLOCK, int ITEMS>
__device__ __noinline__ u32 pick_meet_large(u32 *contact, u32 m, u32 olo, u32 ohi, u64 *first, u64 *sum, const u64 *ot_sig,
                                            bool sigma_small, bool cleared, SampleStream &rng, BlockShared<BLOCK, ITEMS> &sh,
                                            u32 &meet_count, u128 &total_weight
#ifdef EBC_PHASE_COUNTS
                                            , long long *pht
#endif
                                            ) {
#ifdef EBC_PHASE_COUNTS
    long long pt0 = clock64();
#define EBC_PT(i) { const long long t = clock64(); pht[i] += t - pt0; pt0 = t; }
#else
#define EBC_PT(i)
#endif
    constexpr int WARPS = BLOCK / 32;
    constexpr int PE = 4; // edges per thread and batch
    constexpr int PR = 2; // records per thread and batch
    const u32 tid = threadIdx.x;
    const u32 L = ohi - olo;
    const u64 *e64 = reinterpret_cast<const u64 *>(contact); // an edge: {position | index << 32, v | oi << 32, sigma}
    // Positions in two lists for P flagged items per thread: `a` items count upwards from na, `b` items from nb
    // (any order inside a list).  Uniform call; one barrier when WARPS > 1, and the caller keeps another one
    // before the next call.
    auto place = [&](auto P, const bool *fa, const bool *fb, u32 *pa, u32 *pb, u32 &na, u32 &nb) {
        constexpr int N = decltype(P)::value;
        u32 wa = 0, wb = 0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            const u32 ba = __ballot_sync(0xffffffffu, fa[q]), bb = __ballot_sync(0xffffffffu, fb[q]);
            pa[q] = wa + __popc(ba & lanemask_lt());
            pb[q] = wb + __popc(bb & lanemask_lt());
            wa += __popc(ba);
            wb += __popc(bb);
        }
        u32 before = 0, tot = wa | (wb << 16); // (at most 4 * 32 of each kind per warp, 4 * BLOCK <= 2048 in all)
        if (WARPS > 1) {
            if (lane_id() == 0)
                sh.warp_cnt[tid >> 5] = tot;
            __syncthreads();
            tot = 0;
#pragma unroll 1
            for (u32 w = 0; w < static_cast<u32>(WARPS); ++w) {
                const u32 c = sh.warp_cnt[w];
                before += w < (tid >> 5) ? c : 0u;
                tot += c;
            }
        }
#pragma unroll
        for (int q = 0; q < N; ++q) {
            pa[q] += na + (before & 0xffffu);
            pb[q] += nb + (before >> 16);
        }
        na += tot & 0xffffu;
        nb += tot >> 16;
    };
    if (!cleared) { // (probe_level has done it on the way when it could)
#pragma unroll 1
    for (u32 i0 = 0; i0 < m; i0 += PE * BLOCK) { // pass A
        u32 r[PE];
#pragma unroll
        for (int q = 0; q < PE; ++q) {
            const u32 i = i0 + q * BLOCK + tid;
            r[q] = i < m ? static_cast<u32>(ld_cg(e64 + 3 * static_cast<u64>(i) + 1) >> 32) - olo : L;
        }
#pragma unroll
        for (int q = 0; q < PE; ++q)
            if (r[q] < L) {
                st_cg(first + r[q], ~0ull);
                st_cg(sum + r[q], static_cast<u64>(0));
            }
    }
    }
    __syncthreads();
    u32 *members = contact + 16 * static_cast<u64>(m); // other-side idx of every member, unordered
    u32 count = 0, unused = 0;
#pragma unroll 1
    for (u32 i0 = 0; i0 < m; i0 += PE * BLOCK) { // pass B
        u64 key[PE], sg[PE];
        u32 oi[PE];
#pragma unroll
        for (int q = 0; q < PE; ++q) {
            const u32 i = i0 + q * BLOCK + tid;
            const u64 *w = e64 + 3 * static_cast<u64>(i);
            oi[q] = i < m ? static_cast<u32>(ld_cg(w + 1) >> 32) : olo + L;
            const u64 k = i < m ? ld_cg(w) : 0ull;
            key[q] = (k << 32) | (k >> 32);
            sg[q] = i < m ? ld_cg(w + 2) : 0ull;
        }
        bool fresh[PE], none[PE];
#pragma unroll
        for (int q = 0; q < PE; ++q) {
            fresh[q] = oi[q] - olo < L && atom_min_u64(first + (oi[q] - olo), key[q]) == ~0ull;
            none[q] = false;
        }
#pragma unroll
        for (int q = 0; q < PE; ++q)
            if (oi[q] - olo < L)
                sat_atomic_add(sum + (oi[q] - olo), sg[q], sigma_small);
        u32 pa[PE], pb[PE];
        place(std::integral_constant<int, PE>{}, fresh, none, pa, pb, count, unused);
#pragma unroll
        for (int q = 0; q < PE; ++q)
            if (fresh[q])
                st_cg(members + pa[q], oi[q]);
        if (WARPS > 1)
            __syncthreads();
    }
    __syncthreads();
    EBC_PT(0)
    // records of four 8-byte words {key, weight lo, weight hi, oi}: two buffers of `count` records
    u64 *cur = reinterpret_cast<u64 *>(contact + 8 * static_cast<u64>(m));
    u64 *oth = reinterpret_cast<u64 *>(contact); // (over the edges, which nobody reads any more)
    u128 wsum = 0;
#pragma unroll 1
    for (u32 i0 = 0; i0 < count; i0 += PR * BLOCK) { // pass C
        u32 oi[PR];
#pragma unroll
        for (int q = 0; q < PR; ++q) {
            const u32 i = i0 + q * BLOCK + tid;
            oi[q] = i < count ? ld_cg(members + i) : 0xffffffffu;
        }
        u64 key[PR], sm[PR], so[PR];
#pragma unroll
        for (int q = 0; q < PR; ++q)
            key[q] = sm[q] = so[q] = 0;
#pragma unroll
        for (int q = 0; q < PR; ++q)
            if (oi[q] != 0xffffffffu) {
                key[q] = ld_cg(first + (oi[q] - olo));
                sm[q] = ld_cg(sum + (oi[q] - olo));
                so[q] = ld_cg(ot_sig + oi[q]);
            }
#pragma unroll
        for (int q = 0; q < PR; ++q)
            if (oi[q] != 0xffffffffu) {
                const u128 w = static_cast<u128>(sm[q]) * so[q];
                wsum += w;
                u64 *rec = cur + 4 * static_cast<u64>(i0 + q * BLOCK + tid);
                st_cg(rec + 0, key[q]);
                st_cg(rec + 1, static_cast<u64>(w));
                st_cg(rec + 2, static_cast<u64>(w >> 64));
                st_cg(rec + 3, static_cast<u64>(oi[q]));
            }
    }
    u64 wlo, whi, wov;
    block_sum_u128<BLOCK>(wsum, wlo, whi, wov, sh.red64);
    __syncthreads(); // (also: the records are visible)
    total_weight = wov ? ~static_cast<u128>(0) : ((static_cast<u128>(whi) << 64) | wlo);
    meet_count = count;
    const u128 pick = uniform_below_u128(rng, total_weight); // sampler.cpp:124
    EBC_PT(1)
    u64 *cur_buf = cur;
    u32 n_act = count;
    u128 acc = 0; // exact weight of the members below the active keys; acc <= pick
    u32 ans = static_cast<u32>(ld_cg(cur + 3));
#pragma unroll 1
    while (n_act > 32) {
        const u64 *pv = cur + 4 * static_cast<u64>(n_act >> 1);
        const u64 kp = ld_cg(pv);
        const u128 wp = (static_cast<u128>(ld_cg(pv + 2)) << 64) | ld_cg(pv + 1);
        ans = static_cast<u32>(ld_cg(pv + 3));
        u128 s_lt = 0;
        u32 n_lt = 0, n_gt = 0;
#pragma unroll 1
        for (u32 i0 = 0; i0 < n_act; i0 += PR * BLOCK) {
            u64 rec[PR][4];
#pragma unroll
            for (int q = 0; q < PR; ++q) {
                const u32 i = i0 + q * BLOCK + tid;
                const u64 *w = cur + 4 * static_cast<u64>(i);
                rec[q][0] = kp, rec[q][1] = rec[q][2] = rec[q][3] = 0;
                if (i < n_act) {
                    rec[q][0] = ld_cg(w);
                    rec[q][1] = ld_cg(w + 1);
                    rec[q][2] = ld_cg(w + 2);
                    rec[q][3] = ld_cg(w + 3);
                }
            }
            bool lt[PR], gt[PR];
#pragma unroll
            for (int q = 0; q < PR; ++q) {
                lt[q] = rec[q][0] < kp;
                gt[q] = rec[q][0] > kp;
                if (lt[q])
                    s_lt += (static_cast<u128>(rec[q][2]) << 64) | rec[q][1];
            }
            u32 pa[PR], pb[PR];
            place(std::integral_constant<int, PR>{}, lt, gt, pa, pb, n_lt, n_gt);
#pragma unroll
            for (int q = 0; q < PR; ++q)
                if (lt[q] || gt[q]) {
                    u64 *w = oth + 4 * static_cast<u64>(lt[q] ? pa[q] : n_act - 1 - pb[q]);
                    st_cg(w + 0, rec[q][0]);
                    st_cg(w + 1, rec[q][1]);
                    st_cg(w + 2, rec[q][2]);
                    st_cg(w + 3, rec[q][3]);
                }
            if (WARPS > 1)
                __syncthreads();
        }
        u64 lo, hi, ov;
        block_sum_u128<BLOCK>(s_lt, lo, hi, ov, sh.red64);
        const u128 below = acc + ((static_cast<u128>(hi) << 64) | lo);
        if (ov || below < acc || below > pick) { // the answer has a smaller key than the pivot
            u64 *t = cur_buf;
            cur = oth, cur_buf = oth, oth = t;
            n_act = n_lt;
        } else {
            const u128 incl = below + wp;
            if (incl < below || incl > pick || n_gt == 0)
                n_act = 0; // the pivot it is
            else {
                acc = incl;
                u64 *t = cur_buf;
                cur = oth + 4 * static_cast<u64>(n_act - n_gt), cur_buf = oth, oth = t;
                n_act = n_gt;
            }
        }
        __syncthreads(); // the new lists are visible; red64 and warp_cnt may be reused
    }
    if (n_act > 0) { // the last 32: one record per lane, every warp for itself (as in pick_meet_warp)
        const u64 *w = cur + 4 * static_cast<u64>(lane_id());
        const bool have = lane_id() < n_act;
        const u64 key = have ? ld_cg(w) : ~0ull, wl = have ? ld_cg(w + 1) : 0ull, wh = have ? ld_cg(w + 2) : 0ull;
        const u32 oi = have ? static_cast<u32>(ld_cg(w + 3)) : 0u;
        const u32 chosen = warp_first_exceeding(key, wl, wh, n_act, acc, pick);
        if (chosen != 32u) // (else: cannot happen, the last pivot stands)
            ans = __shfl_sync(0xffffffffu, oi, chosen);
    }
    return ans;
}

// Meet set of a normally expanded final level: the contacts (in discovery order)
// whose other-side idx lies in [olo, ohi), written to meetbuf like meet_from_edges.
template <int BLOCK, int ITEMS>
__device__ u32 meet_from_contacts(const u32 *contact, u32 contact_n, const SideRegs &ex, u32 olo, u32 ohi,
                                  u32 *meetbuf, BlockShared<BLOCK, ITEMS> &sh) {
    const u32 tid = threadIdx.x;
    u32 count = 0;
    for (u32 c0 = 0; c0 < contact_n; c0 += BLOCK) {
        const u32 c = c0 + tid;
        bool in[1] = {false};
        u32 ei = 0, oi = 0;
        if (c < contact_n) {
            oi = ld_cg(contact + 2 * static_cast<u64>(c) + 1);
            in[0] = oi - olo < ohi - olo;
            if (in[0])
                ei = ld_cg(contact + 2 * static_cast<u64>(c));
        }
        u32 rank[1];
        const u32 tot = block_ranks<BLOCK, 1>(in, rank, sh.warp_cnt);
        if (in[0]) {
            const u64 sg = ld_cg(ex.pp->sig + ei);
            u32 *w = meetbuf + 4 * static_cast<u64>(count + rank[0]);
            st_cg(w + 0, ld_cg(ex.pp->list + ei));
            st_cg(w + 1, oi);
            st_cg(w + 2, static_cast<u32>(sg));
            st_cg(w + 3, static_cast<u32>(sg >> 32));
        }
        count += tot;
        __syncthreads();
    }
    __syncthreads();
    return count;
}

// One sigma-weighted step chain from `u` (at depth d on side `x`) to the side's
// root (sampler.cpp:135-155).  Emits every vertex strictly between into the
// frame and, optionally, into path_out[pos], pos advancing by pos_step.
//
// predecessors(u) = { w in N(u) : visited(w) && dist[w] + 1 == dist[u] }
//                 = N(u) ∩ level(d-1), chosen in CSR (= ascending id) order.
// They are enumerated either by scanning the row of u and testing each label
// against the idx range of level d-1, or -- when level d-1 is much smaller than
// the row, the common case for hub vertices -- by binary-searching every vertex
// of level d-1 in the sorted row.  Both yield the same set with the same row
// positions, hence the same pick.
template <int BLOCK, int ITEMS>
__device__ void walk_side(const SamplerParams &p, const u32 *lab, int x, const SideRegs &sd, u32 u, u32 d,
                          SampleStream &rng, u32 *path_out, long long pos, int pos_step, u32 &emitted,
                          BlockShared<BLOCK, ITEMS> &sh, WorkRegs &wk) {
    const u32 tid = threadIdx.x;
    while (d > 0) {
        const u64 beg = __ldg(p.offsets + u), end = __ldg(p.offsets + u + 1);
        if (tid == 0) {
            EBC_STAT(sh.ws[kW_S_walk] += 1;)
            EBC_STAT(sh.ws[kW_E_walk] += end - beg;)
        }
        u32 chosen = u;
        if (d == 1) {
            // the only vertex at depth 0 is the root and sigma[root] == 1: total = 1, r = 0
            (void)uniform_below_u128(rng, 1);
            chosen = ld_cg(sd.pp->list);
            if (tid == 0)
                EBC_STAT(wk.p_walk += 1;)
        } else {
            const u32 lo = ld_cg(sd.pp->lvl + (d - 1)), hi = ld_cg(sd.pp->lvl + d);
            const u32 span = hi - lo;
            const u64 degu = end - beg;
            if (tid == 0)
                sh.pred_cnt = 0;
            __syncthreads();
            // pass 1 (sampler.cpp:138-141): total = sum of sigma over predecessors
            u128 total_local = 0;
            const bool by_level = static_cast<u64>(span) * (66 - __clzll(degu)) < degu;
            if (by_level) {
                // rows are ascending in EXTERNAL ids: search the uploaded graph's row of u
                const u64 xbeg = __ldg(p.ext_offsets + ext_id(p, u)), xend = xbeg + degu;
                // A hub's row is searched by every vertex of the level: the first steps of all those searches -- a
                // dozen dependent loads each -- are taken in a table of kSplit evenly spaced entries of the row,
                // fetched once by the CTA (in f_v, which only the meet phase uses).
                constexpr u32 kSplit = 64;
                static_assert(kSplit <= FinalEdgeCap<BLOCK>::value, "splitter table aliases f_v");
                const bool split = degu >= 16 * kSplit;
                if (split) {
                    for (u32 j = tid; j < kSplit; j += BLOCK)
                        sh.f_v[j] = __ldg(p.ext_targets + xbeg + (static_cast<u64>(j) * degu) / kSplit);
                    __syncthreads();
                }
                for (u32 i = lo + tid; i < hi; i += BLOCK) {
                    const u32 w = ld_cg(sd.pp->list + i);
                    const u32 wx = ext_id(p, w);
                    u64 a = xbeg, b = xend; // lower_bound of w in the row of u
                    if (split) {
                        if (wx < sh.f_v[0]) {
                            b = a; // before the row's first entry
                        } else {
                            u32 jl = 0, jh = kSplit; // last j with f_v[j] <= wx
                            while (jh - jl > 1) {
                                const u32 jm = (jl + jh) >> 1;
                                if (sh.f_v[jm] <= wx)
                                    jl = jm;
                                else
                                    jh = jm;
                            }
                            a = xbeg + (static_cast<u64>(jl) * degu) / kSplit;
                            b = jl + 1 < kSplit ? xbeg + (static_cast<u64>(jl + 1) * degu) / kSplit + 1 : xend;
                            b = b < xend ? b : xend;
                        }
                    }
                    while (a < b) {
                        const u64 mid = (a + b) >> 1;
                        if (__ldg(p.ext_targets + mid) < wx)
                            a = mid + 1;
                        else
                            b = mid;
                    }
                    if (a < xend && __ldg(p.ext_targets + a) == wx) {
                        const u64 sg = ld_cg(sd.pp->sig + i);
                        total_local += sg;
                        EBC_STAT(wk.p_walk += 1;)
                        const u32 slot = atomicAdd(&sh.pred_cnt, 1u);
                        if (slot < kPredCache) {
                            sh.pred_pos[slot] = static_cast<u32>(a - xbeg);
                            sh.pred_sig[slot] = sg;
                            sh.pred_vtx[slot] = w;
                        }
                    }
                }
            } else {
                for (u64 k = beg + tid; k < end; k += BLOCK) {
                    const u32 w = __ldg(p.targets + k);
                    const u32 rel = label_idx(ld_cg(lab + w), sd.base, x) - lo;
                    if (rel < span) {
                        const u64 sg = ld_cg(sd.pp->sig + lo + rel);
                        total_local += sg;
                        EBC_STAT(wk.p_walk += 1;)
                        const u32 slot = atomicAdd(&sh.pred_cnt, 1u);
                        if (slot < kPredCache) {
                            sh.pred_pos[slot] = static_cast<u32>(k - beg);
                            sh.pred_sig[slot] = sg;
                            sh.pred_vtx[slot] = w;
                        }
                    }
                }
            }
            u64 tlo, thi, tov;
            block_sum_u128<BLOCK>(total_local, tlo, thi, tov, sh.red64);
            const u128 total = (static_cast<u128>(thi) << 64) | tlo; // < 2^96, cannot overflow
            __syncthreads();
            const u32 npred = sh.pred_cnt;
            const u128 r = uniform_below_u128(rng, total); // sampler.cpp:142
            if (npred <= kPredCache) {
                // pass 2 on the cached predecessors, in CSR order (sampler.cpp:143-151)
                if (tid < kPredCache) {
                    const bool have = tid < npred;
                    const u32 mypos = have ? sh.pred_pos[tid] : 0xffffffffu;
                    const u64 mysig = have ? sh.pred_sig[tid] : 0;
                    u128 before = 0;
#pragma unroll 1
                    for (u32 q = 0; q < npred; ++q)
                        if (sh.pred_pos[q] < mypos)
                            before += sh.pred_sig[q];
                    if (have && before <= r && r - before < mysig)
                        sh.bcast[0] = sh.pred_vtx[tid];
                }
                __syncthreads();
                chosen = sh.bcast[0];
            } else {
                // pass 2 by re-scanning the row in order with a block-wide prefix search
                u128 running = 0;
                bool running_ovf = false;
                for (u64 k0 = beg; k0 < end; k0 += BLOCK) {
                    const u64 k = k0 + tid;
                    u128 wv = 0;
                    u32 w = 0;
                    if (k < end) {
                        w = __ldg(p.targets + k);
                        const u32 rel = label_idx(ld_cg(lab + w), sd.base, x) - lo;
                        if (rel < span)
                            wv = ld_cg(sd.pp->sig + lo + rel);
                    }
                    const u32 f = block_first_exceeding<BLOCK>(wv, running, running_ovf, r, sh.red64, &sh.found_lane);
                    if (f != BLOCK) {
                        if (tid == f)
                            sh.bcast[0] = w;
                        __syncthreads();
                        chosen = sh.bcast[0];
                        break;
                    }
                }
            }
            __syncthreads();
        }
        u = chosen;
        d -= 1;
        if (d > 0) { // sampler.cpp:152-153: endpoints are never counted
            if (tid == 0) {
                const u32 ux = ext_id(p, u);
                atomicAdd(p.frame + 1 + ux, 1u); // apply_sample (sampler.hpp:77)
                if (path_out && pos >= 0 && static_cast<u64>(pos) < p.path_stride)
                    path_out[pos] = ux; // longer paths are truncated to path_stride entries
            }
            pos += pos_step;
            emitted += 1;
        }
    }
}

// walk_side for graphs with fixed-stride rows: a row has at most eight entries, so lane k of EVERY warp takes entry k
// (the warps compute the same step redundantly: no shared memory, no block barrier, and the random stream -- which
// all threads advance alike -- needs no broadcast).  Per step three dependent trips: the row (one sector), the labels
// of its targets, sigma of the predecessors; the pick is an 8-lane prefix scan in row (= CSR) order (sampler.cpp:139-151).
template <int BLOCK, int ITEMS, int RW>
__device__ void walk_side_ell(const SamplerParams &p, const u32 *lab, int x, const SideRegs &sd, u32 u, u32 d,
                              SampleStream &rng, u32 *path_out, long long pos, int pos_step, u32 &emitted,
                              BlockShared<BLOCK, ITEMS> &sh, WorkRegs &wk) {
    const u32 tid = threadIdx.x;
    const u32 k = lane_id();
    const u32 *lvl = sd.pp->lvl;
    const u64 *sig = sd.pp->sig;
    const u32 base = sd.base;
    (void)sh;
    (void)wk;
    while (d > 0) {
        u32 chosen;
        if (d == 1) {
            // the only vertex at depth 0 is the root and sigma[root] == 1: total = 1, r = 0
            (void)uniform_below_u128(rng, 1);
            chosen = ld_cg(sd.pp->list);
            EBC_STAT(if (tid == 0) {
                sh.ws[kW_S_walk] += 1;
                sh.ws[kW_E_walk] += __ldg(p.offsets + u + 1) - __ldg(p.offsets + u);
                wk.p_walk += 1;
            })
        } else {
            const u32 lo = ld_cg(lvl + (d - 1)), span = ld_cg(lvl + d) - lo;
            const u32 ent = k < RW ? __ldg(p.ell + RW * static_cast<u64>(u) + k) : kEllEmpty;
            const u32 w = ent & kEllIdMask;
            u64 sg = 0;
            bool pred = false;
            if (ent != kEllEmpty) {
                const u32 rel = label_idx(ld_cg(lab + w), base, x) - lo;
                pred = rel < span;
                if (pred)
                    sg = ld_cg(sig + lo + rel);
            }
            EBC_STAT(if (tid < 32) {
                const u32 entries = __popc(__ballot_sync(0xffffffffu, ent != kEllEmpty));
                if (tid == 0) {
                    sh.ws[kW_S_walk] += 1;
                    sh.ws[kW_E_walk] += entries;
                }
                wk.p_walk += pred ? 1 : 0;
            })
            // inclusive prefix of sigma over the lanes (at most 8 x (2^64 - 1): 67 bits)
            u64 plo = sg;
            u32 phi = 0;
#pragma unroll
            for (int o = 1; o < RW; o <<= 1) {
                const u64 tlo = __shfl_up_sync(0xffffffffu, plo, o);
                const u32 thi = __shfl_up_sync(0xffffffffu, phi, o);
                if (k >= static_cast<u32>(o)) {
                    const u64 nlo = plo + tlo;
                    phi += thi + (nlo < plo ? 1u : 0u);
                    plo = nlo;
                }
            }
            const u64 tot_lo = __shfl_sync(0xffffffffu, plo, RW - 1);
            const u32 tot_hi = __shfl_sync(0xffffffffu, phi, RW - 1);
            const u128 total = (static_cast<u128>(tot_hi) << 64) | tot_lo;
            const u128 r = uniform_below_u128(rng, total); // sampler.cpp:142
            const u128 mine = (static_cast<u128>(phi) << 64) | plo;
            const u32 hit = __ballot_sync(0xffffffffu, pred && mine > r) & ((1u << RW) - 1);
            chosen = __shfl_sync(0xffffffffu, w, __ffs(hit) - 1); // first prefix above r (a predecessor exists: total > 0)
        }
        u = chosen;
        d -= 1;
        if (d > 0) { // sampler.cpp:152-153: endpoints are never counted
            if (tid == 0) {
                const u32 ux = ext_id(p, u);
                atomicAdd(p.frame + 1 + ux, 1u); // apply_sample (sampler.hpp:77)
                if (path_out && pos >= 0 && static_cast<u64>(pos) < p.path_stride)
                    path_out[pos] = ux; // longer paths are truncated to path_stride entries
            }
            pos += pos_step;
            emitted += 1;
        }
    }
}

// Resident CTAs per SM the kernel is compiled for (register budget = 65536 / (BLOCK * this)).
// Measured on config 2 (profiles/r01_occupancy_sweep.txt): 16 -> 3.26M, 24 -> 3.80M, 32 -> 3.88M,
// 40 -> 3.68M, 48 -> 2.99M samples/s.  The kernel is latency bound, so resident warps matter more than
// the spills a 64-register budget causes.
#ifndef EBC_WARPS_PER_SM
#define EBC_WARPS_PER_SM 32
#endif
#ifndef EBC_FIXED_WARPS_PER_SM
#define EBC_FIXED_WARPS_PER_SM 32
#endif
template <int BLOCK, int FIXED> constexpr int min_blocks_per_sm() {
    constexpr int warps = FIXED ? EBC_FIXED_WARPS_PER_SM : EBC_WARPS_PER_SM;
    return (warps * 32) / BLOCK > 0 ? (warps * 32) / BLOCK : 1;
}

// BITS: the launch uses visited bitmaps (kFlagUseBitmap); a template parameter so that each kernel
// carries only its own variant of the probe code -- the instruction footprint matters, see above.
// FIXED: the graph has fixed-stride rows (SamplerParams::ell).  That kernel consists of expand_level_ell, the
// contact-list meet and the walk only -- no read-only probe (a lattice-like search does not end in a level much
// wider than the ones before), no general expansion, no bitmaps: a third of the instruction footprint.
template <int BLOCK, int ITEMS, bool BITS, int FIXED = 0>
__global__ void __launch_bounds__(BLOCK, min_blocks_per_sm<BLOCK, FIXED>()) sample_kernel(const SamplerParams p) {
    static_assert(!(FIXED && BITS) && (!FIXED || BLOCK <= 128), "fixed-stride rows: no bitmaps, at most 128 threads");
    __shared__ BlockShared<BLOCK, ITEMS> sh;
    __shared__ u32 vf[BITS ? VisitedFilter<BLOCK>::kWords : 1]; // visited filter of the sample in flight
    const u32 tid = threadIdx.x;
    if (BITS)
        for (u32 i = tid; i < VisitedFilter<BLOCK>::kWords; i += BLOCK)
            vf[i] = 0;
    if (p.reserved_sms) { // (before a slot is taken; uniform over the CTA)
        u32 smid, nsmid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        asm volatile("mov.u32 %0, %%nsmid;" : "=r"(nsmid));
        if (smid + p.reserved_sms >= nsmid) {
            // A reserved SM: hold the place until the rest of the grid is running elsewhere, then leave.  Should that
            // never happen (about a second), sample here after all: progress does not depend on CTA placement.
            if (tid == 0) {
                const long long t0 = clock64();
                u32 seen;
                while ((seen = *reinterpret_cast<volatile u32 *>(p.started)) < p.reserve_target && clock64() - t0 < (1ll << 31))
                    __nanosleep(2000);
                sh.bcast[2] = seen >= p.reserve_target ? 1u : 0u;
            }
            __syncthreads();
            if (sh.bcast[2])
                return;
            __syncthreads();
        } else if (tid == 0) {
            atomicAdd(p.started, 1u);
        }
    }
    // Slot hand-out.  Launches of consecutive epochs overlap on two streams, so a CTA cannot own
    // slot blockIdx.x: it takes a free slot id from a ring (at most ring_size CTAs are resident, each
    // holds one slot, so a free one is always there or about to be returned) and puts it back at exit.
    u64 slot = p.slot_base + blockIdx.x;
    if (p.ring) {
        if (tid == 0) {
            u32 got = 0xffffffffu;
            while (got == 0xffffffffu) {
                const unsigned long long h = atomicAdd(p.ring_pos, 1ull);
                got = atomicExch(p.ring + (static_cast<u32>(h) % p.ring_size), 0xffffffffu); // (any position works)
            }
            __threadfence();
            sh.bcast[2] = got;
        }
        __syncthreads();
        slot = sh.bcast[2];
    }
    const u64 n = p.n;
    u64 ticket_count = p.count;
    if (p.count_ptr) {
        const u64 listed = *p.count_ptr;
        ticket_count = listed < ticket_count ? listed : ticket_count;
    }

    SideRegs side[2];
    for (int k = 0; k < 2; ++k) {
        if (tid == 0) {
            if (k == 0) {
                sh.lab = p.lab + slot * n; // one label per vertex
                sh.bits = BITS ? p.bits + slot * 2 * p.bit_words : nullptr;
                sh.contact = p.contact + slot * 6 * p.aux_cap; // 2*aux_cap words: contacts / contact edges
                sh.meetbuf = sh.contact + 2 * p.aux_cap;       // 4*aux_cap words: ordered meet set
            }
            sh.sp[k].list = p.list + (slot * 2 + k) * p.cap;
            sh.sp[k].sig = p.sig + (slot * 2 + k) * p.cap;
            sh.sp[k].lvl = p.lvl + (slot * 2 + k) * (p.aux_cap + 2);
            sh.sp[k].pm = FIXED ? p.pm + (slot * 2 + k) * p.pm_words : nullptr;
        }
        side[k].pp = &sh.sp[k];
        side[k].base = ld_cg(p.hdr + slot * kHdrWords + kHdrBase0); // written by another SM's CTA
    }
    __syncthreads();
    auto edge_cap = [&]() -> u32 { // contact edges the probe may collect (recomputed: not worth a register)
        return static_cast<u32>((2 * p.aux_cap) / 6);
    };
    WorkRegs wk;
    u64 tot_e_lvl = 0, tot_p_walk = 0;
    if (tid == 0)
        for (int c = 0; c < kWorkCounters; ++c)
            sh.wk[c] = 0;
    if (tid == 0)
        for (int c = 0; c < 6; ++c)
            EBC_STAT(sh.last[c] = 0;)
#ifdef EBC_PHASE_TIMERS // experiment only: cycles per phase replace the work counters
    long long ph[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}; // 7: large meet sets, 8: small ones, 9: pick, 10: number of large ones
    long long ph_t = clock64();
#define EBC_PH(i)                         \
    {                                     \
        const long long ph_n = clock64(); \
        ph[i] += ph_n - ph_t;             \
        ph_t = ph_n;                      \
    }
#else
#define EBC_PH(i)
#endif

    for (;;) {
        if (tid == 0)
            sh.ticket = atomicAdd(p.ticket, 1ull);
        __syncthreads();
        const u64 ticket = sh.ticket;
        __syncthreads();
        if (ticket >= ticket_count)
            break;
        const u64 local = p.relist ? p.relist[ticket] : ticket;
        const u64 index = p.first + local;

        // ---- label-space housekeeping: labels must stay below the claim range ----
        {
            const u64 limit = static_cast<u64>(kClaimTop) - kMaxTileSlots - 4;
            if (static_cast<u64>(side[0].base) + 2 * p.cap + 2 >= limit) { // the sample's labels reach base + 2 cap + 1
                for (u64 i = tid; i < n; i += BLOCK)
                    st_cg(sh.lab + i, 0u);
                side[0].base = side[1].base = 1;
                __syncthreads();
            }
        }

        // ---- (s, t): sample_pair (sampler.cpp:45-52) ----
        SampleStream rng(p.seed, p.tag, index);
        u32 s, t;
        if (p.pairs) {
            s = p.pairs[2 * local];
            t = p.pairs[2 * local + 1];
        } else {
            const u64 a = rng.next_below(n);
            u64 b = rng.next_below(n - 1);
            if (b >= a)
                ++b;
            s = static_cast<u32>(a);
            t = static_cast<u32>(b);
        }
        [[maybe_unused]] const u32 s_ext = s, t_ext = t; // (for the record)
        if (p.to_dense) {
            s = __ldg(p.to_dense + s);
            t = __ldg(p.to_dense + t);
        }

        // ---- init both sides (sampler.cpp:65-76) ----
        for (int k = 0; k < 2; ++k) {
            const u32 root = k == 0 ? s : t;
            side[k].cnt = 1;
            side[k].fb = 0;
            side[k].depth = 0;
            side[k].pending = __ldg(p.offsets + root + 1) - __ldg(p.offsets + root);
            if (tid == 0) {
                st_cg(sh.lab + root, make_label(side[k].base, 0, k));
                if (BITS) {
                    red_or_u32(sh.bits + 2 * static_cast<u64>(root >> 5) + k, 1u << (root & 31));
                    filter_insert<BLOCK>(vf, root);
                }
                st_cg(side[k].pp->list, root);
                st_cg(side[k].pp->sig, static_cast<u64>(1));
                st_cg(side[k].pp->lvl, 0u);
                if (FIXED)
                    st_cg(side[k].pp->pm, 0u); // a root has no parents
            }
        }
        if (tid == 0) {
            for (int c = 0; c < kWorkCounters; ++c)
                EBC_STAT(sh.ws[c] = 0;)
            EBC_STAT(sh.ws[kW_V_set] = 2;)
            EBC_STAT(sh.ws[kW_samples] = 1;)
            sh.sigma_small[0] = sh.sigma_small[1] = 1; // sigma[root] = 1
            sh.prev_pending[0] = sh.prev_pending[1] = 0;
        }
        wk.e_lvl = 0;
        wk.p_walk = 0;
        __syncthreads();

#if EBC_STATS
        if (tid == 0) { // the sample's record is kept in shared memory, written by thread 0 only
            SampleRecordDev &rec = sh.rec;
            rec.s = s_ext;
            rec.t = t_ext;
            rec.dist = 0xffffffffu;
            rec.meet = 0xffffffffu;
            rec.meet_count = 0;
            rec.path_len = 0;
            rec.flags = 0;
            rec.weight_lo = rec.weight_hi = 0;
        }
#endif

        // ---- level loop (sampler.cpp:81-116) ----
        EBC_PH(0)
        bool found = false, aborted = false, probed = false;
        bool scratch_ready = false; // the last probe cleared pick_meet_large's scratch entries
        int e = 0;
        u32 contact_n = 0, edge_n = 0;
        while (!found) {
            if (side[0].cnt == side[0].fb || side[1].cnt == side[1].fb)
                break; // a frontier ran empty: t unreachable, empty sample (sampler.cpp:82-83)
            e = side[0].pending <= side[1].pending ? 0 : 1; // tie -> forward (sampler.cpp:84)
            // A probe that finds no contact is a wasted scan of the level, so it is only tried where the
            // level can plausibly be the last one: on a side whose frontier at least doubled.  Searches in
            // expanding graphs (R-MAT, Erdos-Renyi) end in their widest level; on lattice-like graphs the
            // frontier grows by a few per cent per level, almost no level is the last, and probing every wide
            // level cost config 3 a quarter of its time.
            if constexpr (!FIXED)
            if (!(p.flags & kFlagMaterializeFinal) && edge_cap() > 0 && side[e].pending >= p.probe_min_slots &&
                4 * side[e].pending >= p.probe_growth_x4 * sh.prev_pending[e] &&
                static_cast<u64>(side[e].depth) + 2 <= p.aux_cap) {
                u64 new_slots = 0, total_slots = 0;
                // (scratch of pick_meet_large behind both sides' sigma arrays, if there is room for it)
                const u64 o_front = side[1 - e].cnt - side[1 - e].fb;
                scratch_ready = BITS && o_front + side[e].cnt <= p.cap && o_front + side[1 - e].cnt <= p.cap;
                edge_n = probe_level<BLOCK, ITEMS, BITS>(p, sh.lab, sh.bits, vf, e, side[e], side[1 - e], sh.contact, edge_cap(), sh,
                                                         new_slots, total_slots,
                                                         scratch_ready ? side[e].pp->sig + side[e].cnt : nullptr,
                                                         scratch_ready ? side[1 - e].pp->sig + side[1 - e].cnt : nullptr);
                EBC_PH(2)
                bool resolvable = edge_n > 0 && edge_n <= edge_cap();
                if (resolvable && edge_n > static_cast<u32>(FinalEdgeCap<BLOCK>::value)) {
                    // pick_meet_large needs ohi - olo scratch words behind both sides' sigma arrays
                    const SideRegs &ot = side[1 - e];
                    u32 best = ot.depth;
                    while (ld_cg(ot.pp->lvl + best) > sh.min_contact)
                        --best;
                    const u64 span = (best == ot.depth ? ot.cnt : ld_cg(ot.pp->lvl + best + 1)) - ld_cg(ot.pp->lvl + best);
                    resolvable = span + side[e].cnt <= p.cap && span + ot.cnt <= p.cap;
                }
                if (resolvable) {
                    // final level: account its scan, open the (virtual) level for the walk, stop
                    EBC_STAT(wk.e_lvl += new_slots;)
                    if (tid == 0) {
                        EBC_STAT(sh.ws[kW_E_bfs] += total_slots;)
                        EBC_STAT(sh.ws[kW_V_exp] += side[e].cnt - side[e].fb;)
                        EBC_STAT(sh.ws[kW_levels] += 1;)
                        st_cg(side[e].pp->lvl + side[e].depth + 1, side[e].cnt);
                    }
                    __syncthreads();
                    probed = true;
                    found = true;
                    break;
                }
                if (tid == 0 && edge_n > 0)
                    sh.rec.flags |= 4u; // the probe found more contact edges than it can resolve
                __syncthreads(); // no sh.contact (or too many sh.contact edges): expand normally
            }
            bool ok;
            if constexpr (FIXED) // (also takes the new frontier's pending edges)
                ok = expand_level_ell<BLOCK, ITEMS, FIXED>(p, sh.lab, e, side[e], side[1 - e], sh.contact, contact_n, sh, wk);
            else
                ok = expand_level<BLOCK, ITEMS, BITS>(p, sh.lab, sh.bits, vf, e, side[e], side[1 - e], sh.contact, contact_n, sh, wk);
            if (!ok) {
                aborted = true;
                break;
            }
            EBC_PH(1)
            found = sh.min_contact != 0xffffffffu;
            if constexpr (!FIXED) {
                if (!found) { // next_pending (sampler.cpp:95,102); evaluated fused into the level it was 3 % slower
                    if (tid == 0)
                        sh.prev_pending[e] = side[e].pending; // (read after the barriers of sum_frontier_degrees)
                    side[e].pending = sum_frontier_degrees<BLOCK>(p, side[e], sh.red64, &sh.sigma_small[e]);
                } else
                    __syncthreads();
            }
            EBC_PH(3)
        }

        if (aborted) {
            if (tid == 0) {
                EBC_STAT(sh.rec.flags |= 1u;)
                const u32 k = atomicAdd(p.overflow_count, 1u);
                if (k < p.overflow_cap)
                    p.overflow_list[k] = static_cast<u32>(local);
                atomicAdd(p.overflow_total, 1ull);
            }
        } else if (found) {
            SideRegs &ex = side[e];
            SideRegs &ot = side[1 - e];
            const u32 d_ex = probed ? ex.depth + 1 : ex.depth; // depth of the level that touched the other side
            // best = min other.dist over contacts = level of the smallest other-side idx
            const u32 min_idx = sh.min_contact;
            u32 best = ot.depth;
            while (ld_cg(ot.pp->lvl + best) > min_idx)
                --best;
            const u32 olo = ld_cg(ot.pp->lvl + best);
            const u32 ohi = best == ot.depth ? ot.cnt : ld_cg(ot.pp->lvl + best + 1);
            if (tid == 0) {
                EBC_STAT(sh.rec.dist = d_ex + best;)
                if (probed)
                    EBC_STAT(sh.rec.flags |= 2u;)
            }
            __syncthreads();

            u32 meet_count = 0;
            u128 total_weight = 0;
            u32 meet = 0xffffffffu;
            bool searched = false; // a large probed level: the meet vertex is selected, the set is never ordered
            EBC_STAT(if (tid == 0 && probed && edge_n > static_cast<u32>(FinalEdgeCap<BLOCK>::value)) sh.rec.flags |= 8u;) // resolved in global memory
            if constexpr (!FIXED) {
                if (probed && edge_n <= 32) {
                    meet = pick_meet_warp(sh.contact, edge_n, olo, ohi, ot.pp->sig, rng, meet_count, total_weight);
                    searched = true;
                    EBC_STAT(if (tid == 0) sh.rec.flags |= 16u;)
                }
            }
            if constexpr (!FIXED)
                if (probed && edge_n > static_cast<u32>(FinalEdgeCap<BLOCK>::value)) {
                    const u32 oi = pick_meet_large<BLOCK, ITEMS>(sh.contact, edge_n, olo, ohi, ex.pp->sig + ex.cnt, ot.pp->sig + ot.cnt,
                                                                 ot.pp->sig, sh.sigma_small[e] != 0, scratch_ready && olo == ot.fb, rng, sh,
                                                                 meet_count, total_weight
#ifdef EBC_PHASE_COUNTS
                                                                 , ph + 8
#endif
                                                                 );
                    meet = ld_cg(ot.pp->list + oi); // (a member's other-side idx names it)
                    searched = true;
                    EBC_PH(7)
#ifdef EBC_PHASE_TIMERS
                    ph[10] += 1;
#endif
                }
            if (!searched) {
            // meet set in discovery order (sampler.cpp:109-113) -> sh.meetbuf
            if constexpr (FIXED)
                meet_count = meet_from_contacts<BLOCK, ITEMS>(sh.contact, contact_n, ex, olo, ohi, sh.meetbuf, sh);
            else
                meet_count = !probed ? meet_from_contacts<BLOCK, ITEMS>(sh.contact, contact_n, ex, olo, ohi, sh.meetbuf, sh)
                                     : meet_from_edges<BLOCK, ITEMS>(sh.contact, edge_n, olo, ohi, sh.meetbuf, sh);
#ifndef EBC_PHASE_COUNTS
            EBC_PH(8)
#endif

            // total weight over the meet set (sampler.cpp:121-123), saturating at 2^128-1
            u128 wsum = 0;
            for (u32 c = tid; c < meet_count; c += BLOCK) {
                const u32 *w = sh.meetbuf + 4 * static_cast<u64>(c);
                const u64 sg = static_cast<u64>(ld_cg(w + 2)) | (static_cast<u64>(ld_cg(w + 3)) << 32);
                wsum += static_cast<u128>(sg) * ld_cg(ot.pp->sig + ld_cg(w + 1));
            }
            u64 wlo, whi, wov;
            block_sum_u128<BLOCK>(wsum, wlo, whi, wov, sh.red64);
            __syncthreads();
            total_weight = wov ? ~static_cast<u128>(0) : ((static_cast<u128>(whi) << 64) | wlo);

            // pick and ordered prefix search (sampler.cpp:124-133).  pick < total_weight <=
            // sum of the weights, so a hit always exists; the reference's fall-through
            // default (last meet vertex, sampler.cpp:125) is kept for completeness.
            const u128 pick = uniform_below_u128(rng, total_weight);
            {
                u128 running = 0;
                bool running_ovf = false;
                for (u32 c0 = 0; c0 < meet_count && meet == 0xffffffffu; c0 += BLOCK) {
                    const u32 c = c0 + tid;
                    u128 wv = 0;
                    u32 mv = 0;
                    if (c < meet_count) {
                        const u32 *w = sh.meetbuf + 4 * static_cast<u64>(c);
                        const u64 sg = static_cast<u64>(ld_cg(w + 2)) | (static_cast<u64>(ld_cg(w + 3)) << 32);
                        wv = static_cast<u128>(sg) * ld_cg(ot.pp->sig + ld_cg(w + 1));
                        mv = ld_cg(w);
                    }
                    const u32 f = block_first_exceeding<BLOCK>(wv, running, running_ovf, pick, sh.red64, &sh.found_lane);
                    if (f != BLOCK) {
                        if (tid == f)
                            sh.bcast[0] = mv;
                        __syncthreads();
                        meet = sh.bcast[0];
                        __syncthreads();
                    }
                }
                if (meet == 0xffffffffu)
                    meet = ld_cg(sh.meetbuf + 4 * static_cast<u64>(meet_count - 1));
            }
#ifndef EBC_PHASE_COUNTS
            EBC_PH(9)
#endif
            }
            if (tid == 0) {
                EBC_STAT(sh.rec.weight_lo = static_cast<u64>(total_weight);)
                EBC_STAT(sh.rec.weight_hi = static_cast<u64>(total_weight >> 64);)
                EBC_STAT(sh.rec.meet_count = meet_count;)
                EBC_STAT(sh.ws[kW_M] += meet_count;)
            }
            if (tid == 0)
                EBC_STAT(sh.rec.meet = ext_id(p, meet);)
            EBC_PH(4)

            // walks (sampler.cpp:157-163): path order s .. meet .. t
            const u32 d_ot = best;
            const u32 dist_f = e == 0 ? d_ex : d_ot; // depth of meet on the forward side
            const u32 dist_b = e == 0 ? d_ot : d_ex;
            u32 emitted = 0;
            // forward side: vertices at forward depth d sit at internal position d-1
#pragma unroll 1 // one copy of the walk in the instruction stream
            for (int x = 0; x < 2; ++x) {
                const SideRegs sd = x == 0 ? side[0] : side[1];
                if constexpr (FIXED)
                    walk_side_ell<BLOCK, ITEMS, FIXED>(p, sh.lab, x, sd, meet, x == 0 ? dist_f : dist_b, rng,
                                                p.paths ? p.paths + local * p.path_stride : nullptr,
                                                x == 0 ? static_cast<long long>(dist_f) - 2 : static_cast<long long>(dist_f),
                                                x == 0 ? -1 : +1, emitted, sh, wk);
                else
                walk_side<BLOCK, ITEMS>(p, sh.lab, x, sd, meet, x == 0 ? dist_f : dist_b, rng,
                                        p.paths ? p.paths + local * p.path_stride : nullptr,
                                        x == 0 ? static_cast<long long>(dist_f) - 2 : static_cast<long long>(dist_f),
                                        x == 0 ? -1 : +1, emitted, sh, wk);
                if (x == 0 && meet != s && meet != t) {
                    if (tid == 0) {
                        const u32 mx = ext_id(p, meet);
                        atomicAdd(p.frame + 1 + mx, 1u);
                        if (p.paths && static_cast<u64>(dist_f - 1) < p.path_stride)
                            p.paths[local * p.path_stride + (dist_f - 1)] = mx;
                    }
                    emitted += 1;
                }
            }
            if (tid == 0)
                EBC_STAT(sh.rec.path_len = emitted;)
            EBC_PH(5)
            if (tid == 0)
                EBC_STAT(sh.ws[kW_L] += emitted;)
        }

        // ---- apply_sample: tau += 1 (sampler.hpp:75); retire the sample's labels ----
        if (tid == 0)
            EBC_STAT(sh.rec.draws = rng.draws();)
        if (!aborted) {
            tot_e_lvl += wk.e_lvl;
            tot_p_walk += wk.p_walk;
            if (tid == 0) {
                atomicAdd(p.frame, 1u);
                for (int c = 0; c < kWorkCounters; ++c)
                    EBC_STAT(sh.wk[c] += sh.ws[c];)
            }
        }
        if (p.records && tid == 0)
            p.records[local] = sh.rec;
        if (BITS) { // clear the bitmap words of every settled vertex (both sides share the 8-byte word), and the filter
            for (u32 i = tid; i < VisitedFilter<BLOCK>::kWords; i += BLOCK)
                vf[i] = 0;
            u64 *bits64 = reinterpret_cast<u64 *>(sh.bits);
#pragma unroll 1
            for (int k = 0; k < 2; ++k) {
                const u32 c = k == 0 ? side[0].cnt : side[1].cnt;
                const u32 *lst = sh.sp[k].list;
                for (u32 i0 = 0; i0 < c; i0 += 4 * BLOCK) { // four independent loads in flight per thread
                    u32 w[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const u32 i = i0 + q * BLOCK + tid;
                        w[q] = i < c ? ld_cg(lst + i) >> 5 : 0xffffffffu;
                    }
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (w[q] != 0xffffffffu)
                            st_zero_sector(bits64 + (w[q] & ~3u));
                }
            }
        }
        for (int k = 0; k < 2; ++k) {
            if (tid == 0) {
                EBC_STAT(sh.last[k] = side[k].base;)
                EBC_STAT(sh.last[2 + k] = side[k].cnt;)
                EBC_STAT(sh.last[4 + k] = side[k].depth;)
            }
        }
        {
            const u32 used = side[0].cnt > side[1].cnt ? side[0].cnt : side[1].cnt;
            side[0].base += 2 * used;
            side[1].base = side[0].base;
        }
        __syncthreads();
        EBC_PH(6)
    }

    // ---- persist slot header and work counters ----
    if (tid == 0) {
        u32 *h = p.hdr + slot * kHdrWords;
        h[kHdrBase0] = side[0].base;
        h[kHdrBase1] = side[1].base;
        h[kHdrLastBase0] = sh.last[0];
        h[kHdrLastBase1] = sh.last[1];
        h[kHdrLastCnt0] = sh.last[2];
        h[kHdrLastCnt1] = sh.last[3];
        h[kHdrLastDepth0] = sh.last[4];
        h[kHdrLastDepth1] = sh.last[5];
    }
    const u64 e_lvl = block_sum_u64<BLOCK>(tot_e_lvl, sh.red64);
    __syncthreads();
    const u64 p_walk = block_sum_u64<BLOCK>(tot_p_walk, sh.red64);
    if (tid == 0 && sh.wk[kW_samples]) {
        sh.wk[kW_E_lvl] = e_lvl;
        sh.wk[kW_P_walk] = p_walk;
        for (int c = 0; c < kWorkCounters; ++c)
            atomicAdd(p.work + c, static_cast<unsigned long long>(sh.wk[c]));
#ifdef EBC_PHASE_TIMERS
        for (int c = 0; c < 11; ++c)
            atomicAdd(p.work + c, static_cast<unsigned long long>(ph[c]) - static_cast<unsigned long long>(sh.wk[c]));
#endif
    }
    if (p.ring) { // hand the slot back (its header and labels are written; make them visible first)
        __syncthreads();
        if (tid == 0) {
            __threadfence();
            for (;;) {
                const unsigned long long t = atomicAdd(p.ring_pos + 1, 1ull);
                if (atomicCAS(p.ring + (static_cast<u32>(t) % p.ring_size), 0xffffffffu, static_cast<u32>(slot)) == 0xffffffffu)
                    break;
            }
        }
    }
}

} // namespace EBC_VARIANT
} // namespace ebc

#undef EBC_VARIANT
#undef EBC_STAT
