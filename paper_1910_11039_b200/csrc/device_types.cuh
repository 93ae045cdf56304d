// Device-side data layout of the B200 KADABRA sampler ("Data
// layout in HBM").  Everything a sample needs lives in one *slot*; a slot is
// owned by exactly one resident CTA for the duration of a kernel.
#pragma once

#include <cstdint>

namespace ebc {

using u32 = std::uint32_t;
using u64 = std::uint64_t;

// Work counters; indices shared with the C ABI
// (ebc_sampler_work) and with the oracle's instrumented restatement.
enum WorkCounter : int {
    kW_E_bfs = 0,
    kW_E_lvl,
    kW_V_exp,
    kW_V_set,
    kW_F_chk,
    kW_M,
    kW_S_walk,
    kW_E_walk,
    kW_P_walk,
    kW_L,
    kW_levels,
    kW_samples,
    kWorkCounters
};

// Labels.  ONE u32 per vertex (both sides share it, see SideRegs in sampler_kernels.cuh) replaces the
// reference's per-side (stamp, dist, sigma) triple (sampler.hpp:39-54): label = base + 2 * idx + side,
// where idx is the vertex' position in the side's discovery-ordered settle list and base advances by
// twice the larger settled count after every sample (O(1) reset like SearchScratch::round_,
// sampler.cpp:63).  visited on side s <=> (label - base - s) even and (label - base - s) / 2 < settled
// count of s; dist is implied by idx (levels occupy contiguous idx ranges).
constexpr u32 kClaimTop = 0xffffffffu;     // transient claim values: kClaimTop - slot_in_tile
constexpr u32 kMaxBlockThreads = 1024;
constexpr u32 kMaxTileSlots = 4096;        // BLOCK * ITEMS never exceeds this
constexpr u32 kFlagUseBitmap = 2u;        // per-slot visited bitmaps are maintained and used by probe_level
constexpr u32 kFlagMaterializeFinal = 1u; // always settle the final level (state dumps, exact V_set / F_chk)
constexpr u32 kFlagStats = 4u;            // launch the kernels that keep work counters, sample records, paths and state-dump bookkeeping
constexpr u32 kEllWidth = 8;               // entries per fixed-stride row (SamplerParams::ell), at most ...
constexpr u32 kEllNarrow = 4;              // ... and on graphs of maximum degree <= 4 (SamplerParams::ell_width): 16-byte rows
constexpr u32 kEllRevShift = 26;           // bits 26..28 of an entry: position of the reverse arc in the target's row
constexpr u32 kEllDegShift = 29;           // bits 29..31: degree of the target, minus one
constexpr u32 kEllIdMask = (1u << kEllRevShift) - 1;
constexpr u32 kEllEmpty = 0xffffffffu;     // (a graph with fixed-stride rows has fewer than 2^26 - 1 vertices)
constexpr u32 kEllEscape = 0xfffffffeu;    // first word of a row of SamplerParams::ell4 whose vertex has more than four entries
constexpr u32 kHdrWords = 16;              // per-slot header (u32)
// header word indices
enum : int { kHdrBase0 = 0, kHdrBase1 = 1, kHdrLastBase0 = 2, kHdrLastBase1 = 3, kHdrLastCnt0 = 4,
             kHdrLastCnt1 = 5, kHdrLastDepth0 = 6, kHdrLastDepth1 = 7 };

struct SampleRecordDev { // mirrors ebc_sample_record
    u32 s, t, dist, meet, meet_count, draws, path_len, flags;
    u64 weight_lo, weight_hi;
};

struct SamplerParams {
    // graph (replicated CSR)
    u64 n;
    const u64 *offsets;
    const u32 *targets;
    // Hub-clustered numbering (optional).  The search state (labels, bitmaps) is indexed by DENSE ids:
    // vertices renumbered by descending degree, so the probes of hub targets share cache lines.
    // offsets/targets above are then the dense graph: row i = the row of vertex to_ext[i], its entries
    // in the ORIGINAL (ascending external id) order but holding dense ids, so discovery order, meet
    // order and row positions are those of the external graph.  ext_offsets/ext_targets are the graph
    // as uploaded (rows ascending), used to locate a vertex inside a row.  Without renumbering
    // to_dense == to_ext == nullptr and ext_* alias offsets/targets.
    const u32 *to_dense; // external id -> dense id
    const u32 *to_ext;   // dense id -> external id
    const u64 *ext_offsets;
    const u32 *ext_targets;
    // Fixed-stride rows (optional; symmetric graphs whose maximum degree is at most kEllWidth, e.g. grids and road
    // networks): ell[kEllWidth * v + k] = k-th entry of row v of the graph above, packed as
    // target | (position of v in the target's row) << 26 | (degree(target) - 1) << 29, or kEllEmpty behind the
    // row's end.  A row is one 32-byte sector at a computable address; the degree of a settled vertex comes with the
    // entry that discovered it, and the reverse position lets it remember which of its own entries lead back to
    // its discoverers (expand_level_ell in sampler_kernels.cuh).
    // ell_width = 8, or 4 when no row has more than four entries (a 2-D lattice): row v is then the 16 bytes at
    // ell + 4 v, two rows per sector, the whole table half the size (config 3: 64 MB, below the L2 capacity).
    const u32 *ell;
    u32 ell_width;
    // ell_width = 8 on a graph where FEW rows have more than four entries (a lattice with some shortcuts, config 3):
    // ell4[4 v ..] = the first four entries of row v (16 bytes, the 64 MB the expansion streams), or kEllEscape in
    // word 0 if the row is longer -- the expansion then reads the row in `ell`.  Null otherwise.
    const u32 *ell4;
    u32 *pm;       // [slots][2][pm_words] with fixed-stride rows: per settled vertex (indexed like list, one byte each)
                   // the mask of row entries that lead to its parents
    u64 pm_words;
    // slots
    u32 *lab;      // [slots][n]
    u32 *list;     // [slots][2][cap]   settled vertices in discovery order
    u64 *sig;      // [slots][2][cap]   sigma, same indexing
    u32 *lvl;      // [slots][2][aux_cap+2] level start offsets into list
    u32 *contact;  // [slots][6*aux_cap] contacts / contact edges, then the ordered meet set
    u32 *hdr;      // [slots][kHdrWords]
    u64 cap;                    // settled vertices per side (list, sig)
    u64 aux_cap;                // levels per side and contacts per sample (lvl, contact); <= cap
    // work
    u64 seed;
    u32 tag;
    u64 first;
    u64 count;
    unsigned long long *ticket; // dynamic sample dispenser
    u32 *frame;                 // epoch frame, n+1 u32 (word 0 = tau)
    const u32 *pairs;           // optional explicit (s,t) pairs, 2*count
    SampleRecordDev *records;   // optional
    u32 *paths;                 // optional, path_stride per sample
    u64 path_stride;
    unsigned long long *work;   // kWorkCounters
    u32 *overflow_list;         // local sample indices that overflowed slot capacity
    u32 *overflow_count;
    u32 overflow_cap;
    // re-run pass over an earlier launch's overflow list (large slots): local
    // sample index = relist[ticket], number of tickets = min(*count_ptr, count)
    const u32 *relist;
    const u32 *count_ptr;
    u64 slot_base;              // first slot used by this launch
    unsigned long long *overflow_total; // persistent count of abandoned samples of this pass
    u32 flags;                  // kFlag*
    u32 *bits;                  // [slots][2 * bit_words] visited bitmaps, bits[2*(v>>5) + side]
    u64 probe_growth_x4;        // ... and only if 4 x pending edges >= this x the pending edges of the side's previous level
    u64 probe_min_slots;        // a level with fewer adjacency slots is expanded without trying the read-only probe
    u64 bit_words;              // ceil(n / 32), rounded up to a multiple of 4 (32-byte sectors)
    // dynamic slot hand-out (main pass): ring of free slot ids, ring_pos = {head, tail}; null => slot = slot_base + blockIdx.x
    u32 *ring;
    u32 ring_size;
    unsigned long long *ring_pos;
    // Main pass only: CTAs that land on one of the last `reserved_sms` SMs do not sample.  They wait until
    // `reserve_target` CTAs of this launch have started on the other SMs -- all the grid minus what the reserved
    // SMs hold -- and leave; from then on those SMs are empty for a kernel of another stream (NCCL's all-reduce of
    // the previous epoch's frame).  (Leaving at once would drain the whole grid through the reserved SMs while the
    // other SMs are still held by the previous epoch's kernel.)
    u32 reserved_sms;
    u32 reserve_target;
    u32 *started; // CTAs of this launch that started on an SM that is not reserved
};

} // namespace ebc
