// kernels.cuh — the hot path, as an edge-centric gather + a vertex epilogue.
//
// Replaces the reference's iteration body (engine.hpp:177-241):
//   edge_kernel    gather fold (GG-Gather, engine.hpp:198-213) over the
//                  current list; in a superstep (kEdgeChain) also the
//                  influence + GG-EStatus of every processed edge into the
//                  active-edge bitmap (engine.hpp:204-211), with the carry
//                  into each task's continuing vertex from a look-back over
//                  the other tasks' published pieces (chain_carry);
//   edge_kernel_hot the approximate fold with the hottest message slots in
//                  shared memory (4-byte messages);
//   vertex_kernel  skip test (:196), GG-Apply / GG-VStatus / valid (:216-224),
//                  next = prev carry-over (:183), iteration counters.
//
// Layout (per rank): the list (full or sparsified CSC) is addressed by PADDED
// positions P = pad + local edge index, with pad chosen so that P equals the
// global position modulo kChunkEdges; sources/weights are stored at [P].
//   run  r = padded positions [16r, 16r+16): folded SEQUENTIALLY by one lane
//            (the reference's inner loop over that stretch); sources come in
//            as four aligned 128-bit loads, the 16 message gathers are issued
//            back to back (registers);
//   task t = runs [32t, 32t+32) = 512 positions = one warp. The task's
//            non-empty vertices' start offsets are staged in shared memory
//            (empty vertices are never visited); runs that share a
//            destination are joined by one segmented warp scan; vertices
//            that end inside the task get their final accumulator (acc_out),
//            the task's continuing head / tail pieces go to hv[t] / tv[t] and
//            are joined in task order by the vertex kernel.
// Every vertex's fold structure is therefore a function of global edge
// positions only: results are bitwise identical for any grid, launch order
// and GPU count (the analogue of test_engine.cpp:161-182).
#pragma once

#include <type_traits>

#include "common.cuh"

namespace ggb {

enum : int { kModeApprox = GG_MODE_APPROXIMATE, kModeAccurate = GG_MODE_ACCURATE,
             kModeSuperstep = GG_MODE_SUPERSTEP };

// status byte per position (ONE buffer: an iteration's kernels read the
// byte before its vertex kernel rewrites it; a skipped vertex's status is
// already 0, engine.hpp:196, so skipped vertices cost no write)
constexpr uint8_t kStActive = 1;     // vstatus result (engine.hpp:220)
constexpr uint8_t kStInvalid = 4;    // !valid(fresh) (deferred superstep check)
constexpr uint8_t kStWasActive = 8;  // superstep: the status before the iteration (engine.hpp:229)

// Per-iteration reductions (engine.hpp:186-189). Field groups are laid out
// for the multi-GPU allreduce: [u64 sum x2][u32 sum x3][u32 min].
struct IterCounters {
    unsigned long long gathered;
    unsigned long long processed;
    unsigned int changed;
    unsigned int any_invalid;
    unsigned int empty_active;  // some in-degree-0 vertex ended active (the next
                                // vertex kernel must walk those positions)
    unsigned int bad_min;       // smallest invalid vertex (global id), 0xffffffff = none
};

__global__ void reset_counters_kernel(IterCounters* __restrict__ c, int n);

// Device-side early exit inside a batch of enqueued iterations: the kernels
// of iteration u+1 return at once when iteration u changed nothing or hit an
// invalid property (engine.hpp:226-240). A skipped iteration leaves its
// (zeroed) counters "unchanged", so the rest of the batch is skipped too.
__device__ __forceinline__ bool stop_after(const IterCounters* prev) {
    if (!prev) return false;
    // written by an earlier kernel of the stream: the read-only path is
    // coherent here, and every warp after the first per SM hits in L1
    return __ldg(&prev->changed) == 0 || __ldg(&prev->bad_min) != 0xffffffffu;
}

// edge kernel flavours
enum : int {
    kEdgePlain = 0,  // every edge of the list belongs to a processed vertex
    kEdgeCheck = 1,  // full list, skip edges of unprocessed vertices
    kEdgeChain = 2,  // superstep in one pass: fold + influence / estatus, the carry
                     // into a task's continuing vertex from the chain (chain_carry)
};

// chain states (EdgeArgs::chain), per task, for the vertex continuing past it
constexpr uint32_t kChainPiece = 1;  // hv[t] holds the task's whole piece
constexpr uint32_t kChainIncl = 2;   // tv[t] holds its inclusive fold (from the vertex start)

// non-empty vertex starts of one task, relative to the task start, clamped
// to [-1, 513] (-1: began in an earlier task, 513: ends in a later one)
constexpr int kStageStarts = kChunkEdges + 2;

template <class P, class W>
struct EdgeArgs {
    P prog;
    const uint32_t* __restrict__ src;       // [padded position]; sparsified list: [sp_slot(position)]
    bool src_quads;                         // src is in sp_slot order (common.cuh)
    const W* __restrict__ w;                // [padded position]
    const uint32_t* __restrict__ run_i;     // [run] non-empty vertex at its first position
    const uint32_t* __restrict__ nz_row;    // [nz] row of the list's i-th non-empty vertex
                                            // (nullptr: the full list, row = i)
    const uint64_t* __restrict__ nz_start;  // [nz+1] local edge offset
    uint64_t pad, e_end;                    // valid padded positions [pad, e_end)
    uint64_t ntasks, nruns;
    const uint64_t* __restrict__ a_off;     // [R+1] active_in_degree offsets by row (engine.hpp:154-161)
    const uint8_t* __restrict__ st_cur;     // status by position
    const typename P::Message* __restrict__ msg_cur;  // global ids
    // Message-gather cache classes (hot-first slots: low ids are the most read):
    //   slot < hot_limit: L1 evict_last + L2 evict_last   (register-resident runs)
    //   slot < l2_limit:  L2 evict_last                    (heavy programs' runs)
    //   otherwise:        L1 no_allocate + L2 evict_normal, or (cold_last: the
    //                     whole array fits L2) as the first class
    uint32_t hot_limit;
    uint32_t l2_limit;
    uint32_t cold_last;
    typename P::Accum* __restrict__ acc_out;  // [row]
    typename P::Accum* __restrict__ hv;       // [task] continuing head piece
    typename P::Accum* __restrict__ tv;       // [task] continuing tail piece (chain: inclusive)
    // kEdgeChain: per task {state, value} (16-byte slots, accumulators of <= 8
    // bytes) or the state alone (values in hv / tv), and the task ticket
    ulonglong2* __restrict__ cdesc;
    uint32_t* __restrict__ chain;
    uint32_t* __restrict__ ticket;
    uint32_t* __restrict__ bitmap;          // [local edge / 32] active flags
    double theta;
    // theta * (1 +- 2^-40) (NaN when theta is not a normal positive number):
    // the division-free influence test of programs with relative-growth
    // influence (see rel_growth_flags)
    double theta_hi, theta_lo;
    // run > 0, finite, and run * theta_hi/lo inside [2^-998, 2^998], as one
    // unsigned test on the accumulator's high word: (hi32(run) - pn_lo) < pn_span
    // (pn_span = 0: never, every edge takes the exact walk)
    uint32_t pn_lo, pn_span;
    const IterCounters* stop_if;            // batched iterations: the previous iteration's counters
};

// Per-vertex run state is indexed by POSITION p (graph.cuh): rows (vertices
// with in-edges) at [0, nrows), in-degree-0 vertices at [nrows, nloc).
template <class P, class W>
struct VertexArgs {
    P prog;
    uint64_t n;
    uint32_t v_begin, nloc, nrows;
    const uint64_t* __restrict__ off;   // [nrows+1] offsets of the gathered list by row (unpadded)
    uint64_t pad;
    const uint64_t* __restrict__ a_off; // [nrows+1] active_in_degree offsets by row
    uint8_t* __restrict__ st;                         // status by position
    typename P::Property* __restrict__ prop;          // by position
    typename P::Message* __restrict__ msg;            // message slots (one buffer)
    const uint32_t* __restrict__ vid_of_p;            // local vertex of position p
    const uint32_t* __restrict__ slot_p;              // message slot of position p
    const uint32_t* __restrict__ deg_p;               // out-degree of position p
    const typename P::Accum* __restrict__ acc_out;    // [row]
    const typename P::Accum* __restrict__ hv;
    const typename P::Accum* __restrict__ tv;
    // Fused exchange (exchange.cuh): the message of a gathered slot s of this
    // rank (gb0 <= s < ge0 or gb1 <= s < ge1, out-degree > 0) is also stored
    // into every other rank's replica, peers[r] (npeers = 0: no fused exchange)
    typename P::Message* peers[kMaxPeers];
    int npeers, self;
    uint64_t gb0, ge0, gb1, ge1;
    IterCounters* __restrict__ ctr;
    IterCounters* __restrict__ ctr_next;              // reset here for the next iteration
    const IterCounters* ctr_prev;                     // the previous iteration's (empty_active)
    const IterCounters* stop_if;                      // see EdgeArgs::stop_if
};

__device__ __forceinline__ bool vertex_processed(const uint8_t* st, const uint64_t* a_off, uint32_t row) {
    return (st[row] & kStActive) || a_off[row + 1] > a_off[row];  // engine.hpp:196
}
template <class P, class W>
__device__ __forceinline__ uint32_t row_of(const EdgeArgs<P, W>& a, uint64_t i) {
    return a.nz_row ? a.nz_row[i] : (uint32_t)i;
}

// Fold loops are fully unrolled (messages stay in registers) unless the
// program's gather is long (BP: three f64 divisions and two passes over the
// states), where 2 x 16 inlined copies thrash the instruction cache; those
// loops run rolled over a local-memory message array.
template <class P>
__host__ __device__ constexpr int fold_unroll() {
    if constexpr (requires { P::kHeavyGather; }) return P::kHeavyGather ? 1 : kRun;
    else return kRun;
}
// f(j) for j = 0..kRun-1, unrolled per fold_unroll (a plain `#pragma unroll`
// for light programs: an explicit count changes ptxas's allocation).
template <class P, class F>
__device__ __forceinline__ void for_run(F&& f) {
    if constexpr (fold_unroll<P>() == 1) {
#pragma unroll 1
        for (int j = 0; j < kRun; ++j) f(j);
    } else {
#pragma unroll
        for (int j = 0; j < kRun; ++j) f(j);
    }
}

template <class W>
using WStore = std::conditional_t<std::is_void_v<W>, char, W>;

// Load this lane's sources (aligned run -> 4 x 128-bit) and issue its
// message gathers back to back.
// Shared-memory copy of the hottest message slots (edge_kernel_hot).
struct HotTable {
    uint32_t base = 0;  // shared-space address of slot 0
    uint32_t n = 0;     // slots [0, n) are in shared memory
};

// SQ: the list may be a sparsified one in sp_slot order (a.src_quads); false
// for the superstep kernels, which only ever walk the full list.
template <class P, class W, bool HOT = false, bool SQ = true>
__device__ __forceinline__ void load_run(const EdgeArgs<P, W>& a, uint64_t P0, uint64_t lo,
                                         uint64_t hi, typename P::Message (&m)[kRun],
                                         WStore<W> (&wr)[kRun], uint64_t pol_stream,
                                         uint64_t pol_hot, uint64_t pol_cold,
                                         HotTable ht = {}) {
    uint32_t s[kRun];
    if (lo == P0 && hi == P0 + kRun) {
        // sp_slot order: quad i of this lane's run at quad i * 32 + lane of the task block
        const bool quads = SQ && a.src_quads;
        const int L = (int)((P0 >> 4) & 31ull);
        const uint4* sp = quads ? reinterpret_cast<const uint4*>(a.src + (P0 & ~511ull))
                                : reinterpret_cast<const uint4*>(a.src + P0);
#pragma unroll
        for (int i = 0; i < kRun / 4; ++i) {
            uint4 q;
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
                         : "=r"(q.x), "=r"(q.y), "=r"(q.z), "=r"(q.w) : "l"(sp + (quads ? sp_quad(L, i) : i)), "l"(pol_stream));
            s[4 * i] = q.x; s[4 * i + 1] = q.y; s[4 * i + 2] = q.z; s[4 * i + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kRun; ++j) {
            const uint64_t p = P0 + j;
            s[j] = (p >= lo && p < hi)
                       ? ld_stream_u32(a.src + (SQ && a.src_quads ? sp_slot(p) : p), pol_stream) : 0u;
        }
    }
    // Every gather is issued unconditionally and independently (positions
    // outside [lo, hi) read slot 0, always L2-resident; their values are never
    // folded), so all 16 are in flight together. The weights of a run lie
    // inside the padded allocation.
#pragma unroll
    for (int j = 0; j < kRun; ++j) {
        if constexpr (HOT)
            m[j] = ld_msg_hot(a.msg_cur + s[j], ht.base + s[j] * (uint32_t)sizeof(typename P::Message),
                              s[j] < ht.n ? 0u : (s[j] < a.hot_limit ? 1u : 2u), pol_hot, pol_cold);
        else if constexpr (fold_unroll<P>() != 1)
            // (a message array that fits L2 takes the hot instruction for every
            // slot: the cold one does not allocate in L1)
            m[j] = ld_msg2(a.msg_cur + s[j], a.cold_last || s[j] < a.hot_limit, pol_hot, pol_cold);
        else
            m[j] = ld_msg(a.msg_cur + s[j], s[j] < a.l2_limit ? pol_hot : pol_cold);
        if constexpr (!std::is_void_v<W>) wr[j] = __ldg(a.w + P0 + j);
    }
}

// Rewrite the flags of a task's processed edges (lane bits `own`, relative
// to its run) to `kbits`; flags of edges of skipped vertices persist
// (engine.hpp:204-211). Warp-collective: the lanes' 16-bit fields are
// reassembled into bitmap words (word k of the task starts at task position
// 32k - q); a word that lies inside the task belongs to this warp alone and
// is stored (read-modify-write only where some of its flags persist), the
// two words shared with the neighbouring tasks take atomics.
__device__ __forceinline__ void warp_write_flags(uint32_t* __restrict__ bitmap, uint64_t pad,
                                                 uint64_t tstart, uint32_t own, uint32_t kbits,
                                                 int lane) {
    const int64_t b = (int64_t)tstart - (int64_t)pad;  // local edge id of task position 0
    const int64_t w0 = b >> 5;                          // floor
    const int q = (int)(b - (w0 << 5));
    const int s = 32 * lane - q;  // first task position of word w0 + lane
    const int l = s >> 4, off = s & 15;
    auto get = [&](uint32_t v, int src) -> uint64_t {
        const uint32_t x = __shfl_sync(0xffffffffu, v, src & 31);
        return (src >= 0 && src < kWarp) ? (uint64_t)(x & 0xffffu) : 0ull;
    };
    const uint64_t O = get(own, l) | get(own, l + 1) << 16 | get(own, l + 2) << 32;
    const uint64_t K = get(kbits, l) | get(kbits, l + 1) << 16 | get(kbits, l + 2) << 32;
    const uint32_t o = (uint32_t)(O >> off), k = (uint32_t)(K >> off);
    if (lane <= 16 && o) {
        uint32_t* wp = bitmap + (w0 + lane);
        if (s >= 0 && s + 32 <= kChunkEdges) *wp = o == 0xffffffffu ? k : ((*wp & ~o) | k);
        else { atomicAnd(wp, ~o); atomicOr(wp, k); }
    }
}

// The carry into task t's first vertex (which began in an earlier task t0):
// tv[t0] (+) hv[t0+1] (+) ... (+) hv[t-1], folded left to right -- the value
// the vertex kernel's task-order join produces. Every task a vertex continues
// past publishes its piece (kChainPiece) as soon as its fold is done and, once
// it has its own carry, the inclusive fold (kChainIncl; the vertex's first
// task publishes its tail piece as inclusive at once). The warp looks back
// from t-1 for the nearest inclusive value and folds the pieces after it in
// order; any inclusive value it meets is itself that same left-to-right fold,
// so the result does not depend on timing. Tasks are claimed in order
// (ticket), so every task looked at is held by a running warp that never
// waits on a later task: the look-back always completes.
//
// Accumulators of up to 32 bytes travel with their state in H = size/8
// 16-byte halves {state, 8 value bytes}, each written and read as ONE
// relaxed .b128 memory operation (single-copy atomic in the PTX memory
// model; a .v2.u64 access would be two operations there, although both
// compile to the same STG/LDG.E.128.STRONG.GPU), so no fence is needed; a slot
// is ready when all its halves carry the same non-zero state (a reader that
// catches a piece -> inclusive rewrite half way sees mixed states and
// retries). Larger accumulators are written to hv / tv and published by a
// release store of the state.
template <class Accum>
__host__ __device__ constexpr int chain_halves() { return (int)((sizeof(Accum) + 7) / 8); }
template <class Accum>
__host__ __device__ constexpr bool chain_packed() { return sizeof(Accum) <= 32; }

template <class Accum>
__device__ __forceinline__ void chain_put(ulonglong2* d, uint32_t state, const Accum& v) {
    constexpr int H = chain_halves<Accum>();
    unsigned long long bits[H] = {};
    memcpy(bits, &v, sizeof(Accum));
#pragma unroll
    for (int h = 0; h < H; ++h)  // one 128-bit memory operation (.b128: single-copy atomic)
        asm volatile("{ .reg .b128 t; mov.b128 t, {%1, %2}; st.relaxed.gpu.global.b128 [%0], t; }"
                     :: "l"(d + h), "l"((unsigned long long)state), "l"(bits[h]) : "memory");
}
template <class Accum>
__device__ __forceinline__ uint32_t chain_get(const ulonglong2* d, Accum& v) {
    constexpr int H = chain_halves<Accum>();
    unsigned long long st[H], bits[H];
#pragma unroll
    for (int h = 0; h < H; ++h)
        asm volatile("{ .reg .b128 t; ld.relaxed.gpu.global.b128 t, [%2]; mov.b128 {%0, %1}, t; }"
                     : "=l"(st[h]), "=l"(bits[h]) : "l"(d + h) : "memory");
    memcpy(&v, bits, sizeof(Accum));
    bool same = true;
#pragma unroll
    for (int h = 1; h < H; ++h) same = same && st[h] == st[0];
    return same ? (uint32_t)st[0] : 0u;
}

#ifdef GGB_CHAIN_STATS
__device__ unsigned long long g_chain_stats[8];
#endif
template <class P, class W>
__device__ __forceinline__ typename P::Accum chain_carry(const EdgeArgs<P, W>& a, uint64_t t, int lane) {
    using Accum = typename P::Accum;
    constexpr bool kPacked = chain_packed<Accum>();
    int64_t base = (int64_t)t - 1;  // newest task of the window; lane i looks at base - i
    Accum v = a.prog.gather_identity();
    int L;
#ifdef GGB_CHAIN_STATS
    unsigned sleeps = 0, adv = 0;
#endif
    for (;;) {
        const int64_t j = base - lane;
        uint32_t s = kChainIncl;
        if (j >= 0) {
            if constexpr (kPacked) s = chain_get(a.cdesc + j * chain_halves<Accum>(), v);
            else s = ld_acquire(a.chain + j);
        }
        const uint32_t incl = __ballot_sync(0xffffffffu, s == kChainIncl);
        const uint32_t none = __ballot_sync(0xffffffffu, s == 0);
        if (incl) {
            L = __ffs(incl) - 1;
            if ((none & ((1u << L) - 1u)) == 0) break;
        } else if (!none) {
            base -= kWarp;  // 32 pieces, no inclusive value yet: look further back
#ifdef GGB_CHAIN_STATS
            ++adv;
#endif
            continue;
        }
#ifdef GGB_CHAIN_STATS
        ++sleeps;
#endif
        __nanosleep(64);  // a piece in between is still being folded
    }
#ifdef GGB_CHAIN_STATS
    if (lane == 0) {
        atomicAdd(&g_chain_stats[0], 1ull);
        atomicAdd(&g_chain_stats[1], (unsigned long long)sleeps);
        atomicAdd(&g_chain_stats[2], (unsigned long long)adv);
        if (sleeps == 0) atomicAdd(&g_chain_stats[3], 1ull);
        if (sleeps > 8) atomicAdd(&g_chain_stats[4], 1ull);
        if (sleeps > 64) atomicAdd(&g_chain_stats[5], 1ull);
        if (adv > 4) atomicAdd(&g_chain_stats[6], 1ull);
        atomicMax(&g_chain_stats[7], (unsigned long long)(sleeps + adv));
    }
#endif
    if constexpr (!kPacked) {  // values from L2 after the acquire
        __syncwarp();
        const int64_t j = base - lane;
        if (lane <= L) v = lane == L ? ld_l2(a.tv + j) : ld_l2(a.hv + j);
    }
    // inclusive value at lane L, pieces at lanes L-1 .. 0 (ascending tasks)
    Accum acc = shfl_idx_any(v, L);
    for (int i = L - 1; i >= 0; --i) acc = a.prog.combine(acc, shfl_idx_any(v, i));
    // later windows (all published when they were passed over); an inclusive
    // value met there equals the fold so far, so it replaces it exactly
    for (int64_t wb = base + kWarp; wb <= (int64_t)t - 1; wb += kWarp) {
        const int64_t j = wb - lane;
        uint32_t s;
        if constexpr (kPacked) {
            do {  // published; a multi-half slot caught mid-rewrite reads 0
                s = chain_get(a.cdesc + j * chain_halves<Accum>(), v);
            } while (__any_sync(0xffffffffu, s == 0));
        } else {
            s = ld_acquire(a.chain + j);
            __syncwarp();
            v = s == kChainIncl ? ld_l2(a.tv + j) : ld_l2(a.hv + j);
        }
        const uint32_t incl = __ballot_sync(0xffffffffu, s == kChainIncl);
        int start = kWarp - 1;
        if (incl) {
            const int L2 = __ffs(incl) - 1;
            acc = shfl_idx_any(v, L2);
            start = L2 - 1;
        }
        for (int i = start; i >= 0; --i) acc = a.prog.combine(acc, shfl_idx_any(v, i));
    }
    return acc;
}

#ifndef GGB_SHIFT_GROUP
#define GGB_SHIFT_GROUP 8
#endif
// Programs whose influence is the relative growth of the accumulator,
// (acc - before) / acc with 0 for acc <= 0 (PageRank, algorithms.hpp:25-30),
// and whose estatus is `influence > theta`.
template <class P>
__host__ __device__ constexpr bool rel_growth_influence() {
    if constexpr (requires { P::kRelGrowthInfluence; }) return P::kRelGrowthInfluence;
    else return false;
}

template <class P, class W, int MODE, bool HOT = false>
__device__ __forceinline__ void edge_task(const EdgeArgs<P, W>& a, int16_t* st0, uint8_t* sp0,
                                          uint64_t t, int lane, uint64_t pol_stream,
                                          uint64_t pol_hot, uint64_t pol_cold, HotTable ht = {},
                                          uint32_t* claim = nullptr) {
    using Accum = typename P::Accum;
    using Message = typename P::Message;
    constexpr bool CHAIN = MODE == kEdgeChain;
    const uint64_t tstart = t * kChunkEdges;
    const uint64_t r = t * kWarp + lane;
    const uint64_t P0 = r * kRun;
    const uint64_t lo = P0 > a.pad ? P0 : a.pad;
    const uint64_t hi = P0 + kRun < a.e_end ? P0 + kRun : a.e_end;
    // non-empty vertices touching the task: [i0, i_next], starts staged
    const uint32_t i0 = a.run_i[t * kWarp];
    // the next task's first run (run_i[nruns] = nz - 1 is the sentinel): loaded
    // before the gathers' inline asm, which the compiler may not move loads across
    const uint32_t i_next = a.run_i[(t + 1) * kWarp];
    Message m[kRun];
    WStore<W> wr[kRun];
    int len = 0;
    uint32_t ri = 0;  // run_i[r]: the non-empty vertex at the run's first position
    // Sources and message gathers do not depend on the staged starts: for
    // register-resident runs issue them first so their latency overlaps the
    // staging loads (local-memory runs of heavy programs measured better
    // the other way round).
    constexpr bool kEarly = fold_unroll<P>() != 1;
    if constexpr (kEarly) {
        len = hi > lo ? (int)(hi - lo) : 0;
        if (len > 0) {
            ri = a.run_i[r];
            load_run<P, W, HOT, MODE == kEdgePlain>(a, P0, lo, hi, m, wr, pol_stream, pol_hot, pol_cold, ht);
        }
    }
    const uint32_t cnt = i_next - i0 + 2;  // <= kStageStarts
    for (uint32_t j = lane; j < cnt; j += kWarp) {
        const int64_t rel = (int64_t)(a.nz_start[i0 + j] + a.pad) - (int64_t)tstart;
        st0[j] = (int16_t)(rel < 0 ? -1 : (rel > kChunkEdges ? kChunkEdges + 1 : rel));
        // skip test of the task's vertices (engine.hpp:196), staged with the
        // starts so the fold does not wait on it at every vertex boundary
        if constexpr (MODE != kEdgePlain)
            if (j + 1 < cnt) sp0[j] = vertex_processed(a.st_cur, a.a_off, row_of(a, i0 + j)) ? 1 : 0;
    }
    __syncwarp();
    const bool cont = st0[0] < 0;  // the task's first vertex began in an earlier task
    if constexpr (!kEarly) {
        len = hi > lo ? (int)(hi - lo) : 0;
        if (len > 0) {
            ri = a.run_i[r];
            load_run<P, W, HOT, MODE == kEdgePlain>(a, P0, lo, hi, m, wr, pol_stream, pol_hot, pol_cold, ht);
        }
    }
    const int rlo = (int)(lo - tstart), rhi = (int)(hi - tstart);  // task-relative
    auto wv = [&](int j) -> double {
        if constexpr (std::is_void_v<W>) return 1.0;
        else return (double)wr[j];
    };

    // sequential fold of the run, closing the vertices that end inside it
    // (k: index relative to i0; nb: task-relative end of vertex k)
    int k = len > 0 ? (int)(ri - i0) : 0;
    const int hk = k;
    int nb = len > 0 ? st0[k + 1] : 0;
    bool pk = true;
    if constexpr (MODE != kEdgePlain)
        if (len > 0) pk = sp0[k];
    const bool pk_first = pk;  // lane 0: the task's first vertex
    uint32_t pmask = 0;  // edges of processed vertices (flags we own)
    uint32_t bmask = 0;  // run positions at which a new vertex starts
    Accum x = a.prog.gather_identity(), hvv = x;
    bool head_closed = false;
    auto fold_step = [&](int j, const Message& mj, double wj) {
        const int p = (int)(P0 - tstart) + j;
        if (p >= rlo && p < rhi) {
            if (p >= nb) {  // vertex k ended before p: next non-empty vertex
                if (!head_closed) {
                    hvv = x;
                    head_closed = true;
                } else {
                    a.acc_out[row_of(a, i0 + k)] = x;  // began and ended inside this run
                }
                x = a.prog.gather_identity();
                ++k;
                nb = st0[k + 1];
                if constexpr (MODE != kEdgePlain) pk = sp0[k];
                if constexpr (CHAIN) bmask |= 1u << j;
            }
            if (pk) {
                (void)a.prog.gather(x, mj, wj);
                pmask |= 1u << j;
            }
        }
    };
    // Heavy programs fold the run in a rolled loop (one inlined gather);
    // without a second pass over the messages they shift the run through
    // registers (element 0 each step) instead of indexing a local array.
    constexpr bool kShift = fold_unroll<P>() == 1 && !CHAIN &&
                            sizeof(Message) <= 16;  // larger runs stay in local memory
    if constexpr (kShift) {
        // GGB_SHIFT_GROUP positions folded per step (inlined copies), then the
        // run shifts down by the group: 16/G shifts of 16-G elements instead
        // of 16 shifts of 15 (c4 approximate gather 2.27 -> 2.07 ms with G = 8;
        // G = 16, the fully unrolled fold, measured 2.48 ms)
        constexpr int G = GGB_SHIFT_GROUP;
#pragma unroll 1
        for (int j0 = 0; j0 < kRun; j0 += G) {
#pragma unroll
            for (int g = 0; g < G; ++g) fold_step(j0 + g, m[g], wv(g));
#pragma unroll
            for (int i = 0; i + G < kRun; ++i) {
                m[i] = m[i + G];
                if constexpr (!std::is_void_v<W>) wr[i] = wr[i + G];
            }
        }
    } else {
        for_run<P>([&](int j) { fold_step(j, m[j], wv(j)); });
    }
    const uint32_t tk = len > 0 ? (uint32_t)k : 0x7fffff00u + (uint32_t)lane;  // unique when empty
    // join runs sharing a destination: segmented inclusive scan keyed by tk
    Accum S = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Accum y = shfl_up_any(S, d);
        const uint32_t ky = __shfl_up_sync(0xffffffffu, tk, d);
        if (lane >= d && ky == tk) S = a.prog.combine(y, S);
    }
    const Accum prevS = shfl_up_any(S, 1);
    const uint32_t prevK = __shfl_up_sync(0xffffffffu, tk, 1);
    const bool joins_prev = len > 0 && lane > 0 && prevK == (uint32_t)hk;
    {
        if (head_closed) {
            const Accum hval = joins_prev ? a.prog.combine(prevS, hvv) : hvv;
            if (cont && hk == 0) a.hv[t] = hval;
            else a.acc_out[row_of(a, i0 + hk)] = hval;
        }
        const int nextLen = __shfl_down_sync(0xffffffffu, len, 1);
        const uint32_t nextHK = __shfl_down_sync(0xffffffffu, (uint32_t)hk, 1);
        const bool tail_here = len > 0 && (lane == 31 || nextLen == 0 || nextHK != tk);
        if (tail_here) {
            const bool cont_after = nb > rhi;  // the vertex goes on past this task
            const bool first_cont = cont && tk == 0;
            if (first_cont) a.hv[t] = S;
            if (cont_after && !(CHAIN && first_cont)) a.tv[t] = S;
            else if (!cont_after && !first_cont) a.acc_out[row_of(a, i0 + tk)] = S;
            if (CHAIN && cont_after) {  // publish for the tasks this vertex continues into
                const uint32_t state = first_cont ? kChainPiece : kChainIncl;
                if constexpr (chain_packed<Accum>()) {
                    chain_put(a.cdesc + t * chain_halves<Accum>(), state, S);
                } else {
                    __threadfence();
                    st_release(a.chain + t, state);
                }
            }
        }
    }
    Accum carry_in = a.prog.gather_identity();
    // the vertex spans the task: lane 31 (which published the piece S)
    // publishes the inclusive fold once the carry is known
    auto publish_incl = [&](const Accum& carry) {
        if (st0[1] > kChunkEdges && lane == kWarp - 1) {
            const Accum inc = a.prog.combine(carry, S);
            a.tv[t] = inc;
            if constexpr (chain_packed<Accum>()) {
                chain_put(a.cdesc + t * chain_halves<Accum>(), kChainIncl, inc);
            } else {
                __threadfence();
                st_release(a.chain + t, kChainIncl);
            }
        }
    };
    if constexpr (CHAIN) {
        if (cont) {  // warp-uniform
            // the carry of a vertex the skip test leaves out is never read:
            // its chain is closed at once (no look-back). The look-back comes
            // right after the fold: the chain advances at the rate tasks
            // publish inclusive values (measured: any later point is slower;
            // so is deciding the other vertices' edges while the look-back's
            // first window is in flight -- a second walk over the run:
            // c5 superstep 13.2 -> 16.7 ms, c2 1.2 -> 1.75 ms)
            if (__shfl_sync(0xffffffffu, pk_first, 0)) carry_in = chain_carry(a, t, lane);
            publish_incl(carry_in);
        }
        // PageRank's warp claims its next task now: the ticket's L2 round
        // trip overlaps the f64 influence pass, whose length varies little,
        // so tasks still start in claim order (c5 superstep -1.6 %; a claim
        // made before the look-back or the fold lets successors wait up to a
        // whole task for a piece: 13.8 -> 66 ms when claimed at task start).
        // Programs with short influence passes claim after the task (c2 SSSP
        // measured 8 % slower with the early claim).
        if constexpr (rel_growth_influence<P>())
            if (claim && lane == 0) *claim = atomicAdd(a.ticket, 1u);
    }
    if constexpr (CHAIN) {
        // influence of each edge against its exclusive running prefix
        // (engine.hpp:204-211): the carry into the task, the run's prefix in
        // the task, then the run's own sequential gathers; identity at each
        // later vertex start
        Accum run0 = (cont && hk == 0) ? carry_in : a.prog.gather_identity();
        if (joins_prev) run0 = a.prog.combine(run0, prevS);
        uint32_t kbits = 0;
        if constexpr (rel_growth_influence<P>()) {
            // Division-free pass: with s = acc after the edge and d = s - before,
            // the reference's test fl(d / s) > theta is decided as d > theta_hi*s
            // (true) or d < theta_lo*s (false): a quotient outside
            // theta*(1 +- 2^-41) is more than one ulp of theta away from it, so
            // its correctly rounded value cannot fall on the other side. Edges
            // in between (or with s, theta*s out of the normal range) are
            // "unsure" and re-decided by an exact walk with the division
            // (c5 superstep 13.6 -> 13.2 ms; tests: exact ties and one-ulp
            // thresholds, test_pagerank_exact_influence_ties).
            // (vertex starts and the run's valid range come from the fold:
            // bmask marks the positions where it moved to the next vertex,
            // pmask holds only in-range positions of processed vertices)
            Accum run = run0;
            uint32_t unsure = 0;
            for_run<P>([&](int j) {
                {
                    if ((bmask >> j) & 1u) run = a.prog.gather_identity();
                    if ((pmask >> j) & 1u) {
                        const double before = run;
                        run = run + m[j];
                        const double d = run - before;
                        const double th = run * a.theta_hi, tl = run * a.theta_lo;
                        // positive, finite, products in the normal range: one
                        // integer test on the high word; anything else (acc <= 0,
                        // NaN, extreme magnitudes) goes to the exact walk
                        const bool pn = (uint32_t)__double2hiint(run) - a.pn_lo < a.pn_span;
                        const bool hi_side = d > th;
                        kbits |= ((pn && hi_side) ? 1u : 0u) << j;
                        unsure |= ((pn && (hi_side || d < tl)) ? 0u : 1u) << j;
                    }
                }
            });
            // (theta not a normal number: pn_span = 0, every edge is unsure)
            if (unsure) {  // rare: the exact walk for the unsure edges
                run = run0;
                int nb2 = len > 0 ? st0[hk + 1] : 0, kk = hk;
                for_run<P>([&](int j) {
                    const int p = (int)(P0 - tstart) + j;
                    if (p >= rlo && p < rhi) {
                        if (p >= nb2) {
                            ++kk;
                            nb2 = st0[kk + 1];
                            run = a.prog.gather_identity();
                        }
                        if ((pmask >> j) & 1u) {
                            const double infl = a.prog.gather(run, m[j], wv(j));
                            if ((unsure >> j) & 1u)
                                kbits = (kbits & ~(1u << j)) |
                                        ((a.prog.estatus(infl, a.theta) ? 1u : 0u) << j);
                        }
                    }
                });
            }
        } else {
            Accum run = run0;
            for_run<P>([&](int j) {
                if ((bmask >> j) & 1u) run = a.prog.gather_identity();
                if ((pmask >> j) & 1u) {
                    const double infl = a.prog.gather(run, m[j], wv(j));
                    if (a.prog.estatus(infl, a.theta)) kbits |= 1u << j;
                }
            });
        }
        // The next task (claimed above; its ticket has arrived by now): pull its
        // sources and run map into L2 while this task writes its flags, so the
        // task starts with L2 hits (c5 superstep 13.26 -> 12.92 ms; also
        // prefetching its vertices' starts and skip-test inputs needs the run
        // map's value first and measured slower, 13.14 ms)
        if constexpr (rel_growth_influence<P>()) {
            if (claim) {
                const uint32_t tn = __shfl_sync(0xffffffffu, *claim, 0);
                if (tn < a.ntasks && lane <= 16) {
                    const void* pf = lane < 16 ? (const void*)(a.src + (uint64_t)tn * kChunkEdges + lane * 32)
                                               : (const void*)(a.run_i + (uint64_t)tn * kWarp);
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(pf));
                }
            }
        }
        warp_write_flags(a.bitmap, a.pad, tstart, pmask, kbits, lane);
        if constexpr (!rel_growth_influence<P>())
            if (claim && lane == 0) *claim = atomicAdd(a.ticket, 1u);
    }
    __syncwarp();  // st0 is restaged by the warp's next task
}

template <class P, class W, int MODE>
__global__ void __launch_bounds__(kBlockThreads)
edge_kernel(const EdgeArgs<P, W> a) {
    if (stop_after(a.stop_if)) return;
    __shared__ int16_t st_all[kWarpsPerBlock][kStageStarts];
    __shared__ uint8_t sp_all[MODE == kEdgePlain ? 1 : kWarpsPerBlock][kStageStarts];
    uint8_t* sp0 = MODE == kEdgePlain ? nullptr : sp_all[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_hot = policy_evict_last();
    const uint64_t pol_cold = a.cold_last ? policy_evict_last() : policy_evict_normal();
    if constexpr (MODE == kEdgeChain) {  // tasks claimed in order (see chain_carry)
        uint32_t t = 0;
        if (lane == 0) t = atomicAdd(a.ticket, 1u);
        t = __shfl_sync(0xffffffffu, t, 0);
        while (t < a.ntasks) {
            uint32_t tn = 0;
            edge_task<P, W, MODE>(a, st_all[threadIdx.x >> 5], sp0, t, lane, pol_stream, pol_hot,
                                  pol_cold, {}, &tn);
            t = __shfl_sync(0xffffffffu, tn, 0);
        }
        return;
    }
    const uint64_t warps = (uint64_t)gridDim.x * kWarpsPerBlock;
    for (uint64_t t = (uint64_t)blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); t < a.ntasks;
         t += warps) {
        edge_task<P, W, MODE>(a, st_all[threadIdx.x >> 5], sp0, t, lane, pol_stream, pol_hot,
                              pol_cold);
    }
}


// The superstep chain kernel for light programs (unweighted, or 4-byte
// messages), held to 80 registers (6 CTAs per SM): warps waiting in the
// look-back issue no gathers, so it needs more resident warps than the plain
// fold (c5 superstep 16.8 -> 15.4 ms; 7 CTAs spill and lose). Other programs
// (their runs spill at 80 registers) run edge_kernel<kEdgeChain>.
template <class P, class W>
constexpr bool chain_bounded() {
    return fold_unroll<P>() != 1 && (std::is_void_v<W> || sizeof(typename P::Message) == 4);
}
template <class P, class W>
__global__ void __launch_bounds__(kBlockThreads, 6)
edge_chain_kernel(const EdgeArgs<P, W> a) {
    __shared__ int16_t st_all[kWarpsPerBlock][kStageStarts];
    __shared__ uint8_t sp_all[kWarpsPerBlock][kStageStarts];
    const int lane = threadIdx.x & 31;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_hot = policy_evict_last();
    const uint64_t pol_cold = a.cold_last ? policy_evict_last() : policy_evict_normal();
    // Tasks are claimed in order (see chain_carry); the next claim is made
    // inside the current task, after its look-back (see edge_task).
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(a.ticket, 1u);
    t = __shfl_sync(0xffffffffu, t, 0);
    while (t < a.ntasks) {
        uint32_t tn = 0;  // lane 0: the next task, claimed inside the task
        edge_task<P, W, kEdgeChain>(a, st_all[threadIdx.x >> 5], sp_all[threadIdx.x >> 5], t, lane,
                                    pol_stream, pol_hot, pol_cold, {}, &tn);
        t = __shfl_sync(0xffffffffu, tn, 0);
    }
}

// The approximate gather with the hottest message slots copied into shared
// memory: one 24-warp CTA per SM; gathers of slots < nhot are LDS (no L1 tag
// or L2 request), the rest go to global memory as in edge_kernel. Every
// result is identical to edge_kernel's (the table is a copy of msg_cur).
constexpr int kHotWarps = 24;
template <class P, class W, int MODE>
__global__ void __launch_bounds__(kHotWarps * 32, 1)
edge_kernel_hot(const EdgeArgs<P, W> a, uint32_t nhot) {
    static_assert(MODE == kEdgePlain, "the hot-table gather has no skip test");
    if (stop_after(a.stop_if)) return;
    using Message = typename P::Message;
    extern __shared__ __align__(16) unsigned char hot_raw[];
    __shared__ int16_t st_all[kHotWarps][kStageStarts];
    Message* hot = reinterpret_cast<Message*>(hot_raw);
    for (uint32_t i = threadIdx.x; i < nhot; i += blockDim.x) hot[i] = a.msg_cur[i];
    __syncthreads();
    HotTable ht;
    ht.base = smem_u32(hot);
    ht.n = nhot;
    const int lane = threadIdx.x & 31;
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_hot = policy_evict_last();
    const uint64_t pol_cold = a.cold_last ? policy_evict_last() : policy_evict_normal();
    const uint64_t warps = (uint64_t)gridDim.x * kHotWarps;
    for (uint64_t t = (uint64_t)blockIdx.x * kHotWarps + (threadIdx.x >> 5); t < a.ntasks;
         t += warps)
        edge_task<P, W, MODE, true>(a, st_all[threadIdx.x >> 5], nullptr, t, lane, pol_stream, pol_hot,
                                    pol_cold, ht);
}

// Vertex epilogue over the POSITIONS: the rows [0, nrows) every iteration,
// the in-degree-0 tail [nrows, nloc) only while one of them is active (all
// are at t = 1; an in-degree-0 vertex is processed iff its status is set,
// engine.hpp:196). The accumulator of row p is acc_out[p] when its list lies
// inside one task, else tv[t0] (+) hv[t0+1] (+) ... (+) hv[t1] in task order;
// an in-degree-0 vertex folds nothing (gather_identity). Then GG-Apply,
// GG-VStatus, valid, message (in place: the iteration's gathers are done),
// status, counters. Skipped vertices keep property, message and (zero)
// status: no write. SUPER: after a kEdgeChain superstep tv[t1-1] already
// holds the left-to-right fold up to task t1-1, so the join is one combine.
template <class P, class W, bool SUPER, bool PEERS = false>
__global__ void __launch_bounds__(256)
vertex_kernel(const VertexArgs<P, W> a) {
    using Accum = typename P::Accum;
    using Property = typename P::Property;
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // the next iteration's counters, even if skipped
        IterCounters z{};
        z.bad_min = 0xffffffffu;
        *a.ctr_next = z;
    }
    if (stop_after(a.stop_if)) return;
    unsigned long long g = 0, pcount = 0;
    unsigned int changed = 0, inv = 0, bad = 0xffffffffu, eact = 0;
    const uint32_t pend = __ldg(&a.ctr_prev->empty_active) ? a.nloc : a.nrows;
    // U positions per thread per step, every load of the step issued before
    // any use (the accumulator of a single-task row is read speculatively):
    // one memory latency per U positions instead of a dependent chain each.
    constexpr int U = 2;  // measured on c5: 2 beats 1 (0.90 -> 0.75 ms) and 4 (register pressure)
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t base = blockIdx.x * blockDim.x + threadIdx.x; base < pend; base += U * stride) {
        uint8_t st[U];
        uint64_t o0[U], o1[U], q0[U], q1[U];
        uint32_t sv[U], deg[U], lv[U];
        Property prev[U];
        Accum acc1[U];
#pragma unroll
        for (int i = 0; i < U; ++i) {
            const uint32_t p = base + i * stride;
            if (p < pend) {
                lv[i] = a.vid_of_p[p];
                sv[i] = a.slot_p[p];
                st[i] = a.st[p];
                prev[i] = a.prop[p];
                o0[i] = o1[i] = q0[i] = q1[i] = 0;
                if (p < a.nrows) {
                    o0[i] = a.off[p];
                    o1[i] = a.off[p + 1];
                    q0[i] = a.a_off[p];
                    q1[i] = a.a_off[p + 1];
                    acc1[i] = a.acc_out[p];
                }
                deg[i] = 0;
                if constexpr (P::kNeedsDegree) deg[i] = a.deg_p[p];
            }
        }
#pragma unroll
        for (int i = 0; i < U; ++i) {
            const uint32_t p = base + i * stride;
            if (p >= pend) continue;
            const uint32_t v = a.v_begin + lv[i];
            const bool proc = (st[i] & kStActive) || q1[i] > q0[i];  // engine.hpp:196
            if (proc) {
                Accum acc = a.prog.gather_identity();
                if (o1[i] > o0[i]) {
                    const uint64_t t0 = (o0[i] + a.pad) / kChunkEdges,
                                   t1 = (o1[i] - 1 + a.pad) / kChunkEdges;
                    if (t0 == t1) {
                        acc = acc1[i];
                    } else if constexpr (SUPER) {
                        acc = a.prog.combine(a.tv[t1 - 1], a.hv[t1]);
                    } else {
                        acc = a.tv[t0];
                        for (uint64_t t = t0 + 1; t <= t1; ++t) acc = a.prog.combine(acc, a.hv[t]);
                    }
                }
                const Property fresh = a.prog.apply(v, acc, prev[i], a.n);  // GG-Apply (:216)
                const bool active = a.prog.vstatus(prev[i], fresh);         // GG-VStatus (:217)
                const bool ok = a.prog.valid(fresh);                        // (:218)
                a.prop[p] = fresh;
                const typename P::Message mnew = a.prog.message(fresh, deg[i]);
                a.msg[sv[i]] = mnew;
                if (PEERS) {  // fused exchange: the other replicas (NVLink stores)
                    const uint64_t sl = sv[i];
                    if ((sl >= a.gb0 && sl < a.ge0) || (sl >= a.gb1 && sl < a.ge1)) {
#pragma unroll
                        for (int r = 0; r < kMaxPeers; ++r)
                            if (r < a.npeers && r != a.self) a.peers[r][sl] = mnew;
                    }
                }
                a.st[p] = (uint8_t)((active ? kStActive : 0) | (ok ? 0 : kStInvalid) |
                                    (SUPER && (st[i] & kStActive) ? kStWasActive : 0));
                g += o1[i] - o0[i];
                pcount += 1;
                changed |= active ? 1u : 0u;
                if (active && p >= a.nrows) eact = 1;
                if (!ok) {
                    inv = 1;
                    // outside supersteps the reference's scan condition
                    // (status || active_in_degree > 0, engine.hpp:229) is exactly
                    // "processed"; in a superstep an in-degree-0 vertex's is its
                    // status (it keeps no edge), rows are re-checked after the rebuild
                    if (!SUPER || p >= a.nrows) bad = min(bad, v);
                }
            } else if (st[i]) {
                a.st[p] = 0;  // stale bits of an earlier superstep
            }
        }
    }
    // block reduction, one atomic per counter per block
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        g += __shfl_down_sync(0xffffffffu, g, d);
        pcount += __shfl_down_sync(0xffffffffu, pcount, d);
    }
    changed = __reduce_or_sync(0xffffffffu, changed);
    inv = __reduce_or_sync(0xffffffffu, inv);
    eact = __reduce_or_sync(0xffffffffu, eact);
    bad = __reduce_min_sync(0xffffffffu, bad);
    __shared__ unsigned long long s_g[8], s_p[8];
    __shared__ unsigned int s_c[8], s_i[8], s_b[8], s_e[8];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    if (lane == 0) {
        s_g[wib] = g; s_p[wib] = pcount; s_c[wib] = changed; s_i[wib] = inv; s_b[wib] = bad;
        s_e[wib] = eact;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nw = blockDim.x / 32;
        for (int i = 1; i < nw; ++i) {
            g += s_g[i]; pcount += s_p[i]; changed |= s_c[i]; inv |= s_i[i]; bad = min(bad, s_b[i]);
            eact |= s_e[i];
        }
        if (g) atomicAdd(&a.ctr->gathered, g);
        if (pcount) atomicAdd(&a.ctr->processed, pcount);
        if (changed) atomicOr(&a.ctr->changed, changed);
        if (inv) atomicOr(&a.ctr->any_invalid, inv);
        if (eact) atomicOr(&a.ctr->empty_active, eact);
        if (bad != 0xffffffffu) atomicMin(&a.ctr->bad_min, bad);
    }
}

// Superstep bad-vertex rule, engine.hpp:226-233: after the flag rewrite the
// reference scans (status || active_in_degree > 0) && !valid(next[v]) with
// active_in_degree already replaced by the kept counts.
__global__ void superstep_invalid_kernel(uint32_t nrows, uint32_t v_begin,
                                         const uint32_t* __restrict__ vid_of_p,
                                         const uint8_t* __restrict__ st,
                                         const uint64_t* __restrict__ s_off,
                                         IterCounters* __restrict__ ctr);

}  // namespace ggb
