// kernels.cuh — the hot path: one fused gather + GG-EStatus + GG-Apply +
// GG-VStatus kernel per iteration, plus the superstep hub pass.
//
// Replaces the reference's iteration body (engine.hpp:177-241):
//   * skip test            engine.hpp:196
//   * gather fold          engine.hpp:198-213 (GG-Gather, influence inline)
//   * superstep estatus    engine.hpp:207-211, 214 (GG-EStatus -> bitmap)
//   * apply/vstatus/valid  engine.hpp:216-224 (GG-Apply, GG-VStatus)
//
// Work decomposition (B200-first, power-law safe):
//   window  = 32 consecutive destination vertices (aligned), lane k owns
//             vertex k's accumulator and apply;
//   row     = 32 consecutive in-edges of the window's list (one per lane,
//             coalesced 128 B source loads), reduced by a segmented warp scan
//             keyed by destination;
//   task    = up to kRowsPerChunk rows of one window = one warp. Windows with
//             more edges are split into chunks; the last chunk to finish
//             (atomic ticket) combines the per-chunk partials IN CHUNK ORDER
//             and applies.
// Every vertex's fold structure depends only on its window-relative edge
// positions, so results are bitwise identical for any grid size, any launch
// order and any 32-aligned multi-GPU partition (the analogue of the
// reference's thread-count invariance, test_engine.cpp:161-182).
#pragma once

#include "common.cuh"

namespace ggb {

enum : int { kModeApprox = GG_MODE_APPROXIMATE, kModeAccurate = GG_MODE_ACCURATE,
             kModeSuperstep = GG_MODE_SUPERSTEP };

// status byte bits (double-buffered per vertex)
constexpr uint8_t kStActive = 1;     // vstatus result (engine.hpp:220)
constexpr uint8_t kStProcessed = 2;  // processed this iteration (msg buffers differ)
constexpr uint8_t kStInvalid = 4;    // !valid(fresh) (deferred superstep check)

// Per-iteration reductions (engine.hpp:186-189). Field groups are laid out
// for the multi-GPU allreduce: [u64 sum x2][u32 sum x2][u32 min].
struct IterCounters {
    unsigned long long gathered;
    unsigned long long processed;
    unsigned int changed;
    unsigned int any_invalid;
    unsigned int bad_min;      // smallest invalid vertex (global id), 0xffffffff = none
    unsigned int pad;
};

template <class P, class W>
struct IterArgs {
    P prog;
    uint64_t n;                 // global vertex count
    uint32_t v_begin;           // first owned vertex (multiple of 32)
    uint32_t nloc;              // owned vertices
    // gather list (full CSC or sparsified CSC), local vertex / edge ids
    const uint64_t* __restrict__ g_off;
    const uint32_t* __restrict__ g_src;
    const W* __restrict__ g_w;
    const uint4* __restrict__ tasks;   // {window, chunk, nchunks, partial slot of chunk 0}
    uint32_t ntasks;
    // active_in_degree source (engine.hpp:154-161, :214): offsets of the
    // current flag set (full CSC offsets under the accurate scheme)
    const uint64_t* __restrict__ a_off;
    const uint8_t* __restrict__ st_cur;
    uint8_t* __restrict__ st_next;
    typename P::Property* __restrict__ prop;          // local ids (unused if kMsgIsProp)
    const typename P::Message* __restrict__ msg_cur;  // global ids
    typename P::Message* __restrict__ msg_next;       // global ids
    const uint32_t* __restrict__ outdeg;              // global ids
    uint32_t* __restrict__ bitmap;                    // local full-CSC edge ids
    double theta;
    typename P::Accum* __restrict__ partials;         // [multi-chunk tasks][32]
    uint32_t* __restrict__ win_ticket;                // [windows]
    IterCounters* __restrict__ ctr;
};

struct WarpCounters {
    unsigned long long gathered = 0, processed = 0;
    unsigned int changed = 0, any_invalid = 0, bad_min = 0xffffffffu;
};

template <class P>
struct WarpSmem {
    uint32_t rel[kWindow + 1];                  // window-relative list offsets
    typename P::Accum part[2][kWindow];         // row partials, double buffered
};

// Fold one row of 32 edges (one per lane) into the owners' accumulators.
// Returns nothing; `acc` is lane k's accumulator for window vertex k.
// If SUPER, also evaluates each edge's influence against the exclusive
// prefix (carry + in-row segmented prefix) and writes the active-edge bitmap.
template <class P, bool SUPER>
__device__ __forceinline__ void fold_row(const P& prog, WarpSmem<P>& sm, int lane, int parity,
                                         bool valid, bool eproc, int key,
                                         const typename P::Message& m, double w,
                                         typename P::Accum& acc, double theta,
                                         uint32_t* bitmap, uint64_t row_e0, bool do_flags) {
    using Accum = typename P::Accum;
    Accum x = prog.gather_identity();
    if (eproc) (void)prog.gather(x, m, w);
    // inclusive segmented scan (Hillis-Steele) keyed by destination
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const Accum y = shfl_up_any(x, d);
        const int ky = __shfl_up_sync(0xffffffffu, key, d);
        if (lane >= d && ky == key) x = prog.combine(y, x);
    }
    const int knext = __shfl_down_sync(0xffffffffu, key, 1);
    const bool tail = valid && (lane == 31 || knext != key);
    if (SUPER && do_flags) {  // warp-uniform
        const Accum xe_raw = shfl_up_any(x, 1);
        const int kprev = __shfl_up_sync(0xffffffffu, key, 1);
        const Accum carry = shfl_idx_any(acc, key & 31);
        Accum pre = (lane > 0 && kprev == key) ? prog.combine(carry, xe_raw) : carry;
        double infl = 0.0;
        if (eproc) infl = prog.gather(pre, m, w);  // GG-Gather influence (engine.hpp:204-206)
        const bool keep = eproc && prog.estatus(infl, theta);  // GG-EStatus (:208)
        const uint32_t K = __ballot_sync(0xffffffffu, keep);
        const uint32_t O = __ballot_sync(0xffffffffu, eproc);
        if (O != 0 && lane < 2) {
            const uint32_t sh = (uint32_t)(row_e0 & 31);
            const uint64_t word0 = row_e0 >> 5;
            const uint64_t K64 = (uint64_t)K << sh, O64 = (uint64_t)O << sh;
            const uint32_t o = lane == 0 ? (uint32_t)O64 : (uint32_t)(O64 >> 32);
            const uint32_t k = lane == 0 ? (uint32_t)K64 : (uint32_t)(K64 >> 32);
            if (o) {
                // flags of edges of skipped vertices persist (SPEC: superstep scope)
                atomicAnd(bitmap + word0 + lane, ~o);
                atomicOr(bitmap + word0 + lane, k & o);
            }
        }
    }
    if (tail) sm.part[parity][key] = x;
    const uint32_t have = __reduce_or_sync(0xffffffffu, tail ? (1u << (key & 31)) : 0u);
    __syncwarp();
    if ((have >> lane) & 1u) acc = prog.combine(acc, sm.part[parity][lane]);
}

template <class P, class W>
__device__ __forceinline__ void apply_vertex(const IterArgs<P, W>& a, uint32_t lv, bool proc,
                                             uint8_t st, uint64_t list_deg,
                                             const typename P::Accum& acc, int mode,
                                             WarpCounters& wc) {
    using Property = typename P::Property;
    const uint32_t v = a.v_begin + lv;
    if (proc) {
        Property prev;
        if constexpr (P::kMsgIsProp) prev = a.msg_cur[v];
        else prev = a.prop[lv];
        const Property fresh = a.prog.apply(v, acc, prev, a.n);    // GG-Apply (:216)
        const bool active = a.prog.vstatus(prev, fresh);           // GG-VStatus (:217)
        const bool ok = a.prog.valid(fresh);                       // (:218)
        if constexpr (!P::kMsgIsProp) a.prop[lv] = fresh;
        uint32_t deg = 0;
        if constexpr (P::kNeedsDegree) deg = a.outdeg[v];
        a.msg_next[v] = a.prog.message(fresh, deg);
        a.st_next[lv] = (uint8_t)((active ? kStActive : 0) | kStProcessed | (ok ? 0 : kStInvalid));
        wc.gathered += list_deg;
        wc.processed += 1;
        wc.changed |= active ? 1u : 0u;
        if (!ok) {
            wc.any_invalid = 1;
            // outside supersteps the reference's scan condition
            // (status || active_in_degree > 0, engine.hpp:229) is exactly
            // "processed"; supersteps are re-checked after the rebuild.
            if (mode != kModeSuperstep) wc.bad_min = min(wc.bad_min, v);
        }
    } else {
        // skipped: next = prev (engine.hpp:183), status 0. The message
        // buffers only differ if the vertex was processed last iteration.
        if (st & kStProcessed) a.msg_next[v] = a.msg_cur[v];
        a.st_next[lv] = 0;
    }
}

template <class P, class W, bool SUPER, int U>
__global__ void __launch_bounds__(kBlockThreads)
iteration_kernel(const IterArgs<P, W> a) {
    using Accum = typename P::Accum;
    using Message = typename P::Message;
    constexpr int MODE = SUPER ? kModeSuperstep : kModeAccurate;
    __shared__ WarpSmem<P> smem_all[kWarpsPerBlock];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpSmem<P>& sm = smem_all[wib];
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    WarpCounters wc;
    const uint32_t total_warps = gridDim.x * kWarpsPerBlock;

    for (uint32_t t = blockIdx.x * kWarpsPerBlock + wib; t < a.ntasks; t += total_warps) {
        const uint4 tk = a.tasks[t];
        const uint32_t win = tk.x, chunk = tk.y, nch = tk.z, slot0 = tk.w;
        const uint32_t lv0 = win * kWindow;
        const uint32_t nv = min((uint32_t)kWindow, a.nloc - lv0);
        const uint64_t base = a.g_off[lv0];
        const uint64_t my_off = lane < (int)nv ? a.g_off[lv0 + lane] : 0;
        const uint64_t wend = a.g_off[lv0 + nv];
        const uint32_t wedges = (uint32_t)(wend - base);
        sm.rel[lane] = lane < (int)nv ? (uint32_t)(my_off - base) : wedges;
        if (lane == 0) sm.rel[32] = wedges;
        // processed test (engine.hpp:196)
        uint8_t st = 0;
        uint64_t aid = 0;
        if (lane < (int)nv) {
            st = a.st_cur[lv0 + lane];
            aid = a.a_off[lv0 + lane + 1] - a.a_off[lv0 + lane];
        }
        const bool proc = lane < (int)nv && ((st & kStActive) || aid > 0);
        const uint32_t proc_mask = __ballot_sync(0xffffffffu, proc);
        __syncwarp();
        const uint32_t nrows = (wedges + 31) >> 5;
        const bool multi = nch > 1;
        const uint32_t r0 = chunk * kRowsPerChunk;
        const uint32_t r1 = min(nrows, r0 + kRowsPerChunk);

        Accum acc = a.prog.gather_identity();
        // initial destination of this lane's first edge: largest k with rel[k] <= p
        int k = 0;
        {
            const uint32_t p = r0 * 32 + lane;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1)
                if (k + step < (int)nv && sm.rel[k + step] <= p) k += step;
        }
        for (uint32_t row = r0; row < r1; row += U) {
            uint32_t s[U];
            double wv[U];
            Message m[U];
            int key[U];
            bool val[U], ep[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t p = (row + u) * 32 + lane;
                val[u] = (row + u) < r1 && p < wedges;
                while (k + 1 < (int)nv && sm.rel[k + 1] <= p) ++k;
                key[u] = val[u] ? k : 32;
                ep[u] = val[u] && ((proc_mask >> k) & 1u);
                s[u] = ep[u] ? ld_stream_u32(a.g_src + base + p, pol_stream) : 0u;
                wv[u] = ep[u] ? WeightIO<W>::load(a.g_w, base + p) : 1.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (ep[u]) m[u] = ld_msg(a.msg_cur + s[u], pol_keep);
                else memset(&m[u], 0, sizeof(Message));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (row + u < r1)
                    fold_row<P, SUPER>(a.prog, sm, lane, (row + u) & 1, val[u], ep[u], key[u],
                                       m[u], wv[u], acc, a.theta, a.bitmap,
                                       base + (uint64_t)(row + u) * 32, !multi);
            }
        }
        // Multi-chunk windows get their superstep flags from
        // superstep_hub_kernel, which has the carry of earlier chunks.
        if (!multi) {
            if (lane < (int)nv)
                apply_vertex(a, lv0 + lane, proc, st, (uint64_t)(sm.rel[lane + 1] - sm.rel[lane]),
                             acc, MODE, wc);
        } else {
            a.partials[(uint64_t)(slot0 + chunk) * kWindow + lane] = acc;
            __threadfence();
            uint32_t ticket = 0;
            if (lane == 0) ticket = atomicAdd(a.win_ticket + win, 1u);
            ticket = __shfl_sync(0xffffffffu, ticket, 0);
            if (ticket == nch - 1) {
                __threadfence();
                const uint64_t first = slot0;
                Accum run = a.prog.gather_identity();
                for (uint32_t c = 0; c < nch; ++c) {
                    const Accum pc = ld_cg_any(a.partials + (first + c) * kWindow + lane);
                    if constexpr (SUPER) a.partials[(first + c) * kWindow + lane] = run;
                    run = a.prog.combine(run, pc);
                }
                if (lane == 0) a.win_ticket[win] = 0;
                if (lane < (int)nv)
                    apply_vertex(a, lv0 + lane, proc, st,
                                 (uint64_t)(sm.rel[lane + 1] - sm.rel[lane]), run, MODE, wc);
            }
        }
        __syncwarp();
    }

    // block-level counter aggregation, one atomic per counter per block
    __shared__ unsigned long long s_g[kWarpsPerBlock], s_p[kWarpsPerBlock];
    __shared__ unsigned int s_c[kWarpsPerBlock], s_i[kWarpsPerBlock], s_b[kWarpsPerBlock];
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) {
        wc.gathered += __shfl_down_sync(0xffffffffu, wc.gathered, d);
        wc.processed += __shfl_down_sync(0xffffffffu, wc.processed, d);
    }
    wc.changed = __reduce_or_sync(0xffffffffu, wc.changed);
    wc.any_invalid = __reduce_or_sync(0xffffffffu, wc.any_invalid);
    wc.bad_min = __reduce_min_sync(0xffffffffu, wc.bad_min);
    if (lane == 0) {
        s_g[wib] = wc.gathered; s_p[wib] = wc.processed; s_c[wib] = wc.changed;
        s_i[wib] = wc.any_invalid; s_b[wib] = wc.bad_min;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long g = 0, p = 0;
        unsigned int c = 0, inv = 0, b = 0xffffffffu;
        for (int i = 0; i < kWarpsPerBlock; ++i) {
            g += s_g[i]; p += s_p[i]; c |= s_c[i]; inv |= s_i[i]; b = min(b, s_b[i]);
        }
        if (g) atomicAdd(&a.ctr->gathered, g);
        if (p) atomicAdd(&a.ctr->processed, p);
        if (c) atomicOr(&a.ctr->changed, c);
        if (inv) atomicOr(&a.ctr->any_invalid, inv);
        if (b != 0xffffffffu) atomicMin(&a.ctr->bad_min, b);
    }
}

// Superstep pass for windows split into several chunks: re-walks their rows
// with the exclusive chunk carry (written by the last chunk of
// iteration_kernel) to evaluate each edge's influence against its exact
// running-fold prefix and rewrite the bitmap.
template <class P, class W, int U>
__global__ void __launch_bounds__(kBlockThreads)
superstep_hub_kernel(const IterArgs<P, W> a, const uint4* __restrict__ mtasks, uint32_t nmtasks) {
    using Accum = typename P::Accum;
    using Message = typename P::Message;
    __shared__ WarpSmem<P> smem_all[kWarpsPerBlock];
    const int lane = threadIdx.x & 31;
    const int wib = threadIdx.x >> 5;
    WarpSmem<P>& sm = smem_all[wib];
    const uint64_t pol_stream = policy_evict_first();
    const uint64_t pol_keep = policy_evict_last();
    const uint32_t total_warps = gridDim.x * kWarpsPerBlock;
    for (uint32_t i = blockIdx.x * kWarpsPerBlock + wib; i < nmtasks; i += total_warps) {
        const uint4 tk = mtasks[i];
        const uint32_t win = tk.x, chunk = tk.y, slot0 = tk.w;
        const uint32_t lv0 = win * kWindow;
        const uint32_t nv = min((uint32_t)kWindow, a.nloc - lv0);
        const uint64_t base = a.g_off[lv0];
        const uint64_t my_off = lane < (int)nv ? a.g_off[lv0 + lane] : 0;
        const uint64_t wend = a.g_off[lv0 + nv];
        const uint32_t wedges = (uint32_t)(wend - base);
        sm.rel[lane] = lane < (int)nv ? (uint32_t)(my_off - base) : wedges;
        if (lane == 0) sm.rel[32] = wedges;
        uint8_t st = 0;
        uint64_t aid = 0;
        if (lane < (int)nv) {
            st = a.st_cur[lv0 + lane];
            aid = a.a_off[lv0 + lane + 1] - a.a_off[lv0 + lane];
        }
        const bool proc = lane < (int)nv && ((st & kStActive) || aid > 0);
        const uint32_t proc_mask = __ballot_sync(0xffffffffu, proc);
        __syncwarp();
        const uint32_t nrows = (wedges + 31) >> 5;
        const uint32_t r0 = chunk * kRowsPerChunk;
        const uint32_t r1 = min(nrows, r0 + kRowsPerChunk);
        Accum acc = a.partials[(uint64_t)(slot0 + chunk) * kWindow + lane];  // exclusive chunk carry
        int k = 0;
        {
            const uint32_t p = r0 * 32 + lane;
#pragma unroll
            for (int step = 16; step >= 1; step >>= 1)
                if (k + step < (int)nv && sm.rel[k + step] <= p) k += step;
        }
        for (uint32_t row = r0; row < r1; row += U) {
            uint32_t s[U];
            double wv[U];
            Message m[U];
            int key[U];
            bool val[U], ep[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t p = (row + u) * 32 + lane;
                val[u] = (row + u) < r1 && p < wedges;
                while (k + 1 < (int)nv && sm.rel[k + 1] <= p) ++k;
                key[u] = val[u] ? k : 32;
                ep[u] = val[u] && ((proc_mask >> k) & 1u);
                s[u] = ep[u] ? ld_stream_u32(a.g_src + base + p, pol_stream) : 0u;
                wv[u] = ep[u] ? WeightIO<W>::load(a.g_w, base + p) : 1.0;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (ep[u]) m[u] = ld_msg(a.msg_cur + s[u], pol_keep);
                else memset(&m[u], 0, sizeof(Message));
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (row + u < r1)
                    fold_row<P, true>(a.prog, sm, lane, (row + u) & 1, val[u], ep[u], key[u], m[u],
                                      wv[u], acc, a.theta, a.bitmap,
                                      base + (uint64_t)(row + u) * 32, true);
            }
        }
        __syncwarp();
    }
}

// Superstep bad-vertex rule, engine.hpp:226-233: after the flag rewrite the
// reference scans (status || active_in_degree > 0) && !valid(next[v]) with
// active_in_degree already replaced by the kept counts.
__global__ void superstep_invalid_kernel(uint32_t nloc, uint32_t v_begin,
                                         const uint8_t* __restrict__ st_cur,
                                         const uint8_t* __restrict__ st_next,
                                         const uint64_t* __restrict__ s_off,
                                         IterCounters* __restrict__ ctr);

}  // namespace ggb
