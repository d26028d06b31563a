// engine.cuh — host side of the engine: gg::run (engine.hpp:141-249) driving
// the device kernels. Instantiated per (program, weight type) in capi.cu.
#pragma once

#include <cstdlib>

#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "exchange.cuh"
#include "graph.cuh"
#include "kernels.cuh"

namespace ggb {

// engine.cpp:92-107
inline int mode_for(int scheme, uint64_t t, uint64_t alpha) {
    switch (scheme) {
        case GG_SCHEME_ACCURATE: return GG_MODE_ACCURATE;
        case GG_SCHEME_SP: return GG_MODE_APPROXIMATE;
        case GG_SCHEME_SMS:
            if (t <= alpha) return GG_MODE_APPROXIMATE;
            if (t == alpha + 1) return GG_MODE_SUPERSTEP;
            return GG_MODE_ACCURATE;
        case GG_SCHEME_GG:
            return t % (alpha + 1) == 0 ? GG_MODE_SUPERSTEP : GG_MODE_APPROXIMATE;
    }
    return GG_MODE_ACCURATE;
}

// engine.cpp:45-61 (same messages, checked in the same order)
inline void validate(const gg_engine_config& c) {
    if (!(c.sigma >= 0.0 && c.sigma <= 1.0)) throw Error(GG_INVALID_ARGUMENT, "sigma must be in [0,1]");
    if (!(c.theta >= 0.0)) throw Error(GG_INVALID_ARGUMENT, "theta must be >= 0");
    if (c.alpha < 1) throw Error(GG_INVALID_ARGUMENT, "alpha must be >= 1");
    if (c.max_iterations < 1) throw Error(GG_INVALID_ARGUMENT, "max_iterations must be >= 1");
    if (c.threads < 1) throw Error(GG_INVALID_ARGUMENT, "threads must be >= 1");
    if (c.scheme < 0 || c.scheme > 3) throw Error(GG_INVALID_ARGUMENT, "unknown scheme");
}

struct RunIO {
    const gg_engine_config* cfg = nullptr;
    gg_iter_record* recs = nullptr;
    uint64_t rec_cap = 0;
    gg_run_summary* sum = nullptr;
    const gg_run_opts* opts = nullptr;
    void* out_props = nullptr;   // host: double[n*S] or uint32[n] (kRawOutput)
    int out_states = 1;
};

// Initial messages of every (global) vertex, and the owned vertices'
// properties and statuses by position (engine.hpp:163-167).
template <class P>
__global__ void init_kernel(P prog, uint64_t n, uint32_t v_begin, uint32_t nloc,
                            const uint32_t* __restrict__ outdeg,
                            const uint32_t* __restrict__ slot_of,
                            const uint32_t* __restrict__ vid_of_p,
                            typename P::Message* __restrict__ msg,
                            typename P::Property* __restrict__ prop, uint8_t* __restrict__ st) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const typename P::Property p = prog.init_property((uint32_t)v, n);  // engine.hpp:164
        uint32_t deg = 0;
        if constexpr (P::kNeedsDegree) deg = outdeg[v];
        msg[slot_of[v]] = prog.message(p, deg);
        if (v < nloc) {  // position v of this rank
            prop[v] = prog.init_property(v_begin + vid_of_p[v], n);
            st[v] = kStActive;  // status starts at 1 (engine.hpp:166)
        }
    }
}

// position order -> vertex order (out[lv] = props[p], lv = vid_of_p[p])
template <class T>
__global__ void to_vertex_order_kernel(const T* __restrict__ by_pos, const uint32_t* __restrict__ vid_of_p,
                                       uint64_t nloc, T* __restrict__ out) {
    for (uint64_t p = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; p < nloc;
         p += (uint64_t)gridDim.x * blockDim.x)
        out[vid_of_p[p]] = by_pos[p];
}

template <class P>
__global__ void export_kernel(P prog, const typename P::Property* __restrict__ props, uint64_t n,
                              int S, double* __restrict__ out) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x)
        for (int i = 0; i < S; ++i) out[v * S + i] = prog.to_double(props[v], i);
}

inline unsigned grid1d(uint64_t n, int block = 256) {
    uint64_t g = (n + block - 1) / block;
    if (g > 148ull * 32) g = 148ull * 32;
    return (unsigned)(g ? g : 1);
}

inline double event_ms(cudaEvent_t a, cudaEvent_t b) {
    float f = 0.f;
    GGB_CUDA(cudaEventElapsedTime(&f, a, b));
    return (double)f;
}

template <class P, class W>
struct Engine {
    using Prop = typename P::Property;
    using Msg = typename P::Message;
    using Acc = typename P::Accum;

    // CTAs of one launch: `full` (the occupancy-sized grid) unless the run's
    // grid_ctas test hook caps it (gg_run_opts; results do not depend on it)
    static unsigned capped(unsigned full, unsigned cap) { return cap && cap < full ? cap : full; }
    template <int MODE>
    static int grid_edge(DevGraph& g) {
        static const int per_sm = occupancy_grid((const void*)edge_kernel<P, W, MODE>, kBlockThreads,
                                                 0, 1);
        return per_sm * g.num_sms;
    }
    // L1+L2 evict_last prefix of the message slots (GGB_HOT_KB overrides the
    // measured default of 24 MB for message arrays larger than L2's share)
    static size_t hot_bytes() {
        static size_t b = [] {
            const char* e = std::getenv("GGB_HOT_KB");
            return (size_t)(e ? std::atol(e) : 24 * 1024) << 10;
        }();
        return b;
    }
    // Algorithmic HBM bytes (SURVEY §8(d) byte formula B = E_p*b_e + N*b_v;
    // a superstep adds the bitmap write E_p/8).
    static uint64_t edge_bytes(uint64_t edges, bool super) {
        const uint64_t be = 4 + sizeof(Msg) + (uint64_t)weight_bytes<W>();
        return edges * be + (super ? edges / 8 : 0);
    }
    static uint64_t vertex_bytes(uint64_t positions) {
        uint64_t bv = 8 + 2 + 2 * sizeof(Prop) + (P::kMsgIsProp ? 0 : sizeof(Msg)) +
                      (P::kNeedsDegree ? 4 : 0);
        if constexpr (requires { P::kReadsPrior; }) bv += 8;
        return positions * bv;
    }

    // shared-memory hot-slot table of edge_kernel_hot (GGB_SMEM_HOT_KB, default
    // 160 KB; 0 disables the hot kernel)
    static constexpr int kMaxBatch = 8;            // iterations enqueued per host sync
    static constexpr int kRing = kMaxBatch + 1;    // counter slots
    static constexpr bool kHotOK =
        fold_unroll<P>() != 1 && (sizeof(Msg) == 4 || sizeof(Msg) == 8 || sizeof(Msg) == 16);
    // Measured (approximate gather, one B200): 4-byte messages gain 18% (c3
    // WCC) / 5% (c2 SSSP) with a 64 KB table; 8-byte PageRank messages lose
    // at every size (the L1 evict_last class already holds their hot lines
    // and the 24-warp CTA spills), so the table is off for them.
    static size_t smem_hot_bytes() {
        static size_t b = [] {
            const char* e = std::getenv("GGB_SMEM_HOT_KB");
            return (size_t)(e ? std::atol(e) : (sizeof(Msg) == 4 ? 64 : 0)) << 10;
        }();
        return b;
    }
    static void launch_edge_hot(DevGraph& g, const EdgeArgs<P, W>& ea, uint32_t nhot, unsigned cap) {
        const size_t bytes = (size_t)nhot * sizeof(Msg);
        // the dynamic shared-memory limit is per device context: set once per device
        static bool attr_set[64] = {};
        if (g.device < 0 || g.device >= 64 || !attr_set[g.device]) {
            GGB_CUDA(cudaFuncSetAttribute((const void*)edge_kernel_hot<P, W, kEdgePlain>,
                                          cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)std::max<size_t>(smem_hot_bytes(), 16)));
            if (g.device >= 0 && g.device < 64) attr_set[g.device] = true;
        }
        edge_kernel_hot<P, W, kEdgePlain><<<capped(g.num_sms, cap), kHotWarps * 32, bytes, g.stream>>>(
            ea, nhot);
        GGB_CUDA(cudaGetLastError());
    }

    template <int MODE>
    static void launch_edge(DevGraph& g, const EdgeArgs<P, W>& ea, unsigned cap) {
        edge_kernel<P, W, MODE><<<capped(grid_edge<MODE>(g), cap), kBlockThreads, 0, g.stream>>>(ea);
        GGB_CUDA(cudaGetLastError());
    }

    static void launch_chain(DevGraph& g, const EdgeArgs<P, W>& ea, unsigned cap) {
        if constexpr (chain_bounded<P, W>()) {
            static const int per_sm = occupancy_grid((const void*)edge_chain_kernel<P, W>,
                                                     kBlockThreads, 0, 1);
            edge_chain_kernel<P, W><<<capped(per_sm * g.num_sms, cap), kBlockThreads, 0, g.stream>>>(ea);
            GGB_CUDA(cudaGetLastError());
        } else {
            launch_edge<kEdgeChain>(g, ea, cap);
        }
    }

    static void run(DevGraph& g, const P& prog, RunIO& io) {
        const gg_engine_config& cfg = *io.cfg;
        const bool timing = io.opts && io.opts->timing;
        GGB_CUDA(cudaSetDevice(g.device));
        const uint64_t n = g.n, nloc = g.nloc;
        const bool sparse = cfg.scheme != GG_SCHEME_ACCURATE;
        int launches = 0;
        Workspace& ws = g.ws;
        g.project_last = nullptr;  // no valid run until this one completes
        const unsigned cap = io.opts ? io.opts->grid_ctas : 0u;

        // one message buffer: an iteration's gathers complete before its
        // vertex kernel rewrites the messages (same stream; several ranks with
        // the fused exchange: a barrier, since the vertex kernels also write
        // the other ranks' replicas); per-vertex state by position (graph.cuh)
        Msg* msg = static_cast<Msg*>(exchange_msg_buffer(g, n * sizeof(Msg)));
        const bool fused = exchange_register_peers(g, msg, n * sizeof(Msg));
        Prop* prop = ws.get<Prop>("prop", nloc + 1);
        uint8_t* st = ws.get<uint8_t>("st", nloc + 1);
        const uint64_t R = g.nrows;
        // Counters live in a ring of kRing slots: iteration u accumulates into
        // ring[u % kRing] and its vertex kernel resets ring[(u + 1) % kRing]
        // for the next one, so no memset is enqueued per iteration and a
        // batch of up to kMaxBatch iterations is read back with one copy.
        IterCounters* ring = ws.get<IterCounters>("ctr", kRing);
        IterCounters* h_ring =
            static_cast<IterCounters*>(g.host_counters(kRing * sizeof(IterCounters)));
        reset_counters_kernel<<<1, kRing, 0, g.stream>>>(ring, kRing);
        GGB_CUDA(cudaGetLastError());
        Acc* acc_out = ws.get<Acc>("acc_out", R + 1);
        const uint64_t ntask_cap = g.full.ntasks + 2;
        Acc* hv = ws.get<Acc>("hv", ntask_cap);
        Acc* tv = ws.get<Acc>("tv", ntask_cap);
        // superstep chain (kEdgeChain): per-task slots + the task ticket,
        // cleared before each superstep
        constexpr size_t kSlot =
            chain_packed<Acc>() ? sizeof(ulonglong2) * chain_halves<Acc>() : sizeof(uint32_t);
        char* chain = nullptr;
        if (cfg.scheme == GG_SCHEME_SMS || cfg.scheme == GG_SCHEME_GG)
            chain = static_cast<char*>(ws.get("chain", ntask_cap * kSlot + 16));
        const uint64_t nwords = (g.e_loc + 31) / 32;
        const size_t wsz = (size_t)weight_bytes<W>();
        uint32_t* bitmap = nullptr;
        uint64_t* s_off = nullptr;
        uint32_t* s_src = nullptr;
        void* s_w = nullptr;
        ListMeta sp;
        cudaEvent_t e4 = timing ? g.event(4) : nullptr, e5 = timing ? g.event(5) : nullptr;

        init_kernel<P><<<grid1d(std::max<uint64_t>(n, nloc)), 256, 0, g.stream>>>(
            prog, n, (uint32_t)g.v_begin, (uint32_t)nloc, g.outdeg, g.slot_of, g.vid_of_p, msg, prop, st);
        GGB_CUDA(cudaGetLastError());
        ++launches;
        uint64_t kept = g.e_loc;
        if (sparse) {  // engine.hpp:151-161
            bitmap = ws.get<uint32_t>("bitmap", nwords + 1);
            s_off = ws.get<uint64_t>("s_off", R + 1);
            s_src = ws.get<uint32_t>("s_src", g.e_loc + 2 * kChunkEdges + kRun);
            s_w = wsz ? ws.get("s_w", (g.e_loc + kChunkEdges + kRun) * wsz) : nullptr;
            if (g.pre_sparse && g.pre_sigma == cfg.sigma && g.pre_seed == cfg.seed) {
                kept = presparse_finish(g, s_off, sp);  // sparsified during the upload
                launches += 1;  // sp_layout
            } else {
                const SparsifySpec hs = sparsify_spec(cfg.sigma, cfg.seed, false);
                kept = rebuild_sparse(g, bitmap, s_off, s_src, s_w, sp, nullptr, nullptr, &launches,
                                      &hs);
            }
        }
        g.pre_sparse = false;  // one run uses it (its supersteps rewrite the bitmap)
        const uint64_t* a_off = sparse ? s_off : g.full.nz_start;  // by row
        // Gather cache classes (EdgeArgs::hot_limit). A message array that fits
        // half of L2 is kept there whole; a larger one protects its hottest
        // prefix in L1 and L2 (measured on c5: 24 MB best of 4..80 MB). The
        // hot-first slot order makes the hottest slots a prefix: with one
        // rank the whole order is by out-degree class; with several, the
        // tier-0 slots (every rank's highest out-degree octaves, compute_slots)
        // are the global prefix the classes may use.
        const uint64_t hot_prefix = g.nranks == 1 ? n : g.hot_slots;
        const bool msgs_fit_l2 = (uint64_t)n * sizeof(Msg) <= (64ull << 20);
        const uint32_t hot_limit = !msgs_fit_l2
            ? (uint32_t)std::min<uint64_t>(hot_prefix, hot_bytes() / sizeof(Msg)) : 0u;
        // hot slots copied into shared memory by the approximate gather
        const uint32_t nhot = kHotOK
            ? (uint32_t)std::min<uint64_t>(hot_prefix, smem_hot_bytes() / sizeof(Msg)) : 0u;
        const uint32_t l2_limit = (uint32_t)std::min<uint64_t>(hot_prefix, (80ull << 20) / sizeof(Msg));

        uint64_t iterations_run = 0, total_edges = 0;
        bool prev_empty_active = true;  // every status starts active: t = 1 walks every position
        double total_wall = 0.0;
        // Iterations are enqueued in batches: a stretch of consecutive
        // non-superstep iterations (one rank) is launched back to back with
        // device-side early exit (stop_after) and read back with one sync;
        // supersteps and multi-rank iterations form batches of one. Results
        // and records are those of the one-at-a-time loop (engine.hpp:177-241).
        // Several ranks batch too: every rank enqueues the same iterations,
        // a stopped iteration's kernels return at once but its exchange still
        // runs (unchanged messages, zero counters) on every rank, so the
        // collectives stay matched; NCCL calls are stream-ordered (one host
        // sync per batch), the in-process transport syncs inside each call.
        auto batchable = [&](uint64_t u) {
            return mode_for(cfg.scheme, u, cfg.alpha) != GG_MODE_SUPERSTEP;
        };
        bool done = false;
        for (uint64_t t = 1; t <= cfg.max_iterations && !done;) {  // engine.hpp:177
            const auto t0 = std::chrono::steady_clock::now();
            int B = 1;
            if (batchable(t))
                while (t + B <= cfg.max_iterations && B < kMaxBatch && batchable(t + B)) ++B;
            double rb_ms = 0.0;
            bool super = false;
            // timing events of batch member k (single iterations keep e0..e7)
            auto ev = [&](int k, int i) { return B == 1 ? g.event(i) : g.batch_event(8 * k + i); };
            for (int k = 0; k < B; ++k) {
            const uint64_t u = t + k;
            const int mode = mode_for(cfg.scheme, u, cfg.alpha);
            const bool approx = mode == GG_MODE_APPROXIMATE;
            super = mode == GG_MODE_SUPERSTEP;
            const ListMeta& L = approx ? sp : g.full;
            EdgeArgs<P, W> ea{};
            ea.prog = prog;
            ea.src = approx ? s_src : g.src;
            ea.src_quads = approx && sp_quads(g);  // as the compaction wrote it
            ea.w = static_cast<const W*>(approx ? s_w : g.w);
            ea.run_i = L.run_i;
            ea.nz_row = approx ? L.nz_vid : nullptr;  // the full list's rows are its nz indices
            ea.nz_start = L.nz_start;
            ea.pad = L.pad;
            ea.e_end = L.e_end();
            ea.ntasks = L.ntasks;
            ea.nruns = L.nruns;
            ea.a_off = a_off;
            ea.st_cur = st;
            ea.msg_cur = msg;
            ea.hot_limit = hot_limit;
            ea.l2_limit = l2_limit;
            ea.cold_last = msgs_fit_l2 ? 1u : 0u;
            ea.acc_out = acc_out;
            ea.hv = hv;
            ea.tv = tv;
            if (chain) {
                ea.cdesc = reinterpret_cast<ulonglong2*>(chain);
                ea.chain = reinterpret_cast<uint32_t*>(chain);
                ea.ticket = reinterpret_cast<uint32_t*>(chain + L.ntasks * kSlot);
            }
            ea.bitmap = bitmap;
            ea.theta = cfg.theta;
            {
                const bool normal = cfg.theta > 0x1p-900 && cfg.theta < 0x1p+900;
                ea.theta_hi = normal ? cfg.theta * (1.0 + 0x1p-40) : std::nan("");
                ea.theta_lo = normal ? cfg.theta * (1.0 - 0x1p-40) : std::nan("");
                // accumulators whose products with theta_hi/lo stay inside
                // [2^-998, 2^998]: binary exponents [lo_e, hi_e]
                ea.pn_lo = ea.pn_span = 0;
                if (normal) {
                    int et = 0;
                    (void)std::frexp(cfg.theta, &et);  // theta = f * 2^et, f in [0.5, 1)
                    int lo_e = -998 - (et - 1) + 1, hi_e = 998 - et - 1;
                    lo_e = std::max(lo_e, -1022);
                    hi_e = std::min(hi_e, 1023);
                    if (lo_e <= hi_e) {
                        ea.pn_lo = (uint32_t)(lo_e + 1023) << 20;
                        ea.pn_span = (uint32_t)(hi_e - lo_e + 1) << 20;
                    }
                }
            }
            ea.stop_if = k ? ring + (u - 1) % kRing : nullptr;
            VertexArgs<P, W> va{};
            va.prog = prog;
            va.n = n;
            va.v_begin = (uint32_t)g.v_begin;
            va.nloc = (uint32_t)nloc;
            va.nrows = (uint32_t)R;
            va.off = approx ? s_off : g.full.nz_start;
            va.pad = L.pad;
            va.a_off = a_off;
            va.st = st;
            va.prop = prop;
            va.msg = msg;
            va.vid_of_p = g.vid_of_p;
            va.slot_p = g.slot_p;
            va.deg_p = g.deg_p;
            va.acc_out = acc_out;
            va.hv = hv;
            va.tv = tv;
            IterCounters* ctr = ring + u % kRing;
            va.npeers = 0;
            if (fused) {
                va.npeers = g.nranks;
                va.self = g.rank;
                for (int r = 0; r < g.nranks; ++r) va.peers[r] = static_cast<Msg*>(g.peer_msg[r]);
                const uint64_t* gr = g.gather_ranges.data() + 4 * g.rank;
                va.gb0 = gr[0]; va.ge0 = gr[1]; va.gb1 = gr[2]; va.ge1 = gr[3];
            }
            va.ctr = ctr;
            va.ctr_next = ring + (u + 1) % kRing;
            va.ctr_prev = ring + (u - 1) % kRing;  // u = 1: slot 0 = "all statuses active"
            va.stop_if = ea.stop_if;

            if (timing) GGB_CUDA(cudaEventRecord(ev(k, 0), g.stream));
            if (L.ntasks) {
                // every edge of the sparsified list (and of the full list under
                // the accurate scheme) belongs to a processed vertex
                const bool all_proc = approx || cfg.scheme == GG_SCHEME_ACCURATE;
                if (super) {
                    GGB_CUDA(cudaMemsetAsync(chain, 0, L.ntasks * kSlot + 4, g.stream));
                    launch_chain(g, ea, cap);
                } else if (all_proc && nhot) {
                    if constexpr (kHotOK) launch_edge_hot(g, ea, nhot, cap);
                }
                else if (all_proc) launch_edge<kEdgePlain>(g, ea, cap);
                else launch_edge<kEdgeCheck>(g, ea, cap);
                ++launches;
            }
            if (timing) GGB_CUDA(cudaEventRecord(ev(k, 1), g.stream));
            // fused exchange: every rank's gathers are done before any vertex
            // kernel writes the replicas
            if (fused) exchange_barrier(g);
            {
                const unsigned vg = capped(grid1d(nloc), cap);
                if (fused) {
                    if (super) vertex_kernel<P, W, true, true><<<vg, 256, 0, g.stream>>>(va);
                    else vertex_kernel<P, W, false, true><<<vg, 256, 0, g.stream>>>(va);
                } else {
                    if (super) vertex_kernel<P, W, true><<<vg, 256, 0, g.stream>>>(va);
                    else vertex_kernel<P, W, false><<<vg, 256, 0, g.stream>>>(va);
                }
            }
            GGB_CUDA(cudaGetLastError());
            ++launches;
            if (timing) GGB_CUDA(cudaEventRecord(ev(k, 2), g.stream));
            if (super) {  // new flag set -> new sparsified CSC (engine.hpp:207-214)
                kept = rebuild_sparse(g, bitmap, s_off, s_src, s_w, sp, timing ? e4 : nullptr,
                                      timing ? e5 : nullptr, &launches);
                // bad-vertex rescan against the kept counts; exits at once on
                // the device unless the vertex kernel saw an invalid property
                launch_superstep_invalid(g, st, s_off, ctr);
                ++launches;
            }
            if (g.nranks > 1) {  // property exchange + counter allreduce
                if (timing) GGB_CUDA(cudaEventRecord(ev(k, 6), g.stream));
                if (!fused) exchange_slices(g, msg, sizeof(Msg), /*slots=*/true);
                exchange_counters(g, ctr);
                if (timing) GGB_CUDA(cudaEventRecord(ev(k, 7), g.stream));
            }
            }  // batch member k
            GGB_CUDA(cudaMemcpyAsync(h_ring, ring, kRing * sizeof(IterCounters),
                                     cudaMemcpyDeviceToHost, g.stream));
            GGB_CUDA(cudaStreamSynchronize(g.stream));
            const double batch_wall =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (timing && super) rb_ms = event_ms(e4, e5);
            for (int k = 0; k < B; ++k) {
                const uint64_t u = t + k;
                const IterCounters& hc = h_ring[u % kRing];
                const int mode = mode_for(cfg.scheme, u, cfg.alpha);
                const bool approx = mode == GG_MODE_APPROXIMATE;
                if (hc.bad_min != 0xffffffffu) {  // engine.hpp:226-233
                    Error e(GG_INVALID_PROPERTY,
                            "invalid property at iteration " + std::to_string(u) + ", vertex " +
                                std::to_string(hc.bad_min));
                    e.iteration = u;
                    e.vertex = hc.bad_min;
                    if (io.sum) {
                        io.sum->iterations_run = iterations_run;
                        io.sum->total_processed_edges = total_edges;
                        io.sum->kernel_launches = (uint32_t)launches;
                    }
                    throw e;
                }
                // host wall time: exact for single iterations, the batch's
                // share for batch members (each member's GPU time is in the
                // kernel fields when timing is on)
                const double wall = batch_wall / B;
                if (u - 1 < io.rec_cap && io.recs) {  // engine.hpp:235-236
                    gg_iter_record& r = io.recs[u - 1];
                    r.mode = mode;
                    r.processed_edges = hc.gathered;
                    r.active_vertices = hc.processed;
                    r.wall_seconds = wall;
                    r.edge_ms = timing ? event_ms(ev(k, 0), ev(k, 1)) : 0.0;
                    r.vertex_ms = timing ? event_ms(ev(k, 1), ev(k, 2)) : 0.0;
                    r.kernel_ms = r.edge_ms + r.vertex_ms;
                    r.rebuild_ms = rb_ms;
                    r.exchange_ms = (timing && g.nranks > 1) ? event_ms(ev(k, 6), ev(k, 7)) : 0.0;
                    // per-rank algorithmic bytes of this rank's launches
                    const uint64_t local_edges = approx ? kept : g.e_loc;
                    r.edge_bytes = edge_bytes(local_edges, super);
                    // positions the vertex kernel walked: the rows, and the
                    // in-degree-0 tail when one of them was active (always at t = 1)
                    r.vertex_bytes = vertex_bytes(prev_empty_active ? nloc : R);
                    r.algo_bytes = r.edge_bytes + r.vertex_bytes;
                }
                prev_empty_active = hc.empty_active != 0;
                iterations_run = u;
                total_edges += hc.gathered;
                total_wall += wall;
                if (!hc.changed) {                      // engine.hpp:240
                    done = true;
                    break;
                }
            }
            t += B;
        }

        // final properties (engine.hpp:243): owned positions back to vertex
        // order, gathered from every rank
        Prop* final_all = ws.get<Prop>("final", n);
        if (nloc) {
            to_vertex_order_kernel<Prop><<<grid1d(nloc), 256, 0, g.stream>>>(prop, g.vid_of_p, nloc,
                                                                             final_all + g.v_begin);
            GGB_CUDA(cudaGetLastError());
            ++launches;
        }
        if (g.nranks > 1) exchange_slices(g, final_all, sizeof(Prop));
        g.project_last = [&g, prog, final_all, n]() -> const double* {  // metrics.cu
            double* proj = g.ws.get<double>("proj", n + 1);
            export_kernel<P><<<grid1d(n), 256, 0, g.stream>>>(prog, final_all, n, 1, proj);
            GGB_CUDA(cudaGetLastError());
            GGB_CUDA(cudaStreamSynchronize(g.stream));
            return proj;
        };
        if (io.out_props && !(io.opts && io.opts->device_output)) {
            if constexpr (requires { P::kRawOutput; }) {  // WCC: uint32 labels as-is
                GGB_CUDA(cudaMemcpyAsync(io.out_props, final_all, n * 4, cudaMemcpyDeviceToHost,
                                         g.stream));
            } else if constexpr (std::is_same_v<Prop, double>) {  // PR, f64 SSSP: the doubles as-is
                GGB_CUDA(cudaMemcpyAsync(io.out_props, final_all, n * 8, cudaMemcpyDeviceToHost,
                                         g.stream));
            } else {
                double* stage = ws.get<double>("export", n * io.out_states);
                export_kernel<P><<<grid1d(n), 256, 0, g.stream>>>(prog, final_all, n, io.out_states,
                                                                   stage);
                GGB_CUDA(cudaGetLastError());
                ++launches;
                GGB_CUDA(cudaMemcpyAsync(io.out_props, stage, n * io.out_states * 8,
                                         cudaMemcpyDeviceToHost, g.stream));
            }
        }
        if (io.opts && io.opts->out_flags) {
            if (sparse)
                GGB_CUDA(cudaMemcpyAsync(io.opts->out_flags, bitmap, nwords * 4,
                                         cudaMemcpyDeviceToHost, g.stream));
            else
                for (uint64_t i = 0; i < nwords; ++i)
                    io.opts->out_flags[i] = (i + 1 < nwords || g.e_loc % 32 == 0)
                                                ? 0xffffffffu : ((1u << (g.e_loc % 32)) - 1u);
        }
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        if (io.sum) {
            io.sum->iterations_run = iterations_run;
            io.sum->total_processed_edges = total_edges;
            io.sum->total_wall_seconds = total_wall;
            io.sum->kept_edges = kept;
            io.sum->kernel_launches = (uint32_t)launches;
            io.sum->exchange_fused = fused ? 1u : 0u;
        }
    }
};

}  // namespace ggb
