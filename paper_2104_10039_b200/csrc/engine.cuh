// engine.cuh — host side of the engine: gg::run (engine.hpp:141-249) driving
// the device kernels. Instantiated per (program, weight type) in capi.cu.
#pragma once

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
    void* out_props = nullptr;   // host: double[n*S] or uint32[n] (kRawOut)
    int out_states = 1;
};

template <class P>
__global__ void init_kernel(P prog, uint64_t n, uint32_t v_begin, uint32_t nloc,
                            const uint32_t* __restrict__ outdeg,
                            typename P::Message* __restrict__ msg,
                            typename P::Property* __restrict__ prop, uint8_t* __restrict__ st) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const typename P::Property p = prog.init_property((uint32_t)v, n);  // engine.hpp:164
        uint32_t deg = 0;
        if constexpr (P::kNeedsDegree) deg = outdeg[v];
        msg[v] = prog.message(p, deg);
        if (v >= v_begin && v < (uint64_t)v_begin + nloc) {
            if constexpr (!P::kMsgIsProp) prop[v - v_begin] = p;
            st[v - v_begin] = kStActive;  // status starts at 1 (engine.hpp:166)
        }
    }
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

struct EventPair {
    cudaEvent_t a = nullptr, b = nullptr;
    void make() {
        if (!a) {
            GGB_CUDA(cudaEventCreate(&a));
            GGB_CUDA(cudaEventCreate(&b));
        }
    }
    ~EventPair() {
        if (a) cudaEventDestroy(a);
        if (b) cudaEventDestroy(b);
    }
    double ms() const {
        float f = 0.f;
        GGB_CUDA(cudaEventElapsedTime(&f, a, b));
        return (double)f;
    }
};

template <class P, class W>
struct Engine {
    using Prop = typename P::Property;
    using Msg = typename P::Message;
    using Acc = typename P::Accum;
    static constexpr int U = sizeof(Msg) <= 8 ? 4 : 2;

    static int grid_main(DevGraph& g, bool super) {
        static int cached[2] = {0, 0};
        int& c = cached[super ? 1 : 0];
        if (!c) {
            const void* k = super ? (const void*)iteration_kernel<P, W, true, U>
                                  : (const void*)iteration_kernel<P, W, false, U>;
            c = occupancy_grid(k, kBlockThreads, 0, g.num_sms);
        }
        return c;
    }

    // Algorithmic HBM bytes of one gather launch (SURVEY §8(d) byte formula:
    // E_p * b_e + N * b_v, superstep adds the bitmap write E_p / 8).
    static uint64_t algo_bytes(uint64_t edges, uint64_t nloc, bool super) {
        const uint64_t be = 4 + sizeof(Msg) + (uint64_t)weight_bytes<W>();
        uint64_t bv = 8 + 2 + 2 * sizeof(Prop) + (P::kMsgIsProp ? 0 : sizeof(Msg)) +
                      (P::kNeedsDegree ? 4 : 0);
        if constexpr (requires { P::kReadsPrior; }) bv += 8;
        uint64_t b = edges * be + nloc * bv;
        if (super) b += edges / 8;
        return b;
    }

    static void run(DevGraph& g, const P& prog, RunIO& io) {
        const gg_engine_config& cfg = *io.cfg;
        const bool timing = io.opts && io.opts->timing;
        GGB_CUDA(cudaSetDevice(g.device));
        const uint64_t n = g.n, nloc = g.nloc;
        const bool sparse = cfg.scheme != GG_SCHEME_ACCURATE;
        int launches = 0;
        Workspace& ws = g.ws;

        Msg* msg[2] = {ws.get<Msg>("msg0", n), ws.get<Msg>("msg1", n)};
        Prop* prop = P::kMsgIsProp ? nullptr : ws.get<Prop>("prop", nloc);
        uint8_t* st[2] = {ws.get<uint8_t>("st0", nloc + 1), ws.get<uint8_t>("st1", nloc + 1)};
        IterCounters* ctr = ws.get<IterCounters>("ctr", 1);
        const uint64_t nwords = (g.e_loc + 31) / 32;
        const size_t wsz = (size_t)weight_bytes<W>();
        uint32_t* bitmap = nullptr;
        uint64_t* s_off = nullptr;
        uint32_t* s_src = nullptr;
        void* s_w = nullptr;
        TaskList sp;
        const uint64_t nwin = (nloc + kWindow - 1) / kWindow;
        // partial slots: the full list has the most multi-chunk tasks
        Acc* partials = ws.get<Acc>("partials", ((uint64_t)g.full.nmtasks + 1) * kWindow);
        uint32_t* tickets;
        {
            const bool fresh = ws.bufs.find("tickets") == ws.bufs.end() ||
                               ws.bufs["tickets"].bytes < (nwin + 1) * 4;
            tickets = ws.get<uint32_t>("tickets", nwin + 1);
            if (fresh) GGB_CUDA(cudaMemsetAsync(tickets, 0, (nwin + 1) * 4, g.stream));
        }
        IterCounters* h_ctr = nullptr;
        GGB_CUDA(cudaHostAlloc(&h_ctr, sizeof(IterCounters), cudaHostAllocDefault));
        struct HostFree {
            IterCounters* p;
            ~HostFree() { cudaFreeHost(p); }
        } hf{h_ctr};

        EventPair ev_k, ev_rb, ev_x;
        if (timing) { ev_k.make(); ev_rb.make(); ev_x.make(); }

        init_kernel<P><<<grid1d(n), 256, 0, g.stream>>>(prog, n, (uint32_t)g.v_begin,
                                                         (uint32_t)nloc, g.outdeg, msg[0], prop,
                                                         st[0]);
        GGB_CUDA(cudaGetLastError());
        ++launches;
        uint64_t kept = g.e_loc;
        if (sparse) {  // engine.hpp:151-161
            bitmap = ws.get<uint32_t>("bitmap", nwords + 1);
            s_off = ws.get<uint64_t>("s_off", nloc + 1);
            s_src = ws.get<uint32_t>("s_src", g.e_loc + 1);
            s_w = wsz ? ws.get("s_w", (g.e_loc + 1) * wsz) : nullptr;
            sparsify_bitmap(g, bitmap, cfg.sigma, cfg.seed, false);
            ++launches;
            kept = rebuild_sparse(g, bitmap, s_off, s_src, s_w, sp, "sp", nullptr, nullptr, &launches);
        }
        const uint64_t* a_off = sparse ? s_off : g.off;

        IterArgs<P, W> a{};
        a.prog = prog;
        a.n = n;
        a.v_begin = (uint32_t)g.v_begin;
        a.nloc = (uint32_t)nloc;
        a.a_off = a_off;
        a.prop = prop;
        a.outdeg = g.outdeg;
        a.bitmap = bitmap;
        a.theta = cfg.theta;
        a.partials = partials;
        a.win_ticket = tickets;
        a.ctr = ctr;

        int cur = 0;
        uint64_t iterations_run = 0, total_edges = 0;
        double total_wall = 0.0;
        for (uint64_t t = 1; t <= cfg.max_iterations; ++t) {  // engine.hpp:177
            const auto t0 = std::chrono::steady_clock::now();
            const int mode = mode_for(cfg.scheme, t, cfg.alpha);
            const bool approx = mode == GG_MODE_APPROXIMATE;
            const bool super = mode == GG_MODE_SUPERSTEP;
            if (approx) {
                a.g_off = s_off; a.g_src = s_src; a.g_w = static_cast<const W*>(s_w);
                a.tasks = sp.tasks; a.ntasks = sp.ntasks;
            } else {
                a.g_off = g.off; a.g_src = g.src; a.g_w = static_cast<const W*>(g.w);
                a.tasks = g.full.tasks; a.ntasks = g.full.ntasks;
            }
            a.msg_cur = msg[cur]; a.msg_next = msg[cur ^ 1];
            a.st_cur = st[cur]; a.st_next = st[cur ^ 1];
            GGB_CUDA(cudaMemsetAsync(ctr, 0, sizeof(IterCounters), g.stream));
            GGB_CUDA(cudaMemsetAsync(&ctr->bad_min, 0xff, 4, g.stream));
            if (timing) GGB_CUDA(cudaEventRecord(ev_k.a, g.stream));
            if (super) {
                iteration_kernel<P, W, true, U><<<grid_main(g, true), kBlockThreads, 0, g.stream>>>(a);
                GGB_CUDA(cudaGetLastError());
                ++launches;
                if (g.full.nmtasks) {
                    superstep_hub_kernel<P, W, U><<<grid_main(g, true), kBlockThreads, 0, g.stream>>>(
                        a, g.full.mtasks, g.full.nmtasks);
                    GGB_CUDA(cudaGetLastError());
                    ++launches;
                }
            } else {
                iteration_kernel<P, W, false, U><<<grid_main(g, false), kBlockThreads, 0, g.stream>>>(a);
                GGB_CUDA(cudaGetLastError());
                ++launches;
            }
            if (timing) GGB_CUDA(cudaEventRecord(ev_k.b, g.stream));
            double rb_ms = 0.0;
            if (super) {  // new flag set -> new sparsified CSC (engine.hpp:207-214)
                kept = rebuild_sparse(g, bitmap, s_off, s_src, s_w, sp, "sp",
                                      timing ? ev_rb.a : nullptr, timing ? ev_rb.b : nullptr,
                                      &launches);
                if (timing) rb_ms = ev_rb.ms();
                GGB_CUDA(cudaMemcpyAsync(h_ctr, ctr, sizeof(IterCounters), cudaMemcpyDeviceToHost,
                                         g.stream));
                GGB_CUDA(cudaStreamSynchronize(g.stream));
                if (h_ctr->any_invalid) {
                    launch_superstep_invalid(g, st[cur], st[cur ^ 1], s_off, ctr);
                    ++launches;
                }
            }
            if (g.nranks > 1) {  // property exchange + counter allreduce
                if (timing) GGB_CUDA(cudaEventRecord(ev_x.a, g.stream));
                exchange_slices(g, msg[cur ^ 1], sizeof(Msg));
                exchange_counters(g, ctr);
                if (timing) GGB_CUDA(cudaEventRecord(ev_x.b, g.stream));
            }
            GGB_CUDA(cudaMemcpyAsync(h_ctr, ctr, sizeof(IterCounters), cudaMemcpyDeviceToHost,
                                     g.stream));
            GGB_CUDA(cudaStreamSynchronize(g.stream));
            const double wall =
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
            if (h_ctr->bad_min != 0xffffffffu) {  // engine.hpp:226-233
                Error e(GG_INVALID_PROPERTY,
                        "invalid property at iteration " + std::to_string(t) + ", vertex " +
                            std::to_string(h_ctr->bad_min));
                e.iteration = t;
                e.vertex = h_ctr->bad_min;
                if (io.sum) {
                    io.sum->iterations_run = iterations_run;
                    io.sum->total_processed_edges = total_edges;
                    io.sum->kernel_launches = (uint32_t)launches;
                }
                throw e;
            }
            if (t - 1 < io.rec_cap && io.recs) {  // engine.hpp:235-236
                gg_iter_record& r = io.recs[t - 1];
                r.mode = mode;
                r.processed_edges = h_ctr->gathered;
                r.active_vertices = h_ctr->processed;
                r.wall_seconds = wall;
                r.kernel_ms = timing ? ev_k.ms() : 0.0;
                r.rebuild_ms = rb_ms;
                r.exchange_ms = (timing && g.nranks > 1) ? ev_x.ms() : 0.0;
                r.algo_bytes = algo_bytes(h_ctr->gathered, g.n, super);
            }
            iterations_run = t;
            total_edges += h_ctr->gathered;
            total_wall += wall;
            cur ^= 1;                               // engine.hpp:238-239
            if (!h_ctr->changed) break;             // engine.hpp:240
        }

        // final properties (engine.hpp:243)
        const Prop* final_local;
        Prop* final_all;
        if constexpr (P::kMsgIsProp) {
            final_all = msg[cur];  // exchanged every iteration: full on every rank
            final_local = final_all + g.v_begin;
        } else {
            final_all = ws.get<Prop>("final", n);
            GGB_CUDA(cudaMemcpyAsync(final_all + g.v_begin, prop, nloc * sizeof(Prop),
                                     cudaMemcpyDeviceToDevice, g.stream));
            if (g.nranks > 1) exchange_slices(g, final_all, sizeof(Prop));
            final_local = prop;
        }
        (void)final_local;
        if (io.out_props && !(io.opts && io.opts->device_output)) {
            if constexpr (requires { P::kRawOutput; }) {  // WCC: uint32 labels as-is
                GGB_CUDA(cudaMemcpyAsync(io.out_props, final_all, n * 4, cudaMemcpyDeviceToHost,
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
        }
    }
};

}  // namespace ggb
