// exchange.cu — NCCL transport for the partitioned engine (see exchange.cuh).
#include <dlfcn.h>

#include <algorithm>
#include <cstddef>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include "exchange.cuh"
#include "kernels.cuh"

namespace ggb {

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    static std::string load_error;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            load_error = dlerror() ? dlerror() : "dlopen libnccl.so.2 failed";
            return;
        }
#define GGB_SYM(field, name) api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name))
        GGB_SYM(GetUniqueId, "ncclGetUniqueId");
        GGB_SYM(CommInitRank, "ncclCommInitRank");
        GGB_SYM(CommDestroy, "ncclCommDestroy");
        GGB_SYM(Broadcast, "ncclBroadcast");
        GGB_SYM(AllReduce, "ncclAllReduce");
        GGB_SYM(GroupStart, "ncclGroupStart");
        GGB_SYM(GroupEnd, "ncclGroupEnd");
        GGB_SYM(GetErrorString, "ncclGetErrorString");
#undef GGB_SYM
    });
    if (!api.GetUniqueId || !api.CommInitRank || !api.Broadcast || !api.AllReduce)
        throw Error(GG_NCCL, "NCCL unavailable: " + load_error);
    return api;
}

// In-process transport: the ranks are host threads of one process, each
// with its own DevGraph and stream (any devices, including one shared
// device). Collectives are host barriers plus device-to-device copies; no
// kernel ever waits on another rank's kernel. It runs the partitioned engine
// end to end where only one GPU is available (tests/test_gpu_multirank.py);
// the NCCL transport carries the same calls across processes and GPUs.
struct LocalGroup {
    explicit LocalGroup(int n) : nranks(n), bufs(n), vals(n), ctrs(n) {}
    int nranks;
    std::mutex m;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t phase = 0;
    std::vector<void*> bufs;
    std::vector<uint64_t> vals;
    std::vector<IterCounters> ctrs;
    void barrier() {
        std::unique_lock<std::mutex> lk(m);
        const uint64_t my = phase;
        if (++arrived == nranks) {
            arrived = 0;
            ++phase;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return phase != my; });
        }
    }
};

// element ranges of rank r's slice: the vertex range, or (slots) the slot
// ranges of its gathered messages (graph.cuh gather_ranges)
static inline int ranges_of(const DevGraph& g, int r, bool slots, uint64_t (&b)[2], uint64_t (&e)[2]) {
    if (slots && !g.gather_ranges.empty()) {
        b[0] = g.gather_ranges[4 * r]; e[0] = g.gather_ranges[4 * r + 1];
        b[1] = g.gather_ranges[4 * r + 2]; e[1] = g.gather_ranges[4 * r + 3];
        return 2;
    }
    b[0] = g.bounds[r];
    e[0] = g.bounds[r + 1];
    return 1;
}

static void local_slices(DevGraph& g, LocalGroup& L, void* buf, size_t elem, bool slots) {
    GGB_CUDA(cudaStreamSynchronize(g.stream));  // this rank's slice is written
    L.bufs[g.rank] = buf;
    L.barrier();
    for (int r = 0; r < g.nranks; ++r) {
        if (r == g.rank) continue;
        uint64_t b[2], e[2];
        const int k = ranges_of(g, r, slots, b, e);
        for (int i = 0; i < k; ++i) {
            if (e[i] == b[i]) continue;
            GGB_CUDA(cudaMemcpyAsync(static_cast<char*>(buf) + b[i] * elem,
                                     static_cast<const char*>(L.bufs[r]) + b[i] * elem,
                                     (e[i] - b[i]) * elem, cudaMemcpyDefault, g.stream));
        }
    }
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    L.barrier();  // nobody rewrites its buffer while another rank copies from it
}

static void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) {
        const char* s = nccl().GetErrorString ? nccl().GetErrorString(r) : "?";
        throw Error(GG_NCCL, std::string(what) + ": " + s);
    }
}

void exchange_slices(DevGraph& g, void* global_buf, size_t elem_size, bool slots) {
    if (g.nranks <= 1) return;
    if (g.exchange && g.exchange->local)
        return local_slices(g, *g.exchange->local, global_buf, elem_size, slots);
    if (!g.exchange || !g.exchange->comm) throw Error(GG_NCCL, "multi-rank graph without exchange");
    const NcclApi& api = nccl();
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < g.nranks; ++r) {
        uint64_t b[2], e[2];
        const int k = ranges_of(g, r, slots, b, e);
        for (int i = 0; i < k; ++i) {
            if (e[i] == b[i]) continue;
            char* p = static_cast<char*>(global_buf) + b[i] * elem_size;
            nccl_check(api.Broadcast(p, p, (e[i] - b[i]) * elem_size, ncclChar, r, g.exchange->comm,
                                     g.stream), "ncclBroadcast");
        }
    }
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

// every rank's `local` (allgather of one u64 per rank)
static std::vector<uint64_t> exchange_all(DevGraph& g, uint64_t local) {
    if (g.nranks <= 1) return {local};
    if (g.exchange && g.exchange->local) {
        LocalGroup& L = *g.exchange->local;
        L.vals[g.rank] = local;
        L.barrier();
        std::vector<uint64_t> h(L.vals.begin(), L.vals.end());
        L.barrier();
        return h;
    }
    const NcclApi& api = nccl();
    uint64_t* d = g.ws.get<uint64_t>("xbase", (uint64_t)g.nranks + 1);
    GGB_CUDA(cudaMemcpyAsync(d + g.rank, &local, 8, cudaMemcpyHostToDevice, g.stream));
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < g.nranks; ++r)
        nccl_check(api.Broadcast(d + r, d + r, 1, ncclUint64, r, g.exchange->comm, g.stream),
                   "ncclBroadcast(kept)");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    std::vector<uint64_t> h(g.nranks);
    GGB_CUDA(cudaMemcpyAsync(h.data(), d, 8 * g.nranks, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    return h;
}

// every rank's n bytes, in rank order (setup only)
static std::vector<uint8_t> exchange_all_bytes(DevGraph& g, const void* mine, size_t n) {
    std::vector<uint8_t> out(g.nranks * n);
    if (g.exchange && g.exchange->local) {
        LocalGroup& L = *g.exchange->local;
        L.bufs[g.rank] = const_cast<void*>(mine);
        L.barrier();
        for (int r = 0; r < g.nranks; ++r) std::memcpy(out.data() + r * n, L.bufs[r], n);
        L.barrier();
        return out;
    }
    const NcclApi& api = nccl();
    uint8_t* d = g.ws.get<uint8_t>("xbytes", g.nranks * n);
    GGB_CUDA(cudaMemcpyAsync(d + g.rank * n, mine, n, cudaMemcpyHostToDevice, g.stream));
    nccl_check(api.GroupStart(), "ncclGroupStart");
    for (int r = 0; r < g.nranks; ++r)
        nccl_check(api.Broadcast(d + r * n, d + r * n, n, ncclChar, r, g.exchange->comm, g.stream),
                   "ncclBroadcast(bytes)");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
    GGB_CUDA(cudaMemcpyAsync(out.data(), d, g.nranks * n, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    return out;
}

// true on every rank iff `ok` on every rank
static bool exchange_all_true(DevGraph& g, bool ok) {
    for (uint64_t v : exchange_all(g, ok ? 1 : 0))
        if (!v) return false;
    return true;
}

void exchange_release_peers(DevGraph& g) {
    for (void* p : g.ipc_opened) cudaIpcCloseMemHandle(p);
    g.ipc_opened.clear();
    g.peer_msg.clear();
    g.peer_msg_for = nullptr;
    g.peer_msg_bytes = 0;
}

void* exchange_msg_buffer(DevGraph& g, size_t bytes) {
    if (g.nranks > 1 && g.exchange && g.exchange->comm && g.exchange->fused) {
        if (g.ipc_msg_bytes < bytes) {
            // every rank grows its buffer in the same run (same n, same
            // message type), and re-registers its peers before the run uses them
            exchange_release_peers(g);
            if (g.ipc_msg) GGB_CUDA(cudaFree(g.ipc_msg));
            g.ipc_msg = nullptr;
            GGB_CUDA(cudaMalloc(&g.ipc_msg, bytes ? bytes : 16));
            g.ipc_msg_bytes = bytes;
        }
        return g.ipc_msg;
    }
    return g.ws.get("msg", bytes);
}

bool exchange_register_peers(DevGraph& g, void* msg, size_t bytes) {
    if (g.nranks <= 1 || !g.exchange) return false;
    if (!g.peer_msg.empty() && g.peer_msg_for == msg && g.peer_msg_bytes >= bytes) return true;
    exchange_release_peers(g);
    // every step ends in an agreement round: all ranks take the same path
    const bool want = g.exchange->fused && g.nranks <= kMaxPeers;
    if (!exchange_all_true(g, want)) return false;
    std::vector<void*> ptrs(g.nranks, nullptr);
    bool ok = true;
    if (g.exchange->local) {
        GGB_CUDA(cudaStreamSynchronize(g.stream));  // init writes of this rank's replica
        struct Rec { void* p; int device; };
        const Rec mine{msg, g.device};
        const std::vector<uint8_t> all = exchange_all_bytes(g, &mine, sizeof(Rec));
        for (int r = 0; r < g.nranks; ++r) {
            Rec x;
            std::memcpy(&x, all.data() + r * sizeof(Rec), sizeof(Rec));
            ptrs[r] = x.p;
            if (x.device == g.device) continue;
            int can = 0;
            if (cudaDeviceCanAccessPeer(&can, g.device, x.device) != cudaSuccess || !can) {
                cudaGetLastError();
                ok = false;
                continue;
            }
            const cudaError_t e = cudaDeviceEnablePeerAccess(x.device, 0);
            if (e != cudaSuccess) {
                cudaGetLastError();  // cudaErrorPeerAccessAlreadyEnabled is fine
                if (e != cudaErrorPeerAccessAlreadyEnabled) ok = false;
            }
        }
    } else {
        struct Rec { uint64_t ok; cudaIpcMemHandle_t h; };
        Rec mine{};
        mine.ok = msg == g.ipc_msg && cudaIpcGetMemHandle(&mine.h, msg) == cudaSuccess;
        if (!mine.ok) cudaGetLastError();
        const std::vector<uint8_t> all = exchange_all_bytes(g, &mine, sizeof(Rec));
        for (int r = 0; r < g.nranks && ok; ++r) {
            Rec x;
            std::memcpy(&x, all.data() + r * sizeof(Rec), sizeof(Rec));
            if (!x.ok) ok = false;
        }
        for (int r = 0; r < g.nranks && ok; ++r) {
            if (r == g.rank) {
                ptrs[r] = msg;
                continue;
            }
            Rec x;
            std::memcpy(&x, all.data() + r * sizeof(Rec), sizeof(Rec));
            void* p = nullptr;
            if (cudaIpcOpenMemHandle(&p, x.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
                cudaGetLastError();
                ok = false;
                break;
            }
            g.ipc_opened.push_back(p);
            ptrs[r] = p;
        }
    }
    if (!exchange_all_true(g, ok)) {
        exchange_release_peers(g);
        return false;
    }
    g.peer_msg = ptrs;
    g.peer_msg_for = msg;
    g.peer_msg_bytes = bytes;
    return true;
}

void exchange_barrier(DevGraph& g) {
    if (g.nranks <= 1) return;
    if (g.exchange && g.exchange->local) {
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        g.exchange->local->barrier();
        return;
    }
    // a one-word all-reduce completes on no rank before every rank has
    // reached it in stream order
    uint32_t* d = g.ws.get<uint32_t>("xbarrier", 1);
    nccl_check(nccl().AllReduce(d, d, 1, ncclUint32, ncclMax, g.exchange->comm, g.stream),
               "ncclAllReduce(barrier)");
}

uint64_t exchange_exclusive_base(DevGraph& g, uint64_t local) {
    if (g.nranks <= 1) return 0;
    const std::vector<uint64_t> h = exchange_all(g, local);
    uint64_t base = 0;
    for (int r = 0; r < g.rank; ++r) base += h[r];
    return base;
}

uint64_t exchange_sum(DevGraph& g, uint64_t local) {
    if (g.nranks <= 1) return local;
    uint64_t s = 0;
    for (uint64_t v : exchange_all(g, local)) s += v;
    return s;
}

__global__ void add_u32_kernel(uint32_t* __restrict__ acc, const uint32_t* __restrict__ x,
                               uint64_t count) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        acc[i] += x[i];
}

void exchange_allreduce_u32(DevGraph& g, uint32_t* buf, uint64_t count) {
    if (g.nranks <= 1 || !count) return;
    if (g.exchange && g.exchange->local) {
        LocalGroup& L = *g.exchange->local;
        // every rank publishes a copy of its input, then sums the others' copies
        uint32_t* mine = g.ws.get<uint32_t>("xred.mine", count);
        uint32_t* tmp = g.ws.get<uint32_t>("xred.tmp", count);
        GGB_CUDA(cudaMemcpyAsync(mine, buf, count * 4, cudaMemcpyDeviceToDevice, g.stream));
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        L.bufs[g.rank] = mine;
        L.barrier();
        const unsigned grid = (unsigned)std::min<uint64_t>((count + 255) / 256, 148ull * 16);
        for (int r = 0; r < g.nranks; ++r) {
            if (r == g.rank) continue;
            GGB_CUDA(cudaMemcpyAsync(tmp, L.bufs[r], count * 4, cudaMemcpyDefault, g.stream));
            add_u32_kernel<<<grid, 256, 0, g.stream>>>(buf, tmp, count);
            GGB_CUDA(cudaGetLastError());
        }
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        L.barrier();  // nobody frees or rewrites its copy while another rank reads it
        return;
    }
    nccl_check(nccl().AllReduce(buf, buf, count, ncclUint32, ncclSum, g.exchange->comm, g.stream),
               "allreduce(u32)");
}

void exchange_counters(DevGraph& g, void* ctr_v) {
    if (g.nranks <= 1) return;
    if (g.exchange && g.exchange->local) {
        LocalGroup& L = *g.exchange->local;
        IterCounters* d = static_cast<IterCounters*>(ctr_v);
        GGB_CUDA(cudaMemcpyAsync(&L.ctrs[g.rank], d, sizeof(IterCounters), cudaMemcpyDeviceToHost,
                                 g.stream));
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        L.barrier();
        IterCounters s{};
        s.bad_min = 0xffffffffu;
        for (const IterCounters& c : L.ctrs) {  // same reductions as the NCCL path
            s.gathered += c.gathered;
            s.processed += c.processed;
            s.changed += c.changed;
            s.any_invalid += c.any_invalid;
            s.empty_active += c.empty_active;
            s.bad_min = std::min(s.bad_min, c.bad_min);
        }
        L.barrier();
        GGB_CUDA(cudaMemcpyAsync(d, &s, sizeof(IterCounters), cudaMemcpyHostToDevice, g.stream));
        GGB_CUDA(cudaStreamSynchronize(g.stream));  // `s` is a stack variable
        return;
    }
    const NcclApi& api = nccl();
    IterCounters* ctr = static_cast<IterCounters*>(ctr_v);
    nccl_check(api.GroupStart(), "ncclGroupStart");
    nccl_check(api.AllReduce(&ctr->gathered, &ctr->gathered, 2, ncclUint64, ncclSum,
                             g.exchange->comm, g.stream), "allreduce(edges)");
    static_assert(offsetof(IterCounters, empty_active) == offsetof(IterCounters, changed) + 8 &&
                      offsetof(IterCounters, bad_min) == offsetof(IterCounters, changed) + 12,
                  "counter layout: [u64 x2][u32 sums x3][u32 min]");
    nccl_check(api.AllReduce(&ctr->changed, &ctr->changed, 3, ncclUint32, ncclSum,
                             g.exchange->comm, g.stream), "allreduce(changed)");
    nccl_check(api.AllReduce(&ctr->bad_min, &ctr->bad_min, 1, ncclUint32, ncclMin,
                             g.exchange->comm, g.stream), "allreduce(bad)");
    nccl_check(api.GroupEnd(), "ncclGroupEnd");
}

}  // namespace ggb

extern "C" {

gg_status gg_nccl_unique_id(uint8_t out[128]) {
    return ggb::guarded(nullptr, [&] {
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId id;
        ggb::nccl_check(ggb::nccl().GetUniqueId(&id), "ncclGetUniqueId");
        std::memcpy(out, &id, 128);
    });
}

gg_status gg_exchange_nccl_create(const uint8_t unique_id[128], int rank, int nranks,
                                  gg_exchange** out, gg_error* err) {
    return ggb::guarded(err, [&] {
        if (nranks < 1 || rank < 0 || rank >= nranks)
            throw ggb::Error(GG_INVALID_ARGUMENT, "rank/nranks out of range");
        ncclUniqueId id;
        std::memcpy(&id, unique_id, 128);
        auto* x = new gg_exchange;
        x->rank = rank;
        x->nranks = nranks;
        ncclResult_t r = ggb::nccl().CommInitRank(&x->comm, nranks, id, rank);
        if (r != ncclSuccess) {
            delete x;
            ggb::nccl_check(r, "ncclCommInitRank");
        }
        *out = x;
    });
}

gg_status gg_exchange_local_group(int nranks, gg_exchange** out) {
    return ggb::guarded(nullptr, [&] {
        if (nranks < 1) throw ggb::Error(GG_INVALID_ARGUMENT, "nranks must be >= 1");
        auto grp = std::make_shared<ggb::LocalGroup>(nranks);
        for (int r = 0; r < nranks; ++r) {
            auto* x = new gg_exchange;
            x->rank = r;
            x->nranks = nranks;
            x->local = grp;
            out[r] = x;
        }
    });
}

gg_status gg_exchange_set_fused(gg_exchange* x, int on) {
    return ggb::guarded(nullptr, [&] {
        if (!x) throw ggb::Error(GG_INVALID_ARGUMENT, "null exchange");
        x->fused = on != 0;
    });
}

// Transport health check. Every rank fills its own slice of a small buffer
// with a rank pattern, the slices are all-gathered with the grouped
// ncclBroadcast of exchange_slices (ragged slice lengths, rank r owns
// 1000 + 37 r words), a rank vector is sum-all-reduced and the one-word
// barrier all-reduce is issued, all on one private stream; the results are
// read back and compared with the closed forms.
gg_status gg_exchange_selftest(gg_exchange* x, gg_error* err) {
    return ggb::guarded(err, [&] {
        if (!x) throw ggb::Error(GG_INVALID_ARGUMENT, "null exchange");
        if (x->local) return;  // host barriers + device copies: covered by the engine runs
        if (!x->comm) throw ggb::Error(GG_NCCL, "exchange without communicator");
        const ggb::NcclApi& api = ggb::nccl();
        const int R = x->nranks, me = x->rank;
        std::vector<uint64_t> base(R + 1, 0);
        for (int r = 0; r < R; ++r) base[r + 1] = base[r] + 1000 + 37 * (uint64_t)r;
        const uint64_t total = base[R], nred = 4096;
        auto pat = [](int r, uint64_t i) { return (uint32_t)(0x9E3779B9u * (uint32_t)(r + 1) + (uint32_t)i); };
        std::vector<uint32_t> h(total + nred + 1, 0);
        for (uint64_t i = base[me]; i < base[me + 1]; ++i) h[i] = pat(me, i);
        for (uint64_t i = 0; i < nred; ++i) h[total + i] = (uint32_t)(me + 1) * (uint32_t)(i + 1);
        h[total + nred] = (uint32_t)me;
        cudaStream_t st = nullptr;
        uint32_t* d = nullptr;
        GGB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        GGB_CUDA(cudaMalloc(&d, h.size() * 4));
        try {
            GGB_CUDA(cudaMemcpyAsync(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
            ggb::nccl_check(api.GroupStart(), "ncclGroupStart");
            for (int r = 0; r < R; ++r)
                ggb::nccl_check(api.Broadcast(d + base[r], d + base[r], (base[r + 1] - base[r]) * 4,
                                              ncclChar, r, x->comm, st), "ncclBroadcast(selftest)");
            ggb::nccl_check(api.GroupEnd(), "ncclGroupEnd");
            ggb::nccl_check(api.AllReduce(d + total, d + total, nred, ncclUint32, ncclSum, x->comm, st),
                            "ncclAllReduce(selftest sum)");
            ggb::nccl_check(api.AllReduce(d + total + nred, d + total + nred, 1, ncclUint32, ncclMax,
                                          x->comm, st), "ncclAllReduce(selftest max)");
            GGB_CUDA(cudaMemcpyAsync(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost, st));
            GGB_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cudaFree(d);
            cudaStreamDestroy(st);
            throw;
        }
        cudaFree(d);
        cudaStreamDestroy(st);
        for (int r = 0; r < R; ++r)
            for (uint64_t i = base[r]; i < base[r + 1]; ++i)
                if (h[i] != pat(r, i))
                    throw ggb::Error(GG_NCCL, "exchange selftest: gathered slice of rank " +
                                                  std::to_string(r) + " differs");
        const uint32_t tri = (uint32_t)((uint64_t)R * (R + 1) / 2);
        for (uint64_t i = 0; i < nred; ++i)
            if (h[total + i] != tri * (uint32_t)(i + 1))
                throw ggb::Error(GG_NCCL, "exchange selftest: all-reduce sum differs");
        if (h[total + nred] != (uint32_t)(R - 1))
            throw ggb::Error(GG_NCCL, "exchange selftest: all-reduce max differs");
    });
}

gg_status gg_exchange_destroy(gg_exchange* x) {
    return ggb::guarded(nullptr, [&] {
        if (!x) return;
        if (x->comm) ggb::nccl().CommDestroy(x->comm);
        delete x;
    });
}

}  // extern "C"
