// capi.cu — the extern "C" boundary (include/ggb.h) and the program
// dispatch. Each gg_run_* is the device counterpart of
// gg::run<Program>(graph, program, config) (engine.hpp:141-143).
#include <algorithm>
#include <cmath>
#include <numeric>
#include <vector>

#include "engine.cuh"
#include "exchange.cuh"
#include "programs.cuh"

namespace ggb {

// 32-aligned, edge-balanced destination ranges.
constexpr uint64_t kPartAlign = 32;  // rank ranges start at multiples of 32 vertices

static std::vector<uint64_t> plan_partition(uint64_t n, const uint64_t* off, int nranks) {
    std::vector<uint64_t> b(nranks + 1, 0);
    b[nranks] = n;
    const uint64_t e = off[n];
    for (int r = 1; r < nranks; ++r) {
        const uint64_t target = (uint64_t)((long double)e * r / nranks);
        uint64_t v = (uint64_t)(std::lower_bound(off, off + n + 1, target) - off);
        v = (v / kPartAlign) * kPartAlign;
        if (v < b[r - 1]) v = b[r - 1];
        if (v > n) v = n;
        b[r] = v;
    }
    return b;
}

__global__ void rebase_kernel(const uint64_t* __restrict__ in, uint64_t count, uint64_t base,
                              uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i] - base;
}

void setup_common(DevGraph& g, const gg_part_opts* opts) {
    int dev = 0;
    if (opts && opts->device >= 0) dev = opts->device;
    else GGB_CUDA(cudaGetDevice(&dev));
    int count = 0;
    GGB_CUDA(cudaGetDeviceCount(&count));
    if (count < 1) throw Error(GG_CUDA, "no CUDA device");
    g.device = dev;
    GGB_CUDA(cudaSetDevice(dev));
    int major = 0, sms = 0;  // attribute queries: cheap on the e2e path
    GGB_CUDA(cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev));
    GGB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    if (major < 10) {
        cudaDeviceProp prop;
        GGB_CUDA(cudaGetDeviceProperties(&prop, dev));
        throw Error(GG_CUDA, std::string("libggb.so needs an sm_100 device, found ") + prop.name);
    }
    g.num_sms = sms;
    GGB_CUDA(cudaStreamCreateWithFlags(&g.stream, cudaStreamNonBlocking));
    g.ws.stream = g.stream;
    // keep freed device memory cached in the stream-ordered pool (graphs are
    // re-created on the end-to-end path; see graph.cuh dev_alloc)
    cudaMemPool_t pool;
    GGB_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
    uint64_t threshold = UINT64_MAX;
    GGB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    g.rank = opts ? opts->rank : 0;
    g.nranks = opts ? std::max(1, opts->nranks) : 1;
    g.exchange = opts ? static_cast<gg_exchange*>(opts->exchange) : nullptr;
    if (g.nranks > 1 && !g.exchange)
        throw Error(GG_INVALID_ARGUMENT, "nranks > 1 needs an exchange (gg_exchange_nccl_create)");
    if (g.rank < 0 || g.rank >= g.nranks) throw Error(GG_INVALID_ARGUMENT, "rank out of range");
}

void finish_graph(DevGraph& g, const uint64_t* host_off_full) {
    g.bounds = plan_partition(g.n, host_off_full, g.nranks);
    g.ebounds.resize(g.nranks + 1);
    for (int r = 0; r <= g.nranks; ++r) g.ebounds[r] = host_off_full[g.bounds[r]];
    g.v_begin = g.bounds[g.rank];
    g.v_end = g.bounds[g.rank + 1];
    g.nloc = g.v_end - g.v_begin;
    g.e_base = g.ebounds[g.rank];
    g.e_loc = g.ebounds[g.rank + 1] - g.e_base;
    if (g.n > 0xffffffffull) throw Error(GG_INVALID_ARGUMENT, "more than 2^32-1 vertices");
}

}  // namespace ggb

using namespace ggb;

extern "C" {

const char* gg_status_string(gg_status s) {
    switch (s) {
        case GG_OK: return "ok";
        case GG_INVALID_ARGUMENT: return "invalid argument";
        case GG_INVALID_PROPERTY: return "invalid property";
        case GG_CUDA: return "CUDA error";
        case GG_NCCL: return "NCCL error";
        case GG_OOM: return "out of memory";
        case GG_INTERNAL: return "internal error";
    }
    return "unknown status";
}

int gg_abi_version(void) { return GGB_ABI_VERSION; }

gg_status gg_partition_plan(uint64_t n, const uint64_t* offsets, int nranks, uint64_t* bounds) {
    return guarded(nullptr, [&] {
        if (nranks < 1) throw Error(GG_INVALID_ARGUMENT, "nranks must be >= 1");
        auto b = plan_partition(n, offsets, nranks);
        std::copy(b.begin(), b.end(), bounds);
    });
}

// Copy stream + events of one pipelined upload (released on every exit path).
constexpr size_t kUploadChunks = 16;
struct Upload {
    cudaStream_t cs = nullptr;
    cudaEvent_t ready = nullptr, deg = nullptr, off = nullptr, done = nullptr;
    std::vector<cudaEvent_t> chunk;
    Upload(cudaStream_t, size_t nchunks) : chunk(nchunks, nullptr) {
        GGB_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
        for (cudaEvent_t* e : {&ready, &deg, &off, &done})
            GGB_CUDA(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
        for (cudaEvent_t& e : chunk) GGB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    ~Upload() {
        if (cs) cudaStreamSynchronize(cs);
        for (cudaEvent_t e : {ready, deg, off, done})
            if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : chunk)
            if (e) cudaEventDestroy(e);
        if (cs) cudaStreamDestroy(cs);
    }
};

static gg_status create_impl(const gg_csc_view* csc, const gg_part_opts* opts,
                             const SparsifySpec* pre, double pre_sigma, uint64_t pre_seed,
                             gg_dev_graph** out, gg_error* err) {
    return guarded(err, [&] {
        if (!csc || !out) throw Error(GG_INVALID_ARGUMENT, "null argument");
        if (csc->n && !csc->offsets) throw Error(GG_INVALID_ARGUMENT, "offsets is null");
        if (csc->offsets && csc->offsets[csc->n] != csc->e)
            throw Error(GG_INVALID_ARGUMENT, "offsets[n] != e");
        if (csc->e && !csc->sources) throw Error(GG_INVALID_ARGUMENT, "sources is null");
        if (csc->weight_kind != GG_W_NONE && csc->e && !csc->weights)
            throw Error(GG_INVALID_ARGUMENT, "weights is null");
        auto* h = new gg_dev_graph;
        try {
            DevGraph& g = h->g;
            setup_common(g, opts);
            g.n = csc->n;
            g.e_global = csc->e;
            g.wkind = csc->weight_kind;
            const uint64_t zero = 0;
            finish_graph(g, csc->offsets ? csc->offsets : &zero);
            const uint64_t pad = g.e_base % kChunkEdges;  // padded = global position mod 512
            g.off = static_cast<decltype(g.off)>(dev_alloc((g.nloc + 1) * 8, g.stream));
            g.src = static_cast<decltype(g.src)>(dev_alloc((pad + g.e_loc + kRun) * 4, g.stream));
            g.outdeg = static_cast<decltype(g.outdeg)>(dev_alloc((g.n + 1) * 4, g.stream));
            const size_t wb = weight_size(g.wkind);
            if (wb) g.w = static_cast<decltype(g.w)>(dev_alloc((pad + g.e_loc + kRun) * wb, g.stream));
            g.full.pad = pad;
            std::vector<uint32_t> host_deg;
            if (!csc->out_degree) {  // reference graphs carry it; computed here for bare CSC views
                host_deg.assign(g.n, 0);
                for (uint64_t i = 0; i < csc->e; ++i) {
                    if (csc->sources[i] >= g.n)
                        throw Error(GG_INVALID_ARGUMENT, "edge source out of range");
                    ++host_deg[csc->sources[i]];
                }
            }
            // device-side validation flags: [0] source >= n, [1] offsets decrease
            unsigned int* bad = g.ws.get<unsigned int>("create.bad", 4);
            GGB_CUDA(cudaMemsetAsync(bad, 0, 16, g.stream));
            const uint32_t* deg = csc->out_degree ? csc->out_degree : host_deg.data();
            // Pipelined upload: the copy stream carries out-degrees, offsets,
            // then the sources in chunks and the weights over PCIe while the
            // graph stream computes the slot order, the run map and relabels
            // each source chunk as it lands.
            Upload up(g.stream, g.e_loc ? kUploadChunks : 0);
            GGB_CUDA(cudaEventRecord(up.ready, g.stream));  // allocations above
            GGB_CUDA(cudaStreamWaitEvent(up.cs, up.ready, 0));
            if (g.n) GGB_CUDA(cudaMemcpyAsync(g.outdeg, deg, g.n * 4, cudaMemcpyHostToDevice, up.cs));
            GGB_CUDA(cudaEventRecord(up.deg, up.cs));
            GGB_CUDA(cudaMemcpyAsync(g.off, csc->offsets ? csc->offsets + g.v_begin : &zero,
                                     (g.nloc + 1) * 8, cudaMemcpyHostToDevice, up.cs));
            GGB_CUDA(cudaEventRecord(up.off, up.cs));
            // the initial sparsification of the coming run rides along with the
            // upload (one rank; graphs of >= 2^24 edges -- below that the extra
            // launches cost more than the overlap saves): chunks are whole scan
            // tiles, and a chunk's weights travel right after its sources
            // (GGB_PRESPARSE_MIN_EDGES overrides the 2^24 cut, for tests)
            const char* cut_env = std::getenv("GGB_PRESPARSE_MIN_EDGES");
            const uint64_t cut = cut_env ? std::strtoull(cut_env, nullptr, 10) : (1ull << 24);
            const bool presp = pre && g.nranks == 1 && g.e_loc >= cut;
            uint64_t step = (g.e_loc + up.chunk.size() - 1) / std::max<size_t>(up.chunk.size(), 1);
            if (presp) {
                const uint64_t te = presparse_tile_edges();
                step = (step + te - 1) / te * te;
            }
            for (size_t k = 0; k < up.chunk.size(); ++k) {
                const uint64_t b = std::min(g.e_loc, k * step), e = std::min(g.e_loc, b + step);
                if (e > b) {
                    GGB_CUDA(cudaMemcpyAsync(g.src + pad + b, csc->sources + g.e_base + b, (e - b) * 4,
                                             cudaMemcpyHostToDevice, up.cs));
                    if (presp && wb)
                        GGB_CUDA(cudaMemcpyAsync(static_cast<char*>(g.w) + (pad + b) * wb,
                                                 static_cast<const char*>(csc->weights) +
                                                     (g.e_base + b) * wb,
                                                 (e - b) * wb, cudaMemcpyHostToDevice, up.cs));
                }
                GGB_CUDA(cudaEventRecord(up.chunk[k], up.cs));
            }
            if (wb && g.e_loc && !presp)
                GGB_CUDA(cudaMemcpyAsync(static_cast<char*>(g.w) + pad * wb,
                                         static_cast<const char*>(csc->weights) + g.e_base * wb,
                                         g.e_loc * wb, cudaMemcpyHostToDevice, up.cs));
            GGB_CUDA(cudaEventRecord(up.done, up.cs));
            // graph stream
            GGB_CUDA(cudaStreamWaitEvent(g.stream, up.deg, 0));
            compute_slots(g);
            GGB_CUDA(cudaStreamWaitEvent(g.stream, up.off, 0));
            if (g.e_base) {
                rebase_kernel<<<256, 256, 0, g.stream>>>(g.off, g.nloc + 1, g.e_base, g.off);
                GGB_CUDA(cudaGetLastError());
            }
            check_offsets(g, bad + 1);
            build_full(g);
            for (size_t k = 0; k < up.chunk.size(); ++k) {
                const uint64_t b = std::min(g.e_loc, k * step), e = std::min(g.e_loc, b + step);
                GGB_CUDA(cudaStreamWaitEvent(g.stream, up.chunk[k], 0));
                relabel_sources(g, g.src + pad + b, e - b, csc->out_degree ? bad : nullptr);
                if (presp && e > b) presparse_chunk(g, *pre, b, e);
            }
            if (presp) {
                g.pre_sparse = true;
                g.pre_sigma = pre_sigma;
                g.pre_seed = pre_seed;
            }
            GGB_CUDA(cudaStreamWaitEvent(g.stream, up.done, 0));
            unsigned int hbad[4];
            GGB_CUDA(cudaMemcpyAsync(hbad, bad, 16, cudaMemcpyDeviceToHost, g.stream));
            GGB_CUDA(cudaStreamSynchronize(g.stream));
            // every rank fails together (a rank that failed alone would leave
            // the others waiting in the first exchange)
            const uint64_t code = exchange_sum(g, (hbad[1] ? 1ull << 32 : 0ull) | (hbad[0] ? 1ull : 0ull));
            if (code >> 32) throw Error(GG_INVALID_ARGUMENT, "graph: offsets decrease");
            if (code & 0xffffffffull) throw Error(GG_INVALID_ARGUMENT, "edge source out of range");
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

gg_status gg_dev_graph_create(const gg_csc_view* csc, const gg_part_opts* opts,
                              gg_dev_graph** out, gg_error* err) {
    return create_impl(csc, opts, nullptr, 0.0, 0, out, err);
}

gg_status gg_dev_graph_create_for_run(const gg_csc_view* csc, const gg_part_opts* opts,
                                      double sigma, uint64_t seed, gg_dev_graph** out,
                                      gg_error* err) {
    if (!(sigma >= 0.0 && sigma <= 1.0))  // the run reports the field (engine.cpp:45-61)
        return create_impl(csc, opts, nullptr, 0.0, 0, out, err);
    const SparsifySpec h = sparsify_spec(sigma, seed, false);
    return create_impl(csc, opts, &h, sigma, seed, out, err);
}

}  // extern "C"

namespace ggb {
// A graph from a full CSC already in HBM (device R-MAT, device
// symmetrization): one rank adopts the arrays, several ranks copy their
// slice; then slots, relabel, the full list's layout.
void adopt_csc(DevGraph& g, RmatCsc r, gg_weight_kind wk) {
    g.n = r.n;
    g.e_global = r.e;
    g.wkind = wk;
    std::vector<uint64_t> off(r.n + 1);
    GGB_CUDA(cudaMemcpyAsync(off.data(), r.off, (r.n + 1) * 8, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    finish_graph(g, off.data());
    g.outdeg = r.outdeg;
    if (g.nranks == 1) {
        g.off = r.off;
        g.src = r.src;
        g.w = r.w;
    } else {
        g.off = static_cast<decltype(g.off)>(dev_alloc((g.nloc + 1) * 8, g.stream));
        rebase_kernel<<<256, 256, 0, g.stream>>>(r.off + g.v_begin, g.nloc + 1, g.e_base, g.off);
        GGB_CUDA(cudaGetLastError());
        const uint64_t pad = g.e_base % kChunkEdges;
        g.src = static_cast<decltype(g.src)>(dev_alloc((pad + g.e_loc + kRun) * 4, g.stream));
        GGB_CUDA(cudaMemcpyAsync(g.src + pad, r.src + g.e_base, g.e_loc * 4, cudaMemcpyDeviceToDevice,
                                 g.stream));
        const size_t wb = weight_size(g.wkind);
        if (wb) {
            g.w = static_cast<decltype(g.w)>(dev_alloc((pad + g.e_loc + kRun) * wb, g.stream));
            GGB_CUDA(cudaMemcpyAsync(static_cast<char*>(g.w) + pad * wb,
                                     static_cast<char*>(r.w) + g.e_base * wb, g.e_loc * wb,
                                     cudaMemcpyDeviceToDevice, g.stream));
        }
        g.full.pad = pad;
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        dev_free(r.off, g.stream);
        dev_free(r.src, g.stream);
        if (r.w) dev_free(r.w, g.stream);
    }
    assign_slots(g);
    build_full(g);
    GGB_CUDA(cudaStreamSynchronize(g.stream));
}
}  // namespace ggb

extern "C" {

gg_status gg_dev_graph_create_rmat(const gg_rmat_params* p, const gg_part_opts* opts,
                                   gg_dev_graph** out, gg_error* err) {
    return guarded(err, [&] {
        if (!p || !out) throw Error(GG_INVALID_ARGUMENT, "null argument");
        auto* h = new gg_dev_graph;
        try {
            DevGraph& g = h->g;
            setup_common(g, opts);
            adopt_csc(g, rmat_generate(*p, g.stream), p->weight_kind);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

gg_status gg_dev_graph_symmetrized(const gg_dev_graph* in, const gg_part_opts* opts,
                                   gg_dev_graph** out, gg_error* err) {
    return guarded(err, [&] {
        if (!in || !out) throw Error(GG_INVALID_ARGUMENT, "null argument");
        if (in->g.nranks != 1) throw Error(GG_INVALID_ARGUMENT, "symmetrized needs a single-rank graph");
        auto* h = new gg_dev_graph;
        try {
            DevGraph& g = h->g;
            gg_part_opts o{};
            if (opts) o = *opts;
            else o.device = in->g.device;
            if (o.device < 0) o.device = in->g.device;
            setup_common(g, &o);
            adopt_csc(g, symmetrize_device(in->g, g.stream), in->g.wkind);
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

gg_status gg_dev_graph_destroy(gg_dev_graph* g) {
    return guarded(nullptr, [&] {
        if (g) {
            cudaSetDevice(g->g.device);
            delete g;
        }
    });
}

gg_status gg_dev_graph_info(const gg_dev_graph* h, uint64_t* n, uint64_t* e, uint64_t* vb,
                            uint64_t* ve, uint64_t* el) {
    return guarded(nullptr, [&] {
        if (!h) throw Error(GG_INVALID_ARGUMENT, "null graph");
        const DevGraph& g = h->g;
        if (n) *n = g.n;
        if (e) *e = g.e_global;
        if (vb) *vb = g.v_begin;
        if (ve) *ve = g.v_end;
        if (el) *el = g.e_loc;
    });
}

gg_status gg_dev_graph_export(const gg_dev_graph* h, uint64_t* offsets, uint32_t* sources,
                              void* weights, uint32_t* out_degree) {
    return guarded(nullptr, [&] {
        if (!h) throw Error(GG_INVALID_ARGUMENT, "null graph");
        const DevGraph& g = h->g;
        if (g.nranks != 1 && (offsets || sources || weights))  // out_degree is replicated
            throw Error(GG_INVALID_ARGUMENT, "CSC export needs a single-rank graph");
        GGB_CUDA(cudaSetDevice(g.device));
        if (offsets) GGB_CUDA(cudaMemcpy(offsets, g.off, (g.nloc + 1) * 8, cudaMemcpyDeviceToHost));
        if (sources && g.e_loc)
            export_sources(g, sources);  // slot ids back to vertex ids
        const size_t wb = weight_size(g.wkind);
        if (weights && wb && g.e_loc)
            GGB_CUDA(cudaMemcpy(weights, static_cast<const char*>(g.w) + g.full.pad * wb,
                                g.e_loc * wb, cudaMemcpyDeviceToHost));
        if (out_degree && g.n)
            GGB_CUDA(cudaMemcpy(out_degree, g.outdeg, g.n * 4, cudaMemcpyDeviceToHost));
    });
}

gg_status gg_bp_priors(uint64_t n, uint64_t seed, float* out) {
    return guarded(nullptr, [&] {
        float* d = nullptr;
        d = static_cast<decltype(d)>(dev_alloc((2 * n + 2) * 4, 0));
        bp_priors_device(n, seed, d, 0);
        GGB_CUDA(cudaMemcpy(out, d, 2 * n * 4, cudaMemcpyDeviceToHost));
        dev_free(d, 0);
    });
}

gg_status gg_bp_priors_device(uint64_t n, uint64_t seed, float** dev_out) {
    return guarded(nullptr, [&] {
        if (!dev_out) throw Error(GG_INVALID_ARGUMENT, "null argument");
        float* d = nullptr;
        GGB_CUDA(cudaMalloc(&d, (2 * n + 2) * 4));
        bp_priors_device(n, seed, d, 0);
        GGB_CUDA(cudaStreamSynchronize(0));
        *dev_out = d;
    });
}

gg_status gg_device_upload(const void* host, uint64_t bytes, void** dev_out) {
    return guarded(nullptr, [&] {
        if (!dev_out || (bytes && !host)) throw Error(GG_INVALID_ARGUMENT, "null argument");
        void* d = nullptr;
        GGB_CUDA(cudaMalloc(&d, bytes ? bytes : 16));
        if (bytes) GGB_CUDA(cudaMemcpy(d, host, bytes, cudaMemcpyHostToDevice));
        *dev_out = d;
    });
}

gg_status gg_device_free(void* dev) {
    return guarded(nullptr, [&] {
        if (dev) GGB_CUDA(cudaFree(dev));
    });
}

gg_status gg_validate(const gg_engine_config* cfg, gg_error* err) {
    return guarded(err, [&] { validate(*cfg); });
}

int32_t gg_mode_for(int32_t scheme, uint64_t t, uint64_t alpha) { return mode_for(scheme, t, alpha); }

uint64_t gg_select_superstep_iterations(uint64_t alpha, uint64_t max_it, int32_t scheme,
                                        uint64_t* out, uint64_t cap) {
    uint64_t k = 0;  // engine.cpp:77-90
    if (alpha < 1) return 0;
    if (scheme == GG_SCHEME_GG) {
        for (uint64_t t = alpha + 1; t <= max_it; t += alpha + 1) {
            if (k < cap && out) out[k] = t;
            ++k;
        }
    } else if (scheme == GG_SCHEME_SMS && alpha + 1 <= max_it) {
        if (k < cap && out) out[k] = alpha + 1;
        ++k;
    }
    return k;
}

gg_status gg_sparsify(uint64_t e, double sigma, uint64_t seed, uint32_t* out_bitmap, gg_error* err) {
    return guarded(err, [&] {
        if (!(sigma >= 0.0 && sigma <= 1.0)) throw Error(GG_INVALID_ARGUMENT, "sigma must be in [0,1]");
        DevGraph g;
        setup_common(g, nullptr);
        g.e_loc = e;
        const uint64_t nwords = (e + 31) / 32;
        uint32_t* bm = g.ws.get<uint32_t>("bm", nwords + 1);
        sparsify_bitmap(g, bm, sigma, seed, false);
        GGB_CUDA(cudaMemcpyAsync(out_bitmap, bm, nwords * 4, cudaMemcpyDeviceToHost, g.stream));
        GGB_CUDA(cudaStreamSynchronize(g.stream));
    });
}

// ---- runs -----------------------------------------------------------------
static RunIO make_io(const gg_engine_config* cfg, gg_iter_record* recs, uint64_t cap,
                     gg_run_summary* sum, const gg_run_opts* opts, void* props, int S) {
    RunIO io;
    io.cfg = cfg; io.recs = recs; io.rec_cap = cap; io.sum = sum; io.opts = opts;
    io.out_props = props; io.out_states = S;
    if (sum) std::memset(sum, 0, sizeof(*sum));
    return io;
}

static void check_run(gg_dev_graph* h, const gg_engine_config* cfg) {
    if (!h || !cfg) throw Error(GG_INVALID_ARGUMENT, "null argument");
    validate(*cfg);  // engine.hpp:145
}

gg_status gg_run_pr(gg_dev_graph* h, const gg_engine_config* cfg, const gg_pr_params* p,
                    double* out_props, gg_iter_record* recs, uint64_t cap, gg_run_summary* sum,
                    const gg_run_opts* opts, gg_error* err) {
    return guarded(err, [&] {
        check_run(h, cfg);
        RunIO io = make_io(cfg, recs, cap, sum, opts, out_props, 1);
        if (h->g.n == 0) return;  // engine.hpp:149
        PageRank prog;
        prog.damping = p ? p->damping : 0.85;
        prog.epsilon = p ? p->epsilon : 1e-7;
        Engine<PageRank, void>::run(h->g, prog, io);  // PR ignores edge weights
    });
}

gg_status gg_run_sssp(gg_dev_graph* h, const gg_engine_config* cfg, const gg_sssp_params* p,
                      double* out_props, gg_iter_record* recs, uint64_t cap, gg_run_summary* sum,
                      const gg_run_opts* opts, gg_error* err) {
    return guarded(err, [&] {
        check_run(h, cfg);
        RunIO io = make_io(cfg, recs, cap, sum, opts, out_props, 1);
        if (h->g.n == 0) return;
        const uint32_t source = p ? p->source : 0;
        const bool graded = p ? p->graded != 0 : false;
        if (source >= h->g.n)  // algorithms.hpp:55-57
            throw Error(GG_INVALID_ARGUMENT, "sssp source vertex out of range");
        DevGraph& g = h->g;
        if (g.wkind == GG_W_NONE || g.wkind == GG_W_U32) {
            SsspU32 prog;
            prog.source = source;
            prog.graded = graded;
            prog.overflow = g.ws.get<unsigned int>("sssp.overflow", 1);
            GGB_CUDA(cudaMemsetAsync(prog.overflow, 0, 4, g.stream));
            if (g.wkind == GG_W_NONE) Engine<SsspU32, void>::run(g, prog, io);
            else Engine<SsspU32, uint32_t>::run(g, prog, io);
            unsigned int ovf = 0;
            GGB_CUDA(cudaMemcpyAsync(&ovf, prog.overflow, 4, cudaMemcpyDeviceToHost, g.stream));
            GGB_CUDA(cudaStreamSynchronize(g.stream));
            if (exchange_sum(g, ovf)) {  // a distance beyond u32: redo with f64 distances
                SsspF64 p64;
                p64.source = source;
                p64.graded = graded;
                io = make_io(cfg, recs, cap, sum, opts, out_props, 1);
                if (g.wkind == GG_W_NONE) Engine<SsspF64, void>::run(g, p64, io);
                else Engine<SsspF64, uint32_t>::run(g, p64, io);
            }
        } else {
            SsspF64 prog;
            prog.source = source;
            prog.graded = graded;
            if (g.wkind == GG_W_F32) Engine<SsspF64, float>::run(g, prog, io);
            else Engine<SsspF64, double>::run(g, prog, io);
        }
    });
}

gg_status gg_run_wcc(gg_dev_graph* h, const gg_engine_config* cfg, uint32_t* out_props,
                     gg_iter_record* recs, uint64_t cap, gg_run_summary* sum,
                     const gg_run_opts* opts, gg_error* err) {
    return guarded(err, [&] {
        check_run(h, cfg);
        RunIO io = make_io(cfg, recs, cap, sum, opts, out_props, 1);
        if (h->g.n == 0) return;
        Engine<Wcc, void>::run(h->g, Wcc{}, io);
    });
}

gg_status gg_run_bp(gg_dev_graph* h, const gg_engine_config* cfg, const gg_bp_params* p,
                    double* out_props, gg_iter_record* recs, uint64_t cap, gg_run_summary* sum,
                    const gg_run_opts* opts, gg_error* err) {
    return guarded(err, [&] {
        check_run(h, cfg);
        if (!p) throw Error(GG_INVALID_ARGUMENT, "bp params are required");
        DevGraph& g = h->g;
        if (p->prior_table) {
            if (p->states != 2) throw Error(GG_INVALID_ARGUMENT, "bp with a prior table needs states == 2");
            if (g.wkind != GG_W_F32 && g.wkind != GG_W_F64)
                throw Error(GG_INVALID_ARGUMENT, "bp with a prior table needs per-edge couplings (f32/f64 weights)");
            RunIO io = make_io(cfg, recs, cap, sum, opts, out_props, 2);
            if (g.n == 0) return;
            const float2* table = reinterpret_cast<const float2*>(p->prior_table);
            if (!p->prior_on_device) {  // host table: one copy per run
                float2* d = g.ws.get<float2>("bp.prior", g.n);
                GGB_CUDA(cudaMemcpyAsync(d, p->prior_table, g.n * 8, cudaMemcpyHostToDevice, g.stream));
                table = d;
            }
            BeliefPropEdge prog;
            prog.prior_table = table;
            prog.epsilon = p->epsilon;
            if (g.wkind == GG_W_F32) Engine<BeliefPropEdge, float>::run(g, prog, io);
            else Engine<BeliefPropEdge, double>::run(g, prog, io);
            return;
        }
        RunIO io = make_io(cfg, recs, cap, sum, opts, out_props, p->states);
        if (g.n == 0) return;
        switch (p->states) {
            case 2: { BeliefProp<2> b; b.coupling = p->coupling; b.epsilon = p->epsilon;
                      Engine<BeliefProp<2>, void>::run(g, b, io); break; }
            case 3: { BeliefProp<3> b; b.coupling = p->coupling; b.epsilon = p->epsilon;
                      Engine<BeliefProp<3>, void>::run(g, b, io); break; }
            case 4: { BeliefProp<4> b; b.coupling = p->coupling; b.epsilon = p->epsilon;
                      Engine<BeliefProp<4>, void>::run(g, b, io); break; }
            default: {
                if (p->states < 2) throw Error(GG_INVALID_ARGUMENT, "bp states must be >= 2");
                if (p->states > kBpMaxStates)
                    throw Error(GG_INVALID_ARGUMENT, "bp states must be <= 64 on device");
                auto dyn = [&](auto b) {
                    b.states = p->states;
                    b.coupling = p->coupling;
                    b.epsilon = p->epsilon;
                    Engine<decltype(b), void>::run(g, b, io);
                };
                if (p->states <= 16) dyn(BeliefPropDyn<16>{});
                else if (p->states <= 32) dyn(BeliefPropDyn<32>{});
                else dyn(BeliefPropDyn<64>{});
                break;
            }
        }
    });
}

// ---- host metrics (metrics.cpp) ------------------------------------------
gg_status gg_topk_error(const double* approx, const double* exact, uint64_t n, uint64_t k,
                        double* err_out) {
    return guarded(nullptr, [&] {
        if (k < 1 || k > n) throw Error(GG_INVALID_ARGUMENT, "topk k must be in [1, N]");
        auto topk = [&](const double* vals) {
            std::vector<uint32_t> idx(n);
            std::iota(idx.begin(), idx.end(), 0u);
            std::partial_sort(idx.begin(), idx.begin() + (long)k, idx.end(),
                              [&](uint32_t a, uint32_t b) {
                                  if (vals[a] != vals[b]) return vals[a] > vals[b];
                                  return a < b;
                              });
            idx.resize(k);
            return idx;
        };
        const auto ta = topk(approx), te = topk(exact);
        std::vector<uint8_t> in_exact(n, 0);
        for (uint32_t v : te) in_exact[v] = 1;
        uint64_t missing = 0;
        for (uint32_t v : ta) missing += in_exact[v] ? 0 : 1;
        *err_out = (double)missing / (double)k;
    });
}

gg_status gg_relative_error(const double* approx, const double* exact, uint64_t n, double* err_out) {
    return guarded(nullptr, [&] {
        if (n == 0) { *err_out = 0.0; return; }
        double s = 0.0;
        for (uint64_t v = 0; v < n; ++v) {
            const double a = approx[v] + 1.0, e = exact[v] + 1.0;
            s += std::min(1.0, std::fabs(e - a) / e);
        }
        *err_out = s / (double)n;
    });
}

gg_status gg_stretch_error(const double* approx, const double* exact, uint64_t n, double* err_out) {
    return guarded(nullptr, [&] {
        double s = 0.0;
        uint64_t counted = 0;
        for (uint64_t v = 0; v < n; ++v) {
            const double e = exact[v], a = approx[v];
            if (a < e)
                throw Error(GG_INVALID_ARGUMENT, "stretch_error: approximate distance below exact at vertex " +
                                                     std::to_string(v) + " (engine bug)");
            if (std::isinf(e)) continue;
            if (e == 0.0 && a == 0.0) continue;
            ++counted;
            if (std::isinf(a) || e == 0.0) { s += 1.0; continue; }
            s += 1.0 - e / a;
        }
        *err_out = counted == 0 ? 0.0 : s / (double)counted;
    });
}

#ifdef GGB_CHAIN_STATS
// diagnostic build only: look-back statistics of the chain kernels since the last call
void ggb_debug_chain_stats(unsigned long long* out) {
    unsigned long long z[8] = {};
    cudaMemcpyFromSymbol(out, ggb::g_chain_stats, sizeof(z));
    cudaMemcpyToSymbol(ggb::g_chain_stats, z, sizeof(z));
}
#endif
}  // extern "C"
