// graph_io.cu — binary CSC files straight to HBM.
//
// Reads the reference's cache format GGCSR1 (graph.cpp:259-300: "GGCSR1",
// little-endian u64 N, E, weighted, u64 offsets[N+1], u64 sources[E], f64
// weights[E]) and this engine's GGCSR2 (same header with the weight KIND in
// the third word, u64 offsets, u32 sources, weights of that kind, u32
// out-degrees[N]): half the source bytes of GGCSR1 and no out-degree pass.
//
// Loading streams each section through two pinned staging buffers: the file
// read of chunk i+1 overlaps the PCIe copy of chunk i; u64 sources are
// narrowed (and range-checked) on the device; out-degrees of a GGCSR1 file
// are counted on the device. Validation and messages follow read_binary /
// Graph::validate (graph.cpp:80-100, :272-296): bad magic, truncation,
// offsets not starting at 0 / decreasing / not ending at E, sources >= N,
// negative or non-finite weights.
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include <cmath>
#include <cstring>

#include "exchange.cuh"
#include "graph.cuh"

namespace ggb {
namespace {

constexpr char kMagic1[6] = {'G', 'G', 'C', 'S', 'R', '1'};
constexpr char kMagic2[6] = {'G', 'G', 'C', 'S', 'R', '2'};
constexpr size_t kStage = 64ull << 20;  // bytes per staging buffer
constexpr uint64_t kHeader = 6 + 3 * 8;

struct File {
    int fd = -1;
    std::string path;
    explicit File(const std::string& p, bool write = false) : path(p) {
        fd = write ? ::open(p.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644) : ::open(p.c_str(), O_RDONLY);
    }
    ~File() {
        if (fd >= 0) ::close(fd);
    }
    // exactly `bytes` at `off`, else false (truncated)
    bool read_at(void* dst, size_t bytes, uint64_t off) const {
        char* p = static_cast<char*>(dst);
        while (bytes) {
            const ssize_t r = ::pread(fd, p, bytes, (off_t)off);
            if (r <= 0) return false;
            p += r;
            off += (uint64_t)r;
            bytes -= (size_t)r;
        }
        return true;
    }
    bool write_all(const void* src, size_t bytes) const {
        const char* p = static_cast<const char*>(src);
        while (bytes) {
            const ssize_t r = ::write(fd, p, bytes);
            if (r <= 0) return false;
            p += r;
            bytes -= (size_t)r;
        }
        return true;
    }
};

// Pinned double buffer for host<->device streaming.
struct Stager {
    void* buf[2] = {nullptr, nullptr};
    cudaEvent_t ev[2] = {nullptr, nullptr};
    int next = 0;
    Stager() {
        for (int i = 0; i < 2; ++i) {
            GGB_CUDA(cudaHostAlloc(&buf[i], kStage, cudaHostAllocDefault));
            GGB_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
        }
    }
    ~Stager() {
        for (int i = 0; i < 2; ++i) {
            if (ev[i]) {
                cudaEventSynchronize(ev[i]);
                cudaEventDestroy(ev[i]);
            }
            if (buf[i]) cudaFreeHost(buf[i]);
        }
    }
    // a free buffer (its previous copy has completed)
    void* take(int& slot) {
        slot = next;
        next ^= 1;
        GGB_CUDA(cudaEventSynchronize(ev[slot]));
        return buf[slot];
    }
    void done(int slot, cudaStream_t st) { GGB_CUDA(cudaEventRecord(ev[slot], st)); }
};

__global__ void narrow_kernel(const uint64_t* __restrict__ in, uint64_t count, uint64_t n,
                              uint32_t* __restrict__ out, unsigned int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = (uint32_t)in[i];  // read_binary: static_cast<VertexId>
        if (s >= n) *bad = 1;
        out[i] = s;
    }
}

__global__ void count_kernel(const uint32_t* __restrict__ src, uint64_t count, uint64_t n,
                             uint32_t* __restrict__ deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = src[i];
        if (s < n) atomicAdd(deg + s, 1u);
    }
}

__global__ void range_kernel(const uint32_t* __restrict__ src, uint64_t count, uint64_t n,
                             unsigned int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (src[i] >= n) *bad = 1;
}

__global__ void deg_check_kernel(const uint32_t* __restrict__ counted,
                                 const uint32_t* __restrict__ stored, uint64_t n,
                                 unsigned int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        if (counted[i] != stored[i]) *bad = 1;
}

template <class T>
__global__ void weight_check_kernel(const T* __restrict__ w, uint64_t count,
                                    unsigned int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const double x = (double)w[i];
        if (!(x >= 0.0) || !isfinite(x)) *bad = 1;
    }
}

unsigned grid_n(uint64_t n) {
    uint64_t g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 148ull * 32 ? 148ull * 32 : g));
}

[[noreturn]] void fail(const std::string& m) { throw Error(GG_INVALID_ARGUMENT, m); }

}  // namespace
}  // namespace ggb

using namespace ggb;

extern "C" {

gg_status gg_dev_graph_load(const char* path, const gg_part_opts* opts, gg_dev_graph** out,
                            gg_error* err) {
    return guarded(err, [&] {
        if (!path || !out) throw Error(GG_INVALID_ARGUMENT, "null argument");
        const std::string p(path);
        File f(p);
        if (f.fd < 0) fail("cannot open binary graph: " + p);
        char magic[6];
        uint64_t hdr[3];
        if (!f.read_at(magic, 6, 0) ||
            (std::memcmp(magic, kMagic1, 6) != 0 && std::memcmp(magic, kMagic2, 6) != 0))
            fail(p + ": not a GGCSR1 file");
        const bool v2 = std::memcmp(magic, kMagic2, 6) == 0;
        const std::string fmt = v2 ? "GGCSR2" : "GGCSR1";
        if (!f.read_at(hdr, sizeof(hdr), 6)) fail(p + ": truncated " + fmt + " file");
        const uint64_t n = hdr[0], m = hdr[1];
        gg_weight_kind wk = v2 ? (gg_weight_kind)hdr[2] : (hdr[2] ? GG_W_F64 : GG_W_NONE);
        if (v2 && (hdr[2] > 3)) fail(p + ": corrupt GGCSR2 header");
        const size_t sb = v2 ? 4 : 8, wb = weight_size(wk);
        const uint64_t off_pos = kHeader, src_pos = off_pos + (n + 1) * 8,
                       w_pos = src_pos + m * sb, deg_pos = w_pos + m * wb;
        struct stat stt;  // size first: a short file never triggers a huge allocation
        const uint64_t want = (v2 ? deg_pos + n * 4 : w_pos + m * wb);
        if (n >= (1ull << 40) || m >= (1ull << 44) || ::fstat(f.fd, &stt) != 0 ||
            (uint64_t)stt.st_size < want)
            fail(p + ": truncated " + fmt + " file");
        // offsets: host copy (partition plan) + validation (graph.cpp:83-87)
        std::vector<uint64_t> off(n + 1);
        if (!f.read_at(off.data(), (n + 1) * 8, off_pos)) fail(p + ": truncated " + fmt + " file");
        if (off[0] != 0) fail("graph: first offset is not zero");
        for (uint64_t v = 0; v < n; ++v)
            if (off[v] > off[v + 1]) fail("graph: offsets decrease");
        if (off[n] != m) fail("graph: last offset != edge count");

        auto* h = new gg_dev_graph;
        try {
            DevGraph& g = h->g;
            setup_common(g, opts);
            g.n = n;
            g.e_global = m;
            g.wkind = wk;
            finish_graph(g, off.data());
            const uint64_t pad = g.e_base % kChunkEdges;
            g.off = static_cast<uint64_t*>(dev_alloc((g.nloc + 1) * 8, g.stream));
            g.src = static_cast<uint32_t*>(dev_alloc((pad + g.e_loc + kRun) * 4, g.stream));
            g.outdeg = static_cast<uint32_t*>(dev_alloc((n + 1) * 4, g.stream));
            if (wb) g.w = dev_alloc((pad + g.e_loc + kRun) * wb, g.stream);
            g.full.pad = pad;
            unsigned int* bad = static_cast<unsigned int*>(dev_alloc(16, g.stream));
            GGB_CUDA(cudaMemsetAsync(bad, 0, 16, g.stream));
            GGB_CUDA(cudaMemsetAsync(g.outdeg, 0, (n + 1) * 4, g.stream));
            std::vector<uint64_t> loc(off.begin() + g.v_begin, off.begin() + g.v_end + 1);
            for (uint64_t& x : loc) x -= g.e_base;
            GGB_CUDA(cudaMemcpyAsync(g.off, loc.data(), loc.size() * 8, cudaMemcpyHostToDevice, g.stream));
            GGB_CUDA(cudaStreamSynchronize(g.stream));
            {
                Stager sg;
                uint64_t* dtmp = v2 ? nullptr
                                    : static_cast<uint64_t*>(dev_alloc(2 * kStage, g.stream));
                uint32_t* dnar = v2 ? nullptr
                                    : static_cast<uint32_t*>(dev_alloc(kStage, g.stream));
                // sources: GGCSR1 all of them (out-degrees are global), GGCSR2 this rank's
                const uint64_t s_begin = v2 ? g.e_base : 0, s_end = v2 ? g.e_base + g.e_loc : m;
                const uint64_t per = kStage / sb;
                for (uint64_t b = s_begin; b < s_end; b += per) {
                    const uint64_t cnt = std::min(per, s_end - b);
                    int slot;
                    void* hb = sg.take(slot);
                    if (!f.read_at(hb, cnt * sb, src_pos + b * sb)) fail(p + ": truncated " + fmt + " file");
                    if (v2) {
                        GGB_CUDA(cudaMemcpyAsync(g.src + pad + (b - g.e_base), hb, cnt * 4,
                                                 cudaMemcpyHostToDevice, g.stream));
                    } else {
                        uint64_t* dt = dtmp + slot * (kStage / 8);
                        GGB_CUDA(cudaMemcpyAsync(dt, hb, cnt * 8, cudaMemcpyHostToDevice, g.stream));
                        // narrow into a scratch slice, count out-degrees, keep the owned part
                        uint32_t* narrow = dnar + slot * (kStage / 8);
                        narrow_kernel<<<grid_n(cnt), 256, 0, g.stream>>>(dt, cnt, n, narrow, bad);
                        count_kernel<<<grid_n(cnt), 256, 0, g.stream>>>(narrow, cnt, n, g.outdeg);
                        const uint64_t lo = std::max(b, g.e_base), hi = std::min(b + cnt, g.e_base + g.e_loc);
                        if (hi > lo)
                            GGB_CUDA(cudaMemcpyAsync(g.src + pad + (lo - g.e_base), narrow + (lo - b),
                                                     (hi - lo) * 4, cudaMemcpyDeviceToDevice, g.stream));
                        GGB_CUDA(cudaGetLastError());
                    }
                    sg.done(slot, g.stream);
                }
                if (v2) {  // out-degrees stored in the file
                    for (uint64_t b = 0; b < n; b += kStage / 4) {
                        const uint64_t cnt = std::min<uint64_t>(kStage / 4, n - b);
                        int slot;
                        void* hb = sg.take(slot);
                        if (!f.read_at(hb, cnt * 4, deg_pos + b * 4)) fail(p + ": truncated " + fmt + " file");
                        GGB_CUDA(cudaMemcpyAsync(g.outdeg + b, hb, cnt * 4, cudaMemcpyHostToDevice, g.stream));
                        sg.done(slot, g.stream);
                    }
                    range_kernel<<<grid_n(g.e_loc), 256, 0, g.stream>>>(g.src + pad, g.e_loc, n,
                                                                         bad);
                    // the stored out-degrees must be those of the sources
                    // (Graph::validate, graph.cpp:88-93): count this rank's
                    // sources, sum over ranks, compare
                    uint32_t* cnt = static_cast<uint32_t*>(dev_alloc((n + 1) * 4, g.stream));
                    GGB_CUDA(cudaMemsetAsync(cnt, 0, (n + 1) * 4, g.stream));
                    count_kernel<<<grid_n(g.e_loc), 256, 0, g.stream>>>(g.src + pad, g.e_loc, n, cnt);
                    GGB_CUDA(cudaGetLastError());
                    exchange_allreduce_u32(g, cnt, n);
                    deg_check_kernel<<<grid_n(n), 256, 0, g.stream>>>(cnt, g.outdeg, n, bad + 1);
                    GGB_CUDA(cudaGetLastError());
                    GGB_CUDA(cudaStreamSynchronize(g.stream));
                    dev_free(cnt, g.stream);
                }
                if (wb) {
                    const uint64_t per_w = kStage / wb;
                    for (uint64_t b = g.e_base; b < g.e_base + g.e_loc; b += per_w) {
                        const uint64_t cnt = std::min(per_w, g.e_base + g.e_loc - b);
                        int slot;
                        void* hb = sg.take(slot);
                        if (!f.read_at(hb, cnt * wb, w_pos + b * wb)) fail(p + ": truncated " + fmt + " file");
                        GGB_CUDA(cudaMemcpyAsync(static_cast<char*>(g.w) + (pad + b - g.e_base) * wb, hb,
                                                 cnt * wb, cudaMemcpyHostToDevice, g.stream));
                        sg.done(slot, g.stream);
                    }
                    const void* wl = static_cast<const char*>(g.w) + pad * wb;
                    if (wk == GG_W_F64)
                        weight_check_kernel<<<grid_n(g.e_loc), 256, 0, g.stream>>>(
                            static_cast<const double*>(wl), g.e_loc, bad + 3);
                    else if (wk == GG_W_F32)
                        weight_check_kernel<<<grid_n(g.e_loc), 256, 0, g.stream>>>(
                            static_cast<const float*>(wl), g.e_loc, bad + 3);
                    GGB_CUDA(cudaGetLastError());
                }
                GGB_CUDA(cudaStreamSynchronize(g.stream));
                if (dtmp) dev_free(dtmp, g.stream);
                if (dnar) dev_free(dnar, g.stream);
            }
            unsigned int hb[4] = {0, 0, 0, 0};
            GGB_CUDA(cudaMemcpy(hb, bad, 16, cudaMemcpyDeviceToHost));
            dev_free(bad, g.stream);
            if (hb[0]) fail(p + ": corrupt " + fmt + " source array");
            if (hb[1]) fail("graph: out_degree inconsistent with edges");
            if (hb[3]) fail("graph: negative or non-finite weight");
            assign_slots(g);
            build_full(g);
            GGB_CUDA(cudaStreamSynchronize(g.stream));
        } catch (...) {
            delete h;
            throw;
        }
        *out = h;
    });
}

int32_t gg_dev_graph_weight_kind(const gg_dev_graph* h) { return h ? (int32_t)h->g.wkind : -1; }

gg_status gg_dev_graph_save(const gg_dev_graph* h, const char* path, gg_error* err) {
    return guarded(err, [&] {
        if (!h || !path) throw Error(GG_INVALID_ARGUMENT, "null argument");
        const DevGraph& g = h->g;
        if (g.nranks != 1) throw Error(GG_INVALID_ARGUMENT, "save needs a single-rank graph");
        GGB_CUDA(cudaSetDevice(g.device));
        File f(path, true);
        if (f.fd < 0) fail(std::string("cannot open for writing: ") + path);
        const uint64_t hdr[3] = {g.n, g.e_loc, (uint64_t)g.wkind};
        std::vector<uint64_t> off(g.nloc + 1);
        GGB_CUDA(cudaMemcpy(off.data(), g.off, off.size() * 8, cudaMemcpyDeviceToHost));
        bool ok = f.write_all(kMagic2, 6) && f.write_all(hdr, sizeof(hdr)) &&
                  f.write_all(off.data(), off.size() * 8);
        std::vector<uint32_t> buf(g.e_loc);
        if (ok && g.e_loc) {
            export_sources(g, buf.data());
            ok = f.write_all(buf.data(), g.e_loc * 4);
        }
        const size_t wb = weight_size(g.wkind);
        if (ok && wb && g.e_loc) {
            std::vector<char> wbuf(g.e_loc * wb);
            GGB_CUDA(cudaMemcpy(wbuf.data(), static_cast<const char*>(g.w) + g.full.pad * wb,
                                wbuf.size(), cudaMemcpyDeviceToHost));
            ok = f.write_all(wbuf.data(), wbuf.size());
        }
        if (ok && g.n) {
            buf.resize(g.n);
            GGB_CUDA(cudaMemcpy(buf.data(), g.outdeg, g.n * 4, cudaMemcpyDeviceToHost));
            ok = f.write_all(buf.data(), g.n * 4);
        }
        if (!ok) fail(std::string("I/O error while writing ") + path);
    });
}

}  // extern "C"
