// build.cu — flag set maintenance: sparsify, bitmap -> sparsified CSC
// compaction, work-list construction, deferred superstep validity scan.
//
// The reference keeps one flag BYTE per edge and re-tests it inside every
// approximate iteration (engine.hpp:203). Here the flags are a bitmap that
// is touched only when it changes (initial sparsify, each superstep); the
// approximate iterations then stream a compacted CSC holding exactly the
// flagged edges in their original order, so the fold order per vertex is
// unchanged and no flag is read on the hot path.
#include <cub/cub.cuh>

#include "graph.cuh"
#include "kernels.cuh"

namespace ggb {

size_t weight_size(gg_weight_kind k) {
    switch (k) {
        case GG_W_U32: return 4;
        case GG_W_F32: return 4;
        case GG_W_F64: return 8;
        default: return 0;
    }
}

int occupancy_grid(const void* kernel, int block, size_t smem, int num_sms) {
    int per_sm = 0;
    GGB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, smem));
    if (per_sm < 1) per_sm = 1;
    return per_sm * num_sms;
}

static inline unsigned grid_for(uint64_t n, int block, uint64_t cap = 148ull * 64) {
    uint64_t g = (n + block - 1) / block;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (unsigned)g;
}

// --------------------------------------------------------------------------
// sparsify (engine.cpp:63-75): u = (mix64(mix64(seed) ^ e) >> 11) * 2^-53,
// flag = u < sigma, hashed on the GLOBAL edge id so every partition agrees.
// --------------------------------------------------------------------------
__global__ void sparsify_kernel(uint32_t* __restrict__ bitmap, uint64_t nwords, uint64_t e_loc,
                                uint64_t e_base, double sigma, uint64_t key, int all_ones) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nwords;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t word = 0;
        if (i < nwords) {
#pragma unroll 4
            for (int b = 0; b < 32; ++b) {
                const uint64_t e = i * 32 + b;
                if (e >= e_loc) break;
                bool f;
                if (all_ones) {
                    f = true;
                } else {
                    const double u = (double)(mix64(key ^ (e_base + e)) >> 11) * 0x1.0p-53;
                    f = u < sigma;
                }
                word |= (f ? 1u : 0u) << b;
            }
        }
        bitmap[i] = word;  // bitmap[nwords] is the zero guard word
    }
}

void sparsify_bitmap(DevGraph& g, uint32_t* bitmap, double sigma, uint64_t seed, bool all_ones) {
    const uint64_t nwords = (g.e_loc + 31) / 32;
    sparsify_kernel<<<grid_for(nwords + 1, 256), 256, 0, g.stream>>>(
        bitmap, nwords, g.e_loc, g.e_base, sigma, mix64(seed), all_ones ? 1 : 0);
    GGB_CUDA(cudaGetLastError());
}

// --------------------------------------------------------------------------
// work lists
// --------------------------------------------------------------------------
__device__ __forceinline__ uint32_t window_chunks(uint64_t edges) {
    const uint64_t nrows = (edges + 31) >> 5;
    return nrows > (uint64_t)kRowsPerChunk
               ? (uint32_t)((nrows + kRowsPerChunk - 1) / kRowsPerChunk) : 1u;
}

__global__ void task_count_kernel(const uint64_t* __restrict__ off, uint64_t nloc, uint64_t nwin,
                                  uint64_t* __restrict__ cnt) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w <= nwin;
         w += (uint64_t)gridDim.x * blockDim.x) {
        if (w == nwin) { cnt[w] = 0; continue; }
        const uint64_t v0 = w * kWindow;
        const uint64_t v1 = v0 + kWindow < nloc ? v0 + kWindow : nloc;
        const uint32_t nch = window_chunks(off[v1] - off[v0]);
        cnt[w] = (uint64_t)nch | (nch > 1 ? (uint64_t)nch << 32 : 0ull);
    }
}

__global__ void task_fill_kernel(const uint64_t* __restrict__ pref, uint64_t nwin,
                                 uint4* __restrict__ tasks, uint4* __restrict__ mtasks) {
    for (uint64_t w = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; w < nwin;
         w += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p0 = pref[w], p1 = pref[w + 1];
        const uint32_t first = (uint32_t)p0, nch = (uint32_t)p1 - first;
        const uint32_t mfirst = (uint32_t)(p0 >> 32);
        for (uint32_t c = 0; c < nch; ++c) {
            const uint4 t = make_uint4((uint32_t)w, c, nch, nch > 1 ? mfirst : 0xffffffffu);
            tasks[first + c] = t;
            if (nch > 1) mtasks[mfirst + c] = t;
        }
    }
}

void build_tasks(DevGraph& g, const uint64_t* off, const std::string& tag, TaskList& out) {
    const uint64_t nwin = (g.nloc + kWindow - 1) / kWindow;
    uint64_t* cnt = g.ws.get<uint64_t>(tag + ".cnt", nwin + 1);
    uint64_t* pref = g.ws.get<uint64_t>(tag + ".pref", nwin + 1);
    task_count_kernel<<<grid_for(nwin + 1, 256), 256, 0, g.stream>>>(off, g.nloc, nwin, cnt);
    GGB_CUDA(cudaGetLastError());
    size_t tmp = 0;
    GGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, pref, nwin + 1, g.stream));
    void* tmpp = g.ws.get("cub.tmp." + tag, tmp);
    GGB_CUDA(cub::DeviceScan::ExclusiveSum(tmpp, tmp, cnt, pref, nwin + 1, g.stream));
    uint64_t total = 0;
    GGB_CUDA(cudaMemcpyAsync(&total, pref + nwin, 8, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    out.ntasks = (uint32_t)total;
    out.nmtasks = (uint32_t)(total >> 32);
    out.tasks = g.ws.get<uint4>(tag + ".tasks", out.ntasks + 1);
    out.mtasks = g.ws.get<uint4>(tag + ".mtasks", out.nmtasks + 1);
    if (nwin)
        task_fill_kernel<<<grid_for(nwin, 256), 256, 0, g.stream>>>(pref, nwin, out.tasks,
                                                                    out.mtasks);
    GGB_CUDA(cudaGetLastError());
}

// --------------------------------------------------------------------------
// bitmap -> sparsified CSC
// --------------------------------------------------------------------------
__global__ void popc_kernel(const uint32_t* __restrict__ bitmap, uint64_t nwords,
                            uint64_t* __restrict__ cnt) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nwords;
         i += (uint64_t)gridDim.x * blockDim.x)
        cnt[i] = i < nwords ? (uint64_t)__popc(bitmap[i]) : 0ull;
}

__device__ __forceinline__ uint64_t bit_rank(const uint32_t* bitmap, const uint64_t* wpref,
                                             uint64_t e) {
    const uint64_t w = e >> 5;
    const uint32_t b = (uint32_t)(e & 31);
    return wpref[w] + (uint64_t)__popc(bitmap[w] & ((1u << b) - 1u));
}

__global__ void soff_kernel(const uint64_t* __restrict__ off, uint64_t nloc,
                            const uint32_t* __restrict__ bitmap,
                            const uint64_t* __restrict__ wpref, uint64_t* __restrict__ s_off) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= nloc;
         v += (uint64_t)gridDim.x * blockDim.x)
        s_off[v] = bit_rank(bitmap, wpref, off[v]);
}

template <int WB>
__global__ void compact_kernel(const uint32_t* __restrict__ src, const void* __restrict__ w,
                               uint64_t e_loc, const uint32_t* __restrict__ bitmap,
                               const uint64_t* __restrict__ wpref, uint32_t* __restrict__ s_src,
                               void* __restrict__ s_w) {
    // warp-aligned: lane == e & 31, so the word and its prefix are shared
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < e_loc;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t word = __ldg(bitmap + (e >> 5));
        const uint32_t b = (uint32_t)(e & 31);
        if ((word >> b) & 1u) {
            const uint64_t pos = __ldg(wpref + (e >> 5)) + (uint64_t)__popc(word & ((1u << b) - 1u));
            s_src[pos] = __ldg(src + e);
            if constexpr (WB == 4)
                static_cast<uint32_t*>(s_w)[pos] = __ldg(static_cast<const uint32_t*>(w) + e);
            if constexpr (WB == 8)
                static_cast<unsigned long long*>(s_w)[pos] =
                    __ldg(static_cast<const unsigned long long*>(w) + e);
        }
    }
}

uint64_t rebuild_sparse(DevGraph& g, const uint32_t* bitmap, uint64_t* s_off, uint32_t* s_src,
                        void* s_w, TaskList& out, const std::string& tag, cudaEvent_t ev0,
                        cudaEvent_t ev1, int* launches) {
    const uint64_t nwords = (g.e_loc + 31) / 32;
    uint64_t* cnt = g.ws.get<uint64_t>("rb.cnt", nwords + 1);
    uint64_t* wpref = g.ws.get<uint64_t>("rb.wpref", nwords + 1);
    if (ev0) GGB_CUDA(cudaEventRecord(ev0, g.stream));
    popc_kernel<<<grid_for(nwords + 1, 256), 256, 0, g.stream>>>(bitmap, nwords, cnt);
    GGB_CUDA(cudaGetLastError());
    size_t tmp = 0;
    GGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, cnt, wpref, nwords + 1, g.stream));
    void* tmpp = g.ws.get("cub.tmp.rb", tmp);
    GGB_CUDA(cub::DeviceScan::ExclusiveSum(tmpp, tmp, cnt, wpref, nwords + 1, g.stream));
    soff_kernel<<<grid_for(g.nloc + 1, 256), 256, 0, g.stream>>>(g.off, g.nloc, bitmap, wpref,
                                                                  s_off);
    GGB_CUDA(cudaGetLastError());
    const size_t wb = weight_size(g.wkind);
    const unsigned gr = grid_for(g.e_loc, 256, 148ull * 16 * 8);
    if (g.e_loc) {
        if (wb == 0)
            compact_kernel<0><<<gr, 256, 0, g.stream>>>(g.src, g.w, g.e_loc, bitmap, wpref, s_src, s_w);
        else if (wb == 4)
            compact_kernel<4><<<gr, 256, 0, g.stream>>>(g.src, g.w, g.e_loc, bitmap, wpref, s_src, s_w);
        else
            compact_kernel<8><<<gr, 256, 0, g.stream>>>(g.src, g.w, g.e_loc, bitmap, wpref, s_src, s_w);
        GGB_CUDA(cudaGetLastError());
    }
    build_tasks(g, s_off, tag, out);
    if (ev1) GGB_CUDA(cudaEventRecord(ev1, g.stream));
    if (launches) *launches += 6;
    uint64_t kept = 0;
    GGB_CUDA(cudaMemcpyAsync(&kept, wpref + nwords, 8, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    return kept;
}

__global__ void superstep_invalid_kernel(uint32_t nloc, uint32_t v_begin,
                                         const uint8_t* __restrict__ st_cur,
                                         const uint8_t* __restrict__ st_next,
                                         const uint64_t* __restrict__ s_off,
                                         IterCounters* __restrict__ ctr) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < nloc; v += gridDim.x * blockDim.x) {
        if ((st_next[v] & kStInvalid) && ((st_cur[v] & kStActive) || s_off[v + 1] > s_off[v]))
            atomicMin(&ctr->bad_min, v_begin + v);
    }
}

void launch_superstep_invalid(DevGraph& g, const uint8_t* st_cur, const uint8_t* st_next,
                              const uint64_t* s_off, void* ctr) {
    superstep_invalid_kernel<<<grid_for(g.nloc, 256), 256, 0, g.stream>>>(
        (uint32_t)g.nloc, (uint32_t)g.v_begin, st_cur, st_next, s_off,
        static_cast<IterCounters*>(ctr));
    GGB_CUDA(cudaGetLastError());
}

DevGraph::~DevGraph() {
    ws.release();
    if (off) cudaFree(off);
    if (src) cudaFree(src);
    if (w) cudaFree(w);
    if (outdeg) cudaFree(outdeg);
    if (stream) cudaStreamDestroy(stream);
}

}  // namespace ggb
