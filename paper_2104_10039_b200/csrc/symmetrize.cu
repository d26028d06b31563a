// symmetrize.cu — graph.cpp:249-257 symmetrized() on the device: the
// multiset union of the graph and its reverse, built by a STABLE scatter by
// destination of [the edges in edge-id order, then their reversals in
// edge-id order]. Per destination d that is: d's own in-edges in CSC order,
// then the reversals of d's out-edges in ascending edge id (= ascending
// original destination). One radix sort of 64-bit keys
// (new destination, part, edge id) reproduces that order exactly; WCC runs
// on this graph (bench.cpp:280-287), and its masks depend on the order.
#include <cub/cub.cuh>

#include "graph.cuh"

namespace ggb {
namespace {

unsigned grid_of(uint64_t n) {
    uint64_t g = (n + 255) / 256;
    return (unsigned)(g < 1 ? 1 : (g > 148ull * 64 ? 148ull * 64 : g));
}

// destination (global vertex id) of every edge: one warp per row
__global__ void edge_dst_kernel(const uint64_t* __restrict__ row_start, uint64_t nrows,
                                const uint32_t* __restrict__ vid_of_p, uint32_t* __restrict__ dst) {
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const int lane = threadIdx.x & 31;
    for (uint64_t p = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; p < nrows; p += warps) {
        const uint32_t v = vid_of_p[p];
        for (uint64_t e = row_start[p] + lane; e < row_start[p + 1]; e += 32) dst[e] = v;
    }
}

// keys of both orientations: (new dst << 32) | (part << 31) | edge id
__global__ void sym_edge_keys_kernel(const uint32_t* __restrict__ src_slot, const uint32_t* __restrict__ vtx_of_slot,
                                     const uint32_t* __restrict__ dst, uint64_t e,
                                     uint64_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t s = vtx_of_slot[src_slot[i]], d = dst[i];
        keys[i] = (d << 32) | i;
        keys[e + i] = (s << 32) | (1ull << 31) | i;
    }
}

// sorted keys -> CSC: sources, offsets, weights, out-degrees
template <class WT>
__global__ void sym_fill_kernel(const uint64_t* __restrict__ keys, uint64_t e2, uint64_t n,
                                const uint32_t* __restrict__ src_slot,
                                const uint32_t* __restrict__ vtx_of_slot,
                                const uint32_t* __restrict__ dst, const WT* __restrict__ w_in,
                                uint32_t* __restrict__ src, WT* __restrict__ w_out,
                                uint64_t* __restrict__ off, uint32_t* __restrict__ deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= e2;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t d = i < e2 ? (int64_t)(keys[i] >> 32) : (int64_t)n;
        const int64_t dp = i > 0 ? (int64_t)(keys[i - 1] >> 32) : -1;
        for (int64_t v = dp + 1; v <= d; ++v) off[v] = i;
        if (i == e2) continue;
        const uint64_t k = keys[i];
        const uint64_t id = k & 0x7fffffffull;
        const uint32_t s = (k >> 31) & 1ull ? dst[id] : vtx_of_slot[src_slot[id]];
        src[i] = s;
        atomicAdd(deg + s, 1u);
        if constexpr (!std::is_void_v<WT>) w_out[i] = w_in[id];
    }
}

}  // namespace

RmatCsc symmetrize_device(const DevGraph& g, cudaStream_t st) {
    const uint64_t e = g.e_loc, n = g.n;
    if (e >= (1ull << 31)) throw Error(GG_INVALID_ARGUMENT, "symmetrized: at most 2^31-1 edges");
    RmatCsc out;
    out.n = n;
    out.e = 2 * e;
    uint32_t* dst = static_cast<uint32_t*>(dev_alloc((e + 1) * 4, st));
    uint64_t* k0 = static_cast<uint64_t*>(dev_alloc((2 * e + 1) * 8, st));
    uint64_t* k1 = static_cast<uint64_t*>(dev_alloc((2 * e + 1) * 8, st));
    // the input's own stream must be done with its arrays (creation finished)
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    const uint32_t* src_slot = g.src + g.full.pad;
    if (g.nrows) {
        edge_dst_kernel<<<grid_of(g.nrows * 32), 256, 0, st>>>(g.full.nz_start, g.nrows, g.vid_of_p, dst);
        GGB_CUDA(cudaGetLastError());
    }
    if (e) {
        sym_edge_keys_kernel<<<grid_of(e), 256, 0, st>>>(src_slot, g.vtx_of_slot, dst, e, k0);
        GGB_CUDA(cudaGetLastError());
    }
    int vbits = 1;
    while (vbits < 32 && (1ull << vbits) < n) ++vbits;
    size_t tmp = 0;
    GGB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp, k0, k1, 2 * e, 0, 32 + vbits, st));
    void* tmpp = dev_alloc(tmp, st);
    GGB_CUDA(cub::DeviceRadixSort::SortKeys(tmpp, tmp, k0, k1, 2 * e, 0, 32 + vbits, st));
    dev_free(tmpp, st);
    dev_free(k0, st);
    out.off = static_cast<uint64_t*>(dev_alloc((n + 1) * 8, st));
    out.src = static_cast<uint32_t*>(dev_alloc((2 * e + 1) * 4, st));
    out.outdeg = static_cast<uint32_t*>(dev_alloc((n + 1) * 4, st));
    GGB_CUDA(cudaMemsetAsync(out.outdeg, 0, (n + 1) * 4, st));
    const size_t wb = weight_size(g.wkind);
    if (wb) out.w = dev_alloc((2 * e + 1) * wb, st);
    const unsigned gr = grid_of(2 * e + 1);
    const char* w_in = g.w ? static_cast<const char*>(g.w) + g.full.pad * wb : nullptr;
    if (wb == 0)
        sym_fill_kernel<void><<<gr, 256, 0, st>>>(k1, 2 * e, n, src_slot, g.vtx_of_slot, dst, nullptr,
                                                  out.src, nullptr, out.off, out.outdeg);
    else if (wb == 4)
        sym_fill_kernel<uint32_t><<<gr, 256, 0, st>>>(
            k1, 2 * e, n, src_slot, g.vtx_of_slot, dst, reinterpret_cast<const uint32_t*>(w_in), out.src,
            static_cast<uint32_t*>(out.w), out.off, out.outdeg);
    else
        sym_fill_kernel<unsigned long long><<<gr, 256, 0, st>>>(
            k1, 2 * e, n, src_slot, g.vtx_of_slot, dst, reinterpret_cast<const unsigned long long*>(w_in),
            out.src, static_cast<unsigned long long*>(out.w), out.off, out.outdeg);
    GGB_CUDA(cudaGetLastError());
    GGB_CUDA(cudaStreamSynchronize(st));
    dev_free(k1, st);
    dev_free(dst, st);
    return out;
}

}  // namespace ggb
