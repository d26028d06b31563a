// rmat.cu — R-MAT inputs generated straight into HBM.
//
// Same specification as the CPU checker (oracle/gg_oracle.c, og_rmat):
//   key = mix64(seed); edge i, level l: u = to_unit(mix64(key ^ (i*64 + l)))
//   quadrant a | b | c | d by u < a, a+b, a+b+c (MSB first; a = (0,0),
//   b = (src 0, dst 1), c = (1, 0), d = (1, 1)); self-loops and duplicate
//   pairs removed; CSC sorted by (dst, src); no permutation.
// The edge set is a deterministic function of the spec, so the GPU build
// (radix sort + unique) and the CPU build (counting sort) are identical.
#include <cub/cub.cuh>

#include "graph.cuh"

namespace ggb {

__global__ void rmat_keys_kernel(uint64_t m, uint32_t scale, uint64_t key, double t1, double t2,
                                 double t3, uint64_t* __restrict__ keys) {
    const uint64_t invalid = 1ull << (2 * scale);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t s = 0, d = 0;
        for (uint32_t l = 0; l < scale; ++l) {
            const double u = to_unit(mix64(key ^ (i * 64 + l)));
            uint32_t sb, db;
            if (u < t1) { sb = 0; db = 0; }
            else if (u < t2) { sb = 0; db = 1; }
            else if (u < t3) { sb = 1; db = 0; }
            else { sb = 1; db = 1; }
            s = (s << 1) | sb;
            d = (d << 1) | db;
        }
        keys[i] = s == d ? invalid : (((uint64_t)d << scale) | s);
    }
}

// reference symmetrized() order (graph.cpp:249-257): per destination, the
// original in-edges (ascending source) then the reversed out-edges
// (ascending original destination) -> key (dst, part, src).
__global__ void sym_keys_kernel(const uint64_t* __restrict__ in, uint64_t e, uint32_t scale,
                                uint64_t* __restrict__ out) {
    const uint64_t mask = (1ull << scale) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t k = in[i];
        const uint64_t s = k & mask, d = k >> scale;
        out[i] = (d << (scale + 1)) | s;
        out[e + i] = (s << (scale + 1)) | (1ull << scale) | d;
    }
}

__global__ void csc_from_keys_kernel(const uint64_t* __restrict__ keys, uint64_t e, uint64_t n,
                                     uint32_t scale, uint32_t dshift, uint32_t* __restrict__ src,
                                     uint64_t* __restrict__ off) {
    const uint64_t mask = (1ull << scale) - 1;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= e;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t d = i < e ? (int64_t)(keys[i] >> dshift) : (int64_t)n;
        const int64_t dp = i > 0 ? (int64_t)(keys[i - 1] >> dshift) : -1;
        if (i < e) src[i] = (uint32_t)(keys[i] & mask);
        for (int64_t v = dp + 1; v <= d; ++v) off[v] = i;
    }
}

__global__ void outdeg_kernel(const uint32_t* __restrict__ src, uint64_t e,
                              uint32_t* __restrict__ deg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x)
        atomicAdd(deg + src[i], 1u);
}

// BASELINE C2 weights: 1 + mix64(kw ^ e) % 255, kw = mix64(mix64(seed) ^ "weights")
__global__ void weights_u32_kernel(uint64_t e, uint64_t seed, uint32_t* __restrict__ w) {
    const uint64_t kw = mix64(mix64(seed) ^ 0x77656967687473ull);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x)
        w[i] = 1u + (uint32_t)(mix64(kw ^ i) % 255u);
}

// BASELINE C4 couplings: c_e = fp32(0.5 + 0.4 * to_unit(mix64(kc ^ e)))
__global__ void couplings_kernel(uint64_t e, uint64_t seed, float* __restrict__ w) {
    const uint64_t kc = mix64(mix64(seed) ^ 0x636f75706c65ull);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < e;
         i += (uint64_t)gridDim.x * blockDim.x)
        w[i] = (float)(0.5 + 0.4 * to_unit(mix64(kc ^ i)));
}

// BASELINE C4 priors: uniform (0,1) per state, normalised, fp32.
__global__ void priors_kernel(uint64_t n, uint64_t seed, float* __restrict__ out) {
    const uint64_t kp = mix64(mix64(seed) ^ 0x7072696f7273ull);
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const double p0 = ((double)(mix64(kp ^ (2 * v)) >> 11) + 0.5) * 0x1.0p-53;
        const double p1 = ((double)(mix64(kp ^ (2 * v + 1)) >> 11) + 0.5) * 0x1.0p-53;
        const double s = p0 + p1;
        out[2 * v] = (float)(p0 / s);
        out[2 * v + 1] = (float)(p1 / s);
    }
}

static unsigned g1(uint64_t n) {
    uint64_t g = (n + 255) / 256;
    if (g > 148ull * 64) g = 148ull * 64;
    return (unsigned)(g ? g : 1);
}

// Generates the full graph on the current device.
RmatCsc rmat_generate(const gg_rmat_params& p, cudaStream_t st) {
    if (p.scale < 1 || p.scale > 31) throw Error(GG_INVALID_ARGUMENT, "rmat scale must be in [1,31]");
    RmatCsc out;
    const uint64_t n = 1ull << p.scale;
    const uint64_t m = (uint64_t)p.edge_factor << p.scale;
    out.n = n;
    if (m >= (1ull << 31)) throw Error(GG_INVALID_ARGUMENT, "rmat: at most 2^31-1 raw edges");
    uint64_t *k0 = nullptr, *k1 = nullptr;
    k0 = static_cast<decltype(k0)>(dev_alloc((m + 1) * 8, st));
    k1 = static_cast<decltype(k1)>(dev_alloc((m + 1) * 8, st));
    rmat_keys_kernel<<<g1(m), 256, 0, st>>>(m, p.scale, mix64(p.seed), p.a, p.a + p.b,
                                            p.a + p.b + p.c, k0);
    GGB_CUDA(cudaGetLastError());
    size_t tmp_sort = 0, tmp_uniq = 0;
    int* d_num = nullptr;
    d_num = static_cast<decltype(d_num)>(dev_alloc(8, st));
    GGB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tmp_sort, k0, k1, m, 0, 2 * p.scale + 1, st));
    GGB_CUDA(cub::DeviceSelect::Unique(nullptr, tmp_uniq, k1, k0, d_num, m, st));
    void* tmp = nullptr;
    tmp = static_cast<decltype(tmp)>(dev_alloc(std::max(tmp_sort, tmp_uniq), st));
    GGB_CUDA(cub::DeviceRadixSort::SortKeys(tmp, tmp_sort, k0, k1, m, 0, 2 * p.scale + 1, st));
    GGB_CUDA(cub::DeviceSelect::Unique(tmp, tmp_uniq, k1, k0, d_num, m, st));
    int num = 0;
    GGB_CUDA(cudaMemcpyAsync(&num, d_num, 4, cudaMemcpyDeviceToHost, st));
    GGB_CUDA(cudaStreamSynchronize(st));
    uint64_t e = (uint64_t)(uint32_t)num;
    if (e) {
        uint64_t last = 0;
        GGB_CUDA(cudaMemcpy(&last, k0 + e - 1, 8, cudaMemcpyDeviceToHost));
        if (last == (1ull << (2 * p.scale))) --e;  // the (single, deduplicated) self-loop key
    }
    uint64_t* keys = k0;
    uint32_t dshift = p.scale;
    if (p.symmetrize) {
        dev_free(k1, st);
        k1 = nullptr;
        uint64_t *s0 = nullptr, *s1 = nullptr;
        s0 = static_cast<decltype(s0)>(dev_alloc((2 * e + 1) * 8, st));
        sym_keys_kernel<<<g1(e), 256, 0, st>>>(k0, e, p.scale, s0);
        GGB_CUDA(cudaGetLastError());
        GGB_CUDA(cudaStreamSynchronize(st));
        dev_free(k0, st);
        k0 = nullptr;
        s1 = static_cast<decltype(s1)>(dev_alloc((2 * e + 1) * 8, st));
        size_t t2 = 0;
        GGB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, t2, s0, s1, 2 * e, 0, 2 * p.scale + 2, st));
        if (t2 > std::max(tmp_sort, tmp_uniq)) {
            dev_free(tmp, st);
            tmp = static_cast<decltype(tmp)>(dev_alloc(t2, st));
        }
        GGB_CUDA(cub::DeviceRadixSort::SortKeys(tmp, t2, s0, s1, 2 * e, 0, 2 * p.scale + 2, st));
        GGB_CUDA(cudaStreamSynchronize(st));
        dev_free(s0, st);
        keys = s1;
        k0 = s1;
        e = 2 * e;
        dshift = p.scale + 1;
    }
    out.e = e;
    out.off = static_cast<decltype(out.off)>(dev_alloc((n + 1) * 8, st));
    out.src = static_cast<decltype(out.src)>(dev_alloc((e + 1) * 4, st));
    out.outdeg = static_cast<decltype(out.outdeg)>(dev_alloc(n * 4, st));
    GGB_CUDA(cudaMemsetAsync(out.outdeg, 0, n * 4, st));
    csc_from_keys_kernel<<<g1(e + 1), 256, 0, st>>>(keys, e, n, p.scale, dshift, out.src, out.off);
    GGB_CUDA(cudaGetLastError());
    outdeg_kernel<<<g1(e), 256, 0, st>>>(out.src, e, out.outdeg);
    GGB_CUDA(cudaGetLastError());
    if (p.weight_kind == GG_W_U32) {
        out.w = static_cast<decltype(out.w)>(dev_alloc((e + 1) * 4, st));
        weights_u32_kernel<<<g1(e), 256, 0, st>>>(e, p.seed, static_cast<uint32_t*>(out.w));
    } else if (p.weight_kind == GG_W_F32) {
        out.w = static_cast<decltype(out.w)>(dev_alloc((e + 1) * 4, st));
        couplings_kernel<<<g1(e), 256, 0, st>>>(e, p.seed, static_cast<float*>(out.w));
    } else if (p.weight_kind != GG_W_NONE) {
        throw Error(GG_INVALID_ARGUMENT, "rmat weight_kind must be none, u32 or f32");
    }
    GGB_CUDA(cudaGetLastError());
    GGB_CUDA(cudaStreamSynchronize(st));
    if (k0) dev_free(k0, st);
    if (k1) dev_free(k1, st);
    dev_free(tmp, st);
    dev_free(d_num, st);
    return out;
}

void bp_priors_device(uint64_t n, uint64_t seed, float* out, cudaStream_t st) {
    priors_kernel<<<g1(n), 256, 0, st>>>(n, seed, out);
    GGB_CUDA(cudaGetLastError());
}

}  // namespace ggb
