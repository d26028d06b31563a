// metrics.cu — the reference's error metrics (metrics.cpp:23-113) on device
// arrays, so a sweep compares an approximate run with the exact one without
// moving either property vector to the host.
//
//   top-k:    both vectors ranked by (value desc, vertex asc) with a stable
//             radix sort of order-preserving keys (metrics.cpp:23-36 uses
//             partial_sort with the same comparator): identical sets, so the
//             missing count — and the error — are exact.
//   relative: mean of min(1, |e+1 - (a+1)| / (e+1))   (metrics.cpp:74-86)
//   stretch:  mean of 1 - e/a over exactly-reachable vertices, a < e aborts
//             naming the vertex                       (metrics.cpp:88-113)
// The two sums are reduced in a fixed order (deterministic run to run); they
// differ from the reference's left-to-right double sum only by rounding.
#include <cub/cub.cuh>

#include "graph.cuh"

namespace ggb {
namespace {

constexpr int kRedThreads = 256;
constexpr int kRedBlocks = 148 * 4;

// ascending order of the unsigned key == descending order of the double;
// -0.0 ranks with +0.0 (the reference comparator treats them as equal)
__global__ void topk_keys_kernel(const double* __restrict__ v, uint64_t n,
                                 uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        double x = v[i];
        if (x == 0.0) x = 0.0;
        uint64_t b = (uint64_t)__double_as_longlong(x);
        b = (b >> 63) ? ~b : (b | 0x8000000000000000ull);  // ascending-order key
        keys[i] = ~b;                                      // descending
        idx[i] = (uint32_t)i;
    }
}

__global__ void mark_kernel(const uint32_t* __restrict__ idx, uint64_t k, uint8_t* __restrict__ in) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x)
        in[idx[i]] = 1;
}

__global__ void missing_kernel(const uint32_t* __restrict__ idx, uint64_t k,
                               const uint8_t* __restrict__ in, unsigned long long* __restrict__ out) {
    unsigned long long c = 0;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < k;
         i += (uint64_t)gridDim.x * blockDim.x)
        c += in[idx[i]] ? 0 : 1;
    for (int d = 16; d; d >>= 1) c += __shfl_down_sync(0xffffffffu, c, d);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// Fixed-order reduction: thread partials in grid-stride order, a fixed tree
// per block, then one thread adds the block partials in block order.
__device__ void block_sum(double s, unsigned long long c, double* part_s,
                          unsigned long long* part_c) {
    __shared__ double ss[kRedThreads];
    __shared__ unsigned long long cc[kRedThreads];
    ss[threadIdx.x] = s;
    cc[threadIdx.x] = c;
    __syncthreads();
    for (int d = kRedThreads / 2; d; d >>= 1) {
        if (threadIdx.x < (unsigned)d) {
            ss[threadIdx.x] += ss[threadIdx.x + d];
            cc[threadIdx.x] += cc[threadIdx.x + d];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part_s[blockIdx.x] = ss[0];
        part_c[blockIdx.x] = cc[0];
    }
}

__global__ void __launch_bounds__(kRedThreads)
relative_kernel(const double* __restrict__ a, const double* __restrict__ e, uint64_t n,
                double* __restrict__ part_s, unsigned long long* __restrict__ part_c) {
    double s = 0.0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const double av = a[v] + 1.0, ev = e[v] + 1.0;
        const double t = fabs(ev - av) / ev;
        s += t < 1.0 ? t : 1.0;
    }
    block_sum(s, 0, part_s, part_c);
}

__global__ void __launch_bounds__(kRedThreads)
stretch_kernel(const double* __restrict__ a, const double* __restrict__ e, uint64_t n,
               double* __restrict__ part_s, unsigned long long* __restrict__ part_c,
               unsigned int* __restrict__ bad) {
    double s = 0.0;
    unsigned long long c = 0;
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const double ev = e[v], av = a[v];
        if (av < ev) {
            atomicMin(bad, (unsigned int)v);
            continue;
        }
        if (isinf(ev)) continue;               // unreachable either way
        if (ev == 0.0 && av == 0.0) continue;  // the source
        ++c;
        s += (isinf(av) || ev == 0.0) ? 1.0 : 1.0 - ev / av;
    }
    block_sum(s, c, part_s, part_c);
}

__global__ void finish_kernel(const double* __restrict__ part_s,
                              const unsigned long long* __restrict__ part_c, int nb,
                              double* __restrict__ out_s, unsigned long long* __restrict__ out_c) {
    double s = 0.0;
    unsigned long long c = 0;
    for (int b = 0; b < nb; ++b) {
        s += part_s[b];
        c += part_c[b];
    }
    *out_s = s;
    *out_c = c;
}

struct Scratch {  // one-call device scratch from the stream-ordered pool
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    template <class T>
    T* get(size_t count) {
        ptrs.push_back(dev_alloc(count * sizeof(T), st));
        return static_cast<T*>(ptrs.back());
    }
    ~Scratch() {
        for (void* p : ptrs) dev_free(p, st);
        cudaStreamSynchronize(st);
    }
};

void sorted_indices(const double* v, uint64_t n, uint32_t* idx_out, Scratch& sc, cudaStream_t st) {
    uint64_t* k0 = sc.get<uint64_t>(n);
    uint64_t* k1 = sc.get<uint64_t>(n);
    uint32_t* i0 = sc.get<uint32_t>(n);
    topk_keys_kernel<<<kRedBlocks, 256, 0, st>>>(v, n, k0, i0);
    GGB_CUDA(cudaGetLastError());
    size_t tmp = 0;
    GGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, i0, idx_out, n, 0, 64, st));
    void* t = sc.get<char>(tmp);
    GGB_CUDA(cub::DeviceRadixSort::SortPairs(t, tmp, k0, k1, i0, idx_out, n, 0, 64, st));
}

double reduce_mean(bool stretch, const double* a, const double* e, uint64_t n, uint32_t* bad_out,
                   cudaStream_t st) {
    Scratch sc(st);
    double* ps = sc.get<double>(kRedBlocks);
    unsigned long long* pc = sc.get<unsigned long long>(kRedBlocks);
    double* os = sc.get<double>(1);
    unsigned long long* oc = sc.get<unsigned long long>(1);
    unsigned int* bad = sc.get<unsigned int>(1);
    GGB_CUDA(cudaMemsetAsync(bad, 0xff, 4, st));
    if (stretch)
        stretch_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(a, e, n, ps, pc, bad);
    else
        relative_kernel<<<kRedBlocks, kRedThreads, 0, st>>>(a, e, n, ps, pc);
    GGB_CUDA(cudaGetLastError());
    finish_kernel<<<1, 1, 0, st>>>(ps, pc, kRedBlocks, os, oc);
    GGB_CUDA(cudaGetLastError());
    double s = 0.0;
    unsigned long long c = 0;
    unsigned int b = 0;
    GGB_CUDA(cudaMemcpyAsync(&s, os, 8, cudaMemcpyDeviceToHost, st));
    GGB_CUDA(cudaMemcpyAsync(&c, oc, 8, cudaMemcpyDeviceToHost, st));
    GGB_CUDA(cudaMemcpyAsync(&b, bad, 4, cudaMemcpyDeviceToHost, st));
    GGB_CUDA(cudaStreamSynchronize(st));
    if (bad_out) *bad_out = b;
    if (stretch) return c == 0 ? 0.0 : s / (double)c;
    return s / (double)n;
}

}  // namespace
}  // namespace ggb

using namespace ggb;

extern "C" {

gg_status gg_topk_error_dev(const double* approx, const double* exact, uint64_t n, uint64_t k,
                            double* err_out) {
    return guarded(nullptr, [&] {
        if (k < 1 || k > n) throw Error(GG_INVALID_ARGUMENT, "topk k must be in [1, N]");
        if (n > 0xffffffffull) throw Error(GG_INVALID_ARGUMENT, "topk: n exceeds 32-bit ids");
        cudaStream_t st = nullptr;
        GGB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        double err = 0.0;
        {
            Scratch sc(st);
            uint32_t* ia = sc.get<uint32_t>(n);
            uint32_t* ie = sc.get<uint32_t>(n);
            uint8_t* in = sc.get<uint8_t>(n);
            unsigned long long* miss = sc.get<unsigned long long>(1);
            sorted_indices(approx, n, ia, sc, st);
            sorted_indices(exact, n, ie, sc, st);
            GGB_CUDA(cudaMemsetAsync(in, 0, n, st));
            GGB_CUDA(cudaMemsetAsync(miss, 0, 8, st));
            mark_kernel<<<kRedBlocks, 256, 0, st>>>(ie, k, in);
            missing_kernel<<<kRedBlocks, 256, 0, st>>>(ia, k, in, miss);
            GGB_CUDA(cudaGetLastError());
            unsigned long long m = 0;
            GGB_CUDA(cudaMemcpyAsync(&m, miss, 8, cudaMemcpyDeviceToHost, st));
            GGB_CUDA(cudaStreamSynchronize(st));
            err = (double)m / (double)k;
        }
        cudaStreamDestroy(st);
        *err_out = err;
    });
}

gg_status gg_relative_error_dev(const double* approx, const double* exact, uint64_t n,
                                double* err_out) {
    return guarded(nullptr, [&] {
        if (n == 0) {
            *err_out = 0.0;
            return;
        }
        cudaStream_t st = nullptr;
        GGB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        double r = 0.0;
        try {
            r = reduce_mean(false, approx, exact, n, nullptr, st);
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        cudaStreamDestroy(st);
        *err_out = r;
    });
}

gg_status gg_stretch_error_dev(const double* approx, const double* exact, uint64_t n,
                               double* err_out, gg_error* err) {
    return guarded(err, [&] {
        cudaStream_t st = nullptr;
        GGB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        uint32_t bad = 0xffffffffu;
        double r = 0.0;
        try {
            r = n ? reduce_mean(true, approx, exact, n, &bad, st) : 0.0;
        } catch (...) {
            cudaStreamDestroy(st);
            throw;
        }
        cudaStreamDestroy(st);
        if (bad != 0xffffffffu) {  // metrics.cpp:96-100
            Error e(GG_INVALID_ARGUMENT,
                    "stretch_error: approximate distance below exact at vertex " +
                        std::to_string(bad) + " (engine bug)");
            e.vertex = bad;
            throw e;
        }
        *err_out = r;
    });
}

gg_status gg_last_projection(gg_dev_graph* g, const double** dev_out) {
    return guarded(nullptr, [&] {
        if (!g || !dev_out) throw Error(GG_INVALID_ARGUMENT, "null argument");
        if (!g->g.project_last) throw Error(GG_INVALID_ARGUMENT, "no run on this graph yet");
        GGB_CUDA(cudaSetDevice(g->g.device));
        *dev_out = g->g.project_last();
    });
}

gg_status gg_device_copy(const void* dev_src, uint64_t bytes, void** dev_out) {
    return guarded(nullptr, [&] {
        if (!dev_out || (bytes && !dev_src)) throw Error(GG_INVALID_ARGUMENT, "null argument");
        void* d = nullptr;
        GGB_CUDA(cudaMalloc(&d, bytes ? bytes : 16));
        if (bytes) GGB_CUDA(cudaMemcpy(d, dev_src, bytes, cudaMemcpyDeviceToDevice));
        *dev_out = d;
    });
}

}  // extern "C"
