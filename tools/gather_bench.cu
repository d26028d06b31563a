// gather_bench.cu — calibration microbenchmark (not part of the product):
// sustained bandwidth of index-driven 8-byte gathers on this B200, with
// the index stream read coalesced (like the engine's edge sources).
#include <cstdint>
#include <cuda_runtime.h>

template <int U>
__global__ void gather_sum(const uint32_t* __restrict__ idx, const double* __restrict__ x,
                           uint64_t n, double* __restrict__ out) {
    double acc = 0.0;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
    for (uint64_t base = ((uint64_t)blockIdx.x * blockDim.x) * U + threadIdx.x; base < n;
         base += stride) {
        uint32_t s[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t i = base + (uint64_t)u * blockDim.x;
            s[u] = i < n ? __ldg(idx + i) : 0u;
        }
        double v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = __ldg(x + s[u]);
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u];
    }
    if (acc == 1.2345) out[0] = acc;
}

extern "C" float gbench(const uint32_t* idx, const double* x, uint64_t n, double* out, int unroll,
                        int blocks, int threads, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&] {
        switch (unroll) {
            case 4: gather_sum<4><<<blocks, threads>>>(idx, x, n, out); break;
            case 8: gather_sum<8><<<blocks, threads>>>(idx, x, n, out); break;
            case 16: gather_sum<16><<<blocks, threads>>>(idx, x, n, out); break;
            default: gather_sum<32><<<blocks, threads>>>(idx, x, n, out); break;
        }
    };
    launch();
    cudaEventRecord(a);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}
