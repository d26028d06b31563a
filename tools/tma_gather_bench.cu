// tma_gather_bench.cu — calibration microbenchmark (not part of the product):
// can the TMA engine's tile::gather4 (sm_100a) serve index-driven 8-byte
// message gathers at a rate that adds to the LDG path, whose random gathers
// are bound by the L1TEX wavefront rate (~1 line per cycle per SM)?
//
//   ./tma_gather_bench <mode> <skew> [reps]
//     mode: ldg | tma | mix (half the warps LDG, half TMA)
//     skew: index = floor(n * u^skew), u uniform (1 = uniform; 6 ~ the
//           hot-first R-MAT slot marginal: 2^14 of 2^26 slots take ~25%)
//
// Messages: f64[n], n = 2^26 (537 MB). The TMA view is a 2-D tensor of n/2
// rows x 2 f64 (16-byte rows, the minimum box width): gather4 fetches four
// rows by index into shared memory; the lane keeps element idx & 1.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, \
                        __LINE__);                                                    \
            std::exit(1);                                                             \
        }                                                                             \
    } while (0)

__host__ __device__ inline uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

// skew 0: the hot-first slot of an R-MAT s26 source (a + b = 0.76 per bit):
// a source's out-degree falls with its popcount k, so the hot-first slot
// order is (k asc, id): slot = #(ids with popcount < k) + rank within class
__global__ void make_idx(uint32_t* idx, uint64_t m, uint64_t n, int skew) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (skew == 0) {
            int k = 0;
            for (int l = 0; l < 26; ++l)
                k += (double)(mix64(i * 64 + l + 99) >> 11) * 0x1.0p-53 < 0.24 ? 1 : 0;
            double c = 1.0, cum = 0.0;  // C(26, j)
            for (int j = 0; j < k; ++j) { cum += c; c = c * (26 - j) / (j + 1); }
            const double u2 = (double)(mix64(i * 64 + 63) >> 11) * 0x1.0p-53;
            idx[i] = (uint32_t)(cum + floor(u2 * c));
            continue;
        }
        double u = (double)(mix64(i * 0x9e37ull + 17) >> 11) * 0x1.0p-53;
        double p = u;
        for (int k = 1; k < skew; ++k) p *= u;
        uint64_t v = (uint64_t)(p * (double)n);
        idx[i] = (uint32_t)(v < n ? v : n - 1);
    }
}

__global__ void fill(double* x, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x)
        x[i] = (double)(i & 1023) * 0.5;
}

// LDG path: 16 gathers in flight per lane, indices read coalesced.
__device__ __forceinline__ double ldg_chunk(const uint32_t* __restrict__ idx, const double* __restrict__ x,
                                            uint64_t base, int lane) {
    uint32_t s[16];
    const uint4* ip = reinterpret_cast<const uint4*>(idx + base) + lane * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        uint4 v = __ldg(ip + q);
        s[4 * q] = v.x; s[4 * q + 1] = v.y; s[4 * q + 2] = v.z; s[4 * q + 3] = v.w;
    }
    double acc = 0.0, m[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) m[j] = __ldg(x + s[j]);
#pragma unroll
    for (int j = 0; j < 16; ++j) acc += m[j];
    return acc;
}

constexpr int kStages = 4;
constexpr int kChunk = 128;  // indices per warp per stage (32 lanes x one gather4)

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(b)),
                 "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    const uint32_t a = (uint32_t)__cvta_generic_to_shared(b);
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}" ::"r"(a),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_gather4(const CUtensorMap* tm, void* dst, uint64_t* bar, int r0, int r1,
                                            int r2, int r3) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"((uint32_t)__cvta_generic_to_shared(dst)),
        "l"(tm), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
        "r"((uint32_t)__cvta_generic_to_shared(bar))
        : "memory");
}

// mode 0: LDG, 1: TMA, 2: mix (odd warps TMA)
__global__ void __launch_bounds__(256) bench(const __grid_constant__ CUtensorMap tm,
                                             const uint32_t* __restrict__ idx, uint64_t m,
                                             const double* __restrict__ x, int mode,
                                             double* __restrict__ out, double tma_share) {
    extern __shared__ __align__(128) unsigned char dyn[];
    // one 128-byte aligned 64-byte landing slot per lane (TMA destinations
    // are 128-byte aligned)
    unsigned char* base = dyn + ((128 - ((uint32_t)__cvta_generic_to_shared(dyn) & 127)) & 127);
    auto buf = reinterpret_cast<unsigned char (*)[kStages][32 * 128]>(base);
    __shared__ __align__(8) uint64_t bars[8][kStages];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double acc = 0.0;
    const bool tma = mode == 1 || (mode == 2 && (w & 1));
    // mix: LDG warps (even) take the first half of the indices, TMA warps the second
    uint64_t gw = (uint64_t)blockIdx.x * 8 + w, nw = (uint64_t)gridDim.x * 8;
    uint64_t lo = 0, hi = m;
    if (mode == 2) {
        gw = (uint64_t)blockIdx.x * 4 + (w >> 1);
        nw = (uint64_t)gridDim.x * 4;
        const uint64_t cut = ((uint64_t)((double)m * (1.0 - tma_share)) / 512) * 512;
        lo = tma ? cut : 0;
        hi = tma ? m : cut;
    }
    idx += lo;
    m = hi - lo;
    const uint64_t nchunks = m / kChunk;
    if (!tma) {
        // LDG warps take 512-index chunks (16 per lane)
        for (uint64_t c = gw; c < m / 512; c += nw) acc += ldg_chunk(idx, x, c * 512, lane);
    } else {
        if (lane < kStages) mbar_init(&bars[w][lane], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        __syncwarp();
        uint32_t keep[kStages][4];
        uint32_t phase = 0;  // bit s: parity of stage s
        uint64_t it = 0;
        // chunks of 128 indices: lane issues one gather4 (its 4 indices)
        for (uint64_t c = gw; c < nchunks + (uint64_t)(kStages - 1) * nw; c += nw, ++it) {
            const int s = (int)(it % kStages);
            if (c < nchunks) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(idx + c * kChunk) + lane);
                keep[s][0] = v.x; keep[s][1] = v.y; keep[s][2] = v.z; keep[s][3] = v.w;
                if (lane == 0) mbar_expect(&bars[w][s], kChunk * 16);
                __syncwarp();
                tma_gather4(&tm, buf[w][s] + lane * 128, &bars[w][s], (int)(v.x >> 1), (int)(v.y >> 1),
                            (int)(v.z >> 1), (int)(v.w >> 1));
            }
            // consume the stage issued kStages-1 chunks ago
            if (it >= (uint64_t)(kStages - 1)) {
                const uint64_t pc = c - (uint64_t)(kStages - 1) * nw;
                if (pc < nchunks) {
                    const int ps = (int)((it - (kStages - 1)) % kStages);
                    mbar_wait(&bars[w][ps], (phase >> ps) & 1u);
                    phase ^= 1u << ps;
                    const double* rows = reinterpret_cast<const double*>(buf[w][ps] + lane * 128);
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc += rows[2 * k + (keep[ps][k] & 1)];
                }
            }
            __syncwarp();
        }
    }
    if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "ldg";
    const int skew = argc > 2 ? std::atoi(argv[2]) : 6;
    const int reps = argc > 3 ? std::atoi(argv[3]) : 5;
    const double share = argc > 4 ? std::atof(argv[4]) : 0.5;
    const uint64_t n = 1ull << 26, m = 1ull << 28;
    double* x;
    uint32_t* idx;
    double* out;
    CK(cudaMalloc(&x, n * 8));
    CK(cudaMalloc(&idx, m * 4));
    CK(cudaMalloc(&out, 8));
    fill<<<4096, 256>>>(x, n);
    make_idx<<<4096, 256>>>(idx, m, n, skew);
    CK(cudaDeviceSynchronize());

    CUtensorMap tm;
    std::memset(&tm, 0, sizeof(tm));
    typedef CUresult (*Encode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    const cuuint64_t dims[2] = {2, n / 2};
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {2, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = ((Encode)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::printf("cuTensorMapEncodeTiled failed: %d\n", (int)r);
        return 1;
    }
    const int md = mode == "ldg" ? 0 : mode == "tma" ? 1 : 2;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const int smem = 8 * kStages * 32 * 128 + 128;
    CK(cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    for (int blocks_per_sm : {1}) {
        const int grid = sms * blocks_per_sm;
        bench<<<grid, 256, smem>>>(tm, idx, m, x, md, out, share);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int i = 0; i < reps; ++i) bench<<<grid, 256, smem>>>(tm, idx, m, x, md, out, share);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        std::printf("mode=%s skew=%d share=%.2f blocks/SM=%d: %.3f ms, %.1f G gathers/s\n", mode.c_str(),
                    skew, share, blocks_per_sm, ms, (double)m / (ms * 1e-3) / 1e9);
    }
    return 0;
}
