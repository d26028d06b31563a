// common.cuh — shared device/host helpers for libggb.so (sm_100a only).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "ggb.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "libggb.so is built for sm_100a (B200) only"
#endif

namespace ggb {

// ranks of one NVSwitch node: the fused exchange stores into at most this many replicas
constexpr int kMaxPeers = 8;


constexpr int kWarp = 32;
constexpr int kRun = 16;                 // consecutive in-edges folded by one lane
constexpr int kChunkEdges = kWarp * kRun;  // in-edges per warp task (512)

// Storage order of a SPARSIFIED list's sources (written only by the
// compaction kernels, read only by the approximate gather): inside every
// aligned task block of 512 positions the 4-source quads are transposed, quad
// q of lane L's run lies at quad q * 32 + L. A lane's four 128-bit source
// loads then touch 4 x 512 contiguous bytes per warp instead of 16 lines at a
// 64-byte lane stride each (4x fewer L1TEX wavefronts on the source stream).
// The full list keeps position order (compaction, export and the loaders
// index it by edge).
static_assert(kRun == 16 && kWarp == 32, "sp_slot assumes 16-position runs in 512-position tasks");
__host__ __device__ __forceinline__ uint64_t sp_slot(uint64_t p) {
    return (p & ~511ull) | (((p >> 2) & 3ull) << 7) | (((p >> 4) & 31ull) << 2) | (p & 3ull);
}
// uint4 index (inside the task block) of quad i of lane L's run
__host__ __device__ __forceinline__ int sp_quad(int L, int i) { return i * 32 + L; }
constexpr int kBlockThreads = 128;       // edge kernels: 4 warps per CTA
constexpr int kWarpsPerBlock = kBlockThreads / kWarp;

// splitmix64 finalizer: engine.cpp:9-14 (bit-identical on host and device).
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}
__host__ __device__ __forceinline__ double to_unit(uint64_t h) {
    return (double)(h >> 11) * 0x1.0p-53;
}

// Engine error carried to the C ABI boundary.
struct Error : std::runtime_error {
    gg_status status;
    uint64_t iteration = 0;
    uint32_t vertex = 0;
    Error(gg_status s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess) {
        char buf[512];
        std::snprintf(buf, sizeof(buf), "%s: %s (%s:%d)", what, cudaGetErrorString(e), file,
                      line);
        throw Error(e == cudaErrorMemoryAllocation ? GG_OOM : GG_CUDA, buf);
    }
}
#define GGB_CUDA(x) ::ggb::cuda_check((x), #x, __FILE__, __LINE__)

inline void fill_error(gg_error* err, const Error& e) {
    if (!err) return;
    err->iteration = e.iteration;
    err->vertex = e.vertex;
    std::strncpy(err->msg, e.what(), sizeof(err->msg) - 1);
    err->msg[sizeof(err->msg) - 1] = 0;
}

// Every extern "C" entry wraps its body with this: exceptions never cross
// the C boundary.
template <class F>
gg_status guarded(gg_error* err, F&& f) {
    try {
        f();
        if (err) err->msg[0] = 0;
        return GG_OK;
    } catch (const Error& e) {
        fill_error(err, e);
        return e.status;
    } catch (const std::bad_alloc&) {
        if (err) std::strncpy(err->msg, "host out of memory", sizeof(err->msg) - 1);
        return GG_OOM;
    } catch (const std::exception& e) {
        if (err) {
            std::strncpy(err->msg, e.what(), sizeof(err->msg) - 1);
            err->msg[sizeof(err->msg) - 1] = 0;
        }
        return GG_INTERNAL;
    }
}

// -------------------------------------------------------------------------
// Device-side warp helpers
// -------------------------------------------------------------------------
template <class T>
__device__ __forceinline__ T shfl_up_any(T v, int d) {
    static_assert(sizeof(T) % 4 == 0, "32-bit granular types only");
    T out;
    const int* src = reinterpret_cast<const int*>(&v);
    int* dst = reinterpret_cast<int*>(&out);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / 4); ++i) dst[i] = __shfl_up_sync(0xffffffffu, src[i], d);
    return out;
}
template <class T>
__device__ __forceinline__ T shfl_idx_any(T v, int lane) {
    static_assert(sizeof(T) % 4 == 0, "32-bit granular types only");
    T out;
    const int* src = reinterpret_cast<const int*>(&v);
    int* dst = reinterpret_cast<int*>(&out);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / 4); ++i) dst[i] = __shfl_sync(0xffffffffu, src[i], lane);
    return out;
}

// Inter-warp hand-over within one kernel (the superstep carry chain): a value
// is written with plain stores, then published by a release store of its
// state word; readers acquire the state and read the value from L2.
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
template <class T>
__device__ __forceinline__ T ld_l2(const T* p) {
    T out;
    if constexpr (sizeof(T) % 8 == 0) {
        const unsigned long long* s = reinterpret_cast<const unsigned long long*>(p);
        unsigned long long* d = reinterpret_cast<unsigned long long*>(&out);
#pragma unroll
        for (int i = 0; i < (int)(sizeof(T) / 8); ++i) d[i] = __ldcg(s + i);
    } else {
        static_assert(sizeof(T) % 4 == 0, "32-bit granular types only");
        const unsigned int* s = reinterpret_cast<const unsigned int*>(p);
        unsigned int* d = reinterpret_cast<unsigned int*>(&out);
#pragma unroll
        for (int i = 0; i < (int)(sizeof(T) / 4); ++i) d[i] = __ldcg(s + i);
    }
    return out;
}

// L2 eviction policies (createpolicy) for the two access streams of the
// gather: edge arrays are read once per iteration (evict_first), the
// per-vertex message array is re-read randomly (evict_last).
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// Streaming (read-once) 32-bit load: bypass L1, evict-first in L2.
__device__ __forceinline__ uint32_t ld_stream_u32(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
// Random message loads, kept in L2.
__device__ __forceinline__ uint32_t ld_keep(const uint32_t* p, uint64_t pol) {
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint2 ld_keep(const uint2* p, uint64_t pol) {
    uint2 v;
    asm("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                 : "=r"(v.x), "=r"(v.y) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint4 ld_keep(const uint4* p, uint64_t pol) {
    uint4 v;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
    return v;
}
// Load a trivially-copyable message of 4/8/16/32 bytes with the keep policy.
template <class M>
__device__ __forceinline__ M ld_msg(const M* p, uint64_t pol) {
    M out;
    if constexpr (sizeof(M) == 4) {
        uint32_t v = ld_keep(reinterpret_cast<const uint32_t*>(p), pol);
        memcpy(&out, &v, 4);
    } else if constexpr (sizeof(M) == 8) {
        uint2 v = ld_keep(reinterpret_cast<const uint2*>(p), pol);
        memcpy(&out, &v, 8);
    } else if constexpr (sizeof(M) % 16 == 0) {
        uint4 v[sizeof(M) / 16];
#pragma unroll
        for (int i = 0; i < (int)(sizeof(M) / 16); ++i)
            v[i] = ld_keep(reinterpret_cast<const uint4*>(p) + i, pol);
        memcpy(&out, v, sizeof(M));
    } else {
        out = *p;
    }
    return out;
}

// Message gather with a per-lane choice of two fixed L2 policies: two
// predicated loads whose policy operands stay warp-uniform (a per-lane
// SELect of the policy costs a select + R2UR pair per gather).
#ifndef GGB_COLD_L1
#define GGB_COLD_L1 ".L1::no_allocate"  // measured: +1% on the c5 approximate gather
#endif
__device__ __forceinline__ uint32_t ld_keep2(const uint32_t* p, bool hot, uint64_t ph, uint64_t pc) {
    uint32_t v;
    asm("{ .reg .pred q; setp.ne.u32 q, %2, 0;\n"
        " @q ld.global.nc.L1::evict_last.L2::cache_hint.u32 %0, [%1], %3;\n"
        " @!q ld.global.nc" GGB_COLD_L1 ".L2::cache_hint.u32 %0, [%1], %4; }"
        : "=r"(v) : "l"(p), "r"((uint32_t)hot), "l"(ph), "l"(pc));
    return v;
}
__device__ __forceinline__ uint2 ld_keep2(const uint2* p, bool hot, uint64_t ph, uint64_t pc) {
    uint2 v;
    asm("{ .reg .pred q; setp.ne.u32 q, %3, 0;\n"
        " @q ld.global.nc.L1::evict_last.L2::cache_hint.v2.u32 {%0, %1}, [%2], %4;\n"
        " @!q ld.global.nc" GGB_COLD_L1 ".L2::cache_hint.v2.u32 {%0, %1}, [%2], %5; }"
        : "=r"(v.x), "=r"(v.y) : "l"(p), "r"((uint32_t)hot), "l"(ph), "l"(pc));
    return v;
}
__device__ __forceinline__ uint4 ld_keep2(const uint4* p, bool hot, uint64_t ph, uint64_t pc) {
    uint4 v;
    asm("{ .reg .pred q; setp.ne.u32 q, %5, 0;\n"
        " @q ld.global.nc.L1::evict_last.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %6;\n"
        " @!q ld.global.nc" GGB_COLD_L1 ".L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %7; }"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p), "r"((uint32_t)hot), "l"(ph), "l"(pc));
    return v;
}
// Three-way message gather: class 0 from a shared-memory copy of the hot
// slots (saddr), 1 = global with L1+L2 evict_last, 2 = global with policy pc.
#define GGB_LDS3(VEC, OUTS, SADDR, GADDR, CLS, PH, PC)                                   \
    "{ .reg .pred q0, q1, q2;\n"                                                          \
    " setp.eq.u32 q0, " CLS ", 0; setp.eq.u32 q1, " CLS ", 1; setp.eq.u32 q2, " CLS ", 2;\n" \
    " @q0 ld.shared" VEC " " OUTS ", [" SADDR "];\n"                                      \
    " @q1 ld.global.nc.L1::evict_last.L2::cache_hint" VEC " " OUTS ", [" GADDR "], " PH ";\n" \
    " @q2 ld.global.nc.L2::cache_hint" VEC " " OUTS ", [" GADDR "], " PC "; }"
__device__ __forceinline__ uint32_t ld_hot3(const uint32_t* p, uint32_t sa, uint32_t cls, uint64_t ph,
                                            uint64_t pc) {
    uint32_t v;
    asm(GGB_LDS3(".u32", "%0", "%1", "%2", "%3", "%4", "%5")
        : "=r"(v) : "r"(sa), "l"(p), "r"(cls), "l"(ph), "l"(pc));
    return v;
}
__device__ __forceinline__ uint2 ld_hot3(const uint2* p, uint32_t sa, uint32_t cls, uint64_t ph,
                                         uint64_t pc) {
    uint2 v;
    asm(GGB_LDS3(".v2.u32", "{%0, %1}", "%2", "%3", "%4", "%5", "%6")
        : "=r"(v.x), "=r"(v.y) : "r"(sa), "l"(p), "r"(cls), "l"(ph), "l"(pc));
    return v;
}
__device__ __forceinline__ uint4 ld_hot3(const uint4* p, uint32_t sa, uint32_t cls, uint64_t ph,
                                         uint64_t pc) {
    uint4 v;
    asm(GGB_LDS3(".v4.u32", "{%0, %1, %2, %3}", "%4", "%5", "%6", "%7", "%8")
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(sa), "l"(p), "r"(cls), "l"(ph), "l"(pc));
    return v;
}
#undef GGB_LDS3
template <class M>
__device__ __forceinline__ M ld_msg_hot(const M* p, uint32_t sa, uint32_t cls, uint64_t ph, uint64_t pc) {
    M out;
    if constexpr (sizeof(M) == 4) {
        uint32_t v = ld_hot3(reinterpret_cast<const uint32_t*>(p), sa, cls, ph, pc);
        memcpy(&out, &v, 4);
    } else if constexpr (sizeof(M) == 8) {
        uint2 v = ld_hot3(reinterpret_cast<const uint2*>(p), sa, cls, ph, pc);
        memcpy(&out, &v, 8);
    } else {
        static_assert(sizeof(M) % 16 == 0, "message size");
        uint4 v[sizeof(M) / 16];
#pragma unroll
        for (int i = 0; i < (int)(sizeof(M) / 16); ++i)
            v[i] = ld_hot3(reinterpret_cast<const uint4*>(p) + i, sa + 16 * i, cls, ph, pc);
        memcpy(&out, v, sizeof(M));
    }
    return out;
}

template <class M>
__device__ __forceinline__ M ld_msg2(const M* p, bool hot, uint64_t ph, uint64_t pc) {
    M out;
    if constexpr (sizeof(M) == 4) {
        uint32_t v = ld_keep2(reinterpret_cast<const uint32_t*>(p), hot, ph, pc);
        memcpy(&out, &v, 4);
    } else if constexpr (sizeof(M) == 8) {
        uint2 v = ld_keep2(reinterpret_cast<const uint2*>(p), hot, ph, pc);
        memcpy(&out, &v, 8);
    } else if constexpr (sizeof(M) % 16 == 0) {
        uint4 v[sizeof(M) / 16];
#pragma unroll
        for (int i = 0; i < (int)(sizeof(M) / 16); ++i)
            v[i] = ld_keep2(reinterpret_cast<const uint4*>(p) + i, hot, ph, pc);
        memcpy(&out, v, sizeof(M));
    } else {
        out = *p;
    }
    return out;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t pol;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}

template <class W>
constexpr int weight_bytes() { return sizeof(W); }
template <>
constexpr int weight_bytes<void>() { return 0; }

}  // namespace ggb
