// build.cu — flag-set maintenance and list layout: sparsify, bitmap ->
// sparsified CSC compaction, the run -> vertex map of a list, and the
// deferred superstep validity scan.
//
// The reference keeps one flag BYTE per edge and re-tests it inside every
// approximate iteration (engine.hpp:203). Here the flags are a bitmap that
// is touched only when it changes (initial sparsify, each superstep); the
// approximate iterations then stream a compacted CSC holding exactly the
// flagged edges in their original order, so the fold order per vertex is
// unchanged and no flag is read on the hot path.
#include <cub/cub.cuh>

#include "exchange.cuh"
#include <cmath>
#include <cstdlib>
#include <vector>
#include <type_traits>

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
// engine.cpp:63-75: flag(e) = (mix64(key ^ e) >> 11) * 2^-53 < sigma.
// The product is exact (a 53-bit integer times a power of two), so the test
// is the integer compare (mix64(key ^ e) >> 11) < ceil(sigma * 2^53) = thr,
// i.e. mix64(key ^ e) < T = thr << 11 (thr < 2^53; sigma = 1 keeps all).
// One thread per bitmap word (32 independent hashes in flight). The test
// needs only the high word of the final mix: h_hi = x_hi ^ (x_hi >> 31) of
// the last product x, whose high word is three 32-bit multiplies; the low
// word is computed only when h_hi ties T's high word.
// High word of mix64's last product for x (the part the test needs).
__device__ __forceinline__ uint32_t mix_hi(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    const uint64_t y = x ^ (x >> 27);
    const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
    constexpr uint32_t c_lo = 0x133111ebu, c_hi = 0x94d049bbu;  // 0x94d049bb133111eb
    const uint32_t xhi = __umulhi(ylo, c_lo) + ylo * c_hi + yhi * c_lo;
    return xhi ^ (xhi >> 31);
}
constexpr uint64_t kMixC1 = 0xbf58476d1ce4e5b9ull;
// mix_hi from mix64's first product P on: high word of the final mix.
__device__ __forceinline__ uint32_t mix_hi_tail(uint64_t P) {
    const uint64_t y = P ^ (P >> 27);
    const uint32_t ylo = (uint32_t)y, yhi = (uint32_t)(y >> 32);
    constexpr uint32_t c_lo = 0x133111ebu, c_hi = 0x94d049bbu;  // 0x94d049bb133111eb
    const uint32_t xhi = __umulhi(ylo, c_lo) + ylo * c_hi + yhi * c_lo;
    return xhi ^ (xhi >> 31);
}
// Bit i of the result = bit (i ^ k) of w, k < 32 (five conditional swaps of
// adjacent 2^j-bit groups).
__device__ __forceinline__ uint32_t xor_permute_bits(uint32_t w, uint32_t k) {
    if (k & 1u) w = ((w & 0x55555555u) << 1) | ((w >> 1) & 0x55555555u);
    if (k & 2u) w = ((w & 0x33333333u) << 2) | ((w >> 2) & 0x33333333u);
    if (k & 4u) w = ((w & 0x0f0f0f0fu) << 4) | ((w >> 4) & 0x0f0f0f0fu);
    if (k & 8u) w = ((w & 0x00ff00ffu) << 8) | ((w >> 8) & 0x00ff00ffu);
    if (k & 16u) w = (w << 16) | (w >> 16);
    return w;
}
__device__ __forceinline__ bool keep_edge(uint64_t x, uint64_t T) {
    const uint32_t hhi = mix_hi(x), Thi = (uint32_t)(T >> 32);
    if (hhi != Thi) return hhi < Thi;
    return mix64(x) < T;  // tie on the high word (rare)
}

// Flags of bitmap word i (engine.cpp:63-75); e_base = global id of local edge 0.
// The aligned full-word path decides all 32 edges on the high words without
// branches and resolves high-word ties (probability ~2^-32 each) afterwards.
__device__ __forceinline__ uint32_t sparsify_word(uint64_t i, uint64_t e_loc, uint64_t e_base,
                                                  uint64_t T, uint64_t key, int keep_all) {
    const uint64_t e0 = i * 32;
    const int nb = e_loc - e0 < 32 ? (int)(e_loc - e0) : 32;
    uint32_t word = 0;
    if (keep_all) {
        word = nb == 32 ? 0xffffffffu : ((1u << nb) - 1u);
    } else if (nb == 32 && (e_base & 31) == 0) {
        // The 32 hashed values k0 ^ b are the aligned block U0 + c, c = kc ^ b
        // (kc = k0 & 31). After mix64's first step they are A0 + 21 + c
        // (A0 = U0 + (golden & ~31), 32-aligned): c <= 10 falls in block A0
        // at offset r = c + 21, c >= 11 in block A0 + 32 at r = c - 11. Inside
        // a block A the shifted term S = (A | r) >> 30 = A >> 30 is constant,
        // so x ^ (x >> 30) = ((A ^ S) & ~31) + (r ^ (S & 31)) and the first
        // product is P0 + (r ^ m) * C1 with P0 = ((A ^ S) & ~31) * C1, m =
        // S & 31: two multiply-adds per edge instead of the add, the
        // xor-shift and the 64-bit product (all mod 2^64, so block A0 + 32
        // wrapping or crossing a 2^30 boundary needs no special case).
        // Flags are collected at bit c and moved to bit b = c ^ kc at the end.
        const uint64_t k0 = key ^ (e_base + e0);
        const uint32_t kc = (uint32_t)k0 & 31u;
        const uint64_t A0 = (k0 & ~31ull) + (0x9e3779b97f4a7c15ull & ~31ull);
        const uint64_t Qa = A0 ^ (A0 >> 30), A1 = A0 + 32, Qb = A1 ^ (A1 >> 30);
        const uint64_t Pa = (Qa & ~31ull) * kMixC1, Pb = (Qb & ~31ull) * kMixC1;
        const uint32_t ma = (uint32_t)Qa & 31u, mb = (uint32_t)Qb & 31u;
        const uint32_t Thi = (uint32_t)(T >> 32);
        uint32_t wp = 0, tp = 0;
        auto hash_c = [&](int c) {  // c is a compile-time constant after unrolling
            const uint32_t rp = (uint32_t)((c + 21) & 31) ^ (c >= 11 ? mb : ma);
            return mix_hi_tail((c >= 11 ? Pb : Pa) + (uint64_t)rp * kMixC1);
        };
        // T's low word 0 (sigma a multiple of 2^-32, e.g. 0.5): a high-word tie
        // means h >= T, so the high-word test alone decides
        const bool ties = (uint32_t)T != 0;
        if (!ties) {
#pragma unroll
            for (int c = 0; c < 32; ++c) wp |= (hash_c(c) < Thi ? 1u : 0u) << c;
        } else {
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                const uint32_t h = hash_c(c);
                wp |= (h < Thi ? 1u : 0u) << c;
                tp |= (h == Thi ? 1u : 0u) << c;
            }
        }
        word = xor_permute_bits(wp, kc);
        uint32_t tie = ties ? xor_permute_bits(tp, kc) : 0u;
        while (tie) {  // probability ~2^-32 per edge
            const int b = __ffs(tie) - 1;
            tie &= tie - 1;
            if (mix64(k0 ^ (uint64_t)b) < T) word |= 1u << b;
        }
    } else {
        for (int b = 0; b < nb; ++b) word |= (keep_edge(key ^ (e_base + e0 + b), T) ? 1u : 0u) << b;
    }
    return word;
}

__global__ void sparsify_kernel(uint32_t* __restrict__ bitmap, uint64_t nwords, uint64_t e_loc,
                                uint64_t e_base, uint64_t T, uint64_t key, int keep_all) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i <= nwords;
         i += (uint64_t)gridDim.x * blockDim.x)
        bitmap[i] = i < nwords ? sparsify_word(i, e_loc, e_base, T, key, keep_all) : 0u;  // [nwords]: zero guard word
}

SparsifySpec sparsify_spec(double sigma, uint64_t seed, bool all_ones) {
    const uint64_t thr = all_ones ? (1ull << 53) : (uint64_t)std::ceil(sigma * 0x1.0p53);
    SparsifySpec h;
    h.keep_all = thr >= (1ull << 53) ? 1 : 0;  // (h >> 11) < 2^53 always
    h.T = h.keep_all ? 0 : thr << 11;
    h.key = mix64(seed);
    return h;
}

void sparsify_bitmap(DevGraph& g, uint32_t* bitmap, double sigma, uint64_t seed, bool all_ones) {
    const uint64_t nwords = (g.e_loc + 31) / 32;
    const SparsifySpec h = sparsify_spec(sigma, seed, all_ones);
    sparsify_kernel<<<grid_for(nwords + 1, 256), 256, 0, g.stream>>>(
        bitmap, nwords, g.e_loc, g.e_base, h.T, h.key, h.keep_all);
    GGB_CUDA(cudaGetLastError());
}

// --------------------------------------------------------------------------
// List layout: the non-empty vertices (nz_vid / nz_start) and the run map
// run_i[r] = max{i : nz_start[i] + pad <= first valid position of run r}
// (= the non-empty vertex containing it): every non-empty vertex marks the
// first run whose first valid position is >= its start, then a max-scan.
// --------------------------------------------------------------------------
__global__ void nonempty_flag_kernel(const uint64_t* __restrict__ off, uint64_t nloc,
                                     uint32_t* __restrict__ flag) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= nloc;
         v += (uint64_t)gridDim.x * blockDim.x)
        flag[v] = v < nloc && off[v + 1] > off[v] ? 1u : 0u;
}

__global__ void nonempty_fill_kernel(const uint64_t* __restrict__ off, uint64_t nloc, uint64_t pad,
                                     const uint32_t* __restrict__ idx, uint64_t nruns,
                                     uint32_t* __restrict__ nz_vid, uint64_t* __restrict__ nz_start,
                                     uint32_t* __restrict__ marks) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v <= nloc;
         v += (uint64_t)gridDim.x * blockDim.x) {
        if (v == nloc) {
            nz_start[idx[nloc]] = off[nloc];  // sentinel: end of the last vertex
            marks[nruns] = idx[nloc] ? idx[nloc] - 1 : 0u;  // copied to run_i[nruns] below
            continue;
        }
        if (off[v + 1] <= off[v]) continue;
        const uint32_t i = idx[v];
        nz_vid[i] = (uint32_t)v;
        nz_start[i] = off[v];
        const uint64_t s = off[v] + pad;
        const uint64_t r = s <= pad ? 0 : (s + kRun - 1) / kRun;
        if (r < nruns) atomicMax(marks + r, i);
    }
}

struct MaxU32 {
    __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

void build_runs(DevGraph& g, const uint64_t* off, uint64_t pad, uint64_t e, const std::string& tag,
                ListMeta& meta) {
    meta.pad = pad;
    meta.e = e;
    meta.ntasks = (pad + e + kChunkEdges - 1) / kChunkEdges;
    if (e == 0) meta.ntasks = 0;
    meta.nruns = meta.ntasks * kWarp;
    uint32_t* flag = g.ws.get<uint32_t>(tag + ".nzflag", g.nloc + 1);
    uint32_t* idx = g.ws.get<uint32_t>(tag + ".nzidx", g.nloc + 1);
    uint32_t* marks = g.ws.get<uint32_t>(tag + ".runmark", meta.nruns + 1);
    meta.run_i = g.ws.get<uint32_t>(tag + ".run_i", meta.nruns + 1);
    nonempty_flag_kernel<<<grid_for(g.nloc + 1, 256), 256, 0, g.stream>>>(off, g.nloc, flag);
    GGB_CUDA(cudaGetLastError());
    size_t tmp = 0, tmp2 = 0;
    GGB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp, flag, idx, g.nloc + 1, g.stream));
    GGB_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tmp2, marks, meta.run_i, MaxU32{},
                                            meta.nruns ? meta.nruns : 1, g.stream));
    void* tmpp = g.ws.get("cub.tmp." + tag, std::max(tmp, tmp2));
    GGB_CUDA(cub::DeviceScan::ExclusiveSum(tmpp, tmp, flag, idx, g.nloc + 1, g.stream));
    uint32_t nz = 0;
    GGB_CUDA(cudaMemcpyAsync(&nz, idx + g.nloc, 4, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    meta.nz = nz;
    meta.nz_vid = g.ws.get<uint32_t>(tag + ".nz_vid", (uint64_t)nz + 1);
    meta.nz_start = g.ws.get<uint64_t>(tag + ".nz_start", (uint64_t)nz + 1);
    if (meta.nruns) GGB_CUDA(cudaMemsetAsync(marks, 0, meta.nruns * 4, g.stream));
    nonempty_fill_kernel<<<grid_for(g.nloc + 1, 256), 256, 0, g.stream>>>(
        off, g.nloc, pad, idx, meta.nruns, meta.nz_vid, meta.nz_start, marks);
    GGB_CUDA(cudaGetLastError());
    if (!meta.nruns) return;
    GGB_CUDA(cub::DeviceScan::InclusiveScan(tmpp, tmp2, marks, meta.run_i, MaxU32{}, meta.nruns,
                                            g.stream));
    GGB_CUDA(cudaMemcpyAsync(meta.run_i + meta.nruns, marks + meta.nruns, 4, cudaMemcpyDeviceToDevice,
                             g.stream));  // sentinel run_i[nruns] = nz - 1
}

// Position order of the local vertices (graph.cuh): rows (non-empty, in
// vertex order) at [0, R), in-degree-0 vertices at [R, nloc).
__global__ void positions_kernel(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ idx,
                                 uint64_t nloc, uint64_t nrows, uint64_t v_begin,
                                 const uint32_t* __restrict__ slot_of,
                                 const uint32_t* __restrict__ outdeg, uint32_t* __restrict__ vid_of_p,
                                 uint32_t* __restrict__ slot_p, uint32_t* __restrict__ deg_p) {
    for (uint64_t lv = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; lv < nloc;
         lv += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t p = flag[lv] ? idx[lv] : nrows + (lv - idx[lv]);
        vid_of_p[p] = (uint32_t)lv;
        slot_p[p] = slot_of[v_begin + lv];
        deg_p[p] = outdeg[v_begin + lv];
    }
}

void build_full(DevGraph& g) {
    build_runs(g, g.off, g.full.pad, g.e_loc, "full", g.full);
    g.nrows = g.full.nz;
    g.vid_of_p = static_cast<uint32_t*>(dev_alloc((g.nloc + 1) * 4, g.stream));
    g.slot_p = static_cast<uint32_t*>(dev_alloc((g.nloc + 1) * 4, g.stream));
    g.deg_p = static_cast<uint32_t*>(dev_alloc((g.nloc + 1) * 4, g.stream));
    if (!g.nloc) return;
    positions_kernel<<<grid_for(g.nloc, 256), 256, 0, g.stream>>>(
        g.ws.get<uint32_t>("full.nzflag", g.nloc + 1), g.ws.get<uint32_t>("full.nzidx", g.nloc + 1),
        g.nloc, g.nrows, g.v_begin, g.slot_of, g.outdeg, g.vid_of_p, g.slot_p, g.deg_p);
    GGB_CUDA(cudaGetLastError());
}

// --------------------------------------------------------------------------
// bitmap -> sparsified CSC
// --------------------------------------------------------------------------

__device__ __forceinline__ uint64_t bit_rank(const uint32_t* bitmap, const uint64_t* wpref,
                                             uint64_t e) {
    const uint64_t w = e >> 5;
    const uint32_t b = (uint32_t)(e & 31);
    return wpref[w] + (uint64_t)__popc(bitmap[w] & ((1u << b) - 1u));
}

// Stream compaction of the kept edges (sources, weights) into the padded
// sparsified list. A warp takes 8 bitmap words (256 edges) per step: lane l
// owns bit l of each word; all loads of the step are issued before any store,
// so one memory latency covers 256 edges.
template <int WB>
__global__ void compact_kernel(const uint32_t* __restrict__ src, const void* __restrict__ w,
                               uint64_t e_loc, uint64_t in_pad, const uint32_t* __restrict__ bitmap,
                               const uint64_t* __restrict__ wpref, uint32_t* __restrict__ s_src,
                               void* __restrict__ s_w, uint64_t out_pad, bool quads) {
    using WT = std::conditional_t<WB == 8, unsigned long long, uint32_t>;
    constexpr int kW = 8;
    const int lane = threadIdx.x & 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint64_t nw = (e_loc + 31) / 32;
    const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t w0 = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * kW; w0 < nw;
         w0 += warps * kW) {
        uint32_t word[kW], sv[kW];
        uint64_t base[kW];
        WT wv[kW];
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            const bool in = w0 + k < nw;
            word[k] = in ? __ldg(bitmap + w0 + k) : 0u;
            base[k] = in ? __ldg(wpref + w0 + k) : 0ull;
            const uint64_t e = (w0 + k) * 32 + lane;
            const bool ine = e < e_loc;
            sv[k] = ine ? __ldg(src + in_pad + e) : 0u;
            if constexpr (WB != 0) wv[k] = ine ? __ldg(static_cast<const WT*>(w) + in_pad + e) : WT(0);
        }
#pragma unroll
        for (int k = 0; k < kW; ++k) {
            if ((word[k] >> lane) & 1u) {
                const uint64_t pos = out_pad + base[k] + (uint64_t)__popc(word[k] & lt);
                s_src[quads ? sp_slot(pos) : pos] = sv[k];
                if constexpr (WB != 0) static_cast<WT*>(s_w)[pos] = wv[k];
            }
        }
    }
}

// Single-pass flags -> prefix -> compaction (one rank). A CTA takes a tile of
// kScanTile bitmap words (tiles claimed in order from a ticket; warp w owns
// the tile's words [128w, 128w + 128), lane l words 32j + l), computes the
// words (HASH: the sparsify hash; otherwise read from the bitmap), scans their
// popcounts, gets the tile's exclusive prefix by a decoupled look-back over
// the earlier tiles' {flag, value} words (one 64-bit relaxed store each: no
// fence), writes the per-word prefix `wpref` (for the list layout) and compacts
// the tile's kept sources / weights. Replaces sparsify + popc + scan +
// compact (four passes; the sources are read once).
constexpr int kScanThreads = 256, kScanWPL = 4;             // words per lane
constexpr int kScanTile = kScanThreads * kScanWPL;          // words per tile
constexpr int kScanWarpWords = 32 * kScanWPL;
constexpr uint64_t kScanAgg = 1ull << 62, kScanIncl = 2ull << 62, kScanVal = (1ull << 62) - 1;

__device__ __forceinline__ void st_relaxed_u64(unsigned long long* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const unsigned long long* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// Decoupled look-back of tile t (one warp): publishes the tile's aggregate,
// walks back over earlier tiles (lane i reads tile j - i; the nearest
// inclusive value ends the walk, tiles before 0 count as inclusive 0),
// publishes the inclusive prefix and returns the exclusive one.
__device__ __forceinline__ uint64_t tile_lookback(unsigned long long* tstate, uint64_t t,
                                                  uint64_t agg, int lane) {
    if (lane == 0) st_relaxed_u64(tstate + t, (t == 0 ? kScanIncl : kScanAgg) | agg);
    uint64_t excl = 0;
    for (int64_t j = (int64_t)t - 1; j >= 0; j -= 32) {
        const int64_t q = j - lane;
        uint64_t st;
        do {
            st = q >= 0 ? ld_relaxed_u64(tstate + q) : kScanIncl;
        } while (__any_sync(0xffffffffu, (st >> 62) == 0));
        const uint32_t im = __ballot_sync(0xffffffffu, (st >> 62) == 2);
        uint64_t v = st & kScanVal;
        if (im) v = lane <= __ffs(im) - 1 ? v : 0ull;
#pragma unroll
        for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        excl += v;
        if (im) break;
    }
    if (t && lane == 0) st_relaxed_u64(tstate + t, kScanIncl | (excl + agg));
    return excl;
}

// Held to 4 / 4 / 3 CTAs per SM (weight bytes 0 / 4 / 8). WB = -1: scan
// only (flags + per-word prefix + kept total, no compaction) -- several
// ranks need every rank's kept count before the list's padded base is known.
template <int WB, bool HASH>
__global__ void __launch_bounds__(kScanThreads, WB <= 0 ? 4 : WB == 4 ? 4 : 3)
scan_compact_kernel(const uint32_t* __restrict__ src, const void* __restrict__ w, uint64_t e_loc,
                    uint64_t in_pad, uint32_t* __restrict__ bitmap, uint64_t nwords, uint64_t e_base,
                    SparsifySpec h, uint64_t* __restrict__ wpref, uint32_t* __restrict__ s_src,
                    void* __restrict__ s_w, unsigned long long* __restrict__ tstate,
                    uint32_t* __restrict__ ticket, uint64_t tile_base, uint64_t ntiles,
                    bool quads) {
    using WT = std::conditional_t<WB == 8, unsigned long long, uint32_t>;
    constexpr int kWarps = kScanThreads / 32;
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wsum[kWarps];
    __shared__ uint64_t s_wbase[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lt = (1u << lane) - 1u;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t t = tile_base + s_tile;  // tiles [tile_base, ntiles) of this launch
        if (t >= ntiles) break;
        const uint64_t w0 = t * kScanTile + (uint64_t)warp * kScanWarpWords;
        // sources of 8 words (lane l: edge l of each), loaded one batch ahead;
        // the first batch before the flags and the look-back
        // batches in registers: unweighted lists keep three batches in
        // flight ahead of the one being stored (64 registers, 4 CTAs per SM:
        // c5 compaction 2.35 -> 2.18 ms, sparsify + compaction 4.63 -> 4.40
        // ms; one ahead at 6 CTAs, two at 5 and 6, four at 4 and five at 3
        // measured slower)
        constexpr bool kCompact = WB >= 0;
        constexpr int D = WB <= 0 ? 4 : 2;
        uint32_t sv[D][8];
        WT wv[D][8];
        auto load_batch = [&](int k0, uint32_t (&s8)[8], WT (&w8)[8]) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint64_t e = (w0 + k0 + k) * 32 + lane;
                const bool ine = e < e_loc;
                s8[k] = ine ? __ldg(src + in_pad + e) : 0u;
                if constexpr (WB > 0) w8[k] = ine ? __ldg(static_cast<const WT*>(w) + in_pad + e) : WT(0);
            }
        };
        if constexpr (kCompact) {
#pragma unroll
            for (int b = 0; b < D - 1; ++b) load_batch(8 * b, sv[b], wv[b]);
        }
        uint32_t word[kScanWPL], off[kScanWPL];  // off: exclusive popcount within the warp
        uint32_t run = 0;
        if constexpr (HASH) {
            // one copy of the 32 unrolled hashes (rolled over the lane's words:
            // four inlined copies overflow the instruction cache)
#pragma unroll 1
            for (int j = 0; j < kScanWPL; ++j) {
                const uint64_t wi = w0 + 32 * j + lane;
                uint32_t x = 0;
                if (wi < nwords) x = sparsify_word(wi, e_loc, e_base, h.T, h.key, h.keep_all);
                if (wi <= nwords) bitmap[wi] = x;  // [nwords]: zero guard word
#pragma unroll
                for (int q = 0; q < kScanWPL; ++q) word[q] = q == j ? x : word[q];
            }
        }
#pragma unroll
        for (int j = 0; j < kScanWPL; ++j) {
            const uint64_t wi = w0 + 32 * j + lane;
            uint32_t x = 0;
            if constexpr (HASH) {
                x = word[j];
            } else {
                if (wi < nwords) x = __ldg(bitmap + wi);
            }
            word[j] = x;
            uint32_t incl = __popc(x);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            off[j] = run + incl - __popc(x);
            run += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) s_wsum[warp] = run;
        __syncthreads();
        if (warp == 0) {
            const uint64_t ws = lane < kWarps ? s_wsum[lane] : 0u;
            uint64_t wincl = ws;
#pragma unroll
            for (int o = 1; o < kWarps; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, wincl, o);
                if (lane >= o) wincl += y;
            }
            const uint64_t agg = __shfl_sync(0xffffffffu, wincl, kWarps - 1);
            const uint64_t excl = tile_lookback(tstate, t, agg, lane);
            if (lane < kWarps) s_wbase[lane] = excl + wincl - ws;  // warp's exclusive base
        }
        __syncthreads();
        const uint64_t wbase = s_wbase[warp];
#pragma unroll
        for (int j = 0; j < kScanWPL; ++j) {
            const uint64_t wi = w0 + 32 * j + lane;
            if (wi <= nwords) wpref[wi] = wbase + off[j];  // wpref[nwords] = kept total
        }
#pragma unroll
        for (int b = 0; b < kScanWarpWords / 8; ++b) {
            if (!kCompact || w0 + 8 * b >= nwords) break;
            if (b + D - 1 < kScanWarpWords / 8)
                load_batch(8 * (b + D - 1), sv[(b + D - 1) % D], wv[(b + D - 1) % D]);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int kw = 8 * b + k;  // word of the warp: lane kw % 32 of word[kw / 32]
                const uint32_t wk = __shfl_sync(0xffffffffu, word[kw / 32], kw % 32);
                const uint32_t ok = __shfl_sync(0xffffffffu, off[kw / 32], kw % 32);
                if ((wk >> lane) & 1u) {
                    const uint64_t pos = wbase + ok + (uint32_t)__popc(wk & lt);
                    s_src[quads ? sp_slot(pos) : pos] = sv[b % D][k];
                    if constexpr (WB > 0) static_cast<WT*>(s_w)[pos] = wv[b % D][k];
                }
            }
        }
        __syncthreads();  // s_tile / s_wsum / s_wbase reuse
    }
}

// Tiles [tile_lo, tile_hi) (tile_hi = ~0: through the last tile). Launches
// over consecutive tile ranges continue one scan: the tile states are
// cleared by the launch starting at tile 0, and every earlier tile is
// complete when a later range starts (same stream).
template <bool HASH>
static void launch_scan_compact(DevGraph& g, uint32_t* bitmap, const SparsifySpec& h,
                                uint64_t* wpref, uint32_t* s_src, void* s_w, uint64_t tile_lo = 0,
                                uint64_t tile_hi = ~0ull, bool scan_only = false) {
    const uint64_t nwords = (g.e_loc + 31) / 32;
    const uint64_t ntiles = (nwords + 1 + kScanTile - 1) / kScanTile;
    if (tile_hi > ntiles) tile_hi = ntiles;
    if (tile_lo >= tile_hi) return;
    auto* tstate = g.ws.get<unsigned long long>("rb.tstate", ntiles + 1);
    auto* ticket = reinterpret_cast<uint32_t*>(tstate + ntiles);
    if (tile_lo == 0) GGB_CUDA(cudaMemsetAsync(tstate, 0, (ntiles + 1) * 8, g.stream));
    else GGB_CUDA(cudaMemsetAsync(ticket, 0, 4, g.stream));
    // programs that ignore the graph's weights (PR, WCC) compact sources only
    const size_t wb = s_w ? weight_size(g.wkind) : 0;
    // resident CTAs per SM of each instantiation (thread-safe one-time init)
    auto per_sm = [](const void* k) { return occupancy_grid(k, kScanThreads, 0, 1); };
    static const int ps0 = per_sm((const void*)scan_compact_kernel<0, HASH>);
    static const int ps4 = per_sm((const void*)scan_compact_kernel<4, HASH>);
    static const int ps8 = per_sm((const void*)scan_compact_kernel<8, HASH>);
    static const int psn = per_sm((const void*)scan_compact_kernel<-1, HASH>);
    const int ps = scan_only ? psn : wb == 0 ? ps0 : wb == 4 ? ps4 : ps8;
    const uint64_t gr = std::min<uint64_t>(tile_hi - tile_lo, (uint64_t)ps * g.num_sms);
    if (scan_only)
        scan_compact_kernel<-1, HASH><<<gr, kScanThreads, 0, g.stream>>>(
            g.src, g.w, g.e_loc, g.full.pad, bitmap, nwords, g.e_base, h, wpref, s_src, s_w, tstate,
            ticket, tile_lo, tile_hi, sp_quads(g));
    else if (wb == 0)
        scan_compact_kernel<0, HASH><<<gr, kScanThreads, 0, g.stream>>>(
            g.src, g.w, g.e_loc, g.full.pad, bitmap, nwords, g.e_base, h, wpref, s_src, s_w, tstate,
            ticket, tile_lo, tile_hi, sp_quads(g));
    else if (wb == 4)
        scan_compact_kernel<4, HASH><<<gr, kScanThreads, 0, g.stream>>>(
            g.src, g.w, g.e_loc, g.full.pad, bitmap, nwords, g.e_base, h, wpref, s_src, s_w, tstate,
            ticket, tile_lo, tile_hi, sp_quads(g));
    else
        scan_compact_kernel<8, HASH><<<gr, kScanThreads, 0, g.stream>>>(
            g.src, g.w, g.e_loc, g.full.pad, bitmap, nwords, g.e_base, h, wpref, s_src, s_w, tstate,
            ticket, tile_lo, tile_hi, sp_quads(g));
    GGB_CUDA(cudaGetLastError());
}

// Sparsified-list layout in one pass over the owned vertices (replaces
// soff + nonempty flag / scan / fill of build_runs and the run-map max-scan):
// s_off[v] = rank of off[v] among the kept edges; the non-empty vertices get
// consecutive nz indices (decoupled look-back over tiles of kLayoutTile
// vertices; warp w owns the tile's vertices [128w, 128w + 128), lane l
// vertices 32j + l) with nz_vid / nz_start, and every run r whose first
// padded position lies in non-empty vertex i's positions [s, e) gets
// run_i[r] = i, i.e. runs [ceil(s/16), ceil(e/16)) (the first non-empty
// vertex also takes the runs before it); a vertex of more than 32 runs is
// written by its whole warp. The thread holding v = nloc writes the
// sentinels nz_start[nz] and run_i[r] = nz - 1 for the runs after the last
// kept edge, run_i[nruns] included.
constexpr int kLayoutVPT = 8;  // vertices per thread (c5: 8 -> 0.75 ms, 4 -> 0.89, 2 -> 1.20, 16 -> 0.75)
constexpr int kLayoutTile = 256 * kLayoutVPT;

__global__ void __launch_bounds__(256)
sp_layout_kernel(const uint64_t* __restrict__ off, uint64_t nloc,
                 const uint32_t* __restrict__ bitmap, const uint64_t* __restrict__ wpref,
                 uint64_t pad, uint64_t nruns, uint64_t* __restrict__ s_off,
                 uint32_t* __restrict__ nz_vid, uint64_t* __restrict__ nz_start,
                 uint32_t* __restrict__ run_i,
                 unsigned long long* __restrict__ tstate, uint32_t* __restrict__ ticket,
                 uint64_t ntiles) {
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_wsum[8];
    __shared__ uint64_t s_wbase[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (;;) {
        if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
        __syncthreads();
        const uint64_t t = s_tile;
        if (t >= ntiles) break;
        const uint64_t vb = t * kLayoutTile + (uint64_t)warp * 32 * kLayoutVPT;  // warp's first vertex
        uint64_t so[kLayoutVPT];
#pragma unroll
        for (int j = 0; j < kLayoutVPT; ++j) {
            const uint64_t v = vb + 32 * j + lane;
            so[j] = v <= nloc ? bit_rank(bitmap, wpref, __ldg(off + v)) : 0ull;
        }
        const uint64_t vend = vb + 32 * kLayoutVPT;  // lane 31's last successor
        const uint64_t so_end = (lane == 31 && vend <= nloc) ? bit_rank(bitmap, wpref, __ldg(off + vend)) : 0ull;
        // kept offset of vertex (vb + 32j + lane) + 1
        auto next_of = [&](int j) -> uint64_t {
            uint64_t nx = __shfl_down_sync(0xffffffffu, so[j], 1);
            const uint64_t nx0 = __shfl_sync(0xffffffffu, j + 1 < kLayoutVPT ? so[j + 1 < kLayoutVPT ? j + 1 : j] : so_end, 0);
            if (lane == 31) nx = j + 1 < kLayoutVPT ? nx0 : so_end;
            return nx;
        };
        uint32_t fl = 0, off_in[kLayoutVPT], run = 0;
#pragma unroll
        for (int j = 0; j < kLayoutVPT; ++j) {
            const uint64_t v = vb + 32 * j + lane;
            const uint64_t nx = next_of(j);  // warp-collective: every lane, no short-circuit
            const bool f = v < nloc && nx > so[j];
            fl |= (f ? 1u : 0u) << j;
            const uint32_t b = __ballot_sync(0xffffffffu, f);
            off_in[j] = run + __popc(b & ((1u << lane) - 1u));
            run += __popc(b);
        }
        if (lane == 0) s_wsum[warp] = run;
        __syncthreads();
        if (warp == 0) {
            const uint64_t ws = lane < 8 ? s_wsum[lane] : 0u;
            uint64_t wincl = ws;
#pragma unroll
            for (int o = 1; o < 8; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, wincl, o);
                if (lane >= o) wincl += y;
            }
            const uint64_t agg = __shfl_sync(0xffffffffu, wincl, 7);
            const uint64_t excl = tile_lookback(tstate, t, agg, lane);
            if (lane < 8) s_wbase[lane] = excl + wincl - ws;
        }
        __syncthreads();
        const uint64_t wbase = s_wbase[warp];
        auto run_ceil = [&](uint64_t kept_off) { return (kept_off + pad + kRun - 1) / kRun; };
#pragma unroll
        for (int j = 0; j < kLayoutVPT; ++j) {  // every lane runs every j (warp-wide writes below)
            const uint64_t v = vb + 32 * j + lane;
            const uint64_t nx = next_of(j);
            const uint64_t i = wbase + off_in[j];
            uint64_t r_lo = 0, r_hi = 0;  // runs of this lane's vertex
            uint32_t val = 0;
            if (v <= nloc) s_off[v] = so[j];
            if (v == nloc) {  // sentinels: i = nz
                nz_start[i] = so[j];
                r_lo = i ? run_ceil(so[j]) : 0;
                r_hi = nruns + 1;
                val = i ? (uint32_t)(i - 1) : 0u;
            } else if (v < nloc && ((fl >> j) & 1u)) {
                nz_vid[i] = (uint32_t)v;
                nz_start[i] = so[j];
                r_lo = i ? run_ceil(so[j]) : 0;
                r_hi = run_ceil(nx);
                if (r_hi > nruns) r_hi = nruns;
                val = (uint32_t)i;
            }
            const bool longv = r_hi > r_lo + 32;
            if (!longv)
                for (uint64_t r = r_lo; r < r_hi; ++r) run_i[r] = val;
            uint32_t lb = __ballot_sync(0xffffffffu, longv);
            while (lb) {  // long vertices: the warp writes their runs together
                const int src = __ffs(lb) - 1;
                lb &= lb - 1;
                const uint64_t a0 = __shfl_sync(0xffffffffu, r_lo, src);
                const uint64_t a1 = __shfl_sync(0xffffffffu, r_hi, src);
                const uint32_t x = __shfl_sync(0xffffffffu, val, src);
                for (uint64_t r = a0 + lane; r < a1; r += 32) run_i[r] = x;
            }
        }
        __syncthreads();  // s_tile / s_wsum / s_wbase reuse
    }
}

// Layout of the sparsified list (kept edges at `pad`) in ROW space: s_off[p]
// for the rows p in [0, R] (the in-degree-0 vertices keep nothing), nz_vid =
// the rows with kept edges, run map. Asynchronous (the non-empty count stays
// on the device: the edge kernel reads the run_i[nruns] sentinel instead).
static void build_sparse_layout(DevGraph& g, const uint32_t* bitmap, const uint64_t* wpref,
                                uint64_t* s_off, uint64_t pad, uint64_t kept, ListMeta& meta) {
    meta.pad = pad;
    meta.e = kept;
    meta.ntasks = kept ? (pad + kept + kChunkEdges - 1) / kChunkEdges : 0;
    meta.nruns = meta.ntasks * kWarp;
    meta.nz = 0;  // on the device only
    meta.nz_vid = g.ws.get<uint32_t>("sp.nz_vid", g.nrows + 1);
    meta.nz_start = g.ws.get<uint64_t>("sp.nz_start", g.nrows + 1);
    meta.run_i = g.ws.get<uint32_t>("sp.run_i", meta.nruns + 1);
    const uint64_t ntiles = (g.nrows + 1 + kLayoutTile - 1) / kLayoutTile;
    auto* tstate = g.ws.get<unsigned long long>("sp.tstate", ntiles + 1);
    auto* ticket = reinterpret_cast<uint32_t*>(tstate + ntiles);
    GGB_CUDA(cudaMemsetAsync(tstate, 0, (ntiles + 1) * 8, g.stream));
    static const int per_sm = occupancy_grid((const void*)sp_layout_kernel, 256, 0, 1);
    const uint64_t gr = std::min<uint64_t>(ntiles, (uint64_t)per_sm * g.num_sms);
    sp_layout_kernel<<<gr, 256, 0, g.stream>>>(g.full.nz_start, g.nrows, bitmap, wpref, pad, meta.nruns,
                                               s_off, meta.nz_vid, meta.nz_start, meta.run_i,
                                               tstate, ticket, ntiles);
    GGB_CUDA(cudaGetLastError());
}

// Initial sparsification overlapped with the graph upload
// (gg_dev_graph_create_for_run): the hash + compaction of the edges
// [0, e_hi) once their sources are resident; e_hi is a multiple of the scan
// tile (32768 edges) except for the last call (e_hi = e_loc).
uint64_t presparse_tile_edges() { return (uint64_t)kScanTile * 32; }
void presparse_chunk(DevGraph& g, const SparsifySpec& h, uint64_t e_lo, uint64_t e_hi) {
    const uint64_t nwords = (g.e_loc + 31) / 32;
    uint32_t* bitmap = g.ws.get<uint32_t>("bitmap", nwords + 1);
    uint64_t* wpref = g.ws.get<uint64_t>("rb.wpref", nwords + 1);
    uint32_t* s_src = g.ws.get<uint32_t>("s_src", g.e_loc + 2 * kChunkEdges + kRun);
    const size_t wsz = weight_size(g.wkind);
    void* s_w = wsz ? g.ws.get("s_w", (g.e_loc + kChunkEdges + kRun) * wsz) : nullptr;
    const uint64_t te = presparse_tile_edges();
    const uint64_t tlo = e_lo / te;
    const uint64_t thi = e_hi >= g.e_loc ? ~0ull : e_hi / te;
    launch_scan_compact<true>(g, bitmap, h, wpref, s_src, s_w, tlo, thi);
}
// The run side: the list layout of a pre-sparsified graph; returns kept.
uint64_t presparse_finish(DevGraph& g, uint64_t* s_off, ListMeta& meta) {
    const uint64_t nwords = (g.e_loc + 31) / 32;
    uint32_t* bitmap = g.ws.get<uint32_t>("bitmap", nwords + 1);
    uint64_t* wpref = g.ws.get<uint64_t>("rb.wpref", nwords + 1);
    uint64_t kept = 0;
    GGB_CUDA(cudaMemcpyAsync(&kept, wpref + nwords, 8, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    build_sparse_layout(g, bitmap, wpref, s_off, 0, kept, meta);
    return kept;
}

uint64_t sparse_pad(DevGraph& g, uint64_t kept_local) {
    if (g.nranks <= 1) return 0;
    return exchange_exclusive_base(g, kept_local) % kChunkEdges;
}

uint64_t rebuild_sparse(DevGraph& g, uint32_t* bitmap, uint64_t* s_off, uint32_t* s_src,
                        void* s_w, ListMeta& meta, cudaEvent_t ev0, cudaEvent_t ev1,
                        int* launches, const SparsifySpec* hash) {
    const uint64_t nwords = (g.e_loc + 31) / 32;
    uint64_t* wpref = g.ws.get<uint64_t>("rb.wpref", nwords + 1);
    if (ev0) GGB_CUDA(cudaEventRecord(ev0, g.stream));
    uint64_t kept = 0;
    if (g.nranks == 1) {
        // one pass: (sparsify +) scan + compaction at pad 0
        if (hash) launch_scan_compact<true>(g, bitmap, *hash, wpref, s_src, s_w);
        else launch_scan_compact<false>(g, bitmap, SparsifySpec{}, wpref, s_src, s_w);
        GGB_CUDA(cudaMemcpyAsync(&kept, wpref + nwords, 8, cudaMemcpyDeviceToHost, g.stream));
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        build_sparse_layout(g, bitmap, wpref, s_off, 0, kept, meta);
        if (ev1) GGB_CUDA(cudaEventRecord(ev1, g.stream));
        if (launches) *launches += 2;  // scan_compact, sp_layout
        return kept;
    }
    // several ranks: the list's padded base needs the kept counts of all
    // ranks before compaction: one scan-only pass (flags + word prefix +
    // kept total), the kept counts exchanged, then the compaction
    if (hash) launch_scan_compact<true>(g, bitmap, *hash, wpref, s_src, s_w, 0, ~0ull, true);
    else launch_scan_compact<false>(g, bitmap, SparsifySpec{}, wpref, s_src, s_w, 0, ~0ull, true);
    if (launches) ++*launches;
    GGB_CUDA(cudaMemcpyAsync(&kept, wpref + nwords, 8, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    const uint64_t pad = sparse_pad(g, kept);
    const size_t wb = s_w ? weight_size(g.wkind) : 0;  // weights only for programs that read them
    const unsigned gr = grid_for((nwords + 7) / 8 * 32, 256, 148ull * 8);
    if (g.e_loc) {
        if (wb == 0)
            compact_kernel<0><<<gr, 256, 0, g.stream>>>(g.src, g.w, g.e_loc, g.full.pad, bitmap,
                                                        wpref, s_src, s_w, pad, sp_quads(g));
        else if (wb == 4)
            compact_kernel<4><<<gr, 256, 0, g.stream>>>(g.src, g.w, g.e_loc, g.full.pad, bitmap,
                                                        wpref, s_src, s_w, pad, sp_quads(g));
        else
            compact_kernel<8><<<gr, 256, 0, g.stream>>>(g.src, g.w, g.e_loc, g.full.pad, bitmap,
                                                        wpref, s_src, s_w, pad, sp_quads(g));
        GGB_CUDA(cudaGetLastError());
    }
    build_sparse_layout(g, bitmap, wpref, s_off, pad, kept, meta);
    if (ev1) GGB_CUDA(cudaEventRecord(ev1, g.stream));
    if (launches) *launches += 2;  // compact, sp_layout
    return kept;
}

// --------------------------------------------------------------------------
// hot-first message slots
// --------------------------------------------------------------------------
// floor(log2 out-degree) of every vertex (bin 32: out-degree 0)
__global__ void octave_hist_kernel(const uint32_t* __restrict__ outdeg, uint64_t n,
                                   unsigned long long* __restrict__ hist) {
    __shared__ unsigned int h[33];
    for (int i = threadIdx.x; i < 33; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t d = outdeg[v];
        atomicAdd(&h[d ? 31 - __clz(d) : 32], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 33; i += blockDim.x)
        if (h[i]) atomicAdd(hist + i, (unsigned long long)h[i]);
}

// Slot key: (tier, rank, out-degree class desc); ties keep vertex order
// (stable radix sort of (key, v)). tier 0 = out-degree octave >= hot_oct
// (the hot vertices of EVERY rank, a global prefix); with one rank the tier
// only refines nothing (it is monotone in the class), so the order is (class
// desc, id).
__global__ void slot_key_kernel(const uint32_t* __restrict__ outdeg, uint64_t n,
                                const uint64_t* __restrict__ bounds, int nranks, int rank_bits,
                                int hot_oct, uint64_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                int qbits) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t r = 0;
        while (r + 1 < (uint64_t)nranks && v >= bounds[r + 1]) ++r;
        const uint32_t d = outdeg[v];
        uint32_t h = d;
        if (qbits >= 0 && d) {  // degree class: floor(log2 d) and the next qbits bits
            const int lz = 31 - __clz(d);
            const uint32_t frac = qbits ? ((d << (31 - lz)) >> (31 - qbits)) & ((1u << qbits) - 1u) : 0u;
            h = 1u + ((uint32_t)lz << qbits) + frac;
        }
        const uint64_t tier = (d && 31 - __clz(d) >= hot_oct) ? 0ull : 1ull;
        keys[v] = (tier << (32 + rank_bits)) | (r << 32) | (uint64_t)(0xffffffffu - h);
        vals[v] = (uint32_t)v;
    }
}

__global__ void slot_fill_kernel(const uint32_t* __restrict__ sorted_v, uint64_t n,
                                 uint32_t* __restrict__ slot_of, uint32_t* __restrict__ vtx_of_slot) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t v = sorted_v[i];
        slot_of[v] = (uint32_t)i;
        vtx_of_slot[i] = v;
    }
}

// vertex ids -> message slots; with `bad`, sources >= n are flagged (and
// mapped to slot 0) instead of read out of bounds
__global__ void relabel_kernel(uint32_t* __restrict__ src, uint64_t count,
                               const uint32_t* __restrict__ slot_of, uint64_t n,
                               unsigned int* __restrict__ bad) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t s = src[i];
        if (bad && s >= n) {
            *bad = 1;
            src[i] = 0;
        } else {
            src[i] = __ldg(slot_of + s);
        }
    }
}

// local offsets must not decrease (Graph::validate, graph.cpp:83-86)
__global__ void offsets_check_kernel(const uint64_t* __restrict__ off, uint64_t nloc,
                                     unsigned int* __restrict__ bad) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < nloc;
         v += (uint64_t)gridDim.x * blockDim.x)
        if (off[v] > off[v + 1]) *bad = 1;
}
void check_offsets(DevGraph& g, unsigned int* bad) {
    if (!g.nloc) return;
    offsets_check_kernel<<<grid_for(g.nloc, 256), 256, 0, g.stream>>>(g.off, g.nloc, bad);
    GGB_CUDA(cudaGetLastError());
}

// per rank: [3r] tier-0 (hot) vertices, [3r+1] out-degree > 0 vertices
__global__ void gathered_count_kernel(const uint32_t* __restrict__ outdeg, uint64_t n,
                                      const uint64_t* __restrict__ bounds, int nranks, int hot_oct,
                                      unsigned long long* __restrict__ cnt) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n;
         v += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t d = outdeg[v];
        if (!d) continue;
        int r = 0;
        while (r + 1 < nranks && v >= bounds[r + 1]) ++r;
        if (31 - __clz(d) >= hot_oct) atomicAdd(cnt + 3 * r, 1ull);
        atomicAdd(cnt + 3 * r + 1, 1ull);
    }
}

// message slots of the tier-0 (hot) class: the L1+L2 evict_last prefix of an
// 8-byte message array (engine.cuh hot_bytes, 24 MB)
constexpr uint64_t kHotTierSlots = (24ull << 20) / 8;

void compute_slots(DevGraph& g) {
    const uint64_t n = g.n;
    g.slot_of = static_cast<decltype(g.slot_of)>(dev_alloc((n + 1) * 4, g.stream));
    g.vtx_of_slot = static_cast<decltype(g.vtx_of_slot)>(dev_alloc((n + 1) * 4, g.stream));
    if (n == 0) return;
    uint64_t *k0 = nullptr, *k1 = nullptr, *db = nullptr;
    uint32_t *v0 = nullptr, *v1 = nullptr;
    k0 = static_cast<decltype(k0)>(dev_alloc(n * 8, g.stream));
    k1 = static_cast<decltype(k1)>(dev_alloc(n * 8, g.stream));
    v0 = static_cast<decltype(v0)>(dev_alloc(n * 4, g.stream));
    v1 = static_cast<decltype(v1)>(dev_alloc(n * 4, g.stream));
    db = static_cast<decltype(db)>(dev_alloc(g.bounds.size() * 8, g.stream));
    GGB_CUDA(cudaMemcpyAsync(db, g.bounds.data(), g.bounds.size() * 8, cudaMemcpyHostToDevice,
                             g.stream));
    int qbits = 0;  // octave classes (GGB_SLOT_QBITS: -1 exact degree, q > 0 finer classes)
    if (const char* e = std::getenv("GGB_SLOT_QBITS")) qbits = std::atoi(e);
    int rank_bits = 0;
    while ((1 << rank_bits) < g.nranks) ++rank_bits;
    // hot tier (several ranks): the highest out-degree octaves holding at most
    // kHotTierSlots vertices; one rank: no tier (the class order is already
    // hot-first)
    int hot_oct = 33;
    if (g.nranks > 1) {
        auto* hist = static_cast<unsigned long long*>(dev_alloc(33 * 8, g.stream));
        GGB_CUDA(cudaMemsetAsync(hist, 0, 33 * 8, g.stream));
        octave_hist_kernel<<<grid_for(n, 256), 256, 0, g.stream>>>(g.outdeg, n, hist);
        GGB_CUDA(cudaGetLastError());
        uint64_t h[33];
        GGB_CUDA(cudaMemcpyAsync(h, hist, 33 * 8, cudaMemcpyDeviceToHost, g.stream));
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        dev_free(hist, g.stream);
        uint64_t cum = 0;
        for (int o = 31; o >= 0; --o) {
            if (cum + h[o] > kHotTierSlots) break;
            cum += h[o];
            hot_oct = o;
        }
    }
    slot_key_kernel<<<grid_for(n, 256), 256, 0, g.stream>>>(g.outdeg, n, db, g.nranks, rank_bits,
                                                           hot_oct, k0, v0, qbits);
    GGB_CUDA(cudaGetLastError());
    const int key_bits = 32 + rank_bits + (g.nranks > 1 ? 1 : 0);
    size_t tmp = 0;
    GGB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, k0, k1, v0, v1, n, 0, key_bits, g.stream));
    void* tmpp = nullptr;
    tmpp = static_cast<decltype(tmpp)>(dev_alloc(tmp, g.stream));
    GGB_CUDA(cub::DeviceRadixSort::SortPairs(tmpp, tmp, k0, k1, v0, v1, n, 0, key_bits, g.stream));
    slot_fill_kernel<<<grid_for(n, 256), 256, 0, g.stream>>>(v1, n, g.slot_of, g.vtx_of_slot);
    GGB_CUDA(cudaGetLastError());
    if (g.nranks > 1) {  // per-rank slot ranges of the messages the exchange carries
        const int R = g.nranks;
        auto* cnt = static_cast<unsigned long long*>(dev_alloc(8 * 3 * R, g.stream));
        GGB_CUDA(cudaMemsetAsync(cnt, 0, 8 * 3 * R, g.stream));
        gathered_count_kernel<<<grid_for(n, 256), 256, 0, g.stream>>>(g.outdeg, n, db, R, hot_oct, cnt);
        GGB_CUDA(cudaGetLastError());
        std::vector<uint64_t> c(3 * R);
        GGB_CUDA(cudaMemcpyAsync(c.data(), cnt, 8 * 3 * R, cudaMemcpyDeviceToHost, g.stream));
        GGB_CUDA(cudaStreamSynchronize(g.stream));
        dev_free(cnt, g.stream);
        uint64_t hot_total = 0;
        for (int r = 0; r < R; ++r) hot_total += c[3 * r];
        g.hot_slots = hot_total;
        g.gather_ranges.assign(4 * R, 0);
        uint64_t hb = 0, cb = hot_total;
        for (int r = 0; r < R; ++r) {
            const uint64_t nv = g.bounds[r + 1] - g.bounds[r], hot = c[3 * r], gat = c[3 * r + 1];
            g.gather_ranges[4 * r + 0] = hb;
            g.gather_ranges[4 * r + 1] = hb + hot;
            g.gather_ranges[4 * r + 2] = cb;
            g.gather_ranges[4 * r + 3] = cb + (gat - hot);
            hb += hot;
            cb += nv - hot;
        }
    }
    dev_free(k0, g.stream); dev_free(k1, g.stream); dev_free(v0, g.stream); dev_free(v1, g.stream); dev_free(db, g.stream); dev_free(tmpp, g.stream);
}

void relabel_sources(DevGraph& g, uint32_t* src, uint64_t count, unsigned int* bad) {
    if (!count) return;
    relabel_kernel<<<grid_for(count, 256), 256, 0, g.stream>>>(src, count, g.slot_of, g.n, bad);
    GGB_CUDA(cudaGetLastError());
}

void assign_slots(DevGraph& g) {
    compute_slots(g);
    relabel_sources(g, g.src + g.full.pad, g.e_loc);
    GGB_CUDA(cudaStreamSynchronize(g.stream));
}

__global__ void unlabel_kernel(const uint32_t* __restrict__ src, uint64_t count,
                               const uint32_t* __restrict__ vtx_of_slot, uint32_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
         i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = __ldg(vtx_of_slot + src[i]);
}

void export_sources(const DevGraph& g, uint32_t* host_out) {
    uint32_t* tmp = nullptr;
    tmp = static_cast<decltype(tmp)>(dev_alloc((g.e_loc + 1) * 4, g.stream));
    unlabel_kernel<<<grid_for(g.e_loc, 256), 256, 0, g.stream>>>(g.src + g.full.pad, g.e_loc,
                                                                  g.vtx_of_slot, tmp);
    GGB_CUDA(cudaGetLastError());
    GGB_CUDA(cudaMemcpyAsync(host_out, tmp, g.e_loc * 4, cudaMemcpyDeviceToHost, g.stream));
    GGB_CUDA(cudaStreamSynchronize(g.stream));
    dev_free(tmp, g.stream);
}

// Rows only: an in-degree-0 vertex keeps no edges, so its condition is its
// pre-iteration status alone and the vertex kernel reports it directly.
__global__ void superstep_invalid_kernel(uint32_t nrows, uint32_t v_begin,
                                         const uint32_t* __restrict__ vid_of_p,
                                         const uint8_t* __restrict__ st,
                                         const uint64_t* __restrict__ s_off,
                                         IterCounters* __restrict__ ctr) {
    if (!__ldg(&ctr->any_invalid)) return;  // the common case: nothing to rescan
    for (uint32_t p = blockIdx.x * blockDim.x + threadIdx.x; p < nrows; p += gridDim.x * blockDim.x) {
        const uint8_t s = st[p];
        if ((s & kStInvalid) && ((s & kStWasActive) || s_off[p + 1] > s_off[p]))
            atomicMin(&ctr->bad_min, v_begin + vid_of_p[p]);
    }
}

void launch_superstep_invalid(DevGraph& g, const uint8_t* st, const uint64_t* s_off, void* ctr) {
    if (!g.nrows) return;
    superstep_invalid_kernel<<<grid_for(g.nrows, 256), 256, 0, g.stream>>>(
        (uint32_t)g.nrows, (uint32_t)g.v_begin, g.vid_of_p, st, s_off,
        static_cast<IterCounters*>(ctr));
    GGB_CUDA(cudaGetLastError());
}

DevGraph::~DevGraph() {
    exchange_release_peers(*this);
    if (ipc_msg) cudaFree(ipc_msg);
    ws.release();
    if (h_ctr) cudaFreeHost(h_ctr);
    for (cudaEvent_t e : ev)
        if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : bev) cudaEventDestroy(e);
    dev_free(off, stream);
    dev_free(src, stream);
    dev_free(w, stream);
    dev_free(outdeg, stream);
    dev_free(slot_of, stream);
    dev_free(vtx_of_slot, stream);
    dev_free(vid_of_p, stream);
    dev_free(slot_p, stream);
    dev_free(deg_p, stream);
    if (stream) {
        cudaStreamSynchronize(stream);
        cudaStreamDestroy(stream);
    }
}

// slot 0 stands for "iteration 0": every status starts active, so the
// first vertex kernel walks the in-degree-0 positions too
__global__ void reset_counters_kernel(IterCounters* __restrict__ c, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        IterCounters z{};
        z.bad_min = 0xffffffffu;
        z.empty_active = i == 0 ? 1u : 0u;
        c[i] = z;
    }
}

}  // namespace ggb
