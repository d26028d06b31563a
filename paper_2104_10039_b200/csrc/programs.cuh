// programs.cuh — device vertex programs.
//
// The device program concept is the reference's VertexProgram
// (engine.hpp:80-93: init_property, gather_identity, gather -> influence,
// apply, vstatus, estatus, valid) with the SAME formulas, plus the two
// members a parallel gather needs:
//   message(p, out_degree)  the per-source value every gather reads. The
//                           reference passes (src property, src out-degree)
//                           to gather; precomputing e.g. PR's p/deg once per
//                           source yields the identical double per edge.
//   combine(a, b)           the accumulator after folding b's edges after
//                           a's. Exact for PR? no (FP sum association, the
//                           stated tolerance), exact for SSSP/WCC (min).
// Property types are trivially copyable (BP uses a fixed-S array instead of
// std::vector, algorithms.hpp:121).
#pragma once

#include <cmath>
#include <cstdint>

#include "common.cuh"

namespace ggb {

// PageRankProgram, algorithms.hpp:15-40.
struct PageRank {
    using Property = double;
    using Message = double;
    using Accum = double;
    static constexpr bool kRelGrowthInfluence = true;  // gather's influence, estatus `> theta`
    static constexpr bool kMsgIsProp = false;
    static constexpr bool kNeedsDegree = true;
    double damping = 0.85, epsilon = 1e-7;

    __device__ Property init_property(uint32_t, uint64_t n) const { return 1.0 / (double)n; }
    __device__ Accum gather_identity() const { return 0.0; }
    __device__ Message message(const Property& p, uint32_t deg) const {
        return p / (double)deg;  // the per-edge `src / double(src_out_degree)` (:28)
    }
    __device__ double gather(Accum& acc, const Message& m, double) const {  // :25-30
        const double before = acc;
        acc = acc + m;
        return acc > 0.0 ? (acc - before) / acc : 0.0;
    }
    __device__ Accum combine(const Accum& a, const Accum& b) const { return a + b; }
    __device__ Property apply(uint32_t, const Accum& acc, const Property&, uint64_t n) const {
        return (1.0 - damping) / (double)n + damping * acc;  // :31-34
    }
    __device__ bool vstatus(const Property& b, const Property& a) const {
        return fabs(b - a) > epsilon;  // :35-37
    }
    __device__ bool estatus(double infl, double theta) const { return infl > theta; }
    __device__ bool valid(const Property& p) const { return isfinite(p); }
    __device__ double to_double(const Property& p, int) const { return p; }
};

// SsspProgram with f64 distances (algorithms.hpp:46-83) — any weights.
struct SsspF64 {
    using Property = double;
    using Message = double;
    using Accum = double;
    static constexpr bool kMsgIsProp = true;
    static constexpr bool kNeedsDegree = false;
    uint32_t source = 0;
    bool graded = false;

    __device__ Property init_property(uint32_t v, uint64_t) const {
        return v == source ? 0.0 : INFINITY;
    }
    __device__ Accum gather_identity() const { return INFINITY; }
    __device__ Message message(const Property& p, uint32_t) const { return p; }
    __device__ double gather(Accum& acc, const Message& m, double w) const {  // :61-73
        const double cand = m + w;
        if (cand < acc) {
            double infl = 1.0;
            if (graded && isfinite(acc)) infl = (acc - cand) / acc;
            acc = cand;
            return infl;
        }
        return 0.0;
    }
    __device__ Accum combine(const Accum& a, const Accum& b) const { return b < a ? b : a; }
    __device__ Property apply(uint32_t, const Accum& acc, const Property& prev, uint64_t) const {
        return prev < acc ? prev : acc;  // std::min(acc, prev)
    }
    __device__ bool vstatus(const Property& b, const Property& a) const { return a < b; }
    __device__ bool estatus(double infl, double theta) const { return infl > theta; }
    __device__ bool valid(const Property& p) const { return !isnan(p) && p >= 0.0; }
    __device__ double to_double(const Property& p, int) const { return p; }
};

// SsspProgram with u32 distances (BASELINE C2: u32 weights, or unit
// weights). Integer sums are exact in f64, so every comparison and every
// graded influence (computed in f64 from the exact integers) is bit-identical
// to the f64 program. 0xffffffff encodes +inf. A candidate distance that does
// not fit raises *overflow; the run is then repeated with SsspF64 (capi.cu),
// so results stay those of the reference's f64 distances.
struct SsspU32 {
    using Property = uint32_t;
    using Message = uint32_t;
    using Accum = uint32_t;
    static constexpr bool kMsgIsProp = true;
    static constexpr bool kNeedsDegree = false;
    static constexpr uint32_t kInf = 0xffffffffu;
    uint32_t source = 0;
    bool graded = false;
    unsigned int* overflow = nullptr;

    __device__ Property init_property(uint32_t v, uint64_t) const { return v == source ? 0u : kInf; }
    __device__ Accum gather_identity() const { return kInf; }
    __device__ Message message(const Property& p, uint32_t) const { return p; }
    __device__ double gather(Accum& acc, const Message& m, double w) const {
        if (m == kInf) return 0.0;  // inf + w < acc is false for every acc
        const uint64_t c64 = (uint64_t)m + (uint64_t)w;
        if (c64 >= kInf) *overflow = 1;  // the run is redone with f64 distances
        const uint32_t cand = c64 >= kInf ? kInf - 1 : (uint32_t)c64;
        if (cand < acc) {
            double infl = 1.0;
            if (graded && acc != kInf) infl = ((double)acc - (double)cand) / (double)acc;
            acc = cand;
            return infl;
        }
        return 0.0;
    }
    __device__ Accum combine(const Accum& a, const Accum& b) const { return b < a ? b : a; }
    __device__ Property apply(uint32_t, const Accum& acc, const Property& prev, uint64_t) const {
        return prev < acc ? prev : acc;
    }
    __device__ bool vstatus(const Property& b, const Property& a) const { return a < b; }
    __device__ bool estatus(double infl, double theta) const { return infl > theta; }
    __device__ bool valid(const Property&) const { return true; }
    __device__ double to_double(const Property& p, int) const {
        return p == kInf ? INFINITY : (double)p;
    }
};

// WccProgram, algorithms.hpp:88-112.
struct Wcc {
    using Property = uint32_t;
    using Message = uint32_t;
    using Accum = uint32_t;
    static constexpr bool kMsgIsProp = true;
    static constexpr bool kNeedsDegree = false;
    static constexpr bool kRawOutput = true;  // labels leave as uint32 (VertexId)

    __device__ Property init_property(uint32_t v, uint64_t) const { return v; }
    __device__ Accum gather_identity() const { return 0xffffffffu; }
    __device__ Message message(const Property& p, uint32_t) const { return p; }
    __device__ double gather(Accum& acc, const Message& m, double) const {
        if (m < acc) { acc = m; return 1.0; }
        return 0.0;
    }
    __device__ Accum combine(const Accum& a, const Accum& b) const { return b < a ? b : a; }
    __device__ Property apply(uint32_t, const Accum& acc, const Property& prev, uint64_t) const {
        return prev < acc ? prev : acc;
    }
    __device__ bool vstatus(const Property& b, const Property& a) const { return a != b; }
    __device__ bool estatus(double infl, double theta) const { return infl > theta; }
    __device__ bool valid(const Property&) const { return true; }
    __device__ double to_double(const Property& p, int) const { return (double)p; }
};

template <int S>
struct Belief {
    double x[S];
};
struct BeliefF2 {
    float x[2];
};

// BP gather core, algorithms.cpp:25-48 (coupling passed in: global for the
// reference program, per edge for BASELINE C4).
template <int S, class Src>
__device__ __forceinline__ double bp_gather_core(double* acc, const Src& src, double coupling) {
    const double off = (1.0 - coupling) / (double)(S - 1);
    double src_sum = 0.0;
#pragma unroll
    for (int i = 0; i < S; ++i) src_sum += (double)src.x[i];
    double l1_after = 0.0, l1_diff = 0.0, acc_sum = 0.0;
#pragma unroll
    for (int i = 0; i < S; ++i) {
        const double si = (double)src.x[i];
        const double msg = off * (src_sum - si) + coupling * si;
        const double updated = acc[i] * msg;
        l1_after += fabs(updated);
        l1_diff += fabs(acc[i] - updated);
        acc[i] = updated;
        acc_sum += updated;
    }
    if (acc_sum > 0.0) {
#pragma unroll
        for (int i = 0; i < S; ++i) acc[i] /= acc_sum;
    }
    if (l1_after <= 0.0) return 0.0;
    const double r = l1_diff / l1_after;
    return r < 1.0 ? r : 1.0;
}

template <int S>
__device__ __forceinline__ bool bp_is_identity(const Belief<S>& a) {
#pragma unroll
    for (int i = 0; i < S; ++i)
        if (a.x[i] != 1.0) return false;
    return true;
}

// combine: elementwise product then renormalise (the fold's own per-edge
// renormalisation, algorithms.cpp:41-43). The identity (all ones, never a
// normalised vector) is an exact neutral element.
template <int S>
__device__ __forceinline__ Belief<S> bp_combine(const Belief<S>& a, const Belief<S>& b) {
    if (bp_is_identity(a)) return b;
    if (bp_is_identity(b)) return a;
    Belief<S> r;
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < S; ++i) { r.x[i] = a.x[i] * b.x[i]; s += r.x[i]; }
    if (s > 0.0) {
#pragma unroll
        for (int i = 0; i < S; ++i) r.x[i] /= s;
    }
    return r;
}

// BeliefPropagationProgram, algorithms.hpp:120-145 / algorithms.cpp:9-69.
template <int S>
struct BeliefProp {
    using Property = Belief<S>;
    using Message = Belief<S>;
    using Accum = Belief<S>;
    static constexpr bool kMsgIsProp = true;
    static constexpr bool kNeedsDegree = false;
    static constexpr bool kHeavyGather = true;
    double coupling = 0.8, epsilon = 1e-6;

    __device__ Property prior(uint32_t v) const {  // algorithms.cpp:9-23
        Property p;
        double sum = 0.0;
#pragma unroll
        for (int i = 0; i < S; ++i) {
            const uint64_t h = mix64((uint64_t)v * (uint64_t)S + (uint64_t)i);
            p.x[i] = 1.0 + (double)(h >> 11) * 0x1.0p-53;
            sum += p.x[i];
        }
#pragma unroll
        for (int i = 0; i < S; ++i) p.x[i] /= sum;
        return p;
    }
    __device__ Property init_property(uint32_t v, uint64_t) const { return prior(v); }
    __device__ Accum gather_identity() const {
        Accum a;
#pragma unroll
        for (int i = 0; i < S; ++i) a.x[i] = 1.0;
        return a;
    }
    __device__ Message message(const Property& p, uint32_t) const { return p; }
    __device__ double gather(Accum& acc, const Message& m, double) const {
        return bp_gather_core<S>(acc.x, m, coupling);
    }
    __device__ Accum combine(const Accum& a, const Accum& b) const { return bp_combine<S>(a, b); }
    __device__ Property apply(uint32_t v, const Accum& acc, const Property&, uint64_t) const {
        Property out = prior(v);  // algorithms.cpp:50-62
        double sum = 0.0;
#pragma unroll
        for (int i = 0; i < S; ++i) { out.x[i] *= acc.x[i]; sum += out.x[i]; }
        if (sum > 0.0) {
#pragma unroll
            for (int i = 0; i < S; ++i) out.x[i] /= sum;
        }
        return out;
    }
    __device__ bool vstatus(const Property& b, const Property& a) const {  // :64-69
        double l1 = 0.0;
#pragma unroll
        for (int i = 0; i < S; ++i) l1 += fabs(b.x[i] - a.x[i]);
        return l1 > epsilon;
    }
    __device__ bool estatus(double infl, double theta) const { return infl > theta; }
    __device__ bool valid(const Property& p) const {
#pragma unroll
        for (int i = 0; i < S; ++i)
            if (!isfinite(p.x[i])) return false;
        return true;
    }
    __device__ double to_double(const Property& p, int i) const { return p.x[i]; }
};

// BeliefPropagationProgram with any state count 5..kBpMaxStates chosen at run
// time (BeliefProp<S> covers 2..4 with compile-time loops); storage is a
// fixed Belief<MaxS> of the smallest tier (16, 32, 64 states) that holds S,
// states >= S are never touched. Same formulas and operation order as
// BeliefProp<S> (algorithms.cpp:9-69).
constexpr int kBpMaxStates = 64;
template <int MaxS>
struct BeliefPropDyn {
    using Property = Belief<MaxS>;
    using Message = Property;
    using Accum = Property;
    static constexpr bool kMsgIsProp = true;
    static constexpr bool kNeedsDegree = false;
    static constexpr bool kHeavyGather = true;
    int states = 5;
    double coupling = 0.8, epsilon = 1e-6;

    __device__ Property prior(uint32_t v) const {  // algorithms.cpp:9-23
        Property p;
        double sum = 0.0;
        for (int i = 0; i < states; ++i) {
            const uint64_t h = mix64((uint64_t)v * (uint64_t)states + (uint64_t)i);
            p.x[i] = 1.0 + (double)(h >> 11) * 0x1.0p-53;
            sum += p.x[i];
        }
        for (int i = 0; i < states; ++i) p.x[i] /= sum;
        return p;
    }
    __device__ Property init_property(uint32_t v, uint64_t) const { return prior(v); }
    __device__ Accum gather_identity() const {
        Accum a;
        for (int i = 0; i < states; ++i) a.x[i] = 1.0;
        return a;
    }
    __device__ Message message(const Property& p, uint32_t) const { return p; }
    __device__ double gather(Accum& acc, const Message& src, double) const {  // :25-48
        const double off = (1.0 - coupling) / (double)(states - 1);
        double src_sum = 0.0;
        for (int i = 0; i < states; ++i) src_sum += src.x[i];
        double l1_after = 0.0, l1_diff = 0.0, acc_sum = 0.0;
        for (int i = 0; i < states; ++i) {
            const double si = src.x[i];
            const double msg = off * (src_sum - si) + coupling * si;
            const double updated = acc.x[i] * msg;
            l1_after += fabs(updated);
            l1_diff += fabs(acc.x[i] - updated);
            acc.x[i] = updated;
            acc_sum += updated;
        }
        if (acc_sum > 0.0)
            for (int i = 0; i < states; ++i) acc.x[i] /= acc_sum;
        if (l1_after <= 0.0) return 0.0;
        const double r = l1_diff / l1_after;
        return r < 1.0 ? r : 1.0;
    }
    __device__ bool is_identity(const Accum& a) const {
        for (int i = 0; i < states; ++i)
            if (a.x[i] != 1.0) return false;
        return true;
    }
    __device__ Accum combine(const Accum& a, const Accum& b) const {
        if (is_identity(a)) return b;
        if (is_identity(b)) return a;
        Accum r;
        double s = 0.0;
        for (int i = 0; i < states; ++i) { r.x[i] = a.x[i] * b.x[i]; s += r.x[i]; }
        if (s > 0.0)
            for (int i = 0; i < states; ++i) r.x[i] /= s;
        return r;
    }
    __device__ Property apply(uint32_t v, const Accum& acc, const Property&, uint64_t) const {
        Property out = prior(v);  // algorithms.cpp:50-62
        double sum = 0.0;
        for (int i = 0; i < states; ++i) { out.x[i] *= acc.x[i]; sum += out.x[i]; }
        if (sum > 0.0)
            for (int i = 0; i < states; ++i) out.x[i] /= sum;
        return out;
    }
    __device__ bool vstatus(const Property& b, const Property& a) const {  // :64-69
        double l1 = 0.0;
        for (int i = 0; i < states; ++i) l1 += fabs(b.x[i] - a.x[i]);
        return l1 > epsilon;
    }
    __device__ bool estatus(double infl, double theta) const { return infl > theta; }
    __device__ bool valid(const Property& p) const {
        for (int i = 0; i < states; ++i)
            if (!isfinite(p.x[i])) return false;
        return true;
    }
    __device__ double to_double(const Property& p, int i) const { return p.x[i]; }
};

// BASELINE C4 BP: reference formulas, S = 2, coupling = the edge's fp32 c_e,
// prior from an fp32 table, beliefs STORED as fp32 (arithmetic in f64).
struct BeliefPropEdge {
    using Property = BeliefF2;
    using Message = BeliefF2;
    using Accum = Belief<2>;
    static constexpr bool kMsgIsProp = true;
    static constexpr bool kNeedsDegree = false;
    static constexpr bool kReadsPrior = true;
    static constexpr bool kHeavyGather = true;
    const float2* prior_table = nullptr;
    double epsilon = 1e-6;

    __device__ Property init_property(uint32_t v, uint64_t) const {
        const float2 p = prior_table[v];
        return Property{{p.x, p.y}};
    }
    __device__ Accum gather_identity() const { return Accum{{1.0, 1.0}}; }
    __device__ Message message(const Property& p, uint32_t) const { return p; }
    __device__ double gather(Accum& acc, const Message& m, double c) const {
        return bp_gather_core<2>(acc.x, m, c);
    }
    __device__ Accum combine(const Accum& a, const Accum& b) const { return bp_combine<2>(a, b); }
    __device__ Property apply(uint32_t v, const Accum& acc, const Property&, uint64_t) const {
        const float2 p = prior_table[v];
        double o0 = (double)p.x * acc.x[0], o1 = (double)p.y * acc.x[1];
        const double sum = o0 + o1;
        if (sum > 0.0) { o0 /= sum; o1 /= sum; }
        return Property{{(float)o0, (float)o1}};
    }
    __device__ bool vstatus(const Property& b, const Property& a) const {
        const double l1 = fabs((double)b.x[0] - (double)a.x[0]) + fabs((double)b.x[1] - (double)a.x[1]);
        return l1 > epsilon;
    }
    __device__ bool estatus(double infl, double theta) const { return infl > theta; }
    __device__ bool valid(const Property& p) const { return isfinite(p.x[0]) && isfinite(p.x[1]); }
    __device__ double to_double(const Property& p, int i) const { return (double)p.x[i]; }
};

}  // namespace ggb
