// ggb_gg.hpp — drop-in for the reference engine call
//
//     template <VertexProgram A>
//     RunReport<typename A::Property> gg::run(const Graph&, const A&, const EngineConfig&);
//                                      (proj/core/include/gg/engine.hpp:141-143)
//
// A caller of the reference switches `gg::run(g, program, cfg)` to
// `ggb::run(g, program, cfg)` (or, keeping the graph resident across runs,
// `ggb::DeviceGraph dg = ggb::upload(g); ggb::run(dg, program, cfg)`) and gets
// the same gg::RunReport back, with the same exceptions:
//   std::invalid_argument naming the field     (engine.cpp:45-61, algorithms.hpp:55-57)
//   gg::EngineError(iteration, vertex)          (engine.hpp:60-74)
//
// The four reference programs (algorithms.hpp:15-151) map at compile time to
// their compiled device programs (csrc/programs.cuh). A VertexProgram with no
// device entry is a compile error — there is no CPU fallback.
//
// Requires the reference's headers on the include path ("gg/engine.hpp",
// "gg/algorithms.hpp"); links against libggb.so only (no reference code runs).
#pragma once

#include <cstdint>
#include <type_traits>
#include <vector>

#include "gg/algorithms.hpp"
#include "gg/engine.hpp"
#include "ggb.hpp"

namespace ggb {

// gg::Graph (graph.hpp:29-49) as a borrowed C view; weights are f64.
inline gg_csc_view view_of(const gg::Graph& g) {
    gg_csc_view v{};
    v.n = g.num_vertices();
    v.e = g.num_edges();
    v.offsets = g.in_offsets.data();
    v.sources = g.in_sources.data();
    v.weight_kind = g.weighted() ? GG_W_F64 : GG_W_NONE;
    v.weights = g.weighted() ? static_cast<const void*>(g.weights.data()) : nullptr;
    v.out_degree = g.out_degree.data();
    return v;
}

inline DeviceGraph upload(const gg::Graph& g, int device = -1) { return DeviceGraph(view_of(g), device); }

// gg::EngineConfig (engine.hpp:28-36); enum values are identical.
inline gg_engine_config config_of(const gg::EngineConfig& c) {
    return gg_engine_config{static_cast<std::int32_t>(c.scheme), c.sigma, c.theta, c.alpha,
                            c.max_iterations, c.seed, c.threads};
}

namespace detail {

template <class P, class T, class F>
gg::RunReport<P> report_of(Run<T>&& r, F&& convert) {
    gg::RunReport<P> rep;
    rep.final_properties = std::forward<F>(convert)(r.properties);
    rep.iterations_run = r.summary.iterations_run;
    rep.total_wall_seconds = r.summary.total_wall_seconds;
    rep.total_processed_edges = r.summary.total_processed_edges;
    rep.per_iteration.reserve(r.records.size());
    for (const gg_iter_record& x : r.records) {
        gg::IterationRecord ir;
        ir.mode = static_cast<gg::IterationMode>(x.mode);
        ir.processed_edges = x.processed_edges;
        ir.active_vertices = x.active_vertices;
        ir.wall_seconds = x.wall_seconds;
        rep.per_iteration.push_back(ir);
    }
    return rep;
}

// ggb::PropertyError -> gg::EngineError, everything else passes through.
template <class F>
auto rethrow_as_reference(F&& f) -> decltype(f()) {
    try {
        return f();
    } catch (const PropertyError& e) {
        throw gg::EngineError(e.iteration(), e.vertex());
    }
}

inline const auto same = [](auto& v) { return std::move(v); };

template <class>
inline constexpr bool kNoDeviceEntry = false;

}  // namespace detail

// --- device entries, one per reference program -----------------------------

inline gg::RunReport<double> run(const DeviceGraph& g, const gg::PageRankProgram& a,
                                 const gg::EngineConfig& cfg) {
    return detail::rethrow_as_reference([&] {
        return detail::report_of<double>(
            run_pr(g, config_of(cfg), gg_pr_params{a.damping, a.epsilon}), detail::same);
    });
}

inline gg::RunReport<double> run(const DeviceGraph& g, const gg::SsspProgram& a,
                                 const gg::EngineConfig& cfg) {
    return detail::rethrow_as_reference([&] {
        return detail::report_of<double>(
            run_sssp(g, config_of(cfg), gg_sssp_params{a.source, a.graded ? 1 : 0}), detail::same);
    });
}

inline gg::RunReport<std::uint32_t> run(const DeviceGraph& g, const gg::WccProgram&,
                                        const gg::EngineConfig& cfg) {
    return detail::rethrow_as_reference([&] {
        return detail::report_of<std::uint32_t>(run_wcc(g, config_of(cfg)), detail::same);
    });
}

inline gg::RunReport<std::vector<double>> run(const DeviceGraph& g,
                                              const gg::BeliefPropagationProgram& a,
                                              const gg::EngineConfig& cfg) {
    const std::size_t s = a.states > 0 ? static_cast<std::size_t>(a.states) : 1;
    return detail::rethrow_as_reference([&] {
        return detail::report_of<std::vector<double>>(
            run_bp(g, config_of(cfg), gg_bp_params{a.states, a.coupling, a.epsilon, nullptr}),
            [s](const std::vector<double>& flat) {
                std::vector<std::vector<double>> out(flat.size() / s);
                for (std::size_t v = 0; v < out.size(); ++v)
                    out[v].assign(flat.begin() + v * s, flat.begin() + (v + 1) * s);
                return out;
            });
    });
}

// Any other VertexProgram: no device entry, no fallback.
template <class A>
gg::RunReport<typename A::Property> run(const DeviceGraph&, const A&, const gg::EngineConfig&) {
    static_assert(detail::kNoDeviceEntry<A>,
                  "ggb::run: this VertexProgram has no compiled device program "
                  "(add one to paper_2104_10039_b200/csrc/programs.cuh and a C-ABI entry)");
    return {};
}

// The reference signature: uploads the graph for this call.
template <class A>
auto run(const gg::Graph& g, const A& a, const gg::EngineConfig& cfg) {
    const DeviceGraph dg = cfg.scheme == gg::Scheme::accurate
                               ? upload(g)
                               : DeviceGraph::for_run(view_of(g), cfg.sigma, cfg.seed);
    return run(dg, a, cfg);
}

}  // namespace ggb
