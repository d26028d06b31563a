// ggb.hpp — header-only C++ face of libggb.so (include/ggb.h).
//
// RAII ownership of the HBM-resident graph and typed run entries that turn
// gg_status codes back into the exceptions the reference throws:
//   GG_INVALID_ARGUMENT -> std::invalid_argument   (engine.cpp:45-61)
//   GG_INVALID_PROPERTY -> ggb::PropertyError       (gg::EngineError, engine.hpp:60-74)
//   anything else       -> ggb::DeviceError         (CUDA / NCCL / OOM)
// No reference types appear here; include/ggb_gg.hpp binds them.
#pragma once

#include <algorithm>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ggb.h"

namespace ggb {

class DeviceError : public std::runtime_error {
  public:
    DeviceError(gg_status s, const std::string& what) : std::runtime_error(what), status_(s) {}
    gg_status status() const { return status_; }

  private:
    gg_status status_;
};

class PropertyError : public std::runtime_error {
  public:
    PropertyError(std::uint64_t iteration, std::uint32_t vertex, const std::string& what)
        : std::runtime_error(what), iteration_(iteration), vertex_(vertex) {}
    std::uint64_t iteration() const { return iteration_; }
    std::uint32_t vertex() const { return vertex_; }

  private:
    std::uint64_t iteration_;
    std::uint32_t vertex_;
};

inline void check(gg_status s, const gg_error& e) {
    if (s == GG_OK) return;
    if (s == GG_INVALID_ARGUMENT) throw std::invalid_argument(e.msg);
    if (s == GG_INVALID_PROPERTY) throw PropertyError(e.iteration, e.vertex, e.msg);
    throw DeviceError(s, std::string(gg_status_string(s)) + ": " + e.msg);
}

// One rank's slice of the pull CSC, resident in HBM (gg::Graph, graph.hpp:29-49).
class DeviceGraph {
  public:
    DeviceGraph() = default;
    explicit DeviceGraph(const gg_csc_view& csc, int device = -1) {
        gg_part_opts o{device, 0, 1, nullptr};
        gg_error e{};
        check(gg_dev_graph_create(&csc, &o, &g_, &e), e);
    }
    DeviceGraph(const gg_csc_view& csc, const gg_part_opts& opts) {
        gg_error e{};
        check(gg_dev_graph_create(&csc, &opts, &g_, &e), e);
    }
    // uploaded for one sparse-scheme run: its sparsification overlaps the upload
    static DeviceGraph for_run(const gg_csc_view& csc, double sigma, std::uint64_t seed,
                               int device = -1) {
        DeviceGraph d;
        gg_part_opts o{device, 0, 1, nullptr};
        gg_error e{};
        check(gg_dev_graph_create_for_run(&csc, &o, sigma, seed, &d.g_, &e), e);
        return d;
    }
    static DeviceGraph rmat(const gg_rmat_params& p, const gg_part_opts& opts) {
        DeviceGraph d;
        gg_error e{};
        check(gg_dev_graph_create_rmat(&p, &opts, &d.g_, &e), e);
        return d;
    }
    DeviceGraph(const DeviceGraph&) = delete;
    DeviceGraph& operator=(const DeviceGraph&) = delete;
    DeviceGraph(DeviceGraph&& o) noexcept : g_(std::exchange(o.g_, nullptr)) {}
    DeviceGraph& operator=(DeviceGraph&& o) noexcept {
        if (this != &o) {
            reset();
            g_ = std::exchange(o.g_, nullptr);
        }
        return *this;
    }
    ~DeviceGraph() { reset(); }

    gg_dev_graph* get() const { return g_; }
    std::uint64_t num_vertices() const { return info().n; }
    std::uint64_t num_edges() const { return info().e; }

    struct Info {
        std::uint64_t n, e, v_begin, v_end, e_local;
    };
    Info info() const {
        Info i{};
        gg_error e{};
        check(gg_dev_graph_info(g_, &i.n, &i.e, &i.v_begin, &i.v_end, &i.e_local), e);
        return i;
    }

  private:
    void reset() {
        if (g_) gg_dev_graph_destroy(g_);
        g_ = nullptr;
    }
    gg_dev_graph* g_ = nullptr;
};

// What a run returns (gg::RunReport, engine.hpp:49-56), with properties in
// the C-ABI layout (flat; BP: `states` doubles per vertex).
template <class T>
struct Run {
    std::vector<T> properties;
    std::vector<gg_iter_record> records;
    gg_run_summary summary{};
};

namespace detail {
// Records kept per run: every executed iteration up to 65,536 (the engine
// still runs past the cap; only the per-iteration log stops).
inline std::size_t record_cap(const gg_engine_config& c) {
    return static_cast<std::size_t>(std::min<std::uint64_t>(c.max_iterations, 1u << 16));
}
template <class T>
void trim(Run<T>& r) {
    r.records.resize(std::min<std::uint64_t>(r.summary.iterations_run, r.records.size()));
}
}  // namespace detail

inline Run<double> run_pr(const DeviceGraph& g, const gg_engine_config& c, const gg_pr_params& p) {
    Run<double> r;
    r.properties.resize(g.num_vertices());
    r.records.resize(detail::record_cap(c));
    gg_error e{};
    check(gg_run_pr(g.get(), &c, &p, r.properties.data(), r.records.data(), r.records.size(),
                    &r.summary, nullptr, &e), e);
    detail::trim(r);
    return r;
}

inline Run<double> run_sssp(const DeviceGraph& g, const gg_engine_config& c, const gg_sssp_params& p) {
    Run<double> r;
    r.properties.resize(g.num_vertices());
    r.records.resize(detail::record_cap(c));
    gg_error e{};
    check(gg_run_sssp(g.get(), &c, &p, r.properties.data(), r.records.data(), r.records.size(),
                      &r.summary, nullptr, &e), e);
    detail::trim(r);
    return r;
}

inline Run<std::uint32_t> run_wcc(const DeviceGraph& g, const gg_engine_config& c) {
    Run<std::uint32_t> r;
    r.properties.resize(g.num_vertices());
    r.records.resize(detail::record_cap(c));
    gg_error e{};
    check(gg_run_wcc(g.get(), &c, r.properties.data(), r.records.data(), r.records.size(),
                     &r.summary, nullptr, &e), e);
    detail::trim(r);
    return r;
}

inline Run<double> run_bp(const DeviceGraph& g, const gg_engine_config& c, const gg_bp_params& p) {
    Run<double> r;
    r.properties.resize(g.num_vertices() * static_cast<std::uint64_t>(p.states > 0 ? p.states : 1));
    r.records.resize(detail::record_cap(c));
    gg_error e{};
    check(gg_run_bp(g.get(), &c, &p, r.properties.data(), r.records.data(), r.records.size(),
                    &r.summary, nullptr, &e), e);
    detail::trim(r);
    return r;
}

}  // namespace ggb
