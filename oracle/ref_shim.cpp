// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" face over the UNMODIFIED GraphGuess reference, compiled
// together with the reference's own sources (/root/reference/proj/core/src)
// by oracle/Makefile into oracle/_ref/libggref.so. Nothing here re-implements
// the engine: every run goes through the reference's gg::run template
// (engine.hpp:141-249) and its programs (algorithms.hpp). The two extra
// program types below are NEW VertexProgram types (BASELINE C4's per-edge BP
// and test_engine.cpp:23-50's PoisonProgram) handed, unchanged, to gg::run.
//
// Used for (1) pinning oracle/gg_oracle.c bit-for-bit against the reference,
// and (2) bench.py --impl reference / cpu_baseline (reference CPU timing).
#include <array>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "gg/algorithms.hpp"
#include "gg/bench.hpp"
#include "gg/engine.hpp"
#include "gg/graph.hpp"
#include "gg/metrics.hpp"

namespace {

// BASELINE C4: reference BP formulas (algorithms.cpp:25-62) with S = 2, the
// coupling taken from the edge weight, a table prior, fp32 belief storage.
struct BpEdgeProgram {
    using Property = std::array<double, 2>;
    const float* prior_table = nullptr;
    double epsilon = 1e-6;

    Property prior(gg::VertexId v) const {
        return {double(prior_table[2 * std::uint64_t(v)]),
                double(prior_table[2 * std::uint64_t(v) + 1])};
    }
    Property init_property(gg::VertexId v, std::size_t) const { return prior(v); }
    Property gather_identity() const { return {1.0, 1.0}; }
    double gather(Property& acc, const Property& src, double coupling,
                  std::uint32_t) const {
        const double off = (1.0 - coupling) / 1.0;
        double src_sum = 0.0;
        for (double x : src) src_sum += x;
        double l1_after = 0.0, l1_diff = 0.0, acc_sum = 0.0;
        for (int i = 0; i < 2; ++i) {
            const double msg = off * (src_sum - src[i]) + coupling * src[i];
            const double updated = acc[i] * msg;
            l1_after += std::fabs(updated);
            l1_diff += std::fabs(acc[i] - updated);
            acc[i] = updated;
            acc_sum += updated;
        }
        if (acc_sum > 0.0) {
            for (double& x : acc) x /= acc_sum;
        }
        if (l1_after <= 0.0) return 0.0;
        return std::min(1.0, l1_diff / l1_after);
    }
    Property apply(gg::VertexId v, const Property& acc, const Property&,
                   std::size_t) const {
        Property out = prior(v);
        double sum = 0.0;
        for (int i = 0; i < 2; ++i) {
            out[i] *= acc[i];
            sum += out[i];
        }
        if (sum > 0.0) {
            for (double& x : out) x /= sum;
        }
        for (double& x : out) x = double(float(x));
        return out;
    }
    bool vstatus(const Property& b, const Property& a) const {
        return std::fabs(b[0] - a[0]) + std::fabs(b[1] - a[1]) > epsilon;
    }
    bool estatus(double influence, double theta) const { return influence > theta; }
    bool valid(const Property& p) const {
        return std::isfinite(p[0]) && std::isfinite(p[1]);
    }
};

// test_engine.cpp:23-50
struct PoisonProgram {
    using Property = double;
    gg::VertexId poison_vertex = 2;
    int poison_iteration = 3;
    mutable std::atomic<int> applies_of_poison{0};
    PoisonProgram(gg::VertexId v, int it) : poison_vertex(v), poison_iteration(it) {}
    PoisonProgram(const PoisonProgram& o)
        : poison_vertex(o.poison_vertex), poison_iteration(o.poison_iteration) {}
    Property init_property(gg::VertexId, std::size_t) const { return 1.0; }
    Property gather_identity() const { return 0.0; }
    double gather(Property& acc, const Property& src, double, std::uint32_t) const {
        acc += src;
        return 0.0;
    }
    Property apply(gg::VertexId v, const Property& acc, const Property& prev,
                   std::size_t) const {
        if (v == poison_vertex && ++applies_of_poison == poison_iteration) {
            return std::numeric_limits<double>::quiet_NaN();
        }
        return prev + acc * 1e-6;
    }
    bool vstatus(const Property&, const Property&) const { return true; }
    bool estatus(double influence, double theta) const { return influence > theta; }
    bool valid(const Property& p) const { return !std::isnan(p); }
};

gg::Graph make_graph(std::uint64_t n, std::uint64_t e, const std::uint64_t* off,
                     const std::uint32_t* src, const double* w) {
    gg::Graph g;
    g.in_offsets.assign(off, off + n + 1);
    g.in_sources.assign(src, src + e);
    if (w) g.weights.assign(w, w + e);
    g.out_degree.assign(n, 0);
    for (std::uint64_t i = 0; i < e; ++i) ++g.out_degree[src[i]];
    return g;
}

void copy_msg(char* msg, std::size_t cap, const char* text) {
    if (msg && cap) {
        std::strncpy(msg, text, cap - 1);
        msg[cap - 1] = 0;
    }
}

}  // namespace

extern "C" {

struct ref_config {
    int scheme;
    double sigma, theta;
    std::uint64_t alpha, max_iterations, seed;
    std::uint32_t threads;
};
struct ref_params {
    double damping, epsilon;
    std::uint32_t source;
    int graded;
    int states;
    double coupling;
    const float* prior_table;
    std::uint32_t poison_vertex;
    int poison_iteration;
};
struct ref_record {
    std::int32_t mode;
    std::uint64_t processed_edges, active_vertices;
    double wall_seconds;
};
struct ref_summary {
    std::uint64_t iterations_run, total_processed_edges;
    std::uint64_t err_iteration;
    std::uint32_t err_vertex;
    double total_wall_seconds;
};

// A reference gg::Graph held across calls (so that big graphs are copied once).
void* ref_graph_create(std::uint64_t n, std::uint64_t e, const std::uint64_t* off,
                       const std::uint32_t* src, const double* w) {
    return new gg::Graph(make_graph(n, e, off, src, w));
}
void ref_graph_destroy(void* g) { delete static_cast<gg::Graph*>(g); }

// Runs the reference gg::run. prog: 0 pr, 1 sssp, 2 wcc, 3 bp, 4 bp_edge,
// 5 poison. Return: 0 ok, 1 std::invalid_argument, 2 gg::EngineError, 3 other.
int ref_run(const void* graph, int prog, const ref_params* p, const ref_config* c,
            void* out_props, ref_record* recs, std::uint64_t cap, ref_summary* sum,
            std::uint8_t* out_flags, char* msg, std::size_t msg_cap) {
    const gg::Graph& g = *static_cast<const gg::Graph*>(graph);
    std::memset(sum, 0, sizeof(*sum));
    gg::EngineConfig cfg;
    cfg.scheme = static_cast<gg::Scheme>(c->scheme);
    cfg.sigma = c->sigma;
    cfg.theta = c->theta;
    cfg.alpha = c->alpha;
    cfg.max_iterations = c->max_iterations;
    cfg.seed = c->seed;
    cfg.threads = c->threads;
    auto fill = [&](const auto& report, auto&& store) {
        sum->iterations_run = report.iterations_run;
        sum->total_processed_edges = report.total_processed_edges;
        sum->total_wall_seconds = report.total_wall_seconds;
        for (std::size_t i = 0; i < report.per_iteration.size() && i < cap; ++i) {
            recs[i].mode = static_cast<int>(report.per_iteration[i].mode);
            recs[i].processed_edges = report.per_iteration[i].processed_edges;
            recs[i].active_vertices = report.per_iteration[i].active_vertices;
            recs[i].wall_seconds = report.per_iteration[i].wall_seconds;
        }
        if (out_props) {
            for (std::size_t v = 0; v < report.final_properties.size(); ++v) {
                store(v, report.final_properties[v]);
            }
        }
    };
    try {
        switch (prog) {
            case 0: {
                auto r = gg::run(g, gg::pagerank_spec(p->damping, p->epsilon), cfg);
                fill(r, [&](std::size_t v, double x) { static_cast<double*>(out_props)[v] = x; });
                break;
            }
            case 1: {
                auto r = gg::run(g, gg::sssp_spec(p->source, p->graded != 0), cfg);
                fill(r, [&](std::size_t v, double x) { static_cast<double*>(out_props)[v] = x; });
                break;
            }
            case 2: {
                auto r = gg::run(g, gg::wcc_spec(), cfg);
                fill(r, [&](std::size_t v, gg::VertexId x) {
                    static_cast<std::uint32_t*>(out_props)[v] = x;
                });
                break;
            }
            case 3: {
                auto r = gg::run(g, gg::bp_spec(p->states, p->coupling, p->epsilon), cfg);
                fill(r, [&](std::size_t v, const std::vector<double>& x) {
                    for (int i = 0; i < p->states; ++i)
                        static_cast<double*>(out_props)[v * p->states + i] = x[i];
                });
                break;
            }
            case 4: {
                BpEdgeProgram prog4{p->prior_table, p->epsilon};
                auto r = gg::run(g, prog4, cfg);
                fill(r, [&](std::size_t v, const std::array<double, 2>& x) {
                    static_cast<double*>(out_props)[2 * v] = x[0];
                    static_cast<double*>(out_props)[2 * v + 1] = x[1];
                });
                break;
            }
            case 5: {
                PoisonProgram prog5(p->poison_vertex, p->poison_iteration);
                auto r = gg::run(g, prog5, cfg);
                fill(r, [&](std::size_t v, double x) { static_cast<double*>(out_props)[v] = x; });
                break;
            }
            default:
                copy_msg(msg, msg_cap, "unknown program");
                return 3;
        }
    } catch (const gg::EngineError& e) {
        sum->err_iteration = e.iteration();
        sum->err_vertex = e.vertex();
        copy_msg(msg, msg_cap, e.what());
        return 2;
    } catch (const std::invalid_argument& e) {
        copy_msg(msg, msg_cap, e.what());
        return 1;
    } catch (const std::exception& e) {
        copy_msg(msg, msg_cap, e.what());
        return 3;
    }
    // Final flags are engine-internal in the reference; reproduce them from
    // the reference's own sparsify() only when asked for the initial mask.
    (void)out_flags;
    return 0;
}

// GGCSR1 files through the reference's own writer / reader (graph.cpp:259-300).
int ref_write_binary(const void* graph, const char* path, char* msg, std::size_t msg_cap) {
    try {
        gg::write_binary(*static_cast<const gg::Graph*>(graph), path);
        return 0;
    } catch (const std::exception& e) {
        copy_msg(msg, msg_cap, e.what());
        return 1;
    }
}

void* ref_read_binary(const char* path, std::uint64_t* n, std::uint64_t* e, char* msg,
                      std::size_t msg_cap) {
    try {
        auto* g = new gg::Graph(gg::read_binary(path));
        *n = g->num_vertices();
        *e = g->num_edges();
        return g;
    } catch (const std::exception& ex) {
        copy_msg(msg, msg_cap, ex.what());
        return nullptr;
    }
}

int ref_sparsify(const void* graph, double sigma, std::uint64_t seed, std::uint8_t* out) {
    try {
        gg::EdgeFlags f = gg::sparsify(*static_cast<const gg::Graph*>(graph), sigma, seed);
        std::memcpy(out, f.data(), f.size());
        return 0;
    } catch (const std::invalid_argument&) {
        return 1;
    }
}

int ref_mode_for(int scheme, std::uint64_t t, std::uint64_t alpha) {
    return static_cast<int>(gg::mode_for(static_cast<gg::Scheme>(scheme), t, alpha));
}

std::uint64_t ref_supersteps(std::uint64_t alpha, std::uint64_t max_it, int scheme,
                             std::uint64_t* out, std::uint64_t cap) {
    auto v = gg::select_superstep_iterations(alpha, max_it, static_cast<gg::Scheme>(scheme));
    for (std::size_t i = 0; i < v.size() && i < cap; ++i) out[i] = v[i];
    return v.size();
}

// Graph export: the reference generators, for pinning the oracle's copies.
static void* export_graph(const gg::Graph& g, std::uint64_t* n, std::uint64_t* e) {
    *n = g.num_vertices();
    *e = g.num_edges();
    return new gg::Graph(g);
}
void* ref_generate_dumbbell(std::uint64_t k, std::uint64_t* n, std::uint64_t* e) {
    return export_graph(gg::generate_dumbbell(k), n, e);
}
void* ref_generate_power_law(std::uint64_t nv, double avg, double ex, std::uint64_t seed,
                             std::uint64_t* n, std::uint64_t* e) {
    return export_graph(gg::generate_power_law(nv, avg, ex, seed), n, e);
}
void* ref_symmetrized(const void* graph, std::uint64_t* n, std::uint64_t* e) {
    return export_graph(gg::symmetrized(*static_cast<const gg::Graph*>(graph)), n, e);
}
void ref_graph_arrays(const void* graph, std::uint64_t* off, std::uint32_t* src,
                      double* w, std::uint32_t* outdeg) {
    const gg::Graph& g = *static_cast<const gg::Graph*>(graph);
    std::memcpy(off, g.in_offsets.data(), g.in_offsets.size() * 8);
    std::memcpy(src, g.in_sources.data(), g.in_sources.size() * 4);
    if (w && g.weighted()) std::memcpy(w, g.weights.data(), g.weights.size() * 8);
    std::memcpy(outdeg, g.out_degree.data(), g.out_degree.size() * 4);
}
int ref_graph_weighted(const void* graph) {
    return static_cast<const gg::Graph*>(graph)->weighted() ? 1 : 0;
}

// metrics.cpp; which: 0 topk, 1 relative, 2 stretch. Returns 0 / 1 on error.
int ref_metric(int which, const double* approx, const double* exact, std::uint64_t n,
               std::uint64_t k, double* err) {
    try {
        std::span<const double> a(approx, n), x(exact, n);
        gg::ErrorReport r = which == 0   ? gg::topk_error(a, x, k)
                            : which == 1 ? gg::relative_error(a, x)
                                         : gg::stretch_error(a, x);
        *err = r.error;
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// bench.cpp run_sweep + emit_csv for golden comparison. schemes: bitmask of
// {1 sp, 2 sms, 4 gg}. Returns bytes written (or -1).
long ref_sweep_csv(const void* graph, const char* label, int algo, int schemes,
                   const double* sigmas, int n_sigma, const double* thetas, int n_theta,
                   const std::uint64_t* alphas, int n_alpha, std::uint64_t iterations,
                   int repeats, const std::uint64_t* seeds, int n_seeds,
                   std::uint32_t sssp_source, int sssp_graded, double epsilon,
                   char* out, std::size_t cap) {
    try {
        gg::SweepPlan plan;
        plan.algo = static_cast<gg::Algo>(algo);
        plan.graph = *static_cast<const gg::Graph*>(graph);
        plan.graph_label = label;
        plan.schemes.clear();
        if (schemes & 1) plan.schemes.push_back(gg::Scheme::sp);
        if (schemes & 2) plan.schemes.push_back(gg::Scheme::sms);
        if (schemes & 4) plan.schemes.push_back(gg::Scheme::gg);
        plan.sigma_grid.assign(sigmas, sigmas + n_sigma);
        plan.theta_grid.assign(thetas, thetas + n_theta);
        plan.alpha_grid.assign(alphas, alphas + n_alpha);
        plan.iterations = iterations;
        plan.repeats = repeats;
        plan.seeds.assign(seeds, seeds + n_seeds);
        plan.sssp_source = sssp_source;
        plan.sssp_graded = sssp_graded != 0;
        plan.epsilon = epsilon;
        std::ostringstream os;
        gg::emit_csv(gg::run_sweep(plan), plan, os);
        const std::string s = os.str();
        if (s.size() + 1 > cap) return -1;
        std::memcpy(out, s.c_str(), s.size() + 1);
        return static_cast<long>(s.size());
    } catch (const std::exception&) {
        return -1;
    }
}

}  // extern "C"
