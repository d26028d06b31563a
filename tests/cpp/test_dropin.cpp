// test_dropin.cpp — the C++ drop-in check (test infrastructure).
//
// Calls the UNMODIFIED reference engine gg::run (engine.hpp:141-249, linked
// from oracle/_ref/libggref.so, the reference compiled from its own sources)
// and ggb::run (include/ggb_gg.hpp -> libggb.so on the GPU) with the SAME
// gg::Graph, gg:: program and gg::EngineConfig objects, and checks:
//   * iterations_run, and per iteration mode / processed_edges / active_vertices;
//   * final properties: WCC and SSSP bit-exact, PR rel 1e-9, BP rel 1e-6;
//   * exceptions: std::invalid_argument with the same what(), gg::EngineError
//     with the same iteration and vertex;
//   * a resident ggb::DeviceGraph reused across runs gives identical reports.
// Modelled on test_engine.cpp / test_algorithms.cpp's cases (programs x
// schemes on generated graphs). Exit 0 = all cases pass.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "gg/algorithms.hpp"
#include "gg/engine.hpp"
#include "gg/graph.hpp"
#include "ggb_gg.hpp"

namespace {

int g_cases = 0, g_fail = 0;

void fail(const std::string& what) {
    ++g_fail;
    std::fprintf(stderr, "FAIL %s\n", what.c_str());
}

bool close(double a, double b, double rtol) {
    if (a == b) return true;  // covers +inf
    if (std::isnan(a) || std::isnan(b)) return false;
    return std::fabs(a - b) <= rtol * std::fmax(std::fabs(a), std::fabs(b));
}
bool close(std::uint32_t a, std::uint32_t b, double) { return a == b; }
bool close(const std::vector<double>& a, const std::vector<double>& b, double rtol) {
    if (a.size() != b.size()) return false;
    for (std::size_t i = 0; i < a.size(); ++i)
        if (!close(a[i], b[i], rtol)) return false;
    return true;
}

template <class P>
void compare(const std::string& name, const gg::RunReport<P>& ref, const gg::RunReport<P>& dev,
             double rtol) {
    ++g_cases;
    if (ref.iterations_run != dev.iterations_run) {
        fail(name + ": iterations_run " + std::to_string(ref.iterations_run) + " vs " +
             std::to_string(dev.iterations_run));
        return;
    }
    if (ref.per_iteration.size() != dev.per_iteration.size()) {
        fail(name + ": record count");
        return;
    }
    for (std::size_t t = 0; t < ref.per_iteration.size(); ++t) {
        const auto& a = ref.per_iteration[t];
        const auto& b = dev.per_iteration[t];
        if (a.mode != b.mode || a.processed_edges != b.processed_edges ||
            a.active_vertices != b.active_vertices) {
            fail(name + ": record " + std::to_string(t) + " (" + std::to_string(a.processed_edges) +
                 "," + std::to_string(a.active_vertices) + ") vs (" +
                 std::to_string(b.processed_edges) + "," + std::to_string(b.active_vertices) + ")");
            return;
        }
    }
    if (ref.total_processed_edges != dev.total_processed_edges) {
        fail(name + ": total_processed_edges");
        return;
    }
    if (ref.final_properties.size() != dev.final_properties.size()) {
        fail(name + ": property count");
        return;
    }
    for (std::size_t v = 0; v < ref.final_properties.size(); ++v) {
        if (!close(ref.final_properties[v], dev.final_properties[v], rtol)) {
            fail(name + ": property of vertex " + std::to_string(v));
            return;
        }
    }
}

gg::EngineConfig config(gg::Scheme s, double sigma, double theta, std::uint64_t alpha,
                        std::uint64_t max_it, std::uint64_t seed) {
    gg::EngineConfig c;
    c.scheme = s;
    c.sigma = sigma;
    c.theta = theta;
    c.alpha = alpha;
    c.max_iterations = max_it;
    c.seed = seed;
    c.threads = 4;
    return c;
}

const gg::Scheme kSchemes[] = {gg::Scheme::accurate, gg::Scheme::sp, gg::Scheme::sms, gg::Scheme::gg};

template <class A>
void all_schemes(const std::string& name, const gg::Graph& g, const ggb::DeviceGraph& dg,
                 const A& prog, double theta, double rtol, std::uint64_t max_it) {
    for (gg::Scheme s : kSchemes) {
        for (double sigma : {0.3, 0.7}) {
            const gg::EngineConfig c = config(s, sigma, theta, 2, max_it, 11);
            const std::string tag = name + "/" + gg::scheme_name(s) + "/sigma" + std::to_string(sigma);
            compare(tag, gg::run(g, prog, c), ggb::run(dg, prog, c), rtol);
            if (s == gg::Scheme::accurate) break;
        }
    }
}

// Integer-valued f64 weights in [1, 16], keyed by edge id.
gg::Graph with_weights(gg::Graph g) {
    g.weights.resize(g.num_edges());
    for (std::uint64_t e = 0; e < g.num_edges(); ++e)
        g.weights[e] = 1.0 + double((e * 2654435761ull >> 7) % 16);
    return g;
}

template <class F>
std::string what_of(F&& f) {
    try {
        f();
    } catch (const std::invalid_argument& e) {
        return std::string("invalid_argument: ") + e.what();
    } catch (const gg::EngineError& e) {
        return "EngineError " + std::to_string(e.iteration()) + " " + std::to_string(e.vertex());
    } catch (const std::exception& e) {
        return std::string("other: ") + e.what();
    }
    return "no exception";
}

void expect_same_error(const std::string& name, const std::string& ref, const std::string& dev) {
    ++g_cases;
    if (ref != dev || ref == "no exception") fail(name + ": [" + ref + "] vs [" + dev + "]");
}

}  // namespace

int main() {
    // Graphs from the reference's own generators (graph.hpp:88-106).
    const gg::Graph pl = gg::generate_power_law(3000, 8.0, 2.1, 7);
    const gg::Graph pl_big = gg::generate_power_law(60000, 12.0, 2.0, 9);
    const gg::Graph dumbbell = gg::generate_dumbbell(12);
    const gg::Graph sym = gg::symmetrized(pl);
    const gg::Graph wpl = with_weights(pl);

    const ggb::DeviceGraph d_pl = ggb::upload(pl);
    const ggb::DeviceGraph d_big = ggb::upload(pl_big);
    const ggb::DeviceGraph d_db = ggb::upload(dumbbell);
    const ggb::DeviceGraph d_sym = ggb::upload(sym);
    const ggb::DeviceGraph d_wpl = ggb::upload(wpl);

    const gg::PageRankProgram pr = gg::pagerank_spec(0.85, 1e-7);
    all_schemes("pr/power_law", pl, d_pl, pr, 0.01, 1e-9, 50);
    all_schemes("pr/power_law_60k", pl_big, d_big, pr, 0.01, 1e-9, 40);
    all_schemes("pr/dumbbell", dumbbell, d_db, pr, 0.05, 1e-9, 50);

    all_schemes("sssp/unweighted", pl, d_pl, gg::sssp_spec(0, false), 0.0, 0.0, 3001);
    all_schemes("sssp/weighted_graded", wpl, d_wpl, gg::sssp_spec(1, true), 0.05, 0.0, 3001);
    all_schemes("sssp/weighted", wpl, d_wpl, gg::sssp_spec(2, false), 0.0, 0.0, 3001);

    all_schemes("wcc/symmetrized", sym, d_sym, gg::wcc_spec(), 0.0, 0.0, 3001);
    all_schemes("wcc/dumbbell", dumbbell, d_db, gg::wcc_spec(), 0.0, 0.0, 25);

    all_schemes("bp2/power_law", pl, d_pl, gg::bp_spec(2, 0.8, 1e-6), 0.01, 1e-6, 30);
    all_schemes("bp3/power_law", pl, d_pl, gg::bp_spec(3, 0.7, 1e-6), 0.01, 1e-6, 30);
    all_schemes("bp6/power_law", pl, d_pl, gg::bp_spec(6, 0.6, 1e-6), 0.01, 1e-6, 30);

    // The reference signature (graph uploaded inside the call).
    {
        const gg::EngineConfig c = config(gg::Scheme::gg, 0.5, 0.01, 4, 50, 5);
        compare("pr/gg::Graph overload", gg::run(pl, pr, c), ggb::run(pl, pr, c), 1e-9);
    }
    // A resident graph reused across runs gives identical reports.
    {
        const gg::EngineConfig c = config(gg::Scheme::gg, 0.5, 0.01, 3, 50, 3);
        const auto a = ggb::run(d_big, pr, c);
        const auto b = ggb::run(d_big, pr, c);
        compare("pr/resident reuse", a, b, 0.0);
    }
    // Errors: std::invalid_argument naming the field (engine.cpp:45-61).
    {
        gg::EngineConfig c = config(gg::Scheme::gg, 1.5, 0.01, 4, 10, 1);
        expect_same_error("sigma", what_of([&] { gg::run(pl, pr, c); }),
                          what_of([&] { ggb::run(d_pl, pr, c); }));
        c = config(gg::Scheme::gg, 0.5, -1.0, 4, 10, 1);
        expect_same_error("theta", what_of([&] { gg::run(pl, pr, c); }),
                          what_of([&] { ggb::run(d_pl, pr, c); }));
        c = config(gg::Scheme::gg, 0.5, 0.0, 0, 10, 1);
        expect_same_error("alpha", what_of([&] { gg::run(pl, pr, c); }),
                          what_of([&] { ggb::run(d_pl, pr, c); }));
        c = config(gg::Scheme::gg, 0.5, 0.0, 1, 0, 1);
        expect_same_error("max_iterations", what_of([&] { gg::run(pl, pr, c); }),
                          what_of([&] { ggb::run(d_pl, pr, c); }));
        c = config(gg::Scheme::gg, 0.5, 0.0, 1, 10, 1);
        c.threads = 0;
        expect_same_error("threads", what_of([&] { gg::run(pl, pr, c); }),
                          what_of([&] { ggb::run(d_pl, pr, c); }));
        c.threads = 1;
        const gg::SsspProgram bad = gg::sssp_spec(1u << 30, false);
        expect_same_error("sssp source", what_of([&] { gg::run(pl, bad, c); }),
                          what_of([&] { ggb::run(d_pl, bad, c); }));
    }
    // gg::EngineError (engine.hpp:60-74): a negative edge weight makes SSSP
    // produce a negative distance, which SsspProgram::valid rejects.
    {
        gg::Graph neg = with_weights(dumbbell);
        neg.weights[neg.in_offsets[5]] = -100.0;
        const ggb::DeviceGraph d_neg = ggb::upload(neg);
        const gg::EngineConfig c = config(gg::Scheme::accurate, 1.0, 0.0, 1, 100, 0);
        const gg::SsspProgram sp = gg::sssp_spec(0, false);
        expect_same_error("EngineError", what_of([&] { gg::run(neg, sp, c); }),
                          what_of([&] { ggb::run(d_neg, sp, c); }));
    }

    std::printf("test_dropin: %d cases, %d failed\n", g_cases, g_fail);
    return g_fail == 0 ? 0 : 1;
}
