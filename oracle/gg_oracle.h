/*
 * gg_oracle.h — CPU ORACLE. TEST INFRASTRUCTURE ONLY.
 *
 * This is a plain-C restatement of the GraphGuess reference engine
 * (/root/reference/proj/core, C++20 + OpenMP) used as the CHECKER for the
 * B200 product in paper_2104_10039_b200/. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The
 * product never links, calls or falls back to anything in oracle/.
 *
 * Parity pinning: tests/test_oracle_pins.py checks this restatement against
 *   (1) the reference's own known-answer tests (test_engine.cpp,
 *       test_algorithms.cpp, acceptance_main.cpp, golden_dumbbell4.csv), and
 *   (2) the reference itself, compiled from its own sources by
 *       oracle/Makefile into oracle/_ref/libggref.so (when /root/reference is
 *       present), on many seeded graphs, bit for bit.
 */
#ifndef GG_ORACLE_H
#define GG_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Pull CSC, mirrors gg::Graph (graph.hpp:29-49). Edge id = position in src. */
typedef struct og_graph {
    uint64_t n, e;
    uint64_t* off;     /* n+1 */
    uint32_t* src;     /* e */
    double* w;         /* e, or NULL when unweighted */
    uint32_t* outdeg;  /* n */
} og_graph;

/* Schemes / modes: engine.hpp:19, :24 (same integer order). */
enum { OG_ACCURATE = 0, OG_SP = 1, OG_SMS = 2, OG_GG = 3 };
enum { OG_MODE_APPROXIMATE = 0, OG_MODE_ACCURATE = 1, OG_MODE_SUPERSTEP = 2 };

/* Programs. PR/SSSP/WCC/BP are the reference programs (algorithms.hpp);
 * BP_EDGE is the BASELINE C4 extension (per-edge coupling = edge weight,
 * table priors, fp32 storage of beliefs); POISON is test_engine.cpp:23-50. */
enum { OG_PR = 0, OG_SSSP = 1, OG_WCC = 2, OG_BP = 3, OG_BP_EDGE = 4, OG_POISON = 5 };

typedef struct og_config { /* engine.hpp:28-36 */
    int scheme;
    double sigma, theta;
    uint64_t alpha, max_iterations, seed;
    uint32_t threads;
} og_config;

typedef struct og_params {
    double damping, epsilon;      /* PR (algorithms.hpp:18-19), BP epsilon */
    uint32_t source; int graded;  /* SSSP (algorithms.hpp:49-50) */
    int states; double coupling;  /* BP (algorithms.hpp:123-125) */
    const float* prior_table;     /* BP_EDGE: float[2*n] */
    uint32_t poison_vertex; int poison_iteration; /* POISON */
} og_params;

typedef struct og_record { /* engine.hpp:42-47 (wall time omitted: not compared) */
    int32_t mode;
    uint64_t processed_edges, active_vertices;
} og_record;

typedef struct og_summary {
    uint64_t iterations_run, total_processed_edges;
    uint64_t err_iteration; uint32_t err_vertex;
} og_summary;

/* status codes */
enum { OG_OK = 0, OG_INVALID_ARGUMENT = 1, OG_INVALID_PROPERTY = 2, OG_ERROR = 3 };

uint64_t og_mix64(uint64_t x);
double og_to_unit(uint64_t h);

/* graph construction (graph.cpp) */
og_graph* og_build_graph(uint64_t n, uint64_t m, const uint32_t* esrc,
                         const uint32_t* edst, const double* ew);
og_graph* og_from_csc(uint64_t n, uint64_t e, const uint64_t* off,
                      const uint32_t* src, const double* w);
void og_free_graph(og_graph* g);
og_graph* og_generate_dumbbell(uint64_t k);
og_graph* og_generate_power_law(uint64_t n, double avg_degree, double exponent,
                                uint64_t seed);
og_graph* og_random_graph(uint64_t n, uint64_t m, uint64_t seed, int weighted);
og_graph* og_symmetrized(const og_graph* g);
og_graph* og_reverse(const og_graph* g);

/* R-MAT input layer shared (by specification) with the GPU generator. */
og_graph* og_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed,
                  double a, double b, double c, int threads);
void og_rmat_weights_u32(uint64_t e, uint64_t seed, uint32_t* out);
void og_bp_priors(uint64_t n, uint64_t seed, float* out /* 2n */);
void og_bp_couplings(uint64_t e, uint64_t seed, float* out);
uint32_t og_max_outdeg_vertex(const og_graph* g);

/* engine pieces (engine.cpp) */
int og_validate(const og_config* cfg, char* msg, size_t cap);
int og_sparsify(uint64_t e, double sigma, uint64_t seed, uint8_t* flags);
int og_mode_for(int scheme, uint64_t t, uint64_t alpha);
uint64_t og_supersteps(uint64_t alpha, uint64_t max_iterations, int scheme,
                       uint64_t* out, uint64_t cap);

/* gg::run restatement (engine.hpp:141-249). out_props layout: PR/SSSP/
 * POISON double[n]; WCC uint32[n]; BP double[n*states]; BP_EDGE double[2n].
 * out_flags (nullable): final per-edge flag bytes. */
int og_run(const og_graph* g, int prog, const og_params* params,
           const og_config* cfg, void* out_props, og_record* recs,
           uint64_t rec_cap, og_summary* sum, uint8_t* out_flags,
           char* msg, size_t msg_cap);

/* Lock-step comparison with the device's superstep flags (og_run_ex).
 * An edge is NEAR-THRESHOLD when |infl - theta| <= band with
 *   band = tol_unit * ((k + 4) * max(|infl|, theta) + 4),
 * k = the edge's position in its vertex's in-list (the number of gathers
 * folded before it). tol_unit is the program's rounding unit (times a
 * safety factor): it bounds how far a re-associated prefix accumulator (the
 * device joins 16-edge runs, engine.hpp:198-211 folds left to right) can
 * move the influence; 0 for the min programs (SSSP, WCC), whose folds are
 * exact under any grouping (no edge is near-threshold then: an exact tie
 * with theta is decided identically on both sides). */
typedef struct og_lockstep {
    const uint32_t* const* dev_bitmaps; /* [n_dev]: device flags right after superstep s (bit e of word e/32), NULL = none */
    uint64_t n_dev;
    double tol_unit;
    uint64_t* stats;      /* out, 4 per superstep: near-threshold edges, adopted (device differs, near), real (device differs, not near), kept */
    uint64_t stats_cap;   /* supersteps the stats array holds */
    uint64_t n_supersteps; /* out: supersteps run */
} og_lockstep;

int og_run_ex(const og_graph* g, int prog, const og_params* params,
              const og_config* cfg, void* out_props, og_record* recs,
              uint64_t rec_cap, og_summary* sum, uint8_t* out_flags,
              char* msg, size_t msg_cap, og_lockstep* ls);

/* Per-edge influences of destinations [v_begin, v_end) folded over their
 * full in-lists from prev (the superstep fold, engine.hpp:198-211). */
int og_influences(const og_graph* g, int prog, const og_params* params, const void* prev,
                  uint64_t v_begin, uint64_t v_end, int threads, double* out);

/* One iteration of engine.hpp:194-224 restricted to destinations
 * [v_begin, v_end) — the per-rank step of a destination partition (used by
 * the multi-rank protocol tests). prev/next/status/status_next/aid are
 * global-length arrays; only the owned range of next/status_next/aid/flags
 * is written. counters: [gathered, processed, changed, bad_vertex+1 (0 =
 * none; the smallest invalid owned vertex checked like :228-230)]. */
int og_step_range(const og_graph* g, int prog, const og_params* params, int mode, double theta,
                  uint8_t* flags, uint32_t* aid, const void* prev, const uint8_t* status,
                  void* next, uint8_t* status_next, uint64_t v_begin, uint64_t v_end,
                  uint64_t counters[4]);
/* Initial property of every vertex (engine.hpp:163-164) into out. */
int og_init_props(const og_graph* g, int prog, const og_params* params, void* out);

/* metrics.cpp */
int og_topk_error(const double* approx, const double* exact, uint64_t n,
                  uint64_t k, double* err);
int og_relative_error(const double* approx, const double* exact, uint64_t n,
                      double* err);
int og_stretch_error(const double* approx, const double* exact, uint64_t n,
                     double* err);

#ifdef __cplusplus
}
#endif
#endif
