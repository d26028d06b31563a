/*
 * ggb.h — C ABI of the B200-native GraphGuess engine (libggb.so).
 *
 * Drop-in boundary for the reference's hot path:
 *   template <VertexProgram A> RunReport<P> gg::run(const Graph&, const A&,
 *                                                  const EngineConfig&)
 *   (/root/reference/proj/core/include/gg/engine.hpp:141-143)
 * with the four reference programs (algorithms.hpp:15-151) compiled as device
 * programs. Plain pointers and sizes only; no torch / C++ types.
 *
 * Every entry returns a gg_status. Errors mirror the reference's exceptions:
 *   GG_INVALID_ARGUMENT  <- std::invalid_argument (engine.cpp:45-61,
 *                           algorithms.hpp:55-57); err->msg names the field
 *   GG_INVALID_PROPERTY  <- gg::EngineError(iteration, vertex)
 *                           (engine.hpp:60-74); err->iteration / err->vertex
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry returns GG_CUDA.
 */
#ifndef GGB_H
#define GGB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GGB_ABI_VERSION 5

typedef enum gg_status {
    GG_OK = 0,
    GG_INVALID_ARGUMENT = 1,
    GG_INVALID_PROPERTY = 2,
    GG_CUDA = 3,
    GG_NCCL = 4,
    GG_OOM = 5,
    GG_INTERNAL = 6
} gg_status;

/* Schemes and iteration modes: same integer values as gg::Scheme /
 * gg::IterationMode (engine.hpp:19, :24). */
typedef enum gg_scheme { GG_SCHEME_ACCURATE = 0, GG_SCHEME_SP = 1, GG_SCHEME_SMS = 2, GG_SCHEME_GG = 3 } gg_scheme;
typedef enum gg_mode { GG_MODE_APPROXIMATE = 0, GG_MODE_ACCURATE = 1, GG_MODE_SUPERSTEP = 2 } gg_mode;

/* Edge weight storage (gg::Graph::weights is f64 or empty, graph.hpp:32). */
typedef enum gg_weight_kind { GG_W_NONE = 0, GG_W_U32 = 1, GG_W_F32 = 2, GG_W_F64 = 3 } gg_weight_kind;

/* Host pull-CSC view, borrowed for the call (gg::Graph, graph.hpp:29-49). */
typedef struct gg_csc_view {
    uint64_t n;                 /* vertices */
    uint64_t e;                 /* edges */
    const uint64_t* offsets;    /* n+1, offsets[0] == 0, offsets[n] == e */
    const uint32_t* sources;    /* e; edge id = position */
    gg_weight_kind weight_kind;
    const void* weights;        /* e elements of weight_kind, or NULL */
    const uint32_t* out_degree; /* n (trusted: gg::Graph's invariant), or NULL: counted on the
                                   host from the sources. Sources >= n and decreasing offsets
                                   fail creation either way (checked on the device). */
} gg_csc_view;

/* Placement: one process per GPU. nranks == 1 -> single GPU. For nranks > 1
 * the destination range is 1-D partitioned (edge balanced, 32-vertex aligned)
 * and gg_exchange carries the per-iteration property exchange. */
typedef struct gg_part_opts {
    int device;                 /* CUDA ordinal, -1 = current */
    int rank, nranks;
    void* exchange;             /* gg_exchange* (from gg_exchange_nccl_create) or NULL */
} gg_part_opts;

typedef struct gg_dev_graph gg_dev_graph;
typedef struct gg_exchange gg_exchange;

/* Mirrors gg::EngineConfig (engine.hpp:28-36). threads is validated (>= 1)
 * like the reference and otherwise ignored (the device grid replaces it). */
typedef struct gg_engine_config {
    int32_t scheme;
    double sigma;
    double theta;
    uint64_t alpha;
    uint64_t max_iterations;
    uint64_t seed;
    uint32_t threads;
} gg_engine_config;

/* Mirrors gg::IterationRecord (engine.hpp:42-47) plus device evidence. */
typedef struct gg_iter_record {
    int32_t mode;
    uint64_t processed_edges;
    uint64_t active_vertices;
    double wall_seconds;        /* host wall time of the iteration */
    double kernel_ms;           /* CUDA-event time of the gather step (edge + vertex kernels) */
    double rebuild_ms;          /* CUDA-event time of the sparse rebuild (supersteps) */
    double exchange_ms;         /* multi-GPU exchange time (0 for 1 GPU) */
    uint64_t algo_bytes;        /* algorithmic HBM bytes of the gather step */
    double edge_ms;             /* edge kernel (+ superstep pass 2) */
    double vertex_ms;           /* vertex epilogue kernel */
    uint64_t edge_bytes;        /* algorithmic bytes of the edge kernel: E_p * b_e */
    uint64_t vertex_bytes;      /* algorithmic bytes of the vertex kernel: N * b_v */
} gg_iter_record;

typedef struct gg_run_summary {
    uint64_t iterations_run;
    uint64_t total_processed_edges;
    double total_wall_seconds;
    uint64_t kept_edges;        /* active edges after the run (flag popcount) */
    uint32_t kernel_launches;   /* our kernels launched by this run */
    uint32_t exchange_fused;    /* several ranks: 1 = messages stored into the peer replicas
                                   by the vertex kernel, 0 = all-gathered after it */
} gg_run_summary;

typedef struct gg_error {
    uint64_t iteration;
    uint32_t vertex;
    char msg[256];
} gg_error;

/* Optional run outputs / instrumentation. */
typedef struct gg_run_opts {
    uint32_t* out_flags;        /* host bitmap, ceil(e/32) words, final active-edge flags (nullable) */
    int timing;                 /* 1: CUDA-event timing of every kernel into records */
    int device_output;          /* 1: leave properties on device (out_props may be NULL) */
    uint32_t grid_ctas;         /* test hook: cap on the CTAs of every engine launch (0 = the
                                   occupancy-sized default); results must not depend on it */
} gg_run_opts;

/* Program parameters (algorithms.hpp). */
typedef struct gg_pr_params { double damping; double epsilon; } gg_pr_params;      /* :15-40 */
typedef struct gg_sssp_params { uint32_t source; int32_t graded; } gg_sssp_params; /* :46-83 */
typedef struct gg_bp_params {                                                      /* :120-145 */
    int32_t states;             /* 2..64 (2..4 compile-time programs, 5..64 run-time S) */
    double coupling;            /* global coupling (reference BP) */
    double epsilon;
    /* BASELINE C4 extension: when prior_table != NULL the prior comes from the
     * table (float[n*2]), the coupling from each edge's weight, and beliefs
     * are stored as fp32 (states must be 2). */
    const float* prior_table;
    int32_t prior_on_device;    /* 1: prior_table is device memory (no per-run copy) */
} gg_bp_params;

const char* gg_status_string(gg_status s);
int gg_abi_version(void);

/* Graph residency. */
gg_status gg_dev_graph_create(const gg_csc_view* csc, const gg_part_opts* opts,
                              gg_dev_graph** out, gg_error* err);
/* gg_dev_graph_create for one coming sparse-scheme run (sp / sms / gg): the
   run's initial sparsification (engine.cpp:63-75 with this sigma and seed)
   and the compaction of the kept edges proceed chunk by chunk while the
   sources are still being uploaded (one rank, at least 2^24 edges; otherwise
   a plain create). The next gg_run_* with the same sigma and seed uses that
   list instead of sparsifying; any run clears it. Host arrays are borrowed
   for the call only. This is what the drop-in gg::run(Graph, ...) path uses. */
gg_status gg_dev_graph_create_for_run(const gg_csc_view* csc, const gg_part_opts* opts,
                                      double sigma, uint64_t seed, gg_dev_graph** out,
                                      gg_error* err);
gg_status gg_dev_graph_destroy(gg_dev_graph* g);
gg_status gg_dev_graph_info(const gg_dev_graph* g, uint64_t* n, uint64_t* e,
                            uint64_t* v_begin, uint64_t* v_end, uint64_t* e_local);

/* R-MAT generated straight into HBM (a/b/c/d quadrant probabilities, no
 * noise, no permutation, self-loops and duplicates removed, CSC by (dst,src)).
 * symmetrize: reference symmetrized() order (graph.cpp:249-257).
 * weight_kind GG_W_U32: 1 + mix64(kw ^ e) % 255;  GG_W_F32: BP couplings. */
typedef struct gg_rmat_params {
    uint32_t scale, edge_factor;
    uint64_t seed;
    double a, b, c;
    int32_t symmetrize;
    gg_weight_kind weight_kind;
} gg_rmat_params;
gg_status gg_dev_graph_create_rmat(const gg_rmat_params* p, const gg_part_opts* opts,
                                   gg_dev_graph** out, gg_error* err);
/* Copy the (full, single-rank) CSC back to host buffers (any may be NULL). */
/* graph.cpp:249-257 symmetrized() of a resident single-rank graph, built on
 * the device (per destination: its in-edges in order, then its out-edges in
 * ascending original destination; weights carried); opts may be NULL (same
 * device, one rank) or place / partition the result like gg_dev_graph_create. */
gg_status gg_dev_graph_symmetrized(const gg_dev_graph* g, const gg_part_opts* opts,
                                   gg_dev_graph** out, gg_error* err);
gg_status gg_dev_graph_export(const gg_dev_graph* g, uint64_t* offsets, uint32_t* sources,
                              void* weights, uint32_t* out_degree);
/* Binary CSC files straight to HBM (graph.cpp:259-300). Reads the
 * reference's GGCSR1 (u64 sources) and GGCSR2 (u32 sources, weight kind,
 * stored out-degrees); errors name the file like read_binary. Save writes
 * GGCSR2 from a single-rank graph. */
gg_status gg_dev_graph_load(const char* path, const gg_part_opts* opts, gg_dev_graph** out,
                            gg_error* err);
gg_status gg_dev_graph_save(const gg_dev_graph* g, const char* path, gg_error* err);
/* Weight storage of a resident graph (gg_weight_kind), -1 for a null graph. */
int32_t gg_dev_graph_weight_kind(const gg_dev_graph* g);
/* BASELINE C4 priors generated on device (float[2n]); copied to host if out != NULL. */
gg_status gg_bp_priors(uint64_t n, uint64_t seed, float* out);
/* ... or left in device memory (*dev_out, free with gg_device_free). */
gg_status gg_bp_priors_device(uint64_t n, uint64_t seed, float** dev_out);
/* Device copy of a host buffer (e.g. a caller's prior table kept resident
 * across runs); free with gg_device_free. */
gg_status gg_device_upload(const void* host, uint64_t bytes, void** dev_out);
gg_status gg_device_free(void* dev);

/* Runs (engine.hpp:141-249). out_props: host buffer of n * prop_size
 * (pr/sssp: double; wcc: uint32; bp: double[states]). recs: rec_cap
 * records (iterations beyond rec_cap are run but not recorded). */
gg_status gg_run_pr(gg_dev_graph* g, const gg_engine_config* cfg, const gg_pr_params* p,
                    double* out_props, gg_iter_record* recs, uint64_t rec_cap,
                    gg_run_summary* out, const gg_run_opts* opts, gg_error* err);
gg_status gg_run_sssp(gg_dev_graph* g, const gg_engine_config* cfg, const gg_sssp_params* p,
                      double* out_props, gg_iter_record* recs, uint64_t rec_cap,
                      gg_run_summary* out, const gg_run_opts* opts, gg_error* err);
gg_status gg_run_wcc(gg_dev_graph* g, const gg_engine_config* cfg,
                     uint32_t* out_props, gg_iter_record* recs, uint64_t rec_cap,
                     gg_run_summary* out, const gg_run_opts* opts, gg_error* err);
gg_status gg_run_bp(gg_dev_graph* g, const gg_engine_config* cfg, const gg_bp_params* p,
                    double* out_props, gg_iter_record* recs, uint64_t rec_cap,
                    gg_run_summary* out, const gg_run_opts* opts, gg_error* err);

/* Engine pieces, exposed for parity tests (engine.cpp:63-107). */
gg_status gg_validate(const gg_engine_config* cfg, gg_error* err);
int32_t gg_mode_for(int32_t scheme, uint64_t t, uint64_t alpha);
uint64_t gg_select_superstep_iterations(uint64_t alpha, uint64_t max_iterations,
                                        int32_t scheme, uint64_t* out, uint64_t cap);
/* Device sparsify of edge ids [0, e) into a host bitmap (ceil(e/32) words). */
gg_status gg_sparsify(uint64_t e, double sigma, uint64_t seed, uint32_t* out_bitmap,
                      gg_error* err);

/* Partition plan: 32-aligned, edge-balanced destination ranges
 * (bounds[nranks+1]); pure host logic. */
gg_status gg_partition_plan(uint64_t n, const uint64_t* offsets, int nranks, uint64_t* bounds);

/* Multi-GPU exchange over NCCL (dlopen'ed libnccl.so.2). unique_id is the
 * 128-byte ncclUniqueId made by rank 0 (gg_nccl_unique_id) and broadcast by
 * the caller. */
gg_status gg_nccl_unique_id(uint8_t out[128]);
gg_status gg_exchange_nccl_create(const uint8_t unique_id[128], int rank, int nranks,
                                  gg_exchange** out, gg_error* err);
/* In-process transport: nranks handles (out[nranks]) for ranks that are host
 * threads of ONE process, each with its own graph and stream, on any devices
 * (one GPU may host them all). Same engine code path as NCCL; collectives are
 * host barriers + device copies. For single-GPU validation of the partitioned
 * engine and for multi-tenant hosts. Destroy each handle. */
gg_status gg_exchange_local_group(int nranks, gg_exchange** out);
/* Fused exchange on (default) or off. On: the vertex kernel stores every new
 * message into each rank's replica (peer memory over NVLink; CUDA IPC maps the
 * replicas of the NCCL transport), with one barrier per iteration between the
 * gathers and the vertex kernels. Off, or when some rank cannot map its peers:
 * the messages are all-gathered after the vertex kernel (grouped
 * ncclBroadcast). Set the same value on every rank before a run. */
gg_status gg_exchange_set_fused(gg_exchange* x, int on);
/* Transport health check (collective: every rank calls it). Over NCCL it
 * all-gathers ragged rank slices with the engine's grouped ncclBroadcast,
 * sum- and max-all-reduces rank vectors and compares the results with their
 * closed forms; GG_NCCL with a message on any difference. A one-rank
 * communicator is valid (runs the same calls). Call it with the
 * communicator's device current (the one current at gg_exchange_nccl_create).
 * No-op for the in-process transport. */
gg_status gg_exchange_selftest(gg_exchange* x, gg_error* err);
gg_status gg_exchange_destroy(gg_exchange* x);

/* Host metrics (metrics.cpp:60-113); accuracy = (1 - err) * 100. */
gg_status gg_topk_error(const double* approx, const double* exact, uint64_t n, uint64_t k,
                        double* err_out);
gg_status gg_relative_error(const double* approx, const double* exact, uint64_t n,
                            double* err_out);
gg_status gg_stretch_error(const double* approx, const double* exact, uint64_t n,
                           double* err_out);

/* The same metrics on DEVICE arrays (e.g. gg_last_projection of an exact and
 * an approximate run): only the scalar returns to the host. top-k is exact;
 * the two means are reduced in a fixed order (deterministic; equal to the
 * reference's left-to-right sum up to rounding). stretch: a vertex with
 * approx < exact returns GG_INVALID_ARGUMENT with err->vertex set. */
gg_status gg_topk_error_dev(const double* approx, const double* exact, uint64_t n, uint64_t k,
                            double* err_out);
gg_status gg_relative_error_dev(const double* approx, const double* exact, uint64_t n,
                                double* err_out);
gg_status gg_stretch_error_dev(const double* approx, const double* exact, uint64_t n,
                               double* err_out, gg_error* err);
/* double[n] device projection of the graph's last run (PR rank, SSSP
 * distance with +inf for unreached, WCC label, BP belief[0]); valid until the
 * next run on this graph. Copy it (gg_device_copy) to keep it. */
gg_status gg_last_projection(gg_dev_graph* g, const double** dev_out);
gg_status gg_device_copy(const void* dev_src, uint64_t bytes, void** dev_out);

#ifdef __cplusplus
}
#endif
#endif /* GGB_H */
