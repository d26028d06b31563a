/*
 * gg_oracle.c — CPU ORACLE (TEST INFRASTRUCTURE ONLY; see gg_oracle.h).
 *
 * Plain-C restatement of the GraphGuess reference path. Every function cites
 * the reference file:line it follows (paths relative to
 * /root/reference/proj/). Each vertex's fold is sequential in CSC order; the
 * vertex loop of an iteration (a Jacobi update) and the R-MAT input
 * generator run over OpenMP threads. The reference's results are
 * independent of its thread count (engine.hpp:139-140), so they are also
 * this restatement's for any thread count.
 */
#include "gg_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif
#include <stdint.h>

/* largest property (bytes) the run loops keep on the stack: BP up to 64 states */
#define OG_MAX_PSIZE 512

/* engine.cpp:9-14 (and graph.cpp:22-27, test_support.hpp:12-17) */
uint64_t og_mix64(uint64_t x) {
    x += 0x9e3779b97f4a7c15ull;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
    return x ^ (x >> 31);
}

/* graph.cpp:29-31 */
double og_to_unit(uint64_t h) { return (double)(h >> 11) * 0x1.0p-53; }

static void* xmalloc(size_t sz) {
    void* p = malloc(sz ? sz : 1);
    if (!p) { fprintf(stderr, "oracle: out of memory (%zu bytes)\n", sz); abort(); }
    return p;
}
static void* xcalloc(size_t n, size_t sz) {
    void* p = calloc(n ? n : 1, sz ? sz : 1);
    if (!p) { fprintf(stderr, "oracle: out of memory\n"); abort(); }
    return p;
}

void og_free_graph(og_graph* g) {
    if (!g) return;
    free(g->off); free(g->src); free(g->w); free(g->outdeg); free(g);
}

/* graph.cpp:102-124: counting pass, partial sum, stable scatter by dst. */
og_graph* og_build_graph(uint64_t n, uint64_t m, const uint32_t* esrc,
                         const uint32_t* edst, const double* ew) {
    og_graph* g = (og_graph*)xcalloc(1, sizeof(og_graph));
    g->n = n; g->e = m;
    g->off = (uint64_t*)xcalloc(n + 1, 8);
    g->outdeg = (uint32_t*)xcalloc(n, 4);
    for (uint64_t i = 0; i < m; ++i) {
        if (esrc[i] >= n || edst[i] >= n) { og_free_graph(g); return NULL; }
        g->off[edst[i] + 1]++;
        g->outdeg[esrc[i]]++;
    }
    for (uint64_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
    g->src = (uint32_t*)xmalloc(m * 4);
    g->w = ew ? (double*)xmalloc(m * 8) : NULL;
    uint64_t* cur = (uint64_t*)xmalloc((n ? n : 1) * 8);
    memcpy(cur, g->off, n * 8);
    for (uint64_t i = 0; i < m; ++i) {
        uint64_t p = cur[edst[i]]++;
        g->src[p] = esrc[i];
        if (ew) g->w[p] = ew[i];
    }
    free(cur);
    return g;
}

og_graph* og_from_csc(uint64_t n, uint64_t e, const uint64_t* off,
                      const uint32_t* src, const double* w) {
    og_graph* g = (og_graph*)xcalloc(1, sizeof(og_graph));
    g->n = n; g->e = e;
    g->off = (uint64_t*)xmalloc((n + 1) * 8);
    memcpy(g->off, off, (n + 1) * 8);
    g->src = (uint32_t*)xmalloc(e * 4);
    memcpy(g->src, src, e * 4);
    if (w) { g->w = (double*)xmalloc(e * 8); memcpy(g->w, w, e * 8); }
    g->outdeg = (uint32_t*)xcalloc(n, 4);
    for (uint64_t i = 0; i < e; ++i) g->outdeg[src[i]]++;
    return g;
}

/* graph.cpp:69-78 edge_list() in edge-id order: (src, dst, weight). */
static void edge_list(const og_graph* g, uint32_t* s, uint32_t* d, double* w) {
    for (uint64_t v = 0; v < g->n; ++v)
        for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
            s[e] = g->src[e]; d[e] = (uint32_t)v;
            if (w) w[e] = g->w ? g->w[e] : 1.0;
        }
}

/* graph.cpp:184-203 */
og_graph* og_generate_dumbbell(uint64_t k) {
    if (k < 2) return NULL;
    uint64_t m = 2 * k * (k - 1) + 2, i = 0;
    uint32_t* s = (uint32_t*)xmalloc(m * 4);
    uint32_t* d = (uint32_t*)xmalloc(m * 4);
    for (uint64_t c = 0; c < 2; ++c) {
        uint32_t base = (uint32_t)(c * k);
        for (uint64_t u = 0; u < k; ++u)
            for (uint64_t v = 0; v < k; ++v) {
                if (u == v) continue;
                s[i] = base + (uint32_t)u; d[i] = base + (uint32_t)v; ++i;
            }
    }
    s[i] = (uint32_t)(k - 1); d[i] = (uint32_t)k; ++i;
    s[i] = (uint32_t)k; d[i] = (uint32_t)(k - 1); ++i;
    og_graph* g = og_build_graph(2 * k, m, s, d, NULL);
    free(s); free(d);
    return g;
}

/* graph.cpp:205-241 (Chung-Lu style, upper_bound over a Zipf cdf) */
og_graph* og_generate_power_law(uint64_t n, double avg_degree, double exponent,
                                uint64_t seed) {
    if (n < 1 || !(avg_degree > 0.0) || !(exponent > 1.0)) return NULL;
    const double rank_exp = 1.0 / (exponent - 1.0);
    double* cdf = (double*)xmalloc(n * 8);
    double total = 0.0;
    for (uint64_t v = 0; v < n; ++v) {
        total += pow((double)(v + 1), -rank_exp);
        cdf[v] = total;
    }
    for (uint64_t v = 0; v < n; ++v) cdf[v] /= total;
    const uint64_t m = (uint64_t)llround((double)n * avg_degree);
    uint32_t* s = (uint32_t*)xmalloc(m * 4);
    uint32_t* d = (uint32_t*)xmalloc(m * 4);
    const uint64_t key = og_mix64(seed);
    for (uint64_t e = 0; e < m; ++e) {
        const double u_dst = og_to_unit(og_mix64(key ^ (2 * e + 1)));
        const double u_src = og_to_unit(og_mix64(key ^ (2 * e + 2)));
        /* std::upper_bound: first index with cdf[i] > u_dst */
        uint64_t lo = 0, hi = n;
        while (lo < hi) {
            uint64_t mid = lo + (hi - lo) / 2;
            if (u_dst < cdf[mid]) hi = mid; else lo = mid + 1;
        }
        uint64_t dst = lo < n - 1 ? lo : n - 1;
        uint64_t sv = (uint64_t)(u_src * (double)n);
        s[e] = (uint32_t)(sv < n - 1 ? sv : n - 1);
        d[e] = (uint32_t)dst;
    }
    og_graph* g = og_build_graph(n, m, s, d, NULL);
    free(cdf); free(s); free(d);
    return g;
}

/* test_support.hpp:33-48 */
og_graph* og_random_graph(uint64_t n, uint64_t m, uint64_t seed, int weighted) {
    uint32_t* s = (uint32_t*)xmalloc(m * 4);
    uint32_t* d = (uint32_t*)xmalloc(m * 4);
    double* w = (double*)xmalloc(m * 8);
    for (uint64_t e = 0; e < m; ++e) {
        uint32_t u = (uint32_t)(og_to_unit(og_mix64(seed * 3 + 17 + 2 * e)) * (double)n);
        uint32_t v = (uint32_t)(og_to_unit(og_mix64(seed * 3 + 18 + 2 * e)) * (double)n);
        w[e] = 0.1 + 2.0 * og_to_unit(og_mix64(seed * 5 + 23 + e));
        s[e] = u < (uint32_t)(n - 1) ? u : (uint32_t)(n - 1);
        d[e] = v < (uint32_t)(n - 1) ? v : (uint32_t)(n - 1);
    }
    og_graph* g = og_build_graph(n, m, s, d, weighted ? w : NULL);
    free(s); free(d); free(w);
    return g;
}

/* graph.cpp:249-257: edge_list() then the reversed copies, stable build. */
og_graph* og_symmetrized(const og_graph* g) {
    uint64_t m = g->e;
    uint32_t* s = (uint32_t*)xmalloc(2 * m * 4 + 4);
    uint32_t* d = (uint32_t*)xmalloc(2 * m * 4 + 4);
    double* w = (double*)xmalloc(2 * m * 8 + 8);
    edge_list(g, s, d, w);
    for (uint64_t i = 0; i < m; ++i) { s[m + i] = d[i]; d[m + i] = s[i]; w[m + i] = w[i]; }
    og_graph* r = og_build_graph(g->n, 2 * m, s, d, g->w ? w : NULL);
    free(s); free(d); free(w);
    return r;
}

/* graph.cpp:243-247 */
og_graph* og_reverse(const og_graph* g) {
    uint64_t m = g->e;
    uint32_t* s = (uint32_t*)xmalloc(m * 4 + 4);
    uint32_t* d = (uint32_t*)xmalloc(m * 4 + 4);
    double* w = (double*)xmalloc(m * 8 + 8);
    edge_list(g, s, d, w);
    og_graph* r = og_build_graph(g->n, m, d, s, g->w ? w : NULL);
    free(s); free(d); free(w);
    return r;
}

/* ---------------------------------------------------------------------------
 * R-MAT (NEW input layer; the reference has no R-MAT generator).
 * Specification shared with the GPU generator (csrc/rmat.cu):
 *   key = mix64(seed); for edge i in [0, ef*2^scale), level l in [0, scale):
 *     u = to_unit(mix64(key ^ (i*64 + l)));  quadrant by u < a | a+b | a+b+c
 *     (a: src0 dst0, b: src0 dst1, c: src1 dst0, d: src1 dst1), MSB first.
 *   self-loops and duplicate (src,dst) pairs removed; CSC sorted by (dst,src).
 * ------------------------------------------------------------------------- */
static inline void rmat_edge(uint64_t key, uint64_t i, uint32_t scale, double t1,
                             double t2, double t3, uint32_t* ps, uint32_t* pd) {
    uint32_t s = 0, d = 0;
    for (uint32_t l = 0; l < scale; ++l) {
        double u = og_to_unit(og_mix64(key ^ (i * 64 + l)));
        uint32_t sb, db;
        if (u < t1) { sb = 0; db = 0; }
        else if (u < t2) { sb = 0; db = 1; }
        else if (u < t3) { sb = 1; db = 0; }
        else { sb = 1; db = 1; }
        s = (s << 1) | sb; d = (d << 1) | db;
    }
    *ps = s; *pd = d;
}

static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

/* Two-level bucketing, contention free: per-thread counts by the top
 * `bbits` destination bits, a regenerate-and-scatter pass of (dst,src) keys,
 * then each bucket sorted and de-duplicated independently. */
og_graph* og_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed,
                  double a, double b, double c, int threads) {
    if (scale < 1 || scale > 31) return NULL;
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
    const int T = omp_get_max_threads();
#else
    (void)threads;
    const int T = 1;
#endif
    const uint64_t n = 1ull << scale;
    const uint64_t m = (uint64_t)edge_factor << scale;
    const double t1 = a, t2 = a + b, t3 = a + b + c;
    const uint64_t key = og_mix64(seed);
    const uint32_t bbits = scale < 16 ? scale : 16;
    const uint32_t bshift = scale - bbits;
    const uint64_t B = 1ull << bbits;
    uint64_t* cnt = (uint64_t*)xcalloc((size_t)T * B + 1, 8); /* [bucket][thread] */
#pragma omp parallel num_threads(T)
    {
#ifdef _OPENMP
        const int t = omp_get_thread_num();
#else
        const int t = 0;
#endif
        const uint64_t lo = m * (uint64_t)t / (uint64_t)T, hi = m * (uint64_t)(t + 1) / (uint64_t)T;
        for (uint64_t i = lo; i < hi; ++i) {
            uint32_t s, d;
            rmat_edge(key, i, scale, t1, t2, t3, &s, &d);
            if (s == d) continue;
            cnt[(uint64_t)(d >> bshift) * T + t]++;
        }
    }
    uint64_t total = 0;
    for (uint64_t i = 0; i < (uint64_t)T * B; ++i) { uint64_t x = cnt[i]; cnt[i] = total; total += x; }
    cnt[(uint64_t)T * B] = total;
    uint64_t* keys = (uint64_t*)xmalloc(total * 8 + 8);
#pragma omp parallel num_threads(T)
    {
#ifdef _OPENMP
        const int t = omp_get_thread_num();
#else
        const int t = 0;
#endif
        const uint64_t lo = m * (uint64_t)t / (uint64_t)T, hi = m * (uint64_t)(t + 1) / (uint64_t)T;
        for (uint64_t i = lo; i < hi; ++i) {
            uint32_t s, d;
            rmat_edge(key, i, scale, t1, t2, t3, &s, &d);
            if (s == d) continue;
            keys[cnt[(uint64_t)(d >> bshift) * T + t]++] = ((uint64_t)d << 32) | s;
        }
    }
    /* after pass 2, cnt[b*T + t] is the end of (b, t); bucket b = [start, end) */
    uint64_t* bstart = (uint64_t*)xmalloc((B + 1) * 8);
    uint64_t* ucnt = (uint64_t*)xcalloc(B + 1, 8);
    bstart[0] = 0;
    for (uint64_t bk = 0; bk < B; ++bk) bstart[bk + 1] = cnt[bk * T + (T - 1)];
    free(cnt);
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
    for (int64_t bk = 0; bk < (int64_t)B; ++bk) {
        uint64_t* p = keys + bstart[bk];
        const uint64_t len = bstart[bk + 1] - bstart[bk];
        if (len > 1) qsort(p, len, 8, cmp_u64);
        uint64_t k = 0;
        for (uint64_t j = 0; j < len; ++j)
            if (j == 0 || p[j] != p[j - 1]) p[k++] = p[j];
        ucnt[bk + 1] = k;
    }
    for (uint64_t bk = 0; bk < B; ++bk) ucnt[bk + 1] += ucnt[bk];
    og_graph* g = (og_graph*)xcalloc(1, sizeof(og_graph));
    g->n = n; g->e = ucnt[B];
    g->off = (uint64_t*)xcalloc(n + 1, 8);
    g->src = (uint32_t*)xmalloc(g->e * 4 + 4);
#pragma omp parallel for schedule(dynamic, 1) num_threads(T)
    for (int64_t bk = 0; bk < (int64_t)B; ++bk) {
        const uint64_t* p = keys + bstart[bk];
        const uint64_t len = ucnt[bk + 1] - ucnt[bk];
        uint64_t o = ucnt[bk];
        for (uint64_t j = 0; j < len; ++j) {
            g->src[o + j] = (uint32_t)p[j];
            g->off[(p[j] >> 32) + 1]++; /* dst owned by this bucket only */
        }
    }
    for (uint64_t v = 0; v < n; ++v) g->off[v + 1] += g->off[v];
    free(keys); free(bstart); free(ucnt);
    g->w = NULL;
    g->outdeg = (uint32_t*)xcalloc(n, 4);
    for (uint64_t e = 0; e < g->e; ++e) g->outdeg[g->src[e]]++;
    return g;
}

/* BASELINE C2 weights: 1 + mix64(kw ^ e) % 255 over canonical edge ids. */
void og_rmat_weights_u32(uint64_t e, uint64_t seed, uint32_t* out) {
    const uint64_t kw = og_mix64(og_mix64(seed) ^ 0x77656967687473ull);
    for (uint64_t i = 0; i < e; ++i) out[i] = 1u + (uint32_t)(og_mix64(kw ^ i) % 255u);
}

/* BASELINE C4 priors: uniform (0,1) per state, normalised, stored fp32. */
void og_bp_priors(uint64_t n, uint64_t seed, float* out) {
    const uint64_t kp = og_mix64(og_mix64(seed) ^ 0x7072696f7273ull);
    for (uint64_t v = 0; v < n; ++v) {
        double p0 = ((double)(og_mix64(kp ^ (2 * v)) >> 11) + 0.5) * 0x1.0p-53;
        double p1 = ((double)(og_mix64(kp ^ (2 * v + 1)) >> 11) + 0.5) * 0x1.0p-53;
        double s = p0 + p1;
        out[2 * v] = (float)(p0 / s);
        out[2 * v + 1] = (float)(p1 / s);
    }
}

/* BASELINE C4 potentials: diagonal c_e uniform in [0.5, 0.9], fp32. */
void og_bp_couplings(uint64_t e, uint64_t seed, float* out) {
    const uint64_t kc = og_mix64(og_mix64(seed) ^ 0x636f75706c65ull);
    for (uint64_t i = 0; i < e; ++i)
        out[i] = (float)(0.5 + 0.4 * og_to_unit(og_mix64(kc ^ i)));
}

uint32_t og_max_outdeg_vertex(const og_graph* g) {
    uint32_t best = 0;
    for (uint64_t v = 1; v < g->n; ++v)
        if (g->outdeg[v] > g->outdeg[best]) best = (uint32_t)v;
    return best;
}

/* ---------------------------------------------------------------------------
 * engine.cpp
 * ------------------------------------------------------------------------- */
static int fail_msg(char* msg, size_t cap, const char* text) {
    if (msg && cap) { strncpy(msg, text, cap - 1); msg[cap - 1] = 0; }
    return OG_INVALID_ARGUMENT;
}

/* engine.cpp:45-61 */
int og_validate(const og_config* cfg, char* msg, size_t cap) {
    if (!(cfg->sigma >= 0.0 && cfg->sigma <= 1.0)) return fail_msg(msg, cap, "sigma must be in [0,1]");
    if (!(cfg->theta >= 0.0)) return fail_msg(msg, cap, "theta must be >= 0");
    if (cfg->alpha < 1) return fail_msg(msg, cap, "alpha must be >= 1");
    if (cfg->max_iterations < 1) return fail_msg(msg, cap, "max_iterations must be >= 1");
    if (cfg->threads < 1) return fail_msg(msg, cap, "threads must be >= 1");
    return OG_OK;
}

/* engine.cpp:63-75 */
int og_sparsify(uint64_t e, double sigma, uint64_t seed, uint8_t* flags) {
    if (!(sigma >= 0.0 && sigma <= 1.0)) return OG_INVALID_ARGUMENT;
    const uint64_t key = og_mix64(seed);
    for (uint64_t i = 0; i < e; ++i) {
        const double u = (double)(og_mix64(key ^ i) >> 11) * 0x1.0p-53;
        flags[i] = u < sigma ? 1 : 0;
    }
    return OG_OK;
}

/* engine.cpp:92-107 */
int og_mode_for(int scheme, uint64_t t, uint64_t alpha) {
    switch (scheme) {
        case OG_ACCURATE: return OG_MODE_ACCURATE;
        case OG_SP: return OG_MODE_APPROXIMATE;
        case OG_SMS:
            if (t <= alpha) return OG_MODE_APPROXIMATE;
            if (t == alpha + 1) return OG_MODE_SUPERSTEP;
            return OG_MODE_ACCURATE;
        case OG_GG:
            return t % (alpha + 1) == 0 ? OG_MODE_SUPERSTEP : OG_MODE_APPROXIMATE;
    }
    return OG_MODE_ACCURATE;
}

/* engine.cpp:77-90 */
uint64_t og_supersteps(uint64_t alpha, uint64_t max_iterations, int scheme,
                       uint64_t* out, uint64_t cap) {
    uint64_t k = 0;
    if (alpha < 1) return 0;
    if (scheme == OG_GG) {
        for (uint64_t t = alpha + 1; t <= max_iterations; t += alpha + 1) {
            if (k < cap) out[k] = t;
            ++k;
        }
    } else if (scheme == OG_SMS) {
        if (alpha + 1 <= max_iterations) { if (k < cap) out[k] = alpha + 1; ++k; }
    }
    return k;
}

/* ---------------------------------------------------------------------------
 * Vertex programs (algorithms.hpp / algorithms.cpp) behind one vtable that
 * mirrors the VertexProgram concept (engine.hpp:80-93).
 * ------------------------------------------------------------------------- */
typedef struct prog {
    size_t psize;
    const og_params* p;
    uint64_t n;
    int* poison_count; /* POISON's mutable apply counter (test_engine.cpp:27) */
    void (*init)(const struct prog*, uint32_t v, void* out);
    void (*identity)(const struct prog*, void* out);
    double (*gather)(const struct prog*, void* acc, const void* src, double w, uint32_t deg);
    void (*apply)(const struct prog*, uint32_t v, const void* acc, const void* prev, void* out);
    int (*vstatus)(const struct prog*, const void* before, const void* after);
    int (*valid)(const struct prog*, const void* p);
} prog;

/* estatus is `influence > theta` for every reference program
 * (algorithms.hpp:38, :81, :110, :138). */
static int estatus(double influence, double theta) { return influence > theta; }

/* PageRankProgram, algorithms.hpp:15-40 */
static void pr_init(const prog* P, uint32_t v, void* o) { (void)v; *(double*)o = 1.0 / (double)P->n; }
static void pr_id(const prog* P, void* o) { (void)P; *(double*)o = 0.0; }
static double pr_gather(const prog* P, void* a, const void* s, double w, uint32_t deg) {
    (void)P; (void)w;
    double* acc = (double*)a;
    const double before = *acc;
    *acc += *(const double*)s / (double)deg;
    return *acc > 0.0 ? (*acc - before) / *acc : 0.0;
}
static void pr_apply(const prog* P, uint32_t v, const void* a, const void* prev, void* o) {
    (void)v; (void)prev;
    *(double*)o = (1.0 - P->p->damping) / (double)P->n + P->p->damping * *(const double*)a;
}
static int pr_vstatus(const prog* P, const void* b, const void* a) {
    return fabs(*(const double*)b - *(const double*)a) > P->p->epsilon;
}
static int pr_valid(const prog* P, const void* p) { (void)P; return isfinite(*(const double*)p); }

/* SsspProgram, algorithms.hpp:46-83 */
static void sssp_init(const prog* P, uint32_t v, void* o) {
    *(double*)o = v == P->p->source ? 0.0 : INFINITY;
}
static void sssp_id(const prog* P, void* o) { (void)P; *(double*)o = INFINITY; }
static double sssp_gather(const prog* P, void* a, const void* s, double w, uint32_t deg) {
    (void)deg;
    double* acc = (double*)a;
    const double cand = *(const double*)s + w;
    if (cand < *acc) {
        double infl = 1.0;
        if (P->p->graded && isfinite(*acc)) infl = (*acc - cand) / *acc;
        *acc = cand;
        return infl;
    }
    return 0.0;
}
static void sssp_apply(const prog* P, uint32_t v, const void* a, const void* prev, void* o) {
    (void)P; (void)v;
    double x = *(const double*)a, y = *(const double*)prev;
    *(double*)o = y < x ? y : x; /* std::min(acc, prev): returns acc unless prev < acc */
}
static int sssp_vstatus(const prog* P, const void* b, const void* a) {
    (void)P; return *(const double*)a < *(const double*)b;
}
static int sssp_valid(const prog* P, const void* p) {
    (void)P; double x = *(const double*)p; return !isnan(x) && x >= 0.0;
}

/* WccProgram, algorithms.hpp:88-112 */
static void wcc_init(const prog* P, uint32_t v, void* o) { (void)P; *(uint32_t*)o = v; }
static void wcc_id(const prog* P, void* o) { (void)P; *(uint32_t*)o = 0xffffffffu; }
static double wcc_gather(const prog* P, void* a, const void* s, double w, uint32_t deg) {
    (void)P; (void)w; (void)deg;
    uint32_t* acc = (uint32_t*)a;
    if (*(const uint32_t*)s < *acc) { *acc = *(const uint32_t*)s; return 1.0; }
    return 0.0;
}
static void wcc_apply(const prog* P, uint32_t v, const void* a, const void* prev, void* o) {
    (void)P; (void)v;
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)prev;
    *(uint32_t*)o = y < x ? y : x;
}
static int wcc_vstatus(const prog* P, const void* b, const void* a) {
    (void)P; return *(const uint32_t*)a != *(const uint32_t*)b;
}
static int wcc_valid(const prog* P, const void* p) { (void)P; (void)p; return 1; }

/* BeliefPropagationProgram, algorithms.cpp:9-69. S = params->states. */
static void bp_prior(const prog* P, uint32_t v, double* out) {
    const int S = P->p->states;
    double sum = 0.0;
    for (int i = 0; i < S; ++i) {
        const uint64_t h = og_mix64((uint64_t)v * (uint64_t)S + (uint64_t)i);
        out[i] = 1.0 + (double)(h >> 11) * 0x1.0p-53;
        sum += out[i];
    }
    for (int i = 0; i < S; ++i) out[i] /= sum;
}
static void bp_init(const prog* P, uint32_t v, void* o) { bp_prior(P, v, (double*)o); }
static void bp_id(const prog* P, void* o) {
    for (int i = 0; i < P->p->states; ++i) ((double*)o)[i] = 1.0;
}
/* algorithms.cpp:25-48, with the coupling passed in (global or per edge). */
static double bp_gather_c(int S, double coupling, double* acc, const double* src) {
    const double off = (1.0 - coupling) / (double)(S - 1);
    double src_sum = 0.0;
    for (int i = 0; i < S; ++i) src_sum += src[i];
    double l1_before = 0.0, l1_after = 0.0, l1_diff = 0.0, acc_sum = 0.0;
    for (int i = 0; i < S; ++i) {
        const double msg = off * (src_sum - src[i]) + coupling * src[i];
        const double updated = acc[i] * msg;
        l1_before += fabs(acc[i]);
        l1_after += fabs(updated);
        l1_diff += fabs(acc[i] - updated);
        acc[i] = updated;
        acc_sum += updated;
    }
    (void)l1_before;
    if (acc_sum > 0.0)
        for (int i = 0; i < S; ++i) acc[i] /= acc_sum;
    if (l1_after <= 0.0) return 0.0;
    const double r = l1_diff / l1_after;
    return r < 1.0 ? r : 1.0; /* std::min(1.0, r) */
}
static double bp_gather(const prog* P, void* a, const void* s, double w, uint32_t deg) {
    (void)w; (void)deg;
    return bp_gather_c(P->p->states, P->p->coupling, (double*)a, (const double*)s);
}
/* algorithms.cpp:50-62 */
static void bp_apply(const prog* P, uint32_t v, const void* a, const void* prev, void* o) {
    (void)prev;
    const int S = P->p->states;
    double* out = (double*)o;
    bp_prior(P, v, out);
    double sum = 0.0;
    for (int i = 0; i < S; ++i) { out[i] *= ((const double*)a)[i]; sum += out[i]; }
    if (sum > 0.0)
        for (int i = 0; i < S; ++i) out[i] /= sum;
}
/* algorithms.cpp:64-69 */
static int bp_vstatus(const prog* P, const void* b, const void* a) {
    double l1 = 0.0;
    for (int i = 0; i < P->p->states; ++i)
        l1 += fabs(((const double*)b)[i] - ((const double*)a)[i]);
    return l1 > P->p->epsilon;
}
/* algorithms.hpp:139-144 */
static int bp_valid(const prog* P, const void* p) {
    for (int i = 0; i < P->p->states; ++i)
        if (!isfinite(((const double*)p)[i])) return 0;
    return 1;
}

/* BP_EDGE (BASELINE C4): the reference BP formulas with S = 2, coupling =
 * the edge weight (fp32 c_e widened), prior = fp32 table entry, and beliefs
 * rounded to fp32 after apply (fp32 storage, f64 arithmetic). */
static void bpe_init(const prog* P, uint32_t v, void* o) {
    ((double*)o)[0] = (double)P->p->prior_table[2 * (uint64_t)v];
    ((double*)o)[1] = (double)P->p->prior_table[2 * (uint64_t)v + 1];
}
static double bpe_gather(const prog* P, void* a, const void* s, double w, uint32_t deg) {
    (void)P; (void)deg;
    return bp_gather_c(2, w, (double*)a, (const double*)s);
}
static void bpe_apply(const prog* P, uint32_t v, const void* a, const void* prev, void* o) {
    (void)prev;
    double* out = (double*)o;
    bpe_init(P, v, out);
    double sum = 0.0;
    for (int i = 0; i < 2; ++i) { out[i] *= ((const double*)a)[i]; sum += out[i]; }
    if (sum > 0.0)
        for (int i = 0; i < 2; ++i) out[i] /= sum;
    for (int i = 0; i < 2; ++i) out[i] = (double)(float)out[i];
}

/* PoisonProgram, test_engine.cpp:23-50 */
static void poi_init(const prog* P, uint32_t v, void* o) { (void)P; (void)v; *(double*)o = 1.0; }
static double poi_gather(const prog* P, void* a, const void* s, double w, uint32_t deg) {
    (void)P; (void)w; (void)deg;
    *(double*)a += *(const double*)s;
    return 0.0;
}
static void poi_apply(const prog* P, uint32_t v, const void* a, const void* prev, void* o) {
    if (v == P->p->poison_vertex && ++*P->poison_count == P->p->poison_iteration) {
        *(double*)o = NAN;
        return;
    }
    *(double*)o = *(const double*)prev + *(const double*)a * 1e-6;
}
static int poi_vstatus(const prog* P, const void* b, const void* a) { (void)P; (void)b; (void)a; return 1; }
static int poi_valid(const prog* P, const void* p) { (void)P; return !isnan(*(const double*)p); }

static int make_prog(int which, const og_params* p, uint64_t n, int* counter, prog* out) {
    memset(out, 0, sizeof(*out));
    out->p = p; out->n = n; out->poison_count = counter;
    switch (which) {
        case OG_PR:
            out->psize = 8; out->init = pr_init; out->identity = pr_id; out->gather = pr_gather;
            out->apply = pr_apply; out->vstatus = pr_vstatus; out->valid = pr_valid; break;
        case OG_SSSP:
            out->psize = 8; out->init = sssp_init; out->identity = sssp_id; out->gather = sssp_gather;
            out->apply = sssp_apply; out->vstatus = sssp_vstatus; out->valid = sssp_valid; break;
        case OG_WCC:
            out->psize = 4; out->init = wcc_init; out->identity = wcc_id; out->gather = wcc_gather;
            out->apply = wcc_apply; out->vstatus = wcc_vstatus; out->valid = wcc_valid; break;
        case OG_BP:
            if (p->states < 2 || 8 * (size_t)p->states > OG_MAX_PSIZE) return -1;
            out->psize = 8 * (size_t)p->states; out->init = bp_init; out->identity = bp_id;
            out->gather = bp_gather; out->apply = bp_apply; out->vstatus = bp_vstatus;
            out->valid = bp_valid; break;
        case OG_BP_EDGE:
            if (!p->prior_table) return -1;
            out->psize = 16; out->init = bpe_init; out->identity = bp_id; out->gather = bpe_gather;
            out->apply = bpe_apply; out->vstatus = bp_vstatus; out->valid = bp_valid; break;
        case OG_POISON:
            out->psize = 8; out->init = poi_init; out->identity = pr_id; out->gather = poi_gather;
            out->apply = poi_apply; out->vstatus = poi_vstatus; out->valid = poi_valid; break;
        default: return -1;
    }
    return 0;
}

/* ---------------------------------------------------------------------------
 * gg::run restatement — engine.hpp:141-249.
 *
 * The vertex loop of one iteration is a Jacobi update (each vertex reads
 * only prev[] and writes only its own next[] / status / edge flags), so it
 * runs over OpenMP threads (cfg->threads) with each vertex's fold kept
 * sequential in CSC order: the results are those of the reference for any
 * thread count (engine.hpp:139-140, test_engine.cpp:161-182).
 *
 * Lock-step mode (og_run_ex with `ls`): in superstep s the device's flags
 * after that superstep (ls->dev_bitmaps[s]) are compared edge by edge with
 * the oracle's own estatus decision. An edge whose influence lies within the
 * program's rounding band of theta (|infl - theta| <= band, see
 * og_lockstep) and whose device flag differs is ADOPTED (counted as
 * near-threshold), so the rest of the run follows the same flag set as the
 * device; a differing edge outside the band is a REAL mismatch (counted,
 * the oracle keeps its own decision).
 * ------------------------------------------------------------------------- */
static inline double near_band(const og_lockstep* ls, uint64_t k, double infl, double theta) {
    const double m = fabs(infl) > theta ? fabs(infl) : theta;
    return ls->tol_unit * ((double)(k + 4) * m + 4.0);
}

int og_run_ex(const og_graph* g, int which, const og_params* params,
              const og_config* cfg, void* out_props, og_record* recs,
              uint64_t rec_cap, og_summary* sum, uint8_t* out_flags,
              char* msg, size_t msg_cap, og_lockstep* ls) {
    memset(sum, 0, sizeof(*sum));
    int rc = og_validate(cfg, msg, msg_cap);                       /* :145 */
    if (rc) return rc;
    const uint64_t n = g->n;
    if (n == 0) return OG_OK;                                      /* :149 */
    if (which == OG_SSSP && params->source >= n)                   /* algorithms.hpp:55-57 */
        return fail_msg(msg, msg_cap, "sssp source vertex out of range");
    int counter = 0;
    prog P;
    if (make_prog(which, params, n, &counter, &P)) return fail_msg(msg, msg_cap, "bad program parameters");
    if (which == OG_BP_EDGE && !g->w) return fail_msg(msg, msg_cap, "bp_edge needs coupling weights");
    const size_t ps = P.psize;
#ifdef _OPENMP
    const int T = which == OG_POISON ? 1 : (int)(cfg->threads ? cfg->threads : 1);
#endif
    if (ls && ls->stats) memset(ls->stats, 0, 4 * ls->stats_cap * sizeof(uint64_t));

    uint8_t* flags = (uint8_t*)xmalloc(g->e + 1);                  /* :151-153 */
    if (cfg->scheme == OG_ACCURATE) memset(flags, 1, g->e);
    else {
        const uint64_t key = og_mix64(cfg->seed);                  /* engine.cpp:63-75 */
#pragma omp parallel for schedule(static) num_threads(T)
        for (int64_t i = 0; i < (int64_t)g->e; ++i)
            flags[i] = (double)(og_mix64(key ^ (uint64_t)i) >> 11) * 0x1.0p-53 < cfg->sigma ? 1 : 0;
    }
    uint32_t* aid = (uint32_t*)xmalloc(n * 4);                     /* :154-161 */
#pragma omp parallel for schedule(static) num_threads(T)
    for (int64_t v = 0; v < (int64_t)n; ++v) {
        uint32_t c = 0;
        for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) c += flags[e] ? 1 : 0;
        aid[v] = c;
    }
    uint8_t* prev = (uint8_t*)xmalloc(n * ps);                     /* :163-167 */
    uint8_t* next = (uint8_t*)xmalloc(n * ps);
    for (uint64_t v = 0; v < n; ++v) P.init(&P, (uint32_t)v, prev + v * ps);
    memcpy(next, prev, n * ps);
    uint8_t* status = (uint8_t*)xmalloc(n);
    uint8_t* status_next = (uint8_t*)xcalloc(n, 1);
    memset(status, 1, n);
    uint64_t s_ord = 0;  /* supersteps so far */

    for (uint64_t t = 1; t <= cfg->max_iterations; ++t) {          /* :177 */
        const int mode = og_mode_for(cfg->scheme, t, cfg->alpha);
        const int approx = mode == OG_MODE_APPROXIMATE;
        const int superstep = mode == OG_MODE_SUPERSTEP;
        const uint32_t* dev = (superstep && ls && s_ord < ls->n_dev) ? ls->dev_bitmaps[s_ord] : NULL;
        uint64_t* st = (superstep && ls && ls->stats && s_ord < ls->stats_cap) ? ls->stats + 4 * s_ord : NULL;
        memcpy(next, prev, n * ps);                                /* :183-184 */
        memset(status_next, 0, n);
        uint64_t gathered = 0, processed = 0, n_near = 0, n_adopt = 0, n_real = 0, n_kept = 0;
        int changed = 0;
        int64_t bad_vertex = INT64_MAX;
#pragma omp parallel num_threads(T) reduction(+ : gathered, processed, n_near, n_adopt, n_real, n_kept) \
    reduction(| : changed) reduction(min : bad_vertex)
        {
            uint8_t acc[OG_MAX_PSIZE], fresh[OG_MAX_PSIZE];
#pragma omp for schedule(dynamic, 2048)
            for (int64_t vi = 0; vi < (int64_t)n; ++vi) {          /* :194 */
                const uint64_t v = (uint64_t)vi;
                if (!status[v] && aid[v] == 0) continue;           /* :196 */
                P.identity(&P, acc);                               /* :198 */
                uint64_t local_edges = 0;
                uint32_t new_active = 0;
                for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) { /* :202 */
                    if (approx && !flags[e]) continue;             /* :203 */
                    const uint32_t s = g->src[e];
                    const double w = g->w ? g->w[e] : 1.0;         /* :205 */
                    const double infl = P.gather(&P, acc, prev + (uint64_t)s * ps, w, g->outdeg[s]);
                    if (superstep) {                               /* :207-211 */
                        int keep = estatus(infl, cfg->theta);
                        if (ls) {
                            const int near = ls->tol_unit > 0.0 && fabs(infl - cfg->theta) <=
                                             near_band(ls, e - g->off[v], infl, cfg->theta);
                            n_near += near;
                            if (dev) {
                                const int d = (int)((dev[e >> 5] >> (e & 31)) & 1u);
                                if (d != keep) {
                                    if (near) { keep = d; ++n_adopt; }
                                    else ++n_real;
                                }
                            }
                        }
                        flags[e] = keep ? 1 : 0;
                        new_active += keep ? 1 : 0;
                    }
                    ++local_edges;
                }
                if (superstep) { aid[v] = new_active; n_kept += new_active; }  /* :214 */
                P.apply(&P, (uint32_t)v, acc, prev + v * ps, fresh);   /* :216 */
                const int active = P.vstatus(&P, prev + v * ps, fresh);
                if (!P.valid(&P, fresh) && vi < bad_vertex) bad_vertex = vi;  /* :218 (min below) */
                memcpy(next + v * ps, fresh, ps);
                status_next[v] = active ? 1 : 0;
                changed |= active ? 1 : 0;
                gathered += local_edges;
                ++processed;
            }
        }
        if (st) { st[0] = n_near; st[1] = n_adopt; st[2] = n_real; st[3] = n_kept; }
        if (superstep) ++s_ord;
        if (bad_vertex != INT64_MAX) {                             /* :226-233 */
            for (uint64_t v = 0; v < n; ++v) {
                if ((status[v] || aid[v] > 0) && !P.valid(&P, next + v * ps)) {
                    sum->err_iteration = t; sum->err_vertex = (uint32_t)v;
                    if (msg && msg_cap)
                        snprintf(msg, msg_cap, "invalid property at iteration %llu, vertex %llu",
                                 (unsigned long long)t, (unsigned long long)v);
                    free(flags); free(aid); free(prev); free(next); free(status); free(status_next);
                    return OG_INVALID_PROPERTY;
                }
            }
        }
        if (t - 1 < rec_cap) {                                     /* :235-236 */
            recs[t - 1].mode = mode;
            recs[t - 1].processed_edges = gathered;
            recs[t - 1].active_vertices = processed;
        }
        sum->iterations_run = t;
        sum->total_processed_edges += gathered;
        uint8_t* tp = prev; prev = next; next = tp;                /* :238-239 */
        tp = status; status = status_next; status_next = tp;
        if (!changed) break;                                       /* :240 */
    }
    if (ls) ls->n_supersteps = s_ord;
    if (out_props) {
        if (which == OG_WCC) memcpy(out_props, prev, n * 4);
        else memcpy(out_props, prev, n * ps);
    }
    if (out_flags) memcpy(out_flags, flags, g->e);
    free(flags); free(aid); free(prev); free(next); free(status); free(status_next);
    return OG_OK;
}

int og_run(const og_graph* g, int which, const og_params* params,
           const og_config* cfg, void* out_props, og_record* recs,
           uint64_t rec_cap, og_summary* sum, uint8_t* out_flags,
           char* msg, size_t msg_cap) {
    return og_run_ex(g, which, params, cfg, out_props, recs, rec_cap, sum, out_flags, msg,
                     msg_cap, NULL);
}

/* Influence of every in-edge of destinations [v_begin, v_end) against the
 * running accumulator of its vertex's full in-list (engine.hpp:198-211, the
 * superstep fold) given prev[]; out[e - off[v_begin]]. */
int og_influences(const og_graph* g, int which, const og_params* params, const void* prev_v,
                  uint64_t v_begin, uint64_t v_end, int threads, double* out) {
    int counter = 0;
    prog P;
    if (make_prog(which, params, g->n, &counter, &P) || which == OG_POISON) return OG_INVALID_ARGUMENT;
    if (v_end > g->n || v_begin > v_end) return OG_INVALID_ARGUMENT;
    const size_t ps = P.psize;
    const uint8_t* prev = (const uint8_t*)prev_v;
    const uint64_t base = g->off[v_begin];
#ifdef _OPENMP
    const int T = threads > 0 ? threads : 1;
#else
    (void)threads;
#endif
#pragma omp parallel num_threads(T)
    {
        uint8_t acc[OG_MAX_PSIZE];
#pragma omp for schedule(dynamic, 2048)
        for (int64_t vi = (int64_t)v_begin; vi < (int64_t)v_end; ++vi) {
            P.identity(&P, acc);
            for (uint64_t e = g->off[vi]; e < g->off[vi + 1]; ++e) {
                const uint32_t s = g->src[e];
                const double w = g->w ? g->w[e] : 1.0;
                out[e - base] = P.gather(&P, acc, prev + (uint64_t)s * ps, w, g->outdeg[s]);
            }
        }
    }
    return OG_OK;
}

/* engine.hpp:163-164 */
int og_init_props(const og_graph* g, int which, const og_params* params, void* out) {
    int counter = 0;
    prog P;
    if (make_prog(which, params, g->n, &counter, &P)) return OG_INVALID_ARGUMENT;
    for (uint64_t v = 0; v < g->n; ++v) P.init(&P, (uint32_t)v, (uint8_t*)out + v * P.psize);
    return OG_OK;
}

/* engine.hpp:194-224 over one destination range, plus the owned part of the
 * :226-233 scan. Sequential per vertex exactly like og_run. */
int og_step_range(const og_graph* g, int which, const og_params* params, int mode, double theta,
                  uint8_t* flags, uint32_t* aid, const void* prev_v, const uint8_t* status,
                  void* next_v, uint8_t* status_next, uint64_t v_begin, uint64_t v_end,
                  uint64_t counters[4]) {
    int counter = 0;
    prog P;
    if (make_prog(which, params, g->n, &counter, &P)) return OG_INVALID_ARGUMENT;
    const size_t ps = P.psize;
    const uint8_t* prev = (const uint8_t*)prev_v;
    uint8_t* next = (uint8_t*)next_v;
    const int approx = mode == OG_MODE_APPROXIMATE, superstep = mode == OG_MODE_SUPERSTEP;
    uint8_t acc[OG_MAX_PSIZE], fresh[OG_MAX_PSIZE];
    uint64_t gathered = 0, processed = 0, changed = 0;
    int any_bad = 0;
    for (uint64_t v = v_begin; v < v_end; ++v) {
        memcpy(next + v * ps, prev + v * ps, ps);                  /* :183 */
        status_next[v] = 0;
        if (!status[v] && aid[v] == 0) continue;                   /* :196 */
        P.identity(&P, acc);
        uint64_t local_edges = 0;
        uint32_t new_active = 0;
        for (uint64_t e = g->off[v]; e < g->off[v + 1]; ++e) {
            if (approx && !flags[e]) continue;
            const uint32_t s = g->src[e];
            const double w = g->w ? g->w[e] : 1.0;
            const double infl = P.gather(&P, acc, prev + (uint64_t)s * ps, w, g->outdeg[s]);
            if (superstep) {
                const int keep = estatus(infl, theta);
                flags[e] = keep ? 1 : 0;
                new_active += keep ? 1 : 0;
            }
            ++local_edges;
        }
        if (superstep) aid[v] = new_active;
        P.apply(&P, (uint32_t)v, acc, prev + v * ps, fresh);
        const int active = P.vstatus(&P, prev + v * ps, fresh);
        if (!P.valid(&P, fresh)) any_bad = 1;
        memcpy(next + v * ps, fresh, ps);
        status_next[v] = active ? 1 : 0;
        changed |= active ? 1u : 0u;
        gathered += local_edges;
        ++processed;
    }
    uint64_t bad = 0;
    if (any_bad)
        for (uint64_t v = v_begin; v < v_end && !bad; ++v)
            if ((status[v] || aid[v] > 0) && !P.valid(&P, next + v * ps)) bad = v + 1;
    counters[0] = gathered; counters[1] = processed; counters[2] = changed; counters[3] = bad;
    return OG_OK;
}

/* ---------------------------------------------------------------------------
 * metrics.cpp
 * ------------------------------------------------------------------------- */
static const double* g_sort_vals;
/* descending value, ties by ascending id (metrics.cpp:23-34) */
static int cmp_topk(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    double vx = g_sort_vals[x], vy = g_sort_vals[y];
    if (vx != vy) return vx > vy ? -1 : 1;
    return x < y ? -1 : (x > y);
}
static uint32_t* topk_indices(const double* vals, uint64_t n, uint64_t k) {
    uint32_t* idx = (uint32_t*)xmalloc(n * 4);
    for (uint64_t i = 0; i < n; ++i) idx[i] = (uint32_t)i;
    g_sort_vals = vals;
    qsort(idx, n, 4, cmp_topk);
    (void)k;
    return idx;
}

/* metrics.cpp:60-74 */
int og_topk_error(const double* approx, const double* exact, uint64_t n,
                  uint64_t k, double* err) {
    if (k < 1 || k > n) return OG_INVALID_ARGUMENT;
    uint32_t* ta = topk_indices(approx, n, k);
    uint32_t* te = topk_indices(exact, n, k);
    uint8_t* in_exact = (uint8_t*)xcalloc(n, 1);
    for (uint64_t i = 0; i < k; ++i) in_exact[te[i]] = 1;
    uint64_t missing = 0;
    for (uint64_t i = 0; i < k; ++i) missing += in_exact[ta[i]] ? 0 : 1;
    *err = (double)missing / (double)k;
    free(ta); free(te); free(in_exact);
    return OG_OK;
}

/* metrics.cpp:76-87 */
int og_relative_error(const double* approx, const double* exact, uint64_t n, double* err) {
    if (n == 0) { *err = 0.0; return OG_OK; }
    double s = 0.0;
    for (uint64_t v = 0; v < n; ++v) {
        const double a = approx[v] + 1.0, e = exact[v] + 1.0;
        const double r = fabs(e - a) / e;
        s += r < 1.0 ? r : 1.0;
    }
    *err = s / (double)n;
    return OG_OK;
}

/* metrics.cpp:89-113 */
int og_stretch_error(const double* approx, const double* exact, uint64_t n, double* err) {
    double s = 0.0;
    uint64_t counted = 0;
    for (uint64_t v = 0; v < n; ++v) {
        const double e = exact[v], a = approx[v];
        if (a < e) return OG_ERROR;
        if (isinf(e)) continue;
        if (e == 0.0 && a == 0.0) continue;
        ++counted;
        if (isinf(a) || e == 0.0) { s += 1.0; continue; }
        s += 1.0 - e / a;
    }
    *err = counted == 0 ? 0.0 : s / (double)counted;
    return OG_OK;
}
