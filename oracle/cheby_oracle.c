/*
 * oracle/cheby_oracle.c -- CPU restatement of the reference ChebyPower path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker, never the product:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path
 * (paper_2412_10789_b200/, libcpg.so) never links or calls it and fails
 * loudly when its CUDA library is missing.
 *
 * Parity pinning: this restatement is checked against
 *   (1) the reference library itself, compiled from /root/reference sources
 *       into oracle/_ref/ by oracle/Makefile (tests/test_oracle_pin.py), and
 *   (2) the known-answer values of the reference's own tests
 *       (test_kernels.cpp:14-58, test_solvers.cpp:89-128,
 *        acceptance.cpp:74-90, 139-157, 349-360),
 *       and the committed golden vectors under tests/golden/.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to the reference's proj/ directory).  Arithmetic order is kept identical to
 * the reference so the restatement is bit-exact with it (no FMA: compiled with
 * -ffp-contract=off, like the reference's default x86-64 build).
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define CPO_OK 0
#define CPO_EINVAL 1
#define CPO_ENOMEM 4

/* ---- SplitMix64: include/chebyprop/rng.hpp:9-39 ---------------------- */
typedef struct { uint64_t state; } cpo_rng;

static uint64_t rng_next(cpo_rng* r) { /* rng.hpp:13-18 */
    uint64_t z = (r->state += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static double rng_next_double(cpo_rng* r) { /* rng.hpp:21 */
    return (double)(rng_next(r) >> 11) * 0x1.0p-53;
}
static uint64_t rng_next_below(cpo_rng* r, uint64_t bound) { /* rng.hpp:24-27 */
    return (uint64_t)(((unsigned __int128)rng_next(r) * bound) >> 64);
}

uint64_t cpo_splitmix_next(uint64_t* state) {
    cpo_rng r = {*state};
    uint64_t v = rng_next(&r);
    *state = r.state;
    return v;
}

/* ---- Chebyshev coefficients: src/kernels.cpp:157-194 ----------------- */
int cpo_ppr_cheby_coeffs(double alpha, uint64_t max_index, double* c) {
    if (!(alpha > 0.0 && alpha < 1.0)) return CPO_EINVAL; /* kernels.cpp:26-29 */
    const double root = sqrt(2.0 * alpha - alpha * alpha);   /* :159 */
    const double gamma = alpha / root;                        /* :160 */
    const double beta = (1.0 - alpha) / (1.0 + root);         /* :161 */
    c[0] = gamma;                                             /* :163 */
    double term = 2.0 * gamma;                                /* :164 */
    for (uint64_t k = 1; k <= max_index; ++k) {               /* :165-168 */
        term *= beta;
        c[k] = term;
    }
    return CPO_OK;
}

int cpo_hkpr_cheby_coeffs(double t, uint64_t max_index, double* c) {
    if (!(t > 0.0)) return CPO_EINVAL; /* kernels.cpp:31-33 */
    /* Miller backward recurrence, kernels.cpp:177-186 */
    uint64_t tc = (uint64_t)ceil(t);
    const uint64_t start = (max_index > tc ? max_index : tc) + 40;
    double* f = (double*)calloc(start + 2, sizeof(double));
    if (!f) return CPO_ENOMEM;
    f[start] = 1e-30;
    for (uint64_t n = start; n >= 1; --n) {
        f[n - 1] = f[n + 1] + (2.0 * (double)n / t) * f[n];
        if (f[n - 1] > 1e280)
            for (uint64_t j = n - 1; j <= start + 1; ++j) f[j] *= 1e-280;
    }
    /* normalisation e^-t (I_0 + 2 sum I_k) = 1, kernels.cpp:188-192 */
    double norm = f[0];
    for (uint64_t k = 1; k <= start; ++k) norm += 2.0 * f[k];
    c[0] = f[0] / norm;
    for (uint64_t k = 1; k <= max_index; ++k) c[k] = 2.0 * f[k] / norm;
    free(f);
    return CPO_OK;
}

/* Taylor (power-basis) coefficients, kernels.cpp:78-96 (ground truth / PwMethod). */
int cpo_taylor_coeffs(int family, double param, uint64_t max_index, double* zeta) {
    if (family == 0) {
        if (!(param > 0.0 && param < 1.0)) return CPO_EINVAL;
        double z = param;
        for (uint64_t k = 0; k <= max_index; ++k) { zeta[k] = z; z *= 1.0 - param; }
    } else if (family == 1) {
        if (!(param > 0.0)) return CPO_EINVAL;
        double z = exp(-param);
        for (uint64_t k = 0; k <= max_index; ++k) { zeta[k] = z; z *= param / (double)(k + 1); }
    } else {
        return CPO_EINVAL;
    }
    return CPO_OK;
}

/* ---- plan_truncation: src/kernels.cpp:237-341 (family 0 = PPR, 1 = HKPR) */
typedef struct {
    uint64_t cheby_steps;
    uint64_t taylor_steps;
    double epsilon;
    double tail_bound;
} cpo_plan;

#define CPO_TRUNC_CAP 1000000ull /* kernels.cpp:233 */

int cpo_plan_truncation(int family, double param, double epsilon, cpo_plan* plan) {
    if (!(epsilon > 0.0 && epsilon < 1.0)) return CPO_EINVAL; /* :254-255 */
    plan->epsilon = epsilon;
    plan->cheby_steps = 1;
    plan->taylor_steps = 1;
    plan->tail_bound = 0.0;
    if (family == 0) { /* :261-289 */
        const double alpha = param;
        if (!(alpha > 0.0 && alpha < 1.0)) return CPO_EINVAL;
        const double root = sqrt(2.0 * alpha - alpha * alpha);
        const double gamma = alpha / root;
        const double beta = (1.0 - alpha) / (1.0 + root);
#define CHEBY_TAIL(KK) (2.0 * gamma / (1.0 - beta) * exp((double)((KK) + 1) * log(beta)))
        uint64_t K = 1;
        while (CHEBY_TAIL(K) >= epsilon)
            if (++K > CPO_TRUNC_CAP) return CPO_EINVAL;
        plan->cheby_steps = K;
        plan->tail_bound = CHEBY_TAIL(K);
#undef CHEBY_TAIL
        uint64_t N = 1;
        double tail = 1.0 - alpha;
        while (tail >= epsilon) {
            tail *= 1.0 - alpha;
            if (++N > CPO_TRUNC_CAP) return CPO_EINVAL;
        }
        plan->taylor_steps = N;
        return CPO_OK;
    }
    if (family == 1) { /* :290-322 */
        const double t = param;
        if (!(t > 0.0)) return CPO_EINVAL;
        uint64_t horizon = 64;
        for (;;) {
            double* c = (double*)malloc((horizon + 1) * sizeof(double));
            if (!c) return CPO_ENOMEM;
            cpo_hkpr_cheby_coeffs(t, horizon, c);
            /* cheby_steps_from_prefix, :237-249 */
            double prefix = 0.0;
            uint64_t found = 0;
            for (uint64_t k = 0; k <= horizon; ++k) {
                prefix += c[k];
                double tail = 1.0 - prefix;
                if (tail < 0.0) tail = 0.0;
                if (k >= 1 && tail < epsilon) {
                    plan->tail_bound = tail;
                    found = k;
                    break;
                }
            }
            free(c);
            if (found) { plan->cheby_steps = found; break; }
            if (horizon >= CPO_TRUNC_CAP) return CPO_EINVAL;
            horizon = horizon * 2 < CPO_TRUNC_CAP ? horizon * 2 : CPO_TRUNC_CAP;
        }
        double z = exp(-t), prefix = 0.0;
        uint64_t N = 0;
        for (;;) {
            prefix += z;
            ++N;
            if (1.0 - prefix < epsilon) break;
            if (N > CPO_TRUNC_CAP) return CPO_EINVAL;
            z *= t / (double)N;
        }
        plan->taylor_steps = N < 1 ? 1 : N;
        return CPO_OK;
    }
    return CPO_EINVAL;
}

/* ---- walk operator: src/graph.cpp:257-267 ----------------------------- */
/* y = A D^-1 x as the reference's push/scatter loop (ascending u, zero skip). */
void cpo_apply_walk(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                    const double* x, double* out) {
    memset(out, 0, (size_t)n * sizeof(double));        /* graph.cpp:260 */
    for (uint32_t u = 0; u < n; ++u) {                 /* :261 */
        const double xu = x[u];
        if (xu == 0.0) continue;                       /* :263 */
        /* inv_degree_[u] = 1.0 / d, graph.cpp:79 */
        const double w = xu * (1.0 / (double)(offsets[u + 1] - offsets[u])); /* :264 */
        for (uint64_t i = offsets[u]; i < offsets[u + 1]; ++i) out[nbrs[i]] += w; /* :265 */
    }
}

/* ---- ChebyPower: src/solvers.cpp:197-234 ------------------------------ */
/*
 * values <- sum_{k=0..K} c_k T_k(P) seed with the reference's exact update
 * order.  Optional traces: mass_out[k] = sum(r_k) for k = 0..K (the
 * quantity acceptance.cpp:349-360 / C13 checks), r_trace (K+1)*n residuals
 * and est_trace (K+1)*n partial estimates (the StepObserver arguments,
 * solvers.cpp:215,219,226).  Returns push_work (solvers.cpp:214,223).
 */
int cpo_cheby_power_vec(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                        const double* coeffs, uint64_t K, const double* seed,
                        double* values, double* mass_out, double* r_trace,
                        double* est_trace, uint64_t* push_work) {
    if (K < 1) return CPO_EINVAL; /* :201 */
    double* r_prev = (double*)malloc((size_t)n * sizeof(double));
    double* r_cur = (double*)malloc((size_t)n * sizeof(double));
    double* tmp = (double*)malloc((size_t)n * sizeof(double));
    if (!r_prev || !r_cur || !tmp) { free(r_prev); free(r_cur); free(tmp); return CPO_ENOMEM; }
    const uint64_t vol = offsets[n];
    for (uint32_t u = 0; u < n; ++u) values[u] = coeffs[0] * seed[u]; /* :209 */
    memcpy(r_prev, seed, (size_t)n * sizeof(double));                 /* :211 */
    cpo_apply_walk(n, offsets, nbrs, seed, r_cur);                    /* :212 */
    uint64_t work = vol;                                              /* :214 */
#define OBSERVE(k, r)                                                              \
    do {                                                                           \
        if (mass_out) { double s_ = 0.0; for (uint32_t u = 0; u < n; ++u) s_ += (r)[u]; mass_out[k] = s_; } \
        if (r_trace) memcpy(r_trace + (size_t)(k) * n, (r), (size_t)n * sizeof(double)); \
        if (est_trace) memcpy(est_trace + (size_t)(k) * n, values, (size_t)n * sizeof(double)); \
    } while (0)
    OBSERVE(0, r_prev);                                               /* :215 */
    for (uint64_t k = 1; k < K; ++k) {                                /* :217 */
        const double ck = coeffs[k];
        for (uint32_t u = 0; u < n; ++u) values[u] += ck * r_cur[u];  /* :218 */
        OBSERVE(k, r_cur);                                            /* :219 */
        cpo_apply_walk(n, offsets, nbrs, r_cur, tmp);                 /* :220 */
        for (uint32_t u = 0; u < n; ++u) r_prev[u] = 2.0 * tmp[u] - r_prev[u]; /* :221 */
        double* sw = r_prev; r_prev = r_cur; r_cur = sw;              /* :222 */
        work += vol;                                                  /* :223 */
    }
    for (uint32_t u = 0; u < n; ++u) values[u] += coeffs[K] * r_cur[u]; /* :225 */
    OBSERVE(K, r_cur);                                                /* :226 */
#undef OBSERVE
    if (push_work) *push_work = work;
    free(r_prev); free(r_cur); free(tmp);
    return CPO_OK;
}

/* cheby_power with a unit seed, solvers.cpp:236-239 + unit_vector :27-33. */
int cpo_cheby_power(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                    const double* coeffs, uint64_t K, uint32_t source, double* values,
                    double* mass_out, uint64_t* push_work) {
    if (source >= n) return CPO_EINVAL; /* solvers.cpp:28-29 */
    double* e = (double*)calloc(n, sizeof(double));
    if (!e) return CPO_ENOMEM;
    e[source] = 1.0;
    int rc = cpo_cheby_power_vec(n, offsets, nbrs, coeffs, K, e, values, mass_out, NULL,
                                 NULL, push_work);
    free(e);
    return rc;
}

/* Power method (PwMethod), solvers.cpp:87-116; used for ground truth. */
int cpo_power_method(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                     const double* zeta, uint64_t n_steps, uint32_t source, double* values) {
    if (source >= n || n_steps < 1) return CPO_EINVAL;
    double* r = (double*)calloc(n, sizeof(double));
    double* next = (double*)calloc(n, sizeof(double));
    if (!r || !next) { free(r); free(next); return CPO_ENOMEM; }
    r[source] = 1.0;
    memset(values, 0, (size_t)n * sizeof(double));
    for (uint64_t k = 0; k < n_steps; ++k) {
        const double z = zeta[k];
        for (uint32_t u = 0; u < n; ++u) values[u] += z * r[u];
        if (k + 1 < n_steps) {
            cpo_apply_walk(n, offsets, nbrs, r, next);
            double* sw = r; r = next; next = sw;
        }
    }
    free(r); free(next);
    return CPO_OK;
}

/* ---- select_sources (Uniform): src/eval.cpp:67-90 --------------------- */
int cpo_select_sources_uniform(uint32_t n, uint64_t count, uint64_t seed, uint32_t* out) {
    if (count > n) return CPO_EINVAL; /* eval.cpp:70 */
    uint32_t* ids = (uint32_t*)malloc((size_t)n * sizeof(uint32_t));
    if (!ids) return CPO_ENOMEM;
    for (uint32_t i = 0; i < n; ++i) ids[i] = i;
    cpo_rng rng = {seed};
    for (uint64_t i = 0; i < count; ++i) { /* eval.cpp:75-79 */
        const uint64_t j = i + rng_next_below(&rng, n - i);
        uint32_t t = ids[i]; ids[i] = ids[j]; ids[j] = t;
    }
    memcpy(out, ids, (size_t)count * sizeof(uint32_t));
    free(ids);
    return CPO_OK;
}

/* ---- ring + chords fixture: tests/oracles.hpp:162-178 -----------------
 * Emits the edge pairs of ring_chord_edge_text (labels, in text order);
 * returns the pair count.  pairs must hold 2*(n + extra) int64. */
uint64_t cpo_ring_chord_edges(uint64_t n, uint64_t extra, uint64_t seed, int64_t* pairs) {
    cpo_rng rng = {seed};
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; ++i) { pairs[2 * m] = (int64_t)i; pairs[2 * m + 1] = (int64_t)((i + 1) % n); ++m; }
    for (uint64_t e = 0; e < extra; ++e) {
        const uint64_t a = rng_next_below(&rng, n);
        const uint64_t b = rng_next_below(&rng, n);
        if (a != b) { pairs[2 * m] = (int64_t)a; pairs[2 * m + 1] = (int64_t)b; ++m; }
    }
    return m;
}

/* Random vector fixture, tests/oracles.hpp:191-197. */
void cpo_random_vector(uint64_t n, uint64_t seed, double lo, double hi, double* x) {
    cpo_rng rng = {seed};
    for (uint64_t i = 0; i < n; ++i) x[i] = lo + (hi - lo) * rng_next_double(&rng);
}

/* ---- multi-threaded query pool: tools/chebyprop.cpp:305-334 ------------
 * P workers pull sources from a shared cursor (the reference bench's
 * std::atomic cursor); each runs one single-threaded cheby_power. */
typedef struct {
    uint32_t n;
    const uint64_t* offsets;
    const uint32_t* nbrs;
    const double* coeffs;
    uint64_t K;
    const uint32_t* sources;
    uint64_t n_sources;
    double* out; /* n_sources * n, or NULL (results discarded) */
    uint64_t cursor;
    int rc;
} cpo_pool;

static void* pool_worker(void* arg) {
    cpo_pool* p = (cpo_pool*)arg;
    double* scratch = NULL;
    if (!p->out) scratch = (double*)malloc((size_t)p->n * sizeof(double));
    for (;;) {
        uint64_t i = __atomic_fetch_add(&p->cursor, 1, __ATOMIC_RELAXED);
        if (i >= p->n_sources) break;
        double* dst = p->out ? p->out + i * (uint64_t)p->n : scratch;
        int rc = cpo_cheby_power(p->n, p->offsets, p->nbrs, p->coeffs, p->K, p->sources[i],
                                 dst, NULL, NULL);
        if (rc) p->rc = rc;
    }
    free(scratch);
    return NULL;
}

int cpo_cheby_power_pool(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                         const double* coeffs, uint64_t K, const uint32_t* sources,
                         uint64_t n_sources, double* out, int n_threads) {
    cpo_pool p = {n, offsets, nbrs, coeffs, K, sources, n_sources, out, 0, 0};
    if (n_threads <= 1) { pool_worker(&p); return p.rc; }
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, pool_worker, &p);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
    free(th);
    return p.rc;
}

/* ---- edge-list ingest: src/graph.cpp:113-171 ----------------------------
 * Label pairs -> CSR with self-loops dropped (:149), ids interned in
 * first-seen order from surviving edges (:120-124, :150-151), symmetrised
 * (:152-153), sorted and deduplicated (:158-160).  Two calls: first with
 * offsets/nbrs NULL to get n and nnz, then with buffers of that size. */
static int cmp_u64(const void* a, const void* b) {
    uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    return x < y ? -1 : x > y;
}

typedef struct { int64_t label; uint32_t id; int used; } intern_slot;

int cpo_edges_to_csr(const int64_t* pairs, uint64_t m, uint32_t* n_out, uint64_t* nnz_out,
                     uint64_t* offsets, uint32_t* nbrs) {
    uint64_t cap = 16;
    while (cap < 4 * m + 16) cap <<= 1;
    intern_slot* tab = (intern_slot*)calloc(cap, sizeof(intern_slot));
    uint64_t* half = (uint64_t*)malloc((2 * m + 1) * sizeof(uint64_t));
    if (!tab || !half) { free(tab); free(half); return CPO_ENOMEM; }
    uint32_t n = 0;
    uint64_t h = 0;
    for (uint64_t e = 0; e < m; ++e) {
        int64_t a = pairs[2 * e], b = pairs[2 * e + 1];
        if (a == b) continue;
        uint32_t id[2];
        int64_t lab[2] = {a, b};
        for (int s = 0; s < 2; ++s) {
            uint64_t hh = ((uint64_t)lab[s] * 0x9e3779b97f4a7c15ull) & (cap - 1);
            while (tab[hh].used && tab[hh].label != lab[s]) hh = (hh + 1) & (cap - 1);
            if (!tab[hh].used) { tab[hh].used = 1; tab[hh].label = lab[s]; tab[hh].id = n++; }
            id[s] = tab[hh].id;
        }
        half[h++] = ((uint64_t)id[0] << 32) | id[1];
        half[h++] = ((uint64_t)id[1] << 32) | id[0];
    }
    free(tab);
    if (h == 0) { free(half); return CPO_EINVAL; } /* graph.cpp:156 */
    qsort(half, h, sizeof(uint64_t), cmp_u64);
    uint64_t u = 0;
    for (uint64_t i = 0; i < h; ++i)
        if (i == 0 || half[i] != half[i - 1]) half[u++] = half[i];
    *n_out = n;
    *nnz_out = u;
    if (offsets && nbrs) {
        memset(offsets, 0, ((size_t)n + 1) * sizeof(uint64_t));
        for (uint64_t i = 0; i < u; ++i) {
            offsets[(half[i] >> 32) + 1]++;
            nbrs[i] = (uint32_t)(half[i] & 0xffffffffu);
        }
        for (uint32_t i = 1; i <= n; ++i) offsets[i] += offsets[i - 1];
    }
    free(half);
    return CPO_OK;
}

/* ---- steady-state iteration sample for huge graphs --------------------------
 * n_threads threads each run the reference's apply_walk inner loop
 * (graph.cpp:261-266: w = x[u] * inv_deg[u]; out[v] += w for v in N(u)) over a
 * dense seeded vector for a contiguous run of source rows starting at a
 * thread-specific offset until ~edges_per_thread edges are processed (0 =
 * the whole graph, i.e. one full iteration).  The scatter still targets the
 * full-length out vector, so the memory behaviour is the reference's.
 * Vector allocation and fill run before a start barrier, outside the clock.
 * Returns wall seconds; *edges_done = edges processed by all threads. */
typedef struct {
    uint32_t n;
    const uint64_t* offsets;
    const uint32_t* nbrs;
    uint64_t seed;
    uint32_t row0;
    uint64_t edge_budget;
    uint64_t edges;
    int failed;
    pthread_barrier_t* start;
    double t_end;
} cpo_walk_job;

static double now_secs(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static void* walk_worker(void* arg) {
    cpo_walk_job* j = (cpo_walk_job*)arg;
    double* x = (double*)malloc((size_t)j->n * sizeof(double));
    double* out = (double*)calloc((size_t)j->n, sizeof(double));
    if (!x || !out) j->failed = 1;
    else cpo_random_vector(j->n, j->seed, 0.0, 1.0, x);
    pthread_barrier_wait(j->start);
    if (j->failed) { free(x); free(out); return NULL; }
    uint64_t done = 0;
    uint32_t u = j->row0;
    for (uint32_t cnt = 0; cnt < j->n && done < j->edge_budget; ++cnt) {
        const double xu = x[u];
        if (xu != 0.0) {
            const double w = xu * (1.0 / (double)(j->offsets[u + 1] - j->offsets[u]));
            for (uint64_t i = j->offsets[u]; i < j->offsets[u + 1]; ++i) out[j->nbrs[i]] += w;
        }
        done += j->offsets[u + 1] - j->offsets[u];
        if (++u == j->n) u = 0;
    }
    j->edges = done;
    j->t_end = now_secs();
    free(x); free(out);
    return NULL;
}

double cpo_apply_walk_pool(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs, int n_threads,
                           uint64_t edges_per_thread, uint64_t* edges_done) {
    if (n_threads < 1) n_threads = 1;
    if (edges_per_thread == 0) edges_per_thread = offsets[n];
    pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)n_threads);
    cpo_walk_job* jobs = (cpo_walk_job*)calloc((size_t)n_threads, sizeof(cpo_walk_job));
    pthread_barrier_t start;
    pthread_barrier_init(&start, NULL, (unsigned)n_threads + 1u);
    for (int i = 0; i < n_threads; ++i) {
        jobs[i] = (cpo_walk_job){n, offsets, nbrs, (uint64_t)(1000 + i),
                                 (uint32_t)(((uint64_t)i * n) / (uint64_t)n_threads), edges_per_thread, 0, 0,
                                 &start, 0.0};
        pthread_create(&th[i], NULL, walk_worker, &jobs[i]);
    }
    pthread_barrier_wait(&start);
    const double t = now_secs();
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
    pthread_barrier_destroy(&start);
    double wall = 0.0;
    uint64_t total = 0;
    for (int i = 0; i < n_threads; ++i) {
        if (jobs[i].failed) wall = -1;
        else if (wall >= 0 && jobs[i].t_end - t > wall) wall = jobs[i].t_end - t;
        total += jobs[i].edges;
    }
    if (edges_done) *edges_done = total;
    free(th); free(jobs);
    return wall;
}

/* ---- row-parallel pull restatement of cheby_power (multi-threaded) ---------
 * Same arithmetic as cpo_cheby_power_vec / the reference, bit for bit, but the
 * walk operator is evaluated row by row (pull) so the rows can be split over
 * threads:
 *
 *   reference (graph.cpp:260-266): out[v] = 0; for u = 0..n-1 ascending, if
 *   x[u] != 0: out[v] += x[u] * inv_degree(u) for every v in N(u).
 *
 * On a symmetric CSR with sorted rows (Graph::from_csr's invariants,
 * graph.cpp:84-95) the u that add into out[v] are exactly N(v), met in
 * ascending order, so out[v] = (((0 + y[u1]) + y[u2]) + ...) over N(v) sorted,
 * with y[u] = x[u] * (1.0 / d_u).  A skipped zero x[u] is represented by
 * y[u] = -0.0, which is an exact additive identity (s + -0.0 == s for every s,
 * including +0.0), so skipping and adding agree bit for bit.
 *
 * The dense passes (solvers.cpp:209, 218, 221, 225) are per-element and are
 * fused into the row pass with the same expressions:
 *   values[v] += c_k * r_cur[v];  r_next[v] = 2.0 * tmp[v] - r_prev[v].
 * S columns (sources or dense seeds) run interleaved ([n][S] layout) so one
 * gathered cache line serves all of them; each column's arithmetic is the
 * single-column arithmetic.  Pinned bit-for-bit against the reference library
 * in tests/test_oracle_pin.py. */
typedef struct {
    uint32_t n, S;
    const uint64_t* off;
    const uint32_t* nb;
    const double* y;     /* [n][S] gathered: x * inv_degree, -0.0 where x == 0 */
    double* y_next;      /* [n][S] next step's y */
    double* r_prev;      /* [n][S] in: T_{k-1}, out: T_{k+1} (in place) */
    const double* r_cur; /* [n][S] T_k */
    double* values;      /* [n][S] */
    double ck;           /* c_k added before the walk (solvers.cpp:218) */
    int mode;            /* 0: first walk (r_prev <- P seed), 1: recurrence step */
    const uint32_t* chunk_rows; /* chunk boundaries (rows) */
    uint32_t n_chunks;
    uint32_t cursor;
} pull_job;

static inline double pull_y(double x, uint64_t d) {
    return x == 0.0 ? -0.0 : x * (1.0 / (double)d); /* graph.cpp:79, :263-264 */
}

static void* pull_worker(void* arg) {
    pull_job* j = (pull_job*)arg;
    const uint32_t S = j->S;
    double acc[64];
    for (;;) {
        const uint32_t c = __atomic_fetch_add(&j->cursor, 1, __ATOMIC_RELAXED);
        if (c >= j->n_chunks) break;
        for (uint32_t v = j->chunk_rows[c]; v < j->chunk_rows[c + 1]; ++v) {
            for (uint32_t s = 0; s < S; ++s) acc[s] = 0.0; /* out.assign(n, 0.0), graph.cpp:260 */
            const uint64_t b = j->off[v], e = j->off[v + 1];
            for (uint64_t i = b; i < e; ++i) {
                if (i + 16 < e) __builtin_prefetch(j->y + (size_t)j->nb[i + 16] * S);
                const double* yu = j->y + (size_t)j->nb[i] * S;
                for (uint32_t s = 0; s < S; ++s) acc[s] += yu[s]; /* :265 */
            }
            const uint64_t dv = e - b;
            double* rp = j->r_prev + (size_t)v * S;
            double* yn = j->y_next + (size_t)v * S;
            if (j->mode == 0) { /* r_cur = apply_walk(seed), solvers.cpp:212 */
                for (uint32_t s = 0; s < S; ++s) { rp[s] = acc[s]; yn[s] = pull_y(acc[s], dv); }
            } else {
                const double* rc = j->r_cur + (size_t)v * S;
                double* val = j->values + (size_t)v * S;
                for (uint32_t s = 0; s < S; ++s) {
                    val[s] += j->ck * rc[s];                   /* :218 */
                    const double r = 2.0 * acc[s] - rp[s];     /* :221 */
                    rp[s] = r;
                    yn[s] = pull_y(r, dv);
                }
            }
        }
    }
    return NULL;
}

static void pull_run(pull_job* j, int n_threads) {
    j->cursor = 0;
    if (n_threads <= 1) { pull_worker(j); return; }
    pthread_t th[256];
    if (n_threads > 256) n_threads = 256;
    for (int i = 0; i < n_threads; ++i) pthread_create(&th[i], NULL, pull_worker, j);
    for (int i = 0; i < n_threads; ++i) pthread_join(th[i], NULL);
}

/* values[S][n] <- cheby_power_vec for S dense seeds (seeds[S][n]), pull form. */
int cpo_cheby_power_vec_pull(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                             const double* coeffs, uint64_t K, const double* seeds, uint32_t S,
                             double* values_out, int n_threads) {
    if (K < 1 || S < 1 || S > 64) return CPO_EINVAL; /* solvers.cpp:201 */
    const size_t N = (size_t)n * S;
    double* y0 = (double*)malloc(N * sizeof(double));
    double* y1 = (double*)malloc(N * sizeof(double));
    double* ra = (double*)malloc(N * sizeof(double));
    double* rb = (double*)malloc(N * sizeof(double));
    double* val = (double*)malloc(N * sizeof(double));
    /* chunks of ~2^16 edges or 4096 rows, claimed dynamically (hub rows are long) */
    uint32_t cap = 1024, nc = 0;
    uint32_t* rows = (uint32_t*)malloc(sizeof(uint32_t) * (cap + 1));
    if (!y0 || !y1 || !ra || !rb || !val || !rows) {
        free(y0); free(y1); free(ra); free(rb); free(val); free(rows);
        return CPO_ENOMEM;
    }
    rows[0] = 0;
    for (uint32_t v = 0; v < n;) {
        uint32_t e = v;
        const uint64_t start = offsets[v];
        while (e < n && e - v < 4096 && offsets[e + 1] - start < (1u << 16)) ++e;
        if (e == v) ++e;
        if (nc + 1 >= cap) {
            cap *= 2;
            uint32_t* nr = (uint32_t*)realloc(rows, sizeof(uint32_t) * (cap + 1));
            if (!nr) { free(y0); free(y1); free(ra); free(rb); free(val); free(rows); return CPO_ENOMEM; }
            rows = nr;
        }
        rows[++nc] = e;
        v = e;
    }
    /* k = 0: values = c0 * seed (:209), r_prev = seed (:211), y0 = seed * inv_deg */
    for (uint32_t u = 0; u < n; ++u) {
        const uint64_t d = offsets[u + 1] - offsets[u];
        for (uint32_t s = 0; s < S; ++s) {
            const double x = seeds[(size_t)s * n + u];
            val[(size_t)u * S + s] = coeffs[0] * x;
            rb[(size_t)u * S + s] = x;
            y0[(size_t)u * S + s] = pull_y(x, d);
        }
    }
    pull_job j = {n, S, offsets, nbrs, y0, y1, ra, NULL, val, 0.0, 0, rows, nc, 0};
    pull_run(&j, n_threads); /* ra = P seed = r_cur (:212); y1 = its y */
    double* r_prev = rb;     /* T_{k-1} */
    double* r_cur = ra;      /* T_k */
    double* y_cur = y1;
    double* y_nxt = y0;
    for (uint64_t k = 1; k < K; ++k) { /* :217-224 */
        j.y = y_cur; j.y_next = y_nxt; j.r_prev = r_prev; j.r_cur = r_cur;
        j.ck = coeffs[k]; j.mode = 1;
        pull_run(&j, n_threads);
        double* t = r_prev; r_prev = r_cur; r_cur = t; /* :222 */
        t = y_cur; y_cur = y_nxt; y_nxt = t;
    }
    const double cK = coeffs[K];
    for (uint32_t u = 0; u < n; ++u)
        for (uint32_t s = 0; s < S; ++s) {
            const double v = val[(size_t)u * S + s] + cK * r_cur[(size_t)u * S + s]; /* :225 */
            values_out[(size_t)s * n + u] = v;
        }
    free(y0); free(y1); free(ra); free(rb); free(val); free(rows);
    return CPO_OK;
}

/* cheby_power for S unit seeds (solvers.cpp:236-239), pull form, values[S][n]. */
int cpo_cheby_power_pull(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs,
                         const double* coeffs, uint64_t K, const uint32_t* sources, uint32_t S,
                         double* values_out, int n_threads) {
    if (S < 1 || S > 64) return CPO_EINVAL;
    for (uint32_t s = 0; s < S; ++s)
        if (sources[s] >= n) return CPO_EINVAL; /* solvers.cpp:28-29 */
    double* seeds = (double*)calloc((size_t)n * S, sizeof(double));
    if (!seeds) return CPO_ENOMEM;
    for (uint32_t s = 0; s < S; ++s) seeds[(size_t)s * n + sources[s]] = 1.0;
    const int rc = cpo_cheby_power_vec_pull(n, offsets, nbrs, coeffs, K, seeds, S, values_out, n_threads);
    free(seeds);
    return rc;
}
