/*
 * oracle/graphgen_port.c -- CPU restatement of the repo's seeded synthetic
 * graph generators (paper_2412_10789_b200/csrc/graphgen.cu).
 *
 * TEST INFRASTRUCTURE ONLY.  The generators are input preparation, not the
 * reference's algorithm (the reference ships no R-MAT / Chung-Lu generator;
 * SURVEY.md 8d defines the configs).  This restatement exists so that the CPU
 * arms (bench.py --impl reference, the cpu_baseline leg) can build the same
 * CSR on the host without loading the product library.  It is pinned equal
 * to the product's host and device builds in tests/test_oracle_pin.py.
 *
 * Draw i of a graph uses the SplitMix64 stream addressed by (seed, i) (the
 * rng.hpp:30-35 stream idea; state = seed ^ golden*(i+1), advanced once).
 * R-MAT picks a quadrant per level with probabilities (a, b, c, d); Chung-Lu
 * draws both endpoints by inverse-CDF search over power-law expected-degree
 * weights.  Self-loops are dropped, every edge is symmetrised, rows are sorted
 * and deduplicated, and isolated ids are compacted in ascending order -- the
 * invariants Graph::from_csr demands (graph.cpp:48-104).
 *
 * Layout of the build (multi-threaded; memory ~ 8.5 B per sampled edge end
 * plus 4 B per id per thread):
 *   pass 1: draw every pair, count row lengths (with duplicates) per thread
 *   pass 2: draw again, scatter each end into its row at a per-thread cursor
 *   rows sorted + deduplicated in place, ids compacted, rows copied out.
 */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GP_OK 0
#define GP_EINVAL 1
#define GP_ENOMEM 4

static inline uint64_t gp_next(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
static inline double gp_double(uint64_t* s) { return (double)(gp_next(s) >> 11) * 0x1.0p-53; }
static inline uint64_t gp_stream(uint64_t seed, uint64_t tag) {
    uint64_t s = seed ^ (0x9e3779b97f4a7c15ull * (tag + 1));
    gp_next(&s);
    return s;
}

typedef struct {
    int kind; /* 0 = R-MAT, 1 = Chung-Lu */
    uint64_t seed;
    uint32_t scale;
    double a, ab, abc;
    const double* cdf;
    uint32_t n_ids;
} gp_model;

/* returns 0 for a self-loop */
static inline int gp_pair(const gp_model* m, uint64_t i, uint32_t* pu, uint32_t* pv) {
    uint64_t s = gp_stream(m->seed, i);
    uint32_t u = 0, v = 0;
    if (m->kind == 0) {
        for (uint32_t l = 0; l < m->scale; ++l) {
            const double r = gp_double(&s);
            /* branch-free: the quadrant draws are unpredictable */
            const uint32_t bu = (uint32_t)(r >= m->ab);
            const uint32_t bv = ((uint32_t)(r >= m->a) & (uint32_t)(r < m->ab)) | (uint32_t)(r >= m->abc);
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
    } else {
        const double total = m->cdf[m->n_ids - 1];
        for (int side = 0; side < 2; ++side) {
            const double x = gp_double(&s) * total;
            uint32_t lo = 0, hi = m->n_ids - 1; /* first i with cdf[i] > x */
            while (lo < hi) {
                const uint32_t mid = (lo + hi) >> 1;
                if (m->cdf[mid] > x) hi = mid; else lo = mid + 1;
            }
            if (side == 0) u = lo; else v = lo;
        }
    }
    *pu = u;
    *pv = v;
    return u != v;
}

typedef struct {
    const gp_model* m;
    uint64_t i0, i1;
    int pass;
    uint32_t* cnt;  /* this thread's row counters: pass 1 counts, pass 2 write cursors */
    const uint64_t* start;
    uint32_t* slots;
    uint64_t* pairs; /* [n_samples] (u << 32 | v) from pass 1, replayed by pass 2 */
} gp_draw_job;

/* Pass 1 draws (and keeps the pairs: 8 B per sample), pass 2 replays them.
 * Thread-private counters (no atomics: hot R-MAT rows share cache lines, and
 * contended atomics on them cost more than the draws).  Pass 2 writes each
 * end at slots[start[row] + cursor_t[row]++], with cursor_t[row] = the counts
 * of the threads before t (within-row, so 32 bits), so the row contents are
 * in draw order. */
static void* gp_draw_worker(void* arg) {
    gp_draw_job* j = (gp_draw_job*)arg;
    uint32_t u, v;
    uint32_t* cnt = j->cnt;
    if (j->pass == 1) {
        for (uint64_t i = j->i0; i < j->i1; ++i) {
            const int keep = gp_pair(j->m, i, &u, &v);
            j->pairs[i] = ((uint64_t)u << 32) | v;
            if (keep) { ++cnt[u]; ++cnt[v]; }
        }
    } else {
        for (uint64_t i = j->i0; i < j->i1; ++i) {
            u = (uint32_t)(j->pairs[i] >> 32);
            v = (uint32_t)j->pairs[i];
            if (u == v) continue; /* self-loop */
            j->slots[j->start[u] + cnt[u]++] = v;
            j->slots[j->start[v] + cnt[v]++] = u;
        }
    }
    return NULL;
}

static int cmp_u32(const void* a, const void* b) {
    const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

typedef struct {
    uint32_t ids;
    const uint64_t* start;
    uint32_t* slots;
    uint32_t* len; /* in: raw length; out: deduplicated length */
    uint32_t cursor;
    /* copy phase */
    const uint32_t* newid;
    const uint64_t* off_of_id; /* new offsets indexed by old id */
    uint32_t* nbr;
    int phase;
} gp_row_job;

#define GP_ROW_CHUNK 4096u

static void* gp_row_worker(void* arg) {
    gp_row_job* j = (gp_row_job*)arg;
    for (;;) {
        const uint32_t c = __atomic_fetch_add(&j->cursor, 1u, __ATOMIC_RELAXED);
        const uint64_t r0 = (uint64_t)c * GP_ROW_CHUNK;
        if (r0 >= j->ids) break;
        const uint64_t r1 = r0 + GP_ROW_CHUNK < j->ids ? r0 + GP_ROW_CHUNK : j->ids;
        for (uint64_t r = r0; r < r1; ++r) {
            uint32_t* row = j->slots + j->start[r];
            const uint32_t L = j->len[r];
            if (j->phase == 0) {
                if (L < 2) continue;
                if (L <= 24) { /* insertion sort */
                    for (uint32_t a = 1; a < L; ++a) {
                        const uint32_t x = row[a];
                        uint32_t b = a;
                        while (b > 0 && row[b - 1] > x) { row[b] = row[b - 1]; --b; }
                        row[b] = x;
                    }
                } else {
                    qsort(row, L, sizeof(uint32_t), cmp_u32);
                }
                uint32_t w = 1;
                for (uint32_t a = 1; a < L; ++a)
                    if (row[a] != row[w - 1]) row[w++] = row[a];
                j->len[r] = w;
            } else if (L) {
                uint32_t* dst = j->nbr + j->off_of_id[r];
                for (uint32_t a = 0; a < L; ++a) dst[a] = j->newid[row[a]];
            }
        }
    }
    return NULL;
}

static int gp_threads(int n_threads) {
    if (n_threads < 1) n_threads = 1;
    return n_threads > 256 ? 256 : n_threads;
}

static void gp_run_rows(gp_row_job* j, int nt) {
    if (nt > 256) nt = 256;
    pthread_t th[256];
    j->cursor = 0;
    for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, gp_row_worker, j);
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
}

typedef struct {
    uint32_t ids, nt, r0, r1;
    uint32_t** cnt; /* [nt][ids] */
    uint64_t* len;  /* [ids] total per row */
} gp_merge_job;

static void* gp_merge_worker(void* arg) { /* per row: total count */
    gp_merge_job* j = (gp_merge_job*)arg;
    for (uint32_t r = j->r0; r < j->r1; ++r) {
        uint64_t s = 0;
        for (uint32_t t = 0; t < j->nt; ++t) s += j->cnt[t][r];
        j->len[r] = s;
    }
    return NULL;
}

typedef struct {
    uint32_t nt, r0, r1;
    uint32_t** cnt;
    const uint64_t* start;
} gp_cursor_job;

static void* gp_cursor_worker(void* arg) { /* per row: thread t's first slot */
    gp_cursor_job* j = (gp_cursor_job*)arg;
    for (uint32_t r = j->r0; r < j->r1; ++r) {
        uint32_t p = 0; /* a row holds < 2^32 ends (checked by the caller) */
        for (uint32_t t = 0; t < j->nt; ++t) {
            const uint32_t c = j->cnt[t][r];
            j->cnt[t][r] = p;
            p += c;
        }
    }
    return NULL;
}

static int gp_build(const gp_model* m, uint32_t ids, uint64_t n_samples, int n_threads, uint64_t** off_out,
                    uint32_t** nbr_out, uint32_t* n_out, uint64_t* nnz_out) {
    const int nt = gp_threads(n_threads);
    uint32_t* cnt[256];
    pthread_t th[256];
    memset(cnt, 0, sizeof(cnt));
    uint64_t* start = (uint64_t*)malloc(((size_t)ids + 1) * sizeof(uint64_t));
    uint64_t* len = (uint64_t*)malloc((size_t)ids * sizeof(uint64_t));
    int rc = GP_ENOMEM;
    uint32_t* slots = NULL;
    uint64_t* pairs = (uint64_t*)malloc((n_samples ? n_samples : 1) * sizeof(uint64_t));
    if (!start || !len || !pairs) goto out;
    for (int t = 0; t < nt; ++t)
        if (!(cnt[t] = (uint32_t*)calloc((size_t)ids, sizeof(uint32_t)))) goto out;
    gp_draw_job jobs[256];
    for (int t = 0; t < nt; ++t) {
        jobs[t] = (gp_draw_job){m, n_samples * (uint64_t)t / (uint64_t)nt, n_samples * (uint64_t)(t + 1) / (uint64_t)nt,
                                1, cnt[t], start, NULL, pairs};
        pthread_create(&th[t], NULL, gp_draw_worker, &jobs[t]);
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    {
        gp_merge_job mj[256];
        for (int t = 0; t < nt; ++t) {
            mj[t] = (gp_merge_job){ids, (uint32_t)nt, (uint32_t)((uint64_t)ids * t / nt),
                                   (uint32_t)((uint64_t)ids * (t + 1) / nt), cnt, len};
            pthread_create(&th[t], NULL, gp_merge_worker, &mj[t]);
        }
        for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    }
    start[0] = 0;
    for (uint32_t r = 0; r < ids; ++r) {
        if (len[r] >= (1ull << 32)) { rc = GP_EINVAL; goto out; } /* 32-bit in-row cursors */
        start[r + 1] = start[r] + len[r];
    }
    if (!(slots = (uint32_t*)malloc((start[ids] ? start[ids] : 1) * sizeof(uint32_t)))) goto out;
    {
        gp_cursor_job cj[256];
        for (int t = 0; t < nt; ++t) {
            cj[t] = (gp_cursor_job){(uint32_t)nt, (uint32_t)((uint64_t)ids * t / nt),
                                    (uint32_t)((uint64_t)ids * (t + 1) / nt), cnt, start};
            pthread_create(&th[t], NULL, gp_cursor_worker, &cj[t]);
        }
        for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    }
    for (int t = 0; t < nt; ++t) {
        jobs[t].pass = 2;
        jobs[t].slots = slots;
        pthread_create(&th[t], NULL, gp_draw_worker, &jobs[t]);
    }
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    for (int t = 1; t < nt; ++t) { free(cnt[t]); cnt[t] = NULL; }
    free(pairs);
    pairs = NULL;
    {
        /* sort + dedup every row; cnt[0] becomes the deduplicated length */
        uint32_t* dl = cnt[0];
        for (uint32_t r = 0; r < ids; ++r) dl[r] = (uint32_t)len[r];
        gp_row_job rj = {ids, start, slots, dl, 0, NULL, NULL, NULL, 0};
        gp_run_rows(&rj, nt);
        uint32_t* newid = (uint32_t*)malloc((size_t)ids * sizeof(uint32_t));
        uint64_t* off_of_id = len; /* reuse */
        if (!newid) goto out;
        uint32_t n = 0;
        uint64_t nnz = 0;
        for (uint32_t r = 0; r < ids; ++r) {
            newid[r] = n;
            off_of_id[r] = nnz;
            if (dl[r]) { ++n; nnz += dl[r]; }
        }
        if (nnz == 0) { free(newid); rc = GP_EINVAL; goto out; } /* empty graph */
        uint64_t* off = (uint64_t*)malloc(((size_t)n + 1) * sizeof(uint64_t));
        uint32_t* nbr = (uint32_t*)malloc(nnz * sizeof(uint32_t));
        if (!off || !nbr) { free(off); free(nbr); free(newid); goto out; }
        for (uint32_t r = 0; r < ids; ++r)
            if (dl[r]) off[newid[r]] = off_of_id[r];
        off[n] = nnz;
        gp_row_job cpj = {ids, start, slots, dl, 0, newid, off_of_id, nbr, 1};
        gp_run_rows(&cpj, nt);
        free(newid);
        *off_out = off;
        *nbr_out = nbr;
        *n_out = n;
        *nnz_out = nnz;
        rc = GP_OK;
    }
out:
    for (int t = 0; t < nt; ++t) free(cnt[t]);
    free(slots);
    free(pairs);
    free(start);
    free(len);
    return rc;
}

/* R-MAT over 2^scale ids (graphgen.cu: cpg_gen_rmat).  Caller frees with cpo_gen_free. */
int cpo_gen_rmat(uint32_t scale, uint64_t n_samples, double a, double b, double c, uint64_t seed,
                 int n_threads, uint64_t** off, uint32_t** nbr, uint32_t* n, uint64_t* nnz) {
    if (scale < 1 || scale > 31 || a < 0 || b < 0 || c < 0 || a + b + c > 1.0) return GP_EINVAL;
    gp_model m = {0, seed, scale, a, a + b, a + b + c, NULL, 0};
    return gp_build(&m, 1u << scale, n_samples, n_threads, off, nbr, n, nnz);
}

/* Chung-Lu (graphgen.cu: chunglu_cdf + cpg_gen_chunglu): w_i = (i+1)^(-1/(gamma-1)),
 * rescaled to the target mean degree with the cap enforced, as a CDF. */
int cpo_gen_chunglu(uint32_t n_ids, uint64_t n_samples, double exponent, double mean_degree,
                    uint32_t max_degree, uint64_t seed, int n_threads, uint64_t** off, uint32_t** nbr,
                    uint32_t* n, uint64_t* nnz) {
    if (n_ids < 2 || !(exponent > 1.0)) return GP_EINVAL;
    double* w = (double*)malloc((size_t)n_ids * sizeof(double));
    if (!w) return GP_ENOMEM;
    const double beta = 1.0 / (exponent - 1.0);
    for (uint32_t i = 0; i < n_ids; ++i) w[i] = pow((double)i + 1.0, -beta);
    const double target = mean_degree * n_ids;
    for (int round = 0; round < 50; ++round) {
        double sum = 0.0;
        for (uint32_t i = 0; i < n_ids; ++i) sum += w[i];
        const double s = target / sum;
        int capped = 0;
        for (uint32_t i = 0; i < n_ids; ++i) {
            w[i] *= s;
            if (max_degree && w[i] > max_degree) { w[i] = max_degree; capped = 1; }
        }
        if (!capped) break;
    }
    double acc = 0.0;
    for (uint32_t i = 0; i < n_ids; ++i) w[i] = (acc += w[i]); /* in place: the CDF */
    gp_model m = {1, seed, 0, 0, 0, 0, w, n_ids};
    const int rc = gp_build(&m, n_ids, n_samples, n_threads, off, nbr, n, nnz);
    free(w);
    return rc;
}

void cpo_gen_free(uint64_t* off, uint32_t* nbr) {
    free(off);
    free(nbr);
}
