/*
 * cpg.h -- C ABI of the B200-native ChebyPower library (libcpg.so).
 *
 * This is the drop-in boundary for the reference's ChebyPower path
 * (reference paths relative to /root/reference/proj):
 *
 *   Estimate cheby_power(const Graph&, const Kernel&, NodeId source,
 *                        std::size_t cheby_steps, const StepObserver& = {})
 *                                               include/chebyprop/solvers.hpp:59-61
 *   Estimate cheby_power_vec(const Graph&, const Kernel&, const NodeVector& seed,
 *                            std::size_t cheby_steps, ...)   solvers.hpp:62-64
 *   std::vector<double> ppr_cheby_coeffs / hkpr_cheby_coeffs   kernels.hpp:69-74
 *   TruncationPlan plan_truncation(const Kernel&, double)      kernels.hpp:81
 *   Graph::from_csr validation                                  graph.hpp:51-53
 *   general_gp_matrix (batched columns)                         solvers.hpp:107-111
 *
 * Plain pointers and sizes only; no C++ or torch types.  Every entry returns
 * a status code; cpg_last_error() gives the calling thread's message for the
 * last failure.  Status mapping to the reference's exceptions (error.hpp):
 *   CPG_EINVAL  -> ParameterError   (bad source, K < 1, bad alpha/t/eps, length)
 *   CPG_ESTRUCT -> StructuralError  (invalid CSR, empty graph after cleaning)
 *   CPG_EPARSE  -> ParseError       (edge-list text, CPGR / CPGT headers)
 *   CPG_EIO     -> IoError          (cannot open / write a file)
 *   CPG_ECUDA / CPG_ENOMEM / CPG_ENCCL -> runtime failures (no CPU fallback).
 *
 * Node ids, offsets and the CSR layout are the reference's own
 * (Graph::offsets() uint64[n+1], Graph::neighbor_array() uint32[2m],
 * graph.hpp:40-41), so a reference Graph can be handed over without copies.
 */
#ifndef CPG_H
#define CPG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    CPG_OK = 0,
    CPG_EINVAL = 1,
    CPG_ECUDA = 2,
    CPG_ENCCL = 3,
    CPG_ENOMEM = 4,
    CPG_ESTRUCT = 5,
    CPG_EPARSE = 6,   /* ParseError: malformed text / binary cache (error.hpp:8-10) */
    CPG_EIO = 7       /* IoError: cannot open / read / write (error.hpp:28-30)      */
};

enum { CPG_PPR = 0, CPG_HKPR = 1 };

typedef struct cpg_graph cpg_graph;
typedef struct cpg_loopback_group cpg_loopback_group;

/* SolveStats (solvers.hpp:18-25) plus device-side evidence. */
typedef struct {
    uint32_t iterations;   /* K per query (solvers.cpp:228)                  */
    uint64_t push_work;    /* K * vol summed over queries (solvers.cpp:214)  */
    double wall_seconds;   /* host wall time of the call                     */
    double device_ms;      /* CUDA-event time of the K steps (all queries)   */
    double mass_err_max;   /* max_k |sum T_k - sum seed| over queries/steps  */
    double bytes_model;    /* algorithmic HBM bytes           */
    uint32_t launches;     /* kernels launched by this call                  */
    double step_ms;        /* summed CUDA-event time of the step kernels only
                              (filled when cpg_set_profiling(1); else 0)     */
    uint32_t step_launches;/* step-kernel launches behind step_ms            */
} cpg_stats;

/* TruncationPlan (kernels.hpp:48-53). */
typedef struct {
    uint64_t cheby_steps;
    uint64_t taylor_steps;
    double epsilon;
    double tail_bound;
} cpg_plan;

/* Graph description produced at upload (read-only). */
typedef struct {
    uint32_t n;            /* nodes of the whole graph                       */
    uint64_t nnz;          /* 2m of the whole graph                          */
    uint32_t n_local;      /* rows owned by this handle (shard)              */
    uint64_t nnz_local;
    uint32_t row_begin;    /* first owned row in the device (relabelled) order */
    uint32_t n_padded;     /* length of the replicated iterate (ranks*rows)  */
    uint32_t n_hubs;       /* rows split across CTAs                         */
    uint32_t n_items;      /* work items per single-source step              */
    uint32_t max_degree;
    int rank, nranks, device;
    uint64_t structure_hash; /* FNV-1a of (n, m, offsets, neighbors), graph.cpp:97-102 */
    int chunks;            /* row chunks per rank (one all-gather each)      */
    int fused_allgather;   /* 1: batched steps store rows into every rank's replica
                              (CPG_P2P=1, NCCL symmetric windows); 0: NCCL all-gather */
} cpg_graph_info;

const char* cpg_last_error(void);
const char* cpg_version(void);
/* Bracket every step-kernel launch with CUDA events (cpg_stats.step_ms). */
void cpg_set_profiling(int on);

/* ---- host-side math (kernels.cpp restated in C++) ------------------------ */
int cpg_ppr_cheby_coeffs(double alpha, uint64_t max_index, double* out);   /* kernels.cpp:157-170 */
int cpg_hkpr_cheby_coeffs(double t, uint64_t max_index, double* out);      /* kernels.cpp:172-194 */
int cpg_cheby_coeffs(int family, double param, uint64_t max_index, double* out);
int cpg_plan_truncation(int family, double param, double epsilon, cpg_plan* out); /* :253-341 */
/* Taylor (power-basis) coefficients zeta_0..zeta_max (kernels.cpp:78-96). */
int cpg_taylor_coeffs(int family, double param, uint64_t max_index, double* out);
/* Ground-truth truncation N (eval.cpp:39-50): ceil(ln 1e20 / alpha), ceil(2 t ln 1e20). */
uint64_t cpg_ground_truth_steps(int family, double param);
/* "ppr:alpha=0.2" / "hkpr:t=5" (kernels.cpp:343-362) */
int cpg_parse_kernel_spec(const char* spec, int* family, double* param);

/* Graph::from_csr invariants (graph.cpp:48-104) + FNV-1a structure hash. */
int cpg_validate_csr(const uint64_t* offsets, const uint32_t* neighbors, uint64_t n,
                     uint64_t nnz, uint64_t* structure_hash);

/* ---- graph upload --------------------------------------------------------
 * Copies the CSR to `device`, relabels rows by descending degree (results are
 * reported in the caller's ids), and builds the load-balanced work tables.
 * The host arrays are only borrowed for the call.  validate != 0 runs the
 * from_csr checks first (CPG_ESTRUCT on failure). */
int cpg_graph_create(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n,
                     uint64_t nnz, int device, int validate, cpg_graph** out);

/* Same, from arrays already resident on `device` (e.g. produced by the device
 * generator); the arrays stay owned by the caller. */
int cpg_graph_create_device(const uint64_t* d_offsets, const uint32_t* d_neighbors,
                            uint32_t n, uint64_t nnz, int device, cpg_graph** out);

/* Row-partitioned shard for multi-GPU: rank `rank` of
 * `nranks` keeps the rows it owns plus a full-length iterate replica and joins
 * an NCCL communicator identified by `nccl_unique_id` (128 bytes from
 * cpg_nccl_unique_id on one rank, broadcast by the caller).  Every rank passes
 * the whole CSR (host or device pointers per `on_device`). */
int cpg_nccl_unique_id(void* out128);
int cpg_graph_create_sharded(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n,
                             uint64_t nnz, int on_device, int device, int rank, int nranks,
                             const void* nccl_unique_id, cpg_graph** out);

/* TEST HOOK (no reference counterpart): a loopback data plane that runs the
 * nranks shards of the row-partitioned path inside ONE process on ONE device.
 * Rank r's handle comes from cpg_graph_create_loopback(..., rank, group); the
 * exchange steps (per-chunk all-gathers, the mass all-reduce, the result
 * gather) become peer-buffer copies between the handles, with host barriers
 * between the ranks' threads.  Each rank must be driven by its own host thread
 * making the same sequence of calls, as one process per GPU would.  This runs
 * the product's own shard layout and exchange sequence (the same code as the
 * NCCL path up to the data plane) on a single-GPU box. */
int cpg_loopback_group_create(int nranks, cpg_loopback_group** out);
int cpg_loopback_group_destroy(cpg_loopback_group* grp);
int cpg_graph_create_loopback(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n,
                              uint64_t nnz, int on_device, int device, int rank,
                              cpg_loopback_group* grp, cpg_graph** out);

/* One handle over n_devices GPUs of THIS process (SURVEY.md 8b's cpg_graph_create
 * with a device list): the host CSR is row-partitioned across the devices, one
 * shard handle per device (cpg_graph_create_sharded, the NCCL communicator
 * created from one host thread per device).  cpg_chebypower / _vec / _batched /
 * _batched_async / _device, cpg_power_method and cpg_general_gp on it run every
 * shard's call from its own host thread; rank 0 (devices[0]) writes the output
 * and stats.  n_devices == 1 gives a plain single-GPU handle.  topk / measure /
 * trace entries reject it (use them per process on shard handles). */
int cpg_graph_create_multi(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz,
                           const int* devices, int n_devices, cpg_graph** out);
/* Test hook: the same facade over n_ranks shards on ONE device with the
 * loopback data plane (no NCCL; rank r's "all-gather" copies peer slices). */
int cpg_graph_create_multi_loopback(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz,
                                    int device, int n_ranks, cpg_graph** out);
/* Host restatement of the device relabel/partition (graph_build.cu): nodes
 * ordered by (degree desc, id asc); with cr = ceil(n / (nranks*chunks)),
 * position i goes to rank = i % nranks, t = i / nranks, chunk = t % chunks,
 * j = t / chunks: global id = chunk*nranks*cr + rank*cr + j, local row
 * chunk*cr + j.  Fills new_of_old[n]; returns cr in *rows_per_chunk. */
int cpg_shard_plan(const uint64_t* offsets, uint32_t n, int nranks, int chunks, uint32_t* new_of_old,
                   uint32_t* rows_per_chunk);

int cpg_graph_info_get(const cpg_graph* g, cpg_graph_info* info);
int cpg_graph_destroy(cpg_graph* g);

/* ---- the hot path ----------------------------------------------------------
 * ChebyPower (solvers.cpp:197-239): for each source s_j,
 *   out[j*n : (j+1)*n] = sum_{k=0..K} c_k T_k(P) e_{s_j},   P = A D^-1,
 * with coeffs[0..K] supplied by the caller (cpg_cheby_coeffs).  K fused
 * SpMV+recurrence steps per query on the device.  `out` is a HOST buffer
 * (n_sources*n doubles) or NULL to discard; stats may be NULL.
 * Sharded handles: every rank calls collectively; out is filled on every rank. */
int cpg_chebypower(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                   uint32_t n_sources, double* out, cpg_stats* stats);

/* Device-resident variant: d_out is a DEVICE buffer (n_sources*n doubles, or
 * NULL), work is enqueued on `stream` (cudaStream_t, NULL = the handle's own
 * stream) and the call returns without synchronising. */
int cpg_chebypower_device(cpg_graph* g, const double* coeffs, uint32_t K,
                          const uint32_t* sources, uint32_t n_sources, double* d_out,
                          void* stream, cpg_stats* stats);

/* cheby_power_vec (solvers.cpp:197-234): dense seeds (n_seeds x n, host). */
int cpg_chebypower_vec(cpg_graph* g, const double* coeffs, uint32_t K, const double* seeds,
                       uint32_t n_seeds, double* out, cpg_stats* stats);

/* Batched multi-source variant: sources processed in tiles of `tile` (1..64)
 * columns with one SpMM per step (the general_gp_matrix loop of
 * solvers.cpp:405-414 with a = 0 fused into one sweep). */
int cpg_chebypower_batched(cpg_graph* g, const double* coeffs, uint32_t K,
                           const uint32_t* sources, uint32_t n_sources, uint32_t tile,
                           double* out, cpg_stats* stats);
int cpg_chebypower_batched_device(cpg_graph* g, const double* coeffs, uint32_t K,
                                  const uint32_t* sources, uint32_t n_sources, uint32_t tile,
                                  double* d_out, void* stream, cpg_stats* stats);
/* Pipelined host output (no reference counterpart; for throughput callers that
 * issue query after query, like the reference bench's worker loop
 * tools/chebyprop.cpp:305-334): same as cpg_chebypower_batched, but it returns
 * once the steps are computed, with the device->host copy of the last tile into
 * `out` still in flight on the handle's copy stream, so it overlaps the next
 * call's steps.  `out` (pinned host memory for a true overlap) must stay valid
 * and unread until cpg_graph_sync returns.  With stats == NULL the call does not
 * wait for its steps either: it returns once everything is queued, so the host
 * enqueues the next query while the GPU computes this one. */
int cpg_chebypower_batched_async(cpg_graph* g, const double* coeffs, uint32_t K,
                                 const uint32_t* sources, uint32_t n_sources, uint32_t tile,
                                 double* out, cpg_stats* stats);
/* Wait for every result copy the handle has in flight. */
int cpg_graph_sync(cpg_graph* g);

/* ChebyPower ranked on the device: for each source the
 * k best (caller id, score) pairs by (score desc, id asc), the order of the
 * reference's query output (tools/chebyprop.cpp:148-156).  ids/vals are host
 * arrays of n_sources*min(k,n). */
int cpg_chebypower_topk(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                        uint32_t n_sources, uint32_t k, uint32_t* ids, double* vals, cpg_stats* stats);

/* general_gp_vector / general_gp_matrix with ChebyPower (solvers.cpp:390-414):
 * z_j = D^-a f(P) D^a x_j for n_cols dense host columns X (n_cols x n), with the
 * D^{+-a} scalings fused into the seed and output kernels; tile > 1 runs tiles
 * of `tile` columns (<= 64) through the batched step. */
int cpg_general_gp(cpg_graph* g, const double* coeffs, uint32_t K, double a, const double* X,
                   uint32_t n_cols, uint32_t tile, double* out, cpg_stats* stats);

/* Test/observer slow path: T_k(P)e_s for k = 0..K ((K+1) x n, host) and the
 * partial estimates after each step ((K+1) x n), the StepObserver arguments of
 * solvers.cpp:215,219,226.  Either trace pointer may be NULL. */
int cpg_chebypower_trace(cpg_graph* g, const double* coeffs, uint32_t K, uint32_t source,
                         double* out, double* r_trace, double* est_trace);
/* The same observer slow path for a dense seed vector x (length n, caller ids):
 * cheby_power_vec with a non-empty StepObserver (solvers.hpp:62-64,
 * solvers.cpp:197-234).  r_trace[k*n..] = T_k(P) x, est_trace[k*n..] = the
 * partial estimate after step k (est_0 = c_0 x, solvers.cpp:209). */
int cpg_chebypower_vec_trace(cpg_graph* g, const double* coeffs, uint32_t K, const double* seed,
                             double* out, double* r_trace, double* est_trace);

/* PwMethod (solvers.cpp:87-121), the reference's ground-truth engine
 * (eval.cpp:52-59): out = sum_{k<n_steps} zeta_k P^k e_s, n_steps - 1 fused
 * SpMV steps per source (same kernels, Taylor epilogue). */
int cpg_power_method(cpg_graph* g, const double* zeta, uint32_t n_steps, const uint32_t* sources,
                     uint32_t n_sources, double* out, cpg_stats* stats);

/* Single walk y = A D^-1 x (graph.cpp:257-267) for tests; host vectors. */
int cpg_apply_walk(cpg_graph* g, const double* x, double* y);

/* Algorithmic bytes of one single-source step for this handle. */
double cpg_bytes_per_step(const cpg_graph* g, uint32_t tile);

/* After a call made under cpg_set_profiling(1): the mean CUDA-event time of the two
 * kernels of its split batched steps (hub-piece kernel, plain-row kernel) and how many
 * steps were bracketed (0 when the call ran no split step).  bench.py's roofline of
 * the dominant kernel. */
int cpg_last_split_profile(cpg_graph* g, double* pieces_ms, double* rows_ms, uint32_t* steps);

/* Steps at the head of a one-hot query on this handle that gather only the rows
 * of w_{k-1} with a nonzero entry, as the reference's scatter skips zero entries
 * (graph.cpp:262); tile <= 1 = the single-source step.  Results are bit-identical
 * to full steps; the count is the library's measured default or
 * the CPG_SPARSE_STEPS override. */
uint32_t cpg_sparse_early_steps(const cpg_graph* g, uint32_t tile, uint32_t K);

/* ---- synthetic inputs (bench/test harness; deterministic, seed-addressed) ----
 * R-MAT (a,b,c,d) with 2^scale ids and n_samples draws, or Chung-Lu with
 * power-law weights; both symmetrised, deduplicated, self-loops dropped,
 * isolated ids compacted (ascending).  Output CSR lands on `device` (pass
 * device = -1 to build on the host).  Buffers are allocated by the library and
 * released with cpg_free_csr. */
int cpg_gen_rmat(uint32_t scale, uint64_t n_samples, double a, double b, double c,
                 uint64_t seed, int device, uint64_t** offsets, uint32_t** neighbors,
                 uint32_t* n, uint64_t* nnz);
int cpg_gen_chunglu(uint32_t n_ids, uint64_t n_samples, double exponent, double mean_degree,
                    uint32_t max_degree, uint64_t seed, int device, uint64_t** offsets,
                    uint32_t** neighbors, uint32_t* n, uint64_t* nnz);
int cpg_free_csr(uint64_t* offsets, uint32_t* neighbors, int device);
/* GPU ingest with the reference loader's semantics (graph.cpp:113-171): host
 * label pairs (m x 2 int64) -> device CSR; self-loops dropped, labels interned
 * in first-seen order, symmetrised, sorted, deduplicated.  original_ids_host
 * (capacity original_ids_cap) receives the label of every compact id
 * (Graph::original_ids, graph.hpp:45), or NULL. */
int cpg_ingest_edges(const int64_t* pairs, uint64_t m, int device, uint64_t** offsets, uint32_t** neighbors,
                     uint32_t* n, uint64_t* nnz, int64_t* original_ids_host, uint64_t original_ids_cap);
/* Copy a device-resident CSR (e.g. from the generator) into caller host arrays. */
int cpg_csr_to_host(const uint64_t* d_offsets, const uint32_t* d_neighbors, uint32_t n, uint64_t nnz,
                    int device, uint64_t* offsets, uint32_t* neighbors);

/* ---- the formats and metrics either side of the path ---- */

/* ErrorReport (eval.hpp:15-20). */
typedef struct {
    double l1;
    double l2;
    double deg_norm_inf;
    uint32_t argmax_node;
} cpg_error_report;

/* measure(truth, estimate, g) (eval.cpp:18-37) for n_cols column pairs
 * ([n_cols][n] each, caller ids) on the graph's device.  on_device != 0: both
 * pointers are device memory; else host memory (uploaded).  l1/l2 are
 * compensated sums (within the reference's own rounding of its sequential
 * sum), deg_norm_inf and argmax_node are exact (ties keep the smaller id). */
int cpg_measure(cpg_graph* g, const double* truth, const double* estimate, uint32_t n_cols, int on_device,
                cpg_error_report* reports);
/* n_sources ChebyPower queries measured against truths[n_sources][n] on the
 * device (the eval harness's run_query: estimate + measure, eval.cpp:18-37,
 * tools/chebyprop.cpp:140-160) -- no n-vector crosses PCIe.  truths_on_device
 * != 0: truths is device memory (e.g. from cpg_power_method's device output). */
int cpg_chebypower_measure(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                           uint32_t n_sources, const double* truths, int truths_on_device,
                           cpg_error_report* reports, cpg_stats* stats);

/* Edge-list text with the reference loader's line rules (graph.cpp:126-151):
 * blank lines and lines whose first non-blank char is `comment` are skipped;
 * every other line must start with two integers (istream >> int64 rules),
 * optionally followed by ONE token that parses fully as a number (a weight).
 * Errors: CPG_EPARSE with the reference's message ("line N: expected two
 * integers, got \"...\"" / "line N: trailing garbage \"...\"") for the
 * first bad line.  pairs == NULL counts only; else cap_pairs >= the count.
 * Self-loops are kept here (cpg_ingest_edges drops them, graph.cpp:149). */
int cpg_parse_edge_text(const char* text, uint64_t len, char comment, int64_t* pairs, uint64_t cap_pairs,
                        uint64_t* n_pairs, int n_threads);
/* CPGR binary CSR cache (graph.hpp:87-90, graph.cpp:217-255): "CPGR", u32 1,
 * u64 n, u64 m, u64 offsets[n+1], u32 neighbors[2m].  info reads the header
 * (CPG_EPARSE bad magic / version / short header, CPG_ESTRUCT n out of
 * range); read fills caller arrays (CPG_EPARSE "truncated CSR cache").
 * Validation is Graph::from_csr's (cpg_validate_csr). */
int cpg_csr_cache_write(const char* path, const uint64_t* offsets, const uint32_t* neighbors, uint64_t n,
                        uint64_t nnz);
int cpg_csr_cache_info(const char* path, uint64_t* n, uint64_t* m);
int cpg_csr_cache_read(const char* path, uint64_t* offsets, uint32_t* neighbors, uint64_t n, uint64_t m);
/* CPGT ground-truth cache (eval.cpp:92-145): "CPGT", u32 1, u32 len,
 * descriptor, u64 source, u64 n, f64 values[n]; and truth_cache_filename
 * (eval.cpp:147-156). */
int cpg_truth_cache_write(const char* path, const char* kernel_descriptor, uint64_t source, const double* values,
                          uint64_t n);
int cpg_truth_cache_info(const char* path, char* desc, uint64_t desc_cap, uint64_t* source, uint64_t* n);
int cpg_truth_cache_read(const char* path, double* values, uint64_t n);
int cpg_truth_cache_filename(uint64_t structure_hash, const char* kernel_descriptor, uint64_t source, char* out,
                             uint64_t cap);

#ifdef __cplusplus
}
#endif
#endif /* CPG_H */
