// cpg_graph.hpp -- host-side handle behind cpg_graph* (not part of the ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <condition_variable>
#include <map>
#include <mutex>
#include <vector>

#include "cpg_common.hpp"
#include "device_graph.cuh"

namespace cpg {
// Work table for one chunk of local rows [row_begin, row_end).
struct ItemTable {
    WorkItem* items = nullptr;
    uint32_t n_items = 0, n_hubs = 0, n_hub_items = 0;
    uint32_t row_begin = 0, row_end = 0;
    uint2* meta = nullptr;  // column-window hub pieces: (first slot, piece count) per hub row, or null
};
} // namespace cpg

namespace cpg {
// Data plane of a row-sharded handle: the exchange steps of the 1-D row
// partition.  NCCL in production (nccl_dl.cpp); a test-only
// loopback plane (loopback.cu) runs the R shards of one process on one GPU
// with peer-buffer copies, so the sharded layout and choreography run on a
// single-GPU box.
struct Comm {
    int rank = 0, nranks = 1;
    virtual ~Comm() = default;
    // recv[p*count, (p+1)*count) <- rank p's send (in place when send == recv + rank*count)
    virtual void allgather(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
    virtual void allreduce_sum(double* buf, size_t count, cudaStream_t st) = 0;
    // wait for st; a failed communicator surfaces as CPG_ENCCL instead of a hang
    virtual void sync(cudaStream_t st) = 0;
    virtual void* nccl() { return nullptr; }  // ncclComm_t of an NCCL plane
};
Comm* make_nccl_comm(const void* id128, int nranks, int rank);
struct LoopbackGroup;
LoopbackGroup* loopback_group_create(int nranks);
void loopback_group_destroy(LoopbackGroup* grp);
int loopback_group_size(const LoopbackGroup* grp);
Comm* make_loopback_comm(LoopbackGroup* grp, int rank);

// Batched work tables of one (tile width, kernel path): hub pieces per chunk.
struct BatchTables {
    std::vector<ItemTable> tables;
    uint32_t n_bpartials = 0;
};

// Per-call device state: streams, iterates, accumulators, partials, staging.
// A graph handle keeps a pool of these, so concurrent calls on one handle (the
// reference allows concurrent queries on a shared Graph) each
// run on their own streams and buffers.  Grown on demand, owned by the pool.
struct Workspace {
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    cudaStream_t comm_stream = nullptr;  // per-chunk all-gathers (sharded)
    std::vector<cudaEvent_t> chunk_ev;   // chunk computed / chunk gathered
    // ev[0..1]: slot copied out; ev[2..3]: slot computed; ev[4]: caller-stream join
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};

    double* w_a = nullptr;          // iterates (replicated over ranks), [n_pad][cols]
    double* w_b = nullptr;
    double* acc = nullptr;          // [n_loc][cols]
    double* full = nullptr;         // gathered final result (sharded)
    size_t ws_cols = 0;             // columns the iterates are sized for (1, a query group, or B)

    double* hub_partial = nullptr;  // single-source hub pieces, [hub_q][n_partials]
    unsigned int* hub_count = nullptr;  // [hub_q][n_loc]
    uint32_t hub_q = 0;
    double* bhub_partial = nullptr; // batched hub pieces [n_bpartials][B]
    size_t bhub_cap = 0;
    unsigned int* bhub_count = nullptr; // [n_loc]
    unsigned int* d_job_ctr = nullptr;  // fused batched kernel: one job counter per (step, chunk)
    size_t job_ctr_cap = 0;
    unsigned int* d_wctr = nullptr;     // warp-tile single-source step: one item counter per (step, chunk)
    size_t wctr_cap = 0;

    double* d_coeffs = nullptr;
    size_t coeff_cap = 0;
    uint32_t* d_sources = nullptr;
    size_t src_cap = 0;
    double* d_mass_partial = nullptr;   // per (step, chunk, kernel, CTA[, column]) mass partials
    size_t mass_cap = 0;
    double* d_mass_err = nullptr;       // mapped pinned [2]: running max, scratch
    double* d_step_mass = nullptr;      // [queries][K]
    size_t step_mass_cap = 0;
    double* d_mass0 = nullptr;          // per-column conserved mass (dense batched seeds)
    size_t mass0_cap = 0;
    double* d_seeds = nullptr;          // dense seeds of one call slice
    size_t seeds_cap = 0;
    double* d_stage = nullptr;          // device result staging for host output (2 slots)
    uint32_t stage_seq = 0;             // slot of the next batch: slots alternate across calls too,
                                        // so a pipelined call's last copy overlaps the next call
    size_t stage_cap = 0;               // doubles per slot (allocation)
    size_t stage_slot = 0;              // doubles per slot of the last call (slot layout)
    double* d_topk = nullptr;           // device-ranked queries: [Q][n] results
    size_t topk_cap = 0;
    uint32_t* d_nz = nullptr;           // support bitmaps of w_0 .. w_{M-1} (sparse early steps), nz_words(n_pad) each
    size_t nz_cap = 0;                  // words

    // Fused all-gather (CPG_P2P=1 on a sharded graph): w_a / w_b are NCCL
    // symmetric windows and the batched epilogue stores each computed row into
    // every rank's replica through the LSA peer pointers.
    void* win_a = nullptr;
    void* win_b = nullptr;
    double** d_peers_a = nullptr;   // [nranks] peer pointers of w_a's window
    double** d_peers_b = nullptr;
    double* d_barrier = nullptr;    // one-element all-reduce per iteration (the barrier)
};
} // namespace cpg

struct cpg_graph {
    // last profiled call (cpg_set_profiling): mean ms of the piece / row kernels of its split batched steps
    double split_prof_pieces_ms = 0.0, split_prof_rows_ms = 0.0;
    uint32_t split_prof_steps = 0;
    int device = 0;
    int rank = 0, nranks = 1;
    int chunks = 1;                 // row chunks per rank (one all-gather each)
    uint32_t cr = 0;                // rows per (rank, chunk)
    uint32_t n = 0, n_loc = 0, n_pad = 0, row0 = 0, max_degree = 0;
    uint64_t nnz = 0, nnz_loc = 0, hash = 0;

    int64_t* rowptr = nullptr;      // [n_loc+1]
    uint32_t* col = nullptr;        // [nnz_loc]
    uint32_t* gdeg = nullptr;       // [n_pad]
    uint32_t* new_of_old = nullptr; // [n]

    std::vector<cpg::ItemTable> tables;   // single-source items, one table per chunk
    std::vector<cpg::ItemTable> wtables;  // warp-tile items (cheby_step_warp_kernel), one per chunk
    uint32_t n_items = 0, n_hubs = 0, n_hub_items = 0, n_tiles = 0, n_partials = 0;
    int tile = 0;                   // kTileSmall / kTileMid / kTileLarge
    bool step_split = false;        // single-source step as hub + tile kernels (iterate > L2)
    // batched tables per (B, split) key (built on first use, kept: read-only after)
    std::map<int, cpg::BatchTables> btabs;
    std::mutex tab_mu;

    cudaStream_t stream = nullptr;  // build / upload stream
    int sm_count = 0, step_grid = 0;

    // Workspace pool: calls acquire one (blocking when max_ws are in use) and
    // return it when they finish.  Sharded handles use exactly one (their NCCL
    // collectives must be issued in the same order on every rank).
    std::vector<cpg::Workspace*> ws_all, ws_free;
    size_t max_ws = 4;
    std::mutex ws_mu;
    std::condition_variable ws_cv;

    std::vector<cpg_graph*> members;  // multi-device facade (cpg_graph_create_multi): one shard per rank
    cpg::LoopbackGroup* own_group = nullptr;  // facade over loopback shards: the group it owns
    cpg::Comm* comm = nullptr;      // data plane when sharded (NCCL or test loopback), else null
    bool p2p = false;               // fused all-gather through NCCL symmetric windows
    int p2p_self = 0;               // test hook: also store through this rank's own LSA alias
};

namespace cpg {

// graph_build.cu
void build_device_graph(cpg_graph* g, const uint64_t* d_off, const uint32_t* d_nbr, cudaStream_t st);
const BatchTables& ensure_batch_tables(cpg_graph* g, int B);
// Device buffers that the steps touch all over every step (gathered iterates,
// per-row index/offset/accumulator arrays), at 512 MB-aligned addresses when
// large; freed with dfree_aligned (api.cu).
void* dalloc_aligned(size_t bytes);
void dfree_aligned(void* p);
ItemTable build_item_table(const int64_t* rowptr, uint32_t row0, uint32_t row1, int64_t chunk, uint32_t max_rows,
                           int64_t piece, uint32_t slot_off, cudaStream_t st, int64_t hub_thr = 0, int64_t solo = 0);
void launch_step_warp(const StepArgs& a, unsigned int* ctr, int grid, cudaStream_t st);
int step_warp_occupancy();

// step_kernels.cu
void launch_step(const StepArgs& a, int grid, cudaStream_t st, const StepGroup* gq = nullptr, bool pdl = false);
int step_occupancy(int tile);
void launch_step_hubs(const StepArgs& a, int grid, cudaStream_t st, bool pdl = false);
void launch_step_tiles(const StepArgs& a, int tile, int grid, cudaStream_t st, bool pdl = false);
int step_tiles_occupancy(int tile);
int step_hubs_occupancy();
// batched launches return the grid they used (mass partial rows = grid * warps)
int launch_batch(const BatchArgs& a, int B, int grid, cudaStream_t st, const PeerArgs* pa = nullptr,
                 bool pdl = false);
int batch_occupancy();
bool batch_split(uint64_t nnz_loc);
int launch_batch_rows(const BatchArgs& a, int B, int grid, cudaStream_t st, const PeerArgs* pa = nullptr);
// Sparse early batched step (scan + fill kernels); returns the mass rows in CTAs.
int launch_sparse_step(const BatchArgs& a, int B, uint32_t* done, const uint32_t* fill_mask, const uint32_t* coarse,
                       uint32_t coarse_words, int cshift, uint32_t row_begin, int64_t hb, int grid, cudaStream_t st);
int launch_first_push(const BatchArgs& a, const uint32_t* gdeg, const uint32_t* new_of_old, const uint32_t* sources,
                      uint32_t q0, uint32_t count, uint32_t B, int grid, cudaStream_t st);
void launch_coarsen(const uint32_t* fine, uint64_t fine_words, uint32_t* coarse, uint32_t coarse_words, int cshift,
                    cudaStream_t st);
// Coarse-bitmap geometry for n_pad rows: rows per bit = 1 << cshift (>= 64), at most 8192 words (32 KB).
inline int coarse_shift(uint64_t n_pad) {
    int s = 6;
    while ((n_pad >> s) > 8192ull * 32) ++s;
    return s;
}
inline uint32_t coarse_words(uint64_t n_pad, int cshift) {
    return static_cast<uint32_t>((((n_pad + (1ull << cshift) - 1) >> cshift) + 31) / 32);
}
int launch_batch_pieces(const BatchArgs& a, int B, int grid, cudaStream_t st, const PeerArgs* pa = nullptr);

void launch_init_onehot(double* w, uint64_t stride, const uint32_t* gdeg, const uint32_t* no, const uint32_t* src,
                        uint32_t q0, uint32_t count, cudaStream_t st, uint32_t* nz0 = nullptr);
void launch_init_onehot_batch(double* W, const uint32_t* gdeg, const uint32_t* no, const uint32_t* src,
                              uint32_t q0, uint32_t count, uint32_t B, cudaStream_t st, uint32_t* nz0 = nullptr);
void launch_init_dense(double* w, const uint32_t* gdeg, const uint32_t* no, const double* seed,
                       uint32_t n, double a, cudaStream_t st);
void launch_init_dense_batch(double* W, const uint32_t* gdeg, const uint32_t* no, const double* X, uint32_t n,
                             uint32_t count, uint32_t B, double a, cudaStream_t st);
void launch_unpermute(double* out, const double* full, uint64_t stride, const uint32_t* no, uint32_t n,
                      uint32_t count, const uint32_t* gdeg, double a, cudaStream_t st);
void launch_unpermute_batch(double* out, const double* full, const uint32_t* no, uint32_t n,
                            uint32_t count, uint32_t B, const uint32_t* gdeg, double a, cudaStream_t st);
void launch_mass_steps(const double* mp, uint32_t n_part, uint64_t q_stride, uint32_t K, uint32_t count,
                       double* steps, cudaStream_t st);
void launch_zero_f64(double* p, cudaStream_t st);
void launch_mass_err(const double* steps, uint32_t K, double mass0, double* err, cudaStream_t st);
void launch_mass_steps_batch(const double* mp, uint32_t stride, uint32_t used, uint32_t B, uint32_t K,
                             uint32_t count, double* steps, cudaStream_t st);
void launch_mass_err_cols(const double* steps, uint32_t K, uint32_t count, const double* mass0, double* err,
                          cudaStream_t st);

// topk.cu
void device_topk_batch(const double* d_vals, uint32_t n, uint32_t Q, uint32_t k, uint32_t* ids, double* vals,
                       cudaStream_t st);
// measure (eval.cpp:18-37) of [cols][n] device column pairs into d_reports[cols] (measure.cu)
size_t measure_scratch_bytes(const cpg_graph* g, uint32_t cols);
void launch_measure(const cpg_graph* g, const double* d_truth, const double* d_est, uint32_t cols, void* scratch,
                    cpg_error_report* d_reports, cudaStream_t st);

// nccl_dl.cpp
void nccl_get_unique_id(void* out128);
void* nccl_comm_init(const void* id128, int nranks, int rank);
void nccl_allgather_f64(const double* send, double* recv, size_t count, void* comm, cudaStream_t st);
void nccl_allreduce_sum_f64(const double* send, double* recv, size_t count, void* comm, cudaStream_t st);
void nccl_comm_destroy(void* comm);
void nccl_check_async(void* comm);
// nccl_sym.cu (NCCL symmetric windows; see there)
bool nccl_sym_supported(void* comm, int nranks, int rank);
void* nccl_sym_alloc(size_t bytes);
void nccl_sym_free(void* p);
void* nccl_sym_register(void* comm, void* buf, size_t bytes);
void nccl_sym_deregister(void* comm, void* win);
void nccl_sym_peer_ptrs(void* win, int n, double** d_out, cudaStream_t st);

} // namespace cpg
