// api.cu -- C-ABI entry points (include/cpg.h): graph handles and the query
// drivers that sequence the fused step kernels.
//
// Per single-source query (cheby_power, solvers.cpp:197-239):
//   memset(w_a) ; w_a[s] = 1/d_s                       (w_0 = D^-1 e_s)
//   for k = 1..K: step(w_cur = w_{k-1}, w_io = w_{k-2} -> w_k)   [+ all-gather if sharded]
//   per-step mass sums -> |sum T_k - 1| check           (acceptance C13)
//   unpermute d*acc into the caller's ids
// Host outputs are copied on a second stream, one query behind the compute
// stream, so D2H of query q overlaps the K steps of query q+1.
//
// Concurrency: the graph handle is immutable after create (like the
// reference's Graph); every call leases a Workspace
// (streams + buffers) from the handle's pool, so calls from several host
// threads on one handle run concurrently.  Sharded handles keep one workspace:
// their collectives must be issued in the same order on every rank.
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // header-only; ranges cost a pointer check unless a tool is attached

#include <algorithm>
#include <atomic>
#include <chrono>
#include <functional>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "cpg_graph.hpp"

using namespace cpg;

namespace {

template <typename T>
T* dalloc(size_t count) {
    T* p = nullptr;
    CPG_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
    return p;
}

template <typename T>
void dfree(T*& p) {
    if (p) cudaFree(p);
    p = nullptr;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        CPG_CUDA(cudaSetDevice(dev));
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

std::atomic<int> g_profile{0};

// Event pairs around step-kernel launches (profiling mode only).
struct StepProf {
    std::vector<cudaEvent_t> ev;
    std::vector<cudaEvent_t> mid;  // split batched step: between the piece kernel and the row kernel
    void before(cudaStream_t st) { rec(st); }
    void after(cudaStream_t st) { rec(st); }
    void rec(cudaStream_t st) {
        cudaEvent_t e;
        CPG_CUDA(cudaEventCreate(&e));
        CPG_CUDA(cudaEventRecord(e, st));
        ev.push_back(e);
    }
    void between(cudaStream_t st) {  // pairs with the last before()
        cudaEvent_t e;
        CPG_CUDA(cudaEventCreate(&e));
        CPG_CUDA(cudaEventRecord(e, st));
        mid.resize(ev.size() / 2 + 1, nullptr);
        mid[ev.size() / 2] = e;
    }
    // mean milliseconds of the two kernels of the split steps that recorded a mid event
    uint32_t split_ms(double* first, double* second) {
        double a = 0.0, b = 0.0;
        uint32_t n = 0;
        for (size_t i = 0; i < mid.size() && 2 * i + 1 < ev.size(); ++i) {
            if (!mid[i]) continue;
            float m0 = 0.f, m1 = 0.f;
            cudaEventSynchronize(ev[2 * i + 1]);
            cudaEventElapsedTime(&m0, ev[2 * i], mid[i]);
            cudaEventElapsedTime(&m1, mid[i], ev[2 * i + 1]);
            a += m0;
            b += m1;
            ++n;
        }
        if (n) {
            *first = a / n;
            *second = b / n;
        }
        return n;
    }
    double total_ms() {
        double t = 0.0;
        for (size_t i = 0; i + 1 < ev.size(); i += 2) {
            float ms = 0.f;
            cudaEventSynchronize(ev[i + 1]);
            cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
            t += ms;
        }
        return t;
    }
    ~StepProf() {
        // CPG_PROF_DUMP=1 (diagnostics): each bracketed step's milliseconds on stderr
        if (const char* d = std::getenv("CPG_PROF_DUMP"); d && d[0] == '1' && ev.size() >= 2) {
            std::fprintf(stderr, "[cpg prof] step ms:");
            for (size_t i = 0; i + 1 < ev.size(); i += 2) {
                float ms = 0.f;
                cudaEventSynchronize(ev[i + 1]);
                cudaEventElapsedTime(&ms, ev[i], ev[i + 1]);
                std::fprintf(stderr, " %.3f", ms);
            }
            std::fprintf(stderr, "\n");
        }
        for (auto e : ev) cudaEventDestroy(e);
        for (auto e : mid)
            if (e) cudaEventDestroy(e);
    }
};

// NVTX range for the duration of a scope (calls, queries, steps show up by name in
// Nsight Systems / ncu --nvtx; near-free without a tool).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// Row chunks per rank: one all-gather per chunk, overlapped with the next
// chunk's step kernel.  1 on a single GPU; CPG_CHUNKS overrides (tests).
int default_chunks(int nranks) {
    int c = nranks > 1 ? 4 : 1;
    if (const char* e = std::getenv("CPG_CHUNKS")) c = std::max(1, std::min(64, std::atoi(e)));
    return c;
}

int table_grid(const cpg_graph* g, uint32_t n_items, int occ) {
    return static_cast<int>(
        std::max<uint64_t>(1, std::min<uint64_t>(n_items, static_cast<uint64_t>(occ) * g->sm_count)));
}

// Mass-partial rows (one per warp) of one batched launch, at most.
size_t batch_warp_cap(const cpg_graph* g) {
    return static_cast<size_t>(kBatchMaxCtasPerSm) * g->sm_count * (kBatchThreads / 32);
}

// ---- workspace pool ---------------------------------------------------------------------
Workspace* ws_create(cpg_graph* g) {
    auto w = std::make_unique<Workspace>();
    CPG_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
    CPG_CUDA(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
    CPG_CUDA(cudaStreamCreateWithFlags(&w->comm_stream, cudaStreamNonBlocking));
    for (auto& e : w->ev) CPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    w->chunk_ev.resize(2 * static_cast<size_t>(g->chunks));
    for (auto& e : w->chunk_ev) CPG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // the per-query mass check lives in mapped pinned host memory: the host reads it
    // without a device->host copy, which would queue behind a pipelined result copy
    CPG_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w->d_mass_err), 2 * sizeof(double), cudaHostAllocMapped));
    w->d_mass_err[0] = w->d_mass_err[1] = 0.0;
    return w.release();
}

void free_iterates(cpg_graph* g, Workspace* w) {
    if (g->p2p && w->win_a) {
        nccl_sym_deregister(g->comm->nccl(), w->win_a);
        nccl_sym_deregister(g->comm->nccl(), w->win_b);
        nccl_sym_free(w->w_a);
        nccl_sym_free(w->w_b);
        w->win_a = w->win_b = nullptr;
    } else {
        dfree_aligned(w->w_a);
        dfree_aligned(w->w_b);
    }
    w->w_a = w->w_b = nullptr;
}

void ws_destroy(cpg_graph* g, Workspace* w) {
    if (!w) return;
    if (w->stream) cudaStreamSynchronize(w->stream);
    if (w->copy_stream) cudaStreamSynchronize(w->copy_stream);
    free_iterates(g, w);
    dfree_aligned(w->acc);
    w->acc = nullptr;
    for (void* p : {(void*)w->full, (void*)w->hub_partial, (void*)w->hub_count, (void*)w->bhub_partial,
                    (void*)w->bhub_count, (void*)w->d_job_ctr, (void*)w->d_wctr, (void*)w->d_coeffs, (void*)w->d_sources,
                    (void*)w->d_mass_partial, (void*)w->d_step_mass, (void*)w->d_mass0, (void*)w->d_seeds,
                    (void*)w->d_stage, (void*)w->d_topk, (void*)w->d_peers_a, (void*)w->d_peers_b,
                    (void*)w->d_barrier, (void*)w->d_nz})
        if (p) cudaFree(p);
    if (w->d_mass_err) cudaFreeHost(w->d_mass_err);
    for (auto e : w->ev)
        if (e) cudaEventDestroy(e);
    for (auto e : w->chunk_ev)
        if (e) cudaEventDestroy(e);
    for (cudaStream_t s : {w->stream, w->copy_stream, w->comm_stream})
        if (s) cudaStreamDestroy(s);
    delete w;
}

// A leased workspace, returned to the pool (and its waiters woken) on scope exit.
struct WsLease {
    cpg_graph* g;
    Workspace* w;
    explicit WsLease(cpg_graph* gg) : g(gg), w(nullptr) {
        std::unique_lock<std::mutex> lock(g->ws_mu);
        g->ws_cv.wait(lock, [&] { return !g->ws_free.empty() || g->ws_all.size() < g->max_ws; });
        if (!g->ws_free.empty()) {
            w = g->ws_free.back();
            g->ws_free.pop_back();
            return;
        }
        g->ws_all.push_back(nullptr);  // reserve the slot while creating outside the lock
        lock.unlock();
        Workspace* nw = nullptr;
        try {
            DeviceGuard dg(g->device);
            nw = ws_create(g);
        } catch (...) {
            std::lock_guard<std::mutex> l2(g->ws_mu);
            g->ws_all.erase(std::find(g->ws_all.begin(), g->ws_all.end(), nullptr));
            g->ws_cv.notify_one();
            throw;
        }
        std::lock_guard<std::mutex> l2(g->ws_mu);
        *std::find(g->ws_all.begin(), g->ws_all.end(), nullptr) = nw;
        w = nw;
    }
    ~WsLease() {
        std::lock_guard<std::mutex> lock(g->ws_mu);
        g->ws_free.push_back(w);
        g->ws_cv.notify_one();
    }
    WsLease(const WsLease&) = delete;
    WsLease& operator=(const WsLease&) = delete;
};

size_t default_max_ws(const cpg_graph* g) {
    if (g->comm) return 1;
    size_t m = 4;  // device memory bounds the pool, not host threads: config 5 batched needs ~39 GB each
    if (const char* e = std::getenv("CPG_MAX_WORKSPACES")) m = static_cast<size_t>(std::max(1, std::atoi(e)));
    return m;
}

// L2 set-aside for persisting lines (CPG_L2_PERSIST_MB, A/B hook; unset = leave the
// device setting alone).  The hot prefix of the batched iterate is gathered with an
// L2::evict_last policy; the set-aside is the portion of L2 such lines may claim.
void l2_set_aside(int device) {
    const char* e = std::getenv("CPG_L2_PERSIST_MB");
    if (!e) return;
    cudaDeviceProp prop{};
    CPG_CUDA(cudaGetDeviceProperties(&prop, device));
    const size_t want = std::min<size_t>(static_cast<size_t>(std::atoll(e)) << 20,
                                         static_cast<size_t>(prop.persistingL2CacheMaxSize));
    CPG_CUDA(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want));
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
    std::fprintf(stderr, "[cpg] L2 persisting set-aside %zu MB (max %d MB)\n", got >> 20,
                 prop.persistingL2CacheMaxSize >> 20);
}

cpg_graph* create_common(const uint64_t* d_off, const uint32_t* d_nbr, uint32_t n, uint64_t nnz, int device,
                         int rank, int nranks, Comm* comm, int chunks = 0) {
    auto g = std::make_unique<cpg_graph>();
    g->device = device;
    g->rank = rank;
    g->nranks = nranks;
    g->chunks = chunks > 0 ? chunks : default_chunks(nranks);
    g->n = n;
    g->nnz = nnz;
    CPG_CUDA(cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking));
    CPG_CUDA(cudaDeviceGetAttribute(&g->sm_count, cudaDevAttrMultiProcessorCount, device));
    build_device_graph(g.get(), d_off, d_nbr, g->stream);
    const int occ = std::max(1, step_occupancy(g->tile));
    g->step_grid = 1;  // max over chunks: the mass-partial stride
    for (const auto& t : g->tables) g->step_grid = std::max(g->step_grid, table_grid(g.get(), t.n_items, occ));
    // the warp-tile step's hub + warp grids share one mass-partial row too
    g->step_grid = std::max(g->step_grid, (std::max(1, step_hubs_occupancy()) +
                                           std::max(1, step_warp_occupancy())) * g->sm_count);
    // the split step's two grids share one mass-partial row
    g->step_grid = std::max(g->step_grid, (std::max(1, step_hubs_occupancy()) +
                                           std::max(1, step_tiles_occupancy(g->tile))) * g->sm_count);
    g->comm = comm;
    g->max_ws = default_max_ws(g.get());
    l2_set_aside(device);
    CPG_CUDA(cudaStreamSynchronize(g->stream));
    return g.release();
}

// Column width of the batched step for a tile of `tile` sources.
uint32_t batch_width(uint32_t tile) {
    uint32_t B = 4;
    while (B < tile) B <<= 1;
    return B;
}

// The replicated iterates (NCCL symmetric windows on p2p graphs; collective:
// every rank calls this in the same order with the same size).
void alloc_iterates(cpg_graph* g, Workspace* w, size_t cols) {
    const size_t bytes = sizeof(double) * g->n_pad * cols;
    if (!g->p2p) {
        w->w_a = static_cast<double*>(dalloc_aligned(bytes));
        w->w_b = static_cast<double*>(dalloc_aligned(bytes));
        return;
    }
    void* nc = g->comm->nccl();
    w->w_a = static_cast<double*>(nccl_sym_alloc(bytes));
    w->w_b = static_cast<double*>(nccl_sym_alloc(bytes));
    w->win_a = nccl_sym_register(nc, w->w_a, bytes);
    w->win_b = nccl_sym_register(nc, w->w_b, bytes);
    if (!w->d_peers_a) {
        w->d_peers_a = dalloc<double*>(static_cast<size_t>(g->nranks));
        w->d_peers_b = dalloc<double*>(static_cast<size_t>(g->nranks));
        w->d_barrier = dalloc<double>(1);
        CPG_CUDA(cudaMemset(w->d_barrier, 0, sizeof(double)));
    }
    nccl_sym_peer_ptrs(w->win_a, g->nranks, w->d_peers_a, w->stream);
    nccl_sym_peer_ptrs(w->win_b, g->nranks, w->d_peers_b, w->stream);
    CPG_CUDA(cudaStreamSynchronize(w->stream));
}

void ensure_ws(cpg_graph* g, Workspace* w, size_t cols) {
    if (w->ws_cols == cols) return;
    CPG_CUDA(cudaStreamSynchronize(w->stream));
    free_iterates(g, w);
    dfree_aligned(w->acc);
    w->acc = nullptr;
    dfree(w->full);
    alloc_iterates(g, w, cols);
    w->acc = static_cast<double*>(dalloc_aligned(sizeof(double) * g->n_loc * cols));
    if (g->comm) w->full = dalloc<double>(static_cast<size_t>(g->n_pad) * cols);
    CPG_CUDA(cudaMemset(w->w_a, 0, sizeof(double) * g->n_pad * cols));
    CPG_CUDA(cudaMemset(w->w_b, 0, sizeof(double) * g->n_pad * cols));
    w->ws_cols = cols;
}

// Mass-partial columns per (step, chunk) of a query group of Q queries: the
// launch grid of the group (single queries keep the per-graph step_grid).
uint32_t mass_cols(const cpg_graph* g, uint32_t Q) {
    if (Q <= 1) return static_cast<uint32_t>(g->step_grid);
    return static_cast<uint32_t>(std::max(1, step_occupancy(g->tile)) * g->sm_count);
}

void ensure_mass(Workspace* w, size_t partials, size_t steps) {
    if (w->mass_cap < partials) {
        dfree(w->d_mass_partial);
        w->d_mass_partial = dalloc<double>(partials);
        w->mass_cap = partials;
    }
    if (w->step_mass_cap < steps) {
        dfree(w->d_step_mass);
        w->d_step_mass = dalloc<double>(steps);
        w->step_mass_cap = steps;
    }
}

// Per-query device state for a group of Q single-source queries: hub partial
// slots and tickets, and the mass arrays.
void ensure_group(cpg_graph* g, Workspace* w, uint32_t K, uint32_t Q) {
    if (w->hub_q < Q) {
        dfree(w->hub_partial);
        dfree(w->hub_count);
        w->hub_partial = dalloc<double>(static_cast<size_t>(g->n_partials) * Q);
        w->hub_count = dalloc<unsigned int>(static_cast<size_t>(g->n_loc) * Q);
        CPG_CUDA(cudaMemset(w->hub_count, 0, sizeof(unsigned int) * std::max<size_t>(1, static_cast<size_t>(g->n_loc) * Q)));
        w->hub_q = Q;
    }
    ensure_mass(w, static_cast<size_t>(K) * g->chunks * mass_cols(g, Q) * Q, static_cast<size_t>(K) * Q);
}

// Sparse early steps: the first M steps of a one-hot query gather
// only rows of w_{k-1} whose support bit is set (the reference's scatter skips
// zero entries the same way, graph.cpp:262).  Step k reads bitmap k-1 and, for
// k < M, builds bitmap k in its epilogue; the init kernel sets bitmap 0 (the
// sources).  Results are bit-identical to the unmasked steps.  A sharded rank
// builds only its own rows' bits, so there only step 1 (the sources' bitmap,
// known to every rank) is masked; the fused all-gather path is never masked.
// Defaults from the A/B on one B200 (profiles/r02/sparse/): a batched tile masks
// its first 2 steps on graphs of >= 1.5 M directed edges (configs 2-5: +3..11%;
// config 1's 31-us steps lose more to the extra launches than the skipped
// gathers give back, and a third masked step always loses: the 2-hop ball already
// carries most of the volume); one source masks 2 steps only where the iterate
// exceeds the L2 (split step, config 5: +1%; an L2-resident iterate loses 3-5%).
// CPG_SPARSE_STEPS=M overrides (0 = off).
uint32_t sparse_steps(const cpg_graph* g, bool single, uint32_t K) {
    if (g->p2p) return 0;
    uint32_t M = single ? (g->step_split ? 2 : 0)
                        : (g->nnz_loc >= 1500000ull ? 2 : 0);
    if (const char* e = std::getenv("CPG_SPARSE_STEPS")) M = static_cast<uint32_t>(std::max(0, std::atoi(e)));
    if (g->comm) M = std::min<uint32_t>(M, 1);
    return std::min(M, K);
}

// M zeroed bitmaps (stream-ordered), or null for M = 0.
uint32_t* ensure_nz(cpg_graph* g, Workspace* w, uint32_t M, cudaStream_t st) {
    if (!M) return nullptr;
    const size_t need = static_cast<size_t>(M) * nz_words(g->n_pad);
    if (w->nz_cap < need) {
        dfree(w->d_nz);
        w->d_nz = dalloc<uint32_t>(need);
        w->nz_cap = need;
    }
    CPG_CUDA(cudaMemsetAsync(w->d_nz, 0, sizeof(uint32_t) * need, st));
    return w->d_nz;
}

void ensure_params(Workspace* w, uint32_t K, uint32_t n_sources) {
    if (w->coeff_cap < K + 1) {
        dfree(w->d_coeffs);
        w->d_coeffs = dalloc<double>(K + 1);
        w->coeff_cap = K + 1;
    }
    if (w->src_cap < n_sources) {
        dfree(w->d_sources);
        w->d_sources = dalloc<uint32_t>(n_sources);
        w->src_cap = n_sources;
    }
}

// Staging slots for host output.  A pipelined call's last copy may still be
// reading a slot: the slots alternate across calls, and when the slot layout
// changes (another tile or group size) the copies in flight are drained first,
// since the new slot boundaries no longer line up with the old ones.
void ensure_stage(Workspace* w, size_t doubles) {
    if (w->stage_slot != doubles && w->stage_slot != 0) CPG_CUDA(cudaStreamSynchronize(w->copy_stream));
    w->stage_slot = doubles;
    if (w->stage_cap >= doubles) return;
    CPG_CUDA(cudaStreamSynchronize(w->copy_stream));
    dfree(w->d_stage);
    w->d_stage = dalloc<double>(2 * doubles);
    w->stage_cap = doubles;
}

void check_query(const cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources, uint32_t ns) {
    require(g != nullptr, "null graph handle");
    require(K >= 1, "cheby_power: cheby_steps must be >= 1");  // solvers.cpp:201
    require(coeffs != nullptr, "null coefficient array");
    require(ns == 0 || sources != nullptr, "null source array");
    for (uint32_t i = 0; i < ns; ++i)
        require(sources[i] < g->n, "source node " + std::to_string(sources[i]) + " out of range");  // :28-29
}

// Global id of local row 0 of chunk c (cpg_graph layout, graph_build.cu):
// gid(l) = l + chunk_row0(c) for l in chunk c.
uint32_t chunk_row0(const cpg_graph* g, uint32_t c) {
    return c * (static_cast<uint32_t>(g->nranks) - 1) * g->cr + static_cast<uint32_t>(g->rank) * g->cr;
}

// In-place all-gather of chunk c of a replicated [n_pad][cols] iterate on the
// comm stream, after the chunk's step kernel (event chunk_ev[c]); the next use
// of the iterate waits for chunk_ev[C + C-1] (the comm stream is in order).
void gather_chunk(cpg_graph* g, Workspace* w, double* v, uint32_t c, size_t cols, cudaStream_t st) {
    if (!g->comm) return;
    const size_t C = static_cast<size_t>(g->chunks);
    const size_t R = static_cast<size_t>(g->nranks);
    double* base = v + static_cast<size_t>(c) * R * g->cr * cols;
    CPG_CUDA(cudaEventRecord(w->chunk_ev[c], st));
    CPG_CUDA(cudaStreamWaitEvent(w->comm_stream, w->chunk_ev[c], 0));
    g->comm->allgather(base + static_cast<size_t>(g->rank) * g->cr * cols, base, g->cr * cols, w->comm_stream);
    if (c + 1 == C) CPG_CUDA(cudaEventRecord(w->chunk_ev[C + c], w->comm_stream));
}

void wait_gathers(cpg_graph* g, Workspace* w, cudaStream_t st) {
    if (!g->comm) return;
    const size_t C = static_cast<size_t>(g->chunks);
    CPG_CUDA(cudaStreamWaitEvent(st, w->chunk_ev[C + C - 1], 0));
}

// Final d*acc (local rows) -> full [n_pad][cols] replicated, chunk by chunk.
const double* gather_result(cpg_graph* g, Workspace* w, size_t cols, cudaStream_t st) {
    if (!g->comm) return w->acc;
    const size_t R = static_cast<size_t>(g->nranks);
    for (uint32_t c = 0; c < static_cast<uint32_t>(g->chunks); ++c)
        g->comm->allgather(w->acc + static_cast<size_t>(c) * g->cr * cols,
                           w->full + static_cast<size_t>(c) * R * g->cr * cols, g->cr * cols, st);
    return w->full;
}

// Single-source L2 residency split (CPG_HOT1_MB, default 0 = off): ids below
// the budget are gathered evict_last, the rest evict_first.
uint32_t single_hot_rows(const cpg_graph* g) {
    const char* e = std::getenv("CPG_HOT1_MB");
    if (!e) return 0;
    return static_cast<uint32_t>(std::min<uint64_t>(g->n_pad, (static_cast<uint64_t>(std::atoll(e)) << 20) / 8));
}

// Single-source step as CTA hub pieces + barrier-free warp tiles
// (cheby_step_warp_kernel); CPG_WARP_TILES=1/0 (read per call).
bool warp_tiles(const cpg_graph*) {
    const char* e = std::getenv("CPG_WARP_TILES");
    return e && e[0] == '1';
}

// Single-source step as hub-piece + row-tile kernels: by default when the
// iterate exceeds L2 (build_device_graph); CPG_STEP_SPLIT=1/0 forces (read per call).
bool step_split(const cpg_graph* g) {
    const char* e = std::getenv("CPG_STEP_SPLIT");
    return e ? e[0] == '1' : g->step_split;
}

// The K fused steps of one query (group), chunk by chunk (last = write d*acc).
uint32_t run_steps(cpg_graph* g, Workspace* w, uint32_t k_first, uint32_t k_last, uint32_t K, bool last_writes_out,
                   cudaStream_t st, StepProf* prof, bool taylor = false, uint32_t Q = 1, uint32_t M = 0,
                   uint32_t* nz = nullptr) {
    uint32_t launches = 0;
    const int occ = std::max(1, step_occupancy(g->tile));
    const uint32_t C = static_cast<uint32_t>(g->chunks);
    const uint32_t MG = mass_cols(g, Q);
    // programmatic dependent launch between consecutive step kernels: only when
    // nothing else sits between them in the stream (one chunk, no data plane, no
    // profiling events)
    const bool pdl = !g->comm && C == 1 && !prof;
    const bool wt = Q == 1 && warp_tiles(g);
    if (wt) {  // one item counter per (step, chunk) of this call
        const size_t need = static_cast<size_t>(k_last - k_first + 1) * C;
        if (w->wctr_cap < need) {
            dfree(w->d_wctr);
            w->d_wctr = dalloc<unsigned int>(need);
            w->wctr_cap = need;
        }
        CPG_CUDA(cudaMemsetAsync(w->d_wctr, 0, sizeof(unsigned int) * need, st));
    }
    for (uint32_t k = k_first; k <= k_last; ++k) {
        NvtxRange step_range("cpg.step");
        StepArgs a;
        a.rowptr = g->rowptr;
        a.col = g->col;
        a.w_cur = (k & 1) ? w->w_a : w->w_b;
        a.w_io = (k & 1) ? w->w_b : w->w_a;
        a.acc = w->acc;
        a.out = w->acc;
        a.hub_partial = w->hub_partial;
        a.hub_count = w->hub_count;
        a.coeffs = w->d_coeffs;
        a.tile = g->tile;
        a.hot_rows = single_hot_rows(g);
        a.k = static_cast<int>(k);
        a.first = k == 1;
        a.taylor = taylor;
        a.last = last_writes_out && k == K;
        const size_t nzw = nz_words(g->n_pad);
        a.nz_in = nz && k <= M ? nz + (k - 1) * nzw : nullptr;  // masked (sparse early) step
        a.nz_out = nz && k < M ? nz + k * nzw : nullptr;
#if CPG_CHECKED
        a.chk_nnz = g->nnz_loc;
        a.chk_npad = g->n_pad;
        a.chk_nloc = g->n_loc;
        a.chk_parts = g->n_partials;
        a.chk_mass = MG;
#endif
        StepGroup gq;
        gq.nq = Q;
        gq.vec_stride = g->n_pad;
        gq.acc_stride = g->n_loc;
        gq.part_stride = g->n_partials;
        gq.cnt_stride = g->n_loc;
        gq.mass_stride = K * C * MG;
        if (k > 1) wait_gathers(g, w, st);
        for (uint32_t c = 0; c < C; ++c) {
            const ItemTable& t = g->tables[c];
            a.items = t.items;
            a.n_items = t.n_items;
            a.row0 = chunk_row0(g, c);
            a.mass_partial = w->d_mass_partial + (static_cast<size_t>(k - 1) * C + c) * MG;
            const ItemTable& tw = g->wtables[c];
            if (wt && tw.n_items) {  // CTA hub pieces, then barrier-free warp tiles
                if (prof) prof->before(st);
                StepArgs h = a;
                h.items = tw.items;
                h.n_items = tw.n_hub_items;
                const int gh = tw.n_hub_items ? table_grid(g, tw.n_hub_items, std::max(1, step_hubs_occupancy())) : 0;
                if (gh) {
                    launch_step_hubs(h, gh, st);
                    ++launches;
                }
                StepArgs r = a;
                r.items = tw.items + tw.n_hub_items;
                r.n_items = tw.n_items - tw.n_hub_items;
                r.mass_partial = a.mass_partial + gh;
#if CPG_CHECKED
                r.chk_mass = MG - static_cast<uint32_t>(gh);
#endif
                if (r.n_items) {
                    launch_step_warp(r, w->d_wctr + static_cast<size_t>(k - k_first) * C + c,
                                     std::max(1, step_warp_occupancy()) * g->sm_count, st);
                    ++launches;
                }
                if (prof) prof->after(st);
            } else if (t.n_items && Q == 1 && step_split(g)) {  // hub pieces, then row tiles at higher occupancy
                if (prof) prof->before(st);
                StepArgs h = a;
                h.n_items = t.n_hub_items;
                const int gh = t.n_hub_items ? table_grid(g, t.n_hub_items, std::max(1, step_hubs_occupancy())) : 0;
                if (gh) {
                    launch_step_hubs(h, gh, st, pdl);
                    ++launches;
                }
                StepArgs r = a;
                r.items = t.items + t.n_hub_items;
                r.n_items = t.n_items - t.n_hub_items;
                r.mass_partial = a.mass_partial + gh;
#if CPG_CHECKED
                r.chk_mass = MG - static_cast<uint32_t>(gh);
#endif
                if (r.n_items) {
                    launch_step_tiles(r, g->tile, table_grid(g, r.n_items, std::max(1, step_tiles_occupancy(g->tile))),
                                      st, pdl);
                    ++launches;
                }
                if (prof) prof->after(st);
            } else if (t.n_items) {
                const int grid = table_grid(g, t.n_items * Q, occ);
                if (prof) prof->before(st);
                launch_step(a, grid, st, &gq, pdl);
                if (prof) prof->after(st);
                ++launches;
            }
            gather_chunk(g, w, a.w_io, c, 1, st);
        }
    }
    wait_gathers(g, w, st);
    return launches;
}

// A group of Q single-source queries (sources q0 .. q0+Q-1) in one launch per
// step, or one dense-seed query (seed_dev != null, Q = 1); results d*acc
// unpermuted into d_dst[Q][n] (caller ids) if non-null.
uint32_t run_single(cpg_graph* g, Workspace* w, uint32_t K, uint32_t q0, uint32_t Q, const double* seed_dev,
                    double mass0, double* d_dst, cudaStream_t st, StepProf* prof, bool taylor = false,
                    double gp_a = 0.0) {
    uint32_t launches = 0;
    const uint32_t C = static_cast<uint32_t>(g->chunks);
    ensure_group(g, w, K, Q);
    const size_t mstride = static_cast<size_t>(K) * C * mass_cols(g, Q);
    CPG_CUDA(cudaMemsetAsync(w->w_a, 0, sizeof(double) * g->n_pad * Q, st));
    CPG_CUDA(cudaMemsetAsync(w->d_mass_partial, 0, sizeof(double) * mstride * Q, st));
    const uint32_t M = !seed_dev && Q == 1 && !warp_tiles(g) ? sparse_steps(g, true, K) : 0;
    uint32_t* nz = ensure_nz(g, w, M, st);
    if (seed_dev)
        launch_init_dense(w->w_a, g->gdeg, g->new_of_old, seed_dev, g->n, gp_a, st);
    else
        launch_init_onehot(w->w_a, g->n_pad, g->gdeg, g->new_of_old, w->d_sources, q0, Q, st, nz);
    ++launches;
    launches += run_steps(g, w, 1, K, K, true, st, prof, taylor, Q, M, nz);
    launch_mass_steps(w->d_mass_partial, C * mass_cols(g, Q), mstride, K, Q, w->d_step_mass, st);
    ++launches;
    if (g->comm) g->comm->allreduce_sum(w->d_step_mass, static_cast<size_t>(K) * Q, st);
    launch_mass_err(w->d_step_mass, K * Q, mass0, w->d_mass_err, st);
    ++launches;
    if (d_dst) {
        launch_unpermute(d_dst, gather_result(g, w, 1, st), g->n_loc, g->new_of_old, g->n, Q, g->gdeg, gp_a, st);
        ++launches;
    } else if (g->comm) {
        gather_result(g, w, 1, st);  // a collective: every rank takes part, with or without an output
    }
    CPG_CUDA(cudaGetLastError());
    return launches;
}

// One tile of up to B sources (q0 .. q0+count) through the batched step.
// mass0_dev: per-column conserved mass of dense seeds (null: unit seeds, 1 each;
// mass_check false: no conservation to check, general_gp with a != 0).
uint32_t run_batch(cpg_graph* g, Workspace* w, uint32_t K, uint32_t B, uint32_t q0, uint32_t count, double* d_dst,
                   cudaStream_t st, StepProf* prof, const double* seeds_dev = nullptr, double gp_a = 0.0,
                   const double* mass0_dev = nullptr, bool mass_check = true) {
    uint32_t launches = 0;
    const size_t cols = B;
    const uint32_t C = static_cast<uint32_t>(g->chunks);
    const int occ = batch_occupancy();
    const BatchTables& bt = ensure_batch_tables(g, static_cast<int>(B));
    // L2 budget for the degree-sorted hot prefix of the gathered iterate: its rows are
    // loaded evict_last, the rest evict_first.  64 MB of the 126 MB L2 measured best
    // (profiles/r01/hot_prefix_sweep.txt); CPG_HOT_MB overrides, 0 = plain loads.
    uint64_t hot_mb = 64;
    if (const char* e = std::getenv("CPG_HOT_MB")) hot_mb = static_cast<uint64_t>(std::atoll(e));
    const uint32_t hot_rows = static_cast<uint32_t>(std::min<uint64_t>(g->n_pad, (hot_mb << 20) / (8 * cols)));
    // the column-window piece kernel's own hot prefix (graph_build.cu cw_params: the same variable)
    uint64_t cw_hot_mb = 32;
    if (const char* e = std::getenv("CPG_CW_HOT_MB")) cw_hot_mb = static_cast<uint64_t>(std::atoll(e));
    const uint32_t cw_hot_rows = static_cast<uint32_t>(std::min<uint64_t>(g->n_pad, (cw_hot_mb << 20) / (8 * cols)));
    // the plain-row kernel's own hot prefix (CPG_ROWS_HOT_MB; default: the same)
    uint32_t rows_hot_rows = hot_rows;
    if (const char* e = std::getenv("CPG_ROWS_HOT_MB"))
        rows_hot_rows = static_cast<uint32_t>(std::min<uint64_t>(g->n_pad, (static_cast<uint64_t>(std::atoll(e)) << 20) / (8 * cols)));
    CPG_CUDA(cudaMemsetAsync(w->w_a, 0, sizeof(double) * g->n_pad * cols, st));
    // mass partials: one [B] row per warp of every launch, packed per step (the
    // launches, and so the rows, are the same every step: `used` rows per step)
    const size_t step_rows = static_cast<size_t>(C) * 2 * batch_warp_cap(g);
    ensure_mass(w, static_cast<size_t>(K) * step_rows * B, static_cast<size_t>(K) * count);
    size_t used = 0;
    constexpr size_t W = kBatchThreads / 32;
    // Fused kernel (small graphs): warps claim jobs from a counter instead of a static
    // stride, so a warp that drew short rows takes more (CPG_DYN_JOBS=0: static).
    static const bool dyn_jobs = [] {
        const char* e = std::getenv("CPG_DYN_JOBS");
        return !e || e[0] != '0';
    }();
    const bool split = batch_split(g->nnz_loc);
    // column-window piece tables: the piece kernel claims its pieces in list order
    bool cw_tables = false;
    for (const ItemTable& t : bt.tables) cw_tables = cw_tables || t.meta != nullptr;
    const bool use_ctr = (dyn_jobs && !split) || cw_tables;
    // PDL between the fused step kernels (see run_steps): one chunk, no data plane, no profiling
    const bool pdl = !g->comm && C == 1 && !prof;
    if (use_ctr) {
        const size_t need = static_cast<size_t>(K) * C;
        if (w->job_ctr_cap < need) {
            dfree(w->d_job_ctr);
            w->d_job_ctr = dalloc<unsigned int>(need);
            w->job_ctr_cap = need;
        }
        CPG_CUDA(cudaMemsetAsync(w->d_job_ctr, 0, sizeof(unsigned int) * need, st));
    }
    const uint32_t M = seeds_dev ? 0 : sparse_steps(g, false, K);
    // bitmaps [0, M): supports of w_0 .. w_{M-1}; [M, 2M): rows done by each sparse step's scan;
    // then the coarse bitmap of the current sparse step's input (coarse_words words)
    const int cshift = coarse_shift(g->n_pad);
    const uint32_t cwords = coarse_words(g->n_pad, cshift);
    const size_t nzw = nz_words(g->n_pad);
    uint32_t* nz = ensure_nz(g, w, 2 * M + (M ? (cwords + nzw - 1) / nzw : 0), st);
    uint32_t* coarse = nz ? nz + 2 * M * nzw : nullptr;
    const int64_t hb = split ? batch_piece_edges(static_cast<int>(B)) : batch_hub_edges(static_cast<int>(B));
    const bool sparse_kern = cw_tables || [] {  // CPG_SPARSE_KERNEL=0: masked full-step kernels instead (A/B; read per call)
        const char* e = std::getenv("CPG_SPARSE_KERNEL");
        return !e || e[0] != '0';
    }();
    // a sparse step writes fewer mass rows than a full one: the rows it leaves are zero
    if (M) CPG_CUDA(cudaMemsetAsync(w->d_mass_partial, 0, sizeof(double) * K * step_rows * B, st));
    if (seeds_dev)
        launch_init_dense_batch(w->w_a, g->gdeg, g->new_of_old, seeds_dev, g->n, count, B, gp_a, st);
    else
        launch_init_onehot_batch(w->w_a, g->gdeg, g->new_of_old, w->d_sources, q0, count, B, st, nz);
    ++launches;
    for (uint32_t k = 1; k <= K; ++k) {
        NvtxRange step_range("cpg.batch_step");
        BatchArgs b;
        b.rowptr = g->rowptr;
        b.col = g->col;
        b.w_cur = (k & 1) ? w->w_a : w->w_b;
        b.w_io = (k & 1) ? w->w_b : w->w_a;
        b.acc = w->acc;
        b.out = w->acc;
        b.hub_partial = w->bhub_partial;
        b.hub_count = w->bhub_count;
        b.coeffs = w->d_coeffs;
        b.hot_rows = hot_rows;
        b.k = static_cast<int>(k);
        b.first = k == 1;
        b.last = k == K;
        b.job_ctr = nullptr;
        b.nz_in = nz && k <= M ? nz + (k - 1) * nzw : nullptr;  // masked (sparse early) step
        b.nz_out = nz && k < M ? nz + k * nzw : nullptr;
        b.hub_meta = nullptr;
        b.meta_row0 = 0;
        b.n_pad_rows = g->n_pad;
#if CPG_CHECKED
        b.chk_nnz = g->nnz_loc;
        b.chk_npad = g->n_pad;
        b.chk_nloc = g->n_loc;
        b.chk_parts = bt.n_bpartials;
#endif
        PeerArgs peer_args{nullptr, 0, 0};
        const PeerArgs* pa = nullptr;
        if (g->p2p) {  // fused all-gather: the epilogue stores into every replica
            peer_args.peer_io = (k & 1) ? w->d_peers_b : w->d_peers_a;
            peer_args.n_peer = g->nranks;
            peer_args.self = g->p2p_self ? -1 : g->rank;
            pa = &peer_args;
        }
        if (k > 1 && !g->p2p) wait_gathers(g, w, st);
        size_t rows = 0;  // mass-partial rows of this step so far
        double* const mp_step = w->d_mass_partial + static_cast<size_t>(k - 1) * step_rows * B;
        for (uint32_t c = 0; c < C; ++c) {
            const ItemTable& t = bt.tables[c];
            b.hub_items = t.items;
            b.n_hub_items = t.n_hub_items;
            b.hub_rows = t.row_begin + t.n_hubs;  // first non-hub row of the chunk
            b.n_loc = t.row_end;                  // end row of the chunk
            b.row0 = chunk_row0(g, c);
            b.hub_meta = t.meta;
            b.meta_row0 = t.row_begin;
            if (sparse_kern && b.nz_in) {  // sparse early step: edge scan + fill
                b.mass_partial = mp_step + rows * B;
#if CPG_CHECKED
                b.chk_mass = step_rows - rows;
#endif
                if (prof) prof->before(st);
                // rows that can change with y = 0: those with w_{k-2} != 0 (first step: w_0 != 0, the
                // rest pre-zeroed below); every row on the last step (it writes d * acc)
                const uint32_t* fill_mask = b.last ? nullptr : (k == 1 ? b.nz_in : nz + (k - 2) * nzw);
                if (c == 0 && k == 1 && !b.last) {  // w_1 and acc start at zero off the sources' rows
                    CPG_CUDA(cudaMemsetAsync(b.w_io, 0, sizeof(double) * g->n_pad * cols, st));
                    CPG_CUDA(cudaMemsetAsync(w->acc, 0, sizeof(double) * g->n_loc * cols, st));
                }
                if (k == 1 && !b.last && !g->comm && C == 1) {  // one-term sums: push from the sources (exact)
                    rows += W * launch_first_push(b, g->gdeg, g->new_of_old, w->d_sources, q0, count,
                                                  static_cast<uint32_t>(B), 2 * g->sm_count, st);
                } else {
                    if (c == 0) launch_coarsen(b.nz_in, nzw, coarse, cwords, cshift, st);
                    rows += W * launch_sparse_step(b, static_cast<int>(B), nz + (M + k - 1) * nzw, fill_mask, coarse,
                                                   cwords, cshift, t.row_begin, hb, occ * g->sm_count, st);
                }
                if (prof) prof->after(st);
                launches += 2;
            } else if (split) {
                // hub pieces (fused kernel with no plain rows), then the plain rows
                if (prof) prof->before(st);
                if (t.n_hub_items) {
                    BatchArgs h = b;
                    h.n_loc = b.hub_rows;
                    if (t.meta) {
                        h.job_ctr = w->d_job_ctr + static_cast<size_t>(k - 1) * C + c;
                        h.hot_rows = cw_hot_rows;
                    }
                    h.mass_partial = mp_step + rows * B;
#if CPG_CHECKED
                    h.chk_mass = step_rows - rows;
#endif
                    const uint32_t warps = (t.n_hub_items + 64 / B - 1) / (64 / B);
                    // (launch_capped trims the grid to the instance's own occupancy)
                    const int hocc = t.meta ? kBatchMaxCtasPerSm : occ;
                    const int hgrid = static_cast<int>(std::max<uint32_t>(
                        1, std::min<uint32_t>((warps + 7) / 8, static_cast<uint32_t>(hocc * g->sm_count))));
                    const int pg = launch_batch_pieces(h, static_cast<int>(B), hgrid, st, pa);
                    if (pg < 0) fail(CPG_ECUDA, "column-window pieces: unsupported launch");
                    rows += W * pg;
                    ++launches;
                }
                if (prof && t.n_hub_items && t.row_end > b.hub_rows) prof->between(st);
                if (t.row_end > b.hub_rows) {
                    BatchArgs r = b;
                    r.hot_rows = rows_hot_rows;
                    r.mass_partial = mp_step + rows * B;
#if CPG_CHECKED
                    r.chk_mass = step_rows - rows;
#endif
                    rows += W * launch_batch_rows(r, static_cast<int>(B), occ * g->sm_count, st, pa);
                    ++launches;
                }
                if (prof) prof->after(st);
            } else {
                const uint32_t jobs = t.n_hub_items + (t.row_end - b.hub_rows);
                if (jobs) {
                    const int grid = occ * g->sm_count;
                    if (use_ctr) b.job_ctr = w->d_job_ctr + static_cast<size_t>(k - 1) * C + c;
                    b.mass_partial = mp_step + rows * B;
#if CPG_CHECKED
                    b.chk_mass = step_rows - rows;
#endif
                    if (prof) prof->before(st);
                    rows += W * launch_batch(b, static_cast<int>(B), grid, st, pa, pdl && !pa);
                    if (prof) prof->after(st);
                    ++launches;
                }
            }
            if (!g->p2p) gather_chunk(g, w, b.w_io, c, cols, st);
        }
        if (rows > step_rows) fail(CPG_ECUDA, "batched mass partials overflow");
        if (k > 1 && rows != used && !M) fail(CPG_ECUDA, "batched launches differ between steps");
        used = std::max(used, rows);
        // iteration barrier: every rank's rows of w_k are in every replica before step k+1
        if (g->p2p) g->comm->allreduce_sum(w->d_barrier, 1, st);
    }
    if (!g->p2p) wait_gathers(g, w, st);
    if (mass_check && count) {
        launch_mass_steps_batch(w->d_mass_partial, static_cast<uint32_t>(step_rows), static_cast<uint32_t>(used), B, K,
                                count, w->d_step_mass, st);
        ++launches;
        if (g->comm) g->comm->allreduce_sum(w->d_step_mass, static_cast<size_t>(K) * count, st);
        launch_mass_err_cols(w->d_step_mass, K, count, mass0_dev, w->d_mass_err, st);
        ++launches;
    }
    if (d_dst) {
        launch_unpermute_batch(d_dst, gather_result(g, w, cols, st), g->new_of_old, g->n, count, B, g->gdeg, gp_a,
                               st);
        ++launches;
    } else if (g->comm) {
        gather_result(g, w, cols, st);  // a collective: every rank takes part, with or without an output
    }
    CPG_CUDA(cudaGetLastError());
    return launches;
}

void upload_params(Workspace* w, const double* coeffs, uint32_t K, const uint32_t* sources, uint32_t ns,
                   cudaStream_t st) {
    ensure_params(w, K, std::max<uint32_t>(ns, 1));
    CPG_CUDA(cudaMemcpyAsync(w->d_coeffs, coeffs, sizeof(double) * (K + 1), cudaMemcpyHostToDevice, st));
    if (ns) CPG_CUDA(cudaMemcpyAsync(w->d_sources, sources, sizeof(uint32_t) * ns, cudaMemcpyHostToDevice, st));
    launch_zero_f64(w->d_mass_err, st);
}

void fill_stats(cpg_graph* g, Workspace* w, cpg_stats* stats, uint32_t K, uint64_t queries, double wall,
                float dev_ms, uint32_t launches, uint32_t cols, bool mass_checked) {
    if (!stats) return;
    const double merr = *static_cast<volatile double*>(w->d_mass_err);  // mapped; the stream was synchronized
    stats->iterations = K;
    stats->push_work = static_cast<uint64_t>(K) * g->nnz * queries;
    stats->wall_seconds = wall;
    stats->device_ms = dev_ms;
    stats->mass_err_max = mass_checked ? merr : std::nan("");
    const double tiles = cols == 1 ? static_cast<double>(queries) : std::ceil(static_cast<double>(queries) / cols);
    stats->bytes_model = tiles * K * cpg_bytes_per_step(g, cols);
    stats->launches = launches;
    stats->step_ms = 0.0;
    stats->step_launches = 0;
}

// Single-source queries per launch: enough to give every resident CTA several
// work items when the graph alone cannot (small graphs are latency-bound at
// one query per launch), capped at 16 and by a 2 GB workspace.  One rank only
// (the all-gathers move one iterate).  CPG_GROUP_Q overrides (tests), capped at
// 32: the one-hot seed kernel seeds up to 32 queries of a group.
uint32_t single_group(const cpg_graph* g, uint32_t nq) {
    if (nq <= 1 || g->comm) return 1;
    uint32_t Q;
    if (const char* e = std::getenv("CPG_GROUP_Q")) {
        Q = static_cast<uint32_t>(std::max(1, std::min(32, std::atoi(e))));
    } else {
        // measured: config 1 (0.95 M edges) best at 16, config 2 (2.1 M) at 8, config 3 (86 M) at 1
        Q = static_cast<uint32_t>(std::min<uint64_t>(16, std::max<uint64_t>(1, (16ull << 20) / std::max<uint64_t>(1, g->nnz_loc))));
        const uint64_t bytes_per_q = 8ull * (2ull * g->n_pad + g->n_loc);
        Q = static_cast<uint32_t>(std::min<uint64_t>(Q, std::max<uint64_t>(1, (2ull << 30) / bytes_per_q)));
    }
    Q = std::max(1u, std::min(Q, nq));
    const uint32_t groups = (nq + Q - 1) / Q;  // balance the group sizes (no ragged tail group)
    return (nq + groups - 1) / groups;
}

template <typename T>
void ensure_buf(T*& p, size_t& cap, size_t need) {
    if (cap >= need) return;
    dfree(p);
    p = dalloc<T>(need);
    cap = need;
}

// Shared driver for host / device outputs.  mode 0 = one-hot single source,
// 1 = dense seeds (seeds_host), 2 = batched tiles of `tile` sources,
// 3 = power method (Taylor), 4 = batched dense seed columns (general_gp_matrix).
int drive(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources, const double* seeds_host,
          uint32_t nq, uint32_t tile, int mode, double* out, bool out_on_device, void* user_stream,
          cpg_stats* stats, double gp_a = 0.0, bool pipelined = false) {
    static const char* const kModeName[] = {"cpg.chebypower", "cpg.chebypower_vec", "cpg.chebypower_batched",
                                             "cpg.power_method", "cpg.general_gp"};
    NvtxRange range(kModeName[mode >= 0 && mode <= 4 ? mode : 0]);
    if (g && !g->members.empty()) {
        // multi-device handle: every shard runs the same call from its own host thread (the
        // per-step collectives meet across them); rank 0 writes the caller's output and stats
        const size_t R = g->members.size();
        std::vector<int> rc(R, CPG_OK);
        std::vector<std::string> msg(R);
        std::vector<std::thread> th;
        for (size_t r = 0; r < R; ++r)
            th.emplace_back([&, r] {
                rc[r] = drive(g->members[r], coeffs, K, sources, seeds_host, nq, tile, mode, r == 0 ? out : nullptr,
                              out_on_device, r == 0 ? user_stream : nullptr, r == 0 ? stats : nullptr, gp_a,
                              pipelined);
                if (rc[r] != CPG_OK) msg[r] = cpg_last_error();
            });
        for (auto& t : th) t.join();
        for (size_t r = 0; r < R; ++r)
            if (rc[r] != CPG_OK) return guarded([&] { fail(rc[r], "shard " + std::to_string(r) + ": " + msg[r]); });
        return CPG_OK;
    }
    return guarded([&] {
        require(g != nullptr, "null graph handle");
        require(std::isfinite(gp_a), "general_gp: exponent must be finite");
        const bool dense = mode == 1 || mode == 4;
        if (dense) {
            require(K >= 1, "cheby_power: cheby_steps must be >= 1");
            require(coeffs && (nq == 0 || seeds_host), "null argument");
        } else {
            check_query(g, coeffs, K, sources, nq);
        }
        const bool batched = mode == 2 || mode == 4;
        if (batched) require(tile >= 1 && tile <= kBatchCols, "batched tile must be in [1, 64]");
        DeviceGuard dg(g->device);
        WsLease lease(g);
        Workspace* w = lease.w;
        const double t0 = now_s();
        cudaStream_t st = w->stream;
        cudaEvent_t e0, e1;
        CPG_CUDA(cudaEventCreate(&e0));
        CPG_CUDA(cudaEventCreate(&e1));
        if (user_stream) {
            CPG_CUDA(cudaEventRecord(w->ev[4], static_cast<cudaStream_t>(user_stream)));
            CPG_CUDA(cudaStreamWaitEvent(st, w->ev[4], 0));
        }
        const uint32_t B = batched ? batch_width(tile) : 1;
        const size_t cols = B;
        if (batched) {
            const BatchTables& bt = ensure_batch_tables(g, static_cast<int>(B));
            ensure_buf(w->bhub_partial, w->bhub_cap, std::max<size_t>(1, static_cast<size_t>(bt.n_bpartials) * B));
            if (!w->bhub_count) {
                w->bhub_count = dalloc<unsigned int>(g->n_loc);
                CPG_CUDA(cudaMemset(w->bhub_count, 0, sizeof(unsigned int) * std::max<uint32_t>(1, g->n_loc)));
            }
        }
        const uint32_t per = batched ? tile : (mode == 0 || mode == 3) ? single_group(g, nq) : 1;
        ensure_ws(g, w, batched ? cols : per);
        upload_params(w, coeffs, K, sources, dense ? 0 : nq, st);
        const size_t n = g->n;
        const uint32_t nbatches = (nq + per - 1) / per;
        const size_t slot = n * per;  // doubles per result slot
        if (dense) ensure_buf(w->d_seeds, w->seeds_cap, n * per);
        // conserved mass of dense seed columns: sum of the seed (a = 0); a != 0 has none
        const bool mass_checked = !(dense && gp_a != 0.0);
        std::vector<double> mass0;
        if (mode == 4 && mass_checked) {
            mass0.resize(nq);
            for (uint32_t q = 0; q < nq; ++q) {
                double m = 0.0;
                for (size_t v = 0; v < n; ++v) m += seeds_host[q * n + v];
                mass0[q] = m;
            }
            ensure_buf(w->d_mass0, w->mass0_cap, std::max<size_t>(1, nq));
            CPG_CUDA(cudaMemcpyAsync(w->d_mass0, mass0.data(), sizeof(double) * nq, cudaMemcpyHostToDevice, st));
        }
        if (!out_on_device && out) ensure_stage(w, slot);
        uint32_t launches = 0;
        std::unique_ptr<StepProf> prof(g_profile.load() ? new StepProf : nullptr);
        CPG_CUDA(cudaEventRecord(e0, st));
        for (uint32_t b = 0; b < nbatches; ++b) {
            const uint32_t q0 = b * per;
            const uint32_t count = std::min<uint32_t>(per, nq - q0);
            double* dst = nullptr;
            if (out && out_on_device) {
                dst = out + static_cast<size_t>(q0) * n;
            } else if (out) {
                const uint32_t sl = (w->stage_seq + b) & 1;
                dst = w->d_stage + sl * slot;
                CPG_CUDA(cudaStreamWaitEvent(st, w->ev[sl], 0));  // slot free (its previous copy done)
            }
            if (mode == 0 || mode == 3) {
                launches += run_single(g, w, K, q0, count, nullptr, 1.0, dst, st, prof.get(), mode == 3);
            } else if (mode == 1) {
                const double* sh = seeds_host + static_cast<size_t>(q0) * n;
                double m0 = 0.0;  // sum of the D^a-scaled seed: the conserved mass
                for (size_t v = 0; v < n; ++v) m0 += sh[v];
                CPG_CUDA(cudaMemcpyAsync(w->d_seeds, sh, sizeof(double) * n, cudaMemcpyHostToDevice, st));
                launches += run_single(g, w, K, q0, 1, w->d_seeds, gp_a == 0.0 ? m0 : std::nan(""), dst, st,
                                       prof.get(), false, gp_a);
            } else if (mode == 4) {
                CPG_CUDA(cudaMemcpyAsync(w->d_seeds, seeds_host + static_cast<size_t>(q0) * n,
                                         sizeof(double) * n * count, cudaMemcpyHostToDevice, st));
                launches += run_batch(g, w, K, B, q0, count, dst, st, prof.get(), w->d_seeds, gp_a,
                                      mass_checked ? w->d_mass0 + q0 : nullptr, mass_checked);
            } else {
                launches += run_batch(g, w, K, B, q0, count, dst, st, prof.get());
            }
            if (out && !out_on_device) {
                // compute of batch b is queued; now drain batch b-1 (overlaps b's steps)
                const uint32_t sl = (w->stage_seq + b) & 1, ps = sl ^ 1u;
                CPG_CUDA(cudaEventRecord(w->ev[2 + sl], st));
                if (b >= 1) {
                    CPG_CUDA(cudaStreamWaitEvent(w->copy_stream, w->ev[2 + ps], 0));
                    const uint32_t pq0 = (b - 1) * per, pc = std::min<uint32_t>(per, nq - pq0);
                    CPG_CUDA(cudaMemcpyAsync(out + static_cast<size_t>(pq0) * n, w->d_stage + ps * slot,
                                             sizeof(double) * n * pc, cudaMemcpyDeviceToHost, w->copy_stream));
                    CPG_CUDA(cudaEventRecord(w->ev[ps], w->copy_stream));
                }
            }
        }
        CPG_CUDA(cudaEventRecord(e1, st));
        if (out && !out_on_device && nbatches > 0) {
            const uint32_t b = nbatches - 1;
            const uint32_t sl = (w->stage_seq + b) & 1;
            const uint32_t pq0 = b * per, pc = std::min<uint32_t>(per, nq - pq0);
            CPG_CUDA(cudaStreamWaitEvent(w->copy_stream, w->ev[2 + sl], 0));
            CPG_CUDA(cudaMemcpyAsync(out + static_cast<size_t>(pq0) * n, w->d_stage + sl * slot,
                                     sizeof(double) * n * pc, cudaMemcpyDeviceToHost, w->copy_stream));
            CPG_CUDA(cudaEventRecord(w->ev[sl], w->copy_stream));
            w->stage_seq += nbatches;
            if (!pipelined) CPG_CUDA(cudaStreamSynchronize(w->copy_stream));
        }
        if (user_stream) {
            CPG_CUDA(cudaEventRecord(w->ev[4], st));
            CPG_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(user_stream), w->ev[4], 0));
        }
        float ms = 0.f;
        // A pipelined call without stats returns with its steps still queued: the host
        // enqueues the next query while the GPU works (cpg_graph_sync waits for all).
        const bool defer = pipelined && !stats;
        if (!defer && (!user_stream || stats)) {
            if (g->comm)
                g->comm->sync(st);  // polls the communicator's async error
            else
                CPG_CUDA(cudaStreamSynchronize(st));
            CPG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        }
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        fill_stats(g, w, stats, K, nq, now_s() - t0, ms, launches, batched ? tile : 1u, mass_checked);
        if (stats && prof) {
            stats->step_ms = prof->total_ms();
            stats->step_launches = static_cast<uint32_t>(prof->ev.size() / 2);
        }
        if (prof) {
            std::lock_guard<std::mutex> lock(g->ws_mu);
            g->split_prof_steps = prof->split_ms(&g->split_prof_pieces_ms, &g->split_prof_rows_ms);
        }
    });
}

} // namespace

extern "C" {

void cpg_set_profiling(int on) { g_profile.store(on ? 1 : 0); }

int cpg_graph_create(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz, int device,
                     int validate, cpg_graph** out) {
    return guarded([&] {
        require(offsets && neighbors && out, "null argument");
        require(n > 0, "empty graph");
        uint64_t h = 0;
        if (validate) h = validate_csr(offsets, neighbors, n, nnz);
        DeviceGuard dg(device);
        uint64_t* d_off = dalloc<uint64_t>(static_cast<size_t>(n) + 1);
        uint32_t* d_nbr = dalloc<uint32_t>(nnz);
        cpg_graph* g = nullptr;
        try {
            CPG_CUDA(cudaMemcpy(d_off, offsets, sizeof(uint64_t) * (static_cast<size_t>(n) + 1), cudaMemcpyHostToDevice));
            CPG_CUDA(cudaMemcpy(d_nbr, neighbors, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice));
            g = create_common(d_off, d_nbr, n, nnz, device, 0, 1, nullptr);
        } catch (...) {
            cudaFree(d_off);
            cudaFree(d_nbr);
            throw;
        }
        cudaFree(d_off);
        cudaFree(d_nbr);
        g->hash = h;
        *out = g;
    });
}

int cpg_graph_create_device(const uint64_t* d_offsets, const uint32_t* d_neighbors, uint32_t n, uint64_t nnz,
                            int device, cpg_graph** out) {
    return guarded([&] {
        require(d_offsets && d_neighbors && out, "null argument");
        require(n > 0, "empty graph");
        DeviceGuard dg(device);
        *out = create_common(d_offsets, d_neighbors, n, nnz, device, 0, 1, nullptr);
    });
}

int cpg_nccl_unique_id(void* out128) {
    return guarded([&] {
        require(out128 != nullptr, "null argument");
        nccl_get_unique_id(out128);
    });
}

} // extern "C"

namespace {
// Shared tail of the sharded constructors: CSR to the device if needed, the
// shard of `rank`, and the data plane (made by make_comm; owned by the graph).
template <typename MakeComm>
int create_sharded(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz, int on_device,
                   int device, int rank, int nranks, bool allow_p2p, MakeComm make_comm, cpg_graph** out) {
    return guarded([&] {
        require(offsets && neighbors && out, "null argument");
        require(n > 0, "empty graph");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "bad rank/nranks");
        DeviceGuard dg(device);
        const uint64_t* d_off = offsets;
        const uint32_t* d_nbr = neighbors;
        uint64_t* t_off = nullptr;
        uint32_t* t_nbr = nullptr;
        cpg_graph* g = nullptr;
        Comm* comm = nullptr;
        try {
            if (!on_device) {
                t_off = dalloc<uint64_t>(static_cast<size_t>(n) + 1);
                t_nbr = dalloc<uint32_t>(nnz);
                CPG_CUDA(cudaMemcpy(t_off, offsets, sizeof(uint64_t) * (static_cast<size_t>(n) + 1),
                                    cudaMemcpyHostToDevice));
                CPG_CUDA(cudaMemcpy(t_nbr, neighbors, sizeof(uint32_t) * nnz, cudaMemcpyHostToDevice));
                d_off = t_off;
                d_nbr = t_nbr;
            }
            comm = make_comm();
            // CPG_P2P=1: fused all-gather through NCCL symmetric windows when the
            // NCCL in the process has the device API and all ranks share one
            // NVLink domain (one chunk: no separate collective to overlap)
            const char* pe = std::getenv("CPG_P2P");
            const bool p2p = allow_p2p && comm && comm->nccl() && pe && pe[0] == '1' &&
                             nccl_sym_supported(comm->nccl(), nranks, rank);
            g = create_common(d_off, d_nbr, n, nnz, device, rank, nranks, comm,
                              p2p && !std::getenv("CPG_CHUNKS") ? 1 : 0);
            comm = nullptr;  // owned by g
            g->p2p = p2p;
            if (const char* ps = std::getenv("CPG_P2P_SELF")) g->p2p_self = ps[0] == '1';
        } catch (...) {
            delete comm;
            if (t_off) cudaFree(t_off);
            if (t_nbr) cudaFree(t_nbr);
            if (g) cpg_graph_destroy(g);
            throw;
        }
        if (t_off) cudaFree(t_off);
        if (t_nbr) cudaFree(t_nbr);
        *out = g;
    });
}
} // namespace

extern "C" {

int cpg_graph_create_sharded(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz,
                             int on_device, int device, int rank, int nranks, const void* nccl_unique_id,
                             cpg_graph** out) {
    if (nranks > 1 && !nccl_unique_id) {
        return guarded([&] { fail(CPG_EINVAL, "sharded graph needs an NCCL unique id"); });
    }
    // NCCL whenever an id is given (also for one rank: exercises the collective path)
    return create_sharded(offsets, neighbors, n, nnz, on_device, device, rank, nranks, true,
                          [&]() -> Comm* { return nccl_unique_id ? make_nccl_comm(nccl_unique_id, nranks, rank) : nullptr; },
                          out);
}

int cpg_loopback_group_create(int nranks, cpg_loopback_group** out) {
    return guarded([&] {
        require(out && nranks >= 1 && nranks <= 64, "loopback: 1..64 ranks and an output pointer");
        *out = reinterpret_cast<cpg_loopback_group*>(loopback_group_create(nranks));
    });
}

int cpg_loopback_group_destroy(cpg_loopback_group* grp) {
    return guarded([&] { loopback_group_destroy(reinterpret_cast<LoopbackGroup*>(grp)); });
}

int cpg_graph_create_loopback(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz,
                              int on_device, int device, int rank, cpg_loopback_group* grp, cpg_graph** out) {
    auto* lg = reinterpret_cast<LoopbackGroup*>(grp);
    if (!lg) return guarded([&] { fail(CPG_EINVAL, "loopback: null group"); });
    const int nranks = loopback_group_size(lg);
    return create_sharded(offsets, neighbors, n, nnz, on_device, device, rank, nranks, false,
                          [&]() -> Comm* { return make_loopback_comm(lg, rank); }, out);
}

}  // extern "C"

namespace {
// A multi-device facade over one shard handle per rank, created from R host threads
// (the shards' communicator inits meet across them).
int create_multi(int R, const std::function<int(int, cpg_graph**)>& make_shard, LoopbackGroup* own, cpg_graph** out) {
    return guarded([&] {
        std::vector<cpg_graph*> shards(static_cast<size_t>(R), nullptr);
        std::vector<int> rc(static_cast<size_t>(R), CPG_OK);
        std::vector<std::string> msg(static_cast<size_t>(R));
        std::vector<std::thread> th;
        for (int r = 0; r < R; ++r)
            th.emplace_back([&, r] {
                rc[r] = make_shard(r, &shards[r]);
                if (rc[r] != CPG_OK) msg[r] = cpg_last_error();
            });
        for (auto& t : th) t.join();
        for (int r = 0; r < R; ++r)
            if (rc[r] != CPG_OK) {
                for (cpg_graph* s : shards) cpg_graph_destroy(s);
                if (own) loopback_group_destroy(own);
                fail(rc[r], "shard " + std::to_string(r) + ": " + msg[r]);
            }
        auto g = std::make_unique<cpg_graph>();
        const cpg_graph* s0 = shards[0];
        g->device = s0->device;
        g->rank = 0;
        g->nranks = R;
        g->chunks = s0->chunks;
        g->n = s0->n;
        g->nnz = s0->nnz;
        g->n_loc = s0->n;
        g->nnz_loc = s0->nnz;
        g->n_pad = s0->n_pad;
        g->hash = s0->hash;
        g->max_degree = s0->max_degree;
        g->members = shards;
        g->own_group = own;
        *out = g.release();
    });
}
}  // namespace

extern "C" {

int cpg_graph_create_multi(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz,
                           const int* devices, int n_devices, cpg_graph** out) {
    if (!devices || n_devices < 1 || n_devices > 64)
        return guarded([&] { fail(CPG_EINVAL, "multi-device graph: 1..64 devices"); });
    if (n_devices == 1) return cpg_graph_create(offsets, neighbors, n, nnz, devices[0], 0, out);
    unsigned char id[128];
    const int rc = cpg_nccl_unique_id(id);
    if (rc != CPG_OK) return rc;
    return create_multi(n_devices, [&](int r, cpg_graph** s) {
        return cpg_graph_create_sharded(offsets, neighbors, n, nnz, 0, devices[r], r, n_devices, id, s);
    }, nullptr, out);
}

int cpg_graph_create_multi_loopback(const uint64_t* offsets, const uint32_t* neighbors, uint32_t n, uint64_t nnz,
                                    int device, int n_ranks, cpg_graph** out) {
    if (n_ranks < 1 || n_ranks > 64) return guarded([&] { fail(CPG_EINVAL, "loopback: 1..64 ranks"); });
    LoopbackGroup* grp = loopback_group_create(n_ranks);
    return create_multi(n_ranks, [&](int r, cpg_graph** s) {
        return cpg_graph_create_loopback(offsets, neighbors, n, nnz, 0, device, r,
                                         reinterpret_cast<cpg_loopback_group*>(grp), s);
    }, grp, out);
}

int cpg_graph_info_get(const cpg_graph* g, cpg_graph_info* info) {
    return guarded([&] {
        require(g && info, "null argument");
        info->n = g->n;
        info->nnz = g->nnz;
        info->n_local = g->n_loc;
        info->nnz_local = g->nnz_loc;
        info->row_begin = g->row0;
        info->n_padded = g->n_pad;
        info->n_hubs = g->n_hubs;
        info->n_items = g->n_items;
        info->max_degree = g->max_degree;
        info->rank = g->rank;
        info->nranks = g->nranks;
        info->device = g->device;
        info->structure_hash = g->hash;
        info->chunks = g->chunks;
        info->fused_allgather = g->p2p ? 1 : 0;
    });
}

int cpg_graph_destroy(cpg_graph* g) {
    if (!g) return CPG_OK;
    if (!g->members.empty()) {  // multi-device facade: its shards, then its loopback group
        int rc = CPG_OK;
        for (cpg_graph* s : g->members) rc = std::max(rc, cpg_graph_destroy(s));
        if (g->own_group) loopback_group_destroy(g->own_group);
        delete g;
        return rc;
    }
    return guarded([&] {
        DeviceGuard dg(g->device);
        cudaDeviceSynchronize();
        {
            std::lock_guard<std::mutex> lock(g->ws_mu);
            for (Workspace* w : g->ws_all) ws_destroy(g, w);  // p2p windows go through the communicator first
            g->ws_all.clear();
            g->ws_free.clear();
        }
        delete g->comm;
        g->comm = nullptr;
        for (auto& t : g->tables) cudaFree(t.items);
        for (auto& t : g->wtables) cudaFree(t.items);
        for (auto& kv : g->btabs)
            for (auto& t : kv.second.tables)
            {
                if (t.items) cudaFree(t.items);
                if (t.meta) cudaFree(t.meta);
            }
        for (void* p : {(void*)g->rowptr, (void*)g->col})
            dfree_aligned(p);
        for (void* p : {(void*)g->gdeg, (void*)g->new_of_old})
            if (p) cudaFree(p);
        if (g->stream) cudaStreamDestroy(g->stream);
        delete g;
    });
}

int cpg_chebypower(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources, uint32_t n_sources,
                   double* out, cpg_stats* stats) {
    return drive(g, coeffs, K, sources, nullptr, n_sources, 1, 0, out, false, nullptr, stats);
}

int cpg_chebypower_device(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                          uint32_t n_sources, double* d_out, void* stream, cpg_stats* stats) {
    return drive(g, coeffs, K, sources, nullptr, n_sources, 1, 0, d_out, true, stream, stats);
}

int cpg_chebypower_vec(cpg_graph* g, const double* coeffs, uint32_t K, const double* seeds, uint32_t n_seeds,
                       double* out, cpg_stats* stats) {
    return drive(g, coeffs, K, nullptr, seeds, n_seeds, 1, 1, out, false, nullptr, stats);
}

int cpg_chebypower_batched(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                           uint32_t n_sources, uint32_t tile, double* out, cpg_stats* stats) {
    return drive(g, coeffs, K, sources, nullptr, n_sources, tile, 2, out, false, nullptr, stats);
}

int cpg_chebypower_batched_async(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                                 uint32_t n_sources, uint32_t tile, double* out, cpg_stats* stats) {
    return drive(g, coeffs, K, sources, nullptr, n_sources, tile, 2, out, false, nullptr, stats, 0.0, true);
}

int cpg_graph_sync(cpg_graph* g) {
    if (g && !g->members.empty()) {
        int rc = CPG_OK;
        for (cpg_graph* s : g->members) rc = std::max(rc, cpg_graph_sync(s));
        return rc;
    }
    return guarded([&] {
        require(g != nullptr, "null graph handle");
        DeviceGuard dg(g->device);
        std::vector<Workspace*> all;
        {
            std::lock_guard<std::mutex> lock(g->ws_mu);
            all = g->ws_all;
        }
        for (Workspace* w : all) {
            if (!w) continue;
            CPG_CUDA(cudaStreamSynchronize(w->copy_stream));
            CPG_CUDA(cudaStreamSynchronize(w->stream));
        }
    });
}

int cpg_chebypower_batched_device(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                                  uint32_t n_sources, uint32_t tile, double* d_out, void* stream, cpg_stats* stats) {
    return drive(g, coeffs, K, sources, nullptr, n_sources, tile, 2, d_out, true, stream, stats);
}

// PwMethod (solvers.cpp:87-121): yhat = sum_{k<N} zeta_k P^k e_s with N-1
// fused SpMV steps; N = 1 is zeta_0 e_s.
int cpg_power_method(cpg_graph* g, const double* zeta, uint32_t n_steps, const uint32_t* sources,
                     uint32_t n_sources, double* out, cpg_stats* stats) {
    if (n_steps >= 2) return drive(g, zeta, n_steps - 1, sources, nullptr, n_sources, 1, 3, out, false, nullptr, stats);
    return guarded([&] {
        require(n_steps >= 1, "power_method: n_steps must be >= 1");  // solvers.cpp:91
        check_query(g, zeta, 1, sources, n_sources);
        if (!out) return;
        for (uint32_t q = 0; q < n_sources; ++q) {
            double* o = out + static_cast<size_t>(q) * g->n;
            std::fill(o, o + g->n, 0.0);
            o[sources[q]] = zeta[0];
        }
        if (stats) *stats = cpg_stats{1, 0, 0.0, 0.0, 0.0, 0.0, 0, 0.0, 0};
    });
}

// Queries ranked on the device: only the top-k (caller id, score) pairs per
// source come back (the reference ranks on the host, tools/chebyprop.cpp:148-156).
// Sources run in groups (one device-resident [Q][n] result buffer per group) and
// each result column is ranked on the device while the next group computes.
int cpg_chebypower_topk(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources, uint32_t n_sources,
                        uint32_t k, uint32_t* ids, double* vals, cpg_stats* stats) {
    return guarded([&] {
        check_query(g, coeffs, K, sources, n_sources);
        require(g->members.empty(), "topk: not supported on a multi-device handle (use one shard per process)");
        require(k >= 1 && ids && vals, "topk: k >= 1 and output arrays required");
        const uint32_t kk = std::min(k, g->n);
        DeviceGuard dg(g->device);
        // group size: the single-source grouping rule, bounded by a 2 GB result buffer
        const uint32_t Q = std::max<uint32_t>(
            1, std::min<uint32_t>(single_group(g, n_sources),
                                  static_cast<uint32_t>(std::max<uint64_t>(1, (2ull << 30) / (8ull * g->n)))));
        double* d_res = dalloc<double>(static_cast<size_t>(g->n) * Q);
        cudaStream_t st = nullptr;
        cpg_stats acc{};
        try {
            CPG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            for (uint32_t q0 = 0; q0 < n_sources; q0 += Q) {
                const uint32_t cnt = std::min(Q, n_sources - q0);
                cpg_stats s{};
                const int rc = drive(g, coeffs, K, sources + q0, nullptr, cnt, 1, 0, d_res, true, st, &s);
                if (rc != CPG_OK) fail(rc, cpg_last_error());
                device_topk_batch(d_res, g->n, cnt, kk, ids + static_cast<size_t>(q0) * kk,
                                  vals + static_cast<size_t>(q0) * kk, st);
                acc.iterations = s.iterations;
                acc.push_work += s.push_work;
                acc.wall_seconds += s.wall_seconds;
                acc.device_ms += s.device_ms;
                acc.mass_err_max = std::max(acc.mass_err_max, s.mass_err_max);
                acc.bytes_model += s.bytes_model;
                acc.launches += s.launches;
            }
        } catch (...) {
            if (st) cudaStreamDestroy(st);
            cudaFree(d_res);
            throw;
        }
        cudaStreamDestroy(st);
        cudaFree(d_res);
        if (stats) *stats = acc;
    });
}

// measure (eval.cpp:18-37) on the device: n_cols (truth, estimate) column pairs.
int cpg_measure(cpg_graph* g, const double* truth, const double* estimate, uint32_t n_cols, int on_device,
                cpg_error_report* reports) {
    return guarded([&] {
        require(g && truth && estimate && (reports || n_cols == 0), "null argument");
        require(g->members.empty(), "measure: not supported on a multi-device handle");
        if (!n_cols) return;
        DeviceGuard dg(g->device);
        WsLease lease(g);
        Workspace* w = lease.w;
        cudaStream_t st = w->stream;
        const size_t n = g->n, cols = n_cols;
        const double* dt = truth;
        const double* de = estimate;
        double* tmp = nullptr;
        if (!on_device) {
            tmp = dalloc<double>(2 * n * cols);
            CPG_CUDA(cudaMemcpyAsync(tmp, truth, sizeof(double) * n * cols, cudaMemcpyHostToDevice, st));
            CPG_CUDA(cudaMemcpyAsync(tmp + n * cols, estimate, sizeof(double) * n * cols, cudaMemcpyHostToDevice, st));
            dt = tmp;
            de = tmp + n * cols;
        }
        char* scratch = dalloc<char>(measure_scratch_bytes(g, n_cols) + sizeof(cpg_error_report) * cols);
        cpg_error_report* d_rep =
            reinterpret_cast<cpg_error_report*>(scratch + measure_scratch_bytes(g, n_cols));
        launch_measure(g, dt, de, n_cols, scratch, d_rep, st);
        CPG_CUDA(cudaMemcpyAsync(reports, d_rep, sizeof(cpg_error_report) * cols, cudaMemcpyDeviceToHost, st));
        CPG_CUDA(cudaStreamSynchronize(st));
        dfree(scratch);
        if (tmp) dfree(tmp);
    });
}

// The eval harness's query (tools/chebyprop.cpp:140-160: estimate, then
// measure against the truth) with both steps on the device: per group of
// queries the estimates stay in a device [Q][n] buffer and only the reports
// come back.
int cpg_chebypower_measure(cpg_graph* g, const double* coeffs, uint32_t K, const uint32_t* sources,
                           uint32_t n_sources, const double* truths, int truths_on_device,
                           cpg_error_report* reports, cpg_stats* stats) {
    return guarded([&] {
        check_query(g, coeffs, K, sources, n_sources);
        require(g->members.empty(), "measure: not supported on a multi-device handle");
        require(truths && reports, "null argument");
        DeviceGuard dg(g->device);
        const size_t n = g->n;
        const uint32_t Q = std::max<uint32_t>(
            1, std::min<uint32_t>(single_group(g, n_sources),
                                  static_cast<uint32_t>(std::max<uint64_t>(1, (1ull << 30) / (8ull * n)))));
        double* d_res = dalloc<double>(n * Q);
        double* d_truth = truths_on_device ? nullptr : dalloc<double>(n * Q);
        char* scratch = dalloc<char>(measure_scratch_bytes(g, Q) + sizeof(cpg_error_report) * n_sources);
        cpg_error_report* d_rep = reinterpret_cast<cpg_error_report*>(scratch + measure_scratch_bytes(g, Q));
        cudaStream_t st = nullptr;
        cpg_stats acc{};
        auto cleanup = [&] {
            if (st) cudaStreamDestroy(st);
            cudaFree(d_res);
            if (d_truth) cudaFree(d_truth);
            cudaFree(scratch);
        };
        try {
            CPG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
            for (uint32_t q0 = 0; q0 < n_sources; q0 += Q) {
                const uint32_t cnt = std::min(Q, n_sources - q0);
                const double* t = truths + static_cast<size_t>(q0) * n;
                if (!truths_on_device) {
                    CPG_CUDA(cudaMemcpyAsync(d_truth, t, sizeof(double) * n * cnt, cudaMemcpyHostToDevice, st));
                    t = d_truth;
                }
                cpg_stats s{};
                const int rc = drive(g, coeffs, K, sources + q0, nullptr, cnt, 1, 0, d_res, true, st, &s);
                if (rc != CPG_OK) fail(rc, cpg_last_error());
                launch_measure(g, t, d_res, cnt, scratch, d_rep + q0, st);
                acc.iterations = s.iterations;
                acc.push_work += s.push_work;
                acc.wall_seconds += s.wall_seconds;
                acc.device_ms += s.device_ms;
                acc.mass_err_max = std::max(acc.mass_err_max, s.mass_err_max);
                acc.bytes_model += s.bytes_model;
                acc.launches += s.launches + 2;
            }
            CPG_CUDA(cudaMemcpyAsync(reports, d_rep, sizeof(cpg_error_report) * n_sources, cudaMemcpyDeviceToHost,
                                     st));
            CPG_CUDA(cudaStreamSynchronize(st));
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
        if (stats) *stats = acc;
    });
}

// general_gp_vector / general_gp_matrix with ChebyPower (solvers.cpp:390-414):
// z_j = D^-a f(P) D^a x_j for n_cols dense columns, in tiles of `tile` columns
// through the batched step (tile 1: single-column path).
int cpg_general_gp(cpg_graph* g, const double* coeffs, uint32_t K, double a, const double* X, uint32_t n_cols,
                   uint32_t tile, double* out, cpg_stats* stats) {
    if (tile <= 1) return drive(g, coeffs, K, nullptr, X, n_cols, 1, 1, out, false, nullptr, stats, a);
    return drive(g, coeffs, K, nullptr, X, n_cols, tile, 4, out, false, nullptr, stats, a);
}

int cpg_apply_walk(cpg_graph* g, const double* x, double* y) {
    const double c[2] = {0.0, 1.0};  // c0 T0 + c1 T1 = P x
    return cpg_chebypower_vec(g, c, 1, x, 1, y, nullptr);
}

}  // extern "C"

namespace {
// Observer slow path for one source (seed == null) or one dense seed vector
// (cheby_power_vec, solvers.cpp:197-234): T_k(P)x and the partial estimate
// after every step come back to the host (solvers.cpp:215, 219, 226).
int trace_impl(cpg_graph* g, const double* coeffs, uint32_t K, uint32_t source, const double* seed, double* out,
               double* r_trace, double* est_trace) {
    return guarded([&] {
        if (seed) {
            require(g != nullptr, "null graph handle");
            require(K >= 1, "cheby_power: cheby_steps must be >= 1");  // solvers.cpp:201
            require(coeffs != nullptr, "null argument");
        } else {
            check_query(g, coeffs, K, &source, 1);
        }
        require(g->nranks == 1 && g->members.empty(), "trace is single-GPU only");
        DeviceGuard dg(g->device);
        WsLease lease(g);
        Workspace* w = lease.w;
        cudaStream_t st = w->stream;
        ensure_ws(g, w, 1);
        ensure_group(g, w, K, 1);
        upload_params(w, coeffs, K, &source, 1, st);
        const size_t n = g->n, np = g->n_pad;
        std::vector<uint32_t> no(n), gdeg(np);
        CPG_CUDA(cudaMemcpy(no.data(), g->new_of_old, sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
        CPG_CUDA(cudaMemcpy(gdeg.data(), g->gdeg, sizeof(uint32_t) * np, cudaMemcpyDeviceToHost));
        std::vector<double> wv(np), acc(np);
        auto emit = [&](uint32_t k, const double* wk, const double* av, double a_scale) {
            for (size_t v = 0; v < n; ++v) {
                const uint32_t gv = no[v];
                const double d = static_cast<double>(gdeg[gv]);
                if (r_trace) r_trace[k * n + v] = d * wk[gv];
                if (est_trace) est_trace[k * n + v] = a_scale * d * av[gv];
            }
        };
        // k = 0: T_0 = x, est = c0 x (solvers.cpp:209, 215); x = e_s or the seed
        for (size_t v = 0; v < n; ++v) {
            const double x = seed ? seed[v] : (v == source ? 1.0 : 0.0);
            if (r_trace) r_trace[v] = x;
            if (est_trace) est_trace[v] = coeffs[0] * x;
        }
        CPG_CUDA(cudaMemsetAsync(w->w_a, 0, sizeof(double) * np, st));
        if (seed) {
            ensure_buf(w->d_seeds, w->seeds_cap, n);
            CPG_CUDA(cudaMemcpyAsync(w->d_seeds, seed, sizeof(double) * n, cudaMemcpyHostToDevice, st));
            launch_init_dense(w->w_a, g->gdeg, g->new_of_old, w->d_seeds, g->n, 0.0, st);
        } else {
            launch_init_onehot(w->w_a, g->n_pad, g->gdeg, g->new_of_old, w->d_sources, 0, 1, st);
        }
        CPG_CUDA(cudaMemsetAsync(w->d_mass_partial, 0, sizeof(double) * K * g->chunks * g->step_grid, st));
        for (uint32_t k = 1; k <= K; ++k) {
            run_steps(g, w, k, k, K, false, st, nullptr);
            CPG_CUDA(cudaGetLastError());
            const double* w_io = (k & 1) ? w->w_b : w->w_a;
            CPG_CUDA(cudaMemcpyAsync(wv.data(), w_io, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
            CPG_CUDA(cudaMemcpyAsync(acc.data(), w->acc, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
            CPG_CUDA(cudaStreamSynchronize(st));
            emit(k, wv.data(), acc.data(), 1.0);
            if (k == K && out)
                for (size_t v = 0; v < n; ++v) out[v] = static_cast<double>(gdeg[no[v]]) * acc[no[v]];
        }
    });
}
}  // namespace

extern "C" {

int cpg_chebypower_trace(cpg_graph* g, const double* coeffs, uint32_t K, uint32_t source, double* out,
                         double* r_trace, double* est_trace) {
    return trace_impl(g, coeffs, K, source, nullptr, out, r_trace, est_trace);
}

int cpg_chebypower_vec_trace(cpg_graph* g, const double* coeffs, uint32_t K, const double* seed, double* out,
                             double* r_trace, double* est_trace) {
    if (!seed) return guarded([] { require(false, "null argument"); });
    return trace_impl(g, coeffs, K, 0, seed, out, r_trace, est_trace);
}

int cpg_last_split_profile(cpg_graph* g, double* pieces_ms, double* rows_ms, uint32_t* steps) {
    return guarded([&] {
        require(g != nullptr && pieces_ms && rows_ms && steps, "null argument");
        cpg_graph* h = g->members.empty() ? g : g->members[0];
        std::lock_guard<std::mutex> lock(h->ws_mu);
        *pieces_ms = h->split_prof_pieces_ms;
        *rows_ms = h->split_prof_rows_ms;
        *steps = h->split_prof_steps;
    });
}

uint32_t cpg_sparse_early_steps(const cpg_graph* g, uint32_t tile, uint32_t K) {
    if (!g) return 0;
    if (!g->members.empty()) return cpg_sparse_early_steps(g->members[0], tile, K);
    return sparse_steps(g, tile <= 1, K);
}

double cpg_bytes_per_step(const cpg_graph* g, uint32_t tile) {
    if (!g) return 0.0;
    if (!g->members.empty()) return cpg_bytes_per_step(g->members[0], tile);  // per rank
    // 4 B index + 8*B B gathered row per edge, 8 B row pointer
    // per row, 4 streams of 8*B B per row (read w_{k-1}, write w_{k+1}, read+write
    // acc); sharded adds the received all-gather bytes 8*B*n*(R-1)/R.
    const double B = tile <= 1 ? 1.0 : static_cast<double>(batch_width(tile));
    const double nnz = static_cast<double>(g->nnz_loc), nl = static_cast<double>(g->n_loc);
    double bytes = nnz * (4.0 + 8.0 * B) + 8.0 * (nl + 1) + 32.0 * nl * B;
    if (g->nranks > 1)
        bytes += 8.0 * B * static_cast<double>(g->n_pad) * (g->nranks - 1) / g->nranks;
    return bytes;
}

} // extern "C"
