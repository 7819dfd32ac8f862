// step_kernels.cu -- the hot path: one fused Chebyshev step per launch.
//
// Replaces, per step, the reference's scatter SpMV apply_walk_into
// (graph.cpp:257-267) plus the two dense passes around it in cheby_power_vec
// (solvers.cpp:218 accumulate, :221 recurrence, :222 swap) with ONE pull-SpMV
// kernel in the D^-1-scaled basis  w_k = D^-1 T_k(P) s :
//
//   y(v)      = sum_{u in N(v)} w_k(u)                  (pattern-only A, 4 B index + 8 B gather)
//   w_{k+1}(v)= 2 y(v)/d_v - w_{k-1}(v)                 (in place over w_{k-1})
//   acc(v)   += c_{k+1} w_{k+1}(v)                      (acc = D^-1 yhat)
//   mass     += d_v w_{k+1}(v)                          (= sum T_{k+1}, checks C13)
//   last step: out(v) = d_v acc(v)                      (= yhat, solvers.cpp:225)
//
// Load balance for power-law degrees (rows are degree-sorted at upload):
//   * row tiles: <= 2048 edges; indices streamed coalesced (L1 no-allocate),
//     gathered values staged in shared memory, then each row reduced by a
//     power-of-two lane group sized to the tile's mean degree;
//   * hub rows (deg > 1024): split into 4096-edge pieces, one CTA each; the
//     last-arriving piece (device-scope atomic ticket) sums the piece partials
//     in piece order and runs the epilogue.
// Every reduction has a fixed order, so results are bit-reproducible run to
// run (no floating-point atomics).
#include <cuda_runtime.h>

#include <string>

#include "device_graph.cuh"

namespace cpg {

// L2 residency policy (CPG_L2_HINTS, default on): the index stream is read
// once per step (evict_first), the gathered iterate is re-read across the whole
// step (evict_last), so hub rows stay in the 126 MB L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}

#ifndef CPG_L2_HINTS
#define CPG_L2_HINTS 0  // measured neutral on configs 3-5 (profiles/r01/l2_hints_ab.txt)
#endif

__device__ __forceinline__ uint32_t ld_index(const uint32_t* p) {
    uint32_t v;
#if CPG_L2_HINTS
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v)
                 : "l"(p), "l"(policy_evict_first()));
#else
    asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(p));
#endif
    return v;
}

__device__ __forceinline__ double ld_gather(const double* p) {
#if CPG_L2_HINTS
    double v;
    asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(policy_evict_last()));
    return v;
#else
    return __ldg(p);
#endif
}

__device__ __forceinline__ double2 ld_gather2(const double* p) {
#if CPG_L2_HINTS
    double2 v;
    asm volatile("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(policy_evict_last()));
    return v;
#else
    return __ldg(reinterpret_cast<const double2*>(p));
#endif
}

// Deterministic CTA sum: xor butterfly per warp, warp partials summed in warp
// order by thread 0.  Result valid in thread 0 only.
template <int THREADS>
__device__ __forceinline__ double block_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < THREADS / 32; ++i) s += red[i];
    }
    return s;
}

// Recurrence + accumulation + mass for local row r with neighbour sum y.
// w_prev = w_{k-1}(v) (for the first step: w_0(v)), acc_old = acc(v) (unused
// in the first step).
__device__ __forceinline__ void step_epilogue(const StepArgs& a, uint32_t r, double y, int64_t d, double w_prev,
                                              double acc_old, double& mass) {
    const uint32_t gr = a.row0 + r;
    double w_new = 0.0, acc_new = 0.0;
    if (d > 0) {
        const double dd = static_cast<double>(d);
        if (a.first) {
            w_new = y / dd;  // w_1 = D^-1 A w_0   (T_1 = P T_0, solvers.cpp:212)
            acc_new = a.coeffs[0] * w_prev + a.coeffs[1] * w_new;
        } else {
            w_new = 2.0 * y / dd - w_prev;  // solvers.cpp:221
            acc_new = acc_old + a.coeffs[a.k] * w_new;  // solvers.cpp:218 (for k+1)
        }
        mass += dd * w_new;
    }
    a.w_io[gr] = w_new;
    if (a.last)
        a.out[r] = static_cast<double>(d) * acc_new;
    else
        a.acc[r] = acc_new;
}

__device__ __forceinline__ void load_prev(const StepArgs& a, uint32_t r, double& w_prev, double& acc_old) {
    const uint32_t gr = a.row0 + r;
    if (a.first) {
        w_prev = a.w_cur[gr];
        acc_old = 0.0;
    } else {
        w_prev = a.w_io[gr];
        acc_old = a.acc[r];
    }
}

template <int TILE>
struct TileSmem {
    double vals[TILE];            // gathered w_k(col) of the tile's edges
    double ysum[kTileMaxRows];    // per-row neighbour sums
    int rp[kTileMaxRows + 1];     // row offsets relative to the tile's first edge
};

// One row tile: every global load is issued up front (row offsets, the index
// stream, the epilogue operands of the rows this thread finalises), then the
// gathers; one barrier; lane-group row sums from shared memory; one barrier;
// the fused epilogue with thread t owning rows t and t + 256.
template <int THREADS, int TILE>
__device__ __forceinline__ void process_tile(const StepArgs& a, const WorkItem it, TileSmem<TILE>& sm,
                                             double& mass) {
    constexpr int PER = TILE / THREADS;
    constexpr int RPT = kTileMaxRows / THREADS;
    const uint32_t rb = it.a;
    const int nrows = static_cast<int>(it.b - it.a);
    const int64_t e0 = static_cast<int64_t>(it.c & ((1ull << 40) - 1));
    const int cnt = static_cast<int>((it.c >> 40) & 0x3fff);
    const int lg = static_cast<int>((it.c >> 54) & 7);
    const uint32_t* colp = a.col + e0;

    uint32_t idx[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int j = i * THREADS + threadIdx.x;
        idx[i] = j < cnt ? ld_index(colp + j) : 0u;
    }
    for (int j = threadIdx.x; j <= nrows; j += THREADS) sm.rp[j] = static_cast<int>(a.rowptr[rb + j] - e0);
    double w_prev[RPT], acc_old[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = q * THREADS + threadIdx.x;
        if (r < nrows) load_prev(a, rb + r, w_prev[q], acc_old[q]);
    }
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int j = i * THREADS + threadIdx.x;
        if (j < cnt) sm.vals[j] = ld_gather(a.w_cur + idx[i]);
    }
    __syncthreads();

    const int g = 1 << lg;
    const int sub = threadIdx.x & (g - 1);
    const int grp = threadIdx.x >> lg;
    const int ngrp = THREADS >> lg;
    for (int base = 0; base < nrows; base += ngrp) {
        const int r = base + grp;
        double s = 0.0;
        if (r < nrows) {
            const int b1 = sm.rp[r + 1];
            for (int j = sm.rp[r] + sub; j < b1; j += g) s += sm.vals[j];
        }
        for (int o = g >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (r < nrows && sub == 0) sm.ysum[r] = s;
    }
    __syncthreads();

#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = q * THREADS + threadIdx.x;
        if (r < nrows)
            step_epilogue(a, rb + r, sm.ysum[r], sm.rp[r + 1] - sm.rp[r], w_prev[q], acc_old[q], mass);
    }
    __syncthreads();  // shared memory is reused by the next item
}

template <int THREADS>
__device__ __forceinline__ void process_hub(const StepArgs& a, const WorkItem it, double* red,
                                            int* flag, double& mass) {
    constexpr int PER = kHubPieceEdges / THREADS;
    const uint32_t r = it.a, slot_base = it.b, hub = it.a;
    const int64_t p0 = code_e0(it.c);
    const int64_t p1 = p0 + code_cnt(it.c);
    const int64_t rs = a.rowptr[r], re = a.rowptr[r + 1];
    const int64_t d = re - rs;
    const uint32_t piece = static_cast<uint32_t>((p0 - rs) / kHubPieceEdges);
    const uint32_t P = static_cast<uint32_t>((d + kHubPieceEdges - 1) / kHubPieceEdges);

    uint32_t idx[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int64_t e = p0 + i * THREADS + threadIdx.x;
        idx[i] = e < p1 ? ld_index(a.col + e) : 0u;
    }
    double vals[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int64_t e = p0 + i * THREADS + threadIdx.x;
        vals[i] = e < p1 ? ld_gather(a.w_cur + idx[i]) : 0.0;
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) s += vals[i];
    s = block_sum<THREADS>(s, red);

    if (P == 1) {
        if (threadIdx.x == 0) {
            double wp, ao;
            load_prev(a, r, wp, ao);
            step_epilogue(a, r, s, d, wp, ao, mass);
        }
        return;
    }
    if (threadIdx.x == 0) {
        a.hub_partial[slot_base + piece] = s;
        __threadfence();
        const unsigned prev = atomicAdd(&a.hub_count[hub], 1u);
        *flag = (prev == P - 1);
    }
    __syncthreads();
    if (*flag && threadIdx.x < 32) {  // last piece: ordered sum of the P partials
        __threadfence();
        double y = 0.0;
        for (uint32_t p = threadIdx.x; p < P; p += 32) y += __ldcg(a.hub_partial + slot_base + p);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
        if (threadIdx.x == 0) {
            a.hub_count[hub] = 0u;  // re-arm for the next step
            double wp, ao;
            load_prev(a, r, wp, ao);
            step_epilogue(a, r, y, d, wp, ao, mass);
        }
    }
    __syncthreads();
}

template <int THREADS, int TILE>
__global__ void __launch_bounds__(THREADS) cheby_step_kernel(const StepArgs a) {
    __shared__ TileSmem<TILE> sm;
    __shared__ double red[THREADS / 32];
    __shared__ int flag;
    double mass = 0.0;
    for (uint32_t i = blockIdx.x; i < a.n_items; i += gridDim.x) {
        WorkItem it;
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.items) + i);
        it.a = raw.x;
        it.b = raw.y;
        it.c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
        if (it.c & kHubBit)
            process_hub<THREADS>(a, it, red, &flag, mass);
        else
            process_tile<THREADS, TILE>(a, it, sm, mass);
    }
    mass = block_sum<THREADS>(mass, red);
    if (threadIdx.x == 0) a.mass_partial[blockIdx.x] = mass;
}

// ---------------------------------------------------------------------------
// Batched step: B sources per tile (B in {4,8,16,32,64}), iterates row-major
// [n_pad][B] fp64.  A row is owned by a lane sub-group of L = B/2 lanes (one
// double2 each), so a warp works on RPW = 32/L rows at once and every edge
// costs ONE B*8-byte row fetch shared by the B queries (vs one 8-byte fetch per
// query in the single-source step).  Per row: the epilogue operands are
// prefetched with the first index chunk, then 32-edge chunks: each lane loads
// 32/L indices (coalesced within the sub-group), and U row gathers per lane are
// kept in flight.  Edge order within a row is sequential, so results are
// bit-reproducible.  Rows above kBatchHubEdges are split into pieces combined
// by the ordered last-arriver reduction.
// ---------------------------------------------------------------------------
template <int B>
struct BatchJob {
    uint32_t r;
    int64_t e0, e1, d;
    uint32_t slot, piece, P;
    bool valid, hub;
};

template <int B>
__device__ __forceinline__ BatchJob<B> batch_job(const BatchArgs& a, uint32_t job, uint32_t n_jobs) {
    BatchJob<B> j;
    j.valid = job < n_jobs;
    j.hub = false;
    j.r = 0;
    j.e0 = j.e1 = j.d = 0;
    j.slot = j.piece = j.P = 0;
    if (!j.valid) return j;
    if (job < a.n_hub_items) {
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.hub_items) + job);
        j.hub = true;
        j.r = raw.x;
        j.slot = raw.y;
        const uint64_t c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
        j.e0 = code_e0(c);
        j.e1 = j.e0 + code_cnt(c);
        const int64_t rs = a.rowptr[j.r], re = a.rowptr[j.r + 1];
        j.d = re - rs;
        constexpr int HB = batch_hub_edges(B);
        j.piece = static_cast<uint32_t>((j.e0 - rs) / HB);
        j.P = static_cast<uint32_t>((j.d + HB - 1) / HB);
    } else {
        j.r = a.hub_rows + (job - a.n_hub_items);
        j.e0 = a.rowptr[j.r];
        j.e1 = a.rowptr[j.r + 1];
        j.d = j.e1 - j.e0;
    }
    return j;
}

template <int B>
__device__ __forceinline__ void batch_epilogue(const BatchArgs& a, uint32_t r, double2 y, int64_t d, int cl,
                                               double2 wp, double2 ac) {
    const uint32_t gr = a.row0 + r;
    double2 w_new = {0.0, 0.0}, acc_new = {0.0, 0.0};
    if (d > 0) {
        const double dd = static_cast<double>(d);
        if (a.first) {  // wp holds w_0 of this row
            w_new.x = y.x / dd;
            w_new.y = y.y / dd;
            acc_new.x = a.coeffs[0] * wp.x + a.coeffs[1] * w_new.x;
            acc_new.y = a.coeffs[0] * wp.y + a.coeffs[1] * w_new.y;
        } else {
            const double ck = a.coeffs[a.k];
            w_new.x = 2.0 * y.x / dd - wp.x;
            w_new.y = 2.0 * y.y / dd - wp.y;
            acc_new.x = ac.x + ck * w_new.x;
            acc_new.y = ac.y + ck * w_new.y;
        }
    }
    reinterpret_cast<double2*>(a.w_io + static_cast<size_t>(gr) * B)[cl] = w_new;
    if (a.last) {
        const double dd = static_cast<double>(d);
        reinterpret_cast<double2*>(a.out + static_cast<size_t>(r) * B)[cl] = make_double2(dd * acc_new.x, dd * acc_new.y);
    } else {
        reinterpret_cast<double2*>(a.acc + static_cast<size_t>(r) * B)[cl] = acc_new;
    }
}

template <int B>
__device__ __forceinline__ void batch_prefetch(const BatchArgs& a, uint32_t r, int cl, double2& wp, double2& ac) {
    const uint32_t gr = a.row0 + r;
    if (a.first) {
        wp = reinterpret_cast<const double2*>(a.w_cur + static_cast<size_t>(gr) * B)[cl];
        ac = make_double2(0.0, 0.0);
    } else {
        wp = reinterpret_cast<const double2*>(a.w_io + static_cast<size_t>(gr) * B)[cl];
        ac = reinterpret_cast<const double2*>(a.acc + static_cast<size_t>(r) * B)[cl];
    }
}

// Occupancy over registers: 4 CTAs x 8 warps per SM (64 regs) measured best
// for B = 16 and 64 (profiles/r01/slot_sweep.txt), even with small spills.
template <int B, int U = 8, int MINB = 4>
__global__ void __launch_bounds__(kBatchThreads, MINB) cheby_batch_kernel(const BatchArgs a) {
    constexpr int L = B / 2;      // lanes per row slot
    constexpr int RPW = 32 / L;   // row slots per warp
    constexpr int V = 32 / L;     // indices per lane per 32-edge chunk
    // U: row gathers in flight per lane
    const int lane = threadIdx.x & 31;
    const int slot = lane / L, cl = lane % L;
    const unsigned smask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (slot * L));
    const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n_jobs = a.n_hub_items + (a.n_loc - a.hub_rows);
    for (uint32_t base_job = wg * RPW; base_job < n_jobs; base_job += nw * RPW) {
        const BatchJob<B> j = batch_job<B>(a, base_job + slot, n_jobs);
        double2 wp = {0.0, 0.0}, ac = {0.0, 0.0};
        if (j.valid && !j.hub) batch_prefetch<B>(a, j.r, cl, wp, ac);
        double2 s = {0.0, 0.0};
        for (int64_t e = j.e0; __any_sync(0xffffffffu, e < j.e1); e += 32) {
            const int m = static_cast<int>(e < j.e1 ? (j.e1 - e < 32 ? j.e1 - e : 32) : 0);
            uint32_t c[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int t = v * L + cl;
                c[v] = t < m ? ld_index(a.col + e + t) : 0u;
            }
#pragma unroll
            for (int t0 = 0; t0 < 32; t0 += U) {
                if (!__any_sync(0xffffffffu, t0 < m)) break;
                double2 val[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int t = t0 + q;
                    const uint32_t u = __shfl_sync(0xffffffffu, c[t / L], slot * L + (t % L));
                    val[q] = t < m ? ld_gather2(a.w_cur + static_cast<size_t>(u) * B + 2 * cl) : make_double2(0.0, 0.0);
                }
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    s.x += val[q].x;
                    s.y += val[q].y;
                }
            }
        }
        bool do_epi = j.valid && !j.hub;
        double2 y = s;
        if (__any_sync(0xffffffffu, j.hub)) {
            if (j.hub)
                reinterpret_cast<double2*>(a.hub_partial + static_cast<size_t>(j.slot + j.piece) * B)[cl] = s;
            __threadfence();
            __syncwarp();
            unsigned prev = 0;
            if (j.hub && cl == 0) prev = atomicAdd(&a.hub_count[j.r], 1u);
            prev = __shfl_sync(0xffffffffu, prev, slot * L);
            if (j.hub && prev == j.P - 1) {
                __threadfence();
                y = make_double2(0.0, 0.0);
                for (uint32_t p = 0; p < j.P; ++p) {
                    const double2 v =
                        __ldcg(reinterpret_cast<const double2*>(a.hub_partial + static_cast<size_t>(j.slot + p) * B) + cl);
                    y.x += v.x;
                    y.y += v.y;
                }
                if (cl == 0) a.hub_count[j.r] = 0u;
                batch_prefetch<B>(a, j.r, cl, wp, ac);
                do_epi = true;
            }
        }
        (void)smask;
        if (do_epi) batch_epilogue<B>(a, j.r, y, j.d, cl, wp, ac);
    }
}

// ---------------------------------------------------------------------------
// Staged batched step (B <= 32): persistent CTAs walk the batched item table
// (hub pieces, then row tiles).  For each item the gathered neighbour rows
// (E = 32 KB / (8B) edges x B columns) are copied HBM/L2 -> shared memory with
// cp.async (16 B per copy, no register staging), double-buffered so the copies
// of item t+1 are in flight while item t is reduced.  In-flight bytes are
// bounded by shared memory (2 x 32 KB per CTA), not by registers.  Row slots of
// L = B/2 lanes then sum their rows' staged vectors in edge order
// (deterministic) and run the fused epilogue.  Hub pieces reduce over their E
// edges (fixed slot order) and use the ordered last-arriver combine.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

template <int B>
struct StagedTile {
    static constexpr int L = B / 2;                  // lanes (double2 columns) per row slot
    static constexpr int SLOTS = kBatchThreads / L;  // row slots per CTA
    static constexpr int E = batch_tile_edges(B);    // staged edges per item
    static constexpr int R = batch_tile_rows(B);     // rows per tile
    static constexpr int RPS = R / SLOTS;            // epilogue rows per slot
    static constexpr int PER = E * L / kBatchThreads; // 16-B copies per thread per item
    double2 buf[2][E][L];
    int64_t rp[2][R + 1];
    double2 red[SLOTS][L];
    int flag;
};

// Raw 16-B work item; fields decoded on use (keeps the 3-deep pipeline in registers).
struct ItemInfo {
    uint32_t a, b;
    uint64_t c;
    __device__ __forceinline__ bool hub() const { return (c & kHubBit) != 0; }
    __device__ __forceinline__ uint32_t rb() const { return a; }
    __device__ __forceinline__ uint32_t re() const { return hub() ? a + 1 : b; }
    __device__ __forceinline__ uint32_t slot() const { return b; }
    __device__ __forceinline__ int64_t e0() const { return code_e0(c); }
    __device__ __forceinline__ int cnt() const { return code_cnt(c); }
};

template <int B>
__device__ __forceinline__ ItemInfo decode_item(const BatchArgs& a, uint32_t i) {
    const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.hub_items) + i);
    ItemInfo it;
    it.a = raw.x;
    it.b = raw.y;
    it.c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
    return it;
}

// Issue the cp.async copies of one item into buffer `b`, given its column ids.
template <int B>
__device__ __forceinline__ void stage_item(const BatchArgs& a, StagedTile<B>& sm, int b, const ItemInfo& it,
                                           const uint32_t (&cols)[StagedTile<B>::PER]) {
    using T = StagedTile<B>;
    const int cnt = it.cnt();
#pragma unroll
    for (int i = 0; i < T::PER; ++i) {
        const int k = i * kBatchThreads + threadIdx.x;
        const int e = k / T::L, part = k % T::L;
        if (e < cnt) cp_async16(&sm.buf[b][e][part], a.w_cur + static_cast<size_t>(cols[i]) * B + 2 * part);
    }
    if (!it.hub()) {
        const int nr = static_cast<int>(it.re() - it.rb());
        for (int j = threadIdx.x; j <= nr; j += kBatchThreads) cp_async8(&sm.rp[b][j], a.rowptr + it.rb() + j);
    }
}

template <int B>
__device__ __forceinline__ void load_cols(const BatchArgs& a, const ItemInfo& it,
                                          uint32_t (&cols)[StagedTile<B>::PER]) {
    using T = StagedTile<B>;
    const int cnt = it.cnt();
    const uint32_t* colp = a.col + it.e0();
#pragma unroll
    for (int i = 0; i < T::PER; ++i) {
        const int e = (i * kBatchThreads + static_cast<int>(threadIdx.x)) / T::L;
        cols[i] = e < cnt ? ld_index(colp + e) : 0u;
    }
}

template <int B>
__device__ __forceinline__ void reduce_item(const BatchArgs& a, StagedTile<B>& sm, int b, const ItemInfo& it) {
    using T = StagedTile<B>;
    const int slot = threadIdx.x / T::L, cl = threadIdx.x % T::L;
    const uint32_t rb = it.rb();
    if (!it.hub()) {
        const int nr = static_cast<int>(it.re() - rb);
        const int64_t e0 = sm.rp[b][0];
        // prefetch epilogue operands of this slot's rows, then sum staged rows
        double2 wp[T::RPS], ac[T::RPS];
#pragma unroll
        for (int q = 0; q < T::RPS; ++q) {
            const int r = q * T::SLOTS + slot;
            if (r < nr) batch_prefetch<B>(a, rb + r, cl, wp[q], ac[q]);
        }
#pragma unroll
        for (int q = 0; q < T::RPS; ++q) {
            const int r = q * T::SLOTS + slot;
            if (r < nr) {
                const int b0 = static_cast<int>(sm.rp[b][r] - e0), b1 = static_cast<int>(sm.rp[b][r + 1] - e0);
                double2 s = {0.0, 0.0};
                for (int e = b0; e < b1; ++e) {
                    const double2 v = sm.buf[b][e][cl];
                    s.x += v.x;
                    s.y += v.y;
                }
                batch_epilogue<B>(a, rb + r, s, b1 - b0, cl, wp[q], ac[q]);
            }
        }
        return;
    }
    // hub piece: slot s sums edges s, s+SLOTS, ...; slots combined in order.
    double2 s = {0.0, 0.0};
    const int cnt = it.cnt();
    for (int e = slot; e < cnt; e += T::SLOTS) {
        const double2 v = sm.buf[b][e][cl];
        s.x += v.x;
        s.y += v.y;
    }
    sm.red[slot][cl] = s;
    __syncthreads();
    if (slot == 0) {
        double2 t = {0.0, 0.0};
        for (int q = 0; q < T::SLOTS; ++q) {
            t.x += sm.red[q][cl].x;
            t.y += sm.red[q][cl].y;
        }
        const int64_t rs = a.rowptr[rb];
        const int64_t d = a.rowptr[rb + 1] - rs;
        const uint32_t P = static_cast<uint32_t>((d + T::E - 1) / T::E);
        const uint32_t piece = static_cast<uint32_t>((it.e0() - rs) / T::E);
        if (P == 1) {
            double2 wp, ac;
            batch_prefetch<B>(a, rb, cl, wp, ac);
            batch_epilogue<B>(a, rb, t, d, cl, wp, ac);
        } else {
            reinterpret_cast<double2*>(a.hub_partial + static_cast<size_t>(it.slot() + piece) * B)[cl] = t;
            __threadfence();
            if (T::L < 32) __syncwarp((1u << T::L) - 1u);
            else __syncwarp();
            if (cl == 0) {
                const unsigned prev = atomicAdd(&a.hub_count[rb], 1u);
                sm.flag = prev == P - 1;
            }
            if (T::L < 32) __syncwarp((1u << T::L) - 1u);
            else __syncwarp();
            if (sm.flag) {
                __threadfence();
                double2 y = {0.0, 0.0};
                for (uint32_t p = 0; p < P; ++p) {
                    const double2 v = __ldcg(
                        reinterpret_cast<const double2*>(a.hub_partial + static_cast<size_t>(it.slot() + p) * B) + cl);
                    y.x += v.x;
                    y.y += v.y;
                }
                if (cl == 0) a.hub_count[rb] = 0u;
                double2 wp, ac;
                batch_prefetch<B>(a, rb, cl, wp, ac);
                batch_epilogue<B>(a, rb, y, d, cl, wp, ac);
            }
        }
    }
}

template <int B>
__global__ void __launch_bounds__(kBatchThreads, 3) cheby_batch_staged_kernel(const BatchArgs a) {
    using T = StagedTile<B>;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    T& sm = *reinterpret_cast<T*>(smem_raw);
    uint32_t i = blockIdx.x;
    if (i >= a.n_items) return;
    // software pipeline: item i reduced while the rows of i+G are in flight
    // (cp.async) and the column ids of i+2G are being loaded (registers).
    uint32_t cols[T::PER];
    ItemInfo cur = decode_item<B>(a, i);
    load_cols<B>(a, cur, cols);
    stage_item<B>(a, sm, 0, cur, cols);
    cp_async_commit();
    ItemInfo nxt{0u, 0u, 0ull};
    if (i + gridDim.x < a.n_items) {
        nxt = decode_item<B>(a, i + gridDim.x);
        load_cols<B>(a, nxt, cols);
    }
    int b = 0;
    for (; i < a.n_items; i += gridDim.x) {
        const bool has_next = i + gridDim.x < a.n_items;
        if (has_next) stage_item<B>(a, sm, b ^ 1, nxt, cols);
        cp_async_commit();
        ItemInfo nn{0u, 0u, 0ull};
        const uint32_t i2 = i + 2 * gridDim.x;
        if (i2 < a.n_items) {
            nn = decode_item<B>(a, i2);
            load_cols<B>(a, nn, cols);
        }
        cp_async_wait<1>();  // the copies of item i have landed
        __syncthreads();
        reduce_item<B>(a, sm, b, cur);
        __syncthreads();  // buffer b is free again
        cur = nxt;
        nxt = nn;
        b ^= 1;
    }
    cp_async_wait<0>();
}

template <int B>
size_t staged_smem() {
    return sizeof(StagedTile<B>);
}

// ---------------------------------------------------------------------------
// Streaming batched step (the default batched path).  The chunk's edges are
// split into n_slots equal contiguous ranges; a slot of L = B/2 lanes walks its
// range as one stream of stages: per row it owns entirely, two operand stages
// (the row of w_{k-1} and of acc) then one stage per edge (the gathered
// B*8-byte row of w_k); rows cut by a slot boundary are summed per segment and
// combined by the ordered last-arriver reduction.  Every stage is one 16-B
// cp.async per lane into a per-warp ring of kStreamStages stages, so up to
// 16 x 512 B per warp are in flight without holding registers; no CTA
// barriers.  The consumer (kStreamStages-1 stages behind the producer)
// accumulates in edge order, so results are bit-reproducible.
// ---------------------------------------------------------------------------
enum : uint32_t { kEvNone = 0, kEvOpW = 1, kEvOpAcc = 2, kEvEdge = 3, kEvEndFull = 4, kEvEndPart = 5 };

template <int B>
struct StreamCfg {
    static constexpr int L = B / 2;     // lanes per slot
    static constexpr int RPW = 32 / L;  // slots per warp
    static constexpr int S = kStreamStages;
};

template <int B>
size_t stream_smem_bytes() {
    return static_cast<size_t>(kStreamWarps) * kStreamStages * 32 * (sizeof(double2) + sizeof(uint2));
}

__device__ __forceinline__ uint32_t slot_of_edge(const int64_t* slot_edge, uint32_t n_slots, int64_t e) {
    uint32_t lo = 0, hi = n_slots;  // last s with slot_edge[s] <= e
    while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (slot_edge[mid] <= e) lo = mid; else hi = mid;
    }
    return lo;
}

template <int V>
__device__ __forceinline__ uint32_t pick(const uint32_t (&w)[V], int v) {
    uint32_t r = w[0];
#pragma unroll
    for (int i = 1; i < V; ++i) r = v == i ? w[i] : r;
    return r;
}
template <int V>
__device__ __forceinline__ int64_t pick(const int64_t (&w)[V], int v) {
    int64_t r = w[0];
#pragma unroll
    for (int i = 1; i < V; ++i) r = v == i ? w[i] : r;
    return r;
}

template <int B>
__global__ void __launch_bounds__(kStreamWarps * 32, 2) cheby_batch_stream_kernel(const BatchArgs a) {
    using C = StreamCfg<B>;
    constexpr int W = 32;          // index / row-end window per slot
    constexpr int V = W / C::L;    // window entries per lane
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sl = lane / C::L, cl = lane % C::L;
    const int lane0 = sl * C::L;   // first lane of this slot
    double2* ring = reinterpret_cast<double2*>(smem_raw) + static_cast<size_t>(warp) * C::S * 32;
    uint2* desc = reinterpret_cast<uint2*>(smem_raw + static_cast<size_t>(kStreamWarps) * C::S * 32 * sizeof(double2)) +
                  static_cast<size_t>(warp) * C::S * 32;
    const uint32_t slot = (blockIdx.x * kStreamWarps + warp) * C::RPW + sl;
    const bool live = slot < a.n_slots;
    const unsigned smask = C::L == 32 ? 0xffffffffu : (((1u << C::L) - 1u) << lane0);

    // ---- producer state (replicated across the slot's lanes) ----
    int64_t p_e = 0, p_end = 0, p_rs = 0, p_re = 0, s_begin = 0;
    uint32_t p_row = 0;
    int p_phase = 2;  // 0: operand w, 1: operand acc, 2: edges
    bool p_full = false;
    if (live) {
        s_begin = a.slot_edge[slot];
        p_end = a.slot_edge[slot + 1];
        p_e = s_begin;
        p_row = a.slot_row[slot];
    }
    // windows: column ids of edges [cb, cb+W) and row ends rowptr[rb+1 .. rb+W]
    int64_t cb = p_e, rb = p_row;
    uint32_t cw[V], cn[V];
    int64_t rw[V], rn[V];
    const uint32_t row_lim = a.n_loc;  // rows of this chunk end here (rowptr has row_lim+1 valid entries)
#pragma unroll
    for (int v = 0; v < V; ++v) {
        const int64_t e = cb + v * C::L + cl, e2 = e + W;
        cw[v] = live && e < p_end ? ld_index(a.col + e) : 0u;
        cn[v] = live && e2 < p_end ? ld_index(a.col + e2) : 0u;
        const int64_t r = rb + 1 + v * C::L + cl, r2 = r + W;
        rw[v] = live && r <= row_lim ? a.rowptr[r] : 0;
        rn[v] = live && r2 <= row_lim ? a.rowptr[r2] : 0;
    }
    if (live) {
        p_rs = a.rowptr[p_row];
        p_re = __shfl_sync(smask, rw[0], lane0);  // rowptr[p_row + 1]
        p_full = p_rs >= s_begin && p_re <= p_end;
        p_phase = p_full ? 0 : 2;
    }

    // ---- consumer state ----
    double2 c_sum = {0.0, 0.0}, c_wp = {0.0, 0.0}, c_ac = {0.0, 0.0};

    auto produce = [&](int stage) {
        // window lookups (all lanes, converged): current edge's column and the next row's end
        const int ie = static_cast<int>(p_e - cb);
        const uint32_t u = __shfl_sync(0xffffffffu, pick<V>(cw, ie / C::L), lane0 + ie % C::L);
        const int ir = static_cast<int>(p_row + 1 - rb);  // window slot of rowptr[p_row + 2]
        const int64_t next_re = __shfl_sync(0xffffffffu, pick<V>(rw, ir / C::L), lane0 + ir % C::L);
        uint2 d = make_uint2(0u, kEvNone << 29);
        if (p_e < p_end) {
            const uint32_t gr = a.row0 + p_row;
            const uint32_t deg = static_cast<uint32_t>(p_re - p_rs);
            if (p_phase == 0) {
                const double* src = (a.first ? a.w_cur : a.w_io) + static_cast<size_t>(gr) * B + 2 * cl;
                cp_async16(&ring[stage * 32 + lane], src);
                d = make_uint2(p_row, (kEvOpW << 29) | deg);
                p_phase = 1;
            } else if (p_phase == 1) {
                if (!a.first) cp_async16(&ring[stage * 32 + lane], a.acc + static_cast<size_t>(p_row) * B + 2 * cl);
                d = make_uint2(p_row, (kEvOpAcc << 29) | deg);
                p_phase = 2;
            } else {
                cp_async16(&ring[stage * 32 + lane], a.w_cur + static_cast<size_t>(u) * B + 2 * cl);
                const bool row_done = p_e + 1 == p_re, slot_done = p_e + 1 == p_end;
                uint32_t ev = kEvEdge;
                if (row_done && p_full) ev = kEvEndFull;
                else if (row_done || slot_done) ev = kEvEndPart;
                d = make_uint2(p_row, (ev << 29) | deg);
                ++p_e;
                if (p_e - cb == W) {  // slide the column window
                    cb += W;
#pragma unroll
                    for (int v = 0; v < V; ++v) {
                        cw[v] = cn[v];
                        const int64_t e2 = cb + W + v * C::L + cl;
                        cn[v] = e2 < p_end ? ld_index(a.col + e2) : 0u;
                    }
                }
                if (row_done && p_e < p_end) {  // advance to the next row
                    ++p_row;
                    p_rs = p_re;
                    p_re = next_re;
                    p_full = p_re <= p_end;
                    p_phase = p_full ? 0 : 2;
                    if (p_row + 1 - rb == W) {  // slide the row-end window
                        rb += W;
#pragma unroll
                        for (int v = 0; v < V; ++v) {
                            rw[v] = rn[v];
                            const int64_t r2 = rb + 1 + W + v * C::L + cl;
                            rn[v] = r2 <= row_lim ? a.rowptr[r2] : 0;
                        }
                    }
                }
            }
        }
        desc[stage * 32 + lane] = d;
    };

    auto consume = [&](int stage) {
        const uint2 d = desc[stage * 32 + lane];
        const uint32_t ev = d.y >> 29;
        if (ev == kEvNone) return;
        const double2 v = ring[stage * 32 + lane];
        if (ev == kEvOpW) {
            c_wp = v;
            return;
        }
        if (ev == kEvOpAcc) {
            c_ac = a.first ? make_double2(0.0, 0.0) : v;
            return;
        }
        c_sum.x += v.x;
        c_sum.y += v.y;
        if (ev == kEvEdge) return;
        const uint32_t row = d.x;
        const int64_t deg = d.y & ((1u << 28) - 1);
        if (ev == kEvEndFull) {
            batch_epilogue<B>(a, row, c_sum, deg, cl, c_wp, c_ac);
        } else {  // segment of a row shared with neighbouring slots
            const int64_t rs = a.rowptr[row], re = rs + deg;
            const int64_t seg0 = rs > s_begin ? rs : s_begin;
            const int64_t seg1 = re < p_end ? re : p_end;
            const uint32_t pidx = seg0 == s_begin ? 0u : 1u;
            reinterpret_cast<double2*>(a.hub_partial + (static_cast<size_t>(slot) * 2 + pidx) * B)[cl] = c_sum;
            __threadfence();
            __syncwarp(smask);
            unsigned prev = 0;
            const unsigned seg_len = static_cast<unsigned>(seg1 - seg0);
            if (cl == 0) prev = atomicAdd(&a.hub_count[row], seg_len);
            prev = __shfl_sync(smask, prev, lane0);
            if (prev + seg_len == static_cast<unsigned>(deg)) {  // last segment: ordered combine
                __threadfence();
                const uint32_t s0 = slot_of_edge(a.slot_edge, a.n_slots, rs);
                const uint32_t s1 = slot_of_edge(a.slot_edge, a.n_slots, re - 1);
                double2 y = {0.0, 0.0};
                for (uint32_t q = s0; q <= s1; ++q) {
                    const int64_t qb = a.slot_edge[q];
                    if (a.slot_edge[q + 1] == qb) continue;  // empty slot
                    const uint32_t qi = (rs > qb ? rs : qb) == qb ? 0u : 1u;
                    const double2 t = __ldcg(reinterpret_cast<const double2*>(
                                                 a.hub_partial + (static_cast<size_t>(q) * 2 + qi) * B) + cl);
                    y.x += t.x;
                    y.y += t.y;
                }
                if (cl == 0) a.hub_count[row] = 0u;
                double2 wp, ac;
                batch_prefetch<B>(a, row, cl, wp, ac);
                batch_epilogue<B>(a, row, y, deg, cl, wp, ac);
            }
        }
        c_sum = make_double2(0.0, 0.0);
    };

#pragma unroll 1
    for (int st = 0; st < C::S - 1; ++st) {
        produce(st);
        cp_async_commit();
    }
    int stage_p = C::S - 1, stage_c = 0;
#pragma unroll 1
    while (true) {
        produce(stage_p);
        cp_async_commit();
        cp_async_wait<C::S - 1>();  // this lane's copies of stage_c have landed
        consume(stage_c);
        stage_p = stage_p + 1 == C::S ? 0 : stage_p + 1;
        stage_c = stage_c + 1 == C::S ? 0 : stage_c + 1;
        if (!__any_sync(0xffffffffu, p_e < p_end)) {  // drain the S-1 stages in flight
            cp_async_wait<0>();
#pragma unroll 1
            for (int st = 0; st < C::S - 1; ++st) {
                consume(stage_c);
                stage_c = stage_c + 1 == C::S ? 0 : stage_c + 1;
            }
            break;
        }
    }
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA) batched step, B in {4, 8, 16, 32}.  Each warp owns an
// edge-balanced contiguous edge range.  Per stage of 32 edges every lane issues
// ONE cp.async.bulk (the TMA engine) copying the gathered B*8-byte row of
// w_k for its edge into a per-warp shared-memory ring; completion is tracked
// by an mbarrier per stage (expect_tx), so in-flight bytes cost neither
// registers nor LSU issue slots.  B lanes then walk the staged edges in order
// (segmented by row, bit-reproducible), finished rows are queued in shared
// memory and their fused epilogues run 32 rows at a time so the operand loads
// overlap.  Rows cut by a warp boundary use the ordered last-arriver combine.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t ok = 0;
    while (!ok) {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int B>
struct BulkCfg {
    static constexpr int WARPS = 8;
    static constexpr int STAGE_BYTES = 32 * B * 8;
    static constexpr int S0 = (20 * 1024) / STAGE_BYTES;
    static constexpr int S = S0 < 2 ? 2 : (S0 > 8 ? 8 : S0);  // ring stages per warp
    static constexpr int FR = 32;                              // queued finished rows
    static constexpr int RAW_BYTES = S * STAGE_BYTES + FR * B * 8 + FR * 16 + S * 8;
    static constexpr int WARP_BYTES = (RAW_BYTES + 127) / 128 * 128;  // 16-B bulk-copy alignment per warp
};

template <int B>
size_t bulk_smem_bytes() {
    return static_cast<size_t>(BulkCfg<B>::WARPS) * BulkCfg<B>::WARP_BYTES;
}

template <int B>
__device__ __forceinline__ void bulk_flush(const BatchArgs& a, const double* fin, const uint2* fin_meta, int nf,
                                           int lane) {
    // nf finished rows x B columns: each lane takes (row, column pair) items.
    constexpr int PAIRS = B / 2;
    for (int it = lane; it < nf * PAIRS; it += 32) {
        const int q = it / PAIRS, cl = it % PAIRS;
        const uint32_t row = fin_meta[q].x;
        const int64_t deg = fin_meta[q].y;
        double2 wp, ac;
        batch_prefetch<B>(a, row, cl, wp, ac);
        const double2 y = reinterpret_cast<const double2*>(fin + static_cast<size_t>(q) * B)[cl];
        batch_epilogue<B>(a, row, y, deg, cl, wp, ac);
    }
}

template <int B>
__global__ void __launch_bounds__(BulkCfg<B>::WARPS * 32, 1) cheby_batch_bulk_kernel(const BatchArgs a) {
    using C = BulkCfg<B>;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* base = smem_raw + static_cast<size_t>(warp) * C::WARP_BYTES;
    double* ring = reinterpret_cast<double*>(base);                              // [S][32][B]
    double* fin = reinterpret_cast<double*>(base + C::S * C::STAGE_BYTES);       // [FR][B]
    uint2* fin_meta = reinterpret_cast<uint2*>(base + C::S * C::STAGE_BYTES + C::FR * B * 8);  // [FR]
    uint64_t* bar = reinterpret_cast<uint64_t*>(base + C::S * C::STAGE_BYTES + C::FR * B * 8 + C::FR * 16);

    const uint32_t w = blockIdx.x * C::WARPS + warp;
    if (w >= a.n_slots) return;
    const int64_t e_begin = a.slot_edge[w], e_end = a.slot_edge[w + 1];
    if (e_begin >= e_end) return;

    if (lane == 0)
        for (int st = 0; st < C::S; ++st) mbar_init(&bar[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();

    // producer: stage t covers edges [e_begin + 32t, +32)
    const int64_t n_edges = e_end - e_begin;
    const int64_t n_stages = (n_edges + 31) / 32;
    uint32_t col_next = lane < n_edges ? ld_index(a.col + e_begin + lane) : 0u;
    auto issue = [&](int64_t t) {
        const int st = static_cast<int>(t % C::S);
        const int64_t e0 = e_begin + 32 * t;
        const int nvalid = static_cast<int>(e_end - e0 < 32 ? e_end - e0 : 32);
        const uint32_t u = col_next;
        // prefetch the next stage's column ids
        const int64_t en = e0 + 32 + lane;
        col_next = en < e_end ? ld_index(a.col + en) : 0u;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // slot was read by generic loads
        if (lane == 0) mbar_arrive_expect_tx(&bar[st], static_cast<uint32_t>(nvalid) * B * 8);
        __syncwarp();
        if (lane < nvalid)
            bulk_g2s(ring + (static_cast<size_t>(st) * 32 + lane) * B, a.w_cur + static_cast<size_t>(u) * B, B * 8,
                     &bar[st]);
    };

    // consumer state (uniform across the warp; lanes < B hold one column each)
    uint32_t row = a.slot_row[w];
    int64_t row_rs = a.rowptr[row], row_re = a.rowptr[row + 1];
    double sum = 0.0;
    int nf = 0;

    int64_t t_issue = 0;
    for (; t_issue < n_stages && t_issue < C::S; ++t_issue) issue(t_issue);

    for (int64_t t = 0; t < n_stages; ++t) {
        const int st = static_cast<int>(t % C::S);
        mbar_wait(&bar[st], static_cast<uint32_t>((t / C::S) & 1));
        const int64_t e0 = e_begin + 32 * t;
        const int nvalid = static_cast<int>(e_end - e0 < 32 ? e_end - e0 : 32);
        const double* stage = ring + static_cast<size_t>(st) * 32 * B;
        for (int j = 0; j < nvalid; ++j) {
            if (lane < B) sum += stage[j * B + lane];
            const int64_t e = e0 + j + 1;
            if (e == row_re || e == e_end) {  // row (or this warp's segment of it) ends here
                const bool full = row_rs >= e_begin && row_re <= e_end;
                const int64_t deg = row_re - row_rs;
                if (full) {
                    if (lane < B) fin[nf * B + lane] = sum;
                    if (lane == 0) fin_meta[nf] = make_uint2(row, static_cast<uint32_t>(deg));
                    ++nf;
                    if (nf == C::FR) {
                        __syncwarp();
                        bulk_flush<B>(a, fin, fin_meta, nf, lane);
                        __syncwarp();
                        nf = 0;
                    }
                } else {
                    const int64_t seg0 = row_rs > e_begin ? row_rs : e_begin;
                    const int64_t seg1 = row_re < e_end ? row_re : e_end;
                    const uint32_t pidx = seg0 == e_begin ? 0u : 1u;
                    if (lane < B) a.hub_partial[(static_cast<size_t>(w) * 2 + pidx) * B + lane] = sum;
                    __threadfence();
                    __syncwarp();
                    unsigned prev = 0;
                    if (lane == 0) prev = atomicAdd(&a.hub_count[row], static_cast<unsigned>(seg1 - seg0));
                    prev = __shfl_sync(0xffffffffu, prev, 0);
                    if (prev + static_cast<unsigned>(seg1 - seg0) == static_cast<unsigned>(deg)) {
                        __threadfence();
                        const uint32_t s0 = slot_of_edge(a.slot_edge, a.n_slots, row_rs);
                        const uint32_t s1 = slot_of_edge(a.slot_edge, a.n_slots, row_re - 1);
                        double y = 0.0;
                        for (uint32_t q = s0; q <= s1; ++q) {
                            const int64_t qb = a.slot_edge[q];
                            if (a.slot_edge[q + 1] == qb) continue;
                            const uint32_t qi = (row_rs > qb ? row_rs : qb) == qb ? 0u : 1u;
                            if (lane < B) y += __ldcg(a.hub_partial + (static_cast<size_t>(q) * 2 + qi) * B + lane);
                        }
                        if (lane == 0) a.hub_count[row] = 0u;
                        if (lane < B) fin[nf * B + lane] = y;
                        if (lane == 0) fin_meta[nf] = make_uint2(row, static_cast<uint32_t>(deg));
                        ++nf;
                        if (nf == C::FR) {
                            __syncwarp();
                            bulk_flush<B>(a, fin, fin_meta, nf, lane);
                            __syncwarp();
                            nf = 0;
                        }
                    }
                }
                sum = 0.0;
                if (e < e_end) {  // next row (rows never have degree 0 inside an edge range)
                    ++row;
                    row_rs = row_re;
                    row_re = a.rowptr[row + 1];
                }
            }
        }
        __syncwarp();  // every lane is done reading this stage
        if (t_issue < n_stages) issue(t_issue++);
    }
    __syncwarp();
    bulk_flush<B>(a, fin, fin_meta, nf, lane);
}

// ---------------------------------------------------------------------------
// Small kernels around the steps.
// ---------------------------------------------------------------------------

// w_0 = D^-1 e_s in the global (relabelled) ids; vector pre-zeroed.
__global__ void init_onehot_kernel(double* w, const uint32_t* gdeg, const uint32_t* new_of_old,
                                   const uint32_t* sources, uint32_t q) {
    const uint32_t s = new_of_old[sources[q]];
    w[s] = 1.0 / static_cast<double>(gdeg[s]);
}

// Batched: column j of W_0 = D^-1 e_{s_j}; matrix [n_pad][B] pre-zeroed.
__global__ void init_onehot_batch_kernel(double* W, const uint32_t* gdeg, const uint32_t* new_of_old,
                                         const uint32_t* sources, uint32_t q0, uint32_t count, uint32_t B) {
    const uint32_t j = threadIdx.x;
    if (j < count) {
        const uint32_t s = new_of_old[sources[q0 + j]];
        W[static_cast<size_t>(s) * B + j] = 1.0 / static_cast<double>(gdeg[s]);
    }
}

// w_0 = D^-1 seed for a dense seed given in caller ids.
__global__ void init_dense_kernel(double* w, const uint32_t* gdeg, const uint32_t* new_of_old,
                                  const double* seed, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t s = new_of_old[v];
        w[s] = seed[v] / static_cast<double>(gdeg[s]);
    }
}

// out[v] = full[new_of_old[v]]  (back to the caller's ids).
__global__ void unpermute_kernel(double* out, const double* full, const uint32_t* new_of_old, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        out[v] = full[new_of_old[v]];
}

// Batched: out[j][v] = full[new_of_old[v]][j] for j < count (full is [n_pad][B]).
__global__ void unpermute_batch_kernel(double* out, const double* full, const uint32_t* new_of_old,
                                       uint32_t n, uint32_t count, uint32_t B) {
    const uint64_t total = static_cast<uint64_t>(n) * count;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t j = static_cast<uint32_t>(i / n), v = static_cast<uint32_t>(i % n);
        out[i] = full[static_cast<size_t>(new_of_old[v]) * B + j];
    }
}

// steps[k] = sum_b mass_partial[k][b]  (ordered, one CTA per step).
__global__ void mass_steps_kernel(const double* mass_partial, uint32_t n_part, double* steps) {
    __shared__ double red[kStepThreads / 32];
    const uint32_t k = blockIdx.x;
    double s = 0.0;
    for (uint32_t b = threadIdx.x; b < n_part; b += blockDim.x) s += mass_partial[static_cast<size_t>(k) * n_part + b];
    s = block_sum<kStepThreads>(s, red);
    if (threadIdx.x == 0) steps[k] = s;
}

// err = max(err, max_k |steps[k] - mass0|).
__global__ void mass_err_kernel(const double* steps, uint32_t K, double mass0, double* err) {
    double worst = *err;
    for (uint32_t k = 0; k < K; ++k) worst = fmax(worst, fabs(steps[k] - mass0));
    *err = worst;
}

// Host-side launch wrappers ---------------------------------------------------
void launch_step(const StepArgs& a, int grid, cudaStream_t st) {
    if (a.tile == kTileLarge)
        cheby_step_kernel<kStepThreads, kTileLarge><<<grid, kStepThreads, 0, st>>>(a);
    else
        cheby_step_kernel<kStepThreads, kTileSmall><<<grid, kStepThreads, 0, st>>>(a);
}
int step_occupancy(int tile) {
    int blocks = 0;
    if (tile == kTileLarge)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_kernel<kStepThreads, kTileLarge>,
                                                      kStepThreads, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_kernel<kStepThreads, kTileSmall>,
                                                      kStepThreads, 0);
    return blocks;
}
template <int B>
void launch_staged(const BatchArgs& a, int grid, cudaStream_t st) {
    static bool configured = false;
    const size_t bytes = staged_smem<B>();
    if (!configured) {
        cudaFuncSetAttribute(cheby_batch_staged_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(bytes));
        configured = true;
    }
    cheby_batch_staged_kernel<B><<<grid, kBatchThreads, bytes, st>>>(a);
}

template <int B>
int staged_occupancy() {
    const size_t bytes = staged_smem<B>();
    cudaFuncSetAttribute(cheby_batch_staged_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(bytes));
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_staged_kernel<B>, kBatchThreads, bytes);
    return blocks;
}

template <int B>
void launch_stream_t(const BatchArgs& a, int grid, cudaStream_t st) {
    static bool configured = false;
    const size_t bytes = stream_smem_bytes<B>();
    if (!configured) {
        cudaFuncSetAttribute(cheby_batch_stream_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(bytes));
        configured = true;
    }
    cheby_batch_stream_kernel<B><<<grid, kStreamWarps * 32, bytes, st>>>(a);
}

template <int B>
int stream_occupancy_t() {
    const size_t bytes = stream_smem_bytes<B>();
    cudaFuncSetAttribute(cheby_batch_stream_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(bytes));
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_stream_kernel<B>, kStreamWarps * 32, bytes);
    return blocks;
}

// The register-pipelined slot kernel is the batched default (fastest measured,
// profiles/r01); CPG_BATCH_KERNEL=stream selects the cp.async streaming kernel
// (issue-bound: ~25 instructions per gathered row) for comparison.
template <int B>
void launch_bulk_t(const BatchArgs& a, int grid, cudaStream_t st) {
    static bool configured = false;
    const size_t bytes = bulk_smem_bytes<B>();
    if (!configured) {
        cudaFuncSetAttribute(cheby_batch_bulk_kernel<B>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(bytes));
        configured = true;
    }
    cheby_batch_bulk_kernel<B><<<grid, BulkCfg<B>::WARPS * 32, bytes, st>>>(a);
}

void launch_bulk(const BatchArgs& a, int B, int grid, cudaStream_t st) {
    switch (B) {
    case 4: launch_bulk_t<4>(a, grid, st); break;
    case 8: launch_bulk_t<8>(a, grid, st); break;
    case 16: launch_bulk_t<16>(a, grid, st); break;
    default: launch_bulk_t<32>(a, grid, st); break;
    }
}

int bulk_occupancy(int B) {
    const size_t bytes = B == 4 ? bulk_smem_bytes<4>() : B == 8 ? bulk_smem_bytes<8>() : B == 16 ? bulk_smem_bytes<16>()
                                                                                                   : bulk_smem_bytes<32>();
    int blocks = 0;
    switch (B) {
    case 4:
        cudaFuncSetAttribute(cheby_batch_bulk_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_bulk_kernel<4>, 256, bytes);
        break;
    case 8:
        cudaFuncSetAttribute(cheby_batch_bulk_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_bulk_kernel<8>, 256, bytes);
        break;
    case 16:
        cudaFuncSetAttribute(cheby_batch_bulk_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_bulk_kernel<16>, 256, bytes);
        break;
    default:
        cudaFuncSetAttribute(cheby_batch_bulk_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_bulk_kernel<32>, 256, bytes);
        break;
    }
    return blocks;
}

// CPG_BATCH_KERNEL=bulk selects the TMA bulk-copy kernel for B <= 32.
bool batch_uses_bulk(int B) {
    static const bool on = [] {
        const char* e = std::getenv("CPG_BATCH_KERNEL");
        return e && std::string(e) == "bulk";
    }();
    return on && B <= 32;
}

bool batch_uses_stream() {
    static const bool on = [] {
        const char* e = std::getenv("CPG_BATCH_KERNEL");
        return e && std::string(e) == "stream";
    }();
    return on;
}

void launch_stream(const BatchArgs& a, int B, int grid, cudaStream_t st) {
    switch (B) {
    case 4: launch_stream_t<4>(a, grid, st); break;
    case 8: launch_stream_t<8>(a, grid, st); break;
    case 16: launch_stream_t<16>(a, grid, st); break;
    case 32: launch_stream_t<32>(a, grid, st); break;
    default: launch_stream_t<64>(a, grid, st); break;
    }
}

int stream_occupancy(int B) {
    switch (B) {
    case 4: return stream_occupancy_t<4>();
    case 8: return stream_occupancy_t<8>();
    case 16: return stream_occupancy_t<16>();
    case 32: return stream_occupancy_t<32>();
    default: return stream_occupancy_t<64>();
    }
}

int batch_staged_occupancy(int B) {
    switch (B) {
    case 4: return staged_occupancy<4>();
    case 8: return staged_occupancy<8>();
    case 16: return staged_occupancy<16>();
    default: return staged_occupancy<32>();
    }
}

template <int B, int U, int MINB>
void launch_slot(const BatchArgs& a, cudaStream_t st) {
    int occ = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cheby_batch_kernel<B, U, MINB>, kBatchThreads, 0);
    cheby_batch_kernel<B, U, MINB><<<occ * sms, kBatchThreads, 0, st>>>(a);
}

template <int B>
bool launch_slot_b(const BatchArgs& a, int cfg, cudaStream_t st) {
    switch (cfg) {
    case 41: launch_slot<B, 4, 4>(a, st); return true;
    case 45: launch_slot<B, 4, 5>(a, st); return true;
    case 46: launch_slot<B, 4, 6>(a, st); return true;
    case 64: launch_slot<B, 6, 4>(a, st); return true;
    case 84: launch_slot<B, 8, 4>(a, st); return true;
    case 85: launch_slot<B, 8, 5>(a, st); return true;
    default: return false;
    }
}

bool launch_slot_cfg(const BatchArgs& a, int B, int cfg, cudaStream_t st) {
    switch (B) {
    case 16: return launch_slot_b<16>(a, cfg, st);
    case 32: return launch_slot_b<32>(a, cfg, st);
    case 64: return launch_slot_b<64>(a, cfg, st);
    default: return false;
    }
}

void launch_batch(const BatchArgs& a, int B, int grid, cudaStream_t st) {
    if (batch_uses_tiles(B)) {
        switch (B) {
        case 4: launch_staged<4>(a, grid, st); return;
        case 8: launch_staged<8>(a, grid, st); return;
        case 16: launch_staged<16>(a, grid, st); return;
        default: launch_staged<32>(a, grid, st); return;
        }
    }
    static const int cfg = [] {  // tuning hook: CPG_SLOT_CFG = U*10 + MINB
        const char* e = std::getenv("CPG_SLOT_CFG");
        return e ? std::atoi(e) : 0;
    }();
    if (cfg && launch_slot_cfg(a, B, cfg, st)) return;
    switch (B) {
    case 4: cheby_batch_kernel<4><<<grid, kBatchThreads, 0, st>>>(a); break;
    case 8: cheby_batch_kernel<8><<<grid, kBatchThreads, 0, st>>>(a); break;
    case 16: cheby_batch_kernel<16><<<grid, kBatchThreads, 0, st>>>(a); break;
    case 32: cheby_batch_kernel<32><<<grid, kBatchThreads, 0, st>>>(a); break;
    default: cheby_batch_kernel<64><<<grid, kBatchThreads, 0, st>>>(a); break;
    }
}
int batch_occupancy() {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_kernel<64>, kBatchThreads, 0);
    return blocks;
}
void launch_init_onehot(double* w, const uint32_t* gdeg, const uint32_t* no, const uint32_t* src,
                        uint32_t q, cudaStream_t st) {
    init_onehot_kernel<<<1, 1, 0, st>>>(w, gdeg, no, src, q);
}
void launch_init_onehot_batch(double* W, const uint32_t* gdeg, const uint32_t* no, const uint32_t* src,
                              uint32_t q0, uint32_t count, uint32_t B, cudaStream_t st) {
    init_onehot_batch_kernel<<<1, 64, 0, st>>>(W, gdeg, no, src, q0, count, B);
}
void launch_init_dense(double* w, const uint32_t* gdeg, const uint32_t* no, const double* seed,
                       uint32_t n, cudaStream_t st) {
    init_dense_kernel<<<1184, 256, 0, st>>>(w, gdeg, no, seed, n);
}
void launch_unpermute(double* out, const double* full, const uint32_t* no, uint32_t n, cudaStream_t st) {
    unpermute_kernel<<<1184, 256, 0, st>>>(out, full, no, n);
}
void launch_unpermute_batch(double* out, const double* full, const uint32_t* no, uint32_t n,
                            uint32_t count, uint32_t B, cudaStream_t st) {
    unpermute_batch_kernel<<<2368, 256, 0, st>>>(out, full, no, n, count, B);
}
void launch_mass_steps(const double* mp, uint32_t n_part, uint32_t K, double* steps, cudaStream_t st) {
    mass_steps_kernel<<<K, kStepThreads, 0, st>>>(mp, n_part, steps);
}
void launch_mass_err(const double* steps, uint32_t K, double mass0, double* err, cudaStream_t st) {
    mass_err_kernel<<<1, 1, 0, st>>>(steps, K, mass0, err);
}

} // namespace cpg
