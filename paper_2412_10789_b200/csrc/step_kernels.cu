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
//   * row tiles: <= 1024 or 4096 edges (per graph); indices streamed coalesced (L1 no-allocate),
//     gathered values staged in shared memory, then each row reduced by a
//     power-of-two lane group sized to the tile's mean degree;
//   * hub rows (deg > 1024): split into 4096-edge pieces, one CTA each; the
//     last-arriving piece (device-scope atomic ticket) sums the piece partials
//     in piece order and runs the epilogue.
// Every reduction has a fixed order, so results are bit-reproducible run to
// run (no floating-point atomics).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "device_graph.cuh"

namespace cpg {

// L2 residency policy (CPG_L2_HINTS, default off): the index stream is read
// once per step (evict_first), the gathered iterate is re-read across the whole
// step (evict_last), so hub rows stay in the 126 MB L2.
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t policy_evict_normal() {
    uint64_t p;
    asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
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

__device__ __forceinline__ uint32_t ld_index(const uint32_t* p);
__device__ __forceinline__ uint32_t ld_index_b(const uint32_t* p) {  // batched kernels' index stream
#if CPG_STREAM_EF
    uint32_t v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;"
                 : "=r"(v)
                 : "l"(p), "l"(policy_evict_first()));
    return v;
#else
    return ld_index(p);
#endif
}
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

// CPG_GATHER_NA (A/B hook, default off): gathers of the iterate skip L1
// allocation (a random gather over a table far larger than L1 never re-hits).
#ifndef CPG_GATHER_NA
#define CPG_GATHER_NA 0
#endif
#if CPG_GATHER_NA
#define CPG_GL1 ".L1::no_allocate"
#else
#define CPG_GL1 ""
#endif

__device__ __forceinline__ double ld_gather(const double* p) {
#if CPG_GATHER_NA && !CPG_L2_HINTS
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
#elif CPG_L2_HINTS
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
#elif CPG_GATHER_NA
    double2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
#else
    return __ldg(reinterpret_cast<const double2*>(p));
#endif
}

__device__ __forceinline__ double ld_gather_hot(const double* p, bool hot, uint64_t pol_last, uint64_t pol_first) {
    double v;
    asm volatile("ld.global.nc" CPG_GL1 ".L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(hot ? pol_last : pol_first));
    return v;
}

// Batched gathers with an L2 residency split: the degree-sorted hot prefix of
// the iterate (rows < hot) is loaded evict_last, the cold tail evict_first.
__device__ __forceinline__ double2 ld_gather2_hot(const double* p, bool hot, uint64_t pol_last, uint64_t pol_first) {
    double2 v;
    asm volatile("ld.global.nc" CPG_GL1 ".L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(hot ? pol_last : pol_first));
    return v;
}

// One warp-uniform policy for the whole gathered iterate: addresses in the hot prefix
// [base, base + hot_bytes) are loaded evict_last, the rest of the window (up to 4 GB - 1:
// the sizes are 32-bit) evict_first.  A per-row choice between two policies costs ~9
// instructions per gather (compare, two selects, two moves to uniform registers, two
// predicated loads); this costs none.
__device__ __forceinline__ uint64_t policy_range_hot(const double* base, uint64_t hot_bytes, uint64_t total_bytes) {
    uint64_t p;
    const uint32_t prim = static_cast<uint32_t>(hot_bytes < 0xffffffffull ? hot_bytes : 0xffffffffull);
    const uint32_t tot = static_cast<uint32_t>(total_bytes < 0xffffffffull ? total_bytes : 0xffffffffull);
    asm("createpolicy.range.global.L2::evict_last.L2::evict_first.b64 %0, [%1], %2, %3;"
        : "=l"(p)
        : "l"(base), "r"(prim), "r"(tot));
    return p;
}
__device__ __forceinline__ double2 ld_gather2_pol(const double* p, uint64_t pol) {
    double2 v;
    asm volatile("ld.global.nc" CPG_GL1 ".L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(pol));
    return v;
}

// Programmatic dependent launch (sm_90+): the step kernels are launched with
// programmatic stream serialization, so step k+1's CTAs can become resident as
// step k's retire and run their prologue (work-item decode, row offsets, the
// first index chunk: static graph data) before griddepcontrol.wait returns,
// which is when step k has completed and its stores are visible.  Everything a
// previous step wrote (iterates, acc, hub tickets/partials) is read after the
// wait.  launch_dependents lets the next step's grid be scheduled at once.
// The L1 is not coherent and is invalidated only at a kernel launch; under PDL
// that launch precedes the end of the previous step, whose CTAs on the same SM
// keep caching lines of the buffers it overwrites (its w_{k-1} rows, read
// before they are rewritten) -- the gathers would hit them stale (measured:
// config 3 lost parity).  So the wait is followed by a gpu-scope fence, which
// invalidates the SM's L1 (CCTL.IVALL in the SASS).
#ifndef CPG_PDL_FENCE
#define CPG_PDL_FENCE 1  // A/B hook only: 0 is wrong under PDL (stale L1 lines)
#endif
__device__ __forceinline__ void pdl_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
#if CPG_PDL_FENCE
    __threadfence();
#endif
}
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" :::); }

// Batched-step streams (CPG_STREAM_EF, A/B hook): the epilogue's loads of w_{k-1}
// and acc and its stores of w_{k+1} and acc touch each line once per step; with
// an L2::evict_first policy they neither displace the gathered hot prefix
// (evict_last) nor keep the previous step's hot lines -- the buffer now being
// overwritten -- at evict_last priority beside the current ones.
#ifndef CPG_STREAM_EF
#define CPG_STREAM_EF 1  // +0.3-1.6% on configs 1-5 (profiles/r02/ab/ab_streamef.txt)
#endif
__device__ __forceinline__ double2 ld_stream2(const double* p) {
#if CPG_STREAM_EF
    double2 v;
    asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(v.x), "=d"(v.y)
                 : "l"(p), "l"(policy_evict_first()));
    return v;
#else
    return *reinterpret_cast<const double2*>(p);
#endif
}
__device__ __forceinline__ void st_stream2(double* p, double2 v) {
#if CPG_STREAM_EF
    asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y),
                 "l"(policy_evict_first())
                 : "memory");
#else
    *reinterpret_cast<double2*>(p) = v;
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
template <bool MASK = false>
__device__ __forceinline__ void step_epilogue(const StepArgs& a, uint32_t r, double y, int64_t d, double w_prev,
                                              double acc_old, double& mass) {
    const uint32_t gr = a.row0 + r;
    double w_new = 0.0, acc_new = 0.0;
    if (d > 0) {
        const double dd = static_cast<double>(d);
        if (a.first) {
            w_new = y / dd;  // w_1 = D^-1 A w_0   (T_1 = P T_0, solvers.cpp:212)
            acc_new = a.coeffs[0] * w_prev + a.coeffs[1] * w_new;
        } else if (a.taylor) {
            w_new = y / dd;  // r_{k} = P r_{k-1} (solvers.cpp:105-106)
            acc_new = acc_old + a.coeffs[a.k] * w_new;  // solvers.cpp:102
        } else {
            w_new = 2.0 * y / dd - w_prev;  // solvers.cpp:221
            acc_new = acc_old + a.coeffs[a.k] * w_new;  // solvers.cpp:218 (for k+1)
        }
        mass += dd * w_new;
    }
    CPG_CHECK(gr < a.chk_npad && r < a.chk_nloc, "step epilogue row", gr, a.chk_npad);
    if (MASK && a.nz_out && w_new != 0.0) nz_set(a.nz_out, gr);  // support of w_{k+1} for the next masked step
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
template <int THREADS, int TILE, bool PDL, bool MASK = false>
__device__ __forceinline__ void process_tile(const StepArgs& a, const WorkItem it, TileSmem<TILE>& sm,
                                             double& mass, bool& wait_pending) {
    constexpr int PER = TILE / THREADS;
    constexpr int RPT = kTileMaxRows / THREADS;
    const uint32_t rb = it.a;
    const int nrows = static_cast<int>(it.b - it.a);
    const int64_t e0 = static_cast<int64_t>(it.c & ((1ull << 40) - 1));
    const int cnt = static_cast<int>((it.c >> 40) & 0x3fff);
    const int lg = static_cast<int>((it.c >> 54) & 7);
    const uint32_t* colp = a.col + e0;
    CPG_CHECK(static_cast<uint64_t>(e0) + cnt <= a.chk_nnz && nrows <= kTileMaxRows && cnt <= TILE, "tile edges",
              e0 + cnt, a.chk_nnz);

    uint32_t idx[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int j = i * THREADS + threadIdx.x;
        idx[i] = j < cnt ? ld_index(colp + j) : 0u;
    }
    for (int j = threadIdx.x; j <= nrows; j += THREADS) sm.rp[j] = static_cast<int>(a.rowptr[rb + j] - e0);
    if (PDL && wait_pending) {  // first item of this CTA: the previous step's iterate from here on
        pdl_wait();
        wait_pending = false;
    }
    double w_prev[RPT], acc_old[RPT];
#pragma unroll
    for (int q = 0; q < RPT; ++q) {
        const int r = q * THREADS + threadIdx.x;
        if (r < nrows) load_prev(a, rb + r, w_prev[q], acc_old[q]);
    }
    if constexpr (MASK) {  // masked (sparse early) step: every support word first, then the set rows
        uint32_t wd[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = i * THREADS + threadIdx.x;
            wd[i] = j < cnt ? __ldg(a.nz_in + (idx[i] >> 5)) : 0u;
        }
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = i * THREADS + threadIdx.x;
            if (j < cnt) sm.vals[j] = (wd[i] >> (idx[i] & 31)) & 1u ? ld_gather(a.w_cur + idx[i]) : 0.0;
        }
    } else if (a.hot_rows) {
        const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = i * THREADS + threadIdx.x;
            if (j < cnt) sm.vals[j] = ld_gather_hot(a.w_cur + idx[i], idx[i] < a.hot_rows, pol_last, pol_first);
        }
    } else {
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = i * THREADS + threadIdx.x;
            CPG_CHECK(j >= cnt || idx[i] < a.chk_npad, "tile gather", idx[i], a.chk_npad);
            if (j < cnt) sm.vals[j] = ld_gather(a.w_cur + idx[i]);
        }
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
            step_epilogue<MASK>(a, rb + r, sm.ysum[r], sm.rp[r + 1] - sm.rp[r], w_prev[q], acc_old[q], mass);
    }
    __syncthreads();  // shared memory is reused by the next item
}

template <int THREADS, bool PDL, bool MASK = false>
__device__ __forceinline__ void process_hub(const StepArgs& a, const WorkItem it, double* red,
                                            int* flag, double& mass, bool& wait_pending) {
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
    if (PDL && wait_pending) {
        pdl_wait();
        wait_pending = false;
    }
    double vals[PER];
#pragma unroll
    for (int i = 0; i < PER; ++i) {
        const int64_t e = p0 + i * THREADS + threadIdx.x;
        CPG_CHECK(e >= p1 || (idx[i] < a.chk_npad && static_cast<uint64_t>(e) < a.chk_nnz), "hub gather", idx[i],
                  a.chk_npad);
        if constexpr (MASK) {
            vals[i] = 0.0;
        } else {
            vals[i] = e < p1 ? ld_gather(a.w_cur + idx[i]) : 0.0;
        }
    }
    if constexpr (MASK) {  // support words first, then the set rows (see process_tile)
        uint32_t wd[PER];
#pragma unroll
        for (int i = 0; i < PER; ++i) wd[i] = p0 + i * THREADS + threadIdx.x < p1 ? __ldg(a.nz_in + (idx[i] >> 5)) : 0u;
#pragma unroll
        for (int i = 0; i < PER; ++i)
            if ((wd[i] >> (idx[i] & 31)) & 1u) vals[i] = ld_gather(a.w_cur + idx[i]);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < PER; ++i) s += vals[i];
    s = block_sum<THREADS>(s, red);

    if (P == 1) {
        if (threadIdx.x == 0) {
            double wp, ao;
            load_prev(a, r, wp, ao);
            step_epilogue<MASK>(a, r, s, d, wp, ao, mass);
        }
        return;
    }
    if (threadIdx.x == 0) {
        CPG_CHECK(slot_base + P <= a.chk_parts, "hub partial slot", slot_base + P, a.chk_parts);
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
            step_epilogue<MASK>(a, r, y, d, wp, ao, mass);
        }
    }
    __syncthreads();
}

template <int THREADS, int TILE, bool MASK = false>
__global__ void __launch_bounds__(THREADS) cheby_step_kernel(const StepArgs a) {
    __shared__ TileSmem<TILE> sm;
    __shared__ double red[THREADS / 32];
    __shared__ int flag;
    double mass = 0.0;
    bool wait_pending = true;
    pdl_launch_dependents();
    for (uint32_t i = blockIdx.x; i < a.n_items; i += gridDim.x) {
        WorkItem it;
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.items) + i);
        it.a = raw.x;
        it.b = raw.y;
        it.c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
        if (it.c & kHubBit)
            process_hub<THREADS, true, MASK>(a, it, red, &flag, mass, wait_pending);
        else
            process_tile<THREADS, TILE, true, MASK>(a, it, sm, mass, wait_pending);
    }
    mass = block_sum<THREADS>(mass, red);
    CPG_CHECK(threadIdx.x != 0 || blockIdx.x < a.chk_mass, "step mass slot", blockIdx.x, a.chk_mass);
    if (threadIdx.x == 0) a.mass_partial[blockIdx.x] = mass;
}

// Split single-source step (CPG_STEP_SPLIT): the hub pieces of the table
// (items [0, n_hub_items)) and the row tiles (the rest) in two kernels, so the
// tile kernel drops the hub path's registers and fits more CTAs per SM.  Each
// writes its own CTAs' mass partials (the tile kernel's start after the hub
// kernel's grid).
template <int THREADS, bool MASK = false>
__global__ void __launch_bounds__(THREADS) cheby_step_hubs_kernel(const StepArgs a) {
    __shared__ double red[THREADS / 32];
    __shared__ int flag;
    double mass = 0.0;
    bool wait_pending = true;
    for (uint32_t i = blockIdx.x; i < a.n_items; i += gridDim.x) {
        WorkItem it;
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.items) + i);
        it.a = raw.x;
        it.b = raw.y;
        it.c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
        process_hub<THREADS, false, MASK>(a, it, red, &flag, mass, wait_pending);
    }
    mass = block_sum<THREADS>(mass, red);
    CPG_CHECK(threadIdx.x != 0 || blockIdx.x < a.chk_mass, "step mass slot", blockIdx.x, a.chk_mass);
    if (threadIdx.x == 0) a.mass_partial[blockIdx.x] = mass;
}

template <int THREADS, int TILE, int MINB, bool MASK = false>
__global__ void __launch_bounds__(THREADS, MINB) cheby_step_tiles_kernel(const StepArgs a) {
    __shared__ TileSmem<TILE> sm;
    __shared__ double red[THREADS / 32];
    double mass = 0.0;
    bool wait_pending = true;
    for (uint32_t i = blockIdx.x; i < a.n_items; i += gridDim.x) {
        WorkItem it;
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.items) + i);
        it.a = raw.x;
        it.b = raw.y;
        it.c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
        process_tile<THREADS, TILE, false, MASK>(a, it, sm, mass, wait_pending);
    }
    mass = block_sum<THREADS>(mass, red);
    CPG_CHECK(threadIdx.x != 0 || blockIdx.x < a.chk_mass, "step mass slot", blockIdx.x, a.chk_mass);
    if (threadIdx.x == 0) a.mass_partial[blockIdx.x] = mass;
}

// ---------------------------------------------------------------------------
// Warp-tile single-source step (CPG_WARP_TILES; round 2): every warp works its
// own items with no CTA barrier.  Items (graph_build.cu build_warp_table):
//   * tiles of <= kWarpTileEdges edges and <= 64 rows of degree <= kWarpTileEdges/2:
//     the warp loads the 16 indices per lane (coalesced), the rows' offsets and
//     epilogue operands, issues its 16 gathers, stages them in its own shared
//     slice, sums each row with a lane group sized to the tile's mean degree
//     (__syncwarp only), and runs the fused epilogue for rows lane, lane + 32;
//   * single rows of kWarpTileEdges/2 < degree <= kWarpLongRow: the warp sweeps
//     the row 32*U edges at a time, sums in registers and reduces with shuffles;
//   * rows above kWarpLongRow are CTA hub pieces (cheby_step_hubs_kernel).
// Warps claim items from a per-(step, chunk) counter (one atomic per item).
// Summation orders are fixed (lane groups / xor trees), so results are
// bit-reproducible run to run, like the CTA tiles.
struct WarpTileSmem {
    double vals[kWarpTileEdges];
    double ysum[kWarpTileRows];
    int rp[kWarpTileRows + 1];
};

template <int WARPS>
__global__ void __launch_bounds__(WARPS * 32, 4) cheby_step_warp_kernel(const StepArgs a, unsigned int* ctr) {
    __shared__ WarpTileSmem smw[WARPS];
    __shared__ double red[WARPS];
    constexpr int PER = kWarpTileEdges / 32;  // indices / gathers per lane of a tile
    constexpr int U = 16;                     // gathers in flight per lane on a long row
    const int lane = threadIdx.x & 31;
    WarpTileSmem& sm = smw[threadIdx.x >> 5];
    double mass = 0.0;
    for (;;) {
        uint32_t i = 0;
        if (lane == 0) i = atomicAdd(ctr, 1u);
        i = __shfl_sync(0xffffffffu, i, 0);
        if (i >= a.n_items) break;
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.items) + i);
        const uint32_t rb = raw.x;
        const int nrows = static_cast<int>(raw.y - raw.x);
        const uint64_t c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
        const int64_t e0 = code_e0(c);
        const int cnt = code_cnt(c);
        const int lg = static_cast<int>((c >> 54) & 7);
        CPG_CHECK(static_cast<uint64_t>(e0) + cnt <= a.chk_nnz && nrows <= kWarpTileRows, "warp tile", e0 + cnt,
                  a.chk_nnz);
        if (nrows == 1 && cnt > kWarpTileEdges / 2) {  // one long row, swept by the whole warp
            double w_prev = 0.0, acc_old = 0.0;
            if (lane == 0) load_prev(a, rb, w_prev, acc_old);
            double s = 0.0;
            for (int base = 0; base < cnt; base += 32 * U) {
                uint32_t idx[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int j = base + q * 32 + lane;
                    idx[q] = j < cnt ? ld_index(a.col + e0 + j) : 0u;
                }
                double v[U];
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    const int j = base + q * 32 + lane;
                    CPG_CHECK(j >= cnt || idx[q] < a.chk_npad, "warp long gather", idx[q], a.chk_npad);
                    v[q] = j < cnt ? ld_gather(a.w_cur + idx[q]) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < U; ++q) s += v[q];
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
            if (lane == 0) step_epilogue(a, rb, s, cnt, w_prev, acc_old, mass);
            continue;
        }
        uint32_t idx[PER];
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int j = q * 32 + lane;
            idx[q] = j < cnt ? ld_index(a.col + e0 + j) : 0u;
        }
        for (int j = lane; j <= nrows; j += 32) sm.rp[j] = static_cast<int>(a.rowptr[rb + j] - e0);
        double w_prev[2], acc_old[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int r = q * 32 + lane;
            if (r < nrows) load_prev(a, rb + r, w_prev[q], acc_old[q]);
        }
#pragma unroll
        for (int q = 0; q < PER; ++q) {
            const int j = q * 32 + lane;
            CPG_CHECK(j >= cnt || idx[q] < a.chk_npad, "warp tile gather", idx[q], a.chk_npad);
            if (j < cnt) sm.vals[j] = ld_gather(a.w_cur + idx[q]);
        }
        __syncwarp();
        const int g = 1 << lg;
        const int sub = lane & (g - 1);
        const int grp = lane >> lg;
        const int ngrp = 32 >> lg;
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
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const int r = q * 32 + lane;
            if (r < nrows) step_epilogue(a, rb + r, sm.ysum[r], sm.rp[r + 1] - sm.rp[r], w_prev[q], acc_old[q], mass);
        }
        __syncwarp();  // the warp's shared slice is reused by its next item
    }
    mass = block_sum<WARPS * 32>(mass, red);
    CPG_CHECK(threadIdx.x != 0 || blockIdx.x < a.chk_mass, "step mass slot", blockIdx.x, a.chk_mass);
    if (threadIdx.x == 0) a.mass_partial[blockIdx.x] = mass;
}

// Query group: nq single-source queries per launch (small graphs, where one
// query cannot fill the GPU).  Items x queries: job x = q * n_items + i, so a
// CTA's queries are nondecreasing and its mass partial is flushed once per
// query it touched.  The one-query launch keeps cheby_step_kernel: sharing its
// code measured 2.6% slower on config 3 (instruction schedule).
template <int THREADS, int TILE>
__global__ void __launch_bounds__(THREADS) cheby_step_group_kernel(const StepArgs a, const StepGroup gq) {
    __shared__ TileSmem<TILE> sm;
    __shared__ double red[THREADS / 32];
    __shared__ int flag;
    double mass = 0.0;
    bool wait_pending = false;  // launched plainly (PDL measured slower for query groups)
    const uint32_t total = a.n_items * gq.nq;
    uint32_t q_cur = 0u;
    for (uint32_t x = blockIdx.x; x < total; x += gridDim.x) {
        WorkItem it;
        const uint32_t q = x / a.n_items;
        const uint32_t i = x - q * a.n_items;
        if (q != q_cur) {  // CTA-uniform
            mass = block_sum<THREADS>(mass, red);
            if (threadIdx.x == 0) a.mass_partial[static_cast<size_t>(q_cur) * gq.mass_stride + blockIdx.x] = mass;
            mass = 0.0;
            q_cur = q;
        }
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.items) + i);
        it.a = raw.x;
        it.b = raw.y;
        it.c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
        {  // the query's slices
            StepArgs aq = a;
            aq.w_cur = a.w_cur + q_cur * gq.vec_stride;
            aq.w_io = a.w_io + q_cur * gq.vec_stride;
            aq.acc = a.acc + q_cur * gq.acc_stride;
            aq.out = a.out + q_cur * gq.acc_stride;
            aq.hub_partial = a.hub_partial + static_cast<size_t>(q_cur) * gq.part_stride;
            aq.hub_count = a.hub_count + static_cast<size_t>(q_cur) * gq.cnt_stride;
            if (it.c & kHubBit)
                process_hub<THREADS, false>(aq, it, red, &flag, mass, wait_pending);
            else
                process_tile<THREADS, TILE, false>(aq, it, sm, mass, wait_pending);
        }
    }
    mass = block_sum<THREADS>(mass, red);
    if (threadIdx.x == 0) a.mass_partial[static_cast<size_t>(q_cur) * gq.mass_stride + blockIdx.x] = mass;
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
// bit-reproducible.  Rows above batch_hub_edges(B) are split into pieces combined
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

// Per-warp column sums of the mass (acceptance C13), two ways (MODE):
//   1 = each lane keeps its two columns' sums in registers across its rows and
//       the warp folds its row slots with an xor-shuffle tree at the end (no
//       shared memory: the L1 carve-out stays whole for the gathers);
//   0 = per-lane shared-memory cells mcells[warp][slot][column] (no registers
//       held across the row loop).
// The fused kernel uses 1 for B <= 16 and 0 for wider rows, whose instances
// already spill; the split kernels use 0 (profiles/r02/ab_mass.txt).
// CPG_MASS_MODE (compile-time A/B hook) forces 0, 1, or 2 = no mass (timing
// only; batched mass_err then reads 1).  Every order is fixed (the warps are
// summed in order by mass_steps_batch_kernel), so with a static job stride the
// value is reproducible run to run.
#ifndef CPG_MASS_MODE
#define CPG_MASS_MODE -1
#endif
// Ordered sum of a hub row's P piece partials (rows of B doubles; this lane's
// double2 at column pair cl): the loads go out 8 at a time, the adds stay in
// piece order, so the result is the plain sequential sum -- bit-identical --
// with P/8 dependent L2 round trips instead of one per piece.
// UN = loads in flight.  The split path's piece kernel uses 8 (config 5: +0.9%); the
// fused kernel keeps 1 -- its B = 16 instance spills more with 8 and lost 4% on configs
// 1-2 (profiles/r02/ab/ab_unroll.txt).  CPG_PARTIAL_UNROLL overrides both (A/B hook).
template <int B, uint32_t UN_DEFAULT>
__device__ __forceinline__ double2 sum_partials(const double* hp, uint32_t slot, uint32_t P, int cl) {
#ifdef CPG_PARTIAL_UNROLL
    constexpr uint32_t UN = CPG_PARTIAL_UNROLL;
#else
    constexpr uint32_t UN = UN_DEFAULT;
#endif
    double2 y = make_double2(0.0, 0.0);
    uint32_t p = 0;
    for (; p + UN <= P; p += UN) {
        double2 v[UN];
#pragma unroll
        for (uint32_t q = 0; q < UN; ++q)
            v[q] = __ldcg(reinterpret_cast<const double2*>(hp + static_cast<size_t>(slot + p + q) * B) + cl);
#pragma unroll
        for (uint32_t q = 0; q < UN; ++q) {
            y.x += v[q].x;
            y.y += v[q].y;
        }
    }
    for (; p < P; ++p) {
        const double2 v = __ldcg(reinterpret_cast<const double2*>(hp + static_cast<size_t>(slot + p) * B) + cl);
        y.x += v.x;
        y.y += v.y;
    }
    return y;
}

template <int PREF>
constexpr int mass_mode() {
    return CPG_MASS_MODE >= 0 ? CPG_MASS_MODE : PREF;
}

template <int B>
__device__ __forceinline__ double* batch_mass_cell() {
    __shared__ __align__(16) double mcells[kBatchThreads / 32][64];  // [warp][slot * B + column], RPW * B = 64
    const int lane = threadIdx.x & 31;
    return &mcells[threadIdx.x >> 5][(lane / (B / 2)) * B + 2 * (lane % (B / 2))];
}

template <int B, int MODE>
__device__ __forceinline__ void batch_mass_init(double2& msum) {
    msum = make_double2(0.0, 0.0);
    if (MODE == 0) {
        double* c = batch_mass_cell<B>();
        c[0] = 0.0;
        c[1] = 0.0;
    }
}

template <int B, int MODE>
__device__ __forceinline__ void batch_mass_add(double2& msum, double m0, double m1) {
    if (MODE == 0) {  // one 16-B shared load and store (the cell pair is 16-B aligned)
        double2* mcell = reinterpret_cast<double2*>(batch_mass_cell<B>());
        double2 c = *mcell;
        c.x += m0;
        c.y += m1;
        *mcell = c;
    } else if (MODE == 1) {
        msum.x += m0;
        msum.y += m1;
    }
}

template <int B, int MODE>
__device__ __forceinline__ void batch_mass_flush(const BatchArgs& a, double2 msum) {
    if (!a.mass_partial) return;  // uniform over the launch
    constexpr int L = B / 2;
    const int lane = threadIdx.x & 31;
    double* dst = a.mass_partial + (static_cast<size_t>(blockIdx.x) * (kBatchThreads / 32) + (threadIdx.x >> 5)) * B;
    CPG_CHECK(static_cast<uint64_t>(blockIdx.x + 1) * (kBatchThreads / 32) <= a.chk_mass, "batch mass row",
              (blockIdx.x + 1) * (kBatchThreads / 32), a.chk_mass);
    if (MODE == 1) {
        // lane = slot * L + cl: fold the row slots (lane bits >= log2 L) into slot 0
#pragma unroll
        for (int o = 16; o >= L; o >>= 1) {
            msum.x += __shfl_xor_sync(0xffffffffu, msum.x, o);
            msum.y += __shfl_xor_sync(0xffffffffu, msum.y, o);
        }
        if (lane < L) {
            dst[2 * lane] = msum.x;
            dst[2 * lane + 1] = msum.y;
        }
        return;
    }
    __syncwarp();
    if (lane < L) {  // lane l sums its warp's row slots for columns 2l, 2l+1 (warp barrier only)
        double s0 = 0.0, s1 = 0.0;
        if (MODE == 0) {
            const double* c = batch_mass_cell<B>();  // slot 0 cells of this lane's columns
#pragma unroll
            for (int r = 0; r < 64 / B; ++r) {
                s0 += c[r * B];
                s1 += c[r * B + 1];
            }
        }
        dst[2 * lane] = s0;
        dst[2 * lane + 1] = s1;
    }
}

// U row gathers of a masked (sparse early) step: the U edges' support words
// are loaded together first (one L2 round trip for all U), then only the rows
// whose bit is set are gathered -- testing and gathering edge by edge would
// chain U dependent round trips.
template <int B, int U>
__device__ __forceinline__ void gather_rows_masked(const BatchArgs& a, const uint32_t* c, int t0, int m, int slot,
                                                   int cl, double2* val, uint64_t pol_last, uint64_t pol_first) {
    constexpr int L = B / 2;
    uint32_t uq[U], wd[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const int t = t0 + q;
        uq[q] = __shfl_sync(0xffffffffu, c[t / L], slot * L + (t % L));
        CPG_CHECK(t >= m || uq[q] < a.chk_npad, "batch gather", uq[q], a.chk_npad);
        wd[q] = t < m ? __ldg(a.nz_in + (uq[q] >> 5)) : 0u;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
        const uint32_t u = uq[q];
        val[q] = (wd[q] >> (u & 31)) & 1u
                     ? (a.hot_rows ? ld_gather2_hot(a.w_cur + static_cast<size_t>(u) * B + 2 * cl, u < a.hot_rows,
                                                    pol_last, pol_first)
                                   : ld_gather2(a.w_cur + static_cast<size_t>(u) * B + 2 * cl))
                     : make_double2(0.0, 0.0);
    }
}

template <int B, bool PEER, int MM, bool MASK = false>
__device__ __forceinline__ void batch_epilogue(const BatchArgs& a, const PeerArgs& pa, uint32_t r, double2 y,
                                               int64_t d, int cl, double2 wp, double2 ac, double2& msum) {
    const uint32_t gr = a.row0 + r;
    CPG_CHECK(gr < a.chk_npad && r < a.chk_nloc, "batch epilogue row", gr, a.chk_npad);
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
        // sum_v d_v w_{k+1}(v) = sum_v T_{k+1}(v), per column
        batch_mass_add<B, MM>(msum, dd * w_new.x, dd * w_new.y);
    }
    // support of w_{k+1} for the next masked step (any column of the row nonzero)
    if (MASK && a.nz_out && (w_new.x != 0.0 || w_new.y != 0.0)) nz_set(a.nz_out, gr);
    st_stream2(a.w_io + static_cast<size_t>(gr) * B + 2 * cl, w_new);
    if (PEER) {  // fused all-gather: the row into every other rank's replica (NVLink stores)
        for (int p = 0; p < pa.n_peer; ++p)
            if (p != pa.self) reinterpret_cast<double2*>(pa.peer_io[p] + static_cast<size_t>(gr) * B)[cl] = w_new;
    }
    if (a.last) {
        const double dd = static_cast<double>(d);
        st_stream2(a.out + static_cast<size_t>(r) * B + 2 * cl, make_double2(dd * acc_new.x, dd * acc_new.y));
    } else {
        st_stream2(a.acc + static_cast<size_t>(r) * B + 2 * cl, acc_new);
    }
}

// Lane 0 claims the next n jobs of the launch for its warp (warp-uniform result).
__device__ __forceinline__ uint32_t claim_jobs(unsigned int* ctr, int lane, uint32_t n) {
    uint32_t j = 0;
    if (lane == 0) j = atomicAdd(ctr, n);
    return __shfl_sync(0xffffffffu, j, 0);
}

template <int B>
__device__ __forceinline__ void batch_prefetch(const BatchArgs& a, uint32_t r, int cl, double2& wp, double2& ac) {
    const uint32_t gr = a.row0 + r;
    if (a.first) {
        wp = reinterpret_cast<const double2*>(a.w_cur + static_cast<size_t>(gr) * B)[cl];
        ac = make_double2(0.0, 0.0);
    } else {
        wp = ld_stream2(a.w_io + static_cast<size_t>(gr) * B + 2 * cl);
        ac = ld_stream2(a.acc + static_cast<size_t>(r) * B + 2 * cl);
    }
}

// Occupancy over registers: 4 CTAs x 8 warps per SM (64 regs) measured best
// for B = 16 and 64 (profiles/r01/slot_sweep.txt), even with small spills.
template <int B, int U = 8, int MINB = 4, bool PEER = false, bool MASK = false>
__global__ void __launch_bounds__(kBatchThreads, MINB) cheby_batch_kernel(const BatchArgs a, const PeerArgs pa) {
    constexpr int L = B / 2;      // lanes per row slot
    constexpr int RPW = 32 / L;   // row slots per warp
    constexpr int V = 32 / L;     // indices per lane per 32-edge chunk
    // U: row gathers in flight per lane
    const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
    const int lane = threadIdx.x & 31;
    const int slot = lane / L, cl = lane % L;
    const unsigned smask = (L == 32) ? 0xffffffffu : (((1u << L) - 1u) << (slot * L));
    const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n_jobs = a.n_hub_items + (a.n_loc - a.hub_rows);
    // Dynamic claiming: a warp claims CLAIM consecutive jobs per atomic and works them RPW
    // at a time.  CLAIM >= 4 rows: at B = 64 one atomic per row lost 25% on config 2
    // (profiles/r01/fused_piece/dyn_jobs_ab.txt).
#ifndef CPG_CLAIM_ROWS
#define CPG_CLAIM_ROWS 4
#endif
    constexpr uint32_t CLAIM = RPW > CPG_CLAIM_ROWS ? RPW : (CPG_CLAIM_ROWS / RPW) * RPW;
    unsigned int* const ctr = a.job_ctr;
    pdl_launch_dependents();
    // registers where they are free: B <= 16, or instances with fewer gathers in flight / CTAs
    constexpr int MM = mass_mode<(B <= 16 || U <= 6 || MINB <= 3) ? 1 : 0>();
    double2 msum;
    batch_mass_init<B, MM>(msum);
    uint32_t claim_end = 0;
    uint32_t base_job = wg * RPW;
    if (ctr) {
        base_job = claim_jobs(ctr, lane, CLAIM);
        claim_end = base_job + CLAIM;
    }
    bool wait_pending = true;
    for (; base_job < n_jobs;) {
        const BatchJob<B> j = batch_job<B>(a, base_job + slot, n_jobs);
        double2 s = {0.0, 0.0};
        uint32_t c[V], cn[V];
        {
            const int m0 = static_cast<int>(j.e0 < j.e1 ? (j.e1 - j.e0 < 32 ? j.e1 - j.e0 : 32) : 0);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int t = v * L + cl;
                cn[v] = t < m0 ? ld_index_b(a.col + j.e0 + t) : 0u;
            }
        }
        if (wait_pending) {  // the previous step's iterate, acc and hub tickets from here on
            pdl_wait();
            wait_pending = false;
        }
        double2 wp = {0.0, 0.0}, ac = {0.0, 0.0};
        if (j.valid && !j.hub) batch_prefetch<B>(a, j.r, cl, wp, ac);
        for (int64_t e = j.e0; __any_sync(0xffffffffu, e < j.e1); e += 32) {
            const int m = static_cast<int>(e < j.e1 ? (j.e1 - e < 32 ? j.e1 - e : 32) : 0);
            // current chunk <- prefetched one; prefetch the next chunk (in flight during the gathers)
            const int64_t en = e + 32;
            const int mn = static_cast<int>(en < j.e1 ? (j.e1 - en < 32 ? j.e1 - en : 32) : 0);
#pragma unroll
            for (int v = 0; v < V; ++v) {
                c[v] = cn[v];
                const int t = v * L + cl;
                cn[v] = t < mn ? ld_index_b(a.col + en + t) : 0u;
            }
#pragma unroll
            for (int t0 = 0; t0 < 32; t0 += U) {
                if (!__any_sync(0xffffffffu, t0 < m)) break;
                double2 val[U];
                if constexpr (MASK) {
                    gather_rows_masked<B, U>(a, c, t0, m, slot, cl, val, pol_last, pol_first);
                } else {
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const int t = t0 + q;
                        const uint32_t u = __shfl_sync(0xffffffffu, c[t / L], slot * L + (t % L));
                        CPG_CHECK(t >= m || u < a.chk_npad, "batch gather", u, a.chk_npad);
                        val[q] = t < m ? (a.hot_rows ? ld_gather2_hot(a.w_cur + static_cast<size_t>(u) * B + 2 * cl,
                                                                      u < a.hot_rows, pol_last, pol_first)
                                                     : ld_gather2(a.w_cur + static_cast<size_t>(u) * B + 2 * cl))
                                       : make_double2(0.0, 0.0);
                    }
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
            {
                CPG_CHECK(!j.hub || j.slot + j.P <= a.chk_parts, "batch hub slot", j.slot + j.P, a.chk_parts);
                reinterpret_cast<double2*>(a.hub_partial + static_cast<size_t>(j.slot + j.piece) * B)[cl] = s;
            }
            __threadfence();
            __syncwarp();
            unsigned prev = 0;
            if (j.hub && cl == 0) prev = atomicAdd(&a.hub_count[j.r], 1u);
            prev = __shfl_sync(0xffffffffu, prev, slot * L);
            if (j.hub && prev == j.P - 1) {
                __threadfence();
                y = sum_partials<B, 1>(a.hub_partial, j.slot, j.P, cl);
                if (cl == 0) a.hub_count[j.r] = 0u;
                batch_prefetch<B>(a, j.r, cl, wp, ac);
                do_epi = true;
            }
        }
        (void)smask;
        if (do_epi) batch_epilogue<B, PEER, MM, MASK>(a, pa, j.r, y, j.d, cl, wp, ac, msum);
        if (!ctr) {
            base_job += nw * RPW;
        } else if (base_job + RPW < claim_end) {
            base_job += RPW;
        } else {
            base_job = claim_jobs(ctr, lane, CLAIM);
            claim_end = base_job + CLAIM;
        }
    }
    if (PEER) __threadfence_system();  // peer stores performed before the iteration barrier
    batch_mass_flush<B, MM>(a, msum);
}

// Plain-row batched step (rows [hub_rows, n_loc) of the chunk; hub pieces run
// in cheby_batch_kernel first).  Without the hub path the kernel fits more
// warps, and the next row's range and first index chunk are prefetched while
// the current row's gathers and epilogue are in flight.
template <int B, int U = 8, int MINB = 4, bool PEER = false, bool MASK = false, bool RP = false>
__global__ void __launch_bounds__(kBatchThreads, MINB) cheby_batch_rows_kernel(const BatchArgs a, const PeerArgs pa) {
    constexpr int L = B / 2;     // lanes per row slot
    constexpr int RPW = 32 / L;  // row slots per warp
    constexpr int V = 32 / L;    // indices per lane per 32-edge chunk
    const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
    // RP instances: one range policy over the iterate instead of a policy choice per row
    const uint64_t pol_range = RP ? policy_range_hot(a.w_cur, static_cast<uint64_t>(a.hot_rows) * B * 8,
                                                     static_cast<uint64_t>(a.n_pad_rows) * B * 8)
                                  : pol_first;
    const int lane = threadIdx.x & 31;
    const int slot = lane / L, cl = lane % L;
    const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t r_end = a.n_loc;
    const uint32_t stride = nw * RPW;
    uint32_t r = a.hub_rows + wg * RPW + slot;
    int64_t e0 = 0, e1 = 0;
    if (r < r_end) {
        e0 = a.rowptr[r];
        e1 = a.rowptr[r + 1];
    }
    uint32_t c[V];
    auto load_chunk = [&](int64_t e, int64_t end) {
        const int m = static_cast<int>(e < end ? (end - e < 32 ? end - e : 32) : 0);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int t = v * L + cl;
            c[v] = t < m ? ld_index_b(a.col + e + t) : 0u;
        }
    };
    load_chunk(e0, e1);
    constexpr int MM = mass_mode<0>();
    double2 msum;
    batch_mass_init<B, MM>(msum);
    while (__any_sync(0xffffffffu, r < r_end)) {
        const uint32_t rn = r + stride;
        int64_t ne0 = 0, ne1 = 0;
        if (rn < r_end) {  // next row's range, in flight during this row
            ne0 = a.rowptr[rn];
            ne1 = a.rowptr[rn + 1];
        }
        double2 wp = {0.0, 0.0}, ac = {0.0, 0.0};
        if (r < r_end) batch_prefetch<B>(a, r, cl, wp, ac);
        double2 s = {0.0, 0.0};
        uint32_t cn[V];
        for (int64_t e = e0; __any_sync(0xffffffffu, e < e1); e += 32) {
            const int m = static_cast<int>(e < e1 ? (e1 - e < 32 ? e1 - e : 32) : 0);
            if (e != e0) {
#pragma unroll
                for (int v = 0; v < V; ++v) c[v] = cn[v];
            }
            if (__any_sync(0xffffffffu, e + 32 < e1)) {  // long row: prefetch the next chunk
                const int64_t en = e + 32;
                const int mn = static_cast<int>(en < e1 ? (e1 - en < 32 ? e1 - en : 32) : 0);
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const int t = v * L + cl;
                    cn[v] = t < mn ? ld_index_b(a.col + en + t) : 0u;
                }
            }
#pragma unroll
            for (int t0 = 0; t0 < 32; t0 += U) {
                if (!__any_sync(0xffffffffu, t0 < m)) break;
                double2 val[U];
                if constexpr (MASK) {
                    gather_rows_masked<B, U>(a, c, t0, m, slot, cl, val, pol_last, pol_first);
                } else {
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        const int t = t0 + q;
                        const uint32_t u = __shfl_sync(0xffffffffu, c[t / L], slot * L + (t % L));
                        CPG_CHECK(t >= m || u < a.chk_npad, "batch gather", u, a.chk_npad);
                        if constexpr (RP) {
                            val[q] = t < m ? ld_gather2_pol(a.w_cur + static_cast<size_t>(u) * B + 2 * cl, pol_range)
                                           : make_double2(0.0, 0.0);
                        } else {
                            val[q] = t < m ? (a.hot_rows ? ld_gather2_hot(a.w_cur + static_cast<size_t>(u) * B + 2 * cl,
                                                                          u < a.hot_rows, pol_last, pol_first)
                                                         : ld_gather2(a.w_cur + static_cast<size_t>(u) * B + 2 * cl))
                                           : make_double2(0.0, 0.0);
                        }
                    }
                }
#pragma unroll
                for (int q = 0; q < U; ++q) {
                    s.x += val[q].x;
                    s.y += val[q].y;
                }
            }
        }
        load_chunk(ne0, ne1);  // next row's first chunk, overlapping this epilogue
        if (r < r_end) batch_epilogue<B, PEER, MM, MASK>(a, pa, r, s, e1 - e0, cl, wp, ac, msum);
        r = rn;
        e0 = ne0;
        e1 = ne1;
    }
    if (PEER) __threadfence_system();  // peer stores performed before the iteration barrier
    batch_mass_flush<B, MM>(a, msum);
}

// Hub-piece batched step (split path): the jobs are the hub pieces of the
// chunk.  The 16-B item carries the piece's first edge and length, so the next
// piece's item and first index chunk are prefetched while the current piece's
// gathers are in flight (as in cheby_batch_rows_kernel); pieces are combined
// by the ordered last-arriver reduction.
// CW instances (column-window piece tables): the pieces are claimed in list
// order from a.job_ctr (RPW per warp per claim, the next claim made while the current
// pieces run), so the pieces in flight are consecutive in the window-major list; an item
// carries its own partial slot and a.hub_meta the row's first slot and piece count; the
// gathers of a warm-window piece are loaded with the normal L2 priority (they are re-read
// by the other rows' pieces of the same window, then age out when the sweep moves on).
template <int B, int U = 8, int MINB = 4, bool PEER = false, bool MASK = false, bool CW = false, bool RP = false>
__global__ void __launch_bounds__(kBatchThreads, MINB) cheby_batch_pieces_kernel(const BatchArgs a, const PeerArgs pa) {
    constexpr int L = B / 2;
    constexpr int RPW = 32 / L;
    constexpr int V = 32 / L;
    constexpr int HB = batch_piece_edges(B);
    const uint64_t pol_last = policy_evict_last(), pol_first = policy_evict_first();
    const uint64_t pol_normal = CW ? policy_evict_normal() : pol_first;
    // RP instances: one range policy over the iterate instead of a policy choice per row
    const uint64_t pol_range = RP ? policy_range_hot(a.w_cur, static_cast<uint64_t>(a.hot_rows) * B * 8,
                                                     static_cast<uint64_t>(a.n_pad_rows) * B * 8)
                                  : pol_first;
    const int lane = threadIdx.x & 31;
    const int slot = lane / L, cl = lane % L;
    const unsigned smask = L == 32 ? 0xffffffffu : (((1u << L) - 1u) << (slot * L));
    const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n_jobs = a.n_hub_items;
    const uint32_t stride = nw * RPW;
    uint32_t job = CW ? claim_jobs(a.job_ctr, lane, RPW) + slot : wg * RPW + slot;
    bool warm = false, nwarm = false;
    auto load_item = [&](uint32_t jb, uint32_t& r, uint32_t& sb, int64_t& e0, int64_t& e1, bool& wm) {
        if (jb < n_jobs) {
            const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.hub_items) + jb);
            const uint64_t c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
            r = raw.x;
            sb = raw.y;
            e0 = code_e0(c);
            e1 = e0 + code_cnt(c);
            wm = CW && (c & kWarmBit) != 0;
        } else {
            r = sb = 0;
            e0 = e1 = 0;
            wm = false;
        }
    };
    uint32_t c[V], cn[V];
    auto load_chunk = [&](uint32_t (&dst)[V], int64_t e, int64_t end) {
        const int m = static_cast<int>(e < end ? (end - e < 32 ? end - e : 32) : 0);
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int t = v * L + cl;
            dst[v] = t < m ? ld_index_b(a.col + e + t) : 0u;
        }
    };
    uint32_t r, sb;
    int64_t e0, e1;
    load_item(job, r, sb, e0, e1, warm);
    load_chunk(c, e0, e1);
    constexpr int MM = mass_mode<0>();
    double2 msum;
    batch_mass_init<B, MM>(msum);
    while (__any_sync(0xffffffffu, job < n_jobs)) {
        uint32_t nr, nsb;
        int64_t ne0, ne1;
        const uint32_t njob = CW ? claim_jobs(a.job_ctr, lane, RPW) + slot : job + stride;
        load_item(njob, nr, nsb, ne0, ne1, nwarm);  // in flight during this piece
        int64_t rs = 0, re = 0;
        uint2 meta = make_uint2(0u, 0u);
        if (job < n_jobs) {
            rs = a.rowptr[r];
            re = a.rowptr[r + 1];
            if (CW) meta = __ldg(a.hub_meta + (r - a.meta_row0));
        }
        const uint64_t pol_cold = warm ? pol_normal : pol_first;
        double2 s = {0.0, 0.0};
        // GM = 0: a policy per gathered row (hot prefix evict_last, the rest pol_cold);
        // 1: plain loads (normal L2 priority: a warp whose pieces are all warm-window pieces);
        // 2: one range policy over the iterate (RP instances).
        auto sweep = [&](auto mode) {
            constexpr int GM = decltype(mode)::value;
            for (int64_t e = e0; __any_sync(0xffffffffu, e < e1); e += 32) {
                const int m = static_cast<int>(e < e1 ? (e1 - e < 32 ? e1 - e : 32) : 0);
                if (e != e0) {
#pragma unroll
                    for (int v = 0; v < V; ++v) c[v] = cn[v];
                }
                if (__any_sync(0xffffffffu, e + 32 < e1)) load_chunk(cn, e + 32, e1);
#pragma unroll
                for (int t0 = 0; t0 < 32; t0 += U) {
                    if (!__any_sync(0xffffffffu, t0 < m)) break;
                    double2 val[U];
                    if constexpr (MASK) {
                        gather_rows_masked<B, U>(a, c, t0, m, slot, cl, val, pol_last, pol_cold);
                    } else {
#pragma unroll
                        for (int q = 0; q < U; ++q) {
                            const int t = t0 + q;
                            const uint32_t u = __shfl_sync(0xffffffffu, c[t / L], slot * L + (t % L));
                            CPG_CHECK(t >= m || u < a.chk_npad, "batch gather", u, a.chk_npad);
                            const double* src = a.w_cur + static_cast<size_t>(u) * B + 2 * cl;
                            if constexpr (GM == 1) {
                                val[q] = t < m ? __ldg(reinterpret_cast<const double2*>(src)) : make_double2(0.0, 0.0);
                            } else if constexpr (GM == 2) {
                                val[q] = t < m ? ld_gather2_pol(src, pol_range) : make_double2(0.0, 0.0);
                            } else {
                                val[q] = t < m ? (a.hot_rows ? ld_gather2_hot(src, u < a.hot_rows, pol_last, pol_cold)
                                                             : ld_gather2(src))
                                               : make_double2(0.0, 0.0);
                            }
                        }
                    }
#pragma unroll
                    for (int q = 0; q < U; ++q) {
                        s.x += val[q].x;
                        s.y += val[q].y;
                    }
                }
            }
        };
        if constexpr (CW) {
            if (__all_sync(0xffffffffu, warm || job >= n_jobs))
                sweep(std::integral_constant<int, 1>{});
            else
                sweep(std::integral_constant<int, RP ? 2 : 0>{});
        } else {
            sweep(std::integral_constant<int, 0>{});
        }
        load_chunk(c, ne0, ne1);  // next piece's first chunk
        const bool live = job < n_jobs;
        const int64_t d = re - rs;
        const uint32_t P = live ? (CW ? meta.y : static_cast<uint32_t>((d + HB - 1) / HB)) : 0u;
        const uint32_t piece = live && !CW ? static_cast<uint32_t>((e0 - rs) / HB) : 0u;  // CW: sb is the piece's own slot
        if (CW) {
            const uint32_t own = sb;
            sb = meta.x;
            CPG_CHECK(!live || (own >= sb && own - sb < P), "column-window piece slot", own, sb);
            if (live) reinterpret_cast<double2*>(a.hub_partial + static_cast<size_t>(own) * B)[cl] = s;
        }
        CPG_CHECK(!live || sb + piece < a.chk_parts, "piece hub slot", sb + piece, a.chk_parts);
        if (live && !CW) reinterpret_cast<double2*>(a.hub_partial + static_cast<size_t>(sb + piece) * B)[cl] = s;
        __threadfence();
        __syncwarp();
        unsigned prev = 0;
        if (live && cl == 0) prev = atomicAdd(&a.hub_count[r], 1u);
        prev = __shfl_sync(0xffffffffu, prev, slot * L);
        if (live && prev == P - 1) {  // last piece of the row: ordered combine + epilogue
            __threadfence();
            const double2 y = sum_partials<B, 8>(a.hub_partial, sb, P, cl);
            if (cl == 0) a.hub_count[r] = 0u;
            double2 wp, ac;
            batch_prefetch<B>(a, r, cl, wp, ac);
            batch_epilogue<B, PEER, MM, MASK>(a, pa, r, y, d, cl, wp, ac, msum);
        }
        (void)smask;
        job = njob;
        r = nr;
        sb = nsb;
        e0 = ne0;
        e1 = ne1;
        warm = nwarm;
    }
    if (PEER) __threadfence_system();  // peer stores performed before the iteration barrier
    batch_mass_flush<B, MM>(a, msum);
}

// ---------------------------------------------------------------------------
// Sparse early steps of the batched step.  In the first steps
// of a one-hot query only a few rows of w_{k-1} are nonzero (the sources, then
// their neighbours); the reference's scatter skips every zero entry
// (graph.cpp:262).  The pull step does the same in two kernels:
//   * scan: a warp per job (a hub piece of the batched table, or a block of 32
//     plain rows) streams the index once, one edge per lane, tests each edge's
//     support bit (bitmap nz_in), and gathers only the rows whose bit is set, in
//     edge order -- so every row / piece sum is the same sequential sum as in
//     the full step, bit for bit (adding an exact zero changes nothing).  Rows
//     with a set edge, and every hub row (through the ordered last-arriver
//     combine of its pieces), get the epilogue here and a `done` bit;
//   * fill: every other row has y = 0: w_{k+1} = -w_{k-1} (first step: 0), acc
//     += c_k w_{k+1}, streamed and coalesced; a row whose w_{k-1} is zero keeps
//     its (zero) iterate and acc, so only the first step (acc starts there) and
//     the last (writes d*acc) store it.
// The per-warp mass rows (C13) are written as in the full step.
// ---------------------------------------------------------------------------
struct SparseExtra {
    uint32_t* done;              // rows finished by the scan kernel (global ids), pre-zeroed
    const uint32_t* fill_mask;   // fill kernel: rows that can change with y = 0 (support of w_{k-1}'s
                                 // predecessor; first step: of w_0); null = every row (last step)
    const uint32_t* coarse;      // coarse support bitmap: bit i = any of rows [i << cshift, (i+1) << cshift)
    uint32_t coarse_words;       // staged in shared memory by the scan kernel
    int cshift;
    uint32_t row_begin;          // first row of the chunk (fill kernel)
    int64_t hb;                  // piece length of the batched table's hub rows
};

// Coarse support bitmap: word i, bit b = OR of the fine bits of rows
// [(32 i + b) << cshift, (32 i + b + 1) << cshift).
__global__ void coarsen_kernel(const uint32_t* fine, uint64_t fine_words, uint32_t* coarse, uint32_t coarse_words,
                               int cshift) {
    const uint32_t per = 1u << (cshift - 5);  // fine words per coarse bit
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < coarse_words; i += gridDim.x * blockDim.x) {
        uint32_t out = 0;
        for (uint32_t b = 0; b < 32; ++b) {
            const uint64_t f0 = (static_cast<uint64_t>(i) * 32 + b) * per;
            uint32_t any = 0;
            for (uint32_t j = 0; j < per && f0 + j < fine_words; ++j) any |= fine[f0 + j];
            out |= (any ? 1u : 0u) << b;
        }
        coarse[i] = out;
    }
}

template <int B>
__device__ __forceinline__ void sparse_finalize(const BatchArgs& a, const SparseExtra& x, uint32_t r, double2 y,
                                                int64_t d, int lane, double2& msum) {
    constexpr int L = B / 2;
    if (lane < L) {
        double2 wp, ac;
        batch_prefetch<B>(a, r, lane, wp, ac);
        batch_epilogue<B, false, 1, true>(a, PeerArgs{}, r, y, d, lane, wp, ac, msum);
    }
    if (lane == 0) nz_set(x.done, a.row0 + r);
}

// Edge scan of [e0, e1): SC chunks of 32 edges per round, their index loads and then
// their support-word loads all in flight together (a round trip per round, not per
// chunk); each set edge, in edge order, goes to visit(edge, source row).
constexpr int kSparseChunks = 8;
template <typename Visit>
__device__ __forceinline__ void sparse_scan_edges(const BatchArgs& a, const uint32_t* cs, int cshift, int64_t e0,
                                                  int64_t e1, int lane, Visit visit) {
    constexpr int SC = kSparseChunks;
    uint32_t un[SC];  // next round's indices: in flight while this round is tested and visited
#pragma unroll
    for (int j = 0; j < SC; ++j) {
        const int64_t ej = e0 + 32 * j + lane;
        un[j] = ej < e1 ? ld_index_b(a.col + ej) : 0u;
    }
    for (int64_t e = e0; e < e1; e += 32 * SC) {
        uint32_t u[SC];
        bool bit[SC];
#pragma unroll
        for (int j = 0; j < SC; ++j) u[j] = un[j];
        if (e + 32 * SC < e1) {
#pragma unroll
            for (int j = 0; j < SC; ++j) {
                const int64_t ej = e + 32 * (SC + j) + lane;
                un[j] = ej < e1 ? ld_index_b(a.col + ej) : 0u;
            }
        }
#pragma unroll
        for (int j = 0; j < SC; ++j) {  // the coarse bit (shared memory) gates the fine test
            const uint32_t c = u[j] >> cshift;
            bit[j] = e + 32 * j + lane < e1 && ((cs[c >> 5] >> (c & 31)) & 1u) && nz_bit(a.nz_in, u[j]);
        }
#pragma unroll
        for (int j = 0; j < SC; ++j) {
            unsigned m = __ballot_sync(0xffffffffu, bit[j]);
            while (m) {
                const int i = __ffs(m) - 1;
                m &= m - 1;
                visit(e + 32 * j + i, __shfl_sync(0xffffffffu, u[j], i));
            }
        }
    }
}

template <int B>
__global__ void __launch_bounds__(kBatchThreads, 4) cheby_sparse_scan_kernel(const BatchArgs a, const SparseExtra x) {
    constexpr int L = B / 2;
    const int lane = threadIdx.x & 31;
    const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    const uint32_t n_plain = a.n_loc - a.hub_rows;
    const uint32_t n_jobs = a.n_hub_items + (n_plain + 31) / 32;
    extern __shared__ uint32_t cs[];  // coarse support bitmap
    for (uint32_t i = threadIdx.x; i < x.coarse_words; i += blockDim.x) cs[i] = x.coarse[i];
    __syncthreads();
    double2 msum = make_double2(0.0, 0.0);
    for (uint32_t job = wg; job < n_jobs; job += nw) {
        if (job < a.n_hub_items) {  // one hub piece: [e0, e1) of row r
            const uint4 raw = __ldg(reinterpret_cast<const uint4*>(a.hub_items) + job);
            const uint32_t r = raw.x;
            const uint64_t c = (static_cast<uint64_t>(raw.w) << 32) | raw.z;
            const int64_t e0 = code_e0(c), e1 = e0 + code_cnt(c);
            const int64_t rs = a.rowptr[r], re = a.rowptr[r + 1], d = re - rs;
            uint32_t P = static_cast<uint32_t>((d + x.hb - 1) / x.hb);
            uint32_t piece = static_cast<uint32_t>((e0 - rs) / x.hb);
            uint32_t sb = raw.y;
            if (a.hub_meta) {  // column-window table: the item holds its own slot
                const uint2 meta = __ldg(a.hub_meta + (r - a.meta_row0));
                P = meta.y;
                piece = raw.y - meta.x;
                sb = meta.x;
            }
            double2 s = make_double2(0.0, 0.0);
            sparse_scan_edges(a, cs, x.cshift, e0, e1, lane, [&](int64_t, uint32_t v) {
                if (lane < L) {
                    const double2 g = ld_gather2(a.w_cur + static_cast<size_t>(v) * B + 2 * lane);
                    s.x += g.x;
                    s.y += g.y;
                }
            });
            if (P == 1) {
                sparse_finalize<B>(a, x, r, s, d, lane, msum);
                continue;
            }
            CPG_CHECK(sb + piece < a.chk_parts, "sparse hub slot", sb + piece, a.chk_parts);
            if (lane < L) reinterpret_cast<double2*>(a.hub_partial + static_cast<size_t>(sb + piece) * B)[lane] = s;
            __threadfence();
            __syncwarp();
            unsigned prev = 0;
            if (lane == 0) prev = atomicAdd(&a.hub_count[r], 1u);
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if (prev == P - 1) {  // last piece: ordered combine, as sum_partials in the full step
                __threadfence();
                double2 y = make_double2(0.0, 0.0);
                if (lane < L) y = sum_partials<B, 8>(a.hub_partial, sb, P, lane);
                if (lane == 0) a.hub_count[r] = 0u;
                sparse_finalize<B>(a, x, r, y, d, lane, msum);
            }
        } else {  // 32 plain rows [r0, r0 + nr)
            const uint32_t r0 = a.hub_rows + (job - a.n_hub_items) * 32;
            const uint32_t nr = min(32u, a.n_loc - r0);
            const int64_t rp = lane < static_cast<int>(nr) ? a.rowptr[r0 + lane] : INT64_MAX;
            const int64_t E0 = __shfl_sync(0xffffffffu, rp, 0);
            const int64_t E1 = a.rowptr[r0 + nr];
            int cur = -1;
            double2 s = make_double2(0.0, 0.0);
            sparse_scan_edges(a, cs, x.cshift, E0, E1, lane, [&](int64_t ee, uint32_t v) {
                const int rr = __popc(__ballot_sync(0xffffffffu, rp <= ee)) - 1;  // row of edge ee
                if (rr != cur) {
                    if (cur >= 0) {
                        const int64_t b0 = __shfl_sync(0xffffffffu, rp, cur);
                        const int64_t b1 = cur + 1 < static_cast<int>(nr) ? __shfl_sync(0xffffffffu, rp, cur + 1) : E1;
                        sparse_finalize<B>(a, x, r0 + cur, s, b1 - b0, lane, msum);
                    }
                    cur = rr;
                    s = make_double2(0.0, 0.0);
                }
                if (lane < L) {
                    const double2 g = ld_gather2(a.w_cur + static_cast<size_t>(v) * B + 2 * lane);
                    s.x += g.x;
                    s.y += g.y;
                }
            });
            if (cur >= 0) {
                const int64_t b0 = __shfl_sync(0xffffffffu, rp, cur);
                const int64_t b1 = cur + 1 < static_cast<int>(nr) ? __shfl_sync(0xffffffffu, rp, cur + 1) : E1;
                sparse_finalize<B>(a, x, r0 + cur, s, b1 - b0, lane, msum);
            }
        }
    }
    batch_mass_flush<B, 1>(a, msum);
}

template <int B>
__global__ void __launch_bounds__(kBatchThreads, 4) cheby_sparse_fill_kernel(const BatchArgs a, const SparseExtra x) {
    constexpr int L = B / 2;
    constexpr int RPW = 32 / L;
    const int lane = threadIdx.x & 31;
    const int slot = lane / L, cl = lane % L;
    const uint32_t wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    double2 msum = make_double2(0.0, 0.0);
    if (x.fill_mask) {
        // Few rows to fill (the support of an early iterate): a lane tests 32 rows with one
        // word of each bitmap, the warp skips 1024 rows per round, and the slots share the
        // set bits of a live word, RPW at a time.
        const uint64_t g0 = static_cast<uint64_t>(a.row0) + x.row_begin, g1 = static_cast<uint64_t>(a.row0) + a.n_loc;
        const uint32_t w0 = static_cast<uint32_t>(g0 >> 5), w1 = static_cast<uint32_t>((g1 + 31) >> 5);
        for (uint64_t wb = static_cast<uint64_t>(w0) + static_cast<uint64_t>(wg) * 32; wb < w1;
             wb += static_cast<uint64_t>(nw) * 32) {
            const uint64_t wi = wb + lane;
            uint32_t live = 0;
            if (wi < w1) {
                live = __ldg(x.fill_mask + wi) & ~x.done[wi];
                const uint64_t b0 = wi * 32;
                if (b0 < g0) live &= ~0u << (g0 - b0);
                if (b0 + 32 > g1) live &= (1u << (g1 - b0)) - 1u;
            }
            unsigned any = __ballot_sync(0xffffffffu, live != 0u);
            while (any) {
                const int src = __ffs(any) - 1;
                any &= any - 1;
                uint32_t word = __shfl_sync(0xffffffffu, live, src);
                const uint64_t base = (wb + src) * 32;
                while (word) {
                    uint32_t mine = word;
                    for (int s = 0; s < slot; ++s) mine &= mine - 1;  // slot s takes the s-th set bit
                    if (mine) {
                        const uint32_t gr = static_cast<uint32_t>(base) + static_cast<uint32_t>(__ffs(mine) - 1);
                        const uint32_t r = gr - a.row0;
                        const int64_t d = a.rowptr[r + 1] - a.rowptr[r];
                        const double2 wp = a.first ? reinterpret_cast<const double2*>(a.w_cur + static_cast<size_t>(gr) * B)[cl]
                                                   : ld_stream2(a.w_io + static_cast<size_t>(gr) * B + 2 * cl);
                        // w_{k-1} = 0 and y = 0: w_{k+1} = 0 is already stored and acc += 0 keeps acc
                        if (a.first || a.last || wp.x != 0.0 || wp.y != 0.0) {
                            const double2 ac = a.first ? make_double2(0.0, 0.0)
                                                       : ld_stream2(a.acc + static_cast<size_t>(r) * B + 2 * cl);
                            batch_epilogue<B, false, 1, true>(a, PeerArgs{}, r, make_double2(0.0, 0.0), d, cl, wp, ac, msum);
                        }
                    }
                    for (int s = 0; s < RPW && word; ++s) word &= word - 1;
                }
            }
        }
        batch_mass_flush<B, 1>(a, msum);
        return;
    }
    constexpr int FU = 4;  // rows per lane per round: their loads in flight together
    const uint32_t stride = nw * RPW;
    for (uint32_t rb = x.row_begin + wg * RPW + slot; rb < a.n_loc; rb += FU * stride) {
        bool live[FU];
        int64_t d[FU];
        double2 wp[FU];
#pragma unroll
        for (int f = 0; f < FU; ++f) {
            const uint32_t r = rb + f * stride;
            live[f] = r < a.n_loc && !nz_bit(x.done, a.row0 + r) && (!x.fill_mask || nz_bit(x.fill_mask, a.row0 + r));
            d[f] = 0;
            wp[f] = make_double2(0.0, 0.0);
            if (live[f]) {
                const uint32_t gr = a.row0 + r;
                d[f] = a.rowptr[r + 1] - a.rowptr[r];
                wp[f] = a.first ? reinterpret_cast<const double2*>(a.w_cur + static_cast<size_t>(gr) * B)[cl]
                                : ld_stream2(a.w_io + static_cast<size_t>(gr) * B + 2 * cl);
            }
        }
#pragma unroll
        for (int f = 0; f < FU; ++f) {
            const uint32_t r = rb + f * stride;
            // w_{k-1} = 0 and y = 0: w_{k+1} = 0 is already stored and acc += 0 keeps acc
            if (!live[f] || (!a.first && !a.last && wp[f].x == 0.0 && wp[f].y == 0.0)) continue;
            const double2 ac = a.first ? make_double2(0.0, 0.0) : ld_stream2(a.acc + static_cast<size_t>(r) * B + 2 * cl);
            batch_epilogue<B, false, 1, true>(a, PeerArgs{}, r, make_double2(0.0, 0.0), d[f], cl, wp[f], ac, msum);
        }
    }
    batch_mass_flush<B, 1>(a, msum);
}

// First step of a one-hot batched query by push (unsharded graphs).  Column q of
// w_0 has one nonzero, at s_q, and rows never list themselves, so
//   w_1(v, q) = w_0(s_q, q) / d_v   for v in N(s_q)      (a one-term sum: exact)
//   acc(v, q) = c_1 w_1(v, q)  ( = c_0 * 0 + c_1 w_1 ),   acc(s_q, q) = c_0 w_0(s_q, q)
// and every other entry of w_1 and acc is zero (pre-zeroed by the caller).  This
// is the full step's result bit for bit.  CTA b takes pieces b, b + G, ... of
// every column's adjacency list, so each CTA's per-column mass partial (one row of
// B doubles, mass_partial + b * warps * B) has a fixed order.
constexpr int kPushThreads = 256;
constexpr int kPushPer = 8;  // edges per thread per piece
__global__ void __launch_bounds__(kPushThreads) cheby_first_push_kernel(const BatchArgs a, const uint32_t* gdeg,
                                                                        const uint32_t* new_of_old,
                                                                        const uint32_t* sources, uint32_t q0,
                                                                        uint32_t count, uint32_t B) {
    __shared__ double red[kPushThreads / 32];
    __shared__ double mrow[kBatchCols];
    constexpr int64_t PIECE = static_cast<int64_t>(kPushThreads) * kPushPer;
    for (uint32_t q = threadIdx.x; q < B; q += blockDim.x) mrow[q] = 0.0;
    __syncthreads();
    const double c1 = a.coeffs[1];
    for (uint32_t q = 0; q < count; ++q) {
        const uint32_t s = new_of_old[sources[q0 + q]];
        const int64_t rs = a.rowptr[s], re = a.rowptr[s + 1];
        const double w0 = a.w_cur[static_cast<size_t>(s) * B + q];
        const int64_t P = (re - rs + PIECE - 1) / PIECE;
        if (blockIdx.x == 0 && threadIdx.x == 0)  // the source's own row: w_1 = 0 there, acc = c_0 w_0
            a.acc[static_cast<size_t>(s) * B + q] = re > rs ? a.coeffs[0] * w0 : 0.0;
        for (int64_t p = blockIdx.x; p < P; p += gridDim.x) {
            double m = 0.0;
#pragma unroll
            for (int i = 0; i < kPushPer; ++i) {
                const int64_t e = rs + p * PIECE + i * kPushThreads + threadIdx.x;
                if (e < re) {
                    const uint32_t v = a.col[e];
                    const double dd = static_cast<double>(gdeg[v]);
                    const double w1 = w0 / dd;
                    a.w_io[static_cast<size_t>(v) * B + q] = w1;
                    a.acc[static_cast<size_t>(v) * B + q] = c1 * w1;
                    if (a.nz_out) nz_set(a.nz_out, v);
                    m += dd * w1;
                }
            }
            m = block_sum<kPushThreads>(m, red);
            if (threadIdx.x == 0) mrow[q] += m;
        }
    }
    __syncthreads();
    if (a.mass_partial)
        for (uint32_t q = threadIdx.x; q < B; q += blockDim.x)
            a.mass_partial[static_cast<size_t>(blockIdx.x) * (kBatchThreads / 32) * B + q] = mrow[q];
}

// ---------------------------------------------------------------------------
// Small kernels around the steps.
// ---------------------------------------------------------------------------

// w_0 = D^-1 e_s in the global (relabelled) ids; vector pre-zeroed.
// Query group: thread t seeds slice t (w + t*stride) for source q0 + t.
// nz0 (optional, pre-zeroed): support bitmap of w_0 (the union over the group).
__global__ void init_onehot_kernel(double* w, uint64_t stride, const uint32_t* gdeg, const uint32_t* new_of_old,
                                   const uint32_t* sources, uint32_t q0, uint32_t count, uint32_t* nz0) {
    const uint32_t t = threadIdx.x;
    if (t >= count) return;
    const uint32_t s = new_of_old[sources[q0 + t]];
    w[t * stride + s] = 1.0 / static_cast<double>(gdeg[s]);
    if (nz0) nz_set(nz0, s);
}

// Batched: column j of W_0 = D^-1 e_{s_j}; matrix [n_pad][B] pre-zeroed.
__global__ void init_onehot_batch_kernel(double* W, const uint32_t* gdeg, const uint32_t* new_of_old,
                                         const uint32_t* sources, uint32_t q0, uint32_t count, uint32_t B,
                                         uint32_t* nz0) {
    const uint32_t j = threadIdx.x;
    if (j < count) {
        const uint32_t s = new_of_old[sources[q0 + j]];
        W[static_cast<size_t>(s) * B + j] = 1.0 / static_cast<double>(gdeg[s]);
        if (nz0) nz_set(nz0, s);
    }
}

// w_0 = D^-1 (D^a seed) for a dense seed given in caller ids (a = 0: plain
// cheby_power_vec; a != 0: general_gp_vector's D^a scaling, solvers.cpp:396-397).
__global__ void init_dense_kernel(double* w, const uint32_t* gdeg, const uint32_t* new_of_old,
                                  const double* seed, uint32_t n, double a) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t s = new_of_old[v];
        const double d = static_cast<double>(gdeg[s]);
        const double x = a == 0.0 ? seed[v] : pow(d, a) * seed[v];
        w[s] = x / d;
    }
}

// Batched dense seeds: column j of W_0 ([n_pad][B]) = D^-1 D^a X[j] (X is count x n).
__global__ void init_dense_batch_kernel(double* W, const uint32_t* gdeg, const uint32_t* new_of_old,
                                        const double* X, uint32_t n, uint32_t count, uint32_t B, double a) {
    const uint64_t total = static_cast<uint64_t>(n) * count;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t j = static_cast<uint32_t>(i / n), v = static_cast<uint32_t>(i % n);
        const uint32_t s = new_of_old[v];
        const double d = static_cast<double>(gdeg[s]);
        const double x = a == 0.0 ? X[i] : pow(d, a) * X[i];
        W[static_cast<size_t>(s) * B + j] = x / d;
    }
}

// out[v] = d_v^-a full[new_of_old[v]]  (back to the caller's ids; a != 0 only
// for general_gp_vector, solvers.cpp:400-401).
// out[q][v] = full[q*stride + new_of_old[v]] for the count queries of a group.
__global__ void unpermute_kernel(double* out, const double* full, uint64_t stride, const uint32_t* new_of_old,
                                 uint32_t n, uint32_t count, const uint32_t* gdeg, double a) {
    const uint64_t total = static_cast<uint64_t>(n) * count;
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const uint32_t q = static_cast<uint32_t>(i / n), v = static_cast<uint32_t>(i - static_cast<uint64_t>(q) * n);
        const uint32_t s = new_of_old[v];
        const double y = full[q * stride + s];
        out[i] = a == 0.0 ? y : pow(static_cast<double>(gdeg[s]), -a) * y;
    }
}

// Batched: out[j][v] = full[new_of_old[v]][j] for j < count (full is [n_pad][B]).
// One thread per caller id v: it reads its relabelled row once (B*8 contiguous
// bytes, double2 loads) and writes one value per query; the writes of a warp
// are coalesced for every j.
__global__ void unpermute_batch_kernel(double* out, const double* full, const uint32_t* new_of_old,
                                       uint32_t n, uint32_t count, uint32_t B, const uint32_t* gdeg, double a) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t s = new_of_old[v];
        const double scale = a == 0.0 ? 1.0 : pow(static_cast<double>(gdeg[s]), -a);
        const double2* row = reinterpret_cast<const double2*>(full + static_cast<size_t>(s) * B);
        for (uint32_t j = 0; j < count; j += 2) {
            const double2 y = __ldg(row + j / 2);
            out[static_cast<size_t>(j) * n + v] = a == 0.0 ? y.x : scale * y.x;
            if (j + 1 < count) out[static_cast<size_t>(j + 1) * n + v] = a == 0.0 ? y.y : scale * y.y;
        }
    }
}

// steps[k] = sum_b mass_partial[k][b]  (ordered, one CTA per step).
// (query group: blockIdx.y = q, partials at q*q_stride, steps at q*K)
__global__ void mass_steps_kernel(const double* mass_partial, uint32_t n_part, uint64_t q_stride, double* steps,
                                  uint32_t K) {
    __shared__ double red[kStepThreads / 32];
    const uint32_t k = blockIdx.x, q = blockIdx.y;
    const double* mp = mass_partial + q * q_stride;
    double s = 0.0;
    for (uint32_t b = threadIdx.x; b < n_part; b += blockDim.x) s += mp[static_cast<size_t>(k) * n_part + b];
    s = block_sum<kStepThreads>(s, red);
    if (threadIdx.x == 0) steps[static_cast<size_t>(q) * K + k] = s;
}

// err = max(err, max_k |steps[k] - mass0|).
__global__ void mass_err_kernel(const double* steps, uint32_t K, double mass0, double* err) {
    double worst = *err;
    for (uint32_t k = 0; k < K; ++k) worst = fmax(worst, fabs(steps[k] - mass0));
    *err = worst;
}  // (over all K*count entries of a query group: called with K*count)

// Batched: steps[j*K + k] = sum_{i < used} mp[(k*stride + i)*B + j] for the
// count live columns (i over the step's warp rows in launch order; one CTA
// per (k, j); fixed order).
__global__ void mass_steps_batch_kernel(const double* mp, uint32_t stride, uint32_t used, uint32_t B, uint32_t K,
                                        double* steps) {
    __shared__ double red[kStepThreads / 32];
    const uint32_t k = blockIdx.x, j = blockIdx.y;
    double s = 0.0;
    for (uint32_t i = threadIdx.x; i < used; i += blockDim.x)
        s += mp[(static_cast<size_t>(k) * stride + i) * B + j];
    s = block_sum<kStepThreads>(s, red);
    if (threadIdx.x == 0) steps[static_cast<size_t>(j) * K + k] = s;
}

// err = max(err, max_{j,k} |steps[j*K + k] - mass0[j]|) (mass0 null: 1 for every column).
__global__ void mass_err_cols_kernel(const double* steps, uint32_t K, uint32_t count, const double* mass0,
                                     double* err) {
    double worst = *err;
    for (uint32_t j = 0; j < count; ++j) {
        const double m0 = mass0 ? mass0[j] : 1.0;
        for (uint32_t k = 0; k < K; ++k) worst = fmax(worst, fabs(steps[static_cast<size_t>(j) * K + k] - m0));
    }
    *err = worst;
}

// Host-side launch wrappers ---------------------------------------------------
// Step kernels go out with programmatic stream serialization (PDL, see
// pdl_wait); CPG_PDL=0 launches them plainly (A/B hook; same results).
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("CPG_PDL");
        return !e || e[0] != '0';
    }();
    return on;
}

// pdl: the caller's promise that the previous operation in `st` is the previous
// step's kernel (no event record / wait or collective in between: those are not
// ordered by griddepcontrol.wait, and a sharded run with them lost parity).
template <typename... KArgs, typename... Args>
void launch_pdl(bool pdl, void (*kern)(KArgs...), int grid, int block, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(block));
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl && pdl_enabled() ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, args...);
}

void launch_step(const StepArgs& a, int grid, cudaStream_t st, const StepGroup* gq, bool pdl) {
    const bool group = gq && gq->nq > 1;
    if (a.nz_in && !group) {  // masked (sparse early) step
        if (a.tile == kTileMid)
            launch_pdl(pdl, cheby_step_kernel<kStepThreads, kTileMid, true>, grid, kStepThreads, st, a);
        else if (a.tile == kTileLarge)
            launch_pdl(pdl, cheby_step_kernel<kStepThreads, kTileLarge, true>, grid, kStepThreads, st, a);
        else
            launch_pdl(pdl, cheby_step_kernel<kStepThreads, kTileSmall, true>, grid, kStepThreads, st, a);
        return;
    }
    // query groups launch plainly: PDL measured 3% slower on config 1 (profiles/r02/pdl_ab.txt)
    if (a.tile == kTileMid) {
        if (group)
            launch_pdl(false, cheby_step_group_kernel<kStepThreads, kTileMid>, grid, kStepThreads, st, a, *gq);
        else
            launch_pdl(pdl, cheby_step_kernel<kStepThreads, kTileMid>, grid, kStepThreads, st, a);
    } else if (a.tile == kTileLarge) {
        if (group)
            launch_pdl(false, cheby_step_group_kernel<kStepThreads, kTileLarge>, grid, kStepThreads, st, a, *gq);
        else
            launch_pdl(pdl, cheby_step_kernel<kStepThreads, kTileLarge>, grid, kStepThreads, st, a);
    } else {
        if (group)
            launch_pdl(false, cheby_step_group_kernel<kStepThreads, kTileSmall>, grid, kStepThreads, st, a, *gq);
        else
            launch_pdl(pdl, cheby_step_kernel<kStepThreads, kTileSmall>, grid, kStepThreads, st, a);
    }
}
// Split step: tile kernel instance for a tile width (MINB CTAs per SM).
#define CPG_TILES_SWITCH(X)                                  \
    switch (tile) {                                          \
    case kTileSmall: X(kTileSmall, 8); break;                \
    case kTileMid: X(kTileMid, 6); break;                    \
    default: X(kTileLarge, 5); break;                        \
    }
void launch_step_hubs(const StepArgs& a, int grid, cudaStream_t st, bool) {
    // the split step launches plainly: no PDL gain at its 20 ms steps, and the
    // post-wait L1 invalidation cost 3% (profiles/r02/ab_fence.txt)
    if (a.nz_in)
        launch_pdl(false, cheby_step_hubs_kernel<kStepThreads, true>, grid, kStepThreads, st, a);
    else
        launch_pdl(false, cheby_step_hubs_kernel<kStepThreads>, grid, kStepThreads, st, a);
}
void launch_step_tiles(const StepArgs& a, int tile, int grid, cudaStream_t st, bool) {
    if (a.nz_in) {
#define CPG_L(T, M) launch_pdl(false, cheby_step_tiles_kernel<kStepThreads, T, M, true>, grid, kStepThreads, st, a)
        CPG_TILES_SWITCH(CPG_L)
#undef CPG_L
        return;
    }
#define CPG_L(T, M) launch_pdl(false, cheby_step_tiles_kernel<kStepThreads, T, M>, grid, kStepThreads, st, a)
    CPG_TILES_SWITCH(CPG_L)
#undef CPG_L
}
constexpr int kWarpKernelWarps = 8;
void launch_step_warp(const StepArgs& a, unsigned int* ctr, int grid, cudaStream_t st) {
    cheby_step_warp_kernel<kWarpKernelWarps><<<grid, kWarpKernelWarps * 32, 0, st>>>(a, ctr);
}
int step_warp_occupancy() {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_warp_kernel<kWarpKernelWarps>,
                                                  kWarpKernelWarps * 32, 0);
    return blocks;
}
int step_tiles_occupancy(int tile) {
    int blocks = 0;
#define CPG_O(T, M) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_tiles_kernel<kStepThreads, T, M>, kStepThreads, 0)
    CPG_TILES_SWITCH(CPG_O)
#undef CPG_O
    return blocks;
}
int step_hubs_occupancy() {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_hubs_kernel<kStepThreads>, kStepThreads, 0);
    return blocks;
}

int step_occupancy(int tile) {  // same for both instances (64 registers, same shared memory)
    int blocks = 0;
    if (tile == kTileMid)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_group_kernel<kStepThreads, kTileMid>,
                                                      kStepThreads, 0);
    else if (tile == kTileLarge)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_group_kernel<kStepThreads, kTileLarge>,
                                                      kStepThreads, 0);
    else
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_step_group_kernel<kStepThreads, kTileSmall>,
                                                      kStepThreads, 0);
    return blocks;
}
template <int B, int U, int MINB>
int launch_slot(const BatchArgs& a, cudaStream_t st) {
    int occ = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, cheby_batch_kernel<B, U, MINB>, kBatchThreads, 0);
    const int grid = std::max(1, std::min(occ, kBatchMaxCtasPerSm)) * sms;
    cheby_batch_kernel<B, U, MINB><<<grid, kBatchThreads, 0, st>>>(a, PeerArgs{});
    return grid;
}

template <int B>
int launch_slot_b(const BatchArgs& a, int cfg, cudaStream_t st) {
    switch (cfg) {
    case 41: return launch_slot<B, 4, 4>(a, st);
    case 45: return launch_slot<B, 4, 5>(a, st);
    case 46: return launch_slot<B, 4, 6>(a, st);
    case 64: return launch_slot<B, 6, 4>(a, st);
    case 44: return launch_slot<B, 4, 4>(a, st);
    case 83: return launch_slot<B, 8, 3>(a, st);
    case 63: return launch_slot<B, 6, 3>(a, st);
    case 84: return launch_slot<B, 8, 4>(a, st);
    case 85: return launch_slot<B, 8, 5>(a, st);
    default: return 0;
    }
}

int launch_slot_cfg(const BatchArgs& a, int B, int cfg, cudaStream_t st) {
    switch (B) {
    case 16: return launch_slot_b<16>(a, cfg, st);
    case 32: return launch_slot_b<32>(a, cfg, st);
    case 64: return launch_slot_b<64>(a, cfg, st);
    default: return 0;
    }
}

// PEER instances (fused all-gather), default geometry.
#define CPG_PEER_SWITCH(KERNEL, B, grid, st, a, pa)                                                        \
    switch (B) {                                                                                            \
    case 4: KERNEL<4, 8, 4, true><<<grid, kBatchThreads, 0, st>>>(a, pa); break;                            \
    case 8: KERNEL<8, 8, 4, true><<<grid, kBatchThreads, 0, st>>>(a, pa); break;                            \
    case 16: KERNEL<16, 8, 4, true><<<grid, kBatchThreads, 0, st>>>(a, pa); break;                          \
    case 32: KERNEL<32, 8, 4, true><<<grid, kBatchThreads, 0, st>>>(a, pa); break;                          \
    default: KERNEL<64, 8, 4, true><<<grid, kBatchThreads, 0, st>>>(a, pa); break;                          \
    }

int launch_batch(const BatchArgs& a, int B, int grid, cudaStream_t st, const PeerArgs* pa, bool pdl) {
    if (pa) {
        CPG_PEER_SWITCH(cheby_batch_kernel, B, grid, st, a, *pa);
        return grid;
    }
    if (a.nz_in) {  // masked (sparse early) step: the default geometry of each width
        switch (B) {
        case 4: launch_pdl(pdl, cheby_batch_kernel<4, 8, 4, false, true>, grid, kBatchThreads, st, a, PeerArgs{}); break;
        case 8: launch_pdl(pdl, cheby_batch_kernel<8, 8, 4, false, true>, grid, kBatchThreads, st, a, PeerArgs{}); break;
        case 16: launch_pdl(pdl, cheby_batch_kernel<16, 8, 4, false, true>, grid, kBatchThreads, st, a, PeerArgs{}); break;
        case 32: launch_pdl(pdl, cheby_batch_kernel<32, 4, 4, false, true>, grid, kBatchThreads, st, a, PeerArgs{}); break;
        default: launch_pdl(pdl, cheby_batch_kernel<64, 4, 4, false, true>, grid, kBatchThreads, st, a, PeerArgs{}); break;
        }
        return grid;
    }
    static const int cfg = [] {  // tuning hook: CPG_SLOT_CFG = U*10 + MINB
        const char* e = std::getenv("CPG_SLOT_CFG");
        return e ? std::atoi(e) : 0;
    }();
    if (cfg)
        if (const int g = launch_slot_cfg(a, B, cfg, st)) return g;
    switch (B) {
    case 4: launch_pdl(pdl, cheby_batch_kernel<4>, grid, kBatchThreads, st, a, PeerArgs{}); break;
    case 8: launch_pdl(pdl, cheby_batch_kernel<8>, grid, kBatchThreads, st, a, PeerArgs{}); break;
    case 16: launch_pdl(pdl, cheby_batch_kernel<16>, grid, kBatchThreads, st, a, PeerArgs{}); break;
    // B >= 32: 4 row gathers in flight per lane (the rows are 256-512 B; with the mass
    // check in registers this beat U = 8 by 6% on config 2, profiles/r02/ab_slot64.txt)
    case 32: launch_pdl(pdl, cheby_batch_kernel<32, 4>, grid, kBatchThreads, st, a, PeerArgs{}); break;
    default: launch_pdl(pdl, cheby_batch_kernel<64, 4>, grid, kBatchThreads, st, a, PeerArgs{}); break;
    }
    return grid;
}
// Split path: hub pieces through cheby_batch_kernel, then plain rows through
// cheby_batch_rows_kernel.  Faster on every graph with >= 8M local edges
// (profiles/r01/batch_split_ab.txt); tiny graphs keep the single fused launch.
// CPG_BATCH_SPLIT=0/1 forces either.
bool batch_split(uint64_t nnz_loc) {
    const char* e = std::getenv("CPG_BATCH_SPLIT");  // read per call: tests force either path
    if (e) return e[0] != '0';
    return nnz_loc >= (8ull << 20);
}

// Launch a persistent batched kernel instance with its grid capped at its own
// occupancy x SMs (callers size `grid` for the default 4 CTAs/SM).
template <typename Kern>
int launch_capped(Kern kernel, const BatchArgs& a, int grid, cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int occ = 0;  // per kernel instance; the same on every B200
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kBatchThreads, 0);
    const int g = std::max(1, std::min(grid, std::max(1, std::min(occ, kBatchMaxCtasPerSm)) * sms));
    kernel<<<g, kBatchThreads, 0, st>>>(a, PeerArgs{});
    return g;
}

// Geometry of the split kernels (U row gathers in flight per lane, MINB CTAs
// per SM).  B = 16 runs U = 8 at 3 CTAs/SM (80 registers, no spills; config 5:
// 887 -> 911-916 GTEPS); B = 64 keeps 4 CTAs/SM (3 lost 6-9% on configs 3-4;
// profiles/r01/split_occupancy/).  CPG_PIECES_CFG / CPG_ROWS_CFG = U*10 + MINB
// select other instances.
int split_cfg(const char* env, int B) {
    if (const char* e = std::getenv(env)) return std::atoi(e);
    return B == 16 ? 83 : 84;
}

#define CPG_SPLIT_CFG_SWITCH(KERNEL, B)                                                             \
    switch (cfg) {                                                                                  \
    case 83: return launch_capped(KERNEL<B, 8, 3>, a, grid, st);                                    \
    case 63: return launch_capped(KERNEL<B, 6, 3>, a, grid, st);                                    \
    case 162: return launch_capped(KERNEL<B, 16, 2>, a, grid, st);                                  \
    default: return launch_capped(KERNEL<B, 8, 4>, a, grid, st);                                    \
    }

// Masked (sparse early) instances of the split kernels, at the default geometry of each width.
#define CPG_MASK_SWITCH(KERNEL, B)                                                                   \
    switch (B) {                                                                                    \
    case 4: return launch_capped(KERNEL<4, 8, 4, false, true>, a, grid, st);                        \
    case 8: return launch_capped(KERNEL<8, 8, 4, false, true>, a, grid, st);                        \
    case 16: return launch_capped(KERNEL<16, 8, 3, false, true>, a, grid, st);                      \
    case 32: return launch_capped(KERNEL<32, 8, 4, false, true>, a, grid, st);                      \
    default: return launch_capped(KERNEL<64, 8, 4, false, true>, a, grid, st);                      \
    }

int launch_batch_pieces(const BatchArgs& a, int B, int grid, cudaStream_t st, const PeerArgs* pa) {
    if (a.hub_meta) {  // column-window piece table (built for B = 16 and 64, one GPU, unmasked)
        if (pa || a.nz_in || !a.job_ctr || (B != 16 && B != 64)) return -1;  // api.cu never builds such a launch
        static const int cw16 = split_cfg("CPG_CW_CFG", 16);
        if (B == 16) {
            switch (cw16) {
            case 84: return launch_capped(cheby_batch_pieces_kernel<16, 8, 4, false, false, true>, a, grid, st);
            case 85: return launch_capped(cheby_batch_pieces_kernel<16, 8, 5, false, false, true>, a, grid, st);
            case 162: return launch_capped(cheby_batch_pieces_kernel<16, 16, 2, false, false, true>, a, grid, st);
            case 163: return launch_capped(cheby_batch_pieces_kernel<16, 16, 3, false, false, true>, a, grid, st);
            case 44: return launch_capped(cheby_batch_pieces_kernel<16, 4, 4, false, false, true>, a, grid, st);
            case 46: return launch_capped(cheby_batch_pieces_kernel<16, 4, 6, false, false, true>, a, grid, st);
            case 830: return launch_capped(cheby_batch_pieces_kernel<16, 8, 3, false, false, true>, a, grid, st);
            case 841: return launch_capped(cheby_batch_pieces_kernel<16, 8, 4, false, false, true, true>, a, grid, st);
            case 1631: return launch_capped(cheby_batch_pieces_kernel<16, 16, 3, false, false, true, true>, a, grid, st);
            case 1031: return launch_capped(cheby_batch_pieces_kernel<16, 10, 3, false, false, true, true>, a, grid, st);
            case 1041: return launch_capped(cheby_batch_pieces_kernel<16, 10, 4, false, false, true, true>, a, grid, st);
            case 831: return launch_capped(cheby_batch_pieces_kernel<16, 8, 3, false, false, true, true>, a, grid, st);
            // 12 gathers in flight per lane at 3 CTAs/SM (80 registers, no spills): 21.0 ms against 21.9 at 8
            default: return launch_capped(cheby_batch_pieces_kernel<16, 12, 3, false, false, true, true>, a, grid, st);
            }
        }
        if (cw16 == 830) return launch_capped(cheby_batch_pieces_kernel<64, 8, 4, false, false, true>, a, grid, st);
        static const int cw64 = [] {  // A/B: geometry of the B = 64 range-policy instance
            const char* e = std::getenv("CPG_CW_CFG64");
            return e ? std::atoi(e) : 84;
        }();
        if (cw64 == 124) return launch_capped(cheby_batch_pieces_kernel<64, 12, 4, false, false, true, true>, a, grid, st);
        if (cw64 == 123) return launch_capped(cheby_batch_pieces_kernel<64, 12, 3, false, false, true, true>, a, grid, st);
        if (cw64 == 163) return launch_capped(cheby_batch_pieces_kernel<64, 16, 3, false, false, true, true>, a, grid, st);
        if (cw64 == 85) return launch_capped(cheby_batch_pieces_kernel<64, 8, 5, false, false, true, true>, a, grid, st);
        return launch_capped(cheby_batch_pieces_kernel<64, 8, 4, false, false, true, true>, a, grid, st);
    }
    if (pa) {
        CPG_PEER_SWITCH(cheby_batch_pieces_kernel, B, grid, st, a, *pa);
        return grid;
    }
    if (a.nz_in) CPG_MASK_SWITCH(cheby_batch_pieces_kernel, B)
    static const int cfg16 = split_cfg("CPG_PIECES_CFG", 16), cfg64 = split_cfg("CPG_PIECES_CFG", 64);
    if (B == 16) {
        const int cfg = cfg16;
        CPG_SPLIT_CFG_SWITCH(cheby_batch_pieces_kernel, 16)
    }
    if (B == 64) {
        const int cfg = cfg64;
        CPG_SPLIT_CFG_SWITCH(cheby_batch_pieces_kernel, 64)
    }
    switch (B) {
    case 4: cheby_batch_pieces_kernel<4><<<grid, kBatchThreads, 0, st>>>(a, PeerArgs{}); break;
    case 8: cheby_batch_pieces_kernel<8><<<grid, kBatchThreads, 0, st>>>(a, PeerArgs{}); break;
    default: cheby_batch_pieces_kernel<32><<<grid, kBatchThreads, 0, st>>>(a, PeerArgs{}); break;
    }
    return grid;
}

int launch_batch_rows(const BatchArgs& a, int B, int grid, cudaStream_t st, const PeerArgs* pa) {
    if (pa) {
        CPG_PEER_SWITCH(cheby_batch_rows_kernel, B, grid, st, a, *pa);
        return grid;
    }
    if (a.nz_in) CPG_MASK_SWITCH(cheby_batch_rows_kernel, B)
    // One range policy over the iterate instead of a policy choice per gathered row
    // (CPG_ROWS_RP=0 = a policy per row): config 4 (B = 64) +2.6%; at B = 16 level at the same
    // geometry, but it frees the registers for more gathers in flight (below).
    static const int rows_rp = [] {
        const char* e = std::getenv("CPG_ROWS_RP");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    // B = 16: without the per-row policy registers the range-policy instance fits 10 gathers in
    // flight per lane at 4 CTAs/SM in 64 registers, no spills (the per-row-policy instance needs 80
    // for 8 at 3 CTAs/SM): config 5 row kernel 31.8 -> 30.7 ms, 1131 -> 1160 GTEPS
    // (profiles/r02/cw/ab_rows_geometry.txt; CPG_ROWS_RP_CFG = 83, 84, 123, 163 select others).
    if (a.hot_rows && B == 16 && rows_rp != 0) {
        static const int cfg_rp = [] {
            const char* e = std::getenv("CPG_ROWS_RP_CFG");
            return e ? std::atoi(e) : 104;
        }();
        if (cfg_rp == 84) return launch_capped(cheby_batch_rows_kernel<16, 8, 4, false, false, true>, a, grid, st);
        if (cfg_rp == 83) return launch_capped(cheby_batch_rows_kernel<16, 8, 3, false, false, true>, a, grid, st);
        if (cfg_rp == 123) return launch_capped(cheby_batch_rows_kernel<16, 12, 3, false, false, true>, a, grid, st);
        if (cfg_rp == 163) return launch_capped(cheby_batch_rows_kernel<16, 16, 3, false, false, true>, a, grid, st);
        return launch_capped(cheby_batch_rows_kernel<16, 10, 4, false, false, true>, a, grid, st);
    }
    if (a.hot_rows && B == 64 && rows_rp != 0)
        return launch_capped(cheby_batch_rows_kernel<64, 8, 4, false, false, true>, a, grid, st);
    static const int cfg16 = split_cfg("CPG_ROWS_CFG", 16), cfg64 = split_cfg("CPG_ROWS_CFG", 64);
    if (B == 16) {
        const int cfg = cfg16;
        CPG_SPLIT_CFG_SWITCH(cheby_batch_rows_kernel, 16)
    }
    if (B == 64) {
        const int cfg = cfg64;
        CPG_SPLIT_CFG_SWITCH(cheby_batch_rows_kernel, 64)
    }
    switch (B) {
    case 4: cheby_batch_rows_kernel<4><<<grid, kBatchThreads, 0, st>>>(a, PeerArgs{}); break;
    case 8: cheby_batch_rows_kernel<8><<<grid, kBatchThreads, 0, st>>>(a, PeerArgs{}); break;
    default: cheby_batch_rows_kernel<32><<<grid, kBatchThreads, 0, st>>>(a, PeerArgs{}); break;
    }
    return grid;
}

int launch_first_push(const BatchArgs& a, const uint32_t* gdeg, const uint32_t* new_of_old, const uint32_t* sources,
                      uint32_t q0, uint32_t count, uint32_t B, int grid, cudaStream_t st) {
    cheby_first_push_kernel<<<grid, kPushThreads, 0, st>>>(a, gdeg, new_of_old, sources, q0, count, B);
    return grid;  // mass rows in CTAs (one row per CTA written, the rest stay zero)
}

void launch_coarsen(const uint32_t* fine, uint64_t fine_words, uint32_t* coarse, uint32_t coarse_words, int cshift,
                    cudaStream_t st) {
    coarsen_kernel<<<(coarse_words + 255) / 256, 256, 0, st>>>(fine, fine_words, coarse, coarse_words, cshift);
}

int launch_sparse_step(const BatchArgs& a, int B, uint32_t* done, const uint32_t* fill_mask, const uint32_t* coarse,
                       uint32_t coarse_words, int cshift, uint32_t row_begin, int64_t hb, int grid, cudaStream_t st) {
    const SparseExtra x{done, fill_mask, coarse, coarse_words, cshift, row_begin, hb};
    const size_t smem = sizeof(uint32_t) * coarse_words;
#define CPG_SPARSE(BB)                                                                   \
    cheby_sparse_scan_kernel<BB><<<grid, kBatchThreads, smem, st>>>(a, x);               \
    {                                                                                    \
        BatchArgs f = a;                                                                 \
        f.mass_partial = a.mass_partial ? a.mass_partial + static_cast<size_t>(grid) * (kBatchThreads / 32) * BB : nullptr; \
        cheby_sparse_fill_kernel<BB><<<grid, kBatchThreads, 0, st>>>(f, x);              \
    }
    switch (B) {
    case 4: CPG_SPARSE(4) break;
    case 8: CPG_SPARSE(8) break;
    case 16: CPG_SPARSE(16) break;
    case 32: CPG_SPARSE(32) break;
    default: CPG_SPARSE(64) break;
    }
#undef CPG_SPARSE
    return 2 * grid;  // mass rows: one per warp of each kernel, in units of CTAs
}

int batch_occupancy() {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, cheby_batch_kernel<64>, kBatchThreads, 0);
    return blocks;
}
void launch_init_onehot(double* w, uint64_t stride, const uint32_t* gdeg, const uint32_t* no, const uint32_t* src,
                        uint32_t q0, uint32_t count, cudaStream_t st, uint32_t* nz0) {
    init_onehot_kernel<<<1, 32, 0, st>>>(w, stride, gdeg, no, src, q0, count, nz0);
}
void launch_init_onehot_batch(double* W, const uint32_t* gdeg, const uint32_t* no, const uint32_t* src,
                              uint32_t q0, uint32_t count, uint32_t B, cudaStream_t st, uint32_t* nz0) {
    init_onehot_batch_kernel<<<1, 64, 0, st>>>(W, gdeg, no, src, q0, count, B, nz0);
}
void launch_init_dense(double* w, const uint32_t* gdeg, const uint32_t* no, const double* seed,
                       uint32_t n, double a, cudaStream_t st) {
    init_dense_kernel<<<1184, 256, 0, st>>>(w, gdeg, no, seed, n, a);
}
void launch_init_dense_batch(double* W, const uint32_t* gdeg, const uint32_t* no, const double* X, uint32_t n,
                             uint32_t count, uint32_t B, double a, cudaStream_t st) {
    init_dense_batch_kernel<<<2368, 256, 0, st>>>(W, gdeg, no, X, n, count, B, a);
}
void launch_unpermute(double* out, const double* full, uint64_t stride, const uint32_t* no, uint32_t n,
                      uint32_t count, const uint32_t* gdeg, double a, cudaStream_t st) {
    unpermute_kernel<<<1184, 256, 0, st>>>(out, full, stride, no, n, count, gdeg, a);
}
void launch_unpermute_batch(double* out, const double* full, const uint32_t* no, uint32_t n,
                            uint32_t count, uint32_t B, const uint32_t* gdeg, double a, cudaStream_t st) {
    unpermute_batch_kernel<<<2368, 256, 0, st>>>(out, full, no, n, count, B, gdeg, a);
}
void launch_mass_steps(const double* mp, uint32_t n_part, uint64_t q_stride, uint32_t K, uint32_t count,
                       double* steps, cudaStream_t st) {
    mass_steps_kernel<<<dim3(K, count), kStepThreads, 0, st>>>(mp, n_part, q_stride, steps, K);
}
__global__ void zero_f64_kernel(double* p) { *p = 0.0; }
void launch_zero_f64(double* p, cudaStream_t st) { zero_f64_kernel<<<1, 1, 0, st>>>(p); }
void launch_mass_err(const double* steps, uint32_t K, double mass0, double* err, cudaStream_t st) {
    mass_err_kernel<<<1, 1, 0, st>>>(steps, K, mass0, err);
}
void launch_mass_steps_batch(const double* mp, uint32_t stride, uint32_t used, uint32_t B, uint32_t K,
                             uint32_t count, double* steps, cudaStream_t st) {
    mass_steps_batch_kernel<<<dim3(K, count), kStepThreads, 0, st>>>(mp, stride, used, B, K, steps);
}
void launch_mass_err_cols(const double* steps, uint32_t K, uint32_t count, const double* mass0, double* err,
                          cudaStream_t st) {
    mass_err_cols_kernel<<<1, 1, 0, st>>>(steps, K, count, mass0, err);
}

} // namespace cpg
