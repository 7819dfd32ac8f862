// device_graph.cuh -- device-side graph layout and kernel parameter blocks.
//
// Layout in HBM (one handle = one GPU = one row shard):
//   rows are relabelled by (degree desc, id asc) and dealt round-robin to the
//   R ranks ("degree snake"), so rank r owns the contiguous global id range
//   [r*n_loc, (r+1)*n_loc) and every rank gets ~n/R rows and ~nnz/R edges;
//   within a rank rows stay degree-descending (hubs first: the most-gathered
//   iterate entries share L2 lines).
//   rowptr  int64 [n_loc+1]   local row offsets
//   col     uint32[nnz_loc]   global (relabelled) neighbour ids, sorted per row
//   gdeg    uint32[n_pad]     degree of every global id (0 for padding)
//   new_of_old uint32[n]      caller id -> global id
//   items   WorkItem[...]     hub pieces first, then row tiles (single-source)
//   iterates: w_a, w_b fp64[n_pad] (replicated), acc fp64[n_loc]
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

namespace cpg {

// Bounds-checked build (tools/build_variant.sh checked -DCPG_CHECKED=1): every
// index into the CSR, the iterates, acc, the hub partials and the mass partials
// is checked against the buffer sizes the host passes in the chk_* fields, and a
// violation traps with the kernel, the index and the bound.  The default build
// compiles the checks and the fields out.  (The pool's compute-sanitizer is
// closed; this is the substitute, profiles/r02/checked/.)
#ifndef CPG_CHECKED
#define CPG_CHECKED 0
#endif
#if CPG_CHECKED
#define CPG_CHECK(cond, what, idx, bound)                                                              \
    do {                                                                                              \
        if (!(cond)) {                                                                                \
            printf("CPG_CHECK failed: %s index %llu bound %llu (block %d thread %d)\n", what,           \
                   (unsigned long long)(idx), (unsigned long long)(bound), (int)blockIdx.x, (int)threadIdx.x); \
            __trap();                                                                                 \
        }                                                                                             \
    } while (0)
#define CPG_CHK_FIELDS uint64_t chk_nnz, chk_npad, chk_nloc, chk_parts, chk_mass;
#else
#define CPG_CHECK(cond, what, idx, bound) \
    do {                                  \
    } while (0)
#define CPG_CHK_FIELDS
#endif

// Tile geometry of the single-source step (cheby_step_kernel).  The tile
// width is chosen per graph at upload: kTileLarge when there are enough edges
// to give every SM several tiles, kTileSmall otherwise.
constexpr int kStepThreads = 256;
constexpr int kTileSmall = 1024;                 // edges staged per tile ( 8 KB smem)
constexpr int kTileMid = 2048;                   // edges staged per tile (16 KB smem)
constexpr int kTileLarge = 4096;                 // edges staged per tile (32 KB smem)
constexpr int kTileMaxRows = 512;                // rows per tile (2 epilogue rows per thread)
constexpr int kHubPieceEdges = 4096;             // edges per hub piece (16 per thread)
constexpr int kWarpTileEdges = 512;              // warp tiles: edges per tile (16 per lane)
constexpr int kWarpTileRows = 64;                // warp tiles: rows per tile (2 epilogue rows per lane)
constexpr int kWarpLongRow = 4096;               // warp tiles: longest row swept by one warp

// Batched (SpMM) geometry: one warp per row job, 64 columns, double2 per lane.
constexpr int kBatchCols = 64;
constexpr int kBatchThreads = 256;
constexpr int kBatchMaxCtasPerSm = 6;            // grid cap of every batched launch (mass-partial sizing)
constexpr int kBatchHubEdges = 2048;             // B = 64: rows above this are split
// Hub piece in the fused batched kernel (small graphs): rows above this many
// edges are split into pieces of this length.  One row slot (B/2 lanes) works
// a piece U = 8 gathers per round, so a piece costs edges/8 dependent L2
// round trips whatever B is, and on a small graph the longest job bounds the
// step: the same edge count for every B.  96 edges measured best at B = 16
// and 64 (config 1: 512 -> 96 edges 230 -> 512 GTEPS; config 2: 2048 -> 96
// edges 295 -> 550; 64/128/192/256 slower; profiles/r01/fused_piece/).
#ifndef CPG_FUSED_HUB_EDGES
#define CPG_FUSED_HUB_EDGES 96
#endif
__host__ __device__ constexpr int batch_hub_edges(int) { return CPG_FUSED_HUB_EDGES; }
// Hub piece in the split path's piece kernel (large graphs): 64*B edges (B = 16:
// 1024), capped at 2048 for B = 64.  A piece is a run of column-sorted
// gathers; longer runs sweep the iterate more locally (config 5, B = 16:
// 512 -> 1024 edges +2.9%; config 4, B = 64: 2048 -> 4096 -1%;
// profiles/r01/hub_piece_size_c{4,5}.txt).
__host__ __device__ constexpr int batch_piece_edges(int B) { return B >= 32 ? kBatchHubEdges : 64 * B; }

// Work item (16 B, one vector load).
//   tile: a = first row, b = end row,
//         c = first edge | edge count << 40 | lg(lane group) << 54
//   hub piece (bit 63 of c set): a = row (== hub index, hubs are the row
//         prefix), b = first partial slot of this hub,
//         c = first edge | edge count << 40 | 1 << 63
//         (piece index = (first edge - rowptr[row]) / piece size)
struct __align__(16) WorkItem {
    uint32_t a, b;
    uint64_t c;
};
constexpr uint64_t kHubBit = 1ull << 63;
// Column-window hub pieces: b = the piece's OWN partial slot (the row's
// first slot and piece count come from BatchArgs::hub_meta), and bit 54 marks a piece
// whose columns all lie in one window of the warm tier of the iterate.
constexpr uint64_t kWarmBit = 1ull << 54;
__host__ __device__ inline uint64_t tile_code(uint64_t e0, uint32_t cnt, uint32_t lg) {
    return e0 | (static_cast<uint64_t>(cnt) << 40) | (static_cast<uint64_t>(lg) << 54);
}
__host__ __device__ inline int64_t code_e0(uint64_t c) { return static_cast<int64_t>(c & ((1ull << 40) - 1)); }
__host__ __device__ inline int code_cnt(uint64_t c) { return static_cast<int>((c >> 40) & 0x3fff); }

struct StepArgs {
    const int64_t* rowptr;
    const uint32_t* col;
    const WorkItem* items;
    const double* w_cur;   // gather source w_k (global ids, replicated)
    double* w_io;          // in: w_{k-1}, out: w_{k+1} (global ids)
    double* acc;           // local rows
    double* out;           // final d*acc (local rows), used when last
    double* hub_partial;   // per hub piece
    unsigned int* hub_count;
    double* mass_partial;  // [n_items] for this step
    const double* coeffs;  // device copy of c_0..c_K
    uint32_t row0;         // global id of local row 0
    uint32_t n_items;
    int tile;              // kTileSmall or kTileLarge (must match the table)
    uint32_t hot_rows;     // gathers of ids < hot_rows kept in L2 (evict_last); 0 = off
    int k;                 // computing w_k (1..K)
    int first;             // k == 1: w_k = D^-1 A w_0, acc = c0 w0 + c1 w1
    int taylor;            // power method (PwMethod, solvers.cpp:87-116): w_k = D^-1 A w_{k-1}
    int last;              // write out = d * acc instead of acc
    const uint32_t* nz_in; // MASK instances: support bitmap of w_cur (bit u = row u may be nonzero)
    uint32_t* nz_out;      // MASK instances: support bitmap of w_{k+1} to build (pre-zeroed), or null
    CPG_CHK_FIELDS         // CPG_CHECKED builds only: nnz_loc, n_pad, n_loc, hub partial slots, mass slots
};

// Query group (cheby_step_group_kernel): nq single-source queries in one
// launch; query q uses the slices w + q*vec_stride, acc/out + q*acc_stride,
// hub_partial + q*part_stride, hub_count + q*cnt_stride, mass_partial +
// q*mass_stride of the StepArgs arrays.  (A separate parameter block, so the
// one-query kernel's StepArgs and its code are unchanged.)
struct StepGroup {
    uint32_t nq;
    uint64_t vec_stride, acc_stride;
    uint32_t part_stride, cnt_stride, mass_stride;
};


struct BatchArgs {
    const int64_t* rowptr;
    const uint32_t* col;
    const WorkItem* hub_items;  // hub pieces (row, partial slot base, first edge | count | hub bit)
    uint32_t n_hub_items;
    uint32_t hub_rows;          // rows [0, hub_rows) are hubs
    uint32_t n_loc;
    const double* w_cur;        // [n_pad][64]
    double* w_io;               // [n_pad][64]
    double* acc;                // [n_loc][64]
    double* out;                // [n_loc][64] when last
    double* hub_partial;        // [slots][64]
    unsigned int* hub_count;
    const double* coeffs;
    uint32_t row0;
    uint32_t hot_rows;          // gathers of rows < hot_rows are kept in L2 (evict_last); 0 = off
    int k, first, last;
    unsigned int* job_ctr;      // fused kernel: zeroed job counter (warps claim RPW jobs each); null = static stride
    double* mass_partial;       // [gridDim.x * warps][B] per-warp column sums of d_v w_{k+1}(v) (acceptance C13); null = off
    const uint32_t* nz_in;      // MASK instances: support bitmap of w_cur's rows (any column nonzero)
    uint32_t* nz_out;           // MASK instances: support bitmap of w_{k+1}'s rows to build (pre-zeroed), or null
    const uint2* hub_meta;      // column-window pieces: (first partial slot, piece count) of hub row meta_row0 + i; null = uniform pieces
    uint32_t meta_row0;
    uint32_t n_pad_rows;        // rows of the replicated iterate (range-policy window)
    CPG_CHK_FIELDS              // CPG_CHECKED builds only (partial / mass bounds in rows of B doubles)
};

// Support bitmaps (sparse early steps).  The reference's scatter
// skips every source entry that is exactly zero (graph.cpp:262: `if (xu == 0.0)
// continue;`); the pull step does the same with one bit per row of the iterate:
// a gather of row u is issued only if bit u is set, and a row whose bit is clear
// holds exact zeros, so skipping its add leaves every sum bit-identical.  Bit u of
// nz is set if row u of the iterate may be nonzero (a superset is always exact).
#ifdef __CUDACC__
__device__ __forceinline__ bool nz_bit(const uint32_t* nz, uint32_t u) {
    return (__ldg(nz + (u >> 5)) >> (u & 31)) & 1u;
}
__device__ __forceinline__ void nz_set(uint32_t* nz, uint32_t u) { atomicOr(nz + (u >> 5), 1u << (u & 31)); }
#endif
__host__ __device__ inline uint64_t nz_words(uint64_t n_pad) { return (n_pad + 31) / 32; }

// Fused all-gather (second parameter of the PEER instances of the batched
// kernels): w_io's row also goes to peer_io[p] for p in [0, n_peer), p != self.
// A separate block keeps BatchArgs, and the code of the plain instances, as is.
struct PeerArgs {
    double* const* peer_io;     // device array of the ranks' w_io replicas (LSA pointers)
    int n_peer, self;
};

} // namespace cpg
