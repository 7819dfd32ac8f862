// graph_build.cu -- CSR upload: degree-sorted relabel, row-shard extraction and
// the load-balanced work tables.  One-time work per graph handle, off the timed
// path (the reference's Graph::from_csr + inv_degree_, graph.cpp:48-104, is the
// host analogue).  All of it runs on the device with CUB primitives.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <unordered_map>
#include <mutex>

#include "cpg_graph.hpp"

namespace cpg {

namespace {

constexpr int kT = 256;

inline int grid_for(uint64_t n, int cap = 148 * 16) {
    return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + kT - 1) / kT, cap)));
}

template <typename T>
T* dalloc(size_t count) {
    T* p = nullptr;
    CPG_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
    return p;
}

struct DevTemp {
    void* p = nullptr;
    size_t bytes = 0;
    void ensure(size_t b) {
        if (b > bytes) {
            if (p) cudaFree(p);
            CPG_CUDA(cudaMalloc(&p, b));
            bytes = b;
        }
    }
    ~DevTemp() {
        if (p) cudaFree(p);
    }
};

__global__ void k_deg_ids(const uint64_t* off, uint32_t n, uint32_t* deg, uint32_t* ids) {
    for (uint64_t v = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; v < n; v += (uint64_t)gridDim.x * blockDim.x) {
        deg[v] = static_cast<uint32_t>(off[v + 1] - off[v]);
        ids[v] = static_cast<uint32_t>(v);
    }
}

// Layout for R ranks x C chunks, cr = ceil(n / (R*C)) rows per (rank, chunk):
// position i of the degree order -> rank = i % R, t = i / R, chunk = t % C,
// j = t / C; global id = chunk*R*cr + rank*cr + j; local row = chunk*cr + j.
// Every (rank, chunk) gets every (R*C)-th node of the degree order (balanced
// rows and edges), and the rows of chunk c of all ranks are one contiguous
// block of the replicated iterate, so each chunk is one in-place all-gather.
__global__ void k_assign(const uint32_t* order, const uint32_t* sdeg, uint32_t n, uint32_t R, uint32_t C,
                         uint32_t cr, uint32_t* new_of_old, uint32_t* gdeg) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = i / R;
        const uint32_t g = static_cast<uint32_t>((t % C) * R * cr + (i % R) * cr + t / C);
        new_of_old[order[i]] = g;
        gdeg[g] = sdeg[i];
    }
}

__global__ void k_local(const uint32_t* order, const uint32_t* sdeg, uint32_t n, uint32_t R, uint32_t C, uint32_t cr,
                        uint32_t rank, uint32_t n_loc, int64_t* ldeg, uint32_t* lold) {
    for (uint64_t l = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; l <= n_loc; l += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = ((l % cr) * C + l / cr) * R + rank;
        const bool real = l < n_loc && i < n;
        ldeg[l] = real ? sdeg[i] : 0;
        if (l < n_loc) lold[l] = real ? order[i] : 0xffffffffu;
    }
}

// One warp per local row: relabelled neighbours keyed by (row, new id).
__global__ void k_fill_keys(const int64_t* rowptr, const uint32_t* lold, const uint64_t* off, const uint32_t* nbr,
                            const uint32_t* new_of_old, uint32_t n_loc, uint64_t* keys) {
    const uint64_t lane = threadIdx.x & 31;
    for (uint64_t j = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5; j < n_loc;
         j += ((uint64_t)gridDim.x * blockDim.x) >> 5) {
        const uint32_t old = lold[j];
        if (old == 0xffffffffu) continue;
        const uint64_t s = off[old], d = off[old + 1] - s;
        const int64_t dst = rowptr[j];
        for (uint64_t t = lane; t < d; t += 32)
            keys[dst + t] = (j << 32) | new_of_old[nbr[s + t]];
    }
}

__global__ void k_extract(const uint64_t* keys, uint64_t nnz, uint32_t* col) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz; e += (uint64_t)gridDim.x * blockDim.x)
        col[e] = static_cast<uint32_t>(keys[e] & 0xffffffffu);
}

// Rows of a range are degree-descending, so hubs are a prefix: count = last
// index with deg > thr, +1 (rowptr points at the range's first row).
__global__ void k_count_above(const int64_t* rowptr, uint32_t n_rows, int64_t thr, unsigned int* count) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_rows; j += (uint64_t)gridDim.x * blockDim.x) {
        const int64_t d = rowptr[j + 1] - rowptr[j];
        const int64_t dn = j + 1 < n_rows ? rowptr[j + 2] - rowptr[j + 1] : -1;
        if (d > thr && dn <= thr) *count = static_cast<unsigned int>(j + 1);
    }
}

__global__ void k_pieces(const int64_t* rowptr, uint32_t n_hub, int64_t piece, uint32_t* P) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= n_hub; j += gridDim.x * blockDim.x)
        P[j] = j < n_hub ? static_cast<uint32_t>((rowptr[j + 1] - rowptr[j] + piece - 1) / piece) : 0u;
}  // rowptr points at the range's first row

// Hub piece p of hub row row0+j: {row, first partial slot of the hub (+ slot
// offset), first edge | edge count | hub bit}.
__global__ void k_hub_items(const int64_t* rowptr, uint32_t row0, const uint32_t* P, const uint32_t* base,
                            uint32_t n_hub, int64_t piece, uint32_t slot_off, WorkItem* items) {
    const int lane = threadIdx.x & 31;
    for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n_hub; j += (gridDim.x * blockDim.x) >> 5) {
        const int64_t rs = rowptr[row0 + j], d = rowptr[row0 + j + 1] - rs;
        for (uint32_t p = lane; p < P[j]; p += 32) {
            const int64_t e0 = rs + static_cast<int64_t>(p) * piece;
            const uint32_t cnt = static_cast<uint32_t>(min(piece, d - static_cast<int64_t>(p) * piece));
            items[base[j] + p] =
                WorkItem{row0 + j, slot_off + base[j], tile_code(static_cast<uint64_t>(e0), cnt, 0) | kHubBit};
        }
    }
}

// A row starts a tile when its first edge falls in a new chunk of tile/2 edges
// (or every kTileMaxRows rows).  All rows of a tile start inside one chunk and
// non-hub rows have <= tile/2 edges, so a tile holds <= tile edges.
// solo > 0: rows of more than `solo` edges form a tile of their own (warp tiles).
__global__ void k_tile_flags(const int64_t* rowptr, uint32_t first, uint32_t n_loc, int64_t chunk, uint32_t max_rows,
                             uint8_t* flags, int64_t solo = 0) {
    for (uint64_t j = first + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_loc;
         j += (uint64_t)gridDim.x * blockDim.x) {
        bool start = (j == first) || ((j - first) % max_rows == 0) ||
                     (rowptr[j] / chunk != rowptr[j - 1] / chunk);
        if (solo > 0 && j > first)
            start = start || rowptr[j + 1] - rowptr[j] > solo || rowptr[j] - rowptr[j - 1] > solo;
        flags[j - first] = start ? 1 : 0;
    }
}

__global__ void k_tile_items(const int64_t* rowptr, const uint32_t* starts, uint32_t n_tiles, uint32_t n_loc,
                             WorkItem* items) {
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles; t += gridDim.x * blockDim.x) {
        const uint32_t rb = starts[t];
        const uint32_t re = t + 1 < n_tiles ? starts[t + 1] : n_loc;
        const int64_t edges = rowptr[re] - rowptr[rb];
        const double avg = static_cast<double>(edges) / static_cast<double>(re - rb);
        int lg = 0;
        while (lg < 5 && static_cast<double>(2 << lg) <= avg / 2.0) ++lg;  // g <= mean/2
        items[t] = WorkItem{rb, re, tile_code(static_cast<uint64_t>(rowptr[rb]), static_cast<uint32_t>(edges),
                                               static_cast<uint32_t>(lg))};
    }
}

// Hub-piece items for rows [row0, row1) with degree > thr (pieces of `piece`
// edges; the hubs are a prefix of the range).  Items are allocated here.
void build_hub_items(const int64_t* rowptr, uint32_t row0, uint32_t row1, int64_t thr, int64_t piece,
                     uint32_t slot_off, WorkItem** out, uint32_t* n_hub_out, uint32_t* n_items_out,
                     uint32_t reserve_tail, cudaStream_t st) {
    const uint32_t n_rows = row1 - row0;
    unsigned int* d_cnt = dalloc<unsigned int>(1);
    CPG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned int), st));
    if (n_rows) k_count_above<<<grid_for(n_rows), kT, 0, st>>>(rowptr + row0, n_rows, thr, d_cnt);
    unsigned int n_hub = 0;
    CPG_CUDA(cudaMemcpyAsync(&n_hub, d_cnt, sizeof(n_hub), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_cnt);
    uint32_t* P = dalloc<uint32_t>(n_hub + 1);
    uint32_t* base = dalloc<uint32_t>(n_hub + 1);
    k_pieces<<<grid_for(n_hub + 1), kT, 0, st>>>(rowptr + row0, n_hub, piece, P);
    DevTemp tmp;
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, P, base, n_hub + 1, st);
    tmp.ensure(bytes);
    CPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, P, base, n_hub + 1, st));
    uint32_t total = 0;
    CPG_CUDA(cudaMemcpyAsync(&total, base + n_hub, sizeof(total), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    WorkItem* items = dalloc<WorkItem>(static_cast<size_t>(total) + reserve_tail);
    if (n_hub)
        k_hub_items<<<grid_for(static_cast<uint64_t>(n_hub) * 32), kT, 0, st>>>(rowptr, row0, P, base, n_hub, piece,
                                                                                 slot_off, items);
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(P);
    cudaFree(base);
    *out = items;
    *n_hub_out = n_hub;
    *n_items_out = total;
}

// ---------------------------------------------------------------------------
// Column-window hub pieces.  The gathers of a hub row are column
// sorted.  The rows of the iterate past the L2-resident hot prefix but still
// gathered hundreds of times per step (the "warm tier", [lo, lo + W*S) in the
// degree order) are cut into W windows of S rows, each small enough to stay in
// L2; the biggest hubs (degree > cw_deg) are cut at those boundaries, and the
// piece list is ordered window-major, so the pieces in flight (claimed in list
// order by the piece kernel) gather from one window at a time.
// ---------------------------------------------------------------------------

// bnd[h * (W + 1) + j] = first edge of hub row row0 + h with column >= lo + j * S.
__global__ void k_cw_bounds(const int64_t* rowptr, const uint32_t* col, uint32_t row0, uint32_t n_cw, uint32_t lo,
                            uint32_t S, uint32_t W, int64_t* bnd) {
    const uint64_t total = static_cast<uint64_t>(n_cw) * (W + 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t h = static_cast<uint32_t>(i / (W + 1)), j = static_cast<uint32_t>(i % (W + 1));
        int64_t a = rowptr[row0 + h], b = rowptr[row0 + h + 1];
        const uint64_t key = static_cast<uint64_t>(lo) + static_cast<uint64_t>(j) * S;
        while (a < b) {
            const int64_t mid = a + (b - a) / 2;
            if (col[mid] < key) a = mid + 1;
            else b = mid;
        }
        bnd[i] = a;
    }
}

// Segment s of a column-window row: 0 = hot prefix, 1..W = warm windows, W + 1 = cold tail.
__device__ __forceinline__ void cw_segment(const int64_t* bnd_h, int64_t rs, int64_t re, uint32_t W, uint32_t s,
                                           int64_t& b, int64_t& e) {
    b = s == 0 ? rs : bnd_h[s - 1];
    e = s == W + 1 ? re : bnd_h[s];
}

__global__ void k_cw_pieces(const int64_t* rowptr, uint32_t row0, uint32_t n_hub, uint32_t n_cw, const int64_t* bnd,
                            uint32_t W, int64_t piece, uint32_t* P) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j <= n_hub; j += gridDim.x * blockDim.x) {
        uint32_t p = 0;
        if (j < n_hub) {
            const int64_t rs = rowptr[row0 + j], re = rowptr[row0 + j + 1];
            if (j < n_cw) {
                for (uint32_t s = 0; s <= W + 1; ++s) {
                    int64_t b, e;
                    cw_segment(bnd + static_cast<size_t>(j) * (W + 1), rs, re, W, s, b, e);
                    p += static_cast<uint32_t>((e - b + piece - 1) / piece);
                }
            } else {
                p = static_cast<uint32_t>((re - rs + piece - 1) / piece);
            }
        }
        P[j] = p;
    }
}

// One warp per hub row: the row's pieces in column order (piece index = slot order, so
// the ordered combine adds them left to right), each with its own slot and a sort key
// phase << 32 | list index.  Warm-window pieces get phase = window; the others phase 0,
// or (spread) one of the W phases round-robin, so every phase mixes L2-resident window
// gathers with DRAM-bound ones.
__global__ void k_cw_items(const int64_t* rowptr, uint32_t row0, const uint32_t* P, const uint32_t* base,
                           uint32_t n_hub, uint32_t n_cw, const int64_t* bnd, uint32_t W, int64_t piece,
                           uint32_t slot_off, int spread, WorkItem* items, uint64_t* keys, uint2* meta) {
    const int lane = threadIdx.x & 31;
    for (uint32_t j = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n_hub; j += (gridDim.x * blockDim.x) >> 5) {
        const int64_t rs = rowptr[row0 + j], re = rowptr[row0 + j + 1];
        if (lane == 0) meta[j] = make_uint2(slot_off + base[j], P[j]);
        uint32_t p0 = 0;
        const uint32_t n_seg = j < n_cw ? W + 2 : 1;
        for (uint32_t s = 0; s < n_seg; ++s) {
            int64_t b = rs, e = re;
            if (j < n_cw) cw_segment(bnd + static_cast<size_t>(j) * (W + 1), rs, re, W, s, b, e);
            const uint32_t np = static_cast<uint32_t>((e - b + piece - 1) / piece);
            const bool warm = j < n_cw && s >= 1 && s <= W;
            for (uint32_t p = lane; p < np; p += 32) {
                const int64_t e0 = b + static_cast<int64_t>(p) * piece;
                const uint32_t cnt = static_cast<uint32_t>(min(piece, e - e0));
                const uint32_t idx = base[j] + p0 + p;
                items[idx] = WorkItem{row0 + j, slot_off + idx,
                                      tile_code(static_cast<uint64_t>(e0), cnt, 0) | kHubBit | (warm ? kWarmBit : 0ull)};
                // spread & 4: the uncut pieces go to the window phases in blocks of 256 list positions, and
                // inside a block the warm pieces come first, so a warp's RPW pieces stay of one kind while
                // DRAM-bound and L2-bound warps run side by side in every phase
                const uint32_t phase = warm ? s : ((spread & 4) ? 1 + (idx >> 8) % W : ((spread & 1) ? 1 + idx % W : 0));
                // spread & 2: the pieces of a window longest first (a warp's RPW pieces run in lock-step)
                uint32_t sec = warm && (spread & 2) ? ((static_cast<uint32_t>(piece) - cnt) << 20) | (idx & 0xfffffu) : idx;
                if (spread & 4) sec = ((idx >> 8) << 9) | (warm ? 0u : 256u) | (idx & 255u);
                keys[idx] = (static_cast<uint64_t>(phase) << 32) | sec;
            }
            p0 += np;
        }
    }
}

__global__ void k_permute_items(const WorkItem* in, const uint32_t* perm, uint32_t n, WorkItem* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) out[i] = in[perm[i]];
}

__global__ void k_iota(uint32_t* v, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

// Column-window hub items of rows [row0, row1): hubs = rows of degree > piece (as in
// build_hub_items), the first n_cw of them (degree > cw_deg) cut at the window
// boundaries.  Returns false (nothing allocated) when no row qualifies.
bool build_cw_hub_items(const int64_t* rowptr, const uint32_t* col, uint32_t row0, uint32_t row1, int64_t piece,
                        int64_t hub_thr, int64_t cw_deg, uint32_t lo, uint32_t S, uint32_t W, int spread,
                        uint32_t min_cut, uint32_t slot_off, ItemTable* t, cudaStream_t st) {
    const uint32_t n_rows = row1 - row0;
    if (!n_rows || !W) return false;
    unsigned int* d_cnt = dalloc<unsigned int>(2);
    CPG_CUDA(cudaMemsetAsync(d_cnt, 0, 2 * sizeof(unsigned int), st));
    k_count_above<<<grid_for(n_rows), kT, 0, st>>>(rowptr + row0, n_rows, hub_thr, d_cnt);
    k_count_above<<<grid_for(n_rows), kT, 0, st>>>(rowptr + row0, n_rows, std::max(cw_deg, hub_thr), d_cnt + 1);
    unsigned int cnt[2] = {0, 0};
    CPG_CUDA(cudaMemcpyAsync(cnt, d_cnt, sizeof(cnt), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_cnt);
    const uint32_t n_hub = cnt[0], n_cw = cnt[1];
    // Each window phase holds about one piece per cut row.  The pieces in flight (claimed in list
    // order) must be a small part of a phase, or several windows are swept at once and none stays
    // resident: below min_cut rows the table keeps uniform pieces (a sharded rank's chunk tables).
    if (!n_cw || n_cw < min_cut) return false;
    int64_t* bnd = dalloc<int64_t>(static_cast<size_t>(n_cw) * (W + 1));
    k_cw_bounds<<<grid_for(static_cast<uint64_t>(n_cw) * (W + 1)), kT, 0, st>>>(rowptr, col, row0, n_cw, lo, S, W, bnd);
    uint32_t* P = dalloc<uint32_t>(n_hub + 1);
    uint32_t* base = dalloc<uint32_t>(n_hub + 1);
    k_cw_pieces<<<grid_for(n_hub + 1), kT, 0, st>>>(rowptr, row0, n_hub, n_cw, bnd, W, piece, P);
    DevTemp tmp;
    size_t bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, P, base, n_hub + 1, st);
    tmp.ensure(bytes);
    CPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, P, base, n_hub + 1, st));
    uint32_t total = 0;
    CPG_CUDA(cudaMemcpyAsync(&total, base + n_hub, sizeof(total), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    WorkItem* unsorted = dalloc<WorkItem>(total);
    uint64_t* keys = dalloc<uint64_t>(total);
    uint64_t* keys_out = dalloc<uint64_t>(total);
    uint32_t* iota = dalloc<uint32_t>(total);
    uint32_t* perm = dalloc<uint32_t>(total);
    t->meta = dalloc<uint2>(n_hub);
    k_cw_items<<<grid_for(static_cast<uint64_t>(n_hub) * 32), kT, 0, st>>>(rowptr, row0, P, base, n_hub, n_cw, bnd, W,
                                                                            piece, slot_off, spread, unsorted, keys,
                                                                            t->meta);
    k_iota<<<grid_for(total), kT, 0, st>>>(iota, total);
    bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys, keys_out, iota, perm, total, 0, 40, st);
    tmp.ensure(bytes);
    CPG_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys, keys_out, iota, perm, total, 0, 40, st));
    t->items = dalloc<WorkItem>(total);
    k_permute_items<<<grid_for(total), kT, 0, st>>>(unsorted, perm, total, t->items);
    CPG_CUDA(cudaStreamSynchronize(st));
    for (void* q : {(void*)bnd, (void*)P, (void*)base, (void*)unsorted, (void*)keys, (void*)keys_out, (void*)iota,
                    (void*)perm})
        cudaFree(q);
    t->n_hubs = n_hub;
    t->n_hub_items = total;
    if (std::getenv("CPG_CW_DEBUG"))
        std::fprintf(stderr, "[cpg] column-window pieces: rows [%u, %u): %u hubs, %u cut (degree > %lld), %u windows x %u rows "
                     "from row %u, %u pieces\n", row0, row1, n_hub, n_cw, static_cast<long long>(cw_deg), W, S, lo, total);
    return true;
}

} // namespace

// Work table over local rows [row0, row1): hub pieces (rows with deg > chunk,
// split into `piece`-edge pieces, partial slots from slot_off) then row tiles
// (<= 2*chunk edges, <= max_rows rows).
ItemTable build_item_table(const int64_t* rowptr, uint32_t row0, uint32_t row1, int64_t chunk, uint32_t max_rows,
                           int64_t piece, uint32_t slot_off, cudaStream_t st, int64_t hub_thr, int64_t solo) {
    DevTemp tmp;
    size_t bytes = 0;
    WorkItem* hub_items = nullptr;
    uint32_t n_hub = 0, n_hub_items = 0;
    build_hub_items(rowptr, row0, row1, hub_thr > 0 ? hub_thr : chunk, piece, slot_off, &hub_items, &n_hub,
                    &n_hub_items, 0, st);
    uint32_t n_tiles = 0;
    uint32_t* starts = nullptr;
    const uint32_t first = row0 + n_hub;
    if (first < row1) {
        const uint32_t rows = row1 - first;
        uint8_t* flags = dalloc<uint8_t>(rows);
        starts = dalloc<uint32_t>(rows);
        unsigned int* d_sel = dalloc<unsigned int>(1);
        k_tile_flags<<<grid_for(rows), kT, 0, st>>>(rowptr, first, row1, chunk, max_rows, flags, solo);
        cub::CountingInputIterator<uint32_t> it(first);
        cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, starts, d_sel, rows, st);
        tmp.ensure(bytes);
        CPG_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, flags, starts, d_sel, rows, st));
        CPG_CUDA(cudaMemcpyAsync(&n_tiles, d_sel, sizeof(n_tiles), cudaMemcpyDeviceToHost, st));
        CPG_CUDA(cudaStreamSynchronize(st));
        cudaFree(flags);
        cudaFree(d_sel);
    }
    ItemTable t;
    t.items = dalloc<WorkItem>(static_cast<size_t>(n_hub_items) + n_tiles);
    if (n_hub_items)
        CPG_CUDA(cudaMemcpyAsync(t.items, hub_items, sizeof(WorkItem) * n_hub_items, cudaMemcpyDeviceToDevice, st));
    if (n_tiles) k_tile_items<<<grid_for(n_tiles), kT, 0, st>>>(rowptr, starts, n_tiles, row1, t.items + n_hub_items);
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(hub_items);
    if (starts) cudaFree(starts);
    t.n_items = n_hub_items + n_tiles;
    t.n_hubs = n_hub;
    t.n_hub_items = n_hub_items;
    t.row_begin = row0;
    t.row_end = row1;
    return t;
}

void build_device_graph(cpg_graph* g, const uint64_t* d_off, const uint32_t* d_nbr, cudaStream_t st) {
    const uint32_t n = g->n;
    const uint32_t R = static_cast<uint32_t>(g->nranks);
    const uint32_t rank = static_cast<uint32_t>(g->rank);
    const uint32_t C = static_cast<uint32_t>(std::max(1, g->chunks));
    const uint64_t RC = static_cast<uint64_t>(R) * C;
    g->cr = static_cast<uint32_t>((n + RC - 1) / RC);
    g->n_loc = g->cr * C;
    g->n_pad = g->n_loc * R;
    g->row0 = rank * g->cr;  // global id of local row 0 (chunk 0)
    const uint32_t n_loc = g->n_loc;
    DevTemp tmp;
    size_t bytes = 0;

    // 1. degree order: (degree desc, id asc) -- radix sort is stable.
    uint32_t* deg = dalloc<uint32_t>(n);
    uint32_t* ids = dalloc<uint32_t>(n);
    uint32_t* sdeg = dalloc<uint32_t>(n);
    uint32_t* order = dalloc<uint32_t>(n);
    k_deg_ids<<<grid_for(n), kT, 0, st>>>(d_off, n, deg, ids);
    cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, deg, sdeg, ids, order, n, 0, 32, st);
    tmp.ensure(bytes);
    CPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp.p, bytes, deg, sdeg, ids, order, n, 0, 32, st));
    CPG_CUDA(cudaMemcpyAsync(&g->max_degree, sdeg, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    cudaFree(deg);
    cudaFree(ids);

    // 2. relabel + shard assignment.
    g->new_of_old = dalloc<uint32_t>(n);
    g->gdeg = dalloc<uint32_t>(g->n_pad);
    CPG_CUDA(cudaMemsetAsync(g->gdeg, 0, sizeof(uint32_t) * g->n_pad, st));
    k_assign<<<grid_for(n), kT, 0, st>>>(order, sdeg, n, R, C, g->cr, g->new_of_old, g->gdeg);
    int64_t* ldeg = dalloc<int64_t>(static_cast<size_t>(n_loc) + 1);
    uint32_t* lold = dalloc<uint32_t>(n_loc);
    k_local<<<grid_for(static_cast<uint64_t>(n_loc) + 1), kT, 0, st>>>(order, sdeg, n, R, C, g->cr, rank, n_loc, ldeg,
                                                                        lold);
    cudaFree(sdeg);
    cudaFree(order);

    // 3. local row pointers.
    g->rowptr = static_cast<int64_t*>(dalloc_aligned(sizeof(int64_t) * (static_cast<size_t>(n_loc) + 1)));
    bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, ldeg, g->rowptr, n_loc + 1, st);
    tmp.ensure(bytes);
    CPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, ldeg, g->rowptr, n_loc + 1, st));
    int64_t nnz_loc = 0;
    CPG_CUDA(cudaMemcpyAsync(&nnz_loc, g->rowptr + n_loc, sizeof(nnz_loc), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(ldeg);
    g->nnz_loc = static_cast<uint64_t>(nnz_loc);

    // 4. relabelled column ids, sorted within each row (64-bit (row,col) radix sort).
    {
        uint64_t* keys = dalloc<uint64_t>(g->nnz_loc);
        uint64_t* keys_sorted = dalloc<uint64_t>(g->nnz_loc);
        k_fill_keys<<<grid_for(static_cast<uint64_t>(n_loc) * 32), kT, 0, st>>>(g->rowptr, lold, d_off, d_nbr,
                                                                                 g->new_of_old, n_loc, keys);
        int row_bits = 1;
        while (row_bits < 32 && (1ull << row_bits) < n_loc) ++row_bits;
        bytes = 0;
        cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys, keys_sorted, g->nnz_loc, 0, 32 + row_bits, st);
        tmp.ensure(bytes);
        CPG_CUDA(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, keys, keys_sorted, g->nnz_loc, 0, 32 + row_bits, st));
        cudaFree(keys);
        g->col = static_cast<uint32_t*>(dalloc_aligned(sizeof(uint32_t) * std::max<uint64_t>(1, g->nnz_loc)));
        k_extract<<<grid_for(g->nnz_loc), kT, 0, st>>>(keys_sorted, g->nnz_loc, g->col);
        CPG_CUDA(cudaStreamSynchronize(st));
        cudaFree(keys_sorted);
    }
    cudaFree(lold);

    // 5. single-source work table: hub pieces, then row tiles.  Large tiles
    //    when every SM gets >= 8 of them, small tiles otherwise.
    //    An iterate larger than L2 makes the gathers DRAM-latency bound: the
    //    step then runs split (hub-piece kernel + 1024-edge tile kernel at 8
    //    CTAs/SM; config 5: 146 -> 165 GTEPS, profiles/r01/single_split/).
    int l2 = 0;
    CPG_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, g->device));
    g->step_split = static_cast<uint64_t>(g->n_pad) * sizeof(double) > static_cast<uint64_t>(l2);
    //    Large tiles when a launch holds >= 8 of them per SM.  Small graphs run
    //    several queries per launch (query groups, up to 16; one rank), which
    //    counts here: configs 1/2 went from 121/101 to 198/135 GTEPS with
    //    4096-edge tiles (profiles/r01/single_groups/tile_rule.txt).
    const uint64_t q_max = g->nranks > 1 ? 1 : std::min<uint64_t>(16, std::max<uint64_t>(1, (16ull << 20) /
                                                                      std::max<uint64_t>(1, g->nnz_loc)));
    g->tile = g->nnz_loc * q_max >= static_cast<uint64_t>(kTileLarge) * g->sm_count * 8 ? kTileLarge : kTileSmall;
    if (g->step_split) g->tile = kTileSmall;
    if (const char* force = std::getenv("CPG_TILE")) {  // test hook: exercise either width
        const int t = std::atoi(force);
        if (t == kTileSmall || t == kTileMid || t == kTileLarge) g->tile = t;
    }
    g->tables.clear();
    uint32_t slots = 0;
    for (uint32_t c = 0; c < C; ++c) {
        ItemTable t = build_item_table(g->rowptr, c * g->cr, (c + 1) * g->cr, g->tile / 2, kTileMaxRows,
                                       kHubPieceEdges, slots, st);
        slots += t.n_hub_items;  // one partial slot per hub piece
        g->tables.push_back(t);
    }
    // warp-tile tables (cheby_step_warp_kernel): rows above kWarpLongRow edges are hub
    // pieces, rows above kWarpTileEdges/2 single-row items, the rest tiles of <= 512 edges
    // and <= 64 rows.  Their hub pieces take partial slots after the CTA tables'.
    g->wtables.clear();
    uint32_t wslots = 0;
    for (uint32_t c = 0; c < C; ++c) {
        ItemTable t = build_item_table(g->rowptr, c * g->cr, (c + 1) * g->cr, kWarpTileEdges / 2, kWarpTileRows,
                                       kHubPieceEdges, wslots, st, kWarpLongRow, kWarpTileEdges / 2);
        wslots += t.n_hub_items;
        g->wtables.push_back(t);
    }
    g->n_partials = std::max(slots, wslots);
    g->n_items = g->n_hubs = g->n_hub_items = g->n_tiles = 0;
    for (const auto& t : g->tables) {
        g->n_items += t.n_items;
        g->n_hubs += t.n_hubs;
        g->n_hub_items += t.n_hub_items;
        g->n_tiles += t.n_items - t.n_hub_items;
    }
    CPG_CUDA(cudaGetLastError());
}

// Large buffers the steps touch all over every step -- the gathered iterates
// (every edge reads a random row of w_k) and the per-row arrays read at the
// positions of the rows in flight (col, rowptr, acc) -- are placed at 512
// MB-aligned addresses.  Measured on config 5: 68.7 -> 66.3 ms per step for
// the iterates alone, the same as a fresh region
// (profiles/r01/iterate_alignment.txt); presumably larger translation entries.
namespace {
std::mutex g_align_mu;
std::unordered_map<void*, void*> g_align_base;  // aligned pointer -> cudaMalloc'd block
}  // namespace

void* dalloc_aligned(size_t bytes) {
    const size_t align = bytes >= (256ull << 20) ? (512ull << 20) : 0;
    void* base = nullptr;
    if (cudaMalloc(&base, std::max<size_t>(bytes, 8) + align) != cudaSuccess)
        fail(CPG_ENOMEM, "cudaMalloc of " + std::to_string(bytes + align) + " bytes failed");
    void* p = align ? reinterpret_cast<void*>((reinterpret_cast<uintptr_t>(base) + align - 1) / align * align) : base;
    std::lock_guard<std::mutex> lock(g_align_mu);
    g_align_base[p] = base;
    return p;
}

void dfree_aligned(void* p) {
    if (!p) return;
    void* base = p;
    {
        std::lock_guard<std::mutex> lock(g_align_mu);
        auto it = g_align_base.find(p);
        if (it != g_align_base.end()) {
            base = it->second;
            g_align_base.erase(it);
        }
    }
    cudaFree(base);
}

namespace {
struct CwParams {
    int64_t deg = 0, hub = 1 << 30;  // rows above `hub` edges run in the piece kernel (default: the piece length)
    uint32_t lo = 0, S = 0, W = 0;
    int spread = 1;
    uint32_t min_cut = 0;
};
uint64_t env_u64(const char* name, uint64_t dflt) {
    const char* e = std::getenv(name);
    return e ? static_cast<uint64_t>(std::atoll(e)) : dflt;
}
CwParams cw_params(const cpg_graph* g, int B, bool split) {
    CwParams p;
    // B = 64 (512-B rows): a short window segment still moves kilobytes, so more rows pay: 768 at
    // both thresholds (config 3 831 -> 870-880 GTEPS, config 4 1584 -> 1617); at B = 16 rows of
    // 513-1024 edges lose 5% when cut (profiles/r02/cw/ab_column_windows.txt)
    p.deg = static_cast<int64_t>(env_u64("CPG_CW_DEG", B == 64 ? 768 : 2048));
    // (the fused all-gather's PEER instances keep uniform pieces)
    if (!split || p.deg <= 0 || g->p2p || (B != 16 && B != 64)) return p;
    const uint64_t row_bytes = 8ull * static_cast<uint64_t>(B);
    // The piece kernel's own hot prefix: with the windows serving the warm tier it wants most of the
    // L2 for the window, so 32 MB (not the 64 MB of the other kernels): config 5 piece kernel 20.0 ->
    // 17.9 ms (8-32 MB level; profiles/r02/cw/ab_hot_window.txt).  api.cu passes the same rows.
    const uint64_t lo = (env_u64("CPG_CW_HOT_MB", 32) << 20) / row_bytes;
    const uint64_t S = std::max<uint64_t>(1024, (env_u64("CPG_CW_MB", 48) << 20) / row_bytes);
    const uint64_t end = std::min<uint64_t>(g->n_pad, (env_u64("CPG_CW_WARM_MB", 1024) << 20) / row_bytes);
    if (end <= lo + S / 2) return p;  // no warm tier: the iterate is (almost) inside the hot prefix
    p.lo = static_cast<uint32_t>(lo);
    p.S = static_cast<uint32_t>(S);
    p.W = static_cast<uint32_t>(std::min<uint64_t>(64, (end - lo + S - 1) / S));
    p.spread = static_cast<int>(env_u64("CPG_CW_SPREAD", 0));
    p.hub = static_cast<int64_t>(env_u64("CPG_CW_HUB", B == 64 ? 768 : 1 << 30));
    // B = 16: 4 pieces per warp, 3 CTAs of 8 warps per SM in flight; twice that many cut rows at least
    // (one rank: 397 K rows; 4 chunks of one rank, 99 K: level with uniform pieces; 8 ranks x 4 chunks,
    // 12 K: fewer pieces per phase than are in flight).  B = 64 keeps its windows at any size: there
    // the gain is as much the lower hub threshold and the range policy (config 3: 3-6 K cut rows, +5%).
    p.min_cut = static_cast<uint32_t>(env_u64("CPG_CW_MIN_ROWS", B == 16 ? 2ull * g->sm_count * 3 * 8 * 4 : 0));
    return p;
}
}  // namespace

const BatchTables& ensure_batch_tables(cpg_graph* g, int B) {
    const bool split = batch_split(g->nnz_loc);  // piece length depends on the kernel that runs them
    const int key = B * 2 + (split ? 1 : 0);
    std::lock_guard<std::mutex> lock(g->tab_mu);
    auto it = g->btabs.find(key);
    if (it != g->btabs.end()) return it->second;
    BatchTables bt;
    uint32_t slots = 0;
    const uint32_t C = static_cast<uint32_t>(std::max(1, g->chunks));
    const int64_t hb = split ? batch_piece_edges(B) : batch_hub_edges(B);
    cudaStream_t st = nullptr;
    CPG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    // Column-window pieces (split path, one GPU, B = 16 or 64).  Measured
    // defaults (profiles/r02/cw/): rows above 2048 edges are cut, 48 MB windows, warm tier
    // up to 1 GB of the iterate.  CPG_CW_DEG = min degree of the rows cut (0 = off),
    // CPG_CW_MB = window, CPG_CW_WARM_MB = end of the warm tier, CPG_CW_SPREAD = 1 spreads
    // the uncut pieces over the windows (slower), 2 orders a window's pieces longest first.
    const CwParams cw = cw_params(g, B, split);
    for (uint32_t c = 0; c < C; ++c) {
        ItemTable t;
        t.row_begin = c * g->cr;
        t.row_end = (c + 1) * g->cr;
        if (cw.W && build_cw_hub_items(g->rowptr, g->col, t.row_begin, t.row_end, hb, std::min<int64_t>(hb, cw.hub),
                                       cw.deg, cw.lo, cw.S, cw.W, cw.spread, cw.min_cut, slots, &t, st)) {
            t.n_items = t.n_hub_items;
            slots += t.n_hub_items;
            bt.tables.push_back(t);
            continue;
        }
        build_hub_items(g->rowptr, t.row_begin, t.row_end, hb, hb, slots, &t.items, &t.n_hubs, &t.n_hub_items, 0, st);
        t.n_items = t.n_hub_items;
        slots += t.n_hub_items;
        bt.tables.push_back(t);
    }
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaStreamDestroy(st);
    bt.n_bpartials = slots;
    CPG_CUDA(cudaGetLastError());
    return g->btabs.emplace(key, std::move(bt)).first->second;
}

} // namespace cpg
