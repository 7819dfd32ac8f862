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
__global__ void k_tile_flags(const int64_t* rowptr, uint32_t first, uint32_t n_loc, int64_t chunk, uint32_t max_rows,
                             uint8_t* flags) {
    for (uint64_t j = first + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < n_loc;
         j += (uint64_t)gridDim.x * blockDim.x) {
        bool start = (j == first) || ((j - first) % max_rows == 0) ||
                     (rowptr[j] / chunk != rowptr[j - 1] / chunk);
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

} // namespace

// Work table over local rows [row0, row1): hub pieces (rows with deg > chunk,
// split into `piece`-edge pieces, partial slots from slot_off) then row tiles
// (<= 2*chunk edges, <= max_rows rows).
ItemTable build_item_table(const int64_t* rowptr, uint32_t row0, uint32_t row1, int64_t chunk, uint32_t max_rows,
                           int64_t piece, uint32_t slot_off, cudaStream_t st) {
    DevTemp tmp;
    size_t bytes = 0;
    WorkItem* hub_items = nullptr;
    uint32_t n_hub = 0, n_hub_items = 0;
    build_hub_items(rowptr, row0, row1, chunk, piece, slot_off, &hub_items, &n_hub, &n_hub_items, 0, st);
    uint32_t n_tiles = 0;
    uint32_t* starts = nullptr;
    const uint32_t first = row0 + n_hub;
    if (first < row1) {
        const uint32_t rows = row1 - first;
        uint8_t* flags = dalloc<uint8_t>(rows);
        starts = dalloc<uint32_t>(rows);
        unsigned int* d_sel = dalloc<unsigned int>(1);
        k_tile_flags<<<grid_for(rows), kT, 0, st>>>(rowptr, first, row1, chunk, max_rows, flags);
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
    g->rowptr = dalloc<int64_t>(static_cast<size_t>(n_loc) + 1);
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
        g->col = dalloc<uint32_t>(g->nnz_loc);
        k_extract<<<grid_for(g->nnz_loc), kT, 0, st>>>(keys_sorted, g->nnz_loc, g->col);
        CPG_CUDA(cudaStreamSynchronize(st));
        cudaFree(keys_sorted);
    }
    cudaFree(lold);

    // 5. single-source work table: hub pieces, then row tiles.  Large tiles
    //    when every SM gets >= 8 of them, small tiles otherwise.
    g->tile = g->nnz_loc >= static_cast<uint64_t>(kTileLarge) * g->sm_count * 8 ? kTileLarge : kTileSmall;
    if (const char* force = std::getenv("CPG_TILE")) {  // test hook: exercise either width
        const int t = std::atoi(force);
        if (t == kTileSmall || t == kTileLarge) g->tile = t;
    }
    g->tables.clear();
    uint32_t slots = 0;
    for (uint32_t c = 0; c < C; ++c) {
        ItemTable t = build_item_table(g->rowptr, c * g->cr, (c + 1) * g->cr, g->tile / 2, kTileMaxRows,
                                       kHubPieceEdges, slots, st);
        slots += t.n_hub_items;  // one partial slot per hub piece
        g->tables.push_back(t);
    }
    g->n_partials = slots;
    g->n_items = g->n_hubs = g->n_hub_items = g->n_tiles = 0;
    for (const auto& t : g->tables) {
        g->n_items += t.n_items;
        g->n_hubs += t.n_hubs;
        g->n_hub_items += t.n_hub_items;
        g->n_tiles += t.n_items - t.n_hub_items;
    }
    CPG_CUDA(cudaGetLastError());
}

// Column blocks of the neighbour lists of the CB hubs (rows [row0, row0+n_cb)):
// bnd[h*(nb+1)+b] = first edge of hub h whose column is >= b*S (sorted lists).
__global__ void k_cb_bounds(const int64_t* rowptr, const uint32_t* col, uint32_t row0, uint32_t n_cb, uint32_t S,
                            uint32_t nb, int64_t* bnd) {
    const uint64_t total = static_cast<uint64_t>(n_cb) * (nb + 1);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t h = static_cast<uint32_t>(i / (nb + 1)), b = static_cast<uint32_t>(i % (nb + 1));
        int64_t lo = rowptr[row0 + h], hi = rowptr[row0 + h + 1];
        const uint64_t key = static_cast<uint64_t>(b) * S;
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (col[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        bnd[i] = lo;
    }
}

// Column-blocked hub pieces for the largest hubs of [row0, row1): rows with
// degree > thr are cut at column-block boundaries (blocks of S rows of the
// B-wide iterate, sized to stay L2-resident) and each block segment into
// pieces of <= hb edges.  Pieces are ordered block-major, so the warps in
// flight gather from one window of the iterate at a time.  Returns the number
// of CB rows; items/meta are allocated here (null when none).
static uint32_t build_cb_items(const cpg_graph* g, uint32_t row0, uint32_t row1, int64_t thr, int64_t hb, uint32_t S,
                        uint32_t slot_off, WorkItem** items_out, uint2** meta_out, uint32_t* n_items_out,
                        uint32_t* n_slots_out, cudaStream_t st) {
    *items_out = nullptr;
    *meta_out = nullptr;
    *n_items_out = *n_slots_out = 0;
    const uint32_t n_rows = row1 - row0;
    if (!n_rows) return 0;
    unsigned int* d_cnt = dalloc<unsigned int>(1);
    CPG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned int), st));
    k_count_above<<<grid_for(n_rows), kT, 0, st>>>(g->rowptr + row0, n_rows, thr, d_cnt);
    unsigned int n_cb = 0;
    CPG_CUDA(cudaMemcpyAsync(&n_cb, d_cnt, sizeof(n_cb), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_cnt);
    const uint32_t nb = static_cast<uint32_t>((static_cast<uint64_t>(g->n_pad) + S - 1) / S);
    if (!n_cb || nb < 2) return 0;
    const size_t nbnd = static_cast<size_t>(n_cb) * (nb + 1);
    int64_t* d_bnd = dalloc<int64_t>(nbnd);
    k_cb_bounds<<<grid_for(nbnd), kT, 0, st>>>(g->rowptr, g->col, row0, n_cb, S, nb, d_bnd);
    std::vector<int64_t> bnd(nbnd);
    CPG_CUDA(cudaMemcpyAsync(bnd.data(), d_bnd, sizeof(int64_t) * nbnd, cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_bnd);
    // per hub: pieces per block, first slot, piece count
    std::vector<uint32_t> first_piece(nbnd);  // piece index of (h, b) within hub h
    std::vector<uint2> meta(n_cb);
    uint32_t slots = slot_off;
    uint64_t n_items = 0;
    for (uint32_t h = 0; h < n_cb; ++h) {
        const int64_t* bh = bnd.data() + static_cast<size_t>(h) * (nb + 1);
        uint32_t p = 0;
        for (uint32_t b = 0; b < nb; ++b) {
            first_piece[static_cast<size_t>(h) * (nb + 1) + b] = p;
            p += static_cast<uint32_t>((bh[b + 1] - bh[b] + hb - 1) / hb);
        }
        meta[h] = make_uint2(slots, p);
        slots += p;
        n_items += p;
    }
    if (n_items > 0xffffffffull) throw Error(CPG_ENOMEM, "column-blocked hub pieces overflow");
    std::vector<WorkItem> items;
    items.reserve(n_items);
    for (uint32_t b = 0; b < nb; ++b)
        for (uint32_t h = 0; h < n_cb; ++h) {
            const size_t i = static_cast<size_t>(h) * (nb + 1) + b;
            const int64_t e_begin = bnd[i], e_end = bnd[i + 1];
            uint32_t slot = meta[h].x + first_piece[i];
            for (int64_t e = e_begin; e < e_end; e += hb, ++slot) {
                const uint32_t cnt = static_cast<uint32_t>(std::min<int64_t>(hb, e_end - e));
                items.push_back(WorkItem{row0 + h, slot, tile_code(static_cast<uint64_t>(e), cnt, 0) | kHubBit | kCbBit});
            }
        }
    WorkItem* d_items = dalloc<WorkItem>(items.size());
    uint2* d_meta = dalloc<uint2>(n_cb);
    CPG_CUDA(cudaMemcpyAsync(d_items, items.data(), sizeof(WorkItem) * items.size(), cudaMemcpyHostToDevice, st));
    CPG_CUDA(cudaMemcpyAsync(d_meta, meta.data(), sizeof(uint2) * n_cb, cudaMemcpyHostToDevice, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    *items_out = d_items;
    *meta_out = d_meta;
    *n_items_out = static_cast<uint32_t>(items.size());
    *n_slots_out = slots - slot_off;
    if (std::getenv("CPG_CB_DEBUG")) {
        const int64_t e0 = bnd[0], e1 = bnd[nbnd - 1];
        std::fprintf(stderr, "[cpg] column-blocked hubs: rows %u (deg > %lld), blocks %u x %u rows, pieces %zu, edges %lld\n",
                     n_cb, static_cast<long long>(thr), nb, S, items.size(), static_cast<long long>(e1 - e0));
    }
    return n_cb;
}

// Column-blocking parameters: CPG_CB_DEG (min degree, 0 = off), CPG_CB_MB
// (window of the iterate, MB).
static int64_t cb_min_degree() {
    const char* e = std::getenv("CPG_CB_DEG");
    return e ? std::atoll(e) : 32768;
}
static uint32_t cb_rows(int B) {
    const char* e = std::getenv("CPG_CB_MB");
    const double mb = e ? std::atof(e) : 48.0;
    return static_cast<uint32_t>(std::max(1024.0, mb * 1048576.0 / (8.0 * B)));
}

// Sweep bounds: for row rank i of the sweep range (launch l = i / cap, rank j
// in the launch) and block boundary b, the first edge of the row whose column
// is >= b*S, relative to the row start.  Written at the kernel's position of
// the row: j -> (p = j / (G*SL), slot sl, CTA snake(c)) as in
// cheby_batch_sweep_kernel.
__global__ void k_sweep_bounds(const int64_t* rowptr, const uint32_t* col, uint32_t row0, uint32_t n_rows, uint32_t S,
                               uint32_t nb, uint32_t G, uint32_t SL, uint32_t cap, uint32_t* out) {
    const uint64_t total = static_cast<uint64_t>(n_rows) * (nb + 1);
    for (uint64_t x = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; x < total; x += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = static_cast<uint32_t>(x / (nb + 1)), b = static_cast<uint32_t>(x % (nb + 1));
        const int64_t rs = rowptr[row0 + i], re = rowptr[row0 + i + 1];
        int64_t lo = rs, hi = re;
        const uint64_t key = static_cast<uint64_t>(b) * S;
        if (b == nb) lo = re;
        while (lo < hi) {
            const int64_t mid = lo + (hi - lo) / 2;
            if (col[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        const uint32_t l = i / cap, j = i % cap;
        const uint32_t p = j / (G * SL), r = j % (G * SL);
        const uint32_t sl = r / G, c = r % G;
        const uint32_t cta = (sl & 1) ? G - 1 - c : c;
        const size_t pos = ((static_cast<size_t>(l) * (nb + 1) + b) * G + cta) * SL * kSweepRows +
                           static_cast<size_t>(sl) * kSweepRows + p;
        out[pos] = static_cast<uint32_t>(lo - rs);
    }
}

// Rows of [row0, row1) with degree > thr (a prefix: rows are degree-descending).
static uint32_t count_prefix_above(const int64_t* rowptr, uint32_t row0, uint32_t row1, int64_t thr, cudaStream_t st) {
    const uint32_t n_rows = row1 - row0;
    if (!n_rows) return 0;
    unsigned int* d_cnt = dalloc<unsigned int>(1);
    CPG_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned int), st));
    k_count_above<<<grid_for(n_rows), kT, 0, st>>>(rowptr + row0, n_rows, thr, d_cnt);
    unsigned int n = 0;
    CPG_CUDA(cudaMemcpyAsync(&n, d_cnt, sizeof(n), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(d_cnt);
    return n;
}

// Column-sweep setting: CPG_SWEEP=0/1 forces it off/on (default: on when the
// B-wide iterate is >= 512 MB, i.e. far larger than L2); CPG_SWEEP_MB is the
// column window (MB of the iterate), CPG_SWEEP_DEG the minimum degree.
static bool sweep_enabled(const cpg_graph* g, int B) {
    const char* e = std::getenv("CPG_SWEEP");
    (void)g;
    (void)B;
    return e && e[0] != '0';
}
static uint32_t sweep_rows_per_block(int B) {
    const char* e = std::getenv("CPG_SWEEP_MB");
    const double mb = e ? std::atof(e) : 40.0;
    return static_cast<uint32_t>(std::max(256.0, mb * 1048576.0 / (8.0 * B)));
}
static int64_t sweep_min_degree(int B) {
    const char* e = std::getenv("CPG_SWEEP_DEG");
    return e ? std::atoll(e) : batch_hub_edges(B);
}

static void build_sweep(const cpg_graph* g, ItemTable& t, uint32_t n_sw, int B, cudaStream_t st) {
    t.n_sw = n_sw;
    if (!n_sw) return;
    const uint32_t S = sweep_rows_per_block(B);
    t.sw_nb = static_cast<uint32_t>((static_cast<uint64_t>(g->n_pad) + S - 1) / S);
    t.sw_grid = sweep_grid(B);
    const uint32_t SL = static_cast<uint32_t>(sweep_slots_per_cta(B));
    t.sw_cap = static_cast<uint32_t>(t.sw_grid) * SL * kSweepRows;
    t.sw_launches = (n_sw + t.sw_cap - 1) / t.sw_cap;
    const size_t n_bnd = static_cast<size_t>(t.sw_launches) * (t.sw_nb + 1) * t.sw_cap;
    t.sw_bnd = dalloc<uint32_t>(n_bnd);
    t.sw_cnt = dalloc<unsigned int>(static_cast<size_t>(t.sw_launches) * t.sw_nb);
    CPG_CUDA(cudaMemsetAsync(t.sw_bnd, 0, sizeof(uint32_t) * n_bnd, st));
    k_sweep_bounds<<<grid_for(static_cast<uint64_t>(n_sw) * (t.sw_nb + 1)), kT, 0, st>>>(
        g->rowptr, g->col, t.sw_begin, n_sw, S, t.sw_nb, static_cast<uint32_t>(t.sw_grid), SL, t.sw_cap, t.sw_bnd);
    CPG_CUDA(cudaStreamSynchronize(st));
    if (std::getenv("CPG_CB_DEBUG"))
        std::fprintf(stderr, "[cpg] column sweep: rows %u, blocks %u x %u rows, grid %d, %u launches of %u rows\n",
                     n_sw, t.sw_nb, S, t.sw_grid, t.sw_launches, t.sw_cap);
}

void ensure_batch_tables(cpg_graph* g, int B) {
    if (!g->btables.empty() && g->bitems_width == B) return;
    for (auto& t : g->btables)
        for (void* p : {(void*)t.items, (void*)t.cb_meta, (void*)t.sw_bnd, (void*)t.sw_cnt})
            if (p) cudaFree(p);
    g->btables.clear();
    uint32_t slots = 0;
    const uint32_t C = static_cast<uint32_t>(std::max(1, g->chunks));
    const int64_t hb = batch_hub_edges(B);
    const int64_t cb_deg = cb_min_degree();
    for (uint32_t c = 0; c < C; ++c) {
        ItemTable t;
        t.row_begin = c * g->cr;
        t.row_end = (c + 1) * g->cr;
        WorkItem* cb_items = nullptr;
        uint32_t cb_slots = 0;
        if (cb_deg > 0)
            t.n_cb = build_cb_items(g, t.row_begin, t.row_end, std::max<int64_t>(cb_deg - 1, hb), hb, cb_rows(B), slots,
                                    &cb_items, &t.cb_meta, &t.n_cb_items, &cb_slots, g->stream);
        slots += cb_slots;
        t.sw_begin = t.row_begin + t.n_cb;
        if (sweep_enabled(g, B))
            build_sweep(g, t,
                        count_prefix_above(g->rowptr, t.sw_begin, t.row_end,
                                           std::max<int64_t>(sweep_min_degree(B), 0), g->stream),
                        B, g->stream);
        WorkItem* rest = nullptr;
        uint32_t n_rest_hubs = 0, n_rest_items = 0;
        build_hub_items(g->rowptr, t.sw_begin + t.n_sw, t.row_end, hb, hb, slots, &rest, &n_rest_hubs,
                        &n_rest_items, 0, g->stream);
        slots += n_rest_items;
        t.n_hubs = t.n_cb + t.n_sw + n_rest_hubs;
        t.n_hub_items = t.n_cb_items + n_rest_items;
        if (t.n_cb_items) {
            t.items = dalloc<WorkItem>(t.n_hub_items);
            CPG_CUDA(cudaMemcpyAsync(t.items, cb_items, sizeof(WorkItem) * t.n_cb_items, cudaMemcpyDeviceToDevice,
                                     g->stream));
            if (n_rest_items)
                CPG_CUDA(cudaMemcpyAsync(t.items + t.n_cb_items, rest, sizeof(WorkItem) * n_rest_items,
                                         cudaMemcpyDeviceToDevice, g->stream));
            CPG_CUDA(cudaStreamSynchronize(g->stream));
            cudaFree(cb_items);
            cudaFree(rest);
        } else {
            t.items = rest;
        }
        t.n_items = t.n_hub_items;
        g->btables.push_back(t);
    }
    g->n_bpartials = slots;
    g->bitems_width = B;
    CPG_CUDA(cudaGetLastError());
}

} // namespace cpg
