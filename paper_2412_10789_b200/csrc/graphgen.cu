// graphgen.cu -- seeded synthetic inputs for the parity tests and the bench
// (stand-ins for the paper's SNAP datasets).  Not the hot path.
//
// Every edge draw is addressed by its sample index i through
// SplitMix64::stream(seed, i) (include/chebyprop/rng.hpp:30-35 semantics), so
// the host build (device = -1) and the device build produce the same CSR:
// both symmetrise, drop self-loops, sort, deduplicate and compact isolated ids
// in ascending order -- the invariants Graph::from_csr demands
// (graph.cpp:48-104).
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

#include "cpg_common.hpp"

namespace cpg {
namespace {

__host__ __device__ __forceinline__ uint64_t sm_next(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ull);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ double sm_double(uint64_t& s) {
    return static_cast<double>(sm_next(s) >> 11) * 0x1.0p-53;
}
__host__ __device__ __forceinline__ uint64_t sm_stream(uint64_t seed, uint64_t tag) {
    uint64_t s = seed ^ (0x9e3779b97f4a7c15ull * (tag + 1));
    sm_next(s);
    return s;
}

constexpr uint64_t kLoop = ~0ull;  // self-loop sentinel (sorts last)

// R-MAT: per level pick a quadrant with probabilities (a, b, c, d).
__host__ __device__ __forceinline__ void rmat_pair(uint64_t seed, uint64_t i, uint32_t scale, double a, double ab,
                                                   double abc, uint64_t& k1, uint64_t& k2) {
    uint64_t s = sm_stream(seed, i);
    uint32_t u = 0, v = 0;
    for (uint32_t l = 0; l < scale; ++l) {
        const double r = sm_double(s);
        const uint32_t bu = r >= ab ? 1u : 0u;
        const uint32_t bv = (r >= a && r < ab) || r >= abc ? 1u : 0u;
        u = (u << 1) | bu;
        v = (v << 1) | bv;
    }
    if (u == v) {
        k1 = k2 = kLoop;
    } else {
        k1 = (static_cast<uint64_t>(u) << 32) | v;
        k2 = (static_cast<uint64_t>(v) << 32) | u;
    }
}

// Chung-Lu: both endpoints drawn proportionally to w (inverse CDF search).
__host__ __device__ __forceinline__ uint32_t cdf_search(const double* cdf, uint32_t n, double x) {
    uint32_t lo = 0, hi = n - 1;  // first i with cdf[i] > x
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (cdf[mid] > x) hi = mid; else lo = mid + 1;
    }
    return lo;
}
__host__ __device__ __forceinline__ void chunglu_pair(uint64_t seed, uint64_t i, const double* cdf, uint32_t n,
                                                      uint64_t& k1, uint64_t& k2) {
    uint64_t s = sm_stream(seed, i);
    const double total = cdf[n - 1];
    const uint32_t u = cdf_search(cdf, n, sm_double(s) * total);
    const uint32_t v = cdf_search(cdf, n, sm_double(s) * total);
    if (u == v) {
        k1 = k2 = kLoop;
    } else {
        k1 = (static_cast<uint64_t>(u) << 32) | v;
        k2 = (static_cast<uint64_t>(v) << 32) | u;
    }
}

__global__ void k_rmat(uint64_t seed, uint64_t m, uint32_t scale, double a, double ab, double abc, uint64_t* keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        rmat_pair(seed, i, scale, a, ab, abc, keys[2 * i], keys[2 * i + 1]);
}

__global__ void k_chunglu(uint64_t seed, uint64_t m, const double* cdf, uint32_t n, uint64_t* keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x)
        chunglu_pair(seed, i, cdf, n, keys[2 * i], keys[2 * i + 1]);
}

__global__ void k_mark(const uint64_t* keys, uint64_t nnz, uint32_t* present) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz; e += (uint64_t)gridDim.x * blockDim.x)
        present[keys[e] >> 32] = 1u;
}

__global__ void k_csr(const uint64_t* keys, uint64_t nnz, const uint32_t* newid, uint64_t* off, uint32_t* nbr,
                      uint32_t n) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < nnz; e += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t u = static_cast<uint32_t>(keys[e] >> 32);
        nbr[e] = newid[static_cast<uint32_t>(keys[e] & 0xffffffffu)];
        if (e == 0 || (keys[e - 1] >> 32) != u) off[newid[u]] = e;
        if (e == 0) off[n] = nnz;
    }
}

int grid_for(uint64_t n) { return static_cast<int>(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 32))); }

// Shared tail: keys (2m, unsorted) -> CSR.  Device path.
void keys_to_csr_device(uint64_t* keys, uint64_t nk, uint32_t id_space, uint32_t id_bits, uint64_t** off_out,
                        uint32_t** nbr_out, uint32_t* n_out, uint64_t* nnz_out) {
    cudaStream_t st = 0;
    uint64_t* sorted = nullptr;
    CPG_CUDA(cudaMalloc(&sorted, nk * sizeof(uint64_t)));
    void* tmp = nullptr;
    size_t bytes = 0;
    cub::DeviceRadixSort::SortKeys(nullptr, bytes, keys, sorted, nk, 0, 64, st);
    CPG_CUDA(cudaMalloc(&tmp, bytes));
    CPG_CUDA(cub::DeviceRadixSort::SortKeys(tmp, bytes, keys, sorted, nk, 0, 64, st));
    cudaFree(tmp);
    uint64_t* d_cnt = nullptr;
    CPG_CUDA(cudaMalloc(&d_cnt, sizeof(uint64_t)));
    bytes = 0;
    cub::DeviceSelect::Unique(nullptr, bytes, sorted, keys, d_cnt, nk, st);
    CPG_CUDA(cudaMalloc(&tmp, bytes));
    CPG_CUDA(cub::DeviceSelect::Unique(tmp, bytes, sorted, keys, d_cnt, nk, st));
    cudaFree(tmp);
    cudaFree(sorted);
    uint64_t nu = 0, last = 0;
    CPG_CUDA(cudaMemcpy(&nu, d_cnt, sizeof(nu), cudaMemcpyDeviceToHost));
    cudaFree(d_cnt);
    if (nu) CPG_CUDA(cudaMemcpy(&last, keys + nu - 1, sizeof(last), cudaMemcpyDeviceToHost));
    if (nu && last == kLoop) --nu;
    require(nu > 0, "generator produced an empty graph");
    uint32_t *present = nullptr, *newid = nullptr;
    CPG_CUDA(cudaMalloc(&present, (static_cast<size_t>(id_space) + 1) * sizeof(uint32_t)));
    CPG_CUDA(cudaMalloc(&newid, (static_cast<size_t>(id_space) + 1) * sizeof(uint32_t)));
    CPG_CUDA(cudaMemset(present, 0, (static_cast<size_t>(id_space) + 1) * sizeof(uint32_t)));
    k_mark<<<grid_for(nu), 256, 0, st>>>(keys, nu, present);
    bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, bytes, present, newid, id_space + 1, st);
    CPG_CUDA(cudaMalloc(&tmp, bytes));
    CPG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, bytes, present, newid, id_space + 1, st));
    cudaFree(tmp);
    uint32_t n = 0;
    CPG_CUDA(cudaMemcpy(&n, newid + id_space, sizeof(n), cudaMemcpyDeviceToHost));
    uint64_t* off = nullptr;
    uint32_t* nbr = nullptr;
    CPG_CUDA(cudaMalloc(&off, (static_cast<size_t>(n) + 1) * sizeof(uint64_t)));
    CPG_CUDA(cudaMalloc(&nbr, nu * sizeof(uint32_t)));
    k_csr<<<grid_for(nu), 256, 0, st>>>(keys, nu, newid, off, nbr, n);
    CPG_CUDA(cudaDeviceSynchronize());
    CPG_CUDA(cudaGetLastError());
    cudaFree(present);
    cudaFree(newid);
    (void)id_bits;
    *off_out = off;
    *nbr_out = nbr;
    *n_out = n;
    *nnz_out = nu;
}

// Host path (tests / small graphs): identical keys -> identical CSR.
void keys_to_csr_host(std::vector<uint64_t>& keys, uint32_t id_space, uint64_t** off_out, uint32_t** nbr_out,
                      uint32_t* n_out, uint64_t* nnz_out) {
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    if (!keys.empty() && keys.back() == kLoop) keys.pop_back();
    require(!keys.empty(), "generator produced an empty graph");
    std::vector<uint32_t> newid(static_cast<size_t>(id_space) + 1, 0);
    for (uint64_t k : keys) newid[k >> 32] = 1;
    uint32_t n = 0;
    for (size_t i = 0; i <= id_space; ++i) {
        const uint32_t p = newid[i];
        newid[i] = n;
        n += p;
    }
    const uint64_t nnz = keys.size();
    auto* off = static_cast<uint64_t*>(std::malloc((static_cast<size_t>(n) + 1) * sizeof(uint64_t)));
    auto* nbr = static_cast<uint32_t*>(std::malloc(std::max<uint64_t>(1, nnz) * sizeof(uint32_t)));
    if (!off || !nbr) fail(CPG_ENOMEM, "host generator out of memory");
    for (uint64_t e = 0; e < nnz; ++e) {
        const uint32_t u = static_cast<uint32_t>(keys[e] >> 32);
        nbr[e] = newid[static_cast<uint32_t>(keys[e] & 0xffffffffu)];
        if (e == 0 || (keys[e - 1] >> 32) != u) off[newid[u]] = e;
    }
    off[n] = nnz;
    *off_out = off;
    *nbr_out = nbr;
    *n_out = n;
    *nnz_out = nnz;
}

template <typename F>
void host_fill(std::vector<uint64_t>& keys, uint64_t m, F&& pair) {
    keys.resize(2 * m);
    const unsigned nt = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    std::vector<std::thread> th;
    for (unsigned t = 0; t < nt; ++t)
        th.emplace_back([&, t] {
            for (uint64_t i = t; i < m; i += nt) pair(i, keys[2 * i], keys[2 * i + 1]);
        });
    for (auto& x : th) x.join();
}

// Expected-degree weights w_i ~ (i + 1)^(-1/(gamma-1)), scaled to the target
// mean degree with the cap enforced (a few rescale rounds), as a CDF.
std::vector<double> chunglu_cdf(uint32_t n, double exponent, double mean_degree, uint32_t max_degree) {
    require(exponent > 1.0, "chung-lu exponent must exceed 1");
    std::vector<double> w(n);
    const double beta = 1.0 / (exponent - 1.0);
    for (uint32_t i = 0; i < n; ++i) w[i] = std::pow(static_cast<double>(i) + 1.0, -beta);
    const double target = mean_degree * n;
    for (int round = 0; round < 50; ++round) {
        double sum = 0.0;
        for (double x : w) sum += x;
        const double s = target / sum;
        bool capped = false;
        for (double& x : w) {
            x *= s;
            if (max_degree && x > max_degree) {
                x = max_degree;
                capped = true;
            }
        }
        if (!capped) break;
    }
    std::vector<double> cdf(n);
    double acc = 0.0;
    for (uint32_t i = 0; i < n; ++i) cdf[i] = (acc += w[i]);
    return cdf;
}

// ---- GPU ingest: the reference's load_edge_list semantics (graph.cpp:113-171) ----
// Self-loops dropped (:149); labels interned in first-seen order over the
// surviving edges, a before b (:120-124, :150-151); symmetrised (:152-153);
// sorted and deduplicated (:158-160).
__global__ void k_keep(const int64_t* pairs, uint64_t m, uint8_t* keep) {
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < m; e += (uint64_t)gridDim.x * blockDim.x)
        keep[e] = pairs[2 * e] != pairs[2 * e + 1];
}

// endpoint j of kept edge i: key = label with the sign bit flipped (unsigned order = signed order),
// value = position 2i + side (first-seen order).
__global__ void k_endpoints(const int64_t* pairs, const uint64_t* kept, uint64_t mk, uint64_t* key, uint64_t* pos) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < mk; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t e = kept[i];
        key[2 * i] = static_cast<uint64_t>(pairs[2 * e]) ^ 0x8000000000000000ull;
        key[2 * i + 1] = static_cast<uint64_t>(pairs[2 * e + 1]) ^ 0x8000000000000000ull;
        pos[2 * i] = 2 * i;
        pos[2 * i + 1] = 2 * i + 1;
    }
}

// run heads of the label-sorted endpoints: head[j] = 1 if a new label starts at j
__global__ void k_heads(const uint64_t* key, uint64_t cnt, uint32_t* head) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < cnt; j += (uint64_t)gridDim.x * blockDim.x)
        head[j] = (j == 0 || key[j] != key[j - 1]) ? 1u : 0u;
}

// for each run head (unique label u = run index = run[j] - 1): first position and label
__global__ void k_uniques(const uint64_t* key, const uint64_t* pos, const uint32_t* head, const uint32_t* run,
                          uint64_t cnt, uint64_t* first_pos, uint64_t* label) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < cnt; j += (uint64_t)gridDim.x * blockDim.x)
        if (head[j]) {
            first_pos[run[j] - 1] = pos[j];  // stable sort: the run's first entry has the smallest position
            label[run[j] - 1] = key[j];
        }
}

__global__ void k_iota32(uint32_t* v, uint32_t n) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] = i;
}

// id_of[run] = rank of the run's first position
__global__ void k_rank(const uint32_t* run_by_pos, uint32_t n, uint32_t* id_of) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) id_of[run_by_pos[r]] = r;
}

__global__ void k_endpoint_ids(const uint64_t* pos, const uint32_t* run, const uint32_t* id_of, uint64_t cnt,
                               uint32_t* id_at) {
    for (uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; j < cnt; j += (uint64_t)gridDim.x * blockDim.x)
        id_at[pos[j]] = id_of[run[j] - 1];
}

__global__ void k_edge_keys(const uint32_t* id_at, uint64_t mk, uint64_t* keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < mk; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t u = id_at[2 * i], v = id_at[2 * i + 1];
        keys[2 * i] = (u << 32) | v;
        keys[2 * i + 1] = (v << 32) | u;
    }
}

__global__ void k_labels_in_id_order(const uint64_t* label, const uint32_t* run_by_pos, uint32_t n, int64_t* out) {
    for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x)
        out[r] = static_cast<int64_t>(label[run_by_pos[r]] ^ 0x8000000000000000ull);
}

template <typename F>
void cub_call(F&& f, cudaStream_t st) {
    size_t bytes = 0;
    f(nullptr, bytes);
    void* tmp = nullptr;
    CPG_CUDA(cudaMalloc(&tmp, std::max<size_t>(bytes, 1)));
    f(tmp, bytes);
    CPG_CUDA(cudaStreamSynchronize(st));
    cudaFree(tmp);
}

template <typename T>
T* dm(size_t count) {
    T* p = nullptr;
    CPG_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
    return p;
}

void ingest_device(const int64_t* d_pairs, uint64_t m, uint64_t** off_out, uint32_t** nbr_out, uint32_t* n_out,
                   uint64_t* nnz_out, int64_t** labels_out) {
    cudaStream_t st = 0;
    uint8_t* keep = dm<uint8_t>(m);
    uint64_t* kept = dm<uint64_t>(m);
    uint64_t* d_cnt = dm<uint64_t>(1);
    k_keep<<<grid_for(m), 256, 0, st>>>(d_pairs, m, keep);
    cub::CountingInputIterator<uint64_t> iota(0);
    cub_call([&](void* t, size_t& b) { cub::DeviceSelect::Flagged(t, b, iota, keep, kept, d_cnt, m, st); }, st);
    uint64_t mk = 0;
    CPG_CUDA(cudaMemcpy(&mk, d_cnt, sizeof(mk), cudaMemcpyDeviceToHost));
    cudaFree(keep);
    if (mk == 0) fail(CPG_ESTRUCT, "empty graph after cleaning");  // graph.cpp:156 (StructuralError)
    const uint64_t cnt = 2 * mk;
    uint64_t *key = dm<uint64_t>(cnt), *pos = dm<uint64_t>(cnt), *key_s = dm<uint64_t>(cnt), *pos_s = dm<uint64_t>(cnt);
    k_endpoints<<<grid_for(mk), 256, 0, st>>>(d_pairs, kept, mk, key, pos);
    cudaFree(kept);
    cub_call([&](void* t, size_t& b) { cub::DeviceRadixSort::SortPairs(t, b, key, key_s, pos, pos_s, cnt, 0, 64, st); },
             st);
    cudaFree(key);
    cudaFree(pos);
    uint32_t *head = dm<uint32_t>(cnt), *run = dm<uint32_t>(cnt);
    k_heads<<<grid_for(cnt), 256, 0, st>>>(key_s, cnt, head);
    // run[j] = number of run heads in [0, j] = 1 + run index of endpoint j
    cub_call([&](void* t, size_t& b) { cub::DeviceScan::InclusiveSum(t, b, head, run, cnt, st); }, st);
    uint32_t n = 0;
    CPG_CUDA(cudaMemcpy(&n, run + cnt - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost));
    uint64_t *first_pos = dm<uint64_t>(n), *label = dm<uint64_t>(n), *first_pos_s = dm<uint64_t>(n);
    k_uniques<<<grid_for(cnt), 256, 0, st>>>(key_s, pos_s, head, run, cnt, first_pos, label);
    cudaFree(head);
    // order the labels by first appearance: id = rank of first position
    uint32_t *runs = dm<uint32_t>(n), *run_by_pos = dm<uint32_t>(n), *id_of = dm<uint32_t>(n);
    k_iota32<<<grid_for(n), 256, 0, st>>>(runs, n);
    cub_call([&](void* t, size_t& b) {
        cub::DeviceRadixSort::SortPairs(t, b, first_pos, first_pos_s, runs, run_by_pos, n, 0, 64, st);
    }, st);
    k_rank<<<grid_for(n), 256, 0, st>>>(run_by_pos, n, id_of);
    uint32_t* id_at = dm<uint32_t>(cnt);
    k_endpoint_ids<<<grid_for(cnt), 256, 0, st>>>(pos_s, run, id_of, cnt, id_at);
    int64_t* labels = dm<int64_t>(n);
    k_labels_in_id_order<<<grid_for(n), 256, 0, st>>>(label, run_by_pos, n, labels);
    CPG_CUDA(cudaDeviceSynchronize());
    for (void* p : {(void*)key_s, (void*)pos_s, (void*)run, (void*)first_pos, (void*)label, (void*)first_pos_s,
                    (void*)runs, (void*)run_by_pos, (void*)id_of})
        cudaFree(p);
    uint64_t* keys = dm<uint64_t>(cnt);
    k_edge_keys<<<grid_for(mk), 256, 0, st>>>(id_at, mk, keys);
    cudaFree(id_at);
    cudaFree(d_cnt);
    try {
        keys_to_csr_device(keys, cnt, n, 32, off_out, nbr_out, n_out, nnz_out);
    } catch (...) {
        cudaFree(keys);
        cudaFree(labels);
        throw;
    }
    cudaFree(keys);
    require(*n_out == n, "ingest: id compaction mismatch");
    *labels_out = labels;
}

} // namespace
} // namespace cpg

using namespace cpg;

extern "C" {

int cpg_gen_rmat(uint32_t scale, uint64_t n_samples, double a, double b, double c, uint64_t seed, int device,
                 uint64_t** offsets, uint32_t** neighbors, uint32_t* n, uint64_t* nnz) {
    return guarded([&] {
        require(scale >= 1 && scale <= 31, "rmat scale must be in [1, 31]");
        require(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0, "rmat probabilities");
        require(offsets && neighbors && n && nnz, "null argument");
        const double ab = a + b, abc = a + b + c;
        const uint32_t ids = 1u << scale;
        if (device < 0) {
            std::vector<uint64_t> keys;
            host_fill(keys, n_samples, [&](uint64_t i, uint64_t& k1, uint64_t& k2) {
                rmat_pair(seed, i, scale, a, ab, abc, k1, k2);
            });
            keys_to_csr_host(keys, ids, offsets, neighbors, n, nnz);
            return;
        }
        CPG_CUDA(cudaSetDevice(device));
        uint64_t* keys = nullptr;
        CPG_CUDA(cudaMalloc(&keys, 2 * n_samples * sizeof(uint64_t)));
        k_rmat<<<grid_for(n_samples), 256>>>(seed, n_samples, scale, a, ab, abc, keys);
        CPG_CUDA(cudaGetLastError());
        try {
            keys_to_csr_device(keys, 2 * n_samples, ids, scale, offsets, neighbors, n, nnz);
        } catch (...) {
            cudaFree(keys);
            throw;
        }
        cudaFree(keys);
    });
}

int cpg_gen_chunglu(uint32_t n_ids, uint64_t n_samples, double exponent, double mean_degree, uint32_t max_degree,
                    uint64_t seed, int device, uint64_t** offsets, uint32_t** neighbors, uint32_t* n, uint64_t* nnz) {
    return guarded([&] {
        require(n_ids >= 2, "chung-lu needs at least two ids");
        require(offsets && neighbors && n && nnz, "null argument");
        const std::vector<double> cdf = chunglu_cdf(n_ids, exponent, mean_degree, max_degree);
        if (device < 0) {
            std::vector<uint64_t> keys;
            host_fill(keys, n_samples, [&](uint64_t i, uint64_t& k1, uint64_t& k2) {
                chunglu_pair(seed, i, cdf.data(), n_ids, k1, k2);
            });
            keys_to_csr_host(keys, n_ids, offsets, neighbors, n, nnz);
            return;
        }
        CPG_CUDA(cudaSetDevice(device));
        double* d_cdf = nullptr;
        uint64_t* keys = nullptr;
        CPG_CUDA(cudaMalloc(&d_cdf, n_ids * sizeof(double)));
        CPG_CUDA(cudaMemcpy(d_cdf, cdf.data(), n_ids * sizeof(double), cudaMemcpyHostToDevice));
        CPG_CUDA(cudaMalloc(&keys, 2 * n_samples * sizeof(uint64_t)));
        k_chunglu<<<grid_for(n_samples), 256>>>(seed, n_samples, d_cdf, n_ids, keys);
        CPG_CUDA(cudaGetLastError());
        cudaFree(d_cdf);
        try {
            keys_to_csr_device(keys, 2 * n_samples, n_ids, 32, offsets, neighbors, n, nnz);
        } catch (...) {
            cudaFree(keys);
            throw;
        }
        cudaFree(keys);
    });
}

int cpg_csr_to_host(const uint64_t* d_offsets, const uint32_t* d_neighbors, uint32_t n, uint64_t nnz, int device,
                    uint64_t* offsets, uint32_t* neighbors) {
    return guarded([&] {
        require(d_offsets && d_neighbors && offsets && neighbors, "null argument");
        CPG_CUDA(cudaSetDevice(device));
        CPG_CUDA(cudaMemcpy(offsets, d_offsets, (static_cast<size_t>(n) + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost));
        CPG_CUDA(cudaMemcpy(neighbors, d_neighbors, nnz * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    });
}

int cpg_ingest_edges(const int64_t* pairs, uint64_t m, int device, uint64_t** offsets, uint32_t** neighbors,
                     uint32_t* n, uint64_t* nnz, int64_t* original_ids_host, uint64_t original_ids_cap) {
    return guarded([&] {
        require((pairs || m == 0) && offsets && neighbors && n && nnz, "null argument");
        require(device >= 0, "ingest runs on a device");
        CPG_CUDA(cudaSetDevice(device));
        int64_t* d_pairs = nullptr;
        CPG_CUDA(cudaMalloc(&d_pairs, std::max<uint64_t>(1, 2 * m) * sizeof(int64_t)));
        CPG_CUDA(cudaMemcpy(d_pairs, pairs, 2 * m * sizeof(int64_t), cudaMemcpyHostToDevice));
        int64_t* labels = nullptr;
        try {
            if (m == 0) fail(CPG_ESTRUCT, "empty graph after cleaning");  // graph.cpp:156
            ingest_device(d_pairs, m, offsets, neighbors, n, nnz, &labels);
        } catch (...) {
            cudaFree(d_pairs);
            throw;
        }
        cudaFree(d_pairs);
        if (original_ids_host) {
            require(original_ids_cap >= *n, "original_ids buffer too small");
            CPG_CUDA(cudaMemcpy(original_ids_host, labels, *n * sizeof(int64_t), cudaMemcpyDeviceToHost));
        }
        cudaFree(labels);
    });
}

int cpg_free_csr(uint64_t* offsets, uint32_t* neighbors, int device) {
    return guarded([&] {
        if (device < 0) {
            std::free(offsets);
            std::free(neighbors);
        } else {
            CPG_CUDA(cudaSetDevice(device));
            if (offsets) CPG_CUDA(cudaFree(offsets));
            if (neighbors) CPG_CUDA(cudaFree(neighbors));
        }
    });
}

} // extern "C"
