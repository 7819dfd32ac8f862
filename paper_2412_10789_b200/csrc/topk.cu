// topk.cu -- device top-k of a score vector.
//
// The reference's query path ranks the full score vector on the host
// (tools/chebyprop.cpp:148-156: partial_sort by value desc, id asc, top-50)
// after the whole n-vector is materialised.  Here the ranking runs on the
// device, so only k (id, value) pairs cross PCIe:
//   1. histogram of the top 16 bits of an order-preserving 64-bit key;
//   2. one block finds the bin holding the k-th largest key;
//   3. cub::DeviceSelect keeps every element at or above that bin, in id
//      order (deterministic), and a stable descending radix sort of the
//      candidates by value gives (value desc, id asc), the reference's order.
// If the threshold bin holds too many elements (massive ties), a stable sort
// of the whole vector is used instead.  All columns of a query group share one
// histogram pass, one host synchronisation and one scratch allocation.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "cpg_graph.hpp"

namespace cpg {
namespace {

__device__ __forceinline__ uint64_t order_key(double v) {
    uint64_t b;
    memcpy(&b, &v, sizeof(b));
    return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);  // ascending <=> value ascending
}

__global__ void k_hist16(const double* vals, uint32_t n, unsigned int* hist) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&hist[order_key(vals[i]) >> 48], 1u);
}

// Single block: bin b* such that count(bins > b*) < k <= count(bins >= b*).
__global__ void k_threshold(const unsigned int* hist, uint32_t k, unsigned int* out_bin, unsigned int* out_count) {
    if (threadIdx.x != 0) return;
    uint64_t acc = 0;
    for (int b = (1 << 16) - 1; b >= 0; --b) {
        acc += hist[b];
        if (acc >= k || b == 0) {
            *out_bin = static_cast<unsigned int>(b);
            *out_count = static_cast<unsigned int>(acc);
            return;
        }
    }
}

struct AtLeastBin {
    const double* vals;
    unsigned int bin;
    __device__ bool operator()(uint32_t i) const { return (order_key(vals[i]) >> 48) >= bin; }
};

__global__ void k_gather_vals(const double* vals, const uint32_t* ids, uint32_t m, double* out) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) out[i] = vals[ids[i]];
}

template <typename T>
T* dmalloc(size_t count) {
    T* p = nullptr;
    CPG_CUDA(cudaMalloc(&p, std::max<size_t>(1, count) * sizeof(T)));
    return p;
}

} // namespace

// Top-k of Q columns d_vals[q*n .. q*n + n) by (value desc, id asc) into host
// arrays ids/vals [Q][k].  One histogram launch and one threshold launch for
// all columns, ONE host synchronisation to learn the candidate counts, then per
// column a select + stable sort (device scratch allocated once per call and
// grown to the largest candidate set), one D2H of every column's result and a
// final synchronisation.
void device_topk_batch(const double* d_vals, uint32_t n, uint32_t Q, uint32_t k, uint32_t* ids, double* vals,
                       cudaStream_t st) {
    k = std::min(k, n);
    if (k == 0 || Q == 0) return;
    unsigned int* hist = dmalloc<unsigned int>(static_cast<size_t>(Q) << 16);
    unsigned int* meta = dmalloc<unsigned int>(4 * static_cast<size_t>(Q));
    std::vector<void*> owned{hist, meta};
    auto release = [&] {
        for (void* p : owned) cudaFree(p);
    };
    try {
        CPG_CUDA(cudaMemsetAsync(hist, 0, (sizeof(unsigned int) << 16) * Q, st));
        for (uint32_t q = 0; q < Q; ++q) {
            k_hist16<<<1184, 256, 0, st>>>(d_vals + static_cast<size_t>(q) * n, n, hist + (static_cast<size_t>(q) << 16));
            k_threshold<<<1, 32, 0, st>>>(hist + (static_cast<size_t>(q) << 16), k, meta + 2 * q, meta + 2 * q + 1);
        }
        std::vector<unsigned int> bc(2 * static_cast<size_t>(Q));
        CPG_CUDA(cudaMemcpyAsync(bc.data(), meta, sizeof(unsigned int) * 2 * Q, cudaMemcpyDeviceToHost, st));
        CPG_CUDA(cudaStreamSynchronize(st));
        uint32_t mmax = 0;
        for (uint32_t q = 0; q < Q; ++q) {
            const bool full = bc[2 * q + 1] > (1u << 24);  // pathological ties: stable sort of everything
            mmax = std::max(mmax, full ? n : bc[2 * q + 1]);
        }
        uint32_t* c_ids = dmalloc<uint32_t>(mmax);
        double* c_vals = dmalloc<double>(mmax);
        uint32_t* s_ids = dmalloc<uint32_t>(mmax);
        double* s_vals = dmalloc<double>(mmax);
        uint32_t* r_ids = dmalloc<uint32_t>(static_cast<size_t>(Q) * k);
        double* r_vals = dmalloc<double>(static_cast<size_t>(Q) * k);
        owned.insert(owned.end(), {c_ids, c_vals, s_ids, s_vals, r_ids, r_vals});
        cub::CountingInputIterator<uint32_t> iota(0);
        size_t b_sel = 0, b_sort = 0;
        cub::DeviceSelect::If(nullptr, b_sel, iota, c_ids, meta + 2 * Q, n, AtLeastBin{d_vals, 0u}, st);
        cub::DeviceRadixSort::SortPairsDescending(nullptr, b_sort, c_vals, s_vals, c_ids, s_ids, mmax, 0, 64, st);
        const size_t bytes = std::max(b_sel, b_sort);
        void* tmp = dmalloc<char>(bytes);
        owned.push_back(tmp);
        for (uint32_t q = 0; q < Q; ++q) {
            const double* v = d_vals + static_cast<size_t>(q) * n;
            const bool full = bc[2 * q + 1] > (1u << 24);
            const uint32_t m = full ? n : bc[2 * q + 1];
            const unsigned bin = full ? 0u : bc[2 * q];
            size_t b = bytes;
            CPG_CUDA(cub::DeviceSelect::If(tmp, b, iota, c_ids, meta + 2 * Q + q, n, AtLeastBin{v, bin}, st));
            k_gather_vals<<<std::max<uint32_t>(1, std::min<uint32_t>((m + 255) / 256, 1184)), 256, 0, st>>>(v, c_ids, m,
                                                                                                          c_vals);
            // stable descending sort by value: ties keep ascending id order (candidates are in id order)
            b = bytes;
            CPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, b, c_vals, s_vals, c_ids, s_ids, m, 0, 64, st));
            CPG_CUDA(cudaMemcpyAsync(r_ids + static_cast<size_t>(q) * k, s_ids, sizeof(uint32_t) * k,
                                     cudaMemcpyDeviceToDevice, st));
            CPG_CUDA(cudaMemcpyAsync(r_vals + static_cast<size_t>(q) * k, s_vals, sizeof(double) * k,
                                     cudaMemcpyDeviceToDevice, st));
        }
        CPG_CUDA(cudaMemcpyAsync(ids, r_ids, sizeof(uint32_t) * k * Q, cudaMemcpyDeviceToHost, st));
        CPG_CUDA(cudaMemcpyAsync(vals, r_vals, sizeof(double) * k * Q, cudaMemcpyDeviceToHost, st));
        CPG_CUDA(cudaStreamSynchronize(st));
    } catch (...) {
        cudaStreamSynchronize(st);
        release();
        throw;
    }
    release();
}

} // namespace cpg
