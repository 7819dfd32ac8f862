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
// of the whole vector is used instead.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>

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

// Top-k of d_vals[0..n) by (value desc, id asc) into host arrays.
void device_topk(const double* d_vals, uint32_t n, uint32_t k, uint32_t* ids, double* vals, cudaStream_t st) {
    k = std::min(k, n);
    if (k == 0) return;
    unsigned int* hist = dmalloc<unsigned int>(1 << 16);
    unsigned int* meta = dmalloc<unsigned int>(3);
    CPG_CUDA(cudaMemsetAsync(hist, 0, sizeof(unsigned int) << 16, st));
    k_hist16<<<1184, 256, 0, st>>>(d_vals, n, hist);
    k_threshold<<<1, 32, 0, st>>>(hist, k, meta, meta + 1);
    unsigned int bin_count[2] = {0, 0};
    CPG_CUDA(cudaMemcpyAsync(bin_count, meta, sizeof(bin_count), cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    const uint32_t cand = bin_count[1];
    const bool full = cand > (1u << 24);  // pathological ties: stable sort of everything
    const uint32_t m = full ? n : cand;
    uint32_t* c_ids = dmalloc<uint32_t>(m);
    double* c_vals = dmalloc<double>(m);
    uint32_t* s_ids = dmalloc<uint32_t>(m);
    double* s_vals = dmalloc<double>(m);
    void* tmp = nullptr;
    size_t bytes = 0;
    cub::CountingInputIterator<uint32_t> iota(0);
    if (full) {
        CPG_CUDA(cudaMemcpyAsync(c_vals, d_vals, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
        bytes = 0;
        cub::DeviceSelect::If(nullptr, bytes, iota, c_ids, meta + 2, n, AtLeastBin{d_vals, 0u}, st);
        CPG_CUDA(cudaMalloc(&tmp, bytes));
        CPG_CUDA(cub::DeviceSelect::If(tmp, bytes, iota, c_ids, meta + 2, n, AtLeastBin{d_vals, 0u}, st));
        cudaFree(tmp);
    } else {
        bytes = 0;
        cub::DeviceSelect::If(nullptr, bytes, iota, c_ids, meta + 2, n, AtLeastBin{d_vals, bin_count[0]}, st);
        CPG_CUDA(cudaMalloc(&tmp, bytes));
        CPG_CUDA(cub::DeviceSelect::If(tmp, bytes, iota, c_ids, meta + 2, n, AtLeastBin{d_vals, bin_count[0]}, st));
        cudaFree(tmp);
        k_gather_vals<<<std::max<uint32_t>(1, std::min<uint32_t>((m + 255) / 256, 1184)), 256, 0, st>>>(d_vals, c_ids,
                                                                                                          m, c_vals);
    }
    // stable descending sort by value: ties keep ascending id order (candidates are in id order)
    bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, c_vals, s_vals, c_ids, s_ids, m, 0, 64, st);
    CPG_CUDA(cudaMalloc(&tmp, bytes));
    CPG_CUDA(cub::DeviceRadixSort::SortPairsDescending(tmp, bytes, c_vals, s_vals, c_ids, s_ids, m, 0, 64, st));
    cudaFree(tmp);
    CPG_CUDA(cudaMemcpyAsync(ids, s_ids, sizeof(uint32_t) * k, cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaMemcpyAsync(vals, s_vals, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    CPG_CUDA(cudaStreamSynchronize(st));
    for (void* p : {(void*)hist, (void*)meta, (void*)c_ids, (void*)c_vals, (void*)s_ids, (void*)s_vals}) cudaFree(p);
}

} // namespace cpg
