// tools/gather_peak.cu -- microbenchmark: achievable HBM bandwidth for random
// row gathers on this B200, the access pattern of the ChebyPower steps.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_peak tools/gather_peak.cu
//   ./gather_peak          (prints one JSON line per row width)
//
// A table of `rows` rows of W bytes (W = 8, 128, 512: single-source values,
// 16-column and 64-column batched rows) far larger than L2 is gathered at
// uniformly random row indices (pre-generated, streamed coalesced like the CSR
// index array), lanes grouped so one row is read by W/16 lanes with 16-B
// loads, 8 gathers in flight per lane.  Reported: gathered bytes / time and
// the fraction of the copy peak in MEASURED_PEAKS.json (6545 GB/s).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            std::printf("{\"error\": \"%s\"}\n", cudaGetErrorString(e));        \
            return 1;                                                           \
        }                                                                       \
    } while (0)

__global__ void k_fill_idx(uint32_t* idx, uint64_t m, uint32_t rows, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + 0x9e3779b97f4a7c15ull * (i + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        idx[i] = static_cast<uint32_t>((z >> 11) % rows);
    }
}

// L lanes per row (16 B each), 32/L rows per warp instruction, U in flight.
template <int L, int U>
__global__ void __launch_bounds__(256, 4) k_gather(const double* __restrict__ table, const uint32_t* __restrict__ idx,
                                                    uint64_t m, double* sink) {
    constexpr int RPW = 32 / L;
    const int lane = threadIdx.x & 31, slot = lane / L, cl = lane % L;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (uint64_t base = warp * RPW * U; base < m; base += nw * RPW * U) {
        double2 v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t i = base + q * RPW + slot;
            const uint32_t r = i < m ? __ldg(idx + i) : 0u;
            v[q] = i < m ? __ldg(reinterpret_cast<const double2*>(table + static_cast<size_t>(r) * (2 * L)) + cl)
                         : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y;
    }
    if (acc == 123.456) *sink = acc;
}

// Single 8-B values (single-source step): one value per lane.
template <int U>
__global__ void __launch_bounds__(256, 4) k_gather8(const double* __restrict__ table, const uint32_t* __restrict__ idx,
                                                     uint64_t m, double* sink) {
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    const uint64_t nt = (uint64_t)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (uint64_t base = t; base < m; base += nt * U) {
        double v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t i = base + q * nt;
            v[q] = i < m ? __ldg(table + __ldg(idx + i)) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q];
    }
    if (acc == 123.456) *sink = acc;
}

template <typename F>
float time_ms(F&& launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    launch();
    cudaEventRecord(a);
    for (int i = 0; i < 5; ++i) launch();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms / 5.f;
}

int main(int argc, char** argv) {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t table_bytes = 8ull << 30;  // 8 GB, >> 126 MB L2
    double* table = nullptr;
    double* sink = nullptr;
    // argv[1] = alignment of the table in MB (0: wherever cudaMalloc puts it).  The
    // library places its gathered iterates 512 MB-aligned (translation reach).
    const size_t align = (argc > 1 ? static_cast<size_t>(std::atoll(argv[1])) : 0) << 20;
    void* base = nullptr;
    CK(cudaMalloc(&base, table_bytes + align));
    table = align ? reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(base) + align - 1) / align * align)
                  : static_cast<double*>(base);
    CK(cudaMalloc(&sink, sizeof(double)));
    CK(cudaMemset(table, 0, table_bytes));
    const uint64_t m = 256ull << 20;  // 268M gathers
    uint32_t* idx = nullptr;
    CK(cudaMalloc(&idx, m * sizeof(uint32_t)));
    const int grid = sms * 4;
    struct Case {
        int width;
        double ms;
    };
    std::vector<Case> out;
    {
        const uint32_t rows = static_cast<uint32_t>(table_bytes / 8);
        k_fill_idx<<<sms * 8, 256>>>(idx, m, rows, 1);
        CK(cudaDeviceSynchronize());
        out.push_back({8, time_ms([&] { k_gather8<8><<<grid, 256>>>(table, idx, m, sink); })});
    }
    {
        const uint32_t rows = static_cast<uint32_t>(table_bytes / 128);
        k_fill_idx<<<sms * 8, 256>>>(idx, m, rows, 2);
        CK(cudaDeviceSynchronize());
        out.push_back({128, time_ms([&] { k_gather<8, 8><<<grid, 256>>>(table, idx, m, sink); })});
    }
    {
        const uint32_t rows = static_cast<uint32_t>(table_bytes / 512);
        k_fill_idx<<<sms * 8, 256>>>(idx, m / 4, rows, 3);
        CK(cudaDeviceSynchronize());
        out.push_back({512, time_ms([&] { k_gather<32, 8><<<grid, 256>>>(table, idx, m / 4, sink); })});
    }
    CK(cudaGetLastError());
    for (const auto& c : out) {
        const uint64_t gathers = c.width == 512 ? m / 4 : m;
        const double bytes = static_cast<double>(gathers) * c.width;
        const double idx_bytes = static_cast<double>(gathers) * 4;
        std::printf("{\"align_mb\": %zu, \"row_bytes\": %d, \"gathers\": %llu, \"ms\": %.3f, \"gathered_GBps\": %.1f, "
                    "\"gathered_plus_index_GBps\": %.1f, \"gathers_per_s\": %.3e}\n",
                    align >> 20, c.width, static_cast<unsigned long long>(gathers), c.ms, bytes / c.ms / 1e6,
                    (bytes + idx_bytes) / c.ms / 1e6, gathers / (c.ms / 1e3));
    }
    return 0;
}
