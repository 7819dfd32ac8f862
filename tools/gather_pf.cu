// tools/gather_pf.cu -- what limits random row gathers on B200, and whether
// fire-and-forget L2 prefetches lift it.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_pf tools/gather_pf.cu
//   tools/gather_pf            (one JSON line per case)
//
// Cases (uniformly random rows, indices streamed coalesced as in the CSR):
//   * table size sweep 0.5 / 2 / 8 GB at 128-B rows (translation reach vs DRAM);
//   * row width 8 / 64 / 128 / 256 B from an 8 GB table;
//   * 128-B and 8-B rows with prefetch.global.L2 issued PD row-groups ahead of
//     the demand loads: if the ceiling is per-SM outstanding L1 misses x DRAM
//     latency, demand loads that hit L2 free those slots sooner.
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

__device__ __forceinline__ void pf_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// L lanes per row (16 B each; L = 0 means one 8-B value per lane), 32/L rows per
// warp instruction, U row groups in flight, prefetch PD row groups ahead (0: off).
template <int L, int U, int PD>
__global__ void __launch_bounds__(256, 4) k_gather(const double* __restrict__ table, const uint32_t* __restrict__ idx,
                                                    uint64_t m, double* sink) {
    constexpr int RPW = L ? 32 / L : 32;
    constexpr int W = L ? 2 * L : 1;  // doubles per row
    const int lane = threadIdx.x & 31, slot = L ? lane / L : lane, cl = L ? lane % L : 0;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t step = nw * RPW * U;
    double acc = 0.0;
    for (uint64_t base = warp * RPW * U; base < m; base += step) {
        if (PD) {  // rows of the group PD steps ahead: one prefetch per 32-B sector
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const uint64_t i = base + PD * step + q * RPW + slot;
                if (i < m && (L == 0 || (cl & 1) == 0)) {
                    const uint32_t r = __ldg(idx + i);
                    pf_l2(table + static_cast<size_t>(r) * W + 2 * cl);
                }
            }
        }
        double2 v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t i = base + q * RPW + slot;
            const uint32_t r = i < m ? __ldg(idx + i) : 0u;
            if (L)
                v[q] = i < m ? __ldg(reinterpret_cast<const double2*>(table + static_cast<size_t>(r) * W) + cl)
                             : make_double2(0.0, 0.0);
            else
                v[q] = make_double2(i < m ? __ldg(table + r) : 0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y;
    }
    if (acc == 123.456) *sink = acc;
}

__device__ __forceinline__ uint32_t smid() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(r));
    return r;
}

// 128-B rows; every SM gathers only inside its own window of win_rows rows
// (windows staggered over the table): translation locality per SM, no
// locality across SMs.  idx holds offsets in [0, win_rows).
template <int U>
__global__ void __launch_bounds__(256, 4) k_gather_win(const double* __restrict__ table, const uint32_t* __restrict__ idx,
                                                        uint64_t m, uint32_t rows, uint32_t win_rows, double* sink) {
    constexpr int L = 8, RPW = 4, W = 16;
    const int lane = threadIdx.x & 31, slot = lane / L, cl = lane % L;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t step = nw * RPW * U;
    const uint32_t w0 = static_cast<uint32_t>((static_cast<uint64_t>(smid()) * 2654435761ull) % (rows - win_rows));
    double acc = 0.0;
    for (uint64_t base = warp * RPW * U; base < m; base += step) {
        double2 v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t i = base + q * RPW + slot;
            const uint32_t r = i < m ? w0 + __ldg(idx + i) : 0u;
            v[q] = i < m ? __ldg(reinterpret_cast<const double2*>(table + static_cast<size_t>(r) * W) + cl)
                         : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y;
    }
    if (acc == 123.456) *sink = acc;
}

// Sorted groups: group g holds len(g) random rows sorted ascending (a row
// group's edges in column order); one 8-lane slot streams one group at a time,
// U gathers in flight per lane.  len(g) in [G/2, 3G/2) when jitter, else G.
__global__ void k_fill_groups(uint32_t* idx, uint32_t* len, uint64_t n_groups, int G, bool jitter, uint32_t rows,
                              uint64_t seed, bool sorted) {
    for (uint64_t g = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; g < n_groups;
         g += (uint64_t)gridDim.x * blockDim.x) {
        auto mix = [](uint64_t x) {
            x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
            x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
            return x ^ (x >> 31);
        };
        const uint64_t z0 = mix(mix(seed + 0x632be59bd9b4e019ull * (g + 1)));
        uint64_t z = z0;
        auto next = [&]() {
            z += 0x9e3779b97f4a7c15ull;
            uint64_t x = z;
            x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
            x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
            return x ^ (x >> 31);
        };
        const int L = jitter ? G / 2 + static_cast<int>(next() % G) : G;
        len[g] = L;
        // sorted uniform sample: cumulative exponential spacings
        double tot = 0.0;
        for (int j = 0; j <= L; ++j) tot += -log((next() >> 11) * (1.0 / 9007199254740992.0) + 1e-300);
        double c = 0.0;
        uint64_t s2 = z;
        (void)s2;
        z = z0;
        if (jitter) next();
        for (int j = 0; j < L; ++j) {
            c += -log((next() >> 11) * (1.0 / 9007199254740992.0) + 1e-300);
            uint64_t r = sorted ? static_cast<uint64_t>(c / tot * rows) : next() % rows;
            idx[g * 2 * G + j] = static_cast<uint32_t>(r < rows ? r : rows - 1);
        }
    }
}

template <int U>
__global__ void __launch_bounds__(256, 4) k_gather_groups(const double* __restrict__ table, const uint32_t* __restrict__ idx,
                                                           const uint32_t* __restrict__ len, uint64_t n_groups, int G,
                                                           double* sink) {
    constexpr int L = 8, RPW = 4, W = 16;
    const int lane = threadIdx.x & 31, slot = lane / L, cl = lane % L;
    const uint64_t gs = ((blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5) * RPW + slot;
    const uint64_t ns = (((uint64_t)gridDim.x * blockDim.x) >> 5) * RPW;
    double acc = 0.0;
    for (uint64_t g = gs; __any_sync(0xffffffffu, g < n_groups); g += ns) {
        const int m = g < n_groups ? static_cast<int>(len[g]) : 0;
        const uint32_t* p = idx + g * 2 * G;
        for (int t0 = 0; __any_sync(0xffffffffu, t0 < m); t0 += U) {
            double2 v[U];
#pragma unroll
            for (int q = 0; q < U; ++q) {
                const int t = t0 + q;
                const uint32_t r = t < m ? __ldg(p + t) : 0u;
                v[q] = t < m ? __ldg(reinterpret_cast<const double2*>(table + static_cast<size_t>(r) * W) + cl)
                             : make_double2(0.0, 0.0);
            }
#pragma unroll
            for (int q = 0; q < U; ++q) acc += v[q].x + v[q].y;
        }
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

int main() {
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    const size_t max_table = 8ull << 30;
    const size_t align = 512ull << 20;
    void* base = nullptr;
    double* sink = nullptr;
    CK(cudaMalloc(&base, max_table + align));
    double* table = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(base) + align - 1) / align * align);
    CK(cudaMalloc(&sink, sizeof(double)));
    CK(cudaMemset(table, 0, max_table));
    const uint64_t m = 256ull << 20;
    uint32_t* idx = nullptr;
    CK(cudaMalloc(&idx, m * sizeof(uint32_t)));
    const int grid = sms * 4;
    auto run = [&](const char* name, int row_bytes, size_t tbytes, uint64_t gathers, auto launch) {
        k_fill_idx<<<sms * 8, 256>>>(idx, gathers, static_cast<uint32_t>(tbytes / row_bytes), 7);
        cudaDeviceSynchronize();
        const float ms = time_ms(launch);
        std::printf("{\"case\": \"%s\", \"row_bytes\": %d, \"table_mb\": %zu, \"gathers\": %llu, \"ms\": %.3f, "
                    "\"gathers_per_s\": %.3e, \"gathered_GBps\": %.1f}\n",
                    name, row_bytes, tbytes >> 20, static_cast<unsigned long long>(gathers), ms,
                    gathers / (ms / 1e3), gathers * (double)row_bytes / ms / 1e6);
        std::fflush(stdout);
    };
    run("size", 128, max_table, m, [&] { k_gather<8, 8, 0><<<grid, 256>>>(table, idx, m, sink); });
    {
        const uint32_t rows = static_cast<uint32_t>(max_table / 128);
        uint32_t* len = nullptr;
        for (int G : {64, 480, 2048}) {
            for (int jit : {0, 1, 2}) {  // 2: unsorted control
                const uint64_t ng = m / (2 * G);
                CK(cudaMalloc(&len, ng * 4));
                k_fill_groups<<<sms * 4, 256>>>(idx, len, ng, G, jit == 1, rows, 11, jit != 2);
                CK(cudaDeviceSynchronize());
                const float ms = time_ms([&] { k_gather_groups<8><<<grid, 256>>>(table, idx, len, ng, G, sink); });
                std::vector<uint32_t> h(ng);
                cudaMemcpy(h.data(), len, ng * 4, cudaMemcpyDeviceToHost);
                uint64_t tot = 0;
                for (auto x : h) tot += x;
                std::printf("{\"case\": \"sorted_groups\", \"G\": %d, \"jitter\": %d, \"gathers\": %llu, \"ms\": %.3f, "
                            "\"gathers_per_s\": %.3e, \"gathered_GBps\": %.1f}\n",
                            G, jit, (unsigned long long)tot, ms, tot / (ms / 1e3), tot * 128.0 / ms / 1e6);
                std::fflush(stdout);
                cudaFree(len);
            }
        }
    }
    CK(cudaGetLastError());
    return 0;
}
