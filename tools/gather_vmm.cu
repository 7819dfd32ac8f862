// tools/gather_vmm.cu -- microbenchmark: does the way the gathered table is
// allocated change the random-row gather rate?  (DESIGN.md 4.2 found the rate
// limited by address-translation reach: 35 G rows/s over 8 GB against 47 G/s
// when each SM stays inside 512 MB.)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_vmm tools/gather_vmm.cu -lcuda
//   tools/gather_vmm            (one JSON line per allocation mode and row width)
//
// Modes: cudaMalloc; cudaMalloc + 512 MB alignment; the driver's virtual memory
// API (cuMemCreate + cuMemMap) with one physical handle for the whole table at
// the minimum and at the recommended granularity, the virtual range aligned to
// 512 MB / to the table size; and the table built from 2 MB handles (forces
// small translation entries, the lower bound).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e = (x);                                                    \
        if (e != cudaSuccess) {                                                 \
            std::printf("{\"error\": \"%s\", \"line\": %d}\n", cudaGetErrorString(e), __LINE__); \
            return 1;                                                           \
        }                                                                       \
    } while (0)
#define CU(x)                                                                   \
    do {                                                                        \
        CUresult e = (x);                                                       \
        if (e != CUDA_SUCCESS) {                                                \
            const char* s = nullptr;                                            \
            cuGetErrorString(e, &s);                                            \
            std::printf("{\"error\": \"%s\", \"line\": %d}\n", s ? s : "?", __LINE__); \
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
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms / 5.f;
}

static uint32_t* g_idx = nullptr;
static double* g_sink = nullptr;
static int g_sms = 0;

int run_table(const char* mode, double* table, size_t table_bytes, size_t gran) {
    const uint64_t m = 256ull << 20;
    const int grid = g_sms * 4;
    CK(cudaMemset(table, 0, table_bytes));
    const int widths[3] = {8, 128, 512};
    for (int w : widths) {
        const uint32_t rows = static_cast<uint32_t>(table_bytes / w);
        const uint64_t gathers = w == 512 ? m / 4 : m;
        k_fill_idx<<<g_sms * 8, 256>>>(g_idx, gathers, rows, w);
        CK(cudaDeviceSynchronize());
        float ms = 0.f;
        if (w == 8) ms = time_ms([&] { k_gather8<8><<<grid, 256>>>(table, g_idx, gathers, g_sink); });
        if (w == 128) ms = time_ms([&] { k_gather<8, 8><<<grid, 256>>>(table, g_idx, gathers, g_sink); });
        if (w == 512) ms = time_ms([&] { k_gather<32, 8><<<grid, 256>>>(table, g_idx, gathers, g_sink); });
        CK(cudaGetLastError());
        std::printf("{\"mode\": \"%s\", \"granularity\": %zu, \"table_gb\": %.2f, \"row_bytes\": %d, \"ms\": %.3f, "
                    "\"gathered_GBps\": %.1f, \"gathers_per_s\": %.3e}\n",
                    mode, gran, table_bytes / 1073741824.0, w, ms, static_cast<double>(gathers) * w / ms / 1e6,
                    gathers / (ms / 1e3));
        std::fflush(stdout);
    }
    return 0;
}

struct VmmTable {
    CUdeviceptr va = 0;
    size_t va_size = 0;
    std::vector<CUmemGenericAllocationHandle> handles;
};

// Map `bytes` of device memory at a virtual range aligned to `va_align`, from
// physical handles of `handle_bytes` each (0: one handle).
int vmm_alloc(VmmTable* t, size_t bytes, size_t gran, size_t va_align, size_t handle_bytes) {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    if (!handle_bytes) handle_bytes = bytes;
    handle_bytes = (handle_bytes + gran - 1) / gran * gran;
    const size_t total = (bytes + handle_bytes - 1) / handle_bytes * handle_bytes;
    CU(cuMemAddressReserve(&t->va, total, va_align, 0, 0));
    t->va_size = total;
    for (size_t off = 0; off < total; off += handle_bytes) {
        CUmemGenericAllocationHandle h;
        CU(cuMemCreate(&h, handle_bytes, &prop, 0));
        CU(cuMemMap(t->va + off, handle_bytes, 0, h, 0));
        t->handles.push_back(h);
    }
    CUmemAccessDesc acc = {};
    acc.location = prop.location;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemSetAccess(t->va, total, &acc, 1));
    return 0;
}

void vmm_free(VmmTable* t) {
    if (!t->va) return;
    cuMemUnmap(t->va, t->va_size);
    for (auto h : t->handles) cuMemRelease(h);
    cuMemAddressFree(t->va, t->va_size);
    *t = VmmTable();
}

int main(int argc, char** argv) {
    CK(cudaSetDevice(0));
    CK(cudaFree(0));
    CK(cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, 0));
    // argv[2] = table size in MB: the plain-cudaMalloc case only (an L2-resident table gives
    // the gather rate of L2 hits)
    const size_t table_bytes = argc > 2 ? static_cast<size_t>(std::atoll(argv[2])) << 20
                                        : (argc > 1 ? static_cast<size_t>(std::atoll(argv[1])) : 8) << 30;
    CK(cudaMalloc(&g_sink, sizeof(double)));
    CK(cudaMalloc(&g_idx, (256ull << 20) * sizeof(uint32_t)));

    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gmin = 0, grec = 0;
    CU(cuMemGetAllocationGranularity(&gmin, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    CU(cuMemGetAllocationGranularity(&grec, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    std::printf("{\"granularity_min\": %zu, \"granularity_recommended\": %zu}\n", gmin, grec);

    {  // plain cudaMalloc
        void* p = nullptr;
        CK(cudaMalloc(&p, table_bytes));
        if (run_table("cudaMalloc", static_cast<double*>(p), table_bytes, 0)) return 1;
        CK(cudaFree(p));
    }
    if (argc > 2) return 0;
    {  // cudaMalloc, 512 MB aligned (the library's dalloc_aligned)
        const size_t align = 512ull << 20;
        void* p = nullptr;
        CK(cudaMalloc(&p, table_bytes + align));
        double* t = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(p) + align - 1) / align * align);
        if (run_table("cudaMalloc_align512M", t, table_bytes, 0)) return 1;
        CK(cudaFree(p));
    }
    struct Mode {
        const char* name;
        size_t gran, va_align, handle;
    };
    const Mode modes[] = {
        {"vmm_one_handle_min_gran_va512M", gmin, 512ull << 20, 0},
        {"vmm_one_handle_rec_gran_va512M", grec, 512ull << 20, 0},
        {"vmm_one_handle_va_table_size", grec, table_bytes, 0},
        {"vmm_handles_512M", grec, 512ull << 20, 512ull << 20},
        {"vmm_handles_32M", grec, 512ull << 20, 32ull << 20},
        {"vmm_handles_2M", gmin, 512ull << 20, 2ull << 20},
    };
    for (const Mode& md : modes) {
        VmmTable t;
        if (vmm_alloc(&t, table_bytes, md.gran, md.va_align, md.handle)) {
            vmm_free(&t);
            continue;
        }
        run_table(md.name, reinterpret_cast<double*>(t.va), table_bytes, md.gran);
        CK(cudaDeviceSynchronize());
        vmm_free(&t);
    }
    return 0;
}
