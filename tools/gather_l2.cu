// tools/gather_l2.cu -- microbenchmark: what issues random 8-B gathers fastest on
// B200 (the single-source step's inner operation, DESIGN.md 4.1/4.3).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_l2 tools/gather_l2.cu
//   ./tools/gather_l2 [n_table] [zipf_k]
//
// A table of n doubles (default 4.85 M = config 3's iterate, 39 MB, L2-resident)
// is gathered at m = 86 M indices streamed coalesced (like the CSR index
// array).  Index distribution: idx = floor(n * u^k), u uniform (k = 1 uniform;
// k = 3.81 puts 25% / 37% / 53% of the gathers below 24 K / 100 K / 400 K like
// config 3's degree-sorted columns).  Variants:
//   ldg      ld.global.nc per lane, U in flight         (the step kernels' form)
//   ldg_na   ld.global.nc.L1::no_allocate
//   ldg_cg   ld.global.cg (L2 only)
//   smem     the first H entries staged in shared memory (one 1024-thread CTA
//            per SM, 192 KB), the rest ld.global.nc
//   tma4     cp.async.bulk.tensor.2d tile::gather4 of 16-B rows into shared
//            memory (4 gathers per instruction through the TMA unit), S stages
// Prints one JSON line per variant: gathers/s.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#define CK(x)                                                                     \
    do {                                                                          \
        cudaError_t e = (x);                                                      \
        if (e != cudaSuccess) {                                                   \
            std::printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e), __LINE__); \
            std::exit(1);                                                         \
        }                                                                         \
    } while (0)

__global__ void k_fill_idx(uint32_t* idx, uint64_t m, uint32_t n, double k, uint64_t seed) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t z = seed + 0x9e3779b97f4a7c15ull * (i + 1);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        z ^= z >> 31;
        const double u = (z >> 11) * (1.0 / 9007199254740992.0);
        uint64_t v = static_cast<uint64_t>(n * pow(u, k));
        idx[i] = static_cast<uint32_t>(v < n ? v : n - 1);
    }
}

__global__ void k_fill_table(double* t, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        t[i] = 1e-9 * static_cast<double>(i % 1000);
}

template <int MODE>
__device__ __forceinline__ double ld(const double* p) {
    double v;
    if (MODE == 0) {
        v = __ldg(p);
    } else if (MODE == 1) {
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
    } else {
        asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(v) : "l"(p));
    }
    return v;
}

// Each warp takes 32*U consecutive indices (coalesced index loads), U gathers per lane in flight.
template <int MODE, int U>
__global__ void __launch_bounds__(256) k_ldg(const double* __restrict__ table, const uint32_t* __restrict__ idx,
                                             uint64_t m, double* sink) {
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (uint64_t base = warp * 32 * U; base < m; base += nw * 32 * U) {
        uint32_t r[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t i = base + q * 32 + lane;
            r[q] = i < m ? __ldg(idx + i) : 0u;
        }
        double v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = ld<MODE>(table + r[q]);
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q];
    }
    atomicAdd(sink, acc);
}

// Hot prefix [0, H) in shared memory; one 1024-thread CTA per SM.
template <int U>
__global__ void __launch_bounds__(1024, 1) k_smem(const double* __restrict__ table, const uint32_t* __restrict__ idx,
                                                  uint64_t m, uint32_t H, double* sink) {
    extern __shared__ double hot[];
    for (uint32_t i = threadIdx.x; i < H; i += blockDim.x) hot[i] = __ldg(table + i);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    double acc = 0.0;
    for (uint64_t base = warp * 32 * U; base < m; base += nw * 32 * U) {
        uint32_t r[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
            const uint64_t i = base + q * 32 + lane;
            r[q] = i < m ? __ldg(idx + i) : 0u;
        }
        double v[U];
#pragma unroll
        for (int q = 0; q < U; ++q) v[q] = r[q] < H ? hot[r[q]] : __ldg(table + r[q]);
#pragma unroll
        for (int q = 0; q < U; ++q) acc += v[q];
    }
    atomicAdd(sink, acc);
}

// ---- TMA gather4 -----------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// S stages per warp, each 32 gathers = 8 gather4 of 16-B rows (512 B) + one mbarrier.
template <int S>
__global__ void __launch_bounds__(256) k_tma4(const __grid_constant__ CUtensorMap tmap, const uint32_t* __restrict__ idx,
                                              uint64_t m, double* sink) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 127) & ~uintptr_t(127));
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    // [S][8 groups][8 double2]: each gather4 lands 64 B at a 128-B aligned slot (TMA alignment)
    double2* buf = reinterpret_cast<double2*>(smem) + static_cast<size_t>(wib) * S * 64;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8 * S * 64 * 16) + wib * S;
    if (lane == 0)
        for (int s = 0; s < S; ++s)
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(bar + s)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
    const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
    const uint64_t nchunks = (m + 31) / 32;
    double acc = 0.0;
    uint32_t phase = 0;  // bit s = parity of stage s
    uint32_t held[S];    // the lane's own index of chunk in stage s
    uint64_t c = warp;
    // prologue: fill S stages
    auto issue = [&](int s, uint64_t chunk) {
        const uint64_t i = chunk * 32 + lane;
        const uint32_t r = i < m ? __ldg(idx + i) : 0u;
        held[s] = r;
        const uint32_t row = r >> 1;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(bar + s)), "r"(512u)
                         : "memory");
        __syncwarp();
#pragma unroll
        for (int g = 0; g < 8; ++g) {
            const int r0 = __shfl_sync(0xffffffffu, row, 4 * g), r1 = __shfl_sync(0xffffffffu, row, 4 * g + 1);
            const int r2 = __shfl_sync(0xffffffffu, row, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, row, 4 * g + 3);
            if (lane == 0)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
                    "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + s * 64 + 8 * g)),
                    "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(smem_u32(bar + s))
                    : "memory");
        }
    };
    int s = 0;
    for (int p = 0; p < S; ++p) {
        if (c + static_cast<uint64_t>(p) * nw < nchunks) issue(p, c + static_cast<uint64_t>(p) * nw);
    }
    for (; c < nchunks; c += nw) {
        // wait stage s
        const uint32_t par = (phase >> s) & 1u;
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(smem_u32(bar + s)), "r"(par)
                : "memory");
        }
        phase ^= 1u << s;
        const double2 v = buf[s * 64 + (lane >> 2) * 8 + (lane & 3)];
        acc += (held[s] & 1) ? v.y : v.x;
        __syncwarp();
        const uint64_t nxt = c + static_cast<uint64_t>(S) * nw;
        if (nxt < nchunks) issue(s, nxt);
        s = (s + 1 == S) ? 0 : s + 1;
    }
    atomicAdd(sink, acc);
}

typedef CUresult (*EncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <typename F>
float time_it(F&& f, int reps) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    f();
    CK(cudaDeviceSynchronize());
    cudaEventRecord(a);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

int main(int argc, char** argv) {
    const uint32_t n = argc > 1 ? static_cast<uint32_t>(std::atoll(argv[1])) : 4'846'609u;
    const double zk = argc > 2 ? std::atof(argv[2]) : 3.81;
    const uint64_t m = 86'000'000ull;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    double* table;
    uint32_t* idx;
    double* sink;
    const uint32_t n2 = (n + 1) & ~1u;
    CK(cudaMalloc(&table, sizeof(double) * n2));
    CK(cudaMalloc(&idx, sizeof(uint32_t) * m));
    CK(cudaMalloc(&sink, 8));
    k_fill_table<<<1184, 256>>>(table, n2);
    k_fill_idx<<<1184, 256>>>(idx, m, n, zk, 12345);
    CK(cudaDeviceSynchronize());
    const int reps = 10;
    auto report = [&](const char* name, float ms) {
        double s = 0;
        CK(cudaMemcpy(&s, sink, 8, cudaMemcpyDeviceToHost));
        CK(cudaMemset(sink, 0, 8));
        std::printf("{\"variant\": \"%s\", \"n\": %u, \"zipf_k\": %.2f, \"ms\": %.4f, \"G_gathers_per_s\": %.1f, "
                    "\"checksum_per_rep\": %.9e}\n", name, n, zk, ms, m / (ms * 1e-3) / 1e9, s / (reps + 1));
        std::fflush(stdout);
    };
    CK(cudaMemset(sink, 0, 8));
    for (int occ : {4, 8}) {
        const int grid = sms * occ;
        char nm[64];
        std::snprintf(nm, sizeof nm, "ldg_U8_occ%d", occ);
        report(nm, time_it([&] { k_ldg<0, 8><<<grid, 256>>>(table, idx, m, sink); }, reps));
        std::snprintf(nm, sizeof nm, "ldg_U16_occ%d", occ);
        report(nm, time_it([&] { k_ldg<0, 16><<<grid, 256>>>(table, idx, m, sink); }, reps));
        std::snprintf(nm, sizeof nm, "ldg_na_U8_occ%d", occ);
        report(nm, time_it([&] { k_ldg<1, 8><<<grid, 256>>>(table, idx, m, sink); }, reps));
        std::snprintf(nm, sizeof nm, "ldg_cg_U8_occ%d", occ);
        report(nm, time_it([&] { k_ldg<2, 8><<<grid, 256>>>(table, idx, m, sink); }, reps));
    }
    for (uint32_t H : {8192u, 16384u, 24576u}) {
        const size_t sm = sizeof(double) * H;
        CK(cudaFuncSetAttribute(k_smem<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        char nm[64];
        std::snprintf(nm, sizeof nm, "smem_H%u_U8", H);
        report(nm, time_it([&] { k_smem<8><<<sms, 1024, sm>>>(table, idx, m, H, sink); }, reps));
    }
    // TMA gather4 over a [n2/2][2] f64 view (16-B rows)
    EncodeTiled enc = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&enc), cudaEnableDefault, &q));
    if (!enc) {
        std::printf("{\"error\": \"no cuTensorMapEncodeTiled\"}\n");
        return 0;
    }
    CUtensorMap tmap;
    const cuuint64_t dims[2] = {2, n2 / 2};
    const cuuint64_t strides[1] = {16};
    const cuuint32_t box[2] = {2, 1};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, table, dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        std::printf("{\"error\": \"encode %d\"}\n", static_cast<int>(r));
        return 0;
    }
    auto tma = [&](auto kern, int S, int occ, const char* nm) {
        const size_t sm = 8 * (static_cast<size_t>(S) * 64 * 16 + S * 8) + 128;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)));
        report(nm, time_it([&] { kern<<<sms * occ, 256, sm>>>(tmap, idx, m, sink); }, reps));
    };
    tma(k_tma4<4>, 4, 4, "tma4_S4_occ4");
    tma(k_tma4<8>, 8, 4, "tma4_S8_occ4");
    tma(k_tma4<8>, 8, 8, "tma4_S8_occ8");
    tma(k_tma4<16>, 16, 4, "tma4_S16_occ4");
    // correctness spot check of the gather4 path: sum of gathered values vs ldg
    return 0;
}
