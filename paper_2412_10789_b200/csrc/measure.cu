// measure.cu -- the eval harness's error metrics on the device.
//
// measure (src/eval.cpp:18-37): with d_u = |truth_u - est_u|,
//   l1 = sum_u d_u,  l2 = sqrt(sum_u d_u^2),
//   deg_norm_inf = max_u d_u / deg(u), argmax_node = the FIRST u attaining it
//   (the reference updates on a strict '>', so ties keep the smaller id and an
//   all-zero difference reports node 0).
// Here every column of [cols][n] caller-id vectors is reduced on the device, so
// only four numbers per query cross PCIe instead of the n-vector.
//
// Order: block b owns the contiguous id range [b*span, (b+1)*span); threads sum
// strided elements with Neumaier compensation, the block combines its threads
// in a fixed tree (value pairs with their compensations), and one warp per
// column adds the block partials in block order.  The sums are deterministic
// and carry ~1 ulp of error, so they differ from the reference's sequential
// left-to-right sum only by that sum's own rounding (the reference's test
// allows 1e-14 relative, test_eval.cpp:66).  The max and argmax are exact.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "cpg_graph.hpp"

namespace cpg {
namespace {

constexpr int kMeasureThreads = 256;

struct Part {
    double l1, l1c, sq, sqc, dn;
    uint32_t arg;
};

__device__ __forceinline__ void add_comp(double& s, double& c, double x) {  // Neumaier
    const double t = s + x;
    c += (fabs(s) >= fabs(x)) ? (s - t) + x : (x - t) + s;
    s = t;
}

__device__ __forceinline__ void merge(Part& a, const Part& b) {
    add_comp(a.l1, a.l1c, b.l1);
    a.l1c += b.l1c;
    add_comp(a.sq, a.sqc, b.sq);
    a.sqc += b.sqc;
    // max of d/deg; ties keep the smaller id (the reference's first strict '>')
    if (b.dn > a.dn || (b.dn == a.dn && b.arg < a.arg)) {
        a.dn = b.dn;
        a.arg = b.arg;
    }
}

__device__ __forceinline__ Part shfl_part(const Part& p, int off) {
    Part q;
    q.l1 = __shfl_down_sync(0xffffffffu, p.l1, off);
    q.l1c = __shfl_down_sync(0xffffffffu, p.l1c, off);
    q.sq = __shfl_down_sync(0xffffffffu, p.sq, off);
    q.sqc = __shfl_down_sync(0xffffffffu, p.sqc, off);
    q.dn = __shfl_down_sync(0xffffffffu, p.dn, off);
    q.arg = __shfl_down_sync(0xffffffffu, p.arg, off);
    return q;
}

// Fixed-order block reduction; thread 0 returns the block's Part.
__device__ Part block_reduce(Part p) {
    __shared__ Part sh[kMeasureThreads / 32];
    for (int off = 16; off; off >>= 1) {
        const Part q = shfl_part(p, off);
        merge(p, q);
    }
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = p;
    __syncthreads();
    if (threadIdx.x == 0)
        for (int w = 1; w < kMeasureThreads / 32; ++w) merge(p, sh[w]);
    return p;
}

// grid (blocks per column, cols); truth/est are [cols][n] in caller ids.
__global__ void __launch_bounds__(kMeasureThreads) k_measure(const double* __restrict__ truth,
                                                             const double* __restrict__ est, uint32_t n,
                                                             const uint32_t* __restrict__ no,
                                                             const uint32_t* __restrict__ gdeg, uint32_t span,
                                                             Part* __restrict__ parts) {
    const size_t col = blockIdx.y;
    const double* t = truth + col * n;
    const double* e = est + col * n;
    Part p{0.0, 0.0, 0.0, 0.0, 0.0, 0u};
    const uint64_t lo = static_cast<uint64_t>(blockIdx.x) * span;
    const uint64_t hi = lo + span < n ? lo + span : n;
    for (uint64_t u = lo + threadIdx.x; u < hi; u += kMeasureThreads) {
        const double d = fabs(__ldg(t + u) - __ldg(e + u));
        add_comp(p.l1, p.l1c, d);
        add_comp(p.sq, p.sqc, d * d);
        const double dn = d / static_cast<double>(__ldg(gdeg + __ldg(no + u)));
        if (dn > p.dn) {  // per thread ids ascend: strict '>' keeps the first
            p.dn = dn;
            p.arg = static_cast<uint32_t>(u);
        }
    }
    p = block_reduce(p);
    if (threadIdx.x == 0) parts[col * gridDim.x + blockIdx.x] = p;
}

// One warp per column: block partials in block order.
__global__ void k_measure_final(const Part* __restrict__ parts, uint32_t nb, cpg_error_report* __restrict__ out) {
    const size_t col = blockIdx.x;
    if (threadIdx.x != 0) return;
    Part p = parts[col * nb];
    for (uint32_t b = 1; b < nb; ++b) merge(p, parts[col * nb + b]);
    cpg_error_report r;
    r.l1 = p.l1 + p.l1c;
    r.l2 = sqrt(p.sq + p.sqc);
    r.deg_norm_inf = p.dn;
    r.argmax_node = p.arg;
    out[col] = r;
}

}  // namespace

// Error reports of `cols` (truth, estimate) column pairs, device-resident, into
// d_reports[cols] (device).  scratch: >= measure_scratch_bytes(g, cols) bytes.
size_t measure_scratch_bytes(const cpg_graph* g, uint32_t cols) {
    const uint32_t nb = static_cast<uint32_t>(std::max(1, 2 * g->sm_count));
    return sizeof(Part) * nb * cols;
}

void launch_measure(const cpg_graph* g, const double* d_truth, const double* d_est, uint32_t cols, void* scratch,
                    cpg_error_report* d_reports, cudaStream_t st) {
    if (!cols) return;
    const uint32_t n = g->n;
    uint32_t nb = static_cast<uint32_t>(std::max(1, 2 * g->sm_count));
    const uint32_t span = (n + nb - 1) / nb;
    nb = std::max<uint32_t>(1, (n + span - 1) / span);
    Part* parts = static_cast<Part*>(scratch);
    k_measure<<<dim3(nb, cols), kMeasureThreads, 0, st>>>(d_truth, d_est, n, g->new_of_old, g->gdeg, span, parts);
    k_measure_final<<<cols, 32, 0, st>>>(parts, nb, d_reports);
    CPG_CUDA(cudaGetLastError());
}

}  // namespace cpg
