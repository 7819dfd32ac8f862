// loopback.cu -- test-only data plane for the row-sharded path on ONE GPU.
//
// R shard handles of one process live on the same device; rank r's "all-gather"
// copies every peer's slice of the replicated buffer into its own replica, and
// the "all-reduce" sums the ranks' buffers in rank order.  Each rank is driven
// by its own host thread (one query call per rank, concurrently, exactly as
// one process per GPU would issue them), and the ranks meet at host barriers:
//
//   allgather(send, recv, count, st), rank r:
//     record "my slice is computed" on st; publish send; barrier
//     st waits for every peer's event; cudaMemcpyAsync peer slices -> recv
//     synchronize st; barrier     (no peer moves on before every copy landed)
//
// The point is coverage, not speed: it drives the product's own layout and
// exchange code (k_assign / k_local relabel, chunk_row0, gather_chunk,
// gather_result, the mass all-reduce, unpermute) with nranks > 1 on a box
// that has one GPU.  Multi-GPU runs use the NCCL plane (nccl_dl.cpp).
#include <cuda_runtime.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "cpg_graph.hpp"

namespace cpg {

struct LoopbackGroup {
    int R = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    uint64_t generation = 0;
    std::vector<const double*> send;
    std::vector<double*> buf;
    std::vector<cudaEvent_t> ev;

    void barrier() {
        std::unique_lock<std::mutex> lock(mu);
        const uint64_t gen = generation;
        if (++arrived == R) {
            arrived = 0;
            ++generation;
            cv.notify_all();
        } else {
            cv.wait(lock, [&] { return generation != gen; });
        }
    }
};

namespace {

__global__ void k_sum_ranks(double* const* bufs, int R, size_t count, double* out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < R; ++p) s += bufs[p][i];
        out[i] = s;
    }
}

struct LoopbackComm final : Comm {
    LoopbackGroup* g = nullptr;
    double* scratch = nullptr;
    size_t scratch_cap = 0;
    double** d_bufs = nullptr;

    ~LoopbackComm() override {
        if (scratch) cudaFree(scratch);
        if (d_bufs) cudaFree(d_bufs);
    }
    void publish(cudaStream_t st) {
        CPG_CUDA(cudaEventRecord(g->ev[rank], st));
        g->barrier();
        for (int p = 0; p < nranks; ++p)
            if (p != rank) CPG_CUDA(cudaStreamWaitEvent(st, g->ev[p], 0));
    }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
        g->send[rank] = send;
        publish(st);
        for (int p = 0; p < nranks; ++p) {
            const double* src = p == rank ? send : g->send[p];
            double* dst = recv + static_cast<size_t>(p) * count;
            if (src != dst) CPG_CUDA(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
        }
        CPG_CUDA(cudaStreamSynchronize(st));
        g->barrier();
    }
    void allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
        if (scratch_cap < count) {
            if (scratch) cudaFree(scratch);
            CPG_CUDA(cudaMalloc(&scratch, count * sizeof(double)));
            scratch_cap = count;
        }
        if (!d_bufs) CPG_CUDA(cudaMalloc(&d_bufs, sizeof(double*) * nranks));
        g->buf[rank] = buf;
        publish(st);
        CPG_CUDA(cudaMemcpyAsync(d_bufs, g->buf.data(), sizeof(double*) * nranks, cudaMemcpyHostToDevice, st));
        k_sum_ranks<<<static_cast<int>(std::min<size_t>((count + 255) / 256, 1184)) + 0, 256, 0, st>>>(d_bufs, nranks,
                                                                                                    count, scratch);
        CPG_CUDA(cudaGetLastError());
        CPG_CUDA(cudaStreamSynchronize(st));
        g->barrier();  // every rank has read every buffer
        CPG_CUDA(cudaMemcpyAsync(buf, scratch, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
        CPG_CUDA(cudaStreamSynchronize(st));
    }
    void sync(cudaStream_t st) override { CPG_CUDA(cudaStreamSynchronize(st)); }
};

} // namespace

LoopbackGroup* loopback_group_create(int nranks) {
    auto* grp = new LoopbackGroup;
    grp->R = nranks;
    grp->send.assign(nranks, nullptr);
    grp->buf.assign(nranks, nullptr);
    grp->ev.assign(nranks, nullptr);
    for (auto& e : grp->ev) {
        if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) {
            loopback_group_destroy(grp);
            fail(CPG_ECUDA, "loopback: cudaEventCreate failed");
        }
    }
    return grp;
}

void loopback_group_destroy(LoopbackGroup* grp) {
    if (!grp) return;
    for (auto e : grp->ev)
        if (e) cudaEventDestroy(e);
    delete grp;
}

int loopback_group_size(const LoopbackGroup* grp) { return grp->R; }

Comm* make_loopback_comm(LoopbackGroup* grp, int rank) {
    require(grp != nullptr && rank >= 0 && rank < grp->R, "loopback: bad group or rank");
    auto* c = new LoopbackComm;
    c->g = grp;
    c->rank = rank;
    c->nranks = grp->R;
    return c;
}

} // namespace cpg
