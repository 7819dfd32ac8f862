// nccl_dl.cpp -- NCCL entry points resolved at run time.
//
// The library does not link libnccl: in a PyTorch process the torch-bundled
// libnccl.so.2 is already loaded, and dlopen by soname returns that same copy
// (one NCCL per process); standalone C++ hosts get the system libnccl.so.2.
// Only the sharded (multi-GPU) path touches NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <thread>
#include <string>

#include "cpg_graph.hpp"

namespace cpg {

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_async_error)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
            if (!a.h) a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) return;
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(a.h, "ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(a.h, "ncclCommInitRank"));
        a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(a.h, "ncclAllGather"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(a.h, "ncclAllReduce"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(a.h, "ncclCommDestroy"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(a.h, "ncclGetErrorString"));
        a.get_async_error = reinterpret_cast<decltype(a.get_async_error)>(dlsym(a.h, "ncclCommGetAsyncError"));
        a.comm_abort = reinterpret_cast<decltype(a.comm_abort)>(dlsym(a.h, "ncclCommAbort"));
    });
    if (!a.h || !a.get_unique_id || !a.comm_init_rank || !a.all_gather || !a.all_reduce)
        fail(CPG_ENCCL, "libnccl.so.2 not loadable: " + std::string(dlerror() ? dlerror() : "missing symbols"));
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(CPG_ENCCL, std::string(what) + ": " + (api().error_string ? api().error_string(r) : "nccl error"));
}

} // namespace

void nccl_get_unique_id(void* out128) {
    ncclUniqueId id;
    check(api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, sizeof(id));
}

void* nccl_comm_init(const void* id128, int nranks, int rank) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm = nullptr;
    check(api().comm_init_rank(&comm, nranks, id, rank), "ncclCommInitRank");
    return comm;
}

// In place when send == recv + rank*count (the replicated iterate).
void nccl_allgather_f64(const double* send, double* recv, size_t count, void* comm, cudaStream_t st) {
    check(api().all_gather(send, recv, count, ncclFloat64, static_cast<ncclComm_t>(comm), st), "ncclAllGather");
}

void nccl_allreduce_sum_f64(const double* send, double* recv, size_t count, void* comm, cudaStream_t st) {
    check(api().all_reduce(send, recv, count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm), st),
          "ncclAllReduce");
}

// Asynchronous communicator errors (a peer died, a network failure): polled
// while a sharded query waits for its stream, so a dead peer surfaces as
// CPG_ENCCL instead of a hang.  On error the communicator is aborted, which
// releases the kernels blocked in it.
void nccl_check_async(void* comm) {
    if (!comm || !api().get_async_error) return;
    ncclResult_t st = ncclSuccess;
    const ncclResult_t r = api().get_async_error(static_cast<ncclComm_t>(comm), &st);
    if (r == ncclSuccess && (st == ncclSuccess || st == ncclInProgress)) return;
    const ncclResult_t bad = r != ncclSuccess ? r : st;
    fail(CPG_ENCCL, std::string("NCCL communicator failed: ") + (api().error_string ? api().error_string(bad) : "error"));
}

void nccl_comm_destroy(void* comm) {
    if (comm && api().comm_destroy) api().comm_destroy(static_cast<ncclComm_t>(comm));
}

namespace {
struct NcclComm final : Comm {
    void* c = nullptr;
    ~NcclComm() override { nccl_comm_destroy(c); }
    void allgather(const double* send, double* recv, size_t count, cudaStream_t st) override {
        nccl_allgather_f64(send, recv, count, c, st);
    }
    void allreduce_sum(double* buf, size_t count, cudaStream_t st) override {
        nccl_allreduce_sum_f64(buf, buf, count, c, st);
    }
    void sync(cudaStream_t st) override {
        for (;;) {
            const cudaError_t e = cudaStreamQuery(st);
            if (e == cudaSuccess) return;
            if (e != cudaErrorNotReady) CPG_CUDA(e);
            nccl_check_async(c);
            std::this_thread::sleep_for(std::chrono::microseconds(50));
        }
    }
    void* nccl() override { return c; }
};
} // namespace

Comm* make_nccl_comm(const void* id128, int nranks, int rank) {
    auto* m = new NcclComm;
    try {
        m->c = nccl_comm_init(id128, nranks, rank);
    } catch (...) {
        delete m;
        throw;
    }
    m->rank = rank;
    m->nranks = nranks;
    return m;
}

} // namespace cpg
