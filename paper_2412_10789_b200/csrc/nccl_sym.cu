// nccl_sym.cu -- NCCL symmetric-memory windows for the fused step + all-gather.
//
// With NCCL >= 2.28 (the torch-bundled libnccl.so.2), buffers from
// ncclMemAlloc registered with ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)
// are mapped into every rank of the NVLink (LSA) team at one flat address
// range: peer p's copy of byte `off` is ncclGetLsaPointer(win, off, p).  The
// batched step kernels use these peer pointers to store every row they compute
// into all replicas of the iterate straight from the epilogue (SURVEY.md 8e
// "stretch"), so no separate all-gather runs; a one-element all-reduce per
// iteration is the barrier.
//
// Only this file includes the NCCL device headers (from the NCCL the build
// found, CPG_NCCL_DEVICE_API); the entry points are resolved at run time like
// nccl_dl.cpp.  Without them every function reports "unsupported" and the
// sharded path keeps the NCCL all-gather.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "cpg_graph.hpp"

#if CPG_NCCL_DEVICE_API
#include <nccl.h>
#include <nccl_device.h>
#endif

namespace cpg {

#if CPG_NCCL_DEVICE_API
namespace {

struct SymApi {
    void* h = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    ncclResult_t (*mem_alloc)(void**, size_t) = nullptr;
    ncclResult_t (*mem_free)(void*) = nullptr;
    ncclResult_t (*win_register)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
    ncclResult_t (*win_deregister)(ncclComm_t, ncclWindow_t) = nullptr;
    ncclTeam_t (*team_lsa)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
};

SymApi& sym() {
    static SymApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* nm : {"libnccl.so.2", "libnccl.so"}) {
            a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
            if (!a.h) a.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) return;
        auto get = [&](const char* s) { return dlsym(a.h, s); };
        a.get_version = reinterpret_cast<decltype(a.get_version)>(get("ncclGetVersion"));
        a.mem_alloc = reinterpret_cast<decltype(a.mem_alloc)>(get("ncclMemAlloc"));
        a.mem_free = reinterpret_cast<decltype(a.mem_free)>(get("ncclMemFree"));
        a.win_register = reinterpret_cast<decltype(a.win_register)>(get("ncclCommWindowRegister"));
        a.win_deregister = reinterpret_cast<decltype(a.win_deregister)>(get("ncclCommWindowDeregister"));
        a.team_lsa = reinterpret_cast<decltype(a.team_lsa)>(get("ncclTeamLsa"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(get("ncclGetErrorString"));
        int v = 0;
        // the window layout read by ncclGetLsaPointer is the one of the headers compiled here
        a.ok = a.get_version && a.get_version(&v) == ncclSuccess && v >= NCCL_VERSION_CODE - NCCL_PATCH &&
               v < NCCL_VERSION(NCCL_MAJOR, NCCL_MINOR + 1, 0) && a.mem_alloc && a.mem_free && a.win_register &&
               a.win_deregister && a.team_lsa;
    });
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        fail(CPG_ENCCL, std::string(what) + ": " + (sym().error_string ? sym().error_string(r) : "nccl error"));
}

__global__ void k_lsa_ptrs(ncclWindow_t w, int n, double** out) {
    for (int p = threadIdx.x; p < n; p += blockDim.x) out[p] = static_cast<double*>(ncclGetLsaPointer(w, 0, p));
}

} // namespace

bool nccl_sym_supported(void* comm, int nranks, int rank) {
    if (!comm || !sym().ok) return false;
    const ncclTeam_t t = sym().team_lsa(static_cast<ncclComm_t>(comm));
    return t.nRanks == nranks && t.rank == rank && t.stride == 1;  // one NVLink domain: LSA rank == world rank
}

void* nccl_sym_alloc(size_t bytes) {
    void* p = nullptr;
    check(sym().mem_alloc(&p, bytes), "ncclMemAlloc");
    return p;
}

void nccl_sym_free(void* p) {
    if (p && sym().mem_free) sym().mem_free(p);
}

void* nccl_sym_register(void* comm, void* buf, size_t bytes) {
    ncclWindow_t w = nullptr;
    check(sym().win_register(static_cast<ncclComm_t>(comm), buf, bytes, &w, NCCL_WIN_COLL_SYMMETRIC),
          "ncclCommWindowRegister");
    return w;
}

void nccl_sym_deregister(void* comm, void* win) {
    if (win && sym().win_deregister) sym().win_deregister(static_cast<ncclComm_t>(comm), static_cast<ncclWindow_t>(win));
}

void nccl_sym_peer_ptrs(void* win, int n, double** d_out, cudaStream_t st) {
    k_lsa_ptrs<<<1, 32, 0, st>>>(static_cast<ncclWindow_t>(win), n, d_out);
    CPG_CUDA(cudaGetLastError());
}

#else  // built without the NCCL device headers

bool nccl_sym_supported(void*, int, int) { return false; }
void* nccl_sym_alloc(size_t) { fail(CPG_ENCCL, "built without NCCL symmetric memory"); }
void nccl_sym_free(void*) {}
void* nccl_sym_register(void*, void*, size_t) { fail(CPG_ENCCL, "built without NCCL symmetric memory"); }
void nccl_sym_deregister(void*, void*) {}
void nccl_sym_peer_ptrs(void*, int, double**, cudaStream_t) { fail(CPG_ENCCL, "built without NCCL symmetric memory"); }

#endif

} // namespace cpg
