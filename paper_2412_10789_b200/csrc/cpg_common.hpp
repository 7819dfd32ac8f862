// cpg_common.hpp -- shared internals of libcpg.so (not part of the ABI).
#pragma once

#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "cpg.h"

namespace cpg {

// Exceptions thrown inside the library and mapped to status codes at the
// C-ABI edge (mirrors the reference's error.hpp taxonomy).
struct Error : std::runtime_error {
    int code;
    Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const std::string& msg) {
    if (!ok) fail(CPG_EINVAL, msg);
}

void set_last_error(const std::string& msg);

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return CPG_OK;
    } catch (const Error& e) {
        set_last_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        set_last_error("out of host memory");
        return CPG_ENOMEM;
    } catch (const std::exception& e) {
        set_last_error(e.what());
        return CPG_ECUDA;
    }
}

// Host-side math restated from the reference (host_math.cpp).
void ppr_cheby_coeffs(double alpha, uint64_t max_index, double* out);
void hkpr_cheby_coeffs(double t, uint64_t max_index, double* out);
cpg_plan plan_truncation(int family, double param, double epsilon);
uint64_t validate_csr(const uint64_t* offsets, const uint32_t* nbrs, uint64_t n, uint64_t nnz);
uint64_t structure_hash(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n, uint64_t nnz);

} // namespace cpg

#define CPG_CUDA(call)                                                                  \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess)                                                          \
            ::cpg::fail(e_ == cudaErrorMemoryAllocation ? CPG_ENOMEM : CPG_ECUDA,       \
                        std::string(#call) + ": " + cudaGetErrorString(e_));            \
    } while (0)
