// chebyprop_b200.hpp -- header-only C++ drop-in for the reference's ChebyPower.
//
//   #include "chebyprop_b200/chebyprop_b200.hpp"
//   chebyprop::Estimate est = chebyprop::cuda::cheby_power(g, kernel, source, K);
//
// Same signature and semantics as the reference's
//   Estimate cheby_power(const Graph&, const Kernel&, NodeId, std::size_t,
//                        const StepObserver& = {})       include/chebyprop/solvers.hpp:59-61
//   Estimate cheby_power_vec(const Graph&, const Kernel&, const NodeVector&,
//                            std::size_t, const StepObserver& = {})  solvers.hpp:62-64
// (reference paths relative to /root/reference/proj), running on a B200
// through the C ABI in cpg.h.  The graph, kernel and estimate types are
// template parameters so the reference's own chebyprop::Graph / Kernel /
// Estimate plug in unchanged (duck-typed on node_count(), offsets(),
// neighbor_array(), volume(), structure_hash(), family(), alpha(), t(),
// cheby_coeffs()).  The device copy of a graph is cached per structure hash
// (graph.hpp:48) for the life of the process.
//
// Errors: CPG_EINVAL -> ParameterErrorT (the reference's ParameterError when
// passed as the template argument), anything else -> std::runtime_error.
#pragma once

#include <chrono>
#include <cstdint>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "cpg.h"

namespace chebyprop_b200 {

struct GraphHandle {
    cpg_graph* g = nullptr;
    ~GraphHandle() {
        if (g) cpg_graph_destroy(g);
    }
};

template <typename ParameterErrorT>
inline void check(int rc) {
    if (rc == CPG_OK) return;
    const std::string msg = cpg_last_error();
    if (rc == CPG_EINVAL) throw ParameterErrorT(msg);
    throw std::runtime_error("cpg status " + std::to_string(rc) + ": " + msg);
}

// Device copy of a host CSR graph, cached by structure hash (+ size) per device.
template <typename Graph, typename ParameterErrorT>
cpg_graph* device_graph(const Graph& g, int device) {
    static std::mutex mu;
    static std::map<std::tuple<uint64_t, uint64_t, uint64_t, int>, std::shared_ptr<GraphHandle>> cache;
    const auto key = std::make_tuple(static_cast<uint64_t>(g.structure_hash()), static_cast<uint64_t>(g.node_count()),
                                     static_cast<uint64_t>(g.volume()), device);
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second->g;
    auto h = std::make_shared<GraphHandle>();
    check<ParameterErrorT>(cpg_graph_create(g.offsets().data(), g.neighbor_array().data(),
                                            static_cast<uint32_t>(g.node_count()), g.volume(), device, 0, &h->g));
    cache[key] = h;
    return h->g;
}

} // namespace chebyprop_b200

namespace chebyprop {
namespace cuda {

// cheby_power (solvers.cpp:236-239) on the GPU.  Coefficients come from the
// kernel inside the call (solvers.cpp:205); stats mirror solvers.cpp:228-232.
// A non-empty observer takes the slow trace path: T_k(P)e_s and the partial
// estimate after every step are copied back (solvers.cpp:215, 219, 226).
template <typename Estimate, typename Graph, typename Kernel, typename ParameterErrorT, typename Observer>
Estimate cheby_power_t(const Graph& g, const Kernel& kernel, uint32_t source, std::size_t cheby_steps,
                       const Observer& observer, int device = 0) {
    if (cheby_steps < 1) throw ParameterErrorT("cheby_power: cheby_steps must be >= 1");
    if (source >= g.node_count())
        throw ParameterErrorT("source node " + std::to_string(source) + " out of range");
    // the first call's upload is graph loading, which the reference's wall_seconds
    // excludes (README.md:93-95): the clock starts once the device graph exists
    cpg_graph* dg = chebyprop_b200::device_graph<Graph, ParameterErrorT>(g, device);
    const auto start = std::chrono::steady_clock::now();
    const std::vector<double> c = kernel.cheby_coeffs(cheby_steps);
    const std::size_t n = g.node_count();
    Estimate est;
    est.values.assign(n, 0.0);
    const uint32_t K = static_cast<uint32_t>(cheby_steps);
    if (observer) {
        std::vector<double> rt((K + 1) * n), et((K + 1) * n);
        chebyprop_b200::check<ParameterErrorT>(
            cpg_chebypower_trace(dg, c.data(), K, source, est.values.data(), rt.data(), et.data()));
        std::vector<double> r(n), e(n);
        for (uint32_t k = 0; k <= K; ++k) {
            r.assign(rt.begin() + k * n, rt.begin() + (k + 1) * n);
            e.assign(et.begin() + k * n, et.begin() + (k + 1) * n);
            observer(k, r, e);
        }
    } else {
        cpg_stats st{};
        chebyprop_b200::check<ParameterErrorT>(cpg_chebypower(dg, c.data(), K, &source, 1, est.values.data(), &st));
    }
    est.stats.iterations = K;
    est.stats.push_work = static_cast<std::uint64_t>(K) * g.volume();
    est.stats.algorithm = "chebypower";
    est.stats.params = "K=" + std::to_string(K);
    est.stats.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    return est;
}

// cheby_power_vec (solvers.cpp:197-234) on the GPU.  A non-empty observer takes
// the trace slow path (solvers.cpp:215, 219, 226), as cheby_power_t does.
template <typename Estimate, typename Graph, typename Kernel, typename ParameterErrorT, typename Observer>
Estimate cheby_power_vec_t(const Graph& g, const Kernel& kernel, const std::vector<double>& seed,
                           std::size_t cheby_steps, const Observer& observer, int device = 0) {
    if (seed.size() != g.node_count()) throw ParameterErrorT("seed vector length mismatch");
    if (cheby_steps < 1) throw ParameterErrorT("cheby_power: cheby_steps must be >= 1");
    cpg_graph* dg = chebyprop_b200::device_graph<Graph, ParameterErrorT>(g, device);
    const auto start = std::chrono::steady_clock::now();
    const std::vector<double> c = kernel.cheby_coeffs(cheby_steps);
    const std::size_t n = g.node_count();
    Estimate est;
    est.values.assign(n, 0.0);
    const uint32_t K = static_cast<uint32_t>(cheby_steps);
    if (observer) {
        std::vector<double> rt((K + 1) * n), et((K + 1) * n);
        chebyprop_b200::check<ParameterErrorT>(
            cpg_chebypower_vec_trace(dg, c.data(), K, seed.data(), est.values.data(), rt.data(), et.data()));
        std::vector<double> r(n), e(n);
        for (uint32_t k = 0; k <= K; ++k) {
            r.assign(rt.begin() + k * n, rt.begin() + (k + 1) * n);
            e.assign(et.begin() + k * n, et.begin() + (k + 1) * n);
            observer(k, r, e);
        }
    } else {
        cpg_stats st{};
        chebyprop_b200::check<ParameterErrorT>(
            cpg_chebypower_vec(dg, c.data(), K, seed.data(), 1, est.values.data(), &st));
    }
    est.stats.iterations = K;
    est.stats.push_work = static_cast<std::uint64_t>(K) * g.volume();
    est.stats.algorithm = "chebypower";
    est.stats.params = "K=" + std::to_string(K);
    est.stats.wall_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - start).count();
    return est;
}

} // namespace cuda
} // namespace chebyprop

// With the reference headers on the include path, define CHEBYPROP_B200_REFERENCE_TYPES
// before including this file to get the exact reference signatures:
//   chebyprop::cuda::cheby_power(const Graph&, const Kernel&, NodeId, std::size_t,
//                                const StepObserver& = {})
//   chebyprop::cuda::cheby_power_vec(const Graph&, const Kernel&, const NodeVector&,
//                                    std::size_t, const StepObserver& = {})
#ifdef CHEBYPROP_B200_REFERENCE_TYPES
#include "chebyprop/error.hpp"
#include "chebyprop/solvers.hpp"
namespace chebyprop {
namespace cuda {
inline Estimate cheby_power(const Graph& g, const Kernel& kernel, NodeId source, std::size_t cheby_steps,
                            const StepObserver& observer = {}) {
    return cheby_power_t<Estimate, Graph, Kernel, ParameterError>(g, kernel, source, cheby_steps, observer);
}
inline Estimate cheby_power_vec(const Graph& g, const Kernel& kernel, const NodeVector& seed,
                                std::size_t cheby_steps, const StepObserver& observer = {}) {
    return cheby_power_vec_t<Estimate, Graph, Kernel, ParameterError>(g, kernel, seed, cheby_steps, observer);
}
} // namespace cuda
} // namespace chebyprop
#endif
