// tests/cpp/dropin_test.cpp -- the drop-in C++ API against the reference's own
// types.  Built by oracle/Makefile (target `dropin`) with the UNMODIFIED
// reference sources + libcpg.so; run by tests/test_gpu_dropin.py on a B200.
//
// Restates the reference's ChebyPower cases (test_solvers.cpp:88-129,
// acceptance.cpp:139-157 C4, :349-360 C13) with chebyprop::cuda::cheby_power
// in place of chebyprop::cheby_power, plus vector parity against the
// reference on seeded graphs.
#define CHEBYPROP_B200_REFERENCE_TYPES
#include "chebyprop_b200/chebyprop_b200.hpp"

#include <cmath>
#include <cstdio>
#include <sstream>

#include "chebyprop/eval.hpp"
#include "chebyprop/rng.hpp"

using namespace chebyprop;

static int failures = 0;
#define CHECK(cond)                                                          \
    do {                                                                     \
        if (!(cond)) {                                                       \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                      \
        }                                                                    \
    } while (0)

static Graph text_graph(const std::string& t) {
    std::istringstream in(t);
    return load_edge_list(in);
}

// tests/oracles.hpp:162-178 restated (ring + seeded chords).
static Graph make_graph(std::size_t n, std::size_t extra, std::uint64_t seed) {
    SplitMix64 rng(seed);
    std::ostringstream out;
    for (std::size_t i = 0; i < n; ++i) out << i << ' ' << (i + 1) % n << '\n';
    for (std::size_t e = 0; e < extra; ++e) {
        const auto a = rng.next_below(n), b = rng.next_below(n);
        if (a != b) out << a << ' ' << b << '\n';
    }
    return text_graph(out.str());
}

static double linf(const NodeVector& a, const NodeVector& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.size(); ++i) m = std::max(m, std::abs(a[i] - b[i]));
    return m;
}

int main() {
    const Graph star = text_graph("0 1\n0 2\n0 3\n");
    const Graph path3 = text_graph("0 1\n1 2\n");
    {  // K = 1 is the two-term truncation (test_solvers.cpp:89-100)
        const Kernel k = Kernel::ppr(0.2);
        const auto c = k.cheby_coeffs(1);
        const auto est = cuda::cheby_power(star, k, 1, 1);
        NodeVector e(4, 0.0);
        e[1] = 1.0;
        const NodeVector pe = apply_walk(star, e);
        for (NodeId u = 0; u < 4; ++u) CHECK(std::abs(est.values[u] - (c[0] * e[u] + c[1] * pe[u])) <= 1e-14);
        CHECK(est.stats.iterations == 1);
    }
    {  // star r_3 lands back on the hub (:101-113), observer path
        NodeVector r3;
        cuda::cheby_power(star, Kernel::ppr(0.2), 1, 3, [&](std::uint32_t k, const NodeVector& r, const NodeVector&) {
            if (k == 3) r3 = r;
        });
        CHECK(r3.size() == 4);
        CHECK(std::abs(r3[0] - 1.0) <= 1e-14);
        CHECK(std::abs(r3[1]) < 1e-14 && std::abs(r3[2]) < 1e-14 && std::abs(r3[3]) < 1e-14);
    }
    {  // path3 reaches 1e-8 at the planned K (:114-121): compare with the exact PPR
        const Kernel k = Kernel::ppr(0.2);
        const auto plan = plan_truncation(k, 1e-8);
        const auto est = cuda::cheby_power(path3, k, 1, plan.cheby_steps);
        // exact: (I - 0.8 P) y = 0.2 e_1 on the path 0-1-2  =>  y = [0.25, 0.5, 0.25] * ... solve:
        // P = A D^-1: y0 = 0.8*0.5*y1, y2 = 0.8*0.5*y1, y1 = 0.2 + 0.8*(y0 + y2) => y1 = 0.2/(1-0.64)
        const double y1 = 0.2 / (1.0 - 0.64), y0 = 0.4 * y1;
        const double l2 = std::sqrt(std::pow(est.values[0] - y0, 2) + std::pow(est.values[1] - y1, 2) +
                                    std::pow(est.values[2] - y0, 2));
        CHECK(l2 < 1e-8);
    }
    {  // mass conservation at every degree (:122-128, C13)
        const Graph g = make_graph(50, 80, 17);
        double worst = 0.0;
        cuda::cheby_power(g, Kernel::ppr(0.2), 7, 30, [&](std::uint32_t, const NodeVector& r, const NodeVector&) {
            double s = 0;
            for (double v : r) s += v;
            worst = std::max(worst, std::abs(s - 1.0));
        });
        CHECK(worst <= 1e-9);
    }
    {  // C4: l2 error within the tail bound, and vector parity with the reference
        for (std::uint64_t seed = 1; seed <= 5; ++seed) {
            const Graph g = make_graph(200 * seed, 300 * seed, seed);
            const NodeId s = g.node_count() / 2;
            for (const Kernel& kernel : {Kernel::ppr(0.2), Kernel::hkpr(5.0)}) {
                const NodeVector truth = ground_truth(g, kernel, s).values;
                for (double eps : {1e-3, 1e-6, 1e-8}) {
                    const auto plan = plan_truncation(kernel, eps);
                    const auto gpu = cuda::cheby_power(g, kernel, s, plan.cheby_steps);
                    const auto cpu = chebyprop::cheby_power(g, kernel, s, plan.cheby_steps);
                    double l2 = 0;
                    for (std::size_t i = 0; i < truth.size(); ++i) l2 += std::pow(truth[i] - gpu.values[i], 2);
                    CHECK(std::sqrt(l2) <= plan.tail_bound);
                    CHECK(linf(gpu.values, cpu.values) <= 1e-12);
                    CHECK(gpu.stats.push_work == cpu.stats.push_work);
                    CHECK(gpu.stats.iterations == cpu.stats.iterations);
                }
            }
        }
    }
    {  // cheby_power_vec parity
        const Graph g = make_graph(300, 500, 9);
        SplitMix64 rng(92);
        NodeVector x(g.node_count());
        for (auto& v : x) v = rng.next_double();
        const auto gpu = cuda::cheby_power_vec(g, Kernel::hkpr(5.0), x, 25);
        const auto cpu = chebyprop::cheby_power_vec(g, Kernel::hkpr(5.0), x, 25);
        CHECK(linf(gpu.values, cpu.values) <= 1e-12);
        // observer on cheby_power_vec (solvers.hpp:62-64): the same (k, r_k, yhat_k) sequence
        std::vector<NodeVector> gr, ge, cr, ce;
        const auto gpu_o = cuda::cheby_power_vec(g, Kernel::hkpr(5.0), x, 25,
                                                 [&](std::size_t, const NodeVector& r, const NodeVector& e) {
                                                     gr.push_back(r);
                                                     ge.push_back(e);
                                                 });
        chebyprop::cheby_power_vec(g, Kernel::hkpr(5.0), x, 25,
                                   [&](std::size_t, const NodeVector& r, const NodeVector& e) {
                                       cr.push_back(r);
                                       ce.push_back(e);
                                   });
        CHECK(gr.size() == cr.size() && gr.size() == 26);
        double worst = 0;
        for (std::size_t k = 0; k < std::min(gr.size(), cr.size()); ++k)
            worst = std::max({worst, linf(gr[k], cr[k]), linf(ge[k], ce[k])});
        CHECK(worst <= 1e-12);
        CHECK(linf(gpu_o.values, cpu.values) <= 1e-12);
    }
    {  // error behaviour (solvers.cpp:28-29, :201)
        bool threw = false;
        try {
            cuda::cheby_power(path3, Kernel::ppr(0.2), 99, 5);
        } catch (const ParameterError&) {
            threw = true;
        }
        CHECK(threw);
        threw = false;
        try {
            cuda::cheby_power(path3, Kernel::ppr(0.2), 0, 0);
        } catch (const ParameterError&) {
            threw = true;
        }
        CHECK(threw);
    }
    std::printf("%s (%d failures)\n", failures ? "FAILED" : "OK", failures);
    return failures ? 1 : 0;
}
