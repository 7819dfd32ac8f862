// host_math.cpp -- host-side part of the drop-in surface, restated in C++:
// Chebyshev coefficients, the truncation rule, kernel spec strings and the
// Graph::from_csr invariants.  O(K) / O(nnz) host work, off the device path.
// References are to /root/reference/proj.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cpg_common.hpp"

namespace cpg {

namespace {
thread_local std::string t_last_error;

void check_alpha(double alpha) { // kernels.cpp:26-29
    require(alpha > 0.0 && alpha < 1.0, "ppr: alpha must lie in (0,1), got " + std::to_string(alpha));
}
void check_t(double t) { // kernels.cpp:31-33
    require(t > 0.0, "hkpr: t must be positive, got " + std::to_string(t));
}
constexpr uint64_t kTruncationCap = 1000000; // kernels.cpp:233
} // namespace

void set_last_error(const std::string& msg) { t_last_error = msg; }

// gamma = alpha/sqrt(2a-a^2), beta = (1-a)/(1+sqrt(2a-a^2)); c0 = gamma,
// c_k = 2 gamma beta^k built by repeated multiplication (kernels.cpp:157-170).
void ppr_cheby_coeffs(double alpha, uint64_t max_index, double* c) {
    check_alpha(alpha);
    const double root = std::sqrt(2.0 * alpha - alpha * alpha);
    const double gamma = alpha / root;
    const double beta = (1.0 - alpha) / (1.0 + root);
    c[0] = gamma;
    double term = 2.0 * gamma;
    for (uint64_t k = 1; k <= max_index; ++k) {
        term *= beta;
        c[k] = term;
    }
}

// e^-t I_k(t) via Miller's backward recurrence from max(K, ceil t) + 40,
// rescaled near the double range, normalised by e^-t (I0 + 2 sum Ik) = 1
// (kernels.cpp:172-194).
void hkpr_cheby_coeffs(double t, uint64_t max_index, double* c) {
    check_t(t);
    const uint64_t start = std::max<uint64_t>(max_index, static_cast<uint64_t>(std::ceil(t))) + 40;
    std::vector<double> f(start + 2, 0.0);
    f[start] = 1e-30;
    for (uint64_t n = start; n >= 1; --n) {
        f[n - 1] = f[n + 1] + (2.0 * static_cast<double>(n) / t) * f[n];
        if (f[n - 1] > 1e280)
            for (uint64_t j = n - 1; j <= start + 1; ++j) f[j] *= 1e-280;
    }
    double norm = f[0];
    for (uint64_t k = 1; k <= start; ++k) norm += 2.0 * f[k];
    c[0] = f[0] / norm;
    for (uint64_t k = 1; k <= max_index; ++k) c[k] = 2.0 * f[k] / norm;
}

// Smallest K >= 1 whose exact Chebyshev tail is below eps (kernels.cpp:253-341).
cpg_plan plan_truncation(int family, double param, double epsilon) {
    require(epsilon > 0.0 && epsilon < 1.0, "plan_truncation: epsilon must lie in (0,1)");
    cpg_plan plan{1, 1, epsilon, 0.0};
    if (family == CPG_PPR) {
        const double alpha = param;
        check_alpha(alpha);
        const double root = std::sqrt(2.0 * alpha - alpha * alpha);
        const double gamma = alpha / root;
        const double beta = (1.0 - alpha) / (1.0 + root);
        auto tail = [&](uint64_t K) { // 2 gamma beta^{K+1} / (1 - beta), :266-270
            return 2.0 * gamma / (1.0 - beta) * std::exp(static_cast<double>(K + 1) * std::log(beta));
        };
        uint64_t K = 1;
        while (tail(K) >= epsilon)
            require(++K <= kTruncationCap, "plan_truncation: Chebyshev tail stuck above epsilon");
        plan.cheby_steps = K;
        plan.tail_bound = tail(K);
        uint64_t N = 1; // Taylor tail (1-alpha)^N, :279-287
        double t = 1.0 - alpha;
        while (t >= epsilon) {
            t *= 1.0 - alpha;
            require(++N <= kTruncationCap, "plan_truncation: Taylor tail stuck above epsilon");
        }
        plan.taylor_steps = N;
        return plan;
    }
    require(family == CPG_HKPR, "plan_truncation: unknown kernel family");
    const double t = param;
    check_t(t);
    for (uint64_t horizon = 64;; horizon = std::min(horizon * 2, kTruncationCap)) { // :294-308
        std::vector<double> c(horizon + 1);
        hkpr_cheby_coeffs(t, horizon, c.data());
        double prefix = 0.0;
        for (uint64_t k = 0; k <= horizon; ++k) { // cheby_steps_from_prefix, :237-249
            prefix += c[k];
            const double tail = std::max(0.0, 1.0 - prefix);
            if (k >= 1 && tail < epsilon) {
                plan.cheby_steps = k;
                plan.tail_bound = tail;
                goto taylor;
            }
        }
        require(horizon < kTruncationCap, "plan_truncation: Chebyshev tail stuck above epsilon");
    }
taylor: {
    double z = std::exp(-t), prefix = 0.0; // :310-322
    uint64_t N = 0;
    for (;;) {
        prefix += z;
        ++N;
        if (1.0 - prefix < epsilon) break;
        require(N <= kTruncationCap, "plan_truncation: Taylor tail stuck above epsilon");
        z *= t / static_cast<double>(N);
    }
    plan.taylor_steps = std::max<uint64_t>(N, 1);
}
    return plan;
}

// FNV-1a over (n as u32, m as u64, offsets, neighbors): graph.cpp:24-31, 97-102.
uint64_t structure_hash(const uint64_t* offsets, const uint32_t* nbrs, uint32_t n, uint64_t nnz) {
    uint64_t h = 0xcbf29ce484222325ull;
    auto mix = [&h](const void* data, size_t len) {
        const auto* p = static_cast<const unsigned char*>(data);
        for (size_t i = 0; i < len; ++i) {
            h ^= p[i];
            h *= 0x100000001b3ull;
        }
    };
    const uint64_t m = nnz / 2;
    mix(&n, sizeof(n));
    mix(&m, sizeof(m));
    mix(offsets, (static_cast<size_t>(n) + 1) * sizeof(uint64_t));
    mix(nbrs, nnz * sizeof(uint32_t));
    return h;
}

// Graph::from_csr invariants (graph.cpp:51-95), checked with host threads.
uint64_t validate_csr(const uint64_t* offsets, const uint32_t* nbrs, uint64_t n, uint64_t nnz) {
    auto bad = [](const char* m) { fail(CPG_ESTRUCT, m); };
    if (offsets == nullptr || offsets[0] != 0) bad("CSR offsets must start at 0");
    if (n == 0) bad("empty graph after cleaning");
    if (n > 0xffffffffull) bad("node count exceeds 32-bit id range");
    if (offsets[n] != nnz) bad("CSR offsets do not cover the neighbor array");
    if (nnz % 2 != 0) bad("undirected CSR needs an even neighbor count");
    unsigned nt = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    std::vector<std::string> errs(nt);
    auto rows = [&](unsigned tid, bool symmetry) {
        for (uint64_t u = tid; u < n; u += nt) {
            const uint64_t b = offsets[u], e = offsets[u + 1];
            if (!symmetry) {
                if (e < b) { errs[tid] = "CSR offsets not monotone"; return; }
                if (e == b) { errs[tid] = "node with degree 0"; return; }
                if (e > nnz) { errs[tid] = "CSR offsets exceed the neighbor array"; return; }
                for (uint64_t i = b; i < e; ++i) {
                    const uint32_t v = nbrs[i];
                    if (v >= n) { errs[tid] = "neighbor id out of range"; return; }
                    if (v == u) { errs[tid] = "self-loop in CSR"; return; }
                    if (i > b && nbrs[i - 1] >= v) { errs[tid] = "neighbor list not sorted/deduplicated"; return; }
                }
            } else {
                for (uint64_t i = b; i < e; ++i) {
                    const uint32_t v = nbrs[i];
                    const uint32_t* lo = nbrs + offsets[v];
                    const uint32_t* hi = nbrs + offsets[v + 1];
                    if (!std::binary_search(lo, hi, static_cast<uint32_t>(u))) {
                        errs[tid] = "adjacency not symmetric";
                        return;
                    }
                }
            }
        }
    };
    for (int pass = 0; pass < 2; ++pass) {
        std::vector<std::thread> th;
        for (unsigned t = 0; t < nt; ++t) th.emplace_back(rows, t, pass == 1);
        for (auto& x : th) x.join();
        for (auto& e : errs)
            if (!e.empty()) bad(e.c_str());
    }
    return structure_hash(offsets, nbrs, static_cast<uint32_t>(n), nnz);
}

} // namespace cpg

using namespace cpg;

extern "C" {

const char* cpg_last_error(void) { return t_last_error.c_str(); }
const char* cpg_version(void) { return "cpg 0.1 (sm_100a)"; }

int cpg_ppr_cheby_coeffs(double alpha, uint64_t max_index, double* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        ppr_cheby_coeffs(alpha, max_index, out);
    });
}

int cpg_hkpr_cheby_coeffs(double t, uint64_t max_index, double* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        hkpr_cheby_coeffs(t, max_index, out);
    });
}

int cpg_cheby_coeffs(int family, double param, uint64_t max_index, double* out) {
    if (family == CPG_PPR) return cpg_ppr_cheby_coeffs(param, max_index, out);
    if (family == CPG_HKPR) return cpg_hkpr_cheby_coeffs(param, max_index, out);
    set_last_error("unknown kernel family");
    return CPG_EINVAL;
}

// zeta_k: alpha (1-alpha)^k (PPR) or e^-t t^k / k! (HKPR), kernels.cpp:78-96.
int cpg_taylor_coeffs(int family, double param, uint64_t max_index, double* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        if (family == CPG_PPR) {
            check_alpha(param);
            double z = param;
            for (uint64_t k = 0; k <= max_index; ++k) {
                out[k] = z;
                z *= 1.0 - param;
            }
        } else {
            require(family == CPG_HKPR, "unknown kernel family");
            check_t(param);
            double z = std::exp(-param);
            for (uint64_t k = 0; k <= max_index; ++k) {
                out[k] = z;
                z *= param / static_cast<double>(k + 1);
            }
        }
    });
}

// N = ceil(ln(1e20)/alpha) (PPR) or ceil(2 t ln(1e20)) (HKPR), eval.cpp:39-50.
uint64_t cpg_ground_truth_steps(int family, double param) {
    const double target = std::log(1e20);
    if (family == CPG_PPR) return static_cast<uint64_t>(std::ceil(target / param));
    return static_cast<uint64_t>(std::ceil(2.0 * param * target));
}

int cpg_plan_truncation(int family, double param, double epsilon, cpg_plan* out) {
    return guarded([&] {
        require(out != nullptr, "null output");
        *out = plan_truncation(family, param, epsilon);
    });
}

// kernels.cpp:343-362: "<family>:<key>=<value>" with a full-string numeric parse.
int cpg_parse_kernel_spec(const char* spec_c, int* family, double* param) {
    return guarded([&] {
        require(spec_c && family && param, "null argument");
        const std::string spec(spec_c);
        const auto colon = spec.find(':');
        const std::string fam = spec.substr(0, colon);
        const std::string rest = colon == std::string::npos ? "" : spec.substr(colon + 1);
        const auto eq = rest.find('=');
        const std::string key = rest.substr(0, eq);
        const std::string value = eq == std::string::npos ? "" : rest.substr(eq + 1);
        auto parse = [&](const char* expected) {
            require(key == expected && !value.empty(), "bad kernel spec \"" + spec + "\"");
            double v = 0.0;
            auto [ptr, ec] = std::from_chars(value.data(), value.data() + value.size(), v);
            require(ec == std::errc{} && ptr == value.data() + value.size(),
                    "bad kernel parameter in \"" + spec + "\"");
            return v;
        };
        if (fam == "ppr") {
            const double a = parse("alpha");
            check_alpha(a);
            *family = CPG_PPR;
            *param = a;
        } else if (fam == "hkpr") {
            const double t = parse("t");
            check_t(t);
            *family = CPG_HKPR;
            *param = t;
        } else {
            fail(CPG_EINVAL, "unknown kernel family in \"" + spec + "\"");
        }
    });
}

int cpg_shard_plan(const uint64_t* offsets, uint32_t n, int nranks, int chunks, uint32_t* new_of_old,
                   uint32_t* rows_per_chunk) {
    return guarded([&] {
        require(offsets && new_of_old && rows_per_chunk && nranks >= 1 && chunks >= 1 && n > 0, "bad argument");
        std::vector<uint32_t> order(n);
        for (uint32_t i = 0; i < n; ++i) order[i] = i;
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
            return offsets[a + 1] - offsets[a] > offsets[b + 1] - offsets[b];
        });
        const uint64_t R = static_cast<uint64_t>(nranks), C = static_cast<uint64_t>(chunks);
        const uint64_t cr = (n + R * C - 1) / (R * C);
        for (uint64_t i = 0; i < n; ++i) {
            const uint64_t t = i / R;
            new_of_old[order[i]] = static_cast<uint32_t>((t % C) * R * cr + (i % R) * cr + t / C);
        }
        *rows_per_chunk = static_cast<uint32_t>(cr);
    });
}

int cpg_validate_csr(const uint64_t* offsets, const uint32_t* neighbors, uint64_t n, uint64_t nnz,
                     uint64_t* hash) {
    return guarded([&] {
        const uint64_t h = validate_csr(offsets, neighbors, n, nnz);
        if (hash) *hash = h;
    });
}

} // extern "C"
