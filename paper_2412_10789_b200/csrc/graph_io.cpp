// graph_io.cpp -- the host-side formats either side of the path: the edge-list
// text rules of the reference loader, the CPGR binary CSR cache and the CPGT
// ground-truth cache.  Reference paths are relative to /root/reference/proj.
//
//   load_edge_list line rules        src/graph.cpp:126-151
//   write_csr_cache / read_csr_cache src/graph.cpp:217-255 (graph.hpp:87-90)
//   CPGT write / read / filename     src/eval.cpp:92-160
//
// The text parser is multi-threaded (chunks split at newlines); the error it
// reports is the one the reference's sequential loop would hit first (smallest
// line number), with the reference's message.  Label pairs go to the GPU
// ingest (graphgen.cu) for interning / symmetrising / dedup.
#include <algorithm>
#include <cctype>
#include <cerrno>
#include <cinttypes>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <string>
#include <thread>
#include <vector>

#include "cpg_common.hpp"

namespace cpg {
namespace {

// isspace in the "C" locale: what istream's skipws skips.
inline bool ws(char c) { return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r'; }

// istream >> int64_t (num_get, decimal): skip whitespace, optional sign, >= 1
// digit, stop at the first non-digit; overflow fails.  Returns false on failure.
bool read_i64(const char*& p, const char* end, int64_t& v) {
    while (p < end && ws(*p)) ++p;
    bool neg = false;
    if (p < end && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p >= end || *p < '0' || *p > '9') return false;
    uint64_t mag = 0;
    const uint64_t lim = neg ? (uint64_t{1} << 63) : static_cast<uint64_t>(std::numeric_limits<int64_t>::max());
    bool over = false;
    while (p < end && *p >= '0' && *p <= '9') {
        const uint64_t d = static_cast<uint64_t>(*p - '0');
        if (mag > (lim - d) / 10) over = true;
        else mag = mag * 10 + d;
        ++p;
    }
    if (over) return false;
    v = neg ? static_cast<int64_t>(0 - mag) : static_cast<int64_t>(mag);
    return true;
}

struct ChunkResult {
    std::vector<int64_t> pairs;
    uint64_t lines = 0;        // lines started in this chunk
    uint64_t err_line = 0;     // 1-based line within the chunk, 0 = none
    std::string err;
};

// One chunk [b, e) that starts at a line start; every line that starts in it is parsed.
void parse_chunk(const char* b, const char* e, char comment, ChunkResult& r) {
    const char* p = b;
    while (p < e) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(e - p)));
        const char* le = nl ? nl : e;
        ++r.lines;
        // graph.cpp:129-130: blank (only " \t\r") or comment lines are skipped
        const char* q = p;
        while (q < le && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
        if (q < le && *q != comment) {
            const char* s = p;
            int64_t a = 0, c = 0;
            if (!read_i64(s, le, a) || !read_i64(s, le, c)) {  // graph.cpp:132-135
                r.err_line = r.lines;
                r.err = ": expected two integers, got \"" + std::string(p, le) + "\"";
                return;
            }
            while (s < le && ws(*s)) ++s;
            if (s < le) {  // graph.cpp:137-147: the next token must parse fully as a number
                const char* t = s;
                while (t < le && !ws(*t)) ++t;
                const std::string extra(s, t);
                char* stop = nullptr;
                std::strtod(extra.c_str(), &stop);
                if (stop == extra.c_str() || *stop != '\0') {
                    r.err_line = r.lines;
                    r.err = ": trailing garbage \"" + extra + "\"";
                    return;
                }
            }
            r.pairs.push_back(a);
            r.pairs.push_back(c);
        }
        p = nl ? nl + 1 : e;
    }
}

[[noreturn]] void fail_parse(const std::string& m) { fail(CPG_EPARSE, m); }

struct File {
    FILE* f = nullptr;
    File(const char* path, const char* mode) : f(std::fopen(path, mode)) {}
    ~File() {
        if (f) std::fclose(f);
    }
};

template <typename T>
bool read_raw(FILE* f, T& v) {
    return std::fread(&v, sizeof(T), 1, f) == 1;
}

constexpr char kCsrMagic[4] = {'C', 'P', 'G', 'R'};
constexpr char kTruthMagic[4] = {'C', 'P', 'G', 'T'};
constexpr uint32_t kVersion = 1;  // both formats (graph.cpp:219, eval.cpp:95)

// Header of a CPGR file; leaves f positioned at the offsets array.
void csr_header(FILE* f, uint64_t* n, uint64_t* m) {
    char magic[4] = {};
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kCsrMagic, 4) != 0)
        fail_parse("bad CSR cache magic");  // graph.cpp:237-238
    uint32_t version = 0;
    if (!read_raw(f, version)) fail_parse("unexpected end of binary stream");
    if (version != kVersion) fail_parse("unsupported CSR cache version " + std::to_string(version));
    if (!read_raw(f, *n) || !read_raw(f, *m)) fail_parse("unexpected end of binary stream");
    if (*n == 0 || *n > std::numeric_limits<uint32_t>::max())
        fail(CPG_ESTRUCT, "CSR cache node count out of range");  // graph.cpp:245-246
}

void truth_header(FILE* f, std::string* desc, uint64_t* source, uint64_t* n) {
    char magic[4] = {};
    if (std::fread(magic, 1, 4, f) != 4 || std::memcmp(magic, kTruthMagic, 4) != 0)
        fail_parse("bad truth cache magic");  // eval.cpp:128-129
    uint32_t version = 0, len = 0;
    if (!read_raw(f, version)) fail_parse("unexpected end of truth cache");
    if (version != kVersion) fail_parse("unsupported truth cache version " + std::to_string(version));
    if (!read_raw(f, len)) fail_parse("unexpected end of truth cache");
    desc->resize(len);
    if (len && std::fread(&(*desc)[0], 1, len, f) != len) fail_parse("truncated truth cache");
    if (!read_raw(f, *source) || !read_raw(f, *n)) fail_parse("unexpected end of truth cache");
}

}  // namespace
}  // namespace cpg

using namespace cpg;

extern "C" {

int cpg_parse_edge_text(const char* text, uint64_t len, char comment, int64_t* pairs, uint64_t cap_pairs,
                        uint64_t* n_pairs, int n_threads) {
    return guarded([&] {
        require((text || len == 0) && n_pairs, "null argument");
        const char* end = text + len;
        int T = n_threads > 0 ? n_threads : static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
        T = static_cast<int>(std::min<uint64_t>(static_cast<uint64_t>(T), std::max<uint64_t>(1, len >> 20)));
        // chunk starts: line starts at ~len/T
        std::vector<const char*> cut{text};
        for (int i = 1; i < T; ++i) {
            const char* p = std::max(cut.back(), text + len * static_cast<uint64_t>(i) / T);
            const char* nl = p < end ? static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)))
                                     : nullptr;
            if (!nl) break;
            cut.push_back(nl + 1);
        }
        cut.push_back(end);
        const size_t C = cut.size() - 1;
        std::vector<ChunkResult> res(C);
        std::vector<std::thread> th;
        for (size_t c = 1; c < C; ++c)
            th.emplace_back([&, c] { parse_chunk(cut[c], cut[c + 1], comment, res[c]); });
        if (C) parse_chunk(cut[0], cut[1], comment, res[0]);
        for (auto& t : th) t.join();
        // the first error in file order is the one the sequential loader reports
        uint64_t line0 = 0, total = 0;
        for (size_t c = 0; c < C; ++c) {
            if (res[c].err_line) fail_parse("line " + std::to_string(line0 + res[c].err_line) + res[c].err);
            line0 += res[c].lines;
            total += res[c].pairs.size() / 2;
        }
        *n_pairs = total;
        if (!pairs) return;
        require(cap_pairs >= total, "edge pair buffer too small");
        uint64_t at = 0;
        for (size_t c = 0; c < C; ++c) {
            std::memcpy(pairs + 2 * at, res[c].pairs.data(), res[c].pairs.size() * sizeof(int64_t));
            at += res[c].pairs.size() / 2;
        }
    });
}

int cpg_csr_cache_write(const char* path, const uint64_t* offsets, const uint32_t* neighbors, uint64_t n,
                        uint64_t nnz) {
    return guarded([&] {
        require(path && offsets && neighbors, "null argument");
        File f(path, "wb");
        if (!f.f) fail(CPG_EIO, std::string("cannot open CSR cache for writing: ") + path);
        const uint64_t m = nnz / 2;  // Graph::edge_count() (graph.hpp:29)
        bool ok = std::fwrite(kCsrMagic, 1, 4, f.f) == 4;
        ok = ok && std::fwrite(&kVersion, sizeof(kVersion), 1, f.f) == 1;
        ok = ok && std::fwrite(&n, 8, 1, f.f) == 1 && std::fwrite(&m, 8, 1, f.f) == 1;
        ok = ok && std::fwrite(offsets, 8, n + 1, f.f) == n + 1;
        ok = ok && (nnz == 0 || std::fwrite(neighbors, 4, nnz, f.f) == nnz);
        ok = std::fflush(f.f) == 0 && ok;
        if (!ok) fail(CPG_EIO, "write failure while emitting CSR cache");  // graph.cpp:231
    });
}

int cpg_csr_cache_info(const char* path, uint64_t* n, uint64_t* m) {
    return guarded([&] {
        require(path && n && m, "null argument");
        File f(path, "rb");
        if (!f.f) fail(CPG_EIO, std::string("cannot open CSR cache: ") + path);
        csr_header(f.f, n, m);
    });
}

int cpg_csr_cache_read(const char* path, uint64_t* offsets, uint32_t* neighbors, uint64_t n, uint64_t m) {
    return guarded([&] {
        require(path && offsets && (neighbors || m == 0), "null argument");
        File f(path, "rb");
        if (!f.f) fail(CPG_EIO, std::string("cannot open CSR cache: ") + path);
        uint64_t hn = 0, hm = 0;
        csr_header(f.f, &hn, &hm);
        require(hn == n && hm == m, "CSR cache header changed between info and read");
        if (std::fread(offsets, 8, n + 1, f.f) != n + 1 || (m && std::fread(neighbors, 4, 2 * m, f.f) != 2 * m))
            fail_parse("truncated CSR cache");  // graph.cpp:253
    });
}

int cpg_truth_cache_write(const char* path, const char* kernel_descriptor, uint64_t source, const double* values,
                          uint64_t n) {
    return guarded([&] {
        require(path && kernel_descriptor && (values || n == 0), "null argument");
        File f(path, "wb");
        if (!f.f) fail(CPG_EIO, std::string("cannot open truth cache for writing: ") + path);
        const uint32_t len = static_cast<uint32_t>(std::strlen(kernel_descriptor));
        bool ok = std::fwrite(kTruthMagic, 1, 4, f.f) == 4;
        ok = ok && std::fwrite(&kVersion, 4, 1, f.f) == 1 && std::fwrite(&len, 4, 1, f.f) == 1;
        ok = ok && (len == 0 || std::fwrite(kernel_descriptor, 1, len, f.f) == len);
        ok = ok && std::fwrite(&source, 8, 1, f.f) == 1 && std::fwrite(&n, 8, 1, f.f) == 1;
        ok = ok && (n == 0 || std::fwrite(values, 8, n, f.f) == n);
        ok = std::fflush(f.f) == 0 && ok;
        if (!ok) fail(CPG_EIO, "write failure while emitting truth cache");  // eval.cpp:123
    });
}

int cpg_truth_cache_info(const char* path, char* desc, uint64_t desc_cap, uint64_t* source, uint64_t* n) {
    return guarded([&] {
        require(path && desc && desc_cap && source && n, "null argument");
        File f(path, "rb");
        if (!f.f) fail(CPG_EIO, std::string("cannot open truth cache: ") + path);
        std::string d;
        truth_header(f.f, &d, source, n);
        require(d.size() < desc_cap, "descriptor buffer too small");
        std::memcpy(desc, d.c_str(), d.size() + 1);
    });
}

int cpg_truth_cache_read(const char* path, double* values, uint64_t n) {
    return guarded([&] {
        require(path && (values || n == 0), "null argument");
        File f(path, "rb");
        if (!f.f) fail(CPG_EIO, std::string("cannot open truth cache: ") + path);
        std::string d;
        uint64_t s = 0, hn = 0;
        truth_header(f.f, &d, &s, &hn);
        require(hn == n, "truth cache length changed between info and read");
        if (n && std::fread(values, 8, n, f.f) != n) fail_parse("truncated truth cache");  // eval.cpp:141
    });
}

// truth_cache_filename (eval.cpp:147-156): "cpgt-<hash hex16>-<descriptor, [^A-Za-z0-9.-] -> _>-s<source>.bin"
int cpg_truth_cache_filename(uint64_t structure_hash, const char* kernel_descriptor, uint64_t source, char* out,
                             uint64_t cap) {
    return guarded([&] {
        require(kernel_descriptor && out, "null argument");
        std::string desc(kernel_descriptor);
        for (char& c : desc)
            if (!std::isalnum(static_cast<unsigned char>(c)) && c != '.' && c != '-') c = '_';
        char hex[17];
        std::snprintf(hex, sizeof(hex), "%016llx", static_cast<unsigned long long>(structure_hash));
        const std::string name = std::string("cpgt-") + hex + "-" + desc + "-s" + std::to_string(source) + ".bin";
        require(name.size() < cap, "filename buffer too small");
        std::memcpy(out, name.c_str(), name.size() + 1);
    });
}

}  // extern "C"
