// engine_graphio.cuh — graph ingestion at GB scale: psp::load_graph /
// read_graph (src/graph_io.cpp:53-170) with the text parsed on the GPU.
//
// The reference reads line by line (getline + from_chars) and merges DIMACS
// arcs in a std::map. Here the whole file goes to HBM once and is parsed in
// parallel, with results identical to the reference's, errors included:
//   L1  newline index: per-256-byte chunk counts, a scan, the positions;
//   L2  one thread per line: trim, classify (blank / comment / header /
//       edge or arc / other), tokenize, parse the ids (exact u64 with
//       overflow) and the weight, correctly rounded on the device by
//       Eisel-Lemire (decimal_parse.cuh: digits[.digits][e[+-]digits],
//       <= 19 significant digits, normal results). Anything else (signs,
//       "inf", subnormal or overflowing values, malformed tokens, ids out
//       of range) marks the line HARD or ERR;
//   host the HARD / ERR lines, in file order up to the first real error,
//       are re-parsed by a line-for-line restatement of the reference's
//       loop body with std::from_chars -- the function the reference calls
//       -- in one batch, so values and ParseError messages are the
//       reference's. Header lines, "more edges than declared" and the
//       end-of-file checks follow the reference's order;
//   DIMACS normalisation on the device: arcs keyed (min, max) << 32, radix
//       sorted (stable, so file order survives among equal keys) and reduced
//       by key with min -- the std::map's first-inserted-wins on equal
//       weights and its (u, v) iteration order.
// The Graph itself (CSR + invariant checks) is build_csr, whose messages
// are the reference Graph constructor's.
#pragma once

#include <charconv>
#include <thread>
#include <fcntl.h>
#include <sys/stat.h>
#include <unistd.h>

#include "decimal_parse.cuh"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>

struct psp_graph {  // a parsed, validated graph (psp::Graph's edge input)
    uint64_t n = 0;
    std::vector<uint32_t> eu, ev;
    std::vector<double> ew;
};

namespace {

constexpr int PARSE_CHUNK = 256;

// min that keeps the earlier value on ties (std::map's first insert wins
// unless a later weight is strictly smaller, src/graph_io.cpp:129-130)
struct KeepFirstMin {
    __device__ __forceinline__ double operator()(double a, double b) const { return b < a ? b : a; }
};

__global__ void nl_count(const char* __restrict__ buf, uint64_t len, uint32_t* __restrict__ cnt,
                         uint64_t nchunks) {
    const uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const uint64_t a = c * PARSE_CHUNK, b = min(len, a + PARSE_CHUNK);
    uint32_t k = 0;
    for (uint64_t i = a; i < b; ++i) k += buf[i] == '\n';
    cnt[c] = k;
}

__global__ void nl_write(const char* __restrict__ buf, uint64_t len,
                         const uint32_t* __restrict__ off, uint64_t nchunks,
                         uint64_t* __restrict__ nl) {
    const uint64_t c = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (c >= nchunks) return;
    const uint64_t a = c * PARSE_CHUNK, b = min(len, a + PARSE_CHUNK);
    uint64_t at = off[c];
    for (uint64_t i = a; i < b; ++i)
        if (buf[i] == '\n') nl[at++] = i;
}

// line status
enum : uint8_t { LN_SKIP = 0, LN_HEADER = 1, LN_EDGE = 2, LN_ERR = 3, LN_HARD = 4 };
// line classes (first pass)
enum : uint8_t { CL_SKIP = 0, CL_SIG = 1, CL_P = 2, CL_A = 3, CL_OTHER = 4 };

struct LineSpan {
    uint64_t a, b;  // trimmed body [a, b)
};

__device__ __forceinline__ LineSpan line_body(const char* buf, uint64_t len, const uint64_t* nl,
                                              uint64_t nnl, uint64_t i) {
    uint64_t a = i == 0 ? 0 : nl[i - 1] + 1;
    uint64_t b = i < nnl ? nl[i] : len;
    // trim " \t\r" both ends (src/graph_io.cpp:19-23)
    while (a < b && (buf[a] == ' ' || buf[a] == '\t' || buf[a] == '\r')) ++a;
    while (b > a && (buf[b - 1] == ' ' || buf[b - 1] == '\t' || buf[b - 1] == '\r')) --b;
    return {a, b};
}

__global__ void classify_lines(const char* __restrict__ buf, uint64_t len,
                               const uint64_t* __restrict__ nl, uint64_t nnl, uint64_t nlines,
                               int dimacs, uint8_t* __restrict__ cls,
                               unsigned long long* __restrict__ firsts) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nlines) return;
    const LineSpan s = line_body(buf, len, nl, nnl, i);
    uint8_t c = CL_SKIP;
    if (s.a < s.b) {
        const char f = buf[s.a];
        if (!dimacs) c = f == '#' ? CL_SKIP : CL_SIG;
        else c = f == 'c' ? CL_SKIP : f == 'p' ? CL_P : f == 'a' ? CL_A : CL_OTHER;
    }
    cls[i] = c;
    // firsts[0] = first significant / 'p' line; firsts[1] = first 'a' or
    // other line (DIMACS: an error if it precedes the problem line)
    if (c == CL_SIG || c == CL_P) atomicMin(&firsts[0], (unsigned long long)i);
    if (c == CL_A || c == CL_OTHER) atomicMin(&firsts[1], (unsigned long long)i);
}

// Splits [a, b) on runs of ' '/'\t' (src/graph_io.cpp:26-37); up to 5 tokens.
__device__ __forceinline__ int split_tokens(const char* buf, uint64_t a, uint64_t b,
                                            uint64_t (&ta)[5], uint64_t (&tb)[5]) {
    int n = 0;
    uint64_t i = a;
    while (i < b) {
        while (i < b && (buf[i] == ' ' || buf[i] == '\t')) ++i;
        uint64_t j = i;
        while (j < b && buf[j] != ' ' && buf[j] != '\t') ++j;
        if (j > i) {
            if (n < 5) {
                ta[n] = i;
                tb[n] = j;
            }
            ++n;
        }
        i = j;
    }
    return n;
}

// from_chars<uint64_t> on a whole token: digits only, no overflow
__device__ __forceinline__ bool parse_u64(const char* buf, uint64_t a, uint64_t b, uint64_t& v) {
    if (a >= b) return false;
    uint64_t x = 0;
    for (uint64_t i = a; i < b; ++i) {
        const unsigned d = static_cast<unsigned char>(buf[i]) - '0';
        if (d > 9) return false;
        if (x > (~0ull - d) / 10) return false;  // overflow -> result_out_of_range
        x = x * 10 + d;
    }
    v = x;
    return true;
}

// Second pass, one thread per line: status + (u, v, w) of edge / arc lines.
// Edge list: header = line `first`, every later significant line an edge.
// DIMACS: arcs after the problem line (ids 1-based, checked against n).
__global__ void parse_lines(const char* __restrict__ buf, uint64_t len,
                            const uint64_t* __restrict__ nl, uint64_t nnl, uint64_t nlines,
                            int dimacs, const uint8_t* __restrict__ cls, uint64_t first,
                            uint64_t n, uint8_t* __restrict__ st, uint64_t* __restrict__ uu,
                            uint64_t* __restrict__ vv, double* __restrict__ ww) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nlines) return;
    const uint8_t c = cls[i];
    uint8_t s = LN_SKIP;
    if (i == first) {
        s = LN_HEADER;
    } else if (!dimacs && c == CL_SIG && i > first) {
        s = LN_EDGE;
    } else if (dimacs && i > first && (c == CL_P || c == CL_OTHER)) {
        s = LN_ERR;  // duplicate problem line / unrecognized line type
    } else if (dimacs && c == CL_A && i > first) {
        s = LN_EDGE;
    }
    if (s == LN_EDGE) {
        const LineSpan sp = line_body(buf, len, nl, nnl, i);
        uint64_t ta[5], tb[5];
        const int nt = split_tokens(buf, sp.a, sp.b, ta, tb);
        const int t0 = dimacs ? 1 : 0;
        uint64_t u = 0, v = 0;
        double w = 0;
        if (nt != 3 + t0 || !parse_u64(buf, ta[t0], tb[t0], u) ||
            !parse_u64(buf, ta[t0 + 1], tb[t0 + 1], v)) {
            s = LN_ERR;
        } else if (!parse_decimal(buf + ta[t0 + 2], tb[t0 + 2] - ta[t0 + 2], w)) {
            s = LN_HARD;  // exact value (or its error) from the host
        } else if (dimacs ? (u < 1 || u > n || v < 1 || v > n) : (u >= n || v >= n)) {
            s = LN_ERR;
        } else {
            uu[i] = u;
            vv[i] = v;
            ww[i] = w;
        }
    }
    st[i] = s;
}

// DIMACS normalisation keys: (min, max) 0-based, self-loop arcs dropped
__global__ void arc_keys(const uint8_t* __restrict__ st, const uint64_t* __restrict__ uu,
                         const uint64_t* __restrict__ vv, const double* __restrict__ ww,
                         const uint32_t* __restrict__ pos, uint64_t nlines,
                         uint64_t* __restrict__ key, double* __restrict__ w) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nlines || st[i] != LN_EDGE) return;
    uint64_t a = uu[i] - 1, b = vv[i] - 1;
    if (a == b) return;
    if (a > b) {
        const uint64_t t = a; a = b; b = t;
    }
    key[pos[i]] = (a << 32) | b;
    w[pos[i]] = ww[i];
}

__global__ void edge_compact(const uint8_t* __restrict__ st, const uint64_t* __restrict__ uu,
                             const uint64_t* __restrict__ vv, const double* __restrict__ ww,
                             const uint32_t* __restrict__ pos, uint64_t nlines,
                             uint32_t* __restrict__ eu, uint32_t* __restrict__ ev,
                             double* __restrict__ ew) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nlines || st[i] != LN_EDGE) return;
    eu[pos[i]] = static_cast<uint32_t>(uu[i]);
    ev[pos[i]] = static_cast<uint32_t>(vv[i]);
    ew[pos[i]] = ww[i];
}

// mode 0: edge / arc lines; 1: arcs without self-loops (DIMACS keys);
// 2: every line after the header that is not skipped (edge, error, hard)
__global__ void flag_to_u32(const uint8_t* __restrict__ st, uint64_t nlines, int mode,
                            uint32_t* __restrict__ f, const uint64_t* __restrict__ uu,
                            const uint64_t* __restrict__ vv) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= nlines) return;
    const uint8_t s = st[i];
    bool on;
    if (mode == 2) on = s == LN_EDGE || s == LN_ERR || s == LN_HARD;
    else if (mode == 3) on = s == LN_ERR || s == LN_HARD;
    else on = s == LN_EDGE && !(mode == 1 && uu[i] == vv[i]);
    f[i] = on ? 1u : 0u;
}

// compacted (line, body begin, body end) of the ERR / HARD lines < bound
__global__ void collect_lines(const char* __restrict__ buf, uint64_t len,
                              const uint64_t* __restrict__ nl, uint64_t nnl,
                              const uint8_t* __restrict__ st, const uint32_t* __restrict__ pos,
                              uint64_t bound, uint64_t* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= bound || (st[i] != LN_ERR && st[i] != LN_HARD)) return;
    const LineSpan sp = line_body(buf, len, nl, nnl, i);
    out[3 * uint64_t(pos[i]) + 0] = i;
    out[3 * uint64_t(pos[i]) + 1] = sp.a;
    out[3 * uint64_t(pos[i]) + 2] = sp.b;
}

// host-resolved HARD lines: (line, u, v, w bits) -> edge
__global__ void apply_lines(const uint64_t* __restrict__ rec, uint64_t count,
                            uint8_t* __restrict__ st, uint64_t* __restrict__ uu,
                            uint64_t* __restrict__ vv, double* __restrict__ ww) {
    const uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= count) return;
    const uint64_t i = rec[4 * j];
    uu[i] = rec[4 * j + 1];
    vv[i] = rec[4 * j + 2];
    ww[i] = __longlong_as_double(static_cast<long long>(rec[4 * j + 3]));
    st[i] = LN_EDGE;
}

// psp::Graph(n, edges) checks for a parsed edge list (src/graph.cpp:22-56):
// ids, weights are already valid, so the first self-loop in edge order,
// then the lexicographically smallest duplicated pair (the first the
// constructor's sorted-adjacency scan meets).
__global__ void edge_checks(const uint32_t* __restrict__ eu, const uint32_t* __restrict__ ev,
                            uint64_t m, uint64_t* __restrict__ key,
                            unsigned long long* __restrict__ first_loop) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= m) return;
    const uint32_t a = eu[e], b = ev[e];
    if (a == b) atomicMin(first_loop, (unsigned long long)e);
    key[e] = (uint64_t(min(a, b)) << 32) | max(a, b);
}

__global__ void first_duplicate(const uint64_t* __restrict__ key, uint64_t m,
                                unsigned long long* __restrict__ dup) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e + 1 < m && key[e] == key[e + 1]) atomicMin(dup, (unsigned long long)key[e]);
}

// ------------------------------------------------------------- host side --
// Host re-check of the header and of the lines the device declines
// (malformed, signed, non-finite or subnormal weights, > 19 significant
// digits). Verdicts, their order and the messages are the reference's
// psp::ParseError ones (src/graph_io.cpp:50-90 edge list, :93-140 DIMACS).
[[noreturn]] void parse_fail(const std::string& name, uint64_t line, const std::string& msg) {
    throw ParseFail{name + ":" + std::to_string(line) + ": " + msg, line};
}

// One line scanned in place: ' ', '\t' and '\r' stripped from both ends,
// fields = maximal runs of bytes other than ' ' and '\t' (a '\r' inside the
// line is part of a field). The count saturates at kMax, more than any
// valid line has, so "wrong field count" verdicts are unchanged.
struct LineFields {
    static constexpr int kMax = 5;
    std::string_view f[kMax];
    int n = 0;
    char lead = 0;  // first byte of the stripped line, 0 when it is empty
};

LineFields scan_fields(std::string_view line) {
    auto blank = [](char c) { return c == ' ' || c == '\t'; };
    size_t lo = 0, hi = line.size();
    while (lo < hi && (blank(line[lo]) || line[lo] == '\r')) ++lo;
    while (hi > lo && (blank(line[hi - 1]) || line[hi - 1] == '\r')) --hi;
    LineFields out;
    out.lead = lo < hi ? line[lo] : 0;
    size_t i = lo;
    while (i < hi && out.n < LineFields::kMax) {
        if (blank(line[i])) {
            ++i;
            continue;
        }
        const size_t start = i;
        while (i < hi && !blank(line[i])) ++i;
        out.f[out.n++] = line.substr(start, i - start);
    }
    return out;
}

// A field that must be one whole number of type T (std::from_chars, as the
// reference parses it): anything else is "expected <what>, got '<field>'".
template <typename T>
T field_value(std::string_view f, const char* what, const std::string& name, uint64_t line) {
    T v{};
    const char* end = f.data() + f.size();
    const std::from_chars_result r = std::from_chars(f.data(), end, v);
    if (r.ec != std::errc{} || r.ptr != end)
        parse_fail(name, line, std::string("expected ") + what + ", got '" + std::string(f) + "'");
    return v;
}

struct HostEdge {
    uint64_t u, v;
    double w;
};

// An edge line ('u v w', 0-based) or a DIMACS arc line ('a u v w', 1-based).
// Throws ParseFail; returns the parsed edge.
HostEdge host_edge_line(std::string_view line, bool dimacs, uint64_t n, const std::string& name,
                        uint64_t ln) {
    const LineFields lf = scan_fields(line);
    const int at = dimacs ? 1 : 0;  // arcs carry the leading 'a' field
    if (lf.n != 3 + at)
        parse_fail(name, ln, dimacs ? "arc line must be 'a u v w'" : "edge line must be 'u v w'");
    HostEdge e;
    e.u = field_value<uint64_t>(lf.f[at], "vertex id", name, ln);
    e.v = field_value<uint64_t>(lf.f[at + 1], "vertex id", name, ln);
    e.w = field_value<double>(lf.f[at + 2], "weight", name, ln);
    auto valid_id = [&](uint64_t x) { return dimacs ? (x >= 1 && x <= n) : x < n; };
    if (!valid_id(e.u) || !valid_id(e.v))
        parse_fail(name, ln, dimacs ? "vertex id out of range (ids are 1-based)" : "vertex id out of range");
    if (e.w < 0.0) parse_fail(name, ln, "negative weight");
    if (!std::isfinite(e.w)) parse_fail(name, ln, "non-finite weight");
    return e;
}

struct ParsedGraph {
    uint64_t n = 0;
    std::vector<uint32_t> eu, ev;
    std::vector<double> ew;
};

struct DevText {
    DBuf buf;            // the text in HBM
    const char* host = nullptr;  // the same bytes on the host
    uint64_t len = 0;
    char* pinned = nullptr;      // owned host copy (files)
    DevText() = default;
    DevText(const DevText&) = delete;
    DevText& operator=(const DevText&) = delete;
    ~DevText() {
        if (pinned) cudaFreeHost(pinned);
    }
};

// Reads a file into pinned host memory (parallel preads) and HBM.
void read_to_device(const std::string& path, cudaStream_t s, DevText& t) {
    const int fd = ::open(path.c_str(), O_RDONLY);
    if (fd < 0) throw Fail{PSP_EIO, "cannot open '" + path + "' for reading"};
    struct stat sb;
    if (fstat(fd, &sb) != 0 || !S_ISREG(sb.st_mode)) {
        ::close(fd);
        throw Fail{PSP_EIO, "cannot open '" + path + "' for reading"};
    }
    t.len = static_cast<uint64_t>(sb.st_size);
    t.buf.alloc(t.len + 1);
    if (cudaMallocHost(&t.pinned, t.len + 1) != cudaSuccess) {
        ::close(fd);
        throw Fail{PSP_ENOMEM, "pinned host buffer for '" + path + "'"};
    }
    t.host = t.pinned;
    const unsigned nt = std::max(1u, std::min(16u, unsigned(t.len >> 24) + 1));
    std::vector<std::thread> pool;
    std::atomic<bool> failed{false};
    for (unsigned k = 0; k < nt; ++k)
        pool.emplace_back([&, k] {
            uint64_t off = t.len * k / nt;
            const uint64_t end = t.len * (k + 1) / nt;
            while (off < end) {
                const ssize_t r = ::pread(fd, t.pinned + off, std::min<uint64_t>(end - off, 1ull << 30), off);
                if (r <= 0) {
                    failed = true;
                    return;
                }
                off += uint64_t(r);
            }
        });
    for (auto& th : pool) th.join();
    ::close(fd);
    if (failed) throw Fail{PSP_EIO, "read from '" + path + "' failed"};
    if (t.len) CK(cudaMemcpyAsync(t.buf.p, t.pinned, t.len, cudaMemcpyHostToDevice, s));
}

void text_to_device(const char* text, uint64_t len, cudaStream_t s, DevText& t) {
    t.len = len;
    t.host = text;
    t.buf.alloc(len + 1);
    if (len) CK(cudaMemcpyAsync(t.buf.p, text, len, cudaMemcpyHostToDevice, s));
}

std::string host_line(const DevText& t, const std::vector<uint64_t>& r) {
    return std::string(t.host + r[0], t.host + r[1]);  // r = {begin, end} of the line
}

ParsedGraph parse_graph_device(const DevText& t, bool dimacs, const std::string& name,
                               cudaStream_t s, int sms) {
    const char* buf = t.buf.as<char>();
    const uint64_t len = t.len;
    const uint64_t nchunks = (len + PARSE_CHUNK - 1) / PARSE_CHUNK;
    // L1: newline positions
    DBuf cnt((nchunks + 1) * 4), off((nchunks + 1) * 4);
    CK(cudaMemsetAsync(cnt.p, 0, (nchunks + 1) * 4, s));
    if (nchunks) {
        nl_count<<<unsigned((nchunks + 255) / 256), 256, 0, s>>>(buf, len, cnt.as<uint32_t>(), nchunks);
        CK_LAUNCH();
    }
    size_t tb = 0;
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt.as<uint32_t>(), off.as<uint32_t>(),
                                     int(nchunks + 1), s));
    DBuf tmp(tb);
    CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cnt.as<uint32_t>(), off.as<uint32_t>(),
                                     int(nchunks + 1), s));
    uint32_t nnl32 = 0;
    CK(cudaMemcpyAsync(&nnl32, off.as<uint32_t>() + nchunks, 4, cudaMemcpyDeviceToHost, s));
    char last = '\n';
    if (len) CK(cudaMemcpyAsync(&last, buf + len - 1, 1, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t nnl = nnl32;
    // getline: a final line without '\n' still counts
    const uint64_t nlines = nnl + (len > 0 && last != '\n' ? 1 : 0);
    DBuf nl(std::max<uint64_t>(nnl, 1) * 8);
    if (nchunks) {
        nl_write<<<unsigned((nchunks + 255) / 256), 256, 0, s>>>(buf, len, off.as<uint32_t>(), nchunks,
                                                                 nl.as<uint64_t>());
        CK_LAUNCH();
    }
    const uint64_t* d_nl = nl.as<uint64_t>();
    auto line_range = [&](uint64_t i) {
        std::vector<uint64_t> r(2);
        uint64_t prev = 0, cur = len;
        if (i > 0) CK(cudaMemcpyAsync(&prev, d_nl + i - 1, 8, cudaMemcpyDeviceToHost, s));
        if (i < nnl) CK(cudaMemcpyAsync(&cur, d_nl + i, 8, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        r[0] = i > 0 ? prev + 1 : 0;
        r[1] = cur;
        return r;
    };
    auto body_of = [&](uint64_t i) { return host_line(t, line_range(i)); };
    const unsigned lb = unsigned((std::max<uint64_t>(nlines, 1) + 255) / 256);
    const uint64_t lineno_end = nlines ? nlines : 1;  // "lineno ? lineno : 1"

    // L2a: classes and the first header line
    DBuf cls(std::max<uint64_t>(nlines, 1)), firsts(16);
    std::vector<unsigned long long> hf = {~0ull, ~0ull};
    CK(cudaMemcpyAsync(firsts.p, hf.data(), 16, cudaMemcpyHostToDevice, s));
    if (nlines) {
        classify_lines<<<lb, 256, 0, s>>>(buf, len, d_nl, nnl, nlines, dimacs ? 1 : 0,
                                          cls.as<uint8_t>(), firsts.as<unsigned long long>());
        CK_LAUNCH();
    }
    CK(cudaMemcpyAsync(hf.data(), firsts.p, 16, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t first = hf[0];
    // DIMACS lines before the problem line: 'a' or unknown -> error there
    if (dimacs && hf[1] != ~0ull && hf[1] < first) {
        const std::string line = body_of(hf[1]);
        const char lead = scan_fields(line).lead;
        if (lead == 'a') parse_fail(name, hf[1] + 1, "arc line before problem line");
        parse_fail(name, hf[1] + 1, "unrecognized line type '" + std::string(1, lead) + "'");
    }
    if (first == ~0ull)
        parse_fail(name, lineno_end, dimacs ? "missing 'p sp n m' line" : "missing 'n m' header");
    // the header (src/graph_io.cpp:58-66, :103-110)
    uint64_t n = 0, m = 0;
    {
        const std::string line = body_of(first);
        const LineFields hdr = scan_fields(line);
        const uint64_t ln = first + 1;
        const int at = dimacs ? 2 : 0;  // 'p sp n m' | 'n m'
        if (dimacs ? (hdr.n != 4 || hdr.f[1] != "sp") : hdr.n != 2)
            parse_fail(name, ln, dimacs ? "problem line must be 'p sp n m'" : "header must be 'n m'");
        n = field_value<size_t>(hdr.f[at], "vertex count", name, ln);
        m = field_value<size_t>(hdr.f[at + 1], dimacs ? "arc count" : "edge count", name, ln);
    }
    // L2b: every later line
    DBuf st(std::max<uint64_t>(nlines, 1)), uu(std::max<uint64_t>(nlines, 1) * 8),
        vv(std::max<uint64_t>(nlines, 1) * 8), ww(std::max<uint64_t>(nlines, 1) * 8);
    parse_lines<<<lb, 256, 0, s>>>(buf, len, d_nl, nnl, nlines, dimacs ? 1 : 0, cls.as<uint8_t>(),
                                   first, n, st.as<uint8_t>(), uu.as<uint64_t>(), vv.as<uint64_t>(),
                                   ww.as<double>());
    CK_LAUNCH();
    // positions of the edge / arc lines in file order
    DBuf flag(std::max<uint64_t>(nlines, 1) * 4 + 4), pos(std::max<uint64_t>(nlines, 1) * 4 + 4);
    auto positions = [&](int mode) -> uint64_t {
        CK(cudaMemsetAsync(flag.p, 0, flag.bytes, s));
        if (nlines) {
            flag_to_u32<<<lb, 256, 0, s>>>(st.as<uint8_t>(), nlines, mode, flag.as<uint32_t>(),
                                           uu.as<uint64_t>(), vv.as<uint64_t>());
            CK_LAUNCH();
        }
        size_t b2 = 0;
        CK(cub::DeviceScan::ExclusiveSum(nullptr, b2, flag.as<uint32_t>(), pos.as<uint32_t>(),
                                         int(nlines + 1), s));
        DBuf t2(b2);
        CK(cub::DeviceScan::ExclusiveSum(t2.p, b2, flag.as<uint32_t>(), pos.as<uint32_t>(),
                                         int(nlines + 1), s));
        uint32_t total = 0;
        CK(cudaMemcpyAsync(&total, pos.as<uint32_t>() + nlines, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        return total;
    };
    // Edge list: the (m+1)-th line after the header stops the reference with
    // "more edges than declared" (:80) unless it, or an earlier line, fails
    // first -- so errors are only searched up to and including that line.
    uint64_t cut = nlines;  // search bound (exclusive)
    bool more = false;
    if (!dimacs) {
        const uint64_t nsig = positions(2);
        if (nsig > m) {
            more = true;
            std::vector<uint32_t> hpos(nlines + 1);
            CK(cudaMemcpyAsync(hpos.data(), pos.p, (nlines + 1) * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            cut = std::upper_bound(hpos.begin(), hpos.end(), uint32_t(m)) - hpos.begin();
        }
    }
    // resolve the HARD / ERR lines before the bound in file order, in one
    // batch: the first real error throws the reference's ParseError; the
    // HARD lines that parse are written back as edges
    {
        const uint64_t nflag = positions(3);
        uint64_t nres = 0;
        if (nflag) {
            DBuf recs(nflag * 24);
            collect_lines<<<lb, 256, 0, s>>>(buf, len, d_nl, nnl, st.as<uint8_t>(), pos.as<uint32_t>(),
                                             cut, recs.as<uint64_t>());
            CK_LAUNCH();
            uint32_t nb = 0;  // flagged lines below the bound
            CK(cudaMemcpyAsync(&nb, pos.as<uint32_t>() + cut, 4, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<uint64_t> h(uint64_t(nb) * 3);
            if (nb) CK(cudaMemcpyAsync(h.data(), recs.p, h.size() * 8, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            std::vector<uint64_t> ok;
            ok.reserve(uint64_t(nb) * 4);
            for (uint64_t j = 0; j < nb; ++j) {
                const uint64_t f = h[3 * j], ln = f + 1;
                const std::string_view body(t.host + h[3 * j + 1], h[3 * j + 2] - h[3 * j + 1]);
                const char lead = scan_fields(body).lead;
                if (dimacs && lead == 'p') parse_fail(name, ln, "duplicate problem line");
                if (dimacs && lead != 'a')
                    parse_fail(name, ln, "unrecognized line type '" + std::string(1, lead) + "'");
                const HostEdge e = host_edge_line(body, dimacs, n, name, ln);  // ERR lines throw
                uint64_t wb;
                std::memcpy(&wb, &e.w, 8);
                ok.insert(ok.end(), {f, e.u, e.v, wb});
            }
            nres = ok.size() / 4;
            if (nres) {
                DBuf d(ok.size() * 8);
                CK(cudaMemcpyAsync(d.p, ok.data(), ok.size() * 8, cudaMemcpyHostToDevice, s));
                apply_lines<<<unsigned((nres + 255) / 256), 256, 0, s>>>(
                    d.as<uint64_t>(), nres, st.as<uint8_t>(), uu.as<uint64_t>(), vv.as<uint64_t>(),
                    ww.as<double>());
                CK_LAUNCH();
                CK(cudaStreamSynchronize(s));
            }
        }
    }
    if (more) parse_fail(name, cut, "more edges than declared in header");
    const uint64_t nedge_lines = positions(0);
    ParsedGraph G;
    G.n = n;
    if (!dimacs) {
        if (nedge_lines != m)
            parse_fail(name, lineno_end,
                       "declared " + std::to_string(m) + " edges, found " + std::to_string(nedge_lines));
        G.eu.resize(m);
        G.ev.resize(m);
        G.ew.resize(m);
        DBuf du(m * 4 + 4), dv(m * 4 + 4), dw(m * 8 + 8);
        if (nlines) {
            edge_compact<<<lb, 256, 0, s>>>(st.as<uint8_t>(), uu.as<uint64_t>(), vv.as<uint64_t>(),
                                            ww.as<double>(), pos.as<uint32_t>(), nlines,
                                            du.as<uint32_t>(), dv.as<uint32_t>(), dw.as<double>());
            CK_LAUNCH();
        }
        if (m) {
            CK(cudaMemcpyAsync(G.eu.data(), du.p, m * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(G.ev.data(), dv.p, m * 4, cudaMemcpyDeviceToHost, s));
            CK(cudaMemcpyAsync(G.ew.data(), dw.p, m * 8, cudaMemcpyDeviceToHost, s));
            // the Graph constructor's remaining checks, on the device
            DBuf keys(m * 8), sorted(m * 8), flags(16);
            std::vector<unsigned long long> hf = {~0ull, ~0ull};
            CK(cudaMemcpyAsync(flags.p, hf.data(), 16, cudaMemcpyHostToDevice, s));
            const unsigned eb = unsigned((m + 255) / 256);
            edge_checks<<<eb, 256, 0, s>>>(du.as<uint32_t>(), dv.as<uint32_t>(), m, keys.as<uint64_t>(),
                                           flags.as<unsigned long long>());
            CK_LAUNCH();
            size_t b5 = 0;
            CK(cub::DeviceRadixSort::SortKeys(nullptr, b5, keys.as<uint64_t>(), sorted.as<uint64_t>(),
                                              int(m), 0, 64, s));
            DBuf t5(b5);
            CK(cub::DeviceRadixSort::SortKeys(t5.p, b5, keys.as<uint64_t>(), sorted.as<uint64_t>(),
                                              int(m), 0, 64, s));
            first_duplicate<<<eb, 256, 0, s>>>(sorted.as<uint64_t>(), m,
                                               flags.as<unsigned long long>() + 1);
            CK_LAUNCH();
            CK(cudaMemcpyAsync(hf.data(), flags.p, 16, cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (hf[0] != ~0ull)
                throw GraphError("self-loop at vertex " + std::to_string(G.eu[hf[0]]));
            if (hf[1] != ~0ull)
                throw GraphError("duplicate edge (" + std::to_string(hf[1] >> 32) + "," +
                                 std::to_string(hf[1] & 0xffffffffu) + ")");
        }
        CK(cudaStreamSynchronize(s));
        return G;
    }
    // DIMACS: arcs_seen counts self-loop arcs too (src/graph_io.cpp:123-124)
    if (nedge_lines != m)
        parse_fail(name, lineno_end,
                   "declared " + std::to_string(m) + " arcs, found " + std::to_string(nedge_lines));
    const uint64_t na = positions(1);  // keyed arcs: self-loops dropped
    DBuf k1(na * 8 + 8), k2(na * 8 + 8), w1(na * 8 + 8), w2(na * 8 + 8), uk(na * 8 + 8),
        uw(na * 8 + 8), nrun(8);
    if (nlines) {
        arc_keys<<<lb, 256, 0, s>>>(st.as<uint8_t>(), uu.as<uint64_t>(), vv.as<uint64_t>(),
                                    ww.as<double>(), pos.as<uint32_t>(), nlines, k1.as<uint64_t>(),
                                    w1.as<double>());
        CK_LAUNCH();
    }
    uint64_t runs = 0;
    if (na) {
        size_t b3 = 0;
        CK(cub::DeviceRadixSort::SortPairs(nullptr, b3, k1.as<uint64_t>(), k2.as<uint64_t>(),
                                           w1.as<double>(), w2.as<double>(), int(na), 0, 64, s));
        DBuf t3(b3);
        CK(cub::DeviceRadixSort::SortPairs(t3.p, b3, k1.as<uint64_t>(), k2.as<uint64_t>(),
                                           w1.as<double>(), w2.as<double>(), int(na), 0, 64, s));
        size_t b4 = 0;
        CK(cub::DeviceReduce::ReduceByKey(nullptr, b4, k2.as<uint64_t>(), uk.as<uint64_t>(),
                                          w2.as<double>(), uw.as<double>(), nrun.as<int>(),
                                          KeepFirstMin{}, int(na), s));
        DBuf t4(b4);
        CK(cub::DeviceReduce::ReduceByKey(t4.p, b4, k2.as<uint64_t>(), uk.as<uint64_t>(),
                                          w2.as<double>(), uw.as<double>(), nrun.as<int>(),
                                          KeepFirstMin{}, int(na), s));
        int r = 0;
        CK(cudaMemcpyAsync(&r, nrun.p, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        runs = uint64_t(r);
    }
    std::vector<uint64_t> keys(runs);
    G.ew.resize(runs);
    if (runs) {
        CK(cudaMemcpyAsync(keys.data(), uk.p, runs * 8, cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(G.ew.data(), uw.p, runs * 8, cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    G.eu.resize(runs);
    G.ev.resize(runs);
    for (uint64_t i = 0; i < runs; ++i) {
        G.eu[i] = static_cast<uint32_t>(keys[i] >> 32);
        G.ev[i] = static_cast<uint32_t>(keys[i] & 0xffffffffu);
    }
    (void)sms;
    return G;
}

// ------------------------------------------------------------- writer --
// format_weight (src/graph_io.cpp:147-151): shortest round-trip decimal.
uint32_t format_weight_into(double w, char* buf) {
    auto r = std::to_chars(buf, buf + 32, w);
    return static_cast<uint32_t>(r.ptr - buf);
}

// write_graph (src/graph_io.cpp:160-176) of the CSR's edge list (u < v,
// lexicographic, Graph::edge_list), formatted on all host threads.
std::string write_graph_text(const Csr& g, bool dimacs, unsigned threads) {
    std::vector<uint64_t> ecount(g.n + 1, 0);  // edges with u < v per vertex, prefix
    for (uint64_t u = 0; u < g.n; ++u) {
        uint64_t c = 0;
        for (uint64_t e = g.off[u]; e < g.off[u + 1]; ++e) c += g.to[e] > u;
        ecount[u + 1] = ecount[u] + c;
    }
    const uint64_t m = ecount[g.n];
    std::string head = dimacs ? "p sp " + std::to_string(g.n) + " " + std::to_string(2 * m) + "\n"
                              : std::to_string(g.n) + " " + std::to_string(m) + "\n";
    threads = std::max(1u, std::min<unsigned>(threads, unsigned(std::max<uint64_t>(1, g.n / 4096))));
    std::vector<std::string> part(threads);
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            const uint64_t u0 = g.n * t / threads, u1 = g.n * (t + 1) / threads;
            std::string& out = part[t];
            out.reserve((ecount[u1] - ecount[u0]) * (dimacs ? 48 : 24));
            char wb[32], ib[24];
            for (uint64_t u = u0; u < u1; ++u)
                for (uint64_t e = g.off[u]; e < g.off[u + 1]; ++e) {
                    const uint64_t v = g.to[e];
                    if (v <= u) continue;
                    const uint32_t wl = format_weight_into(g.w[e], wb);
                    auto put = [&](uint64_t x) {
                        auto r = std::to_chars(ib, ib + sizeof ib, x);
                        out.append(ib, r.ptr);
                    };
                    if (!dimacs) {
                        put(u); out.push_back(' '); put(v); out.push_back(' ');
                        out.append(wb, wl); out.push_back('\n');
                    } else {  // both arc directions, 1-based
                        out.append("a "); put(u + 1); out.push_back(' '); put(v + 1); out.push_back(' ');
                        out.append(wb, wl); out.push_back('\n');
                        out.append("a "); put(v + 1); out.push_back(' '); put(u + 1); out.push_back(' ');
                        out.append(wb, wl); out.push_back('\n');
                    }
                }
        });
    for (auto& th : pool) th.join();
    size_t total = head.size();
    for (auto& p : part) total += p.size();
    std::string out;
    out.reserve(total);
    out += head;
    for (auto& p : part) out += p;
    return out;
}

}  // namespace
