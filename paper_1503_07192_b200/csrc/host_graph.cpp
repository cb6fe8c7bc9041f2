// host_graph.cpp — CSR build, boundary flags, boundary-first reordering and
// the synthetic grid generators. See host_graph.hpp for the reference
// interfaces each routine reproduces.
#include "host_graph.hpp"

#include <algorithm>
#include <atomic>
#include <cstring>
#include <cmath>
#include <limits>
#include <numeric>
#include <random>
#include <thread>

namespace pspg {

namespace {
std::string pair_str(uint32_t u, uint32_t v) {
    return "(" + std::to_string(u) + "," + std::to_string(v) + ")";
}

// fn(lo, hi) over [0, n) in contiguous slices on up to 16 host threads
// (serial below 64K items, where thread start-up would dominate)
template <class F>
void par_slices(uint64_t n, F&& fn) {
    const unsigned hw = std::max(1u, std::min(16u, std::thread::hardware_concurrency()));
    const uint64_t t = n < (uint64_t(1) << 16) ? 1 : std::min<uint64_t>(hw, n);
    if (t <= 1) {
        fn(uint64_t(0), n);
        return;
    }
    std::vector<std::thread> pool;
    for (uint64_t i = 1; i < t; ++i) pool.emplace_back([&, i] { fn(n * i / t, n * (i + 1) / t); });
    fn(uint64_t(0), n / t);
    for (auto& th : pool) th.join();
}
}  // namespace

Csr build_csr(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev, const double* ew) {
    Csr g;
    g.n = n;
    g.off.assign(n + 1, 0);
    // validation order of src/graph.cpp:22-36: range, self-loop, NaN/inf,
    // negative; the first offending edge is found in parallel, then reported
    // exactly as a serial scan would
    auto bad = [&](uint64_t e) {
        const uint32_t u = eu[e], v = ev[e];
        const double w = ew[e];
        return u >= n || v >= n || u == v || std::isnan(w) || std::isinf(w) || w < 0.0;
    };
    std::atomic<uint64_t> first_bad{m};
    par_slices(m, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e)
            if (bad(e)) {
                uint64_t cur = first_bad.load();
                while (e < cur && !first_bad.compare_exchange_weak(cur, e)) {}
                return;
            }
    });
    if (first_bad.load() < m) {
        const uint64_t e = first_bad.load();
        const uint32_t u = eu[e], v = ev[e];
        const double w = ew[e];
        if (u >= n || v >= n)
            throw GraphError("edge " + pair_str(u, v) + " references vertex outside 0.." +
                             std::to_string(n ? n - 1 : 0));
        if (u == v) throw GraphError("self-loop at vertex " + std::to_string(u));
        if (std::isnan(w) || std::isinf(w))
            throw GraphError("non-finite weight on edge " + pair_str(u, v));
        throw GraphError("negative weight on edge " + pair_str(u, v));
    }
    // degree count and scatter with relaxed atomics: the slot order inside a
    // neighbour list is arbitrary, but the sort below makes the result unique
    // (equal keys are duplicates, which are rejected)
    par_slices(m, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e) {
            std::atomic_ref<uint64_t>(g.off[eu[e] + 1]).fetch_add(1, std::memory_order_relaxed);
            std::atomic_ref<uint64_t>(g.off[ev[e] + 1]).fetch_add(1, std::memory_order_relaxed);
        }
    });
    for (uint64_t v = 0; v < n; ++v) g.off[v + 1] += g.off[v];
    g.to.resize(2 * m);
    g.w.resize(2 * m);
    std::vector<uint64_t> cur(g.off.begin(), g.off.end() - 1);
    par_slices(m, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t e = lo; e < hi; ++e) {
            const uint64_t a = std::atomic_ref<uint64_t>(cur[eu[e]]).fetch_add(1, std::memory_order_relaxed);
            const uint64_t b = std::atomic_ref<uint64_t>(cur[ev[e]]).fetch_add(1, std::memory_order_relaxed);
            g.to[a] = ev[e];
            g.w[a] = ew[e];
            g.to[b] = eu[e];
            g.w[b] = ew[e];
        }
    });
    // per-vertex neighbour sort; the lowest vertex holding a duplicate is the
    // one a serial scan reports
    std::atomic<uint64_t> dup_v{n};
    par_slices(n, [&](uint64_t vlo, uint64_t vhi) {
        std::vector<std::pair<uint32_t, double>> tmp;
        for (uint64_t v = vlo; v < vhi; ++v) {
            const uint64_t lo = g.off[v], hi = g.off[v + 1];
            tmp.clear();
            for (uint64_t e = lo; e < hi; ++e) tmp.emplace_back(g.to[e], g.w[e]);
            std::sort(tmp.begin(), tmp.end(),
                      [](const auto& a, const auto& b) { return a.first < b.first; });
            bool dup = false;
            for (uint64_t e = lo; e < hi; ++e) {
                g.to[e] = tmp[e - lo].first;
                g.w[e] = tmp[e - lo].second;
                dup |= e > lo && g.to[e] == g.to[e - 1];
            }
            if (dup) {
                uint64_t cur = dup_v.load();
                while (v < cur && !dup_v.compare_exchange_weak(cur, v)) {}
                return;
            }
        }
    });
    if (dup_v.load() < n) {
        const uint64_t v = dup_v.load();
        for (uint64_t e = g.off[v] + 1; e < g.off[v + 1]; ++e)
            if (g.to[e] == g.to[e - 1])
                throw GraphError("duplicate edge " + pair_str(static_cast<uint32_t>(v), g.to[e]));
    }
    return g;
}

std::vector<uint8_t> compute_boundary(const Csr& g, const std::vector<uint32_t>& a) {
    std::vector<uint8_t> flags(g.n, 0);
    par_slices(g.n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t v = lo; v < hi; ++v)
            for (uint64_t e = g.off[v]; e < g.off[v + 1]; ++e)
                if (a[g.to[e]] != a[v]) {
                    flags[v] = 1;
                    break;
                }
    });
    return flags;
}

std::vector<uint32_t> reorder_permutation(uint32_t k, const std::vector<uint32_t>& a,
                                          const std::vector<uint8_t>& flags) {
    const uint64_t n = a.size();
    std::vector<uint64_t> bsize(k, 0), tsize(k, 0);
    for (uint64_t v = 0; v < n; ++v) {
        ++tsize[a[v]];
        if (flags[v]) ++bsize[a[v]];
    }
    std::vector<uint64_t> bcur(k), icur(k);
    uint64_t start = 0;
    for (uint32_t c = 0; c < k; ++c) {
        bcur[c] = start;
        icur[c] = start + bsize[c];
        start += tsize[c];
    }
    std::vector<uint32_t> perm(n);
    for (uint64_t v = 0; v < n; ++v)
        perm[v] = static_cast<uint32_t>(flags[v] ? bcur[a[v]]++ : icur[a[v]]++);
    return perm;
}

Reordered reorder(const Csr& g, uint32_t k, const std::vector<uint32_t>& assignment) {
    const uint64_t n = g.n;
    if (assignment.size() != n) throw ArgError("reorder: assignment must cover all vertices");
    for (uint64_t v = 0; v < n; ++v)
        if (assignment[v] >= k) throw ArgError("reorder: component id out of range");
    Reordered r;
    r.n = n;
    r.k = k;
    const std::vector<uint8_t> flags0 = compute_boundary(g, assignment);
    r.perm = reorder_permutation(k, assignment, flags0);
    r.inv.resize(n);
    r.assign.resize(n);
    r.flags.resize(n);
    Csr& rg = r.g;
    rg.n = n;
    rg.off.assign(n + 1, 0);
    // perm is a bijection, so the scatters below write disjoint slots
    par_slices(n, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t v = lo; v < hi; ++v) {
            const uint32_t p = r.perm[v];
            r.inv[p] = static_cast<uint32_t>(v);
            r.assign[p] = assignment[v];
            r.flags[p] = flags0[v];
            rg.off[p + 1] = g.degree(static_cast<uint32_t>(v));
        }
    });
    // relabelled CSR, neighbour lists re-sorted by new id (:458-470)
    for (uint64_t v = 0; v < n; ++v) rg.off[v + 1] += rg.off[v];
    rg.to.resize(g.to.size());
    rg.w.resize(g.w.size());
    par_slices(n, [&](uint64_t lo, uint64_t hi) {
        std::vector<std::pair<uint32_t, double>> tmp;
        for (uint64_t v = lo; v < hi; ++v) {
            tmp.clear();
            for (uint64_t e = g.off[v]; e < g.off[v + 1]; ++e) tmp.emplace_back(r.perm[g.to[e]], g.w[e]);
            std::sort(tmp.begin(), tmp.end(),
                      [](const auto& a, const auto& b) { return a.first < b.first; });
            uint64_t at = rg.off[r.perm[v]];
            for (const auto& t : tmp) {
                rg.to[at] = t.first;
                rg.w[at++] = t.second;
            }
        }
    });
    r.comp_off.assign(k + 1, 0);
    r.bnd_off.assign(k + 1, 0);
    for (uint64_t v = 0; v < n; ++v) {
        ++r.comp_off[r.assign[v] + 1];
        if (r.flags[v]) ++r.bnd_off[r.assign[v] + 1];
    }
    for (uint32_t c = 0; c < k; ++c) {
        r.comp_off[c + 1] += r.comp_off[c];
        r.bnd_off[c + 1] += r.bnd_off[c];
    }
    return r;
}

void generate_grid(int kind, uint64_t rows, uint64_t cols, bool unit, double lo, double hi,
                   uint64_t seed, std::vector<uint32_t>& eu, std::vector<uint32_t>& ev,
                   std::vector<double>& ew) {
    // checked_vertex_count (src/generators.cpp:28-35), WeightModel::uniform (:39-47)
    if (rows == 0 || cols == 0) throw ArgError("grid dimensions must be positive");
    if (cols > std::numeric_limits<uint64_t>::max() / rows ||
        rows * cols > std::numeric_limits<uint32_t>::max())
        throw ArgError("rows*cols exceeds the supported vertex-count range");
    if (!unit && (lo < 0.0 || hi < lo || std::isnan(lo) || std::isnan(hi) || std::isinf(hi)))
        throw ArgError("uniform weight bounds must satisfy 0 <= lo <= hi < inf");
    std::mt19937_64 rng(seed);
    // WeightDrawer (:14-26): 1025 lattice points including both endpoints
    auto draw = [&]() -> double {
        if (unit) return 1.0;
        const double step = static_cast<double>(rng() % 1025u);
        return lo + (hi - lo) * (step / 1024.0);
    };
    eu.clear();
    ev.clear();
    ew.clear();
    auto push = [&](uint64_t a, uint64_t b, double w) {
        eu.push_back(static_cast<uint32_t>(a));
        ev.push_back(static_cast<uint32_t>(b));
        ew.push_back(w);
    };
    for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t c = 0; c < cols; ++c) {
            const uint64_t v = r * cols + c;
            // argument evaluation order matters for the rng stream: the
            // reference draws the weight inside push_back({v, v+1, draw()})
            if (c + 1 < cols) push(v, v + 1, draw());
            if (r + 1 < rows) push(v, v + cols, draw());
            if (kind == 1 && c + 1 < cols && r + 1 < rows) {
                const bool down_right = (rng() & 1u) != 0;
                if (down_right) push(v, v + cols + 1, draw());
                else push(v + 1, v + cols, draw());
            }
        }
}

void min_spanning_forest(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                         const double* key, uint8_t* in_tree) {
    // stable LSD radix sort of the edge ids by key: non-negative doubles
    // order like their bit patterns (negative keys: sorted by value below)
    std::vector<uint64_t> bits(m);
    bool nonneg = true;
    for (uint64_t e = 0; e < m; ++e) {
        if (!(key[e] >= 0.0)) nonneg = false;
        std::memcpy(&bits[e], &key[e], 8);
    }
    std::vector<uint32_t> order(m), tmp(m);
    std::iota(order.begin(), order.end(), 0u);
    if (nonneg) {
        uint64_t diff = 0;  // only the bit positions that vary need passes
        for (uint64_t e = 1; e < m; ++e) diff |= bits[e] ^ bits[0];
        for (int shift = 0; shift < 64 && (diff >> shift); shift += 16) {
            std::vector<uint64_t> cnt(65537, 0);
            for (uint64_t e = 0; e < m; ++e) ++cnt[((bits[order[e]] >> shift) & 0xffff) + 1];
            for (int d = 0; d < 65536; ++d) cnt[d + 1] += cnt[d];
            for (uint64_t e = 0; e < m; ++e) tmp[cnt[(bits[order[e]] >> shift) & 0xffff]++] = order[e];
            order.swap(tmp);
        }
    } else {
        std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return key[a] < key[b]; });
    }
    std::vector<uint32_t> parent(n), size(n, 1);
    std::iota(parent.begin(), parent.end(), 0u);
    auto find = [&](uint32_t x) {
        while (parent[x] != x) {
            parent[x] = parent[parent[x]];
            x = parent[x];
        }
        return x;
    };
    std::fill(in_tree, in_tree + m, uint8_t(0));
    for (uint32_t e : order) {
        uint32_t a = find(eu[e]), b = find(ev[e]);
        if (a == b) continue;
        if (size[a] < size[b]) std::swap(a, b);
        parent[b] = a;
        size[a] += size[b];
        in_tree[e] = 1;
    }
}

}  // namespace pspg
