// k1_order.hpp — elimination order of the per-component FW (K1).
//
// The component table of src/oracle.cpp:162-169 (apsp_dense on the induced
// subgraph, src/shortest_paths.cpp:107-172) does not depend on the pivot
// order, but the work of the sparse walk does (see bg_order.hpp for the
// boundary graph): when pivot block p is processed only the rows with a
// path to p through already processed pivots are finite, and phase 3 walks
// only active x active tiles. The reference numbering inside a component is
// boundary-first (src/partition.cpp:452-481), which makes almost every row
// finite after the first k-block. A nested-dissection order keeps the reach
// of a k-block to its own region plus the separators around it: leaves of
// <= LEAF vertices first, each separator after the two halves it splits.
// On a 90 x 91 grid (nb = 64) this is ~6.2k tile products instead of 133k
// for the dense walk (tools/k1_order_sim.py).
//
// Bisection: BFS levels from a pseudo-peripheral vertex (two sweeps) and the
// median level as the vertex separator; each side holds at most half of the
// part, so the recursion depth is <= log2 n. Disconnected parts are ordered
// one after the other.
#pragma once
#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

namespace pspg {

class NdOrder {
public:
    static constexpr uint32_t LEAF = 64;

    // n local vertices, undirected edges (u, v), u != v. Returns pos[v] =
    // elimination position of v (a permutation of 0..n-1).
    std::vector<uint32_t> positions(uint32_t n, const std::vector<std::pair<uint32_t, uint32_t>>& edges) {
        n_ = n;
        off_.assign(n + 1, 0);
        for (auto& e : edges) {
            ++off_[e.first + 1];
            ++off_[e.second + 1];
        }
        for (uint32_t v = 0; v < n; ++v) off_[v + 1] += off_[v];
        to_.resize(off_[n]);
        std::vector<uint32_t> fill(off_.begin(), off_.end() - 1);
        for (auto& e : edges) {
            to_[fill[e.first]++] = e.second;
            to_[fill[e.second]++] = e.first;
        }
        set_.assign(n, 0);
        seen_.assign(n, 0);
        lev_.assign(n, 0);
        stamp_ = 0;
        next_set_ = 2;
        order_.clear();
        order_.reserve(n);
        std::vector<uint32_t> all(n);
        for (uint32_t v = 0; v < n; ++v) all[v] = v;
        dissect(all, 1);
        std::vector<uint32_t> pos(n);
        for (uint32_t i = 0; i < n; ++i) pos[order_[i]] = i;
        return pos;
    }

private:
    uint32_t n_ = 0;
    std::vector<uint32_t> off_, to_, set_, seen_, lev_, order_;
    uint32_t stamp_ = 0, next_set_ = 2;

    // BFS inside the vertices whose set_ == sid from src; fills `out` in
    // BFS order and lev_ with levels
    void bfs(uint32_t src, uint32_t sid, std::vector<uint32_t>& out) {
        ++stamp_;
        out.clear();
        out.push_back(src);
        seen_[src] = stamp_;
        lev_[src] = 0;
        for (size_t h = 0; h < out.size(); ++h) {
            const uint32_t u = out[h];
            for (uint32_t e = off_[u]; e < off_[u + 1]; ++e) {
                const uint32_t w = to_[e];
                if (set_[w] == sid && seen_[w] != stamp_) {
                    seen_[w] = stamp_;
                    lev_[w] = lev_[u] + 1;
                    out.push_back(w);
                }
            }
        }
    }

    // order the vertices of S (all carry set_ == sid) and append them
    void dissect(std::vector<uint32_t>& S, uint32_t sid) {
        for (uint32_t v : S) set_[v] = sid;
        std::vector<uint32_t> part, tmp;
        // connected parts of S, one after the other
        std::vector<uint32_t> members = S;
        for (uint32_t s0 : members) {
            if (set_[s0] != sid) continue;  // already handled in an earlier part
            bfs(s0, sid, part);
            const uint32_t mine = fresh();
            for (uint32_t v : part) set_[v] = mine;
            if (part.size() <= LEAF) {
                order_.insert(order_.end(), part.begin(), part.end());
                continue;
            }
            // pseudo-peripheral vertex, then levels from it
            bfs(part.back(), mine, tmp);
            bfs(tmp.back(), mine, part);
            const uint32_t L = lev_[part.back()];
            std::vector<uint32_t> cnt(L + 2, 0);
            for (uint32_t v : part) ++cnt[lev_[v]];
            uint64_t cum = 0;
            uint32_t m = 0;
            for (; m <= L; ++m) {
                cum += cnt[m];
                if (2 * cum >= part.size()) break;
            }
            std::vector<uint32_t> A, B, sep;
            for (uint32_t v : part) {
                if (lev_[v] < m) A.push_back(v);
                else if (lev_[v] > m) B.push_back(v);
                else sep.push_back(v);
            }
            if (!A.empty()) dissect(A, fresh());
            if (!B.empty()) dissect(B, fresh());
            for (uint32_t v : sep) set_[v] = 0;
            order_.insert(order_.end(), sep.begin(), sep.end());
        }
    }
    uint32_t fresh() { return next_set_++; }
};

}  // namespace pspg
