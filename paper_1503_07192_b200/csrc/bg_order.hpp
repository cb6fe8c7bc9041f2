// bg_order.hpp — elimination order of the boundary-graph FW.
//
// The FW result does not depend on the pivot order, but its work does once
// phase 3 skips tiles whose panel slot is all INF (fw_active_list): when
// pivot block p is processed, exactly the rows i with a path i -> p through
// already-processed pivots are finite in the panel, and the update costs
// |B(p)| * (sum of B over those rows)^2 / 2 relaxations. The reference
// numbers components by the partitioner (src/partition.cpp), which after
// ~30% of the pivots makes every row finite (cfg2: 71% of the dense work).
// A greedy minimum-reach order, the minimum-degree heuristic of sparse
// elimination, keeps the reach small far longer. Its unit is a PIECE: the
// boundary vertices of one connected part of a component. A component's
// boundary clique (src/oracle.cpp:110-122) only joins vertices at finite
// distance, and the partitioner leaves small fragments of a component
// inside its neighbours (cfg2: 979 pieces in 256 components), so whole
// components as units would tie unrelated regions together (component
// graph degree ~15, piece graph ~5.4). Simulated work on cfg2: 2.4e12
// relaxations for pieces, 8.5e12 for components, 1.5e13 for the reference
// numbering, 2.1e13 dense.
//
// Tile packing (bg_pack): the device walks T-wide tiles, and a unit cut by a
// tile boundary makes both tiles active for its whole reach. Units are laid
// out in the greedy order, except that a unit which would straddle a tile
// boundary is swapped for the first of the next LOOK units that fits the
// room left, and the rest of the tile is padding when none does (isolated
// positions: INF rows, zero diagonal). The tile-level simulation
// (tools/k2_layout_sim.cpp) predicts cfg3 1.17e14 -> 9.3e13 relaxations (nb
// 1055 -> 1120); measured (PSP_K2_TRACE per k-block active slots), the
// simulation tracks the device early on but underestimates the late reach,
// and the walked work drops only 3% (K2 8.29 -> 8.05 s). Used from 128
// tiles per side.
//
// The order only relabels where each boundary vertex sits in the device
// matrix during K2; the finished table is permuted back to the reference's
// boundary ids (permute_sym) before anything reads it.
#pragma once
#include <algorithm>
#include <cstdint>
#include <utility>
#include <vector>

namespace pspg {

struct BgOrder {
    std::vector<uint32_t> order;    // units in elimination order
    double work = 0.0, natural = 0.0;  // simulated relaxations (order / identity)
};

// bsize[u] = boundary vertices of unit u; adj = unit pairs joined by a
// cross edge.
inline BgOrder bg_unit_order(uint32_t k, const std::vector<uint64_t>& bsize,
                                  const std::vector<std::pair<uint32_t, uint32_t>>& adj) {
    BgOrder out;
    const uint32_t W = (k + 63) / 64;
    auto simulate = [&](const std::vector<uint32_t>* fixed, std::vector<uint32_t>* picked) {
        std::vector<uint64_t> F(uint64_t(k) * W, 0);
        auto set = [&](uint32_t i, uint32_t j) { F[uint64_t(i) * W + j / 64] |= 1ull << (j % 64); };
        for (uint32_t c = 0; c < k; ++c) set(c, c);
        for (auto& e : adj) {
            set(e.first, e.second);
            set(e.second, e.first);
        }
        // reach weight of every row: sum of |B| over its set bits
        std::vector<double> w(k, 0.0);
        for (uint32_t i = 0; i < k; ++i)
            for (uint32_t x = 0; x < W; ++x)
                for (uint64_t bits = F[uint64_t(i) * W + x]; bits; bits &= bits - 1)
                    w[i] += double(bsize[x * 64 + __builtin_ctzll(bits)]);
        std::vector<char> done(k, 0);
        std::vector<uint64_t> Rrow(W);
        std::vector<uint32_t> members;
        double work = 0.0;
        for (uint32_t step = 0; step < k; ++step) {
            uint32_t p;
            if (fixed) {
                p = (*fixed)[step];
            } else {
                p = k;
                for (uint32_t c = 0; c < k; ++c)
                    if (!done[c] && (p == k || w[c] < w[p])) p = c;
                picked->push_back(p);
            }
            work += double(bsize[p]) * w[p] * w[p] * 0.5;
            std::copy(F.begin() + uint64_t(p) * W, F.begin() + uint64_t(p + 1) * W, Rrow.begin());
            members.clear();
            for (uint32_t x = 0; x < W; ++x)
                for (uint64_t bits = Rrow[x]; bits; bits &= bits - 1)
                    members.push_back(x * 64 + __builtin_ctzll(bits));
            done[p] = 1;
            // the reach set becomes a clique; only rows still to be pivoted
            // are read again
            for (uint32_t i : members) {
                if (done[i]) continue;
                uint64_t* row = &F[uint64_t(i) * W];
                for (uint32_t x = 0; x < W; ++x) {
                    for (uint64_t add = Rrow[x] & ~row[x]; add; add &= add - 1)
                        w[i] += double(bsize[x * 64 + __builtin_ctzll(add)]);
                    row[x] |= Rrow[x];
                }
            }
        }
        return work;
    };
    std::vector<uint32_t> ident(k);
    for (uint32_t c = 0; c < k; ++c) ident[c] = c;
    out.natural = simulate(&ident, nullptr);
    out.work = simulate(nullptr, &out.order);
    if (!(out.work < out.natural)) {
        out.order = ident;
        out.work = out.natural;
    }
    return out;
}

// start position of every unit (and the padded position count) for the
// greedy order `order` packed into tiles of `tile` positions
inline uint64_t bg_pack(const std::vector<uint32_t>& order, const std::vector<uint64_t>& bsize,
                        uint32_t tile, uint32_t look, std::vector<uint64_t>& start) {
    const size_t nu = order.size();
    std::vector<char> used(nu, 0);
    start.assign(bsize.size(), 0);
    uint64_t p = 0;
    size_t head = 0, placed = 0;
    while (placed < nu) {
        while (used[head]) ++head;
        const uint64_t room = tile - p % tile;
        size_t pick = head;
        const uint64_t s0 = bsize[order[head]];
        if (s0 <= tile && s0 > room) {
            pick = nu;
            for (size_t i = head + 1, seen = 0; i < nu && seen < look; ++i) {
                if (used[i]) continue;
                ++seen;
                if (bsize[order[i]] <= room) {
                    pick = i;
                    break;
                }
            }
            if (pick == nu) {
                p = (p / tile + 1) * tile;
                pick = head;
            }
        }
        used[pick] = 1;
        start[order[pick]] = p;
        p += bsize[order[pick]];
        ++placed;
    }
    return p;
}

}  // namespace pspg
