// Tile-level work of the sparse boundary-graph FW (K2) for unit layouts
// (diagnostic for bg_order.hpp; unit graph from tools/k2_units.py).
// A layout = elimination order of the units + their start positions. At
// k-block kb every not yet eliminated unit overlapping [kb T, kb T + T) is
// eliminated (fill as in bg_unit_order); the active tiles are the tiles
// covered by the units in the union of their reach sets, and the block costs
// a (a + 1) / 2 tile products.
//   g++ -O2 -std=c++17 -Ipaper_1503_07192_b200/csrc tools/k2_layout_sim.cpp -o /tmp/k2sim
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include "bg_order.hpp"

using namespace pspg;
static const uint32_t T = 128;

struct Units {
    uint32_t nu;
    std::vector<uint64_t> bsize;
    std::vector<std::pair<uint32_t, uint32_t>> adj;
};

struct Fill {
    uint32_t k, W;
    std::vector<uint64_t> F;
    std::vector<double> w;
    std::vector<char> done;
    const std::vector<uint64_t>& bs;
    Fill(const Units& U) : k(U.nu), W((U.nu + 63) / 64), F(uint64_t(U.nu) * W, 0), w(U.nu, 0), done(U.nu, 0), bs(U.bsize) {
        auto set = [&](uint32_t i, uint32_t j) { F[uint64_t(i) * W + j / 64] |= 1ull << (j % 64); };
        for (uint32_t c = 0; c < k; ++c) set(c, c);
        for (auto& e : U.adj) { set(e.first, e.second); set(e.second, e.first); }
        for (uint32_t i = 0; i < k; ++i) w[i] = weight(&F[uint64_t(i) * W]);
    }
    double weight(const uint64_t* r) const {
        double s = 0;
        for (uint32_t x = 0; x < W; ++x)
            for (uint64_t b = r[x]; b; b &= b - 1) s += double(bs[x * 64 + __builtin_ctzll(b)]);
        return s;
    }
    const uint64_t* row(uint32_t p) const { return &F[uint64_t(p) * W]; }
    void eliminate(uint32_t p) {
        std::vector<uint64_t> R(row(p), row(p) + W);
        done[p] = 1;
        for (uint32_t x = 0; x < W; ++x)
            for (uint64_t b = R[x]; b; b &= b - 1) {
                const uint32_t i = x * 64 + __builtin_ctzll(b);
                if (done[i]) continue;
                uint64_t* r = &F[uint64_t(i) * W];
                for (uint32_t y = 0; y < W; ++y) {
                    for (uint64_t add = R[y] & ~r[y]; add; add &= add - 1) w[i] += double(bs[y * 64 + __builtin_ctzll(add)]);
                    r[y] |= R[y];
                }
            }
    }
};

// tile products of a layout
double simulate(const Units& U, const std::vector<uint32_t>& order, const std::vector<uint64_t>& start, uint64_t npos,
                const char* trace = nullptr) {
    FILE* tf = trace ? std::fopen(trace, "w") : nullptr;
    Fill f(U);
    const uint32_t nb = uint32_t((npos + T - 1) / T);
    std::vector<uint64_t> reach(f.W);
    double work = 0;
    size_t oi = 0;
    std::vector<char> tileact(nb);
    for (uint32_t kb = 0; kb < nb; ++kb) {
        std::fill(reach.begin(), reach.end(), 0);
        bool any = false;
        while (oi < order.size() && start[order[oi]] < uint64_t(kb + 1) * T) {
            const uint32_t p = order[oi++];
            for (uint32_t x = 0; x < f.W; ++x) reach[x] |= f.row(p)[x];
            f.eliminate(p);
            any = true;
        }
        std::fill(tileact.begin(), tileact.end(), 0);
        tileact[kb] = 1;
        if (any)
            for (uint32_t x = 0; x < f.W; ++x)
                for (uint64_t b = reach[x]; b; b &= b - 1) {
                    const uint32_t u = x * 64 + __builtin_ctzll(b);
                    for (uint64_t t = start[u] / T; t <= (start[u] + U.bsize[u] - 1) / T; ++t) tileact[t] = 1;
                }
        double a = 0;
        for (char c : tileact) a += c;
        work += a * (a + 1) / 2;
        if (tf) std::fprintf(tf, "%u %.0f\n", kb, a);
    }
    if (tf) std::fclose(tf);
    return work;
}

void contiguous(const Units& U, const std::vector<uint32_t>& order, bool pad, std::vector<uint64_t>& start, uint64_t& npos) {
    start.assign(U.nu, 0);
    uint64_t p = 0;
    for (uint32_t u : order) {
        const uint64_t s = U.bsize[u];
        if (pad && s <= T && (p % T) + s > T) p = (p / T + 1) * T;
        start[u] = p;
        p += s;
    }
    npos = p;
}

// tile-aware greedy: a tile starts with the minimum-reach unit; it is then
// filled from the units of the running reach union (fewest new weight
// first) that fit; padding when none fits (straddle = false)
void tile_greedy(const Units& U, bool straddle, std::vector<uint32_t>& order, std::vector<uint64_t>& start, uint64_t& npos) {
    Fill f(U);
    order.clear();
    start.assign(U.nu, 0);
    uint64_t p = 0;
    std::vector<uint64_t> uni(f.W);
    uint32_t left = U.nu;
    while (left) {
        // new tile
        uint32_t best = U.nu;
        for (uint32_t c = 0; c < U.nu; ++c)
            if (!f.done[c] && (best == U.nu || f.w[c] < f.w[best])) best = c;
        std::copy(f.row(best), f.row(best) + f.W, uni.begin());
        auto place = [&](uint32_t u) {
            start[u] = p;
            p += U.bsize[u];
            order.push_back(u);
            f.eliminate(u);
            --left;
        };
        place(best);
        while (left && p % T != 0) {
            const uint64_t room = T - p % T;
            uint32_t cand = U.nu;
            double cw = 0;
            for (uint32_t x = 0; x < f.W; ++x)
                for (uint64_t b = uni[x]; b; b &= b - 1) {
                    const uint32_t u = x * 64 + __builtin_ctzll(b);
                    if (f.done[u] || (!straddle && U.bsize[u] > room)) continue;
                    // new weight this unit adds to the union
                    double add = 0;
                    const uint64_t* r = f.row(u);
                    for (uint32_t y = 0; y < f.W; ++y)
                        for (uint64_t q = r[y] & ~uni[y]; q; q &= q - 1) add += double(U.bsize[y * 64 + __builtin_ctzll(q)]);
                    if (cand == U.nu || add < cw) { cand = u; cw = add; }
                }
            if (cand == U.nu) {
                if (straddle) break;  // start a new group right here
                p = (p / T + 1) * T;  // pad
                break;
            }
            for (uint32_t y = 0; y < f.W; ++y) uni[y] |= f.row(cand)[y];
            place(cand);
        }
    }
    npos = p;
}

// greedy order packed into tiles: a unit that would straddle a tile
// boundary is swapped for the first of the next `look` units that fits the
// room left; padding when none does
void lookahead(const Units& U, const std::vector<uint32_t>& order, uint32_t look, std::vector<uint32_t>& out,
               std::vector<uint64_t>& start, uint64_t& npos) {
    std::vector<uint32_t> q(order);
    std::vector<char> used(q.size(), 0);
    out.clear();
    start.assign(U.nu, 0);
    uint64_t p = 0;
    size_t head = 0;
    while (out.size() < q.size()) {
        while (used[head]) ++head;
        const uint64_t room = T - p % T;
        size_t pick = head;
        if (U.bsize[q[head]] <= T && U.bsize[q[head]] > room) {
            pick = SIZE_MAX;
            for (size_t i = head + 1, seen = 0; i < q.size() && seen < look; ++i) {
                if (used[i]) continue;
                ++seen;
                if (U.bsize[q[i]] <= room) { pick = i; break; }
            }
            if (pick == SIZE_MAX) { p = (p / T + 1) * T; pick = head; }
        }
        used[pick] = 1;
        start[q[pick]] = p;
        p += U.bsize[q[pick]];
        out.push_back(q[pick]);
    }
    npos = p;
}

int main(int argc, char** argv) {
    FILE* fp = std::fopen(argv[1], "rb");
    Units U;
    std::fread(&U.nu, 4, 1, fp);
    U.bsize.resize(U.nu);
    std::fread(U.bsize.data(), 8, U.nu, fp);
    uint64_t na;
    std::fread(&na, 8, 1, fp);
    std::vector<uint32_t> raw(2 * na);
    std::fread(raw.data(), 4, 2 * na, fp);
    for (uint64_t i = 0; i < na; ++i) U.adj.emplace_back(raw[2 * i], raw[2 * i + 1]);
    uint64_t b = 0;
    for (auto s : U.bsize) b += s;
    const double T3 = double(T) * T * T;
    BgOrder g = bg_unit_order(U.nu, U.bsize, U.adj);
    std::printf("units %u, b %llu: unit-level simulated work greedy %.3e, natural %.3e relaxations\n", U.nu,
                (unsigned long long)b, g.work, g.natural);
    std::vector<uint32_t> ident(U.nu);
    for (uint32_t i = 0; i < U.nu; ++i) ident[i] = i;
    std::vector<uint64_t> st;
    uint64_t np;
    contiguous(U, ident, false, st, np);
    std::printf("natural contiguous       : %.3e relax (nb %llu)\n", simulate(U, ident, st, np) * T3, (unsigned long long)((np + T - 1) / T));
    contiguous(U, g.order, false, st, np);
    std::printf("greedy contiguous (now)  : %.3e relax (nb %llu)\n", simulate(U, g.order, st, np, argc > 3 ? argv[3] : nullptr) * T3, (unsigned long long)((np + T - 1) / T));
    contiguous(U, g.order, true, st, np);
    std::printf("greedy, no straddle      : %.3e relax (nb %llu)\n", simulate(U, g.order, st, np) * T3, (unsigned long long)((np + T - 1) / T));
    std::vector<uint32_t> o2;
    tile_greedy(U, false, o2, st, np);
    std::printf("tile greedy, padded      : %.3e relax (nb %llu)\n", simulate(U, o2, st, np) * T3, (unsigned long long)((np + T - 1) / T));
    tile_greedy(U, true, o2, st, np);
    std::printf("tile greedy, straddling  : %.3e relax (nb %llu)\n", simulate(U, o2, st, np) * T3, (unsigned long long)((np + T - 1) / T));
    for (uint32_t look : {4u, 16u, 64u, 256u}) {
        lookahead(U, g.order, look, o2, st, np);
        std::printf("greedy, lookahead %4u   : %.3e relax (nb %llu)\n", look,
                    simulate(U, o2, st, np, look == 16 && argc > 2 ? argv[2] : nullptr) * T3, (unsigned long long)((np + T - 1) / T));
    }
    return 0;
}
