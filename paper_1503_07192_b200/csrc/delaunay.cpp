// delaunay.cpp — Delaunay triangulation of the benchmark point sets
// (BASELINE.json configs[1]/[2]: n uniform points in [0,1)^2 drawn by numpy
// default_rng, workloads.py), so the 1M-vertex input is generated in ~1 s
// instead of scipy Qhull's ~12 s. The edge set must be the one Qhull gives
// (tests/test_host.py::test_delaunay_generator_matches_qhull): for points in
// general position the Delaunay triangulation is unique, and every decision
// here is exact.
//
// * Exact predicates. numpy's doubles in [0,1) are k * 2^-53 with k < 2^53
//   (53-bit mantissa draws), so X = x * 2^53 is an exact int64. orient2d is
//   then exact in __int128 (products < 2^107); incircle is filtered in
//   double (Shewchuk's static bound) and decided exactly in 256-bit
//   integers (products < 2^216) when the filter cannot.
// * Bowyer-Watson insertion with an infinite vertex (ghost triangles on the
//   hull edges, so the hull is exact without a bounding triangle), points
//   inserted along a Hilbert curve and located by a visibility walk from the
//   last new triangle (O(1) expected steps).
// * Output: unique undirected edges u < v of the real triangles, sorted.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <stdexcept>
#include <vector>

namespace pspg {

namespace {

using i128 = __int128;
using u128 = unsigned __int128;

constexpr uint32_t INF_V = 0xffffffffu;  // the infinite vertex
constexpr uint32_t NONE = 0xffffffffu;

struct P {
    int64_t x, y;   // exact: coordinate * 2^53
    double fx, fy;  // the original doubles
};

int sign_i128(i128 v) { return (v > 0) - (v < 0); }

// sign of det [b-a, c-a]: > 0 when a, b, c turn counter-clockwise
int orient(const P& a, const P& b, const P& c) {
    const i128 l = i128(b.x - a.x) * i128(c.y - a.y);
    const i128 r = i128(b.y - a.y) * i128(c.x - a.x);
    return sign_i128(l - r);
}

// 256-bit two's complement, 4 little-endian limbs
struct I256 {
    uint64_t w[4] = {0, 0, 0, 0};
};

I256 mul_i128(i128 a, i128 b) {  // exact signed product, |a|, |b| < 2^127
    const bool neg = (a < 0) != (b < 0);
    const u128 ua = a < 0 ? u128(-a) : u128(a);
    const u128 ub = b < 0 ? u128(-b) : u128(b);
    const uint64_t a0 = uint64_t(ua), a1 = uint64_t(ua >> 64);
    const uint64_t b0 = uint64_t(ub), b1 = uint64_t(ub >> 64);
    const u128 p00 = u128(a0) * b0, p01 = u128(a0) * b1, p10 = u128(a1) * b0, p11 = u128(a1) * b1;
    I256 r;
    r.w[0] = uint64_t(p00);
    u128 mid = (p00 >> 64) + uint64_t(p01) + uint64_t(p10);
    r.w[1] = uint64_t(mid);
    u128 hi = (mid >> 64) + (p01 >> 64) + (p10 >> 64) + uint64_t(p11);
    r.w[2] = uint64_t(hi);
    r.w[3] = uint64_t((hi >> 64) + (p11 >> 64));
    if (neg) {  // two's complement negation
        uint64_t carry = 1;
        for (auto& x : r.w) {
            const u128 t = u128(~x) + carry;
            x = uint64_t(t);
            carry = uint64_t(t >> 64);
        }
    }
    return r;
}

I256 add(const I256& a, const I256& b) {
    I256 r;
    uint64_t carry = 0;
    for (int i = 0; i < 4; ++i) {
        const u128 t = u128(a.w[i]) + b.w[i] + carry;
        r.w[i] = uint64_t(t);
        carry = uint64_t(t >> 64);
    }
    return r;
}

int sign(const I256& a) {
    if (a.w[3] >> 63) return -1;
    return (a.w[0] | a.w[1] | a.w[2] | a.w[3]) ? 1 : 0;
}

// > 0 when d lies strictly inside the circle through a, b, c (ccw)
int incircle(const P& a, const P& b, const P& c, const P& d) {
    const double adx = a.fx - d.fx, ady = a.fy - d.fy;
    const double bdx = b.fx - d.fx, bdy = b.fy - d.fy;
    const double cdx = c.fx - d.fx, cdy = c.fy - d.fy;
    const double bdxcdy = bdx * cdy, cdxbdy = cdx * bdy;
    const double cdxady = cdx * ady, adxcdy = adx * cdy;
    const double adxbdy = adx * bdy, bdxady = bdx * ady;
    const double alift = adx * adx + ady * ady;
    const double blift = bdx * bdx + bdy * bdy;
    const double clift = cdx * cdx + cdy * cdy;
    const double det = alift * (bdxcdy - cdxbdy) + blift * (cdxady - adxcdy) +
                       clift * (adxbdy - bdxady);
    const double perm = (std::fabs(bdxcdy) + std::fabs(cdxbdy)) * alift +
                        (std::fabs(cdxady) + std::fabs(adxcdy)) * blift +
                        (std::fabs(adxbdy) + std::fabs(bdxady)) * clift;
    constexpr double eps = 1.1102230246251565e-16;  // 2^-53
    const double bound = (10.0 + 96.0 * eps) * eps * perm;
    if (det > bound) return 1;
    if (-det > bound) return -1;
    // exact: differences < 2^53, lifts < 2^107, crosses < 2^107
    const i128 ax = a.x - d.x, ay = a.y - d.y, bx = b.x - d.x, by = b.y - d.y;
    const i128 cx = c.x - d.x, cy = c.y - d.y;
    const i128 la = ax * ax + ay * ay, lb = bx * bx + by * by, lc = cx * cx + cy * cy;
    const I256 t = add(add(mul_i128(la, bx * cy - cx * by), mul_i128(lb, cx * ay - ax * cy)),
                       mul_i128(lc, ax * by - bx * ay));
    return sign(t);
}

struct Tri {
    uint32_t v[3];   // counter-clockwise; a ghost holds INF_V at v[2]
    uint32_t nb[3];  // nb[i]: across the edge opposite v[i]
};

class Triangulator {
public:
    explicit Triangulator(const std::vector<P>& pts) : p_(pts) {}

    void run(const std::vector<uint32_t>& order) {
        // first triangle: the first three points of the order that are not
        // collinear (later ones are re-inserted normally)
        size_t i2 = 2;
        while (i2 < order.size() && orient(p_[order[0]], p_[order[1]], p_[order[i2]]) == 0) ++i2;
        if (i2 == order.size()) throw std::invalid_argument("delaunay: all points collinear");
        uint32_t a = order[0], b = order[1], c = order[i2];
        if (orient(p_[a], p_[b], p_[c]) < 0) std::swap(b, c);
        // the triangle and one ghost per edge (the edge reversed, so the
        // outside lies on the ghost edge's left), linked by shared edges
        const uint32_t t4[4] = {make(a, b, c), make(b, a, INF_V), make(c, b, INF_V),
                                make(a, c, INF_V)};
        for (uint32_t x : t4)
            for (uint32_t y : t4)
                if (x != y)
                    for (int e = 0; e < 3; ++e) {
                        const uint32_t u = T(y).v[(e + 1) % 3], w = T(y).v[(e + 2) % 3];
                        if (has_edge(x, u, w)) set_nb(x, u, w, y);
                    }
        last_ = t4[0];
        for (size_t i = 2; i < order.size(); ++i)
            if (i != i2) insert(order[i]);
    }

    template <typename F>
    void for_each_edge(F&& f) const {
        for (size_t t = 0; t < tris_.size(); ++t) {
            if (dead_[t]) continue;
            const Tri& x = tris_[t];
            if (x.v[2] == INF_V) continue;
            for (int e = 0; e < 3; ++e) {
                const uint32_t u = x.v[(e + 1) % 3], w = x.v[(e + 2) % 3];
                // each interior edge once (from the lower triangle index),
                // hull edges (ghost neighbour) always
                const uint32_t o = x.nb[e];
                if (tris_[o].v[2] == INF_V || t < o) f(std::min(u, w), std::max(u, w));
            }
        }
    }

private:
    const std::vector<P>& p_;
    std::vector<Tri> tris_;
    std::vector<char> dead_;
    std::vector<uint32_t> free_;
    uint32_t last_ = 0;
    // Bowyer-Watson scratch
    std::vector<uint32_t> cavity_, stack_;
    std::vector<char> in_cav_;
    struct BEdge {
        uint32_t x, y, outside;  // boundary edge x->y (cavity on its left), outer triangle
    };
    std::vector<BEdge> bnd_;

    Tri& T(uint32_t t) { return tris_[t]; }

    uint32_t make(uint32_t a, uint32_t b, uint32_t c) {
        uint32_t t;
        if (!free_.empty()) {
            t = free_.back();
            free_.pop_back();
            dead_[t] = 0;
        } else {
            t = uint32_t(tris_.size());
            tris_.push_back({});
            dead_.push_back(0);
            in_cav_.push_back(0);
        }
        // canonical ghost: INF_V last, keeping the cyclic order
        if (a == INF_V) { const uint32_t s = a; a = b; b = c; c = s; }
        else if (b == INF_V) { const uint32_t s = b; b = a; a = c; c = s; }
        tris_[t].v[0] = a, tris_[t].v[1] = b, tris_[t].v[2] = c;
        tris_[t].nb[0] = tris_[t].nb[1] = tris_[t].nb[2] = NONE;
        return t;
    }
    bool has_edge(uint32_t t, uint32_t a, uint32_t b) const {
        const Tri& x = tris_[t];
        for (int e = 0; e < 3; ++e) {
            const uint32_t u = x.v[(e + 1) % 3], w = x.v[(e + 2) % 3];
            if ((u == a && w == b) || (u == b && w == a)) return true;
        }
        return false;
    }

    // circumcircle of t strictly contains point q (ghosts: q strictly on the
    // outer side of the hull edge, or on the open hull edge)
    bool contains(uint32_t t, uint32_t q) const {
        const Tri& x = tris_[t];
        const P& d = p_[q];
        if (x.v[2] == INF_V) {
            const P& a = p_[x.v[0]];
            const P& b = p_[x.v[1]];
            const int o = orient(a, b, d);
            if (o != 0) return o > 0;
            // collinear: inside the open segment (a, b)
            const i128 dot = i128(d.x - a.x) * (b.x - a.x) + i128(d.y - a.y) * (b.y - a.y);
            const i128 len = i128(b.x - a.x) * (b.x - a.x) + i128(b.y - a.y) * (b.y - a.y);
            return dot > 0 && dot < len;
        }
        return incircle(p_[x.v[0]], p_[x.v[1]], p_[x.v[2]], d) > 0;
    }

    // visibility walk to a triangle whose circumcircle contains q
    uint32_t locate(uint32_t q) {
        uint32_t t = last_;
        if (dead_[t]) t = 0;
        while (dead_[t]) ++t;
        uint32_t rot = 0;
        for (uint64_t steps = 0;; ++steps) {
            const Tri& x = tris_[t];
            if (x.v[2] == INF_V) return t;  // outside the hull: this ghost sees q
            bool moved = false;
            for (int k = 0; k < 3 && !moved; ++k) {
                const int e = int((k + rot) % 3);
                const P& a = p_[x.v[(e + 1) % 3]];
                const P& b = p_[x.v[(e + 2) % 3]];
                if (orient(a, b, p_[q]) < 0) {
                    t = x.nb[e];
                    moved = true;
                }
            }
            if (!moved) return t;  // q inside or on the boundary of t
            rot = (rot + 1) % 3;
            if (steps > tris_.size() + 16) throw std::runtime_error("delaunay: walk did not end");
        }
    }

    void insert(uint32_t q) {
        const uint32_t start = locate(q);
        // cavity: triangles whose circumcircle contains q (connected, star
        // shaped around q); the located triangle always belongs to it
        cavity_.clear();
        stack_.clear();
        stack_.push_back(start);
        in_cav_[start] = 1;
        while (!stack_.empty()) {
            const uint32_t t = stack_.back();
            stack_.pop_back();
            cavity_.push_back(t);
            for (int e = 0; e < 3; ++e) {
                const uint32_t o = tris_[t].nb[e];
                if (in_cav_[o]) continue;
                if (contains(o, q)) {
                    in_cav_[o] = 1;
                    stack_.push_back(o);
                }
            }
        }
        // its boundary edges, oriented with the cavity on the left
        bnd_.clear();
        for (uint32_t t : cavity_) {
            const Tri& x = tris_[t];
            for (int e = 0; e < 3; ++e) {
                const uint32_t o = x.nb[e];
                if (!in_cav_[o]) bnd_.push_back({x.v[(e + 1) % 3], x.v[(e + 2) % 3], o});
            }
        }
        for (uint32_t t : cavity_) {
            in_cav_[t] = 0;
            dead_[t] = 1;
            free_.push_back(t);
        }
        // fan of new triangles (x, y, q) over the boundary
        const size_t nbnd = bnd_.size();
        std::vector<uint32_t>& made = stack_;  // reuse
        made.assign(nbnd, 0);
        for (size_t i = 0; i < nbnd; ++i) {
            const BEdge& e = bnd_[i];
            const uint32_t t = make(e.x, e.y, q);
            made[i] = t;
            // across (x, y): the outer triangle; fix its back link
            set_nb(t, e.x, e.y, e.outside);
            set_nb(e.outside, e.y, e.x, t);
        }
        // neighbours among the new triangles: (x, y, q) and the one whose
        // boundary edge starts at y share edge (y, q)
        for (size_t i = 0; i < nbnd; ++i) {
            for (size_t j = 0; j < nbnd; ++j) {
                if (bnd_[j].x != bnd_[i].y) continue;
                set_nb(made[i], bnd_[i].y, q, made[j]);
                set_nb(made[j], q, bnd_[j].x, made[i]);
                break;
            }
        }
        // continue walking from a real new triangle
        for (size_t i = 0; i < nbnd; ++i)
            if (tris_[made[i]].v[2] != INF_V) {
                last_ = made[i];
                break;
            }
    }

    // in triangle t, set the neighbour across the edge {a, b}
    void set_nb(uint32_t t, uint32_t a, uint32_t b, uint32_t o) {
        Tri& x = tris_[t];
        for (int e = 0; e < 3; ++e) {
            const uint32_t u = x.v[(e + 1) % 3], w = x.v[(e + 2) % 3];
            if ((u == a && w == b) || (u == b && w == a)) {
                x.nb[e] = o;
                return;
            }
        }
        throw std::runtime_error("delaunay: broken adjacency");
    }
};

// Hilbert index of (x, y) on a 2^16 grid
uint64_t hilbert(uint32_t x, uint32_t y) {
    uint64_t d = 0;
    for (uint32_t s = 1u << 15; s > 0; s >>= 1) {
        const uint32_t rx = (x & s) ? 1 : 0, ry = (y & s) ? 1 : 0;
        d += uint64_t(s) * s * ((3 * rx) ^ ry);
        if (ry == 0) {
            if (rx == 1) {
                x = s - 1 - x;
                y = s - 1 - y;
            }
            std::swap(x, y);
        }
    }
    return d;
}

}  // namespace

// Unique undirected Delaunay edges (u < v, lexicographic) of points xy
// (n x 2, row-major, every coordinate in [0, 1) with a 53-bit mantissa grid).
void delaunay_edges(uint64_t n, const double* xy, std::vector<uint32_t>& eu,
                    std::vector<uint32_t>& ev) {
    if (n < 3) throw std::invalid_argument("delaunay: needs at least 3 points");
    if (n >= INF_V) throw std::invalid_argument("delaunay: too many points");
    std::vector<P> pts(n);
    const double scale = 9007199254740992.0;  // 2^53
    for (uint64_t i = 0; i < n; ++i) {
        const double x = xy[2 * i], y = xy[2 * i + 1];
        if (!(x >= 0.0 && x < 1.0 && y >= 0.0 && y < 1.0))
            throw std::invalid_argument("delaunay: coordinates must lie in [0, 1)");
        const double sx = x * scale, sy = y * scale;
        if (sx != std::floor(sx) || sy != std::floor(sy))
            throw std::invalid_argument("delaunay: coordinates must be multiples of 2^-53");
        pts[i] = {int64_t(sx), int64_t(sy), x, y};
    }
    std::vector<std::pair<uint64_t, uint32_t>> key(n);
    for (uint64_t i = 0; i < n; ++i)
        key[i] = {hilbert(uint32_t(xy[2 * i] * 65536.0), uint32_t(xy[2 * i + 1] * 65536.0)),
                  uint32_t(i)};
    std::sort(key.begin(), key.end());
    std::vector<uint32_t> order(n);
    for (uint64_t i = 0; i < n; ++i) order[i] = key[i].second;
    // duplicate points would make the triangulation ill-defined
    {
        std::vector<std::pair<int64_t, int64_t>> c(n);
        for (uint64_t i = 0; i < n; ++i) c[i] = {pts[i].x, pts[i].y};
        std::sort(c.begin(), c.end());
        if (std::adjacent_find(c.begin(), c.end()) != c.end())
            throw std::invalid_argument("delaunay: duplicate points");
    }
    Triangulator tr(pts);
    tr.run(order);
    std::vector<uint64_t> keys;
    keys.reserve(3 * n);
    tr.for_each_edge([&](uint32_t u, uint32_t v) { keys.push_back((uint64_t(u) << 32) | v); });
    std::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
    eu.resize(keys.size());
    ev.resize(keys.size());
    for (size_t i = 0; i < keys.size(); ++i) {
        eu[i] = uint32_t(keys[i] >> 32);
        ev[i] = uint32_t(keys[i]);
    }
}

}  // namespace pspg
