// partition.cpp — host k-way partitioner with output identical to the
// reference's partition_graph (src/partition.cpp:259-450).
//
// Why restate it: BASELINE.json keeps the reference's partition + boundary
// extraction on the host "so component assignment matches the oracle"; the
// product library must not link reference sources, so the algorithm is
// re-expressed here and checked for identical assignments against the
// reference build (tests/test_partition.py).
//
// What is the same (bit for bit): the mt19937_64 stream and its order of use,
// seed selection (farthest-point first restart, best-of-8 candidates after),
// hop-count Voronoi growth with smallest-id tie breaking, recentering,
// finalize = fill unreached + rebalance + refine sweeps, the cost
// sum |B(C)|^2 and the first-strict-minimum candidate choice over
// (restart, round).
//
// What differs (speed only):
//  * the 8 restarts are independent once their seed sets are drawn, and
//    finalize() never feeds back into a chain (recentering reads the
//    un-finalized growth), so the work runs as a dataflow on a task pool:
//    the seed draws stay sequential (they share the rng and the id
//    shuffle), each restart's grow/recenter chain starts as soon as its
//    seeds exist, and each of the 8 x 13 grown states spawns its
//    finalize() (the expensive part) on any free host thread; the winner
//    is the first minimum in (restart, round) order exactly as the
//    reference's strict `<` scan picks it, kept as the passes finish.
//  * all per-vertex state lives in a BFS-ordered relabelling of the graph
//    (struct Local), so neighbourhoods are compact in memory; rules that
//    depend on id order compare original ids, loops whose order matters
//    still run in original id order, and grow/recenter evaluate their
//    order-free closed forms (smallest-id claimant, smallest-id deepest
//    vertex) instead of replaying the reference's sorted frontiers.
//  * the seed draws' argmax keeps per-block maxima; refine keeps per-vertex
//    foreign-neighbour counts (O(deg) per candidate move instead of
//    O(deg^2)), walks the flagged vertices through a bitset and prefetches
//    ahead of its random-order sweep.
//  * rebalance collects each oversized component's members from per-
//    component buckets instead of rescanning all n vertices; the member
//    order is fixed by the reference's total (hop desc, id asc) sort anyway.
// tools/part_bench.cpp times it without Python; tests/test_host.py checks
// the assignments against the reference build, including scrambled ids.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <atomic>
#include <condition_variable>
#include <deque>
#include <functional>
#include <cstdint>
#include <exception>
#include <limits>
#include <mutex>
#include <numeric>
#include <random>
#include <stdexcept>
#include <barrier>
#include <thread>
#include <vector>

#include "host_graph.hpp"

namespace pspg {

namespace {

constexpr uint32_t kNone = 0xffffffffu;   // kUnassigned (:14)
constexpr int kMaxRefineSweeps = 10;      // (:15)
constexpr int kRecenterRounds = 12;       // (:16)
constexpr int kRestarts = 8;              // (:17)
constexpr uint64_t kSeedCandidates = 8;   // (:18)
constexpr int kAhead = 16;                // refine's prefetch distance, in flagged vertices

// balance_cap (:191-194): ceil(1.1 n / k) in integers
uint64_t cap_of(uint64_t n, uint32_t k) { return (11 * n + 10 * uint64_t(k) - 1) / (10 * uint64_t(k)); }

// A small work pool for the partition dataflow (cf. psp::parallel_for,
// include/psp/parallel.hpp:15-47, which the reference runs per phase):
// `threads - 1` workers plus the thread that calls join(). High-priority
// tasks run first. Tasks may push further tasks. The first exception stops
// the pool (queued tasks are dropped) and is rethrown by join().
class TaskPool {
public:
    explicit TaskPool(unsigned threads) {
        for (unsigned t = 1; t < threads; ++t) pool_.emplace_back([this] { work(); });
    }
    ~TaskPool() {
        {
            std::lock_guard<std::mutex> lock(mu_);
            closed_ = stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : pool_) t.join();
    }
    void push(bool high, std::function<void()> fn) {
        {
            std::lock_guard<std::mutex> lock(mu_);
            (high ? hi_ : lo_).push_back(std::move(fn));
            ++pending_;
        }
        cv_.notify_one();
    }
    void join() {
        {
            std::lock_guard<std::mutex> lock(mu_);
            closed_ = true;
        }
        cv_.notify_all();
        work();
        for (auto& t : pool_) t.join();
        pool_.clear();
        if (err_) std::rethrow_exception(err_);
    }

private:
    void work() {
        std::unique_lock<std::mutex> lock(mu_);
        for (;;) {
            cv_.wait(lock, [&] { return stop_ || !hi_.empty() || !lo_.empty() || (closed_ && pending_ == 0); });
            if (stop_ || (hi_.empty() && lo_.empty())) return;
            auto& q = hi_.empty() ? lo_ : hi_;
            std::function<void()> fn = std::move(q.front());
            q.pop_front();
            lock.unlock();
            try {
                fn();
            } catch (...) {
                lock.lock();
                if (!err_) err_ = std::current_exception();
                stop_ = true;
                pending_ -= 1 + hi_.size() + lo_.size();
                hi_.clear();
                lo_.clear();
                cv_.notify_all();
                return;
            }
            lock.lock();
            if (--pending_ == 0) cv_.notify_all();
        }
    }

    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::function<void()>> hi_, lo_;
    size_t pending_ = 0;
    bool closed_ = false, stop_ = false;
    std::exception_ptr err_;
    std::vector<std::thread> pool_;
};

// The graph relabelled in BFS order (every connected piece, pieces in id
// order of their first vertex). Vertex ids in the reference's inputs need
// carry no locality -- a Delaunay mesh of random points scatters every
// neighbourhood over the whole id range -- so every pass below is bound by
// cache misses on the original numbering. All per-vertex state lives at
// `pos[v]`; every comparison the reference makes on vertex ids is made on
// `id[u]`, the original id, and every loop whose order matters still runs
// in original id order (u = pos[v] for v = 0, 1, ...).
struct Local {
    uint64_t n = 0;
    std::vector<uint32_t> pos, id;  // original -> local, local -> original
    std::vector<uint64_t> off;
    std::vector<uint32_t> to;

    explicit Local(const Csr& g) : n(g.n), pos(g.n), id(g.n), off(g.n + 1), to(g.to.size()) {
        std::vector<uint8_t> seen(n, 0);
        uint64_t tail = 0;
        for (uint64_t r = 0; r < n; ++r) {
            if (seen[r]) continue;
            seen[r] = 1;
            uint64_t head = tail;
            id[tail++] = static_cast<uint32_t>(r);
            for (; head < tail; ++head) {
                const uint32_t u = id[head];
                for (uint64_t e = g.off[u]; e < g.off[u + 1]; ++e)
                    if (!seen[g.to[e]]) {
                        seen[g.to[e]] = 1;
                        id[tail++] = g.to[e];
                    }
            }
        }
        for (uint64_t i = 0; i < n; ++i) pos[id[i]] = static_cast<uint32_t>(i);
        off[0] = 0;
        for (uint64_t i = 0; i < n; ++i) {
            const uint32_t u = id[i];
            uint64_t o = off[i];
            for (uint64_t e = g.off[u]; e < g.off[u + 1]; ++e) to[o++] = pos[g.to[e]];
            off[i + 1] = o;
        }
    }
    uint64_t begin(uint32_t u) const { return off[u]; }
    uint64_t end(uint32_t u) const { return off[u + 1]; }
};

// compute_boundary (:196-212) on local storage
std::vector<uint8_t> local_boundary(const Local& g, const std::vector<uint32_t>& a) {
    std::vector<uint8_t> flags(g.n, 0);
    for (uint64_t u = 0; u < g.n; ++u)
        for (uint64_t e = g.begin(u); e < g.end(u); ++e)
            if (a[g.to[e]] != a[u]) {
                flags[u] = 1;
                break;
            }
    return flags;
}

// The seed draws' hop-count distances (relax_seed_dist, :272-284). After
// relax_from(s) every vertex holds min(old, hop(s, v)) whatever order the
// FIFO visits neighbours in (a vertex improves only if every vertex on a
// shortest path from s to it does), so the relabelling cannot change them.
// farthest_seeds' argmax (the first maximum in id order, :320-324) comes
// from per-block maxima that a relax only dirties where it changed one.
class SeedSpace {
public:
    explicit SeedSpace(const Local& g) : g_(g), dist_(g.n) {
        nblk_ = (g.n + kBlock - 1) / kBlock;
        barg_.resize(nblk_);
        dirty_.assign(nblk_, 0);
    }
    void reset() {
        std::fill(dist_.begin(), dist_.end(), kNone);
        std::fill(dirty_.begin(), dirty_.end(), 1);
        dirty_list_.resize(nblk_);
        std::iota(dirty_list_.begin(), dirty_list_.end(), 0u);
    }
    uint32_t dist_of(uint32_t v) const { return dist_[g_.pos[v]]; }
    void relax_from(uint32_t v) {
        const uint32_t s = g_.pos[v];
        set(s, 0);
        q_.assign(1, s);
        for (size_t head = 0; head < q_.size(); ++head) {
            const uint32_t u = q_[head];
            const uint32_t du = dist_[u] + 1;
            for (uint64_t e = g_.begin(u); e < g_.end(u); ++e) {
                const uint32_t x = g_.to[e];
                if (dist_[x] > du) {
                    set(x, du);
                    q_.push_back(x);
                }
            }
        }
    }
    uint32_t farthest() {
        for (uint32_t b : dirty_list_) {
            const uint64_t lo = uint64_t(b) * kBlock, hi = std::min<uint64_t>(lo + kBlock, g_.n);
            uint32_t best = static_cast<uint32_t>(lo);
            for (uint64_t i = lo + 1; i < hi; ++i)
                if (better(static_cast<uint32_t>(i), best)) best = static_cast<uint32_t>(i);
            barg_[b] = best;
            dirty_[b] = 0;
        }
        dirty_list_.clear();
        uint32_t best = barg_[0];
        for (uint64_t b = 1; b < nblk_; ++b)
            if (better(barg_[b], best)) best = barg_[b];
        return g_.id[best];
    }

private:
    static constexpr uint64_t kBlock = 256;
    bool better(uint32_t a, uint32_t b) const {
        return dist_[a] > dist_[b] || (dist_[a] == dist_[b] && g_.id[a] < g_.id[b]);
    }
    void set(uint32_t x, uint32_t d) {
        dist_[x] = d;
        const uint32_t b = static_cast<uint32_t>(x / kBlock);
        if (!dirty_[b]) {
            dirty_[b] = 1;
            dirty_list_.push_back(b);
        }
    }
    const Local& g_;
    uint64_t nblk_ = 0;
    std::vector<uint32_t> dist_, q_, barg_, dirty_list_;
    std::vector<uint8_t> dirty_;
};

// PSP_PART_PROFILE: summed thread time of the phases (ns)
std::atomic<uint64_t> g_ns_grow{0}, g_ns_recenter{0}, g_ns_finalize{0};
struct PhaseTimer {
    std::atomic<uint64_t>& acc;
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    ~PhaseTimer() {
        acc += uint64_t(std::chrono::duration_cast<std::chrono::nanoseconds>(
                            std::chrono::steady_clock::now() - t0).count());
    }
};

// The restart chain and finalize on local storage: `assign` and `hop` are
// indexed by local position, seeds are original ids.
struct Part {
    const Local& g;
    uint32_t k;
    uint64_t cap;

    // voronoi_grow (:40-72). The reference visits the frontier in id order
    // and lets the first visitor claim, so x goes to the component of its
    // smallest-id frontier neighbour; that rule is order-free and is what
    // is evaluated here, in local order.
    void grow(const std::vector<uint32_t>& seeds, std::vector<uint32_t>& assign,
              std::vector<uint32_t>& hop) const {
        PhaseTimer pt{g_ns_grow};
        const uint64_t n = g.n;
        assign.assign(n, kNone);
        hop.assign(n, kNone);
        // claim[x]: the claimant's position; claim_id[x] its original id (the
        // comparison key, kept beside it so a contest needs no id lookup)
        std::vector<uint32_t> frontier, next, claim(n, kNone), claim_id(n);
        for (uint32_t c = 0; c < seeds.size(); ++c) {
            const uint32_t u = g.pos[seeds[c]];
            assign[u] = c;  // a repeated seed keeps its last component, as in the reference
            hop[u] = 0;
            frontier.push_back(u);
        }
        uint32_t round = 0;
        while (!frontier.empty()) {
            ++round;
            next.clear();
            for (uint32_t u : frontier) {
                const uint32_t iu = g.id[u];
                for (uint64_t e = g.begin(u); e < g.end(u); ++e) {
                    const uint32_t x = g.to[e];
                    if (assign[x] != kNone) continue;
                    if (claim[x] == kNone) {
                        claim[x] = u;
                        claim_id[x] = iu;
                        next.push_back(x);
                    } else if (iu < claim_id[x]) {
                        claim[x] = u;
                        claim_id[x] = iu;
                    }
                }
            }
            for (uint32_t x : next) {
                assign[x] = assign[claim[x]];
                hop[x] = round;
            }
            frontier.swap(next);
        }
    }

    // grow() on `T` threads, level-synchronous: the claim of x is the packed
    // (original id, position) of its smallest-id frontier neighbour, settled by
    // compare-and-swap, so any visiting order gives grow()'s result. Used for
    // the last restarts' chains, which are the partitioner's critical path
    // (the other cores are busy with earlier chains and finalize passes).
    void grow_par(const std::vector<uint32_t>& seeds, std::vector<uint32_t>& assign,
                  std::vector<uint32_t>& hop, unsigned T) const {
        PhaseTimer pt{g_ns_grow};
        const uint64_t n = g.n;
        assign.assign(n, kNone);
        hop.assign(n, kNone);
        std::vector<std::atomic<uint64_t>> claim(n);
        std::vector<uint32_t> frontier, next;
        for (uint32_t c = 0; c < seeds.size(); ++c) {
            const uint32_t u = g.pos[seeds[c]];
            assign[u] = c;  // a repeated seed keeps its last component, as in the reference
            hop[u] = 0;
        }
        for (uint32_t c = 0; c < seeds.size(); ++c) frontier.push_back(g.pos[seeds[c]]);
        std::vector<std::vector<uint32_t>> local(T);
        std::barrier sync(static_cast<std::ptrdiff_t>(T));
        uint32_t round = 0;
        bool done = false;
        auto work = [&](unsigned t) {
            // claims start empty (~0): every thread clears its share
            for (uint64_t x = t; x < n; x += T) claim[x].store(~uint64_t(0), std::memory_order_relaxed);
            sync.arrive_and_wait();
            for (;;) {
                if (done) return;
                // phase 1: claims
                std::vector<uint32_t>& mine = local[t];
                mine.clear();
                const size_t f = frontier.size(), lo = f * t / T, hi = f * (t + 1) / T;
                for (size_t i = lo; i < hi; ++i) {
                    const uint32_t u = frontier[i];
                    const uint64_t key = (uint64_t(g.id[u]) << 32) | u;
                    for (uint64_t e = g.begin(u); e < g.end(u); ++e) {
                        const uint32_t x = g.to[e];
                        if (assign[x] != kNone) continue;
                        uint64_t cur = claim[x].load(std::memory_order_relaxed);
                        while (key < cur) {
                            if (claim[x].compare_exchange_weak(cur, key, std::memory_order_relaxed)) {
                                if (cur == ~uint64_t(0)) mine.push_back(x);
                                break;
                            }
                        }
                    }
                }
                sync.arrive_and_wait();
                if (t == 0) {  // the next frontier, then its assignment
                    ++round;
                    next.clear();
                    for (auto& l : local) next.insert(next.end(), l.begin(), l.end());
                }
                sync.arrive_and_wait();
                const size_t m = next.size(), a0 = m * t / T, a1 = m * (t + 1) / T;
                for (size_t i = a0; i < a1; ++i) {
                    const uint32_t x = next[i];
                    assign[x] = assign[uint32_t(claim[x].load(std::memory_order_relaxed))];
                    hop[x] = round;
                }
                sync.arrive_and_wait();
                if (t == 0) {
                    frontier.swap(next);
                    done = frontier.empty();
                }
                sync.arrive_and_wait();
            }
        };
        std::vector<std::thread> team;
        for (unsigned t = 1; t < T; ++t) team.emplace_back(work, t);
        work(0);
        for (auto& th : team) th.join();
    }

    // recenter (:77-119): per component, the smallest-id vertex of the
    // deepest BFS round from the component's boundary (round 0 = the
    // smallest-id boundary vertex), again an order-free rule.
    std::vector<uint32_t> recenter(const std::vector<uint32_t>& a,
                                   const std::vector<uint32_t>& old) const {
        PhaseTimer pt{g_ns_recenter};
        const uint64_t n = g.n;
        std::vector<uint32_t> seeds(old);
        const std::vector<uint8_t> flags = local_boundary(g, a);
        std::vector<uint32_t> best_hop(seeds.size(), 0), best(seeds.size(), kNone);
        std::vector<uint8_t> visited(n, 0);
        std::vector<uint32_t> frontier, next;
        for (uint64_t u = 0; u < n; ++u)
            if (flags[u]) {
                visited[u] = 1;
                frontier.push_back(static_cast<uint32_t>(u));
                const uint32_t c = a[u];
                if (best[c] == kNone || g.id[u] < g.id[best[c]]) best[c] = static_cast<uint32_t>(u);
            }
        uint32_t round = 0;
        while (!frontier.empty()) {
            ++round;
            next.clear();
            for (uint32_t u : frontier)
                for (uint64_t e = g.begin(u); e < g.end(u); ++e) {
                    const uint32_t x = g.to[e];
                    if (visited[x] || a[x] != a[u]) continue;
                    visited[x] = 1;
                    next.push_back(x);
                }
            for (uint32_t x : next) {
                const uint32_t c = a[x];
                if (round > best_hop[c]) {
                    best_hop[c] = round;
                    best[c] = x;
                } else if (g.id[x] < g.id[best[c]]) {
                    best[c] = x;
                }
            }
            frontier.swap(next);
        }
        for (uint32_t c = 0; c < seeds.size(); ++c)
            if (best[c] != kNone) seeds[c] = g.id[best[c]];
        return seeds;
    }

    // recenter() on `T` threads for the last restarts' chains: the BFS
    // levels (depth from the component's boundary inside the component) do
    // not depend on the visiting order, and the pick -- the smallest id at
    // the deepest level -- is taken after the BFS from per-thread minima, so
    // the seeds are recenter()'s.
    std::vector<uint32_t> recenter_par(const std::vector<uint32_t>& a,
                                       const std::vector<uint32_t>& old, unsigned T) const {
        PhaseTimer pt{g_ns_recenter};
        const uint64_t n = g.n;
        std::vector<uint32_t> seeds(old);
        std::vector<std::atomic<uint8_t>> visited(n);
        std::vector<uint32_t> depth(n, kNone), frontier;
        std::vector<std::vector<uint32_t>> local(T);
        // per thread and component: (depth, id) of the best vertex seen
        std::vector<std::vector<uint64_t>> pick(T);
        std::barrier sync(static_cast<std::ptrdiff_t>(T));
        uint32_t round = 0;
        bool done = false;
        auto work = [&](unsigned t) {
            std::vector<uint32_t>& mine = local[t];
            mine.clear();
            const uint64_t v0 = n * t / T, v1 = n * (t + 1) / T;
            for (uint64_t u = v0; u < v1; ++u) {
                visited[u].store(0, std::memory_order_relaxed);
                for (uint64_t e = g.begin(u); e < g.end(u); ++e)
                    if (a[g.to[e]] != a[u]) {
                        visited[u].store(1, std::memory_order_relaxed);
                        depth[u] = 0;
                        mine.push_back(static_cast<uint32_t>(u));
                        break;
                    }
            }
            sync.arrive_and_wait();
            if (t == 0) {
                frontier.clear();
                for (auto& l : local) frontier.insert(frontier.end(), l.begin(), l.end());
                done = frontier.empty();
            }
            sync.arrive_and_wait();
            while (!done) {
                const uint32_t level = round + 1;
                mine.clear();
                const size_t f = frontier.size(), lo = f * t / T, hi = f * (t + 1) / T;
                for (size_t i = lo; i < hi; ++i) {
                    const uint32_t u = frontier[i];
                    for (uint64_t e = g.begin(u); e < g.end(u); ++e) {
                        const uint32_t x = g.to[e];
                        if (a[x] != a[u] || visited[x].load(std::memory_order_relaxed)) continue;
                        if (visited[x].exchange(1, std::memory_order_relaxed) == 0) {
                            depth[x] = level;
                            mine.push_back(x);
                        }
                    }
                }
                sync.arrive_and_wait();
                if (t == 0) {
                    round = level;
                    frontier.clear();
                    for (auto& l : local) frontier.insert(frontier.end(), l.begin(), l.end());
                    done = frontier.empty();
                }
                sync.arrive_and_wait();
            }
            // deepest level first, then the smallest original id
            std::vector<uint64_t>& pk = pick[t];
            pk.assign(seeds.size(), ~uint64_t(0));
            for (uint64_t u = v0; u < v1; ++u) {
                if (depth[u] == kNone) continue;
                const uint64_t key = (uint64_t(kNone - depth[u]) << 32) | g.id[u];
                pk[a[u]] = std::min(pk[a[u]], key);
            }
        };
        std::vector<std::thread> team;
        for (unsigned t = 1; t < T; ++t) team.emplace_back(work, t);
        work(0);
        for (auto& th : team) th.join();
        for (uint32_t c = 0; c < seeds.size(); ++c) {
            uint64_t best = ~uint64_t(0);
            for (unsigned t = 0; t < T; ++t) best = std::min(best, pick[t][c]);
            if (best != ~uint64_t(0)) seeds[c] = static_cast<uint32_t>(best);
        }
        return seeds;
    }

    // rebalance (:125-175)
    void rebalance(std::vector<uint32_t>& a, const std::vector<uint32_t>& hop,
                   std::vector<uint64_t>& size) const {
        const uint64_t n = g.n;
        bool any = false;
        for (uint32_t c = 0; c < k; ++c) any |= size[c] > cap;
        if (!any) return;
        auto smallest_with_room = [&](uint32_t exclude) {
            uint32_t target = kNone;
            for (uint32_t t = 0; t < k; ++t) {
                if (t == exclude || size[t] + 1 > cap) continue;
                if (target == kNone || size[t] < size[target]) target = t;
            }
            return target;
        };
        // members of c when c is processed = its vertices at entry plus
        // those moved into it while earlier components were trimmed
        std::vector<std::vector<uint32_t>> bucket(k);
        for (uint64_t u = 0; u < n; ++u)
            if (size[a[u]] > cap) bucket[a[u]].push_back(static_cast<uint32_t>(u));
        std::vector<std::vector<uint32_t>> moved_in(k);
        std::vector<uint32_t> members;
        for (uint32_t c = 0; c < k; ++c) {
            if (size[c] <= cap) continue;
            members.clear();
            for (uint32_t u : bucket[c]) if (a[u] == c) members.push_back(u);
            for (uint32_t u : moved_in[c]) if (a[u] == c) members.push_back(u);
            std::sort(members.begin(), members.end(), [&](uint32_t x, uint32_t y) {
                if (hop[x] != hop[y]) return hop[x] > hop[y];
                return g.id[x] < g.id[y];
            });
            for (uint32_t u : members) {
                if (size[c] <= cap) break;
                uint32_t target = kNone;
                for (uint64_t e = g.begin(u); e < g.end(u); ++e) {
                    const uint32_t t = a[g.to[e]];
                    if (t == c || t == kNone || size[t] + 1 > cap) continue;
                    if (target == kNone || size[t] < size[target] ||
                        (size[t] == size[target] && t < target))
                        target = t;
                }
                if (target == kNone) target = smallest_with_room(c);
                a[u] = target;
                --size[c];
                ++size[target];
                if (target > c) moved_in[target].push_back(u);
            }
        }
    }

    // the refine lambda (:334-387), sweeping in original id order. The
    // reference re-derives every boundary flag it needs from scratch
    // (is_boundary_with_move, O(deg) per vertex, so O(deg^2) per candidate
    // move). Here each vertex keeps the number of its neighbours in other
    // components, `foreign`, with flags[x] == (foreign[x] > 0) at all times.
    // On a simple graph (build_csr rejects loops and duplicates) moving v
    // from `from` to `to` changes a neighbour x's count by
    // [a[x] != to] - [a[x] != from], and v's own count becomes
    // deg(v) - #(neighbours in `to`), so a candidate's delta costs O(deg)
    // and the decisions -- same sweep order, same target order, same strict
    // `<` -- are the reference's.
    void refine(std::vector<uint32_t>& a, std::vector<uint64_t>& size,
                std::vector<uint8_t>& flags) const {
        const uint64_t n = g.n;
        std::vector<uint32_t> foreign(n, 0);
        for (uint64_t u = 0; u < n; ++u) {
            if (!flags[u]) continue;
            uint32_t f = 0;
            for (uint64_t e = g.begin(u); e < g.end(u); ++e) f += a[g.to[e]] != a[u];
            foreign[u] = f;
        }
        // flags mirrored as a bitset in original id order, so a sweep skips
        // interior vertices 64 at a time instead of touching each one
        const uint64_t nw = (n + 63) / 64;
        std::vector<uint64_t> bits(nw, 0);
        for (uint64_t u = 0; u < n; ++u)
            if (flags[u]) bits[g.id[u] >> 6] |= uint64_t(1) << (g.id[u] & 63);
        auto set_flag = [&](uint32_t x, bool on) {
            flags[x] = on ? 1 : 0;
            const uint64_t bit = uint64_t(1) << (g.id[x] & 63);
            if (on) bits[g.id[x] >> 6] |= bit;
            else bits[g.id[x] >> 6] &= ~bit;
        };
        // next flagged original id >= v (forward) / <= v (backward), or n;
        // re-read every time: a move may flag or clear vertices ahead
        auto next_fwd = [&](uint64_t v) -> uint64_t {
            if (v >= n) return n;
            uint64_t w = v >> 6, word = bits[w] & (~uint64_t(0) << (v & 63));
            while (!word) {
                if (++w == nw) return n;
                word = bits[w];
            }
            return (w << 6) + __builtin_ctzll(word);
        };
        auto next_bwd = [&](uint64_t v) -> uint64_t {  // v < n, or n for "none"
            if (v >= n) return n;
            uint64_t w = v >> 6, word = bits[w] & (~uint64_t(0) >> (63 - (v & 63)));
            while (!word) {
                if (w-- == 0) return n;
                word = bits[w];
            }
            return (w << 6) + 63 - __builtin_clzll(word);
        };
        std::vector<uint32_t> targets;
        for (int sweep = 0; sweep < kMaxRefineSweeps; ++sweep) {
            bool improved = false;
            const bool fwd = sweep % 2 == 0;
            auto advance = [&](uint64_t ov) {  // next flagged id after ov in sweep order
                return fwd ? next_fwd(ov + 1) : (ov == 0 ? n : next_bwd(ov - 1));
            };
            const uint64_t first = fwd ? next_fwd(0) : next_bwd(n - 1);
            // Software prefetch: the sweep visits vertices in id order, which
            // is random in memory, so it is latency-bound. Three cursors run
            // ahead through the current flags (a hint only: flags may change
            // before the sweep gets there) and pull in, in dependency order,
            // a vertex's state, its adjacency slice and its neighbours' state.
            uint64_t p1 = first, p2 = first, p3 = first;
            for (int i = 0; i < kAhead && p1 < n; ++i) p1 = advance(p1);
            for (int i = 0; i < kAhead / 2 && p2 < n; ++i) p2 = advance(p2);
            for (int i = 0; i < kAhead / 4 && p3 < n; ++i) p3 = advance(p3);
            for (uint64_t ov = first; ov < n; ov = advance(ov)) {
                if (p1 < n) {
                    const uint32_t u = g.pos[p1];
                    __builtin_prefetch(&g.off[u]);
                    __builtin_prefetch(&a[u]);
                    __builtin_prefetch(&foreign[u]);
                    p1 = advance(p1);
                }
                if (p2 < n) {
                    __builtin_prefetch(&g.to[g.off[g.pos[p2]]]);
                    p2 = advance(p2);
                }
                if (p3 < n) {
                    const uint32_t u = g.pos[p3];
                    for (uint64_t e = g.begin(u); e < g.end(u); ++e) {
                        __builtin_prefetch(&a[g.to[e]]);
                        __builtin_prefetch(&foreign[g.to[e]]);
                    }
                    p3 = advance(p3);
                }
                const uint32_t v = g.pos[ov];
                const uint32_t from = a[v];
                if (size[from] <= 1) continue;
                targets.clear();
                for (uint64_t e = g.begin(v); e < g.end(v); ++e) {
                    const uint32_t c = a[g.to[e]];
                    if (c != from && std::find(targets.begin(), targets.end(), c) == targets.end())
                        targets.push_back(c);
                }
                std::sort(targets.begin(), targets.end());
                const uint32_t deg = static_cast<uint32_t>(g.end(v) - g.begin(v));
                int best_delta = 0;
                uint32_t best_to = kNone;
                for (uint32_t to : targets) {
                    if (size[to] + 1 > cap) continue;
                    uint32_t same = 0;  // neighbours of v already in `to`
                    int delta = -1;     // flags[v] is set
                    for (uint64_t e = g.begin(v); e < g.end(v); ++e) {
                        const uint32_t x = g.to[e];
                        const uint32_t ax = a[x];
                        same += ax == to;
                        const uint32_t after = foreign[x] + (ax != to) - (ax != from);
                        delta += (after > 0 ? 1 : 0) - (foreign[x] > 0 ? 1 : 0);
                    }
                    delta += same != deg ? 1 : 0;
                    if (delta < best_delta) {
                        best_delta = delta;
                        best_to = to;
                    }
                }
                if (best_to != kNone) {
                    a[v] = best_to;
                    --size[from];
                    ++size[best_to];
                    uint32_t f = 0;
                    for (uint64_t e = g.begin(v); e < g.end(v); ++e) {
                        const uint32_t x = g.to[e];
                        const uint32_t ax = a[x];
                        f += ax != best_to;
                        foreign[x] = foreign[x] + (ax != best_to) - (ax != from);
                        set_flag(x, foreign[x] > 0);
                    }
                    foreign[v] = f;
                    set_flag(v, f > 0);
                    improved = true;
                }
            }
            if (!improved) break;
        }
    }

    // the finalize lambda (:393-420); returns the candidate's cost and,
    // when `out` is given, the assignment in original id order
    // `out`: the assignment in original ids; `local_out`: in local positions
    uint64_t finalize(std::vector<uint32_t> assign, const std::vector<uint32_t>& hop,
                      std::vector<uint32_t>* out, std::vector<uint32_t>* local_out = nullptr) const {
        PhaseTimer pt{g_ns_finalize};
        const uint64_t n = g.n;
        std::vector<uint64_t> sz(k, 0);
        for (uint64_t u = 0; u < n; ++u)
            if (assign[u] != kNone) ++sz[assign[u]];
        for (uint64_t v = 0; v < n; ++v) {
            const uint32_t u = g.pos[v];
            if (assign[u] != kNone) continue;
            uint32_t best = kNone;
            for (uint32_t c = 0; c < k; ++c)
                if (sz[c] < cap && (best == kNone || sz[c] < sz[best])) best = c;
            assign[u] = best;
            ++sz[best];
        }
        rebalance(assign, hop, sz);
        std::vector<uint8_t> flags = local_boundary(g, assign);
        refine(assign, sz, flags);
        std::vector<uint64_t> bsz(k, 0);
        for (uint64_t u = 0; u < n; ++u)
            if (flags[u]) ++bsz[assign[u]];
        uint64_t cost = 0;
        for (uint32_t c = 0; c < k; ++c) cost += bsz[c] * bsz[c];
        if (out) {
            out->resize(n);
            for (uint64_t v = 0; v < n; ++v) (*out)[v] = assign[g.pos[v]];
        }
        if (local_out) local_out->swap(assign);
        return cost;
    }
};

}  // namespace

std::vector<uint32_t> partition_graph(const Csr& g, uint32_t k, uint64_t seed, unsigned threads) {
    const uint64_t n = g.n;
    if (k < 1) throw ArgError("partition_graph: k must be at least 1");
    if (k > n) throw ArgError("partition_graph: k exceeds vertex count");
    const auto t_start = std::chrono::steady_clock::now();
    const Local L(g);
    Part P{L, k, cap_of(n, k)};

    // --- seed sets for all restarts, in the reference's rng order (:268-329)
    std::mt19937_64 rng(seed);
    std::vector<uint32_t> ids(n);
    std::iota(ids.begin(), ids.end(), 0u);
    SeedSpace S(L);
    if (std::getenv("PSP_PART_PROFILE"))
        std::fprintf(stderr, "[partition] relabelled graph %.3f s\n",
                     std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
    // --- restart chains (:430-444) as a dataflow. finalize() never feeds
    // back into the chain (recenter reads the un-finalized growth), and
    // the seed draws only feed their own restart, so
    //   * restart r's grow/recenter chain starts as soon as its seed set is
    //     drawn (the draws stay sequential on this thread: they share the
    //     rng and the id shuffle);
    //   * every grown (restart, round) state immediately spawns its
    //     finalize(), costs only, on whichever pool thread is free (chain
    //     steps first: they are the critical path);
    // the reference's winner -- the first strict minimum in (restart, round)
    // order -- is the finalized state kept by the pass that produced it.
    constexpr int kRounds = kRecenterRounds + 1;
    struct Grown {
        std::vector<uint32_t> assign, hop;
    };
    std::vector<std::vector<uint32_t>> seed_sets(kRestarts, std::vector<uint32_t>(k));
    std::vector<std::vector<Grown>> grown(kRestarts, std::vector<Grown>(kRounds));
    std::vector<uint64_t> cost(size_t(kRestarts) * kRounds);
    const bool prof = std::getenv("PSP_PART_PROFILE") != nullptr;
    auto lap = [&](const char* what) {
        if (prof)
            std::fprintf(stderr, "[partition] %s %.3f s\n", what,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start)
                             .count());
    };
    // the best finalized state so far: the smallest (cost, restart * rounds
    // + round), i.e. the reference's first strict minimum, kept in local order
    std::mutex win_mu;
    uint64_t win_cost = ~uint64_t(0);
    size_t win_idx = ~size_t(0);
    std::vector<uint32_t> win_local;
    std::function<void(int, int)> chain_step;  // outlives the pool (running tasks call it)
    TaskPool tasks(std::max(1u, threads));
    // the last restarts' chains finish last (their seeds are drawn last):
    // their grows and recenters run on a few threads each (last 2 chains
    // x 4 threads measured best on 16 cores; 4 chains oversubscribe)
    const unsigned par = std::getenv("PSP_PART_SERIAL") ? 1u : std::min(4u, std::max(1u, threads / 4));
    const char* pl = std::getenv("PSP_PART_PAR_LAST");  // A/B: how many of the last chains
    const int par_last = pl ? std::atoi(pl) : 2;
    const bool serial_recenter = std::getenv("PSP_PART_SERIAL_RECENTER") != nullptr;  // A/B
    auto grow_step = [&](int r, std::vector<uint32_t>& as, std::vector<uint32_t>& hp) {
        if (par > 1 && r >= kRestarts - par_last) P.grow_par(seed_sets[r], as, hp, par);
        else P.grow(seed_sets[r], as, hp);
    };
    chain_step = [&](int r, int round) {
        if (round == 0) {
            grow_step(r, grown[r][0].assign, grown[r][0].hop);
        } else {
            seed_sets[r] = par > 1 && r >= kRestarts - par_last && !serial_recenter
                               ? P.recenter_par(grown[r][round - 1].assign, seed_sets[r], par)
                               : P.recenter(grown[r][round - 1].assign, seed_sets[r]);
            grow_step(r, grown[r][round].assign, grown[r][round].hop);
        }
        if (prof && round + 1 == kRounds)
            std::fprintf(stderr, "[partition] chain %d grown %.3f s\n", r,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
        tasks.push(false, [&, r, round] {
            const Grown& gr = grown[r][round];
            std::vector<uint32_t> fin;
            const size_t idx = size_t(r) * kRounds + round;
            const uint64_t c = P.finalize(gr.assign, gr.hop, nullptr, &fin);
            cost[idx] = c;
            std::lock_guard<std::mutex> lk(win_mu);
            if (c < win_cost || (c == win_cost && idx < win_idx)) {
                win_cost = c;
                win_idx = idx;
                win_local.swap(fin);
            }
        });
        if (round + 1 < kRounds) tasks.push(true, [&, r, round] { chain_step(r, round + 1); });
    };
    {  // farthest_seeds (:315-329)
        auto& s = seed_sets[0];
        S.reset();
        s[0] = static_cast<uint32_t>(rng() % n);
        S.relax_from(s[0]);
        for (uint32_t c = 1; c < k; ++c) {
            s[c] = S.farthest();
            S.relax_from(s[c]);
        }
    }
    lap("farthest seeds");
    tasks.push(true, [&] { chain_step(0, 0); });
    for (int r = 1; r < kRestarts; ++r) {  // draw_seeds (:285-306)
        std::vector<uint32_t> s(k);
        S.reset();
        for (uint32_t c = 0; c < k; ++c) {
            const uint64_t m = std::min<uint64_t>(kSeedCandidates, n - c);
            for (uint64_t t = 0; t < m; ++t) {
                const uint64_t j = c + t + static_cast<uint64_t>(rng() % (n - c - t));
                std::swap(ids[c + t], ids[j]);
            }
            uint64_t best = c;
            for (uint64_t t = 1; t < m; ++t) {
                const uint32_t cand = ids[c + t], cur = ids[best];
                const uint32_t dc = S.dist_of(cand), du = S.dist_of(cur);
                if (dc > du || (dc == du && cand < cur)) best = c + t;
            }
            std::swap(ids[c], ids[best]);
            s[c] = ids[c];
            S.relax_from(s[c]);
        }
        seed_sets[r] = std::move(s);
        if (prof)
            std::fprintf(stderr, "[partition] seeds of restart %d drawn %.3f s\n", r,
                         std::chrono::duration<double>(std::chrono::steady_clock::now() - t_start).count());
        tasks.push(true, [&, r] { chain_step(r, 0); });
    }
    lap("seeds drawn");
    tasks.join();  // this thread helps until every chain and finalize is done
    lap("chains + finalize");
    size_t win = 0;
    for (size_t t = 1; t < cost.size(); ++t)
        if (cost[t] < cost[win]) win = t;
    if (win != win_idx) throw std::logic_error("partition_graph: winner bookkeeping mismatch");
    std::vector<uint32_t> assignment(n);
    for (uint64_t v = 0; v < n; ++v) assignment[v] = win_local[L.pos[v]];
    lap("winner assignment");
    if (prof)
        std::fprintf(stderr, "[partition] thread time: grow %.3f s, recenter %.3f s, finalize %.3f s\n",
                     g_ns_grow.load() / 1e9, g_ns_recenter.load() / 1e9, g_ns_finalize.load() / 1e9);
    std::vector<uint64_t> sz(k, 0);
    for (uint32_t c : assignment) ++sz[c];
    for (uint32_t c = 0; c < k; ++c)
        if (sz[c] > P.cap) throw std::logic_error("partition_graph: balance cap violated");
    return assignment;
}

}  // namespace pspg
