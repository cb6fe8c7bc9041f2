// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A thin extern "C" wrapper over the UNMODIFIED reference library (`psp`,
// compiled straight from /root/reference/proj/src/*.cpp by oracle/Makefile
// into oracle/_ref/libpspref.so). Python tests and bench.py's CPU arm reach
// the reference through these entry points with ctypes; nothing here
// re-implements reference behaviour, it only marshals plain arrays in and out.
//
// Reference interfaces wrapped (paths under /root/reference/proj):
//   generate_grid / generate_triangulated_grid   include/psp/generators.hpp:24-30
//   Graph(n, edges)                              include/psp/graph.hpp:50
//   partition_graph / reorder_vertices           include/psp/partition.hpp:42,57
//   build_oracle + BuildStats                    include/psp/oracle.hpp:29-37,85-86
//   build_boundary_graph / boundary_apsp         include/psp/oracle.hpp:90-96
//   apsp_dense / dijkstra_sssp                   include/psp/shortest_paths.hpp:39-43
//   query / batch_query                          include/psp/query.hpp:36-46

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <random>
#include <sstream>
#include <string>
#include <thread>
#include <utility>
#include <vector>

#include "psp/cluster.hpp"
#include "psp/generators.hpp"
#include "psp/graph.hpp"
#include "psp/errors.hpp"
#include "psp/graph_io.hpp"
#include "psp/oracle.hpp"
#include "psp/oracle_io.hpp"
#include "psp/partition.hpp"
#include "psp/placement.hpp"
#include "psp/query.hpp"
#include "psp/shortest_paths.hpp"
#include "support/reference.hpp"  // ref::random_pairs (tests/support/reference.hpp:80-91)

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    } catch (...) {
        g_err = "unknown C++ exception";
        return 1;
    }
}

struct RefGraph {
    psp::Graph g;
};

struct RefOracle {
    psp::Oracle o;
    psp::BuildStats stats;
};

// Parallel task pool of `workers` threads over [0, count) (the reference's
// parallel_for, include/psp/parallel.hpp:15-47, is header-only and
// internal; this is the same static fan-out with dynamic pickup).
template <typename F>
void pool_for(std::size_t count, uint32_t workers, F&& f) {
    std::atomic<std::size_t> next{0};
    std::vector<std::thread> pool;
    for (uint32_t w = 0; w < std::max<uint32_t>(workers, 1); ++w) {
        pool.emplace_back([&] {
            for (;;) {
                const std::size_t i = next.fetch_add(1);
                if (i >= count) return;
                f(i);
            }
        });
    }
    for (auto& t : pool) t.join();
}

// Seeded choice of `n_comps` distinct components (partial Fisher-Yates).
std::vector<uint32_t> sample_components(uint32_t k, uint32_t n_comps, uint64_t seed) {
    std::vector<uint32_t> ids(k);
    for (uint32_t c = 0; c < k; ++c) ids[c] = c;
    std::mt19937_64 rng(seed);
    n_comps = std::min(n_comps, k);
    for (uint32_t i = 0; i < n_comps; ++i) std::swap(ids[i], ids[i + rng() % (k - i)]);
    ids.resize(n_comps);
    std::sort(ids.begin(), ids.end());
    return ids;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

void ref_graph_free(void* g) { delete static_cast<RefGraph*>(g); }
void ref_oracle_free(void* o) { delete static_cast<RefOracle*>(o); }

// kind: 0 grid, 1 triangulated grid. unit != 0 selects WeightModel::unit().
int ref_generate(int kind, uint64_t rows, uint64_t cols, int unit, double lo, double hi,
                 uint64_t seed, void** out) {
    return guarded([&] {
        const psp::WeightModel wm = unit ? psp::WeightModel::unit() : psp::WeightModel::uniform(lo, hi);
        auto* rg = new RefGraph;
        rg->g = kind == 0 ? psp::generate_grid(rows, cols, wm, seed)
                          : psp::generate_triangulated_grid(rows, cols, wm, seed);
        *out = rg;
    });
}

int ref_graph_from_edges(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                         const double* ew, void** out) {
    return guarded([&] {
        std::vector<psp::Edge> edges(m);
        for (uint64_t i = 0; i < m; ++i) edges[i] = {eu[i], ev[i], ew[i]};
        auto* rg = new RefGraph;
        rg->g = psp::Graph(n, edges);
        *out = rg;
    });
}

uint64_t ref_graph_n(const void* g) { return static_cast<const RefGraph*>(g)->g.num_vertices(); }
uint64_t ref_graph_m(const void* g) { return static_cast<const RefGraph*>(g)->g.num_edges(); }

// Edges with u < v in lexicographic order (Graph::edge_list, graph.hpp:66).
int ref_graph_edges(const void* g, uint32_t* eu, uint32_t* ev, double* ew) {
    return guarded([&] {
        const auto el = static_cast<const RefGraph*>(g)->g.edge_list();
        for (size_t i = 0; i < el.size(); ++i) {
            eu[i] = el[i].u;
            ev[i] = el[i].v;
            ew[i] = el[i].weight;
        }
    });
}

int ref_partition(const void* g, uint32_t k, uint64_t seed, uint32_t* assignment,
                  double* elapsed_ms) {
    return guarded([&] {
        auto t0 = std::chrono::steady_clock::now();
        psp::Partition p = psp::partition_graph(static_cast<const RefGraph*>(g)->g, k, seed);
        if (elapsed_ms)
            *elapsed_ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        std::memcpy(assignment, p.assignment.data(), p.assignment.size() * sizeof(uint32_t));
    });
}

int ref_apsp_dense(const void* g, uint64_t block, double* out) {
    return guarded([&] {
        psp::Matrix m = psp::apsp_dense(static_cast<const RefGraph*>(g)->g, block);
        std::memcpy(out, m.data().data(), m.data().size() * sizeof(double));
    });
}

int ref_dijkstra(const void* g, uint32_t src, double* out) {
    return guarded([&] {
        auto d = psp::dijkstra_sssp(static_cast<const RefGraph*>(g)->g, src);
        std::memcpy(out, d.data(), d.size() * sizeof(double));
    });
}

// stats: partition_ms, component_apsp_ms, boundary_ms, boundary_total,
// bg_edges, stored_entries, peak_table_entries_per_worker (7 doubles).
int ref_build_oracle(const void* g, uint32_t k, uint32_t workers, uint64_t seed, double* stats,
                     void** out) {
    return guarded([&] {
        auto* ro = new RefOracle;
        try {
            ro->o = psp::build_oracle(static_cast<const RefGraph*>(g)->g, k, workers, seed,
                                      &ro->stats);
        } catch (...) {
            delete ro;
            throw;
        }
        if (stats) {
            stats[0] = ro->stats.partition_ms;
            stats[1] = ro->stats.component_apsp_ms;
            stats[2] = ro->stats.boundary_ms;
            stats[3] = static_cast<double>(ro->stats.boundary_total);
            stats[4] = static_cast<double>(ro->stats.bg_edges);
            stats[5] = static_cast<double>(ro->stats.stored_entries);
            stats[6] = static_cast<double>(ro->stats.peak_table_entries_per_worker);
        }
        *out = ro;
    });
}

// info: n, k, b
void ref_oracle_info(const void* o, uint64_t* info) {
    const psp::Oracle& r = static_cast<const RefOracle*>(o)->o;
    info[0] = r.n;
    info[1] = r.k;
    info[2] = r.b();
}

// permutation (n), reordered assignment (n), component_offset (k+1),
// boundary_offset (k+1), boundary_vertex (b), boundary_flags (n, reordered).
void ref_oracle_ids(const void* o, uint32_t* perm, uint32_t* assign, uint64_t* comp_off,
                    uint64_t* bnd_off, uint32_t* bvert, uint8_t* flags) {
    const psp::Oracle& r = static_cast<const RefOracle*>(o)->o;
    for (size_t i = 0; i < r.n; ++i) {
        perm[i] = r.permutation[i];
        assign[i] = r.partition.assignment[i];
        flags[i] = r.partition.boundary_flags[i];
    }
    for (size_t c = 0; c <= r.k; ++c) {
        comp_off[c] = r.component_offset[c];
        bnd_off[c] = r.boundary_offset[c];
    }
    for (size_t i = 0; i < r.b(); ++i) bvert[i] = r.boundary_vertex[i];
}

void ref_oracle_component(const void* o, uint32_t c, double* out) {
    const psp::Matrix& m = static_cast<const RefOracle*>(o)->o.component_tables[c];
    std::memcpy(out, m.data().data(), m.data().size() * sizeof(double));
}

void ref_oracle_boundary_rows(const void* o, uint32_t c, double* out) {
    const psp::Matrix& m = static_cast<const RefOracle*>(o)->o.boundary_tables[c];
    std::memcpy(out, m.data().data(), m.data().size() * sizeof(double));
}

// dist (count doubles); ops (count u64, minplus_ops) may be null.
int ref_batch_query(const void* o, uint64_t count, const uint32_t* v1, const uint32_t* v2,
                    uint32_t workers, double* dist, uint64_t* ops, double* elapsed_ms) {
    return guarded([&] {
        std::vector<std::pair<psp::VertexId, psp::VertexId>> pairs(count);
        for (uint64_t i = 0; i < count; ++i) pairs[i] = {v1[i], v2[i]};
        auto t0 = std::chrono::steady_clock::now();
        auto res = psp::batch_query(static_cast<const RefOracle*>(o)->o, pairs, workers);
        if (elapsed_ms)
            *elapsed_ms = std::chrono::duration<double, std::milli>(
                              std::chrono::steady_clock::now() - t0).count();
        for (uint64_t i = 0; i < count; ++i) {
            dist[i] = res[i].distance;
            if (ops) ops[i] = res[i].stats.minplus_ops;
        }
    });
}

// Phase-3 sampling for configurations whose full f64 boundary tables exceed
// host RAM: partition + reorder + component APSP in full,
// build the boundary graph, then time `rows` Dijkstra runs on it.
// times: partition_ms, component_apsp_ms, bg_build_ms, sampled_dijkstra_ms
// info: b, bg_edges
int ref_sampled_build(const void* g, uint32_t k, uint32_t workers, uint64_t seed, uint32_t rows,
                      uint64_t sample_seed, double* times, uint64_t* info) {
    return guarded([&] {
        using Clock = std::chrono::steady_clock;
        auto ms = [](Clock::time_point t) {
            return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
        };
        const psp::Graph& gg = static_cast<const RefGraph*>(g)->g;
        auto t0 = Clock::now();
        psp::Partition op = psp::partition_graph(gg, k, seed);
        auto [rg, part] = psp::reorder_vertices(gg, op);
        times[0] = ms(t0);
        std::vector<std::size_t> off(k + 1, 0);
        for (uint32_t c = 0; c < k; ++c) off[c + 1] = off[c] + part.component_members[c].size();
        // component tables via the public apsp_dense on each induced range
        t0 = Clock::now();
        std::vector<psp::Matrix> tables(k);
        std::vector<std::thread> pool;
        std::atomic<uint32_t> next{0};
        for (uint32_t w = 0; w < workers; ++w) {
            pool.emplace_back([&] {
                for (;;) {
                    uint32_t c = next.fetch_add(1);
                    if (c >= k) return;
                    const std::size_t base = off[c], size = off[c + 1] - off[c];
                    std::vector<psp::Edge> edges;
                    for (std::size_t i = 0; i < size; ++i) {
                        for (const psp::Neighbor& nb : rg.neighbors(static_cast<psp::VertexId>(base + i))) {
                            if (nb.to >= base && nb.to < base + size && nb.to > base + i)
                                edges.push_back({static_cast<psp::VertexId>(i),
                                                 static_cast<psp::VertexId>(nb.to - base), nb.weight});
                        }
                    }
                    tables[c] = psp::apsp_dense(psp::Graph(size, edges));
                }
            });
        }
        for (auto& t : pool) t.join();
        times[1] = ms(t0);
        t0 = Clock::now();
        psp::BoundaryGraph bg = psp::build_boundary_graph(rg, part, tables);
        times[2] = ms(t0);
        info[0] = bg.global_of.size();
        info[1] = bg.graph.num_edges();
        std::mt19937_64 rng(sample_seed);
        const std::size_t b = bg.global_of.size();
        t0 = Clock::now();
        for (uint32_t r = 0; r < rows && b > 0; ++r) {
            auto d = psp::dijkstra_sssp(bg.graph, static_cast<psp::VertexId>(rng() % b));
            (void)d;
        }
        times[3] = ms(t0);
    });
}

// The reference's build_oracle (src/oracle.cpp:144-194) for configurations
// whose f64 boundary tables exceed host RAM (cfg3 needs
// 145.8 GB): Phase 1 (partition_graph + reorder_vertices) and Phase 2
// (apsp_dense per component on `workers` threads) run in FULL; Phase 3
// builds the boundary graph in full (build_boundary_graph) and runs the
// reference's dijkstra_sssp rows (exactly boundary_apsp's per-row work,
// oracle.cpp:127-142) only for the boundary vertices of `n_comps` seeded
// components, fanned out over `workers` threads. The result is a real
// psp::Oracle on which the reference's own query/batch_query answer every
// pair whose source lies in a sampled component (query reads only
// boundary_tables[c1], src/query.cpp:29-46).
// times: partition_ms, component_apsp_ms, bg_build_ms, sampled_rows_ms
// info: b, bg_edges, rows computed; comps_out: the sampled components
int ref_sampled_oracle(const void* g, uint32_t k, uint32_t workers, uint64_t seed,
                       uint32_t n_comps, uint64_t sample_seed, double* times, uint64_t* info,
                       uint32_t* comps_out, void** out) {
    return guarded([&] {
        using Clock = std::chrono::steady_clock;
        auto ms = [](Clock::time_point t) {
            return std::chrono::duration<double, std::milli>(Clock::now() - t).count();
        };
        const psp::Graph& gg = static_cast<const RefGraph*>(g)->g;
        auto ro = std::make_unique<RefOracle>();
        psp::Oracle& o = ro->o;
        auto t0 = Clock::now();
        psp::Partition op = psp::partition_graph(gg, k, seed);
        auto [rg, part] = psp::reorder_vertices(gg, op);
        times[0] = ms(t0);
        o.n = gg.num_vertices();
        o.k = k;
        o.permutation = std::move(op.permutation);
        o.inverse_permutation = std::move(op.inverse_permutation);
        o.component_offset.assign(k + 1, 0);
        for (uint32_t c = 0; c < k; ++c)
            o.component_offset[c + 1] = o.component_offset[c] + part.component_members[c].size();
        t0 = Clock::now();
        o.component_tables.resize(k);
        pool_for(k, std::min(workers, k), [&](std::size_t c) {
            const std::size_t base = o.component_offset[c];
            const std::size_t size = o.component_offset[c + 1] - base;
            std::vector<psp::Edge> edges;
            for (std::size_t i = 0; i < size; ++i)
                for (const psp::Neighbor& nb : rg.neighbors(static_cast<psp::VertexId>(base + i)))
                    if (nb.to >= base && nb.to < base + size && nb.to > base + i)
                        edges.push_back({static_cast<psp::VertexId>(i),
                                         static_cast<psp::VertexId>(nb.to - base), nb.weight});
            o.component_tables[c] = psp::apsp_dense(psp::Graph(size, edges));
        });
        times[1] = ms(t0);
        t0 = Clock::now();
        psp::BoundaryGraph bg = psp::build_boundary_graph(rg, part, o.component_tables);
        times[2] = ms(t0);
        o.boundary_vertex = bg.global_of;
        o.boundary_offset = bg.component_offset;
        const std::size_t b = bg.global_of.size();
        info[0] = b;
        info[1] = bg.graph.num_edges();
        const std::vector<uint32_t> comps = sample_components(k, n_comps, sample_seed);
        std::vector<std::pair<uint32_t, std::size_t>> rows;  // (component, boundary id)
        o.boundary_tables.resize(k);
        for (uint32_t c : comps) {
            const std::size_t lo = bg.component_offset[c], hi = bg.component_offset[c + 1];
            o.boundary_tables[c] = psp::Matrix(hi - lo, b, psp::kUnreachable);
            for (std::size_t i = lo; i < hi; ++i) rows.emplace_back(c, i);
        }
        t0 = Clock::now();
        pool_for(rows.size(), workers, [&](std::size_t r) {
            const auto [c, i] = rows[r];
            std::vector<double> row = psp::dijkstra_sssp(bg.graph, static_cast<psp::VertexId>(i));
            std::copy(row.begin(), row.end(),
                      o.boundary_tables[c].row(i - bg.component_offset[c]));
        });
        times[3] = ms(t0);
        info[2] = rows.size();
        for (std::size_t i = 0; i < comps.size(); ++i) comps_out[i] = comps[i];
        o.partition = std::move(part);
        o.placement = psp::place_components(k, 1);
        *out = ro.release();
    });
}

// A psp::Oracle assembled from plain arrays (e.g. tables exported from the
// GPU build, bit-identical to the reference's): the reference's own
// batch_query then runs on it. bt[c] may be null (component not sampled:
// queries must not start there). assign/flags are in the reordered space.
int ref_oracle_assemble(uint64_t n, uint32_t k, const uint32_t* perm, const uint32_t* assign,
                        const uint8_t* flags, const uint64_t* comp_off, const uint64_t* bnd_off,
                        const uint32_t* bvert, const double* const* ct, const double* const* bt,
                        void** out) {
    return guarded([&] {
        auto ro = std::make_unique<RefOracle>();
        psp::Oracle& o = ro->o;
        o.n = n;
        o.k = k;
        o.permutation.assign(perm, perm + n);
        o.inverse_permutation.resize(n);
        for (uint64_t v = 0; v < n; ++v) o.inverse_permutation[perm[v]] = static_cast<uint32_t>(v);
        o.component_offset.assign(comp_off, comp_off + k + 1);
        o.boundary_offset.assign(bnd_off, bnd_off + k + 1);
        const uint64_t b = bnd_off[k];
        o.boundary_vertex.assign(bvert, bvert + b);
        o.partition.k = k;
        o.partition.assignment.assign(assign, assign + n);
        o.partition.boundary_flags.assign(flags, flags + n);
        o.partition.component_members.assign(k, {});
        for (uint64_t v = 0; v < n; ++v)
            o.partition.component_members[assign[v]].push_back(static_cast<uint32_t>(v));
        o.partition.permutation.resize(n);
        o.partition.inverse_permutation.resize(n);
        for (uint64_t v = 0; v < n; ++v)
            o.partition.permutation[v] = o.partition.inverse_permutation[v] = static_cast<uint32_t>(v);
        o.component_tables.resize(k);
        o.boundary_tables.resize(k);
        for (uint32_t c = 0; c < k; ++c) {
            const uint64_t s = comp_off[c + 1] - comp_off[c], bc = bnd_off[c + 1] - bnd_off[c];
            if (ct[c]) {  // NULL: component not sampled (queries never touch it)
                o.component_tables[c] = psp::Matrix(s, s, psp::kUnreachable);
                std::memcpy(o.component_tables[c].data().data(), ct[c], s * s * sizeof(double));
            }
            if (bt[c]) {
                o.boundary_tables[c] = psp::Matrix(bc, b, psp::kUnreachable);
                std::memcpy(o.boundary_tables[c].data().data(), bt[c], bc * b * sizeof(double));
            }
        }
        o.placement = psp::place_components(k, 1);
        *out = ro.release();
    });
}

// save_oracle / load_oracle (include/psp/oracle_io.hpp:31-32)
int ref_save_oracle(const void* o, const char* path) {
    return guarded([&] { psp::save_oracle(static_cast<const RefOracle*>(o)->o, path); });
}

int ref_load_oracle(const char* path, void** out) {
    return guarded([&] {
        auto* ro = new RefOracle;
        try {
            ro->o = psp::load_oracle(path);
        } catch (...) {
            delete ro;
            throw;
        }
        *out = ro;
    });
}

// --- graph text (include/psp/graph_io.hpp) ---
// kind: 0 ok, 1 ParseError (line set), 2 GraphInvariantError, 3 IoError, 4 other
int ref_read_graph(const char* text, uint64_t len, int format, const char* name, void** out,
                   int* kind, uint64_t* line) {
    *kind = 0;
    *line = 0;
    try {
        std::istringstream in(std::string(text, len));
        auto* rg = new RefGraph{psp::read_graph(
            in, format == 1 ? psp::FileFormat::DimacsGr : psp::FileFormat::EdgeList, name)};
        *out = rg;
        return 0;
    } catch (const psp::ParseError& e) {
        g_err = e.what();
        *kind = 1;
        *line = e.line();
    } catch (const psp::GraphInvariantError& e) {
        g_err = e.what();
        *kind = 2;
    } catch (const psp::IoError& e) {
        g_err = e.what();
        *kind = 3;
    } catch (const std::exception& e) {
        g_err = e.what();
        *kind = 4;
    }
    return 1;
}

// write_graph into buf (cap bytes); *len = full length
int ref_write_graph(const void* g, int format, char* buf, uint64_t cap, uint64_t* len) {
    return guarded([&] {
        std::ostringstream out;
        psp::write_graph(static_cast<const RefGraph*>(g)->g, out,
                         format == 1 ? psp::FileFormat::DimacsGr : psp::FileFormat::EdgeList);
        const std::string t = out.str();
        *len = t.size();
        if (buf) std::memcpy(buf, t.data(), std::min<uint64_t>(cap, t.size()));
    });
}

// --- cluster layer (include/psp/placement.hpp, include/psp/cluster.hpp) ---
static psp::PlacementPolicy policy_of(int p) {
    return p == 1 ? psp::PlacementPolicy::PairsPerGpu : psp::PlacementPolicy::RoundRobin;
}

int ref_place_components(uint32_t k, uint32_t p, int policy, uint32_t* owner) {
    return guarded([&] {
        const psp::Placement pl = psp::place_components(k, p, policy_of(policy));
        std::copy(pl.owner.begin(), pl.owner.end(), owner);
    });
}

// out: distance, minplus_ops, b1, b2, same, transfer_entries, executed_on,
// column_owner, has_transfer, rec.src, rec.dst, rec.entries, rec.bytes,
// overlap_cost, serial_cost
int ref_routed_query(const void* o, uint32_t p, int policy, uint32_t v1, uint32_t v2,
                     uint64_t qid, double* out) {
    return guarded([&] {
        const psp::Oracle& orc = static_cast<const RefOracle*>(o)->o;
        const psp::Placement pl = psp::place_components(orc.k, p, policy_of(policy));
        const psp::RoutedQueryResult r = psp::routed_query(orc, pl, v1, v2, qid);
        const auto& st = r.result.stats;
        double v[15] = {r.result.distance, double(st.minplus_ops), double(st.boundary_size_1),
                        double(st.boundary_size_2), st.same_component ? 1.0 : 0.0,
                        double(st.transfer_entries), double(r.executed_on), double(r.column_owner),
                        r.transfer ? 1.0 : 0.0, r.transfer ? double(r.transfer->src_worker) : 0.0,
                        r.transfer ? double(r.transfer->dst_worker) : 0.0,
                        r.transfer ? double(r.transfer->entries) : 0.0,
                        r.transfer ? double(r.transfer->bytes) : 0.0, r.overlap_cost, r.serial_cost};
        std::memcpy(out, v, sizeof(v));
    });
}

// ClusterSim::run_batch; ledger rows (query_id, src, dst, entries, bytes)
// into rec (count * 5 u64 max), their number into *nrec.
int ref_cluster_run_batch(const void* o, uint32_t p, int policy, uint64_t count,
                          const uint32_t* v1, const uint32_t* v2, double* dist, uint64_t* rec,
                          uint64_t* nrec) {
    return guarded([&] {
        const psp::Oracle& orc = static_cast<const RefOracle*>(o)->o;
        psp::ClusterSim sim(orc, psp::place_components(orc.k, p, policy_of(policy)));
        std::vector<std::pair<psp::VertexId, psp::VertexId>> pairs(count);
        for (uint64_t i = 0; i < count; ++i) pairs[i] = {v1[i], v2[i]};
        const auto res = sim.run_batch(pairs);
        for (uint64_t i = 0; i < count; ++i) dist[i] = res[i].distance;
        const auto recs = sim.ledger().records();
        *nrec = recs.size();
        for (size_t i = 0; i < recs.size(); ++i) {
            rec[5 * i + 0] = recs[i].query_id;
            rec[5 * i + 1] = recs[i].src_worker;
            rec[5 * i + 2] = recs[i].dst_worker;
            rec[5 * i + 3] = recs[i].entries;
            rec[5 * i + 4] = recs[i].bytes;
        }
    });
}

int ref_simulate_build_schedule(uint32_t k, uint32_t p, const double* costs, int policy,
                                double* worker_cost, double* makespan, double* mean_load) {
    return guarded([&] {
        const psp::ScheduleProfile prof = psp::simulate_build_schedule(
            k, p, std::span<const double>(costs, k), policy_of(policy));
        std::copy(prof.worker_cost.begin(), prof.worker_cost.end(), worker_cost);
        *makespan = prof.makespan;
        *mean_load = prof.mean_load;
    });
}

void ref_random_pairs(uint64_t n, uint64_t count, uint64_t seed, uint32_t* v1, uint32_t* v2) {
    const auto pairs = ref::random_pairs(n, count, seed);
    for (uint64_t i = 0; i < count; ++i) {
        v1[i] = pairs[i].first;
        v2[i] = pairs[i].second;
    }
}

}  // extern "C"
