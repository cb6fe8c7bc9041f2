// TEST INFRASTRUCTURE: the shim's device-oracle registry
// (integration/psp_gpu_shim.cpp) against stale-table reuse.
//
// Built by oracle/Makefile against the reference library with its hot-path
// symbols routed to the GPU shim (like the reference's own suites), run from
// tests/test_reference_suites.py on a B200. Ground truth is the reference's
// dijkstra_sssp (src/shortest_paths.cpp:13-105) on the original graph.
//
//   1. an Oracle built through the shim answers correctly;
//   2. it is destroyed and an Oracle of the SAME shape for a DIFFERENT graph
//      is read back with load_oracle (not built by the shim, so never
//      registered) - typically into the same heap storage: its queries must
//      come from its own tables, not the destroyed oracle's device copy;
//   3. more oracles than the registry holds stay correct (eviction);
//   4. copies answer like their source.
#include <cstdio>
#include <filesystem>
#include <string>
#include <vector>

#include "psp/generators.hpp"
#include "psp/oracle.hpp"
#include "psp/oracle_io.hpp"
#include "psp/query.hpp"
#include "psp/shortest_paths.hpp"

using namespace psp;

static int failures = 0;

static std::size_t mismatches(const Oracle& o, const Graph& g) {
    std::size_t bad = 0;
    const std::size_t n = g.num_vertices();
    for (VertexId u = 0; u < n; ++u) {
        const std::vector<double> d = dijkstra_sssp(g, u);
        std::vector<std::pair<VertexId, VertexId>> pairs;
        for (VertexId v = 0; v < n; ++v) pairs.emplace_back(u, v);
        const auto res = batch_query(o, pairs, 1);
        for (VertexId v = 0; v < n; ++v) bad += res[v].distance != d[v];
        bad += query(o, u, (u * 7) % n).distance != d[(u * 7) % n];
    }
    return bad;
}

static void expect(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    failures += ok ? 0 : 1;
}

int main() {
    namespace fs = std::filesystem;
    const fs::path file = fs::temp_directory_path() / "psp_shim_registry_b.bin";
    const Graph ga = generate_grid(12, 12, WeightModel::uniform(1, 8), 7);
    const Graph gb = generate_grid(12, 12, WeightModel::uniform(1, 8), 8);
    {
        const Oracle xb = build_oracle(gb, 6, 1, 0);
        save_oracle(xb, file.string());
    }
    const void* addr_a = nullptr;
    {
        const Oracle a = build_oracle(ga, 6, 1, 0);
        addr_a = a.component_tables.data();
        expect(mismatches(a, ga) == 0, "shim-built oracle answers its own graph");
    }
    // same n, k and table shapes as `a`, different distances
    const Oracle b = load_oracle(file.string());
    std::printf("info: loaded oracle reuses the destroyed oracle's storage: %s\n",
                b.component_tables.data() == addr_a ? "yes" : "no");
    expect(b.n == ga.num_vertices() && b.k == 6, "loaded oracle has the destroyed one's shape");
    expect(mismatches(b, gb) == 0, "loaded oracle answers from its own tables");
    {
        std::vector<Oracle> many;
        std::vector<Graph> graphs;
        for (int i = 0; i < 20; ++i) {
            graphs.push_back(generate_grid(6 + i % 3, 7, WeightModel::uniform(1, 4), 100 + i));
            many.push_back(build_oracle(graphs.back(), 3, 1, 0));
        }
        std::size_t bad = 0;
        for (int round = 0; round < 2; ++round)
            for (int i = 0; i < 20; ++i) bad += mismatches(many[i], graphs[i]);
        expect(bad == 0, "20 live oracles (more than the registry holds) stay correct");
    }
    const Oracle c = b;  // a copy: different storage, same content
    expect(mismatches(c, gb) == 0, "a copy answers like its source");
    fs::remove(file);
    std::printf("%d failed\n", failures);
    return failures;
}
