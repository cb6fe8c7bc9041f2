// host_graph.hpp — host-side graph plumbing around the GPU hot path.
//
// The reference keeps partitioning and reordering on the host and so do we
// (BASELINE.json north_star): these routines reproduce the reference's
// id-space conventions exactly, because component assignment and the
// boundary-first order decide every table entry's position.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pspg {

struct GraphError : std::runtime_error {   // psp::GraphInvariantError
    using std::runtime_error::runtime_error;
};
struct ArgError : std::invalid_argument {  // std::invalid_argument
    using std::invalid_argument::invalid_argument;
};

// Sorted symmetric CSR (psp::Graph, include/psp/graph.hpp:42-76).
struct Csr {
    uint64_t n = 0;
    std::vector<uint64_t> off;  // n+1
    std::vector<uint32_t> to;   // 2m, sorted per vertex
    std::vector<double> w;      // 2m
    uint64_t degree(uint32_t v) const { return off[v + 1] - off[v]; }
};

// psp::Graph(n, edges) (src/graph.cpp:19-56): validates ids, self-loops,
// finite non-negative weights and duplicates, in the reference's order.
Csr build_csr(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev, const double* ew);

// compute_boundary (src/partition.cpp:196-212)
std::vector<uint8_t> compute_boundary(const Csr& g, const std::vector<uint32_t>& assignment);

// compute_reorder_permutation (src/partition.cpp:214-240): stable
// boundary-first counting sort, old id -> new id.
std::vector<uint32_t> reorder_permutation(uint32_t k, const std::vector<uint32_t>& assignment,
                                          const std::vector<uint8_t>& flags);

// The partitioned + reordered view the device build consumes.
struct Reordered {
    uint64_t n = 0;
    uint32_t k = 0;
    std::vector<uint32_t> perm, inv;         // original <-> reordered
    std::vector<uint32_t> assign;            // reordered -> component
    std::vector<uint8_t> flags;              // reordered boundary flags
    std::vector<uint32_t> comp_off, bnd_off; // k+1 each
    Csr g;                                   // reordered graph (sorted)
    uint64_t b() const { return bnd_off[k]; }
};

// reorder_vertices (src/partition.cpp:452-481) given an assignment in
// original ids; also builds component / boundary offsets
// (src/oracle.cpp:45-54, :80-89).
Reordered reorder(const Csr& g, uint32_t k, const std::vector<uint32_t>& assignment);

// partition_graph (src/partition.cpp:259-450), restated in partition.cpp.
std::vector<uint32_t> partition_graph(const Csr& g, uint32_t k, uint64_t seed, unsigned threads);

// generators (src/generators.cpp:50-93)
// Minimum spanning forest under edge keys (Kruskal: keys sorted stably, ties
// by edge index; union-find). in_tree[e] = 1 for forest edges. With distinct
// keys the forest is unique, so it equals scipy's minimum_spanning_tree.
void min_spanning_forest(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                         const double* key, uint8_t* in_tree);

void generate_grid(int kind, uint64_t rows, uint64_t cols, bool unit, double lo, double hi,
                   uint64_t seed, std::vector<uint32_t>& eu, std::vector<uint32_t>& ev,
                   std::vector<double>& ew);

// Delaunay edges of points in [0,1)^2 on the 2^-53 grid (delaunay.cpp)
void delaunay_edges(uint64_t n, const double* xy, std::vector<uint32_t>& eu,
                    std::vector<uint32_t>& ev);

}  // namespace pspg
