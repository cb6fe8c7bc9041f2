/* TEST INFRASTRUCTURE ONLY — the CPU checker for the GPU hot path.
 *
 * Plain-C restatement of the reference's preprocessing (Phase 2 + Phase 3)
 * and query algorithm, in the reference's own f64 arithmetic. It shares no
 * code with the reference; every function cites the reference file:line it
 * follows (paths under /root/reference/proj). Only tests/, the smoke() check
 * in __graft_entry__.py and bench.py's cpu_baseline leg may load it; the
 * product library never does.
 *
 * Parity of this restatement is PINNED against (a) the reference library
 * itself, compiled unmodified into oracle/_ref/libpspref.so (see Makefile),
 * and (b) the golden vectors spelled out in the reference tests
 * (tests/test_oracle.cpp:28-79, :90-112; tests/test_query.cpp:30-89, :155-164;
 * tests/test_shortest_paths.cpp:14-20, :85-105) — tests/test_oracle_pin.py.
 *
 * All graph inputs are in the REORDERED id space (psp::reorder_vertices,
 * src/partition.cpp:452-481): component c owns reordered ids
 * [comp_off[c], comp_off[c+1]) with its boundary vertices first.
 */
#ifndef PSP_ORACLE_H
#define PSP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pso_oracle pso_oracle;

/* apsp_dense (src/shortest_paths.cpp:128-172): blocked Floyd-Warshall in f64
 * over a CSR graph, output n*n row-major. Returns 0, or -1 if block == 0. */
int pso_apsp_dense(uint64_t n, const uint64_t* off, const uint32_t* to, const double* w,
                   uint64_t block, double* out);

/* dijkstra_sssp (src/shortest_paths.cpp:84-105) with the indexed binary heap
 * of src/shortest_paths.cpp:13-80. */
void pso_dijkstra(uint64_t n, const uint64_t* off, const uint32_t* to, const double* w,
                  uint32_t source, double* dist);

/* min_plus_combine (src/shortest_paths.cpp:174-179). */
double pso_min_plus_combine(uint64_t len, const double* a, const double* b);

/* build_oracle Phase 2 + Phase 3 (src/oracle.cpp:162-177) on an already
 * partitioned + reordered graph. perm: original -> reordered (n entries),
 * assign: reordered vertex -> component, flags: reordered boundary flags.
 * Returns NULL on allocation failure. */
pso_oracle* pso_build(uint64_t n, const uint64_t* off, const uint32_t* to, const double* w,
                      uint32_t k, const uint32_t* perm, const uint32_t* assign,
                      const uint8_t* flags);
void pso_free(pso_oracle* o);

/* n, k, b, bg_edges, stored_entries */
void pso_info(const pso_oracle* o, uint64_t* info);
/* component_offset (k+1), boundary_offset (k+1) */
void pso_offsets(const pso_oracle* o, uint64_t* comp_off, uint64_t* bnd_off);
/* |C|x|C| table / |B(C)|x b rows (views, owned by the oracle). */
const double* pso_component_table(const pso_oracle* o, uint32_t c);
const double* pso_boundary_rows(const pso_oracle* o, uint32_t c);

/* query (src/query.cpp:85-88): distance and minplus_ops for original ids.
 * Returns 0, or -1 if an id is out of range (reference throws). */
int pso_query(const pso_oracle* o, uint32_t v1, uint32_t v2, double* dist, uint64_t* ops);
/* batch_query (src/query.cpp:106-114), sequential. Returns index+1 of the
 * first bad pair, or 0. */
uint64_t pso_batch_query(const pso_oracle* o, uint64_t count, const uint32_t* v1,
                         const uint32_t* v2, double* dist, uint64_t* ops);

#ifdef __cplusplus
}
#endif

#endif
