/* psp_gpu.h — C-ABI of the B200-native preprocessing + query engine for the
 * partitioned planar shortest-path oracle (Chapuis & Djidjev, arXiv 1503.07192).
 *
 * This is the drop-in boundary for the hot path of the reference library
 * `psp` (/root/reference/proj). Every entry point names the reference
 * interface it replaces (paths relative to /root/reference/proj). Signatures
 * use only plain pointers and sizes; a C++ shim restores the reference's
 * types (psp::Graph, psp::Oracle, psp::Matrix, exceptions) on top — see
 * INTEGRATION.md.
 *
 * Semantics shared by all entry points
 *  - Distances cross the boundary as IEEE f64 exactly like the reference
 *    (include/psp/graph.hpp:14): unreachable = +infinity.
 *  - Inside the library distances are u32 (exact: integral weights, or dyadic
 *    weights w*2^q integral, "fixed point") or f32 (tolerance path, relative
 *    error <= 1e-5). PSP_VALUE_AUTO picks u32 whenever it is exact.
 *  - Errors: every call returns a psp_status; psp_gpu_last_error() gives a
 *    thread-local message. The shim maps PSP_EINVAL / PSP_EOVERFLOW to
 *    std::invalid_argument, PSP_EGRAPH to psp::GraphInvariantError and the
 *    rest to std::runtime_error (reference conventions, include/psp/errors.hpp).
 *  - There is no CPU fallback: without a usable CUDA device every compute
 *    entry point fails with PSP_ECUDA.
 */
#ifndef PSP_GPU_H
#define PSP_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PSP_GPU_ABI_VERSION 5

typedef enum psp_status {
    PSP_OK = 0,
    PSP_EINVAL = 1,     /* bad argument (reference: std::invalid_argument)      */
    PSP_ENOMEM = 2,     /* device or host allocation failed                      */
    PSP_ECUDA = 3,      /* CUDA runtime error / no device                        */
    PSP_ENCCL = 4,      /* NCCL error (multi-GPU)                                */
    PSP_EOVERFLOW = 5,  /* u32 requested but weights not representable exactly   */
    PSP_EGRAPH = 6,     /* graph invariant violated (psp::GraphInvariantError)   */
    PSP_EIO = 7,        /* file unreadable / truncated / inconsistent (psp::IoError) */
    PSP_EFORMAT = 8,    /* not a PSP1 file or wrong version (psp::FormatVersionError) */
    PSP_ECHECKSUM = 9,  /* CRC-64 mismatch (psp::ChecksumError)                  */
    PSP_EPARSE = 10     /* malformed graph text (psp::ParseError); line: psp_gpu_last_parse_line */
} psp_status;

enum {
    PSP_VALUE_AUTO = 0, /* u32 when exact (integral or dyadic weights), else f32 */
    PSP_VALUE_U32 = 1,  /* exact; fails with PSP_EOVERFLOW when not exact         */
    PSP_VALUE_F32 = 2   /* tolerance path                                         */
};

typedef struct psp_gpu_ctx psp_gpu_ctx;
typedef struct psp_gpu_oracle psp_gpu_oracle;

/* BuildStats (include/psp/oracle.hpp:29-37) plus device-side detail. */
typedef struct psp_build_stats {
    double partition_ms;       /* phase 1: partition + reorder (host)          */
    double component_apsp_ms;  /* phase 2: upload + K0 + K1 (wall clock)       */
    double boundary_ms;        /* phase 3: BG init + K2 + query tables (wall)  */
    uint64_t boundary_total;   /* b                                            */
    uint64_t bg_edges;         /* cross edges + finite clique pairs            */
    uint64_t stored_entries;   /* sum |C|^2 + |B(C)| * b                       */
    uint64_t peak_table_entries_per_worker;
    /* device detail (CUDA events on the build stream) */
    double k1_device_ms;       /* batched component Floyd-Warshall             */
    double k2_device_ms;       /* boundary-graph Floyd-Warshall                */
    double init_device_ms;     /* K0 + BG init + query-table extraction        */
    uint64_t k1_relaxations;   /* min-plus relaxations executed by K1 (padded) */
    uint64_t k2_relaxations;   /* min-plus relaxations executed by K2 (padded) */
    int32_t value_kind;        /* PSP_VALUE_U32 or PSP_VALUE_F32               */
    int32_t fixed_point_shift; /* q: device value = weight * 2^q (u32 only)    */
    uint64_t device_bytes;     /* device memory held by the oracle             */
    /* K2 working layout (ABI 4) */
    uint64_t k2_positions;     /* rows of the K2 working matrix (>= b: tile-packing padding) */
    int32_t k2_order;          /* 0 reference numbering, 1 elimination order   */
    int32_t k2_spilled;        /* component tables left the device during K2   */
    /* host sub-phases of the wall-clock phases (ABI 4) */
    double split_ms;           /* reordered CSR -> per-component edge lists    */
    double k1_order_ms;        /* nested-dissection orders (host threads)      */
    double bg_order_ms;        /* K2 elimination order + layout (host)         */
} psp_build_stats;

typedef struct psp_oracle_info {
    uint64_t n;
    uint32_t k;
    uint64_t b;
    int32_t value_kind;
    int32_t fixed_point_shift;
    int32_t device;
    int32_t tile; /* Floyd-Warshall tile edge T */
} psp_oracle_info;

/* ------------------------------------------------------------ runtime -- */
int psp_gpu_abi_version(void);
const char* psp_gpu_last_error(void);
int psp_gpu_device_count(void);

/* One context per GPU (one process per GPU). `rank`/`world` describe the
 * job; world == 1 is a single GPU. For world > 1 pass the 128-byte NCCL
 * unique id produced by psp_gpu_nccl_unique_id on rank 0 and broadcast by
 * the caller (e.g. through torch.distributed). */
psp_status psp_gpu_ctx_create(int device, int rank, int world, const void* nccl_id,
                              psp_gpu_ctx** out);
void psp_gpu_ctx_destroy(psp_gpu_ctx* ctx);
psp_status psp_gpu_nccl_unique_id(void* out128);
/* The context's CUDA stream (cudaStream_t) for callers that time kernels. */
void* psp_gpu_ctx_stream(psp_gpu_ctx* ctx);

/* Where later multi-GPU builds keep the boundary-graph table (the reference
 * keeps Oracle::boundary_tables, |B(C)| x b per component, on one host,
 * include/psp/oracle.hpp:60):
 *   PSP_STORAGE_REPLICATED  every rank ends the build with the whole table
 *                           (default; all query entry points work);
 *   PSP_STORAGE_ROW_SHARDED each rank keeps only the tile rows it computed in
 *                           the row-sharded K2 (about 1/world of the table, so
 *                           a table larger than one GPU builds across
 *                           several). Such an oracle answers through
 *                           psp_gpu_shard_create + psp_gpu_routed_query_batch
 *                           only; the replicated query, export-boundary-rows
 *                           and save entry points return PSP_EINVAL.
 * With world == 1 both mean replicated. */
enum psp_boundary_storage { PSP_STORAGE_REPLICATED = 0, PSP_STORAGE_ROW_SHARDED = 1 };
psp_status psp_gpu_ctx_set_boundary_storage(psp_gpu_ctx* ctx, int storage);

/* Process totals of the host time spent inside cudaMalloc / cudaFree of the
 * library's device buffers (diagnostics: single calls can stall for 0.1-1 s
 * on a busy driver): out4 = {malloc ns, malloc calls, free ns, free calls}. */
psp_status psp_gpu_alloc_stats(uint64_t* out4);

/* ------------------------------------------------------- preprocessing -- */
/* psp::build_oracle (include/psp/oracle.hpp:85-86, src/oracle.cpp:144-194):
 * partition + reorder on the host (identical assignment to the reference's
 * partition_graph, include/psp/partition.hpp:42), then Phase 2 (K0+K1) and
 * Phase 3 (BG init + K2) on the device. Edges are undirected, listed once
 * (psp::Graph(n, edges), include/psp/graph.hpp:50). workers < 1 or k outside
 * 1..n -> PSP_EINVAL (src/oracle.cpp:146, src/partition.cpp:261-262);
 * `workers` sizes the host partitioner's thread pool only and never changes
 * the result (include/psp/oracle.hpp:80-84). */
psp_status psp_gpu_build_oracle(psp_gpu_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* eu,
                                const uint32_t* ev, const double* ew, uint32_t k,
                                uint32_t workers, uint64_t seed, int value_kind,
                                psp_gpu_oracle** out, psp_build_stats* stats);

/* Same pipeline with the partition supplied by the caller as a component
 * assignment in ORIGINAL ids (psp::make_partition semantics,
 * include/psp/partition.hpp:61): boundary flags and the boundary-first
 * permutation are derived here exactly as src/partition.cpp:196-240 does. */
psp_status psp_gpu_build_partitioned(psp_gpu_ctx* ctx, uint64_t n, uint64_t m,
                                     const uint32_t* eu, const uint32_t* ev, const double* ew,
                                     uint32_t k, const uint32_t* assignment, int value_kind,
                                     psp_gpu_oracle** out, psp_build_stats* stats);

/* Import a host oracle into device memory for queries: e.g. one read by
 * psp::load_oracle (include/psp/oracle_io.hpp:22-34) or copied by value.
 * permutation: original -> reordered (n); assignment: reordered vertex ->
 * component (n); component_offset / boundary_offset (k+1);
 * component_tables[c]: |C| x |C| f64 row-major; boundary_tables[c]:
 * |B(C)| x b f64 (Oracle::component_tables / boundary_tables,
 * include/psp/oracle.hpp:59-60). PSP_VALUE_AUTO stores u32 when every finite
 * entry is exact in u32 fixed point, else f32. */
psp_status psp_gpu_oracle_import(psp_gpu_ctx* ctx, uint64_t n, uint32_t k,
                                 const uint32_t* permutation, const uint32_t* assignment,
                                 const uint64_t* component_offset,
                                 const uint64_t* boundary_offset,
                                 const double* const* component_tables,
                                 const double* const* boundary_tables, int value_kind,
                                 psp_gpu_oracle** out);

/* psp::save_oracle / load_oracle (include/psp/oracle_io.hpp:22-34,
 * src/oracle_io.cpp:106-255): the PSP1 file written straight from the device
 * tables (f64 conversion and CRC-64/XZ on the GPU), byte-identical to the
 * reference's image of the same oracle; and read back (same validation and
 * error classes as read_oracle) into a device oracle for queries. */
psp_status psp_gpu_oracle_save(const psp_gpu_oracle* o, const char* path);
psp_status psp_gpu_oracle_load(psp_gpu_ctx* ctx, const char* path, int value_kind,
                               psp_gpu_oracle** out);

void psp_gpu_oracle_free(psp_gpu_oracle* o);
psp_status psp_gpu_oracle_info(const psp_gpu_oracle* o, psp_oracle_info* out);

/* Oracle id maps (include/psp/oracle.hpp:47-62). Any pointer may be NULL.
 * permutation/inverse (n), assignment + boundary_flags in reordered ids (n),
 * component_offset / boundary_offset (k+1), boundary_vertex (b). */
psp_status psp_gpu_oracle_ids(const psp_gpu_oracle* o, uint32_t* permutation,
                              uint32_t* inverse_permutation, uint32_t* assignment,
                              uint8_t* boundary_flags, uint64_t* component_offset,
                              uint64_t* boundary_offset, uint32_t* boundary_vertex);

/* Materialise Oracle::component_tables[c] (|C| x |C|, row-major) and
 * Oracle::boundary_tables[c] (|B(C)| x b) as f64, for parity checks and for
 * persisting through save_oracle (include/psp/oracle_io.hpp). */
psp_status psp_gpu_export_component(const psp_gpu_oracle* o, uint32_t c, double* dst);
psp_status psp_gpu_export_boundary_rows(const psp_gpu_oracle* o, uint32_t c, double* dst);

/* ------------------------------------------------------------- queries -- */
/* psp::batch_query (include/psp/query.hpp:45-46, src/query.cpp:106-114) on
 * HOST arrays: ids in the original space, distances out as f64 (+inf when
 * unreachable), optional minplus_ops = |B(C1)|*|B(C2)| + |B(C2)|
 * (src/query.cpp:73). Host<->device copies happen inside the call. Any id
 * >= n -> PSP_EINVAL and no output (src/query.cpp:30). */
psp_status psp_gpu_query_batch(const psp_gpu_oracle* o, uint64_t count, const uint32_t* v1,
                               const uint32_t* v2, double* dist, uint64_t* minplus_ops);

/* Device-resident variant: v1, v2, dist are DEVICE pointers on the oracle's
 * GPU; enqueued on `stream` (a cudaStream_t, NULL = the context stream) and
 * returns without synchronising. Out-of-range ids are answered as (0, 0)
 * and not reported (the host variant reports them). */
psp_status psp_gpu_query_batch_device(const psp_gpu_oracle* o, uint64_t count,
                                      const uint32_t* v1, const uint32_t* v2, double* dist,
                                      void* stream);

/* Pipelined host batches: the same answers as psp_gpu_query_batch, with up
 * to `depth` batches in flight. A submit enqueues the host->device copy of
 * its pairs on an input copy stream, the query kernels on the pipe's compute
 * stream and the distance copy back on an output copy stream (ordered by
 * events) and returns at once, so the copies of neighbouring batches overlap
 * the kernels of this one (the serving loop of src/query.cpp:106-114 run as
 * a stream). Host arrays must stay valid until psp_gpu_query_pipe_wait, and
 * be pinned for the copies to be asynchronous. A submit blocks only while
 * all `depth` slots are busy. wait() drains every submitted batch and
 * returns PSP_EINVAL if any held an id >= n (src/query.cpp:30); the dist
 * array of such a batch is then unspecified. One thread per pipe. */
typedef struct psp_gpu_query_pipe psp_gpu_query_pipe;
psp_status psp_gpu_query_pipe_create(const psp_gpu_oracle* o, int depth,
                                     psp_gpu_query_pipe** out);
psp_status psp_gpu_query_pipe_submit(psp_gpu_query_pipe* p, uint64_t count, const uint32_t* v1,
                                     const uint32_t* v2, double* dist);
psp_status psp_gpu_query_pipe_wait(psp_gpu_query_pipe* p);
void psp_gpu_query_pipe_destroy(psp_gpu_query_pipe* p);

/* -------------------------------------------------- routed (sharded) -- */
/* The paper's distributed query mode on real GPUs: psp::routed_query and
 * psp::ClusterSim (include/psp/cluster.hpp:58-109, src/cluster.cpp) with
 * psp::Placement (include/psp/placement.hpp:8-31) mapping components to
 * the ranks of a multi-GPU context. */
enum psp_placement_policy {
    PSP_PLACE_ROUND_ROBIN = 0,  /* owner(c) = c mod p                         */
    PSP_PLACE_PAIRS_PER_GPU = 1 /* contiguous blocks, sizes differ by <= 1    */
};

typedef struct psp_gpu_shard psp_gpu_shard;

typedef struct psp_routed_stats {
    uint64_t queries;          /* pairs this rank submitted                    */
    uint64_t executed_here;    /* pairs this rank executed (owner(C1) == rank) */
    uint64_t sent_to_peers;    /* submitted pairs executed on another rank     */
    uint64_t transfer_queries; /* submitted pairs with owner(C1) != owner(C2)  */
    uint64_t transfer_entries; /* their col2 entries (B2 each)                 */
    uint64_t transfer_bytes;   /* 8 * entries (the reference's f64 ledger)     */
    double route_ms;           /* device time of the pair exchange             */
    double exec_ms;            /* device time of the executed batch            */
} psp_routed_stats;

/* psp::place_components (src/placement.cpp:7-33): owner[k]. p < 1 or
 * p > k -> PSP_EINVAL. */
psp_status psp_place_components(uint32_t k, uint32_t p, int policy, uint32_t* owner);

/* COLLECTIVE over the oracle's context (every rank calls it with the same
 * owner[k], each owner < world): keeps on this rank only the tables of the
 * components it owns -- their full boundary rows, to-boundary rows and
 * component tables -- and maps every peer's to-boundary rows through CUDA
 * IPC. The oracle may be freed afterwards. */
psp_status psp_gpu_shard_create(const psp_gpu_oracle* o, const uint32_t* owner,
                                psp_gpu_shard** out);
/* COLLECTIVE: barrier (peers may still read this rank's tables), then free. */
psp_status psp_gpu_shard_free(psp_gpu_shard* sh);
/* Device bytes this rank holds for the shard. */
psp_status psp_gpu_shard_bytes(const psp_gpu_shard* sh, uint64_t* bytes);

/* COLLECTIVE routed batch: every rank passes its own pairs (count may be
 * 0); each executes at owner(C1) (NCCL send/recv of the ids), col2 comes
 * from owner(C2)'s memory over NVLink, and dist[] returns in this rank's
 * order, equal to psp_gpu_query_batch on the replicated oracle (bit-exact
 * for u32). Optional per-query outputs (NULL to skip): executed_on,
 * column_owner, transfer_entries (B2 when the owners differ, else 0;
 * src/cluster.cpp:77-85). Host pointers. An id >= n on any rank fails the
 * batch on every rank with PSP_EINVAL. */
psp_status psp_gpu_routed_query_batch(psp_gpu_shard* sh, uint64_t count, const uint32_t* v1,
                                      const uint32_t* v2, double* dist, uint32_t* executed_on,
                                      uint32_t* column_owner, uint32_t* transfer_entries,
                                      psp_routed_stats* stats);

/* ------------------------------------------------------ graph ingestion -- */
/* psp::load_graph / read_graph / save_graph / write_graph / format_weight
 * (include/psp/graph_io.hpp:10-25). The text is parsed on the GPU; graphs,
 * values and ParseError messages ("<name>:<line>: <msg>") are the
 * reference's. Edge lists are strict; DIMACS arcs are normalised (min weight
 * per unordered pair, symmetrised, self-loops dropped, (u, v) order). */
enum psp_graph_format {
    PSP_FORMAT_EDGE_LIST = 0, /* "n m" header, one "u v w" line per edge   */
    PSP_FORMAT_DIMACS = 1     /* "p sp n m", "a u v w" arcs, 1-based ids  */
};
typedef struct psp_graph psp_graph;

/* File -> graph (PSP_EIO if unreadable, PSP_EPARSE / PSP_EGRAPH as the
 * reference throws ParseError / GraphInvariantError). */
psp_status psp_gpu_load_graph(psp_gpu_ctx* ctx, const char* path, int format, psp_graph** out);
/* In-memory text -> graph; `name` prefixes parse errors (reference: "<stream>"). */
psp_status psp_gpu_read_graph(psp_gpu_ctx* ctx, const char* text, uint64_t len, int format,
                              const char* name, psp_graph** out);
psp_status psp_graph_size(const psp_graph* g, uint64_t* n, uint64_t* m);
/* Edges as parsed (edge list: file order; DIMACS: normalised order). */
psp_status psp_graph_edges(const psp_graph* g, uint32_t* eu, uint32_t* ev, double* ew);
void psp_graph_free(psp_graph* g);
/* Line of the last PSP_EPARSE on this thread (psp::ParseError::line()). */
uint64_t psp_gpu_last_parse_line(void);

/* write_graph: text of the graph (edges validated as psp::Graph does, then
 * written from its sorted edge list) into buf; call with buf == NULL for
 * the length. save_graph writes it to a file. */
psp_status psp_write_graph(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                           const double* ew, int format, char* buf, uint64_t cap, uint64_t* len);
psp_status psp_save_graph(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                          const double* ew, const char* path, int format);
/* Shortest decimal that parses back to w (std::to_chars); buf >= 32 bytes;
 * returns the length. */
uint32_t psp_format_weight(double w, char* buf);

/* ---------------------------------------------------------- primitives -- */
/* psp::apsp_dense (include/psp/shortest_paths.hpp:43): dense APSP of one
 * graph on the device (K0 + K1 with a batch of one). block_size is the
 * reference's CPU tiling hint: ignored except that 0 -> PSP_EINVAL
 * (src/shortest_paths.cpp:131). out: n*n f64 row-major. */
psp_status psp_gpu_apsp_dense(psp_gpu_ctx* ctx, uint64_t n, uint64_t m, const uint32_t* eu,
                              const uint32_t* ev, const double* ew, uint64_t block_size,
                              int value_kind, double* out);

/* psp::boundary_apsp (include/psp/oracle.hpp:94-96): all-pairs distances of
 * a boundary graph given as an edge list over b vertices; out is b*b f64,
 * rows in boundary-id order, i.e. the concatenation of the reference's
 * per-component |B(C)| x b matrices. */
psp_status psp_gpu_boundary_apsp(psp_gpu_ctx* ctx, uint64_t b, uint64_t m, const uint32_t* eu,
                                 const uint32_t* ev, const double* ew, int value_kind,
                                 double* out);

/* Measured min-plus ALU peak of this GPU (relaxations/s) for the roofline:
 * kind PSP_VALUE_U32 (VIADDMNMX) or PSP_VALUE_F32 (FADD + FMNMX). */
psp_status psp_gpu_minplus_peak(psp_gpu_ctx* ctx, int value_kind, double* relax_per_s,
                                double* sm_clock_mhz);

/* ------------------------------------------------------- host helpers -- */
/* psp::partition_graph (include/psp/partition.hpp:42, src/partition.cpp:
 * 259-450): identical assignment for identical (graph, k, seed); the eight
 * independent restarts run on up to `threads` host threads. */
psp_status psp_partition_graph(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                               const double* ew, uint32_t k, uint64_t seed, uint32_t threads,
                               uint32_t* assignment);

/* Synthetic inputs: psp::generate_grid / generate_triangulated_grid
 * (include/psp/generators.hpp:24-30; kind 0 / 1; unit != 0 -> unit weights,
 * else the uniform 1/1024 lattice on [lo, hi]). Call with eu == NULL to get
 * the edge count in *m. */
psp_status psp_generate_grid(int kind, uint64_t rows, uint64_t cols, int unit, double lo,
                             double hi, uint64_t seed, uint64_t* m, uint32_t* eu, uint32_t* ev,
                             double* ew);

/* Delaunay triangulation of n points in [0,1)^2 (xy row-major, coordinates
 * on the 2^-53 grid numpy's uniform doubles lie on): the unique undirected
 * edges u < v in lexicographic order, exactly the edge set scipy Qhull gives
 * for points in general position (exact predicates). Generates BASELINE.json
 * configs[1]/[2] (workloads.py defines them with scipy). `cap` >= 3n; the
 * edge count goes to *m. Not a reference symbol: bench/test input tooling. */
psp_status psp_delaunay_edges(uint64_t n, const double* xy, uint64_t cap, uint32_t* eu,
                              uint32_t* ev, uint64_t* m);

/* Minimum spanning forest of an edge list under the keys `key` (Kruskal;
 * in_tree[e] = 1 for forest edges). With distinct keys it is the unique
 * forest scipy's minimum_spanning_tree returns; used by the road-like grid of
 * BASELINE.json configs[3] (workloads.py road_grid). Not a reference symbol:
 * bench/test input tooling. */
psp_status psp_min_spanning_forest(uint64_t n, uint64_t m, const uint32_t* eu, const uint32_t* ev,
                                   const double* key, uint8_t* in_tree);

/* ref::random_pairs / the CLI's random_pairs (tests/support/reference.hpp:
 * 80-91, tools/psp_main.cpp:108-120): mt19937_64, v1 = rng() % n then v2. */
void psp_random_pairs(uint64_t n, uint64_t count, uint64_t seed, uint32_t* v1, uint32_t* v2);

#ifdef __cplusplus
}
#endif

#endif /* PSP_GPU_H */
