// minplus.cuh — value semantics and tile geometry shared by every kernel.
//
// Two value kinds (BASELINE.json north_star):
//   u32  exact. INF = 0x7FFFFFFF so INF + INF = 0xFFFFFFFE never wraps; the
//        host guarantees every finite distance < 2^31 - 1
//        (max_w * 2^q * (n - 1) < 2^31 - 1), so one add of two stored values
//        never wraps either, and min() clamps anything >= INF back to <= INF.
//        min(a + b, c) compiles to one VIADDMNMX.U32 on sm_100a.
//   f32  tolerance path. INF = +inf; relaxations are paired so that two of
//        them cost FADD + FADD + one 3-input FMNMX3 (addmin2).
//
// The reference skips unreachable rows explicitly
// (src/shortest_paths.cpp:117, src/query.cpp:53); with these encodings the
// skip is implicit because INF + x >= INF never wins a min.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace pspg {

constexpr int T = 128;          // Floyd-Warshall tile edge
constexpr int TT = T * T;       // elements per tile
constexpr int NTHREADS = 256;   // 16 x 16 threads, 8 x 8 register block each
constexpr uint32_t U32_INF = 0x7FFFFFFFu;

template <class V> struct Ops;

template <> struct Ops<uint32_t> {
    static __host__ __device__ __forceinline__ uint32_t inf() { return U32_INF; }
    static __device__ __forceinline__ uint32_t addmin(uint32_t a, uint32_t b, uint32_t c) {
        return min(a + b, c);
    }
    // two relaxations of one accumulator: two VIADDMNMX
    static __device__ __forceinline__ uint32_t addmin2(uint32_t a0, uint32_t b0, uint32_t a1,
                                                       uint32_t b1, uint32_t c) {
        return min(a1 + b1, min(a0 + b0, c));
    }
    static __device__ __forceinline__ uint32_t vmin(uint32_t a, uint32_t b) { return min(a, b); }
    static __device__ __forceinline__ uint32_t from_bits(uint32_t u) { return u; }
    static __device__ __forceinline__ uint32_t to_bits(uint32_t v) { return v; }
    static __device__ __forceinline__ double to_f64(uint32_t v, double scale) {
        return v >= U32_INF ? __longlong_as_double(0x7ff0000000000000ll) : double(v) * scale;
    }
};

template <> struct Ops<float> {
    static __host__ __device__ __forceinline__ float inf() { return __builtin_huge_valf(); }
    static __device__ __forceinline__ float addmin(float a, float b, float c) {
        return fminf(a + b, c);
    }
    // two relaxations of one accumulator: FADD x2 + one 3-input FMNMX3
    // (1.5 instructions per relaxation instead of 2)
    static __device__ __forceinline__ float addmin2(float a0, float b0, float a1, float b1,
                                                    float c) {
        return fminf(fminf(c, a0 + b0), a1 + b1);  // ptxas fuses to FMNMX3
    }
    static __device__ __forceinline__ float vmin(float a, float b) { return fminf(a, b); }
    static __device__ __forceinline__ float from_bits(uint32_t u) { return __uint_as_float(u); }
    static __device__ __forceinline__ uint32_t to_bits(float v) { return __float_as_uint(v); }
    static __device__ __forceinline__ double to_f64(float v, double) { return double(v); }
};

// ---------------------------------------------------------------- layout --
// A symmetric n x n distance matrix is stored as the upper triangle of its
// nb x nb grid of T x T tiles (nb = ceil(n / T)), "tile-packed": tile (I, J)
// with I <= J is one contiguous T*T row-major block at index
//   tidx(I, J) = I * (2 nb - I + 1) / 2 + (J - I).
// Diagonal tiles hold both triangles. Padding rows/columns (>= n) are
// isolated dummy vertices (INF, 0 on the diagonal) that never shorten a
// path. Element (i, j) lives in tile (min(I,J), max(I,J)); the rule for
// writers is: write (i, j) iff i / T <= j / T.
__host__ __device__ __forceinline__ uint64_t tidx(uint32_t I, uint32_t J, uint32_t nb) {
    return uint64_t(I) * (2ull * nb - I + 1) / 2 + (J - I);
}
__host__ __device__ __forceinline__ uint64_t ntiles_upper(uint32_t nb) {
    return uint64_t(nb) * (nb + 1) / 2;
}
// Offset (in elements, relative to the matrix's first tile) of element (i, j).
__host__ __device__ __forceinline__ uint64_t sym_off(uint32_t i, uint32_t j, uint32_t nb) {
    if (i / T > j / T) {
        const uint32_t t = i;
        i = j;
        j = t;
    }
    return tidx(i / T, j / T, nb) * TT + uint64_t(i % T) * T + (j % T);
}

// Row stride of the query-side to-boundary tables: |B(C)| rounded up to 16
// (INF padded), so a query's row1 for any 16-row chunk of its pair block
// (rows < B1 rounded up to 16) lies inside its row: the grouped product
// stages it with unpredicated 16-byte copies.
__host__ __device__ __forceinline__ uint32_t cb_stride(uint32_t B) { return (B + 15u) & ~15u; }

// A batch of matrices sharing one tile arena (component tables: k matrices;
// boundary graph: one). Arrays are device pointers indexed by matrix.
template <class V> struct MatSet {
    V* tiles;                   // tile arena
    V* panel;                   // per-matrix row-panel slots (nb * T*T each)
    const uint64_t* tile_base;  // element offset of matrix m's first tile
    const uint64_t* panel_base; // element offset of matrix m's panel slots
    const uint64_t* work_prefix;// prefix sum of upper-tile counts (nmat + 1)
    const uint32_t* nb;         // tiles per side
    uint32_t nmat;
    uint32_t nb_max;
    // multi-GPU boundary graph (nmat == 1): tile rows owned by this rank
    // (owner(I) = I mod world), phase 3 walks only these rows
    const uint32_t* rows;       // owned tile rows, ascending (nullptr: all rows)
    const uint64_t* row_prefix; // prefix of their upper-tile counts (nrows + 1)
    uint32_t nrows;
    uint32_t rank, world;
    // peer-to-peer panel exchange (engine_fw.cuh run_fw_sharded): phase 2
    // leaves the slots other ranks compute untouched (they are pulled over
    // NVLink instead of min-allreduced)
    uint32_t p2p;
    // the closed diagonal tile of the current k-block when it is not in this
    // rank's storage (row-sharded table, pulled from its owner); null: the
    // matrix's own tile (kb, kb)
    const V* diag;
    // sparse walk (null: dense). Per k-block phase 2 writes act_flag[s + J]
    // (s = panel_base[m] / TT, matrix m's first panel slot; V-typed so the
    // sharded build min-allreduces it with the panel: 0 = panel slot J holds
    // a finite entry, 1 = all INF; a panel tile that is all INF on input is
    // not computed). fw_active_list compacts matrix m's active slots into
    // act_list[s..] and the rows this rank processes into act_rows[s..]
    // (positions in act_list) with the prefix of their upper-tile counts in
    // act_prefix[s + m ..]; act_meta[2m..2m+1] = {active slots, rows};
    // fw_mat_prefix scans the per-matrix totals into mat_prefix (nmat + 1).
    // A phase-3 tile (I, J) whose panel slot I or J is all INF cannot change
    // (INF + x >= INF), so only active x active tiles are walked.
    V* act_flag;
    uint32_t* act_list;
    uint32_t* act_rows;
    uint64_t* act_prefix;
    uint32_t* act_meta;
    uint64_t* mat_prefix;
    unsigned long long* act_work;  // running count of tile products executed (all phases)
};

}  // namespace pspg
