// query_kernels.cuh — K3: batched distance queries (Algorithm 2).
//
// Replaces query / batch_query (src/query.cpp:29-114):
//   through[j] = min_i row1[i] + BG[g1 + i][g2 + j]     (stitch_into :49-59)
//   d          = min_j through[j] + col2[j]             (min_plus_combine :61-65)
//   d          = min(d, CT[c1](l1, l2)) if c1 == c2     (finish :70-72)
// One warp per query: lanes own target boundary columns j, the source
// boundary row values row1[i] are fetched 32 at a time and broadcast with
// SHFL, the final min is a warp reduction (REDUX.MIN for u32).
//
// Undirected symmetry (dist(v,w) = dist(w,v), tests/test_query.cpp:144-153)
// lets every query be turned around so that c1 <= c2: the B1 x B2 block
// BG[g1.., g2..] then lies in the stored upper triangle (g1 + B1 <= g2), and
// rows advance by a constant stride inside a tile. In u32 the result is
// exact either way; in f32 the three-term sums may round differently, which
// the 1e-5 tolerance covers.
#pragma once
#include "minplus.cuh"

namespace pspg {

template <class V> struct QueryView {
    const uint32_t* perm;       // original -> reordered id
    const uint32_t* assign;     // reordered id -> component
    const uint32_t* comp_off;   // k+1
    const uint32_t* bnd_off;    // k+1 (boundary-id space)
    const uint64_t* cb_off;     // k: offset of CB[c]
    const V* cb;                // |C| x |B(C)| to-boundary tables
    MatSet<V> comps;            // full component tables (same-component cap)
    const V* bg;                // boundary-graph tiles
    uint32_t bg_nb;
    double scale;               // 2^-q (u32 fixed point) or 1
};

template <class V>
__device__ __forceinline__ V warp_min(V v);
template <>
__device__ __forceinline__ uint32_t warp_min<uint32_t>(uint32_t v) {
    return __reduce_min_sync(0xffffffffu, v);
}
template <>
__device__ __forceinline__ float warp_min<float>(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

template <class V>
__global__ void __launch_bounds__(256) query_warp(QueryView<V> q, const uint32_t* __restrict__ v1,
                                                  const uint32_t* __restrict__ v2, uint64_t count,
                                                  double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t qi = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; qi < count;
         qi += nwarps) {
        uint32_t r1 = q.perm[v1[qi]], r2 = q.perm[v2[qi]];
        uint32_t c1 = q.assign[r1], c2 = q.assign[r2];
        if (c1 > c2) {
            uint32_t t = r1; r1 = r2; r2 = t;
            t = c1; c1 = c2; c2 = t;
        }
        const uint32_t l1 = r1 - q.comp_off[c1], l2 = r2 - q.comp_off[c2];
        const uint32_t g1 = q.bnd_off[c1], B1 = q.bnd_off[c1 + 1] - g1;
        const uint32_t g2 = q.bnd_off[c2], B2 = q.bnd_off[c2 + 1] - g2;
        const V* row1 = q.cb + q.cb_off[c1] + uint64_t(l1) * B1;
        const V* col2 = q.cb + q.cb_off[c2] + uint64_t(l2) * B2;
        const uint32_t nb = q.bg_nb;
        V best = Ops<V>::inf();
        for (uint32_t j0 = 0; j0 < B2; j0 += 32) {
            const uint32_t j = j0 + lane;
            const bool active = j < B2;
            const uint32_t gj = g2 + (active ? j : B2 - 1);
            const uint32_t Jt = gj / T, jj = gj % T;
            V acc = Ops<V>::inf();
            for (uint32_t i0 = 0; i0 < B1; i0 += 32) {
                const uint32_t ni = min(32u, B1 - i0);
                const V rv = (lane < ni) ? row1[i0 + lane] : Ops<V>::inf();
                const uint32_t gi0 = g1 + i0;
                if (c1 != c2) {
                    // rows gi0.. cross at most one tile boundary (32 < T)
                    const uint32_t It = gi0 / T;
                    const uint32_t split = min(ni, T - gi0 % T);
                    const V* pa = q.bg + tidx(It, Jt, nb) * TT + uint64_t(gi0 % T) * T + jj;
                    const V* pb = q.bg + tidx(It + 1 < nb ? It + 1 : It, Jt, nb) * TT + jj;
                    pb -= uint64_t(split) * T;
                    if (ni == 32) {
#pragma unroll
                        for (uint32_t t = 0; t < 32; ++t) {
                            const V* p = (t < split) ? pa : pb;
                            acc = Ops<V>::addmin(__shfl_sync(0xffffffffu, rv, t), p[t * T], acc);
                        }
                    } else {
                        for (uint32_t t = 0; t < ni; ++t) {
                            const V* p = (t < split) ? pa : pb;
                            acc = Ops<V>::addmin(__shfl_sync(0xffffffffu, rv, t), p[t * T], acc);
                        }
                    }
                } else {
                    // diagonal block: both triangles, symmetric lookup
                    for (uint32_t t = 0; t < ni; ++t) {
                        const V e = q.bg[sym_off(gi0 + t, gj, nb)];
                        acc = Ops<V>::addmin(__shfl_sync(0xffffffffu, rv, t), e, acc);
                    }
                }
            }
            if (active) best = Ops<V>::addmin(acc, col2[j], best);
        }
        best = warp_min<V>(best);
        if (lane == 0) {
            if (c1 == c2) {
                const V same =
                    q.comps.tiles[q.comps.tile_base[c1] + sym_off(l1, l2, q.comps.nb[c1])];
                best = Ops<V>::vmin(best, same);
            }
            out[qi] = Ops<V>::to_f64(best, q.scale);
        }
    }
}

}  // namespace pspg
