// fw_kernels.cuh — K0/K1/K2: batched, symmetric, tile-packed blocked
// Floyd-Warshall (min-plus) for sm_100a.
//
// Replaces the reference's apsp_dense (src/shortest_paths.cpp:107-172, Phase 2)
// and the Dijkstra-per-boundary-vertex boundary_apsp
// (src/oracle.cpp:127-142, Phase 3) with one engine:
//
//   for each k-block kb (T = 128 intermediates):
//     phase 1  diagonal tile (kb,kb): sequential FW over its 128 vertices,
//              8x8 register block per thread, row/column k broadcast through
//              double-buffered shared memory (one barrier per k).
//     phase 2  row panel R_J = D[kb-rows][J-cols] for every J != kb, as the
//              single min-plus product R_J <- Dkk* (x) R_J (the closed diagonal
//              tile has a zero diagonal, so R_J itself is included). The
//              updated panel is written to its home tile and to the per-matrix
//              panel buffer in [k][j] layout.
//     phase 3  every upper tile (I,J), I,J != kb:
//              D_IJ <- min(D_IJ, R_I^T (x) R_J). Symmetry gives the column
//              panel for free (D[i][k] = D[k][i] = R_I[k][i]), so both
//              operands are panel slots, already in the k-major layout the
//              register-blocked inner loop wants, and only the upper triangle
//              is computed: half the relaxations and half the bytes of a
//              full-matrix FW.
//
// Exactness: u32 min-plus is exact, so the result equals the reference's f64
// tables bit for bit after conversion (every FW order yields the same exact
// shortest-path distances). FW keeps the matrix exactly symmetric even in f32
// because a + b == b + a.
//
// The inner loop (phase 2/3) per k: 2 LDS.128 for A (broadcast within a
// warp), 2 LDS.128 for B, 64 fused add-min (VIADDMNMX.U32 / FADD+FMNMX).
#pragma once
#include <type_traits>

#include "minplus.cuh"

namespace pspg {

// ------------------------------------------------------------ PTX utils --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
                 : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D TMA: contiguous global -> shared bulk copy completing on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// --------------------------------------------------- register blocking --
// Thread (ty, tx) of a 16x16 block owns rows {4ty..4ty+3, 64+4ty..64+4ty+3}
// and the same pattern of columns with tx: two aligned 4-vectors per side.
__device__ __forceinline__ int blk(int t, int a) { return (a < 4) ? 4 * t + a : 60 + 4 * t + a; }

template <class V>
__device__ __forceinline__ void ld4(const V* p, V* r) {
    const uint4 u = *reinterpret_cast<const uint4*>(p);
    r[0] = Ops<V>::from_bits(u.x);
    r[1] = Ops<V>::from_bits(u.y);
    r[2] = Ops<V>::from_bits(u.z);
    r[3] = Ops<V>::from_bits(u.w);
}
template <class V>
__device__ __forceinline__ void st4(V* p, const V* r) {
    uint4 u;
    u.x = Ops<V>::to_bits(r[0]);
    u.y = Ops<V>::to_bits(r[1]);
    u.z = Ops<V>::to_bits(r[2]);
    u.w = Ops<V>::to_bits(r[3]);
    *reinterpret_cast<uint4*>(p) = u;
}

// acc <- 8x8 block of a row-major T x T tile
template <class V>
__device__ __forceinline__ void load_block(const V* tile, V (&acc)[8][8], int ty, int tx) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        const V* row = tile + blk(ty, a) * T;
        ld4(row + 4 * tx, &acc[a][0]);
        ld4(row + 64 + 4 * tx, &acc[a][4]);
    }
}
template <class V>
__device__ __forceinline__ void store_block(V* tile, const V (&acc)[8][8], int ty, int tx) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
        V* row = tile + blk(ty, a) * T;
        st4(row + 4 * tx, &acc[a][0]);
        st4(row + 64 + 4 * tx, &acc[a][4]);
    }
}
// transposed store: tile[col][row] <- acc[row][col]; rows come in aligned
// 4-groups, so every store is still a 16-byte vector.
template <class V>
__device__ __forceinline__ void store_block_t(V* tile, const V (&acc)[8][8], int ty, int tx) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        V* row = tile + blk(tx, b) * T;
        V lo[4] = {acc[0][b], acc[1][b], acc[2][b], acc[3][b]};
        V hi[4] = {acc[4][b], acc[5][b], acc[6][b], acc[7][b]};
        st4(row + 4 * ty, lo);
        st4(row + 64 + 4 * ty, hi);
    }
}

// acc[a][b] <- min_k A(row a, k) + sB[k][col b] over k in [0, T).
// A_KMAJOR: sA[k][row] (the panel layout); otherwise sA[row][k].
template <class V, bool A_KMAJOR>
__device__ __forceinline__ void load_ab(const V* __restrict__ sA, const V* __restrict__ sB, int k,
                                        int ty, int tx, V (&a)[8], V (&b)[8]) {
    if (A_KMAJOR) {
        ld4(sA + k * T + 4 * ty, &a[0]);
        ld4(sA + k * T + 64 + 4 * ty, &a[4]);
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = sA[blk(ty, i) * T + k];
    }
    ld4(sB + k * T + 4 * tx, &b[0]);
    ld4(sB + k * T + 64 + 4 * tx, &b[4]);
}

// k advances in pairs so each accumulator takes two relaxations per update
// (Ops::addmin2: 2 x VIADDMNMX for u32, FADD x2 + FMNMX3 for f32). Eight
// pairs per loop trip cut the loop's address/branch ALU work (cfg3 K2: 8.05 s
// with one pair, 7.83 s with two, 7.74 s with four, 7.64 s with eight, 7.69 s
// with sixteen; road4m f32 K2 20.2 s with one, 19.2 s with two, 20.0 s with
// eight, so f32 keeps two; one CTA/SM either way).
template <class V, bool A_KMAJOR>
__device__ __forceinline__ void minplus_tile(const V* __restrict__ sA, const V* __restrict__ sB,
                                             V (&acc)[8][8], int ty, int tx) {
    constexpr int kUnroll = std::is_same<V, float>::value ? 2 : 8;
#pragma unroll kUnroll
    for (int k = 0; k < T; k += 2) {
        V a0[8], b0[8], a1[8], b1[8];
        load_ab<V, A_KMAJOR>(sA, sB, k, ty, tx, a0, b0);
        load_ab<V, A_KMAJOR>(sA, sB, k + 1, ty, tx, a1, b1);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                acc[i][j] = Ops<V>::addmin2(a0[i], b0[j], a1[i], b1[j], acc[i][j]);
    }
}

// ---------------------------------------------------------------- phase 1 --
// grid: nmat CTAs; one diagonal tile each.
template <class V>
__global__ void __launch_bounds__(NTHREADS) fw_phase1(MatSet<V> ms, uint32_t kb) {
    const uint32_t m = blockIdx.x;
    const uint32_t nb = ms.nb[m];
    if (kb >= nb) return;
    __shared__ __align__(16) V rowbuf[2][T];
    __shared__ __align__(16) V colbuf[2][T];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    V* tile = ms.tiles + ms.tile_base[m] + tidx(kb, kb, nb) * TT;
    V acc[8][8];
    load_block(tile, acc, ty, tx);

    // k runs over the two halves; within a half, k = half*64 + 4*q + r is
    // owned (as a row) by ty == q at register row a = 4*half + r, and (as a
    // column) by tx == q at register column 4*half + r.
#pragma unroll
    for (int half = 0; half < 2; ++half) {
#pragma unroll 1
        for (int q = 0; q < 16; ++q) {
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                const int k = half * 64 + 4 * q + r;
                const int buf = k & 1;
                const int a = 4 * half + r;
                if (ty == q) {
                    st4(&rowbuf[buf][4 * tx], &acc[a][0]);
                    st4(&rowbuf[buf][64 + 4 * tx], &acc[a][4]);
                }
                if (tx == q) {
                    V lo[4] = {acc[0][a], acc[1][a], acc[2][a], acc[3][a]};
                    V hi[4] = {acc[4][a], acc[5][a], acc[6][a], acc[7][a]};
                    st4(&colbuf[buf][4 * ty], lo);
                    st4(&colbuf[buf][64 + 4 * ty], hi);
                }
                __syncthreads();
                V cv[8], rv[8];
                ld4(&colbuf[buf][4 * ty], &cv[0]);
                ld4(&colbuf[buf][64 + 4 * ty], &cv[4]);
                ld4(&rowbuf[buf][4 * tx], &rv[0]);
                ld4(&rowbuf[buf][64 + 4 * tx], &rv[4]);
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 8; ++j) acc[i][j] = Ops<V>::addmin(cv[i], rv[j], acc[i][j]);
            }
        }
    }
    store_block(tile, acc, ty, tx);
}

// ---------------------------------------------------------------- phase 2 --
// grid: (nmat, nb_max). CTA (m, J) updates row-panel tile J of matrix m.
template <class V>
__global__ void __launch_bounds__(NTHREADS, 1) fw_phase2(MatSet<V> ms, uint32_t kb) {
    const uint32_t m = blockIdx.x;
    const uint32_t nb = ms.nb[m];
    const uint32_t J = blockIdx.y;
    if (kb >= nb || J >= nb || J == kb) return;
    if (ms.world > 1) {
        // the panel tile's home row is kb (J > kb) or J (J < kb); its owner
        // computes it, every other rank contributes INF to the min-allreduce
        const uint32_t home_row = J > kb ? kb : J;
        if (home_row % ms.world != ms.rank) {
            if (ms.p2p) return;  // its owner computes it, this rank pulls it
            V* panel = ms.panel + ms.panel_base[m] + uint64_t(J) * TT;
            for (int e = threadIdx.x * 4; e < TT; e += NTHREADS * 4) {
                const V inf4[4] = {Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf()};
                st4(panel + e, inf4);
            }
            if (ms.act_flag && threadIdx.x == 0) ms.act_flag[J] = V(1);  // min-allreduce neutral (nmat == 1)
            return;
        }
    }
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V* sA = reinterpret_cast<V*>(smem_raw);
    V* sB = sA + TT;
    __shared__ uint64_t bar;
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
    V* base = ms.tiles + ms.tile_base[m];
    const V* diag = ms.diag ? ms.diag : base + tidx(kb, kb, nb) * TT;
    V* panel = ms.panel + ms.panel_base[m] + uint64_t(J) * TT;
    const bool upper = J > kb;
    V* home = base + (upper ? tidx(kb, J, nb) : tidx(J, kb, nb)) * TT;
    if (tid == 0) {
        mbar_init(&bar, 1);
        mbar_expect_tx(&bar, 2 * TT * sizeof(V));
        if (upper) {
            bulk_g2s(sA, diag, TT * sizeof(V), &bar);  // Dkk* (symmetric: [k'][k])
            bulk_g2s(sB, home, TT * sizeof(V), &bar);  // R_J [k'][j]
        } else {
            bulk_g2s(sA, home, TT * sizeof(V), &bar);  // Y = R_J^T [j][k']
            bulk_g2s(sB, diag, TT * sizeof(V), &bar);  // Dkk* [k'][k]
        }
    }
    __syncthreads();
    V acc[8][8];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = Ops<V>::inf();
    mbar_wait(&bar, 0);
    if (ms.act_flag) {
        // sparse walk: a panel tile that is all INF stays all INF (and its
        // slot inactive); one that holds a finite entry stays finite (Dkk*
        // has a zero diagonal), so the flag is known before the product
        const V* in = upper ? sB : sA;
        bool fin = false;
        for (int e = tid * 4; e < TT; e += NTHREADS * 4) {
            const uint4 u = *reinterpret_cast<const uint4*>(in + e);
            fin |= (Ops<V>::from_bits(u.x) < Ops<V>::inf()) | (Ops<V>::from_bits(u.y) < Ops<V>::inf()) |
                   (Ops<V>::from_bits(u.z) < Ops<V>::inf()) | (Ops<V>::from_bits(u.w) < Ops<V>::inf());
        }
        fin = __syncthreads_or(fin);
        if (tid == 0) ms.act_flag[ms.panel_base[m] / TT + J] = fin ? V(0) : V(1);
        if (!fin) return;
    }
    if (upper) {
        // out[k][j] = min_k' Dkk[k][k'] + R_J[k'][j]
        minplus_tile<V, true>(sA, sB, acc, ty, tx);
        store_block(home, acc, ty, tx);
        store_block(panel, acc, ty, tx);
    } else {
        // out^T[j][k] = min_k' Y[j][k'] + Dkk[k'][k]; the home tile (J, kb)
        // is stored [j][k] = out^T, the panel slot wants [k][j].
        minplus_tile<V, false>(sA, sB, acc, ty, tx);
        store_block(home, acc, ty, tx);
        store_block_t(panel, acc, ty, tx);
    }
}

// Sparse phase 3 work lists for k-block kb, one CTA of 1024 threads per
// matrix m: its active panel slots J != kb in ascending order, the rows this
// rank walks (all of them, or I mod world == rank) as positions in that
// list, and the prefix of their tile counts (row at position p walks
// J = list[p..na)). act_work counts the tile products of the k-block: the
// walked phase-3 tiles plus the diagonal and the computed panel tiles
// (counted once, on rank 0, in the sharded build).
template <class V>
__global__ void __launch_bounds__(1024) fw_active_list(MatSet<V> ms, uint32_t kb) {
    __shared__ uint32_t warp_sum[32];
    __shared__ uint32_t carry;
    const uint32_t mi = blockIdx.x;
    const uint32_t nb = ms.nb[mi];
    const uint64_t sb = ms.panel_base[mi] / TT, ab = sb + mi;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (kb >= nb) {  // finished (or empty) matrix: no work
        if (tid == 0) {
            ms.act_meta[2 * mi] = 0;
            ms.act_meta[2 * mi + 1] = 0;
            ms.act_prefix[ab] = 0;
        }
        return;
    }
    const V* flag = ms.act_flag + sb;
    uint32_t* list = ms.act_list + sb;
    if (tid == 0) carry = 0;
    __syncthreads();
    // pass 1: compact the active slots
    for (uint32_t base = 0; base < nb; base += 1024) {
        const uint32_t J = base + tid;
        const bool act = J < nb && J != kb && flag[J] == V(0);
        const uint32_t bal = __ballot_sync(0xffffffffu, act);
        if (lane == 0) warp_sum[wid] = __popc(bal);
        __syncthreads();
        uint32_t before = carry;
        for (int w = 0; w < wid; ++w) before += warp_sum[w];
        before += __popc(bal & ((1u << lane) - 1u));
        if (act) list[before] = J;
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
            for (int w = 0; w < 32; ++w) t += warp_sum[w];
            carry += t;
        }
        __syncthreads();
    }
    const uint32_t na = carry;
    __syncthreads();
    if (tid == 0) carry = 0;
    __syncthreads();
    // pass 2: rows of this rank (positions p) and the exclusive prefix of
    // their tile counts (na - p), one block-wide scan per 1024 positions
    __shared__ unsigned long long wsum64[32];
    __shared__ unsigned long long carry64;
    if (tid == 0) carry64 = 0;
    __syncthreads();
    for (uint32_t base = 0; base < na; base += 1024) {
        const uint32_t p = base + tid;
        const bool own = p < na && (ms.world <= 1 || list[p] % ms.world == ms.rank);
        const uint32_t bal = __ballot_sync(0xffffffffu, own);
        unsigned long long v = own ? (unsigned long long)(na - p) : 0ull, incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) { warp_sum[wid] = __popc(bal); wsum64[wid] = incl; }
        __syncthreads();
        uint32_t before = carry;
        unsigned long long pre = carry64;
        for (int w = 0; w < wid; ++w) { before += warp_sum[w]; pre += wsum64[w]; }
        before += __popc(bal & ((1u << lane) - 1u));
        if (own) {
            ms.act_rows[sb + before] = p;
            ms.act_prefix[ab + before] = pre + incl - v;
        }
        __syncthreads();
        if (tid == 0) {
            for (int w = 0; w < 32; ++w) { carry += warp_sum[w]; carry64 += wsum64[w]; }
        }
        __syncthreads();
    }
    if (tid == 0) {
        ms.act_prefix[ab + carry] = carry64;
        ms.act_meta[2 * mi] = na;
        ms.act_meta[2 * mi + 1] = carry;
        atomicAdd(ms.act_work, carry64 + ((ms.world <= 1 || ms.rank == 0) ? na + 1ull : 0ull));
    }
}

// mat_prefix = exclusive prefix over the matrices of their phase-3 work
// (one CTA of 1024 threads).
template <class V>
__global__ void __launch_bounds__(1024) fw_mat_prefix(MatSet<V> ms) {
    __shared__ unsigned long long wsum[32];
    __shared__ unsigned long long carry;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) {
        carry = 0;
        ms.mat_prefix[0] = 0;
    }
    __syncthreads();
    for (uint32_t base = 0; base < ms.nmat; base += 1024) {
        const uint32_t mi = base + tid;
        unsigned long long v = 0;
        if (mi < ms.nmat) v = ms.act_prefix[ms.panel_base[mi] / TT + mi + ms.act_meta[2 * mi + 1]];
        unsigned long long incl = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += t;
        }
        if (lane == 31) wsum[wid] = incl;
        __syncthreads();
        unsigned long long pre = carry;
        for (int w = 0; w < wid; ++w) pre += wsum[w];
        if (mi < ms.nmat) ms.mat_prefix[mi + 1] = pre + incl;
        __syncthreads();
        if (tid == 0)
            for (int w = 0; w < 32; ++w) carry += wsum[w];
        __syncthreads();
    }
}

// ---------------------------------------------------------------- phase 3 --
// Persistent: gridDim.x CTAs split the flat list of (matrix, upper tile)
// items into contiguous ranges, so consecutive items share the tile row I
// and the A operand (panel slot I) is reloaded only when I changes.
// Software pipeline per CTA: the B operand is double-buffered in shared
// memory and the next item's panel slot is fetched by 1-D TMA while the
// current item computes; the C tile is loaded into registers alongside the
// min-plus product and folded in at the end (min is associative), so the
// ALU pipe no longer waits for either transfer. Shared memory: A 64 KB +
// 2 x B 64 KB.
__device__ __forceinline__ uint32_t row_start(uint32_t I, uint32_t nb) {
    return I * nb - (I * (I - 1u)) / 2u;  // first flat index of tile row I
}

struct P3Cursor {
    uint64_t w;
    uint32_t m, ri, nb, I, J;
    uint32_t p, q, am, anr;  // sparse mode: positions of I and J in act_list, |list|, rows
    uint64_t sb;             // sparse mode: matrix m's first panel slot (its lists start there)
};

// sparse mode: enter matrix m at its first walked row
template <class V>
__device__ __forceinline__ void p3_enter(const MatSet<V>& ms, P3Cursor& c, uint32_t m) {
    c.m = m;
    c.nb = ms.nb[m];
    c.sb = ms.panel_base[m] / TT;
    c.am = ms.act_meta[2 * m];
    c.anr = ms.act_meta[2 * m + 1];
    c.ri = 0;
}

template <class V>
__device__ __forceinline__ void p3_advance(const MatSet<V>& ms, P3Cursor& c) {
    ++c.w;
    if (ms.act_flag != nullptr) {
        if (++c.q == c.am && ++c.ri < c.anr) {
            c.p = ms.act_rows[c.sb + c.ri];
            c.q = c.p;
        }
        if (c.ri >= c.anr) {  // next matrix with work
            uint32_t m = c.m;
            do {
                ++m;
            } while (m < ms.nmat && ms.mat_prefix[m + 1] == ms.mat_prefix[m]);
            if (m >= ms.nmat) return;  // past the end: c.w >= total
            p3_enter(ms, c, m);
            c.p = ms.act_rows[c.sb];
            c.q = c.p;
        }
        c.I = ms.act_list[c.sb + c.p];
        c.J = ms.act_list[c.sb + c.q];
    } else if (ms.rows != nullptr) {
        if (++c.J == c.nb && ++c.ri < ms.nrows) {
            c.I = ms.rows[c.ri];
            c.J = c.I;
        }
    } else if (++c.J == c.nb) {
        if (++c.I == c.nb) {
            do {
                ++c.m;
            } while (c.m < ms.nmat && ms.nb[c.m] == 0);  // empty components own no tiles
            if (c.m < ms.nmat) c.nb = ms.nb[c.m];
            c.I = 0;
        }
        c.J = c.I;
    }
}

template <class V>
__device__ __forceinline__ bool p3_valid(const P3Cursor& c, uint64_t w1, uint32_t kb) {
    return c.w < w1 && kb < c.nb && c.I != kb && c.J != kb;
}

template <class V>
__global__ void __launch_bounds__(NTHREADS, 1) fw_phase3(MatSet<V> ms, uint32_t kb) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    V* sA = reinterpret_cast<V*>(smem_raw);
    V* sB0 = sA + TT;  // two B buffers: sB0, sB0 + TT
    __shared__ uint64_t bars[2];
    const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;

    const bool sparse = ms.act_flag != nullptr;
    const bool rowlist = !sparse && ms.rows != nullptr;
    const uint64_t total = sparse ? ms.mat_prefix[ms.nmat]
                                  : rowlist ? ms.row_prefix[ms.nrows] : ms.work_prefix[ms.nmat];
    const uint64_t per = (total + gridDim.x - 1) / gridDim.x;
    const uint64_t w0 = uint64_t(blockIdx.x) * per;
    const uint64_t w1 = min(total, w0 + per);
    if (w0 >= w1) return;

    P3Cursor cur;
    cur.w = w0;
    cur.m = 0;
    cur.ri = 0;
    if (sparse) {
        // matrix: the last m with mat_prefix[m] <= w0 (it has work, since
        // w0 < mat_prefix[m + 1]); then its row by the row prefix
        uint32_t lo = 0, hi = ms.nmat;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (ms.mat_prefix[mid] <= w0) lo = mid; else hi = mid;
        }
        p3_enter(ms, cur, lo);
        const uint64_t local = w0 - ms.mat_prefix[lo];
        const uint64_t* pre = ms.act_prefix + cur.sb + lo;
        uint32_t rlo = 0, rhi = cur.anr;
        while (rhi - rlo > 1) {
            const uint32_t mid = (rlo + rhi) / 2;
            if (pre[mid] <= local) rlo = mid; else rhi = mid;
        }
        cur.ri = rlo;
        cur.p = ms.act_rows[cur.sb + rlo];
        cur.q = cur.p + static_cast<uint32_t>(local - pre[rlo]);
        cur.I = ms.act_list[cur.sb + cur.p];
        cur.J = ms.act_list[cur.sb + cur.q];
    } else if (rowlist) {
        // owned rows only (multi-GPU boundary graph): binary search the row
        uint32_t lo = 0, hi = ms.nrows;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (ms.row_prefix[mid] <= w0) lo = mid; else hi = mid;
        }
        cur.ri = lo;
        cur.nb = ms.nb[0];
        cur.I = ms.rows[lo];
        cur.J = cur.I + static_cast<uint32_t>(w0 - ms.row_prefix[lo]);
    } else {
        // locate the first item: matrix by binary search, tile row by solving
        // row_start(I) <= t < row_start(I+1).
        uint32_t lo = 0, hi = ms.nmat;
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (ms.work_prefix[mid] <= w0) lo = mid; else hi = mid;
        }
        cur.m = lo;
        cur.nb = ms.nb[lo];
        const uint32_t nb = cur.nb;
        const uint32_t t = static_cast<uint32_t>(w0 - ms.work_prefix[lo]);
        const double b2 = 2.0 * nb + 1.0;
        double est = floor((b2 - sqrt(b2 * b2 - 8.0 * t)) * 0.5);
        uint32_t I = est < 0 ? 0u : static_cast<uint32_t>(est);
        if (I >= nb) I = nb - 1;
        while (I > 0 && row_start(I, nb) > t) --I;
        while (I + 1 < nb && row_start(I + 1, nb) <= t) ++I;
        cur.I = I;
        cur.J = I + (t - row_start(I, nb));
    }
    while (cur.w < w1 && !p3_valid<V>(cur, w1, kb)) p3_advance(ms, cur);
    if (cur.w >= w1) return;

    if (tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
    }
    __syncthreads();

    auto panel_of = [&](const P3Cursor& c) { return ms.panel + ms.panel_base[c.m]; };
    uint32_t parity[2] = {0, 0};
    int buf = 0;
    uint64_t a_key = (uint64_t(cur.m) << 32) | cur.I;
    if (tid == 0) {
        const V* P = panel_of(cur);
        mbar_expect_tx(&bars[0], 2u * TT * sizeof(V));
        bulk_g2s(sA, P + uint64_t(cur.I) * TT, TT * sizeof(V), &bars[0]);
        bulk_g2s(sB0, P + uint64_t(cur.J) * TT, TT * sizeof(V), &bars[0]);
    }
    while (cur.w < w1) {
        P3Cursor nxt = cur;
        do {
            p3_advance(ms, nxt);
        } while (nxt.w < w1 && !p3_valid<V>(nxt, w1, kb));
        const bool has_next = nxt.w < w1;
        const uint64_t next_key = (uint64_t(nxt.m) << 32) | nxt.I;
        const bool next_needs_a = has_next && next_key != a_key;
        V* sBcur = sB0 + buf * TT;
        V* sBnxt = sB0 + (buf ^ 1) * TT;
        // same tile row next: its B slot can stream in during this compute
        // (sBnxt was last read by the previous item, before its barrier)
        if (has_next && !next_needs_a && tid == 0) {
            fence_proxy_async();
            mbar_expect_tx(&bars[buf ^ 1], TT * sizeof(V));
            bulk_g2s(sBnxt, panel_of(nxt) + uint64_t(nxt.J) * TT, TT * sizeof(V), &bars[buf ^ 1]);
        }
        V* C = ms.tiles + ms.tile_base[cur.m] + tidx(cur.I, cur.J, cur.nb) * TT;
        V cr[8][8];
        load_block(C, cr, ty, tx);  // in flight during the product
        V acc[8][8];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = Ops<V>::inf();
        mbar_wait(&bars[buf], parity[buf]);
        parity[buf] ^= 1;
        minplus_tile<V, true>(sA, sBcur, acc, ty, tx);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[i][j] = Ops<V>::vmin(acc[i][j], cr[i][j]);
        store_block(C, acc, ty, tx);
        __syncthreads();  // all reads of sA / sBcur done
        if (next_needs_a && tid == 0) {
            const V* P = panel_of(nxt);
            fence_proxy_async();
            mbar_expect_tx(&bars[buf ^ 1], 2u * TT * sizeof(V));
            bulk_g2s(sA, P + uint64_t(nxt.I) * TT, TT * sizeof(V), &bars[buf ^ 1]);
            bulk_g2s(sBnxt, P + uint64_t(nxt.J) * TT, TT * sizeof(V), &bars[buf ^ 1]);
        }
        if (next_needs_a) a_key = next_key;
        cur = nxt;
        buf ^= 1;
    }
}

// ------------------------------------------------------------- K0: init --
template <class V>
__global__ void fill_value(V* __restrict__ p, uint64_t count, V value) {
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
        p[i] = value;
}

// grid: nmat CTAs. Zero diagonal incl. padding vertices.
template <class V>
__global__ void set_diag_zero(MatSet<V> ms) {
    const uint32_t m = blockIdx.x;
    const uint32_t nb = ms.nb[m];
    for (uint32_t v = threadIdx.x; v < nb * T; v += blockDim.x)
        ms.tiles[ms.tile_base[m] + tidx(v / T, v / T, nb) * TT + uint64_t(v % T) * T + v % T] = V(0);
}

// Symmetric scatter of weighted pairs (i, j) into matrix mat[e] (or 0).
template <class V>
__global__ void scatter_pairs(MatSet<V> ms, const uint32_t* __restrict__ mat,
                              const uint32_t* __restrict__ ii, const uint32_t* __restrict__ jj,
                              const V* __restrict__ w, uint64_t count) {
    const uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (e >= count) return;
    const uint32_t m = mat ? mat[e] : 0u;
    const uint32_t nb = ms.nb[m];
    V* base = ms.tiles + ms.tile_base[m];
    const uint32_t i = ii[e], j = jj[e];
    if (i / T <= j / T) base[tidx(i / T, j / T, nb) * TT + uint64_t(i % T) * T + j % T] = w[e];
    if (j / T <= i / T) base[tidx(j / T, i / T, nb) * TT + uint64_t(j % T) * T + i % T] = w[e];
}

// Phase 3 init, clique part (src/oracle.cpp:110-122): the |B(C)| x |B(C)|
// boundary prefix of every component table lands on the BG block diagonal;
// counts finite pairs i < j for BuildStats::bg_edges.
// grid: k CTAs, one component each (block-stride over its B x B block)
// pos[id] = where boundary id sits in the BG matrix (the id itself, or its
// K2 elimination-order position, bg_order.hpp).
template <class V>
__global__ void copy_boundary_blocks(MatSet<V> comps, const uint32_t* __restrict__ bnd_off,
                                     const uint32_t* __restrict__ pos, MatSet<V> bg,
                                     unsigned long long* clique_edges) {
    const uint32_t c = blockIdx.x;
    const uint32_t* p = pos + bnd_off[c];
    const uint32_t B = bnd_off[c + 1] - bnd_off[c];
    const uint64_t total = uint64_t(B) * B;
    uint32_t finite = 0;
    for (uint64_t base = 0; base < total; base += blockDim.x) {
        const uint64_t idx = base + threadIdx.x;
        if (idx < total) {
            const uint32_t i = static_cast<uint32_t>(idx / B), j = static_cast<uint32_t>(idx % B);
            const V val = comps.tiles[comps.tile_base[c] + sym_off(i, j, comps.nb[c])];
            const uint32_t gi = p[i], gj = p[j];
            if (gi / T <= gj / T)
                bg.tiles[tidx(gi / T, gj / T, bg.nb[0]) * TT + uint64_t(gi % T) * T + gj % T] = val;
            finite += (i < j && val < Ops<V>::inf()) ? 1u : 0u;
        }
    }
    const uint32_t warp_total = __reduce_add_sync(0xffffffffu, finite);
    if ((threadIdx.x & 31) == 0 && warp_total) atomicAdd(clique_edges, warp_total);
}

// R <- P with boundary ids restored: element (i, j) of R's upper tiles is
// P(pos[i], pos[j]) (pos = boundary id -> K2 position, bg_order.hpp; P has
// nbP >= nb tiles per side, the tile-packing padding);
// padding vertices are isolated (INF, 0 on the diagonal).
// grid: (nb, nb) CTAs, tile (I = y, J = x), lower ones exit.
template <class V>
__global__ void permute_sym(const V* __restrict__ P, uint32_t nbP, V* __restrict__ R, uint32_t nb,
                            uint32_t b, const uint32_t* __restrict__ pos) {
    const uint32_t I = blockIdx.y, J = blockIdx.x;
    if (I > J) return;
    V* out = R + tidx(I, J, nb) * TT;
    for (uint32_t e = threadIdx.x; e < uint32_t(TT); e += blockDim.x) {
        const uint32_t i = I * T + e / T, j = J * T + e % T;
        V v;
        if (i < b && j < b) v = P[sym_off(pos[i], pos[j], nbP)];
        else v = i == j ? V(0) : Ops<V>::inf();
        out[e] = v;
    }
}

// K1 elimination order (k1_order.hpp), undone: matrix g0 + z of the final
// component arena R gets element (i, j) = W_z(pos[i], pos[j]) of working
// matrix z (pos = pos_all + pos_off[z], the local vertex -> FW position
// map); padding vertices are isolated (INF, 0 on the diagonal).
// grid: (nb_max, nb_max, matrices), tile (I = y, J = x), others exit.
template <class V>
__global__ void permute_batch(MatSet<V> W, MatSet<V> R, uint32_t g0,
                              const uint32_t* __restrict__ pos_all,
                              const uint64_t* __restrict__ pos_off) {
    const uint32_t z = blockIdx.z, I = blockIdx.y, J = blockIdx.x;
    const uint32_t nb = W.nb[z];
    if (I > J || J >= nb) return;
    const uint32_t* pos = pos_all + pos_off[z];
    const uint32_t n = static_cast<uint32_t>(pos_off[z + 1] - pos_off[z]);
    const V* P = W.tiles + W.tile_base[z];
    V* out = R.tiles + R.tile_base[g0 + z] + tidx(I, J, nb) * TT;
    __shared__ uint32_t prow[T], pcol[T];
    for (uint32_t t = threadIdx.x; t < uint32_t(T); t += blockDim.x) {
        prow[t] = I * T + t < n ? pos[I * T + t] : UINT32_MAX;
        pcol[t] = J * T + t < n ? pos[J * T + t] : UINT32_MAX;
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < uint32_t(TT); e += blockDim.x) {
        const uint32_t r = e / T, c = e % T;
        const uint32_t pi = prow[r], pj = pcol[c];
        V v;
        if (pi != UINT32_MAX && pj != UINT32_MAX) v = P[sym_off(pi, pj, nb)];
        else v = (I * T + r == J * T + c) ? V(0) : Ops<V>::inf();
        out[e] = v;
    }
}

// Query side table CB[c] = rows 0..|C| of component c restricted to its
// boundary columns, |C| x cb_stride(|B(C)|) row-major (rows padded to a
// multiple of 4 with INF so each row starts 16-byte aligned): row1/col2 of
// Algorithm 2 (src/query.cpp:29-45) become contiguous, vector-loadable
// reads.  grid: k CTAs
template <class V>
__global__ void extract_to_boundary(MatSet<V> comps, const uint32_t* __restrict__ comp_off,
                                    const uint32_t* __restrict__ bnd_off,
                                    const uint64_t* __restrict__ cb_off, V* __restrict__ cb) {
    const uint32_t c = blockIdx.x;
    const uint32_t S = comp_off[c + 1] - comp_off[c];
    const uint32_t B = bnd_off[c + 1] - bnd_off[c];
    const uint32_t Bp = cb_stride(B);  // rows padded to 16 bytes with INF
    const uint64_t total = uint64_t(S) * Bp;
    for (uint64_t idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const uint32_t l = static_cast<uint32_t>(idx / Bp), j = static_cast<uint32_t>(idx % Bp);
        cb[cb_off[c] + idx] =
            j < B ? comps.tiles[comps.tile_base[c] + sym_off(l, j, comps.nb[c])] : Ops<V>::inf();
    }
}

// Dense import of a row window of matrix m (rows row0.., columns 0..ncols):
// writes element (i, j) iff its tile is in the stored upper triangle.
template <class V>
__global__ void pack_window(MatSet<V> ms, uint32_t m, uint32_t row0, uint32_t nrows,
                            uint32_t ncols, const V* __restrict__ dense) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(nrows) * ncols) return;
    const uint32_t i = row0 + static_cast<uint32_t>(idx / ncols);
    const uint32_t j = static_cast<uint32_t>(idx % ncols);
    if (i / T <= j / T)
        ms.tiles[ms.tile_base[m] + tidx(i / T, j / T, ms.nb[m]) * TT + uint64_t(i % T) * T + j % T] =
            dense[idx];
}

// Dense export of a row/column window of matrix m: out[r][c] = D[row0+r][col0+c].
template <class V>
__global__ void unpack_window(MatSet<V> ms, uint32_t m, uint32_t row0, uint32_t nrows,
                              uint32_t col0, uint32_t ncols, V* __restrict__ out) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(nrows) * ncols) return;
    const uint32_t r = static_cast<uint32_t>(idx / ncols), c = static_cast<uint32_t>(idx % ncols);
    out[idx] = ms.tiles[ms.tile_base[m] + sym_off(row0 + r, col0 + c, ms.nb[m])];
}

// ------------------------------------------------------ ALU peak probe ----
// The phase-3 inner loop without memory: 64 independent add-min chains per
// thread, operands rotated through the accumulators so nothing folds.
template <class V>
__global__ void __launch_bounds__(NTHREADS) minplus_peak_kernel(V* out, uint32_t iters, V seed) {
    // the FW / query inner loop's mix: 8x8 accumulators, k taken in pairs
    // through addmin2 (2 x VIADDMNMX for u32; FADD, FADD, FMNMX3 for f32),
    // 128 relaxations per thread per iteration. The operand rotation is
    // tools/minplus_probe.cu's, whose register allocation reaches the
    // highest f32 rate found (profiles/r1_minplus_peak.json).
    V acc[8][8];
    V a0[8], b0[8], a1[8], b1[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a0[i] = seed + V(threadIdx.x & 7) + V(i);
        b0[i] = seed + V(i * 3);
        a1[i] = seed + V(i + 1);
        b1[i] = seed + V(2 * i);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = seed + V(1000 + i * 8 + j);
    }
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j)
                acc[i][j] = Ops<V>::addmin2(a0[i], b0[j], a1[i], b1[j], acc[i][j]);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            a0[i] = acc[i][(i + 1) & 7];
            b0[i] = acc[(i + 3) & 7][i];
            a1[i] = acc[(i + 5) & 7][(i + 2) & 7];
            b1[i] = acc[(i + 6) & 7][(i + 7) & 7];
        }
    }
    V s = acc[0][0];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s = Ops<V>::vmin(s, acc[i][j]);
    if (s == V(12345)) out[blockIdx.x] = s;
}

}  // namespace pspg
