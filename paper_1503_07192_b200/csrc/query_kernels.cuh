// query_kernels.cuh — K3: batched distance queries (Algorithm 2).
//
// Replaces query / batch_query (src/query.cpp:29-114):
//   through[j] = min_i row1[i] + BG[g1 + i][g2 + j]     (stitch_into :49-59)
//   d          = min_j through[j] + col2[j]             (min_plus_combine :61-65)
//   d          = min(d, CT[c1](l1, l2)) if c1 == c2     (finish :70-72)
//
// Undirected symmetry (dist(v,w) = dist(w,v), tests/test_query.cpp:144-153)
// turns every query around so that c1 <= c2: the B1 x B2 block
// BG[g1.., g2..] then lies in the stored upper triangle (g1 + B1 <= g2 when
// c1 < c2). In u32 the result is exact either way; in f32 the three-term sums
// may round differently, which the 1e-5 tolerance covers.
//
// Kernels:
//  * query_grouped (batches above 16K pairs): queries are grouped by the
//    component pair (c1, c2); one warp takes up to 32 queries of one pair x
//    one 32-column group and streams that block through shared memory ONCE
//    for all of them, as a register-blocked min-plus product followed by
//    the combine with col2. HBM traffic drops from B1*B2*4 bytes per query
//    to per (pair, 32 queries); the kernel is then bound by the min-plus
//    ALU rate.
//  * query_cta (batches up to 16K pairs, no grouping pass): one CTA per
//    query over the same block layout; latency-bound, so shaped for
//    residency (64 warps per SM).
//  * query_server: one resident CTA answering point queries from a mailbox
//    in mapped host memory (no launch per call).
//  * query_warp (PSP_QUERY_KERNEL=warp, k^2 past 31-bit keys): one warp per
//    query, lanes own target columns, every row segment of the block is
//    fetched by the whole warp at once so DRAM sees full segments.
#pragma once
#include "fw_kernels.cuh"  // mbarrier / bulk-copy helpers
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
    uint32_t k;
    uint32_t n;                 // vertex count: ids >= n are rejected
    uint32_t* bad_id;           // set to 1 when a query id is out of range
    double scale;               // 2^-q (u32 fixed point) or 1
    // routed (sharded) mode only, see engine_shard.cuh: this rank holds the
    // full boundary rows of the components it owns, dense row-major; `cb`
    // is its own compact to-boundary arena and cb_peer[r] rank r's, mapped
    // over NVLink; cb_off[c] is c's offset in its owner's arena
    const V* bt;                // [owned boundary rows][bt_stride]
    uint64_t bt_stride;         // >= b, multiple of 4
    const uint32_t* bt_row0;    // k: first local BT row of an owned component
    const uint32_t* owner;      // k: rank owning component c
    const V* const* cb_peer;    // world: every rank's compact CB arena
    // block query layout (optional, engine_oracle.cuh build_query_blocks):
    // block (c1 <= c2) at bq + bq_off[c1 * k + c2], stored [cg][B1p][32]
    // with B1p = B1 rounded up to GK, INF padding rows and columns
    const V* bq;
    const uint64_t* bq_off;
    // 16-bit residual layout (u32 tables, QM_BLOCKS16): block (c1 <= c2) of
    // saturated residuals at bq16 + bq16_off[c1 * k + c2] ([cg][B1p][32]
    // u16), its potentials at bqaux + aux_off[c1 * k + c2] (bqaux_words:
    // 4 reserved, a[B1p], b[ncg*32]). cb16 / cb16_off / rbase: unused (null)
    const uint16_t* bq16;
    const uint64_t* bq16_off;
    const uint32_t* bqaux;
    const uint64_t* aux_off;
    const uint16_t* cb16;
    const uint64_t* cb16_off;
    const uint32_t* rbase;
    uint32_t u16_sat;           // saturation S (U16_SAT; smaller only to test the fallback)
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
__device__ __forceinline__ V same_component_entry(const QueryView<V>& q, uint32_t c,
                                                  uint32_t l1, uint32_t l2) {
    return q.comps.tiles[q.comps.tile_base[c] + sym_off(l1, l2, q.comps.nb[c])];
}

// Resolve a query to (c1 <= c2, l1, l2); routed mode keeps the caller's
// orientation (the query executes at owner(C1), src/cluster.cpp:88-90).
// Where a task's B1 x B2 block comes from (template parameter of the
// grouped kernel): the FW's tile-packed symmetric arena, the dense owned
// rows of a routed shard, or the block query layout (one contiguous 2 KB
// bulk copy per 16-row chunk).
// QM_BLOCKS_LANE / QM_BLOCKS_8X8 are the block layout with earlier products
// (PSP_QUERY_PRODUCT=lane|8x8, kept for A/B measurement).
// QM_BLOCKS16: the 16-bit residual block layout (u32 tables only, see the
// "16-bit residual product" section below).
enum QueryMode : int { QM_TILES = 0, QM_ROUTED = 1, QM_BLOCKS = 2, QM_BLOCKS_LANE = 3, QM_BLOCKS_8X8 = 4,
                       QM_BLOCKS16 = 5 };

template <class V, bool ROUTED = false>
__device__ __forceinline__ void resolve(const QueryView<V>& q, uint32_t v1, uint32_t v2,
                                        uint32_t& c1, uint32_t& c2, uint32_t& l1, uint32_t& l2) {
    // src/query.cpp:30: out-of-range ids invalidate the batch (the host API
    // reports PSP_EINVAL); the query is answered as (0, 0) meanwhile
    if (v1 >= q.n || v2 >= q.n) {
        if (q.bad_id) *q.bad_id = 1u;
        v1 = v2 = 0;
    }
    uint32_t r1 = q.perm[v1], r2 = q.perm[v2];
    c1 = q.assign[r1];
    c2 = q.assign[r2];
    if (!ROUTED && c1 > c2) {
        uint32_t t = r1; r1 = r2; r2 = t;
        t = c1; c1 = c2; c2 = t;
    }
    l1 = r1 - q.comp_off[c1];
    l2 = r2 - q.comp_off[c2];
}

// ---------------------------------------------------- sparse: warp/query --
// One warp per query. Lanes own target columns (a window of 32 x WQ_SLOTS);
// source rows are walked in chunks of 32 with row1 broadcast by SHFL, and
// rows are unrolled by 4 so 4 x WQ_SLOTS independent row-segment loads are
// in flight per warp (each a full 128-byte row segment of the block).
constexpr int WQ_SLOTS = 8;  // 256 target boundary columns per window
constexpr int GK = 16;        // rows per staged chunk (grouped kernel) = block-layout row padding

// One lane's partial answer of a resolved query over the source-row chunks
// i0 = row0, row0 + rstep, ... (32 rows each): min over those rows b1 and the
// lane's target columns j of row1[b1] + BG[b1][j] + col2[j]. Taking the min
// over all lanes (and over row splits) gives Algorithm 2's stitch
// (src/query.cpp:49-65) exactly, in any split: min distributes over +, and
// the f32 rounding of x + col2[j] is monotone in x.
template <class V>
__device__ __forceinline__ V warp_partial(const QueryView<V>& q, uint32_t c1, uint32_t c2,
                                          uint32_t l1, uint32_t l2, uint32_t row0,
                                          uint32_t rstep) {
    const int lane = threadIdx.x & 31;
    const uint32_t nb = q.bg_nb;
    const uint32_t g1 = q.bnd_off[c1], B1 = q.bnd_off[c1 + 1] - g1;
    const uint32_t g2 = q.bnd_off[c2], B2 = q.bnd_off[c2 + 1] - g2;
    const V* row1 = q.cb + q.cb_off[c1] + uint64_t(l1) * cb_stride(B1);
    const V* col2 = q.cb + q.cb_off[c2] + uint64_t(l2) * cb_stride(B2);
    V best = Ops<V>::inf();
    for (uint32_t j0 = 0; j0 < B2; j0 += 32 * WQ_SLOTS) {
        const uint32_t nslot = min(uint32_t(WQ_SLOTS), (B2 - j0 + 31) / 32);
        V acc[WQ_SLOTS];
#pragma unroll
        for (int s = 0; s < WQ_SLOTS; ++s) acc[s] = Ops<V>::inf();
        for (uint32_t i0 = row0; i0 < B1; i0 += rstep) {
            const uint32_t ni = min(32u, B1 - i0);
            const V rv = (uint32_t(lane) < ni) ? row1[i0 + lane] : Ops<V>::inf();
            const uint32_t gi0 = g1 + i0;
            if (c1 != c2) {
                // rows gi0.. span at most two tile rows (32 < T): per slot
                // a pointer for each, p1 pre-shifted so p[t * T] works
                const uint32_t I0 = gi0 >> 7, split = T - (gi0 & (T - 1));
                const V* p0[WQ_SLOTS];
                const V* p1[WQ_SLOTS];
#pragma unroll
                for (int s = 0; s < WQ_SLOTS; ++s) {
                    const uint32_t gj = g2 + min(j0 + s * 32 + lane, B2 - 1);
                    const uint32_t Jt = gj >> 7;
                    p0[s] = q.bg + tidx(I0, Jt, nb) * TT + uint64_t(gi0 & (T - 1)) * T + (gj & (T - 1));
                    p1[s] = (I0 + 1 <= Jt) ? q.bg + tidx(I0 + 1, Jt, nb) * TT + (gj & (T - 1)) -
                                                 uint64_t(split) * T
                                           : p0[s];
                }
                for (uint32_t t0 = 0; t0 < ni; t0 += 4) {
#pragma unroll
                    for (uint32_t dt = 0; dt < 4; ++dt) {
                        const uint32_t t = t0 + dt;
                        const V r = __shfl_sync(0xffffffffu, rv, t & 31);
                        if (t < ni) {
#pragma unroll
                            for (int s = 0; s < WQ_SLOTS; ++s)
                                if (uint32_t(s) < nslot)
                                    acc[s] = Ops<V>::addmin(r, (t < split ? p0[s] : p1[s])[t * T], acc[s]);
                        }
                    }
                }
            } else {  // diagonal block: both triangles, generic lookup
                for (uint32_t t = 0; t < ni; ++t) {
                    const V r = __shfl_sync(0xffffffffu, rv, t);
#pragma unroll
                    for (int s = 0; s < WQ_SLOTS; ++s)
                        if (uint32_t(s) < nslot) {
                            const uint32_t gj = g2 + min(j0 + s * 32 + lane, B2 - 1);
                            acc[s] = Ops<V>::addmin(r, q.bg[sym_off(gi0 + t, gj, nb)], acc[s]);
                        }
                }
            }
        }
#pragma unroll
        for (int s = 0; s < WQ_SLOTS; ++s) {
            const uint32_t j = j0 + s * 32 + lane;
            if (uint32_t(s) < nslot && j < B2) best = Ops<V>::addmin(acc[s], col2[j], best);
        }
    }
    return best;
}

template <class V>
__global__ void __launch_bounds__(256) query_warp(QueryView<V> q, const uint32_t* __restrict__ v1,
                                                  const uint32_t* __restrict__ v2, uint64_t count,
                                                  double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    for (uint64_t qi = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; qi < count;
         qi += nwarps) {
        uint32_t c1, c2, l1, l2;
        resolve(q, v1[qi], v2[qi], c1, c2, l1, l2);
        V best = warp_min<V>(warp_partial(q, c1, c2, l1, l2, 0, 32));
        if (lane == 0) {
            if (c1 == c2) best = Ops<V>::vmin(best, same_component_entry(q, c1, l1, l2));
            out[qi] = Ops<V>::to_f64(best, q.scale);
        }
    }
}

// ------------------------------------------- small batches: CTA/query --
// One CTA (QC_WARPS warps; QC_BATCH_WARPS for batches, below) per query, for
// batches far smaller than k^2 (no
// pair reuse to gain, no sort to pay) and for the point-query server, where
// latency rules: the warps take interleaved 4-row groups of the B1 source
// rows (warp w: rows 4w..4w+3, 4w+32.., ...), lanes take target columns (up
// to WQ_SLOTS per lane), so a 60 x 60 block is fetched in two rounds of
// independent loads. Min distributes over + and f32 rounding of x + col2 is
// monotone in x, so any split of rows and columns gives Algorithm 2's value
// exactly (src/query.cpp:49-65). Result on thread 0.
constexpr int QC_WARPS = 8;

template <class V, int UNR = 8>
__device__ __forceinline__ double cta_query(const QueryView<V>& q, uint32_t v1, uint32_t v2,
                                            V* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t c1, c2, l1, l2;
    resolve(q, v1, v2, c1, c2, l1, l2);
    const uint32_t nb = q.bg_nb;
    const uint32_t g1 = q.bnd_off[c1], B1 = q.bnd_off[c1 + 1] - g1;
    const uint32_t g2 = q.bnd_off[c2], B2 = q.bnd_off[c2 + 1] - g2;
    const V* row1 = q.cb + q.cb_off[c1] + uint64_t(l1) * cb_stride(B1);
    const V* col2 = q.cb + q.cb_off[c2] + uint64_t(l2) * cb_stride(B2);
    // every load below depends only on the resolved ids: issue the
    // same-component entry and the lane's col2 values before the block rows
    // so that one memory round trip covers them all (point-query latency)
    V same = Ops<V>::inf();
    if (c1 == c2 && threadIdx.x == 0) same = same_component_entry(q, c1, l1, l2);
    V best = Ops<V>::inf();
    if (q.bq) {
        // block query layout, block (c1 <= c2) stored [cg][B1p][32]: thread
        // t owns a quad of 4 adjacent columns (16-byte loads, a warp reads
        // 4 full 128-byte row segments) and the rows of one phase
        // (r = phase, phase + nphase, ...), so every load of the block is
        // independent and a whole block arrives in ~B1 / nphase / 4 rounds;
        // each thread adds col2 to its own partial minima (min distributes)
        const uint32_t B1p = (B1 + GK - 1) / GK * GK;
        const uint32_t ncg = (B2 + 31) / 32, nquad = ncg * 8;
        const uint32_t nt = blockDim.x;
        const uint32_t nphase = nquad >= nt ? 1u : nt / nquad;
        const V* bb = q.bq + q.bq_off[c1 * q.k + c2];
        for (uint32_t t = threadIdx.x; t < nquad * nphase; t += nt) {
            const uint32_t quad = t % nquad, phase = t / nquad;
            const uint32_t cg = quad >> 3, j = cg * 32 + (quad & 7) * 4;
            V cv[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) cv[u] = j + u < B2 ? col2[j + u] : Ops<V>::inf();
            const V* col = bb + uint64_t(cg) * B1p * 32 + (quad & 7) * 4;
            V acc[4] = {Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf()};
#pragma unroll UNR
            for (uint32_t r = phase; r < B1; r += nphase) {
                const V a = row1[r];
                const uint4 m = *reinterpret_cast<const uint4*>(col + uint64_t(r) * 32);
                acc[0] = Ops<V>::addmin(a, Ops<V>::from_bits(m.x), acc[0]);
                acc[1] = Ops<V>::addmin(a, Ops<V>::from_bits(m.y), acc[1]);
                acc[2] = Ops<V>::addmin(a, Ops<V>::from_bits(m.z), acc[2]);
                acc[3] = Ops<V>::addmin(a, Ops<V>::from_bits(m.w), acc[3]);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) best = Ops<V>::addmin(acc[u], cv[u], best);
        }
    } else {
        for (uint32_t j0 = 0; j0 < B2; j0 += 32 * WQ_SLOTS) {
            const uint32_t nslot = min(uint32_t(WQ_SLOTS), (B2 - j0 + 31) / 32);
            V acc[WQ_SLOTS], cv[WQ_SLOTS];
            #pragma unroll
            for (int s = 0; s < WQ_SLOTS; ++s) {
                const uint32_t j = j0 + s * 32 + lane;
                acc[s] = Ops<V>::inf();
                cv[s] = (uint32_t(s) < nslot && j < B2) ? col2[j] : Ops<V>::inf();
            }
            for (uint32_t r0 = 4u * warp; r0 < B1; r0 += 4u * (blockDim.x >> 5)) {
                #pragma unroll
                for (uint32_t dr = 0; dr < 4; ++dr) {
                    const uint32_t r = r0 + dr;
                    if (r < B1) {
                        const V a = row1[r];
                        const uint32_t gi = g1 + r;
                        #pragma unroll
                        for (int s = 0; s < WQ_SLOTS; ++s) {
                            const uint32_t j = j0 + s * 32 + lane;
                            if (uint32_t(s) < nslot && j < B2) {
                                const uint32_t gj = g2 + j;
                                // c1 < c2: gi < gj, tile (gi/T, gj/T) is stored
                                const V m = c1 != c2 ? q.bg[tidx(gi >> 7, gj >> 7, nb) * TT +
                                                            uint64_t(gi & (T - 1)) * T + (gj & (T - 1))]
                                                     : q.bg[sym_off(gi, gj, nb)];
                                acc[s] = Ops<V>::addmin(a, m, acc[s]);
                            }
                        }
                    }
                }
            }
            #pragma unroll
            for (int s = 0; s < WQ_SLOTS; ++s) best = Ops<V>::addmin(acc[s], cv[s], best);
        }
    }
    best = warp_min<V>(best);
    if (lane == 0) red[warp] = best;
    __syncthreads();
    double out = 0.0;
    if (threadIdx.x == 0) {
        V b = red[0];
        for (uint32_t w = 1; w < (blockDim.x >> 5); ++w) b = Ops<V>::vmin(b, red[w]);
        out = Ops<V>::to_f64(Ops<V>::vmin(b, same), q.scale);
    }
    __syncthreads();  // red is reused by the next query
    return out;
}

// Batch kernel: NW warps per CTA, UNR rows of independent loads in flight
// per thread, MINB CTAs per SM. The batch is latency-bound (a chain of
// dependent id/offset loads, then a few rounds of block-row loads per
// thread), so residency decides: 16 warps x 4 CTAs (64 warps per SM, 32
// registers) runs 44.3 M queries/s at 1K pairs on cfg3 against 24.3 M for
// 8 warps at 70 registers (3 CTAs per SM, 2.25 waves) and 19.0 M at 90
// (profiles/r2/query_cta_shapes_cfg3.jsonl: 17 shapes).
constexpr int QC_BATCH_WARPS = 16, QC_BATCH_MINB = 4;
template <class V, int NW, int UNR, int MINB = 1>
__global__ void __launch_bounds__(32 * NW, MINB) query_cta(QueryView<V> q, const uint32_t* __restrict__ v1,
                                                     const uint32_t* __restrict__ v2, uint64_t count,
                                                     double* __restrict__ out) {
    __shared__ V red[NW];
    for (uint64_t qi = blockIdx.x; qi < count; qi += gridDim.x) {
        const double d = cta_query<V, UNR>(q, v1[qi], v2[qi], red);
        if (threadIdx.x == 0) out[qi] = d;
    }
}

// ------------------------------------------------ point-query server --
// Host API calls with a handful of pairs (the reference's query(o, v1, v2)
// called in a loop, e.g. acceptance criterion 1: 18.3M single queries) are
// latency-bound: a launch + stream sync per call costs more than the query.
// One resident CTA instead polls a mailbox in mapped pinned host memory and
// answers with cta_query. Every 8-byte word of a request or answer carries
// the request number in its top 16 bits (as NCCL's LL protocol does), so a
// word is valid on its own, and the first pair and the pair count share one
// 16-byte line: one PCIe read per poll fetches a whole single-pair request.
// Two polls stay in flight (tools/pcie_probe: a host<->GPU ping-pong takes
// 2.3 us with one poll, 2.0 us with two, 3.6 us with four). After idle_ns
// without a request the CTA clears `alive` and exits (device-wide syncs
// elsewhere never wait on it for long); the host relaunches it on demand.
//   req[0] = seq << 48 | count << 32 | v1_0     req[2i]   = seq << 48 | v1_i
//   req[1] = seq << 48 | v2_0                    req[2i+1] = seq << 48 | v2_i
//   ans[2i] = seq << 48 | low 32 bits of dist_i, ans[2i+1] = seq << 48 | high 32
//   ans[2 count] = seq << 48 | bad-id flag
constexpr int MAILBOX_PAIRS = 32;
struct __align__(16) QueryMailbox {
    volatile unsigned long long req[2 * MAILBOX_PAIRS];
    volatile unsigned long long ans[2 * MAILBOX_PAIRS + 2];
    volatile uint32_t alive;                  // device: server loop running
    uint32_t pad_;
    volatile unsigned long long prof[2];      // globaltimer: request seen, answered
};
__host__ __device__ inline uint32_t mb_tag(unsigned long long w) { return uint32_t(w >> 48); }

__device__ __forceinline__ unsigned long long global_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ void ld_sys_v2(const volatile unsigned long long* p,
                                          unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.volatile.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// Shared-memory copy of the id maps and per-component offsets the server
// reads first on every query (perm, assign, comp_off, bnd_off, cb_off and the
// component tables' tile_base / nb): a query then starts with shared-memory
// lookups instead of four dependent global loads. Taken when they fit
// (server_smem_bytes != 0).
__host__ __device__ inline size_t server_smem_bytes(uint64_t n, uint32_t k) {
    // cb_off + tile_base (u64), perm + assign (u32 x n), comp_off + bnd_off
    // (u32 x k+1), nb (u32)
    const size_t b = 16 * uint64_t(k) + 8 * n + 8 * (uint64_t(k) + 1) + 4 * uint64_t(k);
    return b <= (size_t(192) << 10) ? (b + 15) / 16 * 16 : 0;
}

template <class V>
__global__ void __launch_bounds__(32 * QC_WARPS) query_server(QueryView<V> q, QueryMailbox* mb,
                                                              uint32_t last_seq,
                                                              unsigned long long idle_ns,
                                                              int cache) {
    __shared__ V red[QC_WARPS];
    __shared__ uint32_t s_v[2 * MAILBOX_PAIRS], s_count, s_seq;
    __shared__ int s_stop;
    __shared__ double s_out[MAILBOX_PAIRS];
    extern __shared__ __align__(16) unsigned char srv_smem[];
    if (cache) {
        const uint32_t n = q.n, k = q.k, nt = blockDim.x;
        uint64_t* cbo = reinterpret_cast<uint64_t*>(srv_smem);
        uint64_t* tb = cbo + k;
        uint32_t* perm = reinterpret_cast<uint32_t*>(tb + k);
        uint32_t* asg = perm + n;
        uint32_t* co = asg + n;
        uint32_t* bo = co + (k + 1);
        uint32_t* nbm = bo + (k + 1);
        for (uint32_t i = threadIdx.x; i < n; i += nt) {
            perm[i] = q.perm[i];
            asg[i] = q.assign[i];
        }
        for (uint32_t i = threadIdx.x; i <= k; i += nt) {
            co[i] = q.comp_off[i];
            bo[i] = q.bnd_off[i];
            if (i < k) {
                cbo[i] = q.cb_off[i];
                tb[i] = q.comps.tile_base[i];
                nbm[i] = q.comps.nb[i];
            }
        }
        __syncthreads();
        q.perm = perm, q.assign = asg, q.comp_off = co, q.bnd_off = bo, q.cb_off = cbo;
        q.comps.tile_base = tb, q.comps.nb = nbm;
    }
    uint32_t last = last_seq;
    if (threadIdx.x == 0) {
        mb->alive = 1u;
        __threadfence_system();
    }
    unsigned long long t_idle = global_ns();
    for (;;) {
        if (threadIdx.x == 0) {
            s_stop = 0;
            // a request is taken from one poll (req[0..1]: tag, count and the
            // first pair); further pairs, if any, are read after
            auto take = [&](unsigned long long w0, unsigned long long w1) -> bool {
                const uint32_t seq = mb_tag(w0);
                if (seq == last || mb_tag(w1) != seq) return false;
                const uint32_t cnt = max(1u, min((uint32_t(w0 >> 32) & 0xffffu), uint32_t(MAILBOX_PAIRS)));
                s_v[0] = uint32_t(w0);
                s_v[1] = uint32_t(w1);
                for (uint32_t i = 1; i < cnt; ++i) {
                    unsigned long long x, y;
                    ld_sys_v2(&mb->req[2 * i], x, y);
                    if (mb_tag(x) != seq || mb_tag(y) != seq) return false;  // still landing
                    s_v[2 * i] = uint32_t(x);
                    s_v[2 * i + 1] = uint32_t(y);
                }
                s_count = cnt;
                s_seq = seq;
                return true;
            };
            // two polls in flight, about half a PCIe round trip apart (the
            // loop consumes and reissues them in turn, so it keeps that
            // spacing by itself)
            unsigned long long a0, a1, b0, b1;
            ld_sys_v2(&mb->req[0], a0, a1);
            __nanosleep(500);
            ld_sys_v2(&mb->req[0], b0, b1);
            for (;;) {
                if (take(a0, a1)) break;
                ld_sys_v2(&mb->req[0], a0, a1);
                if (take(b0, b1)) break;
                ld_sys_v2(&mb->req[0], b0, b1);
                if (global_ns() - t_idle > idle_ns) {
                    mb->alive = 0u;
                    __threadfence_system();
                    unsigned long long h, w0;
                    ld_sys_v2(&mb->req[0], h, w0);
                    if (mb_tag(h) == last) {
                        s_stop = 1;
                        break;
                    }
                    mb->alive = 1u;  // a request raced the exit
                }
            }
        }
        __syncthreads();
        if (s_stop) return;
        const unsigned long long t_seen = global_ns();
        const uint32_t seq = s_seq, cnt = s_count;
        uint32_t bad = 0;
        for (uint32_t i = 0; i < cnt; ++i) {
            const uint32_t a = s_v[2 * i], b = s_v[2 * i + 1];
            if (a >= q.n || b >= q.n) bad = 1;
            const double d = cta_query(q, a < q.n ? a : 0u, b < q.n ? b : 0u, red);
            if (threadIdx.x == 0) s_out[i] = d;
        }
        __syncthreads();
        // answers: lanes of warp 0 write one word each (posted PCIe writes)
        if (threadIdx.x < 32) {
            const unsigned long long tag = (unsigned long long)seq << 48;
            for (uint32_t w = threadIdx.x; w < 2 * cnt + 1; w += 32) {
                unsigned long long val;
                if (w == 2 * cnt) {
                    val = bad;
                } else {
                    const unsigned long long bits = __double_as_longlong(s_out[w >> 1]);
                    val = (w & 1) ? (bits >> 32) : (bits & 0xffffffffull);
                }
                mb->ans[w] = tag | val;
            }
            if (threadIdx.x == 0) {
                mb->prof[0] = t_seen;
                mb->prof[1] = global_ns();
            }
        }
        last = seq;
        t_idle = global_ns();
        __syncthreads();
    }
}

// ------------------------------------------- dense: grouped by (c1, c2) --
// Scheduling unit = one WARP TASK (item, column group): an item is up to 32
// queries of one component pair (c1 <= c2); a column group is 32 consecutive
// target boundary columns j of that pair. Lane = column. Each lane streams
// its own column of the B1 x B2 block straight from HBM/L2 (a warp reads one
// 128-byte row segment per load), and keeps one accumulator per query. The
// queries' row1 values for a 32-row chunk are staged once per warp in shared
// memory with an XOR swizzle (word (kk, q) at column q ^ (kk & 7)) that the
// compute reads as LDS.128 broadcasts at compile-time offsets (the row loop
// is unrolled by 8). Per row: Q/4 LDS.128 +
// Q VIADDMNMX for Q queries (Q = m rounded up to 4, templated), no padding
// in the query or row dimensions. Partial results of the column groups of a
// query meet in a global atomicMin (value bits are order-preserving: all
// distances are >= 0), a last tiny kernel applies the same-component cap.
constexpr int GQ = 32;           // queries per item (= max Q)
constexpr int GWARPS = 8;        // warps per CTA
constexpr int GTHREADS = 32 * GWARPS;

// Per-batch workspace (device pointers), all sized by the caller.
struct GroupWork {
    uint32_t* key;        // [count] c1 * k + c2
    uint32_t* l1;         // [count]
    uint32_t* l2;         // [count]
    uint32_t* best;       // [count] running min (value bits)
    uint32_t* lb;         // [count] QM_BLOCKS16: smallest lower bound of a saturated column
    uint32_t* base16;     // [count] QM_BLOCKS16: min_i row1_i + a_i of the query's block
    uint32_t* fb_list;    // [count] QM_BLOCKS16: queries left to the u32 fallback
    uint32_t* fb_count;   // [1]
    uint32_t* sorted;     // [count] query ids ordered by key
    uint32_t* s_l1;       // [count] l1 in sorted order
    uint32_t* s_l2;       // [count] l2 in sorted order
    uint32_t* bin_cnt;    // [nbins + 1] counts, then reused as scatter cursors
    uint32_t* bin_start;  // [nbins + 1]
    uint32_t* task_cnt;   // [nbins + 1] warp tasks per bin
    uint32_t* task_start; // [nbins + 1]
    uint4* tasks;         // [max tasks] (c1, c2, first sorted query, m | cg << 8)
    uint32_t nbins;
    // sparse grouping (batches far smaller than k^2): the "bins" are the
    // runs of the radix-sorted keys, bin b holds pair bin_key[b]; null: the
    // bin index is the pair key itself
    const uint32_t* bin_key;
    uint32_t* idx;        // [count] iota for the sort's values
};

template <class V, bool ROUTED>
__global__ void group_prep(QueryView<V> q, const uint32_t* __restrict__ v1,
                           const uint32_t* __restrict__ v2, uint64_t count, GroupWork w) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    uint32_t c1, c2, l1, l2;
    resolve<V, ROUTED>(q, v1[i], v2[i], c1, c2, l1, l2);
    const uint32_t key = c1 * q.k + c2;
    w.key[i] = key;
    w.l1[i] = l1;
    w.l2[i] = l2;
    w.best[i] = Ops<V>::to_bits(Ops<V>::inf());
    if (w.lb) w.lb[i] = U32_INF;
    if (w.bin_key) w.idx[i] = static_cast<uint32_t>(i);  // sparse: sorted later
    else atomicAdd(&w.bin_cnt[key], 1u);
}

__global__ void group_tasks(GroupWork w, const uint32_t* __restrict__ bnd_off, uint32_t k) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b < w.nbins) {
        const uint32_t cnt = w.bin_cnt[b];
        if (cnt == 0) {  // (sparse: runs past the last are zero-filled)
            w.task_cnt[b] = 0;
            return;
        }
        const uint32_t c2 = (w.bin_key ? w.bin_key[b] : b) % k;
        const uint32_t B2 = bnd_off[c2 + 1] - bnd_off[c2];
        w.task_cnt[b] = ((cnt + GQ - 1) / GQ) * ((B2 + 31) / 32);
    } else if (b == w.nbins) {
        w.task_cnt[b] = 0;
    }
}

// one thread per bin writes the bin's complete (item, column group) task
// records, so a warp starts a task with one 16-byte load
__global__ void group_emit(GroupWork w, const uint32_t* __restrict__ bnd_off, uint32_t k, bool balanced) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= w.nbins) return;
    const uint32_t n = w.task_cnt[b];
    if (n == 0) return;
    const uint32_t key = w.bin_key ? w.bin_key[b] : b;
    const uint32_t c1 = key / k, c2 = key % k;
    const uint32_t B2 = bnd_off[c2 + 1] - bnd_off[c2], ncg = (B2 + 31) / 32;
    const uint32_t start = w.bin_start[b], end = w.bin_start[b + 1];
    // balanced (register-blocked block-layout product, queries in steps of
    // 4): the bin's queries split into items of near-equal size (e.g. 36 ->
    // 20 + 16 instead of 32 + 4), the same query slots, but no item is left
    // with a 1-query-group remainder, whose product has little instruction-
    // level parallelism for the same block traffic (items <= GQ, so
    // (items - 1) * mbig < queries). The lane products (8/16/32 slots) keep
    // full items.
    const uint32_t nq = end - start, items = (nq + GQ - 1) / GQ;
    const uint32_t mbig = balanced ? min(uint32_t(GQ), ((nq + items - 1) / items + 3) & ~3u) : uint32_t(GQ);
    uint4* out = w.tasks + w.task_start[b];
    for (uint32_t t = 0; t < n; ++t) {
        const uint32_t item = t / ncg, cg = t % ncg;
        const uint32_t q0 = start + item * mbig;
        const uint32_t m = min(mbig, end - q0);
        // bit 6: the pair's last column group holds <= 16 columns (the
        // register-blocked block-layout kernel then runs a 16-column task)
        const uint32_t half = (cg + 1 == ncg && B2 - cg * 32 <= 16) ? 1u : 0u;
        out[t] = make_uint4(c1, c2, q0, m | (half << 6) | (cg << 8));
    }
}

// sparse grouping: the radix sort already ordered the query ids
__global__ void group_scatter_sorted(uint64_t count, const uint32_t* __restrict__ order, GroupWork w) {
    const uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (p >= count) return;
    const uint32_t i = order[p];
    w.sorted[p] = i;
    w.s_l1[p] = w.l1[i];
    w.s_l2[p] = w.l2[i];
}

__global__ void group_scatter(uint64_t count, GroupWork w) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t key = w.key[i];
    const uint32_t pos = w.bin_start[key] + atomicAdd(&w.bin_cnt[key], 1u);
    w.sorted[pos] = static_cast<uint32_t>(i);
    w.s_l1[pos] = w.l1[i];
    w.s_l2[pos] = w.l2[i];
}

template <class V>
__device__ __forceinline__ void atomic_min_bits(uint32_t* p, V v) {
    atomicMin(p, Ops<V>::to_bits(v));  // non-negative: bit order == value order
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, bool valid) {
    // 4-byte asynchronous global->shared copy; invalid lanes zero-fill (their
    // values never reach a used accumulator)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem), "r"(valid ? 4 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Shared staging per warp and chunk (GK = 16 rows):
//   A [query][row]  : row1_q[k0 + kk], GK + 4 word rows (16-byte aligned, the
//                     lane-per-query async fill is 4-way conflicted at most)
//   B [row][column] : block rows for the 36-column, 16-byte-aligned superset
//                     [A0, A0 + 36) of this task's 32 columns starting at
//                     G0 = A0 + shift; lane j reads column shift + j.
// Rows past the block end hold INF in B (their A values are don't-care), so
// the compute never needs a row predicate; it walks rows in groups of 4,
// reading each query's 4 row values as one broadcast LDS.128.
constexpr int GA_STRIDE = GK + 4;  // 16-byte aligned rows, <= 4-way conflicted fill
constexpr int GB_STRIDE = 36;  // the 9 staged 4-column chunks, conflict-free reads

template <class V, int NQ4, int BSTRIDE>
__device__ __forceinline__ void group_chunk(const V* __restrict__ sA, const V* __restrict__ sB,
                                            V (&acc)[4 * NQ4], uint32_t rows4, uint32_t shift,
                                            int lane) {
    const V* bcol = sB + shift + lane;
    for (uint32_t k4 = 0; k4 < rows4; k4 += 4) {
        V b[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) b[r] = bcol[(k4 + r) * BSTRIDE];
#pragma unroll
        for (int qq = 0; qq < 4 * NQ4; ++qq) {
            const uint4 u = *reinterpret_cast<const uint4*>(sA + qq * GA_STRIDE + k4);
            acc[qq] = Ops<V>::addmin2(Ops<V>::from_bits(u.x), b[0], Ops<V>::from_bits(u.y), b[1],
                                      acc[qq]);
            acc[qq] = Ops<V>::addmin2(Ops<V>::from_bits(u.z), b[2], Ops<V>::from_bits(u.w), b[3],
                                      acc[qq]);
        }
    }
}

// Per-warp shared state: two staged chunks of A and B, the item's query
// ids and col2 row offsets.
// ------------------------------------------- 16-bit residual product --
// VIADDMNMX.U16x2 does two 16-bit relaxations per instruction at the u32
// instruction rate (profiles/r2/minplus_probe.json: 125.9 vs 62.1 relax /clk
// /SM), but its add wraps at 2^16. The stitch min_ij r_i + M_ij + c_j is
// rewritten with two-sided potentials of each pair block,
//   M_ij = a_i + R_ij + b_j,  a_i = min_j M_ij,  b_j = min_i (M_ij - a_i),
// so R >= 0 carries only what is not additive, and with the query's base
//   base = min_i (r_i + a_i)
// the product runs on 15-bit saturated offsets (S = 0x7FFF):
//   t16_j = min_i ( min(r_i + a_i - base, S) + min(R_ij, S) )  (< 2^16: no wrap).
// If t16_j < S the minimising term saturated nowhere, so t16_j is exact:
//   candidate t16_j + base + b_j + c_j. If t16_j >= S every term of column j
// is >= S, so S + base + b_j + c_j is a lower bound. A query whose best exact
// candidate is <= the smallest lower bound (or whose same-component entry
// is) is exact; the others are recomputed in u32 by query_fallback
// (tools/u16_feasibility.py --potentials: 2,117 of 2,117 sampled cfg3
// queries settle). u32 tables only: u32 fixed point is exact integer
// arithmetic; f32 keeps the 32-bit product.
constexpr uint32_t U16_SAT = 0x7FFFu;
__host__ __device__ __forceinline__ uint32_t cb16_stride(uint32_t B) { return (B + 15u) & ~15u; }
// per block: [4 reserved][a: B1p u32][b: ncg*32 u32], 16-byte aligned
__host__ __device__ __forceinline__ uint64_t bqaux_words(uint32_t B1, uint32_t B2) {
    const uint32_t B1p = (B1 + GK - 1) / GK * GK, ncg = (B2 + 31) / 32;
    return 4 + B1p + uint64_t(ncg) * 32;
}

// One CTA per pair block (c1 <= c2): potentials, residuals, y16 offsets.
// dynamic smem: a[maxB1] + b[maxB2] (u32)
__global__ void __launch_bounds__(256) pack_query_blocks16(
    const uint32_t* __restrict__ bg, uint32_t nb, const uint32_t* __restrict__ bnd_off, uint32_t k,
    const uint64_t* __restrict__ blk_off, const uint64_t* __restrict__ aux_off,
    uint16_t* __restrict__ bq16, uint32_t* __restrict__ aux, uint32_t maxB, uint32_t sat) {
    const uint32_t c1 = blockIdx.x / k, c2 = blockIdx.x % k;
    if (c2 < c1) return;
    extern __shared__ uint32_t p16_smem[];
    uint32_t* sa = p16_smem;          // a_i
    uint32_t* sb = p16_smem + maxB;   // b_j
    __shared__ uint32_t s_amin;
    const uint32_t g1 = bnd_off[c1], B1 = bnd_off[c1 + 1] - g1;
    const uint32_t g2 = bnd_off[c2], B2 = bnd_off[c2 + 1] - g2;
    const uint32_t B1p = (B1 + GK - 1) / GK * GK, ncg = (B2 + 31) / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    auto M = [&](uint32_t i, uint32_t j) { return bg[sym_off(g1 + i, g2 + j, nb)]; };
    // a_i = min_j M_ij (a warp per row)
    for (uint32_t i = warp; i < B1; i += nw) {
        uint32_t m = U32_INF;
        for (uint32_t j = lane; j < B2; j += 32) m = min(m, M(i, j));
        m = __reduce_min_sync(0xffffffffu, m);
        if (lane == 0) sa[i] = m;
    }
    if (threadIdx.x == 0) s_amin = U32_INF;
    __syncthreads();
    // b_j = min_i (M_ij - a_i) over finite entries (a thread per column)
    for (uint32_t j = threadIdx.x; j < B2; j += blockDim.x) {
        uint32_t m = U32_INF;
        for (uint32_t i = 0; i < B1; ++i) {
            const uint32_t v = M(i, j), a = sa[i];
            if (v < U32_INF && a < U32_INF) m = min(m, v - a);
        }
        sb[j] = m;
    }
    {
        uint32_t m = U32_INF;
        for (uint32_t i = threadIdx.x; i < B1; i += blockDim.x) m = min(m, sa[i]);
        m = __reduce_min_sync(0xffffffffu, m);
        if (lane == 0) atomicMin(&s_amin, m);
    }
    __syncthreads();
    const uint32_t amin = s_amin;
    uint32_t* ax = aux + aux_off[blockIdx.x];
    if (threadIdx.x < 4) ax[threadIdx.x] = threadIdx.x == 0 ? amin : 0u;
    uint32_t* ai = ax + 4;
    for (uint32_t i = threadIdx.x; i < B1p; i += blockDim.x) ai[i] = i < B1 ? sa[i] : U32_INF;
    uint32_t* bj = ax + 4 + B1p;
    for (uint32_t j = threadIdx.x; j < ncg * 32; j += blockDim.x) bj[j] = j < B2 ? sb[j] : U32_INF;
    uint16_t* out = bq16 + blk_off[blockIdx.x];
    const uint64_t total = uint64_t(ncg) * B1p * 32;
    for (uint64_t idx = threadIdx.x; idx < total; idx += blockDim.x) {
        const uint64_t cg = idx / (uint64_t(B1p) * 32), rem = idx - cg * B1p * 32;
        const uint32_t r = uint32_t(rem >> 5), j = uint32_t(cg * 32 + (rem & 31));
        uint32_t v = sat;
        if (r < B1 && j < B2) {
            const uint32_t m = M(r, j), a = sa[r], b = sb[j];
            if (m < U32_INF && a < U32_INF && b < U32_INF) v = min(m - a - b, sat);
        }
        out[idx] = uint16_t(v);
    }
}

// Per to-boundary row (component c, local vertex l): rbase = min_i CB[l][i]
// and x16_i = min(CB[l][i] - rbase, S) (S where unreachable), a warp per row.
__global__ void __launch_bounds__(256) make_cb16(const uint32_t* __restrict__ cb,
                                                 const uint64_t* __restrict__ cb_off,
                                                 const uint32_t* __restrict__ comp_off,
                                                 const uint32_t* __restrict__ bnd_off,
                                                 const uint64_t* __restrict__ cb16_off,
                                                 uint16_t* __restrict__ cb16,
                                                 uint32_t* __restrict__ rbase, uint32_t sat) {
    const uint32_t c = blockIdx.x;
    const uint32_t S = comp_off[c + 1] - comp_off[c], B = bnd_off[c + 1] - bnd_off[c];
    const uint32_t Bp = cb_stride(B), Bp16 = cb16_stride(B);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (uint32_t l = warp; l < S; l += nw) {
        const uint32_t* row = cb + cb_off[c] + uint64_t(l) * Bp;
        uint32_t m = U32_INF;
        for (uint32_t i = lane; i < B; i += 32) m = min(m, row[i]);
        m = __reduce_min_sync(0xffffffffu, m);
        if (lane == 0) rbase[comp_off[c] + l] = m;
        uint16_t* x = cb16 + cb16_off[c] + uint64_t(l) * Bp16;
        for (uint32_t i = lane; i < Bp16; i += 32) {
            uint32_t v = sat;
            if (i < B && row[i] < U32_INF && m < U32_INF) v = min(row[i] - m, sat);
            x[i] = uint16_t(v);
        }
    }
}

template <class V> struct WarpStage {
    V a[2][GQ * GA_STRIDE];
    V b[2][GK * GB_STRIDE];
    V c2[GQ * 32];  // col2_q[j] per (query, lane), fetched at task start
    uint32_t id[GQ], c2off[GQ];
    uint64_t bar[2];  // QM_BLOCKS: completion of the B bulk copies
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(
                     static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
                 "l"(gmem), "r"(valid ? 16 : 0)
                 : "memory");
}

template <class V, int NQ4, int MODE>
__device__ __forceinline__ void group_task(const QueryView<V>& q, const GroupWork& w,
                                           WarpStage<V>* st, uint32_t c1, uint32_t c2,
                                           uint32_t q0, uint32_t m, uint32_t cg,
                                           uint32_t& phase) {
    constexpr bool ROUTED = MODE == QM_ROUTED;
    const int lane = threadIdx.x & 31;
    const uint32_t nb = q.bg_nb;
    const uint32_t g1 = q.bnd_off[c1], B1 = q.bnd_off[c1 + 1] - g1;
    const uint32_t g2 = q.bnd_off[c2], B2 = q.bnd_off[c2 + 1] - g2;
    const uint32_t Bp1 = cb_stride(B1), Bp2 = cb_stride(B2);
    const V* __restrict__ cb1 = q.cb + q.cb_off[c1];
    // routed: col2 comes from owner(C2)'s arena, a peer GPU's memory when
    // the owners differ (the paper's Alg. 2 line 8 transfer)
    const V* __restrict__ cb2 = (ROUTED ? q.cb_peer[q.owner[c2]] : q.cb) + q.cb_off[c2];
    const uint32_t j = cg * 32 + lane;
    const bool col_ok = j < B2;
    // 16-byte-aligned column superset of this task's 32 columns
    const uint32_t G0 = g2 + cg * 32, A0 = G0 & ~3u, shift = G0 - A0;
    const uint32_t Jlo = A0 >> 7;
    const V* bq_task = nullptr;  // QM_BLOCKS: this column group's [B1p][32] slab
    if (MODE == QM_BLOCKS)
        bq_task = q.bq + q.bq_off[c1 * q.k + c2] + uint64_t(cg) * ((B1 + GK - 1) / GK * GK) * 32;
    // this lane's staging slots for B: e = t*32 + lane -> (row kk, chunk u)
    // over the 32 x 9 chunks of 4 columns
    __syncwarp();
    const V* my_row1 = cb1;  // lane q: its query's row1 (16-byte aligned)
    if (uint32_t(lane) < m) {
        const uint32_t id = w.sorted[q0 + lane];
        st->id[lane] = id;
        st->c2off[lane] = w.s_l2[q0 + lane] * Bp2;
        my_row1 = cb1 + uint64_t(w.s_l1[q0 + lane]) * Bp1;
    }
    __syncwarp();

    auto issue = [&](uint32_t k0, int buf) {
        const uint32_t rows = min(uint32_t(GK), B1 - k0);
        V* sa = st->a[buf] + lane * GA_STRIDE;
        // A: lane q copies row1_q[k0 .. k0+32) (padding past Bp1 zero-fills;
        // those rows meet INF in B)
        if (uint32_t(lane) < m) {
#pragma unroll
            for (int t = 0; t < GK / 4; ++t) cp_async16(sa + 4 * t, my_row1 + k0 + 4 * t, k0 + 4 * t < Bp1);
        }
        V* sb = st->b[buf];
        if (MODE == QM_BLOCKS) {  // one contiguous 16 x 32 chunk of the block
            if (lane == 0) {
                fence_proxy_async();
                mbar_expect_tx(&st->bar[buf], GK * 32 * sizeof(V));
                bulk_g2s(sb, bq_task + uint64_t(k0) * 32, GK * 32 * sizeof(V), &st->bar[buf]);
            }
        } else if (ROUTED) {  // dense full rows of c1 (owned): any column block
            const V* rows0 = q.bt + uint64_t(q.bt_row0[c1] + k0) * q.bt_stride;
#pragma unroll
            for (int t = 0; t < (GK * 9 + 31) / 32; ++t) {
                const uint32_t e = t * 32 + lane;
                if (e >= uint32_t(GK * 9)) break;
                const uint32_t kk = e / 9, u = e - kk * 9;
                const uint32_t col = A0 + 4 * u;
                V* dst = sb + kk * GB_STRIDE + 4 * u;
                if (kk < rows && col < q.bt_stride) {
                    cp_async16(dst, rows0 + uint64_t(kk) * q.bt_stride + col, true);
                } else {
                    const V inf4[4] = {Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf()};
                    st4(dst, inf4);
                }
            }
        } else if (c1 != c2) {
            const uint32_t gi0 = g1 + k0;
            const uint32_t I0 = gi0 >> 7, r0 = gi0 & (T - 1);
#pragma unroll
            for (int t = 0; t < (GK * 9 + 31) / 32; ++t) {
                const uint32_t e = t * 32 + lane;
                if (e >= uint32_t(GK * 9)) break;
                const uint32_t kk = e / 9, u = e - kk * 9;
                const uint32_t I = I0 + ((r0 + kk) >> 7);
                const uint32_t col = A0 + 4 * u, J = col >> 7;
                V* dst = sb + kk * GB_STRIDE + 4 * u;
                if (kk < rows && I <= J && J < nb) {
                    const V* src = q.bg + tidx(I, J, nb) * TT + uint64_t((r0 + kk) & (T - 1)) * T +
                                   (col & (T - 1));
                    cp_async16(dst, src, true);
                } else {
                    const V inf4[4] = {Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf(), Ops<V>::inf()};
                    st4(dst, inf4);
                }
            }
        } else {  // diagonal block (c1 == c2, 1/k of the pairs): generic lookup
#pragma unroll 1
            for (int kk = 0; kk < GK; ++kk) {
                const uint32_t col = G0 + lane;
                V v = Ops<V>::inf();
                if (uint32_t(kk) < rows && col_ok) v = q.bg[sym_off(g1 + k0 + kk, col, nb)];
                sb[kk * GB_STRIDE + shift + lane] = v;
            }
        }
        cp_async_commit();
    };
    (void)Jlo;

    V acc[4 * NQ4];
#pragma unroll
    for (int i = 0; i < 4 * NQ4; ++i) acc[i] = Ops<V>::inf();
    // col2_q[j] for every query, fetched asynchronously now (first commit
    // group, so it has landed by the first chunk's wait) into shared memory
#pragma unroll 4
    for (int i = 0; i < 4 * NQ4; ++i) {
        const bool ok = col_ok && uint32_t(i) < m;
        cp_async4(st->c2 + i * 32 + lane, cb2 + (ok ? st->c2off[i] + j : 0), ok);
    }
    cp_async_commit();
    if (B1 > 0) issue(0, 0);
    int buf = 0;
    for (uint32_t k0 = 0; k0 < B1; k0 += GK) {
        const bool more = k0 + GK < B1;
        if (more) issue(k0 + GK, buf ^ 1);
        if (more) cp_async_wait<1>(); else cp_async_wait<0>();
        if (MODE == QM_BLOCKS) {
            mbar_wait(&st->bar[buf], (phase >> buf) & 1u);
            phase ^= 1u << buf;
        }
        __syncwarp();
        if (MODE == QM_BLOCKS)
            group_chunk<V, NQ4, 32>(st->a[buf], st->b[buf], acc,
                                    (min(uint32_t(GK), B1 - k0) + 3) & ~3u, 0, lane);
        else
            group_chunk<V, NQ4, GB_STRIDE>(st->a[buf], st->b[buf], acc,
                                           (min(uint32_t(GK), B1 - k0) + 3) & ~3u, shift, lane);
        __syncwarp();  // buffer `buf` is refilled two chunks later
        buf ^= 1;
    }
    // combine with col2 (t_q = acc_q + col2_q[j]), then per-query minimum over
    // the 32 columns through a padded shared transpose (conflict free)
    cp_async_wait<0>();  // col2 group (also covers B1 == 0)
    __syncwarp();
    static_assert(2 * GQ * GA_STRIDE >= 32 * 33, "transpose scratch fits both A buffers");
    V* sT = st->a[0];  // 32 x 33 words over a[0..1], free after the last chunk
#pragma unroll
    for (int i = 0; i < 4 * NQ4; ++i) {
        const V c2v = st->c2[i * 32 + lane];  // zero-filled when !ok: masked below
        const bool ok = col_ok && uint32_t(i) < m;
        sT[i * 33 + lane] = ok ? Ops<V>::addmin(acc[i], c2v, Ops<V>::inf()) : Ops<V>::inf();
    }
    __syncwarp();
    if (uint32_t(lane) < m) {
        V mine = Ops<V>::inf();
#pragma unroll 8
        for (int c = 0; c < 32; ++c) mine = Ops<V>::vmin(mine, sT[lane * 33 + c]);
        atomic_min_bits<V>(&w.best[st->id[lane]], mine);
    }
}

// ------------------------- block layout: register-blocked warp task --
// Same task and staging as group_task<QM_BLOCKS> (one 2 KB bulk copy per
// 16-row chunk of the column group, row1 by 16-byte cp.async into
// [query][row]), but the product is register-blocked. Lane layout
// <NQG, CPL>: query group qg = lane % NQG, column slot cq = lane / NQG; the
// lane owns queries qg + NQG*i (i < QPT) x columns cq*CPL .. cq*CPL+CPL-1,
// i.e. QPT x CPL independent accumulators. Per 4 rows a lane issues QPT
// LDS.128 of row1 (NQG distinct conflict-free addresses per warp,
// GA_STRIDE = 20), 2*CPL/4 ... CPL LDS.128 of block rows and 4*CPL*QPT
// relaxations (~90% of the issued instructions are VIADDMNMX).
//   <4, 4>: 32 columns, queries in steps of 4 (QPT 1..8)
//   <8, 4>: 16 columns, the last column group of a pair when <= 16 of its
//           columns exist (task flag), queries in steps of 8 (QPT 1..4)
//   <8, 8>: 32 columns, steps of 8 (PSP_QUERY_PRODUCT=8x8, A/B only)
// On cfg2 the finer steps lift useful / issued relaxations from 0.80 to
// 0.90 (query padding to 4 instead of 8, column padding to 16 instead of 32).
// col2 is staged [query][32] with its 16-byte chunks XOR-swizzled by the
// query (chunk u of query q at u ^ (q & 7)), so the epilogue's LDS.128s
// are conflict-free; the column-slot lanes of a query meet by SHFL.
template <class V, int NQG, int CPL, int QPT>
__device__ __forceinline__ void rb_chunk(const V* __restrict__ sA, const V* __restrict__ sB,
                                         V (&acc)[32], uint32_t rows4, int lane) {
    const int qg = lane % NQG, cq = lane / NQG;
    const V* a0 = sA + qg * GA_STRIDE;
    const V* b0 = sB + cq * CPL;
    // not unrolled: one 4-row step is 4 * CPL * QPT relaxations, and four
    // unrolled copies per variant overflow the instruction cache
#pragma unroll 1
    for (uint32_t k4 = 0; k4 < rows4; k4 += 4) {
        uint4 a[QPT];
#pragma unroll
        for (int i = 0; i < QPT; ++i)
            a[i] = *reinterpret_cast<const uint4*>(a0 + NQG * i * GA_STRIDE + k4);
#pragma unroll
        for (int r = 0; r < 4; r += 2) {
            uint32_t bx[CPL], by[CPL];
#pragma unroll
            for (int h = 0; h < CPL / 4; ++h) {
                const uint4 x = *reinterpret_cast<const uint4*>(b0 + (k4 + r) * 32 + 4 * h);
                const uint4 y = *reinterpret_cast<const uint4*>(b0 + (k4 + r + 1) * 32 + 4 * h);
                bx[4 * h] = x.x; bx[4 * h + 1] = x.y; bx[4 * h + 2] = x.z; bx[4 * h + 3] = x.w;
                by[4 * h] = y.x; by[4 * h + 1] = y.y; by[4 * h + 2] = y.z; by[4 * h + 3] = y.w;
            }
#pragma unroll
            for (int i = 0; i < QPT; ++i) {
                const V ar0 = Ops<V>::from_bits(r == 0 ? a[i].x : a[i].z);
                const V ar1 = Ops<V>::from_bits(r == 0 ? a[i].y : a[i].w);
#pragma unroll
                for (int c = 0; c < CPL; ++c)
                    acc[i * CPL + c] = Ops<V>::addmin2(ar0, Ops<V>::from_bits(bx[c]), ar1,
                                                       Ops<V>::from_bits(by[c]), acc[i * CPL + c]);
            }
        }
    }
}

// Epilogue of one variant: t = min over the lane's columns of acc + col2 per
// query slot, written to red[query][column slot] for the generic reduction.
template <class V, int NQG, int CPL, int QPT>
__device__ __forceinline__ void rb_combine(const V (&acc)[32], const V* __restrict__ c2s,
                                           V* __restrict__ red, int lane) {
    constexpr int NCS = 32 / NQG;
    const int qg = lane % NQG, cq = lane / NQG;
#pragma unroll
    for (int i = 0; i < QPT; ++i) {
        const uint32_t qq = qg + NQG * i;
        const V* crow = c2s + qq * 32;
        V d = Ops<V>::inf();
#pragma unroll
        for (int h = 0; h < CPL / 4; ++h) {
            const uint4 cv = *reinterpret_cast<const uint4*>(
                crow + 4 * ((cq * (CPL / 4) + h) ^ (qq & 7)));
            d = Ops<V>::addmin(acc[i * CPL + 4 * h], Ops<V>::from_bits(cv.x), d);
            d = Ops<V>::addmin(acc[i * CPL + 4 * h + 1], Ops<V>::from_bits(cv.y), d);
            d = Ops<V>::addmin(acc[i * CPL + 4 * h + 2], Ops<V>::from_bits(cv.z), d);
            d = Ops<V>::addmin(acc[i * CPL + 4 * h + 3], Ops<V>::from_bits(cv.w), d);
        }
        red[qq * 9 + cq] = d;  // 9-word rows: conflict-free over qg
        (void)NCS;
    }
}

// Variant table (the task's lane layout and query slots), one switch per
// chunk over a flat 32-register accumulator array so all variants share the
// staging, pipeline and reduction code (the kernel stays inside the
// instruction cache):
//   0..7   <4, 4, QPT = v + 1>   32 columns, 4 .. 32 queries in steps of 4
//   8..11  <8, 4, QPT = v - 7>   16 columns (last column group of a pair
//                                 with <= 16 columns), steps of 8
//   ALT:   <8, 8, QPT = v + 1>   32 columns, steps of 8 (PSP_QUERY_PRODUCT=8x8)
template <class V, bool ALT>
__device__ __forceinline__ void rb_chunk_v(int v, const V* sA, const V* sB, V (&acc)[32],
                                           uint32_t rows4, int lane) {
    if constexpr (ALT) {
        switch (v) {
            case 0: rb_chunk<V, 8, 8, 1>(sA, sB, acc, rows4, lane); break;
            case 1: rb_chunk<V, 8, 8, 2>(sA, sB, acc, rows4, lane); break;
            case 2: rb_chunk<V, 8, 8, 3>(sA, sB, acc, rows4, lane); break;
            default: rb_chunk<V, 8, 8, 4>(sA, sB, acc, rows4, lane); break;
        }
    } else {
        switch (v) {
            case 0: rb_chunk<V, 4, 4, 1>(sA, sB, acc, rows4, lane); break;
            case 1: rb_chunk<V, 4, 4, 2>(sA, sB, acc, rows4, lane); break;
            case 2: rb_chunk<V, 4, 4, 3>(sA, sB, acc, rows4, lane); break;
            case 3: rb_chunk<V, 4, 4, 4>(sA, sB, acc, rows4, lane); break;
            case 4: rb_chunk<V, 4, 4, 5>(sA, sB, acc, rows4, lane); break;
            case 5: rb_chunk<V, 4, 4, 6>(sA, sB, acc, rows4, lane); break;
            case 6: rb_chunk<V, 4, 4, 7>(sA, sB, acc, rows4, lane); break;
            case 7: rb_chunk<V, 4, 4, 8>(sA, sB, acc, rows4, lane); break;
            case 8: rb_chunk<V, 8, 4, 1>(sA, sB, acc, rows4, lane); break;
            case 9: rb_chunk<V, 8, 4, 2>(sA, sB, acc, rows4, lane); break;
            case 10: rb_chunk<V, 8, 4, 3>(sA, sB, acc, rows4, lane); break;
            default: rb_chunk<V, 8, 4, 4>(sA, sB, acc, rows4, lane); break;
        }
    }
}
template <class V, bool ALT>
__device__ __forceinline__ void rb_combine_v(int v, const V (&acc)[32], const V* c2s, V* red,
                                             int lane) {
    if constexpr (ALT) {
        switch (v) {
            case 0: rb_combine<V, 8, 8, 1>(acc, c2s, red, lane); break;
            case 1: rb_combine<V, 8, 8, 2>(acc, c2s, red, lane); break;
            case 2: rb_combine<V, 8, 8, 3>(acc, c2s, red, lane); break;
            default: rb_combine<V, 8, 8, 4>(acc, c2s, red, lane); break;
        }
    } else {
        switch (v) {
            case 0: rb_combine<V, 4, 4, 1>(acc, c2s, red, lane); break;
            case 1: rb_combine<V, 4, 4, 2>(acc, c2s, red, lane); break;
            case 2: rb_combine<V, 4, 4, 3>(acc, c2s, red, lane); break;
            case 3: rb_combine<V, 4, 4, 4>(acc, c2s, red, lane); break;
            case 4: rb_combine<V, 4, 4, 5>(acc, c2s, red, lane); break;
            case 5: rb_combine<V, 4, 4, 6>(acc, c2s, red, lane); break;
            case 6: rb_combine<V, 4, 4, 7>(acc, c2s, red, lane); break;
            case 7: rb_combine<V, 4, 4, 8>(acc, c2s, red, lane); break;
            case 8: rb_combine<V, 8, 4, 1>(acc, c2s, red, lane); break;
            case 9: rb_combine<V, 8, 4, 2>(acc, c2s, red, lane); break;
            case 10: rb_combine<V, 8, 4, 3>(acc, c2s, red, lane); break;
            default: rb_combine<V, 8, 4, 4>(acc, c2s, red, lane); break;
        }
    }
}

// A task's per-lane query metadata (lane < m): id, l1 and l2 in sorted
// order, loaded one task ahead (TaskMeta::load inside the previous task) so
// the task start does not wait on them.
struct TaskMeta {
    uint32_t id = 0, l1 = 0, l2 = 0;
    __device__ __forceinline__ void load(const GroupWork& w, const uint4& rec, int lane) {
        const uint32_t q0 = rec.z, m = rec.w & 0x3fu;
        if (uint32_t(lane) < m) {
            id = w.sorted[q0 + lane];
            l1 = w.s_l1[q0 + lane];
            l2 = w.s_l2[q0 + lane];
        }
    }
};

template <class V, bool ALT>
__device__ __forceinline__ void group_task_rb(const QueryView<V>& q, const GroupWork& w,
                                              WarpStage<V>* st, uint32_t c1, uint32_t c2,
                                              uint32_t q0, uint32_t m, uint32_t cg, bool half,
                                              uint32_t& phase, const TaskMeta& me,
                                              const uint4& rec_next, TaskMeta& me_next) {
    const int lane = threadIdx.x & 31;
    // variant and its column-slot count (NCS lanes share a query)
    int v, ncs;
    if (ALT) { v = int((m + 7) / 8) - 1; ncs = 4; }
    else if (half) { v = 7 + int((m + 7) / 8); ncs = 4; }
    else { v = int((m + 3) / 4) - 1; ncs = 8; }
    const uint32_t cch = half ? 4u : 8u;  // 4-column chunks of col2 the task uses
    const uint32_t g1 = q.bnd_off[c1], B1 = q.bnd_off[c1 + 1] - g1;
    const uint32_t g2 = q.bnd_off[c2], B2 = q.bnd_off[c2 + 1] - g2;
    const uint32_t Bp1 = cb_stride(B1), Bp2 = cb_stride(B2);
    const V* __restrict__ cb1 = q.cb + q.cb_off[c1];
    const V* __restrict__ cb2 = q.cb + q.cb_off[c2];
    const V* bq_task = q.bq + q.bq_off[c1 * q.k + c2] + uint64_t(cg) * ((B1 + GK - 1) / GK * GK) * 32;
    (void)q0;
    __syncwarp();
    const V* my_row1 = cb1;
    if (uint32_t(lane) < m) {
        st->id[lane] = me.id;
        st->c2off[lane] = me.l2 * Bp2 + cg * 32;
        my_row1 = cb1 + uint64_t(me.l1) * Bp1;
    }
    __syncwarp();
    // col2: chunk u (4 columns) of query qq -> st->c2[qq * 32 + 4 * (u ^ (qq & 7))];
    // chunks past the row's padded end zero-fill (their block columns are
    // INF, so those sums never win). Slots >= m are never reported.
    for (uint32_t e = lane; e < m * cch; e += 32) {
        const uint32_t qq = e / cch, u = e % cch;
        const bool ok = cg * 32 + 4 * u < Bp2;
        cp_async16(st->c2 + qq * 32 + 4 * (u ^ (qq & 7)), cb2 + (ok ? st->c2off[qq] + 4 * u : 0), ok);
    }
    cp_async_commit();

    auto issue = [&](uint32_t k0, int buf) {
        V* sa = st->a[buf] + lane * GA_STRIDE;
        if (uint32_t(lane) < m) {
#pragma unroll
            for (int t = 0; t < GK / 4; ++t) cp_async16(sa + 4 * t, my_row1 + k0 + 4 * t, true);  // k0 + 16 <= B1p <= Bp1
        }
        cp_async_commit();
        if (lane == 0) {
            // no proxy fence: b[] is only ever written by these bulk copies
            // (its previous contents were read by LDS whose results the
            // product already consumed before the __syncwarp that precedes
            // this issue), so there is no generic write to order against
            mbar_expect_tx(&st->bar[buf], GK * 32 * sizeof(V));
            bulk_g2s(st->b[buf], bq_task + uint64_t(k0) * 32, GK * 32 * sizeof(V), &st->bar[buf]);
        }
    };

    V acc[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = Ops<V>::inf();
    if (B1 > 0) issue(0, 0);
    // the next task's metadata, in flight while this task computes
    me_next.load(w, rec_next, lane);
    int buf = 0;
    for (uint32_t k0 = 0; k0 < B1; k0 += GK) {
        const bool more = k0 + GK < B1;
        if (more) issue(k0 + GK, buf ^ 1);
        if (more) cp_async_wait<1>(); else cp_async_wait<0>();
        mbar_wait(&st->bar[buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;
        __syncwarp();
        rb_chunk_v<V, ALT>(v, st->a[buf], st->b[buf], acc, (min(uint32_t(GK), B1 - k0) + 3) & ~3u, lane);
        __syncwarp();  // buffer `buf` is refilled by the next issue
        buf ^= 1;
    }
    cp_async_wait<0>();  // col2 (also covers B1 == 0)
    __syncwarp();
    static_assert(GQ * 9 <= GQ * GA_STRIDE, "reduction scratch fits a[0]");
    V* red = st->a[0];  // [query][9]: free after the last chunk
    rb_combine_v<V, ALT>(v, acc, st->c2, red, lane);
    __syncwarp();
    if (uint32_t(lane) < m) {
        V d = red[lane * 9];
        for (int c = 1; c < ncs; ++c) d = Ops<V>::vmin(d, red[lane * 9 + c]);
        atomic_min_bits<V>(&w.best[st->id[lane]], d);
    }
}

// ---- 16-bit residual product (QM_BLOCKS16): chunk, epilogue, task ------
// Lane layout <NQG, 4 columns = 2 u16x2 words, QPT>: query group qg = lane %
// NQG, column slot cq = lane / NQG. A: [query][row] u32 words, each the
// row's 15-bit offset in both halves; B: [row][32] u16 residuals.
template <int NQG, int QPT>
__device__ __forceinline__ void rb16_chunk(const uint32_t* __restrict__ sA,
                                           const uint16_t* __restrict__ sB, uint32_t (&acc)[16],
                                           uint32_t rows4, int lane) {
    const int qg = lane % NQG, cq = lane / NQG;
    const uint32_t* a0 = sA + qg * GA_STRIDE;
    const uint16_t* b0 = sB + cq * 4;
#pragma unroll 1
    for (uint32_t k4 = 0; k4 < rows4; k4 += 4) {
        uint4 a[QPT];
#pragma unroll
        for (int i = 0; i < QPT; ++i)
            a[i] = *reinterpret_cast<const uint4*>(a0 + NQG * i * GA_STRIDE + k4);
        uint2 b[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) b[r] = *reinterpret_cast<const uint2*>(b0 + (k4 + r) * 32);
#pragma unroll
        for (int r = 0; r < 4; ++r) {
#pragma unroll
            for (int i = 0; i < QPT; ++i) {
                const uint32_t ar = r == 0 ? a[i].x : r == 1 ? a[i].y : r == 2 ? a[i].z : a[i].w;
                acc[2 * i] = __viaddmin_u16x2(ar, b[r].x, acc[2 * i]);
                acc[2 * i + 1] = __viaddmin_u16x2(ar, b[r].y, acc[2 * i + 1]);
            }
        }
    }
}

// Per query slot of this lane: the best exact candidate and the smallest
// lower bound over the lane's 4 columns, into red_e / red_l [query][9].
template <int NQG, int QPT>
__device__ __forceinline__ void rb16_combine(const uint32_t (&acc)[16], const uint32_t* c2s,
                                             const uint32_t* base, uint4 bj, uint32_t j0,
                                             uint32_t B2, uint32_t* red_e, uint32_t* red_l,
                                             int lane, uint32_t sat) {
    const int qg = lane % NQG, cq = lane / NQG;
    const uint32_t bjv[4] = {bj.x, bj.y, bj.z, bj.w};
#pragma unroll
    for (int i = 0; i < QPT; ++i) {
        const uint32_t qq = qg + NQG * i;
        const uint4 cv = *reinterpret_cast<const uint4*>(c2s + qq * 32 + 4 * (cq ^ (qq & 7)));
        const uint32_t cvv[4] = {cv.x, cv.y, cv.z, cv.w};
        const uint64_t bq = base[qq];
        uint64_t d = U32_INF, l = U32_INF;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t j = j0 + cq * 4 + u;
            if (j < B2) {
                const uint32_t t = (acc[2 * i + (u >> 1)] >> (16 * (u & 1))) & 0xFFFFu;
                const uint64_t tail = bq + uint64_t(cvv[u]) + bjv[u];
                if (t < sat) d = min(d, tail + t);
                else l = min(l, tail + sat);
            }
        }
        red_e[qq * 9 + cq] = uint32_t(min(d, uint64_t(U32_INF)));
        red_l[qq * 9 + cq] = uint32_t(min(l, uint64_t(U32_INF)));
    }
}

__device__ __forceinline__ void rb16_chunk_v(int v, const uint32_t* sA, const uint16_t* sB,
                                             uint32_t (&acc)[16], uint32_t rows4, int lane) {
    switch (v) {
        case 0: rb16_chunk<4, 1>(sA, sB, acc, rows4, lane); break;
        case 1: rb16_chunk<4, 2>(sA, sB, acc, rows4, lane); break;
        case 2: rb16_chunk<4, 3>(sA, sB, acc, rows4, lane); break;
        case 3: rb16_chunk<4, 4>(sA, sB, acc, rows4, lane); break;
        case 4: rb16_chunk<4, 5>(sA, sB, acc, rows4, lane); break;
        case 5: rb16_chunk<4, 6>(sA, sB, acc, rows4, lane); break;
        case 6: rb16_chunk<4, 7>(sA, sB, acc, rows4, lane); break;
        case 7: rb16_chunk<4, 8>(sA, sB, acc, rows4, lane); break;
        case 8: rb16_chunk<8, 1>(sA, sB, acc, rows4, lane); break;
        case 9: rb16_chunk<8, 2>(sA, sB, acc, rows4, lane); break;
        case 10: rb16_chunk<8, 3>(sA, sB, acc, rows4, lane); break;
        default: rb16_chunk<8, 4>(sA, sB, acc, rows4, lane); break;
    }
}
__device__ __forceinline__ void rb16_combine_v(int v, const uint32_t (&acc)[16], const uint32_t* c2s,
                                               const uint32_t* base, uint4 bj, uint32_t j0,
                                               uint32_t B2, uint32_t* re, uint32_t* rl, int lane,
                                               uint32_t sat) {
    switch (v) {
        case 0: rb16_combine<4, 1>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 1: rb16_combine<4, 2>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 2: rb16_combine<4, 3>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 3: rb16_combine<4, 4>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 4: rb16_combine<4, 5>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 5: rb16_combine<4, 6>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 6: rb16_combine<4, 7>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 7: rb16_combine<4, 8>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 8: rb16_combine<8, 1>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 9: rb16_combine<8, 2>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        case 10: rb16_combine<8, 3>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
        default: rb16_combine<8, 4>(acc, c2s, base, bj, j0, B2, re, rl, lane, sat); break;
    }
}

// One warp task of the 16-bit product: the task records, bulk-copy pipeline
// and col2 staging of group_task_rb. A comes in as the queries' u32 row1
// values by cp.async (as in the u32 product) plus the block's row potentials
// a_i; after the chunk lands each lane turns its query's 16 rows in place
// into min(row1 + a_i - base, S) in both halves (base = the query's exact
// min_i row1 + a_i, from group_bases16). Two results per query (best exact
// candidate, smallest lower bound) go to w.best / w.lb.
template <class V>
__device__ __forceinline__ void group_task_rb16(const QueryView<V>& q, const GroupWork& w,
                                                WarpStage<V>* st, uint32_t c1, uint32_t c2,
                                                uint32_t q0, uint32_t m, uint32_t cg, bool half,
                                                uint32_t& phase) {
    const int lane = threadIdx.x & 31;
    int v;
    if (half) v = 7 + int((m + 7) / 8);
    else v = int((m + 3) / 4) - 1;
    const int ncs = half ? 4 : 8;
    const uint32_t cch = half ? 4u : 8u;
    const uint32_t g1 = q.bnd_off[c1], B1 = q.bnd_off[c1 + 1] - g1;
    const uint32_t g2 = q.bnd_off[c2], B2 = q.bnd_off[c2 + 1] - g2;
    const uint32_t Bp1 = cb_stride(B1), Bp2 = cb_stride(B2), B1p = (B1 + GK - 1) / GK * GK;
    const uint64_t blk = uint64_t(c1) * q.k + c2;
    const uint16_t* bq_task = q.bq16 + q.bq16_off[blk] + uint64_t(cg) * B1p * 32;
    const uint32_t* ax = q.bqaux + q.aux_off[blk];
    const uint32_t* arow = ax + 4;                  // a_i, B1p entries
    const uint32_t* bj = ax + 4 + B1p + cg * 32;    // b_j of this column group
    const V* __restrict__ cb1 = q.cb + q.cb_off[c1];
    const V* __restrict__ cb2 = q.cb + q.cb_off[c2];
    // chunk buffers by arithmetic (arrays of pointers indexed by `buf` went to local memory)
    uint16_t* const b16_0 = reinterpret_cast<uint16_t*>(st->b[0]);
    auto b16 = [&](int bb) { return b16_0 + bb * (16 * 32); };
    uint32_t* base = reinterpret_cast<uint32_t*>(st->b[1]);     // [GQ]
    auto abuf = [&](int bb) { return base + GQ + 16 * bb; };    // a_i of each chunk
    auto sa = [&](int bb) { return reinterpret_cast<uint32_t*>(st->a[bb]); };
    __syncwarp();
    const V* my_row1 = cb1;
    if (uint32_t(lane) < m) {
        const uint32_t id = w.sorted[q0 + lane];
        st->id[lane] = id;
        st->c2off[lane] = w.s_l2[q0 + lane] * Bp2 + cg * 32;
        my_row1 = cb1 + uint64_t(w.s_l1[q0 + lane]) * Bp1;
        base[lane] = w.base16[id];
    }
    const uint4 bjq = *reinterpret_cast<const uint4*>(bj + (lane / (half ? 8 : 4)) * 4);
    __syncwarp();
    for (uint32_t e = lane; e < m * cch; e += 32) {
        const uint32_t qq = e / cch, u = e % cch;
        const bool ok = cg * 32 + 4 * u < Bp2;
        cp_async16(reinterpret_cast<V*>(st->c2) + qq * 32 + 4 * (u ^ (qq & 7)),
                   cb2 + (ok ? st->c2off[qq] + 4 * u : 0), ok);
    }
    cp_async_commit();
    auto issue = [&](uint32_t k0, int buf) {
        uint32_t* sa_l = sa(buf) + lane * GA_STRIDE;
        if (uint32_t(lane) < m) {
#pragma unroll
            for (int t = 0; t < GK / 4; ++t)
                cp_async16(sa_l + 4 * t, my_row1 + k0 + 4 * t, k0 + 4 * t < Bp1);
        }
        if (lane < GK / 4) cp_async16(abuf(buf) + 4 * lane, arow + k0 + 4 * lane, true);
        cp_async_commit();
        if (lane == 0) {
            mbar_expect_tx(&st->bar[buf], GK * 32 * sizeof(uint16_t));
            bulk_g2s(b16(buf), bq_task + uint64_t(k0) * 32, GK * 32 * sizeof(uint16_t), &st->bar[buf]);
        }
    };
    uint32_t acc[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = 0xFFFFFFFFu;  // both halves at the 16-bit maximum
    const uint32_t sat = q.u16_sat;
    if (B1 > 0) issue(0, 0);
    int buf = 0;
    for (uint32_t k0 = 0; k0 < B1; k0 += GK) {
        const bool more = k0 + GK < B1;
        if (more) issue(k0 + GK, buf ^ 1);
        if (more) cp_async_wait<1>(); else cp_async_wait<0>();
        __syncwarp();
        if (uint32_t(lane) < m) {  // row1 + a_i - base, saturated, in both halves
            uint32_t* row = sa(buf) + lane * GA_STRIDE;
            const uint64_t bq = base[lane];
            const uint32_t rows = min(uint32_t(GK), B1 - k0);
#pragma unroll
            for (int t = 0; t < GK / 4; ++t) {
                const uint4 r4 = *reinterpret_cast<const uint4*>(row + 4 * t);
                const uint4 a4 = *reinterpret_cast<const uint4*>(abuf(buf) + 4 * t);
                const uint32_t rv[4] = {r4.x, r4.y, r4.z, r4.w}, av[4] = {a4.x, a4.y, a4.z, a4.w};
                uint32_t o[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint64_t x = uint64_t(rv[u]) + av[u];
                    uint32_t y = sat;
                    if (uint32_t(4 * t + u) < rows && rv[u] < U32_INF && av[u] < U32_INF)
                        y = uint32_t(min(x - bq, uint64_t(sat)));
                    o[u] = y * 0x10001u;
                }
                *reinterpret_cast<uint4*>(row + 4 * t) = make_uint4(o[0], o[1], o[2], o[3]);
            }
        }
        mbar_wait(&st->bar[buf], (phase >> buf) & 1u);
        phase ^= 1u << buf;
        __syncwarp();
        rb16_chunk_v(v, sa(buf), b16(buf), acc, (min(uint32_t(GK), B1 - k0) + 3) & ~3u, lane);
        __syncwarp();  // buffer `buf` is refilled by the next issue
        buf ^= 1;
    }
    cp_async_wait<0>();  // col2 (also covers B1 == 0)
    __syncwarp();
    uint32_t* red_e = sa(0);          // [query][9] over a[0], free after the last chunk
    uint32_t* red_l = sa(0) + GQ * 9;
    static_assert(2 * GQ * 9 <= GQ * GA_STRIDE, "reduction scratch fits a[0]");
    rb16_combine_v(v, acc, reinterpret_cast<const uint32_t*>(st->c2), base, bjq, cg * 32, B2, red_e,
                   red_l, lane, sat);
    __syncwarp();
    if (uint32_t(lane) < m) {
        uint32_t d = red_e[lane * 9], l = red_l[lane * 9];
        for (int c = 1; c < ncs; ++c) {
            d = min(d, red_e[lane * 9 + c]);
            l = min(l, red_l[lane * 9 + c]);
        }
        atomicMin(&w.best[st->id[lane]], d);
        atomicMin(&w.lb[st->id[lane]], l);
    }
}

// Exact per-query bases of the 16-bit product: base = min_i row1_i + a_i
// over the pair block's rows (INF when none is finite), a warp per query.
template <class V>
__global__ void group_bases16(QueryView<V> q, uint64_t count, GroupWork w) {
    const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (uint64_t i = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; i < count; i += nw) {
        const uint32_t key = w.key[i];
        const uint32_t c1 = key / q.k, c2 = key % q.k;
        const uint32_t B1 = q.bnd_off[c1 + 1] - q.bnd_off[c1], B1p = (B1 + GK - 1) / GK * GK;
        const V* row1 = q.cb + q.cb_off[c1] + uint64_t(w.l1[i]) * cb_stride(B1);
        const uint32_t* arow = q.bqaux + q.aux_off[uint64_t(c1) * q.k + c2] + 4;
        uint64_t bmin = U32_INF;
        for (uint32_t r = lane; r < B1; r += 32) {
            const uint32_t x = Ops<V>::to_bits(row1[r]), a = arow[r];
            if (x < U32_INF && a < U32_INF) bmin = min(bmin, uint64_t(x) + a);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) bmin = min(bmin, __shfl_xor_sync(0xffffffffu, bmin, o));
        if (lane == 0) w.base16[i] = uint32_t(min(bmin, uint64_t(U32_INF)));
        (void)B1p;
    }
}

template <class V, int MODE>
__global__ void __launch_bounds__(GTHREADS, 2) query_grouped(QueryView<V> q, GroupWork w) {
    extern __shared__ __align__(16) unsigned char g_smem[];
    WarpStage<V>* st = reinterpret_cast<WarpStage<V>*>(g_smem) + (threadIdx.x >> 5);
    uint32_t phase = 0;  // QM_BLOCKS*: parity of each B buffer's barrier
    if (MODE == QM_BLOCKS || MODE == QM_BLOCKS_LANE || MODE == QM_BLOCKS_8X8 || MODE == QM_BLOCKS16) {
        if ((threadIdx.x & 31) == 0) {
            mbar_init(&st->bar[0], 1);
            mbar_init(&st->bar[1], 1);
        }
        __syncwarp();
    }
    const uint32_t total = w.task_start[w.nbins];
    const uint32_t nwarps = gridDim.x * GWARPS;
    // dynamic task queue: a warp's first task is its global warp id, later
    // ones come from a counter (task_cnt[nbins], zeroed by group_tasks and
    // free after the scans) fetched one task ahead so the atomic's latency
    // hides behind the current task. Static striding left the last warps
    // running ~20% past the mean (tasks differ in B1 and query count).
    uint32_t* const queue = w.task_cnt + w.nbins;
    const bool lead = (threadIdx.x & 31) == 0;
    uint32_t task = blockIdx.x * GWARPS + (threadIdx.x >> 5);
    if constexpr (MODE == QM_BLOCKS || MODE == QM_BLOCKS_8X8) {
        // two tasks ahead: the atomic for task t + 2 and the descriptor and
        // per-lane metadata of task t + 1 are in flight while task t runs
        const int lane = threadIdx.x & 31;
        uint32_t nxt = 0;
        if (lead) nxt = atomicAdd(queue, 1u) + nwarps;
        uint4 rec = task < total ? w.tasks[task] : make_uint4(0, 0, 0, 0);
        TaskMeta me;
        me.load(w, rec, lane);
        nxt = __shfl_sync(0xffffffffu, nxt, 0);
        while (task < total) {
            uint32_t nn = 0;
            if (lead) nn = atomicAdd(queue, 1u) + nwarps;
            const uint4 rec_next = nxt < total ? w.tasks[nxt] : make_uint4(0, 0, 0, 0);
            TaskMeta me_next;
            const uint32_t c1 = rec.x, c2 = rec.y, q0 = rec.z, m = rec.w & 0x3fu, cg = rec.w >> 8;
            const bool half = (rec.w >> 6) & 1u;
            group_task_rb<V, MODE == QM_BLOCKS_8X8>(q, w, st, c1, c2, q0, m, cg, half, phase, me,
                                                    rec_next, me_next);
            task = nxt;
            rec = rec_next;
            me = me_next;
            nxt = __shfl_sync(0xffffffffu, nn, 0);
        }
    } else {
        while (task < total) {
            uint32_t next = 0;
            if (lead) next = atomicAdd(queue, 1u) + nwarps;
            const uint4 rec = w.tasks[task];
            const uint32_t c1 = rec.x, c2 = rec.y, q0 = rec.z, m = rec.w & 0x3fu, cg = rec.w >> 8;
            const bool half = (rec.w >> 6) & 1u;  // last column group, <= 16 columns
            // block layout: the register-blocked product (12 variants behind one
            // switch, see group_task_rb). Tile arena / routed / lane product:
            // three query-count variants (32/16/8 slots; finer ones grew that
            // kernel past the instruction cache), 24 slots for the lane product
            if constexpr (MODE == QM_BLOCKS16) {  // 16-bit residual product (u32 tables)
                group_task_rb16<V>(q, w, st, c1, c2, q0, m, cg, half, phase);
            } else {
                constexpr int TM = MODE == QM_BLOCKS_LANE ? QM_BLOCKS : MODE;
                if (m > 24 || (TM != QM_BLOCKS && m > 16)) group_task<V, 8, TM>(q, w, st, c1, c2, q0, m, cg, phase);
                else if (TM == QM_BLOCKS && m > 16) group_task<V, 6, TM>(q, w, st, c1, c2, q0, m, cg, phase);
                else if (m > 8) group_task<V, 4, TM>(q, w, st, c1, c2, q0, m, cg, phase);
                else group_task<V, 2, TM>(q, w, st, c1, c2, q0, m, cg, phase);
            }
            task = __shfl_sync(0xffffffffu, next, 0);
        }
    }
}

// QM_BLOCKS16: a query is exact when its best exact candidate is <= every
// lower bound (or the same-component entry is); the rest go to the list
// query_fallback answers in u32.
template <class V>
__global__ void group_finish16(QueryView<V> q, uint64_t count, GroupWork w, double* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    const uint32_t d = w.best[i], l = w.lb[i];
    const uint32_t key = w.key[i];
    const uint32_t c1 = key / q.k, c2 = key % q.k;
    const uint32_t cap = c1 == c2 ? Ops<V>::to_bits(same_component_entry(q, c1, w.l1[i], w.l2[i]))
                                  : U32_INF;
    if (d <= l) {
        out[i] = Ops<V>::to_f64(Ops<V>::from_bits(min(d, cap)), q.scale);
    } else if (cap <= l) {
        out[i] = Ops<V>::to_f64(Ops<V>::from_bits(cap), q.scale);
    } else {
        w.fb_list[atomicAdd(w.fb_count, 1u)] = static_cast<uint32_t>(i);
    }
}

// The u32 answer of every query group_finish16 could not settle (grid-
// stride over the device-side count; cta_query on the u32 tables).
template <class V>
__global__ void __launch_bounds__(32 * QC_WARPS) query_fallback(QueryView<V> q,
                                                                const uint32_t* __restrict__ v1,
                                                                const uint32_t* __restrict__ v2,
                                                                GroupWork w, double* __restrict__ out) {
    __shared__ V red[QC_WARPS];
    const uint32_t n = *w.fb_count;
    for (uint32_t f = blockIdx.x; f < n; f += gridDim.x) {
        const uint32_t i = w.fb_list[f];
        const double d = cta_query(q, v1[i], v2[i], red);
        if (threadIdx.x == 0) out[i] = d;
    }
}

// out[i] = min(best[i], same-component entry) as f64 (src/query.cpp:70-72).
template <class V>
__global__ void group_finish(QueryView<V> q, const uint32_t* __restrict__ v1,
                             const uint32_t* __restrict__ v2, uint64_t count, GroupWork w,
                             double* __restrict__ out) {
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= count) return;
    V d = Ops<V>::from_bits(w.best[i]);
    const uint32_t key = w.key[i];
    const uint32_t c1 = key / q.k, c2 = key % q.k;
    if (c1 == c2) d = Ops<V>::vmin(d, same_component_entry(q, c1, w.l1[i], w.l2[i]));
    out[i] = Ops<V>::to_f64(d, q.scale);
}

}  // namespace pspg
