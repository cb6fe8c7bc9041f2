// oracle_file.cuh — the reference's PSP1 oracle file (src/oracle_io.cpp:
// 106-255, include/psp/oracle_io.hpp:10-20) written from and read into device
// tables, and the CRC-64/XZ it is sealed with (include/psp/crc64.hpp:9-39).
//
// Layout (little-endian): "PSP1", version u32 = 1, n u64, k u64, b u64,
// permutation n x u64, assignment n x u64 (reordered -> component), boundary
// flags n bits LSB-first, component offsets (k+1) x u64, component tables
// (|C| x |C| f64 row-major, +inf unreachable) then boundary tables
// (|B(C)| x b f64), CRC-64/XZ of every preceding byte.
//
// The tables never exist in f64 on the device for long: a window of rows is
// unpacked from the tile-packed u32/f32 store straight to f64 (u32 / 2^q,
// INF -> +inf), its CRC is computed on the GPU as independent per-segment raw
// CRCs, and the host folds those into the running checksum with the CRC
// "append" operator x^(8 len) mod P (CRC is linear over GF(2)).
#pragma once
#include <cstdint>

#include "minplus.cuh"

namespace pspg {

constexpr uint64_t CRC64_POLY = 0xC96C5795D7870F42ull;  // reflected ECMA-182

struct Crc64Table {
    uint64_t t[256];
};

inline Crc64Table make_crc64_table() {
    Crc64Table tb{};
    for (uint32_t i = 0; i < 256; ++i) {
        uint64_t crc = i;
        for (int bit = 0; bit < 8; ++bit) crc = (crc >> 1) ^ ((crc & 1) ? CRC64_POLY : 0);
        tb.t[i] = crc;
    }
    return tb;
}

// CRC of the bulk bytes on the GPU: one CTA per CRC_BLOCK (64 KB) bytes.
// The block is staged into shared memory with coalesced 16-byte loads; each
// of the 256 threads takes a 256-byte leaf (slicing-by-8 over 8 tables in
// shared memory, 8 bytes per step); the leaves are folded in a tree of 8
// levels with the CRC append operator x^(8 L) mod P for L = 256 * 2^j bytes
// (GF(2) 64x64 matrices in constant memory). Output: the raw CRC (zero
// initial state, no final xor) of each full block; the host appends the
// blocks and the sub-block tail.
constexpr uint32_t CRC_LEAF = 256;
constexpr uint32_t CRC_THREADS = 256;
constexpr uint32_t CRC_BLOCK = CRC_LEAF * CRC_THREADS;  // 64 KB

struct Crc64Slices {
    uint64_t t[8][256];
};
struct CrcFold {
    uint64_t col[8][64];  // append operator for 256 * 2^j bytes, j = 0..7
};
__constant__ CrcFold c_crc_fold;

inline Crc64Slices make_crc64_slices() {
    Crc64Slices sl{};
    for (uint32_t i = 0; i < 256; ++i) {
        uint64_t crc = i;
        for (int bit = 0; bit < 8; ++bit) crc = (crc >> 1) ^ ((crc & 1) ? CRC64_POLY : 0);
        sl.t[0][i] = crc;
    }
    for (int k = 1; k < 8; ++k)
        for (uint32_t i = 0; i < 256; ++i)
            sl.t[k][i] = (sl.t[k - 1][i] >> 8) ^ sl.t[0][sl.t[k - 1][i] & 0xff];
    return sl;
}

__global__ void __launch_bounds__(CRC_THREADS) crc64_blocks(const uint8_t* __restrict__ data,
                                                            const Crc64Slices* __restrict__ slices,
                                                            uint64_t* __restrict__ out) {
    extern __shared__ __align__(16) unsigned char crc_smem[];
    uint64_t* t = reinterpret_cast<uint64_t*>(crc_smem);            // 8 x 256
    uint4* blk = reinterpret_cast<uint4*>(crc_smem + 8 * 256 * 8);  // CRC_BLOCK bytes
    __shared__ uint64_t part[CRC_THREADS];
    for (uint32_t i = threadIdx.x; i < 8 * 256; i += CRC_THREADS) t[i] = (&slices->t[0][0])[i];
    const uint4* src = reinterpret_cast<const uint4*>(data + uint64_t(blockIdx.x) * CRC_BLOCK);
#pragma unroll 4
    for (uint32_t i = threadIdx.x; i < CRC_BLOCK / 16; i += CRC_THREADS) blk[i] = src[i];
    __syncthreads();
    // leaf: 32 words of 8 bytes; word w of thread x at w * 256 + x would be
    // conflict-free, but the leaf must be contiguous: read word-by-word
    const uint64_t* leaf = reinterpret_cast<const uint64_t*>(blk) + threadIdx.x * (CRC_LEAF / 8);
    uint64_t crc = 0;
#pragma unroll 4
    for (uint32_t w = 0; w < CRC_LEAF / 8; ++w) {
        crc ^= leaf[w];
        crc = t[7 * 256 + (crc & 0xff)] ^ t[6 * 256 + ((crc >> 8) & 0xff)] ^
              t[5 * 256 + ((crc >> 16) & 0xff)] ^ t[4 * 256 + ((crc >> 24) & 0xff)] ^
              t[3 * 256 + ((crc >> 32) & 0xff)] ^ t[2 * 256 + ((crc >> 40) & 0xff)] ^
              t[1 * 256 + ((crc >> 48) & 0xff)] ^ t[0 * 256 + (crc >> 56)];
    }
    part[threadIdx.x] = crc;
    __syncthreads();
    // tree: at level j, leaf run x (x % 2^(j+1) == 0) absorbs run x + 2^j,
    // both 256 * 2^j bytes long: crc = M_j crc ^ crc'
    for (int j = 0; j < 8; ++j) {
        const uint32_t stride = 1u << j;
        if ((threadIdx.x & (2 * stride - 1)) == 0) {
            uint64_t v = part[threadIdx.x], r = 0;
#pragma unroll 8
            for (int b = 0; b < 64; ++b)
                if ((v >> b) & 1) r ^= c_crc_fold.col[j][b];
            part[threadIdx.x] = r ^ part[threadIdx.x + stride];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) out[blockIdx.x] = part[0];
}

// u32 / f32 tile-packed window -> dense f64 rows (the file's value format).
template <class V>
__global__ void window_to_f64(MatSet<V> ms, uint32_t m, uint32_t row0, uint32_t nrows,
                              uint32_t ncols, double scale, double* __restrict__ out) {
    const uint64_t idx = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= uint64_t(nrows) * ncols) return;
    const uint32_t r = static_cast<uint32_t>(idx / ncols), c = static_cast<uint32_t>(idx % ncols);
    out[idx] = Ops<V>::to_f64(ms.tiles[ms.tile_base[m] + sym_off(row0 + r, c, ms.nb[m])], scale);
}

// ---- PSP1 load on the device: the table section streamed in chunks.
// Pieces in file order: start[t] (elements) for t < k the component tables
// (s_c x s_c), for k <= t < 2k the boundary rows (B_c x b), start[2k] = end.
struct Psp1Map {
    const uint64_t* start;    // [2k + 1]
    const uint32_t* size;     // [k] component sizes s_c
    const uint32_t* bnd_off;  // [k + 1]
    uint32_t k, b;
};

// Fixed-point need of one value (choose_kind_tables semantics): the
// smallest q with x * 2^q integral, 0 for +inf (unreachable), 1 << 20 when
// no q works (negative or NaN).
__device__ __forceinline__ int psp1_need_q(double x) {
    if (isinf(x) && x > 0) return 0;
    if (!(x >= 0)) return 1 << 20;
    if (x == 0) return 0;
    const unsigned long long bits = __double_as_longlong(x);
    const int ef = int((bits >> 52) & 0x7ff);
    unsigned long long sig = bits & ((1ull << 52) - 1);
    int e;
    if (ef == 0) {
        e = -1074;  // subnormal
    } else {
        sig |= 1ull << 52;
        e = ef - 1075;
    }
    e += __ffsll(static_cast<long long>(sig)) - 1;  // drop trailing zero bits
    return e >= 0 ? 0 : -e;
}

// One chunk of f64 elements [e0, e0 + cnt): each thread takes PER
// consecutive elements (one binary search over the pieces), writes the
// upper-tile entries of the tables (the writers' rule, minplus.cuh) as V at
// fixed point 2^shift, and folds the chunk's largest finite value and
// fixed-point need into maxbits / need (atomicMax).
template <class V, int PER>
__global__ void __launch_bounds__(256) psp1_convert(const double* __restrict__ chunk, uint64_t e0,
                                                    uint64_t cnt, Psp1Map map, MatSet<V> comps,
                                                    MatSet<V> bg, int shift,
                                                    unsigned long long* __restrict__ maxbits,
                                                    int* __restrict__ need) {
    const uint64_t i0 = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) * PER;
    double mx = 0.0;
    int nq = 0;
    if (i0 < cnt) {
        uint64_t e = e0 + i0;
        uint32_t lo = 0, hi = 2 * map.k;  // piece t: start[t] <= e < start[t + 1]
        while (hi - lo > 1) {
            const uint32_t mid = (lo + hi) / 2;
            if (map.start[mid] <= e) lo = mid;
            else hi = mid;
        }
        uint32_t t = lo;
        const double scale = ldexp(1.0, shift);
        for (int u = 0; u < PER && i0 + u < cnt; ++u, ++e) {
            while (e >= map.start[t + 1]) ++t;
            const double x = chunk[i0 + u];
            if (isfinite(x)) mx = fmax(mx, x);
            nq = max(nq, psp1_need_q(x));
            V v;
            if (std::is_same<V, float>::value) v = Ops<V>::from_bits(__float_as_uint(float(x)));
            else v = isinf(x) ? Ops<V>::inf() : V(static_cast<uint32_t>(x * scale));
            const uint64_t local = e - map.start[t];
            if (t < map.k) {
                const uint32_t sz = map.size[t];
                const uint32_t i = uint32_t(local / sz), j = uint32_t(local - uint64_t(i) * sz);
                if (i / T <= j / T)
                    comps.tiles[comps.tile_base[t] + tidx(i / T, j / T, comps.nb[t]) * TT +
                                uint64_t(i % T) * T + j % T] = v;
            } else {
                const uint32_t c = t - map.k;
                const uint32_t r = uint32_t(local / map.b), j = uint32_t(local - uint64_t(r) * map.b);
                const uint32_t g = map.bnd_off[c] + r;
                if (g / T <= j / T)
                    bg.tiles[tidx(g / T, j / T, bg.nb[0]) * TT + uint64_t(g % T) * T + j % T] = v;
            }
        }
    }
    // block reduction, one atomic per block
    __shared__ double smx[8];
    __shared__ int snq[8];
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        nq = max(nq, __shfl_xor_sync(0xffffffffu, nq, o));
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) {
        smx[w] = mx;
        snq[w] = nq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 1; i < int(blockDim.x >> 5); ++i) {
            mx = fmax(mx, smx[i]);
            nq = max(nq, snq[i]);
        }
        atomicMax(maxbits, static_cast<unsigned long long>(__double_as_longlong(mx)));
        atomicMax(need, nq);
    }
}

// GF(2) 64x64 matrices for the CRC append operator.
struct Gf2Mat {
    uint64_t col[64];  // image of bit i
};

inline uint64_t gf2_apply(const Gf2Mat& m, uint64_t v) {
    uint64_t r = 0;
    for (int i = 0; v; ++i, v >>= 1)
        if (v & 1) r ^= m.col[i];
    return r;
}

inline Gf2Mat gf2_mul(const Gf2Mat& a, const Gf2Mat& b) {  // a after b
    Gf2Mat r;
    for (int i = 0; i < 64; ++i) r.col[i] = gf2_apply(a, b.col[i]);
    return r;
}

// Running CRC-64/XZ whose bulk bytes may be appended as (raw CRC, length).
class Crc64Stream {
public:
    // append operator for 2^i bytes (i < 48)
    const Gf2Mat& shift_pow2(int i) const { return pow2_[i]; }
    Crc64Stream() : tb_(make_crc64_table()) {
        // one zero byte: s -> T[s & 0xff] ^ (s >> 8)
        Gf2Mat z;
        for (int i = 0; i < 64; ++i) {
            const uint64_t s = 1ull << i;
            z.col[i] = tb_.t[s & 0xff] ^ (s >> 8);
        }
        pow2_[0] = z;  // 1 byte
        for (int i = 1; i < 48; ++i) pow2_[i] = gf2_mul(pow2_[i - 1], pow2_[i - 1]);
    }
    const Crc64Table& table() const { return tb_; }
    // host bytes
    void update(const void* data, size_t len) {
        const auto* p = static_cast<const uint8_t*>(data);
        for (size_t i = 0; i < len; ++i) state_ = tb_.t[(state_ ^ p[i]) & 0xff] ^ (state_ >> 8);
    }
    // bytes whose raw CRC (zero initial state) is `raw`
    void append_raw(uint64_t raw, uint64_t len) { state_ = shift(state_, len) ^ raw; }
    uint64_t shift(uint64_t s, uint64_t len) const {
        for (int i = 0; len; ++i, len >>= 1)
            if (len & 1) s = gf2_apply(pow2_[i], s);
        return s;
    }
    uint64_t value() const { return state_ ^ ~0ull; }

private:
    Crc64Table tb_;
    Gf2Mat pow2_[48];
    uint64_t state_ = ~0ull;
};

}  // namespace pspg
