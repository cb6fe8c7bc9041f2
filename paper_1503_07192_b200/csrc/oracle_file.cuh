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
