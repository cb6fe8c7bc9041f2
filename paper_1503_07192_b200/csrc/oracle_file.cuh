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
constexpr uint32_t CRC_SEG = 4096;                      // bytes per GPU segment

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

// Raw (init 0, no final xor) CRC of each CRC_SEG-byte segment; the last
// segment may be short.
__global__ void crc64_segments(const uint8_t* __restrict__ data, uint64_t len, Crc64Table tb,
                               uint64_t* __restrict__ out) {
    __shared__ uint64_t t[256];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) t[i] = tb.t[i];
    __syncthreads();
    const uint64_t seg = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const uint64_t begin = seg * CRC_SEG;
    if (begin >= len) return;
    const uint64_t end = min(len, begin + CRC_SEG);
    uint64_t crc = 0;
    uint64_t i = begin;
    for (; i + 8 <= end; i += 8) {
        uint64_t w = *reinterpret_cast<const uint64_t*>(data + i);  // 8-byte aligned
#pragma unroll
        for (int b = 0; b < 8; ++b) {
            crc = t[(crc ^ w) & 0xff] ^ (crc >> 8);
            w >>= 8;
        }
    }
    for (; i < end; ++i) crc = t[(crc ^ data[i]) & 0xff] ^ (crc >> 8);
    out[seg] = crc;
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
