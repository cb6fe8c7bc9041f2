// decimal_parse.cuh — exact decimal -> binary64 for the GPU graph parser.
//
// The reference parses weights with std::from_chars (src/graph_io.cpp:42),
// i.e. correctly rounded. This is the Eisel-Lemire algorithm (Lemire,
// "Number parsing at a gigabyte per second", Software: Practice and
// Experience 51(8), 2021; the fast_float library's compute_float with the
// proof that the 128-bit product always suffices for <= 19 digits), written
// for __host__ __device__ so the host build can be checked exhaustively
// against from_chars (tools/decimal_check.cpp).
//
// parse_decimal() accepts the plain grammar digits[.digits][(e|E)[+-]digits]
// with at most 19 significant digits and a normal (finite, non-subnormal,
// non-zero unless the digits are all zero) result. Everything else --
// signs, "inf"/"nan", longer mantissas, out-of-range or subnormal results,
// malformed text -- returns false and is left to the host's from_chars,
// which also produces the reference's error for it.
#pragma once
#include <cstdint>

#include "pow5_table.cuh"

#if defined(__CUDACC__)
#define PSPG_HD __host__ __device__
#else
#define PSPG_HD
#endif

namespace pspg {

PSPG_HD inline void mul_64x64(uint64_t a, uint64_t b, uint64_t& hi, uint64_t& lo) {
#if defined(__CUDA_ARCH__)
    lo = a * b;
    hi = __umul64hi(a, b);
#else
    const unsigned __int128 r = static_cast<unsigned __int128>(a) * b;
    lo = static_cast<uint64_t>(r);
    hi = static_cast<uint64_t>(r >> 64);
#endif
}

PSPG_HD inline int clz_64(uint64_t x) {
#if defined(__CUDA_ARCH__)
    return __clzll(static_cast<long long>(x));
#else
    return __builtin_clzll(x);
#endif
}

PSPG_HD inline const uint64_t* pow5_table() {
#if defined(__CUDA_ARCH__)
    return kPow5;
#else
    return kPow5Host;
#endif
}

// w * 10^q (w != 0, POW5_MIN_Q <= q <= POW5_MAX_Q) correctly rounded to a
// binary64; false when the result is not a normal finite number.
PSPG_HD inline bool eisel_lemire(uint64_t w, int q, double& out) {
    constexpr int kMant = 52, kMinExp = -1023, kInf = 0x7FF;
    const int lz = clz_64(w);
    w <<= lz;
    const uint64_t* t = pow5_table() + 2 * (q - POW5_MIN_Q);
    uint64_t hi, lo;
    mul_64x64(w, t[0], hi, lo);
    constexpr uint64_t mask = ~uint64_t(0) >> (kMant + 3);
    if ((hi & mask) == mask) {  // refine with the next 64 bits of 5^q
        uint64_t hi2, lo2;
        mul_64x64(w, t[1], hi2, lo2);
        lo += hi2;
        if (hi2 > lo) ++hi;
    }
    const int upper = static_cast<int>(hi >> 63);
    const int shift = upper + 64 - kMant - 3;
    uint64_t mant = hi >> shift;
    int p2 = static_cast<int>(((152170 + 65536) * static_cast<int64_t>(q)) >> 16) + 63 + upper - lz -
             kMinExp;
    if (p2 <= 0) return false;  // subnormal or zero: from_chars decides
    // round to even on an exact halfway case (only possible for small q)
    if (lo <= 1 && q >= -4 && q <= 23 && (mant & 3) == 1 && (mant << shift) == hi) mant &= ~uint64_t(1);
    mant += mant & 1;
    mant >>= 1;
    if (mant >= (uint64_t(2) << kMant)) {
        mant = uint64_t(1) << kMant;
        ++p2;
    }
    mant &= ~(uint64_t(1) << kMant);
    if (p2 >= kInf) return false;  // overflow: from_chars reports it
    const uint64_t bits = (static_cast<uint64_t>(p2) << kMant) | mant;
#if defined(__CUDA_ARCH__)
    out = __longlong_as_double(static_cast<long long>(bits));
#else
    __builtin_memcpy(&out, &bits, 8);
#endif
    return true;
}

// Parses s[0..n) completely; see the file comment for what it declines.
PSPG_HD inline bool parse_decimal(const char* s, uint64_t n, double& out) {
    uint64_t i = 0, w = 0;
    int digits = 0;     // significant digits taken into w
    int dexp = 0;       // decimal exponent adjustment from the '.'
    bool any = false, dot = false;
    for (; i < n; ++i) {
        const char c = s[i];
        if (c == '.') {
            if (dot) return false;
            dot = true;
            continue;
        }
        const unsigned d = static_cast<unsigned char>(c) - '0';
        if (d > 9) break;
        any = true;
        if (w == 0 && d == 0) {  // leading zero: not significant
            if (dot) --dexp;
            continue;
        }
        if (++digits > 19) return false;
        w = w * 10 + d;
        if (dot) --dexp;
    }
    if (!any) return false;
    if (i < n) {  // exponent
        if (s[i] != 'e' && s[i] != 'E') return false;
        ++i;
        bool neg = false;
        if (i < n && (s[i] == '+' || s[i] == '-')) {
            neg = s[i] == '-';
            ++i;
        }
        if (i >= n) return false;
        int e = 0;
        for (; i < n; ++i) {
            const unsigned d = static_cast<unsigned char>(s[i]) - '0';
            if (d > 9) return false;
            if (e < 100000) e = e * 10 + static_cast<int>(d);
        }
        dexp += neg ? -e : e;
    }
    if (w == 0) {
        out = 0.0;
        return true;
    }
    if (dexp < POW5_MIN_Q || dexp > POW5_MAX_Q) return false;
    return eisel_lemire(w, dexp, out);
}

}  // namespace pspg
