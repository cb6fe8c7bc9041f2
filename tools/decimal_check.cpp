// Host check of decimal_parse.cuh (the GPU graph parser's weight conversion)
// against std::from_chars, the function the reference parses weights with
// (src/graph_io.cpp:42):
//   g++ -O2 -std=c++20 -I paper_1503_07192_b200/csrc tools/decimal_check.cpp -o /tmp/decimal_check
//   /tmp/decimal_check [count]
// Every string parse_decimal accepts must give from_chars's exact bits (and
// from_chars must accept it); the acceptance rate is printed.
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>

#include "decimal_parse.cuh"

int main(int argc, char** argv) {
    const long count = argc > 1 ? std::atol(argv[1]) : 2000000;
    std::mt19937_64 rng(12345);
    long accepted = 0, bad = 0;
    char buf[64];
    for (long it = 0; it < count; ++it) {
        std::string s;
        const int form = int(rng() % 6);
        if (form == 0) {  // shortest round-trip of a random double
            uint64_t bits = rng() & 0x7fffffffffffffffull;
            double d;
            std::memcpy(&d, &bits, 8);
            if (!std::isfinite(d)) continue;
            auto r = std::to_chars(buf, buf + 64, d);
            s.assign(buf, r.ptr);
        } else if (form == 1) {  // random double in a graph-like range
            const double d = std::ldexp(double(rng() >> 11), -53) * std::pow(10.0, int(rng() % 12) - 4);
            auto r = std::to_chars(buf, buf + 64, d);
            s.assign(buf, r.ptr);
        } else if (form == 2) {  // f32 values as doubles (the road weights)
            const float f = std::ldexp(float(rng() >> 40), -24) * float(1 + rng() % 1000);
            auto r = std::to_chars(buf, buf + 64, double(f));
            s.assign(buf, r.ptr);
        } else {  // random digit strings, dots, exponents, junk
            const int len = 1 + int(rng() % 24);
            const char* alpha = form == 5 ? "0123456789.eE+-x" : "0123456789.";
            const int na = int(std::strlen(alpha));
            for (int i = 0; i < len; ++i) s.push_back(alpha[rng() % na]);
            if (form == 4 && rng() % 2) s += "e" + std::to_string(int(rng() % 700) - 350);
        }
        double mine = 0;
        if (!pspg::parse_decimal(s.data(), s.size(), mine)) continue;
        ++accepted;
        double ref = 0;
        auto [ptr, ec] = std::from_chars(s.data(), s.data() + s.size(), ref);
        uint64_t a, b;
        std::memcpy(&a, &mine, 8);
        std::memcpy(&b, &ref, 8);
        if (ec != std::errc{} || ptr != s.data() + s.size() || a != b) {
            if (++bad <= 10)
                std::printf("MISMATCH '%s': mine %.17g ref %.17g (ec %d)\n", s.c_str(), mine, ref, int(ec));
        }
    }
    std::printf("decimal_check: %ld strings, %ld accepted on the fast path, %ld mismatches\n", count,
                accepted, bad);
    return bad ? 1 : 0;
}
