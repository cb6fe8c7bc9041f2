// latency_probe.cpp — single-query latency through the C-ABI (the path the
// reference's query(o, u, v) takes through the shim): builds the 44x44 unit
// grid oracle of acceptance criterion 1 (k = 44), then times
//   host     psp_gpu_query_batch(count = 1) calls, answered by the point-query
//            server (mailbox in mapped host memory);
//   launch   the same with PSP_NO_QUERY_SERVER (kernel launch + sync per call);
// and prints per-call microseconds.
//
// Build: g++ -O2 -std=c++17 -Iinclude tools/latency_probe.cpp \
//          -Lpaper_1503_07192_b200 -l:libpsp_gpu.so -Wl,-rpath,$PWD/paper_1503_07192_b200
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "psp_gpu.h"

#define CK(x) do { psp_status s_ = (x); if (s_ != PSP_OK) { \
    std::fprintf(stderr, "%s: %s\n", #x, psp_gpu_last_error()); return 1; } } while (0)

int main(int argc, char** argv) {
    const int side = argc > 1 ? std::atoi(argv[1]) : 44;
    const int k = argc > 2 ? std::atoi(argv[2]) : side;
    const int calls = argc > 3 ? std::atoi(argv[3]) : 200000;
    psp_gpu_ctx* ctx = nullptr;
    CK(psp_gpu_ctx_create(0, 0, 1, nullptr, &ctx));
    uint64_t m = 0;
    CK(psp_generate_grid(0, side, side, 1, 1.0, 1.0, 0, &m, nullptr, nullptr, nullptr));
    std::vector<uint32_t> eu(m), ev(m);
    std::vector<double> ew(m);
    CK(psp_generate_grid(0, side, side, 1, 1.0, 1.0, 0, &m, eu.data(), ev.data(), ew.data()));
    const uint64_t n = uint64_t(side) * side;
    psp_gpu_oracle* o = nullptr;
    psp_build_stats st{};
    CK(psp_gpu_build_oracle(ctx, n, m, eu.data(), ev.data(), ew.data(), k, 1, 0, PSP_VALUE_AUTO,
                            &o, &st));
    auto run = [&](const char* name) -> int {
        double d = 0, sum = 0;
        for (int i = 0; i < 1000; ++i) {  // warm-up
            uint32_t a = i % n, b = (i * 7) % n;
            CK(psp_gpu_query_batch(o, 1, &a, &b, &d, nullptr));
        }
        const auto t0 = std::chrono::steady_clock::now();
        for (int i = 0; i < calls; ++i) {
            uint32_t a = i % n, b = (i * 13 + 5) % n;
            CK(psp_gpu_query_batch(o, 1, &a, &b, &d, nullptr));
            sum += d;
        }
        const double us =
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        std::printf("{\"path\": \"%s\", \"grid\": %d, \"k\": %d, \"calls\": %d, \"us_per_call\": %.3f, "
                    "\"checksum\": %.1f}\n", name, side, k, calls, us / calls, sum);
        return 0;
    };
    if (run("point-query server")) return 1;
    setenv("PSP_NO_QUERY_SERVER", "1", 1);
    if (run("launch per call")) return 1;
    unsetenv("PSP_NO_QUERY_SERVER");
    psp_gpu_oracle_free(o);
    psp_gpu_ctx_destroy(ctx);
    return 0;
}
