// Host partitioner timing harness (no GPU, no Python):
//   g++ -O3 -std=c++20 -pthread -I paper_1503_07192_b200/csrc tools/part_bench.cpp
//       paper_1503_07192_b200/csrc/partition.cpp paper_1503_07192_b200/csrc/host_graph.cpp -o /tmp/part_bench
//   /tmp/part_bench graph.bin k threads [reps]
// graph.bin = u64 n, u64 m, u32 eu[m], u32 ev[m], f64 w[m].
// Prints the wall time per run and an FNV-1a hash of the assignment.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "host_graph.hpp"

int main(int argc, char** argv) {
    if (argc < 4) {
        std::fprintf(stderr, "usage: %s graph.bin k threads [reps]\n", argv[0]);
        return 2;
    }
    FILE* f = std::fopen(argv[1], "rb");
    if (!f) return 2;
    uint64_t hdr[2];
    if (std::fread(hdr, 8, 2, f) != 2) return 2;
    const uint64_t n = hdr[0], m = hdr[1];
    std::vector<uint32_t> eu(m), ev(m);
    std::vector<double> w(m);
    if (std::fread(eu.data(), 4, m, f) != m || std::fread(ev.data(), 4, m, f) != m ||
        std::fread(w.data(), 8, m, f) != m)
        return 2;
    std::fclose(f);
    const pspg::Csr g = pspg::build_csr(n, m, eu.data(), ev.data(), w.data());
    const uint32_t k = std::atoi(argv[2]);
    const unsigned threads = std::atoi(argv[3]);
    const int reps = argc > 4 ? std::atoi(argv[4]) : 1;
    for (int r = 0; r < reps; ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        const std::vector<uint32_t> a = pspg::partition_graph(g, k, 0, threads);
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        uint64_t h = 1469598103934665603ull;
        for (uint32_t x : a) h = (h ^ x) * 1099511628211ull;
        std::printf("partition n=%llu k=%u threads=%u: %.3f s  hash %016llx\n",
                    (unsigned long long)n, k, threads, s, (unsigned long long)h);
    }
    return 0;
}
