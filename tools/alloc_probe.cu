// Host latency of cudaMalloc / cudaFree / fill on this box (diagnostic for
// the build's wall-clock noise): sizes 16 MB .. 8 GB, 5 rounds each.
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    using C = std::chrono::steady_clock;
    auto ms = [](C::time_point a) { return std::chrono::duration<double, std::milli>(C::now() - a).count(); };
    cudaFree(0);
    for (size_t mb : {16ul, 256ul, 2048ul, 8192ul})
        for (int r = 0; r < 5; ++r) {
            void* p = nullptr;
            auto t = C::now();
            cudaMalloc(&p, mb << 20);
            const double a = ms(t);
            t = C::now();
            cudaMemset(p, 0, mb << 20);
            cudaDeviceSynchronize();
            const double f = ms(t);
            t = C::now();
            cudaFree(p);
            const double d = ms(t);
            std::printf("%5zu MB round %d: malloc %.2f ms, memset %.2f ms, free %.2f ms\n", mb, r, a, f, d);
        }
    return 0;
}
