// Are the build's wall-clock stalls tied to cudaFree, or global? Thread A
// loops cudaMalloc/cudaFree (64 MB), thread B loops tiny kernel launches +
// stream syncs; every call slower than 5 ms is logged with its timestamp.
#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>
#include <cuda_runtime.h>
__global__ void tiny(int* p) { if (p) p[threadIdx.x] += 1; }
int main() {
    using C = std::chrono::steady_clock;
    const auto t0 = C::now();
    auto now_ms = [&] { return std::chrono::duration<double, std::milli>(C::now() - t0).count(); };
    cudaFree(0);
    std::atomic<bool> stop{false};
    std::thread a([&] {
        cudaSetDevice(0);
        long n = 0;
        while (!stop) {
            void* p;
            double s = now_ms();
            cudaMalloc(&p, 64 << 20);
            double m = now_ms();
            cudaFree(p);
            double f = now_ms();
            if (m - s > 5) std::printf("A %.1f malloc %.1f ms\n", s, m - s);
            if (f - m > 5) std::printf("A %.1f free %.1f ms\n", m, f - m);
            ++n;
        }
        std::printf("A iterations %ld\n", n);
    });
    std::thread b([&] {
        cudaSetDevice(0);
        cudaStream_t st;
        cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
        long n = 0;
        while (!stop) {
            double s = now_ms();
            tiny<<<1, 32, 0, st>>>(nullptr);
            cudaStreamSynchronize(st);
            double e = now_ms();
            if (e - s > 5) std::printf("B %.1f launch+sync %.1f ms\n", s, e - s);
            ++n;
        }
        std::printf("B iterations %ld\n", n);
    });
    std::this_thread::sleep_for(std::chrono::seconds(20));
    stop = true;
    a.join();
    b.join();
    return 0;
}
