// pcie_probe.cu — the floor under the point-query server's latency: how long
// a GPU takes to read mapped pinned host memory, and a host <-> GPU ping-pong
// through it (host writes a word, a resident GPU thread polls for it and
// writes an answer word back, the host polls for that), with 1, 2 or 4 GPU
// polls in flight.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/pcie_probe tools/pcie_probe.cu
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ unsigned long long ldv(const volatile unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// dependent loads: each address depends on the previous value
__global__ void read_latency(const volatile unsigned long long* host, int iters,
                             unsigned long long* out, unsigned long long* ns) {
    unsigned long long t0, t1, idx = 0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (int i = 0; i < iters; ++i) idx = ldv(host + (idx & 7));
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    *out = idx;
    *ns = t1 - t0;
}

template <int INFLIGHT>
__global__ void echo(volatile unsigned long long* req, volatile unsigned long long* ans, int iters) {
    unsigned long long last = 0;
    unsigned long long v[INFLIGHT];
#pragma unroll
    for (int s = 0; s < INFLIGHT; ++s) {
        v[s] = ldv(req);
        __nanosleep(2000 / INFLIGHT);
    }
    for (int done = 0; done < iters;) {
#pragma unroll
        for (int s = 0; s < INFLIGHT; ++s) {
            const unsigned long long x = v[s];
            v[s] = ldv(req);
            if (x != last) {
                last = x;
                *ans = x;
                ++done;
            }
        }
    }
}

int main() {
    unsigned long long* h = nullptr;
    CK(cudaHostAlloc(&h, 4096, cudaHostAllocMapped | cudaHostAllocPortable));
    for (int i = 0; i < 512; ++i) h[i] = 0;
    unsigned long long *d_out, *d_ns;
    CK(cudaMalloc(&d_out, 8));
    CK(cudaMalloc(&d_ns, 8));
    read_latency<<<1, 1>>>(h, 2000, d_out, d_ns);
    CK(cudaDeviceSynchronize());
    unsigned long long ns = 0;
    CK(cudaMemcpy(&ns, d_ns, 8, cudaMemcpyDeviceToHost));
    std::printf("{\"gpu_read_of_host_memory_ns\": %.1f", ns / 2000.0);
    volatile unsigned long long* req = h + 64;
    volatile unsigned long long* ans = h + 128;
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    const int iters = 100000;
    auto pingpong = [&](auto kernel, const char* name) -> int {
        *req = 0;
        *ans = 0;
        kernel<<<1, 1, 0, s>>>(req, ans, iters);
        const auto t0 = std::chrono::steady_clock::now();
        for (unsigned long long i = 1; i <= (unsigned long long)iters; ++i) {
            *req = i;
            std::atomic_thread_fence(std::memory_order_seq_cst);
            while (*ans != i) {
            }
        }
        const double us =
            std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        CK(cudaStreamSynchronize(s));
        std::printf(", \"%s_us\": %.3f", name, us / iters);
        return 0;
    };
    if (pingpong(echo<1>, "pingpong_1_poll")) return 1;
    if (pingpong(echo<2>, "pingpong_2_polls")) return 1;
    if (pingpong(echo<4>, "pingpong_4_polls")) return 1;
    if (pingpong(echo<8>, "pingpong_8_polls")) return 1;
    std::printf("}\n");
    return 0;
}
