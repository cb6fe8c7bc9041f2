// Where the build's allocation time goes (diagnostic for a physical-memory
// pool filled while the host partitions): per size, cudaMalloc vs the VMM
// steps (cuMemCreate, cuMemAddressReserve + cuMemMap + cuMemSetAccess) and
// the first touch; the same sizes twice, the second time after the first
// round freed its memory (the bench's situation: big frees, then a build).
//   nvcc -O2 -arch=sm_100a tools/alloc_probe2.cu -lcuda -o /tmp/alloc_probe2
#include <chrono>
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>
#include <vector>

using Clk = std::chrono::steady_clock;
static double ms(Clk::time_point a) { return std::chrono::duration<double, std::milli>(Clk::now() - a).count(); }

int main() {
    cudaFree(0);
    CUmemAllocationProp prop{};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = 0;
    size_t gran = 0;
    cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED);
    std::printf("granularity %zu\n", gran);
    for (int round = 0; round < 2; ++round) {
        for (size_t gb : {1ul, 8ul, 36ul, 48ul}) {
            const size_t bytes = gb << 30;
            void* p = nullptr;
            auto t = Clk::now();
            cudaError_t e = cudaMalloc(&p, bytes);
            const double a = ms(t);
            t = Clk::now();
            cudaMemsetAsync(p, 0, bytes);
            cudaDeviceSynchronize();
            const double touch = ms(t);
            t = Clk::now();
            cudaFree(p);
            const double fr = ms(t);
            // VMM: physical in 2 GB chunks
            const size_t chunk = size_t(2) << 30, nch = (bytes + chunk - 1) / chunk;
            std::vector<CUmemGenericAllocationHandle> h(nch);
            t = Clk::now();
            for (auto& x : h) cuMemCreate(&x, chunk, &prop, 0);
            const double create = ms(t);
            CUdeviceptr va = 0;
            t = Clk::now();
            cuMemAddressReserve(&va, nch * chunk, gran, 0, 0);
            for (size_t i = 0; i < nch; ++i) cuMemMap(va + i * chunk, chunk, 0, h[i], 0);
            CUmemAccessDesc acc{};
            acc.location = prop.location;
            acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
            cuMemSetAccess(va, nch * chunk, &acc, 1);
            const double map = ms(t);
            t = Clk::now();
            cudaMemsetAsync(reinterpret_cast<void*>(va), 0, nch * chunk);
            cudaDeviceSynchronize();
            const double vtouch = ms(t);
            t = Clk::now();
            for (size_t i = 0; i < nch; ++i) cuMemUnmap(va + i * chunk, chunk);
            cuMemAddressFree(va, nch * chunk);
            for (auto& x : h) cuMemRelease(x);
            const double vfree = ms(t);
            std::printf("round %d %3zu GB: cudaMalloc %7.2f (%s) touch %6.2f free %7.2f | cuMemCreate %7.2f map %6.2f touch %6.2f release %7.2f ms\n",
                        round, gb, a, e == cudaSuccess ? "ok" : "fail", touch, fr, create, map, vtouch, vfree);
        }
    }
    return 0;
}
