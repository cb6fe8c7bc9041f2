// minplus_probe.cu — measures the min-plus ALU peak of this GPU, and which
// instruction mix reaches it. The roofline denominator for K1/K2 (BASELINE.md
// §3: "ALU min-plus peak: to be microbenchmarked").
//
// Every variant performs the same FW-shaped work: an 8x8 register block of
// accumulators relaxed against 8 row values and 8 column values per k-step,
// with the operands rotated through the accumulators so nothing folds.
//   viaddmnmx  acc = min(a + b, acc)                 1 VIADDMNMX.U32 / relax
//   imad_min3  acc = min3(acc, a*1+b, a'*1+b')       2 IMAD + 1 VIMNMX3 / 2 relax
//   mix3       one viaddmnmx step + one imad_min3    (ALU: 2/3 instr per relax,
//                                                    FMA: 2/3 -> balanced pipes)
//   f32        fminf(fminf(acc, a+b), a'+b')         2 FADD + 1 FMNMX3 / 2 relax
//   f32_ffma   fma(a, one, b) instead of a + b       2 FFMA + 1 FMNMX3 / 2 relax
//   u16x2      __viaddmin_u16x2 (DPX): two 16-bit relaxations per
//              VIADDMNMX.U16x2 (packed halves)
// `one` is a kernel argument equal to 1, so the compiler cannot fold a*one+b
// into the add-min instruction.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o minplus_probe minplus_probe.cu
// Run:   ./minplus_probe > profiles/minplus_peak_r1.json
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

enum { VIADD = 0, IMAD_MIN3 = 1, MIX3 = 2, F32 = 3, F32_FFMA = 4, U16X2 = 5 };

template <int MODE, class V>
__global__ void __launch_bounds__(256) probe(V* out, uint32_t iters, V one) {
    V acc[8][8], a[8], b[8], c[8], d[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        a[i] = V(threadIdx.x & 7) + V(i);
        b[i] = V(i * 3);
        c[i] = V(i + 1);
        d[i] = V(2 * i);
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = V(1000 + i * 8 + j);
    }
    for (uint32_t it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if constexpr (MODE == VIADD) {
                    acc[i][j] = min(a[i] + b[j], acc[i][j]);
                    acc[i][j] = min(c[i] + d[j], acc[i][j]);
                } else if constexpr (MODE == IMAD_MIN3) {
                    acc[i][j] = __vimin3_u32(acc[i][j], a[i] * one + b[j], c[i] * one + d[j]);
                } else if constexpr (MODE == MIX3) {
                    // three relaxations: one fused, two through IMAD + VIMNMX3
                    V t = min(a[i] + b[j], acc[i][j]);
                    acc[i][j] = __vimin3_u32(t, c[i] * one + d[j], a[i] * one + d[j]);
                } else if constexpr (MODE == U16X2) {
                    acc[i][j] = __viaddmin_u16x2(a[i], b[j], acc[i][j]);
                    acc[i][j] = __viaddmin_u16x2(c[i], d[j], acc[i][j]);
                } else if constexpr (MODE == F32) {
                    acc[i][j] = fminf(fminf(acc[i][j], a[i] + b[j]), c[i] + d[j]);
                } else {
                    acc[i][j] = fminf(fminf(acc[i][j], fmaf(a[i], one, b[j])),
                                      fmaf(c[i], one, d[j]));
                }
            }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            a[i] = acc[i][(i + 1) & 7];
            b[i] = acc[(i + 3) & 7][i];
            c[i] = acc[(i + 5) & 7][(i + 2) & 7];
            d[i] = acc[(i + 6) & 7][(i + 7) & 7];
        }
    }
    V s = acc[0][0];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) s = s < acc[i][j] ? s : acc[i][j];
    if (s == V(12345)) out[blockIdx.x] = s;
}

__global__ void dpx_semantics(unsigned* out) {
    out[0] = __viaddmin_u16x2(0x0000fff0u, 0x00000020u, 0xffffffffu);
    out[1] = __viaddmin_u16x2(0x00008000u, 0x00008000u, 0xffffffffu);
    out[2] = __viaddmin_u16x2(0x00000003u, 0x00000004u, 0x00000009u);
    out[3] = __viaddmin_u16x2(0x7fff0000u, 0x7fff0000u, 0xffffffffu);
}

template <int MODE, class V>
int run(const char* name, int relax_per_iter, int sms, bool last) {
    V* out;
    CK(cudaMalloc(&out, sizeof(V) * sms * 64));
    const int blocks = sms * 4;
    const uint32_t iters = 1 << 13;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 4; ++rep) {
        CK(cudaEventRecord(e0));
        probe<MODE, V><<<blocks, 256>>>(out, iters, V(1));
        CK(cudaGetLastError());
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (rep > 0 && ms < best) best = ms;
    }
    const double relax = double(blocks) * 256 * 64 * relax_per_iter * iters;
    const double rate = relax / (best * 1e-3);
    int khz = 0;
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0);
    printf("    \"%s\": {\"relax_per_s\": %.4e, \"relax_per_clk_per_sm_at_max_clock\": %.2f, "
           "\"ms\": %.3f}%s\n",
           name, rate, rate / (sms * khz * 1e3), best, last ? "" : ",");
    cudaFree(out);
    return 0;
}

int main() {
    int sms = 0, khz = 0;
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, 0));
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"max_sm_mhz\": %.0f,\n  \"variants\": {\n", p.name,
           sms, khz / 1e3);
    if (run<VIADD, uint32_t>("u32_viaddmnmx", 2, sms, false)) return 1;
    if (run<IMAD_MIN3, uint32_t>("u32_imad_vimnmx3", 2, sms, false)) return 1;
    if (run<MIX3, uint32_t>("u32_mix_viaddmnmx_imad_vimnmx3", 3, sms, false)) return 1;
    if (run<F32, float>("f32_fadd_fmnmx3", 2, sms, false)) return 1;
    if (run<F32_FFMA, float>("f32_ffma_fmnmx3", 2, sms, false)) return 1;
    // two 16-bit relaxations per instruction
    if (run<U16X2, uint32_t>("u16x2_viaddmnmx", 4, sms, true)) return 1;
    printf("  },\n");
    // semantics of the packed add: wrap or saturate at 0xffff?
    unsigned* d;
    CK(cudaMalloc(&d, 16));
    dpx_semantics<<<1, 1>>>(d);
    unsigned h[4];
    CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
    printf("  \"u16x2_semantics\": {\"min(0xfff0+0x0020, 0xffff)\": \"0x%04x\", "
           "\"min(0x8000+0x8000, 0xffff)\": \"0x%04x\", \"min(0x0003+0x0004, 0x0009)\": "
           "\"0x%04x\", \"hi half min(0x7fff+0x7fff, 0xffff)\": \"0x%04x\"}\n}\n",
           h[0] & 0xffff, h[1] & 0xffff, h[2] & 0xffff, h[3] >> 16);
    return 0;
}
