// Pipe throughput microbenchmark (per SM per clock) for the ops the softmax uses:
// MUFU ex2.approx.f32, cvt.rn.f16x2.f32 (F2FP pack), fma.rn.f32x2 (FFMA2), FMNMX3, FSEL.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_tput pipe_tput.cu && ./pipe_tput
#include <cstdio>
#include <cuda_runtime.h>
constexpr int kIters = 4096, kChains = 8;
template <int OP>
__global__ void k(float* out, float seed) {
    float x[kChains];
    unsigned u[kChains];
#pragma unroll
    for (int c = 0; c < kChains; ++c) { x[c] = seed + threadIdx.x * 1e-6f + c; u[c] = threadIdx.x + c; }
    for (int i = 0; i < kIters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) {
            if (OP == 0) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(x[c]));
            if (OP == 1) asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[c]) : "f"(x[c]), "f"(__uint_as_float(u[c])));
            if (OP == 2) asm volatile("{.reg .b64 a; mov.b64 a, {%0, %1}; fma.rn.f32x2 a, a, a, a; mov.b64 {%0, %1}, a;}" : "+f"(x[c]), "+f"(x[(c + 1) % kChains]));
            if (OP == 3) asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(x[c]) : "f"(x[(c + 1) % kChains]), "f"(x[(c + 2) % kChains]));
            if (OP == 4) asm volatile("{.reg .pred p; setp.ne.b32 p, %1, 0; selp.f32 %0, %0, 0fFF800000, p;}" : "+f"(x[c]) : "r"(u[c]));
            if (OP == 5) asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(u[c]));
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c] + __uint_as_float(u[c]);
    if (s == 12345.f) out[0] = s;
}
int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    float* out;
    cudaMalloc(&out, 4);
    const char* names[] = {"MUFU ex2.f32", "F2FP cvt.f16x2.f32", "FFMA2 fma.f32x2", "FMNMX3 max3", "FSEL", "ex2.f16x2"};
    void (*ks[])(float*, float) = {k<0>, k<1>, k<2>, k<3>, k<4>, k<5>};
    for (int op = 0; op < 6; ++op) {
        const int threads = 512, blocks = sms * 4;
        ks[op]<<<blocks, threads>>>(out, 0.5f);
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        ks[op]<<<blocks, threads>>>(out, 0.5f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double ops = double(blocks) * threads * kIters * kChains;
        const double per_clk_sm = ops / (ms * 1e-3) / sms / (clk * 1e3);
        printf("%-22s %8.2f lane-ops/clk/SM (%.3f ms)\n", names[op], per_clk_sm, ms);
    }
    return 0;
}
