// TMEM read/write throughput per SM: W warps each repeatedly tcgen05.ld (32x32b.x32 or .x16) /
// tcgen05.st of their lane quarter, `per_wait` loads between waits. Prints bytes per SM-clock.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2506_06095_b200/csrc -o tmem_bw tmem_bw.cu
#include <cstdio>
#include "tc.cuh"

namespace sf {
sf_status fail(sf_status st, const std::string&) { return st; }
void note_launch(int64_t) {}
}  // namespace sf
using namespace sf;

constexpr int kIters = 2048;

template <int MODE, int PER_WAIT>  // MODE 0: ld x32, 1: ld x16, 2: st x32
__global__ void k(unsigned long long* cyc, unsigned* sink) {
    __shared__ uint32_t tptr;
    const uint32_t warp = threadIdx.x / 32;
    if (warp == 0) tc::tmem_alloc<512>(&tptr);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tm = tptr + (((warp & 3) * 32) << 16) + 32 * ((warp >> 2) & 15);
    uint32_t acc = 0;
    uint32_t r[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) r[e] = threadIdx.x + e;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < kIters; i += PER_WAIT) {
#pragma unroll
        for (int u = 0; u < PER_WAIT; ++u) {
            if (MODE == 0) {
                tc::tmem_ld32(tm, r);
            } else if (MODE == 1) {
                uint32_t h[16];
                tc::tmem_ld16(tm, h);
#pragma unroll
                for (int e = 0; e < 16; ++e) r[e] += h[e];
            } else {
                tc::tmem_st32(tm, r);
            }
        }
        if (MODE == 2) {
            tc::tmem_st_wait();
        } else {
            tc::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 32; ++e) acc += r[e];
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (acc == 0xdeadbeef) sink[0] = acc;
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<512>(tptr);
}

template <int MODE, int PER_WAIT>
void run(int warps) {
    unsigned long long* d;
    unsigned* s;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&s, 4);
    k<MODE, PER_WAIT><<<148, 32 * warps>>>(d, s);
    k<MODE, PER_WAIT><<<148, 32 * warps>>>(d, s);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    const double bytes = (MODE == 1 ? 16.0 : 32.0) * 4 * 32 * kIters * warps;
    std::printf("%-6s per_wait %d warps %2d: %8llu cycles  %6.1f B/clk/SM  (err %s)\n",
                MODE == 0 ? "ld.x32" : MODE == 1 ? "ld.x16" : "st.x32", PER_WAIT, warps, h[0], bytes / h[0],
                cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
    cudaFree(s);
}

int main() {
    for (int w : {4, 8, 16}) {
        run<0, 1>(w);
        run<0, 2>(w);
        run<1, 2>(w);
        run<2, 1>(w);
        run<2, 4>(w);
    }
    return 0;
}
