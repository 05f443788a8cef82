// Probe of the tcgen05 M=64 (cta_group::1) TMEM layouts the 64-row attention design relies on:
//   (1) SS MMA M=64 N=64 K=64 with D at TMEM lane offset 0 and 16: rows of the two tiles land in
//       lanes {16q + (0..15)} + 32q... i.e. row r -> DP (r % 16) + 32 * (r / 16) (+16 for tile B);
//   (2) TS MMA M=64 with A (P, packed fp16) read from TMEM at the same lane offsets.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2506_06095_b200/csrc -o umma64 umma64.cu
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>
#include "tc.cuh"

namespace sf {
sf_status fail(sf_status st, const std::string&) { return st; }
void note_launch(int64_t) {}
}
using namespace sf;

// K-major SW128 tile of R rows x 64 fp16 (128 B rows, 8-row 1024-B atoms)
__device__ void store_sw128(unsigned char* base, int r, int c16, uint4 v) {
    *reinterpret_cast<uint4*>(base + r * 128 + ((c16 ^ (r & 7)) << 4)) = v;
}

__global__ void probe(const __half* q2, const __half* k2, const __half* v2, float* s_out, float* o_out) {
    // q2: [2][64][64] (tiles A, B), k2: [2][64 keys][64], v2: [2][64 keys][64 d]
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    unsigned char (*sQ)[8192] = reinterpret_cast<unsigned char (*)[8192]>(base);
    unsigned char (*sK)[8192] = reinterpret_cast<unsigned char (*)[8192]>(base + 16384);
    unsigned char (*sV)[8192] = reinterpret_cast<unsigned char (*)[8192]>(base + 32768);
    __shared__ uint64_t bar;
    __shared__ uint32_t tptr;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
    for (int i = t; i < 2 * 64 * 8; i += blockDim.x) {
        const int tile = i / 512, r = (i / 8) % 64, c = i % 8;
        store_sw128(sQ[tile], r, c, reinterpret_cast<const uint4*>(q2 + tile * 4096 + r * 64)[c]);
        store_sw128(sK[tile], r, c, reinterpret_cast<const uint4*>(k2 + tile * 4096 + r * 64)[c]);
        store_sw128(sV[tile], r, c, reinterpret_cast<const uint4*>(v2 + tile * 4096 + r * 64)[c]);  // MN-major V
    }
    if (t == 0) { tc::mbar_init(&bar, 1); tc::fence_barrier_init(); }
    if (warp == 0) tc::tmem_alloc<256>(&tptr);
    tc::fence_proxy_async();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tptr;
    const uint32_t idesc_s = tc::idesc_f16(64, 64, 0, 0, 0), idesc_o = tc::idesc_f16(64, 64, 0, 0, 1);
    if (warp == 0 && tc::elect_one()) {
        for (int tile = 0; tile < 2; ++tile)
            for (int k = 0; k < 4; ++k)
                tc::mma_f16_ss(tmem + ((16u * tile) << 16), tc::sdesc_sw128(tc::smem_u32(sQ[tile]) + 32 * k),
                               tc::sdesc_sw128(tc::smem_u32(sK[tile]) + 32 * k), idesc_s, k != 0);
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 0);
    tc::fence_after_sync();
    // read S back: lane L of warp q holds DP 32q + L
    uint32_t raw[32], raw2[32];
    tc::tmem_ld32(tmem + ((32u * warp) << 16), raw);
    tc::tmem_ld32(tmem + ((32u * warp) << 16) + 32, raw2);
    tc::tmem_ld_wait();
    const int dp = 32 * warp + lane;
    for (int c = 0; c < 32; ++c) {
        s_out[dp * 64 + c] = __uint_as_float(raw[c]);
        s_out[dp * 64 + 32 + c] = __uint_as_float(raw2[c]);
    }
    // P = S as fp16 pairs into TMEM cols 64..95 at the same lanes, then O = P V (TS MMA, M=64)
    uint32_t pk[32];
    for (int c = 0; c < 32; ++c) {
        const float a = c < 16 ? __uint_as_float(raw[2 * c]) : __uint_as_float(raw2[2 * c - 32]);
        const float b = c < 16 ? __uint_as_float(raw[2 * c + 1]) : __uint_as_float(raw2[2 * c - 31]);
        __half2 h = __floats2half2_rn(a * 0.01f, b * 0.01f);
        pk[c] = *reinterpret_cast<uint32_t*>(&h);
    }
    tc::tmem_st32(tmem + ((32u * warp) << 16) + 64, pk);
    tc::tmem_st_wait();
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    if (warp == 0 && tc::elect_one()) {
        for (int tile = 0; tile < 2; ++tile)
            for (int k = 0; k < 4; ++k)
                tc::mma_f16_ts(tmem + 128 + ((16u * tile) << 16), tmem + 64 + ((16u * tile) << 16) + 8 * k,
                               tc::sdesc_sw128_mn(tc::smem_u32(sV[tile]) + 2048 * k), idesc_o, k != 0);
        tc::mma_commit(&bar);
    }
    tc::mbar_wait(&bar, 1);
    tc::fence_after_sync();
    tc::tmem_ld32(tmem + ((32u * warp) << 16) + 128, raw);
    tc::tmem_ld32(tmem + ((32u * warp) << 16) + 160, raw2);
    tc::tmem_ld_wait();
    for (int c = 0; c < 32; ++c) {
        o_out[dp * 64 + c] = __uint_as_float(raw[c]);
        o_out[dp * 64 + 32 + c] = __uint_as_float(raw2[c]);
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc<256>(tmem);
}

int main() {
    std::vector<__half> q(8192), k(8192), v(8192);
    std::vector<float> qf(8192), kf(8192), vf(8192);
    srand(1);
    for (int i = 0; i < 8192; ++i) {
        qf[i] = __half2float(q[i] = __float2half((rand() % 17 - 8) / 8.f));
        kf[i] = __half2float(k[i] = __float2half((rand() % 17 - 8) / 8.f));
        vf[i] = __half2float(v[i] = __float2half((rand() % 17 - 8) / 8.f));
    }
    __half *dq, *dk, *dv; float *ds, *dO;
    cudaMalloc(&dq, 16384); cudaMalloc(&dk, 16384); cudaMalloc(&dv, 16384);
    cudaMalloc(&ds, 128 * 64 * 4); cudaMalloc(&dO, 128 * 64 * 4);
    cudaMemcpy(dq, q.data(), 16384, cudaMemcpyHostToDevice);
    cudaMemcpy(dk, k.data(), 16384, cudaMemcpyHostToDevice);
    cudaMemcpy(dv, v.data(), 16384, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 50 * 1024);
    probe<<<1, 128, 50 * 1024>>>(dq, dk, dv, ds, dO);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("cuda error %s\n", cudaGetErrorString(e)); return 1; }
    std::vector<float> s(128 * 64), o(128 * 64);
    cudaMemcpy(s.data(), ds, s.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(o.data(), dO, o.size() * 4, cudaMemcpyDeviceToHost);
    // expected: DP = (r % 16) + 32 * (r / 16) + 16 * tile
    double es = 0, eo = 0;
    for (int tile = 0; tile < 2; ++tile)
        for (int r = 0; r < 64; ++r) {
            const int dp = (r % 16) + 32 * (r / 16) + 16 * tile;
            std::vector<float> p(64);
            for (int j = 0; j < 64; ++j) {
                float acc = 0;
                for (int d = 0; d < 64; ++d) acc += qf[tile * 4096 + r * 64 + d] * kf[tile * 4096 + j * 64 + d];
                es = std::max(es, (double)std::fabs(acc - s[dp * 64 + j]));
                p[j] = __half2float(__float2half(acc * 0.01f));
            }
            for (int d = 0; d < 64; ++d) {
                float acc = 0;
                for (int j = 0; j < 64; ++j) acc += p[j] * vf[tile * 4096 + j * 64 + d];
                eo = std::max(eo, (double)std::fabs(acc - o[dp * 64 + d]));
            }
        }
    printf("M=64 two-tile layout: max |S - ref| = %.3g, max |O - ref| = %.3g -> %s\n", es, eo,
           (es < 1e-2 && eo < 1e-2) ? "MATCH" : "MISMATCH");
    return 0;
}
