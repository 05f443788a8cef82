// Cost of the attention kernel's tensor-core step without data movement or softmax math:
//   mode 0  throughput: one thread issues S = Q K^T (SS, M=128 N=NS K=64 as K=16 MMAs) and
//           O += P V (TS: P from TMEM, N=64, K=NS) back to back, one commit per step, no waits
//   mode 1  S latency: 4 SS MMAs + commit, then wait for that commit before the next step
//   mode 2  the kernel's two-buffer ping-pong with a zero-math "softmax": 4 warps wait S_j,
//           tcgen05.ld it (2 x 32 columns), arrive; the issuer waits that arrive, issues P_j V_j and
//           S_{j+2} (what attn_tc does per 64-key step, minus TMA and math)
// Grid = CTAS_PER_SM x 148. Prints cycles per step (clock64 of CTA 0).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2506_06095_b200/csrc -o mma_pipe mma_pipe.cu
#include <cstdio>
#include <cstdlib>
#include "tc.cuh"

namespace sf {
sf_status fail(sf_status st, const std::string&) { return st; }
void note_launch(int64_t) {}
}  // namespace sf
using namespace sf;

template <int NS>
__global__ void __launch_bounds__(192, 1) pipe(int mode, int steps, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    unsigned char* sQ = base;               // 128 x 64 fp16 (16 KB)
    unsigned char* sK = base + 16384;       // NS x 64
    unsigned char* sV = sK + NS * 128;      // NS x 64
    __shared__ uint64_t s_full[2], p_full[2], done;
    __shared__ uint32_t tmem_base;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2; ++i) { tc::mbar_init(&s_full[i], 1); tc::mbar_init(&p_full[i], 128); }
        tc::mbar_init(&done, 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<256>(&tmem_base);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = tmem_base;
    constexpr uint32_t idesc_s = tc::idesc_f16(128, NS, 0, 0, 0);
    constexpr uint32_t idesc_o = tc::idesc_f16(128, 64, 0, 0, 1);
    // S[b] at cols b*NS (NS <= 96 so 2 buffers + P + O fit in 256), P at 2*NS..., O at 192
    const uint32_t tP = tmem + (NS == 64 ? 128 : 0), tO = tmem + 192;
    auto issue_s = [&](int j) {
        const uint32_t d = tmem + (NS == 64 ? 64 * (j & 1) : 0);
#pragma unroll
        for (int k = 0; k < 4; ++k)
            tc::mma_f16_ss(d, tc::sdesc_sw128(tc::smem_u32(sQ) + 32 * k), tc::sdesc_sw128(tc::smem_u32(sK) + 32 * k),
                           idesc_s, k != 0);
    };
    auto issue_pv = [&](int j) {
#pragma unroll
        for (int k = 0; k < NS / 16; ++k)
            tc::mma_f16_ts(tO, tP + 32 * (j & 1) * (NS == 64) + 8 * k, tc::sdesc_sw128_mn(tc::smem_u32(sV) + 2048 * k),
                           idesc_o, 1);
    };
    unsigned long long t0 = clock64();
    if (mode == 0) {
        if (warp == 1 && tc::elect_one()) {
            for (int j = 0; j < steps; ++j) {
                issue_s(j);
                issue_pv(j);
                tc::mma_commit(&s_full[j & 1]);
            }
            tc::mma_commit(&done);
            tc::mbar_wait(&done, 0);
        }
    } else if (mode == 1) {
        if (warp == 1 && tc::elect_one()) {
            for (int j = 0; j < steps; ++j) {
                issue_s(j);
                tc::mma_commit(&s_full[0]);
                tc::mbar_wait(&s_full[0], j & 1);
            }
        }
    } else {
        if (warp == 1) {
            if (tc::elect_one()) {
                issue_s(0);
                tc::mma_commit(&s_full[0]);
                issue_s(1);
                tc::mma_commit(&s_full[1]);
                for (int j = 0; j < steps; ++j) {
                    tc::mbar_wait(&p_full[j & 1], (j >> 1) & 1);
                    tc::fence_after_sync();
                    issue_pv(j);
                    if (j + 2 < steps) {
                        issue_s(j + 2);
                        tc::mma_commit(&s_full[j & 1]);
                    }
                }
                tc::mma_commit(&done);
                tc::mbar_wait(&done, 0);
            }
        } else if (warp >= 2) {
            const uint32_t q = warp & 3;
            for (int j = 0; j < steps; ++j) {
                tc::mbar_wait(&s_full[j & 1], (j >> 1) & 1);
                tc::fence_after_sync();
                uint32_t r0[32], r1[32];
                tc::tmem_ld32(tmem + ((q * 32) << 16) + 64 * (j & 1), r0);
                tc::tmem_ld32(tmem + ((q * 32) << 16) + 64 * (j & 1) + 32, r1);
                tc::tmem_ld_wait();
                if (r0[5] == 0x12345u && r1[7] == 0x777u) out[1] = 1;  // keep the loads
                tc::fence_before_sync();
                tc::mbar_arrive(&p_full[j & 1]);
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 32 && blockIdx.x == 0) out[0] = clock64() - t0;
    if (warp == 1) tc::tmem_dealloc<256>(tmem);
}

int main(int argc, char** argv) {
    unsigned long long* d;
    cudaMalloc(&d, 16);
    const int steps = 4096;
    for (int per_sm : {1, 2}) {
        for (int mode : {0, 1, 2}) {
            for (int ns : {64, 96}) {
                if (ns == 96 && mode == 2) continue;
                auto k = ns == 64 ? pipe<64> : pipe<96>;
                const int smem = 16384 + 2 * ns * 128 + 2048;
                cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
                k<<<148 * per_sm, 192, smem>>>(mode, steps, d);  // warm
                k<<<148 * per_sm, 192, smem>>>(mode, steps, d);
                unsigned long long c = 0;
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
                printf("ctas/SM %d mode %d keys/step %d: %7.1f cycles per step (%s)\n", per_sm, mode, ns,
                       double(c) / steps, cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
