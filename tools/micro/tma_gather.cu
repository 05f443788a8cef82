// Throughput of the attention producer's access pattern: per 64-key step, K and V rows of
// 64/BOX randomly chosen column blocks, each a BOX-row x 128-B box of a 4-D (d, n, h, b) tensor
// map over the fused-QKV activation layout (row stride 3*768 elements), into a STAGES-deep ring.
// The consumer releases each stage as soon as it lands, so the number is the producer's ceiling.
//   variants: BOX 16/64, CTAs per SM 1/2, issuing lanes 1/4, ring depth 4/8.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2506_06095_b200/csrc \
//      -o tma_gather tma_gather.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda.h>
#include "tc.cuh"

namespace sf {
sf_status fail(sf_status st, const std::string&) { return st; }
void note_launch(int64_t) {}
}  // namespace sf
using namespace sf;

__device__ __forceinline__ void tma4(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ uint32_t hash(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352d; x ^= x >> 15; x *= 0x846ca68b; x ^= x >> 16;
    return x;
}

template <int BOX, int STAGES, int ISSUERS, int PW = 1>
__global__ void __launch_bounds__(64 + 32 * PW) gather(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                                            int steps, int nblk, int h, int bs) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int G = 64 / BOX;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::fence_barrier_init();
    }
    __syncthreads();
    if (warp < PW) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            const uint32_t ph = ((g / STAGES) & 1) ^ 1;
            if (lane == 0) {
                tc::mbar_wait(&empty[st], ph);
                if (warp == 0) tc::mbar_expect_tx(&full[st], 2 * 64 * 128);
            }
            __syncwarp();
            const uint32_t hs = hash(blockIdx.x * 7919u + g);
            const int slice = hs % (h * bs);
            if (lane < ISSUERS) {
                for (int gg = lane * PW + warp; gg < G; gg += ISSUERS * PW) {
                    const int cb = hash(hs + gg) % nblk;
                    unsigned char* k = base + st * 16384 + gg * BOX * 128;
                    tma4(k, &tk, &full[st], 0, cb * BOX, slice % h, slice / h);
                    tma4(k + 8192, &tv, &full[st], 0, cb * BOX, slice % h, slice / h);
                }
            }
        }
    } else if (warp == PW && lane == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            tc::mbar_wait(&full[st], (g / STAGES) & 1);
            tc::mbar_arrive(&empty[st]);
        }
    }
}

// NB barriers per stage: box gg (K and V) completes on barrier gg % NB, the consumer waits all NB
// (is the per-CTA box rate limited by complete_tx updates to ONE mbarrier?)
template <int BOX, int STAGES, int NB>
__global__ void __launch_bounds__(96) gather_nb(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                                              int steps, int nblk, int h, int bs) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES][NB], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int G = 64 / BOX;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { for (int b = 0; b < NB; ++b) tc::mbar_init(&full[s][b], 1); tc::mbar_init(&empty[s], 1); }
        tc::fence_barrier_init();
    }
    __syncthreads();
    if (warp == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            const uint32_t ph = ((g / STAGES) & 1) ^ 1;
            if (lane == 0) {
                tc::mbar_wait(&empty[st], ph);
                for (int b = 0; b < NB; ++b) tc::mbar_expect_tx(&full[st][b], 2 * 64 * 128 / NB);
            }
            __syncwarp();
            const uint32_t hs = hash(blockIdx.x * 7919u + g);
            const int slice = hs % (h * bs);
            if (lane < G) {
                const int gg = lane;
                const int cb = hash(hs + gg) % nblk;
                unsigned char* k = base + st * 16384 + gg * BOX * 128;
                tma4(k, &tk, &full[st][gg % NB], 0, cb * BOX, slice % h, slice / h);
                tma4(k + 8192, &tv, &full[st][(gg + (NB > G ? G : 0)) % NB], 0, cb * BOX, slice % h, slice / h);
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            for (int b = 0; b < NB; ++b) tc::mbar_wait(&full[st][b], (g / STAGES) & 1);
            tc::mbar_arrive(&empty[st]);
        }
    }
}

template <int BOX, int STAGES, int NB>
void run_nb(const CUtensorMap& tk, const CUtensorMap& tv, int n, int h, int bs, int sms, int cps) {
    auto kern = gather_nb<BOX, STAGES, NB>;
    const int smem = STAGES * 16384 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int steps = 2000, grid = sms * cps;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) kern<<<grid, 96, smem>>>(tk, tv, steps, n / BOX, h, bs);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int it = 0; it < reps; ++it) kern<<<grid, 96, smem>>>(tk, tv, steps, n / BOX, h, bs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(reps) * grid * steps * 16384.0;
    const double s = ms * 1e-3;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("box %2d stages %d barriers/stage %d ctas/SM %d: %7.1f GB/s  %5.1f B/clk/SM  %6.0f clk per 64-key step per CTA\n",
           BOX, STAGES, NB, cps, bytes / s / 1e9, bytes / s / (clk * 1e3) / sms, s * clk * 1e3 / (double(reps) * steps));
    if (cudaGetLastError() != cudaSuccess) { printf("error\n"); exit(1); }
}

// the same 16-row boxes through a 2-D map (rows = b*n, cols = 3H): per-op cost vs dimensionality
template <int BOX, int STAGES, int ISSUERS>
__global__ void __launch_bounds__(96) gather_2d(const __grid_constant__ CUtensorMap t2, int steps, int nblk, int n, int h,
                                              int bs, int H) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int G = 64 / BOX;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::fence_barrier_init();
    }
    __syncthreads();
    if (warp == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            const uint32_t ph = ((g / STAGES) & 1) ^ 1;
            if (lane == 0) {
                tc::mbar_wait(&empty[st], ph);
                tc::mbar_expect_tx(&full[st], 2 * 64 * 128);
            }
            __syncwarp();
            const uint32_t hs = hash(blockIdx.x * 7919u + g);
            const int slice = hs % (h * bs);
            const int hh = slice % h, b = slice / h;
            if (lane < ISSUERS) {
                for (int gg = lane; gg < G; gg += ISSUERS) {
                    const int cb = hash(hs + gg) % nblk;
                    unsigned char* k = base + st * 16384 + gg * BOX * 128;
                    tc::tma_load_2d(k, &t2, &full[st], H + hh * 64, b * n + cb * BOX);
                    tc::tma_load_2d(k + 8192, &t2, &full[st], 2 * H + hh * 64, b * n + cb * BOX);
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            tc::mbar_wait(&full[st], (g / STAGES) & 1);
            tc::mbar_arrive(&empty[st]);
        }
    }
}

// HEADS heads per box ({64, BOX, HEADS, 1}): one TMA instruction fetches the same key block of
// HEADS adjacent heads (items of one row block share the load list across heads); a stage holds
// HEADS x 64 keys of K and of V.
template <int BOX, int STAGES, int ISSUERS, int HEADS>
__global__ void __launch_bounds__(96) gather_heads(const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tv,
                                                   int steps, int nblk, int h, int bs) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int G = 64 / BOX;
    constexpr int kStage = HEADS * 16384;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 1); tc::mbar_init(&empty[s], 1); }
        tc::fence_barrier_init();
    }
    __syncthreads();
    if (warp == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            const uint32_t ph = ((g / STAGES) & 1) ^ 1;
            if (lane == 0) {
                tc::mbar_wait(&empty[st], ph);
                tc::mbar_expect_tx(&full[st], kStage);
            }
            __syncwarp();
            const uint32_t hs = hash(blockIdx.x * 7919u + g);
            const int hp = hs % (h / HEADS), b = (hs / 97) % bs;
            if (lane < ISSUERS) {
                for (int gg = lane; gg < G; gg += ISSUERS) {
                    const int cb = hash(hs + gg) % nblk;
                    unsigned char* k = base + st * kStage + gg * BOX * 128 * HEADS;
                    tma4(k, &tk, &full[st], 0, cb * BOX, hp * HEADS, b);
                    tma4(k + kStage / 2, &tv, &full[st], 0, cb * BOX, hp * HEADS, b);
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            tc::mbar_wait(&full[st], (g / STAGES) & 1);
            tc::mbar_arrive(&empty[st]);
        }
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 encode;
static CUtensorMap map4(const void* base, int n, int h, int bs, long sn, long sh, long sb, int box, int bh = 1);

// The same gather with cp.async (LDGSTS, 16 B per thread) from PW producer warps; each thread
// signals the stage barrier with cp.async.mbarrier.arrive.noinc once its copies land.
// SPLIT: K by TMA (one lane of warp 0), V by LDGSTS (all producer warps).
template <int BOX, int STAGES, int PW, bool SPLIT>
__global__ void __launch_bounds__(32 * PW + 32) gather_lsu(const __grid_constant__ CUtensorMap tk, const __half* kbase,
                                                         const __half* vbase, int steps, int nblk, int h, int bs, int n) {
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(dsm) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t full[STAGES], empty[STAGES];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int G = 64 / BOX;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { tc::mbar_init(&full[s], 32 * PW + (SPLIT ? 1 : 0)); tc::mbar_init(&empty[s], 1); }
        tc::fence_barrier_init();
    }
    __syncthreads();
    const long rs = 3 * 768;  // row stride (elements)
    if (warp < PW) {
        const int t = threadIdx.x;
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            const uint32_t ph = ((g / STAGES) & 1) ^ 1;
            tc::mbar_wait(&empty[st], ph);
            const uint32_t hs = hash(blockIdx.x * 7919u + g);
            const int slice = hs % (h * bs);
            const int hh = slice % h, b = slice / h;
            if (SPLIT && t == 0) {
                tc::mbar_expect_tx(&full[st], 64 * 128);
                for (int gg = 0; gg < G; ++gg) {
                    const int cb = hash(hs + gg) % nblk;
                    tma4(base + st * 16384 + gg * BOX * 128, &tk, &full[st], 0, cb * BOX, hh, b);
                }
            }
            // 16-byte chunks: (SPLIT ? V only : K and V), 64 rows x 8 chunks each
            constexpr int kChunks = (SPLIT ? 1 : 2) * 64 * 8;
#pragma unroll
            for (int c = t; c < kChunks; c += 32 * PW) {
                const int which = SPLIT ? 1 : c / 512;
                const int r = (c / 8) % 64, ch = c % 8;
                const int cb = hash(hs + r / BOX) % nblk;
                const int row = cb * BOX + r % BOX;
                const __half* src = (which ? vbase : kbase) + (long(b) * n + row) * rs + hh * 64 + ch * 8;
                const uint32_t dst = tc::smem_u32(base + st * 16384 + which * 8192 + r * 128 + ((ch ^ (r & 7)) << 4));
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(tc::smem_u32(&full[st])) : "memory");
        }
    } else if (lane == 0) {
        for (int g = 0; g < steps; ++g) {
            const int st = g % STAGES;
            tc::mbar_wait(&full[st], (g / STAGES) & 1);
            tc::mbar_arrive(&empty[st]);
        }
    }
}

template <int BOX, int STAGES, int PW, bool SPLIT>
void run_lsu(const CUtensorMap& tk, const __half* kb, const __half* vb, int n, int h, int bs, int sms, int cps) {
    auto kern = gather_lsu<BOX, STAGES, PW, SPLIT>;
    const int smem = STAGES * 16384 + 1024;
    if (cps * smem > 228 * 1024) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int steps = 2000, grid = sms * cps;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) kern<<<grid, 32 * PW + 32, smem>>>(tk, kb, vb, steps, n / BOX, h, bs, n);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int it = 0; it < reps; ++it) kern<<<grid, 32 * PW + 32, smem>>>(tk, kb, vb, steps, n / BOX, h, bs, n);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(reps) * grid * steps * 16384.0;
    const double s = ms * 1e-3;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("LDGSTS%s box %2d stages %d pwarps %d ctas/SM %d: %7.1f GB/s  %5.1f B/clk/SM  %6.0f clk per 64-key step per CTA\n",
           SPLIT ? "(V; K by TMA)" : "", BOX, STAGES, PW, cps, bytes / s / 1e9, bytes / s / (clk * 1e3) / sms,
           s * clk * 1e3 / (double(reps) * steps));
    if (cudaGetLastError() != cudaSuccess) { printf("error\n"); exit(1); }
}

static CUtensorMap map4(const void* base, int n, int h, int bs, long sn, long sh, long sb, int box, int bh) {
    CUtensorMap m;
    const cuuint64_t dims[4] = {64, (cuuint64_t)n, (cuuint64_t)h, (cuuint64_t)bs};
    const cuuint64_t strides[3] = {(cuuint64_t)sn * 2, (cuuint64_t)sh * 2, (cuuint64_t)sb * 2};
    const cuuint32_t boxd[4] = {64, (cuuint32_t)box, (cuuint32_t)bh, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(base), dims, strides, boxd, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); exit(1); }
    return m;
}

template <int BOX, int STAGES, int ISSUERS, int HEADS>
void run_heads(const CUtensorMap& tk, const CUtensorMap& tv, int n, int h, int bs, int sms, int cps) {
    auto kern = gather_heads<BOX, STAGES, ISSUERS, HEADS>;
    const int smem = STAGES * HEADS * 16384 + 1024;
    if (cps * smem > 228 * 1024) return;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int steps = 2000, grid = sms * cps;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) kern<<<grid, 96, smem>>>(tk, tv, steps, n / BOX, h, bs);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int it = 0; it < reps; ++it) kern<<<grid, 96, smem>>>(tk, tv, steps, n / BOX, h, bs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(reps) * grid * steps * 16384.0 * HEADS;
    const double s = ms * 1e-3;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("box %2dx%d heads stages %d issuers %d ctas/SM %d: %7.1f GB/s  %5.1f B/clk/SM  %6.0f clk per 64-key step (all heads) per CTA\n",
           BOX, HEADS, STAGES, ISSUERS, cps, bytes / s / 1e9, bytes / s / (clk * 1e3) / sms,
           s * clk * 1e3 / (double(reps) * steps));
    if (cudaGetLastError() != cudaSuccess) { printf("error\n"); exit(1); }
}

template <int BOX, int STAGES, int ISSUERS, int PW = 1>
void run(const CUtensorMap& tk, const CUtensorMap& tv, int n, int h, int bs, int sms, int cps) {
    if (cps == 2 && STAGES == 8) return;
    auto kern = gather<BOX, STAGES, ISSUERS, PW>;
    const int smem = STAGES * 16384 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int steps = 2000, grid = sms * cps;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int it = 0; it < 2; ++it) kern<<<grid, 64 + 32 * PW, smem>>>(tk, tv, steps, n / BOX, h, bs);
    cudaEventRecord(e0);
    const int reps = 5;
    for (int it = 0; it < reps; ++it) kern<<<grid, 64 + 32 * PW, smem>>>(tk, tv, steps, n / BOX, h, bs);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = double(reps) * grid * steps * 16384.0;
    const double s = ms * 1e-3;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("box %2d stages %d issuers %d pwarps %d ctas/SM %d: %7.1f GB/s  %5.1f B/clk/SM  %6.0f clk per 64-key step per CTA\n",
           BOX, STAGES, ISSUERS, PW, cps, bytes / s / 1e9, bytes / s / (clk * 1e3) / sms,
           s * clk * 1e3 / (double(reps) * steps));
    if (cudaGetLastError() != cudaSuccess) { printf("error\n"); exit(1); }
}

int main() {
    cudaDriverEntryPointQueryResult q;
    void* fn;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int bs = 16, n = 1024, h = 12, H = 768;
    __half* qkv;
    cudaMalloc(&qkv, size_t(bs) * n * 3 * H * 2);
    cudaMemset(qkv, 0x3c, size_t(bs) * n * 3 * H * 2);
    // (d, n, h, b) strides in elements: row 3H, head 64, batch n*3H
    if (getenv("NB_ONLY")) {
        CUtensorMap tk = map4(qkv + H, n, h, bs, 3 * H, 64, long(n) * 3 * H, 16);
        CUtensorMap tv = map4(qkv + 2 * H, n, h, bs, 3 * H, 64, long(n) * 3 * H, 16);
        for (int cps : {1, 2}) {
            run_nb<16, 4, 1>(tk, tv, n, h, bs, sms, cps);
            run_nb<16, 4, 2>(tk, tv, n, h, bs, sms, cps);
            run_nb<16, 4, 4>(tk, tv, n, h, bs, sms, cps);
            run_nb<16, 4, 8>(tk, tv, n, h, bs, sms, cps);
        }
        CUtensorMap t2;
        {
            const cuuint64_t dims[2] = {(cuuint64_t)3 * H, (cuuint64_t)bs * n};
            const cuuint64_t strides[1] = {(cuuint64_t)3 * H * 2};
            const cuuint32_t boxd[2] = {64, 16};
            const cuuint32_t estr[2] = {1, 1};
            encode(&t2, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, qkv, dims, strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        }
        for (int cps : {1, 2}) {
            auto kern = gather_2d<16, 4, 4>;
            const int smem = 4 * 16384 + 1024;
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const int steps = 2000, grid = sms * cps;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            for (int it = 0; it < 2; ++it) kern<<<grid, 96, smem>>>(t2, steps, n / 16, n, h, bs, H);
            cudaEventRecord(e0);
            for (int it = 0; it < 5; ++it) kern<<<grid, 96, smem>>>(t2, steps, n / 16, n, h, bs, H);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
            printf("2-D map box 16 stages 4 issuers 4 ctas/SM %d: %6.0f clk per 64-key step per CTA (%s)\n", cps,
                   ms * 1e-3 * clk * 1e3 / (5.0 * steps), cudaGetErrorString(cudaGetLastError()));
        }
        return 0;
    }
    for (int box : {16, 64}) {
        CUtensorMap tk = map4(qkv + H, n, h, bs, 3 * H, 64, long(n) * 3 * H, box);
        CUtensorMap tv = map4(qkv + 2 * H, n, h, bs, 3 * H, 64, long(n) * 3 * H, box);
        for (int cps : {1, 2}) {
            if (box == 16) {
                run<16, 4, 1>(tk, tv, n, h, bs, sms, cps);
                run<16, 8, 1>(tk, tv, n, h, bs, sms, cps);
                run<16, 4, 4>(tk, tv, n, h, bs, sms, cps);
                run<16, 8, 4>(tk, tv, n, h, bs, sms, cps);
                run<16, 4, 1, 2>(tk, tv, n, h, bs, sms, cps);
                run<16, 4, 1, 4>(tk, tv, n, h, bs, sms, cps);
                run<16, 4, 2, 4>(tk, tv, n, h, bs, sms, cps);
            } else {
                run<64, 4, 1>(tk, tv, n, h, bs, sms, cps);
                run<64, 8, 1>(tk, tv, n, h, bs, sms, cps);
            }
        }
    }
    for (int hb : {2, 4}) {
        CUtensorMap tk = map4(qkv + H, n, h, bs, 3 * H, 64, long(n) * 3 * H, 16, hb);
        CUtensorMap tv = map4(qkv + 2 * H, n, h, bs, 3 * H, 64, long(n) * 3 * H, 16, hb);
        for (int cps : {1, 2}) {
            if (hb == 2) {
                run_heads<16, 2, 4, 2>(tk, tv, n, h, bs, sms, cps);
                run_heads<16, 3, 4, 2>(tk, tv, n, h, bs, sms, cps);
                run_heads<16, 2, 1, 2>(tk, tv, n, h, bs, sms, cps);
            } else {
                run_heads<16, 2, 4, 4>(tk, tv, n, h, bs, sms, cps);
            }
        }
    }
    {
        CUtensorMap tk = map4(qkv + H, n, h, bs, 3 * H, 64, long(n) * 3 * H, 16);
        for (int cps : {1, 2}) {
            run_lsu<16, 4, 1, false>(tk, qkv + H, qkv + 2 * H, n, h, bs, sms, cps);
            run_lsu<16, 4, 2, false>(tk, qkv + H, qkv + 2 * H, n, h, bs, sms, cps);
            run_lsu<16, 4, 4, false>(tk, qkv + H, qkv + 2 * H, n, h, bs, sms, cps);
            run_lsu<16, 4, 1, true>(tk, qkv + H, qkv + 2 * H, n, h, bs, sms, cps);
            run_lsu<16, 4, 2, true>(tk, qkv + H, qkv + 2 * H, n, h, bs, sms, cps);
            run_lsu<16, 4, 4, true>(tk, qkv + H, qkv + 2 * H, n, h, bs, sms, cps);
        }
    }
    return 0;
}
