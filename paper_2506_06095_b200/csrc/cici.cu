// cici.cu — the CiCi template (backend.hpp:270-306) chained ON CHIP for short activations:
//   out = post( mid( X . W1^T ) . W2^T )      mid = +b1 -> GELU/ReLU, post = +b2 -> +aux -> [LN]
// The reference's search forms CiCi segments only for bs * seq <= 4096 (search.hpp:228), where the
// two CiMi launches are latency-bound (cfg1, 512 rows: FFN1 14 us + FFN2 25 us for 2 x 2.4 GFLOP).
// Here the intermediate never leaves the SM:
//   CTA (chunk c, row block r), one per 128 columns of the intermediate and 128 rows:
//     H   = X[r] . W1[c]^T        tcgen05 (M 128, N 128), TMEM [0, 128), K streamed by TMA
//     Hs  = mid(H) in fp16        written by the epilogue warps straight into shared memory in the
//                                 128-byte-swizzled K-major layout the next MMA reads as operand A
//     Y_p = Hs . W2[:, c]^T       tcgen05 (M 128, N 192 / 128 / 64) per pass of the output,
//                                 double-buffered in TMEM from column 128, so pass p+1's
//                                 MMAs run under pass p's drain
//     Yacc[r, p] += Y_p           fp32 vector reductions (red.global.add.v4.f32) into an L2-resident
//                                 accumulator: the split over intermediate chunks is a split-K of
//                                 the second GEMM
//   then one warp-per-row pass applies post (+b2, +aux, LayerNorm) to Yacc and writes the output.
// Warps: 0 TMA producer (X / W1 k-blocks, then W2 k-blocks, one 32 KB ring), 1 TMEM allocator +
// MMA issuer, 2-5 epilogue (TMEM lane quarter = warp % 4, one thread per row).
#include <algorithm>
#include <cstring>

#include "epilogue.cuh"

namespace sf {
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t st);
namespace {

#ifndef SF_CICI_C1
#define SF_CICI_C1 128
#endif
constexpr int kC1 = SF_CICI_C1;   // intermediate columns per CTA (128 or 256)
constexpr int kNPMax = kC1 == 128 ? 192 : 128;  // output columns per pass (N of the second MMA), max
constexpr int kStagesC = kC1 == 128 ? 4 : 3;
constexpr int kStageBytes = BM * BK * 2 + kC1 * BK * 2;  // X + W1 k-block (W2 k-blocks fit too)
constexpr int kHBytes = BM * kC1 * 2;  // 32 / 64 KB
constexpr int kThreadsC = 192;
constexpr int kSmemC = 1024 + kStagesC * kStageBytes + kHBytes + 256;
constexpr uint32_t kColY = kC1;

struct CiciParams {
    CUtensorMap tx, tw1, tw2;  // X (M x K1), W1 (N1 x K1), W2 (N2 x N1); 64-col boxes, SW128
    int32_t M, K1, N1, N2;
    int32_t np;                // output columns per pass: 192, 128 or 64, dividing N2
    const float* b1;
    int32_t act;
    float* yacc;               // M x N2 fp32, zeroed before the launch
};

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kThreadsC, 1) cici_kernel(const __grid_constant__ CiciParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sRing = smem;
    unsigned char* sH = smem + kStagesC * kStageBytes;  // [kC1 / 64 k-blocks][128 rows][128 B], SW128
    uint64_t* full = reinterpret_cast<uint64_t*>(sH + kHBytes);
    uint64_t* empty = full + kStagesC;
    uint64_t* h_full = empty + kStagesC;   // H accumulated
    uint64_t* h_ready = h_full + 1;        // mid(H) in shared memory (128 epilogue arrivals)
    uint64_t* y_full = h_ready + 1;        // [2]
    uint64_t* y_empty = y_full + 2;        // [2] (128 epilogue arrivals)
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(y_empty + 2);

    pdl_enter();
    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const int c = static_cast<int>(blockIdx.x);   // intermediate chunk
    const int rb = static_cast<int>(blockIdx.y);  // row block
    const int nk1 = p.K1 / BK;
    const int np = p.np;
    const int npass = p.N2 / np;
    constexpr int nk2 = kC1 / BK;                  // 2

    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&p.tx);
        tc::prefetch_tmap(&p.tw1);
        tc::prefetch_tmap(&p.tw2);
        for (int s = 0; s < kStagesC; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(h_full, 1);
        tc::mbar_init(h_ready, 128);
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&y_full[b], 1);
            tc::mbar_init(&y_empty[b], 128);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<512>(tmem_ptr);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (lane == 0) {
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nk1; ++kb) {
                tc::mbar_wait(&empty[s], ph ^ 1);
                tc::mbar_expect_tx(&full[s], kStageBytes);
                tc::tma_load_2d(sRing + s * kStageBytes, &p.tx, &full[s], kb * BK, rb * BM);
                tc::tma_load_2d(sRing + s * kStageBytes + BM * BK * 2, &p.tw1, &full[s], kb * BK, c * kC1);
                if (++s == kStagesC) { s = 0; ph ^= 1; }
            }
            for (int pp = 0; pp < npass; ++pp)
                for (int kb = 0; kb < nk2; ++kb) {
                    tc::mbar_wait(&empty[s], ph ^ 1);
                    tc::mbar_expect_tx(&full[s], np * BK * 2);
                    tc::tma_load_2d(sRing + s * kStageBytes, &p.tw2, &full[s], c * kC1 + kb * BK, pp * np);
                    if (++s == kStagesC) { s = 0; ph ^= 1; }
                }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        constexpr bool bf = std::is_same<T, __nv_bfloat16>::value;
        constexpr uint32_t idesc1 = tc::idesc_f16(BM, kC1, bf, 0, 0);
        const uint32_t idesc2 = tc::idesc_f16(BM, static_cast<uint32_t>(np), bf, 0, 0);
        if (tc::elect_one()) {
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nk1; ++kb) {
                tc::mbar_wait(&full[s], ph);
                tc::fence_after_sync();
                const uint32_t a0 = tc::smem_u32(sRing + s * kStageBytes);
                const uint32_t b0 = a0 + BM * BK * 2;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    tc::mma_f16_ss(tmem, tc::sdesc_sw128(a0 + 32 * k), tc::sdesc_sw128(b0 + 32 * k), idesc1, (kb | k) != 0);
                tc::mma_commit(&empty[s]);
                if (++s == kStagesC) { s = 0; ph ^= 1; }
            }
            tc::mma_commit(h_full);
            tc::mbar_wait(h_ready, 0);  // mid(H) is in shared memory (async-proxy visible)
            tc::fence_after_sync();
            const uint32_t h0 = tc::smem_u32(sH);
            for (int pp = 0; pp < npass; ++pp) {
                const int yb = pp & 1;
                if (pp >= 2) {
                    tc::mbar_wait(&y_empty[yb], ((pp >> 1) - 1) & 1);
                    tc::fence_after_sync();
                }
                const uint32_t d = tmem + kColY + static_cast<uint32_t>(np * yb);
                for (int kb = 0; kb < nk2; ++kb) {
                    tc::mbar_wait(&full[s], ph);
                    tc::fence_after_sync();
                    const uint32_t b0 = tc::smem_u32(sRing + s * kStageBytes);
                    const uint32_t a0 = h0 + kb * (BM * BK * 2);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc::mma_f16_ss(d, tc::sdesc_sw128(a0 + 32 * k), tc::sdesc_sw128(b0 + 32 * k), idesc2, (kb | k) != 0);
                    tc::mma_commit(&empty[s]);
                    if (++s == kStagesC) { s = 0; ph ^= 1; }
                }
                tc::mma_commit(&y_full[yb]);
            }
        }
    } else {
        // ------------------------------------------------------------------ epilogue (warps 2-5)
        const uint32_t q = warp & 3;
        const int r = static_cast<int>(q * 32 + lane);  // row within the block = TMEM lane
        const uint32_t tl = tmem + ((q * 32) << 16);
        // mid(H) -> fp16 -> shared memory, 128-byte swizzle: 16-byte chunk j of row r in k-block
        // kb at kb * 16 KB + (r / 8) * 1 KB + (r % 8) * 128 + (j ^ (r % 8)) * 16
        tc::mbar_wait(h_full, 0);
        tc::fence_after_sync();
        const uint32_t hrow = tc::smem_u32(sH) + static_cast<uint32_t>((r >> 3) * 1024 + (r & 7) * 128);
#pragma unroll 1
        for (int h4 = 0; h4 < kC1 / 32; ++h4) {
            uint32_t v[32];
            tc::tmem_ld32(tl + 32 * h4, v);
            tc::tmem_ld_wait();
            float x[32];
            const float* b1 = p.b1 ? p.b1 + c * kC1 + 32 * h4 : nullptr;
#pragma unroll
            for (int j = 0; j < 32; ++j) {
                float t = __uint_as_float(v[j]) + (b1 ? __ldg(b1 + j) : 0.f);
                x[j] = act_fn(t, p.act);
            }
#pragma unroll
            for (int j8 = 0; j8 < 4; ++j8) {
                const int col = 32 * h4 + 8 * j8;  // first of the 8 values
                const uint32_t kb = static_cast<uint32_t>(col >> 6), j = static_cast<uint32_t>((col & 63) >> 3);
                const uint32_t a = hrow + kb * (BM * BK * 2) + ((j ^ static_cast<uint32_t>(r & 7)) << 4);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pack2<T>(x[8 * j8], x[8 * j8 + 1])),
                             "r"(pack2<T>(x[8 * j8 + 2], x[8 * j8 + 3])), "r"(pack2<T>(x[8 * j8 + 4], x[8 * j8 + 5])),
                             "r"(pack2<T>(x[8 * j8 + 6], x[8 * j8 + 7]))
                             : "memory");
            }
        }
        tc::fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
        tc::fence_before_sync();
        tc::mbar_arrive(h_ready);
        // drain each output pass into the fp32 accumulator
        const int64_t row = static_cast<int64_t>(rb) * BM + r;
        const bool row_ok = row < p.M;
        for (int pp = 0; pp < npass; ++pp) {
            const int yb = pp & 1;
            tc::mbar_wait(&y_full[yb], (pp >> 1) & 1);
            tc::fence_after_sync();
            float* dst = p.yacc + row * p.N2 + pp * np;
#pragma unroll 1
            for (int h4 = 0; h4 < np / 32; ++h4) {
                uint32_t v[32];
                tc::tmem_ld32(tl + kColY + static_cast<uint32_t>(np * yb + 32 * h4), v);
                tc::tmem_ld_wait();
                if (row_ok) {
#pragma unroll
                    for (int j = 0; j < 32; j += 4)
                        red_add_v4(dst + 32 * h4 + j, __uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                   __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
                }
            }
            tc::fence_before_sync();
            tc::mbar_arrive(&y_empty[yb]);
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

__device__ __forceinline__ float wsum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// post ops on the fp32 accumulator: + b2 -> + aux -> [LayerNorm] (backend.hpp:111-153), one warp
// per row; lane l holds columns 4 (l + 32 i) .. +3
template <typename T, int V>
__global__ void __launch_bounds__(256) cici_post_kernel(int32_t M, int32_t N, const float* __restrict__ yacc,
                                                       sf_gemm_epilogue e, T* __restrict__ out, int64_t ldout) {
    pdl_enter();
    const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
    if (row >= M) return;
    const int lane = threadIdx.x & 31;
    const float* b2 = static_cast<const float*>(e.bias);
    const T* aux = static_cast<const T*>(e.aux);
    float v[V][4];
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int col = 4 * (lane + 32 * i);
        if (col < N) {
            const float4 a = *reinterpret_cast<const float4*>(yacc + row * N + col);
            v[i][0] = a.x; v[i][1] = a.y; v[i][2] = a.z; v[i][3] = a.w;
            if (b2) {
                const float4 b = *reinterpret_cast<const float4*>(b2 + col);
                v[i][0] += b.x; v[i][1] += b.y; v[i][2] += b.z; v[i][3] += b.w;
            }
            if (aux) {
                const T* ap = aux + row * e.ldaux + col;
#pragma unroll
                for (int j = 0; j < 4; ++j) v[i][j] += DT<T>::to_f(ap[j]);
            }
        } else {
#pragma unroll
            for (int j = 0; j < 4; ++j) v[i][j] = 0.f;
        }
    }
    float mean = 0.f, inv = 1.f;
    if (e.ln_gamma) {  // two-pass mean / biased variance, eps 1e-5 (backend.hpp:141-154)
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) s += v[i][j];
        mean = wsum(s) / static_cast<float>(N);
        float qq = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i)
            if (4 * (lane + 32 * i) < N)
#pragma unroll
                for (int j = 0; j < 4; ++j) qq += (v[i][j] - mean) * (v[i][j] - mean);
        inv = 1.0f / sqrtf(wsum(qq) / static_cast<float>(N) + kLnEps);
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
        const int col = 4 * (lane + 32 * i);
        if (col >= N) continue;
        T* op = out + row * ldout + col;
        T* pp = e.out_pre_ln ? static_cast<T*>(e.out_pre_ln) + row * ldout + col : nullptr;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            float y = v[i][j];
            if (pp) pp[j] = DT<T>::from_f(y);
            if (e.ln_gamma)
                y = (y - mean) * inv * static_cast<const float*>(e.ln_gamma)[col + j] +
                    static_cast<const float*>(e.ln_beta)[col + j];
            op[j] = DT<T>::from_f(y);
        }
    }
}

template <typename T>
sf_status launch_cici(const sf_gemm_chain_args& a, cudaStream_t st) {
    const bool bf = std::is_same<T, __nv_bfloat16>::value;
    CiciParams p{};
    SF_TRY(make_tmap_2d(&p.tx, a.x, a.M, a.K1, a.ldx, BK, BM, bf));
    SF_TRY(make_tmap_2d(&p.tw1, a.w1, a.N1, a.K1, a.ldw1, BK, kC1, bf));
    p.np = a.N2 % 192 == 0 && kNPMax >= 192 ? 192 : (a.N2 % 128 == 0 ? 128 : 64);
    SF_TRY(make_tmap_2d(&p.tw2, a.w2, a.N2, a.N1, a.ldw2, BK, static_cast<uint32_t>(p.np), bf));
    p.M = a.M; p.K1 = a.K1; p.N1 = a.N1; p.N2 = a.N2;
    p.b1 = static_cast<const float*>(a.mid.bias);
    p.act = a.mid.act;
    void* acc = nullptr;
    const size_t acc_bytes = static_cast<size_t>(a.M) * a.N2 * sizeof(float);
    SF_CUDA_TRY(pool_malloc(&acc, acc_bytes, st));
    p.yacc = static_cast<float*>(acc);
    sf_status status = SF_OK;
    if (cudaMemsetAsync(acc, 0, acc_bytes, st) != cudaSuccess) status = fail(SF_CUDA_ERROR, "cici: memset");
    if (status == SF_OK) {
        auto kern = cici_kernel<T>;
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemC) != cudaSuccess ||
            launch_pdl(kern, dim3(a.N1 / kC1, static_cast<unsigned>(ceil_div(a.M, BM))), dim3(kThreadsC), kSmemC, st,
                       nullptr, p) != cudaSuccess)
            status = fail(SF_CUDA_ERROR, std::string("cici kernel: ") + cudaGetErrorString(cudaGetLastError()));
    }
    if (status == SF_OK) {
        const unsigned grid = static_cast<unsigned>(ceil_div(a.M, 8));
        const float* acc_f = static_cast<const float*>(acc);
        T* out = static_cast<T*>(a.out);
        cudaError_t e = cudaSuccess;
        if (a.N2 <= 128 * 4) e = launch_pdl(cici_post_kernel<T, 4>, dim3(grid), dim3(256), 0, st, nullptr, a.M, a.N2, acc_f, a.post, out, a.ldout);
        else if (a.N2 <= 128 * 8) e = launch_pdl(cici_post_kernel<T, 8>, dim3(grid), dim3(256), 0, st, nullptr, a.M, a.N2, acc_f, a.post, out, a.ldout);
        else e = launch_pdl(cici_post_kernel<T, 16>, dim3(grid), dim3(256), 0, st, nullptr, a.M, a.N2, acc_f, a.post, out, a.ldout);
        if (e != cudaSuccess) status = fail(SF_CUDA_ERROR, std::string("cici post: ") + cudaGetErrorString(e));
    }
    cudaFreeAsync(acc, st);  // stream-ordered: after the post kernel has read it
    if (status == SF_OK) SF_LAUNCH_CHECK();
    return status;
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" sf_status sf_gemm_chain(const sf_gemm_chain_args* a, void* stream) {
    if (!a) return fail(SF_INVALID_PARAMETER, "null argument");
    if (!a->x || !a->w1 || !a->w2 || !a->out) return fail(SF_INVALID_PARAMETER, "null tensor pointer");
    if (a->M < 1 || a->K1 < 1 || a->N1 < 1 || a->N2 < 1) return fail(SF_SHAPE_ERROR, "empty gemm chain");
    if (a->dtype != SF_F16 && a->dtype != SF_BF16) return fail(SF_INVALID_PARAMETER, "dtype must be f16/bf16");
    if (a->mid.aux || a->mid.ln_gamma || a->mid.softmax || a->mid.out_pre_ln)
        return fail(SF_BACKEND_ERROR, "gemm chain: mid ops are bias and activation");
    if (a->post.softmax) return fail(SF_BACKEND_ERROR, "gemm chain: post Softmax is not fused");
    if (a->K1 % BK || a->N1 % kC1 || a->N2 % 64 || a->N2 > 2048 || (a->post.ln_gamma && !a->post.ln_beta))
        return fail(SF_BACKEND_ERROR, "gemm chain: needs K1 % 64 == 0, N1 % " + std::to_string(kC1) +
                                          " == 0, N2 % 64 == 0, N2 <= 2048");
    if ((a->ldx | a->ldw1 | a->ldw2 | a->ldout) % 8)
        return fail(SF_INVALID_PARAMETER, "gemm chain: row strides must be multiples of 8 elements");
    cudaStream_t st = as_stream(stream);
    return a->dtype == SF_BF16 ? launch_cici<__nv_bfloat16>(*a, st) : launch_cici<__half>(*a, st);
}
