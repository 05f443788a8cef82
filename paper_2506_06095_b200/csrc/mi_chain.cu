// mi_chain.cu — the MiChain template (backend.hpp:228-235): a run of memory-intensive ops
// (Bias, GELU/ReLU, Add, LayerNorm) applied to each row in ONE pass over HBM. One 256-thread CTA
// per row; each thread keeps up to 16 values of the row in registers, so the row is read once
// and written once regardless of how many ops are fused (HBM-bound: 2*N*2 bytes per row + aux).
#include "common.cuh"

namespace sf {
namespace {

constexpr int kT = 256, kPer = 16;

__device__ __forceinline__ float block_sum(float v, float* sh) {
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) t += sh[w];
    __syncthreads();
    return t;
}

template <typename T>
__global__ void __launch_bounds__(kT) mi_chain_kernel(int32_t M, int32_t N, const T* __restrict__ x, int64_t ldx,
                                                      sf_gemm_epilogue e, T* __restrict__ out, int64_t ldout) {
    __shared__ float sh[kT / 32];
    const int64_t row = blockIdx.x;
    float v[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int c = threadIdx.x + i * kT;
        float a = 0.f;
        if (c < N) {
            a = DT<T>::to_f(x[row * ldx + c]);
            if (e.bias) a += static_cast<const float*>(e.bias)[c];
            if (e.act == SF_ACT_GELU) a = 0.5f * a * (1.0f + erff(a * 0.7071067811865475f));
            else if (e.act == SF_ACT_RELU) a = a > 0.f ? a : 0.f;
            if (e.aux) a += DT<T>::to_f(static_cast<const T*>(e.aux)[row * e.ldaux + c]);
        }
        v[i] = a;
    }
    if (e.ln_gamma) {
        float s = 0.f;
#pragma unroll
        for (int i = 0; i < kPer; ++i) s += v[i];
        const float mean = block_sum(s, sh) / static_cast<float>(N);
        float q = 0.f;
#pragma unroll
        for (int i = 0; i < kPer; ++i)
            if (threadIdx.x + i * kT < N) q += (v[i] - mean) * (v[i] - mean);
        const float inv = 1.0f / sqrtf(block_sum(q, sh) / static_cast<float>(N) + 1e-5f);
        const float* g = static_cast<const float*>(e.ln_gamma);
        const float* b = static_cast<const float*>(e.ln_beta);
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int c = threadIdx.x + i * kT;
            if (c < N) {
                if (e.out_pre_ln) static_cast<T*>(e.out_pre_ln)[row * ldout + c] = DT<T>::from_f(v[i]);
                out[row * ldout + c] = DT<T>::from_f((v[i] - mean) * inv * g[c] + b[c]);
            }
        }
    } else {
#pragma unroll
        for (int i = 0; i < kPer; ++i) {
            const int c = threadIdx.x + i * kT;
            if (c < N) out[row * ldout + c] = DT<T>::from_f(v[i]);
        }
    }
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" sf_status sf_mi_chain(int32_t M, int32_t N, int32_t dtype, const void* x, int64_t ldx,
                                 const sf_gemm_epilogue* epi, void* out, int64_t ldout, void* stream) {
    if (M < 1 || N < 1) return fail(SF_SHAPE_ERROR, "empty matrix");
    if (N > kT * kPer) return fail(SF_SHAPE_ERROR, "mi_chain supports N <= 4096");
    sf_gemm_epilogue e = epi ? *epi : sf_gemm_epilogue{};
    if (e.ln_gamma && !e.ln_beta) return fail(SF_INVALID_PARAMETER, "LayerNorm needs gamma and beta");
    cudaStream_t st = as_stream(stream);
    if (dtype == SF_F16)
        mi_chain_kernel<__half><<<M, kT, 0, st>>>(M, N, static_cast<const __half*>(x), ldx, e,
                                                  static_cast<__half*>(out), ldout);
    else if (dtype == SF_BF16)
        mi_chain_kernel<__nv_bfloat16><<<M, kT, 0, st>>>(M, N, static_cast<const __nv_bfloat16*>(x), ldx, e,
                                                         static_cast<__nv_bfloat16*>(out), ldout);
    else
        return fail(SF_INVALID_PARAMETER, "dtype must be f16/bf16");
    SF_LAUNCH_CHECK();
    return SF_OK;
}
