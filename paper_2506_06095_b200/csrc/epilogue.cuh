// epilogue.cuh — pieces shared by the CiMi GEMM kernels (gemm_tc.cu: one CTA per tile,
// gemm2_tc.cu: CTA pairs): kernel parameters and the register-level MI epilogue
// (bias -> GELU/ReLU -> +aux, backend.hpp:111-167).
#pragma once

#include "tc.cuh"

namespace sf {

constexpr int BM = 128, BK = 64;
constexpr float kLnEps = 1e-5f;  // backend.hpp:111
constexpr int kMaxCluster = 8;

struct GemmParams {
    CUtensorMap ta;  // X: rows M, cols K
    CUtensorMap tb;  // W: rows N, cols K
    CUtensorMap tc;    // out: rows M, cols N; 32 x 32 boxes, 64-byte swizzle (TMA-store epilogue)
    CUtensorMap taux;  // residual (aux), same boxes (TMA-load epilogue)
    CUtensorMap tpre;  // out_pre_ln, same boxes
    int32_t M, N, K;
    void* out;
    int64_t ldout;
    const float* bias;
    int32_t act;
    const void* aux;
    int64_t ldaux;
    const float* gamma;
    const float* beta;
    void* out_pre_ln;
    int32_t mc;   // single-CTA non-LN: CTAs per cluster along M sharing (multicasting) the weight tile
    int32_t nct;  // pair kernel, LN: n-tiles per row (cluster = 2 x nct CTAs)
    unsigned long long* trace;  // optional clock64 timeline of pair 0 (built with -DSF_GEMM_TRACE)
};

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// GELU(x) = 0.5 x (1 + erf(x / sqrt 2)) (backend.hpp:128-131, exact-erf semantics) evaluated as
// 0.5 x (1 + tanh(u)) with u(x) an odd polynomial least-squares fitted to atanh(erf(x / sqrt 2))
// (x clamped to +-8, where tanh has saturated): |formula - exact GELU| <= 2.8e-5 over all x.
// One MUFU op (tanh.approx.f32, relative error ~2^-11, below the fp16 output rounding) and 7
// FMA-pipe ops, against rcp + ex2 + ~15 ops for the Abramowitz-Stegun erf this replaced — the
// GELU epilogue was the bottleneck of the FFN1 GEMM.
__device__ __forceinline__ float tanh_approx(float u) {
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
    return t;
}
// (clamping x^2 at 64 keeps u monotone beyond |x| = 8, where tanh(u) is already +-1)
__device__ __forceinline__ float gelu_fast(float x) {
    const float x2 = fminf(x * x, 64.0f);
    const float u = x * fmaf(x2, fmaf(x2, -3.53932780e-4f, 3.70247480e-2f), 7.97482758e-1f);
    return x * fmaf(0.5f, tanh_approx(u), 0.5f);
}
// the same on a packed pair (FMUL2 / FFMA2: half the FMA-pipe instructions)
__device__ __forceinline__ float2 gelu_fast2(float2 x) {
    float2 x2 = tc::fmul2(x, x);
    x2.x = fminf(x2.x, 64.0f);
    x2.y = fminf(x2.y, 64.0f);
    float2 pl = tc::ffma2(x2, make_float2(-3.53932780e-4f, -3.53932780e-4f), make_float2(3.70247480e-2f, 3.70247480e-2f));
    pl = tc::ffma2(x2, pl, make_float2(7.97482758e-1f, 7.97482758e-1f));
    const float2 u = tc::fmul2(x, pl);
    const float2 h = tc::ffma2(make_float2(0.5f, 0.5f), make_float2(tanh_approx(u.x), tanh_approx(u.y)), make_float2(0.5f, 0.5f));
    return tc::fmul2(x, h);
}

__device__ __forceinline__ float act_fn(float x, int act) {
    if (act == SF_ACT_GELU) return gelu_fast(x);  // backend.hpp:128-131
    if (act == SF_ACT_RELU) return x > 0.f ? x : 0.f;                                    // backend.hpp:132-134
    return x;
}

// residual values of row `row`, columns [col, col+32) (issued one chunk ahead of their use)
template <typename T>
__device__ __forceinline__ void load_aux(const GemmParams& p, bool ok, int64_t row, int64_t col, uint4 (&a)[4]) {
    if (!p.aux || !ok) return;
    const uint4* a4 = reinterpret_cast<const uint4*>(static_cast<const T*>(p.aux) + row * p.ldaux + col);
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = __ldg(a4 + j);
}

// 32 consecutive values: bias -> act -> + prefetched residual.
template <typename T>
__device__ __forceinline__ void epi_chunk_pre(const GemmParams& p, const uint32_t (&r)[32], int64_t col,
                                              const uint4 (&aux)[4], float (&x)[32]) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(r[j]);
    if (p.bias) {
        const float4* b4 = reinterpret_cast<const float4*>(p.bias + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 b = __ldg(b4 + j);
            x[4 * j] += b.x; x[4 * j + 1] += b.y; x[4 * j + 2] += b.z; x[4 * j + 3] += b.w;
        }
    }
    if (p.act) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = act_fn(x[j], p.act);
    }
    if (p.aux) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const T* h = reinterpret_cast<const T*>(&aux[j]);
#pragma unroll
            for (int e = 0; e < 8; ++e) x[8 * j + e] += DT<T>::to_f(h[e]);
        }
    }
}

// 32 consecutive values of row `row`, columns [col, col+32): bias -> act -> +aux.
template <typename T>
__device__ __forceinline__ void epi_chunk(const GemmParams& p, const uint32_t (&r)[32], int64_t row, int64_t col,
                                          float (&x)[32], bool with_aux = true) {
#pragma unroll
    for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(r[j]);
    if (p.bias) {
        const float4* b4 = reinterpret_cast<const float4*>(p.bias + col);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const float4 b = __ldg(b4 + j);
            const float2 lo = tc::fadd2(make_float2(x[4 * j], x[4 * j + 1]), make_float2(b.x, b.y));
            const float2 hi = tc::fadd2(make_float2(x[4 * j + 2], x[4 * j + 3]), make_float2(b.z, b.w));
            x[4 * j] = lo.x; x[4 * j + 1] = lo.y; x[4 * j + 2] = hi.x; x[4 * j + 3] = hi.y;
        }
    }
    if (p.act == SF_ACT_GELU) {
#pragma unroll
        for (int j = 0; j < 32; j += 2) {
            const float2 g = gelu_fast2(make_float2(x[j], x[j + 1]));
            x[j] = g.x; x[j + 1] = g.y;
        }
    } else if (p.act == SF_ACT_RELU) {
#pragma unroll
        for (int j = 0; j < 32; ++j) x[j] = x[j] > 0.f ? x[j] : 0.f;
    }
    if (p.aux && with_aux) {
        const uint4* a4 = reinterpret_cast<const uint4*>(static_cast<const T*>(p.aux) + row * p.ldaux + col);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint4 u = __ldg(a4 + j);
            const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
            for (int e = 0; e < 8; ++e) x[8 * j + e] += DT<T>::to_f(h[e]);
        }
    }
}

// 32 consecutive values of row r (0..31) into a warp's 32 x 32 staging box in the SWIZZLE_64B
// layout TMA expects: 16-byte chunk j of row r at r*64 + ((j ^ ((r >> 1) & 3)) * 16). A warp's
// 8-lane phases then hit 8 distinct 16-byte bank groups (conflict-free).
template <typename T>
__device__ __forceinline__ void stage_chunk(uint32_t sbase, int r, const float (&x)[32]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t a = sbase + static_cast<uint32_t>(r) * 64u + ((static_cast<uint32_t>(j) ^ ((r >> 1) & 3)) << 4);
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pack2<T>(x[8 * j], x[8 * j + 1])),
                     "r"(pack2<T>(x[8 * j + 2], x[8 * j + 3])), "r"(pack2<T>(x[8 * j + 4], x[8 * j + 5])),
                     "r"(pack2<T>(x[8 * j + 6], x[8 * j + 7]))
                     : "memory");
    }
}

template <typename T>
__device__ __forceinline__ void store_chunk(void* base, int64_t ld, int64_t row, int64_t col, const float (&x)[32]) {
    uint4* o = reinterpret_cast<uint4*>(static_cast<T*>(base) + row * ld + col);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint4 u;
        u.x = pack2<T>(x[8 * j + 0], x[8 * j + 1]);
        u.y = pack2<T>(x[8 * j + 2], x[8 * j + 3]);
        u.z = pack2<T>(x[8 * j + 4], x[8 * j + 5]);
        u.w = pack2<T>(x[8 * j + 6], x[8 * j + 7]);
        o[j] = u;
    }
}

sf_status gemm_pair_dispatch(const sf_gemm_args& a, bool ln, cudaStream_t st);  // gemm2_tc.cu
bool gemm_pair_supported(const sf_gemm_args& a, bool ln);
int num_sms();

}  // namespace sf
