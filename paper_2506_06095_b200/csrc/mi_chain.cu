// mi_chain.cu — the MiChain template (backend.hpp:228-235): a run of memory-intensive ops
// (Bias, GELU/ReLU, Add, then a LayerNorm or Softmax row op) applied to each row in ONE pass
// over HBM.
//
// One warp per row, 8 rows per 256-thread CTA. Each lane holds chunks of 8 consecutive
// elements (16-byte vector loads/stores; a scalar variant covers ragged widths), so a row is read once and written once however many
// ops are fused; the LayerNorm statistics are warp-shuffle reductions (two-pass mean / biased
// variance, eps 1e-5, backend.hpp:141-154). HBM-bound: 2*N*2 bytes per row (+aux).
#include <algorithm>

#include "epilogue.cuh"

namespace sf {
namespace {

constexpr int kWarpsPerCta = 8;

__device__ __forceinline__ float gelu_erf(float x) { return gelu_fast(x); }  // epilogue.cuh

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// W = 8: one 16-byte vector per lane chunk; W = 1: scalar fallback for ragged widths / strides.
template <typename T, int W>
__device__ __forceinline__ void loadw(const T* p, float* f) {
    if constexpr (W == 8) {
        const uint4 raw = *reinterpret_cast<const uint4*>(p);
        const T* h = reinterpret_cast<const T*>(&raw);
#pragma unroll
        for (int e = 0; e < 8; ++e) f[e] = DT<T>::to_f(h[e]);
    } else {
        f[0] = DT<T>::to_f(*p);
    }
}
template <typename T, int W>
__device__ __forceinline__ void storew(T* p, const float* f) {
    if constexpr (W == 8) {
        uint4 raw;
        T* h = reinterpret_cast<T*>(&raw);
#pragma unroll
        for (int e = 0; e < 8; ++e) h[e] = DT<T>::from_f(f[e]);
        *reinterpret_cast<uint4*>(p) = raw;
    } else {
        *p = DT<T>::from_f(f[0]);
    }
}

template <typename T, int V, int W>
__global__ void __launch_bounds__(kWarpsPerCta * 32) mi_chain_kernel(int32_t M, int32_t N, const T* __restrict__ x,
                                                                     int64_t ldx, sf_gemm_epilogue e,
                                                                     T* __restrict__ out, int64_t ldout) {
    pdl_enter();
    const int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + (threadIdx.x >> 5);
    if (row >= M) return;
    const int lane = threadIdx.x & 31;
    const float* bias = static_cast<const float*>(e.bias);
    const T* aux = static_cast<const T*>(e.aux);
    float v[V][W];
#pragma unroll
    for (int k = 0; k < V; ++k) {
        const int c = (k * 32 + lane) * W;  // chunk k of W elements: lanes interleave -> coalesced
        if (c < N) {
            loadw<T, W>(x + row * ldx + c, v[k]);
            if (bias)
#pragma unroll
                for (int i = 0; i < W; ++i) v[k][i] += bias[c + i];
            if (e.act == SF_ACT_GELU)
#pragma unroll
                for (int i = 0; i < W; ++i) v[k][i] = gelu_erf(v[k][i]);
            else if (e.act == SF_ACT_RELU)
#pragma unroll
                for (int i = 0; i < W; ++i) v[k][i] = v[k][i] > 0.f ? v[k][i] : 0.f;
            if (aux) {
                float a[W];
                loadw<T, W>(aux + row * e.ldaux + c, a);
#pragma unroll
                for (int i = 0; i < W; ++i) v[k][i] += a[i];
            }
        } else {
#pragma unroll
            for (int i = 0; i < W; ++i) v[k][i] = 0.f;
        }
    }
    if (e.softmax) {  // apply_row_op Softmax (backend.hpp:155-167): max, exp(x - max), / sum
        float m = -INFINITY;
#pragma unroll
        for (int k = 0; k < V; ++k)
            if ((k * 32 + lane) * W < N)
#pragma unroll
                for (int i = 0; i < W; ++i) m = fmaxf(m, v[k][i]);
        m = warp_max(m);
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k)
            if ((k * 32 + lane) * W < N)
#pragma unroll
                for (int i = 0; i < W; ++i) {
                    v[k][i] = __expf(v[k][i] - m);
                    s += v[k][i];
                }
        const float inv = 1.0f / warp_sum(s);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const int c = (k * 32 + lane) * W;
            if (c >= N) continue;
#pragma unroll
            for (int i = 0; i < W; ++i) v[k][i] *= inv;
            storew<T, W>(out + row * ldout + c, v[k]);
        }
    } else if (e.ln_gamma) {
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k)
#pragma unroll
            for (int i = 0; i < W; ++i) s += v[k][i];
        const float mean = warp_sum(s) / static_cast<float>(N);
        float q = 0.f;
#pragma unroll
        for (int k = 0; k < V; ++k)
            if ((k * 32 + lane) * W < N)
#pragma unroll
                for (int i = 0; i < W; ++i) q += (v[k][i] - mean) * (v[k][i] - mean);
        const float inv = 1.0f / sqrtf(warp_sum(q) / static_cast<float>(N) + 1e-5f);
        const float* g = static_cast<const float*>(e.ln_gamma);
        const float* b = static_cast<const float*>(e.ln_beta);
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const int c = (k * 32 + lane) * W;
            if (c >= N) continue;
            if (e.out_pre_ln) storew<T, W>(static_cast<T*>(e.out_pre_ln) + row * ldout + c, v[k]);
            float y[W];
#pragma unroll
            for (int i = 0; i < W; ++i) y[i] = (v[k][i] - mean) * inv * g[c + i] + b[c + i];
            storew<T, W>(out + row * ldout + c, y);
        }
    } else {
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const int c = (k * 32 + lane) * W;
            if (c < N) storew<T, W>(out + row * ldout + c, v[k]);
        }
    }
}

// Persistent-warp variant for rows of <= 1024 columns (16-byte vectors). The per-row variant
// above re-reads bias / gamma / beta through L1 for every row with 32-byte-strided lanes
// (~400 L1 wavefronts per row, which dominated its run time); here each CTA stages them once in
// shared memory in a lane-permuted layout — the float4 lane l reads for (chunk k, half h) sits at
// float4 index (2k + h) * 32 + l, so a warp's read is 4 conflict-free wavefronts — and every warp
// walks rows (one row's vectors per warp in flight; a one-row-ahead prefetch measured no faster).
template <typename T, int V, int ACT>
__global__ void __launch_bounds__(kWarpsPerCta * 32, V >= 4 ? 2 : 3) mi_chain_rows_kernel(int32_t M, int32_t N,
                                                                          const T* __restrict__ x, int64_t ldx,
                                                                          sf_gemm_epilogue e, T* __restrict__ out,
                                                                          int64_t ldout) {
    __shared__ float4 sprm[3][2 * V * 32];  // bias, gamma, beta
    const int lane = threadIdx.x & 31;
    const T* aux = static_cast<const T*>(e.aux);
    const bool ln = e.ln_gamma != nullptr;
    const float* src[3] = {static_cast<const float*>(e.bias), static_cast<const float*>(e.ln_gamma),
                           static_cast<const float*>(e.ln_beta)};
    for (int t = threadIdx.x; t < 2 * V * 32; t += blockDim.x) {
        const int l = t & 31, kh = t >> 5;            // float4 slot (2k + h) * 32 + l
        const int c = ((kh >> 1) * 32 + l) * 8 + (kh & 1) * 4;  // first column it holds
#pragma unroll
        for (int j = 0; j < 3; ++j)
            sprm[j][t] = (src[j] && c < N) ? *reinterpret_cast<const float4*>(src[j] + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    __syncthreads();
    pdl_enter();  // the parameter staging above overlaps the stream predecessor's tail
    const int64_t stride = static_cast<int64_t>(gridDim.x) * kWarpsPerCta;
    int64_t row = static_cast<int64_t>(blockIdx.x) * kWarpsPerCta + (threadIdx.x >> 5);
    bool ok[V];
#pragma unroll
    for (int k = 0; k < V; ++k) ok[k] = (k * 32 + lane) * 8 < N;
    // volatile shared loads: re-read per row (cheap, conflict-free) instead of being hoisted out of
    // the row loop into registers by the compiler, which spilled
    auto prm = [&](int j, int k, float (&f)[8]) {
        const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(&sprm[j][(2 * k) * 32 + lane]));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(f[0]), "=f"(f[1]), "=f"(f[2]), "=f"(f[3]) : "r"(a));
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(f[4]), "=f"(f[5]), "=f"(f[6]), "=f"(f[7]) : "r"(a + 512));
    };
    uint4 nx[V], na[V];
    auto fetch = [&](int64_t r) {
        if (r >= M) return;
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const int c = (k * 32 + lane) * 8;
            if (!ok[k]) continue;
            nx[k] = *reinterpret_cast<const uint4*>(x + r * ldx + c);
            if (aux) na[k] = *reinterpret_cast<const uint4*>(aux + r * e.ldaux + c);
        }
    };
#pragma unroll 1
    for (; row < M; row += stride) {
        fetch(row);
        float v[V][8];
#pragma unroll
        for (int k = 0; k < V; ++k) {
            const T* hx = reinterpret_cast<const T*>(&nx[k]);
            const T* ha = reinterpret_cast<const T*>(&na[k]);
            float bs[8];
            prm(0, k, bs);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float a = DT<T>::to_f(hx[i]) + bs[i];
                if constexpr (ACT == SF_ACT_GELU) a = gelu_erf(a);
                else if constexpr (ACT == SF_ACT_RELU) a = a > 0.f ? a : 0.f;
                if (aux) a += DT<T>::to_f(ha[i]);
                v[k][i] = ok[k] ? a : 0.f;
            }
        }
        if (ln) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < V; ++k)
#pragma unroll
                for (int i = 0; i < 8; ++i) s += v[k][i];
            const float mean = warp_sum(s) / static_cast<float>(N);
            float q = 0.f;
#pragma unroll
            for (int k = 0; k < V; ++k)
                if (ok[k])
#pragma unroll
                    for (int i = 0; i < 8; ++i) q += (v[k][i] - mean) * (v[k][i] - mean);
            const float inv = 1.0f / sqrtf(warp_sum(q) / static_cast<float>(N) + 1e-5f);
#pragma unroll
            for (int k = 0; k < V; ++k) {
                if (!ok[k]) continue;
                const int c = (k * 32 + lane) * 8;
                if (e.out_pre_ln) storew<T, 8>(static_cast<T*>(e.out_pre_ln) + row * ldout + c, v[k]);
                float g[8], b[8], y[8];
                prm(1, k, g);
                prm(2, k, b);
#pragma unroll
                for (int i = 0; i < 8; ++i) y[i] = (v[k][i] - mean) * inv * g[i] + b[i];
                storew<T, 8>(out + row * ldout + c, y);
            }
        } else {
#pragma unroll
            for (int k = 0; k < V; ++k)
                if (ok[k]) storew<T, 8>(out + row * ldout + (k * 32 + lane) * 8, v[k]);
        }
    }
}

template <typename T, int V, int ACT>
void launch_rows_act(int32_t M, int32_t N, const T* x, int64_t ldx, const sf_gemm_epilogue& e, T* out,
                     int64_t ldout, cudaStream_t st) {
    static int per_sm = 0;
    if (!per_sm) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mi_chain_rows_kernel<T, V, ACT>, kWarpsPerCta * 32, 0);
        if (per_sm <= 0) per_sm = 1;
    }
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t need = ceil_div(M, kWarpsPerCta);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(need, static_cast<int64_t>(sms) * per_sm));
    (void)launch_pdl(mi_chain_rows_kernel<T, V, ACT>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, x, ldx, e, out,
                     ldout);  // errors surface in the caller's SF_LAUNCH_CHECK
}

template <typename T, int V>
void launch_rows(int32_t M, int32_t N, const T* x, int64_t ldx, const sf_gemm_epilogue& e, T* out, int64_t ldout,
                 cudaStream_t st) {
    if (e.act == SF_ACT_GELU) launch_rows_act<T, V, SF_ACT_GELU>(M, N, x, ldx, e, out, ldout, st);
    else if (e.act == SF_ACT_RELU) launch_rows_act<T, V, SF_ACT_RELU>(M, N, x, ldx, e, out, ldout, st);
    else launch_rows_act<T, V, SF_ACT_NONE>(M, N, x, ldx, e, out, ldout, st);
}

// Chains without LayerNorm are elementwise: one thread per 8-element vector (grid-stride),
// bias as two float4 loads. HBM-bound at any row width.
template <typename T, int ACT>
__global__ void __launch_bounds__(256) mi_chain_ew_kernel(int32_t M, int32_t N, const T* __restrict__ x, int64_t ldx,
                                                          sf_gemm_epilogue e, T* __restrict__ out, int64_t ldout) {
    pdl_enter();
    const int64_t vpr = N / 8;  // vectors per row
    const int64_t total = static_cast<int64_t>(M) * vpr;
    const float* bias = static_cast<const float*>(e.bias);
    const T* aux = static_cast<const T*>(e.aux);
    for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
         t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = t / vpr;
        const int c = static_cast<int>(t - r * vpr) * 8;
        float v[8];
        loadw<T, 8>(x + r * ldx + c, v);
        if (bias) {
            const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + c));
            const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + c + 4));
            v[0] += b0.x; v[1] += b0.y; v[2] += b0.z; v[3] += b0.w;
            v[4] += b1.x; v[5] += b1.y; v[6] += b1.z; v[7] += b1.w;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if constexpr (ACT == SF_ACT_GELU) v[i] = gelu_erf(v[i]);
            else if constexpr (ACT == SF_ACT_RELU) v[i] = v[i] > 0.f ? v[i] : 0.f;
        }
        if (aux) {
            float a[8];
            loadw<T, 8>(aux + r * e.ldaux + c, a);
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] += a[i];
        }
        storew<T, 8>(out + r * ldout + c, v);
    }
}

template <typename T>
void launch_ew(int32_t M, int32_t N, const T* x, int64_t ldx, const sf_gemm_epilogue& e, T* out, int64_t ldout,
               cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t total = static_cast<int64_t>(M) * (N / 8);
    const unsigned grid = static_cast<unsigned>(std::min<int64_t>(ceil_div(total, 256), static_cast<int64_t>(sms) * 8));
    if (e.act == SF_ACT_GELU) (void)launch_pdl(mi_chain_ew_kernel<T, SF_ACT_GELU>, grid, dim3(256), 0, st, nullptr, M, N, x, ldx, e, out, ldout);
    else if (e.act == SF_ACT_RELU) (void)launch_pdl(mi_chain_ew_kernel<T, SF_ACT_RELU>, grid, dim3(256), 0, st, nullptr, M, N, x, ldx, e, out, ldout);
    else (void)launch_pdl(mi_chain_ew_kernel<T, SF_ACT_NONE>, grid, dim3(256), 0, st, nullptr, M, N, x, ldx, e, out, ldout);
}

template <typename T, int W>
sf_status launch(int32_t M, int32_t N, const void* x, int64_t ldx, const sf_gemm_epilogue& e, void* out, int64_t ldout,
                 cudaStream_t st) {
    const unsigned grid = static_cast<unsigned>(ceil_div(M, kWarpsPerCta));
    const T* xp = static_cast<const T*>(x);
    T* op = static_cast<T*>(out);
    const int chunks = static_cast<int>(ceil_div(N, 32 * W));  // chunks of 32 lanes x W elements
    constexpr int kMax = 4096 / (32 * W);
    // the row kernel keeps a row in registers (N <= 4096); vectorised elementwise chains run
    // grid-stride at any width. A width limit is a backend limit, not a shape mismatch, so the
    // search skips such candidates (search.hpp:339) instead of aborting.
    const bool row_op = e.ln_gamma || e.softmax;
    if (chunks > kMax && (W != 8 || row_op))
        return fail(SF_BACKEND_ERROR, "mi_chain: LayerNorm / Softmax / unaligned rows support N <= 4096");
    if constexpr (W == 8) {
        if (!row_op) {
            launch_ew<T>(M, N, xp, ldx, e, op, ldout, st);
            SF_LAUNCH_CHECK();
            return SF_OK;
        }
        if (chunks <= 4 && !e.softmax) {
            if (chunks == 1) launch_rows<T, 1>(M, N, xp, ldx, e, op, ldout, st);
            else if (chunks == 2) launch_rows<T, 2>(M, N, xp, ldx, e, op, ldout, st);
            else if (chunks == 3) launch_rows<T, 3>(M, N, xp, ldx, e, op, ldout, st);
            else launch_rows<T, 4>(M, N, xp, ldx, e, op, ldout, st);
            SF_LAUNCH_CHECK();
            return SF_OK;
        }
    }
    if (chunks <= 1) SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 1, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
    else if (chunks <= 2) SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 2, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
    else if (chunks <= 4) SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 4, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
    else if (chunks <= 8) SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 8, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
    else if (chunks <= 16) SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 16, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
    else if constexpr (kMax > 16) {
        if (chunks <= 32) SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 32, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
        else if (chunks <= 64) SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 64, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
        else SF_CUDA_TRY(launch_pdl(mi_chain_kernel<T, 128, W>, grid, dim3(kWarpsPerCta * 32), 0, st, nullptr, M, N, xp, ldx, e, op, ldout));
    }
    SF_LAUNCH_CHECK();
    return SF_OK;
}

template <typename T>
sf_status launch_any(int32_t M, int32_t N, const void* x, int64_t ldx, const sf_gemm_epilogue& e, void* out,
                     int64_t ldout, cudaStream_t st) {
    const bool vec = N % 8 == 0 && ldx % 8 == 0 && ldout % 8 == 0 && (!e.aux || e.ldaux % 8 == 0) &&
                     ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out) |
                       reinterpret_cast<uintptr_t>(e.aux) | reinterpret_cast<uintptr_t>(e.out_pre_ln)) & 15) == 0;
    return vec ? launch<T, 8>(M, N, x, ldx, e, out, ldout, st) : launch<T, 1>(M, N, x, ldx, e, out, ldout, st);
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" sf_status sf_mi_chain(int32_t M, int32_t N, int32_t dtype, const void* x, int64_t ldx,
                                 const sf_gemm_epilogue* epi, void* out, int64_t ldout, void* stream) {
    if (M < 1 || N < 1) return fail(SF_SHAPE_ERROR, "empty matrix");
    sf_gemm_epilogue e = epi ? *epi : sf_gemm_epilogue{};
    if (e.ln_gamma && !e.ln_beta) return fail(SF_INVALID_PARAMETER, "LayerNorm needs gamma and beta");
    if (e.ln_gamma && e.softmax) return fail(SF_INVALID_PARAMETER, "LayerNorm and Softmax are separate row ops");
    if (e.softmax && e.out_pre_ln) return fail(SF_INVALID_PARAMETER, "out_pre_ln belongs to LayerNorm");
    cudaStream_t st = as_stream(stream);
    if (dtype == SF_F16) return launch_any<__half>(M, N, x, ldx, e, out, ldout, st);
    if (dtype == SF_BF16) return launch_any<__nv_bfloat16>(M, N, x, ldx, e, out, ldout, st);
    return fail(SF_INVALID_PARAMETER, "dtype must be f16/bf16");
}
