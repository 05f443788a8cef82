// attn_dense.cu — the dense masked SDPA reference on the device, fp64 accumulation.
// Replaces dense_sdpa_oracle (attention.hpp:15-56): scores Q.K^T * scale over the DENSE bit mask
// (no storage format involved), masked positions -inf, exact two-pass softmax (row max, then
// Σ exp(s - max) and Σ exp(s - max) V), query rows with no valid position stay exactly zero.
// It is an executor independent of the BSR / CSR builders, so `sparsefuse attn verify` can check
// both sparse executors against it on the GPU; it is not on any hot path.
//
// One warp per query row; lane l holds head dims 2l, 2l+1 of q and of the output accumulator;
// the key loop walks the row's mask words and skips masked keys 32 at a time.
#include "common.cuh"

namespace sf {
sf_status check_attn_args(const sf_attn_args& a);  // attn_simt.cu
namespace {

template <typename T>
__device__ __forceinline__ double2 ld2(const T* p);
template <>
__device__ __forceinline__ double2 ld2<__half>(const __half* p) {
    const __half2 h = *reinterpret_cast<const __half2*>(p);
    return make_double2(__half2float(h.x), __half2float(h.y));
}
template <>
__device__ __forceinline__ double2 ld2<__nv_bfloat16>(const __nv_bfloat16* p) {
    const __nv_bfloat162 h = *reinterpret_cast<const __nv_bfloat162*>(p);
    return make_double2(__bfloat162float(h.x), __bfloat162float(h.y));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <typename T>
__global__ void __launch_bounds__(256) dense_sdpa_kernel(sf_attn_args a, double scale, const uint32_t* __restrict__ bits,
                                                         double* __restrict__ o64) {
    const int lane = threadIdx.x & 31;
    const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const int64_t rows = static_cast<int64_t>(a.bs) * a.h * a.seq_len;
    if (row >= rows) return;
    const int n = a.seq_len;
    const int i = static_cast<int>(row % n);
    const int bh = static_cast<int>(row / n);
    const int b = bh / a.h, hh = bh % a.h;
    const T* q = static_cast<const T*>(a.q) + b * a.q_sb + hh * a.q_sh + static_cast<int64_t>(i) * a.q_sn;
    const T* kb = static_cast<const T*>(a.k) + b * a.q_sb + hh * a.q_sh;
    const T* vb = static_cast<const T*>(a.v) + b * a.q_sb + hh * a.q_sh;
    const bool have = 2 * lane < a.head_size;  // head_size <= 64, even (checked on the host)
    const double2 qv = have ? ld2<T>(q + 2 * lane) : make_double2(0.0, 0.0);
    const int words = (n + 31) / 32;
    const uint32_t* mrow = bits + static_cast<int64_t>(i) * words;
    auto score = [&](int j) {
        const double2 kv = have ? ld2<T>(kb + static_cast<int64_t>(j) * a.q_sn + 2 * lane) : make_double2(0.0, 0.0);
        return warp_sum(qv.x * kv.x + qv.y * kv.y) * scale;
    };
    // pass 1: row max over valid positions (attention.hpp:27-38)
    double mx = -INFINITY;
    for (int w = 0; w < words; ++w) {
        uint32_t m = mrow[w];
        while (m) {
            const int j = 32 * w + __ffs(m) - 1;
            m &= m - 1;
            mx = fmax(mx, score(j));
        }
    }
    double2 acc = make_double2(0.0, 0.0);
    if (mx != -INFINITY) {
        // pass 2: denominator and the unnormalised P.V (attention.hpp:40-51)
        double den = 0.0;
        for (int w = 0; w < words; ++w) {
            uint32_t m = mrow[w];
            while (m) {
                const int j = 32 * w + __ffs(m) - 1;
                m &= m - 1;
                const double p = exp(score(j) - mx);
                den += p;
                const double2 vv = have ? ld2<T>(vb + static_cast<int64_t>(j) * a.q_sn + 2 * lane) : make_double2(0.0, 0.0);
                acc.x += p * vv.x;
                acc.y += p * vv.y;
            }
        }
        acc.x /= den;
        acc.y /= den;
    }  // else: a fully masked row stays zero (attention.hpp:39)
    if (have) {
        double* dst = o64 + row * a.head_size + 2 * lane;
        dst[0] = acc.x;
        dst[1] = acc.y;
    }
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" sf_status sf_mha_dense_oracle(const sf_attn_args* args, const uint32_t* d_bits, double* o64, void* stream) {
    if (!args || !d_bits || !o64) return fail(SF_INVALID_PARAMETER, "null argument");
    SF_TRY(check_attn_args(*args));
    if (args->head_size > 64 || (args->head_size & 1))
        return fail(SF_SHAPE_ERROR, "dense oracle: head_size must be even and <= 64");
    if (args->q_sn % 2 || args->q_sh % 2 || args->q_sb % 2 || (reinterpret_cast<uintptr_t>(args->q) & 3) ||
        (reinterpret_cast<uintptr_t>(args->k) & 3) || (reinterpret_cast<uintptr_t>(args->v) & 3))
        return fail(SF_INVALID_PARAMETER, "dense oracle: Q/K/V strides must be even, pointers 4-byte aligned");
    const sf_attn_args a = *args;
    // 0 selects the reference's 1/sqrt(head_size), taken in double as the reference does
    const double scale = a.scale == 0.f ? 1.0 / std::sqrt(static_cast<double>(a.head_size)) : static_cast<double>(a.scale);
    const int64_t rows = static_cast<int64_t>(a.bs) * a.h * a.seq_len;
    const dim3 grid(static_cast<unsigned>((rows + 7) / 8)), block(256);
    cudaStream_t st = as_stream(stream);
    if (a.dtype == SF_F16) dense_sdpa_kernel<__half><<<grid, block, 0, st>>>(a, scale, d_bits, o64);
    else dense_sdpa_kernel<__nv_bfloat16><<<grid, block, 0, st>>>(a, scale, d_bits, o64);
    SF_LAUNCH_CHECK();
    return SF_OK;
}
