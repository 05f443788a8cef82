// strided.cu — masked MHA for the strided pattern by MASK DECOMPOSITION (the planner extension of
// DESIGN §6): strided(w) = { j <= i : i - j < w  or  (i - j) % w == 0 } is the disjoint union of
//   A = causal-local(w)                      { j <= i, i - j < w }            (a narrow band)
//   B = the strided diagonals beyond it      { i - j >= w, (i - j) % w == 0 }
// In the (128,16) BSR the diagonals of B cross every tile of the causal triangle (~1% useful cells
// at n = 8192), while A is a band the tcgen05 block kernel runs near its best rate.
// So A runs on attn_tc with a per-row log2-sum-exp2 output, and B is exact dense causal attention
// inside each residue class: rows i = r + w a and keys j = r + w b of class r (b < a) form a
// strictly-causal problem of ceil(n / w) rows, which this kernel computes with warp-level tensor
// core MMAs (mma.sync m16n8k16, fp32 accumulation) and merges into A's output:
//   O = (O_A 2^lse_A + O_B 2^lse_B) / (2^lse_A + 2^lse_B)  (attention.hpp:71-172 semantics over A u B).
// One CTA per (class, b*h slice); the class's Q / K / V rows (<= 128) are staged in shared memory
// with a 16-byte XOR swizzle (ldmatrix conflict-free); warp q owns class rows [16q, 16q + 16).
#include <algorithm>
#include <cmath>
#include <string>

#include "common.cuh"

namespace sf {
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t st);
sf_status attn_tc(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st, bool probe_only, float* lse);
sf_status check_attn_args(const sf_attn_args& a);
namespace {

constexpr int kMaxClassRows = 128;
constexpr int kDs = 64;

struct StridedParams {
    const void *q, *k, *v;
    void* o;
    int64_t q_sb, q_sh, q_sn, o_sb, o_sh, o_sn;
    int32_t n, h, w;
    float scale_log2;
    const float* lse;  // part A's per-row log2-sum-exp2, [b*h][n]
};

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ldsm_x4(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t a, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]) : "r"(a));
}
template <typename T>
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1);
template <>
__device__ __forceinline__ void mma16816<__half>(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
                 "{%0, %1, %2, %3};"
                 : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <typename T>
__device__ __forceinline__ uint32_t pack2t(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2t<__half>(float a, float b) {
    __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2t<__nv_bfloat16>(float a, float b) {
    __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
    return *reinterpret_cast<uint32_t*>(&h);
}

// byte offset of 16-byte chunk c of staged row a (row = 128 B, chunk index XOR row % 8)
__device__ __forceinline__ uint32_t swz(int a, int c) { return static_cast<uint32_t>(a * 128 + ((c ^ (a & 7)) << 4)); }

template <typename T>
__global__ void __launch_bounds__(256) strided_class_kernel(const StridedParams p) {
    // Q, K, V of the class: [3][apad rows][128 B]; apad = 16 x warps covers the longest class
    extern __shared__ __align__(128) unsigned char sm_dyn[];
    const int apad = static_cast<int>(blockDim.x >> 1);  // 16 rows per warp
    unsigned char* const sm[3] = {sm_dyn, sm_dyn + apad * 128, sm_dyn + 2 * apad * 128};
    pdl_enter();
    const int r = static_cast<int>(blockIdx.x);
    const int slice = static_cast<int>(blockIdx.y);
    const int b = slice / p.h, hh = slice % p.h;
    const int rows = (p.n - r + p.w - 1) / p.w;  // class rows i = r + w a < n
    const T* src[3] = {static_cast<const T*>(p.q), static_cast<const T*>(p.k), static_cast<const T*>(p.v)};
    const int64_t base = b * p.q_sb + hh * p.q_sh;
    // all rows in flight at once (cp.async; rows past the class are zero-filled)
    for (int idx = threadIdx.x; idx < 3 * apad * 8; idx += blockDim.x) {
        const int t = idx / (apad * 8), rem = idx % (apad * 8);
        const int a = rem >> 3, c = rem & 7;
        const bool ok = a < rows;
        const T* g = src[t] + base + (ok ? static_cast<int64_t>(r + p.w * a) * p.q_sn + 8 * c : 0);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(sm[t] + swz(a, c))), "l"(g),
                     "r"(ok ? 16 : 0)
                     : "memory");
    }
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    const int warp = static_cast<int>(threadIdx.x >> 5), lane = static_cast<int>(threadIdx.x & 31);
    const int row0 = 16 * warp;
    if (row0 >= rows || rows <= 1) return;  // class row 0 has no key in B
    const int g = lane >> 2, t4 = lane & 3;
    const uint32_t sQ = smem_addr(sm[0]), sK = smem_addr(sm[1]), sV = smem_addr(sm[2]);  // apad x 128 B each
    // Q fragments of the warp's 16 rows, four 16-wide k-steps over d
    uint32_t qa[4][4];
    {
        const int j = lane >> 3, ra = row0 + (j & 1) * 8 + (lane & 7);
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) ldsm_x4(sQ + swz(ra, 2 * ks + (j >> 1)), qa[ks]);
    }
    float acc[8][4];
#pragma unroll
    for (int dt = 0; dt < 8; ++dt)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[dt][e] = 0.f;
    float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
    const int a_r[2] = {row0 + g, row0 + g + 8};
    const float sl2 = p.scale_log2;
    for (int kt = 0; kt <= warp; ++kt) {  // keys b < a <= row0 + 15: key tiles 0 .. warp
        float s[2][4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) s[nt][e] = 0.f;
        {
            const int j = lane >> 3, kb = 16 * kt + (j >> 1) * 8 + (lane & 7);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
                uint32_t kf[4];
                ldsm_x4(sK + swz(kb, 2 * ks + (j & 1)), kf);
                mma16816<T>(s[0], qa[ks], kf[0], kf[1]);
                mma16816<T>(s[1], qa[ks], kf[2], kf[3]);
            }
        }
        // strictly causal inside the class (b < a), rows past the class masked, log2 domain
        float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int hr = e >> 1, kb = 16 * kt + 8 * nt + 2 * t4 + (e & 1);
                const bool ok = kb < a_r[hr] && a_r[hr] < rows;
                s[nt][e] = ok ? s[nt][e] * sl2 : -INFINITY;
                mx[hr] = fmaxf(mx[hr], s[nt][e]);
            }
        float alpha[2];
#pragma unroll
        for (int hr = 0; hr < 2; ++hr) {
            mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 1));
            mx[hr] = fmaxf(mx[hr], __shfl_xor_sync(0xffffffffu, mx[hr], 2));
            const float mn = fmaxf(m[hr], mx[hr]);
            alpha[hr] = (m[hr] == -INFINITY) ? 0.f : exp2f(m[hr] - mn);
            m[hr] = mn;
            l[hr] *= alpha[hr];
        }
        uint32_t pa[4];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
            float pv[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int hr = e >> 1;
                pv[e] = (m[hr] == -INFINITY) ? 0.f : exp2f(s[nt][e] - m[hr]);
                l[hr] += pv[e];
            }
            pa[2 * nt] = pack2t<T>(pv[0], pv[1]);      // row g,   keys 8nt + 2t4 .. +1
            pa[2 * nt + 1] = pack2t<T>(pv[2], pv[3]);  // row g+8
        }
        const uint32_t a4[4] = {pa[0], pa[1], pa[2], pa[3]};
#pragma unroll
        for (int dt = 0; dt < 8; ++dt) {
            acc[dt][0] *= alpha[0];
            acc[dt][1] *= alpha[0];
            acc[dt][2] *= alpha[1];
            acc[dt][3] *= alpha[1];
        }
        {
            const int j = lane >> 3, kb = 16 * kt + (j & 1) * 8 + (lane & 7);
#pragma unroll
            for (int d2 = 0; d2 < 4; ++d2) {
                uint32_t vf[4];
                ldsm_x4_t(sV + swz(kb, 2 * d2 + (j >> 1)), vf);
                mma16816<T>(acc[2 * d2], a4, vf[0], vf[1]);
                mma16816<T>(acc[2 * d2 + 1], a4, vf[2], vf[3]);
            }
        }
    }
    // merge with part A's output (normalised) and log2-sum-exp2, in place
#pragma unroll
    for (int hr = 0; hr < 2; ++hr) {
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 1);
        l[hr] += __shfl_xor_sync(0xffffffffu, l[hr], 2);
        const int a = a_r[hr];
        if (a < 1 || a >= rows || l[hr] <= 0.f) continue;
        const int64_t i = r + static_cast<int64_t>(p.w) * a;
        const float lse_b = m[hr] + __log2f(l[hr]);
        const float lse_a = p.lse[static_cast<int64_t>(slice) * p.n + i];
        const float mm = fmaxf(lse_a, lse_b);
        const float wa = lse_a == -INFINITY ? 0.f : exp2f(lse_a - mm), wb = exp2f(lse_b - mm);
        const float inv = 1.f / (wa + wb);
        const float cb = wb * inv / l[hr], ca = wa * inv;
        T* orow = static_cast<T*>(p.o) + b * p.o_sb + hh * p.o_sh + i * p.o_sn;
#pragma unroll
        for (int dt = 0; dt < 8; ++dt) {
            uint32_t* op = reinterpret_cast<uint32_t*>(orow + 8 * dt + 2 * t4);
            const uint32_t ov = *op;
            const T* oh = reinterpret_cast<const T*>(&ov);
            const float o0 = DT<T>::to_f(oh[0]) * ca + acc[dt][2 * hr] * cb;
            const float o1 = DT<T>::to_f(oh[1]) * ca + acc[dt][2 * hr + 1] * cb;
            *op = pack2t<T>(o0, o1);
        }
    }
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" sf_status sf_mha_strided(const sf_attn_args* args, int32_t band_width, const sf_bsr_dev* band_bsr,
                                    void* stream) {
    if (!args || !band_bsr) return fail(SF_INVALID_PARAMETER, "null argument");
    SF_TRY(check_attn_args(*args));
    const sf_attn_args& a0 = *args;
    if (band_width < 1 || band_width > a0.seq_len) return fail(SF_INVALID_PARAMETER, "band_width must be in [1, seq_len]");
    if (band_bsr->seq_len != a0.seq_len) return fail(SF_SHAPE_ERROR, "band BSR seq_len differs from input");
    if (a0.head_size != kDs || (band_bsr->block_m != 128 && band_bsr->block_m != 64) ||
        (a0.seq_len + band_width - 1) / band_width > kMaxClassRows || static_cast<int64_t>(a0.bs) * a0.h > 65535)
        return fail(SF_PLAN_ERROR, "strided decomposition needs head_size 64, a block_m 128 (or 64: head pairs) band BSR, "
                                   "ceil(seq_len / band_width) <= 128 and bs * h <= 65535");
    if ((a0.q_sn | a0.q_sh | a0.q_sb | a0.o_sn | a0.o_sh | a0.o_sb) % 8 ||
        ((reinterpret_cast<uintptr_t>(a0.q) | reinterpret_cast<uintptr_t>(a0.k) | reinterpret_cast<uintptr_t>(a0.v) |
          reinterpret_cast<uintptr_t>(a0.o)) & 15))
        return fail(SF_INVALID_PARAMETER, "strides must be multiples of 8 elements and tensors 16-byte aligned");
    cudaStream_t st = as_stream(stream);
    sf_attn_args a = a0;
    if (a.scale == 0.f) a.scale = 1.0f / std::sqrt(static_cast<float>(a.head_size));
    void* lse = nullptr;
    const size_t lse_bytes = static_cast<size_t>(a.bs) * a.h * a.seq_len * sizeof(float);
    SF_CUDA_TRY(pool_malloc(&lse, lse_bytes, st));
    // part A: the causal-local band on the tcgen05 block kernel, with per-row log2-sum-exp2
    sf_status status = attn_tc(a, *band_bsr, st, false, static_cast<float*>(lse));
    if (status == SF_OK) {
        StridedParams p{};
        p.q = a.q; p.k = a.k; p.v = a.v; p.o = a.o;
        p.q_sb = a.q_sb; p.q_sh = a.q_sh; p.q_sn = a.q_sn;
        p.o_sb = a.o_sb; p.o_sh = a.o_sh; p.o_sn = a.o_sn;
        p.n = a.seq_len; p.h = a.h; p.w = band_width;
        p.scale_log2 = a.scale * 1.4426950408889634f;
        p.lse = static_cast<const float*>(lse);
        const dim3 grid(static_cast<unsigned>(band_width), static_cast<unsigned>(a.bs * a.h));
        const int warps = (ceil_div(a.seq_len, band_width) + 15) / 16;  // 16 class rows per warp
        const int smem = 3 * 16 * warps * 128;
        auto kern = a.dtype == SF_BF16 ? strided_class_kernel<__nv_bfloat16> : strided_class_kernel<__half>;
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 3 * kMaxClassRows * 128);
        if (e == cudaSuccess) e = launch_pdl(kern, grid, dim3(32 * warps), smem, st, nullptr, p);
        if (e != cudaSuccess) status = fail(SF_CUDA_ERROR, std::string("strided class kernel: ") + cudaGetErrorString(e));
        else note_launch();
    }
    cudaFreeAsync(lse, st);
    return status;
}
