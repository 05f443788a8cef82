// attn_simt.cu — CUDA-core attention executors.
//
// attn_rowwise: replaces rowwise_sdpa (attention.hpp:177-213). One warp per (b, h, query row),
//   split into 4 groups of 8 lanes; each group handles one gathered key at a time, so a K/V row
//   of d fp16 is read by 8 lanes with 16-byte vector loads (coalesced 128-byte row for d=64).
//   Per-group online softmax in fp32, merged across the 4 groups with shuffles at the end.
//   attn_rowwise64: the head-size-64 specialisation (four keys in flight per group, FFMA2, lazy
//   max update).
//
// attn_bsr_generic: the block-skipping executor (attention.hpp:71-172) for ANY tile shape the
//   reference accepts (the tcgen05 kernel in attn_tc.cu covers block_m = 128). One CTA per
//   (row block, b*h); one thread per query row; K/V tiles staged through shared memory; the
//   per-load-entry tile id (-1 = full) replaces the merge walk.
#include <cmath>
#include <algorithm>
#include <type_traits>

#include "common.cuh"

namespace sf {
namespace {

template <typename T>
__device__ __forceinline__ void load8(const T* p, float* f) {
    // 8 consecutive 16-bit elements -> fp32 (16-byte aligned vector load)
    const uint4 raw = *reinterpret_cast<const uint4*>(p);
    const T* h = reinterpret_cast<const T*>(&raw);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = DT<T>::to_f(h[e]);
}

// DPL = dims per lane (ceil(d / 8)); VEC = 16-byte vector loads (d % 64 == 0, aligned strides).
template <typename T, int DPL, bool VEC>
__global__ void __launch_bounds__(256) attn_rowwise_kernel(sf_attn_args a, const int32_t* __restrict__ row_ptr,
                                                           const int32_t* __restrict__ col_idx) {
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t rows = static_cast<int64_t>(a.bs) * a.h * a.seq_len;
    if (gw >= rows) return;
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const int64_t i = gw % a.seq_len;
    const int64_t bh = gw / a.seq_len;
    const int64_t b = bh / a.h, hh = bh % a.h;
    const T* Q = static_cast<const T*>(a.q) + b * a.q_sb + hh * a.q_sh;
    const T* K = static_cast<const T*>(a.k) + b * a.q_sb + hh * a.q_sh;
    const T* V = static_cast<const T*>(a.v) + b * a.q_sb + hh * a.q_sh;
    T* O = static_cast<T*>(a.o) + b * a.o_sb + hh * a.o_sh + i * a.o_sn;
    const int d = a.head_size;
    const int d0 = gl * DPL;
    const float sl2 = a.scale * 1.4426950408889634f;
    float q[DPL], acc[DPL];
#pragma unroll
    for (int e = 0; e < DPL; ++e) {
        q[e] = (d0 + e < d) ? DT<T>::to_f(Q[i * a.q_sn + d0 + e]) : 0.f;
        acc[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    const int32_t r0 = row_ptr[i], r1 = row_ptr[i + 1];
    for (int32_t kk = r0 + grp; kk < r1; kk += 4) {
        const int64_t j = col_idx[kk];
        float kv[DPL];
        if constexpr (VEC) {
#pragma unroll
            for (int e = 0; e < DPL; e += 8) load8(K + j * a.q_sn + d0 + e, kv + e);
        } else {
#pragma unroll
            for (int e = 0; e < DPL; ++e) kv[e] = (d0 + e < d) ? DT<T>::to_f(K[j * a.q_sn + d0 + e]) : 0.f;
        }
        float dot = 0.f;
#pragma unroll
        for (int e = 0; e < DPL; ++e) dot += q[e] * kv[e];
        // groups run different trip counts: reduce within the group's own 8 lanes only
        const unsigned gmask = 0xffu << (grp * 8);
        dot += __shfl_xor_sync(gmask, dot, 1);
        dot += __shfl_xor_sync(gmask, dot, 2);
        dot += __shfl_xor_sync(gmask, dot, 4);
        const float s = dot * sl2;  // log2-domain score
        const float mn = fmaxf(m, s);
        const float alpha = exp2f(m - mn);  // m == -inf -> 0
        const float p = exp2f(s - mn);
        l = l * alpha + p;
        if constexpr (VEC) {
#pragma unroll
            for (int e = 0; e < DPL; e += 8) load8(V + j * a.q_sn + d0 + e, kv + e);
        } else {
#pragma unroll
            for (int e = 0; e < DPL; ++e) kv[e] = (d0 + e < d) ? DT<T>::to_f(V[j * a.q_sn + d0 + e]) : 0.f;
        }
#pragma unroll
        for (int e = 0; e < DPL; ++e) acc[e] = acc[e] * alpha + p * kv[e];
        m = mn;
    }
    // merge the 4 groups (lanes gl, gl+8, gl+16, gl+24 hold the same dims)
#pragma unroll
    for (int o = 8; o < 32; o <<= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float l2 = __shfl_xor_sync(0xffffffffu, l, o);
        const float mn = fmaxf(m, m2);
        const float a1 = (m == -INFINITY) ? 0.f : exp2f(m - mn);
        const float a2 = (m2 == -INFINITY) ? 0.f : exp2f(m2 - mn);
#pragma unroll
        for (int e = 0; e < DPL; ++e) {
            const float x2 = __shfl_xor_sync(0xffffffffu, acc[e], o);
            acc[e] = acc[e] * a1 + x2 * a2;
        }
        l = l * a1 + l2 * a2;
        m = mn;
    }
    if (grp == 0) {
        const float inv = l > 0.f ? 1.f / l : 0.f;  // rows without valid columns stay zero
#pragma unroll
        for (int e = 0; e < DPL; ++e)
            if (d0 + e < d) O[d0 + e] = DT<T>::from_f(acc[e] * inv);
    }
}

// Head size 64, 16-byte aligned rows (the common case): same warp/group geometry, but each
// group keeps FOUR gathered keys in flight (8 x 16-byte loads issued before any use), the dot and
// P.V updates run as packed fp32 pairs (FFMA2), and the running max is updated lazily (rescale
// only when a score exceeds the max by > 2^8, so p <= 256): one exp2 per key instead of two.
__device__ __forceinline__ void h8_to_f(const uint4& raw, float2 (&f)[4]) {
    const __half2* h = reinterpret_cast<const __half2*>(&raw);
#pragma unroll
    for (int e = 0; e < 4; ++e) f[e] = __half22float2(h[e]);
}
__device__ __forceinline__ void h8_to_f(const uint4& raw, float2 (&f)[4], __nv_bfloat16) {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&raw);
#pragma unroll
    for (int e = 0; e < 4; ++e) f[e] = __bfloat1622float2(h[e]);
}
template <typename T>
__device__ __forceinline__ void cvt8(const uint4& raw, float2 (&f)[4]) {
    if constexpr (std::is_same<T, __half>::value) h8_to_f(raw, f);
    else h8_to_f(raw, f, __nv_bfloat16{});
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\tmov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
        "mov.b64 rc, {%6, %7};\n\tfma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

// RPW = rows per warp: 1 -> the four groups split one row's keys and merge at the end; 4 -> each
// group owns a row (short rows: no idle groups, no merge, a quarter of the warps).
template <typename T, int RPW>
#ifndef SF_RW_MINB
#define SF_RW_MINB 4  // <= 64 registers: 32 warps per SM hide the row_ptr -> col_idx -> K/V chain (10-14% faster)
#endif
__global__ void __launch_bounds__(256, SF_RW_MINB) attn_rowwise64_kernel(sf_attn_args a, const int32_t* __restrict__ row_ptr,
                                                             const int32_t* __restrict__ col_idx) {
    constexpr float kLazy = 8.0f;
    constexpr int kStride = RPW == 1 ? 4 : 1;  // key stride of one group
    const int64_t gw = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t rows = static_cast<int64_t>(a.bs) * a.h * a.seq_len;
    const int lane = threadIdx.x & 31, grp = lane >> 3, gl = lane & 7;
    const int64_t row_id = RPW == 1 ? gw : gw * 4 + grp;
    if (row_id >= rows) return;  // RPW 4: a whole group leaves (its shuffles are group-local)
    const int64_t i = row_id % a.seq_len;
    const int64_t bh = row_id / a.seq_len;
    const int64_t b = bh / a.h, hh = bh % a.h;
    const int64_t base = b * a.q_sb + hh * a.q_sh + gl * 8;
    const T* Q = static_cast<const T*>(a.q) + base;
    const T* K = static_cast<const T*>(a.k) + base;
    const T* V = static_cast<const T*>(a.v) + base;
    const float sl2 = a.scale * 1.4426950408889634f;
    float2 q[4], acc[4];
    {
        cvt8<T>(*reinterpret_cast<const uint4*>(Q + i * a.q_sn), q);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            q[e] = make_float2(q[e].x * sl2, q[e].y * sl2);  // scores come out in the log2 domain
            acc[e] = make_float2(0.f, 0.f);
        }
    }
    float m = -INFINITY, l = 0.f;
    const unsigned gmask = 0xffu << (grp * 8);
    const int32_t r0 = row_ptr[i], r1 = row_ptr[i + 1];
    // kNK keys per group in flight: all column indices, then all K and V rows are requested before
    // any is used (the loop is bound by dependent gather latency, not by arithmetic)
    constexpr int kNK = 4;
    for (int32_t kk = r0 + (RPW == 1 ? grp : 0); kk < r1; kk += kStride * kNK) {
        int64_t jj[kNK];
        bool live[kNK];
#pragma unroll
        for (int t = 0; t < kNK; ++t) {
            live[t] = kk + kStride * t < r1;  // group-uniform
            jj[t] = live[t] ? col_idx[kk + kStride * t] : 0;
        }
        uint4 kr[kNK], vr[kNK];
#pragma unroll
        for (int t = 0; t < kNK; ++t) kr[t] = *reinterpret_cast<const uint4*>(K + jj[t] * a.q_sn);
#pragma unroll
        for (int t = 0; t < kNK; ++t) vr[t] = *reinterpret_cast<const uint4*>(V + jj[t] * a.q_sn);
        float sc[kNK];
#pragma unroll
        for (int t = 0; t < kNK; ++t) {
            float2 kf[4], dd = make_float2(0.f, 0.f);
            cvt8<T>(kr[t], kf);
#pragma unroll
            for (int e = 0; e < 4; ++e) dd = f2fma(q[e], kf[e], dd);
            sc[t] = dd.x + dd.y;
        }
#pragma unroll
        for (int o = 1; o < 8; o <<= 1)
#pragma unroll
            for (int t = 0; t < kNK; ++t) sc[t] += __shfl_xor_sync(gmask, sc[t], o);
        float mx = -INFINITY;
#pragma unroll
        for (int t = 0; t < kNK; ++t) {
            if (!live[t]) sc[t] = -INFINITY;
            mx = fmaxf(mx, sc[t]);
        }
        if (mx > m + kLazy || m == -INFINITY) {  // group-uniform
            const float a1 = m == -INFINITY ? 0.f : exp2f(m - mx);
            l *= a1;
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] = make_float2(acc[e].x * a1, acc[e].y * a1);
            m = mx;
        }
#pragma unroll
        for (int t = 0; t < kNK; ++t) {
            const float pt = exp2f(sc[t] - m);  // dead slots: -inf -> 0
            l += pt;
            float2 vf[4];
            cvt8<T>(vr[t], vf);
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[e] = f2fma(make_float2(pt, pt), vf[e], acc[e]);
        }
    }
    // merge the 4 groups (lanes gl, gl+8, gl+16, gl+24 hold the same dims)
#pragma unroll
    for (int o = 8; o < 32 && RPW == 1; o <<= 1) {
        const float m2 = __shfl_xor_sync(0xffffffffu, m, o);
        const float l2 = __shfl_xor_sync(0xffffffffu, l, o);
        const float mn = fmaxf(m, m2);
        const float a1 = (m == -INFINITY) ? 0.f : exp2f(m - mn);
        const float a2 = (m2 == -INFINITY) ? 0.f : exp2f(m2 - mn);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float x2 = __shfl_xor_sync(0xffffffffu, acc[e].x, o);
            const float y2 = __shfl_xor_sync(0xffffffffu, acc[e].y, o);
            acc[e] = make_float2(acc[e].x * a1 + x2 * a2, acc[e].y * a1 + y2 * a2);
        }
        l = l * a1 + l2 * a2;
        m = mn;
    }
    if (RPW == 4 || grp == 0) {
        const float inv = l > 0.f ? 1.f / l : 0.f;  // rows without valid columns stay zero
        T* O = static_cast<T*>(a.o) + b * a.o_sb + hh * a.o_sh + i * a.o_sn + gl * 8;
        uint4 u;
        T* h = reinterpret_cast<T*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            h[2 * e] = DT<T>::from_f(acc[e].x * inv);
            h[2 * e + 1] = DT<T>::from_f(acc[e].y * inv);
        }
        *reinterpret_cast<uint4*>(O) = u;
    }
}

// Generic block executor. DM = max head size handled (template), BN_MAX staged columns.
template <typename T, int DM>
__global__ void attn_bsr_generic_kernel(sf_attn_args a, sf_bsr_dev bsr) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int bm = bsr.block_m, bn = bsr.block_n, d = a.head_size;
    T* Ks = reinterpret_cast<T*>(smem_raw);
    T* Vs = Ks + static_cast<size_t>(bn) * d;
    const int64_t br = blockIdx.x;
    const int64_t bh = blockIdx.y;
    const int64_t b = bh / a.h, hh = bh % a.h;
    const int n = a.seq_len;
    const T* Q = static_cast<const T*>(a.q) + b * a.q_sb + hh * a.q_sh;
    const T* K = static_cast<const T*>(a.k) + b * a.q_sb + hh * a.q_sh;
    const T* V = static_cast<const T*>(a.v) + b * a.q_sb + hh * a.q_sh;
    T* O = static_cast<T*>(a.o) + b * a.o_sb + hh * a.o_sh;
    const int r = threadIdx.x;
    const int64_t i = br * bm + r;
    const bool active = r < bm && i < n;
    const float sl2 = a.scale * 1.4426950408889634f;
    float q[DM], acc[DM];
#pragma unroll
    for (int e = 0; e < DM; ++e) {
        q[e] = (active && e < d) ? DT<T>::to_f(Q[i * a.q_sn + e]) : 0.f;
        acc[e] = 0.f;
    }
    float m = -INFINITY, l = 0.f;
    const int32_t l0 = bsr.load_row_ptr[br], l1 = bsr.load_row_ptr[br + 1];
    for (int32_t lk = l0; lk < l1; ++lk) {
        const int64_t j0 = static_cast<int64_t>(bsr.load_col_idx[lk]) * bn;
        const int cols = static_cast<int>(imin64(bn, n - j0));
        const int32_t tid = bsr.load_tile[lk];
        __syncthreads();
        for (int t = threadIdx.x; t < cols * d; t += blockDim.x) {
            const int c = t / d, e = t - c * d;
            Ks[t] = K[(j0 + c) * a.q_sn + e];
            Vs[t] = V[(j0 + c) * a.q_sn + e];
        }
        __syncthreads();
        if (!active) continue;
        const uint8_t* tile = tid < 0 ? nullptr : bsr.pool + static_cast<int64_t>(tid) * bsr.tile_bytes;
        // tile max over valid columns, then rescale once per tile (attention.hpp:136-157)
        float tmax = -INFINITY;
        for (int c = 0; c < cols; ++c) {
            if (tile) {
                const int bit = r * bn + c;
                if (!((tile[bit >> 3] >> (bit & 7)) & 1)) continue;
            }
            float dot = 0.f;
#pragma unroll
            for (int e = 0; e < DM; ++e)
                if (e < d) dot += q[e] * DT<T>::to_f(Ks[c * d + e]);
            tmax = fmaxf(tmax, dot * sl2);
        }
        const float mn = fmaxf(m, tmax);
        if (mn == -INFINITY) continue;
        const float alpha = exp2f(m - mn);
        l *= alpha;
#pragma unroll
        for (int e = 0; e < DM; ++e) acc[e] *= alpha;
        for (int c = 0; c < cols; ++c) {
            if (tile) {
                const int bit = r * bn + c;
                if (!((tile[bit >> 3] >> (bit & 7)) & 1)) continue;
            }
            float dot = 0.f;
#pragma unroll
            for (int e = 0; e < DM; ++e)
                if (e < d) dot += q[e] * DT<T>::to_f(Ks[c * d + e]);
            const float p = exp2f(dot * sl2 - mn);
            l += p;
#pragma unroll
            for (int e = 0; e < DM; ++e)
                if (e < d) acc[e] += p * DT<T>::to_f(Vs[c * d + e]);
        }
        m = mn;
    }
    if (active) {
        const float inv = l > 0.f ? 1.f / l : 0.f;
#pragma unroll
        for (int e = 0; e < DM; ++e)
            if (e < d) O[i * a.o_sn + e] = DT<T>::from_f(acc[e] * inv);
    }
}

template <typename T, int DPL, bool VEC = false>
sf_status launch_rowwise(const sf_attn_args& a, const sf_csr_dev& c, cudaStream_t st) {
    const int64_t warps = static_cast<int64_t>(a.bs) * a.h * a.seq_len;
    attn_rowwise_kernel<T, DPL, VEC><<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, st>>>(a, c.row_ptr,
                                                                                                  c.col_idx);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

template <typename T>
sf_status rowwise_dispatch(const sf_attn_args& a, const sf_csr_dev& c, cudaStream_t st) {
    const int d = a.head_size;
    const bool vec = (d % 64 == 0) && (a.q_sn % 8 == 0) && (a.q_sb % 8 == 0) && (a.q_sh % 8 == 0) &&
                     (reinterpret_cast<uintptr_t>(a.k) % 16 == 0) && (reinterpret_cast<uintptr_t>(a.v) % 16 == 0);
    if (d == 64 && vec && a.o_sn % 8 == 0 && reinterpret_cast<uintptr_t>(a.o) % 16 == 0 &&
        reinterpret_cast<uintptr_t>(a.q) % 16 == 0) {
        const int64_t rows = static_cast<int64_t>(a.bs) * a.h * a.seq_len;
        // short rows (<= 32 keys on average): one 8-lane group per row
        if (c.nnz <= 32ll * a.seq_len) {
            const int64_t warps = ceil_div(rows, 4);
            attn_rowwise64_kernel<T, 4><<<static_cast<unsigned>(ceil_div(warps * 32, 256)), 256, 0, st>>>(a, c.row_ptr,
                                                                                                      c.col_idx);
        } else {
            attn_rowwise64_kernel<T, 1><<<static_cast<unsigned>(ceil_div(rows * 32, 256)), 256, 0, st>>>(a, c.row_ptr,
                                                                                                     c.col_idx);
        }
        SF_LAUNCH_CHECK();
        return SF_OK;
    }
    if (d == 64 && vec) return launch_rowwise<T, 8, true>(a, c, st);
    if (d == 128 && vec) return launch_rowwise<T, 16, true>(a, c, st);
    if (d <= 8) return launch_rowwise<T, 1>(a, c, st);
    if (d <= 16) return launch_rowwise<T, 2>(a, c, st);
    if (d <= 32) return launch_rowwise<T, 4>(a, c, st);
    if (d <= 64) return launch_rowwise<T, 8>(a, c, st);
    if (d <= 128) return launch_rowwise<T, 16>(a, c, st);
    return fail(SF_SHAPE_ERROR, "row-wise kernel supports head_size <= 128");
}

template <typename T, int DM>
sf_status launch_generic(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st) {
    const int threads = static_cast<int>(imax64(32, ceil_div(b.block_m, 32) * 32));
    if (threads > 1024) return fail(SF_PLAN_ERROR, "generic block kernel supports block_m <= 1024");
    const size_t smem = static_cast<size_t>(b.block_n) * a.head_size * sizeof(T) * 2;
    if (smem > 200 * 1024) return fail(SF_PLAN_ERROR, "tile too large for shared memory");
    auto k = attn_bsr_generic_kernel<T, DM>;
    if (smem > 48 * 1024) SF_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid(b.n_rows, static_cast<unsigned>(a.bs) * a.h);
    k<<<grid, threads, smem, st>>>(a, b);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

template <typename T>
sf_status generic_dispatch(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st) {
    const int d = a.head_size;
    if (d <= 8) return launch_generic<T, 8>(a, b, st);
    if (d <= 16) return launch_generic<T, 16>(a, b, st);
    if (d <= 32) return launch_generic<T, 32>(a, b, st);
    if (d <= 64) return launch_generic<T, 64>(a, b, st);
    if (d <= 128) return launch_generic<T, 128>(a, b, st);
    return fail(SF_SHAPE_ERROR, "block kernel supports head_size <= 128");
}

}  // namespace

sf_status check_attn_args(const sf_attn_args& a) {
    if (a.bs < 1 || a.h < 1 || a.seq_len < 1 || a.head_size < 1)
        return fail(SF_SHAPE_ERROR, "empty attention input");                    // tensor.hpp:47
    if (!a.q || !a.k || !a.v || !a.o) return fail(SF_INVALID_PARAMETER, "null tensor pointer");
    if (a.dtype != SF_F16 && a.dtype != SF_BF16) return fail(SF_INVALID_PARAMETER, "dtype must be f16/bf16");
    // 0 selects the reference's 1/sqrt(head_size) (attention.hpp:77); the tcgen05 softmax takes the
    // row max of the raw scores, which commutes with a positive scale only
    if (!(a.scale >= 0.f) || !std::isfinite(a.scale))
        return fail(SF_INVALID_PARAMETER, "scale must be finite and >= 0 (0 = 1/sqrt(head_size))");
    return SF_OK;
}

sf_status attn_generic(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st) {
    return a.dtype == SF_F16 ? generic_dispatch<__half>(a, b, st) : generic_dispatch<__nv_bfloat16>(a, b, st);
}

}  // namespace sf

using namespace sf;

extern "C" sf_status sf_mha_rowwise(const sf_attn_args* args, const sf_csr_dev* csr, void* stream) {
    if (!args || !csr) return fail(SF_INVALID_PARAMETER, "null argument");
    SF_TRY(check_attn_args(*args));
    if (csr->seq_len != args->seq_len)
        return fail(SF_SHAPE_ERROR, "rowwise mask seq_len differs from input");   // attention.hpp:179
    sf_attn_args a = *args;
    if (a.scale == 0.f) a.scale = 1.0f / sqrtf(static_cast<float>(a.head_size));
    cudaStream_t st = as_stream(stream);
    return a.dtype == SF_F16 ? rowwise_dispatch<__half>(a, *csr, st) : rowwise_dispatch<__nv_bfloat16>(a, *csr, st);
}
