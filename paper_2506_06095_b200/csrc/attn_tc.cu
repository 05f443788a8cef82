// attn_tc.cu — block-wise masked attention on tcgen05 / TMEM / TMA (sm_100a).
// Replaces block_sparse_sdpa (attention.hpp:71-172) for BSR tiles of block_m = 128 query rows
// and block_n in {16, 32, 64} key columns, head_size 64, fp16/bf16.
//
// One CTA per (128-row block, b*h slice); 192 threads, 2 CTAs per SM:
//   warp 0     TMA producer. Q tile once (128 x 64, 128B-swizzled), then per step the K and V rows
//              of G = 64/block_n load-list column blocks, GATHERED into one contiguous 64-key
//              stage (a 4-D tensor map over (d, n, h, b) reads Q/K/V in any (b,h,i) stride layout,
//              including the fused-QKV activation, in place).
//   warp 1     TMEM allocator + MMA issuer (one elected thread):
//                S_j = Q K_j^T     tcgen05.mma M=128 N=64 K=16 x4  -> TMEM S[j%2] (fp32)
//                O_j = P_j V_j     tcgen05.mma M=128 N=64 K=16 x4  -> TMEM O[j%2] (fp32), V as
//                                  an MN-major B operand straight from the TMA stage
//   warps 2-5  softmax / correction / epilogue, one thread per query row (TMEM lane):
//                tcgen05.ld S_j row; apply the tile's mask bits (full tile -> all ones, part tile
//                -> its pool bits; columns past seq_len are 0 bits in edge tiles) as -inf;
//                online softmax in the log2 domain; P_j (fp16) written 128B-swizzled to smem as
//                the A operand of the P.V MMA; O_j folded into a register accumulator
//                acc = acc * alpha_j + O_j one step later (so softmax j+1 overlaps P_j V_j).
// Empty tiles are never touched (only the BSR load set is iterated, attention.hpp:104-109);
// rows whose running max stays -inf produce exact zeros (attention.hpp:160-166).
#include <algorithm>

#include "tc.cuh"

namespace sf {
namespace {

constexpr int kBM = 128, kD = 64, kNS = 64;  // query rows, head size, keys per step
constexpr int kThreads = 192;
constexpr int kStages = 3;
constexpr int kMaxLoads = 1024;  // load-list entries per row block staged in smem
constexpr int kQBytes = kBM * kD * 2;
constexpr int kKVBytes = kNS * kD * 2;  // one 64-key stage of K (or V)
constexpr int kPBytes = kBM * kNS * 2;
constexpr int kSmem = 1024 + kQBytes + 2 * kStages * kKVBytes + 2 * kPBytes + kMaxLoads * 8 + 256;

struct AttnParams {
    CUtensorMap tq, tk, tv;  // 4-D (d, n, h, b) maps; boxes {64,128,1,1} / {64,bn,1,1}
    int32_t n, h, bn, G;
    const int32_t* load_row_ptr;
    const int32_t* load_col_idx;
    const int32_t* load_tile;
    const uint8_t* pool;
    int32_t tile_bytes;
    void* o;
    int64_t o_sb, o_sh, o_sn;
    float scale_log2;
};

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

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

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 2) attn_tc_kernel(const __grid_constant__ AttnParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sQ = sm;
    unsigned char* sK = sQ + kQBytes;
    unsigned char* sV = sK + kStages * kKVBytes;
    unsigned char* sP = sV + kStages * kKVBytes;
    int32_t* s_col = reinterpret_cast<int32_t*>(sP + 2 * kPBytes);
    int32_t* s_tile = s_col + kMaxLoads;
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_tile + kMaxLoads);
    uint64_t* q_full = bars;
    uint64_t* kv_full = bars + 1;
    uint64_t* kv_empty = kv_full + kStages;
    uint64_t* s_full = kv_empty + kStages;  // [2]
    uint64_t* p_full = s_full + 2;          // [2]
    uint64_t* o_full = p_full + 2;          // [2]
    uint64_t* o_free = o_full + 2;          // [2]
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(o_free + 2);

    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const int br = blockIdx.x;
    const int bh = blockIdx.y;
    const int b = bh / p.h, hh = bh % p.h;
    const int l0 = p.load_row_ptr[br];
    const int L = p.load_row_ptr[br + 1] - l0;
    const int nsteps = (L + p.G - 1) / p.G;

    for (int i = threadIdx.x; i < L; i += kThreads) {
        s_col[i] = p.load_col_idx[l0 + i];
        s_tile[i] = p.load_tile[l0 + i];
    }
    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&p.tq);
        tc::prefetch_tmap(&p.tk);
        tc::prefetch_tmap(&p.tv);
        tc::mbar_init(q_full, 1);
        for (int s = 0; s < kStages; ++s) {
            tc::mbar_init(&kv_full[s], 1);
            tc::mbar_init(&kv_empty[s], 1);
        }
        for (int s = 0; s < 2; ++s) {
            tc::mbar_init(&s_full[s], 1);
            tc::mbar_init(&p_full[s], 128);
            tc::mbar_init(&o_full[s], 1);
            tc::mbar_init(&o_free[s], 128);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<256>(tmem_ptr);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;  // S[0] @ +0, S[1] @ +64, O[0] @ +128, O[1] @ +192

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (tc::elect_one() && nsteps > 0) {
            tc::mbar_expect_tx(q_full, kQBytes);
            tma_load_4d(sQ, &p.tq, q_full, 0, br * kBM, hh, b);
            const int chunk = p.bn * kD * 2;
            int s = 0;
            uint32_t ph = 0;
            for (int j = 0; j < nsteps; ++j) {
                tc::mbar_wait(&kv_empty[s], ph ^ 1);
                tc::mbar_expect_tx(&kv_full[s], 2 * kKVBytes);
                for (int g = 0; g < p.G; ++g) {
                    const int e = j * p.G + g;
                    const int col = (e < L ? s_col[e] : s_col[0]) * p.bn;  // pad: a valid, fully masked block
                    tma_load_4d(sK + s * kKVBytes + g * chunk, &p.tk, &kv_full[s], 0, col, hh, b);
                    tma_load_4d(sV + s * kKVBytes + g * chunk, &p.tv, &kv_full[s], 0, col, hh, b);
                }
                if (++s == kStages) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        constexpr bool bf = std::is_same<T, __nv_bfloat16>::value;
        constexpr uint32_t idesc_s = tc::idesc_f16(kBM, kNS, bf, 0, 0);  // Q (K-major) x K (K-major)
        constexpr uint32_t idesc_o = tc::idesc_f16(kBM, kD, bf, 0, 1);   // P (K-major) x V (MN-major)
        if (tc::elect_one() && nsteps > 0) {
            const uint32_t q0 = tc::smem_u32(sQ);
            tc::mbar_wait(q_full, 0);
            auto issue_s = [&](int j) {
                const int s = j % kStages;
                tc::mbar_wait(&kv_full[s], (j / kStages) & 1);
                tc::fence_after_sync();
                const uint32_t k0 = tc::smem_u32(sK + s * kKVBytes);
#pragma unroll
                for (int k = 0; k < kD / 16; ++k)
                    tc::mma_f16_ss(tmem + (j & 1) * 64, tc::sdesc_sw128(q0 + 32 * k), tc::sdesc_sw128(k0 + 32 * k),
                                   idesc_s, k != 0);
                tc::mma_commit(&s_full[j & 1]);
            };
            issue_s(0);
            if (nsteps > 1) issue_s(1);
            for (int j = 0; j < nsteps; ++j) {
                const int s = j % kStages;
                tc::mbar_wait(&p_full[j & 1], (j >> 1) & 1);  // P_j in smem; S[j&1] consumed
                if (j >= 2) tc::mbar_wait(&o_free[j & 1], ((j - 2) >> 1) & 1);  // O_{j-2} folded
                tc::fence_after_sync();
                const uint32_t pa = tc::smem_u32(sP + (j & 1) * kPBytes);
                const uint32_t v0 = tc::smem_u32(sV + s * kKVBytes);
#pragma unroll
                for (int k = 0; k < kNS / 16; ++k)
                    tc::mma_f16_ss(tmem + 128 + (j & 1) * 64, tc::sdesc_sw128(pa + 32 * k),
                                   tc::sdesc_sw128_mn(v0 + 2048 * k), idesc_o, k != 0);
                tc::mma_commit(&o_full[j & 1]);
                tc::mma_commit(&kv_empty[s]);
                if (j + 2 < nsteps) issue_s(j + 2);
            }
        }
    } else {
        // ------------------------------------------------------------------ softmax / epilogue
        const uint32_t q = warp & 3;
        const int r = static_cast<int>(q * 32 + lane);
        const uint32_t trow = tmem + ((q * 32) << 16);
        const int bn = p.bn;
        const uint32_t full_bits = bn >= 32 ? 0xffffffffu : ((1u << bn) - 1u);
        float acc[kD];
#pragma unroll
        for (int e = 0; e < kD; ++e) acc[e] = 0.f;
        float m = -INFINITY, l = 0.f, alpha_prev = 1.f;
        unsigned char* prow_base = sP + r * 128;
        const int rsw = r & 7;
        for (int j = 0; j < nsteps; ++j) {
            // ---- mask bits of this row for the 64 columns of step j
            uint64_t bits = 0;
            for (int g = 0; g < p.G; ++g) {
                const int e = j * p.G + g;
                uint64_t gb = 0;
                if (e < L) {
                    const int t = s_tile[e];
                    if (t < 0) {
                        gb = bn == 64 ? ~0ull : full_bits;
                    } else {
                        const uint8_t* tp = p.pool + static_cast<int64_t>(t) * p.tile_bytes + r * (bn >> 3);
                        if (bn == 16) gb = *reinterpret_cast<const uint16_t*>(tp);
                        else if (bn == 32) gb = *reinterpret_cast<const uint32_t*>(tp);
                        else gb = *reinterpret_cast<const uint64_t*>(tp);
                    }
                }
                bits |= gb << (g * bn);
            }
            // ---- S_j row from TMEM
            tc::mbar_wait(&s_full[j & 1], (j >> 1) & 1);
            tc::fence_after_sync();
            uint32_t lo[32], hi[32];
            tc::tmem_ld32(trow + (j & 1) * 64, lo);
            tc::tmem_ld32(trow + (j & 1) * 64 + 32, hi);
            tc::tmem_ld_wait();
            float sr[64];
            float mx = -INFINITY;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                sr[c] = ((bits >> c) & 1ull) ? __uint_as_float(lo[c]) * p.scale_log2 : -INFINITY;
                sr[c + 32] = ((bits >> (c + 32)) & 1ull) ? __uint_as_float(hi[c]) * p.scale_log2 : -INFINITY;
                mx = fmaxf(mx, fmaxf(sr[c], sr[c + 32]));
            }
            const float mn = fmaxf(m, mx);
            float alpha = 1.f;
            float rs = 0.f;
            uint32_t pk[32];
            if (mn == -INFINITY) {
#pragma unroll
                for (int c = 0; c < 32; ++c) pk[c] = 0u;
            } else {
                alpha = ex2(m - mn);  // m = -inf -> 0
#pragma unroll
                for (int c = 0; c < 64; c += 2) {
                    const float p0 = ex2(sr[c] - mn);
                    const float p1 = ex2(sr[c + 1] - mn);
                    rs += p0 + p1;
                    pk[c >> 1] = pack2<T>(p0, p1);
                }
                m = mn;
            }
            l = l * alpha + rs;
            // P_j row -> smem, 128B-swizzled K-major A operand (row r: 8 chunks of 16 B)
            unsigned char* prow = prow_base + (j & 1) * kPBytes;
#pragma unroll
            for (int c = 0; c < 8; ++c)
                *reinterpret_cast<uint4*>(prow + ((c ^ rsw) << 4)) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
            tc::fence_proxy_async();
            tc::fence_before_sync();
            tc::mbar_arrive(&p_full[j & 1]);
            // ---- fold O_{j-1} (P_{j-1} V_{j-1}) into the register accumulator
            if (j >= 1) {
                const int jp = j - 1;
                tc::mbar_wait(&o_full[jp & 1], (jp >> 1) & 1);
                tc::fence_after_sync();
                uint32_t ov[32];
#pragma unroll
                for (int h2 = 0; h2 < 2; ++h2) {
                    tc::tmem_ld32(trow + 128 + (jp & 1) * 64 + h2 * 32, ov);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int e = 0; e < 32; ++e) acc[h2 * 32 + e] = acc[h2 * 32 + e] * alpha_prev + __uint_as_float(ov[e]);
                }
                tc::fence_before_sync();
                tc::mbar_arrive(&o_free[jp & 1]);
            }
            alpha_prev = alpha;
        }
        if (nsteps > 0) {
            const int jp = nsteps - 1;
            tc::mbar_wait(&o_full[jp & 1], (jp >> 1) & 1);
            tc::fence_after_sync();
            uint32_t ov[32];
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                tc::tmem_ld32(trow + 128 + (jp & 1) * 64 + h2 * 32, ov);
                tc::tmem_ld_wait();
#pragma unroll
                for (int e = 0; e < 32; ++e) acc[h2 * 32 + e] = acc[h2 * 32 + e] * alpha_prev + __uint_as_float(ov[e]);
            }
        }
        // ---- epilogue: out = acc / l; rows without a valid column stay exactly zero
        const int64_t i = static_cast<int64_t>(br) * kBM + r;
        if (i < p.n) {
            const float inv = l > 0.f ? 1.f / l : 0.f;
            uint4* dst = reinterpret_cast<uint4*>(static_cast<T*>(p.o) + b * p.o_sb + hh * p.o_sh + i * p.o_sn);
#pragma unroll
            for (int c = 0; c < 8; ++c)
                dst[c] = make_uint4(pack2<T>(acc[8 * c] * inv, acc[8 * c + 1] * inv),
                                    pack2<T>(acc[8 * c + 2] * inv, acc[8 * c + 3] * inv),
                                    pack2<T>(acc[8 * c + 4] * inv, acc[8 * c + 5] * inv),
                                    pack2<T>(acc[8 * c + 6] * inv, acc[8 * c + 7] * inv));
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc<256>(tmem);
}

// 4-D map over (d, n, h, b) with element strides (1, sn, sh, sb); box {64, rows, 1, 1}, SW128.
sf_status make_tmap_4d(CUtensorMap* map, const void* base, int n, int h, int bs, int64_t sn, int64_t sh, int64_t sb,
                       uint32_t box_rows, bool bf16) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        SF_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(kD), static_cast<cuuint64_t>(n), static_cast<cuuint64_t>(h),
                                static_cast<cuuint64_t>(bs)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(sn * 2), static_cast<cuuint64_t>(sh * 2),
                                   static_cast<cuuint64_t>(sb * 2)};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(kD), box_rows, 1, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled (4d) failed: " + std::to_string(int(r)));
    return SF_OK;
}

}  // namespace

sf_status attn_tc(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st, bool probe_only) {
    const bool shape_ok = b.block_m == kBM && (b.block_n == 16 || b.block_n == 32 || b.block_n == 64) &&
                          a.head_size == kD && b.n_cols <= kMaxLoads;
    const bool layout_ok = a.q_sn % 8 == 0 && a.q_sh % 8 == 0 && a.q_sb % 8 == 0 && a.o_sn % 8 == 0 &&
                           a.o_sh % 8 == 0 && a.o_sb % 8 == 0 &&
                           ((reinterpret_cast<uintptr_t>(a.q) | reinterpret_cast<uintptr_t>(a.k) |
                             reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.o)) & 15) == 0;
    if (!shape_ok || !layout_ok)
        return fail(SF_PLAN_ERROR, "tcgen05 attention needs block_m 128, block_n 16/32/64, head_size 64, "
                                   "16-byte aligned strides");
    if (probe_only) return SF_OK;
    AttnParams p{};
    const bool bf = a.dtype == SF_BF16;
    SF_TRY(make_tmap_4d(&p.tq, a.q, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, kBM, bf));
    SF_TRY(make_tmap_4d(&p.tk, a.k, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_n, bf));
    SF_TRY(make_tmap_4d(&p.tv, a.v, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_n, bf));
    p.n = a.seq_len;
    p.h = a.h;
    p.bn = b.block_n;
    p.G = kNS / b.block_n;
    p.load_row_ptr = b.load_row_ptr;
    p.load_col_idx = b.load_col_idx;
    p.load_tile = b.load_tile;
    p.pool = b.pool;
    p.tile_bytes = b.tile_bytes;
    p.o = a.o;
    p.o_sb = a.o_sb;
    p.o_sh = a.o_sh;
    p.o_sn = a.o_sn;
    p.scale_log2 = a.scale * 1.4426950408889634f;
    auto kern = bf ? attn_tc_kernel<__nv_bfloat16> : attn_tc_kernel<__half>;
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    dim3 grid(b.n_rows, static_cast<unsigned>(a.bs) * a.h);
    kern<<<grid, kThreads, kSmem, st>>>(p);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

}  // namespace sf
