// gemm_tc.cu — the CiMi fused template (backend.hpp:240-264) as one sm_100a kernel:
//   out[M x N] = epilogue( X[M x K] . W[N x K]^T )
//   epilogue = +bias[N] -> GELU/ReLU -> +aux[M x N] (residual Add) -> LayerNorm over the row
// (op semantics: backend.hpp:111-167; order = the chain's MI order after the Gemm).
//
// Structure (one 128 x BN output tile per CTA, 256 threads):
//   warp 0      TMA producer: X and W tiles (BK = 64 fp16 = one 128-byte swizzle row) into a
//               STAGES-deep smem ring, mbarrier complete_tx.
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma (M=128, N=BN, K=16) into a
//               TMEM fp32 accumulator; tcgen05.commit frees each smem stage.
//   warp 2      TMEM allocator.
//   warps 4-7   epilogue: tcgen05.ld rows of the accumulator (warp w owns TMEM lanes
//               32*(w%4)..+31 = tile rows), apply the MI ops in registers, store fp16.
// LayerNorm needs whole rows: the N/BN CTAs of a row block form a thread-block cluster; each CTA
// stages its x = acc+bias+aux slice as fp32 in the (now idle) pipeline smem, and the per-row
// partial sums Σx and Σ(x-mean)² are exchanged through distributed shared memory (two-pass,
// biased variance, eps 1e-5, exactly the reference's order of operations).
#include <algorithm>
#include <cstring>

#include "tc.cuh"

namespace sf {
namespace {

constexpr int BM = 128, BK = 64;
constexpr int kThreads = 256;
constexpr float kLnEps = 1e-5f;  // backend.hpp:111

struct GemmParams {
    CUtensorMap ta;  // X: rows M, cols K
    CUtensorMap tb;  // W: rows N, cols K
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
};

template <int BN>
struct Cfg {
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int XS_STRIDE = BN + 4;  // fp32 staging row stride (bank-conflict free float4)
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 /*align*/ + 512 /*barriers*/ + 2 * BM * 4;
    static_assert(BM * XS_STRIDE * 4 <= STAGES * (A_BYTES + B_BYTES), "LN staging must fit the ring");
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

__device__ __forceinline__ float act_fn(float x, int act) {
    if (act == SF_ACT_GELU) return 0.5f * x * (1.0f + erff(x * 0.7071067811865475f));  // backend.hpp:128-131
    if (act == SF_ACT_RELU) return x > 0.f ? x : 0.f;                                  // backend.hpp:132-134
    return x;
}

// 32 consecutive values of row `row`, columns [col, col+32): bias -> act -> +aux.
template <typename T>
__device__ __forceinline__ void epi_chunk(const GemmParams& p, const uint32_t (&r)[32], int64_t row, int64_t col,
                                          float (&x)[32]) {
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

template <typename T, int BN, bool LN>
__global__ void __launch_bounds__(kThreads, 1) gemm_fused_kernel(const __grid_constant__ GemmParams p) {
    using C = Cfg<BN>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + C::STAGES * C::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
    uint64_t* empty = full + C::STAGES;
    uint64_t* accum_full = empty + C::STAGES;
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(accum_full + 1);
    float* red_sum = reinterpret_cast<float*>(tmem_ptr + 4);
    float* red_sq = red_sum + BM;

    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const int n0 = blockIdx.x * BN;
    const int m0 = blockIdx.y * BM;
    const int nk = (p.K + BK - 1) / BK;

    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&p.ta);
        tc::prefetch_tmap(&p.tb);
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        tc::mbar_init(accum_full, 1);
        tc::fence_barrier_init();
    }
    if (warp == 2) tc::tmem_alloc<BN>(tmem_ptr);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;

    if (warp == 0) {
        if (tc::elect_one()) {
            const uint64_t pol_a = tc::policy_evict_first();  // X tile rows are re-read by N/BN CTAs only
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nk; ++kb) {
                tc::mbar_wait(&empty[s], ph ^ 1);
                tc::mbar_expect_tx(&full[s], C::A_BYTES + C::B_BYTES);
                tc::tma_load_2d_hint(sA + s * C::A_BYTES, &p.ta, &full[s], kb * BK, m0, pol_a);
                tc::tma_load_2d(sB + s * C::B_BYTES, &p.tb, &full[s], kb * BK, n0);
                if (++s == C::STAGES) { s = 0; ph ^= 1; }
            }
        }
    } else if (warp == 1) {
        constexpr uint32_t idesc = tc::idesc_f16(BM, BN, sizeof(T) == 2 && !std::is_same<T, __half>::value, 0, 0);
        if (tc::elect_one()) {
            int s = 0;
            uint32_t ph = 0;
            for (int kb = 0; kb < nk; ++kb) {
                tc::mbar_wait(&full[s], ph);
                tc::fence_after_sync();
                const uint32_t a0 = tc::smem_u32(sA + s * C::A_BYTES);
                const uint32_t b0 = tc::smem_u32(sB + s * C::B_BYTES);
#pragma unroll
                for (int k = 0; k < BK / 16; ++k)
                    tc::mma_f16_ss(tmem, tc::sdesc_sw128(a0 + 32 * k), tc::sdesc_sw128(b0 + 32 * k), idesc,
                                   (kb | k) != 0);
                tc::mma_commit(&empty[s]);
                if (++s == C::STAGES) { s = 0; ph ^= 1; }
            }
            tc::mma_commit(accum_full);
        }
    } else if (warp >= 4) {
        const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
        const int r_local = static_cast<int>(q * 32 + lane);
        const int64_t row = m0 + r_local;
        const bool row_ok = row < p.M;
        const uint32_t taddr = tmem + ((q * 32) << 16);
        tc::mbar_wait(accum_full, 0);
        tc::fence_after_sync();
        uint32_t r[32];
        float x[32];
        if constexpr (!LN) {
            for (int c = 0; c < BN / 32; ++c) {
                tc::tmem_ld32(taddr + c * 32, r);
                tc::tmem_ld_wait();
                const int64_t col = n0 + c * 32;
                if (!row_ok || col >= p.N) continue;
                epi_chunk<T>(p, r, row, col, x);
                store_chunk<T>(p.out, p.ldout, row, col, x);
            }
        } else {
            float* xs = reinterpret_cast<float*>(smem) + r_local * C::XS_STRIDE;  // reuse the ring
            float sum = 0.f;
            for (int c = 0; c < BN / 32; ++c) {
                tc::tmem_ld32(taddr + c * 32, r);
                tc::tmem_ld_wait();
                const int64_t col = n0 + c * 32;
                if (row_ok) epi_chunk<T>(p, r, row, col, x);
                else
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = 0.f;
#pragma unroll
                for (int j = 0; j < 32; j += 4) {
                    *reinterpret_cast<float4*>(xs + c * 32 + j) = make_float4(x[j], x[j + 1], x[j + 2], x[j + 3]);
                    sum += (x[j] + x[j + 1]) + (x[j + 2] + x[j + 3]);
                }
            }
            red_sum[r_local] = sum;
        }
    }
    if constexpr (LN) {
        // Cross-CTA row reductions. Every thread of every CTA in the cluster takes part in the
        // three cluster barriers (non-epilogue warps simply pass through).
        const uint32_t nct = gridDim.x;  // cluster spans the full row: cluster dims == (N/BN, 1, 1)
        tc::cluster_sync_all();
        float mean = 0.f, inv = 0.f;
        const bool epi = warp >= 4;
        const int r_local = static_cast<int>((warp & 3) * 32 + lane);
        float* xs = reinterpret_cast<float*>(smem) + r_local * C::XS_STRIDE;
        if (epi) {
            float tot = 0.f;
            for (uint32_t c = 0; c < nct; ++c) tot += tc::ld_dsmem_f32(&red_sum[r_local], c);
            mean = tot / static_cast<float>(p.N);
            float sq = 0.f;
            for (int j = 0; j < BN; j += 4) {
                const float4 v = *reinterpret_cast<const float4*>(xs + j);
                const float d0 = v.x - mean, d1 = v.y - mean, d2 = v.z - mean, d3 = v.w - mean;
                sq += (d0 * d0 + d1 * d1) + (d2 * d2 + d3 * d3);
            }
            red_sq[r_local] = sq;
        }
        tc::cluster_sync_all();
        if (epi) {
            float tot = 0.f;
            for (uint32_t c = 0; c < nct; ++c) tot += tc::ld_dsmem_f32(&red_sq[r_local], c);
            inv = 1.0f / sqrtf(tot / static_cast<float>(p.N) + kLnEps);
            const int64_t row = static_cast<int64_t>(blockIdx.y) * BM + r_local;
            if (row < p.M) {
                float y[32], xx[32];
                for (int c = 0; c < BN / 32; ++c) {
                    const int64_t col = n0 + c * 32;
#pragma unroll
                    for (int j = 0; j < 32; j += 4) {
                        const float4 v = *reinterpret_cast<const float4*>(xs + c * 32 + j);
                        xx[j] = v.x; xx[j + 1] = v.y; xx[j + 2] = v.z; xx[j + 3] = v.w;
                    }
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        y[j] = (xx[j] - mean) * inv * __ldg(p.gamma + col + j) + __ldg(p.beta + col + j);
                    store_chunk<T>(p.out, p.ldout, row, col, y);
                    if (p.out_pre_ln) store_chunk<T>(p.out_pre_ln, p.ldout, row, col, xx);
                }
            }
        }
        tc::cluster_sync_all();  // no CTA leaves while a peer may still read its partials
    }
    tc::fence_before_sync();
    __syncthreads();
    if (warp == 2) tc::tmem_dealloc<BN>(tmem);
}

template <typename T, int BN, bool LN>
sf_status launch_gemm(const sf_gemm_args& a, cudaStream_t st) {
    using Cf = Cfg<BN>;
    GemmParams p{};
    const bool bf = std::is_same<T, __nv_bfloat16>::value;
    SF_TRY(make_tmap_2d(&p.ta, a.x, a.M, a.K, a.ldx, BK, BM, bf));
    SF_TRY(make_tmap_2d(&p.tb, a.w, a.N, a.K, a.ldw, BK, BN, bf));
    p.M = a.M; p.N = a.N; p.K = a.K;
    p.out = a.out; p.ldout = a.ldout;
    p.bias = static_cast<const float*>(a.epi.bias);
    p.act = a.epi.act;
    p.aux = a.epi.aux; p.ldaux = a.epi.ldaux;
    p.gamma = static_cast<const float*>(a.epi.ln_gamma);
    p.beta = static_cast<const float*>(a.epi.ln_beta);
    p.out_pre_ln = a.epi.out_pre_ln;
    auto kern = gemm_fused_kernel<T, BN, LN>;
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(ceil_div(a.N, BN)), static_cast<unsigned>(ceil_div(a.M, BM)));
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = Cf::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    if (LN) {
        if (a.N / BN > 8) SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(a.N / BN);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    }
    SF_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    SF_LAUNCH_CHECK();
    return SF_OK;
}

template <typename T>
sf_status gemm_dispatch(const sf_gemm_args& a, cudaStream_t st) {
    const bool ln = a.epi.ln_gamma != nullptr;
    // widest tile that divides N (LN needs whole rows inside one <= 16-CTA cluster)
    if (ln) {
        if (a.N % 256 == 0 && a.N / 256 <= 8) return launch_gemm<T, 256, true>(a, st);
        if (a.N % 128 == 0 && a.N / 128 <= 8) return launch_gemm<T, 128, true>(a, st);
        return fail(SF_SHAPE_ERROR, "fused LayerNorm needs N % 128 == 0 and N <= 2048");
    }
    if (a.N % 256 == 0) return launch_gemm<T, 256, false>(a, st);
    return launch_gemm<T, 128, false>(a, st);
}

}  // namespace

sf_status make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                       uint32_t box_cols, uint32_t box_rows, bool bf16, bool swizzle128) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        SF_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {row_stride_elems * 2};
    const cuuint32_t box[2] = {box_cols, box_rows};
    const cuuint32_t estr[2] = {1, 1};
    CUresult r = encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled failed: " + std::to_string(int(r)));
    return SF_OK;
}

}  // namespace sf

using namespace sf;

extern "C" sf_status sf_gemm_fused(const sf_gemm_args* a, void* stream) {
    if (!a) return fail(SF_INVALID_PARAMETER, "null argument");
    if (a->M < 1 || a->N < 1 || a->K < 1) return fail(SF_SHAPE_ERROR, "empty GEMM");
    if (a->K % 8 || a->ldx % 8 || a->ldw % 8) return fail(SF_SHAPE_ERROR, "K and leading dims must be multiples of 8");
    if (a->N % 32 || a->ldout % 8 || (a->epi.aux && a->epi.ldaux % 8))
        return fail(SF_SHAPE_ERROR, "N must be a multiple of 32, ldout/ldaux multiples of 8");
    if ((reinterpret_cast<uintptr_t>(a->x) | reinterpret_cast<uintptr_t>(a->w) | reinterpret_cast<uintptr_t>(a->out)) & 15)
        return fail(SF_INVALID_PARAMETER, "GEMM operands must be 16-byte aligned");
    if (a->epi.ln_gamma && !a->epi.ln_beta) return fail(SF_INVALID_PARAMETER, "LayerNorm needs gamma and beta");
    cudaStream_t st = as_stream(stream);
    if (a->dtype == SF_F16) return gemm_dispatch<__half>(*a, st);
    if (a->dtype == SF_BF16) return gemm_dispatch<__nv_bfloat16>(*a, st);
    return fail(SF_INVALID_PARAMETER, "dtype must be f16/bf16");
}
