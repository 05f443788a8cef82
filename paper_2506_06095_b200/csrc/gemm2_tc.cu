// gemm2_tc.cu — the CiMi fused template (backend.hpp:240-264) on two-SM CTA pairs.
//
// Why pairs: a single CTA computing a 128 x 256 tile pulls 16 KB of X and 32 KB of W per
// 64-deep k-block (87 FLOP/B); at ~148 SMs that saturates the L2 (LTS) throughput cap well
// before the tensor cores (measured ~900 TFLOP/s ceiling, independent of TMA multicast at
// cluster size 2). A tcgen05 cta_group::2 MMA computes a 256 x 256 tile on two SMs of one TPC:
// each CTA stages its own 128 rows of X and HALF (128 rows) of W, so each SM pulls 32 KB per
// k-block for the same 128 x 256 of output (128 FLOP/B).
//
//   warp 0 (both CTAs)  TMA producer: X rows [128*(2mp+px), +128), W rows [256nb + 128px, +128)
//                       into a 6-deep ring; completion bytes land on the LEADER's full barrier.
//   warp 1 (leader)     MMA issuer: M=256, N=256, K=16 x 4 per stage; commits multicast to both
//                       CTAs (free the stage / hand the accumulator to both epilogues).
//   warp 1 (both)       TMEM allocation (cta_group::2: same 512 columns in both CTAs).
//   warps 4..           epilogue on this CTA's 128 accumulator lanes; per-warp release of the
//                       accumulator to the leader's tempty barrier (remote arrive from the peer).
// LayerNorm: the cluster is (2 x nct) CTAs — nct pairs along the row — and each CTA exchanges
// per-row partial sums with the nct CTAs holding the same rows (ranks px + 2y), as in gemm_tc.cu.
#include <algorithm>
#include <cstring>

#include "epilogue.cuh"

namespace sf {
namespace {

constexpr int BN2 = 256;  // pair tile N; each CTA holds BN2/2 rows of W
constexpr int kMaxNct = 4;  // LN cluster 2 x nct <= 8 CTAs (portable cluster size)

template <bool LN>
struct Cfg2 {
    static constexpr int STAGES = 6;
    static constexpr int EPI_WARPS = LN ? 8 : 16;
    static constexpr int THREADS = 128 + 32 * EPI_WARPS;
    static constexpr int A_BYTES = BM * BK * 2;         // 16 KB
    static constexpr int B_BYTES = (BN2 / 2) * BK * 2;  // 16 KB
    static constexpr int RED_FLOATS = LN ? 2 * 2 * kMaxNct * 2 * BM : 0;  // [par][pass][y][half][row]
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 + 256 + RED_FLOATS * 4;
    static constexpr int TMEM_COLS = 2 * BN2;  // double-buffered 128 x 256 fp32 accumulators
};

template <typename T, bool LN>
__global__ void __launch_bounds__(Cfg2<LN>::THREADS, 1) gemm2_kernel(const __grid_constant__ GemmParams p) {
    using C = Cfg2<LN>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + C::STAGES * C::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;  // [2]
    uint64_t* tempty = tfull + 2;        // [2] (leader's are used)
    uint64_t* lnb = tempty + 2;          // [2 parity][2 pass]
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(lnb + 4);
    float* red = reinterpret_cast<float*>(smem + C::STAGES * (C::A_BYTES + C::B_BYTES) + 256);

    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_rank();
    const uint32_t px = rank & 1u;          // 0: leader, rows [0,128) of the pair tile; 1: rows [128,256)
    const uint32_t leader = rank & ~1u;
    const uint32_t nct = LN ? static_cast<uint32_t>(p.nct) : 1u;
    const int nk = (p.K + BK - 1) / BK;
    const int n_tiles = (p.N + BN2 - 1) / BN2;
    const int mp_tiles = (p.M + 2 * BM - 1) / (2 * BM);

    auto tile_of = [&](int i, int& mp, int& nb) -> bool {
        if constexpr (LN) {  // cluster c walks row blocks; its pair y owns n-tile y
            const int ncl = static_cast<int>(gridDim.y / nct);
            nb = static_cast<int>(blockIdx.y % nct);
            mp = static_cast<int>(blockIdx.y / nct) + i * ncl;
            return mp < mp_tiles;
        } else {  // pair blockIdx.y walks t = pair + i * pairs, n fastest (X rows reused from L2)
            const int t = static_cast<int>(blockIdx.y) + i * static_cast<int>(gridDim.y);
            mp = t / n_tiles;
            nb = t - mp * n_tiles;
            return mp < mp_tiles;
        }
    };

    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&p.ta);
        tc::prefetch_tmap(&p.tb);
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 2 * C::EPI_WARPS);  // one arrive per epilogue warp of both CTAs
        }
        if (LN)
            for (int b = 0; b < 4; ++b) tc::mbar_init(&lnb[b], 32 * C::EPI_WARPS * nct);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc2<C::TMEM_COLS>(tmem_ptr);
    tc::fence_before_sync();
    __syncthreads();
    tc::cluster_sync_all();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer (both CTAs)
        if (tc::elect_one()) {
            const uint64_t pol_a = tc::policy_evict_first();
            const uint64_t pol_b = tc::policy_evict_last();
            const uint32_t full0 = tc::mapa_u32(&full[0], leader);
            int s = 0;
            uint32_t ph = 0;
            int mp, nb;
            for (int i = 0; tile_of(i, mp, nb); ++i) {
                const int arow = (2 * mp + static_cast<int>(px)) * BM;
                const int brow = nb * BN2 + static_cast<int>(px) * (BN2 / 2);
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&empty[s], ph ^ 1);
                    if (px == 0) tc::mbar_expect_tx(&full[s], 2 * (C::A_BYTES + C::B_BYTES));
                    tc::tma_load_2d_pair(sA + s * C::A_BYTES, &p.ta, full0 + 8u * s, kb * BK, arow, pol_a);
                    tc::tma_load_2d_pair(sB + s * C::B_BYTES, &p.tb, full0 + 8u * s, kb * BK, brow, pol_b);
                    if (++s == C::STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer (leader)
        constexpr uint32_t idesc = tc::idesc_f16(2 * BM, BN2, std::is_same<T, __nv_bfloat16>::value, 0, 0);
        if (px == 0 && tc::elect_one()) {
            const uint16_t pair_mask = static_cast<uint16_t>(3u << leader);
            int s = 0;
            uint32_t ph = 0;
            int mp, nb;
            for (int i = 0; tile_of(i, mp, nb); ++i) {
                const int acc = i & 1;
                tc::mbar_wait_cluster(&tempty[acc], ((i >> 1) & 1) ^ 1);  // both epilogues drained it
                tc::fence_after_sync();
                const uint32_t d = tmem + acc * BN2;
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&full[s], ph);
                    tc::fence_after_sync();
                    const uint32_t a0 = tc::smem_u32(sA + s * C::A_BYTES);
                    const uint32_t b0 = tc::smem_u32(sB + s * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc::mma2_f16_ss(d, tc::sdesc_sw128(a0 + 32 * k), tc::sdesc_sw128(b0 + 32 * k), idesc,
                                        (kb | k) != 0);
                    tc::mma2_commit_mc(&empty[s], pair_mask);
                    if (++s == C::STAGES) { s = 0; ph ^= 1; }
                }
                tc::mma2_commit_mc(&tfull[acc], pair_mask);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------------ epilogue (both CTAs)
        const uint32_t q = warp & 3;
        const int r_local = static_cast<int>(q * 32 + lane);
        constexpr int CHUNKS = BN2 / 32;
        constexpr int GROUPS = C::EPI_WARPS / 4;
        const int grp = static_cast<int>((warp - 4) >> 2);
        const int c_begin = grp * (CHUNKS / GROUPS);
        const int c_end = c_begin + CHUNKS / GROUPS;
        auto release = [&](int acc) {  // this warp's TMEM reads are complete: tell the leader's MMA
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) {
                if (px == 0) tc::mbar_arrive(&tempty[acc]);
                else tc::mbar_arrive_cluster(&tempty[acc], leader);
            }
        };
        int mp, nb;
        for (int i = 0; tile_of(i, mp, nb); ++i) {
            const int acc = i & 1;
            tc::mbar_wait(&tfull[acc], (i >> 1) & 1);
            tc::fence_after_sync();
            const uint32_t taddr = tmem + acc * BN2 + ((q * 32) << 16);
            const int64_t row = static_cast<int64_t>(2 * mp + static_cast<int>(px)) * BM + r_local;
            const bool row_ok = row < p.M;
            const int n0 = nb * BN2;
            uint32_t r[32];
            float x[32];
            if constexpr (!LN) {
                for (int c = c_begin; c < c_end; ++c) {
                    __syncwarp();
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    if (c == c_end - 1) release(acc);
                    const int64_t col = n0 + c * 32;
                    if (!row_ok || col >= p.N) continue;
                    epi_chunk<T>(p, r, row, col, x);
                    store_chunk<T>(p.out, p.ldout, row, col, x);
                }
            } else {
                const int par = i & 1;
                const uint32_t my_y = rank >> 1;
                float sum = 0.f;
                uint4 aux_cur[4], aux_nxt[4];
                load_aux<T>(p, row_ok, row, n0 + c_begin * 32, aux_cur);
                for (int c = c_begin; c < c_end; ++c) {
                    if (c + 1 < c_end) load_aux<T>(p, row_ok, row, n0 + (c + 1) * 32, aux_nxt);
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    if (row_ok) epi_chunk_pre<T>(p, r, n0 + c * 32, aux_cur, x);
                    else
#pragma unroll
                        for (int j = 0; j < 32; ++j) x[j] = 0.f;
                    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        s4[j & 3] += x[j];
                        r[j] = __float_as_uint(x[j]);
                    }
                    sum += (s4[0] + s4[1]) + (s4[2] + s4[3]);
                    tc::tmem_st32(taddr + c * 32, r);
#pragma unroll
                    for (int j = 0; j < 4; ++j) aux_cur[j] = aux_nxt[j];
                }
                tc::tmem_st_wait();
                auto exchange = [&](float v, int pass) -> float {
                    float* slot = red + ((par * 2 + pass) * nct) * 2 * BM;  // [y][grp][row]
                    const int mine = (static_cast<int>(my_y) * 2 + grp) * BM + r_local;
                    slot[mine] = v;
                    for (uint32_t y = 0; y < nct; ++y)
                        if (y != my_y) tc::st_dsmem_f32(&slot[mine], px + 2 * y, v);
                    for (uint32_t y = 0; y < nct; ++y)
                        if (y != my_y) tc::mbar_arrive_cluster(&lnb[par * 2 + pass], px + 2 * y);
                    tc::mbar_arrive(&lnb[par * 2 + pass]);
                    tc::mbar_wait_cluster(&lnb[par * 2 + pass], (i >> 1) & 1);
                    float t = 0.f;
                    for (uint32_t c = 0; c < 2 * nct; ++c) t += slot[c * BM + r_local];
                    return t;
                };
                const float mean = exchange(sum, 0) / static_cast<float>(p.N);
                float sq4[4] = {0.f, 0.f, 0.f, 0.f};
                for (int c = c_begin; c < c_end; ++c) {
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float d = __uint_as_float(r[j]) - mean;
                        sq4[j & 3] = fmaf(d, d, sq4[j & 3]);
                    }
                }
                const float sq = (sq4[0] + sq4[1]) + (sq4[2] + sq4[3]);
                const float inv = 1.0f / sqrtf(exchange(sq, 1) / static_cast<float>(p.N) + kLnEps);
                float y[32];
                for (int c = c_begin; c < c_end; ++c) {
                    __syncwarp();
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    if (c == c_end - 1) release(acc);
                    if (!row_ok) continue;
                    const int64_t col = n0 + c * 32;
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        x[j] = __uint_as_float(r[j]);
                        y[j] = (x[j] - mean) * inv * __ldg(p.gamma + col + j) + __ldg(p.beta + col + j);
                    }
                    store_chunk<T>(p.out, p.ldout, row, col, y);
                    if (p.out_pre_ln) store_chunk<T>(p.out_pre_ln, p.ldout, row, col, x);
                }
            }
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::cluster_sync_all();  // the peer's MMAs / remote arrives are done before TMEM goes away
    if (warp == 1) tc::tmem_dealloc2<C::TMEM_COLS>(tmem);
}

// clusters of `cdim` CTAs of this kernel that fit on the device at once (cached per config)
template <typename T, bool LN>
int max_clusters(int cdim_y) {
    static int cache[kMaxNct + 1] = {};
    int& c = cache[std::min(cdim_y, kMaxNct)];
    if (c) return c;
    using Cf = Cfg2<LN>;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2, cdim_y * 64);
    cfg.blockDim = dim3(Cf::THREADS);
    cfg.dynamicSmemBytes = Cf::SMEM;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = static_cast<unsigned>(cdim_y);
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm2_kernel<T, LN>, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = num_sms() / (2 * cdim_y);
    }
    return c = n;
}

template <typename T, bool LN>
sf_status launch_pair(const sf_gemm_args& a, cudaStream_t st) {
    using Cf = Cfg2<LN>;
    GemmParams p{};
    const bool bf = std::is_same<T, __nv_bfloat16>::value;
    SF_TRY(make_tmap_2d(&p.ta, a.x, a.M, a.K, a.ldx, BK, BM, bf));
    SF_TRY(make_tmap_2d(&p.tb, a.w, a.N, a.K, a.ldw, BK, BN2 / 2, bf));
    p.M = a.M; p.N = a.N; p.K = a.K;
    p.out = a.out; p.ldout = a.ldout;
    p.bias = static_cast<const float*>(a.epi.bias);
    p.act = a.epi.act;
    p.aux = a.epi.aux; p.ldaux = a.epi.ldaux;
    p.gamma = static_cast<const float*>(a.epi.ln_gamma);
    p.beta = static_cast<const float*>(a.epi.ln_beta);
    p.out_pre_ln = a.epi.out_pre_ln;
    p.mc = 1;
    const int n_tiles = static_cast<int>(ceil_div(a.N, BN2));
    const int mp_tiles = static_cast<int>(ceil_div(a.M, 2 * BM));
    const int nct = LN ? n_tiles : 1;
    p.nct = nct;
    auto kern = gemm2_kernel<T, LN>;
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int units = LN ? mp_tiles : mp_tiles * n_tiles;  // work items of one cluster
    const int clusters = std::max(1, std::min(units, max_clusters<T, LN>(nct)));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2, nct * clusters);
    cfg.blockDim = dim3(Cf::THREADS);
    cfg.dynamicSmemBytes = Cf::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = static_cast<unsigned>(nct);
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    SF_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    SF_LAUNCH_CHECK();
    return SF_OK;
}

}  // namespace

bool gemm_pair_supported(const sf_gemm_args& a, bool ln) {
    if (a.M <= BM) return false;  // a pair would leave one SM idle
    if (ln) return a.N % BN2 == 0 && a.N / BN2 <= kMaxNct;
    return true;
}

sf_status gemm_pair_dispatch(const sf_gemm_args& a, bool ln, cudaStream_t st) {
    if (!gemm_pair_supported(a, ln))
        return fail(SF_SHAPE_ERROR, ln ? "CTA-pair LayerNorm GEMM needs M > 128, N % 256 == 0 and N <= 1024"
                                       : "CTA-pair GEMM needs M > 128");
    if (a.dtype == SF_BF16) return ln ? launch_pair<__nv_bfloat16, true>(a, st) : launch_pair<__nv_bfloat16, false>(a, st);
    return ln ? launch_pair<__half, true>(a, st) : launch_pair<__half, false>(a, st);
}

}  // namespace sf
