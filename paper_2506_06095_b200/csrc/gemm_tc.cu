// gemm_tc.cu — the CiMi fused template (backend.hpp:240-264) as one persistent sm_100a kernel:
//   out[M x N] = epilogue( X[M x K] . W[N x K]^T )
//   epilogue = +bias[N] -> GELU/ReLU -> +aux[M x N] (residual Add) -> LayerNorm over the row
// (op semantics: backend.hpp:111-167; order = the chain's MI order after the Gemm).
//
// Persistent CTAs (one per SM) walk a static tile schedule of 128 x BN output tiles:
//   warp 0        TMA producer: X and W tiles (BK = 64 fp16 = one 128-byte swizzle row) into a
//                 STAGES-deep smem ring (mbarrier complete_tx).
//   warp 1        TMEM allocator + MMA issuer: one elected thread issues tcgen05.mma
//                 (M=128, N=BN, K=16) into one of TWO TMEM accumulators, so the epilogue of tile i
//                 overlaps the mainloop of tile i+1; tcgen05.commit frees smem stages / signals
//                 the epilogue.
//   warps 4..     epilogue: tcgen05.ld accumulator rows (warp w owns TMEM lanes 32*(w%4)..+31),
//                 apply the MI ops in registers, store fp16.
// LayerNorm needs whole rows. The N/BN CTAs of a row block form a thread-block cluster (the
// cluster walks row blocks together). x = acc+bias(+act)+aux is written back into the TMEM
// accumulator, and the per-row partial sums Σx and Σ(x-mean)^2 are pushed into every peer's
// shared memory (st.shared::cluster) followed by a remote mbarrier arrive; each CTA then reduces
// its peers' partials locally. Two-pass mean / biased variance, eps 1e-5, as the reference.
#include <algorithm>
#include <cstring>

#include "epilogue.cuh"

namespace sf {
namespace {

template <int BN, bool LN>
struct Cfg {
    static constexpr int STAGES = BN == 256 ? 4 : 6;
    static constexpr int EPI_WARPS = LN ? 8 : 16;  // per lane quarter: 2 (LN) or 4 column groups
    static constexpr int THREADS = 128 + 32 * EPI_WARPS;
    static constexpr int A_BYTES = BM * BK * 2;
    static constexpr int B_BYTES = BN * BK * 2;
    static constexpr int RED_FLOATS = LN ? 2 * 2 * kMaxCluster * 2 * BM : 0;  // [par][pass][cta][half][row]
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + 1024 /*align*/ + 256 /*barriers*/ + RED_FLOATS * 4;
    static constexpr int TMEM_COLS = 2 * BN;  // two accumulator buffers
};

template <typename T, int BN, bool LN>
__global__ void __launch_bounds__(Cfg<BN, LN>::THREADS, 1) gemm_fused_kernel(const __grid_constant__ GemmParams p) {
    using C = Cfg<BN, LN>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + C::STAGES * C::A_BYTES;
    uint64_t* full = reinterpret_cast<uint64_t*>(sB + C::STAGES * C::B_BYTES);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;  // [2]
    uint64_t* tempty = tfull + 2;        // [2]
    uint64_t* lnb = tempty + 2;          // [2 parity][2 pass]
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(lnb + 4);
    float* red = reinterpret_cast<float*>(smem + C::STAGES * (C::A_BYTES + C::B_BYTES) + 256);  // [2][2][8][128]

    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const int nk = (p.K + BK - 1) / BK;
    const int n_tiles = (p.N + BN - 1) / BN;
    const int m_tiles = (p.M + BM - 1) / BM;
    const uint32_t nct = LN ? gridDim.x : 1;  // cluster spans the row: cluster dims == (N/BN, 1, 1)
    // CTAs that share operand tiles through TMA multicast: the LN row cluster shares the
    // activation tile; plain GEMMs pair CTAs along M that share the weight tile
    const uint32_t csz = LN ? nct : static_cast<uint32_t>(p.mc);
    const uint32_t me = csz > 1 ? tc::cluster_rank() : 0;
    const uint16_t cmask = static_cast<uint16_t>((1u << csz) - 1u);

    // tile i of this CTA -> (m_blk, n_blk)
    auto tile_of = [&](int i, int& mb, int& nb) -> bool {
        if constexpr (LN) {
            mb = blockIdx.y + i * gridDim.y;
            nb = blockIdx.x;
            return mb < m_tiles;
        } else {
            // cluster c walks tiles t = c + i * n_clusters; its CTAs take consecutive m blocks
            const int t = static_cast<int>(blockIdx.x / csz) + i * static_cast<int>(gridDim.x / csz);
            const int mg = t / n_tiles;
            nb = t - mg * n_tiles;
            mb = mg * static_cast<int>(csz) + static_cast<int>(me);
            return t < (m_tiles / static_cast<int>(csz)) * n_tiles;
        }
    };

    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&p.ta);
        tc::prefetch_tmap(&p.tb);
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], csz);  // consumed by every CTA that receives the stage
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 32 * C::EPI_WARPS);
        }
        if (LN)  // every epilogue thread of every cluster CTA arrives once per (tile, pass)
            for (int b = 0; b < 4; ++b) tc::mbar_init(&lnb[b], 32 * C::EPI_WARPS * nct);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<C::TMEM_COLS>(tmem_ptr);
    tc::fence_before_sync();
    __syncthreads();
    if (csz > 1) tc::cluster_sync_all();  // peers' barriers are initialised before any remote traffic
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;
    pdl_enter();  // the prologue above overlaps the stream predecessor's tail under PDL

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer
        if (tc::elect_one()) {
            const uint64_t pol_a = tc::policy_evict_first();
            int s = 0;
            uint32_t ph = 0;
            int mb, nb;
            for (int i = 0; tile_of(i, mb, nb); ++i) {
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&empty[s], ph ^ 1);
                    tc::mbar_expect_tx(&full[s], C::A_BYTES + C::B_BYTES);  // full A and B arrive in every CTA
                    if (LN && csz > 1) {
                        // row cluster: k-blocks round-robin over the CTAs, each multicasting A
                        if (static_cast<uint32_t>(kb) % csz == me)
                            tc::tma_load_2d_mc(sA + s * C::A_BYTES, &p.ta, &full[s], kb * BK, mb * BM, cmask);
                        tc::tma_load_2d(sB + s * C::B_BYTES, &p.tb, &full[s], kb * BK, nb * BN);
                    } else if (csz > 1) {
                        // M pair: own A; each CTA loads 1/csz of the weight rows and multicasts them
                        const int rows = BN / static_cast<int>(csz);
                        tc::tma_load_2d_hint(sA + s * C::A_BYTES, &p.ta, &full[s], kb * BK, mb * BM, pol_a);
                        tc::tma_load_2d_mc(sB + s * C::B_BYTES + me * rows * 128, &p.tb, &full[s], kb * BK,
                                           nb * BN + static_cast<int>(me) * rows, cmask);
                    } else {
                        tc::tma_load_2d_hint(sA + s * C::A_BYTES, &p.ta, &full[s], kb * BK, mb * BM, pol_a);
                        tc::tma_load_2d(sB + s * C::B_BYTES, &p.tb, &full[s], kb * BK, nb * BN);
                    }
                    if (++s == C::STAGES) { s = 0; ph ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        constexpr uint32_t idesc = tc::idesc_f16(BM, BN, std::is_same<T, __nv_bfloat16>::value, 0, 0);
        if (tc::elect_one()) {
            int s = 0;
            uint32_t ph = 0;
            int mb, nb;
            for (int i = 0; tile_of(i, mb, nb); ++i) {
                const int acc = i & 1;
                tc::mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);  // epilogue drained this buffer
                tc::fence_after_sync();
                const uint32_t d = tmem + acc * BN;
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&full[s], ph);
                    tc::fence_after_sync();
                    const uint32_t a0 = tc::smem_u32(sA + s * C::A_BYTES);
                    const uint32_t b0 = tc::smem_u32(sB + s * C::B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k)
                        tc::mma_f16_ss(d, tc::sdesc_sw128(a0 + 32 * k), tc::sdesc_sw128(b0 + 32 * k), idesc,
                                       (kb | k) != 0);
                    if (csz > 1) tc::mma_commit_mc(&empty[s], cmask);  // free the stage in every sharer
                    else tc::mma_commit(&empty[s]);
                    if (++s == C::STAGES) { s = 0; ph ^= 1; }
                }
                tc::mma_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------------ epilogue
        const uint32_t q = warp & 3;
        const int r_local = static_cast<int>(q * 32 + lane);
        constexpr int CHUNKS = BN / 32;
        // each TMEM lane quarter (32 rows) is split into GROUPS column groups of CHUNKS/GROUPS
        // 32-column chunks; `half` (the group index) is 0/1 for the LayerNorm variant
        constexpr int GROUPS = C::EPI_WARPS / 4;
        const int half = static_cast<int>((warp - 4) >> 2);
        const int c_begin = half * (CHUNKS / GROUPS);
        const int c_end = c_begin + CHUNKS / GROUPS;
        int mb, nb;
        for (int i = 0; tile_of(i, mb, nb); ++i) {
            const int acc = i & 1;
            tc::mbar_wait(&tfull[acc], (i >> 1) & 1);
            tc::fence_after_sync();
            const uint32_t taddr = tmem + acc * BN + ((q * 32) << 16);
            const int64_t row = static_cast<int64_t>(mb) * BM + r_local;
            const bool row_ok = row < p.M;
            const int n0 = nb * BN;
            uint32_t r[32];
            float x[32];
            if constexpr (!LN) {
                for (int c = c_begin; c < c_end; ++c) {
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    if (c == c_end - 1) {  // accumulator fully read: hand it back to the MMA warp
                        tc::fence_before_sync();
                        tc::mbar_arrive(&tempty[acc]);
                    }
                    const int64_t col = n0 + c * 32;
                    if (!row_ok || col >= p.N) continue;
                    epi_chunk<T>(p, r, row, col, x);
                    store_chunk<T>(p.out, p.ldout, row, col, x);
                }
            } else {
                const int par = i & 1;
                // pass 1: x = acc + bias (+act) + aux, kept in TMEM; partial Σx. The residual
                // values of the next chunk are in flight while this chunk is processed.
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
                // Row reduction over the 2 column halves x nct cluster CTAs: every epilogue thread
                // of every CTA writes its partial into every CTA's slot array (peers through
                // DSMEM) and arrives on that CTA's barrier; one wait then covers all partials.
                auto exchange = [&](float v, int pass) -> float {
                    float* slot = red + ((par * 2 + pass) * nct) * 2 * BM;  // [cta][half][row]
                    const int mine = (static_cast<int>(me) * 2 + half) * BM + r_local;
                    slot[mine] = v;
                    for (uint32_t c = 0; c < nct; ++c)
                        if (c != me) tc::st_dsmem_f32(&slot[mine], c, v);
                    for (uint32_t c = 0; c < nct; ++c)
                        if (c != me) tc::mbar_arrive_cluster(&lnb[par * 2 + pass], c);
                    tc::mbar_arrive(&lnb[par * 2 + pass]);
                    tc::mbar_wait_cluster(&lnb[par * 2 + pass], (i >> 1) & 1);
                    float t = 0.f;
                    for (uint32_t c = 0; c < 2 * nct; ++c) t += slot[c * BM + r_local];
                    return t;
                };
                const float mean = exchange(sum, 0) / static_cast<float>(p.N);
                // pass 2: Σ(x - mean)^2
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
                // pass 3: normalise, store
                float y[32];
                for (int c = c_begin; c < c_end; ++c) {
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    if (c == c_end - 1) {
                        tc::fence_before_sync();
                        tc::mbar_arrive(&tempty[acc]);
                    }
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
    if (csz > 1) tc::cluster_sync_all();  // no CTA exits while a peer may still write its smem
    if (warp == 1) tc::tmem_dealloc<C::TMEM_COLS>(tmem);
}


template <typename T, int BN, bool LN>
sf_status launch_gemm(const sf_gemm_args& a, cudaStream_t st) {
    using Cf = Cfg<BN, LN>;
    GemmParams p{};
    const bool bf = std::is_same<T, __nv_bfloat16>::value;
    SF_TRY(make_tmap_2d(&p.ta, a.x, a.M, a.K, a.ldx, BK, BM, bf));
    const int m_tiles = static_cast<int>(ceil_div(a.M, BM)), n_tiles = static_cast<int>(ceil_div(a.N, BN));
    // plain GEMMs: pairs of CTAs along M share the weight tile by multicast (halves the per-CTA
    // weight traffic through L2) when the M tiles pair up and the grid has more than one wave
    const int mc = (!LN && m_tiles % 2 == 0 && m_tiles * n_tiles >= 2 * num_sms()) ? 2 : 1;
    SF_TRY(make_tmap_2d(&p.tb, a.w, a.N, a.K, a.ldw, BK, BN / mc, bf));
    p.mc = mc;
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
    cfg.blockDim = dim3(Cf::THREADS);
    cfg.dynamicSmemBytes = Cf::SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    if (LN) {
        const int nct = n_tiles;  // whole row per cluster
        const int clusters = std::max(1, std::min(m_tiles, num_sms() / nct));
        cfg.gridDim = dim3(nct, clusters);
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = static_cast<unsigned>(nct);
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
    } else {
        const int ctas = std::min(m_tiles * n_tiles, num_sms()) / mc * mc;
        cfg.gridDim = dim3(std::max(ctas, mc));
        if (mc > 1) {
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = static_cast<unsigned>(mc);
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
        }
    }
    cudaLaunchAttribute pdl;
    pdl.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl.val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[cfg.numAttrs] = pdl;
    cfg.numAttrs += 1;
    cfg.attrs = attr;
    SF_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, p));
    SF_LAUNCH_CHECK();
    return SF_OK;
}

template <typename T>
sf_status gemm_dispatch(const sf_gemm_args& a, cudaStream_t st) {
    const bool ln = a.epi.ln_gamma != nullptr;
    if (a.tile_n != SF_TILE_AUTO && a.tile_n != SF_TILE_PAIR && a.tile_n != 128 && a.tile_n != 256)
        return fail(SF_INVALID_PARAMETER, "tile_n must be SF_TILE_AUTO, SF_TILE_PAIR, 128 or 256");
    if (a.tile_n == SF_TILE_PAIR) return gemm_pair_dispatch(a, ln, st);
    if (a.tile_n == 128) {
        if (ln && (a.N % 128 || a.N / 128 > kMaxCluster)) return fail(SF_SHAPE_ERROR, "LayerNorm row does not fit 128-wide tiles");
        return ln ? launch_gemm<T, 128, true>(a, st) : launch_gemm<T, 128, false>(a, st);
    }
    if (a.tile_n == 256) {
        if (ln && (a.N % 256 || a.N / 256 > kMaxCluster)) return fail(SF_SHAPE_ERROR, "LayerNorm row does not fit 256-wide tiles");
        return ln ? launch_gemm<T, 256, true>(a, st) : launch_gemm<T, 256, false>(a, st);
    }
    // auto: CTA pairs whenever their 256 x 256 tiles still fill every SM (the L2-feed-bound
    // single-CTA tiles are kept for small problems); otherwise the widest tile that divides N
    // (LN needs whole rows inside one <= 8-CTA cluster)
    if (gemm_pair_supported(a, ln)) {
        const int64_t pair_ctas = 2 * ceil_div(a.M, 2 * BM) * ceil_div(a.N, 256);
        if (pair_ctas >= num_sms()) return gemm_pair_dispatch(a, ln, st);
    }
    // small problems: 128-wide tiles when 256-wide ones would leave most SMs idle (twice the CTAs
    // on a latency-bound GEMM, e.g. the M = 512 layers of cfg1)
    const bool few = ceil_div(a.M, BM) * ceil_div(a.N, 256) < num_sms();
    const bool ln_clusters = (a.N % 256 == 0 && a.N / 256 <= kMaxCluster) || (a.N % 128 == 0 && a.N / 128 <= kMaxCluster);
    if (ln && a.N <= 4096 && (!ln_clusters || ceil_div(a.M, BM) * ceil_div(a.N, 128) < num_sms() / 4)) {
        // a LayerNorm row cluster per 128 rows would occupy under a quarter of the SMs (or the row
        // does not split into <= 8 CTAs of 128/256 columns): the GEMM (+bias/act/residual) and a
        // MiChain LayerNorm pass over its output (in place, or from out_pre_ln) as two launches
        // (cfg1: 68.5 -> 61.6 us per layer step)
        sf_gemm_args g = a;
        g.epi.ln_gamma = g.epi.ln_beta = nullptr;
        g.epi.out_pre_ln = nullptr;
        void* mid = a.epi.out_pre_ln ? a.epi.out_pre_ln : a.out;
        g.out = mid;
        SF_TRY((launch_gemm<T, 128, false>(g, st)));
        sf_gemm_epilogue e{};
        e.ln_gamma = a.epi.ln_gamma;
        e.ln_beta = a.epi.ln_beta;
        return sf_mi_chain(a.M, a.N, a.dtype, mid, a.ldout, &e, a.out, a.ldout, st);
    }
    if (ln) {
        const bool fit256 = a.N % 256 == 0 && a.N / 256 <= kMaxCluster;
        const bool fit128 = a.N % 128 == 0 && a.N / 128 <= kMaxCluster;
        if (fit256 && !(few && fit128)) return launch_gemm<T, 256, true>(a, st);
        if (fit128) return launch_gemm<T, 128, true>(a, st);
        return fail(SF_SHAPE_ERROR, "fused LayerNorm needs N % 128 == 0 and N <= 2048");
    }
    if (a.N % 256 == 0 && !few) return launch_gemm<T, 256, false>(a, st);
    return launch_gemm<T, 128, false>(a, st);
}

}  // namespace

int num_sms() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

sf_status make_tmap_2d(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint64_t row_stride_elems,
                       uint32_t box_cols, uint32_t box_rows, bool bf16, int swizzle_bytes) {
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
                        swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                        : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                        : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                              : CU_TENSOR_MAP_SWIZZLE_NONE,
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
    if (a->epi.softmax && (a->epi.ln_gamma || a->epi.out_pre_ln))
        return fail(SF_INVALID_PARAMETER, "Softmax excludes LayerNorm / out_pre_ln");
    cudaStream_t st = as_stream(stream);
    if (a->epi.softmax) {
        // the row softmax needs the whole row's max and sum: GEMM (+bias/act/residual), then a
        // MiChain softmax pass over the output in place (the split LayerNorm path's shape)
        sf_gemm_args g = *a;
        g.epi.softmax = 0;
        SF_TRY(sf_gemm_fused(&g, stream));
        sf_gemm_epilogue e{};
        e.softmax = 1;
        return sf_mi_chain(a->M, a->N, a->dtype, a->out, a->ldout, &e, a->out, a->ldout, stream);
    }
    if (a->dtype == SF_F16) return gemm_dispatch<__half>(*a, st);
    if (a->dtype == SF_BF16) return gemm_dispatch<__nv_bfloat16>(*a, st);
    return fail(SF_INVALID_PARAMETER, "dtype must be f16/bf16");
}
