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
// per-row (mean, M2) partials with the nct CTAs holding the same rows (ranks px + 2y): one DSMEM
// exchange per tile, one remote arrive per warp and peer.
#include <algorithm>
#include <cstring>

#include "epilogue.cuh"

namespace sf {
extern unsigned long long* g_gemm_trace;
namespace {

constexpr int BN2 = 256;  // pair tile N; each CTA holds BN2/2 rows of W
constexpr int kMaxNct = 4;  // LN cluster 2 x nct <= 8 CTAs (portable cluster size)

// clock64 timeline of the leader CTA of pair 0 (tools/gemm_trace.py); -DSF_GEMM_TRACE only
#ifdef SF_GEMM_TRACE
#define GTRACE(i, ev)                                                                              \
    do {                                                                                           \
        if (p.trace && blockIdx.y == 0 && px == 0 && (i) < 64) p.trace[(i) * 8 + (ev)] = clock64(); \
    } while (0)
// per-CTA globaltimer (ns): entry, after the PDL wait, before teardown, cluster arrive, cluster wait
#define GSPAN(ev)                                                                                       \
    do {                                                                                                \
        if (p.trace && threadIdx.x == 0) {                                                              \
            unsigned long long t_;                                                                      \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                      \
            p.trace[512 + 8 * (blockIdx.y * gridDim.x + blockIdx.x) + (ev)] = t_;                      \
        }                                                                                               \
    } while (0)
#else
#define GTRACE(i, ev) \
    do {              \
    } while (0)
#define GSPAN(ev) \
    do {          \
    } while (0)
#endif

template <bool LN>
struct Cfg2 {
    static constexpr int STAGES = LN ? 5 : 6;
    static constexpr int EPI_WARPS = LN ? 8 : 16;
    static constexpr int THREADS = 128 + 32 * EPI_WARPS;
    static constexpr int A_BYTES = BM * BK * 2;         // 16 KB
    static constexpr int B_BYTES = (BN2 / 2) * BK * 2;  // 16 KB
    // LN: (mean, M2) partials [par][y][grp][row] as float2, then this CTA's bias/gamma/beta slice
    static constexpr int RED_FLOATS = LN ? 2 * kMaxNct * 2 * BM * 2 + 3 * BN2 : 0;
    // 32 x 32 fp16 staging boxes per epilogue warp (64-byte swizzle): the residual tile arrives by
    // TMA load and the output leaves by TMA store through them (LN: a second box for out_pre_ln)
    static constexpr int NBOX = LN ? 2 : 1;
    static constexpr int STG_BYTES = EPI_WARPS * NBOX * 2048;
    static constexpr int BAR_BYTES = 512;
    static constexpr int SMEM = STAGES * (A_BYTES + B_BYTES) + STG_BYTES + 1024 + BAR_BYTES + RED_FLOATS * 4;
    static constexpr int TMEM_COLS = 2 * BN2;  // double-buffered 128 x 256 fp32 accumulators
};

template <typename T, bool LN>
__global__ void __launch_bounds__(Cfg2<LN>::THREADS, 1) gemm2_kernel(const __grid_constant__ GemmParams p) {
    using C = Cfg2<LN>;
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + C::STAGES * C::A_BYTES;
    unsigned char* sStg = sB + C::STAGES * C::B_BYTES;  // [EPI_WARPS][NBOX][2 KB], 1024-aligned
    uint64_t* full = reinterpret_cast<uint64_t*>(sStg + C::STG_BYTES);
    uint64_t* empty = full + C::STAGES;
    uint64_t* tfull = empty + C::STAGES;  // [2]
    uint64_t* tempty = tfull + 2;        // [2] (leader's are used)
    uint64_t* lnb = tempty + 2;          // [2 parity]
    uint64_t* abar = lnb + 4;            // [EPI_WARPS][2]: residual box landed
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(abar + 2 * C::EPI_WARPS);
    float* red = reinterpret_cast<float*>(smem + C::STAGES * (C::A_BYTES + C::B_BYTES) + C::STG_BYTES + C::BAR_BYTES);

    GSPAN(0);
#ifdef SF_GEMM_TRACE
    const long long c_entry = clock64();
#endif
    GSPAN(1);
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
        tc::prefetch_tmap(&p.tc);
        if (p.aux) tc::prefetch_tmap(&p.taux);
        for (int s = 0; s < C::STAGES; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(&tfull[b], 1);
            tc::mbar_init(&tempty[b], 2 * C::EPI_WARPS);  // one arrive per epilogue warp of both CTAs
        }
        if (LN)  // one arrive per epilogue warp of every CTA holding these rows
            for (int b = 0; b < 2; ++b) tc::mbar_init(&lnb[b], C::EPI_WARPS * nct);
        for (int w = 0; w < 2 * C::EPI_WARPS; ++w) tc::mbar_init(&abar[w], 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc2<C::TMEM_COLS>(tmem_ptr);
    float2* part = reinterpret_cast<float2*>(red);                 // [2][nct][2][BM]
    float* sprm = red + 2 * kMaxNct * 2 * BM * 2;                  // [3][BN2]: bias, gamma, beta
    if constexpr (LN) {  // the n-tile is fixed per CTA in LN mode: stage its epilogue vectors once
        const int c0 = static_cast<int>(blockIdx.y % nct) * BN2;
        for (int t = threadIdx.x; t < BN2; t += blockDim.x) {
            sprm[t] = p.bias ? p.bias[c0 + t] : 0.f;
            sprm[BN2 + t] = p.gamma[c0 + t];
            sprm[2 * BN2 + t] = p.beta[c0 + t];
        }
    }
    tc::fence_before_sync();
    __syncthreads();
    tc::cluster_sync_all();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;
    // the prologue above reads only parameters (bias / LayerNorm vectors): it overlaps the stream
    // predecessor's tail under PDL; activations are read and outputs written only after this wait
    pdl_enter();

    if (warp == 0) {
        // ------------------------------------------------------------------ TMA producer (both CTAs)
        if (tc::elect_one()) {
            // X rows are re-read by the n_tiles pairs working on the same row block at about the
            // same time: evict_first made them miss in L2 (5x DRAM re-reads measured)
            const uint64_t pol_a = tc::policy_evict_normal();
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
                    if (kb == 0) GTRACE(i, 0);
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
                GTRACE(i, 1);
                tc::fence_after_sync();
                const uint32_t d = tmem + acc * BN2;
                for (int kb = 0; kb < nk; ++kb) {
                    tc::mbar_wait(&full[s], ph);
                    if (kb == 0) GTRACE(i, 2);
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
                GTRACE(i, 3);
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
        // this warp's staging boxes (box 0: residual in / output out; box 1: LN out_pre_ln)
        unsigned char* const boxp = sStg + (warp - 4) * (C::NBOX * 2048u);
        const uint32_t box = tc::smem_u32(boxp);
        uint64_t* const my_abar = &abar[2 * (warp - 4)];
        uint32_t aph = 0;
        auto aux_issue = [&](int col, int row0) {  // lane 0: residual box -> box 0 once its last store read it
            if (lane == 0) {
                tc::bulk_wait_read<0>();
                tc::mbar_expect_tx(my_abar, 2048);
                tc::tma_load_2d(boxp, &p.taux, my_abar, col, row0);
            }
        };
        auto aux_add = [&](float (&xx)[32]) {  // wait for the box and add this lane's row of it
            tc::mbar_wait(my_abar, aph);
            aph ^= 1;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint4 u;
                const uint32_t ad = box + lane * 64u + ((static_cast<uint32_t>(j) ^ ((lane >> 1) & 3)) << 4);
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(ad));
                const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
                for (int e = 0; e < 8; ++e) xx[8 * j + e] += DT<T>::to_f(h[e]);
            }
        };
        auto store_box = [&](int k, const CUtensorMap* map, const float (&xx)[32], int col, int row0, bool waited) {
            if (!waited && lane == 0) tc::bulk_wait_read<0>();
            __syncwarp();
            stage_chunk<T>(box + k * 2048u, static_cast<int>(lane), xx);
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                tc::tma_store_2d(map, boxp + k * 2048u, col, row0);
                tc::bulk_commit();
            }
        };
        int mp, nb;
        for (int i = 0; tile_of(i, mp, nb); ++i) {
            const int acc = i & 1;
            tc::mbar_wait(&tfull[acc], (i >> 1) & 1);
            if (warp == 4 && lane == 0) GTRACE(i, 4);
            tc::fence_after_sync();
            const uint32_t taddr = tmem + acc * BN2 + ((q * 32) << 16);
            const int64_t row = static_cast<int64_t>(2 * mp + static_cast<int>(px)) * BM + r_local;
            const bool row_ok = row < p.M;
            const int n0 = nb * BN2;
            uint32_t r[32];
            float x[32];
            const int row0 = (2 * mp + static_cast<int>(px)) * BM + static_cast<int>(q) * 32;
            if constexpr (!LN) {
                // each 32-row x 32-column chunk: the residual box (if any) arrives by TMA while the
                // accumulator is read; registers -> swizzled staging box -> one TMA store
                // (coalesced full-line traffic; rows >= M / cols >= N are clipped by the TMA unit)
                for (int c = c_begin; c < c_end; ++c) {
                    const int col = n0 + c * 32;
                    const bool in_range = col < p.N;  // warp-uniform
                    if (p.aux && in_range) aux_issue(col, row0);
                    __syncwarp();
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    if (c == c_end - 1) {
                        release(acc);
                        if (warp == 4 && lane == 0) GTRACE(i, 5);
                    }
                    if (!in_range) continue;
                    epi_chunk<T>(p, r, row, col, x, false);
                    if (p.aux) aux_add(x);
                    store_box(0, &p.tc, x, col, row0, p.aux != nullptr);
                }
                if (warp == 4 && lane == 0) GTRACE(i, 6);
            } else {
                // LayerNorm over the row split across nct CTAs x GROUPS warps: each thread owns
                // one row and CPT chunks of 32 columns. Pass 1 below; then one exchange of (mean,
                // M2) partials and a Chan combination (numerically the two-pass variance); pass 3:
                // normalise, store.
                const int par = i & 1;
                const uint32_t my_y = rank >> 1;
                // pass 1, per 32-column chunk: x = acc + bias (+act) + residual back into TMEM and
                // the chunk's (mean, M2) from registers; the chunks combine by Chan's formula, so
                // no second TMEM pass is needed for the variance. The residual boxes are double-
                // buffered: chunk c+1's load flies while c is added.
                constexpr int CPT = CHUNKS / GROUPS;
                uint32_t bph = 0u;  // bit b: phase of residual box b
                auto res_issue = [&](int b_, int col) {
                    __syncwarp();  // every lane's reads of the box are done
                    if (lane == 0) {
                        tc::bulk_wait_read<0>();
                        tc::mbar_expect_tx(&my_abar[b_], 2048);
                        tc::tma_load_2d(boxp + b_ * 2048, &p.taux, &my_abar[b_], col, row0);
                    }
                };
                if (p.aux) res_issue(0, n0 + c_begin * 32);
                // the chunk loops stay rolled: the epilogue runs a handful of times per CTA, so an
                // unrolled body is fetched cold each time (no_instructions stalls)
                float run_n = 0.f, run_mean = 0.f, run_m2 = 0.f;  // Chan's running (count, mean, M2)
#pragma unroll 1
                for (int cc = 0; cc < CPT; ++cc) {
                    const int c = c_begin + cc;
                    if (p.aux && cc + 1 < CPT) res_issue((cc + 1) & 1, n0 + (c + 1) * 32);
                    tc::tmem_ld32(taddr + c * 32, r);
                    tc::tmem_ld_wait();
                    const float4* b4 = reinterpret_cast<const float4*>(sprm + c * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 bb = b4[j];
                        x[4 * j] = __uint_as_float(r[4 * j]) + bb.x;
                        x[4 * j + 1] = __uint_as_float(r[4 * j + 1]) + bb.y;
                        x[4 * j + 2] = __uint_as_float(r[4 * j + 2]) + bb.z;
                        x[4 * j + 3] = __uint_as_float(r[4 * j + 3]) + bb.w;
                    }
                    if (p.act) {
#pragma unroll
                        for (int j = 0; j < 32; ++j) x[j] = act_fn(x[j], p.act);
                    }
                    if (p.aux) {
                        const int b_ = cc & 1;
                        tc::mbar_wait(&my_abar[b_], (bph >> b_) & 1u);
                        bph ^= 1u << b_;
                        const uint32_t bx = box + b_ * 2048u;
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            uint4 u;
                            const uint32_t ad = bx + lane * 64u + ((static_cast<uint32_t>(j) ^ ((lane >> 1) & 3)) << 4);
                            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                         : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w) : "r"(ad));
                            const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
                            for (int e = 0; e < 8; ++e) x[8 * j + e] += DT<T>::to_f(h[e]);
                        }
                    }
                    float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        s4[j & 3] += x[j];
                        r[j] = __float_as_uint(x[j]);
                    }
                    tc::tmem_st32(taddr + c * 32, r);
                    const float mc = ((s4[0] + s4[1]) + (s4[2] + s4[3])) * (1.f / 32.f);
                    float q4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float d = x[j] - mc;
                        q4[j & 3] = fmaf(d, d, q4[j & 3]);
                    }
                    {  // Chan: merge (32, mc, m2c) into the running statistics
                        const float m2c = (q4[0] + q4[1]) + (q4[2] + q4[3]);
                        const float n_new = run_n + 32.f;
                        const float dd = mc - run_mean;
                        run_mean += dd * (32.f / n_new);
                        run_m2 += m2c + dd * dd * (run_n * 32.f / n_new);
                        run_n = n_new;
                    }
                }
                tc::tmem_st_wait();
                const float lmean = run_mean, lm2 = run_m2;
                constexpr float kCols = 32.f * CPT;
                const float2 mine = make_float2(lmean, lm2);
                // exchange: every lane writes its row's partial into each row-sharing CTA, then one
                // arrive per warp and peer (release.cluster after the warp's stores)
                float2* slot = part + par * (kMaxNct * 2 * BM);
                const int my_idx = (static_cast<int>(my_y) * 2 + grp) * BM + r_local;
                slot[my_idx] = mine;
                for (uint32_t yy = 0; yy < nct; ++yy)
                    if (yy != my_y) tc::st_dsmem_f32x2(&slot[my_idx], px + 2 * yy, mine);
                __syncwarp();
                if (lane == 0) {
                    for (uint32_t yy = 0; yy < nct; ++yy)
                        if (yy != my_y) tc::mbar_arrive_cluster(&lnb[par], px + 2 * yy);
                    tc::mbar_arrive(&lnb[par]);
                }
                if (warp == 4 && lane == 0) GTRACE(i, 7);  // partials out (passes 1-2 done)
                tc::mbar_wait_cluster(&lnb[par], (i >> 1) & 1);
                if (warp == 4 && lane == 0) GTRACE(i, 6);  // exchange complete
                const int parts = static_cast<int>(2 * nct);
                float msum = 0.f;
                for (int j = 0; j < parts; ++j) msum += slot[j * BM + r_local].x;
                const float mean = msum / static_cast<float>(parts);
                float m2 = 0.f;
                for (int j = 0; j < parts; ++j) {
                    const float2 v = slot[j * BM + r_local];
                    const float d = v.x - mean;
                    m2 += v.y + kCols * d * d;
                }
                const float inv = 1.0f / sqrtf(m2 / static_cast<float>(p.N) + kLnEps);
                // pass 3: normalise and store; the next chunk's TMEM load is in flight while this
                // chunk is staged, and the two boxes alternate so a store only waits for the one
                // before last (out_pre_ln: both boxes per chunk)
                tc::tmem_ld32(taddr + c_begin * 32, r);
#pragma unroll 1
                for (int cc = 0; cc < CPT; ++cc) {
                    const int c = c_begin + cc;
                    const int col = n0 + c * 32;
                    tc::tmem_ld_wait();
                    if (cc == CPT - 1) release(acc);
                    float y[32];
                    const float4* g4 = reinterpret_cast<const float4*>(sprm + BN2 + c * 32);
                    const float4* e4 = reinterpret_cast<const float4*>(sprm + 2 * BN2 + c * 32);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 g = g4[j], e = e4[j];
                        x[4 * j] = __uint_as_float(r[4 * j]);
                        x[4 * j + 1] = __uint_as_float(r[4 * j + 1]);
                        x[4 * j + 2] = __uint_as_float(r[4 * j + 2]);
                        x[4 * j + 3] = __uint_as_float(r[4 * j + 3]);
                        y[4 * j] = (x[4 * j] - mean) * inv * g.x + e.x;
                        y[4 * j + 1] = (x[4 * j + 1] - mean) * inv * g.y + e.y;
                        y[4 * j + 2] = (x[4 * j + 2] - mean) * inv * g.z + e.z;
                        y[4 * j + 3] = (x[4 * j + 3] - mean) * inv * g.w + e.w;
                    }
                    if (cc + 1 < CPT) {
                        __syncwarp();
                        tc::tmem_ld32(taddr + (c + 1) * 32, r);
                    }
                    if (p.out_pre_ln) {
                        store_box(0, &p.tc, y, col, row0, false);
                        store_box(1, &p.tpre, x, col, row0, true);
                    } else {
                        if (lane == 0) tc::bulk_wait_read<1>();
                        store_box(cc & 1, &p.tc, y, col, row0, true);
                    }
                }
            }
        }
    }
    if (warp >= 4 && lane == 0) tc::bulk_wait<0>();  // staged stores done before smem goes away
    tc::fence_before_sync();
    __syncthreads();
    GSPAN(2);
#ifdef SF_GEMM_TRACE
    {
        const long long c0 = clock64();
        asm volatile("barrier.cluster.arrive.release;" ::: "memory");
        const long long c1 = clock64();
        GSPAN(3);
        if (p.trace && threadIdx.x == 0) p.trace[512 + 8 * (blockIdx.y * gridDim.x + blockIdx.x) + 5] = c1 - c0;
        if (p.trace && threadIdx.x == 128) p.trace[512 + 8 * (blockIdx.y * gridDim.x + blockIdx.x) + 6] = c1 - c0;
    }
    asm volatile("barrier.cluster.wait.acquire;" ::: "memory");
    GSPAN(4);
    if (p.trace && threadIdx.x == 0) p.trace[512 + 8 * (blockIdx.y * gridDim.x + blockIdx.x) + 7] = clock64() - c_entry;
#else
    tc::cluster_sync_all();
#endif  // the peer's MMAs / remote arrives are done before TMEM goes away
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
    SF_TRY(make_tmap_2d(&p.tc, a.out, a.M, a.N, a.ldout, 32, 32, bf, 64));
    if (a.epi.aux) SF_TRY(make_tmap_2d(&p.taux, a.epi.aux, a.M, a.N, a.epi.ldaux, 32, 32, bf, 64));
    if (a.epi.out_pre_ln) SF_TRY(make_tmap_2d(&p.tpre, a.epi.out_pre_ln, a.M, a.N, a.ldout, 32, 32, bf, 64));
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
    p.trace = g_gemm_trace;
    auto kern = gemm2_kernel<T, LN>;
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM));
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    const int units = LN ? mp_tiles : mp_tiles * n_tiles;  // work items of one cluster
    const int clusters = std::max(1, std::min(units, max_clusters<T, LN>(nct)));
    cudaLaunchAttribute cl;
    cl.id = cudaLaunchAttributeClusterDimension;
    cl.val.clusterDim.x = 2;
    cl.val.clusterDim.y = static_cast<unsigned>(nct);
    cl.val.clusterDim.z = 1;
    SF_CUDA_TRY(launch_pdl(kern, dim3(2, nct * clusters), dim3(Cf::THREADS), Cf::SMEM, st, &cl, p));
    SF_LAUNCH_CHECK();
    return SF_OK;
}

}  // namespace

unsigned long long* g_gemm_trace = nullptr;

bool gemm_pair_supported(const sf_gemm_args& a, bool ln) {
    if (a.M <= BM) return false;  // a pair would leave one SM idle
    if (ln) return a.N % BN2 == 0 && a.N / BN2 <= kMaxNct;
    return true;
}

bool gemm_ln_panel_supported(const sf_gemm_args& a);          // gemm2_ln.cu
sf_status gemm_ln_panel(const sf_gemm_args& a, cudaStream_t st);

sf_status gemm_pair_dispatch(const sf_gemm_args& a, bool ln, cudaStream_t st) {
    if (ln && gemm_ln_panel_supported(a)) return gemm_ln_panel(a, st);  // one pair per 256-row panel
    if (!gemm_pair_supported(a, ln))
        return fail(SF_SHAPE_ERROR, ln ? "CTA-pair LayerNorm GEMM needs M > 128, N % 256 == 0 and N <= 1024"
                                       : "CTA-pair GEMM needs M > 128");
    if (a.dtype == SF_BF16) return ln ? launch_pair<__nv_bfloat16, true>(a, st) : launch_pair<__nv_bfloat16, false>(a, st);
    return ln ? launch_pair<__half, true>(a, st) : launch_pair<__half, false>(a, st);
}

}  // namespace sf

// Debug hook (not part of the boundary): clock64 timeline of pair 0 of subsequent CTA-pair GEMM
// launches into a device buffer of >= 64*8 uint64 (only in builds with -DSF_GEMM_TRACE).
extern "C" sf_status sf_debug_gemm_trace(void* dev_buf) {
    sf::g_gemm_trace = static_cast<unsigned long long*>(dev_buf);
    return SF_OK;
}
