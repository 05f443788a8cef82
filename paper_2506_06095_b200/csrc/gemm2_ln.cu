// gemm2_ln.cu — the CiMi GEMM + bias (+act) + residual + LayerNorm template (backend.hpp:240-264,
// LayerNorm backend.hpp:140-153) on two-SM CTA pairs with a ROW-PANEL schedule, for N = 512 / 768.
//
// The cluster form in gemm2_tc.cu splits a row's N = 768 columns over three pairs (a 6-CTA
// cluster) and exchanges per-row (mean, M2) partials through DSMEM once per 256 x 256 tile. Its
// LayerNorm epilogue (~11 K cycles per tile) runs against a K = 768 mainloop of ~5.5 K cycles, and
// 6-CTA clusters place on 132 of 148 SMs: the out-projection ran at ~28% of the tensor peak.
// Here ONE pair owns all N columns of its 256 rows, so the whole LayerNorm stays inside the pair's
// CTAs (no cluster exchange) and every SM can hold a pair. The row's N/256 sub-tiles go through
// the pair's 512 TMEM columns (per CTA: 128 rows x 512 fp32):
//   sub-tile 0 -> A = [0, 256)   epilogue E0: + bias (+act) + residual, (mean, M2) per 32-column
//                                chunk, the pre-LN row packed to fp16 IN PLACE into
//                                A[128g, 128g + 64) (g = the warp's column half);
//   sub-tile 1 -> B = [256, 512) E1: same, packed into A[128g + 64, 128g + 128); B is released;
//   sub-tile 2 -> B              E2: same, kept in fp32 in B.
// (N = 512: sub-tile 1 is the last and stays in B.) The MMAs of sub-tile s+1 run under E_s, except
// sub-tile 2, which waits for E1 to have read B. One exchange of (mean, M2) between the two warps
// sharing a TMEM lane quarter, then the normalise pass reads the packed fp16 pre-LN values (the
// value the unfused form would write to HBM, SURVEY finding 3) and the fp32 last sub-tile, and
// stores through the per-warp swizzled staging boxes by TMA.
//   warp 0 (both CTAs)  TMA producer: X rows [128 (2 mp + px), +128) and W rows
//                       [256 s + 128 px, +128) of every sub-tile s into a 5-deep ring.
//   warp 1 (leader)     MMA issuer: M = 256, N = 256, K = 16 x 4 per stage (cta_group::2).
//   warps 4..11         epilogue: two warps per TMEM lane quarter, columns [0, 128) / [128, 256)
//                       of every sub-tile.
#include <algorithm>
#include <cstdlib>

#include "epilogue.cuh"

namespace sf {
extern unsigned long long* g_gemm_trace;
namespace {

constexpr int BNP = 256;              // N per sub-tile (one pair MMA tile)
constexpr int kMaxSub = 3;            // N <= 768
#ifndef SF_LNP_EPI
#define SF_LNP_EPI 8
#endif
constexpr int kEpiWarpsP = SF_LNP_EPI;          // 8 or 16: 2 or 4 warps per TMEM lane quarter
constexpr int kGroups = kEpiWarpsP / 4;         // column groups of a sub-tile
constexpr int kGW = BNP / kGroups;              // columns of a sub-tile per group (128 / 64)
constexpr int kCPG = kGW / 32;                  // 32-column chunks per group and sub-tile
constexpr int kStagesP = kEpiWarpsP == 8 ? 5 : 4;
constexpr int kThreadsP = 128 + 32 * kEpiWarpsP;
constexpr int kABytes = BM * BK * 2;          // 16 KB
constexpr int kBBytes = (BNP / 2) * BK * 2;   // 16 KB
constexpr int kStgBytesP = kEpiWarpsP * 2 * 2048;
constexpr int kPrmFloats = 3 * kMaxSub * BNP;  // bias, gamma, beta over N
constexpr int kPartFloats = 2 * kGroups * BM * 2;  // [parity][grp][row] float2
constexpr int kSmemP = 1024 + kStagesP * (kABytes + kBBytes) + kStgBytesP + 512 + (kPrmFloats + kPartFloats) * 4;
constexpr uint32_t kColB = 256;

// clock64 events of the leader CTA of pair 0, first row block (tools/gemm_ln_trace.py), and
// per-CTA globaltimer spans; -DSF_GEMM_TRACE builds only
#ifdef SF_GEMM_TRACE
#define LTRACE(ev)                                                                  \
    do {                                                                            \
        if (p.trace && blockIdx.y == 0 && px == 0 && i == 0) p.trace[ev] = clock64(); \
    } while (0)
#define LSPAN(ev)                                                                                   \
    do {                                                                                            \
        if (p.trace && threadIdx.x == 0) {                                                          \
            unsigned long long t_;                                                                  \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                                  \
            p.trace[512 + 8 * (blockIdx.y * gridDim.x + blockIdx.x) + (ev)] = t_;                  \
        }                                                                                           \
    } while (0)
#else
#define LTRACE(ev) \
    do {           \
    } while (0)
#define LSPAN(ev) \
    do {          \
    } while (0)
#endif

template <typename T, int NSUB>
__global__ void __launch_bounds__(kThreadsP, 1) gemm2_ln_kernel(const __grid_constant__ GemmParams p) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sA = smem;
    unsigned char* sB = smem + kStagesP * kABytes;
    unsigned char* sStg = sB + kStagesP * kBBytes;  // [8 warps][2][2 KB]
    uint64_t* full = reinterpret_cast<uint64_t*>(sStg + kStgBytesP);
    uint64_t* empty = full + kStagesP;
    uint64_t* tfull = empty + kStagesP;   // [kMaxSub] sub-tile s accumulated (both CTAs)
    uint64_t* afree = tfull + kMaxSub;    // leader: the normalise pass has read A (both CTAs' epilogues)
    uint64_t* bfree1 = afree + 1;         // leader: E1 has read B (N = 768)
    uint64_t* bfree2 = bfree1 + 1;        // leader: the normalise pass has read B
    uint64_t* abar = bfree2 + 1;          // [kEpiWarpsP][2] residual boxes landed
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(abar + 2 * kEpiWarpsP);
    float* sprm = reinterpret_cast<float*>(sStg + kStgBytesP + 512);  // [3][N]: bias, gamma, beta
    float2* part = reinterpret_cast<float2*>(sprm + kPrmFloats);       // [2][2][BM]

    LSPAN(1);
    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t rank = tc::cluster_rank();
    const uint32_t px = rank & 1u;
    const uint32_t leader = rank & ~1u;
#ifdef SF_GEMM_TRACE
    const uint32_t i = 0;  // LTRACE outside the row-block loops: the first block
    if (p.trace && blockIdx.y == 0 && px == 0 && threadIdx.x == 0) p.trace[26] = clock64();
#endif
    const int nk = (p.K + BK - 1) / BK;
    constexpr int nsub = NSUB;
    const int mp_tiles = (p.M + 2 * BM - 1) / (2 * BM);

    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&p.ta);
        tc::prefetch_tmap(&p.tb);
        tc::prefetch_tmap(&p.tc);
        if (p.aux) tc::prefetch_tmap(&p.taux);
        for (int s = 0; s < kStagesP; ++s) {
            tc::mbar_init(&full[s], 1);
            tc::mbar_init(&empty[s], 1);
        }
        for (int s = 0; s < kMaxSub; ++s) tc::mbar_init(&tfull[s], 1);
        tc::mbar_init(afree, 2 * kEpiWarpsP);
        tc::mbar_init(bfree1, 2 * kEpiWarpsP);
        tc::mbar_init(bfree2, 2 * kEpiWarpsP);
        for (int w = 0; w < 2 * kEpiWarpsP; ++w) tc::mbar_init(&abar[w], 1);
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc2<512>(tmem_ptr);
    for (int t = threadIdx.x; t < p.N; t += blockDim.x) {
        sprm[t] = p.bias ? p.bias[t] : 0.f;
        sprm[p.N + t] = p.gamma[t];
        sprm[2 * p.N + t] = p.beta[t];
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
            const uint64_t pol_a = tc::policy_evict_normal();  // X panel: re-read once per sub-tile
            const uint64_t pol_b = tc::policy_evict_last();    // W: read by every pair
            const uint32_t full0 = tc::mapa_u32(&full[0], leader);
            int s = 0;
            uint32_t ph = 0;
            for (int mp = static_cast<int>(blockIdx.y); mp < mp_tiles; mp += static_cast<int>(gridDim.y)) {
                const int arow = (2 * mp + static_cast<int>(px)) * BM;
                for (int sub = 0; sub < nsub; ++sub) {
                    const int brow = sub * BNP + static_cast<int>(px) * (BNP / 2);
                    for (int kb = 0; kb < nk; ++kb) {
                        tc::mbar_wait(&empty[s], ph ^ 1);
                        if (px == 0) tc::mbar_expect_tx(&full[s], 2 * (kABytes + kBBytes));
                        tc::tma_load_2d_pair(sA + s * kABytes, &p.ta, full0 + 8u * s, kb * BK, arow, pol_a);
                        tc::tma_load_2d_pair(sB + s * kBBytes, &p.tb, full0 + 8u * s, kb * BK, brow, pol_b);
                        if (++s == kStagesP) { s = 0; ph ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer (leader)
        constexpr uint32_t idesc = tc::idesc_f16(2 * BM, BNP, std::is_same<T, __nv_bfloat16>::value, 0, 0);
        if (px == 0 && tc::elect_one()) {
            const uint16_t pair_mask = static_cast<uint16_t>(3u << leader);
            int s = 0;
            uint32_t ph = 0;
            uint32_t i = 0;
            for (int mp = static_cast<int>(blockIdx.y); mp < mp_tiles; mp += static_cast<int>(gridDim.y), ++i) {
                for (int sub = 0; sub < nsub; ++sub) {
                    const bool last = sub == nsub - 1;
                    const uint32_t d = tmem + (sub == 0 && !last ? 0u : kColB);
                    if (sub == 0 && !last) {
                        if (i > 0) tc::mbar_wait_cluster(afree, (i - 1) & 1);
                    } else if (!last || nsub == 2) {
                        if (i > 0) tc::mbar_wait_cluster(bfree2, (i - 1) & 1);
                    } else {
                        tc::mbar_wait_cluster(bfree1, i & 1);  // E1 has moved sub-tile 1 out of B
                    }
                    tc::fence_after_sync();
                    LTRACE(8 * sub + 0);
                    for (int kb = 0; kb < nk; ++kb) {
                        tc::mbar_wait(&full[s], ph);
                        tc::fence_after_sync();
                        const uint32_t a0 = tc::smem_u32(sA + s * kABytes);
                        const uint32_t b0 = tc::smem_u32(sB + s * kBBytes);
#pragma unroll
                        for (int k = 0; k < BK / 16; ++k)
                            tc::mma2_f16_ss(d, tc::sdesc_sw128(a0 + 32 * k), tc::sdesc_sw128(b0 + 32 * k), idesc,
                                            (kb | k) != 0);
                        tc::mma2_commit_mc(&empty[s], pair_mask);
                        if (++s == kStagesP) { s = 0; ph ^= 1; }
                    }
                    tc::mma2_commit_mc(&tfull[sub], pair_mask);
                    LTRACE(8 * sub + 1);
                }
            }
        }
    } else if (warp >= 4) {
        // ------------------------------------------------------------------ epilogue (both CTAs)
        const uint32_t q = warp & 3;
        const int grp = static_cast<int>((warp - 4) >> 2);
        const int r_local = static_cast<int>(q * 32 + lane);
        const uint32_t tl = tmem + ((q * 32) << 16);
        unsigned char* const boxp = sStg + (warp - 4) * 4096u;
        const uint32_t box = tc::smem_u32(boxp);
        uint64_t* const my_abar = &abar[2 * (warp - 4)];
        auto arrive_leader = [&](uint64_t* bar) {
            tc::fence_before_sync();
            __syncwarp();
            if (lane == 0) {
                if (px == 0) tc::mbar_arrive(bar);
                else tc::mbar_arrive_cluster(bar, leader);
            }
        };
        auto res_issue = [&](int b_, int col, int row0) {  // residual 32 x 32 box into staging box b_
            __syncwarp();
            if (lane == 0) {
                tc::bulk_wait_read<0>();
                tc::fence_proxy_async();  // the box's generic-proxy staging reads/writes come first
                tc::mbar_expect_tx(&my_abar[b_], 2048);
                tc::tma_load_2d(boxp + b_ * 2048, &p.taux, &my_abar[b_], col, row0);
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
        // Stores go through the warp's 4 KB staging box: a lane stages 32 values of its row into
        // half h of its 128-byte staging row (16-byte piece j of row r at r * 128 + (j ^ (r & 7)) *
        // 16, conflict-free), then the warp writes the box as 4-row groups, eight lanes per row:
        // half 0 to (base0, col0), half 1 to (base1, col1) — two column chunks of one output, or
        // one chunk of the output and of out_pre_ln.
        auto stage = [&](const float (&yy)[32], int h) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t pc = static_cast<uint32_t>(4 * h + j);
                const uint32_t a = box + lane * 128u + ((pc ^ (lane & 7u)) << 4);
                asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(pack2<T>(yy[8 * j], yy[8 * j + 1])),
                             "r"(pack2<T>(yy[8 * j + 2], yy[8 * j + 3])), "r"(pack2<T>(yy[8 * j + 4], yy[8 * j + 5])),
                             "r"(pack2<T>(yy[8 * j + 6], yy[8 * j + 7]))
                             : "memory");
            }
        };
        auto flush = [&](void* base0, int col0, void* base1, int col1, int row0_) {
            __syncwarp();
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t rr = 4u * k + (lane >> 3), pc = lane & 7u;
                uint4 u;
                asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                             : "=r"(u.x), "=r"(u.y), "=r"(u.z), "=r"(u.w)
                             : "r"(box + rr * 128u + ((pc ^ (rr & 7u)) << 4)));
                const int64_t grow = static_cast<int64_t>(row0_) + rr;
                void* base = pc < 4 ? base0 : base1;
                const int c = (pc < 4 ? col0 : col1) + 8 * static_cast<int>(pc & 3u);
                if (grow < p.M) *reinterpret_cast<uint4*>(static_cast<T*>(base) + grow * p.ldout + c) = u;
            }
            __syncwarp();  // the box's reads are done before the next staging
        };
        uint32_t i = 0;
        uint32_t bph = 0;  // bit b: phase of residual box b
        // The chunk loops stay rolled: a pair runs one or two row panels, so unrolled code would be
        // fetched cold from L2 once per panel (an unrolled 12-chunk body measured ~2.5 K cycles per
        // chunk of instruction-fetch stalls).
        for (int mp = static_cast<int>(blockIdx.y); mp < mp_tiles; mp += static_cast<int>(gridDim.y), ++i) {
            const int row0 = (2 * mp + static_cast<int>(px)) * BM + static_cast<int>(q) * 32;
            float run_n = 0.f, run_mean = 0.f, run_m2 = 0.f;  // Chan's running (count, mean, M2)
            uint32_t r[32];
            float x[32];
            if (p.aux) {  // the residual ring runs two chunks ahead, across sub-tiles
                res_issue(0, grp * kGW, row0);
                res_issue(1, grp * kGW + 32, row0);
            }
            // ---- E_sub: bias (+act) + residual, chunk statistics, pre-LN values parked in TMEM
#pragma unroll 1
            for (int k = 0; k < kCPG * nsub; ++k) {
                const int sub = k / kCPG, cc = k % kCPG;
                const bool last = sub == nsub - 1;
                const uint32_t src = (sub == 0 && !last ? 0u : kColB) + kGW * grp;
                if (cc == 0) {
                    tc::mbar_wait(&tfull[sub], i & 1);
                    if (warp == 4 && lane == 0) LTRACE(8 * sub + 2);
                    tc::fence_after_sync();
                }
                const int col = sub * BNP + grp * kGW + cc * 32;
                if (cc == 0) tc::tmem_ld32(tl + src, r);  // later chunks were issued one chunk ahead
                tc::tmem_ld_wait();
#pragma unroll
                for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(r[j]);
                if (cc + 1 < kCPG) tc::tmem_ld32(tl + src + 32 * (cc + 1), r);
                const float4* b4 = reinterpret_cast<const float4*>(sprm + col);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 bb = b4[j];
                    const float2 lo = tc::fadd2(make_float2(x[4 * j], x[4 * j + 1]), make_float2(bb.x, bb.y));
                    const float2 hi = tc::fadd2(make_float2(x[4 * j + 2], x[4 * j + 3]), make_float2(bb.z, bb.w));
                    x[4 * j] = lo.x; x[4 * j + 1] = lo.y; x[4 * j + 2] = hi.x; x[4 * j + 3] = hi.y;
                }
                if (p.act) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = act_fn(x[j], p.act);
                }
                if (p.aux) {
                    const int b_ = k & 1;
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
                    const int k2 = k + 2;  // chunk k + 2 of the warp's walk into the box just read
                    if (k2 < kCPG * nsub) res_issue(b_, (k2 / kCPG) * BNP + grp * kGW + (k2 % kCPG) * 32, row0);
                }
                float2 s2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
                for (int j = 0; j < 32; j += 2) s2[(j >> 1) & 1] = tc::fadd2(s2[(j >> 1) & 1], make_float2(x[j], x[j + 1]));
                const float mc = ((s2[0].x + s2[0].y) + (s2[1].x + s2[1].y)) * (1.f / 32.f);
                float2 q2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                const float2 nmc = make_float2(-mc, -mc);
#pragma unroll
                for (int j = 0; j < 32; j += 2) {
                    const float2 dd = tc::fadd2(make_float2(x[j], x[j + 1]), nmc);
                    q2[(j >> 1) & 1] = tc::ffma2(dd, dd, q2[(j >> 1) & 1]);
                }
                {  // Chan: merge (32, mc, m2c) into the running statistics
                    const float m2c = (q2[0].x + q2[0].y) + (q2[1].x + q2[1].y);
                    const float n_new = run_n + 32.f;
                    const float dd = mc - run_mean;
                    run_mean += dd * (32.f / n_new);
                    run_m2 += m2c + dd * dd * (run_n * 32.f / n_new);
                    run_n = n_new;
                }
                if (last) {  // fp32 back in place
                    uint32_t w[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) w[j] = __float_as_uint(x[j]);
                    tc::tmem_st32(tl + src + 32 * cc, w);
                } else {     // fp16 pairs into A: sub-tile 0 at 128g + 16cc, sub-tile 1 at 128g + 64 + 16cc
                    uint32_t pk[16];
#pragma unroll
                    for (int j = 0; j < 16; ++j) pk[j] = pack2<T>(x[2 * j], x[2 * j + 1]);
                    tc::tmem_st16(tl + kGW * grp + (kGW / 2) * sub + 16u * cc, pk);
                }
                if (cc == kCPG - 1) {
                    tc::tmem_st_wait();
                    if (warp == 4 && lane == 0) LTRACE(8 * sub + 3);
                    if (sub == 1 && !last) arrive_leader(bfree1);  // B may take sub-tile 2
                }
            }
            // ---- the row's (mean, M2): this thread's columns, then the other column half's warp
            float2* slot = part + (i & 1) * (kGroups * BM);
            slot[grp * BM + r_local] = make_float2(run_mean, run_m2);
            asm volatile("bar.sync 1, %0;" ::"n"(32 * kEpiWarpsP) : "memory");
            if (warp == 4 && lane == 0) LTRACE(24);
            float2 part_g[kGroups];  // every group's (mean, M2) over an equal share of the row
            float mean = 0.f;
#pragma unroll
            for (int g2 = 0; g2 < kGroups; ++g2) {
                part_g[g2] = slot[g2 * BM + r_local];
                mean += part_g[g2].x;
            }
            mean *= 1.f / kGroups;
            const float group_cols = static_cast<float>(p.N / kGroups);
            float m2 = 0.f;
#pragma unroll
            for (int g2 = 0; g2 < kGroups; ++g2) {
                const float dd = part_g[g2].x - mean;
                m2 += part_g[g2].y + group_cols * dd * dd;
            }
            const float inv = 1.0f / sqrtf(m2 / static_cast<float>(p.N) + kLnEps);
            // ---- normalise and store; chunk k + 1's TMEM load flies while chunk k is normalised
            auto norm_load = [&](int k) {
                const int sub = k / kCPG, cc = k % kCPG;
                if (sub == nsub - 1) tc::tmem_ld32(tl + kColB + kGW * grp + 32u * cc, r);
                else tc::tmem_ld16(tl + kGW * grp + (kGW / 2) * sub + 16u * cc, *reinterpret_cast<uint32_t(*)[16]>(r));
            };
            norm_load(0);
#pragma unroll 1
            for (int k = 0; k < kCPG * nsub; ++k) {
                const int sub = k / kCPG, cc = k % kCPG;
                const bool last = sub == nsub - 1;
                const int col = sub * BNP + grp * kGW + cc * 32;
                tc::tmem_ld_wait();
                if (last) {
#pragma unroll
                    for (int j = 0; j < 32; ++j) x[j] = __uint_as_float(r[j]);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const T* h = reinterpret_cast<const T*>(&r[j]);
                        x[2 * j] = DT<T>::to_f(h[0]);
                        x[2 * j + 1] = DT<T>::to_f(h[1]);
                    }
                }
                if (k + 1 < kCPG * nsub) norm_load(k + 1);
                // y = ((x - mean) inv) g + e as two packed FMAs per pair
                float y[32];
                const float4* g4 = reinterpret_cast<const float4*>(sprm + p.N + col);
                const float4* e4 = reinterpret_cast<const float4*>(sprm + 2 * p.N + col);
                const float2 inv2 = make_float2(inv, inv), nmi2 = make_float2(-mean * inv, -mean * inv);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const float4 g = g4[j], e = e4[j];
                    const float2 t0 = tc::ffma2(make_float2(x[4 * j], x[4 * j + 1]), inv2, nmi2);
                    const float2 t1 = tc::ffma2(make_float2(x[4 * j + 2], x[4 * j + 3]), inv2, nmi2);
                    const float2 y0 = tc::ffma2(t0, make_float2(g.x, g.y), make_float2(e.x, e.y));
                    const float2 y1 = tc::ffma2(t1, make_float2(g.z, g.w), make_float2(e.z, e.w));
                    y[4 * j] = y0.x; y[4 * j + 1] = y0.y; y[4 * j + 2] = y1.x; y[4 * j + 3] = y1.y;
                }
                if (p.out_pre_ln) {  // the chunk of both outputs per box
                    stage(y, 0);
                    stage(x, 1);
                    flush(p.out, col, p.out_pre_ln, col, row0);
                } else {             // two chunks of the output per box
                    stage(y, cc & 1);
                    if (cc & 1) flush(p.out, col - 32, p.out, col, row0);
                }
            }
            if (warp == 4 && lane == 0) LTRACE(25);
            arrive_leader(afree);
            arrive_leader(bfree2);
        }
    }
    if (warp >= 4 && lane == 0) tc::bulk_wait<0>();  // staged stores done before smem goes away
    tc::fence_before_sync();
    __syncthreads();
    LSPAN(2);
    tc::cluster_sync_all();  // the peer's MMAs / remote arrives are done before TMEM goes away
    if (warp == 1) tc::tmem_dealloc2<512>(tmem);
}

int max_pairs_ln() {
    static int cache = 0;
    if (cache) return cache;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(2, 128);
    cfg.blockDim = dim3(kThreadsP);
    cfg.dynamicSmemBytes = kSmemP;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm2_ln_kernel<__half, 3>, &cfg) != cudaSuccess || n <= 0) {
        cudaGetLastError();
        n = num_sms() / 2;
    }
    return cache = n;
}

template <typename T>
sf_status launch_ln_panel(const sf_gemm_args& a, cudaStream_t st) {
    GemmParams p{};
    const bool bf = std::is_same<T, __nv_bfloat16>::value;
    SF_TRY(make_tmap_2d(&p.ta, a.x, a.M, a.K, a.ldx, BK, BM, bf));
    SF_TRY(make_tmap_2d(&p.tb, a.w, a.N, a.K, a.ldw, BK, BNP / 2, bf));
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
    p.trace = g_gemm_trace;
    auto kern = a.N == 768 ? gemm2_ln_kernel<T, 3> : gemm2_ln_kernel<T, 2>;
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemP));
    const int units = static_cast<int>(ceil_div(a.M, 2 * BM));
    const int pairs = std::max(1, std::min(units, max_pairs_ln()));
    cudaLaunchAttribute cl;
    cl.id = cudaLaunchAttributeClusterDimension;
    cl.val.clusterDim.x = 2;
    cl.val.clusterDim.y = 1;
    cl.val.clusterDim.z = 1;
    SF_CUDA_TRY(launch_pdl(kern, dim3(2, pairs), dim3(kThreadsP), kSmemP, st, &cl, p));
    SF_LAUNCH_CHECK();
    return SF_OK;
}

}  // namespace

// the row-panel form covers N = 512 and 768 (two or three sub-tiles in the pair's 512 TMEM
// columns); SF_GEMM_LN_CLUSTER=1 selects the cluster form of gemm2_tc.cu instead
bool gemm_ln_panel_supported(const sf_gemm_args& a) {
    const char* e = std::getenv("SF_GEMM_LN_CLUSTER");
    if (e && *e == '1') return false;
    const char* f = std::getenv("SF_GEMM_LN_PANEL");  // test aid: the panel form whenever the shape fits
    const bool force = f && *f == '1';
    // the panel form reads the X panel once per sub-tile: from L2 when K is short (the out-projection,
    // K = 768: 41 vs 43 us cold); at K = 3072 the re-reads come from HBM and the cluster form, whose
    // three pairs read one panel together, is faster (70 vs 84 us; tools/ln_time.py)
    // and the pairs run one panel each: a second panel per pair cannot overlap the first one's
    // normalise pass (T5 cfg4, M = 32768: 87 vs 82 us), so longer M keeps the cluster form
    // Fewer panels than ~3/4 of the pairs would leave SMs idle that the cluster form (one pair per
    // 256 x 256 tile) keeps busy.
    const int64_t panels = ceil_div(a.M, 2 * BM);
    return a.M > BM && (a.N == 512 || a.N == 768) && a.K <= 1024 && a.epi.ln_gamma && a.epi.ln_beta &&
           panels <= max_pairs_ln() && (force || 4 * panels >= 3 * max_pairs_ln());
}

sf_status gemm_ln_panel(const sf_gemm_args& a, cudaStream_t st) {
    return a.dtype == SF_BF16 ? launch_ln_panel<__nv_bfloat16>(a, st) : launch_ln_panel<__half>(a, st);
}

}  // namespace sf
