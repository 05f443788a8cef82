// attn_tc3.cu — block-wise masked attention over HEAD GROUPS on tcgen05 / TMEM / TMA (sm_100a).
// Replaces block_sparse_sdpa (attention.hpp:71-172) for BSR tiles of block_m = 128 query rows,
// block_n in {16, 32, 64}, head_size 64, fp16/bf16, when the slice has >= kHG heads.
//
// The mask is per (row, column), the same for every head (attention.hpp:58-59: the load set is
// mask-level), so a work item here is one 128-row block of kHG = 3 heads of one sequence. One
// CTA per SM; per 64-key step all three heads share:
//   * one K stage and one V stage, gathered with ONE 5-D TMA box per column block that carries
//     the block's rows of all three heads (the fused-QKV activation holds a row's heads side by
//     side, so a box row is 3 x 128 B contiguous). The 5-D map (d, row%8, head, row/8, b) lays the
//     stage out as [8-row group][head][8 rows][128 B]: head t's operand is a uniform run of 1 KB
//     swizzle atoms at stride kHG KB, which the UMMA descriptor expresses with SBO = kHG KB;
//   * the step's packed mask bits (bulk-copied part tiles, producer-filled full / padding rows).
// Per head, TMEM holds S (64 fp32 columns), P (32 columns of packed fp16 pairs) and O (64 fp32
// columns): 3 x 160 of 512 columns. S is single-buffered: the softmax releases S_t(j) as soon as
// it has read it (s_free), so the MMA issuer computes S_t(j+1) under the rest of step j's
// softmax; P_t(j+1) is written once P_t(j).V_j has completed (o_full).
// 512 threads: warps 0..11 softmax — four warps (one per TMEM lane quarter) per head, so every SM
// sub-partition runs three softmax warps (the two-CTA, one-head kernel in attn_tc.cu runs two) —
// warp 12 K producer (Q, K, mask bits), 13 TMEM allocator + MMA issuer, 14 V producer, 15 idle.
// setmaxnreg moves registers from warpgroup 3 (56 each) to the softmax warps (152 each).
// Scheduling, the lazy max update, the exp2 MUFU/FMA split and the deferred epilogue follow
// attn_tc.cu.
#include <algorithm>
#include <cstdlib>
#include <string>

#include "attn_common.cuh"

namespace sf {
unsigned* attn_counter_for(cudaStream_t st);
extern unsigned long long* g_attn_trace;

namespace {

constexpr int kHG = 3;                      // heads per work item
constexpr int kD3 = 64, kNS3 = 64, kBM3 = 128;
constexpr int kSoftWarps = 4 * kHG;         // 12
constexpr int kThreads3 = 128 + 32 * kSoftWarps;  // + warpgroup 3: producer, MMA, two idle warps
constexpr int kWarpProd = kSoftWarps, kWarpMma = kSoftWarps + 1, kWarpVProd = kSoftWarps + 2;
// registers: 128 per thread at launch (4 warps per SM sub-partition); warpgroup 3 drops to 56 and
// the softmax warpgroups take the rest: (3 x 152 + 56) x 32 = 16384 per sub-partition
constexpr int kRegCtl = 56, kRegSoft = 152;
constexpr int kKSt = 3, kVSt = 2;           // K (+ mask bits) and V ring depths
constexpr int kQBytes3 = kHG * kBM3 * kD3 * 2;   // 48 KB, double-buffered across items
constexpr int kKVBytes3 = kHG * kNS3 * kD3 * 2;  // 24 KB per stage
constexpr int kMaskBytes3 = kBM3 * 8;
constexpr uint32_t kHeadCols = 160, kPOff = 64, kOOff = 96;
constexpr int kMaxRB3 = 64;                 // n <= 8192
constexpr float kRescaleLog2_3 = 8.0f;
constexpr int kSmem3 = 1024 + 2 * kQBytes3 + kKSt * kKVBytes3 + kVSt * kKVBytes3 + kKSt * kMaskBytes3 +
                       kMaxRB3 * 4 + (kMaxRB3 + 4) * 4 + 1024;

struct Attn3Params {
    CUtensorMap tq, tk, tv;  // tq: 4-D (d, n, h, b), box {64, 128, kHG, 1}; tk/tv: see kv_grouped
    int32_t n, h, bs, hgroups, units, n_rows, n_items;
    int32_t kv_grouped;      // 1: 5-D (d, n%8, h, n/8, b) maps, one box per column block for all heads
                             // 0: 4-D maps, one {64, bn, 1, 1} box per column block and head
    const int32_t* load_row_ptr;
    const int32_t* load_col_idx;
    const int32_t* load_tile;
    const uint8_t* pool;
    void* o;
    int64_t o_sb, o_sh, o_sn;
    float scale_log2;
    unsigned* work;
    unsigned long long* trace;  // -DSF_ATTN_TRACE builds: per-step events of CTA 0, per-CTA spans
};

#ifdef SF_ATTN_TRACE
#define T3(g, ev)                                                                              \
    do {                                                                                       \
        if (p.trace && blockIdx.x == 0 && (g) < 64) p.trace[(g) * 32 + (ev)] = clock64();      \
    } while (0)
#else
#define T3(g, ev) \
    do {          \
    } while (0)
#endif

// exp2 on the FMA pipe for 1 of every 8 pairs: this kernel is issue-bound (three softmax warps per
// sub-partition), and the polynomial costs ~6.5 issue slots per element against MUFU's 2.5
constexpr int kEmuPairs3 = 1;

// mbarrier wait with a suspend-time hint: a waiting warp sleeps in the barrier unit instead of
// re-issuing the probe, so it does not take issue slots from the two other softmax warps of its
// sub-partition (~70 probe/branch instructions per warp-step without it)
__device__ __forceinline__ void wait3(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
        "@!P1 bra WAIT_%=;\n\t}" ::"r"(tc::smem_u32(bar)),
        "r"(parity), "n"(200)
        : "memory");
}

template <typename T, int BN>
__global__ void __launch_bounds__(kThreads3, 1) attn_tc3_kernel(const __grid_constant__ Attn3Params p) {
    constexpr int G = kNS3 / BN;       // column blocks per 64-key step
    constexpr int TB = kBM3 * BN / 8;  // packed bytes of one part tile
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sQ = sm;                               // [2][kHG][128 x 64]
    unsigned char* sK = sQ + 2 * kQBytes3;                // [kKSt] stages
    unsigned char* sV = sK + kKSt * kKVBytes3;            // [kVSt]
    unsigned char* sMask = sV + kVSt * kKVBytes3;         // [kKSt][128 x 8 B]
    int32_t* s_order = reinterpret_cast<int32_t*>(sMask + kKSt * kMaskBytes3);  // [kMaxRB3]
    int32_t* s_lrp = s_order + kMaxRB3;                                          // [n_rows + 1]
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_lrp + kMaxRB3 + 4);
    uint64_t* q_full = bars;                   // [2]
    uint64_t* q_empty = q_full + 2;            // [2]
    uint64_t* k_full = q_empty + 2;            // [kKSt]  K rows + mask bits landed
    uint64_t* k_empty = k_full + kKSt;         // [kKSt]  all softmax threads hold S of the step
    uint64_t* v_full = k_empty + kKSt;         // [kVSt]
    uint64_t* v_empty = v_full + kVSt;         // [kVSt]  P.V of the step done (all heads)
    uint64_t* s_full = v_empty + kVSt;         // [kHG]   S_t landed
    uint64_t* s_free = s_full + kHG;           // [kHG]   S_t read by head t's softmax
    uint64_t* p_full = s_free + kHG;           // [kHG]   P_t written (and O_t rescaled)
    uint64_t* o_full = p_full + kHG;           // [kHG]   P_t.V done
    uint64_t* item_full = o_full + kHG;        // [kItemRing]
    uint64_t* item_empty = item_full + kItemRing;
    int32_t* s_item = reinterpret_cast<int32_t*>(item_empty + kItemRing);
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(s_item + kItemRing);

#ifdef SF_ATTN_TRACE
    if (p.trace && threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        p.trace[4096 + 2 * blockIdx.x] = t_;
    }
#endif
    pdl_enter();
    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;

    if (static_cast<int>(threadIdx.x) < p.n_rows) {  // row blocks ranked by descending load count
        const int r = threadIdx.x;
        const int Lr = p.load_row_ptr[r + 1] - p.load_row_ptr[r];
        int rank = 0;
        for (int i = 0; i < p.n_rows; ++i) {
            const int Li = p.load_row_ptr[i + 1] - p.load_row_ptr[i];
            rank += (Li > Lr) || (Li == Lr && i < r);
        }
        s_order[rank] = r;
        s_lrp[r] = p.load_row_ptr[r];
        if (r == p.n_rows - 1) s_lrp[p.n_rows] = p.load_row_ptr[p.n_rows];
    }
    if (warp == kWarpProd && lane == 0) {
        tc::prefetch_tmap(&p.tq);
        tc::prefetch_tmap(&p.tk);
        tc::prefetch_tmap(&p.tv);
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&q_full[i], 1);
            tc::mbar_init(&q_empty[i], 1);
        }
        for (int s = 0; s < kKSt; ++s) {
            tc::mbar_init(&k_full[s], 1);
            tc::mbar_init(&k_empty[s], 32 * kSoftWarps);
        }
        for (int s = 0; s < kVSt; ++s) {
            tc::mbar_init(&v_full[s], 1);
            tc::mbar_init(&v_empty[s], 1);
        }
        for (int t = 0; t < kHG; ++t) {
            tc::mbar_init(&s_full[t], 1);
            tc::mbar_init(&s_free[t], 128);
            tc::mbar_init(&p_full[t], 128);
            tc::mbar_init(&o_full[t], 1);
        }
        for (int s = 0; s < kItemRing; ++s) {
            tc::mbar_init(&item_full[s], 1);
            tc::mbar_init(&item_empty[s], 3 + kSoftWarps);  // MMA cursors, V producer, softmax warps
        }
        tc::fence_barrier_init();
    }
    if (warp == kWarpMma) tc::tmem_alloc<512>(tmem_ptr);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;
    const Items items{s_lrp, s_order, p.units, p.n_items, G};
    const ItemFeed feed{s_item, item_full, item_empty};
    // head t's operand inside a Q tile / K or V stage, and the stride of its 8-row atoms
    const uint32_t kv_head_off = p.kv_grouped ? 1024u : static_cast<uint32_t>(kNS3 * kD3 * 2);
    const uint32_t kv_sbo = p.kv_grouped ? 1024u * kHG : 1024u;

    if (warp == kWarpProd) {
        // ------------------------------------------------------------------ producer
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
        uint32_t gk = 0;
        int qi = 0;
        for (uint32_t it = 0;; ++it) {
            int idx = 0;
            if (lane == 0) {
                wait3(&item_empty[it % kItemRing], ((it / kItemRing) & 1) ^ 1);
                if (p.work) {
                    idx = static_cast<int>(atomicAdd(p.work, 1u));
                    if (idx >= p.n_items) idx = -1;
                } else {
                    idx = items.static_idx(static_cast<int>(it));
                }
                s_item[it % kItemRing] = idx;
                tc::mbar_arrive(&item_full[it % kItemRing]);
            }
            idx = __shfl_sync(0xffffffffu, idx, 0);
            if (idx < 0) break;
            int rb, unit, l0, L, nsteps;
            items.decode(idx, rb, unit, l0, L, nsteps);
            if (nsteps == 0) continue;
            const int b = unit / p.hgroups, h0 = (unit % p.hgroups) * kHG;
            if (lane == 0) {
                wait3(&q_empty[qi & 1], ((qi >> 1) & 1) ^ 1);
                tc::mbar_expect_tx(&q_full[qi & 1], kQBytes3);
                tma_load_4d(sQ + (qi & 1) * kQBytes3, &p.tq, &q_full[qi & 1], 0, rb * kBM3, h0, b);
            }
            ++qi;
            for (int c = 0; c < L; c += 32) {
                const int e = c + static_cast<int>(lane);
                const int my_col = p.load_col_idx[l0 + (e < L ? e : 0)];  // pad: valid, fully masked
                const int my_tile = e < L ? p.load_tile[l0 + e] : -2;
                const int j1 = min(nsteps, (c + 32) / G);
                for (int j = c / G; j < j1; ++j) {
                    const int src = j * G + static_cast<int>(lane % G) - c;
                    const int gcol = __shfl_sync(0xffffffffu, my_col, src);
                    const int gtile = __shfl_sync(0xffffffffu, my_tile, src);
                    const int parts = __popc(__ballot_sync(0xffffffffu, lane < G && gtile >= 0));
                    // K + bits
                    const int st = gk % kKSt;
                    if (lane == 0) wait3(&k_empty[st], ((gk / kKSt) & 1) ^ 1);
                    __syncwarp();
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        const int tg = __shfl_sync(0xffffffffu, gtile, gg);
                        if (tg < 0) {
                            const uint32_t fv = tg == -1 ? ~0u : 0u;
                            for (int c16 = static_cast<int>(lane); c16 < TB / 16; c16 += 32)
                                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(
                                                 tc::smem_u32(sMask + st * kMaskBytes3 + gg * TB + 16 * c16)),
                                             "r"(fv)
                                             : "memory");
                        }
                    }
                    __syncwarp();
                    if (lane == 0) tc::mbar_expect_tx(&k_full[st], kKVBytes3 + parts * TB);
                    __syncwarp();
                    if (lane < G) {
                        const int gg = static_cast<int>(lane);
                        unsigned char* dk = sK + st * kKVBytes3 + gg * (kHG * BN * kD3 * 2);
                        if (p.kv_grouped) {
                            tma_load_5d(dk, &p.tk, &k_full[st], 0, 0, h0, gcol * (BN / 8), b);
                        } else {
#pragma unroll
                            for (int t = 0; t < kHG; ++t)
                                tma_load_4d(sK + st * kKVBytes3 + t * (kNS3 * kD3 * 2) + gg * BN * kD3 * 2, &p.tk,
                                            &k_full[st], 0, gcol * BN, h0 + t, b);
                        }
                        if (gtile >= 0)
                            tc::bulk_load(sMask + st * kMaskBytes3 + gg * TB, p.pool + static_cast<int64_t>(gtile) * TB,
                                          TB, &k_full[st]);
                    }
                    if (lane == 0) T3(gk, 2);
                    ++gk;
                }
            }
        }
    } else if (warp == kWarpVProd) {
        // ------------------------------------------------------------------ V producer
        // V has its own warp so the K ring (which gates S) runs ahead independently of the V ring
        // (which P.V drains a step later)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
        uint32_t gv = 0;
        for (uint32_t it = 0;; ++it) {
            const int idx = feed.read(it);
            __syncwarp();
            if (lane == 0) feed.release(it);
            if (idx < 0) break;
            int rb, unit, l0, L, nsteps;
            items.decode(idx, rb, unit, l0, L, nsteps);
            const int b = unit / p.hgroups, h0 = (unit % p.hgroups) * kHG;
            for (int j = 0; j < nsteps; ++j, ++gv) {
                const int e = j * G + static_cast<int>(lane);
                const int gcol = (lane < G && e < L) ? p.load_col_idx[l0 + e] : p.load_col_idx[l0];
                const int sv = gv % kVSt;
                if (lane == 0) {
                    wait3(&v_empty[sv], ((gv / kVSt) & 1) ^ 1);
                    tc::mbar_expect_tx(&v_full[sv], kKVBytes3);
                }
                __syncwarp();
                if (lane < G) {
                    const int gg = static_cast<int>(lane);
                    if (p.kv_grouped) {
                        tma_load_5d(sV + sv * kKVBytes3 + gg * (kHG * BN * kD3 * 2), &p.tv, &v_full[sv], 0, 0, h0,
                                    gcol * (BN / 8), b);
                    } else {
#pragma unroll
                        for (int t = 0; t < kHG; ++t)
                            tma_load_4d(sV + sv * kKVBytes3 + t * (kNS3 * kD3 * 2) + gg * BN * kD3 * 2, &p.tv,
                                        &v_full[sv], 0, gcol * BN, h0 + t, b);
                    }
                }
                if (lane == 0) T3(gv, 3);
            }
        }
    } else if (warp == kWarpMma) {
        // ------------------------------------------------------------------ MMA issuer
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));
        constexpr bool bf = std::is_same<T, __nv_bfloat16>::value;
        constexpr uint32_t idesc_s = tc::idesc_f16(kBM3, kNS3, bf, 0, 0);  // Q (K-major) x K (K-major)
        constexpr uint32_t idesc_o = tc::idesc_f16(kBM3, kD3, bf, 0, 1);   // P (TMEM) x V (MN-major)
        if (tc::elect_one()) {
            Cursor cs, cp;
            cs.next_item(items, feed);
            cp.next_item(items, feed);
            uint32_t gS = 0;
            auto issue_s = [&]() {
                if (cs.j == 0) {
                    wait3(&q_full[cs.qi & 1], (cs.qi >> 1) & 1);
                    tc::fence_after_sync();
                }
                const int st = gS % kKSt;
                wait3(&k_full[st], (gS / kKSt) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int t = 0; t < kHG; ++t) {
                    if (gS > 0) {  // head t's softmax has read S_t of the previous step
                        wait3(&s_free[t], (gS - 1) & 1);
                        tc::fence_after_sync();
                    }
                    const uint32_t q0 = tc::smem_u32(sQ + (cs.qi & 1) * kQBytes3 + t * (kBM3 * kD3 * 2));
                    const uint32_t k0 = tc::smem_u32(sK + st * kKVBytes3) + t * kv_head_off;
#pragma unroll
                    for (int k = 0; k < kD3 / 16; ++k)
                        tc::mma_f16_ss(tmem + kHeadCols * t, tc::sdesc_sw128(q0 + 32 * k), sdesc_sw128_sbo(k0 + 32 * k, kv_sbo),
                                       idesc_s, k != 0);
                    tc::mma_commit(&s_full[t]);
                }
                if (cs.j == cs.ns - 1) tc::mma_commit(&q_empty[cs.qi & 1]);  // last S of the item: Q free
                T3(gS, 0);
                ++gS;
                cs.advance(items, feed);
            };
            auto issue_pv = [&](uint32_t g) {
                const int sv = g % kVSt;
                wait3(&v_full[sv], (g / kVSt) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int t = 0; t < kHG; ++t) {
                    wait3(&p_full[t], g & 1);
                    tc::fence_after_sync();
                    const uint32_t v0 = tc::smem_u32(sV + sv * kKVBytes3) + t * kv_head_off;
                    const uint32_t base = tmem + kHeadCols * t;
#pragma unroll
                    for (int k = 0; k < kNS3 / 16; ++k)  // 16 keys per MMA: two 8-key atoms
                        tc::mma_f16_ts(base + kOOff, base + kPOff + 8 * k, sdesc_sw128_sbo(v0 + 2 * kv_sbo * k, kv_sbo),
                                       idesc_o, (cp.j | k) != 0);
                    tc::mma_commit(&o_full[t]);
                }
                tc::mma_commit(&v_empty[sv]);
                T3(g, 1);
            };
            if (cs.valid) issue_s();
            for (uint32_t g = 0; cp.valid; ++g) {
                // S_{g+1} first (its inputs are ready early: S_g was read at the top of step g),
                // unless it opens a new item, whose Q may still be landing: then P_g.V_g first
                const bool boundary = cs.valid && cs.j == 0;
                if (cs.valid && !boundary) issue_s();
                issue_pv(g);
                if (boundary) issue_s();
                cp.advance(items, feed);
            }
        }
    } else if (warp < kSoftWarps) {
        // ------------------------------------------------------------------ softmax / epilogue
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kRegSoft));
        const uint32_t q = warp & 3;                       // TMEM lane quarter
        const int t = static_cast<int>(warp) >> 2;         // head of the group
        const int r = static_cast<int>(q * 32 + lane);     // query row within the block
        const uint32_t tlane = (q * 32) << 16;
        const uint32_t tS = tmem + kHeadCols * t + tlane;
        const uint32_t tP = tS + kPOff;
        const uint32_t tO = tS + kOOff;
        const float sl2 = p.scale_log2;
        auto epilogue = [&](int rb_, int unit_, float l_, bool have_o) {
            const int b = unit_ / p.hgroups, hh = (unit_ % p.hgroups) * kHG + t;
            const int64_t i = static_cast<int64_t>(rb_) * kBM3 + r;
            const float inv = (have_o && l_ > 0.f) ? 1.f / l_ : 0.f;
            uint4* dst = reinterpret_cast<uint4*>(static_cast<T*>(p.o) + b * p.o_sb + hh * p.o_sh + i * p.o_sn);
            const bool ok = i < p.n && hh < p.h;
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t ov[32];
                if (have_o) {
                    tc::tmem_ld32(tO + 32 * h2, ov);
                    tc::tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) ov[e] = 0u;
                }
                if (ok) {
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        float v[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) v[e] = __uint_as_float(ov[c * 8 + e]) * inv;
                        dst[4 * h2 + c] = make_uint4(pack2<T>(v[0], v[1]), pack2<T>(v[2], v[3]), pack2<T>(v[4], v[5]),
                                                     pack2<T>(v[6], v[7]));
                    }
                }
            }
        };
        bool pend = false;
        int pend_rb = 0, pend_unit = 0;
        float pend_l = 0.f;
        uint32_t g = 0;
        for (uint32_t k = 0;; ++k) {
            const int idx = feed.read(k);
            __syncwarp();
            if (lane == 0) feed.release(k);
            if (idx < 0) break;
            int rb, unit, l0, L, nsteps;
            items.decode(idx, rb, unit, l0, L, nsteps);
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < nsteps; ++j, ++g) {
                const int st = g % kKSt;
                const bool trw = lane == 0 && q == 0;  // events 4 + 4t + {0 top, 1 S seen, 2 max, 3 P arrived}
                if (trw) T3(g, 4 + 4 * t);
                wait3(&k_full[st], (g / kKSt) & 1);
                uint32_t bits[2];
                {
                    const uint32_t mb = tc::smem_u32(sMask + st * kMaskBytes3);
                    if constexpr (BN == 16) {
#pragma unroll
                        for (int w = 0; w < 2; ++w)
                            bits[w] = lds_u16(mb + (2 * w) * TB + r * 2) | (lds_u16(mb + (2 * w + 1) * TB + r * 2) << 16);
                    } else if constexpr (BN == 32) {
#pragma unroll
                        for (int w = 0; w < 2; ++w) bits[w] = lds_u32(mb + w * TB + r * 4);
                    } else {
#pragma unroll
                        for (int w = 0; w < 2; ++w) bits[w] = lds_u32(mb + r * 8 + 4 * w);
                    }
                }
                wait3(&s_full[t], g & 1);
                if (trw) T3(g, 5 + 4 * t);
                tc::fence_after_sync();
                uint32_t raw0[32], raw1[32];
                tc::tmem_ld32(tS, raw0);
                tc::tmem_ld32(tS + 32, raw1);
                bool act[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) act[a] = __any_sync(0xffffffffu, ((bits[a >> 1] >> (16 * (a & 1))) & 0xffffu) != 0);
                tc::tmem_ld_wait();
                tc::fence_before_sync();
                tc::mbar_arrive(&s_free[t]);      // S_t may be overwritten by the next step's MMA
                tc::mbar_arrive(&k_empty[st]);    // this thread is done with K_g's step (S landed) and its bits
                float sr[64];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const uint32_t* rw = a < 2 ? raw0 : raw1;
                    const uint32_t bw = bits[a >> 1];
#ifdef SF_ATTN_SKIPINACT
                    if (!act[a]) continue;  // no valid cell for the warp: never read again
#endif
#ifdef SF_ATTN_SKIPFULL
                    // a 16-column group valid for all 32 rows of the warp needs no selects
                    if (__all_sync(0xffffffffu, ((bw >> (16 * (a & 1))) & 0xffffu) == 0xffffu)) {
#pragma unroll
                        for (int c = 0; c < 16; ++c) sr[16 * a + c] = __uint_as_float(rw[16 * (a & 1) + c]);
                        continue;
                    }
#endif
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const int cc = 16 * (a & 1) + c;
                        sr[16 * a + c] = mask_sel(bw, 1u << cc, __uint_as_float(rw[cc]));
                    }
                }
                float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    if (act[a]) {
#pragma unroll
                        for (int c = 16 * a; c < 16 * a + 16; c += 4)
                            mx4[(c >> 2) & 3] = fmax3(mx4[(c >> 2) & 3], fmax3(sr[c], sr[c + 1], sr[c + 2]), sr[c + 3]);
                    }
                }
                // scale > 0 (checked at the boundary) commutes with max
                const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
                const bool upd = mx > m + kRescaleLog2_3 || (m == -INFINITY && mx > -INFINITY);
                const float m_new = upd ? mx : m;
                const bool resc = upd && m > -INFINITY && j > 0;
                const float resc_a = resc ? ex2(m - m_new) : 1.f;
                m = m_new;
                if (trw) T3(g, 6 + 4 * t);
                // P_g in two 32-key halves (16 packed columns each), stored as they are ready
                float2 rs2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m, -m);
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    uint32_t pk[16];
#pragma unroll
                    for (int a = 2 * hf; a < 2 * hf + 2; ++a) {
                        if (!act[a] || m == -INFINITY) {
#pragma unroll
                            for (int c = 8 * (a & 1); c < 8 * (a & 1) + 8; ++c) pk[c] = 0u;
                            continue;
                        }
#pragma unroll
                        for (int c = 16 * a; c < 16 * a + 16; c += 2) {
                            const float2 arg = ffma2(make_float2(sr[c], sr[c + 1]), sl2x2, negm);
#ifdef SF_EXPERIMENT_NO_EXP  // timing experiment only: exponentials replaced by the argument
                            const float2 pp = arg;
#else
                            const float2 pp = ((c >> 1) & 7) >= 8 - kEmuPairs3 ? ex2_emu2(arg)
                                                                              : make_float2(ex2(arg.x), ex2(arg.y));
#endif
                            rs2[(c >> 1) & 1] = fadd2(rs2[(c >> 1) & 1], pp);
                            pk[(c >> 1) & 15] = pack2<T>(pp.x, pp.y);
                        }
                    }
                    if (hf == 0) {
                        // P_t(g-1).V has completed: P_t is free and O_t holds every earlier step
                        if (g > 0) {
                            wait3(&o_full[t], (g - 1) & 1);
                            tc::fence_after_sync();
                        }
                        if (__any_sync(0xffffffffu, resc)) {  // lazy rescale of O (warp-collective)
#pragma unroll
                            for (int h2 = 0; h2 < 4; ++h2) {
                                uint32_t ov[16];
                                tc::tmem_ld16(tO + 16 * h2, ov);
                                tc::tmem_ld_wait();
#pragma unroll
                                for (int e = 0; e < 16; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * resc_a);
                                tc::tmem_st16(tO + 16 * h2, ov);
                            }
                        }
                    }
                    tc::tmem_st16(tP + 16 * hf, pk);
                }
                l = l * resc_a + ((rs2[0].x + rs2[0].y) + (rs2[1].x + rs2[1].y));
                if (j == 0 && pend) {  // the previous item's output, before P_0.V overwrites O
                    epilogue(pend_rb, pend_unit, pend_l, true);
                    pend = false;
                }
                tc::tmem_st_wait();
                tc::fence_before_sync();
                tc::mbar_arrive(&p_full[t]);
                if (trw) T3(g, 7 + 4 * t);
            }
            if (nsteps > 0) {
                pend = true;
                pend_rb = rb;
                pend_unit = unit;
                pend_l = l;
            } else {
                epilogue(rb, unit, 0.f, false);  // an empty row block: zeros, no TMEM access
            }
        }
        if (pend) {
            wait3(&o_full[t], (g - 1) & 1);
            tc::fence_after_sync();
            epilogue(pend_rb, pend_unit, pend_l, true);
        }
    } else {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kRegCtl));  // idle warp 15
    }
    tc::fence_before_sync();
    __syncthreads();
#ifdef SF_ATTN_TRACE
    if (p.trace && threadIdx.x == 0) {
        unsigned long long t_;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));
        p.trace[4096 + 2 * blockIdx.x + 1] = t_;
    }
#endif
    if (p.work && threadIdx.x == 0) {  // every fetch of this launch is done: the last CTA resets
        if (atomicAdd(p.work + 1, 1u) == gridDim.x - 1) {
            p.work[0] = 0;
            p.work[1] = 0;
        }
    }
    if (warp == kWarpMma) tc::tmem_dealloc<512>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn ||
            q != cudaDriverEntryPointSuccess)
            return nullptr;
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    return encode;
}

CUresult encode_map(CUtensorMap* map, const void* base, bool bf16, int rank, const cuuint64_t* dims,
                    const cuuint64_t* strides, const cuuint32_t* box) {
    auto encode = tmap_encoder();
    if (!encode) return CUDA_ERROR_NOT_FOUND;
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    return encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
}

}  // namespace

bool attn_tc3_eligible(const sf_attn_args& a, const sf_bsr_dev& b) {
    // opt-in (SF_ATTN_HEADGROUP=1): measured at parity with attn_tc.cu standalone and slower inside
    // the layer step, so the one-head kernel stays the default
    const char* e = std::getenv("SF_ATTN_HEADGROUP");
    if (!e || *e != '1') return false;
    return b.block_m == 128 && (b.block_n == 16 || b.block_n == 32 || b.block_n == 64) && a.head_size == kD3 &&
           a.h >= kHG && a.seq_len % 8 == 0 && b.n_rows <= kMaxRB3;
}

sf_status attn_tc3(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st) {
    Attn3Params p{};
    const bool bf = a.dtype == SF_BF16;
    {  // Q: (d, n, h, b), box {64, 128, kHG, 1}
        const cuuint64_t dims[4] = {64, static_cast<cuuint64_t>(a.seq_len), static_cast<cuuint64_t>(a.h),
                                    static_cast<cuuint64_t>(a.bs)};
        const cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.q_sn * 2), static_cast<cuuint64_t>(a.q_sh * 2),
                                       static_cast<cuuint64_t>(a.q_sb * 2)};
        const cuuint32_t box[4] = {64, 128, kHG, 1};
        const CUresult r = encode_map(&p.tq, a.q, bf, 4, dims, strides, box);
        if (r != CUDA_SUCCESS) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled (Q head group) failed: " + std::to_string(int(r)));
    }
    const char* ge = std::getenv("SF_ATTN_KV_PER_HEAD");  // test aid: per-head K/V boxes
    p.kv_grouped = (ge && *ge == '1') ? 0 : 1;
    for (int pass = 0; pass < 2; ++pass) {
        CUresult rk = CUDA_SUCCESS, rv = CUDA_SUCCESS;
        if (p.kv_grouped) {  // (d, n%8, h, n/8, b), box {64, 8, kHG, bn/8, 1}
            const cuuint64_t dims[5] = {64, 8, static_cast<cuuint64_t>(a.h), static_cast<cuuint64_t>(a.seq_len / 8),
                                        static_cast<cuuint64_t>(a.bs)};
            const cuuint64_t strides[4] = {static_cast<cuuint64_t>(a.q_sn * 2), static_cast<cuuint64_t>(a.q_sh * 2),
                                           static_cast<cuuint64_t>(a.q_sn * 16), static_cast<cuuint64_t>(a.q_sb * 2)};
            const cuuint32_t box[5] = {64, 8, kHG, static_cast<cuuint32_t>(b.block_n / 8), 1};
            rk = encode_map(&p.tk, a.k, bf, 5, dims, strides, box);
            rv = encode_map(&p.tv, a.v, bf, 5, dims, strides, box);
        } else {  // (d, n, h, b), box {64, bn, 1, 1}
            const cuuint64_t dims[4] = {64, static_cast<cuuint64_t>(a.seq_len), static_cast<cuuint64_t>(a.h),
                                        static_cast<cuuint64_t>(a.bs)};
            const cuuint64_t strides[3] = {static_cast<cuuint64_t>(a.q_sn * 2), static_cast<cuuint64_t>(a.q_sh * 2),
                                           static_cast<cuuint64_t>(a.q_sb * 2)};
            const cuuint32_t box[4] = {64, static_cast<cuuint32_t>(b.block_n), 1, 1};
            rk = encode_map(&p.tk, a.k, bf, 4, dims, strides, box);
            rv = encode_map(&p.tv, a.v, bf, 4, dims, strides, box);
        }
        if (rk == CUDA_SUCCESS && rv == CUDA_SUCCESS) break;
        if (!p.kv_grouped)
            return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled (K/V) failed: " + std::to_string(int(rk)) + "/" +
                                           std::to_string(int(rv)));
        p.kv_grouped = 0;  // the driver rejected the head-interleaved 5-D map: one box per head
    }
    p.n = a.seq_len;
    p.h = a.h;
    p.bs = a.bs;
    p.hgroups = (a.h + kHG - 1) / kHG;
    p.units = a.bs * p.hgroups;
    p.n_rows = b.n_rows;
    p.n_items = b.n_rows * p.units;
    p.load_row_ptr = b.load_row_ptr;
    p.load_col_idx = b.load_col_idx;
    p.load_tile = b.load_tile;
    p.pool = b.pool;
    p.o = a.o;
    p.o_sb = a.o_sb;
    p.o_sh = a.o_sh;
    p.o_sn = a.o_sn;
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.work = attn_counter_for(st);
    p.trace = g_attn_trace;
    void (*kern)(Attn3Params) = nullptr;
    if (b.block_n == 16) kern = bf ? attn_tc3_kernel<__nv_bfloat16, 16> : attn_tc3_kernel<__half, 16>;
    else if (b.block_n == 32) kern = bf ? attn_tc3_kernel<__nv_bfloat16, 32> : attn_tc3_kernel<__half, 32>;
    else kern = bf ? attn_tc3_kernel<__nv_bfloat16, 64> : attn_tc3_kernel<__half, 64>;
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem3));
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        SF_CUDA_TRY(cudaGetDevice(&dev));
        SF_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    int64_t ctas = std::min<int64_t>(p.n_items, n_sm);  // persistent, one CTA per SM
    if (const char* e = std::getenv("SF_ATTN_MAX_CTAS"))
        ctas = std::max<int64_t>(1, std::min<int64_t>(ctas, std::atoll(e)));
    SF_CUDA_TRY(launch_pdl(kern, dim3(static_cast<unsigned>(ctas)), dim3(kThreads3), kSmem3, st, nullptr, p));
    SF_LAUNCH_CHECK();
    return SF_OK;
}

}  // namespace sf
