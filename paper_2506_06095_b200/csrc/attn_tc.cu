// attn_tc.cu — block-wise masked attention on tcgen05 / TMEM / TMA (sm_100a).
// Replaces block_sparse_sdpa (attention.hpp:71-172) for BSR tiles of block_m = 128 query rows
// and block_n in {16, 32, 64} key columns, head_size 64, fp16/bf16.
//
// Persistent: two CTAs per SM (grid = min(items, 2 x SMs)); a CTA walks its work items (128-row
// block, b*h slice) round-robin, row blocks ranked by descending load count. Every role runs
// ahead across item boundaries (Q is double-buffered, the K/V ring and the S/P/O TMEM buffers
// continue), so the next item's loads and first QK^T overlap the current item's tail. 192 threads:
//   warp 0     producer: Q of each item (128 x 64, 128B-swizzled TMA), then per step the K and V
//              rows of G = 64/block_n load-list column blocks, GATHERED into one contiguous 64-key
//              stage (4-D tensor maps over (d, n, h, b) read Q/K/V in any (b,h,i) stride layout in
//              place, e.g. the fused-QKV activation), the packed bit tiles of the step's PART tiles
//              bulk-copied from the BSR pool; full / padding tiles' bit rows are
//              filled with ones / zeros by the producer lanes (no per-tile branches in the softmax).
//              kStages-deep ring, one transaction barrier per stage.
//   warp 1     TMEM allocator + MMA issuer (one elected thread):
//                S_j = Q K_j^T   tcgen05.mma (SS) M=128 N=64 K=16 x4 -> TMEM S[j%2] (fp32)
//                O  += P_j V_j   tcgen05.mma (TS) M=128 N=64 K=16 x4, A = P_j read straight from
//                                TMEM P[j%2] (fp16 pairs), B = V as an MN-major operand from the
//                                TMA stage; O accumulates in TMEM. No P round trip through smem.
//   warps 2-5  softmax, one thread per query row (TMEM lane), 64 columns per step: tcgen05.ld S_j,
//              masked row max, p = 2^(s*scale*log2e - m) with a lazily updated max m (O is
//              rescaled in TMEM only when the row max grows by more than 2^8, FA4-style, so
//              P <= 256 fits fp16), P_j packed to fp16 and tcgen05.st back into TMEM. 16-column
//              groups masked for all 32 rows of a warp skip their exp/max work.
//   epilogue   (same warps, per item) out = O / l; rows that never saw a valid score are exactly
//              zero (attention.hpp:160-166).
// Only the BSR load set is iterated: empty tiles are never touched (attention.hpp:104-109).
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>

#include "attn_common.cuh"

namespace sf {
namespace {

constexpr int kBM = 128, kD = 64, kNS = 64;  // query rows, head size, keys per step
constexpr int kThreads = 192;                // producer warp, MMA warp, 4 softmax warps
constexpr int kStages = 4;                   // K/V ring depth (two CTAs per SM share 228 KB)
// TMEM columns: S[s] at 64*s (fp32), P[s] at 128 + 32*s (packed fp16 pairs), O at 192. P gets its
// own buffers: an in-flight P.V MMA may still read P_j while the next S MMA is writing, so P
// must not alias S. S_{j+2}'s commit covers P_j V_j, so P[j%2] is free again at step j+2.
constexpr int kSBuf = 2;
constexpr uint32_t kPCol = 128, kOCol = 192;
constexpr int kMaxRowBlocks = 128;           // n <= 8192 at block_m 64
constexpr float kRescaleLog2 = 8.0f;         // lazy-rescale threshold (P <= 2^8)
#ifndef SF_PAIR_KS
#define SF_PAIR_KS 2
#endif
#ifndef SF_PAIR_VS
#define SF_PAIR_VS 3
#endif
#ifndef SF_PAIR_QBUF
#define SF_PAIR_QBUF 1
#endif
#ifndef SF_ONE_KS
#define SF_ONE_KS 4
#endif
#ifndef SF_ONE_VS
#define SF_ONE_VS 4
#endif
#ifndef SF_ONE_QBUF
#define SF_ONE_QBUF 2
#endif

// Geometry per query-block height. BM = 128: one (b, h) slice per work item, M = 128 MMAs.
// BM = 64 ("head pair"): a work item is one 64-row block of TWO heads that share the block's load
// list (the mask is per (row, column), the same for every head). Each head's tiles are M = 64
// MMAs whose accumulators sit in TMEM lanes {32q + 0..15} (head A) and {32q + 16..31} (head B)
// (the cta_group::1 M = 64 layout, lane offset 0 / 16; tools/micro/umma64.cu), so the same 128
// softmax threads serve both heads and every column group is skipped at 16-row granularity.
// 64-row blocks execute a third fewer cells than 128-row blocks on BigBird-like masks.
template <int BM>
struct AttnGeo {
    static constexpr bool kPair = BM == 64;
    static constexpr int kHeads = kPair ? 2 : 1;
    // ring depths: K (with the stage's mask bits), V, and Q buffers. Head pairs hold 32 KB per
    // K + V stage; two CTAs per SM fit 2 K + SF_PAIR_VS V stages with Q single-buffered
    static constexpr int kKS = kPair ? SF_PAIR_KS : SF_ONE_KS;
    static constexpr int kVS = kPair ? SF_PAIR_VS : SF_ONE_VS;
    static constexpr int kQBuf = kPair ? SF_PAIR_QBUF : SF_ONE_QBUF;
    static constexpr int kQB = BM * kD * 2 * kHeads;          // 16 KB either way
    static constexpr int kKVB = kHeads * kNS * kD * 2;         // one stage of K (or V), all heads
    static constexpr int kMaskB = BM * 8;                      // 64 bits per query row per stage
    static constexpr int kSmemG = 1024 + kQBuf * kQB + (kKS + kVS) * kKVB + kKS * kMaskB + (kKS + kVS) * 8 +
                                  kMaxRowBlocks * 4 + (kMaxRowBlocks + 4) * 4 + 512;
};

struct AttnParams {
    CUtensorMap tq, tk, tv;  // 4-D (d, n, h, b) maps; boxes {64,128,1,1} / {64,bn,1,1}
    // head pairs (BM 64) with pair5: 5-D K / V maps (d, row % 8, h, row / 8, b), box {64, 8, 2, bn / 8, 1}:
    // ONE box per column block carries both heads' rows as [row / 8][head][8 rows][128 B], so head
    // t's swizzle atoms sit at t * 1 KB + a 2 KB stride (half the boxes of one box per head)
    CUtensorMap tk2, tv2;
    CUtensorMap tk4, tv4;  // the same maps with a 64-row box: a step whose column blocks are consecutive
    int32_t pair5;
    int32_t run64;         // one head (BM 128): tk4 / tv4 are 4-D maps with a 64-row box
    int32_t n, h, bh, n_rows, n_items;  // bh: work units per row block (slices, or head pairs at BM 64)
    int32_t bh_total;                   // b * h slices
    const int32_t* load_row_ptr;
    const int32_t* load_col_idx;
    const int32_t* load_tile;
    const uint8_t* pool;
    void* o;
    int64_t o_sb, o_sh, o_sn;
    float scale_log2;
    unsigned* work;  // [2]: next item, CTAs done (dynamic schedule), or null (static deal)
    float* lse;      // optional [b*h][n] log2-sum-exp2 per row (null: not written)
    unsigned long long* trace;  // optional clock64 trace of CTA 0 (sf_debug_attn_trace)
};

// clock64 timeline of CTA 0 for tools/attn_trace.py; compiled in only with -DSF_ATTN_TRACE
// (the predicated stores otherwise cost issue slots in the softmax loop)
#ifdef SF_ATTN_TRACE
#define SF_TRACE(j, ev)                                                                   \
    do {                                                                                  \
        if (p.trace && blockIdx.x == 0 && (j) < 64) p.trace[(j) * 32 + (ev)] = clock64(); \
    } while (0)
#else
#define SF_TRACE(j, ev) \
    do {                \
    } while (0)
#endif

template <typename T, int BN, int BM>
__global__ void __launch_bounds__(kThreads, 2) attn_tc_kernel(const __grid_constant__ AttnParams p) {
    using Geo = AttnGeo<BM>;
    constexpr bool kPair = Geo::kPair;
    constexpr int kKS = Geo::kKS, kVS = Geo::kVS, kQBuf = Geo::kQBuf;
    constexpr int kQBytes = Geo::kQB;
    constexpr int kKVBytes = Geo::kKVB;
    constexpr int kMaskBytes = Geo::kMaskB;
    constexpr int G = kNS / BN;          // column tiles gathered per 64-key step
    constexpr int TB = BM * BN / 8;      // packed bytes of one part tile (pool stride)
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    unsigned char* sQ = sm;                               // [2] Q tiles (double-buffered across items)
    unsigned char* sK = sQ + kQBuf * kQBytes;
    unsigned char* sV = sK + kKS * kKVBytes;
    unsigned char* sMask = sV + kVS * kKVBytes;            // [kKS][BM * 8 B]: packed part-tile bits
    int32_t* s_order = reinterpret_cast<int32_t*>(sMask + kKS * kMaskBytes) + 2 * (kKS + kVS);  // [kMaxRowBlocks]
    // load_row_ptr cached in smem: item decodes at item boundaries read no global memory
    int32_t* s_lrp = s_order + kMaxRowBlocks;  // [n_rows + 1]
    uint64_t* bars = reinterpret_cast<uint64_t*>(s_lrp + kMaxRowBlocks + 4);
    uint64_t* q_full = bars;                  // [2]
    uint64_t* q_empty = q_full + 2;           // [2]
    // K (with the stage's bit rows) and V have separate barriers: a K slot is
    // released as soon as the softmax holds S of that step (and read its bits), a V slot when
    // P.V of that step is done, so K loads run about a step further ahead than V loads
    uint64_t* k_full = q_empty + 2;           // [kKS]
    uint64_t* k_empty = k_full + kKS;         // [kKS] (128 softmax arrivals)
    uint64_t* v_full = k_empty + kKS;         // [kVS]
    uint64_t* v_empty = v_full + kVS;         // [kVS]
    uint64_t* s_full = v_empty + kVS;         // [kSBuf]
    uint64_t* p_full = s_full + kSBuf;        // [kSBuf]
    uint64_t* o_full = p_full + kSBuf;        // [2]: P.V step g completes o_full[g&1] (parity waits are
                                              // unambiguous only within one phase of lag)
    uint64_t* item_full = o_full + 2;               // [kItemRing]
    uint64_t* item_empty = item_full + kItemRing;  // [kItemRing]
    int32_t* s_item = reinterpret_cast<int32_t*>(item_empty + kItemRing);  // [kItemRing]
    uint32_t* tmem_ptr = reinterpret_cast<uint32_t*>(s_item + kItemRing);

    const uint32_t warp = tc::warp_id();
    const uint32_t lane = threadIdx.x & 31;

    // row blocks ranked by descending load count (ties by index)
    if (static_cast<int>(threadIdx.x) < p.n_rows) {
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
    if (warp == 0 && lane == 0) {
        tc::prefetch_tmap(&p.tq);
        tc::prefetch_tmap(&p.tk);
        tc::prefetch_tmap(&p.tv);
        if (kPair && p.pair5) {
            tc::prefetch_tmap(&p.tk2);
            tc::prefetch_tmap(&p.tv2);
        }
        if ((kPair && p.pair5 == 2) || (!kPair && p.run64)) {
            tc::prefetch_tmap(&p.tk4);
            tc::prefetch_tmap(&p.tv4);
        }
        for (int i = 0; i < 2; ++i) {
            tc::mbar_init(&q_full[i], 1);
            tc::mbar_init(&q_empty[i], 1);
            tc::mbar_init(&o_full[i], 1);
        }
        for (int s = 0; s < kKS; ++s) {
            tc::mbar_init(&k_full[s], 1);
            tc::mbar_init(&k_empty[s], 128);
        }
        for (int s = 0; s < kVS; ++s) {
            tc::mbar_init(&v_full[s], 1);
            tc::mbar_init(&v_empty[s], 1);
        }
        for (int s = 0; s < kSBuf; ++s) {
            tc::mbar_init(&s_full[s], 1);
            tc::mbar_init(&p_full[s], 128);
        }
        for (int s = 0; s < kItemRing; ++s) {
            tc::mbar_init(&item_full[s], 1);
            tc::mbar_init(&item_empty[s], 6);
        }
        tc::fence_barrier_init();
    }
    if (warp == 1) tc::tmem_alloc<256>(tmem_ptr);
    tc::fence_before_sync();
    __syncthreads();
    tc::fence_after_sync();
    const uint32_t tmem = *tmem_ptr;
    // the prologue above reads only the BSR (not written by the stream predecessor): it overlaps the
    // predecessor's tail under PDL; Q/K/V and O are touched only after this wait
    pdl_enter();
    const uint32_t tO = tmem + kOCol;
    const Items items{s_lrp, s_order, p.bh, p.n_items, G};
    const ItemFeed feed{s_item, item_full, item_empty};

    if (warp == 0) {
        // ------------------------------------------------------------------ producer (one warp)
        // Lanes fetch 32 load-list entries at a time; lane 0 issues the TMA for each step.
        uint32_t g = 0;  // step counters unsigned: the ring index / phase math is one LOP3 each
        int qi = 0;
        for (uint32_t it = 0;; ++it) {
            int idx = 0;
            if (lane == 0) {  // pick and publish the CTA's next item
                tc::mbar_wait(&item_empty[it % kItemRing], ((it / kItemRing) & 1) ^ 1);
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
            int rb, bh, l0, L, nsteps;
            items.decode(idx, rb, bh, l0, L, nsteps);
            if (nsteps == 0) continue;
            // the unit's heads: one slice, or the pair (2u, 2u+1) (an odd last pair repeats head A)
            int hb[2], hh2[2];
#pragma unroll
            for (int t = 0; t < Geo::kHeads; ++t) {
                int s_ = kPair ? 2 * bh + t : bh;
                if (s_ >= p.bh_total) s_ = 2 * bh;
                hb[t] = s_ / p.h;
                hh2[t] = s_ % p.h;
            }
            if (lane == 0) {
                tc::mbar_wait(&q_empty[qi % kQBuf], ((qi / kQBuf) & 1) ^ 1);
                tc::mbar_expect_tx(&q_full[qi % kQBuf], kQBytes);
                if (kPair && p.pair5) {
                    tma_load_4d(sQ + (qi % kQBuf) * kQBytes, &p.tq, &q_full[qi % kQBuf], 0, rb * BM, hh2[0], hb[0]);
                } else {
#pragma unroll
                    for (int t = 0; t < Geo::kHeads; ++t)
                        tma_load_4d(sQ + (qi % kQBuf) * kQBytes + t * (BM * kD * 2), &p.tq, &q_full[qi % kQBuf], 0, rb * BM,
                                    hh2[t], hb[t]);
                }
            }
            ++qi;
            for (int c = 0; c < L; c += 32) {
                const int e = c + static_cast<int>(lane);
                const int my_col = p.load_col_idx[l0 + (e < L ? e : 0)];  // pad: valid, fully masked
                const int my_tile = e < L ? p.load_tile[l0 + e] : -2;
                const int j1 = min(nsteps, (c + 32) / G);
                for (int j = c / G; j < j1; ++j, ++g) {
                    const int st = g % kKS, sv = g % kVS;
                    // lane gg < G owns column block gg of the step: its K / V boxes and bit tile
                    // are issued from G lanes in parallel (one issuing thread sustains only one
                    // 16-row TMA box per ~160 cycles; tools/micro/tma_gather.cu)
                    const int src = j * G + static_cast<int>(lane % G) - c;
                    const int gcol = __shfl_sync(0xffffffffu, my_col, src);
                    const int gtile = __shfl_sync(0xffffffffu, my_tile, src);
                    const int parts = __popc(__ballot_sync(0xffffffffu, lane < G && gtile >= 0));
                    // a step over G consecutive column blocks (band interiors) loads each tensor with
                    // ONE 64-row box instead of G: the same bytes land at the same stage addresses
                    const int gcol0 = __shfl_sync(0xffffffffu, gcol, 0);
                    const bool run = G > 1 && (kPair ? p.pair5 == 2 : p.run64 != 0) &&
                                     __all_sync(0xffffffffu, lane >= G || gcol == gcol0 + static_cast<int>(lane));
                    const uint32_t ph = ((g / kKS) & 1) ^ 1, phv = ((g / kVS) & 1) ^ 1;
                    if (lane == 0) {
                        SF_TRACE(g, 4);
                        tc::mbar_wait(&k_empty[st], ph);
                        SF_TRACE(g, 5);
                    }
                    __syncwarp();
                    // the stage's bit rows of full (all ones) and padding (zero) tiles are written
                    // here, so the softmax reads every tile's bits the same way, without branches;
                    // part tiles' rows arrive by bulk copy from the pool
#pragma unroll
                    for (int gg = 0; gg < G; ++gg) {
                        const int tg = __shfl_sync(0xffffffffu, gtile, gg);
                        if (tg < 0) {
                            const uint32_t fv = tg == -1 ? ~0u : 0u;
                            for (int c16 = static_cast<int>(lane); c16 < TB / 16; c16 += 32)
                                asm volatile("st.shared.v4.b32 [%0], {%1, %1, %1, %1};" ::"r"(
                                                 tc::smem_u32(sMask + st * kMaskBytes + gg * TB + 16 * c16)),
                                             "r"(fv)
                                             : "memory");
                        }
                    }
                    __syncwarp();
                    if (lane == 0) tc::mbar_expect_tx(&k_full[st], kKVBytes + parts * TB);  // release: the filled bit rows
                    __syncwarp();
                    if (lane < G) {
                        const int gg = static_cast<int>(lane);
                        if (kPair && p.pair5) {
                            if (!run)
                                tma_load_5d(sK + st * kKVBytes + gg * BN * kD * 2 * 2, &p.tk2, &k_full[st], 0, 0, hh2[0],
                                            gcol * (BN / 8), hb[0]);
                            else if (gg == 0)
                                tma_load_5d(sK + st * kKVBytes, &p.tk4, &k_full[st], 0, 0, hh2[0], gcol0 * (BN / 8), hb[0]);
                        } else if (run) {
                            if (gg == 0) tma_load_4d(sK + st * kKVBytes, &p.tk4, &k_full[st], 0, gcol0 * BN, hh2[0], hb[0]);
                        } else {
#pragma unroll
                            for (int t = 0; t < Geo::kHeads; ++t)  // head t's 64 keys at t * 8 KB
                                tma_load_4d(sK + st * kKVBytes + t * (kNS * kD * 2) + gg * BN * kD * 2, &p.tk, &k_full[st],
                                            0, gcol * BN, hh2[t], hb[t]);
                        }
                        if (gtile >= 0)
                            tc::bulk_load(sMask + st * kMaskBytes + gg * TB, p.pool + static_cast<int64_t>(gtile) * TB, TB,
                                          &k_full[st]);
                    }
                    if (lane == 0) {
                        SF_TRACE(g, 7);
                        tc::mbar_wait(&v_empty[sv], phv);
                        SF_TRACE(g, 11);
                        tc::mbar_expect_tx(&v_full[sv], kKVBytes);
                    }
                    __syncwarp();
                    if (lane < G) {
                        const int gg = static_cast<int>(lane);
                        if (kPair && p.pair5) {
                            if (!run)
                                tma_load_5d(sV + sv * kKVBytes + gg * BN * kD * 2 * 2, &p.tv2, &v_full[sv], 0, 0, hh2[0],
                                            gcol * (BN / 8), hb[0]);
                            else if (gg == 0)
                                tma_load_5d(sV + sv * kKVBytes, &p.tv4, &v_full[sv], 0, 0, hh2[0], gcol0 * (BN / 8), hb[0]);
                        } else if (run) {
                            if (gg == 0) tma_load_4d(sV + sv * kKVBytes, &p.tv4, &v_full[sv], 0, gcol0 * BN, hh2[0], hb[0]);
                        } else {
#pragma unroll
                            for (int t = 0; t < Geo::kHeads; ++t)
                                tma_load_4d(sV + sv * kKVBytes + t * (kNS * kD * 2) + gg * BN * kD * 2, &p.tv, &v_full[sv],
                                            0, gcol * BN, hh2[t], hb[t]);
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------------ MMA issuer
        constexpr bool bf = std::is_same<T, __nv_bfloat16>::value;
        constexpr uint32_t idesc_s = tc::idesc_f16(BM, kNS, bf, 0, 0);  // Q (K-major) x K (K-major)
        constexpr uint32_t idesc_o = tc::idesc_f16(BM, kD, bf, 0, 1);   // P (TMEM) x V (MN-major)
        if (tc::elect_one()) {
            Cursor cs, cp;
            cs.next_item(items, feed);
            cp.next_item(items, feed);
            uint32_t gS = 0;
            auto issue_s = [&]() {
                if (cs.j == 0) {
                    tc::mbar_wait(&q_full[cs.qi % kQBuf], (cs.qi / kQBuf) & 1);
                    tc::fence_after_sync();
                }
                const int s = gS % kKS;
                SF_TRACE(gS, 13);
                tc::mbar_wait(&k_full[s], (gS / kKS) & 1);
                SF_TRACE(gS, 14);
                tc::fence_after_sync();
#pragma unroll
                for (int t = 0; t < Geo::kHeads; ++t) {  // head t: M = BM rows at TMEM lane offset 16t
                    const uint32_t q0 = tc::smem_u32(sQ + (cs.qi % kQBuf) * kQBytes + t * (BM * kD * 2));
                    const bool p5 = kPair && p.pair5;
                    const uint32_t k0 = tc::smem_u32(sK + s * kKVBytes) + (p5 ? 1024u * t : static_cast<uint32_t>(t * (kNS * kD * 2)));
                    const uint32_t kv_sbo = p5 ? 2048u : 1024u;
#pragma unroll
                    for (int k = 0; k < kD / 16; ++k)
                        tc::mma_f16_ss(tmem + ((16u * t) << 16) + 64 * (gS % kSBuf), tc::sdesc_sw128(q0 + 32 * k),
                                       sdesc_sw128_sbo(k0 + 32 * k, kv_sbo), idesc_s, k != 0);
                }
                tc::mma_commit(&s_full[gS % kSBuf]);
                if (cs.j == cs.ns - 1) tc::mma_commit(&q_empty[cs.qi % kQBuf]);  // last S of the item: Q free
                ++gS;
                cs.advance(items, feed);
            };
            for (int j = 0; j < kSBuf && cs.valid; ++j) issue_s();
            for (uint32_t g = 0; cp.valid; ++g) {
                const int s = g % kVS;
                const int sb = g % kSBuf;
                tc::mbar_wait(&p_full[sb], (g / kSBuf) & 1);  // P_g in TMEM (S_g consumed), O rescaled
                SF_TRACE(g, 8);
                tc::mbar_wait(&v_full[s], (g / kVS) & 1);
                tc::fence_after_sync();
#pragma unroll
                for (int t = 0; t < Geo::kHeads; ++t) {
                    const bool p5 = kPair && p.pair5;
                    const uint32_t v0 = tc::smem_u32(sV + s * kKVBytes) + (p5 ? 1024u * t : static_cast<uint32_t>(t * (kNS * kD * 2)));
                    const uint32_t kv_sbo = p5 ? 2048u : 1024u;
                    const uint32_t lo = (16u * t) << 16;
#pragma unroll
                    for (int k = 0; k < kNS / 16; ++k)  // P_g: 64 keys = 32 packed columns, 8 per K=16
                        tc::mma_f16_ts(tO + lo, tmem + lo + kPCol + 32 * sb + 8 * k, sdesc_sw128_sbo(v0 + 2 * kv_sbo * k, kv_sbo),
                                       idesc_o, (cp.j | k) != 0);
                }
                tc::mma_commit(&o_full[g & 1]);
                tc::mma_commit(&v_empty[s]);
                SF_TRACE(g, 9);
                if (cs.valid) issue_s();
                SF_TRACE(g, 10);
                cp.advance(items, feed);
            }
        }
    } else {
        // ------------------------------------------------------------------ softmax / epilogue
        // One thread per query row (TMEM lane), all 64 columns of the step.
        const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
        // the query row this thread (TMEM lane) holds: BM 128 -> 32q + lane; head pairs (BM 64)
        // -> row 16q + lane%16 of head lane/16 (the M = 64 accumulator layout)
        const int r = kPair ? static_cast<int>(q * 16 + (lane & 15)) : static_cast<int>(q * 32 + lane);
        const int my_head = kPair ? static_cast<int>(lane >> 4) : 0;
        const uint32_t trow = tmem + ((q * 32) << 16);
        const float sl2 = p.scale_log2;
        // ---- epilogue of an item: out = O / l; rows without a valid column stay zero
        // (attention.hpp:160-166). It is DEFERRED: the item's last P.V is still running when its
        // last P is published, so the warps first compute the next item's step-0 probabilities and
        // only then wait for that P.V and read O, just before publishing P_0 of the next item (whose
        // P.V overwrites O). The wait for the last P.V hides behind a softmax step.
        auto epilogue = [&](int rb_, int bh_, float l_, float m_, bool have_o, uint32_t g_last) {
            const int slice = kPair ? 2 * bh_ + my_head : bh_;
            const bool slice_ok = slice < p.bh_total;  // an odd last head pair has no head B
            const int b = slice_ok ? slice / p.h : 0, hh = slice_ok ? slice % p.h : 0;
            const int64_t i = static_cast<int64_t>(rb_) * BM + r;
            // optional per-row log2-sum-exp2 of the scaled scores (m + log2 l), for merging partial
            // attentions over disjoint key sets (sf_mha_strided); -inf for rows without a valid key
            if (p.lse && slice_ok && i < p.n)
                p.lse[static_cast<int64_t>(slice) * p.n + i] = (have_o && l_ > 0.f) ? m_ + __log2f(l_) : -INFINITY;
            if (have_o) {
                tc::mbar_wait(&o_full[g_last & 1], (g_last >> 1) & 1);
                tc::fence_after_sync();
            }
            const float inv = (have_o && l_ > 0.f) ? 1.f / l_ : 0.f;
            uint4* dst = reinterpret_cast<uint4*>(static_cast<T*>(p.o) + b * p.o_sb + hh * p.o_sh + i * p.o_sn);
#pragma unroll
            for (int h2 = 0; h2 < 2; ++h2) {
                uint32_t ov[32];
                if (have_o) {
                    tc::tmem_ld32(tO + ((q * 32) << 16) + 32 * h2, ov);
                    tc::tmem_ld_wait();
                } else {
#pragma unroll
                    for (int e = 0; e < 32; ++e) ov[e] = 0u;
                }
                if (i < p.n && slice_ok) {
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
            tc::fence_before_sync();  // O reads ordered before the next item's first P.V (p_full)
        };
        bool pend = false;  // an item whose epilogue is deferred into the next item's step 0
        int pend_rb = 0, pend_bh = 0;
        float pend_l = 0.f, pend_m = 0.f;
        uint32_t pend_g = 0;
        uint32_t g = 0;
        for (uint32_t k = 0;; ++k) {
            const int idx = feed.read(k);
            __syncwarp();
            if (lane == 0) feed.release(k);
            if (idx < 0) break;
            int rb, bh, l0, L, nsteps;
            items.decode(idx, rb, bh, l0, L, nsteps);
            float m = -INFINITY, l = 0.f;
            for (int j = 0; j < nsteps; ++j, ++g) {
                const int st = g % kKS;
                const int sb = g % kSBuf;
                const bool tr = warp == 2 && lane == 0 && k == 0;
                const bool trw = lane == 0;  // per-warp events 16 + 4 (warp - 2) + {0..3}, by CTA step g
                if (tr) SF_TRACE(j, 0);
                if (trw) SF_TRACE(g, 16 + 4 * (warp - 2));
                tc::mbar_wait(&k_full[st], (g / kKS) & 1);
                if (tr) SF_TRACE(j, 1);
                // this row's 64 mask bits (the producer staged every tile's rows: full -> ones,
                // part -> its pool rows, padding -> 0)
                uint32_t bits[2];
                {
                    const uint32_t mb = tc::smem_u32(sMask + st * kMaskBytes);
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
                tc::mbar_wait(&s_full[sb], (g / kSBuf) & 1);
                if (tr) SF_TRACE(j, 2);
                if (trw) SF_TRACE(g, 17 + 4 * (warp - 2));
                tc::fence_after_sync();
                uint32_t raw0[32], raw1[32];
                tc::tmem_ld32(trow + 64 * sb, raw0);
                tc::tmem_ld32(trow + 64 * sb + 32, raw1);
                bool act[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) act[a] = __any_sync(0xffffffffu, ((bits[a >> 1] >> (16 * (a & 1))) & 0xffffu) != 0);
                tc::tmem_ld_wait();
                tc::mbar_arrive(&k_empty[st]);  // S_g is here (so its MMA read K_g) and the bits were read
                // masked cells -> -inf once: they drop out of the max and 2^(-inf) = 0 later
                float sr[64];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    const uint32_t* rw = a < 2 ? raw0 : raw1;
                    const uint32_t bw = bits[a >> 1];
#pragma unroll
                    for (int c = 0; c < 16; ++c) {
                        const int cc = 16 * (a & 1) + c;
#ifdef SF_EXPERIMENT_NO_MASK  // timing experiment only
                        sr[16 * a + c] = __uint_as_float(rw[cc]) + 0.f * bw;
#else
                        sr[16 * a + c] = mask_sel(bw, 1u << cc, __uint_as_float(rw[cc]));
#endif
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
                // max of the raw scores, then scaled: scale > 0 commutes with max (log2 domain)
                const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3])) * sl2;
                if (tr) SF_TRACE(j, 3);
                if (trw) SF_TRACE(g, 18 + 4 * (warp - 2));
                // lazy max update: rescale O / l only when the max grows by > 2^8 (or first time).
                // tcgen05.ld/st are warp-collective: the rescale is voted warp-uniformly and lanes
                // that do not need it scale by 1.
                const bool upd = mx > m + kRescaleLog2 || (m == -INFINITY && mx > -INFINITY);
                const float m_new = upd ? mx : m;
                const bool resc = upd && m > -INFINITY && j > 0;
                if (__any_sync(0xffffffffu, resc)) {
                    const float a = resc ? ex2(m - m_new) : 1.f;
                    l *= a;
                    tc::mbar_wait(&o_full[(g - 1) & 1], ((g - 1) >> 1) & 1);  // P_{g-1} V_{g-1} landed in O
                    tc::fence_after_sync();
#pragma unroll
                    for (int h2 = 0; h2 < 2; ++h2) {
                        uint32_t ov[32];
                        tc::tmem_ld32(tO + ((q * 32) << 16) + 32 * h2, ov);
                        tc::tmem_ld_wait();
#pragma unroll
                        for (int e = 0; e < 32; ++e) ov[e] = __float_as_uint(__uint_as_float(ov[e]) * a);
                        tc::tmem_st32(tO + ((q * 32) << 16) + 32 * h2, ov);
                    }
                }
                m = m_new;
                uint32_t pk[32];
                float2 rs2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
                const float2 sl2x2 = make_float2(sl2, sl2), negm = make_float2(-m, -m);
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    if (!act[a] || m == -INFINITY) {
#pragma unroll
                        for (int c = 8 * a; c < 8 * a + 8; ++c) pk[c] = 0u;
                        continue;
                    }
#pragma unroll
                    for (int c = 16 * a; c < 16 * a + 16; c += 2) {
                        const float2 arg = ffma2(make_float2(sr[c], sr[c + 1]), sl2x2, negm);
                        // the last kEmuPairs pairs of each group on the FMA pipe, the rest on MUFU
#ifdef SF_EXPERIMENT_NO_EXP  // timing experiment only: exponentials replaced by the argument
                        const float2 pp = arg;
#else
                        const float2 pp = ((c >> 1) & 7) >= 8 - kEmuPairs ? ex2_emu2(arg)
                                                                          : make_float2(ex2(arg.x), ex2(arg.y));
#endif
                        rs2[(c >> 1) & 1] = fadd2(rs2[(c >> 1) & 1], pp);
                        pk[c >> 1] = pack2<T>(pp.x, pp.y);
                    }
                }
                l += (rs2[0].x + rs2[0].y) + (rs2[1].x + rs2[1].y);
                if (j == 0 && pend) {  // the previous item's O is read before P_0 lets P.V overwrite it
                    epilogue(pend_rb, pend_bh, pend_l, pend_m, true, pend_g);
                    pend = false;
                }
                // P_g (64 keys = 32 packed columns) into P[sb] in TMEM
                tc::tmem_st32(trow + kPCol + 32 * sb, pk);
                tc::tmem_st_wait();
                tc::fence_before_sync();
                tc::mbar_arrive(&p_full[sb]);
                if (tr) SF_TRACE(j, 6);
                if (trw) SF_TRACE(g, 19 + 4 * (warp - 2));
            }
            if (nsteps > 0) {
                pend = true;
                pend_rb = rb;
                pend_bh = bh;
                pend_l = l;
                pend_m = m;
                pend_g = g - 1;
            } else {
                epilogue(rb, bh, 0.f, 0.f, false, 0);  // an empty row block: zeros, no TMEM access
            }
        }
        if (pend) epilogue(pend_rb, pend_bh, pend_l, pend_m, true, pend_g);
    }
    tc::fence_before_sync();
    __syncthreads();
    if (p.work && threadIdx.x == 0) {  // every fetch of this launch is done: the last CTA resets
        if (atomicAdd(p.work + 1, 1u) == gridDim.x - 1) {
            p.work[0] = 0;
            p.work[1] = 0;
        }
    }
    if (warp == 1) tc::tmem_dealloc<256>(tmem);
}

// 4-D map over (d, n, h, b) with element strides (1, sn, sh, sb); box {64, rows, 1, 1}, SW128.
sf_status make_tmap_4d(CUtensorMap* map, const void* base, int n, int h, int bs, int64_t sn, int64_t sh, int64_t sb,
                       uint32_t box_rows, bool bf16, uint32_t box_heads = 1) {
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
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(kD), box_rows, box_heads, 1};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    CUresult r = encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled (4d) failed: " + std::to_string(int(r)));
    return SF_OK;
}

// Head-pair K / V map: 5-D (d, row % 8, h, row / 8, b) with byte strides (sn, sh, 8 sn, sb) (x 2 B),
// box {64, 8, 2, bn / 8, 1}, SW128 (n % 8 == 0).
sf_status make_tmap_pair5(CUtensorMap* map, const void* base, int n, int h, int bs, int64_t sn, int64_t sh, int64_t sb,
                          uint32_t bn, bool bf16) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        cudaDriverEntryPointQueryResult q{};
        void* fn = nullptr;
        SF_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
        if (!fn || q != cudaDriverEntryPointSuccess) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled unavailable");
        encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    const cuuint64_t dims[5] = {static_cast<cuuint64_t>(kD), 8, static_cast<cuuint64_t>(h), static_cast<cuuint64_t>(n / 8),
                                static_cast<cuuint64_t>(bs)};
    const cuuint64_t strides[4] = {static_cast<cuuint64_t>(sn * 2), static_cast<cuuint64_t>(sh * 2),
                                   static_cast<cuuint64_t>(sn * 16), static_cast<cuuint64_t>(sb * 2)};
    const cuuint32_t box[5] = {static_cast<cuuint32_t>(kD), 8, 2, bn / 8, 1};
    const cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = encode(map, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 5,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(SF_CUDA_ERROR, "cuTensorMapEncodeTiled (head pair) failed: " + std::to_string(int(r)));
    return SF_OK;
}

}  // namespace

unsigned long long* g_attn_trace = nullptr;

// The dynamic schedule's work counter (next item, CTAs done). The last CTA of a launch resets it,
// so a counter is reusable by any later launch ordered after it, never by a concurrent one:
//  * eager launches take the counter of their (device, stream): launches on one stream are
//    ordered (PDL included: the next launch's griddepcontrol.wait follows this one's reset);
//  * a launch captured into a CUDA graph takes a PRIVATE counter, used by nothing else: replays
//    of one graph exec are ordered, but graphs captured on one stream may be replayed
//    concurrently on different streams, and next to eager launches on their capture stream.
// Counters come from a per-device pool of zeroed pairs created outside any capture (by
// sf_bsr_build, or by the first eager attention launch); with the pool spent the launch uses the
// static deal. SF_ATTN_STATIC=1 forces the static deal.
namespace {
constexpr int kCounterPool = 8192;
std::mutex g_counter_mu;
std::map<int, std::pair<unsigned*, int>> g_counter_pool;                // device -> (pool, next free)
std::map<std::pair<int, cudaStream_t>, unsigned*> g_counters;          // (device, stream) -> counter

void reserve_pool_locked(int dev, cudaStream_t st) {  // st: not capturing
    if (g_counter_pool.count(dev)) return;
    unsigned* w = nullptr;
    if (cudaMalloc(&w, kCounterPool * 2 * sizeof(unsigned)) != cudaSuccess ||
        cudaMemsetAsync(w, 0, kCounterPool * 2 * sizeof(unsigned), st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess) {
        cudaGetLastError();
        if (w) cudaFree(w);
        return;
    }
    g_counter_pool.emplace(dev, std::make_pair(w, 0));
}

unsigned* take_counter_locked(int dev) {
    const auto pool = g_counter_pool.find(dev);
    if (pool == g_counter_pool.end() || pool->second.second >= kCounterPool) return nullptr;
    return pool->second.first + 2 * pool->second.second++;
}

bool attn_force_static() {
    const char* e = std::getenv("SF_ATTN_STATIC");  // read per launch so tests can switch it
    return e && *e == '1';
}

unsigned* attn_work_counter(cudaStream_t st) {
    if (attn_force_static()) return nullptr;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(g_counter_mu);
    if (cs != cudaStreamCaptureStatusNone) return take_counter_locked(dev);  // private to this graph node
    const auto key = std::make_pair(dev, st);
    const auto it = g_counters.find(key);
    if (it != g_counters.end()) return it->second;
    reserve_pool_locked(dev, st);
    unsigned* w = take_counter_locked(dev);
    if (w) g_counters.emplace(key, w);
    return w;
}
}  // namespace

unsigned* attn_counter_for(cudaStream_t st) { return attn_work_counter(st); }
bool attn_tc3_eligible(const sf_attn_args& a, const sf_bsr_dev& b);
sf_status attn_tc3(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st);

// called by sf_bsr_build (never inside a capture: it reads the output sizes back)
void attn_reserve_counters(cudaStream_t st) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lock(g_counter_mu);
    reserve_pool_locked(dev, st);
}

sf_status attn_tc(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st, bool probe_only, float* lse) {
    const bool shape_ok = (b.block_m == 128 || b.block_m == 64) && (b.block_n == 16 || b.block_n == 32 || b.block_n == 64) &&
                          a.head_size == kD && b.n_rows <= kMaxRowBlocks;
    const bool layout_ok = a.q_sn % 8 == 0 && a.q_sh % 8 == 0 && a.q_sb % 8 == 0 && a.o_sn % 8 == 0 &&
                           a.o_sh % 8 == 0 && a.o_sb % 8 == 0 &&
                           ((reinterpret_cast<uintptr_t>(a.q) | reinterpret_cast<uintptr_t>(a.k) |
                             reinterpret_cast<uintptr_t>(a.v) | reinterpret_cast<uintptr_t>(a.o)) & 15) == 0;
    if (!shape_ok || !layout_ok)
        return fail(SF_PLAN_ERROR, "tcgen05 attention needs block_m 64/128, block_n 16/32/64, head_size 64, "
                                   "16-byte aligned strides");
    if (probe_only) return SF_OK;
    if (b.tile_bytes != b.block_m * b.block_n / 8) return fail(SF_PLAN_ERROR, "BSR tile_bytes does not match block shape");
    // head groups sharing one mask per work item (attn_tc3.cu) where the slice has >= 3 heads
    if (!lse && attn_tc3_eligible(a, b)) return attn_tc3(a, b, st);
    AttnParams p{};
    const bool bf = a.dtype == SF_BF16;
    SF_TRY(make_tmap_4d(&p.tq, a.q, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_m, bf));
    SF_TRY(make_tmap_4d(&p.tk, a.k, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_n, bf));
    SF_TRY(make_tmap_4d(&p.tv, a.v, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_n, bf));
    // head pairs with an even head count (a pair never straddles two sequences) and rows a multiple
    // of 8: both heads of a column block in one 5-D box
    if (b.block_m == 64 && a.h % 2 == 0 && a.seq_len % 8 == 0) {
        const char* e = std::getenv("SF_ATTN_PAIR5");
        if (!(e && *e == '0')) {
            SF_TRY(make_tmap_pair5(&p.tk2, a.k, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_n, bf));
            SF_TRY(make_tmap_pair5(&p.tv2, a.v, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_n, bf));
            const char* re = std::getenv("SF_ATTN_RUNBOX");
            if (b.block_n < 64 && !(re && *re == '0')) {  // 64-row boxes for runs of consecutive blocks
                SF_TRY(make_tmap_pair5(&p.tk4, a.k, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, 64, bf));
                SF_TRY(make_tmap_pair5(&p.tv4, a.v, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, 64, bf));
            }
            // Q of both heads in one box {64, 64, 2, 1}: [head][64 rows][128 B], head t at t * 8 KB
            SF_TRY(make_tmap_4d(&p.tq, a.q, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, b.block_m, bf, 2));
            p.pair5 = (b.block_n < 64 && !(re && *re == '0')) ? 2 : 1;
        }
    }
    if (b.block_m == 128 && b.block_n < 64) {  // 64-row boxes for runs of consecutive blocks
        const char* re = std::getenv("SF_ATTN_RUNBOX");
        if (!(re && *re == '0')) {
            SF_TRY(make_tmap_4d(&p.tk4, a.k, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, 64, bf));
            SF_TRY(make_tmap_4d(&p.tv4, a.v, a.seq_len, a.h, a.bs, a.q_sn, a.q_sh, a.q_sb, 64, bf));
            p.run64 = 1;
        }
    }
    p.n = a.seq_len;
    p.h = a.h;
    p.bh_total = a.bs * a.h;
    p.bh = b.block_m == 64 ? (p.bh_total + 1) / 2 : p.bh_total;  // head pairs at block_m 64
    p.n_rows = b.n_rows;
    p.n_items = b.n_rows * p.bh;
    p.load_row_ptr = b.load_row_ptr;
    p.load_col_idx = b.load_col_idx;
    p.load_tile = b.load_tile;
    p.pool = b.pool;
    p.o = a.o;
    p.o_sb = a.o_sb;
    p.o_sh = a.o_sh;
    p.o_sn = a.o_sn;
    p.scale_log2 = a.scale * 1.4426950408889634f;
    p.trace = g_attn_trace;
    p.work = attn_work_counter(st);
    p.lse = lse;
    void (*kern)(AttnParams) = nullptr;
    int smem = AttnGeo<128>::kSmemG;
    if (b.block_m == 128) {
        if (b.block_n == 16) kern = bf ? attn_tc_kernel<__nv_bfloat16, 16, 128> : attn_tc_kernel<__half, 16, 128>;
        else if (b.block_n == 32) kern = bf ? attn_tc_kernel<__nv_bfloat16, 32, 128> : attn_tc_kernel<__half, 32, 128>;
        else kern = bf ? attn_tc_kernel<__nv_bfloat16, 64, 128> : attn_tc_kernel<__half, 64, 128>;
    } else {
        smem = AttnGeo<64>::kSmemG;
        if (b.block_n == 16) kern = bf ? attn_tc_kernel<__nv_bfloat16, 16, 64> : attn_tc_kernel<__half, 16, 64>;
        else if (b.block_n == 32) kern = bf ? attn_tc_kernel<__nv_bfloat16, 32, 64> : attn_tc_kernel<__half, 32, 64>;
        else kern = bf ? attn_tc_kernel<__nv_bfloat16, 64, 64> : attn_tc_kernel<__half, 64, 64>;
    }
    if (b.tile_bytes != b.block_m * b.block_n / 8) return fail(SF_PLAN_ERROR, "BSR tile_bytes does not match block shape");
    SF_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    static int n_sm = 0;
    if (!n_sm) {
        int dev = 0;
        SF_CUDA_TRY(cudaGetDevice(&dev));
        SF_CUDA_TRY(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, dev));
    }
    // persistent: two CTAs per SM (smem and TMEM are sized for it), items round-robin
    int64_t ctas = std::min<int64_t>(p.n_items, 2 * n_sm);
    if (const char* e = std::getenv("SF_ATTN_MAX_CTAS"))  // test aid: many items per CTA at small shapes
        ctas = std::max<int64_t>(1, std::min<int64_t>(ctas, std::atoll(e)));
    dim3 grid(static_cast<unsigned>(ctas));
    SF_CUDA_TRY(launch_pdl(kern, grid, dim3(kThreads), smem, st, nullptr, p));
    SF_LAUNCH_CHECK();
    return SF_OK;
}

}  // namespace sf

// Debug hook (not part of the boundary): record clock64 timestamps of CTA (0,0) of subsequent
// tcgen05 attention launches into a device buffer of >= 64*32 uint64 (NULL disables).
extern "C" sf_status sf_debug_attn_trace(void* dev_buf) {
    sf::g_attn_trace = static_cast<unsigned long long*>(dev_buf);
    return SF_OK;
}
