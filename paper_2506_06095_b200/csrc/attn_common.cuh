// attn_common.cuh — device helpers shared by the tcgen05 attention kernels (attn_tc.cu: one
// (b, h) slice per work item; attn_tc3.cu: head groups sharing one mask per work item).
#pragma once
#include "tc.cuh"

namespace sf {
namespace {

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

// 2^x for a pair on the FMA pipe (FA4's MUFU offload): x = j + f with j = rint(x) from the
// 1.5*2^23 rounding trick, 2^f on [-0.5, 0.5] by a degree-4 Taylor polynomial (rel. error
// < 5e-5, well under the fp16 spacing of P), and j added straight into the exponent field.
// x is clamped at -125 so masked (-inf) cells give a tiny positive value that packs to 0.
#ifndef SF_ATTN_EMU
#define SF_ATTN_EMU 1  // 1 of 8 pairs on the FMA pipe: the softmax is issue-bound (profiles/r02/attn_headgroup.txt)
#endif
constexpr int kEmuPairs = SF_ATTN_EMU;  // of the 8 pairs in each 16-column group
__device__ __forceinline__ float2 ex2_emu2(float2 x) {
    x = make_float2(fmaxf(x.x, -125.f), fmaxf(x.y, -125.f));
    const float2 t = tc::fadd2(x, make_float2(12582912.f, 12582912.f));
    const float2 jf = tc::fadd2(t, make_float2(-12582912.f, -12582912.f));
    const float2 f = tc::ffma2(jf, make_float2(-1.f, -1.f), x);
    float2 p = tc::ffma2(make_float2(9.6181291e-3f, 9.6181291e-3f), f, make_float2(5.5504109e-2f, 5.5504109e-2f));
    p = tc::ffma2(p, f, make_float2(2.4022651e-1f, 2.4022651e-1f));
    p = tc::ffma2(p, f, make_float2(6.9314718e-1f, 6.9314718e-1f));
    p = tc::ffma2(p, f, make_float2(1.f, 1.f));
    return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                       __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}

// v if bit `bit` of `bits` is set, else -inf. Written as and/setp/selp so ptxas lowers a run of
// them to one R2P (7 predicates from a register byte) + one FSEL per element.
__device__ __forceinline__ float mask_sel(uint32_t bits, uint32_t bit, float v) {
    float o;
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\tand.b32 t, %1, %2;\n\tsetp.ne.b32 p, t, 0;\n\t"
        "selp.f32 %0, %3, 0fFF800000, p;\n\t}"
        : "=f"(o)
        : "r"(bits), "r"(bit), "f"(v));
    return o;
}

using tc::fadd2;
using tc::ffma2;
using tc::fmax3;

__device__ __forceinline__ uint32_t lds_u32(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t addr) {
    uint16_t v;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(addr));
    return v;
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
        "[%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

// SW128 smem descriptor with a given stride between 8-row groups (SBO): K / V stages whose 1 KB
// swizzle atoms of several heads are interleaved at a fixed stride
__device__ __forceinline__ uint64_t sdesc_sw128_sbo(uint32_t smem_addr, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((smem_addr >> 4) & 0x3FFFu);
    d |= static_cast<uint64_t>(1u) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
    d |= static_cast<uint64_t>(1u) << 46;
    d |= static_cast<uint64_t>(2u) << 61;
    return d;
}

__device__ __forceinline__ void tma_load_5d(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1,
                                            int32_t c2, int32_t c3, int32_t c4) {
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, "
        "%7}], [%2];" ::"r"(tc::smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(tc::smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
        : "memory");
}

// Work items (row-block rank, b*h) are numbered with row blocks ranked by descending load count,
// so the longest items come first. The producer warp picks the CTA's next item and publishes it
// to the MMA and softmax roles through a small shared-memory ring (kItemRing slots with full /
// empty barriers). With a work counter (p.work) it takes the next global index by atomicAdd —
// greedy longest-first list scheduling, which keeps CTAs balanced when a few row blocks are much
// longer than the rest (global rows: cfg4's items range 5-64 steps, a static deal left the
// longest CTA 46% above the mean); the last CTA to finish resets the counter, so the launch
// replays in a CUDA graph. Without one, items are dealt statically in snake order (round k goes
// c = 0..G-1 when k is even, G-1..0 when odd).
constexpr int kItemRing = 4;
struct Items {
    const int32_t* lrp;
    const int32_t* order;  // smem: row block of each rank
    int bh_count, n_items, G;
    // the static deal: the CTA's k-th item index, or -1 past its last
    __device__ __forceinline__ int static_idx(int k) const {
        return k < count() ? k * static_cast<int>(gridDim.x) + pos(k) : -1;
    }
    __device__ __forceinline__ void decode(int idx, int& rb, int& bh, int& l0, int& L, int& nsteps) const {
        rb = order[idx / bh_count];
        bh = idx % bh_count;
        l0 = lrp[rb];
        L = lrp[rb + 1] - l0;
        nsteps = (L + G - 1) / G;
    }
    __device__ __forceinline__ int pos(int k) const {
        const int c = static_cast<int>(blockIdx.x), g = static_cast<int>(gridDim.x);
        return (k & 1) ? g - 1 - c : c;
    }
    __device__ __forceinline__ int count() const {
        const int g = static_cast<int>(gridDim.x);
        const int full = n_items / g, rem = n_items % g;
        return full + (rem > 0 && pos(full) < rem ? 1 : 0);
    }
};

// Consumer side of the item ring: the item at ring position `it` (waits for the producer to
// publish it; `release` frees the slot once this consumer has its copy).
struct ItemFeed {
    const int32_t* slots;  // smem [kItemRing]
    uint64_t* full;        // [kItemRing], one producer arrive
    uint64_t* empty;       // [kItemRing], 2 (the MMA issuer's two cursors) + 4 (softmax warps) arrives
    __device__ __forceinline__ int read(uint32_t it) const {
        tc::mbar_wait(&full[it % kItemRing], (it / kItemRing) & 1);
        return *reinterpret_cast<const volatile int32_t*>(&slots[it % kItemRing]);
    }
    __device__ __forceinline__ void release(uint32_t it) const { tc::mbar_arrive(&empty[it % kItemRing]); }
};

// Flat walk over the steps of the CTA's non-empty items (the MMA issuer keeps two of these: the
// S cursor runs kSBuf steps ahead of the P.V cursor). Each cursor releases a ring slot as soon as
// it has read it, so the S cursor can read past a run of empty items while the P.V cursor still
// works on an earlier one.
struct Cursor {
    uint32_t it = 0;
    int qi = -1, j = 0, ns = 0;
    bool valid = false;
    __device__ __forceinline__ bool next_item(const Items& items, const ItemFeed& feed) {
        int rb, bh, l0, L;
        do {
            const int idx = feed.read(it);
            feed.release(it);
            ++it;
            if (idx < 0) return valid = false;
            items.decode(idx, rb, bh, l0, L, ns);
        } while (ns == 0);
        ++qi;
        j = 0;
        return valid = true;
    }
    __device__ __forceinline__ void advance(const Items& items, const ItemFeed& feed) {
        if (++j == ns) next_item(items, feed);
    }
};


}  // namespace
}  // namespace sf
