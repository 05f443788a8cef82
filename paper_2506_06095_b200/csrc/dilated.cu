// dilated.cu — masked MHA for dilated masks by MASK DECOMPOSITION (the planner extension of
// DESIGN §6, alongside strided.cu). dilated(w, r) = { |i - j| < w s, (i - j) % s == 0 } with
// s = r + 1 (mask.hpp:89-103) only pairs rows and keys of the same residue class p = i mod s, and
// inside class p (rows i = p + s a, keys j = p + s b) it is the sliding window |a - b| < w
// (mask.hpp:74-84) over n / s rows. In the (128, 16) BSR of the whole mask every loaded tile is
// 1/s useful at best; per class the band is dense. So:
//   part A  for each class p, the block executor (attn_tc) over the class's rows — the same Q / K /
//           V / O tensors viewed with row stride s * sn from row p — with the sliding(w) BSR of
//           n / s rows (one BSR serves every class);
//   part B  the rest of the session mask (e.g. T5's global(g) columns and rows), minus the dilated
//           cells, on the block executor over the full rows into a scratch output;
// both with per-row log2-sum-exp2, merged per row: O = (O_A 2^lse_A + O_B 2^lse_B) / (2^lse_A + 2^lse_B)
// (attention.hpp:71-172 semantics over A u B; rows valid in neither stay exactly zero). Without a
// rest the classes write their rows of O directly and nothing is merged.
#include <cmath>
#include <string>

#include "common.cuh"

namespace sf {
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t st);
sf_status attn_tc(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st, bool probe_only, float* lse);
sf_status check_attn_args(const sf_attn_args& a);
namespace {

struct MergeParams {
    void* o;                 // part A's output, merged in place
    const void* ob;          // part B's output, contiguous [b*h][n][64]
    const float* lse_a;      // [s][b*h][n / s]
    const float* lse_b;      // [b*h][n]
    int64_t o_sb, o_sh, o_sn;
    int32_t n, h, s, slices;
};

// one thread per (row, 8-element chunk): 16-byte loads and stores
template <typename T>
__global__ void __launch_bounds__(256) dilated_merge_kernel(const __grid_constant__ MergeParams p) {
    pdl_enter();
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t rows = static_cast<int64_t>(p.slices) * p.n;
    if (t >= rows * 8) return;
    const int64_t r = t >> 3;
    const int c = static_cast<int>(t & 7);
    const int slice = static_cast<int>(r / p.n);
    const int i = static_cast<int>(r - static_cast<int64_t>(slice) * p.n);
    const int cls = i % p.s, a = i / p.s, nc = p.n / p.s;
    const float la = p.lse_a[(static_cast<int64_t>(cls) * p.slices + slice) * nc + a];
    const float lb = p.lse_b[r];
    const float m = fmaxf(la, lb);
    T* dst = static_cast<T*>(p.o) + (slice / p.h) * p.o_sb + (slice % p.h) * p.o_sh + static_cast<int64_t>(i) * p.o_sn + 8 * c;
    uint4 ua = *reinterpret_cast<const uint4*>(dst);
    const uint4 ub = reinterpret_cast<const uint4*>(static_cast<const T*>(p.ob) + r * 64)[c];
    if (m == -INFINITY) {  // no valid key in either part: the row is exactly zero
        *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);
        return;
    }
    const float wa = exp2f(la - m), wb = exp2f(lb - m);
    const float inv = 1.f / (wa + wb);
    const T* ha = reinterpret_cast<const T*>(&ua);
    const T* hb = reinterpret_cast<const T*>(&ub);
    T out[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) out[e] = DT<T>::from_f((wa * DT<T>::to_f(ha[e]) + wb * DT<T>::to_f(hb[e])) * inv);
    *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(out);
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" sf_status sf_mha_dilated(const sf_attn_args* args, int32_t stride, const sf_bsr_dev* class_bsr,
                                    const sf_bsr_dev* rest_bsr, void* stream) {
    if (!args || !class_bsr) return fail(SF_INVALID_PARAMETER, "null argument");
    SF_TRY(check_attn_args(*args));
    const sf_attn_args& a0 = *args;
    if (stride < 2) return fail(SF_INVALID_PARAMETER, "stride (dilation_rate + 1) must be >= 2");
    if (a0.seq_len % stride != 0) return fail(SF_PLAN_ERROR, "dilated decomposition needs seq_len % stride == 0");
    if (class_bsr->seq_len != a0.seq_len / stride) return fail(SF_SHAPE_ERROR, "class BSR seq_len must be seq_len / stride");
    if (rest_bsr && rest_bsr->seq_len != a0.seq_len) return fail(SF_SHAPE_ERROR, "rest BSR seq_len differs from input");
    auto tc_tile = [](const sf_bsr_dev* b) { return b->block_m == 128 || b->block_m == 64; };
    if (a0.head_size != 64 || !tc_tile(class_bsr) || (rest_bsr && !tc_tile(rest_bsr)))
        return fail(SF_PLAN_ERROR, "dilated decomposition needs head_size 64 and block_m 128 or 64 (head pairs) BSRs");
    cudaStream_t st = as_stream(stream);
    sf_attn_args a = a0;
    if (a.scale == 0.f) a.scale = 1.0f / std::sqrt(static_cast<float>(a.head_size));
    const int64_t slices = static_cast<int64_t>(a.bs) * a.h;
    const bool rest = rest_bsr && rest_bsr->n_load > 0;
    const size_t el = 2;
    float* lse_a = nullptr;
    float* lse_b = nullptr;
    void* ob = nullptr;
    if (rest) {
        SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&lse_a), slices * a.seq_len * sizeof(float), st));
        if (pool_malloc(reinterpret_cast<void**>(&lse_b), slices * a.seq_len * sizeof(float), st) != cudaSuccess ||
            pool_malloc(&ob, slices * a.seq_len * 64 * el, st) != cudaSuccess) {
            cudaGetLastError();
            cudaFreeAsync(lse_a, st);
            if (lse_b) cudaFreeAsync(lse_b, st);
            return fail(SF_CUDA_ERROR, "dilated decomposition scratch allocation failed");
        }
    }
    sf_status status = SF_OK;
    // part A: class p = rows p, p + s, ... of every tensor (row stride s * sn), sliding(w) over n / s rows
    const int nc = a.seq_len / stride;
    for (int p = 0; p < stride && status == SF_OK; ++p) {
        sf_attn_args c = a;
        c.seq_len = nc;
        c.q = static_cast<const char*>(a.q) + p * a.q_sn * el;
        c.k = static_cast<const char*>(a.k) + p * a.q_sn * el;
        c.v = static_cast<const char*>(a.v) + p * a.q_sn * el;
        c.o = static_cast<char*>(a.o) + p * a.o_sn * el;
        c.q_sn = a.q_sn * stride;
        c.o_sn = a.o_sn * stride;
        status = attn_tc(c, *class_bsr, st, false, rest ? lse_a + p * slices * nc : nullptr);
    }
    if (status == SF_OK && rest) {
        // part B: the rest of the mask over the full rows into the scratch output, then the merge
        sf_attn_args b = a;
        b.o = ob;
        b.o_sn = 64;
        b.o_sh = static_cast<int64_t>(a.seq_len) * 64;
        b.o_sb = a.h * b.o_sh;
        status = attn_tc(b, *rest_bsr, st, false, lse_b);
        if (status == SF_OK) {
            MergeParams mp{};
            mp.o = a.o; mp.ob = ob; mp.lse_a = lse_a; mp.lse_b = lse_b;
            mp.o_sb = a.o_sb; mp.o_sh = a.o_sh; mp.o_sn = a.o_sn;
            mp.n = a.seq_len; mp.h = a.h; mp.s = stride; mp.slices = static_cast<int32_t>(slices);
            const int64_t threads = slices * a.seq_len * 8;
            auto kern = a.dtype == SF_BF16 ? dilated_merge_kernel<__nv_bfloat16> : dilated_merge_kernel<__half>;
            cudaError_t e = launch_pdl(kern, dim3(static_cast<unsigned>(ceil_div(threads, 256))), dim3(256), 0, st,
                                       nullptr, mp);
            if (e != cudaSuccess) status = fail(SF_CUDA_ERROR, std::string("dilated merge kernel: ") + cudaGetErrorString(e));
            else note_launch();
        }
    }
    if (rest) {
        cudaFreeAsync(lse_a, st);
        cudaFreeAsync(lse_b, st);
        cudaFreeAsync(ob, st);
    }
    return status;
}
