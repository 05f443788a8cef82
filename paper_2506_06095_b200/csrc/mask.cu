// mask.cu — descriptor -> bit-packed dense mask on device.
// Replaces generate_mask / compose / gen_* (io.hpp:192-204, mask.hpp:74-179).
//
// Layout: row-major, W = ceil(n/32) uint32 words per row, bit j of row i = bit j%32 of word
// j/32. One thread produces one word: every term's predicate is evaluated for the word's 32
// columns and OR-ed (compose, mask.hpp:146-166). HBM-bound write of n*W*4 bytes.
//
// Random tiles (mask.hpp:124-143) consume one mt19937_64 draw per tile in row-major tile order.
// The stream is generated on device by a single CTA: 312 threads run the twist in two
// dependency phases, then temper in parallel, and set tile bits in a ceil(n/block)^2 bitmap
// that the word kernel reads. Bit-exact with the reference: the comparison
// (x >> 11) * 2^-53 < filling_rate is exact in double precision.
#include <cstring>
#include <vector>

#include "common.cuh"

namespace sf {
namespace {

constexpr int kMtN = 312, kMtM = 156;

__device__ __forceinline__ uint64_t mt_twist_one(uint64_t cur, uint64_t next, uint64_t far) {
    const uint64_t x = (cur & 0xFFFFFFFF80000000ull) | (next & 0x7FFFFFFFull);
    uint64_t xa = x >> 1;
    if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
    return far ^ xa;
}

__device__ __forceinline__ uint64_t mt_temper(uint64_t x) {
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

// One CTA of kMtN threads. tiles[(bi*grid+bj)/32] bit set iff draw #(bi*grid+bj) < fill.
__global__ void __launch_bounds__(kMtN) random_tiles_kernel(uint64_t seed, int64_t n_draws,
                                                            double fill, uint32_t* tiles) {
    __shared__ uint64_t mt[kMtN];
    const int i = threadIdx.x;
    if (i == 0) {
        uint64_t v = seed;
        mt[0] = v;
        for (int k = 1; k < kMtN; ++k) {
            v = 6364136223846793005ull * (v ^ (v >> 62)) + static_cast<uint64_t>(k);
            mt[k] = v;
        }
    }
    __syncthreads();
    for (int64_t base = 0; base < n_draws; base += kMtN) {
        // twist: phase A (i < 156) reads only old values; phase B (i >= 156) reads old
        // mt[i], mt[i+1] captured before any write and the new mt[i-156] (and new mt[0] for
        // i == 311), matching the sequential recurrence exactly.
        const uint64_t cur = mt[i];
        const uint64_t nxt = (i + 1 < kMtN) ? mt[i + 1] : 0ull;
        const uint64_t far_old = (i < kMtN - kMtM) ? mt[i + kMtM] : 0ull;
        __syncthreads();
        if (i < kMtN - kMtM) mt[i] = mt_twist_one(cur, nxt, far_old);
        __syncthreads();
        if (i >= kMtN - kMtM) {
            const uint64_t nx = (i == kMtN - 1) ? mt[0] : nxt;
            mt[i] = mt_twist_one(cur, nx, mt[i - (kMtN - kMtM)]);
        }
        __syncthreads();
        const int64_t k = base + i;
        if (k < n_draws) {
            const double u = static_cast<double>(mt_temper(mt[i]) >> 11) * 0x1.0p-53;
            if (u < fill) atomicOr(&tiles[k >> 5], 1u << (k & 31));
        }
    }
}

struct TermDev {
    int32_t pattern, band, global, dilation, block, rgrid;
    const uint32_t* rtiles;  // random tile bitmap (RANDOM / BIGBIRD)
};

constexpr int kMaxTerms = 8;
struct Terms {
    int32_t count;
    TermDev t[kMaxTerms];
};

__device__ __forceinline__ uint32_t band_bits(int64_t i, int64_t j0, int64_t lo, int64_t hi) {
    // bits for columns j0..j0+31 inside [lo, hi]
    const int64_t a = max(lo, j0), b = min(hi, j0 + 31);
    if (a > b) return 0u;
    const int len = static_cast<int>(b - a + 1);
    const uint32_t m = len >= 32 ? 0xffffffffu : ((1u << len) - 1u);
    return m << static_cast<int>(a - j0);
}

__global__ void mask_words_kernel(Terms terms, int32_t n, int32_t words, uint32_t* bits) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(n) * words) return;
    const int64_t i = idx / words;
    const int64_t wj = idx - i * words;
    const int64_t j0 = wj * 32;
    const int64_t jmax = imin64(n - 1, j0 + 31);
    uint32_t acc = 0u;
    for (int t = 0; t < terms.count; ++t) {
        const TermDev& d = terms.t[t];
        const int p = d.pattern;
        if (p == SF_PATTERN_GLOBAL || p == SF_PATTERN_LONGFORMER || p == SF_PATTERN_BIGBIRD) {
            if (i < d.global) acc |= band_bits(i, j0, 0, n - 1);
            else acc |= band_bits(i, j0, 0, static_cast<int64_t>(d.global) - 1);
        }
        if (p == SF_PATTERN_SLIDING || p == SF_PATTERN_LONGFORMER || p == SF_PATTERN_BIGBIRD)
            acc |= band_bits(i, j0, i - d.band + 1, imin64(n - 1, i + d.band - 1));
        if (p == SF_PATTERN_CAUSAL) acc |= band_bits(i, j0, 0, i);
        if (p == SF_PATTERN_CAUSAL_LOCAL) acc |= band_bits(i, j0, i - d.band + 1, i);
        if (p == SF_PATTERN_STRIDED) {
            acc |= band_bits(i, j0, i - d.band + 1, i);
            for (int64_t j = j0; j <= min(jmax, i); ++j)
                if ((i - j) % d.band == 0) acc |= 1u << static_cast<int>(j - j0);
        }
        if (p == SF_PATTERN_DILATED) {
            const int64_t stride = static_cast<int64_t>(d.dilation) + 1;
            const int64_t reach = static_cast<int64_t>(d.band) * stride;
            for (int64_t j = j0; j <= jmax; ++j) {
                const int64_t dd = i - j;
                if ((dd < 0 ? -dd : dd) < reach && dd % stride == 0) acc |= 1u << static_cast<int>(j - j0);
            }
        }
        if (p == SF_PATTERN_RANDOM || p == SF_PATTERN_BIGBIRD) {
            const int64_t bi = i / d.block;
            for (int64_t j = j0; j <= jmax; ++j) {
                const int64_t k = bi * d.rgrid + j / d.block;
                if ((d.rtiles[k >> 5] >> (k & 31)) & 1u) acc |= 1u << static_cast<int>(j - j0);
            }
        }
    }
    bits[idx] = acc;
}

__global__ void pack_u8_kernel(const uint8_t* __restrict__ m, int32_t n, int32_t words,
                               uint32_t* __restrict__ bits) {
    const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (idx >= static_cast<int64_t>(n) * words) return;
    const int64_t i = idx / words, wj = idx - i * words;
    uint32_t acc = 0u;
    for (int b = 0; b < 32; ++b) {
        const int64_t j = wj * 32 + b;
        if (j < n && m[i * n + j]) acc |= 1u << b;
    }
    bits[idx] = acc;
}

__global__ void popcount_kernel(const uint32_t* __restrict__ bits, int64_t count,
                                unsigned long long* out) {
    unsigned long long local = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x)
        local += __popc(bits[i]);
    for (int o = 16; o; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(out, local);
}

// Same checks and error classes as the reference generators.
sf_status check_term(const sf_mask_desc& t) {
    const int n = t.seq_len;
    auto bad = [](const char* m) { return fail(SF_INVALID_PARAMETER, m); };
    if (n <= 0) return bad("seq_len must be positive");                          // mask.hpp:23
    const bool band = t.pattern == SF_PATTERN_SLIDING || t.pattern == SF_PATTERN_DILATED ||
                      t.pattern == SF_PATTERN_LONGFORMER || t.pattern == SF_PATTERN_BIGBIRD ||
                      t.pattern == SF_PATTERN_CAUSAL_LOCAL || t.pattern == SF_PATTERN_STRIDED;
    const bool glob = t.pattern == SF_PATTERN_GLOBAL || t.pattern == SF_PATTERN_LONGFORMER ||
                      t.pattern == SF_PATTERN_BIGBIRD;
    const bool rnd = t.pattern == SF_PATTERN_RANDOM || t.pattern == SF_PATTERN_BIGBIRD;
    if (t.pattern < 0 || t.pattern > SF_PATTERN_STRIDED) return bad("unknown mask pattern");
    if (glob && (t.global_width < 0 || t.global_width > n))
        return bad("global_width must be in [0, seq_len]");                     // mask.hpp:108
    if (band && (t.band_width < 1 || t.band_width > n))
        return bad("band_width must be in [1, seq_len]");                       // mask.hpp:75
    if (t.pattern == SF_PATTERN_DILATED && t.dilation_rate < 0)
        return bad("dilation_rate must be >= 0");                               // mask.hpp:92
    if (rnd && t.block < 1) return bad("block must be >= 1");                    // mask.hpp:125
    if (rnd && !(t.filling_rate >= 0.0 && t.filling_rate <= 1.0))
        return bad("filling_rate must be in [0, 1]");                           // mask.hpp:127
    return SF_OK;
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" int32_t sf_mask_words(int32_t seq_len) { return (seq_len + 31) / 32; }

extern "C" sf_status sf_mask_validate(const sf_mask_desc* terms, int32_t n_terms) {
    if (!terms || n_terms < 1) return fail(SF_INVALID_PARAMETER, "compose needs at least one mask");
    if (n_terms > kMaxTerms) return fail(SF_INVALID_PARAMETER, "too many mask terms (max 8)");
    for (int t = 0; t < n_terms; ++t) {
        SF_TRY(check_term(terms[t]));
        if (terms[t].seq_len != terms[0].seq_len)
            return fail(SF_SHAPE_ERROR, "compose: mismatched seq_len");          // mask.hpp:150
    }
    return SF_OK;
}

extern "C" sf_status sf_mask_generate(const sf_mask_desc* terms, int32_t n_terms, uint32_t* d_bits,
                                      void* stream) {
    SF_TRY(sf_mask_validate(terms, n_terms));
    cudaStream_t st = as_stream(stream);
    const int32_t n = terms[0].seq_len, words = sf_mask_words(n);
    Terms td{};
    td.count = n_terms;
    std::vector<uint32_t*> scratch;
    for (int t = 0; t < n_terms; ++t) {
        const sf_mask_desc& d = terms[t];
        TermDev& e = td.t[t];
        e.pattern = d.pattern;
        e.band = d.band_width;
        e.global = d.global_width;
        e.dilation = d.dilation_rate;
        e.block = d.block > 0 ? d.block : 16;
        e.rgrid = (n + e.block - 1) / e.block;
        e.rtiles = nullptr;
        if (d.pattern == SF_PATTERN_RANDOM || d.pattern == SF_PATTERN_BIGBIRD) {
            const int64_t draws = static_cast<int64_t>(e.rgrid) * e.rgrid;
            uint32_t* rt = nullptr;
            SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&rt), ceil_div(draws, 32) * 4, st));
            SF_CUDA_TRY(cudaMemsetAsync(rt, 0, ceil_div(draws, 32) * 4, st));
            random_tiles_kernel<<<1, kMtN, 0, st>>>(d.seed, draws, d.filling_rate, rt);
            SF_LAUNCH_CHECK();
            e.rtiles = rt;
            scratch.push_back(rt);
        }
    }
    const int64_t total = static_cast<int64_t>(n) * words;
    mask_words_kernel<<<static_cast<unsigned>(ceil_div(total, 256)), 256, 0, st>>>(td, n, words, d_bits);
    SF_LAUNCH_CHECK();
    for (auto* p : scratch) SF_CUDA_TRY(cudaFreeAsync(p, st));
    return SF_OK;
}

extern "C" sf_status sf_mask_pack_u8(const uint8_t* d_mask_u8, int32_t seq_len, uint32_t* d_bits,
                                     void* stream) {
    if (seq_len <= 0) return fail(SF_INVALID_PARAMETER, "seq_len must be positive");
    const int32_t words = sf_mask_words(seq_len);
    const int64_t total = static_cast<int64_t>(seq_len) * words;
    pack_u8_kernel<<<static_cast<unsigned>(ceil_div(total, 256)), 256, 0, as_stream(stream)>>>(
        d_mask_u8, seq_len, words, d_bits);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

namespace sf {
namespace {
__global__ void or_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ acc, int64_t total) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < total) acc[i] |= src[i];
}
__global__ void andnot_kernel(const uint32_t* __restrict__ src, uint32_t* __restrict__ acc, int64_t total) {
    const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < total) acc[i] &= ~src[i];
}
}  // namespace
}  // namespace sf

extern "C" sf_status sf_mask_or(const uint32_t* d_src, uint32_t* d_acc, int32_t seq_len, void* stream) {
    if (seq_len <= 0) return fail(SF_INVALID_PARAMETER, "seq_len must be positive");
    const int64_t total = static_cast<int64_t>(seq_len) * sf_mask_words(seq_len);
    or_kernel<<<static_cast<unsigned>(ceil_div(total, 256)), 256, 0, as_stream(stream)>>>(d_src, d_acc, total);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

extern "C" sf_status sf_mask_andnot(const uint32_t* d_src, uint32_t* d_acc, int32_t seq_len, void* stream) {
    if (seq_len <= 0) return fail(SF_INVALID_PARAMETER, "seq_len must be positive");
    const int64_t total = static_cast<int64_t>(seq_len) * sf_mask_words(seq_len);
    andnot_kernel<<<static_cast<unsigned>(ceil_div(total, 256)), 256, 0, as_stream(stream)>>>(d_src, d_acc, total);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

extern "C" sf_status sf_mask_count(const uint32_t* d_bits, int32_t seq_len, int64_t* count,
                                   void* stream) {
    cudaStream_t st = as_stream(stream);
    unsigned long long* d = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&d), 8, st));
    SF_CUDA_TRY(cudaMemsetAsync(d, 0, 8, st));
    const int64_t total = static_cast<int64_t>(seq_len) * sf_mask_words(seq_len);
    popcount_kernel<<<296, 256, 0, st>>>(d_bits, total, d);
    SF_LAUNCH_CHECK();
    unsigned long long h = 0;
    SF_CUDA_TRY(cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st));
    SF_CUDA_TRY(cudaFreeAsync(d, st));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    *count = static_cast<int64_t>(h);
    return SF_OK;
}

// ---------------------------------------------------------------------------------------------
// SFMK dense-mask dump (io.hpp:61-95 write_dense_mask / read_dense_mask): 16-byte header
// ("SFMK", version 1, seq_len, reserved 0) then the n*n bits row-major, packed LSB-first with no
// per-row padding. The device rows are word-padded, so the flat stream is re-packed on device:
// one thread per output byte gathers its 8 bits.
namespace sf {
namespace {
__global__ void sfmk_pack_kernel(const uint32_t* __restrict__ bits, int32_t n, int32_t words, int64_t nbytes,
                                 uint8_t* __restrict__ out) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= nbytes) return;
    const int64_t total = static_cast<int64_t>(n) * n;
    uint32_t v = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) {
        const int64_t f = 8 * k + b;
        if (f >= total) break;
        const int64_t i = f / n, j = f - i * n;
        v |= ((bits[i * words + (j >> 5)] >> (j & 31)) & 1u) << b;
    }
    out[k] = static_cast<uint8_t>(v);
}
__global__ void sfmk_unpack_kernel(const uint8_t* __restrict__ in, int32_t n, int32_t words, uint32_t* __restrict__ bits) {
    const int64_t w = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (w >= static_cast<int64_t>(n) * words) return;
    const int64_t i = w / words, j0 = (w - i * words) * 32;
    uint32_t v = 0;
    for (int b = 0; b < 32 && j0 + b < n; ++b) {
        const int64_t f = i * n + j0 + b;
        v |= ((in[f >> 3] >> (f & 7)) & 1u) << b;
    }
    bits[w] = v;
}
}  // namespace
}  // namespace sf

extern "C" sf_status sf_mask_serialize(const uint32_t* d_bits, int32_t seq_len, uint8_t* buf, int64_t cap,
                                       int64_t* nbytes, void* stream) {
    if (seq_len <= 0) return fail(SF_INVALID_PARAMETER, "seq_len must be positive");
    const int64_t payload = (static_cast<int64_t>(seq_len) * seq_len + 7) / 8;
    if (nbytes) *nbytes = 16 + payload;
    if (!buf) return SF_OK;
    if (cap < 16 + payload) return fail(SF_INVALID_PARAMETER, "buffer too small for the SFMK dump");
    cudaStream_t st = as_stream(stream);
    uint8_t* d = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&d), static_cast<size_t>(payload), st));
    sfmk_pack_kernel<<<static_cast<unsigned>(ceil_div(payload, 256)), 256, 0, st>>>(d_bits, seq_len,
                                                                                   sf_mask_words(seq_len), payload, d);
    SF_LAUNCH_CHECK();
    const uint32_t hdr[4] = {0x4B4D4653u /* "SFMK" */, 1u, static_cast<uint32_t>(seq_len), 0u};
    std::memcpy(buf, hdr, 16);
    SF_CUDA_TRY(cudaMemcpyAsync(buf + 16, d, static_cast<size_t>(payload), cudaMemcpyDeviceToHost, st));
    SF_CUDA_TRY(cudaFreeAsync(d, st));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    return SF_OK;
}

extern "C" sf_status sf_mask_deserialize(const uint8_t* buf, int64_t nbytes, int32_t* seq_len, uint32_t* d_bits,
                                         void* stream) {
    if (!buf || nbytes < 16) return fail(SF_IO_ERROR, "truncated mask dump");
    uint32_t hdr[4];
    std::memcpy(hdr, buf, 16);
    if (hdr[0] != 0x4B4D4653u) return fail(SF_IO_ERROR, "bad mask dump magic");           // io.hpp:80
    if (hdr[1] != 1u) return fail(SF_IO_ERROR, "unsupported mask dump version");          // io.hpp:82
    const int32_t n = static_cast<int32_t>(hdr[2]);
    const int64_t payload = (static_cast<int64_t>(n) * n + 7) / 8;
    if (n <= 0 || nbytes < 16 + payload) return fail(SF_IO_ERROR, "truncated mask dump");  // io.hpp:88
    if (seq_len) *seq_len = n;
    if (!d_bits) return SF_OK;
    cudaStream_t st = as_stream(stream);
    uint8_t* d = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&d), static_cast<size_t>(payload), st));
    SF_CUDA_TRY(cudaMemcpyAsync(d, buf + 16, static_cast<size_t>(payload), cudaMemcpyHostToDevice, st));
    const int32_t words = sf_mask_words(n);
    sfmk_unpack_kernel<<<static_cast<unsigned>(ceil_div(static_cast<int64_t>(n) * words, 256)), 256, 0, st>>>(
        d, n, words, d_bits);
    SF_LAUNCH_CHECK();
    SF_CUDA_TRY(cudaFreeAsync(d, st));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    return SF_OK;
}
