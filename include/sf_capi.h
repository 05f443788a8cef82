/*
 * sf_capi.h — C ABI of the B200-native sparse-Transformer hot path (STOF, arXiv 2506.06095).
 *
 * This is the drop-in boundary. The reference (`/root/reference/proj/include/sparsefuse/` headers)
 * is a header-only C++20 CPU library; every entry point below replaces one reference function
 * on the hot path (cited per declaration). Plain pointers and sizes only: no torch, no C++
 * types, no exceptions cross this boundary. Errors come back as `sf_status` values that mirror
 * the reference's exception taxonomy (`common.hpp:14-36`); the C++ host layer
 * (`include/sparsefuse_b200/sparsefuse.hpp`) rethrows the matching exception type.
 *
 * Device data layouts (all device pointers, all stream-ordered on the `stream` argument):
 *   - Dense mask: bit-packed, row-major, `sf_mask_words(n)` uint32 words per row, bit j of
 *     row i is bit (j % 32) of word (j / 32). Bits at j >= n are zero.
 *   - BSR mask (`sf_bsr_dev`): the seven int32 index arrays of the reference `BsrMask`
 *     (`bsr.hpp:21-37`) plus the part-tile pool, bit-packed per tile exactly like
 *     `pack_bits(tile)` (`common.hpp:77-83`), and a device-only `load_tile` array (one int32
 *     per load entry: -1 = full tile, else pool id) that replaces the reference executor's
 *     merge walk (`attention.hpp:100-119`).
 *   - Row-wise CSR (`sf_csr_dev`): `row_ptr` (n+1) and `col_idx` (nnz), as `RowwiseMask`
 *     (`bsr.hpp:41-45`).
 *   - Attention tensors: fp16 (or bf16), addressed by (b, h, i) element strides so the
 *     (bs*seq, heads*head_size) activation layout of `exec_mha` (`backend.hpp:327-356`) and
 *     a fused QKV projection output are both read in place.
 */
#ifndef SF_CAPI_H
#define SF_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes: one per reference exception type (common.hpp:14-36) plus CUDA failures. */
typedef enum sf_status {
    SF_OK = 0,
    SF_INVALID_PARAMETER = 1,     /* invalid_parameter      common.hpp:14 */
    SF_SHAPE_ERROR = 2,           /* shape_error            common.hpp:17 */
    SF_PLAN_ERROR = 3,            /* plan_error             common.hpp:20 */
    SF_DEGENERATE_INPUT = 4,      /* degenerate_input       common.hpp:23 */
    SF_ILLEGAL_SEGMENT = 5,       /* illegal_segment        common.hpp:26 */
    SF_INTERNAL_INCONSISTENCY = 6,/* internal_inconsistency common.hpp:29 */
    SF_BACKEND_ERROR = 7,         /* backend_error          common.hpp:32 */
    SF_IO_ERROR = 8,              /* io_error               common.hpp:35 */
    SF_CUDA_ERROR = 9             /* device failure (no reference counterpart) */
} sf_status;

/* Last error message of the calling thread (static storage, never NULL). */
const char* sf_last_error(void);
/* Library version string, e.g. "sparsefuse-b200 0.1 sm_100a". */
const char* sf_version(void);

/* ------------------------------------------------------------------------------------------
 * Mask descriptors (io.hpp:158-204 MaskDescriptor / generate_mask; mask.hpp:64-179).
 * A generated mask is the OR of `n_terms` descriptors (mask.hpp:146-166 compose).
 * ---------------------------------------------------------------------------------------- */
typedef enum sf_pattern {
    SF_PATTERN_SLIDING = 0,      /* |i-j| < band_width                         mask.hpp:74-84   */
    SF_PATTERN_DILATED = 1,      /* |i-j| < w(r+1) and (i-j)%(r+1)==0          mask.hpp:89-103  */
    SF_PATTERN_GLOBAL = 2,       /* i < g or j < g                             mask.hpp:107-117 */
    SF_PATTERN_RANDOM = 3,       /* seeded block x block tiles, one mt19937_64 draw per tile,
                                    row-major, set iff unit_real < filling_rate mask.hpp:124-143 */
    SF_PATTERN_LONGFORMER = 4,   /* global | sliding                           mask.hpp:169-171 */
    SF_PATTERN_BIGBIRD = 5,      /* global | sliding | random                  mask.hpp:175-179 */
    /* Additions with no reference generator (SURVEY §0 finding 5, H9): pinned by predicates. */
    SF_PATTERN_CAUSAL = 6,       /* j <= i */
    SF_PATTERN_CAUSAL_LOCAL = 7, /* j <= i and i-j < band_width */
    SF_PATTERN_STRIDED = 8       /* j <= i and (i-j < band_width or (i-j) % band_width == 0) */
} sf_pattern;

typedef struct sf_mask_desc {
    int32_t pattern;        /* sf_pattern */
    int32_t seq_len;
    int32_t band_width;
    int32_t global_width;
    int32_t dilation_rate;
    int32_t block;          /* random-tile edge, default 16 (mask.hpp:70) */
    double filling_rate;
    uint64_t seed;
} sf_mask_desc;

/* uint32 words per bit-packed mask row. */
int32_t sf_mask_words(int32_t seq_len);

/* Validate descriptors exactly like the reference generators (same error classes). */
sf_status sf_mask_validate(const sf_mask_desc* terms, int32_t n_terms);

/* Generate the OR of the terms into d_bits (n * sf_mask_words(n) uint32, device).
 * Replaces generate_mask (io.hpp:192-204) + compose (mask.hpp:146-166). The random-tile
 * mt19937_64 stream is generated on device (one CTA, parallel twist). */
sf_status sf_mask_generate(const sf_mask_desc* terms, int32_t n_terms, uint32_t* d_bits,
                           void* stream);

/* Pack a device uint8 n*n mask (DenseMask::raw(), mask.hpp:18-54) into the bit layout. */
sf_status sf_mask_pack_u8(const uint8_t* d_mask_u8, int32_t seq_len, uint32_t* d_bits,
                          void* stream);

/* SFMK dense-mask dump (write_dense_mask / read_dense_mask, io.hpp:61-95): header "SFMK", version 1,
 * seq_len, reserved, then the n*n bits row-major LSB-first. serialize: buf == NULL -> *nbytes only;
 * synchronizes. deserialize: d_bits == NULL -> *seq_len only; d_bits holds n * sf_mask_words(n)
 * words. SF_IO_ERROR on bad magic / version / truncation (the reference's io_error). */
sf_status sf_mask_serialize(const uint32_t* d_bits, int32_t seq_len, uint8_t* buf, int64_t cap, int64_t* nbytes,
                            void* stream);
sf_status sf_mask_deserialize(const uint8_t* buf, int64_t nbytes, int32_t* seq_len, uint32_t* d_bits, void* stream);

/* d_acc |= d_src over n rows of sf_mask_words(n) words: compose of arbitrary masks
 * (mask.hpp:146-166) when they are not all descriptor-generated. */
sf_status sf_mask_or(const uint32_t* d_src, uint32_t* d_acc, int32_t seq_len, void* stream);

/* d_acc &= ~d_src over n rows: the cells of one mask not covered by another (mask decomposition,
 * sf_mha_dilated's rest). No reference counterpart. */
sf_status sf_mask_andnot(const uint32_t* d_src, uint32_t* d_acc, int32_t seq_len, void* stream);

/* Valid-cell count of a device bit mask (DenseMask::true_count, mask.hpp:39-43). Synchronizes. */
sf_status sf_mask_count(const uint32_t* d_bits, int32_t seq_len, int64_t* count, void* stream);

/* ------------------------------------------------------------------------------------------
 * Storage formats (bsr.hpp:47-101 build_bsr, bsr.hpp:198-209 build_rowwise).
 * ---------------------------------------------------------------------------------------- */
typedef struct sf_bsr_dev {
    int32_t seq_len, block_m, block_n, n_rows, n_cols;
    int32_t n_full, n_part, n_load, n_pool;
    int32_t tile_bytes;         /* ceil(block_m*block_n/8): bytes per packed pool tile */
    int32_t* full_row_ptr;      /* n_rows+1 */
    int32_t* full_col_idx;      /* n_full   */
    int32_t* part_row_ptr;      /* n_rows+1 */
    int32_t* part_col_idx;      /* n_part   */
    int32_t* part_tile_ids;     /* n_part   */
    int32_t* load_row_ptr;      /* n_rows+1 */
    int32_t* load_col_idx;      /* n_load   */
    int32_t* load_tile;         /* n_load: -1 full, else pool id (device-only addition) */
    uint8_t* pool;              /* n_pool * tile_bytes, pack_bits order (common.hpp:77-83) */
    void* _alloc;               /* owned device block; release with sf_bsr_free */
} sf_bsr_dev;

/* Build the dual BSR of a device bit mask, bit-exact with build_bsr: tile classes, row-major
 * column order, and the part pool interned in first-occurrence row-major order
 * (bsr.hpp:64-94). Allocates device arrays (stream-ordered); synchronizes once to size them. */
sf_status sf_bsr_build(const uint32_t* d_bits, int32_t seq_len, int32_t block_m, int32_t block_n,
                       sf_bsr_dev* out, void* stream);
sf_status sf_bsr_free(sf_bsr_dev* bsr, void* stream);

/* Graph-capturable rebuilds (masks that change per request): sf_bsr_workspace allocates a BSR
 * sized for the whole tile grid (n_full / n_part / n_load / n_pool then hold capacities);
 * sf_bsr_build_async rebuilds it from a device mask with no host synchronisation, so the call can
 * sit inside a CUDA graph; the arrays equal sf_bsr_build's and d_counts[4] (device, optional)
 * receives n_full, n_part, n_load, n_pool. The attention executors walk the row pointers, so a
 * workspace BSR can be passed to sf_mha_blockwise directly (its stats report capacities). */
sf_status sf_bsr_workspace(int32_t seq_len, int32_t block_m, int32_t block_n, sf_bsr_dev* ws, void* stream);
sf_status sf_bsr_build_async(const uint32_t* d_bits, sf_bsr_dev* ws, int32_t* d_counts, void* stream);

/* Copy a device BSR into host arrays sized from the counts in `bsr` (any pointer may be NULL
 * to skip). `pool` receives n_pool*tile_bytes packed bytes. Synchronizes. */
sf_status sf_bsr_to_host(const sf_bsr_dev* bsr, int32_t* full_row_ptr, int32_t* full_col_idx,
                         int32_t* part_row_ptr, int32_t* part_col_idx, int32_t* part_tile_ids,
                         int32_t* load_row_ptr, int32_t* load_col_idx, uint8_t* pool,
                         void* stream);

/* SFBR dump bytes (io.hpp:97-122 write_bsr) of a device BSR. Pass buf=NULL to get the size
 * in *nbytes; otherwise writes min(cap, size) bytes. Synchronizes. */
sf_status sf_bsr_serialize(const sf_bsr_dev* bsr, uint8_t* buf, int64_t cap, int64_t* nbytes,
                           void* stream);

/* validate_bsr (bsr.hpp:104-153) on the device: SF_INTERNAL_INCONSISTENCY carrying the
 * reference's message for the first violation it would throw. Synchronizes. */
sf_status sf_bsr_validate(const sf_bsr_dev* bsr, void* stream);

/* to_dense (bsr.hpp:155-177): validate, then expand the full / part tiles into a device bit mask
 * of seq_len rows x sf_mask_words(seq_len) words (edge padding discarded). */
sf_status sf_bsr_to_dense(const sf_bsr_dev* bsr, uint32_t* d_bits, void* stream);

/* Device copy of host BSR arrays (e.g. a deserialised SFBR dump or a hand-built BsrMask);
 * `pool` holds n_pool packed tiles of ceil(block_m*block_n/8) bytes. Release with sf_bsr_free. */
sf_status sf_bsr_from_host(int32_t seq_len, int32_t block_m, int32_t block_n, int32_t n_full, int32_t n_part,
                           int32_t n_load, int32_t n_pool, const int32_t* full_row_ptr, const int32_t* full_col_idx,
                           const int32_t* part_row_ptr, const int32_t* part_col_idx, const int32_t* part_tile_ids,
                           const int32_t* load_row_ptr, const int32_t* load_col_idx, const uint8_t* pool,
                           sf_bsr_dev* out, void* stream);

typedef struct sf_csr_dev {
    int32_t seq_len;
    int64_t nnz;
    int32_t* row_ptr;   /* n+1 */
    int32_t* col_idx;   /* nnz */
    void* _alloc;
} sf_csr_dev;

/* Row-wise CSR of a device bit mask, bit-exact with build_rowwise (bsr.hpp:198-209). */
sf_status sf_rowwise_build(const uint32_t* d_bits, int32_t seq_len, sf_csr_dev* out,
                           void* stream);
sf_status sf_csr_free(sf_csr_dev* csr, void* stream);
/* Copy a device CSR to host arrays (n+1 and nnz int32). Synchronizes. */
sf_status sf_csr_to_host(const sf_csr_dev* csr, int32_t* row_ptr, int32_t* col_idx, void* stream);

/* ------------------------------------------------------------------------------------------
 * Analytical selector (planner.hpp:20-161). Host-side, exact doubles; the 16x16 load count
 * comes from the device builder.
 * ---------------------------------------------------------------------------------------- */
typedef struct sf_hw_spec {
    char name[32];
    int32_t sm_num;
    int64_t smem_size;
    int32_t max_warp;
    int32_t element_bytes;
} sf_hw_spec;

typedef enum sf_kernel_kind { SF_ROW_WISE = 0, SF_BLOCK_WISE = 1 } sf_kernel_kind;

typedef struct sf_plan {
    int32_t kind;       /* sf_kernel_kind */
    int32_t block_m, block_n, num_warps;
    double score;
    double threshold;   /* NaN when the n <= 16 shortcut fired */
    int32_t fallback;
} sf_plan;

typedef enum sf_plan_mode {
    SF_PLAN_REFERENCE = 0,  /* reference grid {16,32,64,128}^2 x {1,2,4,8}, planner.hpp:115-161 */
    SF_PLAN_B200 = 1        /* same Eq. 1/2, grid restricted to tiles the tcgen05 kernel runs;
                               then (sf_select_plan only: it needs the mask, head_size 64) both
                               executors are priced by the B200-calibrated cost model and the
                               faster one is kept, overriding Eq. 1 in either direction */
} sf_plan_mode;

/* hw_preset (planner.hpp:36-40) plus "b200". */
sf_status sf_hw_preset(const char* name, sf_hw_spec* out);
/* Eq. 1 threshold from a device mask (planner.hpp:67-76). */
sf_status sf_threshold(const uint32_t* d_bits, int32_t seq_len, double tau, double* out,
                       void* stream);
/* Eq. 1 from a precomputed 16x16 load count (the device builder's n_load). */
double sf_threshold_from_loads(int32_t seq_len, int64_t loads16, double tau);
sf_status sf_select_plan(const uint32_t* d_bits, const sf_hw_spec* hw, int64_t seq_len, int32_t h,
                         int64_t bs, int32_t head_size, int32_t mode, sf_plan* out, void* stream);
sf_status sf_select_plan_from_loads(int64_t loads16, const sf_hw_spec* hw, int64_t seq_len,
                                    int32_t h, int64_t bs, int32_t head_size, int32_t mode,
                                    sf_plan* out);

/* ------------------------------------------------------------------------------------------
 * Masked MHA (attention.hpp:71-213, planner.hpp:165-172).
 * ---------------------------------------------------------------------------------------- */
typedef enum sf_dtype { SF_F16 = 0, SF_BF16 = 1 } sf_dtype;

typedef struct sf_attn_args {
    int32_t bs, h, seq_len, head_size;
    int32_t dtype;                           /* sf_dtype */
    const void* q; const void* k; const void* v;
    void* o;
    int64_t q_sb, q_sh, q_sn;                /* element strides of q, k, v (shared) */
    int64_t o_sb, o_sh, o_sn;                /* element strides of o */
    float scale;                             /* 0 => 1/sqrt(head_size) (attention.hpp:77) */
} sf_attn_args;

typedef struct sf_attn_stats {               /* BlockExecStats, attention.hpp:60-64 */
    int64_t tiles_loaded, full_tiles, part_tiles;
} sf_attn_stats;

/* Block-wise executor over a device BSR. Replaces block_sparse_sdpa (attention.hpp:71-172) and
 * its plan-checked entry (planner.hpp:165-172): if `plan` is non-NULL it must be BlockWise
 * with matching block sizes or SF_PLAN_ERROR is returned. Dispatches to the tcgen05/TMA kernel
 * when (block_m, block_n, head_size, dtype) is one it implements, else the generic
 * CUDA-core block kernel (any tile shape). The tcgen05 kernel balances its work items through a
 * device work counter that the kernel resets itself: eager launches use the counter of their
 * stream (ordered launches), every launch captured into a CUDA graph gets a private one (so
 * graphs may be replayed concurrently on any streams, next to eager launches). Counters come from
 * a per-device pool that sf_bsr_build or the first eager launch creates. SF_ATTN_STATIC=1
 * selects the counter-free static deal. */
sf_status sf_mha_blockwise(const sf_attn_args* args, const sf_bsr_dev* bsr, const sf_plan* plan,
                           sf_attn_stats* stats, void* stream);
/* Row-wise gather executor over a device CSR. Replaces rowwise_sdpa (attention.hpp:177-213). */
sf_status sf_mha_rowwise(const sf_attn_args* args, const sf_csr_dev* csr, void* stream);

/* Masked MHA for the strided pattern (sf_pattern SF_PATTERN_STRIDED, band w) by mask decomposition:
 * strided(w) = causal-local(w) (disjoint-)union the diagonals i - j = k w, k >= 1. The band runs on
 * the tcgen05 block kernel over `band_bsr` (the block_m 128 or 64 — head pairs, the faster — BSR of
 * the causal-local(w) mask, e.g.
 * sf_mask_generate of {SF_PATTERN_CAUSAL_LOCAL, w} then sf_bsr_build), emitting per-row
 * log-sum-exp; the diagonals are exact dense causal attention inside each residue class i % w
 * (warp-level tensor-core MMAs) merged into the band's output. Same result semantics as
 * sf_mha_blockwise over the strided mask (attention.hpp:71-172). Needs head_size 64 and
 * ceil(seq_len / w) <= 128, else SF_PLAN_ERROR. */
sf_status sf_mha_strided(const sf_attn_args* args, int32_t band_width, const sf_bsr_dev* band_bsr, void* stream);

/* block_sparse_sdpa (attention.hpp:71-172) over a mask containing dilated(w, r) (mask.hpp:89-103),
 * by decomposition: dilated(w, r) pairs only rows and keys of one residue class mod s = r + 1, and
 * inside a class it is sliding(w) (mask.hpp:74-84) over n / s rows. Each class runs the tcgen05
 * block executor on the tensors' rows p, p + s, ... with class_bsr = build_bsr(sliding(w) over
 * n / s rows, 128, bn); rest_bsr (NULL or empty: none) = build_bsr(mask AND NOT dilated(w, r), 128, bn)
 * runs over the full rows, and the two parts are merged per row by log-sum-exp. Needs n % s == 0,
 * head_size 64, block_m 128 or 64 (head pairs) BSRs. SF_PLAN_ERROR otherwise (no launch). */
sf_status sf_mha_dilated(const sf_attn_args* args, int32_t stride, const sf_bsr_dev* class_bsr,
                         const sf_bsr_dev* rest_bsr, void* stream);

/* Dense masked SDPA reference on the device (dense_sdpa_oracle, attention.hpp:15-56): reads the
 * DENSE bit mask (sf_mask_generate's layout), accumulates in fp64 with the reference's exact
 * two-pass softmax, and writes fp64 output (bs, h, n, head_size) contiguous to `o64`. Rows with no
 * valid position are exactly zero. head_size even and <= 64. An executor independent of the
 * storage formats, used by `sparsefuse attn verify`; not a hot path. */
sf_status sf_mha_dense_oracle(const sf_attn_args* args, const uint32_t* d_bits, double* o64, void* stream);

/* Kernel selection for sf_mha_blockwise: 0 = auto, 1 = force generic CUDA-core kernel,
 * 2 = force tcgen05 kernel (fails with SF_PLAN_ERROR if the shape is unsupported). */
sf_status sf_set_attn_impl(int32_t impl);
int32_t sf_get_attn_impl(void);

/* ------------------------------------------------------------------------------------------
 * Fused segment templates (backend.hpp:109-306). GEMM operands fp16 (or bf16), row-major:
 * X (M x K), W^T stored as (N x K) row-major ("K-major", what TMA/tcgen05 read), out (M x N).
 * The epilogue applies, in order: +bias[N], activation, +aux[M x N] (residual Add),
 * LayerNorm over the full row (biased variance, eps 1e-5, backend.hpp:111,141-154) or a row
 * Softmax (max-subtracted, backend.hpp:155-167).
 * ---------------------------------------------------------------------------------------- */
typedef enum sf_act { SF_ACT_NONE = 0, SF_ACT_GELU = 1, SF_ACT_RELU = 2 } sf_act;

typedef struct sf_gemm_epilogue {
    const void* bias;        /* N, fp32 or NULL */
    int32_t act;             /* sf_act, applied after bias (backend.hpp:128-134) */
    const void* aux;         /* M x N residual (same dtype as out) or NULL; row stride ldaux */
    int64_t ldaux;
    const void* ln_gamma;    /* N fp32 or NULL: LayerNorm after the residual */
    const void* ln_beta;     /* N fp32 */
    void* out_pre_ln;        /* optional second output: the pre-LN row (residual stream) */
    int32_t softmax;         /* nonzero: row softmax after the residual (backend.hpp:155-167),
                                exclusive with LayerNorm; in sf_gemm_fused it runs as a MiChain
                                pass over the GEMM output */
} sf_gemm_epilogue;

#define SF_TILE_AUTO 0
#define SF_TILE_PAIR 1

typedef struct sf_gemm_args {
    int32_t M, N, K;
    int32_t dtype;           /* sf_dtype of X, W, out */
    const void* x; int64_t ldx;
    const void* w; int64_t ldw;   /* (N x K) row-major */
    void* out; int64_t ldout;
    sf_gemm_epilogue epi;
    int32_t tile_n;          /* output tiling (a tuning knob, params.hpp): SF_TILE_AUTO, 128 or 256
                                (one CTA per 128 x tile_n tile) or SF_TILE_PAIR (two-SM CTA pairs,
                                256 x 256 tiles, tcgen05 cta_group::2) */
} sf_gemm_args;

/* CiCi template (backend.hpp:270-306), chained on chip: out = post(mid(X . W1^T) . W2^T) with
 * mid = bias + activation (N1) and post = bias + aux residual + LayerNorm (N2) or any subset.
 * Each CTA computes a 128 x 128 block of the intermediate with tcgen05, applies mid in registers,
 * keeps it in shared memory as the next MMA's operand, multiplies it by its slice of W2 and
 * reduces into an fp32 accumulator (split-K over the intermediate); a row pass applies post. Meant
 * for the short activations where the reference's search forms CiCi segments (bs*seq <= 4096,
 * search.hpp:228). SF_BACKEND_ERROR when the shape is outside the kernel (K1 % 64, N1 % 128,
 * N2 % 64, N2 <= 2048) or mid carries more than bias + activation. Measured slower than two
 * sf_gemm_fused launches at the BERT FFN shapes (the split-K reduction), so only the
 * C++ GpuBackend offers it to the search, which times it against the split forms. */
typedef struct sf_gemm_chain_args {
    int32_t M, K1, N1, N2;
    int32_t dtype;                   /* sf_dtype of X, W1, W2, out, aux */
    const void* x; int64_t ldx;      /* M x K1 */
    const void* w1; int64_t ldw1;    /* N1 x K1 row-major */
    const void* w2; int64_t ldw2;    /* N2 x N1 row-major */
    void* out; int64_t ldout;        /* M x N2 */
    sf_gemm_epilogue mid;            /* bias (N1) and act only */
    sf_gemm_epilogue post;           /* bias (N2), aux, LayerNorm, out_pre_ln */
} sf_gemm_chain_args;
sf_status sf_gemm_chain(const sf_gemm_chain_args* args, void* stream);

/* Programmatic dependent launch for the hot-path kernels (default on; env SF_PDL=0 disables):
 * each kernel is scheduled while its stream predecessor drains and waits for it on device
 * (griddepcontrol) before touching global data. Not part of the reference API. */
sf_status sf_set_pdl(int32_t on);

/* CiMi template (backend.hpp:240-264): tcgen05 GEMM + fused epilogue. */
sf_status sf_gemm_fused(const sf_gemm_args* args, void* stream);

/* MiChain template (backend.hpp:228-235): out = LN/bias/act/add chain over a row-major M x N
 * fp16 matrix in one pass (same epilogue semantics as above, no GEMM). */
sf_status sf_mi_chain(int32_t M, int32_t N, int32_t dtype, const void* x, int64_t ldx,
                      const sf_gemm_epilogue* epi, void* out, int64_t ldout, void* stream);

/* ------------------------------------------------------------------------------------------
 * Measurement hook (backend.hpp:391-402): CUDA-event timing of a launch sequence.
 * ---------------------------------------------------------------------------------------- */
typedef sf_status (*sf_launch_fn)(void* user, void* stream);
/* Runs fn `warmup` times, then `reps` times each bracketed by CUDA events on `stream`;
 * writes the best (min) duration in milliseconds (CpuBackend protocol, backend.hpp:488-500). */
sf_status sf_time_best(sf_launch_fn fn, void* user, int32_t warmup, int32_t reps,
                       float* best_ms, void* stream);

/* Number of device kernels this library launched since load (counted host-side per launch). */
int64_t sf_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* SF_CAPI_H */
