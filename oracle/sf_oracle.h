/*
 * sf_oracle.h — CPU restatement of the STOF reference hot path, in plain C.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library, and only as the checker or the timed CPU
 * baseline — never as the product path. The product (paper_2506_06095_b200/csrc) does not link
 * it and fails loudly when its CUDA library is missing.
 *
 * Every function cites the reference file:line it restates
 * (/root/reference/proj/include/sparsefuse/...). Parity of this restatement is pinned against
 * the reference itself: oracle/_ref/libsfref.so is compiled from the unmodified reference
 * headers (oracle/Makefile) and tests/test_oracle_vs_ref.py compares the two bit-for-bit;
 * tests/golden/ holds fixtures produced by the reference (tests/golden/make_golden.py).
 */
#ifndef SF_ORACLE_H
#define SF_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/sf_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ---- foundation (common.hpp:39-83) ---- */
typedef struct sfo_mt64 { uint64_t mt[312]; int idx; } sfo_mt64;
void sfo_mt64_seed(sfo_mt64* g, uint64_t seed);
uint64_t sfo_mt64_next(sfo_mt64* g);
double sfo_unit_real(sfo_mt64* g);                      /* common.hpp:44-46 */
uint64_t sfo_mix_seed(uint64_t seed, uint64_t tag);     /* common.hpp:49-54 */
uint64_t sfo_fnv1a(const uint8_t* s, size_t n, uint64_t h); /* common.hpp:57-63 */
void sfo_pack_bits(const uint8_t* bits, size_t n, uint8_t* out); /* common.hpp:77-83 */

/* ---- masks: uint8 n*n row-major, 1 = valid (mask.hpp:18-54) ---- */
sf_status sfo_mask_generate(const sf_mask_desc* terms, int32_t n_terms, uint8_t* out);
int64_t sfo_mask_count(const uint8_t* m, int32_t n);

/* ---- formats (bsr.hpp) ---- */
typedef struct sfo_bsr {
    int32_t seq_len, block_m, block_n, n_rows, n_cols;
    int32_t n_full, n_part, n_load, n_pool;
    int32_t *full_row_ptr, *full_col_idx, *part_row_ptr, *part_col_idx, *part_tile_ids;
    int32_t *load_row_ptr, *load_col_idx;
    uint8_t* pool; /* n_pool * block_m*block_n bytes, unpacked like part_mask_pool */
} sfo_bsr;
sf_status sfo_build_bsr(const uint8_t* mask, int32_t n, int32_t bm, int32_t bn, sfo_bsr* out);
void sfo_bsr_free(sfo_bsr* b);
/* SFBR bytes (io.hpp:103-122); returns the byte count, writes when buf != NULL. */
int64_t sfo_bsr_serialize(const sfo_bsr* b, uint8_t* buf);
sf_status sfo_build_rowwise(const uint8_t* mask, int32_t n, int32_t* row_ptr, int32_t* col_idx,
                            int64_t cap, int64_t* nnz);

/* ---- attention (attention.hpp) ---- */
/* fp32 block-skipping online softmax, same loop order as attention.hpp:71-172. Slices
 * (b,h) are independent; n_threads > 1 runs them on pthreads. */
sf_status sfo_block_sparse_sdpa(const float* q, const float* k, const float* v, int32_t bs,
                                int32_t h, int32_t n, int32_t d, const sfo_bsr* bsr, float* out,
                                int64_t* stats3, int32_t n_threads);
/* fp64 row gather, exact two-pass softmax (attention.hpp:177-213). */
sf_status sfo_rowwise_sdpa(const double* q, const double* k, const double* v, int32_t bs,
                           int32_t h, int32_t n, int32_t d, const int32_t* row_ptr,
                           const int32_t* col_idx, double* out);
/* fp64 dense ground truth (attention.hpp:19-56). */
sf_status sfo_dense_sdpa(const double* q, const double* k, const double* v, int32_t bs, int32_t h,
                         int32_t n, int32_t d, const uint8_t* mask, double* out);
/* random_attention_input (tensor.hpp:62-73): q, k, v filled in that order from one stream. */
void sfo_random_attention_input(int32_t bs, int32_t h, int32_t n, int32_t d, uint64_t seed,
                                float* q, float* k, float* v);

/* ---- planner (planner.hpp) ---- */
sf_status sfo_hw_preset(const char* name, sf_hw_spec* out);
sf_status sfo_threshold(const uint8_t* mask, int32_t n, double tau, double* out);
double sfo_threshold_from_loads(int32_t n, int64_t loads16, double tau);
int64_t sfo_req_smem(int32_t bm, int32_t bn, int32_t head, int32_t padding);
double sfo_occupancy(int32_t warps, int64_t req_elems, const sf_hw_spec* hw);
double sfo_plan_score(int32_t bm, int32_t bn, int32_t w, const sf_hw_spec* hw, int64_t seq,
                      int32_t h, int64_t bs, int32_t head);
sf_status sfo_select_plan_from_loads(int64_t loads16, const sf_hw_spec* hw, int64_t seq,
                                     int32_t h, int64_t bs, int32_t head, int32_t mode,
                                     sf_plan* out);

/* ---- fused-template semantics (backend.hpp:43-306) ---- */
void sfo_random_matrix(int64_t rows, int64_t cols, uint64_t seed, float lo, float hi, float* out);
/* out[M x N] = in[M x K] * w[K x N] (w row-major K x N as GraphData stores it) */
void sfo_gemm(const float* in, const float* w, int64_t M, int64_t N, int64_t K, float* out,
              int32_t n_threads);
void sfo_bias(float* x, int64_t M, int64_t N, const float* bias);
void sfo_add(float* x, int64_t M, int64_t N, const float* aux);
void sfo_gelu(float* x, int64_t count);
void sfo_relu(float* x, int64_t count);
void sfo_layernorm(float* x, int64_t M, int64_t N, const float* gamma, const float* beta);
void sfo_softmax_rows(float* x, int64_t M, int64_t N);

#ifdef __cplusplus
}
#endif
#endif
