/*
 * sf_oracle.c — plain-C restatement of the reference hot path. TEST INFRASTRUCTURE ONLY
 * (see sf_oracle.h). Citations are to /root/reference/proj/include/sparsefuse/.
 *
 * Parity pinned against the compiled reference (oracle/_ref/libsfref.so) in
 * tests/test_oracle_vs_ref.py and against tests/golden/ fixtures.
 */
#include "sf_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------------------------
 * mt19937_64 (ISO C++ [rand.predef]); the reference draws through std::mt19937_64.
 * ---------------------------------------------------------------------------------------- */
#define MT_N 312
#define MT_M 156
void sfo_mt64_seed(sfo_mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < MT_N; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}
static void mt64_twist(sfo_mt64* g) {
    const uint64_t up = 0xFFFFFFFF80000000ULL, lo = 0x7FFFFFFFULL, a = 0xB5026F5AA96619E9ULL;
    for (int i = 0; i < MT_N; ++i) {
        uint64_t x = (g->mt[i] & up) | (g->mt[(i + 1) % MT_N] & lo);
        uint64_t xa = x >> 1;
        if (x & 1ULL) xa ^= a;
        g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ xa;
    }
    g->idx = 0;
}
uint64_t sfo_mt64_next(sfo_mt64* g) {
    if (g->idx >= MT_N) mt64_twist(g);
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}
/* common.hpp:44-46: top 53 bits scaled by 2^-53 */
double sfo_unit_real(sfo_mt64* g) { return (double)(sfo_mt64_next(g) >> 11) * 0x1.0p-53; }
/* common.hpp:49-54: splitmix64 finalizer over seed + golden*(tag+1) */
uint64_t sfo_mix_seed(uint64_t seed, uint64_t tag) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
/* common.hpp:57-63 */
uint64_t sfo_fnv1a(const uint8_t* s, size_t n, uint64_t h) {
    for (size_t i = 0; i < n; ++i) { h ^= s[i]; h *= 0x100000001b3ULL; }
    return h;
}
/* common.hpp:77-83: row-major, LSB-first within each byte */
void sfo_pack_bits(const uint8_t* bits, size_t n, uint8_t* out) {
    memset(out, 0, (n + 7) / 8);
    for (size_t i = 0; i < n; ++i)
        if (bits[i]) out[i >> 3] |= (uint8_t)(1u << (i & 7));
}

/* ------------------------------------------------------------------------------------------
 * Masks. Each term is written as a predicate / tile fill and OR-ed into the output
 * (compose, mask.hpp:146-166). Parameter checks follow the generators' throw sites.
 * ---------------------------------------------------------------------------------------- */
static sf_status check_term(const sf_mask_desc* t) {
    const int n = t->seq_len;
    if (n <= 0) return SF_INVALID_PARAMETER;                       /* mask.hpp:23 */
    switch (t->pattern) {
        case SF_PATTERN_SLIDING:
        case SF_PATTERN_CAUSAL_LOCAL:
        case SF_PATTERN_STRIDED:
            if (t->band_width < 1 || t->band_width > n) return SF_INVALID_PARAMETER; /* :75 */
            return SF_OK;
        case SF_PATTERN_DILATED:
            if (t->band_width < 1 || t->band_width > n) return SF_INVALID_PARAMETER; /* :90 */
            if (t->dilation_rate < 0) return SF_INVALID_PARAMETER;                   /* :92 */
            return SF_OK;
        case SF_PATTERN_GLOBAL:
            if (t->global_width < 0 || t->global_width > n) return SF_INVALID_PARAMETER; /* :108 */
            return SF_OK;
        case SF_PATTERN_RANDOM:
            if (t->block < 1) return SF_INVALID_PARAMETER;                           /* :125 */
            if (!(t->filling_rate >= 0.0 && t->filling_rate <= 1.0)) return SF_INVALID_PARAMETER;
            return SF_OK;
        case SF_PATTERN_LONGFORMER:  /* mask.hpp:169-171: global then sliding */
            if (t->global_width < 0 || t->global_width > n) return SF_INVALID_PARAMETER;
            if (t->band_width < 1 || t->band_width > n) return SF_INVALID_PARAMETER;
            return SF_OK;
        case SF_PATTERN_BIGBIRD:     /* mask.hpp:175-179: global, sliding, random */
            if (t->global_width < 0 || t->global_width > n) return SF_INVALID_PARAMETER;
            if (t->band_width < 1 || t->band_width > n) return SF_INVALID_PARAMETER;
            if (t->block < 1) return SF_INVALID_PARAMETER;
            if (!(t->filling_rate >= 0.0 && t->filling_rate <= 1.0)) return SF_INVALID_PARAMETER;
            return SF_OK;
        case SF_PATTERN_CAUSAL:
            return SF_OK;
        default:
            return SF_INVALID_PARAMETER;                               /* io.hpp:203 */
    }
}

static void or_sliding(uint8_t* m, int n, int w) {            /* mask.hpp:74-84 */
    for (int i = 0; i < n; ++i) {
        int lo = i - w + 1 < 0 ? 0 : i - w + 1;
        int hi = i + w - 1 > n - 1 ? n - 1 : i + w - 1;
        memset(m + (size_t)i * n + lo, 1, (size_t)(hi - lo + 1));
    }
}
static void or_dilated(uint8_t* m, int n, int w, int r) {      /* mask.hpp:89-103 */
    const int64_t stride = (int64_t)r + 1, reach = (int64_t)w * stride;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            int64_t d = (int64_t)i - j;
            int64_t ad = d < 0 ? -d : d;
            if (ad < reach && d % stride == 0) m[(size_t)i * n + j] = 1;
        }
}
static void or_global(uint8_t* m, int n, int g) {              /* mask.hpp:107-117 */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (i < g || j < g) m[(size_t)i * n + j] = 1;
}
static void or_random_blocks(uint8_t* m, int n, int block, double fill, uint64_t seed) {
    /* mask.hpp:124-143: one draw per tile of the ceil(n/block)^2 grid, row-major */
    const int grid = (n + block - 1) / block;
    sfo_mt64 g;
    sfo_mt64_seed(&g, seed);
    for (int bi = 0; bi < grid; ++bi)
        for (int bj = 0; bj < grid; ++bj) {
            double u = sfo_unit_real(&g);
            if (u >= fill) continue;
            int ie = (bi + 1) * block < n ? (bi + 1) * block : n;
            int je = (bj + 1) * block < n ? (bj + 1) * block : n;
            for (int i = bi * block; i < ie; ++i)
                memset(m + (size_t)i * n + (size_t)bj * block, 1, (size_t)(je - bj * block));
        }
}
static void or_causal_family(uint8_t* m, int n, int kind, int w) {
    /* No reference generator (SPEC.md:114 non-goal); predicates documented in sf_capi.h. */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            int d = i - j, ok;
            if (kind == SF_PATTERN_CAUSAL) ok = 1;
            else if (kind == SF_PATTERN_CAUSAL_LOCAL) ok = d < w;
            else ok = d < w || d % w == 0;
            if (ok) m[(size_t)i * n + j] = 1;
        }
}

sf_status sfo_mask_generate(const sf_mask_desc* terms, int32_t n_terms, uint8_t* out) {
    if (n_terms < 1) return SF_INVALID_PARAMETER;              /* mask.hpp:147 */
    const int n = terms[0].seq_len;
    for (int t = 0; t < n_terms; ++t) {
        sf_status s = check_term(&terms[t]);
        if (s != SF_OK) return s;
        if (terms[t].seq_len != n) return SF_SHAPE_ERROR;      /* mask.hpp:150 */
    }
    memset(out, 0, (size_t)n * n);
    for (int t = 0; t < n_terms; ++t) {
        const sf_mask_desc* d = &terms[t];
        switch (d->pattern) {
            case SF_PATTERN_SLIDING: or_sliding(out, n, d->band_width); break;
            case SF_PATTERN_DILATED: or_dilated(out, n, d->band_width, d->dilation_rate); break;
            case SF_PATTERN_GLOBAL: or_global(out, n, d->global_width); break;
            case SF_PATTERN_RANDOM:
                or_random_blocks(out, n, d->block, d->filling_rate, d->seed);
                break;
            case SF_PATTERN_LONGFORMER:
                or_global(out, n, d->global_width);
                or_sliding(out, n, d->band_width);
                break;
            case SF_PATTERN_BIGBIRD:
                or_global(out, n, d->global_width);
                or_sliding(out, n, d->band_width);
                or_random_blocks(out, n, d->block, d->filling_rate, d->seed);
                break;
            default: or_causal_family(out, n, d->pattern, d->band_width); break;
        }
    }
    return SF_OK;
}

int64_t sfo_mask_count(const uint8_t* m, int32_t n) {
    int64_t c = 0;
    for (size_t i = 0; i < (size_t)n * n; ++i) c += m[i];
    return c;
}

/* ------------------------------------------------------------------------------------------
 * build_bsr (bsr.hpp:47-101). Tiles are scanned row-major; mixed tiles are interned by their
 * packed bit content (a chained hash table keyed by FNV-1a of the packed bytes, compared by
 * memcmp) so pool ids are first-occurrence ranks.
 * ---------------------------------------------------------------------------------------- */
typedef struct { uint64_t h; int32_t id; } pool_slot;

sf_status sfo_build_bsr(const uint8_t* mask, int32_t n, int32_t bm, int32_t bn, sfo_bsr* b) {
    memset(b, 0, sizeof(*b));
    if (bm < 1 || bn < 1) return SF_INVALID_PARAMETER;         /* bsr.hpp:48 */
    if (n < 1) return SF_INVALID_PARAMETER;
    b->seq_len = n; b->block_m = bm; b->block_n = bn;
    b->n_rows = (n + bm - 1) / bm;
    b->n_cols = (n + bn - 1) / bn;
    const int64_t tiles = (int64_t)b->n_rows * b->n_cols;
    const size_t tsz = (size_t)bm * bn, psz = (tsz + 7) / 8;
    b->full_row_ptr = calloc((size_t)b->n_rows + 1, 4);
    b->part_row_ptr = calloc((size_t)b->n_rows + 1, 4);
    b->load_row_ptr = calloc((size_t)b->n_rows + 1, 4);
    /* first pass: classes, so the arrays can be sized exactly */
    uint8_t* cls = malloc((size_t)tiles);
    uint8_t* tile = malloc(tsz);
    for (int br = 0; br < b->n_rows; ++br)
        for (int bc = 0; bc < b->n_cols; ++bc) {
            int any_t = 0, any_f = 0;
            for (int di = 0; di < bm && !(any_t && any_f); ++di) {
                int i = br * bm + di;
                for (int dj = 0; dj < bn; ++dj) {
                    int j = bc * bn + dj;
                    int v = (i < n && j < n) ? mask[(size_t)i * n + j] != 0 : 0; /* bsr.hpp:72 */
                    if (v) any_t = 1; else any_f = 1;
                }
            }
            uint8_t c = !any_t ? 0 : (!any_f ? 1 : 2);
            cls[(size_t)br * b->n_cols + bc] = c;
            if (c == 1) { b->n_full++; b->full_row_ptr[br + 1]++; }
            if (c == 2) { b->n_part++; b->part_row_ptr[br + 1]++; }
            if (c) { b->n_load++; b->load_row_ptr[br + 1]++; }
        }
    for (int r = 0; r < b->n_rows; ++r) {                      /* bsr.hpp:95-99 */
        b->full_row_ptr[r + 1] += b->full_row_ptr[r];
        b->part_row_ptr[r + 1] += b->part_row_ptr[r];
        b->load_row_ptr[r + 1] += b->load_row_ptr[r];
    }
    b->full_col_idx = malloc((size_t)(b->n_full ? b->n_full : 1) * 4);
    b->part_col_idx = malloc((size_t)(b->n_part ? b->n_part : 1) * 4);
    b->part_tile_ids = malloc((size_t)(b->n_part ? b->n_part : 1) * 4);
    b->load_col_idx = malloc((size_t)(b->n_load ? b->n_load : 1) * 4);
    b->pool = malloc((size_t)(b->n_part ? b->n_part : 1) * tsz);
    uint8_t* packed_pool = malloc((size_t)(b->n_part ? b->n_part : 1) * psz);
    size_t cap = 16;
    while (cap < (size_t)b->n_part * 2) cap <<= 1;
    pool_slot* table = malloc(cap * sizeof(pool_slot));
    for (size_t s = 0; s < cap; ++s) table[s].id = -1;
    uint8_t* packed = malloc(psz);
    int fk = 0, pk = 0, lk = 0;
    for (int br = 0; br < b->n_rows; ++br)
        for (int bc = 0; bc < b->n_cols; ++bc) {
            uint8_t c = cls[(size_t)br * b->n_cols + bc];
            if (!c) continue;
            if (c == 1) {
                b->full_col_idx[fk++] = bc;
            } else {
                for (int di = 0; di < bm; ++di) {
                    int i = br * bm + di;
                    for (int dj = 0; dj < bn; ++dj) {
                        int j = bc * bn + dj;
                        tile[(size_t)di * bn + dj] =
                            (i < n && j < n) ? mask[(size_t)i * n + j] != 0 : 0;
                    }
                }
                sfo_pack_bits(tile, tsz, packed);
                uint64_t h = sfo_fnv1a(packed, psz, 0xcbf29ce484222325ULL);
                size_t s = (size_t)h & (cap - 1);
                int32_t id = -1;
                while (table[s].id >= 0) {
                    if (table[s].h == h &&
                        memcmp(packed_pool + (size_t)table[s].id * psz, packed, psz) == 0) {
                        id = table[s].id;
                        break;
                    }
                    s = (s + 1) & (cap - 1);
                }
                if (id < 0) {                                  /* bsr.hpp:84-86 */
                    id = b->n_pool++;
                    table[s].h = h;
                    table[s].id = id;
                    memcpy(packed_pool + (size_t)id * psz, packed, psz);
                    memcpy(b->pool + (size_t)id * tsz, tile, tsz);
                }
                b->part_col_idx[pk] = bc;
                b->part_tile_ids[pk++] = id;
            }
            b->load_col_idx[lk++] = bc;
        }
    free(packed); free(table); free(packed_pool); free(tile); free(cls);
    return SF_OK;
}

void sfo_bsr_free(sfo_bsr* b) {
    free(b->full_row_ptr); free(b->full_col_idx); free(b->part_row_ptr); free(b->part_col_idx);
    free(b->part_tile_ids); free(b->load_row_ptr); free(b->load_col_idx); free(b->pool);
    memset(b, 0, sizeof(*b));
}

static uint8_t* put_u32(uint8_t* p, uint32_t v) {
    if (p) { p[0] = (uint8_t)v; p[1] = (uint8_t)(v >> 8); p[2] = (uint8_t)(v >> 16); p[3] = (uint8_t)(v >> 24); return p + 4; }
    return NULL;
}
static int64_t put_arr(uint8_t** p, const int32_t* a, int32_t cnt) {
    if (*p) {
        *p = put_u32(*p, (uint32_t)cnt);
        for (int32_t i = 0; i < cnt; ++i) *p = put_u32(*p, (uint32_t)a[i]);
    }
    return 4 + 4 * (int64_t)cnt;
}
/* io.hpp:103-122: magic, version 1, seq_len, block_m, block_n, 7 arrays, pool count, tiles */
int64_t sfo_bsr_serialize(const sfo_bsr* b, uint8_t* buf) {
    uint8_t* p = buf;
    int64_t n = 0;
    if (p) { memcpy(p, "SFBR", 4); p += 4; }
    n += 4;
    p = put_u32(p, 1); p = put_u32(p, (uint32_t)b->seq_len);
    p = put_u32(p, (uint32_t)b->block_m); p = put_u32(p, (uint32_t)b->block_n);
    n += 16;
    n += put_arr(&p, b->full_row_ptr, b->n_rows + 1);
    n += put_arr(&p, b->full_col_idx, b->n_full);
    n += put_arr(&p, b->part_row_ptr, b->n_rows + 1);
    n += put_arr(&p, b->part_col_idx, b->n_part);
    n += put_arr(&p, b->part_tile_ids, b->n_part);
    n += put_arr(&p, b->load_row_ptr, b->n_rows + 1);
    n += put_arr(&p, b->load_col_idx, b->n_load);
    p = put_u32(p, (uint32_t)b->n_pool);
    n += 4;
    const size_t tsz = (size_t)b->block_m * b->block_n, psz = (tsz + 7) / 8;
    for (int32_t t = 0; t < b->n_pool; ++t) {
        if (p) { sfo_pack_bits(b->pool + (size_t)t * tsz, tsz, p); p += psz; }
        n += (int64_t)psz;
    }
    return n;
}

/* bsr.hpp:198-209 */
sf_status sfo_build_rowwise(const uint8_t* mask, int32_t n, int32_t* row_ptr, int32_t* col_idx,
                            int64_t cap, int64_t* nnz) {
    int64_t k = 0;
    row_ptr[0] = 0;
    for (int i = 0; i < n; ++i) {
        for (int j = 0; j < n; ++j)
            if (mask[(size_t)i * n + j]) {
                if (col_idx && k < cap) col_idx[k] = j;
                ++k;
            }
        row_ptr[i + 1] = (int32_t)k;
    }
    *nnz = k;
    return (col_idx && k > cap) ? SF_INVALID_PARAMETER : SF_OK;
}

/* ------------------------------------------------------------------------------------------
 * Attention.
 * ---------------------------------------------------------------------------------------- */
typedef struct {
    const float *q, *k, *v;
    float* out;
    int32_t h, n, d;
    const sfo_bsr* b;
    int64_t slice_begin, slice_end;
    int64_t stats[3];
} bsdpa_job;

/* One (b,h) slice of attention.hpp:87-167: per row block reset state, walk the load list with
 * the full/part merge walk, per row masked dot (scale after the dot), online rescale, exp*V. */
static void bsdpa_slice(const bsdpa_job* jb, int64_t slice, int count_tiles, int64_t* stats) {
    const sfo_bsr* b = jb->b;
    const int n = jb->n, d = jb->d, bm = b->block_m, bn = b->block_n;
    const float scale = 1.0f / sqrtf((float)d);
    const float ninf = -INFINITY;
    const size_t base = (size_t)slice * n * d;
    const float *Q = jb->q + base, *K = jb->k + base, *V = jb->v + base;
    float* O = jb->out + base;
    float* m_run = malloc(sizeof(float) * bm);
    float* l_run = malloc(sizeof(float) * bm);
    float* acc = malloc(sizeof(float) * (size_t)bm * d);
    float* s = malloc(sizeof(float) * (size_t)bm * bn);
    const size_t tsz = (size_t)bm * bn;
    for (int br = 0; br < b->n_rows; ++br) {
        const int i0 = br * bm;
        const int rows = bm < n - i0 ? bm : n - i0;
        if (rows <= 0) break;
        for (int r = 0; r < bm; ++r) { m_run[r] = ninf; l_run[r] = 0.0f; }
        memset(acc, 0, sizeof(float) * (size_t)bm * d);
        int32_t fk = b->full_row_ptr[br], fend = b->full_row_ptr[br + 1], pk = b->part_row_ptr[br];
        for (int32_t lk = b->load_row_ptr[br]; lk < b->load_row_ptr[br + 1]; ++lk) {
            const int bc = b->load_col_idx[lk];
            const int j0 = bc * bn;
            const int cols = bn < n - j0 ? bn : n - j0;
            if (cols <= 0) continue;
            const int is_full = fk < fend && b->full_col_idx[fk] == bc;
            const uint8_t* tile = NULL;
            if (is_full) ++fk;
            else tile = b->pool + (size_t)b->part_tile_ids[pk++] * tsz;
            if (count_tiles) { stats[0]++; stats[is_full ? 1 : 2]++; }
            for (int r = 0; r < rows; ++r) {
                float* srow = s + (size_t)r * bn;
                float tmax = ninf;
                const float* qr = Q + (size_t)(i0 + r) * d;
                for (int c = 0; c < cols; ++c) {
                    if (tile && !tile[(size_t)r * bn + c]) { srow[c] = ninf; continue; }
                    const float* kc = K + (size_t)(j0 + c) * d;
                    float dot = 0.0f;
                    for (int kk = 0; kk < d; ++kk) dot += qr[kk] * kc[kk];
                    srow[c] = dot * scale;
                    if (srow[c] > tmax) tmax = srow[c];
                }
                const float m_new = m_run[r] > tmax ? m_run[r] : tmax;
                if (m_new == ninf) continue;
                const float rescale = m_run[r] == ninf ? 0.0f : expf(m_run[r] - m_new);
                l_run[r] *= rescale;
                float* arow = acc + (size_t)r * d;
                for (int kk = 0; kk < d; ++kk) arow[kk] *= rescale;
                for (int c = 0; c < cols; ++c) {
                    if (srow[c] == ninf) continue;
                    const float p = expf(srow[c] - m_new);
                    l_run[r] += p;
                    const float* vc = V + (size_t)(j0 + c) * d;
                    for (int kk = 0; kk < d; ++kk) arow[kk] += p * vc[kk];
                }
                m_run[r] = m_new;
            }
        }
        for (int r = 0; r < rows; ++r) {                       /* attention.hpp:160-166 */
            const float l = l_run[r];
            if (l <= 0.0f) continue;
            const float inv = 1.0f / l;
            for (int kk = 0; kk < d; ++kk) O[(size_t)(i0 + r) * d + kk] = acc[(size_t)r * d + kk] * inv;
        }
    }
    free(m_run); free(l_run); free(acc); free(s);
}

static void* bsdpa_worker(void* arg) {
    bsdpa_job* jb = (bsdpa_job*)arg;
    for (int64_t sl = jb->slice_begin; sl < jb->slice_end; ++sl)
        bsdpa_slice(jb, sl, sl == 0, jb->stats);
    return NULL;
}

sf_status sfo_block_sparse_sdpa(const float* q, const float* k, const float* v, int32_t bs,
                                int32_t h, int32_t n, int32_t d, const sfo_bsr* bsr, float* out,
                                int64_t* stats3, int32_t n_threads) {
    if (bs < 1 || h < 1 || n < 1 || d < 1) return SF_SHAPE_ERROR;  /* tensor.hpp:23 */
    if (bsr->seq_len != n) return SF_SHAPE_ERROR;                  /* attention.hpp:74 */
    memset(out, 0, sizeof(float) * (size_t)bs * h * n * d);
    const int64_t slices = (int64_t)bs * h;
    if (n_threads < 1) n_threads = 1;
    if (n_threads > slices) n_threads = (int32_t)slices;
    bsdpa_job* jobs = calloc((size_t)n_threads, sizeof(bsdpa_job));
    pthread_t* th = calloc((size_t)n_threads, sizeof(pthread_t));
    for (int t = 0; t < n_threads; ++t) {
        jobs[t] = (bsdpa_job){q, k, v, out, h, n, d, bsr,
                              slices * t / n_threads, slices * (t + 1) / n_threads, {0, 0, 0}};
        if (n_threads > 1) pthread_create(&th[t], NULL, bsdpa_worker, &jobs[t]);
        else bsdpa_worker(&jobs[t]);
    }
    if (n_threads > 1)
        for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    if (stats3) {
        stats3[0] = stats3[1] = stats3[2] = 0;
        for (int t = 0; t < n_threads; ++t)
            for (int c = 0; c < 3; ++c) stats3[c] += jobs[t].stats[c];
    }
    free(jobs); free(th);
    return SF_OK;
}

sf_status sfo_rowwise_sdpa(const double* q, const double* k, const double* v, int32_t bs,
                           int32_t h, int32_t n, int32_t d, const int32_t* row_ptr,
                           const int32_t* col_idx, double* out) {
    if (bs < 1 || h < 1 || n < 1 || d < 1) return SF_SHAPE_ERROR;
    const double scale = 1.0 / sqrt((double)d);
    memset(out, 0, sizeof(double) * (size_t)bs * h * n * d);
    double* s = malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int64_t sl = 0; sl < (int64_t)bs * h; ++sl) {
        const size_t base = (size_t)sl * n * d;
        for (int i = 0; i < n; ++i) {
            const int32_t b0 = row_ptr[i], b1 = row_ptr[i + 1];
            if (b0 == b1) continue;                               /* attention.hpp:189 */
            double mx = -INFINITY;
            for (int32_t kk = b0; kk < b1; ++kk) {
                const int j = col_idx[kk];
                double dot = 0.0;
                for (int c = 0; c < d; ++c) dot += q[base + (size_t)i * d + c] * k[base + (size_t)j * d + c];
                s[kk - b0] = dot * scale;
                if (dot * scale > mx) mx = dot * scale;
            }
            double den = 0.0;
            for (int32_t kk = b0; kk < b1; ++kk) { s[kk - b0] = exp(s[kk - b0] - mx); den += s[kk - b0]; }
            for (int32_t kk = b0; kk < b1; ++kk) {
                const int j = col_idx[kk];
                const double p = s[kk - b0] / den;
                for (int c = 0; c < d; ++c) out[base + (size_t)i * d + c] += p * v[base + (size_t)j * d + c];
            }
        }
    }
    free(s);
    return SF_OK;
}

sf_status sfo_dense_sdpa(const double* q, const double* k, const double* v, int32_t bs, int32_t h,
                         int32_t n, int32_t d, const uint8_t* mask, double* out) {
    if (bs < 1 || h < 1 || n < 1 || d < 1) return SF_SHAPE_ERROR;
    const double scale = 1.0 / sqrt((double)d);
    memset(out, 0, sizeof(double) * (size_t)bs * h * n * d);
    double* s = malloc(sizeof(double) * (size_t)n);
    for (int64_t sl = 0; sl < (int64_t)bs * h; ++sl) {
        const size_t base = (size_t)sl * n * d;
        for (int i = 0; i < n; ++i) {
            double mx = -INFINITY;
            for (int j = 0; j < n; ++j) {
                if (!mask[(size_t)i * n + j]) { s[j] = -INFINITY; continue; }
                double dot = 0.0;
                for (int c = 0; c < d; ++c) dot += q[base + (size_t)i * d + c] * k[base + (size_t)j * d + c];
                s[j] = dot * scale;
                if (s[j] > mx) mx = s[j];
            }
            if (mx == -INFINITY) continue;                        /* attention.hpp:40 */
            double den = 0.0;
            for (int j = 0; j < n; ++j) if (s[j] != -INFINITY) den += exp(s[j] - mx);
            for (int j = 0; j < n; ++j) {
                if (s[j] == -INFINITY) continue;
                const double p = exp(s[j] - mx) / den;
                for (int c = 0; c < d; ++c) out[base + (size_t)i * d + c] += p * v[base + (size_t)j * d + c];
            }
        }
    }
    free(s);
    return SF_OK;
}

void sfo_random_attention_input(int32_t bs, int32_t h, int32_t n, int32_t d, uint64_t seed,
                                float* q, float* k, float* v) {
    sfo_mt64 g;
    sfo_mt64_seed(&g, seed);
    const size_t cnt = (size_t)bs * h * n * d;
    float* t[3] = {q, k, v};
    for (int a = 0; a < 3; ++a)
        for (size_t i = 0; i < cnt; ++i) t[a][i] = (float)(2.0 * sfo_unit_real(&g) - 1.0);
}

/* ------------------------------------------------------------------------------------------
 * Planner (planner.hpp:20-161).
 * ---------------------------------------------------------------------------------------- */
sf_status sfo_hw_preset(const char* name, sf_hw_spec* out) {
    memset(out, 0, sizeof(*out));
    if (!strcmp(name, "rtx4090")) { strcpy(out->name, "rtx4090"); out->sm_num = 128; out->smem_size = 128 * 1024; out->max_warp = 48; out->element_bytes = 2; return SF_OK; }
    if (!strcmp(name, "a100")) { strcpy(out->name, "a100"); out->sm_num = 108; out->smem_size = 192 * 1024; out->max_warp = 64; out->element_bytes = 2; return SF_OK; }
    /* Addition: B200 (sm_100a): 148 SMs, 228 KiB smem per SM, 64 warps per SM. */
    if (!strcmp(name, "b200")) { strcpy(out->name, "b200"); out->sm_num = 148; out->smem_size = 228 * 1024; out->max_warp = 64; out->element_bytes = 2; return SF_OK; }
    return SF_INVALID_PARAMETER;
}

double sfo_threshold_from_loads(int32_t n, int64_t loads16, double tau) {
    /* planner.hpp:67-76: L/N^2 - tau/(log2 N)^2, N = ceil(n/16) */
    const double big_n = (double)((n + 15) / 16);
    const double loads = (double)loads16;
    const double log_n = log2(big_n);
    return loads / (big_n * big_n) - tau / (log_n * log_n);
}

sf_status sfo_threshold(const uint8_t* mask, int32_t n, double tau, double* out) {
    if (n <= 16) return SF_DEGENERATE_INPUT;                      /* planner.hpp:69 */
    sfo_bsr b;
    sf_status s = sfo_build_bsr(mask, n, 16, 16, &b);
    if (s != SF_OK) return s;
    *out = sfo_threshold_from_loads(n, b.n_load, tau);
    sfo_bsr_free(&b);
    return SF_OK;
}

int64_t sfo_req_smem(int32_t bm, int32_t bn, int32_t head, int32_t padding) {
    /* planner.hpp:80-85 */
    return (int64_t)(2 * bm + bn) * (head + padding) + (int64_t)bm * (bn + padding);
}

double sfo_occupancy(int32_t warps, int64_t req_elems, const sf_hw_spec* hw) {
    /* planner.hpp:90-100 */
    const int64_t bytes = req_elems * hw->element_bytes;
    const int64_t by_smem = bytes > hw->smem_size ? 0 : hw->smem_size / bytes;
    const int64_t by_warp = hw->max_warp / warps;
    const int64_t blocks = by_smem < by_warp ? by_smem : by_warp;
    return (double)warps * (double)blocks / (double)hw->max_warp;
}

double sfo_plan_score(int32_t bm, int32_t bn, int32_t w, const sf_hw_spec* hw, int64_t seq,
                      int32_t h, int64_t bs, int32_t head) {
    /* planner.hpp:104-113 */
    const double occ = sfo_occupancy(w, sfo_req_smem(bm, bn, head, 16), hw);
    if (occ == 0.0) return 0.0;
    const double gran = sqrt((double)hw->sm_num / ((double)bm * bn));
    const double work = (double)seq * h * (double)bs / (double)bm;
    return occ * gran * work;
}

sf_status sfo_select_plan_from_loads(int64_t loads16, const sf_hw_spec* hw, int64_t seq,
                                     int32_t h, int64_t bs, int32_t head, int32_t mode,
                                     sf_plan* out) {
    /* planner.hpp:130-161 */
    if (hw->sm_num <= 0 || hw->smem_size <= 0 || hw->max_warp <= 0 || hw->element_bytes <= 0)
        return SF_INVALID_PARAMETER;
    if (h <= 0 || bs <= 0 || head <= 0) return SF_INVALID_PARAMETER;
    memset(out, 0, sizeof(*out));
    out->kind = SF_ROW_WISE;
    out->threshold = NAN;
    if (seq <= 16) return SF_OK;
    out->threshold = sfo_threshold_from_loads((int32_t)seq, loads16, 1.2);
    if (out->threshold < 0.0) return SF_OK;
    static const int sizes[4] = {16, 32, 64, 128};
    static const int warps[4] = {1, 2, 4, 8};
    double best = -1.0;
    for (int a = 0; a < 4; ++a)
        for (int c = 0; c < 4; ++c)
            for (int w = 0; w < 4; ++w) {
                /* B200 mode: only the tile shapes the tcgen05 kernel executes (M = 128). */
                if (mode == SF_PLAN_B200 && !(sizes[a] == 128 && head == 64)) continue;
                const double s = sfo_plan_score(sizes[a], sizes[c], warps[w], hw, seq, h, bs, head);
                if (s > 0.0 && s > best) {
                    best = s;
                    out->kind = SF_BLOCK_WISE;
                    out->block_m = sizes[a]; out->block_n = sizes[c]; out->num_warps = warps[w];
                    out->score = s;
                }
            }
    if (out->kind != SF_BLOCK_WISE) out->fallback = 1;
    return SF_OK;
}

/* ------------------------------------------------------------------------------------------
 * Fused-template semantics (backend.hpp:43-196; oracles.hpp:114-194 naive per-op form).
 * ---------------------------------------------------------------------------------------- */
void sfo_random_matrix(int64_t rows, int64_t cols, uint64_t seed, float lo, float hi, float* out) {
    /* backend.hpp:43-49 */
    sfo_mt64 g;
    sfo_mt64_seed(&g, seed);
    for (int64_t i = 0; i < rows * cols; ++i) out[i] = lo + (float)sfo_unit_real(&g) * (hi - lo);
}

typedef struct { const float *in, *w; int64_t M, N, K, r0, r1; float* out; } gemm_job;
static void* gemm_worker(void* arg) {
    gemm_job* j = (gemm_job*)arg;
    for (int64_t i = j->r0; i < j->r1; ++i) {
        float* o = j->out + (size_t)i * j->N;
        memset(o, 0, sizeof(float) * (size_t)j->N);
        for (int64_t k = 0; k < j->K; ++k) {
            const float x = j->in[(size_t)i * j->K + k];
            const float* wr = j->w + (size_t)k * j->N;
            for (int64_t c = 0; c < j->N; ++c) o[c] += x * wr[c];
        }
    }
    return NULL;
}
void sfo_gemm(const float* in, const float* w, int64_t M, int64_t N, int64_t K, float* out,
              int32_t n_threads) {
    if (n_threads < 1) n_threads = 1;
    if (n_threads > M) n_threads = (int32_t)(M > 0 ? M : 1);
    gemm_job* jobs = calloc((size_t)n_threads, sizeof(gemm_job));
    pthread_t* th = calloc((size_t)n_threads, sizeof(pthread_t));
    for (int t = 0; t < n_threads; ++t) {
        jobs[t] = (gemm_job){in, w, M, N, K, M * t / n_threads, M * (t + 1) / n_threads, out};
        if (n_threads > 1) pthread_create(&th[t], NULL, gemm_worker, &jobs[t]);
        else gemm_worker(&jobs[t]);
    }
    if (n_threads > 1)
        for (int t = 0; t < n_threads; ++t) pthread_join(th[t], NULL);
    free(jobs); free(th);
}
void sfo_bias(float* x, int64_t M, int64_t N, const float* bias) {     /* backend.hpp:119-121 */
    for (int64_t i = 0; i < M; ++i)
        for (int64_t j = 0; j < N; ++j) x[i * N + j] += bias[j];
}
void sfo_add(float* x, int64_t M, int64_t N, const float* aux) {       /* backend.hpp:122-127 */
    for (int64_t i = 0; i < M * N; ++i) x[i] += aux[i];
}
void sfo_gelu(float* x, int64_t count) {                               /* backend.hpp:128-131 */
    for (int64_t i = 0; i < count; ++i)
        x[i] = 0.5f * x[i] * (1.0f + erff(x[i] * 0.7071067811865475f));
}
void sfo_relu(float* x, int64_t count) {                               /* backend.hpp:132-134 */
    for (int64_t i = 0; i < count; ++i) x[i] = x[i] > 0.0f ? x[i] : 0.0f;
}
void sfo_layernorm(float* x, int64_t M, int64_t N, const float* gamma, const float* beta) {
    /* backend.hpp:141-154: two-pass mean / biased variance, eps 1e-5 */
    for (int64_t i = 0; i < M; ++i) {
        float* r = x + (size_t)i * N;
        float mean = 0.0f;
        for (int64_t j = 0; j < N; ++j) mean += r[j];
        mean /= (float)N;
        float var = 0.0f;
        for (int64_t j = 0; j < N; ++j) { const float dd = r[j] - mean; var += dd * dd; }
        var /= (float)N;
        const float inv = 1.0f / sqrtf(var + 1e-5f);
        for (int64_t j = 0; j < N; ++j) r[j] = (r[j] - mean) * inv * gamma[j] + beta[j];
    }
}
void sfo_softmax_rows(float* x, int64_t M, int64_t N) {                /* backend.hpp:155-163 */
    for (int64_t i = 0; i < M; ++i) {
        float* r = x + (size_t)i * N;
        float m = r[0];
        for (int64_t j = 1; j < N; ++j) m = r[j] > m ? r[j] : m;
        float den = 0.0f;
        for (int64_t j = 0; j < N; ++j) { r[j] = expf(r[j] - m); den += r[j]; }
        for (int64_t j = 0; j < N; ++j) r[j] /= den;
    }
}
