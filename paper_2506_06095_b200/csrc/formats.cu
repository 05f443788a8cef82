// formats.cu — device builders for the storage formats, bit-exact with the reference.
//   sf_bsr_build     <- build_bsr     (bsr.hpp:47-101)
//   sf_rowwise_build <- build_rowwise (bsr.hpp:198-209)
//
// BSR pipeline (all stream-ordered; two small D2H syncs to size the outputs):
//   1. classify: one warp per tile; lanes walk the tile's rows, extract the bn-bit row slices
//      from the bit mask (cells past n read as 0, bsr.hpp:72), popcount -> empty/full/part,
//      and fold a 64-bit content hash (row index mixed in, so the fold is order-free).
//   2. per-tile-row counts -> single-CTA exclusive scans -> full/part/load row pointers.
//   3. compaction: one CTA per tile row; a block-wide scan of the full/part flags writes the
//      column lists in ascending column order (bsr.hpp:64-65 loop order).
//   4. dedup: open-addressing table keyed by content (hash compared first, then the tile bits
//      themselves); each slot keeps the MIN row-major tile index of its content via atomicMin.
//      A part entry whose own tile index equals its slot's minimum is a first occurrence.
//   5. exclusive scan of the first-occurrence flags over the row-major part list = pool ids in
//      first-occurrence order (bsr.hpp:84-88); ids are scattered back through the slots.
//   6. pool: one warp per distinct tile writes pack_bits(tile) (common.hpp:77-83).
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "scan.cuh"

namespace sf {
namespace {

struct Geo {
    int32_t n, words, bm, bn, n_rows, n_cols;
};

// Content hash + popcount of tile (br, bc); executed by one full warp.
__device__ __forceinline__ void tile_scan(const uint32_t* __restrict__ bits, const Geo& g,
                                          int64_t br, int64_t bc, int64_t* count_out,
                                          uint64_t* hash_out) {
    const int lane = threadIdx.x & 31;
    int64_t cnt = 0;
    uint64_t h = 0;
    const int64_t j0 = bc * g.bn;
    const int64_t jlim = imin64(g.n, j0 + g.bn);
    for (int di = lane; di < g.bm; di += 32) {
        // rows past n are all-invalid cells (bsr.hpp:72): they hash as zero bits, exactly like
        // an in-range all-zero row, so equal tile contents always get equal hashes.
        const int64_t i = br * g.bm + di;
        const uint32_t* row = bits + imin64(i, g.n - 1) * g.words;
        for (int64_t c = 0; c * 64 < g.bn; ++c) {
            const uint64_t v = i < g.n ? row_bits64(row, j0 + 64 * c, jlim) : 0ull;
            cnt += __popcll(v);
            h += mix64(v ^ (0x9e3779b97f4a7c15ull * static_cast<uint64_t>(di * 1024 + c + 1)));
        }
    }
    for (int o = 16; o; o >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        h += __shfl_xor_sync(0xffffffffu, h, o);
    }
    *count_out = cnt;
    *hash_out = h;
}

// cls: 0 empty, 1 full, 2 part
__global__ void classify_kernel(const uint32_t* __restrict__ bits, Geo g, uint8_t* __restrict__ cls,
                                uint64_t* __restrict__ hash) {
    const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int64_t tiles = static_cast<int64_t>(g.n_rows) * g.n_cols;
    if (warp >= tiles) return;
    const int64_t br = warp / g.n_cols, bc = warp - br * g.n_cols;
    int64_t cnt;
    uint64_t h;
    tile_scan(bits, g, br, bc, &cnt, &h);
    if ((threadIdx.x & 31) == 0) {
        const int64_t full = static_cast<int64_t>(g.bm) * g.bn;
        cls[warp] = cnt == 0 ? 0 : (cnt == full ? 1 : 2);
        hash[warp] = h;
    }
}

__device__ __forceinline__ int32_t block_excl_scan(int32_t v, int32_t* sh, int32_t* total) {
    // blockDim.x == 256
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int32_t x = v;
    for (int o = 1; o < 32; o <<= 1) {
        int32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sh[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int32_t s = lane < 8 ? sh[lane] : 0;
        for (int o = 1; o < 8; o <<= 1) {
            int32_t y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < 8) sh[lane] = s;
    }
    __syncthreads();
    const int32_t r = x - v + (wid ? sh[wid - 1] : 0);
    *total = sh[7];
    __syncthreads();
    return r;
}

__global__ void row_count_kernel(const uint8_t* __restrict__ cls, Geo g, int32_t* full_cnt,
                                 int32_t* part_cnt, int32_t* load_cnt) {
    const int64_t br = blockIdx.x;
    int32_t f = 0, p = 0;
    for (int64_t bc = threadIdx.x; bc < g.n_cols; bc += blockDim.x) {
        const uint8_t c = cls[br * g.n_cols + bc];
        f += c == 1;
        p += c == 2;
    }
    for (int o = 16; o; o >>= 1) {
        f += __shfl_xor_sync(0xffffffffu, f, o);
        p += __shfl_xor_sync(0xffffffffu, p, o);
    }
    __shared__ int32_t sf_[8], sp_[8];
    if ((threadIdx.x & 31) == 0) {
        sf_[threadIdx.x >> 5] = f;
        sp_[threadIdx.x >> 5] = p;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t F = 0, P = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { F += sf_[w]; P += sp_[w]; }
        full_cnt[br] = F;
        part_cnt[br] = P;
        load_cnt[br] = F + P;
    }
}

// One 256-thread CTA per tile row: ordered compaction of the three column lists.
__global__ void compact_kernel(const uint8_t* __restrict__ cls, Geo g,
                               const int32_t* __restrict__ full_ptr, const int32_t* __restrict__ part_ptr,
                               const int32_t* __restrict__ load_ptr, int32_t* full_col,
                               int32_t* part_col, int32_t* load_col, int32_t* part_lin,
                               int32_t* load_part) {
    __shared__ int32_t sh[8];
    const int64_t br = blockIdx.x;
    int32_t fo = full_ptr[br], po = part_ptr[br], lo = load_ptr[br];
    for (int64_t c0 = 0; c0 < g.n_cols; c0 += blockDim.x) {
        const int64_t bc = c0 + threadIdx.x;
        const uint8_t c = bc < g.n_cols ? cls[br * g.n_cols + bc] : 0;
        int32_t tf, tp;
        const int32_t ef = block_excl_scan(c == 1, sh, &tf);
        const int32_t ep = block_excl_scan(c == 2, sh, &tp);
        if (c == 1) full_col[fo + ef] = static_cast<int32_t>(bc);
        if (c == 2) {
            part_col[po + ep] = static_cast<int32_t>(bc);
            part_lin[po + ep] = static_cast<int32_t>(br * g.n_cols + bc);
        }
        if (c) {
            load_col[lo + ef + ep] = static_cast<int32_t>(bc);
            load_part[lo + ef + ep] = c == 2 ? po + ep : -1;
        }
        fo += tf;
        po += tp;
        lo += tf + tp;
    }
}

// Tile equality, one full warp: lanes take rows di = lane, lane+32, ... (independent loads, one
// ballot) instead of one thread walking all block_m rows serially.
__device__ __forceinline__ bool tiles_equal_warp(const uint32_t* __restrict__ bits, const Geo& g, int64_t ta,
                                                 int64_t tb) {
    const int lane = threadIdx.x & 31;
    const int64_t ar = ta / g.n_cols, ac = ta - ar * g.n_cols;
    const int64_t br_ = tb / g.n_cols, bc_ = tb - br_ * g.n_cols;
    bool diff = false;
    for (int di = lane; di < g.bm; di += 32) {
        const int64_t ia = ar * g.bm + di, ib = br_ * g.bm + di;
        for (int64_t c = 0; c * 64 < g.bn; ++c) {
            const int64_t ja = ac * g.bn + 64 * c, jb = bc_ * g.bn + 64 * c;
            const uint64_t va = ia < g.n ? row_bits64(bits + ia * g.words, ja, imin64(g.n, ac * g.bn + g.bn)) : 0ull;
            const uint64_t vb = ib < g.n ? row_bits64(bits + ib * g.words, jb, imin64(g.n, bc_ * g.bn + g.bn)) : 0ull;
            diff |= va != vb;
        }
    }
    return __ballot_sync(0xffffffffu, diff) == 0u;
}

// Intern part tiles by content: one warp per part tile; lane 0 probes the open-addressing table,
// the warp compares contents on a hash match. Each slot ends holding the smallest row-major tile
// id of its content class (atomicMin), which fixes the pool order to first occurrence
// (bsr.hpp:83-91).
__global__ void dedup_insert_kernel(const uint32_t* __restrict__ bits, Geo g, const int32_t* __restrict__ n_part_dev,
                                    const int32_t* __restrict__ part_lin, const uint64_t* __restrict__ hash,
                                    int32_t* table, uint32_t cap_mask, int32_t* part_slot) {
    const int64_t k = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (k >= *n_part_dev) return;
    const int lane = threadIdx.x & 31;
    const int32_t lin = part_lin[k];
    const uint64_t h = hash[lin];
    uint32_t s = static_cast<uint32_t>(h ^ (h >> 32)) & cap_mask;
    for (;;) {
        int32_t cur = 0;
        if (lane == 0) cur = atomicCAS(&table[s], -1, lin);
        cur = __shfl_sync(0xffffffffu, cur, 0);
        if (cur == -1) break;  // claimed an empty slot
        if (hash[cur] == h && tiles_equal_warp(bits, g, cur, lin)) {
            if (lane == 0) atomicMin(&table[s], lin);
            break;
        }
        s = (s + 1) & cap_mask;
    }
    if (lane == 0) part_slot[k] = static_cast<int32_t>(s);
}

// first-occurrence flags over the part list, 0 past the device count (so a scan over the
// capacity equals a scan over the list)
__global__ void first_flag_kernel(int64_t cap, const int32_t* __restrict__ n_part_dev, const int32_t* __restrict__ part_lin,
                                  const int32_t* __restrict__ table, const int32_t* __restrict__ part_slot,
                                  int32_t* first) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= cap) return;
    first[k] = k < *n_part_dev && table[part_slot[k]] == part_lin[k] ? 1 : 0;
}

__global__ void slot_id_kernel(const int32_t* __restrict__ n_part_dev, const int32_t* __restrict__ first,
                               const int32_t* __restrict__ first_scan, const int32_t* __restrict__ part_slot,
                               int32_t* slot_id, int32_t* pool_src) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= *n_part_dev) return;
    if (first[k]) {
        slot_id[part_slot[k]] = first_scan[k];
        pool_src[first_scan[k]] = static_cast<int32_t>(k);
    }
}

__global__ void tile_ids_kernel(const int32_t* __restrict__ n_part_dev, const int32_t* __restrict__ part_slot,
                                const int32_t* __restrict__ slot_id, int32_t* tile_ids) {
    const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (k >= *n_part_dev) return;
    tile_ids[k] = slot_id[part_slot[k]];
}

__global__ void load_tile_kernel(const int32_t* __restrict__ n_load_dev, const int32_t* __restrict__ load_part,
                                 const int32_t* __restrict__ tile_ids, int32_t* load_tile) {
    const int64_t l = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (l >= *n_load_dev) return;
    const int32_t k = load_part[l];
    load_tile[l] = k < 0 ? -1 : tile_ids[k];
}

// One warp per pool tile; each lane assembles whole 32-bit words of pack_bits(tile) (cells 32w ..
// 32w + 31, LSB first) from the tile's row segments with 64-bit row extracts, then stores the
// word's bytes. Launched for every part tile (an upper bound of the pool); the pool size is read
// on device, so the build needs no host round trip between the dedup and the pool write.
__global__ void pool_write_kernel(const uint32_t* __restrict__ bits, Geo g, const int32_t* __restrict__ n_pool_dev,
                                  const int32_t* __restrict__ pool_src,
                                  const int32_t* __restrict__ part_lin, int32_t tile_bytes,
                                  uint8_t* __restrict__ pool) {
    const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= *n_pool_dev) return;
    const int lane = threadIdx.x & 31;
    const int64_t lin = part_lin[pool_src[w]];
    const int64_t br = lin / g.n_cols, bc = lin - br * g.n_cols;
    const int64_t nbits = static_cast<int64_t>(g.bm) * g.bn;
    const int64_t jlim = imin64(g.n, bc * g.bn + g.bn);
    uint8_t* dst = pool + w * tile_bytes;
    for (int64_t word = lane; word * 4 < tile_bytes; word += 32) {
        uint32_t v = 0;
        int64_t t = word * 32;
        const int64_t tend = imin64(nbits, t + 32);
        while (t < tend) {
            const int64_t di = t / g.bn, dj = t - di * g.bn;
            const int len = static_cast<int>(imin64(g.bn - dj, tend - t));  // <= 32
            const int64_t i = br * g.bm + di;
            if (i < g.n) {
                const uint64_t seg = row_bits64(bits + i * g.words, bc * g.bn + dj, jlim);
                const uint32_t m = len == 32 ? ~0u : ((1u << len) - 1u);
                v |= (static_cast<uint32_t>(seg) & m) << (t - word * 32);
            }
            t += len;
        }
#pragma unroll
        for (int b = 0; b < 4; ++b)
            if (word * 4 + b < tile_bytes) dst[word * 4 + b] = static_cast<uint8_t>(v >> (8 * b));
    }
}

// ---- row-wise CSR ----
__global__ void row_popc_kernel(const uint32_t* __restrict__ bits, int32_t n, int32_t words,
                                int32_t* cnt) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const int lane = threadIdx.x & 31;
    int32_t c = 0;
    for (int w = lane; w < words; w += 32) c += __popc(bits[i * words + w]);
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) cnt[i] = c;
}

__global__ void row_compact_kernel(const uint32_t* __restrict__ bits, int32_t n, int32_t words,
                                   const int32_t* __restrict__ row_ptr, int32_t* __restrict__ col) {
    const int64_t i = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (i >= n) return;
    const int lane = threadIdx.x & 31;
    int32_t base = row_ptr[i];
    for (int w0 = 0; w0 < words; w0 += 32) {
        const int w = w0 + lane;
        uint32_t v = w < words ? bits[i * words + w] : 0u;
        const int c = __popc(v);
        int x = c;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        int pos = base + x - c;
        while (v) {
            const int b = __ffs(v) - 1;
            col[pos++] = w * 32 + b;
            v &= v - 1;
        }
        base += __shfl_sync(0xffffffffu, x, 31);
    }
}

// ---- validate_bsr / to_dense (bsr.hpp:104-177) ----
// The first violation the reference's validate_bsr would throw is the smallest 64-bit key
// (check group, row, position): groups in the reference's order (full, part, load CSRs, then the
// tile ids, the pool, the per-row union), rows ascending, within a CSR row "decreasing row_ptr"
// before the entries' "out of range" / "not strictly increasing" in column order.
enum : uint32_t {
    kVFront = 0, kVDecr = 1, kVRange = 2, kVIncr = 3, kVLen = 4,        // per CSR group (x 5 + group)
    kVIdRange = 15, kVPoolMixed = 16, kVLoadSum = 17, kVOverlap = 18, kVUnion = 19
};
__device__ __forceinline__ unsigned long long vkey(uint32_t group, int64_t row, uint32_t pos, uint32_t code) {
    return (static_cast<unsigned long long>(group) << 58) | (static_cast<unsigned long long>(row & 0x3ffffff) << 32) |
           (static_cast<unsigned long long>(pos & 0xffffff) << 8) | code;
}

struct VCsr {
    const int32_t* ptr;
    const int32_t* col;
    int32_t len;
};

// one thread per (CSR, row): group g in {0 full, 1 part, 2 load}
__global__ void validate_csr_kernel(VCsr f, VCsr pa, VCsr lo, int32_t n_rows, int32_t n_cols,
                                    unsigned long long* err) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= 3ll * (n_rows + 1)) return;
    const uint32_t gi = static_cast<uint32_t>(t / (n_rows + 1));
    const int64_t r = t - static_cast<int64_t>(gi) * (n_rows + 1);
    const VCsr c = gi == 0 ? f : (gi == 1 ? pa : lo);
    const uint32_t G = gi;  // key group
    if (r == n_rows) {  // trailing checks of check_csr: front == 0, col length == ptr.back()
        if (c.ptr[0] != 0) atomicMin(err, vkey(G, 0, 0, gi * 5 + kVFront));
        if (c.ptr[n_rows] != c.len) atomicMin(err, vkey(G, n_rows, 0, gi * 5 + kVLen));
        return;
    }
    const int32_t a = c.ptr[r], b = c.ptr[r + 1];
    if (a > b) {
        atomicMin(err, vkey(G, r, 0, gi * 5 + kVDecr));
        return;
    }
    for (int32_t k = a; k < b; ++k) {
        const uint32_t pos = static_cast<uint32_t>(k - a) * 2 + 1;
        if (k < 0 || k >= c.len) {  // the reference would read past the column array here
            atomicMin(err, vkey(G, n_rows, 0, gi * 5 + kVLen));
            return;
        }
        const int32_t v = c.col[k];
        if (v < 0 || v >= n_cols) {
            atomicMin(err, vkey(G, r, pos, gi * 5 + kVRange));
            return;
        }
        if (k > a && v <= c.col[k - 1]) {
            atomicMin(err, vkey(G, r, pos + 1, gi * 5 + kVIncr));
            return;
        }
    }
}

// tile ids in pool range (group 3), pool tiles mixed (group 4), per-row sum / disjointness /
// union (group 5). Launched only when the three CSRs passed (their indices are then safe).
__global__ void validate_rest_kernel(VCsr f, VCsr pa, VCsr lo, const int32_t* __restrict__ tile_ids, int32_t n_pool,
                                     const uint8_t* __restrict__ pool, int32_t tile_bytes, int64_t nbits,
                                     int32_t n_rows, unsigned long long* err) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t < pa.len) {
        const int32_t id = tile_ids[t];
        if (id < 0 || id >= n_pool) atomicMin(err, vkey(3, 0, static_cast<uint32_t>(t), kVIdRange));
    }
    if (t < n_pool) {
        int64_t ones = 0;
        const uint8_t* tp = pool + t * tile_bytes;
        for (int64_t byte = 0; byte * 8 < nbits; ++byte) {
            uint32_t v = tp[byte];
            const int64_t left = nbits - byte * 8;
            if (left < 8) v &= (1u << left) - 1u;
            ones += __popc(v);
        }
        if (ones == 0 || ones == nbits) atomicMin(err, vkey(4, t, 0, kVPoolMixed));
    }
    if (t < n_rows) {
        const int32_t f0 = f.ptr[t], f1 = f.ptr[t + 1], p0 = pa.ptr[t], p1 = pa.ptr[t + 1];
        const int32_t l0 = lo.ptr[t], l1 = lo.ptr[t + 1];
        if (l1 != f1 + p1) {  // the reference compares the raw prefix values
            atomicMin(err, vkey(5, t, 0, kVLoadSum));
            return;
        }
        // both lists are strictly increasing (checked): merge, look for a common column, then
        // compare the merged run with the load row
        int32_t i = f0, j = p0, k = l0;
        uint32_t code = 0;
        while (i < f1 || j < p1) {
            int32_t v;
            if (j >= p1 || (i < f1 && f.col[i] < pa.col[j])) v = f.col[i++];
            else if (i >= f1 || pa.col[j] < f.col[i]) v = pa.col[j++];
            else { code = kVOverlap; break; }
            if (code == 0 && (k >= l1 || lo.col[k] != v)) code = kVUnion;
            ++k;
        }
        if (code == 0 && k != l1) code = kVUnion;
        // std::equal(merged, load + ptr[r]) only reads merged.size() load entries: a longer load
        // row passes the union check itself (the sum check above already fixed the lengths)
        if (code) atomicMin(err, vkey(5, t, 0, code));
    }
}

// to_dense: one thread per (full or part entry, tile row); ORs the row's block_n bits into the
// bit-packed mask (neighbouring tiles may share a 32-bit word)
__global__ void to_dense_kernel(const int32_t* __restrict__ frp, const int32_t* __restrict__ fci, int32_t n_full,
                                const int32_t* __restrict__ prp, const int32_t* __restrict__ pci,
                                const int32_t* __restrict__ pti, int32_t n_part, const uint8_t* __restrict__ pool,
                                int32_t tile_bytes, Geo g, uint32_t* __restrict__ out) {
    const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t entries = static_cast<int64_t>(n_full) + n_part;
    if (t >= entries * g.bm) return;
    const int64_t e = t / g.bm;
    const int di = static_cast<int>(t - e * g.bm);
    const bool full = e < n_full;
    const int64_t k = full ? e : e - n_full;
    const int32_t* rp = full ? frp : prp;
    // row block of entry k: the last row whose pointer is <= k (binary search)
    int lo_ = 0, hi_ = g.n_rows;
    while (hi_ - lo_ > 1) {
        const int mid = (lo_ + hi_) >> 1;
        if (rp[mid] <= k) lo_ = mid; else hi_ = mid;
    }
    const int64_t br = lo_;
    const int64_t bc = full ? fci[k] : pci[k];
    const int64_t i = br * g.bm + di;
    if (i >= g.n) return;
    const uint8_t* tile = full ? nullptr : pool + static_cast<int64_t>(pti[k]) * tile_bytes;
    uint32_t* row = out + i * g.words;
    for (int dj0 = 0; dj0 < g.bn; dj0 += 32) {
        const int64_t j0 = bc * g.bn + dj0;
        if (j0 >= g.n) break;
        const int len = static_cast<int>(imin64(imin64(32, g.bn - dj0), g.n - j0));
        uint32_t v;
        if (full) {
            v = len == 32 ? ~0u : ((1u << len) - 1u);
        } else {  // bits [di*bn + dj0, +len) of the LSB-first packed tile
            const int64_t b0 = static_cast<int64_t>(di) * g.bn + dj0;
            uint64_t w = 0;
            for (int q = 0; q < 5; ++q) {
                const int64_t byte = (b0 >> 3) + q;
                if (byte < tile_bytes) w |= static_cast<uint64_t>(tile[byte]) << (8 * q);
            }
            v = static_cast<uint32_t>(w >> (b0 & 7));
            if (len < 32) v &= (1u << len) - 1u;
        }
        // place bits j0..j0+len-1 into the row's words
        const int64_t w0 = j0 >> 5;
        const int sh = static_cast<int>(j0 & 31);
        if (v << sh) atomicOr(&row[w0], v << sh);
        if (sh && sh + len > 32 && (v >> (32 - sh))) atomicOr(&row[w0 + 1], v >> (32 - sh));
    }
}

template <typename T>
T* carve(char*& p, int64_t count) {
    T* r = reinterpret_cast<T*>(p);
    p += ((count * static_cast<int64_t>(sizeof(T)) + 255) / 256) * 256;
    return r;
}

unsigned blocks_for(int64_t threads, int per = 256) {
    return static_cast<unsigned>(imax64(1, ceil_div(threads, per)));
}

}  // namespace
}  // namespace sf

using namespace sf;

namespace sf {
void attn_reserve_counters(cudaStream_t st);  // attn_tc.cu: the attention work-counter pool of this device
}

namespace {
// Phase-1 scratch: per-tile class + hash, per-row counts and row pointers, device totals
// (n_full, n_part, n_load, n_pool).
struct Scratch1 {
    uint8_t* cls;
    uint64_t* hash;
    int32_t *fcnt, *pcnt, *lcnt, *fptr, *pptr, *lptr, *totals;
};
int64_t scratch1_bytes(int64_t tiles, int64_t n_rows) {
    return ceil_div(tiles, 256) * 256 + ceil_div(tiles * 8, 256) * 256 + 6 * (ceil_div((n_rows + 1) * 4, 256) * 256) + 256;
}
Scratch1 carve_scratch1(char*& p, int64_t tiles, int64_t n_rows) {
    Scratch1 s;
    s.cls = carve<uint8_t>(p, tiles);
    s.hash = carve<uint64_t>(p, tiles);
    s.fcnt = carve<int32_t>(p, n_rows + 1);
    s.pcnt = carve<int32_t>(p, n_rows + 1);
    s.lcnt = carve<int32_t>(p, n_rows + 1);
    s.fptr = carve<int32_t>(p, n_rows + 1);
    s.pptr = carve<int32_t>(p, n_rows + 1);
    s.lptr = carve<int32_t>(p, n_rows + 1);
    s.totals = carve<int32_t>(p, 4);
    return s;
}
// Phase-2 (dedup) scratch for up to part_cap part tiles and load_cap loads.
struct Scratch2 {
    int32_t *part_lin, *part_slot, *first, *first_scan, *pool_src, *table, *slot_id, *load_part;
    uint32_t cap;
};
uint32_t table_cap(int64_t part_cap) {
    uint32_t cap = 16;
    while (cap < static_cast<uint32_t>(imax64(1, part_cap)) * 2u) cap <<= 1;
    return cap;
}
int64_t scratch2_bytes(int64_t part_cap, int64_t load_cap) {
    const int64_t np1 = imax64(1, part_cap);
    return 5 * ceil_div((np1 + 1) * 4, 256) * 256 + 2 * ceil_div(table_cap(part_cap) * 4ll, 256) * 256 +
           ceil_div(imax64(1, load_cap) * 4, 256) * 256;
}
Scratch2 carve_scratch2(char*& p, int64_t part_cap, int64_t load_cap) {
    Scratch2 s;
    const int64_t np1 = imax64(1, part_cap);
    s.cap = table_cap(part_cap);
    s.part_lin = carve<int32_t>(p, np1);
    s.part_slot = carve<int32_t>(p, np1);
    s.first = carve<int32_t>(p, np1);
    s.first_scan = carve<int32_t>(p, np1 + 1);
    s.pool_src = carve<int32_t>(p, np1);
    s.table = carve<int32_t>(p, s.cap);
    s.slot_id = carve<int32_t>(p, s.cap);
    s.load_part = carve<int32_t>(p, imax64(1, load_cap));
    return s;
}
// Output arrays of a BSR with room for the given counts.
int64_t out_bytes(int64_t n_rows, int64_t n_full, int64_t n_part, int64_t n_load, int64_t pool_bytes) {
    const int64_t rp = n_rows + 1;
    return 3 * ceil_div(rp * 4, 256) * 256 + ceil_div(imax64(1, n_full) * 4, 256) * 256 +
           2 * ceil_div(imax64(1, n_part) * 4, 256) * 256 + 2 * ceil_div(imax64(1, n_load) * 4, 256) * 256 +
           ceil_div(imax64(1, pool_bytes), 256) * 256;
}
void carve_out(char*& p, sf_bsr_dev* out, int64_t n_rows, int64_t n_full, int64_t n_part, int64_t n_load,
               int64_t pool_bytes) {
    const int64_t rp = n_rows + 1;
    out->full_row_ptr = carve<int32_t>(p, rp);
    out->part_row_ptr = carve<int32_t>(p, rp);
    out->load_row_ptr = carve<int32_t>(p, rp);
    out->full_col_idx = carve<int32_t>(p, imax64(1, n_full));
    out->part_col_idx = carve<int32_t>(p, imax64(1, n_part));
    out->part_tile_ids = carve<int32_t>(p, imax64(1, n_part));
    out->load_col_idx = carve<int32_t>(p, imax64(1, n_load));
    out->load_tile = carve<int32_t>(p, imax64(1, n_load));
    out->pool = carve<uint8_t>(p, imax64(1, pool_bytes));
}

// classify -> per-row counts -> the three row-pointer scans (written to fptr/pptr/lptr), device totals
sf_status bsr_phase1(const uint32_t* d_bits, const Geo& g, const Scratch1& s, int32_t* fptr, int32_t* pptr,
                     int32_t* lptr, cudaStream_t st) {
    const int64_t tiles = static_cast<int64_t>(g.n_rows) * g.n_cols;
    classify_kernel<<<blocks_for(tiles * 32), 256, 0, st>>>(d_bits, g, s.cls, s.hash);
    SF_LAUNCH_CHECK();
    row_count_kernel<<<g.n_rows, 256, 0, st>>>(s.cls, g, s.fcnt, s.pcnt, s.lcnt);
    SF_LAUNCH_CHECK();
    scan_exclusive3_kernel<<<dim3(1, 3), 1024, 0, st>>>(s.fcnt, s.pcnt, s.lcnt, fptr, pptr, lptr, g.n_rows, s.totals);
    SF_LAUNCH_CHECK();
    return SF_OK;
}

// compaction, content dedup, pool ids, pool bytes, load tile kinds; every count read on device
// (totals), launches sized by the capacities
sf_status bsr_phase2(const uint32_t* d_bits, const Geo& g, const sf_bsr_dev* out, const int32_t* fptr,
                     const int32_t* pptr, const int32_t* lptr, const Scratch1& s1, const Scratch2& s2,
                     int64_t part_cap, int64_t load_cap, int32_t tile_bytes, cudaStream_t st) {
    SF_CUDA_TRY(cudaMemsetAsync(s2.table, 0xff, s2.cap * 4ll, st));
    if (load_cap > 0) {
        compact_kernel<<<g.n_rows, 256, 0, st>>>(s1.cls, g, fptr, pptr, lptr, out->full_col_idx, out->part_col_idx,
                                                 out->load_col_idx, s2.part_lin, s2.load_part);
        SF_LAUNCH_CHECK();
    }
    const int32_t* n_part = s1.totals + 1;
    const int32_t* n_load = s1.totals + 2;
    int32_t* n_pool = s1.totals + 3;
    if (part_cap > 0) {
        dedup_insert_kernel<<<blocks_for(part_cap * 32), 256, 0, st>>>(d_bits, g, n_part, s2.part_lin, s1.hash,
                                                                       s2.table, s2.cap - 1, s2.part_slot);
        SF_LAUNCH_CHECK();
        first_flag_kernel<<<blocks_for(part_cap), 256, 0, st>>>(part_cap, n_part, s2.part_lin, s2.table, s2.part_slot,
                                                               s2.first);
        SF_LAUNCH_CHECK();
        SF_TRY(scan_exclusive(s2.first, s2.first_scan, part_cap, n_pool, st));
        slot_id_kernel<<<blocks_for(part_cap), 256, 0, st>>>(n_part, s2.first, s2.first_scan, s2.part_slot, s2.slot_id,
                                                            s2.pool_src);
        SF_LAUNCH_CHECK();
        tile_ids_kernel<<<blocks_for(part_cap), 256, 0, st>>>(n_part, s2.part_slot, s2.slot_id, out->part_tile_ids);
        SF_LAUNCH_CHECK();
        pool_write_kernel<<<blocks_for(part_cap * 32), 256, 0, st>>>(d_bits, g, n_pool, s2.pool_src, s2.part_lin,
                                                                     tile_bytes, out->pool);
        SF_LAUNCH_CHECK();
    } else {
        SF_CUDA_TRY(cudaMemsetAsync(n_pool, 0, 4, st));
    }
    if (load_cap > 0) {
        load_tile_kernel<<<blocks_for(load_cap), 256, 0, st>>>(n_load, s2.load_part, out->part_tile_ids, out->load_tile);
        SF_LAUNCH_CHECK();
    }
    return SF_OK;
}

bool bsr_args_ok(const uint32_t* d_bits, int32_t seq_len, int32_t block_m, int32_t block_n, sf_status* st) {
    if (block_m < 1 || block_n < 1) { *st = fail(SF_INVALID_PARAMETER, "block sizes must be >= 1"); return false; }
    if (seq_len < 1) { *st = fail(SF_INVALID_PARAMETER, "seq_len must be positive"); return false; }
    if (!d_bits) { *st = fail(SF_INVALID_PARAMETER, "null mask"); return false; }
    const int64_t tiles = ceil_div(seq_len, block_m) * ceil_div(seq_len, block_n);
    if (tiles > (1ll << 31) - 1) { *st = fail(SF_INVALID_PARAMETER, "tile grid too large"); return false; }
    return true;
}
}  // namespace

extern "C" sf_status sf_bsr_build(const uint32_t* d_bits, int32_t seq_len, int32_t block_m,
                                  int32_t block_n, sf_bsr_dev* out, void* stream) {
    if (!out) return fail(SF_INVALID_PARAMETER, "null output");
    *out = sf_bsr_dev{};
    sf_status bad = SF_OK;
    if (!bsr_args_ok(d_bits, seq_len, block_m, block_n, &bad)) return bad;
    cudaStream_t st = as_stream(stream);
    sf::attn_reserve_counters(st);
    Geo g{seq_len, sf_mask_words(seq_len), block_m, block_n,
          static_cast<int32_t>(ceil_div(seq_len, block_m)), static_cast<int32_t>(ceil_div(seq_len, block_n))};
    const int64_t tiles = static_cast<int64_t>(g.n_rows) * g.n_cols;
    const int32_t tile_bytes = static_cast<int32_t>(ceil_div(static_cast<int64_t>(block_m) * block_n, 8));

    // phase 1, then the exact output sizes read back (this entry's one host round trip; use
    // sf_bsr_build_async on a worst-case workspace to rebuild inside a CUDA graph)
    char* s1b = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&s1b), scratch1_bytes(tiles, g.n_rows), st));
    char* p = s1b;
    const Scratch1 s1 = carve_scratch1(p, tiles, g.n_rows);
    sf_status rc = bsr_phase1(d_bits, g, s1, s1.fptr, s1.pptr, s1.lptr, st);
    int32_t h_tot[3] = {0, 0, 0};
    if (rc == SF_OK && cudaMemcpyAsync(h_tot, s1.totals, 12, cudaMemcpyDeviceToHost, st) != cudaSuccess)
        rc = fail(SF_CUDA_ERROR, "cudaMemcpyAsync (BSR sizes)");
    if (rc == SF_OK && cudaStreamSynchronize(st) != cudaSuccess) rc = fail(SF_CUDA_ERROR, "cudaStreamSynchronize");
    if (rc != SF_OK) {
        cudaFreeAsync(s1b, st);
        return rc;
    }
    const int32_t n_full = h_tot[0], n_part = h_tot[1], n_load = h_tot[2];

    // outputs (owned by the sf_bsr_dev), sized exactly; the pool for the worst case of n_part
    char* ob = nullptr;
    char* s2b = nullptr;
    const int64_t pool_cap = static_cast<int64_t>(n_part) * tile_bytes;
    if (pool_malloc(reinterpret_cast<void**>(&ob), out_bytes(g.n_rows, n_full, n_part, n_load, pool_cap), st) !=
            cudaSuccess ||
        pool_malloc(reinterpret_cast<void**>(&s2b), scratch2_bytes(n_part, n_load), st) != cudaSuccess) {
        cudaGetLastError();
        if (ob) cudaFreeAsync(ob, st);
        cudaFreeAsync(s1b, st);
        return fail(SF_CUDA_ERROR, "BSR output allocation failed");
    }
    p = ob;
    carve_out(p, out, g.n_rows, n_full, n_part, n_load, pool_cap);
    out->_alloc = ob;
    p = s2b;
    const Scratch2 s2 = carve_scratch2(p, n_part, n_load);
    // the three row-pointer arrays are carved identically (256-byte aligned, back to back) in the
    // scratch and in the output block: one copy moves all three
    rc = cudaMemcpyAsync(out->full_row_ptr, s1.fptr,
                         static_cast<size_t>(reinterpret_cast<char*>(out->load_row_ptr) -
                                             reinterpret_cast<char*>(out->full_row_ptr)) + (g.n_rows + 1) * 4ll,
                         cudaMemcpyDeviceToDevice, st) == cudaSuccess
             ? SF_OK
             : fail(SF_CUDA_ERROR, "cudaMemcpyAsync (row pointers)");
    if (rc == SF_OK) rc = bsr_phase2(d_bits, g, out, s1.fptr, s1.pptr, s1.lptr, s1, s2, n_part, n_load, tile_bytes, st);
    int32_t n_pool = 0;
    if (rc == SF_OK && n_part > 0) {  // the pool size for the host struct: the build's trailing sync
        if (cudaMemcpyAsync(&n_pool, s1.totals + 3, 4, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            rc = fail(SF_CUDA_ERROR, "BSR pool size read-back");
    }
    cudaFreeAsync(s2b, st);
    cudaFreeAsync(s1b, st);
    if (rc != SF_OK) {
        cudaFreeAsync(ob, st);
        *out = sf_bsr_dev{};
        return rc;
    }
    out->seq_len = seq_len;
    out->block_m = block_m;
    out->block_n = block_n;
    out->n_rows = g.n_rows;
    out->n_cols = g.n_cols;
    out->n_full = n_full;
    out->n_part = n_part;
    out->n_load = n_load;
    out->n_pool = n_pool;
    out->tile_bytes = tile_bytes;
    return SF_OK;
}

// Worst-case workspace: outputs sized for the whole tile grid (every tile full, part and loaded;
// the pool for every tile), followed by both scratch blocks, in one owned allocation.
extern "C" sf_status sf_bsr_workspace(int32_t seq_len, int32_t block_m, int32_t block_n, sf_bsr_dev* ws,
                                      void* stream) {
    if (!ws) return fail(SF_INVALID_PARAMETER, "null output");
    *ws = sf_bsr_dev{};
    sf_status bad = SF_OK;
    const uint32_t dummy = 0;
    if (!bsr_args_ok(&dummy, seq_len, block_m, block_n, &bad)) return bad;
    cudaStream_t st = as_stream(stream);
    sf::attn_reserve_counters(st);
    const int64_t n_rows = ceil_div(seq_len, block_m), n_cols = ceil_div(seq_len, block_n), tiles = n_rows * n_cols;
    const int32_t tile_bytes = static_cast<int32_t>(ceil_div(static_cast<int64_t>(block_m) * block_n, 8));
    const int64_t total = out_bytes(n_rows, tiles, tiles, tiles, tiles * tile_bytes) + scratch1_bytes(tiles, n_rows) +
                          scratch2_bytes(tiles, tiles);
    char* blk = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&blk), total, st));
    char* p = blk;
    carve_out(p, ws, n_rows, tiles, tiles, tiles, tiles * tile_bytes);
    ws->_alloc = blk;
    ws->seq_len = seq_len;
    ws->block_m = block_m;
    ws->block_n = block_n;
    ws->n_rows = static_cast<int32_t>(n_rows);
    ws->n_cols = static_cast<int32_t>(n_cols);
    ws->n_full = ws->n_part = ws->n_load = ws->n_pool = static_cast<int32_t>(tiles);  // capacities
    ws->tile_bytes = tile_bytes;
    return SF_OK;
}

extern "C" sf_status sf_bsr_build_async(const uint32_t* d_bits, sf_bsr_dev* ws, int32_t* d_counts, void* stream) {
    if (!ws || !ws->_alloc) return fail(SF_INVALID_PARAMETER, "BSR workspace not allocated (sf_bsr_workspace)");
    sf_status bad = SF_OK;
    if (!bsr_args_ok(d_bits, ws->seq_len, ws->block_m, ws->block_n, &bad)) return bad;
    cudaStream_t st = as_stream(stream);
    const Geo g{ws->seq_len, sf_mask_words(ws->seq_len), ws->block_m, ws->block_n, ws->n_rows, ws->n_cols};
    const int64_t tiles = static_cast<int64_t>(g.n_rows) * g.n_cols;
    char* p = static_cast<char*>(ws->_alloc);
    sf_bsr_dev layout{};
    carve_out(p, &layout, g.n_rows, tiles, tiles, tiles, tiles * ws->tile_bytes);  // skip the output block
    const Scratch1 s1 = carve_scratch1(p, tiles, g.n_rows);
    const Scratch2 s2 = carve_scratch2(p, tiles, tiles);
    // the row pointers are scanned straight into the workspace's output arrays
    SF_TRY(bsr_phase1(d_bits, g, s1, ws->full_row_ptr, ws->part_row_ptr, ws->load_row_ptr, st));
    SF_TRY(bsr_phase2(d_bits, g, ws, ws->full_row_ptr, ws->part_row_ptr, ws->load_row_ptr, s1, s2, tiles, tiles,
                      ws->tile_bytes, st));
    if (d_counts) SF_CUDA_TRY(cudaMemcpyAsync(d_counts, s1.totals, 16, cudaMemcpyDeviceToDevice, st));
    return SF_OK;
}

extern "C" sf_status sf_bsr_free(sf_bsr_dev* bsr, void* stream) {
    if (!bsr) return SF_OK;
    if (bsr->_alloc) SF_CUDA_TRY(cudaFreeAsync(bsr->_alloc, as_stream(stream)));
    *bsr = sf_bsr_dev{};
    return SF_OK;
}

extern "C" sf_status sf_bsr_to_host(const sf_bsr_dev* b, int32_t* full_row_ptr, int32_t* full_col_idx,
                                    int32_t* part_row_ptr, int32_t* part_col_idx, int32_t* part_tile_ids,
                                    int32_t* load_row_ptr, int32_t* load_col_idx, uint8_t* pool,
                                    void* stream) {
    cudaStream_t st = as_stream(stream);
    const int64_t rp = (b->n_rows + 1) * 4ll;
    auto cp = [&](void* dst, const void* src, int64_t bytes) -> sf_status {
        if (dst && bytes > 0) SF_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
        return SF_OK;
    };
    SF_TRY(cp(full_row_ptr, b->full_row_ptr, rp));
    SF_TRY(cp(part_row_ptr, b->part_row_ptr, rp));
    SF_TRY(cp(load_row_ptr, b->load_row_ptr, rp));
    SF_TRY(cp(full_col_idx, b->full_col_idx, b->n_full * 4ll));
    SF_TRY(cp(part_col_idx, b->part_col_idx, b->n_part * 4ll));
    SF_TRY(cp(part_tile_ids, b->part_tile_ids, b->n_part * 4ll));
    SF_TRY(cp(load_col_idx, b->load_col_idx, b->n_load * 4ll));
    SF_TRY(cp(pool, b->pool, static_cast<int64_t>(b->n_pool) * b->tile_bytes));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    return SF_OK;
}

extern "C" sf_status sf_bsr_serialize(const sf_bsr_dev* b, uint8_t* buf, int64_t cap, int64_t* nbytes,
                                      void* stream) {
    // io.hpp:103-122 layout
    const int64_t rp = b->n_rows + 1;
    const int64_t size = 4 + 16 + 7 * 4 + 4 * (3 * rp + b->n_full + 2ll * b->n_part + b->n_load) + 4 +
                         static_cast<int64_t>(b->n_pool) * b->tile_bytes;
    if (nbytes) *nbytes = size;
    if (!buf) return SF_OK;
    if (cap < size) return fail(SF_INVALID_PARAMETER, "buffer smaller than the SFBR dump (query the size first)");
    std::vector<int32_t> frp(rp), fci(b->n_full), prp(rp), pci(b->n_part), pti(b->n_part), lrp(rp), lci(b->n_load);
    std::vector<uint8_t> pool(static_cast<size_t>(b->n_pool) * b->tile_bytes);
    SF_TRY(sf_bsr_to_host(b, frp.data(), fci.data(), prp.data(), pci.data(), pti.data(), lrp.data(), lci.data(),
                          pool.data(), stream));
    std::vector<uint8_t> o;
    o.reserve(static_cast<size_t>(size));
    auto u32 = [&](uint32_t v) { for (int s = 0; s < 32; s += 8) o.push_back(static_cast<uint8_t>(v >> s)); };
    auto arr = [&](const std::vector<int32_t>& a) { u32(static_cast<uint32_t>(a.size())); for (auto x : a) u32(static_cast<uint32_t>(x)); };
    o.insert(o.end(), {'S', 'F', 'B', 'R'});
    u32(1);
    u32(static_cast<uint32_t>(b->seq_len));
    u32(static_cast<uint32_t>(b->block_m));
    u32(static_cast<uint32_t>(b->block_n));
    arr(frp); arr(fci); arr(prp); arr(pci); arr(pti); arr(lrp); arr(lci);
    u32(static_cast<uint32_t>(b->n_pool));
    o.insert(o.end(), pool.begin(), pool.end());
    std::memcpy(buf, o.data(), o.size());
    return SF_OK;
}

extern "C" sf_status sf_rowwise_build(const uint32_t* d_bits, int32_t seq_len, sf_csr_dev* out, void* stream) {
    if (!out) return fail(SF_INVALID_PARAMETER, "null output");
    *out = sf_csr_dev{};
    if (seq_len < 1) return fail(SF_INVALID_PARAMETER, "seq_len must be positive");
    cudaStream_t st = as_stream(stream);
    const int32_t words = sf_mask_words(seq_len);
    int32_t* cnt = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&cnt), (seq_len + 1) * 4ll + 256, st));
    int32_t* total = cnt + seq_len;
    char* blk = nullptr;
    row_popc_kernel<<<blocks_for(static_cast<int64_t>(seq_len) * 32), 256, 0, st>>>(d_bits, seq_len, words, cnt);
    SF_LAUNCH_CHECK();
    int32_t* rp_tmp = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&rp_tmp), (seq_len + 1) * 4ll, st));
    SF_TRY(scan_exclusive(cnt, rp_tmp, seq_len, total, st));
    int32_t nnz = 0;
    SF_CUDA_TRY(cudaMemcpyAsync(&nnz, total, 4, cudaMemcpyDeviceToHost, st));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    const int64_t rp_bytes = ceil_div((seq_len + 1) * 4ll, 256) * 256;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&blk), rp_bytes + imax64(4, nnz * 4ll), st));
    out->row_ptr = reinterpret_cast<int32_t*>(blk);
    out->col_idx = reinterpret_cast<int32_t*>(blk + rp_bytes);
    SF_CUDA_TRY(cudaMemcpyAsync(out->row_ptr, rp_tmp, (seq_len + 1) * 4ll, cudaMemcpyDeviceToDevice, st));
    row_compact_kernel<<<blocks_for(static_cast<int64_t>(seq_len) * 32), 256, 0, st>>>(d_bits, seq_len, words,
                                                                                       out->row_ptr, out->col_idx);
    SF_LAUNCH_CHECK();
    SF_CUDA_TRY(cudaFreeAsync(rp_tmp, st));
    SF_CUDA_TRY(cudaFreeAsync(cnt, st));
    out->seq_len = seq_len;
    out->nnz = nnz;
    out->_alloc = blk;
    return SF_OK;
}

extern "C" sf_status sf_csr_free(sf_csr_dev* csr, void* stream) {
    if (!csr) return SF_OK;
    if (csr->_alloc) SF_CUDA_TRY(cudaFreeAsync(csr->_alloc, as_stream(stream)));
    *csr = sf_csr_dev{};
    return SF_OK;
}

extern "C" sf_status sf_csr_to_host(const sf_csr_dev* csr, int32_t* row_ptr, int32_t* col_idx, void* stream) {
    cudaStream_t st = as_stream(stream);
    if (row_ptr)
        SF_CUDA_TRY(cudaMemcpyAsync(row_ptr, csr->row_ptr, (csr->seq_len + 1) * 4ll, cudaMemcpyDeviceToHost, st));
    if (col_idx && csr->nnz > 0)
        SF_CUDA_TRY(cudaMemcpyAsync(col_idx, csr->col_idx, csr->nnz * 4ll, cudaMemcpyDeviceToHost, st));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    return SF_OK;
}

static const char* validate_message(unsigned long long key) {
    const uint32_t code = static_cast<uint32_t>(key & 0xff);
    static const char* csr_msg[5] = {"bad row_ptr shape", "decreasing row_ptr", "col out of range",
                                     "cols not strictly increasing", "col length mismatch"};
    static const char* what[3] = {"full: ", "part: ", "load: "};
    static thread_local std::string m;
    if (code < 15) {
        m = std::string(what[code / 5]) + csr_msg[code % 5];
        return m.c_str();
    }
    switch (code) {
        case kVIdRange: return "part tile id out of pool range";
        case kVPoolMixed: return "pool tile is not mixed";
        case kVLoadSum: return "load_row_ptr is not the sum of full and part";
        case kVOverlap: return "full and part columns overlap";
        default: return "load columns are not the union of full and part";
    }
}

extern "C" sf_status sf_bsr_validate(const sf_bsr_dev* b, void* stream) {
    if (!b || !b->full_row_ptr || !b->part_row_ptr || !b->load_row_ptr)
        return fail(SF_INVALID_PARAMETER, "null BSR");
    if (b->n_rows < 0 || b->n_cols < 0 || b->block_m < 1 || b->block_n < 1)
        return fail(SF_INTERNAL_INCONSISTENCY, "full: bad row_ptr shape");
    cudaStream_t st = as_stream(stream);
    unsigned long long* err = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&err), 8, st));
    SF_CUDA_TRY(cudaMemsetAsync(err, 0xff, 8, st));
    const VCsr f{b->full_row_ptr, b->full_col_idx, b->n_full}, pa{b->part_row_ptr, b->part_col_idx, b->n_part},
        lo{b->load_row_ptr, b->load_col_idx, b->n_load};
    validate_csr_kernel<<<blocks_for(3ll * (b->n_rows + 1)), 256, 0, st>>>(f, pa, lo, b->n_rows, b->n_cols, err);
    SF_LAUNCH_CHECK();
    unsigned long long h = ~0ull;
    SF_CUDA_TRY(cudaMemcpyAsync(&h, err, 8, cudaMemcpyDeviceToHost, st));
    SF_CUDA_TRY(cudaStreamSynchronize(st));
    if (h == ~0ull) {
        const int64_t span = imax64(imax64(b->n_part, b->n_pool), b->n_rows);
        validate_rest_kernel<<<blocks_for(span), 256, 0, st>>>(
            f, pa, lo, b->part_tile_ids, b->n_pool, b->pool, b->tile_bytes,
            static_cast<int64_t>(b->block_m) * b->block_n, b->n_rows, err);
        SF_LAUNCH_CHECK();
        SF_CUDA_TRY(cudaMemcpyAsync(&h, err, 8, cudaMemcpyDeviceToHost, st));
        SF_CUDA_TRY(cudaStreamSynchronize(st));
    }
    SF_CUDA_TRY(cudaFreeAsync(err, st));
    if (h != ~0ull) return fail(SF_INTERNAL_INCONSISTENCY, validate_message(h));
    return SF_OK;
}

extern "C" sf_status sf_bsr_to_dense(const sf_bsr_dev* b, uint32_t* d_bits, void* stream) {
    SF_TRY(sf_bsr_validate(b, stream));  // to_dense validates first (bsr.hpp:156)
    if (!d_bits) return fail(SF_INVALID_PARAMETER, "null output mask");
    cudaStream_t st = as_stream(stream);
    const Geo g{b->seq_len, sf_mask_words(b->seq_len), b->block_m, b->block_n, b->n_rows, b->n_cols};
    SF_CUDA_TRY(cudaMemsetAsync(d_bits, 0, static_cast<size_t>(b->seq_len) * g.words * 4, st));
    const int64_t work = (static_cast<int64_t>(b->n_full) + b->n_part) * b->block_m;
    if (work > 0) {
        to_dense_kernel<<<blocks_for(work), 256, 0, st>>>(b->full_row_ptr, b->full_col_idx, b->n_full, b->part_row_ptr,
                                                           b->part_col_idx, b->part_tile_ids, b->n_part, b->pool,
                                                           b->tile_bytes, g, d_bits);
        SF_LAUNCH_CHECK();
    }
    return SF_OK;
}

// Device copy of host BSR arrays (a deserialised or hand-built BsrMask). load_tile is derived on
// the host from the full / part lists (-1 where a load column is not a part column).
extern "C" sf_status sf_bsr_from_host(int32_t seq_len, int32_t block_m, int32_t block_n, int32_t n_full, int32_t n_part,
                                      int32_t n_load, int32_t n_pool, const int32_t* full_row_ptr,
                                      const int32_t* full_col_idx, const int32_t* part_row_ptr,
                                      const int32_t* part_col_idx, const int32_t* part_tile_ids,
                                      const int32_t* load_row_ptr, const int32_t* load_col_idx, const uint8_t* pool,
                                      sf_bsr_dev* out, void* stream) {
    if (!out) return fail(SF_INVALID_PARAMETER, "null output");
    *out = sf_bsr_dev{};
    if (seq_len < 1 || block_m < 1 || block_n < 1) return fail(SF_INVALID_PARAMETER, "bad BSR geometry");
    if (n_full < 0 || n_part < 0 || n_load < 0 || n_pool < 0) return fail(SF_INVALID_PARAMETER, "negative BSR counts");
    cudaStream_t st = as_stream(stream);
    const int32_t n_rows = static_cast<int32_t>(ceil_div(seq_len, block_m));
    const int32_t tile_bytes = static_cast<int32_t>(ceil_div(static_cast<int64_t>(block_m) * block_n, 8));
    const int64_t rp = n_rows + 1;
    std::vector<int32_t> load_tile(static_cast<size_t>(std::max(1, n_load)), -1);
    for (int64_t r = 0; r < n_rows; ++r) {  // map each load column to its part pool id, if any
        const int32_t p0 = part_row_ptr[r], p1 = part_row_ptr[r + 1];
        for (int32_t k = load_row_ptr[r]; k < load_row_ptr[r + 1] && k < n_load; ++k)
            for (int32_t q = std::max(0, p0); q < p1 && q < n_part; ++q)
                if (part_col_idx[q] == load_col_idx[k]) load_tile[static_cast<size_t>(k)] = part_tile_ids[q];
    }
    const int64_t out_bytes = 3 * ceil_div(rp * 4, 256) * 256 + ceil_div(std::max(1, n_full) * 4ll, 256) * 256 +
                              2 * ceil_div(std::max(1, n_part) * 4ll, 256) * 256 +
                              2 * ceil_div(std::max(1, n_load) * 4ll, 256) * 256 +
                              ceil_div(imax64(1, static_cast<int64_t>(n_pool) * tile_bytes), 256) * 256;
    char* ob = nullptr;
    SF_CUDA_TRY(pool_malloc(reinterpret_cast<void**>(&ob), out_bytes, st));
    char* p = ob;
    out->full_row_ptr = carve<int32_t>(p, rp);
    out->part_row_ptr = carve<int32_t>(p, rp);
    out->load_row_ptr = carve<int32_t>(p, rp);
    out->full_col_idx = carve<int32_t>(p, std::max(1, n_full));
    out->part_col_idx = carve<int32_t>(p, std::max(1, n_part));
    out->part_tile_ids = carve<int32_t>(p, std::max(1, n_part));
    out->load_col_idx = carve<int32_t>(p, std::max(1, n_load));
    out->load_tile = carve<int32_t>(p, std::max(1, n_load));
    out->pool = carve<uint8_t>(p, imax64(1, static_cast<int64_t>(n_pool) * tile_bytes));
    out->_alloc = ob;
    auto up = [&](void* dst, const void* src, int64_t bytes) -> sf_status {
        if (bytes > 0 && src) SF_CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
        return SF_OK;
    };
    SF_TRY(up(out->full_row_ptr, full_row_ptr, rp * 4));
    SF_TRY(up(out->part_row_ptr, part_row_ptr, rp * 4));
    SF_TRY(up(out->load_row_ptr, load_row_ptr, rp * 4));
    SF_TRY(up(out->full_col_idx, full_col_idx, n_full * 4ll));
    SF_TRY(up(out->part_col_idx, part_col_idx, n_part * 4ll));
    SF_TRY(up(out->part_tile_ids, part_tile_ids, n_part * 4ll));
    SF_TRY(up(out->load_col_idx, load_col_idx, n_load * 4ll));
    SF_TRY(up(out->load_tile, load_tile.data(), n_load * 4ll));
    SF_TRY(up(out->pool, pool, static_cast<int64_t>(n_pool) * tile_bytes));
    SF_CUDA_TRY(cudaStreamSynchronize(st));  // the host staging vector dies here
    out->seq_len = seq_len;
    out->block_m = block_m;
    out->block_n = block_n;
    out->n_rows = n_rows;
    out->n_cols = static_cast<int32_t>(ceil_div(seq_len, block_n));
    out->n_full = n_full;
    out->n_part = n_part;
    out->n_load = n_load;
    out->n_pool = n_pool;
    out->tile_bytes = tile_bytes;
    return SF_OK;
}
