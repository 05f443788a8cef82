// capi.cu — host side of the C ABI: error state, launch accounting, the analytical selector
// (planner.hpp:20-161, exact doubles, host C++), attention dispatch and the CUDA-event timing
// hook behind the MeasurementBackend contract (backend.hpp:391-402, 488-500).
#include <cstdlib>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "common.cuh"

namespace sf {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};
static std::atomic<int32_t> g_attn_impl{0};

void set_error(const std::string& msg) { g_last_error = msg; }
sf_status fail(sf_status st, const std::string& msg) {
    g_last_error = msg;
    return st;
}
void note_launch(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

sf_status check_attn_args(const sf_attn_args& a);
sf_status attn_generic(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st);
// attn_tc.cu: returns SF_PLAN_ERROR (without launching) when the shape is not supported.
sf_status attn_tc(const sf_attn_args& a, const sf_bsr_dev& b, cudaStream_t st, bool probe_only, float* lse = nullptr);

namespace {

// B200 executor cost model, fitted to `bench.py --sweep --both` and `--band-sweep`
// (profiles/r01/sweep_mha_both_v2.jsonl, band_sweep_v1.jsonl): the persistent tcgen05 block
// executor has a ~12 us floor (cfg1: 12.3 us measured, profiles/r01/bench_cfg1_v8.json) and retires ~1.8e12 executed cells/s (cells of the loaded 128x16
// tiles); the row-wise gather has a ~10 us floor, a per-row cost (0.2 ns with one 8-lane group
// per row when rows average <= 32 keys, 0.65 ns with a warp per row) and ~6e10 valid cells/s.
constexpr double kBlockCellsPerUs = 1.8e6;
constexpr double kBlockFloorUs = 12.0;
constexpr double kWideTileCellRatio = 1.05;  // block_n 64 / 32 when their cells are <= 1.05x block_n 16's
constexpr double kPairCellRatio = 0.80;  // block_m 64 when its executed cells < 0.80x block_m 128's
constexpr double kRowNnzPerUs = 6.0e4;
constexpr double kRowFloorUs = 10.0;

double threshold_from_loads(int32_t n, int64_t loads16, double tau) {
    // planner.hpp:67-76: L / N^2 - tau / (log2 N)^2 with N = ceil(n/16)
    const double big_n = static_cast<double>((n + 15) / 16);
    const double log_n = std::log2(big_n);
    return static_cast<double>(loads16) / (big_n * big_n) - tau / (log_n * log_n);
}

int64_t req_smem(int bm, int bn, int head, int padding = 16) {  // planner.hpp:80-85
    return static_cast<int64_t>(2 * bm + bn) * (head + padding) + static_cast<int64_t>(bm) * (bn + padding);
}

double occupancy(int warps, int64_t req, const sf_hw_spec& hw) {  // planner.hpp:90-100
    const int64_t bytes = req * hw.element_bytes;
    const int64_t by_smem = bytes > hw.smem_size ? 0 : hw.smem_size / bytes;
    const int64_t by_warp = hw.max_warp / warps;
    return static_cast<double>(warps) * static_cast<double>(std::min(by_smem, by_warp)) /
           static_cast<double>(hw.max_warp);
}

double plan_score(int bm, int bn, int w, const sf_hw_spec& hw, int64_t seq, int h, int64_t bs, int head) {
    // planner.hpp:104-113
    const double occ = occupancy(w, req_smem(bm, bn, head), hw);
    if (occ == 0.0) return 0.0;
    const double gran = std::sqrt(static_cast<double>(hw.sm_num) / (static_cast<double>(bm) * bn));
    const double work = static_cast<double>(seq) * h * static_cast<double>(bs) / static_cast<double>(bm);
    return occ * gran * work;
}

}  // namespace
}  // namespace sf

using namespace sf;

extern "C" const char* sf_last_error(void) { return g_last_error.c_str(); }
namespace sf {
static std::atomic<int> g_pdl{-1};
bool pdl_enabled() {
    int v = g_pdl.load();
    if (v < 0) {
        const char* e = std::getenv("SF_PDL");
        v = (e && e[0] == '0') ? 0 : 1;
        g_pdl.store(v);
    }
    return v != 0;
}
}  // namespace sf

namespace sf {
cudaError_t pool_malloc(void** p, size_t bytes, cudaStream_t st) {
    static std::atomic<int> ready{0};
    if (!ready.load()) {
        int dev = 0;
        cudaMemPool_t pool;
        if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        ready.store(1);
    }
    return cudaMallocAsync(p, bytes, st);
}
}  // namespace sf

extern "C" sf_status sf_set_pdl(int32_t on) {
    sf::g_pdl.store(on ? 1 : 0);
    return SF_OK;
}

extern "C" const char* sf_version(void) { return "sparsefuse-b200 0.1 sm_100a"; }
extern "C" int64_t sf_launch_count(void) { return g_launches.load(); }

extern "C" sf_status sf_set_attn_impl(int32_t impl) {
    if (impl < 0 || impl > 2) return fail(SF_INVALID_PARAMETER, "impl must be 0, 1 or 2");
    g_attn_impl.store(impl);
    return SF_OK;
}
extern "C" int32_t sf_get_attn_impl(void) { return g_attn_impl.load(); }

extern "C" sf_status sf_hw_preset(const char* name, sf_hw_spec* out) {
    // planner.hpp:36-40 presets, plus the B200 this library targets.
    if (!name || !out) return fail(SF_INVALID_PARAMETER, "null argument");
    auto set = [&](const char* nm, int sm, int64_t smem, int warps) {
        std::memset(out, 0, sizeof(*out));
        std::strncpy(out->name, nm, sizeof(out->name) - 1);
        out->sm_num = sm;
        out->smem_size = smem;
        out->max_warp = warps;
        out->element_bytes = 2;
        return SF_OK;
    };
    if (!std::strcmp(name, "rtx4090")) return set("rtx4090", 128, 128 * 1024, 48);
    if (!std::strcmp(name, "a100")) return set("a100", 108, 192 * 1024, 64);
    if (!std::strcmp(name, "b200")) return set("b200", 148, 228 * 1024, 64);
    return fail(SF_INVALID_PARAMETER, std::string("unknown hardware preset: ") + name);
}

extern "C" double sf_threshold_from_loads(int32_t seq_len, int64_t loads16, double tau) {
    return threshold_from_loads(seq_len, loads16, tau);
}

static sf_status loads16_of(const uint32_t* d_bits, int32_t n, int64_t* loads, void* stream) {
    sf_bsr_dev b{};
    SF_TRY(sf_bsr_build(d_bits, n, 16, 16, &b, stream));
    *loads = b.n_load;
    return sf_bsr_free(&b, stream);
}

extern "C" sf_status sf_threshold(const uint32_t* d_bits, int32_t seq_len, double tau, double* out,
                                  void* stream) {
    if (seq_len <= 16)
        return fail(SF_DEGENERATE_INPUT, "threshold undefined for seq_len <= 16 (log2(1) = 0)");  // planner.hpp:69
    int64_t loads = 0;
    SF_TRY(loads16_of(d_bits, seq_len, &loads, stream));
    *out = threshold_from_loads(seq_len, loads, tau);
    return SF_OK;
}

extern "C" sf_status sf_select_plan_from_loads(int64_t loads16, const sf_hw_spec* hw, int64_t seq_len, int32_t h,
                                               int64_t bs, int32_t head_size, int32_t mode, sf_plan* out) {
    // planner.hpp:130-161 (strict '>' scan over bm, bn, warps ascending: first maximum wins)
    if (!hw || !out) return fail(SF_INVALID_PARAMETER, "null argument");
    if (hw->sm_num <= 0 || hw->smem_size <= 0 || hw->max_warp <= 0 || hw->element_bytes <= 0)
        return fail(SF_INVALID_PARAMETER, "hardware spec fields must be positive");
    if (h <= 0 || bs <= 0 || head_size <= 0) return fail(SF_INVALID_PARAMETER, "hyperparameters must be positive");
    std::memset(out, 0, sizeof(*out));
    out->kind = SF_ROW_WISE;
    out->threshold = std::nan("");
    if (seq_len <= 16) return SF_OK;
    out->threshold = threshold_from_loads(static_cast<int32_t>(seq_len), loads16, 1.2);
    if (out->threshold < 0.0) return SF_OK;
    static const int sizes[4] = {16, 32, 64, 128};
    static const int warps[4] = {1, 2, 4, 8};
    double best = -1.0;
    for (int bm : sizes)
        for (int bn : sizes)
            for (int w : warps) {
                // B200 mode: Eq. 2 over the tiles the tcgen05 kernel executes (M = 128 MMA
                // rows, head_size 64); the reference grid otherwise.
                if (mode == SF_PLAN_B200 && !(bm == 128 && head_size == 64)) continue;
                const double s = plan_score(bm, bn, w, *hw, seq_len, h, bs, head_size);
                if (s > 0.0 && s > best) {
                    best = s;
                    out->kind = SF_BLOCK_WISE;
                    out->block_m = bm;
                    out->block_n = bn;
                    out->num_warps = w;
                    out->score = s;
                }
            }
    if (out->kind != SF_BLOCK_WISE) out->fallback = 1;
    return SF_OK;
}

extern "C" sf_status sf_select_plan(const uint32_t* d_bits, const sf_hw_spec* hw, int64_t seq_len, int32_t h,
                                    int64_t bs, int32_t head_size, int32_t mode, sf_plan* out, void* stream) {
    if (!hw || !out) return fail(SF_INVALID_PARAMETER, "null argument");
    if (hw->sm_num <= 0 || hw->smem_size <= 0 || hw->max_warp <= 0 || hw->element_bytes <= 0)
        return fail(SF_INVALID_PARAMETER, "hardware spec fields must be positive");
    if (h <= 0 || bs <= 0 || head_size <= 0) return fail(SF_INVALID_PARAMETER, "hyperparameters must be positive");
    int64_t loads = 0;
    if (seq_len > 16) SF_TRY(loads16_of(d_bits, static_cast<int32_t>(seq_len), &loads, stream));
    SF_TRY(sf_select_plan_from_loads(loads, hw, seq_len, h, bs, head_size, mode, out));
    if (mode == SF_PLAN_B200 && seq_len > 16 && head_size == 64) {
        // B200 calibration of the Eq. 1 decision: both executors are priced with the
        // fitted cost model above and the faster one is kept, whichever way Eq. 1 routed. Eq. 1
        // assumes a row-wise executor that is competitive per valid cell; on B200 the tcgen05
        // block executor runs ~30x more cells per second than the CUDA-core row-wise gather, so
        // most of Eq. 1's row-wise verdicts (narrow bands) flip to block-wise, while unstructured
        // low-density masks (every (128,16) tile loaded, nearly empty) flip the other way.
        const int bn = out->kind == SF_BLOCK_WISE ? out->block_n : 16;
        sf_bsr_dev b{};
        SF_TRY(sf_bsr_build(d_bits, static_cast<int32_t>(seq_len), 128, bn, &b, stream));
        const int64_t n_load = b.n_load;
        SF_TRY(sf_bsr_free(&b, stream));
        int64_t nnz = 0;
        SF_TRY(sf_mask_count(d_bits, static_cast<int32_t>(seq_len), &nnz, stream));
        const double slices = static_cast<double>(bs) * h;
        const double rows = slices * static_cast<double>(seq_len);
        const double per_row_us = nnz <= 32 * seq_len ? 0.0002 : 0.00065;
        const double t_bw = kBlockFloorUs + static_cast<double>(n_load) * 128.0 * bn * slices / kBlockCellsPerUs;
        const double t_rw = kRowFloorUs + rows * per_row_us + static_cast<double>(nnz) * slices / kRowNnzPerUs;
        if (out->kind == SF_ROW_WISE && t_bw < t_rw) {
            out->kind = SF_BLOCK_WISE;
            out->block_m = 128;
            out->block_n = 16;
            out->num_warps = 8;
            out->score = plan_score(128, 16, 8, *hw, seq_len, h, bs, head_size);
            out->fallback = 0;
        } else if (out->kind == SF_BLOCK_WISE && t_rw < t_bw) {
            out->kind = SF_ROW_WISE;
            out->block_m = out->block_n = out->num_warps = 0;
            out->score = 0.0;
            out->fallback = 0;
        }
        // block_m 64 (the tcgen05 kernel's head-pair mode: M = 64 tiles of two heads per work item,
        // one 5-D TMA box per column block for both heads) retires executed cells at 0.7-0.9x the
        // rate of block_m 128, so it wins only where 64-row blocks execute clearly fewer cells:
        // BigBird-like random blocks (cfg2: 0.67x the cells, 0.83x the time), narrow bands,
        // longformer; never causal or wide bands (0.75-0.98x the cells, 1.04-1.08x the time)
        // (tools/bm_sweep.py, profiles/r02/bm_sweep.txt). SF_PLAN_PAIR=0 keeps block_m 128.
        const char* pe = std::getenv("SF_PLAN_PAIR");
        // (the tcgen05 kernel holds <= 128 row blocks: head pairs up to n = 8192)
        if (out->kind == SF_BLOCK_WISE && out->block_m == 128 && seq_len <= 64 * 128 && !(pe && *pe == '0')) {
            sf_bsr_dev b64{};
            SF_TRY(sf_bsr_build(d_bits, static_cast<int32_t>(seq_len), 64, out->block_n, &b64, stream));
            const int64_t n_load64 = b64.n_load;
            SF_TRY(sf_bsr_free(&b64, stream));
            if (static_cast<double>(n_load64) * 64.0 < kPairCellRatio * static_cast<double>(n_load) * 128.0) {
                out->block_m = 64;
                out->score = plan_score(64, out->block_n, out->num_warps, *hw, seq_len, h, bs, head_size);
            }
        }
        // block_n last: the widest of 64 / 32 whose tiles execute at most 5% more cells than the
        // plan's. A step gathers 64 keys in 64 / block_n boxes per tensor, so wider tiles cut the
        // TMA boxes and the bit-row fills per step (T5 cfg4 at (64, 64): 91.7 vs 100.7 us with the
        // same cells; cfg2's BigBird keeps 16: 1.36x the cells at 32; tools/tile_test.py).
        const char* be = std::getenv("SF_PLAN_BN");
        if (out->kind == SF_BLOCK_WISE && out->block_n == 16 && !(be && *be == '0')) {
            sf_bsr_dev b0{};
            SF_TRY(sf_bsr_build(d_bits, static_cast<int32_t>(seq_len), out->block_m, 16, &b0, stream));
            const double cells16 = static_cast<double>(b0.n_load) * 16.0;
            SF_TRY(sf_bsr_free(&b0, stream));
            for (int bn : {64, 32}) {
                sf_bsr_dev bw{};
                SF_TRY(sf_bsr_build(d_bits, static_cast<int32_t>(seq_len), out->block_m, bn, &bw, stream));
                const double cells = static_cast<double>(bw.n_load) * bn;
                SF_TRY(sf_bsr_free(&bw, stream));
                if (cells <= kWideTileCellRatio * cells16) {
                    out->block_n = bn;
                    out->score = plan_score(out->block_m, bn, out->num_warps, *hw, seq_len, h, bs, head_size);
                    break;
                }
            }
        }
    }
    return SF_OK;
}

extern "C" sf_status sf_mha_blockwise(const sf_attn_args* args, const sf_bsr_dev* bsr, const sf_plan* plan,
                                      sf_attn_stats* stats, void* stream) {
    if (!args || !bsr) return fail(SF_INVALID_PARAMETER, "null argument");
    SF_TRY(check_attn_args(*args));
    if (bsr->seq_len != args->seq_len) return fail(SF_SHAPE_ERROR, "bsr seq_len differs from input");  // attention.hpp:74
    if (plan) {  // planner.hpp:165-172
        if (plan->kind != SF_BLOCK_WISE) return fail(SF_PLAN_ERROR, "plan does not select the block-wise kernel");
        if (plan->block_m != bsr->block_m || plan->block_n != bsr->block_n)
            return fail(SF_PLAN_ERROR, "BSR block sizes do not match the active plan");
    }
    sf_attn_args a = *args;
    if (a.scale == 0.f) a.scale = 1.0f / std::sqrt(static_cast<float>(a.head_size));
    if (stats) {  // BlockExecStats of one (b,h) slice: the load set is mask-level (attention.hpp:58-59)
        stats->tiles_loaded = bsr->n_load;
        stats->full_tiles = bsr->n_full;
        stats->part_tiles = bsr->n_part;
    }
    if (bsr->n_load == 0 || a.seq_len == 0) {
        // every row fully masked: output is exactly zero (attention.hpp:160-166)
        cudaStream_t st = as_stream(stream);
        const size_t el = 2;
        if (a.o_sn == a.head_size && a.o_sh == static_cast<int64_t>(a.seq_len) * a.head_size &&
            a.o_sb == static_cast<int64_t>(a.h) * a.o_sh) {
            SF_CUDA_TRY(cudaMemsetAsync(a.o, 0, static_cast<size_t>(a.bs) * a.o_sb * el, st));
        } else {
            for (int b = 0; b < a.bs; ++b)
                for (int hh = 0; hh < a.h; ++hh)
                    SF_CUDA_TRY(cudaMemset2DAsync(static_cast<char*>(a.o) + (b * a.o_sb + hh * a.o_sh) * el,
                                                  a.o_sn * el, 0, a.head_size * el, a.seq_len, st));
        }
        return SF_OK;
    }
    const int impl = g_attn_impl.load();
    cudaStream_t st = as_stream(stream);
    if (impl != 1) {
        sf_status s = attn_tc(a, *bsr, st, /*probe_only=*/false);
        if (s == SF_OK || impl == 2 || s != SF_PLAN_ERROR) return s;
    }
    return attn_generic(a, *bsr, st);
}

extern "C" sf_status sf_time_best(sf_launch_fn fn, void* user, int32_t warmup, int32_t reps, float* best_ms,
                                  void* stream) {
    if (!fn || !best_ms || reps < 1) return fail(SF_INVALID_PARAMETER, "bad timing arguments");
    cudaStream_t st = as_stream(stream);
    for (int i = 0; i < warmup; ++i) SF_TRY(fn(user, stream));
    struct Events {  // destroyed on every return path, error returns included
        cudaEvent_t e[2] = {nullptr, nullptr};
        ~Events() {
            for (cudaEvent_t x : e)
                if (x) cudaEventDestroy(x);
        }
    } ev;
    SF_CUDA_TRY(cudaEventCreate(&ev.e[0]));
    SF_CUDA_TRY(cudaEventCreate(&ev.e[1]));
    cudaEvent_t e0 = ev.e[0], e1 = ev.e[1];
    float best = INFINITY;
    for (int i = 0; i < reps; ++i) {
        SF_CUDA_TRY(cudaEventRecord(e0, st));
        SF_TRY(fn(user, stream));
        SF_CUDA_TRY(cudaEventRecord(e1, st));
        SF_CUDA_TRY(cudaEventSynchronize(e1));
        float ms = 0.f;
        SF_CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    *best_ms = best;
    return SF_OK;
}
