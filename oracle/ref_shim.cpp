// ref_shim.cpp — extern "C" entry points over the UNMODIFIED reference headers
// (/root/reference/proj/include/sparsefuse/*.hpp), compiled in place by oracle/Makefile into
// oracle/_ref/libsfref.so. TEST INFRASTRUCTURE ONLY: used to pin the C restatement
// (oracle/sf_oracle.c), to generate tests/golden/ fixtures, and as bench.py's CPU baseline
// ("kind": "reference"). Nothing here is on the product path. No reference source is copied:
// this file only #includes the headers where they lie.
#include <sparsefuse/attention.hpp>
#include <sparsefuse/backend.hpp>
#include <sparsefuse/bsr.hpp>
#include <sparsefuse/io.hpp>
#include <sparsefuse/mask.hpp>
#include <sparsefuse/planner.hpp>
#include <sparsefuse/search.hpp>

#include <barrier>
#include <chrono>
#include <cstring>
#include <sstream>
#include <thread>
#include <vector>

#include "../include/sf_capi.h"

using namespace sparsefuse;

namespace {

template <typename F>
int guard(F&& f) {
    try {
        f();
        return SF_OK;
    } catch (const invalid_parameter&) { return SF_INVALID_PARAMETER; }
    catch (const shape_error&) { return SF_SHAPE_ERROR; }
    catch (const plan_error&) { return SF_PLAN_ERROR; }
    catch (const degenerate_input&) { return SF_DEGENERATE_INPUT; }
    catch (const illegal_segment&) { return SF_ILLEGAL_SEGMENT; }
    catch (const internal_inconsistency&) { return SF_INTERNAL_INCONSISTENCY; }
    catch (const backend_error&) { return SF_BACKEND_ERROR; }
    catch (const io_error&) { return SF_IO_ERROR; }
    catch (...) { return SF_BACKEND_ERROR; }
}

DenseMask from_u8(const uint8_t* m, int n) {
    DenseMask d(n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j)
            if (m[static_cast<size_t>(i) * n + j]) d.set(i, j, true);
    return d;
}

const char* pattern_name(int p) {
    switch (p) {
        case SF_PATTERN_SLIDING: return "sliding";
        case SF_PATTERN_DILATED: return "dilated";
        case SF_PATTERN_GLOBAL: return "global";
        case SF_PATTERN_RANDOM: return "random";
        case SF_PATTERN_LONGFORMER: return "longformer";
        case SF_PATTERN_BIGBIRD: return "bigbird";
        default: return "unsupported";
    }
}

}  // namespace

extern "C" {

// generate_mask over MaskDescriptor (io.hpp:192) for each term, then compose (mask.hpp:146).
// Causal-family terms have no reference generator; they are rejected (SF_INVALID_PARAMETER).
int ref_mask_generate(const sf_mask_desc* terms, int n_terms, uint8_t* out) {
    return guard([&] {
        std::vector<DenseMask> ms;
        for (int t = 0; t < n_terms; ++t) {
            MaskDescriptor d;
            d.pattern = pattern_name(terms[t].pattern);
            d.seq_len = terms[t].seq_len;
            d.params.band_width = terms[t].band_width;
            d.params.global_width = terms[t].global_width;
            d.params.dilation_rate = terms[t].dilation_rate;
            d.params.filling_rate = terms[t].filling_rate;
            d.params.block = terms[t].block;
            d.params.seed = terms[t].seed;
            ms.push_back(generate_mask(d));
        }
        const DenseMask m = ms.size() == 1 ? ms[0] : compose(std::span<const DenseMask>(ms));
        std::memcpy(out, m.raw().data(), m.raw().size());
    });
}

// build_bsr (bsr.hpp:47) + write_bsr (io.hpp:103). Returns bytes via *nbytes; writes if buf.
int ref_build_bsr_sfbr(const uint8_t* mask, int n, int bm, int bn, uint8_t* buf, int64_t cap,
                       int64_t* nbytes, int64_t* counts4) {
    return guard([&] {
        const BsrMask b = build_bsr(from_u8(mask, n), bm, bn);
        std::ostringstream os;
        write_bsr(os, b);
        const std::string s = os.str();
        *nbytes = static_cast<int64_t>(s.size());
        if (buf) std::memcpy(buf, s.data(), std::min<size_t>(s.size(), static_cast<size_t>(cap)));
        if (counts4) {
            const auto st = block_stats(b);
            counts4[0] = st.full_count;
            counts4[1] = st.part_count;
            counts4[2] = st.empty_count;
            counts4[3] = static_cast<int64_t>(b.part_mask_pool.size());
        }
    });
}

// write_dense_mask (io.hpp:66-76) of a uint8 mask: the reference's SFMK bytes.
int ref_mask_sfmk(const uint8_t* mask, int n, uint8_t* buf, int64_t cap, int64_t* nbytes) {
    return guard([&] {
        std::ostringstream os;
        write_dense_mask(os, from_u8(mask, n));
        const std::string s = os.str();
        *nbytes = static_cast<int64_t>(s.size());
        if (buf) std::memcpy(buf, s.data(), std::min<size_t>(s.size(), static_cast<size_t>(cap)));
    });
}

// build_rowwise (bsr.hpp:198).
int ref_build_rowwise(const uint8_t* mask, int n, int32_t* row_ptr, int32_t* col_idx, int64_t cap,
                      int64_t* nnz) {
    return guard([&] {
        const RowwiseMask r = build_rowwise(from_u8(mask, n));
        *nnz = static_cast<int64_t>(r.col_idx.size());
        std::memcpy(row_ptr, r.row_ptr.data(), r.row_ptr.size() * 4);
        if (col_idx)
            std::memcpy(col_idx, r.col_idx.data(),
                        std::min<size_t>(r.col_idx.size(), static_cast<size_t>(cap)) * 4);
    });
}

// block_sparse_sdpa (attention.hpp:71) on a BSR built at (bm, bn). (b,h) slices are
// independent; n_threads > 1 runs them on std::threads, each slice calling the
// unmodified executor on a (1,1,n,d) input.
int ref_block_sparse_sdpa(const float* q, const float* k, const float* v, int bs, int h, int n,
                          int d, const uint8_t* mask, int bm, int bn, float* out, int64_t* stats3,
                          int n_threads) {
    return guard([&] {
        const BsrMask b = build_bsr(from_u8(mask, n), bm, bn);
        const int64_t slices = static_cast<int64_t>(bs) * h;
        const size_t sl = static_cast<size_t>(n) * d;
        std::vector<BlockExecStats> st(static_cast<size_t>(std::max(1, n_threads)));
        auto work = [&](int t, int64_t s0, int64_t s1) {
            for (int64_t s = s0; s < s1; ++s) {
                AttentionInput<float> in{Tensor4<float>(1, 1, n, d), Tensor4<float>(1, 1, n, d),
                                         Tensor4<float>(1, 1, n, d)};
                std::memcpy(in.q.v.data(), q + s * sl, sl * 4);
                std::memcpy(in.k.v.data(), k + s * sl, sl * 4);
                std::memcpy(in.v.v.data(), v + s * sl, sl * 4);
                BlockExecStats one;
                const auto o = block_sparse_sdpa(in, b, &one);
                if (s == 0) st[static_cast<size_t>(t)] = one;
                std::memcpy(out + s * sl, o.v.data(), sl * 4);
            }
        };
        if (n_threads <= 1) {
            work(0, 0, slices);
        } else {
            std::vector<std::thread> th;
            for (int t = 0; t < n_threads; ++t)
                th.emplace_back(work, t, slices * t / n_threads, slices * (t + 1) / n_threads);
            for (auto& x : th) x.join();
        }
        if (stats3) {
            stats3[0] = stats3[1] = stats3[2] = 0;
            for (const auto& x : st) {
                stats3[0] += x.tiles_loaded;
                stats3[1] += x.full_tiles;
                stats3[2] += x.part_tiles;
            }
        }
    });
}

int ref_rowwise_sdpa(const double* q, const double* k, const double* v, int bs, int h, int n, int d,
                     const uint8_t* mask, double* out) {
    return guard([&] {
        AttentionInput<double> in{Tensor4<double>(bs, h, n, d), Tensor4<double>(bs, h, n, d),
                                  Tensor4<double>(bs, h, n, d)};
        const size_t cnt = in.q.v.size();
        std::memcpy(in.q.v.data(), q, cnt * 8);
        std::memcpy(in.k.v.data(), k, cnt * 8);
        std::memcpy(in.v.v.data(), v, cnt * 8);
        const auto o = rowwise_sdpa(in, build_rowwise(from_u8(mask, n)));
        std::memcpy(out, o.v.data(), cnt * 8);
    });
}

int ref_dense_sdpa(const double* q, const double* k, const double* v, int bs, int h, int n, int d,
                   const uint8_t* mask, double* out) {
    return guard([&] {
        AttentionInput<double> in{Tensor4<double>(bs, h, n, d), Tensor4<double>(bs, h, n, d),
                                  Tensor4<double>(bs, h, n, d)};
        const size_t cnt = in.q.v.size();
        std::memcpy(in.q.v.data(), q, cnt * 8);
        std::memcpy(in.k.v.data(), k, cnt * 8);
        std::memcpy(in.v.v.data(), v, cnt * 8);
        const auto o = dense_sdpa_oracle(in, from_u8(mask, n));
        std::memcpy(out, o.v.data(), cnt * 8);
    });
}

void ref_random_attention_input(int bs, int h, int n, int d, uint64_t seed, float* q, float* k,
                                float* v) {
    const auto in = random_attention_input<float>(bs, h, n, d, seed);
    std::memcpy(q, in.q.v.data(), in.q.v.size() * 4);
    std::memcpy(k, in.k.v.data(), in.k.v.size() * 4);
    std::memcpy(v, in.v.v.data(), in.v.v.size() * 4);
}

int ref_threshold(const uint8_t* mask, int n, double tau, double* out) {
    return guard([&] { *out = threshold(from_u8(mask, n), tau); });
}

// select_plan (planner.hpp:130) with an explicit HardwareSpec.
int ref_select_plan(const uint8_t* mask, int n, const sf_hw_spec* hw, int64_t seq, int h, int64_t bs,
                    int head, sf_plan* out) {
    return guard([&] {
        HardwareSpec s{hw->name, hw->sm_num, hw->smem_size, hw->max_warp, hw->element_bytes};
        const KernelPlan p = select_plan(from_u8(mask, n), s, seq, h, bs, head);
        out->kind = p.kind == KernelKind::BlockWise ? SF_BLOCK_WISE : SF_ROW_WISE;
        out->block_m = p.block_m;
        out->block_n = p.block_n;
        out->num_warps = p.num_warps;
        out->score = p.score;
        out->threshold = p.threshold;
        out->fallback = p.fallback ? 1 : 0;
    });
}

int ref_hw_preset(const char* name, sf_hw_spec* out) {
    return guard([&] {
        const HardwareSpec s = hw_preset(name);
        std::memset(out, 0, sizeof(*out));
        std::strncpy(out->name, s.name.c_str(), sizeof(out->name) - 1);
        out->sm_num = s.sm_num;
        out->smem_size = s.smem_size;
        out->max_warp = s.max_warp;
        out->element_bytes = s.element_bytes;
    });
}

// One GraphData parameter tensor (backend.hpp:65-106) of a preset chain, for pinning the
// restatement of the seeded parameters. which: 0 input, 1 weight, 2 bias, 3 gamma, 4 beta, 5 aux.
int ref_graph_param(const char* model, int64_t bs, int64_t seq, int64_t hidden, int heads,
                    int head_size, uint64_t seed, int node, int which, float* out, int64_t cap,
                    int64_t* count) {
    return guard([&] {
        GraphHyper hy{bs, seq, hidden, heads, head_size, 0};
        const OpGraph g = build_preset_graph(model, hy);
        const GraphData gd = GraphData::make(g, seed);
        const std::vector<float>* src = nullptr;
        const NodeParams& p = gd.params.at(static_cast<size_t>(std::max(node, 0)));
        switch (which) {
            case 0: src = &gd.input.a; break;
            case 1: src = &p.weight.a; break;
            case 2: src = &p.bias; break;
            case 3: src = &p.gamma; break;
            case 4: src = &p.beta; break;
            default: src = &p.aux.a; break;
        }
        *count = static_cast<int64_t>(src->size());
        if (out) std::memcpy(out, src->data(), std::min<size_t>(src->size(), static_cast<size_t>(cap)) * 4);
    });
}

// CpuBackend-style chain run (backend.hpp:430-441) of a preset graph under the given scheme
// code (empty = unfused) with default settings, the MHA context built from `mask` at the
// given plan tile. Output rows*hidden floats. n_threads > 1 runs `n_threads` independent
// copies of the chain (one sequence each when bs == 1) for throughput timing; out receives
// copy 0. `seconds` (optional) receives the wall time of the run_chain calls alone: every thread
// first builds its CpuBackend (GraphData::make regenerates all weights, backend.hpp:408-410,456),
// then all start together at a barrier; the clock runs from the barrier to the last join.
int ref_run_chain(const char* model, int64_t bs, int64_t seq, int64_t hidden, int heads,
                  int head_size, uint64_t seed, const uint8_t* mask, int bm, int bn,
                  const char* code, float* out, int n_threads, double* seconds) {
    return guard([&] {
        GraphHyper hy{bs, seq, hidden, heads, head_size, 0};
        const OpGraph g = build_preset_graph(model, hy);
        const DenseMask dm = from_u8(mask, static_cast<int>(seq));
        KernelPlan plan;
        plan.kind = KernelKind::BlockWise;
        plan.block_m = bm;
        plan.block_n = bn;
        const MhaContext ctx = MhaContext::make(dm, plan);
        const FusionScheme scheme = (code && *code) ? make_scheme(decode(code)) : unfused_scheme(g.size());
        validate_scheme(scheme, g);
        const int nt = std::max(1, n_threads);
        std::barrier start(nt + 1);
        std::chrono::steady_clock::time_point t0;
        auto one = [&](float* dst) {
            CpuBackend be(g, seed, ctx);
            start.arrive_and_wait();
            const Matrix r = be.run_chain(g, scheme, {});
            if (dst) std::memcpy(dst, r.a.data(), r.a.size() * 4);
        };
        std::vector<std::thread> th;
        for (int t = 0; t < nt; ++t) th.emplace_back(one, t == 0 ? out : nullptr);
        start.arrive_and_wait();
        t0 = std::chrono::steady_clock::now();
        for (auto& x : th) x.join();
        if (seconds) *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

// A preset graph, or "spec:<nodes>" — a linear chain over rows = bs*seq starting at width
// `hidden`, nodes comma-separated: g<cols> Gemm (inner = current width), b Bias, a Add,
// l LayerNorm, e Gelu, r Relu, s Softmax, m MhaFused. The same grammar is parsed by
// tests/cpp/host_api_test.cpp for the C++ API under test.
OpGraph graph_of(const std::string& model, const GraphHyper& hy) {
    if (model.rfind("spec:", 0) != 0) return build_preset_graph(model, hy);
    OpGraph g;
    g.name = model;
    g.hyper = hy;
    const std::int64_t rows = hy.bs * hy.seq_len;
    std::int64_t w = hy.hidden_dim;
    std::stringstream ss(model.substr(5));
    std::string tok;
    while (std::getline(ss, tok, ',')) {
        const int id = static_cast<int>(g.nodes.size());
        switch (tok.at(0)) {
            case 'g': { const std::int64_t c = std::stoll(tok.substr(1)); g.nodes.push_back({id, OpKind::Gemm, rows, c, w}); w = c; break; }
            case 'b': g.nodes.push_back({id, OpKind::Bias, rows, w, 0}); break;
            case 'a': g.nodes.push_back({id, OpKind::Add, rows, w, 0}); break;
            case 'l': g.nodes.push_back({id, OpKind::LayerNorm, rows, w, 0}); break;
            case 'e': g.nodes.push_back({id, OpKind::Gelu, rows, w, 0}); break;
            case 'r': g.nodes.push_back({id, OpKind::Relu, rows, w, 0}); break;
            case 's': g.nodes.push_back({id, OpKind::Softmax, rows, w, 0}); break;
            case 'm': g.nodes.push_back({id, OpKind::MhaFused, rows, w, 0}); break;
            default: throw invalid_parameter("bad graph spec token " + tok);
        }
    }
    return g;
}

// exec_segment (backend.hpp:360) of one segment of a preset / spec graph on GraphData(seed), fed
// `in`; with a mask (n x n uint8, may be null) the MHA context is built at block (bm, bn).
int ref_exec_segment(const char* model, int64_t bs, int64_t seq, int64_t hidden, int heads,
                     int head_size, uint64_t seed, int seg_begin, int seg_end, const float* in,
                     float* out, const uint8_t* mask, int bm, int bn) {
    return guard([&] {
        GraphHyper hy{bs, seq, hidden, heads, head_size, 0};
        const OpGraph g = graph_of(model, hy);
        const GraphData gd = GraphData::make(g, seed);
        const Segment seg{seg_begin, seg_end};
        const TemplateKind kind = classify_segment(seg, g);
        Matrix x(g.nodes[static_cast<size_t>(seg_begin)].rows,
                 g.nodes[static_cast<size_t>(seg_begin)].kind == OpKind::Gemm
                     ? g.nodes[static_cast<size_t>(seg_begin)].inner
                     : g.nodes[static_cast<size_t>(seg_begin)].cols);
        std::memcpy(x.a.data(), in, x.a.size() * 4);
        std::optional<MhaContext> ctx;
        if (mask) {
            KernelPlan plan;
            plan.kind = KernelKind::BlockWise;
            plan.block_m = bm;
            plan.block_n = bn;
            ctx = MhaContext::make(from_u8(mask, static_cast<int>(seq)), plan);
        }
        const Matrix r = exec_segment(g, gd, ctx ? &*ctx : nullptr, seg, default_setting(kind), x);
        std::memcpy(out, r.a.data(), r.a.size() * 4);
    });
}

// run_pipeline (search.hpp:514) on the reference SyntheticBackend (backend.hpp:516-671): the
// canonical report line the C++ host API test prints for its own search.
int ref_run_pipeline_synthetic(const char* model, int64_t bs, int64_t seq, uint64_t model_seed, uint64_t cfg_seed,
                               int planted, char* out, int64_t cap) {
    return guard([&] {
        GraphHyper hy{bs, seq, 768, 12, 64, 0};
        const OpGraph g = build_preset_graph(model, hy);
        SyntheticCostModel m = SyntheticCostModel::random_model(model_seed);
        if (planted) m.planted = SyntheticCostModel::Planted{{{0, 1}, {1, 5}, {5, 9}, {9, 12}}};
        SyntheticBackend be(m);
        SearchConfig cfg;
        cfg.seed = cfg_seed;
        TuningCache cache;
        const TuningReport r = run_pipeline(g, hw_preset("a100"), DenseMask(static_cast<int>(seq), true), be, cfg, cache);
        std::ostringstream o;
        o.precision(17);
        o << "code=" << r.code << ";hex=" << r.code_hex << ";e2e=" << r.end_to_end_s;
        for (const auto& s : r.segments)
            o << ";seg=" << s.seg.begin << "-" << s.seg.end << ":" << s.setting.key() << ":" << s.duration << ":"
              << s.untuned;
        const auto& t = r.stats;
        o << ";stats=" << t.measure_calls << "," << t.sample_evals << "," << t.cache_hits << "," << t.e2e_calls << ","
          << t.e2e_hits << "," << t.schemes_evaluated << "," << t.stage1_accepted << "," << t.stage2_iterations;
        const std::string s = o.str();
        std::strncpy(out, s.c_str(), static_cast<size_t>(cap - 1));
        out[cap - 1] = '\0';
    });
}

// Two-stage search on the SyntheticBackend with tuning-cache persistence (io.hpp:407-458): load the
// context's entries from path_in (if given), run, append the session's entries to path_out.
// Returns the report line (same format as above) — cross-implementation cache files must yield
// identical warm sessions.
int ref_cache_session(const char* model, int64_t bs, int64_t seq, uint64_t model_seed, uint64_t cfg_seed,
                      const char* path_in, const char* path_out, char* out, int64_t cap) {
    return guard([&] {
        GraphHyper hy{bs, seq, 768, 12, 64, 0};
        const OpGraph g = build_preset_graph(model, hy);
        SyntheticCostModel m = SyntheticCostModel::random_model(model_seed);
        SyntheticBackend be(m);
        SearchConfig cfg;
        cfg.seed = cfg_seed;
        const std::string ctx = cache_context(g, be.id(), "a100");
        TuningCache cache = (path_in && path_in[0]) ? load_cache_file(path_in, ctx) : TuningCache{};
        const TuningReport r = run_pipeline(g, hw_preset("a100"), DenseMask(static_cast<int>(seq), true), be, cfg, cache);
        if (path_out && path_out[0]) append_cache_file(path_out, ctx, cache);
        std::ostringstream o;
        o.precision(17);
        o << "ctx=" << ctx << ";code=" << r.code << ";e2e=" << r.end_to_end_s;
        for (const auto& sg : r.segments) o << ";seg=" << sg.seg.begin << "-" << sg.seg.end << ":" << sg.setting.key() << ":" << sg.duration;
        const auto& t = r.stats;
        o << ";stats=" << t.measure_calls << "," << t.sample_evals << "," << t.cache_hits << "," << t.e2e_calls << ","
          << t.e2e_hits;
        const std::string str = o.str();
        std::strncpy(out, str.c_str(), static_cast<size_t>(cap - 1));
        out[cap - 1] = '\0';
    });
}

// validate_bsr (bsr.hpp:104-153) of host arrays, e.g. a built BSR with one field corrupted: returns
// the status and the exception message (empty when valid).
int ref_validate_bsr(int seq_len, int bm, int bn, const int32_t* frp, int64_t n_frp, const int32_t* fci, int64_t n_fci,
                     const int32_t* prp, int64_t n_prp, const int32_t* pci, int64_t n_pci, const int32_t* pti,
                     int64_t n_pti, const int32_t* lrp, int64_t n_lrp, const int32_t* lci, int64_t n_lci,
                     const uint8_t* pool_tiles, int64_t n_pool, char* msg, int64_t cap) {
    msg[0] = '\0';
    try {
        BsrMask b;
        b.seq_len = seq_len;
        b.block_m = bm;
        b.block_n = bn;
        b.n_rows = (seq_len + bm - 1) / bm;
        b.n_cols = (seq_len + bn - 1) / bn;
        b.full_row_ptr.assign(frp, frp + n_frp);
        b.full_col_idx.assign(fci, fci + n_fci);
        b.part_row_ptr.assign(prp, prp + n_prp);
        b.part_col_idx.assign(pci, pci + n_pci);
        b.part_tile_ids.assign(pti, pti + n_pti);
        b.load_row_ptr.assign(lrp, lrp + n_lrp);
        b.load_col_idx.assign(lci, lci + n_lci);
        const size_t tb = static_cast<size_t>(bm) * bn;
        for (int64_t t = 0; t < n_pool; ++t)
            b.part_mask_pool.emplace_back(pool_tiles + t * tb, pool_tiles + (t + 1) * tb);
        validate_bsr(b);
        return SF_OK;
    } catch (const internal_inconsistency& e) {
        std::strncpy(msg, e.what(), static_cast<size_t>(cap - 1));
        msg[cap - 1] = '\0';
        return SF_INTERNAL_INCONSISTENCY;
    } catch (...) {
        return SF_BACKEND_ERROR;
    }
}

}  // extern "C"
