// host_api_test.cpp — exercises the C++ host API (include/sparsefuse_b200/) the way the
// reference's own Catch2 suites exercise theirs. Driven by tests/test_cpp_host_api.py.
//
//   host_api_test search <model> <bs> <seq> <model_seed> <cfg_seed> <planted 0|1>
//       run_pipeline on the SyntheticBackend (host only); prints a canonical report line that the
//       Python test compares with the reference's run_pipeline (oracle/_ref).
//   host_api_test gpu-basics       masks / formats / selector / attention through the C++ API
//   host_api_test gpu-backend      GpuBackend: chain on the device + a device-timed search
//   host_api_test exec-segment ... exec_segment / exec_mha (host Matrix API) on one segment
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>

#include "sparsefuse_b200/gpu_backend.hpp"
#include "sparsefuse_b200/io.hpp"

using namespace sparsefuse;

#define REQUIRE(c)                                                                  \
    do {                                                                            \
        if (!(c)) {                                                                 \
            std::fprintf(stderr, "REQUIRE failed %s:%d: %s\n", __FILE__, __LINE__, #c); \
            std::exit(1);                                                           \
        }                                                                           \
    } while (0)

template <typename E, typename F>
bool throws_as(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static std::string report_line(const TuningReport& r) {
    std::ostringstream o;
    o.precision(17);
    o << "code=" << r.code << ";hex=" << r.code_hex << ";e2e=" << r.end_to_end_s;
    for (const auto& s : r.segments)
        o << ";seg=" << s.seg.begin << "-" << s.seg.end << ":" << s.setting.key() << ":" << s.duration << ":" << s.untuned;
    const auto& t = r.stats;
    o << ";stats=" << t.measure_calls << "," << t.sample_evals << "," << t.cache_hits << "," << t.e2e_calls << ","
      << t.e2e_hits << "," << t.schemes_evaluated << "," << t.stage1_accepted << "," << t.stage2_iterations;
    return o.str();
}

static int cmd_search(int argc, char** argv) {
    if (argc < 8) return 2;
    const std::string model = argv[2];
    GraphHyper hy{std::atoll(argv[3]), std::atoll(argv[4]), 768, 12, 64, 0};
    OpGraph g = build_preset_graph(model, hy);
    SyntheticCostModel m = SyntheticCostModel::random_model(std::strtoull(argv[5], nullptr, 10));
    if (std::atoi(argv[7])) m.planted = SyntheticCostModel::Planted{{{0, 1}, {1, 5}, {5, 9}, {9, 12}}};
    SyntheticBackend be(m);
    SearchConfig cfg;
    cfg.seed = std::strtoull(argv[6], nullptr, 10);
    TuningCache cache;
    KernelPlan plan;  // the analytical MHA plan does not take part in the search itself
    const TuningReport r = run_pipeline(g, HardwareSpec{"a100", 108, 192 * 1024, 64, 2}, plan, be, cfg, cache);
    std::cout << report_line(r) << "\n";
    // a warm re-run on the same cache re-finds the same scheme (stage 1 is fully cache-served)
    const TuningReport r2 = run_pipeline(g, HardwareSpec{"a100", 108, 192 * 1024, 64, 2}, plan, be, cfg, cache);
    REQUIRE(r2.code == r.code);
    return 0;
}

// host_api_test cache <model> <bs> <seq> <model_seed> <cfg_seed> <path_in|-> <path_out|->
// the reference's ref_cache_session, through this API (tests/test_cpp_host_api.py)
static int cmd_cache(int argc, char** argv) {
    if (argc < 9) return 2;
    GraphHyper hy{std::atoll(argv[3]), std::atoll(argv[4]), 768, 12, 64, 0};
    const OpGraph g = build_preset_graph(argv[2], hy);
    SyntheticBackend be(SyntheticCostModel::random_model(std::strtoull(argv[5], nullptr, 10)));
    SearchConfig cfg;
    cfg.seed = std::strtoull(argv[6], nullptr, 10);
    const std::string in = argv[7], out = argv[8];
    const std::string ctx = cache_context(g, be.id(), "a100");
    TuningCache cache = in != "-" ? load_cache_file(in, ctx) : TuningCache{};
    KernelPlan plan;
    const TuningReport r = run_pipeline(g, HardwareSpec{"a100", 108, 192 * 1024, 64, 2}, plan, be, cfg, cache);
    if (out != "-") append_cache_file(out, ctx, cache);
    std::ostringstream o;
    o.precision(17);
    o << "ctx=" << ctx << ";code=" << r.code << ";e2e=" << r.end_to_end_s;
    for (const auto& s : r.segments) o << ";seg=" << s.seg.begin << "-" << s.seg.end << ":" << s.setting.key() << ":" << s.duration;
    const auto& t = r.stats;
    o << ";stats=" << t.measure_calls << "," << t.sample_evals << "," << t.cache_hits << "," << t.e2e_calls << "," << t.e2e_hits;
    std::cout << o.str() << "\n";
    return 0;
}

static double max_abs(const Tensor4<float>& a, const Tensor4<double>& b) {
    double m = 0;
    for (std::size_t i = 0; i < a.v.size(); ++i) m = std::max(m, std::abs(static_cast<double>(a.v[i]) - b.v[i]));
    return m;
}

// fp64 dense reference for the checks below (attention.hpp:19-56 semantics), test-local
static Tensor4<double> dense_ref(const AttentionInput<float>& in, const DenseMask& mask) {
    const int n = in.seq_len(), d = in.head_size();
    Tensor4<double> out(in.bs(), in.h(), n, d);
    const double sc = 1.0 / std::sqrt(static_cast<double>(d));
    for (int b = 0; b < in.bs(); ++b)
        for (int h = 0; h < in.h(); ++h)
            for (int i = 0; i < n; ++i) {
                std::vector<double> s(static_cast<std::size_t>(n), -INFINITY);
                double mx = -INFINITY;
                for (int j = 0; j < n; ++j) {
                    if (!mask.get(i, j)) continue;
                    double dot = 0;
                    for (int k = 0; k < d; ++k)
                        dot += static_cast<double>(__half2float(__float2half(in.q.at(b, h, i, k)))) *
                               __half2float(__float2half(in.k.at(b, h, j, k)));
                    s[static_cast<std::size_t>(j)] = dot * sc;
                    mx = std::max(mx, dot * sc);
                }
                if (mx == -INFINITY) continue;
                double den = 0;
                for (double x : s)
                    if (x != -INFINITY) den += std::exp(x - mx);
                for (int j = 0; j < n; ++j) {
                    if (s[static_cast<std::size_t>(j)] == -INFINITY) continue;
                    const double p = std::exp(s[static_cast<std::size_t>(j)] - mx) / den;
                    for (int k = 0; k < d; ++k) out.at(b, h, i, k) += p * __half2float(__float2half(in.v.at(b, h, j, k)));
                }
            }
    return out;
}

static int cmd_gpu_basics() {
    // test_mask.cpp-style
    REQUIRE(gen_sliding_window(4, 4).true_count() == 16);
    REQUIRE(gen_dilated(8, 2, 1).true_count() == 20);
    REQUIRE(std::abs(sparsity(gen_sliding_window(1024, 32)) - 0.938) <= 0.005);
    REQUIRE(throws_as<invalid_parameter>([] { gen_sliding_window(16, 0); }));
    REQUIRE(throws_as<invalid_parameter>([] { gen_sliding_window(16, 17); }));
    REQUIRE(gen_bigbird(512, 22, 22, 0.3, 4) == gen_bigbird(512, 22, 22, 0.3, 4));
    const DenseMask bb = gen_bigbird(128, 8, 8, 0.2, 9);
    REQUIRE(bb == compose({gen_global(128, 8), gen_sliding_window(128, 8), gen_random_blocks(128, 16, 0.2, 9)}));
    DenseMask edited(32, false);
    edited.set(3, 4, true);
    REQUIRE(edited.true_count() == 1 && edited.get(3, 4) && !edited.get(4, 3));
    // test_bsr.cpp-style
    {
        const auto b = build_bsr(DenseMask(64, true), 16, 16);
        REQUIRE(b.full_row_ptr.back() == 16 && b.part_row_ptr.back() == 0 && b.part_mask_pool.empty());
        REQUIRE(block_stats(b).valid_block_ratio == 1.0);
        const auto e = build_bsr(DenseMask(64, false), 16, 16);
        REQUIRE(e.load_row_ptr.back() == 0);
        REQUIRE(throws_as<invalid_parameter>([] { build_bsr(DenseMask(16, true), 0, 4); }));
    }
    {
        const auto r = build_rowwise(gen_sliding_window(40, 3));
        REQUIRE(r.row_ptr.back() == static_cast<int>(gen_sliding_window(40, 3).true_count()));
    }
    // test_planner.cpp-style
    REQUIRE(std::abs(threshold(DenseMask(1024, true)) - (1.0 - 1.2 / 36.0)) <= 1e-12);
    REQUIRE(throws_as<degenerate_input>([] { threshold(DenseMask(16, true)); }));
    REQUIRE(hw_preset("a100").sm_num == 108 && hw_preset("rtx4090").max_warp == 48);
    REQUIRE(throws_as<invalid_parameter>([] { hw_preset("h100"); }));
    const auto p = select_plan(DenseMask(1024, true), hw_preset("a100"), 1024, 12, 8, 64);
    REQUIRE(p.kind == KernelKind::BlockWise && p.block_m == 16 && p.block_n == 16 && p.num_warps == 4);
    REQUIRE(std::isnan(select_plan(DenseMask(16, true), hw_preset("a100"), 16, 12, 8, 64).threshold));
    const auto pb = select_plan(gen_bigbird(1024, 32, 32, 0.1, 0), hw_preset("b200"), 1024, 12, 16, 64, PlanMode::B200);
    REQUIRE(pb.kind == KernelKind::BlockWise && pb.block_m == 64 && pb.block_n == 16);  // head pairs for BigBird
    // test_attention.cpp-style, through the host-tensor signatures
    {
        const auto in = random_attention_input<float>(2, 2, 16, 8, 1);
        const auto blk = block_sparse_sdpa(in, build_bsr(DenseMask(16, false), 4, 4));
        for (float v : blk.v) REQUIRE(v == 0.0f);
    }
    for (int impl : {1, 0}) {  // generic kernel, then auto (tcgen05 where the tile allows)
        check(sf_set_attn_impl(impl));
        const DenseMask m = gen_bigbird(300, 17, 17, 0.1, 0);
        const auto in = random_attention_input<float>(1, 2, 300, 64, 1);
        BlockExecStats st;
        const auto bsr = build_bsr(m, 128, 16);
        const auto out = block_sparse_sdpa(in, bsr, &st);
        REQUIRE(st.tiles_loaded == bsr.load_row_ptr.back());
        REQUIRE(max_abs(out, dense_ref(in, m)) <= 2e-2);
        KernelPlan wrong;
        wrong.kind = KernelKind::BlockWise;
        wrong.block_m = 16;
        wrong.block_n = 16;
        REQUIRE(throws_as<plan_error>([&] { block_sparse_sdpa(in, bsr, wrong); }));
    }
    check(sf_set_attn_impl(0));
    {
        const DenseMask m = gen_longformer(96, 8, 8);
        const auto in = random_attention_input<float>(1, 2, 96, 32, 7);
        const auto ind = AttentionInput<double>{in.q.cast<double>(), in.k.cast<double>(), in.v.cast<double>()};
        const auto rw = rowwise_sdpa(ind, build_rowwise(m));
        const auto ref = dense_ref(in, m);
        double mx = 0;
        for (std::size_t i = 0; i < rw.v.size(); ++i) mx = std::max(mx, std::abs(rw.v[i] - ref.v[i]));
        REQUIRE(mx <= 2e-2);
    }
    std::cout << "gpu-basics ok\n";
    return 0;
}

static int cmd_gpu_backend() {
    // bert-layer on the device, all-true session mask planned by the B200 selector
    GraphHyper hy{1, 256, 256, 4, 64, 0};
    for (const char* model : {"bert-layer", "gpt-layer", "t5-layer"}) {
        OpGraph g = build_preset_graph(model, hy);
        GpuBackend be(g, 1, gen_bigbird(256, 16, 16, 0.1, 0));
        // fused and unfused schemes compute the same chain
        SearchConfig cfg;
        cfg.space = ParamSpace::b200();
        const FusionScheme init = init_scheme(g, cfg);
        const auto y_unfused = be.run_chain(g, unfused_scheme(g.size()), {});
        const auto y_init = be.run_chain(g, init, {});
        double md = 0, mr = 0;
        for (std::size_t i = 0; i < y_unfused.size(); ++i) {
            md = std::max(md, static_cast<double>(std::abs(y_unfused[i] - y_init[i])));
            mr = std::max(mr, static_cast<double>(std::abs(y_unfused[i])));
        }
        REQUIRE(md <= 2e-2 * std::max(1.0, mr));
        TuningCache cache;
        const TuningReport r = run_pipeline(g, hw_preset("b200"), *be.plan(), be, cfg, cache);
        REQUIRE(r.end_to_end_s > 0 && r.stats.measure_calls > 0);
        std::cout << model << " " << report_line(r) << "\n";
    }
    std::cout << "gpu-backend ok\n";
    return 0;
}

// Same grammar as oracle/ref_shim.cpp graph_of: a preset, or "spec:<nodes>".
static OpGraph graph_of(const std::string& model, const GraphHyper& hy) {
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
        OpNode n{id, OpKind::Bias, rows, w, 0};
        switch (tok.at(0)) {
            case 'g': n.kind = OpKind::Gemm; n.inner = w; n.cols = w = std::stoll(tok.substr(1)); break;
            case 'b': n.kind = OpKind::Bias; break;
            case 'a': n.kind = OpKind::Add; break;
            case 'l': n.kind = OpKind::LayerNorm; break;
            case 'e': n.kind = OpKind::Gelu; break;
            case 'r': n.kind = OpKind::Relu; break;
            case 's': n.kind = OpKind::Softmax; break;
            case 'm': n.kind = OpKind::MhaFused; break;
            default: throw invalid_parameter("bad graph spec token " + tok);
        }
        g.nodes.push_back(n);
    }
    return g;
}

static std::vector<char> read_file(const std::string& path) {
    std::FILE* f = std::fopen(path.c_str(), "rb");
    REQUIRE(f);
    std::vector<char> b;
    char buf[1 << 16];
    std::size_t k;
    while ((k = std::fread(buf, 1, sizeof buf, f)) > 0) b.insert(b.end(), buf, buf + k);
    std::fclose(f);
    return b;
}

// exec-segment <model> <bs> <seq> <hidden> <heads> <head_size> <seed> <seg_begin> <seg_end> <in.f32>
//              <out.f32> [<mask.u8> <bm> <bn> [<strided band>]]
// The reference-signature free functions (exec_segment / exec_mha with host Matrix in / out and an
// MhaContext) on GraphData(seed); the Python test compares the output with the reference's own
// exec_segment (oracle/_ref).
static int cmd_exec_segment(int argc, char** argv) {
    if (argc < 12) return 2;
    GraphHyper hy{std::atoll(argv[3]), std::atoll(argv[4]), std::atoll(argv[5]), std::atoi(argv[6]), std::atoi(argv[7]), 0};
    const OpGraph g = graph_of(argv[2], hy);
    const GraphData gd = GraphData::make(g, std::strtoull(argv[8], nullptr, 10));
    const Segment seg{std::atoi(argv[9]), std::atoi(argv[10])};
    const OpNode& first = g.nodes.at(static_cast<std::size_t>(seg.begin));
    Matrix x(first.rows, first.kind == OpKind::Gemm ? first.inner : first.cols);
    const auto raw = read_file(argv[11]);
    REQUIRE(raw.size() == x.a.size() * 4);
    std::memcpy(x.a.data(), raw.data(), raw.size());
    std::optional<MhaContext> ctx;
    if (argc >= 16) {
        const auto mb = read_file(argv[13]);
        const int n = static_cast<int>(hy.seq_len);
        REQUIRE(mb.size() == static_cast<std::size_t>(n) * n);
        DenseMask m(n);
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j)
                if (mb[static_cast<std::size_t>(i) * n + j]) m.set(i, j, true);
        KernelPlan plan;
        plan.kind = KernelKind::BlockWise;
        plan.block_m = std::atoi(argv[14]);
        plan.block_n = std::atoi(argv[15]);
        // a strided(band) mask may be run by the decomposed executor (MhaContext::make_strided), a
        // mask holding dilated(band, rate) by the class decomposition ("dil:<band>:<rate>", make_dilated)
        if (argc >= 17 && std::strncmp(argv[16], "dil:", 4) == 0) {
            int band = 0, rate = 0;
            REQUIRE(std::sscanf(argv[16], "dil:%d:%d", &band, &rate) == 2);
            ctx = MhaContext::make_dilated(m, plan, band, rate);
        } else {
            ctx = argc >= 17 ? MhaContext::make_strided(m, plan, std::atoi(argv[16])) : MhaContext::make(m, plan);
        }
    }
    const Matrix y = exec_segment(g, gd, ctx ? &*ctx : nullptr, seg, default_setting(classify_segment(seg, g)), x);
    std::FILE* f = std::fopen(argv[12], "wb");
    REQUIRE(f);
    std::fwrite(y.a.data(), 4, y.a.size(), f);
    std::fclose(f);
    std::cout << "exec-segment ok " << y.rows << "x" << y.cols << "\n";
    return 0;
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string cmd = argv[1];
    try {
        if (cmd == "search") return cmd_search(argc, argv);
        if (cmd == "cache") return cmd_cache(argc, argv);
        if (cmd == "gpu-basics") return cmd_gpu_basics();
        if (cmd == "gpu-backend") return cmd_gpu_backend();
        if (cmd == "exec-segment") return cmd_exec_segment(argc, argv);
    } catch (const std::exception& e) {
        std::fprintf(stderr, "exception: %s\n", e.what());
        return 1;
    }
    return 2;
}
