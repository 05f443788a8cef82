// sf_tune — the two-stage fusion search (search.hpp:514-554 run_pipeline) at a BASELINE
// configuration, measured on the B200 (GpuBackend: segments executed by the fused kernels,
// CUDA-event timed with the reference's 3-warm-up best-of-N protocol, backend.hpp:488-500), with a
// JSON tuning report on stdout (the fields of the reference's report, io.hpp:360-458).
//
//   sf_tune <bert-layer|gpt-layer|t5-layer> <bs> <seq_len> <mask> [seed] [--cache file.jsonl]
//   mask := term("+"term)*, term := pattern[:band[:global[:dilation[:fill[:seed]]]]]
//   e.g.   sf_tune t5-layer 8 4096 dilated:64:0:1+global:0:64
// --cache: the tuning cache persisted across sessions (io.hpp:407-458 schema and context hash,
// interchangeable with the reference's files): the context's entries are loaded before the
// search and the session's new measurements appended after it.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <sstream>

#include "sparsefuse_b200/gpu_backend.hpp"
#include "sparsefuse_b200/io.hpp"

using namespace sparsefuse;

static std::vector<std::string> split(const std::string& s, char c) {
    std::vector<std::string> out;
    std::string cur;
    for (char ch : s) {
        if (ch == c) {
            out.push_back(cur);
            cur.clear();
        } else {
            cur += ch;
        }
    }
    out.push_back(cur);
    return out;
}

static DenseMask parse_mask(const std::string& spec, int n) {
    std::vector<MaskDescriptor> terms;
    for (const auto& t : split(spec, '+')) {
        const auto f = split(t, ':');
        MaskDescriptor d;
        d.pattern = f[0];
        d.seq_len = n;
        auto num = [&](std::size_t i, double dflt) { return f.size() > i && !f[i].empty() ? std::atof(f[i].c_str()) : dflt; };
        d.params.band_width = static_cast<int>(num(1, 0));
        d.params.global_width = static_cast<int>(num(2, 0));
        d.params.dilation_rate = static_cast<int>(num(3, 0));
        d.params.filling_rate = num(4, 0.0);
        d.params.block = 16;
        d.params.seed = static_cast<std::uint64_t>(num(5, 0));
        terms.push_back(d);
    }
    return generate_mask(terms);
}

static std::string jstr(const std::string& s) { return "\"" + s + "\""; }

int main(int argc, char** argv) {
    std::string cache_path;
    std::vector<char*> pos;
    for (int i = 1; i < argc; ++i) {
        if (std::string(argv[i]) == "--cache" && i + 1 < argc) cache_path = argv[++i];
        else pos.push_back(argv[i]);
    }
    if (pos.size() < 4) {
        std::fprintf(stderr, "usage: sf_tune <model> <bs> <seq_len> <mask> [seed] [--cache file.jsonl]\n");
        return 2;
    }
    argc = static_cast<int>(pos.size()) + 1;
    pos.insert(pos.begin(), argv[0]);
    argv = pos.data();
    try {
        const std::string model = argv[1];
        GraphHyper hy{std::atoll(argv[2]), std::atoll(argv[3]), 768, 12, 64, 0};
        const std::uint64_t seed = argc > 5 ? std::strtoull(argv[5], nullptr, 10) : 0;
        const OpGraph g = build_preset_graph(model, hy);
        const auto t_mask = std::chrono::steady_clock::now();
        const DenseMask mask = parse_mask(argv[4], static_cast<int>(hy.seq_len));
        const KernelPlan plan = select_plan(mask, hw_preset("b200"), hy.seq_len, hy.heads, hy.bs, hy.head_size, PlanMode::B200);
        const double plan_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t_mask).count();
        GpuBackend be(g, 1, mask, plan);
        SearchConfig cfg;
        cfg.space = ParamSpace::b200();
        cfg.seed = seed;
        const std::string ctx = cache_context(g, be.id(), "b200");
        TuningCache cache = cache_path.empty() ? TuningCache{} : load_cache_file(cache_path, ctx);
        const std::int64_t preloaded = cache.size();
        const TuningReport r = run_pipeline(g, hw_preset("b200"), plan, be, cfg, cache);
        if (!cache_path.empty()) append_cache_file(cache_path, ctx, cache);
        const auto unfused = unfused_scheme(g.size());
        const double e2e_unfused = be.end_to_end(g, unfused, {});
        std::ostringstream o;
        o.precision(9);
        o << "{\"version\": " << r.version << ", \"graph\": " << jstr(r.graph_name) << ", \"hyper\": {\"bs\": " << hy.bs
          << ", \"seq_len\": " << hy.seq_len << ", \"hidden\": " << hy.hidden_dim << ", \"heads\": " << hy.heads
          << ", \"head_size\": " << hy.head_size << "}, \"mask\": " << jstr(argv[4]) << ", \"hw\": " << jstr(r.hw_name)
          << ", \"backend\": " << jstr(r.backend_id) << ", \"plan\": {\"kind\": "
          << jstr(plan.kind == KernelKind::BlockWise ? "block_wise" : "row_wise") << ", \"block_m\": " << plan.block_m
          << ", \"block_n\": " << plan.block_n << ", \"threshold\": " << plan.threshold << ", \"select_s\": " << plan_s
          << "}, \"code\": " << jstr(r.code) << ", \"code_hex\": " << jstr(r.code_hex) << ", \"segments\": [";
        for (std::size_t i = 0; i < r.segments.size(); ++i) {
            const auto& s = r.segments[i];
            o << (i ? ", " : "") << "{\"begin\": " << s.seg.begin << ", \"end\": " << s.seg.end << ", \"ops\": [";
            for (std::size_t k = 0; k < s.ops.size(); ++k) o << (k ? ", " : "") << jstr(s.ops[k]);
            o << "], \"setting\": " << jstr(s.setting.key()) << ", \"duration_s\": " << s.duration
              << ", \"untuned\": " << (s.untuned ? "true" : "false") << "}";
        }
        const auto& t = r.stats;
        o << "], \"end_to_end_s\": " << r.end_to_end_s << ", \"end_to_end_unfused_s\": " << e2e_unfused
          << ", \"seed\": " << r.seed << ", \"stats\": {\"measure_calls\": " << t.measure_calls
          << ", \"sample_evals\": " << t.sample_evals << ", \"cache_hits\": " << t.cache_hits << ", \"e2e_calls\": "
          << t.e2e_calls << ", \"schemes_evaluated\": " << t.schemes_evaluated << ", \"stage1_accepted\": "
          << t.stage1_accepted << ", \"stage2_iterations\": " << t.stage2_iterations
          << "}, \"cache\": {\"ctx\": " << jstr(ctx) << ", \"file\": " << jstr(cache_path)
          << ", \"preloaded_entries\": " << preloaded << "}, \"tuning_wall_s\": " << r.wall_time_s << "}";
        std::cout << o.str() << std::endl;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "sf_tune: %s\n", e.what());
        return 1;
    }
    return 0;
}
