// sparsefuse — command-line surface over the B200 host API (SPEC.md "cli" module; the
// reference's tools/sparsefuse.cpp is a stub). JSON on stdout; exit 0 success, 1 verification
// failure, 2 usage.
//
//   sparsefuse mask gen    <mask flags> [--dump file.sfmk]
//   sparsefuse mask stats  <mask flags> --block BMxBN
//   sparsefuse plan select <mask flags> --hw NAME --heads H --bs B [--head-size D] [--mode reference|b200]
//   sparsefuse fuse encode 0-1,1-3,3-4
//   sparsefuse fuse decode 0110
//   sparsefuse attn verify <mask flags | --pattern none --seq-len N> [--bs B] [--heads H] [--head-size D]
//                          [--seed S] [--tol A] [--tol-rel R] [--inject-fault tile]
//   sparsefuse report show <report.jsonl> [--line K] [--output text|json]
//   mask flags: --pattern P --seq-len N [--band W] [--global G] [--dilation R] [--fill F]
//               [--block-rand B] [--seed S]   (or --sfmk file.sfmk)
// `tune run` is sf_tune (same directory); `report show` renders one of its JSON reports.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <random>
#include <sstream>

#include "sparsefuse_b200/ops.hpp"
#include "sparsefuse_b200/fusion.hpp"
#include "sparsefuse_b200/io.hpp"

using namespace sparsefuse;

namespace {

struct Args {
    std::vector<std::string> pos;
    std::map<std::string, std::string> kv;
    std::string get(const std::string& k, const std::string& d = "") const {
        const auto it = kv.find(k);
        return it == kv.end() ? d : it->second;
    }
    bool has(const std::string& k) const { return kv.count(k) != 0; }
};

Args parse(int argc, char** argv, int from) {
    Args a;
    for (int i = from; i < argc; ++i) {
        const std::string s = argv[i];
        if (s.rfind("--", 0) == 0 && i + 1 < argc) a.kv[s.substr(2)] = argv[++i];
        else a.pos.push_back(s);
    }
    return a;
}

[[noreturn]] void usage(const std::string& why) {
    std::cout << "{\"error\": \"usage\", \"message\": \"" << why << "\"}" << std::endl;
    std::exit(2);
}

std::string num(double v) {
    std::ostringstream o;
    o.precision(17);
    o << v;
    return o.str();
}

MaskDescriptor descriptor(const Args& a) {
    if (!a.has("pattern") || !a.has("seq-len")) usage("mask flags need --pattern and --seq-len");
    MaskDescriptor d;
    d.pattern = a.get("pattern");
    d.seq_len = std::atoi(a.get("seq-len").c_str());
    d.params.band_width = std::atoi(a.get("band", "0").c_str());
    d.params.global_width = std::atoi(a.get("global", "0").c_str());
    d.params.dilation_rate = std::atoi(a.get("dilation", "0").c_str());
    d.params.filling_rate = std::atof(a.get("fill", "0").c_str());
    d.params.block = std::atoi(a.get("block-rand", "16").c_str());
    d.params.seed = std::strtoull(a.get("seed", "0").c_str(), nullptr, 10);
    return d;
}

DenseMask mask_of(const Args& a) {
    if (a.has("sfmk")) {
        std::ifstream f(a.get("sfmk"), std::ios::binary);
        if (!f) usage("cannot open " + a.get("sfmk"));
        const std::string data((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
        int32_t n = 0;
        check(sf_mask_deserialize(reinterpret_cast<const uint8_t*>(data.data()), static_cast<int64_t>(data.size()), &n,
                                  nullptr, nullptr));
        DenseMask m(n);
        check(sf_mask_deserialize(reinterpret_cast<const uint8_t*>(data.data()), static_cast<int64_t>(data.size()), &n,
                                  m.mutable_device_bits(), nullptr));
        return m;
    }
    return generate_mask(descriptor(a));
}

int64_t count(const DenseMask& m) {
    int64_t c = 0;
    check(sf_mask_count(m.device_bits(), m.seq_len(), &c, nullptr));
    return c;
}

int mask_gen(const Args& a) {
    const MaskDescriptor d = descriptor(a);
    const DenseMask m = generate_mask(d);
    const int64_t nnz = count(m);
    const double n2 = static_cast<double>(m.seq_len()) * m.seq_len();
    if (a.has("dump")) {
        int64_t nb = 0;
        check(sf_mask_serialize(m.device_bits(), m.seq_len(), nullptr, 0, &nb, nullptr));
        std::vector<uint8_t> buf(static_cast<size_t>(nb));
        check(sf_mask_serialize(m.device_bits(), m.seq_len(), buf.data(), nb, &nb, nullptr));
        std::ofstream(a.get("dump"), std::ios::binary).write(reinterpret_cast<const char*>(buf.data()), nb);
    }
    std::cout << "{\"pattern\": \"" << d.pattern << "\", \"seq_len\": " << d.seq_len << ", \"band_width\": "
              << d.params.band_width << ", \"global_width\": " << d.params.global_width << ", \"dilation_rate\": "
              << d.params.dilation_rate << ", \"filling_rate\": " << num(d.params.filling_rate) << ", \"block\": "
              << d.params.block << ", \"seed\": " << d.params.seed << ", \"nnz\": " << nnz
              << ", \"sparsity\": " << num(1.0 - nnz / n2) << "}" << std::endl;
    return 0;
}

int mask_stats(const Args& a) {
    const DenseMask m = mask_of(a);
    int bm = 16, bn = 16;
    const std::string b = a.get("block", "16x16");
    if (std::sscanf(b.c_str(), "%dx%d", &bm, &bn) < 2) bn = bm;
    const BsrMask bsr = build_bsr(m, bm, bn);
    const BlockStats s = block_stats(bsr);
    const double n2 = static_cast<double>(m.seq_len()) * m.seq_len();
    std::cout << "{\"seq_len\": " << m.seq_len() << ", \"block_m\": " << bm << ", \"block_n\": " << bn
              << ", \"full_count\": " << s.full_count << ", \"part_count\": " << s.part_count << ", \"empty_count\": "
              << s.empty_count << ", \"valid_block_ratio\": " << num(s.valid_block_ratio) << ", \"sparsity\": "
              << num(1.0 - count(m) / n2) << ", \"pool\": " << bsr.part_mask_pool.size() << "}" << std::endl;
    return 0;
}

int plan_select(const Args& a) {
    const DenseMask m = mask_of(a);
    const HardwareSpec hw = hw_preset(a.get("hw", "b200"));
    const PlanMode mode = a.get("mode", "reference") == "b200" ? PlanMode::B200 : PlanMode::Reference;
    const KernelPlan p = select_plan(m, hw, m.seq_len(), std::atoi(a.get("heads", "12").c_str()),
                                     std::atoll(a.get("bs", "1").c_str()), std::atoi(a.get("head-size", "64").c_str()), mode);
    std::cout << "{\"kind\": \"" << to_string(p.kind) << "\", \"block_m\": " << p.block_m << ", \"block_n\": "
              << p.block_n << ", \"num_warps\": " << p.num_warps << ", \"score\": " << num(p.score)
              << ", \"threshold\": " << (std::isnan(p.threshold) ? std::string("null") : num(p.threshold))
              << ", \"fallback\": " << (p.fallback ? "true" : "false") << ", \"hw\": \"" << hw.name << "\"}" << std::endl;
    return 0;
}

int fuse(const Args& a, const std::string& op) {
    if (a.pos.empty()) usage("fuse " + op + " needs an argument");
    if (op == "decode") {
        const auto segs = decode(a.pos[0]);
        std::cout << "{\"code\": \"" << a.pos[0] << "\", \"segments\": [";
        for (size_t i = 0; i < segs.size(); ++i) std::cout << (i ? ", " : "") << "[" << segs[i].begin << ", " << segs[i].end << "]";
        std::cout << "]}" << std::endl;
        return 0;
    }
    std::vector<Segment> segs;
    std::stringstream ss(a.pos[0]);
    std::string item;
    while (std::getline(ss, item, ',')) {
        int b = 0, e = 0;
        if (std::sscanf(item.c_str(), "%d-%d", &b, &e) != 2) usage("segments look like 0-1,1-3");
        segs.push_back({b, e});
    }
    std::cout << "{\"code\": \"" << encode(segs) << "\"}" << std::endl;
    return 0;
}

// attn verify: the dense oracle (dense_sdpa_oracle on the device, fp64, from
// the DENSE mask) vs the block-wise executor (tcgen05 at the B200 plan's tile, over the BSR) vs
// the row-wise executor (over the CSR) on the same seeded inputs; max-abs and mean-rel errors of
// each sparse executor against the oracle, and the loaded-tile count against block_stats.
// --inject-fault flips one tile of the BSR before the block-wise run (a full tile dropped, a part
// tile's bits inverted, or, for a mask with no valid tile, tile (0,0) made full): the run must
// then fail (exit 1) with a diff report.
namespace {
struct Diff {
    double max_abs = 0.0, sum_abs = 0.0, sum_ref = 0.0;
    int64_t at = -1;
    double got = 0.0, want = 0.0;
    double mean_rel() const { return sum_ref > 0.0 ? sum_abs / sum_ref : sum_abs; }
};
template <typename T>
Diff diff(const Tensor4<T>& got, const Tensor4<double>& want) {
    Diff r;
    for (size_t i = 0; i < want.v.size(); ++i) {
        const double e = std::abs(static_cast<double>(got.v[i]) - want.v[i]);
        r.sum_abs += e;
        r.sum_ref += std::abs(want.v[i]);
        if (e > r.max_abs) {
            r.max_abs = e;
            r.at = static_cast<int64_t>(i);
            r.got = static_cast<double>(got.v[i]);
            r.want = want.v[i];
        }
    }
    return r;
}

// flip one tile of a host BsrMask (keeps the arrays structurally valid); returns what was done
std::string flip_one_tile(BsrMask& b) {
    const size_t tb = static_cast<size_t>(b.block_m) * b.block_n;
    auto shift = [](std::vector<int32_t>& rp, int from, int by) {
        for (size_t r = static_cast<size_t>(from); r < rp.size(); ++r) rp[r] += by;
    };
    for (int r = 0; r < b.n_rows; ++r) {
        if (b.full_row_ptr[r + 1] > b.full_row_ptr[r]) {  // drop the row block's first full tile
            const int c = b.full_col_idx[b.full_row_ptr[r]];
            b.full_col_idx.erase(b.full_col_idx.begin() + b.full_row_ptr[r]);
            shift(b.full_row_ptr, r + 1, -1);
            for (int k = b.load_row_ptr[r]; k < b.load_row_ptr[r + 1]; ++k)
                if (b.load_col_idx[k] == c) {
                    b.load_col_idx.erase(b.load_col_idx.begin() + k);
                    break;
                }
            shift(b.load_row_ptr, r + 1, -1);
            return "full tile (" + std::to_string(r) + ", " + std::to_string(c) + ") dropped";
        }
        if (b.part_row_ptr[r + 1] > b.part_row_ptr[r]) {  // invert the bits of its first part tile
            const int k = b.part_row_ptr[r];
            std::vector<uint8_t> inv = b.part_mask_pool[b.part_tile_ids[k]];
            for (auto& x : inv) x = x ? 0 : 1;
            b.part_mask_pool.push_back(std::move(inv));
            b.part_tile_ids[k] = static_cast<int32_t>(b.part_mask_pool.size() - 1);
            (void)tb;
            return "part tile (" + std::to_string(r) + ", " + std::to_string(b.part_col_idx[k]) + ") bits inverted";
        }
    }
    // no valid tile at all: make tile (0, 0) full
    b.full_col_idx.insert(b.full_col_idx.begin(), 0);
    shift(b.full_row_ptr, 1, 1);
    b.load_col_idx.insert(b.load_col_idx.begin(), 0);
    shift(b.load_row_ptr, 1, 1);
    return "empty tile (0, 0) made full";
}
}  // namespace

int attn_verify(const Args& a) {
    const DenseMask m = a.get("pattern") == "none" ? DenseMask(std::atoi(a.get("seq-len", "0").c_str()), false) : mask_of(a);
    const int bs = std::atoi(a.get("bs", "1").c_str()), h = std::atoi(a.get("heads", "2").c_str());
    const int d = std::atoi(a.get("head-size", "64").c_str());
    const auto in = random_attention_input<float>(bs, h, m.seq_len(), d, std::strtoull(a.get("seed", "1").c_str(), nullptr, 10));
    const AttentionInput<double> ind{in.q.cast<double>(), in.k.cast<double>(), in.v.cast<double>()};
    const KernelPlan p = select_plan(m, hw_preset("b200"), m.seq_len(), h, bs, d, PlanMode::B200);
    const int bm = p.kind == KernelKind::BlockWise ? p.block_m : 128, bn = p.kind == KernelKind::BlockWise ? p.block_n : 16;
    BsrMask bsr = build_bsr(m, bm, bn);
    const BlockStats bs_ = block_stats(bsr);
    std::string fault;
    if (a.has("inject-fault")) {
        fault = flip_one_tile(bsr);
        bsr.device = upload_bsr(bsr);
    }
    const Tensor4<double> want = dense_sdpa_oracle(ind, m);
    BlockExecStats st;
    const Diff dbw = diff(block_sparse_sdpa(in, bsr, &st), want);
    const Diff drw = diff(rowwise_sdpa(ind, build_rowwise(m)), want);
    const bool tiles_ok = st.tiles_loaded == bs_.full_count + bs_.part_count;
    const double tol = std::atof(a.get("tol", "2e-2").c_str()), tol_rel = std::atof(a.get("tol-rel", "1e-3").c_str());
    const bool bw_ok = dbw.max_abs <= tol && dbw.mean_rel() <= tol_rel, rw_ok = drw.max_abs <= tol && drw.mean_rel() <= tol_rel;
    const bool pass = bw_ok && rw_ok && tiles_ok;
    std::cout << "{\"pass\": " << (pass ? "true" : "false") << ", \"oracle\": \"dense_sdpa_oracle (device, fp64)\""
              << ", \"max_abs_blockwise\": " << num(dbw.max_abs) << ", \"mean_rel_blockwise\": " << num(dbw.mean_rel())
              << ", \"max_abs_rowwise\": " << num(drw.max_abs) << ", \"mean_rel_rowwise\": " << num(drw.mean_rel())
              << ", \"tolerance\": {\"max_abs\": " << num(tol) << ", \"mean_rel\": " << num(tol_rel) << "}"
              << ", \"block\": [" << bm << ", " << bn << "], \"tiles_loaded\": " << st.tiles_loaded
              << ", \"valid_tiles\": " << bs_.full_count + bs_.part_count << ", \"fault_injected\": "
              << (fault.empty() ? "null" : "\"" + fault + "\"");
    if (!pass) {  // diff report: the worst element of the failing executor
        const bool bw_bad = !bw_ok || !tiles_ok;
        const Diff& w = bw_bad ? dbw : drw;
        const int64_t n = m.seq_len(), i = w.at < 0 ? 0 : w.at;
        std::cout << ", \"diff\": {\"executor\": \"" << (bw_bad ? "block_wise" : "row_wise") << "\", \"b\": " << i / (int64_t(h) * n * d)
                  << ", \"h\": " << (i / (n * d)) % h << ", \"row\": " << (i / d) % n << ", \"col\": " << i % d
                  << ", \"got\": " << num(w.got) << ", \"want\": " << num(w.want) << "}";
    }
    std::cout << "}" << std::endl;
    return pass ? 0 : 1;
}

// report show: a human-readable summary of a tuning report (sf_tune's JSON line, the fields of
// the reference's report); --output json re-emits the selected line unchanged
int report_show(const Args& a) {
    if (a.pos.empty()) usage("report show needs a report file");
    std::ifstream f(a.pos[0]);
    if (!f) usage("cannot open " + a.pos[0]);
    const int want = std::atoi(a.get("line", "0").c_str());
    std::string line;
    for (int i = 0; std::getline(f, line); ++i)
        if (i == want) break;
    if (line.find_first_not_of(" \t\r") == std::string::npos) usage("no report on line " + std::to_string(want));
    if (a.get("output", "text") == "json") {
        std::cout << line << std::endl;
        return 0;
    }
    using io_detail::Value;
    const Value r = io_detail::Parser(line).parse();
    auto num_of = [](const Value& v) { return v.number(); };
    auto us = [](double s) {
        char b[32];
        std::snprintf(b, sizeof b, "%.1f us", s * 1e6);
        return std::string(b);
    };
    const Value& hy = r.at("hyper");
    const Value& pl = r.at("plan");
    std::cout << r.at("graph").str() << "  bs " << num_of(hy.at("bs")) << "  seq " << num_of(hy.at("seq_len"))
              << "  hidden " << num_of(hy.at("hidden")) << "  heads " << num_of(hy.at("heads")) << " x "
              << num_of(hy.at("head_size")) << "  mask " << r.at("mask").str() << "  hw " << r.at("hw").str()
              << " / backend " << r.at("backend").str() << "\n";
    std::cout << "plan: " << pl.at("kind").str() << " (" << num_of(pl.at("block_m")) << " x " << num_of(pl.at("block_n"))
              << "), threshold " << num_of(pl.at("threshold")) << "\n";
    const double e2e = num_of(r.at("end_to_end_s"));
    std::cout << "scheme " << r.at("code").str() << " (hex " << r.at("code_hex").str() << "), end-to-end " << us(e2e);
    if (r.has("end_to_end_unfused_s")) {
        const double u = num_of(r.at("end_to_end_unfused_s"));
        char b[64];
        std::snprintf(b, sizeof b, " (unfused %s, %.2fx)", us(u).c_str(), e2e > 0 ? u / e2e : 0.0);
        std::cout << b;
    }
    std::cout << "\n";
    const auto& segs = std::get<std::vector<Value>>(r.at("segments").v);
    for (const auto& sg : segs) {
        std::string ops;
        for (const auto& o : std::get<std::vector<Value>>(sg.at("ops").v)) ops += (ops.empty() ? "" : "+") + o.str();
        char b[256];
        std::snprintf(b, sizeof b, "  [%2d,%2d) %-34s %-22s %12s%s\n", static_cast<int>(num_of(sg.at("begin"))),
                      static_cast<int>(num_of(sg.at("end"))), ops.c_str(), sg.at("setting").str().c_str(),
                      us(num_of(sg.at("duration_s"))).c_str(),
                      std::get<bool>(sg.at("untuned").v) ? "  (untuned)" : "");
        std::cout << b;
    }
    const Value& st = r.at("stats");
    const double meas = num_of(st.at("measure_calls")), hits = num_of(st.at("cache_hits"));
    char b[256];
    std::snprintf(b, sizeof b,
                  "search: %.0f measurements, %.0f sample evals, %.0f cache hits (%.1f%%), %.0f end-to-end runs, %.0f "
                  "schemes, stage-1 accepted %.0f, stage-2 iterations %.0f; tuning %.3f s\n",
                  meas, num_of(st.at("sample_evals")), hits, meas + hits > 0 ? 100.0 * hits / (meas + hits) : 0.0,
                  num_of(st.at("e2e_calls")), num_of(st.at("schemes_evaluated")), num_of(st.at("stage1_accepted")),
                  num_of(st.at("stage2_iterations")), num_of(r.at("tuning_wall_s")));
    std::cout << b;
    if (r.has("cache")) {
        const Value& c = r.at("cache");
        const std::string file = c.at("file").str();
        std::cout << "cache: ctx " << c.at("ctx").str() << ", file " << (file.empty() ? "-" : file) << ", "
                  << num_of(c.at("preloaded_entries")) << " preloaded entries\n";
    }
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 3) usage("sparsefuse <mask|plan|fuse|attn|report> <command> [flags]");
    const std::string grp = argv[1], cmd = argv[2];
    const Args a = parse(argc, argv, 3);
    try {
        if (grp == "mask" && cmd == "gen") return mask_gen(a);
        if (grp == "mask" && cmd == "stats") return mask_stats(a);
        if (grp == "plan" && cmd == "select") return plan_select(a);
        if (grp == "fuse" && (cmd == "encode" || cmd == "decode")) return fuse(a, cmd);
        if (grp == "attn" && cmd == "verify") return attn_verify(a);
        if (grp == "report" && cmd == "show") return report_show(a);
    } catch (const io_error& e) {
        std::cout << "{\"error\": \"io_error\", \"message\": \"" << e.what() << "\"}" << std::endl;
        return 1;
    } catch (const std::invalid_argument& e) {
        std::cout << "{\"error\": \"invalid_parameter\", \"message\": \"" << e.what() << "\"}" << std::endl;
        return 2;
    } catch (const std::exception& e) {
        std::cout << "{\"error\": \"failure\", \"message\": \"" << e.what() << "\"}" << std::endl;
        return 1;
    }
    usage("unknown command " + grp + " " + cmd);
}
