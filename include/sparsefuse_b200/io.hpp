// io.hpp — tuning-cache persistence of the two-stage search (io.hpp:383-458 of the reference):
// one append-only JSON-lines file; every line carries the context hash of the (graph, backend
// id, hardware) it belongs to, so one file serves many sessions. The line schema and the context
// hash are the reference's, so cache files move between the two implementations:
//   {"ctx": "<hex64>", "type": "seg", "code": "...", "begin": b, "end": e,
//    "setting": {"kind": "ci_mi", "tile_m": .., "tile_n": .., "tile_k": ..}, "dur": seconds}
//   {"ctx": "<hex64>", "type": "e2e", "code": "...", "key": "...", "dur": seconds}
// The reader is a small JSON parser for this flat schema (any key order / whitespace; no
// third-party dependency in the product headers).
#pragma once

#include <cctype>
#include <cstdio>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

#include "search.hpp"

namespace sparsefuse {

// graph_signature / cache_context (io.hpp:386-405): identical strings and hash
inline std::string graph_signature(const OpGraph& g) {
    std::string s = g.name + "|" + std::to_string(g.hyper.bs) + "," + std::to_string(g.hyper.seq_len) + "," +
                    std::to_string(g.hyper.hidden_dim) + "," + std::to_string(g.hyper.heads) + "," +
                    std::to_string(g.hyper.head_size) + "," + std::to_string(g.hyper.ff_dim);
    for (const auto& n : g.nodes) {
        s += "|";
        s += to_string(n.kind);
        s += ":" + std::to_string(n.rows) + "x" + std::to_string(n.cols) + "x" + std::to_string(n.inner);
    }
    return s;
}

inline std::string cache_context(const OpGraph& g, const std::string& backend_id, const std::string& hw_name) {
    return hex64(fnv1a(graph_signature(g) + "#" + backend_id + "#" + hw_name));
}

namespace io_detail {

inline std::string quote(const std::string& s) {
    std::string o = "\"";
    for (char c : s) {
        if (c == '"' || c == '\\') o += '\\';
        o += c;
    }
    return o + "\"";
}

inline std::string num(double d) {
    char b[32];
    std::snprintf(b, sizeof b, "%.17g", d);  // round-trips exactly
    return b;
}

inline std::string setting_json(const Setting& s) {
    std::string j = "{\"kind\":" + quote(to_string(s.kind));
    if (s.kind == TemplateKind::MiChain) {
        j += ",\"chunk_size\":" + std::to_string(s.chunk_size);
    } else {
        if (s.kind == TemplateKind::CiCi) j += ",\"stage_depth\":" + std::to_string(s.stage_depth);
        j += ",\"tile_k\":" + std::to_string(s.tile_k) + ",\"tile_m\":" + std::to_string(s.tile_m) +
             ",\"tile_n\":" + std::to_string(s.tile_n);
    }
    return j + "}";
}

// ---- minimal JSON value + parser (objects, arrays, strings, numbers, true/false/null)
struct Value;
using Object = std::map<std::string, Value>;
struct Value {
    std::variant<std::nullptr_t, bool, double, std::string, std::vector<Value>, Object> v;
    const Value& at(const std::string& k) const {
        const auto* o = std::get_if<Object>(&v);
        if (!o) throw io_error("cache line: expected an object");
        const auto it = o->find(k);
        if (it == o->end()) throw io_error("cache line: missing key " + k);
        return it->second;
    }
    bool has(const std::string& k) const {
        const auto* o = std::get_if<Object>(&v);
        return o && o->count(k);
    }
    const std::string& str() const {
        const auto* s = std::get_if<std::string>(&v);
        if (!s) throw io_error("cache line: expected a string");
        return *s;
    }
    double number() const {
        const auto* d = std::get_if<double>(&v);
        if (!d) throw io_error("cache line: expected a number");
        return *d;
    }
};

class Parser {
public:
    explicit Parser(const std::string& s) : s_(s) {}
    Value parse() {
        Value v = value();
        ws();
        if (i_ != s_.size()) fail("trailing characters");
        return v;
    }

private:
    [[noreturn]] void fail(const char* what) const {
        throw io_error(std::string("cache line: ") + what + " at offset " + std::to_string(i_));
    }
    void ws() {
        while (i_ < s_.size() && std::isspace(static_cast<unsigned char>(s_[i_]))) ++i_;
    }
    char peek() {
        ws();
        if (i_ >= s_.size()) fail("unexpected end");
        return s_[i_];
    }
    void expect(char c) {
        if (peek() != c) fail("unexpected character");
        ++i_;
    }
    Value value() {
        const char c = peek();
        if (c == '{') return object();
        if (c == '[') return array();
        if (c == '"') return Value{string()};
        if (s_.compare(i_, 4, "true") == 0) { i_ += 4; return Value{true}; }
        if (s_.compare(i_, 5, "false") == 0) { i_ += 5; return Value{false}; }
        if (s_.compare(i_, 4, "null") == 0) { i_ += 4; return Value{nullptr}; }
        return Value{number()};
    }
    Value object() {
        expect('{');
        Object o;
        if (peek() == '}') { ++i_; return Value{std::move(o)}; }
        for (;;) {
            std::string k = string();
            expect(':');
            o.emplace(std::move(k), value());
            if (peek() == ',') { ++i_; continue; }
            expect('}');
            return Value{std::move(o)};
        }
    }
    Value array() {
        expect('[');
        std::vector<Value> a;
        if (peek() == ']') { ++i_; return Value{std::move(a)}; }
        for (;;) {
            a.push_back(value());
            if (peek() == ',') { ++i_; continue; }
            expect(']');
            return Value{std::move(a)};
        }
    }
    std::string string() {
        expect('"');
        std::string o;
        while (i_ < s_.size() && s_[i_] != '"') {
            if (s_[i_] == '\\') {
                if (++i_ >= s_.size()) fail("bad escape");
                const char e = s_[i_];
                o += e == 'n' ? '\n' : e == 't' ? '\t' : e;  // the schema's strings are plain ASCII
            } else {
                o += s_[i_];
            }
            ++i_;
        }
        if (i_ >= s_.size()) fail("unterminated string");
        ++i_;
        return o;
    }
    double number() {
        const char* b = s_.c_str() + i_;
        char* e = nullptr;
        const double d = std::strtod(b, &e);
        if (e == b) fail("bad number");
        i_ += static_cast<std::size_t>(e - b);
        return d;
    }
    const std::string& s_;
    std::size_t i_ = 0;
};

inline TemplateKind template_kind_from_string(const std::string& s) {  // io.hpp:281-286
    if (s == "mi_chain") return TemplateKind::MiChain;
    if (s == "ci_mi") return TemplateKind::CiMi;
    if (s == "ci_ci") return TemplateKind::CiCi;
    throw invalid_parameter("unknown template kind: " + s);
}

inline Setting setting_from(const Value& j) {  // io.hpp:288-297 (absent fields read as 0)
    Setting s;
    s.kind = template_kind_from_string(j.at("kind").str());
    auto opt = [&](const char* k) { return j.has(k) ? static_cast<int>(j.at(k).number()) : 0; };
    s.chunk_size = opt("chunk_size");
    s.tile_m = opt("tile_m");
    s.tile_n = opt("tile_n");
    s.tile_k = opt("tile_k");
    s.stage_depth = opt("stage_depth");
    return s;
}

}  // namespace io_detail

// append_cache_file (io.hpp:407-427): the session's new entries, then mark them persisted
inline void append_cache_file(const std::string& path, const std::string& ctx, TuningCache& cache) {
    std::ofstream f(path, std::ios::app);
    if (!f) throw io_error("cannot open cache file for append: " + path);
    using io_detail::num;
    using io_detail::quote;
    for (const auto& e : cache.session_entries())
        f << "{\"begin\":" << e.seg.begin << ",\"code\":" << quote(e.code) << ",\"ctx\":" << quote(ctx)
          << ",\"dur\":" << num(e.duration) << ",\"end\":" << e.seg.end
          << ",\"setting\":" << io_detail::setting_json(e.setting) << ",\"type\":\"seg\"}\n";
    for (const auto& [code, key, dur] : cache.session_e2e())
        f << "{\"code\":" << quote(code) << ",\"ctx\":" << quote(ctx) << ",\"dur\":" << num(dur)
          << ",\"key\":" << quote(key) << ",\"type\":\"e2e\"}\n";
    if (!f) throw io_error("cache file write failed: " + path);
    cache.mark_persisted();
}

// load_cache_file (io.hpp:431-458): the entries of one context; a missing file loads nothing;
// loaded entries count as pre-warmed, not session-new
inline TuningCache load_cache_file(const std::string& path, const std::string& ctx) {
    TuningCache cache;
    std::ifstream f(path);
    if (!f) return cache;
    std::string line;
    while (std::getline(f, line)) {
        if (line.find_first_not_of(" \t\r") == std::string::npos) continue;
        const io_detail::Value j = io_detail::Parser(line).parse();
        if (!j.has("ctx") || j.at("ctx").str() != ctx) continue;
        if (j.at("type").str() == "seg") {
            cache.put(j.at("code").str(),
                      {static_cast<int>(j.at("begin").number()), static_cast<int>(j.at("end").number())},
                      io_detail::setting_from(j.at("setting")), j.at("dur").number());
        } else {
            cache.put_e2e(j.at("code").str(), j.at("key").str(), j.at("dur").number());
        }
    }
    cache.mark_persisted();
    return cache;
}

}  // namespace sparsefuse
