// INI config surface of the planner (include/lightplan/config.hpp; grammar
// and diagnostics of the reference parser, proj/src/config.cpp:148-426):
// the files the reference's `plan` / `sweep` commands read
// (cli.cpp:262-292) drive the B200 plan -> execute loop
// (paper_2411_11217_b200/cli.py).
#include <algorithm>
#include <array>
#include <cctype>
#include <charconv>
#include <cmath>
#include <fstream>
#include <sstream>
#include <string_view>
#include <unordered_map>

#include "lightplan/config.hpp"

namespace lightplan {

namespace {

// How a value's text is read: which unit suffixes it accepts, and whether it
// must be an integer count or a 0/1 flag.
enum class Kind { Bytes, Rate, Flops, Count, Real, Flag };

struct Field {
    std::string_view section, key;
    Kind kind;
};

// Table order = the order "missing key" is reported in (config.cpp:165-190).
constexpr std::array<Field, 24> kFields{{
    {"hardware", "m_g", Kind::Bytes},  {"hardware", "m_c", Kind::Bytes},  {"hardware", "b_g", Kind::Rate},
    {"hardware", "b_c", Kind::Rate},   {"hardware", "b_cg", Kind::Rate},  {"hardware", "p_g", Kind::Flops},
    {"hardware", "p_c", Kind::Flops},  {"model", "l", Kind::Count},       {"model", "h1", Kind::Count},
    {"model", "h2", Kind::Count},      {"model", "n_q", Kind::Count},     {"model", "n_kv", Kind::Count},
    {"model", "n_e", Kind::Count},     {"model", "k", Kind::Count},       {"model", "dt_w", Kind::Real},
    {"model", "dt_kv", Kind::Real},    {"workload", "s", Kind::Count},    {"workload", "n", Kind::Count},
    {"policy", "N", Kind::Count},      {"policy", "mu", Kind::Count},     {"policy", "A_g", Kind::Flag},
    {"policy", "F_g", Kind::Flag},     {"policy", "r_w", Kind::Real},     {"policy", "r_c", Kind::Real},
}};

std::string_view strip(std::string_view s) {
    const auto ws = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
    while (!s.empty() && ws(s.front())) s.remove_prefix(1);
    while (!s.empty() && ws(s.back())) s.remove_suffix(1);
    return s;
}

// Case-insensitive suffix test; the suffix must leave at least one character.
bool cut_suffix(std::string_view& body, std::string_view suffix) {
    if (body.size() <= suffix.size()) return false;
    const std::string_view tail = body.substr(body.size() - suffix.size());
    for (size_t i = 0; i < suffix.size(); ++i)
        if (std::toupper(static_cast<unsigned char>(tail[i])) != suffix[i]) return false;
    body.remove_suffix(suffix.size());
    return true;
}

bool read_number(std::string_view text, Kind kind, double& out) {
    std::string_view body = text;
    double mult = 1.0;
    if (kind == Kind::Flops) {
        if (cut_suffix(body, "TFLOPS")) mult = 1e12;
        else if (cut_suffix(body, "GFLOPS")) mult = 1e9;
    } else if (kind == Kind::Bytes || kind == Kind::Rate) {
        static constexpr std::pair<std::string_view, double> kSi[] = {{"K", 1e3}, {"M", 1e6}, {"G", 1e9}, {"T", 1e12}};
        for (const auto& [suf, m] : kSi)
            if (cut_suffix(body, suf)) {
                mult = m;
                break;
            }
    }
    body = strip(body);
    double v = 0.0;
    const auto [end, ec] = std::from_chars(body.data(), body.data() + body.size(), v);
    if (ec != std::errc{} || end != body.data() + body.size()) return false;
    out = v * mult;
    return true;
}

// Store `v` into the field; "" on success, else the diagnostic.
std::string store(ParsedConfig& c, const Field& f, double v) {
    const std::string key(f.key);
    int64_t count = 0;
    bool flag = false;
    if (f.kind == Kind::Count) {
        if (v != std::floor(v)) return key + " must be an integer";
        count = static_cast<int64_t>(v);
    } else if (f.kind == Kind::Flag) {
        if (v != 0.0 && v != 1.0) return key + " must be 0 or 1";
        flag = v != 0.0;
    }
    HardwareSpec& h = c.hardware;
    ModelSpec& m = c.model;
    const std::unordered_map<std::string, double*> reals = {
        {"hardware.m_g", &h.gpu_mem_bytes}, {"hardware.m_c", &h.cpu_mem_bytes}, {"hardware.b_g", &h.gpu_bw},
        {"hardware.b_c", &h.cpu_bw},        {"hardware.b_cg", &h.link_bw},      {"hardware.p_g", &h.gpu_flops},
        {"hardware.p_c", &h.cpu_flops},     {"model.dt_w", &m.weight_dtype_bytes},
        {"model.dt_kv", &m.kv_dtype_bytes}};
    const std::string dotted = std::string(f.section) + "." + key;
    if (auto it = reals.find(dotted); it != reals.end()) {
        *it->second = v;
        return "";
    }
    const std::unordered_map<std::string, int64_t*> counts = {
        {"model.l", &m.layers},       {"model.h1", &m.hidden_dim}, {"model.h2", &m.ffn_dim},
        {"model.n_q", &m.q_heads},    {"model.n_kv", &m.kv_heads}, {"model.n_e", &m.experts},
        {"model.k", &m.top_k},        {"workload.s", &c.workload.prompt_len},
        {"workload.n", &c.workload.gen_len}};
    if (auto it = counts.find(dotted); it != counts.end()) {
        *it->second = count;
        return "";
    }
    Policy& p = *c.policy;
    if (dotted == "policy.N") p.batch = count;
    else if (dotted == "policy.mu") p.micro_batch = count;
    else if (dotted == "policy.A_g") p.attn_on_gpu = flag;
    else if (dotted == "policy.F_g") p.ffn_on_gpu = flag;
    else if (dotted == "policy.r_w") p.weights_on_gpu = v;
    else if (dotted == "policy.r_c") p.kv_on_gpu = v;
    return "";
}

bool known_section(std::string_view s) {
    return std::any_of(kFields.begin(), kFields.end(), [&](const Field& f) { return f.section == s; });
}

}  // namespace

ConfigResult parse_config_text(const std::string& text) {
    ConfigResult res;
    ParsedConfig cfg;
    auto error = [&](int line, std::string msg) {
        res.parse_error = ConfigParseError{line, std::move(msg)};
        return res;
    };
    std::unordered_map<std::string, int> first_line;  // "section.key" -> line
    bool seen_hw = false, seen_model = false, seen_work = false;
    std::string section;
    std::istringstream lines(text);
    std::string raw;
    for (int no = 1; std::getline(lines, raw); ++no) {
        std::string_view line(raw);
        if (const size_t hash = line.find('#'); hash != std::string_view::npos) line = line.substr(0, hash);
        line = strip(line);
        if (line.empty()) continue;
        if (line.front() == '[') {
            if (line.back() != ']') return error(no, "unterminated section header");
            section = std::string(strip(line.substr(1, line.size() - 2)));
            if (!known_section(section)) return error(no, "unknown section [" + section + "]");
            seen_hw |= section == "hardware";
            seen_model |= section == "model";
            seen_work |= section == "workload";
            if (section == "policy" && !cfg.policy) cfg.policy.emplace();
            continue;
        }
        const size_t eq = line.find('=');
        if (eq == std::string_view::npos) return error(no, "expected `key = value`");
        const std::string key(strip(line.substr(0, eq)));
        const std::string_view value = strip(line.substr(eq + 1));
        if (section.empty()) return error(no, "key `" + key + "` outside any section");
        const auto f = std::find_if(kFields.begin(), kFields.end(),
                                    [&](const Field& x) { return x.section == section && x.key == key; });
        if (f == kFields.end()) return error(no, "unknown key `" + key + "` in section [" + section + "]");
        const std::string dotted = section + "." + key;
        if (auto it = first_line.find(dotted); it != first_line.end())
            return error(no, "duplicate key `" + key + "` (first set on line " + std::to_string(it->second) + ")");
        first_line.emplace(dotted, no);
        double v = 0.0;
        if (!read_number(value, f->kind, v)) return error(no, "cannot parse numeric value '" + std::string(value) + "'");
        if (std::string msg = store(cfg, *f, v); !msg.empty()) return error(no, msg);
    }
    if (!seen_hw) return error(0, "missing required section [hardware]");
    if (!seen_model) return error(0, "missing required section [model]");
    if (!seen_work) return error(0, "missing required section [workload]");
    for (const Field& f : kFields) {
        if (f.section == "policy" && !cfg.policy) continue;
        if (!first_line.count(std::string(f.section) + "." + std::string(f.key)))
            return error(0, "missing key `" + std::string(f.key) + "` in section [" + std::string(f.section) + "]");
    }
    auto add = [&](std::vector<ValidationIssue> v) {
        res.validation_issues.insert(res.validation_issues.end(), v.begin(), v.end());
    };
    add(validate(cfg.hardware));
    add(validate(cfg.model));
    add(validate(cfg.workload));
    if (cfg.policy) add(validate(*cfg.policy));
    if (res.validation_issues.empty()) res.config = std::move(cfg);
    return res;
}

ConfigResult parse_config_file(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) {
        ConfigResult res;
        res.parse_error = ConfigParseError{0, "cannot open config file: " + path};
        return res;
    }
    std::ostringstream text;
    text << in.rdbuf();
    return parse_config_text(text.str());
}

namespace {

std::string shortest(double v) {
    char buf[40];
    const auto r = std::to_chars(buf, buf + sizeof buf, v);
    return std::string(buf, r.ptr);
}

}  // namespace

std::string serialize_config(const ParsedConfig& c) {
    std::ostringstream o;
    auto line = [&](const char* k, const std::string& v) { o << k << " = " << v << "\n"; };
    const auto i = [](int64_t v) { return std::to_string(v); };
    o << "[hardware]\n";
    line("m_g", shortest(c.hardware.gpu_mem_bytes));
    line("m_c", shortest(c.hardware.cpu_mem_bytes));
    line("b_g", shortest(c.hardware.gpu_bw));
    line("b_c", shortest(c.hardware.cpu_bw));
    line("b_cg", shortest(c.hardware.link_bw));
    line("p_g", shortest(c.hardware.gpu_flops));
    line("p_c", shortest(c.hardware.cpu_flops));
    o << "\n[model]\n";
    line("l", i(c.model.layers));
    line("h1", i(c.model.hidden_dim));
    line("h2", i(c.model.ffn_dim));
    line("n_q", i(c.model.q_heads));
    line("n_kv", i(c.model.kv_heads));
    line("n_e", i(c.model.experts));
    line("k", i(c.model.top_k));
    line("dt_w", shortest(c.model.weight_dtype_bytes));
    line("dt_kv", shortest(c.model.kv_dtype_bytes));
    o << "\n[workload]\n";
    line("s", i(c.workload.prompt_len));
    line("n", i(c.workload.gen_len));
    if (c.policy) {
        const Policy& p = *c.policy;
        o << "\n[policy]\n";
        line("N", i(p.batch));
        line("mu", i(p.micro_batch));
        line("A_g", p.attn_on_gpu ? "1" : "0");
        line("F_g", p.ffn_on_gpu ? "1" : "0");
        line("r_w", shortest(p.weights_on_gpu));
        line("r_c", shortest(p.kv_on_gpu));
    }
    return o.str();
}

}  // namespace lightplan
