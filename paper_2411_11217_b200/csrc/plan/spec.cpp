// Spec validation.  Invariants follow proj/src/config.cpp:42-122 (positivity,
// n_q % n_kv, h1 % n_q, k <= n_e, N % mu, r_w/r_c ranges, r_c = 0 without
// A_g, p_g >= p_c, b_g >= b_c); field labels use the reference's INI keys so
// messages read the same.
#include <cmath>
#include <sstream>

#include "lightplan/config.hpp"

namespace lightplan {

const char* to_string(IssueCode code) {
    static const char* const names[] = {"NonPositiveField", "DivisibilityViolation",
                                        "PolicyInconsistency", "RangeViolation",
                                        "OrderingViolation"};
    const int i = static_cast<int>(code);
    return (i >= 0 && i < 5) ? names[i] : "UnknownIssue";
}

namespace {

struct IssueList {
    std::vector<ValidationIssue> v;
    void add(IssueCode c, const char* field, std::string msg) { v.push_back({c, field, std::move(msg)}); }
    void positive(double x, const char* field) {
        if (!(x > 0) || !std::isfinite(x)) add(IssueCode::NonPositiveField, field, std::string(field) + " must be strictly positive");
    }
    void positive(std::int64_t x, const char* field) {
        if (x <= 0) add(IssueCode::NonPositiveField, field, std::string(field) + " must be strictly positive");
    }
};

}  // namespace

std::vector<ValidationIssue> validate(const HardwareSpec& hw) {
    IssueList out;
    const std::pair<double, const char*> fields[] = {
        {hw.gpu_mem_bytes, "hardware.m_g"}, {hw.cpu_mem_bytes, "hardware.m_c"},
        {hw.gpu_bw, "hardware.b_g"},        {hw.cpu_bw, "hardware.b_c"},
        {hw.link_bw, "hardware.b_cg"},      {hw.gpu_flops, "hardware.p_g"},
        {hw.cpu_flops, "hardware.p_c"}};
    for (const auto& [value, name] : fields) out.positive(value, name);
    if (!out.v.empty()) return out.v;
    if (hw.gpu_flops < hw.cpu_flops)
        out.add(IssueCode::OrderingViolation, "hardware.p_g",
                "p_g must be >= p_c (GPU sits above CPU in the hierarchy)");
    if (hw.gpu_bw < hw.cpu_bw)
        out.add(IssueCode::OrderingViolation, "hardware.b_g",
                "b_g must be >= b_c (GPU sits above CPU in the hierarchy)");
    return out.v;
}

std::vector<ValidationIssue> validate(const ModelSpec& m) {
    IssueList out;
    const std::pair<std::int64_t, const char*> ints[] = {
        {m.layers, "model.l"},     {m.hidden_dim, "model.h1"}, {m.ffn_dim, "model.h2"},
        {m.q_heads, "model.n_q"},  {m.kv_heads, "model.n_kv"}, {m.experts, "model.n_e"},
        {m.top_k, "model.k"}};
    for (const auto& [value, name] : ints) out.positive(value, name);
    out.positive(m.weight_dtype_bytes, "model.dt_w");
    out.positive(m.kv_dtype_bytes, "model.dt_kv");
    if (!out.v.empty()) return out.v;
    if (m.q_heads % m.kv_heads != 0)
        out.add(IssueCode::DivisibilityViolation, "model.n_q", "n_q must be divisible by n_kv");
    if (m.hidden_dim % m.q_heads != 0)
        out.add(IssueCode::DivisibilityViolation, "model.h1", "h1 must be divisible by n_q");
    if (m.top_k > m.experts)
        out.add(IssueCode::RangeViolation, "model.k", "k must satisfy 1 <= k <= n_e");
    return out.v;
}

std::vector<ValidationIssue> validate(const WorkloadSpec& w) {
    IssueList out;
    out.positive(w.prompt_len, "workload.s");
    out.positive(w.gen_len, "workload.n");
    return out.v;
}

std::vector<ValidationIssue> validate(const Policy& p) {
    IssueList out;
    out.positive(p.micro_batch, "policy.mu");
    out.positive(p.batch, "policy.N");
    if (!out.v.empty()) return out.v;
    if (p.batch < p.micro_batch)
        out.add(IssueCode::RangeViolation, "policy.N", "N must be >= mu");
    else if (p.batch % p.micro_batch != 0)
        out.add(IssueCode::DivisibilityViolation, "policy.N", "N must be divisible by mu");
    if (!(p.weights_on_gpu >= 0.0 && p.weights_on_gpu <= 1.0))
        out.add(IssueCode::RangeViolation, "policy.r_w", "r_w must lie in [0,1]");
    if (!(p.kv_on_gpu >= 0.0 && p.kv_on_gpu <= 1.0))
        out.add(IssueCode::RangeViolation, "policy.r_c", "r_c must lie in [0,1]");
    if (!p.attn_on_gpu && p.kv_on_gpu > 0.0)
        out.add(IssueCode::PolicyInconsistency, "policy.r_c",
                "r_c must be 0 when A_g = 0 (CPU attention keeps all KV on CPU)");
    return out.v;
}

std::string format_issues(const std::vector<ValidationIssue>& issues) {
    std::ostringstream s;
    const char* sep = "";
    for (const auto& i : issues) {
        s << sep << to_string(i.code) << ": " << i.message;
        sep = "; ";
    }
    return s.str();
}

}  // namespace lightplan
