// Per-layer decode model (Eq. 13-15 of the paper), memory budget and TP
// rule.  Formulas restate proj/src/planner.cpp:17-162 with the same
// floating-point evaluation order so the B200 HRM bound printed by bench.py is
// the number the reference itself would print for the same spec.
#include "lightplan/planner.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

namespace lightplan {

namespace {

inline double d(std::int64_t v) { return static_cast<double>(v); }

// Roofline time of one operator at one device.
inline double roof(double bytes, double bw, double flops, double peak) {
    return std::max(bytes / bw, flops / peak);
}

LatencyBreakdown model_layer(const HardwareSpec& hw, const ModelSpec& m, const Policy& p,
                             double ctx) {
    const double N = d(p.batch);
    const double n_ub = d(p.micro_batch_count());
    const OpProfile attn = attention_decode_profile(m, N, ctx);
    const OpProfile ffn = moe_ffn_profile(m, N, p.weights_on_gpu);
    const ProjectionProfiles proj = projection_profiles(m, N);

    LatencyBreakdown b;
    // QKV before attention, O after: always on the GPU (planner.cpp:32-39).
    b.gpu_attention = roof(proj.qkv.gpu_bytes, hw.gpu_bw, proj.qkv.flops, hw.gpu_flops);
    b.gpu_ffn = roof(proj.output.gpu_bytes, hw.gpu_bw, proj.output.flops, hw.gpu_flops);
    if (p.attn_on_gpu)
        b.gpu_attention += roof(attn.gpu_bytes, hw.gpu_bw, attn.flops, hw.gpu_flops);
    else
        b.cpu_attention = roof(attn.cpu_bytes, hw.cpu_bw, attn.flops, hw.cpu_flops);
    if (p.ffn_on_gpu)
        b.gpu_ffn += roof(ffn.gpu_bytes, hw.gpu_bw, ffn.flops, hw.gpu_flops);
    else
        b.cpu_ffn = roof(ffn.cpu_bytes, hw.cpu_bw, ffn.flops, hw.cpu_flops);

    // Link: streamed weights + per-micro-batch KV (A_g) or all but the first
    // hidden upload (the first hides under the previous layer's stream).
    const TransferSizes t = transfer_sizes(m, p, ctx);
    double up = t.weight_stream;
    up += p.attn_on_gpu ? n_ub * t.kv_upload : (n_ub - 1.0) * t.hidden_upload;
    b.link_upload = up / hw.link_bw;
    b.layer_total = std::max({b.link_upload, b.cpu_total(), b.gpu_total()});
    return b;
}

double prefill_flops_per_layer(const ModelSpec& m, const Policy& p, const WorkloadSpec& w) {
    // planner.cpp:112-127: dense linears per prompt token + causal attention.
    const double h1 = d(m.hidden_dim), h2 = d(m.ffn_dim), dh = d(m.head_dim());
    const double s = d(w.prompt_len);
    const double per_token = 2.0 * h1 * d(m.q_heads + 2 * m.kv_heads) * dh + 2.0 * h1 * h1 +
                             d(m.top_k) * 6.0 * h1 * h2;
    const double causal = 4.0 * d(m.q_heads) * dh * s * (s + 1.0) / 2.0;
    return d(p.batch) * (s * per_token + causal);
}

}  // namespace

// Unchecked per-layer model, shared with the policy search (search.cpp).
LatencyBreakdown layer_latency_model(const HardwareSpec& hw, const ModelSpec& m, const Policy& p,
                                     double ctx) {
    return model_layer(hw, m, p, ctx);
}

MemoryFootprint memory_footprint(const HardwareSpec& hw, const ModelSpec& m,
                                 const WorkloadSpec& w, const Policy& p) {
    const MemoryTotals tot = memory_totals(m, w, p.batch);
    const double layer = layer_weight_bytes(m).total();
    const double streamed = 1.0 - p.weights_on_gpu;
    const double act = d(p.micro_batch) * d(m.hidden_dim + 2 * m.ffn_dim) * m.weight_dtype_bytes;
    MemoryFootprint f;
    // GPU: resident share + double buffer of two streamed layers + resident
    // KV + activation peak.  CPU: offloaded shares + pinned staging mirror.
    f.gpu_bytes = p.weights_on_gpu * tot.weight_bytes + 2.0 * streamed * layer +
                  p.kv_on_gpu * tot.kv_cache_bytes + act;
    f.cpu_bytes = streamed * tot.weight_bytes + (1.0 - p.kv_on_gpu) * tot.kv_cache_bytes +
                  2.0 * streamed * layer;
    f.feasible = f.gpu_bytes <= hw.gpu_mem_bytes && f.cpu_bytes <= hw.cpu_mem_bytes;
    return f;
}

LatencyBreakdown layer_latency(const HardwareSpec& hw, const ModelSpec& m, const WorkloadSpec& w,
                               const Policy& p, double ctx) {
    const MemoryFootprint f = memory_footprint(hw, m, w, p);
    if (!f.feasible)
        throw InfeasiblePolicyError("policy exceeds device memory (gpu " +
                                    std::to_string(f.gpu_bytes) + " / " +
                                    std::to_string(hw.gpu_mem_bytes) + ", cpu " +
                                    std::to_string(f.cpu_bytes) + " / " +
                                    std::to_string(hw.cpu_mem_bytes) + ")");
    return model_layer(hw, m, p, ctx);
}

HardwareSpec apply_tensor_parallelism(const HardwareSpec& hw, int tp) {
    if (tp < 1) throw std::invalid_argument("tensor-parallel degree must be >= 1");
    HardwareSpec s = hw;
    s.gpu_mem_bytes *= tp;
    s.gpu_bw *= tp;
    s.gpu_flops *= tp;
    return s;
}

HardwareSpec apply_tensor_parallelism_b200(const HardwareSpec& hw, int tp, double host_read_cap) {
    HardwareSpec s = apply_tensor_parallelism(hw, tp);
    s.link_bw = hw.link_bw * tp;
    if (host_read_cap > 0) s.link_bw = std::min(s.link_bw, host_read_cap);
    return s;
}

PlanResult estimate_throughput(const HardwareSpec& hw, const ModelSpec& m, const WorkloadSpec& w,
                               const Policy& p) {
    PlanResult r;
    r.policy = p;
    r.memory = memory_footprint(hw, m, w, p);
    if (!r.memory.feasible) throw InfeasiblePolicyError("policy exceeds device memory");

    const double L = d(m.layers);
    double decode = 0.0;
    for (std::int64_t step = 1; step <= w.gen_len; ++step)  // ctx grows one token per step
        decode += L * layer_latency(hw, m, w, p, d(w.prompt_len + step)).layer_total;

    const double stream = transfer_sizes(m, p, 1.0).weight_stream / hw.link_bw;
    const double compute = prefill_flops_per_layer(m, p, w) / hw.gpu_flops;
    const double prefill = L * std::max(stream, compute);

    const double generated = d(p.batch) * d(w.gen_len);
    r.decode_throughput = generated / decode;
    r.generation_throughput = generated / (prefill + decode);
    const double ctx_mid = d(w.prompt_len) + d(w.gen_len) / 2.0;
    r.breakdown = layer_latency(hw, m, w, p, ctx_mid);
    r.objective = r.breakdown.layer_total / d(p.batch);
    return r;
}

double nvlink_allreduce_seconds(const ModelSpec& m, const Policy& p, int tp, double nvlink_bw) {
    if (tp <= 1) return 0.0;
    if (nvlink_bw <= 0) throw std::invalid_argument("nvlink_bw must be > 0");
    const double size = d(p.micro_batch) * d(m.hidden_dim) * 4.0;  // fp32 [mu, h1]
    const double ring = 2.0 * (tp - 1.0) / tp;
    return d(p.micro_batch_count()) * 2.0 * ring * size / nvlink_bw;
}

PlanResult estimate_throughput_b200(const HardwareSpec& hw, const ModelSpec& m, const WorkloadSpec& w,
                                    const Policy& p, int tp, double nvlink_bw) {
    if (tp <= 1) return estimate_throughput(hw, m, w, p);
    const double t_nvl = nvlink_allreduce_seconds(m, p, tp, nvlink_bw);
    PlanResult r;
    r.policy = p;
    r.memory = memory_footprint(hw, m, w, p);
    if (!r.memory.feasible) throw InfeasiblePolicyError("policy exceeds device memory");
    auto layer = [&](double ctx) {
        LatencyBreakdown b = layer_latency(hw, m, w, p, ctx);
        b.gpu_ffn += t_nvl;
        b.layer_total = std::max({b.link_upload, b.cpu_total(), b.gpu_total()});
        return b;
    };
    const double L = d(m.layers);
    double decode = 0.0;
    for (std::int64_t step = 1; step <= w.gen_len; ++step) decode += L * layer(d(w.prompt_len + step)).layer_total;
    const double stream = transfer_sizes(m, p, 1.0).weight_stream / hw.link_bw;
    const double compute = prefill_flops_per_layer(m, p, w) / hw.gpu_flops;
    const double prefill = L * std::max(stream, compute);
    const double generated = d(p.batch) * d(w.gen_len);
    r.decode_throughput = generated / decode;
    r.generation_throughput = generated / (prefill + decode);
    r.breakdown = layer(d(w.prompt_len) + d(w.gen_len) / 2.0);
    r.objective = r.breakdown.layer_total / d(p.batch);
    return r;
}

}  // namespace lightplan
