// A reference-API caller of the B200 engine: plain C++20
// against include/lightplan/*.hpp, linked with libmlt.so — no Python, no C
// ABI.  Builds the CGOPipe DAG with the reference's build_schedule, executes
// it on the GPU with sim::execute, checks the measured timeline with the
// reference's metrics()/verify_timeline(), runs decode_layer, and shows the
// error conventions.  Prints one JSON line (tests/test_cpp_api_gpu.py).
#include <cstdio>
#include <stdexcept>
#include <string>
#include <vector>

#include "lightplan/pipesim.hpp"
#include "lightplan/planner.hpp"
#include "lightplan/runtime.hpp"

using namespace lightplan;

int main(int argc, char** argv) {
    const bool gpu_attn = argc > 1 && std::string(argv[1]) == "gpu-attn";
    ModelSpec m;
    m.layers = 2; m.hidden_dim = 1024; m.ffn_dim = 3584; m.q_heads = 8; m.kv_heads = 2;
    m.experts = 8; m.top_k = 2; m.weight_dtype_bytes = 2; m.kv_dtype_bytes = 2;
    Policy p;
    p.batch = 8; p.micro_batch = 4; p.attn_on_gpu = gpu_attn; p.ffn_on_gpu = true;
    p.weights_on_gpu = gpu_attn ? 1.0 : 0.25; p.kv_on_gpu = gpu_attn ? 1.0 : 0.0;
    RuntimeConfig c;
    c.budget_bytes = 4e9;
    c.max_ctx = 64;
    Runtime rt(m, p, c);
    rt.prefill_synthetic(16, 9012);

    const int steps = 3;
    // the reference's own DAG builder, for this policy (pipesim.hpp build_schedule)
    HardwareSpec hw{4e9, 1e12, 6.5e12, 1.8e11, 5.5e10, 1.4e15, 2e12};
    WorkloadSpec w{16, steps};
    const sim::ScheduleKind kind = gpu_attn ? sim::ScheduleKind::S4 : sim::ScheduleKind::CgoPipe;
    const sim::ScheduleDag dag = sim::build_schedule(hw, m, w, p, kind, static_cast<int>(m.layers), steps);
    std::vector<std::int32_t> tok(8), ids(steps * 8);
    for (int i = 0; i < 8; ++i) tok[i] = 100 + 37 * i;
    sim::ScheduleDag measured;
    const sim::Timeline tl = sim::execute(dag, rt, tok.data(), ids.data(), nullptr, &measured);
    const sim::SimMetrics met = sim::metrics(measured, tl);
    const std::string bad = sim::verify_timeline_tol(measured, tl, 5e-5);

    std::vector<std::int32_t> ids2(steps * 8);
    const LatencyBreakdown lb = decode_layer(rt, ids.data() + (steps - 1) * 8, steps, ids2.data());

    // error conventions: a DAG for another layer count / placement
    std::string err_layers, err_kind;
    try {
        sim::execute(sim::build_schedule(hw, m, w, p, kind, 3, 1), rt, tok.data(), ids2.data());
    } catch (const std::invalid_argument& e) {
        err_layers = "invalid_argument";
    }
    try {
        Policy q = p;
        q.attn_on_gpu = !p.attn_on_gpu;
        q.kv_on_gpu = q.attn_on_gpu ? 1.0 : 0.0;
        q.weights_on_gpu = 1.0;
        sim::execute(sim::build_schedule(hw, m, w, q, gpu_attn ? sim::ScheduleKind::CgoPipe : sim::ScheduleKind::S4,
                                         static_cast<int>(m.layers), 1),
                     rt, tok.data(), ids2.data());
    } catch (const std::invalid_argument&) {
        err_kind = "invalid_argument";
    } catch (const sim::UnsupportedCombinationError&) {
        err_kind = "UnsupportedCombinationError";
    }

    std::printf("{\"tasks\": %zu, \"entries\": %zu, \"makespan\": %.6f, \"verify\": \"%s\", "
                "\"steady_layer_time\": %.6f, \"gpu_util\": %.4f, \"ids\": [",
                dag.tasks.size(), tl.entries.size(), tl.makespan, bad.c_str(), met.steady_layer_time,
                met.utilization[0]);
    for (size_t i = 0; i < ids.size(); ++i) std::printf("%s%d", i ? ", " : "", ids[i]);
    std::printf("], \"decode_layer\": {\"link_upload\": %.6g, \"gpu_attention\": %.6g, \"gpu_ffn\": %.6g, "
                "\"cpu_attention\": %.6g, \"layer_total\": %.6g}, \"err_layers\": \"%s\", \"err_kind\": \"%s\"}\n",
                lb.link_upload, lb.gpu_attention, lb.gpu_ffn, lb.cpu_attention, lb.layer_total, err_layers.c_str(),
                err_kind.c_str());
    return 0;
}
