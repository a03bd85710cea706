// lightplan/runtime.hpp: the reference-style C++ API over mlt::Runtime.
#include "lightplan/runtime.hpp"

#include "runtime.hpp"

namespace lightplan {

Runtime::Runtime(const ModelSpec& model, const Policy& policy, const RuntimeConfig& c) {
    mlt::ModelExt ext;
    ext.vocab = c.vocab;
    ext.seed = c.seed;
    mlt::RuntimeOptions opt;
    opt.device = c.device;
    opt.budget_bytes = c.budget_bytes;
    opt.max_ctx = c.max_ctx;
    opt.weight_codec = c.weight_codec;
    opt.host_threads = c.host_threads;
    rt_ = std::make_unique<mlt::Runtime>(model, ext, policy, opt);
}

Runtime::~Runtime() = default;

void Runtime::prefill_synthetic(int prompt_len, std::uint64_t seed) { rt_->prefill_synthetic(prompt_len, seed); }

sim::ScheduleDag Runtime::schedule(int steps) const { return rt_->schedule(steps); }

namespace sim {
Timeline execute(const ScheduleDag& dag, Runtime& rt, const std::int32_t* tokens, std::int32_t* ids_out,
                 const std::int32_t* forced, ScheduleDag* measured) {
    Timeline tl;
    rt.engine().execute(dag, tokens, forced, ids_out, measured, &tl);
    return tl;
}
}  // namespace sim

LatencyBreakdown decode_layer(Runtime& rt, const std::int32_t* tokens, int steps, std::int32_t* ids_out) {
    return rt.engine().decode(tokens, nullptr, steps, ids_out).measured;
}

}  // namespace lightplan
