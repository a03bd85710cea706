// lightplan/runtime.hpp — the B200 build's additions to the reference C++ API
// (SURVEY.md §8(b)): the decode step is EXECUTED instead of simulated.
//
//   * lightplan::Runtime — one GPU's decode engine (budget-capped HBM arena,
//     paged weight pool fed over PCIe, host KV + host-core attention or the
//     paged GPU KV cache, the sm_100a kernels).  Wraps mlt::Runtime, the same
//     engine the C ABI (include/mlt.h, mlt_runtime_*) exposes.
//   * sim::execute(dag, rt, ...) — runs a build_schedule DAG (pipesim.hpp,
//     reference pipesim.cpp:294-348) on the runtime's resources and returns
//     the MEASURED Timeline, in place of sim::simulate (reference
//     pipesim.hpp:114); metrics()/verify_timeline() accept it unchanged.
//   * decode_layer(rt, ...) — a measured LatencyBreakdown per layer, the
//     executed counterpart of layer_latency (reference planner.hpp:43-44).
//
// Errors are the reference's exception types (UnsupportedCombinationError for
// a placement the engine cannot run, CycleDetectedError, std::invalid_argument
// for a DAG that does not match the runtime), plus std::runtime_error for
// CUDA failures and budget overflow.
#pragma once

#include <cstdint>
#include <memory>

#include "lightplan/config.hpp"
#include "lightplan/pipesim.hpp"
#include "lightplan/planner.hpp"

namespace mlt {
class Runtime;
}

namespace lightplan {

// Build-only knobs of the engine (everything else comes from ModelSpec/Policy).
struct RuntimeConfig {
    int device = 0;
    double budget_bytes = 16e9;  // every device allocation of the engine (weights, pool, KV, activations)
    int max_ctx = 0;             // KV capacity per sequence (>= prompt + generated)
    int vocab = 32000;
    std::uint64_t seed = 1234;   // synthetic weights (counter PRNG)
    bool weight_codec = false;   // lossless encoded weight tiles (fewer PCIe bytes)
    int host_threads = 0;        // host attention threads (0: all cores but the launchers)
};

class Runtime {
  public:
    Runtime(const ModelSpec& model, const Policy& policy, const RuntimeConfig& config);
    ~Runtime();
    Runtime(const Runtime&) = delete;
    Runtime& operator=(const Runtime&) = delete;

    // Synthetic prompt-stage KV for positions [0, prompt_len) of every sequence.
    void prefill_synthetic(int prompt_len, std::uint64_t seed);
    // The build_schedule DAG this engine runs for `steps` decode steps
    // (CGOPipe when A_g = 0, S4 when A_g = 1).
    sim::ScheduleDag schedule(int steps) const;
    mlt::Runtime& engine() { return *rt_; }

  private:
    std::unique_ptr<mlt::Runtime> rt_;
};

namespace sim {
// Executes `dag` on `rt`: tokens = the N step-0 ids, ids_out = [steps][N]
// greedy ids (steps = the DAG's step count), forced = optional [steps][N]
// teacher-forced ids.  Returns the measured Timeline (device clock);
// `measured` (optional) receives the graph as executed — the DAG (with the
// data-exact weight gates) carrying the measured task
// durations — which metrics() / verify_timeline() take with the timeline.
Timeline execute(const ScheduleDag& dag, Runtime& rt, const std::int32_t* tokens, std::int32_t* ids_out,
                 const std::int32_t* forced = nullptr, ScheduleDag* measured = nullptr);
}  // namespace sim

// Runs `steps` decode steps and returns the measured per-layer breakdown
// (link_upload, gpu_attention, gpu_ffn, cpu_attention; layer_total = the
// steady inter-layer time of the measured timeline).
LatencyBreakdown decode_layer(Runtime& rt, const std::int32_t* tokens, int steps, std::int32_t* ids_out);

}  // namespace lightplan
