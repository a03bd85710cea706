// C ABI over the B200 build's lightplan planner + scheduler (include/mlt.h).
#include <cstring>
#include <string>
#include <vector>

#include "lightplan/config.hpp"
#include "lightplan/opcost.hpp"
#include "lightplan/hrm.hpp"
#include "lightplan/pipesim.hpp"
#include "lightplan/planner.hpp"
#include "lightplan/batcher.hpp"
#include <algorithm>
#include "status.hpp"

namespace mlt {
namespace {
thread_local std::string g_error;
thread_local int g_status = 0;
}
void set_error(const char* msg, int code) { g_error = msg ? msg : ""; g_status = code; }
const char* last_error() { return g_error.c_str(); }
int last_status() { return g_status; }
}  // namespace mlt

namespace {
template <class F>
int guard(F&& f) {
    MLT_GUARD_BODY(lightplan)
}
}  // namespace

#define LP_NS lightplan
#define LP_FN(x) mlt_##x
#define LP_PRODUCT 1
#include "plan_glue.inc"

extern "C" {

const char* mlt_last_error(void) { return mlt::last_error(); }

int mlt_last_status(void) { return mlt::last_status(); }

const char* mlt_version(void) { return "mlt-b200 0.1 (sm_100a)"; }

int mlt_estimate_throughput_b200(const mlt_hardware_spec_t* tp_hw, const mlt_model_spec_t* model,
                                 const mlt_workload_spec_t* w, const mlt_policy_t* p, int tp,
                                 double nvlink_bw, mlt_plan_result_t* out) {
    return guard([&] {
        const auto r = lightplan::estimate_throughput_b200(glue::hw_in(tp_hw), glue::model_in(model),
                                                           glue::work_in(w), glue::policy_in(p), tp, nvlink_bw);
        out->policy = glue::policy_out(r.policy);
        out->breakdown = glue::lat_out(r.breakdown);
        out->memory = {r.memory.gpu_bytes, r.memory.cpu_bytes, r.memory.feasible ? 1 : 0};
        out->decode_throughput = r.decode_throughput;
        out->generation_throughput = r.generation_throughput;
        out->objective = r.objective;
        return MLT_OK;
    });
}

int mlt_validate(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                 const mlt_workload_spec_t* workload, const mlt_policy_t* policy, char* msg,
                 size_t cap) {
    return guard([&] {
        std::vector<lightplan::ValidationIssue> all;
        auto take = [&](std::vector<lightplan::ValidationIssue> v) {
            all.insert(all.end(), v.begin(), v.end());
        };
        if (hw) take(lightplan::validate(glue::hw_in(hw)));
        if (model) take(lightplan::validate(glue::model_in(model)));
        if (workload) take(lightplan::validate(glue::work_in(workload)));
        if (policy) take(lightplan::validate(glue::policy_in(policy)));
        glue::copy_out(lightplan::format_issues(all), msg, cap);
        return static_cast<int>(all.size());
    });
}

}  // extern "C"
