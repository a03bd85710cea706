// TEST INFRASTRUCTURE — not product code.  C-ABI shim over the *reference*
// lightplan sources (compiled in place from /root/reference/proj/src by
// oracle/Makefile, namespace renamed to lightplan_ref with
// -Dlightplan=lightplan_ref).  Exposes the same entry points as include/mlt.h
// with a ref_ prefix so tests/test_plan_parity.py and
// tests/test_schedule_parity.py can compare the B200 build against the
// reference itself on identical inputs.
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
#include "event_oracle.hpp"
#include "search_reference.hpp"
#include "batch_reference.hpp"
#include <stdexcept>
#include "latency_oracle.hpp"
#include "../paper_2411_11217_b200/csrc/capi/status.hpp"

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
#define LP_FN(x) ref_##x
#include "../paper_2411_11217_b200/csrc/capi/plan_glue.inc"

extern "C" {

const char* ref_last_error(void) { return mlt::last_error(); }
int ref_last_status(void) { return mlt::last_status(); }

// tests/support/latency_oracle.cpp:8-57 — the reference's independent
// spreadsheet recomputation. out = {comm, t_attn_c, t_ffn_c, t_gpu, t_layer}.
int ref_oracle_layer_latency(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                             const mlt_policy_t* p, double ctx, double out[5]) {
    return guard([&] {
        const auto o = lightplan::testing::oracle_layer_latency(glue::hw_in(hw), glue::model_in(model),
                                                                glue::policy_in(p), ctx);
        out[0] = o.comm; out[1] = o.t_attn_c; out[2] = o.t_ffn_c; out[3] = o.t_gpu; out[4] = o.t_layer;
        return MLT_OK;
    });
}

// tests/support/event_oracle.cpp:9-58 — second event simulator.
int ref_replay_simulate(const mlt_dag* d, mlt_timeline_entry_t* entries, double* makespan,
                        double busy[5]) {
    return guard([&] {
        const auto& dag = *reinterpret_cast<const lightplan::sim::ScheduleDag*>(d);
        const auto tl = lightplan::testing::replay_simulate(dag);
        for (size_t i = 0; i < tl.entries.size(); ++i)
            entries[i] = {tl.entries[i].task, tl.entries[i].start, tl.entries[i].end};
        *makespan = tl.makespan;
        for (int r = 0; r < 5; ++r) busy[r] = tl.busy[r];
        return MLT_OK;
    });
}

// tests/support/search_reference.cpp — serial unpruned enumeration of the
// grid.  Returns 1 with the winner in *policy/*objective, 0 when nothing fits.
int ref_brute_force_search(const mlt_hardware_spec_t* hw, const mlt_model_spec_t* model,
                           const mlt_workload_spec_t* w, const mlt_search_grid_t* grid,
                           mlt_policy_t* policy, double* objective) {
    return guard([&] {
        const auto r = lightplan::testing::brute_force_search(glue::hw_in(hw), glue::model_in(model),
                                                              glue::work_in(w), glue::grid_in(grid));
        if (!r) return 0;
        *policy = glue::policy_out(r->policy);
        *objective = r->objective;
        return 1;
    });
}

// tests/support/batch_reference.cpp — literal replay of Algorithm 2 (no
// flushing).  Same output convention as ref_batch_requests.
int ref_replay_batching(const char* const* ids, const int64_t* input_len, int32_t n,
                        const mlt_batch_params_t* p, int32_t* out_batch, int32_t* out_slot) {
    return guard([&] {
        std::vector<lightplan::Request> q;
        for (int i = 0; i < n; ++i) q.push_back({ids[i], input_len[i]});
        const auto plan = lightplan::testing::replay_batching(q, p->n_ub, p->ubs, p->gen_len, p->cache_size);
        for (int i = 0; i < n; ++i) out_batch[i] = -2, out_slot[i] = -1;
        auto index_of = [&](const std::string& id) {
            for (int i = 0; i < n; ++i)
                if (id == ids[i]) return i;
            throw std::runtime_error("replay returned an unknown id");
        };
        for (size_t b = 0; b < plan.micro_batches.size(); ++b)
            for (size_t s = 0; s < plan.micro_batches[b].size(); ++s) {
                const int i = index_of(plan.micro_batches[b][s].id);
                out_batch[i] = static_cast<int32_t>(b);
                out_slot[i] = static_cast<int32_t>(s);
            }
        for (size_t a = 0; a < plan.aborted.size(); ++a) {
            const int i = index_of(plan.aborted[a].id);
            out_batch[i] = -1;
            out_slot[i] = static_cast<int32_t>(a);
        }
        return static_cast<int>(plan.micro_batches.size());
    });
}

}  // extern "C"
