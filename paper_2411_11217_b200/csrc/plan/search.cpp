// Policy search over (N, mu, A_g, F_g, r_w, r_c): the planner's optimiser,
// run on the measured B200 HardwareSpec to choose the policy the executor
// runs (closes the plan -> execute loop).  Restates
// proj/src/planner.cpp:164-341: exhaustive over the grid with memory
// pruning, OpenMP-parallel, reduced under the plan_preferred total order so
// the winner does not depend on the thread count; results are bit-identical
// to the reference (tests/test_plan_parity.py).
#include <algorithm>
#include <cmath>
#include <limits>
#include <sstream>
#include <tuple>

#include "lightplan/planner.hpp"

namespace lightplan {

// planner.cpp:21-64 evaluated without the feasibility check (the search
// prunes on memory_footprint itself).
LatencyBreakdown layer_latency_model(const HardwareSpec& hw, const ModelSpec& m, const Policy& p,
                                     double ctx);

SearchGrid SearchGrid::defaults() {
    SearchGrid g;
    std::vector<std::int64_t> mu;
    for (std::int64_t v = 1; v <= 1024; v *= 2) mu.push_back(v);
    for (std::int64_t v = 4; v <= 256; v += 4) mu.push_back(v);
    std::sort(mu.begin(), mu.end());
    mu.erase(std::unique(mu.begin(), mu.end()), mu.end());
    g.micro_batch_values = mu;
    for (std::int64_t n = 1; n <= 32; ++n) g.micro_batch_counts.push_back(n);
    for (int i = 0; i <= 20; ++i) {
        g.weight_ratio_values.push_back(static_cast<double>(i) * 0.05);
        g.kv_ratio_values.push_back(static_cast<double>(i) * 0.05);
    }
    g.attn_on_gpu_values = {false, true};
    g.ffn_on_gpu_values = {false, true};
    return g;
}

std::size_t SearchGrid::candidate_count() const {
    std::size_t kv = 0;
    for (bool a : attn_on_gpu_values) kv += a ? kv_ratio_values.size() : 1;
    return micro_batch_values.size() * micro_batch_counts.size() * weight_ratio_values.size() *
           ffn_on_gpu_values.size() * kv;
}

double steady_context(const WorkloadSpec& w, const SearchOptions& o) {
    if (o.ctx_override > 0) return o.ctx_override;
    return static_cast<double>(w.prompt_len) + static_cast<double>(w.gen_len) / 2.0;
}

bool plan_preferred(double oa, double ca, const Policy& a, double ob, double cb, const Policy& b) {
    const auto key = [](double o, double c, const Policy& p) {
        return std::make_tuple(o, c, p.batch, p.micro_batch, static_cast<int>(p.attn_on_gpu),
                               static_cast<int>(p.ffn_on_gpu), p.weights_on_gpu, p.kv_on_gpu);
    };
    return key(oa, ca, a) < key(ob, cb, b);
}

namespace {

struct Best {
    bool valid = false;
    Policy policy;
    double objective = std::numeric_limits<double>::infinity();
    double cpu_bytes = std::numeric_limits<double>::infinity();
    void offer(const Policy& p, double obj, double cpu) {
        if (!valid || plan_preferred(obj, cpu, p, objective, cpu_bytes, policy)) {
            valid = true;
            policy = p;
            objective = obj;
            cpu_bytes = cpu;
        }
    }
};

// Closest-to-fitting infeasible candidate, for the error message.
struct Miss {
    double overflow = std::numeric_limits<double>::infinity();
    bool gpu = true;
    double need = 0, have = 0;
    void offer(const Miss& m) {
        const auto key = [](const Miss& x) { return std::make_tuple(x.overflow, x.gpu ? 0 : 1, x.need); };
        if (key(m) < key(*this)) *this = m;
    }
};

}  // namespace

PlanResult search_policy(const HardwareSpec& hw, const ModelSpec& model, const WorkloadSpec& workload,
                         const SearchGrid& grid, const SearchOptions& options) {
    if (grid.micro_batch_values.empty() || grid.micro_batch_counts.empty() ||
        grid.weight_ratio_values.empty() || grid.attn_on_gpu_values.empty() ||
        grid.ffn_on_gpu_values.empty())
        throw std::invalid_argument("search grid must be non-empty in every dimension");

    std::vector<std::pair<bool, double>> placements;  // (A_g, r_c); r_c searched only with A_g
    for (bool a : grid.attn_on_gpu_values) {
        if (a)
            for (double rc : grid.kv_ratio_values) placements.push_back({true, rc});
        else
            placements.push_back({false, 0.0});
    }
    const std::int64_t n_rw = static_cast<std::int64_t>(grid.weight_ratio_values.size());
    const std::int64_t n_ffn = static_cast<std::int64_t>(grid.ffn_on_gpu_values.size());
    const std::int64_t n_pl = static_cast<std::int64_t>(placements.size());
    const std::int64_t n_mu = static_cast<std::int64_t>(grid.micro_batch_values.size());
    const std::int64_t n_cnt = static_cast<std::int64_t>(grid.micro_batch_counts.size());
    const std::int64_t total = n_rw * n_ffn * n_pl * n_mu * n_cnt;
    const double ctx = steady_context(workload, options);

    Best best;
    Miss miss;
#pragma omp parallel
    {
        Best mine;
        Miss my_miss;
#pragma omp for schedule(static) nowait
        for (std::int64_t i = 0; i < total; ++i) {
            std::int64_t r = i;
            Policy p;
            p.weights_on_gpu = grid.weight_ratio_values[r % n_rw];
            r /= n_rw;
            p.ffn_on_gpu = grid.ffn_on_gpu_values[r % n_ffn];
            r /= n_ffn;
            p.attn_on_gpu = placements[r % n_pl].first;
            p.kv_on_gpu = placements[r % n_pl].second;
            r /= n_pl;
            p.micro_batch = grid.micro_batch_values[r % n_mu];
            p.batch = p.micro_batch * grid.micro_batch_counts[r / n_mu];
            const MemoryFootprint f = memory_footprint(hw, model, workload, p);
            if (!f.feasible) {
                const double og = f.gpu_bytes - hw.gpu_mem_bytes, oc = f.cpu_bytes - hw.cpu_mem_bytes;
                my_miss.offer(og >= oc ? Miss{og, true, f.gpu_bytes, hw.gpu_mem_bytes}
                                       : Miss{oc, false, f.cpu_bytes, hw.cpu_mem_bytes});
                continue;
            }
            const double t = layer_latency_model(hw, model, p, ctx).layer_total;
            mine.offer(p, options.objective == SearchObjective::TokensPerSecond ? t / static_cast<double>(p.batch) : t,
                       f.cpu_bytes);
        }
#pragma omp critical(mlt_search_merge)
        {
            if (mine.valid) best.offer(mine.policy, mine.objective, mine.cpu_bytes);
            miss.offer(my_miss);
        }
    }
    if (!best.valid) {
        std::ostringstream msg;
        msg << "no feasible policy in the grid; tightest violated constraint: " << (miss.gpu ? "gpu" : "cpu")
            << " memory needs " << miss.need << " bytes of " << miss.have << " available";
        throw NoFeasiblePolicyError(msg.str());
    }
    PlanResult res = estimate_throughput(hw, model, workload, best.policy);
    res.breakdown = layer_latency(hw, model, workload, best.policy, ctx);
    res.objective = best.objective;
    return res;
}

}  // namespace lightplan
