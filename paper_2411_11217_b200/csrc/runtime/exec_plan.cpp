// GPU-free executor planning: catalog + residency, pages, exact gates,
// reuse edges (see exec_plan.hpp and executor.cpp's file comment).
#include "exec_plan.hpp"

#include "host_layout.hpp"
#include "lightplan/opcost.hpp"

namespace mlt {

using lightplan::sim::Resource;
using lightplan::sim::ScheduleDag;
using lightplan::sim::Task;
using lightplan::sim::TaskKind;

Catalog build_catalog(const lightplan::ModelSpec& m, const lightplan::Policy& p) {
    Catalog c;
    const int H = static_cast<int>(m.hidden_dim), F = static_cast<int>(m.ffn_dim);
    const int E = static_cast<int>(m.experts);
    const int W = static_cast<int>((m.q_heads + 2 * m.kv_heads) * m.head_dim());
    auto add = [&](int kind, int expert, int rows, int64_t K) {
        for (int rb = 0; rb < rows / 128; ++rb) c.blocks.push_back({kind, expert, rb, K, 128 * K * 2, false, 0});
    };
    add(kWqkv, 0, W, H);
    add(kWo, 0, H, H);
    for (int e = 0; e < E; ++e) {
        add(kW1, e, F, H);
        add(kW3, e, F, H);
        add(kW2, e, H, F);
    }
    const double layer_total = lightplan::layer_weight_bytes(m).total();
    const double router = static_cast<double>(E) * H * 2;
    const double budget = p.weights_on_gpu * layer_total - router;
    bool open = true;
    for (auto& b : c.blocks) {
        if (open && static_cast<double>(c.resident_bytes + b.bytes) <= budget) {
            b.resident = true;
            b.offset = c.resident_bytes;
            c.resident_bytes += b.bytes;
        } else {
            open = false;
            b.offset = c.blob_bytes;
            c.blob_bytes += b.bytes;
        }
    }
    c.achieved_rw = (static_cast<double>(c.resident_bytes) + router) / layer_total;
    return c;
}

std::pair<int64_t, int64_t> page_range(int64_t blob, int M, int page) {
    if (page <= 0) return {0, blob};
    // n_ub pages per layer (pipesim.cpp:150-162), 4 KiB-aligned boundaries
    auto edge = [&](int q) { return q == M ? blob : ((blob * q / M) & ~static_cast<int64_t>(4095)); };
    return {edge(page - 1), edge(page)};
}

void apply_exact_gates(ScheduleDag& dag, const Catalog& cat, int M) {
    const int n = static_cast<int>(dag.tasks.size());
    const int G = dag.layers * dag.steps;
    std::vector<std::vector<std::pair<int, int>>> pages(G + 1);  // g -> (page, task)
    for (int i = 0; i < n; ++i) {
        const Task& t = dag.tasks[i];
        if (t.kind == TaskKind::WeightToGpu) pages[(t.step - 1) * dag.layers + t.layer].push_back({t.page, i});
    }
    auto needs = [&](bool pre, int page) {
        const auto [b, e] = page_range(cat.blob_bytes, M, page);
        for (const auto& blk : cat.blocks) {
            if (blk.resident || (blk.kind == kWqkv) != pre) continue;
            if (blk.offset < e && blk.offset + blk.bytes > b) return true;
        }
        return false;
    };
    for (int i = 0; i < n; ++i) {
        Task& t = dag.tasks[i];
        if (t.kind != TaskKind::PreAttn && t.kind != TaskKind::PostAttn && t.kind != TaskKind::GpuAttn) continue;
        const int g = (t.step - 1) * dag.layers + t.layer;
        std::vector<int> keep;
        for (int d : t.deps)
            if (dag.tasks[d].kind != TaskKind::WeightToGpu) keep.push_back(d);
        if (t.kind != TaskKind::GpuAttn)  // GPU attention reads only the (resident) KV pool
            for (const auto& [pg, idx] : pages[g])
                if (needs(t.kind == TaskKind::PreAttn, pg)) keep.push_back(idx);
        t.deps = std::move(keep);
    }
}

std::vector<std::vector<int>> reuse_edges(const ScheduleDag& dag) {
    const int n = static_cast<int>(dag.tasks.size());
    const int L = dag.layers;
    std::vector<std::vector<int>> extra(n);
    std::vector<std::vector<int>> gpu_of(L * dag.steps + 2), up_of(L * dag.steps + 2);
    for (int i = 0; i < n; ++i) {
        const Task& t = dag.tasks[i];
        const int g = (t.step - 1) * L + t.layer;
        if (t.resource == Resource::Gpu) gpu_of[g].push_back(i);
        if (t.kind == TaskKind::WeightToGpu) up_of[g].push_back(i);
    }
    for (int i = 0; i < n; ++i) {
        const Task& t = dag.tasks[i];
        const int g = (t.step - 1) * L + t.layer;
        if (g <= 2) continue;
        if (t.kind == TaskKind::WeightToGpu) extra[i] = gpu_of[g - 2];       // pool slot of g-2
        else if (t.kind == TaskKind::WeightToPinned) extra[i] = up_of[g - 2];  // staging slot
    }
    return extra;
}

ScheduleDag execution_dag(const ScheduleDag& reference, const Catalog& cat, int M, bool exact) {
    ScheduleDag d = reference;
    if (exact) apply_exact_gates(d, cat, M);
    const auto extra = reuse_edges(d);
    for (size_t i = 0; i < d.tasks.size(); ++i)
        d.tasks[i].deps.insert(d.tasks[i].deps.end(), extra[i].begin(), extra[i].end());
    return d;
}

}  // namespace mlt
