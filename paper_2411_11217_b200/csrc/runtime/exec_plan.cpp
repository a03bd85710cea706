// GPU-free executor planning: catalog + residency, pages, exact gates,
// reuse edges (see exec_plan.hpp and executor.cpp's file comment).
#include "exec_plan.hpp"

#include <cmath>
#include <stdexcept>

#include "host_layout.hpp"
#include "weight_codec.hpp"
#include "lightplan/opcost.hpp"

namespace mlt {

using lightplan::sim::Resource;
using lightplan::sim::ScheduleDag;
using lightplan::sim::Task;
using lightplan::sim::TaskKind;

Shard make_shard(const lightplan::ModelSpec& m, int rank, int size) {
    if (size < 1 || rank < 0 || rank >= size) throw std::invalid_argument("bad tensor-parallel rank/size");
    if (m.q_heads % size || m.kv_heads % size || m.ffn_dim % 128)
        throw std::invalid_argument("tp must divide n_q and n_kv; h2 must be a multiple of 128");
    Shard s;
    s.rank = rank;
    s.size = size;
    s.q_heads = m.q_heads / size;
    s.kv_heads = m.kv_heads / size;
    // h2 in 128-row blocks, as evenly as blocks allow (DBRX h2 = 10752 = 84
    // blocks: tp=8 gives ranks 11 or 10 blocks); every rank keeps UMMA-sized
    // row blocks and the all-reduce sums the uneven partial products exactly
    const int64_t blocks = m.ffn_dim / 128;
    const int64_t b0 = rank * blocks / size, b1 = (rank + 1) * blocks / size;
    s.ffn = (b1 - b0) * 128;
    s.ffn_off = b0 * 128;
    s.qkv_rows = (s.q_heads + 2 * s.kv_heads) * m.head_dim();
    s.o_k = s.q_heads * m.head_dim();
    if (s.qkv_rows % 128 || s.ffn % 128 || s.o_k % 64)
        throw std::invalid_argument("tp shard must keep 128-row weight blocks (qkv rows, h2/tp)");
    return s;
}

ShardMap shard_map(const lightplan::ModelSpec& m, const Shard& s, int kind) {
    ShardMap out;
    const int64_t H = m.hidden_dim, d = m.head_dim(), r = s.rank;
    const double sH = 1.0 / std::sqrt(static_cast<double>(H));
    const double sF = 1.0 / std::sqrt(static_cast<double>(m.ffn_dim));
    switch (kind) {
        case kWqkv: {
            const int64_t qn = s.q_heads * d, kn = s.kv_heads * d;
            for (int64_t i = 0; i < s.qkv_rows; ++i)
                out.rows.push_back(i < qn ? r * qn + i
                                   : i < qn + kn ? m.q_heads * d + r * kn + (i - qn)
                                                 : (m.q_heads + m.kv_heads) * d + r * kn + (i - qn - kn));
            out.k_local = out.k_global = H;
            out.scale = static_cast<float>(sH);
            break;
        }
        case kWo:
            for (int64_t i = 0; i < H; ++i) out.rows.push_back(i);
            out.col0 = r * s.o_k;
            out.k_local = s.o_k;
            out.k_global = m.q_heads * d;
            out.scale = static_cast<float>(sH);
            break;
        case kW1:
        case kW3:
            for (int64_t i = 0; i < s.ffn; ++i) out.rows.push_back(s.ffn_off + i);
            out.k_local = out.k_global = H;
            out.scale = static_cast<float>(sH);
            break;
        case kW2:
            for (int64_t i = 0; i < H; ++i) out.rows.push_back(i);
            out.col0 = s.ffn_off;
            out.k_local = s.ffn;
            out.k_global = m.ffn_dim;
            out.scale = static_cast<float>(sF);
            break;
        default:
            throw std::invalid_argument("shard_map: not a sharded weight kind");
    }
    return out;
}

Catalog build_catalog(const lightplan::ModelSpec& m, const lightplan::Policy& p, const Shard& shard_in,
                      bool codec, const std::vector<uint8_t>* raw_mask, const int* kind_tile_bytes) {
    Catalog c;
    const Shard sh = shard_in.q_heads ? shard_in : make_shard(m, 0, 1);
    const int H = static_cast<int>(m.hidden_dim), F = static_cast<int>(sh.ffn);
    const int E = static_cast<int>(m.experts);
    const int W = static_cast<int>(sh.qkv_rows);
    auto add = [&](int kind, int expert, int rows, int64_t K) {
        for (int rb = 0; rb < rows / 128; ++rb) {
            const size_t i = c.blocks.size();
            const bool raw = codec && raw_mask && i < raw_mask->size() && (*raw_mask)[i];
            const int64_t tile = kind_tile_bytes ? kind_tile_bytes[kind] : kCodecTileBytes;
            const int64_t bytes = (codec && !raw) ? K / 64 * tile : 128 * K * 2;
            c.blocks.push_back({kind, expert, rb, K, bytes, raw, false, 0});
        }
    };
    add(kWqkv, 0, W, H);
    add(kWo, 0, H, sh.o_k);
    for (int e = 0; e < E; ++e) {
        add(kW1, e, F, H);
        add(kW3, e, F, H);
        add(kW2, e, H, F);
    }
    // per-GPU layer bytes as stored (= layer_weight_bytes(m).total() / tp for
    // bf16 blocks, opcost.cpp:49-61); the router stays bf16 and resident
    const double router = static_cast<double>(E) * H * 2;
    double layer_total = router;
    for (const auto& b : c.blocks) layer_total += static_cast<double>(b.bytes);
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
    // page p carries bytes of a QKV block (PreAttn) / of another block
    // (PostAttn): the same for every layer, so tabulated once per page
    std::vector<char> need_pre(M + 1, 0), need_post(M + 1, 0);
    for (int p = 0; p <= M; ++p) {
        const auto [b, e] = page_range(cat.blob_bytes, M, p);
        for (const auto& blk : cat.blocks) {
            if (blk.resident || !(blk.offset < e && blk.offset + blk.bytes > b)) continue;
            (blk.kind == kWqkv ? need_pre : need_post)[p] = 1;
        }
    }
    auto needs = [&](bool pre, int page) {
        return page >= 0 && page <= M && (pre ? need_pre : need_post)[page] != 0;
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
