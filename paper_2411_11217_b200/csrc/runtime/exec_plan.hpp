// Pure (GPU-free) planning pieces of the executor: the per-layer weight
// block catalog with its residency split, page byte ranges, data-exact weight
// gates and buffer-reuse edges.  Exposed through mlt_execution_dag so the
// CPU test suite can check the executed graph without a device.
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "lightplan/config.hpp"
#include "lightplan/pipesim.hpp"

namespace mlt {

// One 128-row block of one weight matrix (packed layout, all of K).
struct WeightBlock {
    int kind;       // TensorKind (kWqkv, kWo, kW1, kW3, kW2)
    int expert;
    int rb;         // row block
    int64_t K;      // reduction length
    int64_t bytes;  // 128 * K * 2
    bool resident;
    int64_t offset;  // resident: offset in the layer's resident region; streamed: in the layer blob
};

struct Catalog {
    std::vector<WeightBlock> blocks;  // identical for every layer
    int64_t resident_bytes = 0;       // per layer, excluding the router
    int64_t blob_bytes = 0;           // streamed bytes per layer (the D3 of this build)
    double achieved_rw = 0;           // realised r_w (router counted resident)
};

// Resident first: QKV, O, then expert row blocks in (expert, W1, W3, W2)
// order while resident + router <= r_w * W_layer.
Catalog build_catalog(const lightplan::ModelSpec& model, const lightplan::Policy& policy);

// Byte range [begin, end) of page p (1..M) of a layer blob; p = 0: whole.
std::pair<int64_t, int64_t> page_range(int64_t blob_bytes, int M, int page);

// Replace the reference's all-pages weight gates by data-exact ones.
void apply_exact_gates(lightplan::sim::ScheduleDag& dag, const Catalog& cat, int M);

// Write-after-read edges for the two-slot page pool / staging ring.
std::vector<std::vector<int>> reuse_edges(const lightplan::sim::ScheduleDag& dag);

// The graph the executor runs: the reference DAG (same issue order), with
// exact gates if requested and the reuse edges folded into deps.
lightplan::sim::ScheduleDag execution_dag(const lightplan::sim::ScheduleDag& reference,
                                          const Catalog& cat, int M, bool exact_gates);

}  // namespace mlt
