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
#include "weight_codec.hpp"

namespace mlt {

// One 128-row block of one weight matrix (packed layout, all of K).
struct WeightBlock {
    int kind;       // TensorKind (kWqkv, kWo, kW1, kW3, kW2)
    int expert;
    int rb;         // row block
    int64_t K;      // reduction length
    int64_t bytes;  // 128 * K * 2, or the encoded size (codec)
    bool raw;       // codec: stored as raw bf16 tiles (per-block fallback, tagged page-table entry)
    bool resident;
    int64_t offset;  // resident: offset in the layer's resident region; streamed: in the layer blob
};

struct Catalog {
    std::vector<WeightBlock> blocks;  // identical for every layer
    int64_t resident_bytes = 0;       // per layer, excluding the router
    int64_t blob_bytes = 0;           // streamed bytes per layer (the D3 of this build)
    double achieved_rw = 0;           // realised r_w (router counted resident)
};

// Tensor-parallel shard of one rank: heads and the expert hidden dim are
// split tp ways (QKV / W1 / W3 by rows, O / W2 by columns); router, norms,
// embedding and lm_head are replicated.
struct Shard {
    int rank = 0, size = 1;
    int64_t q_heads = 0, kv_heads = 0, ffn = 0;  // local counts
    int64_t ffn_off = 0;                         // first global h2 row of this rank's slice
    int64_t qkv_rows = 0;                        // (q_heads + 2 kv_heads) * d
    int64_t o_k = 0;                             // q_heads * d (O projection K)
};
Shard make_shard(const lightplan::ModelSpec& model, int rank, int size);

// Which global rows / columns this rank's local matrix of `kind` covers:
// local (m, k) is global (rows[m], col0 + k) of the [.., k_global] tensor.
// QKV: this rank's q heads, then k heads, then v heads; O: all rows, the
// columns of this rank's heads; W1/W3: rows [r*h2/tp, ...); W2: all rows,
// columns [r*h2/tp, ...).  scale = the synthetic init scale (1/sqrt(fan_in)).
struct ShardMap {
    std::vector<int64_t> rows;
    int64_t col0 = 0, k_local = 0, k_global = 0;
    float scale = 0;
};
ShardMap shard_map(const lightplan::ModelSpec& model, const Shard& shard, int kind);

// Resident first: QKV, O, then expert row blocks in (expert, W1, W3, W2)
// order while resident + router <= r_w * (W_layer / tp) (SURVEY.md
// Appendix B; the reference's uniform share, per GPU under TP).
// codec: blocks are stored encoded (weight_codec.hpp: 12432 B per 64-k tile
// instead of 16384), so the same r_w share holds more weights and the pages
// stream fewer bytes.
// kind_tile_bytes (codec only): stored bytes per encoded 64-k tile, indexed by
// TensorKind (codec 4 sizes its tiles per kind); nullptr: 12432 for every kind.
// raw_mask (codec only): raw_mask[i] != 0 stores catalog block i as raw
// 16 KiB tiles in every layer — the fallback for weights the code cannot hold.
Catalog build_catalog(const lightplan::ModelSpec& model, const lightplan::Policy& policy,
                      const Shard& shard = Shard{}, bool codec = false,
                      const std::vector<uint8_t>* raw_mask = nullptr, const int* kind_tile_bytes = nullptr);

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
