// Host-side synthetic weights (counter PRNG) and packed-layout conversion.
#pragma once

#include <cstdint>

namespace mlt {

// Tensor kinds of the synthetic model (tensor id = ((layer+1) << 16) |
// (kind << 8) | expert); identical numbering in oracle/oracle_numerics.h.
enum TensorKind {
    kEmbed = 0, kLmHead = 1, kFinalNorm = 2, kAttnNorm = 3, kFfnNorm = 4, kWqkv = 5, kWo = 6,
    kRouter = 7, kW1 = 8, kW3 = 9, kW2 = 10, kKCache = 11, kVCache = 12
};

inline uint64_t tensor_id(int layer, int kind, int expert) {
    return (static_cast<uint64_t>(layer + 1) << 16) | (static_cast<uint64_t>(kind) << 8) |
           static_cast<uint64_t>(expert);
}

inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint16_t f32_to_bf16(float f);
float bf16_to_f32(uint16_t v);

// Element i of tensor tid in [begin, end) written to out[0 .. end-begin).
// Values: uniform(-a, a), a = sqrt(3)*scale; norms: 1 + uniform(-0.1, 0.1).
void synth_bf16(uint64_t seed, uint64_t tid, int64_t begin, int64_t end, float scale,
                bool is_norm, uint16_t* out);

// Same values written directly in packed weight layout: tensor [M, K]
// row-major element (m, k) lands at a_packed_off(m, k, K).  Rows
// [row_begin, row_end) only (multiples of 128); dst points at row_begin's
// block.
void synth_bf16_packed(uint64_t seed, uint64_t tid, int64_t M, int64_t K, int64_t row_begin,
                       int64_t row_end, float scale, uint16_t* dst);

// Tensor-parallel shard of a synthetic [M_global, K_global] tensor in packed
// layout: local row m is global row rows[m] (rows.size() = M_local, a multiple
// of 128), local column k is global column col0 + k (k < K_local).  Every
// element equals the unsharded tensor's element, so the union of the shards
// is bit-identical to the full model.  Local rows [row_begin, row_end).
void synth_shard_packed(uint64_t seed, uint64_t tid, int64_t K_global, const int64_t* rows,
                        int64_t col0, int64_t K_local, int64_t row_begin, int64_t row_end,
                        float scale, uint16_t* dst);

void pack_weight(const uint16_t* src, int64_t M, int64_t K, uint16_t* dst);
// The caller-weights counterpart of synth_shard_packed: local rows [row_begin,
// row_end) of this rank's shard of the row-major [M_global, K_global] tensor
// `full` (local row m = global row rows[m], local column k = col0 + k).
void pack_shard_rows(const uint16_t* full, int64_t K_global, const int64_t* rows, int64_t col0, int64_t K_local,
                     int64_t row_begin, int64_t row_end, uint16_t* dst);
void pack_rows(const uint16_t* src, int64_t rows, int64_t K, int64_t R, uint8_t* dst);
void unpack_rows(const uint8_t* packed, int64_t R, int64_t rows, int64_t K, uint16_t* dst);

}  // namespace mlt
