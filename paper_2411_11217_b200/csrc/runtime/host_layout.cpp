// Host synthetic-weight generator and packed-layout conversion, OpenMP over
// rows.  The generator is a from-scratch statement of the counter PRNG of
// DESIGN.md §3 (splitmix64 keyed by seed and tensor id); tests/
// test_oracle_pins.py checks it against the oracle's independent copy.
#include "host_layout.hpp"

#include <cstring>

#include "../kernels/common.cuh"

namespace mlt {

float bf16_to_f32(uint16_t v) {
    const uint32_t u = static_cast<uint32_t>(v) << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

uint16_t f32_to_bf16(float f) {
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7fffu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

namespace {
inline uint16_t draw(uint64_t key, uint64_t i, float a, bool is_norm) {
    const uint64_t h = mix64(key + i);
    const float r = 2.0f * (static_cast<float>(h >> 40) * 0x1p-24f) - 1.0f;
    return f32_to_bf16(is_norm ? 1.0f + r * 0.1f : r * a);
}
inline float amplitude(float scale) { return static_cast<float>(1.7320508075688772 * static_cast<double>(scale)); }
}  // namespace

void synth_bf16(uint64_t seed, uint64_t tid, int64_t begin, int64_t end, float scale,
                bool is_norm, uint16_t* out) {
    const uint64_t key = mix64(seed ^ mix64(tid));
    const float a = amplitude(scale);
#pragma omp parallel for schedule(static)
    for (int64_t i = begin; i < end; ++i) out[i - begin] = draw(key, static_cast<uint64_t>(i), a, is_norm);
}

void synth_bf16_packed(uint64_t seed, uint64_t tid, int64_t M, int64_t K, int64_t row_begin,
                       int64_t row_end, float scale, uint16_t* dst) {
    (void)M;
    const uint64_t key = mix64(seed ^ mix64(tid));
    const float a = amplitude(scale);
    uint8_t* base = reinterpret_cast<uint8_t*>(dst);
    const uint64_t base_off = mltk::a_packed_off(row_begin, 0, K);
#pragma omp parallel for schedule(static)
    for (int64_t m = row_begin; m < row_end; ++m)
        for (int64_t k = 0; k < K; ++k)
            *reinterpret_cast<uint16_t*>(base + mltk::a_packed_off(m, k, K) - base_off) =
                draw(key, static_cast<uint64_t>(m * K + k), a, false);
}

void synth_shard_packed(uint64_t seed, uint64_t tid, int64_t K_global, const int64_t* rows,
                        int64_t col0, int64_t K_local, int64_t row_begin, int64_t row_end,
                        float scale, uint16_t* dst) {
    const uint64_t key = mix64(seed ^ mix64(tid));
    const float a = amplitude(scale);
    uint8_t* base = reinterpret_cast<uint8_t*>(dst);
    const uint64_t base_off = mltk::a_packed_off(row_begin, 0, K_local);
#pragma omp parallel for schedule(static)
    for (int64_t m = row_begin; m < row_end; ++m) {
        const uint64_t g = static_cast<uint64_t>(rows[m]) * static_cast<uint64_t>(K_global) + static_cast<uint64_t>(col0);
        for (int64_t k = 0; k < K_local; ++k)
            *reinterpret_cast<uint16_t*>(base + mltk::a_packed_off(m, k, K_local) - base_off) =
                draw(key, g + static_cast<uint64_t>(k), a, false);
    }
}

void pack_shard_rows(const uint16_t* full, int64_t K_global, const int64_t* rows, int64_t col0, int64_t K_local,
                     int64_t row_begin, int64_t row_end, uint16_t* dst) {
    uint8_t* base = reinterpret_cast<uint8_t*>(dst);
    const uint64_t base_off = mltk::a_packed_off(row_begin, 0, K_local);
#pragma omp parallel for schedule(static)
    for (int64_t m = row_begin; m < row_end; ++m) {
        const uint16_t* src = full + rows[m] * K_global + col0;
        for (int64_t k = 0; k < K_local; k += 8)
            std::memcpy(base + mltk::a_packed_off(m, k, K_local) - base_off, src + k, 16);
    }
}

void pack_weight(const uint16_t* src, int64_t M, int64_t K, uint16_t* dst) {
    uint8_t* d = reinterpret_cast<uint8_t*>(dst);
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m)
        for (int64_t k = 0; k < K; k += 8)
            std::memcpy(d + mltk::a_packed_off(m, k, K), src + m * K + k, 16);
}

void pack_rows(const uint16_t* src, int64_t rows, int64_t K, int64_t R, uint8_t* dst) {
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < rows; ++n)
        for (int64_t k = 0; k < K; k += 8)
            std::memcpy(dst + mltk::b_packed_off(n, k, R), src + n * K + k, 16);
}

void unpack_rows(const uint8_t* packed, int64_t R, int64_t rows, int64_t K, uint16_t* dst) {
#pragma omp parallel for schedule(static)
    for (int64_t n = 0; n < rows; ++n)
        for (int64_t k = 0; k < K; k += 8)
            std::memcpy(dst + n * K + k, packed + mltk::b_packed_off(n, k, R), 16);
}

}  // namespace mlt
