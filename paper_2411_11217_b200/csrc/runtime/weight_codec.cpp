// Host encoder / reference decoder of the weight-tile codec (weight_codec.hpp).
#include "weight_codec.hpp"

#include <algorithm>
#include <cstring>

#include "../kernels/common.cuh"

namespace mlt {

bool codec_encode_tile(const uint8_t* tile, uint8_t* out) {
    uint32_t hist[256] = {};
    for (int i = 0; i < 8192; ++i) ++hist[tile[2 * i + 1]];
    // the 15 most frequent high bytes (ties -> smaller value: deterministic)
    uint8_t order[256];
    for (int v = 0; v < 256; ++v) order[v] = static_cast<uint8_t>(v);
    std::stable_sort(order, order + 256, [&](uint8_t a, uint8_t b) { return hist[a] > hist[b]; });
    uint8_t code_of[256];
    std::memset(code_of, 15, sizeof(code_of));
    uint8_t* table = out + 12288;
    std::memset(table, 0, 16);
    for (int c = 0; c < 15; ++c) {
        if (!hist[order[c]]) break;
        table[c] = order[c];
        code_of[order[c]] = static_cast<uint8_t>(c);
    }
    uint8_t* codes = out + 8192;
    std::memset(codes, 0, 4096);
    int n = 0;
    uint8_t* esc = out + 12308;
    std::memset(out + 12304, 0, kCodecTileBytes - 12304);
    for (int i = 0; i < 8192; ++i) {
        out[i] = tile[2 * i];
        const uint8_t hi = tile[2 * i + 1];
        const uint8_t c = code_of[hi];
        codes[i >> 1] |= static_cast<uint8_t>(c << ((i & 1) * 4));
        if (c == 15) {
            if (n == kCodecMaxEscapes) return false;
            esc[4 * n] = static_cast<uint8_t>(i & 0xff);
            esc[4 * n + 1] = static_cast<uint8_t>(i >> 8);
            esc[4 * n + 2] = hi;
            ++n;
        }
    }
    out[12304] = static_cast<uint8_t>(n & 0xff);
    out[12305] = static_cast<uint8_t>(n >> 8);
    return true;
}

void codec_decode_tile(const uint8_t* enc, uint8_t* tile) {
    const uint8_t* table = enc + 12288;
    for (int i = 0; i < 8192; ++i) {
        const int c = (enc[8192 + (i >> 1)] >> ((i & 1) * 4)) & 15;
        tile[2 * i] = enc[i];
        tile[2 * i + 1] = table[c];
    }
    const int n = enc[12304] | (enc[12305] << 8);
    for (int e = 0; e < n; ++e) {
        const int i = enc[12308 + 4 * e] | (enc[12309 + 4 * e] << 8);
        tile[2 * i + 1] = enc[12310 + 4 * e];
    }
}

namespace {
// packed (SWIZZLE_128B image) byte offset of fragment-order weight i
inline uint32_t frag_src(uint32_t i) {
    const uint32_t u = i >> 3, j = i & 7u;
    const uint32_t lane = u & 31u, kk = (u >> 5) & 3u, mb = u >> 7;
    const uint32_t r = 16u * mb + (lane >> 2) + 8u * ((j >> 1) & 1u);
    const uint32_t k = 16u * kk + 2u * (lane & 3u) + (j & 1u) + 8u * (j >> 2);
    return mltk::swz_off(r, k);
}
}  // namespace

void frag_from_packed(const uint8_t* packed, uint16_t* frag) {
    for (uint32_t i = 0; i < 8192; ++i) std::memcpy(frag + i, packed + frag_src(i), 2);
}

void packed_from_frag(const uint16_t* frag, uint8_t* packed) {
    for (uint32_t i = 0; i < 8192; ++i) std::memcpy(packed + frag_src(i), frag + i, 2);
}

bool codec_encode_frag_tile(const uint8_t* packed, uint8_t* out) {
    uint16_t frag[8192];
    frag_from_packed(packed, frag);
    return codec_encode_tile(reinterpret_cast<const uint8_t*>(frag), out);
}

namespace {
// packed (SWIZZLE_128B image) byte offset of row-plane weight i
inline uint32_t rows_src(uint32_t i) {
    const uint32_t t = i & 15u, r = (i >> 4) & 127u, j = i >> 11;
    return mltk::swz_off(r, 16u * j + t);
}
}  // namespace

void rows_from_packed(const uint8_t* packed, uint16_t* rows) {
    for (uint32_t i = 0; i < 8192; ++i) std::memcpy(rows + i, packed + rows_src(i), 2);
}

void packed_from_rows(const uint16_t* rows, uint8_t* packed) {
    for (uint32_t i = 0; i < 8192; ++i) std::memcpy(packed + rows_src(i), rows + i, 2);
}

bool codec_encode_rows_tile(const uint8_t* packed, uint8_t* out) {
    uint16_t rows[8192];
    rows_from_packed(packed, rows);
    return codec_encode_tile(reinterpret_cast<const uint8_t*>(rows), out);
}

}  // namespace mlt
