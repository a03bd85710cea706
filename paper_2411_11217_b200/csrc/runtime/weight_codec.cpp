// Host encoder / reference decoder of the weight-tile codec (weight_codec.hpp).
#include "weight_codec.hpp"

#include <algorithm>
#include <cstring>
#include <vector>

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

namespace mlt {
namespace {
constexpr int kC4Codes = 8192, kC4Rows = 11264, kC4Table = 11392, kC4Hdr = 11400, kC4QMask = 11408,
              kC4Ent = 11424;
inline uint32_t c4_index(uint32_t r, uint32_t k) { return ((k >> 4) * 128u + r) * 16u + (k & 15u); }
// (code word m, bit shift) of the 3-bit code of weight k of a row; bits 0-2
// of a direct code are contiguous, a spare-bit code is spread over words
// 3H, 3H+1, 3H+2 at bit 4n+3 (see weight_codec.hpp)
inline void c4_put(uint32_t* words, uint32_t k, uint32_t code) {
    const uint32_t H = k >> 5, kk = k & 31u, n = kk & 7u;
    if (kk < 24) {
        words[3 * H + (kk >> 3)] |= code << (4 * n);
    } else {
        for (uint32_t b = 0; b < 3; ++b) words[3 * H + b] |= ((code >> b) & 1u) << (4 * n + 3);
    }
}
inline uint32_t c4_get(const uint32_t* words, uint32_t k) {
    const uint32_t H = k >> 5, kk = k & 31u, n = kk & 7u;
    if (kk < 24) return (words[3 * H + (kk >> 3)] >> (4 * n)) & 7u;
    uint32_t c = 0;
    for (uint32_t b = 0; b < 3; ++b) c |= ((words[3 * H + b] >> (4 * n + 3)) & 1u) << b;
    return c;
}
}  // namespace

bool codec4_encode_rows_tile(const uint8_t* packed, uint8_t* out, int cap, int* entries) {
    uint16_t w[8192];
    rows_from_packed(packed, w);
    bool can_shift = true;  // w + 0x80 must not carry out of the exponent (e = 255)
    for (int i = 0; i < 8192; ++i) can_shift = can_shift && ((w[i] >> 7) & 0xFF) != 0xFF;
    int ph = 0, best_cov = -1;
    uint8_t table[8] = {};
    for (int p = 0; p < (can_shift ? 2 : 1); ++p) {
        uint32_t hist[256] = {};
        for (int i = 0; i < 8192; ++i) ++hist[((w[i] + p * 0x80) >> 8) & 0xFF];
        uint8_t order[256];
        for (int v = 0; v < 256; ++v) order[v] = static_cast<uint8_t>(v);
        std::stable_sort(order, order + 256, [&](uint8_t a, uint8_t b) { return hist[a] > hist[b]; });
        int cov = 0;
        for (int s = 0; s < 8; ++s) cov += static_cast<int>(hist[order[s]]);
        if (cov > best_cov) {
            best_cov = cov, ph = p;
            for (int s = 0; s < 8; ++s) table[s] = order[s];  // descending frequency: slot 7 the rarest
        }
    }
    std::memset(out, 0, codec4_tile_bytes(cap));
    // slots 0-6 are fixed for the tile; slot 7 is per row (override byte) and,
    // inside the 4-weight units a row's record flags, a second per-row byte
    int code_of[256];
    for (int v = 0; v < 256; ++v) code_of[v] = -1;
    for (int s = 0; s < 7; ++s) code_of[table[s]] = s;
    struct Hard { uint32_t q, i; uint16_t v; };
    std::vector<Hard> hard;
    uint32_t qmask[4] = {};
    std::vector<uint32_t> recs;
    for (uint32_t r = 0; r < 128; ++r) {
        uint8_t hi[64];
        for (uint32_t k = 0; k < 64; ++k) {
            const uint32_t i = c4_index(r, k);
            const uint16_t x = static_cast<uint16_t>(w[i] + ph * 0x80);
            out[i] = static_cast<uint8_t>(x & 0xFF);
            hi[k] = static_cast<uint8_t>(x >> 8);
        }
        // the row's out-of-table (slot 7) values
        int vals[64], nv = 0, cnt_v[64] = {};
        uint8_t slot_of[256];  // this row's out-of-table value -> index in vals (first seen)
        for (uint32_t k = 0; k < 64; ++k) {
            if (code_of[hi[k]] >= 0) continue;
            bool seen = false;
            for (int a = 0; a < nv && !seen; ++a) seen = vals[a] == hi[k];  // nv is small unless heavy-tailed
            if (!seen) {
                slot_of[hi[k]] = static_cast<uint8_t>(nv);
                vals[nv++] = hi[k];
            }
            ++cnt_v[slot_of[hi[k]]];
        }
        // hard escapes of an assignment: R row-wide, X[h] in the units of row half
        // h (k / 32) that hold an X[h] (the record's unit mask, bits 8h .. 8h + 7)
        auto cost = [&](int R, const int* X, uint32_t* umask_out) {
            uint32_t um = 0;
            for (uint32_t k = 0; k < 64; ++k)
                if (X[k >> 5] >= 0 && hi[k] == X[k >> 5]) um |= 1u << (k >> 2);
            int h = 0;
            for (uint32_t k = 0; k < 64; ++k) {
                if (code_of[hi[k]] >= 0) continue;
                const int slot7 = (um >> (k >> 2)) & 1u ? X[k >> 5] : R;
                h += hi[k] != slot7;
            }
            if (umask_out) *umask_out = um;
            return h;
        };
        // candidates: the row's most frequent out-of-table values (at most 6).
        // For a given R the two halves are independent: per half, the X (or
        // none) with the fewest hard escapes, from per-unit value counts.
        for (int a = 1; a < nv; ++a)  // stable sort by count, descending
            for (int b = a; b > 0 && cnt_v[b] > cnt_v[b - 1]; --b) {
                std::swap(cnt_v[b], cnt_v[b - 1]);
                std::swap(vals[b], vals[b - 1]);
            }
        const int nc = std::min(nv, 6);
        int cu[6][16] = {}, ou[16] = {};  // per unit: count of candidate c, of out-of-table weights
        for (uint32_t k = 0; k < 64; ++k) {
            if (code_of[hi[k]] >= 0) continue;
            ++ou[k >> 2];
            for (int c = 0; c < nc; ++c) cu[c][k >> 2] += hi[k] == vals[c];
        }
        int R = nv ? vals[0] : table[7], X[2] = {-1, -1}, best = 1 << 30;
        for (int a = 0; a < (nv ? nc : 1) && best; ++a) {
            int tot = 0, xb[2] = {-1, -1};
            for (int h = 0; h < 2; ++h) {
                int hb = 1 << 30;
                for (int x = -1; x < nc; ++x) {
                    if (x == a) continue;
                    int hh = 0;
                    for (int u = 8 * h; u < 8 * h + 8; ++u)
                        hh += (x >= 0 && cu[x][u]) ? ou[u] - cu[x][u] : ou[u] - (nv ? cu[a][u] : 0);
                    if (hh < hb) hb = hh, xb[h] = x;
                }
                tot += hb;
            }
            if (tot < best) {
                best = tot, R = nv ? vals[a] : table[7];
                X[0] = xb[0] < 0 ? -1 : vals[xb[0]], X[1] = xb[1] < 0 ? -1 : vals[xb[1]];
            }
        }
        uint32_t um = 0;
        cost(R, X, &um);
        out[kC4Rows + r] = static_cast<uint8_t>(R);
        if (um) {
            qmask[r / 32] |= 1u << (r % 32);
            recs.push_back(um | (static_cast<uint32_t>(X[0] < 0 ? 0 : X[0]) << 16) |
                           (static_cast<uint32_t>(X[1] < 0 ? 0 : X[1]) << 24));
        }
        uint32_t words[6] = {};
        for (uint32_t k = 0; k < 64; ++k) {
            int c = code_of[hi[k]];
            if (c < 0) {
                const int slot7 = (um >> (k >> 2)) & 1u ? X[k >> 5] : R;
                if (hi[k] == slot7) {
                    c = 7;
                } else {
                    const uint32_t i = c4_index(r, k);
                    hard.push_back({r / 32, i, w[i]});
                    c = 0;
                }
            }
            c4_put(words, k, static_cast<uint32_t>(c));
        }
        for (uint32_t m = 0; m < 6; ++m) std::memcpy(out + kC4Codes + (m * 128 + r) * 4, &words[m], 4);
    }
    const int n_ent = static_cast<int>(recs.size() + hard.size());
    if (entries) *entries = n_ent;
    if (n_ent > cap || hard.size() > 255) return false;
    std::memcpy(out + kC4Table, table, 8);
    uint8_t start[4] = {0, 0, 0, 0};
    for (uint32_t q = 1; q < 4; ++q) {
        uint8_t s = 0;
        while (s < hard.size() && hard[s].q < q) ++s;   // rows were visited in order
        start[q] = s;
    }
    out[kC4Hdr] = static_cast<uint8_t>(ph);
    out[kC4Hdr + 1] = start[1], out[kC4Hdr + 2] = start[2], out[kC4Hdr + 3] = start[3];
    out[kC4Hdr + 4] = static_cast<uint8_t>(hard.size());
    out[kC4Hdr + 5] = static_cast<uint8_t>(recs.size());
    std::memcpy(out + kC4QMask, qmask, 16);
    for (size_t e = 0; e < recs.size(); ++e) std::memcpy(out + kC4Ent + 4 * e, &recs[e], 4);
    const size_t h0 = kC4Ent + 4 * recs.size();
    for (size_t e = 0; e < hard.size(); ++e) {
        const uint16_t i16 = static_cast<uint16_t>(hard[e].i);
        std::memcpy(out + h0 + 4 * e, &i16, 2);
        std::memcpy(out + h0 + 4 * e + 2, &hard[e].v, 2);
    }
    return true;
}

void codec4_decode_rows_tile(const uint8_t* enc, uint8_t* packed) {
    uint16_t w[8192];
    const uint8_t* table = enc + kC4Table;
    const int ph = enc[kC4Hdr];
    const int n_hard = enc[kC4Hdr + 4], n_rec = enc[kC4Hdr + 5];
    uint32_t qmask[4];
    std::memcpy(qmask, enc + kC4QMask, 16);
    int rec = 0;
    for (uint32_t r = 0; r < 128; ++r) {
        uint32_t words[6], um = 0, X[2] = {0, 0};
        if ((qmask[r / 32] >> (r % 32)) & 1u) {
            uint32_t v;
            std::memcpy(&v, enc + kC4Ent + 4 * rec++, 4);
            um = v & 0xffffu, X[0] = (v >> 16) & 0xffu, X[1] = v >> 24;
        }
        for (uint32_t m = 0; m < 6; ++m) std::memcpy(&words[m], enc + kC4Codes + (m * 128 + r) * 4, 4);
        for (uint32_t k = 0; k < 64; ++k) {
            const uint32_t i = c4_index(r, k), c = c4_get(words, k);
            const uint32_t hb = c < 7 ? table[c] : ((um >> (k >> 2)) & 1u) ? X[k >> 5] : enc[kC4Rows + r];
            w[i] = static_cast<uint16_t>(((hb << 8) | enc[i]) - ph * 0x80);
        }
    }
    const uint8_t* hard = enc + kC4Ent + 4 * n_rec;
    for (int e = 0; e < n_hard; ++e) {
        uint16_t i16, v;
        std::memcpy(&i16, hard + 4 * e, 2);
        std::memcpy(&v, hard + 4 * e + 2, 2);
        w[i16] = v;
    }
    (void)rec;
    packed_from_rows(w, packed);
}

}  // namespace mlt
