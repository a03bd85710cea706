// Lossless weight-tile codec ("hi-byte table" code).
//
// The unit is one 16 KiB packed weight tile (128 rows x 64 k, the exact
// SWIZZLE_128B smem image the GEMM consumes, common.cuh): 8192 bf16 values
// w_i at byte 2i.  A bf16 is [sign:1][exponent:8][mantissa:7]; its LOW byte
// (exponent lsb + mantissa) is close to uniformly distributed, its HIGH byte
// (sign + exponent msbs) takes a handful of values for trained or synthetic
// weights (entropy ~2-3 bits).  The encoded tile keeps the low bytes raw and
// replaces each high byte by a 4-bit index into a per-tile table of its 15
// most frequent values; the rare rest are escapes (code 15) listed with
// their position:
//
//   [0, 8192)        low byte of w_i
//   [8192, 12288)    code of w_i in the low (even i) / high (odd i) nibble
//   [12288, 12304)   table[16] of high bytes (entry 15 unused)
//   [12304, 12306)   escape count n (u16), [12306, 12308) reserved
//   [12308, 12432)   escapes: n <= 31 entries {u16 index, u8 high byte, u8 0}
//
// 12432 B instead of 16384 B (-24.1 %), a multiple of 16 so encoded tiles
// pack back to back and stay cp.async.bulk-aligned.  Decoding is exact: the
// tensor cores consume bit-identical bf16 tiles either way.
#pragma once

#include <cstdint>

namespace mlt {

constexpr int kCodecTileBytes = 12432;
constexpr int kCodecMaxEscapes = 31;

// Encode one 16 KiB tile; false if it needs more than kCodecMaxEscapes
// escapes (its high bytes spread over > 15 values too evenly).
bool codec_encode_tile(const uint8_t* tile16k, uint8_t* out);
// Host reference decoder (tests; the GEMM decodes in shared memory).
void codec_decode_tile(const uint8_t* enc, uint8_t* tile16k);

// Fragment order (kernels/gemm_codec.cu, GemmArgs::codec = 2): the same
// 128 x 64 weights reordered so that 8-weight unit u = (mb * 4 + kk) * 32 +
// lane holds lane's mma.sync m16n8k16 A fragment of m16 block mb and k16
// block kk: weight j of the unit is row 16 mb + g + 8 ((j >> 1) & 1), k 16 kk
// + 2 tg + (j & 1) + 8 (j >> 2), g = lane / 4, tg = lane % 4.  The codec
// fields are unchanged (the code is order-independent); escape indices refer
// to fragment order.  A raw fallback block stores 16 KiB fragment-order bf16.
void frag_from_packed(const uint8_t* packed16k, uint16_t* frag8192);
void packed_from_frag(const uint16_t* frag8192, uint8_t* packed16k);
bool codec_encode_frag_tile(const uint8_t* packed16k, uint8_t* out);

// Row-plane order (kernels/gemm_tc.cu, GemmArgs::codec = 3: decoded rows go
// to tensor memory, the MMA reads A from TMEM): weight (r, k) of the tile is
// i = ((k / 16) * 128 + r) * 16 + k % 16, so the 16 low bytes (and 8 code
// bytes) of one row's 16-k chunk are one 16-byte (8-byte) word and a warp's
// 32 rows read 32 consecutive words (bank-conflict-free).  Decoder thread r
// expands its row's 64 weights into the 32 TMEM columns of lane r (k pairs
// per 32-bit column).  The codec fields are unchanged; escape indices refer to
// this order.  A raw fallback block stays 16 KiB packed (SWIZZLE_128B) tiles.
void rows_from_packed(const uint8_t* packed16k, uint16_t* rows8192);
void packed_from_rows(const uint16_t* rows8192, uint8_t* packed16k);
bool codec_encode_rows_tile(const uint8_t* packed16k, uint8_t* out);

}  // namespace mlt
