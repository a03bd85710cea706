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

namespace mlt {

// ---- codec 4: 3-bit code (GemmArgs::codec = 4, kernels/gemm_tc.cu) --------
// Same row-plane weight order and TMEM-operand engine as codec 3, 11 stored
// bits per weight instead of 12.  A per-tile phase ph in {0, 1} shifts every
// weight by ph * 0x80 (one exponent step: ph = 1 pairs binades (2m-1, 2m)
// instead of (2m, 2m+1), whichever leaves fewer weights outside the table):
// w' = w + ph * 0x80.  Stored: w' low byte raw and a 3-bit index of w' high
// byte: slots 0-6 into the tile's table of its most frequent high bytes, slot
// 7 into the row's override byte R_r, except inside the 4-weight units a row
// record flags, where slot 7 means the record's byte X_{r,h} for that row half
// h = k / 32 (up to two more per-row values).  Weights that still miss are
// "hard" escapes {index, bf16}.  Layout:
//   [0, 8192)       low byte of w'_i (i = ((k / 16) * 128 + r) * 16 + k % 16)
//   [8192, 11264)   codes: u32 word m (0..5) of row r at 8192 + (m * 128 + r) * 4;
//                   for H = m / 3, words A, B, C = 3H, 3H+1, 3H+2: nibble n
//                   (bits 4n..4n+2) holds the code of k = 32H + n (A),
//                   32H + 8 + n (B), 32H + 16 + n (C); bit 4n+3 of A, B, C
//                   holds bit 0, 1, 2 of the code of k = 32H + 24 + n
//   [11264, 11392)  R_r, per row
//   [11392, 11400)  table[8] (slot 7 unused by the decoder)
//   [11400, 11404)  {phase, first hard escape of row quarter 1, 2, 3} (u8)
//   [11404, 11408)  {n_hard, n_rec, 0, 0} (u8)
//   [11408, 11424)  u32 per row quarter: bit l = row 32q + l has a record
//   [11424, ...)    n_rec records in row order {u16 unit mask (bit u: k in
//                   [4u, 4u+4)), u8 X_{r,0} (units 0-7), u8 X_{r,1} (units
//                   8-15)}, then n_hard hard escapes
//                   {u16 index i, u16 bf16 w_i} in row order;
//                   n_rec + n_hard <= the tile's capacity
// Decoding: w_i = (slot byte << 8 | low) - ph * 0x80, then hard escapes.
// Capacity: records + hard escapes per tile.  The runtime sizes it per weight
// kind from the weights (scan_raw_blocks: the kind's largest tile), so the
// tile is codec4_tile_bytes(cap) = 11424 + 4 cap rounded up to 16 B; 44 is
// the C-ABI default (mlt_codec4_encode_rows: 11600 B).
constexpr int kCodec4MaxEntries = 44;   // default capacity
constexpr int kCodec4CapLimit = 200;    // beyond: the block is stored raw
constexpr int kCodec4TileBytes = 11600;  // at the default capacity
constexpr int codec4_tile_bytes(int cap) { return (11424 + 4 * cap + 15) & ~15; }
static_assert(codec4_tile_bytes(kCodec4MaxEntries) == kCodec4TileBytes, "default tile size");
// Encode one tile with at most cap entries; false if it needs more.  With
// entries != nullptr the count is reported (also when it exceeds cap; out
// must then hold codec4_tile_bytes(kCodec4CapLimit) bytes).
bool codec4_encode_rows_tile(const uint8_t* packed16k, uint8_t* out, int cap = kCodec4MaxEntries,
                             int* entries = nullptr);
void codec4_decode_rows_tile(const uint8_t* enc, uint8_t* packed16k);

// stored bytes of one encoded 64-k tile in GemmArgs::codec mode m (1-4)
inline int codec_tile_bytes(int mode) { return mode == 4 ? kCodec4TileBytes : kCodecTileBytes; }

}  // namespace mlt
