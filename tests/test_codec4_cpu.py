"""Codec 4, the 3-bit row-plane weight code (runtime/weight_codec.hpp
codec4_encode_rows_tile), on the host.

A numpy decoder written from the format description pins the byte layout:
3-bit codes (nibbles of words A, B, C, and their spare bits for the last 8
weights of each 32), the 8-entry high-byte table with the per-row slot-7
override, the per-tile exponent phase, and the quarter-sorted escapes.
Encode -> decode restores every tile bit for bit (synthetic Mixtral weights,
uniform and Gaussian tiles, zeros, tiles with e = 255); blocks that need more
than 48 escapes are reported raw.  Also the stored size against codec 3.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2411_11217_b200 import capi

TILE4 = 11600


@pytest.fixture(scope="module")
def K():
    return capi.load_kernels()


def bf16(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def pack(K, w16, M, Kd):
    out = np.zeros(M * Kd, np.uint16)
    K.pack_weight(np.ascontiguousarray(w16).ctypes.data_as(C.c_void_p), M, Kd, out.ctypes.data_as(C.c_void_p))
    return out.view(np.uint8)


def np_swz_off(r, k):
    return (r >> 3) * 1024 + (r & 7) * 128 + ((((k & 63) >> 3) ^ (r & 7)) << 4) + (k & 7) * 2


R_I, K_I = np.meshgrid(np.arange(128), np.arange(64), indexing="ij")
ROW_PLANE = ((K_I // 16) * 128 + R_I) * 16 + K_I % 16    # [r, k] -> index i


def np_decode4(enc):
    """Spec decoder -> [128, 64] bf16 (row r, column k of the tile)."""
    enc = np.frombuffer(enc, np.uint8)
    words = enc[8192:11264].view(np.uint32).reshape(6, 128)      # [m, r]
    codes = np.zeros((128, 64), np.uint32)
    for k in range(64):
        H, kk = k // 32, k % 32
        n = kk % 8
        if kk < 24:
            codes[:, k] = (words[3 * H + kk // 8] >> (4 * n)) & 7
        else:
            for b in range(3):
                codes[:, k] |= ((words[3 * H + b] >> (4 * n + 3)) & 1) << b
    table = enc[11392:11400]
    ph = int(enc[11400])
    n_hard, n_rec = int(enc[11404]), int(enc[11405])
    qmask = enc[11408:11424].view(np.uint32)
    slot7 = np.repeat(enc[11264:11392][:, None], 64, axis=1).astype(np.uint32)   # R_r
    rec = 0
    for r in range(128):
        if (int(qmask[r // 32]) >> (r % 32)) & 1:
            v = int(enc[11424 + 4 * rec:11428 + 4 * rec].view(np.uint32)[0])
            rec += 1
            for u in range(16):
                if (v >> u) & 1:
                    slot7[r, 4 * u:4 * u + 4] = (v >> (16 + 8 * (u // 8))) & 0xFF    # X_{r,half} in flagged units
    assert rec == n_rec and n_rec + n_hard <= 44
    hi = np.where(codes == 7, slot7, table[np.minimum(codes, 6)]).astype(np.uint32)
    lo = enc[:8192][ROW_PLANE].astype(np.uint32)
    w = ((hi << 8 | lo) - ph * 0x80).astype(np.uint16)
    starts = [0, int(enc[11401]), int(enc[11402]), int(enc[11403]), n_hard]
    assert starts == sorted(starts)
    h0 = 11424 + 4 * n_rec
    prev = None
    for e in range(n_hard):
        i = int(enc[h0 + 4 * e:h0 + 4 * e + 2].view(np.uint16)[0])
        v = enc[h0 + 4 * e + 2:h0 + 4 * e + 4].view(np.uint16)[0]
        r, k = (i >> 4) & 127, (i >> 11) * 16 + (i & 15)
        q = r // 32
        assert starts[q] <= e < starts[q + 1]       # sorted by row quarter
        assert prev is None or (r, k) > prev        # then row, column
        prev = (r, k)
        w[r, k] = v
    return w


def tile_weights(packed_tile):
    """[128, 64] bf16 of a packed 16 KiB tile."""
    return packed_tile.view(np.uint16)[np_swz_off(R_I, K_I) // 2]


def encode4(K, packed, M, Kd):
    out = np.zeros(M // 128 * (Kd // 64) * 16384, np.uint8)
    raw = np.zeros(M // 128, np.uint8)
    n_raw = K.codec4_encode_rows(packed.ctypes.data_as(C.c_void_p), M, Kd, out.ctypes.data_as(C.c_void_p),
                                 raw.ctypes.data_as(C.c_void_p))
    return out, raw, n_raw


@pytest.mark.parametrize("fan", [4096, 14336])
def test_roundtrip_synthetic_mixtral(K, fan):
    """The runtime's synthetic weights (counter PRNG, uniform(+-sqrt3/sqrt(fan))):
    every block codes, escapes well under the cap, bit-exact round trip."""
    from oracle import bind as orc
    Kd = 1024
    w = orc.gen_bf16(1234, orc.tensor_id(0, 8 if fan == 4096 else 10, 3), 256 * Kd, fan ** -0.5).reshape(256, Kd)
    packed = pack(K, w, 256, Kd)
    out, raw, n_raw = encode4(K, packed, 256, Kd)
    assert n_raw == 0 and not raw.any()
    tiles = 256 // 128 * Kd // 64
    esc = []
    for t in range(tiles):
        enc = out[t * TILE4:(t + 1) * TILE4]
        esc.append(int(enc[11404]) + int(enc[11405]))
        assert np.array_equal(np_decode4(enc.tobytes()), tile_weights(packed[t * 16384:(t + 1) * 16384]))
    assert max(esc) <= 36, esc          # records + hard escapes, of 44
    back = np.zeros_like(packed)
    K.codec4_decode_rows(out.ctypes.data_as(C.c_void_p), tiles, back.ctypes.data_as(C.c_void_p))
    assert np.array_equal(back, packed)
    assert K.codec4_tile_bytes() == TILE4 and TILE4 % 16 == 0
    assert TILE4 / 12432 < 0.934      # >= 6.6 % fewer stored bytes than codec 3


def test_edge_tiles(K):
    """Zeros, signed zeros, denormals, e = 255 (inf / nan: phase 0 forced),
    tiny outliers (escapes), and a block whose tiles overflow -> raw."""
    rng = np.random.default_rng(5)
    M, Kd = 384, 128
    w = bf16(rng.uniform(-0.02, 0.02, (M, Kd)))
    w[0, :64] = 0
    w[1, :8] = 0x8000
    w[2, :4] = [1, 2, 0x8003, 0x0040]                  # denormals
    w[3, 5] = 0x7F80; w[3, 6] = 0xFF80; w[3, 7] = 0x7FC1   # inf, -inf, nan
    w[5, 3] = bf16(np.array([2.0 ** -60]))[0]
    w[100, 60] = bf16(np.array([-(2.0 ** -50)]))[0]
    w[256:] = bf16(rng.normal(0, 1, (128, Kd)) * np.exp(rng.normal(0, 4, (128, Kd))))   # block 2: raw
    packed = pack(K, w, M, Kd)
    out, raw, n_raw = encode4(K, packed, M, Kd)
    assert n_raw == 1 and list(raw) == [0, 0, 1]
    kb = Kd // 64
    for t in range(2 * kb):
        enc = out[t * TILE4:(t + 1) * TILE4]
        assert np.array_equal(np_decode4(enc.tobytes()), tile_weights(packed[t * 16384:(t + 1) * 16384]))
    assert int(out[11400]) == 0                      # tile 0 holds e = 255: no phase shift
    off = 2 * kb * TILE4
    assert np.array_equal(out[off:off + kb * 16384], packed[2 * kb * 16384:])


def test_phase_and_row_override(K):
    """A tile whose binades straddle the high-byte pairing picks phase 1; a
    row whose out-of-table weights share one high byte codes them through its
    slot-7 byte, a second value goes to a unit record, not to escapes."""
    rng = np.random.default_rng(8)
    a = 1.5 * 2.0 ** -7                      # top binade alone in its pair at phase 0
    w = bf16(rng.uniform(-a, a, (128, 64)))
    packed = pack(K, w, 128, 64)
    out, raw, n_raw = encode4(K, packed, 128, 64)
    enc = out[:TILE4]
    assert int(enc[11400]) == 1
    assert np.array_equal(np_decode4(enc.tobytes()), tile_weights(packed[:16384]))
    w2 = bf16(rng.uniform(-0.02, 0.02, (128, 64)))
    w2[9, :6] = bf16(np.full(6, 2.0 ** -30))          # six equal tiny weights in row 9
    w2[9, 40:42] = bf16(np.full(2, -(2.0 ** -33)))     # and a second tiny value in one unit
    packed2 = pack(K, w2, 128, 64)
    out2, _, _ = encode4(K, packed2, 128, 64)
    enc2 = out2[:TILE4]
    assert np.array_equal(np_decode4(enc2.tobytes()), tile_weights(packed2[:16384]))
    n_hard, n_rec = int(enc2[11404]), int(enc2[11405])
    h0 = 11424 + 4 * n_rec
    rows = [((int(enc2[h0 + 4 * e]) | int(enc2[h0 + 1 + 4 * e]) << 8) >> 4) & 127 for e in range(n_hard)]
    assert 9 not in rows
    assert (int(enc2[11408:11412].view(np.uint32)[0]) >> 9) & 1     # row 9 holds a unit record


def test_capacity_per_weight_kind(K):
    """A scale whose top binade is nearly empty (DBRX's down projection,
    sqrt(3/10752) = 1.07 * 2^-6) needs ~28 records + escapes per tile: with
    too small a capacity blocks overflow to raw; the runtime sizes the
    capacity per weight kind (mlt_codec4_encode_rows_cap, tiles of 11424 +
    4 cap bytes), which codes every block and round-trips exactly."""
    from oracle import bind as orc
    M, Kd = 1024, 1024
    w = orc.gen_bf16(1234, orc.tensor_id(0, 10, 1), M * Kd, 10752 ** -0.5).reshape(M, Kd)
    packed = pack(K, w, M, Kd)
    small = np.zeros(M // 128 * (Kd // 64) * 16384, np.uint8)
    raw = np.zeros(M // 128, np.uint8)
    assert K.codec4_encode_rows_cap(packed.ctypes.data_as(C.c_void_p), M, Kd, 16, small.ctypes.data_as(C.c_void_p),
                                    raw.ctypes.data_as(C.c_void_p)) > 0     # too small a capacity: raw blocks
    cap = 80
    tb = K.codec4_tile_bytes_for(cap)
    assert tb == 11424 + 4 * cap and tb % 16 == 0 and K.codec4_tile_bytes_for(44) == TILE4
    out = np.zeros(M // 128 * (Kd // 64) * 16384, np.uint8)
    raw = np.zeros(M // 128, np.uint8)
    assert K.codec4_encode_rows_cap(packed.ctypes.data_as(C.c_void_p), M, Kd, cap, out.ctypes.data_as(C.c_void_p),
                                    raw.ctypes.data_as(C.c_void_p)) == 0
    tiles = M // 128 * Kd // 64
    ent = [int(out[t * tb + 11404]) + int(out[t * tb + 11405]) for t in range(tiles)]
    assert 16 < max(ent) <= cap
    back = np.zeros_like(packed)
    K.codec4_decode_rows_cap(out.ctypes.data_as(C.c_void_p), tiles, cap, back.ctypes.data_as(C.c_void_p))
    assert np.array_equal(back, packed)
    with pytest.raises(capi.MltError):
        K.codec4_encode_rows_cap(packed.ctypes.data_as(C.c_void_p), M, Kd, 201, out.ctypes.data_as(C.c_void_p), None)
