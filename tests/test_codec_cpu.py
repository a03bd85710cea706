"""Lossless weight-tile codec (runtime/weight_codec.hpp) on the host.

A numpy decoder written from the format description (not from the C++ code)
pins the byte layout; encode -> decode must restore every packed tile bit
for bit: synthetic Mixtral-style weights, Gaussian weights, tiles that need
escapes, and the overflow error when a tile's high bytes do not fit.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2411_11217_b200 import capi

TILE = 12432


@pytest.fixture(scope="module")
def K():
    return capi.load_kernels()


def np_decode(enc):
    """Spec decoder: low bytes raw, 4-bit codes into a 16-entry high-byte table,
    escapes {u16 index, u8 high byte, u8 0} at 12308."""
    enc = np.frombuffer(enc, np.uint8)
    lo = enc[:8192]
    nib = enc[8192:12288]
    codes = np.empty(8192, np.uint8)
    codes[0::2] = nib & 15
    codes[1::2] = nib >> 4
    hi = enc[12288:12304][codes].copy()
    n = int(enc[12304]) | (int(enc[12305]) << 8)
    for e in range(n):
        i = int(enc[12308 + 4 * e]) | (int(enc[12309 + 4 * e]) << 8)
        assert codes[i] == 15
        hi[i] = enc[12310 + 4 * e]
    out = np.empty(16384, np.uint8)
    out[0::2], out[1::2] = lo, hi
    return out


def encode(K, packed, M, Kd):
    out = np.zeros(M // 128 * (Kd // 64) * TILE, np.uint8)
    K.codec_encode(packed.ctypes.data_as(C.c_void_p), M, Kd, out.ctypes.data_as(C.c_void_p))
    return out


def pack(K, w16, M, Kd):
    out = np.zeros(M * Kd, np.uint16)
    K.pack_weight(w16.ctypes.data_as(C.c_void_p), M, Kd, out.ctypes.data_as(C.c_void_p))
    return out.view(np.uint8)


def bf16(x):
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


@pytest.mark.parametrize("dist", ["uniform", "gauss"])
def test_roundtrip_weights(K, dist):
    M, Kd = 256, 512
    rng = np.random.default_rng(3)
    sig = Kd ** -0.5
    x = rng.uniform(-3 ** 0.5 * sig, 3 ** 0.5 * sig, (M, Kd)) if dist == "uniform" else rng.normal(0, sig, (M, Kd))
    packed = pack(K, bf16(x), M, Kd)
    enc = encode(K, packed, M, Kd)
    assert enc.nbytes == packed.nbytes * TILE // 16384  # -24.1 %
    tiles = M // 128 * Kd // 64
    for t in range(tiles):
        assert np.array_equal(np_decode(enc[t * TILE:(t + 1) * TILE].tobytes()), packed[t * 16384:(t + 1) * 16384])
    back = np.zeros_like(packed)
    K.codec_decode(enc.ctypes.data_as(C.c_void_p), tiles, back.ctypes.data_as(C.c_void_p))
    assert np.array_equal(back, packed)


def test_escapes_and_overflow(K):
    rng = np.random.default_rng(9)
    w = bf16(rng.uniform(-0.02, 0.02, (128, 64)))
    # 20 rare high bytes beyond the 15 table entries -> escapes
    rare = bf16(np.array([2.0 ** e for e in range(-30, -10)] + [-(2.0 ** e) for e in range(-30, -20)]))
    w.reshape(-1)[[7, 100, 2047, 4096, 8191, 1, 3, 5, 9, 11, 13, 15, 17, 19, 21, 23, 25, 27, 29, 31][:20]] = rare[:20]
    packed = pack(K, w, 128, 64)
    enc = encode(K, packed, 128, 64)
    n = int(enc[12304]) | (int(enc[12305]) << 8)
    assert 0 < n <= 31
    assert np.array_equal(np_decode(enc.tobytes()), packed)
    # > 31 distinct rare high bytes -> the tile cannot be coded
    w2 = w.copy()
    many = bf16(np.concatenate([2.0 ** np.arange(-60, -20, dtype=np.float64), -(2.0 ** np.arange(-60, -20, dtype=np.float64))]))
    w2.reshape(-1)[:80] = many
    with pytest.raises(capi.MltError):
        encode(K, pack(K, w2, 128, 64), 128, 64)


def test_product_synthetic_weights_encode(K):
    """The runtime's synthetic weights (counter PRNG, uniform(-sqrt3 s, sqrt3 s))
    all fit the code with few escapes."""
    from oracle import bind as orc
    Kd = 4096
    w = orc.gen_bf16(1234, orc.tensor_id(0, 8, 3), 256 * Kd, Kd ** -0.5).reshape(256, Kd)
    packed = pack(K, w, 256, Kd)
    enc = encode(K, packed, 256, Kd)
    tiles = 2 * Kd // 64
    esc = [int(enc[t * TILE + 12304]) for t in range(tiles)]
    assert max(esc) <= 8
    back = np.zeros_like(packed)
    K.codec_decode(enc.ctypes.data_as(C.c_void_p), tiles, back.ctypes.data_as(C.c_void_p))
    assert np.array_equal(back, packed)


def np_swz_off(r, k):
    """Byte offset of element (r, k) in a packed 16 KiB tile (SWIZZLE_128B image)."""
    return (r >> 3) * 1024 + (r & 7) * 128 + ((((k & 63) >> 3) ^ (r & 7)) << 4) + (k & 7) * 2


def test_row_plane_order_roundtrip(K):
    """Codec-3 tiles (mlt_codec_encode_rows): the spec decoder yields the tile's
    weights in row-plane order i = ((k // 16) * 128 + r) * 16 + k % 16; mapped
    back through the swizzle they equal the packed tile, escapes included; a
    block that cannot be coded is reported raw and copied as packed tiles."""
    rng = np.random.default_rng(11)
    M, Kd = 256, 256
    w = bf16(rng.normal(0, Kd ** -0.5, (M, Kd)))
    w[3, 17] = bf16(np.array([2.0 ** -40]))[0]          # an escape in block 0
    w[128:] = bf16(rng.normal(0, 1, (128, Kd)) * np.exp(rng.normal(0, 4, (128, Kd))))  # block 1: raw
    packed = pack(K, w, M, Kd)
    out = np.zeros(M * Kd * 2, np.uint8)
    raw = np.zeros(M // 128, np.uint8)
    n_raw = K.codec_encode_rows(packed.ctypes.data_as(C.c_void_p), M, Kd, out.ctypes.data_as(C.c_void_p),
                                raw.ctypes.data_as(C.c_void_p))
    assert n_raw == 1 and list(raw) == [0, 1]
    r_i, k_i = np.meshgrid(np.arange(128), np.arange(64), indexing="ij")
    row_plane = ((k_i // 16) * 128 + r_i) * 16 + k_i % 16
    src = np_swz_off(r_i, k_i)
    kb = Kd // 64
    for t in range(kb):
        dec = np_decode(out[t * TILE:(t + 1) * TILE].tobytes())
        vals = dec.view(np.uint16)[row_plane]
        ref = packed[t * 16384:(t + 1) * 16384].view(np.uint16)[src // 2]
        assert np.array_equal(vals, ref)
    assert int(out[12304]) >= 1 or any(int(out[t * TILE + 12304]) for t in range(kb))
    off = kb * TILE
    assert np.array_equal(out[off:off + kb * 16384], packed[kb * 16384:2 * kb * 16384])
