"""Host-side layout and synthetic-weight parity (CPU only).

* the product's counter PRNG (runtime/host_layout.cpp) and the oracle's
  independent copy (oracle/oracle_numerics.c) produce bit-identical bf16
  tensors — "identical synthetic weights";
* packed weight / activation layouts match the documented byte formula
  (kernels/common.cuh) and round-trip;
* the product's RoPE table equals the oracle's cos/sin.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2411_11217_b200 import capi


@pytest.fixture(scope="module")
def K():
    return capi.load_kernels()


def vp(a):
    return a.ctypes.data_as(C.c_void_p)


@pytest.mark.parametrize("layer,kind,expert,n,scale,norm", [
    (-1, 0, 0, 4096, 1.0, 0), (-1, 1, 0, 8192, 4 / 32, 0), (0, 3, 0, 1024, 0.0, 1),
    (5, 8, 3, 10000, 1 / 64, 0), (31, 10, 7, 3333, 1 / 119.7, 0), (2, 7, 0, 8 * 4096, 1 / 64, 0)])
def test_synthetic_weights_bit_identical_to_oracle(K, layer, kind, expert, n, scale, norm):
    from oracle import bind as orc
    tid = orc.tensor_id(layer, kind, expert)
    ours = np.zeros(n, np.uint16)
    K.synth_bf16(1234, tid, n, scale, norm, vp(ours))
    assert np.array_equal(ours, orc.gen_bf16(1234, tid, n, scale, bool(norm)))
    vals = orc.bf16_to_f32(ours)
    a = 1.0 + 0.1 if norm else 3 ** 0.5 * scale
    lo, hi = (0.9 - 1e-2, 1.1 + 1e-2) if norm else (-a * 1.01, a * 1.01)
    assert vals.min() >= lo and vals.max() <= hi


def swz(r, k):
    return (r // 8) * 1024 + (r % 8) * 128 + (((k % 64) // 8) ^ (r % 8)) * 16 + (k % 8) * 2


def test_pack_weight_layout(K):
    M, Kd = 256, 192
    src = np.arange(M * Kd, dtype=np.uint32).astype(np.uint16).reshape(M, Kd)
    dst = np.zeros(M * Kd, np.uint16)
    K.pack_weight(vp(src), M, Kd, vp(dst))
    b = dst.view(np.uint8)
    rng = np.random.default_rng(0)
    for _ in range(500):
        m, k = int(rng.integers(M)), int(rng.integers(Kd))
        off = ((m // 128) * (Kd // 64) + k // 64) * 16384 + swz(m % 128, k)
        assert b[off:off + 2].view(np.uint16)[0] == src[m, k]


def test_pack_rows_layout_and_roundtrip(K):
    rows, Kd, R = 37, 256, 48
    src = np.random.default_rng(1).integers(0, 65535, (rows, Kd)).astype(np.uint16)
    packed = np.zeros(R * Kd * 2, np.uint8)
    K.pack_rows_host(vp(src), rows, Kd, R, vp(packed))
    for n, k in [(0, 0), (36, 255), (9, 70), (17, 129)]:
        off = (k // 64) * R * 128 + swz(n, k)
        assert packed[off:off + 2].view(np.uint16)[0] == src[n, k]
    back = np.zeros_like(src)
    K.unpack_rows(vp(packed), R, rows, Kd, vp(back))
    assert np.array_equal(back, src)


def test_layout_argument_checks(K):
    a = np.zeros(16, np.uint16)
    with pytest.raises(capi.MltError):
        K.pack_weight(vp(a), 100, 64, vp(a))  # M % 128
    with pytest.raises(capi.MltError):
        K.unpack_rows(vp(a), 8, 9, 64, vp(a))  # rows > R


def test_rope_table_matches_oracle(K):
    from oracle import bind as orc
    d, P = 128, 40
    tab = np.zeros((P, d // 2, 2), np.float32)
    K.rope_table(P, d, 1e6, vp(tab))
    x = np.random.default_rng(2).standard_normal((P, 2 * d)).astype(np.float32)
    ref = orc.rope(x, np.arange(P, dtype=np.int32), 2, d, 1e6)
    c, s = tab[:, None, :, 0], tab[:, None, :, 1]
    v = x.reshape(P, 2, d)
    a, b = v[..., : d // 2], v[..., d // 2:]
    ours = np.concatenate([a * c - b * s, b * c + a * s], axis=-1).reshape(P, 2 * d)
    assert np.array_equal(ours, ref)
