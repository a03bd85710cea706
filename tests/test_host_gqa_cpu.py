"""Host-core GQA decode attention (the CpuAttn kernel of A_g = 0 policies,
runtime/host_attention.cpp, exported as mlt_host_gqa_decode) against the
oracle's orc_attention (oracle_numerics.c), on CPU.

Layout: the runtime's host KV streams [T][nkv][ctx][d]; the oracle's
[T][ctx][nkv][d].  Output is bf16 (RNE) vs the oracle's fp32: tolerance is
the bf16 rounding of |out| <= 1 plus fp32 reassociation."""
import ctypes as C

import numpy as np
import pytest

from oracle import bind as orc
from paper_2411_11217_b200 import capi

D = 128


def _p(x):
    return x.ctypes.data_as(C.c_void_p)


@pytest.fixture(params=["amx", "avx512"])
def path(request):
    k = capi.load_kernels()
    on = k.host_gqa_use_amx(int(request.param == "amx"))
    if request.param == "amx" and not on:
        pytest.skip("no AMX-BF16 on this host")
    yield request.param
    k.host_gqa_use_amx(1)


@pytest.mark.parametrize("nq,nkv", [(32, 8), (48, 8), (8, 8), (16, 2), (64, 4)])
def test_host_gqa_matches_oracle(path, nq, nkv):
    k = capi.load_kernels()
    rng = np.random.default_rng(nq * 100 + nkv)
    ctx = np.array([1, 15, 16, 17, 100, 127, 128, 64], np.int32)
    T, cap = len(ctx), 128
    q = orc.f32_to_bf16(rng.uniform(-1, 1, (T, nq, D)))
    kv = orc.f32_to_bf16(rng.uniform(-1, 1, (2, T, nkv, cap, D)))
    out = np.zeros((T, nq, D), np.uint16)
    k.host_gqa_decode(_p(q), _p(kv[0]), _p(kv[1]), _p(ctx), T, nq, nkv, D, cap, _p(out), 0)
    ref = orc.attention(orc.bf16_to_f32(q).reshape(T, nq * D),
                        np.ascontiguousarray(kv[0].transpose(0, 2, 1, 3)),
                        np.ascontiguousarray(kv[1].transpose(0, 2, 1, 3)), ctx, nq, nkv, D)
    got = orc.bf16_to_f32(out).reshape(T, nq * D)
    assert np.abs(got - ref).max() < 4e-3
    # ctx = 1: the single value row, exactly (softmax weight 1)
    np.testing.assert_array_equal(out[0].reshape(nkv, nq // nkv, D),
                                  np.broadcast_to(kv[1, 0, :, :1, :], (nkv, nq // nkv, D)))


def test_host_gqa_thread_counts_agree(path):
    k = capi.load_kernels()
    rng = np.random.default_rng(7)
    T, nq, nkv, cap = 16, 32, 8, 96
    ctx = rng.integers(1, cap + 1, T).astype(np.int32)
    q = orc.f32_to_bf16(rng.uniform(-1, 1, (T, nq, D)))
    kc = orc.f32_to_bf16(rng.uniform(-1, 1, (T, nkv, cap, D)))
    vc = orc.f32_to_bf16(rng.uniform(-1, 1, (T, nkv, cap, D)))
    outs = []
    for th in (1, 3, 0):
        o = np.zeros((T, nq, D), np.uint16)
        k.host_gqa_decode(_p(q), _p(kc), _p(vc), _p(ctx), T, nq, nkv, D, cap, _p(o), th)
        outs.append(o)
    np.testing.assert_array_equal(outs[0], outs[1])  # one item per (seq, head): no cross-thread reduction
    np.testing.assert_array_equal(outs[0], outs[2])


def test_host_gqa_rejects_bad_shapes():
    k = capi.load_kernels()
    z = np.zeros(1 << 16, np.uint16)
    ctx = np.array([5], np.int32)
    with pytest.raises(capi.MltError):
        k.host_gqa_decode(_p(z), _p(z), _p(z), _p(ctx), 1, 32, 8, 64, 8, _p(z), 1)   # d != 128
    with pytest.raises(capi.MltError):
        k.host_gqa_decode(_p(z), _p(z), _p(z), _p(ctx), 1, 30, 8, 128, 8, _p(z), 1)  # nq % nkv
    with pytest.raises(capi.MltError):
        k.host_gqa_decode(_p(z), _p(z), _p(z), _p(ctx), 1, 32, 8, 128, 4, _p(z), 1)  # ctx > max_ctx


def test_amx_and_avx512_paths_agree():
    """The tile path (P as bf16 hi + lo) matches the fp32 AVX-512 path to
    within one bf16 ulp of the output (2^-7 relative)."""
    k = capi.load_kernels()
    if not k.host_gqa_use_amx(1):
        pytest.skip("no AMX-BF16 on this host")
    rng = np.random.default_rng(11)
    T, nq, nkv, cap = 12, 48, 8, 300
    ctx = rng.integers(1, cap + 1, T).astype(np.int32)
    q = orc.f32_to_bf16(2 * rng.standard_normal((T, nq, D)))
    kc = orc.f32_to_bf16(rng.standard_normal((T, nkv, cap, D)))
    vc = orc.f32_to_bf16(rng.standard_normal((T, nkv, cap, D)))
    outs = []
    for amx in (1, 0):
        k.host_gqa_use_amx(amx)
        o = np.zeros((T, nq, D), np.uint16)
        k.host_gqa_decode(_p(q), _p(kc), _p(vc), _p(ctx), T, nq, nkv, D, cap, _p(o), 0)
        outs.append(orc.bf16_to_f32(o))
    k.host_gqa_use_amx(1)
    a, b = outs
    assert np.all(np.abs(a - b) <= 2.0 ** -7 * np.maximum(np.abs(a), np.abs(b)) + 1e-6)


def test_host_bandwidth_probe_is_vectorised():
    """mlt_measure_host_bw (the b_c of the B200 HardwareSpec): a 4-accumulator
    vector read, not an add-latency-bound scalar sum — it must beat one core's
    scalar dependent-add rate (a few GB/s) by a wide margin on any AVX-512 host."""
    api = capi.load_product()
    f = api.lib.mlt_measure_host_bw
    f.restype, f.argtypes = C.c_int, [C.c_size_t, C.POINTER(C.c_double)]
    out = (C.c_double * 2)()
    api.check(f(256 << 20, out))
    assert out[0] > 10.0 and out[1] > 5.0, list(out)
