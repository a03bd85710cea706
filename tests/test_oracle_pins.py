"""Pin the CPU numerical oracle before trusting it (CPU only).

Numerics parity is unpinned by the reference (it has no numerical path), so
the oracle's building blocks are pinned here against independent numpy
restatements on small cases, and the router's tie-break / stability rules
 against hand-built cases.
"""
import numpy as np
import pytest

from oracle import bind as orc


def bf(a):
    return orc.f32_to_bf16(np.asarray(a, np.float32))


def test_bf16_rounding_is_rne():
    x = np.array([1.0, 1.00390625, 1.01171875, -2.5, 3.0e-39, 65504.0], np.float32)
    r = orc.bf16_to_f32(orc.f32_to_bf16(x))
    assert r[0] == 1.0 and r[1] == 1.0 and r[2] == 1.015625  # ties to even
    assert r[3] == -2.5 and r[5] == 65536.0


def test_linear_expert_rmsnorm_against_numpy():
    rng = np.random.default_rng(0)
    T, H, F = 5, 128, 96
    x = rng.standard_normal((T, H)).astype(np.float32)
    w1, w3 = bf(rng.standard_normal((F, H)) / 11), bf(rng.standard_normal((F, H)) / 11)
    w2 = bf(rng.standard_normal((H, F)) / 10)
    y = orc.linear(x, w1)
    assert np.allclose(y, x.astype(np.float64) @ orc.bf16_to_f32(w1).T, rtol=1e-5, atol=1e-5)
    g = x @ orc.bf16_to_f32(w1).T.astype(np.float64)
    u = x @ orc.bf16_to_f32(w3).T.astype(np.float64)
    ref = (g / (1 + np.exp(-g)) * u) @ orc.bf16_to_f32(w2).T
    assert np.allclose(orc.expert(x, w1, w3, w2), ref, rtol=1e-4, atol=1e-4)
    gamma = bf(1 + rng.uniform(-0.1, 0.1, H))
    rn = x / np.sqrt((x.astype(np.float64) ** 2).mean(1, keepdims=True) + 1e-5) * orc.bf16_to_f32(gamma)
    assert np.allclose(orc.rmsnorm(x, gamma, 1e-5), rn, rtol=1e-5, atol=1e-6)


def test_attention_against_numpy():
    rng = np.random.default_rng(1)
    T, nq, nkv, d, cap = 3, 4, 2, 16, 9
    q = rng.standard_normal((T, nq * d)).astype(np.float32)
    k = bf(rng.standard_normal((T, cap, nkv, d)))
    v = bf(rng.standard_normal((T, cap, nkv, d)))
    ctx = np.array([1, 5, 9], np.int32)
    out = orc.attention(q, k, v, ctx, nq, nkv, d)
    kf, vf = orc.bf16_to_f32(k), orc.bf16_to_f32(v)
    for t in range(T):
        for h in range(nq):
            kh = h // (nq // nkv)
            s = kf[t, :ctx[t], kh] @ q[t, h * d:(h + 1) * d] / np.sqrt(d)
            p = np.exp(s - s.max())
            p /= p.sum()
            assert np.allclose(out[t, h * d:(h + 1) * d], p @ vf[t, :ctx[t], kh], atol=1e-5)


def test_router_topk_ties_and_stable_permutation():
    H, E, K = 256, 8, 2
    hn = np.zeros((4, H), np.uint16)
    w = np.zeros((E, H), np.uint16)
    one = bf(1.0)[()] if np.ndim(bf(1.0)) == 0 else bf([1.0])[0]
    hn[:, 0] = one
    for e in range(E):  # logits: e3 = e5 = 2 (tie), e1 = 1.5, rest 0
        w[e, 0] = bf([{3: 2.0, 5: 2.0, 1: 1.5}.get(e, 0.0)])[0]
    logits, idx, wts, perm, off = orc.router(hn, w, K)
    assert (idx == np.array([[3, 5]] * 4)).all()       # tie -> lower index first
    assert np.allclose(wts, 0.5)
    assert list(off) == [0, 0, 0, 0, 4, 4, 8, 8, 8]
    assert list(perm) == [0, 2, 4, 6, 1, 3, 5, 7]         # stable by (expert, token, slot)


def test_router_logit_tree_is_the_documented_one():
    rng = np.random.default_rng(3)
    H, E = 512, 4
    hn = bf(rng.standard_normal((2, H)))
    w = bf(rng.standard_normal((E, H)) / 20)
    logits, *_ = orc.router(hn, w, 1)
    x, ww = orc.bf16_to_f32(hn), orc.bf16_to_f32(w)
    for t in range(2):
        for e in range(E):
            lane = np.zeros(32, np.float32)
            for l in range(32):
                acc = np.float32(0)
                for c in range(l, H // 8, 32):
                    for j in range(8):
                        # fmaf: exact product + one rounding
                        acc = np.float32(np.float64(x[t, c * 8 + j]) * np.float64(ww[e, c * 8 + j]) + np.float64(acc))
                lane[l] = acc
            for m in (16, 8, 4, 2, 1):
                lane = np.array([np.float32(lane[i] + lane[i ^ m]) for i in range(32)], np.float32)
            assert lane[0] == logits[t, e]


@pytest.mark.parametrize("mode", [orc.FP32, orc.FAITHFUL])
def test_tiny_model_decode_runs_and_is_deterministic(mode):
    a = orc.Model(1, 256, 256, 2, 1, 4, 2, 512, 3, 8, seed=7)
    b = orc.Model(1, 256, 256, 2, 1, 4, 2, 512, 3, 8, seed=7)
    toks = np.array([1, 2, 3], np.int32)
    for s in range(3):
        na, ma = a.decode_step(toks, np.full(3, s, np.int32), mode)
        nb, mb = b.decode_step(toks, np.full(3, s, np.int32), mode)
        assert (na == nb).all() and (ma == mb).all() and (ma >= 0).all()
        toks = na


@pytest.mark.parametrize("T,K,M", [(1, 16, 1), (5, 4096, 14), (64, 1024, 37), (3, 100, 7), (17, 33, 9)])
def test_blocked_linear_is_the_scalar_dot_structure(T, K, M):
    """orc_linear (4x4 register-blocked AVX-512, OpenMP) evaluates exactly the
    oracle's one dot-product structure (16 lane partials of fused
    multiply-adds, summed left to right, then the tail): bit-identical to the
    plain statement orc_linear_scalar for any shape, including M/T/K tails."""
    rng = np.random.default_rng(T * 1000 + K + M)
    x = rng.standard_normal((T, K)).astype(np.float32)
    w = bf(rng.standard_normal((M, K)) * 0.05)
    a = np.zeros((T, M), np.float32)
    b = np.zeros((T, M), np.float32)
    orc.lib().orc_linear(orc.p(x), orc.p(w), T, K, M, orc.p(a))
    orc.lib().orc_linear_scalar(orc.p(x), orc.p(w), T, K, M, orc.p(b))
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_forced_routes_reproduce_own_routes_bitwise():
    """orc_model_force_routes with the oracle's own top-k reproduces the
    unforced step bit for bit (same weights, same permutation); a different
    route changes the residual; out-of-range experts are rejected."""
    def model():
        return orc.Model(2, 256, 384, 2, 1, 8, 2, 512, 4, 8, seed=77)

    toks = np.array([1, 7, 300, 511], np.int32)
    pos = np.zeros(4, np.int32)
    a = model()
    _, _, xa = a.decode_step(toks, pos, orc.FP32, want_x=True)
    own, gap = a.route_info()
    assert own.shape == (2, 4, 2) and np.all(gap >= 0)
    b = model()
    b.force_routes(own)
    _, _, xb = b.decode_step(toks, pos, orc.FP32, want_x=True)
    assert np.array_equal(xa.view(np.uint32), xb.view(np.uint32))
    alt = own.copy()
    alt[1, 2] = [(own[1, 2, 0] + 1) % 8 if (own[1, 2, 0] + 1) % 8 != own[1, 2, 1] else (own[1, 2, 0] + 2) % 8,
                 own[1, 2, 1]]
    c = model()
    c.force_routes(alt)
    _, _, xc = c.decode_step(toks, pos, orc.FP32, want_x=True)
    assert np.array_equal(xc[[0, 1, 3]], xa[[0, 1, 3]]) and not np.array_equal(xc[2], xa[2])
    bad = own.copy()
    bad[0, 0, 0] = 8
    d = model()
    d.force_routes(bad)
    with pytest.raises(AssertionError):
        d.decode_step(toks, pos, orc.FP32)
