"""End-to-end decode on the B200 through the runtime C ABI vs the CPU oracle
(BASELINE.json correctness items 2 and 3; config 1 "Tiny": l=2, h1=1024,
h2=3584, n_q=8, n_kv=2, n_e=8, k=2, vocab 32000, N=8, mu=4, prompt 16 +
32 greedy steps, weights seed 1234, prompt seed 5678).

Greedy parity.  The GPU keeps activations in bf16 between kernels and its
tensor cores accumulate with ~4e-6 relative error (measured,
tools/diag_gemm.py), so values sitting on a bf16 rounding boundary flip one
ulp against any CPU reference; the resulting logit noise is ~1e-3 of the
logit scale.  The test therefore runs both sides FREE-RUNNING for 32 steps
and requires every divergence to start at a step whose oracle top1-top2
margin is below NEAR_TIE (a genuine near-tie; a real bug diverges at large
margins and fails), plus a sanity floor of half the sequences identical for
all 32 steps (measured: 6/8 at seed 5678, both divergences at margins
< 0.02).  The per-stage test below pins each kernel boundary bit-for-bit or
to ~1e-5 on identical inputs.
"""
import ctypes as C

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_11217_b200 import capi  # noqa: E402
from paper_2411_11217_b200.runtime import Runtime  # noqa: E402

N, MU, PROMPT, GEN, VOCAB = 8, 4, 16, 32, 32000
NEAR_TIE = 0.05  # logit units; logits have std ~4 (lm_head_scale 4)


def tiny_model(layers=2):
    return capi.ModelSpec(layers, 1024, 3584, 8, 2, 8, 2, 2.0, 2.0)


def oracle_model(layers=2, batch=N):
    from oracle import bind as orc
    return orc.Model(layers, 1024, 3584, 8, 2, 8, 2, VOCAB, batch, 64, seed=1234)


@pytest.fixture(scope="module")
def prompt():
    return np.random.default_rng(5678).integers(0, VOCAB, size=(PROMPT, N), dtype=np.int32)


@pytest.fixture(scope="module")
def oracle_run(prompt):
    from oracle import bind as orc
    m = oracle_model()
    ids, margins = [], []
    tok = prompt[0]
    for s in range(PROMPT + GEN - 1):
        tok = prompt[s] if s < PROMPT else tok
        nxt, mg = m.decode_step(tok, np.full(N, s, np.int32), orc.FAITHFUL)
        if s >= PROMPT - 1:
            ids.append(nxt)
            margins.append(mg)
        tok = nxt
    return np.array(ids), np.array(margins)


def run_gpu(prompt, r_w, a_g):
    pol = capi.Policy(N, MU, a_g, 1, r_w, 1.0 if a_g else 0.0)
    rt = Runtime(tiny_model(), pol, budget_bytes=4e9, max_ctx=64, vocab=VOCAB, seed=1234)
    first = rt.decode(prompt[0], PROMPT, forced=prompt)
    rest = rt.decode(first.ids[-1], GEN - 1)
    return rt, first, rest, np.array([first.ids[-1]] + list(rest.ids))


@pytest.mark.parametrize("r_w,a_g", [(0.0, 0), (0.5, 0), (1.0, 1)])
def test_tiny_greedy_32_steps(prompt, oracle_run, r_w, a_g):
    ref, margins = oracle_run
    rt, first, rest, gen = run_gpu(prompt, r_w, a_g)
    assert first.report.timeline_ok == 1 and rest.report.timeline_ok == 1
    exact = 0
    for s in range(N):
        bad = np.nonzero(gen[:, s] != ref[:, s])[0]
        if bad.size == 0:
            exact += 1
            continue
        k = bad[0]
        assert margins[k, s] < NEAR_TIE, (
            f"seq {s} diverges at step {k} with oracle margin {margins[k, s]:.4f} >= {NEAR_TIE}")
    print(f"\n[greedy] r_w={r_w} A_g={a_g}: {exact}/8 sequences identical for 32 steps; "
          f"min oracle margin {margins.min():.4f}")
    assert exact >= N // 2  # sanity floor; the near-tie check above is the real gate
    # paging volume: every step streams each layer's non-resident blocks once
    info = rt.info
    layer_bytes = 2 * 1024 * 1536 + 2 * 1024 * 1024 + 8 * 3 * 1024 * 3584 * 2 + 8 * 1024 * 2
    # residency is decided per 128-row block: at most one block (128 x h2 x 2 B) short
    assert info.streamed_bytes_per_layer <= (1 - r_w) * layer_bytes + 128 * 3584 * 2
    assert rest.report.h2d_weight_bytes == pytest.approx((GEN - 1) * 2 * info.streamed_bytes_per_layer)


def test_tiny_layer_output_within_2e2_of_fp32(prompt):
    """BASELINE item 2: layer outputs within 2e-2 relative (bf16 GPU vs fp32 CPU)."""
    from oracle import bind as orc
    m = oracle_model()
    rt = Runtime(tiny_model(), capi.Policy(N, MU, 0, 1, 0.25, 0.0), budget_bytes=4e9,
                 max_ctx=64, vocab=VOCAB, seed=1234)
    worst = 0.0
    for s in range(4):
        _, _, x_ref = m.decode_step(prompt[s], np.full(N, s, np.int32), orc.FP32, want_x=True)
        rt.decode(prompt[s], 1)
        x = rt.residual()
        worst = max(worst, np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
    assert worst <= 2e-2, worst


def test_one_layer_stage_by_stage():
    """Each kernel boundary of one decoder layer against the oracle fed with
    the GPU's own inputs: bf16 outputs bit-equal except rounding-boundary
    ulps, router indices exact, fp32 outputs ~1e-5."""
    from oracle import bind as orc
    KD = capi.load_kernels()
    H, E, Kk = 1024, 8, 2
    m = oracle_model(layers=1)
    rt = Runtime(tiny_model(layers=1), capi.Policy(N, N, 0, 1, 0.0, 0.0), budget_bytes=4e9,
                 max_ctx=64, vocab=VOCAB)
    toks = np.array([5, 17, 300, 4000, 12345, 31999, 7, 8], np.int32)
    rt.decode(toks, 1)

    def rel(a, b):
        return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))

    emb = orc.bf16_to_f32(m.tensor(-1, orc.T_EMBED))[toks]
    xn = orc.rmsnorm(emb, m.tensor(0, orc.T_ATTN_NORM), 1e-5, True)
    qkv = orc.bf16_to_f32(orc.f32_to_bf16(orc.linear(xn, m.tensor(0, orc.T_WQKV))))
    qkv_g = orc.bf16_to_f32(rt.debug_read("qkv_bf16", np.uint16).reshape(N, -1))
    assert np.mean(qkv_g == qkv) > 0.998 and rel(qkv_g, qkv) < 1e-4
    att = rt.debug_read("attn_in", np.uint16)
    rows = np.empty((N, H), np.uint16)
    KD.unpack_rows(att.ctypes.data_as(C.c_void_p), 16, N, H, rows.ctypes.data_as(C.c_void_p))
    att_f = orc.bf16_to_f32(rows)
    v = qkv_g[:, 10 * 128:]
    v_exp = np.concatenate([np.repeat(v[:, h * 128:(h + 1) * 128][:, None, :], 4, axis=1)
                            .reshape(N, -1) for h in range(2)], axis=1)
    assert np.array_equal(att_f, v_exp)  # position 0: attention output == v (host attention)
    h_g = rt.debug_read("h", np.float32).reshape(N, H)
    assert rel(h_g, emb + orc.linear(att_f, m.tensor(0, orc.T_WO))) < 1e-5
    hn_g = rt.debug_read("hn", np.uint16).reshape(N, H)
    hn_ref = orc.f32_to_bf16(orc.rmsnorm(h_g, m.tensor(0, orc.T_FFN_NORM), 1e-5, True))
    assert np.mean(hn_g == hn_ref) > 0.999
    _, idx, w, _, _ = orc.router(hn_g, m.tensor(0, orc.T_ROUTER), Kk)
    assert np.array_equal(rt.debug_read("topk", np.int32).reshape(N, Kk), idx)
    assert np.allclose(rt.debug_read("topw", np.float32).reshape(N, Kk), w, rtol=1e-6, atol=1e-7)
    hnf = orc.bf16_to_f32(hn_g)
    out = h_g.astype(np.float64).copy()
    for t in range(N):
        for s in range(Kk):
            e = idx[t, s]
            y = orc.expert(hnf[t:t + 1], m.tensor(0, orc.T_W1, e), m.tensor(0, orc.T_W3, e),
                           m.tensor(0, orc.T_W2, e), True)
            out[t] += w[t, s] * y[0]
    assert rel(rt.residual(), out) < 1e-4
