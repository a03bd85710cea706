"""End-to-end decode on the B200 through the runtime C ABI vs the CPU oracle
(BASELINE.json correctness items 2 and 3).

Configs: "Tiny" (BASELINE configs[0]: l=2, h1=1024, h2=3584, n_q=8, n_kv=2,
n_e=8, k=2, vocab 32000) and the reduced-depth 8x7B-width model of SURVEY
§8c (l=2, h1=4096, h2=14336, n_q=32, n_kv=8).  N=8 sequences, mu=4, a
16-token prompt (seed 5678) + 32 greedy steps, weights seed 1234.

Greedy parity.  The GPU keeps activations in bf16 between kernels and its
tensor cores accumulate with ~4e-6 relative error (tools/diag_gemm.py), so
values on a bf16 rounding boundary flip one ulp against any CPU reference;
the residual drifts ~3e-3 from the bf16-faithful oracle.  That flips two
kinds of genuinely tied decisions: lm-head argmax near-ties and router
top-k near-ties (a flipped expert moves that token's residual by 10-30%).
So greedy parity is checked TEACHER-FORCED (the GPU decodes the oracle's own
greedy tokens, so one tie cannot cascade) and every discrepancy must be
attributable:
  * each greedy id equals the oracle's, unless the oracle's top1-top2 logit
    margin is < LM_TIE or a router near-tie (< ROUTER_TIE) occurred for that
    sequence at that step;
  * each per-step residual is within 1e-2 (relative) of the oracle, unless a
    router near-tie occurred at that step.
A real bug fails both (large margins, no ties).  The free-running 32-step
comparison is printed for information.
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
LM_TIE = 0.05      # logit units; logits have std ~4 (lm_head_scale 4)
ROUTER_TIE = 0.02  # router logit units (std ~1)
TINY = (1024, 3584, 8, 2)
W8X7B = (4096, 14336, 32, 8)


@pytest.fixture(scope="module")
def prompt():
    return np.random.default_rng(5678).integers(0, VOCAB, size=(PROMPT, N), dtype=np.int32)


def _model(dims, layers=2):
    h1, h2, nq, nkv = dims
    return capi.ModelSpec(layers, h1, h2, nq, nkv, 8, 2, 2.0, 2.0)


def _oracle(dims, layers=2):
    from oracle import bind as orc
    h1, h2, nq, nkv = dims
    return orc.Model(layers, h1, h2, nq, nkv, 8, 2, VOCAB, N, 64, seed=1234)


def teacher_forced_parity(dims, prompt, r_w, a_g, budget, weight_codec=False):
    """Teacher-forced decode, the oracle on the GPU's routes.  Each step the
    router tap returns the GPU's top-k at every layer; the bf16-faithful
    oracle is forced onto those routes (orc_model_force_routes), so a router
    near-tie cannot move one side onto other experts and EVERY sequence's
    residual is checked (<= 1e-2 relative).  Where the oracle's own free
    choice differs from the GPU's it must be a near-tie (gap < ROUTER_TIE);
    ids may differ only at lm-head near-ties (margin < LM_TIE)."""
    from oracle import bind as orc
    ref = _oracle(dims)
    rt = Runtime(_model(dims), capi.Policy(N, MU, a_g, 1, r_w, 1.0 if a_g else 0.0),
                 budget_bytes=budget, max_ctx=64, vocab=VOCAB, seed=1234, weight_codec=weight_codec)
    steps = PROMPT + GEN - 1
    tok = prompt[0]
    events = {"lm_tie": 0, "router_flips": 0, "ids": 0, "min_lm_margin": float("inf")}
    worst = 0.0
    for s in range(steps):
        tok = prompt[s] if s < PROMPT else tok
        rt.capture_router(1)
        out = rt.decode(tok, 1)
        assert out.report.timeline_ok == 1
        _, topk, _ = rt.captured_router()
        ref.force_routes(topk)
        nxt, lm_margin, x_ref = ref.decode_step(tok, np.full(N, s, np.int32), orc.FAITHFUL, want_x=True)
        own, gap = ref.route_info()
        flips = np.argwhere((np.sort(own, axis=2) != np.sort(topk, axis=2)).any(axis=2))
        events["router_flips"] += len(flips)
        for a, b in flips:
            assert gap[a, b] < ROUTER_TIE, (s, int(a), int(b), float(gap[a, b]))
        x = rt.residual()
        rel = np.linalg.norm(x - x_ref, axis=1) / np.linalg.norm(x_ref, axis=1)
        worst = max(worst, float(rel.max()))
        assert rel.max() <= 1e-2, (s, float(rel.max()))
        if s >= PROMPT - 1:
            events["min_lm_margin"] = min(events["min_lm_margin"], float(lm_margin.min()))
            for q in range(N):
                if out.ids[0][q] != nxt[q]:
                    events["ids"] += 1
                    events["lm_tie"] += 1
                    assert lm_margin[q] < LM_TIE, (f"step {s} seq {q}: id {out.ids[0][q]} vs oracle {nxt[q]} at "
                                                   f"lm margin {lm_margin[q]:.3f}")
        tok = nxt
    ref.force_routes(None)
    return rt, events, worst


def free_running(dims, prompt, r_w, a_g, budget):
    """Free-running greedy decode (BASELINE: greedy ids match for the first 32
    steps) against the bf16-faithful oracle running free too.  Asserted: for
    every sequence the GPU's ids equal the oracle's up to that sequence's
    first near-tie — an lm-head margin < LM_TIE or a router gap < ROUTER_TIE
    at any layer of that step — after which the two may legitimately part."""
    from oracle import bind as orc
    ref = _oracle(dims)
    ids, lm, rm = [], [], []
    tok = prompt[0]
    for s in range(PROMPT + GEN - 1):
        tok = prompt[s] if s < PROMPT else tok
        nxt, mg = ref.decode_step(tok, np.full(N, s, np.int32), orc.FAITHFUL)
        rm.append(ref.router_margins())
        if s >= PROMPT - 1:
            ids.append(nxt)
            lm.append(mg)
        tok = nxt
    rt = Runtime(_model(dims), capi.Policy(N, MU, a_g, 1, r_w, 1.0 if a_g else 0.0),
                 budget_bytes=budget, max_ctx=64, vocab=VOCAB, seed=1234)
    first = rt.decode(prompt[0], PROMPT, forced=prompt)
    rest = rt.decode(first.ids[-1], GEN - 1)
    gen = np.array([first.ids[-1]] + list(rest.ids))
    ids, lm, rm = np.array(ids), np.array(lm), np.array(rm)
    # per sequence: first generated step at or after which a near-tie occurred
    # (router ties during the prompt count from generated step 0)
    rtie = rm < ROUTER_TIE  # [PROMPT + GEN - 1, N]
    first_tie = []
    for q in range(N):
        cand = [GEN]
        if rtie[:PROMPT, q].any():
            cand.append(0)
        t_r = np.nonzero(rtie[PROMPT - 1:, q])[0]
        t_l = np.nonzero(lm[:, q] < LM_TIE)[0]
        cand += [int(t_r[0])] if t_r.size else []
        cand += [int(t_l[0])] if t_l.size else []
        first_tie.append(min(cand))
    first_div = [int(np.nonzero(gen[:, q] != ids[:, q])[0][0]) if (gen[:, q] != ids[:, q]).any()
                 else GEN for q in range(N)]
    for q in range(N):
        assert first_div[q] >= first_tie[q], (f"seq {q}: GPU ids leave the oracle's at generated step "
                                              f"{first_div[q]} before any near-tie (first at {first_tie[q]})")
    stats = {"first_divergence": first_div, "first_near_tie": first_tie,
             "sequences_identical_32_steps": int(sum(d == GEN for d in first_div)),
             "min_lm_margin": float(lm.min()), "min_router_gap": float(rm.min())}
    return rt, first, rest, stats


@pytest.mark.parametrize("r_w,a_g", [(0.0, 0), (0.5, 0), (1.0, 1)])
def test_tiny_greedy(prompt, r_w, a_g):
    rt, ev, worst = teacher_forced_parity(TINY, prompt, r_w, a_g, 4e9)
    print(f"\n[tiny r_w={r_w} A_g={a_g}] teacher-forced (oracle on the GPU's routes): {ev}, worst residual "
          f"{worst:.2e}")
    assert ev["ids"] <= 4
    rt2, first, rest, st = free_running(TINY, prompt, r_w, a_g, 4e9)
    print(f"[tiny r_w={r_w} A_g={a_g}] free-running: {st}")
    assert first.report.timeline_ok == 1 and rest.report.timeline_ok == 1
    # paging volume: every step streams each layer's non-resident blocks once
    info = rt2.info
    layer_bytes = 2 * 1024 * 1536 + 2 * 1024 * 1024 + 8 * 3 * 1024 * 3584 * 2 + 8 * 1024 * 2
    # residency is decided per 128-row block: at most one block (128 x h2 x 2 B) short
    assert info.streamed_bytes_per_layer <= (1 - r_w) * layer_bytes + 128 * 3584 * 2
    assert rest.report.h2d_weight_bytes == pytest.approx((GEN - 1) * 2 * info.streamed_bytes_per_layer)


@pytest.mark.parametrize("a_g", [0, 1])
def test_8x7b_width_reduced_depth_greedy(prompt, a_g):
    """Reduced-depth 8x7B-width model: paged at r_w=0.10
    under a 7 GB cap with host attention, resident with GPU attention;
    teacher-forced on the GPU's routes and free-running for 32 steps."""
    r_w, budget = (0.10, 7e9) if a_g == 0 else (1.0, 12e9)
    rt, ev, worst = teacher_forced_parity(W8X7B, prompt, r_w, a_g, budget)
    print(f"\n[8x7B-width l=2 A_g={a_g}] teacher-forced (oracle on the GPU's routes): {ev}, worst residual "
          f"{worst:.2e}")
    assert ev["ids"] <= 6
    rt.close()
    rt2, first, rest, st = free_running(W8X7B, prompt, r_w, a_g, budget)
    print(f"[8x7B-width l=2 A_g={a_g}] free-running: {st}")
    assert first.report.timeline_ok == 1 and rest.report.timeline_ok == 1


SK = (1024, 2432, 8, 2)  # 8 experts x 19 row blocks = 152 gate/up tiles: a 4-tile last wave on 148 SMs


@pytest.mark.parametrize("r_w,a_g", [(0.0, 0), (1.0, 1)])
def test_gateup_stream_k_tail_parity(prompt, r_w, a_g):
    """The gate/up GEMM's stream-K tail (gemm_tc.cu: the 4 tiles of the partial
    last wave split 8 ways along K; every part sums all parts in order for its
    slice of rows, SiLU after) against the fp32 oracle: residual within the
    Tiny model's bar, greedy ids equal except at bf16-vs-fp32 near-ties."""
    rt, ev, worst = teacher_forced_parity(SK, prompt, r_w, a_g, 4e9)
    print(f"\n[stream-K tail r_w={r_w} A_g={a_g}] teacher-forced: {ev}, worst residual {worst:.2e}")
    assert worst <= 1e-2 and ev["ids"] <= ev["lm_tie"]


def test_tiny_layer_output_within_2e2_of_fp32(prompt):
    """BASELINE item 2: layer outputs within 2e-2 relative (bf16 GPU vs fp32 CPU)."""
    from oracle import bind as orc
    m = _oracle(TINY)
    rt = Runtime(_model(TINY), capi.Policy(N, MU, 0, 1, 0.25, 0.0), budget_bytes=4e9,
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
    H, Kk = 1024, 2
    m = _oracle(TINY, layers=1)
    rt = Runtime(_model(TINY, layers=1), capi.Policy(N, N, 0, 1, 0.0, 0.0), budget_bytes=4e9,
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


def test_executed_baseline_schedules_match_cgopipe(prompt):
    """S2 / S3 (pipesim.cpp s2/s3: whole-layer transfers, no page pipelining)
    run through the same executor and kernels as CGOPipe: only the issue order
    and dependencies change, so ids and the residual are bit-identical."""
    outs = {}
    for kind in ("cgopipe", "s2", "s3"):
        rt = Runtime(_model(TINY), capi.Policy(N, MU, 0, 1, 0.25, 0.0), budget_bytes=4e9, max_ctx=64,
                     vocab=VOCAB, seed=1234, schedule=kind)
        first = rt.decode(prompt[0], PROMPT, forced=prompt)
        rest = rt.decode(first.ids[-1], 8)
        assert first.report.timeline_ok == 1 and rest.report.timeline_ok == 1
        assert rest.report.h2d_weight_bytes == pytest.approx(8 * 2 * rt.info.streamed_bytes_per_layer)
        outs[kind] = (np.asarray(first.ids), np.asarray(rest.ids), rt.residual())
    for kind in ("s2", "s3"):
        for a, b in zip(outs[kind], outs["cgopipe"]):
            assert np.array_equal(a, b), kind
    with pytest.raises(capi.UnsupportedCombinationError):
        Runtime(_model(TINY), capi.Policy(N, MU, 0, 1, 0.25, 0.0), budget_bytes=4e9, max_ctx=64,
                vocab=VOCAB, seed=1234, schedule="s4")


@pytest.mark.parametrize("mode", ["1", "2", "3", "4"])
@pytest.mark.parametrize("dims,r_w,a_g,budget", [(TINY, 0.3, 0, 4e9), (TINY, 1.0, 1, 4e9), (SK, 0.5, 0, 4e9),
                                                 (W8X7B, 0.10, 0, 7e9)])
def test_weight_codec_decode_bitwise_equal(prompt, dims, r_w, a_g, budget, mode):
    """Decoding with encoded weights (stored, paged and read as 12432-byte
    tiles; codec 1 = tcgen05 with in-smem decoders, codec 2 = the register-
    decode mma.sync GEMM, codec 3 = decode into TMEM; codec 4 = the 3-bit code
    on the TMEM engine, 11600-byte tiles, the default) returns the same ids
    and residual bits as the same runtime with every block stored as a raw
    fallback block (MLT_CODEC_FORCE_RAW=1: bf16 tiles through the same GEMMs,
    no decode), while the pages carry 24 % fewer bytes — the in-kernel decode
    is exact."""
    import os
    out = []
    for force_raw in (True, False):
        os.environ["MLT_CODEC_FORCE_RAW"] = "1" if force_raw else "0"
        os.environ["MLT_CODEC_MODE"] = mode
        try:
            rt = Runtime(_model(dims), capi.Policy(N, MU, a_g, 1, r_w, 1.0 if a_g else 0.0), budget_bytes=budget,
                         max_ctx=64, vocab=VOCAB, seed=1234, weight_codec=True)
        finally:
            os.environ.pop("MLT_CODEC_FORCE_RAW", None)
            os.environ.pop("MLT_CODEC_MODE", None)
        assert rt.info.codec_engine == int(mode)
        first = rt.decode(prompt[0], PROMPT, forced=prompt)
        rest = rt.decode(first.ids[-1], 8)
        out.append((first.ids.copy(), rest.ids.copy(), rt.residual().copy(), rt.info.streamed_bytes_per_layer,
                    rest.report.h2d_weight_bytes))
        assert rest.report.timeline_ok == 1
        rt.close()
    (f0, r0, x0, s0, b0), (f1, r1, x1, s1, b1) = out
    assert np.array_equal(f0, f1) and np.array_equal(r0, r1)
    assert np.array_equal(x0.view(np.uint32), x1.view(np.uint32))
    if r_w < 1.0:
        ratio = 11600 / 16384 if mode == "4" else 12432 / 16384
        assert s1 < (ratio + 0.04) * s0 and b1 < (ratio + 0.04) * b0  # + block-granular residency


@pytest.mark.parametrize("dims,r_w,a_g,budget", [(TINY, 0.3, 0, 4e9), (W8X7B, 0.10, 0, 7e9)])
def test_weight_codec_parity_vs_oracle(prompt, dims, r_w, a_g, budget):
    """The encoded-weight decode path (register-decode GEMMs) against the
    oracle: teacher-forced on the GPU's routes, every residual within 1e-2,
    ids equal except at lm-head near-ties."""
    rt, ev, worst = teacher_forced_parity(dims, prompt, r_w, a_g, budget, weight_codec=True)
    print(f"\n[codec {dims[0]} r_w={r_w}] teacher-forced: {ev}, worst residual {worst:.2e}")
    assert ev["ids"] <= 4


def test_tp_shard_only_measurement_mode(prompt):
    """tp_shard_only: one rank's shard of a tp=2 job runs alone (all-reduce
    elided): it decodes, streams half of each layer's paged bytes, and its
    measured timeline still verifies.  (Values are partial sums by design.)"""
    model = _model(TINY)
    full = Runtime(model, capi.Policy(N, MU, 0, 1, 0.0, 0.0), budget_bytes=4e9, max_ctx=64, vocab=VOCAB, seed=1234)
    shard = Runtime(model, capi.Policy(N, MU, 0, 1, 0.0, 0.0), budget_bytes=4e9, max_ctx=64, vocab=VOCAB, seed=1234,
                    tp_rank=1, tp_size=2, tp_shard_only=True)
    for rt in (full, shard):
        rt.prefill_synthetic(PROMPT, 9012)
    d = shard.decode(prompt[0], 3)
    assert d.report.timeline_ok == 1 and d.ids.shape == (3, N)
    assert shard.info.streamed_bytes_per_layer == pytest.approx(full.info.streamed_bytes_per_layer / 2, rel=0.02)
    full.close()
    shard.close()


def test_bad_inputs_rejected_before_the_device(prompt):
    """Token ids outside [0, vocab) (decode inputs, teacher-forced ids and
    prefill prompts) and unsupported GQA group sizes fail loudly with
    invalid-argument instead of reaching the kernels."""
    rt = Runtime(_model(TINY), capi.Policy(N, MU, 0, 1, 0.0, 0.0), budget_bytes=4e9, max_ctx=64, vocab=VOCAB,
                 seed=1234)
    bad = prompt[0].copy()
    bad[3] = VOCAB
    with pytest.raises(capi.MltError, match="token id"):
        rt.decode(bad, 1)
    bad[3] = -1
    with pytest.raises(capi.MltError, match="token id"):
        rt.decode(prompt[0], 2, forced=np.stack([prompt[0], bad]))
    with pytest.raises(capi.MltError, match="token id"):
        rt.prefill([np.array([1, 2, VOCAB + 5], np.int32)] * N)
    with pytest.raises(ValueError):
        rt.prefill([np.array([1, 2], np.int32)] * (N - 1))
    d = rt.decode(prompt[0], 1)  # the runtime is still usable
    assert d.report.timeline_ok == 1
    rt.close()
    # G = 32 / 1 = 32 query heads per kv head: beyond the host kernel's 16
    with pytest.raises(capi.MltError, match="q_heads / kv_heads"):
        Runtime(capi.ModelSpec(2, 4096, 3584, 32, 1, 8, 2, 2.0, 2.0), capi.Policy(N, MU, 0, 1, 0.0, 0.0),
                budget_bytes=4e9, max_ctx=64, vocab=VOCAB)
    # G = 3 on the GPU attention path (templated for 1/2/4/6/8)
    with pytest.raises(capi.MltError, match="q_heads / kv_heads"):
        Runtime(capi.ModelSpec(2, 768, 3584, 6, 2, 8, 2, 2.0, 2.0), capi.Policy(N, MU, 1, 1, 1.0, 1.0),
                budget_bytes=4e9, max_ctx=64, vocab=VOCAB)
