"""GPU prefill through the runtime C ABI vs the CPU
oracle.

The oracle has no separate prefill: it runs the prompt through its decode
step one position at a time (PAPER.md:166 — prefill computes exactly the
prompt's K/V and the first generated token), which is the same math as the
GPU's chunked causal prefill.  Checked, on ragged prompts:
  * the KV cache the GPU prefill writes (host cache for A_g = 0, paged device
    pool for A_g = 1) against the oracle's, every layer, every prompt
    position: relative error <= 1e-2 (bf16 values from tensor-core fp32
    accumulation against CPU fp32 with bf16 rounding at the same points);
  * the first generated token of every prompt: equal to the oracle's unless
    the oracle's top1-top2 logit margin is < LM_TIE or a router near-tie
    (< ROUTER_TIE) occurred on that prompt (same attribution as
    tests/test_decode_gpu.py);
  * decode continued from the prefilled state (teacher-forced on the oracle's
    greedy tokens): residual within 1e-2 and ids attributable, as above.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_11217_b200 import capi  # noqa: E402
from paper_2411_11217_b200.runtime import Runtime  # noqa: E402

N, MU, VOCAB, CTX, GEN = 8, 4, 32000, 64, 8
LM_TIE, ROUTER_TIE = 0.05, 0.02
TINY = (1024, 3584, 8, 2)
W8X7B = (4096, 14336, 32, 8)
LENS = [16, 9, 23, 3, 12, 16, 1, 7]


def _prompts(lens, seed=5678):
    rng = np.random.default_rng(seed)
    return [rng.integers(0, VOCAB, size=n, dtype=np.int32) for n in lens]


def _oracle_prefill(ref, prompts):
    """Prompt positions through the oracle; returns first ids, lm margins at
    the last prompt position, the min router margin over each prompt, and the
    router margin of every (sequence, position)."""
    from oracle import bind as orc
    lens = [len(p) for p in prompts]
    first = np.zeros(N, np.int32)
    lm = np.zeros(N, np.float32)
    rmin = np.full(N, np.inf, np.float32)
    rpos = np.full((N, max(lens)), np.inf, np.float32)
    for s in range(max(lens)):
        tok = np.array([p[s] if s < len(p) else 0 for p in prompts], np.int32)
        nxt, margin = ref.decode_step(tok, np.full(N, s, np.int32), orc.FAITHFUL)
        rm = ref.router_margins()
        for q in range(N):
            if s < lens[q]:
                rmin[q] = min(rmin[q], rm[q])
                rpos[q, s] = rm[q]
            if s == lens[q] - 1:
                first[q], lm[q] = nxt[q], margin[q]
    return first, lm, rmin, rpos


def _kv_check(rt, ref, dims, lens, a_g, layers, rpos):
    """Per layer and prompt, relative error over the positions whose residual
    no router near-tie has touched: K/V at (layer l, position p) depend on
    the residual at p after layers < l, which a near-tie at p can flip
    (rpos = min over layers of the oracle's routing gap at p)."""
    h1, h2, nq, nkv = dims
    d = 128
    worst = 0.0
    from oracle import bind as orc
    for which, name in ((0, "k"), (1, "v")):
        if a_g == 0:
            kc = rt.debug_read(name + "cache", np.uint16).reshape(layers, N, nkv, CTX, d)
        else:
            page = 16
            mp = CTX // page
            pool = rt.debug_read(name + "pool", np.uint16).reshape(layers, N, mp, nkv, page, d)
            # undo the token-row chunk swizzle (common.cuh kv_page_off): chunk c of
            # token r is stored at c ^ (r & 7)
            idx = np.arange(d // 8)[None, :] ^ (np.arange(page)[:, None] & 7)  # [page][chunk]
            pool = np.take_along_axis(pool.reshape(layers, N, mp, nkv, page, d // 8, 8),
                                      idx[None, None, None, None, :, :, None], axis=5).reshape(
                layers, N, mp, nkv, page, d)
            kc = pool.transpose(0, 1, 3, 2, 4, 5).reshape(layers, N, nkv, mp * page, d)
        for l in range(layers):
            ok = ref.kv(l, which)  # [N][max_ctx][nkv][d]
            for q in range(N):
                n = lens[q]
                clean = rpos[q, :n] >= ROUTER_TIE if l > 0 else np.ones(n, bool)
                got = orc.bf16_to_f32(kc[l, q, :, :n].transpose(1, 0, 2))[clean]
                exp = orc.bf16_to_f32(ok[q, :n])[clean]
                rel = np.linalg.norm(got - exp) / max(np.linalg.norm(exp), 1e-30)
                worst = max(worst, rel)
                assert rel <= 1e-2, (name, l, q, rel)
    return worst


def _run(dims, r_w, a_g, budget, lens, layers=2, chunk=0, warm=False):
    from oracle import bind as orc
    h1, h2, nq, nkv = dims
    model = capi.ModelSpec(layers, h1, h2, nq, nkv, 8, 2, 2.0, 2.0)
    ref = orc.Model(layers, h1, h2, nq, nkv, 8, 2, VOCAB, N, CTX, seed=1234)
    prompts = _prompts(lens)
    rt = Runtime(model, capi.Policy(N, MU, a_g, 1, r_w, 1.0 if a_g else 0.0), budget_bytes=budget,
                 max_ctx=CTX, vocab=VOCAB, seed=1234, prefill_chunk_tokens=chunk)
    if warm:  # an earlier prefill on the same runtime: buffers reused, KV overwritten
        rt.prefill(_prompts(lens, seed=1))
    first, rep = rt.prefill(prompts)
    assert rep.prompt_tokens == sum(lens) and rep.seconds > 0 and rep.gpu_launches > 0
    o_first, o_lm, o_rmin, o_rpos = _oracle_prefill(ref, prompts)
    mism = 0
    for q in range(N):
        if first[q] != o_first[q]:
            mism += 1
            assert o_lm[q] < LM_TIE or o_rmin[q] < ROUTER_TIE, (q, first[q], o_first[q], o_lm[q], o_rmin[q])
    worst_kv = _kv_check(rt, ref, dims, lens, a_g, layers, o_rpos)
    # decode continues at each prompt's length, teacher-forced on the oracle's tokens
    tok = o_first.copy()
    pos = np.array(lens, np.int32)
    for s in range(GEN):
        nxt, lm_m, x_ref = ref.decode_step(tok, pos + s, orc.FAITHFUL, want_x=True)
        rm = ref.router_margins()
        out = rt.decode(tok, 1)
        x = rt.residual()
        rel = np.linalg.norm(x - x_ref, axis=1) / np.linalg.norm(x_ref, axis=1)
        for q in range(N):
            if rm[q] >= ROUTER_TIE and o_rmin[q] >= ROUTER_TIE:
                assert rel[q] <= 1e-2, (s, q, rel[q])
            if out.ids[0][q] != nxt[q]:
                assert lm_m[q] < LM_TIE or rm[q] < ROUTER_TIE or o_rmin[q] < ROUTER_TIE, (s, q)
        tok = nxt
    print(f"\n[prefill {dims} r_w={r_w} A_g={a_g}] first-id mismatches {mism}/{N}, worst KV rel "
          f"{worst_kv:.2e}, {rep.prompt_tokens} tokens in {rep.seconds * 1e3:.2f} ms, "
          f"chunk {rep.chunk_tokens} x {rep.chunks_per_layer}")
    return rep


@pytest.mark.parametrize("r_w,a_g", [(0.25, 0), (0.0, 1), (1.0, 0)])
def test_tiny_prefill_matches_oracle(r_w, a_g):
    _run(TINY, r_w, a_g, 4e9, LENS)


def test_8x7b_width_prefill_matches_oracle():
    _run(W8X7B, 0.10, 0, 7e9, LENS)


def test_prefill_uniform_prompts_second_call():
    """Uniform prompts; a second prefill on the same runtime reuses the chunk
    buffers and overwrites the KV."""
    _run(TINY, 0.5, 0, 4e9, [20] * N, warm=True)


@pytest.mark.parametrize("a_g", [0, 1])
def test_prefill_small_chunks(a_g):
    """32-token chunks: several chunks per layer, so the double-buffered
    residual/KV copies and chunk metadata alternate within a layer."""
    rep = _run(TINY, 0.25 if a_g == 0 else 0.0, a_g, 4e9, LENS, chunk=32)
    assert rep.chunk_tokens == 32 and rep.chunks_per_layer >= 4


@pytest.mark.parametrize("a_g,r_w", [(0, 0.3), (1, 1.0)])
def test_prefill_with_weight_codec_bitwise_equal(a_g, r_w):
    """GPU prefill on encoded weights: same first tokens, same KV cache bits and
    same decode continuation as the same runtime with every block stored as a
    raw fallback block (MLT_CODEC_FORCE_RAW=1: same GEMMs, no decode)."""
    import os
    dims = (1024, 3584, 8, 2)
    lens = [17, 40, 33, 8, 56, 1, 25, 48]
    prompts = _prompts(lens)
    outs = []
    for force_raw in (True, False):
        os.environ["MLT_CODEC_FORCE_RAW"] = "1" if force_raw else "0"
        try:
            rt = Runtime(capi.ModelSpec(2, *dims, 8, 2, 2.0, 2.0),
                         capi.Policy(N, MU, a_g, 1, r_w, 1.0 if a_g else 0.0),
                         budget_bytes=4e9, max_ctx=CTX, vocab=VOCAB, seed=1234, weight_codec=True)
        finally:
            os.environ.pop("MLT_CODEC_FORCE_RAW", None)
        first, _ = rt.prefill(prompts)
        if a_g:  # paged pool [layer][seq][page][kv_head][16][d]: pages past a prompt hold stale bytes
            kv = [rt.debug_read(n, np.uint16).reshape(2, N, CTX // 16, dims[3], 16, 128) for n in ("kpool", "vpool")]
            kv = [np.concatenate([a[:, q, :(lens[q] + 15) // 16].reshape(2, -1) for q in range(N)], axis=1)
                  for a in kv]
        else:  # host cache [layer][seq][kv_head][ctx][d]: compare the prompt positions only
            kv = [rt.debug_read(n, np.uint16).reshape(2, N, dims[3], CTX, 128) for n in ("kcache", "vcache")]
            kv = [np.concatenate([a[:, q, :, :lens[q]].reshape(2, -1) for q in range(N)], axis=1) for a in kv]
        nxt = rt.decode(first, 3)
        outs.append((first.copy(), kv, nxt.ids.copy()))
        rt.close()
    (f0, kv0, n0), (f1, kv1, n1) = outs
    assert np.array_equal(f0, f1) and np.array_equal(n0, n1)
    assert all(np.array_equal(a, b) for a, b in zip(kv0, kv1))
