"""Caller-owned weights (mlt_runtime_create_with_weights) and the codec's
per-block raw fallback (VERDICT r1 "what's weak" 8).

The weights are NOT the synthetic uniform ones: Student-t (nu = 4) entries,
with outlier rows (x 30) in every fourth 128-row block — the heavy tails and
outlier channels a real checkpoint has, which the 15-entry high-byte table
cannot always hold.  With
the codec on, every 128-row block with a tile of more than 31 escapes is
stored raw (tagged page-table entry) instead of aborting the runtime.
Checked:
  * the runtime builds, reports raw blocks (some, not all) and the achieved
    stored bytes per weight;
  * decoding is bit-identical to the same weights with every block raw
    (MLT_CODEC_FORCE_RAW=1): the in-kernel decode is exact on these values;
  * against the CPU oracle holding the same caller weights (teacher-forced on
    the GPU's routes): residual within BASELINE's 2e-2 every step (the x30
    outlier channels make bf16 activations round coarser than with the
    synthetic weights' 3e-3), ids equal except at lm-head near-ties.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_11217_b200 import capi  # noqa: E402
from paper_2411_11217_b200 import runtime as rtm  # noqa: E402

N, MU, STEPS, VOCAB = 8, 4, 12, 32000
L, H, F, NQ, NKV, E, K = 2, 1024, 3584, 8, 2, 8, 2
D = H // NQ
LM_TIE = 0.05


def _bf16(a):
    from oracle import bind as orc
    return orc.f32_to_bf16(np.asarray(a, np.float32))


def heavy_tailed_weights(seed=2024):
    rng = np.random.default_rng(seed)
    shapes = {rtm.W_EMBED: (VOCAB, H), rtm.W_LM_HEAD: (VOCAB, H), rtm.W_FINAL_NORM: (H,),
              rtm.W_ATTN_NORM: (H,), rtm.W_FFN_NORM: (H,), rtm.W_QKV: ((NQ + 2 * NKV) * D, H),
              rtm.W_O: (H, NQ * D), rtm.W_ROUTER: (E, H), rtm.W_W1: (F, H), rtm.W_W3: (F, H),
              rtm.W_W2: (H, F)}
    out = {}

    def t_matrix(shape, fan_in):
        w = rng.standard_t(4.0, size=shape).astype(np.float32) / np.sqrt(fan_in) * 0.7
        rows = np.arange(shape[0])
        w[((rows // 128) % 4 == 1) & (rows % 41 == 0)] *= 30.0  # outlier rows in some blocks
        return _bf16(w)

    for layer in range(-1, L):
        kinds = [rtm.W_EMBED, rtm.W_LM_HEAD, rtm.W_FINAL_NORM] if layer < 0 else \
            [rtm.W_ATTN_NORM, rtm.W_FFN_NORM, rtm.W_QKV, rtm.W_O, rtm.W_ROUTER]
        for kind in kinds:
            shp = shapes[kind]
            if kind in (rtm.W_FINAL_NORM, rtm.W_ATTN_NORM, rtm.W_FFN_NORM):
                out[(layer, kind, 0)] = _bf16(1.0 + 0.1 * rng.uniform(-1, 1, shp))
            elif kind == rtm.W_EMBED:
                out[(layer, kind, 0)] = _bf16(rng.standard_normal(shp))
            elif kind == rtm.W_LM_HEAD:
                out[(layer, kind, 0)] = _bf16(rng.standard_normal(shp) * 4.0 / np.sqrt(H))
            else:
                out[(layer, kind, 0)] = t_matrix(shp, shp[1])
        if layer >= 0:
            for e in range(E):
                for kind in (rtm.W_W1, rtm.W_W3, rtm.W_W2):
                    shp = shapes[kind]
                    out[(layer, kind, e)] = t_matrix(shp, shp[1])
    return out


@pytest.fixture(scope="module")
def weights():
    return heavy_tailed_weights()


def _runtime(weights, codec, force_raw=False):
    os.environ["MLT_CODEC_FORCE_RAW"] = "1" if force_raw else "0"
    try:
        return rtm.Runtime(capi.ModelSpec(L, H, F, NQ, NKV, E, K, 2.0, 2.0), capi.Policy(N, MU, 0, 1, 0.3, 0.0),
                           budget_bytes=4e9, max_ctx=64, vocab=VOCAB, weight_codec=codec,
                           weights=lambda layer, kind, expert: weights[(layer, kind, expert)])
    finally:
        os.environ.pop("MLT_CODEC_FORCE_RAW", None)


def test_codec_raw_fallback_on_heavy_tailed_weights(weights):
    from oracle import bind as orc
    toks = np.random.default_rng(5678).integers(0, VOCAB, size=(STEPS, N), dtype=np.int32)
    runs = []
    for force_raw in (False, True):
        rt = _runtime(weights, True, force_raw)
        info = rt.info
        ids, xs, routes = [], [], []
        for s in range(STEPS):
            rt.capture_router(1)
            d = rt.decode(toks[s], 1)
            assert d.report.timeline_ok == 1
            ids.append(d.ids[0].copy())
            xs.append(rt.residual())
            routes.append(rt.captured_router()[1])
        runs.append((info, np.array(ids), np.array(xs), np.array(routes)))
        rt.close()
    (info, ids, xs, routes), (info_raw, ids_r, xs_r, _) = runs
    total_blocks = (NQ + 2 * NKV) * D // 128 + H // 128 + E * (2 * F // 128 + H // 128)
    print(f"\n[heavy-tailed weights] codec: {info.raw_blocks:.0f} of {total_blocks} blocks per layer stored raw, "
          f"{info.bytes_per_weight:.4f} B/weight (all-raw: {info_raw.bytes_per_weight:.4f}); "
          f"streamed {info.streamed_bytes_per_layer / 1e6:.1f} vs {info_raw.streamed_bytes_per_layer / 1e6:.1f} MB/layer")
    assert 0 < info.raw_blocks < total_blocks
    assert info_raw.raw_blocks == total_blocks and info_raw.bytes_per_weight == 2.0
    assert 1.5 < info.bytes_per_weight < 2.0
    assert info.codec_engine == 3  # heavy tails: the 11-bit code's capacity rule falls back to the 12-bit code
    assert np.array_equal(ids, ids_r) and np.array_equal(xs.view(np.uint32), xs_r.view(np.uint32))

    # the oracle on the same caller weights, forced onto the GPU's routes
    m = orc.Model(L, H, F, NQ, NKV, E, K, VOCAB, N, 64, seed=1234)
    for (layer, kind, expert), a in weights.items():
        m.set_tensor(layer, kind, expert, a)
    worst = 0.0
    for s in range(STEPS):
        m.force_routes(routes[s])
        nxt, mg, x = m.decode_step(toks[s], np.full(N, s, np.int32), orc.FAITHFUL, want_x=True)
        rel = np.linalg.norm(xs[s] - x, axis=1) / np.linalg.norm(x, axis=1)
        worst = max(worst, float(rel.max()))
        assert rel.max() <= 2e-2, (s, float(rel.max()))
        for q in np.nonzero(ids[s] != nxt)[0]:
            assert mg[q] < LM_TIE, (s, int(q), float(mg[q]))
    print(f"[heavy-tailed weights] vs oracle (same weights, GPU routes): worst residual {worst:.2e}")


def test_caller_weights_without_codec_match_oracle(weights):
    """mlt_runtime_create_with_weights on bf16 tiles (no codec) also matches
    the oracle holding the same weights; a missing tensor is MLT_ERR_INVALID."""
    from oracle import bind as orc
    rt = _runtime(weights, False)
    m = orc.Model(L, H, F, NQ, NKV, E, K, VOCAB, N, 64, seed=1234)
    for (layer, kind, expert), a in weights.items():
        m.set_tensor(layer, kind, expert, a)
    toks = np.random.default_rng(99).integers(0, VOCAB, size=(4, N), dtype=np.int32)
    for s in range(4):
        rt.capture_router(1)
        d = rt.decode(toks[s], 1)
        m.force_routes(rt.captured_router()[1])
        _, _, x = m.decode_step(toks[s], np.full(N, s, np.int32), orc.FAITHFUL, want_x=True)
        rel = np.linalg.norm(rt.residual() - x, axis=1) / np.linalg.norm(x, axis=1)
        assert rel.max() <= 2e-2 and d.report.timeline_ok == 1
    rt.close()
    partial = {k: v for k, v in weights.items() if k[1] != rtm.W_W2}
    with pytest.raises(capi.MltError, match="no tensor"):
        rtm.Runtime(capi.ModelSpec(L, H, F, NQ, NKV, E, K, 2.0, 2.0), capi.Policy(N, MU, 0, 1, 0.3, 0.0),
                    budget_bytes=4e9, max_ctx=64, vocab=VOCAB,
                    weights=lambda layer, kind, expert: partial[(layer, kind, expert)])
