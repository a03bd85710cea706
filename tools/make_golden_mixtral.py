"""Golden vectors for the CPU numerical oracle from an independent Mixtral
implementation: Hugging Face transformers' MixtralForCausalLM (fp32, eager,
CPU), loaded with the oracle's own synthetic bf16-valued weights, with the KV
cache and the router input rounded to bf16 like the oracle's (bf16_kv_cache).  The
reference (MoE-Lightning's planner) has no numerical path, so this pins the
oracle's "per public Mixtral" semantics (RMSNorm eps 1e-5,
rotate-half RoPE theta 1e6, GQA, softmax top-2 router renormalised over the
k, SiLU-gated experts, weighted combine) against the canonical model code.

  python tools/make_golden_mixtral.py [--config toy|baseline_tiny]
      toy           -> tests/golden/mixtral_hf_tiny.npz (2 layers, h1 512, 4 experts, vocab 1000:
                       every position's full logits)
      baseline_tiny -> tests/golden/mixtral_hf_baseline_tiny.npz (BASELINE configs[0]: 2 layers,
                       h1 1024, h2 3584, n_q 8, n_kv 2, 8 experts top-2, vocab 32000: every
                       position's top-64 logits with their ids, to keep the fixture small)

The committed fixture is what tests/test_oracle_golden_hf.py checks; this
script needs transformers (in this container) and is not run by the tests.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import bind as orc  # noqa: E402

CONFIGS = {
    "toy": dict(layers=2, hidden=512, ffn=384, q_heads=4, kv_heads=2, experts=4, top_k=2, vocab=1000),
    "baseline_tiny": dict(layers=2, hidden=1024, ffn=3584, q_heads=8, kv_heads=2, experts=8, top_k=2, vocab=32000),
}
CFG = dict(CONFIGS["toy"])
N, PROMPT, GEN, SEED = 3, 10, 6, 1234
TOPK = 64


def oracle_model(max_ctx=PROMPT + GEN + 2):
    c = CFG
    return orc.Model(c["layers"], c["hidden"], c["ffn"], c["q_heads"], c["kv_heads"], c["experts"], c["top_k"],
                     c["vocab"], N, max_ctx, seed=SEED)


def hf_model(m):
    from transformers import MixtralConfig, MixtralForCausalLM
    c = CFG
    cfg = MixtralConfig(vocab_size=c["vocab"], hidden_size=c["hidden"], intermediate_size=c["ffn"],
                        num_hidden_layers=c["layers"], num_attention_heads=c["q_heads"],
                        num_key_value_heads=c["kv_heads"], num_local_experts=c["experts"],
                        num_experts_per_tok=c["top_k"], rope_theta=1e6, rms_norm_eps=1e-5,
                        max_position_embeddings=64, tie_word_embeddings=False, attn_implementation="eager")
    hf = MixtralForCausalLM(cfg).eval()
    f = lambda a: torch.from_numpy(orc.bf16_to_f32(a).astype(np.float32))  # noqa: E731
    d = c["hidden"] // c["q_heads"]
    nq, nkv = c["q_heads"] * d, c["kv_heads"] * d
    sd = {"model.embed_tokens.weight": f(m.tensor(-1, orc.T_EMBED)), "lm_head.weight": f(m.tensor(-1, orc.T_LM_HEAD)),
          "model.norm.weight": f(m.tensor(-1, orc.T_FINAL_NORM))}
    for l in range(c["layers"]):
        p = f"model.layers.{l}."
        qkv = f(m.tensor(l, orc.T_WQKV))
        sd[p + "self_attn.q_proj.weight"] = qkv[:nq]
        sd[p + "self_attn.k_proj.weight"] = qkv[nq:nq + nkv]
        sd[p + "self_attn.v_proj.weight"] = qkv[nq + nkv:]
        sd[p + "self_attn.o_proj.weight"] = f(m.tensor(l, orc.T_WO))
        sd[p + "mlp.gate.weight"] = f(m.tensor(l, orc.T_ROUTER))
        sd[p + "mlp.experts.gate_up_proj"] = torch.stack(
            [torch.cat([f(m.tensor(l, orc.T_W1, e)), f(m.tensor(l, orc.T_W3, e))]) for e in range(c["experts"])])
        sd[p + "mlp.experts.down_proj"] = torch.stack([f(m.tensor(l, orc.T_W2, e)) for e in range(c["experts"])])
        sd[p + "input_layernorm.weight"] = f(m.tensor(l, orc.T_ATTN_NORM))
        sd[p + "post_attention_layernorm.weight"] = f(m.tensor(l, orc.T_FFN_NORM))
    hf.load_state_dict(sd, strict=True)
    return hf


def bf16_kv_cache(hf):
    """The oracle (like the product) keeps K (after RoPE) and V in a bf16 cache
    and routes on the bf16 normalised hidden state, while q and every other
    activation stay fp32: round HF's tensors at the same three points."""
    from transformers.models.mixtral import modeling_mixtral as mm
    rope = mm.apply_rotary_pos_emb

    def rope_bf16_k(q, k, *a, **kw):
        qe, ke = rope(q, k, *a, **kw)
        return qe, ke.to(torch.bfloat16).float()
    mm.apply_rotary_pos_emb = rope_bf16_k
    for layer in hf.model.layers:
        layer.self_attn.v_proj.register_forward_hook(lambda mod, inp, out: out.to(torch.bfloat16).float())
        # the router reads the bf16 normalised hidden state (the GPU router's
        # exact input); the experts read it in fp32
        layer.mlp.gate.register_forward_pre_hook(lambda mod, inp: (inp[0].to(torch.bfloat16).float(),))


def main():
    import argparse
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="toy", choices=sorted(CONFIGS))
    a = ap.parse_args()
    CFG.clear()
    CFG.update(CONFIGS[a.config])
    torch.manual_seed(0)
    m = oracle_model()
    hf = hf_model(m)
    bf16_kv_cache(hf)
    prompt = np.random.default_rng(5678).integers(0, CFG["vocab"], (N, PROMPT)).astype(np.int64)
    ids = torch.from_numpy(prompt)
    with torch.no_grad():
        for _ in range(GEN):  # greedy, full recompute (tiny)
            nxt = hf(ids).logits[:, -1].argmax(-1, keepdim=True)
            ids = torch.cat([ids, nxt], 1)
        logits = hf(ids[:, :-1]).logits.float().numpy()  # every position's next-token logits
    import transformers
    meta = dict(prompt=prompt.astype(np.int32), ids=ids.numpy().astype(np.int32), seed=SEED,
                transformers=transformers.__version__, torch=torch.__version__, **{k: v for k, v in CFG.items()})
    if a.config == "toy":
        out = os.path.join(ROOT, "tests", "golden", "mixtral_hf_tiny.npz")
        np.savez_compressed(out, logits=logits.astype(np.float32), **meta)
    else:  # top-64 logits per position (+ their ids) and each position's logit range
        out = os.path.join(ROOT, "tests", "golden", f"mixtral_hf_{a.config}.npz")
        top = np.argsort(-logits, axis=-1)[..., :TOPK]
        np.savez_compressed(out, top_ids=top.astype(np.int32),
                            top_logits=np.take_along_axis(logits, top, -1).astype(np.float32),
                            logit_range=np.abs(logits).max(-1).astype(np.float32), **meta)
    print("wrote", out, logits.shape, "greedy", ids[:, PROMPT:].tolist())


if __name__ == "__main__":
    main()
