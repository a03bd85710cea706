"""Diagnostics: GPU runtime vs oracle (faithful / fp32) on the Tiny config."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2411_11217_b200 import capi
from paper_2411_11217_b200.runtime import Runtime
from oracle import bind as orc
N, V = 8, 32000
prompt = np.random.default_rng(5678).integers(0, V, size=(16, N), dtype=np.int32)
model = capi.ModelSpec(2, 1024, 3584, 8, 2, 8, 2, 2.0, 2.0)
for lm_scale in (4.0,):
    mf = orc.Model(2, 1024, 3584, 8, 2, 8, 2, V, N, 64, seed=1234, lm_head_scale=lm_scale)
    m32 = orc.Model(2, 1024, 3584, 8, 2, 8, 2, V, N, 64, seed=1234, lm_head_scale=lm_scale)
    rt = Runtime(model, capi.Policy(N, 4, 0, 1, 0.0, 0.0), budget_bytes=4e9, max_ctx=64, vocab=V, seed=1234, lm_head_scale=lm_scale)
    for s in range(16):
        nf, mgf, xf = mf.decode_step(prompt[s], np.full(N, s, np.int32), orc.FAITHFUL, want_x=True)
        n3, mg3, x3 = m32.decode_step(prompt[s], np.full(N, s, np.int32), orc.FP32, want_x=True)
        d = rt.decode(prompt[s], 1)
        xg = rt.residual()
        relf = np.linalg.norm(xg - xf) / np.linalg.norm(xf)
        rel3 = np.linalg.norm(xg - x3) / np.linalg.norm(x3)
        relfo = np.linalg.norm(xf - x3) / np.linalg.norm(x3)
        print(f"step {s}: rel(gpu,faithful)={relf:.2e} rel(gpu,fp32)={rel3:.2e} rel(faithful,fp32)={relfo:.2e} "
              f"ids gpu==faithful {np.sum(d.ids[0]==nf)}/8 ==fp32 {np.sum(d.ids[0]==n3)}/8 minmargin {mgf.min():.3f} "
              f"tl_ok={d.report.timeline_ok} tok/s={d.report.tokens_per_second:.0f}")
