"""8x7B-width, 2 layers: GPU vs faithful oracle per step under teacher forcing."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_2411_11217_b200 import capi
from paper_2411_11217_b200.runtime import Runtime
from oracle import bind as orc
N, V = 8, 32000
prompt = np.random.default_rng(5678).integers(0, V, size=(16, N), dtype=np.int32)
ref = orc.Model(2, 4096, 14336, 32, 8, 8, 2, V, N, 64, seed=1234)
rt = Runtime(capi.ModelSpec(2, 4096, 14336, 32, 8, 8, 2, 2.0, 2.0), capi.Policy(N, 4, 0, 1, 0.10, 0.0),
             budget_bytes=7e9, max_ctx=64, vocab=V, seed=1234)
tok = prompt[0]
for s in range(30):
    tok = prompt[s] if s < 16 else tok
    nxt, mg, xr = ref.decode_step(tok, np.full(N, s, np.int32), orc.FAITHFUL, want_x=True)
    d = rt.decode(tok, 1)
    xg = rt.residual()
    per_seq = np.linalg.norm(xg - xr, axis=1) / np.linalg.norm(xr, axis=1)
    print(f"step {s:2d}: max rel {per_seq.max():.2e} (seq {per_seq.argmax()}), ids eq {np.sum(d.ids[0]==nxt)}/8, "
          f"min margin {mg.min():.3f}, mism margins {mg[d.ids[0]!=nxt]}")
    tok = nxt
