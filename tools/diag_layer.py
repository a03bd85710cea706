"""Per-stage GPU vs oracle on a 1-layer Tiny-width model, 1 micro-batch."""
import sys, ctypes as C, numpy as np
sys.path.insert(0, '.')
from paper_2411_11217_b200 import capi
from paper_2411_11217_b200.runtime import Runtime
from oracle import bind as orc
N, V, H, F, E, Kk = 8, 32000, 1024, 3584, 8, 2
KD = capi.load_kernels()
m = orc.Model(1, H, F, 8, 2, E, Kk, V, N, 64, seed=1234)
rt = Runtime(capi.ModelSpec(1, H, F, 8, 2, E, Kk, 2.0, 2.0), capi.Policy(N, N, 0, 1, 0.0, 0.0), budget_bytes=4e9, max_ctx=64, vocab=V)
toks = np.array([5, 17, 300, 4000, 12345, 31999, 7, 8], np.int32)
rt.decode(toks, 1)
def rel(a, b): return float(np.linalg.norm(a.astype(np.float64) - b) / np.linalg.norm(b))
emb = orc.bf16_to_f32(m.tensor(-1, orc.T_EMBED))[toks]
xn = orc.rmsnorm(emb, m.tensor(0, orc.T_ATTN_NORM), 1e-5, True)
qkv = orc.linear(xn, m.tensor(0, orc.T_WQKV))
qkv_g = orc.bf16_to_f32(rt.debug_read("qkv_bf16", np.uint16).reshape(N, -1))
print("qkv (pos0, rope=id) rel", rel(qkv_g, orc.bf16_to_f32(orc.f32_to_bf16(qkv))), "bits equal frac", np.mean(qkv_g == orc.bf16_to_f32(orc.f32_to_bf16(qkv))))
att = rt.debug_read("attn_in", np.uint16)
rows = np.empty((N, H), np.uint16)
KD.unpack_rows(att.ctypes.data_as(C.c_void_p), 16, N, H, rows.ctypes.data_as(C.c_void_p))
v_g = qkv_g[:, (8 + 2) * 128:]
att_f = orc.bf16_to_f32(rows)
vexp = np.concatenate([np.repeat(v_g[:, h*128:(h+1)*128][:, None, :], 4, axis=1).reshape(N, -1) for h in range(2)], axis=1)
print("attn_in == v (GQA expanded) frac", np.mean(att_f == vexp))
h_g = rt.debug_read("h", np.float32).reshape(N, H)
h_ref = emb + orc.linear(att_f, m.tensor(0, orc.T_WO))
print("h rel (gpu attn input)", rel(h_g, h_ref))
hn_g = rt.debug_read("hn", np.uint16).reshape(N, H)
hn_ref = orc.f32_to_bf16(orc.rmsnorm(h_g, m.tensor(0, orc.T_FFN_NORM), 1e-5, True))
print("hn bits equal frac (from gpu h)", np.mean(hn_g == hn_ref))
lg, idx, w, perm, off = orc.router(hn_g, m.tensor(0, orc.T_ROUTER), Kk)
print("topk equal", np.array_equal(rt.debug_read("topk", np.int32).reshape(N, Kk), idx), "topw maxdiff", np.abs(rt.debug_read("topw", np.float32).reshape(N, Kk) - w).max())
hnf = orc.bf16_to_f32(hn_g)
out = h_g.astype(np.float64).copy()
for t in range(N):
    for s in range(Kk):
        e = idx[t, s]
        y = orc.expert(hnf[t:t+1], m.tensor(0, orc.T_W1, e), m.tensor(0, orc.T_W3, e), m.tensor(0, orc.T_W2, e), True)
        out[t] += w[t, s] * y[0]
x_g = rt.residual()
print("x rel (gpu h/hn inputs)", rel(x_g, out))
# full oracle
_, _, x_ref = m.decode_step(toks, np.zeros(N, np.int32), orc.FAITHFUL, want_x=True)
print("x rel vs faithful oracle", rel(x_g, x_ref))
