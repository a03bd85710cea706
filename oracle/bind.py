"""TEST INFRASTRUCTURE — ctypes binding of the CPU numerical oracle
(oracle/liboracle.so, oracle_numerics.c).  Importable only by tests/,
__graft_entry__.smoke() and bench.py's CPU legs; the product never loads it.
The reference has no numerical path; the numerics are pinned against
transformers' MixtralForCausalLM golden vectors (tests/test_oracle_golden_hf.py,
see oracle_numerics.h)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liboracle.so")

FP32, FAITHFUL = 0, 1
T_EMBED, T_LM_HEAD, T_FINAL_NORM, T_ATTN_NORM, T_FFN_NORM, T_WQKV, T_WO, T_ROUTER, T_W1, \
    T_W3, T_W2 = range(11)


class OrcConfig(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("layers", "hidden", "ffn", "q_heads", "kv_heads",
                                         "experts", "top_k", "vocab", "batch", "max_ctx")] + \
               [("rms_eps", C.c_float), ("rope_theta", C.c_float), ("lm_head_scale", C.c_float),
                ("seed", C.c_uint64)]


V, I, F = C.c_void_p, C.c_int, C.c_float
_SIGS = {
    "orc_tensor_id": (C.c_uint64, [I, I, I]),
    "orc_gen_bf16": (None, [C.c_uint64, C.c_uint64, C.c_int64, F, I, V]),
    "orc_router": (None, [V, V, I, I, I, I, V, V, V, V, V]),
    "orc_rmsnorm": (None, [V, V, I, I, F, I, V]),
    "orc_attention": (None, [V, V, V, V, I, I, I, I, I, V]),
    "orc_linear": (None, [V, V, I, I, I, V]),
    "orc_linear_scalar": (None, [V, V, I, I, I, V]),
    "orc_expert": (None, [V, V, V, V, I, I, I, I, V]),
    "orc_rope": (None, [V, V, I, I, I, F]),
    "orc_model_create": (V, [C.POINTER(OrcConfig)]),
    "orc_model_free": (None, [V]),
    "orc_model_tensor": (V, [V, I, I, I]),
    "orc_decode_step": (I, [V, V, V, I, V, V, V]),
    "orc_layer_forward": (I, [V, I, V, V, I, V]),
    "orc_fill_kv": (None, [V, C.c_uint64, I]),
    "orc_model_kv": (V, [V, I, I]),
    "orc_num_threads": (I, []),
    "orc_router_margins": (None, [V, V]),
    "orc_model_force_routes": (None, [V, V]),
    "orc_model_set_tensor": (I, [V, I, I, I, V]),
    "orc_model_route_info": (None, [V, V, V]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(SO):
            raise ImportError(f"{SO} missing: make -C oracle")
        _lib = C.CDLL(SO)
        for n, (r, a) in _SIGS.items():
            f = getattr(_lib, n)
            f.restype, f.argtypes = r, a
    return _lib


def p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.c_void_p)


def gen_bf16(seed, tid, n, scale, is_norm=False) -> np.ndarray:
    out = np.empty(n, dtype=np.uint16)
    lib().orc_gen_bf16(seed, tid, n, scale, int(is_norm), p(out))
    return out


def tensor_id(layer, kind, expert=0) -> int:
    return lib().orc_tensor_id(layer, kind, expert)


def bf16_to_f32(a: np.ndarray) -> np.ndarray:
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def router(hn_bf16: np.ndarray, w_bf16: np.ndarray, K: int):
    T, H = hn_bf16.shape
    E = w_bf16.shape[0]
    logits = np.zeros((T, E), np.float32)
    idx = np.zeros((T, K), np.int32)
    wts = np.zeros((T, K), np.float32)
    perm = np.zeros(T * K, np.int32)
    off = np.zeros(E + 1, np.int32)
    lib().orc_router(p(np.ascontiguousarray(hn_bf16)), p(np.ascontiguousarray(w_bf16)), T, H, E,
                     K, p(logits), p(idx), p(wts), p(perm), p(off))
    return logits, idx, wts, perm, off


def linear(x: np.ndarray, w_bf16: np.ndarray) -> np.ndarray:
    T, K = x.shape
    M = w_bf16.shape[0]
    y = np.zeros((T, M), np.float32)
    lib().orc_linear(p(np.ascontiguousarray(x, np.float32)), p(np.ascontiguousarray(w_bf16)), T,
                     K, M, p(y))
    return y


def expert(x, w1, w3, w2, round_bf16=False):
    T, H = x.shape
    Fd = w1.shape[0]
    y = np.zeros((T, H), np.float32)
    lib().orc_expert(p(np.ascontiguousarray(x, np.float32)), p(w1), p(w3), p(w2), T, H, Fd,
                     int(round_bf16), p(y))
    return y


def rmsnorm(x, gamma_bf16, eps, round_bf16=False):
    T, H = x.shape
    out = np.zeros((T, H), np.float32)
    lib().orc_rmsnorm(p(np.ascontiguousarray(x, np.float32)), p(gamma_bf16), T, H, eps,
                      int(round_bf16), p(out))
    return out


def rope(x, pos, n_heads, d, theta):
    x = np.ascontiguousarray(x, np.float32).copy()
    lib().orc_rope(p(x), p(np.ascontiguousarray(pos, np.int32)), x.shape[0], n_heads, d, theta)
    return x


def attention(q, k, v, ctx, n_q, n_kv, d):
    """q [T, n_q*d] f32; k, v [T, cap, n_kv, d] bf16; ctx [T]."""
    T, cap = k.shape[0], k.shape[1]
    out = np.zeros((T, n_q * d), np.float32)
    lib().orc_attention(p(np.ascontiguousarray(q, np.float32)), p(np.ascontiguousarray(k)),
                        p(np.ascontiguousarray(v)), p(np.ascontiguousarray(ctx, np.int32)), T,
                        n_q, n_kv, d, cap, p(out))
    return out


class Model:
    """Whole synthetic model (weights generated from the shared PRNG)."""

    def __init__(self, layers, hidden, ffn, q_heads, kv_heads, experts, top_k, vocab, batch,
                 max_ctx, seed=1234, eps=1e-5, theta=1e6, lm_head_scale=4.0):
        self.cfg = OrcConfig(layers, hidden, ffn, q_heads, kv_heads, experts, top_k, vocab, batch,
                             max_ctx, eps, theta, lm_head_scale, seed)
        self.h = lib().orc_model_create(C.byref(self.cfg))

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_model_free(self.h)
            self.h = None

    def tensor(self, layer, kind, expert=0, shape=None) -> np.ndarray:
        c = self.cfg
        d = c.hidden // c.q_heads
        shapes = {T_EMBED: (c.vocab, c.hidden), T_LM_HEAD: (c.vocab, c.hidden),
                  T_FINAL_NORM: (c.hidden,), T_ATTN_NORM: (c.hidden,), T_FFN_NORM: (c.hidden,),
                  T_WQKV: ((c.q_heads + 2 * c.kv_heads) * d, c.hidden),
                  T_WO: (c.hidden, c.hidden), T_ROUTER: (c.experts, c.hidden),
                  T_W1: (c.ffn, c.hidden), T_W3: (c.ffn, c.hidden), T_W2: (c.hidden, c.ffn)}
        shp = shape or shapes[kind]
        ptr = lib().orc_model_tensor(self.h, layer, kind, expert)
        n = int(np.prod(shp))
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint16)), shape=(n,)).reshape(shp).copy()

    def decode_step(self, tokens, pos, mode=FAITHFUL, want_x=False):
        N = self.cfg.batch
        nxt = np.zeros(N, np.int32)
        margin = np.zeros(N, np.float32)
        x = np.zeros((N, self.cfg.hidden), np.float32) if want_x else None
        rc = lib().orc_decode_step(self.h, p(np.ascontiguousarray(tokens, np.int32)),
                                   p(np.ascontiguousarray(pos, np.int32)), mode, p(nxt), p(margin),
                                   p(x) if want_x else None)
        assert rc == 0, "oracle decode_step failed"
        return (nxt, margin, x) if want_x else (nxt, margin)

    def layer_forward(self, layer, x, pos, mode=FP32):
        x = np.ascontiguousarray(x, np.float32).copy()
        idx = np.zeros((self.cfg.batch, self.cfg.top_k), np.int32)
        rc = lib().orc_layer_forward(self.h, layer, p(x), p(np.ascontiguousarray(pos, np.int32)),
                                     mode, p(idx))
        assert rc == 0
        return x, idx

    def router_margins(self) -> np.ndarray:
        """Per sequence, min over layers of the last step's routing gap
        (k-th selected logit minus best unselected)."""
        out = np.zeros(self.cfg.batch, np.float32)
        lib().orc_router_margins(self.h, p(out))
        return out

    def set_tensor(self, layer, kind, expert, data):
        """Overwrite a model tensor with caller weights (bf16 bits, same shape)."""
        a = np.ascontiguousarray(data, np.uint16)
        assert lib().orc_model_set_tensor(self.h, layer, kind, expert, p(a)) == 0

    def force_routes(self, topk):
        """Take these routes ([L, N, K] int32) in every following step (None: own routing)."""
        if topk is None:
            self._routes = None
            lib().orc_model_force_routes(self.h, None)
            return
        self._routes = np.ascontiguousarray(topk, np.int32)  # kept alive while borrowed
        c = self.cfg
        assert self._routes.shape == (c.layers, c.batch, c.top_k)
        lib().orc_model_force_routes(self.h, p(self._routes))

    def route_info(self):
        """(own top-k [L, N, K], gap [L, N]) of the last step."""
        c = self.cfg
        idx = np.zeros((c.layers, c.batch, c.top_k), np.int32)
        gap = np.zeros((c.layers, c.batch), np.float32)
        lib().orc_model_route_info(self.h, p(idx), p(gap))
        return idx, gap

    def fill_kv(self, seed, upto):
        lib().orc_fill_kv(self.h, seed, upto)

    def kv(self, layer, which):
        c = self.cfg
        d = c.hidden // c.q_heads
        n = c.batch * c.max_ctx * c.kv_heads * d
        ptr = lib().orc_model_kv(self.h, layer, which)
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_uint16)), shape=(n,)).reshape(
            c.batch, c.max_ctx, c.kv_heads, d)
