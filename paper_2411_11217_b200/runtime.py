"""Python handle on the native decode runtime (mlt_runtime_* in include/mlt.h).

Plumbing only: every byte of compute happens in libmlt.so.  Mirrors the
reference's vocabulary: a `Runtime` is built from a ModelSpec and a Policy
(proj/include/lightplan/config.hpp:24-56) and `decode()` returns the greedy
ids plus the measured per-layer LatencyBreakdown (planner.hpp:25-35).
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

import numpy as np

from . import capi


class RuntimeOptions(C.Structure):
    _fields_ = [("device", C.c_int32), ("budget_bytes", C.c_double), ("max_ctx", C.c_int32),
                ("host_threads", C.c_int32), ("pin_weights", C.c_int32), ("vocab", C.c_int32),
                ("rms_eps", C.c_float), ("rope_theta", C.c_float), ("lm_head_scale", C.c_float),
                ("seed", C.c_uint64), ("exact_gates", C.c_int32), ("tp_rank", C.c_int32),
                ("tp_size", C.c_int32), ("nccl_id", C.c_uint8 * 128), ("schedule", C.c_int32),
                ("prefill_chunk_tokens", C.c_int32), ("tp_shard_only", C.c_int32),
                ("weight_codec", C.c_int32), ("disable_pdl", C.c_int32), ("collective", C.c_int32),
                ("expert_down_splits", C.c_int32)]


def host_collective_name() -> bytes:
    """Rendezvous key of a host-staged collective group (collective="host"):
    rank 0 creates it, the launcher broadcasts it like an ncclUniqueId."""
    import secrets
    return f"mlt_coll_{os.getpid()}_{secrets.token_hex(8)}".encode()


def nccl_unique_id() -> bytes:
    """ncclUniqueId for a tensor-parallel group (rank 0 creates, launcher broadcasts)."""
    api = capi.load_product()
    f = api.lib.mlt_nccl_unique_id
    f.restype, f.argtypes = C.c_int, [C.c_void_p]
    buf = (C.c_uint8 * 128)()
    api.check(f(buf))
    return bytes(buf)


class DecodeReport(C.Structure):
    _fields_ = [("seconds", C.c_double), ("tokens_per_second", C.c_double),
                ("measured", capi.LatencyBreakdown), ("h2d_weight_bytes", C.c_double),
                ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double),
                ("steady_layer_time", C.c_double), ("utilization", C.c_double * 5),
                ("gpu_launches", C.c_int32), ("timeline_ok", C.c_int32),
                ("expert_ms_total", C.c_double), ("expert_launches", C.c_int32),
                ("dense_ms_total", C.c_double), ("dense_launches", C.c_int32)]


class PrefillReport(C.Structure):
    _fields_ = [("seconds", C.c_double), ("tokens_per_second", C.c_double),
                ("prompt_tokens", C.c_int64), ("chunk_tokens", C.c_int32),
                ("chunks_per_layer", C.c_int32), ("h2d_weight_bytes", C.c_double),
                ("h2d_bytes", C.c_double), ("d2h_bytes", C.c_double),
                ("gpu_busy_seconds", C.c_double), ("gpu_launches", C.c_int32)]


class RuntimeInfo(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("achieved_weight_ratio", "streamed_bytes_per_layer",
                                          "arena_used", "arena_capacity", "pin_seconds",
                                          "gen_seconds", "bytes_per_weight", "raw_blocks",
                                          "codec_engine")]


# mlt_weight_fn: const uint16_t* get(void* ctx, int layer, int kind, int expert)
WEIGHT_FN = C.CFUNCTYPE(C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int)
# tensor kinds of mlt_runtime_create_with_weights (runtime/host_layout.hpp TensorKind)
W_EMBED, W_LM_HEAD, W_FINAL_NORM, W_ATTN_NORM, W_FFN_NORM, W_QKV, W_O, W_ROUTER, W_W1, W_W3, W_W2 = range(11)


_SIGS = {
    "runtime_create_with_weights": (C.c_void_p, [C.POINTER(capi.ModelSpec), C.POINTER(capi.Policy),
                                                 C.POINTER(RuntimeOptions), WEIGHT_FN, C.c_void_p]),
    "runtime_create": (C.c_void_p, [C.POINTER(capi.ModelSpec), C.POINTER(capi.Policy),
                                    C.POINTER(RuntimeOptions)]),
    "runtime_destroy": (None, [C.c_void_p]),
    "runtime_info": (C.c_int, [C.c_void_p, C.POINTER(RuntimeInfo)]),
    "runtime_prefill_synthetic": (C.c_int, [C.c_void_p, C.c_int, C.c_uint64]),
    "runtime_set_positions": (C.c_int, [C.c_void_p, C.c_void_p]),
    "runtime_prefill": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(PrefillReport)]),
    "runtime_decode": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                 C.POINTER(DecodeReport)]),
    "runtime_timeline_json": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "runtime_read_residual": (C.c_int, [C.c_void_p, C.c_void_p]),
    "runtime_debug_read": (C.c_int, [C.c_void_p, C.c_char_p, C.c_void_p, C.c_size_t]),
    "runtime_capture_router": (C.c_int, [C.c_void_p, C.c_int]),
    "runtime_execute": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.POINTER(DecodeReport)]),
}


def _fns():
    api = capi.load_product()
    out = {}
    for n, (r, a) in _SIGS.items():
        f = getattr(api.lib, "mlt_" + n)
        f.restype, f.argtypes = r, a
        out[n] = f
    return api, out


@dataclass
class Decoded:
    ids: np.ndarray          # [steps, N]
    report: DecodeReport


class Runtime:
    def __init__(self, model: capi.ModelSpec, policy: capi.Policy, *, budget_bytes: float,
                 max_ctx: int, vocab: int = 32000, seed: int = 1234, device: int = 0,
                 host_threads: int = 0, pin_weights: bool = True, rms_eps: float = 1e-5,
                 rope_theta: float = 1e6, lm_head_scale: float = 4.0, exact_gates: bool = True,
                 tp_rank: int = 0, tp_size: int = 1, nccl_id: bytes = b"", schedule: str = "auto",
                 prefill_chunk_tokens: int = 0, tp_shard_only: bool = False, weight_codec: bool = False,
                 pdl: bool = True, down_splits: int = 0, collective: str = "nccl", weights=None):
        """weights: optional callable (layer, kind, expert) -> bf16 bits (uint16
        ndarray, the FULL row-major tensor; kinds W_*) replacing the synthetic
        weights (mlt_runtime_create_with_weights)."""
        self.api, self.f = _fns()
        self.model, self.policy = model, policy
        nid = (C.c_uint8 * 128)(*(nccl_id.ljust(128, b"\0")[:128]))
        self.opts = RuntimeOptions(device, budget_bytes, max_ctx, host_threads, int(pin_weights),
                                   vocab, rms_eps, rope_theta, lm_head_scale, seed,
                                   int(exact_gates), tp_rank, tp_size, nid,
                                   -1 if schedule == "auto" else capi.SCHED[schedule],
                                   prefill_chunk_tokens, int(tp_shard_only), int(weight_codec), int(not pdl),
                                   {"nccl": 0, "host": 1}[collective], down_splits)
        if weights is None:
            self.h = self.f["runtime_create"](C.byref(model), C.byref(policy), C.byref(self.opts))
        else:
            held = []  # arrays handed to the C side stay alive until the call returns

            def get(_ctx, layer, kind, expert):
                try:
                    a = np.ascontiguousarray(weights(layer, kind, expert), dtype=np.uint16)
                except Exception:  # noqa: BLE001 - reported as a NULL tensor (MLT_ERR_INVALID)
                    return None
                held.append(a)
                return a.ctypes.data
            cb = WEIGHT_FN(get)
            self.h = self.f["runtime_create_with_weights"](C.byref(model), C.byref(policy), C.byref(self.opts),
                                                           cb, None)
            del held
        if not self.h:
            code = self.api.fn["last_status"]()
            raise capi._EXC.get(code, capi.MltError)(code, self.api.error())

    def close(self):
        if getattr(self, "h", None):
            self.f["runtime_destroy"](self.h)
            self.h = None

    __del__ = close

    def _ck(self, rc):
        return self.api.check(rc)

    @property
    def info(self) -> RuntimeInfo:
        out = RuntimeInfo()
        self._ck(self.f["runtime_info"](self.h, C.byref(out)))
        return out

    def prefill_synthetic(self, prompt_len: int, seed: int = 9012):
        self._ck(self.f["runtime_prefill_synthetic"](self.h, prompt_len, seed))

    def prefill(self, prompts):
        """GPU prefill of real prompts (mlt_runtime_prefill).  prompts: [N, s]
        array or a list of N 1-D id arrays (ragged).  Returns (first ids [N],
        PrefillReport); decode continues at each prompt's length."""
        if isinstance(prompts, np.ndarray) and prompts.ndim == 2:
            prompts = list(prompts)
        if len(prompts) != self.policy.batch:  # the C side reads exactly N lengths
            raise ValueError(f"prefill needs {self.policy.batch} prompts (policy.batch), got {len(prompts)}")
        lens = np.array([len(p) for p in prompts], np.int32)
        toks = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts]), np.int32)
        first = np.zeros(len(prompts), np.int32)
        rep = PrefillReport()
        self._ck(self.f["runtime_prefill"](self.h, toks.ctypes.data_as(C.c_void_p),
                                           lens.ctypes.data_as(C.c_void_p),
                                           first.ctypes.data_as(C.c_void_p), C.byref(rep)))
        return first, rep

    def set_positions(self, pos):
        pos = np.ascontiguousarray(pos, np.int32)
        self._ck(self.f["runtime_set_positions"](self.h, pos.ctypes.data_as(C.c_void_p)))

    def decode(self, tokens, steps: int, forced=None) -> Decoded:
        N = self.policy.batch
        tokens = np.ascontiguousarray(tokens, np.int32)
        if tokens.size != N:
            raise ValueError(f"decode needs {N} token ids (policy.batch), got {tokens.size}")
        tokens = tokens.reshape(N)
        out = np.zeros((steps, N), np.int32)
        rep = DecodeReport()
        fp = None
        if forced is not None:
            forced = np.ascontiguousarray(forced, np.int32).reshape(steps, N)
            fp = forced.ctypes.data_as(C.c_void_p)
        self._ck(self.f["runtime_decode"](self.h, tokens.ctypes.data_as(C.c_void_p), fp, steps,
                                          out.ctypes.data_as(C.c_void_p), C.byref(rep)))
        return Decoded(out, rep)

    def execute(self, dag, tokens, forced=None) -> Decoded:
        """sim::execute: run a caller-built schedule (a capi.Dag from
        Api.schedule_build for this model/policy) instead of the runtime's own."""
        N = self.policy.batch
        steps = max(t.step for t, _ in dag.tasks())
        tokens = np.ascontiguousarray(tokens, np.int32).reshape(N)
        out = np.zeros((steps, N), np.int32)
        rep = DecodeReport()
        fp = None
        if forced is not None:
            forced = np.ascontiguousarray(forced, np.int32).reshape(steps, N)
            fp = forced.ctypes.data_as(C.c_void_p)
        self._ck(self.f["runtime_execute"](self.h, dag.h, tokens.ctypes.data_as(C.c_void_p), fp,
                                           out.ctypes.data_as(C.c_void_p), C.byref(rep)))
        return Decoded(out, rep)

    def timeline(self) -> dict:
        n = self._ck(self.f["runtime_timeline_json"](self.h, None, 0))
        buf = C.create_string_buffer(n + 1)
        self.f["runtime_timeline_json"](self.h, buf, n + 1)
        return json.loads(buf.value.decode())

    def kernel_profile(self) -> list:
        f = self.api.lib.mlt_runtime_kernel_profile
        f.restype, f.argtypes = C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]
        n = self._ck(f(self.h, None, 0))
        buf = C.create_string_buffer(n + 1)
        f(self.h, buf, n + 1)
        return json.loads(buf.value.decode())

    def residual(self) -> np.ndarray:
        x = np.zeros((self.policy.batch, self.model.hidden_dim), np.float32)
        self._ck(self.f["runtime_read_residual"](self.h, x.ctypes.data_as(C.c_void_p)))
        return x

    def debug_read(self, name: str, dtype) -> np.ndarray:
        n = self._ck(self.f["runtime_debug_read"](self.h, name.encode(), None, 0))
        out = np.zeros(n // np.dtype(dtype).itemsize, dtype)
        self._ck(self.f["runtime_debug_read"](self.h, name.encode(), out.ctypes.data_as(C.c_void_p), n))
        return out

    def capture_router(self, step: int):
        """Arm the router tap for decode step `step` (1-based) of the next decode()."""
        self._ck(self.f["runtime_capture_router"](self.h, step))

    def captured_router(self):
        """(hn [L, N, H] u16, topk [L, N, K] i32, topw [L, N, K] f32) of the tapped step."""
        L, N = self.model.layers, self.policy.batch
        H, K = self.model.hidden_dim, self.model.top_k
        return (self.debug_read("cap_hn", np.uint16).reshape(L, N, H),
                self.debug_read("cap_topk", np.int32).reshape(L, N, K),
                self.debug_read("cap_topw", np.float32).reshape(L, N, K))
