"""ctypes mirror of include/mlt.h (the C ABI of the B200 decode hot path).

The Python side is plumbing only: tests and bench.py call the C ABI through
these bindings exactly as a reference maintainer's ctypes stub would
(INTEGRATION.md).  `bind(lib, prefix)` binds either the product library
(prefix "mlt_") or the reference shim built under oracle/_ref (prefix "ref_",
tests only) with the same struct layouts.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

_HERE = os.path.dirname(os.path.abspath(__file__))
# MLT_LIB overrides the library (diagnostic builds of the same sources, tools/)
LIB_PATH = os.environ.get("MLT_LIB") or os.path.join(_HERE, "libmlt.so")

MLT_OK = 0
ERRORS = {-1: "invalid argument", -2: "infeasible policy", -3: "unsupported combination",
          -4: "cycle detected", -5: "empty timeline", -6: "cuda error", -7: "budget exceeded",
          -8: "internal error"}


class MltError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class InfeasiblePolicyError(MltError):
    pass


class UnsupportedCombinationError(MltError):
    pass


class CycleDetectedError(MltError):
    pass


class EmptyTimelineError(MltError):
    pass


class NoFeasiblePolicyError(MltError):
    pass


_EXC = {-2: InfeasiblePolicyError, -3: UnsupportedCombinationError, -4: CycleDetectedError,
        -5: EmptyTimelineError, -9: NoFeasiblePolicyError}
ERRORS[-9] = "no feasible policy"


class HardwareSpec(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("gpu_mem_bytes", "cpu_mem_bytes", "gpu_bw", "cpu_bw", "link_bw", "gpu_flops",
                 "cpu_flops")]


class ModelSpec(C.Structure):
    _fields_ = [(n, C.c_int64) for n in
                ("layers", "hidden_dim", "ffn_dim", "q_heads", "kv_heads", "experts", "top_k")] + \
               [("weight_dtype_bytes", C.c_double), ("kv_dtype_bytes", C.c_double)]

    def head_dim(self) -> int:
        return self.hidden_dim // self.q_heads if self.q_heads > 0 else 0


class WorkloadSpec(C.Structure):
    _fields_ = [("prompt_len", C.c_int64), ("gen_len", C.c_int64)]


class Policy(C.Structure):
    _fields_ = [("batch", C.c_int64), ("micro_batch", C.c_int64), ("attn_on_gpu", C.c_int32),
                ("ffn_on_gpu", C.c_int32), ("weights_on_gpu", C.c_double),
                ("kv_on_gpu", C.c_double)]

    def micro_batch_count(self) -> int:
        return self.batch // self.micro_batch if self.micro_batch > 0 else 0


class OpProfile(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("flops", "gpu_bytes", "cpu_bytes", "link_bytes")]


class LayerWeightBytes(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("experts", "qkv", "output", "router")]

    def total(self) -> float:
        return self.experts + self.qkv + self.output + self.router


class TransferSizes(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("qkv_offload", "hidden_upload", "weight_stream", "kv_upload")]


class LatencyBreakdown(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("link_upload", "gpu_attention", "gpu_ffn", "cpu_attention", "cpu_ffn",
                 "layer_total")]

    def gpu_total(self):
        return self.gpu_attention + self.gpu_ffn

    def cpu_total(self):
        return self.cpu_attention + self.cpu_ffn


class MemoryFootprint(C.Structure):
    _fields_ = [("gpu_bytes", C.c_double), ("cpu_bytes", C.c_double), ("feasible", C.c_int32)]


class PlanResult(C.Structure):
    _fields_ = [("policy", Policy), ("breakdown", LatencyBreakdown), ("memory", MemoryFootprint),
                ("decode_throughput", C.c_double), ("generation_throughput", C.c_double),
                ("objective", C.c_double)]


class StepDurations(C.Structure):
    _fields_ = [(n, C.c_double) for n in
                ("pre_attn", "offload_qkv", "cpu_attn", "load_hidden", "post_attn",
                 "weight_stage", "weight_upload", "kv_load", "gpu_attn")]


class Task(C.Structure):
    _fields_ = [(n, C.c_int32) for n in
                ("kind", "step", "layer", "microbatch", "page", "resource")] + \
               [("duration", C.c_double), ("n_deps", C.c_int32)]


class TimelineEntry(C.Structure):
    _fields_ = [("task", C.c_int32), ("start", C.c_double), ("end", C.c_double)]


class SimMetrics(C.Structure):
    _fields_ = [("makespan", C.c_double), ("utilization", C.c_double * 5),
                ("steady_layer_time", C.c_double)]


class SearchGrid(C.Structure):
    _fields_ = [("micro_batch_values", C.c_void_p), ("n_micro_batch_values", C.c_int32),
                ("micro_batch_counts", C.c_void_p), ("n_micro_batch_counts", C.c_int32),
                ("weight_ratio_values", C.c_void_p), ("n_weight_ratio_values", C.c_int32),
                ("kv_ratio_values", C.c_void_p), ("n_kv_ratio_values", C.c_int32),
                ("attn_on_gpu_values", C.c_void_p), ("n_attn_on_gpu_values", C.c_int32),
                ("ffn_on_gpu_values", C.c_void_p), ("n_ffn_on_gpu_values", C.c_int32)]


def make_grid(mu, counts, rw, rc, attn=(0, 1), ffn=(0, 1)):
    """A SearchGrid over Python lists (the arrays are kept alive on the struct)."""
    arrs = [(C.c_int64 * len(mu))(*mu), (C.c_int64 * len(counts))(*counts),
            (C.c_double * len(rw))(*rw), (C.c_double * len(rc))(*rc),
            (C.c_int32 * len(attn))(*attn), (C.c_int32 * len(ffn))(*ffn)]
    g = SearchGrid(C.cast(arrs[0], C.c_void_p), len(mu), C.cast(arrs[1], C.c_void_p), len(counts),
                   C.cast(arrs[2], C.c_void_p), len(rw), C.cast(arrs[3], C.c_void_p), len(rc),
                   C.cast(arrs[4], C.c_void_p), len(attn), C.cast(arrs[5], C.c_void_p), len(ffn))
    g._keep = arrs
    return g


class RooflineGrid(C.Structure):
    """RooflineGrid (reference hrm.hpp:57-61)."""
    _fields_ = [("min_intensity", C.c_double), ("max_intensity", C.c_double),
                ("points_per_decade", C.c_int32)]


LEVEL_GPU, LEVEL_CPU = 0, 1  # MemoryLevel (hrm.hpp:15)


class BatchParams(C.Structure):
    _fields_ = [("n_ub", C.c_int64), ("ubs", C.c_int64), ("gen_len", C.c_int64),
                ("cache_size", C.c_int64), ("flush_partials", C.c_int32)]


SCHED = {"cgopipe": 0, "s2": 1, "s3": 2, "s4": 3}
TASK_KINDS = ["pre_attn", "offload_qkv", "cpu_attn", "load_hidden", "post_attn",
              "weight_to_pinned", "weight_to_gpu", "kv_load", "gpu_attn"]
RESOURCES = ["gpu", "cpu", "h2d", "d2h", "ctopin"]

P = C.POINTER
class Config(C.Structure):
    """ParsedConfig (reference config.hpp:89-94); has_policy = the optional [policy]."""
    _fields_ = [("hardware", HardwareSpec), ("model", ModelSpec), ("workload", WorkloadSpec),
                ("policy", Policy), ("has_policy", C.c_int32)]


class ConfigError(ValueError):
    """parse_config_text failure: line >= 1 a parse error on that line, 0 a
    file-level parse error (missing section/key), -1 validation issues."""

    def __init__(self, line: int, message: str):
        super().__init__(f"line {line}: {message}" if line > 0 else message)
        self.line, self.message = line, message


_SIGS = {
    "last_error": (C.c_char_p, []),
    "parse_config": (C.c_int, [C.c_char_p, P(Config), P(C.c_int32), C.c_char_p, C.c_size_t]),
    "serialize_config": (C.c_int, [P(Config), C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "last_status": (C.c_int, []),
    "version": (C.c_char_p, []),
    "op_profiles": (C.c_int, [P(ModelSpec), C.c_double, C.c_double, C.c_double, P(OpProfile)]),
    "layer_weight_bytes": (C.c_int, [P(ModelSpec), P(LayerWeightBytes)]),
    "transfer_sizes": (C.c_int, [P(ModelSpec), P(Policy), C.c_double, P(TransferSizes)]),
    "memory_totals": (C.c_int, [P(ModelSpec), P(WorkloadSpec), C.c_int64, P(C.c_double)]),
    "layer_latency": (C.c_int, [P(HardwareSpec), P(ModelSpec), P(WorkloadSpec), P(Policy),
                                C.c_double, P(LatencyBreakdown)]),
    "memory_footprint": (C.c_int, [P(HardwareSpec), P(ModelSpec), P(WorkloadSpec), P(Policy),
                                   P(MemoryFootprint)]),
    "apply_tensor_parallelism": (C.c_int, [P(HardwareSpec), C.c_int, C.c_int, C.c_double,
                                           P(HardwareSpec)]),
    "estimate_throughput": (C.c_int, [P(HardwareSpec), P(ModelSpec), P(WorkloadSpec), P(Policy),
                                      P(PlanResult)]),
    "hrm_attainable_local": (C.c_int, [C.c_int, C.c_double, P(HardwareSpec), P(C.c_double)]),
    "hrm_attainable_cross": (C.c_int, [C.c_double, C.c_double, P(HardwareSpec), P(C.c_double)]),
    "hrm_turning_point_p1": (C.c_int, [C.c_double, P(HardwareSpec), P(C.c_double)]),
    "hrm_turning_point_p2": (C.c_int, [C.c_double, P(HardwareSpec), P(C.c_double)]),
    "hrm_balance_gap": (C.c_int, [C.c_double, C.c_double, P(HardwareSpec), P(C.c_double)]),
    "roofline_csv": (C.c_int, [P(OpProfile), P(C.c_char_p), C.c_int, P(HardwareSpec), P(RooflineGrid),
                               C.c_char_p, C.c_size_t, P(C.c_size_t)]),
    "search_policy": (C.c_int, [P(HardwareSpec), P(ModelSpec), P(WorkloadSpec), P(SearchGrid),
                                C.c_int, C.c_double, P(PlanResult)]),
    "search_candidate_count": (C.c_int64, [P(SearchGrid)]),
    "validate": (C.c_int, [P(HardwareSpec), P(ModelSpec), P(WorkloadSpec), P(Policy), C.c_char_p,
                           C.c_size_t]),
    "batch_requests": (C.c_int, [P(C.c_char_p), P(C.c_int64), C.c_int32, P(BatchParams),
                                 P(C.c_int32), P(C.c_int32)]),
    "schedule_build": (C.c_void_p, [P(HardwareSpec), P(ModelSpec), P(WorkloadSpec), P(Policy),
                                    C.c_int, C.c_int, C.c_int]),
    "schedule_build_durations": (C.c_void_p, [P(StepDurations), C.c_int, C.c_int, C.c_int,
                                              C.c_int]),
    "dag_from_tasks": (C.c_void_p, [P(Task), C.c_int, P(C.c_int32), C.c_int, C.c_int, C.c_int,
                                    C.c_int]),
    "dag_free": (None, [C.c_void_p]),
    "dag_size": (C.c_int, [C.c_void_p]),
    "dag_task": (C.c_int, [C.c_void_p, C.c_int, P(Task), P(C.c_int32), C.c_int]),
    "dag_dump": (C.c_int, [C.c_void_p, C.c_char_p, C.c_size_t]),
    "simulate": (C.c_int, [C.c_void_p, P(TimelineEntry), P(C.c_double), P(C.c_double)]),
    "metrics": (C.c_int, [C.c_void_p, P(TimelineEntry), C.c_int, C.c_double, P(C.c_double),
                          P(SimMetrics)]),
    "verify_timeline": (C.c_int, [C.c_void_p, P(TimelineEntry), C.c_int, C.c_double,
                                  P(C.c_double), C.c_double, C.c_char_p, C.c_size_t]),
    "timeline_json": (C.c_int, [C.c_void_p, P(TimelineEntry), C.c_int, C.c_double,
                                P(C.c_double), C.c_char_p, C.c_char_p, C.c_size_t]),
}


@dataclass
class Timeline:
    entries: object  # ctypes array of TimelineEntry
    makespan: float
    busy: object     # c_double * 5

    def starts(self):
        return [e.start for e in self.entries]


class Dag:
    """Owning handle on an mlt_dag (ScheduleDag)."""

    def __init__(self, api: "Api", handle):
        self.api, self.h = api, handle

    def __del__(self):
        if getattr(self, "h", None):
            self.api.fn["dag_free"](self.h)
            self.h = None

    def __len__(self):
        return self.api.fn["dag_size"](self.h)

    def task(self, i):
        t = Task()
        deps = (C.c_int32 * 64)()
        n = self.api.check(self.api.fn["dag_task"](self.h, i, C.byref(t), deps, 64))
        return t, [deps[k] for k in range(min(n, 64))]

    def tasks(self):
        return [self.task(i) for i in range(len(self))]

    def dump(self) -> str:
        n = self.api.check(self.api.fn["dag_dump"](self.h, None, 0))
        buf = C.create_string_buffer(n + 1)
        self.api.fn["dag_dump"](self.h, buf, n + 1)
        return buf.value.decode()

    def simulate(self, fn_name="simulate") -> Timeline:
        n = len(self)
        entries = (TimelineEntry * max(n, 1))()
        mk = C.c_double()
        busy = (C.c_double * 5)()
        self.api.check(self.api.fn[fn_name](self.h, entries, C.byref(mk), busy))
        return Timeline(entries, mk.value, busy)

    def metrics(self, tl: Timeline) -> SimMetrics:
        out = SimMetrics()
        self.api.check(self.api.fn["metrics"](self.h, tl.entries, len(self), tl.makespan,
                                              tl.busy, C.byref(out)))
        return out

    def verify(self, tl: Timeline, tol=1e-9) -> str:
        buf = C.create_string_buffer(4096)
        rc = self.api.fn["verify_timeline"](self.h, tl.entries, len(tl.entries), tl.makespan,
                                            tl.busy, tol, buf, 4096)
        if rc < 0:
            self.api.check(rc)
        return buf.value.decode()

    def timeline_json(self, tl: Timeline, manifest="{}") -> str:
        f = self.api.fn["timeline_json"]
        n = self.api.check(f(self.h, tl.entries, len(self), tl.makespan, tl.busy,
                             manifest.encode(), None, 0))
        buf = C.create_string_buffer(n + 1)
        f(self.h, tl.entries, len(self), tl.makespan, tl.busy, manifest.encode(), buf, n + 1)
        return buf.value.decode()


class Api:
    """Typed wrapper over one library's planner/scheduler entry points."""

    def __init__(self, lib: C.CDLL, prefix: str, extra_sigs=None):
        self.lib, self.prefix, self.fn = lib, prefix, {}
        sigs = dict(_SIGS)
        sigs.update(extra_sigs or {})
        for name, (res, args) in sigs.items():
            f = getattr(lib, prefix + name, None)
            if f is None:
                continue
            f.restype, f.argtypes = res, args
            self.fn[name] = f

    def error(self) -> str:
        return (self.fn["last_error"]() or b"").decode()

    def version(self) -> str:
        return (self.fn["version"]() or b"").decode() if "version" in self.fn else ""

    def check(self, rc: int) -> int:
        if rc < 0:
            raise _EXC.get(rc, MltError)(rc, self.error())
        return rc

    # --- cost model ------------------------------------------------------
    def op_profiles(self, model, tokens, ctx, r_w=0.0):
        out = (OpProfile * 4)()
        self.check(self.fn["op_profiles"](C.byref(model), tokens, ctx, r_w, out))
        return {"attention": out[0], "ffn": out[1], "qkv": out[2], "output": out[3]}

    def layer_weight_bytes(self, model):
        out = LayerWeightBytes()
        self.check(self.fn["layer_weight_bytes"](C.byref(model), C.byref(out)))
        return out

    def transfer_sizes(self, model, policy, ctx):
        out = TransferSizes()
        self.check(self.fn["transfer_sizes"](C.byref(model), C.byref(policy), ctx, C.byref(out)))
        return out

    def memory_totals(self, model, workload, batch):
        out = (C.c_double * 2)()
        self.check(self.fn["memory_totals"](C.byref(model), C.byref(workload), batch, out))
        return out[0], out[1]

    # --- planner ---------------------------------------------------------
    def layer_latency(self, hw, model, workload, policy, ctx):
        out = LatencyBreakdown()
        self.check(self.fn["layer_latency"](C.byref(hw), C.byref(model), C.byref(workload),
                                            C.byref(policy), ctx, C.byref(out)))
        return out

    def memory_footprint(self, hw, model, workload, policy):
        out = MemoryFootprint()
        self.check(self.fn["memory_footprint"](C.byref(hw), C.byref(model), C.byref(workload),
                                               C.byref(policy), C.byref(out)))
        return out

    def apply_tensor_parallelism(self, hw, tp, b200_rule=False, host_read_cap=0.0):
        out = HardwareSpec()
        self.check(self.fn["apply_tensor_parallelism"](C.byref(hw), tp, int(b200_rule),
                                                       host_read_cap, C.byref(out)))
        return out

    def estimate_throughput(self, hw, model, workload, policy):
        out = PlanResult()
        self.check(self.fn["estimate_throughput"](C.byref(hw), C.byref(model),
                                                  C.byref(workload), C.byref(policy),
                                                  C.byref(out)))
        return out

    def estimate_throughput_b200(self, tp_hw, model, workload, policy, tp, nvlink_bw=900e9):
        """B200 HRM of a tp-way group incl. the NVLink all-reduce roof (product only)."""
        f = self.lib.mlt_estimate_throughput_b200
        f.restype = C.c_int
        f.argtypes = [P(HardwareSpec), P(ModelSpec), P(WorkloadSpec), P(Policy), C.c_int, C.c_double,
                      P(PlanResult)]
        out = PlanResult()
        self.check(f(C.byref(tp_hw), C.byref(model), C.byref(workload), C.byref(policy), tp, nvlink_bw,
                     C.byref(out)))
        return out

    # --- hierarchical roofline (hrm.hpp:13-74) ---------------------------
    def _d(self, name, *args):
        out = C.c_double()
        self.check(self.fn[name](*args, C.byref(out)))
        return out.value

    def attainable_local(self, level, intensity, hw):
        return self._d("hrm_attainable_local", level, intensity, C.byref(hw))

    def attainable_cross(self, gpu_intensity, cpu_intensity, hw):
        return self._d("hrm_attainable_cross", gpu_intensity, cpu_intensity, C.byref(hw))

    def turning_point_p1(self, cpu_intensity, hw):
        return self._d("hrm_turning_point_p1", cpu_intensity, C.byref(hw))

    def turning_point_p2(self, gpu_intensity, hw):
        return self._d("hrm_turning_point_p2", gpu_intensity, C.byref(hw))

    def balance_gap(self, gpu_intensity, cpu_intensity, hw):
        return self._d("hrm_balance_gap", gpu_intensity, cpu_intensity, C.byref(hw))

    def roofline_csv(self, profiles, names, hw, grid=None) -> str:
        n = len(profiles)
        arr = (OpProfile * max(n, 1))(*profiles)
        nm = (C.c_char_p * max(n, 1))(*[x.encode() for x in names])
        ln = C.c_size_t(0)
        g = C.byref(grid) if grid is not None else None
        self.check(self.fn["roofline_csv"](arr, nm, n, C.byref(hw), g, None, 0, C.byref(ln)))
        buf = C.create_string_buffer(ln.value + 1)
        self.check(self.fn["roofline_csv"](arr, nm, n, C.byref(hw), g, buf, ln.value + 1, C.byref(ln)))
        return buf.value.decode()

    def search_policy(self, hw, model, workload, grid=None, objective=0, ctx_override=-1.0):
        out = PlanResult()
        self.check(self.fn["search_policy"](C.byref(hw), C.byref(model), C.byref(workload),
                                            C.byref(grid) if grid is not None else None, objective,
                                            ctx_override, C.byref(out)))
        return out

    # --- INI config (config.hpp:80-121) -----------------------------------
    def parse_config(self, text: str) -> Config:
        out, line = Config(), C.c_int32(0)
        buf = C.create_string_buffer(4096)
        rc = self.fn["parse_config"](text.encode(), C.byref(out), C.byref(line), buf, 4096)
        if rc == -1:
            raise ConfigError(line.value, buf.value.decode())
        self.check(rc)
        return out

    def parse_config_file(self, path: str) -> Config:
        try:
            with open(path, "rb") as fh:
                text = fh.read().decode("utf-8", "surrogateescape")
        except OSError:
            raise ConfigError(0, "cannot open config file: " + path) from None
        return self.parse_config(text)

    def serialize_config(self, cfg: Config) -> str:
        n = C.c_size_t(0)
        self.check(self.fn["serialize_config"](C.byref(cfg), None, 0, C.byref(n)))
        buf = C.create_string_buffer(n.value + 1)
        self.check(self.fn["serialize_config"](C.byref(cfg), buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def validate(self, hw=None, model=None, workload=None, policy=None):
        """Reference config.hpp validate(): the list of issue lines ([] = valid)."""
        buf = C.create_string_buffer(4096)
        ref = lambda x: C.byref(x) if x is not None else None  # noqa: E731
        n = self.check(self.fn["validate"](ref(hw), ref(model), ref(workload), ref(policy), buf, 4096))
        return buf.value.decode().splitlines() if n else []

    def search_candidate_count(self, grid=None):
        return self.fn["search_candidate_count"](C.byref(grid) if grid is not None else None)

    def batch_requests(self, requests, n_ub, ubs, gen_len, cache_size, flush_partials=True,
                       fn="batch_requests"):
        """requests: list of (id, input_len).  Returns (micro_batches [[ids]], aborted [ids])."""
        n = len(requests)
        ids = (C.c_char_p * max(n, 1))(*[r[0].encode() for r in requests])
        lens = (C.c_int64 * max(n, 1))(*[r[1] for r in requests])
        ob, os_ = (C.c_int32 * max(n, 1))(), (C.c_int32 * max(n, 1))()
        p = BatchParams(n_ub, ubs, gen_len, cache_size, int(flush_partials))
        nb = self.check(self.fn[fn](ids, lens, n, C.byref(p), ob, os_))
        batches = [[None] * 0 for _ in range(nb)]
        slots = {}
        aborted = {}
        for i in range(n):
            if ob[i] == -1:
                aborted[os_[i]] = requests[i][0]
            elif ob[i] >= 0:
                slots[(ob[i], os_[i])] = requests[i][0]
        for (b, s) in sorted(slots):
            batches[b].append(slots[(b, s)])
        return batches, [aborted[k] for k in sorted(aborted)]

    # --- scheduler -------------------------------------------------------
    def _dag(self, h):
        if not h:
            raise _EXC.get(self._last_code(), MltError)(self._last_code(), self.error())
        return Dag(self, h)

    def _last_code(self):
        return self.fn["last_status"]()

    def build_schedule(self, hw, model, workload, policy, kind="cgopipe", layers=None, steps=1):
        layers = model.layers if layers is None else layers
        h = self.fn["schedule_build"](C.byref(hw), C.byref(model), C.byref(workload),
                                      C.byref(policy), SCHED[kind], layers, steps)
        return self._dag(h)

    def build_schedule_durations(self, durations, kind, layers, steps, micro_batches):
        if isinstance(durations, StepDurations):
            durations = [durations] * steps
        arr = (StepDurations * max(len(durations), 1))(*durations)
        h = self.fn["schedule_build_durations"](arr, SCHED[kind], layers, steps, micro_batches)
        return self._dag(h)

    def execution_dag(self, dag: "Dag", model, policy, exact_gates=True):
        """The DAG the executor runs for `dag` (mlt_execution_dag)."""
        f = self.lib.mlt_execution_dag
        f.restype = C.c_void_p
        f.argtypes = [C.c_void_p, P(ModelSpec), P(Policy), C.c_int, C.c_void_p]
        return self._dag(f(dag.h, C.byref(model), C.byref(policy), int(exact_gates), None))

    def dag_from_tasks(self, tasks, layers=1, steps=1, micro_batches=1, kind="cgopipe"):
        """tasks: list of (Task, deps)."""
        arr = (Task * max(len(tasks), 1))()
        flat = []
        for i, (t, deps) in enumerate(tasks):
            t.n_deps = len(deps)
            arr[i] = t
            flat.extend(deps)
        dep_arr = (C.c_int32 * max(len(flat), 1))(*flat)
        h = self.fn["dag_from_tasks"](arr, len(tasks), dep_arr, layers, steps, micro_batches,
                                      SCHED[kind])
        return self._dag(h)


_product = None


def load_product() -> Api:
    """The product library.  Fails loudly when it has not been built."""
    global _product
    if _product is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g;"
                              f" g.build()'` (make -C paper_2411_11217_b200/csrc)")
        _product = Api(C.CDLL(LIB_PATH), "mlt_")
    return _product


# ---------------------------------------------------------------------------
# Kernel-level entry points (device pointers are passed as integers).
# ---------------------------------------------------------------------------
class GemmArgs(C.Structure):
    _fields_ = [("a_table", C.c_void_p), ("n_mats", C.c_int32), ("G", C.c_int32),
                ("RB", C.c_int32), ("K", C.c_int32), ("b", C.c_void_p), ("R", C.c_int32),
                ("b_off", C.c_void_p), ("b_cnt", C.c_void_p), ("rows_dense", C.c_int32),
                ("n_cap", C.c_int32), ("epi", C.c_int32), ("alpha", C.c_float),
                ("out_f32", C.c_void_p), ("ldo", C.c_int32), ("residual", C.c_void_p),
                ("ldr", C.c_int32), ("out_packed", C.c_void_p), ("out_R", C.c_int32),
                ("n_chunks", C.c_int32), ("k_splits", C.c_int32), ("split_stride", C.c_int64),
                ("trace", C.c_void_p), ("codec", C.c_int32), ("ktrace", C.c_void_p),
                ("sk_scratch", C.c_void_p), ("sk_count", C.c_void_p), ("sk_rows", C.c_int32),
                ("dec_groups", C.c_int32), ("codec_raw", C.c_int32), ("enc_tile", C.c_int32)]


V, I, F = C.c_void_p, C.c_int, C.c_float
_KSIGS = {
    "pack_weight": [V, C.c_int64, C.c_int64, V],
    "codec_encode": [V, C.c_int64, C.c_int64, V],
    "codec_decode": [V, C.c_int64, V],
    "codec_encode_frag": [V, C.c_int64, C.c_int64, V, V],
    "codec_encode_rows": [V, C.c_int64, C.c_int64, V, V],
    "codec4_encode_rows": [V, C.c_int64, C.c_int64, V, V],
    "codec4_decode_rows": [V, C.c_int64, V],
    "codec4_tile_bytes": [],
    "codec4_encode_rows_cap": [V, C.c_int64, C.c_int64, I, V, V],
    "codec4_decode_rows_cap": [V, C.c_int64, I, V],
    "codec4_tile_bytes_for": [I],
    "frag_pack": [V, C.c_int64, V],
    "host_gqa_decode": [V, V, V, V, I, I, I, I, I, V, I],
    "host_gqa_use_amx": [I],
    "unpack_rows": [V, C.c_int64, C.c_int64, C.c_int64, V],
    "pack_rows_host": [V, C.c_int64, C.c_int64, C.c_int64, V],
    "gemm": [C.POINTER(GemmArgs), V],
    "embed": [V, V, I, I, V, V],
    "rmsnorm_pack": [V, V, I, I, F, V, I, V],
    "pack_rows": [V, I, I, I, V, I, V],
    "rope_qkv": [V, V, V, I, I, I, I, V, V],
    "router_topk": [V, V, F, V, V, I, I, I, I, V, V, V, V, V],
    "moe_permute": [V, V, I, I, I, I, V, V, V, V, V, I, V],
    "moe_combine": [V, V, I, V, V, I, I, I, V, V],
    "expert_ffn": [V, I, V, V, V, V, I, I, I, I, V, V, V, V, V, I, I, V, V],
    "argmax": [V, I, I, V, V, V],
    "gqa_decode_paged": [V, I, V, V, V, I, V, V, I, I, I, I, I, V, I, V, V],
    "gqa_decode_paged_split": [V, I, V, V, V, I, V, V, I, I, I, I, I, V, I, V, I, I, V, V, V],
    "gqa_decode_paged_flat": [V, I, V, V, V, I, V, V, I, I, I, I, I, V, I, V, I, V, V, V],
    "kv_append": [V, I, I, I, V, V, I, V, I, I, V, V, V],
    "rope_table": [I, I, C.c_double, V],
    "prefill_attention": [V, I, V, I, I, I, I, V, I, V],
    "kv_stage": [V, I, I, I, I, V, V, V, V, I, V, V, V],
    "synth_bf16": [C.c_uint64, C.c_uint64, C.c_int64, F, I, V],
}


class Kernels:
    """Raw kernel entry points; every call raises MltError on failure."""

    def __init__(self, lib: C.CDLL):
        self.lib = lib
        self._err = lib.mlt_last_error
        self._err.restype = C.c_char_p
        for name, args in _KSIGS.items():
            f = getattr(lib, "mlt_" + name)
            f.restype, f.argtypes = C.c_int, args
            setattr(self, "_" + name, f)

    def __getattr__(self, name):
        raw = self.__dict__.get("_" + name)
        if raw is None:
            raise AttributeError(name)

        def call(*args):
            rc = raw(*args)
            if rc < 0:
                raise _EXC.get(rc, MltError)(rc, (self._err() or b"").decode())
            return rc
        return call


_kernels = None


def load_kernels() -> Kernels:
    global _kernels
    if _kernels is None:
        load_product()
        _kernels = Kernels(_product.lib)
    return _kernels
