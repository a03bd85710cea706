#!/usr/bin/env python
"""Headline benchmark: batched decode tokens/sec at a fixed GPU memory budget
and its fraction of the B200 HRM bound (BASELINE.json "metric").

Default workload = BASELINE.json configs[1]: Mixtral-8x7B shape (l=32,
h1=4096, h2=14336, n_q=32, n_kv=8, n_e=8, k=2), 1 x B200, 16 GB cap on every
runtime device allocation, paged expert weights, N=256 sequences, prompt 512
(synthetic prompt-stage KV), greedy decode.  Policy (N=256, mu=64, A_g=0,
F_g=1, r_w=0.10): the reference model's optimum family at 16 GB (BASELINE.md
§2; mu=64 instead of 256 keeps CPU attention overlapped, same bound within
0.1%).  A "step" = one decode step of all 32 layers for all 256 sequences.

  python bench.py [--steps K] [--warmup W] [--impl mlt|reference] [--config NAME]

--impl reference times the CPU numerical restatement (oracle/, the only CPU
decode path there is: the reference artifact has none) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: model (l, h1, h2, n_q, n_kv, n_e, k), policy, budget, prompt, vocab
    "mixtral8x7b-16g": dict(model=(32, 4096, 14336, 32, 8, 8, 2), N=256, mu=64, r_w=0.10, a_g=0,
                            budget=16e9, prompt=512, gen=32, vocab=32000),
    # r_w 0.29, not the reference optimum 0.30: the arena also holds embedding +
    # lm_head (0.52 GB), which ModelSpec does not model (memory_footprint)
    "mixtral8x7b-32g": dict(model=(32, 4096, 14336, 32, 8, 8, 2), N=256, mu=64, r_w=0.29, a_g=0,
                            budget=32e9, prompt=512, gen=32, vocab=32000),
    "mixtral8x7b-64g": dict(model=(32, 4096, 14336, 32, 8, 8, 2), N=256, mu=64, r_w=0.65, a_g=0,
                            budget=64e9, prompt=512, gen=32, vocab=32000),
    # all weights + KV resident in HBM, attention on the GPU (S4 schedule): the
    # GPU-bound regime a 180 GB B200 opens up (HRM bound is HBM, not PCIe)
    "mixtral8x7b-resident": dict(model=(32, 4096, 14336, 32, 8, 8, 2), N=256, mu=256, r_w=1.0,
                                 a_g=1, budget=140e9, prompt=512, gen=32, vocab=32000),
    # BASELINE configs[3]/[4]: tensor-parallel over 2/4/8 B200 (torchrun), 16 GB per GPU;
    # r_w per tp = the reference model's optimum
    "mixtral8x22b-tp": dict(model=(56, 6144, 16384, 48, 8, 8, 2), N=256, mu=64,
                            r_w={1: 0.0, 2: 0.05, 4: 0.15, 8: 0.40}, a_g=0, budget=16e9, prompt=512,
                            gen=32, vocab=32000),
    "dbrx-tp": dict(model=(40, 6144, 10752, 48, 8, 16, 4), N=256, mu=64,
                    # reference optimum r_w 0.05/0.20/0.45 less the arena's embedding + lm_head
                    # (0.79 GB, not in ModelSpec): 0.04/0.18/0.42 fit 16 GB per GPU
                    r_w={1: 0.0, 2: 0.04, 4: 0.18, 8: 0.42}, a_g=0, budget=16e9, prompt=512, gen=128,
                    vocab=32000),
    # BASELINE configs[0] (the CPU reference's own case): 181 MB of weights per layer fit
    # any budget, so weights and KV are resident and attention runs on the GPU (S4)
    "tiny": dict(model=(2, 1024, 3584, 8, 2, 8, 2), N=8, mu=4, r_w=1.0, a_g=1, budget=4e9,
                 prompt=16, gen=32, vocab=32000),
}

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
NVLINK_BW = 900e9       # B200 NVLink 5, bytes/s per direction (nominal; 1 GPU in this pool)
HOST_FLOPS = 2.0e12     # fallback host-core fp32 FLOP/s (16 SPR cores AVX-512); measured live when possible
_host_flops = None
# An 8-GPU B200 node's host DRAM feeds every GPU's PCIe stream and the host
# attention together.  This pool leases one GPU with a 16-core slice of a
# host (its DRAM read bandwidth is measured live); a tp-way job's node is
# modeled as tp such slices but never above this node limit: 2 sockets x 8
# channels of DDR5-5600 (716.8 GB/s peak) at the ~80 % a read stream
# sustains (DGX B200 class host).  Documented assumption.
NODE_HOST_READ_GBS = 573.0


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return PEAKS_FALLBACK, "fallback"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), "--query-gpu=" + self.Q,
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None
        return self

    def __exit__(self, *exc):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.p.kill()

    def summary(self):
        self.f.flush()
        self.f.seek(0)
        rows = [r.strip().split(",") for r in self.f.read().splitlines() if r.strip()]
        os.unlink(self.f.name)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# bytes per weight as stored with --codec: the runtime's default 3-bit code
# (codec 4, 11600 B per 8192-weight tile, runtime/weight_codec.hpp), or the
# 4-bit code's 12432 B when MLT_CODEC_MODE selects engine 1-3; the runtime
# itself always computes in bf16
CODEC_DT = (12432 if os.environ.get("MLT_CODEC_MODE", "4")[:1] in ("1", "2", "3") else 11600) / 8192
def arena_extra(cfg):
    """Arena bytes outside ModelSpec: embedding + lm_head (vocab x h1 bf16 each),
    activations, page tables and other KV-independent buffers (0.2 GB); the runtime
    steps r_w down if the arena still overflows."""
    return 2 * cfg["vocab"] * cfg["model"][1] * 2 + 0.2e9


def model_spec(cfg, stored=False):
    """ModelSpec of the config; stored=True gives the bytes the weights occupy as
    stored/streamed (dt_w = CODEC_DT with --codec), which is what the HRM bound of
    the reference's cost model must see."""
    from paper_2411_11217_b200 import capi
    l, h1, h2, nq, nkv, ne, k = cfg["model"]
    dt = cfg.get("stored_dt", CODEC_DT)  # after runtime creation: the bytes per weight it actually stores
    return capi.ModelSpec(l, h1, h2, nq, nkv, ne, k, dt if stored and cfg.get("codec") else 2.0, 2.0)


def node_host(host_gbs, tp, per_slice_host):
    """(host DRAM read B/s, host FLOP/s) of the job's node: the measured slice,
    x tp slices for a --tp-shard extrapolation, capped at NODE_HOST_READ_GBS."""
    slices = tp if per_slice_host else 1
    bw = host_gbs * slices
    if slices > 1:
        bw = min(bw, NODE_HOST_READ_GBS)
    return bw * 1e9, host_flops() * slices


def b200_hw(cfg, link_gbs, host_gbs, pk, tp=1, per_slice_host=False, budget=None):
    """The measured B200 HardwareSpec (TP-scaled with the B200 rule for tp > 1:
    GPU side x tp, link x tp capped by the node's host read bandwidth)."""
    from paper_2411_11217_b200 import capi
    api = capi.load_product()
    host_bw, host_fl = node_host(host_gbs, tp, per_slice_host)
    hw = capi.HardwareSpec(cfg["budget"] if budget is None else budget, 196e9 * max(tp, 1), pk["hbm_gbs"] * 1e9,
                           host_bw, link_gbs * 1e9, pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) * 1e12,
                           host_fl)
    if tp > 1:
        hw = api.apply_tensor_parallelism(hw, tp, b200_rule=True, host_read_cap=host_bw)
    return hw


def search_rw(cfg, link_gbs, host_gbs, pk, tp=1, per_slice_host=False):
    """Best feasible r_w for the config's (N, mu, A_g) on the measured spec with
    the stored weight bytes (product search_policy, planner.cpp:234-341)."""
    from paper_2411_11217_b200 import capi
    api = capi.load_product()
    hw = b200_hw(cfg, link_gbs, host_gbs, pk, tp, per_slice_host, budget=cfg["budget"] - arena_extra(cfg))
    grid = capi.make_grid([cfg["mu"]], [cfg["N"] // cfg["mu"]], [round(0.01 * i, 2) for i in range(101)],
                          [1.0] if cfg["a_g"] else [0.0], attn=(cfg["a_g"],), ffn=(1,))
    return api.search_policy(hw, model_spec(cfg, stored=True), capi.WorkloadSpec(cfg["prompt"], cfg["gen"]),
                             grid).policy.weights_on_gpu


def policy(cfg):
    from paper_2411_11217_b200 import capi
    return capi.Policy(cfg["N"], cfg["mu"], cfg["a_g"], 1, cfg["r_w"], 1.0 if cfg["a_g"] else 0.0)


def hrm_bound(cfg, link_gbs, host_gbs, pk, tp=1, per_slice_host=False):
    """B200 HRM bound: the reference's own estimate_throughput (planner.cpp:129-162)
    re-parameterised with measured B200 numbers; under TP the B200 rule of
    apply_tensor_parallelism_b200 (GPU side x tp, link x tp capped by the host
    DRAM read bandwidth: every B200 has its own PCIe link)."""
    from paper_2411_11217_b200 import capi
    api = capi.load_product()
    # with --tp-shard the measured box is one GPU's slice of a node (16 cores,
    # 196 GB, its own PCIe link): a tp-way job has tp slices, whose host cores
    # compute their own heads' attention (the reference keeps the CPU side
    # fixed under TP, planner.cpp:101-108), capped at the node's DRAM read limit
    hw = b200_hw(cfg, link_gbs, host_gbs, pk, tp, per_slice_host)
    w = capi.WorkloadSpec(cfg["prompt"], cfg["gen"])
    m = model_spec(cfg, stored=True)
    if tp > 1:  # + the NVLink roof of the 2 all-reduces / layer / micro-batch (nominal NVLink 5)
        return api.estimate_throughput_b200(hw, m, w, policy(cfg), tp, NVLINK_BW)
    r = api.estimate_throughput(hw, m, w, policy(cfg))
    return r


def host_flops():
    """Host fp32 FLOP/s of this box, measured once (numpy / OpenBLAS sgemm 4096^3
    on all cores, best of 2; the HardwareSpec's cpu_flops) in a child process, so
    no BLAS worker threads outlive the measurement next to the runtime's host
    attention pool; the fallback HOST_FLOPS only if the measurement fails."""
    global _host_flops
    if _host_flops is None:
        code = ("import numpy as np, time\n"
                "a = np.random.default_rng(0).standard_normal((4096, 4096), dtype=np.float32)\n"
                "a @ a\nbest = 0.0\n"
                "for _ in range(2):\n"
                "    t = time.perf_counter(); a @ a; best = max(best, 2 * 4096 ** 3 / (time.perf_counter() - t))\n"
                "print(best)\n")
        try:
            r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
            best = float(r.stdout.strip().splitlines()[-1])
            _host_flops = best if best > 1e10 else HOST_FLOPS
        except Exception:  # noqa: BLE001  (no BLAS / no child: keep the stated estimate)
            _host_flops = HOST_FLOPS
    return _host_flops


def measure_host(api):
    import ctypes as C
    f = api.lib.mlt_measure_host_bw
    f.restype, f.argtypes = C.c_int, [C.c_size_t, C.POINTER(C.c_double)]
    out = (C.c_double * 2)()
    api.check(f(4 << 30, out))
    return out[0]


def host_info():
    """CPU model and usable cores of this box (stated in both arms' lines)."""
    model, flags = None, set()
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name") and model is None:
                    model = ln.split(":", 1)[1].strip()
                elif ln.startswith("flags") and not flags:
                    flags = set(ln.split(":", 1)[1].split())
    except OSError:
        pass
    isa = [f for f in ("avx512f", "avx512_bf16", "amx_bf16", "amx_tile") if f in flags]
    return {"cpu_model": model, "cores": len(os.sched_getaffinity(0)), "isa": isa}


def config_obj(args, cfg, world):
    """The workload description, printed identically by both arms."""
    names = {32: "Mixtral-8x7B shape", 56: "Mixtral-8x22B shape", 40: "DBRX shape", 2: "tiny"}
    l = cfg["model"][0]
    return {"workload": args.config, "model": names.get(l, "custom"), "global_batch": cfg["N"],
            "seq_len": cfg["prompt"], "gen_len": cfg["gen"], "micro_batch": cfg["mu"],
            "gpu_budget_gb": cfg["budget"] / 1e9, "A_g": cfg["a_g"],
            "parallelism": f"tp{world}" if world > 1 else "single GPU, weight paging",
            "data": "synthetic weights seed 1234, prompt ids seed 5678, prompt KV seed 9012"}


def cpu_decode(cfg, warmup, steps):
    """The CPU restatement of the decode path (oracle/, fp32 activations,
    OpenMP over all host cores) run for WHOLE decode steps: all l layers for
    all N sequences, greedy, from the synthetic prompt KV at ctx = prompt.
    Returns (per-step seconds of the timed steps, threads, setup seconds)."""
    import numpy as np
    from oracle import bind as orc
    l, h1, h2, nq, nkv, ne, k = cfg["model"]
    N, s = cfg["N"], cfg["prompt"]
    t0 = time.perf_counter()
    m = orc.Model(l, h1, h2, nq, nkv, ne, k, cfg["vocab"], N, s + warmup + steps + 2)
    m.fill_kv(9012, s)
    setup = time.perf_counter() - t0
    tok = np.random.default_rng(5678).integers(0, cfg["vocab"], N, dtype=np.int32)
    times = []
    for i in range(warmup + steps):
        t = time.perf_counter()
        tok, _ = m.decode_step(tok, np.full(N, s + i, np.int32), orc.FP32)
        times.append(time.perf_counter() - t)
    del m
    return times[warmup:], orc.lib().orc_num_threads(), setup


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    times, cores, setup = cpu_decode(cfg, args.warmup, args.steps)
    total = sum(times)
    l = cfg["model"][0]
    value = cfg["N"] * len(times) / total
    sample = (f"{len(times)} whole decode steps (all {l} layers, N={cfg['N']} sequences, ctx "
              f"{cfg['prompt']}..{cfg['prompt'] + args.warmup + args.steps - 1}) of the fp32 CPU oracle "
              f"after {args.warmup} warm-up steps; model build + prompt KV {setup:.1f} s untimed")
    line = {"impl": "reference", "metric": "decode tokens/sec at fixed GPU-mem budget",
            "value": value, "unit": "tok/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_obj(args, cfg, args.tp_shard if args.tp_shard > 1 else world), "host": host_info(),
            "cpu_baseline": {"value": value, "unit": "tok/s", "cores": cores, "kind": "port",
                             "sample": sample},
            "step_seconds": [round(t, 3) for t in times],
            "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def expert_roofline(cfg, rep, pk, traffic_src, tp=1):
    """Dominant GPU kernel = expert FFN (gate/up + down GEMM) per micro-batch.
    Algorithmic bytes per launch: sum over touched experts of
    3*h1*h2*dt (all n_e are touched at mu*k >= 128 slots, P(untouched) <
    1e-7) + mu*k*2*h1*dt + mu*h1*dt."""
    l, h1, h2, nq, nkv, ne, k = cfg["model"]
    traffic, traffic_file = traffic_src
    mu = cfg["mu"]
    wbytes = ne * 3 * h1 * (h2 // tp) * 2
    tokens = mu * k * 2 * h1 * 2 + mu * h1 * 2
    # --codec: the kernel must read the encoded tiles (the runtime's stored
    # bytes/weight, ~CODEC_DT), so those are the bytes that bound it; the bf16
    # figure is reported beside
    stored = wbytes * cfg.get("stored_dt", CODEC_DT) / 2 if cfg.get("codec") else wbytes
    bytes_launch = stored + tokens
    # in-kernel %globaltimer span of the gate/up and down GEMMs of each launch
    # (CUDA-event deltas on the mostly idle compute stream would add host-launch gaps)
    avg_s = rep.expert_ms_total / max(rep.expert_launches, 1) / 1e3
    achieved = bytes_launch / avg_s / 1e9
    peak = pk["hbm_gbs"]
    return {"kernel": "expert_ffn (gemm_tc gate/up+SiLU, gemm_tc down)", "bound": "hbm",
            "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic if tp == 1 else None,
            "traffic_source": (f"ncu dram__bytes_read+write per launch, {traffic_file} (same kernels and shape, "
                               f"captured outside the timed run)") if tp == 1 and traffic else None,
            "bytes_per_launch": bytes_launch,
            "bf16_equivalent_gbs": (wbytes + tokens) / avg_s / 1e9,
            "avg_launch_ms": avg_s * 1e3, "launches": rep.expert_launches}


def hrm_kernels(cfg, hw, rep, prof, steps, tp=1, csv_path=None):
    """Each hot kernel on the B200 hierarchical roofline (lightplan::hrm on the
    measured spec hw, Eq. 7-11): operator FLOPs/bytes per micro-batch
    launch from the reference cost model (opcost.cpp:5-47, stored weight
    bytes, /tp under TP), its operational intensities, attainable_local /
    attainable_cross, the turning points P1/P2, the balance gap, and the FLOP/s
    it achieved in this run (live per-launch timings)."""
    from paper_2411_11217_b200 import capi
    api = capi.load_product()
    mu = cfg["mu"]
    ctx = cfg["prompt"] + steps / 2.0  # mean context over the timed steps
    pr = api.op_profiles(model_spec(cfg, stored=True), mu, ctx, cfg["r_w"])
    for p in pr.values():  # this rank's share
        p.flops, p.gpu_bytes, p.cpu_bytes, p.link_bytes = (p.flops / tp, p.gpu_bytes / tp, p.cpu_bytes / tp,
                                                           p.link_bytes / tp)
    ex = {k["name"]: k for k in prof.get("exec", [])}
    ev = {k["name"]: k for k in prof.get("events", [])}

    def per_launch(d, name):
        k = d.get(name)
        return k["ms"] / k["launches"] / 1e3 if k and k.get("launches") else None

    M = cfg["N"] // mu
    t_ffn = rep.expert_ms_total / rep.expert_launches / 1e3 if rep.expert_launches else None
    t_attn = (per_launch(ev, "gqa_decode_paged") if cfg["a_g"]
              else (rep.measured.cpu_attention / M if rep.measured.cpu_attention > 0 else None))
    items = [("expert_ffn", pr["ffn"], t_ffn, capi.LEVEL_GPU),
             ("attention", pr["attention"], t_attn, capi.LEVEL_GPU if cfg["a_g"] else capi.LEVEL_CPU),
             ("qkv_proj", pr["qkv"], per_launch(ex, "qkv_gemm"), capi.LEVEL_GPU),
             ("o_proj", pr["output"], per_launch(ex, "o_gemm"), capi.LEVEL_GPU)]
    out = {}
    for name, p, t, lv in items:
        gi = p.flops / p.gpu_bytes if p.gpu_bytes else 0.0
        ci = p.flops / p.cpu_bytes if p.cpu_bytes else 0.0
        li = p.flops / p.link_bytes if p.link_bytes else None
        local = api.attainable_local(lv, gi if lv == capi.LEVEL_GPU else ci, hw)
        r = {"where": "gpu" if lv == capi.LEVEL_GPU else "host cores", "flops": p.flops,
             "bytes": p.gpu_bytes if lv == capi.LEVEL_GPU else p.cpu_bytes, "intensity": gi if lv == capi.LEVEL_GPU else ci,
             "attainable_local_tflops": local / 1e12, "p2": api.turning_point_p2(gi, hw)}
        if li is not None:  # streamed over the link: the cross roof binds
            r.update({"link_intensity": li, "attainable_cross_tflops": api.attainable_cross(gi, li, hw) / 1e12,
                      "p1": api.turning_point_p1(li, hw), "balance_gap": api.balance_gap(gi, li, hw)})
        if t:
            r["seconds_per_launch"] = t
            r["achieved_tflops"] = p.flops / t / 1e12
            r["frac_of_attainable_local"] = p.flops / t / local if local else None
        out[name] = r
    if csv_path:
        with open(csv_path, "w") as fh:
            fh.write(api.roofline_csv([p for _, p, _, _ in items], [n for n, _, _, _ in items], hw))
    return out


def load_traffic(codec=False):
    """ncu dram read+write bytes per expert-FFN launch of the same kernels at the
    same shape (an ncu capture cannot run inside the timed bench): (bytes, file)."""
    # codec 3 (4-bit code): expert_ffn_traffic_codec.json; codec 4 (3-bit, default): ..._codec4.json
    name = ("expert_ffn_traffic_codec4.json" if CODEC_DT < 1.45 else "expert_ffn_traffic_codec.json") if codec \
        else "expert_ffn_traffic.json"
    p = os.path.join(ROOT, "profiles", name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f).get("traffic_bytes_per_launch"), "profiles/" + name
    return None, None


def run_mlt(args, cfg):
    from paper_2411_11217_b200 import capi
    from paper_2411_11217_b200.runtime import Runtime, nccl_unique_id
    import ctypes as C
    import numpy as np

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # --tp-shard T: the largest shard of a T-way tensor-parallel job measured alone on
    # this GPU (its own PCIe link, all-reduce elided): the per-GPU step of that job
    tp = args.tp_shard if args.tp_shard > 1 else world
    if args.tp_shard > 1:  # measure the rank with the largest shard (uneven h2 blocks): the job's slowest
        import ctypes as C
        from paper_2411_11217_b200 import capi
        f = capi.load_product().lib.mlt_tp_shard
        f.restype, f.argtypes = C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        sizes = []
        for r in range(tp):
            out = (C.c_int64 * 6)()
            f(C.byref(model_spec(cfg)), r, tp, out)
            sizes.append(out[2])
        shard_rank = max(range(tp), key=lambda r: sizes[r])
    else:
        shard_rank = rank
    dist = None
    nid = b""
    if world > 1:
        # One process per GPU; tensor parallelism across the node: heads and
        # expert h2 sharded, 2 NCCL all-reduces per layer per micro-batch.  The
        # gloo group only ships the ncclUniqueId, barriers and the max-over-ranks.
        import torch
        import torch.distributed as dist
        dist.init_process_group("gloo")
        idt = torch.tensor(list(nccl_unique_id() if rank == 0 else bytes(128)), dtype=torch.uint8)
        dist.broadcast(idt, 0)
        nid = bytes(idt.tolist())
    pk, pk_src = peaks()
    api = capi.load_product()
    f = api.lib.mlt_measure_link
    f.restype, f.argtypes = C.c_int, [C.c_int, C.c_size_t, C.c_int, C.POINTER(C.c_double)]
    link = (C.c_double * 3)()
    api.check(f(local, 1 << 30, 5, link))
    link_gbs = link[0]
    host_gbs = measure_host(api)
    log(f"[bench] rank {rank}: link H2D {link[0]:.2f} GB/s, D2H {link[1]:.2f}, H2D with D2H "
        f"{link[2]:.2f}; host DRAM read {host_gbs:.1f} GB/s; host fp32 {host_flops() / 1e12:.2f} TFLOP/s")

    raw_rw = cfg["r_w"]
    if cfg.get("codec"):  # the stored bytes shrink: re-pick r_w for the budget
        cfg["r_w"] = search_rw(cfg, link_gbs, host_gbs, pk, tp, per_slice_host=args.tp_shard > 1)
        log(f"[bench] rank {rank}: weight codec on, r_w {cfg['r_w']:.2f} (search on {CODEC_DT:.4f} B/weight)")
    t = time.perf_counter()
    while True:
        try:
            rt = Runtime(model_spec(cfg), policy(cfg), budget_bytes=cfg["budget"],
                         max_ctx=cfg["prompt"] + args.warmup + args.steps + 8, vocab=cfg["vocab"],
                         device=local, exact_gates=args.gates == "exact", tp_rank=shard_rank, tp_size=tp,
                         nccl_id=nid, schedule=args.schedule, tp_shard_only=args.tp_shard > 1,
                         weight_codec=bool(cfg.get("codec")), pdl=not args.no_pdl,
                         host_threads=args.host_threads, down_splits=args.down_splits)
            break
        except capi.MltError as e:
            # the searched r_w assumes an even shard; the largest uneven h2 shard
            # (DBRX tp=8) or the arena extras may not fit: step r_w down
            if not (cfg.get("codec") and "budget" in str(e) and cfg["r_w"] > 0.01):
                raise
            cfg["r_w"] = round(cfg["r_w"] - 0.01, 2)
            log(f"[bench] rank {rank}: {e}; retrying with r_w {cfg['r_w']:.2f}")
    info = rt.info
    log(f"[bench] rank {rank}: runtime ready in {time.perf_counter() - t:.1f}s (weights gen "
        f"{info.gen_seconds:.1f}s, pin {info.pin_seconds:.1f}s), r_w achieved "
        f"{info.achieved_weight_ratio:.4f}, streamed {info.streamed_bytes_per_layer / 1e9:.3f} GB/layer, "
        f"arena {info.arena_used / 1e9:.2f} GB")
    prep = None
    if args.prefill:
        # GPU prefill of real (synthetic-id) prompts: KV and first tokens computed, not generated
        prompts = np.random.default_rng(5678).integers(0, cfg["vocab"], (cfg["N"], cfg["prompt"]),
                                                       dtype=np.int32)
        toks, prep = rt.prefill(prompts)
        log(f"[bench] rank {rank}: GPU prefill {prep.prompt_tokens} tokens in {prep.seconds:.3f}s "
            f"({prep.tokens_per_second:.0f} tok/s, chunk {prep.chunk_tokens} x {prep.chunks_per_layer}, "
            f"GPU busy {prep.gpu_busy_seconds:.3f}s)")
    else:
        rt.prefill_synthetic(cfg["prompt"], 9012)
        toks = np.random.default_rng(5678).integers(0, cfg["vocab"], cfg["N"], dtype=np.int32)
    w = rt.decode(toks, args.warmup)
    last = w.ids[-1]
    log(f"[bench] rank {rank}: warm-up {args.warmup} steps: {w.report.tokens_per_second:.1f} tok/s")

    if dist:
        dist.barrier()
    with ClockSampler(local) as clk:
        t0 = time.perf_counter()
        d = rt.decode(last, args.steps)          # host ids in, host ids out (C ABI)
        t1 = time.perf_counter()
    if dist:
        dist.barrier()
    clocks = clk.summary()
    rep = d.report
    dev_s, wall_s = rep.seconds, t1 - t0
    if dist:  # time = max over ranks
        import torch
        tt = torch.tensor([dev_s, wall_s], dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dev_s, wall_s = tt.tolist()
    if not rep.timeline_ok:
        log(f"[bench] measured timeline check: {api.error()}")
    if args.timeline and rank == 0:
        with open(args.timeline, "w") as fh:
            json.dump(rt.timeline(), fh)
    value = cfg["N"] * args.steps / dev_s        # device-timed (CUDA events), whole job
    e2e = cfg["N"] * args.steps / wall_s         # wall clock around the C-ABI call
    if cfg.get("codec"):
        # the bound of the executed run sees the stored bytes per weight the runtime
        # reports: raw-fallback blocks, or the 12-bit code when the 11-bit one does
        # not fit the weights, stream more than the search's CODEC_DT assumed
        cfg["stored_dt"] = info.bytes_per_weight
    try:
        bound = hrm_bound(cfg, link_gbs, host_gbs, pk, tp=tp, per_slice_host=args.tp_shard > 1)
    except capi.InfeasiblePolicyError:
        # the searched r_w does not fit the budget at the stored size (the runtime
        # held fewer weights resident): bound of the best policy at that size
        cfg["r_w_bound"] = search_rw(cfg, link_gbs, host_gbs, pk, tp, per_slice_host=args.tp_shard > 1)
        bound = hrm_bound(dict(cfg, r_w=cfg["r_w_bound"]), link_gbs, host_gbs, pk, tp=tp,
                          per_slice_host=args.tp_shard > 1)
    # the bf16-weight bound at the raw policy: the best the unencoded stream could do
    bound_bf16 = hrm_bound(dict(cfg, codec=False, r_w=raw_rw), link_gbs, host_gbs, pk, tp=tp,
                           per_slice_host=args.tp_shard > 1) if cfg.get("codec") else bound
    prof = rt.kernel_profile()
    l = cfg["model"][0]
    link_s = rep.measured.link_upload * l * args.steps
    h2d_gbs = rep.h2d_weight_bytes / link_s / 1e9 if link_s > 0 else 0.0
    bd = bound.breakdown
    binding = max([("host link (H2D)", bd.link_upload), ("host cores", bd.cpu_attention + bd.cpu_ffn),
                   ("GPU (HBM)", bd.gpu_attention + bd.gpu_ffn)], key=lambda kv: kv[1])[0]
    line = {
        "metric": "decode tokens/sec at fixed GPU-mem budget",
        "value": value, "unit": "tok/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * dev_s / args.steps,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (counter-PRNG weights seed 1234, prompt ids seed 5678, prompt KV seed 9012)",
        "config": config_obj(args, cfg, tp),
        "host": host_info(),
        "run": {"r_w": cfg["r_w"], "weight_codec": "on" if cfg.get("codec") else "off",
                "r_w_achieved": info.achieved_weight_ratio,
                **({"r_w_bound": cfg["r_w_bound"]} if "r_w_bound" in cfg else {}),
                "parallelism_detail": (f"tp{world} (heads + expert h2 sharded, all-reduce x2/layer)"
                                       if world > 1 else
                                       f"tp{tp} job, its largest shard (rank {shard_rank}) measured alone on 1 GPU "
                                       f"(own PCIe link; NVLink all-reduce elided, modeled ~0.5 MB/call)" if tp > 1
                                       else "single GPU, weight paging"),
                "schedule": ("CGOPipe" if cfg["a_g"] == 0 else "S4") if args.schedule == "auto"
                else args.schedule,
                "weight_gates": args.gates,
                "l2": "weights streamed per step (>> 126 MB L2): no flush needed"},
        "hrm": {"bound_tok_s": bound.decode_throughput, "frac": value / bound.decode_throughput,
                "weight_bytes_per_param": cfg.get("stored_dt", CODEC_DT) if cfg.get("codec") else 2.0,
                "weight_bytes_per_param_searched": CODEC_DT if cfg.get("codec") else 2.0,
                "raw_fallback_blocks_per_layer": info.raw_blocks,
                "weight_code": {0: "bf16 tiles", 1: "12-bit (codec 1)", 2: "12-bit (codec 2)", 3: "12-bit (codec 3)",
                                4: "11-bit (codec 4)"}.get(int(info.codec_engine), "?"),
                "bound_bf16_weights_tok_s": bound_bf16.decode_throughput,
                "value_over_bf16_bound": value / bound_bf16.decode_throughput,
                "binding": binding, "link_gbs_measured": link_gbs, "host_read_gbs_measured": host_gbs,
                "host_fp32_tflops_measured": host_flops() / 1e12,
                "modeled_layer_ms": bound.breakdown.layer_total * 1e3,
                "measured_steady_layer_ms": rep.steady_layer_time * 1e3,
                "h2d_weight_gbs_achieved": h2d_gbs,
                "streamed_gb_per_layer_per_gpu": info.streamed_bytes_per_layer / 1e9,
                "utilization": dict(zip(["gpu", "cpu", "h2d", "d2h", "ctopin"], list(rep.utilization)))},
        "roofline": expert_roofline(cfg, rep, pk, load_traffic(bool(cfg.get("codec"))), tp),
        "hrm_kernels": hrm_kernels(cfg, b200_hw(cfg, link_gbs, host_gbs, pk, tp, args.tp_shard > 1), rep, prof,
                                   args.steps, tp, args.roofline_csv),
        "peaks_source": pk_src,
        "e2e": {"value": e2e, "unit": "tok/s",
                "h2d_bytes_per_step": rep.h2d_bytes / args.steps + cfg["N"] * 4 * 2,
                "d2h_bytes_per_step": rep.d2h_bytes / args.steps + cfg["N"] * 4},
        "kernels_ms_per_step": {k["name"]: round(k["ms"] / args.steps, 4) for k in prof["events"]},
        "gemm_exec_ms_per_step": {k["name"]: round(k["ms"] / args.steps, 4) for k in prof["exec"]},
        "gpu_launches": rep.gpu_launches,
        "timeline_ok": bool(rep.timeline_ok),
        "clocks": clocks,
    }
    if prep is not None:
        gen = cfg["gen"]
        n_tok = cfg["N"] * gen
        model_prefill_s = n_tok / bound.generation_throughput - n_tok / bound.decode_throughput
        step_s = dev_s / args.steps
        line["prefill"] = {
            "seconds": prep.seconds, "prompt_tokens": prep.prompt_tokens,
            "tokens_per_second": prep.tokens_per_second,
            "hrm_model_seconds": model_prefill_s, "hrm_frac": model_prefill_s / prep.seconds,
            "chunk_tokens": prep.chunk_tokens, "chunks_per_layer": prep.chunks_per_layer,
            "gpu_busy_seconds": prep.gpu_busy_seconds, "gpu_launches": prep.gpu_launches,
            "h2d_gb": prep.h2d_bytes / 1e9, "d2h_gb": prep.d2h_bytes / 1e9,
            "kv": "computed on the GPU and written to the host cache (A_g=0) / device pool (A_g=1)"}
        line["generation"] = {
            "metric": "generation tok/s = N*gen / (prefill + gen decode steps)",
            "value": n_tok / (prep.seconds + gen * step_s), "unit": "tok/s",
            "decode_steps_measured": args.steps, "gen_len": gen,
            "hrm_bound": bound.generation_throughput,
            "note": "prefill measured; decode time = gen_len x the measured per-step time"}
    del rt
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        # >= 2 whole decode steps of the CPU path on this box's cores
        times, cores, setup = cpu_decode(cfg, 0, 2)
        line["cpu_baseline"] = {"value": cfg["N"] * len(times) / sum(times), "unit": "tok/s", "cores": cores,
                                "kind": "port",
                                "sample": f"2 whole decode steps (all {l} layers, N={cfg['N']}, ctx {cfg['prompt']}"
                                          f"..{cfg['prompt'] + 1}) of the fp32 CPU oracle (step s: "
                                          f"{', '.join(f'{x:.2f}' for x in times)}; build {setup:.1f} s untimed)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mlt", choices=["mlt", "reference"])
    ap.add_argument("--config", default="mixtral8x7b-16g", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gates", default="exact", choices=["exact", "reference"],
                    help="weight gates: data-exact (default) or the reference's all-pages gate")
    ap.add_argument("--schedule", default="auto", choices=["auto", "cgopipe", "s2", "s3", "s4"],
                    help="executed schedule: CGOPipe (S4 when A_g=1) or a baseline of pipesim.hpp")
    ap.add_argument("--prefill", action="store_true",
                    help="run the GPU prefill on synthetic prompt ids instead of synthetic prompt KV")
    ap.add_argument("--timeline", default=None, help="write the measured timeline JSON here")
    ap.add_argument("--roofline-csv", default=None,
                    help="write the hot kernels' roofline series (lightplan::roofline_csv) here")
    ap.add_argument("--codec", default="auto", choices=["auto", "on", "off"],
                    help="store/stream/read weights as lossless encoded tiles (runtime/weight_codec.hpp); "
                         "auto = on when weights are paged over the host link (r_w < 1), off when resident")
    ap.add_argument("--no-pdl", action="store_true",
                    help="no programmatic dependent launch on all-GPU schedules (per-kernel event breakdown)")
    ap.add_argument("--tp-shard", type=int, default=0,
                    help="measure the largest shard of a T-way TP job alone on one GPU (all-reduce elided)")
    ap.add_argument("--down-splits", type=int, default=0,
                    help="K-splits of the expert down GEMM (0 = auto: wave fill with the codec, 1 raw)")
    ap.add_argument("--host-threads", type=int, default=0,
                    help="host attention threads (0 = all cores but two, split across co-located ranks)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    rw0 = cfg["r_w"] if not isinstance(cfg["r_w"], dict) else min(cfg["r_w"].values())
    cfg["codec"] = args.codec == "on" or (args.codec == "auto" and rw0 < 1.0)
    if isinstance(cfg["r_w"], dict):
        world = args.tp_shard if args.tp_shard > 1 else int(os.environ.get("WORLD_SIZE", "1"))
        if world not in cfg["r_w"]:
            raise SystemExit(f"{args.config}: no policy for {world} GPUs (h2/tp must keep 128-row blocks)")
        cfg["r_w"] = cfg["r_w"][world]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_mlt(args, cfg)


if __name__ == "__main__":
    main()
