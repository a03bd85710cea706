"""HRM policy sweep on one B200 (BASELINE.json configs[2]): Mixtral-8x7B shape,
N=256, prompt 512, budgets 16/32/64 GB x micro-batch size x attention
placement.  For every (budget, mu, A_g) the product's search_policy
(planner.cpp:234-341, bit-identical) picks the best feasible r_w on the
MEASURED B200 spec; the runtime then executes that policy and the measured
decode tok/s is compared with its HRM bound.  Also reports whether the
search's global optimum per budget is the measured optimum (the plan ->
execute loop of SURVEY.md §8f rank 3).

  python tools/hrm_sweep.py [--budgets 16,32,64] [--mus 32,64,128,256] [--steps 2]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402  (model/bound helpers, live link + host measurements)
from paper_2411_11217_b200 import capi  # noqa: E402
from paper_2411_11217_b200.runtime import Runtime  # noqa: E402

# the search runs on m_g = budget - bench.arena_extra (embedding + lm_head +
# activations, which ModelSpec does not model), the runtime on the budget
RESERVE = 0.82e9  # bench.arena_extra for the 8x7B shape (reported)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budgets", default="16,32,64")
    ap.add_argument("--mus", default="32,64,128,256")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--out", default=None)
    ap.add_argument("--codec", action="store_true", help="weights stored/streamed/read as encoded tiles")
    a = ap.parse_args()
    import ctypes as C
    api = capi.load_product()
    pk, pk_src = bench.peaks()
    f = api.lib.mlt_measure_link
    f.restype, f.argtypes = C.c_int, [C.c_int, C.c_size_t, C.c_int, C.POINTER(C.c_double)]
    link = (C.c_double * 3)()
    api.check(f(0, 1 << 30, 5, link))
    host = bench.measure_host(api)
    print(f"[sweep] link {link[0]:.2f} GB/s, host read {host:.1f} GB/s", file=sys.stderr, flush=True)
    model_t = (32, 4096, 14336, 32, 8, 8, 2)
    N, prompt, gen = 256, 512, 32
    l = model_t[0]
    rows = []
    for budget_gb in [float(x) for x in a.budgets.split(",")]:
        cfg0 = dict(model=model_t, N=N, prompt=prompt, gen=gen, budget=budget_gb * 1e9, codec=a.codec)
        hw = capi.HardwareSpec(budget_gb * 1e9 - bench.arena_extra(dict(cfg0, vocab=32000)), 196e9, pk["hbm_gbs"] * 1e9, host * 1e9,
                               link[0] * 1e9, pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) * 1e12,
                               bench.host_flops())
        w = capi.WorkloadSpec(prompt, gen)
        for mu in [int(x) for x in a.mus.split(",")]:
            for a_g in (0, 1):
                grid = capi.make_grid([mu], [N // mu], [round(0.01 * i, 2) for i in range(101)],
                                      [1.0] if a_g else [0.0], attn=(a_g,), ffn=(1,))
                try:
                    plan = api.search_policy(hw, bench.model_spec(cfg0, stored=True), w, grid)
                except capi.MltError as e:
                    rows.append({"budget_gb": budget_gb, "mu": mu, "A_g": a_g, "feasible": False,
                                 "why": str(e)[:160]})
                    print(f"[sweep] {budget_gb:.0f} GB mu={mu} A_g={a_g}: infeasible", file=sys.stderr,
                          flush=True)
                    continue
                r_w = plan.policy.weights_on_gpu
                cfg = dict(cfg0, mu=mu, a_g=a_g, r_w=r_w)
                bound = bench.hrm_bound(cfg, link[0], host, pk)
                t = time.perf_counter()
                try:
                    rt = Runtime(bench.model_spec(cfg), bench.policy(cfg), budget_bytes=cfg["budget"],
                                 max_ctx=prompt + a.steps + a.warmup + 8, vocab=32000, weight_codec=a.codec)
                except capi.MltError as e:  # e.g. the arena's extras push it over the cap
                    rows.append({"budget_gb": budget_gb, "mu": mu, "A_g": a_g, "r_w": r_w, "feasible": False,
                                 "why": "runtime: " + str(e)[:160]})
                    continue
                setup = time.perf_counter() - t
                rt.prefill_synthetic(prompt, 9012)
                toks = np.random.default_rng(5678).integers(0, 32000, N, dtype=np.int32)
                wu = rt.decode(toks, a.warmup)
                d = rt.decode(wu.ids[-1], a.steps)
                rep = d.report
                val = N * a.steps / rep.seconds
                if a.codec:  # the bound at the bytes per weight the runtime stored (bench.py does the same)
                    try:
                        bound = bench.hrm_bound(dict(cfg, stored_dt=rt.info.bytes_per_weight), link[0], host, pk)
                    except capi.InfeasiblePolicyError:
                        pass
                row = {"budget_gb": budget_gb, "mu": mu, "A_g": a_g, "r_w": r_w,
                       "r_w_achieved": rt.info.achieved_weight_ratio, "feasible": True,
                       "hrm_bound_tok_s": bound.decode_throughput, "measured_tok_s": val,
                       "stored_bytes_per_weight": rt.info.bytes_per_weight if a.codec else 2.0,
                       "frac": val / bound.decode_throughput,
                       "search_objective_tok_s": plan.decode_throughput,
                       "modeled_layer_ms": bound.breakdown.layer_total * 1e3,
                       "measured_steady_layer_ms": rep.steady_layer_time * 1e3,
                       "utilization": dict(zip(["gpu", "cpu", "h2d", "d2h", "ctopin"], list(rep.utilization))),
                       "timeline_ok": bool(rep.timeline_ok), "setup_s": setup,
                       "arena_gb": rt.info.arena_used / 1e9}
                rows.append(row)
                print(f"[sweep] {budget_gb:.0f} GB mu={mu} A_g={a_g} r_w={r_w:.2f}: {val:.1f} tok/s, "
                      f"bound {bound.decode_throughput:.1f} ({100 * row['frac']:.1f}%)", file=sys.stderr, flush=True)
                rt.close()
                del rt
    summary = {}
    for b in sorted({r["budget_gb"] for r in rows}):
        ok = [r for r in rows if r["budget_gb"] == b and r["feasible"]]
        if not ok:
            continue
        best_model = max(ok, key=lambda r: r["hrm_bound_tok_s"])
        best_meas = max(ok, key=lambda r: r["measured_tok_s"])
        summary[f"{b:.0f}GB"] = {
            "search_optimum": {k: best_model[k] for k in ("mu", "A_g", "r_w", "hrm_bound_tok_s", "measured_tok_s")},
            "measured_optimum": {k: best_meas[k] for k in ("mu", "A_g", "r_w", "hrm_bound_tok_s", "measured_tok_s")},
            "search_pick_within_pct_of_measured_best": 100 * best_model["measured_tok_s"] / best_meas["measured_tok_s"]}
    out = {"what": "HRM policy sweep, Mixtral-8x7B shape, N=256, prompt 512, 1x B200 (tools/hrm_sweep.py)"
                   + (f", weights encoded (weight codec, {bench.CODEC_DT * 8192:.0f} B per 16 KiB tile)" if a.codec else ""),
           "link_gbs": link[0], "host_read_gbs": host, "peaks_source": pk_src, "search_reserve_gb": RESERVE / 1e9,
           "decode_steps": a.steps, "rows": rows, "summary": summary}
    js = json.dumps(out, indent=1)
    if a.out:
        with open(a.out, "w") as fh:
            fh.write(js)
    print(js)


if __name__ == "__main__":
    main()
