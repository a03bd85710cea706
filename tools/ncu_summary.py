"""Condense an ncu --set full report into a per-kernel JSON summary (duration,
DRAM bytes and GB/s, achieved fraction of the measured HBM peak, SM / memory
throughput, tensor-pipe and ALU utilisation, top stall reasons).

  python tools/ncu_summary.py report.ncu-rep [--out summary.json]
"""
import argparse
import csv
import io
import json
import os
import subprocess

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__grid_size", "launch__block_size",
           "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
           "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
           "sm__cycles_elapsed.avg.per_second"]
UNIT = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
        "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--out", default=None)
    ap.add_argument("--peak-gbs", type=float, default=None)
    a = ap.parse_args()
    peak = a.peak_gbs
    if peak is None:
        p = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
        peak = json.load(open(p))["hbm_gbs"] if os.path.exists(p) else 6650.0
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))

        def val(m):
            v = d.get(m, "")
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                return None
            return x * UNIT.get(u.get(m, ""), 1.0)
        t = val("gpu__time_duration.sum")
        rd, wr = val("dram__bytes_read.sum") or 0.0, val("dram__bytes_write.sum") or 0.0
        k = {"kernel": d.get("Kernel Name", "")[:120], "id": d.get("ID"),
             "grid": d.get("launch__grid_size"), "block": d.get("launch__block_size"),
             "duration_us": t * 1e6 if t else None, "dram_read_bytes": rd, "dram_write_bytes": wr,
             "dram_gbs": (rd + wr) / t / 1e9 if t else None}
        k["frac_of_hbm_peak"] = k["dram_gbs"] / peak if k["dram_gbs"] else None
        for m in METRICS[3:]:
            if m in d and m not in ("launch__grid_size", "launch__block_size"):
                k[m] = val(m)
        out.append(k)
    js = json.dumps({"report": os.path.basename(a.rep), "hbm_peak_gbs": peak,
                     "note": "ncu replays each kernel with flushed caches (--cache-control all): durations are "
                             "cold-cache and serialised; shares, traffic and pipe utilisation are the evidence",
                     "kernels": out}, indent=1)
    if a.out:
        open(a.out, "w").write(js)
    print(js)


if __name__ == "__main__":
    main()
