"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum
--clock-control none --csv --log-file X.csv ...`) per kernel: launches,
mean / total microseconds, share of the summed kernel time.

  python tools/launch_summary.py gpurun_out/launches.csv [--json out.json]
"""
import argparse
import collections
import csv
import json
import re


def summarise(path):
    hdr, agg = None, collections.OrderedDict()
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if not hdr or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        u = d["Metric Unit"]
        v = v / 1e3 if u in ("ns", "nsecond") else v * 1e3 if u in ("ms", "msecond") else v
        name = re.sub(r"\(.*", "", d["Kernel Name"]).replace("(anonymous namespace)::", "")
        name = name.split("::")[-1].split("<")[0] + ("<" + d["Kernel Name"].split("<")[1].split(">")[0] + ">"
                                                      if "<" in d["Kernel Name"] else "")
        agg.setdefault(name, []).append(v)
    total = sum(sum(v) for v in agg.values())
    out = {k: {"launches": len(v), "mean_us": sum(v) / len(v), "total_us": sum(v),
               "share": sum(v) / total if total else 0.0} for k, v in agg.items()}
    return out, total


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    out, total = summarise(a.csv)
    for k, v in sorted(out.items(), key=lambda kv: -kv[1]["total_us"]):
        print(f"{k:40s} n={v['launches']:5d} mean={v['mean_us']:9.2f} us  total={v['total_us'] / 1e3:9.3f} ms"
              f"  {100 * v['share']:5.1f}%")
    print(f"{'sum':40s} {total / 1e3:.3f} ms")
    if a.json:
        json.dump({"source": a.csv, "total_us": total, "kernels": out}, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
