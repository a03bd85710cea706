"""One rank of a tensor-parallel decode run through the product runtime
(tests/test_tp_gpu.py launches two of these on ONE GPU).  Not a test module.

  python tests/tp_worker.py --rank R --size S --name KEY --dims h1,h2,nq,nkv
        --out FILE [--a-g 0|1] [--r-w X] [--budget B]

Each rank builds mlt_runtime with tp_rank/tp_size and the host-staged
all-reduce (collective = 1, rendezvous KEY) and decodes STEPS teacher-forced
steps (fixed synthetic ids, seed 5678), one step per call with the router tap
armed, saving per step its greedy ids, residual and every layer's top-k
choice, plus report fields, to FILE (.npz)."""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2411_11217_b200 import capi  # noqa: E402
from paper_2411_11217_b200.runtime import Runtime  # noqa: E402

N, MU, STEPS, VOCAB = 8, 4, 24, 32000


def run(rank, size, name, dims, out, a_g=0, r_w=0.0, budget=4e9, layers=2, experts=8, top_k=2, codec=False):
    h1, h2, nq, nkv = dims
    model = capi.ModelSpec(layers, h1, h2, nq, nkv, experts, top_k, 2.0, 2.0)
    pol = capi.Policy(N, MU, a_g, 1, r_w, 1.0 if a_g else 0.0)
    kw = dict(budget_bytes=budget, max_ctx=64, vocab=VOCAB, seed=1234, weight_codec=codec)
    if size > 1:
        kw.update(tp_rank=rank, tp_size=size, nccl_id=name.encode(), collective="host")
    rt = Runtime(model, pol, **kw)
    toks = forced_tokens()
    ids, xs, routes, ok = [], [], [], 1
    for s in range(STEPS):
        rt.capture_router(1)
        d = rt.decode(toks[s], 1)
        ok = min(ok, d.report.timeline_ok)
        ids.append(d.ids[0])
        xs.append(rt.residual())
        routes.append(rt.captured_router()[1])
    np.savez(out, ids=np.array(ids), x=np.array(xs), routes=np.array(routes),
             streamed=rt.info.streamed_bytes_per_layer, timeline_ok=ok, h2d=d.report.h2d_weight_bytes)
    rt.close()


def forced_tokens():
    return np.random.default_rng(5678).integers(0, VOCAB, size=(STEPS, N), dtype=np.int32)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int, default=0)
    ap.add_argument("--size", type=int, default=1)
    ap.add_argument("--name", default="")
    ap.add_argument("--dims", required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--a-g", type=int, default=0)
    ap.add_argument("--r-w", type=float, default=0.0)
    ap.add_argument("--budget", type=float, default=4e9)
    ap.add_argument("--codec", action="store_true")
    a = ap.parse_args()
    run(a.rank, a.size, a.name, tuple(int(x) for x in a.dims.split(",")), a.out, a.a_g, a.r_w, a.budget,
        codec=a.codec)
