"""Tiling sweep of the tcgen05 weight-streaming GEMM (gemm_tc.cu) at the dense
projection shapes of Mixtral-8x7B decode: QKV (6144 x 4096) and O (4096 x
4096) for mu tokens, over (n_cap, n_chunks, k_splits).  Four weight copies
rotate so every launch streams its weights from HBM (4 x 50 MB > L2).

  python tools/sweep_gemm.py [--mu 256]
"""
import argparse
import ctypes as C
import itertools
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_11217_b200 import capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mu", type=int, default=256)
    ap.add_argument("--reps", type=int, default=40)
    a = ap.parse_args()
    mu, H = a.mu, 4096
    KD = capi.load_kernels()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    Rmu = (mu + 15) // 16 * 16
    xn = (torch.randn(Rmu * H, device="cuda") * 0.1).to(torch.bfloat16)
    out = torch.zeros(8 * Rmu * 6144, device="cuda")
    res = []
    for name, M in (("qkv", 6144), ("o", 4096)):
        copies = []
        for _ in range(4):
            w = (torch.randn(M * H, device="cuda") * 0.02).to(torch.bfloat16)
            tab = torch.tensor([w.data_ptr() + rb * 128 * H * 2 for rb in range(M // 128)],
                               dtype=torch.int64, device="cuda")
            copies.append((w, tab))
        caps = sorted({min(256, Rmu), min(128, Rmu), min(64, Rmu)})
        for cap, ks in itertools.product(caps, (1, 2, 3, 4, 6, 8)):
            ch = (mu + cap - 1) // cap
            if (M // 128) * ch * ks > 4 * 148 or ks > H // 64:
                continue

            def launch(i):
                g = capi.GemmArgs(a_table=copies[i % 4][1].data_ptr(), n_mats=1, G=1, RB=M // 128, K=H,
                                  b=xn.data_ptr(), R=Rmu, rows_dense=mu, n_cap=cap, epi=0, alpha=1.0,
                                  out_f32=out.data_ptr(), ldo=M, n_chunks=ch, k_splits=ks,
                                  split_stride=Rmu * M)
                KD.gemm(C.byref(g), s)
            for i in range(4):
                launch(i)
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            st.record()
            for i in range(a.reps):
                launch(i)
            en.record()
            torch.cuda.synchronize()
            us = st.elapsed_time(en) / a.reps * 1e3
            gbs = M * H * 2 / (us * 1e-6) / 1e9
            tiles = (M // 128) * ch * ks
            print(f"{name:4s} mu={mu:4d} n_cap={cap:4d} chunks={ch} k_splits={ks} tiles={tiles:4d}  "
                  f"{us:7.2f} us  {gbs:7.1f} GB/s", flush=True)
            res.append({"gemm": name, "mu": mu, "n_cap": cap, "n_chunks": ch, "k_splits": ks, "us": us,
                        "weight_gbs": gbs})
    print(json.dumps(res))


if __name__ == "__main__":
    main()
