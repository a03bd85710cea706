"""Per-CTA phase timeline of the tcgen05 GEMM (gemm_tc.cu trace stamps):
entry, setup done, first weight copy issued, first stage full (first data
landed), last MMA issued, first accumulator ready, epilogue done, exit —
as offsets from the earliest CTA entry, min / median / max over CTAs.

  python tools/trace_gemm.py [--mu 64]
"""
import argparse
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_11217_b200 import capi  # noqa: E402

PHASES = ["entry", "setup", "1st_issue", "1st_full", "mma_done", "1st_acc", "epi_done", "exit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mu", type=int, default=64)
    a = ap.parse_args()
    mu, H = a.mu, 4096
    KD = capi.load_kernels()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    Rmu = (mu + 15) // 16 * 16
    xn = (torch.randn(Rmu * H, device="cuda") * 0.1).to(torch.bfloat16)
    out = torch.zeros(8 * Rmu * 6144, device="cuda")
    tr = torch.zeros(148 * 8, dtype=torch.int64, device="cuda")
    for name, M, ks, alpha in (("qkv", 6144, 3, 1.0), ("o", 4096, 4, 1.0)):
        copies = []
        for _ in range(4):
            w = (torch.randn(M * H, device="cuda") * 0.02).to(torch.bfloat16)
            tab = torch.tensor([w.data_ptr() + rb * 128 * H * 2 for rb in range(M // 128)],
                               dtype=torch.int64, device="cuda")
            copies.append((w, tab))
        cap = min(256, Rmu)
        for i in range(6):
            tr.zero_()
            g = capi.GemmArgs(a_table=copies[i % 4][1].data_ptr(), n_mats=1, G=1, RB=M // 128, K=H,
                              b=xn.data_ptr(), R=Rmu, rows_dense=mu, n_cap=cap, epi=0,
                              out_f32=out.data_ptr(), ldo=M, n_chunks=1, k_splits=ks,
                              split_stride=Rmu * M, trace=tr.data_ptr(), alpha=alpha)
            KD.gemm(C.byref(g), s)
            torch.cuda.synchronize()
        t = tr.view(148, 8).cpu().numpy().astype(np.int64)
        t = t[t[:, 0] > 0]
        base = t[:, 0].min()
        rel = (t - base) / 1e3
        print(f"{name} mu={mu} k_splits={ks}: {len(t)} CTAs, span {rel[:, 7].max():.2f} us")
        for j, p in enumerate(PHASES):
            col = rel[:, j]
            print(f"  {p:10s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")


if __name__ == "__main__":
    main()
