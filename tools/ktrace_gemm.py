"""CTA-0 pipeline trace of the expert gate/up GEMM (gemm_tc.cu ktrace):
per k-block %globaltimer stamps of producer issue, decoder start (stage
landed), decoder done and MMA start, raw vs encoded weights.  Prints the
median stage latency and the steady-state issue interval.

  python tools/ktrace_gemm.py [--mu 64]
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

H, F, E = 4096, 14336, 8


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mu", type=int, default=64)
    ap.add_argument("--down", action="store_true", help="the down GEMM (K = h2, 4 K-splits) instead of gate/up")
    ap.add_argument("--dec-groups", type=int, default=0)
    a = ap.parse_args()
    KD = capi.load_kernels()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    per_e = a.mu * 2 // E  # tokens per expert (uniform routing)
    cnt = torch.full((E,), per_e, dtype=torch.int32, device="cuda")
    off = torch.tensor([e * ((per_e + 15) // 16 * 16) for e in range(E + 1)], dtype=torch.int32, device="cuda")
    R = int(off[-1].item()) + 16
    xp = (torch.randn(R * H, device="cuda") * 0.1).to(torch.bfloat16)
    inter = torch.zeros(R * F, dtype=torch.int16, device="cuda")
    M, Kd = (H, F) if a.down else (F, H)  # weight rows, reduction length
    g = torch.Generator().manual_seed(1)
    w = ((torch.rand(M, Kd, generator=g) * 2 - 1) * (3.0 / Kd) ** 0.5).to(torch.bfloat16)
    src = w.view(torch.int16).numpy().view(np.uint16)
    packed = np.empty_like(src)
    KD.pack_weight(src.ctypes.data_as(C.c_void_p), M, Kd, packed.ctypes.data_as(C.c_void_p))
    enc = np.zeros(M // 128 * (Kd // 64) * 12432, np.uint8)
    KD.codec_encode(packed.ctypes.data_as(C.c_void_p), M, Kd, enc.ctypes.data_as(C.c_void_p))
    ym = torch.zeros(4 * R * H, device="cuda")
    raw_d = torch.from_numpy(packed.view(np.int16)).cuda()
    enc_d = torch.from_numpy(enc).cuda()
    kt = torch.zeros(4 * 256, dtype=torch.int64, device="cuda")
    for codec, dev, tile in ((0, raw_d, 16384), (1, enc_d, 12432)):
        # every (mat, expert) uses the same weight matrix: bandwidth is what is measured
        nm = 1 if a.down else 2
        tab = torch.tensor([dev.data_ptr() + rb * (Kd // 64) * tile for m in range(nm) for e in range(E)
                            for rb in range(M // 128)], dtype=torch.int64, device="cuda")
        if a.down:
            args = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=E, RB=M // 128, K=Kd, b=inter.data_ptr(), R=R,
                                 b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=min(128, (a.mu + 15) // 16 * 16),
                                 epi=0, alpha=1.0, out_f32=ym.data_ptr(), ldo=H, codec=codec, k_splits=4,
                                 split_stride=R * H, ktrace=kt.data_ptr(), dec_groups=a.dec_groups)
        else:
            args = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=2, G=E, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                                 b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=min(128, (a.mu + 15) // 16 * 16),
                                 epi=1, alpha=1.0, out_packed=inter.data_ptr(), out_R=R, codec=codec,
                                 ktrace=kt.data_ptr(), dec_groups=a.dec_groups)
        for _ in range(3):
            kt.zero_()
            KD.gemm(C.byref(args), s)
            torch.cuda.synchronize()
        t = kt.view(4, 256).cpu().numpy().astype(np.int64)
        base = t[0, 0]
        rel = (t - base) / 1e3
        n = 200
        issue, dstart, ddone, mma = rel[0, :n], rel[1, :n], rel[2, :n], rel[3, :n]
        iv = np.diff(issue[50:n])
        print(f"codec={codec}: stage issue interval median {np.median(iv) * 1e3:.0f} ns (stage = 2 tiles)")
        if codec:
            print(f"  MMA start interval median {np.median(np.diff(mma[50:n])) * 1e3:.0f} ns")
            print(f"  land latency (issue->decoder start) median {np.median(dstart - issue) * 1e3:.0f} ns, "
                  f"decode median {np.median(ddone - dstart) * 1e3:.0f} ns, "
                  f"decoded->MMA median {np.median(mma - ddone) * 1e3:.0f} ns")
        print(f"  issue->MMA start median {np.median(mma - issue) * 1e3:.0f} ns")
        for i in range(0, 24):
            print(f"   kb {i:3d}: issue {issue[i]:8.3f} dec {dstart[i]:8.3f}-{ddone[i]:8.3f} mma {mma[i]:8.3f}")


if __name__ == "__main__":
    main()
