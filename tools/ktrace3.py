"""CTA-0 pipeline trace of the codec-3 expert GEMM (gemm_tc.cu ktrace, codec 3):
per weight tile %globaltimer stamps — producer issue, landed (decoder saw
the slot full), decoded, TMEM slot granted, stored (dfull), MMA start.
Prints median stage latencies and the steady-state tile interval.

  python tools/ktrace3.py [--mu 64] [--down]
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
    ap.add_argument("--down", action="store_true")
    a = ap.parse_args()
    KD = capi.load_kernels()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    per_e = a.mu * 2 // E
    cnt = torch.full((E,), per_e, dtype=torch.int32, device="cuda")
    off = torch.tensor([e * ((per_e + 15) // 16 * 16) for e in range(E + 1)], dtype=torch.int32, device="cuda")
    R = int(off[-1].item()) + 16
    xp = (torch.randn(R * H, device="cuda") * 0.1).to(torch.bfloat16)
    inter = torch.zeros(R * F, dtype=torch.int16, device="cuda")
    M, Kd = (H, F) if a.down else (F, H)
    g = torch.Generator().manual_seed(1)
    w = ((torch.rand(M, Kd, generator=g) * 2 - 1) * (3.0 / Kd) ** 0.5).to(torch.bfloat16)
    src = w.view(torch.int16).numpy().view(np.uint16)
    packed = np.empty_like(src)
    KD.pack_weight(src.ctypes.data_as(C.c_void_p), M, Kd, packed.ctypes.data_as(C.c_void_p))
    enc = np.zeros(M // 128 * (Kd // 64) * 12432, np.uint8)
    assert KD.codec_encode_rows(packed.ctypes.data_as(C.c_void_p), M, Kd, enc.ctypes.data_as(C.c_void_p), None) == 0
    enc_d = torch.from_numpy(enc).cuda()
    ym = torch.zeros(4 * R * H, device="cuda")
    kt = torch.zeros(6 * 256, dtype=torch.int64, device="cuda")
    nm = 1 if a.down else 2
    tab = torch.tensor([enc_d.data_ptr() + rb * (Kd // 64) * 12432 for m in range(nm) for e in range(E)
                        for rb in range(M // 128)], dtype=torch.int64, device="cuda")
    ncap = min(128, (a.mu + 15) // 16 * 16)
    if a.down:
        args = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=E, RB=M // 128, K=Kd, b=inter.data_ptr(), R=R,
                             b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=ncap, epi=0, alpha=1.0,
                             out_f32=ym.data_ptr(), ldo=H, codec=3, k_splits=4, split_stride=R * H,
                             ktrace=kt.data_ptr())
    else:
        args = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=2, G=E, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                             b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=ncap, epi=1, alpha=1.0,
                             out_packed=inter.data_ptr(), out_R=R, codec=3, ktrace=kt.data_ptr())
    for _ in range(3):
        kt.zero_()
        KD.gemm(C.byref(args), s)
        torch.cuda.synchronize()
    t = kt.view(6, 256).cpu().numpy().astype(np.int64)
    rel = (t - t[0, 0]) / 1e3
    n = 240
    iss, land, dec, slot, stored, mma = (rel[i, :n] for i in range(6))
    lo = 40
    print(f"tile interval (MMA start) median {np.median(np.diff(mma[lo:n])) * 1e3:.0f} ns; "
          f"producer issue interval {np.median(np.diff(iss[lo:n])) * 1e3:.0f} ns")
    for name, x, y in (("issue->landed", iss, land), ("landed->decoded", land, dec), ("decoded->slot", dec, slot),
                       ("slot->stored", slot, stored), ("stored->mma", stored, mma), ("issue->mma", iss, mma)):
        print(f"  {name:16s} median {np.median((y - x)[lo:n]) * 1e3:7.0f} ns")
    for i in range(0, 40):
        print(f"   t {i:3d}: issue {iss[i]:8.3f} land {land[i]:8.3f} dec {dec[i]:8.3f} slot {slot[i]:8.3f} "
              f"st {stored[i]:8.3f} mma {mma[i]:8.3f}")


if __name__ == "__main__":
    main()
