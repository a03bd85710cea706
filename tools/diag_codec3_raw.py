"""Bisect: codec-3 grouped gate/up on ALL-raw (tagged) weight blocks vs codec 0."""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from paper_2411_11217_b200 import capi  # noqa: E402

T, H, Fd, E, Kk, ncap, nm, sk, rawflag = (int(x) for x in sys.argv[1:10])
K = capi.load_kernels()
s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
g = torch.Generator().manual_seed(1)
R = (T * Kk + 16 * E + 15) // 16 * 16
per = max(1, T * Kk // E)
cnt = torch.tensor([per if e < T * Kk // per else 0 for e in range(E)], dtype=torch.int32, device="cuda")
off = torch.tensor([e * ((per + 15) // 16 * 16) for e in range(E + 1)], dtype=torch.int32, device="cuda")
xp = (torch.randn(R * H, generator=g) * 0.1).to(torch.bfloat16).cuda()
w = ((torch.rand(Fd, H, generator=g) * 2 - 1) * 0.03).to(torch.bfloat16)
src = w.view(torch.int16).numpy().view(np.uint16)
packed = np.empty_like(src)
K.pack_weight(src.ctypes.data_as(C.c_void_p), Fd, H, packed.ctypes.data_as(C.c_void_p))
dev = torch.from_numpy(packed.view(np.int16)).cuda()
Rmu = (T + 15) // 16 * 16
sk_scratch = torch.zeros(148 * 2 * Rmu * 128, device="cuda")
sk_count = torch.zeros(148, dtype=torch.int64, device="cuda")
enc = np.zeros(Fd // 128 * (H // 64) * 12432, np.uint8)
assert K.codec_encode_rows(packed.ctypes.data_as(C.c_void_p), Fd, H, enc.ctypes.data_as(C.c_void_p), None) == 0
enc_d = torch.from_numpy(enc).cuda()
outs = []
for codec in (0, 3):
    tag = rawflag if codec == 3 else 0
    src_d, tb = (dev, 128 * H * 2) if (codec == 0 or tag) else (enc_d, (H // 64) * 12432)
    tab = torch.tensor([src_d.data_ptr() + rb * tb + tag for m in range(nm) for e in range(E)
                        for rb in range(Fd // 128)], dtype=torch.int64, device="cuda")
    if nm == 2:
        out = torch.zeros(R * Fd, dtype=torch.int16, device="cuda")
        a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=2, G=E, RB=Fd // 128, K=H, b=xp.data_ptr(), R=R,
                          b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=ncap, epi=1, alpha=1.0,
                          out_packed=out.data_ptr(), out_R=R, codec=codec, codec_raw=tag,
                          sk_scratch=sk_scratch.data_ptr() if sk else None, sk_count=sk_count.data_ptr(), sk_rows=Rmu)
    else:
        out = torch.zeros(R * Fd, device="cuda")
        a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=E, RB=Fd // 128, K=H, b=xp.data_ptr(), R=R,
                          b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=ncap, epi=0, alpha=1.0,
                          out_f32=out.data_ptr(), ldo=Fd, codec=codec, codec_raw=tag)
    K.gemm(C.byref(a), s)
    torch.cuda.synchronize()
    outs.append(out.cpu())
print("equal" if torch.equal(outs[0], outs[1]) else "DIFF", sys.argv[1:])
