"""GEMM accuracy: mlt tcgen05 GEMM vs fp64 ground truth, next to cuBLAS bf16."""
import sys, ctypes as C, numpy as np, torch
sys.path.insert(0, '.')
from paper_2411_11217_b200 import capi
K_ = capi.load_kernels()
def ptr(t): return C.c_void_p(t.data_ptr())
for (T, M, Kd) in [(8, 1536, 1024), (64, 4096, 4096), (64, 1024, 3584)]:
    g = torch.Generator().manual_seed(1)
    w = (torch.rand(M, Kd, generator=g) * 2 - 1).mul(3 ** 0.5 / Kd ** 0.5).to(torch.bfloat16)
    x = (torch.randn(T, Kd, generator=g)).to(torch.bfloat16)
    src = w.contiguous().view(torch.int16).numpy().view(np.uint16)
    dst = np.empty_like(src)
    K_.pack_weight(src.ctypes.data_as(C.c_void_p), M, Kd, dst.ctypes.data_as(C.c_void_p))
    wd = torch.from_numpy(dst.view(np.int16).copy()).cuda()
    tab = torch.tensor([wd.data_ptr() + rb * 128 * Kd * 2 for rb in range(M // 128)], dtype=torch.int64, device='cuda')
    R = (T + 15) // 16 * 16
    xp = torch.zeros(R * Kd, dtype=torch.int16, device='cuda')
    xd = x.cuda()
    K_.pack_rows(ptr(xd), Kd, T, Kd, ptr(xp), R, C.c_void_p(0))
    out = torch.zeros(R, M, device='cuda')
    a = capi.GemmArgs(a_table=tab.data_ptr(), n_mats=1, G=1, RB=M // 128, K=Kd, b=xp.data_ptr(), R=R,
                      rows_dense=T, n_cap=min(256, R), epi=0, alpha=1.0, out_f32=out.data_ptr(), ldo=M)
    K_.gemm(C.byref(a), C.c_void_p(0)); torch.cuda.synchronize()
    exact = x.double() @ w.double().T
    f32seq = (x.float() @ w.float().T)  # CPU fp32 (blocked)
    cub = (xd @ w.cuda().T.contiguous().T.T).float().cpu() if False else torch.matmul(xd.float(), w.cuda().float().T).cpu()
    cub_bf16out = torch.matmul(xd, w.cuda().T).float().cpu()
    def rel(a): return ((a.double() - exact).norm() / exact.norm()).item()
    def mx(a): return ((a.double() - exact).abs().max() / exact.abs().max()).item()
    print(f"T={T} M={M} K={Kd}: mlt rel={rel(out[:T].cpu()):.2e} max={mx(out[:T].cpu()):.2e} | cpu fp32 rel={rel(f32seq):.2e} | torch fp32(TF32?) rel={rel(cub):.2e} | cublas bf16 (bf16 out) rel={rel(cub_bf16out):.2e}")
