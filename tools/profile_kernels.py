"""Kernel microbenchmark at Mixtral-8x7B decode shapes (mu tokens per launch).

Times each hot kernel with CUDA events (warm, back-to-back, weights > L2 so
every launch streams from HBM) and prints achieved GB/s against the
measured HBM peak.  Used standalone and under ncu (`--once` runs each kernel
a fixed small number of times for a capture).

  python tools/profile_kernels.py [--mu 64] [--once]
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_11217_b200 import capi  # noqa: E402

H, F, E, K, NQ, NKV, D, V = 4096, 14336, 8, 2, 32, 8, 128, 32000
W = (NQ + 2 * NKV) * D


def ptr(t):
    return C.c_void_p(t.data_ptr())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mu", type=int, default=64)
    ap.add_argument("--once", action="store_true")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--with-h2d", action="store_true", help="run a concurrent H2D copy stream")
    ap.add_argument("--codec", action="store_true", help="encoded weight tiles (decoder warps in the GEMM)")
    ap.add_argument("--codec2", action="store_true",
                    help="fragment-order encoded tiles, register decode + mma.sync (gemm_codec.cu)")
    ap.add_argument("--codec3", action="store_true",
                    help="row-plane encoded tiles decoded into TMEM, MMA with A from TMEM (gemm_tc codec 3)")
    ap.add_argument("--codec4", action="store_true",
                    help="3-bit row-plane tiles (11600 B) on the TMEM-operand engine (gemm_tc codec 4)")
    ap.add_argument("--only", default="", help="comma-separated case-name prefixes to run")
    ap.add_argument("--ncap-e", type=int, default=0, help="expert GEMM token tile (0: the runtime's min(128, Rmu))")
    ap.add_argument("--no-stream-k", action="store_true", help="gate/up without the stream-K tail")
    ap.add_argument("--dec-groups", type=int, default=0, help="codec decoder groups (0: default)")
    ap.add_argument("--down-splits", type=int, default=0,
                    help="K-splits of the down GEMM (0: the runtime's auto choice, 4 with --codec at 8x7B)")
    a = ap.parse_args()
    if a.codec2 or a.codec3 or a.codec4:
        a.codec = True
    TB = 11600 if a.codec4 else 12432
    mu = a.mu
    KD = capi.load_kernels()
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    torch.manual_seed(0)

    def blocks(rows, k, n_mats=1):
        """n_mats x E packed weight matrices [rows, k] (bandwidth does not depend on
        values; small normals).  --codec: encoded tiles (runtime/weight_codec.hpp)."""
        if not a.codec:
            w = (torch.randn(n_mats * E * rows * k, device="cuda") * 0.02).to(torch.bfloat16)
            per = rows * k * 2
            tab = [w.data_ptr() + (m * E + e) * per + rb * 128 * k * 2
                   for m in range(n_mats) for e in range(E) for rb in range(rows // 128)]
            return w, torch.tensor(tab, dtype=torch.int64, device="cuda")
        per = rows // 128 * (k // 64) * TB
        enc = np.zeros(n_mats * E * per, np.uint8)
        g = torch.Generator().manual_seed(rows + k)
        for i in range(n_mats * E):
            # the runtime's synthetic-weight distribution: uniform(-sqrt3 s, sqrt3 s), s = 1/sqrt(k)
            w = ((torch.rand(rows, k, generator=g) * 2 - 1) * (3.0 / k) ** 0.5).to(torch.bfloat16)
            src = w.view(torch.int16).numpy().view(np.uint16)
            packed = np.empty_like(src)
            KD.pack_weight(src.ctypes.data_as(C.c_void_p), rows, k, packed.ctypes.data_as(C.c_void_p))
            if a.codec4:
                assert KD.codec4_encode_rows(packed.ctypes.data_as(C.c_void_p), rows, k,
                                             enc[i * per:(i + 1) * per].ctypes.data_as(C.c_void_p), None) == 0
            elif a.codec3:
                assert KD.codec_encode_rows(packed.ctypes.data_as(C.c_void_p), rows, k,
                                            enc[i * per:(i + 1) * per].ctypes.data_as(C.c_void_p), None) == 0
            elif a.codec2:
                KD.codec_encode_frag(packed.ctypes.data_as(C.c_void_p), rows, k,
                                     enc[i * per:(i + 1) * per].ctypes.data_as(C.c_void_p), None)
            else:
                KD.codec_encode(packed.ctypes.data_as(C.c_void_p), rows, k,
                                enc[i * per:(i + 1) * per].ctypes.data_as(C.c_void_p))
        dev = torch.from_numpy(enc).cuda()
        tab = [dev.data_ptr() + i * per + rb * (k // 64) * TB
               for i in range(n_mats * E) for rb in range(rows // 128)]
        return dev, torch.tensor(tab, dtype=torch.int64, device="cuda")

    w13, t13 = blocks(F, H, 2)
    w2, t2 = blocks(H, F, 1)
    wqkv = (torch.randn(W * H, device="cuda") * 0.02).to(torch.bfloat16)
    tqkv = torch.tensor([wqkv.data_ptr() + rb * 128 * H * 2 for rb in range(W // 128)],
                        dtype=torch.int64, device="cuda")
    wo = (torch.randn(H * H, device="cuda") * 0.02).to(torch.bfloat16)
    to = torch.tensor([wo.data_ptr() + rb * 128 * H * 2 for rb in range(H // 128)],
                      dtype=torch.int64, device="cuda")
    wr = (torch.randn(E, H, device="cuda") * H ** -0.5).to(torch.bfloat16)
    x = torch.randn(mu, H, device="cuda")
    gamma = torch.ones(H, device="cuda").to(torch.bfloat16)
    hn = torch.zeros(mu, H, dtype=torch.bfloat16, device="cuda")
    idx = torch.zeros(mu, K, dtype=torch.int32, device="cuda")
    wts = torch.zeros(mu, K, device="cuda")
    R = (mu * K + 16 * E + 15) // 16 * 16
    cnt = torch.zeros(E, dtype=torch.int32, device="cuda")
    off = torch.zeros(E + 1, dtype=torch.int32, device="cuda")
    perm = torch.zeros(R, dtype=torch.int32, device="cuda")
    inv = torch.zeros(mu * K, dtype=torch.int32, device="cuda")
    xp = torch.zeros(R * H, dtype=torch.int16, device="cuda")
    inter = torch.zeros(R * F, dtype=torch.int16, device="cuda")
    # runtime.cpp expert_down_splits auto (8 x 32 tiles over 148 SMs; 2 CTAs per SM with codec 2)
    ds = a.down_splits or (8 if a.codec2 else 4 if a.codec else 1)
    cmode = 2 if a.codec2 else 3 if a.codec3 else 4 if a.codec4 else int(a.codec)
    y = torch.zeros(ds * R, H, device="cuda")
    xo = torch.zeros(mu, H, device="cuda")
    Rmu = (mu + 15) // 16 * 16
    xn = torch.zeros(Rmu * H, dtype=torch.int16, device="cuda")
    qkv = torch.zeros(Rmu, W, device="cuda")
    hbuf = torch.zeros(mu, H, device="cuda")
    ncap = a.ncap_e or min(128, Rmu)  # runtime.cpp ncap_e_
    ncap_gu, ncap_dn = (min(32, ncap), min(64, ncap)) if a.codec2 else (ncap, ncap)

    def router():
        KD.router_topk(ptr(x), ptr(gamma), 1e-5, None, ptr(wr), mu, H, E, K, ptr(hn), None,
                       ptr(idx), ptr(wts), s)
        KD.moe_permute(ptr(idx), ptr(hn), mu, H, E, K, ptr(cnt), ptr(off), ptr(perm), ptr(inv),
                       ptr(xp), R, s)

    # the runtime's stream-K tail for the last wave of gate/up tiles (runtime.cpp gu.sk_*)
    sk_scratch = torch.zeros(148 * 2 * Rmu * 128, device="cuda")
    sk_count = torch.zeros(148, dtype=torch.int64, device="cuda")
    gu_args = capi.GemmArgs(a_table=t13.data_ptr(), n_mats=2, G=E, RB=F // 128, K=H, b=xp.data_ptr(), R=R,
                            b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=ncap_gu, epi=1, alpha=1.0,
                            out_packed=inter.data_ptr(), out_R=R, codec=cmode,
                            sk_scratch=None if a.no_stream_k else sk_scratch.data_ptr(),
                            sk_count=sk_count.data_ptr(), sk_rows=Rmu, dec_groups=a.dec_groups)
    dn_args = capi.GemmArgs(a_table=t2.data_ptr(), n_mats=1, G=E, RB=H // 128, K=F, b=inter.data_ptr(), R=R,
                            b_off=off.data_ptr(), b_cnt=cnt.data_ptr(), n_cap=ncap_dn, epi=0, alpha=1.0,
                            out_f32=y.data_ptr(), ldo=H, codec=cmode, k_splits=ds, split_stride=R * H,
                            dec_groups=a.dec_groups)

    def expert():
        KD.gemm(C.byref(gu_args), s)
        KD.gemm(C.byref(dn_args), s)
        # (timing tool: the C ABI's combine sums split 0 only; the runtime's sums all ds parts)
        KD.moe_combine(ptr(hbuf), ptr(y), H, ptr(inv), ptr(wts), mu, H, K, ptr(xo), s)

    def tiling(rb):  # runtime.cpp dense_tiling
        cap = min(256, Rmu)
        ch = (mu + cap - 1) // cap
        return cap, ch, max(1, min(8, 148 // (rb * ch)))

    qkv_parts = torch.zeros(8 * Rmu * W, device="cuda")
    h_parts = torch.zeros(8 * mu * H, device="cuda")

    def dense_qkv():
        KD.rmsnorm_pack(ptr(x), ptr(gamma), mu, H, 1e-5, ptr(xn), Rmu, s)
        cap, ch, ks = tiling(W // 128)
        g = capi.GemmArgs(a_table=tqkv.data_ptr(), n_mats=1, G=1, RB=W // 128, K=H,
                          b=xn.data_ptr(), R=Rmu, rows_dense=mu, n_cap=cap, epi=0, alpha=1.0,
                          out_f32=qkv_parts.data_ptr(), ldo=W, n_chunks=ch, k_splits=ks,
                          split_stride=Rmu * W)
        KD.gemm(C.byref(g), s)

    def dense_o():
        cap, ch, ks = tiling(H // 128)
        g = capi.GemmArgs(a_table=to.data_ptr(), n_mats=1, G=1, RB=H // 128, K=H,
                          b=xn.data_ptr(), R=Rmu, rows_dense=mu, n_cap=cap, epi=0, alpha=1.0,
                          out_f32=h_parts.data_ptr(), ldo=H, residual=x.data_ptr(), ldr=H,
                          n_chunks=ch, k_splits=ks, split_stride=mu * H)
        KD.gemm(C.byref(g), s)

    # paged GQA attention at ctx 528 (identity block table, 16-token pages)
    CTX = 528
    pages_per = (CTX + 15) // 16
    kpool = (torch.randn(mu * pages_per * NKV * 16 * D, device="cuda")).to(torch.bfloat16)
    vpool = (torch.randn(mu * pages_per * NKV * 16 * D, device="cuda")).to(torch.bfloat16)
    bt = torch.arange(mu * pages_per, dtype=torch.int32, device="cuda")
    seq = torch.arange(mu, dtype=torch.int32, device="cuda")
    ctxs = torch.full((mu,), CTX, dtype=torch.int32, device="cuda")
    qrows = (torch.randn(mu, W, device="cuda")).to(torch.bfloat16)
    attn_out = torch.zeros(Rmu * H, dtype=torch.int16, device="cuda")

    def attention():
        KD.gqa_decode_paged(ptr(qrows), W, ptr(kpool), ptr(vpool), ptr(bt), pages_per, ptr(seq),
                            ptr(ctxs), mu, NQ, NKV, D, 16, ptr(attn_out), Rmu, None, s)

    att_scratch = torch.zeros(mu * NQ * 8 * 130, device="cuda")
    att_cnt = torch.zeros(mu * NKV, dtype=torch.int32, device="cuda")

    flat_scratch = torch.zeros(296 * 4 * 2 * (NQ // NKV) * 130, device="cuda")

    def attention_flat():  # stream-K over the flattened (token, head, page) space
        KD.gqa_decode_paged_flat(ptr(qrows), W, ptr(kpool), ptr(vpool), ptr(bt), pages_per, ptr(seq),
                                 ptr(ctxs), mu, NQ, NKV, D, 16, ptr(attn_out), Rmu, None, 0,
                                 ptr(flat_scratch), ptr(att_cnt), s)

    def attention_split():  # the runtime's call: split-KV, auto split count
        KD.gqa_decode_paged_split(ptr(qrows), W, ptr(kpool), ptr(vpool), ptr(bt), pages_per, ptr(seq),
                                  ptr(ctxs), mu, NQ, NKV, D, 16, ptr(attn_out), Rmu, None, 0, 8,
                                  ptr(att_scratch), ptr(att_cnt), s)

    router()
    torch.cuda.synchronize()
    touched = int((cnt > 0).sum().item())
    cases = [
        ("router+permute", router, mu * H * 4 + E * H * 2 + mu * K * 2 * H * 2),
        ("expert_ffn (gate/up+down+combine)", expert,
         touched * 3 * H * F * 2 + mu * K * 2 * H * 2 + mu * H * 2),
        ("expert gate/up gemm", lambda: KD.gemm(C.byref(gu_args), s), touched * 2 * H * F * 2 + mu * K * H * 2),
        ("expert down gemm", lambda: KD.gemm(C.byref(dn_args), s), touched * H * F * 2 + mu * K * F * 2),
        ("qkv (norm+gemm)", dense_qkv, W * H * 2 + mu * H * 4),
        ("o_proj (+residual)", dense_o, H * H * 2 + mu * H * 4 * 2),
        ("gqa_decode_paged (ctx 528)", attention, mu * 2 * CTX * NKV * D * 2),
        ("gqa_decode_paged split-KV (ctx 528)", attention_split, mu * 2 * CTX * NKV * D * 2),
        ("gqa_decode_paged stream-K (ctx 528)", attention_flat, mu * 2 * CTX * NKV * D * 2),
    ]
    reps = 2 if a.once else a.reps
    out = {}
    if a.with_h2d:  # concurrent page-stream DMA into HBM, as during a paged decode
        hsrc = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
        hdst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        cs = torch.cuda.Stream()
        with torch.cuda.stream(cs):
            for _ in range(12):
                hdst.copy_(hsrc, non_blocking=True)
    for name, fn, nbytes in cases:
        if a.only and not any(name.startswith(p) for p in a.only.split(",")):
            continue
        for _ in range(2 if not a.once else 0):
            fn()
        st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        st.record()
        for _ in range(reps):
            fn()
        en.record()
        torch.cuda.synchronize()
        ms = st.elapsed_time(en) / reps
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"ms": ms, "alg_bytes": nbytes, "GBps": gbs, "frac_hbm": gbs / peak}
        extra = ""
        if a.codec and name.startswith("expert"):  # bytes actually read: encoded weight tiles
            wb = touched * {"expert_ffn": 3, "expert gate/up gemm": 2, "expert down gemm": 1}[name.split(" (")[0]] * H * F * 2
            stored = nbytes - wb + wb * TB // 16384
            out[name].update(stored_bytes=stored, stored_GBps=stored / (ms * 1e-3) / 1e9,
                             stored_frac_hbm=stored / (ms * 1e-3) / 1e9 / peak)
            extra = f"  [encoded: {stored / 1e6:.1f} MB, {100 * out[name]['stored_frac_hbm']:.1f}% of HBM]"
        print(f"{name:36s} mu={mu:4d} {ms * 1e3:9.1f} us  {nbytes / 1e6:9.1f} MB  "
              f"{gbs:8.1f} GB/s  {100 * gbs / peak:5.1f}% of {peak} GB/s{extra}", flush=True)
    print(json.dumps({"mu": mu, "touched_experts": touched, "kernels": out}))


if __name__ == "__main__":
    main()
