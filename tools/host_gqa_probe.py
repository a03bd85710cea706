"""Host GQA decode attention (the CpuAttn kernel, mlt_host_gqa_decode) on
this machine's cores: GB/s of KV read per thread count at the 8x7B shape
(nq 32, nkv 8, d 128), ctx ~ prompt 512 + decode steps.

  python tools/host_gqa_probe.py [--T 256] [--ctx 520] [--threads 1,2,4,8,14,16]
"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_11217_b200 import capi  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, default=256)
    ap.add_argument("--ctx", type=int, default=520)
    ap.add_argument("--threads", default="1,2,4,8,14,16")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--h2d", action="store_true",
                    help="keep a host->device copy stream running (the weight pages of a paging policy)")
    a = ap.parse_args()
    stop = None
    if a.h2d:
        import threading

        import torch
        src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
        dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        stop = threading.Event()

        def pump():
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                while not stop.is_set():
                    dst.copy_(src, non_blocking=True)
                    s.synchronize()
        pump_thread = threading.Thread(target=pump, daemon=True)
        pump_thread.start()
        time.sleep(1.0)
    k = capi.load_kernels()
    T, nq, nkv, d, L = a.T, 32, 8, 128, a.ctx
    rng = np.random.default_rng(0)

    def bf16(shape):
        x = rng.standard_normal(shape, dtype=np.float32)
        return (x.view(np.uint32) >> 16).astype(np.uint16)
    q = bf16((T, nq, d))
    kc, vc = bf16((T, nkv, L, d)), bf16((T, nkv, L, d))
    ctx = np.full(T, L, np.int32)
    out = np.zeros((T, nq, d), np.uint16)
    p = lambda x: x.ctypes.data_as(C.c_void_p)  # noqa: E731
    kv_bytes = 2 * T * nkv * L * d * 2
    res = {}
    for th in [int(x) for x in a.threads.split(",")]:
        best = 1e9
        for _ in range(a.reps):
            t = time.perf_counter()
            k.host_gqa_decode(p(q), p(kc), p(vc), p(ctx), T, nq, nkv, d, L, p(out), th)
            best = min(best, time.perf_counter() - t)
        res[th] = best
        print(f"threads {th:3d}: {best * 1e3:8.2f} ms  {kv_bytes / best / 1e9:7.1f} GB/s  "
              f"{kv_bytes / best / 1e9 / th:6.2f} GB/s/thread", flush=True)
    if stop is not None:
        stop.set()
        pump_thread.join()
    return res


if __name__ == "__main__":
    main()
