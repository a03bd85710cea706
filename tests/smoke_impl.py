"""__graft_entry__.smoke(): one tiny decode step of the hot path on cuda:0,
checked against the CPU oracle.  Runs the full CGOPipe executor (weight
paging, host attention, router, tcgen05 expert FFN, lm_head, argmax) on the
Tiny config for 2 steps and compares the residual (<= 2e-2 relative to the
fp32 oracle) and the greedy ids at non-tie margins."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def run():
    from oracle import bind as orc
    from paper_2411_11217_b200 import capi
    from paper_2411_11217_b200.runtime import Runtime

    N, V = 8, 32000
    model = capi.ModelSpec(2, 1024, 3584, 8, 2, 8, 2, 2.0, 2.0)
    rt = Runtime(model, capi.Policy(N, 4, 0, 1, 0.0, 0.0), budget_bytes=2e9, max_ctx=32, vocab=V,
                 seed=1234, device=0)
    ref = orc.Model(2, 1024, 3584, 8, 2, 8, 2, V, N, 32, seed=1234)
    toks = np.random.default_rng(5678).integers(0, V, N, dtype=np.int32)
    for s in range(2):
        out = rt.decode(toks, 1)
        ids, margin, x_ref = ref.decode_step(toks, np.full(N, s, np.int32), orc.FP32, want_x=True)
        x = rt.residual()
        rel = float(np.linalg.norm(x - x_ref) / np.linalg.norm(x_ref))
        assert out.report.timeline_ok == 1, "measured timeline failed verify_timeline"
        assert out.report.gpu_launches > 0, "no kernels launched"
        assert rel <= 2e-2, f"residual rel error {rel}"
        sure = margin > 0.05
        assert (out.ids[0][sure] == ids[sure]).all(), (out.ids[0], ids, margin)
        print(f"[smoke] step {s}: rel(x)={rel:.2e}, ids {np.sum(out.ids[0] == ids)}/{N} equal, "
              f"{out.report.gpu_launches} launches, {out.report.tokens_per_second:.0f} tok/s")
        toks = out.ids[0]
    rt.close()


if __name__ == "__main__":
    run()
