"""Reproduce a codec-3 decode at the 8x7B-width 2-layer test shape (tests/test_decode_gpu.py)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2411_11217_b200 import capi  # noqa: E402
from paper_2411_11217_b200.runtime import Runtime  # noqa: E402

N, MU, PROMPT, VOCAB = 8, 4, 16, 32000
force_raw = sys.argv[1] if len(sys.argv) > 1 else "0"
r_w = float(sys.argv[2]) if len(sys.argv) > 2 else 0.10
layers = int(sys.argv[3]) if len(sys.argv) > 3 else 2
h1, h2 = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (4096, 14336)
os.environ["MLT_CODEC_FORCE_RAW"] = force_raw
os.environ["MLT_CODEC_MODE"] = "3"
prompt = np.random.default_rng(5678).integers(0, VOCAB, size=(PROMPT, N), dtype=np.int32)
rt = Runtime(capi.ModelSpec(layers, h1, h2, 32, 8, 8, 2, 2.0, 2.0), capi.Policy(N, MU, 0, 1, r_w, 0.0),
             budget_bytes=7e9, max_ctx=64, vocab=VOCAB, seed=1234, weight_codec=True)
first = rt.decode(prompt[0], PROMPT, forced=prompt)
print("ok", first.ids[-1])
