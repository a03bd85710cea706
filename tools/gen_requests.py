"""Seeded synthetic request file (`id,input_len` CSV, the reference's
load_requests format, cli.cpp:211-250) with a long-tailed prompt-length mix.

  python tools/gen_requests.py --n 512 --min 32 --max 1000 --seed 7 > requests.csv
"""
import argparse

import numpy as np

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=512)
ap.add_argument("--min", type=int, default=32)
ap.add_argument("--max", type=int, default=1000)
ap.add_argument("--seed", type=int, default=7)
a = ap.parse_args()
rng = np.random.default_rng(a.seed)
lens = np.clip(rng.lognormal(np.log(300), 0.7, a.n).astype(int), a.min, a.max)
for i, n in enumerate(lens):
    print(f"r{i:04d},{n}")
