"""MHA decode attention (Llama-2-7B heads) at small batches: the SIMT kernel
(impl 1, U = 4 tokens in flight per thread group, 5 CTAs/SM) vs its deep
variant (impl 3, U = 8, 2 CTAs/SM), engine launch plan.  JSON lines."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_attn  # noqa: E402

HBM = 6551.7
rng = np.random.default_rng(0)
for n in (1, 2, 4, 8, 16, 32, 64):
    for ctx in (256, 600, 1200, 2000, "mix"):
        c = rng.integers(100, 2048, size=n).astype(np.int32) if ctx == "mix" else np.full(n, ctx, np.int32)
        row = {"n": n, "ctx": ctx}
        for impl in (1, 3):
            us = td_bench_attn(c, 32, 32, 128, iters=20, impl=impl)
            row[f"us{impl}"] = round(us, 2)
            row[f"frac{impl}"] = round(float(c.sum()) * 32 * 128 * 4 / (us * 1e-6) / 1e9 / HBM, 3)
        print(json.dumps(row), flush=True)
