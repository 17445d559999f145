"""MHA decode attention (Llama-2-7B heads): SIMT (impl 1) vs tensor-core kernel
(impl 2) around the dispatch threshold, C2-like contexts (lognormal, mean ~250)
and ShareGPT-mix contexts (mean ~750); engine launch plans, random operands.
JSON lines: n, dist, us per kernel, SIMT/TC time ratio."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_attn  # noqa: E402

for dist, (mu, lo, hi) in (("mix250", (5.2, 16, 2000)), ("mix", (6.3, 32, 4000))):
    for n in (16, 24, 32, 40, 48, 56, 64, 96):
        us = {}
        for seed in range(3):   # three context draws per point
            rng = np.random.default_rng(100 + seed)
            ctx = np.clip(rng.lognormal(mu, 0.8, n), lo, hi).astype(np.int32)
            for impl in (1, 2):
                us.setdefault(impl, []).append(td_bench_attn(ctx, 32, 32, 128, iters=30, impl=impl))
        a, b = float(np.sum(us[1])), float(np.sum(us[2]))
        print(json.dumps({"n": n, "dist": dist, "simt_us": round(a / 3, 2), "tc_us": round(b / 3, 2),
                          "simt_over_tc": round(a / b, 3)}), flush=True)
