"""Sweep split-K for the decode GEMM shapes of Llama-2-7B (weights from HBM)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_gemm  # noqa: E402

HBM = 6535.7
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008), "lm": (32000, 4096)}
res = []
for T in [1, 8, 32, 64, 128, 256]:
    for name, (N, K) in shapes.items():
        best = None
        for s in [1, 2, 3, 4, 6, 8, 12, 16]:
            if (K // 64) // s < 4:
                continue
            us = td_bench_gemm(T, N, K, s, True, iters=40, copies=max(2, int(600e6 // (N * K * 2)) + 1))
            gbs = (N * K * 2 + T * K * 2) / (us * 1e-6) / 1e9
            res.append(dict(T=T, gemm=name, splits=s, us=round(us, 2), GBs=round(gbs, 1), frac=round(gbs / HBM, 3)))
            print(json.dumps(res[-1]), flush=True)
json.dump(res, open("gpurun_out/gemm_sweep.json", "w"), indent=0)
