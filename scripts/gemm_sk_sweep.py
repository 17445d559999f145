"""Decode GEMMs of Llama-2-7B (weights streamed from HBM): stream-K kernel vs
the best split-K grid launch.  python scripts/gemm_sk_sweep.py > gpurun_out/gemm_sk_sweep.txt"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_gemm  # noqa: E402

HBM = 6535.7
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008), "lm": (32000, 4096)}
for T in [1, 8, 16, 32, 64, 96, 128]:
    for name, (N, K) in shapes.items():
        copies = max(2, int(600e6 // (N * K * 2)) + 1)
        byts = N * K * 2 + T * K * 2
        sk = td_bench_gemm(T, N, K, 1, 2, iters=40, copies=copies)
        best = min((td_bench_gemm(T, N, K, s, 1, iters=40, copies=copies), s) for s in (1, 2, 3, 4, 8)
                   if (K // 64) // s >= 4)
        print(json.dumps(dict(T=T, gemm=name, sk_us=round(sk, 2), sk_frac=round(byts / sk / 1e3 / HBM, 3),
                              splitk_us=round(best[0], 2), splitk_frac=round(byts / best[0] / 1e3 / HBM, 3),
                              splits=best[1])), flush=True)
