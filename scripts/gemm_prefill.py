"""Prefill GEMM throughput (T = 2048) for the Llama-2-7B shapes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_gemm  # noqa: E402

shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008)}
for T in [int(x) for x in os.environ.get("TS", "2048,1738,1024").split(",")]:
    for name, (N, K) in shapes.items():
        us = td_bench_gemm(T, N, K, 1, False, iters=20, copies=2)
        tf = 2.0 * T * N * K / (us * 1e-6) / 1e12
        print(json.dumps(dict(T=T, gemm=name, us=round(us, 1), TFLOPs=round(tf, 1),
                              frac_sustained=round(tf / 1412.2, 3), tag=os.environ.get("TAG", ""))), flush=True)
