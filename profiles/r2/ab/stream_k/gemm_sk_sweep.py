"""Token-major GEMM: data-parallel (mode 2) vs stream-K tail (mode 5), isolated,
TFLOP/s fraction of sustained peak.  JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_gemm  # noqa: E402

TC = 1412.2
cases = [("7b_o", 1738, 4096, 4096), ("7b_down", 1738, 4096, 11008), ("7b_qkv", 1738, 12288, 4096),
         ("7b_gu", 1738, 22016, 4096), ("7b_o", 2048, 4096, 4096), ("7b_gu", 256, 22016, 4096),
         ("7b_qkv", 256, 12288, 4096), ("7b_qkv", 512, 12288, 4096), ("70b_qkv", 512, 10240, 8192),
         ("70b_qkv", 256, 10240, 8192), ("70b_gu", 512, 57344, 8192), ("7b_gu", 160, 22016, 4096)]
for name, T, N, K in cases:
    row = {"gemm": name, "T": T}
    for mode in (2, 5):
        us = td_bench_gemm(T, N, K, 1, mode, iters=10, copies=2)
        row[f"m{mode}"] = {"us": round(us, 2), "frac": round(2.0 * T * N * K / (us * 1e-6) / 1e12 / TC, 3)}
    print(json.dumps(row), flush=True)
