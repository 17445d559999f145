"""Decode GEMMs at 65..128 tokens: swap-AB (mode 1, engine split rule) vs the
token-major kernel (mode 2, no split).  HBM fraction of weight bytes."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_gemm  # noqa: E402

HBM = 6551.7
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008),
          "70b_gu": (57344, 8192), "70b_qkv": (10240, 8192)}
for T in (72, 96, 128):
    for name, (N, K) in shapes.items():
        ctas = ((N + 127) // 128) * 1
        sp = max(1, min(8, 288 // ctas))
        while sp > 1 and (K // 64) // sp < 4:
            sp -= 1
        r = {"T": T, "gemm": name}
        for mode, s in ((1, sp), (2, 1)):
            us = td_bench_gemm(T, N, K, s, mode, iters=20, copies=2)
            r[f"m{mode}"] = {"us": round(us, 2), "splits": s, "frac": round(N * K * 2 / (us * 1e-6) / 1e9 / HBM, 3)}
        print(json.dumps(r), flush=True)
