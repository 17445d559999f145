"""Decode GEMMs at 33..128 tokens: swap-AB with the engine's token tile (BN 64 /
128) vs 64- and 32-token tiles (more weight stages in flight per SM; the token
tiles share each weight tile through L2), engine split rule.  HBM fraction of
the weight bytes.  JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_gemm  # noqa: E402

HBM = 6551.7
shapes = {"qkv": (12288, 4096), "o": (4096, 4096), "gu": (22016, 4096), "down": (4096, 11008)}


def splits_for(N, K, T, bn):
    ctas = ((N + 127) // 128) * ((T + bn - 1) // bn)
    s = max(1, min(8, 288 // ctas))
    while s > 1 and (K // 64) // s < 4:
        s -= 1
    return s


for T in (40, 64, 96, 128):
    for name, (N, K) in shapes.items():
        row = {"T": T, "gemm": name}
        auto_bn = 32 if T <= 32 else 64 if T <= 64 else 128
        for mode, bn in ((1, auto_bn), (3, 64), (4, 32)):
            if mode != 1 and bn >= auto_bn:
                continue
            sp = splits_for(N, K, T, bn)
            us = td_bench_gemm(T, N, K, sp, mode, iters=20, copies=4)
            row[f"bn{bn}"] = {"us": round(us, 2), "splits": sp, "frac": round(N * K * 2 / (us * 1e-6) / 1e9 / HBM, 3)}
        print(json.dumps(row), flush=True)
