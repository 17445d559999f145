"""Decode GEMMs at 129..512 tokens (B200): the swap-AB split-K kernel (the
engine's rule for T <= 128: ~288 CTAs, <= 8 splits) vs the token-major
kernel with 1..8 K splits, Llama-2-7B and Llama-2-70B shapes, weights from
HBM.  Fraction of min(HBM, TC x AI) roofline per point.

    python scripts/gemm_sweep_t128.py > gpurun_out/gemm_sweep_t128.jsonl
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import td_bench_gemm  # noqa: E402

P = json.load(open("MEASURED_PEAKS.json")) if os.path.exists("MEASURED_PEAKS.json") else {}
HBM, TC = P.get("hbm_gbs", 6551.7), P.get("bf16_tflops_sustained", 1412.2)
shapes = {"7b_qkv": (12288, 4096), "7b_o": (4096, 4096), "7b_gu": (22016, 4096), "7b_down": (4096, 11008),
          "70b_qkv": (10240, 8192), "70b_o": (8192, 8192), "70b_gu": (57344, 8192), "70b_down": (8192, 28672)}
for T in [160, 256, 384, 512]:
    for name, (N, K) in shapes.items():
        ideal = max((N * K * 2 + T * K * 2 + T * N * 4) / (HBM * 1e9), 2.0 * T * N * K / (TC * 1e12)) * 1e6
        copies = max(2, int(600e6 // (N * K * 2)) + 1)
        rows = []
        # swap-AB decode kernel, engine split rule
        ctas = ((N + 127) // 128) * ((T + 127) // 128)
        s = max(1, min(8, 288 // ctas))
        while s > 1 and (K // 64) // s < 4:
            s -= 1
        us = td_bench_gemm(T, N, K, s, 1, iters=20, copies=copies)
        rows.append(("swapab", s, us))
        for s in [1, 2, 3, 4, 6, 8]:
            if s > 1 and ((K // 64) // s < 8 or s * T * N * 4 > (16 << 20) * 4):
                continue
            us = td_bench_gemm(T, N, K, s, 2, iters=20, copies=copies)
            rows.append(("tokmajor", s, us))
        for kind, s, us in rows:
            print(json.dumps(dict(T=T, gemm=name, kind=kind, splits=s, us=round(us, 2), ideal_us=round(ideal, 2),
                                  frac=round(ideal / us, 3))), flush=True)
