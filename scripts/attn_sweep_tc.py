"""Decode-attention sweep (B200): achieved GB/s of K/V per launch vs batch size,
context length, split size (0 = the engine's launch plan) and kernel (impl 1 =
SIMT, 2 = tensor cores).  One JSON line per point.

    python scripts/attn_sweep_tc.py H HKV HD [impl ...] > gpurun_out/attn_sweep.jsonl
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2506_10470_b200.tdpipe import td_bench_attn  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6551.7
H, HKV, HD = (int(a) for a in sys.argv[1:4]) if len(sys.argv) > 3 else (64, 8, 128)
impls = [int(a) for a in sys.argv[4:]] or [0]
splits = [int(s) for s in os.environ.get("SPLITS", "0,64,128,256,512,1024").split(",")]
rng = np.random.default_rng(0)
for n in (1, 4, 16, 64, 128, 256, 512):
    for dist in ("256", "1024", "3072", "mix", "mix250"):
        if dist == "mix":
            ctx = np.clip(rng.lognormal(6.3, 0.8, n), 32, 4000).astype(np.int32)
        elif dist == "mix250":   # C2-like decode contexts (mean ~250 tokens)
            ctx = np.clip(rng.lognormal(5.2, 0.8, n), 16, 2000).astype(np.int32)
        else:
            ctx = np.full(n, int(dist), np.int32)
        kv_bytes = float(ctx.sum()) * HKV * HD * 2 * 2 + 4.0 * n * H * HD
        for impl in impls:
            for sp in splits:
                if sp and sp > 2 * int(ctx.max()):
                    continue
                us = td_bench_attn(ctx, H, HKV, HD, iters=20, split=sp, impl=impl)
                print(json.dumps({"H": H, "Hkv": HKV, "hd": HD, "impl": impl, "n": n, "ctx": dist,
                                  "sum_ctx": int(ctx.sum()), "split": sp, "us": round(us, 2),
                                  "GBs": round(kv_bytes / us / 1e3, 1),
                                  "frac": round(kv_bytes / us / 1e3 / PEAK, 3)}), flush=True)
