"""Decode-attention sweep (B200): GB/s of K/V streamed per launch vs batch size
and context length, Llama-2-7B heads, the engine's launch plan.  Extra env
knobs (TDPIPE_ATTN_V2=1) select variants for A/B runs.

    python scripts/attn_sweep.py [tag] > gpurun_out/attn_sweep.txt
"""
import json
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2506_10470_b200.tdpipe import td_bench_attn  # noqa: E402

PEAK = 6535.7
tag = sys.argv[1] if len(sys.argv) > 1 else "v1"
# Llama-2-7B heads (MHA) by default; "gqa8" = Llama-2-70B heads (H 64 / Hkv 8)
H, HKV, HD = (64, 8, 128) if "gqa8" in tag else (32, 32, 128)
rng = np.random.default_rng(0)
for n in (1, 2, 4, 8, 16, 32, 64, 128, 256, 512):
    for dist in ("256", "1024", "3072", "mix"):
        if dist == "mix":
            ctx = np.clip(rng.lognormal(6.3, 0.8, n), 32, 4000).astype(np.int32)
        else:
            ctx = np.full(n, int(dist), np.int32)
        kv_bytes = float(ctx.sum()) * HKV * HD * 2 * 2
        us = td_bench_attn(ctx, H, HKV, HD, iters=30)
        print(json.dumps({"tag": tag, "n": n, "ctx": dist, "sum_ctx": int(ctx.sum()), "us": round(us, 2),
                          "GBs": round(kv_bytes / us / 1e3, 1), "frac": round(kv_bytes / us / 1e3 / PEAK, 3)}),
              flush=True)
