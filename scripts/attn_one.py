"""One decode-attention configuration (for ncu): n sequences of ctx tokens,
Llama-2-7B heads (or H HKV HD given).  python scripts/attn_one.py N CTX [ITERS [H HKV HD]]"""
import sys

import numpy as np

sys.path.insert(0, ".")
from paper_2506_10470_b200.tdpipe import td_bench_attn  # noqa: E402

n, ctx = int(sys.argv[1]), int(sys.argv[2])
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 2
H, HKV, HD = (int(a) for a in sys.argv[4:7]) if len(sys.argv) > 6 else (32, 32, 128)
us = td_bench_attn(np.full(n, ctx, np.int32), H, HKV, HD, iters=iters)
print(f"n={n} ctx={ctx}: {us:.2f} us, {n * ctx * HKV * HD * 4 / us / 1e3:.1f} GB/s")
