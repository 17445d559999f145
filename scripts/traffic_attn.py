"""Decode steps through the engine (Llama-2-7B shape, 32 layers) for an ncu
DRAM-traffic capture of the decode-attention launches (the bench's roofline
kernel).  A ShareGPT-like context mix of B sequences is prefilled, then STEPS
decode steps run; the algorithmic bytes of every decode_attn launch (K and V of
each context token + q + o, the engine's own accounting) are
printed for scripts/traffic_summary.py:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum -k regex:decode_attn \
        --clock-control none --csv --log-file gpurun_out/traffic_attn.csv \
        python scripts/traffic_attn.py [B] [STEPS] > gpurun_out/traffic_attn.json
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import TD_BATCH_DECODE, TD_BATCH_PREFILL, TDPipe  # noqa: E402
from workload import SHAPES  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
STEPS = int(sys.argv[2]) if len(sys.argv) > 2 else 2
shape = SHAPES["llama2_7b"]
rng = np.random.default_rng(0)
ctx = np.clip(rng.lognormal(6.3, 0.8, B), 32, 1900).astype(np.int64)
nb = (ctx + STEPS + 15) // 16 + 1
t = TDPipe(shape, 1, kv_blocks=int(nb.sum()) + 16)
# scattered pages: a random permutation of the pool
perm = rng.permutation(int(nb.sum())).astype(np.int32)
maxb = int(nb.max())
bt = np.zeros((B, maxb), np.int32)
o = 0
for i in range(B):
    bt[i, :nb[i]] = perm[o:o + nb[i]]
    o += nb[i]
i = 0
while i < B:   # prefill in chunks of <= 2048 tokens
    j = i
    tot = 0
    while j < B and tot + ctx[j] <= 2048:
        tot += ctx[j]
        j += 1
    j = max(j, i + 1)
    toks = rng.integers(0, shape.vocab, size=int(ctx[i:j].sum())).astype(np.int32)
    t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * (j - i), ctx[i:j].tolist(), bt[i:j], toks)
    i = j
algo = 0.0
launches = 0
for s in range(STEPS):
    toks = rng.integers(0, shape.vocab, size=B).astype(np.int32)
    t.td_stage_forward(0, TD_BATCH_DECODE, (ctx + s).tolist(), [1] * B, bt, toks)
    per = float((ctx + s + 1).sum()) * 2 * shape.n_kv_heads * shape.head_dim * 2 + 4.0 * B * shape.n_heads * shape.head_dim
    algo += per * shape.n_layers
    launches += shape.n_layers
t.close()
print(json.dumps({"launches": launches, "algorithmic_bytes": algo, "B": B, "steps": STEPS,
                  "mean_ctx": float(ctx.mean())}))
