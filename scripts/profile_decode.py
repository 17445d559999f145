"""Decode-phase micro-benchmark for ncu: Llama-2-7B-shaped layers, a batch of
sequences prefilled to ~ctx tokens, then decode steps at batch b.
Usage: python scripts/profile_decode.py [--layers 2] [--b 256] [--ctx 300] [--steps 3]"""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import TD_BATCH_DECODE, TD_BATCH_PREFILL, TDPipe  # noqa: E402
from workload import SHAPES  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=2)
ap.add_argument("--b", type=int, default=256)
ap.add_argument("--ctx", type=int, default=300)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--model", default="llama2_7b")
ap.add_argument("--no-prefill", action="store_true")
ap.add_argument("--prefill-only", action="store_true")
a = ap.parse_args()
shape = SHAPES[a.model].with_layers(a.layers)
t = TDPipe(shape, 1, kv_blocks=a.b * ((a.ctx + a.steps + 15) // 16 + 1) + 16)
nb = (a.ctx + a.steps + 15) // 16 + 1
bt = np.arange(a.b * nb, dtype=np.int32).reshape(a.b, nb)
rng = np.random.default_rng(0)
per = max(1, 2048 // a.ctx)
for s in (range(0, a.b, per) if not a.no_prefill else []):
    idx = list(range(s, min(a.b, s + per)))
    toks = rng.integers(0, shape.vocab, size=a.ctx * len(idx)).astype(np.int32)
    t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * len(idx), [a.ctx] * len(idx), bt[idx], toks)
for step in (range(a.steps) if not a.prefill_only else []):
    toks = rng.integers(0, shape.vocab, size=a.b).astype(np.int32)
    t.td_stage_forward(0, TD_BATCH_DECODE, [a.ctx + step] * a.b, [1] * a.b, bt, toks)
print("done")
