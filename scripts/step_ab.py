"""Decode-step / prefill time of an n-layer Llama-2-7B-shaped stage (td_profile)
at a few batch sizes: quick A/B of engine knobs (run once per env setting).
Usage: TAG=x [ENV=...] python scripts/step_ab.py [--layers 8] [--ctx 600]"""
import argparse
import json
import os
import sys
import tempfile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import TDPipe  # noqa: E402
from workload import SHAPES, read_profile_csv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--ctx", type=int, default=600)
ap.add_argument("--bmax", type=int, default=256)
ap.add_argument("--chain", type=int, default=0)
ap.add_argument("--model", default="llama2_7b")
a = ap.parse_args()
shape = SHAPES[a.model].with_layers(a.layers)
t = TDPipe(shape, 1, kv_blocks=a.bmax * ((a.ctx + 31) // 16 + 2) + 64, decode_chain=a.chain)
csv = os.path.join(tempfile.gettempdir(), f"step_ab_{os.getpid()}.csv")
t.td_profile(csv, a.bmax, 2048, a.ctx)
tdec, tpre = read_profile_csv(csv)
row = {"tag": os.environ.get("TAG", ""), "model": a.model, "chain": a.chain, "layers": a.layers, "ctx": a.ctx}
for b in (1, 4, 8, 16, 32, 64, 128, 256, 384, 512):
    if b <= a.bmax:
        row[f"D{b}"] = round(int(tdec[b]) / 1e3, 1)
for k in (512, 2048):
    row[f"P{k}"] = round(int(tpre[k]) / 1e3, 1)
print(json.dumps(row), flush=True)
t.close()
