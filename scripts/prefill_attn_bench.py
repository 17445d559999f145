"""Prefill attention in context: td_bench_step (prefill micro-batch of n equal
prompts of `len` tokens) on a 2-layer Llama-2-7B-shaped stage; per-launch time
and causal TFLOP/s of the prefill-attention class.  JSON lines."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import TDPipe  # noqa: E402
from workload import SHAPES  # noqa: E402

t = TDPipe(SHAPES["llama2_7b"].with_layers(2), 1, kv_blocks=4096)
for n, L in ((16, 128), (8, 256), (4, 512), (2, 1024), (1, 2048)):
    t.td_set_timing(True)
    us, _ = t.td_bench_step(0, n, L, 10)
    k = t.td_get_timing("prefill_attn")
    t.td_set_timing(False)
    per = k["ms"] * 1e3 / max(k["launches"], 1)
    print(json.dumps({"tag": os.environ.get("TAG", ""), "n": n, "len": L, "attn_us": round(per, 2),
                      "TFLOPs": round(k["flops"] / (k["ms"] * 1e-3) / 1e12, 1), "step_us": round(us, 1)}), flush=True)
t.close()
