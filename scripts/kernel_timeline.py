"""In-context kernel timeline of decode steps (CUPTI activity tracing through
torch.profiler: GPU start / end of every kernel of the process, PDL overlap
intact and no per-kernel CUDA events -- unlike the bench's roofline pass).
An n-layer Llama-2-7B-shaped stage: b sequences are prefilled to `ctx` tokens
with td_stage_forward, then decode steps run under the profiler.  For each
kernel class: launches per step, mean kernel duration, and its MARGINAL time
(how far its end moves the timeline past its predecessor's end; these sum to
the step).  JSON lines.

    python scripts/kernel_timeline.py [--b 1 8 32] [--layers 8] [--ctx 600]
"""
import argparse
import collections
import json
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import TD_BATCH_DECODE, TD_BATCH_PREFILL, TDPipe  # noqa: E402
from workload import SHAPES  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--b", type=int, nargs="+", default=[1, 8, 32])
ap.add_argument("--layers", type=int, default=8)
ap.add_argument("--ctx", type=int, default=600)
ap.add_argument("--model", default="llama2_7b")
ap.add_argument("--chain", type=int, default=0)
ap.add_argument("--steps", type=int, default=3)
ap.add_argument("--trace", default="")
ap.add_argument("--roles", type=int, default=1, help="label the GEMMs QKV / O / gate-up / down / LM head")
a = ap.parse_args()
torch.cuda.init()
shape = SHAPES[a.model].with_layers(a.layers)
nb = (a.ctx + a.steps + 16) // 16 + 1
t = TDPipe(shape, 1, kv_blocks=max(a.b) * nb + 64, decode_chain=a.chain)
ROLES = {}


def short(name):
    for k in ("gemm_tc_kernel", "gemm_tnp_kernel", "decode_attn_tc_kernel", "decode_attn_kernel", "resid_norm_cluster",
              "resid_norm_kernel", "splitk_reduce", "rmsnorm_kernel", "argmax", "embed", "decode_chain", "flash_prefill"):
        if k in name:
            return k
    return name[:40]


for b in a.b:
    bt = (np.arange(b * nb, dtype=np.int32).reshape(nb, b).T).copy()   # interleaved pages
    per = max(1, 2048 // a.ctx)
    rng = np.random.default_rng(b)
    for i in range(0, b, per):
        j = min(b, i + per)
        toks = rng.integers(0, shape.vocab, size=(j - i) * a.ctx).astype(np.int32)
        t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * (j - i), [a.ctx] * (j - i), bt[i:j], toks)
    nxt = np.zeros(b, np.int32)
    t.td_stage_forward(0, TD_BATCH_DECODE, [a.ctx] * b, [1] * b, bt, nxt)   # warm
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for s in range(a.steps):
            t.td_stage_forward(0, TD_BATCH_DECODE, [a.ctx + 1 + s] * b, [1] * b, bt, nxt)
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.name and
          "memcpy" not in e.name.lower() and "memset" not in e.name.lower()]
    ev.sort(key=lambda e: e.time_range.start)
    if a.trace:
        prof.export_chrome_trace(f"{a.trace}_b{b}.json")
    starts = [i for i, e in enumerate(ev) if "embed" in e.name]
    steps = [ev[starts[k]:(starts[k + 1] if k + 1 < len(starts) else len(ev))] for k in range(len(starts))]
    marg, dur, cnt = collections.defaultdict(float), collections.defaultdict(float), collections.Counter()
    spans = []
    roles = ["gemm_qkv", "gemm_o", "gemm_gu", "gemm_down"]
    for st in steps:
        prev = st[0].time_range.start
        ng = sum(1 for e in st if short(e.name).startswith("gemm"))
        gi = 0
        for e in st:
            k = short(e.name)
            if k.startswith("gemm") and a.roles:   # label: 4 per layer, the last one is the LM head
                k = "gemm_lm_head" if gi == ng - 1 else roles[gi % 4]
                gi += 1
            marg[k] += max(0, e.time_range.end - prev)
            dur[k] += e.time_range.end - e.time_range.start
            cnt[k] += 1
            prev = max(prev, e.time_range.end)
        spans.append(prev - st[0].time_range.start)
    ns = len(steps)
    row = {"b": b, "layers": a.layers, "ctx": a.ctx, "step_us": round(float(np.mean(spans)), 1),
           "classes": {k: {"per_step": cnt[k] / ns, "dur_us": round(dur[k] / cnt[k], 2),
                           "marginal_us_per_step": round(marg[k] / ns, 1)} for k in cnt}}
    print(json.dumps(row), flush=True)
t.close()
