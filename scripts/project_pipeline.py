"""Project multi-GPU TD-Pipe vs the naive PP+SB pipeline from MEASURED per-stage
B200 times.

For each (model, S) the per-stage profile table is measured on one B200 with
td_profile on a model of n_layers / S layers (embedding + LM head included, i.e.
the slowest stage); then td_simulate replays the exact TD-Pipe / PP+SB schedules
(the same controller as td_run) on an S-stage FIFO pipeline with those times.
The KV capacity per stage is what one B200 holds next to its stage's weights
(or a cap that reproduces the paper's KV-constrained regime).
Output: one JSON line per (config, policy) -> gpurun_out/projection.jsonl
"""
import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import (TD_EXEC_NULL, TD_POLICY_PPSB_ALT, TD_POLICY_PPHB, TD_POLICY_PPSB_PRIO,  # noqa: E402
                                   TD_POLICY_TDPIPE, TDPipe)
from workload import SHAPES, config_workload  # noqa: E402

HBM = 183_359 * 2 ** 20          # bytes (nvidia-smi total)
RESERVE = 0.06 * HBM + 3e9       # reserve + work buffers


def stage_kv_blocks(shape, S):
    lps = shape.n_layers // S
    hd = shape.head_dim
    w_stage = 2 * (lps * (shape.d_model * (shape.n_heads + 2 * shape.n_kv_heads) * hd + shape.d_model * shape.n_heads * hd
                          + 3 * shape.d_model * shape.d_ffn) + 2 * shape.vocab * shape.d_model)
    per_block = 2 * shape.n_kv_heads * 16 * hd * 2 * lps
    return int((HBM - RESERVE - w_stage) // per_block)


def run(cfg_name, model, S, kv_cap=None, out=None):
    shape = SHAPES[model]
    wl = config_workload(cfg_name)
    n = len(wl.requests)
    L = np.array([len(r.prompt) for r in wl.requests])
    P = np.array([r.predicted_len for r in wl.requests])
    ctx_rep = int(L.sum() // n + (P.sum() // n) // 2)
    prof = f"/tmp/prof_{model}_{S}.csv"
    if not os.path.exists(prof):
        stage = dataclasses.replace(shape.with_layers(shape.n_layers // S), max_seq_len=4096)
        nb = (ctx_rep + 16) // 16 + 1
        lps = shape.n_layers // S
        per_block = 2 * shape.n_kv_heads * 16 * shape.head_dim * 2 * lps
        w_stage = HBM - RESERVE - stage_kv_blocks(shape, S) * per_block
        b_max = int(min(1024, (HBM - RESERVE - w_stage - 8e9) // (nb * per_block)))
        t = TDPipe(stage, 1, kv_blocks=b_max * nb + 64)
        t.td_profile(prof, b_max, 2048, ctx_rep)
        t.close()
    C = kv_cap or stage_kv_blocks(shape, S)
    big = dataclasses.replace(shape, max_seq_len=8192)
    for name, pol, sigma in [("tdpipe", TD_POLICY_TDPIPE, 1), ("tdpipe_sigma", TD_POLICY_TDPIPE, max(1, S - 1)),
                             ("ppsb_alt", TD_POLICY_PPSB_ALT, 1), ("ppsb_prio", TD_POLICY_PPSB_PRIO, 1),
                             ("pphb", TD_POLICY_PPHB, 1)]:
        if name == "tdpipe_sigma" and S <= 2:
            continue
        t = TDPipe(big, S, executor=TD_EXEC_NULL, kv_blocks=C, profile_csv=prof, policy=pol, eq2_bubble_scale=sigma,
                   log_decisions=0)
        t.submit_workload(wl)
        st = t.td_simulate(30_000)
        rec = dict(config=cfg_name, model=model, stages=S, kv_blocks=C, policy=name, gen_tok_s=round(st["gen_tokens_per_s"]),
                   total_tok_s=round(st["total_tokens_per_s"]), bubble=round(st["bubble_frac"], 4),
                   makespan_s=round(st["makespan_ns"] / 1e9, 2), p2d=st["n_p2d"], d2p=st["n_d2p"],
                   stolen=st["n_stolen"], evicted=st["n_evicted"])
        print(json.dumps(rec), flush=True)
        if out:
            out.write(json.dumps(rec) + "\n")
        t.close()


if __name__ == "__main__":
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/projection.jsonl", "w") as out:
        run("C3", "llama2_13b", 2, out=out)
        run("C3", "llama2_13b", 4, out=out)
        run("C4", "opt30b_shaped", 4, out=out)
        run("C4", "opt30b_shaped", 8, out=out)
        run("C5", "llama2_70b", 8, out=out)
        run("C5", "llama2_70b", 8, kv_cap=24000, out=out)
