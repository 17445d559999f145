"""§4.4 ablations of the paper on B200, and the KV-usage
timeline / Chrome trace of a measured run (PAPER.md:580-585 fig:memory_usage).

A. MEASURED, one B200, one stage (W = 1): the C2 request set (Llama-2-7B-shaped,
   256 ShareGPT-length requests) with the KV pool capped so that demand /
   capacity ~ 4 (the paper's memory-constrained regime):
   TD-Pipe vs its ablations -- the P->D switch replaced by a KV-occupancy ratio
   30/50/70 % ("Approach-1") and the D->P switch replaced by a
   request-finish ratio 25/50/90 % ("Approach-3") -- and the
   PP+SB baselines.  Work stealing (Approach-2) needs W > 1 decode batches: it
   is a no-op on one stage and is measured in B only.  Each run's device time
   comes from td_run (CUDA events); one TD-Pipe run is repeated with timing on
   and written as a Chrome trace with the kv_used_blocks timeline.
B. PROJECTION (labelled so): per-stage tables measured on this B200 with
   td_profile on a model of n_layers / S layers, then td_simulate replays every
   policy on an S-stage FIFO pipeline -- stealing on / off,
   KV-ratio and finish-ratio switches, PP+SB -- for the KV-constrained C5-cap
   (Llama-2-70B, S = 8, 24,000 blocks) and C4 (S = 4) configs.

    python scripts/ablations.py [A|B|AB] -> gpurun_out/ablations.jsonl, gpurun_out/trace_c2cap.json
"""
import dataclasses
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2506_10470_b200 as tp  # noqa: E402
from paper_2506_10470_b200 import TDPipe  # noqa: E402
from workload import SHAPES, config_workload  # noqa: E402

OUT = os.path.join(ROOT, "gpurun_out")
POL = {"tdpipe": tp.TD_POLICY_TDPIPE, "ppsb_alt": tp.TD_POLICY_PPSB_ALT, "ppsb_prio": tp.TD_POLICY_PPSB_PRIO,
       "pphb": tp.TD_POLICY_PPHB}
VARIANTS = [("tdpipe", "tdpipe", {}),
            ("kv_ratio_30", "tdpipe", dict(p2d_kv_permille=300)),
            ("kv_ratio_50", "tdpipe", dict(p2d_kv_permille=500)),
            ("kv_ratio_70", "tdpipe", dict(p2d_kv_permille=700)),
            ("finish_25", "tdpipe", dict(d2p_finish_permille=250)),
            ("finish_50", "tdpipe", dict(d2p_finish_permille=500)),
            ("finish_90", "tdpipe", dict(d2p_finish_permille=900)),
            ("ppsb_alt", "ppsb_alt", {}), ("ppsb_prio", "ppsb_prio", {})]


def ctx_rep(wl):
    n = len(wl.requests)
    L = np.array([len(r.prompt) for r in wl.requests])
    P = np.array([r.predicted_len for r in wl.requests])
    return int(L.sum() // n + (P.sum() // n) // 2)


def emit(rec, out):
    print(json.dumps(rec), flush=True)
    out.write(json.dumps(rec) + "\n")
    out.flush()


def measured(out, kv_blocks=1500, steps=2):
    shape = SHAPES["llama2_7b"]
    wl = config_workload("C2")
    demand = sum(-(-(len(r.prompt) + r.max_new_tokens) // 16) for r in wl.requests)
    prof = os.path.join(OUT, "prof_c2.csv")
    t0 = TDPipe(shape, 1, device=0, kv_blocks=kv_blocks)
    t0.td_profile(prof, 512, 2048, ctx_rep(wl))
    t0.close()
    for name, pol, extra in VARIANTS:
        t = TDPipe(shape, 1, device=0, kv_blocks=kv_blocks, profile_csv=prof, policy=POL[pol], **extra)
        t.submit_workload(wl)
        t.td_upload()
        t.td_run()   # warm-up
        sts = []
        for _ in range(steps):
            t.td_reset()
            t.submit_workload(wl)
            t.td_upload()
            sts.append(t.td_run())
        st = sts[-1]
        gen = sum(s["generated_tokens"] for s in sts)
        span = sum(s["makespan_ns"] for s in sts) / 1e9
        rec = dict(kind="measured", config="C2-cap", model="llama2_7b", stages=1, kv_blocks=kv_blocks,
                   demand_over_capacity=round(demand / kv_blocks, 2), variant=name, gen_tok_s=round(gen / span, 1),
                   total_tok_s=round(sum(s["generated_tokens"] + s["prompt_tokens"] for s in sts) / span, 1),
                   makespan_s=round(span / steps, 3), p2d=st["n_p2d"], d2p=st["n_d2p"], evicted=st["n_evicted"],
                   prompt_tokens=st["prompt_tokens"], microbatches=st["n_microbatches"])
        emit(rec, out)
        if name == "tdpipe":   # the measured KV-usage timeline + Chrome trace (timing on)
            t.td_reset()
            t.submit_workload(wl)
            t.td_upload()
            t.td_set_timing(True)
            t.td_run()
            t.td_set_timing(False)
            t.td_write_trace(os.path.join(OUT, "trace_c2cap.json"))
        t.close()


HBM = 183_359 * 2 ** 20
RESERVE = 0.06 * HBM + 3e9


def stage_kv_blocks(shape, S):
    lps = shape.n_layers // S
    hd = shape.head_dim
    w_stage = 2 * (lps * (shape.d_model * (shape.n_heads + 2 * shape.n_kv_heads) * hd + shape.d_model * shape.n_heads * hd
                          + 3 * shape.d_model * shape.d_ffn) + 2 * shape.vocab * shape.d_model)
    per_block = 2 * shape.n_kv_heads * 16 * hd * 2 * lps
    return int((HBM - RESERVE - w_stage) // per_block)


def projection(out, cfg, model, S, kv_cap=None):
    shape = SHAPES[model]
    wl = config_workload(cfg)
    prof = os.path.join(OUT, f"prof_{model}_S{S}.csv")
    if not os.path.exists(prof):
        stage = dataclasses.replace(shape.with_layers(shape.n_layers // S), max_seq_len=4096)
        nb = (ctx_rep(wl) + 16) // 16 + 1
        lps = shape.n_layers // S
        per_block = 2 * shape.n_kv_heads * 16 * shape.head_dim * 2 * lps
        w_stage = HBM - RESERVE - stage_kv_blocks(shape, S) * per_block
        b_max = int(min(1024, (HBM - RESERVE - w_stage - 8e9) // (nb * per_block)))
        t = TDPipe(stage, 1, device=0, kv_blocks=b_max * nb + 64)
        t.td_profile(prof, b_max, 2048, ctx_rep(wl))
        t.close()
    C = kv_cap or stage_kv_blocks(shape, S)
    big = dataclasses.replace(shape, max_seq_len=8192)
    variants = VARIANTS + [("steal_off", "tdpipe", dict(steal=0)), ("tdpipe_sigma", "tdpipe",
                                                                      dict(eq2_bubble_scale=S - 1))]
    for name, pol, extra in variants:
        t = TDPipe(big, S, executor=tp.TD_EXEC_NULL, kv_blocks=C, profile_csv=prof, policy=POL[pol], log_decisions=0,
                   **extra)
        t.submit_workload(wl)
        st = t.td_simulate(30_000)
        emit(dict(kind="projection (B200 per-stage tables + td_simulate)", config=cfg + ("-cap" if kv_cap else ""),
                  model=model, stages=S, kv_blocks=C, variant=name, gen_tok_s=round(st["gen_tokens_per_s"]),
                  bubble=round(st["bubble_frac"], 4), makespan_s=round(st["makespan_ns"] / 1e9, 2), p2d=st["n_p2d"],
                  d2p=st["n_d2p"], stolen=st["n_stolen"], evicted=st["n_evicted"]), out)
        t.close()


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "AB"
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, "ablations.jsonl"), "a") as out:
        if "A" in what:
            measured(out)
        if "B" in what:
            projection(out, "C5", "llama2_70b", 8, kv_cap=24000)
            projection(out, "C4", "opt30b_shaped", 4)
