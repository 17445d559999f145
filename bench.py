#!/usr/bin/env python
"""TD-Pipe hot-path benchmark (contract: one JSON line on rank 0).

Step = one pass of the whole hot path over one batch of synthetic input: the
complete offline job of BASELINE.json config[1] at N=1 -- Llama-2-7B-shaped
random-init weights (all 32 layers), 256 ShareGPT-length requests with
bucket-predicted output lengths, run to completion by the TD-Pipe controller
(prefill phases + decode phases).  Metric: generated
tokens/s (BASELINE.json "metric"), plus bubble %, roofline fractions.

  value  generated tokens / device time of td_run (CUDA events on the library's
         stream), prompts already resident in HBM (td_upload before timing)
  e2e    same metric through the C ABI from HOST buffers: td_submit + td_upload
         (H2D) + td_run + td_get_outputs (D2H) inside the timed region

--impl reference times the oracle (oracle/, numpy fp64) on the host cores on a
bounded sample of the same workload (the tier's reference arm).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from workload import SHAPES, config_workload  # noqa: E402

METRIC = "generated tokens/s (8×B200 pipeline) + bubble %, HBM/TC roofline fraction"
UNIT = "tokens/s"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm=d["hbm_gbs"], tc=d["bf16_tflops"], tc_sus=d.get("bf16_tflops_sustained", d["bf16_tflops"]),
                    src="measured (MEASURED_PEAKS.json)")
    # the driver writes MEASURED_PEAKS.json per pod; without it, the values it
    # held on this pool in round 1 (recorded in profiles/README.md)
    return dict(hbm=6535.7, tc=1673.3, tc_sus=1406.7,
                src="MEASURED_PEAKS.json absent: this pool's round-1 measured peaks (profiles/README.md)")


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------- oracle arm
# SURVEY.md §8(d) "Oracle timing": the oracle as it stands (oracle/, numpy fp32
# as §8(d) states, BLAS threads = the cores this process may use), timed on
# the GPU box's host in the same harness run: C1 end to end; a C2 slice (one
# 2,048-token prefill + 8 decode steps at b = 256); reference-scheduler
# decisions/s on the C5 request set.  A baseline, not the target.
_ORACLE_W = {}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def host_info():
    """cores used, cpu_count, CPU model, BLAS vendor/threads (threadpoolctl)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    blas = None
    try:
        import threadpoolctl
        for d in threadpoolctl.threadpool_info():
            if d.get("user_api") == "blas":
                blas = {"vendor": d.get("internal_api"), "version": d.get("version"),
                        "threads": d.get("num_threads"), "arch": d.get("architecture")}
                break
    except Exception:
        pass
    return {"cores": cpu_cores(), "cpu_count": os.cpu_count(), "cpu_model": model, "blas": blas}


def _blas_threads():
    try:
        import threadpoolctl
        return threadpoolctl.threadpool_limits(limits=cpu_cores(), user_api="blas")
    except Exception:
        import contextlib
        return contextlib.nullcontext()


def oracle_c1():
    """C1 end to end: the 8 C1 requests (prompt 16 / output 16), greedy decode
    per request with the F6 KV cache (oracle/cached.py), tiny model, fp32."""
    from oracle import cached as Cc
    from oracle.weights import OracleWeights
    wl = config_workload("C1")
    W = OracleWeights(SHAPES["tiny"])
    Cc.greedy_generate_cached(W, wl.requests[0].prompt, 2, dtype=np.float32)   # weights + casts: setup
    t0 = time.perf_counter()
    gen = 0
    for r in wl.requests:
        toks, _ = Cc.greedy_generate_cached(W, r.prompt, r.max_new_tokens, dtype=np.float32)
        gen += len(toks)
    dt = time.perf_counter() - t0
    return {"value": gen / dt, "unit": UNIT, "seconds": round(dt, 3), "generated": gen,
            "sample": "C1 end to end: 8 requests x (prompt 16, output 16), tiny model, fp32, per-request KV cache"}


def oracle_c2_slice(layers=2, n_dec=8, b=256):
    """C2 slice: one <= 2,048-token prefill micro-batch of
    C2 prompts, then `n_dec` decode steps of b = 256 C2 requests, through
    `layers` of the 32 Llama-2-7B layers and the LM head, numpy fp32 with the
    F6 per-request KV cache; the per-layer time (measured minus a 0-layer run)
    is scaled to 32 layers.  The decode requests' caches hold seeded random
    K/V at their C2 prompt lengths (their 58k-token prefill is not part of the
    slice).  Returns generated tokens/s (the bench metric) of the slice."""
    from oracle import cached as Cc
    from oracle.weights import OracleWeights
    full = SHAPES["llama2_7b"]
    shape = full.with_layers(layers)
    key = ("c2", layers)
    if key not in _ORACLE_W:
        W = OracleWeights(shape)
        for l in range(layers):
            Cc._weights(W, l, np.float32)
            W.drop_layer(l)
        for g in ("embed", "gf", "lm"):
            Cc._global(W, g, np.float32)
        W._embed = W._lm = None
        _ORACLE_W[key] = W
    W = _ORACLE_W[key]
    wl = config_workload("C2")
    pre, tok = [], 0
    for r in wl.requests:
        if tok + len(r.prompt) > 2048:
            break
        pre.append(r.prompt)
        tok += len(r.prompt)
    rng = np.random.default_rng(0)
    hd, hkv = full.head_dim, full.n_kv_heads

    kvkey = ("kv", layers, b)
    if kvkey not in _ORACLE_W:   # seeded K/V of the decode requests, drawn once (setup, untimed)
        _ORACLE_W[kvkey] = [[(rng.standard_normal((len(r.prompt), hkv, hd), dtype=np.float32),
                              rng.standard_normal((len(r.prompt), hkv, hd), dtype=np.float32))
                             for _ in range(layers)] for r in wl.requests[:b]]

    def caches_for_decode():
        cs = []
        for r, kv in zip(wl.requests[:b], _ORACLE_W[kvkey]):
            c = Cc.Cache(layers)
            for l in range(layers):
                c.k[l], c.v[l] = kv[l]     # a step appends by concatenation: the drawn arrays stay intact
            c.T = len(r.prompt)
            cs.append(c)
        return cs

    def run(lys):
        cs = [Cc.Cache(layers) for _ in pre]
        dec = caches_for_decode()
        toks = [[int(t)] for t in rng.integers(0, full.vocab, size=b)]
        t0 = time.perf_counter()
        Cc.forward_rows(W, cs, pre, layers=lys, dtype=np.float32)
        for _ in range(n_dec):
            lg = Cc.forward_rows(W, dec, toks, layers=lys, dtype=np.float32)
            toks = [[int(t)] for t in np.argmax(lg, -1)]
        return time.perf_counter() - t0

    with _blas_threads():
        t_l = run(range(layers))
        if ("t0", n_dec, b) not in _ORACLE_W:   # the 0-layer part (embedding + LM head), measured once
            _ORACLE_W[("t0", n_dec, b)] = run([])
        t_0 = _ORACLE_W[("t0", n_dec, b)]
    per_layer = max(t_l - t_0, 0.0) / layers
    scaled = t_0 + per_layer * full.n_layers
    gen = len(pre) + n_dec * b
    return {"value": gen / scaled, "unit": UNIT, "seconds": round(t_l + t_0, 2), "scaled_seconds": round(scaled, 2),
            "generated": gen,
            "sample": f"C2 slice: one {tok}-token prefill ({len(pre)} C2 prompts) + {n_dec} decode steps at b={b} "
                      f"(contexts = C2 prompt lengths, seeded random K/V), {layers}/{full.n_layers} Llama-2-7B "
                      f"layers + LM head, numpy fp32, per-request KV cache; per-layer time scaled to "
                      f"{full.n_layers} layers"}


def oracle_sched_c5():
    """Reference-scheduler decisions/s on the C5 request set (4,096 requests,
    8 stages, KV-capped to 24,000 blocks = C5-cap, synthetic frozen profile):
    decision-log lines per second of oracle/scheduler.py."""
    from oracle.scheduler import SchedOptions, schedule
    from workload import synthetic_profile
    wl = config_workload("C5")
    reqs = [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]
    tdec, tpre = synthetic_profile(1024, 2048, knee=64)
    t0 = time.perf_counter()
    s = schedule(reqs, SchedOptions(n_stages=8, block_size=16, kv_blocks=24000), tdec, tpre)
    dt = time.perf_counter() - t0
    return {"value": len(s.log) / dt, "unit": "decisions/s", "seconds": round(dt, 2), "decisions": len(s.log),
            "micro_batches": len(s.plan),
            "sample": "oracle/scheduler.py on C5 (4096 requests, W=8, kv_blocks=24000), decision-log lines/s"}


def cpu_baseline(with_c1=True, with_sched=True):
    c2 = oracle_c2_slice(layers=1)
    out = {"value": c2["value"], "unit": UNIT, "kind": "oracle", "sample": c2["sample"], "c2_slice": c2}
    out.update(host_info())
    if with_c1:
        out["c1_e2e"] = oracle_c1()
    if with_sched:
        out["sched_c5"] = oracle_sched_c5()
    return out


def run_reference(args):
    """The tier's reference arm: the oracle as it stands on the host cores;
    one step = the C2 slice (a bounded sample of the bench workload)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    vals, secs = [], []
    desc = ""
    for i in range(args.warmup + args.steps):
        r = oracle_c2_slice(layers=1, n_dec=2)
        desc = r["sample"]
        if i >= args.warmup:
            vals.append(r["value"])
            secs.append(r["seconds"])
    value = statistics.mean(vals)
    cb = {"value": value, "unit": UNIT, "kind": "oracle", "sample": desc}
    cb.update(host_info())
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(secs),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload_config(args), "cpu_baseline": cb,
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, n_gpus=1):
    shape = SHAPES[args.model]
    wl = config_workload(args.config)
    n_req = len(wl.requests)
    return {"workload": f"{args.config}: {shape.name}-shaped random-init ({shape.n_layers} layers), {n_req} "
                        f"ShareGPT-length requests, bucket-predicted lengths, {max(n_gpus, args.stages)}-stage "
                        f"TD-Pipe ({args.policy})",
            "model": shape.name, "n_requests": n_req, "global_batch": n_req,
            "parallelism": f"pp{max(n_gpus, args.stages)}",
            "l2": "inputs larger than L2 (weights + KV per step >> 126 MB)"}


def job_roofline(stats, peaks):
    """Whole-job speed of light: the engine's per-micro-batch
    algorithmic bytes / FLOPs (td_run_stats), ideal = sum over micro-batches of
    max(bytes / HBM peak, FLOPs / TC peak), divided by the measured makespan."""
    ideal = sum(s["ideal_ns"] for s in stats)
    span = sum(s["makespan_ns"] for s in stats)
    n = max(len(stats), 1)
    return {"frac": round(ideal / span, 4) if span else None, "ideal_ms_per_step": round(ideal / 1e6 / n, 2),
            "ms_per_step": round(span / 1e6 / n, 2), "alg_bytes_per_step": sum(s["alg_bytes"] for s in stats) / n,
            "alg_flops_per_step": sum(s["alg_flops"] for s in stats) / n, "peak_hbm_gbs": peaks["hbm"],
            "peak_tc_tflops": peaks["tc_sus"],
            "def": "sum_mb max(bytes/HBM, flops/TC) / makespan; bytes = weights once + K/V of every context "
                   "token per layer + new K/V; flops = 2*tokens*weights + causal attention"}


def _traffic_record(kernel):
    import glob
    files = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r*",
                                          f"traffic_{kernel}.json")))
    if not files:
        return None
    rec = json.load(open(files[-1]))
    rec["file"] = os.path.relpath(files[-1], os.path.dirname(os.path.abspath(__file__)))
    return rec


# ----------------------------------------------------------- C5 stage record
DEC_CLASSES = ["decode_attn", "gemm_qkv_dec", "gemm_o_dec", "gemm_gu_dec", "gemm_down_dec", "lm_head_dec"]
PRE_CLASSES = ["prefill_attn", "gemm_qkv_pre", "gemm_o_pre", "gemm_gu_pre", "gemm_down_pre", "lm_head_pre"]


def c5_stage(peaks, iters=10):
    """The headline config's per-stage hot path (BASELINE configs[4]: Llama-2-70B,
    8-stage pipeline => 10 of 80 layers per stage), measured on this GPU with
    td_bench_step: decode micro-batches of b = 64 / 256 / 512 sequences at the
    C5 workload's representative context (mean prompt + half the mean
    predicted output) and a 2,048-token prefill (8 x 256).
    Per kernel class: achieved bytes/s and FLOP/s and the fraction of its
    attainable roofline max(bytes / HBM, FLOPs / TC) / time (GQA-8 decode
    attention and the tensor-bound decode GEMMs at b = 512).  Parity of this
    shape is tests/test_gpu_parity.py::test_llama70b_shaped_layer_gqa8*.
    The stage here also holds the embedding and LM head (the last stage)."""
    from paper_2506_10470_b200 import TD_BATCH_DECODE, TD_BATCH_PREFILL, TDPipe
    shape = SHAPES["llama2_70b"].with_layers(10)
    wl = config_workload("C5")
    n_req = len(wl.requests)
    L = np.array([len(r.prompt) for r in wl.requests])
    P = np.array([r.predicted_len for r in wl.requests])
    ctx_rep = int(L.sum() // n_req + (P.sum() // n_req) // 2)
    t = TDPipe(shape, 1, device=0, kv_blocks=12288, hbm_peak_gbs=peaks["hbm"], tc_peak_tflops=peaks["tc_sus"])
    rec = {"model": "Llama-2-70B-shaped, 10 of 80 layers (one stage of the 8-stage pipeline) + embedding + LM head",
           "ctx_rep": ctx_rep, "peak_hbm_gbs": peaks["hbm"], "peak_tc_tflops": peaks["tc_sus"],
           "parity": "tests/test_gpu_parity.py::test_llama70b_shaped_layer_gqa8 (+ _large_decode_batch)", "steps": {}}
    for label, kind, n, ln, classes in [("decode_b64", TD_BATCH_DECODE, 64, ctx_rep, DEC_CLASSES),
                                        ("decode_b256", TD_BATCH_DECODE, 256, ctx_rep, DEC_CLASSES),
                                        ("decode_b512", TD_BATCH_DECODE, 512, ctx_rep, DEC_CLASSES),
                                        ("prefill_T2048", TD_BATCH_PREFILL, 8, 256, PRE_CLASSES)]:
        us, ideal = t.td_bench_step(kind, n, ln, iters)
        ks = {}
        for name in classes:
            v = t.td_get_timing(name)
            if v["ms"] <= 0:
                continue
            sec = v["ms"] * 1e-3
            att = max(v["bytes"] / (peaks["hbm"] * 1e9), v["flops"] / (peaks["tc_sus"] * 1e12))
            ks[name] = {"launches": v["launches"], "us_per_launch": round(v["ms"] * 1e3 / v["launches"], 2),
                        "GB/s": round(v["bytes"] / sec / 1e9, 1), "TFLOP/s": round(v["flops"] / sec / 1e12, 1),
                        "bound": "tensor" if v["flops"] / (peaks["tc_sus"] * 1e12) > v["bytes"] / (peaks["hbm"] * 1e9)
                        else "hbm", "frac": round(att / sec, 4)}
        rec["steps"][label] = {"n_seqs": n, "len": ln, "us": round(us, 1), "ideal_us": round(ideal, 1),
                               "sol_frac": round(ideal / us, 4) if us else None, "kernels": ks}
    t.close()
    return rec


# ---------------------------------------------------------------------- our arm
def run_ours(args):
    import paper_2506_10470_b200 as tp
    from paper_2506_10470_b200 import TDPipe

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        return run_ours_multiprocess(args, world, rank)
    peaks = load_peaks()
    shape = SHAPES[args.model]
    wl = config_workload(args.config)
    n_req = len(wl.requests)
    policy = {"tdpipe": tp.TD_POLICY_TDPIPE, "ppsb_prio": tp.TD_POLICY_PPSB_PRIO,
              "ppsb_alt": tp.TD_POLICY_PPSB_ALT, "pphb": tp.TD_POLICY_PPHB}[args.policy]
    t = TDPipe(shape, args.stages, device=0, policy=policy, eq2_bubble_scale=args.sigma,
               hbm_peak_gbs=peaks["hbm"], tc_peak_tflops=peaks["tc_sus"])
    info = t.td_info()
    # frozen profile table for Eq.1/Eq.2, measured once, untimed
    L = np.array([len(r.prompt) for r in wl.requests])
    P = np.array([r.predicted_len for r in wl.requests])
    ctx_rep = int(L.sum() // n_req + (P.sum() // n_req) // 2)
    prof = os.path.join("gpurun_out" if os.path.isdir("gpurun_out") else tempfile.gettempdir(),
                        f"tdpipe_profile_{args.config}_{os.getpid()}.csv")
    t0 = time.perf_counter()
    t.td_profile(prof, min(1024, max(n_req, 1)), 2048, ctx_rep)
    prof_s = time.perf_counter() - t0

    def one_step():
        t.td_reset()
        t.submit_workload(wl)
        t.td_upload()
        return t.td_run()

    t.td_set_timing(False)
    for _ in range(args.warmup):
        one_step()
    # timed region: K whole-job steps, no per-kernel instrumentation
    sampler = ClockSampler(0)
    sampler.start()
    stats = []
    wall0 = time.perf_counter()
    for _ in range(args.steps):
        stats.append(one_step())
    wall = time.perf_counter() - wall0
    clocks = sampler.stop()
    # roofline pass: the same K steps again with CUDA events around every hot
    # kernel on the library's stream (events serialise PDL overlap, so these
    # per-kernel durations are slightly pessimistic)
    kstats = []
    if not args.no_timing:
        t.td_set_timing(True)
        for _ in range(args.steps):
            kstats.append(one_step())
        t.td_set_timing(False)
    gen = sum(s["generated_tokens"] for s in stats)
    dev_s = sum(s["makespan_ns"] for s in stats) / 1e9
    value = gen / dev_s
    # roofline of the dominant kernel class over the timed region
    kern = {}
    if not args.no_timing:
        for name in ["decode_attn", "prefill_attn", "gemm_qkv_dec", "gemm_o_dec", "gemm_gu_dec", "gemm_down_dec",
                     "lm_head_dec", "gemm_qkv_pre", "gemm_o_pre", "gemm_gu_pre", "gemm_down_pre", "lm_head_pre",
                     "decode_attn@b1-8", "decode_attn@b9-32", "decode_attn@b33-128", "decode_attn@b129+",
                     "gemm_dec@b1-8", "gemm_dec@b9-32", "gemm_dec@b33-128", "gemm_dec@b129+"]:
            kern[name] = t.td_get_timing(name)   # accumulated over the K timed steps
    # e2e: host buffers through the public API, H2D + D2H inside the timed region
    e2e_vals = []
    h2d = d2h = 0
    t.td_set_timing(False)
    for _ in range(max(1, min(args.steps, 2))):
        t.td_reset()
        s0 = time.perf_counter()
        t.submit_workload(wl)
        t.td_upload()
        st = t.td_run()
        out, n = t.td_get_outputs(n_req, int(max(r.max_new_tokens for r in wl.requests)))
        e2e_vals.append(st["generated_tokens"] / (time.perf_counter() - s0))
        h2d = int(sum(len(r.prompt) + r.max_new_tokens + 1 for r in wl.requests) * 4 + st["h2d_bytes"])
        d2h = int(sum(len(r.prompt) + r.max_new_tokens + 1 for r in wl.requests) * 4)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "scope": f"N=1 point of the metric's 1/2/4/8-GPU series: one B200, {args.stages} pipeline stage(s) in one "
                 f"process (the multi-GPU pipeline runs under torchrun)",
        "ms_per_step": dev_s * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic",
        "config": dict(workload_config(args), kv_blocks=info["kv_blocks"], profile_s=round(prof_s, 2)),
        "bubble_pct": 100.0 * statistics.mean(s["bubble_frac"] for s in kstats) if kstats else None,
        "total_tokens_per_s": sum(s["generated_tokens"] + s["prompt_tokens"] for s in stats) / dev_s,
        "wall_tokens_per_s": gen / wall,
        "gpu_launches": int(sum(s["gpu_launches"] for s in stats)),
        "sched": {k: stats[-1][k] for k in ["n_microbatches", "n_prefill_mb", "n_decode_mb", "n_p2d", "n_d2p",
                                            "n_stolen", "n_evicted", "prompt_tokens", "generated_tokens"]},
        "clocks": clocks,
        "e2e": {"value": statistics.mean(e2e_vals), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
        "job_roofline": job_roofline(stats, peaks),
    }
    if kern:
        main = {k: v for k, v in kern.items() if "@" not in k}
        tot_ms = sum(k["ms"] for k in main.values())
        dom = max(main, key=lambda k: main[k]["ms"])
        share = {k: round(v["ms"] / tot_ms, 4) for k, v in main.items() if tot_ms > 0}
        rl = {}
        for k, v in kern.items():
            if v["ms"] <= 0:
                continue
            gbs = v["bytes"] / (v["ms"] * 1e-3) / 1e9
            tfs = v["flops"] / (v["ms"] * 1e-3) / 1e12
            rl[k] = {"launches": v["launches"], "ms": round(v["ms"], 3), "GB/s": round(gbs, 1),
                     "TFLOP/s": round(tfs, 1), "hbm_frac": round(gbs / peaks["hbm"], 4),
                     "tc_frac": round(tfs / peaks["tc_sus"], 4)}
        d = kern[dom]
        if dom.endswith("_pre") or dom == "prefill_attn":
            ach = d["flops"] / (d["ms"] * 1e-3) / 1e12
            line["roofline"] = {"kernel": dom, "bound": "tensor", "achieved": round(ach, 1), "peak": peaks["tc_sus"],
                                "unit": "TFLOP/s", "frac": round(ach / peaks["tc_sus"], 4), "traffic": None,
                                "peak_src": peaks["src"] + " (bf16 sustained)"}
        else:
            ach = d["bytes"] / (d["ms"] * 1e-3) / 1e9
            line["roofline"] = {"kernel": dom, "bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm"],
                                "unit": "GB/s", "frac": round(ach / peaks["hbm"], 4), "traffic": None,
                                "peak_src": peaks["src"]}
            # DRAM bytes per launch measured by ncu over every launch of this
            # kernel in one C2 job (scripts/traffic_attn.py), next to the
            # algorithmic bytes per launch the engine counted for the same job
            tf = _traffic_record(dom)
            if tf:
                line["roofline"].update(traffic=round(tf["dram_bytes_per_launch"]),
                                        traffic_algorithmic=round(tf["algorithmic_bytes_per_launch"]),
                                        traffic_ratio=round(tf["ratio"], 4), traffic_src=tf["file"])
        line["kernels"] = rl
        line["kernel_share"] = share
    t.close()
    if not args.no_c5_stage:
        line["c5_stage"] = c5_stage(peaks)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline()
    print(json.dumps(line), flush=True)
    return 0


def run_ours_multiprocess(args, world, rank):
    """N > 1: one process per GPU = one pipeline stage (torchrun).  The
    controller is replicated on every rank (decisions depend only on logical
    events); the fp32 residual moves stage -> stage and the sampled tokens
    last -> stage 0 through the library's peer-store hand-off (CUDA-IPC
    mailboxes over NVLink, stream-ordered flags; `--handoff nccl` = the NCCL
    send/recv baseline).  torch.distributed (gloo, host only) carries the
    library's allgather callback (IPC handles, KV-capacity min, profile max),
    the barriers and the max over ranks of the per-rank device times.
    TDPIPE_SAME_DEVICE=1 puts every rank on cuda:0 (single-GPU check of the
    multi-process path; the KV pool is then capped by --kv-blocks)."""
    import torch
    import torch.distributed as dist

    import paper_2506_10470_b200 as tp
    from paper_2506_10470_b200 import TDPipe, td_nccl_ids

    same = os.environ.get("TDPIPE_SAME_DEVICE") == "1"
    local = 0 if same else int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")

    def gather(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out

    def max_over_ranks(v):
        x = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
        return float(x.item())

    def sum_over_ranks(v):
        x = torch.tensor([float(v)], dtype=torch.float64)
        dist.all_reduce(x)
        return float(x.item())

    extra = {}
    if args.handoff == "nccl":
        ids = [td_nccl_ids() if rank == 0 else None]
        dist.broadcast_object_list(ids, src=0)
        import ctypes
        idbuf = ctypes.create_string_buffer(ids[0], 256)
        extra = dict(handoff=tp.TD_HANDOFF_NCCL, nccl_ids=ctypes.cast(idbuf, ctypes.c_void_p))
    kvb = args.kv_blocks or (2048 if same else 0)
    peaks = load_peaks()
    shape = SHAPES[args.model]
    wl = config_workload(args.config)
    n_req = len(wl.requests)
    policy = {"tdpipe": tp.TD_POLICY_TDPIPE, "ppsb_prio": tp.TD_POLICY_PPSB_PRIO,
              "ppsb_alt": tp.TD_POLICY_PPSB_ALT, "pphb": tp.TD_POLICY_PPHB}[args.policy]
    t = TDPipe(shape, world, device=local, policy=policy, eq2_bubble_scale=args.sigma, world_size=world, rank=rank,
               allgather=gather, kv_blocks=kvb, hbm_peak_gbs=peaks["hbm"], tc_peak_tflops=peaks["tc_sus"], **extra)
    info = t.td_info()
    L = np.array([len(r.prompt) for r in wl.requests])
    P = np.array([r.predicted_len for r in wl.requests])
    ctx_rep = int(L.sum() // n_req + (P.sum() // n_req) // 2)
    t0 = time.perf_counter()
    t.td_profile(None, min(1024, max(n_req, 1)), 2048, ctx_rep)
    prof_s = time.perf_counter() - t0

    def one_step():
        t.td_reset()
        t.submit_workload(wl)
        t.td_upload()
        dist.barrier()
        torch.cuda.synchronize()
        st = t.td_run()
        torch.cuda.synchronize()
        return st

    t.td_set_timing(False)
    for _ in range(args.warmup):
        one_step()
    sampler = ClockSampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
    stats = [one_step() for _ in range(args.steps)]
    clocks = sampler.stop() if sampler else None
    dev_s = max_over_ranks(sum(s["makespan_ns"] for s in stats) / 1e9)
    # slowest stage's speed of light vs the pipeline makespan
    ideal_s = max_over_ranks(sum(s["ideal_ns"] for s in stats) / 1e9)
    gen = sum(s["generated_tokens"] for s in stats)
    launches = int(sum_over_ranks(sum(s["gpu_launches"] for s in stats)))
    # instrumented pass: per-kernel CUDA events on every rank; bubble from the
    # per-rank stage busy time (PAPER.md:454 reading R19)
    kern, bubble = {}, None
    if not args.no_timing:
        t.td_set_timing(True)
        kst = [one_step() for _ in range(args.steps)]
        t.td_set_timing(False)
        span = max_over_ranks(sum(s["makespan_ns"] for s in kst) / 1e6)
        busy = sum_over_ranks(t.td_get_timing("stage")["ms"])
        bubble = 100.0 * (1.0 - busy / (world * span)) if span > 0 else None
        for name in ["decode_attn", "prefill_attn", "gemm_qkv_dec", "gemm_o_dec", "gemm_gu_dec", "gemm_down_dec",
                     "lm_head_dec", "gemm_qkv_pre", "gemm_o_pre", "gemm_gu_pre", "gemm_down_pre", "lm_head_pre"]:
            kern[name] = t.td_get_timing(name)   # this rank's stage
    # e2e through the public API: prompts H2D, run, outputs D2H (stage 0)
    e2e = []
    for _ in range(max(1, min(args.steps, 2))):
        t.td_reset()
        dist.barrier()
        torch.cuda.synchronize()
        s0 = time.perf_counter()
        t.submit_workload(wl)
        t.td_upload()
        st = t.td_run()
        if rank == 0:
            t.td_get_outputs(n_req, int(max(r.max_new_tokens for r in wl.requests)))
        e2e.append(st["generated_tokens"] / max_over_ranks(time.perf_counter() - s0))
    if rank == 0:
        arena = int(sum(len(r.prompt) + r.max_new_tokens + 1 for r in wl.requests) * 4)
        line = {"metric": METRIC, "value": gen / dev_s, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dev_s * 1e3 / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
                "config": dict(workload_config(args, world), kv_blocks=info["kv_blocks"], handoff=args.handoff,
                               same_device=same, profile_s=round(prof_s, 2)),
                "bubble_pct": bubble, "gpu_launches": launches, "clocks": clocks,
                "sched": {k: stats[-1][k] for k in ["n_microbatches", "n_prefill_mb", "n_decode_mb", "n_p2d",
                                                    "n_d2p", "n_stolen", "n_evicted", "prompt_tokens",
                                                    "generated_tokens"]},
                "e2e": {"value": statistics.mean(e2e), "unit": UNIT, "h2d_bytes_per_step": arena,
                        "d2h_bytes_per_step": arena},
                "job_roofline": {"frac": round(ideal_s / dev_s, 4) if dev_s else None,
                                 "def": "max over stages of sum_mb max(bytes/HBM, flops/TC) / pipeline makespan"}}
        main = {k: v for k, v in kern.items() if v["ms"] > 0}
        if main:
            dom = max(main, key=lambda k: main[k]["ms"])
            d = main[dom]
            if dom.endswith("_pre") or dom == "prefill_attn":
                ach = d["flops"] / (d["ms"] * 1e-3) / 1e12
                line["roofline"] = {"kernel": dom + " (stage 0)", "bound": "tensor", "achieved": round(ach, 1),
                                    "peak": peaks["tc_sus"], "unit": "TFLOP/s", "frac": round(ach / peaks["tc_sus"], 4),
                                    "traffic": None, "peak_src": peaks["src"] + " (bf16 sustained)"}
            else:
                ach = d["bytes"] / (d["ms"] * 1e-3) / 1e9
                line["roofline"] = {"kernel": dom + " (stage 0)", "bound": "hbm", "achieved": round(ach, 1),
                                    "peak": peaks["hbm"], "unit": "GB/s", "frac": round(ach / peaks["hbm"], 4),
                                    "traffic": None, "peak_src": peaks["src"]}
        print(json.dumps(line), flush=True)
    dist.barrier()
    t.close()
    dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2")
    ap.add_argument("--model", default="llama2_7b")
    ap.add_argument("--stages", type=int, default=1)
    ap.add_argument("--policy", default="tdpipe", choices=["tdpipe", "ppsb_prio", "ppsb_alt", "pphb"])
    ap.add_argument("--sigma", type=int, default=1)
    ap.add_argument("--no-timing", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5-stage", action="store_true")
    ap.add_argument("--handoff", default="peer", choices=["peer", "nccl"])
    ap.add_argument("--kv-blocks", type=int, default=0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
