"""T1: the C++ controller (product, via the C ABI with the null executor) must
reproduce the reference scheduler's decision log byte for byte (SURVEY.md
§8(c) S12: batch membership, switch points, stolen requests, KV block tables).
CPU only: the null executor completes micro-batches logically."""
import dataclasses
import os

import numpy as np
import pytest

from oracle.scheduler import SchedOptions, schedule
from workload import generate_workload, random_tiny_workload, synthetic_profile, write_profile_csv

pytest.importorskip("ctypes")
from paper_2506_10470_b200 import TD_EXEC_NULL, TDPipe  # noqa: E402
from workload import SHAPES  # noqa: E402


def _run_both(wl, tmp_path, tag, **o):
    tdec, tpre = o.pop("tables")
    csv = os.path.join(str(tmp_path), f"prof_{tag}.csv")
    write_profile_csv(csv, tdec, tpre)
    reqs = [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]
    so = SchedOptions(n_stages=o["W"], block_size=o["B"], kv_blocks=o["C"], prefill_token_budget=o["budget"],
                      max_batch_seqs=o["max_seqs"], fp_stride=o["stride"], fp_horizon=o["horizon"],
                      policy=o["policy"], steal=o["steal"], alg1_check_before_launch=o["cbl"],
                      eq2_bubble_scale=o["sigma"], p2d_kv_permille=o.get("kvp", 0),
                      d2p_finish_permille=o.get("finp", 0), hb_tokens=o.get("hb", 512))
    ref = schedule(reqs, so, tdec, tpre)
    shape = dataclasses.replace(SHAPES["tiny"].with_layers(max(2, o["W"])), max_seq_len=4096)
    t = TDPipe(shape, o["W"], executor=TD_EXEC_NULL, block_size=o["B"], kv_blocks=o["C"],
               prefill_token_budget=o["budget"], max_batch_seqs=o["max_seqs"], fp_stride=o["stride"],
               fp_horizon=o["horizon"], policy=o["policy"], steal=o["steal"], alg1_check_before_launch=o["cbl"],
               eq2_bubble_scale=o["sigma"], profile_csv=csv, p2d_kv_permille=o.get("kvp", 0),
               d2p_finish_permille=o.get("finp", 0), hb_tokens=o.get("hb", 512))
    t.submit_workload(wl)
    st = t.td_run()
    got = t.td_get_log()
    want = "".join(line + "\n" for line in ref.log)
    n_out = [len(t.td_get_output(i)) for i in range(len(wl.requests))]
    t.close()
    return got, want, st, ref, n_out


def test_parity_random_tiny_workloads(tmp_path):
    """>= 1000 random tiny runs: random W, capacity, lengths, predictions, policy, flags."""
    rng = np.random.default_rng(123)
    kinds = set()
    for seed in range(1, 1101):
        wl = random_tiny_workload(seed, n_max=14, len_max=40)
        W = int(rng.integers(1, 6))
        B = int(rng.choice([1, 4, 16]))
        need = max((len(r.prompt) + r.max_new_tokens + B - 1) // B for r in wl.requests)
        policy = int(rng.choice([0, 0, 0, 1, 2]))
        C = int(need * (W if policy else 1) + rng.integers(0, 3 * need + 1))
        o = dict(W=W, B=B, C=C, budget=int(rng.choice([16, 40, 64, 2048])), max_seqs=int(rng.choice([2, 4, 8, 64])),
                 stride=int(rng.choice([1, 2, 4, 32])), horizon=int(rng.choice([4, 16, 64])), policy=policy,
                 steal=int(rng.integers(0, 2)), cbl=int(rng.integers(0, 2)), sigma=int(rng.choice([1, max(1, W - 1)])),
                 tables=synthetic_profile(int(rng.choice([8, 64])), int(rng.choice([32, 512])),
                                          knee=int(rng.integers(0, 12))),
                 kvp=int(rng.choice([0, 0, 0, 300, 700])), finp=int(rng.choice([0, 0, 0, 250, 500, 900])))
        got, want, st, ref, n_out = _run_both(wl, tmp_path, seed % 7, **o)
        assert got == want, f"seed {seed} opts {o}\n--- first diff at line " + str(
            next((i for i, (a, b) in enumerate(zip(got.splitlines(), want.splitlines())) if a != b), None))
        assert n_out == [r.max_new_tokens for r in wl.requests]
        for line in ref.log:
            kinds.add(line.split()[0] + (line.split()[1] if line.startswith("S") else ""))
    for k in ["P", "G", "A", "F", "D", "R", "SP2D", "SD2P", "E", "W", "U", "X"]:
        assert k in kinds, (k, kinds)


def test_parity_pphb_random(tmp_path):
    """PP+HB baseline [R23]: 400 random tiny runs, C++ controller log == oracle
    log byte for byte (chunk splits, admissions, evictions, finishes)."""
    rng = np.random.default_rng(77)
    kinds = set()
    n_chunked = 0
    for seed in range(2001, 2401):
        wl = random_tiny_workload(seed, n_max=14, len_max=40)
        W = int(rng.integers(1, 6))
        B = int(rng.choice([1, 4, 16]))
        need = max((len(r.prompt) + r.max_new_tokens + B - 1) // B for r in wl.requests)
        C = int(need * W + rng.integers(0, 3 * need + 1))
        o = dict(W=W, B=B, C=C, budget=2048, max_seqs=64, stride=32, horizon=64, policy=3, steal=1, cbl=0, sigma=1,
                 tables=synthetic_profile(8, 32, knee=4), hb=int(rng.choice([1, 7, 16, 32, 512])))
        got, want, st, ref, n_out = _run_both(wl, tmp_path, seed % 7, **o)
        assert got == want, f"seed {seed} opts {o}\n--- first diff at line " + str(
            next((i for i, (a, b) in enumerate(zip(got.splitlines(), want.splitlines())) if a != b), None))
        assert n_out == [r.max_new_tokens for r in wl.requests]
        for line in ref.log:
            kinds.add(line.split()[0])
            if line.startswith("H"):
                n_chunked += sum(1 for x in line.split()[5:] if ":" in x and not x.split(":")[1] == "0")
    for k in ["H", "A", "F", "R", "E"]:
        assert k in kinds, (k, kinds)
    assert n_chunked > 100   # prompts really are split over several micro-batches


def test_parity_sharegpt_shaped(tmp_path):
    """Larger ShareGPT-shaped sets (bucket predictor) at W = 2, 4, 8, KV-constrained."""
    for W, seed in [(2, 31), (4, 32), (8, 33)]:
        wl = generate_workload(300, 256, seed, in_max=500, out_max=400)
        need = sum((len(r.prompt) + r.max_new_tokens + 15) // 16 for r in wl.requests)
        o = dict(W=W, B=16, C=max(need // 4, 64), budget=2048, max_seqs=1024, stride=32, horizon=1024, policy=0,
                 steal=1, cbl=0, sigma=1, tables=synthetic_profile(512, 2048, dec_base_ns=3_000_000,
                                                                   dec_per_req_ns=4_000, knee=96))
        got, want, st, ref, _ = _run_both(wl, tmp_path, W, **o)
        assert got == want
        assert st["n_d2p"] == ref.stats["d2p"] and st["n_evicted"] == ref.stats["evicted"]
