"""Pins for the reference scheduler -- CPU only.

Checked against: the paper's / SPEC's printed examples (tests/golden/
paper_examples.json), a per-step brute-force KV ledger (Alg.1 exactness),
closed-form Eq.1/Eq.2 values, and whole-run invariants (token conservation,
no double-owned block, capacity-infinite => one P->D and no D->P).
"""
import json
import os
from collections import defaultdict

import numpy as np
import pytest

from oracle.scheduler import (PPSB_ALT, PPSB_PRIO, TDPIPE, RefScheduler, SchedOptions, Slot,
                              ceil_div, schedule)
from workload import random_tiny_workload, synthetic_profile

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_examples.json")))


def reqs_of(wl):
    return [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]


# --------------------------------------------------------------- Alg.1 pieces
def test_future_points_default():
    s = RefScheduler(SchedOptions(), [(10, 5, 5)])
    g = GOLD["future_points"]
    assert s.fps[:3] == g["first"] and s.fps[-2:] == g["last"] and len(s.fps) == g["count"]


def test_update_usage_spec_example():
    g = GOLD["update_usage"]
    o = SchedOptions(block_size=1, fp_stride=32, fp_horizon=96)
    s = RefScheduler(o, [(g["input_len"], g["remaining_decode_steps"] + 1, 500)])
    assert s.fps == g["points"]
    U = {fp: 0 for fp in s.fps}
    s.update_usage(U, s.reqs[0])
    assert [U[p] for p in g["points"]] == g["gains"]
    # order independence
    s2 = RefScheduler(o, [(100, 65, 500), (7, 40, 500)])
    U1 = {fp: 0 for fp in s2.fps}; U2 = dict(U1)
    s2.update_usage(U1, s2.reqs[0]); s2.update_usage(U1, s2.reqs[1])
    s2.update_usage(U2, s2.reqs[1]); s2.update_usage(U2, s2.reqs[0])
    assert U1 == U2


def test_check_switch_spec_examples():
    for U, C, want in GOLD["check_switch"]["cases"]:
        assert RefScheduler.check_switch({int(k): v for k, v in U.items()}, C) == want


def test_prefill_budget_spec_example():
    g = GOLD["prefill_budget"]
    tdec, tpre = synthetic_profile(64, 4096)
    s = schedule([(L, 4, 4) for L in g["inputs"]],
                 SchedOptions(prefill_token_budget=g["budget"], block_size=1), tdec, tpre)
    sizes = [int(l.split()[2]) for l in s.log if l.startswith("P ")]
    assert sizes == g["batch_sizes"]
    # a request longer than the budget forms a singleton batch, never dropped
    s = schedule([(3000, 2, 2), (5, 2, 2)], SchedOptions(prefill_token_budget=2048), tdec, tpre)
    assert [l.split()[:3] for l in s.log if l.startswith("P ")] == [["P", "0", "1"], ["P", "1", "1"]]


def test_alg1_forecast_equals_bruteforce_ledger():
    """With the oracle predictor (P = N) and no later admissions, the forecast at
    every futurePoint equals the blocks actually allocated during that decode
    step (Alg.1 exactness under reading R1), and between points the
    excess over the preceding point is <= alive * ceil((stride-1)/B)."""
    rng = np.random.default_rng(0)
    for trial in range(40):
        n = int(rng.integers(1, 20))
        B = int(rng.choice([1, 4, 16]))
        stride = int(rng.choice([1, 2, 4, 8]))
        reqs = [(int(rng.integers(1, 60)), 0, int(rng.integers(1, 50))) for _ in range(n)]
        reqs = [(L, N, N) for L, _, N in reqs]                         # oracle predictor
        o = SchedOptions(n_stages=1, block_size=B, fp_stride=stride, fp_horizon=stride)
        tdec, tpre = synthetic_profile(64, 4096)
        s = RefScheduler(o, reqs, tdec, tpre)
        s._evict_key = {}
        U = {fp: 0 for fp in s.fps}
        for r in s.reqs:
            s.update_usage(U, r)
        s.run()                                                     # infinite capacity, 1 prefill phase
        # brute force ledger: replay the log, blocks owned during decode step j
        owned = defaultdict(int)
        step_usage = []
        for line in s.log:
            t = line.split()
            if t[0] == "A":
                owned[int(t[1])] += len(t) - 2
            elif t[0] == "F":
                owned.pop(int(t[1]), None)
            elif t[0] == "D":
                step_usage.append(sum(owned.values()))
        alive = lambda j: sum(1 for L, P, N in reqs if j <= N - 1)
        for fp in s.fps:
            want = step_usage[fp - 1] if fp - 1 < len(step_usage) else 0
            assert U[fp] == want, (trial, fp, U[fp], want)
        for j in range(1, len(step_usage) + 1):
            if j in s.fps:
                continue
            prev = max([fp for fp in s.fps if fp < j], default=None)
            if prev is not None:
                assert step_usage[j - 1] - step_usage[prev - 1] <= alive(prev) * ceil_div(stride - 1, B)


# ---------------------------------------------------------- §3.4 work stealing
def _steal_fixture(sizes):
    s = RefScheduler(SchedOptions(n_stages=len(sizes)), [(1, 1, 1)] * sum(sizes))
    s._evict_key = {}
    rid = 0
    for i, n in enumerate(sizes):
        s.slots.append(Slot(i, list(range(rid, rid + n))))
        rid += n
    return s


def test_work_stealing_fig_app2():
    g = GOLD["work_stealing_fig_app2"]
    s = _steal_fixture(g["initial"])
    for st in g["steps"] + g["continuation"]:
        sl = s.slots[st["batch"]]
        before_pool = len(s.pool)
        del sl.members[:st["finished"]]           # the returning batch removes its finished requests
        s.steal_refill(sl)
        assert len(sl.members) == st["submit"], st
        if "withheld" in st:
            assert len(s.pool) - before_pool == st["withheld"], st
        if "refilled" in st:
            assert before_pool - len(s.pool) == st["refilled"], st
        if "average" in st:
            others = sum(len(x.members) for x in s.slots if x is not sl)
            assert (others + st["submit"] + len(s.pool)) // len(s.slots) == st["average"]
    assert [len(x.members) for x in s.slots] == [114] * 4 and not s.pool


def test_work_stealing_conservation_and_convergence():
    """submitted + withheld + finished = returned; with completions
    stopped, max-min <= 1 within W rotations; the pool drains."""
    rng = np.random.default_rng(1)
    for trial in range(2000):
        W = int(rng.integers(2, 9))
        sizes = [int(x) for x in rng.integers(0, 300, size=W)]
        if sum(sizes) == 0:
            continue
        s = _steal_fixture(sizes)
        for rot in range(3):
            for i in range(W):
                sl = s.slots[i]
                fin = int(rng.integers(0, len(sl.members) + 1)) if rot == 0 else 0
                ret = len(sl.members)
                del sl.members[:fin]
                p0 = len(s.pool)
                s.steal_refill(sl)
                assert len(sl.members) + (len(s.pool) - p0) + fin == ret
        sz = [len(x.members) for x in s.slots]
        assert max(sz) - min(sz) <= 1 and not s.pool, (trial, sizes, sz)


# --------------------------------------------------------- §3.5 Eq.1 / Eq.2
def _eq_fixture(bs):
    # toy table Tdec[b] = 2 ms + 10 us * b, three pending prefills of 20 ms, W = 4
    tdec = [0] + [2_000_000 + 10_000 * b for b in range(1, 513)]
    tpre = [0] + [20_000_000] * 2048
    o = SchedOptions(n_stages=4, block_size=1, kv_blocks=10 ** 9, prefill_token_budget=100)
    reqs = [(100, 2, 2)] * 3
    s = RefScheduler(o, reqs + [(1, 1, 1)] * bs, tdec, tpre)
    s._evict_key = {}
    s.pending_fresh = type(s.pending_fresh)([0, 1, 2])
    sl = Slot(0, list(range(3, 3 + bs)))
    return s, sl


@pytest.mark.parametrize("bs,switch,spatial,temporal", [
    (512, False, 1.0, 0.873), (256, True, 0.781, 0.835), (128, True, 0.543, 0.814)])
def test_intensity_rule_toy_table(bs, switch, spatial, temporal):
    s, sl = _eq_fixture(bs)
    assert s.Bp == 512
    # closed forms, Eq.1 / Eq.2
    tdb = 2_000_000 + 10_000 * bs
    sp = (bs / tdb) / (512 / s.tdec[512])
    bub = max(0, 20_000_000 - tdb)
    tot = 3 * 20_000_000 + 4 * tdb + bub
    tp = 1 - bub / tot
    assert abs(sp - spatial) < 1e-3 and abs(tp - temporal) < 1e-3
    assert s.decide_switch(sl) == switch == (sp < tp)


def test_temporal_intensity_spec_value():
    g = GOLD["temporal_intensity"]
    assert 1 - g["bubble"] / g["total"] == g["value"]


def test_strict_inequality_remains_in_decode():
    """spatial == temporal -> remain (PAPER.md:465 'less than')."""
    # bs = Bp -> spatial 1; no bubble (prefill shorter than decode) -> temporal 1
    tdec = [0] + [5_000_000] * 16
    tpre = [0] + [1_000_000] * 64
    s = RefScheduler(SchedOptions(n_stages=2, block_size=1, prefill_token_budget=8), [(4, 2, 2)], tdec, tpre)
    s._evict_key = {}
    sl = Slot(0, list(range(16)))
    assert not s.decide_switch(sl)


# ----------------------------------------------------------- whole-run checks
def _check_run(s, reqs):
    owner = {}
    for line in s.log:
        t = line.split()
        if t[0] == "A":
            for b in map(int, t[2:]):
                assert b not in owner, ("double-owned block", line)
                owner[b] = int(t[1])
        elif t[0] in ("F", "E"):
            for b in map(int, t[2:]):
                assert owner.pop(b) == int(t[1])
    assert not owner
    assert s.alloc.free == s.C
    for r, (L, P, N) in zip(s.reqs, reqs):
        assert r.n_out == N, "token conservation (SPEC.md:480)"
        assert r.done


@pytest.mark.parametrize("policy", [TDPIPE, PPSB_ALT, PPSB_PRIO])
def test_random_runs_invariants(policy):
    tdec, tpre = synthetic_profile(64, 512, knee=8)
    for seed in range(1, 120):
        wl = random_tiny_workload(seed)
        reqs = reqs_of(wl)
        W = 1 + seed % 4
        kvb = 24 if policy == TDPIPE else 24 * W
        o = SchedOptions(n_stages=W, block_size=4, kv_blocks=kvb, prefill_token_budget=64,
                         max_batch_seqs=8, fp_stride=4, fp_horizon=16, policy=policy)
        s = schedule(reqs, o, tdec, tpre)
        _check_run(s, reqs)
        s2 = schedule(reqs, o, tdec, tpre)
        assert s.log == s2.log, "determinism"


def test_infinite_capacity_single_cycle():
    tdec, tpre = synthetic_profile(64, 512)
    for seed in range(1, 40):
        reqs = reqs_of(random_tiny_workload(seed))
        s = schedule(reqs, SchedOptions(n_stages=1 + seed % 4, block_size=4, prefill_token_budget=64), tdec, tpre)
        assert s.stats["p2d"] == 1 and s.stats["d2p"] == 0 and s.stats["evicted"] == 0


def test_c1b_exercises_every_log_kind():
    """C1b: kv_blocks=12, budget 64, max_seqs 8, fp_stride 4 over seeds
    1..50 produce P->D, D->P, evictions, steals and refills."""
    tdec, tpre = synthetic_profile(64, 512, knee=8)
    kinds = defaultdict(int)
    for seed in range(1, 51):
        reqs = reqs_of(random_tiny_workload(seed))
        reqs = [(min(L, 40), P, min(N, 40)) for L, P, N in reqs]
        o = SchedOptions(n_stages=2 + seed % 3, block_size=4, kv_blocks=24, prefill_token_budget=64,
                         max_batch_seqs=8, fp_stride=4, fp_horizon=16)
        s = schedule(reqs, o, tdec, tpre)
        _check_run(s, reqs)
        for line in s.log:
            t = line.split()
            kinds[t[0] if t[0] != "S" else t[0] + t[1]] += 1
    for k in ["P", "G", "A", "F", "D", "R", "SP2D", "SD2P", "E", "W", "U"]:
        assert kinds[k] > 0, (k, dict(kinds))


def test_single_stage_equals_pipeline_outputs():
    """Switch policy / stealing / W do not change what each request generates:
    every run generates exactly N tokens per request and recomputed prompts are
    prompt ++ generated (the scheduler never invents or drops tokens)."""
    tdec, tpre = synthetic_profile(64, 512, knee=8)
    reqs = reqs_of(random_tiny_workload(7))
    outs = []
    for W in (1, 2, 3):
        for steal in (0, 1):
            s = schedule(reqs, SchedOptions(n_stages=W, steal=steal, block_size=4, kv_blocks=20,
                                            prefill_token_budget=64, fp_stride=4), tdec, tpre)
            outs.append([r.n_out for r in s.reqs])
    assert all(o == outs[0] for o in outs)


def test_pphb_invariants():
    """PP+HB [R23]: every prompt is prefilled by contiguous chunks 0..L, each
    micro-batch holds <= hb_tokens tokens (decode tokens count one each), each
    engine stays inside its KV quota, and every request emits exactly its N
    tokens (recompute included)."""
    from oracle.scheduler import PPHB
    for seed in range(60):
        rng = np.random.default_rng(seed)
        n, W, hb = int(rng.integers(1, 14)), int(rng.integers(1, 4)), int(rng.choice([8, 32, 64]))
        reqs = [(int(rng.integers(1, 90)), int(rng.integers(1, 20)), int(rng.integers(1, 25))) for _ in range(n)]
        need = max(ceil_div(L + N, 16) for L, _, N in reqs)
        C = need * W + int(rng.integers(0, need + 1))
        s = schedule(reqs, SchedOptions(n_stages=W, kv_blocks=C, policy=PPHB, hb_tokens=hb))
        assert [r.n_out for r in s.reqs] == [N for _, _, N in reqs]
        quota = [C // W + (1 if e < C % W else 0) for e in range(W)]
        held = {}
        for mb in s.plan:
            assert mb.kind == "H" and sum(mb.q_len) <= hb
            assert all(m % W == mb.slot for m in mb.members)
        for line in s.log:
            f = line.split()
            if f[0] in ("A",):
                held.setdefault(int(f[1]), 0)
                held[int(f[1])] += len(f) - 2
            elif f[0] in ("F", "E"):
                held[int(f[1])] = 0
            per = [0] * W
            for rid, b in held.items():
                per[rid % W] += b
            assert all(per[e] <= quota[e] for e in range(W)), (seed, line)
        # chunks of one admission are contiguous: q_start = previous end
        nxt = {}
        for line in s.log:
            f = line.split()
            if f[0] == "E":
                nxt.pop(int(f[1]), None)
            if f[0] == "H":
                for c in f[5 + int(f[3]):]:
                    rid, q0, ql = map(int, c.split(":"))
                    assert q0 == nxt.get(rid, 0), (seed, line)
                    nxt[rid] = q0 + ql


def test_pphb_tiny_example():
    """Hand-checked: one engine, hb = 8, prompts 10 and 3, outputs 2 and 1.
    mb0 = chunk 0:0:8; mb1 = chunk 0:8:2 (prompt 0 done -> first token) +
    1:0:3 (done, first token = its only token); mb2 = decode of request 0."""
    from oracle.scheduler import PPHB
    s = schedule([(10, 2, 2), (3, 1, 1)], SchedOptions(n_stages=1, kv_blocks=100, policy=PPHB, hb_tokens=8))
    H = [l for l in s.log if l.startswith("H")]
    assert H == ["H 0 0 0 1 0:0:8", "H 1 0 0 2 0:8:2 1:0:3", "H 2 0 1 0 0"], H
