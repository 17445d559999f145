"""td_simulate: the timed pipeline replay takes exactly the decisions of td_run
(same decision log) and its timing obeys the pipeline bounds."""
import dataclasses

from paper_2506_10470_b200 import TD_EXEC_NULL, TDPipe
from workload import SHAPES, generate_workload, synthetic_profile, write_profile_csv


def test_simulate_matches_run_and_bounds(tmp_path):
    csv = str(tmp_path / "p.csv")
    tdec, tpre = synthetic_profile(512, 2048, dec_base_ns=3_000_000, dec_per_req_ns=4_000, knee=96)
    write_profile_csv(csv, tdec, tpre)
    wl = generate_workload(200, 256, 7, in_max=500, out_max=400)
    shape = dataclasses.replace(SHAPES["tiny"].with_layers(8), max_seq_len=4096)
    for S in (1, 2, 4):
        for pol in (0, 1, 2, 3):
            kw = dict(executor=TD_EXEC_NULL, kv_blocks=900 * S, profile_csv=csv, policy=pol)
            a = TDPipe(shape, S, **kw)
            a.submit_workload(wl)
            a.td_run()
            b = TDPipe(shape, S, **kw)
            b.submit_workload(wl)
            st = b.td_simulate(20_000)
            assert a.td_get_log() == b.td_get_log()
            assert 0.0 <= st["bubble_frac"] < 1.0
            busy = st["busy_ns"][:S]
            assert st["makespan_ns"] >= max(busy)                 # a stage cannot be busier than the run
            assert st["generated_tokens"] == sum(r.max_new_tokens for r in wl.requests)
            if S == 1:
                assert st["bubble_frac"] < 0.05                   # one stage: only host-return gaps


def test_trace_export(tmp_path):
    """The Chrome trace holds one span per (micro-batch, stage), spans on a stage
    never overlap, and the bubble recomputed from the trace equals td_simulate's."""
    import json
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(512, 2048, dec_base_ns=3_000_000, dec_per_req_ns=4_000, knee=96))
    wl = generate_workload(120, 256, 9, in_max=400, out_max=300)
    shape = dataclasses.replace(SHAPES["tiny"].with_layers(8), max_seq_len=4096)
    t = TDPipe(shape, 4, executor=TD_EXEC_NULL, kv_blocks=1200, profile_csv=csv)
    t.submit_workload(wl)
    st = t.td_simulate(20_000)
    path = str(tmp_path / "trace.json")
    t.td_write_trace(path)
    ev = json.load(open(path))["traceEvents"]
    spans = [e for e in ev if e["ph"] == "X"]
    kv = [e for e in ev if e["ph"] == "C"]
    assert len(spans) == 4 * st["n_microbatches"] and len(kv) == st["n_microbatches"]
    busy = 0.0
    for s in range(4):
        ss = sorted((e["ts"], e["ts"] + e["dur"]) for e in spans if e["tid"] == s)
        assert all(a[1] <= b[0] + 1e-6 for a, b in zip(ss, ss[1:]))
        busy += sum(b - a for a, b in ss)
    bubble = 1 - busy / (4 * st["makespan_ns"] / 1e3)
    assert abs(bubble - st["bubble_frac"]) < 1e-3
    assert max(e["args"]["blocks"] for e in kv) <= 1200


def test_simulate_pphb_cost_model(tmp_path):
    """PP+HB micro-batches in the timed replay [R23]: every H micro-batch costs
    max(P(T), D(1)) + D(n_dec) - D(1) on every stage (read back from the trace),
    so with one stage and no host gap the makespan is the sum of those costs."""
    import json
    from oracle.scheduler import PPHB, SchedOptions, schedule
    csv = str(tmp_path / "p.csv")
    tdec, tpre = synthetic_profile(512, 2048, dec_base_ns=3_000_000, dec_per_req_ns=4_000, knee=96)
    write_profile_csv(csv, tdec, tpre)
    wl = generate_workload(60, 256, 11, in_max=300, out_max=200)
    shape = dataclasses.replace(SHAPES["tiny"].with_layers(4), max_seq_len=4096)
    t = TDPipe(shape, 1, executor=TD_EXEC_NULL, kv_blocks=2000, profile_csv=csv, policy=3, hb_tokens=256)
    t.submit_workload(wl)
    st = t.td_simulate(0)
    path = str(tmp_path / "trace.json")
    t.td_write_trace(path)
    spans = [e for e in json.load(open(path))["traceEvents"] if e["ph"] == "X"]
    ref = schedule([(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests],
                   SchedOptions(n_stages=1, kv_blocks=2000, policy=PPHB, hb_tokens=256))
    L = {}
    want = []
    for mb in ref.plan:
        # decode members lead: q_start >= current prompt length (no evictions here)
        nd = sum(1 for rid, q0 in zip(mb.members, mb.q_start) if q0 >= len(wl.requests[rid].prompt))
        T = sum(mb.q_len)
        cost = max(tpre[min(T, 2048)], tdec[1]) + (tdec[nd] - tdec[1] if nd else 0)
        want.append(cost)
    assert ref.stats["evicted"] == 0
    got = [round(e["dur"] * 1e3) for e in sorted(spans, key=lambda e: e["ts"])]
    assert got == want
    assert st["makespan_ns"] == sum(want)
