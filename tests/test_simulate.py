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
        for pol in (0, 1, 2):
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
