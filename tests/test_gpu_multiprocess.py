"""Multi-process pipeline on ONE GPU: one process per stage, all on cuda:0.

The peer-store hand-off (include/tdpipe.h TD_HANDOFF_PEER) moves the fp32
residual stage s -> s+1 and the sampled tokens last -> stage 0 through CUDA-IPC
mailboxes and stream-ordered sequence flags.  IPC works between processes on
the same device exactly as between NVLink peers, so this exercises the whole
multi-process path (replicated controllers, receive rings, slot-free acks,
token ring, IPC handle exchange through the allgather callback) on the
single-GPU boxes of this round; only the transport differs (local HBM instead
of NVLink).

Checks ("a single point-to-point
communication"):
  * every rank takes the same decisions as the single-process controller
    (decision logs byte-identical);
  * the tokens stage 0 receives equal, bit for bit, the tokens of the
    single-process S-stage run (same kernels, same split choices; the hand-off
    copies fp32 rows exactly);
  * C1: the last stage's logits match the fp64 oracle under teacher forcing
    (2e-2, BASELINE.json north_star).
"""
import os
import socket

import numpy as np
import pytest

from workload import SHAPES, config_workload, random_tiny_workload, synthetic_profile, write_profile_csv

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather(world):
    def g(b):
        out = [None] * world
        dist.all_gather_object(out, b)
        return out
    return g


def _workload(case):
    if case["wl"] == "C1":
        return config_workload("C1")
    return random_tiny_workload(case["seed"], n_max=14, len_max=40)


def _shape(case):
    s = SHAPES["tiny"]
    return s if case["layers"] == s.n_layers else s.with_layers(case["layers"])


def _opts(case, csv):
    return dict(kv_blocks=case["kv_blocks"], profile_csv=csv, prefill_token_budget=case["budget"],
                max_batch_seqs=case.get("max_seqs", 8), hb_tokens=case.get("hb_tokens", 512), fp_stride=4,
                fp_horizon=16, record_logits=case["logits"], device=0)


def _worker(rank, world, port, csv, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_2506_10470_b200 import TDPipe
    try:
        wl = _workload(case)
        t = TDPipe(_shape(case), world, world_size=world, rank=rank, allgather=_gather(world), **_opts(case, csv))
        t.submit_workload(wl)
        st = t.td_run()
        out = {"rank": rank, "log": t.td_get_log(), "tokens": [t.td_get_output(i) for i in range(len(wl.requests))],
               "stats": st}
        if case["logits"] and rank == world - 1:
            out["logits"] = [t.td_get_logits(i) for i in range(len(wl.requests))]
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        t.close()
        if rank == 0:
            q.put(gathered)
    except Exception as e:   # surface the failure to the parent instead of hanging it
        q.put(repr(e))
        raise
    finally:
        dist.destroy_process_group()


def _run_mp(case, csv, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, csv, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert not isinstance(res, str), res
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    return res


CASES = [
    # C1 (BASELINE.json configs[0]): 2 stages, teacher-forced logits vs the oracle
    dict(name="C1_pp2", wl="C1", seed=0, layers=2, world=2, kv_blocks=64, budget=2048, logits=1),
    # KV-starved random runs: evictions / recompute, D->P switches, many
    # micro-batches (wraps the 3-slot residual ring and the 16-slot token ring)
    dict(name="starved_pp2", wl="rand", seed=7, layers=2, world=2, kv_blocks=12, budget=64, logits=0),
    dict(name="starved_pp4", wl="rand", seed=11, layers=4, world=4, kv_blocks=12, budget=64, logits=0),
    # decode groups (n_live / W, + steals) far above max_batch_seqs = 2: the
    # hand-off slots sized at td_create are too small and td_run re-sizes
    # every rank's mailbox before the first launch
    dict(name="big_decode_pp2", wl="rand", seed=9, layers=2, world=2, kv_blocks=400, budget=2048, logits=0,
         max_seqs=2, hb_tokens=0),
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: c["name"])
def test_peer_handoff_pipeline_matches_single_process(case, tmp_path):
    from paper_2506_10470_b200 import TDPipe
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(64, 2048))
    world = case["world"]
    res = _run_mp(case, csv, world)
    # single-process S-stage run of the same job: the reference for decisions and tokens
    wl = _workload(case)
    t = TDPipe(_shape(case), world, **_opts(case, csv))
    t.submit_workload(wl)
    st = t.td_run()
    log = t.td_get_log()
    toks = [t.td_get_output(i) for i in range(len(wl.requests))]
    t.close()
    assert len(res) == world
    for r in res:
        assert r["log"] == log, f"rank {r['rank']}: decision log differs from the single-process controller"
    for i, r in enumerate(wl.requests):
        assert len(res[0]["tokens"][i]) == r.max_new_tokens
        np.testing.assert_array_equal(res[0]["tokens"][i], toks[i], err_msg=f"stage-0 tokens of request {i}")
        np.testing.assert_array_equal(res[-1]["tokens"][i], toks[i], err_msg=f"last-stage tokens of request {i}")
    assert res[0]["stats"]["generated_tokens"] == st["generated_tokens"]
    if case["wl"] == "rand":
        assert st["n_microbatches"] > 16   # the rings wrapped
    if case["logits"]:
        from oracle import forward as F
        from oracle.weights import OracleWeights
        W = OracleWeights(_shape(case))
        for i, r in enumerate(wl.requests):
            ref = F.teacher_forced_logits(W, r.prompt, res[0]["tokens"][i])
            rel = F.max_abs_rel(res[-1]["logits"][i], ref)
            assert rel.max() <= 2e-2, f"request {i}: max-abs-rel {rel.max():.3e}"
