"""N>1 host logic on CPU (world_size 2, gloo): one process per pipeline stage.

Every rank runs its own replica of the controller; the multi-process pipeline
is deadlock-free and correct only if (a) all replicas take identical decisions,
(b) the implied point-to-point schedule pairs up: stage 0 sends the fp32
residual of every micro-batch to stage 1 in launch order, stage 1 receives the
same sizes in the same order, stage 1 returns (position, token) pairs of every
micro-batch and stage 0 receives them in return order (= launch order, FIFO
stages), and (c) the NCCL ids distributed by rank 0 reach every rank intact.
"""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from workload import SHAPES, random_tiny_workload, synthetic_profile, write_profile_csv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _schedule(log, rank, world, d_model):
    """Per-rank P2P op list implied by the decision log."""
    ops = []
    launches = []
    for line in log.splitlines():
        t = line.split()
        if t[0] in ("P", "D"):
            ids = list(map(int, t[3:] if t[0] == "P" else t[4:]))
            launches.append((int(t[1]), t[0], ids))
        elif t[0] == "R":
            mid = int(t[1])
            n = int(t[2])
            if rank == 0:
                ops.append(("recv_tok", world - 1, 2 * n))
            continue
        else:
            continue
        mid, kind, ids = launches[-1]
        if rank > 0:
            ops.append(("recv_x", rank - 1, ("T", mid)))
        if rank < world - 1:
            ops.append(("send_x", rank + 1, ("T", mid)))
        else:
            ops.append(("send_tok", 0, 2 * len(ids)))
    return ops, launches


def _worker(rank, world, port, csv, seeds, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    sys.path.insert(0, ROOT)
    from paper_2506_10470_b200 import TD_EXEC_NULL, TDPipe, td_nccl_ids
    from paper_2506_10470_b200.tdpipe import make_allgather
    ids = [td_nccl_ids() if rank == 0 else None]
    dist.broadcast_object_list(ids, src=0)
    out = {"ids": ids[0], "logs": []}
    # (d) the td_allgather_fn callback the library calls in peer-store mode
    # (IPC handles, KV-capacity min, profile max): rank order, exact bytes
    import ctypes

    def gather(b):
        parts = [None] * world
        dist.all_gather_object(parts, b)
        return parts
    cb = make_allgather(gather)
    mine = bytes([rank + 1]) * 64 + rank.to_bytes(8, "little")
    send = ctypes.create_string_buffer(mine, len(mine))
    recv = ctypes.create_string_buffer(len(mine) * world)
    out["allgather_rc"] = cb(None, ctypes.cast(send, ctypes.c_void_p), ctypes.cast(recv, ctypes.c_void_p), len(mine))
    out["allgather"] = recv.raw
    for seed in seeds:
        wl = random_tiny_workload(seed, n_max=14, len_max=40)
        t = TDPipe(SHAPES["tiny"].with_layers(4), world, executor=TD_EXEC_NULL, kv_blocks=6, block_size=16,
                   prefill_token_budget=64, max_batch_seqs=8, fp_stride=4, fp_horizon=16, profile_csv=csv,
                   world_size=world, rank=rank)
        t.submit_workload(wl)
        t.td_run()
        out["logs"].append(t.td_get_log())
        t.close()
    gathered = [None] * world
    dist.all_gather_object(gathered, out)
    if rank == 0:
        q.put(gathered)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_replicated_controllers_and_p2p_schedule(tmp_path, world):
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(64, 2048, knee=8))
    seeds = list(range(1, 21))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, csv, seeds, q)) for r in range(world)]
    for p in procs:
        p.start()
    gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # (c) ids intact on every rank
    assert all(g["ids"] == gathered[0]["ids"] and len(g["ids"]) == 256 for g in gathered)
    # (d) allgather callback: every rank receives every rank's bytes in rank order
    want = b"".join(bytes([r + 1]) * 64 + r.to_bytes(8, "little") for r in range(world))
    assert all(g["allgather_rc"] == 0 and g["allgather"] == want for g in gathered)
    evictions = 0
    for i, seed in enumerate(seeds):
        logs = [g["logs"][i] for g in gathered]
        # (a) identical decisions on every rank
        assert all(l == logs[0] for l in logs), seed
        evictions += logs[0].count("\nE ")
        # (b) pairwise-matched P2P schedule
        sch = [_schedule(logs[r], r, world, 64) for r in range(world)]
        for r in range(world - 1):
            sends = [o for o in sch[r][0] if o[0] == "send_x"]
            recvs = [o for o in sch[r + 1][0] if o[0] == "recv_x"]
            assert [o[2] for o in sends] == [o[2] for o in recvs]
        tok_s = [o[2] for o in sch[world - 1][0] if o[0] == "send_tok"]
        tok_r = [o[2] for o in sch[0][0] if o[0] == "recv_tok"]
        assert tok_s == tok_r, seed          # returns arrive in launch order
    assert evictions > 0                     # the starved pool exercised recompute too
