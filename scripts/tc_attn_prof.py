"""Where the GQA-8 tensor-core decode attention's warps spend their cycles
(TDP_TC_PROF build): per wait site, the summed cycles of lane 0 of every warp,
as a fraction of that role's total, for n = 512 at short and long contexts.
Usage (GPU box): TDP_NVCC_DEFINES=-DTDP_TC_PROF python -m paper_2506_10470_b200.build --force
                 python scripts/tc_attn_prof.py"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200.tdpipe import lib, td_bench_attn  # noqa: E402

fn = lib().td_tc_prof
fn.argtypes = [C.c_void_p, C.c_int32]
fn.restype = None
buf = np.zeros(16, np.uint64)
NAMES = ["prod.wait_iempty", "prod.wait_ring_slot", "qprep.wait_ifull", "merger.wait_ifull", "merger.wait_oready",
         "cons.wait_qready", "cons.wait_page", "cons.wait_ofree", None, None, None, None,
         "prod.page_issue", "prod.rotate", "merger.combine", "merger.store"]
for n, ctx in ((512, 256), (512, 1024), (64, 314), (256, 314), (512, 128)):
    c = np.full(n, ctx, np.int32)
    td_bench_attn(c, 64, 8, 128, iters=2)
    fn(buf.ctypes.data, 1)
    us = td_bench_attn(c, 64, 8, 128, iters=10)
    fn(buf.ctypes.data, 1)
    tot = {"cons": buf[8], "prod": buf[9], "qprep": buf[10], "merger": buf[11]}
    row = {"n": n, "ctx": ctx, "us": round(us, 2),
           "frac": round(float(c.sum()) * 8 * 128 * 4 / (us * 1e-6) / 1e9 / 6551.7, 3)}
    for i, k in enumerate(NAMES):
        if k is None:
            continue
        role = k.split(".")[0]
        row[k] = round(float(buf[i]) / max(float(tot[role]), 1.0), 3)
    print(json.dumps(row), flush=True)
