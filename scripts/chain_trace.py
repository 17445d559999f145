"""Per-op timeline of one decode-chain launch (the last full post-attention
layer program) from a TDP_CHAIN_TRACE build: for each op, the median / max over
CTAs of op start / end (epilogue warps), last weight load issued, last MMA
committed and activation-barrier passed, in us from the earliest kernel entry.
Usage (GPU box): TDP_NVCC_DEFINES=-DTDP_CHAIN_TRACE python -m paper_2506_10470_b200.build --force
                 python scripts/chain_trace.py [--n 1 8 32 128]"""
import argparse
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_10470_b200 import TDPipe  # noqa: E402
from paper_2506_10470_b200.tdpipe import lib  # noqa: E402
from workload import SHAPES  # noqa: E402

OPS = ["O+resid", "GU+swiglu", "down+resid", "QKV+rope"]
K = ["start", "end", "w_issued", "mma_done", "x_ready", "entry", "drained", "wait_ok", "reduced"]
SHOW = [0, 4, 2, 3, 6, 7, 8, 1]

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, nargs="+", default=[1, 8, 32, 128])
ap.add_argument("--model", default="llama2_7b")
ap.add_argument("--ctx", type=int, default=600)
a = ap.parse_args()
shape = SHAPES[a.model].with_layers(4)
t = TDPipe(shape, 1, kv_blocks=max(a.n) * ((a.ctx + 31) // 16 + 2) + 64)
fn = lib().td_chain_trace
fn.argtypes = [C.c_void_p]
fn.restype = None
buf = np.zeros(160 * 12 * 9, np.uint64)
for n in a.n:
    us, ideal = t.td_bench_step(1, n, a.ctx, 3)
    fn(buf.ctypes.data)
    tr = buf.reshape(160, 12, 9).astype(np.int64)[:148]
    t0 = tr[:, 0, 5].min()
    print(f"n={n}: step {us:.1f} us (ideal {ideal:.1f}); kernel entry spread {((tr[:, 0, 5] - t0).max()) / 1e3:.2f} us")
    for i, name in enumerate(OPS):
        row = []
        for k in SHOW:
            v = tr[:, i, k]
            v = v[v > 0]
            if len(v) == 0:
                row.append("    -    ")
                continue
            d = (v - t0) / 1e3
            row.append(f"{np.median(d):.1f}/{d.max():.1f}")
        print(f"  {i} {name:10s} " + " ".join(f"{K[k]}={r}" for k, r in zip(SHOW, row)))
    end = tr[:, len(OPS) - 1, 1].max()
    print(f"  total {(end - t0) / 1e3:.1f} us", flush=True)
    buf[:] = 0
t.close()
