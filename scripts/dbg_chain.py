"""Debug: td_stage_forward decode with the decode chain on / off vs the oracle
(per step max-abs-rel), tiny and a 2-layer GQA shape."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import forward as F  # noqa: E402
from oracle.weights import OracleWeights  # noqa: E402
from paper_2506_10470_b200 import TD_BATCH_DECODE, TD_BATCH_PREFILL, TDPipe  # noqa: E402
from workload import SHAPES, ModelShape  # noqa: E402


def paged(lengths, start=3):
    nb = [(L + 15) // 16 for L in lengths]
    bt = np.zeros((len(lengths), max(nb)), np.int32)
    nxt = start
    for i, n in enumerate(nb):
        bt[i, :n] = list(range(nxt, nxt + n))[::-1]
        nxt += n + 1
    return bt


def run(shape, chain, nstages=1, layers_out=False):
    W = OracleWeights(shape)
    t = TDPipe(shape, nstages, kv_blocks=512, decode_chain=chain)
    rng = np.random.default_rng(0)
    lengths = [1, 17, 33, 5]
    prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
    bt = paged([L + 4 for L in lengths])
    out = t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * 4, lengths, bt, np.concatenate(prompts))
    seqs = [list(p) for p in prompts]
    res = [max(float(F.max_abs_rel(out[i], F.sequence_logits(W, p)[-1]).max()) for i, p in enumerate(prompts))]
    for step in range(3):
        nxt = [int(np.argmax(o)) for o in out]
        for i in range(4):
            seqs[i].append(nxt[i])
        qs = [len(s) - 1 for s in seqs]
        out = t.td_stage_forward(0, TD_BATCH_DECODE, qs, [1] * 4, bt, np.array(nxt, np.int32))
        res.append(max(float(F.max_abs_rel(out[i], F.sequence_logits(W, np.array(seqs[i]))[-1]).max())
                       for i in range(4)))
    t.close()
    return res


if __name__ == "__main__":
    for name in ("tiny", "tiny_gqa"):
        for chain in (0, 1):
            print(name, "chain", chain, ["%.3e" % r for r in run(SHAPES[name], chain)], flush=True)
    sh = ModelShape("gqa8", 2, 1024, 8, 1, 2816, 4096, max_seq_len=2048)
    for chain in (0, 1):
        print("gqa8 chain", chain, ["%.3e" % r for r in run(sh, chain)], flush=True)
