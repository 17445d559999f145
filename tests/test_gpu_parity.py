"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle.

Tolerance (BASELINE.json north_star): per-step logits under teacher forcing
agree within max-abs-rel 2e-2 (F8 row metric); argmax agrees unless the
oracle's top-2 gap is < 4e-2 * max|o|.  Scheduler decisions are bit-exact.
"""
import dataclasses

import numpy as np
import pytest

from oracle import forward as F
from oracle.scheduler import SchedOptions, schedule
from oracle.weights import OracleWeights
from workload import SHAPES, ModelShape, config_workload, generate_workload, random_tiny_workload, \
    synthetic_profile, write_profile_csv

pytestmark = pytest.mark.gpu
TOL = 2e-2

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2506_10470_b200 import TD_BATCH_DECODE, TD_BATCH_PREFILL, TDPipe  # noqa: E402

GQA8 = ModelShape("gqa8", 2, 1024, 8, 1, 2816, 4096, max_seq_len=2048)
GQA4_64 = ModelShape("gqa4_hd64", 2, 512, 8, 2, 1536, 1024, max_seq_len=2048)
LONG = dataclasses.replace(SHAPES["tiny_gqa"], max_seq_len=2048, name="tiny_long")


def _rows_ok(g, o, tol=TOL):
    rel = F.max_abs_rel(g, o)
    assert rel.max() <= tol, f"max-abs-rel {rel.max():.3e} > {tol}"
    return rel


def _argmax_ok(g, o):
    g = np.atleast_2d(g)
    o = np.atleast_2d(o)
    for gi, oi in zip(g, o):
        s = np.sort(oi)
        if s[-1] - s[-2] >= 4e-2 * np.abs(oi).max():
            assert int(np.argmax(gi)) == int(np.argmax(oi))


def _paged(lengths, start=3):
    """Block tables with scattered (non-contiguous, non-monotone) block ids."""
    nb = [(L + 15) // 16 for L in lengths]
    mx = max(nb)
    bt = np.zeros((len(lengths), mx), np.int32)
    nxt = start
    for i, n in enumerate(nb):
        ids = list(range(nxt, nxt + n))[::-1]
        nxt += n + 1
        bt[i, :n] = ids
    return bt


@pytest.mark.parametrize("shape", [SHAPES["tiny"], SHAPES["tiny_gqa"], GQA8, GQA4_64, LONG],
                         ids=lambda s: s.name)
def test_stage_forward_prefill_then_decode(shape):
    """td_stage_forward: a ragged prefill micro-batch, then decode steps into the
    same paged KV, vs the oracle's causal logits at each position."""
    W = OracleWeights(shape)
    t = TDPipe(shape, 1, kv_blocks=512)
    rng = np.random.default_rng(0)
    lengths = [1, 17, 33, 5] if shape.max_seq_len < 2048 else [1, 17, 700, 1100]
    prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
    bt = _paged([L + 4 for L in lengths])
    out = t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * 4, lengths, bt, np.concatenate(prompts))
    seqs = [list(p) for p in prompts]
    for i, p in enumerate(prompts):
        ref = F.sequence_logits(W, p)[-1]
        _rows_ok(out[i], ref)
        _argmax_ok(out[i], ref)
    for step in range(3):
        nxt = [int(np.argmax(o)) for o in out]
        for i in range(4):
            seqs[i].append(nxt[i])
        qs = [len(s) - 1 for s in seqs]
        out = t.td_stage_forward(0, TD_BATCH_DECODE, qs, [1] * 4, bt, np.array(nxt, np.int32))
        for i in range(4):
            ref = F.sequence_logits(W, np.array(seqs[i]))[-1]
            _rows_ok(out[i], ref)
    t.close()


def test_stage_forward_two_stages_residual_handoff():
    """Pipelined == single-stage: stage 0 hands its fp32 residual to stage 1."""
    shape = SHAPES["tiny"].with_layers(4)
    W = OracleWeights(shape)
    t = TDPipe(shape, 2, kv_blocks=256)
    rng = np.random.default_rng(1)
    lengths = [9, 23]
    prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
    bt = _paged(lengths)
    x = t.td_stage_forward(0, TD_BATCH_PREFILL, [0, 0], lengths, bt, np.concatenate(prompts))
    ref_x = np.concatenate([F.forward_hidden(W, p, layers=range(0, 2)) for p in prompts])
    _rows_ok(x, ref_x)
    lg = t.td_stage_forward(1, TD_BATCH_PREFILL, [0, 0], lengths, bt, x)
    for i, p in enumerate(prompts):
        _rows_ok(lg[i], F.sequence_logits(W, p)[-1])
    t.close()


def _tiny_run(shape, wl, n_stages, csv, **opts):
    t = TDPipe(shape, n_stages, record_logits=1, profile_csv=csv, **opts)
    t.submit_workload(wl)
    st = t.td_run()
    toks = [t.td_get_output(i) for i in range(len(wl.requests))]
    logits = [t.td_get_logits(i) for i in range(len(wl.requests))]
    log = t.td_get_log()
    t.close()
    return st, toks, logits, log


def test_td_run_c1_teacher_forced(tmp_path):
    """BASELINE config 0: tiny model, 8 requests prompt 16 / output 16, 2 stages."""
    shape = SHAPES["tiny"]
    wl = config_workload("C1")
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(64, 2048))
    st, toks, logits, log = _tiny_run(shape, wl, 2, csv, kv_blocks=64)
    W = OracleWeights(shape)
    for r, tk, lg in zip(wl.requests, toks, logits):
        assert len(tk) == r.max_new_tokens and lg.shape == (r.max_new_tokens, shape.vocab)
        assert np.array_equal(np.argmax(lg, -1), tk)
        ref = F.teacher_forced_logits(W, r.prompt, tk)
        _rows_ok(lg, ref)
        _argmax_ok(lg, ref)
    # scheduler decisions bit-exact vs the reference scheduler
    reqs = [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]
    ref = schedule(reqs, SchedOptions(n_stages=2, block_size=16, kv_blocks=64), *synthetic_profile(64, 2048))
    assert log == "".join(l + "\n" for l in ref.log)


def test_td_run_batch_invariance(tmp_path):
    """Stealing / W / switching do not change outputs: with batch-invariant
    kernels the generated tokens are bitwise identical (no eviction)."""
    shape = SHAPES["tiny_gqa"]
    wl = random_tiny_workload(5, n_max=12, len_max=40)
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(64, 2048, knee=8))
    outs = []
    for W, steal in [(1, 1), (2, 1), (2, 0)]:
        _, toks, _, _ = _tiny_run(shape.with_layers(2), wl, W, csv, kv_blocks=400, steal=steal)
        outs.append(toks)
    for o in outs[1:]:
        for a, b in zip(outs[0], o):
            assert np.array_equal(a, b)


def test_td_run_evictions_teacher_forced(tmp_path):
    """KV-starved run (C1b-like): P->D, D->P, steals and recompute evictions all
    happen; outputs still match the oracle under teacher forcing and the log is
    bit-exact."""
    shape = SHAPES["tiny_gqa"].with_layers(3)
    csv = str(tmp_path / "p.csv")
    tables = synthetic_profile(64, 2048, knee=8)
    write_profile_csv(csv, *tables)
    W = OracleWeights(shape)
    kinds = set()
    for seed in (3, 8, 13):
        wl = random_tiny_workload(seed, n_max=14, len_max=40)
        need = max((len(r.prompt) + r.max_new_tokens + 15) // 16 for r in wl.requests)
        C = need + 2
        st, toks, logits, log = _tiny_run(shape, wl, 3, csv, kv_blocks=C, prefill_token_budget=64, max_batch_seqs=8,
                                          fp_stride=4, fp_horizon=16)
        reqs = [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]
        ref = schedule(reqs, SchedOptions(n_stages=3, block_size=16, kv_blocks=C, prefill_token_budget=64,
                                          max_batch_seqs=8, fp_stride=4, fp_horizon=16), *tables)
        assert log == "".join(l + "\n" for l in ref.log)
        kinds |= {l.split()[0] for l in ref.log}
        for r, tk, lg in zip(wl.requests, toks, logits):
            assert len(tk) == r.max_new_tokens
            _rows_ok(lg, F.teacher_forced_logits(W, r.prompt, tk))
    assert "E" in kinds


def test_chunked_prefill_over_paged_prefix():
    """Chunked prefill through td_stage_forward: prompts fed in chunks that
    start at q_start > 0 (attending to their paged prefix, causal on absolute
    positions), several sequences with different offsets in one call, MHA and
    GQA, hd 128 and 64.  The last chunk's logits must match the oracle's
    full-prompt logits, and a decode step after it as well."""
    for shape in (ModelShape("mha128c", 1, 512, 4, 4, 512, 512, max_seq_len=1024),
                  ModelShape("gqa64c", 2, 256, 4, 2, 512, 512, max_seq_len=1024)):
        W = OracleWeights(shape)
        t = TDPipe(shape, 1, kv_blocks=256)
        rng = np.random.default_rng(5)
        lengths = [150, 97, 64, 201]
        prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
        bt = _paged([L + 2 for L in lengths])
        cuts = [[0, 64, 128, 150], [0, 30, 97], [0, 64], [0, 1, 100, 163, 201]]   # chunk boundaries
        done = [0] * 4
        last = [None] * 4
        while any(done[i] < len(cuts[i]) - 1 for i in range(4)):
            idx = [i for i in range(4) if done[i] < len(cuts[i]) - 1]
            qs = [cuts[i][done[i]] for i in idx]
            ql = [cuts[i][done[i] + 1] - cuts[i][done[i]] for i in idx]
            toks = np.concatenate([prompts[i][q:q + n] for i, q, n in zip(idx, qs, ql)])
            out = t.td_stage_forward(0, TD_BATCH_PREFILL, qs, ql, bt[idx], toks)
            for j, i in enumerate(idx):
                done[i] += 1
                last[i] = out[j]
        nxt = np.array([np.argmax(l) for l in last], np.int32)
        out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths, [1] * 4, bt, nxt)
        t.close()
        for i, p in enumerate(prompts):
            ref = F.sequence_logits(W, np.concatenate([p, [nxt[i]]]))
            _rows_ok(last[i], ref[-2])
            _rows_ok(out2[i], ref[-1])


def test_td_run_pphb_chunked_prefill_teacher_forced(tmp_path):
    """PP+HB baseline [R23] on the GPU: hybrid micro-batches mixing decode
    tokens and prefill chunks that attend to their paged prefix (small
    hb_tokens so prompts split over several micro-batches, tight KV so
    recompute evictions happen).  Logits teacher-forced vs the oracle, decision
    log bit-exact vs oracle/scheduler.py."""
    from oracle.scheduler import PPHB
    from paper_2506_10470_b200 import TD_POLICY_PPHB
    csv = str(tmp_path / "p.csv")
    tables = synthetic_profile(64, 2048, knee=8)
    write_profile_csv(csv, *tables)
    kinds, n_chunk = set(), 0
    for shape, seed, W, hb in [(SHAPES["tiny_gqa"].with_layers(2), 4, 2, 16), (SHAPES["tiny"], 9, 1, 7),
                               (ModelShape("hd64", 2, 256, 4, 2, 512, 512, max_seq_len=512), 12, 2, 24)]:
        Wt = OracleWeights(shape)
        wl = random_tiny_workload(seed, vocab=shape.vocab, n_max=10, len_max=60)
        need = max((len(r.prompt) + r.max_new_tokens + 15) // 16 for r in wl.requests)
        C = need * W + 2
        st, toks, logits, log = _tiny_run(shape, wl, W, csv, kv_blocks=C, policy=TD_POLICY_PPHB, hb_tokens=hb)
        reqs = [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]
        ref = schedule(reqs, SchedOptions(n_stages=W, block_size=16, kv_blocks=C, policy=PPHB, hb_tokens=hb), *tables)
        assert log == "".join(l + "\n" for l in ref.log)
        kinds |= {l.split()[0] for l in ref.log}
        n_chunk += sum(1 for mb in ref.plan for q0, ql in zip(mb.q_start, mb.q_len) if ql > 1 and q0 > 0)
        for r, tk, lg in zip(wl.requests, toks, logits):
            assert len(tk) == r.max_new_tokens and lg.shape == (r.max_new_tokens, shape.vocab)
            ref_l = F.teacher_forced_logits(Wt, r.prompt, tk)
            _rows_ok(lg, ref_l)
            _argmax_ok(lg, ref_l)
    assert n_chunk > 0 and "H" in kinds


def _prefill_in_budget(t, prompts, bt, budget=2048):
    """Prefill every prompt through td_stage_forward in <= budget-token
    micro-batches (the controller's prefill budget); returns the
    last-position logits of every sequence."""
    outs, i = [], 0
    while i < len(prompts):
        j, tok = i, 0
        while j < len(prompts) and (j == i or tok + len(prompts[j]) <= budget):
            tok += len(prompts[j])
            j += 1
        L = [len(p) for p in prompts[i:j]]
        outs.append(t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * len(L), L, bt[i:j], np.concatenate(prompts[i:j])))
        i = j
    return np.concatenate(outs)


def _check_sequences(W, prompts, nxt, out, out2, idx):
    for i in idx:
        ref = F.sequence_logits(W, np.concatenate([prompts[i], [nxt[i]]]))
        _rows_ok(out[i], ref[-2])
        _argmax_ok(out[i], ref[-2])
        _rows_ok(out2[i], ref[-1])


@pytest.mark.slow
def test_llama7b_shaped_bench_launch_config():
    """Full-size Llama-2-7B layers (d 4096, F 11008, V 32000) at the bench's
    launch configuration: the C2 request set (256 ShareGPT-length prompts,
    seed 2) prefilled in <= 2048-token micro-batches, then ONE decode
    micro-batch of all 256 sequences -- the b > 128 path the bench takes
    (token-major tcgen05 kernel for the wide QKV / gate-up / LM-head GEMMs,
    n >= 129 attention plan, split-K O / down) -- and a second decode step
    (the fused QKV-reduce attention prologue).  2 of the 32 layers
    (the layers share one structure).  Checked against the fp64
    oracle one by one: the 8 shortest, the 8 longest (multi-split attention)
    and 8 random sequences."""
    shape = SHAPES["llama2_7b"].with_layers(2)
    wl = generate_workload(256, shape.vocab, 2)
    prompts = [r.prompt for r in wl.requests]
    lengths = [len(p) for p in prompts]
    t = TDPipe(shape, 1, kv_blocks=8192)
    bt = _paged([L + 3 for L in lengths])
    out = _prefill_in_budget(t, prompts, bt)
    nxt = np.argmax(out, -1).astype(np.int32)
    out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths, [1] * 256, bt, nxt)
    nxt2 = np.argmax(out2, -1).astype(np.int32)
    out3 = t.td_stage_forward(0, TD_BATCH_DECODE, [L + 1 for L in lengths], [1] * 256, bt, nxt2)
    t.close()
    W = OracleWeights(shape)
    order = sorted(range(256), key=lambda i: lengths[i])
    rng = np.random.default_rng(0)
    idx = sorted(set(order[:8] + order[-8:] + list(rng.choice(256, 8, replace=False))))
    _check_sequences(W, prompts, nxt, out, out2, idx)
    for i in order[-4:]:   # the second decode step of the longest sequences
        ref = F.sequence_logits(W, np.concatenate([prompts[i], [nxt[i], nxt2[i]]]))
        _rows_ok(out3[i], ref[-1])


@pytest.mark.slow
@pytest.mark.parametrize("chain", [0, 1], ids=["per_kernel", "decode_chain"])
def test_llama7b_split_k_decode_tolerance(chain):
    """Decode micro-batches of 1, 8 and 40 sequences at Llama-2-7B width, where
    the decode GEMMs split K (8 / 8 / 4 splits on QKV, O, gate-up, down) and
    attention splits the context: every sequence's logits vs the fp64 oracle,
    and the same sequence decoded in different batch compositions agrees
    within the tolerance (split counts change rounding, never the result).
    decode_chain: the same through the persistent decode-layer kernel."""
    shape = SHAPES["llama2_7b"].with_layers(2)
    wl = generate_workload(48, shape.vocab, 21)
    prompts = [r.prompt for r in wl.requests][:40]
    lengths = [len(p) for p in prompts]
    W = OracleWeights(shape)
    res = {}
    for b in (1, 8, 40):
        t = TDPipe(shape, 1, kv_blocks=4096, decode_chain=chain)
        bt = _paged([L + 2 for L in lengths[:b]])
        out = _prefill_in_budget(t, prompts[:b], bt)
        nxt = np.argmax(out, -1).astype(np.int32)
        out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths[:b], [1] * b, bt, nxt)
        t.close()
        res[b] = (nxt, out2)
    refs = {}
    for b, (nxt, out2) in res.items():
        for i in range(b):
            key = (i, int(nxt[i]))
            if key not in refs:
                refs[key] = F.sequence_logits(W, np.concatenate([prompts[i], [nxt[i]]]))[-1]
            _rows_ok(out2[i], refs[key])
    # batch composition: the same sequence decoded among 1 / 8 / 40 sequences
    for i in range(8):
        if res[8][0][i] == res[40][0][i]:
            assert F.max_abs_rel(res[8][1][i], res[40][1][i]).max() <= TOL
    if res[1][0][0] == res[8][0][0]:
        assert F.max_abs_rel(res[1][1][0], res[8][1][0]).max() <= TOL


@pytest.mark.slow
def test_llama70b_shaped_layer_gqa8():
    """C5 shape (Llama-2-70B: d 8192, H 64 / Hkv 8, F 28672, V 32000), one of
    its 80 layers: a <= 2048-token ShareGPT-mix prefill micro-batch and a decode
    step of all its sequences, i.e. the GQA-8 decode-attention kernel and the
    wide decode / prefill GEMMs at full width.  EVERY sequence is checked
    against the fp64 oracle (prefill and decode logits), including the long
    multi-split ones."""
    shape = SHAPES["llama2_70b"].with_layers(1)
    wl = generate_workload(64, shape.vocab, 5)
    lengths, prompts = [], []
    for r in wl.requests:
        if sum(lengths) + len(r.prompt) > 2048:
            break
        lengths.append(len(r.prompt))
        prompts.append(r.prompt)
    t = TDPipe(shape, 1, kv_blocks=2048)
    bt = _paged([L + 2 for L in lengths])
    out = t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * len(lengths), lengths, bt, np.concatenate(prompts))
    nxt = np.argmax(out, -1).astype(np.int32)
    out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths, [1] * len(lengths), bt, nxt)
    t.close()
    assert max(lengths) > 256   # at least one multi-split decode-attention sequence
    _check_sequences(OracleWeights(shape), prompts, nxt, out, out2, range(len(lengths)))


@pytest.mark.slow
def test_llama70b_shaped_layer_gqa8_large_decode_batch():
    """GQA-8 at the C5 stage's decode batch sizes: 128 ShareGPT-length
    sequences (several prefill micro-batches) decoded in ONE micro-batch at
    Llama-2-70B width (tensor-bound decode GEMMs, GQA decode attention over
    many CTAs); sampled sequences (4 shortest, 4 longest, 4 random) vs the fp64
    oracle."""
    shape = SHAPES["llama2_70b"].with_layers(1)
    wl = generate_workload(128, shape.vocab, 55)
    prompts = [r.prompt for r in wl.requests]
    lengths = [len(p) for p in prompts]
    t = TDPipe(shape, 1, kv_blocks=4096)
    bt = _paged([L + 2 for L in lengths])
    out = _prefill_in_budget(t, prompts, bt)
    nxt = np.argmax(out, -1).astype(np.int32)
    out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths, [1] * 128, bt, nxt)
    t.close()
    order = sorted(range(128), key=lambda i: lengths[i])
    rng = np.random.default_rng(1)
    idx = sorted(set(order[:4] + order[-4:] + list(rng.choice(128, 4, replace=False))))
    _check_sequences(OracleWeights(shape), prompts, nxt, out, out2, idx)


def test_device_weights_bit_identical_to_oracle_recipe():
    """F9: the device and the oracle implement the
    counter-based weight recipe independently; every tensor of the tiny model
    (and a GQA variant) read back through td_get_weight (logical layout) must
    equal oracle/weights.py bit for bit -- compared by SHA-256 of the bf16 bits
    and elementwise."""
    import hashlib
    from oracle import weights as Wt
    for shape, stages in ((SHAPES["tiny"], 1), (SHAPES["tiny_gqa"].with_layers(3), 2)):
        W = OracleWeights(shape)
        t = TDPipe(shape, stages, kv_blocks=16)
        L = shape.n_layers
        names = ["g1", "wq", "wk", "wv", "wo", "g2", "wg", "wu", "wd"]
        want = {0: W.embed(), 1 + 9 * L: W.final_norm()[None, :], 2 + 9 * L: W.lm_head()}
        for l in range(L):
            for j, nm in enumerate(names):
                v = W.layer(l)[nm]
                want[1 + 9 * l + j] = v[None, :] if v.ndim == 1 else v
        for tid, ref in want.items():
            ref_bits = (np.ascontiguousarray(ref, np.float32).view(np.uint32) >> 16).astype(np.uint16)
            got = t.td_get_weight(tid)
            assert got.shape == ref_bits.shape, tid
            assert hashlib.sha256(got.tobytes()).hexdigest() == hashlib.sha256(ref_bits.tobytes()).hexdigest(), tid
            assert np.array_equal(got, ref_bits), tid
        t.close()
        assert Wt.tensor_id(0, "lm", L) == 2 + 9 * L


@pytest.mark.slow
def test_mha_tensor_core_decode_large_batch():
    """MHA decode micro-batches of >= 64 sequences at a mean context >= 512
    tokens run on the tensor-core attention kernel (decode_attn_use_tc), with
    the QKV split-K reduction as its own kernel: sampled sequences vs the fp64
    oracle, and the same sequences decoded in an 8-sequence micro-batch (SIMT
    kernel, reduction folded into it) agree within the tolerance."""
    shape = ModelShape("mha128", 1, 512, 4, 4, 512, 512, max_seq_len=4096)
    W = OracleWeights(shape)
    rng = np.random.default_rng(17)
    n = 72
    lengths = [int(v) for v in rng.integers(300, 1200, size=n)]
    assert sum(lengths) >= 512 * n
    prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
    t = TDPipe(shape, 1, kv_blocks=sum((L + 2 + 15) // 16 + 1 for L in lengths) + 8)   # _paged leaves a gap per sequence
    bt = _paged([L + 2 for L in lengths])
    out = _prefill_in_budget(t, prompts, bt)
    nxt = np.argmax(out, -1).astype(np.int32)
    out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths, [1] * n, bt, nxt)
    out_small = t.td_stage_forward(0, TD_BATCH_DECODE, lengths[:8], [1] * 8, bt[:8], nxt[:8])
    t.close()
    order = sorted(range(n), key=lambda i: lengths[i])
    idx = sorted(set(order[:2] + order[-2:] + [int(i) for i in rng.choice(n, 3, replace=False)]))
    for i in idx:
        ref = F.sequence_logits(W, np.concatenate([prompts[i], [nxt[i]]]))
        _rows_ok(out[i], ref[-2])
        _rows_ok(out2[i], ref[-1])
    for i in range(8):
        assert F.max_abs_rel(out2[i], out_small[i]).max() <= TOL


def test_decode_attention_long_context_many_pages():
    """Long contexts (many KV pages per split, every ring slot reused several
    times) for MHA hd=128 and GQA: decode logits vs the oracle."""
    for shape in (ModelShape("mha128", 1, 512, 4, 4, 512, 512, max_seq_len=4096),
                  ModelShape("gqa8_long", 1, 1024, 8, 1, 1024, 512, max_seq_len=4096)):
        W = OracleWeights(shape)
        t = TDPipe(shape, 1, kv_blocks=1024)
        rng = np.random.default_rng(11)
        lengths = [3000, 1500, 37]
        prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
        bt = _paged([L + 2 for L in lengths])
        out = t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * 3, lengths, bt, np.concatenate(prompts))
        nxt = np.argmax(out, -1).astype(np.int32)
        out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths, [1] * 3, bt, nxt)
        t.close()
        for i, p in enumerate(prompts):
            ref = F.sequence_logits(W, np.concatenate([p, [nxt[i]]]))
            _rows_ok(out[i], ref[-2])
            _rows_ok(out2[i], ref[-1])


def test_td_run_speed_of_light_accounting(tmp_path):
    """td_run_stats.alg_bytes / alg_flops / ideal_ns (the whole-job roofline of
    bench.py) equal the closed form for C1: every micro-batch streams all
    weights once (+ the LM head), every context token's K/V per layer is read
    and each new token's K/V written; FLOPs = 2 x tokens x weights + causal
    attention + the LM head rows.  With oracle predictions and 64 blocks there
    is no eviction, so the per-request contexts are 16 (prefill) and 17..31
    (decode steps)."""
    shape = SHAPES["tiny"]
    wl = config_workload("C1")
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(64, 2048))
    t = TDPipe(shape, 2, kv_blocks=64, profile_csv=csv, hbm_peak_gbs=6535.7, tc_peak_tflops=1406.7)
    t.submit_workload(wl)
    st = t.td_run()
    t.close()
    d, H, Hkv, F_, V, nl = shape.d_model, shape.n_heads, shape.n_kv_heads, shape.d_ffn, shape.vocab, shape.n_layers
    hd = d // H
    w_layer = 2.0 * ((H + 2 * Hkv) * hd * d + d * H * hd + 2 * F_ * d + d * F_ + 2 * d)
    head = 2.0 * V * d + 2.0 * d
    kv_tok = 2.0 * Hkv * hd * 2
    n_req = len(wl.requests)
    L, N = 16, 16
    ctx_sum = n_req * (L + sum(L + k for k in range(1, N)))          # prefill ctx + decode contexts
    new_tok = n_req * (L + N - 1)
    att = n_req * (L * (L + 1) / 2 + sum(L + k for k in range(1, N)))
    n_mb = st["n_microbatches"]
    want_bytes = n_mb * (nl * w_layer + head) + nl * kv_tok * (ctx_sum + new_tok)
    want_flops = nl * (new_tok * w_layer + 4.0 * H * hd * att) + 2.0 * n_req * N * V * d
    assert st["n_evicted"] == 0
    assert st["alg_bytes"] == pytest.approx(want_bytes, rel=1e-9)
    assert st["alg_flops"] == pytest.approx(want_flops, rel=1e-9)
    assert 0 < st["ideal_ns"] < st["makespan_ns"]


def test_gqa_small_batch_32_token_splits():
    """GQA-8 decode at a batch too small to occupy the GPU (2 sequences x 1 kv
    head): the launch plan goes down to 32-token splits, up to 8 per sequence,
    merged in split order (kernels.h kAttnMinSplitGQA).  Context lengths hit
    8 full splits, a ragged last split, and a single split."""
    shape = ModelShape("gqa8_small", 1, 1024, 8, 1, 1024, 512, max_seq_len=1024)
    W = OracleWeights(shape)
    t = TDPipe(shape, 1, kv_blocks=256)
    rng = np.random.default_rng(5)
    for lengths in ([255, 200], [31, 250]):
        prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
        bt = _paged([L + 2 for L in lengths])
        out = t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * 2, lengths, bt, np.concatenate(prompts))
        nxt = np.argmax(out, -1).astype(np.int32)
        out2 = t.td_stage_forward(0, TD_BATCH_DECODE, lengths, [1] * 2, bt, nxt)
        for i, p in enumerate(prompts):
            ref = F.sequence_logits(W, np.concatenate([p, [nxt[i]]]))
            _rows_ok(out[i], ref[-2])
            _rows_ok(out2[i], ref[-1])
    t.close()


def test_td_run_trace_and_kv_timeline(tmp_path):
    """A td_run with timing on leaves its CUDA-event spans and the KV-usage
    timeline (PAPER.md:580-585 fig:memory_usage) for td_write_trace: one span
    per (micro-batch, stage) in launch order, non-overlapping on the single
    stream, and the KV blocks held at every launch equal those of td_simulate
    for the same request set -- both come from the same controller decisions
    (the allocation the GPU run performed is the one the controller planned)."""
    import json
    from paper_2506_10470_b200 import TD_EXEC_NULL
    shape = SHAPES["tiny_gqa"].with_layers(2)
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(64, 2048, knee=8))
    wl = random_tiny_workload(8, n_max=14, len_max=40)
    C = max((len(r.prompt) + r.max_new_tokens + 15) // 16 for r in wl.requests) + 3
    opts = dict(kv_blocks=C, profile_csv=csv, prefill_token_budget=64, max_batch_seqs=8, fp_stride=4, fp_horizon=16)
    t = TDPipe(shape, 2, **opts)
    t.submit_workload(wl)
    t.td_set_timing(True)
    st = t.td_run()
    path = str(tmp_path / "run.json")
    t.td_write_trace(path)
    t.close()
    ev = json.load(open(path))["traceEvents"]
    spans = [e for e in ev if e["ph"] == "X"]
    kv = [e["args"]["blocks"] for e in ev if e["ph"] == "C"]
    assert len(spans) == 2 * st["n_microbatches"] and len(kv) == st["n_microbatches"]
    ss = sorted((e["ts"], e["ts"] + e["dur"]) for e in spans)
    assert all(a[1] <= b[0] + 1e-3 for a, b in zip(ss, ss[1:]))     # one stream: stages back to back
    assert max(e["ts"] + e["dur"] for e in spans) <= st["makespan_ns"] / 1e3 + 1e-3
    s = TDPipe(shape, 2, executor=TD_EXEC_NULL, **opts)
    s.submit_workload(wl)
    s.td_simulate(0)
    path2 = str(tmp_path / "sim.json")
    s.td_write_trace(path2)
    s.close()
    kv_sim = [e["args"]["blocks"] for e in json.load(open(path2))["traceEvents"] if e["ph"] == "C"]
    assert kv == kv_sim
    assert max(kv) <= C


@pytest.mark.parametrize("shape", [GQA8, GQA4_64], ids=lambda s: s.name)
def test_decode_chain_stage_forward(shape):
    """The persistent decode-layer kernel (td_options.decode_chain = 1): a
    ragged prefill, then 3 decode steps; logits vs the fp64 oracle, and equal
    within the tolerance to the per-kernel path on the same inputs."""
    W = OracleWeights(shape)
    rng = np.random.default_rng(5)
    lengths = [1, 17, 300, 5, 64]
    prompts = [rng.integers(0, shape.vocab, size=L).astype(np.int32) for L in lengths]
    bt = _paged([L + 4 for L in lengths])
    outs = {}
    for chain in (0, 1):
        t = TDPipe(shape, 1, kv_blocks=512, decode_chain=chain)
        out = t.td_stage_forward(0, TD_BATCH_PREFILL, [0] * 5, lengths, bt, np.concatenate(prompts))
        seqs = [list(p) for p in prompts]
        steps = []
        for step in range(3):
            nxt = [int(np.argmax(o)) for o in out] if chain == 0 else outs[0][step][0]
            for i in range(5):
                seqs[i].append(nxt[i])
            out = t.td_stage_forward(0, TD_BATCH_DECODE, [len(s) - 1 for s in seqs], [1] * 5, bt,
                                     np.array(nxt, np.int32))
            steps.append((nxt, out, [list(s_) for s_ in seqs]))
        t.close()
        outs[chain] = steps
    for (nxt0, out0, seqs0), (nxt1, out1, _) in zip(outs[0], outs[1]):
        for i in range(5):
            ref = F.sequence_logits(W, np.array(seqs0[i]))[-1]
            _rows_ok(out1[i], ref)
            assert F.max_abs_rel(out1[i], out0[i]).max() <= TOL


def test_decode_chain_td_run_teacher_forced(tmp_path):
    """td_run end to end (2 stages, prefill + decode phases) with the decode
    chain: teacher-forced logits vs the oracle, decisions bit-exact."""
    shape = GQA4_64
    wl = generate_workload(12, shape.vocab, 3, uniform_in=(4, 60), uniform_out=(4, 24))
    csv = str(tmp_path / "p.csv")
    write_profile_csv(csv, *synthetic_profile(64, 2048))
    st, toks, logits, log = _tiny_run(shape, wl, 2, csv, kv_blocks=256, decode_chain=1)
    W = OracleWeights(shape)
    for r, tk, lg in zip(wl.requests, toks, logits):
        assert len(tk) == r.max_new_tokens
        _rows_ok(lg, F.teacher_forced_logits(W, r.prompt, tk))
    reqs = [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]
    ref = schedule(reqs, SchedOptions(n_stages=2, block_size=16, kv_blocks=256), *synthetic_profile(64, 2048))
    assert log == "".join(l + "\n" for l in ref.log)
