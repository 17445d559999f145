"""Hand-computed pins for the reference scheduler's formation, gating,
eviction and baseline rules, and for the F8 tolerance metric.

Every expected value below was worked out by hand from the cited passage (the
derivation is in each docstring), not produced by running the oracle, so that a
plausible mistake -- a round-robin split instead of a contiguous one, the
smallest admission seq as the victim, ALT and PRIO swapped, a wrong
denominator in max_abs_rel -- fails here even though every invariant test
would still pass.
"""
import numpy as np

from oracle import forward as F
from oracle.scheduler import PPHB, PPSB_ALT, PPSB_PRIO, TDPIPE, RefScheduler, SchedOptions, Slot, schedule
from oracle.weights import OracleWeights
from workload import SHAPES, random_tiny_workload, synthetic_profile


def _sched(reqs, **o):
    s = RefScheduler(SchedOptions(**o), reqs)
    s._evict_key = {}
    return s


# ------------------------------------------------------------------ S5 formation
def test_form_decode_contiguous_split_by_admission_order():
    """S5 / PAPER.md:409 §3.4 "divide the requests into batches equal to the
    number of GPUs, with each batch containing the same number of requests";
    SPEC.md:394 "remainder to earlier batches".

    10 live requests, W = 4: sizes 3, 3, 2, 2, contiguous in ADMISSION order
    (not request id).  Admission seq of request i is (7 i) mod 10, so the
    admission order is rid 0, 3, 6, 9, 2, 5, 8, 1, 4, 7:
        slot 0 = [0, 3, 6], slot 1 = [9, 2, 5], slot 2 = [8, 1], slot 3 = [4, 7].
    (A round-robin split would give [0, 9, 8, 4], ... .)"""
    s = _sched([(4, 4, 4)] * 10, n_stages=4, block_size=4)
    for i in range(10):
        s.reqs[i].adm = (7 * i) % 10
        s.live.add(i)
    s.form_decode()
    assert s.log == ["G 0 3 0 3 6", "G 1 3 9 2 5", "G 2 2 8 1", "G 3 2 4 7"]
    assert [sl.members for sl in s.slots] == [[0, 3, 6], [9, 2, 5], [8, 1], [4, 7]]


def test_form_decode_fewer_requests_than_stages():
    """3 live requests, W = 4: min(W, n) = 3 batches of one request each."""
    s = _sched([(4, 4, 4)] * 3, n_stages=4, block_size=4)
    for i, a in enumerate([2, 0, 1]):
        s.reqs[i].adm = a
        s.live.add(i)
    s.form_decode()
    assert s.log == ["G 0 1 1", "G 1 1 2", "G 2 1 0"]


# ------------------------------------------------------------------ S5 gating
def _gating_fixture():
    s = _sched([(4, 8, 8)] * 4, n_stages=3, block_size=4, kv_blocks=100)
    for i in range(4):
        s.reqs[i].adm = i
        s.live.add(i)
    s.slots = [Slot(0, [0, 1]), Slot(1, [2]), Slot(2, [3])]
    for i, sl in enumerate(s.slots):
        for r in sl.members:
            s.reqs[r].slot = i
    return s


def _launches(log):
    return [l for l in log if l.startswith("D ")]


def test_readiness_gating_waits_for_in_flight_members_and_slot_order():
    """S5: "Slot i launches at the first event after which all its members are
    ready AND slot i-1 has launched" (membership fixed at formation).

    Member 1 of slot 0 is still in flight: nothing launches -- slot 1 (all
    members ready) must NOT overtake slot 0.  Once 1 returns, slots 0, 1, 2
    launch in order as micro-batches 0, 1, 2."""
    s = _gating_fixture()
    s.reqs[1].in_flight = True
    s.try_launch_formed()
    assert _launches(s.log) == []
    s.reqs[1].in_flight = False
    s.try_launch_formed()
    assert _launches(s.log) == ["D 0 0 2 0 1", "D 1 1 1 2", "D 2 2 1 3"]


def test_readiness_gating_stops_at_first_unready_slot():
    """Slot 0 ready, slot 1's member in flight, slot 2 ready: only slot 0
    launches; slot 2 waits behind slot 1."""
    s = _gating_fixture()
    s.reqs[2].in_flight = True
    s.try_launch_formed()
    assert _launches(s.log) == ["D 0 0 2 0 1"]
    s.reqs[2].in_flight = False
    s.try_launch_formed()
    assert _launches(s.log) == ["D 0 0 2 0 1", "D 1 1 1 2", "D 2 2 1 3"]


# ------------------------------------------------------------------ S8 eviction
def test_eviction_victim_is_largest_admission_seq_of_slot_and_pool():
    """S8 / PAPER.md:533 §4.1 "the KV cache of recently arrived requests will be
    freed once memory capacity is saturated" (recompute).

    B = 4, C = 6 blocks.  Requests 0..4 each hold one block (ids 0..4, lowest
    first), L = 4, one token generated (g = 1, d = 0), so the next decode step
    needs ceil((4+0+1)/4) - 1 = 1 new block per member.  Slot members [0, 1, 2]
    (admission 0, 5, 2), pool [3] (admission 7), request 4 (admission 3) is in
    another slot and not a candidate.  Free = 1, need = 3:
      victim 1 = max adm over {0:0, 1:5, 2:2, 3:7} = request 3 (pool) -> free 2
      need 3 > 2 -> victim 2 = request 1 (adm 5)                      -> free 3
      need 2 (members 0, 2) <= 3 -> stop.
    Log "E 3 3", "E 1 1"; the evicted requests re-enter pending at the front in
    (old) admission order [1, 3]; request 1 recomputes prompt ++ generated:
    L = 5, N = 6 - 1 = 5, P = max(9 - 1, 1) = 8, g = d = 0."""
    s = _sched([(4, 9, 6)] * 5, n_stages=2, block_size=4, kv_blocks=6)
    for i, a in enumerate([0, 5, 2, 7, 3]):
        r = s.reqs[i]
        r.adm = a
        r.blocks = s.alloc.alloc(1)
        r.g = 1
        s.live.add(i)
    s.pending_fresh.clear()
    sl = Slot(0, [0, 1, 2])
    s.slots = [sl, Slot(1, [4])]
    s.pool.append(3)
    s.ensure_blocks(sl)
    assert s.log == ["E 3 3", "E 1 1"]
    assert sl.members == [0, 2] and list(s.pool) == []
    assert s.pending_evicted == [1, 3]
    r1 = s.reqs[1]
    assert (r1.L, r1.N, r1.P, r1.g, r1.d, r1.blocks, r1.adm) == (5, 5, 8, 0, 0, [], -1)
    assert s.alloc.free == 3


# ------------------------------------------------------------------ S11 baselines
ALT_PRIO_REQS = [(4, 3, 3), (4, 1, 1), (4, 2, 2), (4, 1, 1)]   # (L, P, N); rid mod 2 = engine


def test_ppsb_prio_two_engine_log():
    """S11 PPSB_PRIO (vLLM-0.5.x-like virtual engines, "PP+SB"):
    an engine issues a prefill whenever one is admissible.  W = 2, B = 4,
    budget 4 (one prompt per prefill), C = 20 (quota 10 per engine), lowest
    free block first.  Hand trace (mb = micro-batch id):
      e0: P mb0 [0] (blk 0)          e1: P mb1 [1] (blk 1)
      R0: e0 prefill [2] now (PRIO)  -> P mb2 [2] (blk 2)
      R1: 1 done (F 1 1); e1 prefill [3] -> P mb3 [3] (blk 1, reused)
      R2: e0 decode [0, 2]: +1 block each (3, 4) -> D mb4
      R3: 3 done (F 3 1); e1 idle
      R4: 2 done (F 2 2 4); e0 decode [0] (no new block) -> D mb5
      R5: 0 done (F 0 0 3)."""
    s = schedule(ALT_PRIO_REQS, SchedOptions(n_stages=2, block_size=4, kv_blocks=20, prefill_token_budget=4,
                                             policy=PPSB_PRIO))
    assert s.log == ["A 0 0", "P 0 1 0", "A 1 1", "P 1 1 1",
                     "R 0 1 0", "A 2 2", "P 2 1 2",
                     "R 1 1 1", "F 1 1", "A 3 1", "P 3 1 3",
                     "R 2 1 2", "A 0 3", "A 2 4", "D 4 0 2 0 2",
                     "R 3 1 3", "F 3 1",
                     "R 4 2 0 2", "F 2 2 4", "D 5 0 1 0",
                     "R 5 1 0", "F 0 0 3"]


def test_ppsb_alt_two_engine_log():
    """S11 PPSB_ALT, "naive phase-interleaved" (PAPER.md:108 fig:pipeline_bubble;
    SPEC.md:488 "alternates one prefill batch then one decode step"): same
    inputs as the PRIO pin, but an engine whose last micro-batch was a prefill
    and that has running requests must decode first.
      e0: P mb0 [0] (blk 0)          e1: P mb1 [1] (blk 1)
      R0: e0 last = P, running [0] -> decode: A 0 2, D mb2 [0]
      R1: 1 done (F 1 1); e1 running empty -> prefill [3] (blk 1): P mb3
      R2: e0 last = D -> prefill [2] (blk 3): P mb4
      R3: 3 done (F 3 1); e1 idle
      R4: e0 pending empty -> decode [0, 2]: r0 needs 0, r2 +1 (blk 1): D mb5
      R5: 0 and 2 done (F 0 0 2, F 2 3 1)."""
    s = schedule(ALT_PRIO_REQS, SchedOptions(n_stages=2, block_size=4, kv_blocks=20, prefill_token_budget=4,
                                             policy=PPSB_ALT))
    assert s.log == ["A 0 0", "P 0 1 0", "A 1 1", "P 1 1 1",
                     "R 0 1 0", "A 0 2", "D 2 0 1 0",
                     "R 1 1 1", "F 1 1", "A 3 1", "P 3 1 3",
                     "R 2 1 0", "A 2 3", "P 4 1 2",
                     "R 3 1 3", "F 3 1",
                     "R 4 1 2", "A 2 1", "D 5 0 2 0 2",
                     "R 5 2 0 2", "F 0 0 2", "F 2 3 1"]


# ------------------------------------------------------------------ F8 metric
def test_max_abs_rel_closed_form():
    """F8: max_i |g_i - o_i| / max(max_i |o_i|, 1e-6), one value per row."""
    o = np.array([[1.0, -4.0, 2.0], [0.5, 0.25, -0.5], [0.0, 0.0, 0.0]])
    g = np.array([[1.0, -4.0, 2.5], [0.5, 0.0, -0.5], [1e-7, 0.0, -3e-7]])
    # row 0: 0.5 / 4 ; row 1: 0.25 / 0.5 ; row 2: 3e-7 / 1e-6 (floor)
    np.testing.assert_allclose(F.max_abs_rel(g, o), [0.125, 0.5, 0.3], rtol=0, atol=1e-15)
    # 1-D input is one row; symmetric scaling leaves it unchanged
    np.testing.assert_allclose(F.max_abs_rel(g[0] * 3, o[0] * 3), [0.125], rtol=0, atol=1e-15)


# ------------------------------------------------------------------ plan executed
def _execute_plan(sched, W, prompts):
    """Run the scheduler's micro-batch plan, in launch order, through the
    forward definition: every member's KV prefix must be exactly its prompt ++
    what it generated so far (prefill / recompute: q_start 0 and q_len = that
    length; decode: q_start = length - 1, the last generated token; PP+HB
    chunks: q_start = tokens prefilled so far), and the member's next token is
    argmax of the logits at position q_start + q_len - 1."""
    known = {i: list(map(int, p)) for i, p in enumerate(prompts)}
    gen = {i: [] for i in known}
    filled = {i: 0 for i in known}       # PP+HB: prompt tokens prefilled by chunks so far
    decoding = {i: False for i in known}
    cache = {}

    def next_token(seq):
        key = tuple(seq)
        if key not in cache:
            cache[key] = int(F.greedy_argmax(F.sequence_logits(W, np.array(seq))[-1]))
        return cache[key]

    for mb in sched.plan:
        for rid, q0, ql in zip(mb.members, mb.q_start, mb.q_len):
            seq = known[rid]
            if mb.kind == "P" or (mb.kind == "H" and q0 == 0):
                decoding[rid] = False             # (re)admission: prefill from position 0
                filled[rid] = 0
            if mb.kind == "D" or (mb.kind == "H" and decoding[rid]):
                assert decoding[rid] and (q0, ql) == (len(seq) - 1, 1), (mb, rid)
            elif mb.kind == "P":
                assert (q0, ql) == (0, len(seq)), (mb, rid)
            else:                                 # PP+HB chunk, continuing the last one
                assert q0 == filled[rid] and q0 + ql <= len(seq), (mb, rid)
                filled[rid] = q0 + ql
                if q0 + ql < len(seq):
                    continue                      # no token until the chunk completing the prompt
            t = next_token(seq)
            seq.append(t)
            gen[rid].append(t)
            decoding[rid] = True
    return gen


def test_every_schedule_generates_the_plain_greedy_decode():
    """What TD-Pipe computes is fixed (§2.1): whatever the
    stage count, stealing, switching, eviction (recompute) or baseline policy,
    executing the scheduler's plan through the forward definition yields each
    request's plain greedy decode, token for token."""
    shape = SHAPES["tiny"]
    W = OracleWeights(shape)
    tdec, tpre = synthetic_profile(64, 512, knee=8)
    wl = random_tiny_workload(4, n_max=6, len_max=14)
    prompts = [r.prompt for r in wl.requests]
    reqs = [(len(r.prompt), r.predicted_len, r.max_new_tokens) for r in wl.requests]
    ref = {i: list(map(int, F.greedy_generate(W, p, r.max_new_tokens)[0])) for i, (p, r) in
           enumerate(zip(prompts, wl.requests))}
    n_evicted = 0
    for policy in (TDPIPE, PPSB_ALT, PPSB_PRIO, PPHB):
        for Wst in (1, 2, 3):
            for steal in (0, 1):
                o = SchedOptions(n_stages=Wst, steal=steal, block_size=4, kv_blocks=12, prefill_token_budget=20,
                                 fp_stride=4, policy=policy, hb_tokens=7)
                if policy != TDPIPE and any(-(-(L + N) // 4) > o.kv_blocks // Wst for L, _, N in reqs):
                    continue
                s = schedule(reqs, o, tdec, tpre)
                n_evicted += s.stats["evicted"]
                assert _execute_plan(s, W, prompts) == ref, (policy, Wst, steal)
    assert n_evicted > 0   # the recompute path was exercised
