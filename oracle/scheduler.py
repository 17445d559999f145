"""Reference scheduler -- TEST INFRASTRUCTURE ONLY.

The TD-Pipe control plane, step by step in the paper's order and notation:

* Alg.1 "Prefill-to-Decode Switch Algorithm" (§3.3):
  CheckSwitch / UpdateUsage / SchedulePrefill, futurePoints,
* inter-batch work stealing with a sliding window of W batch sizes
  (§3.4),
* spatial-temporal intensity comparison, Eq.1 / Eq.2 and the rule
  "switches to the prefill phase when the spatial intensity is less than the
  temporal intensity" (§3.5),
* recompute on KV overflow, "KV cache of recently arrived requests will be
  freed" (§4.1),
* the naive PP+SB baselines (PAPER.md:108 fig:pipeline_bubble; 530 §4.1),
* the PP+HB baseline: hybrid batching with chunked prefill (PAPER.md:125-128
  §1, 255-260 §2.3, 531 §4.1) [R23].

Logical time only: the only external events are micro-batch returns, which
arrive in launch order because every stage is FIFO, so
the whole decision sequence is a function of the request set, the options and
the frozen profile table -- no wall clock.

Readings where the paper is silent/ambiguous are DESIGN.md "Readings" R1-R20
(= SURVEY.md §8(c) ambiguity table); the ones this file implements are cited
inline as [R#].  The decision log (S12) is the parity artefact: the C++
controller must reproduce it byte for byte.
"""
from __future__ import annotations

import heapq
from collections import deque
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

TDPIPE, PPSB_PRIO, PPSB_ALT, PPHB = 0, 1, 2, 3


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


@dataclass
class SchedOptions:
    n_stages: int = 1             # W = number of GPUs
    block_size: int = 16          # B
    kv_blocks: int = 1 << 30      # C (capacity in blocks, min over stages)
    prefill_token_budget: int = 2048   # SPEC.md:391 [R5]
    max_batch_seqs: int = 1 << 30
    fp_stride: int = 32           # PAPER.md:385 "32nd, 64th, 96th, ..." [R3]
    fp_horizon: int = 1024        # PAPER.md:385 "... 992nd, 1024th"
    policy: int = TDPIPE
    steal: int = 1
    alg1_check_before_launch: int = 0   # [R11b] verbatim = 0 (launch precedes check)
    eq2_bubble_scale: int = 1           # sigma [R12b]; 1 = verbatim Eq.2
    # ablations (§4.4.1, 660-662 §4.4.3); 0 = the paper's method
    p2d_kv_permille: int = 0            # switch to decode once allocated KV >= ratio * C
    d2p_finish_permille: int = 0        # switch to prefill once this fraction of the decode cohort finished
    hb_tokens: int = 512                # PP+HB: tokens per hybrid micro-batch (decode tokens + prefill chunks) [R23]


@dataclass
class Req:
    rid: int
    n_prompt: int
    L: int          # current prompt length incl. recomputed tokens (S1)
    P: int          # predicted output length
    N: int          # remaining stop length (tokens to generate from this admission)
    g: int = 0      # tokens generated since (re)admission
    d: int = 0      # decode steps returned since (re)admission
    adm: int = -1   # admission sequence number
    n_out: int = 0  # tokens generated in total
    blocks: List[int] = field(default_factory=list)
    in_flight: bool = False
    done: bool = False
    slot: int = -1  # current-formation slot or -1 (pool / none)
    pf: int = 0     # PP+HB: prompt tokens prefilled so far (chunked prefill)


@dataclass
class MicroBatch:
    mid: int
    kind: str                 # 'P', 'D' or 'H' (hybrid: decode members first, then prefill chunks)
    members: List[int]
    q_start: List[int]
    q_len: List[int]
    slot: int = -1
    epoch: int = 0


class Allocator:
    """Paged KV block allocator: lowest free ids first (S0)."""

    def __init__(self, n: int):
        self.n = n
        self.free_heap = []      # released ids (all < watermark)
        self.watermark = 0       # ids >= watermark never handed out yet

    @property
    def free(self) -> int:
        return self.n - self.watermark + len(self.free_heap)

    def alloc(self, k: int) -> List[int]:
        assert k <= self.free
        out = []
        for _ in range(k):
            if self.free_heap:
                out.append(heapq.heappop(self.free_heap))
            else:
                out.append(self.watermark)
                self.watermark += 1
        return out

    def release(self, blocks: List[int]) -> None:
        for b in blocks:
            heapq.heappush(self.free_heap, b)


class Slot:
    def __init__(self, idx: int, members: List[int]):
        self.idx = idx
        self.members = list(members)
        self.launched = False     # has launched at least once in this formation
        self.inflight = False
        self.retired = False

    @property
    def active(self) -> bool:
        return not self.retired


class RefScheduler:
    """Reference control plane.  Use: s = RefScheduler(opts, reqs, tdec, tpre); s.run()."""

    def __init__(self, opts: SchedOptions, requests, tdec=None, tpre=None):
        self.o = opts
        self.W = opts.n_stages
        self.B = opts.block_size
        self.C = opts.kv_blocks
        self.reqs: List[Req] = []
        for i, (L, P, N) in enumerate(requests):
            self.reqs.append(Req(i, L, L, max(int(P), 1), N))     # P<1 -> 1
        self.tdec = None if tdec is None else [int(v) for v in tdec]
        self.tpre = None if tpre is None else [int(v) for v in tpre]
        self.log: List[str] = []
        self.plan: List[MicroBatch] = []
        self.alloc = Allocator(self.C)
        self.pending_evicted: List[int] = []   # sorted by old admission seq [R8-eviction]
        self.pending_fresh = deque(range(len(self.reqs)))   # submission order
        self.live = set()
        self.inflight = deque()
        self.slots: List[Slot] = []
        self.pool = deque()
        self.epoch = 0
        self.adm_counter = 0
        self.mb_counter = 0
        self.stats = dict(p2d=0, d2p=0, stolen=0, evicted=0, refilled=0)
        self.cohort_n = 0          # requests of the current decode phase (ablation A23)
        self.cohort_done = 0
        n = len(self.reqs)
        # futurePoints: s, 2s, ..., H, H >= every remaining length [R3]
        s = opts.fp_stride
        maxP = max([r.P for r in self.reqs], default=1)
        H = max(opts.fp_horizon, s * ceil_div(maxP, s))
        self.fps = list(range(s, H + 1, s))
        # ctx_rep, b_mem and Peak, once, in integers (S9) [R11]
        if n:
            self.ctx_rep = max(1, sum(r.L for r in self.reqs) // n + (sum(r.P for r in self.reqs) // n) // 2)
        else:
            self.ctx_rep = 1
        self.b_mem = max(1, (self.C * self.B) // (self.W * self.ctx_rep))
        self.Bp = None
        if self.tdec is not None:
            bmax = len(self.tdec) - 1
            best = 1
            for b in range(1, min(self.b_mem, bmax) + 1):
                # b/T[b] >= best/T[best]  (ties -> largest b)
                if b * self.tdec[best] >= best * self.tdec[b]:
                    best = b
            self.Bp = best

    # ------------------------------------------------------------------ utils
    def emit(self, *parts) -> None:
        self.log.append(" ".join(str(p) for p in parts))

    def pending_empty(self) -> bool:
        return not self.pending_evicted and not self.pending_fresh

    def pending_list(self) -> List[int]:
        return list(self.pending_evicted) + list(self.pending_fresh)

    def _tdec(self, b: int) -> int:
        return self.tdec[min(max(b, 1), len(self.tdec) - 1)]

    def _tpre(self, k: int) -> int:
        return self.tpre[min(max(k, 1), len(self.tpre) - 1)]

    # ------------------------------------------------------------- Alg.1 (S2, S3)
    def update_usage(self, U: dict, r: Req) -> None:
        """UpdateUsage, block form [R1, R2]:
        for futurePoint <= predictLen: kvUsage[futurePoint] += blocks(inputLen + futurePoint),
        predictLen := remaining predicted decode steps max(P-1-d, 0), inputLen := L+d."""
        rem = max(r.P - 1 - r.d, 0)
        for fp in self.fps:
            if fp <= rem:
                U[fp] += ceil_div(r.L + r.d + fp, self.B)

    def rebuild_usage(self) -> dict:
        """kvUsage rebuilt from live requests at each prefill phase [R4]."""
        U = {fp: 0 for fp in self.fps}
        for rid in sorted(self.live, key=lambda i: self.reqs[i].adm):
            self.update_usage(U, self.reqs[rid])
        return U

    @staticmethod
    def check_switch(U: dict, C: int) -> bool:
        """CheckSwitch: switch to decode iff maxUsage > kvCapacity."""
        max_usage = 0
        for usage in U.values():
            if usage > max_usage:
                max_usage = usage
        return max_usage > C

    # ------------------------------------------------------------ S4 prefill
    def _form_prefill_batch(self, pending: List[int], free: int, quota_free: Optional[int] = None):
        """getPrefillBatch [R5]: FIFO greedy under the token budget,
        max_seqs, and the now-free guard ceil(L/B) <= free blocks."""
        batch, tok, need = [], 0, 0
        limit = free if quota_free is None else quota_free
        for rid in pending:
            r = self.reqs[rid]
            if batch and tok + r.L > self.o.prefill_token_budget:
                break
            if len(batch) >= self.o.max_batch_seqs:
                break
            nb = ceil_div(r.L, self.B)
            if need + nb > limit:
                break
            batch.append(rid)
            tok += r.L
            need += nb
            if tok >= self.o.prefill_token_budget:
                break
        return batch

    def _pop_pending(self, batch: List[int]) -> None:
        for rid in batch:
            if self.pending_evicted and self.pending_evicted[0] == rid:
                self.pending_evicted.pop(0)
            else:
                assert self.pending_fresh[0] == rid
                self.pending_fresh.popleft()

    def _usage_delta(self, batch: List[int]) -> dict:
        U = {fp: 0 for fp in self.fps}
        for rid in batch:
            r = self.reqs[rid]
            rem = max(r.P - 1, 0)
            for fp in self.fps:
                if fp <= rem:
                    U[fp] += ceil_div(r.L + fp, self.B)
        return U

    def prefill_phase(self) -> None:
        """SchedulePrefill loop, eager at one logical instant (S4)."""
        U = self.rebuild_usage()
        launched = 0
        while True:
            if self.pending_empty():
                reason = "queue_empty"
                break
            batch = self._form_prefill_batch(self.pending_list(), self.alloc.free)
            if not batch:
                reason = "now_full"
                break
            if self.o.alg1_check_before_launch and (launched > 0 or self.live):
                delta = self._usage_delta(batch)
                if self.check_switch({fp: U[fp] + delta[fp] for fp in self.fps}, self.C):
                    reason = "forecast_pre"
                    break
            self._pop_pending(batch)
            self.launch_prefill(batch)           # batch = getPrefillBatch().Launch()
            launched += 1
            for rid in batch:                    # foreach request: UpdateUsage
                self.update_usage(U, self.reqs[rid])
            if self.o.p2d_kv_permille:
                # ablation: "switch to decode once <ratio> of the KV cache blocks are occupied"
                if (self.C - self.alloc.free) * 1000 >= self.o.p2d_kv_permille * self.C:
                    reason = "kv_ratio"
                    break
            elif self.check_switch(U, self.C):   # CheckSwitch
                reason = "forecast"
                break
        self.stats["p2d"] += 1
        self.emit("S", "P2D", reason, max(U.values()) if U else 0, self.C)

    def dry_run_prefill(self) -> List[int]:
        """S10 step 1: token counts of the prefill batches S4 would launch now."""
        U = self.rebuild_usage()
        pending = self.pending_list()
        free = self.alloc.free
        ks = []
        launched = 0
        while pending:
            batch = self._form_prefill_batch(pending, free)
            if not batch:
                break
            if self.o.alg1_check_before_launch and (launched > 0 or self.live):
                delta = self._usage_delta(batch)
                if self.check_switch({fp: U[fp] + delta[fp] for fp in self.fps}, self.C):
                    break
            pending = pending[len(batch):]
            free -= sum(ceil_div(self.reqs[i].L, self.B) for i in batch)
            ks.append(sum(self.reqs[i].L for i in batch))
            launched += 1
            for rid in batch:
                r = self.reqs[rid]
                rem = max(r.P - 1, 0)
                for fp in self.fps:
                    if fp <= rem:
                        U[fp] += ceil_div(r.L + fp, self.B)
            if self.o.p2d_kv_permille:
                if (self.C - free) * 1000 >= self.o.p2d_kv_permille * self.C:
                    break
            elif self.check_switch(U, self.C):
                break
        return ks

    def launch_prefill(self, batch: List[int], slot: int = -1) -> None:
        for rid in batch:
            r = self.reqs[rid]
            blk = self.alloc.alloc(ceil_div(r.L, self.B))
            r.blocks.extend(blk)
            self.emit("A", rid, *blk)
        mid = self.mb_counter
        self.mb_counter += 1
        for rid in batch:
            r = self.reqs[rid]
            r.adm = self.adm_counter
            self.adm_counter += 1
            r.in_flight = True
            r.g = 0
            r.d = 0
            self.live.add(rid)
        mb = MicroBatch(mid, "P", list(batch), [0] * len(batch),
                        [self.reqs[i].L for i in batch], slot, self.epoch)
        self.inflight.append(mb)
        self.plan.append(mb)
        self.emit("P", mid, len(batch), *batch)

    # ------------------------------------------------------------ S5 formation
    def form_decode(self) -> None:
        """Decode phase entry: live requests by admission order -> W contiguous
        batches, remainder to earlier ones."""
        self.epoch += 1
        self.pool.clear()
        members = sorted(self.live, key=lambda i: self.reqs[i].adm)
        self.cohort_n = len(members)
        self.cohort_done = 0
        for r in self.reqs:
            r.slot = -1
        self.slots = []
        n = len(members)
        if n == 0:
            return
        Wf = min(self.W, n)
        q, rm = divmod(n, Wf)
        idx = 0
        for i in range(Wf):
            sz = q + (1 if i < rm else 0)
            sl = Slot(i, members[idx: idx + sz])
            idx += sz
            for rid in sl.members:
                self.reqs[rid].slot = i
            self.slots.append(sl)
            self.emit("G", i, sz, *sl.members)

    def try_launch_formed(self) -> None:
        """S5: slot i launches once its members are ready and slot i-1 launched."""
        for sl in self.slots:
            if sl.retired or sl.launched:
                continue
            if any(self.reqs[r].in_flight for r in sl.members):
                break
            self.launch_decode(sl)
            if not (sl.retired or sl.launched):
                break

    # ------------------------------------------------------------ S8 eviction
    def evict(self, rid: int) -> None:
        """Recompute on overflow: free KV, prompt := prompt ++ generated."""
        r = self.reqs[rid]
        self.alloc.release(r.blocks)
        self.emit("E", rid, *r.blocks)
        r.blocks = []
        r.L = r.L + r.g
        r.N = r.N - r.g
        r.P = max(r.P - r.g, 1)
        r.g = 0
        r.d = 0
        self.live.discard(rid)
        old = r.adm
        r.adm = -1
        r.slot = -1
        # pending front, evicted kept in (old) admission order [R16]
        keys = [self._evict_key[i] for i in self.pending_evicted]
        self._evict_key[rid] = old
        pos = 0
        while pos < len(keys) and keys[pos] < old:
            pos += 1
        self.pending_evicted.insert(pos, rid)
        self.stats["evicted"] += 1

    _evict_key: dict = None

    def decode_need(self, members: List[int]) -> int:
        need = 0
        for rid in members:
            r = self.reqs[rid]
            need += max(0, ceil_div(r.L + r.d + 1, self.B) - len(r.blocks))
        return need

    def ensure_blocks(self, sl: Slot) -> None:
        """S8: while the step's blocks exceed free blocks, evict the largest
        admission seq among this slot's members and the withheld pool."""
        while sl.members and self.decode_need(sl.members) > self.alloc.free:
            cands = list(sl.members) + list(self.pool)
            victim = max(cands, key=lambda i: self.reqs[i].adm)
            if victim in sl.members:
                sl.members.remove(victim)
            else:
                self.pool.remove(victim)
            self.evict(victim)

    def launch_decode(self, sl: Slot) -> None:
        self.ensure_blocks(sl)
        if not sl.members:
            self.retire(sl)
            return
        for rid in sl.members:
            r = self.reqs[rid]
            k = ceil_div(r.L + r.d + 1, self.B) - len(r.blocks)
            if k > 0:
                blk = self.alloc.alloc(k)
                r.blocks.extend(blk)
                self.emit("A", rid, *blk)
        mid = self.mb_counter
        self.mb_counter += 1
        q0 = [self.reqs[i].L + self.reqs[i].d for i in sl.members]
        mb = MicroBatch(mid, "D", list(sl.members), q0, [1] * len(sl.members), sl.idx, self.epoch)
        for rid in sl.members:
            self.reqs[rid].in_flight = True
        sl.launched = True
        sl.inflight = True
        self.inflight.append(mb)
        self.plan.append(mb)
        self.emit("D", mid, sl.idx, len(sl.members), *sl.members)

    def retire(self, sl: Slot) -> None:
        if not sl.retired:
            sl.retired = True
            self.emit("X", sl.idx)

    # ------------------------------------------------------------ S7 stealing
    def steal_refill(self, sl: Slot) -> None:
        """Inter-batch work stealing with the pool counted [R7]:
        average over the sliding window of the last W batch sizes, deducting the
        finished requests; withhold the excess, refill from withheld requests."""
        others = [s for s in self.slots if s is not sl and s.active]
        rem = len(sl.members)
        n_live = sum(len(s.members) for s in others) + rem + len(self.pool)
        Wa = len(others) + 1
        q, s_ = divmod(n_live, Wa)
        A = sum(1 for s in others if len(s.members) > q)
        target = q + (1 if A < s_ else 0)
        if rem > target:
            k = rem - target
            moved = sl.members[-k:]
            del sl.members[-k:]
            for rid in moved:
                self.reqs[rid].slot = -1
                self.pool.append(rid)
            self.stats["stolen"] += k
            self.emit("W", sl.idx, *moved)
        elif rem < target and self.pool:
            k = min(target - rem, len(self.pool))
            moved = [self.pool.popleft() for _ in range(k)]
            for rid in moved:
                self.reqs[rid].slot = sl.idx
            sl.members.extend(moved)
            self.stats["refilled"] += k
            self.emit("U", sl.idx, *moved)

    # ---------------------------------------------------------- S9 / S10 rule
    def decide_switch(self, sl: Slot) -> bool:
        """Eq.1 spatial = Achieved/Peak; Eq.2 temporal = 1 - bubble/total;
        switch iff spatial < temporal, exact integers [R10-R14]."""
        ks = self.dry_run_prefill()
        if not ks:
            return False
        if self.o.d2p_finish_permille:
            # ablation: switch "once <ratio> of the requests have completed"
            if self.cohort_done * 1000 >= self.o.d2p_finish_permille * self.cohort_n:
                self.emit("S", "D2P", "finish_ratio", self.cohort_done, self.cohort_n)
                return True
            return False
        bs = len(sl.members)
        tpre = [self._tpre(k) for k in ks]
        if bs == 0:
            self.emit("S", "D2P", 0, 0, self._tdec(self.Bp), self.Bp, 0, sum(tpre))
            return True
        tdb = self._tdec(bs)
        tdp = self._tdec(self.Bp)
        bubble = self.o.eq2_bubble_scale * max(0, max(tpre) - tdb)   # longest prefill - current decode
        total = sum(tpre) + self.W * tdb + bubble                   # pending prefills + one step/batch + bubble
        # (bs/tdb)/(Bp/tdp) < (total-bubble)/total
        if bs * tdp * total < self.Bp * tdb * (total - bubble):
            self.emit("S", "D2P", bs, tdb, tdp, self.Bp, bubble, total)
            return True
        return False

    # ------------------------------------------------------------ S6 returns
    def finish(self, r: Req) -> None:
        r.done = True
        self.cohort_done += 1
        self.alloc.release(r.blocks)
        self.emit("F", r.rid, *r.blocks)
        r.blocks = []
        self.live.discard(r.rid)
        if r.rid in self.pool:
            self.pool.remove(r.rid)
        if r.slot >= 0 and r.slot < len(self.slots):
            sl = self.slots[r.slot]
            if r.rid in sl.members:
                sl.members.remove(r.rid)
        r.slot = -1

    def on_return(self, mb: MicroBatch) -> None:
        self.emit("R", mb.mid, len(mb.members), *mb.members)
        for rid in mb.members:
            r = self.reqs[rid]
            r.in_flight = False
            r.g += 1
            r.n_out += 1
            if mb.kind == "D":
                r.d += 1
            if r.g == r.N:
                self.finish(r)
        current = mb.kind == "D" and mb.epoch == self.epoch
        if not current:
            # prefill or superseded decode: members already sit in the new formation
            for sl in self.slots:
                if sl.active and not sl.launched and not sl.members:
                    self.retire(sl)
            return
        sl = self.slots[mb.slot]
        sl.inflight = False
        if self.o.steal and self.W > 1:
            self.steal_refill(sl)
        if not self.pending_empty() and self.decide_switch(sl):
            self.stats["d2p"] += 1
            self.prefill_phase()
            self.form_decode()
            return
        if not sl.members:
            self.retire(sl)
            return
        self.launch_decode(sl)

    # ------------------------------------------------------------ main loop
    def run(self):
        self._evict_key = {}
        if self.o.policy == PPHB:
            return self._run_hybrid()
        if self.o.policy != TDPIPE:
            return self._run_baseline()
        if not self.reqs:
            return self
        self.prefill_phase()
        self.form_decode()
        self.try_launch_formed()
        while self.inflight:
            mb = self.inflight.popleft()
            self.on_return(mb)
            self.try_launch_formed()
            if not any(s.active for s in self.slots) and (not self.pending_empty() or self.live):
                self.emit("S", "D2P", "idle")
                self.stats["d2p"] += 1
                self.prefill_phase()
                self.form_decode()
                self.try_launch_formed()
        assert self.pending_empty() and not self.live, "scheduler stalled"
        return self

    # ------------------------------------------------------------ S11 baselines
    def _run_baseline(self):
        """Naive phase-interleaved PP+SB (S11): W virtual engines, request r on
        engine r mod W, per-engine KV quota C/W.  ALT: prefill only if the
        engine's previous micro-batch was not a prefill; PRIO: whenever admissible."""
        W = self.W
        quota = [self.C // W + (1 if e < self.C % W else 0) for e in range(W)]
        used = [0] * W
        q_ev = [[] for _ in range(W)]
        q_fr = [deque() for _ in range(W)]
        for r in self.reqs:
            q_fr[r.rid % W].append(r.rid)
        running = [[] for _ in range(W)]
        last = ["-"] * W
        ekey = {}
        for r in self.reqs:
            if ceil_div(r.L + r.N, self.B) > quota[r.rid % W]:
                raise ValueError("request exceeds its engine's KV quota")

        def issue(e):
            while True:
                pend = list(q_ev[e]) + list(q_fr[e])
                batch = self._form_prefill_batch(pend, self.alloc.free, quota[e] - used[e]) if pend else []
                if self.o.policy == PPSB_ALT:
                    do_p = bool(batch) and (last[e] != "P" or not running[e])
                else:
                    do_p = bool(batch)
                if do_p:
                    for rid in batch:
                        if q_ev[e] and q_ev[e][0] == rid:
                            q_ev[e].pop(0)
                        else:
                            q_fr[e].popleft()
                    self.launch_prefill(batch, slot=e)
                    used[e] += sum(len(self.reqs[i].blocks) for i in batch)
                    running[e].extend(batch)
                    last[e] = "P"
                    return
                if running[e]:
                    # own-quota eviction: most recently admitted running request
                    while running[e]:
                        need = self.decode_need(running[e])
                        if need <= quota[e] - used[e]:
                            break
                        victim = max(running[e], key=lambda i: self.reqs[i].adm)
                        running[e].remove(victim)
                        r = self.reqs[victim]
                        used[e] -= len(r.blocks)
                        old = r.adm
                        self.alloc.release(r.blocks)
                        self.emit("E", victim, *r.blocks)
                        r.blocks = []
                        r.L += r.g
                        r.N -= r.g
                        r.P = max(r.P - r.g, 1)
                        r.g = r.d = 0
                        r.adm = -1
                        self.live.discard(victim)
                        ekey[victim] = old
                        pos = 0
                        while pos < len(q_ev[e]) and ekey[q_ev[e][pos]] < old:
                            pos += 1
                        q_ev[e].insert(pos, victim)
                        self.stats["evicted"] += 1
                    if not running[e]:
                        last[e] = "-"
                        continue
                    for rid in running[e]:
                        r = self.reqs[rid]
                        k = ceil_div(r.L + r.d + 1, self.B) - len(r.blocks)
                        if k > 0:
                            blk = self.alloc.alloc(k)
                            r.blocks.extend(blk)
                            used[e] += k
                            self.emit("A", rid, *blk)
                    mid = self.mb_counter
                    self.mb_counter += 1
                    mem = list(running[e])
                    mb = MicroBatch(mid, "D", mem, [self.reqs[i].L + self.reqs[i].d for i in mem],
                                    [1] * len(mem), e, 0)
                    for rid in mem:
                        self.reqs[rid].in_flight = True
                    self.inflight.append(mb)
                    self.plan.append(mb)
                    self.emit("D", mid, e, len(mem), *mem)
                    last[e] = "D"
                    return
                return   # engine idle

        for e in range(W):
            issue(e)
        while self.inflight:
            mb = self.inflight.popleft()
            e = mb.slot
            self.emit("R", mb.mid, len(mb.members), *mb.members)
            for rid in mb.members:
                r = self.reqs[rid]
                r.in_flight = False
                r.g += 1
                r.n_out += 1
                if mb.kind == "D":
                    r.d += 1
                if r.g == r.N:
                    used[e] -= len(r.blocks)
                    r.done = True
                    self.alloc.release(r.blocks)
                    self.emit("F", rid, *r.blocks)
                    r.blocks = []
                    self.live.discard(rid)
                    running[e].remove(rid)
            issue(e)
        assert all(r.done for r in self.reqs), "baseline stalled"
        return self


    # ------------------------------------------------------------ PP+HB
    def _run_hybrid(self):
        """PP+HB baseline [R23]: "hybrid batching combines requests from both
        the prefill and decode phases into the same batch" with "chunked
        prefill [that] splits the prefill into chunks".
        As the PP+SB baselines: W virtual engines (one micro-batch in flight
        each), request r on engine r mod W, per-engine KV quota C/W.  Each
        micro-batch of engine e = all its decoding requests (one token each,
        admission order) + prefill chunks filling the rest of hb_tokens: first
        the engine's partially prefilled requests, then its pending ones
        (evicted first, then fresh).  A chunk takes min(remaining prompt,
        token budget left, tokens whose blocks fit the quota); the chunk that
        completes a prompt produces the first token and the request decodes
        from the next micro-batch on.  KV overflow of the decode step evicts
        (recompute) the most recently admitted running or prefilling request."""
        W = self.W
        T = max(self.o.hb_tokens, 1)
        quota = [self.C // W + (1 if e < self.C % W else 0) for e in range(W)]
        used = [0] * W
        q_ev = [[] for _ in range(W)]
        q_fr = [deque() for _ in range(W)]
        for r in self.reqs:
            q_fr[r.rid % W].append(r.rid)
        running = [[] for _ in range(W)]    # decoding, admission order
        filling = [[] for _ in range(W)]    # 0 < pf < L, admission order
        ekey = {}
        for r in self.reqs:
            if ceil_div(r.L + r.N, self.B) > quota[r.rid % W]:
                raise ValueError("request exceeds its engine's KV quota")

        def evict(e, victim):
            r = self.reqs[victim]
            used[e] -= len(r.blocks)
            old = r.adm
            self.alloc.release(r.blocks)
            self.emit("E", victim, *r.blocks)
            r.blocks = []
            if victim in running[e]:
                running[e].remove(victim)
            else:
                filling[e].remove(victim)
            r.L += r.g
            r.N -= r.g
            r.P = max(r.P - r.g, 1)
            r.g = r.d = r.pf = 0
            r.adm = -1
            self.live.discard(victim)
            ekey[victim] = old
            pos = 0
            while pos < len(q_ev[e]) and ekey[q_ev[e][pos]] < old:
                pos += 1
            q_ev[e].insert(pos, victim)
            self.stats["evicted"] += 1

        def plan(e):
            dec = list(running[e])
            avail = quota[e] - used[e] - self.decode_need(dec)
            budget = T - len(dec)
            chunks = []          # (rid, q_start, q_len)
            for rid in list(filling[e]) + list(q_ev[e]) + list(q_fr[e]):
                if budget <= 0:
                    break
                r = self.reqs[rid]
                fit = (len(r.blocks) + avail) * self.B - r.pf     # tokens whose blocks fit the quota
                take = min(r.L - r.pf, budget, fit)
                if take <= 0:
                    break
                avail -= ceil_div(r.pf + take, self.B) - len(r.blocks)
                chunks.append((rid, r.pf, take))
                budget -= take
            return dec, chunks

        def issue(e):
            # decode step of the running requests; evict while it does not fit
            while running[e] and self.decode_need(running[e]) > quota[e] - used[e]:
                evict(e, max(running[e] + filling[e], key=lambda i: self.reqs[i].adm))
            dec, chunks = plan(e)
            # partially prefilled prompts alone can exhaust the quota: recompute
            # the most recently admitted one until something fits
            while not dec and not chunks and filling[e]:
                evict(e, max(filling[e], key=lambda i: self.reqs[i].adm))
                dec, chunks = plan(e)
            if not dec and not chunks:
                return           # engine idle
            for rid in dec:
                r = self.reqs[rid]
                k = ceil_div(r.L + r.d + 1, self.B) - len(r.blocks)
                if k > 0:
                    blk = self.alloc.alloc(k)
                    r.blocks.extend(blk)
                    used[e] += k
                    self.emit("A", rid, *blk)
            for rid, q0, ql in chunks:
                r = self.reqs[rid]
                if r.pf == 0 and rid not in filling[e]:     # admission
                    if q_ev[e] and q_ev[e][0] == rid:
                        q_ev[e].pop(0)
                    else:
                        q_fr[e].popleft()
                    r.adm = self.adm_counter
                    self.adm_counter += 1
                    r.g = r.d = 0
                    self.live.add(rid)
                    filling[e].append(rid)
                k = ceil_div(q0 + ql, self.B) - len(r.blocks)
                if k > 0:
                    blk = self.alloc.alloc(k)
                    r.blocks.extend(blk)
                    used[e] += k
                    self.emit("A", rid, *blk)
            mid = self.mb_counter
            self.mb_counter += 1
            mem = dec + [c[0] for c in chunks]
            mb = MicroBatch(mid, "H", mem, [self.reqs[i].L + self.reqs[i].d for i in dec] + [c[1] for c in chunks],
                            [1] * len(dec) + [c[2] for c in chunks], e, 0)
            for rid in mem:
                self.reqs[rid].in_flight = True
            self.inflight.append(mb)
            self.plan.append(mb)
            self.emit("H", mid, e, len(dec), len(chunks), *dec, *["%d:%d:%d" % c for c in chunks])

        for e in range(W):
            issue(e)
        while self.inflight:
            mb = self.inflight.popleft()
            e = mb.slot
            self.emit("R", mb.mid, len(mb.members), *mb.members)
            for rid, q0, ql in zip(mb.members, mb.q_start, mb.q_len):
                r = self.reqs[rid]
                r.in_flight = False
                if rid in running[e]:           # decode token
                    r.g += 1
                    r.n_out += 1
                    r.d += 1
                else:                           # prefill chunk
                    r.pf = q0 + ql
                    if r.pf < r.L:
                        continue
                    filling[e].remove(rid)      # prompt complete: first token
                    running[e].append(rid)
                    r.g += 1
                    r.n_out += 1
                if r.g == r.N:
                    used[e] -= len(r.blocks)
                    r.done = True
                    self.alloc.release(r.blocks)
                    self.emit("F", rid, *r.blocks)
                    r.blocks = []
                    self.live.discard(rid)
                    running[e].remove(rid)
            issue(e)
        assert all(r.done for r in self.reqs), "hybrid baseline stalled"
        return self


def schedule(requests, opts: SchedOptions, tdec=None, tpre=None) -> RefScheduler:
    """Convenience: run the reference scheduler; requests = [(L, P, N), ...]."""
    return RefScheduler(opts, requests, tdec, tpre).run()
