"""TD-Pipe oracle -- TEST INFRASTRUCTURE ONLY.

Plain, slow, obviously-correct CPU implementations of what the hot path
computes, written from the paper (arxiv 2506.10470, /root/reference/PAPER.md)
and SURVEY.md §8(c):

* ``oracle.weights``   -- the counter-based splitmix64 weight recipe (F9),
* ``oracle.forward``   -- fp64 numpy Llama-style forward, one request at a time,
                          contiguous KV (F1-F8; §2.1),
* ``oracle.scheduler`` -- the reference scheduler, step by step (S0-S12;
                          Alg.1, work stealing PAPER.md:409-427,
                          Eq.1-2, recompute PAPER.md:533).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import anything under ``oracle/``.  The product
path (``paper_2506_10470_b200``) never imports it and shares no code with it;
both consume inputs from the separate ``workload`` module only.

Parity status: every function is pinned by ``tests/test_oracle_*.py`` (HF
LlamaForCausalLM, closed forms, paper worked examples, brute force) except the
measured profile table, which is an input -- see DESIGN.md "parity unpinned".
"""
