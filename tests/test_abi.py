"""The C-ABI library loads and exports every symbol include/tdpipe.h declares
(CPU: no compute calls), and argument validation behaves as documented."""
import os
import re

import numpy as np
import pytest

from paper_2506_10470_b200 import TD_EXEC_NULL, TDError, TDPipe, lib
from workload import SHAPES

HDR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "tdpipe.h")


def declared():
    src = open(HDR).read()
    return sorted(set(re.findall(r"^(?:td_status|void|const char\*|int64_t)\s+(td_\w+)\(", src, re.M)))


def test_every_declared_symbol_is_exported():
    names = declared()
    assert len(names) >= 15
    L = lib()
    for n in names:
        assert hasattr(L, n), n


def test_create_validation_errors():
    import ctypes as C
    from paper_2506_10470_b200.tdpipe import default_options, make_shape
    s = SHAPES["tiny"]
    L = lib()
    ctx = C.c_void_p()
    o = default_options(executor=TD_EXEC_NULL)
    # n_stages > n_layers
    assert L.td_create(C.byref(make_shape(s)), 3, C.byref(o), C.byref(ctx)) == -1
    # kv heads must divide heads
    bad = make_shape(s)
    bad.n_kv_heads = 3
    assert L.td_create(C.byref(bad), 1, C.byref(o), C.byref(ctx)) == -1
    assert L.td_create(C.byref(make_shape(s)), 2, C.byref(o), C.byref(ctx)) == 0
    L.td_destroy(ctx)


def test_submit_validation_and_null_run():
    t = TDPipe(SHAPES["tiny"], 2, executor=TD_EXEC_NULL, kv_blocks=8, policy=1)
    with pytest.raises(TDError):
        t.td_submit([1, 2, 3], 4, 600)            # > max_seq_len
    with pytest.raises(TDError):
        t.td_submit([1, 2, 300], 4, 4)            # token id >= vocab
    with pytest.raises(TDError):
        t.td_submit(list(range(100)) + [0] * 100, 4, 100)   # exceeds 8 blocks of 16
    assert t.td_submit([1, 2, 3], 4, 5) == 0
    assert t.td_submit([4] * 20, 0, 3) == 1       # predicted_len < 1 -> 1
    st = t.td_run()
    assert st["generated_tokens"] == 8
    assert len(t.td_get_output(0)) == 5 and len(t.td_get_output(1)) == 3
    t.close()


def test_options_layout_and_handoff_validation():
    """td_options as seen through ctypes matches the C defaults (layout check of
    the trailing multi-process fields) and the hand-off options are validated
    before any device is touched."""
    import ctypes as C
    from paper_2506_10470_b200.tdpipe import TD_HANDOFF_NCCL, TD_HANDOFF_PEER, default_options, make_shape
    o = default_options()
    assert o.block_size == 16 and o.prefill_token_budget == 2048 and o.hb_tokens == 512
    assert o.world_size == 1 and o.handoff == TD_HANDOFF_PEER and not o.allgather and not o.allgather_user
    L = lib()
    ctx = C.c_void_p()
    s = make_shape(SHAPES["tiny"])
    # CUDA executor, 2 ranks, peer hand-off without an allgather callback: TD_EINVAL
    o2 = default_options(world_size=2, rank=0)
    assert L.td_create(C.byref(s), 2, C.byref(o2), C.byref(ctx)) == -1
    # unknown hand-off kind: TD_EINVAL
    o3 = default_options(executor=TD_EXEC_NULL, handoff=7)
    assert L.td_create(C.byref(s), 1, C.byref(o3), C.byref(ctx)) == -1
    o4 = default_options(executor=TD_EXEC_NULL, handoff=TD_HANDOFF_NCCL)
    assert L.td_create(C.byref(s), 1, C.byref(o4), C.byref(ctx)) == 0
    L.td_destroy(ctx)
